"""KV content closed form (SURVEY.md §8(c) "KV content (makes every byte checkable)").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper has no model execution on this path (the engine is out of scope,
SURVEY.md P-37), so the bytes a program's KV blocks must hold are defined by a
closed form: for program ``uid``, token ``t``, layer ``l``, ``kv`` in {0, 1},
head ``h`` and 8-byte word ``w < D*2/8``::

    i    = (((t*L + l)*2 + kv)*Hkv + h)*(D/4) + w
    word = splitmix64((uid << 40) + i)          (little-endian)

``splitmix64`` is the standard SplitMix64 finaliser (Steele, Lea, Flood 2014)
with constants 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB.
"Restorable byte-for-byte" (BASELINE.json north_star, invariant I6) means every
valid token slot of every owned block equals this function.

Pinned by: the published SplitMix64 output sequence (tests/test_oracle_content.py).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def splitmix64(x: int) -> int:
    """One SplitMix64 output for state ``x`` (the state is advanced by GAMMA first)."""
    z = (x + GAMMA) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def content_word(uid: int, t: int, l: int, kv: int, h: int, w: int, L: int, Hkv: int, D: int) -> int:
    i = (((t * L + l) * 2 + kv) * Hkv + h) * (D // 4) + w
    return splitmix64(((uid << 40) + i) & M64)


def _splitmix64_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def block_words(uid: int, j: int, bt: int, L: int, Hkv: int, D: int) -> np.ndarray:
    """Expected 8-byte words of logical block ``j`` of program ``uid``.

    Returned shape ``[L, 2, bt, Hkv, D/4]`` (layer, kv, token slot, head, word),
    i.e. the per-(layer, kv) segments of the layer-major pool
    ``pool[l][kv][block][slot][head][D]`` in order.  Token of slot s is j*bt + s.
    """
    W = D // 4
    t = (j * bt + np.arange(bt, dtype=np.uint64))[None, None, :, None, None]
    l = np.arange(L, dtype=np.uint64)[:, None, None, None, None]
    kv = np.arange(2, dtype=np.uint64)[None, :, None, None, None]
    h = np.arange(Hkv, dtype=np.uint64)[None, None, None, :, None]
    w = np.arange(W, dtype=np.uint64)[None, None, None, None, :]
    with np.errstate(over="ignore"):
        i = (((t * np.uint64(L) + l) * np.uint64(2) + kv) * np.uint64(Hkv) + h) * np.uint64(W) + w
        x = (np.uint64(uid) << np.uint64(40)) + i
    return _splitmix64_np(x)
