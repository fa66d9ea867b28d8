"""Trace presets (SURVEY.md §8(d) table "Trace presets").

A trace is a script per program *slot*: prompt tokens ``p0``, and for each turn
``t < T``: tokens generated ``g[t]``, tool latency ``d_ms[t]`` and tool-result
tokens ``o[t]`` (the last turn has no tool call, so ``d_ms[T-1] = o[T-1] = 0``).
This is the reason/act step structure of PAPER.md:160-162.

Draws use numpy PCG64 (``default_rng(seed)``).  ``ln(m, s)`` means
``m * exp(s * Z)`` with Z standard normal, clipped to ``[lo, hi]`` and rounded.
Traces are truncated so that the final context never exceeds ``max_ctx``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# kind: ('U', lo, hi) uniform integer in [lo, hi]; ('LN', m, s, lo, hi); ('C', v)
PRESETS = {
    # SWE-Agent / mini-SWE-agent: predictable local tools, 1-30 s (BASELINE.json configs[1])
    "swe": dict(p0=("U", 2000, 5000), turns=("LN", 20, 0.5, 4, 80),
                gen=("LN", 250, 0.6, 16, 2048), tool_ms=("LN", 3000, 0.8, 1000, 30000),
                out=("LN", 300, 1.0, 8, 4096)),
    # OpenHands: heavier prompts, longer episodes
    "openhands": dict(p0=("U", 5000, 9000), turns=("LN", 25, 0.5, 5, 100),
                      gen=("LN", 300, 0.6, 16, 2048), tool_ms=("LN", 4000, 1.0, 500, 60000),
                      out=("LN", 400, 1.0, 8, 4096)),
    # ToolOrchestra: heavy-tailed remote tools
    "toolorch": dict(p0=("U", 1000, 3000), turns=("U", 3, 12),
                     gen=("LN", 400, 0.6, 16, 2048), tool_ms=("LN", 2000, 1.7, 100, 300000),
                     out=("LN", 800, 1.0, 8, 4096)),
    # toy (BASELINE.json configs[0]): 4 turns, tiny contexts
    "toy": dict(p0=("U", 64, 256), turns=("C", 4), gen=("U", 16, 128),
                tool_ms=("U", 1000, 12000), out=("U", 16, 160)),
}


@dataclass
class Trace:
    """Struct-of-arrays trace.  ``turn_off`` is a CSR offset array (n_slots+1)."""
    uid: np.ndarray        # u32 [n_slots]  program identity used by the KV content function
    p0: np.ndarray         # u32 [n_slots]  prompt tokens
    turn_off: np.ndarray   # u32 [n_slots+1]
    g: np.ndarray          # u32 [total_turns] tokens generated in the turn
    d_ms: np.ndarray       # u32 [total_turns] tool latency after the turn (0 on last turn)
    o: np.ndarray          # u32 [total_turns] tool-result tokens (0 on last turn)
    n_initial: int         # slots [0, n_initial) arrive at tick 0 (closed loop afterwards)
    preset: list           # preset name per slot (metadata only)

    @property
    def n_slots(self) -> int:
        return int(self.p0.shape[0])

    @property
    def total_turns(self) -> int:
        return int(self.turn_off[-1])

    def turns(self, p: int) -> int:
        return int(self.turn_off[p + 1] - self.turn_off[p])

    def final_ctx(self) -> np.ndarray:
        s = np.add.reduceat(self.g.astype(np.int64) + self.o.astype(np.int64),
                            self.turn_off[:-1].astype(np.int64))
        return self.p0.astype(np.int64) + s


def _draw(rng: np.random.Generator, spec, n: int) -> np.ndarray:
    kind = spec[0]
    if kind == "U":
        return rng.integers(spec[1], spec[2] + 1, size=n, dtype=np.int64)
    if kind == "C":
        return np.full(n, spec[1], dtype=np.int64)
    if kind == "LN":
        _, m, s, lo, hi = spec
        z = rng.standard_normal(n)
        v = np.rint(m * np.exp(s * z))
        return np.clip(v, lo, hi).astype(np.int64)
    raise ValueError(kind)


def gen_trace(mix, n: int, seed: int, max_ctx: int, n_initial: int | None = None) -> Trace:
    """Generate ``n`` program slots.  ``mix`` is a list of preset names; slot ``p``
    uses ``mix[p % len(mix)]`` (equal mixes, e.g. 50% swe / 50% openhands)."""
    if isinstance(mix, str):
        mix = [mix]
    rng = np.random.default_rng(seed)
    names = [mix[p % len(mix)] for p in range(n)]
    p0 = np.zeros(n, np.int64)
    T = np.zeros(n, np.int64)
    per_prog = [None] * n
    for name in mix:
        idx = np.array([p for p in range(n) if names[p] == name], dtype=np.int64)
        if idx.size == 0:
            continue
        sp = PRESETS[name]
        p0[idx] = _draw(rng, sp["p0"], idx.size)
        T[idx] = _draw(rng, sp["turns"], idx.size)
        tot = int(T[idx].sum())
        g = _draw(rng, sp["gen"], tot)
        d = _draw(rng, sp["tool_ms"], tot)
        o = _draw(rng, sp["out"], tot)
        off = 0
        for p in idx:
            t = int(T[p])
            per_prog[p] = (g[off:off + t].copy(), d[off:off + t].copy(), o[off:off + t].copy())
            off += t
    gs, ds, os_, offs = [], [], [], [0]
    for p in range(n):
        g, d, o = per_prog[p]
        # truncate so the context never exceeds max_ctx: keep turn t while
        # p0 + sum_{i<=t} g_i + sum_{i<t} o_i <= max_ctx
        ctx = int(p0[p])
        keep = 0
        for t in range(len(g)):
            need = ctx + int(g[t])
            if need > max_ctx:
                if t == 0:
                    g[0] = max(0, max_ctx - ctx)
                    keep = 1
                break
            keep = t + 1
            ctx = need + int(o[t])
            if ctx > max_ctx:
                break
        g, d, o = g[:keep].copy(), d[:keep].copy(), o[:keep].copy()
        d[-1] = 0
        o[-1] = 0
        gs.append(g); ds.append(d); os_.append(o)
        offs.append(offs[-1] + keep)
    return Trace(
        uid=np.arange(1, n + 1, dtype=np.uint32),
        p0=p0.astype(np.uint32),
        turn_off=np.array(offs, dtype=np.uint32),
        g=np.concatenate(gs).astype(np.uint32),
        d_ms=np.concatenate(ds).astype(np.uint32),
        o=np.concatenate(os_).astype(np.uint32),
        n_initial=n if n_initial is None else int(n_initial),
        preset=names,
    )


def tile_trace(tr: Trace, k: int) -> Trace:
    """k interleaved copies of a trace (slot p*k + c is copy c of slot p, uid = slot + 1):
    the weak-scaling workload for k replicas, where each replica sees the 1-replica
    workload (copies of a program are adjacent, so restores alternate between replicas)."""
    if k == 1:
        return tr
    n = tr.n_slots
    src = np.repeat(np.arange(n), k)                     # slot s -> source slot s // k
    lens = (tr.turn_off[1:] - tr.turn_off[:-1]).astype(np.int64)[src]
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
    take = np.concatenate([np.arange(tr.turn_off[p], tr.turn_off[p + 1]) for p in src]).astype(np.int64)
    return Trace(uid=np.arange(1, n * k + 1, dtype=np.uint32), p0=tr.p0[src].copy(), turn_off=offs,
                 g=tr.g[take].copy(), d_ms=tr.d_ms[take].copy(), o=tr.o[take].copy(),
                 n_initial=tr.n_initial * k, preset=[tr.preset[p] for p in src])
