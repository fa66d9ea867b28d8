"""Pins for oracle/content.py (KV content closed form)."""
import numpy as np

from oracle.content import GAMMA, block_words, content_word, splitmix64


def test_splitmix64_published_vectors():
    # SplitMix64 reference outputs (Steele/Lea/Flood; Vigna's splitmix64.c):
    # seed 0 -> first output 0xE220A8397B1DCDAF
    assert splitmix64(0) == 0xE220A8397B1DCDAF
    # seed 1234567 -> 6457827717110365317, 3203168211198807973, 9817491932198370423,
    # 4593380528125082431, 16408922859458223821 (the widely reproduced test sequence)
    want = [6457827717110365317, 3203168211198807973, 9817491932198370423,
            4593380528125082431, 16408922859458223821]
    got = [splitmix64((1234567 + i * GAMMA) & ((1 << 64) - 1)) for i in range(5)]
    assert got == want


def test_block_words_matches_scalar_definition():
    L, Hkv, D, bt = 2, 2, 64, 16
    for uid, j in [(1, 0), (7, 3), (123456, 9)]:
        arr = block_words(uid, j, bt, L, Hkv, D)
        assert arr.shape == (L, 2, bt, Hkv, D // 4)
        for (l, kv, s, h, w) in [(0, 0, 0, 0, 0), (1, 1, 15, 1, 15), (1, 0, 7, 0, 3)]:
            assert int(arr[l, kv, s, h, w]) == content_word(uid, j * bt + s, l, kv, h, w, L, Hkv, D)


def test_content_index_is_injective_over_a_program():
    # i is a mixed-radix number: distinct (t, l, kv, h, w) give distinct words' inputs
    L, Hkv, D, bt = 2, 2, 64, 16
    a = np.concatenate([block_words(5, j, bt, L, Hkv, D).ravel() for j in range(4)])
    assert len(np.unique(a)) == a.size
