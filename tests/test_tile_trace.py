"""The weak-scaling workload of bench.py at N GPUs (tracegen.tile_trace: N interleaved
copies of the 1-replica trace on N replicas) does exactly N times the 1-replica work:
every counter of the oracle run is N times the 1-replica run's, tick by tick."""
import pytest

import oracle
import tracegen

KEYS = ("pauses", "restores", "evict_blocks", "evict_to_host", "fetch_blocks", "h2d_blocks",
        "recompute_blocks", "new_blocks", "stops", "arrivals", "hit_tok", "miss_tok", "new_tok",
        "cost_decode", "cost_recompute", "overshoot_blocks")


@pytest.mark.parametrize("k", [2, 3])
def test_tiled_trace_is_k_copies_of_the_work(k):
    base = dict(hbm_blocks=48, host_blocks=12, compact_every=0, trace=dict(n=12, n_initial=6, seed=5))
    c1 = tracegen.get_config("c1_toy", n_replicas=1, **base)
    ck = tracegen.get_config("c1_toy", n_replicas=k, **base)
    ck["trace"]["tile"] = k
    t1, tk = tracegen.make_trace(c1), tracegen.make_trace(ck)
    assert tk.n_slots == k * t1.n_slots and tk.n_initial == k * t1.n_initial
    assert len(set(tk.uid.tolist())) == tk.n_slots
    o1, ok = oracle.Oracle(c1, t1), oracle.Oracle(ck, tk)
    for _ in range(200):
        o1.sched_step()
        ok.sched_step()
        for key in KEYS:
            assert ok.stats[key] == k * o1.stats[key], key
        used1 = o1.NB - sum(o1.hbm_free[0])
        assert all(ok.NB - sum(ok.hbm_free[r]) == used1 for r in range(k))
    assert o1.stats["evict_blocks"] > 0 and o1.stats["stops"] > 0
