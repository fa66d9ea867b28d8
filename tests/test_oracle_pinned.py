"""NEXT-2 baseline pins: PinnedRouting (SPEC.md BaselinePolicy; "sends
all requests from the same agentic workflow to the same node"; reading A45): per-replica
queues instead of the global program-aware queue."""
import random

import oracle
import tracegen
from tests.helpers import base_cfg, flat_trace, set_program


def test_pinned_leaves_a_replica_idle_hand_computed():
    """R = 2, 10 blocks each (bt = 1); paused slots 0, 2, 4 (all pinned to r0, 6 tokens
    each), r1 empty.  Global queue: slot 0 -> r0, slot 2 -> r1 (least loaded), slot 4
    fits nowhere.  Pinned: slot 0 -> r0, slot 2 does not fit r0 -> r0's queue stops; r1
    has no programs of its own and stays idle (Fig. 2a imbalance)."""
    def build(pinned):
        o = oracle.Oracle(base_cfg(n_replicas=2, hbm_blocks=10, pinned_routing=pinned), flat_trace(5))
        for p in (0, 2, 4):
            set_program(o, p, oracle.PAUSED, oracle.PHASE_R, 6, c_kv=0, paused_since=0)
        o.next_arrival = 5
        o.tick = 1
        return o
    g, pn = build(False), build(True)
    _, dg = g.sched_step()
    _, dp = pn.sched_step()
    assert [(d[1], d[3]) for d in dg if d[0] == oracle.D_RESTORE] == [(0, 0), (2, 1)]
    assert [(d[1], d[3]) for d in dp if d[0] == oracle.D_RESTORE] == [(0, 0)]
    assert g.stats["imbalance_last_blocks"] == 0 and pn.stats["imbalance_last_blocks"] == 6


def test_pinned_equals_global_with_one_replica():
    cfg = tracegen.get_config("c1_toy", n_replicas=1, hbm_blocks=80, host_blocks=16,
                              trace=dict(n=24, n_initial=10, seed=77))
    tr = tracegen.make_trace(cfg)
    a, b = oracle.Oracle(cfg, tr), oracle.Oracle(dict(cfg, pinned_routing=True), tr)
    for _ in range(120):
        assert a.sched_step() == b.sched_step()


def test_pinned_random_traces_stay_on_their_replica():
    for seed in range(3):
        cfg = tracegen.get_config("c1_toy", n_replicas=3, hbm_blocks=48, host_blocks=16, pinned_routing=True,
                                  trace=dict(n=24, n_initial=12, seed=400 + seed))
        o = oracle.Oracle(cfg, tracegen.make_trace(cfg))
        rng = random.Random(seed)
        for _ in range(100):
            st, ds = o.sched_step()
            assert st == oracle.OK
            o.check_invariants()
            for p in range(o.N):
                if o.placement[p] >= 0:
                    assert o.placement[p] == p % 3
            if rng.random() < 0.1:
                o.check_watermark()


def test_ttl_pin_table_step_contribution():
    """TTL-pin baseline (reading A47): f(t) = 1 for t < TTL, 0 after: an acting program of
    10 blocks (bt = 1) contributes 10 before its TTL of 3 s and 0 after (vs 10 >> k for
    the paper's 2^-t)."""
    from tracegen.configs import ttl_pin_table
    o = oracle.Oracle(base_cfg(hbm_blocks=100, decay_table=ttl_pin_table(3)), flat_trace(1, d_ms=10 ** 9))
    set_program(o, 0, oracle.ACTING, oracle.PHASE_A, 10, placement=0, home=0, acting_since=0,
                tool_return=10 ** 12, hbm=range(10))
    o.next_arrival = 1
    o.tick = 0
    seen = []
    for _ in range(3):                         # T = 0, 5000, 10000 ms -> k = 0, 5, 10
        o.sched_step()
        seen.append(o.L[0])
    assert seen == [10, 0, 0]
    assert o.contrib_at(0, 2999, 10) == 10 and o.contrib_at(0, 3000, 10) == 0
