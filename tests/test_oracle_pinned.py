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


def test_request_aware_orders_hand_computed():
    """RequestAware baseline (reading A46): a stateless request-level engine.  Over
    capacity it preempts the latest running program (not the shortest or the acting
    one); acting programs hold no request (load 0); the waiting queue is FCFS; idle
    caches are evicted least-recently-used first, whatever their size or phase."""
    # over capacity: REASONING slots 0 (12 blocks) and 2 (10 blocks) on 20 blocks -> the
    # latest program (slot 2) is preempted
    cfg = base_cfg(hbm_blocks=20, request_aware=True)
    o = oracle.Oracle(cfg, flat_trace(5, g=1000, d_ms=10 ** 9))
    set_program(o, 0, oracle.REASONING, oracle.PHASE_R, 12, placement=0, home=0, satisfied=1, hbm=range(12))
    set_program(o, 2, oracle.REASONING, oracle.PHASE_R, 10, placement=0, home=0, satisfied=1, hbm=())
    o.next_arrival = 5
    o.tick = 3
    st, ds = o.sched_step()
    assert [d[1] for d in ds if d[0] == oracle.D_PAUSE] == [2]
    # an acting program weighs nothing: 12 + 6 blocks resident, load 12, nothing paused
    o2 = oracle.Oracle(base_cfg(hbm_blocks=20, request_aware=True), flat_trace(5, g=1000, d_ms=10 ** 9))
    set_program(o2, 0, oracle.REASONING, oracle.PHASE_R, 12, placement=0, home=0, satisfied=1, hbm=range(12))
    set_program(o2, 1, oracle.ACTING, oracle.PHASE_A, 6, placement=0, home=0, acting_since=14000,
                tool_return=10 ** 12, hbm=range(12, 18))
    o2.next_arrival = 5
    o2.tick = 3
    o2.sched_step()
    assert o2.L[0] == 12 and o2.status[1] == oracle.ACTING
    # FCFS queue: slot 4 (paused at tick 0, 9 blocks) before slot 3 (tick 1, 2 blocks);
    # the 2-block program then no longer fits 10 blocks and the queue stops
    o3 = oracle.Oracle(base_cfg(hbm_blocks=10, request_aware=True), flat_trace(5, g=1000, d_ms=10 ** 9))
    set_program(o3, 3, oracle.PAUSED, oracle.PHASE_R, 2, c_kv=0, paused_since=1)
    set_program(o3, 4, oracle.PAUSED, oracle.PHASE_R, 9, c_kv=0, paused_since=0)
    o3.next_arrival = 5
    o3.tick = 3
    _, ds = o3.sched_step()
    assert [d[1] for d in ds if d[0] == oracle.D_RESTORE] == [4]
    # LRU eviction: two idle caches on r0, the older one goes first regardless of size
    o4 = oracle.Oracle(base_cfg(hbm_blocks=10, request_aware=True), flat_trace(5, g=1000, d_ms=10 ** 9))
    set_program(o4, 0, oracle.ACTING, oracle.PHASE_A, 3, placement=0, home=0, acting_since=9000,
                tool_return=10 ** 12, hbm=range(0, 3))
    set_program(o4, 1, oracle.ACTING, oracle.PHASE_A, 5, placement=0, home=0, acting_since=4000,
                tool_return=10 ** 12, hbm=range(3, 8))
    set_program(o4, 2, oracle.PAUSED, oracle.PHASE_R, 4, c_kv=0, paused_since=0)
    o4.next_arrival = 5
    o4.tick = 2
    _, ds = o4.sched_step()
    ev = [(d[1], d[4]) for d in ds if d[0] == oracle.D_EVICT]
    assert ev == [(1, 2)]                      # need 4, 2 free: evict 2 blocks of the older cache (slot 1)
