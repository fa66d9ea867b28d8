"""NEXT-4 pins: backend health mask with force-pause failover (PAPER.md:699
BackendState.healthy; SPEC.md:499-506 poll_backends: "unhealthy backends flagged,
their programs force-Paused back to the global queue"; readings A37-A39)."""
import random

import oracle
import tracegen
from tests.helpers import flat_trace, set_program
from tests.test_oracle_golden import load_w1


def dec(kind, pid, src=-1, dst=-1, blocks=0, to_host=0, dropped=0):
    """A decision record in ta_decision field order (kind, pid, src, dst, blocks, to_host,
    dropped, hit, peer, host, miss, new), written out here, not by the oracle."""
    return (kind, pid, src, dst, blocks, to_host, dropped, 0, 0, 0, 0, 0)


def test_w1_replica1_fails_hand_computed():
    """W1 state before tick 2 (tests/golden/w1.json): replica 1 fails.  By hand:
    p3 is REASONING on r1 -> PAUSE p3 @1; programs homed on r1: p3 (5 HBM blocks) and
    p5 (2 HBM + 4 host blocks) -> EVICT p3 (5 dropped), EVICT p5 (6 dropped)."""
    _, o = load_w1()
    st, out = o.set_health(1, False)
    assert st == oracle.OK
    assert out == [dec(oracle.D_PAUSE, 3, src=1),
                   dec(oracle.D_EVICT, 3, src=1, blocks=5, dropped=5),
                   dec(oracle.D_EVICT, 5, src=1, blocks=6, dropped=6)]
    assert all(o.hbm_free[1]) and all(o.host_free[1])
    assert o.home[3] == o.home[5] == -1 and o.status[3] == oracle.PAUSED
    assert o.cap_max[1] == o.cap_min[1] == 0
    # idempotent
    assert o.set_health(1, False) == (oracle.OK, [])
    o.check_invariants()
    # the next ticks never place anything on r1; p4 (host tier of r0) restores onto r0 only if it fits
    for _ in range(6):
        st, ds = o.sched_step()
        assert st == oracle.OK
        assert all(o.placement[p] != 1 for p in range(o.N))
        assert all(d[3] != 1 for d in ds if d[0] in (oracle.D_RESTORE, oracle.D_FETCH))
        o.check_invariants()


def test_failover_pauses_everything_on_the_replica_spec_506():
    """one backend marked unhealthy -> its programs appear Paused in the
    next queue snapshot; the other backends keep theirs."""
    cfg = dict(n_replicas=3, block_tokens=1, hbm_blocks=100, host_blocks=20, max_ctx=4096,
               delta_t_ms=5000, decay_x=2, decay_unit_ms=1000, decode_tok_per_s=0,
               lambda_max_q16=65536, lambda_min_q16=65536, compact_every=0, layout=0, kv="mini")
    o = oracle.Oracle(cfg, flat_trace(6))
    nxt = {0: 0, 1: 0, 2: 0}
    for p, r in enumerate([0, 1, 2, 1, 0, 1]):
        set_program(o, p, oracle.REASONING, oracle.PHASE_R, 10, placement=r, home=r, satisfied=1,
                    hbm=range(nxt[r], nxt[r] + 10))
        nxt[r] += 10
    o.next_arrival = 6
    st, out = o.set_health(1, False)
    assert st == oracle.OK
    assert [d[1] for d in out if d[0] == oracle.D_PAUSE] == [1, 3, 5]
    assert [(d[1], d[6]) for d in out if d[0] == oracle.D_EVICT] == [(1, 10), (3, 10), (5, 10)]
    assert [o.status[p] for p in range(6)] == [oracle.REASONING, oracle.PAUSED, oracle.REASONING,
                                               oracle.PAUSED, oracle.REASONING, oracle.PAUSED]
    # next tick: the three paused programs restore onto the healthy replicas and recompute
    st, ds = o.sched_step()
    restored = {d[1]: d[3] for d in ds if d[0] == oracle.D_RESTORE}
    assert set(restored) == {1, 3, 5} and set(restored.values()) <= {0, 2}
    miss = sum(d[10] for d in ds if d[0] == oracle.D_FETCH)
    assert miss == 30                      # every lost token is recomputed (history = 10 each)
    # back to healthy: capacity restored, replica empty, programs placed there again later
    assert o.set_health(1, True) == (oracle.OK, [])
    assert o.cap_max[1] == 100 and o.L[1] == 0
    o.check_invariants()


def test_failover_random_traces_invariants_and_conservation():
    """Random failures / recoveries on stress traces: invariants I1-I10 every tick, the
    failed replica holds nothing while down, and lost blocks == blocks it held."""
    for seed in range(4):
        cfg = tracegen.get_config("c1_toy", n_replicas=3, hbm_blocks=48, host_blocks=16,
                                  trace=dict(n=20, n_initial=10, seed=300 + seed))
        tr = tracegen.make_trace(cfg)
        o = oracle.Oracle(cfg, tr)
        rng = random.Random(seed)
        down = set()
        for k in range(60):
            if rng.random() < 0.15:
                r = rng.randrange(3)
                if r in down:
                    st, out = o.set_health(r, True)
                    down.discard(r)
                    assert out == []
                elif len(down) < 2:
                    held = sum(1 for p in range(o.N) if o.home[p] == r for e in o.loc[p] if e != oracle.NONE)
                    st, out = o.set_health(r, False)
                    down.add(r)
                    assert sum(d[6] for d in out if d[0] == oracle.D_EVICT) == held
                assert st == oracle.OK
                o.check_invariants()
            st, _ = o.sched_step()
            assert st == oracle.OK
            o.check_invariants()
            for r in down:
                assert not any(o.placement[p] == r or o.home[p] == r for p in range(o.N))
                assert all(o.hbm_free[r]) and all(o.host_free[r])


def test_verbs_reject_unhealthy_targets():
    _, o = load_w1()
    o.set_health(0, False)
    st, _ = o.resume(4, 0)                 # p4 PAUSED: explicit unhealthy target
    assert st == oracle.E_CAPACITY
    assert o.set_health(5, False)[0] == oracle.E_INVAL
