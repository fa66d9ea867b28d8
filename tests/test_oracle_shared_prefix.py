"""NEXT-3 pins: the agents' shared system prompt stored once per replica (reading A49;
PAPER.md:230 "agentic system prompts are identical across workflows"; "the
shared prompt across programs implicitly reserves sufficient memory buffer").

The first sb = shared_prefix_tokens / bt blocks of every program reference the top sb
HBM blocks of its replica; they are never allocated, evicted, copied or compacted, and
the load (Eq. 7) still counts every program's full context.  Expected values below are
worked out by hand from that rule, or come from the same run without the shared prefix
(the special case the rule must reduce to)."""
import random

import oracle
import tracegen
from tests.helpers import base_cfg, flat_trace, set_program
from tests.test_oracle_invariants import check_i9, stress_cfg

H = oracle.HOST_BIT


def cfg_small(**kw):
    c = base_cfg(block_tokens=16, hbm_blocks=10, host_blocks=4, max_ctx=1024,
                 shared_prefix_tokens=32)
    c.update(kw)
    return c


def homed(o, p, home, private=(), host=()):
    """Program p homed on `home`: shared prefix entries, then private HBM blocks, then
    host slots (set_program would record the shared blocks as owned by p)."""
    set_program(o, p, o.status[p], o.phase[p], o.c[p], placement=o.placement[p], home=home,
                c_kv=o.c_kv[p], paused_since=o.paused_since[p], satisfied=o.satisfied[p],
                hbm=list(range(o.shared_base, o.NB)) + list(private), host=host)
    for j in range(o.sb):                      # restore the reserved blocks' owner tag
        o.owner_hbm[home][o.shared_base + j] = (oracle.ta_oracle.SHARED, j)


def test_arrivals_share_the_prefix_hand_computed():
    """Two 48-token prompts, bt 16, 32 shared tokens (sb 2) on NB 10: the reserved blocks
    are 8, 9; each program allocates one private block (lowest free, slot order): rows
    [8, 9, 0] and [8, 9, 1], free {2..7}.  Without sharing: [0, 1, 2], [3, 4, 5]."""
    tr = flat_trace(2, turns=2, g=10, p0=48)
    o = oracle.Oracle(cfg_small(), tr)
    assert o.sb == 2 and o.shared_base == 8
    assert [o.hbm_free[0][b] for b in range(10)] == [1] * 8 + [0, 0]
    st, out = o.sched_step()
    assert st == oracle.OK
    assert list(o.loc[0][:4]) == [8, 9, 0, oracle.NONE]
    assert list(o.loc[1][:4]) == [8, 9, 1, oracle.NONE]
    assert [o.hbm_free[0][b] for b in range(10)] == [0, 0] + [1] * 6 + [0, 0]
    fetch = [d for d in out if d[0] == oracle.D_FETCH]
    # (kind, pid, src, dst, blocks, to_host, dropped, hit, peer, host, miss, new)
    assert fetch == [(oracle.D_FETCH, 0, -1, 0, 1, 0, 0, 0, 0, 0, 0, 48),
                     (oracle.D_FETCH, 1, -1, 0, 1, 0, 0, 0, 0, 0, 0, 48)]
    assert o.stats["new_blocks"] == 2 and o.stats["fetch_blocks"] == 2
    assert o.stats["fill_tok"] == 2 * 16                     # tokens [32, 48) of each program
    assert [f[5:] for f in o.fills] == [(32, 48), (32, 48)]
    assert o.L == [6]                                         # load counts the full contexts
    o.check_invariants()
    # the same arrivals without sharing
    p = oracle.Oracle(cfg_small(shared_prefix_tokens=0), tr)
    p.sched_step()
    assert list(p.loc[0][:3]) == [0, 1, 2] and list(p.loc[1][:3]) == [3, 4, 5]


def test_eviction_spares_the_prefix_hand_computed():
    """NB 6 (sb 2: blocks 4, 5 reserved).  A PAUSED homed on 0 with rows [4, 5, 0, 1]
    (c 64); B REASONING on 0, fresh, c 80 -> need = 5 - 2 = 3; free {2, 3}; supply =
    2 + (4 - 2) = 4 >= 3; X = 1: A's tail block j=3 (idx 1) goes to host slot 0.  B then
    takes the lowest free blocks 1, 2, 3: row [4, 5, 1, 2, 3]."""
    tr = flat_trace(2, turns=2, g=10, p0=32)
    o = oracle.Oracle(cfg_small(hbm_blocks=6), tr)
    set_program(o, 0, oracle.PAUSED, oracle.PHASE_R, 64)
    homed(o, 0, 0, private=(0, 1))
    set_program(o, 1, oracle.REASONING, oracle.PHASE_R, 80, placement=0, c_kv=0)
    o.tick = 1
    o.check_invariants()
    st, out = o.sched_step()
    assert st == oracle.OK
    assert (oracle.D_EVICT, 0, 0, -1, 1, 1, 0, 0, 0, 0, 0, 0) in out
    assert list(o.loc[0][:4]) == [4, 5, 0, H | 0]
    assert list(o.loc[1][:5]) == [4, 5, 1, 2, 3]
    assert o.moves[0] == (oracle.ta_oracle.MOVE_D2H, 0, 1, 0, 0, 0, 3)
    o.check_invariants()


def test_resume_elsewhere_counts_the_prefix_as_hit_hand_computed():
    """R 2, NB 6 each.  A PAUSED homed on 0, rows [4, 5, 0, H|0], c = c_kv = 64; replica 0
    is loaded by B (c 80, REASONING, resident) so A restores onto replica 1 (least
    loaded).  Resume-time classes: the 32 shared tokens are resident on 1 (hit), block 2
    is on replica 0's HBM (peer 16), block 3 on its host tier (host 16): need 2 = one
    P2P + one H2D into blocks 0, 1 of replica 1."""
    tr = flat_trace(2, turns=2, g=10, p0=32)
    o = oracle.Oracle(cfg_small(n_replicas=2, hbm_blocks=6, lambda_min_q16=65535), tr)
    set_program(o, 0, oracle.PAUSED, oracle.PHASE_R, 64)
    homed(o, 0, 0, private=(0,), host=(0,))
    set_program(o, 1, oracle.REASONING, oracle.PHASE_R, 80, placement=0, satisfied=1)
    homed(o, 1, 0, private=(1, 2, 3))
    o.tick = 1
    o.check_invariants()
    st, out = o.sched_step()
    assert st == oracle.OK
    assert (oracle.D_RESTORE, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0) in out
    assert (oracle.D_FETCH, 0, 0, 1, 2, 0, 0, 32, 16, 16, 0, 0) in out
    assert list(o.loc[0][:4]) == [4, 5, 0, 1] and o.home[0] == 1
    assert o.hbm_free[0][0] == 1 and o.host_free[0][0] == 1   # deferred frees of the sources
    o.check_invariants()


def test_reduces_to_the_unshared_run_when_nothing_is_evicted():
    """With a pool no run ever fills, sharing changes no scheduling decision (the load
    counts full contexts) and every FETCH asks sb fewer blocks of a program that is not
    resident; per replica, used blocks = sb + (unshared used) - sb * (homed programs)."""
    cross = less_peer = 0
    for seed in range(4):
        # watermarks at 3% of the pool: pauses and cross-replica restores, no eviction
        cfg = stress_cfg(seed, R=2, NB=4096, NH=0, n=24, n0=10, compact=0,
                         lambda_max_q16=1966, lambda_min_q16=1966)
        cfg_s = dict(cfg, shared_prefix_tokens=64)
        tr = tracegen.make_trace(cfg)
        a, b = oracle.Oracle(cfg, tr), oracle.Oracle(cfg_s, tr)
        for _ in range(120):
            sa, da = a.sched_step()
            sb_, db = b.sched_step()
            assert sa == sb_ == oracle.OK
            sched = lambda ds: [d for d in ds if d[0] in (oracle.D_PAUSE, oracle.D_RESTORE, oracle.D_STALL)]
            assert sched(da) == sched(db)
            fa = [d for d in da if d[0] == oracle.D_FETCH]
            fb = [d for d in db if d[0] == oracle.D_FETCH]
            # (kind, pid, src, dst, blocks, to_host, dropped, hit, peer, host, miss, new)
            assert [d[:4] + d[9:] for d in fa] == [d[:4] + d[9:] for d in fb]
            for x, y in zip(fa, fb):
                assert y[7] + y[8] == x[7] + x[8]            # the prefix moves from peer to hit
                assert y[4] == (x[4] if x[2] == x[3] else x[4] - b.sb)
            for r in range(2):
                homed_r = sum(1 for p in range(a.N) if a.home[p] == r)
                used_a = a.NB - sum(a.hbm_free[r])
                used_b = b.NB - sum(b.hbm_free[r])
                assert used_b == b.sb + used_a - b.sb * homed_r, (seed, r)
            b.check_invariants()
        assert a.stats["evict_blocks"] == b.stats["evict_blocks"] == 0
        cross += a.stats["p2p_blocks"]
        less_peer += a.stats["peer_tok"] - b.stats["peer_tok"]
    assert cross > 0 and less_peer > 0


def test_random_stress_invariants_with_shared_prefix():
    """Tight pools, host tier, compaction every 3 ticks, 2 replicas: the invariants
    (I1-I10 plus the shared-prefix rules) after every tick; compaction never moves a
    reserved block; content classes add up."""
    for seed in range(6):
        cfg = stress_cfg(100 + seed, compact=3, shared_prefix_tokens=48)
        tr = tracegen.make_trace(cfg)
        o = oracle.Oracle(cfg, tr)
        assert o.sb == 3
        for _ in range(300):
            st, ds = o.sched_step()
            assert st == oracle.OK
            o.check_invariants()
            o.check_watermark()
            check_i9(o)
            M = oracle.ta_oracle
            for kind, sr, si, dr, di, p, j in o.moves:
                assert j >= o.sb, f"a shared-prefix block moved: {(kind, si, di, p, j)}"
                if kind != M.MOVE_H2D:                       # HBM source
                    assert si < o.shared_base
                if kind in (M.MOVE_P2P, M.MOVE_H2D, M.MOVE_D2D):
                    assert di < o.shared_base
            for f in o.fills:
                assert f[4] >= o.sb and f[2] < o.shared_base, f
            for d in ds:
                if d[0] == oracle.D_FETCH:
                    assert d[7] + d[8] + d[9] + d[10] <= o.c[d[1]]
            if all(s in (oracle.STOPPED, oracle.UNARRIVED) for s in o.status) and o.next_arrival == o.N:
                break


def test_verbs_and_failover_keep_the_reserved_blocks():
    """OFFLOAD pauses evict only private blocks; a failed replica drops its programs'
    private blocks (the reserved ones stay reserved) and counts only those as lost."""
    rng = random.Random(7)
    cfg = stress_cfg(200, NB=64, shared_prefix_tokens=32)
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    for k in range(120):
        o.sched_step()
        act = [p for p in range(o.N) if o.status[p] in (oracle.REASONING, oracle.ACTING)]
        if act and k % 5 == 0:
            p = rng.choice(act)
            nh = sum(1 for j in range(o.nb_of(p)) if o.is_hbm(o.loc[p][j]) and j >= o.sb)
            st, out = o.pause(p, oracle.PAUSE_OFFLOAD)
            assert st == oracle.OK
            ev = [d for d in out if d[0] == oracle.D_EVICT]
            assert (ev[0][4] if ev else 0) == (nh if o.home[p] >= 0 else 0)
            assert all(o.loc[p][j] == o.shared_base + j for j in range(o.sb)) or o.home[p] < 0
        if k == 60:
            homed_1 = {p: sum(1 for j, e in enumerate(o.loc[p]) if e != oracle.NONE and j >= o.sb)
                       for p in range(o.N) if o.home[p] == 1}
            st, out = o.set_health(1, False)
            lost = {d[1]: d[4] for d in out if d[0] == oracle.D_EVICT}
            assert lost == {p: n for p, n in homed_1.items() if n}
            assert sum(o.hbm_free[1]) == o.NB - o.sb
        if k == 80:
            o.set_health(1, True)
        o.check_invariants()


def test_api_arrival_shorter_than_the_prefix_is_rejected():
    o = oracle.Oracle(cfg_small(), api_mode=True, n_slots=4)
    ev = [(oracle.E_ARRIVE, 0, 1, 31, 0)]
    assert o.sched_step(0, ev) == (oracle.E_INVAL, [])
    st, _ = o.sched_step(0, [(oracle.E_ARRIVE, 0, 1, 32, 0)])
    assert st == oracle.OK and list(o.loc[0][:2]) == [8, 9]
