"""Invariants I1-I10 on random traces, determinism, no-thrash I8
 and the discrete C_unused bound I9."""
import pytest

import oracle
import tracegen
from oracle import ACTING, PAUSED, REASONING


def stress_cfg(seed, R=2, NB=56, NH=16, n=24, n0=10, compact=3, **kw):
    return tracegen.get_config("c1_toy", n_replicas=R, hbm_blocks=NB, host_blocks=NH,
                               compact_every=compact,
                               trace=dict(n=n, n_initial=n0, seed=seed), **kw)


def run(cfg, ticks=300, check=True):
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    log = []
    for _ in range(ticks):
        st, dec = o.sched_step()
        assert st == oracle.OK
        log.append((dec, list(o.moves)))
        if check:
            o.check_invariants()
            o.check_watermark()
            check_i9(o)
        if all(s in (oracle.STOPPED, oracle.UNARRIVED) for s in o.status) and o.next_arrival == o.N:
            break
    return o, log


def check_i9(o):
    """I9: after step 4 every replica is at/above lambda_min*C, or the queue is
    exhausted, or its head (first non-oversized) fits nowhere."""
    nb = [o.nb_of(p) for p in range(o.N)]
    Q = sorted((p for p in range(o.N) if o.status[p] == PAUSED), key=lambda p: o.restore_key(p, nb[p]))
    maxcap = max(o.cap_max)
    head = next((p for p in Q if o.contrib_at(p, o.last_T, nb[p]) <= maxcap), None)
    if head is None:
        return
    cr = o.contrib_at(head, o.last_T, nb[head])
    for r in range(o.R):
        assert not (o.L[r] < o.cap_min[r] and o.L[r] + cr <= o.cap_max[r]), "I9"


@pytest.mark.parametrize("seed,R", [(11, 1), (12, 2), (13, 3), (14, 2)])
def test_invariants_random_traces(seed, R):
    o, log = run(stress_cfg(seed, R=R, NB=56 if R > 1 else 80))
    kinds = {d[0] for dec, _ in log for d in dec}
    assert oracle.D_RESTORE in kinds


def test_all_paths_exercised():
    o, _ = run(stress_cfg(12, R=2))
    s = o.stats
    for k in ("pauses", "evict_to_host", "evict_dropped", "p2p_blocks", "h2d_blocks",
              "recompute_blocks", "compact_blocks", "hit_tok", "peer_tok", "host_tok", "miss_tok"):
        assert s[k] > 0, k


def test_determinism():
    cfg = stress_cfg(21, R=3)
    _, a = run(cfg, check=False)
    _, b = run(cfg, check=False)
    assert a == b


def test_conservation_i7():
    """I7: c = P0 + sum(decoded) + sum(tool results); finished programs
    reach exactly the trace's final context."""
    cfg = stress_cfg(31, R=2, NB=80)
    o, _ = run(cfg, ticks=400, check=False)
    tr = o.trace
    fin = tr.final_ctx()
    done = [p for p in range(o.N) if o.status[p] == oracle.STOPPED]
    assert done
    # a STOPPED program's last c is kept: the whole script was consumed
    for p in done:
        assert o.c[p] == fin[p]


def test_no_thrash_i8():
    """With f == 1, lambda = 1 and R = 1, an ACTING program that is not paused
    during its tool call never loses a block: its resume is a 100% hbm hit."""
    cfg = stress_cfg(41, R=1, NB=80, NH=16, decay_x=1, compact=0)
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    tainted = set()
    acting_prev = set()
    checked = 0
    for _ in range(400):
        st, dec = o.sched_step()
        for d in dec:
            if d[0] == oracle.D_PAUSE:
                tainted.add(d[1])
            if d[0] == oracle.D_EVICT:
                # only paused programs may lose blocks
                assert o.status[d[1]] == PAUSED or d[1] in tainted
            if d[0] == oracle.D_FETCH and d[1] in acting_prev and d[1] not in tainted:
                assert d[8] == d[9] == d[10] == 0, d
                checked += 1
        acting_prev = {p for p in range(o.N) if o.status[p] == ACTING}
        for p in range(o.N):
            if o.status[p] == REASONING and p in tainted and p not in acting_prev:
                tainted.discard(p)
        if o.next_arrival == o.N and all(s == oracle.STOPPED for s in o.status):
            break
    assert checked > 0
