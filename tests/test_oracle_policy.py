"""Pins for oracle steps 2-4 (effective load, pause pass, restore pass).

Each test states what fixes the expected value: a SPEC.md worked example
(bt = 1 makes blocks = tokens, reading A4), a closed form from PAPER.md, or
exhaustive enumeration.  None re-derives the value through the oracle's own code.
"""
import itertools
import random

import pytest

import oracle
from oracle import ACTING, PAUSED, PHASE_A, PHASE_R, REASONING
from tests.helpers import base_cfg, set_program


def decide(o, T=0, k=0):
    o._step1_footprint()
    o._step2_load(T)
    pauses, restores = [], []
    o._step3_pause(k, pauses)
    o._step4_restore(restores)
    return [d[1] for d in pauses], [(d[1], d[3]) for d in restores]


# ---------------------------------------------------------------- P1: decay table
def test_decay_table_closed_form_x2():
    F = oracle.decay_table(2)
    assert F[0] == 1 << 32                       # f(0) = 1, Hypothesis 2
    for k in range(64):                          # f(t) = 2^-t
        assert F[k] == (2 ** (32 - k) if k <= 32 else 0)


def test_decay_semigroup_exact_for_x2():
    # f(a+b) = f(a) f(b): the semigroup equation of Theorem E.1
    F = oracle.decay_table(2)
    for a in range(33):
        for b in range(33 - a):
            assert F[a + b] == (F[a] * F[b]) >> 32


def test_decay_contribution_spec_example():
    # SPEC.md:221 "Acting c=1024, Geometric(2), t=10 -> contribution 1.0 token"
    o = oracle.Oracle(base_cfg(), n_slots=1)
    set_program(o, 0, ACTING, PHASE_A, 1024, placement=0, acting_since=0)
    assert o.contrib_at(0, 10_000, 1024) == 1
    assert o.contrib_at(0, 0, 1024) == 1024       # f(0) = 1


def test_effective_load_spec_example():
    # Reasoning c=100 + Acting c=200 with f = 0.5 -> 200  (Eq. 7)
    o = oracle.Oracle(base_cfg(), n_slots=2)
    set_program(o, 0, REASONING, PHASE_R, 100, placement=0)
    set_program(o, 1, ACTING, PHASE_A, 200, placement=0, acting_since=4000)
    o._step1_footprint()
    o._step2_load(5000)
    assert o.L == [200]


def test_eq7_reduces_to_eq6_without_decay():
    # SPEC.md:220 / pin P4: f == 1 (x = 1) gives the plain thrashing check sum(c) (Eq. 6)
    o = oracle.Oracle(base_cfg(decay_x=1), n_slots=3)
    set_program(o, 0, REASONING, PHASE_R, 100, placement=0)
    set_program(o, 1, ACTING, PHASE_A, 200, placement=0, acting_since=0)
    set_program(o, 2, ACTING, PHASE_A, 50, placement=0, acting_since=-10**9)
    o._step1_footprint()
    o._step2_load(10**6)
    assert o.L == [350]


@pytest.mark.parametrize("cap,load,lam_q16,want", [
    (1000, 900, 65536, 0), (1000, 1300, 65536, 300),
    # lambda = 0.9: Q16 58983 is the nearest value that gives floor(0.9*1000) = 900 exactly
    (1000, 950, 58983, 50)])
def test_delta_c_spec_examples(cap, load, lam_q16, want):
    # Delta C = sum c - lambda_max * C_total
    o = oracle.Oracle(base_cfg(hbm_blocks=cap, lambda_max_q16=lam_q16), n_slots=1)
    set_program(o, 0, REASONING, PHASE_R, load, placement=0)
    o._step1_footprint()
    o._step2_load(0)
    assert max(0, o.L[0] - o.cap_max[0]) == want


# ---------------------------------------------------------------- P3: pause pass
def test_select_evictions_3_5_8():
    # c = {3,5,8} all Acting, Delta C = 7 -> {3,5} (sum c^2 = 34 < 64)
    o = oracle.Oracle(base_cfg(hbm_blocks=16 - 7), n_slots=3)
    for p, c in enumerate([8, 3, 5]):
        set_program(o, p, ACTING, PHASE_A, c, placement=0, acting_since=0)
    paused, _ = decide(o)
    assert sorted(o.c[p] for p in paused) == [3, 5]


def test_select_evictions_tier_dominates():
    # Acting {9}, Reasoning {2,2}, Delta C = 4 -> {9}
    o = oracle.Oracle(base_cfg(hbm_blocks=13 - 4), n_slots=3)
    set_program(o, 0, REASONING, PHASE_R, 2, placement=0)
    set_program(o, 1, REASONING, PHASE_R, 2, placement=0)
    set_program(o, 2, ACTING, PHASE_A, 9, placement=0, acting_since=0)
    paused, _ = decide(o)
    assert paused == [2]


def test_tick_over_by_300():
    # backend over by 300 with Acting {100,250,400} -> Pause {100,250}
    o = oracle.Oracle(base_cfg(hbm_blocks=750 - 300), n_slots=3)
    for p, c in enumerate([400, 100, 250]):
        set_program(o, p, ACTING, PHASE_A, c, placement=0, acting_since=0)
    paused, _ = decide(o)
    assert sorted(o.c[p] for p in paused) == [100, 250]


def test_balanced_cluster_noop():
    # balanced cluster under watermark -> no decisions
    o = oracle.Oracle(base_cfg(n_replicas=2, hbm_blocks=100), n_slots=2)
    set_program(o, 0, REASONING, PHASE_R, 60, placement=0)
    set_program(o, 1, ACTING, PHASE_A, 70, placement=1, acting_since=0)
    assert decide(o) == ([], [])


# ---------------------------------------------------------------- P3: restore pass
def test_restore_reasoning_before_acting():
    # Paused Reasoning c=100 and Acting c=50: Reasoning restored first
    o = oracle.Oracle(base_cfg(hbm_blocks=100), n_slots=2)
    set_program(o, 0, PAUSED, PHASE_A, 50, acting_since=0)
    set_program(o, 1, PAUSED, PHASE_R, 100)
    _, restored = decide(o)
    assert restored == [(1, 0)]


def test_restore_all_to_empty_backend():
    # A full, B empty, 3 queued -> all 3 restored to B in the same tick
    o = oracle.Oracle(base_cfg(n_replicas=2, hbm_blocks=100), n_slots=4)
    set_program(o, 0, REASONING, PHASE_R, 100, placement=0)
    for p, c in [(1, 30), (2, 10), (3, 20)]:
        set_program(o, p, PAUSED, PHASE_R, c)
    _, restored = decide(o)
    assert sorted(restored) == [(1, 1), (2, 1), (3, 1)]
    assert [p for p, _ in restored] == [2, 3, 1]          # shortest first


@pytest.mark.parametrize("c,ok", [(400, True), (700, False)])
def test_resume_capacity(c, ok):
    # Paused c onto a backend with load 400, C = 1000, lambda_max = 1
    o = oracle.Oracle(base_cfg(hbm_blocks=1000), n_slots=2)
    set_program(o, 0, REASONING, PHASE_R, 400, placement=0, home=0, satisfied=1,
                hbm=range(400))
    set_program(o, 1, PAUSED, PHASE_R, c)
    o.L = [400]
    st, dec = o.resume(1, 0)
    assert (st == oracle.OK) == ok
    if ok:
        assert dec[0][0] == oracle.D_RESTORE and o.status[1] == REASONING
        o.check_invariants()
    else:
        assert st == oracle.E_CAPACITY and o.status[1] == PAUSED


# ---------------------------------------------------------------- P2: Definition 1 brute force
def _greedy_exact_instance(rng):
    n = rng.randint(1, 12)
    cs = [rng.randint(1, 30) for _ in range(n)]
    m = rng.randint(1, n)
    dC = sum(sorted(cs)[:m])
    return cs, dC


def test_pause_selection_optimal_in_exact_cover_regime():
    """Definition 1: min sum c_i^2 s.t. sum c_i >= Delta C.
    Greedy shortest-first is optimal when its prefix covers Delta C exactly
    (SPEC.md:270, 584).  Checked by exhaustive enumeration."""
    rng = random.Random(7)
    for _ in range(500):
        cs, dC = _greedy_exact_instance(rng)
        o = oracle.Oracle(base_cfg(hbm_blocks=sum(cs) - dC), n_slots=len(cs))
        for p, c in enumerate(cs):
            set_program(o, p, ACTING, PHASE_A, c, placement=0, acting_since=-rng.randint(0, 900))
        paused, _ = decide(o)
        got = sum(o.c[p] ** 2 for p in paused)
        assert sum(o.c[p] for p in paused) >= dC
        best = min(sum(x * x for x in S) for r in range(len(cs) + 1)
                   for S in itertools.combinations(cs, r) if sum(S) >= dC)
        assert got == best, (cs, dC, paused)
        # same-cardinality statement (second regime)
        m = len(paused)
        assert got == min(sum(x * x for x in S) for S in itertools.combinations(cs, m))


# ---------------------------------------------------------------- P9: Fig. 3 scenario
def test_fig3_scenario():
    """Backend #1 thrashes, Backend #3 is underused: the global queue
    pauses acting Program #2 and restores reasoning #6 and #9 onto Backend #3."""
    o = oracle.Oracle(base_cfg(n_replicas=3, hbm_blocks=10), n_slots=10)
    set_program(o, 2, ACTING, PHASE_A, 3, placement=0, acting_since=0)
    set_program(o, 0, REASONING, PHASE_R, 5, placement=0)
    set_program(o, 1, REASONING, PHASE_R, 4, placement=0)       # r0 load 12 > 10
    set_program(o, 3, REASONING, PHASE_R, 10, placement=1)      # r1 full
    set_program(o, 6, PAUSED, PHASE_R, 4)
    set_program(o, 9, PAUSED, PHASE_R, 5)
    paused, restored = decide(o)
    assert paused == [2]
    assert (6, 2) in restored and (9, 2) in restored
    assert o.L[2] == 9 and o.L[0] <= 10
