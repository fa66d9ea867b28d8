"""NEXT-4 (first half) pins: the per-decode-step guard (reading A50; PAPER.md:360-361
"the context length c_p of agentic workflows grows rapidly, which can trigger memory
thrashing mid-execution even without new arrivals"; PAPER.md:544 Delta t ablation;
SURVEY.md 8(f) "Delta t -> one decode step").

The guard is the periodic monitor run with Delta t = one decode step; what it bounds is
the excess L_eff - lambda_max*C the pause pass finds (`overshoot_blocks`, summed over
replica-ticks, and `overshoot_max_blocks`)."""
import oracle
import tracegen
from oracle import ACTING, PHASE_A
from tests.helpers import base_cfg, set_program
from tests.test_oracle_invariants import stress_cfg


def test_overshoot_spec_tick_over_by_300():
    """a backend over by 300 (Acting {400, 100, 250}, capacity 450): the
    monitor finds an excess of 300."""
    o = oracle.Oracle(base_cfg(hbm_blocks=450), n_slots=3)
    for p, c in enumerate([400, 100, 250]):
        set_program(o, p, ACTING, PHASE_A, c, placement=0, acting_since=0)
    o._step1_footprint()
    o._step2_load(0)
    o._step3_pause(0, [])
    assert o.stats["overshoot_blocks"] == 300 and o.stats["overshoot_max_blocks"] == 300


def test_overshoot_sums_replicas_and_keeps_the_max():
    """Two replicas of 100 blocks over by 5 and 7 (fresh acting programs, f(0) = 1):
    sum 12, max 7; a replica under its watermark adds nothing."""
    o = oracle.Oracle(base_cfg(n_replicas=3, hbm_blocks=100), n_slots=3)
    for p, c in enumerate([105, 107, 90]):
        set_program(o, p, ACTING, PHASE_A, c, placement=p, acting_since=0)
    o._step1_footprint()
    o._step2_load(0)
    o._step3_pause(0, [])
    assert o.stats["overshoot_blocks"] == 12 and o.stats["overshoot_max_blocks"] == 7


def check_growth_bound(cfg, ticks, invariants_every=0):
    """Every tick, the excess the monitor finds is covered by the growth of the programs
    that stayed active since the last tick:
        sum_r overshoot_r(k) <= sum_{p active after tick k-1, not released} (contrib_k(p) - contrib_{k-1}(p))^+
    since after step 4 of tick k-1 every replica is at or below lambda_max*C (I3) and
    only releases leave the active set before step 3 (restores come after it).
    Returns the oracle and the number of ticks whose monitor found an excess."""
    o = oracle.Oracle(cfg, tracegen.make_trace(cfg))
    prev_contrib, prev_active, hit = None, set(), 0
    for _ in range(ticks):
        before = o.stats["overshoot_blocks"]
        st, _ = o.sched_step()
        assert st == oracle.OK
        found = o.stats["overshoot_blocks"] - before
        if prev_contrib is not None:
            growth = sum(max(0, o.contrib[p] - prev_contrib[p]) for p in prev_active
                         if o.status[p] != oracle.STOPPED)
            assert found <= growth, (o.tick, found, growth)
            hit += found > 0
        prev_contrib = list(o.contrib)
        prev_active = {p for p in range(o.N) if o.placement[p] >= 0}
        if invariants_every and o.tick % invariants_every == 0:
            o.check_invariants()
            o.check_watermark()
    return o, hit


def test_overshoot_bounded_by_growth_between_checks():
    for seed in range(4):
        o, hit = check_growth_bound(stress_cfg(300 + seed), 250)
        assert hit > 0


def test_decode_step_guard():
    """Delta t = one decode step (1000 / 40 tok/s = 25 ms): a decoding program gains one
    token per check (at most one block), so what the monitor finds beyond that comes
    from events (tool results, the end of a decay step), not from decode growth; the
    same growth bound and the invariants hold over 60 s of simulated time."""
    cfg = stress_cfg(310, NB=48, NH=8, delta_t_ms=25, decay_unit_ms=1000)
    assert cfg["decode_tok_per_s"] * cfg["delta_t_ms"] // 1000 == 1
    o, hit = check_growth_bound(cfg, 2400, invariants_every=50)
    assert hit > 0 and o.stats["pauses"] > 0
