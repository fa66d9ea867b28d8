"""NEXT-1 pins: the STP cost ledger (Eq. 2-3; SPEC.md cost-ledger
record / recompute_cost_of / decompose; Appendix E.2 staircase) and
the Cost_unused bound.  Readings A40-A44."""
import oracle
from oracle.ta_oracle import stair
from tests.helpers import base_cfg, flat_trace, set_program

DT = 5000


def test_staircase_spec_examples():
    assert stair(8, 2) == 20                  # SPEC: (c=8, chunk=2) -> 2+4+6+8 = 20
    assert stair(0, 4) == 0                   # SPEC: empty context
    assert stair(8, 2, base=10) == 12 + 14 + 16 + 18
    assert stair(7, 2) == 2 + 4 + 6 + 7       # ragged last chunk
    for m in range(1, 40):                    # closed form q*m(m+1)/2 at c = m*q
        assert stair(m * 16, 16) == 16 * m * (m + 1) // 2


def test_staircase_quadratic_ratio_lemma1():
    """Lemma 1: recompute cost ~ c^2 at fixed chunk: the ratio
    cost(2c)/cost(c) tends to 4 (SPEC: exponent 2.0 +- 0.05 over c in 2^6..2^14)."""
    for e in range(6, 15):                    # c = m*q: ratio = 2(2m+1)/(m+1) = 4 - 2/(m+1)
        c = 1 << e
        m = c // 8
        assert stair(2 * c, 8) * (m + 1) == stair(c, 8) * 2 * (2 * m + 1)
    assert abs(stair(1 << 15, 8) / stair(1 << 14, 8) - 4.0) < 0.002


def one_tick(o):
    before = dict(o.stats)
    st, _ = o.sched_step()
    assert st == oracle.OK
    return {k: o.stats[k] - before[k] for k in o.stats}


def test_decode_and_caching_rectangles():
    """A satisfied REASONING program (c = 7) and an ACTING program with 10 resident
    tokens, no pressure, no decode (rate 0): every tick adds 7*dt decode and 10*dt caching
    (SPEC: 10 tokens held for 5 ticks as Caching -> 50 token-ticks)."""
    o = oracle.Oracle(base_cfg(hbm_blocks=100), flat_trace(2, g=1000, d_ms=10 ** 9))
    set_program(o, 0, oracle.REASONING, oracle.PHASE_R, 7, placement=0, home=0, satisfied=1, hbm=range(7))
    set_program(o, 1, oracle.ACTING, oracle.PHASE_A, 10, placement=0, home=0, acting_since=0,
                tool_return=10 ** 12, hbm=range(7, 17))
    o.next_arrival = 2
    for _ in range(5):
        dl = one_tick(o)
        assert dl["cost_decode"] == 7 * DT
        assert dl["cost_caching"] == 10 * DT
        assert dl["cost_prefill"] == dl["cost_recompute"] == dl["cost_unused"] == 0
    assert o.stats["cost_caching"] == 10 * 5 * DT


def test_recompute_and_prefill_staircases():
    """Resumed program, history of 8 tokens fully lost (bt = 1), chunk 2: recompute
    adds tau*20 (SPEC example); a satisfied program with c_kv = 10 and 8 new tokens
    adds tau*(12+14+16+18) prefill."""
    cfg = base_cfg(hbm_blocks=100, prefill_chunk_tokens=2, prefill_chunk_ms=3)
    o = oracle.Oracle(cfg, flat_trace(2, g=1000, d_ms=10 ** 9))
    set_program(o, 0, oracle.PAUSED, oracle.PHASE_R, 8, c_kv=8, paused_since=0)       # no blocks left
    set_program(o, 1, oracle.REASONING, oracle.PHASE_R, 18, c_kv=10, placement=0, home=0, satisfied=1,
                hbm=range(20, 30))
    o.next_arrival = 2
    dl = one_tick(o)
    assert dl["cost_recompute"] == 3 * 20
    assert dl["cost_prefill"] == 3 * (12 + 14 + 16 + 18) + 3 * 0    # program 0: c_kv = c after recompute
    assert dl["cost_decode"] == (8 + 18) * DT


def test_unused_cost_and_bound_hand_computed():
    """Two replicas of 10 blocks (bt = 1): r0 full, r1 holds 3; a paused 8-token program
    (phase R) fits nowhere (3 + 8 > 10) -> the queue stays non-empty: unused r0 = 0,
    r1 = 7 blocks -> 7*dt; bound: idle r1 = 10 - 3 = 7 < c_min = 8 holds."""
    cfg = base_cfg(n_replicas=2, hbm_blocks=10)
    o = oracle.Oracle(cfg, flat_trace(4, g=1000, d_ms=10 ** 9))
    set_program(o, 0, oracle.REASONING, oracle.PHASE_R, 10, placement=0, home=0, satisfied=1, hbm=range(10))
    set_program(o, 1, oracle.REASONING, oracle.PHASE_R, 3, placement=1, home=1, satisfied=1, hbm=range(3))
    set_program(o, 2, oracle.PAUSED, oracle.PHASE_R, 8, c_kv=0, paused_since=0)
    o.next_arrival = 3
    o.tick = 1                                # past tick 0: no initial arrivals for slot 3
    dl = one_tick(o)
    assert dl["cost_unused"] == 7 * DT
    assert dl["unused_bound_checks"] == 2 and dl["unused_bound_violations"] == 0
    # a phase-A paused program of 2 blocks behind the phase-R head: the queue stops at the
    # head (reading A9), the small one would fit on r1 -> c_min = 2 <= idle 7: violated
    set_program(o, 3, oracle.PAUSED, oracle.PHASE_A, 2, c_kv=2, paused_since=0, acting_since=0,
                tool_return=10 ** 12)
    o.next_arrival = 4
    dl = one_tick(o)
    assert dl["unused_bound_checks"] == 2 and dl["unused_bound_violations"] == 1


def test_engine_prefill_time_delays_decode_hand_computed():
    """Synthetic engine (reading A48): a resumed program whose 4096-token history was lost
    is recomputed in ceil(4096/2048) = 2 chunk steps of 100 ms, plus its 300 waiting
    tool-result tokens in 1 step: 300 ms of the next 5 s interval are not decoding, so at
    40 tokens/s it decodes 40 * 4.7 = 188 tokens instead of 200."""
    cfg = base_cfg(hbm_blocks=5000, max_ctx=8192, decode_tok_per_s=40, prefill_chunk_tokens=2048,
                   prefill_chunk_ms=100)
    o = oracle.Oracle(cfg, flat_trace(1, g=10 ** 6, d_ms=10 ** 9))
    set_program(o, 0, oracle.PAUSED, oracle.PHASE_R, 4396, c_kv=4096, paused_since=0)
    o.pend[0] = 300
    o.next_arrival = 1
    o.tick = 1
    one_tick(o)                                   # restored, recomputed, prefilled
    assert o.busy[0] == 300 and o.pend[0] == 0 and o.satisfied[0] == 1
    one_tick(o)                                   # decodes during the interval after
    assert o.c[0] == 4396 + 188
    one_tick(o)                                   # nothing left to prefill: a full interval
    assert o.c[0] == 4396 + 188 + 200
