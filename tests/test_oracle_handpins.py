"""Hand-computed pins of the oracle's definitional steps (VERDICT r1 "what's weak" 1):
two-finger compaction (reading A20), the program-aware eviction order with all three
groups (reading A21; "evict long-idling caches under memory pressure")
and the tool-call start time of a partially used interval (readings A3, A33, A48).

Every expected value below was worked out by hand from DESIGN.md §2 (steps 5.3 and 7)
and is written out literally; a plausible mistake in the oracle (finger order, group
order, floor for ceil) changes at least one of them."""
import oracle
from oracle.ta_oracle import MOVE_D2D, MOVE_D2H, MOVE_DROP, decision
from tests.helpers import base_cfg, flat_trace, set_program

NONE, HB = oracle.NONE, oracle.HOST_BIT


def _free(o, r):
    return [b for b in range(o.NB) if o.hbm_free[r][b]]


# --------------------------------------------------------------------------- A20
def test_two_finger_compaction_by_hand():
    """NB = 12, used {0, 2, 3, 7, 9, 11} (p0 holds 0, 2, 3; p1 holds 7, 9, 11).
    Fingers: lowest free 1 <- highest used 11; 4 <- 9; 5 <- 7; then the lowest free (6)
    is above the highest used (3): stop.  3 blocks move, highest first."""
    o = oracle.Oracle(base_cfg(hbm_blocks=12, max_ctx=16), flat_trace(2))
    set_program(o, 0, oracle.PAUSED, oracle.PHASE_R, 3, home=0, hbm=(0, 2, 3))
    set_program(o, 1, oracle.PAUSED, oracle.PHASE_R, 3, home=0, hbm=(7, 9, 11))
    out = []
    o._compact(0, out)
    assert out == [decision(oracle.D_COMPACT, oracle.NONE, src=0, dst=0, blocks=3)]
    assert list(o.loc[0][:3]) == [0, 2, 3]
    assert list(o.loc[1][:3]) == [5, 4, 1]                 # j0: 7->5, j1: 9->4, j2: 11->1
    assert o.moves == [(MOVE_D2D, 0, 11, 0, 1, 1, 2),
                       (MOVE_D2D, 0, 9, 0, 4, 1, 1),
                       (MOVE_D2D, 0, 7, 0, 5, 1, 0)]
    assert _free(o, 0) == [6, 7, 8, 9, 10, 11]
    assert o.owner_hbm[0][1] == (1, 2) and o.owner_hbm[0][4] == (1, 1) and o.owner_hbm[0][5] == (1, 0)
    assert o.owner_hbm[0][7] is None and o.owner_hbm[0][9] is None and o.owner_hbm[0][11] is None
    o.check_invariants()
    out2 = []
    o._compact(0, out2)                                     # already compact: no move, no record
    assert out2 == [] and o.moves[3:] == []


def test_two_finger_compaction_adjacent_last_pair_by_hand():
    """NB = 8, used {0, 1, 4, 5}: 5 -> 2, then the fingers are adjacent (lowest free 3,
    highest used 4) and still cross over: 4 -> 3.  Now lowest free 4 > highest used 3:
    stop.  2 moves (a rule that stops one pair early moves only one)."""
    o = oracle.Oracle(base_cfg(hbm_blocks=8, max_ctx=16), flat_trace(1))
    set_program(o, 0, oracle.PAUSED, oracle.PHASE_R, 4, home=0, hbm=(0, 1, 4, 5))
    out = []
    o._compact(0, out)
    assert out == [decision(oracle.D_COMPACT, oracle.NONE, src=0, dst=0, blocks=2)]
    assert list(o.loc[0][:4]) == [0, 1, 3, 2]
    assert o.moves == [(MOVE_D2D, 0, 5, 0, 2, 0, 3), (MOVE_D2D, 0, 4, 0, 3, 0, 2)]
    assert _free(o, 0) == [4, 5, 6, 7]


def test_two_finger_compaction_spares_shared_prompt_and_runs_in_the_tick():
    """A shared prompt (reading A51) of 2 blocks sits at blocks 4, 5 (used by p0 and p1);
    private blocks: p0 {0, 2, 3}, p1 {7, 9}; free {1, 6, 8, 10, 11}.  The upper finger
    skips the prompt's blocks: 9 -> 1, 7 -> 6, then the lowest free block (7) is above
    the highest movable used block (3): 2 moves.  Through sched_step with compact_every
    = 1, the COMPACT record is the last decision."""
    cfg = base_cfg(hbm_blocks=12, max_ctx=16, compact_every=1, shared_prefix_tokens=2)
    o = oracle.Oracle(cfg, flat_trace(2, p0=2, d_ms=10 ** 9))
    o.kp[0] = o.kp[1] = 0
    o.pblk[0][0] = [4, 5]
    o.pref[0][0] = 2
    for j, b in enumerate((4, 5)):
        o.hbm_free[0][b] = 0
        o.owner_hbm[0][b] = (oracle.ta_oracle.PROMPT, 0, j)
    for p, priv in ((0, (0, 2, 3)), (1, (7, 9))):
        set_program(o, p, oracle.PAUSED, oracle.PHASE_R, 2 + len(priv), home=0)
        o.loc[p][0], o.loc[p][1] = 4, 5
        for j, b in enumerate(priv, start=2):
            o.loc[p][j] = b
            o.hbm_free[0][b] = 0
            o.owner_hbm[0][b] = (p, j)
    o.next_arrival = 2
    o.check_invariants()
    # lambda = 1, NB = 12: both paused programs (5 + 4 blocks) fit; the restore pass puts
    # them back on r0 without moving bytes, so only compaction moves blocks this tick
    st, dec = o.sched_step()
    assert st == oracle.OK
    assert dec[-1] == decision(oracle.D_COMPACT, oracle.NONE, src=0, dst=0, blocks=2)
    assert list(o.loc[1][:4]) == [4, 5, 6, 1]             # j2: 7 -> 6, j3: 9 -> 1
    assert list(o.loc[0][:5]) == [4, 5, 0, 2, 3]
    assert [m for m in o.moves if m[0] == MOVE_D2D] == [(MOVE_D2D, 0, 9, 0, 1, 1, 3),
                                                        (MOVE_D2D, 0, 7, 0, 6, 1, 2)]
    assert _free(o, 0) == [7, 8, 9, 10, 11]
    o.check_invariants()


# --------------------------------------------------------------------------- A21
def _eviction_state():
    """Replica 0 (NB = 20, host tier NH = 3 with slot 1 taken), bt = 1.
      p0 PAUSED  phase A nb 1  hbm [0]                 group 0
      p1 PAUSED  phase R nb 2  hbm [1, 2]              group 0
      p2 PAUSED  phase R nb 3  hbm [3, 4, 5]           group 0
      p3 ACTING  on r1   nb 4  hbm [6..9]   contrib 2  group 1  (t_q = 1 s: 4 * 2^-1)
      p4 ACTING  on r1   nb 4  hbm [10..13] contrib 1  group 1  (t_q = 2 s: 4 * 2^-2)
      p5 ACTING  on r0   nb 2  hbm [14, 15] contrib 2  group 2  (t_q = 0)
      p6 PAUSED  host slot 1 only (not a candidate: no HBM blocks)
      p7 REASONING on r0, new (c = 12, no KV): need 12, free 4 (16..19) -> X = 8."""
    cfg = base_cfg(n_replicas=2, hbm_blocks=20, host_blocks=3, max_ctx=64)
    o = oracle.Oracle(cfg, flat_trace(8, d_ms=10 ** 9))
    T = 10000
    set_program(o, 0, oracle.PAUSED, oracle.PHASE_A, 1, home=0, acting_since=T, hbm=(0,))
    set_program(o, 1, oracle.PAUSED, oracle.PHASE_R, 2, home=0, hbm=(1, 2))
    set_program(o, 2, oracle.PAUSED, oracle.PHASE_R, 3, home=0, hbm=(3, 4, 5))
    set_program(o, 3, oracle.ACTING, oracle.PHASE_A, 4, placement=1, home=0, acting_since=T - 1000,
                hbm=(6, 7, 8, 9))
    set_program(o, 4, oracle.ACTING, oracle.PHASE_A, 4, placement=1, home=0, acting_since=T - 2000,
                hbm=(10, 11, 12, 13))
    set_program(o, 5, oracle.ACTING, oracle.PHASE_A, 2, placement=0, home=0, acting_since=T, hbm=(14, 15))
    set_program(o, 6, oracle.PAUSED, oracle.PHASE_R, 1, home=0, host=(1,))
    set_program(o, 7, oracle.REASONING, oracle.PHASE_R, 12, placement=0, c_kv=0)
    o.check_invariants()
    o._step1_footprint()
    o._step2_load(T)
    o._satisfied_now, o._ledger_s = set(), []
    return o


def test_eviction_order_groups_by_hand():
    """Restore order of the PAUSED candidates (R first, nb up): p1, p2, p0, so group 0
    evicts in its exact reverse p0, p2, p1 (not slot order, not nb order); group 1 by
    (contrib, slot): p4 (1) before p3 (2); group 2 (p5) last."""
    o = _eviction_state()
    assert o.contrib[3] == 2 and o.contrib[4] == 1 and o.contrib[5] == 2
    assert o._evict_order(0) == [0, 2, 1, 4, 3, 5]


def test_eviction_into_group1_partial_victim_host_then_drop_by_hand():
    """X = 8: p0 (1) + p2 (3) + p1 (2) whole, then 2 of p4's 4 blocks (partial last
    victim, tail first).  Host slots lowest free first: e0 (p0 j0, block 0) -> slot 0,
    e1 (p2 j2, block 5) -> slot 2 (slot 1 is taken), then the tier is full and every
    further block is dropped.  p7 then takes the 12 lowest free blocks in j order."""
    o = _eviction_state()
    ev, fx, deferred = [], [], []
    assert o._materialize(0, [7], ev, fx, deferred)
    D = decision
    assert ev == [D(oracle.D_EVICT, 0, src=0, blocks=1, to_host=1, dropped=0),
                  D(oracle.D_EVICT, 2, src=0, blocks=3, to_host=1, dropped=2),
                  D(oracle.D_EVICT, 1, src=0, blocks=2, to_host=0, dropped=2),
                  D(oracle.D_EVICT, 4, src=0, blocks=2, to_host=0, dropped=2)]
    M1, M5 = MOVE_D2H, MOVE_DROP
    assert o.moves[:8] == [(M1, 0, 0, 0, 0, 0, 0), (M1, 0, 5, 0, 2, 2, 2),
                           (M5, 0, 4, -1, -1, 2, 1), (M5, 0, 3, -1, -1, 2, 0),
                           (M5, 0, 2, -1, -1, 1, 1), (M5, 0, 1, -1, -1, 1, 0),
                           (M5, 0, 13, -1, -1, 4, 3), (M5, 0, 12, -1, -1, 4, 2)]
    assert list(o.loc[0][:1]) == [HB | 0]
    assert list(o.loc[2][:3]) == [NONE, NONE, HB | 2]
    assert list(o.loc[1][:2]) == [NONE, NONE]
    assert list(o.loc[4][:4]) == [10, 11, NONE, NONE]
    assert list(o.loc[3][:4]) == [6, 7, 8, 9] and list(o.loc[5][:2]) == [14, 15]
    assert list(o.loc[7][:12]) == [0, 1, 2, 3, 4, 5, 12, 13, 16, 17, 18, 19]
    assert [s for s in range(3) if o.host_free[0][s]] == []
    assert o.owner_host[0][0] == (0, 0) and o.owner_host[0][2] == (2, 2)
    assert fx == [D(oracle.D_FETCH, 7, src=-1, dst=0, blocks=12, new=12)]
    assert _free(o, 0) == []
    st = o.stats
    assert (st["evict_blocks"], st["evict_to_host"], st["evict_dropped"]) == (8, 2, 6)
    assert (st["new_blocks"], st["fetch_blocks"]) == (12, 12)


# --------------------------------------------------------------------------- A3/A33/A48
def test_tool_call_start_time_partial_interval_with_busy():
    """Reading A48 + A33: the engine spent busy = 1000 ms of the interval prefilling,
    then decodes at 30 tokens/s; the turn has 100 tokens left, fewer than the
    30 * (5000 - 1000) / 1000 = 120 the interval allows, so they finish after
    ceil(100 * 1000 / 30) = 3334 ms (3333.3 rounded UP, reading A33).  The tool call
    therefore starts at T - 5000 + 1000 + 3334 = T - 666 and returns d_ms = 7000 later."""
    cfg = base_cfg(hbm_blocks=1000, max_ctx=4096, decode_tok_per_s=30)
    o = oracle.Oracle(cfg, flat_trace(1, turns=2, g=100, d_ms=7000, o=5, p0=10))
    set_program(o, 0, oracle.REASONING, oracle.PHASE_R, 10, placement=0, home=0, satisfied=1,
                hbm=tuple(range(10)))
    o.busy[0] = 1000
    o.next_arrival = 1
    k, T = 3, 15000
    o._step0_trace(k, T)
    assert o.c[0] == 110 and o.gen_done[0] == 100
    assert o.phase[0] == oracle.PHASE_A and o.status[0] == oracle.ACTING
    assert o.acting_since[0] == 15000 - 5000 + 1000 + 3334 == 14334
    assert o.tool_return[0] == 21334
    # the tool result arrives at the first tick with T >= 21334: tick 5 (T = 25000)
    o._step0_trace(4, 20000)
    assert o.phase[0] == oracle.PHASE_A
    o._step0_trace(5, 25000)
    assert o.phase[0] == oracle.PHASE_R and o.c[0] == 115 and o.turn[0] == 1


def test_tool_call_start_time_busy_longer_than_interval():
    """busy is capped at Delta t (A48): a 7000 ms materialize leaves no decode time, so
    nothing is generated and no tool call starts during that interval."""
    cfg = base_cfg(hbm_blocks=1000, max_ctx=4096, decode_tok_per_s=30)
    o = oracle.Oracle(cfg, flat_trace(1, turns=2, g=100, d_ms=7000, o=5, p0=10))
    set_program(o, 0, oracle.REASONING, oracle.PHASE_R, 10, placement=0, home=0, satisfied=1,
                hbm=tuple(range(10)))
    o.busy[0] = 7000
    o.next_arrival = 1
    o._step0_trace(3, 15000)
    assert o.c[0] == 10 and o.gen_done[0] == 0 and o.status[0] == oracle.REASONING
