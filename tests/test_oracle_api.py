"""API-mode events and explicit verbs (SURVEY.md §8(b)/(c) API table; SPEC.md:52-69,
240-257, 490-498).  Expected outcomes are the SPEC's stated contracts."""
import oracle
from oracle import ACTING, PAUSED, PHASE_A, PHASE_R, REASONING
from tests.helpers import base_cfg, set_program

A, DEC, TC, TR, REL = (oracle.E_ARRIVE, oracle.E_DECODE, oracle.E_TOOL_CALL,
                       oracle.E_TOOL_RESULT, oracle.E_RELEASE)


def api(n=4, **kw):
    return oracle.Oracle(base_cfg(**kw), api_mode=True, n_slots=n)


def test_create_program_enters_paused_and_dup_id():
    o = api()
    st, _ = o.sched_step(0, [(A, 0, 11, 512, 0)])
    assert st == oracle.OK
    # arrivals are Paused before first admission ... then restored this tick
    assert o.status[0] == REASONING and o.c[0] == 512
    st, dec = o.sched_step(5000, [(A, 0, 11, 512, 0)])
    assert st == oracle.E_DUP_ID and dec == []


def test_event_batch_is_all_or_nothing():
    o = api()
    o.sched_step(0, [(A, 0, 11, 100, 0)])
    c0 = o.c[0]
    st, _ = o.sched_step(5000, [(DEC, 0, 0, 50, 0), (TR, 0, 0, 30, 0)])   # result without call
    assert st == oracle.E_ILLEGAL_TRANSITION and o.c[0] == c0 and o.tick == 1


def test_reason_act_cycle_and_release_idempotent():
    o = api()
    o.sched_step(0, [(A, 0, 11, 100, 0)])
    o.sched_step(5000, [(DEC, 0, 0, 50, 0)])                          # c 100 -> 150
    assert o.c[0] == 150
    o.sched_step(10000, [(TC, 0, 0, 0, 9000)])
    assert o.status[0] == ACTING and o.phase[0] == PHASE_A and o.step_count[0] == 1
    o.sched_step(15000, [(TR, 0, 0, 30, 0)])                           # 150 -> 180
    assert o.status[0] == REASONING and o.c[0] == 180
    st, _ = o.sched_step(20000, [(REL, 0, 0, 0, 0)])
    assert st == oracle.OK and o.status[0] == oracle.STOPPED and o.placement[0] == -1
    assert all(o.hbm_free[0])                                          # KV reclaimed
    st, _ = o.sched_step(25000, [(REL, 0, 0, 0, 0)])
    assert st == oracle.OK
    st, _ = o.sched_step(30000, [(REL, 3, 0, 0, 0)])
    assert st == oracle.E_UNKNOWN_PROGRAM
    st, _ = o.sched_step(35000, [(DEC, 0, 0, 1, 0)])
    assert st == oracle.E_ILLEGAL_TRANSITION


def test_pause_verb_modes():
    o = oracle.Oracle(base_cfg(hbm_blocks=20, host_blocks=3), n_slots=3)
    set_program(o, 0, REASONING, PHASE_R, 5, placement=0, home=0, satisfied=1, hbm=range(5))
    o.L = [5]
    st, dec = o.pause(0, oracle.PAUSE_OFFLOAD)
    assert st == oracle.OK and o.status[0] == PAUSED and o.L == [0]
    assert dec[1][0] == oracle.D_EVICT and dec[1][4:7] == (5, 3, 2)    # host first, then drop
    o.check_invariants()
    st, _ = o.pause(0)
    assert st == oracle.E_ILLEGAL_TRANSITION


def test_resume_then_migrate_moves_blocks_p2p():
    o = oracle.Oracle(base_cfg(n_replicas=2, hbm_blocks=20), n_slots=2)
    set_program(o, 0, PAUSED, PHASE_R, 6, home=0, hbm=range(6))
    o.L = [0, 0]
    st, dec = o.resume(0, 0)
    assert st == oracle.OK and o.status[0] == REASONING and o.placement[0] == 0
    assert dec[-1][0] == oracle.D_FETCH and dec[-1][7] == 6            # resident: 6 hbm hits
    st, dec = o.migrate(0, 1)
    assert st == oracle.OK and o.placement[0] == 1 and o.home[0] == 1
    assert dec[0][0] == oracle.D_MIGRATE and dec[-1][8] == 6           # 6 peer tokens
    assert sum(1 for m in o.moves if m[0] == oracle.ta_oracle.MOVE_P2P) == 6
    o.check_invariants()
    assert o.L == [0, 6]


def test_resume_capacity_when_fetch_cannot_fit():
    """Load accounting admits the program but the physical fetch cannot be satisfied
    (blocks pinned by a program REASONING elsewhere): TA_E_CAPACITY, nothing changes."""
    o = oracle.Oracle(base_cfg(n_replicas=2, hbm_blocks=10), n_slots=2)
    set_program(o, 0, REASONING, PHASE_R, 8, placement=1, home=0, hbm=range(8))
    set_program(o, 1, PAUSED, PHASE_R, 3)
    o.L = [0, 8]
    st, dec = o.resume(1, 0)
    assert st == oracle.E_CAPACITY and dec == []
    assert o.status[1] == PAUSED and o.placement[1] == -1 and o.L == [0, 8]
    o.check_invariants()
    o.c[1] = 2
    st, dec = o.resume(1, 0)
    assert st == oracle.OK and dec[-1][0] == oracle.D_FETCH and dec[-1][4] == 2


def test_context_bound_rejected():
    """Reading A35: an event that would grow a context beyond max_ctx is rejected (E_INVAL)."""
    o = api(max_ctx=300)
    st, _ = o.sched_step(0, [(A, 0, 11, 301, 0)])
    assert st == oracle.E_INVAL and o.status[0] == oracle.UNARRIVED
    o.sched_step(0, [(A, 0, 11, 250, 0)])
    st, _ = o.sched_step(5000, [(DEC, 0, 0, 40, 0), (DEC, 0, 0, 11, 0)])
    assert st == oracle.E_INVAL and o.c[0] == 250
