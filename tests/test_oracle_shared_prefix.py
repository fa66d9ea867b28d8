"""NEXT-3 pins: shared system prompts, one per agent preset, refcounted per replica
(reading A51; "agentic system prompts are identical across workflows";
PAPER.md:365 "the shared prompt across programs implicitly reserves sufficient memory
buffer").

Program p's first sbk[k] blocks (k = its preset's prompt) are prompt k, stored once per
replica: the first program that needs it on a replica materializes it (its first
requests: lowest free blocks, prefilled), every program homed there points at those
blocks, pref[r][k] counts them, and the last one to leave (release, move elsewhere,
failure) releases the blocks.  Prompt blocks are never evicted, moved or compacted; the
load (Eq. 7) still counts full contexts.  Expected values below are worked out by hand
from that rule, or come from the same run without prompts (the case it reduces to)."""
import random

import oracle
import tracegen
from oracle.ta_oracle import FILL_NEW, FILL_PROMPT, MOVE_D2H, PROMPT, PROMPT_UID, decision
from tests.helpers import base_cfg, flat_trace, set_program
from tests.test_oracle_invariants import check_i9, stress_cfg

H = oracle.HOST_BIT
D = decision


def cfg_small(**kw):
    c = base_cfg(block_tokens=16, hbm_blocks=10, host_blocks=4, max_ctx=1024,
                 shared_prefix_tokens=32)
    c.update(kw)
    return c


def place_prompt(o, r, k, blocks):
    """Prompt k resident on replica r in `blocks` (no users yet)."""
    o.pblk[r][k] = list(blocks)
    for j, b in enumerate(blocks):
        o.hbm_free[r][b] = 0
        o.owner_hbm[r][b] = (PROMPT, k, j)


def homed(o, p, home, k, private=(), host=()):
    """Program p (using prompt k) homed on `home`: prompt entries, private HBM blocks,
    then host slots."""
    o.kp[p] = k
    set_program(o, p, o.status[p], o.phase[p], o.c[p], placement=o.placement[p], home=home,
                c_kv=o.c_kv[p], paused_since=o.paused_since[p], satisfied=o.satisfied[p],
                hbm=list(o.pblk[home][k]) + list(private), host=host)
    for j, b in enumerate(o.pblk[home][k]):     # set_program recorded p as their owner
        o.owner_hbm[home][b] = (PROMPT, k, j)
    o.pref[home][k] += 1


def free_blocks(o, r):
    return [b for b in range(o.NB) if o.hbm_free[r][b]]


def test_first_user_materializes_the_prompt_hand_computed():
    """Two 48-token arrivals, bt 16, a 32-token prompt (2 blocks), NB 10.  F = [p0, p1]:
    p0 brings the prompt (2 extra blocks, its first requests: blocks 0, 1) and its own
    block 2; p1 shares the prompt and takes block 3.  Without prompts: [0, 1, 2], [3, 4, 5]."""
    tr = flat_trace(2, turns=2, g=10, p0=48)
    o = oracle.Oracle(cfg_small(), tr)
    assert o.K == 1 and o.sbk == [2] and free_blocks(o, 0) == list(range(10))
    st, out = o.sched_step()
    assert st == oracle.OK
    assert list(o.loc[0][:4]) == [0, 1, 2, oracle.NONE]
    assert list(o.loc[1][:4]) == [0, 1, 3, oracle.NONE]
    assert o.pblk[0][0] == [0, 1] and o.pref[0][0] == 2
    assert free_blocks(o, 0) == list(range(4, 10))
    fetch = [d for d in out if d[0] == oracle.D_FETCH]
    assert fetch == [D(oracle.D_FETCH, 0, src=-1, dst=0, blocks=3, new=48),
                     D(oracle.D_FETCH, 1, src=-1, dst=0, blocks=1, new=48)]
    assert (o.stats["prefix_blocks"], o.stats["new_blocks"], o.stats["fetch_blocks"]) == (2, 2, 4)
    assert o.fills == [(FILL_PROMPT, 0, 0, PROMPT_UID, 0, 0, 16), (FILL_PROMPT, 0, 1, PROMPT_UID, 1, 16, 32),
                       (FILL_NEW, 0, 2, 0, 2, 32, 48), (FILL_NEW, 0, 3, 1, 2, 32, 48)]
    assert o.stats["fill_tok"] == 64
    assert o.L == [6]                                         # the load counts full contexts
    o.check_invariants()
    p = oracle.Oracle(cfg_small(shared_prefix_tokens=0), tr)
    p.sched_step()
    assert list(p.loc[0][:3]) == [0, 1, 2] and list(p.loc[1][:3]) == [3, 4, 5]


def api_cfg():
    # two prompts: 32 tokens (2 blocks) for preset "a", 16 tokens (1 block) for "b"
    return base_cfg(block_tokens=16, hbm_blocks=12, max_ctx=1024, shared_prefixes=[(32, "a"), (16, "b")])


def test_two_prompts_refcounts_and_release_by_the_last_user_hand_computed():
    """API mode (ARRIVE's t_ms = prompt index).  Tick 0: p0 (prompt 0), p1 (prompt 1),
    p2 (prompt 0), 48 tokens each.  F = [p0, p1, p2]: p0 brings prompt 0 (blocks 0, 1)
    and takes 2; p1 brings prompt 1 (block 3) and takes 4, 5; p2 shares prompt 0 and takes
    6.  Tick 1: p0 stops: its block 2 is freed, prompt 0 keeps one user.  Tick 2: p2
    stops: prompt 0's last user, so blocks 0, 1 are freed with its block 6.  Tick 3: p3
    arrives with prompt 0 and materializes it again in the lowest free blocks 0, 1."""
    o = oracle.Oracle(api_cfg(), api_mode=True, n_slots=4)
    A, REL = oracle.E_ARRIVE, oracle.E_RELEASE
    st, out = o.sched_step(0, [(A, 0, 1, 48, 0), (A, 1, 2, 48, 1), (A, 2, 3, 48, 0)])
    assert st == oracle.OK
    assert [list(o.loc[p][:3]) for p in range(3)] == [[0, 1, 2], [3, 4, 5], [0, 1, 6]]
    assert o.pblk[0] == [[0, 1], [3]] and o.pref[0] == [2, 1]
    assert [d[4] for d in out if d[0] == oracle.D_FETCH] == [3, 3, 1]     # need + prompt blocks
    assert o.stats["prefix_blocks"] == 3 and free_blocks(o, 0) == [7, 8, 9, 10, 11]
    o.check_invariants()
    st, out = o.sched_step(5000, [(REL, 0, 0, 0, 0)])
    assert st == oracle.OK and out == []
    assert o.pref[0] == [1, 1] and o.pblk[0][0] == [0, 1] and free_blocks(o, 0) == [2, 7, 8, 9, 10, 11]
    o.check_invariants()
    st, out = o.sched_step(10000, [(REL, 2, 0, 0, 0)])
    assert st == oracle.OK
    assert o.pref[0] == [0, 1] and o.pblk[0][0] is None
    assert free_blocks(o, 0) == [0, 1, 2, 6, 7, 8, 9, 10, 11]
    o.check_invariants()
    st, out = o.sched_step(15000, [(A, 3, 4, 48, 0)])
    assert st == oracle.OK
    assert list(o.loc[3][:3]) == [0, 1, 2] and o.pblk[0][0] == [0, 1] and o.pref[0] == [1, 1]
    assert o.stats["prefix_blocks"] == 5
    o.check_invariants()


def test_eviction_spares_the_prompt_hand_computed():
    """NB 6, prompt 0 at blocks 4, 5.  A PAUSED homed on 0 with rows [4, 5, 0, 1]
    (c 64); B REASONING on 0, fresh, c 80: the prompt is resident, so need = 5 - 2 = 3,
    no extra; free {2, 3}; supply = 2 + (4 - 2) = 4 >= 3; X = 1: A's tail block j = 3
    (idx 1) goes to host slot 0.  B then takes blocks 1, 2, 3: row [4, 5, 1, 2, 3]."""
    tr = flat_trace(2, turns=2, g=10, p0=32)
    o = oracle.Oracle(cfg_small(hbm_blocks=6), tr)
    place_prompt(o, 0, 0, (4, 5))
    set_program(o, 0, oracle.PAUSED, oracle.PHASE_R, 64)
    homed(o, 0, 0, 0, private=(0, 1))
    set_program(o, 1, oracle.REASONING, oracle.PHASE_R, 80, placement=0, c_kv=0)
    o.kp[1] = 0
    o.tick = 1
    o.check_invariants()
    st, out = o.sched_step()
    assert st == oracle.OK
    assert D(oracle.D_EVICT, 0, src=0, blocks=1, to_host=1) in out
    assert list(o.loc[0][:4]) == [4, 5, 0, H | 0]
    assert list(o.loc[1][:5]) == [4, 5, 1, 2, 3]
    assert o.moves[0] == (MOVE_D2H, 0, 1, 0, 0, 0, 3)
    assert o.pref[0][0] == 2 and o.stats["prefix_blocks"] == 0
    o.check_invariants()


def test_resume_elsewhere_brings_the_prompt_hand_computed():
    """R 2, NB 6 each.  A PAUSED homed on 0, rows [4, 5, 0, H|0], c = c_kv = 64;
    replica 0 is loaded by B (c 80, REASONING, homed there too) so A restores onto
    replica 1, where no program holds the prompt: A brings it (blocks 0, 1 of replica
    1, its 32 tokens recomputed: miss 32), then block 2 <- replica 0's block 0 (P2P,
    peer 16) and block 3 <- replica 0's host slot 0 (H2D, host 16).  Step 7: A's sources
    are freed and A leaves prompt 0 on replica 0, which B keeps."""
    tr = flat_trace(2, turns=2, g=10, p0=32)
    o = oracle.Oracle(cfg_small(n_replicas=2, hbm_blocks=6, lambda_min_q16=65535), tr)
    place_prompt(o, 0, 0, (4, 5))
    set_program(o, 0, oracle.PAUSED, oracle.PHASE_R, 64)
    homed(o, 0, 0, 0, private=(0,), host=(0,))
    set_program(o, 1, oracle.REASONING, oracle.PHASE_R, 80, placement=0, satisfied=1)
    homed(o, 1, 0, 0, private=(1, 2, 3))
    o.tick = 1
    o.check_invariants()
    st, out = o.sched_step()
    assert st == oracle.OK
    assert D(oracle.D_RESTORE, 0, src=0, dst=1) in out
    assert D(oracle.D_FETCH, 0, src=0, dst=1, blocks=4, peer=16, host=16, miss=32) in out
    assert list(o.loc[0][:4]) == [0, 1, 2, 3] and o.home[0] == 1
    assert o.pblk[1][0] == [0, 1] and o.pref == [[1], [1]] and o.pblk[0][0] == [4, 5]
    assert o.hbm_free[0][0] == 1 and o.host_free[0][0] == 1   # deferred frees of the sources
    assert o.busy[0] == 100                                   # one prefill chunk for the 32 missed tokens
    o.check_invariants()


def test_migrating_the_last_user_away_releases_the_prompt():
    """A REASONING program alone with prompt 0 on replica 0 migrates to replica 1 (verb):
    replica 1 materializes the prompt for it, and replica 0's prompt blocks are freed."""
    tr = flat_trace(1, turns=2, g=10, p0=32)
    o = oracle.Oracle(cfg_small(n_replicas=2, hbm_blocks=8), tr)
    place_prompt(o, 0, 0, (6, 7))
    set_program(o, 0, oracle.REASONING, oracle.PHASE_R, 48, placement=0, satisfied=1)
    homed(o, 0, 0, 0, private=(0,))
    o.L = [3, 0]
    o.check_invariants()
    st, out = o.migrate(0, 1)
    assert st == oracle.OK
    assert out[0] == D(oracle.D_MIGRATE, 0, src=0, dst=1)
    assert list(o.loc[0][:3]) == [0, 1, 2] and o.home[0] == 1
    assert o.pblk[1][0] == [0, 1] and o.pblk[0][0] is None and o.pref == [[0], [1]]
    assert free_blocks(o, 0) == list(range(8))
    o.check_invariants()


def test_reduces_to_the_unshared_run_when_nothing_is_evicted():
    """With a pool no run ever fills, a prompt changes no scheduling decision (the load
    counts full contexts); per replica, used blocks = unshared used - sb * (homed
    programs) + sb if any program is homed there."""
    for seed in range(4):
        cfg = stress_cfg(seed, R=2, NB=4096, NH=0, n=24, n0=10, compact=0,
                         lambda_max_q16=1966, lambda_min_q16=1966)
        cfg_s = dict(cfg, shared_prefix_tokens=64)
        tr = tracegen.make_trace(cfg)
        a, b = oracle.Oracle(cfg, tr), oracle.Oracle(cfg_s, tr)
        sb = b.sbk[0]
        for _ in range(120):
            sa, da = a.sched_step()
            sb_, db = b.sched_step()
            assert sa == sb_ == oracle.OK
            sched = lambda ds: [d for d in ds if d[0] in (oracle.D_PAUSE, oracle.D_RESTORE, oracle.D_STALL)]
            assert sched(da) == sched(db)
            for r in range(2):
                homed_r = sum(1 for p in range(a.N) if a.home[p] == r)
                used_a = a.NB - sum(a.hbm_free[r])
                used_b = b.NB - sum(b.hbm_free[r])
                assert used_b == used_a - sb * homed_r + (sb if homed_r else 0), (seed, r)
            b.check_invariants()
        assert a.stats["evict_blocks"] == b.stats["evict_blocks"] == 0


def test_random_stress_invariants_with_two_prompts():
    """Tight pools, host tier, compaction every 3 ticks, 2 replicas, two prompts (one
    per preset of a two-preset mix): the invariants (I1-I10, refcounts, residency,
    prompt rows) after every tick; no move or compaction ever touches a prompt block."""
    made = 0
    for seed in range(6):
        cfg = stress_cfg(100 + seed, compact=3)
        tr = tracegen.make_trace(cfg)
        tr.preset = ["a" if p % 2 == 0 else "b" for p in range(tr.n_slots)]
        cfg["shared_prefixes"] = [(48, "a"), (32, "b")]
        o = oracle.Oracle(cfg, tr)
        assert o.sbk == [3, 2]
        for _ in range(300):
            st, ds = o.sched_step()
            assert st == oracle.OK
            o.check_invariants()
            o.check_watermark()
            check_i9(o)
            for kind, sr, si, dr, di, p, j in o.moves:
                assert j >= o.sbp(p), f"a prompt block moved: {(kind, si, di, p, j)}"
            for f in o.fills:
                if f[0] != FILL_PROMPT:
                    assert f[4] >= o.sbp(f[3]), f
            if all(s in (oracle.STOPPED, oracle.UNARRIVED) for s in o.status) and o.next_arrival == o.N:
                break
        made += o.stats["prefix_blocks"]
    assert made > 0


def test_verbs_and_failover_keep_prompts_consistent():
    """OFFLOAD pauses evict only private blocks; a failed replica loses its programs'
    blocks and its prompts (only private blocks are counted as lost)."""
    rng = random.Random(7)
    cfg = stress_cfg(200, NB=64, shared_prefix_tokens=32)
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    for k in range(120):
        o.sched_step()
        act = [p for p in range(o.N) if o.status[p] in (oracle.REASONING, oracle.ACTING)]
        if act and k % 5 == 0:
            p = rng.choice(act)
            nh = sum(1 for j in range(o.nb_of(p)) if o.is_hbm(o.loc[p][j]) and j >= o.sbp(p))
            st, out = o.pause(p, oracle.PAUSE_OFFLOAD)
            assert st == oracle.OK
            ev = [d for d in out if d[0] == oracle.D_EVICT]
            assert (ev[0][4] if ev else 0) == (nh if o.home[p] >= 0 else 0)
        if k == 60:
            homed_1 = {p: sum(1 for j, e in enumerate(o.loc[p]) if e != oracle.NONE and j >= o.sbp(p))
                       for p in range(o.N) if o.home[p] == 1}
            st, out = o.set_health(1, False)
            lost = {d[1]: d[4] for d in out if d[0] == oracle.D_EVICT}
            assert lost == {p: n for p, n in homed_1.items() if n}
            assert sum(o.hbm_free[1]) == o.NB and o.pblk[1] == [None] and o.pref[1] == [0]
        if k == 80:
            o.set_health(1, True)
        o.check_invariants()


def test_api_arrival_prompt_checks():
    """K = 1: t_ms is ignored, a prompt shorter than the shared prefix is rejected;
    K = 2: t_ms must name a prompt, and the prompt must cover it."""
    o = oracle.Oracle(cfg_small(), api_mode=True, n_slots=4)
    assert o.sched_step(0, [(oracle.E_ARRIVE, 0, 1, 31, 0)]) == (oracle.E_INVAL, [])
    st, _ = o.sched_step(0, [(oracle.E_ARRIVE, 0, 1, 32, 7)])
    assert st == oracle.OK and list(o.loc[0][:2]) == [0, 1] and o.kp[0] == 0
    o2 = oracle.Oracle(api_cfg(), api_mode=True, n_slots=4)
    assert o2.sched_step(0, [(oracle.E_ARRIVE, 0, 1, 48, 2)])[0] == oracle.E_INVAL
    assert o2.sched_step(0, [(oracle.E_ARRIVE, 0, 1, 31, 0)])[0] == oracle.E_INVAL
    st, _ = o2.sched_step(0, [(oracle.E_ARRIVE, 0, 1, 16, 1)])
    assert st == oracle.OK and o2.kp[0] == 1 and o2.pblk[0][1] == [0]
