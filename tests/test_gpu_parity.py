"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, tick by tick,
on identical seeded traces.  Decisions, program table, block tables, free sets and
owners must be bit-identical; KV bytes are checked against the content closed form
(on the GPU for every owned block, and on the CPU for sampled blocks)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import tracegen  # noqa: E402
from tests.gpu_compare import check_blocks_content, compare_state, dec_tuples, oracle_arrays  # noqa: E402
from tests.test_oracle_golden import DK, load_w1  # noqa: E402


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run_parity(cfg, ticks, state_every=1, content_every=1, samples=4, fill=True, flags=0, seed=0,
               host_blocks=None, counters=None):
    need_gpu()
    from paper_2602_13692_b200 import Pool
    if host_blocks is not None:
        cfg = dict(cfg, host_blocks=host_blocks)
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=fill, flags=flags)
    pool.load_trace(tr)
    rng = np.random.default_rng(seed)
    n_dec = 0
    for k in range(ticks):
        st_o, dec_o = o.sched_step()
        st_g, dec_g = pool.step()
        assert st_o == oracle.OK and st_g == 0
        got = dec_tuples(dec_g)
        if got != dec_o:
            for i, (a, b) in enumerate(zip(dec_o, got)):
                if a != b:
                    raise AssertionError(f"tick {k} decision {i}: oracle {a} gpu {b}")
            raise AssertionError(f"tick {k}: {len(dec_o)} oracle decisions vs {len(got)} gpu")
        n_dec += len(got)
        if state_every and (k % state_every == 0 or k == ticks - 1):
            compare_state(o, pool.debug_download(), where=f"tick {k}")
        if fill and content_every and (k % content_every == 0 or k == ticks - 1):
            bad, seen = pool.verify_content()
            assert bad == 0, f"tick {k}: {bad} of {seen} KV words differ from the closed form"
            check_blocks_content(o, pool, samples, rng)
        if o.next_arrival == o.N and all(s == oracle.STOPPED for s in o.status):
            break
    s = pool.stats()
    for key in oracle.ta_oracle.STAT_KEYS:
        assert s[key] == o.stats[key], (key, s[key], o.stats[key])
    if counters is not None:                  # size-branch counters (ta_debug_counters)
        for k, v in pool.debug_counters().items():
            counters[k] = counters.get(k, 0) + v
    pool.close()
    return o, n_dec


def stress(seed, R, NB=56, NH=16, n=24, n0=10, compact=3, **kw):
    return tracegen.get_config("c1_toy", n_replicas=R, hbm_blocks=NB, host_blocks=NH,
                               compact_every=compact, trace=dict(n=n, n_initial=n0, seed=seed), **kw)


def test_gpu_toy_config1_full_run():
    o, n = run_parity(tracegen.get_config("c1_toy"), 400)
    assert all(s == oracle.STOPPED for s in o.status) and n > 0


@pytest.mark.parametrize("seed,R", [(11, 1), (12, 2), (13, 3), (14, 2), (15, 4)])
def test_gpu_stress_full_run(seed, R):
    o, n = run_parity(stress(seed, R, NB=56 if R > 1 else 80), 300, seed=seed)
    assert o.stats["evict_blocks"] > 0 and o.stats["restores"] > 0


def test_gpu_stress_block_major_layout_and_bt1():
    run_parity(stress(21, 2, layout=1), 200)
    run_parity(stress(22, 2, NB=600, NH=200, block_tokens=1, compact=5), 120, state_every=5)


@pytest.mark.parametrize("dt,x,lam", [(1000, 1, 65536), (2500, 4, 65536), (10000, 8, 60000),
                                       (5000, 2, 52000)])
def test_gpu_policy_parameters(dt, x, lam):
    """The ablation axes (NEXT-2): detection period Delta t, decay base
    x of f(t) = x^-t (x = 1: no decay, eq. 6), and lambda_max < 1 (a watermark band:
    lambda_min = lambda_max - 4096)."""
    cfg = stress(40 + x, 2, NB=64, delta_t_ms=dt, decay_x=x, lambda_max_q16=lam,
                 lambda_min_q16=lam - (4096 if lam < 65536 else 0))
    o, n = run_parity(cfg, 200, seed=x)
    assert n > 0


def test_gpu_ttl_pin_baseline():
    """NEXT-2 baseline: TTL-pin decay table (step function) against the oracle."""
    from tracegen.configs import ttl_pin_table
    o, n = run_parity(stress(60, 2, NB=56, decay_table=ttl_pin_table(3)), 200, seed=60)
    assert n > 0


@pytest.mark.parametrize("R", [1, 3])
def test_gpu_request_aware_baseline(R):
    """NEXT-2 baseline: stateless request-level policy (TA_F_REQUEST_AWARE) vs the oracle."""
    o, n = run_parity(stress(70 + R, R, NB=56 if R > 1 else 80, request_aware=True), 200, seed=R)
    assert n > 0 and o.stats["pauses"] > 0


@pytest.mark.parametrize("R", [2, 3])
def test_gpu_pinned_routing_baseline(R):
    """NEXT-2 baseline: per-replica queues (TA_F_PINNED_ROUTING) against the oracle."""
    o, n = run_parity(stress(50 + R, R, NB=56, pinned_routing=True), 200, seed=R)
    assert n > 0 and o.stats["restores"] > 0


def test_gpu_no_graph_and_timing_modes():
    from paper_2602_13692_b200 import binding
    run_parity(stress(31, 2), 80, flags=binding.F_NO_GRAPH)
    run_parity(stress(32, 2), 40, flags=binding.F_TIMING)


@pytest.mark.parametrize("flags_name", ["F_NO_BULK_DEFAULT", "F_NO_FUSE"])
def test_gpu_copy_engine_variants(flags_name):
    """128-bit load/store engine instead of TMA bulk; split instead of fused movement."""
    from paper_2602_13692_b200 import binding
    run_parity(stress(33, 3), 120, flags=getattr(binding, flags_name))


def test_gpu_w1_golden():
    """Hand-computed two-tick example uploaded into the GPU state (tests/golden/w1.json)."""
    need_gpu()
    from paper_2602_13692_b200 import Pool
    g, o = load_w1()
    pool = Pool(o.cfg, o.N, max_turns=o.trace.total_turns, fill=False)
    pool.load_trace(o.trace)
    arrs = oracle_arrays(o)
    arrs["scalars"] = np.array([o.tick, o.next_arrival, 0, 0], np.int64)
    pool.debug_upload(arrs)
    for tk in g["ticks"]:
        st, dec = pool.step()
        assert st == 0
        want = [tuple([DK[d[0]]] + d[1:]) for d in tk["decisions"]]
        assert dec_tuples(dec) == want, tk["tick"]
        o.sched_step()
        compare_state(o, pool.debug_download(), where=f"W1 tick {tk['tick']}")
    pool.close()


def test_gpu_determinism():
    need_gpu()
    from paper_2602_13692_b200 import Pool
    cfg = stress(41, 3)
    outs = []
    for _ in range(2):
        tr = tracegen.make_trace(cfg)
        pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns)
        pool.load_trace(tr)
        log = [dec_tuples(pool.step()[1]) for _ in range(150)]
        st = pool.debug_download()
        outs.append((log, st["loc"].tobytes(), st["hbm_free"].tobytes(),
                     bytes(pool.hbm[0].cpu().numpy())))
        pool.close()
    assert outs[0] == outs[1]


@pytest.mark.slow
def test_gpu_config2_swe_q32_full_size():
    """configs[1] at full size (Qwen3-32B KV, 24,576 x 4 MiB blocks, 16,384 host slots)."""
    run_parity(tracegen.get_config("c2_swe"), 40, state_every=5, content_every=10, samples=3)


@pytest.mark.parametrize("name,ticks", [("c3_mixed", 25), ("c4_rlburst", 40)])
def test_gpu_configs3_4_decisions_full_n(name, ticks):
    """configs[2]/[3] at their full program counts and per-replica pools, all 8 replicas
    on one GPU with the decision-only KV shape (bytes per block do not affect decisions)."""
    cfg = tracegen.get_config(name, kv="mini")
    run_parity(cfg, ticks, state_every=4, content_every=4, samples=8)


@pytest.mark.parametrize("seed,R,spt", [(81, 1, 48), (82, 2, 48), (83, 3, 64), (84, 2, 16)])
def test_gpu_shared_prefix(seed, R, spt):
    """NEXT-3: the shared system prompt stored once per replica (reserved top blocks);
    tight pools with host tier and compaction; the reserved blocks' bytes (uid 0) are
    verified with the rest."""
    o, n = run_parity(stress(seed, R, NB=56 if R > 1 else 80, shared_prefix_tokens=spt), 300, seed=seed)
    assert o.stats["evict_blocks"] > 0 and o.stats["compact_blocks"] > 0 and o.sbk == [spt // 16]


def test_gpu_shared_prefix_swe_decisions_full_n():
    """configs[1] shape (256 SWE programs) with a 1024-token shared system prompt, the
    decision-only KV shape."""
    cfg = tracegen.get_config("c2_swe", kv="mini", shared_prefix_tokens=1024)
    o, n = run_parity(cfg, 40, state_every=5, content_every=10, samples=8)
    assert n > 0


@pytest.mark.parametrize("seed,R", [(86, 1), (87, 2), (88, 3)])
def test_gpu_two_shared_prompts(seed, R):
    """NEXT-3 widened (reading A51): two shared prompts (48 and 32 tokens), one per agent
    label, materialized by their first user on a replica, refcounted and released by
    the last; tight pools with host tier and compaction."""
    cfg = stress(seed, R, NB=56 if R > 1 else 80, n=32, n0=14)
    cfg["trace"]["labels"] = ["a", "b"]
    cfg["shared_prefixes"] = [(48, "a"), (32, "b")]
    o, n = run_parity(cfg, 300, seed=seed)
    assert o.stats["prefix_blocks"] > 0 and o.stats["evict_blocks"] > 0 and o.K == 2


def test_gpu_two_prompts_configs3_full_n():
    """configs[2] (2k programs, 8 replicas on one GPU, decision-only KV) with one shared
    prompt per preset: OpenHands 960 tokens, ToolOrchestra 640 tokens."""
    cfg = tracegen.get_config("c3_mixed", kv="mini", shared_prefixes=[(960, "openhands"), (640, "toolorch")])
    o, n = run_parity(cfg, 20, state_every=4, content_every=4, samples=8)
    assert n > 0 and o.sbk == [60, 40] and o.stats["prefix_blocks"] > 0


def test_gpu_decode_step_guard():
    """NEXT-4 guard: Delta t = one decode step (25 ms at 40 tok/s), 600 ticks; the
    overshoot counters are among the compared stats."""
    o, n = run_parity(stress(85, 2, NB=56, delta_t_ms=25), 600, state_every=10, content_every=20, seed=85)
    assert n > 0 and o.stats["overshoot_blocks"] > 0


def test_gpu_shared_prefix_configs3_full_n():
    """configs[2] (2k mixed programs, 8 replicas on one GPU, decision-only KV shape) with a
    960-token shared system prompt (every preset's prompt is at least 1,000 tokens)."""
    cfg = tracegen.get_config("c3_mixed", kv="mini", shared_prefix_tokens=960)
    o, n = run_parity(cfg, 20, state_every=4, content_every=4, samples=8)
    assert n > 0 and o.sbk == [60]


@pytest.mark.gpu
def test_gpu_decide_only_same_decisions():
    """TA_F_DECIDE_ONLY (the bench's decision-latency probe: no block copies): decisions,
    block tables, free sets, owners and statistics still equal the oracle's tick by tick
    (no decision depends on bytes); the pools' contents are not checked."""
    need_gpu()
    from paper_2602_13692_b200 import binding
    for seed, R in ((41, 1), (42, 3)):
        run_parity(stress(seed, R, compact=4), 200, state_every=2, seed=seed, fill=False,
                   flags=binding.F_DECIDE_ONLY)


@pytest.mark.gpu
def test_gpu_jitter_schedules():
    """TA_F_JITTER (development build): every CTA of the tick kernels sleeps a pseudo-random
    0-20 us at entry and after every grid / cluster barrier, shifting the CTAs against each
    other; results must stay bit-exact (a missing barrier between CTAs -- like the k_close
    race fixed in round 2 -- shows up as a wrong decision).  Trace mode with compaction every
    2 ticks on 3-4 replicas, then API-mode multi-event batches on 3 replicas."""
    need_gpu()
    import random
    from paper_2602_13692_b200 import Pool, binding
    from tests.test_gpu_api import random_event_sequences
    from tests.gpu_compare import same_decisions
    for seed, R in ((51, 3), (52, 4)):
        run_parity(stress(seed, R, compact=2), 120, state_every=3, seed=seed, flags=binding.F_JITTER)
    cfg = tracegen.get_config("c1_toy", n_replicas=3, hbm_blocks=48, host_blocks=16, max_ctx=4096,
                              compact_every=5)
    o = oracle.Oracle(cfg, api_mode=True, n_slots=48)
    pool = Pool(cfg, 48, trace_mode=False, flags=binding.F_JITTER)
    rng = random.Random(23)
    for k in range(120):
        T = 5000 * k
        evs = random_event_sequences(o, rng, T)
        st_o, dec_o = o.sched_step(T, evs)
        st_g, dec_g = pool.step(T, evs, raise_on_error=False)
        assert st_o == st_g, (k, st_o, st_g)
        if st_o == oracle.OK:
            same_decisions(dec_g, dec_o, f"jitter api tick {k}")
    pool.close()


def _lockstep_full_scan(cfg, ticks, verbs_seed=None, n_slots=None):
    """Two pools on the same trace: the product's footprint pass (counts only rows written
    since the previous pass) and TA_F_FULL_SCAN (development build: counts every live row,
    the round-1/2 behaviour the oracle parity was first established on).  After every tick
    and verb: the same status, the same decisions, and the same derived arrays (nb, n_hbm,
    n_host, prefix_hbm, contrib) and block tables."""
    import random
    from paper_2602_13692_b200 import Pool, binding
    tr = tracegen.make_trace(cfg)
    pools = [Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False, flags=f)
             for f in (0, binding.F_FULL_SCAN)]
    for p in pools:
        p.load_trace(tr)
    fields = ["status", "nb", "n_hbm", "n_host", "prefix_hbm", "contrib", "loc"]
    rng = random.Random(verbs_seed)
    for k in range(ticks):
        outs = [p.step() for p in pools]
        assert outs[0][0] == outs[1][0], (k, outs[0][0], outs[1][0])
        assert np.array_equal(outs[0][1], outs[1][1]), f"tick {k}: decisions differ"
        if verbs_seed is not None and k % 3 == 2:       # a verb between ticks (rows rewritten)
            st = pools[0].debug_download(["status"])["status"]
            cand = np.nonzero(st == oracle.REASONING)[0]
            if cand.size:
                pid = int(rng.choice(list(cand)))
                mode = rng.choice((0, 1, 2))
                r0 = [p.pause(pid, mode) for p in pools]
                assert r0[0][0] == r0[1][0], (k, "pause", r0[0][0], r0[1][0])
            cand = np.nonzero(st == oracle.PAUSED)[0]
            if cand.size:
                pid = int(rng.choice(list(cand)))
                r1 = [p.resume(pid, -1) for p in pools]
                assert r1[0][0] == r1[1][0], (k, "resume", r1[0][0], r1[1][0])
        a, b = (p.debug_download(fields) for p in pools)
        for f in fields:
            if not np.array_equal(a[f], b[f]):
                bad = np.argwhere(a[f] != b[f])[:4]
                raise AssertionError(f"tick {k}: {f} differs at {bad.tolist()}")
    for p in pools:
        p.close()


@pytest.mark.gpu
def test_gpu_dirty_rows_equal_full_scan():
    """The footprint pass reads only rows written since its previous pass (DESIGN.md §6,
    dirty rows); with TA_F_FULL_SCAN it counts every live row.  Both give the same
    decisions, derived counts and block tables tick by tick: stress traces with compaction
    and the host tier (R 1 and 3), with pause / resume verbs between ticks, and bench_10k
    (10k programs, mini KV) through its burst."""
    need_gpu()
    _lockstep_full_scan(stress(61, 1, compact=3), 150)
    _lockstep_full_scan(stress(62, 3, compact=2), 150, verbs_seed=7)
    _lockstep_full_scan(tracegen.get_config("bench_10k", kv="mini"), 40)
