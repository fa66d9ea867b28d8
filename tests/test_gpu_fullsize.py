"""GPU parity at full size and on every size branch.

* bench_10k -- the workload bench.py times -- with Qwen3-32B KV (24,576 x 4 MiB HBM
  blocks, 16,384 pinned host slots), ticks 0-40 against the oracle element by element,
  including the eviction-heavy ticks; every owned KV word verified on the GPU and
  sampled blocks on the CPU.
* configs[4] sweep points at block sizes 32 and 64 with 16k and 64k programs (the
  decision-only `mini` KV shape; bytes per block enter no decision), 20 ticks each.
* TA_F_SMALL_PATHS: the size thresholds of the shared-memory fast paths lowered so
  toy-sized traces take every large-size branch (global-memory radix sort, planner
  lists in global memory, sort-ordered F_r, multi-chunk restore), with the per-branch
  counters (ta_debug_counters) asserted > 0; the full-size runs above report theirs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import tracegen  # noqa: E402
from tracegen.configs import sweep_config  # noqa: E402
from tests.test_gpu_parity import need_gpu, run_parity, stress  # noqa: E402


def _record(name, cnt):
    """Size-branch counters of a run, kept as evidence when TA_COUNTERS_DIR is set."""
    import json
    import os
    d = os.environ.get("TA_COUNTERS_DIR")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"{name}.json"), "w") as f:
            json.dump(cnt, f)


def _host_cap_blocks(block_bytes, want):
    """Pinned host tier that fits in half of this box's RAM."""
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal:"):
                return min(want, int(ln.split()[1]) * 1024 // 2 // block_bytes)
    except OSError:
        pass
    return want


def test_gpu_bench10k_q32_ticks_0_40():
    """bench.py's workload at its full size, oracle-checked tick by tick."""
    need_gpu()
    cfg = tracegen.get_config("bench_10k")
    nh = _host_cap_blocks(4 << 20, cfg["host_blocks"])
    cnt = {}
    o, n = run_parity(cfg, 41, state_every=1, content_every=10, samples=3, host_blocks=nh, counters=cnt)
    st = o.stats
    # the window holds the burst's eviction-heavy ticks (D2H to the host tier, drops)
    assert st["evict_blocks"] > 500 and st["evict_to_host"] > 0 and st["h2d_blocks"] > 0, st
    assert cnt["evict_ticks"] > 0, cnt
    _record("bench10k_q32", cnt)


@pytest.mark.parametrize("n,bt", [(16000, 32), (64000, 32), (16000, 64), (64000, 64)])
def test_gpu_configs4_sweep_points(n, bt):
    """configs[4]: 96 GiB of KV per GPU at bt 32 / 64 (NB = 12,288 / 6,144), no host tier,
    16k and 64k programs on one replica; 20 ticks against the oracle."""
    need_gpu()
    point = {16: 0, 32: 7, 64: 14}[bt] + {16000: 4, 64000: 6}[n]
    cfg = sweep_config(n, 1, bt, point)
    cfg["kv"] = "mini"
    cnt = {}
    o, nd = run_parity(cfg, 20, state_every=5, content_every=5, samples=8, counters=cnt)
    assert o.stats["evict_blocks"] > 0 and o.stats["pauses"] > 0 and nd > 0
    _record(f"configs4_{n}_bt{bt}", cnt)


SMALL_RUNS = [
    ("toy R1", dict(seed=91, R=1, NB=80)), ("toy R2", dict(seed=92, R=2, NB=56)),
    ("toy R3", dict(seed=93, R=3, NB=56)), ("toy R4 spt", dict(seed=94, R=4, NB=56, shared_prefix_tokens=32)),
    ("bt1", dict(seed=95, R=2, NB=600, NH=200, block_tokens=1, compact=5)),
    # hundreds of candidates per pass: sorts beyond the lowered limits (radix, bitonic) and
    # planner lists beyond the lowered staging limits
    ("400 programs R2", dict(seed=96, R=2, NB=600, NH=300, n=400, n0=400)),
    ("300 programs R1", dict(seed=97, R=1, NB=900, NH=200, n=300, n0=200)),
]


def test_gpu_small_paths_reach_every_size_branch():
    """TA_F_SMALL_PATHS on stress traces (R 1-4, shared prefix, bt 1), bit-exact vs the
    oracle, and every size-branch counter > 0 over the runs."""
    need_gpu()
    from paper_2602_13692_b200 import binding
    cnt = {}
    for name, kw in SMALL_RUNS:
        kw = dict(kw)
        seed, R = kw.pop("seed"), kw.pop("R")
        run_parity(stress(seed, R, **kw), 250, state_every=3, seed=seed, flags=binding.F_SMALL_PATHS,
                   counters=cnt)
    _record("small_paths", cnt)
    missing = [k for k in binding.DEBUG_COUNTERS if cnt.get(k, 0) == 0]
    assert not missing, (missing, cnt)


def test_gpu_small_paths_api_and_verbs():
    """The API-mode multi-event sort and the verbs' single-program planner under
    TA_F_SMALL_PATHS."""
    need_gpu()
    import random
    from paper_2602_13692_b200 import Pool, binding
    from tests.test_gpu_api import random_event_sequences
    from tests.gpu_compare import compare_state, dec_tuples
    cfg = tracegen.get_config("c1_toy", n_replicas=2, hbm_blocks=48, host_blocks=16, max_ctx=4096,
                              compact_every=3)
    N = 48
    o = oracle.Oracle(cfg, api_mode=True, n_slots=N)
    pool = Pool(cfg, N, trace_mode=False, flags=binding.F_SMALL_PATHS)
    rng = random.Random(31)
    for k in range(120):
        T = 5000 * k
        evs = random_event_sequences(o, rng, T)
        st_o, dec_o = o.sched_step(T, evs)
        st_g, dec_g = pool.step(T, evs, raise_on_error=False)
        assert st_o == st_g, (k, st_o, st_g)
        if st_o == oracle.OK:
            assert dec_tuples(dec_g) == dec_o, f"tick {k}"
        if k % 6 == 0:
            compare_state(o, pool.debug_download(), where=f"tick {k}")
        for _ in range(2):
            q = [p for p in range(N) if o.status[p] == oracle.PAUSED]
            if q:
                p = rng.choice(q)
                st_o, d_o = o.resume(p, -1)
                st_g, d_g = pool.resume(p, -1)
                assert st_o == st_g
                if st_o == oracle.OK:
                    assert dec_tuples(d_g) == d_o
    compare_state(o, pool.debug_download(), where="end")
    bad, _ = pool.verify_content()
    assert bad == 0
    pool.close()
