"""configs[4] scaling sweep of the scheduler tick (developer tool, GPU box).

usage: python tools/sweep.py [--programs 1000,2000,...] [--bt 16,32,64] [--ticks 40] [--preroll 10] [--decide-only]

For each point (N programs, block size bt) of BASELINE.json configs[4] on one GPU
(96 GiB of Qwen3-32B KV per GPU -> NB = 96 GiB / block bytes, no host tier;
tracegen.configs.sweep_config) it runs the full ta_sched_step CUDA graph with the
decision-identical `mini` KV shape (no decision depends on bytes per block) and
reports the per-tick device latency (CUDA events on the context stream, L2 flushed
before every tick).  One JSON line per point."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from tracegen.configs import sweep_config  # noqa: E402
from paper_2602_13692_b200 import Pool, binding  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def main():
    progs = [int(x) for x in arg("--programs", "1000,2000,4000,8000,16000,32000,64000").split(",")]
    bts = [int(x) for x in arg("--bt", "16,32,64").split(",")]
    ticks, preroll = int(arg("--ticks", "40")), int(arg("--preroll", "10"))
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    point = 0
    for bt in bts:
        for n in progs:
            cfg = sweep_config(n, 1, bt, point)
            point += 1
            cfg["kv"] = "mini"
            tr = tracegen.make_trace(cfg)
            pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False,
                        flags=binding.F_DECIDE_ONLY if "--decide-only" in sys.argv else 0)
            pool.load_trace(tr)
            s = pool.stream
            for _ in range(preroll):
                pool.step(decisions=False)
            us = []
            st0 = pool.stats()
            for _ in range(ticks):
                with torch.cuda.stream(s):
                    torch.cuda._sleep(1_000_000)    # host submission ahead of the GPU (bench.py)
                    flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                pool.step(decisions=False)
                b.record(s)
                b.synchronize()
                us.append(a.elapsed_time(b) * 1e3)
            st1 = pool.stats()
            us = np.array(us)
            print(json.dumps({"programs": n, "block_tokens": bt, "hbm_blocks": cfg["hbm_blocks"],
                              "max_blocks_per_program": pool.MAXB,
                              "tick_us_median": round(float(np.median(us)), 1),
                              "tick_us_p99": round(float(np.percentile(us, 99)), 1),
                              "ticks_per_s": round(1e6 / float(np.median(us)), 1),
                              "ticks": f"{preroll}..{preroll + ticks - 1}",
                              "pauses": st1["pauses"] - st0["pauses"], "restores": st1["restores"] - st0["restores"],
                              "evicted_blocks": st1["evict_blocks"] - st0["evict_blocks"],
                              "fetched_blocks": st1["fetch_blocks"] - st0["fetch_blocks"]}), flush=True)
            pool.close()
            del pool
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
