"""NEXT-4 guard: the periodic monitor at Delta t down to one decode step (SURVEY.md 8(f)
"Delta t -> one decode step"), through libta on the GPU.

usage: python tools/decode_step_guard.py [--config bench_10k] [--sim-s 60] [--dts 5000,1000,250,25]

For each Delta t: sim_s seconds of simulated time on the config's trace (mini KV shape,
decision-identical), reporting the device time of one tick (CUDA events on the pool's
stream, median; what a guard at that period costs: tick / Delta t), the excess the
monitor found (overshoot_blocks per simulated second, overshoot_max_blocks) and the
resume hit rate.  One JSON line per point."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def main():
    name = arg("--config", "bench_10k")
    sim_s = int(arg("--sim-s", "60"))
    dts = [int(v) for v in arg("--dts", "5000,1000,250,25").split(",")]
    for dt in dts:
        cfg = tracegen.get_config(name, kv="mini", delta_t_ms=dt)
        tr = tracegen.make_trace(cfg)
        pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False)
        pool.load_trace(tr)
        ticks = sim_s * 1000 // dt
        times = []
        for k in range(ticks):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(pool.stream)
            pool.step(decisions=False)
            e1.record(pool.stream)
            e1.synchronize()
            if k >= 5:
                times.append(e0.elapsed_time(e1) * 1000.0)
        st = pool.stats()
        hist = st["hit_tok"] + st["peer_tok"] + st["host_tok"] + st["miss_tok"]
        tick_us = float(np.median(times))
        out = {"config": name, "programs": tr.n_slots, "delta_t_ms": dt, "ticks": ticks, "sim_s": sim_s,
               "tick_us_median": round(tick_us, 1), "tick_us_p99": round(float(np.percentile(times, 99)), 1),
               "guard_overhead": round(tick_us / (dt * 1000.0), 5),
               "overshoot_blocks_per_sim_s": round(st["overshoot_blocks"] / sim_s, 1),
               "overshoot_max_blocks": st["overshoot_max_blocks"],
               "pauses": st["pauses"], "restores": st["restores"],
               "hit_rate": round(st["hit_tok"] / hist, 4) if hist else None,
               "tokens_per_sim_s": round(st["new_tok"] / sim_s, 1),
               "note": "tick timed with warm L2 (back-to-back ticks); movement bytes ~0 (mini KV)"}
        print(json.dumps(out), flush=True)
        pool.close()


if __name__ == "__main__":
    main()
