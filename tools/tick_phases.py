"""Per-kernel device times of the decision path (developer tool, GPU box).

usage: python tools/tick_phases.py [--config bench_10k] [--start 13] [--ticks 100] [--tile R] [--decide-only]

Runs the full ta_sched_step graph with TA_F_TIMING on the decision-identical `mini` KV
shape (no decision depends on bytes per block), the L2 flushed before every tick, and
prints one JSON line: median / p90 of each phase (ta_phase_times) and of the whole
tick (a separate event pair, no timing nodes).  TA_LIB selects a library variant."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool, binding  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def main():
    name, start, n = arg("--config", "bench_10k"), int(arg("--start", "13")), int(arg("--ticks", "100"))
    cfg = tracegen.get_config(name)
    cfg["kv"] = "mini"
    tile = int(arg("--tile", "1"))            # R replicas on this GPU over R copies of the trace
    if tile > 1:
        cfg["n_replicas"] = tile
        cfg["trace"]["tile"] = tile
    tr = tracegen.make_trace(cfg)
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {"lib": os.environ.get("TA_LIB", "libta.so"), "config": name, "replicas": tile, "programs": tr.n_slots,
           "ticks": f"{start}..{start + n - 1}"}
    for mode in ("timing", "plain"):
        extra = binding.F_DECIDE_ONLY if "--decide-only" in sys.argv else 0
        pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False,
                    flags=(binding.F_TIMING if mode == "timing" else 0) | extra)
        pool.load_trace(tr)
        s = pool.stream
        for _ in range(start):
            pool.step(decisions=False)
        rows = []
        for _ in range(n):
            with torch.cuda.stream(s):
                torch.cuda._sleep(1_000_000)        # host submission ahead of the GPU (bench.py)
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            pool.step(decisions=False)
            b.record(s)
            b.synchronize()
            rows.append([a.elapsed_time(b) * 1e3] + (pool.phase_times() if mode == "timing" else []))
        rows = np.array(rows)
        if mode == "timing":
            names = ["front", "pause_restore", "plan", "move", "-", "-", "close", "compact", "-"]
            for i, nm in enumerate(names):
                if nm != "-":
                    out[nm] = [round(float(np.median(rows[:, i + 1])), 1), round(float(np.percentile(rows[:, i + 1], 90)), 1)]
        else:
            out["tick_us"] = [round(float(np.median(rows[:, 0])), 1), round(float(np.percentile(rows[:, 0], 99)), 1),
                              round(float(rows[:, 0].mean()), 1)]
        pool.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
