"""Where the cold-L2 cost of a decision tick comes from (developer tool, GPU box):
code (instruction fetch of the large planner kernels) or data (the context's metadata).

usage: python tools/cold_split.py [--start 13] [--ticks 60] [--decide-only] [--dev]

Four modes per tick of bench_10k (mini KV), each with the 256 MiB L2 flush first:
  cold  : flush, tick
  code  : flush, one tick of a SECOND bench_10k context (same kernels, other data), tick
  data  : flush, a read of this context's device workspace (its metadata), tick
  warm  : no flush
Prints one JSON line with the median tick (us) of each mode."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool, binding  # noqa: E402


# --decide-only: the decision path alone (TA_F_DECIDE_ONLY); --dev: the development build
FLAGS = (binding.F_DECIDE_ONLY if "--decide-only" in sys.argv else 0) | (binding.F_TIMING if "--dev" in sys.argv else 0)


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def main():
    start, n = int(arg("--start", "13")), int(arg("--ticks", "60"))
    cfg = tracegen.get_config("bench_10k")
    cfg["kv"] = "mini"
    tr = tracegen.make_trace(cfg)
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {"config": "bench_10k", "ticks": f"{start}..{start + n - 1}", "flags": FLAGS}
    for mode in ("cold", "code", "data", "warm"):
        a = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False, flags=FLAGS)
        a.load_trace(tr)
        b = None
        if mode == "code":
            b = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False, flags=FLAGS, stream=a.stream)
            b.load_trace(tr)
        for _ in range(start):
            a.step(decisions=False)
            if b is not None:
                b.step(decisions=False)
        s = a.stream
        us = []
        for _ in range(n):
            with torch.cuda.stream(s):
                torch.cuda._sleep(1_000_000)        # host submission ahead of the GPU (bench.py)
                if mode != "warm":
                    flush.zero_()
                if mode == "data":
                    a.dev_ws.view(torch.int32)[: a.dev_ws.numel() // 4].sum()
            if b is not None:
                b.step(decisions=False)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            a.step(decisions=False)
            e1.record(s)
            e1.synchronize()
            us.append(e0.elapsed_time(e1) * 1e3)
        out[mode] = round(float(np.median(us)), 1)
        out[mode + "_ws_mb"] = round(a.dev_ws.numel() / 2**20, 1)
        a.close()
        if b is not None:
            b.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
