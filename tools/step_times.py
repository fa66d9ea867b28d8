"""Per-step device/host timing of the bench workload (developer tool, GPU box).
usage: python tools/step_times.py [--no-fuse] [--ticks N] [--phases] [--no-timing] [--flush] [--mini] [--decide-only]
--flush: 256 MiB memset before every tick (outside the timed pair); --mini: 4 KiB-block KV shape"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool, binding  # noqa: E402

flags = (0 if "--no-timing" in sys.argv else binding.F_TIMING) | (binding.F_NO_FUSE if "--no-fuse" in sys.argv else 0)
flags |= binding.F_DECIDE_ONLY if "--decide-only" in sys.argv else 0
ticks = int(sys.argv[sys.argv.index("--ticks") + 1]) if "--ticks" in sys.argv else 24
cfg = tracegen.get_config("bench_10k")
if "--mini" in sys.argv:
    cfg["kv"] = "mini"
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if "--flush" in sys.argv else None
tr = tracegen.make_trace(cfg)
pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False, flags=flags)
pool.load_trace(tr)
s = pool.stream
prev = pool.stats()
for k in range(ticks):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if flush is not None:
        with torch.cuda.stream(s):
            flush.zero_()
    t0 = time.perf_counter()
    e0.record(s)
    pool.step(decisions=False)
    e1.record(s)
    e1.synchronize()
    t1 = time.perf_counter()
    ph = pool.phase_times() if flags & binding.F_TIMING and not os.environ.get("TA_NO_EVENTS") else [0.0] * 9
    st = pool.stats()
    d2h = st["evict_to_host"] - prev["evict_to_host"]
    h2d = st["h2d_blocks"] - prev["h2d_blocks"]
    prev = st
    print(f"tick {k:3d} dev {e0.elapsed_time(e1):9.4f} ms host {1e3 * (t1 - t0):9.3f} ms  "
          f"move {ph[3] / 1e3:8.2f} ms  d2h {d2h:5d} h2d {h2d:5d} blocks  sched {sum(ph) / 1e3 - ph[3] / 1e3:6.3f} ms",
          flush=True)
    if "--phases" in sys.argv:
        print("   phases us: " + " ".join(f"{x:.1f}" for x in ph))
        st = pool.phase_stamps(absolute=True)       # in-kernel globaltimer stamps (ns), one origin
        print("   spans    : " + "  ".join(f"{n} {b:.1f}-{e:.1f}" for n, b, e in st.pop("spans", [])))
        for kname, v in st.items():
            print(f"   {kname:9s}: " + " ".join(f"{i}:{c / 1e3:.1f}" if isinstance(i, int) else f"{i}={c}"
                                                 for i, c in v))
