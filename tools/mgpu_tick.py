"""Per-rank decision tick in multi-process mode (developer tool, GPU box).

torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mgpu_tick.py [--start 13] [--ticks 60] [--spans]

bench_10k tiled over N replicas (one per GPU, 10k programs each: tracegen.tile_trace),
decision-identical mini KV, L2 flushed before every tick, a device spin first so the
host's submission is ahead (as bench.py).  Each rank times its own tick with a CUDA
event pair; rank 0 prints the median / p90 over ranks' max per tick.  --spans: the
development build's kernel spans on rank 0 (TA_F_TIMING without event nodes)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool, binding  # noqa: E402
from paper_2602_13692_b200.dist import connect  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def main():
    start, n = int(arg("--start", "13")), int(arg("--ticks", "60"))
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = tracegen.get_config("bench_10k")
    cfg["kv"] = "mini"
    cfg["n_replicas"] = world
    cfg["trace"]["tile"] = world
    tr = tracegen.make_trace(cfg)
    spans = "--spans" in sys.argv
    if spans:
        os.environ["TA_NO_EVENTS"] = "1"
    flags = binding.F_TIMING if spans else 0
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False, replicas_here=1, first_replica=rank,
                device=local, flags=flags)
    connect(pool)
    pool.load_trace(tr)
    dev = torch.device("cuda", local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    s = pool.stream
    for _ in range(start):
        pool.step(decisions=False)
    torch.cuda.synchronize(dev)
    us, sp = [], []
    for _ in range(n):
        dist.barrier()
        with torch.cuda.stream(s):
            torch.cuda._sleep(1_000_000)
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        pool.step(decisions=False)
        b.record(s)
        b.synchronize()
        us.append(a.elapsed_time(b) * 1e3)
        if spans and rank == 0:
            sp.append(pool.phase_stamps(absolute=True).get("spans", []))
    t = torch.tensor(us, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    m = t.cpu().numpy()
    if rank == 0:
        out = {"gpus": world, "programs_per_gpu": tr.n_slots // world, "ticks": f"{start}..{start + n - 1}",
               "tick_us_median": round(float(np.median(m)), 1), "tick_us_p90": round(float(np.percentile(m, 90)), 1),
               "tick_us_mean": round(float(m.mean()), 1), "build": "dev" if spans else "product"}
        if sp:
            acc = {}
            for row in sp:
                for nm, b0, e0 in row:
                    acc.setdefault(nm, []).append((b0, e0))
            out["spans_median"] = {nm: [round(float(np.median([x[0] for x in v])), 1),
                                        round(float(np.median([x[1] for x in v])), 1)] for nm, v in acc.items()}
        print(json.dumps(out), flush=True)
    pool.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
