"""NVLink movement inside the product API: ta_migrate of programs between two GPUs
(developer tool, GPU box, 2 ranks).

torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/migrate_nvlink.py [--ticks 12] [--programs 24]

bench_10k tiled over 2 replicas (one per GPU, Qwen3-32B 4 MiB blocks, 96 GiB pools), the
burst window run for `ticks` ticks, then the `programs` REASONING programs of replica 0
with the most HBM blocks are migrated to replica 1 (collective verb on both ranks; the
destination rank pulls the blocks over NVLink from the peer pool).  Each call is timed
with a CUDA event pair on the context stream of every rank (max over ranks); GB/s =
blocks moved x block bytes / time, against the 770 GB/s measured peer copy
(B200_PROFILING.md; 900 nominal).  Both replicas run at lambda = 1, so replica 1's active
programs are first paused with their blocks dropped (ta_pause, TA_PAUSE_DROP) to make
room.  One JSON summary line from rank 0."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool  # noqa: E402
from paper_2602_13692_b200.dist import connect  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def main():
    ticks, nprog = int(arg("--ticks", "12")), int(arg("--programs", "24"))
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = tracegen.get_config("bench_10k")
    cfg["n_replicas"] = world
    cfg["trace"]["tile"] = world
    tr = tracegen.make_trace(cfg)
    host_cap = 24 << 30                                   # pinned host tier per rank (fits the box)
    nh = min(cfg["host_blocks"], host_cap // (64 * 2 * 8 * 128 * 2 * 16))
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False, replicas_here=1, first_replica=rank,
                device=local, host_blocks=nh)
    connect(pool)
    pool.load_trace(tr)
    for _ in range(ticks):
        pool.step(decisions=False)
    torch.cuda.synchronize()
    st = pool.debug_download(["status", "home", "n_hbm", "satisfied", "placement"])
    # make room on replica 1 (both replicas run at lambda = 1): pause its active programs,
    # dropping their blocks (collective verbs; every rank holds the same state)
    for p in range(tr.n_slots):
        if st["placement"][p] == 1 and st["status"][p] in (2, 3):
            pool.pause(p, 2)
    torch.cuda.synchronize()
    cand = [p for p in range(tr.n_slots) if st["status"][p] == 2 and st["home"][p] == 0 and st["placement"][p] == 0
            and st["satisfied"][p] == 1]                  # materialized: every block in HBM (NVLink only)
    cand.sort(key=lambda p: -int(st["n_hbm"][p]))
    cand = cand[:nprog]
    s = pool.stream
    rows = []
    for p in cand:
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        code, dec = pool.migrate(p, 1)
        b.record(s)
        b.synchronize()
        ms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=torch.device("cuda", local))
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        blocks = int(pool.last_tick()["p2p_blocks"]) if code == 0 else 0   # blocks pulled over NVLink
        rows.append((p, code, blocks, float(ms.item())))
    if rank == 0:
        ok = [(p, b, t) for p, c, b, t in rows if c == 0 and b > 0]
        tot_b = sum(b for _, b, _ in ok)
        tot_ms = sum(t for _, _, t in ok)
        bb = pool.block_bytes
        print(json.dumps({"gpus": world, "migrations": len(ok), "blocks": tot_b, "gb": round(tot_b * bb / 1e9, 2),
                          "verb_time_ms": round(tot_ms, 2),
                          "gbs": round(tot_b * bb / (tot_ms * 1e-3) / 1e9, 1) if tot_ms else None,
                          "peak_gbs": 770.0, "frac": round(tot_b * bb / (tot_ms * 1e-3) / 1e9 / 770.0, 3) if tot_ms else None,
                          "per_call": [(p, b, round(t, 3)) for p, b, t in ok[:8]],
                          "note": "ta_migrate end to end on the device (plan, P2P pull, close), max over ranks"}),
              flush=True)
    pool.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
