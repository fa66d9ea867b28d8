"""Host-link bandwidth with every GPU of the box copying at once, per copy engine:
the DMA copy engines (pinned cudaMemcpyAsync), and libta's SM-driven block movement
(ta_move_blocks: TMA bulk, and the 128-bit load/store engine), D2H and H2D.

usage: torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/pcie_concurrent.py [--blocks 512]

Each rank owns an independent one-replica pool (Qwen3-32B KV shape, 4 MiB blocks).
For each (engine, direction): rank 0 alone (the others wait), then all ranks together
after a barrier; each rank times its own copies with CUDA events (median of 5).  Rank 0 prints one
JSON line: GB/s per rank, alone and concurrent."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool, binding  # noqa: E402


def main():
    nblk = int(sys.argv[sys.argv.index("--blocks") + 1]) if "--blocks" in sys.argv else 512
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = tracegen.get_config("bench_10k", hbm_blocks=2 * nblk + 64, host_blocks=nblk + 64)
    tr = tracegen.make_trace(tracegen.get_config("c1_toy"))
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False, device=local)
    bb = pool.block_bytes
    rng = np.random.default_rng(rank)
    hbm = torch.tensor(rng.permutation(pool.NB)[:nblk].astype(np.int32), device=dev)
    host = torch.tensor(rng.permutation(pool.NH)[:nblk].astype(np.int32), device=dev)
    nbytes = nblk * bb
    hbuf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dbuf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s = pool.stream

    def run(engine, direction):
        if engine == "dma":
            dst, src = (hbuf, dbuf) if direction == "d2h" else (dbuf, hbuf)
            with torch.cuda.stream(s):
                dst.copy_(src, non_blocking=True)
        else:
            pool.set_copy_bulk(engine == "sm_bulk")
            if direction == "d2h":
                pool.move_blocks(binding.MOVE_D2H, 0, 0, hbm, host)
            else:
                pool.move_blocks(binding.MOVE_H2D, 0, 0, host, hbm)

    def timed(engine, direction, reps=5):
        vals = []                                     # median: every copy overlaps the others'
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            run(engine, direction)
            e1.record(s)
            e1.synchronize()
            vals.append(nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        return sorted(vals)[len(vals) // 2]

    out = {"world": world, "bytes_per_copy": nbytes, "block_bytes": bb}
    for engine in ("dma", "sm_bulk", "sm_ldst"):
        for direction in ("d2h", "h2d"):
            timed(engine, direction, reps=1)          # warm-up
            if world > 1:
                dist.barrier()
            alone = timed(engine, direction) if rank == 0 else 0.0
            if world > 1:
                torch.cuda.synchronize()
                dist.barrier()
            together = timed(engine, direction)
            vals = torch.tensor([alone, together], dtype=torch.float64, device=dev)
            if world > 1:
                allv = [torch.zeros_like(vals) for _ in range(world)]
                dist.all_gather(allv, vals)
            else:
                allv = [vals]
            out[f"{engine}_{direction}"] = {"alone_rank0": round(float(allv[0][0]), 1),
                                            "together": [round(float(v[1]), 1) for v in allv]}
    pool.set_copy_bulk(True)
    if rank == 0:
        print(json.dumps(out), flush=True)
    pool.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
