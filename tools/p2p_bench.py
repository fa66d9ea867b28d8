"""Cross-replica KV block migration over NVLink: libta's P2P copy kernel vs the NCCL
send/recv baseline (BASELINE.json north_star: "cross-replica migration as P2P stores
over NVLink, with NCCL send/recv only as the comparison baseline").

torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2p_bench.py [n_blocks]

Both replicas hold a layer-major Qwen3-32B pool (4 MiB blocks = 128 segments of
32 KiB).  n random source blocks of rank 0 move to n random free blocks of rank 1:
  ours_push  ta_move_blocks(P2P, 0 -> 1) on rank 0: loads from local HBM, stores into
             the peer pool mapped with CUDA IPC (one kernel, NVLink writes)
  ours_pull  ta_move_blocks(P2P, 0 -> 1) on rank 1: loads over NVLink from rank 0's pool
  nccl       rank 0 gathers the blocks into a contiguous buffer (torch index_select),
             dist.send -> dist.recv (NCCL), rank 1 scatters them (torch index_copy_)
  nccl_link  dist.send/recv of one contiguous buffer of the same bytes (link reference)
Bytes are checked after every variant.  Times: CUDA events, max over the two ranks.
Rank 0 prints one JSON line."""
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


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert world == 2
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    cfg = tracegen.get_config("bench_10k", n_replicas=2, hbm_blocks=4 * n, host_blocks=0)
    pool = Pool(cfg, 16, max_turns=1, fill=False, device=rank, replicas_here=1, first_replica=rank)
    connect(pool)
    bb = pool.block_bytes
    nseg = 2 * pool.c.n_layers
    seg = bb // nseg
    rng = np.random.default_rng(3)
    perm0 = rng.permutation(pool.NB)
    perm1 = rng.permutation(pool.NB)
    src = torch.tensor(perm0[:n].astype(np.int32), device=dev)
    dst = torch.tensor(perm1[:n].astype(np.int32), device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(11 + rank)
    pool.hbm[rank].view(torch.int64).random_(generator=g)
    s = pool.stream
    torch.cuda.synchronize(dev)

    def blocks(idx):
        return pool.hbm[rank].view(nseg, pool.NB, seg)[:, idx.long(), :]

    want = blocks(src).clone() if rank == 0 else None
    if rank == 1:
        want = torch.empty(nseg, n, seg, dtype=torch.uint8, device=dev)
        dist.recv(want, src=0)
    else:
        dist.send(want, dst=1)

    def timed(fn, reps=3):
        best = 1e30
        for _ in range(reps):
            dist.barrier()
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            with torch.cuda.stream(s):
                fn()
            b.record(s)
            b.synchronize()
            t = torch.tensor([a.elapsed_time(b)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            best = min(best, float(t.item()))
        return best

    def check():
        ok = torch.tensor([1], device=dev)
        if rank == 1:
            ok[0] = int(torch.equal(blocks(dst), want))
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        return bool(ok.item())

    def scrub():
        if rank == 1:
            blocks_view = pool.hbm[1].view(nseg, pool.NB, seg)
            blocks_view[:, dst.long(), :] = 0
        torch.cuda.synchronize(dev)

    res = {}
    # ours: push from rank 0 (rank 1 idle), pull by rank 1 (rank 0 idle)
    for name, actor in (("ours_push", 0), ("ours_pull", 1)):
        scrub()
        ms = timed(lambda: pool.move_blocks(binding.MOVE_P2P, 0, 1, src, dst) if rank == actor else None)
        res[name] = {"ms": round(ms, 3), "gbs": round(n * bb / (ms * 1e-3) / 1e9, 1), "bytes_ok": check()}
    # NCCL baseline: gather -> send/recv -> scatter
    stage = torch.empty(nseg, n, seg, dtype=torch.uint8, device=dev)

    def nccl_fn():
        if rank == 0:
            torch.index_select(pool.hbm[0].view(nseg, pool.NB, seg), 1, src.long(), out=stage)
            dist.send(stage, dst=1)
        else:
            dist.recv(stage, src=0)
            pool.hbm[1].view(nseg, pool.NB, seg).index_copy_(1, dst.long(), stage)
    scrub()
    ms = timed(nccl_fn)
    res["nccl"] = {"ms": round(ms, 3), "gbs": round(n * bb / (ms * 1e-3) / 1e9, 1), "bytes_ok": check(),
                   "how": "torch index_select gather + dist.send/recv (NCCL) + index_copy_ scatter"}

    def link_fn():
        if rank == 0:
            dist.send(stage, dst=1)
        else:
            dist.recv(stage, src=0)
    ms = timed(link_fn)
    res["nccl_link"] = {"ms": round(ms, 3), "gbs": round(n * bb / (ms * 1e-3) / 1e9, 1),
                        "how": "dist.send/recv of one contiguous buffer of the same bytes"}
    if rank == 0:
        out = {"blocks": n, "block_bytes": bb, "bytes": n * bb, "peak_gbs_nvlink_per_direction": 900,
               "measured_peer_copy_gbs": 770, "results": res,
               "frac_of_770": {k: round(v["gbs"] / 770.0, 3) for k, v in res.items()},
               "ours_vs_nccl": round(res["ours_push"]["gbs"] / res["nccl"]["gbs"], 2)}
        print(json.dumps(out), flush=True)
    dist.barrier()
    pool.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
