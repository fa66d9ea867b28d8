"""Cross-replica KV block migration over NVLink: libta's P2P copy kernel vs the NCCL
send/recv baseline (BASELINE.json north_star: "cross-replica migration as P2P stores
over NVLink, with NCCL send/recv only as the comparison baseline").

torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2p_bench.py [n_blocks] [layout]

Both replicas hold a Qwen3-32B pool (4 MiB blocks = 128 segments of 32 KiB); layout 0
is layer-major (a block's 128 segments are 32 KiB pieces NB*32 KiB apart, vLLM-like),
layout 1 block-major (a block is one contiguous 4 MiB range).  n random source blocks
of rank 0 move to n random free blocks of rank 1:
  ours_push   ta_move_blocks(P2P, 0 -> 1) on rank 0: loads from local HBM, stores into
              the peer pool mapped with CUDA IPC (one kernel, NVLink writes)
  ours_pull   ta_move_blocks(P2P, 0 -> 1) on rank 1: loads over NVLink from rank 0's pool
  nccl_p2p    the fair NCCL baseline: grouped ncclSend / ncclRecv
              (torch batch_isend_irecv) straight from the source pool into the
              destination pool, no staging: one send/recv pair per contiguous piece --
              per 4 MiB block in layout 1, per 32 KiB segment in layout 0 (groups of
              4096 pairs)
  nccl_staged rank 0 gathers the blocks into a contiguous buffer (torch index_select),
              dist.send -> dist.recv, rank 1 scatters them (torch index_copy_)
  nccl_link   dist.send/recv of one contiguous buffer of the same bytes (link reference)
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
    layout = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert world == 2
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    cfg = tracegen.get_config("bench_10k", n_replicas=2, hbm_blocks=4 * n, host_blocks=0, layout=layout)
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

    def pool_view():                      # [nseg, NB, seg] whatever the layout
        v = pool.hbm[rank]
        return v.view(nseg, pool.NB, seg) if layout == 0 else v.view(pool.NB, nseg, seg).transpose(0, 1)

    def blocks(idx):
        return pool_view()[:, idx.long(), :]

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
            pool_view()[:, dst.long(), :] = 0
        torch.cuda.synchronize(dev)

    res = {}
    # ours: push from rank 0 (rank 1 idle), pull by rank 1 (rank 0 idle)
    for name, actor in (("ours_push", 0), ("ours_pull", 1)):
        scrub()
        ms = timed(lambda: pool.move_blocks(binding.MOVE_P2P, 0, 1, src, dst) if rank == actor else None)
        res[name] = {"ms": round(ms, 3), "gbs": round(n * bb / (ms * 1e-3) / 1e9, 1), "bytes_ok": check()}
    # the fair NCCL baseline: grouped send/recv of every contiguous piece, pool to pool
    src_l, dst_l = src.tolist(), dst.tolist()
    if layout == 1:
        flat = pool.hbm[rank].view(pool.NB, bb)
        pieces = [flat[b] for b in (src_l if rank == 0 else dst_l)]
    else:
        lv = pool.hbm[rank].view(nseg, pool.NB, seg)
        pieces = [lv[q, b] for b in (src_l if rank == 0 else dst_l) for q in range(nseg)]
    GROUP = 4096

    def nccl_p2p_fn():
        for i in range(0, len(pieces), GROUP):
            ops = [dist.P2POp(dist.isend if rank == 0 else dist.irecv, t, 1 - rank) for t in pieces[i:i + GROUP]]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
    scrub()
    nccl_p2p_fn()                               # NCCL's first grouped call sets up its P2P channels
    scrub()
    ms = timed(nccl_p2p_fn)
    res["nccl_p2p"] = {"ms": round(ms, 3), "gbs": round(n * bb / (ms * 1e-3) / 1e9, 1), "bytes_ok": check(),
                       "pieces": len(pieces), "piece_bytes": bb if layout == 1 else seg,
                       "how": "torch batch_isend_irecv (ncclGroupStart, ncclSend/ncclRecv per contiguous piece, "
                              f"ncclGroupEnd; groups of {GROUP}), pool to pool, no staging"}
    # NCCL with staging: gather -> send/recv -> scatter
    stage = torch.empty(nseg, n, seg, dtype=torch.uint8, device=dev)

    def nccl_fn():
        if rank == 0:
            stage.copy_(blocks(src))
            dist.send(stage, dst=1)
        else:
            dist.recv(stage, src=0)
            pool_view()[:, dst.long(), :] = stage
    scrub()
    ms = timed(nccl_fn)
    res["nccl_staged"] = {"ms": round(ms, 3), "gbs": round(n * bb / (ms * 1e-3) / 1e9, 1), "bytes_ok": check(),
                          "how": "torch gather into a contiguous buffer + dist.send/recv (NCCL) + scatter"}

    def link_fn():
        if rank == 0:
            dist.send(stage, dst=1)
        else:
            dist.recv(stage, src=0)
    ms = timed(link_fn)
    res["nccl_link"] = {"ms": round(ms, 3), "gbs": round(n * bb / (ms * 1e-3) / 1e9, 1),
                        "how": "dist.send/recv of one contiguous buffer of the same bytes"}
    if rank == 0:
        out = {"blocks": n, "layout": "layer-major" if layout == 0 else "block-major", "block_bytes": bb,
               "bytes": n * bb, "peak_gbs_nvlink_per_direction": 900,
               "measured_peer_copy_gbs": 770, "results": res,
               "frac_of_900": {k: round(v["gbs"] / 900.0, 3) for k, v in res.items()},
               "frac_of_770": {k: round(v["gbs"] / 770.0, 3) for k, v in res.items()},
               "ours_push_vs_nccl_p2p": round(res["ours_push"]["gbs"] / res["nccl_p2p"]["gbs"], 2),
               "ours_pull_vs_nccl_p2p": round(res["ours_pull"]["gbs"] / res["nccl_p2p"]["gbs"], 2)}
        print(json.dumps(out), flush=True)
    dist.barrier()
    pool.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
