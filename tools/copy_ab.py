"""A/B the two copy engines (128-bit LDG/STG vs TMA cp.async.bulk) on every path,
checking bytes (developer tool, GPU box).  usage: python tools/copy_ab.py [n_blocks]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool, binding  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = tracegen.get_config("bench_10k", hbm_blocks=8192, host_blocks=4096)
pool = Pool(cfg, 16, max_turns=1, fill=False)
dev = pool.device
bb = pool.block_bytes
rng = np.random.default_rng(0)
g = torch.Generator(device=dev)
g.manual_seed(0)
pool.hbm[0].view(torch.int64).random_(generator=g)
pool.host[0].view(torch.int64)[:].copy_(torch.randint(0, 2**62, (pool.host[0].numel() // 8,)))
perm = rng.permutation(pool.NB)
src = torch.tensor(perm[:n].astype(np.int32), device=dev)
dst = torch.tensor(perm[n:2 * n].astype(np.int32), device=dev)
hs = torch.tensor(rng.permutation(pool.NH)[:n].astype(np.int32), device=dev)
out = {}
nseg = 2 * pool.c.n_layers
seg = bb // nseg


def blocks(buf, nblk, idx):
    v = buf.view(nseg, nblk, seg)
    return v[:, idx.long(), :]


for bulk in (False, True):
    pool.set_copy_bulk(bulk)
    for name, kind, a, b, per in (("d2d", binding.MOVE_D2D, src, dst, 2 * bb),
                                  ("d2h", binding.MOVE_D2H, src, hs, bb),
                                  ("h2d", binding.MOVE_H2D, hs, dst, bb)):
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(pool.stream)
            pool.move_blocks(kind, 0, 0, a, b)
            e1.record(pool.stream)
            e1.synchronize()
            best = max(best, n * per / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        # byte check of the last copy
        s_buf, s_n = (pool.host[0], pool.NH) if kind == binding.MOVE_H2D else (pool.hbm[0], pool.NB)
        d_buf, d_n = (pool.host[0], pool.NH) if kind == binding.MOVE_D2H else (pool.hbm[0], pool.NB)
        want = blocks(s_buf.to(dev) if s_buf.device.type == "cpu" else s_buf, s_n, a.cpu() if s_buf.device.type == "cpu" else a)
        got = blocks(d_buf.to(dev) if d_buf.device.type == "cpu" else d_buf, d_n, b.cpu() if d_buf.device.type == "cpu" else b)
        ok = bool(torch.equal(want.to(dev), got.to(dev)))
        out[f"{name}_{'bulk' if bulk else 'ldst'}"] = {"gbs": round(best, 1), "bytes_ok": ok}
        print(name, "bulk" if bulk else "ldst", round(best, 1), "GB/s", "ok" if ok else "MISMATCH", flush=True)
print(json.dumps(out))
