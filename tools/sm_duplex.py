"""SM-copy duplex on the host link (developer tool, GPU box): libta's block copies
(ta_move_blocks, the kernels' copy path) D2H alone, H2D alone, and both at once from
two contexts on two streams, against pinned cudaMemcpyAsync (DMA engines) both ways.
Tells how much of the fused movement kernel's loss on mixed ticks is the link itself."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool, binding  # noqa: E402


def main():
    nb = 2048
    cfg = tracegen.get_config("bench_10k", hbm_blocks=2 * nb + 64, host_blocks=2 * nb)
    pa = Pool(cfg, 64, fill=False)
    pb = Pool(cfg, 64, fill=False)
    bb = pa.block_bytes
    rng = np.random.default_rng(3)
    dev = pa.device
    def lists():
        perm = rng.permutation(pa.NB)[:nb].astype(np.int32)
        hs = rng.permutation(pa.NH)[:nb].astype(np.int32)
        return torch.tensor(perm, device=dev), torch.tensor(hs, device=dev)
    (sa, ha), (sb, hb) = lists(), lists()
    def run(moves):
        best = 0.0
        for _ in range(3):
            torch.cuda.synchronize()
            evs = []
            for pool, kind, a, b in moves:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(pool.stream)
                pool.move_blocks(kind, pool.first, pool.first, a, b)
                e1.record(pool.stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            t = max(e0.elapsed_time(e1) for e0, e1 in evs) * 1e-3     # streams start together
            best = max(best, len(moves) * nb * bb / t / 1e9)
        return round(best, 1)
    out = {"block_bytes": bb, "blocks_per_direction": nb,
           "sm_d2h_gbs": run([(pa, binding.MOVE_D2H, sa, ha)]),
           "sm_h2d_gbs": run([(pb, binding.MOVE_H2D, hb, sb)]),
           "sm_duplex_total_gbs": run([(pa, binding.MOVE_D2H, sa, ha), (pb, binding.MOVE_H2D, hb, sb)])}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
