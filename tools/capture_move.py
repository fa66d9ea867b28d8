"""Run bench_10k (Q32 KV, 64 GiB pinned host tier) for ticks 0..K and print, per tick, the
movement kernel's algorithmic bytes (ta_last_tick telemetry: blocks per path x block
bytes) as JSON lines -- the denominator of the DRAM-traffic ratio of an ncu capture of
the same launch (developer tool, GPU box):

  ncu --set full -k regex:k_move_fused -s 2 -c 1 -o move python tools/capture_move.py 2
  -> launch index 2 = tick 2; ratio = (dram__bytes_read + dram__bytes_write) / bytes"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool  # noqa: E402


def main():
    last = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    cfg = tracegen.get_config("bench_10k")
    tr = tracegen.make_trace(cfg)
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False, flags=0)
    pool.load_trace(tr)
    for k in range(last + 1):
        pool.step(decisions=False)
        ti = pool.last_tick()
        bb = pool.block_bytes
        print(json.dumps({"tick": k, "d2h_blocks": ti["d2h_blocks"], "h2d_blocks": ti["h2d_blocks"],
                          "p2p_blocks": ti["p2p_blocks"],
                          "algorithmic_bytes": (ti["d2h_blocks"] + ti["h2d_blocks"] + ti["p2p_blocks"]) * bb,
                          "note": "D2H: read from HBM; H2D: written to HBM (1 block_bytes of DRAM each)"}),
              flush=True)
    torch.cuda.synchronize()
    pool.close()


if __name__ == "__main__":
    main()
