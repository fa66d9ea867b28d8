"""NEXT-3: what storing the agents' shared system prompt once per replica buys
("the shared prompt across programs implicitly reserves sufficient memory
buffer"), through libta on the GPU (the kernels tests/test_gpu_parity.py::
test_gpu_shared_prefix checks against the oracle).

usage: python tools/shared_prefix_compare.py [--config c2_swe] [--sim-s 2400] [--spts 0,1024,1984]
       python tools/shared_prefix_compare.py --config c3_mixed --per-preset openhands:960,toolorch:640

Each point runs the config's trace (decision-identical `mini` KV shape) for sim_s
seconds of simulated time with shared_prefix_tokens = spt (one prompt for every program),
or with --per-preset one prompt per listed preset (NEXT-3, reading A51: materialized by
the first user on a replica, refcounted, released by the last), and reports per simulated
second the tokens written, the resume hit rate, evictions and recomputed blocks, and
the mean physical HBM occupancy (sampled every 10 ticks).  The load (Eq. 7) counts full
contexts either way, so pause/restore see the same loads; the reserved-once prompt
leaves physical room that keeps idle programs' KV resident longer.  One JSON line per
point."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def main():
    name = arg("--config", "c2_swe")
    sim_s = int(arg("--sim-s", "2400"))
    spts = [int(v) for v in arg("--spts", "0,1024,1984").split(",")]
    points = [("shared_prefix_tokens", spt) for spt in spts]
    if "--per-preset" in sys.argv:                   # no prompt, then one prompt per preset
        spec = [(int(t), pr) for pr, t in (x.split(":") for x in arg("--per-preset", "").split(","))]
        points = [("shared_prefix_tokens", 0), ("shared_prefixes", spec)]
    for key, val in points:
        cfg = tracegen.get_config(name, kv="mini", **{key: val})
        spt = val
        tr = tracegen.make_trace(cfg)
        pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False)
        pool.load_trace(tr)
        ticks = sim_s * 1000 // int(cfg["delta_t_ms"])
        used = []
        for k in range(ticks):
            pool.step(decisions=False)
            if k % 10 == 0:
                hf = pool.debug_download(fields=["hbm_free"])["hbm_free"]
                free = int(np.unpackbits(hf.view(np.uint8)).sum())
                used.append(cfg["n_replicas"] * cfg["hbm_blocks"] - free)
        st = pool.stats()
        hist = st["hit_tok"] + st["peer_tok"] + st["host_tok"] + st["miss_tok"]
        out = {"config": name, key: spt, "ticks": ticks, "sim_s": sim_s,
               "prefix_blocks": st["prefix_blocks"],
               "tokens_per_sim_s": round(st["new_tok"] / sim_s, 1),
               "hit_rate": round(st["hit_tok"] / hist, 4) if hist else None,
               "no_recompute_rate": round((hist - st["miss_tok"]) / hist, 4) if hist else None,
               "pauses": st["pauses"], "restores": st["restores"], "stops": st["stops"],
               "evict_blocks": st["evict_blocks"], "evict_dropped": st["evict_dropped"],
               "recompute_blocks": st["recompute_blocks"], "h2d_blocks": st["h2d_blocks"],
               "mean_used_blocks": round(float(np.mean(used)), 1),
               "pool_blocks": cfg["n_replicas"] * cfg["hbm_blocks"],
               "stp_recompute_token_s_per_sim_s": round(st["cost_recompute"] / 1000 / sim_s)}
        print(json.dumps(out), flush=True)
        pool.close()


if __name__ == "__main__":
    main()
