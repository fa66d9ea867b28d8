"""In-trace D2D: two-finger compaction of full-size KV blocks inside a real trace
(developer tool, GPU box, VERDICT r1 "turn compaction on in one timed
window").

usage: python tools/compaction_trace.py [--config c2_swe] [--every 4] [--ticks 540]

configs[1] (SWE-Agent shape, 256 programs, Qwen3-32B 4 MiB blocks, one 96 GiB pool) is
run with compaction every `every` ticks.  bench_10k's pool stays full (closed-loop
arrivals keep every block in use, so compaction finds no hole); configs[1] drains once
its programs have all arrived, and its compaction ticks move thousands of blocks.  For
every compaction tick: blocks moved, the k_copy_compact time (TA_F_TIMING event pair
around it) and GB/s read + write against the measured HBM peak.  One JSON line per
compaction tick, then a summary line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool, binding  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def hbm_peak():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p)).get("hbm_gbs", 6549.1))
    except (OSError, ValueError):
        return 6549.1


def main():
    name, every, ticks = arg("--config", "c2_swe"), int(arg("--every", "4")), int(arg("--ticks", "540"))
    cfg = tracegen.get_config(name)
    cfg["compact_every"] = every
    tr = tracegen.make_trace(cfg)
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=True, flags=binding.F_TIMING)
    pool.load_trace(tr)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=pool.device)
    peak = hbm_peak()
    tot_b, tot_us, n, bad, seen = 0, 0.0, 0, 0, 0
    for k in range(ticks):
        with torch.cuda.stream(pool.stream):
            flush.zero_()
        pool.step(decisions=False)
        ph = pool.phase_times()
        ti = pool.last_tick()
        if ti["d2d_blocks"]:
            b = ti["d2d_blocks"]
            by = 2.0 * b * pool.block_bytes
            gbs = by / (ph[7] * 1e-6) / 1e9
            print(json.dumps({"tick": k, "blocks": b, "gb_rw": round(by / 1e9, 3), "kernel_us": round(ph[7], 1),
                              "gbs_rw": round(gbs, 1), "frac_hbm": round(gbs / peak, 4)}), flush=True)
            tot_b += b
            tot_us += ph[7]
            n += 1
            vb, vs = pool.verify_content()       # every owned KV word after the moves
            bad += vb
            seen += vs
    by = 2.0 * tot_b * pool.block_bytes
    print(json.dumps({"summary": True, "config": name, "compact_every": every, "ticks": ticks,
                      "compaction_ticks": n, "blocks": tot_b, "gb_rw": round(by / 1e9, 3),
                      "kernel_s": round(tot_us * 1e-6, 6),
                      "gbs_rw": round(by / (tot_us * 1e-6) / 1e9, 1) if tot_us else None,
                      "peak_gbs": peak, "frac_hbm": round(by / (tot_us * 1e-6) / 1e9 / peak, 4) if tot_us else None,
                      "bytes_verified_bad_words": bad, "words_checked": seen,
                      "block_bytes": pool.block_bytes}), flush=True)
    pool.close()


if __name__ == "__main__":
    main()
