"""NEXT-2 baseline comparison: the global program-aware queue vs PinnedRouting
(per-replica queues) on heterogeneous-lifetime traces (SPEC.md acceptance 8, PAPER.md
Fig. 2a: "Max memory imbalance can achieve 51%"), through libta on the GPU.

usage: python tools/imbalance_compare.py [--replicas 2] [--programs 400] [--ticks 400] [--seeds 3]

Workload: 50% OpenHands / 50% ToolOrchestra programs (heavy-tailed tool latencies),
configs[2]-shaped replicas with the decision-identical `mini` KV shape.  Per tick the
HBM imbalance max_r used - min_r used (blocks) is read from ta_stats; reported: the
fraction of ticks where the global queue's imbalance is below the pinned one (<=, and
strictly), mean and max imbalance as a fraction of a replica's pool, tokens written per
simulated second, unused STP.  One JSON line per seed."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def run(cfg, tr, ticks):
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False)
    pool.load_trace(tr)
    imb = []
    for _ in range(ticks):
        pool.step(decisions=False)
        imb.append(pool.stats()["imbalance_last_blocks"])
    st = pool.stats()
    pool.close()
    return imb, st


def main():
    R = int(arg("--replicas", "2"))
    n = int(arg("--programs", "400"))
    ticks = int(arg("--ticks", "400"))
    for seed in range(int(arg("--seeds", "3"))):
        cfg = tracegen.get_config("c3_mixed", n_replicas=R, kv="mini", hbm_blocks=12288, host_blocks=4096,
                                  trace=dict(n=n, seed=5000 + seed))
        tr = tracegen.make_trace(cfg)
        ig, sg = run(cfg, tr, ticks)
        ip, sp = run(dict(cfg, pinned_routing=True), tr, ticks)
        NB = cfg["hbm_blocks"]
        sim_s = ticks * cfg["delta_t_ms"] / 1000
        print(json.dumps({
            "replicas": R, "programs": n, "ticks": ticks, "seed": 5000 + seed,
            "frac_ticks_global_le_pinned": round(sum(a <= b for a, b in zip(ig, ip)) / ticks, 3),
            "frac_ticks_global_lt_pinned": round(sum(a < b for a, b in zip(ig, ip)) / ticks, 3),
            "mean_imbalance_frac": {"global": round(sum(ig) / ticks / NB, 4), "pinned": round(sum(ip) / ticks / NB, 4)},
            "max_imbalance_frac": {"global": round(max(ig) / NB, 4), "pinned": round(max(ip) / NB, 4)},
            "tokens_per_sim_s": {"global": round(sg["new_tok"] / sim_s, 1), "pinned": round(sp["new_tok"] / sim_s, 1)},
            "unused_stp_token_s": {"global": sg["cost_unused"] // 1000, "pinned": sp["cost_unused"] // 1000},
            "hit_rate": {k: round(s["hit_tok"] / max(1, s["hit_tok"] + s["peer_tok"] + s["host_tok"] + s["miss_tok"]), 4)
                         for k, s in (("global", sg), ("pinned", sp))},
        }), flush=True)


if __name__ == "__main__":
    main()
