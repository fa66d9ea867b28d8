"""NEXT-2 (part): ablation of the detection period Delta t and the decay base x of
f(t) = x^-t (Fig. 7b) on the synthetic engine, through libta on the
GPU (the same kernels the parity tests check against the oracle, including these
parameters: tests/test_gpu_parity.py::test_gpu_policy_parameters).

usage: python tools/ablation.py [--config c2_swe] [--sim-s 2400] [--dts 1000,2500,5000,10000,20000] [--xs 1,2,4,8]

Workload: the config's trace with the decision-identical `mini` KV shape.  Each point
runs sim_s seconds of simulated time (sim_s / Delta t ticks) and reports, per simulated
second: tokens written (decode + tool results, the engine's useful work), the KV hit
rate of resumed programs (hit / (hit + peer + host + miss)), and the STP ledger
(NEXT-1) normalised per simulated second.  One JSON line per point."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def main():
    name = arg("--config", "c2_swe")
    sim_s = int(arg("--sim-s", "2400"))
    dts = [int(v) for v in arg("--dts", "1000,2500,5000,10000,20000").split(",")]
    xs = [int(v) for v in arg("--xs", "1,2,4,8").split(",")]
    for dt in dts:
        for x in xs:
            cfg = tracegen.get_config(name, delta_t_ms=dt, decay_x=x, kv="mini")
            tr = tracegen.make_trace(cfg)
            pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False)
            pool.load_trace(tr)
            ticks = sim_s * 1000 // dt
            for _ in range(ticks):
                pool.step(decisions=False)
            st = pool.stats()
            hist = st["hit_tok"] + st["peer_tok"] + st["host_tok"] + st["miss_tok"]
            out = {"config": name, "delta_t_ms": dt, "decay_x": x, "ticks": ticks, "sim_s": sim_s,
                   "tokens_per_sim_s": round(st["new_tok"] / sim_s, 1),
                   "hit_rate": round(st["hit_tok"] / hist, 4) if hist else None,
                   "no_recompute_rate": round((hist - st["miss_tok"]) / hist, 4) if hist else None,
                   "pauses": st["pauses"], "restores": st["restores"], "stops": st["stops"],
                   "evict_dropped": st["evict_dropped"], "evict_to_host": st["evict_to_host"],
                   "stp_token_s_per_sim_s": {k[5:]: round(st[k] / 1000 / sim_s) for k in
                                             ("cost_decode", "cost_prefill", "cost_recompute", "cost_unused",
                                              "cost_caching")},
                   "unused_bound": [st["unused_bound_checks"], st["unused_bound_violations"]]}
            print(json.dumps(out), flush=True)
            pool.close()


if __name__ == "__main__":
    main()
