"""NEXT-2 baselines on heavy-tailed tool traces (SPEC.md acceptance 6, Fig. 4c/4f
regime: "program-aware steps/min > TtlPin even when TtlPin's hit rate is higher ...
inflates Cost_caching"), through libta on the GPU.

usage: python tools/baseline_compare.py [--programs 256] [--sim-s 2400] [--seeds 2]

Policies (same kernels; parity of each vs the oracle in tests/test_gpu_parity.py):
  program_aware  f(t) = 2^-t
  request_aware  stateless request-level engine (latest-first preemption, FCFS, LRU; A46)
  ttl_pin_p50    f = 1 for t < 2 s (the ToolOrchestra tool-latency median), 0 after
  ttl_pin_p95    f = 1 for t < 33 s (the p95: pins long)
  no_decay       f = 1 (eq. 6: acting programs always count in full)
Workload: ToolOrchestra-shaped programs (heavy-tailed tool latency),
one replica of configs[1]'s pool (24,576 blocks), mini KV shape (decision-identical)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen  # noqa: E402
from tracegen.configs import ttl_pin_table  # noqa: E402
from paper_2602_13692_b200 import Pool  # noqa: E402


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


POLICIES = {"program_aware": dict(decay_x=2), "request_aware": dict(request_aware=True),
            "ttl_pin_p50": dict(decay_table=ttl_pin_table(2)),
            "ttl_pin_p95": dict(decay_table=ttl_pin_table(33)), "no_decay": dict(decay_x=1)}


def main():
    n = int(arg("--programs", "256"))
    sim_s = int(arg("--sim-s", "2400"))
    for seed in range(int(arg("--seeds", "2"))):
        row = {"programs": n, "sim_s": sim_s, "seed": 6000 + seed}
        for name, over in POLICIES.items():
            cfg = tracegen.get_config("c2_swe", kv="mini", trace=dict(mix=["toolorch"], n=n, seed=6000 + seed),
                                      **over)
            tr = tracegen.make_trace(cfg)
            pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False)
            pool.load_trace(tr)
            for _ in range(sim_s * 1000 // cfg["delta_t_ms"]):
                pool.step(decisions=False)
            st = pool.stats()
            pool.close()
            hist = st["hit_tok"] + st["peer_tok"] + st["host_tok"] + st["miss_tok"]
            row[name] = {"tokens_per_sim_s": round(st["new_tok"] / sim_s, 1), "stops": st["stops"],
                         "hit_rate": round(st["hit_tok"] / hist, 4) if hist else None,
                         "caching_token_s_per_s": round(st["cost_caching"] / 1000 / sim_s),
                         "recompute_token_s_per_s": round(st["cost_recompute"] / 1000 / sim_s)}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
