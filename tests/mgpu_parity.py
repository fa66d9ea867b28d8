"""Multi-GPU parity (one replica per GPU, CUDA-IPC P2P, device barriers) vs the oracle.

torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_parity.py [ticks] [--verbs] [--api]
    [--shared TOKENS] [--c3] [--prompts2]
Every rank runs the replicated control plane for all N replicas and moves only its
own replica's bytes; every rank compares its decisions and full state with its own
oracle copy, and verifies the KV content of its local pool.  --api: the same ticks in
API mode (the engine's recorded events, tools/api_events.py) against the trace-mode
oracle.  --shared: NEXT-3 shared system prompt of TOKENS tokens (reserved blocks on
every GPU).  --c3: configs[2] (2k programs) with one replica per GPU, decision-only KV
shape.  --prompts2: two shared prompts, one per agent label (NEXT-3, A51).  Exit code 0 =
parity."""
import os
import random
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool  # noqa: E402
from paper_2602_13692_b200.dist import connect  # noqa: E402
from tests.gpu_compare import compare_state, dec_tuples  # noqa: E402


def main():
    ticks = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 150
    verbs = "--verbs" in sys.argv
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spt = int(sys.argv[sys.argv.index("--shared") + 1]) if "--shared" in sys.argv else 0
    if "--c3" in sys.argv:    # configs[2]'s 2k OpenHands + ToolOrchestra programs, one replica per GPU,
        cfg = tracegen.get_config("c3_mixed", kv="mini", n_replicas=world, compact_every=4)   # decision-only KV
        if "--prompts2" in sys.argv:                   # one shared prompt per preset (NEXT-3, A51)
            cfg["shared_prefixes"] = [(960, "openhands"), (640, "toolorch")]
    else:
        cfg = tracegen.get_config("c1_toy", n_replicas=world, hbm_blocks=64, host_blocks=16, compact_every=3,
                                  trace=dict(n=12 * world, n_initial=5 * world, seed=77),
                                  shared_prefix_tokens=spt)
        if "--prompts2" in sys.argv:                   # two shared prompts, alternating labels (A51)
            cfg["trace"]["labels"] = ["a", "b"]
            cfg["shared_prefixes"] = [(48, "a"), (32, "b")]
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    api = "--api" in sys.argv
    batches = None
    if api:   # the engine's events of this trace, recorded on this rank's GPU (all replicas local)
        from tools.api_events import record
        rc = dict(cfg)
        rc["kv"] = "mini"
        batches, _ = record(rc, tr, ticks, device=local)
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, replicas_here=1, first_replica=rank, device=local,
                trace_mode=not api)
    peers = connect(pool)
    if not api:
        pool.load_trace(tr)
    rng = random.Random(5)
    n_dec = n_p2p = n_verbs = 0
    for k in range(ticks):
        _, want = o.sched_step()
        st, got = pool.step(k * cfg["delta_t_ms"], batches[k]) if api else pool.step()
        assert st == 0, f"rank {rank} tick {k}: status {st}"
        got = dec_tuples(got)
        assert got == want, f"rank {rank} tick {k}: decisions differ"
        n_dec += len(got)
        if not api and (k % 4 == 0 or "--c3" not in sys.argv):   # API mode: decisions + bytes only
            compare_state(o, pool.debug_download(), where=f"rank {rank} tick {k}")
        bad, seen = pool.verify_content()
        assert bad == 0, f"rank {rank} tick {k}: {bad} of {seen} local KV words wrong"
        if verbs and k % 3 == 1:          # collective verbs: same call on every rank
            p = rng.randrange(o.N)
            rep = rng.randrange(world)
            for name, fo, fg, args in (("migrate", o.migrate, pool.migrate, (p, rep)),
                                       ("resume", o.resume, pool.resume, (p, rep)),
                                       ("pause", o.pause, pool.pause, (p, 1))):
                so, do = fo(*args)
                sg, dg = fg(*args)
                assert so == sg, (rank, k, name, so, sg)
                if so == oracle.OK:
                    assert dec_tuples(dg) == do, (rank, k, name)
                    n_verbs += 1
                compare_state(o, pool.debug_download(), where=f"rank {rank} tick {k} {name}")
        if o.next_arrival == o.N and all(s == oracle.STOPPED for s in o.status):
            break
    n_p2p = o.stats["p2p_blocks"]
    s = pool.stats()
    for key in oracle.ta_oracle.STAT_KEYS:
        assert s[key] == o.stats[key], (rank, key, s[key], o.stats[key])
    dist.barrier()
    print(f"rank {rank}: OK peers={peers} ticks={k + 1} decisions={n_dec} p2p_blocks={n_p2p} "
          f"h2d_blocks={o.stats['h2d_blocks']} verbs_ok={n_verbs}", flush=True)
    pool.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
