"""Small end-to-end driver for compute-sanitizer runs (developer tool, GPU box):
trace-mode ticks with fills and compaction, API-mode batches with multi-event
programs, and every verb (pause/resume/migrate/set_health), each checked against the
oracle.  usage: compute-sanitizer --tool memcheck python tests/sanitize_driver.py"""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool  # noqa: E402
from tests.gpu_compare import dec_tuples  # noqa: E402
from tests.test_gpu_api import random_event_sequences  # noqa: E402


def main():
    cfg = tracegen.get_config("c1_toy", n_replicas=2, hbm_blocks=56, host_blocks=16, compact_every=3,
                              trace=dict(n=24, n_initial=10, seed=12))
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns)
    pool.load_trace(tr)
    rng = random.Random(1)
    for k in range(30):
        _, want = o.sched_step()
        _, got = pool.step()
        assert dec_tuples(got) == want, k
        if k % 5 == 2:
            p = rng.randrange(o.N)
            for fo, fg, args in ((o.pause, pool.pause, (p, 1)), (o.resume, pool.resume, (p, -1)),
                                 (o.migrate, pool.migrate, (p, 1)), (o.set_health, pool.set_health, (1, k % 10 != 2))):
                so, _ = fo(*args)
                sg, _ = fg(*args)
                assert so == sg, (k, fo.__name__, so, sg)
    bad, seen = pool.verify_content()
    assert bad == 0 and seen > 0
    pool.close()
    cfg2 = tracegen.get_config("c1_toy", n_replicas=2, hbm_blocks=48, host_blocks=16, max_ctx=4096)
    o2 = oracle.Oracle(cfg2, api_mode=True, n_slots=32)
    pool2 = Pool(cfg2, 32, trace_mode=False)
    for k in range(30):
        evs = random_event_sequences(o2, rng, 5000 * k)
        so, do = o2.sched_step(5000 * k, evs)
        sg, dg = pool2.step(5000 * k, evs, raise_on_error=False)
        assert so == sg, k
        if so == oracle.OK:
            assert dec_tuples(dg) == do, k
    pool2.close()
    print("sanitize driver OK")


if __name__ == "__main__":
    main()
