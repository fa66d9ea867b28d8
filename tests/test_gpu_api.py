"""GPU parity of the API-mode event path and of the explicit verbs (ta_pause /
ta_resume / ta_migrate) against the oracle, on random legal and illegal inputs."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import tracegen  # noqa: E402
from tests.gpu_compare import compare_state, dec_tuples, same_decisions  # noqa: E402
from tests.test_gpu_parity import need_gpu, stress  # noqa: E402

A, DEC, TC, TR, REL = (oracle.E_ARRIVE, oracle.E_DECODE, oracle.E_TOOL_CALL, oracle.E_TOOL_RESULT,
                       oracle.E_RELEASE)


def random_events(o, rng, T, n_max=12, illegal_p=0.1):
    """Events that are legal for the oracle's current state (plus, sometimes, one illegal)."""
    evs = []
    used = set()
    for _ in range(rng.randint(0, n_max)):
        p = rng.randrange(o.N)
        if p in used:
            continue
        st, ph = o.status[p], o.phase[p]
        if st == oracle.UNARRIVED:
            evs.append((A, p, 1000 + p, rng.randint(1, 400), 0))
        elif st == oracle.REASONING:
            r = rng.random()
            if r < 0.5:
                evs.append((DEC, p, 0, rng.randint(1, 200), 0))
            elif r < 0.9:
                evs.append((TC, p, 0, 0, max(0, T - rng.randint(0, 9000))))
            else:
                evs.append((REL, p, 0, 0, 0))
        elif ph == oracle.PHASE_A and st in (oracle.ACTING, oracle.PAUSED):
            evs.append((TR, p, 0, rng.randint(0, 300), 0) if rng.random() < 0.8 else (REL, p, 0, 0, 0))
        elif st == oracle.STOPPED and rng.random() < 0.2:
            evs.append((REL, p, 0, 0, 0))      # idempotent
        used.add(p)
    if rng.random() < illegal_p and evs:
        p = evs[0][1]
        evs.append((DEC, p, 0, 1, 0) if o.status[p] != oracle.REASONING else (A, p, 1, 1, 0))
    return evs


@pytest.mark.parametrize("seed,R,spt", [(1, 1, 0), (2, 2, 0), (3, 3, 0), (4, 2, 32)])
def test_gpu_api_mode_events(seed, R, spt):
    """spt > 0: NEXT-3 shared prefix (arrivals shorter than it are rejected batches)."""
    need_gpu()
    from paper_2602_13692_b200 import Pool
    cfg = tracegen.get_config("c1_toy", n_replicas=R, hbm_blocks=48, host_blocks=16, max_ctx=4096,
                              compact_every=4, shared_prefix_tokens=spt)
    N = 40
    o = oracle.Oracle(cfg, api_mode=True, n_slots=N)
    pool = Pool(cfg, N, trace_mode=False)
    rng = random.Random(seed)
    errs = 0
    for k in range(120):
        T = 5000 * k
        evs = random_events(o, rng, T)
        st_o, dec_o = o.sched_step(T, evs)
        st_g, dec_g = pool.step(T, evs, raise_on_error=False)
        assert st_o == st_g, (k, st_o, st_g, evs)
        if st_o != oracle.OK:
            errs += 1
            continue
        same_decisions(dec_g, dec_o, f"tick {k}")
        if k % 5 == 0:
            compare_state(o, pool.debug_download(), where=f"api tick {k}")
        bad, _ = pool.verify_content()
        assert bad == 0
    assert errs > 0
    pool.close()


@pytest.mark.parametrize("seed,R,spt", [(5, 2, 0), (6, 3, 0), (7, 1, 0), (8, 2, 48)])
def test_gpu_verbs_random(seed, R, spt):
    need_gpu()
    from paper_2602_13692_b200 import Pool
    cfg = stress(seed, R, NB=128 if R > 1 else 192,     # some headroom so resumes can succeed
                 shared_prefix_tokens=spt)
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns)
    pool.load_trace(tr)
    rng = random.Random(seed)
    n_ok = {"pause": 0, "resume": 0, "migrate": 0}
    for k in range(80):
        _, dec_o = o.sched_step()
        _, dec_g = pool.step()
        same_decisions(dec_g, dec_o, f"tick {k}")
        for _ in range(rng.randint(0, 3)):
            verb = rng.choice(["pause", "resume", "migrate"])
            want = {"pause": (oracle.REASONING, oracle.ACTING), "resume": (oracle.PAUSED,),
                    "migrate": (oracle.REASONING, oracle.ACTING)}[verb]
            pool_p = [q for q in range(o.N) if o.status[q] in want]
            p = rng.choice(pool_p) if pool_p and rng.random() < 0.85 else rng.randrange(o.N)
            if verb == "pause":
                mode = rng.randrange(3)
                st_o, d_o = o.pause(p, mode)
                st_g, d_g = pool.pause(p, mode)
            elif verb == "resume":
                rep = rng.randrange(-1, R)
                st_o, d_o = o.resume(p, rep)
                st_g, d_g = pool.resume(p, rep)
            else:
                rep = rng.randrange(R)
                st_o, d_o = o.migrate(p, rep)
                st_g, d_g = pool.migrate(p, rep)
            assert st_o == st_g, (k, verb, p, st_o, st_g)
            if st_o == oracle.OK:
                n_ok[verb] += 1
                same_decisions(d_g, d_o, f"tick {k} verb {verb} pid {p}")
            compare_state(o, pool.debug_download(), where=f"tick {k} after {verb}({p})")
        bad, _ = pool.verify_content()
        assert bad == 0, f"tick {k}: {bad} KV words wrong"
    assert n_ok["pause"] > 0 and n_ok["resume"] > 0 and (R == 1 or n_ok["migrate"] > 0), n_ok
    pool.close()


def random_event_sequences(o, rng, T, n_max=16, illegal_p=0.15):
    """Batches with SEVERAL events per program (legal sequences in batch order, programs
    interleaved), plus sometimes one illegal event somewhere in the batch."""
    per = {}
    for _ in range(rng.randint(0, n_max)):
        p = rng.randrange(o.N)
        if p in per:
            continue
        st, ph = o.status[p], o.phase[p]
        seq = []
        if st == oracle.UNARRIVED:
            seq = [(A, p, 1000 + p, rng.randint(1, 300), 0)]
            if rng.random() < 0.2:
                seq.append((REL, p, 0, 0, 0))
        elif st == oracle.REASONING:
            seq = [(DEC, p, 0, rng.randint(1, 100), 0)]
            r = rng.random()
            if r < 0.4:
                seq.append((TC, p, 0, 0, max(0, T - rng.randint(0, 4000))))
                if rng.random() < 0.5:
                    seq.append((TR, p, 0, rng.randint(0, 200), 0))
                    seq.append((DEC, p, 0, rng.randint(1, 50), 0))
            elif r < 0.5:
                seq.append((REL, p, 0, 0, 0))
                seq.append((REL, p, 0, 0, 0))      # idempotent
        elif ph == oracle.PHASE_A and st in (oracle.ACTING, oracle.PAUSED):
            seq = [(TR, p, 0, rng.randint(0, 300), 0)]
            if st == oracle.ACTING and rng.random() < 0.5:
                seq.append((DEC, p, 0, rng.randint(1, 60), 0))
        per[p] = seq
    # interleave the programs' sequences, keeping each program's order
    evs = []
    queues = [list(s) for s in per.values() if s]
    while queues:
        q = rng.choice(queues)
        evs.append(q.pop(0))
        if not q:
            queues.remove(q)
    if rng.random() < illegal_p and evs:
        p = evs[rng.randrange(len(evs))][1]
        bad = (DEC, p, 0, 1, 0) if o.status[p] != oracle.REASONING else (A, p, 1, 1, 0)
        evs.insert(rng.randrange(len(evs) + 1), bad)
    return evs


@pytest.mark.parametrize("seed,R", [(21, 1), (22, 2), (23, 3)])
def test_gpu_api_mode_event_sequences(seed, R):
    """Several events per program in one batch (the parallel per-program state machines
    and the multi-event sort path) against the oracle's sequential validation."""
    need_gpu()
    from paper_2602_13692_b200 import Pool
    cfg = tracegen.get_config("c1_toy", n_replicas=R, hbm_blocks=48, host_blocks=16, max_ctx=4096,
                              compact_every=5)
    N = 48
    o = oracle.Oracle(cfg, api_mode=True, n_slots=N)
    pool = Pool(cfg, N, trace_mode=False)
    rng = random.Random(seed)
    errs = multi = 0
    for k in range(150):
        T = 5000 * k
        evs = random_event_sequences(o, rng, T)
        pids = [e[1] for e in evs]
        multi += len(pids) - len(set(pids))
        st_o, dec_o = o.sched_step(T, evs)
        st_g, dec_g = pool.step(T, evs, raise_on_error=False)
        assert st_o == st_g, (k, st_o, st_g, evs)
        if st_o != oracle.OK:
            errs += 1
            continue
        same_decisions(dec_g, dec_o, f"tick {k}")
        if k % 7 == 0:
            compare_state(o, pool.debug_download(), where=f"api tick {k}")
        bad, _ = pool.verify_content()
        assert bad == 0
    assert errs > 0 and multi > 50, (errs, multi)
    pool.close()


@pytest.mark.parametrize("name,n,ticks", [("c1_toy", 24, 60), ("bench_10k", 2000, 30)])
def test_gpu_api_replay_equals_trace_mode(name, n, ticks):
    """The engine's event batches recorded from a trace-mode run (tools/api_events.py),
    replayed through an API-mode context, give the same decisions every tick: the API
    event path and the trace engine are the same step 0."""
    need_gpu()
    import numpy as np
    from paper_2602_13692_b200 import Pool
    from tools.api_events import record
    over = dict(trace=dict(n=n, n_initial=n // 2 if name == "c1_toy" else None))
    if name == "bench_10k":
        over["kv"] = "mini"
    else:
        over.update(hbm_blocks=56, host_blocks=16)
    cfg = tracegen.get_config(name, **over)
    tr = tracegen.make_trace(cfg)
    batches, want = record(cfg, tr, ticks)
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, trace_mode=False, fill=False)
    n_ev = 0
    for k in range(ticks):
        st, got = pool.step(k * cfg["delta_t_ms"], batches[k])
        assert st == 0, (k, st)
        n_ev += len(batches[k])
        assert np.array_equal(got, want[k]), f"tick {k}: API replay differs from trace mode"
    assert n_ev > 0
    pool.close()


@pytest.mark.parametrize("seed,spt", [(31, 0), (32, 0), (33, 48)])
def test_gpu_health_failover_random(seed, spt):
    """NEXT-4 health mask: replicas fail and come back between ticks (ta_set_health),
    interleaved with the other verbs; decisions, status codes and full state equal the
    oracle's; the KV left on the healthy replicas stays byte-exact."""
    need_gpu()
    from paper_2602_13692_b200 import Pool
    cfg = tracegen.get_config("c1_toy", n_replicas=3, hbm_blocks=64, host_blocks=16, compact_every=4,
                              trace=dict(n=30, n_initial=12, seed=seed), shared_prefix_tokens=spt)
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns)
    pool.load_trace(tr)
    rng = random.Random(seed)
    down, n_fail = set(), 0
    for k in range(90):
        _, dec_o = o.sched_step()
        _, dec_g = pool.step()
        same_decisions(dec_g, dec_o, f"tick {k}")
        if rng.random() < 0.2:
            r = rng.randrange(3)
            up = r in down or len(down) == 2
            if up and r not in down:
                continue
            so, do = o.set_health(r, up)
            sg, dg = pool.set_health(r, up)
            assert so == sg == oracle.OK
            assert dec_tuples(dg) == do, (k, r, up)
            (down.discard if up else down.add)(r)
            n_fail += not up
            compare_state(o, pool.debug_download(), where=f"tick {k} after set_health({r}, {up})")
        if rng.random() < 0.3:                # verbs must refuse unhealthy targets the same way
            p = rng.randrange(o.N)
            rep = rng.randrange(3)
            so, do = o.resume(p, rep)
            sg, dg = pool.resume(p, rep)
            assert so == sg, (k, p, rep, so, sg)
            if so == oracle.OK:
                assert dec_tuples(dg) == do
        bad, _ = pool.verify_content()
        assert bad == 0, f"tick {k}: {bad} KV words wrong"
    assert n_fail > 0
    pool.close()


def test_gpu_rejected_batch_after_compaction_moves_no_bytes():
    """a rejected batch right after a compaction tick must not replay
    that tick's compaction copies.  Between ticks the engine writes into blocks (here:
    every HBM byte is overwritten with noise); the rejected batch must leave every byte
    as it was, and the oracle-parity run then continues unchanged."""
    need_gpu()
    from paper_2602_13692_b200 import Pool
    cfg = tracegen.get_config("c1_toy", n_replicas=2, hbm_blocks=48, host_blocks=16, max_ctx=4096,
                              compact_every=1)
    N = 40
    o = oracle.Oracle(cfg, api_mode=True, n_slots=N)
    pool = Pool(cfg, N, trace_mode=False)
    rng = random.Random(99)
    hit = 0
    for k in range(200):
        T = 5000 * k
        evs = random_events(o, rng, T, illegal_p=0.0)
        c0 = o.stats["compact_blocks"]
        st_o, dec_o = o.sched_step(T, evs)
        st_g, dec_g = pool.step(T, evs, raise_on_error=False)
        assert st_o == st_g == oracle.OK
        same_decisions(dec_g, dec_o, f"tick {k}")
        if o.stats["compact_blocks"] == c0:
            continue
        # this tick compacted: the engine now writes; then an illegal batch arrives
        torch.cuda.synchronize()
        saved = {r: pool.hbm[r].clone() for r in pool.hbm}
        for r in pool.hbm:
            pool.hbm[r].random_(0, 256)
        noise = {r: pool.hbm[r].clone() for r in pool.hbm}
        unarrived = [p for p in range(N) if o.status[p] == oracle.UNARRIVED]
        bad = [(DEC, unarrived[0] if unarrived else 0, 0, 1, 0)] if unarrived else [(A, 0, 1, 1, 0)]
        st_o, _ = o.sched_step(T + 1, bad)
        st_g, _ = pool.step(T + 1, bad, raise_on_error=False)
        assert st_o == st_g != oracle.OK
        torch.cuda.synchronize()
        for r in pool.hbm:
            assert torch.equal(pool.hbm[r], noise[r]), f"tick {k}: a rejected batch moved KV bytes on r{r}"
            pool.hbm[r].copy_(saved[r])
        compare_state(o, pool.debug_download(), where=f"after rejected batch, tick {k}")
        hit += 1
        if hit >= 3:
            break
    assert hit >= 3
    pool.close()


def test_gpu_api_two_shared_prompts_events_and_verbs():
    """NEXT-3 (reading A51) in API mode: ARRIVE's t_ms names the program's prompt (two
    prompts of 2 and 1 blocks); random legal / illegal batches, then resumes and
    migrations (verbs materialize prompts too), against the oracle."""
    need_gpu()
    from paper_2602_13692_b200 import Pool
    cfg = tracegen.get_config("c1_toy", n_replicas=2, hbm_blocks=64, host_blocks=16, max_ctx=4096,
                              compact_every=4, shared_prefixes=[(32, "a"), (16, "b")])
    N = 40
    o = oracle.Oracle(cfg, api_mode=True, n_slots=N)
    pool = Pool(cfg, N, trace_mode=False)
    rng = random.Random(17)
    errs = verbs = 0
    for k in range(150):
        T = 5000 * k
        evs = []
        for e in random_events(o, rng, T, illegal_p=0.05):
            if e[0] == A:                              # prompt index in t_ms; sometimes too short
                e = (A, e[1], e[2], rng.randint(8, 400), rng.choice((0, 1, 1, 0, 2)))
            evs.append(e)
        st_o, dec_o = o.sched_step(T, evs)
        st_g, dec_g = pool.step(T, evs, raise_on_error=False)
        assert st_o == st_g, (k, st_o, st_g, evs)
        if st_o != oracle.OK:
            errs += 1
            continue
        same_decisions(dec_g, dec_o, f"tick {k}")
        for _ in range(2):
            p = rng.randrange(N)
            if o.status[p] == oracle.PAUSED:
                rep = rng.randrange(-1, 2)
                st_o, d_o = o.resume(p, rep)
                st_g, d_g = pool.resume(p, rep)
                assert st_o == st_g, (k, "resume", p, st_o, st_g)
                if st_o == oracle.OK:
                    same_decisions(d_g, d_o, f"tick {k} verb")
                    verbs += 1
            elif o.status[p] in (oracle.REASONING, oracle.ACTING):
                rep = rng.randrange(2)
                st_o, d_o = o.migrate(p, rep)
                st_g, d_g = pool.migrate(p, rep)
                assert st_o == st_g, (k, "migrate", p, st_o, st_g)
                if st_o == oracle.OK:
                    same_decisions(d_g, d_o, f"tick {k} verb")
                    verbs += 1
        if k % 5 == 0:
            compare_state(o, pool.debug_download(), where=f"api tick {k}")
        bad, _ = pool.verify_content()
        assert bad == 0
    assert errs > 0 and o.stats["prefix_blocks"] > 0 and verbs > 0, (errs, verbs)
    pool.close()
