"""Benchmark of the ThunderAgent KV-manager hot path on B200 (contract: one JSON line).

A step is one scheduler tick through libta (ta_sched_step: ingest, footprint,
decayed load, pause, restore, materialize, KV block movement, finalize) over the
bench workload (tracegen config `bench_10k`: configs[3]'s 10k-program RL-burst
trace, one replica per GPU with a 96 GiB HBM pool of 4 MiB Qwen3-32B blocks and a
64 GiB pinned host tier).

The timed window is FIXED: ticks [1, 1 + K) of a fresh context (tick 0, the arrival
of the 10k programs, runs untimed), whatever W is -- the W warm-up ticks run on a
throw-away context over the same buffers first.  The window opens with the burst:
ticks 1-12 offload ~46k blocks (~190 GB) to the host tier and fetch ~13k back, so
every run at K >= 12 moves KV over every path the workload uses.  Each tick is
bracketed by its own CUDA-event pair; the 256 MiB L2 flush before each tick sits
OUTSIDE the pair.  `value` = K ticks / sum of tick times, normalised to 10k programs
per tick (program-ticks/s / 1e4), summed over ranks (max-over-ranks time).

Usage:
  python bench.py [--gpus N] [--steps K] [--warmup W]          # our CUDA path
  python bench.py --impl reference ...                         # the CPU oracle
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

JSON_OUT = sys.stdout                    # the one JSON line (fd 1 is redirected to stderr when N > 1)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = None


def load_metric():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        return json.load(f)["metric"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="bench_10k")
    ap.add_argument("--window-start", dest="start", type=int, default=1, help="first timed tick of the fresh context")
    ap.add_argument("--host-gib", type=float, default=64.0, help="cap of the pinned host tier")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--sched-ticks", type=int, default=200, help="ticks of the decision-path latency probe")
    ap.add_argument("--sched-start", type=int, default=13, help="first tick of the latency probe (after the burst)")
    ap.add_argument("--compaction-ticks", type=int, default=530,
                    help="configs[1] ticks of the in-trace D2D (compaction) probe at N=1 (0: skip)")
    return ap.parse_args()


# ---------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, which):
        setattr(self, which, time.time())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t_start", 0.0), getattr(self, "t_end", 1e30)
        lines = [ln for t, ln in self.lines if t0 - 0.15 <= t <= t1 + 0.15] or [ln for _, ln in self.lines]
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback B200_PROFILING.md (6.65 TB/s)"


def pcie_peak(torch, dev, barrier=None):
    """Measured pinned cudaMemcpyAsync peak per direction (1 GiB, best of 5).  With a
    `barrier` (all ranks copying at once) each direction starts together on every rank
    and the median of 5 copies is kept: a best-of figure would pick a copy that ran
    while the other ranks were already done (tools/pcie_concurrent.py)."""
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    out = {}
    for name, (dst, src) in (("h2d", (d, h)), ("d2h", (h, d))):
        if barrier is not None:
            torch.cuda.synchronize()
            barrier()
        vals = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            e1.synchronize()
            vals.append(n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        out[name] = max(vals) if barrier is None else sorted(vals)[len(vals) // 2]
    del h, d
    return out


def kv_path_microbench(pool, torch, peaks, hbm_peak, n_blocks=2048, reps=3):
    """Per-mode KV movement through ta_move_blocks with random block lists drawn from a
    fragmented pool (SURVEY.md §8(d) 'Two movement measurements', 1)."""
    import numpy as np
    from paper_2602_13692_b200 import binding
    rng = np.random.default_rng(7)
    dev = pool.device
    bb = pool.block_bytes
    out = {}
    NB, NH = pool.NB, pool.NH
    n_blocks = min(n_blocks, NB // 2, NH if NH else NB // 2)
    perm = rng.permutation(NB)
    src = torch.tensor(perm[:n_blocks].astype(np.int32), device=dev)
    dst = torch.tensor(perm[n_blocks:2 * n_blocks].astype(np.int32), device=dev)
    modes = [("d2d", binding.MOVE_D2D, src, dst, 2 * bb, hbm_peak, "hbm r+w")]
    if NH:
        hs = torch.tensor(rng.permutation(NH)[:n_blocks].astype(np.int32), device=dev)
        modes += [("d2h", binding.MOVE_D2H, src, hs, bb, peaks["d2h"], "pcie d2h (measured memcpy)"),
                  ("h2d", binding.MOVE_H2D, hs, dst, bb, peaks["h2d"], "pcie h2d (measured memcpy)")]
    if pool.R > 1:                      # NVLink: pull blocks from the next rank's HBM pool
        modes.append(("p2p_pull", binding.MOVE_P2P, src, dst, bb, 770.0,
                      "nvlink per direction (770 GB/s measured peer copy, B200_PROFILING.md; 900 nominal)"))
    s = pool.stream
    for name, kind, a, b, bytes_per_block, peak, pname in modes:
        best = 0.0
        srep = (pool.first + 1) % pool.R if kind == binding.MOVE_P2P else pool.first
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            pool.move_blocks(kind, srep, pool.first, a, b)
            e1.record(s)
            e1.synchronize()
            gbs = n_blocks * bytes_per_block / (e0.elapsed_time(e1) * 1e-3) / 1e9
            best = max(best, gbs)
        out[name] = {"gbs": round(best, 1), "peak_gbs": round(peak, 1), "frac": round(best / peak, 3),
                     "peak": pname, "blocks": n_blocks, "block_bytes": bb}
    return out


def sched_tick_latency(cfg, tr, torch, dev, start, n_ticks, flush, world=1, rank=0):
    """Latency of one scheduler tick at the bench's program count, decision path only:
    the same trace and pool sizes with the decision-identical `mini` KV shape (4 KiB
    blocks: no decision depends on bytes per block), so the movement kernels still run
    but move almost nothing.  One CUDA-event pair per tick on the context stream; L2
    flushed before every tick (outside the pair).  Ticks [start, start + n_ticks)."""
    import numpy as np
    from paper_2602_13692_b200 import Pool
    from paper_2602_13692_b200 import binding
    c = dict(cfg)
    c["kv"] = "mini"
    def run(do_flush, flags=binding.F_DECIDE_ONLY):
        pool = Pool(c, tr.n_slots, max_turns=tr.total_turns, fill=False, flags=flags, device=dev.index,
                    replicas_here=1, first_replica=rank)
        if world > 1:                        # one replica per GPU: every rank runs the whole
            from paper_2602_13692_b200.dist import connect   # replicated control plane
            connect(pool)
        pool.load_trace(tr)
        s = pool.stream
        for _ in range(start):
            pool.step(decisions=False)
        us = []
        for _ in range(n_ticks):
            with torch.cuda.stream(s):
                # a ~0.5 ms device-side spin first: the host has submitted the tick's graph
                # before the GPU reaches event a, so the pair times the GPU executing the
                # tick, not host submission jitter (Python / ctypes; the e2e key covers that)
                torch.cuda._sleep(1_000_000)
                if do_flush:
                    flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            pool.step(decisions=False)
            b.record(s)
            b.synchronize()
            us.append(a.elapsed_time(b) * 1e3)
        pool.close()
        us = np.array(us)
        if world > 1:                        # per tick, the slowest rank
            import torch.distributed as dist
            t = torch.tensor(us, dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            us = t.cpu().numpy()
        return us

    us = run(True)
    warm = run(False)           # back-to-back ticks, L2 warm (context only; the headline is flushed)
    mv = run(True, flags=0)     # the same with the (4 KiB-block) copy kernels in the graph
    return {"median_us": round(float(np.median(us)), 1), "p99_us": round(float(np.percentile(us, 99)), 1),
            "warm_l2_median_us": round(float(np.median(warm)), 1),
            "mean_us": round(float(us.mean()), 1), "ticks": f"{start}..{start + n_ticks - 1}",
            "programs": tr.n_slots, "programs_per_gpu": tr.n_slots // world, "gpus": world, "target_us": 100,
            "ranks": "per tick the slowest rank (each runs the replicated control plane over all programs)"
                     if world > 1 else "one GPU",
            "with_copies": {"median_us": round(float(np.median(mv)), 1), "p99_us": round(float(np.percentile(mv, 99)), 1),
                            "note": "the same ticks with the movement kernel copying the mini KV's 4 KiB blocks "
                                    "(hundreds over PCIe on host-tier ticks: the tail)"},
            "kv": "mini (4 KiB blocks; decisions identical to the Q32 run)",
            "note": "the decision path: one ta_sched_step CUDA graph with TA_F_DECIDE_ONLY (front, pause + "
                    "restore, plan, close; no block copies), L2 flushed before each tick; a 0.5 ms device "
                    "spin before the flush keeps the host's graph submission ahead of the GPU"}


def compaction_probe(torch, ticks, hbm_peak):
    """In-trace D2D at full block size: configs[1] (256 SWE programs, Qwen3-32B 4 MiB blocks,
    the same 96 GiB pool and host tier as bench_10k) with two-finger compaction every 4th
    tick.  bench_10k itself never compacts (closed-loop arrivals keep its pool full);
    configs[1] drains once all its programs have arrived, and its compaction ticks
    (452-520) move ~17k blocks.  k_copy_compact is timed by the TA_F_TIMING event pair
    around it (phase 7); bytes = read + write of every moved block."""
    import tracegen
    from paper_2602_13692_b200 import Pool, binding
    cfg = tracegen.get_config("c2_swe", compact_every=4)
    tr = tracegen.make_trace(cfg)
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False, flags=binding.F_TIMING)
    pool.load_trace(tr)
    blocks, us, n = 0, 0.0, 0
    for _ in range(ticks):
        pool.step(decisions=False)
        ti = pool.last_tick()
        if ti["d2d_blocks"]:
            ph = pool.phase_times()
            blocks += ti["d2d_blocks"]
            us += ph[7]
            n += 1
    bb = pool.block_bytes
    pool.close()
    if not blocks:
        return None
    by = 2.0 * blocks * bb
    gbs = by / (us * 1e-6) / 1e9
    return {"config": "configs[1] c2_swe, compact_every 4", "ticks": f"0..{ticks - 1}", "compaction_ticks": n,
            "blocks": blocks, "gb_rw": round(by / 1e9, 3), "kernel_s": round(us * 1e-6, 6),
            "gbs_rw": round(gbs, 1), "peak_gbs": hbm_peak, "frac_hbm": round(gbs / hbm_peak, 4),
            "note": "k_copy_compact per compaction tick (TA_F_TIMING event pair around it, development "
                    "build); bench_10k never compacts"}


def migrate_probe(pool, tr, world, rank, base_flags, torch, n_prog=24, ticks=12):
    """NVLink through the product API at N >= 2: a fresh trace context runs the burst's
    first `ticks` ticks; replica 1's active programs are paused with their blocks dropped
    (collective ta_pause, TA_PAUSE_DROP: both replicas run at lambda = 1, so replica 1
    needs room), then the `n_prog` REASONING programs of replica 0 with the most HBM blocks
    are migrated to replica 1 (collective ta_migrate; replica 1 pulls the blocks over
    NVLink from replica 0's pool).  Each verb is timed on the device (event pair on the
    context stream, max over ranks); GB/s = blocks pulled x block bytes / time."""
    import torch.distributed as dist
    from paper_2602_13692_b200 import binding
    fresh(pool, world, flags=base_flags)
    pool.load_trace(tr)
    for _ in range(ticks):
        pool.step(decisions=False)
    torch.cuda.synchronize()
    st = pool.debug_download(["status", "home", "n_hbm", "satisfied", "placement"])
    for p in range(tr.n_slots):
        if st["placement"][p] == 1 and st["status"][p] in (2, 3):
            pool.pause(p, 2)
    cand = [p for p in range(tr.n_slots) if st["status"][p] == 2 and st["home"][p] == 0 and st["placement"][p] == 0
            and st["satisfied"][p] == 1]                  # materialized: every block in HBM (NVLink only)
    cand = sorted(cand, key=lambda p: -int(st["n_hbm"][p]))[:n_prog]
    s = pool.stream
    blocks, ms_tot = 0, 0.0
    dev = pool.device
    for p in cand:
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        code, _ = pool.migrate(p, 1)
        b.record(s)
        b.synchronize()
        t = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if code == binding.TA_OK:
            blocks += int(pool.last_tick()["p2p_blocks"])
            ms_tot += float(t.item())
    if not blocks:
        return None
    by = blocks * pool.block_bytes
    gbs = by / (ms_tot * 1e-3) / 1e9
    return {"migrations": len(cand), "blocks": blocks, "gb": round(by / 1e9, 2), "verb_time_ms": round(ms_tot, 2),
            "gbs": round(gbs, 1), "peak_gbs": 770.0, "frac": round(gbs / 770.0, 3),
            "note": "ta_migrate replica 0 -> 1 end to end on the device (plan, NVLink pull, close), max over "
                    "ranks; peak = the measured peer copy (B200_PROFILING.md; 900 nominal)"}


def workload(name, world):
    """The bench workload at N GPUs: N replicas, 10k programs per replica (weak scaling):
    N interleaved copies of the 1-GPU trace (tracegen.tile_trace), so every replica sees
    the 1-GPU workload and per-GPU work stays fixed as N grows."""
    import tracegen
    cfg = tracegen.get_config(name)
    cfg["n_replicas"] = world
    cfg["trace"]["tile"] = world
    return cfg


def host_cap_bytes(host_gib, world):
    """Pinned host tier per rank: at most host_gib, and at most 55% of RAM shared by the ranks."""
    cap = int(host_gib * (1 << 30))
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal:"):
                cap = min(cap, int(ln.split()[1]) * 1024 * 55 // 100 // world)
    except OSError:
        pass
    return cap


def metadata_bytes(pool_stats_prev, n_programs, sum_nb, moved_blocks):
    # algorithmic bytes of the decision phase: program records r+w,
    # one block-table scan, bitmaps, table/owner updates of moved blocks
    return n_programs * 96 + sum_nb * 4 + moved_blocks * 8


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, metric):
    """The tier's reference arm: the CPU oracle, as it stands, on the same window."""
    import tracegen
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg = workload(args.config, world)
    tr = tracegen.make_trace(cfg)
    warm = oracle.Oracle(cfg, tr)            # W warm-up ticks on a throw-away instance
    for _ in range(args.warmup):
        warm.sched_step()
    del warm
    o = oracle.Oracle(cfg, tr)
    for _ in range(args.start):
        o.sched_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.sched_step()
    dt = time.perf_counter() - t0
    n_prog = tr.n_slots
    value = args.steps * n_prog / 1e4 / dt
    line = {
        "impl": "reference", "metric": metric, "value": round(value, 4),
        "unit": "ticks/s (10k-program ticks, summed over GPUs)",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.config, "programs": n_prog, "replicas": cfg["n_replicas"],
                   "ticks": f"{args.start}..{args.start + args.steps - 1}"},
        "cpu_baseline": {"value": round(value, 4), "unit": "ticks/s", "cores": 1, "kind": "oracle",
                         "sample": f"oracle (pure Python, 1 thread), ticks {args.start}..{args.start + args.steps - 1} "
                                   f"of a fresh run; it tracks block indices, moves no KV bytes"},
        "e2e": {"value": round(value, 4), "unit": "ticks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, trace, start, seconds):
    """The oracle on the same trace from the same first tick, for ~`seconds`."""
    import oracle
    o = oracle.Oracle(cfg, trace)
    for _ in range(start):
        o.sched_step()                    # untimed, like the GPU window
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < seconds:
        o.sched_step()
        n += 1
    dt = time.perf_counter() - t0
    cpu = os.cpu_count()
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": round(n * trace.n_slots / 1e4 / dt, 4), "unit": "ticks/s", "cores": 1,
            "kind": "oracle",
            "sample": f"ticks {start}..{start + n - 1} of the same trace ({dt:.1f} s, pure-Python oracle, "
                      f"1 of {cpu} cores, {model}); the oracle tracks block indices and moves no KV bytes"}


# per-tick algorithmic bytes of the kernels: the footprint pass reads a
# slot's 64-B program record and writes 24 B of derived values, and reads 4 B per entry
# of the rows written since the previous pass (clean rows are not read);
# the movement kernel moves one block per moved block over its link; compaction reads
# and writes each moved block in HBM
FRONT_SLOT_BYTES = 88


def fresh(pool, world, flags=None):
    """A fresh context over the same buffers (every slot UNARRIVED, all blocks free)."""
    pool.reset(flags=flags)
    if world > 1:
        from paper_2602_13692_b200.dist import connect
        connect(pool)


# ---------------------------------------------------------------------------- our arm
def main():
    args = parse()
    metric = load_metric()
    if args.impl == "reference":
        return run_reference(args, metric)
    import numpy as np
    import torch
    import torch.distributed as dist

    import tracegen
    from paper_2602_13692_b200 import Pool, binding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:                         # native libraries (NCCL's version banner) print to fd 1:
        global JSON_OUT                   # send fd 1 to stderr, keep stdout for the JSON line
        JSON_OUT = os.fdopen(os.dup(1), "w")
        sys.stdout.flush()
        os.dup2(2, 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # keep stdout to the one JSON line
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # weak scaling: N replicas (one per GPU) share one global queue over 10k * N
    # programs; every rank runs the replicated control plane, moves its own replica's
    # bytes, and pulls / pushes migrated blocks over NVLink
    cfg = workload(args.config, world)
    tr = tracegen.make_trace(cfg)
    block_bytes = 2 * 64 * 8 * 128 * 2 * cfg["block_tokens"]
    nh = min(cfg["host_blocks"], host_cap_bytes(args.host_gib, world) // block_bytes)
    cfg["host_blocks"] = nh
    K, W, S0 = args.steps, args.warmup, args.start
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False, flags=0, device=local,
                replicas_here=1, first_replica=rank)
    base_flags = pool.c.flags
    if world > 1:
        from paper_2602_13692_b200.dist import connect
        connect(pool)
    pool.load_trace(tr)
    peaks_file, peak_src = measured_peaks()
    hbm_peak = float(peaks_file.get("hbm_gbs", 6650.0))
    s = pool.stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(s):
        flush.zero_()                    # first touch of the flush buffer outside the timed region

    # the clock sampler starts before warm-up (nvidia-smi start-up can stall the driver);
    # only samples taken inside the timed window are kept
    sampler = ClockSampler(local)
    sampler.start()
    # ---- W warm-up ticks (ticks 0..W-1 of a throw-away context over the same buffers)
    for _ in range(W):
        pool.step(decisions=False)
    torch.cuda.synchronize(dev)
    # ---- the timed window: ticks [S0, S0 + K) of a fresh context
    fresh(pool, world)
    pool.load_trace(tr)
    for _ in range(S0):
        pool.step(decisions=False)
    torch.cuda.synchronize(dev)
    time.sleep(0.3)
    st0 = pool.stats()
    barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    sampler.mark("t_start")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * K)]
    e0.record(s)
    for i in range(K):                # enqueued back to back: no host sync inside the region
        with torch.cuda.stream(s):
            flush.zero_()             # L2 flush (256 MiB > 126 MB L2), outside the tick's event pair
        ev[2 * i].record(s)
        pool.step(decisions=False)
        ev[2 * i + 1].record(s)
    e1.record(s)
    torch.cuda.synchronize(dev)
    sampler.mark("t_end")
    barrier()
    clocks = sampler.stop()
    step_ms = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(K)]
    ms = max_over_ranks(sum(step_ms))
    region_ms = max_over_ranks(e0.elapsed_time(e1))
    st1 = pool.stats()
    progs_total = tr.n_slots
    value = K * progs_total / 1e4 / (ms * 1e-3)

    # ---- per-kernel breakdown: the SAME window again with TA_F_TIMING (event-record
    # nodes in the graph, ~2.7 us each) on the context stream; host-mapped telemetry of
    # every tick (blocks per path and per replica) and the block-table entries scanned
    fresh(pool, world, flags=base_flags | binding.F_TIMING)
    pool.load_trace(tr)
    for _ in range(S0):
        pool.step(decisions=False)
    ticks = []
    st_prev = pool.debug_download(["status"])
    ent_prev = pool.debug_counters()["front_row_entries"]
    for _ in range(K):
        with torch.cuda.stream(s):
            flush.zero_()
        pool.step(decisions=False)
        ph = np.array(pool.phase_times())          # syncs the stream
        ti = pool.last_tick()
        ent = pool.debug_counters()["front_row_entries"]
        # entries read by this tick's footprint pass: the rows written since the previous
        # pass (clean rows keep their counts and class and are not read)
        live = np.isin(st_prev["status"], (1, 2, 3))
        ticks.append((ti, ph, ent - ent_prev, int(live.sum())))
        ent_prev = ent
        st_prev = pool.debug_download(["status"])
    barrier()

    # ---- e2e through the public API as a serving engine drives it: an API-mode context
    # over the same buffers; every step copies that tick's event batch from pinned host
    # memory to the device (ta_event array, H2D inside ta_sched_step) and reads the
    # decisions back (D2H).  The batches are the engine's view of the trace
    # (tools/api_events.py), recorded untimed beforehand on a decision-identical
    # small-KV context; API replay == trace mode is a GPU test (test_gpu_api.py).
    from tools.api_events import record
    rec_cfg = dict(cfg)
    rec_cfg["kv"] = "mini"
    batches, _ = record(rec_cfg, tr, S0 + K, device=local)
    fresh(pool, world, flags=base_flags & ~binding.F_TRACE_MODE)
    dt_ms = cfg["delta_t_ms"]
    for k in range(S0):
        pool.step(k * dt_ms, batches[k], decisions=False)
    torch.cuda.synchronize(dev)
    barrier()
    h2d = d2h = n_events = 0
    e2e_ms = 0.0
    for k in range(S0, S0 + K):
        with torch.cuda.stream(s):
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        st, dec = pool.step(k * dt_ms, batches[k], decisions=True)
        b.record(s)
        if st != 0:
            raise RuntimeError(f"e2e replay: ta_sched_step status {st} at tick {k}")
        b.synchronize()
        e2e_ms += a.elapsed_time(b)
        h2d += batches[k].nbytes + 12    # events + header (now_ms, n_events)
        d2h += dec.nbytes + 8            # decisions + count + status
        n_events += len(batches[k])
    e2e_ms = max_over_ranks(e2e_ms)
    e2e_value = K * progs_total / 1e4 / (e2e_ms * 1e-3)


    # ---- host-link peaks of this run: one GPU alone (rank 0; the movement floor uses these
    # at every N, so the fraction can only fall when the host is shared), and with N > 1
    # every rank copying at once (context: GPUs share host-side PCIe / memory bandwidth; a
    # synchronized DMA measurement of that is noisy and can sit below what the kernels
    # reach, so it does not enter the floor)
    peaks = pcie_peak(torch, dev) if (nh and rank == 0) else {"h2d": 0.0, "d2h": 0.0}
    peaks_concurrent = None
    if world > 1:
        barrier()
        tpk = torch.tensor([peaks["d2h"], peaks["h2d"]], dtype=torch.float64, device=dev)
        dist.all_reduce(tpk, op=dist.ReduceOp.MAX)            # rank 0's to every rank
        peaks = {"d2h": float(tpk[0]) or 1.0, "h2d": float(tpk[1]) or 1.0}
        if nh:
            torch.cuda.synchronize()
            barrier()
            pc = pcie_peak(torch, dev, barrier=dist.barrier)
            tpk = torch.tensor([pc["d2h"], pc["h2d"]], dtype=torch.float64, device=dev)
            dist.all_reduce(tpk, op=dist.ReduceOp.MIN)
            peaks_concurrent = {"d2h": round(float(tpk[0]), 1), "h2d": round(float(tpk[1]), 1)}
        barrier()
    elif not nh:
        peaks = {"h2d": 1.0, "d2h": 1.0}
    peaks_alone = dict(peaks)

    # ---- movement in the window, per path, and the roofline of every kernel.  Tick
    # telemetry counts are cluster totals; the replicas are symmetric (per GPU = total/N).
    bb = pool.block_bytes
    G = 1e9
    nvl = 770.0 if world > 1 else hbm_peak / 2     # co-located "P2P" is an HBM read+write
    ph_sum = np.zeros(9)
    mv = dict(d2h=0.0, h2d=0.0, p2p=0.0, d2d=0.0, floor_s=0.0, d2d_floor_s=0.0)
    front_bytes = 0.0
    for ti, ph, sum_nb, n_live in ticks:
        ph_sum += ph
        mv["d2h"] += ti["d2h_blocks"] * bb / world
        mv["h2d"] += ti["h2d_blocks"] * bb / world
        mv["p2p"] += ti["p2p_blocks"] * bb / world
        mv["d2d"] += ti["d2d_blocks"] * bb / world
        # one fused kernel: the links run in parallel; its floor is the slowest replica's
        # own links (PCIe out / in of its tier, NVLink in); every rank waits for it
        mv["floor_s"] += max(max(ti["d2h_of"][r] * bb / peaks["d2h"], ti["h2d_of"][r] * bb / peaks["h2d"],
                                 ti["p2p_to"][r] * bb / nvl) for r in range(len(ti["d2h_of"]))) / G
        if peaks_concurrent:                         # context: the same floor at the concurrent DMA rates
            mv["floor_conc_s"] = mv.get("floor_conc_s", 0.0) + max(
                max(ti["d2h_of"][r] * bb / max(peaks_concurrent["d2h"], 1e-9),
                    ti["h2d_of"][r] * bb / max(peaks_concurrent["h2d"], 1e-9),
                    ti["p2p_to"][r] * bb / nvl) for r in range(len(ti["d2h_of"]))) / G
        mv["d2d_floor_s"] += 2 * ti["d2d_blocks"] * bb / world / hbm_peak / G
        front_bytes += (FRONT_SLOT_BYTES * progs_total / world + 4 * sum_nb / world)
    move_s = ph_sum[3] * 1e-6                         # fused movement kernel, summed over the window
    move_bytes = mv["d2h"] + mv["h2d"] + mv["p2p"]
    # kernel names by phase slot (ta_phase_times)
    if world == 1:
        names = ["k_tick_front", "k_pause_restore", "k_plan", "k_move_fused", "-", "-", "k_close",
                 "k_copy_compact", "-"]
    else:
        names = ["k_tick_front", "k_pause_restore", "k_plan", "k_barrier+k_move_fused+k_barrier", "-", "k_fill",
                 "k_close", "k_copy_compact", "-"]
    dom = int(np.argmax(ph_sum))
    per_kernel = []
    for i, nm in enumerate(names):
        if nm == "-" or ph_sum[i] <= 0:
            continue
        t = ph_sum[i] * 1e-6
        if i == 3:
            byts, pk, bnd = move_bytes, (move_bytes / mv["floor_s"] / G if mv["floor_s"] > 0 else None), \
                "pcie full duplex (+ nvlink)"
        elif i == 7:
            byts, pk, bnd = 2 * mv["d2d"], hbm_peak, "hbm"
        elif i == 0:                                 # reads only rows written since the last tick
            byts, pk, bnd = front_bytes, hbm_peak, "latency (two dependent round trips; fraction of HBM for context)"
        else:
            byts, pk, bnd = None, None, "latency (serial planner chain)"
        ach = byts / t / G if byts else None
        per_kernel.append({"kernel": nm, "us_per_launch": round(ph_sum[i] / K, 2),
                           "share_of_step": round(float(ph_sum[i] / ph_sum.sum()), 4),
                           "bytes_per_launch": int(byts / K) if byts else None,
                           "achieved_gbs": round(ach, 2) if ach else None,
                           "peak_gbs": round(pk, 1) if pk else None,
                           "frac": round(ach / pk, 4) if (ach and pk) else None, "bound": bnd})
    # traffic: DRAM bytes per launch from the committed ncu --set full capture of the
    # movement kernel in this window (ratio of measured DRAM bytes to algorithmic bytes)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r2_move_traffic.json")) as f:
            traffic = round(move_bytes / K * json.load(f)["ratio_dram_to_algorithmic"])
    except (OSError, KeyError, ValueError):
        traffic = None
    dk = next(k for k in per_kernel if k["kernel"] == names[dom])
    psrc = (f"measured in this run: pinned cudaMemcpyAsync 1 GiB (d2h {peaks['d2h']:.1f}, h2d {peaks['h2d']:.1f}"
            f" GB/s{'' if world == 1 else ', one GPU alone; with all %d GPUs copying at once (DMA, context only): %s' % (world, peaks_concurrent)}"
            f"); peak = bytes / floor, floor = sum over ticks of max over replicas and links of link bytes / link peak"
            ) if dom == 3 else peak_src
    roofline = {"bound": "pcie" if dom == 3 else dk["bound"], "kernel": names[dom],
                "achieved": dk["achieved_gbs"], "peak": dk["peak_gbs"], "unit": "GB/s", "frac": dk["frac"],
                "traffic": traffic if dom == 3 else None,
                "traffic_source": "ncu --set full (profiles/r2_move_traffic.json): DRAM bytes / algorithmic bytes x this run's bytes per launch",
                "share_of_step": dk["share_of_step"], "peak_source": psrc,
                "note": "achieved = algorithmic bytes per launch / mean launch time (CUDA events on the context stream, TA_F_TIMING replay of the same window)"}
    kv_paths = kv_path_microbench(pool, torch, peaks, hbm_peak) if rank == 0 else None
    barrier()                            # peers keep their pools mapped until rank 0 is done
    kv_moved = {
        "window": f"ticks {S0}..{S0 + K - 1}",
        "gb": {p: round(mv[p] / 1e9, 3) for p in ("d2h", "h2d", "p2p", "d2d")},
        "blocks_total_all_replicas": {"d2h": st1["evict_to_host"] - st0["evict_to_host"],
                                      "h2d": st1["h2d_blocks"] - st0["h2d_blocks"],
                                      "p2p": st1["p2p_blocks"] - st0["p2p_blocks"],
                                      "d2d": st1["compact_blocks"] - st0["compact_blocks"],
                                      "dropped": st1["evict_dropped"] - st0["evict_dropped"]},
        "movement_kernel_s": round(move_s, 4),
        "in_trace_gbs": round(move_bytes / move_s / G, 2) if move_s > 0 else None,
        "link_floor_s": round(mv["floor_s"], 4),
        "frac_of_link_floor": round(mv["floor_s"] / move_s, 4) if move_s > 0 else None,
        "frac_of_concurrent_dma_floor": (round(mv["floor_conc_s"] / move_s, 4)
                                         if move_s > 0 and mv.get("floor_conc_s") else None),
        "compaction": ({"gbs_rw": round(2 * mv["d2d"] / (ph_sum[7] * 1e-6) / G, 1),
                        "frac_hbm": round(mv["d2d_floor_s"] / (ph_sum[7] * 1e-6), 4)}
                       if mv["d2d"] > 0 and ph_sum[7] > 0 else None),
        "compaction_in_trace": "bench_10k never compacts (its pool stays full); the N = 1 line runs the "
                               "configs[1] compaction probe (DESIGN.md 8)",
        "host_link_peaks_gbs": peaks,
        "host_link_concurrent_gbs": peaks_concurrent,
    }
    tick_lat = (sched_tick_latency(cfg, tr, torch, dev, args.sched_start, args.sched_ticks, flush, world, rank)
                if args.sched_ticks > 0 else None)   # every rank at N > 1 (max over ranks per tick)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c1 = tracegen.get_config(args.config)
        cpu = cpu_baseline(c1, tracegen.make_trace(c1), S0, args.cpu_seconds)
    dstat = {k: st1[k] - st0[k] for k in binding.STAT_KEYS + binding.LEDGER_KEYS if isinstance(st0[k], int)}
    launches = 5 + (1 if cfg.get("compact_every", 0) > 0 else 0) + (2 if world > 1 else 0)
    nb_main, nh_main = pool.NB, pool.NH
    if world > 1:
        kv_moved["p2p_in_api"] = migrate_probe(pool, tr, world, rank, base_flags, torch)
    if world == 1 and args.compaction_ticks > 0:   # the main pool's memory goes back to torch's caches
        pool.close()
        pool.hbm, pool.host, pool.dev_ws, pool.host_ws = {}, {}, None, None
        kv_moved["compaction_in_trace"] = compaction_probe(torch, args.compaction_ticks, hbm_peak)
    line = {
        "metric": metric, "value": round(value, 4), "unit": "ticks/s (10k-program ticks, summed over GPUs)",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": round(ms / K, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic",
        "config": {"workload": args.config, "programs": tr.n_slots, "replicas": world, "replicas_per_gpu": 1,
                   "kv": "Qwen3-32B GQA L64 H8 D128 bf16, 16-token blocks (4 MiB)",
                   "hbm_blocks": nb_main, "host_blocks": nh_main,
                   "window": f"ticks {S0}..{S0 + K - 1} of a fresh context (fixed; the W warm-up ticks run on a "
                             f"throw-away context first)",
                   "engine_fill": "off (engine stand-in, not a hot-path row)",
                   "l2": "256 MiB memset before every tick, outside the tick's CUDA-event pair; KV pools and "
                         "host tier (160 GiB) exceed L2",
                   "parallelism": f"dp{world} (one replica per GPU)"},
        "clocks": clocks,
        "e2e": {"value": round(e2e_value, 4), "unit": "ticks/s", "h2d_bytes_per_step": int(h2d / K),
                "d2h_bytes_per_step": int(d2h / K), "events_per_step": round(n_events / K, 1),
                "note": "API mode (serving-engine path): per step the tick's event batch H2D from pinned host "
                        "memory, validation + apply + tick on the device, decisions D2H; same window as value"},
        "gpu_launches": K * launches,
        "roofline": roofline,
        "kernels": per_kernel,
        "kv_moved": kv_moved,
        "sched_tick": tick_lat,
        "phases_us_per_step": {n: round(float(v / K), 1) for n, v in zip(names, ph_sum) if n != "-"},
        # NEXT-1: STP cost ledger of the timed ticks (token-ms per step) and
        # the Cost_unused < c_min bound of PAPER.md:415 (replica-ticks checked / violated)
        "stp_ledger_token_ms_per_step": {k[5:]: int(dstat[k] / K) for k in binding.LEDGER_KEYS
                                         if k.startswith("cost_")},
        "unused_bound": {"checks": dstat["unused_bound_checks"], "violations": dstat["unused_bound_violations"]},
        "kv_paths": kv_paths,
        "cpu_baseline": cpu,
        "step_ms": [round(x, 3) for x in step_ms],
        "region_ms_incl_flush": round(region_ms, 3),
    }
    if rank == 0:
        JSON_OUT.write(json.dumps(line) + "\n")
        JSON_OUT.flush()
    pool.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
