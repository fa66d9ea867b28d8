"""Benchmark of the ThunderAgent KV-manager hot path on B200 (contract: one JSON line).

A step is one scheduler tick through libta (ta_sched_step: ingest, footprint,
decayed load, pause, restore, materialize, KV block movement, finalize) over the
bench workload (tracegen config `bench_10k`: configs[3]'s 10k-program RL-burst
trace, one replica per GPU with a 96 GiB HBM pool of 4 MiB Qwen3-32B blocks and a
pinned host tier).  `value` = scheduler ticks/s normalised to 10k programs per tick
(program-ticks/s / 1e4), summed over ranks.  Usage:

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
    ap.add_argument("--preroll", type=int, default=8, help="untimed ticks before warm-up")
    ap.add_argument("--host-gib", type=float, default=64.0, help="cap of the pinned host tier")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--sched-ticks", type=int, default=200, help="ticks of the decision-path latency probe")
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


def sched_tick_latency(cfg, tr, torch, dev, start, n_ticks, flush):
    """Latency of one scheduler tick at the bench's program count, decision path only:
    the same trace and pool sizes with the decision-identical `mini` KV shape (4 KiB
    blocks: no decision depends on bytes per block), so the movement kernels still run
    but move almost nothing.  One CUDA-event pair per tick on the context stream; L2
    flushed before every tick (outside the pair).  Ticks [start, start + n_ticks)."""
    import numpy as np
    from paper_2602_13692_b200 import Pool
    c = dict(cfg)
    c["kv"] = "mini"
    def run(do_flush):
        pool = Pool(c, tr.n_slots, max_turns=tr.total_turns, fill=False, flags=0, device=dev.index,
                    replicas_here=1, first_replica=0)
        pool.load_trace(tr)
        s = pool.stream
        for _ in range(start):
            pool.step(decisions=False)
        us = []
        for _ in range(n_ticks):
            if do_flush:
                with torch.cuda.stream(s):
                    flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            pool.step(decisions=False)
            b.record(s)
            b.synchronize()
            us.append(a.elapsed_time(b) * 1e3)
        pool.close()
        return np.array(us)

    us = run(True)
    warm = run(False)           # back-to-back ticks, L2 warm (context only; the headline is flushed)
    return {"median_us": round(float(np.median(us)), 1), "p99_us": round(float(np.percentile(us, 99)), 1),
            "warm_l2_median_us": round(float(np.median(warm)), 1),
            "mean_us": round(float(us.mean()), 1), "ticks": f"{start}..{start + n_ticks - 1}",
            "programs": tr.n_slots, "target_us": 100,
            "kv": "mini (4 KiB blocks; decisions identical to the Q32 run, movement kernels run but move ~0 B)",
            "note": "one full ta_sched_step CUDA graph (5 kernels), L2 flushed before each tick"}


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
    import tracegen
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = workload(args.config, int(os.environ.get("WORLD_SIZE", "1")))
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    for _ in range(args.preroll + args.warmup):
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
                   "ticks": f"{args.preroll + args.warmup}..{args.preroll + args.warmup + args.steps - 1}"},
        "cpu_baseline": {"value": round(value, 4), "unit": "ticks/s", "cores": 1, "kind": "oracle",
                         "sample": f"oracle (pure Python, 1 thread) ticks after {args.preroll + args.warmup} untimed"},
        "e2e": {"value": round(value, 4), "unit": "ticks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, trace, seconds):
    import oracle
    o = oracle.Oracle(cfg, trace)
    o.sched_step()                    # tick 0 (arrivals) untimed
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
            "sample": f"ticks 1..{n} of the same trace ({dt:.1f} s, pure-Python oracle, 1 of {cpu} cores, {model})"}


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

    # weak scaling: N replicas (one per GPU) share one global queue over 10k * N
    # programs; every rank runs the replicated control plane, moves its own replica's
    # bytes, and pulls / pushes migrated blocks over NVLink
    cfg = workload(args.config, world)
    tr = tracegen.make_trace(cfg)
    block_bytes = 2 * 64 * 8 * 128 * 2 * cfg["block_tokens"]
    nh = min(cfg["host_blocks"], host_cap_bytes(args.host_gib, world) // block_bytes)
    cfg["host_blocks"] = nh
    # the timed run has no timing nodes in its graph; the per-kernel breakdown comes from
    # a replay of the same ticks with TA_F_TIMING (event-record nodes cost ~2.7 us each)
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns, fill=False, flags=0, device=local,
                replicas_here=1, first_replica=rank)
    base_flags = pool.c.flags
    if world > 1:
        from paper_2602_13692_b200.dist import connect
        connect(pool)
    pool.load_trace(tr)
    peaks_file, peak_src = measured_peaks()
    hbm_peak = float(peaks_file.get("hbm_gbs", 6650.0))

    # the clock sampler starts before warm-up (nvidia-smi start-up can stall the driver);
    # only samples taken inside the timed window are kept
    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.preroll + args.warmup):
        pool.step(decisions=False)
    torch.cuda.synchronize(dev)
    time.sleep(0.3)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(pool.stream):
        flush.zero_()                    # first touch of the flush buffer outside the timed region
    torch.cuda.synchronize(dev)
    s = pool.stream
    st0 = pool.stats()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    sampler.mark("t_start")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    e0.record(s)
    for i in range(args.steps):       # enqueued back to back: no host sync inside the region
        ev[2 * i].record(s)
        with torch.cuda.stream(s):
            flush.zero_()             # L2 flush (256 MiB > 126 MB L2) inside the timed region
        pool.step(decisions=False)
        ev[2 * i + 1].record(s)
    e1.record(s)
    torch.cuda.synchronize(dev)
    sampler.mark("t_end")
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    step_ms = [round(ev[2 * i].elapsed_time(ev[2 * i + 1]), 3) for i in range(args.steps)]
    st1 = pool.stats()
    sum_nb = int(pool.debug_download()["nb"].sum())   # block-table entries scanned per tick
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    progs_total = tr.n_slots
    value = args.steps * progs_total / 1e4 / (ms * 1e-3)

    # ---- per-kernel breakdown: the SAME ticks again with TA_F_TIMING (fresh context over
    # the same buffers, same untimed prefix); CUDA-event times of every graph phase
    pool.reset(flags=base_flags | binding.F_TIMING)
    if world > 1:
        connect(pool)
    pool.load_trace(tr)
    for _ in range(args.preroll + args.warmup):
        pool.step(decisions=False)
    phase_sum = np.zeros(9)
    ticks_info = []
    for _ in range(args.steps):
        with torch.cuda.stream(s):
            flush.zero_()
        pool.step(decisions=False)
        ph_step = np.array(pool.phase_times())   # syncs the stream
        phase_sum += ph_step
        ticks_info.append((pool.last_tick(), ph_step))   # host-mapped telemetry
    if world > 1:
        dist.barrier()

    # ---- e2e: the SAME ticks through the public API as a serving engine drives it: an
    # API-mode context over the same buffers; every step copies that tick's event batch
    # from host memory to the device (ta_event array, H2D inside ta_sched_step) and
    # reads the decisions back (D2H).  The batches are the engine's view of the trace
    # (tools/api_events.py), recorded untimed beforehand on a decision-identical
    # small-KV context; API replay == trace mode is a GPU test (test_gpu_api.py).
    from tools.api_events import record
    rec_cfg = dict(cfg)
    rec_cfg["kv"] = "mini"
    n_pre = args.preroll + args.warmup
    batches, _ = record(rec_cfg, tr, n_pre + args.steps, device=local)
    pool.reset(flags=base_flags & ~binding.F_TRACE_MODE)
    if world > 1:
        connect(pool)                    # fresh context: fresh mailboxes to map
    dt_ms = cfg["delta_t_ms"]
    for k in range(n_pre):
        pool.step(k * dt_ms, batches[k], decisions=False)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    h2d = d2h = n_events = 0
    e0.record(s)
    for k in range(n_pre, n_pre + args.steps):
        with torch.cuda.stream(s):
            flush.zero_()
        st, dec = pool.step(k * dt_ms, batches[k], decisions=True)
        if st != 0:
            raise RuntimeError(f"e2e replay: ta_sched_step status {st} at tick {k}")
        h2d += batches[k].nbytes + 12    # events + header (now_ms, n_events)
        d2h += dec.nbytes + 8            # decisions + count + status
        n_events += len(batches[k])
    e1.record(s)
    torch.cuda.synchronize(dev)
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = args.steps * progs_total / 1e4 / (e2e_ms * 1e-3)

    # ---- bytes per path in the timed steps, roofline of the dominant kernel
    dstat = {k: st1[k] - st0[k] for k in binding.STAT_KEYS + binding.LEDGER_KEYS if isinstance(st0[k], int)}
    bb = pool.block_bytes
    ph = phase_sum / args.steps            # us per step
    if world == 1:
        names = ["tick_front(ingest+footprint)", "pause+restore", "plan(cluster)", "movement_fused(d2h+h2d+p2p+fill)",
                 "-", "-", "close(finalize+compact_plan+assemble)", "compact_d2d", "-"]
    elif pool.c.flags & binding.F_NO_FUSE == 0:
        names = ["tick_front(ingest+footprint)", "pause+restore", "plan(cluster)",
                 "barrier+movement_fused(d2h+pull+push)+barrier", "-", "fill", "close(finalize+compact_plan+assemble)",
                 "compact_d2d", "-"]
    else:
        names = ["tick_front(ingest+footprint)", "pause+restore", "plan(cluster)", "evict_d2h+barrier",
                 "fetch_p2p_h2d+push+barrier", "fill", "close(finalize+compact_plan+assemble)", "compact_d2d", "-"]
    # the host-link peak of ONE GPU's link, measured by rank 0 while the others wait; with
    # N > 1 also with every rank copying at once (GPUs can share host-side PCIe / memory
    # bandwidth): the floor uses the concurrent figure of the slowest rank, the physical
    # limit when all replicas stream together
    peaks = pcie_peak(torch, dev) if (nh and rank == 0) else {"h2d": 1.0, "d2h": 1.0}
    peaks_alone = dict(peaks)
    if world > 1:
        dist.barrier()
        if nh:
            torch.cuda.synchronize()
            dist.barrier()
            pc = pcie_peak(torch, dev, barrier=dist.barrier)
            tpk = torch.tensor([pc["d2h"], pc["h2d"]], dtype=torch.float64, device=dev)
            dist.all_reduce(tpk, op=dist.ReduceOp.MIN)
            peaks = {"d2h": float(tpk[0]), "h2d": float(tpk[1])}
        dist.barrier()
    # algorithmic bytes per GPU, tick by tick (telemetry counts are cluster totals; the
    # replicas are symmetric, so per GPU = total / N).  A movement phase's time floor is
    # the slowest link it must cross in that tick (PCIe is full duplex).
    nvl = 770.0 if world > 1 else hbm_peak / 2     # co-located "P2P" is an HBM read+write
    G = 1e9
    tmin = {3: 0.0, 4: 0.0, 7: 0.0}
    byts = {3: 0.0, 4: 0.0, 7: 0.0}
    for ti, _ in ticks_info:
        d2h_b = ti["d2h_blocks"] * bb / world
        h2d_b = ti["h2d_blocks"] * bb / world
        p2p_b = ti["p2p_blocks"] * bb / world
        d2d_b = 2 * ti["d2d_blocks"] * bb / world
        if world == 1 or not pool.c.flags & binding.F_NO_FUSE:   # one fused kernel: links in parallel
            # floor = the slowest replica's own links (PCIe out / in of its tier, NVLink in);
            # every rank waits for it at the closing barrier
            floor = max(max(ti["d2h_of"][r] * bb / peaks["d2h"], ti["h2d_of"][r] * bb / peaks["h2d"],
                            ti["p2p_to"][r] * bb / nvl) for r in range(len(ti["d2h_of"])))
            tmin[3] += floor / G
            byts[3] += d2h_b + h2d_b + p2p_b
        else:
            tmin[3] += d2h_b / peaks["d2h"] / G
            byts[3] += d2h_b
            tmin[4] += max(h2d_b / peaks["h2d"], p2p_b / nvl) / G
            byts[4] += h2d_b + p2p_b
        tmin[7] += d2d_b / hbm_peak / G
        byts[7] += d2d_b
    for k in tmin:                       # per step
        tmin[k] /= args.steps
        byts[k] /= args.steps
    dom = int(np.argmax(ph))
    dname = names[dom]
    if dom in tmin and ph[dom] > 0 and byts[dom] > 0:
        t = ph[dom] * 1e-6
        achieved = byts[dom] / t / 1e9
        peak = byts[dom] / tmin[dom] / G if tmin[dom] > 0 else achieved
        bound = ("hbm" if dom == 7 else "pcie (full duplex)" if (world == 1 or not pool.c.flags & binding.F_NO_FUSE)
                 else ("pcie" if dom == 3 else "pcie/nvlink"))
        psrc = (peak_src if dom == 7 else
                f"measured in this run: pinned cudaMemcpyAsync 1 GiB (d2h {peaks['d2h']:.1f}, h2d {peaks['h2d']:.1f}"
                f" GB/s{'' if world == 1 else ' per GPU with all %d GPUs copying at once; one GPU alone: d2h %.1f, h2d %.1f' % (world, peaks_alone['d2h'], peaks_alone['h2d'])}"
                f"); peak = bytes / floor, floor = max over replicas and links of (link bytes / link peak)")
    else:
        byts_d = metadata_bytes(st0, tr.n_slots, sum_nb, 0)
        achieved = byts_d / (ph[dom] * 1e-6) / 1e9 if ph[dom] > 0 else 0.0
        peak, bound, psrc = hbm_peak, "hbm", peak_src
    # traffic: DRAM bytes per launch, from the committed ncu --set full capture of the same
    # kernel (profiles/r1e_move_traffic.json: measured DRAM / algorithmic bytes of two
    # launch) applied to this run's algorithmic bytes per launch
    traffic = None
    if dom == 3 and world == 1:          # the captured kernel is the single-process fused one
        try:
            with open(os.path.join(ROOT, "profiles", "r1e_move_traffic.json")) as f:
                traffic = round(byts[3] * json.load(f)["ratio_dram_to_algorithmic"])
        except (OSError, KeyError, ValueError):
            traffic = None
    roofline = {"bound": bound, "kernel": dname, "achieved": round(achieved, 2), "peak": round(peak, 1),
                "unit": "GB/s", "frac": round(achieved / peak, 4) if peak else None, "traffic": traffic,
                "traffic_source": "ncu --set full capture (profiles/r1e_move_traffic.json) ratio x algorithmic bytes",
                "share_of_step": round(float(ph[dom] / ph.sum()), 4), "peak_source": psrc}
    kv_paths = kv_path_microbench(pool, torch, peaks, hbm_peak) if rank == 0 else None
    if world > 1:
        dist.barrier()                   # peers keep their pools mapped until rank 0 is done
    moved = {
        "d2h_gb_per_step": round(dstat["evict_to_host"] * bb / args.steps / 1e9, 3),
        "h2d_gb_per_step": round(dstat["h2d_blocks"] * bb / args.steps / 1e9, 3),
        "p2p_gb_per_step": round(dstat["p2p_blocks"] * bb / args.steps / 1e9, 3),
        "d2d_gb_per_step": round(dstat["compact_blocks"] * bb / args.steps / 1e9, 3),
    }
    sched_us = float(ph[0] + ph[1] + ph[2] + ph[6] + ph[8])
    tick_lat = (sched_tick_latency(cfg, tr, torch, dev, args.preroll + args.warmup, args.sched_ticks, flush)
                if rank == 0 and world == 1 and args.sched_ticks > 0 else None)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(tracegen.get_config(args.config), tracegen.make_trace(tracegen.get_config(args.config)),
                           args.cpu_seconds)
    line = {
        "metric": metric, "value": round(value, 4), "unit": "ticks/s (10k-program ticks, summed over GPUs)",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic",
        "config": {"workload": args.config, "programs": tr.n_slots, "replicas": world, "replicas_per_gpu": 1,
                   "kv": "Qwen3-32B GQA L64 H8 D128 bf16, 16-token blocks (4 MiB)",
                   "hbm_blocks": pool.NB, "host_blocks": pool.NH, "preroll_ticks": args.preroll,
                   "engine_fill": "off (engine stand-in, not a hot-path row)",
                   "l2": "256 MiB memset before every timed step (inside the timed region)",
                   "parallelism": f"dp{world} (one replica per GPU)"},
        "clocks": clocks,
        "e2e": {"value": round(e2e_value, 4), "unit": "ticks/s", "h2d_bytes_per_step": int(h2d / args.steps),
                "d2h_bytes_per_step": int(d2h / args.steps), "events_per_step": round(n_events / args.steps, 1),
                "note": "API mode (serving-engine path): per step the tick's event batch H2D from host memory, "
                        "validation + apply + tick on the device, decisions D2H; same ticks as value"},
        # per tick: tick_front, pause+restore (cooperative), plan (one launch of R 8-CTA
        # clusters), movement (1 fused kernel; multi-GPU: barrier, fused kernel, barrier), close
        # (compaction copies only when compaction is configured; off in this workload)
        "gpu_launches": args.steps * (5 if world == 1 else 7),
        "roofline": roofline,
        "phases_us_per_step": {n: round(float(v), 1) for n, v in zip(names, ph)},
        "sched_us_per_tick": round(sched_us, 1),
        # NEXT-1: STP cost ledger of the timed ticks (token-ms per step) and
        # the Cost_unused < c_min bound of PAPER.md:415 (replica-ticks checked / violated)
        "stp_ledger_token_ms_per_step": {k[5:]: int(dstat[k] / args.steps) for k in binding.LEDGER_KEYS
                                         if k.startswith("cost_")},
        "unused_bound": {"checks": dstat["unused_bound_checks"], "violations": dstat["unused_bound_violations"]},
        "sched_tick": tick_lat,
        "kv_moved": moved,
        "kv_paths": kv_paths,
        "cpu_baseline": cpu,
        "step_ms": step_ms,
    }
    if rank == 0:
        JSON_OUT.write(json.dumps(line) + "\n")
        JSON_OUT.flush()
    pool.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
