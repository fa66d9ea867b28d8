"""ctypes binding over libta.so (include/ta.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libta.so; PyTorch is used
for device memory, pinned host memory and the CUDA stream.  There is no CPU
fallback: if libta.so or a CUDA device is missing, constructing a Pool raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# libta.so: the product build; libta_dev.so: the same sources with the development
# options compiled in (DEV_FLAGS; build.py).  TA_LIB: developer A/B aid (a variant of
# the product build made with build.py --out, inside this package).
LIB_PATH = os.path.join(HERE, os.path.basename(os.environ.get("TA_LIB", "libta.so")))
LIB_DEV_PATH = os.path.join(HERE, os.path.basename(os.environ.get("TA_LIB_DEV", "libta_dev.so")))
MAXR = 32
HANDLE_BYTES = 192   # TA_HANDLE_BYTES

TA_OK, TA_E_INVAL, TA_E_NOMEM, TA_E_DUP_ID, TA_E_UNKNOWN_PROGRAM = 0, 1, 2, 3, 4
TA_E_ILLEGAL_TRANSITION, TA_E_CAPACITY, TA_E_TRUNCATED, TA_E_CUDA, TA_E_PEER, TA_E_STATE = 5, 6, 7, 8, 9, 10
F_TRACE_MODE, F_FILL, F_NO_GRAPH, F_TIMING, F_COPY_BULK, F_NO_FUSE, F_PINNED_ROUTING = 1, 2, 4, 8, 16, 32, 64
F_REQUEST_AWARE = 128
F_SMALL_PATHS = 256                  # test aid: small runs take the full-size code paths
F_DECIDE_ONLY = 512                  # measurement aid: decisions without block copies
F_JITTER = 1024                      # test aid: random CTA delays at entry and after barriers
F_FULL_SCAN = 2048                   # test aid: the footprint pass counts every live row
DEV_FLAGS = F_TIMING | F_PINNED_ROUTING | F_REQUEST_AWARE | F_SMALL_PATHS | F_JITTER | F_FULL_SCAN   # libta_dev.so
F_NO_BULK_DEFAULT = 1 << 30          # binding-only: do not turn TA_F_COPY_BULK on
STATUS_NAMES = {0: "OK", 1: "E_INVAL", 2: "E_NOMEM", 3: "E_DUP_ID", 4: "E_UNKNOWN_PROGRAM",
                5: "E_ILLEGAL_TRANSITION", 6: "E_CAPACITY", 7: "E_TRUNCATED", 8: "E_CUDA",
                9: "E_PEER", 10: "E_STATE"}


class TAError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("elem_bytes", C.c_int32), ("block_tokens", C.c_int32), ("layout", C.c_int32),
                ("n_replicas", C.c_int32), ("replicas_here", C.c_int32), ("first_replica", C.c_int32),
                ("max_programs", C.c_int32), ("max_blocks_per_program", C.c_int32),
                ("max_trace_turns", C.c_int32), ("hbm_blocks", C.c_int64), ("host_blocks", C.c_int64),
                ("delta_t_ms", C.c_int64), ("decay_unit_ms", C.c_int64),
                ("lambda_max_q16", C.c_uint32), ("lambda_min_q16", C.c_uint32),
                ("decay_q32", C.c_uint64 * 64), ("decode_tok_per_s", C.c_int32),
                ("compact_every", C.c_int32), ("flags", C.c_uint32), ("prefill_chunk_tokens", C.c_int32),
                ("prefill_chunk_ms", C.c_int32), ("shared_prefix_tokens", C.c_int32),
                ("n_prefixes", C.c_int32), ("prefix_tokens", C.c_int32 * 8)]


class Buffers(C.Structure):
    _fields_ = [("hbm_pool", C.c_void_p * MAXR), ("host_pool", C.c_void_p * MAXR),
                ("dev_workspace", C.c_void_p), ("host_workspace", C.c_void_p)]


class Event(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("pid", C.c_uint32), ("uid", C.c_uint32),
                ("tokens", C.c_uint32), ("t_ms", C.c_int64)]


EVENT_DTYPE = np.dtype([("kind", "<u4"), ("pid", "<u4"), ("uid", "<u4"), ("tokens", "<u4"), ("t_ms", "<i8")])
assert EVENT_DTYPE.itemsize == C.sizeof(Event) == 24

DECISION_DTYPE = np.dtype([("kind", "<u4"), ("pid", "<u4"), ("src", "<i4"), ("dst", "<i4"),
                           ("blocks", "<u4"), ("to_host", "<u4"), ("dropped", "<u4"),
                           ("hit_tok", "<u4"), ("peer_tok", "<u4"), ("host_tok", "<u4"),
                           ("miss_tok", "<u4"), ("new_tok", "<u4")])
assert DECISION_DTYPE.itemsize == 48

STAT_KEYS = ("ticks", "arrivals", "stops", "pauses", "restores", "oversized_skips", "shortfalls",
             "evict_blocks", "evict_to_host", "evict_dropped", "fetch_blocks", "p2p_blocks",
             "h2d_blocks", "recompute_blocks", "new_blocks", "compact_blocks", "stalls",
             "hit_tok", "peer_tok", "host_tok", "miss_tok", "new_tok", "fill_tok",
             "imbalance_max_blocks", "imbalance_last_blocks")


LEDGER_KEYS = ("cost_decode", "cost_prefill", "cost_recompute", "cost_unused", "cost_caching",
               "unused_bound_checks", "unused_bound_violations",
               "overshoot_blocks", "overshoot_max_blocks",       # + the NEXT-4 guard counters
               "prefix_blocks")                                  # + NEXT-3 prompt blocks (A51)


class Stats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in STAT_KEYS] + [
        ("L", C.c_uint64 * MAXR), ("hbm_used", C.c_uint64 * MAXR), ("host_used", C.c_uint64 * MAXR),
        ("block_bytes", C.c_uint64)] + [(k, C.c_uint64) for k in LEDGER_KEYS]


class TickInfo(C.Structure):
    _fields_ = [("tick", C.c_int64)] + [(k, C.c_uint32) for k in (
        "decisions", "d2h_blocks", "h2d_blocks", "p2p_blocks", "d2d_blocks", "fetch_blocks")] + [
        (k, C.c_uint32 * 32) for k in ("d2h_of", "h2d_of", "p2p_to")]


class TraceView(C.Structure):
    _fields_ = [("n_slots", C.c_int32), ("n_initial", C.c_int32)] + [
        (k, C.POINTER(C.c_uint32)) for k in ("uid", "p0", "turn_off", "g", "d_ms", "o")] + [
        ("prefix_id", C.POINTER(C.c_uint8))]


_VIEW_FIELDS = [
    ("uid", C.c_uint32), ("c", C.c_uint32), ("c_kv", C.c_uint32), ("paused_since", C.c_uint32),
    ("step_count", C.c_uint32), ("turn", C.c_uint32), ("gen_done", C.c_uint32),
    ("status", C.c_uint8), ("phase", C.c_uint8), ("satisfied", C.c_uint8),
    ("placement", C.c_int8), ("home", C.c_int8),
    ("acting_since", C.c_int64), ("tool_return", C.c_int64),
    ("loc", C.c_uint32), ("hbm_free", C.c_uint32), ("host_free", C.c_uint32),
    ("owner_hbm", C.c_uint32), ("owner_host", C.c_uint32), ("L", C.c_uint64),
    ("nb", C.c_uint32), ("n_hbm", C.c_uint32), ("n_host", C.c_uint32), ("prefix_hbm", C.c_uint32),
    ("contrib", C.c_uint32), ("scalars", C.c_int64),
    ("prefix_id", C.c_uint8), ("prefix_ref", C.c_uint32), ("prefix_blk", C.c_uint32)]


class StateView(C.Structure):
    _fields_ = [(n, C.POINTER(t)) for n, t in _VIEW_FIELDS]


_libs = {}


def lib(dev: bool = False):
    """Load libta.so, or libta_dev.so with dev=True (fails loudly: there is no fallback
    path)."""
    path = LIB_DEV_PATH if dev else LIB_PATH
    if path not in _libs:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python -m paper_2602_13692_b200.build`")
        L = C.CDLL(path)
        vp, i32, i64, u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32
        sig = {
            "ta_workspace_bytes": [vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)],
            "ta_block_bytes": [vp, C.POINTER(C.c_size_t)],
            "ta_init_pool": [vp, vp, vp, vp, C.POINTER(vp)],
            "ta_load_trace": [vp, vp],
            "ta_sched_step": [vp, i64, vp, i32, vp, i32, C.POINTER(i32)],
            "ta_pause": [vp, u32, u32, vp, i32, C.POINTER(i32)],
            "ta_resume": [vp, u32, i32, vp, i32, C.POINTER(i32)],
            "ta_migrate": [vp, u32, i32, vp, i32, C.POINTER(i32)],
            "ta_set_health": [vp, i32, i32, vp, i32, C.POINTER(i32)],
            "ta_stats": [vp, vp],
            "ta_phase_times": [vp, C.POINTER(C.c_float), i32],
            "ta_debug_phase_stamps": [vp, C.POINTER(C.c_uint64), i32],
            "ta_debug_counters": [vp, C.POINTER(C.c_uint64), i32],
            "ta_verify_content": [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)],
            "ta_debug_state": [vp, i32, vp],
            "ta_move_blocks": [vp, i32, i32, i32, vp, vp, i32],
            "ta_last_tick": [vp, vp],
            "ta_set_copy_bulk": [vp, i32],
            "ta_export_pool_handle": [vp, vp],
            "ta_import_peer_pool": [vp, i32, vp],
            "ta_destroy": [vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.ta_last_error.argtypes = [vp]
        L.ta_last_error.restype = C.c_char_p
        L.ta_abi_version.restype = C.c_int32
        _libs[path] = L
    return _libs[path]


EXPORTED = ("ta_workspace_bytes", "ta_block_bytes", "ta_init_pool", "ta_load_trace", "ta_sched_step",
            "ta_pause", "ta_resume", "ta_migrate", "ta_stats", "ta_phase_times", "ta_verify_content",
            "ta_debug_state", "ta_export_pool_handle", "ta_import_peer_pool", "ta_destroy",
            "ta_last_error", "ta_abi_version", "ta_move_blocks", "ta_last_tick", "ta_set_copy_bulk",
            "ta_debug_phase_stamps", "ta_set_health", "ta_debug_counters")
def e_any(spans):
    return any(e for _, e in spans.values())


SPAN_KERNELS = ("front", "pause_restore", "plan", "move", "close", "compact")   # KSpan k order
DEBUG_COUNTERS = ("radix_sort", "bitonic_sort", "rank_sort", "list_global", "plan_f_global", "plan_e_global",
                  "plan_v_global", "plan_fst_global", "restore_chunks", "evict_ticks",
                  "front_rows_counted", "front_row_entries")
MOVE_D2D, MOVE_P2P, MOVE_D2H, MOVE_H2D = 1, 2, 3, 4


def decay_q32(x: int) -> list:
    """F[k] = floor(2^32 * x^-k) (eq. 7 time decay; f(t) = x^-t,
    PAPER.md:458), by repeated floor division (floor(floor(a/x)/x) = floor(a/x^2))."""
    F = [1 << 32]
    for _ in range(63):
        F.append(F[-1] // x)
    return F


def make_config(cfg: dict, n_programs: int, max_turns: int, trace_mode: bool = True, fill: bool = True,
                flags: int = 0, replicas_here: int | None = None, first_replica: int = 0) -> Config:
    from tracegen import KV_SHAPES   # parameters only
    kv = KV_SHAPES[cfg.get("kv", "toy")] if isinstance(cfg.get("kv", "toy"), str) else cfg["kv"]
    c = Config()
    c.n_layers, c.n_kv_heads, c.head_dim, c.elem_bytes = (kv["n_layers"], kv["n_kv_heads"],
                                                          kv["head_dim"], kv.get("elem_bytes", 2))
    c.block_tokens = cfg["block_tokens"]
    c.layout = cfg.get("layout", 0)
    c.n_replicas = cfg["n_replicas"]
    c.replicas_here = cfg["n_replicas"] if replicas_here is None else replicas_here
    c.first_replica = first_replica
    c.max_programs = n_programs
    c.max_blocks_per_program = -(-cfg["max_ctx"] // cfg["block_tokens"])
    c.max_trace_turns = max(1, max_turns)
    c.hbm_blocks = cfg["hbm_blocks"]
    c.host_blocks = cfg["host_blocks"]
    c.delta_t_ms = cfg["delta_t_ms"]
    c.decay_unit_ms = cfg["decay_unit_ms"]
    c.lambda_max_q16 = cfg["lambda_max_q16"]
    c.lambda_min_q16 = cfg["lambda_min_q16"]
    table = cfg.get("decay_table") or decay_q32(cfg["decay_x"])
    if cfg.get("request_aware", False):              # baseline: no program view (reading A46)
        flags |= F_REQUEST_AWARE
        table = [0] * 64
    for k, v in enumerate(table):
        c.decay_q32[k] = v
    c.decode_tok_per_s = cfg["decode_tok_per_s"]
    c.compact_every = cfg.get("compact_every", 0)
    c.prefill_chunk_tokens = cfg.get("prefill_chunk_tokens", 2048)   # STP ledger (NEXT-1)
    c.prefill_chunk_ms = cfg.get("prefill_chunk_ms", 100)
    from tracegen import prefix_spec  # parameters only
    spec = prefix_spec(cfg)                                             # NEXT-3 prompts (A51)
    c.shared_prefix_tokens = 0
    c.n_prefixes = len(spec)
    for k, (t, _) in enumerate(spec):
        c.prefix_tokens[k] = t
    # TMA bulk copies are the default engine (measured faster or equal on every path);
    # pass flags=F_NO_BULK_DEFAULT to keep the 128-bit load/store engine
    if not flags & F_NO_BULK_DEFAULT:
        flags |= F_COPY_BULK
    if cfg.get("pinned_routing", False):
        flags |= F_PINNED_ROUTING
    c.flags = (flags & ~F_NO_BULK_DEFAULT) | (F_TRACE_MODE if trace_mode else 0) | (F_FILL if fill else 0)
    return c


def _u32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


class Pool:
    """One libta context plus the torch-owned buffers it runs on."""

    def __init__(self, cfg: dict, n_programs: int, max_turns: int = 1, trace_mode: bool = True,
                 fill: bool = True, flags: int = 0, device: int = 0, host_blocks: int | None = None,
                 replicas_here: int | None = None, first_replica: int = 0, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libta needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.cfg = dict(cfg)
        if host_blocks is not None:
            self.cfg["host_blocks"] = host_blocks
        self.device = torch.device("cuda", device)
        flags |= int(os.environ.get("TA_EXTRA_FLAGS", "0"))   # developer aid (e.g. TA_F_NO_GRAPH)
        self.c = make_config(self.cfg, n_programs, max_turns, trace_mode, fill, flags,
                             replicas_here, first_replica)
        L = self.L = lib(dev=(self.c.flags & DEV_FLAGS) != 0)
        dev_b, host_b, blk = C.c_size_t(), C.c_size_t(), C.c_size_t()
        self._chk(L.ta_workspace_bytes(C.byref(self.c), C.byref(dev_b), C.byref(host_b)), "workspace")
        L.ta_block_bytes(C.byref(self.c), C.byref(blk))
        self.block_bytes = blk.value
        self.N = n_programs
        self.R = self.c.n_replicas
        self.MAXB = self.c.max_blocks_per_program
        self.K = self.c.n_prefixes                      # NEXT-3 shared prompts
        self.SBM = max([1] + [self.c.prefix_tokens[k] // self.c.block_tokens for k in range(self.K)])
        self.NB, self.NH = self.c.hbm_blocks, self.c.host_blocks
        self.first, self.here = self.c.first_replica, self.c.replicas_here
        self.dev_ws = torch.empty(dev_b.value, dtype=torch.uint8, device=self.device)
        self.host_ws = torch.empty(host_b.value, dtype=torch.uint8, pin_memory=True)
        self.hbm = {}
        self.host = {}
        b = Buffers()
        for r in range(self.first, self.first + self.here):
            self.hbm[r] = torch.empty(self.NB * self.block_bytes, dtype=torch.uint8, device=self.device)
            b.hbm_pool[r] = self.hbm[r].data_ptr()
            if self.NH > 0:
                self.host[r] = torch.empty(self.NH * self.block_bytes, dtype=torch.uint8, pin_memory=True)
                b.host_pool[r] = self.host[r].data_ptr()
        b.dev_workspace = self.dev_ws.data_ptr()
        b.host_workspace = self.host_ws.data_ptr()
        self.buffers = b
        # a dedicated (capturable) stream: the legacy default stream cannot host a CUDA graph
        self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
        self.ctx = C.c_void_p()
        with torch.cuda.device(self.device):
            st = L.ta_init_pool(C.byref(self.c), C.byref(b), C.c_void_p(self.stream.cuda_stream), None,
                                C.byref(self.ctx))
        if st != TA_OK:
            raise TAError(st, "ta_init_pool failed")
        self.dec_buf = np.zeros(4 * n_programs + self.R + 64, dtype=DECISION_DTYPE)

    def reset(self, flags: int | None = None):
        """Destroy the context and create a fresh one over the same buffers (the
        workspace is re-initialised: every slot UNARRIVED, all blocks free).
        `flags` replaces the context's TA_F_* flags (same buffers and workspace size)."""
        import torch
        self.close()
        if flags is not None:
            self.c.flags = flags
            self.L = lib(dev=(self.c.flags & DEV_FLAGS) != 0)
        self.ctx = C.c_void_p()
        with torch.cuda.device(self.device):
            st = self.L.ta_init_pool(C.byref(self.c), C.byref(self.buffers),
                                    C.c_void_p(self.stream.cuda_stream), None, C.byref(self.ctx))
        if st != TA_OK:
            raise TAError(st, "ta_init_pool (reset) failed")

    # ------------------------------------------------------------------ helpers
    def _chk(self, st, what):
        if st != TA_OK:
            msg = self.L.ta_last_error(self.ctx).decode() if getattr(self, "ctx", None) else ""
            raise TAError(st, f"{what}: {msg}")

    def close(self):
        if getattr(self, "ctx", None) and self.ctx.value:
            self.L.ta_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ ABI calls
    def load_trace(self, tr):
        self._trace_arrays = [np.ascontiguousarray(a, dtype=np.uint32)
                              for a in (tr.uid, tr.p0, tr.turn_off, tr.g, tr.d_ms, tr.o)]
        v = TraceView()
        v.n_slots = tr.n_slots
        v.n_initial = tr.n_initial
        for name, a in zip(("uid", "p0", "turn_off", "g", "d_ms", "o"), self._trace_arrays):
            setattr(v, name, _u32p(a))
        from tracegen import prefix_ids  # input data: each slot's shared prompt (NEXT-3)
        self._trace_kp = np.ascontiguousarray(prefix_ids(self.cfg, tr), dtype=np.uint8)
        v.prefix_id = self._trace_kp.ctypes.data_as(C.POINTER(C.c_uint8))
        self._chk(self.L.ta_load_trace(self.ctx, C.byref(v)), "ta_load_trace")

    def step(self, now_ms: int = -1, events=None, decisions: bool = True, raise_on_error=True):
        """One ta_sched_step.  Returns (status, decisions ndarray or None)."""
        n_ev = 0
        evp = None
        if isinstance(events, np.ndarray):              # EVENT_DTYPE batch: passed as is
            if events.dtype != EVENT_DTYPE or not events.flags.c_contiguous:
                raise ValueError("event arrays must be C-contiguous EVENT_DTYPE")
            if len(events):
                evp, n_ev = C.c_void_p(events.ctypes.data), len(events)
        elif events:
            arr = (Event * len(events))()
            for i, e in enumerate(events):
                arr[i].kind, arr[i].pid, arr[i].uid, arr[i].tokens, arr[i].t_ms = e
            evp, n_ev = arr, len(events)
        n_out = C.c_int32(0)
        if decisions:
            st = self.L.ta_sched_step(self.ctx, now_ms, evp, n_ev, self.dec_buf.ctypes.data,
                                     len(self.dec_buf), C.byref(n_out))
        else:
            st = self.L.ta_sched_step(self.ctx, now_ms, evp, n_ev, None, 0, None)
        if st not in (TA_OK,) and raise_on_error and st in (TA_E_CUDA, TA_E_PEER, TA_E_INVAL, TA_E_STATE):
            self._chk(st, "ta_sched_step")
        if not decisions or st != TA_OK:
            return st, None
        return st, self.dec_buf[:n_out.value].copy()

    def _verb(self, fn, *args):
        n_out = C.c_int32(0)
        st = fn(self.ctx, *args, self.dec_buf.ctypes.data, len(self.dec_buf), C.byref(n_out))
        if st in (TA_E_CUDA, TA_E_PEER):
            self._chk(st, fn.__name__)
        return st, (self.dec_buf[:n_out.value].copy() if st == TA_OK else None)

    def pause(self, pid, mode=0):
        return self._verb(self.L.ta_pause, pid, mode)

    def resume(self, pid, replica=-1):
        return self._verb(self.L.ta_resume, pid, replica)

    def migrate(self, pid, dst):
        return self._verb(self.L.ta_migrate, pid, dst)

    def set_health(self, replica, healthy):
        return self._verb(self.L.ta_set_health, replica, 1 if healthy else 0)

    def stats(self) -> dict:
        s = Stats()
        self._chk(self.L.ta_stats(self.ctx, C.byref(s)), "ta_stats")
        out = {k: getattr(s, k) for k in STAT_KEYS + LEDGER_KEYS}
        out["L"] = list(s.L[:self.R])
        out["hbm_used"] = list(s.hbm_used[:self.R])
        out["host_used"] = list(s.host_used[:self.R])
        out["block_bytes"] = s.block_bytes
        return out

    def set_copy_bulk(self, on: bool):
        self._chk(self.L.ta_set_copy_bulk(self.ctx, 1 if on else 0), "ta_set_copy_bulk")

    def last_tick(self) -> dict:
        t = TickInfo()
        self._chk(self.L.ta_last_tick(self.ctx, C.byref(t)), "ta_last_tick")
        return {k: (list(getattr(t, k))[:self.R] if k.endswith(("_of", "_to")) else getattr(t, k))
                for k, _ in TickInfo._fields_}

    def phase_times(self):
        a = (C.c_float * 9)()
        self._chk(self.L.ta_phase_times(self.ctx, a, 9), "ta_phase_times")
        return list(a)

    def phase_stamps(self, absolute: bool = False):
        """Globaltimer stamps (ns) of the planner kernels' phases in the last tick (TA_F_TIMING):
        {kernel: [(phase index, ns since that kernel's first stamp), ...]}; plan_cta1 / plan_cta3
        are cluster ranks 1 and 3 of replica 0's planner cluster."""
        a = (C.c_uint64 * 256)()
        self._chk(self.L.ta_debug_phase_stamps(self.ctx, a, 256), "ta_debug_phase_stamps")
        out = {}
        names = ("pause", "restore", "plan", "close", "plan_cta1", "plan_cta3", "front_cta0", "front_last")
        # kernel spans (first CTA start, last thread-0 exit) live in slot 3, entries 16..27
        spans = {n: (a[3 * 32 + 16 + 2 * i], a[3 * 32 + 17 + 2 * i]) for i, n in enumerate(SPAN_KERNELS)}
        probes = [a[3 * 32 + 28 + i] for i in range(4)]
        for i in range(16, 32):
            a[3 * 32 + i] = 0
        first = {}
        for k, name in enumerate(names):
            v = [a[32 * k + i] for i in range(32) if a[32 * k + i] and not a[32 * k + i] >> 62]
            first[name] = min(v) if v else 0
        # the planner's cluster ranks share the leader's time origin
        first["plan"] = first["plan_cta1"] = first["plan_cta3"] = min(
            [x for x in (first["plan"], first["plan_cta1"], first["plan_cta3"]) if x] or [0])
        first["front_cta0"] = first["front_last"] = min(
            [x for x in (first["front_cta0"], first["front_last"]) if x] or [0])
        if absolute:                       # one origin for every kernel: the tick's first stamp
            t0 = min([x for x in first.values() if x] or [0])
            first = {k: t0 for k in first}
        for k, name in enumerate(names):
            v = [(i, a[32 * k + i]) for i in range(32) if a[32 * k + i] and not a[32 * k + i] >> 62]
            out[name] = [(i, c - first[name]) for i, c in v] if v else []
            # sizes recorded next to the stamps (bit 62 set): ("n<i>", value)
            out[name] += [(f"n{i}", a[32 * k + i] & ((1 << 62) - 1)) for i in range(32) if a[32 * k + i] >> 62 == 1]
        t0 = min([b for b, e in spans.values() if e] or [0])
        out["spans"] = [(n, round((b - t0) / 1e3, 1), round((e - t0) / 1e3, 1))
                        for n, (b, e) in spans.items() if e]      # (kernel, start us, end us)
        out["spans"] += [(f"probe{i}", round((t - t0) / 1e3, 1), round((t - t0) / 1e3, 1))
                         for i, t in enumerate(probes) if t and e_any(spans)]
        return out

    def debug_counters(self) -> dict:
        """Size-branch counters (ta_debug_counters): how often each large-size path ran."""
        a = (C.c_uint64 * 16)()
        self._chk(self.L.ta_debug_counters(self.ctx, a, 16), "ta_debug_counters")
        return {n: int(a[i]) for i, n in enumerate(DEBUG_COUNTERS)}

    def verify_content(self):
        bad, seen = C.c_uint64(), C.c_uint64()
        self._chk(self.L.ta_verify_content(self.ctx, C.byref(bad), C.byref(seen)), "ta_verify_content")
        return bad.value, seen.value

    def _view_arrays(self, fields=None):
        N, R, NB, NH, MAXB = self.N, self.R, self.NB, self.NH, self.MAXB
        NBW, NHW = -(-NB // 32), -(-NH // 32)
        shapes = dict(uid=N, c=N, c_kv=N, paused_since=N, step_count=N, turn=N, gen_done=N, status=N,
                      phase=N, satisfied=N, placement=N, home=N, acting_since=N, tool_return=N,
                      loc=N * MAXB, hbm_free=R * NBW, host_free=max(1, R * NHW), owner_hbm=R * NB,
                      owner_host=max(1, R * NH), L=R, nb=N, n_hbm=N, n_host=N, prefix_hbm=N, contrib=N,
                      scalars=4, prefix_id=N, prefix_ref=R * max(1, self.K),
                      prefix_blk=R * max(1, self.K) * self.SBM)
        npt = {C.c_uint32: np.uint32, C.c_uint8: np.uint8, C.c_int8: np.int8, C.c_int64: np.int64,
               C.c_uint64: np.uint64}
        return {n: np.zeros(shapes[n], dtype=npt[t]) for n, t in _VIEW_FIELDS if fields is None or n in fields}

    def debug_download(self, fields=None) -> dict:
        """Device state as numpy arrays (all fields, or only the named ones)."""
        arrs = self._view_arrays(fields)
        v = StateView()
        for n, t in _VIEW_FIELDS:
            if n in arrs:
                setattr(v, n, arrs[n].ctypes.data_as(C.POINTER(t)))
        self._chk(self.L.ta_debug_state(self.ctx, 0, C.byref(v)), "ta_debug_state")
        if "loc" in arrs:
            arrs["loc"] = arrs["loc"].reshape(self.N, self.MAXB)
        return arrs

    def debug_upload(self, arrs: dict):
        v = StateView()
        keep = {}
        for n, t in _VIEW_FIELDS:
            if n in ("nb", "n_hbm", "n_host", "prefix_hbm", "contrib") or n not in arrs:
                continue
            a = np.ascontiguousarray(arrs[n]).ravel()
            keep[n] = a
            setattr(v, n, a.ctypes.data_as(C.POINTER(t)))
        self._chk(self.L.ta_debug_state(self.ctx, 1, C.byref(v)), "ta_debug_state upload")

    def move_blocks(self, kind: int, src_r: int, dst_r: int, src_idx, dst_idx):
        """ta_move_blocks with device index tensors (torch int32/uint32 on this device)."""
        n = int(src_idx.numel())
        self._chk(self.L.ta_move_blocks(self.ctx, kind, src_r, dst_r, src_idx.data_ptr(),
                                       dst_idx.data_ptr(), n), "ta_move_blocks")

    def export_handle(self) -> bytes:
        h = (C.c_char * HANDLE_BYTES)()
        self._chk(self.L.ta_export_pool_handle(self.ctx, h), "ta_export_pool_handle")
        return bytes(h)

    def import_peer(self, replica: int, handle: bytes):
        h = (C.c_char * HANDLE_BYTES).from_buffer_copy(handle)
        self._chk(self.L.ta_import_peer_pool(self.ctx, replica, h), "ta_import_peer_pool")

    def read_block(self, r: int, tier: str, idx: int) -> np.ndarray:
        """Bytes of one KV block as uint64 words, shaped [2L, bt, H, D/4] (test aid)."""
        import torch
        c = self.c
        nseg = 2 * c.n_layers
        seg = self.block_bytes // nseg
        nblk = self.NB if tier == "hbm" else self.NH
        buf = self.hbm[r] if tier == "hbm" else self.host[r]
        self.torch.cuda.synchronize(self.device)
        if c.layout == 0:
            v = buf.view(nseg, nblk, seg)[:, idx, :]
        else:
            v = buf.view(nblk, nseg, seg)[idx]
        a = v.contiguous().cpu().numpy().view(np.uint64)
        return a.reshape(nseg, c.block_tokens, c.n_kv_heads, c.head_dim // 4)
