// k_ingest.cuh — step 0 (ingest) and steps 1-2 (footprint, decayed effective load).
#pragma once
#include "common.cuh"

// A slot's values after step 0, handed from the ingesting lane to its warp.
struct SlotNow {
  u32 c;
  i64 as;          // acting_since
  int st, ph, pl, home, released;
};

// Step 0, trace mode, for one slot: decode during the last interval, tool call /
// tool result, release (PAPER.md:160-162 reason/act loop; readings A3, A18).  Split in
// two so the block-table row loads can be issued between them: ingest_load issues
// every program-table load of the slot (one memory round trip), ingest_apply the trace
// script loads of the current turn (a second one) and the state change.
struct SlotFields {
  i64 tr0, as;
  u32 c, t, gd0, busy, pend0, base, base1;
  u8 st, sat, ph;
  i8 pl, home;
};

__device__ __forceinline__ SlotFields ingest_load(const Dev& d, int p) {
  SlotFields f;
  f.st = d.status[p]; f.sat = d.satisfied[p]; f.ph = d.phase[p];
  f.c = d.c[p]; f.t = d.turn[p]; f.gd0 = d.gen_done[p];
  f.tr0 = d.tool_return[p]; f.as = d.acting_since[p];
  f.busy = d.busy[p]; f.pend0 = d.pend[p];
  f.base = d.t_off[p]; f.base1 = d.t_off[p + 1];
  f.pl = d.placement[p]; f.home = d.home[p];
  return f;
}

__device__ __forceinline__ SlotNow ingest_apply(const Dev& d, int p, i64 T, const SlotFields& f) {
  u8 st = f.st, ph = f.ph;
  u32 c = f.c;
  i64 as = f.as;
  const u32 t = f.t, gd0 = f.gd0, busy = f.busy, base = f.base;
  SlotNow o{c, as, st, ph, f.pl, f.home, 0};
  if (st == TA_UNARRIVED || st == TA_STOPPED) return o;
  const u32 nturns = f.base1 - base;
  const u32 g = d.t_g[base + t], dtool = d.t_d[base + t], res = d.t_o[base + t];
  i64 tr = f.tr0;
  u32 tt = t, gd = gd0;
  bool wrote_gd = false, wrote_tool = false;
  if (st == TA_REASONING && f.sat) {
    // decode after the engine's (re)prefill of the last materialize (reading A48)
    const i64 b = min((i64)busy, d.dt);
    const u32 d_tick = (u32)(((i64)d.rate * (d.dt - b)) / 1000);
    const u32 left = g - gd;
    const u32 dd = min(d_tick, left);
    c += dd;
    gd += dd;
    wrote_gd = true;
    if (gd == g) {
      if (t == nturns - 1) {             // last turn: release
        d.gen_done[p] = gd;
        d.c[p] = c;
        d.status[p] = TA_STOPPED;
        d.placement[p] = -1;
        d.satisfied[p] = 0;
        atomicAdd(&d.ctr->stops, 1u);
        o.c = c; o.st = TA_STOPPED; o.pl = -1; o.released = 1;
        return o;
      }
      ph = TA_PHASE_A;                   // tool call: Reasoning -> Acting
      st = TA_ACTING;
      const i64 took = d.rate == 0 ? 0 : ((i64)left * 1000 + d.rate - 1) / d.rate;
      as = T - d.dt + b + took;
      tr = as + (i64)dtool;
      d.acting_since[p] = as;
      d.step_count[p] += 1;
      wrote_tool = true;
    }
  }
  if (ph == TA_PHASE_A && (st == TA_ACTING || st == TA_PAUSED) && T >= tr) {
    c += res;                            // tool result (tools run while paused)
    d.pend[p] = f.pend0 + res;           // ... waits for its prefill
    tt = t + 1;
    gd = 0;
    wrote_gd = true;
    ph = TA_PHASE_R;
    tr = INT64_MAX;
    wrote_tool = true;
    if (st == TA_ACTING) st = TA_REASONING;
    d.turn[p] = tt;
  }
  if (wrote_gd) d.gen_done[p] = gd;
  if (wrote_tool) d.tool_return[p] = tr;
  d.c[p] = c;
  d.phase[p] = ph;
  d.status[p] = st;
  o.c = c; o.as = as; o.st = st; o.ph = ph;
  return o;
}

// Step 0, API mode (SURVEY.md §8(c) event table): the batch
// ev[0, n) is validated in order, all-or-nothing, then applied, in parallel over
// programs.  Events of different programs commute; a program's events are a small
// state machine over (status, phase, c) run in batch order.  The first illegal event
// of the batch (lowest index) is the first illegal event of some program's sequence,
// so the batch error is the minimum over programs of (index, code).
//   k_ev_count   per event: events per pid; out-of-range pids are errors
//   k_ev_single  pids with one event run it at once; the rest go to a list
//   k_ev_multi   one CTA: the list sorted by (pid, index); each pid's sequence run
//                in order; the batch status is decided (ctr->err)
//   k_ev_apply   per event: the owner of each pid writes the final state (only if
//                the batch is legal); per-pid counters are cleared
// Later kernels of the tick return at once when ctr->err != TA_OK (state unchanged).
struct EvRes {                 // final state of one program after its events (owner event)
  i64 as;                      // acting_since (if a TOOL_CALL ran)
  u32 c, uid, calls, pend;     // pend: tokens waiting for prefill (prompt, tool results; A48)
  u8 st, ph, fl, kp, pad[4];   // fl: EVF_*; kp: shared prompt of an ARRIVE (A51)
};
static_assert(sizeof(EvRes) == 32, "EvRes layout (workspace carving)");
enum { EVF_OWNER = 1, EVF_ARRIVE = 2, EVF_CALL = 4 };

// Run the events of pid `p` (indices idx[0, n)) from its current state; returns the
// (index << 8 | code) of the first illegal event, or ~0 and the final state in *o.
template <typename Idx>
__device__ ull ev_run(const Dev& d, const ta_event* ev, u32 p, int n, Idx idx, EvRes* o) {
  const u64 cap = (u64)d.MAXB * (u64)d.bt;   // contexts are bounded by max_ctx (reading A35)
  u8 st = d.status[p], ph = d.phase[p];
  u64 c = d.c[p];
  u32 uid = d.uid[p], calls = 0, fl = 0, pend = d.pend[p];
  u8 kp = d.kp[p];
  i64 as = 0;
  for (int q = 0; q < n; ++q) {
    const u32 i = idx(q);
    const ta_event e = ev[i];
    if (e.kind == TA_EV_ARRIVE || e.kind == TA_EV_DECODE || e.kind == TA_EV_TOOL_RESULT) {
      const u64 cn = e.kind == TA_EV_ARRIVE ? (u64)e.tokens : c + e.tokens;
      if (cn > cap && !(e.kind == TA_EV_ARRIVE && st != TA_UNARRIVED)) return ((ull)i << 8) | TA_E_INVAL;
      if (e.kind == TA_EV_ARRIVE && st == TA_UNARRIVED) {   // its shared prompt (A51): none, the
        const i64 t = e.t_ms;                             // only one, or the one t_ms names
        if (d.K > 1 && (t < 0 || t >= d.K)) return ((ull)i << 8) | TA_E_INVAL;
        const u8 k = d.K == 0 ? (u8)KP_NONE : (d.K == 1 ? (u8)0 : (u8)t);
        if (k != KP_NONE && (u64)e.tokens < (u64)d.sbk[k] * (u64)d.bt)
          return ((ull)i << 8) | TA_E_INVAL;         // the prompt starts with its shared prefix
        kp = k;
      }
      if (!(e.kind == TA_EV_ARRIVE && st != TA_UNARRIVED)) c = cn;
    }
    switch (e.kind) {
      case TA_EV_ARRIVE:
        if (st != TA_UNARRIVED) return ((ull)i << 8) | TA_E_DUP_ID;
        st = TA_PAUSED; ph = TA_PHASE_R; uid = e.uid; fl |= EVF_ARRIVE; calls = 0; fl &= ~EVF_CALL;
        pend = e.tokens;
        break;
      case TA_EV_DECODE:
        if (st != TA_REASONING) return ((ull)i << 8) | TA_E_ILLEGAL_TRANSITION;
        break;
      case TA_EV_TOOL_CALL:
        if (st != TA_REASONING) return ((ull)i << 8) | TA_E_ILLEGAL_TRANSITION;
        if (e.t_ms < 0 || e.t_ms > (i64)AS_MAX) return ((ull)i << 8) | TA_E_INVAL;
        st = TA_ACTING; ph = TA_PHASE_A; as = e.t_ms; ++calls; fl |= EVF_CALL;
        break;
      case TA_EV_TOOL_RESULT:
        if (ph != TA_PHASE_A || (st != TA_ACTING && st != TA_PAUSED)) return ((ull)i << 8) | TA_E_ILLEGAL_TRANSITION;
        ph = TA_PHASE_R;
        pend += e.tokens;
        if (st == TA_ACTING) st = TA_REASONING;
        break;
      case TA_EV_RELEASE:
        if (st == TA_UNARRIVED) return ((ull)i << 8) | TA_E_UNKNOWN_PROGRAM;
        st = TA_STOPPED;
        break;
      default:
        return ((ull)i << 8) | TA_E_INVAL;
    }
  }
  o->as = as; o->c = (u32)c; o->uid = uid; o->calls = calls; o->pend = pend;
  o->st = st; o->ph = ph; o->fl = (u8)(fl | EVF_OWNER); o->kp = kp;
  return ~0ull;
}

__global__ void __launch_bounds__(256) k_ev_count(const __grid_constant__ Dev d) {
  const int n = d.ctr->n_events;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u32 p = d.events[i].pid;
    d.evr[i].fl = 0;
    if (p >= (u32)d.N) atomicMin(&d.ctr->ev_err, ((ull)i << 8) | TA_E_UNKNOWN_PROGRAM);
    else atomicAdd(&d.ev_pcnt[p], 1u);
  }
}

__global__ void __launch_bounds__(256) k_ev_single(const __grid_constant__ Dev d) {
  const int n = d.ctr->n_events;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u32 p = d.events[i].pid;
    if (p >= (u32)d.N) continue;
    if (d.ev_pcnt[p] == 1) {
      EvRes o;
      const ull err = ev_run(d, d.events, p, 1, [&](int) { return (u32)i; }, &o);
      if (err != ~0ull) atomicMin(&d.ctr->ev_err, err);
      else d.evr[i] = o;
    } else {
      const u32 pos = atomicAdd(&d.ctr->ev_multi, 1u);
      d.ev_mk[pos] = ((u64)p << 32) | (u32)i;
    }
  }
}

__global__ void __launch_bounds__(CTA, 1) k_ev_multi(const __grid_constant__ Dev d) {
  __shared__ u32 s_big[8192 + 1];
  __shared__ u32 s_tmp[NWARP + 1];
  extern __shared__ __align__(16) char dsm[];
  SortSmem* sm = reinterpret_cast<SortSmem*>(dsm);
  const int nm = (int)d.ctr->ev_multi;
  if (nm > 0) {
    for (int i = threadIdx.x; i < nm; i += CTA) d.ev_mv[i] = 0;
    __syncthreads();
    const int res = cta_sort(d.ev_mk, d.ev_mv, d.ev_mk2, d.ev_mv2, nm, s_big, s_tmp, sm, sort_lim(d));
    const u64* k = res ? d.ev_mk2 : d.ev_mk;
    for (int q = threadIdx.x; q < nm; q += CTA) {     // one thread per program: its events in order
      const u32 p = (u32)(k[q] >> 32);
      if (q > 0 && (u32)(k[q - 1] >> 32) == p) continue;
      int len = 1;
      while (q + len < nm && (u32)(k[q + len] >> 32) == p) ++len;
      EvRes o;
      const ull err = ev_run(d, d.events, p, len, [&](int t) { return (u32)k[q + t]; }, &o);
      if (err != ~0ull) atomicMin(&d.ctr->ev_err, err);
      else d.evr[(u32)k[q]] = o;                       // owner: the program's first event
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const ull e = d.ctr->ev_err;
    d.ctr->err = e == ~0ull ? TA_OK : (i32)(e & 0xFF);
    d.ctr->ev_err = ~0ull;
    d.ctr->ev_multi = 0;
  }
}

__global__ void __launch_bounds__(256) k_ev_apply(const __grid_constant__ Dev d) {
  const int n = d.ctr->n_events;
  const bool ok = d.ctr->err == TA_OK;
  const u32 k = (u32)d.ctr->tick;
  u32 arr = 0, stops = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u32 p = d.events[i].pid;
    if (p >= (u32)d.N) continue;
    d.ev_pcnt[p] = 0;
    const EvRes o = d.evr[i];
    if (!ok || !(o.fl & EVF_OWNER)) continue;
    const u8 st0 = d.status[p];
    if (o.fl & EVF_ARRIVE) {              // _arrive (reading A12)
      d.uid[p] = o.uid; d.c_kv[p] = 0; d.paused_since[p] = k; d.kp[p] = o.kp;
      d.placement[p] = -1; d.home[p] = -1; d.turn[p] = 0; d.gen_done[p] = 0;
      d.satisfied[p] = 0; d.step_count[p] = 0; d.acting_since[p] = 0;
      d.tool_return[p] = INT64_MAX;
      d.busy[p] = 0;
      ++arr;
    }
    if (o.fl & EVF_CALL) d.acting_since[p] = o.as;
    d.step_count[p] = ((o.fl & EVF_ARRIVE) ? 0u : d.step_count[p]) + o.calls;
    d.c[p] = o.c;
    d.pend[p] = o.pend;
    d.phase[p] = o.ph;
    d.status[p] = o.st;
    if (o.st == TA_STOPPED && st0 != TA_STOPPED) {   // release
      d.placement[p] = -1; d.satisfied[p] = 0;
      d.released[p] = 1;
      ++stops;
    }
  }
  if (arr) atomicAdd(&d.ctr->n_arr, arr);
  if (stops) atomicAdd(&d.ctr->stops, stops);
}

// Steps 0 (release frees) + 1 (footprint) + 2 (contribution, L_eff), one CTA per 32
// slots (FP_SLOTS), four memory round trips for the whole CTA:
//   1. warp 0, lane l = slot base + l: the slot's program-table fields (coalesced SoA
//      loads), hence its row length nbo;
//   2. every thread: the block-table rows of the 32 slots as one flat list of 16-B
//      chunks, copied into shared memory with cp.async (LDGSTS: many loads in flight
//      per thread, no registers held) -- while warp 0 runs the ingest, whose trace
//      script loads overlap the row traffic;
//   3. every warp: a contiguous range of the staged chunks, per-slot counts (n_hbm,
//      n_host, first non-HBM entry) accumulated in registers and flushed to shared
//      memory when the slot changes; rows of programs released this tick are freed;
//   4. warp 0: nb, contribution (Eq. 7), and the planners' candidate lists, appended
//      with one atomic per distinct replica per warp (warp-aggregated).
// A slot whose chunks do not fit the staging buffer is read straight from global memory.
//
// Only entries j < nbo are read: nbo = ceil(c/bt) of the context the row was written
// for (before this tick's ingest).  A row holds no entry at or beyond nb(c) (invariant
// I2: blocks are allocated for j < nb only, and c never shrinks), so entries [nbo, nb)
// are NONE: n_hbm and n_host are the counts over [0, nbo), and the first non-HBM entry
// is the first one in [0, nbo), else nbo.
//
// Only rows written since the last pass are counted (d.dirty: every writer of loc sets
// it -- evictions and fetches in k_plan, satisfaction and compaction in k_close, the
// verbs, a state upload -- and this pass clears it).  A clean row of a live program
// has the counts and HBM prefix the last pass stored: c never shrinks, so its extra
// entries [nbo_then, nbo) are NONE, which add to neither count and leave
// min(first, nbo) where it was.  Its last-history-block class (entry ceil(c_kv/bt) - 1)
// is kept as well: c_kv changes only when the program is satisfied (k_close, which marks
// the row) or arrives (a fresh or released row, class 0), so a clean row's entry and
// index are the ones last classified.
#define FP_SLOTS 32                     // slots per CTA (one lane of warp 0 each)
#ifndef FP_THREADS
#define FP_THREADS 256                   // FP_SLOTS / (FP_THREADS / 32) slots per warp
#endif
#define FP_STAGE (FP_SLOTS * 104)        // 16-B chunks staged per CTA (416 block-table entries per slot, 52 KiB)
#define FP_SMEM (FP_STAGE * 16)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const u32 s = (u32)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n cp.async.wait_group 0;" ::: "memory");
}

// Entries of a slot's row that can hold KV: nb of its context if it is live.
__device__ __forceinline__ u32 row_len_of(const Dev& d, u8 st, u32 c) {
  return (st == TA_PAUSED || st == TA_REASONING || st == TA_ACTING) ? ceil_div_u32(c, d.bt) : 0u;
}

// mode 0: trace-mode tick (ingest + footprint); 1: API-mode tick (events applied);
// 2: verbs (state of the last tick, no L accumulation, no release handling)
template <int MODE>
__device__ __forceinline__ void footprint_cta(const Dev& d) {
  extern __shared__ __align__(16) uint4 s_stage[];   // [FP_STAGE], dynamic (FP_SMEM bytes)
  __shared__ u32 s_off[FP_SLOTS + 1];    // chunk offsets (exclusive prefix of ceil(nbo/4))
  __shared__ u32 s_nbo[FP_SLOTS], s_nh[FP_SLOTS], s_ns[FP_SLOTS], s_first[FP_SLOTS];
  __shared__ int s_home[FP_SLOTS];
  __shared__ u8 s_rel[FP_SLOTS], s_hcls[FP_SLOTS], s_kp[FP_SLOTS];
  __shared__ u32 s_jh[FP_SLOTS];          // entry of the last history block (ceil(c_kv/bt) - 1), or ~0
  __shared__ u8 s_dirty[FP_SLOTS];
  const int warp = threadIdx.x >> 5, lane = (int)lane_id();
  const int p0 = blockIdx.x * FP_SLOTS;
  const int p = p0 + lane;
  const bool w0 = warp == 0;
  if (MODE == 0 && TA_FLAG(d, TA_F_TIMING) && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && threadIdx.x < 32)
    d.pst[(blockIdx.x == 0 ? 6 : 7) * 32 + threadIdx.x] = 0;
  if (MODE == 0) { PSTAMP_B(6, 0, 0); PSTAMP_B(7, gridDim.x - 1, 0); }
  const i64 T = MODE == 0 ? d.ctr->tick * d.dt : (MODE == 1 ? d.ctr->now_ms : d.ctr->T);
  if (MODE == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    d.ctr->T = T;
    if (d.ctr->err != TA_E_PEER) d.ctr->err = TA_OK;   // a failed verb's status does not stop the tick
  }
  if (MODE == 1 && blockIdx.x == 0 && threadIdx.x == 0) d.ctr->T = T;
  // ---- 1. fields (warp 0)
  SlotFields f{};
  SlotNow v{};
  u32 nh_old = 0, ns_old = 0;
  u8 dv = 0, hc_old = 0;
  if (w0) {
    u32 nbo = 0;
    if (p < d.N) {
      dv = d.dirty[p] | (TA_FLAG(d, TA_F_FULL_SCAN) ? 1 : 0);   // a clean row keeps last pass's counts
      nh_old = d.n_hbm[p];
      ns_old = d.n_host[p];
      hc_old = d.hcls[p];
      if (MODE == 0) {
        f = ingest_load(d, p);
        nbo = row_len_of(d, f.st, f.c);
      } else {
        v = SlotNow{d.c[p], d.acting_since[p], d.status[p], d.phase[p], d.placement[p], d.home[p],
                    MODE == 1 ? (int)d.released[p] : 0};
        nbo = max(row_len_of(d, (u8)v.st, v.c), v.released ? ceil_div_u32(v.c, d.bt) : 0u);
      }
    }
    const u32 nch = dv ? (nbo + 3) >> 2 : 0u;     // only written rows are read
    const u32 inc = warp_incl_scan(nch);
    s_off[lane] = inc - nch;
    if (lane == 31) s_off[FP_SLOTS] = inc;
#ifndef TA_PROD_VARIANT
    if (MODE == 0) {                     // rows / entries read (ta_debug_counters; development build)
      const u32 nr = __reduce_add_sync(FULL_MASK, (dv && nbo) ? 1u : 0u);
      const u32 ne = __reduce_add_sync(FULL_MASK, dv ? nbo : 0u);
      if (lane == 0 && nr) { atomicAdd(&d.dbg[DBG_ROWS_COUNTED], (ull)nr); atomicAdd(&d.dbg[DBG_ROW_ENTRIES], (ull)ne); }
    }
#endif
    s_nbo[lane] = nbo;
    s_dirty[lane] = dv;
    s_nh[lane] = 0; s_ns[lane] = 0; s_first[lane] = 0xFFFFFFFFu;
    const u32 ckv = p < d.N ? d.c_kv[p] : 0u;
    s_kp[lane] = p < d.N ? d.kp[p] : (u8)KP_NONE;
    s_jh[lane] = ckv ? ceil_div_u32(ckv, d.bt) - 1 : 0xFFFFFFFFu;
    s_hcls[lane] = dv ? 0 : hc_old;      // clean: c_kv and the row are as last counted
  }
  __syncthreads();
  const u32* rows = d.loc + (size_t)p0 * d.MAXBP;
  if (MODE == 0) { PSTAMP_B(6, 0, 1); PSTAMP_B(7, gridDim.x - 1, 1); }
  // ---- 2 + 3. warps 1..7: each stages its slots' rows (slots w-1, w+6, ...) and counts
  //      them as soon as its own copies land; meanwhile warp 0 runs the ingest and the
  //      per-slot values that need no counts (a slot's chunks go to the staging buffer at
  //      s_off[slot] if they fit, else they are read straight from global memory)
  const bool valid = p < d.N;
  u32 nbv = 0, cb = 0, rbv = 0xFFFFFFFFu;
  bool live = false;
  if (!w0) {
    constexpr int CW = FP_THREADS / 32 - 1;       // counting warps
    for (int sl = warp - 1; sl < FP_SLOTS; sl += CW) {
      const u32 o = s_off[sl], nch = s_off[sl + 1] - o;
      if (s_dirty[sl] && o + nch <= FP_STAGE)    // clean rows are not read
        for (u32 c = lane; c < nch; c += 32) cp_async16(&s_stage[o + c], rows + (size_t)sl * d.MAXBP + 4 * c);
    }
    cp_async_wait_all();
    __syncwarp();
    for (int sl = warp - 1; sl < FP_SLOTS; sl += CW) {
      const u32 o = s_off[sl], nch = s_off[sl + 1] - o, nbo = s_nbo[sl];
      if (!s_dirty[sl]) continue;
      const bool staged = o + nch <= FP_STAGE;
      const uint4* grow = reinterpret_cast<const uint4*>(rows + (size_t)sl * d.MAXBP);
      u32 a_h = 0, a_n = 0, a_f = 0xFFFFFFFFu;   // HBM entries, non-HBM entries, first non-HBM
      const u32 jh = s_jh[sl];
#pragma unroll 4
      for (u32 c = lane; c < nch; c += 32) {
        uint4 q = staged ? s_stage[o + c] : grow[c];
        if (4 * c + 4 > nbo) {           // the row's last chunk: entries j >= nbo do not count
          const u32 k = nbo - 4 * c;     // 1..3
          if (k < 2) q.y = LOC_NONE;
          if (k < 3) q.z = LOC_NONE;
          q.w = LOC_NONE;
        }
        if ((jh >> 2) == c && jh < nbo) {  // the last history block's location class
          const u32 t = jh & 3;
          const u32 x = t == 0 ? q.x : t == 1 ? q.y : t == 2 ? q.z : q.w;
          s_hcls[sl] = is_hbm(x) ? 1 : (is_host(x) ? 2 : 0);
        }
        // HBM entries have bit 31 clear; host entries set it, and so does LOC_NONE
        const u32 n0 = q.x >> 31, n1 = q.y >> 31, n2 = q.z >> 31, n3 = q.w >> 31;
        const u32 nn = n0 + n1 + n2 + n3;
        a_h += 4 - nn;
        a_n += nn - (q.x == LOC_NONE) - (q.y == LOC_NONE) - (q.z == LOC_NONE) - (q.w == LOC_NONE);
        if (nn && a_f == 0xFFFFFFFFu) a_f = 4 * c + (n0 ? 0 : n1 ? 1 : n2 ? 2 : 3);
      }
      a_h = __reduce_add_sync(FULL_MASK, a_h);
      a_n = __reduce_add_sync(FULL_MASK, a_n);
      a_f = __reduce_min_sync(FULL_MASK, a_f);
      if (lane == 0) { s_nh[sl] = a_h; s_ns[sl] = a_n; s_first[sl] = a_f; }
    }
  } else {
    if (MODE == 0 && valid) v = ingest_apply(d, p, T, f);
    const bool rel = MODE != 2 && valid && v.released;
    s_rel[lane] = rel ? 1 : 0;
    s_home[lane] = v.home;
    const u8 st = (u8)v.st;
    live = valid && !rel && (st == TA_PAUSED || st == TA_REASONING || st == TA_ACTING);
    if (live) {
      nbv = ceil_div_u32(v.c, d.bt);
      cb = contrib_of(d, nbv, (u8)v.ph, v.as, T);
      if (st == TA_PAUSED) rbv = restore_bucket(d, (u8)v.ph, nbv);
    }
    // restore-bucket histogram: one atomic per distinct bucket per warp (thousands of
    // PAUSED slots fall in a few buckets; per-lane atomics serialize at L2)
    const u32 peers = __match_any_sync(FULL_MASK, rbv);
    if (rbv != 0xFFFFFFFFu && lane == (int)(__ffs(peers) - 1)) atomicAdd(&d.rhist[rbv], (u32)__popc(peers));
  }
  if (MODE == 0) { PSTAMP_B(6, 0, 2); PSTAMP_B(7, gridDim.x - 1, 2); }
  __syncthreads();
  if (MODE == 0) { PSTAMP_B(6, 0, 3); PSTAMP_B(7, gridDim.x - 1, 3); }
  if (!w0) {
    // ---- 3b. free every block of a program STOPPED this tick (A26), by its counting warp
    constexpr int CW = FP_THREADS / 32 - 1;
    for (int sl = warp - 1; sl < FP_SLOTS; sl += CW) {
      if (!s_rel[sl]) continue;
      const u32 o = s_off[sl], nbo = s_nbo[sl], nch = (nbo + 3) >> 2;
      const bool staged = s_dirty[sl] && o + nch <= FP_STAGE;   // a clean row was not staged
      const uint4* grow = reinterpret_cast<const uint4*>(rows + (size_t)sl * d.MAXBP);
      const int h = s_home[sl];
      const u32 sbs = sb_of(d, s_kp[sl]);
      u32* row = d.loc + (size_t)(p0 + sl) * d.MAXBP;
      for (u32 c = lane; c < nch; c += 32) {
        const uint4 q = staged ? s_stage[o + c] : grow[c];
        const u32 e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const u32 j = 4 * c + t;
          if (j >= nbo || e[t] == LOC_NONE) continue;
          if (j >= sbs) {                  // the shared prompt is a reference, not owned
            if (e[t] & LOC_HOST) {
              const u32 s2 = e[t] & ~LOC_HOST;
              atomicOr(&d.host_free[(size_t)h * d.NHW + (s2 >> 5)], 1u << (s2 & 31));
            } else {
              atomicOr(&d.hbm_free[(size_t)h * d.NBW + (e[t] >> 5)], 1u << (e[t] & 31));
            }
          }
          row[j] = LOC_NONE;
        }
      }
      if (h >= 0 && s_kp[sl] != KP_NONE) {  // it no longer uses its prompt on h: the last
        const u32 k = s_kp[sl];              // user frees the prompt's blocks (A51)
        u32 last = 0;
        if (lane == 0) last = atomicSub(&d.pref[(size_t)h * d.K + k], 1u) == 1u;
        if (__shfl_sync(FULL_MASK, last, 0)) prompt_free(d, h, k, lane, 32);
      }
    }
    return;
  }
  if (MODE == 0) { PSTAMP_B(6, 0, 4); PSTAMP_B(7, gridDim.x - 1, 4); }
  // ---- 4. per slot: derived values and candidate sets (warp 0)
  const u8 st = (u8)v.st;
  u32 n_h = 0, n_s = 0;
  int pl = -1;
  if (live) {
    if (st != TA_PAUSED) pl = v.pl;
    if (dv) {
      n_h = s_nh[lane];
      n_s = s_ns[lane];
      d.prefix_hbm[p] = min(s_first[lane], s_nbo[lane]);   // entries [nbo, nbv) are NONE
    } else {                             // clean: counts and prefix as last counted
      n_h = nh_old;
      n_s = ns_old;
    }
  } else if (valid) {
    d.prefix_hbm[p] = 0;
    if (MODE != 2 && v.released) d.home[p] = -1;
    if (MODE == 1 && v.released) d.released[p] = 0;
  }
  if (valid) {
    d.nb[p] = nbv; d.contrib[p] = cb;
    if (dv || !live) { d.n_hbm[p] = n_h; d.n_host[p] = n_s; }
    if (dv) d.dirty[p] = 0;
    d.rb[p] = rbv; d.hcls[p] = s_rel[lane] ? 0 : s_hcls[lane];
  }
  // candidate bitmaps: this CTA's 32 slots are word blockIdx.x of every replica's maps
  // (whole-word stores, every word rewritten each pass); the decayed load of the actives
  // (Eq. 7) summed per replica (one reduction per replica per warp, a commutative u64 add)
  const int h = v.home;
  const bool ecand = live && n_h > sb_of(d, s_kp[lane]) && h >= 0;
  const size_t wi = blockIdx.x;
  for (int r = 0; r < d.R; ++r) {
    const bool on_r = pl == r;
    const u32 wa = __ballot_sync(FULL_MASK, on_r);
    const u32 wr = __ballot_sync(FULL_MASK, on_r && st == TA_REASONING);
    const u32 we = __ballot_sync(FULL_MASK, ecand && h == r);
    const u32 sum = __reduce_add_sync(FULL_MASK, on_r ? cb : 0u);   // < 32 lanes x 2^23
    if (lane == 0) {
      d.act_bits[(size_t)r * d.NW + wi] = wa;
      d.reas_bits[(size_t)r * d.NW + wi] = wr;
      d.ec_bits[(size_t)r * d.NW + wi] = we;
      if (MODE != 2 && sum) atomicAdd(&d.Lacc[r], (ull)sum);
    }
  }
  if (MODE == 0) { PSTAMP_B(6, 0, 5); PSTAMP_B(7, gridDim.x - 1, 5); }
}

#define FP_GRID(N) (((N) + FP_SLOTS - 1) / FP_SLOTS)
#define FP_BLOCK FP_THREADS
#define FP_DSMEM FP_SMEM
__global__ void __launch_bounds__(FP_THREADS, 4) k_tick_front(Dev d) {   // 592 CTAs in one wave: 18,944 slots
  const ull t_in = gtimer();   // the CTA's first instruction (kernel span, timing mode)
  kspan_begin(d, KS_FRONT, t_in);
  jitter(d, 0u);
  footprint_cta<0>(d);
  kspan_end(d, KS_FRONT);
}
__global__ void __launch_bounds__(FP_THREADS) k_footprint(Dev d, int verb) {
  if (verb) {
    footprint_cta<2>(d);
  } else {
    if (d.ctr->err != TA_OK) return;
    footprint_cta<1>(d);
  }
}
