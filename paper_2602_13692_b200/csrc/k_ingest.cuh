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
// tool result, release (PAPER.md:160-162 reason/act loop; readings A3, A18).  Every
// field is loaded up front (one memory round trip), the trace script entries of the
// current turn in a second one.
__device__ __forceinline__ SlotNow ingest_slot(const Dev& d, int p, i64 T) {
  u8 st = d.status[p];
  const u8 sat = d.satisfied[p];
  u8 ph = d.phase[p];
  u32 c = d.c[p];
  const u32 t = d.turn[p];
  const u32 gd0 = d.gen_done[p];
  const i64 tr0 = d.tool_return[p];
  i64 as = d.acting_since[p];
  const u32 busy = d.busy[p], pend0 = d.pend[p];
  const u32 base = d.t_off[p], base1 = d.t_off[p + 1];
  SlotNow o{c, as, st, ph, d.placement[p], d.home[p], 0};
  if (st == TA_UNARRIVED || st == TA_STOPPED) return o;
  const u32 nturns = base1 - base;
  const u32 g = d.t_g[base + t], dtool = d.t_d[base + t], res = d.t_o[base + t];
  i64 tr = tr0;
  u32 tt = t, gd = gd0;
  bool wrote_gd = false, wrote_tool = false;
  if (st == TA_REASONING && sat) {
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
    d.pend[p] = pend0 + res;             // ... waits for its prefill
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
  u8 st, ph, fl, pad[5];       // fl: EVF_*
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
  i64 as = 0;
  for (int q = 0; q < n; ++q) {
    const u32 i = idx(q);
    const ta_event e = ev[i];
    if (e.kind == TA_EV_ARRIVE || e.kind == TA_EV_DECODE || e.kind == TA_EV_TOOL_RESULT) {
      const u64 cn = e.kind == TA_EV_ARRIVE ? (u64)e.tokens : c + e.tokens;
      if (cn > cap && !(e.kind == TA_EV_ARRIVE && st != TA_UNARRIVED)) return ((ull)i << 8) | TA_E_INVAL;
      if (e.kind == TA_EV_ARRIVE && st == TA_UNARRIVED && (u64)e.tokens < (u64)d.sb * (u64)d.bt)
        return ((ull)i << 8) | TA_E_INVAL;           // the prompt starts with the shared prefix
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
  o->st = st; o->ph = ph; o->fl = (u8)(fl | EVF_OWNER);
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
      d.uid[p] = o.uid; d.c_kv[p] = 0; d.paused_since[p] = k;
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

// Steps 0 (release frees) + 1 (footprint) + 2 (contribution, L_eff) for one slot,
// by one warp, given the slot's values after step 0 (identical in every lane).  The
// block-table row is scanned with 16-byte loads; counts come from ballot/popc,
// prefix_hbm from the first non-HBM entry.  Loads accumulate into Lacc (k_pause
// publishes L).  Closed-loop arrivals are initialised by k_restore.
__device__ __forceinline__ void footprint_warp(const Dev& d, int p, i64 T, int verb, const SlotNow& v) {
  const u32 lane = lane_id();
  u32* row = d.loc + (size_t)p * d.MAXBP;
  if (!verb && v.released) {                      // free every block of a STOPPED program (A26)
    const int h = v.home;
    const u32 nbv = ceil_div_u32(v.c, d.bt);
    for (u32 j = lane; j < nbv; j += 32) {
      u32 e = row[j];
      if (e == LOC_NONE) continue;
      if (j < d.sb) {                              // shared prefix: a reference, not owned
        row[j] = LOC_NONE;
        continue;
      }
      if (e & LOC_HOST) {
        u32 s = e & ~LOC_HOST;
        atomicOr(&d.host_free[(size_t)h * d.NHW + (s >> 5)], 1u << (s & 31));
      } else {
        atomicOr(&d.hbm_free[(size_t)h * d.NBW + (e >> 5)], 1u << (e & 31));
      }
      row[j] = LOC_NONE;
    }
    if (lane == 0) {
      d.home[p] = -1;
      d.released[p] = 0;
      d.nb[p] = d.n_hbm[p] = d.n_host[p] = d.prefix_hbm[p] = d.contrib[p] = 0;
      d.rb[p] = 0xFFFFFFFFu;
      d.fpl[p] = -1;
    }
    return;
  }
  const u8 st = (u8)v.st;
  if (st != TA_PAUSED && st != TA_REASONING && st != TA_ACTING) {
    if (lane == 0) {
      d.nb[p] = d.n_hbm[p] = d.n_host[p] = d.prefix_hbm[p] = d.contrib[p] = 0;
      d.rb[p] = 0xFFFFFFFFu;
      d.fpl[p] = -1;
    }
    return;
  }
  const u32 nbv = ceil_div_u32(v.c, d.bt);
  u32 n_h = 0, n_s = 0, first = 0xFFFFFFFFu;
  for (u32 j0 = 0; j0 < nbv; j0 += 512) {         // four independent 16-B loads per lane in flight
    uint4 q[4];
#pragma unroll
    for (int h2 = 0; h2 < 4; ++h2) {
      const u32 j = j0 + h2 * 128 + lane * 4;
      q[h2] = make_uint4(LOC_NONE, LOC_NONE, LOC_NONE, LOC_NONE);
      if (j < nbv) q[h2] = *reinterpret_cast<const uint4*>(row + j);
    }
#pragma unroll
    for (int h2 = 0; h2 < 4; ++h2) {
      const u32 j = j0 + h2 * 128 + lane * 4;
      u32 e[4] = {q[h2].x, q[h2].y, q[h2].z, q[h2].w};
      u32 lfirst = 0xFFFFFFFFu;
#pragma unroll
      for (int t = 3; t >= 0; --t) {
        if (j + t < nbv) {
          bool h = is_hbm(e[t]);
          n_h += h;
          n_s += is_host(e[t]);
          if (!h) lfirst = j + t;
        }
      }
      first = min(first, lfirst);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    n_h += __shfl_xor_sync(FULL_MASK, n_h, o);
    n_s += __shfl_xor_sync(FULL_MASK, n_s, o);
    first = min(first, __shfl_xor_sync(FULL_MASK, first, o));
  }
  if (lane == 0) {
    d.nb[p] = nbv;
    d.n_hbm[p] = n_h;
    d.n_host[p] = n_s;
    d.prefix_hbm[p] = first == 0xFFFFFFFFu ? nbv : first;
    const u8 ph = (u8)v.ph;
    u32 cb = contrib_of(d, nbv, ph, v.as, T);
    d.contrib[p] = cb;
    // candidate lists of the planner kernels (unordered appends; consumers sort by key
    // and slot, so the append order never reaches a result)
    u32 rbv = 0xFFFFFFFFu;
    i8 pl = -1;
    if (st == TA_PAUSED) {
      rbv = restore_bucket(d, ph, nbv);
      atomicAdd(&d.rhist[rbv], 1u);
    } else {
      pl = (i8)v.pl;
      if (!verb) atomicAdd(&d.Lacc[pl], (ull)cb);     // commutative u64 sum
      d.act_list[(size_t)pl * d.N + atomicAdd(&d.act_cnt[pl], 1u)] = (u32)p;
    }
    const int h = v.home;
    if (n_h > d.sb && h >= 0) d.ec_list[(size_t)h * d.N + atomicAdd(&d.ec_cnt[h], 1u)] = (u32)p;
    d.rb[p] = rbv;
    d.fpl[p] = pl;
  }
}

// The slot's current values (API mode, verbs: step 0 already applied or absent).
__device__ __forceinline__ SlotNow slot_now(const Dev& d, int p) {
  return SlotNow{d.c[p], d.acting_since[p], d.status[p], d.phase[p], d.placement[p], d.home[p], d.released[p]};
}

// broadcast lane 0's SlotNow to the warp
__device__ __forceinline__ SlotNow bcast(SlotNow v) {
  v.c = __shfl_sync(FULL_MASK, v.c, 0);
  v.as = (i64)__shfl_sync(FULL_MASK, (ull)v.as, 0);
  v.st = __shfl_sync(FULL_MASK, v.st, 0);
  v.ph = __shfl_sync(FULL_MASK, v.ph, 0);
  v.pl = __shfl_sync(FULL_MASK, v.pl, 0);
  v.home = __shfl_sync(FULL_MASK, v.home, 0);
  v.released = __shfl_sync(FULL_MASK, v.released, 0);
  return v;
}

// Trace mode: steps 0-2 of the tick in one kernel, one warp per slot (ingest by
// lane 0, then the warp's footprint scan of the same slot).
__global__ void __launch_bounds__(256) k_tick_front(Dev d) {
  const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= d.N) return;
  const i64 T = d.ctr->tick * d.dt;
  if (p == 0 && lane_id() == 0) {
    d.ctr->T = T;
    if (d.ctr->err != TA_E_PEER) d.ctr->err = TA_OK;   // a failed verb's status does not stop the tick
  }
  SlotNow v{};
  if (lane_id() == 0) v = ingest_slot(d, p, T);
  footprint_warp(d, p, T, 0, bcast(v));
}

// API mode and verbs: steps 1-2 (the events were applied by k_ev_*).  Verbs
// act on the state left by the last tick, at its time T (no ingest, L kept).
__global__ void __launch_bounds__(256) k_footprint(Dev d, int verb) {
  const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= d.N || (!verb && d.ctr->err != TA_OK)) return;
  const i64 T = verb ? d.ctr->T : d.ctr->now_ms;
  if (!verb && p == 0 && lane_id() == 0) d.ctr->T = T;
  SlotNow v{};
  if (lane_id() == 0) v = slot_now(d, p);
  footprint_warp(d, p, T, verb, bcast(v));
}
