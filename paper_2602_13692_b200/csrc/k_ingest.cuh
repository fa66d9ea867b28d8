// k_ingest.cuh — step 0 (ingest) and steps 1-2 (footprint, decayed effective load).
#pragma once
#include "common.cuh"

// Step 0, trace mode, for one slot: decode during the last interval, tool call /
// tool result, release (PAPER.md:160-162 reason/act loop; readings A3, A18).
__device__ __forceinline__ void ingest_slot(const Dev& d, int p, i64 T) {
  u8 st = d.status[p];
  if (st == TA_UNARRIVED || st == TA_STOPPED) return;
  const u32 base = d.t_off[p];
  const u32 nturns = d.t_off[p + 1] - base;
  u32 c = d.c[p];
  u8 ph = d.phase[p];
  if (st == TA_REASONING && d.satisfied[p]) {
    const u32 d_tick = (u32)(((i64)d.rate * d.dt) / 1000);
    u32 t = d.turn[p];
    u32 g = d.t_g[base + t];
    u32 gd = d.gen_done[p];
    u32 left = g - gd;
    u32 dd = min(d_tick, left);
    c += dd;
    gd += dd;
    d.gen_done[p] = gd;
    if (gd == g) {
      if (t == nturns - 1) {             // last turn: release
        d.c[p] = c;
        d.status[p] = TA_STOPPED;
        d.placement[p] = -1;
        d.satisfied[p] = 0;
        d.released[p] = 1;
        atomicAdd(&d.ctr->stops, 1u);
        return;
      }
      ph = TA_PHASE_A;                   // tool call: Reasoning -> Acting
      st = TA_ACTING;
      i64 took = d.rate == 0 ? 0 : ((i64)left * 1000 + d.rate - 1) / d.rate;
      i64 as = T - d.dt + took;
      d.acting_since[p] = as;
      d.tool_return[p] = as + (i64)d.t_d[base + t];
      d.step_count[p] += 1;
    }
  }
  if (ph == TA_PHASE_A && (st == TA_ACTING || st == TA_PAUSED) && T >= d.tool_return[p]) {
    u32 t = d.turn[p];
    c += d.t_o[base + t];                 // tool result (tools run while paused)
    d.turn[p] = t + 1;
    d.gen_done[p] = 0;
    ph = TA_PHASE_R;
    d.tool_return[p] = INT64_MAX;
    if (st == TA_ACTING) st = TA_REASONING;
  }
  d.c[p] = c;
  d.phase[p] = ph;
  d.status[p] = st;
}

// Step 0, API mode: validate the event batch in order, all-or-nothing, then apply
// it (one thread: event batches are short and order-dependent).  Tentative
// status/phase of touched pids are tracked in the ska scratch (pid-indexed).
__global__ void k_apply_events(Dev d, const ta_event* ev, int n_ev, int apply) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  u8* tst = d.evs;                       // [N] tentative status (zeroed marks between calls)
  u8* tph = tst + d.N;                   // [N] tentative phase
  u8* touched = tph + d.N;               // [N]
  u32* tc = d.evc;                       // [N] tentative context length
  const u64 cap = (u64)d.MAXB * (u64)d.bt;   // contexts are bounded by max_ctx (reading A35)
  int err = TA_OK;
  for (int i = 0; i < n_ev && err == TA_OK; ++i) {
    u32 pid = ev[i].pid;
    if (pid >= (u32)d.N) { err = TA_E_UNKNOWN_PROGRAM; break; }
    if (!touched[pid]) {
      touched[pid] = 1; tst[pid] = d.status[pid]; tph[pid] = d.phase[pid]; tc[pid] = d.c[pid];
    }
    u8 st = tst[pid], ph = tph[pid];
    const u32 kd = ev[i].kind;
    if (kd == TA_EV_ARRIVE || kd == TA_EV_DECODE || kd == TA_EV_TOOL_RESULT) {
      u64 c = kd == TA_EV_ARRIVE ? (u64)ev[i].tokens : (u64)tc[pid] + ev[i].tokens;
      if (c > cap && !(kd == TA_EV_ARRIVE && st != TA_UNARRIVED)) { err = TA_E_INVAL; break; }
      tc[pid] = (u32)c;
    }
    switch (ev[i].kind) {
      case TA_EV_ARRIVE:
        if (st != TA_UNARRIVED) err = TA_E_DUP_ID; else { tst[pid] = TA_PAUSED; tph[pid] = TA_PHASE_R; }
        break;
      case TA_EV_DECODE:
        if (st != TA_REASONING) err = TA_E_ILLEGAL_TRANSITION;
        break;
      case TA_EV_TOOL_CALL:
        if (st != TA_REASONING) err = TA_E_ILLEGAL_TRANSITION;
        else if (ev[i].t_ms < 0 || ev[i].t_ms > (i64)AS_MAX) err = TA_E_INVAL;
        else { tst[pid] = TA_ACTING; tph[pid] = TA_PHASE_A; }
        break;
      case TA_EV_TOOL_RESULT:
        if (ph != TA_PHASE_A || (st != TA_ACTING && st != TA_PAUSED)) err = TA_E_ILLEGAL_TRANSITION;
        else { tph[pid] = TA_PHASE_R; if (st == TA_ACTING) tst[pid] = TA_REASONING; }
        break;
      case TA_EV_RELEASE:
        if (st == TA_UNARRIVED) err = TA_E_UNKNOWN_PROGRAM; else tst[pid] = TA_STOPPED;
        break;
      default:
        err = TA_E_INVAL;
    }
  }
  for (int i = 0; i < n_ev; ++i) {       // clear scratch marks
    u32 pid = ev[i].pid;
    if (pid < (u32)d.N) touched[pid] = 0;
  }
  d.ctr->err = err;
  if (err != TA_OK || !apply) return;
  const i64 k = d.ctr->tick;
  u32 arr = 0;
  for (int i = 0; i < n_ev; ++i) {
    u32 p = ev[i].pid;
    switch (ev[i].kind) {
      case TA_EV_ARRIVE:
        d.uid[p] = ev[i].uid; d.status[p] = TA_PAUSED; d.phase[p] = TA_PHASE_R;
        d.c[p] = ev[i].tokens; d.c_kv[p] = 0; d.paused_since[p] = (u32)k;
        d.placement[p] = -1; d.home[p] = -1; d.turn[p] = 0; d.gen_done[p] = 0;
        d.satisfied[p] = 0; d.step_count[p] = 0; d.acting_since[p] = 0;
        d.tool_return[p] = INT64_MAX;
        ++arr;
        break;
      case TA_EV_DECODE:
        d.c[p] += ev[i].tokens;
        break;
      case TA_EV_TOOL_CALL:
        d.phase[p] = TA_PHASE_A; d.status[p] = TA_ACTING; d.acting_since[p] = ev[i].t_ms;
        d.step_count[p] += 1;
        break;
      case TA_EV_TOOL_RESULT:
        d.c[p] += ev[i].tokens; d.phase[p] = TA_PHASE_R;
        if (d.status[p] == TA_ACTING) d.status[p] = TA_REASONING;
        break;
      case TA_EV_RELEASE:
        if (d.status[p] != TA_STOPPED) {
          d.status[p] = TA_STOPPED; d.placement[p] = -1; d.satisfied[p] = 0;
          d.released[p] = 1;
          d.ctr->stops += 1;
        }
        break;
    }
  }
  d.ctr->n_arr = arr;
}

// Steps 0 (release frees) + 1 (footprint) + 2 (contribution, L_eff) for one slot,
// by one warp.  The block-table row is scanned with 16-byte loads; counts come from
// ballot/popc, prefix_hbm from the first non-HBM entry.  Loads accumulate into Lacc
// (k_pause publishes L).  Closed-loop arrivals are initialised by k_restore.
__device__ __forceinline__ void footprint_warp(const Dev& d, int p, i64 T, int verb) {
  const u32 lane = lane_id();
  u32* row = d.loc + (size_t)p * d.MAXBP;
  if (!verb && d.released[p]) {                   // free every block of a STOPPED program (A26)
    const int h = d.home[p];
    const u32 nbv = ceil_div_u32(d.c[p], d.bt);
    for (u32 j = lane; j < nbv; j += 32) {
      u32 e = row[j];
      if (e == LOC_NONE) continue;
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
  const u8 st = d.status[p];
  if (st != TA_PAUSED && st != TA_REASONING && st != TA_ACTING) {
    if (lane == 0) {
      d.nb[p] = d.n_hbm[p] = d.n_host[p] = d.prefix_hbm[p] = d.contrib[p] = 0;
      d.rb[p] = 0xFFFFFFFFu;
      d.fpl[p] = -1;
    }
    return;
  }
  const u32 nbv = ceil_div_u32(d.c[p], d.bt);
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
    const u8 ph = d.phase[p];
    u32 cb = contrib_of(d, nbv, ph, d.acting_since[p], T);
    d.contrib[p] = cb;
    // candidate lists of the planner kernels (unordered appends; consumers sort by key
    // and slot, so the append order never reaches a result)
    u32 rbv = 0xFFFFFFFFu;
    i8 pl = -1;
    if (st == TA_PAUSED) {
      rbv = restore_bucket(d, ph, nbv);
      atomicAdd(&d.rhist[rbv], 1u);
    } else {
      pl = d.placement[p];
      if (!verb) atomicAdd(&d.Lacc[pl], (ull)cb);     // commutative u64 sum
      d.act_list[(size_t)pl * d.N + atomicAdd(&d.act_cnt[pl], 1u)] = (u32)p;
    }
    const int h = d.home[p];
    if (n_h > 0 && h >= 0) d.ec_list[(size_t)h * d.N + atomicAdd(&d.ec_cnt[h], 1u)] = (u32)p;
    d.rb[p] = rbv;
    d.fpl[p] = pl;
  }
}

// Trace mode: steps 0-2 of the tick in one kernel, one warp per slot (ingest by
// lane 0, then the warp's footprint scan of the same slot).
__global__ void __launch_bounds__(256) k_tick_front(Dev d) {
  const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= d.N) return;
  const i64 T = d.ctr->tick * d.dt;
  if (p == 0 && lane_id() == 0) d.ctr->T = T;
  if (lane_id() == 0) ingest_slot(d, p, T);
  __syncwarp();
  footprint_warp(d, p, T, 0);
}

// API mode and verbs: steps 1-2 (the events were applied by k_apply_events).  Verbs
// act on the state left by the last tick, at its time T (no ingest, L kept).
__global__ void __launch_bounds__(256) k_footprint(Dev d, int verb) {
  const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= d.N) return;
  const i64 T = verb ? d.ctr->T : d.ctr->now_ms;
  if (!verb && p == 0 && lane_id() == 0) d.ctr->T = T;
  footprint_warp(d, p, T, verb);
}
