// k_sched.cuh — tick bookkeeping, step 3 (pause pass) and step 4 (restore pass).
#pragma once
#include "common.cuh"

#define RESTORE_CHUNK 512u   // queue entries selected per sorted chunk of the restore loop

// Start of a tick: reset per-tick counters and the load accumulators.
__global__ void k_begin(Dev d) {
  int t = threadIdx.x;
  if (t == 0) {
    d.ctr->stops = 0;
    d.ctr->restore_cnt = 0;
    d.ctr->n_arr = 0;
    d.ctr->T = d.api_mode ? d.ctr->now_ms : d.ctr->tick * d.dt;
    d.ctr->t_d2h = d.ctr->t_h2d = d.ctr->t_p2p = d.ctr->t_d2d = d.ctr->t_fetch = 0;
  }
  if (t < d.R) {
    d.L[t] = 0;
    d.pause_cnt[t] = 0; d.f_cnt[t] = 0; d.s_cnt[t] = 0; d.ev_cnt[t] = 0;
    d.evd_cnt[t] = 0; d.fed_cnt[t] = 0; d.fld_cnt[t] = 0; d.dfh_cnt[t] = 0; d.dfs_cnt[t] = 0;
    d.cpd_cnt[t] = 0;
  }
}

// Step 3, one CTA per replica (reading A6): if the decayed
// load exceeds lambda_max*C, pause the minimal prefix of the actives in S_pause
// order (acting first, shortest first) whose contributions cover Delta C.  Only the
// prefix is materialized: buckets (tau, nb) select it exactly, then a stable CTA
// radix sort orders it by the full key.
__global__ void __launch_bounds__(CTA, 1) k_pause(Dev d) {
  __shared__ u32 s_big[8192 + 1];
  __shared__ u32 s_tmp[NWARP + 1];
  const int r = blockIdx.x;
  const ull Lr = d.L[r];
  const ull cap = (ull)d.cap_max[r];
  if (Lr <= cap) return;
  const u32 dC = (u32)(Lr - cap);
  const int N = d.N;
  const u32 NBK = d.nbk, sh = d.nb_shift;
  u64* ka = d.ska + (size_t)r * N;
  u64* kb = d.skb + (size_t)r * N;
  u32* va = d.sva + (size_t)r * N;
  u32* vb = d.svb + (size_t)r * N;
  auto pred = [&](int i) {
    u8 s = d.status[i];
    return (s == TA_REASONING || s == TA_ACTING) && d.placement[i] == r;
  };
  auto bucket = [&](int i) { return (u32)(d.phase[i] == TA_PHASE_R) * NBK + (d.nb[i] >> sh); };
  const u32 T = cta_bucket_threshold(N, 2 * NBK, 0, dC, s_big, s_tmp, pred, bucket,
                                     [&](int i) { return d.contrib[i]; });
  u32 n = cta_ordered_gather(N, s_tmp,
      [&](int i) { return pred(i) && bucket(i) <= T; },
      [&](u32 pos, int i) {
        ka[pos] = pause_key(d.phase[i], d.nb[i], d.acting_since[i]);
        va[pos] = (u32)i;
      });
  int res = cta_radix_sort(ka, va, kb, vb, (int)n, s_big, s_tmp);
  const u32* sv = res ? vb : va;
  u32* cum = (u32*)(res ? ka : kb);             // free key buffer as u32 scratch
  for (u32 i = threadIdx.x; i < n; i += CTA) cum[i] = d.contrib[sv[i]];
  __syncthreads();
  cta_incl_scan_array(cum, (int)n, s_tmp);
  // minimal prefix with sum >= dC: m = #(cum < dC) + 1, clipped to n
  u32 m = (u32)upper_bound_u32(cum, (int)n, dC - 1) + 1;
  bool shortfall = false;
  if (m > n) { m = n; shortfall = true; }
  const u32 k = (u32)d.ctr->tick;
  for (u32 i = threadIdx.x; i < m; i += CTA) {
    u32 p = sv[i];
    d.status[p] = TA_PAUSED;
    d.placement[p] = -1;
    d.paused_since[p] = k;
    d.satisfied[p] = 0;
    d.pause_list[(size_t)r * N + i] = p;
  }
  if (threadIdx.x == 0) {
    d.pause_cnt[r] = m;
    d.L[r] = Lr - (m ? cum[m - 1] : 0);
    atomicAdd(&d.stats[ST_PAUSES], (ull)m);
    if (shortfall) atomicAdd(&d.stats[ST_SHORTFALLS], 1ull);
  }
}

// Step 4, one CTA (readings A8-A11, A14): the global queue
// in S_restore order, consumed sequentially: each program goes to the least-loaded
// replica that is below lambda_min*C and stays <= lambda_max*C.  The queue is
// materialized chunk by chunk (exact bucket prefix + stable radix sort), since the
// loop usually stops early.  Warp 0 runs the loop: lane r holds L[r]; the argmin is
// one __reduce_min_sync over the packed key (L << 6 | [r != home] << 5 | r), which
// fits 32 bits because a candidate has L < cap_min <= NB < 2^17.
__global__ void __launch_bounds__(CTA, 1) k_restore(Dev d) {
  __shared__ u32 s_big[8192 + 1];
  __shared__ u32 s_tmp[NWARP + 1];
  __shared__ u32 s_stop;
  const int N = d.N, R = d.R;
  const u32 NBK = d.nbk, sh = d.nb_shift;
  u64* ka = d.ska + (size_t)R * N;
  u64* kb = d.skb + (size_t)R * N;
  u32* va = d.sva + (size_t)R * N;
  u32* vb = d.svb + (size_t)R * N;
  const u32 lane = lane_id();
  const bool w0 = threadIdx.x < 32;
  ull Lr = 0, cmax = 0, cmin = 0, maxcap = 0;
  if (w0) {
    Lr = lane < (u32)R ? d.L[lane] : 0;
    cmax = lane < (u32)R ? (ull)d.cap_max[lane] : 0;
    cmin = lane < (u32)R ? (ull)d.cap_min[lane] : 0;
    maxcap = cmax;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      ull t = __shfl_xor_sync(FULL_MASK, maxcap, o);
      maxcap = t > maxcap ? t : maxcap;
    }
  }
  u32 cnt = 0, over = 0;
  auto pred = [&](int i) { return d.status[i] == TA_PAUSED; };
  auto bucket = [&](int i) { return (u32)(d.phase[i] == TA_PHASE_A) * NBK + (d.nb[i] >> sh); };
  u32 lo = 0;
  while (true) {
    const u32 T = cta_bucket_threshold(N, 2 * NBK, lo, RESTORE_CHUNK, s_big, s_tmp, pred, bucket,
                                       [](int) { return 1u; });
    u32 n = cta_ordered_gather(N, s_tmp,
        [&](int i) { if (!pred(i)) return false; u32 b = bucket(i); return b >= lo && b <= T; },
        [&](u32 pos, int i) {
          ka[pos] = restore_key(d.phase[i], d.nb[i], d.paused_since[i]);
          va[pos] = (u32)i;
        });
    int res = cta_radix_sort(ka, va, kb, vb, (int)n, s_big, s_tmp);
    const u32* q = res ? vb : va;
    if (w0) {
      bool stop = false;
      for (u32 base = 0; base < n && !stop; base += 32) {
        u32 i = base + lane;
        u32 pl = i < n ? q[i] : 0;
        u32 crl = i < n ? d.contrib[pl] : 0;
        int hml = i < n ? d.home[pl] : -1;
        u32 phl = i < n ? d.phase[pl] : 0;
        u32 mcount = min(32u, n - base);
        for (u32 jj = 0; jj < mcount; ++jj) {
          u32 cr = __shfl_sync(FULL_MASK, crl, jj);
          if (cr > maxcap) { ++over; continue; }       // can never fit (reading A9)
          bool fits = lane < (u32)R && Lr < cmin && Lr + cr <= cmax;
          if (__ballot_sync(FULL_MASK, fits) == 0) { stop = true; break; }
          int hm = __shfl_sync(FULL_MASK, hml, jj);
          u32 key = fits ? (((u32)Lr << 6) | ((u32)((int)lane != hm) << 5) | lane) : 0xFFFFFFFFu;
          u32 t = __reduce_min_sync(FULL_MASK, key) & 31;
          if (lane == t) Lr += cr;
          if (lane == jj) {                       // the lane that holds the entry writes it
            d.status[pl] = phl == TA_PHASE_A ? TA_ACTING : TA_REASONING;
            d.placement[pl] = (i8)t;
            d.restore_pid[cnt] = pl;
            d.restore_dst[cnt] = t | ((u32)(hml + 1) << 8);   // dst | (home before + 1) << 8
          }
          ++cnt;
        }
      }
      if (lane == 0) s_stop = stop || T >= 2 * NBK - 1;
    }
    __syncthreads();
    if (s_stop) break;
    lo = T + 1;
    __syncthreads();
  }
  if (w0) {
    if (lane < (u32)R) d.L[lane] = Lr;
    if (lane == 0) {
      d.ctr->restore_cnt = cnt;
      atomicAdd(&d.stats[ST_RESTORES], (ull)cnt);
      atomicAdd(&d.stats[ST_OVERSIZED], (ull)over);
    }
  }
}
