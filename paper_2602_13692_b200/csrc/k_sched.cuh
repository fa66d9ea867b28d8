// k_sched.cuh — tick bookkeeping, step 3 (pause pass) and step 4 (restore pass).
#pragma once
#include "common.cuh"

// Queue entries selected per sorted chunk of the restore loop: the loop usually stops
// at the head (steady state) or runs long (bursts), so chunks grow geometrically.
#define RESTORE_CHUNK0 32u
#ifndef TA_RESTORE_CHUNK_DIV
#define TA_RESTORE_CHUNK_DIV 512u
#endif
#define RESTORE_CHUNK_MAX 4096u

// Step 3, one CTA per replica (reading A6): if the decayed
// load exceeds lambda_max*C, pause the minimal prefix of the actives in S_pause
// order (acting first, shortest first) whose contributions cover Delta C.  Only the
// prefix is materialized: buckets (tau, nb) select it exactly, then a stable CTA
// radix sort orders it by the full key.
__device__ __forceinline__ void pause_pass(const Dev& d, const int r, u32* s_big, u32* s_tmp) {
  extern __shared__ __align__(16) char dsm[];
  SortSmem* sm = reinterpret_cast<SortSmem*>(dsm);
  __shared__ ull s_L;
  if (d.ctr->err != TA_OK) return;              // API batch rejected: the tick does not run
  if (TA_FLAG(d, TA_F_TIMING) && blockIdx.x == 0 && threadIdx.x < 32) d.pst[threadIdx.x] = 0;
  PSTAMP(0, 0);
  if (threadIdx.x == 0) {                       // publish this tick's load (eq. 7) of replica r
    s_L = d.Lacc[r];
    d.Lacc[r] = 0;
  }
  __syncthreads();
  const ull Lr = s_L;
  const ull cap = (ull)d.cap_max[r];
  if (Lr <= cap) {
    if (threadIdx.x == 0) d.L[r] = Lr;
    return;
  }
  const u32 dC = (u32)(Lr - cap);
  if (threadIdx.x == 0) {                        // NEXT-4 guard: excess found by the monitor (A50)
    atomicAdd(&d.stats[ST_OVERSHOOT], (ull)dC);
    atomicMax(&d.stats[ST_OVERSHOOT_MAX], (ull)dC);
  }
  const int N = d.N;
  const u32 NBK = d.nbk, sh = d.nb_shift;
  u64* ka = d.ska + (size_t)r * N;
  u64* kb = d.skb + (size_t)r * N;
  u32* va = d.sva + (size_t)r * N;
  u32* vb = d.svb + (size_t)r * N;
  // the actives on r are exactly the footprint pass's set for r (statuses have not
  // changed since), as a slot list in the free tail of the dynamic shared memory (or
  // global scratch when it does not fit); ordered below by (S_pause key, slot)
  __shared__ u32 s_cnt;
  const u32* al = nullptr;
  const u32 lcap = small_paths(d) ? 8u : 3u * 4096u;
  const int na = (int)cta_bits_to_list(d.act_bits + (size_t)r * d.NW, d.NW,
                                       reinterpret_cast<u32*>(dsm + sizeof(SortSmem)), lcap,
                                       d.act_list + (size_t)r * N, s_tmp, &al);
  if ((u32)na > lcap) dbg_hit(d, DBG_LIST_GLOBAL);
  PSTAMP(0, 1);
  const bool ra = TA_FLAG(d, TA_F_REQUEST_AWARE);   // RequestAware baseline (A46)
  auto bucket = [&](int i) { return ra ? 0u : (u32)(d.phase[i] == TA_PHASE_R) * NBK + (d.nb[i] >> sh); };
  const u32 T = cta_list_threshold(al, na, 2 * NBK, 0, dC, s_big, s_tmp, [](int) { return true; }, bucket,
                                   [&](int i) { return d.contrib[i]; });
  PSTAMP(0, 2);
  u32 n = cta_list_gather(al, na, &s_cnt,
      [&](int i) { return bucket(i) <= T; },
      [&](u32 pos, int i) {
        ka[pos] = ra ? (((u64)(d.phase[i] == TA_PHASE_A) << 63) | (u64)(0xFFFFFFFFu - (u32)i))
                     : pause_key(d.phase[i], d.nb[i], d.acting_since[i]);
        va[pos] = (u32)i;
      });
  PSTAMP(0, 3);
  int res = cta_sort_kv(ka, va, kb, vb, (int)n, s_big, s_tmp, sm, sort_lim(d));
  PSTAMP(0, 4);
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
    const u32 b = restore_bucket(d, d.phase[p], d.nb[p]);   // joins the restore queue
    d.rb[p] = b;
    atomicAdd(&d.rhist[b], 1u);
  }
  PSTAMP(0, 5);
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
__device__ __forceinline__ void restore_pass(const Dev& d, u32* s_big, u32* s_tmp) {
  __shared__ u32 s_stop;
  if (d.ctr->err != TA_OK) return;              // API batch rejected: the tick does not run
  extern __shared__ __align__(16) char dsm[];
  SortSmem* sm = reinterpret_cast<SortSmem*>(dsm);
  const int N = d.N, R = d.R;
  const u32 NBK = d.nbk;
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
  if (TA_FLAG(d, TA_F_TIMING) && threadIdx.x < 32) d.pst[1 * 32 + threadIdx.x] = 0;
  PSTAMP(1, 0);
  if (!d.api_mode) {                   // closed-loop trace arrivals (reading A12):
    const i64 na = d.ctr->next_arrival;  // the lowest UNARRIVED slots, one per release
    const i64 n_arr = trace_arrivals(d);
    const u32 k = (u32)d.ctr->tick;
    for (i64 q = threadIdx.x; q < n_arr; q += CTA) {
      const int p = (int)(na + q);
      d.uid[p] = d.t_uid[p]; d.status[p] = TA_PAUSED; d.phase[p] = TA_PHASE_R;
      d.c[p] = d.t_p0[p]; d.c_kv[p] = 0; d.paused_since[p] = k;
      d.placement[p] = -1; d.home[p] = -1; d.turn[p] = 0; d.gen_done[p] = 0;
      d.satisfied[p] = 0; d.step_count[p] = 0; d.acting_since[p] = 0;
      d.tool_return[p] = INT64_MAX;
      d.pend[p] = d.t_p0[p]; d.busy[p] = 0;      // the prompt waits for its prefill (A48)
      d.kp[p] = d.t_kp[p];                       // its shared prompt (A51)
      const u32 nbv = ceil_div_u32(d.t_p0[p], d.bt);
      d.nb[p] = nbv; d.n_hbm[p] = 0; d.n_host[p] = 0; d.prefix_hbm[p] = 0; d.contrib[p] = nbv;
      const u32 b = restore_bucket(d, TA_PHASE_R, nbv);
      d.rb[p] = b;
      atomicAdd(&d.rhist[b], 1u);
    }
    __syncthreads();
  }
  u32 cnt = 0, over = 0, it = 0;
  u32 stopped = 0;                      // PinnedRouting: replicas whose queue stopped (warp 0)
  // queue buckets: rb[] / rhist[] from the footprint pass, plus this tick's pauses
  // (k_pause) and arrivals (above), so no pass over the slots is needed to size a chunk
  const u32 chunk_max = small_paths(d) ? 64u : RESTORE_CHUNK_MAX;
  // first chunk: about one queued entry per 512 slots (32 up to 16k programs, 78 at 40k),
  // so that large queues rarely need a second pass over the slots
  u32 lo = 0, chunk = small_paths(d) ? 4u : max(RESTORE_CHUNK0, min(512u, (u32)N / TA_RESTORE_CHUNK_DIV));
  while (true) {
    const u32 T = cta_hist_threshold(d.rhist, 2 * NBK, lo, chunk, s_big, s_tmp);
    if (it < 7) PSTAMP(1, 1 + 4 * it);
    // the chunk's entries (slot order) with their S_restore keys, into the free tail of
    // the dynamic shared memory when they fit (sorted there in place), else global
    const u32 scap = small_paths(d) ? 16u : (u32)SORT_SMALL;
    u64* s_gk = reinterpret_cast<u64*>(dsm + sizeof(SortSmem));
    u32* s_gv = reinterpret_cast<u32*>(s_gk + SORT_SMALL);
    u32 n = cta_ordered_gather_w(N, s_tmp,
        [&](int i) { const u32 b = d.rb[i]; return b >= lo && b <= T; },
        [&](u32 pos, int i, u32 total) {
          const u64 key = TA_FLAG(d, TA_F_REQUEST_AWARE) ? (u64)d.paused_since[i]            // FCFS (A46)
                                                         : restore_key(d.phase[i], d.nb[i], d.paused_since[i]);
          if (total <= scap) { s_gk[pos] = key; s_gv[pos] = (u32)i; }
          else { ka[pos] = key; va[pos] = (u32)i; }
        });
    if (it < 7) PSTAMP(1, 2 + 4 * it);
    if (TA_FLAG(d, TA_F_TIMING) && threadIdx.x == 0 && it < 4) d.pst[1 * 32 + 27 + it] = n | (1ull << 62);
    const u32* q;
    if (n <= scap) {
      const int res = cta_sort(s_gk, s_gv, s_gk, s_gv, (int)n, s_big, s_tmp, sm, sort_lim(d));
      (void)res;                          // in place: the result is in (s_gk, s_gv) either way
      q = s_gv;
    } else {
      dbg_hit(d, DBG_LIST_GLOBAL);
      const int res = cta_sort(ka, va, kb, vb, (int)n, s_big, s_tmp, sm, sort_lim(d));
      q = res ? vb : va;
    }
    if (it < 7) PSTAMP(1, 3 + 4 * it);
    // the entries' contribution, home and phase for the sequential loop, gathered by the
    // whole CTA in one round trip (the keys' space is free after the sort)
    const bool pre = n <= scap;
    u32* s_cr = reinterpret_cast<u32*>(s_gk);
    u32* s_hp = s_cr + SORT_SMALL;                // (home + 1) | phase << 8
    if (pre) {
      for (u32 i = threadIdx.x; i < n; i += CTA) {
        const u32 p = q[i];
        s_cr[i] = d.contrib[p];
        s_hp[i] = (u32)(d.home[p] + 1) | ((u32)d.phase[p] << 8);
      }
      __syncthreads();
    }
    if (w0 && pre && R == 1 && !TA_FLAG(d, TA_F_PINNED_ROUTING)) {
      // one replica: the loop below places entries in order while L < cap_min and
      // L + c <= cap_max, skipping the oversized, up to the first that fails -- so 32
      // entries at a time: L before entry i = L + the placed contributions before it
      // (a warp prefix sum), and the first failing lane ends the pass
      bool stop = false;
      const ull c_min = __shfl_sync(FULL_MASK, cmin, 0), c_max = __shfl_sync(FULL_MASK, cmax, 0);
      ull L0 = __shfl_sync(FULL_MASK, Lr, 0);
      const u32 below = (1u << lane) - 1u;
      for (u32 base = 0; base < n; base += 32) {
        const u32 i = base + lane;
        const bool in = i < n;
        const u32 cr = in ? s_cr[i] : 0u;
        const bool skip = in && cr > maxcap;             // can never fit (reading A9)
        const u32 v = (in && !skip) ? cr : 0u;
        const u32 inc = warp_incl_scan(v);               // < 32 x 2^23
        const ull before = L0 + (ull)(inc - v);
        const bool fit = skip || (before < c_min && before + cr <= c_max);
        const u32 fail = __ballot_sync(FULL_MASK, in && !fit);
        const u32 upto = fail ? (1u << (__ffs(fail) - 1)) - 1u : 0xFFFFFFFFu;   // lanes before it
        const u32 placed = __ballot_sync(FULL_MASK, in && !skip) & upto;
        over += __popc(__ballot_sync(FULL_MASK, skip) & upto);
        if ((placed >> lane) & 1u) {
          const u32 pl = q[i], hp = s_hp[i];
          const bool pa = (hp >> 8) == TA_PHASE_A;
          const u32 at = cnt + __popc(placed & below);
          d.status[pl] = pa ? TA_ACTING : TA_REASONING;
          d.placement[pl] = 0;
          d.restore_pid[at] = pl;
          d.restore_dst[at] = 0u | ((hp & 0xFFu) << 8) | ((u32)pa << 24);
        }
        cnt += __popc(placed);
        const int f = fail ? __ffs(fail) - 1 : 31;      // placed before the first failure: all of them
        L0 += (ull)__shfl_sync(FULL_MASK, fail ? inc - v : inc, f);
        if (fail) { stop = true; break; }
      }
      if (lane == 0) { Lr = L0; s_stop = stop || T >= 2 * NBK - 1; }
    } else if (w0 && pre && !TA_FLAG(d, TA_F_PINNED_ROUTING)) {
      // the global queue (reading A10) with the entries in shared memory: every lane reads
      // entry i (broadcast, independent of the loads), and one min-reduction over the
      // replicas' packed keys both tells whether any replica fits and picks the target
      bool stop = false;
      const bool mine = lane < (u32)R;
#pragma unroll 2
      for (u32 i = 0; i < n; ++i) {
        const u32 cr = s_cr[i], hp = s_hp[i];
        if (cr > maxcap) { ++over; continue; }          // can never fit (reading A9)
        const int hm = (int)(hp & 0xFFu) - 1;
        const u32 key = (mine && Lr < cmin && Lr + cr <= cmax)
                            ? (((u32)Lr << 6) | ((u32)((int)lane != hm) << 5) | lane) : 0xFFFFFFFFu;
        const u32 kmin = __reduce_min_sync(FULL_MASK, key);
        if (kmin == 0xFFFFFFFFu) { stop = true; break; }
        const u32 t = kmin & 31u;
        if (lane == t) Lr += cr;
        if (lane == 0) {
          const u32 pl = q[i];
          const bool pa = (hp >> 8) == TA_PHASE_A;
          d.status[pl] = pa ? TA_ACTING : TA_REASONING;
          d.placement[pl] = (i8)t;
          d.restore_pid[cnt] = pl;
          d.restore_dst[cnt] = t | ((hp & 0xFFu) << 8) | ((u32)pa << 24);   // dst | (home + 1) << 8 | A << 24
        }
        ++cnt;
      }
      if (lane == 0) s_stop = stop || T >= 2 * NBK - 1;
    } else if (w0) {
      bool stop = false;
      const bool pinned = TA_FLAG(d, TA_F_PINNED_ROUTING);
      const u32 all_r = R >= 32 ? 0xFFFFFFFFu : ((1u << R) - 1);
      for (u32 base = 0; base < n && !stop; base += 32) {
        u32 i = base + lane;
        u32 pl = i < n ? q[i] : 0;
        const u32 hp = (i < n && pre) ? s_hp[i] : 0u;
        u32 crl = i < n ? (pre ? s_cr[i] : d.contrib[pl]) : 0;
        int hml = i < n ? (pre ? (int)(hp & 0xFF) - 1 : d.home[pl]) : -1;
        u32 phl = i < n ? (pre ? hp >> 8 : d.phase[pl]) : 0;
        u32 mcount = min(32u, n - base);
        for (u32 jj = 0; jj < mcount; ++jj) {
          u32 cr = __shfl_sync(FULL_MASK, crl, jj);
          u32 t;
          if (pinned) {                           // PinnedRouting baseline (reading A45)
            t = __shfl_sync(FULL_MASK, pl, jj) % (u32)R;
            if ((stopped >> t) & 1u) continue;    // that replica's queue has stopped
            if (cr > __shfl_sync(FULL_MASK, cmax, t)) { ++over; continue; }
            const bool fits = lane == t && Lr < cmin && Lr + cr <= cmax;
            if (__ballot_sync(FULL_MASK, fits) == 0) {
              stopped |= 1u << t;
              if (stopped == all_r) { stop = true; break; }
              continue;
            }
          } else {
            if (cr > maxcap) { ++over; continue; }       // can never fit (reading A9)
            bool fits = lane < (u32)R && Lr < cmin && Lr + cr <= cmax;
            if (__ballot_sync(FULL_MASK, fits) == 0) { stop = true; break; }
            int hm = __shfl_sync(FULL_MASK, hml, jj);
            u32 key = fits ? (((u32)Lr << 6) | ((u32)((int)lane != hm) << 5) | lane) : 0xFFFFFFFFu;
            t = __reduce_min_sync(FULL_MASK, key) & 31;
          }
          if (lane == t) Lr += cr;
          if (lane == jj) {                       // the lane that holds the entry writes it
            d.status[pl] = phl == TA_PHASE_A ? TA_ACTING : TA_REASONING;
            d.placement[pl] = (i8)t;
            d.restore_pid[cnt] = pl;
            // dst | (home before + 1) << 8 | phase A << 24
            d.restore_dst[cnt] = t | ((u32)(hml + 1) << 8) | ((u32)(phl == TA_PHASE_A) << 24);
          }
          ++cnt;
        }
      }
      if (lane == 0) s_stop = stop || T >= 2 * NBK - 1;
    }
    __syncthreads();
    if (it < 7) PSTAMP(1, 4 + 4 * it);
    ++it;
    if (s_stop) break;
    lo = T + 1;
    chunk = min(chunk * 8, chunk_max);
    dbg_hit(d, DBG_RESTORE_CHUNKS);
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
  PSTAMP(1, 31);
}
