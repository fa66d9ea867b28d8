// k_finalize.cuh — step 7: deferred frees, materialized-program updates, two-finger
// compaction plan, statistics and canonical decision assembly.
#pragma once
#include "common.cuh"

// Deferred frees (P2P sources and fetched host slots become free only after the
// movement, reading A16) and the per-program results of step 5.7.
template <int verb>
__device__ __forceinline__ void finalize_part(const Dev& d, int first_cta) {
  const int t = ((int)blockIdx.x - first_cta) * blockDim.x + threadIdx.x;
  const int stride = ((int)gridDim.x - first_cta) * blockDim.x;
  for (int r = 0; r < d.R; ++r) {
    const u32 nh = d.dfh_cnt[r], ns = d.dfs_cnt[r];
    const u32* fh = d.dfh + (size_t)r * d.NB;
    const u32* fs = d.dfs + (size_t)r * d.NB;
    for (u32 e = t; e < nh; e += stride) {
      u32 x = fh[e], h = x >> 27, idx = x & ((1u << 27) - 1);
      atomicOr(&d.hbm_free[(size_t)h * d.NBW + (idx >> 5)], 1u << (idx & 31));
    }
    for (u32 e = t; e < ns; e += stride) {
      u32 x = fs[e], h = x >> 27, s = x & ((1u << 27) - 1);
      atomicOr(&d.host_free[(size_t)h * d.NHW + (s >> 5)], 1u << (s & 31));
    }
  }
  ull cach = 0;                          // NEXT-1: idle resident KV (token count)
  u32 cmin = 0xFFFFFFFFu;                // smallest paused footprint (blocks)
  for (int p = t; p < d.N; p += stride) {
    // every per-program value in one round trip (L2-resident: written this tick)
    const u8 s = d.sat_new[p], st = d.status[p];
    const int h = d.home[p];
    const u32 cp = d.c[p], nbp = d.nb[p], nhp = d.n_hbm[p];
    if (s) {
      const int r = s - 1;
      const u8 k = d.kp[p];
      if (h != r && k != KP_NONE) {      // NEXT-3 (A51): its prompt entries now point at r's copy;
        const u32* blk = d.pblk + ((size_t)r * d.K + k) * d.SBM;   // h's copy loses a user, and
        for (u32 j = 0; j < d.sbk[k]; ++j) d.loc[(size_t)p * d.MAXBP + j] = blk[j];   // the last
        if (h >= 0 && atomicSub(&d.pref[(size_t)h * d.K + k], 1u) == 1u)  // one frees its blocks
          prompt_free(d, h, k, 0, 1);
      }
      d.satisfied[p] = 1;
      d.home[p] = (i8)(s - 1);
      d.c_kv[p] = cp;
      d.n_hbm[p] = nbp;
      d.sat_new[p] = 0;
      d.dirty[p] = 1;                    // its row was written (fetches, prompt entries)
    } else if (!verb) {
      d.satisfied[p] = 0;
      if (st == TA_PAUSED || st == TA_ACTING) {
        if (h >= 0) cach += min((ull)nhp * (ull)d.bt, (ull)cp);
        if (st == TA_PAUSED) cmin = min(cmin, nbp);
      }
    }
  }
  if (!verb) {
    cach = warp_sum_ull(cach);
    cmin = __reduce_min_sync(FULL_MASK, cmin);
    if (lane_id() == 0) {
      if (cach) atomicAdd(&d.stats[ST_COST_CACHING], cach * (ull)d.dt);
      if (cmin != 0xFFFFFFFFu) atomicMin(&d.ctr->cmin, cmin);
    }
  }
}

// Two-finger compaction (reading A20), one CTA per replica, over the movable blocks
// (used, not a shared-prompt block: A51): the m-th lowest free block receives the m-th
// highest movable block while the former lies below the latter -- all moves of the
// sequential two-finger loop, computed at once by rank/select (the fingers only pass
// blocks they have not touched, so the pairs are those of the initial sets).
__device__ __forceinline__ void compact_plan_pass(const Dev& d, const int r, u32* s_big, u32* s_tmp) {
  __shared__ u32 s_K;
  u32* fw = d.hbm_free + (size_t)r * d.NBW;
  const u32* fx = d.pfix + (size_t)r * d.NBW;
  const int nw = d.NBW;
  u32* s_free = s_big;                  // [nw + 1]
  u32* s_used = s_big + nw + 1;         // [nw + 1]
  u32* s_mw = s_big + 2 * (nw + 1);     // [nw] movable words
  auto valid_of = [&](int w) -> u32 {   // bits of word w that are blocks
    const i64 n = (i64)d.NB - (i64)w * 32;
    return n <= 0 ? 0u : (n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1));
  };
  for (int w = threadIdx.x; w < nw; w += CTA) s_mw[w] = ~fw[w] & ~fx[w] & valid_of(w);
  if (threadIdx.x == 0) s_K = 0xFFFFFFFFu;
  __syncthreads();
  cta_bitmap_prefix(fw, nw, s_free, s_tmp);
  cta_bitmap_prefix(s_mw, nw, s_used, s_tmp);
  const u32 F = s_free[nw], U = s_used[nw], lim = min(F, U);
  for (u32 m = threadIdx.x; m < lim; m += CTA)          // first m whose pair does not cross
    if (bitmap_select(fw, s_free, nw, m) > bitmap_select(s_mw, s_used, nw, U - 1 - m)) atomicMin(&s_K, m);
  __syncthreads();
  const u32 K = min(s_K, lim);
  CpDesc* cp = d.cpd + (size_t)r * (d.NB / 2 + 1);
  for (u32 m = threadIdx.x; m < K; m += CTA) {
    const u32 dst = bitmap_select(fw, s_free, nw, m);
    const u32 src = bitmap_select(s_mw, s_used, nw, U - 1 - m);   // m-th highest movable block
    const u32 o = d.owner_hbm[(size_t)r * d.NB + src];
    const u32 p = o / (u32)d.MAXB, j = o % (u32)d.MAXB;
    d.loc[(size_t)p * d.MAXBP + j] = dst;
    d.dirty[p] = 1;
    d.owner_hbm[(size_t)r * d.NB + dst] = o;
    cp[m] = CpDesc{src, dst};
  }
  __syncthreads();
  for (u32 m = threadIdx.x; m < K; m += CTA) {
    CpDesc c = cp[m];
    atomicOr(&fw[c.src >> 5], 1u << (c.src & 31));
    atomicAnd(&fw[c.dst >> 5], ~(1u << (c.dst & 31)));
  }
  if (threadIdx.x == 0) {
    d.cpd_cnt[r] = K;
    atomicAdd(&d.stats[ST_COMPACT], (ull)K);
    atomicAdd(&d.ctr->t_d2d, K);
  }
}

// Canonical decision list (PAUSE by replica, RESTORE in queue order, EVICT by
// replica, FETCH/STALL by replica in slot order, COMPACT by replica), written to
// the host-mapped buffer; tick bookkeeping and occupancy statistics.  In two parts:
// the records of steps 3-5 (their inputs are final when k_close starts), and after the
// frees and the compaction plan, the COMPACT records, statistics and clears.
__device__ __forceinline__ u32 assemble_records(const Dev& d, u32* s_tmp) {
  const int N = d.N, R = d.R;
  const u32 cap = d.dec_cap;
  u32 pos = 0;                           // uniform across the CTA
  auto put = [&](u32 at, const ta_decision& rec) { if (at < cap) d.dec_out[at] = rec; };
  for (int r = 0; r < R; ++r) {          // PAUSE
    u32 n = d.pause_cnt[r];
    for (u32 i = threadIdx.x; i < n; i += CTA) {
      ta_decision rec = {};
      rec.kind = TA_D_PAUSE; rec.pid = d.pause_list[(size_t)r * N + i]; rec.src = r; rec.dst = -1;
      put(pos + i, rec);
    }
    pos += n;
  }
  {                                      // RESTORE / MIGRATE
    u32 n = d.ctr->restore_cnt;
    for (u32 i = threadIdx.x; i < n; i += CTA) {
      ta_decision rec = {};
      u32 x = d.restore_dst[i];
      rec.kind = ((x >> 16) & 1u) ? TA_D_MIGRATE : TA_D_RESTORE;
      rec.pid = d.restore_pid[i];
      rec.src = (int)((x >> 8) & 0xFF) - 1;
      rec.dst = (int)(x & 0xFF);
      put(pos + i, rec);
    }
    pos += n;
  }
  for (int r = 0; r < R; ++r) {          // EVICT
    u32 n = d.ev_cnt[r];
    for (u32 i = threadIdx.x; i < n; i += CTA) put(pos + i, d.dec_ev[(size_t)r * N + i]);
    pos += n;
  }
  PSTAMP(3, 10);
  // FETCH / STALL (kind 0 = no decision): every replica's F records in one ordered pass
  // over their concatenation (replica order, then F order), one CTA scan in all
  __shared__ u32 s_fo[TA_MAX_REPLICAS + 1];
  if (threadIdx.x == 0) {
    u32 o = 0;
    for (int r = 0; r < R; ++r) { s_fo[r] = o; o += d.f_cnt[r]; }
    s_fo[R] = o;
  }
  __syncthreads();
  auto rec_at = [&](int x) -> const ta_decision& {
    int r = 0;
    while ((u32)x >= s_fo[r + 1]) ++r;
    return d.dec_fs[(size_t)r * N + (x - (int)s_fo[r])];
  };
  u32 n = cta_ordered_gather((int)s_fo[R], s_tmp,
      [&](int x) { return rec_at(x).kind != 0; },
      [&](u32 at, int x) { put(pos + at, rec_at(x)); });
  pos += n;
  return pos;
}

template <int verb>
__device__ __forceinline__ void assemble_close(const Dev& d, u32 pos) {
  __shared__ ull s_red[NWARP];
  const int R = d.R;
  const u32 cap = d.dec_cap;
  auto put = [&](u32 at, const ta_decision& rec) { if (at < cap) d.dec_out[at] = rec; };
  for (int r = 0; r < R; ++r) {          // COMPACT
    u32 n = d.cpd_cnt[r];
    if (n) {
      if (threadIdx.x == 0) {
        ta_decision rec = {};
        rec.kind = TA_D_COMPACT; rec.pid = 0xFFFFFFFFu; rec.src = r; rec.dst = r; rec.blocks = n;
        put(pos, rec);
      }
      pos += 1;
    }
  }
  PSTAMP(3, 6);
  // occupancy / imbalance (SPEC.md:151-157 at block granularity): every
  // replica's free words counted at once (NWARP / R warps per replica, one pass)
  __shared__ u32 s_free[TA_MAX_REPLICAS];
  if (threadIdx.x < R) s_free[threadIdx.x] = 0;
  __syncthreads();
  {
    const int wpr = R >= NWARP ? 1 : NWARP / R, w = threadIdx.x >> 5, lane = (int)lane_id();
    for (int rr = w / wpr; rr < R && w < wpr * R; rr += NWARP / wpr) {   // R > NWARP: warps loop
      const u32* hf = d.hbm_free + (size_t)rr * d.NBW;
      u32 fr = 0;
#pragma unroll 4
      for (int x = (w % wpr) * 32 + lane; x < d.NBW; x += wpr * 32) fr += __popc(hf[x]);
      fr = __reduce_add_sync(FULL_MASK, fr);
      if (lane == 0) atomicAdd(&s_free[rr], fr);
    }
  }
  __syncthreads();
  // per replica on warp 0 (lane r; R <= 32): every value loaded in one round trip, the
  // statistics added with fire-and-forget atomics (no read-modify-write chain on thread 0)
  ull umax = 0, umin = ~0ull;
  if (threadIdx.x < 32) {
    const int r = (int)threadIdx.x;
    const u32 cminq = d.ctr->cmin;
    const bool on = r < R;
    const ull used = on ? (ull)d.NB - s_free[r] : 0ull;
    const ull cap = on ? (ull)d.cap_max[r] : 0ull, Lr = on ? d.L[r] : 0ull;
    ull cost = 0, viol = 0;
    if (!verb && cminq != 0xFFFFFFFFu && on) {     // programs wait in the queue
      cost = (cap > used ? cap - used : 0) * (ull)d.bt * (ull)d.dt;
      const ull idle = cap > Lr ? cap - Lr : 0;    // C_unused < c_min
      viol = idle >= cminq ? 1ull : 0ull;
    }
    cost = warp_sum_ull(cost);
    viol = warp_sum_ull(viol);
    ull mx = on ? used : 0ull, mn = on ? used : ~0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const ull a = __shfl_xor_sync(FULL_MASK, mx, o), b = __shfl_xor_sync(FULL_MASK, mn, o);
      mx = a > mx ? a : mx;
      mn = b < mn ? b : mn;
    }
    umax = mx; umin = mn;
    if (threadIdx.x == 0 && !verb && cminq != 0xFFFFFFFFu) {
      atomicAdd(&d.stats[ST_COST_UNUSED], cost);
      atomicAdd(&d.stats[ST_UNUSED_CHECKS], (ull)R);
      if (viol) atomicAdd(&d.stats[ST_UNUSED_VIOL], viol);
    }
  }
  PSTAMP(3, 7);
  if (threadIdx.x < TA_MAX_REPLICAS) {   // per-replica link telemetry (host-mapped), one lane each
    const int r = threadIdx.x;
    d.tick_info->d2h_of[r] = r < R ? d.t_rep[r] : 0;
    d.tick_info->h2d_of[r] = r < R ? d.t_rep[R + r] : 0;
    d.tick_info->p2p_to[r] = r < R ? d.t_rep[2 * R + r] : 0;
  }
  if (threadIdx.x == 0) {
    // every counter read first (one round trip), then stores and fire-and-forget atomics
    Ctr* c = d.ctr;
    const i64 tick = c->tick, nxt = c->next_arrival;
    const u32 t_d2h = c->t_d2h, t_h2d = c->t_h2d, t_p2p = c->t_p2p, t_d2d = c->t_d2d, t_fetch = c->t_fetch;
    const u32 stops = c->stops, narr = c->n_arr;
    *d.dec_out_cnt = pos;
    ta_tick_info* ti = d.tick_info;
    ti->tick = tick;
    ti->decisions = pos;
    ti->d2h_blocks = t_d2h;
    ti->h2d_blocks = t_h2d;
    ti->p2p_blocks = t_p2p;
    ti->d2d_blocks = t_d2d;
    ti->fetch_blocks = t_fetch;
    c->n_dec = pos;
    if (!verb) {
      const ull imb = umax - umin;
      d.stats[ST_IMB_LAST] = imb;
      atomicMax(&d.stats[ST_IMB_MAX], imb);
      i64 n_arr;                                      // trace_arrivals() on the values read above
      if (d.api_mode) {
        n_arr = (i64)narr;
      } else {
        const i64 want = (tick == 0 ? (i64)d.n_initial : 0) + (i64)stops, room = (i64)d.n_slots - nxt;
        n_arr = want < room ? want : room;
        c->next_arrival = nxt + n_arr;
      }
      atomicAdd(&d.stats[ST_ARRIVALS], (ull)n_arr);
      if (stops) atomicAdd(&d.stats[ST_STOPS], (ull)stops);
      atomicAdd(&d.stats[ST_TICKS], 1ull);
      c->tick = tick + 1;
    }
  }
  // clear the per-tick lists and counters for the next tick / call
  __syncthreads();
  PSTAMP(3, 8);
  if (threadIdx.x == 0) {
    d.ctr->cmin = 0xFFFFFFFFu;
    d.ctr->stops = 0;
    d.ctr->restore_cnt = 0;
    d.ctr->n_arr = 0;
    d.ctr->t_d2h = d.ctr->t_h2d = d.ctr->t_p2p = d.ctr->t_d2d = d.ctr->t_fetch = d.ctr->t_cross = 0;
  }
  for (int t = threadIdx.x; t < R; t += CTA) {
    d.pause_cnt[t] = 0; d.f_cnt[t] = 0; d.s_cnt[t] = 0; d.ev_cnt[t] = 0;
    d.evd_cnt[t] = 0; d.fed_cnt[t] = 0; d.fld_cnt[t] = 0; d.dfh_cnt[t] = 0; d.dfs_cnt[t] = 0;
    // cpd_cnt is read by the compaction copies after this kernel
  }
  for (u32 b = threadIdx.x; b < 2 * d.nbk; b += CTA) d.rhist[b] = 0;
  for (int t = threadIdx.x; t < 3 * R; t += CTA) d.t_rep[t] = 0;
}

// Step 7 in one cooperative launch: deferred frees and per-program results over all
// CTAs, grid barrier, the two-finger compaction plan (CTA r, on compaction ticks),
// grid barrier, the canonical decision list and statistics on CTA 0.  The
// compaction copies (k_copy_compact) run after this kernel.
template <int verb>   // 0: tick, 1: verbs (a kernel of its own)
__global__ void __launch_bounds__(CTA, 1) k_close(const __grid_constant__ Dev d) {
  const ull t_in = gtimer();   // the CTA's first instruction (kernel span, timing mode)
  __shared__ u32 s_big[8192 + 1];
  __shared__ u32 s_tmp[NWARP + 1];
  if (!verb && d.ctr->err != TA_OK) return;           // API batch rejected: the tick does not run
  if (TA_FLAG(d, TA_F_TIMING) && blockIdx.x == 0 && threadIdx.x < 16) d.pst[3 * 32 + threadIdx.x] = 0;
  kspan_begin(d, KS_CLOSE, t_in);
  jitter(d, 4u);
  PSTAMP(3, 0);
  // compaction tick: read by every CTA before the first grid barrier (CTA 0 advances the
  // tick counter only after it), so all CTAs take the same barriers below
  const bool ctick = !verb && d.compact_every > 0 && (d.ctr->tick % d.compact_every) == 0;
  // CTA 0 assembles the records of steps 3-5 while the other CTAs finalize (one CTA: both)
  u32 pos = 0;
  if (blockIdx.x == 0) pos = assemble_records(d, s_tmp);
  PSTAMP(3, 5);
  if (gridDim.x == 1 || blockIdx.x > 0) finalize_part<verb>(d, gridDim.x == 1 ? 0 : 1);
  PSTAMP(3, 1);
  grid_sync(d, 1);
  PSTAMP(3, 2);
  if (ctick) {                                        // CTA r plans replica r's moves,
    if (blockIdx.x < (unsigned)d.R) compact_plan_pass(d, blockIdx.x, s_big, s_tmp);
    PSTAMP(3, 3);
    grid_sync(d, 1);                                  // plans -> decisions
  } else {                                            // no moves: CTA 0, which reads the
    if (blockIdx.x == 0)                              // counts, clears them itself (a clear
      for (int t = threadIdx.x; t < d.R; t += CTA) d.cpd_cnt[t] = 0;   // by CTA r raced
    __syncthreads();                                  // CTA 0's read: a stale COMPACT record)
  }
  PSTAMP(3, 4);
  if (blockIdx.x == 0) assemble_close<verb>(d, pos);
  PSTAMP(3, 9);
  kspan_end(d, KS_CLOSE);
}
