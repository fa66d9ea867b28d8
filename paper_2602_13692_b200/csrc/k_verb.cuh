// k_verb.cuh — explicit single-program verbs (ta_pause / ta_resume / ta_migrate).
// They act on the state left by the last tick, at its time T (SURVEY.md §8(c) "API-mode
// events and explicit verbs"); resume/migrate reuse k_footprint, k_plan (F = {pid},
// all-or-nothing), the copy kernels, k_finalize and k_assemble in verb mode.
#pragma once
#include "common.cuh"

// Clear every per-call list so the shared copy / assembly kernels see only this verb.
__global__ void k_verb_reset(Dev d) {
  int t = threadIdx.x;
  if (t == 0) {
    d.ctr->restore_cnt = 0; d.ctr->verb_ok = 1;
    if (d.ctr->err != TA_E_PEER) d.ctr->err = TA_OK;   // a peer failure stays until read
    d.ctr->t_d2h = d.ctr->t_h2d = d.ctr->t_p2p = d.ctr->t_d2d = d.ctr->t_fetch = d.ctr->t_cross = 0;
  }
  if (t < d.R) {
    d.pause_cnt[t] = 0; d.f_cnt[t] = 0; d.s_cnt[t] = 0; d.ev_cnt[t] = 0;
    d.evd_cnt[t] = 0; d.fed_cnt[t] = 0; d.fld_cnt[t] = 0; d.dfh_cnt[t] = 0; d.dfs_cnt[t] = 0;
    d.cpd_cnt[t] = 0;
  }
  for (u32 b = threadIdx.x; b < 2 * d.nbk; b += blockDim.x) d.rhist[b] = 0;
}

// ta_pause: LAZY only unbinds; OFFLOAD evicts every HBM block of the
// program tail-first into the lowest free host slots of its home (drop when full);
// DROP frees them.  One CTA.
__global__ void __launch_bounds__(CTA, 1) k_verb_pause(Dev d, u32 pid, u32 mode) {
  __shared__ u32 s_big[8192 + 1];
  __shared__ u32 s_tmp[NWARP + 1];
  __shared__ int s_err, s_h;
  __shared__ u32 s_nh, s_sb;
  if (threadIdx.x == 0) {
    int err = TA_OK;
    u8 st = pid < (u32)d.N ? d.status[pid] : TA_UNARRIVED;
    if (pid >= (u32)d.N || st == TA_UNARRIVED) err = TA_E_UNKNOWN_PROGRAM;
    else if (st != TA_REASONING && st != TA_ACTING) err = TA_E_ILLEGAL_TRANSITION;
    s_err = err;
    d.ctr->err = err;
    if (err == TA_OK) {
      const int r = d.placement[pid];
      const u32 nbv = ceil_div_u32(d.c[pid], d.bt);
      const u32 cb = contrib_of(d, nbv, d.phase[pid], d.acting_since[pid], d.ctr->T);
      d.L[r] -= cb;
      d.status[pid] = TA_PAUSED;
      d.placement[pid] = -1;
      d.paused_since[pid] = (u32)d.ctr->tick;
      d.satisfied[pid] = 0;
      d.pause_list[(size_t)r * d.N] = pid;
      d.pause_cnt[r] = 1;
      d.stats[ST_PAUSES] += 1;
      s_h = d.home[pid];
      u32 nh = 0;                          // HBM prefix length (I10)
      const u32* row = d.loc + (size_t)pid * d.MAXBP;
      while (nh < nbv && is_hbm(row[nh])) ++nh;
      const u32 sbp = sb_of(d, d.kp[pid]);
      s_sb = sbp;
      s_nh = (mode == TA_PAUSE_LAZY || s_h < 0 || nh <= sbp) ? 0 : nh - sbp;   // private blocks
    }
  }
  __syncthreads();
  if (s_err != TA_OK || s_nh == 0) return;
  const int h = s_h;
  const u32 X = s_nh;
  u32* row = d.loc + (size_t)pid * d.MAXBP;
  if (threadIdx.x == 0) d.dirty[pid] = 1;
  const u32* sf = d.host_free + (size_t)h * d.NHW;
  u32 hfree = 0;
  if (mode == TA_PAUSE_OFFLOAD) {
    cta_bitmap_prefix(sf, d.NHW, s_big, s_tmp);
    hfree = s_big[d.NHW];
  }
  EvDesc* evd = d.evd + (size_t)h * d.NB;
  u32* scr = d.evx + (size_t)h * d.NB;
  for (u32 e = threadIdx.x; e < X; e += CTA) {
    u32 j = s_sb + X - 1 - e;             // tail first, down to the shared prompt
    u32 idx = row[j];
    scr[e] = idx;
    if (e < hfree) {
      if (evp_owner(d, h)) evp_of(d, h)[idx] = 2u * d.nL;
      u32 slot = bitmap_select(sf, s_big, d.NHW, e);
      row[j] = LOC_HOST | slot;
      d.owner_host[(size_t)h * d.NH + slot] = pid * (u32)d.MAXB + j;
      evd[e].src = idx;
      evd[e].dst = slot;
    } else {
      row[j] = LOC_NONE;
    }
  }
  __syncthreads();
  u32* hf = d.hbm_free + (size_t)h * d.NBW;
  u32* shf = d.host_free + (size_t)h * d.NHW;
  for (u32 e = threadIdx.x; e < X; e += CTA) {
    u32 idx = scr[e];
    atomicOr(&hf[idx >> 5], 1u << (idx & 31));
    if (e < hfree) {
      u32 slot = evd[e].dst;
      atomicAnd(&shf[slot >> 5], ~(1u << (slot & 31)));
    }
  }
  if (threadIdx.x == 0) {
    u32 toh = min(X, hfree);
    ta_decision rec = {};
    rec.kind = TA_D_EVICT; rec.pid = pid; rec.src = h; rec.dst = -1; rec.blocks = X;
    rec.to_host = toh; rec.dropped = X - toh;
    d.dec_ev[(size_t)h * d.N] = rec;
    d.ev_cnt[h] = 1;
    d.evd_cnt[h] = toh;
    d.stats[ST_EVICT_BLOCKS] += X;
    d.stats[ST_EVICT_TO_HOST] += toh;
    d.ctr->t_d2h += toh;
    d.stats[ST_EVICT_DROPPED] += X - toh;
  }
}

// ta_resume / ta_migrate admission (one thread): legality, capacity,
// target choice (step-4 argmin when replica < 0), tentative activation.  A phase-R
// program then runs k_plan in verb mode (all-or-nothing); k_verb_commit finishes.
__global__ void k_verb_admit(Dev d, u32 pid, int replica, int migrate) {
  if (threadIdx.x != 0) return;
  int err = TA_OK;
  u8 st = pid < (u32)d.N ? d.status[pid] : TA_UNARRIVED;
  if (pid >= (u32)d.N || st == TA_UNARRIVED) err = TA_E_UNKNOWN_PROGRAM;
  else if (!migrate && st != TA_PAUSED) err = TA_E_ILLEGAL_TRANSITION;
  else if (migrate && st != TA_REASONING && st != TA_ACTING) err = TA_E_ILLEGAL_TRANSITION;
  else if (replica >= d.R || replica < -1 || (migrate && (replica < 0 || replica == d.placement[pid])))
    err = TA_E_INVAL;
  int t = replica;
  const ull cr = err == TA_OK ? d.contrib[pid] : 0;
  if (err == TA_OK) {
    if (t < 0) {                           // least loaded candidate (step 4 rule)
      u64 best = ~0ull;
      for (int r = 0; r < d.R; ++r) {
        ull L = d.L[r];
        if (L < (ull)d.cap_min[r] && L + cr <= (ull)d.cap_max[r]) {
          u64 key = (L << 6) | ((u64)(r != d.home[pid]) << 5) | (u64)r;
          if (key < best) best = key;
        }
      }
      if (best == ~0ull) err = TA_E_CAPACITY; else t = (int)(best & 31);
    } else if (!((d.healthy >> t) & 1u) || d.L[t] + cr > (ull)d.cap_max[t]) {
      err = TA_E_CAPACITY;                 // an unhealthy replica has no capacity (reading A39)
    }
  }
  d.ctr->err = err;
  if (err != TA_OK) return;
  const int src = migrate ? d.placement[pid] : d.home[pid];
  d.ctr->verb_pid = pid;
  d.ctr->verb_replica = t;
  d.ctr->n_arr = (u32)(d.placement[pid] + 1) | ((u32)st << 8);   // saved for a revert
  d.status[pid] = d.phase[pid] == TA_PHASE_R ? TA_REASONING : TA_ACTING;
  d.placement[pid] = (i8)t;
  d.restore_pid[0] = pid;
  d.restore_dst[0] = (u32)t | ((u32)(src + 1) << 8) | ((u32)migrate << 16);
  d.ctr->restore_cnt = 1;
  d.ctr->verb_ok = 1;
}

// After k_plan: revert when the physical fetch could not be satisfied, else book the load.
__global__ void k_verb_commit(Dev d, int migrate) {
  if (threadIdx.x != 0 || d.ctr->err != TA_OK) return;
  const u32 pid = d.ctr->verb_pid;
  const int t = d.ctr->verb_replica;
  if (!d.ctr->verb_ok) {
    u32 saved = d.ctr->n_arr;
    d.placement[pid] = (i8)((int)(saved & 0xFF) - 1);
    d.status[pid] = (u8)(saved >> 8);
    d.ctr->restore_cnt = 0;
    d.ctr->err = TA_E_CAPACITY;
    return;
  }
  const ull cr = d.contrib[pid];
  const int old = (int)(d.ctr->n_arr & 0xFF) - 1;
  if (old >= 0) d.L[old] -= cr;
  d.L[t] += cr;
  if (!migrate) d.stats[ST_RESTORES] += 1;
}

// ta_set_health(r, unhealthy) (NEXT-4; readings A37-A39),
// one CTA: the replica's KV is lost.  Programs active on r are force-paused (PAUSE
// records, slot order); programs homed on r drop every block (EVICT records with all
// blocks dropped, slot order, only those that held blocks); r's HBM and host-tier
// bitmaps become all free; its load is 0.  The caller already set its watermarks to 0.
__global__ void __launch_bounds__(CTA, 1) k_verb_health(const __grid_constant__ Dev d, int r) {
  __shared__ u32 s_tmp[NWARP + 1];
  const int N = d.N;
  const u32 k = (u32)d.ctr->tick;
  u32* pl = d.pause_list + (size_t)r * N;
  const u32 np = cta_ordered_gather(N, s_tmp,
      [&](int i) { const u8 s = d.status[i]; return (s == TA_REASONING || s == TA_ACTING) && d.placement[i] == r; },
      [&](u32 pos, int i) { pl[pos] = (u32)i; });
  for (u32 q = threadIdx.x; q < np; q += CTA) {
    const u32 p = pl[q];
    d.status[p] = TA_PAUSED;
    d.placement[p] = -1;
    d.paused_since[p] = k;
    d.satisfied[p] = 0;
  }
  u32* hl = d.e_pid + (size_t)r * N;                  // programs homed on r, slot order
  const u32 nh = cta_ordered_gather(N, s_tmp, [&](int i) { return d.home[i] == r; },
                                    [&](u32 pos, int i) { hl[pos] = (u32)i; });
  u32* lost = d.e_cum + (size_t)r * N;
  const u32 warp = threadIdx.x >> 5, lane = lane_id();
  for (u32 q = warp; q < nh; q += NWARP) {            // one warp per program: drop its row
    const u32 p = hl[q];
    u32* row = d.loc + (size_t)p * d.MAXBP;
    const u32 nbv = ceil_div_u32(d.c[p], d.bt), sbp = sb_of(d, d.kp[p]);
    u32 cnt = 0;
    for (u32 j = lane; j < nbv; j += 32) {          // lost: private blocks (j >= its prompt)
      if (row[j] != LOC_NONE) { cnt += j >= sbp; row[j] = LOC_NONE; }
    }
    cnt = __reduce_add_sync(FULL_MASK, cnt);
    if (lane == 0) { lost[q] = cnt; d.home[p] = -1; d.dirty[p] = 1; }
  }
  __syncthreads();
  ta_decision* ev = d.dec_ev + (size_t)r * N;
  __shared__ ull s_lost;
  if (threadIdx.x == 0) s_lost = 0;
  __syncthreads();
  const u32 ne = cta_ordered_gather((int)nh, s_tmp, [&](int q) { return lost[q] > 0; },
      [&](u32 pos, int q) {
        ta_decision rec = {};
        rec.kind = TA_D_EVICT; rec.pid = hl[q]; rec.src = r; rec.dst = -1;
        rec.blocks = lost[q]; rec.dropped = lost[q];
        ev[pos] = rec;
        atomicAdd(&s_lost, (ull)lost[q]);
      });
  // every block of r belonged to a program homed on r or to a prompt they used: the pools
  // are empty now, and r holds no prompt (A51)
  for (int w = threadIdx.x; w < d.NBW; w += CTA) {
    const i64 lo = (i64)w * 32, n = (i64)d.NB - lo;
    d.hbm_free[(size_t)r * d.NBW + w] = n <= 0 ? 0u : (n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1));
    d.pfix[(size_t)r * d.NBW + w] = 0u;
  }
  for (int k = threadIdx.x; k < d.K; k += CTA) d.pref[(size_t)r * d.K + k] = 0u;
  for (int w = threadIdx.x; w < d.NHW; w += CTA) {
    const i64 lo = (i64)w * 32, n = d.NH - lo;
    d.host_free[(size_t)r * d.NHW + w] = n <= 0 ? 0u : (n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1));
  }
  if (threadIdx.x == 0) {
    d.pause_cnt[r] = np;
    d.ev_cnt[r] = ne;
    d.L[r] = 0;
    d.stats[ST_PAUSES] += np;
    d.stats[ST_EVICT_BLOCKS] += s_lost;
    d.stats[ST_EVICT_DROPPED] += s_lost;
  }
}
