// k_plan.cuh — step 5 (materialize): stall cut, program-aware eviction, lowest-free
// allocation, sources, hit accounting, fill descriptors.  One CTA per replica.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "k_sched.cuh"

// need(p) on replica r = #{sb <= j < nb : loc[j] is not HBM on r}.  HBM entries of a
// program always form the prefix [0, n_hbm) of its row (invariant I10: growth
// appends, eviction is tail-first), so need = nb - n_hbm on the home replica; the sb
// shared-prefix blocks (NEXT-3) are resident on every replica.
__device__ __forceinline__ u32 need_of(const Dev& d, u32 p, int r) {
  return d.home[p] == r ? d.nb[p] - d.n_hbm[p] : d.nb[p] - sb_of(d, d.kp[p]);
}

// NEXT-3 (A51): the prompt blocks F_r entries bring.  A prompt not resident on r (no
// program homed there uses it) is materialized by the first entry (slot order) that uses
// it: fc[i] += its blocks, f_x[i] = blocks | prompt << 16.  One CTA, fp / fc global.
__device__ __forceinline__ void prompt_extras(const Dev& d, int r, const u32* fp, u32 nF, u32* fc, u32* f_x) {
  __shared__ u32 s_kfirst[TA_MAX_PREFIXES];
  if (threadIdx.x < TA_MAX_PREFIXES) s_kfirst[threadIdx.x] = 0xFFFFFFFFu;
  __syncthreads();
  if (d.K) {
    for (u32 i = threadIdx.x; i < nF; i += CTA) {
      const u8 k = d.kp[fp[i]];
      if (k != KP_NONE && d.pref[(size_t)r * d.K + k] == 0) atomicMin(&s_kfirst[k], i);
    }
    __syncthreads();
  }
  for (u32 i = threadIdx.x; i < nF; i += CTA) {
    const u8 k = d.K ? d.kp[fp[i]] : (u8)KP_NONE;
    const u32 x = (k != KP_NONE && s_kfirst[k] == i) ? d.sbk[k] : 0u;
    fc[i] += x;
    f_x[i] = x | ((u32)k << 16);
  }
  __syncthreads();
}

// warp-aggregated add of a per-thread counter into a shared accumulator
__device__ __forceinline__ void warp_add_shared(ull v, ull* s) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  if (lane_id() == 0 && v) atomicAdd(s, v);
}

enum { PC_P2P, PC_H2D, PC_REC, PC_NEW, PC_FILLTOK, PC_HIT, PC_PEER, PC_HOST, PC_MISS, PC_NEWTOK,
       PC_STALL, PC_PREFIX, PC_N };

// Step 5 of replica r by a thread-block cluster of PLAN_CL CTAs (SM90+ clusters with
// distributed shared memory).  The leader CTA (rank 0) runs the inherently serial
// parts: F_r and the stall cut, the eviction order, host-slot and allocation
// prefixes, hit accounting.  The two per-block loops (one iteration per evicted block,
// one per requested block) are split over all CTAs of the cluster: each copies the
// leader's staged lists into its own shared memory through DSMEM, takes a contiguous
// range, and appends to the leader's shared counters/bitmap with DSMEM atomics.  The
// leader stays off both loops and off everything that does not depend on its chain:
// rank 1 builds the host-tier select prefix (part A) and the allocation prefix (part
// B), rank 2 orders the D2H copies (part B); the loops run on ranks 1..PLAN_CL-1.
// Copy descriptors keep request order: per-CTA compaction into a staging buffer, then
// placement at the prefix of the CTAs' counts.
#define PLAN_CL 8

struct PlanSh {                  // leader's scalars, read by the cluster through DSMEM
  u32 stop, X, hfree, nv, vst, ecs_sm, m, tot, fst, fcs_sm, nF;
  u32 hfree0;                    // free host-tier slots before the evictions (rank 1, part A)
  u32 fcnt[PLAN_CL];
  ull fr, es;                    // free blocks and eviction supply (rank 2, before #0)
};

__device__ __forceinline__ void cl_copy(u32* dst, const u32* src, u32 n) {
  for (u32 i = threadIdx.x; i < n; i += CTA) dst[i] = src[i];
}

// Several (DSMEM) -> shared copies as one index space, four loads in flight per thread
// (one loop per array would serialise their remote-load latencies).
struct CpSeg { u32* dst; const u32* src; u32 n; };
template <int K>
__device__ __forceinline__ void cl_copy_segs(const CpSeg (&sg)[K]) {
  u32 tot = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) tot += sg[k].n;
  for (u32 i0 = threadIdx.x; i0 < tot; i0 += 4 * CTA) {
    u32 v[4];
    u32* dp[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      dp[u] = nullptr;
      v[u] = 0;
      u32 off = i0 + u * CTA;
      if (off >= tot) continue;
      const u32* sp = nullptr;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (sp == nullptr) {
          if (off < sg[k].n) { sp = sg[k].src + off; dp[u] = sg[k].dst + off; }
          else off -= sg[k].n;
        }
      }
      v[u] = *sp;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (dp[u]) *dp[u] = v[u];
  }
}

// VERB (compile time): 0 = tick, 1 = ta_resume / ta_migrate (each a kernel of its own,
// so the tick kernel carries no verb code)
template <int VERB>
__device__ __forceinline__ void plan_pass(const Dev& d, const int r, u32* s_big, u32* s_tmp) {
  constexpr int verb = VERB;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const u32 crank = cl.block_rank();
  const bool lead = crank == 0;
  __shared__ ull s_red[NWARP];
  __shared__ u32 s_app[4];              // appends: fed, fld, dfh, dfs (leader's are the live ones)
  __shared__ ull s_pc[PC_N];
  __shared__ PlanSh sh;
  __shared__ u32 s_h2d_src[TA_MAX_REPLICAS];  // H2D requests by source tier (telemetry)
  extern __shared__ __align__(16) char dsm[];
  SortSmem* sm = reinterpret_cast<SortSmem*>(dsm);
  u32* s_fc = reinterpret_cast<u32*>(dsm + sizeof(SortSmem));   // staged need prefix  [4096]
  u32* s_ec = s_fc + 4096;                                         // staged evict prefix [4096]
  u32* s_hw = s_ec + 4096;                                         // staged HBM free bitmap [4096]
  u32* s_fl = s_hw + 4096;                                         // F_r in slot order, first 4096 [4096]
  // sort buffers, reused once the sorts are done: host-tier free words, victims,
  // per-F-program values of the request loop
  u32* s_sfw = sm->p[0];                               // [8192] >= NHW (NH <= 262112)
  u32* s_vp = reinterpret_cast<u32*>(sm->k[0]);        // [8192]
  u32* s_vn = s_vp + 8192;                             // [8192]
  // [FST_MAX] x 6 per-program values of the request loop, in the F-list region of the
  // request-loop ranks (unused there): the leader writes them into every rank's copy
  // through DSMEM during its hit accounting, so nobody reads them remotely after #2
  constexpr u32 FST_MAX = 576;                         // 7 arrays in the 4096-word region
  u32* s_fp = s_fl;
  u32* s_fj = s_fp + FST_MAX;
  u32* s_fh = s_fp + 2 * FST_MAX;
  u32* s_fk = s_fp + 3 * FST_MAX;
  u32* s_fcn = s_fp + 4 * FST_MAX;
  u32* s_fu = s_fp + 5 * FST_MAX;
  u32* s_fx = s_fp + 6 * FST_MAX;                      // prompt blocks brought | prompt << 16
  PlanSh* L = cl.map_shared_rank(&sh, 0);              // leader's scalars
  const int N = d.N;
  const u32 bt = (u32)d.bt;
  const bool fill = (d.flags & TA_F_FILL) != 0;
  // uniform over the cluster (depends on r and global state only)
  if (!verb && d.ctr->err != TA_OK) return;           // API batch rejected: the tick does not run
  if (verb && (r != d.ctr->verb_replica || d.ctr->err != TA_OK ||
               d.status[d.ctr->verb_pid] != TA_REASONING)) return;   // phase-A restores move no bytes
  if (TA_FLAG(d, TA_F_TIMING) && r == 0 && lead && threadIdx.x < 32) d.pst[2 * 32 + threadIdx.x] = 0;
  if (TA_FLAG(d, TA_F_TIMING) && (blockIdx.x == 1 || blockIdx.x == 3) && threadIdx.x < 32)
    d.pst[(blockIdx.x == 1 ? 4 : 5) * 32 + threadIdx.x] = 0;
  PSTAMP_B(4, 1, 0); PSTAMP_B(5, 3, 0);
  PSTAMP(2, 0);
  if (threadIdx.x < 4) s_app[threadIdx.x] = 0;
  if (threadIdx.x < PC_N) s_pc[threadIdx.x] = 0;
  if (threadIdx.x < TA_MAX_REPLICAS) s_h2d_src[threadIdx.x] = 0;
  u32* fp = d.f_pid + (size_t)r * N;
  u32* fc = d.f_cum + (size_t)r * N;
  u32* hf = d.hbm_free + (size_t)r * d.NBW;
  u32* sf = d.host_free + (size_t)r * d.NHW;
  u32* ep = d.e_pid + (size_t)r * N;
  u32* ec = d.e_cum + (size_t)r * N;
  EvDesc* evt = d.evt + (size_t)r * d.NB;   // (block, slot) in eviction order
  u32 pc[PC_N];
#pragma unroll
  for (int i = 0; i < PC_N; ++i) pc[i] = 0;

  // ================= rank 1, concurrent with part A: host-tier free-word snapshot and
  // its select prefix (the host bitmap is not touched before the eviction loop)
  if (crank == 1) {
    cta_bitmap_prefix(sf, d.NHW, s_big, s_tmp);
    if (threadIdx.x == 0) L->hfree0 = s_big[d.NHW];
    cl_copy(s_sfw, sf, d.NHW);
  }
  // ================= rank 2, concurrent with F_r: free blocks on r and eviction supply
  if (crank == 2) {
    ull fr = 0, es = 0;
    for (int w = threadIdx.x; w < d.NBW; w += CTA) fr += __popc(hf[w]);
    const u32* el = nullptr;                        // home == r with HBM blocks (footprint pass)
    const int nel = (int)cta_bits_to_list(d.ec_bits + (size_t)r * d.NW, d.NW, reinterpret_cast<u32*>(sm->k[0]),
                                          small_paths(d) ? 8u : 8192u, d.ec_list + (size_t)r * N, s_tmp, &el);
    for (int i = threadIdx.x; i < nel; i += CTA) {
      const u32 p = el[i];
      const u8 s = d.status[p];
      if (s == TA_PAUSED || s == TA_ACTING) es += d.n_hbm[p] - sb_of(d, d.kp[p]);   // private HBM blocks
    }
    auto add = [](ull a, ull b) { return a + b; };
    fr = cta_reduce<ull>(fr, s_red, add, 0ull);
    es = cta_reduce<ull>(es, s_red, add, 0ull);
    if (threadIdx.x == 0) { L->fr = fr; L->es = es; }   // into the leader's scalars
  }
  // ================= leader, part A: F_r, stall cut, eviction order, staging
  {                                                    // part A scope
  u32 nF = 0;
  bool fcs_sm = false;
  const u32* fcs = fc;
  if (lead) {
    // ---- 5.1 F_r: REASONING programs placed on r, slot order, with their need
    if (verb) {
      if (threadIdx.x == 0) {
        u32 p = d.ctr->verb_pid;
        fp[0] = p;
        fc[0] = need_of(d, p, r);
      }
      nF = 1;
      __syncthreads();
      prompt_extras(d, r, fp, nF, fc, d.f_x + (size_t)r * N);
    } else {
      // F_r = REASONING placed on r now: the footprint pass's REASONING set on r, minus
      // the programs this tick's pause pass took off r, plus the phase-R programs the
      // restore pass put on r.  The bitmap (in shared memory; NW <= 8192) gives the slot
      // order; the sort buffers are free here.  The words, the pause list and the restore
      // entries are loaded together (one round trip after their counts).
      u32* s_bits = reinterpret_cast<u32*>(sm->k[0]);
      const int NW = d.NW;
      const u32 np = d.pause_cnt[r], nr = d.ctr->restore_cnt;
      for (int w = threadIdx.x; w < NW; w += CTA) s_bits[w] = d.reas_bits[(size_t)r * NW + w];
      u32 pq = 0xFFFFFFFFu, rq = 0xFFFFFFFFu, rx = 0;
      if (threadIdx.x < np) pq = d.pause_list[(size_t)r * N + threadIdx.x];
      if (threadIdx.x < nr) { rx = d.restore_dst[threadIdx.x]; rq = d.restore_pid[threadIdx.x]; }
      __syncthreads();
      for (u32 i = threadIdx.x + CTA; i < np; i += CTA) {          // long lists: the rest
        const u32 q = d.pause_list[(size_t)r * N + i];
        atomicAnd(&s_bits[q >> 5], ~(1u << (q & 31)));
      }
      if (pq != 0xFFFFFFFFu) atomicAnd(&s_bits[pq >> 5], ~(1u << (pq & 31)));
      __syncthreads();
      for (u32 i = threadIdx.x + CTA; i < nr; i += CTA) {
        const u32 x = d.restore_dst[i];
        if ((int)(x & 0xFFu) == r && !((x >> 24) & 1u)) {
          const u32 q = d.restore_pid[i];
          atomicOr(&s_bits[q >> 5], 1u << (q & 31));
        }
      }
      if (rq != 0xFFFFFFFFu && (int)(rx & 0xFFu) == r && !((rx >> 24) & 1u))   // restored onto r, phase R
        atomicOr(&s_bits[rq >> 5], 1u << (rq & 31));
      __syncthreads();
      cta_bitmap_prefix(s_bits, NW, s_big, s_tmp);
      nF = s_big[NW];
      for (int w = threadIdx.x; w < NW; w += CTA) {
        u32 m = s_bits[w], pos = s_big[w];
        while (m) {
          const u32 q = (u32)w * 32u + (u32)(__ffs(m) - 1);
          m &= m - 1;
          fp[pos] = q;
          if (pos < 4096) s_fl[pos] = q;
          ++pos;
        }
      }
      __syncthreads();
      for (u32 i = threadIdx.x; i < nF; i += CTA) fc[i] = need_of(d, i < 4096 ? s_fl[i] : fp[i], r);
      __syncthreads();
      prompt_extras(d, r, fp, nF, fc, d.f_x + (size_t)r * N);
      cta_incl_scan_array(fc, (int)nF, s_tmp);
    }
    // short lists are searched many times below: stage them in shared memory
    fcs_sm = nF <= (small_paths(d) ? 8u : 4096u);
    if (!fcs_sm) dbg_hit(d, DBG_F_GLOBAL);
    if (fcs_sm) {                        // the need prefix, into every rank's s_fc (DSMEM stores)
      for (u32 i = threadIdx.x; i < nF; i += CTA) {
        const u32 v = fc[i];
        s_fc[i] = v;
#pragma unroll
        for (int k = 1; k < PLAN_CL; ++k) cl.map_shared_rank(s_fc, k)[i] = v;
      }
      __syncthreads();
    }
    fcs = fcs_sm ? s_fc : fc;
    PSTAMP(2, 1);
  }
  cl.sync();                                           // #0: rank 2's supply reaches the leader
  jitter(d, 200u);
  if (lead) {
    const u32* el = nullptr;                        // home == r with HBM blocks (footprint pass)
    int nel = 0;
    const ull fr = sh.fr, es = sh.es;
    const ull supply = fr + es;
    // ---- 5.2 stall cut: longest prefix of F_r with sum(need) <= supply
    const u32 m = nF ? (u32)upper_bound_u32(fcs, (int)nF, supply > 0xFFFFFFFFull ? 0xFFFFFFFFu : (u32)supply) : 0;
    u32 stop = 0;
    if (verb) {
      if (m < nF) {                      // all-or-nothing: fail before any mutation
        if (threadIdx.x == 0) d.ctr->verb_ok = 0;
        stop = 1;
      } else if (threadIdx.x == 0) {
        d.ctr->verb_ok = 1;
      }
    }
    PSTAMP(2, 2);
    const u32 tot = m ? fcs[m - 1] : 0;
    const u32 X = stop ? 0 : (tot > fr ? (u32)(tot - fr) : 0);
    u32 nv = 0, hfree = 0, vst = 0, ecs_sm = 0;
    // ---- 5.3 eviction: E_r ordered (group 0 PAUSED, reverse restore order; group 1
    // ACTING placed elsewhere; group 2 ACTING placed on r; groups 1-2 by contrib),
    // whole programs tail-first, last victim partially; host tier first, else drop.
    if (X > 0) {
      u64* ka = d.ska + (size_t)r * N;
      u64* kb = d.skb + (size_t)r * N;
      u32* va = d.sva + (size_t)r * N;
      u32* vb = d.svb + (size_t)r * N;
      // exact prefix of E covering X blocks: buckets monotone in the eviction order
      const u32 NBK = d.nbk, shf = d.nb_shift;
      auto epred = [&](int i) {          // on the list: home == r and n_hbm > 0 already
        u8 s = d.status[i];
        return s == TA_PAUSED || s == TA_ACTING;
      };
      const bool ra = TA_FLAG(d, TA_F_REQUEST_AWARE);   // RequestAware: LRU (A46)
      auto ebucket = [&](int i) -> u32 {
        if (ra) return 0u;
        if (d.status[i] == TA_PAUSED)    // group 0: A first, nb descending
          return (u32)(d.phase[i] == TA_PHASE_A ? 0 : 1) * NBK + (NBK - 1 - (d.nb[i] >> shf));
        return (u32)(d.placement[i] != r ? 2 : 3) * NBK + (d.contrib[i] >> shf);
      };
      // the candidates as a slot list in shared memory (s_ec and s_hw, 8192 words, free
      // until the sorted order is staged), else in global scratch
      {
        const u32 cap = small_paths(d) ? 8u : 8192u;
        nel = (int)cta_bits_to_list(d.ec_bits + (size_t)r * d.NW, d.NW, s_ec, cap, d.ec_list + (size_t)r * N,
                                    s_tmp, &el);
        if ((u32)nel > cap) dbg_hit(d, DBG_LIST_GLOBAL);
      }
      const u32 T = cta_list_threshold(el, nel, 4 * NBK, 0, X, s_big, s_tmp, epred, ebucket,
                                       [&](int i) { return d.n_hbm[i] - sb_of(d, d.kp[i]); });
      PSTAMP(2, 3);
      // keys: group 0 (PAUSED) = exact reverse of the restore order, ties slot-down (the
      // tie-break value N-1-slot); groups 1-2 (ACTING) = (group, contrib), ties slot-up
      __shared__ u32 s_cnt2;
      const u32 ne = cta_list_gather(el, nel, &s_cnt2,
          [&](int i) { return epred(i) && ebucket(i) <= T; },
          [&](u32 pos, int i) {
            if (ra) {                    // idle since (ms), least recent first; ties slot-up
              const u64 idle = d.status[i] == TA_PAUSED ? (u64)d.paused_since[i] * (u64)d.dt
                                                        : (u64)d.acting_since[i];
              ka[pos] = (1ull << 62) | idle;
              va[pos] = (u32)i;
            } else if (d.status[i] == TA_PAUSED) {
              u64 rk = ((u64)(d.phase[i] == TA_PHASE_A) << 55) | ((u64)d.nb[i] << 32) | d.paused_since[i];
              ka[pos] = ((1ull << 56) - 1) - rk;
              va[pos] = (u32)(N - 1 - i);
            } else {
              u64 g = d.placement[i] != r ? 1 : 2;
              ka[pos] = (g << 62) | d.contrib[i];
              va[pos] = (u32)i;
            }
          });
      PSTAMP(2, 4);
      if (TA_FLAG(d, TA_F_TIMING) && r == 0 && threadIdx.x == 0) {
        d.pst[2 * 32 + 27] = ne | (1ull << 62);
        d.pst[2 * 32 + 28] = X | (1ull << 62);
      }
      int res = cta_sort_kv(ka, va, kb, vb, (int)ne, s_big, s_tmp, sm, sort_lim(d));
      const u64* sk = res ? kb : ka;
      const u32* sv = res ? vb : va;
      PSTAMP(2, 5);
      for (u32 i = threadIdx.x; i < ne; i += CTA) {
        const u32 p = (sk[i] >> 62) == 0 ? (u32)(N - 1) - sv[i] : sv[i];   // undo the group-0 tie-break
        ep[i] = p;
        ec[i] = d.n_hbm[p] - sb_of(d, d.kp[p]);
      }
      __syncthreads();
      cta_incl_scan_array(ec, (int)ne, s_tmp);
      ecs_sm = ne <= (small_paths(d) ? 8u : 4096u);
      if (!ecs_sm) dbg_hit(d, DBG_E_GLOBAL);
      dbg_hit(d, DBG_EVICT_TICKS);
      if (ecs_sm) {
        cl_copy(s_ec, ec, ne);
        __syncthreads();
      }
      nv = (u32)upper_bound_u32(ecs_sm ? s_ec : ec, (int)ne, X - 1) + 1;   // victims
      PSTAMP(2, 13);
      // victims' slot and HBM prefix length (the host-tier snapshot and its select
      // prefix are rank 1's)
      vst = nv <= (small_paths(d) ? 8u : 8192u);
      if (!vst) dbg_hit(d, DBG_V_GLOBAL);
      if (vst)
        for (u32 v = threadIdx.x; v < nv; v += CTA) { const u32 p = ep[v]; s_vp[v] = p; s_vn[v] = d.n_hbm[p]; }
      for (int w = threadIdx.x; w < d.NBW; w += CTA) s_hw[w] = 0;   // blocks evicted to host (bitmap)
    }
    PSTAMP(2, 14);
    if (threadIdx.x == 0) {
      sh.stop = stop; sh.X = X; sh.hfree = hfree; sh.nv = nv; sh.vst = vst; sh.ecs_sm = ecs_sm;
      sh.m = m; sh.tot = stop ? 0 : tot; sh.nF = nF; sh.fcs_sm = fcs_sm;
    }
  }
  }                                                    // part A scope
  cl.sync();                                           // #1: part A visible to the cluster
  jitter(d, 201u);
  PSTAMP_B(4, 1, 1); PSTAMP_B(5, 3, 1);

  // ================= all CTAs: the eviction loop, split by cluster rank
  PSTAMP(2, 15);
  const u32 X = L->X;
  if (L->stop) {
    cl.sync();                                         // leader's smem outlives every reader
    return;
  }
  FillDesc* fld = d.fld + (size_t)r * d.NB;
  if (lead) {
    // the leader, while the others evict: hit accounting of S_r (reads only S_r's rows
    // and counters, which the evictions do not touch: victims are PAUSED / ACTING)
    if (X > 0 && threadIdx.x == 0) sh.hfree = cl.map_shared_rank(s_big, 1)[d.NHW];   // rank 1's, before #2
    const u32 m = sh.m, nF = sh.nF;
    const u32* fcs = sh.fcs_sm ? s_fc : fc;
    // per-program values the request loop reads for each of its blocks, staged for
    // S_r programs when they fit: slot, first needed j, home, c_kv, c, uid
    const bool fst = m <= (small_paths(d) ? 4u : FST_MAX);
    if (!fst) dbg_hit(d, DBG_FST_GLOBAL);
    ull l_dec = 0, l_pre = 0, l_rec = 0;             // NEXT-1 STP ledger (token-ms)
    // ---- 5.6 hit accounting, FETCH / STALL records, new tokens into a resident partial block
    for (u32 i = threadIdx.x; i < nF; i += CTA) {
      u32 p = (verb || i >= 4096) ? fp[i] : s_fl[i];
      u32 need = fcs[i] - (i ? fcs[i - 1] : 0);
      // every per-program value up front: one memory round trip for the whole record
      const int h = d.home[p];
      const u32 ckv = d.c_kv[p], c = d.c[p], nhp = d.n_hbm[p], uidp = d.uid[p], nsp = d.n_host[p];
      const u32 pendp = d.pend[p], fx = d.f_x[(size_t)r * N + i];
      const u8 satp = d.satisfied[p], cls = d.hcls[p];
      const u32 sbp = sb_of(d, (u8)(fx >> 16)), xb = fx & 0xFFFFu;   // prompt blocks, brought now
      ta_decision rec;
      rec.pid = p; rec.src = h; rec.dst = r; rec.blocks = need; rec.to_host = 0; rec.dropped = 0;
      rec.hit_tok = rec.peer_tok = rec.host_tok = rec.miss_tok = rec.new_tok = 0;
      if (i < m) {
        if (fst) {
          u32* lf = sm->p[0];                          // leader-local staging, pushed below
          lf[i] = p; lf[FST_MAX + i] = h == r ? nhp : sbp; lf[2 * FST_MAX + i] = (u32)h;
          lf[3 * FST_MAX + i] = ckv; lf[4 * FST_MAX + i] = c; lf[5 * FST_MAX + i] = uidp;
          lf[6 * FST_MAX + i] = fx;
        }
        const bool resumed = !(satp && h == r);
        if (resumed && ckv > 0) {
          u32 hb = ceil_div_u32(ckv, bt);
          u32 shs = bt - (ckv - (hb - 1) * bt);        // missing slots of the last block
          u32 nh = nhp, ns = nsp, nn = hb - nh - ns;
          ull th = (ull)nh * bt, ts = (ull)ns * bt, tn = (ull)nn * bt;
          // cls: entry hb - 1, classified by the footprint pass
          if (cls == 1) th -= shs; else if (cls == 2) ts -= shs; else tn -= shs;
          u32 sh_hit = 0, sh_miss = 0;
          if (sbp) {                                   // the shared prompt: resident on r (hit), or
            const ull sh = (ull)sbp * bt;              // materialized now by this program (miss);
            if (h >= 0) th -= sh; else tn -= sh;       // c_kv >= its prompt >= sbp * bt
            if (xb) sh_miss = (u32)sh; else sh_hit = (u32)sh;
          }
          rec.hit_tok = sh_hit;
          if (h == r) rec.hit_tok += (u32)th; else rec.peer_tok = (u32)th;
          rec.host_tok = (u32)ts;
          rec.miss_tok = (u32)tn + sh_miss;
        }
        rec.new_tok = c - ckv;
        rec.kind = (need > 0 || resumed) ? TA_D_FETCH : 0;
        l_dec += (ull)c * (ull)d.dt;                    // holds c while decoding the interval
        // engine time of this materialize: recompute + prefill of waiting tokens (A48)
        const u32 q = (u32)d.chunk_q;
        d.busy[p] = (u32)d.chunk_ms * (ceil_div_u32(rec.miss_tok, q) + ceil_div_u32(pendp, q));
        d.pend[p] = 0;
        l_pre += (ull)d.chunk_ms * stp_stair(c - ckv, (ull)d.chunk_q, ckv);
        l_rec += (ull)d.chunk_ms * stp_stair(rec.miss_tok, (ull)d.chunk_q, 0);
        pc[PC_HIT] += rec.hit_tok; pc[PC_PEER] += rec.peer_tok; pc[PC_HOST] += rec.host_tok;
        pc[PC_MISS] += rec.miss_tok; pc[PC_NEWTOK] += rec.new_tok;
        if (h == r && c > ckv && (ckv % bt) != 0) {    // partial last block already resident
          u32 j = ckv / bt;
          if (j < nhp) {
            u32 t1 = min((j + 1) * bt, c);
            pc[PC_FILLTOK] += t1 - ckv;
            if (fill) {
              u32 pos = atomicAdd(&s_app[1], 1u);
              fld[pos] = FillDesc{d.loc[(size_t)p * d.MAXBP + j], uidp, ckv, t1, j, 0};
            }
          }
        }
        // it now uses its prompt on r (the rows' prompt entries and the old home's release
        // follow in step 7, after every replica's materialize: k_close)
        if (sbp && h != r) atomicAdd(&d.pref[(size_t)r * d.K + (fx >> 16)], 1u);
        d.sat_new[p] = (u8)(r + 1);
      } else {
        rec.kind = TA_D_STALL;
        pc[PC_STALL] += 1;
      }
      d.dec_fs[(size_t)r * N + i] = rec;
    }
    if (threadIdx.x == 0) sh.fst = fst;
    if (fst && m) {                                    // the six staged arrays into every request-loop
      __syncthreads();                                 // rank's copy (DSMEM stores, published by #2)
      const u32* lf = sm->p[0];
      for (u32 x = threadIdx.x; x < 7 * m; x += CTA) {
        const u32 a6 = x / m, i = x - a6 * m, v = lf[a6 * FST_MAX + i];
#pragma unroll
        for (int k = 1; k < PLAN_CL; ++k) cl.map_shared_rank(s_fp, k)[a6 * FST_MAX + i] = v;
      }
    }
    if (!verb) {
      l_dec = warp_sum_ull(l_dec); l_pre = warp_sum_ull(l_pre); l_rec = warp_sum_ull(l_rec);
      if (lane_id() == 0) {
        if (l_dec) atomicAdd(&d.stats[ST_COST_DECODE], l_dec);
        if (l_pre) atomicAdd(&d.stats[ST_COST_PREFILL], l_pre);
        if (l_rec) atomicAdd(&d.stats[ST_COST_RECOMPUTE], l_rec);
      }
    }
    PSTAMP(2, 10);
    if (TA_FLAG(d, TA_F_TIMING) && r == 0 && threadIdx.x == 0) {
      d.pst[2 * 32 + 29] = nF | (1ull << 62);
      d.pst[2 * 32 + 30] = sh.tot | (1ull << 62);
    }
  } else if (X > 0) {
    const u32 nv = L->nv, vst = L->vst, ecs_sm = L->ecs_sm;
    {                                                  // the leader's lists, rank 1's host snapshot
      const u32 n1 = (crank == 1 || L->hfree0 == 0) ? 0u : 1u;   // no free host slot: all drops
      CpSeg sg[5] = {{s_ec, cl.map_shared_rank(s_ec, 0), ecs_sm ? nv : 0u},
                     {s_vp, cl.map_shared_rank(s_vp, 0), vst ? nv : 0u},
                     {s_vn, cl.map_shared_rank(s_vn, 0), vst ? nv : 0u},
                     {s_sfw, cl.map_shared_rank(s_sfw, 1), n1 * (u32)d.NHW},
                     {s_big, cl.map_shared_rank(s_big, 1), n1 * ((u32)d.NHW + 1)}};
      cl_copy_segs(sg);
      __syncthreads();
    }
    const u32 hfree = (crank == 1 || L->hfree0) ? s_big[d.NHW] : 0u;
    const u32* ecs = ecs_sm ? s_ec : ec;
    u32* Lhw = cl.map_shared_rank(s_hw, 0);            // leader's evicted-to-host bitmap
    const u32 per = (X + PLAN_CL - 2) / (PLAN_CL - 1); // ranks 1..PLAN_CL-1
    const u32 e_lo = (crank - 1) * per, e_hi = min(X, e_lo + per);
    // e-th evicted block: victim v, its block j = n_hbm - 1 - (e - excl) (tail first);
    // four per thread per round so their block-table loads are in flight together
    for (u32 e0 = e_lo; e0 < e_hi; e0 += 4 * CTA) {
      u32 pk[4], jk[4], ik[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const u32 e = e0 + k * CTA + threadIdx.x;
        pk[k] = jk[k] = ik[k] = 0;
        if (e < e_hi) {
          const u32 v = (u32)upper_bound_u32(ecs, (int)nv, e);
          const u32 excl = v ? ecs[v - 1] : 0;
          const u32 p = vst ? s_vp[v] : ep[v];
          const u32 nh = vst ? s_vn[v] : d.n_hbm[p];
          pk[k] = p;
          jk[k] = nh - 1 - (e - excl);
          ik[k] = d.loc[(size_t)p * d.MAXBP + jk[k]];
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const u32 e = e0 + k * CTA + threadIdx.x;
        if (e >= e_hi) continue;
        const u32 idx = ik[k], j = jk[k], p = pk[k];
        u32* ent = d.loc + (size_t)p * d.MAXBP + j;
        d.dirty[p] = 1;
        atomicOr(&hf[idx >> 5], 1u << (idx & 31));          // freed now (intra-replica)
        if (e < hfree) {
          if (evp_owner(d, r)) evp_of(d, r)[idx] = 2u * d.nL;  // segments pending their D2H read
          const u32 slot = bitmap_select(s_sfw, s_big, d.NHW, e);
          *ent = LOC_HOST | slot;
          d.owner_host[(size_t)r * d.NH + slot] = p * (u32)d.MAXB + j;
          evt[e] = EvDesc{idx, slot};
          atomicAnd(&sf[slot >> 5], ~(1u << (slot & 31)));
          atomicOr(&Lhw[idx >> 5], 1u << (idx & 31));
        } else {
          *ent = LOC_NONE;
        }
      }
    }
  }
  PSTAMP(2, 16);
  PSTAMP_B(4, 1, 2); PSTAMP_B(5, 3, 2);
  cl.sync();                                           // #2: evictions done
  jitter(d, 202u);
  PSTAMP_B(4, 1, 3); PSTAMP_B(5, 3, 3);
  PSTAMP(2, 6);

  // ================= part B.  Every request-loop rank (1..7): a snapshot of the free
  // bitmap after the evictions (the live bitmap; nobody writes it until #4, the request
  // loop's allocations are cleared after #4) and its select prefix, in its own shared
  // memory; meanwhile the leader orders the D2H copies and writes the EVICT records.
  if (!lead) {
    cl_copy(s_hw, hf, d.NBW);                          // NBW <= 4095 (NB <= 131040)
    __syncthreads();
    cta_bitmap_prefix(s_hw, d.NBW, s_big, s_tmp);
  }
  PSTAMP_B(4, 1, 4); PSTAMP_B(5, 3, 4);
  if (lead && X > 0) {
    // D2H copies are issued in ascending HBM-block order, the order in which the
    // allocation hands the freed blocks out again, so a fetch that reuses an evicted
    // block rarely waits for its eviction (fused movement kernel).
    const u32 ntoh = min(X, sh.hfree);
    EvDesc* evd = d.evd + (size_t)r * d.NB;
    if (ntoh) cta_bitmap_prefix(s_hw, d.NBW, s_big, s_tmp);   // s_hw: blocks evicted to host (bitmap)
    for (u32 e = threadIdx.x; e < ntoh; e += CTA) {
      const EvDesc x = evt[e];
      const u32 k = s_big[x.src >> 5] + __popc(s_hw[x.src >> 5] & ((1u << (x.src & 31)) - 1));
      evd[k] = x;
    }
  }
  if (lead) {
    const u32 nv = sh.nv, hfree = sh.hfree;
    if (X > 0) {
      const u32* ecs = sh.ecs_sm ? s_ec : ec;
      const u32 ntoh = min(X, hfree);
      PSTAMP(2, 7);
      for (u32 v = threadIdx.x; v < nv; v += CTA) {
        u32 p = ep[v];
        u32 excl = v ? ecs[v - 1] : 0;
        u32 take = (v == nv - 1) ? X - excl : d.n_hbm[p] - sb_of(d, d.kp[p]);
        u32 toh = hfree > excl ? min(take, hfree - excl) : 0;
        ta_decision rec;
        rec.kind = TA_D_EVICT; rec.pid = p; rec.src = r; rec.dst = -1; rec.blocks = take;
        rec.to_host = toh; rec.dropped = take - toh;
        rec.hit_tok = rec.peer_tok = rec.host_tok = rec.miss_tok = rec.new_tok = 0;
        d.dec_ev[(size_t)r * N + v] = rec;
        d.n_hbm[p] -= take;
        d.n_host[p] += toh;
      }
      if (threadIdx.x == 0) {
        d.ev_cnt[r] = nv;
        d.evd_cnt[r] = ntoh;
        d.t_rep[r] = ntoh;
        atomicAdd(&d.stats[ST_EVICT_BLOCKS], (ull)X);
        atomicAdd(&d.stats[ST_EVICT_TO_HOST], (ull)ntoh);
        atomicAdd(&d.ctr->t_d2h, ntoh);
        atomicAdd(&d.stats[ST_EVICT_DROPPED], (ull)(X - ntoh));
      }
      __syncthreads();
    }
    PSTAMP(2, 8);
    PSTAMP(2, 9);
  }

  PSTAMP(2, 17);
  // ================= all CTAs: the request loop, split by cluster rank
  // (p in S_r slot order, needed j ascending) -> q-th lowest free block.  Selects read
  // the staged snapshot of the free bitmap, so each request clears its block in the
  // live bitmap at once.  Only requests that move or write bytes get a descriptor
  // (copies; fills when the engine stand-in is on), compacted in request order.
  const u32 m = L->m, tot = L->tot, fst = L->fst, fcs_sm = L->fcs_sm;
  // (the leader's lists were written into this CTA's shared memory before #2)

  __syncthreads();
  const u32* fcs = fcs_sm ? s_fc : fc;
  const u32* hws = s_hw;
  u32* dfh = d.dfh + (size_t)r * d.NB;
  u32* dfs = d.dfs + (size_t)r * d.NB;
  u32* Lapp = cl.map_shared_rank(s_app, 0);            // leader's append counters
  const u32 per = (tot + PLAN_CL - 2) / (PLAN_CL - 1);  // ranks 1..PLAN_CL-1; the leader has none
  const u32 q_lo = lead ? tot : min(tot, (crank - 1) * per), q_hi = lead ? tot : min(tot, q_lo + per);
  FeDesc* fstage = d.fedt + (size_t)r * d.NB + q_lo;  // this CTA's descriptors, compacted
  u32 nfed = 0;
  for (u32 q0 = q_lo; q0 < q_hi; q0 += 2 * CTA) {
    u32 ik[2], pk[2], jk[2], dk[2], xk[2];
    int hk[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {                       // block-table loads of both in flight
      const u32 q = q0 + k * CTA + threadIdx.x;
      ik[k] = pk[k] = jk[k] = dk[k] = xk[k] = 0;
      hk[k] = 0;
      if (q < q_hi) {
        const u32 i = (u32)upper_bound_u32(fcs, (int)m, q);
        const u32 excl = i ? fcs[i - 1] : 0;
        const u32 p = fst ? s_fp[i] : fp[i];
        const int h = fst ? (int)s_fh[i] : d.home[p];
        const u32 fx = fst ? s_fx[i] : d.f_x[(size_t)r * N + i];
        const u32 xb = fx & 0xFFFFu, off = q - excl;
        dk[k] = bitmap_select(hws, s_big, d.NBW, q);
        pk[k] = fst ? i : p;
        hk[k] = h;
        if (off < xb) {                                 // one of the prompt blocks it brings (A51)
          jk[k] = off;
          xk[k] = 1u | (fx & 0xFFFF0000u);
          ik[k] = LOC_NONE;
        } else {
          const u32 j = (fst ? s_fj[i] : (h == r ? d.n_hbm[p] : sb_of(d, (u8)(fx >> 16)))) + (off - xb);
          jk[k] = j;
          ik[k] = d.loc[(size_t)p * d.MAXBP + j];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const u32 q = q0 + k * CTA + threadIdx.x;
      FeDesc x{MV_NONE, 0, 0, 0, 0, 0, 0, 0};
      if (q < q_hi && xk[k]) {                          // prompt block jj of prompt pk: prefilled
        const u32 pr = xk[k] >> 16, jj = jk[k], dst = dk[k];
        d.pblk[((size_t)r * d.K + pr) * d.SBM + jj] = dst;
        d.owner_hbm[(size_t)r * d.NB + dst] = OWNER_PROMPT | (pr << 20) | jj;
        atomicOr(&d.pfix[(size_t)r * d.NBW + (dst >> 5)], 1u << (dst & 31));
        pc[PC_PREFIX] += 1;
        pc[PC_FILLTOK] += bt;
        if (fill) x = FeDesc{MV_FILL, 0, 0, dst, TA_PROMPT_UID + pr, jj * bt, (jj + 1) * bt, jj};
      } else if (q < q_hi) {
        const u32 p = fst ? s_fp[pk[k]] : pk[k];
        const int h = hk[k];
        const u32 j = jk[k], dst = dk[k], old = ik[k];
        const u32 ckv = fst ? s_fk[pk[k]] : d.c_kv[p];
        const u32 c = fst ? s_fcn[pk[k]] : d.c[p];
        const u32 uid = fst ? s_fu[pk[k]] : d.uid[p];
        const u32 hb = ceil_div_u32(ckv, bt);
        const u32 jb = j * bt, je = min(jb + bt, c);
        if (is_hbm(old) || is_host(old)) {              // copy: P2P (HBM of h != r) or H2D (tier of h)
          // a copied partial block that also receives new tokens carries the fill of its
          // tail [max(jb, c_kv), je) in the same descriptor (written after the copy)
          u32 t0 = 0, t1 = 0;
          if (ckv < c && jb + bt > ckv) {
            t0 = max(jb, ckv);
            t1 = je;
            pc[PC_FILLTOK] += t1 - t0;
            if (!fill) t0 = t1 = 0;
          }
          if (is_hbm(old)) {
            x = FeDesc{MV_P2P, (u32)h, old, dst, uid, t0, t1, j};
            dfh[atomicAdd(&Lapp[2], 1u)] = ((u32)h << 27) | old;
            pc[PC_P2P] += 1;
          } else {
            x = FeDesc{MV_H2D, (u32)h, old & ~LOC_HOST, dst, uid, t0, t1, j};
            dfs[atomicAdd(&Lapp[3], 1u)] = ((u32)h << 27) | (old & ~LOC_HOST);
            atomicAdd(&s_h2d_src[h], 1u);
            pc[PC_H2D] += 1;
          }
        } else {                                        // recompute history / brand-new tokens
          if (j < hb) pc[PC_REC] += 1; else pc[PC_NEW] += 1;
          pc[PC_FILLTOK] += je - jb;
          if (fill) x = FeDesc{MV_FILL, 0, 0, dst, uid, jb, je, j};
        }
        d.loc[(size_t)p * d.MAXBP + j] = dst;
        d.dirty[p] = 1;
        d.owner_hbm[(size_t)r * d.NB + dst] = p * (u32)d.MAXB + j;
      }
      u32 round_n;
      const u32 pos = cta_excl_scan(x.kind != MV_NONE ? 1u : 0u, s_tmp, &round_n);
      if (x.kind != MV_NONE) fstage[nfed + pos] = x;
      nfed += round_n;
    }
  }
  PSTAMP(2, 18);
  PSTAMP_B(4, 1, 7); PSTAMP_B(5, 3, 7);
  // per-CTA counters: warp sums (one redux per counter), then shared 64-bit atomics
#pragma unroll
  for (int i = 0; i < PC_N; ++i) {
    const u32 v = __reduce_add_sync(FULL_MASK, pc[i]);
    if (lane_id() == 0 && v) atomicAdd(&s_pc[i], (ull)v);
  }
  // every CTA's count into every CTA's copy, so nothing is read remotely after #4 and
  // no CTA has to outlive the others (no closing cluster barrier)
  if (threadIdx.x < PLAN_CL) cl.map_shared_rank(&sh, threadIdx.x)->fcnt[crank] = nfed;
  cl.sync();                                           // #4: counts of every CTA known
  jitter(d, 203u);
  PSTAMP_B(4, 1, 8); PSTAMP_B(5, 3, 8);
  if (!lead && tot) {                                  // allocated = the first tot free blocks of the
    for (u32 w = (u32)(crank - 1) * CTA + threadIdx.x; w < (u32)d.NBW; w += (PLAN_CL - 1) * CTA) {
      const u32 pre = s_big[w], fw = s_hw[w];          // snapshot: clear them in the live bitmap
      if (pre >= tot || fw == 0) continue;
      const u32 k = tot - pre;                         // the lowest k free bits of this word are taken
      hf[w] = k >= (u32)__popc(fw) ? 0u : fw & ~((1u << __fns(fw, 0, (int)k + 1)) - 1u);
    }
  }
  u32 base = 0, total_fed = 0;
  for (u32 c = 0; c < PLAN_CL; ++c) {
    const u32 n = sh.fcnt[c];
    if (c < crank) base += n;
    total_fed += n;
  }
  FeDesc* fed = d.fed + (size_t)r * d.NB;
  for (u32 i = threadIdx.x; i < nfed; i += CTA) fed[base + i] = fstage[i];
  if (threadIdx.x < d.R && s_h2d_src[threadIdx.x]) atomicAdd(&d.t_rep[d.R + threadIdx.x], s_h2d_src[threadIdx.x]);
  if (threadIdx.x == 0) {
    if (s_pc[PC_P2P]) atomicAdd(&d.t_rep[2 * d.R + r], (u32)s_pc[PC_P2P]);
    atomicAdd(&d.stats[ST_P2P], s_pc[PC_P2P]);
    atomicAdd(&d.stats[ST_H2D], s_pc[PC_H2D]);
    atomicAdd(&d.ctr->t_p2p, (u32)s_pc[PC_P2P]);
    atomicAdd(&d.ctr->t_h2d, (u32)s_pc[PC_H2D]);
    u32 cross = (u32)s_pc[PC_P2P];                     // copies another process takes part in
    for (int h = 0; h < d.R; ++h)
      if (h != r) cross += s_h2d_src[h];
    if (cross) atomicAdd(&d.ctr->t_cross, cross);
    atomicAdd(&d.stats[ST_RECOMPUTE], s_pc[PC_REC]);
    atomicAdd(&d.stats[ST_NEW_BLOCKS], s_pc[PC_NEW]);
    atomicAdd(&d.stats[ST_FILL_TOK], s_pc[PC_FILLTOK]);
    atomicAdd(&d.stats[ST_HIT], s_pc[PC_HIT]);
    atomicAdd(&d.stats[ST_PEER], s_pc[PC_PEER]);
    atomicAdd(&d.stats[ST_HOST], s_pc[PC_HOST]);
    atomicAdd(&d.stats[ST_MISS], s_pc[PC_MISS]);
    atomicAdd(&d.stats[ST_NEW_TOK], s_pc[PC_NEWTOK]);
    atomicAdd(&d.stats[ST_STALLS], s_pc[PC_STALL]);
    if (s_pc[PC_PREFIX]) atomicAdd(&d.stats[ST_PREFIX_BLOCKS], s_pc[PC_PREFIX]);
    if (lead) {
      d.f_cnt[r] = sh.nF;
      d.s_cnt[r] = m;
      d.fed_cnt[r] = total_fed;          // copy / fill descriptors, in request order
      d.fld_cnt[r] = s_app[1];
      d.dfh_cnt[r] = s_app[2];
      d.dfs_cnt[r] = s_app[3];
      atomicAdd(&d.stats[ST_FETCH_BLOCKS], (ull)tot);
      atomicAdd(&d.ctr->t_fetch, tot);
    }
  }
  PSTAMP(2, 11);
  PSTAMP(2, 12);
}

// Steps 3 and 4 as their own kernels (one CTA per replica; one CTA).  Measured: one
// cooperative kernel for steps 3-5 with grid barriers was slower (register pressure
// of the merged code outweighs the two launch gaps).
__global__ void __launch_bounds__(CTA, 1) k_pause(const __grid_constant__ Dev d) {
  __shared__ u32 s_big[8192 + 1];
  __shared__ u32 s_tmp[NWARP + 1];
  pause_pass(d, blockIdx.x, s_big, s_tmp);
}

__global__ void __launch_bounds__(CTA, 1) k_restore(const __grid_constant__ Dev d) {
  __shared__ u32 s_big[8192 + 1];
  __shared__ u32 s_tmp[NWARP + 1];
  restore_pass(d, s_big, s_tmp);
}

// Steps 3 + 4 in one cooperative launch of R CTAs: CTA r's pause pass, a grid barrier,
// the restore pass on CTA 0 (one launch less per tick than k_pause + k_restore).
__global__ void __launch_bounds__(CTA, 1) k_pause_restore(const __grid_constant__ Dev d) {
  const ull t_in = gtimer();   // the CTA's first instruction (kernel span, timing mode)
  __shared__ u32 s_big[8192 + 1];
  __shared__ u32 s_tmp[NWARP + 1];
  kspan_begin(d, KS_PR, t_in);
  jitter(d, 1u);
  pause_pass(d, blockIdx.x, s_big, s_tmp);
  grid_sync(d, 0);
  if (blockIdx.x == 0) restore_pass(d, s_big, s_tmp);
  kspan_end(d, KS_PR);
}

// Step 5 per replica: cluster r (PLAN_CL CTAs); verb != 0: ta_resume / ta_migrate,
// the verb's program only.  Grid = R * PLAN_CL.
template <int VERB>
__global__ void __cluster_dims__(PLAN_CL, 1, 1) __launch_bounds__(CTA, 1)
k_plan(const __grid_constant__ Dev d) {
  const ull t_in = gtimer();   // the CTA's first instruction (kernel span, timing mode)
  __shared__ u32 s_big[8192 + 1];       // radix histogram / bitmap prefix counts
  __shared__ u32 s_tmp[NWARP + 1];
  kspan_begin(d, KS_PLAN, t_in);
  jitter(d, 2u);
  plan_pass<VERB>(d, blockIdx.x / PLAN_CL, s_big, s_tmp);
  kspan_end(d, KS_PLAN);
}
