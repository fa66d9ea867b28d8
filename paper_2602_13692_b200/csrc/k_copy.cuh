// k_copy.cuh — step 6 (KV block movement) and the engine stand-in (content fill).
//
// A KV block is 2L segments of seg_bytes = bt*Hkv*D*2 bytes.  Layer-major pools
// (layout 0, vLLM-like) place segment s = 2l+kv of block b at base + (s*NB + b)*seg;
// block-major pools (layout 1) at base + (b*2L + s)*seg.  Every copy kernel is
// driven by a device-resident descriptor list whose length is read on the device,
// so the whole tick is one CUDA-graph replay with no host round trip.
#pragma once
#include "common.cuh"

__device__ __forceinline__ char* seg_addr(char* base, int layout, i64 nblk, i64 seg, int nseg, u32 b, int s) {
  return layout == 0 ? base + ((i64)s * nblk + b) * seg : base + ((i64)b * nseg + s) * seg;
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// CTA-wide copy of n16 16-byte words: 8 independent 128-bit loads in flight per thread.
__device__ __forceinline__ void cta_copy16(const uint4* __restrict__ src, uint4* __restrict__ dst, i64 n16) {
  const int T = blockDim.x;
  i64 i = threadIdx.x;
  for (; i + 7 * (i64)T < n16; i += 8 * (i64)T) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ld_stream(src + i + k * T);
#pragma unroll
    for (int k = 0; k < 8; ++k) st_stream(dst + i + k * T, v[k]);
  }
  for (; i < n16; i += T) st_stream(dst + i, ld_stream(src + i));
}

// ---- TMA bulk copy (TA_F_COPY_BULK): one elected thread moves the segment through a
// 32 KiB shared-memory buffer with cp.async.bulk (global -> smem, mbarrier complete_tx)
// and cp.async.bulk (smem -> global, bulk_group).  Large transfers instead of 16-B
// accesses; the other threads of the CTA are free for fills.
#define BULK_CHUNK 32768u

__device__ __forceinline__ void mbar_init(u64* mbar, u32 count) {
  u32 a = (u32)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(u64* mbar, u32 phase) {
  u32 a = (u32)__cvta_generic_to_shared(mbar);
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" :: "r"(a), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem, const void* src, u32 bytes, u64* mbar) {
  u32 s = (u32)__cvta_generic_to_shared(smem), m = (u32)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(m), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(s), "l"(src), "r"(bytes), "r"(m) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* smem, u32 bytes) {
  u32 s = (u32)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst), "r"(s), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct BulkCtx {                 // per-CTA state, used by threadIdx.x == 0 only
  char* smem;
  u64* mbar;
  u32 phase;
};

// Copy `bytes` (multiple of 16) from src to dst through smem.  `before_store(k)` runs
// after chunk k has landed in smem and before it is written (used to wait for the
// destination block's eviction).  Thread 0 only; returns with the smem reusable.
template <typename BeforeStore>
__device__ __forceinline__ void bulk_copy(BulkCtx& b, const char* src, char* dst, u32 bytes, BeforeStore before) {
  for (u32 off = 0; off < bytes; off += BULK_CHUNK) {
    const u32 n = min(BULK_CHUNK, bytes - off);
    bulk_load(b.smem, src + off, n, b.mbar);
    mbar_wait(b.mbar, b.phase);
    b.phase ^= 1;
    before(off);
    bulk_store(dst + off, b.smem, n);
    bulk_wait_read();
  }
}

// Per-kernel setup of the bulk path (dynamic smem of BULK_CHUNK bytes when bulk is on).
__device__ __forceinline__ BulkCtx bulk_begin(const Dev& d) {
  extern __shared__ __align__(128) char dyn_smem[];
  __shared__ u64 mbar;
  BulkCtx b{dyn_smem, &mbar, 0};
  if ((d.flags & TA_F_COPY_BULK) && threadIdx.x == 0) mbar_init(&mbar, 1);
  __syncthreads();
  return b;
}
// Copy one segment (CTA-wide call): TMA bulk by thread 0, or 128-bit loads/stores by all.
__device__ __forceinline__ void seg_copy(const Dev& d, BulkCtx& b, const uint4* src, uint4* dst) {
  if (d.flags & TA_F_COPY_BULK) {
    if (threadIdx.x == 0) bulk_copy(b, (const char*)src, (char*)dst, (u32)d.seg_bytes, [](u32) {});
  } else {
    cta_copy16(src, dst, d.seg_bytes >> 4);
  }
}
// Make a segment's copy complete and visible to the CTA's generic stores (before a tail fill).
__device__ __forceinline__ void seg_copy_fence(const Dev& d) {
  if ((d.flags & TA_F_COPY_BULK) && threadIdx.x == 0) {
    bulk_wait_all();
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncthreads();
}
__device__ __forceinline__ void bulk_end(const Dev& d) {
  if ((d.flags & TA_F_COPY_BULK) && threadIdx.x == 0) bulk_wait_all();
}

// Map a flat item index onto (local replica, entry, segment) given per-replica counts.
__device__ __forceinline__ bool locate(const Dev& d, const u32* cnt, i64 item, int nseg, int* r, u32* e, int* s) {
  for (int q = 0; q < d.n_local; ++q) {
    int rr = d.first_local + q;
    i64 n = (i64)cnt[rr] * nseg;
    if (item < n) { *r = rr; *e = (u32)(item / nseg); *s = (int)(item % nseg); return true; }
    item -= n;
  }
  return false;
}
__device__ __forceinline__ i64 local_items(const Dev& d, const u32* cnt, int nseg) {
  i64 n = 0;
  for (int q = 0; q < d.n_local; ++q) n += (i64)cnt[d.first_local + q] * nseg;
  return n;
}

// D2H evictions: HBM block of replica r -> slot of r's pinned host tier (PCIe).
__global__ void __launch_bounds__(256) k_copy_evict(Dev d) {
  const int nseg = 2 * d.nL;
  const i64 items = local_items(d, d.evd_cnt, nseg);
  BulkCtx bk = bulk_begin(d);
  for (i64 it = blockIdx.x; it < items; it += gridDim.x) {
    int r, s; u32 e;
    locate(d, d.evd_cnt, it, nseg, &r, &e, &s);
    EvDesc x = d.evd[(size_t)r * d.NB + e];
    const uint4* src = (const uint4*)seg_addr(d.hbm[r], d.layout, d.NB, d.seg_bytes, nseg, x.src, s);
    uint4* dst = (uint4*)seg_addr(d.host[r], d.layout, d.NH, d.seg_bytes, nseg, x.dst, s);
    seg_copy(d, bk, src, dst);
  }
  bulk_end(d);
}

// Fetches into the local replicas' HBM: P2P from a peer (or co-located) replica's
// HBM over NVLink, or H2D from a host tier.
__global__ void __launch_bounds__(256) k_copy_fetch(Dev d) {
  const int nseg = 2 * d.nL;
  const i64 items = local_items(d, d.fed_cnt, nseg);
  BulkCtx bk = bulk_begin(d);
  for (i64 it = blockIdx.x; it < items; it += gridDim.x) {
    int r, s; u32 e;
    locate(d, d.fed_cnt, it, nseg, &r, &e, &s);
    FeDesc x = d.fed[(size_t)r * d.NB + e];
    if (x.kind != MV_P2P && x.kind != MV_H2D) continue;   // fills: k_fill
    const char* sbase = x.kind == MV_P2P ? d.hbm[x.src_r] : d.host[x.src_r];
    i64 snb = x.kind == MV_P2P ? d.NB : d.NH;
    if (sbase == nullptr) continue;      // executed by the source's owner (multi-process push)
    const uint4* src = (const uint4*)seg_addr((char*)sbase, d.layout, snb, d.seg_bytes, nseg, x.src, s);
    uint4* dst = (uint4*)seg_addr(d.hbm[r], d.layout, d.NB, d.seg_bytes, nseg, x.dst, s);
    seg_copy(d, bk, src, dst);
  }
  bulk_end(d);
}

// Multi-process push: H2D fetches whose source is THIS process's host tier but whose
// destination replica lives in another process: read the local pinned tier, store
// into the peer's HBM pool over NVLink (mapped with CUDA IPC).
__global__ void __launch_bounds__(256) k_copy_push(Dev d) {
  if (!d.multi) return;
  const int nseg = 2 * d.nL;
  BulkCtx bk = bulk_begin(d);
  for (int r = 0; r < d.R; ++r) {
    if (r >= d.first_local && r < d.first_local + d.n_local) continue;
    const u32 n = d.fed_cnt[r];
    const FeDesc* fe = d.fed + (size_t)r * d.NB;
    for (i64 it = blockIdx.x; it < (i64)n * nseg; it += gridDim.x) {
      FeDesc x = fe[it / nseg];
      const int s = (int)(it % nseg);
      if (x.kind != MV_H2D || d.host[x.src_r] == nullptr || d.hbm[r] == nullptr) continue;
      const uint4* src = (const uint4*)seg_addr(d.host[x.src_r], d.layout, d.NH, d.seg_bytes, nseg, x.src, s);
      uint4* dst = (uint4*)seg_addr(d.hbm[r], d.layout, d.NB, d.seg_bytes, nseg, x.dst, s);
      seg_copy(d, bk, src, dst);
    }
  }
  bulk_end(d);
  __threadfence_system();                // peer stores visible before the barrier flag
}

// Cross-process barrier through IPC-mapped mailboxes (one replica per GPU): lane i
// publishes this rank's epoch into peer i's mailbox, then waits for peer i's epoch
// in its own.  Bounded spin: a dead peer poisons the context instead of hanging.
// A/B aid (env TA_GAP_PROBES at init, timing mode): a one-warp kernel between two tick
// kernels stamps its first instruction into pst[3*32 + 28 + i].
__global__ void k_probe(Dev d, int i) {
  const ull t = gtimer();
  if (threadIdx.x == 0) d.pst[3 * 32 + 28 + i] = t;
}

// Timing mode only: reset the kernel spans (kspan_begin / kspan_end) at the head of a tick.
__global__ void k_span_reset(Dev d) {
  if (threadIdx.x < KS_N) {
    d.pst[3 * 32 + 16 + 2 * threadIdx.x] = ~0ull;
    d.pst[3 * 32 + 17 + 2 * threadIdx.x] = 0;
  }
}

__global__ void k_barrier(Dev d) {
  if (!d.multi) return;
  // The barriers order copies between processes (a push into a peer's freshly evicted
  // block, a pull from a peer's block that it frees at step 7).  A tick whose plan --
  // the same on every rank: the control plane is replicated -- moves nothing between
  // processes needs neither, so every rank skips both (epochs stay in step).
  if (d.ctr->t_cross == 0) return;
  jitter(d, 5u);                        // TA_F_JITTER: ranks reach the barrier out of step
  __shared__ ull e;
  if (threadIdx.x == 0) e = ++(*d.epoch);
  __syncthreads();
  const int i = threadIdx.x;
  if (i >= d.R || i == d.rank || !((d.healthy >> i) & 1u)) return;   // failed replicas are not waited for
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(d.mbox_peer[i] + d.rank), "l"(e) : "memory");
  ull v = 0;
  for (long long spin = 0; spin < (1ll << 26); ++spin) {   // ~15 s worst case
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(d.mbox + i) : "memory");
    if (v >= e) return;
    if (spin > 64) __nanosleep(200);
  }
  d.ctr->err = TA_E_PEER;
}

// Two-finger compaction moves inside one replica's HBM pool (D2D).  A tick that did
// not run (rejected API batch, peer failure) planned no compaction: the descriptor list
// still holds the previous tick's moves, whose destinations the engine may have written
// since, so nothing is copied.
__device__ __forceinline__ void copy_compact(const Dev& d) {
  if (d.ctr->err != TA_OK) return;
  const int nseg = 2 * d.nL;
  const i64 items = local_items(d, d.cpd_cnt, nseg);
  BulkCtx bk = bulk_begin(d);
  for (i64 it = blockIdx.x; it < items; it += gridDim.x) {
    int r, s; u32 e;
    locate(d, d.cpd_cnt, it, nseg, &r, &e, &s);
    CpDesc x = d.cpd[(size_t)r * (d.NB / 2 + 1) + e];
    const uint4* src = (const uint4*)seg_addr(d.hbm[r], d.layout, d.NB, d.seg_bytes, nseg, x.src, s);
    uint4* dst = (uint4*)seg_addr(d.hbm[r], d.layout, d.NB, d.seg_bytes, nseg, x.dst, s);
    seg_copy(d, bk, src, dst);
  }
  bulk_end(d);
}
__global__ void __launch_bounds__(256) k_copy_compact(Dev d) {
  const ull t_in = gtimer();   // the CTA's first instruction (kernel span, timing mode)
  kspan_begin(d, KS_COMPACT, t_in);
  copy_compact(d);
  kspan_end(d, KS_COMPACT);
}

// ta_move_blocks: n whole blocks from one pool to another, block-list driven.
__global__ void __launch_bounds__(256) k_move(Dev d, const char* sbase, i64 snb, char* dbase, i64 dnb,
                                              const u32* __restrict__ src, const u32* __restrict__ dst, int n) {
  const int nseg = 2 * d.nL;
  const i64 items = (i64)n * nseg;
  BulkCtx bk = bulk_begin(d);
  for (i64 it = blockIdx.x; it < items; it += gridDim.x) {
    u32 e = (u32)(it / nseg);
    int s = (int)(it % nseg);
    const uint4* sp = (const uint4*)seg_addr((char*)sbase, d.layout, snb, d.seg_bytes, nseg, src[e], s);
    uint4* dp = (uint4*)seg_addr(dbase, d.layout, dnb, d.seg_bytes, nseg, dst[e], s);
    seg_copy(d, bk, sp, dp);
  }
  bulk_end(d);
}

// ---- KV content closed form: word(uid, t, l, kv, h, w) =
// splitmix64((uid << 40) + (((t*L + l)*2 + kv)*Hkv + h)*(D/4) + w)
__device__ __forceinline__ ull splitmix64(ull x) {
  ull z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Engine stand-in: write the content of tokens [t0, t1) of logical block j of program
// uid into segment s (= 2l + kv) of HBM block idx of replica r (CTA-wide).
__device__ __forceinline__ void fill_segment(const Dev& d, int r, u32 idx, int s, u32 uid, u32 j, u32 t0,
                                             u32 t1) {
  const int nseg = 2 * d.nL;
  const u32 wtok = (u32)(d.Hkv * d.D / 4);            // 8-byte words per (token, layer, kv)
  ull* seg = (ull*)seg_addr(d.hbm[r], d.layout, d.NB, d.seg_bytes, nseg, idx, s);
  const u32 l = (u32)s >> 1, kv = (u32)s & 1;
  const u32 slot0 = t0 - j * (u32)d.bt;
  const u32 nw = (t1 - t0) * wtok;
  const ull ubase = (ull)uid << 40;
  for (u32 q = threadIdx.x * 2; q < nw; q += blockDim.x * 2) {
    u32 t = t0 + q / wtok, rem = q % wtok;            // wtok is even: q, q+1 share t
    ull i = (((ull)t * d.nL + l) * 2 + kv) * wtok + rem;
    ull a = splitmix64(ubase + i), b = splitmix64(ubase + i + 1);
    uint4 v = make_uint4((u32)a, (u32)(a >> 32), (u32)b, (u32)(b >> 32));
    *reinterpret_cast<uint4*>(seg + (size_t)slot0 * wtok + q) = v;
  }
}

// Fills of new / recomputed blocks, then the new-token tails of copied blocks.
__global__ void __launch_bounds__(256) k_fill(Dev d) {
  const int nseg = 2 * d.nL;
  const i64 n1 = local_items(d, d.fld_cnt, nseg);
  const i64 items = n1 + local_items(d, d.fed_cnt, nseg);
  for (i64 it = blockIdx.x; it < items; it += gridDim.x) {
    int r, s; u32 e;
    if (it < n1) {
      locate(d, d.fld_cnt, it, nseg, &r, &e, &s);
      FillDesc x = d.fld[(size_t)r * d.NB + e];
      fill_segment(d, r, x.idx, s, x.uid, x.j, x.t0, x.t1);
    } else {
      locate(d, d.fed_cnt, it - n1, nseg, &r, &e, &s);
      FeDesc x = d.fed[(size_t)r * d.NB + e];
      if (x.t0 < x.t1) fill_segment(d, r, x.dst, s, x.uid, x.j, x.t0, x.t1);
    }
  }
}

// Wait until every segment of the destination block has been read by its eviction.
// The grid is co-resident (cooperative launch), so a local wait always ends; a wait
// over NVLink on a peer's flag is bounded (~10 s): a dead peer sets TA_E_PEER, and the
// CTA skips the copy (returns false) instead of hanging.
__device__ __forceinline__ bool wait_evicted(const Dev& d, const u32* flag, bool sys) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    u32 v;
    long long spin = 0;
    int ok = 1;
    do {
      if (sys) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      if (v) {
        __nanosleep(64);
        if (++spin > (1ll << 27)) { d.ctr->err = TA_E_PEER; ok = 0; break; }
      }
    } while (v);
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// The movement of one tick in ONE kernel (step 6): even CTAs run the D2H evictions,
// odd CTAs the fetches into this process's replicas (P2P pulls over NVLink, H2D from
// its own host tiers, each followed by its new-token tail), then -- one process per
// GPU -- the pushes of this process's host tier into peers' pools over NVLink, then
// the fills of new / recomputed blocks.  D2H and H2D therefore share the
// full-duplex host link instead of running back to back.  A destination block that
// was evicted in this tick is written only after all its segments were read: the
// evictor (the block's owner) decrements its flag per segment (release), writers
// wait for 0 (acquire; over NVLink for pushes).  Evicting CTAs never wait, and the
// grid is fully resident, so the waits always terminate.  Multi-process: fills and
// new-token tails run in k_fill after the closing barrier (a pushed block's tail is
// written by its destination process).
__device__ __forceinline__ void move_fused(const Dev& d) {
  const int nseg = 2 * d.nL;
  const int role = blockIdx.x & 1;
  const int G = gridDim.x >> 1;
  const int me = blockIdx.x >> 1;
  // rejected API batch, or a peer failure in any mode: the lists are not this tick's
  if (d.ctr->err == TA_E_PEER || (d.api_mode && d.ctr->err != TA_OK)) return;
  i64 n_push = 0;
  if (d.multi)
    for (int r = 0; r < d.R; ++r)
      if (r != d.rank) n_push += (i64)d.fed_cnt[r] * nseg;
  {   // CTAs without work for their role leave before any setup (ticks that move little)
    const i64 fl = d.multi ? 0 : local_items(d, d.fld_cnt, nseg);
    const i64 mine = role == 0 ? local_items(d, d.evd_cnt, nseg)
                               : max(local_items(d, d.fed_cnt, nseg) + n_push, fl);
    if (me >= mine) return;
  }
  BulkCtx bk = bulk_begin(d);
  if (role == 0) {
    const i64 items = local_items(d, d.evd_cnt, nseg);
    for (i64 it = me; it < items; it += G) {
      int r, s; u32 e;
      locate(d, d.evd_cnt, it, nseg, &r, &e, &s);
      EvDesc x = d.evd[(size_t)r * d.NB + e];
      const uint4* src = (const uint4*)seg_addr(d.hbm[r], d.layout, d.NB, d.seg_bytes, nseg, x.src, s);
      uint4* dst = (uint4*)seg_addr(d.host[r], d.layout, d.NH, d.seg_bytes, nseg, x.dst, s);
      seg_copy(d, bk, src, dst);
      __syncthreads();                              // every load of the segment has returned
      if (threadIdx.x == 0) {
        __threadfence_system();
        atomicSub(&evp_of(d, r)[x.src], 1u);
      }
    }
    bulk_end(d);
    return;
  }
  const i64 nf = local_items(d, d.fed_cnt, nseg);
  for (i64 it = me; it < nf + n_push; it += G) {
    int r, s; u32 e;
    bool push = it >= nf;
    if (!push) {
      locate(d, d.fed_cnt, it, nseg, &r, &e, &s);
    } else {                                        // remote replicas' fetches, in replica order
      i64 q = it - nf;
      for (r = 0; r < d.R; ++r) {
        if (r == d.rank) continue;
        const i64 n = (i64)d.fed_cnt[r] * nseg;
        if (q < n) break;
        q -= n;
      }
      e = (u32)(q / nseg);
      s = (int)(q % nseg);
    }
    FeDesc x = d.fed[(size_t)r * d.NB + e];
    if (x.kind == MV_NONE) continue;
    if (push && (x.kind != MV_H2D || d.host[x.src_r] == nullptr)) continue;   // not from this tier
    if (push && !((d.healthy >> r) & 1u)) continue;   // a failed replica receives nothing
    if (x.kind == MV_FILL) {                        // new / recomputed tokens (single process)
      if (d.multi) continue;
      if (!wait_evicted(d, &evp_of(d, r)[x.dst], false)) continue;
      fill_segment(d, r, x.dst, s, x.uid, x.j, x.t0, x.t1);
      continue;
    }
    const char* sbase = x.kind == MV_P2P ? d.hbm[x.src_r] : d.host[x.src_r];
    if (sbase == nullptr) continue;                 // H2D from a peer's tier: pushed by its owner
    if (!wait_evicted(d, &evp_of(d, r)[x.dst], push)) continue;
    const i64 snb = x.kind == MV_P2P ? d.NB : d.NH;
    const uint4* src = (const uint4*)seg_addr((char*)sbase, d.layout, snb, d.seg_bytes, nseg, x.src, s);
    uint4* dst = (uint4*)seg_addr(d.hbm[r], d.layout, d.NB, d.seg_bytes, nseg, x.dst, s);
    seg_copy(d, bk, src, dst);
    if (x.t0 < x.t1 && !d.multi) {
      seg_copy_fence(d);                            // copy done before the tail is overwritten
      fill_segment(d, r, x.dst, s, x.uid, x.j, x.t0, x.t1);
    }
  }
  if (!d.multi) {
    const i64 nl = local_items(d, d.fld_cnt, nseg);
    for (i64 it = me; it < nl; it += G) {
      int r, s; u32 e;
      locate(d, d.fld_cnt, it, nseg, &r, &e, &s);
      FillDesc x = d.fld[(size_t)r * d.NB + e];
      if (!wait_evicted(d, &evp_of(d, r)[x.idx], false)) continue;
      fill_segment(d, r, x.idx, s, x.uid, x.j, x.t0, x.t1);
    }
  }
  bulk_end(d);
  if (d.multi) __threadfence_system();             // pushed bytes visible before the barrier
}
__global__ void __launch_bounds__(256, 4) k_move_fused(Dev d) {
  const ull t_in = gtimer();   // the CTA's first instruction (kernel span, timing mode)
  kspan_begin(d, KS_MOVE, t_in);
  jitter(d, 3u);
  move_fused(d);
  kspan_end(d, KS_MOVE);
}

// Test aid: count words of every owned block (HBM and host tier of the local
// replicas) that differ from the closed form, over valid token slots only.
__global__ void __launch_bounds__(256) k_verify(Dev d, int tier) {
  const int nseg = 2 * d.nL;
  const u32 wtok = (u32)(d.Hkv * d.D / 4);
  const i64 nblk = tier ? d.NH : d.NB;
  const i64 items = (i64)d.n_local * nblk * nseg;
  ull bad = 0, seen = 0;
  for (i64 it = blockIdx.x; it < items; it += gridDim.x) {
    int q = (int)(it / (nblk * nseg));
    i64 rem = it % (nblk * nseg);
    u32 b = (u32)(rem / nseg);
    int s = (int)(rem % nseg);
    int r = d.first_local + q;
    const u32* fw = tier ? d.host_free + (size_t)r * d.NHW : d.hbm_free + (size_t)r * d.NBW;
    if (fw[b >> 5] & (1u << (b & 31))) continue;      // free
    u32 o = tier ? d.owner_host[(size_t)r * d.NH + b] : d.owner_hbm[(size_t)r * d.NB + b];
    u32 j, t0, t1, uid;
    if (!tier && o >= OWNER_PROMPT) {                    // shared prompt k's block j: full
      j = o & 0xFFFFFu;
      t0 = j * (u32)d.bt; t1 = t0 + (u32)d.bt; uid = TA_PROMPT_UID + ((o >> 20) & 0x7Fu);
    } else {
      const u32 p = o / (u32)d.MAXB;
      j = o % (u32)d.MAXB;
      t0 = j * (u32)d.bt; t1 = min(t0 + (u32)d.bt, d.c_kv[p]); uid = d.uid[p];
    }
    if (t1 <= t0) continue;
    char* base = tier ? d.host[r] : d.hbm[r];
    const ull* seg = (const ull*)seg_addr(base, d.layout, nblk, d.seg_bytes, nseg, b, s);
    const u32 l = (u32)s >> 1, kv = (u32)s & 1;
    const ull ubase = (ull)uid << 40;
    const u32 nw = (t1 - t0) * wtok;
    for (u32 w = threadIdx.x; w < nw; w += blockDim.x) {
      u32 t = t0 + w / wtok, rw = w % wtok;
      ull i = (((ull)t * d.nL + l) * 2 + kv) * wtok + rw;
      bad += seg[w] != splitmix64(ubase + i);
      seen += 1;
    }
  }
  bad = warp_sum_u64(bad);
  seen = warp_sum_u64(seen);
  if (lane_id() == 0) {
    if (bad) atomicAdd(&d.verify[0], bad);
    atomicAdd(&d.verify[1], seen);
  }
}
