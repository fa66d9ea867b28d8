// common.cuh — device state layout and CTA-level primitives for libta (sm_100a).
//
// Control plane is replicated: every process holds the program table, block
// tables, bitmaps and owner maps of ALL replicas and computes every decision;
// only the copy kernels are restricted to the replicas whose pools it holds.
// Everything is integer arithmetic with total orders ending in the slot index,
// so results are bit-identical to the CPU oracle.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ta.h"

typedef uint32_t u32;
typedef uint64_t u64;
typedef int64_t i64;
typedef int32_t i32;
typedef uint8_t u8;
typedef int8_t i8;
typedef unsigned long long ull;

#define LOC_NONE 0xFFFFFFFFu
#define LOC_HOST 0x80000000u
#define OWNER_PROMPT TA_OWNER_PROMPT      // owner_hbm of a shared-prompt block: | k << 20 | j (NEXT-3)
#define KP_NONE 0xFFu                     // prefix_id of a program without a shared prompt
#define FULL_MASK 0xFFFFFFFFu
#define CTA 1024          // threads of the single-CTA planner kernels
#define NWARP (CTA / 32)

enum StatIdx {
  ST_TICKS = 0, ST_ARRIVALS, ST_STOPS, ST_PAUSES, ST_RESTORES, ST_OVERSIZED, ST_SHORTFALLS,
  ST_EVICT_BLOCKS, ST_EVICT_TO_HOST, ST_EVICT_DROPPED, ST_FETCH_BLOCKS, ST_P2P, ST_H2D,
  ST_RECOMPUTE, ST_NEW_BLOCKS, ST_COMPACT, ST_STALLS, ST_HIT, ST_PEER, ST_HOST, ST_MISS,
  ST_NEW_TOK, ST_FILL_TOK, ST_IMB_MAX, ST_IMB_LAST,
  ST_BASE_N,                                   // counters before block_bytes in ta_stats_t
  ST_COST_DECODE = ST_BASE_N, ST_COST_PREFILL, ST_COST_RECOMPUTE, ST_COST_UNUSED, ST_COST_CACHING,
  ST_UNUSED_CHECKS, ST_UNUSED_VIOL, ST_OVERSHOOT, ST_OVERSHOOT_MAX, ST_PREFIX_BLOCKS, ST_N
};

// per-request descriptor kinds (step 5.5): copy from a peer's HBM, copy from a host
// tier, write new / recomputed tokens, nothing (fills disabled)
enum MoveKind { MV_NONE = 0, MV_P2P = 2, MV_H2D = 3, MV_FILL = 4 };

struct Ctr {                 // device-resident scalars of the context
  i64 tick;                  // k
  i64 next_arrival;          // lowest UNARRIVED slot (arrivals are a suffix)
  i64 T;                     // time of the current tick (ms)
  i64 now_ms;                // API mode: time passed by the host
  u32 stops;                 // releases this tick
  u32 restore_cnt;           // RESTORE decisions this tick
  u32 n_dec;                 // decisions assembled this tick
  u32 n_arr;                 // arrivals this tick
  i32 err;                   // API-mode event validation status
  i32 n_events;              // API-mode events this tick
  u32 verb_pid;              // single-program materialize (verbs)
  i32 verb_replica;
  i32 verb_ok;
  u32 t_d2h, t_h2d, t_p2p, t_d2d, t_fetch;   // this tick's block moves (telemetry)
  u32 t_cross;               // this tick's copies between processes (P2P, a peer tier's H2D)
  u32 cmin;                  // smallest footprint (blocks) among PAUSED programs after step 4 (~0: none)
  ull ev_err;                // API mode: min over programs of (event index << 8 | code); ~0 = legal
  u32 ev_multi;              // API mode: events of programs with several events in the batch
};

struct EvRes;

struct EvDesc { u32 src; u32 dst; };                     // HBM block -> host slot (replica r)
// P2P / H2D into HBM block dst; tokens [t0, t1) of logical block j of program uid are
// (re)written after the copy when t0 < t1 (new tokens landing in a copied partial block)
struct FeDesc { u32 kind; u32 src_r; u32 src; u32 dst; u32 uid; u32 t0; u32 t1; u32 j; };
struct FillDesc { u32 idx; u32 uid; u32 t0; u32 t1; u32 j; u32 pad; };
struct CpDesc { u32 src; u32 dst; };

struct Dev {
  // ---- configuration ----
  int N, MAXB, MAXBP, R, bt, nL, Hkv, D, layout;
  i64 NB, NH;
  int NBW, NHW;
  i64 dt, unit;
  int rate;
  u32 flags;
  int compact_every;
  int chunk_q, chunk_ms;           // STP ledger: prefill chunk tokens / ms per chunk
  int K;                           // NEXT-3 (A51): shared prompts
  u32 sbk[TA_MAX_PREFIXES];        // blocks of each prompt
  u32 SBM;                         // max over sbk (stride of pblk)
  i64 seg_bytes, block_bytes;
  int first_local, n_local;
  int api_mode;
  u32 nbk, nb_shift;               // coarse-key buckets: nb >> nb_shift < nbk <= 2048
  i64 cap_max[TA_MAX_REPLICAS], cap_min[TA_MAX_REPLICAS];   // 0 while a replica is unhealthy
  u32 healthy;                     // bit r: replica r healthy (BackendState.healthy)
  ull F[64];
  char* hbm[TA_MAX_REPLICAS];      // device-addressable HBM pool per replica (NULL if not here)
  char* host[TA_MAX_REPLICAS];     // device alias of the pinned host tier (local replicas)
  // ---- program table (SoA, N slots) ----
  u32 *uid, *c, *c_kv, *paused_since, *step_count, *turn, *gen_done;
  u8 *status, *phase, *satisfied;
  i8 *placement, *home;
  i64 *acting_since, *tool_return;
  u32* loc;                        // [N][MAXBP]
  // ---- per-tick derived values ----
  u32 *nb, *n_hbm, *n_host, *prefix_hbm, *contrib;
  u8* hcls;                        // [N] where the last history block (entry ceil(c_kv/bt) - 1) is:
                                   //     0 NONE, 1 HBM, 2 host tier (footprint pass; hit accounting)
  u8* released;                    // released during this tick's ingest
  u8* sat_new;                     // 1 + replica that satisfied the program this tick
  u8* dirty;                       // [N] row written since the footprint pass last counted it
                                   //     (every writer of loc sets it; the pass clears it)
  u8* kp;                          // [N] shared prompt of each program (KP_NONE: none)
  u8* t_kp;                        // [N] trace mode: prompt of each slot's program
  u32* pref;                       // [R][K] programs homed on r using prompt k
  u32* pblk;                       // [R][K][SBM] blocks of prompt k on r (valid while pref > 0)
  u32* pfix;                       // [R][NBW] prompt blocks (bit set): never evicted, moved or compacted
  u32* f_x;                        // [R][N] F_r entry: prompt blocks it materializes | prompt << 16
  u32 *pend, *busy;                // [N] synthetic engine (A48): tokens waiting for prefill;
                                   //     ms the last materialize spent (re)prefilling
  u8* evs;                         // [3N] API-mode validation scratch (kept zero)
  u32* evc;                        // [N]  API-mode tentative context lengths
  // ---- trace scripts ----
  int n_slots, n_initial;
  u32 *t_uid, *t_p0, *t_off, *t_g, *t_d, *t_o;
  // ---- replica state (all replicas) ----
  u32 *hbm_free, *host_free;       // [R][NBW], [R][NHW]; bit set = free
  u32 *owner_hbm, *owner_host;     // [R][NB], [R][NH]: pid * MAXB + j
  ull* L;                          // [R]  effective load after the last pause/restore pass
  ull* Lacc;                       // [R]  footprint accumulator of this tick (zeroed by k_pause)
  Ctr* ctr;
  ull* stats;                      // [ST_N]
  // ---- scratch ----
  u64 *ska, *skb;                  // sort keys  [R+1][N]
  u32 *sva, *svb;                  // sort values[R+1][N]
  u32* pause_list;                 // [R][N]
  u32* pause_cnt;                  // [R]
  u32 *restore_pid, *restore_dst;  // [N]
  u32 *f_pid, *f_cum;              // [R][N]  REASONING list per replica, inclusive need prefix
  u32 *f_cnt, *s_cnt;              // [R]
  ta_decision* dec_fs;             // [R][N]  FETCH/STALL record per F entry (kind 0 = none)
  ta_decision* dec_ev;             // [R][N]  EVICT records (victim order)
  u32* ev_cnt;                     // [R]     victims
  u32* e_pid;                      // [R][N]  eviction order (sorted candidates)
  u32* e_cum;                      // [R][N]  inclusive n_hbm prefix in eviction order
  EvDesc* evd; u32* evd_cnt;       // [R][NB]
  u32* evx;                        // [R][NB] evicted HBM block per eviction rank
  EvDesc* evt;                     // [R][NB] evictions in victim order (evd: by block index)
  FeDesc* fed; u32* fed_cnt;       // [R][NB]
  FeDesc* fedt;                    // [R][NB] per-CTA staging of k_plan's descriptors
  FillDesc* fld; u32* fld_cnt;     // [R][NB]
  u32* dfh; u32* dfh_cnt;          // deferred HBM frees  [R][NB]: (replica << 27) | idx
  u32* dfs; u32* dfs_cnt;          // deferred host frees [R][NB]
  CpDesc* cpd; u32* cpd_cnt;       // [R][NB/2+1]
  ta_decision* dec_out;            // host-mapped decision buffer (canonical order)
  u32* dec_out_cnt;                // host-mapped count
  ta_tick_info* tick_info;         // host-mapped telemetry of the last tick
  u32 dec_cap;
  ull* verify;                     // [2] mismatches, checked
  ta_event* events;                // [ev_cap] API-mode event batch
  EvRes* evr;                      // [ev_cap] per-event result (owner event of each program)
  u32* ev_pcnt;                    // [N] events per program in the batch (kept zero between calls)
  u64 *ev_mk, *ev_mk2;             // [ev_cap] (pid << 32 | index) of multi-event programs
  u32 *ev_mv, *ev_mv2;             // [ev_cap] sort values (unused payload)
  u32* t_rep;                      // [3][R] this tick's blocks per replica: d2h into, h2d from, p2p into
  // ---- multi-process data plane (one replica per GPU) ----
  int multi, rank;                 // multi: pools of other replicas live in other processes
  int fused;                       // single-process: evict / fetch / fill in one kernel
  u32* evp;                        // [R][NB] segments of a block still to be evicted this tick
                                   // (multi-process: [NB] of the local replica, in the IPC-shared
                                   // mailbox allocation)
  u32* evp_peer[TA_MAX_REPLICAS];  // multi-process: peers' eviction flags (CUDA IPC)
  ull* mbox;                       // [TA_MAX_REPLICAS] this rank's barrier mailbox (epochs)
  ull* mbox_peer[TA_MAX_REPLICAS]; // peers' mailboxes (CUDA IPC)
  ull* epoch;                      // barrier epoch counter (device)
  ull* pst;                        // [8][32] in-kernel phase stamps, globaltimer ns (TA_F_TIMING; developer aid)
  // ---- candidate sets built by the footprint pass as slot bitmaps (one word per 32
  // slots, written whole by the CTA that owns those slots: no atomics), so the planner
  // kernels never scan all N slots except the restore gather; consumers turn a bitmap
  // into a slot-ordered list (cta_bits_to_list)
  int NW;                          // words per bitmap: ceil(N / 32)
  u32* act_bits;                   // [R][NW]: REASONING or ACTING placed on r
  u32* reas_bits;                  // [R][NW]: REASONING placed on r (F_r before steps 3-4)
  u32* ec_bits;                    // [R][NW]: home == r with private HBM blocks (eviction candidates)
  u32 *act_list, *ec_list;         // [R][N]: list scratch when a list does not fit shared memory
  u32* rhist;                      // [2 * nbk] restore-bucket histogram of PAUSED slots
  u32* rb;                         // [N] restore bucket of a PAUSED slot, else 0xFFFFFFFF
  ull* gsync;                      // [2] grid-barrier counters of k_decide / k_close (monotone)
  ull* dbg;                        // [DBG_N] size-branch counters (ta_debug_counters)
};

// Size-branch counters: how often each large-size / fallback code path ran (test
// evidence that parity runs reach them; ta_debug_counters).
enum DbgIdx {
  DBG_RADIX = 0,        // CTA sort of n > sort limit: global-memory radix sort
  DBG_BITONIC,          // register/shared bitonic network (rank limit < n <= sort limit)
  DBG_RANK,             // rank sort (n <= rank limit)
  DBG_LIST_GLOBAL,      // a candidate bitmap's slot list did not fit shared memory (global list)
  DBG_F_GLOBAL,         // k_plan need prefix read from global memory (nF > staging limit)
  DBG_E_GLOBAL,         // k_plan eviction prefix read from global memory (ne > staging limit)
  DBG_V_GLOBAL,         // k_plan victims read from global memory (nv > victim staging limit)
  DBG_FST_GLOBAL,       // k_plan request loop reads per-program values from global (m > FST limit)
  DBG_RESTORE_CHUNKS,   // restore pass chunks after the first
  DBG_EVICT_TICKS,      // k_plan replica-ticks with X > 0
  DBG_ROWS_COUNTED,     // tick footprint pass: block-table rows counted (written since the last pass)
  DBG_ROW_ENTRIES,      // ... and their entries read (the rest of the rows are clean, not read)
  DBG_N = 16
};
__device__ __forceinline__ void dbg_hit(const Dev& d, int i) {
  if (threadIdx.x == 0) atomicAdd(&d.dbg[i], 1ull);
}
// Per-context option flags read by the tick kernels.  TA_PROD_VARIANT (developer A/B
// build) compiles the measurement / baseline / test options out: timing stamps,
// PinnedRouting, RequestAware, small paths.
#ifdef TA_PROD_VARIANT
#define TA_FLAG(d, f) ((((f) & (TA_F_TIMING | TA_F_PINNED_ROUTING | TA_F_REQUEST_AWARE | TA_F_SMALL_PATHS | \
                               TA_F_JITTER | TA_F_FULL_SCAN)) == 0) && \
                       (((d).flags & (f)) != 0))
#else
#define TA_FLAG(d, f) (((d).flags & (f)) != 0)
#endif

// Size thresholds of the shared-memory fast paths.  TA_F_SMALL_PATHS (test aid) lowers
// them so that toy-sized runs take the branches of full-size runs.
__device__ __forceinline__ bool small_paths(const Dev& d) { return TA_FLAG(d, TA_F_SMALL_PATHS); }

// Barrier across the CTAs of a cooperative launch (all co-resident).  Counter k is
// used by one kernel only and grows by gridDim.x per barrier, so arrival t waits for
// the next multiple of gridDim.x.  One CTA: just a CTA barrier.
// TA_F_JITTER (test aid): thread 0 of the CTA sleeps a pseudo-random 0-20 us (a hash of
// the CTA, the site and the tick), then the CTA waits for it.  Called where every thread
// of the CTA is present (kernel entry, right after a grid or cluster barrier).
__device__ __forceinline__ void jitter(const Dev& d, u32 site) {
  if (TA_FLAG(d, TA_F_JITTER)) {
    if (threadIdx.x == 0) {
      u32 h = (blockIdx.x + 1u) * 0x9E3779B1u ^ site * 0x85EBCA77u ^ (u32)d.ctr->tick * 0xC2B2AE3Du;
      h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12;
      const u32 ns = h % 20000u;
      for (u32 t = 0; t < ns; t += 1000u) __nanosleep(1000u);
    }
    __syncthreads();
  }
}
__device__ __forceinline__ void grid_sync(const Dev& d, int k) {
  __syncthreads();
  if (gridDim.x > 1) {
    if (threadIdx.x == 0) {
      __threadfence();
      ull* c = d.gsync + k;
      const ull t = atomicAdd(c, 1ull);
      const ull target = (t / gridDim.x + 1) * gridDim.x;
      ull v;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(c) : "memory");
      } while (v < target);
      __threadfence();
    }
    __syncthreads();
  }
  jitter(d, 100u + (u32)k);
}

// STP staircase of a chunked prefill of n tokens over a resident base (
// SPEC.md recompute_cost_of): sum_{i=1}^{ceil(n/q)} (base + min(i*q, n)), in closed form.
__device__ __forceinline__ ull stp_stair(ull n, ull q, ull base) {
  const ull m = (n + q - 1) / q, k = n / q;
  return m * base + q * k * (k + 1) / 2 + (m > k ? n : 0);
}

// warp sum of a u64 (all lanes)
__device__ __forceinline__ ull warp_sum_ull(ull v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}

// Eviction flags of replica r's HBM blocks (the owner's copy in multi-process mode).
__device__ __forceinline__ u32* evp_of(const Dev& d, int r) {
  if (!d.multi) return d.evp + (size_t)r * d.NB;
  return r == d.rank ? d.evp : d.evp_peer[r];
}
// Only the process that will read an evicted block sets its flag.
__device__ __forceinline__ bool evp_owner(const Dev& d, int r) { return d.fused && (!d.multi || r == d.rank); }

// Phase stamp: SM clock of thread 0 of CTA 0 at a phase boundary of a planner kernel
// (kernel slot kk: 0 pause, 1 restore, 2 plan, 3 other).  Only with TA_F_TIMING.
__device__ __forceinline__ ull gtimer() {
  ull t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PSTAMP(kk, i)                                                              \
  do {                                                                             \
    if (TA_FLAG(d, TA_F_TIMING) && blockIdx.x == 0 && threadIdx.x == 0)            \
      d.pst[(kk) * 32 + (i)] = gtimer();                                           \
  } while (0)
// the same from thread 0 of block `b` into kernel slot kk (cluster ranks of k_plan)
#define PSTAMP_B(kk, b, i)                                                         \
  do {                                                                             \
    if (TA_FLAG(d, TA_F_TIMING) && blockIdx.x == (b) && threadIdx.x == 0)          \
      d.pst[(kk) * 32 + (i)] = gtimer();                                           \
  } while (0)

// Kernel span (TA_F_TIMING only): the earliest CTA start and the latest exit of any
// warp, as globaltimer ns in pst[3*32 + 16 + 2k] / [.. + 1] (reset to ~0 / 0 at
// the head of each tick by k_span_reset).  The kernel wrappers call kspan_begin / the
// body / kspan_end.  k: 0 front, 1 pause+restore, 2 plan, 3 movement, 4 close,
// 5 compaction.
enum { KS_FRONT = 0, KS_PR = 1, KS_PLAN = 2, KS_MOVE = 3, KS_CLOSE = 4, KS_COMPACT = 5, KS_N = 6 };
__device__ __forceinline__ void kspan_begin(const Dev& d, int k, ull t_in) {
  if (TA_FLAG(d, TA_F_TIMING) && threadIdx.x == 0) atomicMin(d.pst + 3 * 32 + 16 + 2 * k, t_in);
}
__device__ __forceinline__ void kspan_end(const Dev& d, int k) {
  if (TA_FLAG(d, TA_F_TIMING) && (threadIdx.x & 31) == 0) atomicMax(d.pst + 3 * 32 + 17 + 2 * k, gtimer());
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ u32 ceil_div_u32(u32 a, u32 b) { return (a + b - 1) / b; }
// blocks of a program's shared prompt (0 without one)
__device__ __forceinline__ u32 sb_of(const Dev& d, u8 k) { return k == KP_NONE ? 0u : d.sbk[k]; }
// Free the blocks of prompt k on replica r (its last user left; A51).
__device__ __forceinline__ void prompt_free(const Dev& d, int r, u32 k, u32 lane, u32 nl) {
  const u32* blk = d.pblk + ((size_t)r * d.K + k) * d.SBM;
  for (u32 j = lane; j < d.sbk[k]; j += nl) {
    const u32 b = blk[j];
    atomicAnd(&d.pfix[(size_t)r * d.NBW + (b >> 5)], ~(1u << (b & 31)));
    atomicOr(&d.hbm_free[(size_t)r * d.NBW + (b >> 5)], 1u << (b & 31));
  }
}
__device__ __forceinline__ bool is_hbm(u32 e) { return e != LOC_NONE && !(e & LOC_HOST); }
__device__ __forceinline__ bool is_host(u32 e) { return e != LOC_NONE && (e & LOC_HOST); }
__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ u32 lanemask_lt() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Eq. 7 contribution in blocks: nb for tau=R, floor(nb * F[k] / 2^32) for tau=A (readings A4, A5).
__device__ __forceinline__ u32 contrib_of(const Dev& d, u32 nbv, u8 ph, i64 acting_since, i64 T) {
  if (ph == TA_PHASE_R) return nbv;
  i64 el = T - acting_since;
  i64 k = el < 0 ? 0 : el / d.unit;
  if (k > 63) k = 63;
  return (u32)(((ull)nbv * d.F[k]) >> 32);
}

// Closed-loop arrivals of this tick (trace mode): n_initial at tick 0, then one per
// release, taking the lowest UNARRIVED slots (reading A12).
__device__ __forceinline__ i64 trace_arrivals(const Dev& d) {
  i64 n = (d.ctr->tick == 0 ? (i64)d.n_initial : 0) + (i64)d.ctr->stops;
  i64 room = (i64)d.n_slots - d.ctr->next_arrival;
  return n < room ? n : room;
}

// Coarse restore bucket (monotone in the S_restore key): tau = R first, then nb.
__device__ __forceinline__ u32 restore_bucket(const Dev& d, u8 ph, u32 nbv) {
  if TA_FLAG(d, TA_F_REQUEST_AWARE) return 0;        // FCFS key: one bucket
  return (u32)(ph == TA_PHASE_A) * d.nbk + (nbv >> d.nb_shift);
}

// S_restore order (reading A8): R first, nb up, paused_since up; ties by slot
// via sort stability on slot-ordered input.
__device__ __forceinline__ u64 restore_key(u8 ph, u32 nbv, u32 ps) {
  return ((u64)(ph == TA_PHASE_A) << 63) | ((u64)nbv << 32) | (u64)ps;
}
// S_pause order (reading A7): A first, nb up, acting_since DOWN; ties by slot.
#define AS_MAX ((1ull << 40) - 1)
__device__ __forceinline__ u64 pause_key(u8 ph, u32 nbv, i64 as) {
  if (ph == TA_PHASE_A) return ((u64)nbv << 40) | (AS_MAX - (u64)as);
  return (1ull << 63) | ((u64)nbv << 40);
}

// ------------------------------------------------------------------ warp / CTA scans
__device__ __forceinline__ u32 warp_incl_scan(u32 v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 t = __shfl_up_sync(FULL_MASK, v, o);
    if (lane_id() >= (u32)o) v += t;
  }
  return v;
}
__device__ __forceinline__ ull warp_sum_u64(ull v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}

// Exclusive scan of one u32 per thread across the CTA (blockDim.x == CTA).
// s_tmp: >= NWARP+1 u32 of shared memory.  Returns exclusive prefix; *total = sum.
__device__ u32 cta_excl_scan(u32 v, u32* s_tmp, u32* total) {
  u32 inc = warp_incl_scan(v);
  int w = threadIdx.x >> 5;
  if (lane_id() == 31) s_tmp[w] = inc;
  __syncthreads();
  if (w == 0) {
    u32 x = lane_id() < NWARP ? s_tmp[lane_id()] : 0;
    u32 xi = warp_incl_scan(x);
    if (lane_id() < NWARP) s_tmp[lane_id()] = xi - x;
    if (lane_id() == NWARP - 1) s_tmp[NWARP] = xi;
  }
  __syncthreads();
  u32 r = s_tmp[w] + inc - v;
  *total = s_tmp[NWARP];
  __syncthreads();
  return r;
}

template <typename T, typename Op>
__device__ T cta_reduce(T v, T* s_tmp, Op op, T ident) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(FULL_MASK, v, o));
  int w = threadIdx.x >> 5;
  if (lane_id() == 0) s_tmp[w] = v;
  __syncthreads();
  if (w == 0) {
    T x = lane_id() < NWARP ? s_tmp[lane_id()] : ident;
#pragma unroll
    for (int o = 16; o; o >>= 1) x = op(x, __shfl_xor_sync(FULL_MASK, x, o));
    if (lane_id() == 0) s_tmp[0] = x;
  }
  __syncthreads();
  T r = s_tmp[0];
  __syncthreads();
  return r;
}

// Ordered stream compaction over [0, n): every thread owns a contiguous chunk, so
// emitted items keep slot order.  pred(i) -> bool; emit(pos, i).  Returns count.
template <typename Pred, typename Emit>
__device__ u32 cta_ordered_gather(int n, u32* s_tmp, Pred pred, Emit emit) {
  int chunk = (n + CTA - 1) / CTA;
  int lo = threadIdx.x * chunk, hi = min(n, lo + chunk);
  u32 cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += pred(i) ? 1u : 0u;
  u32 total;
  u32 pos = cta_excl_scan(cnt, s_tmp, &total);
  for (int i = lo; i < hi; ++i)
    if (pred(i)) emit(pos++, i);
  __syncthreads();
  return total;
}

// Ordered stream compaction over [0, n) with coalesced reads: warp w owns a contiguous
// range of indices and its lanes take consecutive ones (ballot counts per warp, a scan
// over the warps, then the emit pass re-evaluates pred).  Items keep index order.
// emit(pos, i, total) -- the total is known before the first emit.
template <typename Pred, typename Emit>
__device__ u32 cta_ordered_gather_w(int n, u32* s_tmp, Pred pred, Emit emit) {
  const int w = threadIdx.x >> 5, lane = (int)lane_id();
  const int per = (((n + NWARP - 1) / NWARP) + 31) & ~31;
  const int lo = w * per, hi = min(n, lo + per);
  // up to 64 chunks of 32 slots per warp (n <= 64 * 32 * NWARP): the predicate bits of
  // the counting pass are kept (bit c of tb: this lane's slot in chunk c), so the emit
  // pass reloads nothing and issues four chunks' emits back to back
  const bool keep = per <= 64 * 32;
  u32 cnt = 0;
  u64 tb = 0;
  for (int b = lo; b < hi; b += 128) {            // four independent loads per lane in flight
    bool t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { const int i = b + 32 * k + lane; t[k] = i < hi && pred(i); }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cnt += __popc(__ballot_sync(FULL_MASK, t[k]));
      if (keep && t[k]) tb |= 1ull << (((b - lo) >> 5) + k);
    }
  }
  if (lane == 0) s_tmp[w] = cnt;
  __syncthreads();
  if (w == 0) {
    const u32 x = lane < NWARP ? s_tmp[lane] : 0u;
    const u32 xi = warp_incl_scan(x);
    if (lane < NWARP) s_tmp[lane] = xi - x;
    if (lane == NWARP - 1) s_tmp[NWARP] = xi;
  }
  __syncthreads();
  u32 pos = s_tmp[w];
  const u32 total = s_tmp[NWARP];
  if (keep) {
    for (int b = lo; b < hi; b += 128) {
      u32 m[4], at[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        m[k] = __ballot_sync(FULL_MASK, (u32)(tb >> (((b - lo) >> 5) + k)) & 1u);
        at[k] = pos + __popc(m[k] & lanemask_lt());
        pos += __popc(m[k]);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((m[k] >> lane) & 1u) emit(at[k], b + 32 * k + lane, total);
    }
  } else {
    for (int b = lo; b < hi; b += 32) {
      const int i = b + lane;
      const bool t = i < hi && pred(i);
      const u32 m = __ballot_sync(FULL_MASK, t);
      if (t) emit(pos + __popc(m & lanemask_lt()), i, total);
      pos += __popc(m);
    }
  }
  __syncthreads();
  return total;
}

// In-place inclusive scan of a global u32 array a[0..n) by one CTA.
__device__ void cta_incl_scan_array(u32* a, int n, u32* s_tmp) {
  int chunk = (n + CTA - 1) / CTA;
  int lo = threadIdx.x * chunk, hi = min(n, lo + chunk);
  u32 s = 0;
  for (int i = lo; i < hi; ++i) s += a[i];
  u32 total;
  u32 run = cta_excl_scan(s, s_tmp, &total);
  for (int i = lo; i < hi; ++i) { run += a[i]; a[i] = run; }
  __syncthreads();
}

// First index i in [0, n) with a[i] > x for a non-decreasing array (n if none).
__device__ __forceinline__ int upper_bound_u32(const u32* a, int n, u32 x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ------------------------------------------------------------------ stable CTA radix sort
// Sorts (key, val) pairs [0, n) ascending by key, stable.  8-bit digits; only the
// digits in which keys differ are processed (vary = OR ^ AND over all keys).  With
// by_val the order is (key, val) lexicographic: the val digits are processed first
// (LSD), then the key digits.
// Buffers a -> b -> a ...; returns 0 if the result is in (ka, va), 1 if in (kb, vb).
// s_hist: NWARP * 256 u32 of shared memory; s_tmp: >= NWARP + 1 u32.
__device__ __noinline__ int cta_radix_sort(u64* ka, u32* va, u64* kb, u32* vb, int n, u32* s_hist, u32* s_tmp,
                              bool by_val = false) {
  if (n <= 1) return 0;
  // which digits vary
  u64 o = 0, a = ~0ull, vo = 0, vand = ~0ull;
  for (int i = threadIdx.x; i < n; i += CTA) {
    u64 k = ka[i]; o |= k; a &= k;
    if (by_val) { u64 v = va[i]; vo |= v; vand &= v; }
  }
  __shared__ u64 s_red[NWARP];
  o = cta_reduce<u64>(o, s_red, [](u64 x, u64 y) { return x | y; }, 0ull);
  a = cta_reduce<u64>(a, s_red, [](u64 x, u64 y) { return x & y; }, ~0ull);
  u64 vary = o ^ a, vvary = 0;
  if (by_val) {
    vo = cta_reduce<u64>(vo, s_red, [](u64 x, u64 y) { return x | y; }, 0ull);
    vand = cta_reduce<u64>(vand, s_red, [](u64 x, u64 y) { return x & y; }, ~0ull);
    vvary = vo ^ vand;
  }
  const int w = threadIdx.x >> 5, lane = lane_id();
  const int tile = (n + NWARP - 1) / NWARP;
  const int lo = w * tile, hi = min(n, lo + tile);
  int cur = 0;
  for (int pass = by_val ? 0 : 4; pass < 12; ++pass) {   // passes 0-3: val bytes; 4-11: key bytes
    const bool on_val = pass < 4;
    const int shift = on_val ? 8 * pass : 8 * (pass - 4);
    if ((((on_val ? vvary : vary) >> shift) & 0xFF) == 0) continue;
    u64* kin = cur ? kb : ka;
    u32* vin = cur ? vb : va;
    u64* kout = cur ? ka : kb;
    u32* vout = cur ? va : vb;
    for (int i = threadIdx.x; i < NWARP * 256; i += CTA) s_hist[i] = 0;
    __syncthreads();
    for (int base = lo; base < hi; base += 32) {
      int i = base + lane;
      bool v = i < hi;
      u32 dg = v ? (u32)(((on_val ? (u64)vin[i] : kin[i]) >> shift) & 0xFF) : 256u + lane;
      u32 peers = __match_any_sync(FULL_MASK, dg);
      if (v && (__ffs(peers) - 1) == lane) s_hist[dg * NWARP + w] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // exclusive scan over (digit, warp) order: 8 consecutive entries per thread
    {
      u32 loc8[8];
      u32 s = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) { loc8[q] = s_hist[threadIdx.x * 8 + q]; s += loc8[q]; }
      u32 total;
      u32 run = cta_excl_scan(s, s_tmp, &total);
#pragma unroll
      for (int q = 0; q < 8; ++q) { s_hist[threadIdx.x * 8 + q] = run; run += loc8[q]; }
    }
    __syncthreads();
    for (int base = lo; base < hi; base += 32) {
      int i = base + lane;
      bool v = i < hi;
      u64 k = v ? kin[i] : 0;
      u32 vv = v ? vin[i] : 0;
      u32 dg = v ? (u32)(((on_val ? (u64)vv : k) >> shift) & 0xFF) : 256u + lane;
      u32 peers = __match_any_sync(FULL_MASK, dg);
      u32 rank = __popc(peers & lanemask_lt());
      if (v) {
        u32 pos = s_hist[dg * NWARP + w] + rank;
        kout[pos] = k;
        vout[pos] = vin[i];
      }
      __syncwarp();
      if (v && (__ffs(peers) - 1) == lane) s_hist[dg * NWARP + w] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    cur ^= 1;
  }
  return cur;
}

// ------------------------------------------------------------------ small sorts
// The planner's sorts are usually short (a few hundred to a few thousand candidates)
// and latency-bound.  For n <= SORT_SMALL they run as a bitonic network on
// (key, input position) pairs held in registers (E = P/1024 pairs per thread):
// partner distance j < 32 exchanges through warp shuffles, 32 <= j < 1024 through
// double-buffered shared memory (one barrier per stage), j >= 1024 inside a thread.
// Positions are unique, so the network's order is the stable order.  Longer inputs
// fall back to the global-memory radix sort.
#define SORT_SMALL 4096
struct SortSmem {                 // 96 KiB of dynamic shared memory
  u64 k[2][SORT_SMALL];
  u32 p[2][SORT_SMALL];
};
#define PLAN_DSMEM (sizeof(SortSmem) + 4 * 4096 * sizeof(u32))   // sort + staged arrays

// keep the smaller (take_min) or larger pair of self and other; pairs are distinct
__device__ __forceinline__ void bitonic_pick(u64& k, u32& p, u64 ok, u32 op, bool take_min) {
  const bool other_less = ok < k || (ok == k && op < p);
  if (other_less == take_min) { k = ok; p = op; }
}

// Rank sort for short inputs (n <= RANK_SORT_MAX): thread i owns element i and
// counts the elements that precede it in (key, tie) order, reading all keys as
// shared-memory broadcasts; no barrier-separated network stages.  tie: unique per
// element.  Writes (key, out_val) to (kb, vb) at the element's rank.
#define RANK_SORT_MAX 512
__device__ __forceinline__ void cta_rank_sort(const u64* ka, u64* kb, u32* vb, int n, SortSmem* sm,
                                              bool tie_is_val, const u32* va) {
  const int t = threadIdx.x;
  u32 myv = 0;                                  // read before any write: (kb, vb) may be (ka, va)
  if (t < n) {
    myv = va[t];
    sm->k[0][t] = ka[t];
    sm->p[0][t] = tie_is_val ? myv : (u32)t;
  }
  __syncthreads();
  if (t < n) {
    const u64 k = sm->k[0][t];
    const u32 v = sm->p[0][t];
    u32 rank = 0;
#pragma unroll 8
    for (int j = 0; j < n; ++j) {                // independent broadcast loads: unrolled for ILP
      const u64 kj = sm->k[0][j];
      const u32 vj = sm->p[0][j];
      rank += (kj < k) | ((kj == k) & (vj < v));
    }
    kb[rank] = k;
    vb[rank] = myv;
  }
  __syncthreads();
}

// Which sort runs for n items (TA_F_SMALL_PATHS: 64 / 16 instead of 4096 / 512), and
// the counter of the branch taken.
struct SortLim { int small, rank; ull* cnt; };
__device__ __forceinline__ SortLim sort_lim(const Dev& d) {
  return small_paths(d) ? SortLim{64, 16, d.dbg} : SortLim{SORT_SMALL, RANK_SORT_MAX, d.dbg};
}
__device__ __forceinline__ void sort_count(const SortLim& L, int i) {
  if (threadIdx.x == 0) atomicAdd(&L.cnt[i], 1ull);
}

// Stable sort of (ka, va)[0, n) by key.  Returns 0 if the result is in (ka, va),
// 1 if in (kb, vb).  The buffer not holding the result is free scratch afterwards.
__device__ int cta_sort(u64* ka, u32* va, u64* kb, u32* vb, int n, u32* s_hist, u32* s_tmp, SortSmem* sm,
                        const SortLim& L) {
  if (n <= 1) return 0;
  if (n > L.small) { sort_count(L, DBG_RADIX); return cta_radix_sort(ka, va, kb, vb, n, s_hist, s_tmp); }
  if (n <= L.rank) {
    sort_count(L, DBG_RANK);
    cta_rank_sort(ka, kb, vb, n, sm, false, va);
    return 1;
  }
  sort_count(L, DBG_BITONIC);
  int P = 32;
  while (P < n) P <<= 1;
  const int E = P > CTA ? P / CTA : 1;        // 1, 2 or 4 pairs per thread
  const int t = threadIdx.x;
  const bool act = E > 1 || t < P;            // warp-uniform (P is a multiple of 32)
  u64 k[SORT_SMALL / CTA];
  u32 p[SORT_SMALL / CTA];
#pragma unroll
  for (int e = 0; e < SORT_SMALL / CTA; ++e) {
    const int i = t + e * CTA;
    k[e] = (e < E && i < n) ? ka[i] : ~0ull;   // padding sorts last (positions >= n)
    p[e] = (u32)i;
  }
  int buf = 0;
  for (int kk = 2; kk <= P; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= CTA) {                         // both elements in this thread
        // constant register indices only (no local-memory arrays): j / CTA is 1 or 2
        auto cx = [&](u64& ka_, u32& pa_, u64& kb_, u32& pb_, int e) {
          const bool up = ((t + e * CTA) & kk) == 0;
          const bool gt = ka_ > kb_ || (ka_ == kb_ && pa_ > pb_);
          if (gt == up) {
            u64 tk = ka_; ka_ = kb_; kb_ = tk;
            u32 tp = pa_; pa_ = pb_; pb_ = tp;
          }
        };
        if (j == CTA) {
          cx(k[0], p[0], k[1], p[1], 0);
          if (E > 2) cx(k[2], p[2], k[3], p[3], 2);
        } else {
          cx(k[0], p[0], k[2], p[2], 0);
          cx(k[1], p[1], k[3], p[3], 1);
        }
      } else if (j >= 32) {                   // across warps: shared memory
        if (act) {
#pragma unroll
          for (int e = 0; e < SORT_SMALL / CTA; ++e)
            if (e < E) { sm->k[buf][t + e * CTA] = k[e]; sm->p[buf][t + e * CTA] = p[e]; }
        }
        __syncthreads();
        if (act) {
#pragma unroll
          for (int e = 0; e < SORT_SMALL / CTA; ++e) {
            if (e >= E) continue;
            const int i = t + e * CTA, l = i ^ j;
            bitonic_pick(k[e], p[e], sm->k[buf][l], sm->p[buf][l], ((i & j) == 0) == ((i & kk) == 0));
          }
        }
        buf ^= 1;
      } else if (act) {                       // inside a warp: shuffles
#pragma unroll
        for (int e = 0; e < SORT_SMALL / CTA; ++e) {
          if (e >= E) continue;
          const int i = t + e * CTA;
          const u32 lo = __shfl_xor_sync(FULL_MASK, (u32)k[e], j);
          const u32 hi = __shfl_xor_sync(FULL_MASK, (u32)(k[e] >> 32), j);
          const u32 op = __shfl_xor_sync(FULL_MASK, p[e], j);
          bitonic_pick(k[e], p[e], ((u64)hi << 32) | lo, op, ((i & j) == 0) == ((i & kk) == 0));
        }
      }
    }
  }
  // keys first (nothing reads the key array any more: its reads preceded the network's
  // barriers / shuffles); the values through the scratch buffer the network read last
  // two barriers ago (every value read before any is written: in place is allowed)
  if (act) {
#pragma unroll
    for (int e = 0; e < SORT_SMALL / CTA; ++e) {
      const int i = t + e * CTA;
      if (e < E && i < n) { kb[i] = k[e]; sm->p[buf][i] = va[p[e]]; }
    }
  }
  __syncthreads();
  if (act) {
#pragma unroll
    for (int e = 0; e < SORT_SMALL / CTA; ++e) {
      const int i = t + e * CTA;
      if (e < E && i < n) vb[i] = sm->p[buf][i];
    }
  }
  __syncthreads();
  return 1;
}

// Sort (ka, va)[0, n) by (key, val) lexicographic, val unique (a slot or a
// slot-derived tie-break): the result does not depend on the input order, so inputs
// may come from unordered (atomic) appends.  Returns 0 / 1 like cta_sort.
__device__ int cta_sort_kv(u64* ka, u32* va, u64* kb, u32* vb, int n, u32* s_hist, u32* s_tmp, SortSmem* sm,
                           const SortLim& L) {
  if (n <= 1) return 0;
  if (n > L.small) { sort_count(L, DBG_RADIX); return cta_radix_sort(ka, va, kb, vb, n, s_hist, s_tmp, true); }
  if (n <= L.rank) {
    sort_count(L, DBG_RANK);
    cta_rank_sort(ka, kb, vb, n, sm, true, va);
    return 1;
  }
  sort_count(L, DBG_BITONIC);
  int P = 32;
  while (P < n) P <<= 1;
  const int E = P > CTA ? P / CTA : 1;
  const int t = threadIdx.x;
  const bool act = E > 1 || t < P;
  u64 k[SORT_SMALL / CTA];
  u32 p[SORT_SMALL / CTA];
#pragma unroll
  for (int e = 0; e < SORT_SMALL / CTA; ++e) {
    const int i = t + e * CTA;
    const bool in = e < E && i < n;
    k[e] = in ? ka[i] : ~0ull;                 // padding: (max key, max val) sorts last
    p[e] = in ? va[i] : 0xFFFFFFFFu;
  }
  int buf = 0;
  for (int kk = 2; kk <= P; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j >= CTA) {
        auto cx = [&](u64& ka_, u32& pa_, u64& kb_, u32& pb_, int e) {
          const bool up = ((t + e * CTA) & kk) == 0;
          const bool gt = ka_ > kb_ || (ka_ == kb_ && pa_ > pb_);
          if (gt == up) {
            u64 tk = ka_; ka_ = kb_; kb_ = tk;
            u32 tp = pa_; pa_ = pb_; pb_ = tp;
          }
        };
        if (j == CTA) {
          cx(k[0], p[0], k[1], p[1], 0);
          if (E > 2) cx(k[2], p[2], k[3], p[3], 2);
        } else {
          cx(k[0], p[0], k[2], p[2], 0);
          cx(k[1], p[1], k[3], p[3], 1);
        }
      } else if (j >= 32) {
        if (act) {
#pragma unroll
          for (int e = 0; e < SORT_SMALL / CTA; ++e)
            if (e < E) { sm->k[buf][t + e * CTA] = k[e]; sm->p[buf][t + e * CTA] = p[e]; }
        }
        __syncthreads();
        if (act) {
#pragma unroll
          for (int e = 0; e < SORT_SMALL / CTA; ++e) {
            if (e >= E) continue;
            const int i = t + e * CTA, l = i ^ j;
            bitonic_pick(k[e], p[e], sm->k[buf][l], sm->p[buf][l], ((i & j) == 0) == ((i & kk) == 0));
          }
        }
        buf ^= 1;
      } else if (act) {
#pragma unroll
        for (int e = 0; e < SORT_SMALL / CTA; ++e) {
          if (e >= E) continue;
          const int i = t + e * CTA;
          const u32 lo = __shfl_xor_sync(FULL_MASK, (u32)k[e], j);
          const u32 hi = __shfl_xor_sync(FULL_MASK, (u32)(k[e] >> 32), j);
          const u32 op = __shfl_xor_sync(FULL_MASK, p[e], j);
          bitonic_pick(k[e], p[e], ((u64)hi << 32) | lo, op, ((i & j) == 0) == ((i & kk) == 0));
        }
      }
    }
  }
  if (act) {
#pragma unroll
    for (int e = 0; e < SORT_SMALL / CTA; ++e) {
      const int i = t + e * CTA;
      if (e < E && i < n) { kb[i] = k[e]; vb[i] = p[e]; }
    }
  }
  __syncthreads();
  return 1;
}

// ------------------------------------------------------------------ exact prefix selection
// The pause, restore and eviction passes consume only a PREFIX of their sorted
// order.  bucket(i) is a coarse key monotone in the full sort key, so the items of
// buckets [lo, T] are exactly the next stretch of the global order.  One pass
// builds a weighted histogram in shared memory, a scan finds the smallest T whose
// cumulative weight reaches `need`, and an ordered gather emits (slot order) the
// items with lo <= bucket <= T; the caller then sorts only that subset.
// s_hist: >= nbkt u32 (nbkt <= 8192).  Returns T (nbkt - 1 if need is never reached).
template <typename Pred, typename Bucket, typename Weight>
__device__ u32 cta_bucket_threshold(int n, u32 nbkt, u32 lo, ull need, u32* s_hist, u32* s_tmp,
                                    Pred pred, Bucket bucket, Weight weight) {
  __shared__ u32 s_T;
  for (u32 b = threadIdx.x; b < nbkt; b += CTA) s_hist[b] = 0;
  if (threadIdx.x == 0) s_T = nbkt - 1;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += CTA) {
    if (!pred(i)) continue;
    u32 b = bucket(i);
    if (b >= lo) atomicAdd(&s_hist[b], weight(i));
  }
  __syncthreads();
  {                                      // inclusive scan, 8 buckets per thread
    const u32 per = (nbkt + CTA - 1) / CTA;
    const u32 b0 = threadIdx.x * per;
    ull s = 0;
    for (u32 q = 0; q < per && b0 + q < nbkt; ++q) s += s_hist[b0 + q];
    u32 total;
    ull run = cta_excl_scan((u32)min(s, 0xFFFFFFFFull), s_tmp, &total);
    for (u32 q = 0; q < per && b0 + q < nbkt; ++q) {
      run += s_hist[b0 + q];
      if (run >= need) { atomicMin(&s_T, b0 + q); break; }
    }
  }
  __syncthreads();
  const u32 T = s_T;
  __syncthreads();
  return T;
}

// Bucket threshold from a histogram already in global memory (built by other kernels).
__device__ u32 cta_hist_threshold(const u32* ghist, u32 nbkt, u32 lo, ull need, u32* s_hist, u32* s_tmp) {
  __shared__ u32 s_T;
  for (u32 b = threadIdx.x; b < nbkt; b += CTA) s_hist[b] = b >= lo ? ghist[b] : 0u;
  if (threadIdx.x == 0) s_T = nbkt - 1;
  __syncthreads();
  const u32 per = (nbkt + CTA - 1) / CTA;
  const u32 b0 = threadIdx.x * per;
  ull sum = 0;
  for (u32 q = 0; q < per && b0 + q < nbkt; ++q) sum += s_hist[b0 + q];
  u32 total;
  ull run = cta_excl_scan((u32)min(sum, 0xFFFFFFFFull), s_tmp, &total);
  for (u32 q = 0; q < per && b0 + q < nbkt; ++q) {
    run += s_hist[b0 + q];
    if (run >= need) { atomicMin(&s_T, b0 + q); break; }
  }
  __syncthreads();
  const u32 T = s_T;
  __syncthreads();
  return T;
}

// Bucket threshold over an explicit candidate list (lst[0, n), unordered): like
// cta_bucket_threshold, with pred/bucket/weight evaluated on the listed slots.
template <typename Pred, typename Bucket, typename Weight>
__device__ u32 cta_list_threshold(const u32* lst, int n, u32 nbkt, u32 lo, ull need, u32* s_hist, u32* s_tmp,
                                  Pred pred, Bucket bucket, Weight weight) {
  return cta_bucket_threshold(n, nbkt, lo, need, s_hist, s_tmp,
                              [&](int i) { return pred((int)lst[i]); },
                              [&](int i) { return bucket((int)lst[i]); },
                              [&](int i) { return weight((int)lst[i]); });
}

// Append the listed slots that satisfy pred: emit(pos, slot) with pos from a shared
// counter (unordered).  Returns the count.
template <typename Pred, typename Emit>
__device__ u32 cta_list_gather(const u32* lst, int n, u32* s_cnt, Pred pred, Emit emit) {
  if (threadIdx.x == 0) *s_cnt = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += CTA) {               // uniform trip count (warp ballots)
    const int i = i0 + threadIdx.x;
    const int p = i < n ? (int)lst[i] : 0;
    const bool take = i < n && pred(p);
    const u32 m = __ballot_sync(FULL_MASK, take);      // warp-aggregated append
    u32 base = 0;
    if (lane_id() == 0 && m) base = atomicAdd(s_cnt, (u32)__popc(m));
    base = __shfl_sync(FULL_MASK, base, 0);
    if (take) emit(base + __popc(m & lanemask_lt()), p);
  }
  __syncthreads();
  const u32 n_out = *s_cnt;
  __syncthreads();
  return n_out;
}

// ------------------------------------------------------------------ bitmap rank / select
// s_pre[w] = number of set bits in words [0, w) for w in [0, nw]; built by one CTA.
__device__ void cta_bitmap_prefix(const u32* words, int nw, u32* s_pre, u32* s_tmp) {
  int chunk = (nw + CTA - 1) / CTA;
  int lo = threadIdx.x * chunk, hi = min(nw, lo + chunk);
  u32 s = 0;
  // one word per thread up to 32K-word bitmaps: rolled loops (compact code, see DESIGN 6.2)
#pragma unroll 1
  for (int i = lo; i < hi; ++i) s += __popc(words[i]);
  u32 total;
  u32 run = cta_excl_scan(s, s_tmp, &total);
#pragma unroll 1
  for (int i = lo; i < hi; ++i) { s_pre[i] = run; run += __popc(words[i]); }
  if (threadIdx.x == 0) s_pre[nw] = total;
  __syncthreads();
}
// Index of the q-th (0-based) set bit, given prefix counts s_pre (q < s_pre[nw]).
__device__ __forceinline__ u32 bitmap_select(const u32* words, const u32* s_pre, int nw, u32 q) {
  int lo = 0, hi = nw;                    // last word w with s_pre[w] <= q
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (s_pre[mid] <= q) lo = mid; else hi = mid;
  }
  u32 w = words[lo];
  u32 k = q - s_pre[lo];                  // k-th set bit inside w
  u32 pos = __fns(w, 0, (int)k + 1);
  return (u32)lo * 32u + pos;
}

// The slots of a bitmap (bit b of word w = slot 32w + b) in ascending slot order: into
// s_out (shared memory, capacity s_cap) when they fit, else into g_out (global).  One
// CTA; every thread takes a contiguous run of words.  *out receives the list used.
__device__ u32 cta_bits_to_list(const u32* words, int nw, u32* s_out, u32 s_cap, u32* g_out, u32* s_tmp,
                                const u32** out) {
  const int chunk = (nw + CTA - 1) / CTA;
  const int lo = threadIdx.x * chunk, hi = min(nw, lo + chunk);
  u32 cnt = 0;
#pragma unroll 1
  for (int w = lo; w < hi; ++w) cnt += __popc(words[w]);
  u32 total;
  u32 pos = cta_excl_scan(cnt, s_tmp, &total);
  u32* dst = total <= s_cap ? s_out : g_out;
#pragma unroll 1
  for (int w = lo; w < hi; ++w) {
    u32 m = words[w];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      dst[pos++] = (u32)(w * 32 + b);
    }
  }
  __syncthreads();
  *out = dst;
  return total;
}

// Write the listed slots (unique, < N) to out[0, n) in ascending slot order: mark them
// in a shared-memory slot bitmap, rank each by the bitmap prefix.  s_bits: >= nw
// words, s_pre: >= nw + 1 words, nw = ceil(N / 32).
__device__ void cta_slot_order(const u32* lst, int n, int N, u32* out, u32* s_bits, u32* s_pre, u32* s_tmp) {
  const int nw = (N + 31) / 32;
  for (int w = threadIdx.x; w < nw; w += CTA) s_bits[w] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += CTA) {
    const u32 p = lst[i];
    atomicOr(&s_bits[p >> 5], 1u << (p & 31));
  }
  __syncthreads();
  cta_bitmap_prefix(s_bits, nw, s_pre, s_tmp);
  for (int i = threadIdx.x; i < n; i += CTA) {
    const u32 p = lst[i];
    out[s_pre[p >> 5] + __popc(s_bits[p >> 5] & ((1u << (p & 31)) - 1))] = p;
  }
  __syncthreads();
}
