// ta_runtime.cu — host side of libta: the C ABI of include/ta.h.
//
// Owns no memory: every buffer comes from the caller (ta_buffers).  The tick is a
// fixed sequence of kernels on the caller's stream; in trace mode it is captured
// once into a CUDA graph and replayed (all sizes are read on the device).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "k_copy.cuh"
#include "k_finalize.cuh"
#include "k_ingest.cuh"
#include "k_plan.cuh"
#include "k_sched.cuh"
#include "k_verb.cuh"

namespace {

const int kCopyGrid = 148 * 8;   // copy kernels: 8 resident 256-thread CTAs per SM
const size_t kEvpOffset = 512;   // eviction flags inside the mailbox allocation
// API-mode event batch capacity: 4 events per program slot (at least 4096)
static inline size_t ev_capacity(const ta_config* c) {
  return std::max<size_t>(4096, 4 * (size_t)c->max_programs);
}

struct Layout {                  // workspace carving (dry run when base == nullptr)
  char* base;
  size_t off = 0;
  template <class T> T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

struct HostWs {
  ta_decision* dec;              // [dec_cap]
  u32* dec_cnt;
  ta_tick_info* tick_info;
  ta_event* ev;                  // [ev_capacity] pinned staging of the event batch
  i64* scal;                     // [8] small H2D/D2H staging
};

}  // namespace

struct ta_ctx {
  ta_config cfg;
  ta_buffers bufs;
  cudaStream_t stream;
  Dev d;
  HostWs h;
  ta_event* ev_dev = nullptr;
  cudaGraphExec_t graph = nullptr;
  bool trace_loaded = false;
  int poisoned = TA_OK;
  std::string err;
  size_t block_bytes = 0;
  cudaEvent_t ev[10] = {};
  bool timing = false;
  void* mbox_alloc = nullptr;               // barrier mailbox + (multi) eviction flags, library-owned
  int move_grid = 0;                        // resident CTAs of k_move_fused (even)
  int close_grid = 1;                       // CTAs of the cooperative k_close
  void* peer_base[TA_MAX_REPLICAS] = {};    // IPC-opened peer pool allocations
  void* peer_mbox[TA_MAX_REPLICAS] = {};    // IPC-opened peer mailboxes
  bool split_pr = false;                    // A/B aid (env TA_SPLIT_PR at init): k_pause + k_restore
  bool probes = false;                      // A/B aid (env TA_GAP_PROBES, timing mode): k_probe between kernels
  bool no_events = false;                   // A/B aid (env TA_NO_EVENTS): device stamps without event nodes
};

#define FAIL(ctx, code, ...)                                          \
  do {                                                                \
    char _b[512];                                                     \
    snprintf(_b, sizeof(_b), __VA_ARGS__);                            \
    if (ctx) (ctx)->err = _b;                                         \
    return (code);                                                    \
  } while (0)

#define CK(ctx, x)                                                                     \
  do {                                                                                 \
    cudaError_t _e = (x);                                                              \
    if (_e != cudaSuccess) {                                                           \
      if (ctx) {                                                                       \
        (ctx)->err = std::string(#x) + ": " + cudaGetErrorString(_e);                  \
        (ctx)->poisoned = TA_E_CUDA;                                                   \
      }                                                                                \
      return TA_E_CUDA;                                                                \
    }                                                                                  \
  } while (0)

static size_t blk_bytes(const ta_config* c) {
  return (size_t)2 * c->n_layers * c->block_tokens * c->n_kv_heads * c->head_dim * c->elem_bytes;
}

static const char* validate(const ta_config* c) {
  if (!c) return "null config";
  if (c->elem_bytes != 2) return "elem_bytes must be 2";
  if (c->n_layers <= 0 || c->n_kv_heads <= 0 || c->head_dim <= 0 || c->block_tokens <= 0)
    return "KV shape must be positive";
  if ((c->n_kv_heads * c->head_dim) % 8) return "n_kv_heads*head_dim must be a multiple of 8";
  if (c->layout != 0 && c->layout != 1) return "layout must be 0 or 1";
  if (c->n_replicas < 1 || c->n_replicas > TA_MAX_REPLICAS) return "n_replicas out of range";
  if (c->replicas_here < 1 || c->first_replica < 0 || c->first_replica + c->replicas_here > c->n_replicas)
    return "replicas_here/first_replica out of range";
  if (c->max_programs < 1 || c->max_blocks_per_program < 1) return "max_programs/max_blocks must be >= 1";
  if (c->max_programs > 262144) return "max_programs must be <= 262144 (planner slot bitmaps in shared memory)";
  if (c->max_blocks_per_program >= (1 << 23)) return "max_blocks_per_program must be < 2^23";
  if ((uint64_t)c->max_programs * (uint64_t)c->max_blocks_per_program >= (1ull << 32))
    return "max_programs * max_blocks_per_program must be < 2^32";
  if (c->hbm_blocks < 1 || c->hbm_blocks > 131040) return "hbm_blocks must be in [1, 131040]";
  if (c->host_blocks < 0 || c->host_blocks > 262112) return "host_blocks must be in [0, 262112]";
  if (c->delta_t_ms <= 0 || c->decay_unit_ms <= 0) return "delta_t_ms and decay_unit_ms must be > 0";
  if (c->lambda_min_q16 == 0 || c->lambda_min_q16 > c->lambda_max_q16 || c->lambda_max_q16 > 65536)
    return "watermarks must satisfy 0 < lambda_min <= lambda_max <= 1 (SPEC.md:190)";
  if (c->decode_tok_per_s < 0 || c->compact_every < 0 || c->max_trace_turns < 0) return "negative rate/compact/turns";
  if (c->prefill_chunk_tokens < 1 || c->prefill_chunk_ms < 0) return "prefill_chunk_tokens must be >= 1, prefill_chunk_ms >= 0";
  if (c->shared_prefix_tokens < 0 || c->shared_prefix_tokens % c->block_tokens != 0 ||
      c->shared_prefix_tokens / c->block_tokens >= c->hbm_blocks)
    return "shared_prefix_tokens must be a multiple of block_tokens, below hbm_blocks blocks";
  if (c->n_prefixes < 0 || c->n_prefixes > TA_MAX_PREFIXES) return "n_prefixes must be in [0, TA_MAX_PREFIXES]";
  if (c->compact_every > 0 && c->hbm_blocks > 87360) return "compaction needs hbm_blocks <= 87360 (its plan in shared memory)";
  for (int k = 0; k < c->n_prefixes; ++k)
    if (c->prefix_tokens[k] <= 0 || c->prefix_tokens[k] % c->block_tokens != 0 ||
        c->prefix_tokens[k] / c->block_tokens >= c->hbm_blocks || c->prefix_tokens[k] / c->block_tokens >= (1 << 20))
      return "prefix_tokens must be positive multiples of block_tokens, below hbm_blocks blocks";
  if ((uint64_t)c->max_programs * (uint64_t)c->max_blocks_per_program >= (uint64_t)TA_OWNER_PROMPT)
    return "max_programs * max_blocks_per_program must be below TA_OWNER_PROMPT";
#ifdef TA_PROD_VARIANT
  if (c->flags & (TA_F_TIMING | TA_F_PINNED_ROUTING | TA_F_REQUEST_AWARE | TA_F_SMALL_PATHS | TA_F_JITTER |
                  TA_F_FULL_SCAN))
    return "TA_F_TIMING / TA_F_PINNED_ROUTING / TA_F_REQUEST_AWARE / TA_F_SMALL_PATHS / TA_F_JITTER / TA_F_FULL_SCAN "
           "need libta_dev.so "
           "(the development build of the same sources; libta.so compiles them out)";
#endif
  return nullptr;
}

static size_t carve(const ta_config* c, char* base, Dev* d) {
  Layout L{base};
  const size_t N = c->max_programs, R = c->n_replicas, NB = c->hbm_blocks;
  const size_t NH = c->host_blocks > 0 ? c->host_blocks : 1;
  const size_t MAXBP = (c->max_blocks_per_program + 3) & ~3;
  const size_t NBW = (NB + 31) / 32, NHW = (NH + 31) / 32;
  const size_t TT = c->max_trace_turns > 0 ? c->max_trace_turns : 1;
  Dev x{};
  x.ctr = L.take<Ctr>(1);
  x.stats = L.take<ull>(ST_N);
  x.verify = L.take<ull>(2);
  x.uid = L.take<u32>(N); x.c = L.take<u32>(N); x.c_kv = L.take<u32>(N);
  x.paused_since = L.take<u32>(N); x.step_count = L.take<u32>(N); x.turn = L.take<u32>(N);
  x.gen_done = L.take<u32>(N);
  x.status = L.take<u8>(N); x.phase = L.take<u8>(N); x.satisfied = L.take<u8>(N);
  x.placement = L.take<i8>(N); x.home = L.take<i8>(N);
  x.acting_since = L.take<i64>(N); x.tool_return = L.take<i64>(N);
  x.loc = L.take<u32>(N * MAXBP);
  x.nb = L.take<u32>(N); x.n_hbm = L.take<u32>(N); x.n_host = L.take<u32>(N);
  x.prefix_hbm = L.take<u32>(N); x.contrib = L.take<u32>(N);
  x.pend = L.take<u32>(N); x.busy = L.take<u32>(N); x.hcls = L.take<u8>(N);
  {                                        // NEXT-3 prompts (A51)
    int K = c->n_prefixes ? c->n_prefixes : (c->shared_prefix_tokens ? 1 : 0);
    size_t SBM = 1;
    for (int k = 0; k < K; ++k) {
      const int t = c->n_prefixes ? c->prefix_tokens[k] : c->shared_prefix_tokens;
      SBM = std::max<size_t>(SBM, (size_t)(t / c->block_tokens));
    }
    x.kp = L.take<u8>(N); x.t_kp = L.take<u8>(N);
    x.pref = L.take<u32>(R * std::max(K, 1)); x.pblk = L.take<u32>(R * std::max(K, 1) * SBM);
    x.pfix = L.take<u32>(R * NBW); x.f_x = L.take<u32>(R * N);
  }
  x.released = L.take<u8>(N); x.sat_new = L.take<u8>(N); x.dirty = L.take<u8>(N); x.evs = L.take<u8>(3 * N);
  x.evc = L.take<u32>(N);
  x.t_uid = L.take<u32>(N); x.t_p0 = L.take<u32>(N); x.t_off = L.take<u32>(N + 1);
  x.t_g = L.take<u32>(TT); x.t_d = L.take<u32>(TT); x.t_o = L.take<u32>(TT);
  x.hbm_free = L.take<u32>(R * NBW); x.host_free = L.take<u32>(R * NHW);
  x.owner_hbm = L.take<u32>(R * NB); x.owner_host = L.take<u32>(R * NH);
  x.L = L.take<ull>(R); x.Lacc = L.take<ull>(R);
  x.ska = L.take<u64>((R + 1) * N); x.skb = L.take<u64>((R + 1) * N);
  x.sva = L.take<u32>((R + 1) * N); x.svb = L.take<u32>((R + 1) * N);
  x.pause_list = L.take<u32>(R * N); x.pause_cnt = L.take<u32>(R);
  x.restore_pid = L.take<u32>(N); x.restore_dst = L.take<u32>(N);
  x.f_pid = L.take<u32>(R * N); x.f_cum = L.take<u32>(R * N);
  x.f_cnt = L.take<u32>(R); x.s_cnt = L.take<u32>(R);
  x.dec_fs = L.take<ta_decision>(R * N); x.dec_ev = L.take<ta_decision>(R * N);
  x.ev_cnt = L.take<u32>(R);
  x.e_pid = L.take<u32>(R * N); x.e_cum = L.take<u32>(R * N);
  x.evd = L.take<EvDesc>(R * NB); x.evd_cnt = L.take<u32>(R); x.evx = L.take<u32>(R * NB);
  x.evt = L.take<EvDesc>(R * NB);
  x.fed = L.take<FeDesc>(R * NB); x.fedt = L.take<FeDesc>(R * NB); x.fed_cnt = L.take<u32>(R); x.evp = L.take<u32>(R * NB);
  x.fld = L.take<FillDesc>(R * NB); x.fld_cnt = L.take<u32>(R);
  x.dfh = L.take<u32>(R * NB); x.dfh_cnt = L.take<u32>(R);
  x.dfs = L.take<u32>(R * NB); x.dfs_cnt = L.take<u32>(R);
  x.cpd = L.take<CpDesc>(R * (NB / 2 + 1)); x.cpd_cnt = L.take<u32>(R);
  const size_t EC = ev_capacity(c);
  x.events = L.take<ta_event>(EC);
  x.evr = reinterpret_cast<EvRes*>(L.take<char>(EC * 32));
  x.ev_pcnt = L.take<u32>(N);
  x.ev_mk = L.take<u64>(EC); x.ev_mk2 = L.take<u64>(EC);
  x.ev_mv = L.take<u32>(EC); x.ev_mv2 = L.take<u32>(EC);
  x.pst = L.take<ull>(8 * 32);
  x.gsync = L.take<ull>(2);
  x.dbg = L.take<ull>(DBG_N);
  x.t_rep = L.take<u32>(3 * R);
  const size_t NWs = (N + 31) / 32;
  x.act_bits = L.take<u32>(R * NWs); x.reas_bits = L.take<u32>(R * NWs); x.ec_bits = L.take<u32>(R * NWs);
  x.act_list = L.take<u32>(R * N); x.ec_list = L.take<u32>(R * N);
  x.rhist = L.take<u32>(2 * 2048 + 2); x.rb = L.take<u32>(N);
  if (d) *d = x;
  return L.off + 256;
}

static size_t host_carve(const ta_config* c, char* base, HostWs* h) {
  Layout L{base};
  HostWs x{};
  const size_t cap = 4 * (size_t)c->max_programs + c->n_replicas + 64;
  x.dec = L.take<ta_decision>(cap);
  x.dec_cnt = L.take<u32>(1);
  x.tick_info = L.take<ta_tick_info>(1);
  x.ev = L.take<ta_event>(ev_capacity(c));
  x.scal = L.take<i64>(8);
  if (h) *h = x;
  return L.off + 256;
}

__global__ void k_init(Dev d) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  for (int r = 0; r < d.R; ++r) {
    for (int w = t; w < d.NBW; w += stride) {
      i64 lo = (i64)w * 32, n = d.NB - lo;
      d.hbm_free[(size_t)r * d.NBW + w] = n <= 0 ? 0u : (n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1));
    }
    for (int w = t; w < d.NHW; w += stride) {
      i64 lo = (i64)w * 32, n = d.NH - lo;
      d.host_free[(size_t)r * d.NHW + w] = n <= 0 ? 0u : (n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1));
    }
  }
  if (t == 0) { d.ctr->ev_err = ~0ull; d.ctr->cmin = 0xFFFFFFFFu; }
  for (int p = t; p < d.N; p += stride) {
    d.tool_return[p] = INT64_MAX;
    d.placement[p] = -1;
    d.home[p] = -1;
    d.kp[p] = KP_NONE;
    d.t_kp[p] = d.K ? 0 : KP_NONE;                     // trace prompts: ta_load_trace
  }
}

// ------------------------------------------------------------------ tick launch sequence
static void rec(ta_ctx* x, int i, cudaStream_t s = nullptr) {
  if (!x->timing || x->no_events) return;
  cudaStream_t st = s ? s : x->stream;
  // external event-record nodes keep working inside the captured CUDA graph; outside a
  // capture (verbs, TA_F_NO_GRAPH) a plain record
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(x->ev[i], st, cudaEventRecordExternal);
  else
    cudaEventRecord(x->ev[i], st);
}

// dynamic shared memory of the copy kernels: the TMA staging buffer in bulk mode
static inline size_t csm(const Dev& d) { return (d.flags & TA_F_COPY_BULK) ? BULK_CHUNK : 0; }

// Cooperative launch (all CTAs co-resident: the kernel has grid barriers or waits
// across CTAs).
template <typename... Args>
static void launch_coop_b(void (*k)(Args...), int grid, int block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(block);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = grid > 1 ? 1 : 0;       // one CTA needs no co-residency guarantee
  cudaLaunchKernelEx(&lc, k, args...);
}
template <typename... Args>
static void launch_coop(void (*k)(Args...), int grid, size_t smem, cudaStream_t s, Args... args) {
  launch_coop_b(k, grid, CTA, smem, s, args...);
}

// Step 6.  Single process: one fused kernel (D2H overlapped with H2D/P2P and fills).
// Multi-process: evict -> barrier -> fetch (pull) + push -> barrier -> fills.
static void launch_movement(ta_ctx* x, cudaStream_t s) {
  Dev& d = x->d;
  if (d.fused) {
    // one process per GPU: every peer's plan (and its eviction flags) is in place before
    // anyone pushes, and every transfer has landed before anyone reuses a block
    if (d.multi) k_barrier<<<1, 32, 0, s>>>(d);
    // persistent, CTAs wait on each other's evictions: cooperative, so the driver either
    // makes the whole grid co-resident or fails the launch (never a partial grid)
    launch_coop_b(k_move_fused, x->move_grid, 256, csm(d), s, (Dev)d);
    if (d.multi) k_barrier<<<1, 32, 0, s>>>(d);
    rec(x, 4, s);
    rec(x, 5, s);
    if (d.multi && (d.flags & TA_F_FILL)) k_fill<<<kCopyGrid, 256, 0, s>>>(d);
    return;
  }
  k_copy_evict<<<kCopyGrid, 256, csm(d), s>>>(d);
  if (d.multi) k_barrier<<<1, 32, 0, s>>>(d);   // evicted blocks read before peers refill them
  rec(x, 4);
  k_copy_fetch<<<kCopyGrid, 256, csm(d), s>>>(d);
  if (d.multi) {
    k_copy_push<<<kCopyGrid, 256, csm(d), s>>>(d);
    k_barrier<<<1, 32, 0, s>>>(d);               // fetches landed; P2P sources read
  }
  rec(x, 5);
  if (d.flags & TA_F_FILL) k_fill<<<kCopyGrid, 256, 0, s>>>(d);
}

static cudaError_t launch_tick(ta_ctx* x, int) {
  Dev& d = x->d;
  cudaStream_t s = x->stream;
  const int N = d.N, R = d.R;
  if (x->timing) k_span_reset<<<1, 32, 0, s>>>(d);
  rec(x, 0);
  // per-tick lists and counters were cleared by the previous tick's k_assemble
  if (d.api_mode) {
    // events: validate + apply in parallel over programs (n_events read on the device)
    const int eg = (int)std::min<size_t>(148 * 4, (ev_capacity(&x->cfg) + 255) / 256);
    k_ev_count<<<eg, 256, 0, s>>>(d);
    k_ev_single<<<eg, 256, 0, s>>>(d);
    k_ev_multi<<<1, CTA, PLAN_DSMEM, s>>>(d);
    k_ev_apply<<<eg, 256, 0, s>>>(d);
    k_footprint<<<FP_GRID(N), FP_BLOCK, FP_DSMEM, s>>>(d, 0);
  } else {
    k_tick_front<<<FP_GRID(N), FP_BLOCK, FP_DSMEM, s>>>(d);   // ingest + footprint + load
  }
  rec(x, 1);
  if (x->probes) k_probe<<<1, 32, 0, s>>>(d, 0);
  if (x->split_pr) {                       // A/B aid: the two passes as separate kernels
    k_pause<<<R, CTA, PLAN_DSMEM, s>>>(d);
    k_restore<<<1, CTA, PLAN_DSMEM, s>>>(d);
  } else {
    launch_coop(k_pause_restore, R, PLAN_DSMEM, s, (Dev)d);
  }
  rec(x, 2);
  if (x->probes) k_probe<<<1, 32, 0, s>>>(d, 1);
  k_plan<0><<<R * PLAN_CL, CTA, PLAN_DSMEM, s>>>(d);   // one CTA cluster per replica
  rec(x, 3);
  if (x->probes) k_probe<<<1, 32, 0, s>>>(d, 2);
  const bool copies = !(d.flags & TA_F_DECIDE_ONLY);
  if (copies) {
    launch_movement(x, s);
  } else {
    rec(x, 4);
    rec(x, 5);
  }
  rec(x, 6);
  launch_coop(k_close<0>, x->close_grid, 0, s, (Dev)d);     // frees, compaction plan, decisions
  rec(x, 7);
  if (copies && d.compact_every > 0) k_copy_compact<<<kCopyGrid, 256, csm(d), s>>>(d);
  rec(x, 8);
  rec(x, 9);
  return cudaGetLastError();
}

static ta_status check_ctx(ta_ctx* ctx) {
  if (!ctx) return TA_E_INVAL;
  if (ctx->poisoned) return (ta_status)ctx->poisoned;
  return TA_OK;
}

// Multi-process contexts need every peer's pool and mailbox before any data movement.
static ta_status check_peers(ta_ctx* ctx) {
  if (!ctx->d.multi) return TA_OK;
  for (int r = 0; r < ctx->d.R; ++r)
    if (r != ctx->d.rank && (!ctx->d.hbm[r] || !ctx->d.mbox_peer[r]))
      FAIL(ctx, TA_E_STATE, "peer replica %d not imported (ta_import_peer_pool)", r);
  return TA_OK;
}

// A barrier that timed out (dead peer) poisons the context.
static ta_status check_device_err(ta_ctx* ctx) {
  CK(ctx, cudaMemcpyAsync(ctx->h.scal + 2, &ctx->d.ctr->err, sizeof(i32), cudaMemcpyDeviceToHost, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  if (*(i32*)(ctx->h.scal + 2) == TA_E_PEER) {
    ctx->poisoned = TA_E_PEER;
    FAIL(ctx, TA_E_PEER, "cross-process barrier timed out");
  }
  return TA_OK;
}

static ta_status copy_out(ta_ctx* ctx, ta_decision* out, int32_t out_cap, int32_t* n_out) {
  u32 n = *ctx->h.dec_cnt;
  if (n_out) *n_out = (int32_t)n;
  if (!out) return TA_OK;
  u32 m = n < (u32)out_cap ? n : (u32)out_cap;
  memcpy(out, ctx->h.dec, (size_t)m * sizeof(ta_decision));
  return n > (u32)out_cap ? TA_E_TRUNCATED : TA_OK;
}

// ------------------------------------------------------------------ C ABI
extern "C" {

int32_t ta_abi_version(void) { return TA_ABI_VERSION; }

ta_status ta_block_bytes(const ta_config* cfg, size_t* block_bytes) {
  if (!cfg || !block_bytes) return TA_E_INVAL;
  *block_bytes = blk_bytes(cfg);
  return TA_OK;
}

ta_status ta_workspace_bytes(const ta_config* cfg, size_t* dev_bytes, size_t* host_bytes) {
  if (validate(cfg)) return TA_E_INVAL;
  if (dev_bytes) *dev_bytes = carve(cfg, nullptr, nullptr);
  if (host_bytes) *host_bytes = host_carve(cfg, nullptr, nullptr);
  return TA_OK;
}

ta_status ta_init_pool(const ta_config* cfg, const ta_buffers* bufs, void* cuda_stream, void* nccl_comm,
                       ta_ctx** out) {
  if (!out || !bufs) return TA_E_INVAL;
  *out = nullptr;
  if (const char* why = validate(cfg)) {
    fprintf(stderr, "ta_init_pool: %s\n", why);
    return TA_E_INVAL;
  }
  if (nccl_comm) return TA_E_INVAL;
  if (!bufs->dev_workspace || !bufs->host_workspace) return TA_E_NOMEM;
  for (int q = 0; q < cfg->replicas_here; ++q) {
    int r = cfg->first_replica + q;
    if (!bufs->hbm_pool[r]) return TA_E_INVAL;
    if (cfg->host_blocks > 0 && !bufs->host_pool[r]) return TA_E_INVAL;
  }
  ta_ctx* x = new ta_ctx();
  x->cfg = *cfg;
  x->bufs = *bufs;
  x->stream = (cudaStream_t)cuda_stream;
  x->block_bytes = blk_bytes(cfg);
  Dev& d = x->d;
  carve(cfg, (char*)bufs->dev_workspace, &d);
  host_carve(cfg, (char*)bufs->host_workspace, &x->h);
  x->ev_dev = d.events;
  d.N = cfg->max_programs;
  d.NW = (cfg->max_programs + 31) / 32;
  d.MAXB = cfg->max_blocks_per_program;
  d.MAXBP = (cfg->max_blocks_per_program + 3) & ~3;
  d.R = cfg->n_replicas;
  d.bt = cfg->block_tokens;
  d.nL = cfg->n_layers; d.Hkv = cfg->n_kv_heads; d.D = cfg->head_dim; d.layout = cfg->layout;
  d.NB = cfg->hbm_blocks; d.NH = cfg->host_blocks;
  d.NBW = (int)((d.NB + 31) / 32);
  d.NHW = (int)((d.NH + 31) / 32);
  d.dt = cfg->delta_t_ms; d.unit = cfg->decay_unit_ms; d.rate = cfg->decode_tok_per_s;
  d.flags = cfg->flags; d.compact_every = cfg->compact_every;
  d.chunk_q = cfg->prefill_chunk_tokens;
  d.chunk_ms = cfg->prefill_chunk_ms;
  d.K = cfg->n_prefixes ? cfg->n_prefixes : (cfg->shared_prefix_tokens ? 1 : 0);
  d.SBM = 1;
  for (int k = 0; k < TA_MAX_PREFIXES; ++k) {
    const int t = k < d.K ? (cfg->n_prefixes ? cfg->prefix_tokens[k] : cfg->shared_prefix_tokens) : 0;
    d.sbk[k] = (u32)(t / cfg->block_tokens);
    d.SBM = std::max(d.SBM, d.sbk[k]);
  }
  d.seg_bytes = (i64)cfg->block_tokens * cfg->n_kv_heads * cfg->head_dim * cfg->elem_bytes;
  d.block_bytes = (i64)x->block_bytes;
  d.first_local = cfg->first_replica; d.n_local = cfg->replicas_here;
  d.nb_shift = 0;
  const u32 nbk_max = (cfg->flags & TA_F_SMALL_PATHS) ? 8u : 2048u;   // restore / pause buckets
  while (((u32)d.MAXB >> d.nb_shift) + 1 > nbk_max) ++d.nb_shift;
  d.nbk = ((u32)d.MAXB >> d.nb_shift) + 1;
  d.api_mode = (cfg->flags & TA_F_TRACE_MODE) ? 0 : 1;
  for (int r = 0; r < d.R; ++r) {
    d.cap_max[r] = (i64)(((u64)cfg->lambda_max_q16 * (u64)d.NB) >> 16);
    d.cap_min[r] = (i64)(((u64)cfg->lambda_min_q16 * (u64)d.NB) >> 16);
  }
  d.healthy = d.R >= 32 ? 0xFFFFFFFFu : ((1u << d.R) - 1);
  for (int k = 0; k < 64; ++k) d.F[k] = cfg->decay_q32[k];
  for (int r = 0; r < TA_MAX_REPLICAS; ++r) {
    d.hbm[r] = (char*)bufs->hbm_pool[r];
    d.host[r] = nullptr;
    if (bufs->host_pool[r] && cfg->host_blocks > 0) {
      void* dp = nullptr;
      cudaError_t e = cudaHostGetDevicePointer(&dp, bufs->host_pool[r], 0);
      if (e != cudaSuccess) {
        x->err = std::string("host tier is not page-locked/mapped: ") + cudaGetErrorString(e);
        delete x;
        return TA_E_INVAL;
      }
      d.host[r] = (char*)dp;
    }
  }
  {
    void* dp = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&dp, bufs->host_workspace, 0);
    if (e != cudaSuccess) { delete x; return TA_E_INVAL; }
    char* hb = (char*)dp;
    d.dec_out = (ta_decision*)(hb + ((char*)x->h.dec - (char*)bufs->host_workspace));
    d.dec_out_cnt = (u32*)(hb + ((char*)x->h.dec_cnt - (char*)bufs->host_workspace));
    d.tick_info = (ta_tick_info*)(hb + ((char*)x->h.tick_info - (char*)bufs->host_workspace));
    d.dec_cap = (u32)(4 * (size_t)cfg->max_programs + cfg->n_replicas + 64);
  }
  d.n_slots = 0;
  d.n_initial = 0;
  x->timing = (cfg->flags & TA_F_TIMING) != 0;
  x->split_pr = getenv("TA_SPLIT_PR") != nullptr;
  d.multi = cfg->replicas_here < cfg->n_replicas ? 1 : 0;
  d.rank = cfg->first_replica;
  d.fused = !(cfg->flags & TA_F_NO_FUSE) ? 1 : 0;
  {   // the fused movement kernel waits across CTAs: launch only as many as are resident
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_move_fused, 256, BULK_CHUNK);
    if (const char* e = getenv("TA_MOVE_CTAS_PER_SM"))   // A/B aid: fewer resident copy CTAs
      per_sm = std::max(1, std::min(per_sm, atoi(e)));
    x->move_grid = (sms * per_sm) & ~1;
    if (x->move_grid < 2) d.fused = 0;
    // k_close: CTA 0 assembles the records while one 1024-thread CTA per 1024 slots
    // finalizes (at least R CTAs: CTA r plans replica r's compaction), at most one per SM
    const int want = (cfg->max_programs + CTA - 1) / CTA + 1;
    x->close_grid = std::min(std::max(want, cfg->n_replicas), std::max(sms, cfg->n_replicas));
  }
  if (d.multi && cfg->replicas_here != 1) {
    fprintf(stderr, "ta_init_pool: multi-process mode needs replicas_here == 1\n");
    delete x;
    return TA_E_INVAL;
  }
  // mailbox epochs [0, 264) and, one process per GPU, the local replica's eviction
  // flags at kEvpOffset: one IPC handle shares both with the peers
  const size_t mbox_bytes = kEvpOffset + (size_t)cfg->hbm_blocks * sizeof(u32);
  if (cudaMalloc(&x->mbox_alloc, mbox_bytes) != cudaSuccess ||
      cudaMemset(x->mbox_alloc, 0, mbox_bytes) != cudaSuccess) {
    delete x;
    return TA_E_CUDA;
  }
  d.mbox = (ull*)x->mbox_alloc;
  d.epoch = d.mbox + TA_MAX_REPLICAS;
  if (d.multi) d.evp = (u32*)((char*)x->mbox_alloc + kEvpOffset);
  size_t dev_bytes = carve(cfg, nullptr, nullptr);
  cudaError_t e = cudaMemsetAsync(bufs->dev_workspace, 0, dev_bytes, x->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(d.loc, 0xFF, (size_t)d.N * d.MAXBP * sizeof(u32), x->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(d.dirty, 1, (size_t)d.N, x->stream);   // first pass counts every row
  if (e == cudaSuccess) { k_init<<<148, 256, 0, x->stream>>>(d); e = cudaGetLastError(); }

  // planner kernels: small sorts and staged lists in dynamic shared memory
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_pause, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PLAN_DSMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_restore, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PLAN_DSMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_pause_restore, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PLAN_DSMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_plan<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PLAN_DSMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_plan<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PLAN_DSMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_ev_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PLAN_DSMEM);
  if (e == cudaSuccess && FP_DSMEM > 48 * 1024) e = cudaFuncSetAttribute(k_tick_front, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FP_DSMEM);
  if (e == cudaSuccess && FP_DSMEM > 48 * 1024) e = cudaFuncSetAttribute(k_footprint, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FP_DSMEM);
  if (e == cudaSuccess) e = cudaStreamSynchronize(x->stream);
  if (e != cudaSuccess) {
    fprintf(stderr, "ta_init_pool: %s\n", cudaGetErrorString(e));
    cudaFree(x->mbox_alloc);
    delete x;
    return TA_E_CUDA;
  }
  if (x->timing)
    for (int i = 0; i < 10; ++i) cudaEventCreate(&x->ev[i]);
  x->probes = x->timing && getenv("TA_GAP_PROBES") != nullptr;
  x->no_events = getenv("TA_NO_EVENTS") != nullptr;
  *out = x;
  return TA_OK;
}

ta_status ta_load_trace(ta_ctx* ctx, const ta_trace_view* t) {
  if (ta_status s = check_ctx(ctx)) return s;
  if (!t) return TA_E_INVAL;
  if (ctx->d.api_mode) FAIL(ctx, TA_E_STATE, "ta_load_trace: context is not in trace mode");
  if (t->n_slots < 0 || t->n_slots > ctx->d.N) FAIL(ctx, TA_E_INVAL, "n_slots %d > max_programs", t->n_slots);
  if (t->n_initial < 0 || t->n_initial > t->n_slots) FAIL(ctx, TA_E_INVAL, "bad n_initial");
  const u32 total = t->n_slots ? t->turn_off[t->n_slots] : 0;
  if (total > (u32)ctx->cfg.max_trace_turns) FAIL(ctx, TA_E_INVAL, "trace has %u turns > max_trace_turns", total);
  for (int p = 0; p < t->n_slots; ++p) {
    if (t->turn_off[p + 1] <= t->turn_off[p]) FAIL(ctx, TA_E_INVAL, "slot %d has no turns", p);
    const u8 k = t->prefix_id ? t->prefix_id[p] : (ctx->d.K ? 0 : KP_NONE);
    if (k != KP_NONE && (int)k >= ctx->d.K) FAIL(ctx, TA_E_INVAL, "slot %d: prefix_id %u >= n_prefixes", p, k);
    if (k != KP_NONE && (u64)t->p0[p] < (u64)ctx->d.sbk[k] * (u64)ctx->d.bt)
      FAIL(ctx, TA_E_INVAL, "slot %d: prompt shorter than its shared prefix", p);
    u64 ctx_max = t->p0[p];
    for (u32 q = t->turn_off[p]; q < t->turn_off[p + 1]; ++q) ctx_max += (u64)t->g[q] + t->o[q];
    if ((ctx_max + ctx->d.bt - 1) / ctx->d.bt > (u64)ctx->d.MAXB)
      FAIL(ctx, TA_E_INVAL, "slot %d reaches %llu tokens > max_blocks_per_program", p, (unsigned long long)ctx_max);
  }
  cudaStream_t s = ctx->stream;
  Dev& d = ctx->d;
  CK(ctx, cudaMemcpyAsync(d.t_uid, t->uid, sizeof(u32) * t->n_slots, cudaMemcpyHostToDevice, s));
  CK(ctx, cudaMemcpyAsync(d.t_p0, t->p0, sizeof(u32) * t->n_slots, cudaMemcpyHostToDevice, s));
  CK(ctx, cudaMemcpyAsync(d.t_off, t->turn_off, sizeof(u32) * (t->n_slots + 1), cudaMemcpyHostToDevice, s));
  CK(ctx, cudaMemcpyAsync(d.t_g, t->g, sizeof(u32) * total, cudaMemcpyHostToDevice, s));
  CK(ctx, cudaMemcpyAsync(d.t_d, t->d_ms, sizeof(u32) * total, cudaMemcpyHostToDevice, s));
  CK(ctx, cudaMemcpyAsync(d.t_o, t->o, sizeof(u32) * total, cudaMemcpyHostToDevice, s));
  if (t->prefix_id) CK(ctx, cudaMemcpyAsync(d.t_kp, t->prefix_id, t->n_slots, cudaMemcpyHostToDevice, s));
  CK(ctx, cudaStreamSynchronize(s));
  d.n_slots = t->n_slots;
  d.n_initial = t->n_initial;
  if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
  ctx->trace_loaded = true;
  return TA_OK;
}

// One tick on the context stream: the captured CUDA graph (built on first use; the
// same kernels in both modes, API-mode ones reading the batch size on the device), or
// kernel by kernel with TA_F_NO_GRAPH.
static cudaError_t run_tick(ta_ctx* ctx) {
  cudaStream_t s = ctx->stream;
  if (ctx->cfg.flags & TA_F_NO_GRAPH) return launch_tick(ctx, 0);
  if (!ctx->graph) {
    cudaGraph_t g;
    cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return e;
    cudaError_t le = launch_tick(ctx, 0);
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (le != cudaSuccess) return le;
    if (ce != cudaSuccess) return ce;
    e = cudaGraphInstantiate(&ctx->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return e;
  }
  return cudaGraphLaunch(ctx->graph, s);
}

ta_status ta_sched_step(ta_ctx* ctx, int64_t now_ms, const ta_event* ev, int32_t n_ev, ta_decision* out,
                        int32_t out_cap, int32_t* n_out) {
  if (ta_status s = check_ctx(ctx)) return s;
  Dev& d = ctx->d;
  cudaStream_t s = ctx->stream;
  if (n_ev < 0 || (n_ev > 0 && !ev) || out_cap < 0) FAIL(ctx, TA_E_INVAL, "bad event/output arguments");
  if (ta_status ps = check_peers(ctx)) return ps;
  if (!d.api_mode) {
    if (n_ev) FAIL(ctx, TA_E_STATE, "events passed in trace mode");
    if (!ctx->trace_loaded) FAIL(ctx, TA_E_STATE, "no trace loaded");
    if (now_ms >= 0) {
      // must equal tick * delta_t: read the device tick counter
      CK(ctx, cudaMemcpyAsync(ctx->h.scal, &d.ctr->tick, sizeof(i64), cudaMemcpyDeviceToHost, s));
      CK(ctx, cudaStreamSynchronize(s));
      if (now_ms != ctx->h.scal[0] * d.dt) FAIL(ctx, TA_E_INVAL, "now_ms %lld != tick*delta_t", (long long)now_ms);
    }
    CK(ctx, run_tick(ctx));
  } else {
    if (now_ms < 0 || now_ms > (int64_t)AS_MAX) FAIL(ctx, TA_E_INVAL, "API mode needs 0 <= now_ms < 2^40");
    if ((size_t)n_ev > ev_capacity(&ctx->cfg))
      FAIL(ctx, TA_E_INVAL, "at most %zu events per tick", ev_capacity(&ctx->cfg));
    // the batch and its header go to the device; validation, application and the tick
    // run as one graph; a rejected batch makes every later kernel return at once
    if (n_ev) memcpy(ctx->h.ev, ev, sizeof(ta_event) * n_ev);
    ctx->h.scal[0] = now_ms;
    *(i32*)(ctx->h.scal + 1) = n_ev;
    if (n_ev) CK(ctx, cudaMemcpyAsync(ctx->ev_dev, ctx->h.ev, sizeof(ta_event) * n_ev, cudaMemcpyHostToDevice, s));
    CK(ctx, cudaMemcpyAsync(&d.ctr->now_ms, ctx->h.scal, sizeof(i64), cudaMemcpyHostToDevice, s));
    CK(ctx, cudaMemcpyAsync(&d.ctr->n_events, ctx->h.scal + 1, sizeof(i32), cudaMemcpyHostToDevice, s));
    CK(ctx, run_tick(ctx));
    CK(ctx, cudaMemcpyAsync(ctx->h.scal + 2, &d.ctr->err, sizeof(i32), cudaMemcpyDeviceToHost, s));
    CK(ctx, cudaStreamSynchronize(s));
    const int verr = *(i32*)(ctx->h.scal + 2);
    if (verr != TA_OK) FAIL(ctx, (ta_status)verr, "event batch rejected (first illegal event); nothing applied");
  }
  if (!out && !n_out) return TA_OK;
  CK(ctx, cudaStreamSynchronize(s));
  if (d.multi)
    if (ta_status de = check_device_err(ctx)) return de;
  return copy_out(ctx, out, out_cap, n_out);
}

ta_status ta_stats(ta_ctx* ctx, ta_stats_t* out) {
  if (ta_status s = check_ctx(ctx)) return s;
  if (!out) return TA_E_INVAL;
  Dev& d = ctx->d;
  memset(out, 0, sizeof(*out));
  std::vector<ull> st(ST_N);
  std::vector<ull> L(d.R);
  std::vector<u32> hf((size_t)d.R * d.NBW), sf((size_t)d.R * (d.NHW ? d.NHW : 1));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  CK(ctx, cudaMemcpy(st.data(), d.stats, sizeof(ull) * ST_N, cudaMemcpyDeviceToHost));
  CK(ctx, cudaMemcpy(L.data(), d.L, sizeof(ull) * d.R, cudaMemcpyDeviceToHost));
  CK(ctx, cudaMemcpy(hf.data(), d.hbm_free, sizeof(u32) * hf.size(), cudaMemcpyDeviceToHost));
  if (d.NHW) CK(ctx, cudaMemcpy(sf.data(), d.host_free, sizeof(u32) * (size_t)d.R * d.NHW, cudaMemcpyDeviceToHost));
  memcpy(out, st.data(), sizeof(ull) * ST_BASE_N);
  out->cost_decode = st[ST_COST_DECODE];
  out->cost_prefill = st[ST_COST_PREFILL];
  out->cost_recompute = st[ST_COST_RECOMPUTE];
  out->cost_unused = st[ST_COST_UNUSED];
  out->cost_caching = st[ST_COST_CACHING];
  out->unused_bound_checks = st[ST_UNUSED_CHECKS];
  out->unused_bound_violations = st[ST_UNUSED_VIOL];
  out->overshoot_blocks = st[ST_OVERSHOOT];
  out->overshoot_max_blocks = st[ST_OVERSHOOT_MAX];
  out->prefix_blocks = st[ST_PREFIX_BLOCKS];
  for (int r = 0; r < d.R; ++r) {
    out->L[r] = L[r];
    u64 f = 0, g = 0;
    for (int w = 0; w < d.NBW; ++w) f += __builtin_popcount(hf[(size_t)r * d.NBW + w]);
    for (int w = 0; w < d.NHW; ++w) g += __builtin_popcount(sf[(size_t)r * d.NHW + w]);
    out->hbm_used[r] = d.NB - f;
    out->host_used[r] = d.NH - g;
  }
  out->block_bytes = ctx->block_bytes;
  return TA_OK;
}

ta_status ta_set_copy_bulk(ta_ctx* ctx, int32_t on) {
  if (ta_status s = check_ctx(ctx)) return s;
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  if (on) ctx->d.flags |= TA_F_COPY_BULK; else ctx->d.flags &= ~(u32)TA_F_COPY_BULK;
  if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }   // params changed
  return TA_OK;
}

ta_status ta_last_tick(ta_ctx* ctx, ta_tick_info* out) {
  if (ta_status s = check_ctx(ctx)) return s;
  if (!out) return TA_E_INVAL;
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  *out = *ctx->h.tick_info;
  return TA_OK;
}

ta_status ta_phase_times(ta_ctx* ctx, float* us, int32_t n) {
  if (ta_status s = check_ctx(ctx)) return s;
  if (!ctx->timing) FAIL(ctx, TA_E_STATE, "context created without TA_F_TIMING");
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < n && i < 9; ++i) {
    float ms = 0;
    CK(ctx, cudaEventElapsedTime(&ms, ctx->ev[i], ctx->ev[i + 1]));
    us[i] = ms * 1000.f;
  }
  return TA_OK;
}

ta_status ta_debug_phase_stamps(ta_ctx* ctx, uint64_t* out, int32_t n) {
  if (ta_status s = check_ctx(ctx)) return s;
  if (!ctx->timing) FAIL(ctx, TA_E_STATE, "context created without TA_F_TIMING");
  if (!out || n < 0 || n > 256) FAIL(ctx, TA_E_INVAL, "bad stamp buffer");
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  CK(ctx, cudaMemcpy(out, ctx->d.pst, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  return TA_OK;
}

ta_status ta_debug_counters(ta_ctx* ctx, uint64_t* out, int32_t n) {
  if (ta_status s = check_ctx(ctx)) return s;
  if (!out || n < 0 || n > DBG_N) FAIL(ctx, TA_E_INVAL, "bad counter buffer");
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  CK(ctx, cudaMemcpy(out, ctx->d.dbg, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  return TA_OK;
}

ta_status ta_move_blocks(ta_ctx* ctx, int32_t kind, int32_t src_r, int32_t dst_r, const uint32_t* src_blocks,
                         const uint32_t* dst_blocks, int32_t n) {
  if (ta_status s = check_ctx(ctx)) return s;
  Dev& d = ctx->d;
  if (n < 0 || (n > 0 && (!src_blocks || !dst_blocks))) FAIL(ctx, TA_E_INVAL, "bad block lists");
  if (src_r < 0 || src_r >= d.R) FAIL(ctx, TA_E_INVAL, "bad src replica");
  if (kind == TA_MOVE_D2D || kind == TA_MOVE_D2H) dst_r = src_r;
  if (dst_r < 0 || dst_r >= d.R) FAIL(ctx, TA_E_INVAL, "bad dst replica");
  const char* sb = nullptr;
  char* db = nullptr;
  i64 snb = d.NB, dnb = d.NB;
  switch (kind) {
    case TA_MOVE_D2D: case TA_MOVE_P2P: sb = d.hbm[src_r]; db = d.hbm[dst_r]; break;
    case TA_MOVE_D2H: sb = d.hbm[src_r]; db = d.host[src_r]; dnb = d.NH; break;
    case TA_MOVE_H2D: sb = d.host[src_r]; db = d.hbm[dst_r]; snb = d.NH; break;
    default: FAIL(ctx, TA_E_INVAL, "bad move kind %d", kind);
  }
  if (!sb || !db) FAIL(ctx, TA_E_INVAL, "pool not addressable from this process");
  if (n == 0) return TA_OK;
  k_move<<<kCopyGrid, 256, csm(d), ctx->stream>>>(d, sb, snb, db, dnb, src_blocks, dst_blocks, n);
  CK(ctx, cudaGetLastError());
  return TA_OK;
}

ta_status ta_verify_content(ta_ctx* ctx, uint64_t* mismatched, uint64_t* checked) {
  if (ta_status s = check_ctx(ctx)) return s;
  Dev& d = ctx->d;
  CK(ctx, cudaMemsetAsync(d.verify, 0, 2 * sizeof(ull), ctx->stream));
  k_verify<<<148 * 8, 256, 0, ctx->stream>>>(d, 0);
  if (d.NH > 0) k_verify<<<148 * 8, 256, 0, ctx->stream>>>(d, 1);
  CK(ctx, cudaGetLastError());
  ull v[2];
  CK(ctx, cudaMemcpyAsync(v, d.verify, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  if (mismatched) *mismatched = v[0];
  if (checked) *checked = v[1];
  return TA_OK;
}

ta_status ta_debug_state(ta_ctx* ctx, int32_t dir, const ta_state_view* v) {
  if (ta_status s = check_ctx(ctx)) return s;
  if (!v || (dir != 0 && dir != 1)) return TA_E_INVAL;
  Dev& d = ctx->d;
  cudaStream_t s = ctx->stream;
  CK(ctx, cudaStreamSynchronize(s));
  const size_t N = d.N, R = d.R;
  auto mv = [&](void* host, void* dev, size_t bytes) -> cudaError_t {
    if (!host) return cudaSuccess;
    return dir == 0 ? cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost)
                    : cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice);
  };
  CK(ctx, mv(v->uid, d.uid, N * 4)); CK(ctx, mv(v->c, d.c, N * 4)); CK(ctx, mv(v->c_kv, d.c_kv, N * 4));
  CK(ctx, mv(v->paused_since, d.paused_since, N * 4)); CK(ctx, mv(v->step_count, d.step_count, N * 4));
  CK(ctx, mv(v->turn, d.turn, N * 4)); CK(ctx, mv(v->gen_done, d.gen_done, N * 4));
  CK(ctx, mv(v->status, d.status, N)); CK(ctx, mv(v->phase, d.phase, N)); CK(ctx, mv(v->satisfied, d.satisfied, N));
  CK(ctx, mv(v->placement, d.placement, N)); CK(ctx, mv(v->home, d.home, N));
  CK(ctx, mv(v->acting_since, d.acting_since, N * 8)); CK(ctx, mv(v->tool_return, d.tool_return, N * 8));
  if (v->loc) {
    size_t w = (size_t)d.MAXB * 4, sp = (size_t)d.MAXBP * 4;
    if (dir == 0) CK(ctx, cudaMemcpy2D(v->loc, w, d.loc, sp, w, N, cudaMemcpyDeviceToHost));
    else CK(ctx, cudaMemcpy2D(d.loc, sp, v->loc, w, w, N, cudaMemcpyHostToDevice));
  }
  if (dir == 1) {                          // uploaded state: the next footprint pass recounts every row
    CK(ctx, cudaMemset(d.dirty, 1, N));
  }
  CK(ctx, mv(v->hbm_free, d.hbm_free, R * d.NBW * 4));
  if (d.NHW) CK(ctx, mv(v->host_free, d.host_free, R * d.NHW * 4));
  CK(ctx, mv(v->owner_hbm, d.owner_hbm, R * d.NB * 4));
  if (d.NH) CK(ctx, mv(v->owner_host, d.owner_host, R * d.NH * 4));
  CK(ctx, mv(v->L, d.L, R * 8));
  if (dir == 0) {
    CK(ctx, mv(v->nb, d.nb, N * 4)); CK(ctx, mv(v->n_hbm, d.n_hbm, N * 4));
    CK(ctx, mv(v->n_host, d.n_host, N * 4)); CK(ctx, mv(v->prefix_hbm, d.prefix_hbm, N * 4));
    CK(ctx, mv(v->contrib, d.contrib, N * 4));
  }
  {                                        // NEXT-3 prompts (A51)
    const size_t RK = (size_t)R * (d.K ? d.K : 1);
    CK(ctx, mv(v->prefix_id, d.kp, N));
    CK(ctx, mv(v->prefix_ref, d.pref, RK * 4));
    CK(ctx, mv(v->prefix_blk, d.pblk, RK * d.SBM * 4));
    if (dir == 1 && v->prefix_blk && v->prefix_ref) {   // the prompt-block bitmap follows the upload
      std::vector<u32> ref(RK), blk(RK * d.SBM), fix((size_t)R * d.NBW, 0u);
      memcpy(ref.data(), v->prefix_ref, RK * 4);
      memcpy(blk.data(), v->prefix_blk, RK * d.SBM * 4);
      for (size_t r = 0; r < R; ++r)
        for (int k = 0; k < d.K; ++k)
          if (ref[r * d.K + k])
            for (u32 j = 0; j < d.sbk[k]; ++j) {
              const u32 b = blk[(r * d.K + k) * d.SBM + j];
              fix[r * d.NBW + (b >> 5)] |= 1u << (b & 31);
            }
      CK(ctx, cudaMemcpy(d.pfix, fix.data(), fix.size() * 4, cudaMemcpyHostToDevice));
    }
  }
  if (v->scalars) {
    Ctr c;
    CK(ctx, cudaMemcpy(&c, d.ctr, sizeof(Ctr), cudaMemcpyDeviceToHost));
    if (dir == 0) {
      v->scalars[0] = c.tick; v->scalars[1] = c.next_arrival; v->scalars[2] = c.T; v->scalars[3] = 0;
    } else {
      c.tick = v->scalars[0]; c.next_arrival = v->scalars[1]; c.T = v->scalars[2];
      CK(ctx, cudaMemcpy(d.ctr, &c, sizeof(Ctr), cudaMemcpyHostToDevice));
    }
  }
  return TA_OK;
}

// Verbs: enqueue, synchronize, read the device-side status, return the decisions.
static ta_status verb_finish(ta_ctx* ctx, const char* what, ta_decision* out, int32_t out_cap, int32_t* n_out) {
  Dev& d = ctx->d;
  CK(ctx, cudaGetLastError());
  CK(ctx, cudaMemcpyAsync(ctx->h.scal + 1, &d.ctr->err, sizeof(i32), cudaMemcpyDeviceToHost, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  int err = (int)*(i32*)(ctx->h.scal + 1);
  if (n_out) *n_out = 0;
  if (err != TA_OK) FAIL(ctx, (ta_status)err, "%s rejected", what);
  return copy_out(ctx, out, out_cap, n_out);
}

ta_status ta_pause(ta_ctx* ctx, uint32_t pid, uint32_t mode, ta_decision* out, int32_t out_cap, int32_t* n_out) {
  if (ta_status s = check_ctx(ctx)) return s;
  if (mode > TA_PAUSE_DROP || out_cap < 0) FAIL(ctx, TA_E_INVAL, "bad pause mode / out_cap");
  if (ta_status ps = check_peers(ctx)) return ps;
  Dev& d = ctx->d;
  cudaStream_t s = ctx->stream;
  k_verb_reset<<<1, 32, 0, s>>>(d);
  k_verb_pause<<<1, CTA, 0, s>>>(d, pid, mode);
  launch_movement(ctx, ctx->stream);
  launch_coop(k_close<1>, ctx->close_grid, 0, s, (Dev)d);
  return verb_finish(ctx, "ta_pause", out, out_cap, n_out);
}

static ta_status activate(ta_ctx* ctx, uint32_t pid, int32_t replica, int migrate, ta_decision* out,
                          int32_t out_cap, int32_t* n_out) {
  if (ta_status s = check_ctx(ctx)) return s;
  if (out_cap < 0) FAIL(ctx, TA_E_INVAL, "bad out_cap");
  if (ta_status ps = check_peers(ctx)) return ps;
  Dev& d = ctx->d;
  cudaStream_t s = ctx->stream;
  const int N = d.N;
  k_verb_reset<<<1, 32, 0, s>>>(d);
  k_footprint<<<FP_GRID(N), FP_BLOCK, FP_DSMEM, s>>>(d, 1);
  k_verb_admit<<<1, 32, 0, s>>>(d, pid, replica, migrate);
  k_plan<1><<<d.R * PLAN_CL, CTA, PLAN_DSMEM, s>>>(d);
  k_verb_commit<<<1, 32, 0, s>>>(d, migrate);
  launch_movement(ctx, ctx->stream);
  launch_coop(k_close<1>, ctx->close_grid, 0, s, (Dev)d);
  return verb_finish(ctx, migrate ? "ta_migrate" : "ta_resume", out, out_cap, n_out);
}

ta_status ta_set_health(ta_ctx* ctx, int32_t replica, int32_t healthy, ta_decision* out, int32_t out_cap,
                        int32_t* n_out) {
  if (ta_status s = check_ctx(ctx)) return s;
  Dev& d = ctx->d;
  if (replica < 0 || replica >= d.R || out_cap < 0) FAIL(ctx, TA_E_INVAL, "bad replica %d / out_cap", replica);
  if (ta_status ps = check_peers(ctx)) return ps;
  if (n_out) *n_out = 0;
  const u32 bit = 1u << replica;
  if (((d.healthy & bit) != 0) == (healthy != 0)) return TA_OK;    // no change, no decisions
  // watermarks and the health mask are kernel parameters: the tick graph is re-captured
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
  if (healthy) {                         // back in service, empty
    d.healthy |= bit;
    d.cap_max[replica] = (i64)(((u64)ctx->cfg.lambda_max_q16 * (u64)d.NB) >> 16);
    d.cap_min[replica] = (i64)(((u64)ctx->cfg.lambda_min_q16 * (u64)d.NB) >> 16);
    return TA_OK;
  }
  d.healthy &= ~bit;
  d.cap_max[replica] = d.cap_min[replica] = 0;
  cudaStream_t s = ctx->stream;
  k_verb_reset<<<1, 32, 0, s>>>(d);
  k_verb_health<<<1, CTA, 0, s>>>(d, replica);
  launch_coop(k_close<1>, ctx->close_grid, 0, s, (Dev)d);
  return verb_finish(ctx, "ta_set_health", out, out_cap, n_out);
}

ta_status ta_resume(ta_ctx* ctx, uint32_t pid, int32_t replica, ta_decision* out, int32_t out_cap, int32_t* n_out) {
  return activate(ctx, pid, replica, 0, out, out_cap, n_out);
}

ta_status ta_migrate(ta_ctx* ctx, uint32_t pid, int32_t dst, ta_decision* out, int32_t out_cap, int32_t* n_out) {
  return activate(ctx, pid, dst, 1, out, out_cap, n_out);
}

// handle layout: [0,64) pool IPC handle | [64,72) pool offset in its allocation |
// [72,136) mailbox IPC handle | [136,192) reserved
ta_status ta_export_pool_handle(ta_ctx* ctx, void* handle) {
  if (ta_status s = check_ctx(ctx)) return s;
  if (!handle || !ctx->d.multi) FAIL(ctx, TA_E_INVAL, "export needs a multi-process context");
  char* out = (char*)handle;
  memset(out, 0, TA_HANDLE_BYTES);
  void* pool = ctx->bufs.hbm_pool[ctx->cfg.first_replica];
  CUdeviceptr base = 0;
  size_t size = 0;
  // driver entry point through the runtime (no link-time libcuda dependency)
  typedef CUresult (*range_fn)(CUdeviceptr*, size_t*, CUdeviceptr);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
      ((range_fn)fn)(&base, &size, (CUdeviceptr)pool) != CUDA_SUCCESS)
    { ctx->poisoned = TA_E_PEER; FAIL(ctx, TA_E_PEER, "cuMemGetAddressRange failed"); }
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
  if (e == cudaSuccess) {
    memcpy(out, &h, 64);
    u64 off = (u64)((CUdeviceptr)pool - base);
    memcpy(out + 64, &off, 8);
    e = cudaIpcGetMemHandle(&h, ctx->mbox_alloc);
    memcpy(out + 72, &h, 64);
  }
  if (e != cudaSuccess) { ctx->poisoned = TA_E_PEER; FAIL(ctx, TA_E_PEER, "%s", cudaGetErrorString(e)); }
  return TA_OK;
}

ta_status ta_import_peer_pool(ta_ctx* ctx, int32_t replica, const void* handle) {
  if (ta_status s = check_ctx(ctx)) return s;
  if (!handle || replica < 0 || replica >= ctx->d.R || replica == ctx->d.rank || !ctx->d.multi)
    FAIL(ctx, TA_E_INVAL, "bad peer replica %d", replica);
  const char* in = (const char*)handle;
  cudaIpcMemHandle_t h;
  u64 off;
  memcpy(&h, in, 64);
  memcpy(&off, in + 64, 8);
  void* p = nullptr;
  void* m = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e == cudaSuccess) {
    memcpy(&h, in + 72, 64);
    e = cudaIpcOpenMemHandle(&m, h, cudaIpcMemLazyEnablePeerAccess);
  }
  if (e != cudaSuccess) { ctx->poisoned = TA_E_PEER; FAIL(ctx, TA_E_PEER, "%s", cudaGetErrorString(e)); }
  ctx->peer_base[replica] = p;
  ctx->peer_mbox[replica] = m;
  ctx->bufs.hbm_pool[replica] = (char*)p + off;
  ctx->d.hbm[replica] = (char*)p + off;
  ctx->d.mbox_peer[replica] = (ull*)m;
  ctx->d.evp_peer[replica] = (u32*)((char*)m + kEvpOffset);
  if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
  return TA_OK;
}

ta_status ta_destroy(ta_ctx* ctx) {
  if (!ctx) return TA_E_INVAL;
  cudaStreamSynchronize(ctx->stream);
  if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
  for (int i = 0; i < 10; ++i)
    if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
  for (int r = 0; r < TA_MAX_REPLICAS; ++r) {
    if (ctx->peer_base[r]) cudaIpcCloseMemHandle(ctx->peer_base[r]);
    if (ctx->peer_mbox[r]) cudaIpcCloseMemHandle(ctx->peer_mbox[r]);
  }
  if (ctx->mbox_alloc) cudaFree(ctx->mbox_alloc);
  delete ctx;
  return TA_OK;
}

const char* ta_last_error(const ta_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

}  // extern "C"
