/*
 * ta.h — C ABI of the B200-native ThunderAgent KV-manager hot path (libta.so).
 *
 * The library implements, in hand-written sm_100a CUDA, the per-tick scheduler
 * step of ThunderAgent's program-aware KV-cache manager (arXiv 2602.13692,
 * PAPER.md §4.3) over all live agentic programs, and the paged-KV
 * block movement its decisions trigger (HBM <-> pinned host, HBM -> peer HBM,
 * HBM -> HBM compaction).  Policy semantics are defined step by step in
 * DESIGN.md §2 (readings A1-A27).
 *
 * Conventions (apply to every entry point):
 *  - Every call returns ta_status; TA_OK == 0.  No exceptions cross the ABI.
 *    A failed call leaves the context unchanged, except TA_E_CUDA / TA_E_PEER,
 *    which poison the context (every later call returns the same code).
 *    ta_last_error() returns a human-readable reason for the last failure.
 *  - Ownership: the CALLER allocates and owns every buffer (KV pools, host
 *    tiers, workspaces) and the CUDA stream, and keeps them alive until
 *    ta_destroy().  The library never frees caller memory.
 *  - Calls on one context are serialized by the caller (single writer,
 *    SPEC.md:82, 283).  All device work is stream-ordered on the context stream.
 *  - Multi-replica: replica state (program table, block tables, bitmaps) is
 *    replicated on every rank; each rank holds the KV pools of
 *    `replicas_here` replicas starting at `first_replica`.  In multi-process
 *    mode (one replica per process) ta_sched_step, ta_pause, ta_resume,
 *    ta_migrate and ta_set_health are COLLECTIVE: every rank makes the same
 *    call with the same arguments, in the same order (they change replicated
 *    state and run the cross-process device barriers of the movement step; a
 *    call made on one rank only waits ~15 s at the barrier and returns
 *    TA_E_PEER).  Replicas marked unhealthy (ta_set_health) are skipped by the
 *    barriers, so the surviving ranks keep ticking after a failover.
 *  - Block-table entry encoding (u32): TA_LOC_NONE = no KV; bit 31 clear =
 *    HBM block index on the program's home replica; bit 31 set = slot index in
 *    the home replica's pinned host tier.
 */
#ifndef TA_H_
#define TA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TA_ABI_VERSION 3
#define TA_MAX_REPLICAS 32
#define TA_MAX_PREFIXES 8          /* shared system prompts (NEXT-3) */
#define TA_PROMPT_UID 0xFF0000u    /* KV content identity of prompt k: TA_PROMPT_UID + k */
#define TA_OWNER_PROMPT 0xF8000000u /* owner_hbm of prompt k's block j: TA_OWNER_PROMPT | k << 20 | j */
#define TA_LOC_NONE 0xFFFFFFFFu
#define TA_LOC_HOST 0x80000000u

typedef struct ta_ctx ta_ctx;

typedef enum {
  TA_OK = 0,
  TA_E_INVAL = 1,              /* bad argument / config / time */
  TA_E_NOMEM = 2,              /* workspace too small */
  TA_E_DUP_ID = 3,             /* ARRIVE on a used pid */
  TA_E_UNKNOWN_PROGRAM = 4,    /* pid never arrived */
  TA_E_ILLEGAL_TRANSITION = 5, /* event/verb not legal in the program's status */
  TA_E_CAPACITY = 6,           /* restore/migrate would exceed lambda_max*C or cannot be fetched */
  TA_E_TRUNCATED = 7,          /* more decisions than out_cap; *n_out holds the needed count */
  TA_E_CUDA = 8,               /* CUDA error (context poisoned) */
  TA_E_PEER = 9,               /* peer / IPC error (context poisoned) */
  TA_E_STATE = 10              /* call not valid in this mode (e.g. events in trace mode) */
} ta_status;

/* Program status s (PAPER.md:670-676 ProgramStatus, plus UNARRIVED for unused slots). */
enum { TA_UNARRIVED = 0, TA_PAUSED = 1, TA_REASONING = 2, TA_ACTING = 3, TA_STOPPED = 4 };
/* Execution phase tau. */
enum { TA_PHASE_R = 0, TA_PHASE_A = 1 };
/* Decision kinds, emitted in canonical order PAUSE, RESTORE, EVICT, FETCH/STALL, COMPACT. */
enum { TA_D_PAUSE = 1, TA_D_RESTORE = 2, TA_D_EVICT = 3, TA_D_FETCH = 4, TA_D_STALL = 5,
       TA_D_MIGRATE = 6, TA_D_COMPACT = 7 };
/* API-mode events (the three-change protocol). */
enum { TA_EV_ARRIVE = 1, TA_EV_DECODE = 2, TA_EV_TOOL_CALL = 3, TA_EV_TOOL_RESULT = 4,
       TA_EV_RELEASE = 5 };
/* ta_pause modes: LAZY is the paper's Pause (KV becomes evictable). */
enum { TA_PAUSE_LAZY = 0, TA_PAUSE_OFFLOAD = 1, TA_PAUSE_DROP = 2 };
/* ta_config.flags */
enum {
  TA_F_TRACE_MODE = 1u << 0,   /* program scripts come from ta_load_trace (closed-loop) */
  TA_F_FILL = 1u << 1,         /* write KV content for new/recomputed tokens (engine stand-in) */
  TA_F_NO_GRAPH = 1u << 2,     /* launch the tick kernel by kernel instead of a CUDA graph */
  TA_F_TIMING = 1u << 3,       /* record per-phase CUDA events (graph event-record nodes) */
  TA_F_COPY_BULK = 1u << 4,    /* HBM->HBM copies via cp.async.bulk (TMA) instead of LDG/STG.128 */
  TA_F_NO_FUSE = 1u << 5,      /* single process: separate evict / fetch / fill kernels (A/B aid) */
  TA_F_PINNED_ROUTING = 1u << 6, /* baseline (NEXT-2): program p bound to replica p mod R, per-replica
                                  queues instead of the global queue (reading A45) */
  TA_F_REQUEST_AWARE = 1u << 7, /* baseline (NEXT-2): stateless request-level engine -- running
                                  requests preempted latest program first, FCFS waiting queue, LRU
                                  eviction of idle caches; pass an all-zero decay table (A46) */
  TA_F_SMALL_PATHS = 1u << 8,   /* test aid: lower the size thresholds of the shared-memory fast
                                  paths (CTA sort 4096 -> 64, rank sort 512 -> 16, staged planner
                                  lists 4096 / 8192 / 1024 -> 8 / 8 / 4, candidate slot lists in
                                  shared memory 12288 / 8192 -> 8, restore chunks 32..4096 -> 4..64, restore buckets <= 8) so that
                                  small runs take the code paths of full-size runs.  Results are
                                  identical; only the speed differs. */
  TA_F_JITTER = 1u << 10,       /* test aid (development build only): every CTA of the tick kernels
                                  sleeps a pseudo-random 0-20 us at kernel entry and after every
                                  grid / cluster barrier, so that a missing barrier between CTAs
                                  shows up as a wrong result.  Results are identical. */
  TA_F_FULL_SCAN = 1u << 11,    /* test aid (development build only): the footprint pass counts
                                  every live row each tick instead of only the rows written
                                  since the previous pass (the clean-row rule).
                                  Results are identical; tests compare the two. */
  TA_F_DECIDE_ONLY = 1u << 9    /* measurement aid: the tick runs steps 0-5 and 7 (decisions,
                                  block tables, free sets, statistics) but issues no block copy
                                  (no step 6, no compaction copies): the pools' bytes are not
                                  maintained.  Decisions are identical (none depends on bytes);
                                  it times the decision path alone.  In multi-process mode the
                                  device barriers go too (they order copies only). */
};

typedef struct {
  /* KV shape of one token (BackendState.cache_config) */
  int32_t n_layers, n_kv_heads, head_dim, elem_bytes; /* elem_bytes must be 2 */
  int32_t block_tokens;        /* bt: tokens per KV block (16/32/64; 1 for pins) */
  int32_t layout;              /* 0: layer-major pool[l][kv][NB][bt][H][D]; 1: block-major pool[NB][l][kv][bt][H][D] */
  int32_t n_replicas;          /* R data-parallel replicas (<= TA_MAX_REPLICAS) */
  int32_t replicas_here;       /* replicas whose pools this process holds */
  int32_t first_replica;       /* index of the first of them */
  int32_t max_programs;        /* N program slots */
  int32_t max_blocks_per_program; /* MAXB = ceil(max_ctx / bt) */
  int32_t max_trace_turns;     /* capacity of the trace script arrays */
  int64_t hbm_blocks;          /* NB per replica */
  int64_t host_blocks;         /* NH per replica (0 = no host tier) */
  int64_t delta_t_ms;          /* Delta t of the periodic monitor (reading A1) */
  int64_t decay_unit_ms;       /* time unit of t_q in f(t_q) (reading A2) */
  uint32_t lambda_max_q16;     /* high watermark, 65536 == 1.0; 0 < min <= max <= 65536 */
  uint32_t lambda_min_q16;     /* low watermark */
  uint64_t decay_q32[64];      /* F[k] = floor(f(k) * 2^32), F[0] = 2^32 (eq. 7) */
  int32_t decode_tok_per_s;    /* synthetic engine decode rate (trace mode) */
  int32_t compact_every;       /* two-finger compaction every k ticks; 0 = off */
  uint32_t flags;              /* TA_F_* */
  int32_t prefill_chunk_tokens; /* STP ledger (NEXT-1): chunked-prefill tokens per engine step (>= 1) */
  int32_t prefill_chunk_ms;    /* STP ledger: duration of one chunk step in ms (>= 0) */
  /* NEXT-3, single-prompt form: one shared system prompt of this many tokens used by
   * every program (= n_prefixes 1, prefix_tokens[0]); 0 = off.  See n_prefixes. */
  int32_t shared_prefix_tokens;
  /* NEXT-3 (reading A51; "agentic system prompts are identical across
   * workflows"): K = n_prefixes shared system prompts (one per agent
   * preset), prompt k = the first prefix_tokens[k] tokens of every program that uses it
   * (multiples of block_tokens, below hbm_blocks blocks).  A program's prompt comes from
   * the trace (ta_trace_view.prefix_id) or its ARRIVE event (t_ms = prompt index when
   * K > 1; prompt 0 when K == 1).  Prompt k is stored once per replica: the first
   * program (F_r slot order) that needs it on replica r materializes it -- its first
   * requests get the lowest free blocks, prefilled (content: uid TA_PROMPT_UID + k) --
   * every program homed on r points its first entries at those blocks, a per-replica
   * refcount counts them, and the last one to leave (release, fetch to another replica,
   * replica failure) frees them (at step 0 for releases, step 7 otherwise).  Prompt
   * blocks are never evicted, copied or compacted; need, eviction supply and eviction
   * cover a program's private blocks only; a resumed program counts its prompt tokens
   * as hit, or as miss when it materializes the prompt.  The load (Eq. 7) still counts
   * full contexts.  Every prompt (trace p0, ARRIVE tokens) must cover its shared prefix
   * (else TA_E_INVAL).  0 = use shared_prefix_tokens. */
  int32_t n_prefixes;
  int32_t prefix_tokens[TA_MAX_PREFIXES];
} ta_config;

typedef struct {
  /* Device pointer of replica r's HBM KV pool (NB * block_bytes bytes) for every
   * replica this process can address: local replicas, and peers mapped with
   * ta_import_peer_pool().  NULL for replicas it cannot address. */
  void* hbm_pool[TA_MAX_REPLICAS];
  /* Page-locked host pointer of replica r's host tier (NH * block_bytes bytes),
   * local replicas only; NULL otherwise. */
  void* host_pool[TA_MAX_REPLICAS];
  void* dev_workspace;         /* >= dev_bytes from ta_workspace_bytes, 256-B aligned */
  void* host_workspace;        /* page-locked, >= host_bytes from ta_workspace_bytes */
} ta_buffers;

typedef struct {               /* API-mode event */
  uint32_t kind;               /* TA_EV_* */
  uint32_t pid;                /* program slot */
  uint32_t uid;                /* ARRIVE: program identity used by the KV content */
  uint32_t tokens;             /* ARRIVE: prompt tokens; DECODE: n; TOOL_RESULT: result tokens */
  int64_t t_ms;                /* TOOL_CALL: time the tool call started (0 <= t_ms < 2^40) */
} ta_event;

typedef struct {               /* one scheduling decision (48 bytes) */
  uint32_t kind;               /* TA_D_* */
  uint32_t pid;                /* program slot; 0xFFFFFFFF for COMPACT */
  int32_t src;                 /* PAUSE: replica left; RESTORE/FETCH/STALL: KV home before; EVICT/COMPACT: replica */
  int32_t dst;                 /* RESTORE/MIGRATE/FETCH/STALL: target replica; -1 otherwise */
  uint32_t blocks;             /* EVICT: blocks evicted; FETCH/STALL: blocks needed; COMPACT: blocks moved */
  uint32_t to_host, dropped;   /* EVICT: blocks offloaded to the host tier / dropped */
  uint32_t hit_tok, peer_tok, host_tok, miss_tok; /* FETCH of a resumed program: history by location */
  uint32_t new_tok;            /* FETCH: tokens [c_kv, c) written now */
} ta_decision;

typedef struct {               /* cumulative counters (order fixed) */
  uint64_t ticks, arrivals, stops, pauses, restores, oversized_skips, shortfalls;
  uint64_t evict_blocks, evict_to_host, evict_dropped, fetch_blocks, p2p_blocks, h2d_blocks;
  uint64_t recompute_blocks, new_blocks, compact_blocks, stalls;
  uint64_t hit_tok, peer_tok, host_tok, miss_tok, new_tok, fill_tok;
  uint64_t imbalance_max_blocks, imbalance_last_blocks;   /* max_r used - min_r used */
  uint64_t L[TA_MAX_REPLICAS];          /* effective load after the last restore pass (eq. 7) */
  uint64_t hbm_used[TA_MAX_REPLICAS];   /* HBM blocks in use */
  uint64_t host_used[TA_MAX_REPLICAS];  /* host-tier slots in use */
  uint64_t block_bytes;                 /* bytes per KV block (bytes moved = blocks * block_bytes) */
  /* NEXT-1: STP cost ledger in token-ms (Eq. 2-3; readings A40-A44):
   * for the interval after each tick -- decode: satisfied programs hold c; prefill /
   * recompute: chunked staircases of new tokens / missed history; caching: resident
   * tokens of ACTING and PAUSED programs; unused: cap_max - used blocks while programs
   * wait -- and the Cost_unused < c_min bound of PAPER.md:415 per replica-tick. */
  uint64_t cost_decode, cost_prefill, cost_recompute, cost_unused, cost_caching;
  uint64_t unused_bound_checks, unused_bound_violations;
  /* NEXT-4 guard (reading A50; "context growth ... can trigger memory
   * thrashing mid-execution"): at each pause pass, the excess L_eff - lambda_max*C the
   * periodic monitor found on a replica (blocks), summed over replica-ticks, and its
   * maximum.  Shrinking delta_t_ms to one decode step (1000 / decode rate) bounds it by
   * one step's growth. */
  uint64_t overshoot_blocks, overshoot_max_blocks;
  /* NEXT-3 (reading A51): blocks allocated for shared prompts (a prompt materialized on a
   * replica where no program held it). */
  uint64_t prefix_blocks;
} ta_stats_t;

typedef struct {               /* trace-mode program scripts (tracegen layout; host pointers) */
  int32_t n_slots;             /* <= max_programs */
  int32_t n_initial;           /* slots [0, n_initial) arrive at tick 0; then closed loop */
  const uint32_t* uid;         /* [n_slots] */
  const uint32_t* p0;          /* [n_slots] prompt tokens */
  const uint32_t* turn_off;    /* [n_slots + 1] CSR offsets into g / d_ms / o */
  const uint32_t* g;           /* tokens generated per turn */
  const uint32_t* d_ms;        /* tool latency after the turn */
  const uint32_t* o;           /* tool-result tokens after the turn */
  const uint8_t* prefix_id;    /* [n_slots] shared prompt of each slot (< n_prefixes, 255 = none);
                                  NULL: prompt 0 when there is one, else none */
} ta_trace_view;

typedef struct {               /* host mirror of the device state (parity tests); NULL = skip */
  uint32_t *uid, *c, *c_kv, *paused_since, *step_count, *turn, *gen_done;   /* [N] */
  uint8_t *status, *phase, *satisfied;                                      /* [N] */
  int8_t *placement, *home;                                                 /* [N] */
  int64_t *acting_since, *tool_return;                                      /* [N] */
  uint32_t *loc;              /* [N * MAXB] */
  uint32_t *hbm_free;         /* [R * ceil(NB/32)] bit set = free */
  uint32_t *host_free;        /* [R * ceil(NH/32)] */
  uint32_t *owner_hbm;        /* [R * NB]  pid * MAXB + j of the block's owner (valid if used) */
  uint32_t *owner_host;       /* [R * NH] */
  uint64_t *L;                /* [R] */
  uint32_t *nb, *n_hbm, *n_host, *prefix_hbm, *contrib;   /* [N] step-1/2 values of the last tick (download only) */
  int64_t *scalars;           /* [4]: tick, next_arrival, last_T, reserved */
  uint8_t *prefix_id;         /* [N] shared prompt of each program (255 = none) */
  uint32_t *prefix_ref;       /* [R * K] programs homed on r using prompt k */
  uint32_t *prefix_blk;       /* [R * K * max prompt blocks] blocks of prompt k on r (valid if ref > 0) */
} ta_state_view;

/* Bytes of device / page-locked host workspace a context needs for cfg. */
ta_status ta_workspace_bytes(const ta_config* cfg, size_t* dev_bytes, size_t* host_bytes);

/* Bytes of one KV block for cfg (2 * L * bt * H * D * elem_bytes). */
ta_status ta_block_bytes(const ta_config* cfg, size_t* block_bytes);

/* Create a context over caller-owned buffers on the caller's CUDA stream
 * (cudaStream_t passed as void*).  Initialises the program table (all slots
 * UNARRIVED), empty block tables and all-free bitmaps.  nccl_comm is reserved
 * (must be NULL in ABI v1).  Errors: TA_E_INVAL (config), TA_E_NOMEM, TA_E_CUDA. */
ta_status ta_init_pool(const ta_config* cfg, const ta_buffers* bufs, void* cuda_stream,
                       void* nccl_comm, ta_ctx** out);

/* Trace mode: copy program scripts to the device.  Must be
 * called before the first tick.  Errors: TA_E_INVAL (sizes), TA_E_STATE (not trace mode). */
ta_status ta_load_trace(ta_ctx* ctx, const ta_trace_view* trace);

/* One scheduler tick (the periodic monitor, every Delta t):
 *   step 0  ingest (trace script or the API events ev[0..n_ev), validated in
 *           order, all-or-nothing); releases free their blocks;
 *   step 1  per-program footprint and prefix residency from the block table;
 *   step 2  decayed effective load per replica (eq. 7);
 *   step 3  pause pass, shortest-first acting-first;
 *   step 4  restore pass from the global queue;
 *   step 5  materialize: stall cut, program-aware eviction (host tier first),
 *           lowest-free-first allocation, hit accounting;
 *   step 6  block movement: D2H evictions, then P2P/H2D fetches and fills;
 *   step 7  deferred frees, optional compaction, statistics.
 * now_ms: trace mode: -1 (or exactly tick*Delta t); API mode: the tick's time.
 * Decisions are written to out[0..*n_out) in canonical order when out != NULL
 * (the call then returns after they land); with out == NULL the tick is only
 * enqueued on the stream.  Errors: TA_E_INVAL, TA_E_STATE, event errors
 * (TA_E_DUP_ID, TA_E_UNKNOWN_PROGRAM, TA_E_ILLEGAL_TRANSITION: nothing applied,
 * the tick does not run), TA_E_TRUNCATED (tick ran; *n_out = needed count). */
ta_status ta_sched_step(ta_ctx* ctx, int64_t now_ms, const ta_event* ev, int32_t n_ev,
                        ta_decision* out, int32_t out_cap, int32_t* n_out);

/* Pause one active program now.  mode: TA_PAUSE_LAZY (blocks
 * become evictable, no bytes move), TA_PAUSE_OFFLOAD (evict its HBM blocks to the
 * host tier now, dropping when full), TA_PAUSE_DROP (free them).
 * Errors: TA_E_UNKNOWN_PROGRAM, TA_E_ILLEGAL_TRANSITION (not REASONING/ACTING). */
ta_status ta_pause(ta_ctx* ctx, uint32_t pid, uint32_t mode, ta_decision* out, int32_t out_cap,
                   int32_t* n_out);

/* Restore one paused program now on `replica` (-1: the
 * restore pass's least-loaded choice).  Phase R programs fetch their KV now
 * (eviction allowed).  Errors: TA_E_ILLEGAL_TRANSITION (not PAUSED),
 * TA_E_CAPACITY (L + contrib > lambda_max*C, or the fetch cannot be satisfied;
 * nothing changes). */
ta_status ta_resume(ta_ctx* ctx, uint32_t pid, int32_t replica, ta_decision* out, int32_t out_cap,
                    int32_t* n_out);

/* Move an active program to replica dst (dynamic migration):
 * a REASONING program's HBM blocks move to dst now (P2P over NVLink or D2D for
 * co-located replicas); an ACTING program's blocks move when its tool returns.
 * Errors: TA_E_ILLEGAL_TRANSITION, TA_E_INVAL (dst), TA_E_CAPACITY. */
ta_status ta_migrate(ta_ctx* ctx, uint32_t pid, int32_t dst_replica, ta_decision* out,
                     int32_t out_cap, int32_t* n_out);

/* Backend health mask with failover (PAPER.md:699 BackendState.healthy; SPEC.md:499-506:
 * "unhealthy backends flagged, their programs force-Paused back to the global queue").
 * healthy == 0: replica's KV (HBM pool and host tier) is considered lost: programs
 * active on it are paused (PAUSE records, slot order), programs homed on it drop every
 * block (EVICT records, all blocks dropped, slot order), its watermarks become 0 so no
 * restore, resume or migration targets it.  healthy != 0: back in service, empty (no
 * decisions).  No change: TA_OK, no decisions.  Collective in multi-process mode.
 * Errors: TA_E_INVAL (replica).  Synchronizes. */
ta_status ta_set_health(ta_ctx* ctx, int32_t replica, int32_t healthy, ta_decision* out, int32_t out_cap,
                        int32_t* n_out);

/* Cumulative counters and per-replica occupancy (synchronizes the stream). */
ta_status ta_stats(ta_ctx* ctx, ta_stats_t* out);

typedef struct {               /* what the last tick did (written by the device into host-mapped memory) */
  int64_t tick;                /* index of the tick */
  uint32_t decisions;          /* decisions emitted */
  uint32_t d2h_blocks;         /* evicted to the host tier (all replicas) */
  uint32_t h2d_blocks;         /* fetched from host tiers */
  uint32_t p2p_blocks;         /* fetched from another replica's HBM */
  uint32_t d2d_blocks;         /* moved by compaction */
  uint32_t fetch_blocks;       /* all allocated blocks (copies + fills) */
  /* per replica r (what crosses r's own links; a phase's time floor is the max over r): */
  uint32_t d2h_of[TA_MAX_REPLICAS];   /* blocks evicted into r's host tier (PCIe, out of r's GPU) */
  uint32_t h2d_of[TA_MAX_REPLICAS];   /* blocks fetched from r's host tier (PCIe, into r's GPU) */
  uint32_t p2p_to[TA_MAX_REPLICAS];   /* blocks fetched into r's HBM from a peer's HBM (NVLink) */
} ta_tick_info;

/* Telemetry of the last ta_sched_step (synchronizes the stream). */
ta_status ta_last_tick(ta_ctx* ctx, ta_tick_info* out);

/* Switch the copy engine between TMA bulk copies (cp.async.bulk through a 32 KiB
 * shared-memory stage, on != 0) and 128-bit loads/stores (on == 0).  Results are
 * identical; only the speed differs.  Synchronizes the stream. */
ta_status ta_set_copy_bulk(ta_ctx* ctx, int32_t on);

/* Per-phase device times of the last tick in microseconds (TA_F_TIMING only):
 * [0] ingest + footprint (API mode: event kernels + footprint) [1] pause + restore
 * [2] materialize plan [3] movement (one process: the fused kernel; one process per
 * GPU, TA_F_NO_FUSE: D2H evictions + barrier) [4] fetch copies + push + barrier
 * (TA_F_NO_FUSE only) [5] fills (multi-process with TA_F_FILL) [6] finalize +
 * compaction plan + decision assembly [7] compaction copies [8] unused.  n <= 9. */
ta_status ta_phase_times(ta_ctx* ctx, float* us, int32_t n);

/* Developer aid (TA_F_TIMING only): globaltimer stamps (ns) taken by thread 0 of
 * CTA 0 at the phase boundaries of the planner kernels during the last tick:
 * out[32*k + i], k = 0 pause, 1 restore, 2 plan, 3 close, 4 / 5 plan cluster ranks
 * 1 / 3 of replica 0; 0 = phase not reached.  n <= 256.  Synchronizes the stream.
 * Errors: TA_E_STATE (no TA_F_TIMING). */
ta_status ta_debug_phase_stamps(ta_ctx* ctx, uint64_t* out, int32_t n);

/* Developer / test aid: cumulative size-branch counters since ta_init_pool, out[i] =
 * how many times branch i ran: [0] CTA radix sort (n above the shared-memory sort
 * limit) [1] bitonic sort [2] rank sort [3] a candidate set's slot list kept in global
 * memory (beyond the shared-memory list limit) [4] planner need prefix in global memory [5] eviction prefix in global
 * memory [6] victims in global memory [7] request loop reading program values from
 * global memory [8] restore-pass chunks after the first [9] replica-ticks with
 * evictions [10] (development build) block-table rows the tick's footprint pass counted (rows written
 * since the previous pass; clean rows keep their counts and are not read) [11] the
 * entries of those rows; [12, 16) reserved.  n <= 16.  Synchronizes the stream. */
#define TA_DEBUG_COUNTERS 16
ta_status ta_debug_counters(ta_ctx* ctx, uint64_t* out, int32_t n);

/* Block-list-driven KV movement (the copy engine of step 6, exposed directly):
 * copy n whole KV blocks, block src_blocks[i] of the source pool to block
 * dst_blocks[i] of the destination pool.  kind: TA_MOVE_D2D (HBM of src_replica
 * to HBM of the same replica; dst_replica ignored), TA_MOVE_P2P (HBM of
 * src_replica to HBM of dst_replica, over NVLink when the pools live on
 * different GPUs), TA_MOVE_D2H (HBM of src_replica to its host tier),
 * TA_MOVE_H2D (host tier of src_replica to HBM of dst_replica).
 * src_blocks / dst_blocks are DEVICE pointers (caller-owned, n u32 each); the
 * lists must not overlap in the destination.  Block tables and free sets are
 * not touched.  Enqueued on the context stream.  Errors: TA_E_INVAL. */
enum { TA_MOVE_D2D = 1, TA_MOVE_P2P = 2, TA_MOVE_D2H = 3, TA_MOVE_H2D = 4 };
ta_status ta_move_blocks(ta_ctx* ctx, int32_t kind, int32_t src_replica, int32_t dst_replica,
                         const uint32_t* src_blocks, const uint32_t* dst_blocks, int32_t n);

/* Count KV words that differ from the content closed form
 * over every valid token slot of every owned HBM and host block of the local
 * replicas (test aid; needs TA_F_FILL runs).  Synchronizes. */
ta_status ta_verify_content(ta_ctx* ctx, uint64_t* mismatched_words, uint64_t* checked_words);

/* Parity tests: dir 0 = download device state into v, 1 = upload v (all
 * fields required except the download-only ones).  Synchronizes. */
ta_status ta_debug_state(ta_ctx* ctx, int32_t dir, const ta_state_view* v);

/* Multi-GPU, one replica per process (replicas_here == 1, first_replica = rank):
 * ta_export_pool_handle writes TA_HANDLE_BYTES describing this process's HBM pool
 * and its barrier mailbox (CUDA IPC handles + offset); every peer passes it to
 * ta_import_peer_pool, which maps that replica's pool (P2P over NVLink) and
 * mailbox.  All peers must be imported before the first tick; each tick then
 * runs two device-side barriers (after evictions, after fetches/pushes) and
 * pushes host-tier fetches whose destination lives in another process.
 * Errors: TA_E_INVAL (arguments), TA_E_PEER (IPC failure; poisons the context). */
#define TA_HANDLE_BYTES 192
ta_status ta_export_pool_handle(ta_ctx* ctx, void* handle);        /* handle: TA_HANDLE_BYTES */
ta_status ta_import_peer_pool(ta_ctx* ctx, int32_t replica, const void* handle);

ta_status ta_destroy(ta_ctx* ctx);
const char* ta_last_error(const ta_ctx* ctx);
int32_t ta_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TA_H_ */
