"""Plain, slow, integer-only CPU oracle of ThunderAgent's program-aware KV manager.

TEST INFRASTRUCTURE ONLY.  Imported only by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (cpu_baseline / --impl reference).  Shares no code with the
CUDA path; its only input is a ``tracegen`` trace (data) and a config dict.

The method is a heuristic policy applied tick by tick, so the
oracle *is* the algorithm written out step by step in the paper's order
(SURVEY.md §8(c) steps 0-7), with the readings (A1 onwards) listed in DESIGN.md §2.1.
Every order is a total order ending in the slot index, so results are unique.

Paper anchors (PAPER.md line numbers):
  program tuple P=<ID,c,T,L,tau,s>            306-310   (eq. 1)
  Restore / Pause primitives                  337-351   (eqs. 4, 5)
  periodic thrashing check                    356-360   (eq. 6)
  watermarks lambda_max/lambda_min, Delta C   362-365
  time-decayed check with f(t_q)              367-373   (eq. 7)
  shortest-first pause, Definition 1          386-399   (eqs. 8, 9)
  S_restore, S_pause scores                   400-406   (eqs. 10, 11)
  global waiting queue, load-balanced restore 409-415

Parity status: steps 2-4 are pinned by SPEC worked examples, brute force and
closed forms (tests/test_oracle_policy.py); step 5.6 hit accounting by an
independent per-token simulator (tests/test_oracle_tokensim.py); the whole tick
by the hand-computed golden W1 (tests/golden/w1.json) and invariants I1-I10.
Steps 0, 5.1-5.3 (eviction order) and 7 (compaction) are definitional (SURVEY.md
P11: no paper value to compare with); since round 2 they are pinned by hand-computed
states written from DESIGN.md's text (tests/test_oracle_handpins.py: two-finger
compaction, all three eviction groups with a partial victim and host-slot order, the
tool-call start time) and a mutation check that breaks each rule and sees a pin fail
(tests/test_oracle_mutants.py), besides W1 and invariants I1-I10.
"""
from __future__ import annotations

from array import array

NONE = 0xFFFFFFFF          # block-table entry: no KV
HOST_BIT = 0x80000000      # block-table entry: slot in the home replica's host tier

UNARRIVED, PAUSED, REASONING, ACTING, STOPPED = 0, 1, 2, 3, 4   # PAPER.md:670-676 (+UNARRIVED)
PHASE_R, PHASE_A = 0, 1                                          # tau

D_PAUSE, D_RESTORE, D_EVICT, D_FETCH, D_STALL, D_MIGRATE, D_COMPACT = 1, 2, 3, 4, 5, 6, 7
E_ARRIVE, E_DECODE, E_TOOL_CALL, E_TOOL_RESULT, E_RELEASE = 1, 2, 3, 4, 5
OK, E_INVAL, E_NOMEM, E_DUP_ID, E_UNKNOWN_PROGRAM, E_ILLEGAL_TRANSITION, E_CAPACITY = 0, 1, 2, 3, 4, 5, 6
PAUSE_LAZY, PAUSE_OFFLOAD, PAUSE_DROP = 0, 1, 2

MOVE_D2H, MOVE_P2P, MOVE_H2D, MOVE_D2D, MOVE_DROP = 1, 2, 3, 4, 5
FILL_NEW, FILL_RECOMPUTE, FILL_PROMPT = 1, 2, 3

INT64_MAX = (1 << 63) - 1


def decay_table(x: int, n: int = 64) -> list:
    """F[k] = floor(x^-k * 2^32) in exact integers (reading A5; PAPER.md:458 f(t)=2^-t).

    For x = 2 this is 2^(32-k) for k <= 32 and 0 beyond (pin P1)."""
    return [(1 << 32) // (x ** k) for k in range(n)]


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


PROMPT = -1        # owner_hbm tag of a shared-prompt block: (PROMPT, k, j)
PROMPT_UID = 0xFF0000   # KV content identity of shared prompt k: PROMPT_UID + k


def decision(kind, pid=NONE, src=-1, dst=-1, blocks=0, to_host=0, dropped=0,
             hit=0, peer=0, host=0, miss=0, new=0):
    """Decision record; field order matches ``ta_decision`` in include/ta.h."""
    return (kind, pid, src, dst, blocks, to_host, dropped, hit, peer, host, miss, new)


STAT_KEYS = (
    "ticks", "arrivals", "stops", "pauses", "restores", "oversized_skips", "shortfalls",
    "evict_blocks", "evict_to_host", "evict_dropped", "fetch_blocks", "p2p_blocks",
    "h2d_blocks", "recompute_blocks", "new_blocks", "compact_blocks", "stalls",
    "hit_tok", "peer_tok", "host_tok", "miss_tok", "new_tok", "fill_tok",
    "imbalance_max_blocks", "imbalance_last_blocks",
    # NEXT-1: STP cost ledger (token-ms, Eq. 2-3) and the Cost_unused bound
    "cost_decode", "cost_prefill", "cost_recompute", "cost_unused", "cost_caching",
    "unused_bound_checks", "unused_bound_violations",
    # NEXT-4 guard: how far memory pressure had grown when the periodic monitor found it
    # (context growth triggers thrashing mid-execution between checks)
    "overshoot_blocks", "overshoot_max_blocks",
    # NEXT-3 (reading A51): blocks allocated for shared prompts (a prompt materialized on a
    # replica where no program held it)
    "prefix_blocks",
)


def stair(n: int, q: int, base: int = 0) -> int:
    """Tokens held, summed over the chunks of a chunked prefill of n tokens on top of a
    resident base (SPEC.md cost-ledger recompute_cost_of; Appendix E.2:
    chunked prefill processes a constant number of tokens per step, so memory grows
    linearly and the STP integral is a staircase): sum_{i=1}^{ceil(n/q)} (base + min(i*q, n))."""
    total = 0
    i = 1
    while (i - 1) * q < n:
        total += base + min(i * q, n)
        i += 1
    return total


class Oracle:
    """One oracle instance = the whole cluster (all R replicas), single writer."""

    def __init__(self, cfg: dict, trace=None, api_mode: bool = False, n_slots: int | None = None):
        self.cfg = cfg
        self.R = int(cfg["n_replicas"])
        self.bt = int(cfg["block_tokens"])
        self.NB = int(cfg["hbm_blocks"])
        self.NH = int(cfg["host_blocks"])
        self.MAXB = ceil_div(int(cfg["max_ctx"]), self.bt)
        self.dt = int(cfg["delta_t_ms"])
        self.unit = int(cfg["decay_unit_ms"])
        self.rate = int(cfg["decode_tok_per_s"])
        # f(t) as a Q32 table: x^-t, or an explicit table (e.g. the TTL-pin
        # baseline's step function, NEXT-2 reading A47)
        self.F = list(cfg["decay_table"]) if cfg.get("decay_table") else decay_table(int(cfg["decay_x"]))
        # NEXT-2 baseline RequestAware (reading A46): a stateless engine, no program view
        self.request_aware = bool(cfg.get("request_aware", False))
        if self.request_aware:
            self.F = [0] * 64                  # a program in a tool call holds no request
        self.lmax = int(cfg["lambda_max_q16"])
        self.lmin = int(cfg["lambda_min_q16"])
        self.compact_every = int(cfg.get("compact_every", 0))
        # NEXT-2 baseline (SPEC.md BaselinePolicy.PinnedRouting; "sends all
        # requests from the same agentic workflow to the same node"): no global queue
        self.pinned = bool(cfg.get("pinned_routing", False))
        self.chunk_q = int(cfg.get("prefill_chunk_tokens", 2048))   # chunked-prefill tokens per step
        self.chunk_ms = int(cfg.get("prefill_chunk_ms", 100))       # time of one chunk step
        self.api_mode = api_mode
        self.trace = trace
        N = trace.n_slots if trace is not None else int(n_slots)
        self.N = N
        # --- program table (ProgramState) ---
        self.uid = [0] * N
        self.status = [UNARRIVED] * N
        self.phase = [PHASE_R] * N
        self.placement = [-1] * N          # L (curly)
        self.home = [-1] * N               # replica whose HBM / host tier holds the KV
        self.c = [0] * N                   # context tokens
        self.c_kv = [0] * N                # tokens whose KV has been written
        self.acting_since = [0] * N        # ms; t_q = T - acting_since
        self.tool_return = [INT64_MAX] * N
        self.paused_since = [0] * N        # tick
        self.step_count = [0] * N
        self.turn = [0] * N
        self.gen_done = [0] * N
        self.satisfied = [0] * N
        # synthetic engine (reading A48): tokens waiting to be prefilled (prompt, tool
        # results) and the engine time the last materialize spent (re)prefilling
        self.pend = [0] * N
        self.busy = [0] * N
        self.loc = [array("I", [NONE]) * self.MAXB for _ in range(N)]
        # --- per replica pools (BackendState.cache_config) ---
        self.hbm_free = [bytearray([1]) * self.NB for _ in range(self.R)]
        self.host_free = [bytearray([1]) * self.NH for _ in range(self.R)]
        self.owner_hbm = [[None] * self.NB for _ in range(self.R)]
        self.owner_host = [[None] * self.NH for _ in range(self.R)]
        # NEXT-3 (reading A51): K shared system prompts (one per agent preset; PAPER.md:230
        # "agentic system prompts are identical across workflows").  Program p's first
        # sbk[kp[p]] blocks are its prompt, stored once per replica: a program homed on r
        # points them at prompt k's blocks on r (pblk[r][k]); pref[r][k] counts those
        # programs; the prompt is materialized (allocated lowest-free and prefilled) by the
        # first program that needs it on r, and released -- its blocks freed -- when the
        # last one leaves (release, move to another replica, failure).  Prompt blocks are
        # never evicted, moved or compacted.  Load accounting still counts every
        # program's full c.
        import tracegen                                   # input parameters only
        spec = tracegen.prefix_spec(cfg)
        self.K = len(spec)
        assert all(t > 0 and t % self.bt == 0 for t, _ in spec), "shared prompts: whole blocks"
        self.sbk = [t // self.bt for t, _ in spec]
        self.kp = [-1] * N
        self.trace_kp = None
        if trace is not None and self.K:
            ids = tracegen.prefix_ids(cfg, trace)
            self.trace_kp = [int(x) if x != 255 else -1 for x in ids]
            for q in range(N):
                kq = self.trace_kp[q]
                assert kq < 0 or int(trace.p0[q]) >= self.sbk[kq] * self.bt, "a prompt starts with its shared prefix"
        self.pref = [[0] * self.K for _ in range(self.R)]
        self.pblk = [[None] * self.K for _ in range(self.R)]
        self.cap_max = [(self.lmax * self.NB) >> 16 for _ in range(self.R)]
        self.cap_min = [(self.lmin * self.NB) >> 16 for _ in range(self.R)]
        self.L = [0] * self.R
        self.healthy = [True] * self.R     # BackendState.healthy
        self.tick = 0
        self.last_T = 0
        self.next_arrival = 0
        self.stats = {k: 0 for k in STAT_KEYS}
        # per-tick outputs kept for tests / debugging
        self.moves = []      # (kind, src_replica, src_idx, dst_replica, dst_idx, pid, j)
        self.fills = []      # (kind, replica, hbm_idx, pid, j, t0, t1)
        self.fp = None

    # ------------------------------------------------------------------ helpers
    def nb_of(self, p: int) -> int:
        return ceil_div(self.c[p], self.bt)

    def sbp(self, p: int) -> int:
        """Blocks of program p's shared prompt (0 without one)."""
        k = self.kp[p]
        return self.sbk[k] if k >= 0 else 0

    def _unref(self, r: int, k: int):
        """A program using prompt k stopped being homed on r; the last one releases it."""
        self.pref[r][k] -= 1
        assert self.pref[r][k] >= 0
        if self.pref[r][k] == 0:
            for b in self.pblk[r][k]:
                self.hbm_free[r][b] = 1
                self.owner_hbm[r][b] = None
            self.pblk[r][k] = None

    @staticmethod
    def is_hbm(e: int) -> bool:
        return e != NONE and not (e & HOST_BIT)

    @staticmethod
    def is_host(e: int) -> bool:
        return e != NONE and bool(e & HOST_BIT)

    def contrib_at(self, p: int, T: int, nb: int) -> int:
        """Eq. 7: c for tau=R, c*f(t_q) for tau=A, in blocks (A4)
        and floored through the Q32 table (A5).  t_q = T - acting_since, in units of
        decay_unit_ms (A2), capped at 63."""
        if self.phase[p] == PHASE_R:
            return nb
        el = T - self.acting_since[p]
        k = 0 if el < 0 else min(63, el // self.unit)
        return (nb * self.F[k]) >> 32

    def restore_key(self, p: int, nb: int):
        """S_restore = 1/c + I(tau=R): R first, shortest first;
        ties: earlier paused_since, then slot (A8).  RequestAware: FCFS (A46)."""
        if self.request_aware:
            return (0, 0, self.paused_since[p], p)
        return (0 if self.phase[p] == PHASE_R else 1, nb, self.paused_since[p], p)

    def pause_key(self, p: int, nb: int):
        """S_pause = 1/c + I(tau=A): A first, shortest first;
        ties: later acting_since first (phase A only), then slot (A7).  RequestAware:
        running requests, the latest program first (recompute preemption, A46)."""
        if self.request_aware:
            return (1 if self.phase[p] == PHASE_A else 0, -p, 0, 0)
        if self.phase[p] == PHASE_A:
            return (0, nb, -self.acting_since[p], p)
        return (1, nb, 0, p)

    def _free_all(self, p: int):
        h = self.home[p]
        row = self.loc[p]
        sb = self.sbp(p)
        for j in range(self.MAXB):
            e = row[j]
            if e == NONE:
                continue
            assert h >= 0, "KV without a home replica"
            if j < sb:                         # shared prompt: a reference, not an owner
                row[j] = NONE
                continue
            if e & HOST_BIT:
                s = e & ~HOST_BIT
                self.host_free[h][s] = 1
                self.owner_host[h][s] = None
            else:
                self.hbm_free[h][e] = 1
                self.owner_hbm[h][e] = None
            row[j] = NONE
        if h >= 0 and self.kp[p] >= 0:         # it no longer uses its prompt on h
            self._unref(h, self.kp[p])

    def _release(self, p: int):
        """STOPPED: placement cleared, every block freed (A26)."""
        self._free_all(p)
        self.status[p] = STOPPED
        self.placement[p] = -1
        self.home[p] = -1
        self.satisfied[p] = 0
        self.stats["stops"] += 1

    def _arrive(self, p: int, k: int, uid: int, p0: int, prompt: int = -1):
        """Arrivals enter PAUSED, phase R (A12).  prompt: the shared
        prompt the program uses (-1: none; A51)."""
        self.uid[p] = uid
        self.kp[p] = prompt
        self.status[p] = PAUSED
        self.phase[p] = PHASE_R
        self.c[p] = p0
        self.c_kv[p] = 0
        self.paused_since[p] = k
        self.placement[p] = -1
        self.home[p] = -1
        self.turn[p] = 0
        self.gen_done[p] = 0
        self.satisfied[p] = 0
        self.step_count[p] = 0
        self.acting_since[p] = 0
        self.tool_return[p] = INT64_MAX
        self.pend[p] = p0                       # the prompt waits for its prefill
        self.busy[p] = 0
        self.stats["arrivals"] += 1

    def _pause(self, p: int, k: int):
        """Pause: unbind from the backend; KV becomes evictable
        (lazy, A13).  No bytes move."""
        self.status[p] = PAUSED
        self.placement[p] = -1
        self.paused_since[p] = k
        self.satisfied[p] = 0
        self.stats["pauses"] += 1

    # ------------------------------------------------------------------ step 0
    def _step0_trace(self, k: int, T: int):
        """Trace-mode ingest: decode, tool return, release, closed-loop arrivals
        (reason/act loop PAPER.md:160-162; A18)."""
        tr = self.trace
        stops = 0
        for p in range(self.N):
            st = self.status[p]
            if st == UNARRIVED or st == STOPPED:
                continue
            base = int(tr.turn_off[p])
            nturns = int(tr.turn_off[p + 1]) - base
            # 1. decode during the last interval (only if materialized last tick), after
            #    the engine's (re)prefill of that materialize (reading A48)
            if st == REASONING and self.satisfied[p]:
                t = self.turn[p]
                g = int(tr.g[base + t])
                left = g - self.gen_done[p]
                busy = min(self.busy[p], self.dt)
                d = min((self.rate * (self.dt - busy)) // 1000, left)
                self.c[p] += d
                self.gen_done[p] += d
                if self.gen_done[p] == g:
                    if t == nturns - 1:
                        self._release(p)
                        stops += 1
                        continue
                    # tool call: Reasoning -> Acting, t_q starts now (A3)
                    self.phase[p] = PHASE_A
                    self.status[p] = ACTING
                    took = 0 if self.rate == 0 else ceil_div(left * 1000, self.rate)
                    self.acting_since[p] = T - self.dt + busy + took
                    self.tool_return[p] = self.acting_since[p] + int(tr.d_ms[base + t])
                    self.step_count[p] += 1
            # 2. tool result (tools keep running while paused)
            if (self.phase[p] == PHASE_A and self.status[p] in (ACTING, PAUSED)
                    and T >= self.tool_return[p]):
                self.c[p] += int(tr.o[base + self.turn[p]])
                self.pend[p] += int(tr.o[base + self.turn[p]])   # the result waits for prefill
                self.turn[p] += 1
                self.gen_done[p] = 0
                self.phase[p] = PHASE_R
                self.tool_return[p] = INT64_MAX
                if self.status[p] == ACTING:
                    self.status[p] = REASONING
        # 4. arrivals: closed loop, lowest UNARRIVED slots
        n_arr = (tr.n_initial if k == 0 else 0) + stops
        hi = min(self.N, self.next_arrival + n_arr)
        for p in range(self.next_arrival, hi):
            self._arrive(p, k, int(tr.uid[p]), int(tr.p0[p]), self.trace_kp[p] if self.trace_kp else -1)
        self.next_arrival = hi

    # ------------------------------------------------------------------ step 1
    def _step1_footprint(self):
        """Per program: nb = ceil(c/bt), n_hbm, n_host, n_none, prefix_hbm (first
        non-HBM entry) from the block table (BASELINE.json north_star; A4)."""
        N = self.N
        nb = [0] * N
        n_hbm = [0] * N
        n_host = [0] * N
        n_none = [0] * N
        prefix = [0] * N
        for p in range(N):
            if self.status[p] not in (PAUSED, REASONING, ACTING):
                continue
            b = self.nb_of(p)
            row = self.loc[p]
            first = None
            for j in range(b):
                e = row[j]
                if e == NONE:
                    n_none[p] += 1
                elif e & HOST_BIT:
                    n_host[p] += 1
                else:
                    n_hbm[p] += 1
                    continue
                if first is None:
                    first = j
            nb[p] = b
            prefix[p] = b if first is None else first
        self.fp = dict(nb=nb, n_hbm=n_hbm, n_host=n_host, n_none=n_none, prefix_hbm=prefix)
        return self.fp

    # ------------------------------------------------------------------ step 2
    def _step2_load(self, T: int):
        nb = self.fp["nb"]
        contrib = [0] * self.N
        L = [0] * self.R
        for p in range(self.N):
            if self.status[p] in (PAUSED, REASONING, ACTING):
                contrib[p] = self.contrib_at(p, T, nb[p])
                if self.status[p] in (REASONING, ACTING):
                    L[self.placement[p]] += contrib[p]
        self.contrib = contrib
        self.L = L
        return contrib, L

    # ------------------------------------------------------------------ step 3
    def _step3_pause(self, k: int, out: list):
        """Per replica: if L > lambda_max*C, pause the shortest-first (acting-first)
        minimal prefix whose contributions cover Delta C (
        Delta C counts decayed contributions, A6)."""
        nb, contrib = self.fp["nb"], self.contrib
        for r in range(self.R):
            if self.L[r] <= self.cap_max[r]:
                continue
            dC = self.L[r] - self.cap_max[r]
            self.stats["overshoot_blocks"] += dC          # reading A50
            self.stats["overshoot_max_blocks"] = max(self.stats["overshoot_max_blocks"], dC)
            act = [p for p in range(self.N)
                   if self.status[p] in (REASONING, ACTING) and self.placement[p] == r]
            act.sort(key=lambda p: self.pause_key(p, nb[p]))
            s = 0
            chosen = []
            for p in act:
                if s >= dC:
                    break
                chosen.append(p)
                s += contrib[p]
            if s < dC:
                self.stats["shortfalls"] += 1
            for p in chosen:
                self._pause(p, k)
                self.L[r] -= contrib[p]
                out.append(decision(D_PAUSE, p, src=r))

    # ------------------------------------------------------------------ step 4
    def _step4_restore(self, out: list):
        """Global program-aware queue: S_restore order; restore
        while some replica is below lambda_min*C and the program keeps it <=
        lambda_max*C; target = least loaded (A10); skip programs
        that fit nowhere ever (A9); otherwise stop at the head."""
        nb, contrib = self.fp["nb"], self.contrib
        Q = [p for p in range(self.N) if self.status[p] == PAUSED]
        Q.sort(key=lambda p: self.restore_key(p, nb[p]))
        self.queue_order = list(Q)
        if self.pinned:
            self._step4_pinned(Q, out)
            return
        maxcap = max(self.cap_max)
        for p in Q:
            cr = contrib[p]
            if cr > maxcap:
                self.stats["oversized_skips"] += 1
                continue
            cand = [r for r in range(self.R)
                    if self.L[r] < self.cap_min[r] and self.L[r] + cr <= self.cap_max[r]]
            if not cand:
                break
            t = min(cand, key=lambda r: (self.L[r], 0 if r == self.home[p] else 1, r))
            self.status[p] = REASONING if self.phase[p] == PHASE_R else ACTING
            self.placement[p] = t
            self.L[t] += cr
            self.stats["restores"] += 1
            out.append(decision(D_RESTORE, p, src=self.home[p], dst=t))

    def _step4_pinned(self, Q: list, out: list):
        """PinnedRouting baseline (reading A45): program p is bound to replica p mod R for
        its lifetime; each replica restores from its own queue (the global S_restore
        order restricted to its programs) while the head fits there (same watermark
        test) and stops at its first head that does not; programs that can never fit
        their replica are skipped.  Decisions in global queue order."""
        contrib = self.contrib
        stopped = [False] * self.R
        for p in Q:
            t = p % self.R
            if stopped[t]:
                continue
            cr = contrib[p]
            if cr > self.cap_max[t]:
                self.stats["oversized_skips"] += 1
                continue
            if not (self.L[t] < self.cap_min[t] and self.L[t] + cr <= self.cap_max[t]):
                stopped[t] = True
                if all(stopped):
                    break
                continue
            self.status[p] = REASONING if self.phase[p] == PHASE_R else ACTING
            self.placement[p] = t
            self.L[t] += cr
            self.stats["restores"] += 1
            out.append(decision(D_RESTORE, p, src=self.home[p], dst=t))

    # ------------------------------------------------------------------ step 5
    def _need(self, p: int, r: int) -> int:
        """#{sbp <= j < nb : loc[j] is not HBM on r}: the program's private blocks (its
        shared prompt, if it must be materialized on r, is added by _materialize)."""
        row = self.loc[p]
        here = self.home[p] == r
        return sum(1 for j in range(self.sbp(p), self.fp["nb"][p]) if not (here and self.is_hbm(row[j])))

    def _evict_order(self, r: int):
        """Eviction candidates E_r and their order (reading A21):
        group 0 PAUSED in exact reverse of the restore order; group 1 ACTING placed
        elsewhere; group 2 ACTING placed on r; groups 1-2 by (contrib, slot)."""
        nb, n_hbm, contrib = self.fp["nb"], self.fp["n_hbm"], self.contrib
        E = [p for p in range(self.N) if self.home[p] == r and n_hbm[p] > self.sbp(p)
             and self.status[p] in (PAUSED, ACTING)]
        if self.request_aware:                 # LRU over idle caches, not program-aware (A46)
            return sorted(E, key=lambda p: (self.paused_since[p] * self.dt if self.status[p] == PAUSED
                                            else self.acting_since[p], p))
        g0 = sorted([p for p in E if self.status[p] == PAUSED],
                    key=lambda p: self.restore_key(p, nb[p]), reverse=True)
        g1 = sorted([p for p in E if self.status[p] == ACTING and self.placement[p] != r],
                    key=lambda p: (contrib[p], p))
        g2 = sorted([p for p in E if self.status[p] == ACTING and self.placement[p] == r],
                    key=lambda p: (contrib[p], p))
        return g0 + g1 + g2

    def _materialize(self, r: int, F: list, stat_out: list, fetch_out: list, deferred: list,
                     all_or_nothing: bool = False) -> bool:
        """Steps 5.2-5.7 for replica r and the REASONING list F (slot order).
        Returns False (and changes nothing) if all_or_nothing and F does not fit."""
        nb, n_hbm = self.fp["nb"], self.fp["n_hbm"]
        need = {p: self._need(p, r) for p in F}
        # NEXT-3 (A51): a prompt not resident on r is materialized by the first program of
        # F (slot order) that uses it; its blocks are that program's first requests
        extra, claimed = {}, set()
        for p in F:
            k = self.kp[p]
            extra[p] = 0
            if k >= 0 and self.pblk[r][k] is None and k not in claimed:
                extra[p] = self.sbk[k]
                claimed.add(k)
        E = self._evict_order(r)
        free_r = sum(self.hbm_free[r])
        supply = free_r + sum(n_hbm[p] - self.sbp(p) for p in E)   # private HBM blocks
        # 5.2 stall cut: longest prefix of F with sum(need) <= supply
        S, tot = [], 0
        for p in F:
            if tot + need[p] + extra[p] > supply:
                break
            S.append(p)
            tot += need[p] + extra[p]
        if all_or_nothing and len(S) < len(F):
            return False
        stalled = F[len(S):]
        # 5.3 evict: tail-first, host tier first (lowest free slot) else drop
        X = max(0, tot - free_r)
        ev_out = []
        hslot = 0
        for p in E:
            if X == 0:
                break
            row = self.loc[p]
            hbm_js = [j for j in range(self.sbp(p), nb[p]) if self.is_hbm(row[j])]
            take = min(X, len(hbm_js))
            to_host = dropped = 0
            for j in sorted(hbm_js, reverse=True)[:take]:
                idx = row[j]
                while hslot < self.NH and not self.host_free[r][hslot]:
                    hslot += 1
                if hslot < self.NH:
                    self.host_free[r][hslot] = 0
                    self.owner_host[r][hslot] = (p, j)
                    row[j] = HOST_BIT | hslot
                    self.moves.append((MOVE_D2H, r, idx, r, hslot, p, j))
                    to_host += 1
                else:
                    row[j] = NONE
                    self.moves.append((MOVE_DROP, r, idx, -1, -1, p, j))
                    dropped += 1
                self.hbm_free[r][idx] = 1
                self.owner_hbm[r][idx] = None
            n_hbm[p] -= take
            X -= take
            self.stats["evict_blocks"] += take
            self.stats["evict_to_host"] += to_host
            self.stats["evict_dropped"] += dropped
            ev_out.append(decision(D_EVICT, p, src=r, blocks=take, to_host=to_host, dropped=dropped))
        assert X == 0
        # 5.6 hit accounting (before the table is rewritten), 5.4 allocate, 5.5 sources
        hptr = 0
        fx = []
        for p in S:
            row = self.loc[p]
            h = self.home[p]
            k = self.kp[p]
            sb = self.sbp(p)
            resumed = not (self.satisfied[p] and h == r)
            hit = peer = host = miss = 0
            if resumed:
                H = self.c_kv[p]
                for j in range(ceil_div(H, self.bt)):
                    tok = min(self.bt, H - j * self.bt)
                    e = row[j]
                    if j < sb:                         # shared prompt: resident on r, or
                        if extra[p]:                   # prefilled now by this program
                            miss += tok
                        else:
                            hit += tok
                    elif e == NONE:
                        miss += tok
                    elif e & HOST_BIT:
                        host += tok
                    elif h == r:
                        hit += tok
                    else:
                        peer += tok
            c0, c1 = self.c_kv[p], self.c[p]
            hist_blocks = ceil_div(c0, self.bt)
            if extra[p]:                               # materialize prompt k on r
                blocks = []
                for j in range(sb):
                    while not self.hbm_free[r][hptr]:
                        hptr += 1
                    dst = hptr
                    self.hbm_free[r][dst] = 0
                    self.owner_hbm[r][dst] = (PROMPT, k, j)
                    blocks.append(dst)
                    self.fills.append((FILL_PROMPT, r, dst, PROMPT_UID + k, j, j * self.bt, (j + 1) * self.bt))
                    self.stats["fill_tok"] += self.bt
                    self.stats["prefix_blocks"] += 1
                    self.stats["fetch_blocks"] += 1
                self.pblk[r][k] = blocks
            for j in range(sb):                        # the prompt (same blocks for every user on r)
                row[j] = self.pblk[r][k][j]
            for j in range(sb, nb[p]):
                e = row[j]
                recompute = False
                if h == r and self.is_hbm(e):
                    dst = e                                    # resident: hbm hit
                else:
                    while not self.hbm_free[r][hptr]:          # lowest free, request order
                        hptr += 1
                    dst = hptr
                    self.hbm_free[r][dst] = 0
                    self.owner_hbm[r][dst] = (p, j)
                    if e != NONE and not (e & HOST_BIT):      # HBM on h != r: P2P
                        self.moves.append((MOVE_P2P, h, e, r, dst, p, j))
                        deferred.append(("hbm", h, e))
                        self.stats["p2p_blocks"] += 1
                    elif e != NONE:                            # host tier of h: H2D
                        s = e & ~HOST_BIT
                        self.moves.append((MOVE_H2D, h, s, r, dst, p, j))
                        deferred.append(("host", h, s))
                        self.stats["h2d_blocks"] += 1
                    elif j < hist_blocks:                      # evicted history: recompute
                        recompute = True
                        self.stats["recompute_blocks"] += 1
                    else:                                      # brand-new tokens
                        self.stats["new_blocks"] += 1
                    row[j] = dst
                    self.stats["fetch_blocks"] += 1
                # 5.7 KV written into block j: recomputed history and new tokens [c_kv, c)
                t0 = j * self.bt if recompute else max(j * self.bt, c0)
                t1 = min((j + 1) * self.bt, c1)
                if t0 < t1:
                    self.fills.append((FILL_RECOMPUTE if recompute else FILL_NEW,
                                       r, dst, p, j, t0, t1))
                    self.stats["fill_tok"] += t1 - t0
            self.stats["hit_tok"] += hit
            self.stats["peer_tok"] += peer
            self.stats["host_tok"] += host
            self.stats["miss_tok"] += miss
            self.stats["new_tok"] += c1 - c0
            if need[p] + extra[p] > 0 or resumed:
                fx.append(decision(D_FETCH, p, src=h, dst=r, blocks=need[p] + extra[p],
                                   hit=hit, peer=peer, host=host, miss=miss, new=c1 - c0))
            if h != r and k >= 0:                      # the program now uses prompt k on r
                self.pref[r][k] += 1
                if h >= 0:
                    deferred.append(("unref", h, k))   # ... and no longer on h (step 7)
            self.home[p] = r
            self.c_kv[p] = c1
            n_hbm[p] = nb[p]
            # engine time of this materialize: recompute of the lost history plus the
            # prefill of waiting prompt / tool-result tokens, in chunk steps (A48)
            q = self.chunk_q
            self.busy[p] = self.chunk_ms * (ceil_div(miss, q) + ceil_div(self.pend[p], q))
            self.pend[p] = 0
            self._ledger_s.append((p, c0, c1, miss))
        for p in stalled:
            fx.append(decision(D_STALL, p, src=self.home[p], dst=r, blocks=need[p] + extra[p]))
            self.stats["stalls"] += 1
        stat_out.extend(ev_out)
        fetch_out.extend(fx)
        self._satisfied_now.update(S)
        return True

    def _step5(self, evict_out: list, fetch_out: list):
        deferred = []
        self._satisfied_now = set()
        self._ledger_s = []
        for r in range(self.R):
            F = [p for p in range(self.N) if self.status[p] == REASONING and self.placement[p] == r]
            self._materialize(r, F, evict_out, fetch_out, deferred)
        for p in range(self.N):
            self.satisfied[p] = 1 if p in self._satisfied_now else 0
        return deferred

    # ------------------------------------------------------------------ step 7
    def _apply_deferred(self, deferred):
        for kind, h, i in deferred:
            if kind == "hbm":
                self.hbm_free[h][i] = 1
                self.owner_hbm[h][i] = None
            elif kind == "host":
                self.host_free[h][i] = 1
                self.owner_host[h][i] = None
            else:                                      # "unref": a program left prompt i on h
                self._unref(h, i)

    def _compact(self, r: int, out: list):
        """Two-finger compaction (reading A20): move the highest used block to the
        lowest free block until the fingers cross.  Shared-prompt blocks stay put (A51):
        the upper finger skips them."""
        free = self.hbm_free[r]
        owner = self.owner_hbm[r]
        lo, hi, moves = 0, self.NB - 1, 0
        while True:
            while lo < self.NB and not free[lo]:
                lo += 1
            while hi >= 0 and (free[hi] or owner[hi][0] == PROMPT):
                hi -= 1
            if lo >= self.NB or hi < 0 or lo > hi:
                break
            p, j = self.owner_hbm[r][hi]
            self.loc[p][j] = lo
            self.owner_hbm[r][lo] = (p, j)
            self.owner_hbm[r][hi] = None
            free[lo] = 0
            free[hi] = 1
            self.moves.append((MOVE_D2D, r, hi, r, lo, p, j))
            moves += 1
        if moves:
            self.stats["compact_blocks"] += moves
            out.append(decision(D_COMPACT, NONE, src=r, dst=r, blocks=moves))

    def _ledger(self):
        """NEXT-1 STP ledger of this tick (readings A40-A44): for the interval that follows
        the tick, per replica, in token-ms:
          decode     satisfied programs hold their context c for the interval
          prefill    new tokens [c_kv, c) of satisfied programs, chunked on top of the
                     resident history: chunk_ms * stair(c - c_kv, q, base=c_kv)
          recompute  missed history of resumed programs: chunk_ms * stair(miss, q)
          caching    resident tokens of ACTING and PAUSED programs (idle KV), min(n_hbm*bt, c)
          unused     max(0, cap_max - used blocks) * bt while paused programs wait
        and the Cost_unused bound of PAPER.md:415: while the queue is non-empty, every
        replica's idle effective capacity max(0, cap_max - L) after the restore pass
        should be below c_min, the smallest paused footprint (blocks)."""
        dt, q, tau = self.dt, self.chunk_q, self.chunk_ms
        for p, c0, c1, miss in self._ledger_s:
            self.stats["cost_decode"] += c1 * dt
            self.stats["cost_prefill"] += tau * stair(c1 - c0, q, c0)
            self.stats["cost_recompute"] += tau * stair(miss, q)
        nb, n_hbm = self.fp["nb"], self.fp["n_hbm"]
        for p in range(self.N):
            if self.home[p] >= 0 and self.status[p] in (ACTING, PAUSED):
                self.stats["cost_caching"] += min(n_hbm[p] * self.bt, self.c[p]) * dt
        paused = [nb[p] for p in range(self.N) if self.status[p] == PAUSED]
        if paused:
            c_min = min(paused)
            for r in range(self.R):
                used = self.NB - sum(self.hbm_free[r])
                self.stats["cost_unused"] += max(0, self.cap_max[r] - used) * self.bt * dt
                self.stats["unused_bound_checks"] += 1
                if max(0, self.cap_max[r] - self.L[r]) >= c_min:
                    self.stats["unused_bound_violations"] += 1

    def _finalize_stats(self):
        used = [self.NB - sum(self.hbm_free[r]) for r in range(self.R)]
        imb = max(used) - min(used)
        self.stats["imbalance_last_blocks"] = imb
        self.stats["imbalance_max_blocks"] = max(self.stats["imbalance_max_blocks"], imb)
        self.stats["ticks"] += 1

    # ------------------------------------------------------------------ the tick
    def sched_step(self, now_ms: int | None = None, events=None):
        """One scheduler tick k at T = k*Delta t (periodic monitor).
        Returns (status, decisions in canonical order)."""
        k = self.tick
        self.moves = []
        self.fills = []
        if self.api_mode:
            T = int(now_ms)
            if events:
                st = self.validate_events(events)
                if st != OK:
                    return st, []
                self.apply_events(events, k)
        else:
            T = k * self.dt
            if now_ms is not None and now_ms >= 0 and now_ms != T:
                return E_INVAL, []
            self._step0_trace(k, T)
        self.last_T = T
        self._step1_footprint()
        self._step2_load(T)
        pauses, restores, evicts, fetches, compacts = [], [], [], [], []
        self._step3_pause(k, pauses)
        self._step4_restore(restores)
        deferred = self._step5(evicts, fetches)
        # step 6 (movement) is the list self.moves / self.fills, D2H before the rest
        self._apply_deferred(deferred)
        if self.compact_every and k % self.compact_every == 0:
            for r in range(self.R):
                self._compact(r, compacts)
        self._ledger()
        self._finalize_stats()
        self.tick += 1
        return OK, pauses + restores + evicts + fetches + compacts

    # ------------------------------------------------------------------ API mode
    def event_prompt(self, ev) -> int:
        """The shared prompt of an ARRIVE event (A51): none without prompts, prompt 0 with
        one, else t_ms (the prompt index; -2 = invalid)."""
        if self.K == 0:
            return -1
        if self.K == 1:
            return 0
        t = int(ev[4])
        return t if 0 <= t < self.K else -2

    def validate_events(self, events) -> int:
        """All-or-nothing validation in order (SURVEY.md §8(c) API table)."""
        status = {}
        phase = {}
        ctx = {}
        cap = self.MAXB * self.bt          # contexts are bounded by max_ctx (reading A35)
        for ev in events:
            kind, pid = ev[0], ev[1]
            if pid >= self.N:
                return E_UNKNOWN_PROGRAM
            st = status.get(pid, self.status[pid])
            ph = phase.get(pid, self.phase[pid])
            if kind in (E_ARRIVE, E_DECODE, E_TOOL_RESULT):
                c = ev[3] if kind == E_ARRIVE else ctx.get(pid, self.c[pid]) + ev[3]
                if c > cap and not (kind == E_ARRIVE and st != UNARRIVED):
                    return E_INVAL
                if kind == E_ARRIVE and st == UNARRIVED:
                    k = self.event_prompt(ev)
                    if k == -2:
                        return E_INVAL                    # no such shared prompt (A51)
                    if k >= 0 and c < self.sbk[k] * self.bt:
                        return E_INVAL                    # the prompt starts with its shared prefix
                ctx[pid] = c
            if kind == E_ARRIVE:
                if st != UNARRIVED:
                    return E_DUP_ID
                status[pid], phase[pid] = PAUSED, PHASE_R
            elif kind == E_DECODE:
                if st != REASONING:
                    return E_ILLEGAL_TRANSITION
            elif kind == E_TOOL_CALL:
                if st != REASONING:
                    return E_ILLEGAL_TRANSITION
                status[pid], phase[pid] = ACTING, PHASE_A
            elif kind == E_TOOL_RESULT:
                if ph != PHASE_A or st not in (ACTING, PAUSED):
                    return E_ILLEGAL_TRANSITION
                phase[pid] = PHASE_R
                if st == ACTING:
                    status[pid] = REASONING
            elif kind == E_RELEASE:
                if st == UNARRIVED:
                    return E_UNKNOWN_PROGRAM
                status[pid] = STOPPED
            else:
                return E_INVAL
        return OK

    def apply_events(self, events, k: int):
        for ev in events:
            kind, pid, uid, tokens, t_ms = ev
            if kind == E_ARRIVE:
                self._arrive(pid, k, uid, tokens, self.event_prompt(ev))
            elif kind == E_DECODE:
                self.c[pid] += tokens
            elif kind == E_TOOL_CALL:
                self.phase[pid] = PHASE_A
                self.status[pid] = ACTING
                self.acting_since[pid] = t_ms
                self.step_count[pid] += 1
            elif kind == E_TOOL_RESULT:
                self.c[pid] += tokens
                self.pend[pid] += tokens
                self.phase[pid] = PHASE_R
                if self.status[pid] == ACTING:
                    self.status[pid] = REASONING
            elif kind == E_RELEASE:
                if self.status[pid] != STOPPED:          # idempotent
                    self._release(pid)

    # explicit verbs act on the state left by the last tick, on one program
    def _verb_prepare(self):
        self.moves = []
        self.fills = []
        self._step1_footprint()
        self.contrib = [self.contrib_at(p, self.last_T, self.fp["nb"][p])
                        if self.status[p] in (PAUSED, REASONING, ACTING) else 0
                        for p in range(self.N)]

    def pause(self, pid: int, mode: int = PAUSE_LAZY):
        """Pause.  LAZY: blocks become evictable (A13);
        OFFLOAD: evict all HBM blocks now (host first, then drop); DROP: free them."""
        if pid >= self.N or self.status[pid] == UNARRIVED:
            return E_UNKNOWN_PROGRAM, []
        if self.status[pid] not in (REASONING, ACTING):
            return E_ILLEGAL_TRANSITION, []
        self._verb_prepare()
        r = self.placement[pid]
        self.L[r] -= self.contrib[pid]
        self._pause(pid, self.tick)
        out = [decision(D_PAUSE, pid, src=r)]
        if mode in (PAUSE_OFFLOAD, PAUSE_DROP):
            h = self.home[pid]
            row = self.loc[pid]
            hbm_js = [j for j in range(self.sbp(pid), self.fp["nb"][pid]) if self.is_hbm(row[j])]
            to_host = dropped = 0
            hslot = 0
            for j in sorted(hbm_js, reverse=True):
                idx = row[j]
                if mode == PAUSE_OFFLOAD:
                    while hslot < self.NH and not self.host_free[h][hslot]:
                        hslot += 1
                if mode == PAUSE_OFFLOAD and hslot < self.NH:
                    self.host_free[h][hslot] = 0
                    self.owner_host[h][hslot] = (pid, j)
                    row[j] = HOST_BIT | hslot
                    self.moves.append((MOVE_D2H, h, idx, h, hslot, pid, j))
                    to_host += 1
                else:
                    row[j] = NONE
                    self.moves.append((MOVE_DROP, h, idx, -1, -1, pid, j))
                    dropped += 1
                self.hbm_free[h][idx] = 1
                self.owner_hbm[h][idx] = None
            if hbm_js:
                self.stats["evict_blocks"] += len(hbm_js)
                self.stats["evict_to_host"] += to_host
                self.stats["evict_dropped"] += dropped
                out.append(decision(D_EVICT, pid, src=h, blocks=len(hbm_js),
                                    to_host=to_host, dropped=dropped))
        return OK, out

    def resume(self, pid: int, replica: int = -1):
        """Restore one program; capacity check SPEC.md:251-256.
        Phase R fetches now (steps 5-6 for this program alone, eviction allowed)."""
        if pid >= self.N or self.status[pid] == UNARRIVED:
            return E_UNKNOWN_PROGRAM, []
        if self.status[pid] != PAUSED:
            return E_ILLEGAL_TRANSITION, []
        if replica >= self.R or replica < -1:
            return E_INVAL, []
        self._verb_prepare()
        cr = self.contrib[pid]
        if replica == -1:
            cand = [r for r in range(self.R)
                    if self.L[r] < self.cap_min[r] and self.L[r] + cr <= self.cap_max[r]]
            if not cand:
                return E_CAPACITY, []
            replica = min(cand, key=lambda r: (self.L[r], 0 if r == self.home[pid] else 1, r))
        elif not self.healthy[replica] or self.L[replica] + cr > self.cap_max[replica]:
            return E_CAPACITY, []                         # unhealthy: no capacity (reading A39)
        return self._activate(pid, replica, cr, D_RESTORE)

    def migrate(self, pid: int, dst: int):
        """Move an active program to another DP replica:
        a REASONING program's blocks move now (P2P); ACTING ones on tool return."""
        if pid >= self.N or self.status[pid] == UNARRIVED:
            return E_UNKNOWN_PROGRAM, []
        if self.status[pid] not in (REASONING, ACTING):
            return E_ILLEGAL_TRANSITION, []
        if dst < 0 or dst >= self.R or dst == self.placement[pid]:
            return E_INVAL, []
        self._verb_prepare()
        cr = self.contrib[pid]
        if not self.healthy[dst] or self.L[dst] + cr > self.cap_max[dst]:
            return E_CAPACITY, []
        return self._activate(pid, dst, cr, D_MIGRATE)

    def _activate(self, pid: int, r: int, cr: int, kind: int):
        old_status, old_place, old_sat = self.status[pid], self.placement[pid], self.satisfied[pid]
        src = self.placement[pid] if kind == D_MIGRATE else self.home[pid]
        self.status[pid] = REASONING if self.phase[pid] == PHASE_R else ACTING
        self.placement[pid] = r
        evicts, fetches, deferred = [], [], []
        if self.status[pid] == REASONING:
            self._satisfied_now = set()
            self._ledger_s = []                  # verbs are not ticks: no ledger interval
            # all_or_nothing returns before any mutation when the fetch cannot fit
            ok = self._materialize(r, [pid], evicts, fetches, deferred, all_or_nothing=True)
            if not ok:
                self.status[pid], self.placement[pid], self.satisfied[pid] = old_status, old_place, old_sat
                return E_CAPACITY, []
            self.satisfied[pid] = 1
            self._apply_deferred(deferred)
        if old_place >= 0:
            self.L[old_place] -= cr
        self.L[r] += cr
        if kind == D_RESTORE:
            self.stats["restores"] += 1
        return OK, [decision(kind, pid, src=src, dst=r)] + evicts + fetches

    def set_health(self, r: int, healthy: bool):
        """Backend health mask with failover (NEXT-4; PAPER.md:699 BackendState.healthy;
        SPEC.md:502 "unhealthy backends flagged, their programs force-Paused back to the
        global queue").  Readings A37-A39: a replica marked unhealthy loses
        its KV -- its HBM pool and its host tier -- so every program homed there drops
        all its blocks (home -1; the history is recomputed where it resumes); every
        program active on it is paused (paused_since = the current tick); its
        watermarks become 0, so no restore targets it until it is marked healthy again
        (empty).  Decisions: PAUSE (slot order), then EVICT with all blocks dropped
        (slot order, programs that held blocks on r).  Idempotent: no change, no
        decisions."""
        if r < 0 or r >= self.R:
            return E_INVAL, []
        healthy = bool(healthy)
        if healthy == self.healthy[r]:
            return OK, []
        self.healthy[r] = healthy
        if healthy:
            self.cap_max[r] = (self.lmax * self.NB) >> 16
            self.cap_min[r] = (self.lmin * self.NB) >> 16
            return OK, []
        self.cap_max[r] = self.cap_min[r] = 0
        pauses, evicts = [], []
        for p in range(self.N):
            if self.status[p] in (REASONING, ACTING) and self.placement[p] == r:
                self._pause(p, self.tick)
                pauses.append(decision(D_PAUSE, p, src=r))
        for p in range(self.N):
            if self.home[p] != r:
                continue
            lost = sum(1 for j, e in enumerate(self.loc[p]) if e != NONE and j >= self.sbp(p))
            self._free_all(p)
            self.home[p] = -1
            if lost:
                self.stats["evict_blocks"] += lost
                self.stats["evict_dropped"] += lost
                evicts.append(decision(D_EVICT, p, src=r, blocks=lost, dropped=lost))
        self.L[r] = 0
        return OK, pauses + evicts

    # ------------------------------------------------------------------ invariants
    def check_invariants(self):
        """I1-I10; I6 (content) and I8 (no-thrash) are checked by tests."""
        used_h = [[None] * self.NB for _ in range(self.R)]
        used_s = [[None] * self.NH for _ in range(self.R)]
        users = [[0] * self.K for _ in range(self.R)]
        for p in range(self.N):
            row = self.loc[p]
            nb = self.nb_of(p) if self.status[p] in (PAUSED, REASONING, ACTING) else 0
            sb = self.sbp(p)
            if self.home[p] >= 0 and self.kp[p] >= 0:
                users[self.home[p]][self.kp[p]] += 1
            first_non_hbm = None
            n_hbm = 0
            for j in range(self.MAXB):
                e = row[j]
                if e == NONE:
                    if j < nb and first_non_hbm is None:
                        first_non_hbm = j
                    continue
                assert j < nb, f"I2: block beyond nb for p={p}"
                h = self.home[p]
                assert h >= 0, f"I5: KV without home p={p}"
                if j < sb:                                 # NEXT-3: shared prompt reference
                    blk = self.pblk[h][self.kp[p]]
                    assert blk is not None and e == blk[j], f"shared prompt entry p={p} j={j}"
                    n_hbm += 1
                    continue
                if e & HOST_BIT:
                    s = e & ~HOST_BIT
                    assert used_s[h][s] is None and not self.host_free[h][s], "I2 host"
                    assert self.owner_host[h][s] == (p, j), "I2 host owner"
                    used_s[h][s] = (p, j)
                    if first_non_hbm is None:
                        first_non_hbm = j
                else:
                    assert used_h[h][e] is None and not self.hbm_free[h][e], "I2 hbm"
                    assert self.owner_hbm[h][e] == (p, j), "I2 hbm owner"
                    used_h[h][e] = (p, j)
                    n_hbm += 1
            if nb:
                assert (nb if first_non_hbm is None else first_non_hbm) == n_hbm, f"I10 p={p}"
                if sb and self.home[p] >= 0:
                    assert n_hbm >= sb, f"homed program without its shared prompt p={p}"
            st = self.status[p]
            assert (self.placement[p] >= 0) == (st in (REASONING, ACTING)), f"I5 p={p}"
            if st in (UNARRIVED, STOPPED):
                assert self.home[p] == -1 and n_hbm == 0
        for r in range(self.R):
            for k in range(self.K):                    # A51: refcounts and prompt blocks
                assert self.pref[r][k] == users[r][k], f"prompt refcount r={r} k={k}"
                assert (self.pblk[r][k] is not None) == (users[r][k] > 0), f"prompt residency r={r} k={k}"
                for j, b in enumerate(self.pblk[r][k] or ()):
                    assert not self.hbm_free[r][b] and self.owner_hbm[r][b] == (PROMPT, k, j), "prompt block"
                    assert used_h[r][b] is None
                    used_h[r][b] = (PROMPT, k, j)
            for b in range(self.NB):
                assert (used_h[r][b] is None) == bool(self.hbm_free[r][b]), "I1/I2 hbm free-set"
            for s in range(self.NH):
                assert (used_s[r][s] is None) == bool(self.host_free[r][s]), "I1/I2 host free-set"
        return True

    def check_watermark(self):
        """I3 (after step 4): L[r] <= lambda_max * C; I4 pinned fit."""
        for r in range(self.R):
            assert self.L[r] <= self.cap_max[r], f"I3 r={r}"
            pinned = sum(self.nb_of(p) for p in range(self.N)
                         if self.status[p] == REASONING and self.placement[p] == r)
            assert pinned <= self.cap_max[r], f"I4 r={r}"
        return True
