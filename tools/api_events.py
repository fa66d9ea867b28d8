"""The engine's side of API mode, recorded from a trace-mode run (test and bench aid).

In trace mode libta advances every program itself (decode during the interval, tool
call, tool result, release, closed-loop arrival: ta.h TA_F_TRACE_MODE).  In API mode
the engine reports the same changes as events (ta_event).  This module
runs the trace in trace mode on the GPU and turns the per-tick change of each program
into the event batch an engine would have sent, in slot order:
  ARRIVE(p, uid, p0)          the slot left UNARRIVED
  DECODE(p, n)                tokens generated during the interval (c grew beyond o)
  TOOL_CALL(p, acting_since)  step_count grew
  TOOL_RESULT(p, o)           turn grew (o = the trace's result tokens of that turn)
  RELEASE(p)                  the program stopped
Replaying the batches through an API-mode context at now_ms = k * Delta t gives the
same decisions as the trace-mode run (tests/test_gpu_api.py), and bench.py's e2e uses
them as the host-side input of every step.  No scheduling arithmetic lives here: the
batches are differences of observed states plus the trace's own script values."""
from __future__ import annotations

import numpy as np

FIELDS = ("uid", "status", "c", "turn", "step_count", "acting_since")
UNARRIVED, PAUSED, REASONING, ACTING, STOPPED = 0, 1, 2, 3, 4
ARRIVE, DECODE, TOOL_CALL, TOOL_RESULT, RELEASE = 1, 2, 3, 4, 5


def batch_from_states(prev: dict, cur: dict, trace) -> np.ndarray:
    """Events that take `prev` (state after tick k-1) to `cur`'s ingest result."""
    from paper_2602_13692_b200.binding import EVENT_DTYPE
    st0, st1 = prev["status"], cur["status"]
    arrive = (st0 == UNARRIVED) & (st1 != UNARRIVED)
    live = np.isin(st0, (PAUSED, REASONING, ACTING))
    d_turn = np.where(live, cur["turn"].astype(np.int64) - prev["turn"], 0)
    d_call = np.where(live, cur["step_count"].astype(np.int64) - prev["step_count"], 0)
    base = trace.turn_off[:-1].astype(np.int64)
    o = np.where(d_turn > 0, trace.o[np.minimum(base + prev["turn"], len(trace.o) - 1)], 0)
    dec = np.where(live, cur["c"].astype(np.int64) - prev["c"] - o, 0)
    release = live & (st1 == STOPPED)
    rows = []
    for p in np.nonzero(arrive | (dec > 0) | (d_call > 0) | (d_turn > 0) | release)[0]:
        if arrive[p]:
            rows.append((ARRIVE, p, int(trace.uid[p]), int(trace.p0[p]), 0))
            continue
        if dec[p] > 0:
            rows.append((DECODE, p, 0, int(dec[p]), 0))
        if d_call[p] > 0:
            rows.append((TOOL_CALL, p, 0, 0, int(cur["acting_since"][p])))
        if d_turn[p] > 0:
            rows.append((TOOL_RESULT, p, 0, int(o[p]), 0))
        if release[p]:
            rows.append((RELEASE, p, 0, 0, 0))
    return np.array(rows, dtype=EVENT_DTYPE) if rows else np.zeros(0, dtype=EVENT_DTYPE)


def record(cfg: dict, trace, ticks: int, device: int = 0):
    """Run `ticks` trace-mode ticks; return (event batches, decision lists) per tick."""
    from paper_2602_13692_b200 import Pool
    pool = Pool(cfg, trace.n_slots, max_turns=trace.total_turns, fill=False, device=device)
    pool.load_trace(trace)
    prev = pool.debug_download(FIELDS)
    batches, decisions = [], []
    for _ in range(ticks):
        _, dec = pool.step()
        cur = pool.debug_download(FIELDS)
        batches.append(batch_from_states(prev, cur, trace))
        decisions.append(dec)
        prev = cur
    pool.close()
    return batches, decisions
