"""Test helpers: build configs and hand-made oracle states (no method arithmetic here)."""
from __future__ import annotations

import numpy as np

from tracegen.presets import Trace


def base_cfg(**kw):
    cfg = dict(n_replicas=1, block_tokens=1, hbm_blocks=1000, host_blocks=0, max_ctx=4096,
               delta_t_ms=5000, decay_x=2, decay_unit_ms=1000, decode_tok_per_s=0,
               lambda_max_q16=65536, lambda_min_q16=65536, compact_every=0, layout=0,
               kv="mini")
    cfg.update(kw)
    return cfg


def flat_trace(n, turns=3, g=100, d_ms=1000, o=0, p0=1):
    """A trace where every slot has the same simple script (for hand-built states)."""
    g_ = np.full(n * turns, g, np.uint32)
    d_ = np.full(n * turns, d_ms, np.uint32)
    o_ = np.full(n * turns, o, np.uint32)
    d_[turns - 1::turns] = 0
    o_[turns - 1::turns] = 0
    return Trace(uid=np.arange(1, n + 1, dtype=np.uint32), p0=np.full(n, p0, np.uint32),
                 turn_off=(np.arange(n + 1) * turns).astype(np.uint32), g=g_, d_ms=d_, o=o_,
                 n_initial=n, preset=["flat"] * n)


def set_program(o, p, status, phase, c, placement=-1, home=-1, acting_since=0,
                tool_return=None, paused_since=0, c_kv=None, satisfied=0, hbm=(), host=(),
                uid=None):
    """Place program p in a hand-made state.  hbm: block indices on `home` for j=0..;
    host: host-tier slots for the following j."""
    import oracle
    o.uid[p] = p + 1 if uid is None else uid
    o.status[p] = status
    o.phase[p] = phase
    o.c[p] = c
    o.c_kv[p] = c if c_kv is None else c_kv
    o.placement[p] = placement
    o.home[p] = home
    o.acting_since[p] = acting_since
    o.tool_return[p] = (1 << 63) - 1 if tool_return is None else tool_return
    o.paused_since[p] = paused_since
    o.satisfied[p] = satisfied
    j = 0
    for b in hbm:
        o.loc[p][j] = b
        o.hbm_free[home][b] = 0
        o.owner_hbm[home][b] = (p, j)
        j += 1
    for s in host:
        o.loc[p][j] = oracle.HOST_BIT | s
        o.host_free[home][s] = 0
        o.owner_host[home][s] = (p, j)
        j += 1
    o.next_arrival = max(o.next_arrival, p + 1)
