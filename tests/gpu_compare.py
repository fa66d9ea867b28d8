"""Helpers for GPU-vs-oracle parity: convert oracle state to the ta_state_view layout
and compare element by element (exact: all of it is integer / index work)."""
from __future__ import annotations

import numpy as np

import oracle
from oracle.content import block_words


def _bits(flags: bytearray, n: int) -> np.ndarray:
    """bytearray of 0/1 flags -> little-endian u32 words (bit i of word w = flag 32w+i)."""
    nw = -(-n // 32)
    a = np.zeros(nw * 32, np.uint8)
    a[:n] = np.frombuffer(bytes(flags), np.uint8)
    return np.packbits(a, bitorder="little").view("<u4").astype(np.uint32)


def oracle_arrays(o) -> dict:
    N, R, MAXB = o.N, o.R, o.MAXB
    d = dict(
        uid=np.array(o.uid, np.uint32), c=np.array(o.c, np.uint32), c_kv=np.array(o.c_kv, np.uint32),
        paused_since=np.array(o.paused_since, np.uint32), step_count=np.array(o.step_count, np.uint32),
        turn=np.array(o.turn, np.uint32), gen_done=np.array(o.gen_done, np.uint32),
        status=np.array(o.status, np.uint8), phase=np.array(o.phase, np.uint8),
        satisfied=np.array(o.satisfied, np.uint8), placement=np.array(o.placement, np.int8),
        home=np.array(o.home, np.int8), acting_since=np.array(o.acting_since, np.int64),
        tool_return=np.array(o.tool_return, np.int64),
        loc=np.array([np.frombuffer(row, np.uint32) for row in o.loc], np.uint32).reshape(N, MAXB),
        hbm_free=np.concatenate([_bits(o.hbm_free[r], o.NB) for r in range(R)]),
        host_free=(np.concatenate([_bits(o.host_free[r], o.NH) for r in range(R)])
                   if o.NH else np.zeros(1, np.uint32)),
        L=np.array(o.L, np.uint64),
        scalars=np.array([o.tick, o.next_arrival, o.last_T, 0], np.int64),
        prefix_id=np.array([k if k >= 0 else 255 for k in o.kp], np.uint8),
    )
    K, SBM = max(1, o.K), max([1] + o.sbk)                 # NEXT-3 prompts (A51)
    ref = np.zeros(R * K, np.uint32)
    blk = np.zeros(R * K * SBM, np.uint32)
    for r in range(R):
        for k in range(o.K):
            ref[r * K + k] = o.pref[r][k]
            for j, b in enumerate(o.pblk[r][k] or ()):
                blk[(r * K + k) * SBM + j] = b
    d["prefix_ref"], d["prefix_blk"] = ref, blk
    own_h = np.zeros(R * o.NB, np.uint32)
    own_s = np.zeros(max(1, R * o.NH), np.uint32)
    for r in range(R):
        for b, ow in enumerate(o.owner_hbm[r]):
            if ow is not None:       # shared-prompt blocks (NEXT-3): TA_OWNER_PROMPT | k << 20 | j
                own_h[r * o.NB + b] = (0xF8000000 | (ow[1] << 20) | ow[2]) if ow[0] == oracle.ta_oracle.PROMPT \
                    else ow[0] * MAXB + ow[1]
        for s, ow in enumerate(o.owner_host[r]):
            if ow is not None:
                own_s[r * o.NH + s] = ow[0] * MAXB + ow[1]
    d["owner_hbm"], d["owner_host"] = own_h, own_s
    return d


FIELDS = ("uid", "c", "c_kv", "paused_since", "step_count", "turn", "gen_done", "status", "phase",
          "satisfied", "placement", "home", "acting_since", "tool_return", "L")


def compare_state(o, g: dict, where=""):
    """Assert GPU state == oracle state (program table, block tables, free sets,
    owners of used blocks)."""
    a = oracle_arrays(o)
    live = a["status"] != oracle.UNARRIVED
    for f in FIELDS:
        x, y = a[f], g[f]
        if f in ("uid", "c", "c_kv", "paused_since", "step_count", "turn", "gen_done", "acting_since",
                 "tool_return"):
            x, y = x[live], y[live]
        if not np.array_equal(x, y):
            bad = np.nonzero(x != y)[0][:8]
            raise AssertionError(f"{where}: field {f} differs at {bad}: oracle {x[bad]} gpu {y[bad]}")
    if not np.array_equal(a["loc"], g["loc"]):
        p, j = np.argwhere(a["loc"] != g["loc"])[0]
        raise AssertionError(f"{where}: loc[{p}][{j}] oracle {a['loc'][p, j]:#x} gpu {g['loc'][p, j]:#x}")
    assert np.array_equal(a["hbm_free"], g["hbm_free"]), f"{where}: hbm free set differs"
    if o.NH:
        assert np.array_equal(a["host_free"], g["host_free"][:a["host_free"].size]), f"{where}: host free set"
    used_h = ~np.unpackbits(a["hbm_free"].view(np.uint8), bitorder="little").astype(bool)
    for r in range(o.R):
        m = used_h[r * (-(-o.NB // 32) * 32): r * (-(-o.NB // 32) * 32) + o.NB]
        ia, ig = a["owner_hbm"][r * o.NB:(r + 1) * o.NB][m], g["owner_hbm"][r * o.NB:(r + 1) * o.NB][m]
        assert np.array_equal(ia, ig), f"{where}: owner_hbm r={r}"
    assert int(g["scalars"][0]) == o.tick and int(g["scalars"][1]) == o.next_arrival, where
    if o.K:                                                # NEXT-3: prompts, refcounts, blocks
        assert np.array_equal(a["prefix_id"][live], g["prefix_id"][live]), f"{where}: prefix_id"
        assert np.array_equal(a["prefix_ref"], g["prefix_ref"][:a["prefix_ref"].size]), \
            f"{where}: prompt refcounts oracle {a['prefix_ref']} gpu {g['prefix_ref']}"
        SBM = max(o.sbk)
        for r in range(o.R):
            for k in range(o.K):
                if o.pref[r][k]:
                    lo = (r * o.K + k) * SBM
                    assert np.array_equal(a["prefix_blk"][lo:lo + o.sbk[k]], g["prefix_blk"][lo:lo + o.sbk[k]]), \
                        f"{where}: prompt {k} blocks on r{r}"


def dec_tuples(arr) -> list:
    return [tuple(int(x) for x in rec) for rec in arr]


def same_decisions(got_arr, want, where="") -> None:
    """Assert the GPU decision list equals the oracle's; on a mismatch name the first
    differing record and show both (kind, pid, src, dst, blocks, ...)."""
    got = dec_tuples(got_arr)
    if got == want:
        return
    for i, (a, b) in enumerate(zip(want, got)):
        if a != b:
            raise AssertionError(f"{where}: decision {i} of {len(want)} (gpu {len(got)}): oracle {a} gpu {b}")
    n = min(len(want), len(got))
    raise AssertionError(f"{where}: {len(want)} oracle decisions vs {len(got)} gpu; "
                         f"oracle extra {want[n:][:4]}, gpu extra {got[n:][:4]}")


def check_blocks_content(o, pool, samples, rng):
    """Byte-level check of sampled owned blocks against the closed form on the CPU."""
    from tracegen import KV_SHAPES
    kv = KV_SHAPES[o.cfg["kv"]]
    L, H, D, bt = kv["n_layers"], kv["n_kv_heads"], kv["head_dim"], o.bt
    owned = []
    for r in range(o.R):
        owned += [("hbm", r, b, ow) for b, ow in enumerate(o.owner_hbm[r]) if ow is not None]
        owned += [("host", r, s, ow) for s, ow in enumerate(o.owner_host[r]) if ow is not None]
    if not owned:
        return 0
    pick = rng.choice(len(owned), size=min(samples, len(owned)), replace=False)
    n = 0
    for i in pick:
        tier, r, idx, ow = owned[i]
        shared = ow[0] == oracle.ta_oracle.PROMPT                 # shared prompt k: uid PROMPT_UID + k
        if shared:
            _, k, j = ow
        else:
            p, j = ow
        valid = bt if shared else min(bt, o.c_kv[p] - j * bt)
        got = pool.read_block(r, tier, idx)                       # [2L, bt, H, D/4]
        want = block_words(oracle.ta_oracle.PROMPT_UID + k if shared else o.uid[p], j, bt, L, H,
                           D).reshape(2 * L, bt, H, D // 4)
        assert np.array_equal(got[:, :valid], want[:, :valid]), (tier, r, idx, p, j)
        n += 1
    return n
