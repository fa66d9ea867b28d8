"""Run configurations (BASELINE.json configs[0..4]; SURVEY.md §8(d) "Configs").

Pure parameters: no method arithmetic.  Every config uses Delta-t = 5000 ms
(reading A1), f(t) = 2^-t (x = 2, time unit
1000 ms, reading A2), lambda_max = lambda_min = 1, a synthetic
decode rate of 40 tokens/s and closed-loop arrivals.
"""
from __future__ import annotations

import copy

import numpy as np

from .presets import gen_trace, tile_trace

# KV shapes (2-byte elements).  toy: BASELINE.json configs[0]; q32: Qwen3-32B GQA
# (64 layers, 8 KV heads, head dim 128), BASELINE.json configs[1].
KV_SHAPES = {
    "toy": dict(n_layers=2, n_kv_heads=2, head_dim=64, elem_bytes=2),
    "q32": dict(n_layers=64, n_kv_heads=8, head_dim=128, elem_bytes=2),
    # decision-only shape: same block table / scheduling, tiny bytes per block
    # (used to run configs 3-4 with all replicas on one GPU)
    "mini": dict(n_layers=1, n_kv_heads=1, head_dim=64, elem_bytes=2),
}

_COMMON = dict(delta_t_ms=5000, decay_x=2, decay_unit_ms=1000, decode_tok_per_s=40,
               lambda_max_q16=65536, lambda_min_q16=65536, compact_every=0, layout=0)

CONFIGS = {
    # configs[0]: toy, 8 programs, 2 replicas, 4 turns, 256-block pool (128 per replica, reading A19)
    "c1_toy": dict(_COMMON, trace=dict(mix=["toy"], n=8, seed=1001, max_ctx=1024),
                   n_replicas=2, kv="toy", block_tokens=16, hbm_blocks=128, host_blocks=64,
                   max_ctx=1024, tick_cap=400),
    # configs[1]: SWE-Agent-shaped, 256 programs, 1 replica, Qwen3-32B KV
    "c2_swe": dict(_COMMON, trace=dict(mix=["swe"], n=256, seed=1002, max_ctx=65536),
                   n_replicas=1, kv="q32", block_tokens=16, hbm_blocks=24576, host_blocks=16384,
                   max_ctx=65536, tick_cap=2000),
    # configs[2]: OpenHands + ToolOrchestra, 2k programs, 8 replicas
    "c3_mixed": dict(_COMMON, trace=dict(mix=["openhands", "toolorch"], n=2000, seed=1003,
                                         max_ctx=65536),
                     n_replicas=8, kv="q32", block_tokens=16, hbm_blocks=12288, host_blocks=8192,
                     max_ctx=65536, tick_cap=2000),
    # configs[3]: RL-rollout burst, 10k programs at t=0, 8 replicas, max_ctx 32k
    "c4_rlburst": dict(_COMMON, trace=dict(mix=["swe", "openhands"], n=10000, seed=1004,
                                           max_ctx=32768),
                       n_replicas=8, kv="q32", block_tokens=16, hbm_blocks=12288,
                       host_blocks=16384, max_ctx=32768, tick_cap=2000),
    # bench workload (N=1 line of bench.py): configs[3]'s 10k-program RL-burst trace on ONE
    # replica per GPU with the configs[4] per-GPU pool (96 GiB / 4 MiB blocks)
    "bench_10k": dict(_COMMON, trace=dict(mix=["swe", "openhands"], n=10000, seed=1004,
                                          max_ctx=32768),
                      n_replicas=1, kv="q32", block_tokens=16, hbm_blocks=24576,
                      host_blocks=16384, max_ctx=32768, tick_cap=2000),
}


def sweep_config(n_programs: int, gpus: int, block_tokens: int, point: int) -> dict:
    """configs[4]: scaling sweep point (96 GiB of KV per GPU, swe/openhands mix)."""
    blk_bytes = 64 * 2 * 8 * 128 * 2 * block_tokens
    return dict(_COMMON, trace=dict(mix=["swe", "openhands"], n=n_programs, seed=2000 + point,
                                    max_ctx=65536),
                n_replicas=gpus, kv="q32", block_tokens=block_tokens,
                hbm_blocks=(96 << 30) // blk_bytes, host_blocks=0, max_ctx=65536, tick_cap=2000)


def ttl_pin_table(ttl_units: int) -> list:
    """TTL-pin baseline's f(t) (NEXT-2; SPEC.md BaselinePolicy.TtlPin; PAPER.md:2.2 "employs a
    time-to-live (TTL) mechanism to pin KV caches"): an acting program's KV counts in full
    for ttl_units decay units after its tool call, then not at all.  A parameter table
    (Q32, 64 entries), like the decay base x; the policy arithmetic stays on each side."""
    return [(1 << 32) if k < ttl_units else 0 for k in range(64)]


def prefix_spec(cfg: dict):
    """The shared system prompts of a run (NEXT-3, reading A51): a list of K token
    counts and, per prompt, the agent preset whose programs use it.  `shared_prefixes`
    = [(tokens, preset), ...]; the single-prompt form `shared_prefix_tokens` = T means one
    prompt used by every program (preset None).  Parameters only."""
    if cfg.get("shared_prefixes"):
        return [(int(t), p) for t, p in cfg["shared_prefixes"]]
    t = int(cfg.get("shared_prefix_tokens", 0) or 0)
    return [(t, None)] if t else []


def prefix_ids(cfg: dict, trace) -> np.ndarray:
    """Per trace slot, the index of the shared prompt its program uses (255: none): the
    prompt listed for its preset, or prompt 0 for everyone with the single-prompt form.
    Input data for both sides (no method arithmetic)."""
    spec = prefix_spec(cfg)
    out = np.full(trace.n_slots, 255, np.uint8)
    for k, (_, preset) in enumerate(spec):
        if preset is None:
            out[:] = k
        else:
            out[np.array([pr == preset for pr in trace.preset], bool)] = k
    return out


def get_config(name: str, **override) -> dict:
    cfg = copy.deepcopy(CONFIGS[name])
    tr = override.pop("trace", None)
    cfg.update(override)
    if tr:
        cfg["trace"].update(tr)
    return cfg


def make_trace(cfg: dict):
    t = cfg["trace"]
    tr = gen_trace(t["mix"], t["n"], t["seed"], t["max_ctx"], t.get("n_initial"))
    if t.get("labels"):           # agent labels cycled over the slots (e.g. one shared prompt each)
        lab = list(t["labels"])
        tr.preset = [lab[p % len(lab)] for p in range(tr.n_slots)]
    return tile_trace(tr, int(t.get("tile", 1)))
