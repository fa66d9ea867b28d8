"""Seeded synthetic agent-trace generator and run configurations.

This module is the ONLY code shared by the CPU oracle (`oracle/`) and the CUDA
path (`paper_2602_13692_b200/`).  It holds no arithmetic of the scheduling
method: it draws per-program workload scripts (prompt length, turns, tokens
generated per turn, tool latency, tool-result tokens) and lists run parameters.
Everything the method computes from them lives on either side separately.

Shapes follow SURVEY.md §8(d) "Trace presets" (all parameters invented and
labelled synthetic: the paper only gives qualitative tool-latency shapes,
PAPER.md:775-808, 433, 445).
"""
from .presets import PRESETS, Trace, gen_trace, tile_trace  # noqa: F401
from .configs import CONFIGS, KV_SHAPES, get_config, make_trace, prefix_ids, prefix_spec  # noqa: F401
