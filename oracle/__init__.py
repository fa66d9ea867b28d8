"""CPU oracle for the ThunderAgent KV-manager hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  It
shares no code with the CUDA path (``paper_2602_13692_b200``) and never imports
it; the only shared module is the seeded input generator ``tracegen``.

Parity status per function is listed in each module header and in DESIGN.md §3 (readings in §2.1).
"""
from .ta_oracle import (  # noqa: F401
    Oracle, NONE, HOST_BIT, UNARRIVED, PAUSED, REASONING, ACTING, STOPPED, PHASE_R, PHASE_A,
    D_PAUSE, D_RESTORE, D_EVICT, D_FETCH, D_STALL, D_MIGRATE, D_COMPACT,
    E_ARRIVE, E_DECODE, E_TOOL_CALL, E_TOOL_RESULT, E_RELEASE,
    OK, E_INVAL, E_DUP_ID, E_UNKNOWN_PROGRAM, E_ILLEGAL_TRANSITION, E_CAPACITY,
    PAUSE_LAZY, PAUSE_OFFLOAD, PAUSE_DROP, decay_table,
)
from .content import splitmix64, content_word, block_words  # noqa: F401
