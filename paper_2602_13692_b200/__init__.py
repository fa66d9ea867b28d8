"""B200-native (sm_100a) hot path of ThunderAgent's program-aware KV-cache manager.

``libta.so`` (built from ``csrc/`` by ``build.py``) holds every kernel and the C ABI
declared in ``include/ta.h``; ``binding`` is a thin ctypes layer over it.
"""
from .binding import EXPORTED, Pool, TAError, decay_q32, lib, make_config  # noqa: F401

__all__ = ["Pool", "TAError", "lib", "make_config", "decay_q32", "EXPORTED"]
