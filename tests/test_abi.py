"""CPU-side checks of the boundary: libta.so builds, loads without a GPU and exports
every entry point include/ta.h declares; the binding's structs match the header."""
import ctypes as C
import os
import re

import pytest

from paper_2602_13692_b200 import binding, build


@pytest.fixture(scope="module")
def libta():
    build.build()
    return binding.lib()


def header_functions():
    src = open(os.path.join(os.path.dirname(__file__), "..", "include", "ta.h")).read()
    return sorted(set(re.findall(r"^(?:ta_status|const char\*|int32_t)\s+(ta_\w+)\(", src, re.M)))


def test_exports_every_declared_symbol(libta):
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(libta, n), n
    assert set(names) == set(binding.EXPORTED)


def test_dev_build_exports_the_same_abi(libta):
    """libta_dev.so (development options compiled in) exports the same C ABI."""
    dev = binding.lib(dev=True)
    for n in header_functions():
        assert hasattr(dev, n), n
    assert dev.ta_abi_version() == libta.ta_abi_version()


def test_product_build_rejects_development_flags(libta):
    """libta.so compiles the timing / baseline / test options out and refuses a config
    that sets one (ta_workspace_bytes validates the config without a GPU)."""
    import tracegen
    cfg = tracegen.get_config("c1_toy")
    for f in (binding.F_TIMING, binding.F_PINNED_ROUTING, binding.F_REQUEST_AWARE, binding.F_SMALL_PATHS):
        c = binding.make_config(cfg, 8, 4, True, False, f, None, 0)
        d, h = C.c_size_t(), C.c_size_t()
        assert libta.ta_workspace_bytes(C.byref(c), C.byref(d), C.byref(h)) == binding.TA_E_INVAL, f
        assert binding.lib(dev=True).ta_workspace_bytes(C.byref(c), C.byref(d), C.byref(h)) == binding.TA_OK, f


def test_abi_version_and_struct_sizes(libta):
    assert libta.ta_abi_version() == 3
    assert C.sizeof(binding.Event) == 24
    assert binding.DECISION_DTYPE.itemsize == 48
    # ta_stats_t: 25 counters, L/hbm_used/host_used[32], block_bytes, 7 ledger, 2 guard, prefix_blocks (ta.h)
    assert C.sizeof(binding.Stats) == (25 + 3 * 32 + 1 + 7 + 2 + 1) * 8
    # ta_tick_info: tick, 6 u32 counters, 3 x u32[32] per-replica link counts
    assert C.sizeof(binding.TickInfo) == 8 + 6 * 4 + 3 * 32 * 4
    # ta_config ends with flags, prefill_chunk_tokens, prefill_chunk_ms, reserved
    assert binding.Config.prefill_chunk_ms.offset == binding.Config.prefill_chunk_tokens.offset + 4


def test_workspace_query_and_validation(libta):
    import tracegen
    cfg = tracegen.get_config("c1_toy")
    c = binding.make_config(cfg, 8, 32)
    dev, host = C.c_size_t(), C.c_size_t()
    assert libta.ta_workspace_bytes(C.byref(c), C.byref(dev), C.byref(host)) == 0
    assert dev.value > 0 and host.value > 0
    blk = C.c_size_t()
    libta.ta_block_bytes(C.byref(c), C.byref(blk))
    assert blk.value == 2 * 2 * 16 * 2 * 64 * 2          # 2L * bt * H * D * 2 bytes
    c.elem_bytes = 4
    assert libta.ta_workspace_bytes(C.byref(c), C.byref(dev), C.byref(host)) == binding.TA_E_INVAL


def test_binding_decay_table_matches_paper_default():
    # f(t) = 2^-t in Q32: 2^(32-k), 0 beyond k = 32
    F = binding.decay_q32(2)
    assert F == [(1 << 32) >> k if k <= 32 else 0 for k in range(64)]


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import tracegen
    with pytest.raises(RuntimeError):
        binding.Pool(tracegen.get_config("c1_toy"), 8)
