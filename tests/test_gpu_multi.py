"""Multi-GPU parity: one replica per GPU over CUDA IPC + NVLink (tests/mgpu_parity.py under
torchrun).  Skipped unless at least two GPUs are visible."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n,mode", [(2, "trace"), (2, "verbs"), (2, "api"), (2, "shared"), (2, "c3"),
                                    (2, "prompts2"), (4, "trace"), (4, "api"), (4, "shared"), (4, "c3"),
                                    (4, "prompts2")])
def test_multi_gpu_parity(n, mode):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    port = 29530 + {"trace": 1, "verbs": 3, "api": 5, "shared": 7, "c3": 9, "prompts2": 11}[mode] + 20 * n
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mgpu_parity.py"), "30" if mode == "c3" else "120"] + (
               {"trace": [], "verbs": ["--verbs"], "api": ["--api"], "shared": ["--verbs", "--shared", "48"],
                "c3": ["--c3"], "prompts2": ["--verbs", "--prompts2"]}[mode])
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(": OK") == n
    if mode == "trace":   # ticks with copies between processes (the device barriers run) and
        import re         # ticks without (they are skipped) both occur in this run
        assert max(int(x) for x in re.findall(r"p2p_blocks=(\d+)", r.stdout)) > 0, r.stdout[-2000:]
