"""Multi-GPU parity: one replica per GPU over CUDA IPC + NVLink (tools/mgpu_parity.py under
torchrun).  Skipped unless at least two GPUs are visible."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("verbs", [False, True])
def test_two_gpu_parity(verbs):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    n = 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533" if verbs else "29531",
           os.path.join(ROOT, "tools", "mgpu_parity.py"), "120"] + (["--verbs"] if verbs else [])
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(": OK") == n
