"""Build libta.so (all CUDA kernels + the C ABI) in-tree for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libta.so")          # product build (TA_PROD_VARIANT)
LIB_DEV = os.path.join(HERE, "libta_dev.so")  # development build: timing, baselines, test aids
# developer A/B aid: extra nvcc flags (e.g. -DROW_PRE=2) and another output name
EXTRA = os.environ.get("TA_NVCC_EXTRA", "").split()
SRC = os.path.join(HERE, "csrc", "ta_runtime.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def sources():
    d = os.path.join(HERE, "csrc")
    return [os.path.join(d, f) for f in sorted(os.listdir(d))] + [os.path.join(ROOT, "include", "ta.h")]


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(s) <= t for s in sources())


def _nvcc(out: str, defines: list) -> subprocess.CompletedProcess:
    cmd = [NVCC, *FLAGS, *defines, *EXTRA, "-I", os.path.join(ROOT, "include"), "-o", out + ".tmp", SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed building {os.path.basename(out)}")
    return r


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """Both libraries from the same sources: libta.so with the measurement, baseline and
    test options (TA_F_TIMING, TA_F_PINNED_ROUTING, TA_F_REQUEST_AWARE, TA_F_SMALL_PATHS)
    compiled out of the tick kernels, libta_dev.so with them (the binding picks it for a
    context that sets one).  `out`: an A/B variant of the product build only."""
    if out is not None:                   # A/B variant: no log, no default library
        r = _nvcc(out, ["-DTA_PROD_VARIANT"])
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(out + ".tmp", out)
        return out
    if force or not up_to_date(LIB_DEV):
        _nvcc(LIB_DEV, [])
        os.replace(LIB_DEV + ".tmp", LIB_DEV)
    if force or not up_to_date(LIB):
        r = _nvcc(LIB, ["-DTA_PROD_VARIANT"])
        if verbose:
            sys.stderr.write(r.stderr)
        with open(os.path.join(HERE, "csrc", "ptxas.log"), "w") as f:   # registers / spills per kernel
            f.write("".join(ln for ln in r.stderr.splitlines(True) if "Compile time" not in ln))
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose=True, out=out))
