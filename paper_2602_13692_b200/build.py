"""Build libta.so (all CUDA kernels + the C ABI) in-tree for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libta.so")
# developer A/B aid: extra nvcc flags (e.g. -DROW_PRE=2) and another output name
EXTRA = os.environ.get("TA_NVCC_EXTRA", "").split()
SRC = os.path.join(HERE, "csrc", "ta_runtime.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def sources():
    d = os.path.join(HERE, "csrc")
    return [os.path.join(d, f) for f in sorted(os.listdir(d))] + [os.path.join(ROOT, "include", "ta.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    if out is None and not force and up_to_date():
        return LIB
    cmd = [NVCC, *FLAGS, *EXTRA, "-I", os.path.join(ROOT, "include"), "-o", (out or LIB) + ".tmp", SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libta.so")
    if verbose:
        sys.stderr.write(r.stderr)
    if out is not None:                   # A/B variant: no log, no default library
        os.replace(out + ".tmp", out)
        return out
    with open(os.path.join(HERE, "csrc", "ptxas.log"), "w") as f:   # registers / spills per kernel
        f.write("".join(ln for ln in r.stderr.splitlines(True) if "Compile time" not in ln))
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose=True, out=out))
