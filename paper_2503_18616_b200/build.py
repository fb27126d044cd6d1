"""In-tree build of the sm_100a shared library (nvcc; no torch extension, no JIT cache).

    python -m paper_2503_18616_b200.build

Both precisions are compiled with ``-fmad=false`` so the fp64 build rounds
exactly like the reference's C (built with -ffp-contract=off); the fp32 hot
loops place their fused multiply-adds explicitly.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_native")
LIB = os.path.join(OUT_DIR, "libtissuesim_b200.so")
SOURCES = ["capi.cu", "step_f32.cu", "step_f64.cu", "compiler.cpp"]
GENCODE = "arch=compute_100a,code=sm_100a"


def nvcc_bin():
    cand = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "tissuesim_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False):
    """Compile the library for sm_100a into paper_2503_18616_b200/_native/."""
    if not force and not needs_build():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    cmd = [nvcc_bin(), "-gencode", GENCODE, "-lineinfo", "-O3", "-fmad=false", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v" if verbose else "-O3",
           *os.environ.get("TS_NVCC_FLAGS", "").split(),   # development experiments only
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", LIB + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
