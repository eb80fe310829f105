"""Build the in-tree C-ABI library `libburst_b200.so` for sm_100a with nvcc.

    python -m paper_2403_09347_b200.build [--force] [--verbose]

The .so is written next to this file (git-ignored, but it travels to the GPU
box with the repo snapshot).  Rebuilds only when a source is newer than the
library unless --force.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libburst_b200.so")
SOURCES = ["capi.cu", "ring_nccl.cu", "ring_ipc.cu"]
HEADERS = ["ptx.cuh", "common.cuh", "lao_fwd_sm100.cuh", "lao_bwd4_sm100.cuh", "lao_dq_sm100.cuh",
           "simt_f32.cuh", "aux_kernels.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(ROOT, "include", "burst_b200.h"), os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile libburst_b200.so; `out`/`defines` build experiment variants."""
    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    tmp = target + ".tmp"
    cmd = [nvcc_path(), *ARCH, *[f"-D{d}" for d in defines], "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", "-shared", "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES], "-ldl"]
    if verbose:
        cmd.insert(4, "-Xptxas=-v")
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed building libburst_b200.so")
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.out, tuple(a.defines)))
