"""Builds libalp.so in-tree with nvcc for sm_100a (no GPU needed to compile)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "alp.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", n) for n in ("alp_device.cuh", "alp_kernels.cuh")] + [os.path.join(ROOT, "include", "alp.h")]
OUT = os.path.join(HERE, "libalp.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compiles libalp.so (or, for tuning experiments, a variant `out` with extra -D defines)."""
    target = out or OUT
    if not force and out is None and not needs_build():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
           "-o", target + ".tmp", *SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libalp.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(target + ".tmp", target)
    if out is None:
        with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
            fh.write(res.stderr)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
