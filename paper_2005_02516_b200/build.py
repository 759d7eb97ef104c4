"""Build the in-tree CUDA extension libswedg_b200.so for sm_100a.

    python -m paper_2005_02516_b200.build        # or __graft_entry__.build()

nvcc cross-compiles without a GPU; the .so is written next to this file so
it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libswedg_b200.so")
SOURCES = ["swedg_capi.cu", "setup.cpp"]
DEPS = ["swedg_capi.cu", "swedg_common.cuh", "modal_kernels.cuh", "modal_fast.cuh", "modal_pair_n4.cuh", "modal_pair_n3.cuh", "sbp_kernels.cuh", "sbp_pair_n4.cuh", "halo.cuh", "setup.cpp", "quad_data.inc"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-shared",
    "-Xptxas", "-v",
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, d) for d in sorted(set(DEPS) | set(os.listdir(CSRC)))]
    deps.append(os.path.join(os.path.dirname(PKG), "include", "swedg_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc] + NVCC_FLAGS + [os.path.join(CSRC, s) for s in SOURCES] + ["-o", LIB + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libswedg_b200.so")
    with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
        f.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print(r.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
