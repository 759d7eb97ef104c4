#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/*.npz from the REFERENCE itself.

The reference (/root/reference/proj, header-only C++20) is compiled unmodified
against oracle/shim (Eigen/doctest stand-ins) by `make -f oracle/Makefile.ref`
into oracle/_ref/swedg_dump (oracle/ref_dump.cpp).  This script runs that
binary for each fixture case and converts its record container to compressed
.npz files.  It needs /root/reference (this container only); the .npz files it
writes are committed and travel to the GPU box.

    python tests/golden/make_golden.py            # (re)build oracle/_ref and all fixtures
"""
from __future__ import annotations

import os
import struct
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
DUMP = os.path.join(REPO, "oracle", "_ref", "swedg_dump")

# name -> swedg_dump arguments (see oracle/ref_dump.cpp main())
CASES = {
    # operator tables N=1..4, modal and SBP-Legendre, plus volume rules deg 1..16
    "ops": ["ops"],
    # test_solver.cpp Fixture-style cases on [-1,1]^2:  N n warp periodic seed bathy nsteps dt
    "modal_n3_warp": ["modal", "3", "4", "0.1", "1", "23", "1", "3", "0.005"],
    "modal_n4_warp": ["modal", "4", "4", "0.1", "1", "41", "1", "2", "0.004"],
    "modal_n2_walls": ["modal", "2", "4", "0.0", "0", "31", "0", "2", "0.005"],
    "modal_n1_affine": ["modal", "1", "4", "0.0", "1", "53", "1", "1", "0.01"],
    "modal_n4_affine": ["modal", "4", "3", "0.0", "1", "5", "1", "1", "0.004"],
    # named problems through run.hpp:  name N scheme n warp cfl tfinal store_inputs
    # C1: vortex N=3, K1D=16 (512 tris), RK to t=0.5
    "c1_vortex": ["problem", "vortex", "3", "hyb", "16", "0.0", "0.125", "0.5", "1"],
    # C2: lake at rest, N=3, curved (warp 0.1), K1D=8, t=0.5
    "c2_lake": ["problem", "lake", "3", "hyb", "8", "0.1", "0.125", "0.5", "1"],
    # C3-style SBP N=4 dam break (small grid) and SBP lake (curved)
    "sbp_dam_n4": ["problem", "dambreak", "4", "sbp", "10", "0.0", "0.0625", "0.05", "1"],
    "sbp_lake_n3": ["problem", "lake", "3", "sbp", "4", "0.1", "0.125", "0.02", "1"],
    "sbp_vortex_n2": ["problem", "vortex", "2", "sbp", "8", "0.0", "0.125", "0.1", "1"],
    # hybridized dam break (walls + curved dam) N=3, small
    "dam_n3": ["problem", "dambreak", "3", "hyb", "10", "0.0", "0.0625", "0.05", "1"],
    # test_solver.cpp:355-371 positivity failure in element 1
    "positivity": ["positivity"],
    # bench.hpp volume-kernel cost study: matvec / fluxdiff / skew outputs, n = 6..50
    "ratio": ["ratio"],
    # output formats: mesh text (lake, dam) and run()'s CSV / VTK files of a small vortex run
    "io": ["io", "@TMP"],
    # acceptance criterion 5: the reference's vortex convergence studies
    "convergence": ["convergence"],
}


def read_records(path: str) -> dict[str, np.ndarray]:
    out: dict[str, np.ndarray] = {}
    with open(path, "rb") as f:
        data = f.read()
    p = 0
    while p < len(data):
        (n,) = struct.unpack_from("<I", data, p)
        p += 4
        name = data[p : p + n].decode()
        p += n
        dtype = data[p]
        p += 1
        (nd,) = struct.unpack_from("<I", data, p)
        p += 4
        dims = struct.unpack_from("<" + "Q" * nd, data, p)
        p += 8 * nd
        count = int(np.prod(dims)) if nd else 1
        dt = np.float64 if dtype == 0 else np.int32
        arr = np.frombuffer(data, dtype=dt, count=count, offset=p).reshape(dims).copy()
        p += count * arr.itemsize
        out[name] = arr
    return out


def main(argv: list[str]) -> int:
    subprocess.run(["make", "-f", "oracle/Makefile.ref", "-j8"], cwd=REPO, check=True)
    only = set(argv[1:])
    for name, args in CASES.items():
        if only and name not in only:
            continue
        raw = os.path.join(REPO, "oracle", "_ref", name + ".bin")
        with tempfile.TemporaryDirectory() as tmp:  # "@TMP": a scratch output directory
            cmd = [DUMP, args[0], raw] + [tmp if a == "@TMP" else a for a in args[1:]]
            subprocess.run(cmd, check=True)
        recs = read_records(raw)
        dst = os.path.join(HERE, name + ".npz")
        np.savez_compressed(dst, **recs)
        print(f"{name:16s} {len(recs):3d} arrays  {os.path.getsize(dst) / 1024:8.1f} KiB")
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv))
