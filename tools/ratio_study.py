#!/usr/bin/env python3
"""R_GPU study (bench.hpp:55-201).

For each matrix size n of the reference's default_bench_sizes(), time the
traditional DG volume kernel (dense y = Q f(u)) and the ESDG flux-differencing
kernel (y_i = sum_j 2 Q_ij f_S(u_i, u_j)) on the B200 (swedg_ratio_kernels,
CUDA events, median of reps) and report R_GPU = t_ESDG / t_DG, beside the
reference's own R_CPU (oracle/_ref/swedg_refbench ratio: the unmodified
ratio_sweep, serial, on this host).  Random operators/states as ratio_sweep
draws them (Q in [-1,1], h in [0.5,2], velocities in [-1,1]); the element
count is chosen so every launch holds 2^24 nodes (GPU-sized work; the CPU
sweep grows K from 64 until a run takes > 0.1 ms, as ratio_sweep does).

    python tools/ratio_study.py [--nodes 16777216] [--reps 7] [--json out.json]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2005_02516_b200 import capi  # noqa: E402

SIZES = [6, 10, 15, 21, 28, 36, 50, 100, 200]  # bench.hpp:208-210 default_bench_sizes


def states(n, K, rng):
    h = rng.uniform(0.5, 2.0, (K, n))
    u = np.empty((K, 3, n))
    u[:, 0] = h
    u[:, 1] = h * rng.uniform(-1.0, 1.0, (K, n))
    u[:, 2] = h * rng.uniform(-1.0, 1.0, (K, n))
    return u


def cpu_ratios():
    exe = os.path.join(REPO, "oracle", "_ref", "swedg_refbench")
    if not os.path.exists(exe):
        return {}
    out = subprocess.run([exe, "ratio", "64", "1"], capture_output=True, text=True, check=True).stdout
    rows = {}
    for line in out.strip().splitlines()[1:]:
        n, el, reps, te, td, r, sp = line.split(",")
        rows[int(n)] = {"elements": int(el), "t_esdg_s": float(te), "t_dg_s": float(td), "R_CPU": float(r)}
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    cpu = cpu_ratios()
    rng = np.random.default_rng(0)
    rows = []
    for n in SIZES:
        K = max(1, a.nodes // n)
        Q = rng.uniform(-1.0, 1.0, (n, n))
        u = states(n, K, rng)
        row = {"n": n, "elements": K}
        for mode, tag in ((capi.MODE_FAST, "fast"), (capi.MODE_PARITY, "parity")):
            tdg, tes, _, _ = capi.ratio_kernels(Q, u, mode=mode, reps=a.reps, outputs=False)
            pairs = K * n * n
            row[tag] = {"t_dg_ms": round(tdg, 4), "t_esdg_ms": round(tes, 4), "R_GPU": round(tes / tdg, 3),
                        "esdg_gpairs_per_s": round(pairs / (tes * 1e-3) / 1e9, 2),
                        "dg_gbs": round(K * 6 * n * 8 / (tdg * 1e-3) / 1e9, 1)}
        if n in cpu:
            row["cpu_reference"] = cpu[n]
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)
    print("\n| n | elements | t_DG ms | t_ESDG ms | R_GPU (FAST) | R_GPU (PARITY) | R_CPU (reference) |")
    print("|---|---|---|---|---|---|---|")
    for r in rows:
        rc = r.get("cpu_reference", {}).get("R_CPU")
        print(f"| {r['n']} | {r['elements']} | {r['fast']['t_dg_ms']} | {r['fast']['t_esdg_ms']} | "
              f"{r['fast']['R_GPU']} | {r['parity']['R_GPU']} | {'' if rc is None else round(rc, 3)} |")


if __name__ == "__main__":
    sys.exit(main())
