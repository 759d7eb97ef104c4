"""FAST-mode RHS acceptance with an audit trail (TEST INFRASTRUCTURE).

Every FAST-vs-reference RHS comparison in the GPU suite goes through
`assert_fast_rhs`, which records the measured numbers and the branch that
accepted the case.  At the end of the session tests/conftest.py writes the
records to $SWEDG_PARITY_LOG (default gpurun_out/parity_log.jsonl);
tools/parity_table.py turns them into profiles/parity_r2.md.

Acceptance (SURVEY §7 "hard parts", scale convention test_solver.cpp:299-300):
  branch "rel"  max|du_fast - du_ref| / (1 + max|du_ref|) <= 1e-12   (north-star tolerance)
  branch "ld"   only when "rel" fails: FAST no less accurate than the reference,
                max|du_fast - du_exact| <= 4 max|du_ref - du_exact|,
                du_exact = the same algorithm in x87 long double (oracle/liboracle_ld.so).
"""
from __future__ import annotations

import os

import numpy as np

RHS_TOL = 1e-12
LD_FACTOR = 4.0
RECORDS: list[dict] = []


def rel(a, b) -> float:
    return float(np.abs(a - b).max() / (1.0 + np.abs(b).max()))


def _label(label: str | None) -> str:
    cur = os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0]
    return f"{cur}[{label}]" if label else cur


def assert_fast_rhs(du_fast, du_ref, exact_fn, label: str | None = None) -> dict:
    """exact_fn() -> du in long double (called only when the 1e-12 branch fails)."""
    r = rel(du_fast, du_ref)
    rec = {"case": _label(label), "rel": r, "tol": RHS_TOL, "branch": "rel", "e_fast": None, "e_ref": None,
           "ratio": None, "scale": float(np.abs(du_ref).max())}
    if r > RHS_TOL:
        exact = exact_fn()
        e_fast = float(np.abs(du_fast - exact).max())
        e_ref = float(np.abs(du_ref - exact).max())
        rec.update(branch="ld", e_fast=e_fast, e_ref=e_ref, ratio=e_fast / e_ref if e_ref > 0 else float("inf"))
        RECORDS.append(rec)
        assert e_fast <= LD_FACTOR * e_ref, \
            f"FAST error {e_fast:.3e} vs reference rounding error {e_ref:.3e} (rel {r:.3e})"
        return rec
    RECORDS.append(rec)
    return rec


def write(path: str) -> None:
    import json

    if not RECORDS:
        return
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "a") as f:
        for r in RECORDS:
            f.write(json.dumps(r) + "\n")
