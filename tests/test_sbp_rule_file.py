"""SBP rule files: sbp_rule / load_sbp_rule_file
(quadrature.hpp:290-343) restated in the native setup (setup.cpp), checked against
the reference's own loader (oracle/_ref/ref_sbp_rule, built from the unmodified
headers when /root/reference is present) and against the built-in tables.

Gauss-Legendre-edge rules come from the tables; Gauss-Lobatto-edge rules exist only
as data files sbp_lobatto_N<N>.txt (none ships with the reference).  The loader is
exercised on a file written from the Legendre N=2 rule, plus every error path of the
reference (missing file, header mismatch, non-embedding surface nodes, nonpositive
weight, failed exactness)."""
import os
import subprocess

import numpy as np
import pytest

from paper_2005_02516_b200 import capi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref", "ref_sbp_rule")


def write_rule(path, rule, degree, npf, perturb=None):
    x, y, w = rule["x"].copy(), rule["y"].copy(), rule["w"].copy()
    if perturb:
        perturb(x, y, w)
    with open(path, "w") as f:
        f.write(f"degree={degree} nodes_per_face={npf}\n")
        for a, b, c in zip(x, y, w):
            f.write(f"{float(a)!r} {float(b)!r} {float(c)!r}\n")  # shortest round-trip decimal: exact


def ref_rule(N, family, data_dir="-", rule_file="-"):
    """The reference's loader: (dict or None, error message or None)."""
    r = subprocess.run([REF, str(N), str(family), data_dir, rule_file], capture_output=True, text=True)
    lines = r.stdout.strip().splitlines()
    if lines[0].startswith("error"):
        return None, lines[0][6:]
    _, nq, npf = lines[0].split()
    xyw = np.array([[float.fromhex(t) for t in ln.split()] for ln in lines[1:1 + int(nq)]])
    fi = np.array([int(t) for t in lines[1 + int(nq)].split()], dtype=np.int32)
    return {"x": xyw[:, 0], "y": xyw[:, 1], "w": xyw[:, 2], "npf": int(npf), "face_index": fi}, None


def same(a, b):
    for k in ("x", "y", "w", "face_index"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    assert a["npf"] == b["npf"]


def test_rule_file_round_trip_equals_table_rule(tmp_path):
    tab = capi.sbp_rule(2)
    p = tmp_path / "legendre_n2.txt"
    write_rule(p, tab, 3, tab["npf"])
    same(capi.sbp_rule(2, capi.SBP_LEGENDRE, rule_file=str(p)), tab)
    if os.path.exists(REF):
        r, err = ref_rule(2, 0, rule_file=str(p))
        assert err is None
        same(r, tab)
        r, err = ref_rule(2, 0)
        same(r, tab)  # the reference's table rule


def test_case_from_rule_file_equals_table_case(tmp_path):
    tab = capi.sbp_rule(2)
    p = tmp_path / "legendre_n2.txt"
    write_rule(p, tab, 3, tab["npf"])
    a = capi.Case("vortex", scheme=capi.SCHEME_SBP, N=2, nx=4, threads=1)
    b = capi.Case("vortex", scheme=capi.SCHEME_SBP, N=2, nx=4, threads=1, sbp_rule_file=str(p))
    for name in ("Qr", "Qs", "M_diag", "gf", "sJ", "u0", "b", "J_vol"):
        np.testing.assert_array_equal(a.array(name), b.array(name), err_msg=name)
    np.testing.assert_array_equal(a.iarray("face_index"), b.iarray("face_index"))


@pytest.mark.parametrize("what", ["missing", "lobatto_missing", "header", "weight", "exactness", "embed"])
def test_rule_file_errors_match_reference(tmp_path, what):
    """Every failure of the reference's loader, same message (test_quadrature.cpp:127-129)."""
    tab = capi.sbp_rule(2)
    p = tmp_path / "rule.txt"
    fam, data_dir, rule_file, expect = capi.SBP_LEGENDRE, None, str(p), None
    if what == "missing":
        rule_file = str(tmp_path / "nope.txt")
        expect = "unavailable"
    elif what == "lobatto_missing":  # sbp_rule(2, GaussLobatto, "/nonexistent")
        fam, data_dir, rule_file, expect = capi.SBP_LOBATTO, "/nonexistent", None, "unavailable"
    elif what == "header":
        write_rule(p, tab, 2, tab["npf"])  # degree 2 < 2N - 1 = 3
        expect = "header mismatch"
    elif what == "weight":
        write_rule(p, tab, 3, tab["npf"], perturb=lambda x, y, w: w.__setitem__(5, -w[5]))
        expect = "nonpositive weight"
    elif what == "exactness":  # verify_exactness flags a broken rule (test_quadrature.cpp:132-136)
        write_rule(p, tab, 3, tab["npf"], perturb=lambda x, y, w: w.__setitem__(10, w[10] + 1e-6))
        expect = "exactness"
    elif what == "embed":  # Lobatto edge nodes (corners) are not nodes of the Legendre rule
        d = tmp_path / "data"
        d.mkdir()
        write_rule(d / "sbp_lobatto_N2.txt", tab, 3, 4)
        fam, data_dir, rule_file, expect = capi.SBP_LOBATTO, str(d), None, "does not embed"
    with pytest.raises(capi.InvalidArgument) as ei:
        capi.sbp_rule(2, fam, data_dir=data_dir, rule_file=rule_file)
    assert expect in str(ei.value)
    if os.path.exists(REF):
        r, err = ref_rule(2, fam, data_dir or "-", rule_file or "-")
        assert r is None and err == str(ei.value)


def test_gauss_lobatto_edges_match_reference(tmp_path):
    """A rule whose surface is Gauss-Lobatto: the volume rule of the file holds the edge
    nodes of the 4-point Lobatto rule on every face (corners twice) — the reference's
    embedding check rejects shared corner nodes, and so does the restatement."""
    pts = []
    for f in range(3):
        for r in (-1.0, -1 / np.sqrt(5), 1 / np.sqrt(5), 1.0):
            pts.append([(r, -1.0), (-r, r), (-1.0, -r)][f])
    rule = {"x": np.array([p[0] for p in pts]), "y": np.array([p[1] for p in pts]), "w": np.full(len(pts), 1 / 6)}
    d = tmp_path / "d"
    d.mkdir()
    write_rule(d / "sbp_lobatto_N2.txt", rule, 3, 4)
    with pytest.raises(capi.InvalidArgument) as ei:
        capi.sbp_rule(2, capi.SBP_LOBATTO, data_dir=str(d))
    if os.path.exists(REF):
        _, err = ref_rule(2, 1, str(d))
        assert err == str(ei.value)
