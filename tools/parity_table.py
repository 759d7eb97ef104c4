"""gpurun_out/parity_log.jsonl (tests/parity_log.py records of a `pytest -m gpu` run)
-> a markdown table of every FAST-mode RHS comparison: the measured relative error,
the branch that accepted it, and, for the long-double branch, FAST's and the
reference's own error against the long-double evaluation.

    python tools/parity_table.py gpurun_out/parity_log.jsonl > profiles/parity_r2.md
"""
import json
import sys


def main(path):
    recs, seen = [], set()
    for ln in open(path):
        r = json.loads(ln)
        key = (r["case"], r["rel"])
        if key in seen:
            continue
        seen.add(key)
        recs.append(r)
    n_ld = sum(r["branch"] == "ld" for r in recs)
    print("# FAST-mode RHS parity, every comparison of the GPU suite\n")
    print("Acceptance (tests/parity_log.py): branch `rel` = max|du_fast - du_ref| / (1 + max|du_ref|) <= 1e-12")
    print("(the north-star tolerance, scale convention of test_solver.cpp:299-300); branch `ld` only")
    print("when `rel` fails: FAST no less accurate than the reference, max|du_fast - du_exact| <= 4 max|du_ref -")
    print("du_exact|, du_exact = the same algorithm in x87 long double (oracle/liboracle_ld.so).")
    print("PARITY mode is asserted bitwise in every one of these tests and is not listed.\n")
    print(f"{len(recs)} comparisons: {len(recs) - n_ld} pass the 1e-12 bound, {n_ld} only through the "
          "long-double branch (listed first).\n")
    print("| case | rel. error vs reference | branch | FAST err vs long double | reference err vs long double | ratio |")
    print("|---|---|---|---|---|---|")
    for r in sorted(recs, key=lambda r: (r["branch"] != "ld", r["case"])):
        case = r["case"].replace("tests/", "").replace("|", "/")
        e_fast = "—" if r["e_fast"] is None else f"{r['e_fast']:.3e}"
        e_ref = "—" if r["e_ref"] is None else f"{r['e_ref']:.3e}"
        ratio = "—" if r["ratio"] is None else f"{r['ratio']:.2f}"
        print(f"| `{case}` | {r['rel']:.3e} | {r['branch']} | {e_fast} | {e_ref} | {ratio} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_log.jsonl")
