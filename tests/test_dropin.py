"""The C++ drop-in path (include/swedg_b200.hpp) inside a program built from the
UNMODIFIED reference: reference rhs()/entropy_projection()/step_lsrk45 vs the
adapter's, in-process (oracle/dropin_test.cpp, built into oracle/_ref/)."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "oracle", "_ref", "dropin_test")


@pytest.mark.gpu
def test_cpp_dropin_against_reference():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all drop-in checks passed" in r.stdout


def test_dropin_adapter_header_compiles_standalone(tmp_path):
    """The adapter header is self-contained C++17 over the C ABI (no torch, no CUDA types)."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "swedg_b200.hpp"\nint main() { return swedg_abi_version() == SWEDG_ABI_VERSION ? 0 : 1; }\n')
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I", os.path.join(REPO, "include"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
