"""The multi-rank path from C++ through the C ABI (tests/cpp/multirank_test.cpp):
logical partitions with an exchange callback, and one rank exchanging across its own periodic
cut through the peer-memory transport and through a one-rank NCCL communicator."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "tests", "cpp", "multirank_test")


@pytest.mark.gpu
def test_cpp_multirank_partitions_and_nccl():
    assert os.path.exists(BIN), "tests/cpp/multirank_test not built (__graft_entry__.build())"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all multi-rank checks passed" in r.stdout


def test_cpp_multirank_test_builds():
    """The binary links the C ABI, the setup ABI and the adapter only (no torch)."""
    assert os.path.exists(BIN), "tests/cpp/multirank_test not built (__graft_entry__.build())"
