import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionfinish(session, exitstatus):
    """FAST-mode parity audit trail (tests/parity_log.py)."""
    import parity_log

    path = os.environ.get("SWEDG_PARITY_LOG", os.path.join(REPO, "gpurun_out", "parity_log.jsonl"))
    parity_log.write(path)
