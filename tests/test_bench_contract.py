"""bench.py's driver contract on the CPU side: the reference arm's JSON line (it runs
the unmodified reference, oracle/_ref/swedg_refbench, on this host) and the launch
logic (--gpus N without a torchrun environment re-executes under torch.distributed.run;
a mismatched WORLD_SIZE is refused)."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref", "swedg_refbench")
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"}


def run_bench(*args, env=None, timeout=600):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, env=e, cwd=REPO)


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref/swedg_refbench not built")
def test_reference_arm_json_line():
    r = run_bench("--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-k1d", "32", "--no-extra")
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["higher_is_better"] is True and d["dtype"] == "f64"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] == os.cpu_count() and cb["value"] == d["value"]
    assert cb["nproc"] == os.cpu_count() and cb["cpu_model"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_non_zero_ranks_exit_quietly():
    """Under torchrun only rank 0 runs the reference arm; the others exit 0 without work."""
    r = run_bench("--impl", "reference", "--gpus", "2", env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_world_size_must_match_gpus():
    r = run_bench("--gpus", "4", env={"RANK": "0", "WORLD_SIZE": "2", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_gpus_without_torchrun_respawns_under_torch_distributed_run(monkeypatch):
    """--gpus N with no WORLD_SIZE re-executes bench.py under torch.distributed.run with N
    ranks on 127.0.0.1 (checked without launching: the command line is captured)."""
    sys.path.insert(0, REPO)
    import bench

    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8", "--scaling", "strong"])
    assert bench.main() == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-3:] == ["--gpus", "8", "--scaling", "strong"][-3:]
    assert os.environ.get("NCCL_DEBUG") == "INFO"
