"""bench.py's --gpus N launch: re-exec under torch.distributed.run with one process per rank
(gloo + the oracle-backed CPU plan via the --cpu-test hook, so no GPU is needed), the
max-over-ranks timing, and rank 0's single JSON line."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(*argv, env=None):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], capture_output=True, text=True,
                         timeout=300, env=e, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    return lines


def test_launch_command_shapes():
    import bench

    assert bench.launch_command(1, []) is None
    cmd = bench.launch_command(4, ["--gpus", "4", "--steps", "3"])
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "127.0.0.1" in cmd and cmd[-3:] == ["--gpus", "4", "--steps", "3"][-3:]
    os.environ["WORLD_SIZE"] = "2"
    try:
        assert bench.launch_command(2, []) is None  # already under torchrun
        with pytest.raises(SystemExit):
            bench.launch_command(4, [])
    finally:
        del os.environ["WORLD_SIZE"]


@pytest.mark.parametrize("gpus", [1, 2])
def test_gpus_n_spawns_n_ranks(gpus):
    lines = _run("--gpus", str(gpus), "--cpu-test", "--steps", "1", "--warmup", "1")
    assert len(lines) == 1, lines  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["value"] > 0
    owners = {int(r): a for r, a in d["ranks_agents"].items()}
    assert sorted(i for a in owners.values() for i in a) == [0, 1, 2, 3]
    if gpus == 2:
        assert owners[0] == [0, 2] and owners[1] == [1, 3]


def test_multirank_time_to_rmse_path():
    """--gpus 2 with a time-to-RMSE budget: the per-iteration NRMSE of the global consensus image
    from a fresh two-rank solve, the first iteration after which it stays <= 1e-3."""
    lines = _run("--gpus", "2", "--cpu-test", "--steps", "1", "--warmup", "1", "--ttr-iters", "300")
    d = json.loads(lines[0])
    t = d["time_to_rmse_1e-3"]
    assert t["ran_iterations"] == 300 and isinstance(t["iterations"], int) and 1 < t["iterations"] < 300
    assert t["final_nrmse"] <= 1e-3 and t["seconds"] > 0
