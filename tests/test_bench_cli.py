"""bench.py's multi-GPU launch contract on a CPU box:
`--gpus N` outside torchrun must spawn N ranks itself or, when fewer than N
GPUs are visible, exit non-zero with a clear message — never fall back to a
silent world = 1 run that reports n_gpus = 1."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                          capture_output=True, text=True, env=e, timeout=300)


def test_gpus_2_without_enough_gpus_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() >= 2:
        pytest.skip("this box has >= 2 GPUs")
    p = _run(["--gpus", "2", "--steps", "1", "--warmup", "1"])
    assert p.returncode != 0
    assert "needs 2 visible GPUs" in p.stderr
    assert '"n_gpus"' not in p.stdout


def test_world_size_mismatch_fails():
    p = _run(["--gpus", "2", "--steps", "1"], env={"WORLD_SIZE": "1", "RANK": "0",
                                                   "LOCAL_RANK": "0"})
    assert p.returncode != 0
    assert "WORLD_SIZE=1" in p.stderr


def test_reference_arm_rank_nonzero_exits_clean():
    """Under torchrun only rank 0 runs the oracle reference arm."""
    p = _run(["--impl", "reference", "--gpus", "2"], env={"WORLD_SIZE": "2", "RANK": "1",
                                                          "LOCAL_RANK": "1"})
    assert p.returncode == 0 and p.stdout.strip() == ""
