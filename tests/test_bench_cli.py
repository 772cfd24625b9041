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


def test_eq1_counts_the_adapter():
    """Reading A7b: with an adapter of A bytes streaming every invocation,
    Eq. 1 (M_prefetch = max(M - T B, 0)) is applied to M + A, i.e. the planner
    gets T' = T - A / B; T' x B + A = T x B bytes cross PCIe in T."""
    sys.path.insert(0, ROOT)
    import bench
    B = 55.5e9
    assert bench.eq1_t_ttft(0.045, 0, B) == 0.045
    t = bench.eq1_t_ttft(0.045, 125173760, B)
    assert abs(t * B + 125173760 - 0.045 * B) < 1.0
    M = 26_030_000_000
    assert abs((M + 125173760 - 0.045 * B) - (M - t * B)) < 1.0   # same M_prefetch
    assert bench.eq1_t_ttft(0.001, 10**9, B) == 0.0                 # clamped like Eq. 1
