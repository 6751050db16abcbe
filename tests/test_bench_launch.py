"""bench.py's multi-GPU launch path on CPU: `bench.py --gpus 2` with no launcher re-executes
itself under torchrun (2 ranks, rendezvous on 127.0.0.1), times with barriers and the max over
ranks, and rank 0 alone prints exactly one JSON line with n_gpus = 2.  The GPU step is replaced by
a gloo allreduce of gradient rows (GSLIC_BENCH_PLUMBING=1); the device path itself is covered by
tests/test_dp_gpu.py."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(300)
def test_bench_self_spawns_two_ranks():
    env = dict(os.environ, GSLIC_BENCH_PLUMBING="1", OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "5",
                        "--warmup", "3"], capture_output=True, text=True, env=env, timeout=280)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["plumbing"] is True and out["steps"] == 5 and out["warmup"] == 3
    assert out["union_rows"] > 0 and out["config"]["parallelism"] == "dp2"
