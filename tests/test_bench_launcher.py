"""`python bench.py --gpus N` starts N ranks itself when it is not already under torchrun
(the driver's 1/2/4/8-GPU command must reach the multi-rank path).  On CPU the
launcher check runs the GPU arm's rank plumbing -- spawn, contiguous shards, in-place
all-gather, max over ranks -- over gloo with index-derived placeholder results."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    return env


@pytest.mark.parametrize("n", [2, 3])
def test_bench_gpus_n_spawns_n_ranks(n):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--launcher-check",
                        "--config", "cfg1"], capture_output=True, text=True, timeout=600, env=_env(), cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout          # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["launcher_check"] is True and rec["n_gpus"] == n
    per = -(-256 // n)
    assert rec["motions_per_rank"] == [float(min(256, (k + 1) * per) - min(256, k * per)) for k in range(n)]
    assert rec["gathered_ok_per_rank"] == [1.0] * n and rec["max_over_ranks"] == float(n)


def test_bench_refuses_mismatched_world():
    env = _env()
    env.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launcher-check",
                        "--config", "cfg1"], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0 and "--gpus 2 but 1 rank" in (r.stderr + r.stdout)
