"""bench.py's N>1 path end to end under torchrun, on the one GPU this box has.

Both ranks run on cuda:0 with gloo for the host-side plumbing (SCR_BENCH_ONE_GPU test hook):
rank 0 adapts and broadcasts the prediction table, the ranks relocalise disjoint frame shards
with no per-frame collective, and rank 0 prints one JSON line with the max-over-ranks time and
the frames of both ranks. Nothing here waits on another rank's kernels.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_two_ranks_json_line():
    env = dict(os.environ, SCR_BENCH_ONE_GPU="1", SCR_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", "bench.py", "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--batch", "16", "--test-frames", "32", "--adapt-frames", "40", "--lanes", "1",
           "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 3
    assert d["scaling"] == "weak" and d["value"] > 0
    # both ranks' frames are counted: value = 2 ranks x steps x batch / max-over-ranks time
    assert abs(d["value"] * d["ms_per_step"] / 1e3 - 2 * 16) < 0.05 * 2 * 16
    assert d["adapt"]["broadcast_ms"] is not None


@pytest.mark.gpu
def test_bench_self_launches_ranks_for_gpus_flag():
    """`python bench.py --gpus 2` (no torchrun) starts two ranks itself; config 4 shards the
    8 scenes 4 + 4 over them and rank 0 reports the frames of both ranks."""
    env = dict(os.environ, SCR_BENCH_ONE_GPU="1", SCR_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--workload", "scenes", "--steps", "1", "--warmup", "3",
           "--batch", "8", "--test-frames", "16", "--adapt-frames", "30", "--lanes", "1", "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["comm"]["nranks"] == 2 and d["scaling"] == "strong"
    assert d["config"]["scenes_on_rank0"] == [1, 3, 5, 7]
    # 2 ranks x 4 scenes x 1 lane x 8 frames per step
    assert abs(d["value"] * d["ms_per_step"] / 1e3 - 64) < 0.05 * 64
