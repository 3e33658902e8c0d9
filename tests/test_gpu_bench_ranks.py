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
