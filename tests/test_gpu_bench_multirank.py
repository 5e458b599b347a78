"""bench.py's multi-rank path (torchrun, particle shards, max-over-ranks
timing, the stage-time re-run from the restored shard state) run as two ranks
on one GPU with gloo and host-staged exchanges (SMCL_BENCH_GLOO=1). A
functional check of the contract the driver's N-GPU runs use, not a
measurement: the line must count every shard's particle-points once."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_rank_bench_line():
    n = 65536
    env = dict(os.environ, SMCL_BENCH_GLOO="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--particles", str(n)]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 prints one JSON line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 3
    assert d["config"]["pp_per_step"] == 2 * n * d["config"]["scan_points"]
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert "shards x2" in d["config"]["parallelism"]
