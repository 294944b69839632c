"""bench.py --gpus 2 launches two ranks itself (torch.distributed.run re-exec) and runs the sharded
slide path end to end: contiguous tile shards, the size all-gather, the device archive, the host
path into one /dev/shm archive shared by the ranks, max-over-ranks timing.  On a one-GPU box the
ranks share the GPU and exchange through gloo (WBPC_BENCH_BACKEND); measured runs use NCCL."""

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_self_launches_two_ranks():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, WBPC_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--tiles", "8", "--steps", "1",
                        "--warmup", "3", "--no-cpu", "--e2e-steps", "1"], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["tiles"] == 8 and d["run"]["tiles_per_gpu"] == 4
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["encode_mps"] > 0 and d["decode_mps"] > 0
