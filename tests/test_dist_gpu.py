"""Multi-GPU executor (one process per GPU, NCCL P2P hops over NVLink, per-stage replica
all-reduce) on config C1 vs the CPU oracle; skipped on boxes with fewer than 2 GPUs."""

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multi_gpu_parity(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world), os.path.join(ROOT, "tools", "dist_parity.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    r = json.loads(line)
    assert r["order_ok"]
    assert abs(r["loss"] - r["ref_loss"]) / r["ref_loss"] < 2e-2
    assert r["loss2"] < r["loss"]
    for key, (cos, rel) in r["stage_cos_rel"].items():
        assert cos >= 0.99 and rel <= 6e-2, (key, cos, rel)
    assert abs(r["grad_norm"] - r["ref_grad_norm"]) / r["ref_grad_norm"] < 3e-2
