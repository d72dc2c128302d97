"""Multi-GPU (NCCL over NVLink) parity: the sharded path equals the
single-GPU path on every rank. Needs >= 2 GPUs (gpurun --gpus 2); the
host-side logic is covered on CPU by tests/test_parallel_cpu.py (gloo)."""
import json
import os
import socket
import subprocess
import sys
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_graph_and_replay_nccl(ls):
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(n, 4)
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                            "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                            os.path.join(ROOT, "tests", "mp", "nccl_worker.py")],
                           capture_output=True, text=True, timeout=600, env=dict(os.environ, LSG_MP_OUT=d))
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
        lines = [json.load(open(os.path.join(d, f))) for f in sorted(os.listdir(d))]
    assert len(lines) == n and all(all(x["ok"].values()) for x in lines), lines
