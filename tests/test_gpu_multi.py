"""Real multi-GPU runs of the row-sharded solve (one process per GPU, NCCL
communicator, fused peer exchange over NVLink via CUDA IPC for dense C, NCCL
allreduce in CUDA-graph slots for the on-the-fly cost), checked against the
oracle and for identical decisions on every rank (tests/multi/sharded_case.py).
Skipped on boxes with fewer than 2 GPUs -- the GPU pool of this build gives one
GPU per call, so the multi-rank logic is also covered by the emulated-rank
GPU tests and the world-size-2 gloo tests."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("G", [2, 4, 8])
def test_sharded_solve_on_real_gpus(G):
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs, this box has {torch.cuda.device_count()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "multi", "sharded_case.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env=dict(os.environ, PYTHONPATH=ROOT))
    out = p.stdout + p.stderr
    assert p.returncode == 0 and "MULTI OK" in out, out[-5000:]
