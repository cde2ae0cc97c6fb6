"""Expert parallelism across the node's GPUs over NCCL: the
P > 1 exchange with real all-to-alls (graph-captured) equals the single-GPU
decoder bit for bit.  Skipped on a one-GPU box (the P > 1 device path is also
covered in one process: test_gpu_parity.py::test_ep_ranks_in_one_process...)."""

import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ep_over_nccl_on_every_gpu_equals_single_gpu():
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={min(n, 8)}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tools", "ep_multi_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "EP_MULTI_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
