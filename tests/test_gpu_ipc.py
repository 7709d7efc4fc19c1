"""The peer-memory exchange across processes (CUDA IPC, tagc_ctx_peer_open):
tools/peer_ipc_check.py under torch.distributed.run, 2 and 3 processes on
cuda:0, checked against the CPU oracle on rank 0."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("nproc,width", [(2, 4), (3, 4), (2, 1)])
def test_peer_exchange_across_processes(nproc, width):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tools", "peer_ipc_check.py"), "--steps", "3", "--width", str(width)]
    env = dict(os.environ, TAGC_PEER_TIMEOUT_MS="60000")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "IPC peer exchange OK" in r.stdout, r.stdout[-2000:]
