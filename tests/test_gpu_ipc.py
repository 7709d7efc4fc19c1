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


def test_bench_two_ranks_plumbing():
    """bench.py's N > 1 code (rank timing, max over ranks, owner step,
    overlap, e2e, one JSON line from rank 0) with 2 ranks sharing cuda:0 over
    the peer exchange (TAGC_BENCH_SHARE_GPU=1: a plumbing check only)."""
    import json
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3", "--exchange", "peer"]
    env = dict(os.environ, TAGC_BENCH_SHARE_GPU="1", TAGC_PEER_TIMEOUT_MS="60000")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["peel"]["unresolved"] == 0
    g = d["extras"]["gpt2"]  # the owner step and the overlap run on the GPT-2 extra line
    assert g["owner_step"]["fused_ms"] > 0 and g["overlap"]["overlapped_ms"] > 0 and d["e2e"]["value"] > 0
