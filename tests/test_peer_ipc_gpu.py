"""Peer halos across processes (CUDA IPC): two ranks on one GPU, stepped in host
lock step (tests/peer_ipc_worker.py) — bitwise equal to the single-domain run."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("K,nsteps", [(1, 9), (4, 23), (8, 23)])
def test_peer_halo_ipc_two_processes(K, nsteps):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29611", os.path.join(ROOT, "tests", "peer_ipc_worker.py"),
           str(K), str(nsteps)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"peer-ipc ok K={K}" in r.stdout
