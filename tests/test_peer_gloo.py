"""Peer-halo bootstrap host logic on CPU (gloo, world_size 2 and 3): every rank
turns peer halos on, all-gathers its export blob, and maps exactly its slab neighbours — rank − 1
on side 0 and rank + 1 on side 1 — with their own blobs.  (The device side, the IPC mapping and
the stepping are covered by tests/test_peer_gpu.py and tests/test_peer_ipc_gpu.py.)"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_11931_b200 import parallel, tsw


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeSolver:
    def __init__(self, rank, nranks):
        self.rank, self.nranks = rank, nranks
        self.options, self.imports = {}, []

    def set_option(self, key, value):
        self.options[key] = value

    def peer_export(self):
        return f"blob-of-rank-{self.rank}".encode()

    def peer_import(self, side, blob):
        self.imports.append((side, blob.decode()))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = FakeSolver(rank, world)
    parallel.peer_bootstrap(s)
    q.put((rank, s.options, s.imports))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_bootstrap_maps_slab_neighbours(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, opts, imps = q.get(timeout=120)
        res[r] = (opts, imps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        opts, imps = res[r]
        assert opts.get(tsw.TSW_OPT_HALO) == 1
        want = []
        if r > 0:
            want.append((0, f"blob-of-rank-{r - 1}"))
        if r < world - 1:
            want.append((1, f"blob-of-rank-{r + 1}"))
        assert imps == want


def test_peer_neighbours_edges():
    assert parallel.peer_neighbours(0, 1) == []
    assert parallel.peer_neighbours(0, 4) == [(1, 1)]
    assert parallel.peer_neighbours(3, 4) == [(0, 2)]
    assert parallel.peer_neighbours(1, 4) == [(0, 0), (1, 2)]
