"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): row-slab decomposition, ghost-row
exchange schedule and NCCL-id bootstrap of SURVEY §8(e), with the oracle as the per-slab compute.

The library's slab path (tsw_create rank/nranks + exchange_nccl) uses exactly this schedule:
rank r owns global rows [r0, r1) (paper_2005_11931_b200.parallel.slab), keeps one ghost row
above/below, and after every level sends its first owned row to r−1 and its last owned row to
r+1.  Here each rank steps its slab with the oracle and exchanges with torch.distributed
send/recv; the gathered field must equal the single-domain oracle run bitwise.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2005_11931_b200 import inputs, parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg():
    return inputs.config(2, nx=70, ny=53, dx=0.02, dy=0.02, kind=inputs.H_DELTA_LINE_X, eps=[0.2], amp=[1.0], dt=2e-3)


def _exchange(u, rank, world, top_ghost, bot_ghost):
    """Ghost-row exchange of the local array u (rows: [ghost?] owned... [ghost?])."""
    reqs = []
    first = 1 if top_ghost else 0
    last = u.shape[0] - 2 if bot_ghost else u.shape[0] - 1
    send_up = torch.from_numpy(np.ascontiguousarray(u[first]))
    send_dn = torch.from_numpy(np.ascontiguousarray(u[last]))
    recv_up = torch.empty_like(send_up)
    recv_dn = torch.empty_like(send_dn)
    if rank > 0:
        reqs += [dist.isend(send_up, rank - 1), dist.irecv(recv_up, rank - 1)]
    if rank < world - 1:
        reqs += [dist.isend(send_dn, rank + 1), dist.irecv(recv_dn, rank + 1)]
    for r in reqs:
        r.wait()
    if rank > 0:
        u[0] = recv_up.numpy()
    if rank < world - 1:
        u[-1] = recv_dn.numpy()


def _worker(rank, world, port, nsteps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = _cfg()
        r0, r1 = parallel.slab(cfg.ny, rank, world)
        top = rank > 0                    # ghost row above (rank 0 starts at the boundary row)
        bot = rank < world - 1
        j0 = r0 - (1 if top else 0)
        j1 = r1 + (1 if bot else 0)
        _, _, c1, c2 = oracle.member_coefficients(cfg, 0, np.float64, 0, j0, cfg.nx, j1 - j0)
        u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, j0, j1 - j0)
        # start-up (R11), exchange, then leapfrog levels each followed by the exchange
        v = oracle.startup(2, c1, c2, u0, None, cfg.dt)
        _exchange(v, rank, world, top, bot)
        un, unm1 = v, u0
        for _ in range(nsteps - 1):
            un, unm1 = oracle.leapfrog(2, c1, c2, un, unm1, 1)
            _exchange(un, rank, world, top, bot)
        own = un[(1 if top else 0):(un.shape[0] - (1 if bot else 0))]
        assert own.shape[0] == r1 - r0
        out = [None] * world
        dist.all_gather_object(out, (r0, own))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_exchange_equals_single_domain(world):
    nsteps = 40
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nsteps, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = _cfg()
    full, _, _, _ = oracle.run_member(cfg, 0, np.float64, nsteps=nsteps,
                                      u0=inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny))
    got = np.concatenate([own for (_, own) in sorted(parts, key=lambda t: t[0])])
    assert np.array_equal(got, full)


def test_slab_partition_matches_library_and_covers_grid():
    for ny in (3, 53, 4096, 32768):
        for P in (1, 2, 3, 4, 8):
            if ny < 2 * P:
                continue
            rows = [parallel.slab(ny, r, P) for r in range(P)]
            assert rows[0][0] == 0 and rows[-1][1] == ny
            assert all(rows[k][1] == rows[k + 1][0] for k in range(P - 1))
            assert all(inputs.slab_rows(ny, r, P) == rows[r] for r in range(P))
            assert max(b - a for a, b in rows) - min(b - a for a, b in rows) <= 1


def _boot_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2005_11931_b200 import tsw
        got = {}
        tsw.tsw_nccl_unique_id = lambda: bytes([7] * 64 + list(range(64)))   # no GPU needed here
        tsw.tsw_nccl_init = lambda ctx, uid: got.setdefault("uid", uid)

        class S:
            pass
        s = S()
        s.rank, s.nranks, s.ctx = rank, world, None
        parallel.nccl_bootstrap(s)
        out = [None] * world
        dist.all_gather_object(out, got.get("uid"))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_nccl_id_bootstrap_broadcasts_rank0_id():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_boot_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ids = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(i == ids[0] for i in ids) and len(ids[0]) == 128
