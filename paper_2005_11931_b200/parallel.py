"""Process-group plumbing for row slabs: one process per GPU, torch.distributed for
rendezvous and for broadcasting the NCCL unique id; the halo exchange itself runs inside
libtsw.so (ncclSend/ncclRecv on the ctx stream), not in Python."""
from __future__ import annotations

import os
from typing import Tuple

from . import tsw


def env_rank() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process ⇒ 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init_process_group(backend: str = "nccl"):
    """Initialise torch.distributed when WORLD_SIZE > 1 (MASTER_ADDR defaults to 127.0.0.1)."""
    import torch.distributed as dist
    rank, world, local = env_rank()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        kw = {}
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    return rank, world, local


def slab(ny: int, rank: int, nranks: int) -> Tuple[int, int]:
    """Rows [r0, r1) of rank (same split as tsw_create: the first ny % P ranks get one more row)."""
    base, rem = divmod(ny, nranks)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


def nccl_bootstrap(solver: "tsw.Solver") -> None:
    """Rank 0 creates an ncclUniqueId, torch.distributed broadcasts it, every rank joins."""
    import torch.distributed as dist
    if solver.nranks <= 1:
        return
    obj = [tsw.tsw_nccl_unique_id() if solver.rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    tsw.tsw_nccl_init(solver.ctx, obj[0])


def peer_bootstrap(solver: "tsw.Solver") -> None:
    """Peer halos (TSW_OPT_HALO = 1): every rank exports IPC handles of its buffers, an all-gather
    distributes them, each rank maps its neighbours (rank ± 1).  Call after TSW_OPT_TBLOCK and
    before set_initial; no NCCL communicator is needed for the halos."""
    import torch.distributed as dist
    if solver.nranks <= 1:
        return
    solver.set_option(tsw.TSW_OPT_HALO, 1)
    blobs = [None] * solver.nranks
    dist.all_gather_object(blobs, solver.peer_export())
    neighbours = peer_neighbours(solver.rank, solver.nranks)
    for side, r in neighbours:
        solver.peer_import(side, blobs[r])
    dist.barrier()


def peer_neighbours(rank: int, nranks: int):
    """(side, rank) of the slab neighbours: side 0 = rank − 1 (above), side 1 = rank + 1 (below)."""
    out = []
    if rank > 0:
        out.append((0, rank - 1))
    if rank < nranks - 1:
        out.append((1, rank + 1))
    return out
