"""Worker for test_peer_ipc_gpu: two processes, one GPU, peer halos over CUDA IPC handles, stepped
in host lock step (one halo operation per rank per turn, a gloo barrier in between: no waiter
ever spins).  Rank 0 gathers the slabs and compares them with the single-domain run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from paper_2005_11931_b200 import inputs, parallel, tsw
from tests.helpers import check_slabs_against_oracle, slab_record


def lockstep(rank, world, fn):
    """fn() on rank 0, then rank 1, …, each followed by a barrier; returns this rank's result."""
    out = None
    for r in range(world):
        if r == rank:
            out = fn()
            torch.cuda.synchronize()
        dist.barrier()
    return out


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    K, nsteps = int(sys.argv[1]), int(sys.argv[2])
    dist.init_process_group("gloo", init_method="env://")
    torch.cuda.set_device(0)
    cfg = inputs.config(3, nx=700, ny=151, dx=0.01, dy=0.01, eps=[0.1, 0.3], amp=[1.0, 2.0], dt=2e-3)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
    s = tsw.Solver.from_config(cfg, "f64", rank=rank, nranks=world, device=0)
    if K > 1:
        s.set_option(tsw.TSW_OPT_TBLOCK, K)
    parallel.peer_bootstrap(s)                       # CUDA IPC handles through an all-gather
    lockstep(rank, world, lambda: s.set_initial(np.ascontiguousarray(u0[s.r0:s.r0 + s.ny_local]), None, cfg.dt,
                                                flags=tsw.TSW_INIT_SHARED))
    done, ops = 0, 0
    while done < nsteps:
        used = lockstep(rank, world, lambda: tsw.tsw_step_op(s.ctx, nsteps - done))
        used = [used]
        dist.broadcast_object_list(used, src=0)      # every rank advances identically
        done += used[0]
        ops += 1
    E = lockstep(rank, world, lambda: s.energy())
    mine = (s.r0, s.read(0), s.read(1), E, tsw.tsw_peer_state(s.ctx), slab_record(s))
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    if rank == 0:
        ref = tsw.Solver.from_config(cfg, "f64")
        if K > 1:
            ref.set_option(tsw.TSW_OPT_TBLOCK, K)
        ref.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
        ref.step(nsteps)
        g, gp = ref.read(0), ref.read(1)
        for r0, a, b, _, state, _ in allp:
            assert np.array_equal(a, g[:, r0:r0 + a.shape[1]]), f"u^n slab at row {r0}"
            assert np.array_equal(b, gp[:, r0:r0 + b.shape[1]]), f"u^(n-1) slab at row {r0}"
            assert state[3] == 0, "a waiter timed out"
        check_slabs_against_oracle([p[5] for p in allp], cfg, "f64", nsteps, u0)
        Es = sum(p[3] for p in allp)
        np.testing.assert_allclose(Es, ref.energy(), rtol=1e-12)
        print(f"peer-ipc ok K={K} steps={nsteps} ops={ops}", flush=True)
    dist.barrier()
    s.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
