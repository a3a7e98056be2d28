"""Peer halos (TSW_OPT_HALO = 1): the temporally blocked stencil stores its first /
last K owned rows straight into the neighbours' ghost rows through mapped peer pointers, one-level
steps push their boundary row with a copy kernel, and every halo operation is ordered by epochs
(a one-thread waiter on the rank's local mailbox, a signal into the neighbours' mailboxes).  Here
the ranks are ctxs of one process on one GPU sharing one stream, stepped by tsw_group_step epoch by
epoch, so every waiter finds its condition already met (nothing spins on one GPU).  Results must be
bitwise those of the single-domain run, and no waiter may time out."""
import numpy as np
import pytest

from paper_2005_11931_b200 import inputs, tsw
from tests.helpers import check_slabs_against_oracle

pytestmark = pytest.mark.gpu


def _group(cfg, P, K, dtype="f64"):
    import torch
    stream = torch.cuda.Stream()
    parts = [tsw.Solver.from_config(cfg, dtype, rank=r, nranks=P, stream=stream.cuda_stream) for r in range(P)]
    for p in parts:
        if K > 1:
            p.set_option(tsw.TSW_OPT_TBLOCK, K)
        p.set_option(tsw.TSW_OPT_HALO, 1)
    for r, p in enumerate(parts):
        if r > 0:
            p.peer_attach(0, parts[r - 1])
        if r < P - 1:
            p.peer_attach(1, parts[r + 1])
    return parts, stream


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("K", [1, 4, 5, 8, 10])
@pytest.mark.parametrize("ny", [151, 29])
def test_peer_halo_slabs_bitwise(P, K, ny):
    cfg = inputs.config(3, nx=700, ny=ny, dx=0.01, dy=0.01, eps=[0.1, 0.3], amp=[1.0, 2.0], dt=2e-3)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
    n = 3 * K + 5
    ref = tsw.Solver.from_config(cfg, "f64")
    if K > 1:
        ref.set_option(tsw.TSW_OPT_TBLOCK, K)
    ref.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    ref.step(n)
    g, gp = ref.read(0), ref.read(1)
    parts, _ = _group(cfg, P, K)
    for p in parts:
        p.set_initial(np.ascontiguousarray(u0[p.r0:p.r0 + p.ny_local]), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    ctxs = [p.ctx for p in parts]
    tsw.tsw_group_step(ctxs, 1)          # ghost push + the start-up level
    tsw.tsw_group_step(ctxs, n - 1)      # ghost deepening, passes, remainder levels
    for p in parts:
        assert np.array_equal(p.read(0), g[:, p.r0:p.r0 + p.ny_local]), (P, K, ny, p.rank)
        assert np.array_equal(p.read(1), gp[:, p.r0:p.r0 + p.ny_local])
        assert tsw.tsw_peer_state(p.ctx)[3] == 0
    check_slabs_against_oracle(parts, cfg, "f64", n, u0)
    # energy is a ghost-reading collective (one epoch per rank) returning the slab's share
    E = sum(p.energy() for p in parts)
    np.testing.assert_allclose(E, ref.energy(), rtol=1e-12)
    for p in parts:
        p.close()
    ref.close()


@pytest.mark.parametrize("K,n", [(4, 41), (8, 45), (10, 41)])
def test_peer_halo_bench_shape_sampled(K, n):
    """The bench workload split into 2 slabs with K-deep peer halos (K = 8: a 4-level remainder
    pass): the slabs ≡ the single domain stepped one level at a time."""
    cfg = inputs.weak_unit(2, rows_per_rank=512)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
    ref = tsw.Solver.from_config(cfg, "f64")
    ref.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    ref.step(n)
    g = ref.read(0)
    parts, _ = _group(cfg, 2, K)
    for p in parts:
        p.set_initial(np.ascontiguousarray(u0[p.r0:p.r0 + p.ny_local]), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    tsw.tsw_group_step([p.ctx for p in parts], n)
    for p in parts:
        assert np.array_equal(p.read(0), g[:, p.r0:p.r0 + p.ny_local])
    check_slabs_against_oracle(parts, cfg, "f64", n, u0)
    for p in parts:
        p.close()
    ref.close()


@pytest.mark.parametrize("halo", [0, 1])
@pytest.mark.parametrize("K", [4, 8])
def test_slabs_several_calls_ending_in_passes(halo, K):
    """Every stepping call ends on a pass that also reduces the energy (TSW_OPT_ENERGY_FUSE); with
    peer halos that pass must still push its boundary rows (the fused-energy kernel has a peer-store
    variant), with loopback / NCCL-phase halos its rows must still be exchanged — so the NEXT call
    reads correct ghost rows.  Several such calls, energies in between, fields against the oracle."""
    import torch
    from tests.helpers import check_slabs_against_oracle
    cfg = inputs.config(3, nx=700, ny=151, dx=0.01, dy=0.01, eps=[0.1, 0.3], amp=[1.0, 2.0], dt=2e-3)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
    if halo:
        parts, _ = _group(cfg, 2, K)
    else:
        stream = torch.cuda.Stream()
        parts = [tsw.Solver.from_config(cfg, "f64", rank=r, nranks=2, stream=stream.cuda_stream) for r in range(2)]
        for p in parts:
            p.set_option(tsw.TSW_OPT_TBLOCK, K)
    for p in parts:
        p.set_initial(np.ascontiguousarray(u0[p.r0:p.r0 + p.ny_local]), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    ctxs = [p.ctx for p in parts]
    tsw.tsw_group_step(ctxs, 1)
    for _ in range(3):
        tsw.tsw_group_step(ctxs, K)
        for p in parts:
            p.energy()
    check_slabs_against_oracle(parts, cfg, "f64", 1 + 3 * K, u0)
    for p in parts:
        p.close()
