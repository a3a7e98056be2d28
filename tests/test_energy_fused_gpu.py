"""S5 fused into S3 (TSW_OPT_ENERGY_FUSE): the last temporally blocked pass of a
stepping call reduces the discrete energy E^{n−½} (R17, the discrete CL-01 of PAPER.md P:209–213)
of the two levels it writes, in the node form of reading R30 (−Σ u^{n+1}·L(u^n) + Σ (u^{n+1} −
u^n)², the stencil's own L at the pass's last level; per-item fp64 partials summed in a fixed
order by k_tb_energy_final).  It must equal the oracle's (face-form) energy of the same fields
(fp64 accumulation in a different order: ≤ 1e−12 relative) and leave the fields bitwise
unchanged."""
import numpy as np
import pytest

import oracle
from paper_2005_11931_b200 import inputs, tsw
from tests.helpers import NP, host_cores

pytestmark = pytest.mark.gpu
oracle.set_threads(host_cores())


def _oracle_energy(s, cfg, b, dtype):
    h1, h2 = s.read_faces()
    c1 = oracle.prescale(h1[b], cfg.dt, cfg.dx, NP[dtype])
    c2 = oracle.prescale(np.ascontiguousarray(h2[b][1:-1]), cfg.dt, cfg.dy, NP[dtype])
    return oracle.energy(2, c1, c2, s.read(0)[b], s.read(1)[b], cfg.dx, cfg.dy, cfg.dt)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("K,nsteps", [(8, 17), (8, 16), (4, 13), (5, 11), (7, 15), (2, 9), (3, 7), (6, 13), (10, 20), (9, 13)])
@pytest.mark.parametrize("shape", [(97, 700), (300, 2049), (7, 515)])
def test_fused_energy_matches_oracle(dtype, K, nsteps, shape):
    """Every pass depth (the call's last pass is a full K pass or the remainder), both CTA widths
    (2049 columns: 4-warp strips), several strips and chunks, ragged tails, a batch of members."""
    ny, nx = shape
    cfg = inputs.config(3, nx=nx, ny=ny, dx=0.01, dy=0.01, eps=[0.1, 0.3, 0.05], amp=[1.0, 2.0, 0.0], dt=2e-3)
    u0 = inputs.uniform_dense_rows(nx, ny, 0, ny).astype(NP[dtype])
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_option(tsw.TSW_OPT_TBLOCK, K)
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(1)
    s.step(nsteps)
    fused = s.energy()
    g = s.read(0)
    ref = tsw.Solver.from_config(cfg, dtype)
    ref.set_option(tsw.TSW_OPT_TBLOCK, K)
    ref.set_option(tsw.TSW_OPT_ENERGY_FUSE, 0)
    ref.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    ref.step(1)
    ref.step(nsteps)
    standalone = ref.energy()
    assert np.array_equal(g, ref.read(0))                       # fields untouched by the fusion
    for b in range(cfg.batch):
        Eo = _oracle_energy(s, cfg, b, dtype)
        assert abs(fused[b] - Eo) <= 1e-12 * Eo, (b, fused[b], Eo)
    np.testing.assert_allclose(fused, standalone, rtol=1e-12)
    s.close()
    ref.close()


def test_fused_energy_bench_shape_and_cadence():
    """The bench workload (32768 × 4096, dense, K = 8) with the bench's cadence: step(20) ends on a
    remainder pass of 4, step(16) on a full pass; each energy ≡ the standalone kernel's ≤ 1e−12 and
    conserved ≤ 1e−12 (R17)."""
    cfg = inputs.weak_unit(1)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
    s = tsw.Solver.from_config(cfg, "f64")
    s.set_option(tsw.TSW_OPT_TBLOCK, 8)
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    Es = []
    for k in (20, 16, 20):
        s.step(k)
        E = s.energy()
        s.set_option(tsw.TSW_OPT_ENERGY_FUSE, 0)
        Ea = s.energy()                                           # the standalone kernel, same level
        s.set_option(tsw.TSW_OPT_ENERGY_FUSE, 1)
        np.testing.assert_allclose(E, Ea, rtol=1e-12)
        Es.append(E[0])
    assert max(Es) - min(Es) <= 1e-12 * Es[0]
    s.close()


def test_fused_energy_invalidated_by_new_state():
    """A stored fused energy is for its level only: set_state / a one-level step recompute."""
    cfg = inputs.config(3, nx=300, ny=80, dx=0.01, dy=0.01, eps=[0.1], amp=[1.0], dt=2e-3)
    u0 = inputs.uniform_dense_rows(300, 80, 0, 80)
    s = tsw.Solver.from_config(cfg, "f64")
    s.set_option(tsw.TSW_OPT_TBLOCK, 4)
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(9)
    E9 = s.energy()
    s.step(1)                                                      # one-level step: no pass
    assert abs(s.energy()[0] - _oracle_energy(s, cfg, 0, "f64")) <= 1e-12 * E9[0]
    s.set_state(s.read(1), s.read(0), 10, cfg.dt)                  # swapped levels: another energy
    assert abs(s.energy()[0] - _oracle_energy(s, cfg, 0, "f64")) <= 1e-12 * E9[0]
    s.close()


@pytest.mark.parametrize("halo", ["loopback", "peer"])
@pytest.mark.parametrize("P,K,nsteps", [(2, 8, 17), (3, 4, 13), (2, 5, 12)])
def test_fused_energy_slabs(halo, P, K, nsteps):
    """Row slabs (one process, one GPU): with loopback copies (the phases of the NCCL pass) or peer
    halos, each slab's fused energy is its share of E (the node form reads no ghost row); the shares
    sum to the single-domain oracle energy ≤ 1e−12."""
    import torch
    cfg = inputs.config(3, nx=700, ny=151, dx=0.01, dy=0.01, eps=[0.1, 0.3], amp=[1.0, 2.0], dt=2e-3)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
    stream = torch.cuda.Stream()
    parts = [tsw.Solver.from_config(cfg, "f64", rank=r, nranks=P, stream=stream.cuda_stream) for r in range(P)]
    for p in parts:
        p.set_option(tsw.TSW_OPT_TBLOCK, K)
        if halo == "peer":
            p.set_option(tsw.TSW_OPT_HALO, 1)
    if halo == "peer":
        for r, p in enumerate(parts):
            if r > 0:
                p.peer_attach(0, parts[r - 1])
            if r < P - 1:
                p.peer_attach(1, parts[r + 1])
    for p in parts:
        p.set_initial(np.ascontiguousarray(u0[p.r0:p.r0 + p.ny_local]), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    ctxs = [p.ctx for p in parts]
    tsw.tsw_group_step(ctxs, 1)
    tsw.tsw_group_step(ctxs, nsteps)
    E = sum(p.energy() for p in parts)
    one = tsw.Solver.from_config(cfg, "f64")
    one.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    one.step(1 + nsteps)
    for b in range(cfg.batch):
        Eo = _oracle_energy(one, cfg, b, "f64")
        assert abs(E[b] - Eo) <= 1e-12 * Eo, (b, E[b], Eo)
    for p in parts:
        p.close()
    one.close()
