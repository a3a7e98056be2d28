"""Temporally blocked stencil: K levels per HBM pass must give the same bits
as K = 1 and as the oracle (same canonical per-node expression), for every K, both precisions,
ragged strips / row chunks, step counts not divisible by K, and the diagnostics afterwards."""
import numpy as np
import pytest

import oracle
from paper_2005_11931_b200 import inputs, tsw
from tests.helpers import NP, host_cores

pytestmark = pytest.mark.gpu
oracle.set_threads(host_cores())


def _run(cfg, dtype, K, nsteps, u0, rows_per_item=0, profile=None):
    s = tsw.Solver.from_config(cfg, dtype)
    if profile is not None:
        s.set_coeff_profile(*profile)
    s.set_option(tsw.TSW_OPT_TBLOCK, K)
    if rows_per_item:
        s.set_option(tsw.TSW_OPT_ROWS_PER_ITEM, rows_per_item)
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(nsteps)
    return s


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("K", [2, 3, 4, 5, 6, 8])
def test_tblock_bitwise_vs_oracle(dtype, K):
    cfg = inputs.config(3, nx=1300, ny=211, dx=0.01, dy=0.01, eps=[0.05, 0.3], amp=[1.0, 0.0], dt=2e-3)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(NP[dtype])
    n = 3 * K + 1 + 37                                 # a remainder handled by single levels
    s = _run(cfg, dtype, K, n, u0, rows_per_item=50)  # several chunks with a ragged last one
    g, gp = s.read(0), s.read(1)
    h1g, h2g = s.read_faces()
    for b in range(2):
        c1 = oracle.prescale(h1g[b], cfg.dt, cfg.dx, NP[dtype])
        c2 = oracle.prescale(np.ascontiguousarray(h2g[b][1:-1]), cfg.dt, cfg.dy, NP[dtype])
        un, unm1 = oracle.run(2, c1, c2, u0, None, cfg.dt, n)
        assert np.array_equal(g[b], un), f"K={K} member {b}: {np.max(np.abs(g[b] - un))}"
        assert np.array_equal(gp[b], unm1)
    E = s.energy()
    s1 = _run(cfg, dtype, 1, n, u0)
    assert np.array_equal(s1.read(0), g)
    np.testing.assert_allclose(E, s1.energy(), rtol=1e-13)
    s.close()
    s1.close()


@pytest.mark.parametrize("K", [4, 8])
def test_tblock_profile_isotropic_and_auto_chunks(K):
    sc = inputs.paper_2d(dx=0.1)
    cfg = inputs.config(3, nx=sc.nx, ny=sc.ny, dx=sc.dx, dy=sc.dx, eps=[0.8], amp=[1.0], dt=4e-3)
    prof = (sc.seg_value, sc.seg_break, [0.8], [20.0], [3.0], [1], True)
    u0 = sc.initial()
    s = _run(cfg, "f64", K, 200, u0, profile=prof)
    ref = _run(cfg, "f64", 1, 200, u0, profile=prof)
    assert np.array_equal(s.read(0), ref.read(0))
    assert np.array_equal(s.read(1), ref.read(1))
    D = s.family_l2()
    assert D.shape == (1, 1)
    s.close()
    ref.close()


def test_tblock_bench_shape_sampled():
    """The bench workload (32768 × 4096 δ-line slab) with K = 4: sampled nodes ≡ the K = 1 run."""
    cfg = inputs.weak_unit(1)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
    a = _run(cfg, "f64", 4, 41, u0)
    b = _run(cfg, "f64", 1, 41, u0)
    ga, gb = a.read(0)[0], b.read(0)[0]
    assert np.array_equal(ga, gb)
    np.testing.assert_allclose(a.energy(), b.energy(), rtol=1e-13)
    a.close()
    b.close()
