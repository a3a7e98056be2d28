"""GPU parity of the paper's implicit method (R26/R27) through TSW_OPT_SCHEME=1.

1D: Thomas in the oracle's operation order ⇒ bitwise.  2D: cyclic reduction (GPU) vs Thomas (oracle)
solve the same line systems in different orders; B = I − ½L per line is diagonally dominant
(condition number ≤ 1 + 2·max c), so each solve agrees to a few ulps × κ and the difference after
n levels stays ≤ n·κ·ε relative — the tests use 1e−10 at 100 levels.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2005_11931_b200 import inputs, tsw
from tests.helpers import NP, host_cores, rel_maxnorm

pytestmark = pytest.mark.gpu
oracle.set_threads(host_cores())


def _implicit_solver(cfg, dtype="f64"):
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_option(tsw.TSW_OPT_SCHEME, 1)
    return s


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_implicit_1d_bitwise(dtype):
    cfg = inputs.config(1, eps=[0.05, 0.2], amp=[1.0, 1.0], dt=0.02)        # 20× the explicit bound
    s = _implicit_solver(cfg, dtype)
    u0 = cfg.initial().astype(NP[dtype])
    v1 = (0.1 * inputs.uniform_dense((cfg.nx,), seed=2, dim=1)).astype(NP[dtype])
    s.set_initial(u0, v1, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(200)
    g = s.read(0)
    h1g, _ = s.read_faces()
    for b in range(2):
        c1 = oracle.prescale(h1g[b], cfg.dt, cfg.dx, NP[dtype])
        un, _ = oracle.implicit_run(1, c1, None, u0, v1, cfg.dt, 200)
        assert np.array_equal(g[b], un), np.max(np.abs(g[b] - un))
    s.close()


@pytest.mark.parametrize("shape", [(130, 97), (300, 257), (64, 700)])
def test_implicit_2d_vs_oracle(shape):
    ny, nx = shape
    cfg = inputs.config(3, nx=nx, ny=ny, dx=0.02, dy=0.02, eps=[0.1, 0.3], amp=[1.0, 2.0], dt=0.02)
    s = _implicit_solver(cfg)
    u0 = inputs.uniform_dense((ny, nx), seed=4)
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(1)
    g1 = s.read(0)
    s.step(99)
    g = s.read(0)
    h1g, h2g = s.read_faces()
    for b in range(2):
        c1 = oracle.prescale(h1g[b], cfg.dt, cfg.dx, np.float64)
        c2 = oracle.prescale(np.ascontiguousarray(h2g[b][1:-1]), cfg.dt, cfg.dy, np.float64)
        o1, _ = oracle.implicit_run(2, c1, c2, u0, None, cfg.dt, 1)
        assert rel_maxnorm(g1[b], o1) < 1e-13
        un, _ = oracle.implicit_run(2, c1, c2, u0, None, cfg.dt, 100)
        assert rel_maxnorm(g[b], un) < 1e-10
        assert np.all(g[b][0] == 0) and np.all(g[b][:, -1] == 0)
    s.close()


def test_implicit_table1_setup_4096():
    """PAPER §4 Table 1 set-up: 4096² on [0,100]², Δt = 0.05, T = 5 (100 steps), H = h_0(x) —
    the GPU result against the oracle (sampled 100 steps in full), finite and bounded."""
    sc = inputs.paper_2d(dx=100.0 / 4095)
    cfg = inputs.config(3, nx=sc.nx, ny=sc.ny, dx=sc.dx, dy=sc.dx, eps=[0.8], dt=0.05)
    s = tsw.Solver(2, sc.nx, sc.ny, sc.dx, sc.dx, 1, "f64")
    s.set_coeff_profile(sc.seg_value, sc.seg_break, [0.8], isotropic=True)
    s.set_option(tsw.TSW_OPT_SCHEME, 1)
    u0 = sc.initial()
    s.set_initial(u0[None], None, 0.05)
    s.step(100)
    g = s.read(0)[0]
    assert np.all(np.isfinite(g)) and np.max(np.abs(g)) < 60
    h1g, h2g = s.read_faces()
    c1 = oracle.prescale(h1g[0], 0.05, sc.dx, np.float64)
    c2 = oracle.prescale(np.ascontiguousarray(h2g[0][1:-1]), 0.05, sc.dx, np.float64)
    un, _ = oracle.implicit_run(2, c1, c2, u0, None, 0.05, 100)
    assert rel_maxnorm(g, un) < 1e-10
    assert np.array_equal(g, g[::-1, :]) or rel_maxnorm(g, g[::-1, :]) < 1e-12   # y-symmetric data
    s.close()
