"""GPU parity of the paper's implicit method (R26–R28) through TSW_OPT_SCHEME=1.

1D: Thomas in the oracle's operation order ⇒ bitwise.  2D: both line solvers — the scan solvers
(R28: shared-LU affine scans along x, Toeplitz closed form along y; default) and cyclic reduction
(the paper's) — against the oracle's Thomas solves.  They solve the same line systems in other
orders; B = I − ½L per line is diagonally dominant (κ ≤ 1 + 2·max c), so one level agrees to
≲ κ·ε and n levels to ≲ n·κ·ε relative (R28): 1e−12 after one level, 1e−10 after 100 (fp64);
fp32 5e−5 after 100 levels.
"""
import numpy as np
import pytest

import oracle
from paper_2005_11931_b200 import inputs, tsw
from tests.helpers import NP, host_cores, rel_maxnorm

pytestmark = pytest.mark.gpu
oracle.set_threads(host_cores())
SOLVERS = {"scan": 3, "cr": 1, "stream": 2, "auto": 0}


def _implicit_solver(cfg, dtype="f64", solver="scan"):
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_option(tsw.TSW_OPT_SCHEME, 1)
    s.set_option(tsw.TSW_OPT_IMPLICIT_SOLVER, SOLVERS[solver])
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


def _oracle_2d(s, cfg, u0, v1, n, dtype):
    h1g, h2g = s.read_faces()
    out = []
    for b in range(h1g.shape[0]):
        c1 = oracle.prescale(h1g[b], cfg.dt, cfg.dx, NP[dtype])
        c2 = oracle.prescale(np.ascontiguousarray(h2g[b][1:-1]), cfg.dt, cfg.dy, NP[dtype])
        out.append(oracle.implicit_run(2, c1, c2, u0, v1, cfg.dt, n)[0])
    return out


# shapes: every x-solver width class (≤512, ≤1024, ≤2048, ≤4096, >4096 unknowns), ragged y segments,
# the smallest grids (one unknown per line)
SHAPES = [(130, 97), (300, 257), (64, 700), (40, 1500), (33, 3000), (9, 5000), (1029, 40), (3, 3), (4, 70), (70, 4)]


@pytest.mark.parametrize("solver", ["scan", "cr", "stream"])
@pytest.mark.parametrize("shape", SHAPES)
def test_implicit_2d_vs_oracle(shape, solver):
    ny, nx = shape
    cfg = inputs.config(3, nx=nx, ny=ny, dx=0.02, dy=0.02, eps=[0.1, 0.3], amp=[1.0, 2.0], dt=0.02)
    if solver == "cr" and max(nx, ny) - 2 > 4095:
        with pytest.raises(tsw.TswError):                     # CR keeps 4 line arrays of 2^q − 1 in smem
            _implicit_solver(cfg, solver=solver)
        return
    s = _implicit_solver(cfg, solver=solver)
    u0 = inputs.uniform_dense((ny, nx), seed=4)
    v1 = 0.5 * inputs.uniform_dense((ny, nx), seed=5)
    s.set_initial(u0, v1, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(1)
    g1 = s.read(0)
    n = 100 if nx * ny < 400000 else 20
    s.step(n - 1)
    g = s.read(0)
    o1 = _oracle_2d(s, cfg, u0, v1, 1, "f64")
    on = _oracle_2d(s, cfg, u0, v1, n, "f64")
    for b in range(2):
        assert rel_maxnorm(g1[b], o1[b]) < 1e-12
        assert rel_maxnorm(g[b], on[b]) < 1e-10
        assert np.all(g[b][0] == 0) and np.all(g[b][-1] == 0) and np.all(g[b][:, 0] == 0) and np.all(g[b][:, -1] == 0)
    s.close()


@pytest.mark.parametrize("xrows", [1, 2])
@pytest.mark.parametrize("shape", [(257, 300), (40, 1500), (9, 5000)])
def test_implicit_x_rows_per_iteration(shape, xrows):
    """The x-line solve with one and two rows per iteration (odd and even row counts per CTA)."""
    ny, nx = shape
    cfg = inputs.config(3, nx=nx, ny=ny, dx=0.02, dy=0.02, eps=[0.1], amp=[1.0], dt=0.02)
    s = _implicit_solver(cfg)
    s.set_option(tsw.TSW_OPT_IMPLICIT_XROWS, xrows)
    u0 = inputs.uniform_dense((ny, nx), seed=9)
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(10)
    on = _oracle_2d(s, cfg, u0, None, 10, "f64")[0]
    assert rel_maxnorm(s.read(0)[0], on) < 1e-11
    s.close()


@pytest.mark.parametrize("solver", ["scan", "cr", "stream"])
def test_implicit_2d_f32(solver):
    cfg = inputs.config(3, nx=515, ny=260, dx=0.02, dy=0.02, eps=[0.1], amp=[1.0], dt=0.02)
    s = _implicit_solver(cfg, "f32", solver)
    u0 = inputs.uniform_dense((cfg.ny, cfg.nx), seed=6).astype(np.float32)
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(100)
    g = s.read(0)[0]
    on = _oracle_2d(s, cfg, u0, None, 100, "f32")[0]
    assert rel_maxnorm(g, on) < 5e-5
    s.close()


def test_implicit_solvers_agree_and_constant_coeffs_symmetric():
    """Scan vs CR at large Courant numbers (γ up to ~1e4, ρ → 1 where the closed form's boundary
    terms matter) and x↔y symmetry for a constant coefficient on a square grid."""
    cfg = inputs.config(3, nx=257, ny=257, dx=0.01, dy=0.01, eps=[0.3], amp=[0.0], dt=1.0)
    u0 = inputs.uniform_dense((257, 257), seed=8)
    u0 = 0.5 * (u0 + u0.T)
    res = []
    for solver in ("scan", "cr", "stream"):
        s = _implicit_solver(cfg, solver=solver)
        s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
        s.step(30)
        res.append(s.read(0)[0])
        s.close()
    assert rel_maxnorm(res[0], res[1]) < 1e-10
    assert rel_maxnorm(res[0], res[2]) < 1e-10
    assert rel_maxnorm(res[0], res[0].T) < 1e-11


def test_implicit_table1_setup_4096():
    """PAPER §4 Table 1 set-up: 4096² on [0,100]², Δt = 0.05, T = 5 (100 steps), H = h_0(x) —
    the GPU result against the oracle (100 steps in full), finite, bounded, y-symmetric."""
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
    un = _oracle_2d(s, cfg, u0, None, 100, "f64")[0]
    assert rel_maxnorm(g, un) < 1e-10
    assert rel_maxnorm(g, g[::-1, :]) < 1e-12                    # y-symmetric data
    s.close()
