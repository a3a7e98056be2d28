"""GPU parity for the paper's own scenarios through tsw_set_coeff_profile.

Faces: GPU tanh-sinh Φ vs the oracle's adaptive-Simpson Φ (both ≈ 1e−15 absolute) ⇒ faces agree
to ≤ 1e−13·max h.  Stepping: bitwise with the GPU faces given to the oracle; end to end ≤ 1e−12
relative max-norm (fp64).  Paper statements checked on the GPU fields: P:1101 (reflected-wave sign
structure) and the ε-stability of Figs. 3–5 as SPEC S:548's Cauchy trend.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2005_11931_b200 import inputs, tsw
from tests.helpers import abi_faces, host_cores, rel_maxnorm

pytestmark = pytest.mark.gpu
oracle.set_threads(host_cores())


def _solver(sc, batch=None):
    s = tsw.Solver(sc.dim, sc.nx, sc.ny, sc.dx, sc.dx, batch or sc.batch, "f64")
    return s


def _set_profile(s, sc, eps=None, scale=None):
    s.set_coeff_profile(sc.seg_value, sc.seg_break, eps or sc.eps, sc.sing_loc, sc.sing_amp, sc.sing_order,
                        sc.isotropic, scale)


def _oracle_profile(sc):
    return oracle.Profile(sc.seg_value, sc.seg_break, sc.sing_loc, sc.sing_amp, sc.sing_order, sc.isotropic)


def _dt(s, T, frac=0.9):
    dtm = s.info()[2]
    n = int(math.ceil(T / (frac * dtm)))
    return T / n, n


@pytest.mark.parametrize("case", ["1", "2", "3"])
def test_profile_faces_1d(case):
    sc = inputs.paper_case(case, amp=100.0)
    s = _solver(sc)
    _set_profile(s, sc)
    h1g, _ = s.read_faces()
    h1o, _ = oracle.build_faces_profile(1, _oracle_profile(sc), sc.eps[0], sc.nx, 1, sc.dx)
    assert np.max(np.abs(h1g[0] - h1o)) <= 1e-13 * np.max(h1o)
    assert np.array_equal(h1g[0] == 100.0, h1o == 100.0)      # locality is exact on both sides
    s.close()


def test_profile_faces_2d_isotropic_and_vector():
    sc = inputs.paper_2d(dx=0.25)
    for iso in (True, False):
        sc2 = inputs.Scenario(**{**sc.__dict__, "sing_loc": [20.0], "sing_amp": [3.0], "sing_order": [1],
                                 "isotropic": iso})
        s = _solver(sc2)
        _set_profile(s, sc2)
        h1g, h2g = s.read_faces()
        h1o, h2o = oracle.build_faces_profile(2, _oracle_profile(sc2), sc2.eps[0], sc2.nx, sc2.ny, sc2.dx)
        H1, H2 = abi_faces(h1o, h2o)
        assert np.max(np.abs(h1g[0] - H1)) <= 1e-13 * np.max(H1)
        assert np.max(np.abs(h2g[0][1:-1] - H2[1:-1])) <= 1e-13 * np.max(H2)
        s.close()


@pytest.mark.parametrize("case", ["1", "2", "3"])
def test_paper_1d_singularity_runs(case):
    """§3.2.3 set-up (Lorentzian e = 0.1, ε = 0.2, 100δ / 100δ²) to t = 2.5: GPU ≡ oracle (≤ 1e−12),
    bitwise with shared faces, and the paper's P:1101 sign structure on the GPU field."""
    sc = inputs.paper_case(case, data="lorentz", e=0.1, amp=100.0)
    s = _solver(sc)
    _set_profile(s, sc)
    dt, n = _dt(s, 2.5)
    u0 = sc.initial()
    s.set_initial(u0[None], None, dt)
    s.step(n)
    g = s.read(0)[0]
    h1g, _ = s.read_faces()
    un, _ = oracle.run(1, oracle.prescale(h1g[0], dt, sc.dx, np.float64), None, u0, None, dt, n)
    assert np.array_equal(g, un)                                # stepping bitwise, shared faces
    h1o, _ = oracle.build_faces_profile(1, _oracle_profile(sc), sc.eps[0], sc.nx, 1, sc.dx)
    uo, _ = oracle.run(1, oracle.prescale(h1o, dt, sc.dx, np.float64), None, u0, None, dt, n)
    assert rel_maxnorm(g, uo) <= 1e-12                          # end to end
    x = inputs.node_coords(sc.nx, sc.dx)
    main = np.max(np.abs(g[(x > -20.0) & (x < -10.0)]))
    r = g[(x > -5.0) & (x < 19.5)]
    thr = 0.01 * main
    has_pos, has_neg = bool(np.any(r > thr)), bool(np.any(r < -thr))
    assert np.max(np.abs(r)) < main
    if case == "1":
        assert has_pos and not has_neg
    else:
        assert has_pos and has_neg
    s.close()


def test_paper_2d_isotropic_h0():
    """§3.3: H(x, y) = h_0(x), ε = 0.8, Gaussian u0, on a 0.1-spaced grid to t = 2.5."""
    sc = inputs.paper_2d(dx=0.1)
    s = _solver(sc)
    _set_profile(s, sc)
    dt, n = _dt(s, 2.5)
    u0 = sc.initial()
    s.set_initial(u0[None], None, dt)
    s.step(n)
    g = s.read(0)[0]
    assert np.array_equal(g, g[::-1, :])                        # y-mirror symmetry (data symmetric in y)
    h1g, h2g = s.read_faces()
    c1 = oracle.prescale(h1g[0], dt, sc.dx, np.float64)
    c2 = oracle.prescale(np.ascontiguousarray(h2g[0][1:-1]), dt, sc.dx, np.float64)
    un, _ = oracle.run(2, c1, c2, u0, None, dt, n)
    assert np.array_equal(g, un)                                # bitwise, shared faces (LINE c2 vector)
    h1o, h2o = oracle.build_faces_profile(2, _oracle_profile(sc), sc.eps[0], sc.nx, sc.ny, sc.dx)
    uo, _ = oracle.run(2, oracle.prescale(h1o, dt, sc.dx, np.float64), oracle.prescale(h2o, dt, sc.dx, np.float64),
                       u0, None, dt, n)
    assert rel_maxnorm(g, uo) <= 1e-12
    s.close()


def test_eps_stability_cauchy_trend():
    """Figs. 3–5 ("stable as ε → 0"): at t = 5 the ε-family of Cases 1–3 is Cauchy —
    ‖u_{0.05} − u_{0.02}‖ < ‖u_{0.2} − u_{0.1}‖ < ‖u_{0.8} − u_{0.5}‖, one batched run per case."""
    eps = [0.02, 0.05, 0.1, 0.2, 0.5, 0.8]
    for case in ("1", "2", "3"):
        sc = inputs.paper_case(case, data="gauss1d")
        s = _solver(sc, batch=len(eps))
        _set_profile(s, sc, eps=eps)
        dt, n = _dt(s, 5.0)
        s.set_initial(sc.initial(), None, dt, flags=tsw.TSW_INIT_SHARED)
        s.step(n)
        E = s.energy()
        g = s.read(0)
        d = lambda a, b: math.sqrt(np.sum((g[a] - g[b]) ** 2) * sc.dx)
        assert d(1, 0) < d(3, 2) < d(5, 4), (case, d(1, 0), d(3, 2), d(5, 4))
        assert np.all(np.isfinite(E)) and np.all(E > 0)
        s.close()
