"""GPU parity of the ε-family diagnostics against the oracle definitions.

* tsw_family_l2 ≡ oracle.family_l2 (≤ 1e−12 relative: fp64 sums in another order);
* tsw_field_norms ≡ oracle.field_norms (≤ 1e−12 relative);
* tsw_coeff_norms ≡ the analytic W^{1,∞} pieces (≤ 1e−12 relative), and its ε-ladder gives the
  moderateness exponents N0 = 2 (δ) and 3 (δ²) of the Assumption;
* Theorem lem 1's estimate: the ratio of the solution norms to
  (1 + ‖h‖_∞^{1/2})(‖u0‖_{H¹} + ‖u1‖) stays bounded over time and uniformly in ε.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2005_11931_b200 import inputs, tsw
from tests.helpers import NP, host_cores

pytestmark = pytest.mark.gpu
oracle.set_threads(host_cores())


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("dim", [1, 2])
def test_family_l2_and_norms_small(dtype, dim):
    B = 7
    if dim == 1:
        cfg = inputs.config(1, nx=1999, eps=[0.03 + 0.02 * k for k in range(B)], amp=[1.0] * (B - 1) + [0.0], dt=7e-4)
    else:
        cfg = inputs.config(3, nx=301, ny=123, dx=0.02, dy=0.02, eps=[0.05 + 0.05 * k for k in range(B)],
                            amp=[1.0] * (B - 1) + [0.0], dt=2e-3)
    s = tsw.Solver.from_config(cfg, dtype)
    u0 = cfg.initial().astype(NP[dtype])
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(150)
    un, unm1 = s.read(0), s.read(1)
    w = cfg.dx if dim == 1 else cfg.dx * cfg.dy
    D = s.family_l2()
    Do = oracle.family_l2(un, w)
    assert np.all(D == D.T) and np.all(np.diag(D) == 0.0)
    np.testing.assert_allclose(D, Do, rtol=1e-12, atol=1e-300)
    N = s.field_norms()
    for b in range(B):
        No = oracle.field_norms(dim, un[b], unm1[b], cfg.dx, cfg.dy, cfg.dt)
        np.testing.assert_allclose(N[b], No, rtol=1e-12, atol=1e-300)
    s.close()


@pytest.mark.parametrize("dim,B,dtype", [(2, 65, "f64"), (1, 200, "f64"), (2, 37, "f32"), (1, 88, "f32")])
def test_family_l2_many_members(dim, B, dtype):
    """All pairs against the oracle for the member counts that select the pair-block groups and
    node phases of k_family_l2 (B = 65: 3 groups × 51 blocks, H = 5; B = 200: 5 groups, H = 1),
    on grids whose rows end in a ragged tile."""
    eps = [0.03 + 0.2 * k / B for k in range(B)]
    amp = [1.0 + 0.01 * k for k in range(B - 1)] + [0.0]
    if dim == 1:
        cfg = inputs.config(1, nx=3001, eps=eps, amp=amp, dt=5e-4)
    else:
        cfg = inputs.config(3, nx=203, ny=97, dx=0.02, dy=0.02, eps=eps, amp=amp, dt=2e-3)
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_initial(cfg.initial().astype(NP[dtype]), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(60)
    un = s.read(0)
    w = cfg.dx if dim == 1 else cfg.dx * cfg.dy
    D = s.family_l2()
    Do = oracle.family_l2(un, w)
    assert np.all(D == D.T) and np.all(np.diag(D) == 0.0)
    np.testing.assert_allclose(D, Do, rtol=1e-12, atol=1e-300)
    s.close()


def test_family_l2_config5_full_size():
    cfg = inputs.config(5)
    s = tsw.Solver.from_config(cfg, "f64")
    s.set_initial(cfg.initial(), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(400)
    D = s.family_l2()
    g = s.read(0)
    w = cfg.dx * cfg.dy
    rng = np.random.default_rng(0)
    pairs = [(0, 1), (0, 64), (31, 32), (62, 63)] + [tuple(sorted(rng.choice(65, 2, replace=False))) for _ in range(6)]
    for i, j in pairs:
        ref = math.sqrt(w * np.sum((g[i] - g[j]) ** 2))
        assert abs(D[i, j] - ref) <= 1e-12 * ref
    # the ε-family is Cauchy towards small ε at this time: neighbours in the ladder are closer at
    # the small-ε end than at the large-ε end
    assert D[0, 1] < D[62, 63]
    s.close()


def test_coeff_norms_and_moderateness_exponents():
    ladder = [0.2, 0.1, 0.05, 0.025]
    nx, dx = 20001, 0.0005                                       # 50 faces per ε at the smallest ε
    for order, N0 in ((1, 2.0), (2, 3.0)):
        s = tsw.Solver(1, nx, 1, dx, dx, len(ladder), "f64")
        s.set_coeff_profile([100.0], [], ladder, [0.0], [1.0], [order])
        cn = s.coeff_norms()
        P = oracle.Profile([100.0], [], [0.0], [1.0], [order])
        xf = ((2 * np.arange(nx - 1) + 2 - nx) * dx) / 2
        for b, e in enumerate(ladder):
            ref_h = np.max(np.abs(P.eval(xf[np.abs(xf) < 1.1 * e], e)))
            ref_d = np.max(np.abs(oracle.profile_derivative(P, xf, e)))
            assert abs(cn[b, 0] - ref_h) <= 1e-12 * ref_h
            assert abs(cn[b, 1] - ref_d) <= 1e-12 * ref_d
        assert abs(oracle.moderateness_exponent(ladder, cn[:, 1]) - N0) < 0.02
        s.close()
    # δ-line and δ-point kinds against the analytic gradient
    cfg = inputs.config(2, nx=400, ny=300, dx=0.005, dy=0.005, eps=[0.1, 0.2], amp=[1.0, 2.0])
    s = tsw.Solver.from_config(cfg, "f64")
    cn = s.coeff_norms()
    xf = ((2 * np.arange(cfg.nx - 1) + 2 - cfg.nx) * cfg.dx) / 2
    yn = inputs.node_coords(cfg.ny, cfg.dy)
    for b in range(2):
        e, A = cfg.eps[b], cfg.amp[b]
        px, py = oracle.phi_eps(xf, e), oracle.phi_eps(yn, e)
        gx = np.outer(py, oracle.dphi_eps(xf, e))
        gy = np.outer(oracle.dphi_eps(yn, e), px)
        ref = A * np.max(np.sqrt(gx ** 2 + gy ** 2))
        assert abs(cn[b, 1] - ref) <= 1e-12 * ref
        h1o, h2o = oracle.build_faces(2, cfg.kind, 1, 1.0, A, 0.0, 0.0, e, cfg.nx, cfg.ny, cfg.dx, cfg.dy)
        assert abs(cn[b, 0] - h1o.max()) <= 1e-12 * h1o.max()
        assert abs(cn[b, 2] - h2o.max()) <= 1e-12 * h2o.max()
    s.close()


def test_energy_estimate_ratio_bounded_uniformly_in_eps():
    """Theorem lem 1 along runs of Cases 1–3 (Gaussian data, T = 5) for ε ∈ {0.05 … 0.8}."""
    eps = [0.05, 0.1, 0.2, 0.4, 0.8]
    worst = []
    for case in ("1", "2", "3"):
        sc = inputs.paper_case(case, data="gauss1d")
        s = tsw.Solver(1, sc.nx, 1, sc.dx, sc.dx, len(eps), "f64")
        s.set_coeff_profile(sc.seg_value, sc.seg_break, eps, sc.sing_loc, sc.sing_amp, sc.sing_order)
        hinf = s.coeff_norms()[:, 0]
        dtm = s.info()[2]
        n = int(math.ceil(5.0 / (0.9 * dtm)))
        dt = 5.0 / n
        u0 = sc.initial()
        s.set_initial(u0, None, dt, flags=tsw.TSW_INIT_SHARED)
        s.step(1)
        N0 = s.field_norms()
        H1 = N0[:, 0] + N0[:, 2]                    # ‖u0‖_{H¹} ≈ ‖u¹‖ + ‖∂x u¹‖ (first level)
        den = (1.0 + np.sqrt(hinf)) * H1
        ratios = []
        for _ in range(10):
            s.step(n // 10)
            N = s.field_norms()
            ratios.append((N[:, 0] + N[:, 1] + N[:, 2]) / den)
        R = np.array(ratios)
        assert np.all(np.isfinite(R)) and R.max() < 10.0          # SPEC S:250's bound
        worst.append(R.max(axis=0))
        s.close()
    W = np.array(worst)
    assert W.max() / W.min() < 3.0                                  # uniform in ε and case
