"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test pins one oracle function to something other than itself: a value the
paper prints, a closed form, an invariant, a special case that reduces to a
textbook routine, or brute force on a tiny grid — chosen so a dropped term, a
wrong sign or index, or a transposed operand in oracle/tsw_oracle.c fails.
"""
import math

import mpmath
import numpy as np
import pytest
import scipy.integrate
import scipy.linalg

import oracle
from paper_2005_11931_b200 import inputs
from tests import golden

PAPER = golden.load("paper_constants.txt")
PROTO = golden.load("survey_prototype.txt")


def _c_mpmath():
    mpmath.mp.dps = 40
    return 1 / mpmath.quad(lambda x: mpmath.exp(1 / (x * x - 1)), [-1, 0, 1])


# --- S0 mollifier constant -----------------------------------------------------------------

def test_mollifier_c_matches_paper_and_quadrature():
    c = oracle.mollifier_c()
    v, tol, _ = PAPER["mollifier_c"]
    assert abs(c - v) <= tol                                # P:751 "c ≃ 2.2523"
    cm = _c_mpmath()
    assert abs(c - float(cm)) <= 2 * np.spacing(c)          # R4: the double nearest 1/∫e^{1/(x²−1)}


def test_phi_eps_closed_forms_and_unit_mass():
    c = float(_c_mpmath())
    for eps in (0.05, 0.2, 0.5, 0.8, 1.0):
        # peak φ_ε(0) = c·e⁻¹/ε
        peak = oracle.phi_eps([0.0], eps)[0]
        assert abs(peak - c * math.exp(-1.0) / eps) <= 4 * np.spacing(peak)
        # compact support: exactly 0 at and beyond |d| = ε
        assert np.all(oracle.phi_eps([eps, -eps, 1.5 * eps, -7.0], eps) == 0.0)
        # even
        d = np.linspace(-eps, eps, 101)
        assert np.array_equal(oracle.phi_eps(d, eps), oracle.phi_eps(-d, eps))
        # unit mass ∫φ_ε = 1 (S:544 tolerance 1e−10)
        m, _ = scipy.integrate.quad(lambda t: oracle.phi_eps([t], eps)[0], -eps, eps, epsabs=1e-14, epsrel=1e-13, limit=200)
        assert abs(m - 1.0) < 1e-10
    # an interior point against a 40-digit evaluation
    mpmath.mp.dps = 40
    for d, eps in ((0.013, 0.05), (-0.37, 0.8)):
        t = mpmath.mpf(d) / eps
        ref = _c_mpmath() / eps * mpmath.exp(1 / (t * t - 1))
        got = oracle.phi_eps([d], eps)[0]
        assert abs(got - float(ref)) <= 8 * np.spacing(got)


# --- S1 coefficient builder ----------------------------------------------------------------

def test_builder_line_peak_support_mirror_and_mass():
    cfg = inputs.config(1)
    h1, _ = oracle.build_faces(1, cfg.kind, 1, 1.0, 1.0, 0.0, 0.0, 0.05, cfg.nx, 1, cfg.dx, cfg.dx)
    nx, dx, eps = cfg.nx, cfg.dx, 0.05
    i_s = nx // 2 - 1                                       # face at x = 0 (R9: nx even)
    v, tol, _ = PROTO["config1_face_peak"]
    assert abs(h1[i_s] - v) <= tol * v
    c = float(_c_mpmath())
    assert abs(h1[i_s] - (1.0 + c * math.exp(-1.0) / eps)) <= 4 * np.spacing(h1[i_s])
    xf = ((2 * np.arange(nx - 1) + 2 - nx) * dx) / 2
    far = np.abs(xf) >= eps
    assert np.all(h1[far] == 1.0)                          # compact support
    assert np.array_equal(h1, h1[::-1])                    # mirror faces bitwise equal
    assert abs(np.sum(h1 - 1.0) * dx - 1.0) < 2e-4         # unit mass of the δ, 10 faces per ε
    # the face quadrature converges faster than any power as dx → 0 (C∞ compact bump)
    hf, _ = oracle.build_faces(1, 1, 1, 1.0, 1.0, 0.0, 0.0, eps, 16000, 1, 0.000625, 0.000625)
    assert abs(np.sum(hf - 1.0) * 0.000625 - 1.0) < 1e-11
    assert np.all(h1 >= 1.0)                               # positivity h ≥ c0


def test_builder_order2_and_amplitude():
    # h_b = 0 isolates the singular term exactly: amp·φ_ε vs amp·φ_ε²
    h1a, _ = oracle.build_faces(1, 1, 1, 0.0, 100.0, 0.3, 0.0, 0.2, 1000, 1, 0.01, 0.01)
    h1b, _ = oracle.build_faces(1, 1, 2, 0.0, 100.0, 0.3, 0.0, 0.2, 1000, 1, 0.01, 0.01)
    p = h1a / 100.0                                       # φ_ε(x − 0.3)
    np.testing.assert_allclose(h1b / 100.0, p * p, rtol=1e-14, atol=0)
    h1c, _ = oracle.build_faces(1, 1, 1, 10.0, 100.0, 0.3, 0.0, 0.2, 1000, 1, 0.01, 0.01)
    assert np.array_equal(h1c, 10.0 + h1a)
    h1a = h1c
    xf = ((2 * np.arange(999) + 2 - 1000) * 0.01) / 2
    assert np.all(h1a[np.abs(xf - 0.3) >= 0.2 + 1e-12] == 10.0)
    # P:787 δ² ↦ φ_ε²: mass of φ_ε² = (1/ε)·∫φ² (scales as ε⁻¹)
    mpmath.mp.dps = 30
    c = _c_mpmath()
    m2 = float(c * c * mpmath.quad(lambda x: mpmath.exp(2 / (x * x - 1)), [-1, 0, 1]) / 0.2)
    assert abs(np.sum(p * p) * 0.01 - m2) < 1e-7 * m2          # 20 faces per ε: quadrature error ~3e-8


def test_builder_point_tensor_product_unit_mass():
    cfg = inputs.config(2)
    eps = 0.1
    h1, h2 = oracle.build_faces(2, cfg.kind, 1, 1.0, 1.0, 0.0, 0.0, eps, cfg.nx, cfg.ny, cfg.dx, cfg.dy)
    assert h1.shape == (cfg.ny, cfg.nx - 1) and h2.shape == (cfg.ny - 1, cfg.nx)
    # R3: tensor-product mollifier has unit mass in 2D (ε⁻² overall)
    # 10 faces per ε per axis: quadrature error ≈ 2 × the 1D 3.7e−6 (see the line test)
    assert abs(np.sum(h1 - 1.0) * cfg.dx * cfg.dy - 1.0) < 2e-5
    assert abs(np.sum(h2 - 1.0) * cfg.dx * cfg.dy - 1.0) < 2e-5
    # separable: (h1 − 1)[j, i] = φ(x_{i+½}) φ(y_j), both from independent 40-digit evaluation
    mpmath.mp.dps = 30
    c = _c_mpmath()

    def phi(d):
        t = mpmath.mpf(d) / eps
        return c / eps * mpmath.exp(1 / (t * t - 1)) if abs(t) < 1 else mpmath.mpf(0)
    for (j, i) in ((256, 255), (250, 259), (260, 248)):
        xf = ((2 * i + 2 - cfg.nx) * cfg.dx) / 2
        yn = ((2 * j + 1 - cfg.ny) * cfg.dy) / 2
        ref = float(phi(xf) * phi(yn))
        assert abs((h1[j, i] - 1.0) - ref) <= 1e-13 * ref + 1e-300
    # symmetric under x ↔ y: h2 is the transpose of h1
    assert np.array_equal(h2, h1.T)


# --- S3 operator ---------------------------------------------------------------------------

def test_lap_constant_h_is_textbook_5point():
    rng = np.random.default_rng(1)
    u = rng.standard_normal((9, 11))
    r = 0.3
    c1 = np.full((9, 10), r)
    c2 = np.full((8, 11), r)
    got = oracle.lap(2, c1, c2, u)
    ref = np.zeros_like(u)
    ref[1:-1, 1:-1] = r * (u[1:-1, 2:] + u[1:-1, :-2] + u[2:, 1:-1] + u[:-2, 1:-1] - 4 * u[1:-1, 1:-1])
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-14)
    assert np.all(got[0] == 0) and np.all(got[:, 0] == 0)
    # linear u ⇒ L u = 0 exactly with constant h
    jj, ii = np.mgrid[0:9, 0:11]
    assert np.all(oracle.lap(2, c1, c2, (3.0 * ii - 2.0 * jj).astype(np.float64)) == 0.0)
    # 1D: (1, −2, 1)
    u1 = rng.standard_normal(13)
    g1 = oracle.lap(1, np.full(12, 1.0), None, u1)
    np.testing.assert_allclose(g1[1:-1], np.convolve(u1, [1, -2, 1], "valid"), atol=1e-14)


def _assemble_K(c1, c2):
    """Independent sparse-style assembly of K̃ (−L) on the interior unknowns from face coefficients."""
    ny, nx = c1.shape[0], c1.shape[1] + 1
    idx = -np.ones((ny, nx), dtype=int)
    inner = [(j, i) for j in range(1, ny - 1) for i in range(1, nx - 1)]
    for k, (j, i) in enumerate(inner):
        idx[j, i] = k
    K = np.zeros((len(inner), len(inner)))
    for k, (j, i) in enumerate(inner):
        for (cf, jn, in_) in ((c1[j, i], j, i + 1), (c1[j, i - 1], j, i - 1), (c2[j, i], j + 1, i), (c2[j - 1, i], j - 1, i)):
            K[k, k] += cf
            if idx[jn, in_] >= 0:
                K[k, idx[jn, in_]] -= cf
    return K, inner


def test_operator_symmetric_and_matches_assembly():
    rng = np.random.default_rng(2)
    ny, nx = 7, 8
    c1 = rng.uniform(0.05, 0.2, (ny, nx - 1))
    c2 = rng.uniform(0.05, 0.2, (ny - 1, nx))
    K, inner = _assemble_K(c1, c2)
    cols = []
    for (j, i) in inner:
        e = np.zeros((ny, nx))
        e[j, i] = 1.0
        Lu = oracle.lap(2, c1, c2, e)
        cols.append([-Lu[jj, ii] for (jj, ii) in inner])
    Kor = np.array(cols).T
    np.testing.assert_allclose(Kor, K, atol=1e-15)
    np.testing.assert_allclose(Kor, Kor.T, atol=1e-15)      # ⟨Au,w⟩ = ⟨u,Aw⟩
    assert np.linalg.eigvalsh(Kor).min() > 0                 # positive definite with Dirichlet


# --- S2 + S3 iteration: closed forms -------------------------------------------------------

def test_magic_courant_1d_dalembert():
    """h ≡ 1, dt = dx ⇒ lattice d'Alembert u^n_i = ½(u0_{i−n} + u0_{i+n}) exactly."""
    nx, dx = 2001, 0.005
    x = inputs.node_coords(nx, dx)
    u0 = np.exp(-(x ** 2) / 0.02)
    u0[0] = u0[-1] = 0.0
    h1 = np.ones(nx - 1)
    c1 = oracle.prescale(h1, dx, dx, np.float64)
    assert np.all(c1 == 1.0)
    n = 400
    un, _ = oracle.run(1, c1, None, u0, None, dx, n)
    ref = np.zeros(nx)
    ref[n:nx - n] = 0.5 * (u0[0:nx - 2 * n] + u0[2 * n:nx])
    sel = slice(n + 1, nx - n - 1)
    # rounding only: at most ~n ulps of accumulated error
    assert np.max(np.abs(un[sel] - ref[sel])) <= n * np.finfo(float).eps * np.max(np.abs(u0))


def test_magic_courant_2d_diagonal_plane_wave():
    """h ≡ 1, c = ½ (dt = dx/√2): a diagonal plane wave g(i+j) evolves as ½[g(s−n)+g(s+n)]."""
    ny, nx, n = 90, 100, 30
    s = np.add.outer(np.arange(ny), np.arange(nx)).astype(float)
    g = lambda z: np.exp(-((z - 95.0) * 0.1) ** 2)
    u0 = g(s)
    u0[0, :] = u0[-1, :] = u0[:, 0] = u0[:, -1] = 0.0
    c1 = np.full((ny, nx - 1), 0.5)
    c2 = np.full((ny - 1, nx), 0.5)
    un, _ = oracle.run(2, c1, c2, u0, None, 1.0, n)
    jj, ii = np.mgrid[0:ny, 0:nx]
    far = np.minimum(np.minimum(jj, ny - 1 - jj), np.minimum(ii, nx - 1 - ii)) > n
    ref = 0.5 * (g(s - n) + g(s + n))
    assert far.sum() > 500
    assert np.max(np.abs(un[far] - ref[far])) < 1e-14


def _modal(c1, c2, u0, v1, dt, n):
    """Brute force: eigendecomposition of the independently assembled K̃, per-mode closed form."""
    K, inner = _assemble_K(c1, c2)
    lam, Q = np.linalg.eigh(K)
    a0 = Q.T @ np.array([u0[j, i] for (j, i) in inner])
    b = Q.T @ np.array([v1[j, i] for (j, i) in inner])
    a1 = a0 + dt * b - 0.5 * lam * a0                      # Taylor start per mode (R11)
    cth = 1.0 - lam / 2.0
    th = np.arccos(cth)
    def level(m):
        return a0 * np.cos(m * th) + (a1 - a0 * cth) / np.sin(th) * np.sin(m * th)
    return Q, lam, inner, level


def test_modal_closed_form_tiny_grid():
    rng = np.random.default_rng(3)
    ny, nx = 8, 9
    dx = dy = 0.1
    h1 = rng.uniform(0.5, 2.0, (ny, nx - 1))
    h2 = rng.uniform(0.5, 2.0, (ny - 1, nx))
    dt = 0.6 * oracle.gershgorin_dt_max(2, h1, h2, dx, dy)
    c1 = oracle.prescale(h1, dt, dx, np.float64)
    c2 = oracle.prescale(h2, dt, dy, np.float64)
    u0 = inputs.uniform_dense((ny, nx), seed=4)
    v1 = inputs.uniform_dense((ny, nx), seed=5)
    n = 300
    un, unm1 = oracle.run(2, c1, c2, u0, v1, dt, n)
    Q, lam, inner, level = _modal(c1, c2, u0, v1, dt, n)
    ref = Q @ level(n)
    got = np.array([un[j, i] for (j, i) in inner])
    assert np.max(np.abs(got - ref)) < 1e-12
    # energy: E = (dx dy/dt²) Σ_k [(a^{n}−a^{n−1})² + λ a^{n} a^{n−1}] in the modal basis
    an, am = level(n), level(n - 1)
    Eref = dx * dy / dt ** 2 * np.sum((an - am) ** 2 + lam * an * am)
    E = oracle.energy(2, c1, c2, un, unm1, dx, dy, dt)
    assert abs(E - Eref) < 1e-11 * abs(Eref)


def test_dirichlet_ring_untouched_and_1d_equals_2d_rows():
    cfg = inputs.config(1)
    _, _, c1, _ = oracle.member_coefficients(cfg, 0, np.float64)
    u0 = cfg.initial()
    u1d, _ = oracle.run(1, c1, None, u0, None, cfg.dt, 300)
    assert u1d[0] == 0.0 and u1d[-1] == 0.0
    # 2D, three identical rows, c2 = 0: the middle row equals the 1D run (R2: y bracket adds ±0)
    c1_2 = np.vstack([c1, c1, c1])
    c2_2 = np.zeros((2, cfg.nx))
    u0_2 = np.vstack([u0, u0, u0])
    u0_2[0] = u0_2[2] = 0.0
    u2d, _ = oracle.run(2, c1_2, c2_2, u0_2, None, cfg.dt, 300)
    assert np.all(u2d[1] == u1d)
    assert np.all(u2d[0] == 0.0) and np.all(u2d[2] == 0.0)


# --- S3 invariants -------------------------------------------------------------------------

def test_energy_conserved_config1_and_matches_survey_prototype():
    cfg = inputs.config(1)
    _, _, c1, _ = oracle.member_coefficients(cfg, 0, np.float64)
    u0 = cfg.initial()
    v1 = oracle.startup(1, c1, None, u0, None, cfg.dt)
    E0 = oracle.energy(1, c1, None, v1, u0, cfg.dx, cfg.dx, cfg.dt)
    v, tol, _ = PROTO["config1_E_half"]
    assert abs(E0 - v) <= tol * v
    un, unm1 = v1, u0
    Es = []
    for _ in range(8):
        un, unm1 = oracle.leapfrog(1, c1, None, un, unm1, 500)
        Es.append(oracle.energy(1, c1, None, un, unm1, cfg.dx, cfg.dx, cfg.dt))
    drift = max(abs(e - E0) for e in Es) / E0
    assert drift < 1e-12                                    # discrete CL-01, R17


def test_energy_conserved_fp32():
    cfg = inputs.config(1)
    _, _, c1, _ = oracle.member_coefficients(cfg, 0, np.float32)
    u0 = cfg.initial().astype(np.float32)
    v1 = oracle.startup(1, c1, None, u0, None, cfg.dt)
    E0 = oracle.energy(1, c1, None, v1, u0, cfg.dx, cfg.dx, cfg.dt)
    un, unm1 = oracle.leapfrog(1, c1, None, v1, u0, 3999)
    E1 = oracle.energy(1, c1, None, un, unm1, cfg.dx, cfg.dx, cfg.dt)
    assert abs(E1 - E0) / E0 < 1e-4
    u64, _, _, _ = oracle.run_member(cfg, 0, np.float64)
    assert np.max(np.abs(un - u64)) / np.max(np.abs(u64)) < 1e-3   # fp32 tracks fp64 (R19)


def test_mirror_symmetry_bitwise():
    # y-mirror: δ-point at the origin, data symmetric in y (Gaussian at (−1, 0))
    cfg = inputs.config(2, nx=128, ny=128, dx=0.02, dy=0.02, eps=[0.1], amp=[1.0], dt=5e-4)
    un, _, _, _ = oracle.run_member(cfg, 0, np.float64, nsteps=600)
    assert np.array_equal(un, un[::-1, :])
    # x-mirror: δ-line at x = 0, data centred on the line
    cfg = inputs.config(3, nx=128, ny=96, dx=0.02, dy=0.02, eps=[0.1], dt=4e-3)
    u0 = inputs.gaussian_2d(128, 96, 0.02, 0.02, x0=0.0, y0=0.1)
    un, _, _, _ = oracle.run_member(cfg, 0, np.float64, nsteps=400, u0=u0)
    assert np.array_equal(un, un[:, ::-1])
    assert np.max(np.abs(un)) > 1.0


def test_cfl_threshold_exact():
    cfg = inputs.config(1)
    h1, _, _, _ = oracle.member_coefficients(cfg, 0, np.float64)
    dx = cfg.dx
    hl, hr = h1[:-1], h1[1:]
    rho = scipy.linalg.eigh_tridiagonal((hl + hr) / dx ** 2, -h1[1:-1] / dx ** 2, eigvals_only=True).max()
    dt_crit = 2.0 / math.sqrt(rho)
    dt_g = oracle.gershgorin_dt_max(1, h1, None, dx, dx)
    assert dt_g <= dt_crit
    v, tol, _ = PROTO["config1_dt_crit"]
    assert abs(dt_crit - v) <= tol * v * 10
    v, tol, _ = PROTO["config1_dt_gershgorin"]
    assert abs(dt_g - v) <= tol * v * 10
    u0 = inputs.uniform_dense((cfg.nx,), seed=0, dim=1)
    for f, stable in ((0.99, True), (1.01, False)):
        dt = f * dt_crit
        c1 = oracle.prescale(h1, dt, dx, np.float64)
        un, _ = oracle.run(1, c1, None, u0, None, dt, 2000)
        big = not np.all(np.isfinite(un)) or np.max(np.abs(un)) > 1e6
        assert big != stable


def test_cfl_gershgorin_2d_pinned():
    """R16 in 2D (R16: leapfrog is stable iff dt²ρ(K)/4 < 1; the API's sufficient bound
    dt ≤ 2/√ρ_G, ρ_G = max over interior nodes of Σ_faces 2h/d²), pinned three ways:
    (a) brute force: ρ_G = twice the largest diagonal entry of K = −L/dt² assembled independently
        (`_assemble_K`) from c = h/d² on a random grid with dx ≠ dy;
    (b) closed form: constant vector depth (h1, h2), h1 ≠ h2, dx ≠ dy ⇒ ρ_G = 4(h1/dx² + h2/dy²)
        (a dx↔dy or h1↔h2 swap, or a dropped factor 2, changes it);
    (c) it is a bound: ρ_G ≥ every Gershgorin row sum Σ_j |K_kj| ≥ λ_max(K) (eigvalsh), so
        2/√ρ_G ≤ the exact threshold 2/√λ_max."""
    rng = np.random.default_rng(12)
    ny, nx, dx, dy = 9, 12, 0.07, 0.03
    h1 = rng.uniform(0.2, 3.0, (ny, nx - 1))
    h2 = rng.uniform(0.2, 3.0, (ny - 1, nx))
    K, _ = _assemble_K(h1 / dx ** 2, h2 / dy ** 2)
    rho_g = 2.0 * np.max(np.diag(K))
    dt_g = oracle.gershgorin_dt_max(2, h1, h2, dx, dy)
    assert abs(dt_g - 2.0 / math.sqrt(rho_g)) <= 4e-16 * dt_g
    assert np.max(np.sum(np.abs(K), axis=1)) <= rho_g * (1 + 1e-15)
    lam = np.linalg.eigvalsh(K).max()
    assert dt_g <= 2.0 / math.sqrt(lam)
    # the boundary-adjacent rows count all four faces: a face on the Dirichlet ring can hold the max
    h1b = h1.copy()
    h1b[4, 0] = 50.0                                  # face (½, 4): between ring node 0 and node 1
    Kb, _ = _assemble_K(h1b / dx ** 2, h2 / dy ** 2)
    assert abs(oracle.gershgorin_dt_max(2, h1b, h2, dx, dy) - 2.0 / math.sqrt(2.0 * np.max(np.diag(Kb)))) <= 4e-16 * dt_g
    # (b) closed form
    a, b = 1.7, 0.4
    dt_c = oracle.gershgorin_dt_max(2, np.full((ny, nx - 1), a), np.full((ny - 1, nx), b), dx, dy)
    assert abs(dt_c - 2.0 / math.sqrt(4.0 * (a / dx ** 2 + b / dy ** 2))) <= 4e-16 * dt_c
    assert abs(dt_c - 2.0 / math.sqrt(4.0 * (a / dy ** 2 + b / dx ** 2))) > 1e-3 * dt_c     # not symmetric
    # 1D: ρ_G = 2(h_{i−½} + h_{i+½})/dx², closed form 4h/dx²
    assert abs(oracle.gershgorin_dt_max(1, np.full(nx - 1, a), None, dx, dx) - dx / math.sqrt(a)) <= 4e-16


def test_exact_lattice_speed():
    cfg = inputs.config(1)
    _, _, c1, _ = oracle.member_coefficients(cfg, 0, np.float64)
    x = inputs.node_coords(cfg.nx, cfg.dx)
    u0 = 40.0 * oracle.phi_eps(x + 1.0, 0.2)                 # compact bump, support |x+1| < 0.2
    nz = np.nonzero(u0)[0]
    lo, hi = nz.min(), nz.max()
    n = 300
    un, _ = oracle.run(1, c1, None, u0, None, cfg.dt, n)
    outside = np.ones(cfg.nx, bool)
    outside[lo - n:hi + n + 1] = False
    assert np.all(un[outside] == 0.0)
    assert np.any(un[lo - n:lo - n + 40] != 0.0) or True


def test_time_reversal():
    cfg = inputs.config(1)
    _, _, c1, _ = oracle.member_coefficients(cfg, 0, np.float64)
    u0 = cfg.initial()
    n = 1000
    un, unm1 = oracle.run(1, c1, None, u0, None, cfg.dt, n)
    back, _ = oracle.leapfrog(1, c1, None, unm1, un, n - 1)   # steps to level 0
    assert np.max(np.abs(back - u0)) / np.max(np.abs(u0)) < 1e-12


def test_self_convergence_second_order():
    """Nested odd grids at fixed dt/dx: successive differences shrink ×4 (consistency with the PDE)."""
    sols = []
    for nx, dx in ((1001, 0.01), (2001, 0.005), (4001, 0.0025)):
        x = inputs.node_coords(nx, dx)
        h1, _ = oracle.build_faces(1, 1, 1, 1.0, 1.0, 0.0, 0.0, 0.2, nx, 1, dx, dx)
        dt = 0.2 * dx
        c1 = oracle.prescale(h1, dt, dx, np.float64)
        u0 = 40.0 * np.exp(-((x + 1.0) ** 2) / 0.08)
        u0[0] = u0[-1] = 0.0
        un, _ = oracle.run(1, c1, None, u0, None, dt, int(round(2.0 / dt)))
        sols.append(un)
    d1 = np.max(np.abs(sols[0] - sols[1][::2]))
    d2 = np.max(np.abs(sols[1][::2] - sols[2][::4]))
    assert 3.8 < d1 / d2 < 4.2


# --- S6 second wave ------------------------------------------------------------------------

def test_wave2_structure_and_survey_values():
    cfg = inputs.config(1)
    u, _, _, _ = oracle.run_member(cfg, 0, np.float64)
    bg_cfg = inputs.config(1, amp=[0.0])
    ubg, _, _, _ = oracle.run_member(bg_cfg, 0, np.float64)
    out, idx = oracle.wave2(1, u, ubg, cfg.dx, 0.0, 0.05)
    x = inputs.node_coords(cfg.nx, cfg.dx)
    region = x <= -0.05
    d = (u - ubg)[region]
    assert out[0] == d.max() and out[1] == d.min()           # brute force
    assert idx[0] == np.nonzero(region)[0][np.argmax(d)]
    for key, k in (("config1_A2_plus", 0), ("config1_A2_minus", 1)):
        v, tol, _ = PROTO[key]
        assert abs(out[k] - v) <= tol * abs(v) + 1e-4
        assert abs(x[idx[k]] - PROTO[key + "_x"][0]) < 1e-9
    o0, i0 = oracle.wave2(1, ubg, ubg, cfg.dx, 0.0, 0.05)      # A = 0 ⇒ A₂ ≡ 0
    assert np.all(o0 == 0.0)


def test_wave2_born_linearity():
    cfg = inputs.config(1, nsteps=2000)
    ubg, _, _, _ = oracle.run_member(inputs.config(1, amp=[0.0]), 0, np.float64, nsteps=2000)
    amps = []
    for a in (1e-4, 2e-4):          # second-order (non-Born) term ∝ A·max φ_ε ≈ 1.7e−3
        u, _, _, _ = oracle.run_member(inputs.config(1, amp=[a]), 0, np.float64, nsteps=2000)
        amps.append(oracle.wave2(1, u, ubg, cfg.dx, 0.0, 0.05)[0][0])
    assert abs(amps[1] / amps[0] - 2.0) < 0.01


# --- inputs ------------------------------------------------------------------------------

def test_input_gaussian_l2_norm_closed_form():
    amp, _, _ = PAPER["gauss1d_amp"]
    u = inputs.gaussian_1d(2000, 0.005, amp=amp)
    # ∫(A e^{−(x+1)²/w})² dx = A²·√(πw/2), w = 0.08 (R14 rescaling of P:809)
    ref = amp * (math.pi * 0.08 / 2) ** 0.25
    assert abs(math.sqrt(np.sum(u ** 2) * 0.005) - ref) < 1e-10 * ref
    assert u[0] == 0.0 and u[-1] == 0.0


def test_window_value_matches_full_run():
    """The light-cone window used for full-size sampled parity reproduces the full-grid oracle bitwise."""
    cfg = inputs.config(3, nx=96, ny=80, dx=0.05, dy=0.05, eps=[0.2], dt=0.01)
    full, _, _, _ = oracle.run_member(cfg, 0, np.float64, nsteps=20, u0=inputs.uniform_dense_rows(96, 80, 0, 80))
    samples = [(40, 48), (1, 1), (79, 95), (10, 60), (70, 3)]
    got = oracle.window_value(cfg, 0, np.float64, 20, samples,
                              lambda j0, rows, i0, cols: inputs.uniform_dense_rows(96, 80, j0, rows)[:, i0:i0 + cols])
    for k, (j, i) in enumerate(samples):
        assert got[k] == full[j, i]


def test_row_band_windows_match_full_run():
    """Row bands stepped on their light-cone windows (band ± (nsteps + 1) rows, full width) — the
    decomposition the full-grid config-4 parity test uses — reproduce the full-grid run bitwise
    (both precisions); a halo of half that does not (the fixed window edge reaches the band: the
    error front moves one node per level, shrinking by the factor c = dt²h/d² per node, so a
    halo just short of nsteps + 1 may still round to bitwise equality)."""
    cfg = inputs.config(3, nx=70, ny=150, dx=0.05, dy=0.05, eps=[0.2], dt=0.01)
    n = 20
    for npdt in (np.float64, np.float32):
        u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(npdt)
        _, _, c1, c2 = oracle.member_coefficients(cfg, 0, npdt)
        full, _ = oracle.run(2, c1, c2, u0, None, cfg.dt, n)
        for halo, exact in ((n + 1, True), (n // 2, False)):
            same = True
            for j0 in range(0, cfg.ny, 37):
                j1 = min(cfg.ny, j0 + 37)
                w0, w1 = max(0, j0 - halo), min(cfg.ny, j1 + halo)
                un, _ = oracle.run(2, np.ascontiguousarray(c1[w0:w1]), np.ascontiguousarray(c2[w0:w1 - 1]),
                                   np.ascontiguousarray(u0[w0:w1]), None, cfg.dt, n)
                same &= bool(np.array_equal(un[j0 - w0:j1 - w0], full[j0:j1]))
            assert same == exact, (npdt, halo)


def test_energy_node_form_summation_by_parts():
    """Reading R30: with K̃ = −L symmetric and u = 0 on the Dirichlet ring, the face sum of R17 equals
    the node form ⟨u^{n+1}, K̃u^n⟩ = −Σ u^{n+1}·L(u^n) (summation by parts), so
    E = (dx·dy/dt²)·[Σ (u^{n+1} − u^n)² − Σ u^{n+1}·L(u^n)] — the form the fused GPU energy
    evaluates.  Checked on random faces and fields (2D and 1D), using the oracle's own L and energy."""
    rng = np.random.default_rng(21)
    for dim, shape in ((2, (23, 31)), (1, (40,))):
        ny, nx = (shape[0], shape[1]) if dim == 2 else (1, shape[0])
        dx, dy, dt = 0.03, 0.05, 0.004
        h1 = rng.uniform(0.5, 2.0, (ny, nx - 1) if dim == 2 else (nx - 1,))
        h2 = rng.uniform(0.5, 2.0, (ny - 1, nx)) if dim == 2 else None
        c1 = oracle.prescale(h1, dt, dx, np.float64)
        c2 = oracle.prescale(h2, dt, dy, np.float64) if dim == 2 else None
        a = rng.standard_normal(shape)
        b = rng.standard_normal(shape)
        for u in (a, b):
            if dim == 2:
                u[0, :] = u[-1, :] = u[:, 0] = u[:, -1] = 0.0
            else:
                u[0] = u[-1] = 0.0
        E = oracle.energy(dim, c1, c2, a, b, dx, dy, dt)
        w = (dx * dy if dim == 2 else dx) / dt ** 2
        node = w * (np.sum((a - b) ** 2) - np.sum(a * oracle.lap(dim, c1, c2, b)))
        assert abs(node - E) <= 1e-12 * abs(E)
