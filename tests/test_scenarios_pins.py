"""Pins for the paper's own scenarios in the oracle (-m "not gpu").

* Φ, the mollifier's primitive: against 40-digit mpmath quadrature, Φ(0) = ½,
  Φ(t) + Φ(−t) = 1, Φ′ = φ.
* The regularised discontinuous depth (PAPER.md eq. (h2case)) and Cases 2–3
  (P:773–789): SPEC S:545's locality/midpoint checks, h_{1,ε}(70) = h_{0,ε}(70) + φ_ε(0).
* The paper's own statement about the reflected wave (§3.2.3): "In all cases the second
  wave is smaller in size. The reflected wave has only one positive component in Case I, while
  it has both positive and negative parts in Cases II and III" — checked on leapfrog runs of the
  paper's §3.2.3 set-up (Lorentzian u0, e ∈ {0.5, 0.3, 0.1}, ε = 0.2, 100δ / 100δ²).
"""
import math

import mpmath
import numpy as np
import pytest

import oracle
from paper_2005_11931_b200 import inputs

mpmath.mp.dps = 40
C_MP = 1 / mpmath.quad(lambda x: mpmath.exp(1 / (x * x - 1)), [-1, 0, 1])


def _Phi_mp(t):
    return float(C_MP * mpmath.quad(lambda x: mpmath.exp(1 / (x * x - 1)), [-1, t]))


def test_primitive_against_mpmath_and_symmetry():
    ts = np.linspace(-0.999, 0.999, 37)
    got = oracle.mollifier_primitive(ts)
    ref = np.array([_Phi_mp(t) for t in ts])
    assert np.max(np.abs(got - ref)) < 2e-15
    assert oracle.mollifier_primitive([-1.0, -3.0])[0] == 0.0
    assert np.all(oracle.mollifier_primitive([1.0, 7.0]) == 1.0)
    assert abs(oracle.mollifier_primitive([0.0])[0] - 0.5) < 1e-15
    np.testing.assert_allclose(oracle.mollifier_primitive(ts) + oracle.mollifier_primitive(-ts), 1.0, atol=2e-15)
    # Φ′ = φ (central difference)
    h = 1e-5
    for t in (-0.7, -0.2, 0.0, 0.45):
        d = (oracle.mollifier_primitive([t + h])[0] - oracle.mollifier_primitive([t - h])[0]) / (2 * h)
        assert abs(d - oracle.phi_eps([t], 1.0)[0]) < 1e-8


def test_case1_profile_locality_and_midpoint():
    """SPEC S:545 (PAPER eq. (h2case)): ε = 0.2 ⇒ h_ε(50) = 100, h_ε(90) = 10 exactly, h_ε(75) = 55."""
    sc = inputs.paper_case("1")
    P = oracle.Profile(sc.seg_value, sc.seg_break)
    # paper coordinates x_p = x + 50
    assert P.eval([0.0], 0.2)[0] == 100.0
    assert P.eval([40.0], 0.2)[0] == 10.0
    assert abs(P.eval([25.0], 0.2)[0] - 55.0) < 1e-12
    xs = np.linspace(24.7, 25.3, 61)
    v = P.eval(xs, 0.2)
    assert np.all(np.diff(v) <= 0.0)                          # monotone across the jump
    assert np.all(v[xs <= 24.8 - 1e-9] == 100.0) and np.all(v[xs >= 25.2 + 1e-9] == 10.0)
    # the convolution with φ_ε of a step is the primitive (closed form of h_0 * φ_ε)
    for xp in (24.9, 25.05, 25.17):
        ref = 100.0 + (10.0 - 100.0) * _Phi_mp((xp - 25.0) / 0.2)
        assert abs(P.eval([xp], 0.2)[0] - ref) < 1e-12


def test_case2_case3_singular_terms():
    """P:779 h_{1,ε} = h_{0,ε} + φ_ε(x−70); P:787 h_{2,ε} = h_{0,ε} + φ_ε²(x−70); S:87 ≈ 104.14."""
    c2 = inputs.paper_case("2")
    c3 = inputs.paper_case("3")
    P2 = oracle.Profile(c2.seg_value, c2.seg_break, c2.sing_loc, c2.sing_amp, c2.sing_order)
    P3 = oracle.Profile(c3.seg_value, c3.seg_break, c3.sing_loc, c3.sing_amp, c3.sing_order)
    peak = float(C_MP) * math.exp(-1.0) / 0.2
    assert abs(P2.eval([20.0], 0.2)[0] - (100.0 + peak)) < 1e-12
    assert abs(P2.eval([20.0], 0.2)[0] - 104.14) < 5e-3         # SPEC S:87 example
    assert abs(P3.eval([20.0], 0.2)[0] - (100.0 + peak * peak)) < 1e-11
    xs = np.array([19.7, 19.9, 20.1, 20.3])
    np.testing.assert_allclose(P2.eval(xs, 0.2) - 100.0, oracle.phi_eps(xs - 20.0, 0.2), rtol=1e-14, atol=0)


def _reflected_components(sc, e):
    """Leapfrog run of §3.2.3's set-up to t = 2.5; the wave between the left-going main pulse and
    the singular point: sign components above 1 % of the main pulse (SPEC S:354's threshold)."""
    sc = inputs.paper_case(sc, data="lorentz", e=e, amp=100.0)
    P = oracle.Profile(sc.seg_value, sc.seg_break, sc.sing_loc, sc.sing_amp, sc.sing_order)
    h1, _ = oracle.build_faces_profile(1, P, sc.eps[0], sc.nx, 1, sc.dx)
    dt = 0.9 * oracle.gershgorin_dt_max(1, h1, None, sc.dx, sc.dx)
    T = 2.5
    n = int(math.ceil(T / dt))
    dt = T / n
    c1 = oracle.prescale(h1, dt, sc.dx, np.float64)
    un, _ = oracle.run(1, c1, None, sc.initial(), None, dt, n)
    x = inputs.node_coords(sc.nx, sc.dx)
    main = np.max(np.abs(un[(x > -20.0) & (x < -10.0)]))     # left-going half of u0 (x_p ≈ 35)
    r = un[(x > -5.0) & (x < 19.5)]                          # between it and x_p = 70
    thr = 0.01 * main
    signs, prev = [], 0
    for v in np.where(r > thr, 1, np.where(r < -thr, -1, 0)):
        if v != 0 and v != prev:
            signs.append(int(v))
        if v != 0:
            prev = v
    return main, r, signs


@pytest.mark.parametrize("e", [0.5, 0.3, 0.1])
def test_paper_reflected_wave_structure(e):
    # Case I (discontinuous h_0): one positive component
    main, r, signs = _reflected_components("1", e)
    assert signs == [1]
    assert np.max(np.abs(r)) < main                          # "the second wave is smaller in size"
    # Cases II and III (100δ, 100δ²): both positive and negative parts
    for case in ("2", "3"):
        main, r, signs = _reflected_components(case, e)
        assert 1 in signs and -1 in signs
        assert np.max(np.abs(r)) < main


def test_profile_faces_2d_isotropic_and_vector():
    sc = inputs.paper_2d(dx=0.5)
    P = oracle.Profile([100.0, 10.0], [25.0], [20.0], [3.0], [1], isotropic=True)
    h1, h2 = oracle.build_faces_profile(2, P, 0.8, sc.nx, sc.ny, sc.dx)
    x_nodes = inputs.node_coords(sc.nx, sc.dx)
    x_faces = ((2 * np.arange(sc.nx - 1) + 2 - sc.nx) * sc.dx) / 2
    assert np.all(h1 == h1[0]) and np.all(h2 == h2[0])       # x-only
    np.testing.assert_array_equal(h1[0], P.eval(x_faces, 0.8))
    np.testing.assert_array_equal(h2[0], P.eval(x_nodes, 0.8))
    Pv = oracle.Profile([100.0, 10.0], [25.0], [20.0], [3.0], [1], isotropic=False)
    _, h2v = oracle.build_faces_profile(2, Pv, 0.8, sc.nx, sc.ny, sc.dx)
    np.testing.assert_array_equal(h2v[0], Pv.eval(x_nodes, 0.8, with_sing=False))


# --- NEXT 2 diagnostics: pins of the oracle definitions ---------------------------------------

def test_family_l2_metric_and_closed_form():
    x = inputs.node_coords(4001, 0.005)
    g = np.exp(-(x ** 2) / 0.08)                              # ‖g‖² = √(π·0.04) (closed form)
    U = np.stack([g, g + 0.5 * g, g - 2.0 * g, np.sin(x)])
    D = oracle.family_l2(U, 0.005)
    assert np.all(D == D.T) and np.all(np.diag(D) == 0.0)
    ng = (math.pi * 0.04) ** 0.25
    assert abs(D[0, 1] - 0.5 * ng) < 1e-12 and abs(D[0, 2] - 2.0 * ng) < 1e-12
    for i in range(4):
        for j in range(4):
            for k in range(4):
                assert D[i, j] <= D[i, k] + D[k, j] + 1e-14


def test_field_norms_closed_forms():
    """Gaussian g = e^{−(x²+y²)/w}: ‖g‖² = πw/2, ‖∂x g‖² = π/2 (any w) — second-order accurate."""
    n, dx, w = 801, 0.005, 0.08
    x = inputs.node_coords(n, dx)
    g = np.exp(-(x[None, :] ** 2 + x[:, None] ** 2) / w)
    out = oracle.field_norms(2, g, 0.5 * g, dx, dx, 0.1)
    assert abs(out[0] - math.sqrt(math.pi * w / 2)) < 1e-9
    assert abs(out[1] - 5.0 * math.sqrt(math.pi * w / 2)) < 1e-9     # ‖(g − g/2)/0.1‖
    assert abs(out[2] - math.sqrt(math.pi / 2)) < 1e-4 and abs(out[3] - out[2]) < 1e-12


def test_dphi_and_moderateness_exponents():
    """φ_ε′ against central differences; SPEC S:89–97 / S:369–377: N0 ≈ 1, 2, 3 for Cases 1, 2, 3."""
    for eps in (0.05, 0.3):
        d = np.linspace(-0.95 * eps, 0.95 * eps, 41)
        h = 1e-6 * eps
        fd = (oracle.phi_eps(d + h, eps) - oracle.phi_eps(d - h, eps)) / (2 * h)
        np.testing.assert_allclose(oracle.dphi_eps(d, eps), fd, rtol=1e-6, atol=1e-6 / eps ** 2)
    # the derivative seminorm of each singular part scales as an exact power of ε⁻¹ (SPEC S:97:
    # jump 90·φ(0)/ε ⇒ 1; δ: φ_ε′ = ε⁻²φ′ ⇒ 2; δ²: (φ_ε²)′ ∝ ε⁻³ ⇒ 3); the full W^{1,∞} norm
    # approaches these slopes as ε → 0
    ladder = [0.2, 0.1, 0.05, 0.025]
    parts = {"1": oracle.Profile([100.0, 10.0], [25.0]),
             "2": oracle.Profile([100.0], [], [20.0], [1.0], [1]),
             "3": oracle.Profile([100.0], [], [20.0], [1.0], [2])}
    for case, N0 in (("1", 1.0), ("2", 2.0), ("3", 3.0)):
        P = parts[case]
        c0 = 25.0 if case == "1" else 20.0
        semi = []
        for e in ladder:
            xs = c0 + np.linspace(-e, e, 20001)
            semi.append(np.max(np.abs(oracle.profile_derivative(P, xs, e))))
        assert abs(oracle.moderateness_exponent(ladder, semi) - N0) < 0.01

def test_paper_difference_kernel_H():
    """H = h_{ε1} − h_{ε2} = 90 ∫_{(x−75)/ε1}^{(x−75)/ε2} φ(z) dz, and H ≡ 0 away from
    the jump (outside the union of supports)."""
    sc = inputs.paper_case("1")
    P = oracle.Profile(sc.seg_value, sc.seg_break)
    e1, e2 = 0.2, 0.1
    for xp in (24.85, 24.95, 25.0, 25.07, 25.15):
        H = P.eval([xp], e1)[0] - P.eval([xp], e2)[0]
        t1, t2 = (xp - 25.0) / e1, (xp - 25.0) / e2
        ref = 90.0 * float(C_MP * mpmath.quad(lambda z: mpmath.exp(1 / (z * z - 1)) if abs(z) < 1 else 0,
                                              [t1, t2]))
        assert abs(H - ref) < 1e-11
    far = np.array([10.0, 24.79, 25.21, 40.0])
    assert np.all(P.eval(far, e1) - P.eval(far, e2) == 0.0)


def _case1_reflection(eps, dx, T=5.0):
    """Oracle leapfrog runs of Case 1 (h_0 = 100 | 10 at x_p = 75, mollified with ε) and
    of the uniform h = 100 background, both from the paper's Gaussian u0 = 40 e^{−(x_p−40)²/8}
    (P:809); A₂± of R18 over x ≤ 75 − ε, and the transmitted peak beyond the jump."""
    sc = inputs.paper_case("1", eps=eps, dx=dx)
    hj, _ = oracle.build_faces_profile(1, oracle.Profile(sc.seg_value, sc.seg_break), eps, sc.nx, 1, sc.dx)
    hu, _ = oracle.build_faces_profile(1, oracle.Profile([100.0]), eps, sc.nx, 1, sc.dx)
    dt = 0.9 * oracle.gershgorin_dt_max(1, hu, None, sc.dx, sc.dx)
    n = int(math.ceil(T / dt))
    dt = T / n
    u0 = sc.initial()
    a, _ = oracle.run(1, oracle.prescale(hj, dt, sc.dx, np.float64), None, u0, None, dt, n)
    b, _ = oracle.run(1, oracle.prescale(hu, dt, sc.dx, np.float64), None, u0, None, dt, n)
    w, idx = oracle.wave2(1, a, b, sc.dx, 25.0, eps)
    x = inputs.node_coords(sc.nx, sc.dx)
    trans = float(np.max(a[x > 25.0 + eps]))
    return w, float(x[idx[0]]), trans


def test_case1_reflection_is_the_impedance_mismatch():
    """S6 (A₂, R18) pinned to a textbook closed form: for u_tt = (h u_x)_x a wave crossing a jump of
    h from h1 to h2 is reflected with R = (Z1 − Z2)/(Z1 + Z2) and transmitted with T = 2Z1/(Z1 + Z2),
    Z = √h (impedance of unit density), in the limit of a transition short against the pulse.
    Case 1 (h1 = 100, h2 = 10): R = 0.5195, T = 1.5195; the right-going half of u0 has amplitude 20,
    reaches the jump at t = 3.5 (speed √100) and at t = 5 the reflected pulse is centred at
    x_p = 60.  The oracle's A₂⁺ against the uniform-depth run converges to 20R as ε → 0 (second
    order: the error shrinks ×4 per halving of ε), A₂⁻ is round-off (one positive
    component only), and the transmitted peak is 20T."""
    R = (10.0 - math.sqrt(10.0)) / (10.0 + math.sqrt(10.0))
    Tt = 2.0 * 10.0 / (10.0 + math.sqrt(10.0))
    w2, xm2, tr2 = _case1_reflection(0.2, 0.005)
    w1, xm1, tr1 = _case1_reflection(0.1, 0.005)
    e2, e1 = abs(w2[0] / (20 * R) - 1), abs(w1[0] / (20 * R) - 1)
    assert e2 < 1e-2 and e1 < 3e-3
    assert 3.0 < e2 / e1 < 5.0                                   # O(ε²) approach to the closed form
    assert abs(xm1 - 10.0) < 0.15 and abs(xm2 - 10.0) < 0.25     # x_p = 60 (centred x = 10)
    for w in (w1, w2):
        assert w[1] > -1e-9 * w[0]                               # no negative component
    assert abs(tr1 / (20 * Tt) - 1) < 1e-2


def _thin_layer_reflection(eps, dx, sigma=0.5, L=4.0, T=6.0, a=2.0):
    """Oracle runs of the configs' δ-line depth h = 1 + φ_ε(x) (R6/R7, 1D) and of the background
    h = 1, from a Gaussian u0 of amplitude a and width σ centred at x = −L, to t = T; A₂± (R18)."""
    nx = int(round(2 * (L + T + 2) / dx)) + 1
    nx += nx % 2                                     # even: x_s = 0 is a face (R9)
    x = inputs.node_coords(nx, dx)
    u0 = a * np.exp(-(x + L) ** 2 / (2 * sigma ** 2))
    u0[0] = u0[-1] = 0.0
    hl, _ = oracle.build_faces(1, 1, 1, 1.0, 1.0, 0.0, 0.0, eps, nx, 1, dx, dx)
    hb, _ = oracle.build_faces(1, 1, 1, 1.0, 0.0, 0.0, 0.0, eps, nx, 1, dx, dx)
    dt = 0.9 * oracle.gershgorin_dt_max(1, hl, None, dx, dx)
    n = int(math.ceil(T / dt))
    dt = T / n
    A, _ = oracle.run(1, oracle.prescale(hl, dt, dx, np.float64), None, u0, None, dt, n)
    B, _ = oracle.run(1, oracle.prescale(hb, dt, dx, np.float64), None, u0, None, dt, n)
    w, idx = oracle.wave2(1, A, B, dx, 0.0, eps)
    return w, x[idx]


def test_delta_line_reflection_thin_layer_limit():
    """S6 (A₂, R18) on the configs' δ-line pinned to the thin-layer (Born) limit of
    u_tt = (h u_x)_x: a layer much thinner than the pulse reflects u_r = (Δ/2)·∂_s f of the incident
    right-going wave f (amplitude a/2, here a Gaussian: max |f′| = (a/2)e^{−1/2}/σ), with
    Δ = ∫(1 − h_b/h_ε) dx (mpmath quadrature here).  So A₂⁺ → +(Δ/2)·max|f′| and A₂⁻ → −(Δ/2)·max|f′|
    — both signs, as the paper states for the δ singularity — with the positive lobe
    nearer the layer: at t = 6 the reflected pulse is centred at x = −2 (the layer at 0 reached at
    t = 4), its lobes at −2 ± σ.  The approach is second order in ε/σ."""
    sigma, a = 0.5, 2.0
    fmax = (a / 2) / sigma * math.exp(-0.5)
    errs = []
    for eps, dx in ((0.1, 0.002), (0.05, 0.001)):
        w, xi = _thin_layer_reflection(eps, dx, sigma=sigma, a=a)
        Delta = float(mpmath.quad(lambda s: 1 - 1 / (1 + C_MP / eps * mpmath.exp(1 / ((s / eps) ** 2 - 1))),
                                  [-eps, 0, eps]))
        pred = Delta / 2 * fmax
        errs.append(max(abs(w[0] / pred - 1), abs(-w[1] / pred - 1)))
        assert abs(xi[0] - (-2.0 + sigma)) < 0.1 and abs(xi[1] - (-2.0 - sigma)) < 0.1
    assert errs[0] < 3e-2 and errs[1] < 1e-2
    assert 3.0 < errs[0] / errs[1] < 5.0
