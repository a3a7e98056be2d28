"""Pins of the oracle's implicit scheme (R26/R27) — -m "not gpu".

* The Thomas line solves equal a dense solve with the independently assembled
  B = (I − ½K̃x)(I − ½K̃y) (≤ 1e−12); 1D likewise.
* Closed form per mode for constant coefficients (commuting K̃x, K̃y): (1 + ½λx)(1 + ½λy) = 1/cos θ,
  a^n = a^0 cos nθ (u₁ = 0) — brute force on a tiny grid.
* Unconditional stability: the paper's Table-1 time step (Courant ≈ 30× the explicit limit) stays
  bounded, while leapfrog at the same dt overflows.
* Consistency: at a small dt the implicit and leapfrog solutions of the same problem agree to
  second order (difference ratio ≈ 4 when dt halves).
"""
import math

import numpy as np
import pytest

import oracle
from paper_2005_11931_b200 import inputs


def _assemble_xy(c1, c2):
    """K̃x, K̃y (−L_x, −L_y) on the interior unknowns, assembled from the face coefficients."""
    ny, nx = c1.shape[0], c1.shape[1] + 1
    inner = [(j, i) for j in range(1, ny - 1) for i in range(1, nx - 1)]
    idx = {p: k for k, p in enumerate(inner)}
    n = len(inner)
    Kx, Ky = np.zeros((n, n)), np.zeros((n, n))
    for k, (j, i) in enumerate(inner):
        for (cf, nb) in ((c1[j, i], (j, i + 1)), (c1[j, i - 1], (j, i - 1))):
            Kx[k, k] += cf
            if nb in idx:
                Kx[k, idx[nb]] -= cf
        for (cf, nb) in ((c2[j, i], (j + 1, i)), (c2[j - 1, i], (j - 1, i))):
            Ky[k, k] += cf
            if nb in idx:
                Ky[k, idx[nb]] -= cf
    return Kx, Ky, inner


def test_line_solves_equal_dense_solve():
    rng = np.random.default_rng(0)
    ny, nx = 9, 11
    c1 = rng.uniform(0.2, 5.0, (ny, nx - 1))
    c2 = rng.uniform(0.2, 5.0, (ny - 1, nx))
    r = rng.standard_normal((ny, nx))
    s = oracle.implicit_solve(2, c1, c2, r)
    Kx, Ky, inner = _assemble_xy(c1, c2)
    I = np.eye(len(inner))
    B = (I + 0.5 * Kx) @ (I + 0.5 * Ky)
    ref = np.linalg.solve(B, np.array([r[j, i] for (j, i) in inner]))
    got = np.array([s[j, i] for (j, i) in inner])
    assert np.max(np.abs(got - ref)) < 1e-12 * np.max(np.abs(ref))
    assert np.all(s[0] == 0) and np.all(s[-1] == 0) and np.all(s[:, 0] == 0) and np.all(s[:, -1] == 0)
    # 1D
    c = rng.uniform(0.2, 5.0, 40)
    r1 = rng.standard_normal(41)
    s1 = oracle.implicit_solve(1, c, None, r1)
    K1 = np.diag(c[:-1] + c[1:]) - np.diag(c[1:-1], 1) - np.diag(c[1:-1], -1)
    ref1 = np.linalg.solve(np.eye(39) + 0.5 * K1, r1[1:-1])
    assert np.max(np.abs(s1[1:-1] - ref1)) < 1e-12 * np.max(np.abs(ref1))


def test_modal_closed_form_constant_coefficients():
    ny, nx, n = 8, 10, 60
    cx, cy = 3.0, 7.0                                    # Courant² far above the explicit limit
    c1, c2 = np.full((ny, nx - 1), cx), np.full((ny - 1, nx), cy)
    u0 = inputs.uniform_dense((ny, nx), seed=3)
    un, _ = oracle.implicit_run(2, c1, c2, u0, None, 1.0, n)
    Kx, Ky, inner = _assemble_xy(c1, c2)
    lam, Q = np.linalg.eigh(Kx + Ky)                     # Kx, Ky commute: a common eigenbasis
    lx = np.einsum("ij,jk,ki->i", Q.T, Kx, Q)
    ly = np.einsum("ij,jk,ki->i", Q.T, Ky, Q)
    beta = (1 + 0.5 * lx) * (1 + 0.5 * ly)
    th = np.arccos(1.0 / beta)
    a0 = Q.T @ np.array([u0[j, i] for (j, i) in inner])
    ref = Q @ (a0 * np.cos(n * th))
    got = np.array([un[j, i] for (j, i) in inner])
    assert np.max(np.abs(got - ref)) < 1e-11


def test_unconditional_stability_at_table1_step():
    """PAPER §4: Δt = 0.05 with depth up to 100 — ≈ 30× the explicit Courant limit here."""
    sc = inputs.paper_2d(dx=0.5)
    P = oracle.Profile(sc.seg_value, sc.seg_break, isotropic=True)
    h1, h2 = oracle.build_faces_profile(2, P, 0.8, sc.nx, sc.ny, sc.dx)
    # Table 1 at 4096²: dx = 100/4095, bound dx/(10√2) = 1.73e−3, Δt = 0.05 ⇒ ratio ≈ 29
    dt = 29.0 * oracle.gershgorin_dt_max(2, h1, h2, sc.dx, sc.dx)
    c1, c2 = oracle.prescale(h1, dt, sc.dx, np.float64), oracle.prescale(h2, dt, sc.dx, np.float64)
    u0 = inputs.uniform_dense((sc.ny, sc.nx), seed=1)
    un, _ = oracle.implicit_run(2, c1, c2, u0, None, dt, 300)
    assert np.all(np.isfinite(un)) and np.max(np.abs(un)) < 10.0
    lf, _ = oracle.run(2, c1, c2, u0, None, dt, 60)
    assert not np.all(np.isfinite(lf)) or np.max(np.abs(lf)) > 1e6


def test_second_order_agreement_with_leapfrog():
    cfg = inputs.config(3, nx=201, ny=161, dx=0.02, dy=0.02, eps=[0.2], dt=1e-3)
    h1, h2 = oracle.build_faces(2, cfg.kind, 1, 1.0, 1.0, 0.0, 0.0, 0.2, cfg.nx, cfg.ny, cfg.dx, cfg.dy)
    u0 = inputs.gaussian_2d(cfg.nx, cfg.ny, cfg.dx, cfg.dy, x0=-0.5)
    T, diffs = 0.5, []
    for dt in (4e-3, 2e-3):
        n = int(round(T / dt))
        c1, c2 = oracle.prescale(h1, dt, cfg.dx, np.float64), oracle.prescale(h2, dt, cfg.dy, np.float64)
        a, _ = oracle.implicit_run(2, c1, c2, u0, None, dt, n)
        b, _ = oracle.run(2, c1, c2, u0, None, dt, n)
        diffs.append(np.max(np.abs(a - b)))
    assert 3.5 < diffs[0] / diffs[1] < 4.5
