"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bars (BASELINE.json north_star, R19/R20):
  * stepping with SHARED fp64 faces (tsw_set_coeff_faces): bitwise equal (same canonical tree);
  * end to end with the GPU coefficient builder (CUDA exp vs libm exp, ≤ 2 ulp per face):
    relative max-norm ≤ 1e−12 (fp64) / ≤ 1e−5 (fp32);
  * energy: ≤ 1e−12 relative (different fp64 summation order); A₂: exact given equal fields.
"""
import numpy as np
import pytest

import oracle
from paper_2005_11931_b200 import inputs, tsw
from tests.helpers import NP, TOL, abi_faces, check_slabs_against_oracle, host_cores, rel_maxnorm

pytestmark = pytest.mark.gpu

oracle.set_threads(host_cores())


def _solver(cfg, dtype, **kw):
    return tsw.Solver(cfg.dim, cfg.nx, cfg.ny, cfg.dx, cfg.dy, cfg.batch, dtype, **kw)


def _oracle_faces(cfg, b, **kw):
    return oracle.build_faces(cfg.dim, cfg.kind, cfg.order, cfg.h_background, cfg.amp[b], cfg.xs, cfg.ys,
                              cfg.eps[b], cfg.nx, cfg.ny, cfg.dx, cfg.dy, **kw)


def _shared_faces_solver(cfg, dtype, faces):
    """GPU solver whose faces are the oracle's fp64 faces (bitwise stepping check)."""
    s = _solver(cfg, dtype)
    if cfg.dim == 1:
        s.set_coeff_faces(np.stack([f[0] for f in faces]))
    else:
        H = [abi_faces(h1, h2) for (h1, h2) in faces]
        s.set_coeff_faces(np.stack([h[0] for h in H]), np.stack([h[1] for h in H]))
    return s


# ---------------------------------------------------------------------------------------------
# S1 builder
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_builder_faces_within_2ulp(n):
    cfg = inputs.config(n)
    if n == 3:
        cfg = inputs.config(3, ny=64)        # faces of the line kind do not depend on y
    if n == 5:
        cfg = inputs.config(5, ny=8)
    s = tsw.Solver.from_config(cfg, "f64")
    h1g, h2g = s.read_faces()
    ulp = 4 if cfg.kind == inputs.H_DELTA_POINT else 2      # point: product of two exp values
    for b in range(cfg.batch):
        h1o, h2o = _oracle_faces(cfg, b)
        if cfg.dim == 1:
            np.testing.assert_array_max_ulp(h1g[b], h1o, maxulp=ulp)
            assert np.array_equal(h1g[b] == 1.0, h1o == 1.0)   # compact support, bitwise
            continue
        H1, H2 = abi_faces(h1o, h2o)
        np.testing.assert_array_max_ulp(h1g[b], H1, maxulp=ulp)
        np.testing.assert_array_max_ulp(h2g[b][1:-1], H2[1:-1], maxulp=ulp)
        if cfg.kind == inputs.H_DELTA_LINE_X:
            assert np.array_equal(h1g[b] == 1.0, H1 == 1.0)
    s.close()


def test_builder_order2_and_cfl_bound():
    cfg = inputs.config(2, eps=[0.1, 0.2], amp=[100.0, 3.0], order=2, h_background=10.0, dt=1e-4)
    s = tsw.Solver.from_config(cfg, "f64")
    h1g, h2g = s.read_faces()
    for b in range(2):
        h1o, h2o = _oracle_faces(cfg, b)
        np.testing.assert_array_max_ulp(h1g[b], h1o, maxulp=8)   # order 2 squares the exp error
    _, _, dt_max = s.info()
    dto = min(oracle.gershgorin_dt_max(2, *_oracle_faces(cfg, b), cfg.dx, cfg.dy) for b in range(2))
    assert abs(dt_max - dto) <= 1e-12 * dto
    s.close()


# ---------------------------------------------------------------------------------------------
# S2 + S3 stepping, bitwise with shared faces (several tiles + ragged tail)
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("shape", [(77, 300), (5, 67), (3, 3), (130, 129)])
def test_stepping_bitwise_dense_faces_random(dtype, shape):
    ny, nx = shape
    rng = np.random.default_rng(7)
    B = 2
    cfg = inputs.config(3, nx=nx, ny=ny, dx=0.05, dy=0.04, eps=[0.5] * B, amp=[1.0] * B, dt=0.004)
    faces = [(rng.uniform(0.5, 2.0, (ny, nx - 1)), rng.uniform(0.5, 2.0, (ny - 1, nx))) for _ in range(B)]
    dt = 0.6 * min(oracle.gershgorin_dt_max(2, h1, h2, cfg.dx, cfg.dy) for h1, h2 in faces)
    s = _shared_faces_solver(cfg, dtype, faces)
    u0 = np.stack([inputs.uniform_dense((ny, nx), seed=11 + b) for b in range(B)]).astype(NP[dtype])
    u1 = np.stack([inputs.uniform_dense((ny, nx), seed=21 + b) for b in range(B)]).astype(NP[dtype])
    s.set_initial(u0, u1, dt)
    s.step(57)
    g = s.read(0)
    gp = s.read(1)
    for b in range(B):
        c1 = oracle.prescale(faces[b][0], dt, cfg.dx, NP[dtype])
        c2 = oracle.prescale(faces[b][1], dt, cfg.dy, NP[dtype])
        un, unm1 = oracle.run(2, c1, c2, u0[b], u1[b], dt, 57)
        assert np.array_equal(g[b], un), f"member {b}: max diff {np.max(np.abs(g[b] - un))}"
        assert np.array_equal(gp[b], unm1)
    s.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_stepping_bitwise_line_mode_const(dtype):
    """LINE-mode kernel (row-invariant coefficients) bitwise: constant h has identical faces on both sides."""
    cfg = inputs.config(3, nx=520, ny=200, dx=0.01, dy=0.01, eps=[0.3, 0.3], amp=[0.0, 0.0], dt=0.004)
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_coeff(tsw.TSW_H_CONST, cfg.eps, 1.7)
    u0 = inputs.uniform_dense((200, 520), seed=3).astype(NP[dtype])
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(100)
    g = s.read(0)
    h1 = np.full((200, 519), 1.7)
    h2 = np.full((199, 520), 1.7)
    un, _ = oracle.run(2, oracle.prescale(h1, cfg.dt, cfg.dx, NP[dtype]), oracle.prescale(h2, cfg.dt, cfg.dy, NP[dtype]),
                       u0, None, cfg.dt, 100)
    assert np.array_equal(g[0], un) and np.array_equal(g[1], un)
    s.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_stepping_bitwise_line_mode_shared_faces_via_readback(dtype):
    """LINE mode with the GPU-built δ-line faces read back and given to the oracle: bitwise."""
    cfg = inputs.config(3, nx=1000, ny=300, dx=0.004, dy=0.004, eps=[0.05, 0.2], amp=[1.0, 1.0], dt=8e-4)
    s = tsw.Solver.from_config(cfg, dtype)
    h1g, h2g = s.read_faces()
    u0 = cfg.initial().astype(NP[dtype])
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(300)
    g = s.read(0)
    for b in range(2):
        c1 = oracle.prescale(h1g[b], cfg.dt, cfg.dx, NP[dtype])
        c2 = oracle.prescale(h2g[b][1:-1], cfg.dt, cfg.dy, NP[dtype])
        un, _ = oracle.run(2, c1, c2, u0, None, cfg.dt, 300)
        assert np.array_equal(g[b], un)
    s.close()


# ---------------------------------------------------------------------------------------------
# Configs end to end (GPU builder) — tolerance of north_star
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_config1_end_to_end(dtype):
    cfg = inputs.config(1, eps=[0.05, 0.05], amp=[1.0, 0.0])   # + background member for A₂
    s = tsw.Solver.from_config(cfg, dtype)
    u0 = cfg.initial().astype(NP[dtype])
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    E_half = None
    s.step(1)
    E_half = s.energy()
    s.step(cfg.nsteps - 1)
    g = s.read(0)
    E_end = s.energy()
    w2, idx = s.wave2(1)
    ref = []
    for b in range(2):
        un, unm1, c1, _ = oracle.run_member(cfg, b, NP[dtype])
        ref.append(un)
        assert rel_maxnorm(g[b], un) <= TOL[dtype]
        Eo = oracle.energy(1, c1, None, un, unm1, cfg.dx, cfg.dy, cfg.dt)
        assert abs(E_end[b] - Eo) <= (1e-12 if dtype == "f64" else 1e-6) * Eo
    # energy conservation over 4000 steps (R17)
    assert np.all(np.abs(E_end - E_half) <= (1e-12 if dtype == "f64" else 1e-4) * E_half)
    wo, io = oracle.wave2(1, ref[0], ref[1], cfg.dx, 0.0, 0.05)
    np.testing.assert_allclose(w2[0], wo, rtol=0, atol=(1e-11 if dtype == "f64" else 1e-4) * 40)
    assert np.all(w2[1] == 0.0)                               # background member: A₂ ≡ 0
    if dtype == "f64":
        assert np.array_equal(idx[0], io)


def test_config1_stepping_bitwise_shared_faces():
    cfg = inputs.config(1)
    for dtype in ("f64", "f32"):
        faces = [_oracle_faces(cfg, 0)]
        s = _shared_faces_solver(cfg, dtype, faces)
        u0 = cfg.initial().astype(NP[dtype])[None]
        s.set_initial(u0, None, cfg.dt)
        s.step(cfg.nsteps)
        un, unm1, _, _ = oracle.run_member(cfg, 0, NP[dtype])
        g = s.read(0)
        assert np.array_equal(g[0], un)
        assert np.array_equal(s.read(1)[0], unm1)
        s.close()


def test_1d_global_fallback_path_bitwise():
    """nx too large for the shared-memory persistent kernel → per-step global kernel."""
    nx = 20000
    cfg = inputs.config(1, nx=nx, dx=0.0005, eps=[0.05], dt=1e-4)
    faces = [_oracle_faces(cfg, 0)]
    s = _shared_faces_solver(cfg, "f64", faces)
    u0 = inputs.uniform_dense((nx,), seed=1, dim=1)[None]
    s.set_initial(u0, None, cfg.dt)
    s.step(300)
    c1 = oracle.prescale(faces[0][0], cfg.dt, cfg.dx, np.float64)
    un, _ = oracle.run(1, c1, None, u0[0], None, cfg.dt, 300)
    assert np.array_equal(s.read(0)[0], un)


def test_config2_end_to_end():
    cfg = inputs.config(2)
    s = tsw.Solver.from_config(cfg, "f64")
    u0 = cfg.initial()
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(1)
    E_half = s.energy()
    s.step(cfg.nsteps - 1)
    g = s.read(0)
    E = s.energy()
    w2, idx = s.wave2(3)
    ref = []
    for b in range(cfg.batch):
        un, unm1, c1, c2 = oracle.run_member(cfg, b, np.float64)
        ref.append(un)
        assert rel_maxnorm(g[b], un) <= 1e-12, f"member {b}"
        Eo = oracle.energy(2, c1, c2, un, unm1, cfg.dx, cfg.dy, cfg.dt)
        assert abs(E[b] - Eo) <= 1e-12 * Eo
        assert np.array_equal(g[b], g[b][::-1, :])              # y-mirror symmetry, bitwise
    assert np.all(np.abs(E - E_half) <= 1e-12 * E_half)
    for b in range(cfg.batch):
        wo, io = oracle.wave2(2, ref[b], ref[3], cfg.dx, 0.0, cfg.eps[b])
        np.testing.assert_allclose(w2[b], wo, rtol=0, atol=1e-11)
    assert np.all(w2[3] == 0.0)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_config3_full_size(dtype):
    """4096² δ-line, the full 5000 steps against the full oracle run, with
    the energy at n = 100 and n = 5000 against the oracle's.  Invariant drift (R17, discrete
    CL-01): fp64 ≤ 1e−12 relative; fp32 — the fields are rounded every step, so
    the invariant moves by O(ε₃₂) per step on BOTH sides — the GPU's drift is bounded by twice the
    oracle's own fp32 drift on the same run (R29)."""
    cfg = inputs.config(3)
    s = tsw.Solver.from_config(cfg, dtype)
    u0 = cfg.initial().astype(NP[dtype])
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(100)
    E100 = s.energy()[0]
    s.step(cfg.nsteps - 100)
    E = s.energy()[0]
    g = s.read(0)
    s.close()
    un, unm1, c1, c2 = oracle.run_member(cfg, 0, NP[dtype], nsteps=100, u0=u0)
    Eo100 = oracle.energy(2, c1, c2, un, unm1, cfg.dx, cfg.dy, cfg.dt)
    un, unm1 = oracle.leapfrog(2, c1, c2, un, unm1, cfg.nsteps - 100)
    Eo = oracle.energy(2, c1, c2, un, unm1, cfg.dx, cfg.dy, cfg.dt)
    assert rel_maxnorm(g[0], un) <= TOL[dtype]
    etol = 1e-12 if dtype == "f64" else 1e-6
    assert abs(E100 - Eo100) <= etol * Eo100 and abs(E - Eo) <= etol * Eo
    if dtype == "f64":
        assert abs(E - E100) <= 1e-12 * E100
    else:
        assert abs(E - E100) <= 2.0 * abs(Eo - Eo100) + 1e-12 * E100
    assert np.array_equal(g[0], g[0][::-1, :])
    assert np.all(np.isfinite(g))


def _dense_rows(cfg):
    return lambda j0, rows, i0, cols: inputs.uniform_dense_rows(cfg.nx, cfg.ny, j0, rows)[:, i0:i0 + cols]


from bench import TB_DEFAULT as BENCH_K   # bench.py's default temporal-blocking depth per dtype


@pytest.mark.parametrize("dtype,K,full", [("f64", 1, False), ("f32", 1, False), ("f64", BENCH_K["f64"], False),
                                          ("f32", BENCH_K["f32"], False), ("f64", BENCH_K["f64"], True),
                                          ("f32", BENCH_K["f32"], True)])
def test_config4_weak_unit_sampled_windows(dtype, K, full):
    """The bench workload (32768 × 4096 slab, dense data) in the bench's launch configuration
    (temporally blocked, K per dtype; K = 1 too) and the full 32768² config-4 grid
    (`bench.py --scaling strong`): sampled nodes against light-cone oracle windows, bitwise with
    the GPU's own faces."""
    cfg = inputs.config(4) if full else inputs.weak_unit(1)
    s = tsw.Solver.from_config(cfg, dtype)
    if K > 1:
        s.set_option(tsw.TSW_OPT_TBLOCK, K)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(NP[dtype])
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    nsteps = 40
    s.step(nsteps)
    g = s.read(0)[0]
    rng = np.random.default_rng(5)
    V = 2 if dtype == "f64" else 4
    samples = [(0, 0), (1, 1), (cfg.ny - 2, cfg.nx - 2), (cfg.ny - 1, 100), (2048, cfg.nx // 2 - 1),
               (2048, cfg.nx // 2), (17, 32 * V - 1), (17, 32 * V), (300, 64 * V - 1),
               (cfg.ny // 2, 503), (cfg.ny // 2, 504), (cfg.ny // 2, 505), (5, 1007), (cfg.ny - 3, 1008)]
    samples += [(int(rng.integers(0, cfg.ny)), int(rng.integers(0, cfg.nx))) for _ in range(40)]
    thin = tsw.Solver.from_config(inputs.weak_unit(1, rows_per_rank=8), dtype)
    line = thin.read_faces()[0][0, 0]
    thin.close()
    # oracle windows with the GPU-built line faces (bitwise stepping) — faces are x-only
    got = []
    R = nsteps + 1
    for (j, i) in samples:
        i0, i1 = max(0, i - R), min(cfg.nx, i + R + 1)
        j0, j1 = max(0, j - R), min(cfg.ny, j + R + 1)
        c1 = oracle.prescale(np.tile(line[i0:i1 - 1], (j1 - j0, 1)), cfg.dt, cfg.dx, NP[dtype])
        c2 = oracle.prescale(np.full((j1 - j0 - 1, i1 - i0), 1.0), cfg.dt, cfg.dy, NP[dtype])
        w0 = np.ascontiguousarray(u0[j0:j1, i0:i1])
        un, _ = oracle.run(2, c1, c2, w0, None, cfg.dt, nsteps)
        got.append(un[j - j0, i - i0])
    for k, (j, i) in enumerate(samples):
        assert g[j, i] == got[k], f"node {(j, i)}"
    # and against the oracle's own faces, end to end, at a few nodes
    vals = oracle.window_value(cfg, 0, NP[dtype], nsteps, samples[:6], lambda j0, r, i0, c: u0[j0:j0 + r, i0:i0 + c])
    for k, (j, i) in enumerate(samples[:6]):
        assert abs(float(g[j, i]) - float(vals[k])) <= TOL[dtype] * max(1.0, float(np.max(np.abs(g))))
    s.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_config4_full_grid_every_node(dtype):
    """Config 4's full 32768² grid, 20 steps ("oracle parity 20 steps on the full
    grid"), dense data, in the bench's launch configuration (temporally blocked, K =
    bench.TB_DEFAULT): EVERY node of u^20 against the oracle.  The oracle runs in row bands, each on
    its light-cone window (band ± 21 rows): the scheme moves information one node per step, so the
    window's fixed edge cannot reach the band (SURVEY §8(c) exact lattice speed; the window run
    reproducing the full run bitwise is pinned in tests/test_oracle_pins.py).  Bitwise with the
    GPU's own δ-line faces; ≤ TOL with the oracle's own faces."""
    cfg = inputs.config(4)
    nsteps, halo, band = 20, 21, 2048
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_option(tsw.TSW_OPT_TBLOCK, BENCH_K[dtype])
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(NP[dtype])
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    del u0
    s.step(nsteps)
    g = s.read(0)[0]
    s.close()
    assert np.all(np.isfinite(g))
    thin = tsw.Solver.from_config(inputs.config(4, ny=8), dtype)   # δ-line faces depend on x only
    h1g, h2g = thin.read_faces()
    thin.close()
    h1o, h2o = oracle.build_faces(2, cfg.kind, cfg.order, cfg.h_background, cfg.amp[0], cfg.xs, cfg.ys, cfg.eps[0],
                                  cfg.nx, cfg.ny, cfg.dx, cfg.dy, 0, 0, cfg.nx, 2)
    rows = {"gpu": (h1g[0, 0], h2g[0, 1]), "oracle": (h1o[0], h2o[0])}
    gmax = float(np.max(np.abs(g)))
    for j0 in range(0, cfg.ny, band):
        j1 = min(cfg.ny, j0 + band)
        w0, w1 = max(0, j0 - halo), min(cfg.ny, j1 + halo)
        uw = inputs.uniform_dense_rows(cfg.nx, cfg.ny, w0, w1 - w0).astype(NP[dtype])
        for which, (r1, r2) in rows.items():
            c1 = np.ascontiguousarray(np.broadcast_to(oracle.prescale(r1, cfg.dt, cfg.dx, NP[dtype]), (w1 - w0, cfg.nx - 1)))
            c2 = np.ascontiguousarray(np.broadcast_to(oracle.prescale(r2, cfg.dt, cfg.dy, NP[dtype]), (w1 - w0 - 1, cfg.nx)))
            un, _ = oracle.run(2, c1, c2, uw, None, cfg.dt, nsteps)
            got, ref = g[j0:j1], un[j0 - w0:j1 - w0]
            if which == "gpu":
                bad = np.argwhere(got != ref)
                assert bad.size == 0, f"rows {j0}..{j1}: {len(bad)} nodes differ, first {bad[:3].tolist()}"
            else:
                err = float(np.max(np.abs(got.astype(np.float64) - ref.astype(np.float64))))
                assert err <= TOL[dtype] * gmax, f"rows {j0}..{j1}: {err}"


def test_config5_batched_family():
    """65 × 2048² ε family (SURVEY §8(d) config 5 parity plan): all 65 members against the oracle at
    200 steps; ε_min, ε_mid, ε_max and the background member (A = 0) against the oracle for the full
    4000 steps (fields, energy, A₂± with its index); energy conservation of every member over the
    4000 steps; A₂ of other members against brute force; batch ≡ single-member launches, bitwise."""
    cfg = inputs.config(5)
    s = tsw.Solver.from_config(cfg, "f64")
    u0 = cfg.initial()
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(200)
    g200 = s.read(0)
    for b in range(cfg.batch):
        un, _, _, _ = oracle.run_member(cfg, b, np.float64, nsteps=200, u0=u0)
        assert rel_maxnorm(g200[b], un) <= 1e-12, f"member {b} at 200 steps"
    del g200
    E0 = s.energy()
    for _ in range(3):
        s.step(1000)
    s.step(cfg.nsteps - 3200)
    E = s.energy()
    assert np.all(np.abs(E - E0) <= 1e-12 * E0)
    g = s.read(0)
    w2, idx = s.wave2(64)
    full = {}
    for b in (0, 31, 63, 64):          # ε_min, ε_mid, ε_max (R21), background
        un, unm1, c1, c2 = oracle.run_member(cfg, b, np.float64, u0=u0)
        assert rel_maxnorm(g[b], un) <= 1e-12, f"member {b} at {cfg.nsteps} steps"
        Eo = oracle.energy(2, c1, c2, un, unm1, cfg.dx, cfg.dy, cfg.dt)
        assert abs(E[b] - Eo) <= 1e-12 * Eo
        full[b] = un
    for b in (0, 31, 63):
        wo, io = oracle.wave2(2, full[b], full[64], cfg.dx, cfg.xs, cfg.eps[b])
        tol = 1e-12 * np.max(np.abs(full[b]))
        np.testing.assert_allclose(w2[b], wo, rtol=0, atol=tol)
        # the GPU's arg-extremum is an extremum of the oracle's field too (equal up to rounding)
        dd = (full[b] - full[64]).reshape(-1)
        for k in range(2):
            assert inputs.node_coords(cfg.nx, cfg.dx)[idx[b, k] % cfg.nx] <= cfg.xs - cfg.eps[b]
            assert abs(dd[idx[b, k]] - wo[k]) <= 2 * tol
    assert np.all(w2[64] == 0.0)
    x = inputs.node_coords(cfg.nx, cfg.dx)
    for b in (0, 10, 31, 63, 64):
        reg = x <= -cfg.eps[b]
        d = (g[b] - g[64])[:, reg]
        assert w2[b, 0] == d.max() and w2[b, 1] == d.min()
    # batch equivalence: members alone
    for b in (0, 31, 63):
        one = inputs.config(5, eps=[cfg.eps[b]], amp=[cfg.amp[b]])
        s1 = tsw.Solver.from_config(one, "f64")
        s1.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
        s1.step(cfg.nsteps)
        assert np.array_equal(s1.read(0)[0], g[b])
        s1.close()
    s.close()


# ---------------------------------------------------------------------------------------------
# multi-slab decomposition on one device (loopback) ≡ single domain, bitwise
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kind", [inputs.H_DELTA_LINE_X, inputs.H_DELTA_POINT])
def test_loopback_slabs_bitwise(P, dtype, kind):
    cfg = inputs.config(2, nx=260, ny=151, dx=0.01, dy=0.01, kind=kind, eps=[0.2, 0.3], amp=[1.0, 0.0], dt=1e-3)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(NP[dtype])
    one = tsw.Solver.from_config(cfg, dtype)
    one.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    one.step(80)
    ref = one.read(0)
    Eref = one.energy()
    wref, iref = one.wave2(1)
    import torch
    stream = torch.cuda.Stream()
    parts = [tsw.Solver.from_config(cfg, dtype, rank=r, nranks=P, stream=stream.cuda_stream) for r in range(P)]
    for p in parts:
        p.set_initial(np.ascontiguousarray(u0[p.r0:p.r0 + p.ny_local]), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    tsw.tsw_group_step([p.ctx for p in parts], 80)
    for p in parts:
        assert np.array_equal(p.read(0), ref[:, p.r0:p.r0 + p.ny_local])
        assert np.array_equal(p.read(1), one.read(1)[:, p.r0:p.r0 + p.ny_local])
    check_slabs_against_oracle(parts, cfg, dtype, 80, u0)
    E = sum(p.energy() for p in parts)
    np.testing.assert_allclose(E, Eref, rtol=1e-12)
    w = [p.wave2(1) for p in parts]
    for b in range(2):
        assert max(v[0][b, 0] for v in w) == wref[b, 0]
        assert min(v[0][b, 1] for v in w) == wref[b, 1]
    for p in parts:
        p.close()
    one.close()


# ---------------------------------------------------------------------------------------------
# state, resume, reversal, errors
# ---------------------------------------------------------------------------------------------

def test_set_state_resume_bitwise_and_time_reversal():
    cfg = inputs.config(3, nx=700, ny=300, dx=0.01, dy=0.01, eps=[0.1], dt=3e-3)
    u0 = cfg.initial()
    a = tsw.Solver.from_config(cfg, "f64")
    a.set_initial(u0[None], None, cfg.dt)
    a.step(150)
    un, unm1 = a.read(0), a.read(1)
    a.step(150)
    ref = a.read(0)
    b = tsw.Solver.from_config(cfg, "f64")
    b.set_state(un, unm1, 150, cfg.dt)
    b.step(150)
    assert np.array_equal(b.read(0), ref)
    assert b.info()[0] == 300
    # time reversal: (u^N, u^{N−1}) → swapped, N−1 steps → u^0
    c = tsw.Solver.from_config(cfg, "f64")
    c.set_state(a.read(1), a.read(0), 1, cfg.dt)
    c.step(299)
    assert rel_maxnorm(c.read(0)[0], u0) < 1e-12


def test_errors():
    cfg = inputs.config(3, nx=64, ny=64, dx=0.01, dy=0.01, eps=[0.1], dt=3e-3)
    s = tsw.Solver(2, 64, 64, 0.01, 0.01, 1, "f64")
    with pytest.raises(tsw.TswError) as e:
        s.step(1)
    assert e.value.status == tsw.TSW_ERR_STATE
    with pytest.raises(tsw.TswError) as e:
        s.set_initial(np.zeros((1, 64, 64)), None, 1e-3)
    assert e.value.status == tsw.TSW_ERR_STATE
    with pytest.raises(tsw.TswError) as e:
        s.set_coeff(tsw.TSW_H_DELTA_LINE_X, [1.5])
    assert e.value.status == tsw.TSW_ERR_ARG
    with pytest.raises(tsw.TswError) as e:
        s.set_coeff(tsw.TSW_H_DELTA_LINE_X, [0.1], h_background=0.0)
    assert e.value.status == tsw.TSW_ERR_ARG
    s.set_coeff(tsw.TSW_H_DELTA_LINE_X, [0.1])
    dt_max = s.info()[2]
    with pytest.raises(tsw.TswError) as e:
        s.set_initial(np.zeros((1, 64, 64)), None, dt_max * 1.0001)
    assert e.value.status == tsw.TSW_ERR_CFL
    s.set_initial(np.zeros((1, 64, 64)), None, dt_max)
    with pytest.raises(tsw.TswError) as e:
        s.energy()
    assert e.value.status == tsw.TSW_ERR_STATE
    s.step(3)
    assert np.all(s.read(0) == 0.0)
    assert s.energy()[0] == 0.0
    with pytest.raises(tsw.TswError) as e:
        s.wave2(5)
    assert e.value.status == tsw.TSW_ERR_ARG
    bad = np.ones((1, 64, 63))
    bad[0, 3, 3] = -1.0
    with pytest.raises(tsw.TswError) as e:
        s.set_coeff_faces(bad, np.ones((1, 65, 64)))
    assert e.value.status == tsw.TSW_ERR_ARG
    s.close()


def test_boundary_forced_zero_and_velocity_start():
    cfg = inputs.config(3, nx=130, ny=70, dx=0.02, dy=0.02, eps=[0.2], dt=5e-3)
    u0 = np.ones((1, 70, 130))
    u1 = np.full((1, 70, 130), 2.0)
    s = tsw.Solver.from_config(cfg, "f64")
    s.set_initial(u0, u1, cfg.dt)
    s.step(1)
    g = s.read(0)
    assert np.all(g[0, 0] == 0) and np.all(g[0, -1] == 0) and np.all(g[0, :, 0] == 0) and np.all(g[0, :, -1] == 0)
    h1g, h2g = s.read_faces()
    c1 = oracle.prescale(h1g[0], cfg.dt, cfg.dx, np.float64)
    c2 = oracle.prescale(h2g[0][1:-1], cfg.dt, cfg.dy, np.float64)
    z0 = u0[0].copy(); z1 = u1[0].copy()
    for z in (z0, z1):
        z[0] = z[-1] = 0; z[:, 0] = z[:, -1] = 0
    ref = oracle.startup(2, c1, c2, z0, z1, cfg.dt)
    assert np.array_equal(g[0], ref)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_config5_and_config3_bench_launch_configuration(dtype):
    """config 5 (65 × 2048² ε family) and config 3 (4096²) as bench.py runs them — temporally
    blocked at the dtype's K: config 5 bitwise equal to the one-level launch on every member,
    config 3 against the full oracle at 100 steps."""
    K = BENCH_K[dtype]
    cfg = inputs.config(5)
    u0 = cfg.initial().astype(NP[dtype])
    runs = []
    for k in (1, K):
        s = tsw.Solver.from_config(cfg, dtype)
        if k > 1:
            s.set_option(tsw.TSW_OPT_TBLOCK, k)
        s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
        s.step(3 * K + 1)
        runs.append((s.read(0), s.energy()))
        s.close()
    assert np.array_equal(runs[0][0], runs[1][0])
    np.testing.assert_allclose(runs[0][1], runs[1][1], rtol=1e-12)
    del runs
    cfg = inputs.config(3)
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_option(tsw.TSW_OPT_TBLOCK, K)
    u0 = cfg.initial().astype(NP[dtype])
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(100)
    un, _, _, _ = oracle.run_member(cfg, 0, NP[dtype], nsteps=100, u0=u0)
    assert rel_maxnorm(s.read(0)[0], un) <= TOL[dtype]
    s.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("shape", [(37, 1300), (9, 4100), (300, 515)])
def test_wave2_first_extremum_ties(dtype, shape):
    """S6 on fields with many equal extrema: the values are fl_T(u_b − u_bg) exactly and the index is
    the FIRST extremum in row-major order of the region x ≤ x_s − ε (R18) — across threads, CTA
    tiles, row chunks and members (ragged widths, several column tiles)."""
    ny, nx = shape
    eps = [0.05, 0.2, 0.11]
    cfg = inputs.config(3, nx=nx, ny=ny, dx=0.01, dy=0.01, eps=eps + [0.1], amp=[1.0, 1.0, 1.0, 0.0], dt=2e-3)
    rng = np.random.default_rng(11)
    u = rng.integers(-3, 4, size=(cfg.batch, ny, nx)).astype(NP[dtype])    # few distinct values → ties
    u[:, 0, :] = u[:, -1, :] = 0
    u[:, :, 0] = u[:, :, -1] = 0
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_state(u, u, 5, cfg.dt)
    w2, idx = s.wave2(3)
    x = inputs.node_coords(nx, cfg.dx)
    for b in range(cfg.batch):
        reg = x <= 0.0 - cfg.eps[b]
        d = (u[b] - u[3]).astype(NP[dtype])
        masked = np.where(reg[None, :], d.astype(np.float64), np.nan)
        flat = masked.reshape(-1)
        imax, imin = int(np.nanargmax(flat)), int(np.nanargmin(flat))   # first occurrence
        assert w2[b, 0] == flat[imax] and w2[b, 1] == flat[imin]
        assert idx[b, 0] == imax and idx[b, 1] == imin, (b, idx[b], imax, imin)
    s.close()
