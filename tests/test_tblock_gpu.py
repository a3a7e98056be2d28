"""Temporally blocked stencil: K levels per HBM pass must give the same bits
as K = 1 and as the oracle (same canonical per-node expression), for every K, both precisions,
ragged strips / row chunks, step counts not divisible by K, and the diagnostics afterwards."""
import numpy as np
import pytest

import oracle
from paper_2005_11931_b200 import inputs, tsw
from tests.helpers import NP, check_slabs_against_oracle, host_cores

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
@pytest.mark.parametrize("K", [2, 3, 4, 5, 6, 7, 8, 9, 10])
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


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("K,levels", [(8, 13), (8, 10), (5, 7), (4, 3), (10, 23), (9, 9)])
def test_tblock_remainder_is_one_shallower_pass(dtype, K, levels):
    """A stepping call of q·K + r levels (2 ≤ r < K) runs q passes of depth K and ONE pass of depth r
    (not r one-level steps) — one launch per pass — with the bits of one-level stepping."""
    cfg = inputs.config(3, nx=900, ny=97, dx=0.01, dy=0.01, eps=[0.1], amp=[1.0], dt=2e-3)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(NP[dtype])
    s = _run(cfg, dtype, K, 1, u0)  # start-up level
    n0 = s.launches()
    s.step(levels)
    q, r = divmod(levels, K)
    # + the fused energy's final reduction when the call ends on a pass (TSW_OPT_ENERGY_FUSE)
    assert s.launches() - n0 == q + (1 if r >= 2 else r) + (1 if r != 1 else 0)
    ref = _run(cfg, dtype, 1, 1 + levels, u0)
    assert np.array_equal(s.read(0), ref.read(0))
    assert np.array_equal(s.read(1), ref.read(1))
    s.close()
    ref.close()


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


@pytest.mark.parametrize("K", [4, 8, 10])
def test_tblock_bench_shape_sampled(K):
    """The bench workload (32768 × 4096 δ-line slab) with K = 4, 8 and the bench's K = 10 (the
    start-up level, passes and a remainder pass): the whole field ≡ the K = 1 run."""
    cfg = inputs.weak_unit(1)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
    a = _run(cfg, "f64", K, 41 + K // 2, u0)
    b = _run(cfg, "f64", 1, 41 + K // 2, u0)
    ga, gb = a.read(0)[0], b.read(0)[0]
    bad = np.argwhere(ga != gb)
    if len(bad):
        # which run is wrong: oracle light-cone windows at a few nodes
        thin = tsw.Solver.from_config(inputs.weak_unit(1, rows_per_rank=8), "f64")
        line = thin.read_faces()[0][0, 0]
        thin.close()
        info = []
        for (j, i) in [tuple(bad[0]), (2048, 16000)]:
            R = 42 + K // 2
            i0, i1 = max(0, i - R), min(cfg.nx, i + R + 1)
            j0, j1 = max(0, j - R), min(cfg.ny, j + R + 1)
            c1 = oracle.prescale(np.tile(line[i0:i1 - 1], (j1 - j0, 1)), cfg.dt, cfg.dx, np.float64)
            c2 = oracle.prescale(np.full((j1 - j0 - 1, i1 - i0), 1.0), cfg.dt, cfg.dy, np.float64)
            un, _ = oracle.run(2, c1, c2, np.ascontiguousarray(u0[j0:j1, i0:i1]), None, cfg.dt, 41 + K // 2)
            info.append(((int(j), int(i)), un[j - j0, i - i0], ga[j, i], gb[j, i]))
        raise AssertionError((len(bad), bad[:4].tolist(), info))
    np.testing.assert_allclose(a.energy(), b.energy(), rtol=1e-13)
    a.close()
    b.close()


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("K", [2, 5, 8, 10])
@pytest.mark.parametrize("ny", [151, 31])
def test_tblock_loopback_slabs_bitwise(P, K, ny):
    """k-deep ghost rows: P slabs on one GPU (tsw_group_step, K-row exchanges of both levels every
    K levels, boundary rows first when the slab has ≥ 3K rows) ≡ the single-domain run, bitwise."""
    import torch
    cfg = inputs.config(3, nx=700, ny=ny, dx=0.01, dy=0.01, eps=[0.1, 0.3], amp=[1.0, 2.0], dt=2e-3)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
    n = 3 * K + 4
    ref = _run(cfg, "f64", 1, n, u0)
    stream = torch.cuda.Stream()
    parts = [tsw.Solver.from_config(cfg, "f64", rank=r, nranks=P, stream=stream.cuda_stream) for r in range(P)]
    for p in parts:
        p.set_option(tsw.TSW_OPT_TBLOCK, K)
        p.set_initial(np.ascontiguousarray(u0[p.r0:p.r0 + p.ny_local]), None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    tsw.tsw_group_step([p.ctx for p in parts], 1)         # start-up level alone
    tsw.tsw_group_step([p.ctx for p in parts], n - 1)     # TB passes + remainder
    g, gp = ref.read(0), ref.read(1)
    for p in parts:
        assert np.array_equal(p.read(0), g[:, p.r0:p.r0 + p.ny_local])
        assert np.array_equal(p.read(1), gp[:, p.r0:p.r0 + p.ny_local])
    check_slabs_against_oracle(parts, cfg, "f64", n, u0)
    E = sum(p.energy() for p in parts)
    np.testing.assert_allclose(E, ref.energy(), rtol=1e-12)
    for p in parts:
        p.close()
    ref.close()


def test_concurrent_contexts_do_not_interfere():
    """Regression: buffers are zeroed on the ctx's own (non-blocking) stream.  A legacy-stream memset
    was not ordered before the ctx's work and, with another ctx keeping the GPU busy, landed in the
    middle of it.  Run a new ctx while a temporally blocked ctx is still executing."""
    cfg = inputs.weak_unit(1, rows_per_rank=2048)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)
    ref = _run(cfg, "f64", 1, 21, u0).read(0)
    for it in range(4):
        busy = _run(cfg, "f64", 4, 41, u0)          # still running when the next ctx starts
        s = _run(cfg, "f64", 1 if it % 2 else 4, 21, u0)
        assert np.array_equal(s.read(0), ref), f"iteration {it}"
        s.close()
        busy.close()


@pytest.mark.parametrize("K", [2, 4, 8, 10])
@pytest.mark.parametrize("shape", [(3, 3), (4, 5), (5, 67), (6, 2000)])
def test_tblock_degenerate_grids(K, shape):
    """One interior node, a single interior row or column, a strip narrower than the halo: the
    temporally blocked path ≡ the one-level path, bitwise; step(0) changes nothing."""
    ny, nx = shape
    cfg = inputs.config(3, nx=nx, ny=ny, dx=0.05, dy=0.05, eps=[0.2], amp=[1.0], dt=0.005)
    u0 = inputs.uniform_dense((ny, nx), seed=13)
    ref = _run(cfg, "f64", 1, 2 * K + 3, u0)
    s = _run(cfg, "f64", K, 2 * K + 3, u0)
    before = s.read(0)
    s.step(0)
    assert np.array_equal(s.read(0), before)
    assert np.array_equal(before, ref.read(0)) and np.array_equal(s.read(1), ref.read(1))
    s.close()
    ref.close()


@pytest.mark.parametrize("warps", [4, 8])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_tblock_cta_width_bitwise(warps, dtype):
    """Both CTA widths of the temporally blocked stencil (TSW_OPT_TB_WARPS) ≡ the one-level path."""
    cfg = inputs.config(3, nx=2049, ny=97, dx=0.01, dy=0.01, eps=[0.1, 0.3], amp=[1.0, 2.0], dt=2e-3)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(NP[dtype])
    K = 4 if dtype == "f64" else 8
    ref = _run(cfg, dtype, 1, 3 * K + 2, u0)
    s = tsw.Solver.from_config(cfg, dtype)
    s.set_option(tsw.TSW_OPT_TBLOCK, K)
    s.set_option(tsw.TSW_OPT_TB_WARPS, warps)
    s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED)
    s.step(3 * K + 2)
    assert np.array_equal(s.read(0), ref.read(0)) and np.array_equal(s.read(1), ref.read(1))
    s.close()
    ref.close()
