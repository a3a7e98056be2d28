"""Out-of-bounds writes: every kernel family on ragged small grids with the guard zones of all
device arrays armed (TSW_OPT_GUARD_CHECK fills them with 0xFF = NaN) — no guard byte may change,
and the results must be bitwise those of an unarmed run (a stray read of a guard would show)."""
import numpy as np
import pytest

from paper_2005_11931_b200 import inputs, tsw
from tests.helpers import NP

pytestmark = pytest.mark.gpu


def _run(make, nsteps, armed, diag=True):
    s = make()
    if armed:
        s.set_option(tsw.TSW_OPT_GUARD_CHECK, 1)
    s.prime()
    s.step(nsteps)
    out = [s.read(0), s.read(1)]
    if diag:
        out.append(s.energy())
    bad, checked = s.check_guards() if armed else (0, 0)
    s.close()
    return out, (bad, checked)


class _S:
    """A solver plus the set_initial call to make after arming."""

    def __init__(self, solver, init):
        self.s, self.init = solver, init

    def __getattr__(self, k):
        return getattr(self.s, k)

    def prime(self):
        self.init(self.s)


def _cases():
    out = []
    for dtype in ("f64", "f32"):
        npdt = NP[dtype]

        def point(kern, dtype=dtype, npdt=npdt):
            cfg = inputs.config(2, nx=203, ny=151, dx=0.01, dy=0.01, eps=[0.1, 0.2], amp=[1.0, 0.0], dt=3e-4)
            s = tsw.Solver.from_config(cfg, dtype)
            s.set_option(tsw.TSW_OPT_KERNEL, kern)
            return _S(s, lambda s: s.set_initial(cfg.initial().astype(npdt), None, cfg.dt, flags=tsw.TSW_INIT_SHARED))

        out += [(f"point-tma-{dtype}", lambda point=point: point(0), 9, True),
                (f"point-reg-{dtype}", lambda point=point: point(1), 9, True)]
        for K in (2, 4, 8):
            def tb(K=K, dtype=dtype, npdt=npdt):
                cfg = inputs.config(3, nx=701, ny=97, dx=0.01, dy=0.01, eps=[0.1, 0.3], amp=[1.0, 2.0], dt=2e-3)
                s = tsw.Solver.from_config(cfg, dtype)
                s.set_option(tsw.TSW_OPT_TBLOCK, K)
                s.set_option(tsw.TSW_OPT_ROWS_PER_ITEM, 20)
                u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny).astype(npdt)
                return _S(s, lambda s: s.set_initial(u0, None, cfg.dt, flags=tsw.TSW_INIT_SHARED))
            out.append((f"tb{K}-{dtype}", tb, 2 * K + 3, True))
        for solver in (0, 1):
            def imp(solver=solver, dtype=dtype, npdt=npdt):
                sc = inputs.paper_2d(dx=0.45)
                s = tsw.Solver(2, sc.nx, sc.ny, sc.dx, sc.dx, 1, dtype)
                s.set_coeff_profile(sc.seg_value, sc.seg_break, [0.8], isotropic=True)
                s.set_option(tsw.TSW_OPT_SCHEME, 1)
                s.set_option(tsw.TSW_OPT_IMPLICIT_SOLVER, solver)
                return _S(s, lambda s: s.set_initial(sc.initial()[None].astype(npdt), None, 0.05))
            out.append((f"implicit{solver}-{dtype}", imp, 4, False))

        def one_d(dtype=dtype, npdt=npdt):
            cfg = inputs.config(1, eps=[0.05, 0.2], amp=[1.0, 0.0])
            s = tsw.Solver.from_config(cfg, dtype)
            return _S(s, lambda s: s.set_initial(cfg.initial().astype(npdt), None, cfg.dt, flags=tsw.TSW_INIT_SHARED))
        out.append((f"1d-{dtype}", one_d, 40, True))
    return out


CASES = _cases()


@pytest.mark.parametrize("name,make,nsteps,diag", CASES, ids=[c[0] for c in CASES])
def test_no_out_of_bounds_writes(name, make, nsteps, diag):
    ref, _ = _run(make, nsteps, armed=False, diag=diag)
    got, (bad, checked) = _run(make, nsteps, armed=True, diag=diag)
    assert checked >= 2 * 16384 * 4, f"{name}: only {checked} guard bytes armed"   # fields + coefficients
    assert bad == 0, f"{name}: {bad} guard bytes overwritten"
    for a, b in zip(ref, got):
        assert np.array_equal(a, b), name


@pytest.mark.parametrize("K", [1, 4])
def test_blow_up_reported_unstable(K):
    """SURVEY §5 blow-up detection: above the leapfrog stability bound (TSW_ALLOW_UNSTABLE skips the
    R16 check) the discrete energy (R17) is not conserved — tsw_energy reports TSW_ERR_UNSTABLE once
    it drifts past 10^−k (TSW_OPT_ENERGY_DRIFT, default k = 2) and, with the drift check off, once it
    is no longer finite; below the bound the same run never raises."""
    cfg = inputs.config(3, nx=130, ny=90, dx=0.02, dy=0.02, eps=[0.2], amp=[1.0], dt=1e-3)
    u0 = inputs.uniform_dense_rows(cfg.nx, cfg.ny, 0, cfg.ny)

    def run(factor, drift):
        s = tsw.Solver.from_config(cfg, "f64")
        if K > 1:
            s.set_option(tsw.TSW_OPT_TBLOCK, K)
        s.set_option(tsw.TSW_OPT_ENERGY_DRIFT, drift)
        dt = factor * s.info()[2]
        s.set_initial(u0, None, dt, flags=tsw.TSW_INIT_SHARED | tsw.TSW_ALLOW_UNSTABLE)
        for it in range(200):
            s.step(8)
            try:
                s.energy()
            except tsw.TswError as e:
                assert e.status == tsw.TSW_ERR_UNSTABLE
                s.close()
                return it
        s.close()
        return None

    assert run(0.9, 2) is None                       # stable: conserved to round-off, never flagged
    first = run(1.5, 2)                              # the Gershgorin bound is sufficient, not sharp:
    assert first is not None                         # 1.5× is past the exact threshold here
    late = run(1.5, 0)                               # finiteness only: flagged when it overflows
    assert late is not None and late >= first
