"""Test helpers: layout conversion and comparison (no arithmetic of the method here)."""
import os

import numpy as np


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def abi_faces(h1, h2, r0: int = 0, rows: int = None, ny: int = None):
    """Oracle faces (h1 [ny][nx−1], h2 [ny−1][nx]) → tsw_set_coeff_faces layout of one slab.

    h2 row k of the ABI layout is the face between global rows r0+k−1 and r0+k (oracle h2 row
    r0+k−1); rows outside the grid are filled with 1.0 (ignored by the library).
    """
    ny = h1.shape[0] if ny is None else ny
    rows = ny - r0 if rows is None else rows
    H1 = np.ascontiguousarray(h1[r0:r0 + rows])
    nx = h1.shape[1] + 1
    H2 = np.ones((rows + 1, nx))
    for k in range(rows + 1):
        g = r0 + k - 1
        if 0 <= g <= ny - 2:
            H2[k] = h2[g]
    return H1, H2


def rel_maxnorm(a, b) -> float:
    """R20: max|a − b| / max|b|."""
    den = float(np.max(np.abs(b)))
    return float(np.max(np.abs(np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)))) / (den if den > 0 else 1.0)


TOL = {"f64": 1e-12, "f32": 1e-5}     # BASELINE.json north_star relative max-norm
NP = {"f64": np.float64, "f32": np.float32}


def slab_record(p):
    """What the oracle check needs from one slab solver: rows, both levels, its own fp64 faces."""
    f1, f2 = p.read_faces()
    return {"r0": p.r0, "ny_local": p.ny_local, "un": p.read(0), "unm1": p.read(1), "h1": f1, "h2": f2}


def check_slabs_against_oracle(slabs, cfg, dtype, nsteps, u0):
    """Every slab's u^n and u^{n−1} against the CPU oracle's full-grid run (start-up + nsteps − 1
    leapfrog levels): bitwise with the faces the slabs built for themselves (global oracle layout
    assembled from them — h2 storage row k of a slab is the face between global rows r0+k−1 and
    r0+k; the per-node arithmetic is the canonical tree on both sides), and ≤ TOL end to end
    against the oracle's own faces.  `slabs`: solvers or slab_record dicts."""
    import oracle
    oracle.set_threads(host_cores())
    slabs = sorted([s if isinstance(s, dict) else slab_record(s) for s in slabs], key=lambda s: s["r0"])
    npdt = NP[dtype]
    B, nx = slabs[0]["un"].shape[0], slabs[0]["un"].shape[-1]
    ny = sum(s["ny_local"] for s in slabs)
    h1 = np.empty((B, ny, nx - 1))
    h2 = np.empty((B, ny - 1, nx))
    for s in slabs:
        h1[:, s["r0"]:s["r0"] + s["ny_local"]] = s["h1"]
        for k in range(s["ny_local"] + 1):
            g = s["r0"] + k - 1
            if 0 <= g <= ny - 2:
                h2[:, g] = s["h2"][:, k]
    u0 = np.asarray(u0)
    for b in range(B):
        ub = np.ascontiguousarray(u0[b] if u0.ndim == 3 else u0, dtype=npdt)
        c1 = oracle.prescale(h1[b], cfg.dt, cfg.dx, npdt)
        c2 = oracle.prescale(h2[b], cfg.dt, cfg.dy, npdt)
        un, unm1 = oracle.run(2, c1, c2, ub, None, cfg.dt, nsteps)
        for s in slabs:
            sl = slice(s["r0"], s["r0"] + s["ny_local"])
            assert np.array_equal(s["un"][b], un[sl]), f"member {b} slab r0={s['r0']}: u^n differs from the oracle"
            assert np.array_equal(s["unm1"][b], unm1[sl]), f"member {b} slab r0={s['r0']}: u^(n-1) differs"
        uo, _, _, _ = oracle.run_member(cfg, b, npdt, nsteps=nsteps, u0=ub)
        got = np.concatenate([s["un"][b] for s in slabs])
        assert rel_maxnorm(got, uo) <= TOL[dtype], f"member {b}: end to end vs the oracle's faces"
