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
