"""Seeded synthetic inputs and the five BASELINE.json configurations.

This module is shared by the CUDA path's callers (tests, bench) and by the
oracle's callers.  It holds NONE of the method's arithmetic: no mollifier, no
coefficient, no stencil, no energy.  It only says which grid, which ε family,
which dt and which initial data (u0, u1) a run uses, and generates that data.

Readings of the paper used here (DESIGN.md §3 lists them all):
  * R9  grid: "N×N grid" = N nodes per axis including the Dirichlet nodes, on a
        centred grid.  Node i sits at x_i = ((2i + 1 − nx)·dx)/2 (an exact
        integer times dx, halved), so x_s = 0 is a face when nx is even.
  * R14 data: the paper's Gaussians (§3.1 eq. (u0)
        "u_0(x)=40exp(-(x-40)^2/8)"; §3.3
        "u_0(x,y) = 50exp(-((x-40)^2+(y-50)^2)/8)") mapped by x -> (x-50)/10:
        1D  u0 = 40·exp(−(x+1)²/0.08),  2D  u0 = 50·exp(−((x+1)²+y²)/0.08);
        u1 = 0 ("we take u_1(x) ≡ 0").
  * R10 Dirichlet: boundary entries of every generated field are exactly +0.0.
  * R21 ε ladder of config 5: ε_k = 0.02·40^{k/63}, k = 0..63, plus one
        background member (amplitude 0).
  * Dense data-independence guard: uniform [−1, 1], seed 0.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np

# Coefficient kinds, numerically identical to tsw_hkind in include/tsw.h.
H_CONST = 0
H_DELTA_LINE_X = 1
H_DELTA_POINT = 2
H_FACES = 3


def node_coords(n: int, d: float, offset: int = 0, count: Optional[int] = None) -> np.ndarray:
    """Coordinates of nodes offset..offset+count-1 of an n-node centred axis."""
    if count is None:
        count = n - offset
    i = np.arange(offset, offset + count, dtype=np.int64)
    return ((2 * i + 1 - n).astype(np.float64) * d) / 2.0


def zero_boundary(u: np.ndarray, dim: int, row_offset: int = 0, ny_global: Optional[int] = None) -> np.ndarray:
    """Force Dirichlet entries (R10) to +0.0.  u is [..., rows, nx] (2D) or [..., nx] (1D)."""
    u[..., 0] = 0.0
    u[..., -1] = 0.0
    if dim == 2:
        rows = u.shape[-2]
        ny = ny_global if ny_global is not None else rows
        if row_offset == 0:
            u[..., 0, :] = 0.0
        if row_offset + rows == ny:
            u[..., rows - 1, :] = 0.0
    return u


def gaussian_1d(nx: int, dx: float, amp: float = 40.0, x0: float = -1.0, w: float = 0.08) -> np.ndarray:
    """R14: u0 = amp·exp(−(x−x0)²/w) on the centred grid, fp64, boundary zeroed."""
    x = node_coords(nx, dx)
    u = amp * np.exp(-((x - x0) ** 2) / w)
    return zero_boundary(u, 1)


def gaussian_2d(nx: int, ny: int, dx: float, dy: float, amp: float = 50.0, x0: float = -1.0,
                y0: float = 0.0, w: float = 0.08, row_offset: int = 0,
                rows: Optional[int] = None) -> np.ndarray:
    """R14: u0 = amp·exp(−((x−x0)²+(y−y0)²)/w); rows row_offset..row_offset+rows−1 of an ny-row grid."""
    if rows is None:
        rows = ny - row_offset
    x = node_coords(nx, dx)
    y = node_coords(ny, dy, row_offset, rows)
    u = amp * np.exp(-(((x[None, :] - x0) ** 2) + ((y[:, None] - y0) ** 2)) / w)
    return zero_boundary(u, 2, row_offset, ny)


def uniform_dense(shape: Sequence[int], seed: int = 0, dim: int = 2, row_offset: int = 0,
                  ny_global: Optional[int] = None) -> np.ndarray:
    """Dense guard data: uniform [−1, 1] with a counter-free seeded generator (numpy PCG64)."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1.0, 1.0, size=tuple(shape))
    return zero_boundary(u, dim, row_offset, ny_global)


def uniform_dense_rows(nx: int, ny: int, row_offset: int, rows: int, seed: int = 0) -> np.ndarray:
    """Rows [row_offset, row_offset+rows) of the dense field of an ny×nx grid.

    Row j is drawn from its own stream (seed, j) so any slab or window of the
    global field can be generated without generating the rest.
    """
    u = np.empty((rows, nx), dtype=np.float64)
    for k in range(rows):
        rng = np.random.default_rng([seed, row_offset + k])
        u[k] = rng.uniform(-1.0, 1.0, size=nx)
    return zero_boundary(u, 2, row_offset, ny)


def eps_ladder(k_count: int = 64, lo: float = 0.02, ratio: float = 40.0) -> List[float]:
    """R21: ε_k = lo·ratio^{k/(k_count−1)}, k = 0..k_count−1 (0.02 … 0.8, Fig. 3 range P:676)."""
    return [lo * ratio ** (k / (k_count - 1)) for k in range(k_count)]


@dataclasses.dataclass
class Config:
    """One BASELINE.json configuration, as concrete synthetic inputs."""
    name: str
    dim: int
    nx: int
    ny: int
    dx: float
    dy: float
    kind: int
    eps: List[float]
    amp: List[float]
    dt: float
    nsteps: int
    dtypes: List[str]
    h_background: float = 1.0
    order: int = 1
    xs: float = 0.0
    ys: float = 0.0
    data: str = "gaussian"   # or "dense"

    @property
    def batch(self) -> int:
        return len(self.eps)

    def initial(self, row_offset: int = 0, rows: Optional[int] = None, data: Optional[str] = None) -> np.ndarray:
        """u0 (fp64, boundary zeroed) for rows [row_offset, row_offset+rows) — shared by all members."""
        data = data or self.data
        if self.dim == 1:
            if data == "dense":
                return uniform_dense((self.nx,), dim=1)
            return gaussian_1d(self.nx, self.dx)
        if rows is None:
            rows = self.ny - row_offset
        if data == "dense":
            return uniform_dense_rows(self.nx, self.ny, row_offset, rows)
        return gaussian_2d(self.nx, self.ny, self.dx, self.dy, row_offset=row_offset, rows=rows)

    def interior_updates_per_step(self) -> int:
        if self.dim == 1:
            return (self.nx - 2) * self.batch
        return (self.nx - 2) * (self.ny - 2) * self.batch


def config(n: int, **over) -> Config:
    """BASELINE.json configs[n-1] (1-based as in SURVEY §8(d))."""
    if n == 1:
        c = Config("config1_1d_delta_point", 1, 2000, 1, 0.005, 0.005, H_DELTA_LINE_X,
                   [0.05], [1.0], 1.0e-3, 4000, ["f64", "f32"])
    elif n == 2:
        c = Config("config2_2d_delta_point_512", 2, 512, 512, 0.01, 0.01, H_DELTA_POINT,
                   [0.2, 0.1, 0.05, 0.05], [1.0, 1.0, 1.0, 0.0], 3.5e-4, 5000, ["f64"])
    elif n == 3:
        c = Config("config3_2d_delta_line_4096", 2, 4096, 4096, 0.0025, 0.0025, H_DELTA_LINE_X,
                   [0.05], [1.0], 4.0e-4, 5000, ["f32", "f64"])
    elif n == 4:
        c = Config("config4_2d_delta_line_32768", 2, 32768, 32768, 0.0025, 0.0025, H_DELTA_LINE_X,
                   [0.05], [1.0], 4.0e-4, 500, ["f32", "f64"])
    elif n == 5:
        eps = eps_ladder() + [0.02]
        amp = [1.0] * 64 + [0.0]
        c = Config("config5_batched_eps_family_2048", 2, 2048, 2048, 0.005, 0.005, H_DELTA_LINE_X,
                   eps, amp, 5.0e-4, 4000, ["f64", "f32"])
    else:
        raise ValueError(f"no config {n}")
    return dataclasses.replace(c, **over)


def weak_unit(nranks: int, rows_per_rank: int = 4096, nx: int = 32768) -> Config:
    """R22: config-4 weak-scaling unit — nx × rows_per_rank rows per GPU; P ranks ⇒ ny = rows_per_rank·P."""
    return config(4, name=f"config4_weak_{nx}x{rows_per_rank}_per_gpu", ny=rows_per_rank * nranks)


def slab_rows(ny: int, rank: int, nranks: int) -> tuple:
    """Row slab [r0, r1) owned by `rank` of `nranks`; remainder rows go to the first ranks."""
    if not (0 <= rank < nranks) or nranks < 1 or ny < nranks:
        raise ValueError("bad slab decomposition")
    base, rem = divmod(ny, nranks)
    r0 = rank * base + min(rank, rem)
    r1 = r0 + base + (1 if rank < rem else 0)
    return r0, r1


# ---------------------------------------------------------------------------------------------
# The paper's own scenarios, in the centred coordinates of R9: the paper's
# domain [0, 100] is x + 50 here, so its jump at 75 is at x = 25, its δ at 70 is at x = 20.
# ---------------------------------------------------------------------------------------------

@dataclasses.dataclass
class Scenario:
    """A depth profile + data of PAPER.md §3 (configuration only — no arithmetic of the method)."""
    name: str
    dim: int
    nx: int
    ny: int
    dx: float
    seg_value: List[float]
    seg_break: List[float]
    sing_loc: List[float]
    sing_amp: List[float]
    sing_order: List[int]
    isotropic: bool
    eps: List[float]
    scale: List[float]
    T: float
    data: str           # "gauss1d" | "lorentz" | "gauss2d"
    e: float = 0.0      # Lorentzian width

    @property
    def batch(self) -> int:
        return len(self.eps)

    def initial(self) -> np.ndarray:
        x = node_coords(self.nx, self.dx)
        if self.data == "gauss1d":      # P:809 u0 = 40 exp(−(x−40)²/8)  (x_paper = x + 50)
            return zero_boundary(40.0 * np.exp(-((x + 10.0) ** 2) / 8.0), 1)
        if self.data == "lorentz":      # P:1091 u0 = e/((x−60)² + e²)
            return zero_boundary(self.e / ((x - 10.0) ** 2 + self.e ** 2), 1)
        if self.data == "gauss2d":      # P:1156 u0 = 50 exp(−((x−40)² + (y−50)²)/8)
            y = node_coords(self.ny, self.dx)
            u = 50.0 * np.exp(-(((x[None, :] + 10.0) ** 2) + y[:, None] ** 2) / 8.0)
            return zero_boundary(u, 2)
        raise ValueError(self.data)


def paper_case(case: str, eps: float = 0.2, data: str = "gauss1d", e: float = 0.1, T: float = 5.0,
               dx: float = 0.005, amp: float = 1.0) -> Scenario:
    """PAPER.md §3.1 / §3.2.3, 1D on [0, 100] (dx = 0.005 as P:821 ⇒ 20001 nodes).

    case "1": h_0 = 100 on [0,75), 10 on [75,100] (eq. (h2case));
    case "2": h_0 + amp·δ(x−70) (amp = 100 is §3.2.3's singular type I);
    case "3": h_0 + amp·δ²(x−70) (amp = 100 is §3.2.3's singular type II).
    """
    nx = int(round(100.0 / dx)) + 1
    sing = {"1": ([], [], []), "2": ([20.0], [amp], [1]), "3": ([20.0], [amp], [2])}[case]
    return Scenario(f"paper_case{case}_{data}", 1, nx, 1, dx, [100.0, 10.0], [25.0], sing[0], sing[1], sing[2],
                    False, [eps], [1.0], T, data, e)


def paper_2d(eps: float = 0.8, dx: float = 0.05, T: float = 5.0) -> Scenario:
    """PAPER.md §3.3: H(x, y) = h_0(x) isotropic, Gaussian u0, ε = 0.8 (Fig. 6)."""
    n = int(round(100.0 / dx)) + 1
    return Scenario("paper_2d_H_h0", 2, n, n, dx, [100.0, 10.0], [25.0], [], [], [], True, [eps], [1.0], T,
                    "gauss2d")
