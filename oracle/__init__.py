"""CPU oracle for the leapfrog hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product package
(paper_2005_11931_b200) never imports it and shares no code with it: the
arithmetic lives in oracle/tsw_oracle.c (plain C, gcc -O2 -ffp-contract=off),
written from PAPER.md; this module only marshals numpy arrays through ctypes
and composes those C functions in the paper's order.

Every function states the passage it follows.  Pins: tests/test_oracle_pins.py.
Every function is pinned to something other than itself (tests/test_oracle_pins.py,
tests/test_scenarios_pins.py, tests/test_implicit_pins.py).  The second-wave amplitude (R18, our
definition: the paper prints no A₂ value) is pinned by brute force, by invariants and by two
closed forms — the impedance-mismatch reflection coefficient of a depth jump and the thin-layer
(Born) limit of the δ-line.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tsw_oracle.c")
_LIB_PATH = os.path.join(_HERE, "_build", "libtsw_oracle.so")
_lib = None

GCC_FLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=gnu11"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no contraction, no FTZ).  Returns the .so path."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", *GCC_FLAGS, "-o", _LIB_PATH, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB_PATH


def _L():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        d, i64, i32, vp = ctypes.c_double, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        lib.tswo_mollifier_c.restype = d
        lib.tswo_phi_eps.restype = d
        lib.tswo_phi_eps.argtypes = [d, d]
        lib.tswo_phi_eps_array.argtypes = [vp, i64, d, vp]
        lib.tswo_set_threads.argtypes = [i32]
        lib.tswo_max_threads.restype = i32
        lib.tswo_build_faces.argtypes = [i32, i32, i32, d, d, d, d, d, i64, i64, d, d, i64, i64, i64, i64, vp, vp]
        lib.tswo_mollifier_primitive.restype = d
        lib.tswo_mollifier_primitive.argtypes = [d]
        lib.tswo_profile_eval.restype = d
        lib.tswo_profile_eval.argtypes = [d, d, i32, vp, vp, i32, i32, vp, vp, vp, d]
        lib.tswo_build_faces_profile.argtypes = [i32, i32, vp, vp, i32, vp, vp, vp, d, i32, d, i64, i64, d,
                                                 i64, i64, i64, i64, vp, vp]
        lib.tswo_gershgorin_dt_max.restype = d
        lib.tswo_gershgorin_dt_max.argtypes = [i32, i64, i64, vp, vp, d, d]
        for s in ("f64", "f32"):
            getattr(lib, f"tswo_prescale_{s}").argtypes = [vp, i64, d, d, vp]
            getattr(lib, f"tswo_lap_{s}").argtypes = [i32, i64, i64, vp, vp, vp, vp]
            getattr(lib, f"tswo_startup_{s}").argtypes = [i32, i64, i64, vp, vp, vp, vp, d, vp]
            getattr(lib, f"tswo_leapfrog_{s}").argtypes = [i32, i64, i64, vp, vp, vp, vp, i64]
            f = getattr(lib, f"tswo_energy_{s}")
            f.restype = d
            f.argtypes = [i32, i64, i64, vp, vp, vp, vp, d, d, d]
            getattr(lib, f"tswo_wave2_{s}").argtypes = [i32, i64, i64, vp, vp, d, d, d, vp, vp]
            getattr(lib, f"tswo_implicit_solve_{s}").argtypes = [i32, i64, i64, vp, vp, vp, vp]
            getattr(lib, f"tswo_implicit_steps_{s}").argtypes = [i32, i64, i64, vp, vp, vp, vp, i64]
            getattr(lib, f"tswo_implicit_startup_{s}").argtypes = [i32, i64, i64, vp, vp, vp, vp, d, vp]
        _lib = lib
    return _lib


def _sfx(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return "f64"
    if dt == np.float32:
        return "f32"
    raise TypeError(f"oracle precision must be float32/float64, got {dt}")


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def set_threads(n: int) -> None:
    _L().tswo_set_threads(int(n))


def max_threads() -> int:
    return int(_L().tswo_max_threads())


# --- S0 / S1: mollifier and coefficient builder (§3.1, §2) -------

def mollifier_c() -> float:
    """The literal c of φ(x) = c·exp(1/(x²−1)) ("c ≃ 2.2523"; R4)."""
    return float(_L().tswo_mollifier_c())


def phi_eps(d, eps: float) -> np.ndarray:
    """φ_ε(d) = ε⁻¹ φ(d/ε), elementwise in fp64."""
    d = _c(np.atleast_1d(d), np.float64)
    out = np.empty_like(d)
    _L().tswo_phi_eps_array(_p(d), d.size, float(eps), _p(out))
    return out


def build_faces(dim: int, kind: int, order: int, hb: float, amp: float, xs: float, ys: float,
                eps: float, nx: int, ny: int, dx: float, dy: float, i0: int = 0, j0: int = 0,
                wnx: Optional[int] = None, wny: Optional[int] = None) -> Tuple[np.ndarray, Optional[np.ndarray]]:
    """fp64 regularised depth at the half-grid faces of a window (R2–R8).

    Returns h1 [wny][wnx−1] (x faces) and h2 [wny−1][wnx] (y faces; None in 1D).
    """
    wnx = nx - i0 if wnx is None else wnx
    if dim == 1:
        h1 = np.empty(wnx - 1, dtype=np.float64)
        _L().tswo_build_faces(1, kind, order, hb, amp, xs, ys, eps, nx, 1, dx, dy, i0, 0, wnx, 1, _p(h1), None)
        return h1, None
    wny = ny - j0 if wny is None else wny
    h1 = np.empty((wny, wnx - 1), dtype=np.float64)
    h2 = np.empty((wny - 1, wnx), dtype=np.float64)
    _L().tswo_build_faces(2, kind, order, hb, amp, xs, ys, eps, nx, ny, dx, dy, i0, j0, wnx, wny, _p(h1), _p(h2))
    return h1, h2


def mollifier_primitive(t) -> np.ndarray:
    """Φ(t) = ∫_{−1}^{t} φ (adaptive Simpson), elementwise."""
    t = np.atleast_1d(np.asarray(t, dtype=np.float64))
    return np.array([_L().tswo_mollifier_primitive(float(v)) for v in t.ravel()]).reshape(t.shape)


class Profile:
    """Piecewise-constant depth + singular terms (§3.1 Cases 1–3, §3.2.3; NEXT 1)."""

    def __init__(self, seg_value, seg_break=(), sing_loc=(), sing_amp=(), sing_order=(), isotropic=False):
        self.seg_value = np.ascontiguousarray(seg_value, dtype=np.float64)
        self.seg_break = np.ascontiguousarray(seg_break if len(seg_break) else [0.0], dtype=np.float64)
        self.nseg = len(seg_value)
        self.sing_loc = np.ascontiguousarray(sing_loc if len(sing_loc) else [0.0], dtype=np.float64)
        self.sing_amp = np.ascontiguousarray(sing_amp if len(sing_amp) else [0.0], dtype=np.float64)
        self.sing_order = np.ascontiguousarray(sing_order if len(sing_order) else [1], dtype=np.int32)
        self.nsing = len(sing_loc)
        self.isotropic = bool(isotropic)

    def eval(self, x, eps: float, with_sing: bool = True, sing_scale: float = 1.0) -> np.ndarray:
        """h_ε(x) = (h_0 * φ_ε)(x) + Σ A φ_ε(x − x_k)^{o_k}."""
        x = np.atleast_1d(np.asarray(x, dtype=np.float64))
        f = _L().tswo_profile_eval
        return np.array([f(float(v), eps, self.nseg, _p(self.seg_value), _p(self.seg_break), int(with_sing),
                           self.nsing, _p(self.sing_loc), _p(self.sing_amp), _p(self.sing_order), sing_scale)
                         for v in x.ravel()]).reshape(x.shape)


def build_faces_profile(dim: int, prof: "Profile", eps: float, nx: int, ny: int, dx: float, sing_scale: float = 1.0,
                        i0: int = 0, j0: int = 0, wnx: Optional[int] = None, wny: Optional[int] = None):
    """Faces of an x-only profile (h1 at x faces; h2 at y faces from node x_i)."""
    wnx = nx - i0 if wnx is None else wnx
    if dim == 1:
        h1 = np.empty(wnx - 1)
        _L().tswo_build_faces_profile(1, prof.nseg, _p(prof.seg_value), _p(prof.seg_break), prof.nsing,
                                      _p(prof.sing_loc), _p(prof.sing_amp), _p(prof.sing_order), sing_scale,
                                      int(prof.isotropic), eps, nx, 1, dx, i0, 0, wnx, 1, _p(h1), None)
        return h1, None
    wny = ny - j0 if wny is None else wny
    h1 = np.empty((wny, wnx - 1))
    h2 = np.empty((wny - 1, wnx))
    _L().tswo_build_faces_profile(2, prof.nseg, _p(prof.seg_value), _p(prof.seg_break), prof.nsing,
                                  _p(prof.sing_loc), _p(prof.sing_amp), _p(prof.sing_order), sing_scale,
                                  int(prof.isotropic), eps, nx, ny, dx, i0, j0, wnx, wny, _p(h1), _p(h2))
    return h1, h2


def gershgorin_dt_max(dim: int, h1: np.ndarray, h2: Optional[np.ndarray], dx: float, dy: float) -> float:
    """R16: 2/√ρ_G, ρ_G = max_node Σ_faces 2h/d² (sufficient leapfrog CFL bound)."""
    h1 = _c(h1, np.float64)
    if dim == 1:
        return float(_L().tswo_gershgorin_dt_max(1, h1.shape[-1] + 1, 1, _p(h1), None, dx, dy))
    h2 = _c(h2, np.float64)
    ny, nx = h1.shape[0], h1.shape[1] + 1
    return float(_L().tswo_gershgorin_dt_max(2, nx, ny, _p(h1), _p(h2), dx, dy))


def prescale(h: np.ndarray, dt: float, d: float, dtype) -> np.ndarray:
    """O3: c = fl_T((dt·dt)/(d·d) · h)."""
    h = _c(h, np.float64)
    c = np.empty(h.shape, dtype=dtype)
    getattr(_L(), f"tswo_prescale_{_sfx(dtype)}")(_p(h), h.size, dt, d, _p(c))
    return c


# --- S2 / S3: the stepper (north_star leapfrog; R1, R10, R11, R19) ---------------------------

def _shape(dim, u):
    if dim == 1:
        return u.shape[-1], 1
    return u.shape[-1], u.shape[-2]


def lap(dim: int, c1: np.ndarray, c2: Optional[np.ndarray], u: np.ndarray) -> np.ndarray:
    """O5: L(u) at interior nodes (0 on the ring), canonical contraction-free tree."""
    dtype = u.dtype
    u, c1 = _c(u, dtype), _c(c1, dtype)
    c2 = None if dim == 1 else _c(c2, dtype)
    nx, ny = _shape(dim, u)
    out = np.empty_like(u)
    getattr(_L(), f"tswo_lap_{_sfx(dtype)}")(dim, nx, ny, _p(c1), _p(c2), _p(u), _p(out))
    return out


def startup(dim: int, c1, c2, u0: np.ndarray, u1: Optional[np.ndarray], dt: float) -> np.ndarray:
    """O4 / R11: u¹ = (u⁰ + fl(dt·u₁)) + fl(½·L(u⁰))."""
    dtype = u0.dtype
    u0, c1 = _c(u0, dtype), _c(c1, dtype)
    c2 = None if dim == 1 else _c(c2, dtype)
    u1 = None if u1 is None else _c(u1, dtype)
    nx, ny = _shape(dim, u0)
    out = np.empty_like(u0)
    getattr(_L(), f"tswo_startup_{_sfx(dtype)}")(dim, nx, ny, _p(c1), _p(c2), _p(u0), _p(u1), dt, _p(out))
    return out


def leapfrog(dim: int, c1, c2, un: np.ndarray, unm1: np.ndarray, k: int) -> Tuple[np.ndarray, np.ndarray]:
    """O5: k steps of u^{n+1} = (2u^n − u^{n−1}) + L(u^n).  Returns (u^{n+k}, u^{n+k−1})."""
    dtype = un.dtype
    un, unm1 = _c(un, dtype).copy(), _c(unm1, dtype).copy()
    c1 = _c(c1, dtype)
    c2 = None if dim == 1 else _c(c2, dtype)
    nx, ny = _shape(dim, un)
    getattr(_L(), f"tswo_leapfrog_{_sfx(dtype)}")(dim, nx, ny, _p(c1), _p(c2), _p(un), _p(unm1), int(k))
    return un, unm1


def run(dim: int, c1, c2, u0: np.ndarray, u1: Optional[np.ndarray], dt: float, nsteps: int):
    """Start-up then nsteps−1 leapfrog steps: returns (u^N, u^{N−1}) at t = N·dt (R12)."""
    if nsteps < 1:
        raise ValueError("nsteps >= 1")
    v1 = startup(dim, c1, c2, u0, u1, dt)
    return leapfrog(dim, c1, c2, v1, u0, nsteps - 1)


# --- S5 / S6: diagnostics -------------------------------------------------------------------

def energy(dim: int, c1, c2, unp1: np.ndarray, un: np.ndarray, dx: float, dy: float, dt: float) -> float:
    """O6 / R17: E^{n+1/2} with the stepper's own rounded coefficients (discrete CL-01)."""
    dtype = un.dtype
    unp1, un, c1 = _c(unp1, dtype), _c(un, dtype), _c(c1, dtype)
    c2 = None if dim == 1 else _c(c2, dtype)
    nx, ny = _shape(dim, un)
    return float(getattr(_L(), f"tswo_energy_{_sfx(dtype)}")(dim, nx, ny, _p(c1), _p(c2), _p(unp1), _p(un), dx, dy, dt))


def wave2(dim: int, u: np.ndarray, ubg: np.ndarray, dx: float, xs: float, eps: float):
    """O7 / R18: (A₂⁺, A₂⁻) and their row-major indices over {x_i ≤ xs − ε} (pins: brute force,
    A = 0 ⇒ 0, Born linearity, impedance-mismatch and thin-layer closed forms)."""
    dtype = u.dtype
    u, ubg = _c(u, dtype), _c(ubg, dtype)
    nx, ny = _shape(dim, u)
    out = np.zeros(2, dtype=np.float64)
    idx = np.zeros(2, dtype=np.int64)
    getattr(_L(), f"tswo_wave2_{_sfx(dtype)}")(dim, nx, ny, _p(u), _p(ubg), dx, xs, eps, _p(out), _p(idx))
    return out, idx


# --- composition for one configuration member ------------------------------------------------

def member_coefficients(cfg, member: int, dtype, i0: int = 0, j0: int = 0,
                        wnx: Optional[int] = None, wny: Optional[int] = None):
    """(h1, h2, c1, c2) for member b of a config (window optional) — S1 then O3."""
    h1, h2 = build_faces(cfg.dim, cfg.kind, cfg.order, cfg.h_background, cfg.amp[member], cfg.xs, cfg.ys,
                         cfg.eps[member], cfg.nx, cfg.ny, cfg.dx, cfg.dy, i0, j0, wnx, wny)
    c1 = prescale(h1, cfg.dt, cfg.dx, dtype)
    c2 = None if cfg.dim == 1 else prescale(h2, cfg.dt, cfg.dy, dtype)
    return h1, h2, c1, c2


def run_member(cfg, member: int, dtype, nsteps: Optional[int] = None, u0: Optional[np.ndarray] = None):
    """Oracle run of one member on the full grid: returns (u^N, u^{N−1}, c1, c2)."""
    nsteps = cfg.nsteps if nsteps is None else nsteps
    _, _, c1, c2 = member_coefficients(cfg, member, dtype)
    if u0 is None:
        u0 = cfg.initial()
    u0 = np.ascontiguousarray(u0, dtype=dtype)
    un, unm1 = run(cfg.dim, c1, c2, u0, None, cfg.dt, nsteps)
    return un, unm1, c1, c2


def window_value(cfg, member: int, dtype, nsteps: int, samples: Sequence[Tuple[int, int]], u0_rows) -> np.ndarray:
    """u^N at sampled global nodes (j, i) of a full-size run, each from its own light-cone window.

    The window has half-width nsteps+1 (clipped to the grid): the scheme moves
    information one node per step, so the fixed window edge cannot reach the
    centre (SURVEY §8(c) "exact lattice speed").  u0_rows(j0, rows, i0, cols)
    returns that block of the initial field.
    """
    out = np.empty(len(samples), dtype=dtype)
    R = nsteps + 1
    for k, (j, i) in enumerate(samples):
        i0, i1 = max(0, i - R), min(cfg.nx, i + R + 1)
        j0, j1 = max(0, j - R), min(cfg.ny, j + R + 1)
        _, _, c1, c2 = member_coefficients(cfg, member, dtype, i0, j0, i1 - i0, j1 - j0)
        u0 = np.ascontiguousarray(u0_rows(j0, j1 - j0, i0, i1 - i0), dtype=dtype)
        un, _ = run(2, c1, c2, u0, None, cfg.dt, nsteps)
        out[k] = un[j - j0, i - i0]
    return out


# --- NEXT 2: ε-family diagnostics (definitions written out, numpy fp64) ------------------------

def family_l2(U: np.ndarray, w: float) -> np.ndarray:
    """‖u_i − u_j‖_{L²} = sqrt(w·Σ (u_i − u_j)²) for every pair of members."""
    U = np.asarray(U, dtype=np.float64).reshape(U.shape[0], -1)
    B = U.shape[0]
    D = np.zeros((B, B))
    for i in range(B):
        for j in range(i + 1, B):
            D[i, j] = D[j, i] = np.sqrt(w * np.sum((U[i] - U[j]) ** 2))
    return D


def field_norms(dim: int, un: np.ndarray, unm1: np.ndarray, dx: float, dy: float, dt: float) -> np.ndarray:
    """Theorem lem 1's L² quantities: ‖u‖, ‖(u^n − u^{n−1})/dt‖, ‖∂x u‖, ‖∂y u‖
    (forward differences over all faces, rectangle rule)."""
    u = np.asarray(un, dtype=np.float64)
    p = np.asarray(unm1, dtype=np.float64)
    w = dx if dim == 1 else dx * dy
    out = [np.sqrt(w * np.sum(u * u)), np.sqrt(w * np.sum((u - p) ** 2)) / dt,
           np.sqrt(w * np.sum(np.diff(u, axis=-1) ** 2)) / dx]
    out.append(np.sqrt(w * np.sum(np.diff(u, axis=0) ** 2)) / dy if dim == 2 else 0.0)
    return np.array(out)


def dphi_eps(d, eps: float) -> np.ndarray:
    """φ_ε′(d) = φ_ε(d)·(−2t/((t²−1)²·ε)), t = d/ε (derivative of P:745–750's φ_ε)."""
    d = np.atleast_1d(np.asarray(d, dtype=np.float64))
    t = d / eps
    out = np.zeros_like(d)
    m = np.abs(t) < 1.0
    out[m] = phi_eps(d[m], eps) * (-2.0 * t[m] / ((t[m] ** 2 - 1.0) ** 2 * eps))
    return out


def profile_derivative(prof: "Profile", x, eps: float, sing_scale: float = 1.0) -> np.ndarray:
    """h_ε′(x) = Σ_k (v_k − v_{k−1}) φ_ε(x − b_k) + Σ_j s·A_j·(φ_ε^{o_j})′(x − x_j)  (Φ′ = φ)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    d = np.zeros_like(x)
    for k in range(1, prof.nseg):
        d += (prof.seg_value[k] - prof.seg_value[k - 1]) * phi_eps(x - prof.seg_break[k - 1], eps)
    for j in range(prof.nsing):
        p, q = phi_eps(x - prof.sing_loc[j], eps), dphi_eps(x - prof.sing_loc[j], eps)
        d += sing_scale * prof.sing_amp[j] * (2.0 * p * q if prof.sing_order[j] == 2 else q)
    return d


def moderateness_exponent(eps_list, norms) -> float:
    """Least-squares slope N of log‖h_ε‖_{W^{1,∞}} against log(1/ε) (Assumption)."""
    x = np.log(1.0 / np.asarray(eps_list, dtype=np.float64))
    y = np.log(np.asarray(norms, dtype=np.float64))
    return float(np.polyfit(x, y, 1)[0])


# --- NEXT 3: the paper's implicit 2D method (R26/R27; §3.3, Table 1) ---

def implicit_solve(dim: int, c1, c2, r: np.ndarray) -> np.ndarray:
    """s = B⁻¹r, B = (I − ½L_x)(I − ½L_y), Thomas line solves (rows, then columns); ring → 0."""
    dtype = r.dtype
    r, c1 = _c(r, dtype), _c(c1, dtype)
    c2 = None if dim == 1 else _c(c2, dtype)
    nx, ny = _shape(dim, r)
    out = np.empty_like(r)
    getattr(_L(), f"tswo_implicit_solve_{_sfx(dtype)}")(dim, nx, ny, _p(c1), _p(c2), _p(r), _p(out))
    return out


def implicit_run(dim: int, c1, c2, u0: np.ndarray, u1: Optional[np.ndarray], dt: float, nsteps: int):
    """R27 start u¹ = B⁻¹u⁰ + fl(dt·u₁), then u^{n+1} = B⁻¹(2u^n) − u^{n−1}: returns (u^N, u^{N−1})."""
    dtype = u0.dtype
    u0, c1 = _c(u0, dtype), _c(c1, dtype)
    c2 = None if dim == 1 else _c(c2, dtype)
    u1 = None if u1 is None else _c(u1, dtype)
    nx, ny = _shape(dim, u0)
    v = np.empty_like(u0)
    L = _L()
    getattr(L, f"tswo_implicit_startup_{_sfx(dtype)}")(dim, nx, ny, _p(c1), _p(c2), _p(u0), _p(u1), dt, _p(v))
    un, unm1 = v.copy(), u0.copy()
    getattr(L, f"tswo_implicit_steps_{_sfx(dtype)}")(dim, nx, ny, _p(c1), _p(c2), _p(un), _p(unm1), int(nsteps - 1))
    return un, unm1
