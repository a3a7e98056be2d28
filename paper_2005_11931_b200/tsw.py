"""Python binding of include/tsw.h — the same names, argument marshalling only (ctypes).

Every step of the hot path runs inside libtsw.so (hand-written sm_100a CUDA).  There is no
CPU fallback: if libtsw.so is missing or there is no CUDA device, these calls raise.

Arrays: numpy arrays are host buffers (on_device = 0); objects with ``data_ptr()`` and
``is_cuda`` (torch CUDA tensors) are passed as device pointers (on_device = 1).  Field arrays
are [batch][ny_local][nx] (2D) or [batch][nx] (1D) in the ctx dtype.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libtsw.so")

TSW_OK, TSW_ERR_ARG, TSW_ERR_CFL, TSW_ERR_STATE, TSW_ERR_CUDA, TSW_ERR_NCCL, TSW_ERR_OOM, TSW_ERR_UNSTABLE = range(8)
TSW_F32, TSW_F64 = 0, 1
TSW_H_CONST, TSW_H_DELTA_LINE_X, TSW_H_DELTA_POINT, TSW_H_FACES, TSW_H_PROFILE_X = range(5)
TSW_ALLOW_UNSTABLE = 1
TSW_INIT_SHARED = 2
TSW_OPT_ROWS_PER_ITEM = 1
TSW_OPT_TIME_KERNELS = 2
TSW_OPT_KERNEL = 3
TSW_OPT_DEPTH = 4
TSW_OPT_GRAPHS = 5
TSW_OPT_TBLOCK = 6
TSW_OPT_TB_DEPTH = 7
TSW_OPT_SCHEME = 8
TSW_OPT_IMPLICIT_SOLVER = 9
TSW_OPT_GUARD_CHECK = 10
TSW_OPT_HALO = 11
TSW_OPT_IMPLICIT_XROWS = 12
TSW_OPT_TB_WARPS = 13
TSW_OPT_ENERGY_FUSE = 14
TSW_OPT_ENERGY_DRIFT = 15

STATUS_NAMES = {0: "TSW_OK", 1: "TSW_ERR_ARG", 2: "TSW_ERR_CFL", 3: "TSW_ERR_STATE", 4: "TSW_ERR_CUDA",
                5: "TSW_ERR_NCCL", 6: "TSW_ERR_OOM", 7: "TSW_ERR_UNSTABLE"}

# every symbol include/tsw.h declares (tests check the library exports all of them)
EXPORTS = ["tsw_create", "tsw_destroy", "tsw_set_coeff", "tsw_set_coeff_faces", "tsw_set_coeff_profile", "tsw_read_faces", "tsw_set_initial", "tsw_step",
           "tsw_group_step", "tsw_energy", "tsw_wave2", "tsw_read", "tsw_family_l2", "tsw_field_norms", "tsw_coeff_norms", "tsw_set_state", "tsw_info", "tsw_sync",
           "tsw_launch_count", "tsw_set_option", "tsw_kernel_stats", "tsw_kernel_launches", "tsw_alu_probe", "tsw_check_guards", "tsw_peer_export", "tsw_peer_import", "tsw_peer_attach", "tsw_peer_state", "tsw_step_op", "tsw_nccl_unique_id", "tsw_nccl_init", "tsw_last_error",
           "tsw_version"]


class TswError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class tsw_grid_desc(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("nx", ctypes.c_int64), ("ny", ctypes.c_int64),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("batch", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("device", ctypes.c_int32), ("stream", ctypes.c_void_p)]


class tsw_profile_desc(ctypes.Structure):
    _fields_ = [("nseg", ctypes.c_int32), ("seg_value", ctypes.POINTER(ctypes.c_double)),
                ("seg_break", ctypes.POINTER(ctypes.c_double)), ("nsing", ctypes.c_int32),
                ("sing_loc", ctypes.POINTER(ctypes.c_double)), ("sing_amp", ctypes.POINTER(ctypes.c_double)),
                ("sing_order", ctypes.POINTER(ctypes.c_int32)), ("isotropic", ctypes.c_int32)]


class tsw_coeff_desc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("order", ctypes.c_int32), ("h_background", ctypes.c_double),
                ("amp", ctypes.c_double), ("xs", ctypes.c_double), ("ys", ctypes.c_double),
                ("eps", ctypes.POINTER(ctypes.c_double)), ("amp_per_member", ctypes.POINTER(ctypes.c_double))]


_lib = None


def load(path: Optional[str] = None):
    """Load libtsw.so (raises if it has not been built — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("TSW_LIB") or LIB_PATH   # TSW_LIB: an alternative build (A/B timing)
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python paper_2005_11931_b200/build.py` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, i32, i64, d, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_uint32
    sig = {
        "tsw_create": (i32, [ctypes.POINTER(tsw_grid_desc), ctypes.POINTER(vp)]),
        "tsw_destroy": (None, [vp]),
        "tsw_set_coeff": (i32, [vp, ctypes.POINTER(tsw_coeff_desc)]),
        "tsw_set_coeff_faces": (i32, [vp, vp, vp, i32]),
        "tsw_set_coeff_profile": (i32, [vp, ctypes.POINTER(tsw_profile_desc), vp, vp]),
        "tsw_read_faces": (i32, [vp, vp, vp]),
        "tsw_set_initial": (i32, [vp, vp, vp, d, i32, u32]),
        "tsw_step": (i32, [vp, i64]),
        "tsw_group_step": (i32, [ctypes.POINTER(vp), i32, i64]),
        "tsw_energy": (i32, [vp, vp]),
        "tsw_wave2": (i32, [vp, i32, vp, vp]),
        "tsw_read": (i32, [vp, i32, vp, i32]),
        "tsw_family_l2": (i32, [vp, vp]),
        "tsw_field_norms": (i32, [vp, vp]),
        "tsw_coeff_norms": (i32, [vp, vp]),
        "tsw_set_state": (i32, [vp, vp, vp, i64, d, i32, u32]),
        "tsw_info": (i32, [vp, ctypes.POINTER(i64), ctypes.POINTER(d), ctypes.POINTER(d)]),
        "tsw_sync": (i32, [vp]),
        "tsw_launch_count": (i64, [vp]),
        "tsw_set_option": (i32, [vp, i32, i64]),
        "tsw_kernel_stats": (i32, [vp, ctypes.POINTER(d), ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "tsw_kernel_launches": (i32, [vp, i64, vp, vp, vp, ctypes.POINTER(i64)]),
        "tsw_alu_probe": (i32, [i32, i32, ctypes.POINTER(d)]),
        "tsw_check_guards": (i32, [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "tsw_nccl_unique_id": (i32, [vp]),
        "tsw_nccl_init": (i32, [vp, vp]),
        "tsw_peer_export": (i32, [vp, vp, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
        "tsw_peer_import": (i32, [vp, i32, vp, ctypes.c_size_t]),
        "tsw_peer_attach": (i32, [vp, i32, vp]),
        "tsw_peer_state": (i32, [vp, ctypes.POINTER(i64)]),
        "tsw_step_op": (i32, [vp, i64, ctypes.POINTER(i64)]),
        "tsw_last_error": (ctypes.c_char_p, [vp]),
        "tsw_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(st: int, ctx=None) -> None:
    if st != TSW_OK:
        raise TswError(st, load().tsw_last_error(ctx).decode())


def _ptr(a, dtype=None) -> Tuple[Optional[int], int, object]:
    """(pointer, on_device, keep-alive) of a numpy array or a CUDA tensor."""
    if a is None:
        return None, 0, None
    if hasattr(a, "data_ptr") and getattr(a, "is_cuda", False):
        if not a.is_contiguous():
            raise ValueError("device tensors must be contiguous")
        return a.data_ptr(), 1, a
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data, 0, arr


def _np_dtype(code: int):
    return np.float64 if code == TSW_F64 else np.float32


# ---- the ABI, same names ------------------------------------------------------------------

def tsw_version() -> str:
    return load().tsw_version().decode()


def tsw_last_error(ctx=None) -> str:
    return load().tsw_last_error(ctx).decode()


def tsw_create(dim: int, nx: int, ny: int, dx: float, dy: float, batch: int = 1, dtype: int = TSW_F64,
               rank: int = 0, nranks: int = 1, device: int = -1, stream: Optional[int] = None):
    g = tsw_grid_desc(dim, nx, ny, dx, dy, batch, dtype, rank, nranks, device, stream)
    out = ctypes.c_void_p()
    _check(load().tsw_create(ctypes.byref(g), ctypes.byref(out)))
    return out


def tsw_destroy(ctx) -> None:
    if ctx:
        load().tsw_destroy(ctx)


def tsw_set_coeff(ctx, kind: int, eps: Sequence[float], h_background: float = 1.0, amp: float = 1.0,
                  order: int = 1, xs: float = 0.0, ys: float = 0.0,
                  amp_per_member: Optional[Sequence[float]] = None) -> None:
    e = (ctypes.c_double * len(eps))(*eps)
    a = None if amp_per_member is None else (ctypes.c_double * len(amp_per_member))(*amp_per_member)
    desc = tsw_coeff_desc(kind, order, h_background, amp, xs, ys,
                          ctypes.cast(e, ctypes.POINTER(ctypes.c_double)),
                          None if a is None else ctypes.cast(a, ctypes.POINTER(ctypes.c_double)))
    _check(load().tsw_set_coeff(ctx, ctypes.byref(desc)), ctx)


def _dbl(vals):
    vals = list(vals)
    return (ctypes.c_double * max(1, len(vals)))(*vals)


def tsw_set_coeff_profile(ctx, seg_value: Sequence[float], seg_break: Sequence[float], eps: Sequence[float],
                          sing_loc: Sequence[float] = (), sing_amp: Sequence[float] = (),
                          sing_order: Sequence[int] = (), isotropic: bool = False,
                          scale: Optional[Sequence[float]] = None) -> None:
    sv, sb, sl, sa = _dbl(seg_value), _dbl(seg_break), _dbl(sing_loc), _dbl(sing_amp)
    so = (ctypes.c_int32 * max(1, len(sing_order)))(*list(sing_order))
    P = ctypes.POINTER(ctypes.c_double)
    desc = tsw_profile_desc(len(seg_value), ctypes.cast(sv, P), ctypes.cast(sb, P), len(sing_loc),
                            ctypes.cast(sl, P), ctypes.cast(sa, P), ctypes.cast(so, ctypes.POINTER(ctypes.c_int32)),
                            int(bool(isotropic)))
    e = _dbl(eps)
    sc = None if scale is None else _dbl(scale)
    _check(load().tsw_set_coeff_profile(ctx, ctypes.byref(desc), ctypes.cast(e, ctypes.c_void_p),
                                        None if sc is None else ctypes.cast(sc, ctypes.c_void_p)), ctx)


def tsw_set_coeff_faces(ctx, h1, h2=None) -> None:
    p1, d1, k1 = _ptr(h1, np.float64)
    p2, d2, k2 = _ptr(h2, np.float64)
    if h2 is not None and d1 != d2:
        raise ValueError("h1 and h2 must both be host or both be device arrays")
    _check(load().tsw_set_coeff_faces(ctx, p1, p2, d1), ctx)


def tsw_read_faces(ctx, h1_out: np.ndarray, h2_out: Optional[np.ndarray] = None) -> None:
    """Copy the fp64 faces into host arrays (tsw_set_coeff_faces layout)."""
    for a in (h1_out, h2_out):
        if a is not None and not (a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]):
            raise ValueError("face buffers must be C-contiguous float64")
    _check(load().tsw_read_faces(ctx, h1_out.ctypes.data, None if h2_out is None else h2_out.ctypes.data), ctx)


def tsw_set_initial(ctx, u0, u1=None, dt: float = 0.0, flags: int = 0, dtype=None) -> None:
    p0, d0, k0 = _ptr(u0, dtype)
    p1, d1, k1 = _ptr(u1, dtype)
    if u1 is not None and d0 != d1:
        raise ValueError("u0 and u1 must both be host or both be device arrays")
    _check(load().tsw_set_initial(ctx, p0, p1, dt, d0, flags), ctx)


def tsw_set_state(ctx, un, unm1, n: int, dt: float, flags: int = 0, dtype=None) -> None:
    pa, da, ka = _ptr(un, dtype)
    pb, db, kb = _ptr(unm1, dtype)
    _check(load().tsw_set_state(ctx, pa, pb, n, dt, da, flags), ctx)


def tsw_step(ctx, nsteps: int) -> None:
    _check(load().tsw_step(ctx, nsteps), ctx)


def tsw_group_step(ctxs: Sequence, nsteps: int) -> None:
    arr = (ctypes.c_void_p * len(ctxs))(*[c.value for c in ctxs])
    _check(load().tsw_group_step(arr, len(ctxs), nsteps))


def tsw_energy(ctx, batch: int) -> np.ndarray:
    out = np.zeros(batch, dtype=np.float64)
    _check(load().tsw_energy(ctx, out.ctypes.data), ctx)
    return out


def tsw_wave2(ctx, bg_member: int, batch: int) -> Tuple[np.ndarray, np.ndarray]:
    out = np.zeros((batch, 2), dtype=np.float64)
    idx = np.zeros((batch, 2), dtype=np.int64)
    _check(load().tsw_wave2(ctx, bg_member, out.ctypes.data, idx.ctypes.data), ctx)
    return out, idx


def tsw_family_l2(ctx, batch: int) -> np.ndarray:
    """[batch][batch] ‖u_i − u_j‖_{L²} at the current level."""
    out = np.zeros((batch, batch), dtype=np.float64)
    _check(load().tsw_family_l2(ctx, out.ctypes.data), ctx)
    return out


def tsw_field_norms(ctx, batch: int) -> np.ndarray:
    """[batch][4]: ‖u‖, ‖u_t‖, ‖∂x u‖, ‖∂y u‖ (L², Theorem lem 1 P:181–183)."""
    out = np.zeros((batch, 4), dtype=np.float64)
    _check(load().tsw_field_norms(ctx, out.ctypes.data), ctx)
    return out


def tsw_coeff_norms(ctx, batch: int) -> np.ndarray:
    """[batch][3]: sup|h1|, sup|∇h|, sup|h2| (W^{1,∞})."""
    out = np.zeros((batch, 3), dtype=np.float64)
    _check(load().tsw_coeff_norms(ctx, out.ctypes.data), ctx)
    return out


def tsw_read(ctx, which: int, out) -> object:
    """Copy u^n (which=0) or u^{n−1} (which=1) into `out` (numpy host array or CUDA tensor)."""
    if hasattr(out, "data_ptr") and getattr(out, "is_cuda", False):
        _check(load().tsw_read(ctx, which, out.data_ptr(), 1), ctx)
        return out
    if not (isinstance(out, np.ndarray) and out.flags["C_CONTIGUOUS"]):
        raise ValueError("out must be a C-contiguous numpy array or a CUDA tensor")
    _check(load().tsw_read(ctx, which, out.ctypes.data, 0), ctx)
    return out


def tsw_info(ctx) -> Tuple[int, float, float]:
    n, t, m = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    _check(load().tsw_info(ctx, ctypes.byref(n), ctypes.byref(t), ctypes.byref(m)), ctx)
    return n.value, t.value, m.value


def tsw_sync(ctx) -> None:
    _check(load().tsw_sync(ctx), ctx)


def tsw_launch_count(ctx) -> int:
    return int(load().tsw_launch_count(ctx))


def tsw_set_option(ctx, key: int, value: int) -> None:
    _check(load().tsw_set_option(ctx, key, value), ctx)


def tsw_kernel_stats(ctx) -> Tuple[float, int, int]:
    """(total stencil-kernel ms, launches, point-updates) since TSW_OPT_TIME_KERNELS was set."""
    ms, n, u = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
    _check(load().tsw_kernel_stats(ctx, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(u)), ctx)
    return ms.value, n.value, u.value


def tsw_kernel_launches(ctx):
    """Per timed launch: (ms [n], levels [n], point-updates [n]) numpy arrays."""
    n = ctypes.c_int64()
    _check(load().tsw_kernel_launches(ctx, 0, None, None, None, ctypes.byref(n)), ctx)
    ms = np.zeros(n.value, dtype=np.float64)
    lv = np.zeros(n.value, dtype=np.int32)
    up = np.zeros(n.value, dtype=np.int64)
    _check(load().tsw_kernel_launches(ctx, n.value, ms.ctypes.data, lv.ctypes.data, up.ctypes.data,
                                      ctypes.byref(n)), ctx)
    return ms, lv, up


def tsw_alu_probe(device: int, dtype: int) -> float:
    """Measured non-contracted add/multiply throughput of the device in dtype (operations/s)."""
    v = ctypes.c_double()
    _check(load().tsw_alu_probe(int(device), int(dtype), ctypes.byref(v)))
    return v.value


def tsw_check_guards(ctx) -> Tuple[int, int]:
    """(guard bytes changed since TSW_OPT_GUARD_CHECK filled them, guard bytes inspected)."""
    n, m = ctypes.c_int64(), ctypes.c_int64()
    _check(load().tsw_check_guards(ctx, ctypes.byref(n), ctypes.byref(m)), ctx)
    return n.value, m.value


def tsw_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().tsw_nccl_unique_id(buf))
    return buf.raw


def tsw_nccl_init(ctx, uid: bytes) -> None:
    buf = ctypes.create_string_buffer(uid, 128)
    _check(load().tsw_nccl_init(ctx, buf), ctx)


def tsw_peer_export(ctx) -> bytes:
    """Opaque blob with CUDA IPC handles of this ctx's field buffers and halo mailbox."""
    n = ctypes.c_size_t()
    _check(load().tsw_peer_export(ctx, None, 0, ctypes.byref(n)), ctx)
    buf = ctypes.create_string_buffer(n.value)
    _check(load().tsw_peer_export(ctx, buf, n.value, ctypes.byref(n)), ctx)
    return buf.raw[:n.value]


def tsw_peer_import(ctx, side: int, blob: bytes) -> None:
    """Map the neighbour on `side` (0: rank − 1, 1: rank + 1) from its tsw_peer_export blob."""
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(load().tsw_peer_import(ctx, side, buf, len(blob)), ctx)


def tsw_peer_state(ctx) -> Tuple[int, int, int, int]:
    """(halo epochs issued, mailbox from rank − 1, mailbox from rank + 1, wait-timeout word)."""
    out = (ctypes.c_int64 * 4)()
    _check(load().tsw_peer_state(ctx, out), ctx)
    return out[0], out[1], out[2], out[3]


def tsw_step_op(ctx, nsteps: int) -> int:
    """One peer-halo operation of the next `nsteps` levels; returns the levels it advanced."""
    n = ctypes.c_int64()
    _check(load().tsw_step_op(ctx, nsteps, ctypes.byref(n)), ctx)
    return n.value


def tsw_peer_attach(ctx, side: int, neighbour_ctx) -> None:
    """Map a neighbour ctx of this process directly."""
    _check(load().tsw_peer_attach(ctx, side, neighbour_ctx), ctx)


# ---- convenience wrapper ------------------------------------------------------------------

class Solver:
    """One tsw_ctx with its shape: a thin object over the same calls (no arithmetic here)."""

    def __init__(self, dim: int, nx: int, ny: int, dx: float, dy: float, batch: int = 1, dtype: str = "f64",
                 rank: int = 0, nranks: int = 1, device: int = -1, stream: Optional[int] = None):
        self.dim, self.nx, self.ny, self.batch = dim, nx, (ny if dim == 2 else 1), batch
        self.dtype_code = TSW_F64 if dtype in ("f64", "float64", np.float64) else TSW_F32
        self.np_dtype = _np_dtype(self.dtype_code)
        self.rank, self.nranks = rank, nranks
        if dim == 2:
            base, rem = divmod(ny, nranks)
            self.r0 = rank * base + min(rank, rem)
            self.ny_local = base + (1 if rank < rem else 0)
        else:
            self.r0, self.ny_local = 0, 1
        self.ctx = tsw_create(dim, nx, self.ny, dx, dy, batch, self.dtype_code, rank, nranks, device, stream)

    @classmethod
    def from_config(cls, cfg, dtype: str = "f64", rank: int = 0, nranks: int = 1, **kw) -> "Solver":
        s = cls(cfg.dim, cfg.nx, cfg.ny, cfg.dx, cfg.dy, cfg.batch, dtype, rank, nranks, **kw)
        s.set_coeff(cfg.kind, cfg.eps, cfg.h_background, 1.0, cfg.order, cfg.xs, cfg.ys, amp_per_member=cfg.amp)
        return s

    @property
    def field_shape(self):
        return (self.batch, self.nx) if self.dim == 1 else (self.batch, self.ny_local, self.nx)

    def close(self):
        if self.ctx:
            tsw_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_coeff(self, kind, eps, h_background=1.0, amp=1.0, order=1, xs=0.0, ys=0.0, amp_per_member=None):
        tsw_set_coeff(self.ctx, kind, list(eps), h_background, amp, order, xs, ys, amp_per_member)

    def set_coeff_profile(self, seg_value, seg_break, eps, sing_loc=(), sing_amp=(), sing_order=(),
                          isotropic=False, scale=None):
        tsw_set_coeff_profile(self.ctx, seg_value, seg_break, list(eps), sing_loc, sing_amp, sing_order,
                              isotropic, scale)

    def set_coeff_faces(self, h1, h2=None):
        tsw_set_coeff_faces(self.ctx, h1, h2)

    def read_faces(self):
        """(h1, h2) fp64 faces in the tsw_set_coeff_faces layout (h2 None in 1D)."""
        if self.dim == 1:
            h1 = np.empty((self.batch, self.nx - 1))
            tsw_read_faces(self.ctx, h1)
            return h1, None
        h1 = np.empty((self.batch, self.ny_local, self.nx - 1))
        h2 = np.empty((self.batch, self.ny_local + 1, self.nx))
        tsw_read_faces(self.ctx, h1, h2)
        return h1, h2

    def set_initial(self, u0, u1=None, dt=0.0, flags=0):
        tsw_set_initial(self.ctx, u0, u1, dt, flags, self.np_dtype)

    def set_state(self, un, unm1, n, dt, flags=0):
        tsw_set_state(self.ctx, un, unm1, n, dt, flags, self.np_dtype)

    def step(self, nsteps: int):
        tsw_step(self.ctx, nsteps)

    def energy(self) -> np.ndarray:
        return tsw_energy(self.ctx, self.batch)

    def wave2(self, bg_member: int):
        return tsw_wave2(self.ctx, bg_member, self.batch)

    def read(self, which: int = 0, out=None):
        if out is None:
            out = np.empty(self.field_shape, dtype=self.np_dtype)
        return tsw_read(self.ctx, which, out)

    def family_l2(self) -> np.ndarray:
        return tsw_family_l2(self.ctx, self.batch)

    def field_norms(self) -> np.ndarray:
        return tsw_field_norms(self.ctx, self.batch)

    def coeff_norms(self) -> np.ndarray:
        return tsw_coeff_norms(self.ctx, self.batch)

    def info(self):
        return tsw_info(self.ctx)

    def sync(self):
        tsw_sync(self.ctx)

    def launches(self) -> int:
        return tsw_launch_count(self.ctx)

    def set_option(self, key: int, value: int):
        tsw_set_option(self.ctx, key, value)

    def kernel_stats(self):
        return tsw_kernel_stats(self.ctx)

    def kernel_launches(self):
        return tsw_kernel_launches(self.ctx)

    def check_guards(self) -> Tuple[int, int]:
        return tsw_check_guards(self.ctx)

    def peer_export(self) -> bytes:
        return tsw_peer_export(self.ctx)

    def peer_import(self, side: int, blob: bytes) -> None:
        tsw_peer_import(self.ctx, side, blob)

    def peer_attach(self, side: int, neighbour: "Solver") -> None:
        tsw_peer_attach(self.ctx, side, neighbour.ctx)
