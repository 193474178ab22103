"""ctypes binding of ``include/rexi_b200.h`` (the in-tree ``librexi_b200.so``).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, :func:`lib` / :class:`NativePlan` raise :class:`DeviceError`.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import DeviceError, SolverError

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "librexi_b200.so")

REXI_OK = 0
REXI_ERR_INVALID = 1
REXI_ERR_SINGULAR = 2
REXI_ERR_NOCONV = 3
REXI_ERR_BREAKDOWN = 4
REXI_ERR_CUDA = 5
REXI_ERR_NOMEM = 6
REXI_ERR_UNSUPPORTED = 7

SOLVER_AUTO, SOLVER_TRIDIAG, SOLVER_COCG, SOLVER_BAND = 0, 1, 2, 3
MEM_HOST, MEM_DEVICE = 0, 1
ABI_VERSION = 3

EXPORTED = (
    "rexi_plan_create", "rexi_plan_step", "rexi_plan_step_partial", "rexi_combine_partials",
    "rexi_plan_solve", "rexi_plan_info", "rexi_plan_destroy", "rexi_plan_last_error",
    "rexi_last_error", "rexi_device_count", "rexi_abi_version", "rexi_plan_profile",
    "rexi_plan_profile_report", "rexi_plan_run", "rexi_pencil_create", "rexi_pencil_solve_b",
    "rexi_pencil_spectral_radius", "rexi_pencil_cheb_step", "rexi_pencil_last_error",
    "rexi_pencil_destroy", "rexi_assemble_p1", "rexi_plan_wait_stream", "rexi_plan_shift_iters",
    "rexi_pencil_wait_stream",
)


class RexiDesc(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("n", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("indptr", ctypes.c_void_p),
        ("indices", ctypes.c_void_p),
        ("a_vals", ctypes.c_void_p),
        ("a_imag", ctypes.c_void_p),
        ("b_vals", ctypes.c_void_p),
        ("k", ctypes.c_int32),
        ("shifts", ctypes.c_void_p),
        ("weights", ctypes.c_void_p),
        ("shift_offset", ctypes.c_int32),
        ("tau", ctypes.c_double),
        ("device", ctypes.c_int32),
        ("solver", ctypes.c_int32),
        ("refine", ctypes.c_int32),
        ("tol", ctypes.c_double),
        ("max_iters", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("weight_ref", ctypes.c_double),
        ("shift_ids", ctypes.c_void_p),
    ]


class RexiP1Desc(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32), ("m", ctypes.c_int32), ("n_templates", ctypes.c_int32),
        ("n_off", ctypes.c_int32), ("offsets", ctypes.c_void_p), ("n_contrib", ctypes.c_int32),
        ("contrib_start", ctypes.c_void_p), ("contrib_t", ctypes.c_void_p),
        ("contrib_a", ctypes.c_void_p), ("contrib_b", ctypes.c_void_p),
        ("contrib_va", ctypes.c_void_p), ("contrib_stiff", ctypes.c_void_p),
        ("contrib_mass", ctypes.c_void_p), ("device", ctypes.c_int32), ("stream", ctypes.c_void_p),
    ]


class RexiStats(ctypes.Structure):
    _fields_ = [
        ("t_rhs_ms", ctypes.c_double),
        ("t_local_ms", ctypes.c_double),
        ("t_reduce_ms", ctypes.c_double),
        ("steps", ctypes.c_int64),
        ("launches", ctypes.c_int64),
        ("iters_max", ctypes.c_int32),
        ("iters_mean", ctypes.c_double),
        ("refine_rounds", ctypes.c_int32),
        ("bad_shift", ctypes.c_int32),
    ]


class RexiInfo(ctypes.Structure):
    _fields_ = [
        ("solver", ctypes.c_int32),
        ("bandwidth", ctypes.c_int32),
        ("k_pad", ctypes.c_int32),
        ("levels", ctypes.c_int32),
        ("refine", ctypes.c_int32),
        ("device_bytes", ctypes.c_int64),
        ("prepare_ms", ctypes.c_double),
        ("min_pivot_ratio", ctypes.c_double),
        ("persistent", ctypes.c_int32),
        ("screen_pivot_ratio", ctypes.c_double),
    ]


_lib = None


def lib():
    """Load the in-tree native library (raises DeviceError if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"native library {LIB_PATH} is missing; run __graft_entry__.build() "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp = ctypes.c_void_p
    L.rexi_plan_create.argtypes = [ctypes.POINTER(RexiDesc), ctypes.POINTER(vp)]
    L.rexi_plan_step.argtypes = [vp, vp, vp, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(RexiStats)]
    L.rexi_plan_step_partial.argtypes = [vp, vp, vp, ctypes.POINTER(RexiStats)]
    L.rexi_plan_run.argtypes = [vp, vp, vp, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(RexiStats)]
    L.rexi_combine_partials.argtypes = [vp, ctypes.c_int32, ctypes.c_int64, vp, vp]
    L.rexi_plan_solve.argtypes = [vp, vp, vp, ctypes.c_int32]
    L.rexi_plan_info.argtypes = [vp, ctypes.POINTER(RexiInfo)]
    L.rexi_plan_destroy.argtypes = [vp]
    L.rexi_plan_last_error.argtypes = [vp]
    L.rexi_plan_last_error.restype = ctypes.c_char_p
    L.rexi_last_error.restype = ctypes.c_char_p
    L.rexi_device_count.argtypes = [ctypes.POINTER(ctypes.c_int32)]
    L.rexi_abi_version.restype = ctypes.c_int32
    L.rexi_plan_profile.argtypes = [vp, ctypes.c_int32]
    L.rexi_plan_profile_report.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64]
    i32p = ctypes.POINTER(ctypes.c_int32)
    L.rexi_pencil_create.argtypes = [ctypes.POINTER(RexiDesc), ctypes.POINTER(vp)]
    L.rexi_pencil_solve_b.argtypes = [vp, vp, vp, ctypes.c_int32, i32p]
    L.rexi_pencil_spectral_radius.argtypes = [vp, vp, ctypes.c_double, ctypes.c_int32,
                                              ctypes.POINTER(ctypes.c_double), i32p, i32p]
    L.rexi_pencil_cheb_step.argtypes = [vp, vp, ctypes.c_int32, ctypes.c_double, vp, vp,
                                        ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(RexiStats)]
    L.rexi_pencil_last_error.argtypes = [vp]
    L.rexi_pencil_last_error.restype = ctypes.c_char_p
    L.rexi_pencil_destroy.argtypes = [vp]
    L.rexi_plan_wait_stream.argtypes = [vp, vp]
    L.rexi_plan_shift_iters.argtypes = [vp, i32p]
    L.rexi_pencil_wait_stream.argtypes = [vp, vp]
    L.rexi_assemble_p1.argtypes = [ctypes.POINTER(RexiP1Desc), vp, vp, vp, vp, vp]
    if L.rexi_abi_version() != ABI_VERSION:
        raise DeviceError("native library ABI version mismatch")
    _lib = L
    return L


def device_count() -> int:
    c = ctypes.c_int32(0)
    rc = lib().rexi_device_count(ctypes.byref(c))
    return int(c.value) if rc == 0 else 0


def host_empty(shape, dtype=np.complex128) -> np.ndarray:
    """Host output buffer in page-locked memory (torch's caching pinned-host
    allocator, so repeated steps reuse the block), so the device->host copy
    of a step result runs at full link speed; plain numpy if torch is absent."""
    try:
        import torch
        tdt = {np.dtype(np.complex128): torch.complex128, np.dtype(np.float64): torch.float64}[np.dtype(dtype)]
        return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
    except Exception:
        return np.empty(shape, dtype=dtype)


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


class NativeError(Exception):
    pass


def raise_status(rc: int, msg: str, shift_offset: int = 0):
    if rc == REXI_OK:
        return
    if rc in (REXI_ERR_INVALID, REXI_ERR_UNSUPPORTED):
        raise ValueError(msg)
    if rc in (REXI_ERR_SINGULAR, REXI_ERR_NOCONV, REXI_ERR_BREAKDOWN):
        raise SolverError(msg)
    raise DeviceError(msg)


class NativePlan:
    """Owns one ``rexi_plan`` (one device, one shard of shifts)."""

    def __init__(self, indptr, indices, a_vals, b_vals, shifts, weights, tau, *, a_imag=None,
                 device=0, solver=SOLVER_AUTO, refine=-1, tol=0.0, max_iters=0, shift_offset=0,
                 stream=None, weight_ref=0.0, shift_ids=None):
        L = lib()
        self._keep = [np.ascontiguousarray(indptr, dtype=np.int32),
                      np.ascontiguousarray(indices, dtype=np.int32),
                      np.ascontiguousarray(a_vals, dtype=np.float64),
                      np.ascontiguousarray(b_vals, dtype=np.float64),
                      np.ascontiguousarray(shifts, dtype=np.complex128),
                      np.ascontiguousarray(weights, dtype=np.complex128)]
        self._ids = None if shift_ids is None else np.ascontiguousarray(shift_ids, dtype=np.int32)
        if a_imag is not None:
            self._keep.append(np.ascontiguousarray(a_imag, dtype=np.float64))
        ip, ix, av, bv, sh, wt = self._keep[:6]
        d = RexiDesc()
        d.abi_version = ABI_VERSION
        d.n = len(ip) - 1
        d.nnz = len(ix)
        d.indptr = ip.ctypes.data
        d.indices = ix.ctypes.data
        d.a_vals = av.ctypes.data
        d.a_imag = self._keep[6].ctypes.data if a_imag is not None else None
        d.b_vals = bv.ctypes.data
        d.k = len(sh)
        d.shifts = sh.ctypes.data
        d.weights = wt.ctypes.data
        d.shift_offset = int(shift_offset)
        d.tau = float(tau)
        d.device = int(device)
        d.solver = int(solver)
        d.refine = int(refine)
        d.tol = float(tol)
        d.max_iters = int(max_iters)
        d.stream = stream
        d.weight_ref = float(weight_ref)
        d.shift_ids = self._ids.ctypes.data if self._ids is not None else None
        self.n = int(d.n)
        self.k = int(d.k)
        self.device = int(device)
        h = ctypes.c_void_p(None)
        rc = L.rexi_plan_create(ctypes.byref(d), ctypes.byref(h))
        if rc != REXI_OK:
            msg = L.rexi_last_error().decode()
            raise_status(rc, msg)
        self._h = h
        info = RexiInfo()
        L.rexi_plan_info(self._h, ctypes.byref(info))
        self.info = info

    def _err(self) -> str:
        return lib().rexi_plan_last_error(self._h).decode()

    def step_host(self, u: np.ndarray, n_steps: int = 1, stats: RexiStats | None = None) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.complex128)
        out = host_empty(u.shape)
        rc = lib().rexi_plan_step(self._h, _ptr(u), _ptr(out), int(n_steps), MEM_HOST,
                                  ctypes.byref(stats) if stats is not None else None)
        raise_status(rc, self._err())
        return out

    def step_device(self, u_ptr: int, out_ptr: int, n_steps: int = 1,
                    stats: RexiStats | None = None):
        rc = lib().rexi_plan_step(self._h, ctypes.c_void_p(u_ptr), ctypes.c_void_p(out_ptr),
                                  int(n_steps), MEM_DEVICE,
                                  ctypes.byref(stats) if stats is not None else None)
        raise_status(rc, self._err())

    def run_host(self, u: np.ndarray, n_steps: int, stats: RexiStats | None = None) -> np.ndarray:
        """States after each of n_steps steps, shape (n_steps, n) (fresh pinned buffer)."""
        u = np.ascontiguousarray(u, dtype=np.complex128)
        out = host_empty((int(n_steps), self.n))
        rc = lib().rexi_plan_run(self._h, _ptr(u), _ptr(out), int(n_steps), MEM_HOST,
                                 ctypes.byref(stats) if stats is not None else None)
        raise_status(rc, self._err())
        return out

    def wait_stream(self, stream_handle):
        """Order this plan's stream after the work queued on ``stream_handle``
        (a cudaStream_t as int, e.g. torch's current stream)."""
        rc = lib().rexi_plan_wait_stream(self._h, ctypes.c_void_p(stream_handle))
        raise_status(rc, self._err())

    def shift_iters(self) -> np.ndarray:
        """Per-shift COCG iterations of the last step (zeros for the direct solver)."""
        out = np.zeros(self.k, dtype=np.int32)
        rc = lib().rexi_plan_shift_iters(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        raise_status(rc, self._err())
        return out

    def step_partial(self, u_ptr: int, partial_ptr: int, stats: RexiStats | None = None):
        rc = lib().rexi_plan_step_partial(self._h, ctypes.c_void_p(u_ptr), ctypes.c_void_p(partial_ptr),
                                          ctypes.byref(stats) if stats is not None else None)
        raise_status(rc, self._err())

    def solve_host(self, rhs: np.ndarray) -> np.ndarray:
        rhs = np.ascontiguousarray(rhs, dtype=np.complex128)
        x = np.empty((self.k, self.n), dtype=np.complex128)
        rc = lib().rexi_plan_solve(self._h, _ptr(rhs), _ptr(x), MEM_HOST)
        raise_status(rc, self._err())
        return x

    def profile(self, enable: bool = True):
        """Per-kernel CUDA-event timing on the plan's stream (resets counters)."""
        raise_status(lib().rexi_plan_profile(self._h, 1 if enable else 0), self._err())

    def profile_report(self) -> dict:
        """{kernel: (launches, total_ms, algorithmic_bytes or 0)} since profile(True)."""
        buf = ctypes.create_string_buffer(1 << 16)
        raise_status(lib().rexi_plan_profile_report(self._h, buf, len(buf)), self._err())
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms, nbytes = line.split()
            out[name] = (int(cnt), float(ms), float(nbytes))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().rexi_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NativePencil:
    """Owns one ``rexi_pencil``: the pencil (A, B) on one device, for B-solves,
    the spectral-radius power iteration and Chebyshev stepping."""

    def __init__(self, indptr, indices, a_vals, b_vals, *, a_imag=None, device=0, tol=0.0,
                 max_iters=0, stream=None):
        L = lib()
        self._keep = [np.ascontiguousarray(indptr, dtype=np.int32),
                      np.ascontiguousarray(indices, dtype=np.int32),
                      np.ascontiguousarray(a_vals, dtype=np.float64),
                      np.ascontiguousarray(b_vals, dtype=np.float64)]
        if a_imag is not None:
            self._keep.append(np.ascontiguousarray(a_imag, dtype=np.float64))
        ip, ix, av, bv = self._keep[:4]
        d = RexiDesc()
        d.abi_version = ABI_VERSION
        d.n = len(ip) - 1
        d.nnz = len(ix)
        d.indptr = ip.ctypes.data
        d.indices = ix.ctypes.data
        d.a_vals = av.ctypes.data
        d.a_imag = self._keep[4].ctypes.data if a_imag is not None else None
        d.b_vals = bv.ctypes.data
        d.device = int(device)
        d.tol = float(tol)
        d.max_iters = int(max_iters)
        d.stream = stream
        self.n = int(d.n)
        self.device = int(device)
        h = ctypes.c_void_p(None)
        rc = L.rexi_pencil_create(ctypes.byref(d), ctypes.byref(h))
        if rc != REXI_OK:
            raise_status(rc, L.rexi_last_error().decode())
        self._h = h

    def _err(self) -> str:
        return lib().rexi_pencil_last_error(self._h).decode()

    def wait_stream(self, stream_handle):
        rc = lib().rexi_pencil_wait_stream(self._h, ctypes.c_void_p(stream_handle))
        raise_status(rc, self._err())

    def solve_b(self, rhs: np.ndarray):
        rhs = np.ascontiguousarray(rhs, dtype=np.complex128)
        x = np.empty_like(rhs)
        it = ctypes.c_int32(0)
        rc = lib().rexi_pencil_solve_b(self._h, _ptr(rhs), _ptr(x), MEM_HOST, ctypes.byref(it))
        raise_status(rc, self._err())
        return x, int(it.value)

    def spectral_radius(self, v0: np.ndarray, tol: float, max_iters: int):
        v0 = np.ascontiguousarray(v0, dtype=np.complex128)
        val = ctypes.c_double(0.0)
        it = ctypes.c_int32(0)
        conv = ctypes.c_int32(0)
        rc = lib().rexi_pencil_spectral_radius(self._h, _ptr(v0), float(tol), int(max_iters),
                                               ctypes.byref(val), ctypes.byref(it), ctypes.byref(conv))
        raise_status(rc, self._err())
        return float(val.value), int(it.value), bool(conv.value)

    def cheb_step(self, coeffs, scale: float, u_ptr, out_ptr, n_steps: int, mem: int,
                  stats: RexiStats | None = None):
        c = np.ascontiguousarray(coeffs, dtype=np.complex128)
        rc = lib().rexi_pencil_cheb_step(self._h, _ptr(c), len(c) - 1, float(scale),
                                         ctypes.c_void_p(u_ptr), ctypes.c_void_p(out_ptr),
                                         int(n_steps), int(mem),
                                         ctypes.byref(stats) if stats is not None else None)
        raise_status(rc, self._err())

    def cheb_step_host(self, coeffs, scale: float, u: np.ndarray, n_steps: int = 1,
                       stats: RexiStats | None = None) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.complex128)
        out = host_empty(u.shape)
        self.cheb_step(coeffs, scale, u.ctypes.data, out.ctypes.data, n_steps, MEM_HOST, stats)
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().rexi_pencil_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def combine_partials(partials_ptr: int, g: int, n: int, out_ptr: int, stream=None):
    rc = lib().rexi_combine_partials(ctypes.c_void_p(partials_ptr), int(g), int(n),
                                     ctypes.c_void_p(out_ptr), stream)
    raise_status(rc, lib().rexi_last_error().decode())
