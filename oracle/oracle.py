"""ctypes front-end of the CPU oracle.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and
only as the checker or the timed CPU baseline.  The product package
``paper_1912_03312_b200`` never imports it.

``OraclePlan`` restates the reference path (see ``rexi_oracle.c`` for the
file:line map): banded LU with partial pivoting per shift
(``solvers.py:42-80``), ``rhs = 1j*(B@u)`` (``integrate.py:203-206``),
``fl(beta_j*x_j)`` terms and an ascending-j Kahan sum
(``integrate.py:59-68,208-226``).  ``mode="truth"`` refines every shift
against a double-double residual and sums exactly.
``cocg_step`` is the CPU restatement used where the reference cannot run
(2D/3D: its dense-LU fallback, ``solvers.py:108-115``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or any(
            os.path.getmtime(os.path.join(HERE, f)) > os.path.getmtime(LIB_PATH)
            for f in ("rexi_oracle.c", "cocg_oracle.c")):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        p = ctypes.c_void_p
        L.orc_create.restype = p
        L.orc_create.argtypes = [ctypes.c_int64, ctypes.c_int64, p, p, p, p, ctypes.c_int32,
                                 p, p, ctypes.c_double, ctypes.c_int32, p]
        L.orc_destroy.argtypes = [p]
        L.orc_step.argtypes = [p, p, p, ctypes.c_int32, p, p]
        L.orc_step.restype = ctypes.c_int
        L.orc_solve.argtypes = [p, ctypes.c_int32, p, p]
        L.orc_rel_residual.argtypes = [p, ctypes.c_int32, p, p]
        L.orc_rel_residual.restype = ctypes.c_double
        L.orc_bad_shift.argtypes = [p]
        L.orc_bad_shift.restype = ctypes.c_int32
        L.orc_bandwidth.argtypes = [p]
        L.orc_bandwidth.restype = ctypes.c_int32
        L.orc_rhs.argtypes = [p, p, p]
        L.orc_screen.argtypes = [p, p, p, p]
        L.orc_cocg_step.restype = ctypes.c_int
        L.orc_cocg_truth_step.restype = ctypes.c_int
        L.orc_cocg_truth_step.argtypes = [ctypes.c_int64, p, p, p, p, ctypes.c_int32, p, p,
                                          ctypes.c_double, p, p, ctypes.c_double, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_double, ctypes.c_int32, p, p, p]
        L.orc_csr_rel_residual.restype = ctypes.c_double
        L.orc_csr_rel_residual.argtypes = [ctypes.c_int64, p, p, p, p, ctypes.c_double,
                                           ctypes.c_double * 2, p, p, ctypes.c_int32]
        L.orc_cocg_step.argtypes = [ctypes.c_int64, p, p, p, p, ctypes.c_int32, p, p,
                                    ctypes.c_double, p, p, ctypes.c_double, ctypes.c_int32,
                                    ctypes.c_int32, ctypes.c_double, ctypes.c_int32, p]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def union_pattern(A, B):
    """Shared CSR pattern of A and B plus both value arrays on it."""
    A = A.tocsr()
    B = B.tocsr()
    P = (abs(A) + abs(B)).tocsr()
    P.sort_indices()
    n = P.shape[0]
    rows = np.repeat(np.arange(n), np.diff(P.indptr))
    key = rows.astype(np.int64) * n + P.indices

    def vals(M):
        M = M.tocoo()
        mk = M.row.astype(np.int64) * n + M.col
        out = np.zeros(len(key))
        pos = np.searchsorted(key, mk)
        np.add.at(out, pos, M.data.real if np.iscomplexobj(M.data) else M.data)
        return out
    return (P.indptr.astype(np.int32), P.indices.astype(np.int32), vals(A), vals(B))


class OraclePlan:
    """Factor-once / solve-many CPU restatement of ``rexi_prepare``."""

    def __init__(self, sysm, approx, tau, nthreads=0):
        L = lib()
        self.indptr, self.indices, self.a, self.b = union_pattern(sysm.A, sysm.B)
        self.n = int(sysm.n_dof)
        self.k = int(len(approx.shifts))
        self.shifts = np.ascontiguousarray(approx.shifts, dtype=np.complex128)
        self.weights = np.ascontiguousarray(approx.weights, dtype=np.complex128)
        self.tau = float(tau)
        st = ctypes.c_int32(0)
        self._p = L.orc_create(self.n, len(self.indices), _ptr(self.indptr), _ptr(self.indices),
                               _ptr(self.a), _ptr(self.b), self.k, _ptr(self.shifts),
                               _ptr(self.weights), self.tau, int(nthreads), ctypes.byref(st))
        self.status = st.value
        self.bad_shift = L.orc_bad_shift(self._p)
        self.bandwidth = L.orc_bandwidth(self._p)

    def close(self):
        if self._p:
            lib().orc_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, u, mode="reference", return_solutions=False):
        u = np.ascontiguousarray(u, dtype=np.complex128)
        out = np.empty(self.n, dtype=np.complex128)
        xs = np.empty((self.k, self.n), dtype=np.complex128) if return_solutions else None
        corr = ctypes.c_double(0.0)
        lib().orc_step(self._p, _ptr(u), _ptr(out), 1 if mode == "truth" else 0,
                       _ptr(xs) if xs is not None else None, ctypes.byref(corr))
        self.last_correction = corr.value
        return (out, xs) if return_solutions else out

    def run(self, u0, n_steps, mode="reference"):
        u = np.array(u0, dtype=np.complex128, copy=True)
        hist = []
        for _ in range(n_steps):
            u = self.step(u, mode)
            hist.append(u)
        return hist

    def rhs(self, u):
        u = np.ascontiguousarray(u, dtype=np.complex128)
        out = np.empty(self.n, dtype=np.complex128)
        lib().orc_rhs(self._p, _ptr(u), _ptr(out))
        return out

    def solve(self, j, b):
        b = np.ascontiguousarray(b, dtype=np.complex128)
        x = np.empty(self.n, dtype=np.complex128)
        lib().orc_solve(self._p, int(j), _ptr(b), _ptr(x))
        return x

    def screen(self):
        """Per shift (min|U_ii|, max|U_ii|, info) of the partially pivoted band
        LU -- the data of the reference's singularity screen (solvers.py:52-69)."""
        umin = np.zeros(self.k)
        umax = np.zeros(self.k)
        info = np.zeros(self.k, dtype=np.int32)
        lib().orc_screen(self._p, _ptr(umin), _ptr(umax), _ptr(info))
        return umin, umax, info

    def rel_residual(self, j, rhs, x):
        rhs = np.ascontiguousarray(rhs, dtype=np.complex128)
        x = np.ascontiguousarray(x, dtype=np.complex128)
        return lib().orc_rel_residual(self._p, int(j), _ptr(rhs), _ptr(x))


def cocg_step(sysm, approx, tau, u, tol=1e-12, maxit=20000, refine=1, tol_refine=1e-8,
              nthreads=0, pattern=None):
    """CPU Jacobi-COCG restatement of one REXI step; returns (u1, iterations[K])."""
    indptr, indices, a, b = pattern if pattern is not None else union_pattern(sysm.A, sysm.B)
    shifts = np.ascontiguousarray(approx.shifts, dtype=np.complex128)
    weights = np.ascontiguousarray(approx.weights, dtype=np.complex128)
    u = np.ascontiguousarray(u, dtype=np.complex128)
    out = np.empty_like(u)
    iters = np.zeros(len(shifts), dtype=np.int32)
    rc = lib().orc_cocg_step(len(u), _ptr(indptr), _ptr(indices), _ptr(a), _ptr(b), len(shifts),
                             _ptr(shifts), _ptr(weights), float(tau), _ptr(u), _ptr(out),
                             float(tol), int(maxit), int(refine), float(tol_refine),
                             int(nthreads), _ptr(iters))
    if rc:
        raise RuntimeError(f"oracle COCG failed for shift j = {rc - 10}")
    return out, iters


def cocg_truth_step(sysm, approx, tau, u, tol=1e-12, maxit=40000, rounds=6, tol_refine=1e-8,
                    nthreads=0, pattern=None, return_solutions=False):
    """Truth-level CPU step for any CSR pencil (2D/3D, where the banded truth
    of ``OraclePlan`` does not fit): per-shift Jacobi-COCG, double-double
    residual refinement with x kept in double-double, exact-product
    double-double sum (``cocg_oracle.c: orc_cocg_truth_step``).
    Returns (u1, iterations[K], last relative correction[K]) and the fp64
    per-shift solutions when ``return_solutions``."""
    indptr, indices, a, b = pattern if pattern is not None else union_pattern(sysm.A, sysm.B)
    shifts = np.ascontiguousarray(approx.shifts, dtype=np.complex128)
    weights = np.ascontiguousarray(approx.weights, dtype=np.complex128)
    u = np.ascontiguousarray(u, dtype=np.complex128)
    out = np.empty_like(u)
    k = len(shifts)
    iters = np.zeros(k, dtype=np.int32)
    corr = np.zeros(k, dtype=np.float64)
    xs = np.empty((k, len(u)), dtype=np.complex128) if return_solutions else None
    rc = lib().orc_cocg_truth_step(len(u), _ptr(indptr), _ptr(indices), _ptr(a), _ptr(b), k,
                                   _ptr(shifts), _ptr(weights), float(tau), _ptr(u), _ptr(out),
                                   float(tol), int(maxit), int(rounds), float(tol_refine),
                                   int(nthreads), _ptr(iters), _ptr(corr),
                                   _ptr(xs) if xs is not None else None)
    if rc:
        raise RuntimeError(f"oracle COCG failed for shift j = {rc - 10}")
    return (out, iters, corr, xs) if return_solutions else (out, iters, corr)


def csr_rel_residual(pattern, tau, sigma, b, x, nthreads=0):
    """||b - (tau A - 1j sigma B) x|| / ||b|| with a double-double residual
    (entries formed with the reference's rounding, integrate.py:171)."""
    indptr, indices, a, bv = pattern
    b = np.ascontiguousarray(b, dtype=np.complex128)
    x = np.ascontiguousarray(x, dtype=np.complex128)
    s = (ctypes.c_double * 2)(complex(sigma).real, complex(sigma).imag)
    return float(lib().orc_csr_rel_residual(len(b), _ptr(indptr), _ptr(indices), _ptr(a), _ptr(bv),
                                            float(tau), s, _ptr(b), _ptr(x), int(nthreads)))


def rel_l2(x, y):
    x = np.asarray(x)
    y = np.asarray(y)
    d = np.linalg.norm(y)
    return float(np.linalg.norm(x - y) / (d if d > 0 else 1.0))


# ---------------------------------------------------------------------------
# prepare/comparison paths, numpy/scipy restatements
# ---------------------------------------------------------------------------

def _b_solver(B):
    from scipy.sparse.linalg import splu
    return splu(B.tocsc().astype(complex)).solve


def power_iteration(sysm, tol=1e-6, max_iters=500, seed=0):
    """Restates ``spectral_radius_estimate`` (reference spatial.py:314-344):
    power iteration on B^-1 A from default_rng(seed).standard_normal(n),
    Rayleigh quotient |v^H A v / v^H B v|, relative-change stop.  B^-1 by a
    sparse LU (the reference's banded/dense LU).  Returns (value, its, conv)."""
    solve_b = _b_solver(sysm.B)
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(sysm.n_dof).astype(complex)
    v /= np.linalg.norm(v)
    prev = None
    rq = 0.0
    it = 0
    for it in range(1, max_iters + 1):
        av = sysm.A @ v
        rq = abs(np.vdot(v, av) / np.vdot(v, sysm.B @ v))
        if prev is not None and abs(rq - prev) <= tol * max(rq, 1e-300):
            return float(rq), it, True
        prev = rq
        w = solve_b(av)
        v = w / np.linalg.norm(w)
    return float(rq), it, False


def clenshaw_step(sysm, coeffs, tau, radius, u):
    """Restates ``chebyshev_step`` (reference integrate.py:333-356): Clenshaw
    backward recurrence for sum a_k T_k(-(tau/R) B^-1 A) u."""
    solve_b = _b_solver(sysm.B)
    s = -(tau / radius)
    u = np.asarray(u, dtype=complex)
    b1 = np.zeros_like(u)
    b2 = np.zeros_like(u)
    for k in range(len(coeffs) - 1, 0, -1):
        b1, b2 = coeffs[k] * u + 2.0 * s * solve_b(sysm.A @ b1) - b2, b1
    return coeffs[0] * u + s * solve_b(sysm.A @ b1) - b2
