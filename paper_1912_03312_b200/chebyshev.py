"""Chebyshev / Clenshaw stepping on the GPU -- drop-in for the reference's
comparison propagator (``rexiprop.integrate``, ``integrate.py:248-377``).

* :func:`chebyshev_coeffs` (ref ``:257-280``) -- host setup: coefficients
  a_0..a_N of sum a_k T_k(x) ~ exp(i r x) on [-1, 1] from samples at the
  N+1 Chebyshev-Lobatto points (discrete cosine sum with half weights at
  the ends), with the sup-norm error measured on a 100 001-point grid.
* :func:`chebyshev_prepare` (ref ``:303-330``) -- validation, spectral
  radius (GPU power iteration when ``sr_value`` is None), admissibility
  ratio, and the device pencil that replaces ``factorize(sys.B)``.
* :func:`chebyshev_step` / :func:`chebyshev_run` (ref ``:333-377``) -- the
  Clenshaw backward recurrence b_k = a_k u + 2 s B^-1 A b_{k+1} - b_{k+2},
  out = a_0 u + s B^-1 A b_1 - b_2 with s = -tau/R, entirely on the device
  (``rexi_pencil_cheb_step``, ``csrc/pencil.cu``): per stage one fused
  A-multiply + CG start, CG iterations on B, one combine kernel.  Without
  an observer, ``chebyshev_run`` keeps all steps on the device in one call.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np
from numpy.polynomial.chebyshev import chebval

from . import _native
from .integrate import Observer, _admissibility, _is_torch, _require_admissible
from .spectral import pencil_of, spectral_radius_estimate


class ChebyshevCoeffs(NamedTuple):
    coeffs: np.ndarray
    sup_error: float


def chebyshev_coeffs(r: float, n: int) -> ChebyshevCoeffs:
    """Coefficients of the degree-n Chebyshev interpolant of exp(i r x) at
    the Lobatto points cos(pi j / n) (ref ``integrate.py:257-280``)."""
    if n < 1:
        raise ValueError(f"degree must be >= 1, got {n}")
    if not r > 0:
        raise ValueError(f"interval radius must be positive, got {r}")
    j = np.arange(n + 1)
    samples = np.exp(1j * r * np.cos(np.pi * j / n))
    half = np.ones(n + 1)
    half[[0, n]] = 0.5
    table = np.cos(np.pi * np.outer(j, j) / n)
    a = (2.0 / n) * (table @ (half * samples))
    a[0] *= 0.5
    a[n] *= 0.5
    grid = np.linspace(-1.0, 1.0, 100_001)
    sup = float(np.max(np.abs(chebval(grid, a) - np.exp(1j * r * grid))))
    return ChebyshevCoeffs(coeffs=a, sup_error=sup)


class BSolve:
    """``factorize(sys.B)`` seen through the device pencil (the reference's
    solver protocol ``.solve(b)``, ``.matrix``, ``.bandwidth``,
    ``solvers.py:39-115``); solves run as CG on the GPU."""

    def __init__(self, pencil, B):
        self._pencil = pencil
        self.matrix = B
        self.bandwidth = None

    def solve(self, b: np.ndarray) -> np.ndarray:
        b = np.asarray(b, dtype=complex)
        if b.ndim == 2:
            return np.stack([self.solve(b[:, c]) for c in range(b.shape[1])], axis=1)
        x, _ = self._pencil.solve_b(b)
        return x


@dataclass
class ChebyshevStepper:
    """Prepared Clenshaw propagator for p(tau*M) (ref ``integrate.py:283-300``)."""

    coeffs: np.ndarray
    degree: int
    R: float
    tau: float
    B_factorization: object
    sup_error: float
    sr_value: float
    admissibility_ratio: float
    admissible: bool
    override_admissibility: bool = False
    override_used: bool = False
    timers: dict = field(default_factory=lambda: {"rhs": 0.0, "local": 0.0, "reduce": 0.0})
    pencil: object = field(default=None, repr=False)
    device: int = 0
    stats: dict = field(default_factory=dict)

    @property
    def interval_radius(self) -> float:
        return self.R

    @property
    def scale(self) -> float:
        return -(self.tau / self.R)

    def close(self):
        if self.pencil is not None:
            self.pencil.close()
            self.pencil = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def chebyshev_prepare(sys, tau: float, *, degree: int = 26, radius: float = 10.0,
                      sr_value: float | None = None, override_admissibility: bool = False,
                      device: int | None = None, tol: float | None = None,
                      max_iters: int | None = None) -> ChebyshevStepper:
    """Build coefficients for i[-radius, radius] and put the pencil on the
    device (ref ``integrate.py:303-330``).  Extra keyword-only knobs:
    ``device``, ``tol`` / ``max_iters`` of the CG B-solves (default 1e-14 /
    1000)."""
    if not tau > 0:
        raise ValueError(f"tau must be positive, got {tau}")
    dev = 0 if device is None else int(device)
    if sr_value is None:
        sr_value = spectral_radius_estimate(sys, device=dev)
    cc = chebyshev_coeffs(radius, degree)
    ratio, admissible = _admissibility(tau, sr_value, radius)
    pencil = pencil_of(sys, device=dev, tol=0.0 if tol is None else float(tol),
                       max_iters=0 if max_iters is None else int(max_iters))
    return ChebyshevStepper(
        coeffs=cc.coeffs, degree=degree, R=float(radius), tau=tau,
        B_factorization=BSolve(pencil, sys.B), sup_error=cc.sup_error,
        sr_value=float(sr_value), admissibility_ratio=ratio, admissible=admissible,
        override_admissibility=override_admissibility, pencil=pencil, device=dev)


def _cheb_native(stepper: ChebyshevStepper, u, n_steps: int):
    st = _native.RexiStats()
    t0 = time.perf_counter()
    if _is_torch(u):
        import torch
        if not u.is_cuda:
            return torch.from_numpy(_cheb_native(stepper, u.detach().cpu().numpy(), n_steps))
        dev = torch.device("cuda", stepper.device)
        u_t = u.to(device=dev, dtype=torch.complex128).contiguous()
        out = torch.empty_like(u_t)
        # u_t was produced on torch's current stream: order the pencil's stream after it
        stepper.pencil.wait_stream(torch.cuda.current_stream(dev).cuda_stream)
        stepper.pencil.cheb_step(stepper.coeffs, stepper.scale, u_t.data_ptr(), out.data_ptr(),
                                 n_steps, _native.MEM_DEVICE, st)
    else:
        out = stepper.pencil.cheb_step_host(stepper.coeffs, stepper.scale, u, n_steps, st)
    stepper.timers["local"] += time.perf_counter() - t0
    stepper.stats = {"cg_iters_max": int(st.iters_max), "cg_iters_mean": float(st.iters_mean),
                     "launches": int(st.launches), "device_ms": float(st.t_local_ms)}
    return out


def chebyshev_step(stepper: ChebyshevStepper, sys, u):
    """p(tau*M) u by the Clenshaw backward recurrence (ref
    ``integrate.py:333-356``); ``sys`` must be the system the stepper was
    prepared for (its pencil already lives on the device)."""
    if sys is not None and int(sys.n_dof) != stepper.pencil.n:
        raise ValueError(f"system has {sys.n_dof} DOF, stepper was prepared for {stepper.pencil.n}")
    return _cheb_native(stepper, u, 1)


def chebyshev_run(stepper: ChebyshevStepper, sys, u0, n_steps: int,
                  observer: Observer | None = None):
    """Apply chebyshev_step ``n_steps`` times with the observer contract of
    rexi_run (ref ``integrate.py:359-377``)."""
    if n_steps < 0:
        raise ValueError(f"n_steps must be >= 0, got {n_steps}")
    if n_steps > 0:
        _require_admissible("Chebyshev", stepper)
    if _is_torch(u0):
        u = u0.clone()
    else:
        u = np.array(u0, dtype=complex, copy=True)
    if n_steps == 0:
        return u
    if observer is None:
        return _cheb_native(stepper, u, n_steps)
    for k in range(1, n_steps + 1):
        u = chebyshev_step(stepper, sys, u)
        observer(k, k * stepper.tau, u)
    return u
