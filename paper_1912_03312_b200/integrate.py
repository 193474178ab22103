"""REXI stepping on B200 -- drop-in for reference ``rexiprop.integrate``.

Same entry points, signatures, fields, error types and admissibility
semantics as the reference (``pkg/src/rexiprop/integrate.py:43-245``):

* :func:`rexi_prepare` (ref ``:143-190``) validates, computes the
  admissibility ratio and builds the native plan(s): the K shifted
  operators are formed on the device from the shared A/B values with the
  reference's rounding and factored once (1D) or preconditioned (2D/3D).
* :func:`rexi_step` (ref ``:193-226``) runs one step on the GPU and returns
  a fresh array; ``timers`` accumulate seconds per phase.
* :func:`rexi_run` (ref ``:229-245``) with the observer contract
  ``observer(k, k*tau, u)``; without an observer all steps stay on the
  device in one native call.

``workers`` keeps its meaning of "how many pieces the K shifts are split
into" (ref ``:114-120``): each piece is one native plan producing a
double-double partial sum, and the pieces are combined in fixed order, so
the answer does not depend on ``workers`` (ref ``:196-198``,
``test_integrate.py:268-274``).  The default is one piece.  Across GPUs the
same split is driven by :mod:`paper_1912_03312_b200.distributed`.

There is no CPU fallback: without the native library or a CUDA device the
calls raise :class:`DeviceError`.
"""

from __future__ import annotations

import re
import time
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _native
from ._pattern import shared_pattern
from .errors import AdmissibilityError, SolverError

SAFETY_FACTOR = 1.05
# tau * sr(M) above which 1D solves get one round of double-double residual
# refinement by default.
AUTO_REFINE_STIFFNESS = 5e3
# rexi_run with an observer keeps at most this many bytes of states per chunk
RUN_CHUNK_BYTES = 256 << 20

Observer = Callable[[int, float, np.ndarray], None]


def max_step_size(r1: float, sr_m: float) -> float:
    """Largest step keeping tau * sr(M) <= R1 (ref ``integrate.py:50-56``)."""
    if not sr_m > 0:
        raise ValueError(f"spectral radius must be positive, got {sr_m}")
    if not r1 > 0:
        raise ValueError(f"interval radius must be positive, got {r1}")
    return r1 / sr_m


def _admissibility(tau: float, sr_value: float, radius: float):
    ratio = SAFETY_FACTOR * tau * float(sr_value) / radius
    return ratio, ratio <= 1.0


def _require_admissible(kind: str, stepper) -> None:
    """Ref ``integrate.py:76-88``."""
    if stepper.admissible:
        return
    if stepper.override_admissibility:
        stepper.override_used = True
        return
    largest = stepper.interval_radius / (SAFETY_FACTOR * stepper.sr_value)
    raise AdmissibilityError(
        f"{kind} step tau = {stepper.tau:g} is inadmissible: "
        f"{SAFETY_FACTOR} * tau * sr(M) / R1 = {stepper.admissibility_ratio:.4g} "
        f"> 1; the largest admissible step for this system is "
        f"max_step_size = {largest:.6e}"
    )


class ShiftedSystem:
    """``factorizations[j]`` of the reference (``solvers.py:39-80``): the
    shifted operator j as seen through the GPU plan.

    ``matrix`` is the host CSR of ``tau*A - (1j*sigma_j)*B`` (built lazily,
    for inspection; the device forms it on the fly), ``solve(b)`` runs the
    device solve of all shifts of the owning plan and returns column j.
    """

    def __init__(self, stepper: "RexiStepper", j: int):
        self._stepper = stepper
        self._j = j
        self._matrix = None

    @property
    def matrix(self):
        if self._matrix is None:
            s = self._stepper
            sigma = complex(s.approx.shifts[self._j])
            self._matrix = (s.tau * s.system.A - (1j * sigma) * s.system.B).tocsr()
        return self._matrix

    @property
    def bandwidth(self):
        return self._stepper.bandwidth

    def solve(self, b: np.ndarray) -> np.ndarray:
        return self._stepper._solve_shift(self._j, b)


@dataclass
class RexiStepper:
    """Prepared REXI propagator (ref ``integrate.py:95-140``); ``plans`` are
    the native plans, one per shift piece, ``stats`` carries device-side
    diagnostics (levels, refinement, COCG iterations, HBM held)."""

    approx: object
    tau: float
    system: object
    factorizations: list
    workers: int
    sr_value: float
    admissibility_ratio: float
    admissible: bool
    override_admissibility: bool = False
    override_used: bool = False
    timers: dict = field(default_factory=lambda: {"rhs": 0.0, "local": 0.0, "reduce": 0.0})
    plans: list = field(default_factory=list, repr=False)
    pieces: list = field(default_factory=list, repr=False)
    device: int = 0
    refine: int = 0
    solver: str = "auto"
    stats: dict = field(default_factory=dict)

    @property
    def interval_radius(self) -> float:
        return self.approx.domain_radius

    @property
    def bandwidth(self):
        """Bandwidth of the shifted systems (None when not banded, as the
        reference reports for its dense fallback)."""
        return self.stats.get("bandwidth")

    def close(self):
        for p in self.plans:
            p.close()
        self.plans = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- internals --------------------------------------------------------
    def _solve_shift(self, j: int, b: np.ndarray) -> np.ndarray:
        b = np.asarray(b, dtype=complex)
        if b.ndim == 2:
            return np.stack([self._solve_shift(j, b[:, c]) for c in range(b.shape[1])], axis=1)
        for plan, idx in zip(self.plans, self.pieces):
            if idx[0] <= j <= idx[-1]:
                return plan.solve_host(b)[j - idx[0]]
        raise IndexError(j)


_SOLVERS = {"auto": _native.SOLVER_AUTO, "tridiag": _native.SOLVER_TRIDIAG,
            "cocg": _native.SOLVER_COCG}


def rexi_prepare(
    sys,
    approx,
    tau: float,
    *,
    workers: int | None = None,
    sr_value: float | None = None,
    override_admissibility: bool = False,
    device: int | None = None,
    refine: int | None = None,
    solver: str = "auto",
    tol: float | None = None,
    max_iters: int | None = None,
) -> RexiStepper:
    """Form and factor the K shifted systems on the GPU (ref ``:143-190``).

    Extra keyword-only knobs (all optional): ``device`` (CUDA ordinal),
    ``refine`` (double-double residual-refinement rounds; default by
    stiffness), ``solver`` ("auto" | "tridiag" | "cocg"), ``tol`` and
    ``max_iters`` for COCG.
    """
    if not tau > 0:
        raise ValueError(f"tau must be positive, got {tau}")
    shifts = np.asarray(approx.shifts, dtype=complex)
    weights = np.asarray(approx.weights, dtype=complex)
    k = len(shifts)
    if len(np.unique(shifts)) != k:
        raise ValueError("approximation shifts must be distinct")
    requested = workers
    if workers is None:
        workers = 1
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if solver not in _SOLVERS:
        raise ValueError(f"unknown solver {solver!r}")
    if sr_value is None:
        from .spectral import spectral_radius_estimate
        sr_value = spectral_radius_estimate(sys, device=0 if device is None else int(device))
    ratio, admissible = _admissibility(tau, sr_value, approx.domain_radius)
    dev = 0 if device is None else int(device)

    indptr, indices, a_re, a_im, b_re = shared_pattern(sys.A, sys.B)
    if refine is None:
        rows = np.repeat(np.arange(len(indptr) - 1), np.diff(indptr))
        tridiagonal = len(indices) == 0 or int(np.max(np.abs(indices - rows))) <= 1
        if tridiagonal and solver != "cocg":
            refine = 1 if tau * float(sr_value) > AUTO_REFINE_STIFFNESS else 0
        else:
            refine = 1          # COCG: one double-double refinement round
    pieces = [c for c in np.array_split(np.arange(k), min(workers, k)) if len(c)]
    plans = []
    try:
        for idx in pieces:
            try:
                plans.append(_native.NativePlan(
                    indptr, indices, a_re, b_re, shifts[idx], weights[idx], tau, a_imag=a_im,
                    device=dev, solver=_SOLVERS[solver], refine=int(refine),
                    tol=float(tol or 0.0), max_iters=int(max_iters or 0),
                    shift_offset=int(idx[0]), weight_ref=float(np.mean(np.abs(weights)))))
            except SolverError as exc:
                m = re.search(r"j = (\d+)", str(exc))
                j = int(m.group(1)) if m else int(idx[0])
                raise SolverError(
                    f"shifted system j = {j} (sigma = {shifts[j]}) is singular: the "
                    f"shift coincides with an eigenvalue of tau*M ({exc})"
                ) from exc
    except BaseException:
        for p in plans:
            p.close()
        raise

    info = plans[0].info
    band = int(info.bandwidth)
    stepper = RexiStepper(
        approx=approx,
        tau=tau,
        system=sys,
        factorizations=[],
        workers=workers if requested is not None else workers,
        sr_value=float(sr_value),
        admissibility_ratio=ratio,
        admissible=admissible,
        override_admissibility=override_admissibility,
        plans=plans,
        pieces=[list(map(int, c)) for c in pieces],
        device=dev,
        refine=int(info.refine),
        solver={1: "tridiag", 2: "cocg"}.get(int(info.solver), "auto"),
        stats={"bandwidth": band if band <= 32 else None,
               "levels": int(info.levels), "k_pad": int(info.k_pad),
               "device_bytes": int(sum(p.info.device_bytes for p in plans)),
               "prepare_ms": float(sum(p.info.prepare_ms for p in plans)),
               "min_pivot_ratio": float(min(p.info.min_pivot_ratio for p in plans))},
    )
    stepper.factorizations = [ShiftedSystem(stepper, j) for j in range(k)]
    return stepper


def _is_torch(u) -> bool:
    return type(u).__module__.startswith("torch")


def _step_pieces_device(stepper: RexiStepper, u_t, out_t, n_steps: int):
    """Multi-piece stepping on device tensors (torch plumbing only)."""
    import torch
    n = u_t.shape[0]
    g = len(stepper.plans)
    parts = torch.empty((g, 4, n), dtype=torch.float64, device=u_t.device)
    cur = u_t.clone()
    nxt = torch.empty_like(cur)
    for _ in range(n_steps):
        t0 = time.perf_counter()
        for q, plan in enumerate(stepper.plans):
            plan.step_partial(cur.data_ptr(), parts[q].data_ptr())
        t1 = time.perf_counter()
        _native.combine_partials(parts.data_ptr(), g, n, nxt.data_ptr())
        t2 = time.perf_counter()
        stepper.timers["local"] += t1 - t0
        stepper.timers["reduce"] += t2 - t1
        cur, nxt = nxt, cur
    out_t.copy_(cur)


def _run_native(stepper: RexiStepper, u, n_steps: int):
    """n_steps steps; numpy in -> numpy out, torch CUDA in -> torch out."""
    if _is_torch(u):
        import torch
        if not u.is_cuda:
            return torch.from_numpy(_run_native(stepper, u.detach().cpu().numpy(), n_steps))
        u_t = u.to(torch.complex128).contiguous()
        out = torch.empty_like(u_t)
        if len(stepper.plans) == 1:
            t0 = time.perf_counter()
            stepper.plans[0].step_device(u_t.data_ptr(), out.data_ptr(), n_steps)
            stepper.timers["local"] += time.perf_counter() - t0
        else:
            _step_pieces_device(stepper, u_t, out, n_steps)
        return out
    u = np.ascontiguousarray(u, dtype=complex)
    if len(stepper.plans) == 1:
        t0 = time.perf_counter()
        out = stepper.plans[0].step_host(u, n_steps)
        stepper.timers["local"] += time.perf_counter() - t0
        return out
    import torch
    u_t = torch.from_numpy(u).to(f"cuda:{stepper.device}")
    out_t = torch.empty_like(u_t)
    _step_pieces_device(stepper, u_t, out_t, n_steps)
    return out_t.cpu().numpy()


def rexi_step(stepper: RexiStepper, u):
    """One REXI step (ref ``integrate.py:193-226``): rhs = iBu, K shifted
    solves, beta-weighted sum in fixed order (double-double)."""
    return _run_native(stepper, u, 1)


def rexi_run(stepper: RexiStepper, u0, n_steps: int, observer: Observer | None = None):
    """Apply rexi_step ``n_steps`` times (ref ``integrate.py:229-245``)."""
    if n_steps < 0:
        raise ValueError(f"n_steps must be >= 0, got {n_steps}")
    if n_steps > 0:
        _require_admissible("REXI", stepper)
    if _is_torch(u0):
        u = u0.clone()
    else:
        u = np.array(u0, dtype=complex, copy=True)
    if n_steps == 0:
        return u
    if observer is None:
        return _run_native(stepper, u, n_steps)
    if len(stepper.plans) == 1 and not _is_torch(u):
        # every state is produced on the device (rexi_plan_run: one launch for
        # small 1D plans), copied back in chunks, and handed to the observer
        # in order; each state is its own array, as in the reference loop
        n = stepper.plans[0].n
        chunk = max(1, min(n_steps, RUN_CHUNK_BYTES // (16 * max(n, 1))))
        k = 0
        while k < n_steps:
            c = min(chunk, n_steps - k)
            t0 = time.perf_counter()
            states = stepper.plans[0].run_host(u, c)
            stepper.timers["local"] += time.perf_counter() - t0
            for s in range(c):
                k += 1
                observer(k, k * stepper.tau, states[s])
            u = states[c - 1]
        return u
    for k in range(1, n_steps + 1):
        u = rexi_step(stepper, u)
        observer(k, k * stepper.tau, u)
    return u
