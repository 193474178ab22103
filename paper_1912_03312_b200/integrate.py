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
double-double partial sum, the pieces are spread over the visible GPUs of
this process and combined in fixed order, so the answer does not depend on
``workers`` or on the GPU count (ref ``:196-198``,
``test_integrate.py:268-274``).  The default is one piece per GPU.  One
process per GPU (torchrun) uses :mod:`paper_1912_03312_b200.distributed`.

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
    _plan_args: tuple = field(default=None, repr=False)
    _slots: list = field(default_factory=list, repr=False)
    _rebalanced: bool = field(default=True, repr=False)

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
            if j in idx:
                return plan.solve_host(b)[idx.index(j)]
        raise IndexError(j)


_SOLVERS = {"auto": _native.SOLVER_AUTO, "tridiag": _native.SOLVER_TRIDIAG,
            "cocg": _native.SOLVER_COCG, "band": _native.SOLVER_BAND}
# below this many row-shifts (n*K) the default keeps one GPU: a config-1-sized
# step (~1 MB of work) is launch-latency bound and a cross-GPU combine would
# cost more than the solves
MULTI_GPU_MIN_WORK = 1 << 22


def _default_devices(n: int, k: int, device, devices):
    if devices is not None:
        devs = [int(d) for d in devices]
        if not devs:
            raise ValueError("devices must not be empty")
        return devs
    if device is not None:
        return [int(device)]
    visible = _native.device_count()
    if visible <= 1 or n * k < MULTI_GPU_MIN_WORK:
        return [0]
    return list(range(visible))


def _make_plans(stepper_args, pieces, piece_devs):
    """One native plan per piece (shift index list) on its device."""
    (indptr, indices, a_re, a_im, b_re, shifts, weights, tau, solver, refine, tol, max_iters,
     wref) = stepper_args
    plans = []
    try:
        for idx, dev in zip(pieces, piece_devs):
            idx = np.asarray(idx, dtype=np.int64)
            try:
                plans.append(_native.NativePlan(
                    indptr, indices, a_re, b_re, shifts[idx], weights[idx], tau, a_imag=a_im,
                    device=dev, solver=_SOLVERS[solver], refine=int(refine),
                    tol=float(tol or 0.0), max_iters=int(max_iters or 0),
                    shift_offset=int(idx[0]), weight_ref=wref, shift_ids=idx))
            except SolverError as exc:
                # the native message is the reference's factorize() message
                # (solvers.py:52-69) tagged "[shift j = N]" with the global index
                m = re.search(r"j = (\d+)", str(exc))
                j = int(m.group(1)) if m else int(idx[0])
                inner = re.sub(r"\s*\[shift j = \d+\]$", "", str(exc))
                raise SolverError(
                    f"shifted system j = {j} (sigma = {shifts[j]}) is singular: the "
                    f"shift coincides with an eigenvalue of tau*M ({inner})"
                ) from exc
    except BaseException:
        for p in plans:
            p.close()
        raise
    return plans


def max_shifts_per_plan(indptr, indices, solver: str = "auto") -> int:
    """Shifts one native plan takes: 256 for the tridiagonal solver (its
    level-0 lane tile), 1024 for the band solver, and for COCG the largest
    power of two keeping n * k_pad below 2^31 (32-bit element offsets)."""
    indptr = np.asarray(indptr)
    indices = np.asarray(indices)
    n = len(indptr) - 1
    rows = np.repeat(np.arange(n), np.diff(indptr))
    half_band = 0 if len(indices) == 0 else int(np.max(np.abs(indices - rows)))
    if solver == "tridiag" or (solver == "auto" and half_band <= 1):
        return 256
    if solver == "band" or (solver == "auto" and 2 <= half_band <= 4):
        return 1024
    kp = 1
    while 2 * kp * max(n, 1) < 2 ** 31 - 1:
        kp *= 2
    return kp


def default_refine(indptr, indices, tau: float, sr_value: float, solver: str = "auto") -> int:
    """The refinement rounds ``rexi_prepare`` uses when ``refine`` is not
    given: the direct solvers (1D tridiagonal, and the band LU for half
    bandwidths 2..4, the reference's P2 pencils) refine once on stiff pencils
    (tau*sr above AUTO_REFINE_STIFFNESS, where the fp64 solve alone drifts
    past 1e-8 of truth), COCG always refines once (double-double residual
    round)."""
    indptr = np.asarray(indptr)
    indices = np.asarray(indices)
    rows = np.repeat(np.arange(len(indptr) - 1), np.diff(indptr))
    half_band = 0 if len(indices) == 0 else int(np.max(np.abs(indices - rows)))
    direct = half_band <= 1 or (2 <= half_band <= 4 and solver != "tridiag")
    if direct and solver != "cocg":
        return 1 if tau * float(sr_value) > AUTO_REFINE_STIFFNESS else 0
    return 1


def rexi_prepare(
    sys,
    approx,
    tau: float,
    *,
    workers: int | None = None,
    sr_value: float | None = None,
    override_admissibility: bool = False,
    device: int | None = None,
    devices=None,
    refine: int | None = None,
    solver: str = "auto",
    tol: float | None = None,
    max_iters: int | None = None,
) -> RexiStepper:
    """Form and factor the K shifted systems on the GPU(s) (ref ``:143-190``).

    ``workers`` keeps the reference's meaning -- the number of pieces the K
    shifts are split into (ref ``:114-120``) -- and the pieces are spread
    round-robin over the GPUs: ``devices`` (list of CUDA ordinals; default
    all visible GPUs for steps of at least ``MULTI_GPU_MIN_WORK`` row-shifts,
    else GPU 0, or ``[device]`` when ``device`` is given).  ``workers=None``
    gives one piece per GPU and reports ``workers = K`` like the reference's
    default (``:161-162``).  Pieces produce double-double partial sums that
    are combined in fixed piece order, so the answer does not depend on the
    split.  With COCG on several GPUs the pieces are re-balanced once after
    the first step by the measured per-shift iteration counts (LPT).

    Extra keyword-only knobs (all optional): ``refine`` (double-double
    residual-refinement rounds; default by stiffness), ``solver`` ("auto" |
    "tridiag" | "band" | "cocg"), ``tol`` and ``max_iters`` for COCG.
    """
    if not tau > 0:
        raise ValueError(f"tau must be positive, got {tau}")
    shifts = np.asarray(approx.shifts, dtype=complex)
    weights = np.asarray(approx.weights, dtype=complex)
    k = len(shifts)
    if len(np.unique(shifts)) != k:
        raise ValueError("approximation shifts must be distinct")
    if workers is not None and workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if solver not in _SOLVERS:
        raise ValueError(f"unknown solver {solver!r}")
    devs = _default_devices(int(sys.n_dof), k, device, devices)
    if sr_value is None:
        from .spectral import spectral_radius_estimate
        sr_value = spectral_radius_estimate(sys, device=devs[0])
    ratio, admissible = _admissibility(tau, sr_value, approx.domain_radius)

    indptr, indices, a_re, a_im, b_re = shared_pattern(sys.A, sys.B)
    if refine is None:
        refine = default_refine(indptr, indices, tau, sr_value, solver)
    n_pieces = min(workers, k) if workers is not None else min(len(devs), k)
    devs = devs[:n_pieces]          # one concurrent slot (host thread) per entry
    # a plan holds at most max_shifts_per_plan() shifts (the 1D solver's lane
    # tile, COCG's 32-bit element offsets): more pieces when K exceeds it
    n_pieces = max(n_pieces, -(-k // max_shifts_per_plan(indptr, indices, solver)))
    pieces = [list(map(int, c)) for c in np.array_split(np.arange(k), n_pieces) if len(c)]
    piece_devs = [devs[q % len(devs)] for q in range(len(pieces))]
    args = (indptr, indices, a_re, a_im, b_re, shifts, weights, tau, solver, refine, tol, max_iters,
            float(np.mean(np.abs(weights))))
    plans = _make_plans(args, pieces, piece_devs)

    info = plans[0].info
    band = int(info.bandwidth)
    stepper = RexiStepper(
        approx=approx,
        tau=tau,
        system=sys,
        factorizations=[],
        workers=int(workers) if workers is not None else k,
        sr_value=float(sr_value),
        admissibility_ratio=ratio,
        admissible=admissible,
        override_admissibility=override_admissibility,
        plans=plans,
        pieces=pieces,
        device=devs[0],
        refine=int(info.refine),
        solver={1: "tridiag", 2: "cocg", 3: "band"}.get(int(info.solver), "auto"),
        stats={"bandwidth": band if band <= 32 else None,
               "levels": int(info.levels), "k_pad": int(info.k_pad),
               "devices": sorted(set(piece_devs)),
               "device_bytes": int(sum(p.info.device_bytes for p in plans)),
               "prepare_ms": float(sum(p.info.prepare_ms for p in plans)),
               "min_pivot_ratio": float(min(p.info.min_pivot_ratio for p in plans)),
               "steps": 0, "per_step": []},
    )
    stepper._plan_args = args
    stepper._slots = devs
    stepper._rebalanced = len(devs) < 2 or stepper.solver != "cocg"
    stepper.factorizations = [ShiftedSystem(stepper, j) for j in range(k)]
    return stepper


def _is_torch(u) -> bool:
    return type(u).__module__.startswith("torch")


def _record(stepper: RexiStepper, st: _native.RexiStats | None, wall: float, staged: float = 0.0,
            finish: float = 0.0):
    """Fold one native call into the reference timers (seconds, wall clock
    like ``integrate.py:203-225``) and the per-step stats.  The native
    stats split the device time into rhs / local / reduce (see rexi_stats in
    include/rexi_b200.h); host staging counts as rhs, host finishing as reduce."""
    t_rhs = t_red = 0.0
    if st is not None:
        t_rhs, t_red = st.t_rhs_ms * 1e-3, st.t_reduce_ms * 1e-3
    stepper.timers["rhs"] += staged + t_rhs
    stepper.timers["local"] += max(0.0, wall - t_rhs - t_red)
    stepper.timers["reduce"] += finish + t_red
    if st is None:
        return
    stepper.stats["steps"] += int(st.steps)
    stepper.stats["refine_rounds"] = int(st.refine_rounds)
    stepper.stats["launches"] = int(st.launches)
    if stepper.solver == "cocg":
        its = np.zeros(len(stepper.approx.shifts), dtype=np.int32)
        for plan, idx in zip(stepper.plans, stepper.pieces):
            its[idx] = plan.shift_iters()
        stepper.stats["shift_iters"] = its
        stepper.stats["iters_max"] = int(its.max())
        stepper.stats["iters_mean"] = float(its.mean())
        stepper.stats["per_step"].append({"step": stepper.stats["steps"], "steps_in_call": int(st.steps),
                                          "iters_max": int(its.max()), "iters_mean": float(its.mean())})


def _rebalance(stepper: RexiStepper):
    """COCG on several GPUs: after the first step, re-split the shifts by
    the measured per-shift iterations, longest-processing-time first (the
    lockstep cost of a piece grows with its shifts' iterations; SURVEY.md
    8(e)), keeping the piece count and the piece -> slot assignment."""
    stepper._rebalanced = True
    its = stepper.stats.get("shift_iters")
    if its is None:
        return
    from .distributed import shard_indices
    devs = [p.device for p in stepper.plans]
    cost = its.astype(float) + 1.0
    new = shard_indices(len(cost), len(devs), cost)
    # pieces sharing a slot run one after the other: balance slot loads
    slots = stepper._slots
    if len(devs) != len(slots):
        return
    old_load = max(cost[i].sum() for i in stepper.pieces)
    new_load = max(cost[i].sum() for i in new if i)
    if not new_load < 0.9 * old_load or any(not i for i in new):
        return
    plans = _make_plans(stepper._plan_args, new, devs)
    for p in stepper.plans:
        p.close()
    stepper.plans, stepper.pieces = plans, new
    stepper.stats["rebalanced"] = {"old_max_cost": float(old_load), "new_max_cost": float(new_load)}


def _step_pieces_device(stepper: RexiStepper, u_t, n_steps: int):
    """Multi-piece stepping: u_t on the first plan's device (torch plumbing
    only).  Each device gets u, runs its pieces' partial sums (one host
    thread per device: the native calls release the GIL), the partials are
    gathered on the first device and combined there in piece order."""
    cur = u_t.clone()
    done = 0
    while done < n_steps:
        cur, ran = _pieces_chunk(stepper, cur, n_steps - done)
        done += ran
    return cur


def _pieces_chunk(stepper: RexiStepper, cur, n_steps: int):
    """Steps until n_steps are done or the pieces are re-balanced (after
    which the device buffers must be rebuilt); returns (state, steps run)."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    n = cur.shape[0]
    g = len(stepper.plans)
    dev0 = torch.device("cuda", stepper.plans[0].device)
    nslot = max(1, len(stepper._slots))
    by_dev = {}        # slot -> piece indices (one host thread per slot)
    for q in range(g):
        by_dev.setdefault(q % nslot, []).append(q)
    bufs = {d: (torch.empty(n, dtype=torch.complex128, device=f"cuda:{stepper.plans[qs[0]].device}"),
                torch.empty((len(qs), 4, n), dtype=torch.float64,
                            device=f"cuda:{stepper.plans[qs[0]].device}"))
            for d, qs in by_dev.items()}
    parts = torch.empty((g, 4, n), dtype=torch.float64, device=dev0)
    nxt = torch.empty_like(cur)

    def run_dev(d):
        ub, pb = bufs[d]
        stream = torch.cuda.current_stream(stepper.plans[by_dev[d][0]].device).cuda_stream
        for i, q in enumerate(by_dev[d]):
            plan = stepper.plans[q]
            plan.wait_stream(stream)
            plan.step_partial(ub.data_ptr(), pb[i].data_ptr())

    pool = ThreadPoolExecutor(max_workers=len(by_dev)) if len(by_dev) > 1 else None
    ran = 0
    try:
        while ran < n_steps:
            t0 = time.perf_counter()
            for d in by_dev:
                bufs[d][0].copy_(cur)
            t1 = time.perf_counter()
            if pool is None:
                for d in by_dev:
                    run_dev(d)
            else:
                list(pool.map(run_dev, list(by_dev)))
            t2 = time.perf_counter()
            for d, qs in by_dev.items():
                for i, q in enumerate(qs):
                    parts[q].copy_(bufs[d][1][i])
            with torch.cuda.device(dev0):
                _native.combine_partials(parts.data_ptr(), g, n, nxt.data_ptr(),
                                         torch.cuda.current_stream(dev0).cuda_stream)
            torch.cuda.current_stream(dev0).synchronize()
            t3 = time.perf_counter()
            stepper.timers["rhs"] += t1 - t0
            stepper.timers["local"] += t2 - t1
            stepper.timers["reduce"] += t3 - t2
            stepper.stats["steps"] += 1
            if stepper.solver == "cocg":
                its = np.zeros(len(stepper.approx.shifts), dtype=np.int32)
                for plan, idx in zip(stepper.plans, stepper.pieces):
                    its[idx] = plan.shift_iters()
                stepper.stats["shift_iters"] = its
                stepper.stats["iters_max"] = int(its.max())
                stepper.stats["iters_mean"] = float(its.mean())
                stepper.stats["per_step"].append({"step": stepper.stats["steps"], "steps_in_call": 1,
                                                  "iters_max": int(its.max()),
                                                  "iters_mean": float(its.mean())})
            cur, nxt = nxt, cur
            ran += 1
            if not stepper._rebalanced:
                _rebalance(stepper)
                break
    finally:
        if pool is not None:
            pool.shutdown()
    return cur, ran


def _run_native(stepper: RexiStepper, u, n_steps: int):
    """n_steps steps; numpy in -> numpy out, torch CUDA in -> torch out."""
    if _is_torch(u):
        import torch
        if not u.is_cuda:
            return torch.from_numpy(_run_native(stepper, u.detach().cpu().numpy(), n_steps))
        t0 = time.perf_counter()
        dev = torch.device("cuda", stepper.plans[0].device)
        u_t = u.to(device=dev, dtype=torch.complex128).contiguous()
        if len(stepper.plans) == 1:
            out = torch.empty_like(u_t)
            plan = stepper.plans[0]
            # the input was produced on torch's current stream: order the plan after it
            plan.wait_stream(torch.cuda.current_stream(dev).cuda_stream)
            st = _native.RexiStats()
            t1 = time.perf_counter()
            plan.step_device(u_t.data_ptr(), out.data_ptr(), n_steps, st)
            t2 = time.perf_counter()
            _record(stepper, st, t2 - t1, staged=t1 - t0, finish=time.perf_counter() - t2)
            return out
        return _step_pieces_device(stepper, u_t, n_steps)
    t0 = time.perf_counter()
    u = np.ascontiguousarray(u, dtype=complex)
    if len(stepper.plans) == 1:
        st = _native.RexiStats()
        t1 = time.perf_counter()
        out = stepper.plans[0].step_host(u, n_steps, st)
        t2 = time.perf_counter()
        # a fused direct step reports its device time as local only; the
        # host-side staging / finishing around it count as rhs / reduce
        _record(stepper, st, t2 - t1, staged=t1 - t0, finish=time.perf_counter() - t2)
        return out
    import torch
    u_t = torch.from_numpy(u).to(f"cuda:{stepper.plans[0].device}")
    stepper.timers["rhs"] += time.perf_counter() - t0
    out_t = _step_pieces_device(stepper, u_t, n_steps)
    t2 = time.perf_counter()
    out = out_t.cpu().numpy()
    stepper.timers["reduce"] += time.perf_counter() - t2
    return out


def rexi_step(stepper: RexiStepper, u):
    """One REXI step (ref ``integrate.py:193-226``): rhs = iBu, K shifted
    solves, beta-weighted sum in fixed order (double-double)."""
    return _run_native(stepper, u, 1)


def rexi_run(stepper: RexiStepper, u0, n_steps: int, observer: Observer | None = None, *,
             readonly_observer: bool = False):
    """Apply rexi_step ``n_steps`` times (ref ``integrate.py:229-245``).

    With an observer each step starts from the very array the observer was
    handed, as in the reference loop, so an observer that modifies the state
    in place steers the run.  ``readonly_observer=True`` promises the
    observer does not modify its argument: the states of a whole chunk of
    steps are then produced on the device in one native call
    (``rexi_plan_run``: one launch for small 1D plans) and handed out in
    order afterwards -- bitwise the same states, much faster for small
    systems.
    """
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
        if stepper.solver == "cocg" and len(stepper.plans) == 1:
            # one native call per step: per-step stats (iterations) are kept
            for _ in range(n_steps):
                u = _run_native(stepper, u, 1)
            return u
        return _run_native(stepper, u, n_steps)
    if readonly_observer and len(stepper.plans) == 1 and not _is_torch(u):
        n = stepper.plans[0].n
        chunk = max(1, min(n_steps, RUN_CHUNK_BYTES // (16 * max(n, 1))))
        k = 0
        while k < n_steps:
            c = min(chunk, n_steps - k)
            t0 = time.perf_counter()
            st = _native.RexiStats()
            states = stepper.plans[0].run_host(u, c, st)
            _record(stepper, st, time.perf_counter() - t0)
            for s in range(c):
                k += 1
                observer(k, k * stepper.tau, states[s])
            u = np.array(states[c - 1])     # do not keep the pinned chunk alive
        return u
    for k in range(1, n_steps + 1):
        u = rexi_step(stepper, u)
        observer(k, k * stepper.tau, u)
    return u
