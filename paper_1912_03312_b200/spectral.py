"""Spectral radius of M = (iB)^-1 A on the GPU -- drop-in for reference
``rexiprop.spatial.spectral_radius_estimate`` (``spatial.py:296-344``).

Same algorithm and stopping rule as the reference: power iteration on
B^-1 A from ``numpy.random.default_rng(seed).standard_normal(n)`` (so the
start vector is the reference's, bit for bit), Rayleigh quotient
|v^H A v / v^H B v|, converged when two successive quotients agree to
``tol`` relative, at most ``max_iters`` iterations.  The reference applies
B^-1 with an LU factorisation (``factorize(sys.B)``, banded or dense); here
each B-solve is a Jacobi-preconditioned CG on the device
(``rexi_pencil_spectral_radius``, ``csrc/pencil.cu``), which is what makes
the estimate usable for the 2D/3D configurations where the reference falls
back to a dense LU.
"""

from __future__ import annotations

import numpy as np

from . import _native
from ._pattern import shared_pattern


class SpectralRadiusEstimate(float):
    """A float (the estimate) carrying power-iteration diagnostics
    (reference ``spatial.py:296-311``)."""

    iterations: int
    converged: bool

    def __new__(cls, value: float, iterations: int, converged: bool):
        obj = super().__new__(cls, value)
        obj.iterations = iterations
        obj.converged = converged
        return obj

    def __repr__(self):
        return (f"SpectralRadiusEstimate({float(self)!r}, "
                f"iterations={self.iterations}, converged={self.converged})")


def pencil_of(sys, *, device: int = 0, tol: float = 0.0, max_iters: int = 0):
    """Native pencil (A, B) of a ``SystemMatrices`` on one device."""
    indptr, indices, a_re, a_im, b_re = shared_pattern(sys.A, sys.B)
    return _native.NativePencil(indptr, indices, a_re, b_re, a_imag=a_im, device=device,
                                tol=tol, max_iters=max_iters)


def spectral_radius_estimate(sys, tol: float = 1e-6, max_iters: int = 500, seed: int = 0, *,
                             device: int | None = None) -> SpectralRadiusEstimate:
    """Power iteration on B^-1 A with B-pencil Rayleigh quotients (ref
    ``spatial.py:314-344``); ``device`` (keyword-only) is the CUDA ordinal."""
    rng = np.random.default_rng(seed)
    v0 = rng.standard_normal(sys.n_dof).astype(complex)
    pencil = pencil_of(sys, device=0 if device is None else int(device))
    try:
        value, iterations, converged = pencil.spectral_radius(v0, tol, max_iters)
    finally:
        pencil.close()
    return SpectralRadiusEstimate(value, iterations, converged)
