"""Input types of the REXI path, mirrored from the reference.

* :class:`SystemMatrices` mirrors ``rexiprop.spatial.SystemMatrices``
  (reference ``pkg/src/rexiprop/spatial.py:130-136``): the pencil (A, B)
  as scipy CSR float64 on interior DOFs plus ``n_dof``.
* :class:`PartialFractionApproximation` mirrors
  ``rexiprop.approx.PartialFractionApproximation`` (``approx.py:491-517``):
  r(z) = sum_j weights[j] / (z - shifts[j]) on i[-R1, R1].
* :func:`approx_to_json` / :func:`approx_from_json` restate the
  reference's fixed-key-order, 17-significant-digit JSON format
  (``approx.py:691-745``) so frozen pole sets can be read on a box where
  the reference is absent.

The hot path only duck-types these (``.A``, ``.B``, ``.n_dof``;
``.shifts``, ``.weights``, ``.domain_radius``, ``.K``), so the
reference's own objects are accepted unchanged.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np
from scipy.sparse import csr_matrix


@dataclass(frozen=True)
class SystemMatrices:
    """Assembled pencil on interior nodes (Dirichlet rows eliminated)."""

    A: csr_matrix
    B: csr_matrix
    n_dof: int


@dataclass(frozen=True)
class PartialFractionApproximation:
    """r(z) = sum_j weights[j] / (z - shifts[j]) approximating exp on
    i*[-domain_radius, domain_radius] (reference ``approx.py:491-517``)."""

    shifts: np.ndarray
    weights: np.ndarray
    domain_radius: float
    sup_error: float
    stabilized: bool = False
    stabilize_factor: float | None = None
    warnings: tuple = field(default=(), compare=False)

    def __post_init__(self):
        object.__setattr__(self, "shifts", np.asarray(self.shifts, dtype=complex))
        object.__setattr__(self, "weights", np.asarray(self.weights, dtype=complex))
        if len(self.shifts) != len(self.weights):
            raise ValueError("shifts and weights must have equal length")

    @property
    def K(self) -> int:
        return len(self.shifts)


def evaluate_pfd(approx, z):
    """sum_j beta_j / (z - sigma_j) (reference ``approx.py:520-532``)."""
    z_arr = np.asarray(z, dtype=complex)
    diffs = z_arr[..., None] - np.asarray(approx.shifts)
    out = np.sum(np.asarray(approx.weights) / diffs, axis=-1)
    return out if z_arr.ndim else complex(out)


_JSON_KEYS = ("K", "R1", "shifts", "weights", "sup_error", "stabilized",
              "stabilize_factor")


def _fmt17(x: float) -> str:
    return format(float(x), ".17g")


def approx_to_json(approx) -> str:
    """Same byte format as reference ``approx_to_json`` (approx.py:700-721)."""
    def pairs(arr):
        return "[" + ", ".join(
            f"[{_fmt17(v.real)}, {_fmt17(v.imag)}]" for v in arr
        ) + "]"

    factor = ("null" if approx.stabilize_factor is None
              else _fmt17(approx.stabilize_factor))
    body = ", ".join([
        f'"K": {approx.K}',
        f'"R1": {_fmt17(approx.domain_radius)}',
        f'"shifts": {pairs(approx.shifts)}',
        f'"weights": {pairs(approx.weights)}',
        f'"sup_error": {_fmt17(approx.sup_error)}',
        f'"stabilized": {"true" if approx.stabilized else "false"}',
        f'"stabilize_factor": {factor}',
    ])
    return "{" + body + "}"


def approx_from_json(text: str) -> PartialFractionApproximation:
    """Inverse of :func:`approx_to_json`, bit-exact (approx.py:724-745)."""
    try:
        raw = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ValueError(f"not valid JSON: {exc}") from exc
    missing = [k for k in _JSON_KEYS if k not in raw]
    if missing:
        raise ValueError(f"approximation JSON is missing keys: {missing}")
    shifts = np.array([complex(re, im) for re, im in raw["shifts"]])
    weights = np.array([complex(re, im) for re, im in raw["weights"]])
    if len(shifts) != raw["K"] or len(weights) != raw["K"]:
        raise ValueError("K does not match the length of shifts/weights")
    return PartialFractionApproximation(
        shifts=shifts,
        weights=weights,
        domain_radius=float(raw["R1"]),
        sup_error=float(raw["sup_error"]),
        stabilized=bool(raw["stabilized"]),
        stabilize_factor=(None if raw["stabilize_factor"] is None
                          else float(raw["stabilize_factor"])),
    )
