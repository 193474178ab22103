"""paper_1912_03312_b200 -- B200-native REXI time step (arXiv 1912.03312).

Drop-in for the hot path of the reference package ``rexiprop``:
``rexi_prepare`` / ``rexi_step`` / ``rexi_run`` / ``RexiStepper`` with the
reference's signatures, over hand-written sm_100a CUDA behind the C ABI in
``include/rexi_b200.h`` (``librexi_b200.so``, built in-tree); next to it the
reference's prepare/comparison paths on the same device pencil:
``spectral_radius_estimate`` and the Chebyshev/Clenshaw stepper.
"""

from .errors import (AdmissibilityError, ApproximationError, ConfigError, DeviceError,
                     NumericalError, SolverError, SpatialError)
from .integrate import (SAFETY_FACTOR, RexiStepper, ShiftedSystem, max_step_size, rexi_prepare,
                        rexi_run, rexi_step)
from .chebyshev import (ChebyshevCoeffs, ChebyshevStepper, chebyshev_coeffs, chebyshev_prepare,
                        chebyshev_run, chebyshev_step)
from .spectral import SpectralRadiusEstimate, spectral_radius_estimate
from .types import (PartialFractionApproximation, SystemMatrices, approx_from_json, approx_to_json,
                    evaluate_pfd)

__version__ = "0.1.0"

__all__ = [
    "AdmissibilityError", "ApproximationError", "ConfigError", "DeviceError", "NumericalError",
    "SolverError", "SpatialError", "SAFETY_FACTOR", "RexiStepper", "ShiftedSystem",
    "max_step_size", "rexi_prepare", "rexi_run", "rexi_step", "PartialFractionApproximation",
    "SystemMatrices", "approx_from_json", "approx_to_json", "evaluate_pfd",
    "ChebyshevCoeffs", "ChebyshevStepper", "chebyshev_coeffs", "chebyshev_prepare",
    "chebyshev_run", "chebyshev_step", "SpectralRadiusEstimate", "spectral_radius_estimate",
]
