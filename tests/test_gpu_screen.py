"""GPU: the singularity screen matches the reference's.  The reference
rejects a shift when the partially pivoted band LU (zgbtrf) has a zero pivot
or min|U_ii| < 1e-14 max|U_ii| (solvers.py:52-69), for every pattern with
kl + ku + 1 <= 32; the plan recomputes that factor's U diagonal on the device
(csrc/screen.cu) for the direct 1D solver AND for COCG plans on such bands
(P2 pentadiagonal).  Compared here with scipy's own zgbtrf on shifts at, near
and away from an eigenvalue of tau B^-1 A."""
import re

import numpy as np
import pytest

import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from test_oracle import _reference_screen, screen_cases  # noqa: E402

pytestmark = pytest.mark.gpu


def _native_verdict(sysm, tau, sigma):
    from paper_1912_03312_b200 import SolverError, _native
    from paper_1912_03312_b200._pattern import shared_pattern
    ip, ix, ar, ai, br = shared_pattern(sysm.A, sysm.B)
    try:
        plan = _native.NativePlan(ip, ix, ar, br, np.array([sigma]), np.array([1.0 + 0j]), tau, a_imag=ai)
    except SolverError as exc:
        return True, None, str(exc)
    ratio = float(plan.info.screen_pivot_ratio)
    plan.close()
    return False, ratio, ""


@pytest.mark.parametrize("case", range(len(screen_cases())))
def test_screen_verdict_equals_reference(case):
    sysm, tau, sigma = screen_cases()[case]
    rmin, rmax, rinfo = _reference_screen(sysm, sigma, tau)
    ref_bad = rinfo > 0 or rmin < 1e-14 * rmax
    rratio = rmin / rmax
    bad, ratio, msg = _native_verdict(sysm, tau, sigma)
    if 5e-15 < rratio < 2e-14:
        pytest.skip(f"reference ratio {rratio:.2e} within rounding of the 1e-14 floor")
    assert bad == ref_bad, (sigma, rratio, ratio, msg)
    if bad:
        assert re.match(r"matrix is numerically singular \(pivot ratio = [0-9.e+-]+\) \[shift j = 0\]$", msg) \
            or msg.startswith("matrix is singular: zero pivot at index"), msg
    elif rratio > 1e-12:
        assert abs(ratio - rratio) <= 1e-6 * rratio, (ratio, rratio)


def test_prepare_message_is_the_reference_message():
    """rexi_prepare's SolverError text is integrate.py:172-178's, wrapping
    solvers.py:64-67's, for the first singular shift in j order"""
    from paper_1912_03312_b200 import SolverError, rexi_prepare
    from paper_1912_03312_b200.types import PartialFractionApproximation
    sysm, tau, sigma = [c for c in screen_cases() if c[0].A.nnz == 118][3]     # on an eigenvalue
    shifts = np.array([5 + 3j, 6 - 2j, sigma, sigma + 1e-3j * 0 + 7])
    ap = PartialFractionApproximation(shifts, np.ones(4, complex), 10.0, 0.0)
    with pytest.raises(SolverError) as ei:
        rexi_prepare(sysm, ap, tau, sr_value=1.0, override_admissibility=True)
    msg = str(ei.value)
    assert re.fullmatch(
        rf"shifted system j = 2 \(sigma = {re.escape(str(sigma))}\) is singular: the shift coincides with an "
        r"eigenvalue of tau\*M \(matrix is numerically singular \(pivot ratio = [0-9.]+e[+-]\d+\)\)", msg), msg
