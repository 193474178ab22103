"""CPU: the 8(f) oracles (power iteration, Clenshaw) and the host-side
Chebyshev coefficients, pinned to the reference's own outputs
(tests/golden/cheb_*.npz, written by make_golden.py --cheb)."""
import numpy as np
import pytest

from conftest import cheb_names, load_cheb
from oracle.oracle import clenshaw_step, power_iteration, rel_l2
from paper_1912_03312_b200.chebyshev import chebyshev_coeffs


@pytest.mark.parametrize("name", cheb_names())
def test_power_iteration_oracle_matches_reference(name):
    d, sysm = load_cheb(name)
    val, its, conv = power_iteration(sysm)
    assert conv == bool(d["sr_converged"])
    assert abs(its - int(d["sr_iterations"])) <= 1
    assert abs(val - float(d["sr"])) <= 1e-9 * float(d["sr"])


@pytest.mark.parametrize("name", cheb_names())
def test_clenshaw_oracle_matches_reference(name):
    d, sysm = load_cheb(name)
    u = d["u0"]
    for k in range(d["steps"].shape[0]):
        u = clenshaw_step(sysm, d["coeffs"], float(d["tau"]), float(d["radius"]), u)
        assert rel_l2(u, d["steps"][k]) <= 1e-12, (name, k)


def test_chebyshev_coeffs_match_reference():
    d, _ = load_cheb(cheb_names()[0])
    cc = chebyshev_coeffs(float(d["radius"]), int(d["degree"]))
    np.testing.assert_allclose(cc.coeffs, d["coeffs"], rtol=0, atol=1e-15)
    assert abs(cc.sup_error - float(d["sup_error"])) <= 1e-3 * float(d["sup_error"])


def test_chebyshev_coeffs_validation():
    with pytest.raises(ValueError):
        chebyshev_coeffs(10.0, 0)
    with pytest.raises(ValueError):
        chebyshev_coeffs(0.0, 8)


def test_chebyshev_polynomial_approximates_exp():
    # p(z) = sum a_k T_k(-iz/r) ~ exp(z) on i[-r, r]: the reference's certificate
    cc = chebyshev_coeffs(10.0, 26)
    x = np.linspace(-1, 1, 2001)
    from numpy.polynomial.chebyshev import chebval
    assert np.max(np.abs(chebval(x, cc.coeffs) - np.exp(10j * x))) <= cc.sup_error * (1 + 1e-12)
