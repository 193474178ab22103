"""CPU tests of the oracle (test infrastructure): pinned against the golden
vectors the reference itself produced (tests/golden/make_golden.py), plus
internal consistency of its truth mode and of the COCG restatement."""

import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle.oracle import OraclePlan, cocg_step, rel_l2
from paper_1912_03312_b200 import fixtures
from paper_1912_03312_b200.types import PartialFractionApproximation

# fp64 floor of the reference path: weights up to 1.7e7 cancel to O(1), so two
# correct fp64 implementations differ by ~1e-9 per step
FLOOR_PER_STEP = 2.5e-9


@pytest.mark.parametrize("name", golden_names())
def test_oracle_reference_mode_matches_reference(name):
    d, sysm, ap = load_golden(name)
    p = OraclePlan(sysm, ap, float(d["tau"]))
    assert p.status == 0
    if int(d["bandwidth"]) > 0:
        assert p.bandwidth == int(d["bandwidth"])
    u = d["u0"]
    for k in range(d["steps"].shape[0]):
        u = p.step(u)
        assert rel_l2(u, d["steps"][k]) <= FLOOR_PER_STEP * (k + 1), (name, k)


@pytest.mark.parametrize("name", ["cfg1_k32", "fem_p2", "pencil_0", "p1_2d_m16"])
def test_truth_mode_is_converged_and_near_reference(name):
    d, sysm, ap = load_golden(name)
    p = OraclePlan(sysm, ap, float(d["tau"]))
    ut = p.step(d["u0"], "truth")
    assert p.last_correction < 1e-20
    assert rel_l2(ut, d["steps"][0]) <= FLOOR_PER_STEP


def test_truth_per_shift_residuals():
    d, sysm, ap = load_golden("cfg1_k32")
    p = OraclePlan(sysm, ap, float(d["tau"]))
    rhs = p.rhs(d["u0"])
    for j in range(ap.K):
        x = p.solve(j, rhs)
        assert p.rel_residual(j, rhs, x) < 1e-12


def test_oracle_rhs_is_i_B_u():
    d, sysm, ap = load_golden("fem_p2")
    p = OraclePlan(sysm, ap, float(d["tau"]))
    u = d["u0"]
    np.testing.assert_array_equal(p.rhs(u), 1j * (sysm.B @ u))


def test_oracle_singular_shift_detected(flagship):
    from scipy.sparse import csr_matrix, identity
    from paper_1912_03312_b200.types import SystemMatrices
    s0 = complex(flagship.shifts[3])
    sysm = SystemMatrices(A=csr_matrix(np.array([[1j * s0]]).real), B=identity(1, format="csr"), n_dof=1)
    # real part only: not singular
    assert OraclePlan(sysm, flagship, 1.0).status == 0
    sysz = SystemMatrices(A=csr_matrix((2, 2)), B=csr_matrix((2, 2)), n_dof=2)
    assert OraclePlan(sysz, flagship, 1.0).status == 2


def test_cocg_restatement_matches_banded_truth():
    cfg = fixtures.config3(m=24)
    ap = fixtures.load_poles(16)
    tau = 2e-3
    p = OraclePlan(cfg.system, ap, tau)
    truth = p.step(cfg.u0, "truth")
    u1, iters = cocg_step(cfg.system, ap, tau, cfg.u0, tol=1e-12, refine=1, tol_refine=1e-8)
    assert rel_l2(u1, truth) <= 1e-8
    assert np.all(iters > 0)


def test_zero_state_exact_zero():
    d, sysm, ap = load_golden("cfg1_k16")
    p = OraclePlan(sysm, ap, float(d["tau"]))
    assert np.all(p.step(np.zeros(sysm.n_dof, complex)) == 0)


def test_threads_do_not_change_the_answer():
    d, sysm, ap = load_golden("cfg1_k32")
    a = OraclePlan(sysm, ap, float(d["tau"]), nthreads=1).step(d["u0"])
    b = OraclePlan(sysm, ap, float(d["tau"]), nthreads=4).step(d["u0"])
    np.testing.assert_array_equal(a, b)
