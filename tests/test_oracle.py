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


def _pencil_1d(n, p2=False):
    """small 1D pencil: P1 tridiagonal, or a pentadiagonal stand-in with the
    P2 band structure (kl = ku = 2)"""
    from scipy.sparse import diags
    from paper_1912_03312_b200.types import SystemMatrices
    h = 1.0 / (n + 1)
    x = np.linspace(h, 1 - h, n)
    if p2:
        A = diags([0.1 / h * np.ones(n - 2), -0.7 / h * np.ones(n - 1), 1.4 / h + 5 * h * x ** 2,
                   -0.7 / h * np.ones(n - 1), 0.1 / h * np.ones(n - 2)], [-2, -1, 0, 1, 2]).tocsr()
        B = diags([-h / 30 * np.ones(n - 2), h / 15 * np.ones(n - 1), 8 * h / 15 * np.ones(n),
                   h / 15 * np.ones(n - 1), -h / 30 * np.ones(n - 2)], [-2, -1, 0, 1, 2]).tocsr()
    else:
        A = diags([-0.5 / h * np.ones(n - 1), 1.0 / h + 5 * h * x ** 2, -0.5 / h * np.ones(n - 1)],
                  [-1, 0, 1]).tocsr()
        B = diags([h / 6 * np.ones(n - 1), 2 * h / 3 * np.ones(n), h / 6 * np.ones(n - 1)], [-1, 0, 1]).tocsr()
    return SystemMatrices(A=A, B=B, n_dof=n)


def _reference_screen(sysm, sigma, tau):
    """solvers.py:42-69 with scipy's own zgbtrf (the reference's LAPACK):
    (min|U_ii|, max|U_ii|, info)"""
    from scipy.linalg import lapack
    mat = (tau * sysm.A - (1j * sigma) * sysm.B).tocsr()
    coo = mat.tocoo()
    d = coo.col - coo.row
    kl, ku = int(max(0, -d.min())), int(max(0, d.max()))
    n = mat.shape[0]
    ab = np.zeros((2 * kl + ku + 1, n), dtype=complex, order="F")
    for dd in range(-kl, ku + 1):
        ab[kl + ku - dd, max(dd, 0): n + min(dd, 0)] = mat.diagonal(dd)
    lu, piv, info = lapack.zgbtrf(ab, kl, ku)
    u = np.abs(lu[kl + ku, :])
    return u.min(), u.max(), info


def screen_cases():
    """shifts at, near and away from an eigenvalue of tau B^-1 A (sigma =
    -i tau lambda (1 + delta) makes tau A - i sigma B = tau (A - lambda (1 +
    delta) B)), plus ordinary REXI poles"""
    from scipy.linalg import eigh
    out = []
    for p2 in (False, True):
        sysm = _pencil_1d(40, p2)
        lam = eigh(sysm.A.toarray(), sysm.B.toarray(), eigvals_only=True)
        tau = 0.01
        for kidx in (0, 7, 39):
            for delta in (0.0, 1e-9, 1e-4):
                out.append((sysm, tau, complex(0.0, -tau * lam[kidx] * (1 + delta))))
        for s in fixtures.load_poles(16).shifts[:4]:
            out.append((sysm, tau, complex(s)))
    return out


def test_oracle_screen_matches_reference_zgbtrf():
    """the oracle's band LU restatement gives the reference's screen data
    (scipy zgbtrf, solvers.py:52-69) on tridiagonal and pentadiagonal
    pencils, including shifts on an eigenvalue"""
    from paper_1912_03312_b200.types import PartialFractionApproximation
    for sysm, tau, sigma in screen_cases():
        ap = PartialFractionApproximation(np.array([sigma]), np.array([1.0 + 0j]), 10.0, 0.0)
        umin, umax, info = OraclePlan(sysm, ap, tau).screen()
        rmin, rmax, rinfo = _reference_screen(sysm, sigma, tau)
        assert int(info[0]) == int(rinfo)
        assert abs(umax[0] - rmax) <= 1e-12 * rmax
        ref_bad = rinfo > 0 or rmin < 1e-14 * rmax
        bad = info[0] > 0 or umin[0] < 1e-14 * umax[0]
        assert bad == ref_bad, (sigma, umin[0] / umax[0], rmin / rmax)
        if rmin > 1e-12 * rmax:      # away from the rounding floor the ratios agree closely
            assert abs(umin[0] - rmin) <= 1e-6 * rmin
