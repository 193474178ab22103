"""GPU, full BASELINE sizes of the 2D/3D configs (3: 1M DOF K=64, 5: 2M DOF
K=64), where no CPU truth is affordable: size-independent properties.

* solver: the true relative residual ||b - S_j x_j|| / ||b|| of the shifts
  that carry the largest weights |beta_j| is <= 1e-12 (north_star), the
  residual evaluated with 80-bit products and sums so the check's own
  rounding stays far below the bound;
* linearity of the step (test_integrate.py:252-265's property) to 1e-8;
* the step does not grow the B-norm of the physical packet beyond the
  pole set's sup error (test_integrate.py:308-315's property).
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _residual_ld(sysm, tau, sigma, b, x):
    """||b - (tau A - 1j sigma B) x|| / ||b|| with longdouble products/sums;
    the shifted entries are formed in fp64 exactly as the reference does
    (integrate.py:171)."""
    A, B = sysm.A.tocsr(), sysm.B.tocsr()
    assert np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)
    ta = tau * A.data
    re = ta + sigma.imag * B.data          # fl(fl(tau a) + fl(Im sigma b))
    im = -(sigma.real * B.data)
    xr = x.real[A.indices].astype(np.longdouble)
    xi = x.imag[A.indices].astype(np.longdouble)
    er, ei = re.astype(np.longdouble), im.astype(np.longdouble)
    pr = er * xr - ei * xi
    pi = er * xi + ei * xr
    starts = A.indptr[:-1]
    sr = np.add.reduceat(pr, starts)
    si = np.add.reduceat(pi, starts)
    rr = b.real.astype(np.longdouble) - sr
    ri = b.imag.astype(np.longdouble) - si
    num = np.sqrt(np.sum(rr * rr + ri * ri))
    den = np.sqrt(np.sum(b.real.astype(np.longdouble) ** 2 + b.imag.astype(np.longdouble) ** 2))
    return float(num / den)


@pytest.mark.parametrize("c", [3, 5])
def test_full_size_cocg_properties(c):
    from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_step
    cfg = fixtures.build_config(c)
    sysm, ap, tau = cfg.system, cfg.approx, cfg.tau
    stp = rexi_prepare(sysm, ap, tau, sr_value=cfg.sr, override_admissibility=True)
    assert stp.solver == "cocg"
    # solver residuals of the heaviest shifts
    b = 1j * (sysm.B @ cfg.u0)
    xs = stp.plans[0].solve_host(b)
    heavy = np.argsort(-np.abs(np.asarray(ap.weights)))[:3]
    for j in heavy:
        assert _residual_ld(sysm, tau, complex(ap.shifts[j]), b, xs[j]) <= 1e-12, j
    del xs
    # linearity
    u, v = cfg.u0, np.conj(cfg.u0)
    a = 0.5 - 2.0j
    lhs = rexi_step(stp, u + a * v)
    rhs = rexi_step(stp, u) + a * rexi_step(stp, v)
    assert np.linalg.norm(lhs - rhs) <= 1e-8 * np.linalg.norm(rhs)
    # B-norm of the packet
    u1 = rexi_step(stp, u)
    bn0 = np.sqrt(np.vdot(u, sysm.B @ u).real)
    bn1 = np.sqrt(np.vdot(u1, sysm.B @ u1).real)
    assert np.all(np.isfinite(u1))
    assert bn1 <= bn0 * (1.0 + ap.sup_error + 1e-9)
    stp.close()


@pytest.mark.parametrize("c", [3, 4, 5])
def test_full_size_step1_vs_cpu_truth(c):
    """Step 1 of the FULL-SIZE config c (1M / 4.2M / 2M DOF, K = 64 / 128 / 64,
    BASELINE tau)
    against the CPU truth restatement (oracle.cocg_truth_step: COCG refined
    against double-double residuals to 1e-22, exact dd sum), precomputed by
    tests/golden/make_fullsize.py and kept as u1 at 8192 seeded rows plus 4
    seeded projections <w, u1> of the whole vector."""
    import os
    import sys
    from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_step
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    from fullsize_probes import probes
    path = os.path.join(here, "fullsize", f"cfg{c}_step1.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tests/golden/make_fullsize.py {c}: hours of CPU)")
    g = np.load(path)
    cfg = fixtures.build_config(c)
    n = cfg.system.n_dof
    assert n == int(g["n"]) and cfg.tau == float(g["tau"])
    assert abs(np.linalg.norm(cfg.u0) - float(g["norm_u0"])) <= 1e-13 * float(g["norm_u0"])
    stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
    u1 = rexi_step(stp, cfg.u0)
    stp.close()
    rows, w = probes(c, n)
    assert np.array_equal(rows, g["rows"])
    u_ref = g["u1_rows"]
    e_rows = np.linalg.norm(u1[rows] - u_ref) / np.linalg.norm(u_ref)
    proj = w @ u1
    e_proj = np.abs(proj - g["proj"]) / np.abs(g["proj"])
    e_norm = abs(np.linalg.norm(u1) - float(g["norm_u1"])) / float(g["norm_u1"])
    assert e_rows <= 1e-8, e_rows          # north_star: rel-L2 <= 1e-8
    assert np.all(e_proj <= 1e-8), e_proj
    assert e_norm <= 1e-9, e_norm
