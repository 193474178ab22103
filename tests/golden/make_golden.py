"""Generate the frozen pole sets and the reference golden vectors.

Run IN THE BUILD CONTAINER (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from
``/root/reference/pkg/src`` and writes

* ``paper_1912_03312_b200/poles/*.json`` -- pole/weight sets through the
  reference's own ``approx_to_json`` (17 significant digits, bit-exact):
  the flagship ``faber_cf(JoukowskiMap(10))`` (K = 16, the reference's
  test fixture ``conftest.py:7-10``) and the K = 32/64/128 ensembles of
  SURVEY.md A.3 (concatenated degree-16 outputs, weights / n, R1 = min).
* ``tests/golden/*.npz`` -- inputs and the reference's outputs of
  ``rexi_prepare``/``rexi_run``/``rexi_step`` (``integrate.py:143-245``)
  for small systems: scalar Dahlquist systems, the reference's own ``fem``
  P2 fixture (``test_integrate.py:56-68``), random dense pencils
  (``test_integrate.py:71-78``), config 1 (1D P1, K = 32 and 16), and small
  2D/3D P1 pencils (which the reference runs through its dense fallback).

Nothing on the GPU box reads ``/root/reference``; only these files travel.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import rexiprop  # noqa: E402  (the reference, imported unchanged)
from rexiprop import (JoukowskiMap, PartialFractionApproximation, approx_to_json,  # noqa: E402
                      faber_cf, sup_error_on_interval)
from rexiprop.integrate import rexi_prepare, rexi_run, rexi_step  # noqa: E402
from rexiprop.spatial import (PhysicalConstants, PotentialSpec, SystemMatrices,  # noqa: E402
                              WavePacketParams, assemble_system, build_mesh,
                              project_initial, spectral_radius_estimate)

from paper_1912_03312_b200 import fixtures  # noqa: E402

POLE_DIR = os.path.join(ROOT, "paper_1912_03312_b200", "poles")

ENSEMBLES = {
    32: [10.0, 10.5],
    64: [10.0, 10.25, 10.5, 11.5],
    128: [9.5, 9.75, 10.0, 10.25, 10.5, 11.0, 11.5, 12.0],
}


def ensemble(radii):
    parts = [faber_cf(JoukowskiMap(r)) for r in radii]
    n = len(parts)
    shifts = np.concatenate([p.shifts for p in parts])
    weights = np.concatenate([p.weights for p in parts]) / n
    a = PartialFractionApproximation(shifts=shifts, weights=weights,
                                     domain_radius=min(radii), sup_error=0.0)
    return PartialFractionApproximation(
        shifts=a.shifts, weights=a.weights, domain_radius=a.domain_radius,
        sup_error=sup_error_on_interval(a))


def write_poles():
    os.makedirs(POLE_DIR, exist_ok=True)
    flag = faber_cf(JoukowskiMap(10.0))
    sets = {16: flag}
    for k, radii in ENSEMBLES.items():
        sets[k] = ensemble(radii)
        assert sets[k].K == k, (k, sets[k].K)
    for k, a in sets.items():
        with open(os.path.join(POLE_DIR, fixtures.POLE_SETS[k]), "w") as fh:
            fh.write(approx_to_json(a))
        print(f"poles K={k} R1={a.domain_radius} sup={a.sup_error:.3e}")
    return sets


def csr_arrays(prefix, mat):
    mat = mat.tocsr()
    return {f"{prefix}_indptr": mat.indptr.astype(np.int64),
            f"{prefix}_indices": mat.indices.astype(np.int64),
            f"{prefix}_data": mat.data,
            f"{prefix}_shape": np.array(mat.shape)}


def run_ref(name, sysm, approx, tau, u0, n_steps, sr, workers=1, extra=None):
    """Reference outputs after every step, through its public API."""
    stp = rexi_prepare(sysm, approx, tau, sr_value=sr, workers=workers,
                       override_admissibility=True)
    seen = []
    rexi_run(stp, u0, n_steps, observer=lambda k, t, u: seen.append(u.copy()))
    stp.close()
    out = {"tau": np.float64(tau), "sr": np.float64(sr), "u0": np.asarray(u0, complex),
           "steps": np.stack(seen), "shifts": approx.shifts, "weights": approx.weights,
           "R1": np.float64(approx.domain_radius),
           "admissibility_ratio": np.float64(stp.admissibility_ratio),
           "bandwidth": np.int64(-1 if stp.bandwidth is None else stp.bandwidth)}
    out.update(csr_arrays("A", sysm.A))
    out.update(csr_arrays("B", sysm.B))
    if extra:
        out.update(extra)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"golden {name}: n={sysm.n_dof} K={approx.K} steps={n_steps}")


def run_ref_cheb(name, sysm, u0, n_steps, degree=26, radius=10.0):
    """Reference spectral_radius_estimate + chebyshev_prepare/chebyshev_run
    (spatial.py:314-344, integrate.py:257-377) on one system."""
    from rexiprop.integrate import chebyshev_coeffs, chebyshev_prepare, chebyshev_run
    est = spectral_radius_estimate(sysm)
    tau = 0.9 * radius / (1.05 * float(est))
    stp = chebyshev_prepare(sysm, tau, degree=degree, radius=radius, sr_value=float(est))
    seen = []
    chebyshev_run(stp, sysm, u0, n_steps, observer=lambda k, t, u: seen.append(u.copy()))
    cc = chebyshev_coeffs(radius, degree)
    out = {"tau": np.float64(tau), "radius": np.float64(radius), "degree": np.int64(degree),
           "u0": np.asarray(u0, complex), "steps": np.stack(seen), "coeffs": cc.coeffs,
           "sup_error": np.float64(cc.sup_error), "sr": np.float64(float(est)),
           "sr_iterations": np.int64(est.iterations), "sr_converged": np.bool_(est.converged),
           "admissibility_ratio": np.float64(stp.admissibility_ratio)}
    out.update(csr_arrays("A", sysm.A))
    out.update(csr_arrays("B", sysm.B))
    np.savez_compressed(os.path.join(HERE, f"cheb_{name}.npz"), **out)
    print(f"golden cheb_{name}: n={sysm.n_dof} sr={float(est):.6e} its={est.iterations} "
          f"conv={est.converged} steps={n_steps}")


def cheb_main():
    """Golden vectors of the 8(f) rows: spectral radius + Chebyshev stepper."""
    consts = PhysicalConstants()
    mesh = build_mesh(-12.0, 12.0, 64)
    sysm = assemble_system(mesh, PotentialSpec(kind="step", v_max=1.0, c_barr=2.0), consts)
    u0 = project_initial(mesh, WavePacketParams(r_bar=-4.0, p_bar=2.0, sigma=1.0), consts, sysm.B)
    run_ref_cheb("fem_p2", sysm, u0, 3)
    c1 = fixtures.config1()
    run_ref_cheb("cfg1", c1.system, c1.u0, 3)
    c3 = fixtures.config3(m=16)
    run_ref_cheb("p1_2d_m16", c3.system, c3.u0, 2)
    c5 = fixtures.config5(m=8)
    run_ref_cheb("p1_3d_m8", c5.system, c5.u0, 2)
    from scipy.sparse import csr_matrix
    rng = np.random.default_rng(13)
    n = 24
    m0 = rng.standard_normal((n, n))
    r0 = rng.standard_normal((n, n))
    sysn = SystemMatrices(A=csr_matrix(0.5 * (m0 + m0.T)), B=csr_matrix(r0 @ r0.T + n * np.eye(n)),
                          n_dof=n)
    run_ref_cheb("pencil", sysn, rng.standard_normal(n) + 1j * rng.standard_normal(n), 2)


def harness_main():
    """The reference harness's default tunneling experiment (harness.py:68-90,
    205-213): 1D P2, 4000 elements, step barrier, flagship K=16 poles, dt=5e-5;
    a few REXI steps through the reference (the P2 pencil is pentadiagonal)."""
    from rexiprop.harness import ExperimentConfig, _build_experiment
    cfg = ExperimentConfig()
    mesh, consts, system, u0 = _build_experiment(cfg)
    flag = faber_cf(JoukowskiMap(10.0))
    sr = float(spectral_radius_estimate(system))
    run_ref("harness_p2", system, flag, cfg.dt, u0, 3, sr)


def main():
    sets = write_poles()
    flag = sets[16]

    # scalar Dahlquist systems (test_integrate.py:43-48,230-242,277-285)
    from scipy.sparse import csr_matrix, identity
    for omega in (-9.5, -1.0, 0.3, 1.0, 7.25):
        sysm = SystemMatrices(A=csr_matrix(np.array([[omega]])),
                              B=identity(1, format="csr"), n_dof=1)
        run_ref(f"scalar_{omega:+.2f}".replace(".", "p"), sysm, flag, 1.0,
                np.array([1.0 + 0.0j]), 50 if omega == 1.0 else 1, abs(omega))

    # the reference's own fem fixture (test_integrate.py:56-68): P2, pentadiagonal
    consts = PhysicalConstants()
    mesh = build_mesh(-12.0, 12.0, 64)
    sysm = assemble_system(mesh, PotentialSpec(kind="step", v_max=1.0, c_barr=2.0), consts)
    sr = float(spectral_radius_estimate(sysm))
    u0 = project_initial(mesh, WavePacketParams(r_bar=-4.0, p_bar=2.0, sigma=1.0), consts, sysm.B)
    run_ref("fem_p2", sysm, flag, 0.02, u0, 4, sr)

    # random dense pencils (test_integrate.py:71-78, 464-477)
    import scipy.linalg as sla
    rng = np.random.default_rng(11)
    for i in range(3):
        n = 32
        m0 = rng.standard_normal((n, n))
        a_d = 0.5 * (m0 + m0.T)
        r0 = rng.standard_normal((n, n))
        b_d = r0 @ r0.T + n * np.eye(n)
        sysn = SystemMatrices(A=csr_matrix(a_d), B=csr_matrix(b_d), n_dof=n)
        srn = float(np.max(np.abs(sla.eigh(a_d, b_d, eigvals_only=True))))
        tau = 0.9 * 10.0 / (1.05 * srn)
        u = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        run_ref(f"pencil_{i}", sysn, flag, tau, u, 1, srn)

    # config 1 (1D P1, 1023 DOF) with the K=32 ensemble and the flagship
    c1 = fixtures.config1()
    sr_ref = float(spectral_radius_estimate(c1.system))
    run_ref("cfg1_k32", c1.system, sets[32], c1.tau, c1.u0, c1.n_steps, c1.sr,
            extra={"sr_reference_estimator": np.float64(sr_ref)})
    run_ref("cfg1_k16", c1.system, flag, c1.tau, c1.u0, c1.n_steps, c1.sr)

    # small 2D / 3D P1 pencils at the config stiffness scale (dense fallback in the reference)
    c3 = fixtures.config3(m=16)
    run_ref("p1_2d_m16", c3.system, flag, 2e-3, c3.u0, 2, c3.sr)
    c5 = fixtures.config5(m=8)
    run_ref("p1_3d_m8", c5.system, flag, 1e-2, c5.u0, 2, c5.sr)


if __name__ == "__main__":
    if "--cheb" in sys.argv:
        cheb_main()
    elif "--harness" in sys.argv:
        harness_main()
    else:
        main()
