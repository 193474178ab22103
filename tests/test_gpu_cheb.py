"""GPU: the 8(f) rows through the public API -- spectral_radius_estimate
(ref spatial.py:314-344) and the Chebyshev/Clenshaw stepper (ref
integrate.py:257-377) -- against the reference's own outputs
(tests/golden/cheb_*.npz) and the numpy/scipy oracles."""
import numpy as np
import pytest

from conftest import cheb_names, load_cheb, load_golden

pytestmark = pytest.mark.gpu


def _rel(x, y):
    return float(np.linalg.norm(np.asarray(x) - np.asarray(y)) / np.linalg.norm(y))


@pytest.mark.parametrize("name", cheb_names())
def test_spectral_radius_matches_reference(name):
    from paper_1912_03312_b200 import spectral_radius_estimate
    d, sysm = load_cheb(name)
    est = spectral_radius_estimate(sysm)
    assert est.converged == bool(d["sr_converged"])
    assert abs(est.iterations - int(d["sr_iterations"])) <= 1
    assert abs(float(est) - float(d["sr"])) <= 1e-9 * float(d["sr"])
    assert "SpectralRadiusEstimate(" in repr(est)


@pytest.mark.parametrize("name", cheb_names())
def test_chebyshev_run_matches_reference_every_step(name):
    from paper_1912_03312_b200 import chebyshev_prepare, chebyshev_run
    d, sysm = load_cheb(name)
    stp = chebyshev_prepare(sysm, float(d["tau"]), degree=int(d["degree"]), radius=float(d["radius"]),
                            sr_value=float(d["sr"]))
    assert abs(stp.admissibility_ratio - float(d["admissibility_ratio"])) <= 1e-15
    np.testing.assert_allclose(stp.coeffs, d["coeffs"], rtol=0, atol=1e-15)
    seen = []
    chebyshev_run(stp, sysm, d["u0"], d["steps"].shape[0],
                  observer=lambda k, t, u: seen.append((k, t, u.copy())))
    for k, (kk, t, u) in enumerate(seen):
        assert kk == k + 1 and t == pytest.approx((k + 1) * float(d["tau"]))
        assert _rel(u, d["steps"][k]) <= 1e-11, (name, k, _rel(u, d["steps"][k]))
    # device-resident run (no observer) gives the same answer
    u_all = chebyshev_run(stp, sysm, d["u0"], d["steps"].shape[0])
    assert _rel(u_all, d["steps"][-1]) <= 1e-11
    stp.close()


def test_chebyshev_step_is_repeatable_bitwise():
    from paper_1912_03312_b200 import chebyshev_prepare, chebyshev_step
    d, sysm = load_cheb("cheb_cfg1")
    stp = chebyshev_prepare(sysm, float(d["tau"]), sr_value=float(d["sr"]))
    a = chebyshev_step(stp, sysm, d["u0"])
    b = chebyshev_step(stp, sysm, d["u0"])
    assert np.array_equal(a, b)
    assert stp.stats["cg_iters_max"] > 0 and stp.timers["local"] > 0
    stp.close()


def test_chebyshev_run_contract():
    from paper_1912_03312_b200 import AdmissibilityError, chebyshev_prepare, chebyshev_run
    d, sysm = load_cheb("cheb_cfg1")
    tau_bad = 3.0 * float(d["tau"])
    stp = chebyshev_prepare(sysm, tau_bad, sr_value=float(d["sr"]))
    assert not stp.admissible
    with pytest.raises(AdmissibilityError, match="max_step_size"):
        chebyshev_run(stp, sysm, d["u0"], 1)
    with pytest.raises(ValueError):
        chebyshev_run(stp, sysm, d["u0"], -1)
    u0 = chebyshev_run(stp, sysm, d["u0"], 0)
    assert np.array_equal(u0, d["u0"]) and u0 is not d["u0"]
    stp.close()
    stp = chebyshev_prepare(sysm, tau_bad, sr_value=float(d["sr"]), override_admissibility=True)
    chebyshev_run(stp, sysm, d["u0"], 1)
    assert stp.override_used
    stp.close()
    with pytest.raises(ValueError):
        chebyshev_prepare(sysm, 0.0, sr_value=1.0)


def test_chebyshev_torch_roundtrip():
    import torch
    from paper_1912_03312_b200 import chebyshev_prepare, chebyshev_run
    d, sysm = load_cheb("cheb_p1_2d_m16")
    stp = chebyshev_prepare(sysm, float(d["tau"]), sr_value=float(d["sr"]))
    ut = torch.from_numpy(d["u0"]).cuda()
    out = chebyshev_run(stp, sysm, ut, d["steps"].shape[0])
    assert out.is_cuda and out.dtype == torch.complex128
    assert _rel(out.cpu().numpy(), d["steps"][-1]) <= 1e-11
    stp.close()


@pytest.mark.parametrize("name", ["cheb_fem_p2", "cheb_p1_3d_m8", "cheb_pencil"])
def test_b_solve_residual(name):
    from paper_1912_03312_b200 import chebyshev_prepare
    d, sysm = load_cheb(name)
    stp = chebyshev_prepare(sysm, float(d["tau"]), sr_value=float(d["sr"]))
    rng = np.random.default_rng(5)
    b = rng.standard_normal(sysm.n_dof) + 1j * rng.standard_normal(sysm.n_dof)
    x = stp.B_factorization.solve(b)
    assert np.linalg.norm(sysm.B @ x - b) <= 1e-13 * np.linalg.norm(b)
    assert np.array_equal(stp.B_factorization.solve(np.zeros_like(b)), np.zeros_like(b))
    stp.close()


def test_rexi_prepare_estimates_sr_on_gpu():
    from paper_1912_03312_b200 import rexi_prepare
    d, sysm, ap = load_golden("cfg1_k32")
    stp = rexi_prepare(sysm, ap, float(d["tau"]), override_admissibility=True)
    ref = float(d["sr_reference_estimator"])
    assert abs(stp.sr_value - ref) <= 1e-9 * ref
    stp.close()


def test_non_spd_b_rejected():
    from scipy.sparse import csr_matrix
    from paper_1912_03312_b200 import SolverError, SystemMatrices, spectral_radius_estimate
    A = csr_matrix(np.diag([1.0, 2.0, 3.0]))
    B = csr_matrix(np.diag([1.0, -1.0, 1.0]))
    with pytest.raises(SolverError):
        spectral_radius_estimate(SystemMatrices(A, B, 3))


@pytest.mark.slow
def test_spectral_radius_full_size_2d():
    """Config 3 (1M DOF 2D): the reference's estimator needs a dense LU here
    (solvers.py:108-115); the GPU power iteration runs in seconds."""
    from paper_1912_03312_b200 import fixtures, spectral_radius_estimate
    cfg = fixtures.build_config(3)
    est = spectral_radius_estimate(cfg.system)
    assert 0.5 * cfg.sr <= float(est) <= 1.05 * cfg.sr


def test_chebyshev_torch_input_from_a_side_stream():
    """a CUDA tensor produced on a non-default torch stream is consumed after
    that stream's work (the pencil's stream waits on torch's current one)"""
    import torch
    from paper_1912_03312_b200 import chebyshev_prepare, chebyshev_step
    d, sysm = load_cheb("cheb_cfg1")
    cs = chebyshev_prepare(sysm, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True)
    ref = chebyshev_step(cs, sysm, d["u0"])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        big = torch.randn(1 << 24, device="cuda")
        for _ in range(20):
            big = big * 1.0000001          # keep the side stream busy
        u = torch.from_numpy(d["u0"]).to("cuda", non_blocking=False) * 1.0
        out = chebyshev_step(cs, sysm, u)
        torch.cuda.current_stream().synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)
