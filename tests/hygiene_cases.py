"""Workloads for tests/test_gpu_hygiene.py (run in a subprocess so that
REXI_POISON is read when the library loads): python hygiene_cases.py OUT.npz"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
os.environ.setdefault("REXI_FIXTURE_HOST", "1")
import numpy as np  # noqa: E402

from conftest import load_golden  # noqa: E402
from paper_1912_03312_b200 import (chebyshev_prepare, chebyshev_run, fixtures, rexi_prepare,  # noqa: E402
                                   rexi_run, rexi_step, spectral_radius_estimate)


def cases():
    out = {}
    cfg = fixtures.config1()                                     # persistent cluster loop
    stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
    out["cfg1_persist"] = rexi_run(stp, cfg.u0, 3)
    out["cfg1_observer"] = np.stack([u for u in _observed(stp, cfg.u0, 2)])
    stp.close()
    cfg = fixtures.config2(m=20001)                              # TMA / mbarrier level-0 kernels, refined
    for refine in (0, 1):
        stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True,
                           refine=refine)
        out[f"cfg2s_r{refine}"] = rexi_run(stp, cfg.u0, 2)
        out[f"cfg2s_r{refine}_solve"] = stp.plans[0].solve_host(1j * (cfg.system.B @ cfg.u0))[:3]
        stp.close()
    cfg = fixtures.stiffness_matched(3, 32)                      # COCG: staged spmv, repacks, classes
    stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
    out["cocg2d"] = rexi_run(stp, cfg.u0, 2)
    stp.close()
    cfg = fixtures.stiffness_matched(5, 8)
    stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
    out["cocg3d"] = rexi_step(stp, cfg.u0)
    stp.close()
    d, sysm, ap = load_golden("harness_p2")                      # band solver (staged kernels)
    for refine in (0, 1):
        stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True,
                           refine=refine)
        out[f"band_r{refine}"] = rexi_run(stp, d["u0"], 2)
        stp.close()
    cfg = fixtures.config3(m=32)                                 # pencil: CG on B, power iteration, Clenshaw
    est = spectral_radius_estimate(cfg.system)
    out["sr"] = np.array([float(est), est.iterations])
    cs = chebyshev_prepare(cfg.system, cfg.tau, sr_value=float(est), override_admissibility=True)
    out["cheb"] = chebyshev_run(cs, cfg.system, cfg.u0, 2)
    return out


def _observed(stp, u0, n):
    seen = []
    rexi_run(stp, u0, n, observer=lambda k, t, u: seen.append(u.copy()))
    return seen


if __name__ == "__main__":
    res = cases()
    again = cases()                     # the same process, again: run-to-run determinism
    for k in res:
        assert np.array_equal(res[k], again[k]), f"{k}: not bitwise reproducible within a process"
    np.savez(sys.argv[1], **res)
    print("ok", len(res))
