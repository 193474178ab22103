"""Small cases for compute-sanitizer (scripts/sanitize.sh): each exercises
one family of kernels with its synchronisation (mbarriers + cp.async.bulk,
cluster barriers + DSMEM, the COCG atomic work claims and last-CTA finishes).

    python scripts/sanitize_cases.py persist|refined1d|plain1d|chain|cocg2d|cocg3d|pencil
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("REXI_FIXTURE_HOST", "1")     # keep the assembly kernels out of the way
import numpy as np  # noqa: E402

from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_run, rexi_step  # noqa: E402


def case(name):
    if name == "persist":           # cfg 1: one thread-block-cluster launch, DSMEM, cluster barriers
        cfg = fixtures.config1()
        stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
        assert stp.plans[0].info.persistent > 0
        u = rexi_run(stp, cfg.u0, 3)
    elif name in ("refined1d", "plain1d", "chain"):
        # 1D multi-kernel path: TMA bulk copies on mbarriers (S1, K2, K3, k_lv_tma,
        # k_lv32), the level chain cluster launch; m ~ 20k rows, K = 64
        cfg = fixtures.config2(m=20001)
        if name == "chain":
            os.environ.pop("REXI_NO_CHAIN", None)
        stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True,
                           refine=1 if name != "plain1d" else 0)
        u = rexi_step(stp, cfg.u0)
        u = rexi_step(stp, u)
    elif name == "cocg2d":          # staged spmv (bulk copies), finishes, repacks, stencil classes
        cfg = fixtures.stiffness_matched(3, 32)
        stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
        u = rexi_step(stp, cfg.u0)
    elif name == "cocg3d":
        cfg = fixtures.stiffness_matched(5, 8)
        stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
        u = rexi_step(stp, cfg.u0)
    elif name == "pencil":          # CG on B, power iteration, Clenshaw
        from paper_1912_03312_b200 import chebyshev_prepare, chebyshev_run, spectral_radius_estimate
        cfg = fixtures.config3(m=32)
        est = spectral_radius_estimate(cfg.system)
        cs = chebyshev_prepare(cfg.system, cfg.tau, sr_value=float(est), override_admissibility=True)
        u = chebyshev_run(cs, cfg.system, cfg.u0, 2)
        stp = None
    else:
        raise SystemExit(f"unknown case {name}")
    if stp is not None:
        stp.close()
    assert np.all(np.isfinite(u))
    print(f"{name}: ok")


if __name__ == "__main__":
    case(sys.argv[1])
