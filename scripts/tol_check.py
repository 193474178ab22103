"""Accuracy of the current COCG tolerance knobs (REXI_COCG_*) at BASELINE
conditioning: stiffness-matched cfg 3 / 4 / 5 (fixtures.stiffness_matched)
against the truth oracle every step, and the worst per-shift true relative
residual (double-double) of the first solve set (north_star: <= 1e-12)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_run
from oracle.oracle import OraclePlan, rel_l2
out = []
for idx, m, steps in ((3, 64, 4), (4, 64, 3), (5, 16, 3)):
    cfg = fixtures.stiffness_matched(idx, m)
    stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
    seen = []
    rexi_run(stp, cfg.u0, steps, observer=lambda k, t, u: seen.append(u.copy()))
    orc = OraclePlan(cfg.system, cfg.approx, cfg.tau)
    ut = cfg.u0
    err = 0.0
    for u in seen:
        ut = orc.step(ut, "truth")
        err = max(err, rel_l2(u, ut))
    rhs = orc.rhs(cfg.u0)
    xs = stp.plans[0].solve_host(rhs)
    res = max(orc.rel_residual(j, rhs, xs[j]) for j in range(cfg.approx.K))
    stp.close()
    out.append(f"cfg{idx}@m{m}: err {err:.2e} res {res:.2e}")
print(" | ".join(out))
