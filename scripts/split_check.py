"""Accuracy of the current COCG tolerance knobs (REXI_COCG_*): small 2D/3D
cases vs the truth oracle, and the worst per-shift true residual (2D m=32)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_step
from oracle.oracle import OraclePlan, rel_l2
errs = []
for cfg in (fixtures.config3(m=48), fixtures.config5(m=12), fixtures.config4(m=48)):
    stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
    u1 = rexi_step(stp, cfg.u0); stp.close()
    errs.append(rel_l2(u1, OraclePlan(cfg.system, cfg.approx, cfg.tau).step(cfg.u0, "truth")))
cfg = fixtures.config3(m=32)
stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
orc = OraclePlan(cfg.system, cfg.approx, cfg.tau)
rhs = orc.rhs(cfg.u0)
xs = stp.plans[0].solve_host(rhs); stp.close()
res = max(orc.rel_residual(j, rhs, xs[j]) for j in range(cfg.approx.K))
print("vs truth (2D m48, 3D m12, 2D-disordered m48): " + ", ".join(f"{e:.2e}" for e in errs) + f" | max shift residual {res:.2e}")
