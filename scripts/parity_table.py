"""Per-config parity numbers for DESIGN.md: max over steps of rel-L2 vs the
truth oracle for the GPU path and for the reference's algorithm (its C
restatement, or the reference's own stored outputs), plus the worst
per-shift true residual where the oracle can form it.
    python scripts/parity_table.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests")); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np
from conftest import load_golden
from oracle.oracle import OraclePlan, rel_l2
from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_run, rexi_step


def chain(cfg, steps, **kw):
    stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True, **kw)
    seen = []
    rexi_run(stp, cfg.u0, steps, observer=lambda k, t, u: seen.append(u.copy()))
    info = (stp.solver, stp.refine)
    stp.close()
    return seen, info


def row(name, cfg, steps, ref_mode=True, **kw):
    seen, (solver, refine) = chain(cfg, steps, **kw)
    orc = OraclePlan(cfg.system, cfg.approx, cfg.tau)
    ut = ur = cfg.u0
    eg = er = 0.0
    for u in seen:
        ut = orc.step(ut, "truth")
        eg = max(eg, rel_l2(u, ut))
        if ref_mode:
            ur = orc.step(ur, "reference")
            er = max(er, rel_l2(ur, ut))
    print(f"| {name} | {solver}, refine={refine} | {steps} | {eg:.2e} | {er:.2e} |", flush=True)


print("| case | solver | steps | GPU vs truth (max over steps) | reference algorithm vs truth |")
print("|---|---|---|---|---|")
row("cfg 1 (1D P1, 1,023 DOF, K=32)", fixtures.config1(), 10)
row("cfg 2 (1D P1, 1,048,574 DOF, K=64, tau*sr=2.1e7)", fixtures.config2(), 20)
for idx, m in ((3, 64), (4, 64), (5, 16)):
    cfg = fixtures.stiffness_matched(idx, m)
    row(f"cfg {idx} stiffness-matched ({cfg.name})", cfg, cfg.n_steps)
# the reference's own P2 goldens and acceptance workload
for name in ("fem_p2", "harness_p2"):
    d, sysm, ap = load_golden(name)
    stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True)
    seen = []
    rexi_run(stp, d["u0"], len(d["steps"]), observer=lambda k, t, u: seen.append(u.copy()))
    orc = OraclePlan(sysm, ap, float(d["tau"]))
    ut = d["u0"]; eg = er = 0.0
    for k, u in enumerate(seen):
        ut = orc.step(ut, "truth")
        eg = max(eg, rel_l2(u, ut)); er = max(er, rel_l2(d["steps"][k], ut))
    print(f"| {name} (reference golden, P2) | {stp.solver}, refine={stp.refine} | {len(seen)} | {eg:.2e} | {er:.2e} (reference's own output) |")
    stp.close()
d, sysm, ap = load_golden("acceptance_p2")
for refine in (None, 1):
    stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), refine=refine)
    orc = OraclePlan(sysm, ap, float(d["tau"]))
    u, ut, done = d["u0"], d["u0"], 0
    out = []
    for i, k in enumerate(int(c) for c in d["check_steps"]):
        u = rexi_run(stp, u, k - done)
        for _ in range(k - done):
            ut = orc.step(ut, "truth")
        done = k
        out.append(f"step {k}: {rel_l2(u, ut):.1e} vs ref {rel_l2(d['states'][i], ut):.1e}")
    print(f"| acceptance_p2 (7,999 DOF P2, K=16) | {stp.solver}, refine={stp.refine} | 1000 | " + "; ".join(out) + " | (reference's own states) |", flush=True)
    stp.close()
# full-size 2D/3D step 1 against the CPU truth fixtures
from fullsize_probes import probes
for c in (3, 5):
    g = np.load(os.path.join(ROOT, "tests", "golden", "fullsize", f"cfg{c}_step1.npz"))
    cfg = fixtures.build_config(c)
    stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
    u1 = rexi_step(stp, cfg.u0)
    stp.close()
    rows, w = probes(c, cfg.system.n_dof)
    e_rows = np.linalg.norm(u1[rows] - g["u1_rows"]) / np.linalg.norm(g["u1_rows"])
    e_proj = float(np.max(np.abs(w @ u1 - g["proj"]) / np.abs(g["proj"])))
    print(f"| cfg {c} full size, step 1 (8192 sampled rows / 4 projections) | cocg, refine=1 | 1 | {e_rows:.2e} / {e_proj:.2e} | CPU truth fixture |", flush=True)
