"""GPU probe for the COCG path: small 2D/3D pencils vs the oracle truth, then full-size timing."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_step, rexi_run
from oracle.oracle import OraclePlan, rel_l2

def small(cfg, label):
    stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
    t = time.time(); u1 = rexi_step(stp, cfg.u0); dt = time.time() - t
    orc = OraclePlan(cfg.system, cfg.approx, cfg.tau)
    truth = orc.step(cfg.u0, "truth"); ref = orc.step(cfg.u0, "reference")
    print(f"{label}: n={cfg.system.n_dof} K={cfg.approx.K} tau*sr={cfg.tau*cfg.sr:.3g} gpu-truth {rel_l2(u1, truth):.3e} "
          f"refLU-truth {rel_l2(ref, truth):.3e} step {dt*1e3:.1f} ms solver={stp.solver} refine={stp.refine}", flush=True)
    stp.close()

small(fixtures.config3(m=48), "2D m=48 (cfg3 tau)")
small(fixtures.config5(m=12), "3D m=12 (cfg5 tau)")
c = fixtures.config4(m=48); small(c, "2D m=48 (cfg4 V, tau)")
for which in sys.argv[1:]:
    t = time.time()
    cfg = fixtures.build_config(int(which))
    print(f"cfg{which}: build {time.time()-t:.1f}s n={cfg.system.n_dof} nnz={cfg.system.A.nnz} K={cfg.approx.K}", flush=True)
    stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
    from paper_1912_03312_b200 import _native
    st = _native.RexiStats()
    ud = torch.from_numpy(cfg.u0).cuda(); out = torch.empty_like(ud)
    t = time.time(); stp.plans[0].step_device(ud.data_ptr(), out.data_ptr(), 1, st); torch.cuda.synchronize(); dt = time.time() - t
    print(f"  step {dt:.3f} s, iters max {st.iters_max} mean(sum over solves) {st.iters_mean:.1f}, launches {st.launches}", flush=True)
    stp.close()
