"""P2 (pentadiagonal) timing/accuracy on the reference harness default (tests/golden/harness_p2.npz)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from conftest import load_golden
from paper_1912_03312_b200 import rexi_prepare, rexi_run, _native
d, sysm, ap = load_golden("harness_p2")
print("n", sysm.n_dof, "tau*sr", float(d["tau"]) * float(d["sr"]))
for refine in (None, 0):
    stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True, refine=refine)
    u = rexi_run(stp, d["u0"], 3)
    print("refine", refine, "solver", stp.solver, "stats", stp.stats, "rel vs reference step 3",
          np.linalg.norm(u - d["steps"][-1]) / np.linalg.norm(d["steps"][-1]))
    ud = torch.from_numpy(d["u0"]).cuda(); out = torch.empty_like(ud)
    st = _native.RexiStats()
    stp.plans[0].step_device(ud.data_ptr(), out.data_ptr(), 1, st); torch.cuda.synchronize()
    t = time.time(); stp.plans[0].step_device(ud.data_ptr(), out.data_ptr(), 20, st); torch.cuda.synchronize()
    print(f"  {(time.time()-t)/20*1e3:.3f} ms/step, iters max {st.iters_max} mean {st.iters_mean:.1f}")
    stp.close()
