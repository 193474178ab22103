"""Run one REXI step of config C on cuda:0 (for profiling): python scripts/cfg_step.py C [refine] [tol]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1912_03312_b200 import fixtures, rexi_prepare, _native
c = int(sys.argv[1]); refine = int(sys.argv[2]) if len(sys.argv) > 2 else None
tol = float(sys.argv[3]) if len(sys.argv) > 3 else None
cfg = fixtures.build_config(c)
stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True, refine=refine, tol=tol)
ud = torch.from_numpy(cfg.u0).cuda(); out = torch.empty_like(ud)
st = _native.RexiStats()
t = time.time(); stp.plans[0].step_device(ud.data_ptr(), out.data_ptr(), 1, st); torch.cuda.synchronize()
print(f"cfg{c}: {time.time()-t:.3f} s/step, iters max {st.iters_max}, mean {st.iters_mean:.1f}, launches {st.launches}")
stp.close()
