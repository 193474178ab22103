"""Phase timing of the persistent 1D loop: REXI_PERSIST_TRACE=1 python scripts/persist_probe.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1912_03312_b200 import fixtures, rexi_prepare
cfg = fixtures.config1()
stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
print("persistent cluster", stp.plans[0].info.persistent, flush=True)
ud = torch.from_numpy(cfg.u0).cuda(); out = torch.empty_like(ud)
for n in (1, 10, 1000):
    stp.plans[0].step_device(ud.data_ptr(), out.data_ptr(), n); torch.cuda.synchronize()
    t = time.time(); stp.plans[0].step_device(ud.data_ptr(), out.data_ptr(), n); torch.cuda.synchronize()
    print(f"{n} steps: {(time.time()-t)/n*1e6:.1f} us/step", flush=True)
