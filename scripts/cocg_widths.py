"""Per-width COCG kernel profile of one step: REXI_COCG_TRACE=1 python scripts/cocg_widths.py C [pre_steps]
(pre_steps steps from u0 first: later steps see broader-band states)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("REXI_COCG_TRACE", "1")
import torch
from paper_1912_03312_b200 import fixtures, rexi_prepare
c = int(sys.argv[1])
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = fixtures.build_config(c)
stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
ud = torch.from_numpy(cfg.u0).cuda(); out = torch.empty_like(ud)
plan = stp.plans[0]
for _ in range(pre):
    plan.step_device(ud.data_ptr(), out.data_ptr(), 1); torch.cuda.synchronize()
    ud, out = out, ud
plan.step_device(ud.data_ptr(), out.data_ptr(), 1); torch.cuda.synchronize()
plan.profile(True)
plan.step_device(ud.data_ptr(), out.data_ptr(), 1); torch.cuda.synchronize()
rep = plan.profile_report(); plan.profile(False)
tot = sum(v[1] for v in rep.values())
def key(kv):
    n = kv[0]
    return (n.split("@")[0], -int(n.split("@")[1]) if "@" in n else 0)
for name, (cnt, ms, b) in sorted(rep.items(), key=key):
    gbs = b / (ms / 1e3) / 1e9 if b and ms else 0
    print(f"{name:16s} n={cnt:5d} {ms:9.3f} ms ({100*ms/tot:5.1f}%) avg {1e3*ms/max(cnt,1):8.1f} us  {gbs:7.0f} GB/s ({gbs/65.424:4.1f}%)")
print(f"total {tot:.1f} ms")
