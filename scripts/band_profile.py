"""Per-kernel device time of the band solver on the acceptance workload
(tests/golden/acceptance_p2.npz): python scripts/band_profile.py [steps]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
from conftest import load_golden
from paper_1912_03312_b200 import rexi_prepare, _native
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
d, sysm, ap = load_golden("acceptance_p2")
stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]))
plan = stp.plans[0]
print("solver", stp.solver, "prepare_ms", stp.stats["prepare_ms"])
a = torch.from_numpy(d["u0"]).cuda(); b = torch.empty_like(a)
plan.step_device(a.data_ptr(), b.data_ptr(), 5); torch.cuda.synchronize()
t = time.perf_counter(); plan.step_device(a.data_ptr(), b.data_ptr(), steps); torch.cuda.synchronize()
print(f"graph replay: {(time.perf_counter() - t) / steps * 1e6:.1f} us/step")
plan.profile(True)
plan.step_device(a.data_ptr(), b.data_ptr(), steps); torch.cuda.synchronize()
for k, (c, ms, _b) in sorted(plan.profile_report().items()):
    print(f"{k:14s} n={c:6d} avg {1e3 * ms / c:8.2f} us")
plan.profile(False)
