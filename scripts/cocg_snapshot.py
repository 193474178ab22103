"""Save COCG step outputs (bitwise regression reference): python scripts/cocg_snapshot.py OUT.npz"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from conftest import load_golden
from paper_1912_03312_b200 import rexi_prepare, rexi_run, fixtures
out = {}
for name in ("p1_2d_m16", "p1_3d_m8", "fem_p2", "harness_p2"):
    d, sysm, ap = load_golden(name)
    for w in (1, 3):
        stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True, workers=w)
        out[f"{name}_w{w}"] = rexi_run(stp, d["u0"], 2)
        stp.close()
c = fixtures.config3(m=96)
stp = rexi_prepare(c.system, c.approx, c.tau, sr_value=c.sr, override_admissibility=True)
out["cfg3_m96"] = rexi_run(stp, c.u0, 1)
stp.close()
c = fixtures.config5(m=28)
stp = rexi_prepare(c.system, c.approx, c.tau, sr_value=c.sr, override_admissibility=True)
out["cfg5_m28"] = rexi_run(stp, c.u0, 1)
stp.close()
np.savez(sys.argv[1], **out)
print("saved", list(out))
