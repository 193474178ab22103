"""1D outputs for bitwise comparisons: python scripts/tri_snapshot.py OUT.npz"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1912_03312_b200 import rexi_prepare, rexi_run, fixtures
out = {}
c2 = fixtures.config2()
for refine in (0, 1):
    stp = rexi_prepare(c2.system, c2.approx, c2.tau, sr_value=c2.sr, override_admissibility=True, refine=refine)
    out[f"cfg2_r{refine}"] = rexi_run(stp, c2.u0, 3)
    stp.close()
for n in (4097, 70001, 300003):
    import scipy.sparse as sp
    s = type(c2.system)(c2.system.A[:n, :n].tocsr(), c2.system.B[:n, :n].tocsr(), n)
    for refine in (0, 1):
        stp = rexi_prepare(s, c2.approx, c2.tau, sr_value=c2.sr, override_admissibility=True, refine=refine)
        out[f"n{n}_r{refine}"] = rexi_run(stp, c2.u0[:n], 2)
        stp.close()
c1 = fixtures.config1()
for refine in (0, 1):
    stp = rexi_prepare(c1.system, c1.approx, c1.tau, sr_value=c1.sr, override_admissibility=True, refine=refine)
    out[f"cfg1_r{refine}"] = rexi_run(stp, c1.u0, 3)
    stp.close()
np.savez(sys.argv[1], **out)
print("saved", len(out))
