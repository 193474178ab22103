"""Stiffness-matched parity probe: GPU vs the CPU truth oracle every step,
refine 0 and 1 (cfg 3/4/5 at tau*sr of the full configs)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np
from paper_1912_03312_b200 import fixtures as F, rexi_prepare, rexi_run
from oracle.oracle import OraclePlan, rel_l2

cases = [(3, 64), (4, 64), (5, 16)] if len(sys.argv) < 2 else [tuple(map(int, a.split(':'))) for a in sys.argv[1:]]
out = []
for i, m in cases:
    c = F.stiffness_matched(i, m)
    orc = OraclePlan(c.system, c.approx, c.tau)
    truth = []
    ut = c.u0
    for s in range(c.n_steps):
        ut = orc.step(ut, "truth")
        truth.append(ut)
    for refine in (0, 1, 2):
        stp = rexi_prepare(c.system, c.approx, c.tau, sr_value=c.sr, override_admissibility=True, refine=refine)
        seen = []
        t0 = time.time()
        rexi_run(stp, c.u0, c.n_steps, observer=lambda k, t, u: seen.append(u.copy()))
        dt = time.time() - t0
        errs = [rel_l2(u, t) for u, t in zip(seen, truth)]
        rec = dict(case=c.name, refine=refine, errs=errs, secs=dt, stats=dict(stp.stats))
        print(json.dumps(rec, default=str), flush=True)
        out.append(rec)
        stp.close()
json.dump(out, open('gpurun_out/stiff_probe.json', 'w'), indent=1, default=str)
