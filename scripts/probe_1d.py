"""Quick GPU probe: cfg1/cfg2 accuracy vs oracle and step timing."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_step, rexi_run
from oracle.oracle import OraclePlan, rel_l2

for which in sys.argv[1:] or ["1", "2"]:
    t = time.time()
    cfg = fixtures.build_config(int(which))
    print(f"cfg{which}: build {time.time()-t:.1f}s n={cfg.system.n_dof} K={cfg.approx.K}", flush=True)
    for refine in (0, 1):
        t = time.time()
        stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True, refine=refine)
        print(f"  refine={refine} prepare {time.time()-t:.2f}s stats {stp.stats}", flush=True)
        u1 = rexi_step(stp, cfg.u0)
        orc = OraclePlan(cfg.system, cfg.approx, cfg.tau)
        t = time.time(); truth = orc.step(cfg.u0, "truth"); tt = time.time()-t
        t = time.time(); ref = orc.step(cfg.u0, "reference"); tr = time.time()-t
        print(f"  gpu-truth {rel_l2(u1, truth):.3e} gpu-refport {rel_l2(u1, ref):.3e} refport-truth {rel_l2(ref, truth):.3e} (oracle truth {tt:.1f}s ref {tr:.1f}s)", flush=True)
        ud = torch.from_numpy(cfg.u0).cuda()
        for _ in range(3):
            rexi_run(stp, ud, 1)
        torch.cuda.synchronize()
        nst = 20
        t = time.time(); out = rexi_run(stp, ud, nst); torch.cuda.synchronize(); dt = (time.time()-t)/nst
        print(f"  device-resident: {dt*1e3:.3f} ms/step  ({1/dt:.1f} steps/s)", flush=True)
        if os.environ.get("PROBE_PROF"):
            stp.plans[0].profile(True)
            rexi_run(stp, ud, nst); torch.cuda.synchronize()
            rep = stp.plans[0].profile_report(); stp.plans[0].profile(False)
            tot = sum(v[1] for v in rep.values())
            for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1]):
                print(f"    {k:12s} n={v[0]:5d} {v[1]/nst:.4f} ms/step {100*v[1]/tot:5.1f}%")
        stp.close()
