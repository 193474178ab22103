"""COCG pieces running concurrently on ONE GPU (two host threads, two plan
streams): does overlapping the hard shifts' narrow tail with the other
shifts' wide phases pay?  python scripts/concurrent_pieces.py C [n_hard...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_step
from paper_1912_03312_b200.integrate import _make_plans
c = int(sys.argv[1]); hards = [int(a) for a in sys.argv[2:]] or [2, 4, 8]
cfg = fixtures.build_config(c)
u0 = torch.from_numpy(cfg.u0).cuda()


def timed(stp, u):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        u = rexi_step(stp, u)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / 3 * 1e3, u


stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
u1 = rexi_step(stp, u0)
u2 = rexi_step(stp, u1)
its = np.array(stp.stats["shift_iters"])
order = np.argsort(-its)
print("per-shift iterations (step 2), top 8:", its[order[:8]].tolist(), "median", float(np.median(its)))
ms, ref = timed(stp, u2)
print(f"one plan: {ms:.1f} ms/step (steps 3-5)", flush=True)
stp.close()
for nh in hards:
    stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True,
                       workers=2, devices=[0, 0])
    hard = sorted(int(j) for j in order[:nh])
    rest = sorted(int(j) for j in range(cfg.approx.K) if j not in hard)
    for p in stp.plans:
        p.close()
    stp.pieces = [hard, rest]
    stp.plans = _make_plans(stp._plan_args, stp.pieces, [0, 0])
    stp._rebalanced = True
    rexi_step(stp, u2)
    ms, out = timed(stp, u2)
    d = float(torch.max(torch.abs(out - ref)) / torch.max(torch.abs(ref)))
    print(f"hard {nh} || rest {len(rest)}: {ms:.1f} ms/step (steps 3-5), max diff vs one plan {d:.1e}", flush=True)
    stp.close()
