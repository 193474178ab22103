"""Per-rank step time of a pole shard (first K/world shifts of the config) on
one GPU: the compute part of a world-size-W step (no exchange).
python scripts/shard_probe.py C"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1912_03312_b200 import fixtures, _native
from paper_1912_03312_b200._pattern import shared_pattern
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = fixtures.build_config(c)
ip, ix, ar, ai, br = shared_pattern(cfg.system.A, cfg.system.B)
K = cfg.approx.K
refine = 1 if cfg.tau * cfg.sr > 5e3 else 0
u = torch.from_numpy(cfg.u0).cuda()
n = u.shape[0]
for world in (1, 2, 4, 8):
    k = K // world
    sh, wt = cfg.approx.shifts[:k], cfg.approx.weights[:k]
    p = _native.NativePlan(ip, ix, ar, br, sh, wt, cfg.tau, a_imag=ai, device=0, refine=refine,
                           weight_ref=float(np.mean(np.abs(cfg.approx.weights))))
    part = torch.empty((4, n), dtype=torch.float64, device="cuda")
    steps = 50 if c <= 2 else 2
    for _ in range(3):
        p.step_partial(u.data_ptr(), part.data_ptr())
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(steps):
        p.step_partial(u.data_ptr(), part.data_ptr())
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / steps
    print(f"cfg{c} world {world}: shard K={k} {dt*1e3:.3f} ms/step (speedup vs world 1 at equal exchange: see first line)", flush=True)
    if os.environ.get("SHARD_PROF"):
        # per-kernel device time of the same steps (CUDA events around each launch)
        p.profile(True)
        for _ in range(steps):
            p.step_partial(u.data_ptr(), part.data_ptr())
        torch.cuda.synchronize()
        rep = p.profile_report()
        p.profile(False)
        print("   " + ", ".join(f"{kn}: {v[1] / steps * 1e3:.1f} us x{v[0] // steps}" for kn, v in
                                 sorted(rep.items(), key=lambda kv: -kv[1][1])), flush=True)
    p.close() if hasattr(p, "close") else None
