"""Per-call overhead of a one-step host call on cfg 1 (persistent kernel):
bare C call with/without stats, the Python API.  python scripts/e2e_overhead.py"""
import os, sys, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_step, _native
cfg = fixtures.config1()
stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True, device=0)
plan = stp.plans[0]
u = torch.from_numpy(cfg.u0).pin_memory().numpy()
N = 2000


def tm(f):
    f(); f()
    gc.disable()
    t = time.perf_counter()
    for _ in range(N):
        f()
    gc.enable()
    return (time.perf_counter() - t) / N * 1e6


print(f"plan.step_host, no stats: {tm(lambda: plan.step_host(u, 1, None)):.1f} us")
print(f"plan.step_host, stats:    {tm(lambda: plan.step_host(u, 1, _native.RexiStats())):.1f} us")
print(f"rexi_step(numpy):         {tm(lambda: rexi_step(stp, u)):.1f} us")
out = _native.host_empty(u.shape)
import ctypes
L = _native.lib()
h = plan._h
print(f"bare rexi_plan_step:      {tm(lambda: L.rexi_plan_step(h, u.ctypes.data, out.ctypes.data, 1, 0, None)):.1f} us")
print(f"host_empty:               {tm(lambda: _native.host_empty(u.shape)):.1f} us")
