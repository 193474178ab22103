"""Feasibility probe: do two half-width (32-shift) cfg2 plans on two streams overlap
(K2 is FP64/issue-bound, K3/S1 HBM-bound)?  Independent states, no combine."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1912_03312_b200 import fixtures, _native
from paper_1912_03312_b200._pattern import shared_pattern

cfg = fixtures.build_config(2)
ip, ix, ar, ai, br = shared_pattern(cfg.system.A, cfg.system.B)
sh, wt = cfg.approx.shifts, cfg.approx.weights
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
s_full = torch.cuda.Stream(); sA = torch.cuda.Stream(); sB = torch.cuda.Stream()
full = _native.NativePlan(ip, ix, ar, br, sh, wt, cfg.tau, a_imag=ai, device=0, refine=1, stream=s_full.cuda_stream)
pa = _native.NativePlan(ip, ix, ar, br, sh[:32], wt[:32], cfg.tau, a_imag=ai, device=0, refine=1, stream=sA.cuda_stream)
pb = _native.NativePlan(ip, ix, ar, br, sh[32:], wt[32:], cfg.tau, a_imag=ai, device=0, refine=1, stream=sB.cuda_stream)
u = torch.from_numpy(cfg.u0).cuda()
bufs = {k: (u.clone(), torch.empty_like(u)) for k in "fab"}

def run(plan, k, n):
    a, b = bufs[k]
    plan.step_device(a.data_ptr(), b.data_ptr(), n)

for p, k in ((full, "f"), (pa, "a"), (pb, "b")):
    run(p, k, 3)
torch.cuda.synchronize()

def timed(fn):
    torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize(); return (time.perf_counter() - t) * 1e3 / steps

t_full = timed(lambda: run(full, "f", steps))
t_a = timed(lambda: run(pa, "a", steps))
t_ser = timed(lambda: (run(pa, "a", steps), run(pb, "b", steps)))
import threading
def conc():
    # rexi_plan_step synchronises its own stream at the end: one host thread per
    # plan (ctypes drops the GIL), so both streams are fed at once
    th = [threading.Thread(target=run, args=(p, k, steps)) for p, k in ((pa, "a"), (pb, "b"))]
    for t in th: t.start()
    for t in th: t.join()
t_conc = timed(conc)
print(f"full 64-lane step {t_full:.3f} ms | one 32-lane half {t_a:.3f} ms | halves serial {t_ser:.3f} ms | "
      f"halves on two streams (two host threads) {t_conc:.3f} ms")
