"""Per-step COCG timing over several steps of config C (steps after the first see
broader-band states): REXI_COCG_TRACE=1 python scripts/cocg_steps.py C [steps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1912_03312_b200 import fixtures, rexi_prepare, _native
c = int(sys.argv[1]); steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = fixtures.build_config(c)
stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
plan = stp.plans[0]
a = torch.from_numpy(cfg.u0).cuda(); b = torch.empty_like(a)
for s in range(steps):
    st = _native.RexiStats()
    torch.cuda.synchronize(); t = time.perf_counter()
    plan.step_device(a.data_ptr(), b.data_ptr(), 1, st); torch.cuda.synchronize()
    print(f"step {s + 1}: {1e3 * (time.perf_counter() - t):.1f} ms, lockstep iters {st.iters_max} "
          f"(sum over solves {st.iters_mean:.0f})", file=sys.stderr, flush=True)
    a, b = b, a
