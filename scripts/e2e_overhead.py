import sys, os, time, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_step, _native
cfg = fixtures.build_config(1)
stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True)
p = stp.plans[0]
u = _native.host_empty(cfg.u0.shape); u[:] = cfg.u0
for _ in range(50): rexi_step(stp, u)
N = 2000
t = time.perf_counter()
for _ in range(N): rexi_step(stp, u)
t_step = (time.perf_counter() - t) / N
t = time.perf_counter()
for _ in range(N): _native.host_empty(u.shape)
t_alloc = (time.perf_counter() - t) / N
out = _native.host_empty(u.shape)
lib = _native.lib()
t = time.perf_counter()
for _ in range(N): lib.rexi_plan_step(p._h, _native._ptr(u), _native._ptr(out), 1, _native.MEM_HOST, None)
t_c = (time.perf_counter() - t) / N
import torch
ud = torch.from_numpy(cfg.u0).cuda(); od = torch.empty_like(ud)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(N): p.step_device(ud.data_ptr(), od.data_ptr(), 1)
torch.cuda.synchronize()
t_dev = (time.perf_counter() - t) / N
print(f"rexi_step {t_step*1e6:.1f} us | host_empty {t_alloc*1e6:.1f} us | raw C call (host ptrs) {t_c*1e6:.1f} us | step_device {t_dev*1e6:.1f} us")
