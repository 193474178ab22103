"""Fixture build times with the device assembly."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1912_03312_b200 import fixtures
torch.zeros(1).cuda()
for c in (3, 4, 5):
    t = time.time(); cfg = fixtures.build_config(c); torch.cuda.synchronize()
    print(f"cfg{c}: build {time.time()-t:.2f} s (n={cfg.system.n_dof}, nnz={cfg.system.A.nnz})", flush=True)
mesh = fixtures.StructuredMesh(3, 128, fixtures.np.zeros(3), 1 / 128)
v = fixtures._harmonic([0.5] * 3, 30.0)
from paper_1912_03312_b200.assembly import assemble_p1_device
for _ in range(2):
    t = time.time(); s = assemble_p1_device(mesh, v); torch.cuda.synchronize()
    print(f"assemble_p1_device 128^3: {time.time()-t:.3f} s", flush=True)
