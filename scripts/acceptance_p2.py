"""The reference's acceptance workload through the drop-in (tests/golden/
acceptance_p2.npz, test_acceptance.py:95-121): 7,999-DOF P2, K = 16,
dt = 2e-4, 1000 steps.  Prints steps/s, parity against the reference's own
states and the truth oracle, and the B-norm drift (criterion 7).
    python scripts/acceptance_p2.py [solver]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from conftest import load_golden
from paper_1912_03312_b200 import rexi_prepare, rexi_run
from oracle.oracle import OraclePlan, rel_l2
solver = sys.argv[1] if len(sys.argv) > 1 else "auto"
d, sysm, ap = load_golden("acceptance_p2")
tau, sr = float(d["tau"]), float(d["sr"])
checks = [int(c) for c in d["check_steps"]]
stp = rexi_prepare(sysm, ap, tau, sr_value=sr, solver=solver)
rexi_run(stp, d["u0"], 5)                       # warm
t0 = time.perf_counter()
u = rexi_run(stp, d["u0"], 1000)
dt = time.perf_counter() - t0
print(f"solver {stp.solver} refine {stp.refine} bandwidth {stp.bandwidth}: 1000 steps {dt:.3f} s "
      f"({1000 / dt:.0f} steps/s); reference here {float(d['ref_run_s']):.2f} s")
states, done, cur = {}, 0, d["u0"]
for k in checks:
    cur = rexi_run(stp, cur, k - done)
    done = k
    states[k] = cur
orc = OraclePlan(sysm, ap, tau)
ut, done = d["u0"], 0
for i, k in enumerate(checks):
    for _ in range(k - done):
        ut = orc.step(ut, "truth")
    done = k
    print(f"step {k}: vs reference {rel_l2(states[k], d['states'][i]):.2e}, vs truth {rel_l2(states[k], ut):.2e}, "
          f"reference vs truth {rel_l2(d['states'][i], ut):.2e}")
B = sysm.B
bn = lambda v: np.sqrt(np.vdot(v, B @ v).real)
print(f"B-norm drift over 1000 steps {abs(bn(u) - bn(d['u0'])) / bn(d['u0']):.2e} (criterion 7: <= 1e-6)")
stp.close()
