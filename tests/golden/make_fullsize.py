"""Full-size truth samples for the 2D/3D BASELINE configs (TEST INFRASTRUCTURE).

The reference cannot run configs 3-5 (its factorize() falls back to a dense
LU, solvers.py:108-115) and a banded truth does not fit, so step 1 of the
full-size configs is computed here by the CPU truth restatement
``oracle.cocg_truth_step`` (Jacobi-COCG per shift, double-double residual
refinement with x in double-double, exact-product double-double sum of
beta_j x_j -- the 2D/3D counterpart of rexi_oracle.c's truth mode, checked
bit-for-bit against the banded truth in tests/test_oracle.py).

A 1-2M-entry complex vector is too large to commit, so the fixture keeps
size-independent evidence of u1:

* u1 at 8192 seeded random rows (rng = default_rng(20191207 + cfg));
* <w_q, u1> for 4 seeded complex Gaussian vectors w_q (same rng, drawn
  after the rows), which sees an error anywhere in the vector;
* ||u1||_2, ||u0||_2 and per-shift iteration counts / last corrections.

Run in the build container (hours of CPU for cfg 3 and 5 on 8 threads):

    python tests/golden/make_fullsize.py 5 3
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
os.environ.setdefault("REXI_FIXTURE_HOST", "1")

sys.path.insert(0, HERE)
from fullsize_probes import probes  # noqa: E402
from oracle.oracle import cocg_truth_step  # noqa: E402
from paper_1912_03312_b200 import fixtures  # noqa: E402


def main(cfgs):
    for c in cfgs:
        t0 = time.time()
        cfg = fixtures.build_config(c)
        t1 = time.time()
        u1, iters, corr = cocg_truth_step(cfg.system, cfg.approx, cfg.tau, cfg.u0,
                                          tol=1e-12, rounds=4, tol_refine=1e-9)
        t2 = time.time()
        rows, w = probes(c, len(u1))
        out = os.path.join(HERE, "fullsize", f"cfg{c}_step1.npz")
        np.savez_compressed(out, rows=rows, u1_rows=u1[rows], proj=w @ u1,
                            norm_u1=np.linalg.norm(u1), norm_u0=np.linalg.norm(cfg.u0),
                            iters=iters, corr=corr, tau=cfg.tau, n=len(u1),
                            k=len(cfg.approx.shifts), build_s=t1 - t0, truth_s=t2 - t1)
        print(f"cfg{c}: n={len(u1)} build {t1 - t0:.1f}s truth {t2 - t1:.1f}s "
              f"iters max {iters.max()} median {np.median(iters)} corr max {corr.max():.2e}",
              flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [5, 3])
