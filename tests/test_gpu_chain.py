"""GPU: the small reduced levels of the 1D path run as ONE thread-block-cluster
launch (csrc/tridiag_l0.cu k_lv_chain: TMA-staged S1 up, top solve, S3
down).  Bitwise identical to the per-level launches, plain and refined, on
ragged sizes and shard-sized shift counts (fewer lanes start the chain a level
earlier)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

_PROBE = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_run
m, k, refine, steps = (int(a) for a in sys.argv[1:5])
cfg = fixtures.config2(m=m, k=k)
stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True, refine=refine)
out = rexi_run(stp, cfg.u0, steps)
np.save(sys.argv[5], out)
"""


def _run(m, k, refine, steps, env_extra, tmp_path, tag):
    env = dict(os.environ, **env_extra)
    path = str(tmp_path / f"chain_{m}_{k}_{refine}_{tag}.npy")
    subprocess.run([sys.executable, "-c", _PROBE % ROOT, str(m), str(k), str(refine), str(steps), path],
                   check=True, env=env, cwd=ROOT)
    return np.load(path)


@pytest.mark.parametrize("m,k,refine", [(2 ** 18 + 36, 64, 1), (2 ** 18 + 36, 64, 0), (300_001, 16, 1),
                                        (70_001, 32, 1), (5_000, 64, 1)])
def test_chain_equals_per_level_launches_bitwise(m, k, refine, tmp_path):
    chained = _run(m, k, refine, 3, {}, tmp_path, "chain")
    plain = _run(m, k, refine, 3, {"REXI_NO_CHAIN": "1"}, tmp_path, "plain")
    assert np.all(np.isfinite(plain))
    assert np.array_equal(chained, plain)
