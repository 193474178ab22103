"""GPU: COCG layout and format changes must not change the answer.
Repacking the live lanes into a prefix of the same width (cocg.cu cg_solve)
is bitwise identical to the halving-only compaction (layout-independent
reduction tree), and the narrow-layout spmv over stencil classes (CgClass:
columns and B values from a per-class table) is bitwise identical to plain
CSR, on 2D and 3D pencils, plain and refined."""
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
c, m, refine, steps = (int(a) for a in sys.argv[1:5])
cfg = fixtures.build_config(c, m=m)
stp = rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True, refine=refine)
out = rexi_run(stp, cfg.u0, steps)
np.save(sys.argv[5], out)
"""


_DEFAULT_RUNS = {}   # (c, m, refine, steps) -> output of the default (no switch) run


def _run(c, m, refine, steps, env_extra, tmp_path, tag):
    key = (c, m, refine, steps)
    if not env_extra and key in _DEFAULT_RUNS:
        return _DEFAULT_RUNS[key]
    out = _run_uncached(c, m, refine, steps, env_extra, tmp_path, tag)
    if not env_extra:
        _DEFAULT_RUNS[key] = out
    return out


def _run_uncached(c, m, refine, steps, env_extra, tmp_path, tag):
    env = dict(os.environ, **env_extra)
    path = str(tmp_path / f"cocg_{c}_{m}_{refine}_{tag}.npy")
    subprocess.run([sys.executable, "-c", _PROBE % ROOT, str(c), str(m), str(refine), str(steps), path],
                   check=True, env=env, cwd=ROOT)
    return np.load(path)


@pytest.mark.parametrize("c,m,refine", [(3, 64, 1), (3, 64, 0), (5, 12, 1), (4, 48, 1)])
def test_prefix_repack_bitwise(c, m, refine, tmp_path):
    repacked = _run(c, m, refine, 2, {}, tmp_path, "prefix")
    plain = _run(c, m, refine, 2, {"REXI_COCG_NOPREFIX": "1"}, tmp_path, "plain")
    assert np.all(np.isfinite(plain))
    assert np.array_equal(repacked, plain)


@pytest.mark.parametrize("c,m,refine", [(3, 64, 1), (5, 12, 1), (4, 48, 0)])
def test_stencil_classes_bitwise(c, m, refine, tmp_path):
    classed = _run(c, m, refine, 2, {}, tmp_path, "cls")
    plain = _run(c, m, refine, 2, {"REXI_COCG_NOCLS": "1"}, tmp_path, "nocls")
    assert np.all(np.isfinite(plain))
    assert np.array_equal(classed, plain)


# The TMA-pipelined kernels of the wide layouts -- the windowed spmv (p, q, x
# tiles, z windows and the packed matrix blob by bulk copy; two row-lanes per
# thread on 2D patterns, one on 3D patterns), the tile-only TMA spmv and the
# TMA update -- keep the gather kernels' rows per sub-block, per-lane operation
# order and partial tree: the step must be bitwise identical with each of them
# switched off, and with the live-prefix row stride switched off.
@pytest.mark.parametrize("c,m,refine", [(3, 64, 1), (4, 48, 1), (5, 14, 1), (3, 40, 0)])
@pytest.mark.parametrize("off", ["REXI_COCG_NOTMA", "REXI_COCG_NOWIN", "REXI_COCG_NOUTMA", "REXI_COCG_NOLD"])
def test_tma_kernels_bitwise(c, m, refine, off, tmp_path):
    tma = _run(c, m, refine, 2, {}, tmp_path, "tma")
    plain = _run(c, m, refine, 2, {off: "1"}, tmp_path, off.lower())
    assert np.all(np.isfinite(plain))
    assert np.array_equal(tma, plain)


def test_window_tables_cover_ragged_sizes(tmp_path):
    """Row counts that are not multiples of the stage / chunk sizes (the last
    stage and the last chunk are partial): windowed vs gather kernels."""
    for m in (33, 50, 71):
        tma = _run(3, m, 1, 1, {}, tmp_path, f"rag{m}")
        plain = _run(3, m, 1, 1, {"REXI_COCG_NOTMA": "1"}, tmp_path, f"rag{m}_plain")
        assert np.array_equal(tma, plain), m


@pytest.mark.parametrize("c,m", [(3, 64), (4, 48), (5, 14)])
def test_window_tables_are_built(c, m, tmp_path):
    """The bitwise tests above compare against the gather kernels; this one
    makes sure the windowed path is what the default run uses on the 2D
    (K = 64, K = 128) and 3D fixtures: REXI_COCG_REQUIRE_WIN turns a missing
    table into an error."""
    out = _run(c, m, 1, 1, {"REXI_COCG_REQUIRE_WIN": "1"}, tmp_path, "reqwin")
    assert np.all(np.isfinite(out))
