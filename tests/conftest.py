import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the native library")
    config.addinivalue_line("markers", "slow: full-size configs")


def load_golden(name):
    """(npz, SystemMatrices, PartialFractionApproximation) of a golden case
    written by tests/golden/make_golden.py from the reference itself."""
    from scipy.sparse import csr_matrix
    from paper_1912_03312_b200.types import PartialFractionApproximation, SystemMatrices
    d = np.load(os.path.join(GOLDEN, name + ".npz"))

    def csr(p):
        return csr_matrix((d[p + "_data"], d[p + "_indices"], d[p + "_indptr"]),
                          shape=tuple(d[p + "_shape"]))
    sysm = SystemMatrices(csr("A"), csr("B"), int(d["A_shape"][0]))
    ap = PartialFractionApproximation(d["shifts"], d["weights"], float(d["R1"]), 0.0)
    return d, sysm, ap


def golden_names():
    """REXI golden cases (the cheb_* files hold the 8(f) rows)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith(("cheb_", "acceptance_")))


def cheb_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "cheb_*.npz")))


def load_cheb(name):
    """(npz, SystemMatrices) of a spectral-radius / Chebyshev golden case
    (reference spectral_radius_estimate + chebyshev_run, make_golden.py --cheb)."""
    from scipy.sparse import csr_matrix
    from paper_1912_03312_b200.types import SystemMatrices
    d = np.load(os.path.join(GOLDEN, name + ".npz"))

    def csr(p):
        return csr_matrix((d[p + "_data"], d[p + "_indices"], d[p + "_indptr"]),
                          shape=tuple(d[p + "_shape"]))
    return d, SystemMatrices(csr("A"), csr("B"), int(d["A_shape"][0]))


@pytest.fixture(scope="session")
def flagship():
    from paper_1912_03312_b200 import fixtures
    return fixtures.load_poles(16)
