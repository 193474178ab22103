"""Sample rows and projection vectors of the full-size truth fixtures
(shared by make_fullsize.py and tests/test_gpu_fullsize.py)."""
import numpy as np

N_SAMPLES = 8192
N_PROJ = 4


def probes(cfg_idx: int, n: int):
    """u1 is kept at these rows, and as <w_q, u1> for these w_q (seeded)."""
    rng = np.random.default_rng(20191207 + cfg_idx)
    rows = np.sort(rng.choice(n, size=min(N_SAMPLES, n), replace=False))
    w = rng.standard_normal((N_PROJ, n)) + 1j * rng.standard_normal((N_PROJ, n))
    return rows, w
