"""GPU: the one-launch multi-step loop for small 1D plans (SURVEY 8(f)3,
csrc/tridiag_persist.cu) is bitwise identical to the multi-kernel path and
to the reference goldens' tolerance."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu

_PROBE = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from conftest import load_golden
from paper_1912_03312_b200 import rexi_prepare, rexi_run
d, sysm, ap = load_golden(sys.argv[1])
stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True, refine=0)
out = rexi_run(stp, d["u0"], int(sys.argv[2]))
np.save(sys.argv[3], out)
"""


def _run(name, steps, persist, tmp_path):
    env = dict(os.environ, REXI_PERSIST=persist)
    path = str(tmp_path / f"{name}_{persist}.npy")
    subprocess.run([sys.executable, "-c", _PROBE % os.path.join(ROOT, "tests"), name, str(steps), path],
                   check=True, env=env, cwd=ROOT)
    return np.load(path)


def test_persistent_path_is_taken():
    from paper_1912_03312_b200 import rexi_prepare
    d, sysm, ap = load_golden("cfg1_k32")
    stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True)
    assert stp.plans[0].info.persistent >= 4
    stp.close()


@pytest.mark.parametrize("name,steps", [("cfg1_k32", 10), ("cfg1_k16", 10), ("cfg1_k32", 1)])
def test_persistent_equals_multikernel_bitwise(name, steps, tmp_path):
    a = _run(name, steps, "1", tmp_path)
    b = _run(name, steps, "0", tmp_path)
    assert np.array_equal(a, b)


def test_persistent_matches_reference_every_step():
    from paper_1912_03312_b200 import rexi_prepare, rexi_run
    d, sysm, ap = load_golden("cfg1_k32")
    stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True)
    u = d["u0"]
    for k in range(d["steps"].shape[0]):
        u = rexi_run(stp, u, 1)
        assert np.linalg.norm(u - d["steps"][k]) <= 2.5e-9 * np.linalg.norm(d["steps"][k])
    all_steps = rexi_run(stp, d["u0"], d["steps"].shape[0])
    assert np.array_equal(all_steps, u)
    stp.close()


def test_persistent_in_place_device_call():
    import torch
    from paper_1912_03312_b200 import rexi_prepare, rexi_run
    d, sysm, ap = load_golden("cfg1_k32")
    stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True)
    ref = rexi_run(stp, d["u0"], 3)
    ut = torch.from_numpy(d["u0"]).cuda()
    p = stp.plans[0]
    p.step_device(ut.data_ptr(), ut.data_ptr(), 3)
    assert np.array_equal(ut.cpu().numpy(), ref)
    stp.close()


@pytest.mark.parametrize("name,refine", [("cfg1_k32", 0), ("cfg1_k32", 1), ("p1_2d_m16", None), ("fem_p2", None)])
def test_observer_states_equal_step_loop(name, refine):
    """rexi_run(observer) produces every state on the device (rexi_plan_run);
    the observer sees exactly the states of a rexi_step loop, each its own array."""
    from paper_1912_03312_b200 import rexi_prepare, rexi_run, rexi_step
    d, sysm, ap = load_golden(name)
    stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True,
                       refine=refine)
    nst = 5
    seen = []
    final = rexi_run(stp, d["u0"], nst, observer=lambda k, t, u: seen.append((k, t, u)))
    assert [k for k, _, _ in seen] == list(range(1, nst + 1))
    assert all(abs(t - k * float(d["tau"])) < 1e-15 for k, t, _ in seen)
    u = d["u0"]
    for k in range(nst):
        u = rexi_step(stp, u)
        assert np.array_equal(seen[k][2], u), k
    assert np.array_equal(final, u)
    assert len({id(s[2]) for s in seen}) == nst
    stp.close()


@pytest.mark.parametrize("steps", [1, 3])
def test_persistent_pinned_buffers_zero_copy(steps):
    """page-locked input and output: the persistent loop reads u and writes
    its last state over the link (no staging copies) -- bitwise equal to
    pageable buffers and to device-resident stepping"""
    import torch
    from paper_1912_03312_b200 import _native, rexi_prepare
    d, sysm, ap = load_golden("cfg1_k32")
    stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True)
    p = stp.plans[0]
    assert p.info.persistent >= 4
    u_pin = _native.host_empty(d["u0"].shape)
    u_pin[:] = d["u0"]
    zc = p.step_host(u_pin, steps)
    staged = p.step_host(np.array(d["u0"]), steps)
    ud = torch.from_numpy(np.array(d["u0"])).cuda()
    out = torch.empty_like(ud)
    p.step_device(ud.data_ptr(), out.data_ptr(), steps)
    assert np.array_equal(zc, staged)
    assert np.array_equal(zc, out.cpu().numpy())
    stp.close()
