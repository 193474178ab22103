"""GPU: the drop-in surface beyond the numbers -- phase timers, per-step
stats, the observer's feedback semantics, torch-stream ordering, workers /
devices, and cost-balanced pieces (reference integrate.py:95-140, 193-245,
test_integrate.py:268-305)."""
import numpy as np
import pytest

from conftest import load_golden
from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_run, rexi_step

pytestmark = pytest.mark.gpu


def _prep(cfg, **kw):
    return rexi_prepare(cfg.system, cfg.approx, cfg.tau, sr_value=cfg.sr, override_admissibility=True, **kw)


@pytest.mark.parametrize("builder,kw", [("config1", dict(m=256)), ("config3", dict(m=32)),
                                        ("config2", dict(m=50_000, k=32))])
def test_timers_all_phases_accumulate(builder, kw):
    """timers rhs/local/reduce (integrate.py:110-112, 203-225) all grow"""
    cfg = getattr(fixtures, builder)(**kw)
    with _prep(cfg) as stp:
        rexi_run(stp, cfg.u0, 2)
        t1 = dict(stp.timers)
        assert all(t1[p] > 0.0 for p in ("rhs", "local", "reduce")), t1
        rexi_step(stp, cfg.u0)
        assert all(stp.timers[p] > t1[p] for p in ("rhs", "local", "reduce")), (t1, stp.timers)
        assert stp.stats["steps"] == 3


def test_cocg_stats_every_step():
    cfg = fixtures.config3(m=32)
    with _prep(cfg) as stp:
        rexi_run(stp, cfg.u0, 3)
        ps = stp.stats["per_step"]
        assert [p["step"] for p in ps] == [1, 2, 3]
        for p in ps:
            assert p["iters_max"] > 0 and 0 < p["iters_mean"] <= p["iters_max"]
        its = stp.stats["shift_iters"]
        assert its.shape == (cfg.approx.K,) and its.min() > 0
        assert stp.stats["iters_max"] == its.max()
        assert stp.stats["refine_rounds"] == 1


@pytest.mark.parametrize("builder,kw", [("config1", dict(m=256)), ("config3", dict(m=24))])
def test_observer_mutation_steers_the_run(builder, kw):
    """the reference steps from the array it handed the observer
    (integrate.py:241-244): zeroing it in place makes every later state 0"""
    cfg = getattr(fixtures, builder)(**kw)
    seen = []

    def obs(k, t, u):
        seen.append(np.linalg.norm(u))
        if k == 2:
            u[:] = 0.0
    with _prep(cfg) as stp:
        out = rexi_run(stp, cfg.u0, 4, observer=obs)
    assert seen[0] > 0 and seen[1] > 0 and seen[2] == 0.0 and seen[3] == 0.0
    assert np.all(out == 0)


def test_readonly_observer_fast_path_is_bitwise_equal():
    d, sysm, ap = load_golden("cfg1_k32")
    stp = rexi_prepare(sysm, ap, float(d["tau"]), sr_value=float(d["sr"]), override_admissibility=True)
    a, b = [], []
    ua = rexi_run(stp, d["u0"], 10, observer=lambda k, t, u: a.append((k, t, u.copy())))
    ub = rexi_run(stp, d["u0"], 10, observer=lambda k, t, u: b.append((k, t, u.copy())),
                  readonly_observer=True)
    stp.close()
    assert [x[:2] for x in a] == [x[:2] for x in b]
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x[2], y[2])
    np.testing.assert_array_equal(ua, ub)
    assert ub.base is None or ub.base.size == ub.size     # no pinned chunk kept alive


def test_torch_input_on_a_side_stream():
    """device input produced by a long kernel on a non-default torch stream:
    the plan waits for it (rexi_plan_wait_stream), no stale read"""
    import torch
    cfg = fixtures.config2(m=200_000, k=16)
    with _prep(cfg) as stp:
        ref = rexi_step(stp, cfg.u0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            big = torch.ones((8192, 8192), dtype=torch.float64, device="cuda")
            u = torch.zeros(cfg.system.n_dof, dtype=torch.complex128, device="cuda")
            for _ in range(4):
                big = big @ big * 1e-4               # keep the stream busy
            u += torch.from_numpy(cfg.u0).to("cuda", non_blocking=False)
            out = rexi_step(stp, u)
        s.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy(), ref)


def test_workers_field_and_pieces():
    cfg = fixtures.config1(m=256)
    with _prep(cfg) as stp:
        assert stp.workers == cfg.approx.K            # reference default (integrate.py:161-162)
        assert len(stp.plans) == 1
    with _prep(cfg, workers=5) as stp:
        assert stp.workers == 5 and len(stp.plans) == 5
        assert sorted(sum(stp.pieces, [])) == list(range(cfg.approx.K))


def test_two_slots_rebalance_and_agree():
    """two concurrent slots (devices=[0, 0]: two host threads, two plans on
    separate streams of one GPU -- the multi-GPU code path): after step 1
    the shifts are re-split by measured iterations (LPT) and the answer
    stays the single-piece one to 1e-13"""
    cfg = fixtures.config3(m=40)
    with _prep(cfg) as stp:
        single = rexi_run(stp, cfg.u0, 3)
    with _prep(cfg, devices=[0, 0]) as stp:
        assert len(stp.plans) == 2
        before = [list(p) for p in stp.pieces]
        multi = rexi_run(stp, cfg.u0, 3)
        assert sorted(sum(stp.pieces, [])) == list(range(cfg.approx.K))
        if "rebalanced" in stp.stats:
            assert stp.pieces != before
            assert stp.stats["rebalanced"]["new_max_cost"] < stp.stats["rebalanced"]["old_max_cost"]
        assert len(stp.stats["per_step"]) == 3
    assert np.max(np.abs(multi - single)) <= 1e-13 * np.max(np.abs(single))


def test_singular_shift_named_in_noncontiguous_piece():
    """a cost-balanced (non-contiguous) piece names the global j"""
    from paper_1912_03312_b200 import SolverError, _native
    from paper_1912_03312_b200._pattern import shared_pattern
    from scipy.sparse import csr_matrix, identity
    A = csr_matrix(np.array([[2.0]]))
    B = identity(1, format="csr")
    ip, ix, ar, ai, br = shared_pattern(A, B)
    tau = 1.0
    shifts = np.array([1 + 1j, -2j, 3 + 1j])      # tau*2 - i*(-2j) = 0 -> index 1 singular
    with pytest.raises(SolverError, match="j = 7"):
        _native.NativePlan(ip, ix, ar, br, shifts, np.ones(3, complex), tau, a_imag=ai,
                           shift_ids=np.array([3, 7, 9]))
