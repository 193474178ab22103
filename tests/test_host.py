"""CPU tests of the host-side logic: fixtures, pole sets, the shared CSR
pattern, validation semantics of rexi_prepare / rexi_run that precede any
device work (reference integrate.py:50-88, 157-164, 236-239), sharding, and
the C-ABI library's exported symbols (no compute without a GPU)."""

import ctypes
import json
import math
import os
import re
import subprocess

import numpy as np
import pytest
from scipy.sparse import csr_matrix, diags, identity

from conftest import ROOT
from paper_1912_03312_b200 import (AdmissibilityError, PartialFractionApproximation, SystemMatrices,
                                   approx_from_json, approx_to_json, fixtures, max_step_size,
                                   rexi_prepare, rexi_run)
from paper_1912_03312_b200 import integrate as gi
from paper_1912_03312_b200._pattern import shared_pattern
from paper_1912_03312_b200.distributed import dd_combine_host, shard_indices


# ---------------------------------------------------------------------------
# fixtures (P1 Kuhn assembly)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("d,m", [(1, 17), (2, 9), (3, 5)])
def test_p1_pattern_and_symmetry(d, m):
    mesh = fixtures.StructuredMesh(d, m, np.zeros(d), 1.0 / m)
    sysm = fixtures.assemble_p1(mesh, lambda x: 3.0 + np.sum(x * x, axis=1))
    n = m - 1
    nnz = {1: 3 * n - 2,
           2: n * n + 2 * (2 * n * (n - 1) + (n - 1) ** 2),
           3: n ** 3 + 2 * (3 * n * n * (n - 1) + 3 * n * (n - 1) ** 2 + (n - 1) ** 3)}[d]
    assert sysm.n_dof == n ** d
    assert sysm.A.nnz == sysm.B.nnz == nnz
    assert abs(sysm.B - sysm.B.T).max() == 0
    assert abs(sysm.A - sysm.A.T).max() <= 1e-14 * abs(sysm.A).max()
    np.testing.assert_array_equal(sysm.A.indices, sysm.B.indices)
    # B is SPD and sums to the volume of the interior-supported mass
    assert np.all(np.linalg.eigvalsh(sysm.B.toarray()) > 0)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_quadrature_degree4_exact(d):
    lam, w = fixtures._quad_rule(d)
    assert abs(w.sum() - 1.0) < 1e-14
    # integral over the unit simplex of lam0^a lam1^b = a! b! d! / (a+b+d)!
    for a, b in [(4, 0), (2, 2), (1, 3), (3, 1), (2, 1)]:
        exact = math.factorial(a) * math.factorial(b) * math.factorial(d) / math.factorial(a + b + d)
        got = np.sum(w * lam[:, 0] ** a * lam[:, 1] ** b)
        assert abs(got - exact) < 1e-12


def test_config1_matches_survey_numbers():
    c = fixtures.config1()
    assert c.system.n_dof == 1023 and c.system.A.nnz == 3067
    assert abs(c.sr - 4104.0) < 1.0
    assert abs(np.vdot(c.u0, c.system.B @ c.u0).real - 1.0) < 1e-13
    ratio, _ = gi._admissibility(c.tau, c.sr, c.approx.domain_radius)
    assert abs(ratio - 1.05 * 0.1 * c.sr / 10.0) < 1e-12


def test_pole_sets_roundtrip_and_quality():
    for k in (16, 32, 64, 128):
        a = fixtures.load_poles(k)
        assert a.K == k
        assert len(np.unique(a.shifts)) == k
        assert a.sup_error < 1e-9
        b = approx_from_json(approx_to_json(a))
        np.testing.assert_array_equal(a.shifts, b.shifts)
        np.testing.assert_array_equal(a.weights, b.weights)
        assert a.domain_radius == b.domain_radius
    f = fixtures.load_poles(16)
    assert abs(f.sup_error - 7.839809628702543e-10) < 1e-20   # reference flagship (test_output window)


# ---------------------------------------------------------------------------
# shared pattern
# ---------------------------------------------------------------------------

def test_shared_pattern_union_and_values():
    A = csr_matrix(np.array([[1.0, 0, 2.0], [0, 3.0, 0], [4.0, 0, 5.0]]))
    B = identity(3, format="csr") * 2.0
    ip, ix, a, ai, b = shared_pattern(A, B)
    assert ai is None
    M = csr_matrix((a, ix, ip), shape=(3, 3))
    Bm = csr_matrix((b, ix, ip), shape=(3, 3))
    np.testing.assert_array_equal(M.toarray(), A.toarray())
    np.testing.assert_array_equal(Bm.toarray(), B.toarray())


def test_shared_pattern_complex_a():
    A = csr_matrix(np.array([[1.0 + 2.0j]]))
    ip, ix, a, ai, b = shared_pattern(A, identity(1, format="csr"))
    assert a[0] == 1.0 and ai[0] == 2.0 and b[0] == 1.0


def test_shared_pattern_rejects_complex_b():
    with pytest.raises(ValueError):
        shared_pattern(identity(2, format="csr"), identity(2, format="csr") * 1j)


# ---------------------------------------------------------------------------
# reference validation semantics (no device needed)
# ---------------------------------------------------------------------------

def scalar(omega):
    return SystemMatrices(A=csr_matrix(np.array([[omega]])), B=identity(1, format="csr"), n_dof=1)


def test_max_step_size():
    assert max_step_size(10.0, 1e5) == pytest.approx(1e-4)
    for r1, sr in [(0.0, 1.0), (10.0, 0.0), (10.0, -3.0), (-1.0, 5.0)]:
        with pytest.raises(ValueError):
            max_step_size(r1, sr)


def test_prepare_validates_before_device(flagship):
    with pytest.raises(ValueError):
        rexi_prepare(scalar(1.0), flagship, 0.0, sr_value=1.0)
    with pytest.raises(ValueError):
        rexi_prepare(scalar(1.0), flagship, 1.0, sr_value=1.0, workers=0)
    dup = PartialFractionApproximation(np.array([2 + 1j, 2 + 1j]), np.array([1 + 0j, 1 + 0j]), 10.0, 1.0)
    with pytest.raises(ValueError, match="distinct"):
        rexi_prepare(scalar(1.0), dup, 1.0, sr_value=1.0)
    with pytest.raises(ValueError):
        rexi_prepare(scalar(1.0), flagship, 1.0, sr_value=1.0, solver="lu")


class _FakeStepper:
    def __init__(self, admissible, override):
        self.admissible = admissible
        self.override_admissibility = override
        self.override_used = False
        self.interval_radius = 10.0
        self.sr_value = 5.0
        self.tau = 10.0
        self.admissibility_ratio = 5.25


def test_require_admissible_semantics():
    s = _FakeStepper(False, False)
    with pytest.raises(AdmissibilityError, match="max_step_size"):
        gi._require_admissible("REXI", s)
    s = _FakeStepper(False, True)
    gi._require_admissible("REXI", s)
    assert s.override_used
    s = _FakeStepper(True, False)
    gi._require_admissible("REXI", s)
    assert not s.override_used


def test_run_validation_without_device():
    s = _FakeStepper(False, False)
    with pytest.raises(ValueError):
        rexi_run(s, np.array([1.0 + 0j]), -1)
    with pytest.raises(AdmissibilityError):
        rexi_run(s, np.array([1.0 + 0j]), 1)
    u0 = np.array([0.25 - 0.5j])
    out = rexi_run(s, u0, 0)
    assert out is not u0
    np.testing.assert_array_equal(out, u0)


# ---------------------------------------------------------------------------
# sharding and the fixed-order double-double combine
# ---------------------------------------------------------------------------

def test_shard_indices_contiguous_and_lpt():
    assert shard_indices(10, 3) == [[0, 1, 2, 3], [4, 5, 6], [7, 8, 9]]
    cost = [100, 1, 1, 1, 50, 50]
    sh = shard_indices(6, 2, cost)
    loads = [sum(cost[j] for j in s) for s in sh]
    assert sorted(sum(sh, [])) == list(range(6))
    assert max(loads) == 102


def test_dd_combine_is_order_robust():
    rng = np.random.default_rng(0)
    n, g = 1000, 8
    terms = rng.standard_normal((64, n)) * 1e7
    terms[-1] = -terms[:-1].sum(axis=0) + rng.standard_normal(n)   # cancel to O(1)

    def parts(shards):
        out = np.zeros((len(shards), 4, n))
        for q, idx in enumerate(shards):
            hi = np.zeros(n); lo = np.zeros(n)
            for j in idx:
                s = hi + terms[j]; bb = s - hi
                e = (hi - (s - bb)) + (terms[j] - bb)
                hi, lo = s, lo + e
            out[q, 0], out[q, 1] = hi, lo
        return out
    one = dd_combine_host(parts([list(range(64))]))
    eight = dd_combine_host(parts(shard_indices(64, g)))
    np.testing.assert_array_equal(one, eight)


# ---------------------------------------------------------------------------
# the C ABI library: built, loadable, exports every declared symbol
# ---------------------------------------------------------------------------

def _declared_functions():
    text = open(os.path.join(ROOT, "include", "rexi_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*|int32_t)\s*\*?\s*(rexi_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = _declared_functions()
    for required in ("rexi_plan_create", "rexi_plan_step", "rexi_plan_step_partial",
                     "rexi_combine_partials", "rexi_plan_solve", "rexi_plan_destroy"):
        assert required in names


def test_library_exports_all_declared_symbols():
    from paper_1912_03312_b200 import build_native
    lib = build_native.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rexi_\w+)", out))
    missing = [s for s in _declared_functions() if s not in exported]
    assert not missing, missing
    L = ctypes.CDLL(lib)
    L.rexi_abi_version.restype = ctypes.c_int32
    from paper_1912_03312_b200 import _native
    assert L.rexi_abi_version() == _native.ABI_VERSION == 3
    assert set(_declared_functions()) <= set(_native.EXPORTED) | {"rexi_abi_version"}


def test_library_is_sm100a_only():
    from paper_1912_03312_b200 import build_native
    lib = build_native.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_rejects_bad_descriptor_without_gpu():
    from paper_1912_03312_b200 import _native
    with pytest.raises(ValueError):
        _native.NativePlan(np.array([0, 1], np.int32), np.array([0], np.int32), np.array([1.0]),
                           np.array([1.0]), np.array([1 + 1j]), np.array([1 + 0j]), tau=-1.0)


def test_pencil_create_rejects_bad_descriptor_without_gpu():
    from paper_1912_03312_b200 import _native
    with pytest.raises(ValueError, match="column index"):
        _native.NativePencil(np.array([0, 1], np.int32), np.array([3], np.int32), np.array([1.0]),
                             np.array([1.0]))
    with pytest.raises(ValueError, match="nnz"):
        _native.NativePencil(np.array([0, 2], np.int32), np.array([0], np.int32), np.array([1.0]),
                             np.array([1.0]))


def test_solver_selection_policy_without_device():
    """rexi_prepare's host-side policies: default refinement (direct solvers
    refine on stiff pencils only, COCG always) and the per-plan shift limit
    that makes it split K into more pieces"""
    from scipy.sparse import diags
    from paper_1912_03312_b200._pattern import shared_pattern
    from paper_1912_03312_b200.integrate import default_refine, max_shifts_per_plan
    n = 50
    tri = diags([np.ones(n - 1), 2 * np.ones(n), np.ones(n - 1)], [-1, 0, 1]).tocsr()
    penta = diags([np.ones(n - 2), np.ones(n - 1), 4 * np.ones(n), np.ones(n - 1), np.ones(n - 2)],
                  [-2, -1, 0, 1, 2]).tocsr()
    wide = diags([np.ones(n - 7), 4 * np.ones(n), np.ones(n - 7)], [-7, 0, 7]).tocsr()
    for mat, stiff_refine, cap in ((tri, 1, 256), (penta, 1, 1024), (wide, 1, None)):
        ip, ix = shared_pattern(mat, mat)[:2]
        assert default_refine(ip, ix, 1.0, 1e6) == stiff_refine
        lim = max_shifts_per_plan(ip, ix)
        if cap is not None:
            assert lim == cap
        else:
            assert lim >= 1024 and lim & (lim - 1) == 0 and lim * n < 2 ** 31
    ip, ix = shared_pattern(tri, tri)[:2]
    assert default_refine(ip, ix, 1.0, 10.0) == 0            # non-stiff 1D: fp64 suffices
    assert default_refine(ip, ix, 1.0, 10.0, "cocg") == 1    # COCG always refines
    ip, ix = shared_pattern(penta, penta)[:2]
    assert default_refine(ip, ix, 1.0, 10.0) == 0            # P2 band, non-stiff
