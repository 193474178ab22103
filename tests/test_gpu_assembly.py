"""GPU: P1 assembly on the device (csrc/assembly.cu) against
the host assembly it restates (fixtures.assemble_p1_host)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mesh(d, m):
    from paper_1912_03312_b200.fixtures import StructuredMesh
    return StructuredMesh(d, m, np.zeros(d) - 0.5, 1.0 / m)


def _same_structure(a, b):
    assert a.shape == b.shape
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)


@pytest.mark.parametrize("d,m", [(1, 64), (2, 24), (3, 8)])
def test_stiffness_and_mass_bitwise(d, m):
    from paper_1912_03312_b200.assembly import assemble_p1_device
    from paper_1912_03312_b200.fixtures import assemble_p1_host
    mesh = _mesh(d, m)
    zero = lambda x: np.zeros(x.shape[0])   # noqa: E731  (host-evaluated potential path)
    h, g = assemble_p1_host(mesh, zero), assemble_p1_device(mesh, zero)
    _same_structure(h.A, g.A)
    _same_structure(h.B, g.B)
    assert np.array_equal(h.A.data, g.A.data)      # 0.5 K, same summation order
    assert np.array_equal(h.B.data, g.B.data)      # M
    assert h.n_dof == g.n_dof == (m - 1) ** d


@pytest.mark.parametrize("d,m", [(1, 64), (2, 24), (3, 8)])
def test_potential_term_matches_host(d, m):
    from paper_1912_03312_b200.assembly import assemble_p1_device
    from paper_1912_03312_b200.fixtures import _harmonic, assemble_p1_host
    mesh = _mesh(d, m)
    v = _harmonic([0.1] * d, 50.0)
    h, g = assemble_p1_host(mesh, v), assemble_p1_device(mesh, v)
    _same_structure(h.A, g.A)
    assert np.array_equal(h.B.data, g.B.data)
    assert np.max(np.abs(h.A.data - g.A.data)) <= 1e-14 * np.max(np.abs(h.A.data))


def test_fourier_potential_matches_host():
    from paper_1912_03312_b200.assembly import assemble_p1_device
    from paper_1912_03312_b200.fixtures import StructuredMesh, assemble_p1_host, config4_potential
    mesh = StructuredMesh(2, 32, np.zeros(2), 1.0 / 32)
    v = config4_potential(grid_m=32)
    h, g = assemble_p1_host(mesh, v), assemble_p1_device(mesh, v)
    _same_structure(h.A, g.A)
    assert np.max(np.abs(h.A.data - g.A.data)) <= 1e-13 * np.max(np.abs(h.A.data))


def test_fixture_dispatch_uses_device_and_steps():
    """fixtures build 2D/3D pencils on the GPU; REXI on them matches the host-built pencil."""
    from paper_1912_03312_b200 import fixtures, rexi_prepare, rexi_step
    c = fixtures.config3(m=48)        # device assembly (GPU present)
    import os
    os.environ["REXI_FIXTURE_HOST"] = "1"
    try:
        ch = fixtures.config3(m=48)
    finally:
        del os.environ["REXI_FIXTURE_HOST"]
    assert np.max(np.abs(c.system.A.data - ch.system.A.data)) <= 1e-14 * np.max(np.abs(ch.system.A.data))
    s1 = rexi_prepare(c.system, c.approx, c.tau, sr_value=c.sr, override_admissibility=True)
    s2 = rexi_prepare(ch.system, ch.approx, ch.tau, sr_value=ch.sr, override_admissibility=True)
    u1, u2 = rexi_step(s1, c.u0), rexi_step(s2, ch.u0)
    assert np.linalg.norm(u1 - u2) <= 1e-12 * np.linalg.norm(u2)
    s1.close()
    s2.close()
