"""Synthetic inputs for the five BASELINE.json configs (builder-side code).

The reference discretises 1D with P2 elements only (``spatial.py:1-16``);
BASELINE.json asks for P1 pencils in 1D, 2D and 3D, so the assembly here
is new fixture code.  The hot path only consumes the resulting
``SystemMatrices(A, B, n_dof)`` (reference ``spatial.py:130-136``).

Conventions follow the reference (``spatial.py:193-223``): hbar = m = 1,
A = 0.5 * stiffness + potential-weighted mass, B = mass, Dirichlet nodes
eliminated, u0 = nodal interpolant scaled so that u^H B u = 1
(``spatial.py:245-270``).

Meshes are structured Kuhn (Freudenthal) simplicial meshes: the unit cell
of the tensor grid is split into d! simplices, one per permutation of the
axes (1D: intervals; 2D: two triangles sharing the (0,0)-(1,1) diagonal;
3D: six tetrahedra).  Every element is a translate of one of d! templates,
so stiffness and mass element matrices are per-template constants and
only the potential term varies.  Potential integrals use fixed rules:
1D 4-point Gauss-Legendre, 2D 6-point Dunavant (degree 4), 3D 11-point
Keast (degree 4).  RNG draws use ``numpy.random.default_rng(seed)`` in the
order documented in each builder.
"""

from __future__ import annotations

import itertools
import math
import os
from dataclasses import dataclass

import numpy as np
from scipy.sparse import csr_matrix

from .types import SystemMatrices, approx_from_json

_POLE_DIR = os.path.join(os.path.dirname(__file__), "poles")


# ---------------------------------------------------------------------------
# Quadrature on the reference simplex (barycentric points, weights sum to 1)
# ---------------------------------------------------------------------------

def _quad_rule(d: int):
    if d == 1:
        x, w = np.polynomial.legendre.leggauss(4)
        t = 0.5 * (x + 1.0)
        return np.stack([1.0 - t, t], axis=1), 0.5 * w
    if d == 2:
        a1, b1, w1 = 0.108103018168070, 0.445948490915965, 0.223381589678011
        a2, b2, w2 = 0.816847572980459, 0.091576213509771, 0.109951743655322
        pts = []
        for a, b in ((a1, b1), (a2, b2)):
            pts += [(a, b, b), (b, a, b), (b, b, a)]
        return np.array(pts), np.array([w1] * 3 + [w2] * 3)
    if d == 3:
        s = math.sqrt(5.0 / 14.0)
        a, b = (1.0 + s) / 4.0, (1.0 - s) / 4.0
        pts = [(0.25, 0.25, 0.25, 0.25)]
        w = [-148.0 / 1875.0]
        for k in range(4):
            p = [1.0 / 14.0] * 4
            p[k] = 11.0 / 14.0
            pts.append(tuple(p))
            w.append(343.0 / 7500.0)
        for i, j in itertools.combinations(range(4), 2):
            p = [b] * 4
            p[i] = a
            p[j] = a
            pts.append(tuple(p))
            w.append(56.0 / 375.0)
        return np.array(pts), np.array(w)
    raise ValueError(f"unsupported dimension {d}")


def kuhn_templates(d: int):
    """Vertex offsets (d+1, d) of the d! Kuhn simplices of the unit cell."""
    temps = []
    for perm in itertools.permutations(range(d)):
        verts = [np.zeros(d, dtype=np.int64)]
        for k in perm:
            v = verts[-1].copy()
            v[k] += 1
            verts.append(v)
        temps.append(np.array(verts))
    return temps


def _template_blocks(verts: np.ndarray):
    """Unit-scale (h = 1) stiffness and mass element matrices of a simplex."""
    d = verts.shape[1]
    jac = (verts[1:] - verts[0]).T.astype(float)         # columns v_k - v_0
    inv = np.linalg.inv(jac)
    grads = np.vstack([-inv.sum(axis=0), inv])            # (d+1, d)
    grads = np.rint(grads)                                # exact: integer Kuhn gradients
    vol = 1.0 / math.factorial(d)
    stiff = vol * (grads @ grads.T)
    mass = vol / ((d + 1) * (d + 2)) * (np.ones((d + 1, d + 1)) + np.eye(d + 1))
    return stiff, mass, vol


# ---------------------------------------------------------------------------
# Structured P1 assembly
# ---------------------------------------------------------------------------

@dataclass
class StructuredMesh:
    d: int
    m: int                 # cells per axis
    lo: np.ndarray         # (d,) lower corner
    h: float

    @property
    def n_interior(self) -> int:
        return (self.m - 1) ** self.d

    def interior_coords(self) -> np.ndarray:
        axes = [self.lo[k] + self.h * np.arange(1, self.m) for k in range(self.d)]
        grids = np.meshgrid(*axes, indexing="ij")
        return np.stack([g.ravel() for g in grids], axis=1)


def _use_device() -> bool:
    if os.environ.get("REXI_FIXTURE_HOST"):
        return False
    try:
        import torch
        from . import _native
        return torch.cuda.is_available() and os.path.exists(_native.LIB_PATH)
    except Exception:
        return False


def assemble_p1(mesh: StructuredMesh, potential) -> SystemMatrices:
    """The pencil on the GPU when one is available (assembly.assemble_p1_device,
    SURVEY 8(f)4), else on the host (assemble_p1_host)."""
    if mesh.d > 1 and _use_device():
        from .assembly import assemble_p1_device
        return assemble_p1_device(mesh, potential)
    return assemble_p1_host(mesh, potential)


def assemble_p1_host(mesh: StructuredMesh, potential) -> SystemMatrices:
    """A = 0.5*K + M_V, B = M on interior nodes, CSR with sorted columns.

    ``potential(x)`` takes points (n, d) and returns V (n,).  Stencil
    offsets of a Kuhn mesh lie in {-1,0,1}^d with all nonzero components of
    equal sign (3 in 1D, 7 in 2D, 15 in 3D); every offset is stored even
    where an entry happens to be zero, so A and B share one CSR pattern.
    """
    d, m, h = mesh.d, mesh.m, mesh.h
    shape = (m + 1,) * d
    temps = kuhn_templates(d)
    lam, wq = _quad_rule(d)
    offsets = sorted({tuple(int(x) for x in (t[b] - t[a]))
                      for t in temps for a in range(d + 1) for b in range(d + 1)})
    stiff_g = {o: np.zeros(shape) for o in offsets}
    mass_g = {o: np.zeros(shape) for o in offsets}
    pot_g = {o: np.zeros(shape) for o in offsets}

    cell_axes = [np.arange(m, dtype=float) for _ in range(d)]
    cell_grid = np.meshgrid(*cell_axes, indexing="ij")
    cell_lo = np.stack([g.ravel() for g in cell_grid], axis=1)   # (m^d, d) in cells
    del cell_grid
    for t in temps:
        stiff_u, mass_u, vol = _template_blocks(t)
        stiff_e = stiff_u * h ** (d - 2)
        mass_e = mass_u * h ** d
        # potential element matrices: vol h^d sum_q w_q V(x_q) lam_a lam_b
        vq = np.empty((cell_lo.shape[0], len(wq)))
        for q in range(len(wq)):
            off = lam[q] @ t.astype(float)                 # quadrature point, in cell units
            if hasattr(potential, "on_cells"):
                vq[:, q] = potential.on_cells(mesh, off)   # separable fast path
            else:
                vq[:, q] = potential(mesh.lo + h * (cell_lo + off))
        coef = wq[:, None, None] * lam[:, :, None] * lam[:, None, :]   # (nq, d+1, d+1)
        pot_e = (vq @ coef.reshape(len(wq), -1)) * (vol * h ** d)
        pot_e = pot_e.reshape((m,) * d + (d + 1, d + 1))
        for a in range(d + 1):
            sl = tuple(slice(int(t[a][k]), int(t[a][k]) + m) for k in range(d))
            for b in range(d + 1):
                o = tuple(int(x) for x in (t[b] - t[a]))
                stiff_g[o][sl] += stiff_e[a, b]
                mass_g[o][sl] += mass_e[a, b]
                pot_g[o][sl] += pot_e[..., a, b]
        del vq, pot_e
    del cell_lo

    n1 = m - 1
    inner = tuple(slice(1, m) for _ in range(d))
    n_int = n1 ** d
    idx_grid = np.meshgrid(*[np.arange(1, m) for _ in range(d)], indexing="ij")
    strides = [n1 ** (d - 1 - k) for k in range(d)]
    rows_lin = np.arange(n_int, dtype=np.int64)
    # sort offsets by their linear column delta so CSR columns come out sorted
    offsets.sort(key=lambda o: sum(o[k] * strides[k] for k in range(d)))
    masks, a_cols, b_cols, c_cols = [], [], [], []
    for o in offsets:
        ok = np.ones(n_int, dtype=bool)
        for k in range(d):
            nb = idx_grid[k].ravel() + o[k]
            ok &= (nb >= 1) & (nb <= m - 1)
        masks.append(ok)
        a_cols.append((0.5 * stiff_g[o][inner] + pot_g[o][inner]).ravel())
        b_cols.append(mass_g[o][inner].ravel())
        c_cols.append(rows_lin + sum(o[k] * strides[k] for k in range(d)))
    mask = np.stack(masks, axis=1)
    counts = mask.sum(axis=1)
    indptr = np.zeros(n_int + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    flat = mask.ravel()
    a_data = np.stack(a_cols, axis=1).ravel()[flat]
    b_data = np.stack(b_cols, axis=1).ravel()[flat]
    cols = np.stack(c_cols, axis=1).ravel()[flat].astype(np.int32)
    indptr = indptr.astype(np.int32)
    a_mat = csr_matrix((a_data, cols, indptr), shape=(n_int, n_int))
    b_mat = csr_matrix((b_data, cols.copy(), indptr.copy()), shape=(n_int, n_int))
    a_mat.has_sorted_indices = True
    b_mat.has_sorted_indices = True
    return SystemMatrices(A=a_mat, B=b_mat, n_dof=n_int)


def normalized_packet(mesh: StructuredMesh, b_mat, center, std, wavevec) -> np.ndarray:
    """Nodal interpolant of exp(-|x-c|^2/(2 std^2)) e^{i k.x}, scaled so
    u^H B u = 1 (reference ``spatial.py:245-290`` convention, hbar = 1)."""
    x = mesh.interior_coords()
    dx = x - np.asarray(center, dtype=float)
    phase = x @ np.asarray(wavevec, dtype=float)
    u = np.exp(-np.sum(dx * dx, axis=1) / (2.0 * std * std) + 1j * phase)
    quad = complex(np.vdot(u, b_mat @ u))
    return u / math.sqrt(quad.real)


# ---------------------------------------------------------------------------
# Spectral radius of M = (iB)^-1 A
# ---------------------------------------------------------------------------

def element_sr_bound(mesh: StructuredMesh, v_max: float) -> float:
    """Upper bound sr(M) <= max_e lambda_max(A_e, B_e) <= 0.5*max lambda(K_e, M_e) + v_max.

    Assembled Rayleigh quotients are bounded by the worst element quotient;
    used for the large 2D/3D configs where the reference's estimator
    (``spatial.py:314-344``) would need a dense factorisation of B.
    """
    worst = 0.0
    for t in kuhn_templates(mesh.d):
        stiff_u, mass_u, _ = _template_blocks(t)
        ev = np.linalg.eigvals(np.linalg.solve(mass_u, stiff_u)).real.max()
        worst = max(worst, ev)
    return 0.5 * worst / mesh.h ** 2 + v_max


def power_sr_1d(sys_m: SystemMatrices, iters: int = 400, tol: float = 1e-6, seed: int = 0) -> float:
    """Power iteration on B^-1 A with B-Rayleigh quotients (the reference's
    algorithm, ``spatial.py:314-344``) using a banded B solve; 1D only."""
    from scipy.linalg import solve_banded
    b = sys_m.B
    n = sys_m.n_dof
    ab = np.zeros((3, n))
    ab[0, 1:] = b.diagonal(1)
    ab[1, :] = b.diagonal(0)
    ab[2, :-1] = b.diagonal(-1)
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    rq_prev, rq = None, 0.0
    for _ in range(iters):
        av = sys_m.A @ v
        rq = abs(np.dot(v, av) / np.dot(v, b @ v))
        if rq_prev is not None and abs(rq - rq_prev) <= tol * max(rq, 1e-300):
            break
        rq_prev = rq
        w = solve_banded((1, 1), ab, av)
        v = w / np.linalg.norm(w)
    return float(rq)


# ---------------------------------------------------------------------------
# Pole sets (frozen JSON, generated by tests/golden/make_golden.py)
# ---------------------------------------------------------------------------

POLE_SETS = {
    16: "flagship_k16.json",
    32: "ensemble_k32.json",
    64: "ensemble_k64.json",
    128: "ensemble_k128.json",
}


def load_poles(k_or_name):
    """Frozen pole/weight set: 16 = reference flagship faber_cf(R1=10);
    32/64/128 = ensembles of degree-16 generator outputs."""
    name = POLE_SETS.get(k_or_name, k_or_name)
    with open(os.path.join(_POLE_DIR, name)) as fh:
        return approx_from_json(fh.read())


# ---------------------------------------------------------------------------
# The five BASELINE.json configs
# ---------------------------------------------------------------------------

@dataclass
class Config:
    name: str
    system: SystemMatrices
    u0: np.ndarray
    approx: object
    tau: float
    n_steps: int
    sr: float
    mesh: StructuredMesh


def _cell_axis(mesh, k, off, dev):
    """Coordinates lo_k + h (i + off_k) of the cells along axis k (device),
    in the host formula's operation order."""
    import torch
    i = torch.arange(mesh.m, dtype=torch.float64, device=dev)
    return mesh.lo[k] + mesh.h * (i + float(off[k]))


class _Harmonic:
    """V = coef |x - c|^2; device_on_cells evaluates all cells at one
    quadrature offset on the GPU (same operation order as __call__)."""

    def __init__(self, center, coef):
        self.c = np.asarray(center, dtype=float)
        self.coef = coef

    def __call__(self, x):
        dx = x - self.c
        return self.coef * np.sum(dx * dx, axis=1)

    def device_on_cells(self, mesh, off, dev):
        import torch
        d = mesh.d
        s = None
        for k in range(d):
            dx = _cell_axis(mesh, k, off, dev) - float(self.c[k])
            shape = [1] * d
            shape[k] = mesh.m
            term = (dx * dx).reshape(shape)
            s = term if s is None else s + term
        return (self.coef * s).reshape(-1)


def _harmonic(center, coef):
    return _Harmonic(center, coef)


def config1(m: int = 1024, k: int = 32) -> Config:
    """1D P1 on [-20, 20], m elements (m+1 = 1025 nodes), V = x^2/2,
    u0 ~ exp(-(x+5)^2/2) e^{2ix}, tau = 0.1, K = 32, 10 steps."""
    mesh = StructuredMesh(1, m, np.array([-20.0]), 40.0 / m)
    sysm = assemble_p1(mesh, _harmonic([0.0], 0.5))
    u0 = normalized_packet(mesh, sysm.B, [-5.0], 1.0, [2.0])
    sr = power_sr_1d(sysm)
    return Config("cfg1", sysm, u0, load_poles(k), 0.1, 10, sr, mesh)


def config2_potential(seed: int = 1912):
    """Draw order: a[16] ~ U(0,1), phi[16] ~ U(0,2pi), center ~ U(-100,100),
    std ~ U(2,6), wavenumber ~ U(-1.5,1.5)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.0, 1.0, 16)
    phi = rng.uniform(0.0, 2.0 * math.pi, 16)
    center = rng.uniform(-100.0, 100.0)
    std = rng.uniform(2.0, 6.0)
    kw = rng.uniform(-1.5, 1.5)
    modes = np.arange(1, 17)

    class Fourier1D:
        def __call__(self, x):
            arg = 2.0 * math.pi * np.outer(x[:, 0] + 200.0, modes) / 400.0 + phi
            return np.cos(arg) @ a

        def device_on_cells(self, mesh, off, dev):
            import torch
            x = _cell_axis(mesh, 0, off, dev)
            md = torch.from_numpy(modes.astype(float)).to(dev)
            arg = 2.0 * math.pi * torch.outer(x + 200.0, md) / 400.0 + torch.from_numpy(phi).to(dev)
            return torch.cos(arg) @ torch.from_numpy(a).to(dev)

    return Fourier1D(), center, std, kw, float(np.sum(a))


def config2(m: int = 2 ** 20 - 1, k: int = 64, sr: float | None = None) -> Config:
    """1D P1 on [-200, 200] with 2^20 nodes, 16 random Fourier modes
    (seed 1912), K = 64, tau = 0.5, 20 steps."""
    mesh = StructuredMesh(1, m, np.array([-200.0]), 400.0 / m)
    v, center, std, kw, vmax = config2_potential()
    sysm = assemble_p1(mesh, v)
    u0 = normalized_packet(mesh, sysm.B, [center], std, [kw])
    if sr is None:
        sr = 6.0 / mesh.h ** 2 + vmax     # lambda_max(M^-1 K) = 12/h^2 for uniform P1
    return Config("cfg2", sysm, u0, load_poles(k), 0.5, 20, sr, mesh)


def config3(m: int = 1024, k: int = 64) -> Config:
    """2D P1 unit square, m x m cells x 2 triangles, V = 50|x-c|^2,
    packet c=(.5,.5), std .05, k=(20,10), K = 64, tau = 1e-3, 10 steps."""
    mesh = StructuredMesh(2, m, np.zeros(2), 1.0 / m)
    sysm = assemble_p1(mesh, _harmonic([0.5, 0.5], 50.0))
    u0 = normalized_packet(mesh, sysm.B, [0.5, 0.5], 0.05, [20.0, 10.0])
    sr = element_sr_bound(mesh, 50.0 * 0.5)
    return Config("cfg3", sysm, u0, load_poles(k), 1e-3, 10, sr, mesh)


def config4_potential(seed: int = 3312, grid_m: int = 2048):
    """Draw order: (p,q)[64] integers in [-8,8]^2 (rows equal to (0,0)
    redrawn in place, in order), a[64] ~ U(0,1), phi[64] ~ U(0,2pi).
    V = 1e3 * F / max|F| with the max taken over the (grid_m+1)^2 nodes."""
    rng = np.random.default_rng(seed)
    pq = rng.integers(-8, 9, size=(64, 2))
    for i in range(64):
        while pq[i, 0] == 0 and pq[i, 1] == 0:
            pq[i] = rng.integers(-8, 9, size=2)
    a = rng.uniform(0.0, 1.0, 64)
    phi = rng.uniform(0.0, 2.0 * math.pi, 64)

    c = a * np.exp(1j * phi)

    class FourierPotential:
        """V = 1e3 F / max|F|; on_cells() evaluates all cells at one offset as
        Re(X diag(c) Y^T) with X[i,m] = exp(2 pi i p_m x_i), Y[j,m] likewise
        (each mode factorises per axis)."""

        def __init__(self):
            self.scale = 1.0

        def f(self, x):
            arg = 2.0 * math.pi * (np.outer(x[:, 0], pq[:, 0]) + np.outer(x[:, 1], pq[:, 1])) + phi
            return np.cos(arg) @ a

        def f_grid(self, xs, ys):
            X = np.exp(2j * math.pi * np.outer(xs, pq[:, 0]))
            Y = np.exp(2j * math.pi * np.outer(ys, pq[:, 1]))
            return ((X * c) @ Y.T).real                    # [i, j]

        def __call__(self, x):
            return self.scale * self.f(x)

        def on_cells(self, mesh, off):
            m, h = mesh.m, mesh.h
            xs = mesh.lo[0] + h * (np.arange(m) + off[0])
            ys = mesh.lo[1] + h * (np.arange(m) + off[1])
            return self.scale * self.f_grid(xs, ys).ravel()

        def device_on_cells(self, mesh, off, dev):
            import torch
            xs, ys = _cell_axis(mesh, 0, off, dev), _cell_axis(mesh, 1, off, dev)
            p = torch.from_numpy(pq[:, 0].astype(float)).to(dev)
            q = torch.from_numpy(pq[:, 1].astype(float)).to(dev)
            X = torch.exp(2j * math.pi * torch.outer(xs, p).to(torch.complex128))
            Y = torch.exp(2j * math.pi * torch.outer(ys, q).to(torch.complex128))
            cc = torch.from_numpy(c).to(dev)
            return self.scale * ((X * cc) @ Y.T).real.reshape(-1)

    v = FourierPotential()
    g = np.linspace(0.0, 1.0, grid_m + 1)
    fmax = float(np.max(np.abs(v.f_grid(g, g))))
    v.scale = 1e3 / fmax
    return v


def config4(m: int = 2048, k: int = 128) -> Config:
    """2D P1, m x m cells, disordered V (64 seeded Fourier modes, amplitude
    1e3), packet c=(.5,.5), std .05, k=(20,10), K = 128, tau = 5e-4, 10 steps."""
    mesh = StructuredMesh(2, m, np.zeros(2), 1.0 / m)
    v = config4_potential(grid_m=m)
    sysm = assemble_p1(mesh, v)
    u0 = normalized_packet(mesh, sysm.B, [0.5, 0.5], 0.05, [20.0, 10.0])
    sr = element_sr_bound(mesh, 1e3)
    return Config("cfg4", sysm, u0, load_poles(k), 5e-4, 10, sr, mesh)


def config5(m: int = 128, k: int = 64) -> Config:
    """3D P1 unit cube, m^3 cells x 6 Kuhn tets, V = 30|x-c|^2, packet
    c=(.5,.5,.5), std .07, k=(10,5,0), K = 64, tau = 1e-3, 5 steps."""
    mesh = StructuredMesh(3, m, np.zeros(3), 1.0 / m)
    sysm = assemble_p1(mesh, _harmonic([0.5, 0.5, 0.5], 30.0))
    u0 = normalized_packet(mesh, sysm.B, [0.5, 0.5, 0.5], 0.07, [10.0, 5.0, 0.0])
    sr = element_sr_bound(mesh, 30.0 * 0.75)
    return Config("cfg5", sysm, u0, load_poles(k), 1e-3, 5, sr, mesh)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}
FULL_M = {3: 1024, 4: 2048, 5: 128}
V_MAX = {3: 50.0 * 0.5, 4: 1e3, 5: 30.0 * 0.75}


def stiffness_matched(idx: int, m: int) -> Config:
    """Config idx (3, 4 or 5) on an m-cell mesh with tau scaled so that
    tau * sr(M) equals the full-size config's (1.89e4 / 3.77e4 / 559): the
    shifted systems keep the BASELINE conditioning (and the COCG iteration
    counts it drives) at a size a CPU truth oracle solves in seconds."""
    cfg = CONFIGS[idx](m=m)
    d = cfg.mesh.d
    full = StructuredMesh(d, FULL_M[idx], np.zeros(d), 1.0 / FULL_M[idx])
    tau_full = {3: 1e-3, 4: 5e-4, 5: 1e-3}[idx]
    target = tau_full * element_sr_bound(full, V_MAX[idx])
    cfg.tau = target / cfg.sr
    cfg.name = f"{cfg.name}@m={m},tau*sr={target:.4g}"
    return cfg


def build_config(idx: int, **kw) -> Config:
    return CONFIGS[idx](**kw)
