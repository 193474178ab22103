"""P1 assembly of the pencil on the GPU.

The reference assembles its pencils on the host (scipy COO sums,
``spatial.py:143-223``; 1D P2 only).  The 2D/3D configurations are P1 on
structured Kuhn meshes (``fixtures.py``); their host assembly
(``fixtures.assemble_p1``) takes ~25 s at 128^3.  :func:`assemble_p1_device`
builds the same CSR pencil on the GPU:

* the potential at the quadrature points is evaluated on the device when the
  potential object provides ``device_on_cells(mesh, off)`` (torch), otherwise
  on the host and uploaded;
* the element potential matrices are one batched product per template;
* ``rexi_assemble_p1`` (``csrc/assembly.cu``) gathers every (row, stencil
  offset) entry from the element contributions in the host's accumulation
  order, so K and M are bitwise identical to the host assembly and the
  potential term agrees to rounding.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
from scipy.sparse import csr_matrix

from . import _native
from .types import SystemMatrices


def _contribution_table(mesh):
    """Stencil offsets (sorted by column delta) and the (t, a, b) element
    contributions of each, in fixtures.assemble_p1's accumulation order."""
    from .fixtures import _template_blocks, kuhn_templates
    d, m, h = mesh.d, mesh.m, mesh.h
    temps = kuhn_templates(d)
    n1 = m - 1
    strides = [n1 ** (d - 1 - k) for k in range(d)]
    offsets = sorted({tuple(int(x) for x in (t[b] - t[a]))
                      for t in temps for a in range(d + 1) for b in range(d + 1)})
    offsets.sort(key=lambda o: sum(o[k] * strides[k] for k in range(d)))
    blocks = []
    for t in temps:
        stiff_u, mass_u, vol = _template_blocks(t)
        blocks.append((stiff_u * h ** (d - 2), mass_u * h ** d, vol))
    start, ct, ca, cb, cva, cs, cm = [0], [], [], [], [], [], []
    for o in offsets:
        for ti, t in enumerate(temps):
            for a in range(d + 1):
                for b in range(d + 1):
                    if tuple(int(x) for x in (t[b] - t[a])) != o:
                        continue
                    ct.append(ti)
                    ca.append(a)
                    cb.append(b)
                    cva.extend(int(x) for x in t[a])
                    cs.append(blocks[ti][0][a, b])
                    cm.append(blocks[ti][1][a, b])
        start.append(len(ct))
    return temps, blocks, offsets, start, ct, ca, cb, cva, cs, cm


def _potential_on_cells(mesh, potential, off, dev):
    """V at cell_lo + off (cell units) for all m^d cells, as a device tensor."""
    import torch
    if hasattr(potential, "device_on_cells"):
        return potential.device_on_cells(mesh, off, dev)
    if hasattr(potential, "on_cells"):
        v = potential.on_cells(mesh, off)
    else:
        d, m, h = mesh.d, mesh.m, mesh.h
        axes = [np.arange(m, dtype=float) for _ in range(d)]
        grid = np.meshgrid(*axes, indexing="ij")
        cell_lo = np.stack([g.ravel() for g in grid], axis=1)
        v = potential(mesh.lo + h * (cell_lo + off))
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(dev)


def assemble_p1_device(mesh, potential, device: int = 0) -> SystemMatrices:
    """A = 0.5*K + M_V, B = M on the interior nodes (the same pencil as
    fixtures.assemble_p1), assembled on CUDA device ``device``."""
    import torch
    from .fixtures import _quad_rule
    d, m, h = mesh.d, mesh.m, mesh.h
    dev = torch.device("cuda", device)
    temps, blocks, offsets, start, ct, ca, cb, cva, cs, cm = _contribution_table(mesh)
    lam, wq = _quad_rule(d)
    coef = torch.from_numpy((wq[:, None, None] * lam[:, :, None] * lam[:, None, :]).reshape(len(wq), -1)).to(dev)
    ncell = m ** d
    pot_e = torch.empty((len(temps), ncell, (d + 1) ** 2), dtype=torch.float64, device=dev)
    for ti, t in enumerate(temps):
        vq = torch.empty((ncell, len(wq)), dtype=torch.float64, device=dev)
        for q in range(len(wq)):
            vq[:, q] = _potential_on_cells(mesh, potential, lam[q] @ t.astype(float), dev)
        torch.matmul(vq, coef, out=pot_e[ti])
        pot_e[ti] *= blocks[ti][2] * h ** d
        del vq
    n1 = m - 1
    n_int = n1 ** d
    nnz = int(sum(math.prod(n1 - abs(o[k]) for k in range(d)) for o in offsets))
    indptr = torch.empty(n_int + 1, dtype=torch.int32, device=dev)
    indices = torch.empty(nnz, dtype=torch.int32, device=dev)
    a_vals = torch.empty(nnz, dtype=torch.float64, device=dev)
    b_vals = torch.empty(nnz, dtype=torch.float64, device=dev)
    keep = [np.ascontiguousarray(x, dtype=np.int32) for x in
            ([c for o in offsets for c in o], start, ct, ca, cb, cva)]
    keep += [np.ascontiguousarray(cs, dtype=np.float64), np.ascontiguousarray(cm, dtype=np.float64)]
    desc = _native.RexiP1Desc()
    desc.d, desc.m, desc.n_templates = d, m, len(temps)
    desc.n_off = len(offsets)
    desc.offsets = keep[0].ctypes.data
    desc.n_contrib = len(ct)
    desc.contrib_start = keep[1].ctypes.data
    desc.contrib_t = keep[2].ctypes.data
    desc.contrib_a = keep[3].ctypes.data
    desc.contrib_b = keep[4].ctypes.data
    desc.contrib_va = keep[5].ctypes.data
    desc.contrib_stiff = keep[6].ctypes.data
    desc.contrib_mass = keep[7].ctypes.data
    desc.device = device
    desc.stream = torch.cuda.current_stream(dev).cuda_stream
    L = _native.lib()
    rc = L.rexi_assemble_p1(ctypes.byref(desc), ctypes.c_void_p(pot_e.data_ptr()),
                            ctypes.c_void_p(indptr.data_ptr()), ctypes.c_void_p(indices.data_ptr()),
                            ctypes.c_void_p(a_vals.data_ptr()), ctypes.c_void_p(b_vals.data_ptr()))
    _native.raise_status(rc, L.rexi_last_error().decode())
    del pot_e
    ip, ix = indptr.cpu().numpy(), indices.cpu().numpy()
    a_mat = csr_matrix((a_vals.cpu().numpy(), ix, ip), shape=(n_int, n_int))
    b_mat = csr_matrix((b_vals.cpu().numpy(), ix.copy(), ip.copy()), shape=(n_int, n_int))
    a_mat.has_sorted_indices = True
    b_mat.has_sorted_indices = True
    return SystemMatrices(A=a_mat, B=b_mat, n_dof=n_int)
