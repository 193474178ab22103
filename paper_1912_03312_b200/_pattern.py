"""Host-side preparation of the shared CSR pattern of A and B.

The reference forms ``tau*A - (1j*sigma)*B`` with scipy sparse arithmetic
(``integrate.py:171``), i.e. on the union of the two patterns.  The native
plan takes one pattern and both value arrays on it.
"""

from __future__ import annotations

import numpy as np
from scipy.sparse import csr_matrix, issparse


def _as_csr(m):
    if issparse(m):
        return m.tocsr()
    return csr_matrix(np.asarray(m))


def shared_pattern(A, B):
    """Return (indptr int32, indices int32, a_re, a_im or None, b_re).

    A may be complex (the reference's singular-shift test uses one); B must
    be real (the reference's mass matrix).
    """
    A = _as_csr(A)
    B = _as_csr(B)
    if A.shape != B.shape or A.shape[0] != A.shape[1]:
        raise ValueError(f"A and B must be square and of equal shape, got {A.shape}, {B.shape}")
    if np.iscomplexobj(B.data) and np.any(np.imag(B.data) != 0):
        raise ValueError("complex B is not supported (the reference's B is the real mass matrix)")
    n = A.shape[0]
    A.sum_duplicates()
    B.sum_duplicates()
    if A.has_sorted_indices and B.has_sorted_indices and A.nnz == B.nnz and \
            np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices):
        indptr, indices = A.indptr, A.indices
        a = A.data
        b = np.real(B.data).astype(np.float64)
    else:
        P = (abs(A) + abs(B)).tocsr()
        P.sort_indices()
        indptr, indices = P.indptr, P.indices
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
        key = rows * n + indices

        def on_pattern(M):
            M = M.tocoo()
            mk = M.row.astype(np.int64) * n + M.col
            out = np.zeros(len(key), dtype=M.data.dtype)
            np.add.at(out, np.searchsorted(key, mk), M.data)
            return out
        a = on_pattern(A)
        b = np.real(on_pattern(B)).astype(np.float64)
    a_re = np.ascontiguousarray(np.real(a), dtype=np.float64)
    a_im = None
    if np.iscomplexobj(a) and np.any(np.imag(a) != 0):
        a_im = np.ascontiguousarray(np.imag(a), dtype=np.float64)
    return (np.ascontiguousarray(indptr, dtype=np.int32),
            np.ascontiguousarray(indices, dtype=np.int32), a_re, a_im,
            np.ascontiguousarray(b, dtype=np.float64))
