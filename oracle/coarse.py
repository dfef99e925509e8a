"""Oracle: subspace bases as explicit sparse matrices and the Galerkin coarse systems.

Test infrastructure only (see oracle/__init__.py).

* Eq. 7: x = sum_i phi_i(X) P_i(X - X_i) q_i, P_i = I3 kron [1 x y z],
  so the 3x12 block of vertex v and handle i is I3 kron (phi_i(v) [1, X_v - c_i]) and the
  12 coordinates of q_i are ordered [x-row(4), y-row(4), z-row(4)].
* U_s stacks these blocks (L356-362); U_a uses one handle at the centre of mass with
  phi_a = 1 - phi_DBC (L300-302, reading Q14).
* The coarse matrices U^T H U are formed explicitly here (the definition), and factorised by
  dense Cholesky (reading R4: exact coarse solves).
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import fem


def lbs_matrix(X, vptr, handle, phi, origins, n_handles):
    """Sparse (3n x 12 n_handles) matrix of Eq. 7 from per-vertex (handle, phi) lists."""
    n = X.shape[0]
    cnt = np.diff(vptr)
    v = np.repeat(np.arange(n), cnt)
    hnd = np.asarray(handle, dtype=np.int64)
    mono = np.concatenate([np.ones((len(v), 1)), X[v] - origins[hnd]], axis=1)   # (nnz,4)
    w = np.asarray(phi)[:, None] * mono
    rows, cols, vals = [], [], []
    for c in range(3):
        for k in range(4):
            rows.append(3 * v + c)
            cols.append(12 * hnd + 4 * c + k)
            vals.append(w[:, k])
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(3 * n, 12 * n_handles))


def sms_matrix(X, basis):
    """U_s (L356-362)."""
    return lbs_matrix(X, basis.vptr, basis.handle, basis.phi, basis.origins, basis.m)


def affine_matrix(X, basis):
    """U_a: one affine handle at the centre of mass, weight phi_a = 1 - phi_DBC (L300-302)."""
    n = X.shape[0]
    vptr = np.arange(n + 1, dtype=np.int64)
    return lbs_matrix(X, vptr, np.zeros(n, dtype=np.int64), basis.phi_affine,
                      np.asarray(basis.affine_origin, dtype=np.float64)[None, :], 1)


def galerkin(U, H, n_blocks=32):
    """Dense U^T H U (the 'subspace sandwich matrix', L456), formed column block by column
    block, S[:, J] = U^T (H U[:, J]), on a thread pool (the blocks are independent)."""
    H = H.tocsr()
    Ut = U.T.tocsr()
    Uc = U.tocsc()
    n = U.shape[1]
    cuts = np.linspace(0, n, min(n_blocks, n) + 1).astype(int)

    def block(k):
        return (Ut @ (H @ Uc[:, cuts[k]:cuts[k + 1]])).toarray()
    with ThreadPoolExecutor(fem.n_threads()) as ex:
        return np.ascontiguousarray(np.concatenate(list(ex.map(block, range(len(cuts) - 1))), axis=1))


def cholesky(S):
    """Lower Cholesky factor of the SPD coarse matrix (reading R4)."""
    return np.linalg.cholesky(S)


def cho_solve(L, b):
    y = sla.solve_triangular(L, b, lower=True)
    return sla.solve_triangular(L.T, y, lower=False)
