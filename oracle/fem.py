"""Oracle: per-tetrahedron stable Neo-Hookean energy, gradient, Hessian, PSD projection.

Test infrastructure only (see oracle/__init__.py).

Passages followed:
* PAPER.md §3.1 L169 (piecewise-linear tets), L629 ("non-inverting Neo-hookean");
  reading R1 (SURVEY §0.1 / DESIGN.md): Psi = mu/2 (I_C - 3) - mu (J - 1) + lam/2 (J - 1)^2,
  Lame parameters from (E, nu), +inf for J <= 0.
* Reading R2: PSD projection = eigenvalue clamp of the 12x12 element Hessian.
* SURVEY §8(c) steps 1-4 for the kinematics and derivative formulas.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# D_ref maps vertex positions to edge vectors: Ds = X_e @ D_ref, X_e = [x0 x1 x2 x3] (3x4)
D_REF = np.array([[-1.0, -1.0, -1.0],
                  [1.0, 0.0, 0.0],
                  [0.0, 1.0, 0.0],
                  [0.0, 0.0, 1.0]])


def lame(E, nu):
    """mu = E / (2(1+nu)), lam = E nu / ((1+nu)(1-2nu))."""
    E = np.asarray(E, dtype=np.float64)
    nu = np.asarray(nu, dtype=np.float64)
    return E / (2.0 * (1.0 + nu)), E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))


def rest_data(X, tets):
    """Dm = [X1-X0 | X2-X0 | X3-X0] (columns), V = det(Dm)/6, Bm = Dm^-1."""
    Xe = X[tets]                                    # (nt,4,3)
    Dm = np.transpose(Xe[:, 1:] - Xe[:, :1], (0, 2, 1))   # columns are edges
    V = np.linalg.det(Dm) / 6.0
    Bm = np.linalg.inv(Dm)
    return Dm, Bm, V


def deformation_gradient(x, tets, Bm):
    """F = Ds Bm with Ds = [x1-x0 | x2-x0 | x3-x0]."""
    xe = x[tets]
    Ds = np.transpose(xe[:, 1:] - xe[:, :1], (0, 2, 1))
    return Ds @ Bm


def cofactor(F):
    """cof F = [f1 x f2 | f2 x f0 | f0 x f1] (columns f_k of F); cof F = det(F) F^-T."""
    f0, f1, f2 = F[..., :, 0], F[..., :, 1], F[..., :, 2]
    return np.stack([np.cross(f1, f2), np.cross(f2, f0), np.cross(f0, f1)], axis=-1)


def psi(F, mu, lam):
    """Stable Neo-Hookean energy density (R1); +inf where J <= 0."""
    J = np.linalg.det(F)
    Ic = np.sum(F * F, axis=(-2, -1))
    val = 0.5 * mu * (Ic - 3.0) - mu * (J - 1.0) + 0.5 * lam * (J - 1.0) ** 2
    return np.where(J > 0.0, val, np.inf)


def first_piola(F, mu, lam):
    """P = dPsi/dF = mu F + (lam (J-1) - mu) cof F."""
    J = np.linalg.det(F)
    return mu[..., None, None] * F + (lam * (J - 1.0) - mu)[..., None, None] * cofactor(F)


def vec(A):
    """Column-major vectorisation of (...,3,3) -> (...,9)."""
    return np.swapaxes(A, -1, -2).reshape(A.shape[:-2] + (9,))


def skew(a):
    """[a]x such that [a]x b = a x b."""
    z = np.zeros(a.shape[:-1])
    return np.stack([np.stack([z, -a[..., 2], a[..., 1]], -1),
                     np.stack([a[..., 2], z, -a[..., 0]], -1),
                     np.stack([-a[..., 1], a[..., 0], z], -1)], -2)


def hessian_J(F):
    """d^2 J / dF^2 in column-major vec order (9x9 blocks (a,b) = d^2J/df_a df_b)."""
    f = [F[..., :, k] for k in range(3)]
    n = F.shape[:-2]
    H = np.zeros(n + (9, 9))
    # J = f0 . (f1 x f2); d2J/df0 df1 = -[f2]x, d2J/df0 df2 = [f1]x, d2J/df1 df2 = -[f0]x
    blocks = {(0, 1): -skew(f[2]), (0, 2): skew(f[1]), (1, 2): -skew(f[0])}
    for (a, b), M in blocks.items():
        H[..., 3 * a:3 * a + 3, 3 * b:3 * b + 3] = M
        H[..., 3 * b:3 * b + 3, 3 * a:3 * a + 3] = np.swapaxes(M, -1, -2)
    return H


def d2psi_dF2(F, mu, lam):
    """d^2Psi/dF^2 = mu I9 + lam vec(cof F) vec(cof F)^T + (lam (J-1) - mu) H_J."""
    J = np.linalg.det(F)
    g = vec(cofactor(F))
    A = mu[..., None, None] * np.eye(9) + lam[..., None, None] * g[..., :, None] * g[..., None, :]
    return A + (lam * (J - 1.0) - mu)[..., None, None] * hessian_J(F)


def shape_gradient_matrix(Bm):
    """G_e (9x12) with vec(F) = G_e vec(X_e): G_e = (D_ref Bm)^T kron I3."""
    D = D_REF @ Bm                                   # (nt,4,3)
    Dt = np.swapaxes(D, -1, -2)                      # (nt,3,4)
    return np.einsum("...ab,ij->...aibj", Dt, np.eye(3)).reshape(Bm.shape[:-2] + (9, 12))


def element_energy(x, tets, Bm, V, mu, lam):
    """Per-tet V_e Psi(F_e)."""
    return V * psi(deformation_gradient(x, tets, Bm), mu, lam)


def element_gradient(x, tets, Bm, V, mu, lam):
    """Per-tet 12-vector g_e = V_e G_e^T vec P(F_e) (vertex-major, xyz inner)."""
    F = deformation_gradient(x, tets, Bm)
    G = shape_gradient_matrix(Bm)
    return V[:, None] * (np.swapaxes(G, -1, -2) @ vec(first_piola(F, mu, lam))[..., None])[..., 0]


def element_hessian(x, tets, Bm, V, mu, lam):
    """Per-tet 12x12 H_e = V_e G_e^T (d^2Psi/dF^2) G_e (unprojected)."""
    F = deformation_gradient(x, tets, Bm)
    G = shape_gradient_matrix(Bm)
    A = d2psi_dF2(F, mu, lam)
    return V[:, None, None] * (np.swapaxes(G, -1, -2) @ A @ G)


def psd_project(H):
    """P+(H) = Q max(Lambda, 0) Q^T with H = Q Lambda Q^T (R2; LAPACK syevd via numpy.eigh)."""
    H = 0.5 * (H + np.swapaxes(H, -1, -2))
    w, Q = np.linalg.eigh(H)
    return (Q * np.maximum(w, 0.0)[..., None, :]) @ np.swapaxes(Q, -1, -2)


def n_threads():
    """Host threads for the element loops (chunks are independent; results do not depend on it)."""
    return max(1, int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1)))


def map_chunks(fn, n, chunk):
    """Yields fn(slice) for each chunk of range(n) in chunk order, evaluated on a thread pool
    (numpy's batched linear algebra releases the GIL) with a bounded number in flight."""
    sl = [slice(s, min(s + chunk, n)) for s in range(0, n, chunk)]
    nt = n_threads()
    if nt == 1 or len(sl) <= 1:
        for e in sl:
            yield fn(e)
        return
    with ThreadPoolExecutor(nt) as ex:
        pending = [ex.submit(fn, e) for e in sl[:2 * nt]]
        nxt = len(pending)
        while pending:
            r = pending.pop(0).result()
            if nxt < len(sl):
                pending.append(ex.submit(fn, sl[nxt]))
                nxt += 1
            yield r


def element_hessian_psd(x, tets, Bm, V, mu, lam, chunk=32768):
    """P+(H_e) for every tet, evaluated in independent chunks to bound memory."""
    out = np.empty((len(tets), 12, 12))

    def work(e):
        out[e] = psd_project(element_hessian(x, tets[e], Bm[e], V[e], mu[e], lam[e]))
    for _ in map_chunks(work, len(tets), chunk):
        pass
    return out
