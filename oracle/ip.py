"""Oracle: incremental potential E, gradient g and Hessian H (Eq. 2).

Test infrastructure only (see oracle/__init__.py).

E(x) = 1/2 sum_v m_v |x_v - xhat_v|^2 + h^2 [ sum_e V_e Psi(F_e) + kappa sum_v b(d_v) ]

* implicit Euler, alpha = 1 (L182-184); gravity folded into the predictor
  xhat = x^t + h v^t + h^2 g_grav (reading R8 / Q10);
* BDF2 (L185-189; NEXT-4): alpha = 4/9, xhat = (4x^t - x^{t-1})/3 + (2h/9)(4v^t - v^{t-1}) + alpha h^2 g
  (gravity is an external potential inside the alpha-scaled term, so it folds in with alpha h^2);
* lumped mass m_v = sum_{e ni v} rho_e V_e / 4 (reading Q9);
* IPC log barrier against the ground plane, b(d) = -(d - dhat)^2 ln(d/dhat) for
  d < dhat; E = +inf if any d_v <= 0;
* Dirichlet (DBC) vertices: g = 0, H rows/cols -> identity (reading Q13); their
  constant inertia/barrier terms are left out of E (they never move).
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.sparse as sp

from . import fem


@dataclasses.dataclass
class Model:
    X: np.ndarray
    tets: np.ndarray
    Bm: np.ndarray
    V: np.ndarray
    mu: np.ndarray
    lam: np.ndarray
    mass: np.ndarray          # (n_v,)
    free: np.ndarray          # (n_v,) bool, False at DBC vertices
    h: float
    gravity: np.ndarray
    ground: dict | None
    alpha: float = 1.0        # IP scaling of Eq. 2: 1 (implicit Euler), 4/9 (BDF2)

    @property
    def n(self):
        return self.X.shape[0]


def make_model(scene):
    X = np.asarray(scene.X, dtype=np.float64)
    tets = np.asarray(scene.tets, dtype=np.int64)
    _, Bm, V = fem.rest_data(X, tets)
    mu, lam = fem.lame(scene.E, scene.nu)
    mass = np.bincount(tets.ravel(), weights=np.repeat(scene.rho * V / 4.0, 4), minlength=len(X))
    free = np.ones(len(X), dtype=bool)
    free[np.asarray(scene.dbc, dtype=np.int64)] = False
    return Model(X, tets, Bm, V, mu, lam, mass, free, float(scene.h),
                 np.asarray(scene.gravity, dtype=np.float64), scene.ground)


def ah2(model):
    """alpha h^2, the weight of the potential energies in Eq. 2."""
    return model.alpha * model.h ** 2


def predictor(model, x_t, v_t):
    """xhat = x^t + h v^t + h^2 g_grav (P:183 with gravity folded in, R8)."""
    return x_t + model.h * v_t + model.h ** 2 * model.gravity[None, :]


def predictor_bdf2(model, x_t, v_t, x_tm1, v_tm1):
    """BDF2 predictor: xhat = (4x^t - x^{t-1})/3 + (2h/9)(4v^t - v^{t-1}), plus the folded
    gravity alpha h^2 g with alpha = 4/9."""
    h = model.h
    return (4.0 * x_t - x_tm1) / 3.0 + (2.0 * h / 9.0) * (4.0 * v_t - v_tm1) + (4.0 / 9.0) * h ** 2 * model.gravity[None, :]


# ----------------------------------------------------------------------------- barrier

def barrier(d, dhat):
    """b(d) = -(d - dhat)^2 ln(d / dhat) on (0, dhat), 0 for d >= dhat."""
    d = np.asarray(d, dtype=np.float64)
    act = d < dhat
    dd = np.where(act, d, dhat)
    return np.where(act, -(dd - dhat) ** 2 * np.log(dd / dhat), 0.0)


def barrier_d1(d, dhat):
    """b'(d) = -2 (d - dhat) ln(d/dhat) - (d - dhat)^2 / d."""
    d = np.asarray(d, dtype=np.float64)
    act = d < dhat
    dd = np.where(act, d, dhat)
    return np.where(act, -2.0 * (dd - dhat) * np.log(dd / dhat) - (dd - dhat) ** 2 / dd, 0.0)


def barrier_d2(d, dhat):
    """b''(d) = -2 ln(d/dhat) - 4 (d - dhat)/d + (d - dhat)^2 / d^2."""
    d = np.asarray(d, dtype=np.float64)
    act = d < dhat
    dd = np.where(act, d, dhat)
    return np.where(act, -2.0 * np.log(dd / dhat) - 4.0 * (dd - dhat) / dd + (dd - dhat) ** 2 / dd ** 2, 0.0)


def ground_distance(model, x):
    n = np.asarray(model.ground["normal"], dtype=np.float64)
    return x @ n - model.ground["offset"], n


# ----------------------------------------------------------------------------- E, g

def energy_terms(model, x, xhat):
    """(inertia, alpha h^2 elastic, alpha h^2 barrier) with +inf on inversion / penetration."""
    h2 = ah2(model)
    f = model.free
    inertia = 0.5 * np.sum(model.mass[f] * np.sum((x[f] - xhat[f]) ** 2, axis=1))
    elastic = h2 * np.sum(fem.element_energy(x, model.tets, model.Bm, model.V, model.mu, model.lam))
    bar = 0.0
    if model.ground is not None:
        d, _ = ground_distance(model, x)
        d = d[f]
        if np.any(d <= 0.0):
            return inertia, elastic, np.inf
        bar = h2 * model.ground["kappa"] * np.sum(barrier(d, model.ground["dhat"]))
    return inertia, elastic, bar


def energy(model, x, xhat):
    """E(x) of Eq. 2 (IE, alpha = 1)."""
    return float(sum(energy_terms(model, x, xhat)))


def energy_difference(model, x, d, alpha, xhat):
    """E(x + alpha d) - E(x), summed term by term (reading Q12: the strict-decrease test of the
    backtracking line search is evaluated on per-element / per-vertex differences so that the
    large constant parts of E cancel exactly instead of at the scale of |E|)."""
    h2 = ah2(model)
    f = model.free
    y = x + alpha * d
    r = x[f] - xhat[f]
    dv = alpha * d[f]
    dK = 0.5 * np.sum(model.mass[f] * (2.0 * np.sum(r * dv, axis=1) + np.sum(dv * dv, axis=1)))
    e1 = fem.element_energy(y, model.tets, model.Bm, model.V, model.mu, model.lam)
    if not np.all(np.isfinite(e1)):
        return np.inf
    e0 = fem.element_energy(x, model.tets, model.Bm, model.V, model.mu, model.lam)
    dPsi = h2 * np.sum(e1 - e0)
    dB = 0.0
    if model.ground is not None:
        d0, _ = ground_distance(model, x)
        d1, _ = ground_distance(model, y)
        d0, d1 = d0[f], d1[f]
        if np.any(d1 <= 0.0):
            return np.inf
        dh = model.ground["dhat"]
        dB = h2 * model.ground["kappa"] * np.sum(barrier(d1, dh) - barrier(d0, dh))
    return float(dK + dPsi + dB)


def gradient(model, x, xhat):
    """g = M (x - xhat) + alpha h^2 [sum_e G_e^T vec P V_e + kappa b'(d) n]; g = 0 at DBC vertices."""
    h2 = ah2(model)
    ge = fem.element_gradient(x, model.tets, model.Bm, model.V, model.mu, model.lam)
    g = np.zeros_like(x)
    for a in range(4):
        for c in range(3):
            g[:, c] += np.bincount(model.tets[:, a], weights=ge[:, 3 * a + c], minlength=model.n)
    g *= h2
    g += model.mass[:, None] * (x - xhat)
    if model.ground is not None:
        d, nrm = ground_distance(model, x)
        g += h2 * model.ground["kappa"] * barrier_d1(d, model.ground["dhat"])[:, None] * nrm[None, :]
    g[~model.free] = 0.0
    return g


# ----------------------------------------------------------------------------- H

def block_pattern(tets, n):
    """3x3-block sparsity: vertex adjacency through tets, plus the diagonal (CSR, sorted)."""
    r = np.repeat(tets, 4, axis=1).ravel()
    c = np.tile(tets, (1, 4)).ravel()
    A = sp.coo_matrix((np.ones(len(r)), (r, c)), shape=(n, n)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    return A.indptr.astype(np.int64), A.indices.astype(np.int64)


def elastic_blocks(model, x, elem_scale=None, chunk=32768):
    """alpha h^2 sum_e s_e P+(H_e) as 3x3 blocks on the BSR pattern (block_pattern): the (a,b) 3x3
    block of P+(H_e) goes to slot (e[a], e[b]).  s_e = 1 (full integration) or, for the cubature
    Hessian of the subspace solves (§3.8, NEXT-2), s_e = w_e / V_e on the cubature elements and 0
    elsewhere (the weight replaces the element volume)."""
    n = model.n
    h2 = ah2(model)
    indptr, indices = block_pattern(model.tets, n)
    nnzb = len(indices)
    rows = np.repeat(np.arange(n), np.diff(indptr))
    key = rows * n + indices                   # sorted
    blocks = np.zeros((nnzb, 9))
    sel = np.arange(len(model.tets)) if elem_scale is None else np.flatnonzero(elem_scale != 0.0)

    def work(e):
        t = model.tets[sel[e]]
        ids = sel[e]
        He = fem.element_hessian_psd(x, t, model.Bm[ids], model.V[ids], model.mu[ids], model.lam[ids], chunk=len(t))
        if elem_scale is not None:
            He = He * elem_scale[ids][:, None, None]
        slot = np.searchsorted(key, (t[:, :, None] * n + t[:, None, :]).ravel())      # (c*16,)
        sub = He.reshape(-1, 4, 3, 4, 3).transpose(0, 1, 3, 2, 4).reshape(-1, 9)  # (c*16, 9)
        return slot, sub

    for slot, sub in fem.map_chunks(work, len(sel), chunk):     # summed in chunk order
        lo, hi = int(slot.min()), int(slot.max()) + 1
        for q in range(9):
            blocks[lo:hi, q] += np.bincount(slot - lo, weights=sub[:, q], minlength=hi - lo)
    blocks = blocks.reshape(nnzb, 3, 3)
    blocks *= h2
    return blocks


def hessian(model, x, xhat, chunk=32768, elem_scale=None, elastic=None):
    """H = M + alpha h^2 (sum_e s_e P+(H_e) + kappa b''(d) n n^T), DBC rows/cols -> identity.

    Returned as scipy.sparse.bsr_matrix with 3x3 blocks: H_(i,j) = sum over tets e and
    local corners (a,b) with e[a]=i, e[b]=j of the (a,b) 3x3 block of P+(H_e).  elem_scale: see
    elastic_blocks; elastic: precomputed elastic blocks (the lagged Hessian of the refinement,
    §3.7.2: elastic part frozen, inertia and barrier always fresh)."""
    n = model.n
    h2 = ah2(model)
    indptr, indices = block_pattern(model.tets, n)
    rows = np.repeat(np.arange(n), np.diff(indptr))
    key = rows * n + indices
    blocks = (elastic_blocks(model, x, elem_scale, chunk) if elastic is None else elastic).copy()
    diag = np.searchsorted(key, np.arange(n) * n + np.arange(n))
    blocks[diag] += model.mass[:, None, None] * np.eye(3)[None]
    if model.ground is not None:
        d, nrm = ground_distance(model, x)
        kb = h2 * model.ground["kappa"] * barrier_d2(d, model.ground["dhat"])
        blocks[diag] += kb[:, None, None] * np.outer(nrm, nrm)[None]
    # DBC: identity rows/cols
    fixed = ~model.free
    kill = fixed[rows] | fixed[indices]
    blocks[kill] = 0.0
    blocks[diag[fixed]] = np.eye(3)
    return sp.bsr_matrix((blocks, indices, indptr), shape=(3 * n, 3 * n))
