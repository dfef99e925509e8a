"""Modal moment-fitting cubature for the subspace Hessian (BOUNDARY precompute; NEXT-2;
PAPER.md §3.8, Alg. 3; readings C3 and C4 in DESIGN.md).

Like the basis, the cubature is an INPUT of the hot path: the element subset and weights are fed
identically to the CUDA path (ms_cubature_upload) and to the oracle.  No Hessian, projection or
solve lives here.

Per mesh partition (the k-means clusters of the basis, §3.8.2 "we use our mesh partitioning
structure ... to build integration complexes"):
1. the basis functions intersecting the partition -- the scalar SMS weights u_j = phi_j of every
   handle j whose support meets a vertex of the partition (reading C3: the material-aware part of
   the basis; its monomial factors [1, X - c_j] of Eq. 7 are low-degree polynomials, and fitting
   their products too (4x the functions, 16x the constraints) selected 75-97 % of the elements of
   C1 / C2 / the drop scene, against the paper's 1-41 %) -- evaluated per element by averaging the
   element's four vertex values (§3.8.2, "averaging the basis values at each element's vertices");
2. moment constraints for all products of degree <= p = 2 (§3.8.1): 1, u_a, u_a u_b (a <= b),
   weighted by the element's Young's modulus (reading C3: the integrand is the elastic energy
   density, proportional to E_e; unweighted moments left a 54 % error in B^T H B on C2, whose
   partitions mix 1e5 and 1e9 Pa cubes): A[alpha, k] = E_k prod u(e_k), targets
   b = sum_e vol_e E_e prod(u(e)) over all partition elements (§3.8.2), so that
   sum_k w_k E_k prod u(e_k) = sum_e vol_e E_e prod u(e);
3. Alg. 3: NNLS (scipy.optimize.nnls, Lawson-Hanson) on n_init seeded random elements, then while
   ||A w - b|| / ||b|| > tol (1e-9, §3.8.2) add n_add elements drawn without replacement with
   probability ~ rho_k = (A_k . r)^2, r = A w - b; all elements sampled = exact (w = vol solves it).
The rows of A are scaled by 1 / max|row| (both sides), which leaves the NNLS solution set of the
exact system unchanged and keeps the tolerance test meaningful across constraint scales.
"""
from __future__ import annotations

import dataclasses
import os

import numpy as np
from scipy.optimize import nnls

CUBATURE_VERSION = "v2"


@dataclasses.dataclass
class Cubature:
    elements: np.ndarray     # (n_c,) int32 tet ids, ascending
    weights: np.ndarray      # (n_c,) float64 > 0 (replaces the element volume in the elastic integral)
    part_counts: np.ndarray  # (m,) cubature points per partition
    part_residual: np.ndarray  # (m,) final ||A w - b|| / ||b|| per partition
    p: int = 2
    tol: float = 1e-9

    def save(self, path):
        np.savez_compressed(path, **{k: getattr(self, k) for k in self.__dataclass_fields__})

    @staticmethod
    def load(path):
        z = np.load(path)
        return Cubature(elements=z["elements"], weights=z["weights"], part_counts=z["part_counts"],
                        part_residual=z["part_residual"], p=int(z["p"]), tol=float(z["tol"]))


def element_basis_values(X, tets, basis, elems):
    """u(e) for the SMS weights meeting `elems`: (n_e, n_f) per-element averages of the four vertex
    values of phi_j; returns (values, handle ids)."""
    vptr, handle, phi = basis.vptr, basis.handle, basis.phi
    verts = np.unique(tets[elems])
    hs = sorted({int(handle[k]) for v in verts for k in range(vptr[v], vptr[v + 1])})
    col = {h: i for i, h in enumerate(hs)}
    loc = {int(v): i for i, v in enumerate(verts)}
    vals = np.zeros((len(verts), len(hs)))
    for v in verts:
        for k in range(vptr[v], vptr[v + 1]):
            vals[loc[int(v)], col[int(handle[k])]] = phi[k]
    li = np.vectorize(loc.get)(tets[elems])
    ue = (((vals[li[:, 0]] + vals[li[:, 1]]) + vals[li[:, 2]]) + vals[li[:, 3]]) / 4.0
    return ue, hs


def moment_matrix(ue, p=2):
    """Rows: prod_{i in alpha} u_i(e) for |alpha| <= p (alpha a multiset), columns: elements."""
    n_e, n_f = ue.shape
    rows = [np.ones(n_e)]
    if p >= 1:
        rows += [ue[:, a] for a in range(n_f)]
    if p >= 2:
        rows += [ue[:, a] * ue[:, b] for a in range(n_f) for b in range(a, n_f)]
    if p > 2:
        raise NotImplementedError("p <= 2")
    return np.array(rows)


def fit_partition(A, b, rng, tol=1e-9, n_init=None, n_add=None):
    """Alg. 3 on one partition; returns (column ids, weights > 0, relative residual)."""
    m, n = A.shape
    n_init = max(m, 10) if n_init is None else n_init
    n_add = max(m // 2, 5) if n_add is None else n_add
    scale = 1.0 / np.maximum(np.abs(A).max(axis=1), 1e-300)
    As, bs = A * scale[:, None], b * scale
    nb = np.linalg.norm(bs)
    chosen = np.zeros(n, dtype=bool)
    chosen[rng.choice(n, size=min(n_init, n), replace=False)] = True
    while True:
        cols = np.flatnonzero(chosen)
        w, _ = nnls(As[:, cols], bs, maxiter=50 * len(cols))
        r = As[:, cols] @ w - bs
        rel = np.linalg.norm(r) / nb
        if rel <= tol or chosen.all():
            keep = w > 0
            return cols[keep], w[keep], rel
        cand = np.flatnonzero(~chosen)
        rho = (As[:, cand].T @ r) ** 2
        prob = rho / rho.sum() if rho.sum() > 0 else np.full(len(cand), 1.0 / len(cand))
        k = min(n_add, len(cand), int(np.count_nonzero(prob)))
        chosen[rng.choice(cand, size=k, replace=False, p=prob)] = True


def _fit_one(args):
    i, X, tets, basis, elems, vol, E, p, tol, seed = args
    ue, _ = element_basis_values(X, tets, basis, elems)
    A = moment_matrix(ue, p) * E[elems][None, :]
    b = A @ vol[elems]
    cols, w, rel = fit_partition(A, b, np.random.default_rng([seed, i]), tol)
    return i, elems[cols], w, rel


def build_cubature(scene, basis, p=2, tol=1e-9, seed=None, workers=None):
    from .basis import tet_volumes
    X, tets = scene.X, np.asarray(scene.tets, dtype=np.int64)
    vol = tet_volumes(X, tets)
    seed = scene.config if seed is None else seed
    parts = [np.flatnonzero(basis.cluster == i) for i in range(basis.m)]
    E = np.asarray(scene.E, dtype=np.float64)
    jobs = [(i, X, tets, basis, parts[i], vol, E, p, tol, seed) for i in range(basis.m)]
    workers = min(os.cpu_count() or 1, 64) if workers is None else workers
    if workers > 1 and len(jobs) > 4:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(workers) as pool:
            res = pool.map(_fit_one, jobs, chunksize=1)
    else:
        res = [_fit_one(j) for j in jobs]
    res.sort(key=lambda r: r[0])
    elements = np.concatenate([r[1] for r in res])
    weights = np.concatenate([r[2] for r in res])
    o = np.argsort(elements, kind="stable")
    return Cubature(elements=elements[o].astype(np.int32), weights=weights[o],
                    part_counts=np.array([len(r[1]) for r in res]), part_residual=np.array([r[3] for r in res]),
                    p=p, tol=tol)


def cached_cubature(scene, basis, cache_dir=None, **kw) -> Cubature:
    from .basis import BASIS_VERSION
    cache_dir = cache_dir or os.environ.get("MSIM_CACHE", os.path.join(os.path.dirname(__file__), "..", ".cache"))
    os.makedirs(cache_dir, exist_ok=True)
    path = os.path.join(cache_dir, f"{scene.name}_{scene.n_tets}_{basis.m}_{BASIS_VERSION}_cub{CUBATURE_VERSION}.npz")
    if os.path.exists(path):
        return Cubature.load(path)
    c = build_cubature(scene, basis, **kw)
    c.save(path)
    return c
