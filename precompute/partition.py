"""Stiffness- and geometry-aware partitioner (BOUNDARY precompute; NEXT-3 of SURVEY §8(f);
PAPER.md §3.6.1-3.6.3 L404-419 and L635; reading N3 of DESIGN.md).

Like the rest of the basis build this is an INPUT of the hot path (the tet -> cluster map from
which precompute/basis.py builds the handles); no Hessian, projection or solve of the Newton
iteration lives here.

* Distances (§3.6.1, "heat diffusion-based geodesics [Crane et al. 2013] ... stiffness-weighted
  Laplacian, corresponding to diffusion with a spatially varying diffusion coefficient"): for a
  source vertex s
    1. heat flow   (M + t L_k) u = e_s,  t = (mean edge length)^2, L_k = sum_e k_e V_e G_e G_e^T;
    2. unit field  X_e = -grad u_e / |grad u_e| / sqrt(k_e)   (|grad phi| = 1/sqrt(k): the metric in
       which heat travels "faster" in stiff regions, so distances grow slower there);
    3. Poisson     L phi = sum_e V_e G_e X_e (least-squares fit of grad phi to X; L unweighted,
       regularised by 1e-10 M for the constant null space), phi shifted so phi(s) = 0, clipped >= 0.
  k_e = E_e / median(E) with the jump penalty (§3.6.2): an element with a vertex that touches
  elements of different materials gets k_e = jump * (softest k), jump = 0.25 ("0.1 to 0.5",
  0.25 "for others", L415).
* Clustering (§3.6.1): kmeans++ seeding with the same distance (first centre ~ vertex volume,
  next ~ volume * D^2, draws from the seeded SplitMix64 stream shared with basis.py), Lloyd
  relaxation: a tet joins the centre with the smallest mean distance of its four vertices (ties ->
  lowest centre), each centre moves to the cluster vertex nearest to the cluster's volume-weighted
  barycentre (reading N3: the geodesic centroid is not computable without all-pairs distances).
* Pruning (§3.6.3): every 10 Lloyd iterations the clusters with
  median volume >= 1.75 x their volume are candidates; the n = 5 smallest candidates are deleted
  (their tets join the nearest remaining centre at the next assignment).  Stop at an assignment
  fixed point without pruning, or after max_iter iterations.

Cost: 2 sparse solves per centre per Lloyd iteration with two factorisations (SuperLU) of the
vertex Laplacian -- practical for C1 / C2 / the test scenes on the CPU; C3-C5 keep the Euclidean
partitioner (a GPU build is not part of this round).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

JUMP = 0.25
PRUNE_EVERY = 10
PRUNE_RATIO = 1.75
PRUNE_N = 5


def shape_gradients(X, tets):
    """Per-tet gradients of the 4 barycentric coordinates (nt, 4, 3) and volumes (nt,)."""
    D = X[tets[:, 1:]] - X[tets[:, :1]]
    vol = np.linalg.det(D) / 6.0
    g123 = np.transpose(np.linalg.inv(D), (0, 2, 1))
    G = np.concatenate([-g123.sum(axis=1, keepdims=True), g123], axis=1)
    return G, vol


def element_stiffness_weights(tets, E, jump=JUMP):
    """k_e = E_e / median(E); elements with a vertex touching two materials get jump * min(k)
    (jump None: no penalty)."""
    E = np.asarray(E, dtype=np.float64)
    k = E / np.median(E)
    n_v = int(tets.max()) + 1
    t4 = tets.ravel()
    e4 = np.repeat(E, 4)
    vmin = np.full(n_v, np.inf)
    vmax = np.full(n_v, -np.inf)
    np.minimum.at(vmin, t4, e4)
    np.maximum.at(vmax, t4, e4)
    interface_v = vmax > vmin
    interface_e = interface_v[tets].any(axis=1)
    out = k.copy()
    if jump is not None:
        out[interface_e] = jump * k.min()
    return out, interface_e


def laplacian(G, vol, w, tets, n_v):
    Kl = np.einsum("eik,ejk->eij", G, G) * (vol * w)[:, None, None]
    rows = np.repeat(tets, 4, axis=1).ravel()
    cols = np.tile(tets, (1, 4)).ravel()
    return sp.csr_matrix((Kl.ravel(), (rows, cols)), shape=(n_v, n_v))


class HeatGeodesics:
    """Stiffness-weighted heat-method distances on a tet mesh (the two operators factorised once)."""

    def __init__(self, X, tets, E, jump=JUMP):
        self.tets = np.asarray(tets, dtype=np.int64)
        self.n_v = len(X)
        self.G, self.vol = shape_gradients(X, self.tets)
        self.k, self.interface = element_stiffness_weights(self.tets, E, jump)
        e = X[self.tets[:, [0, 0, 0, 1, 1, 2]]] - X[self.tets[:, [1, 2, 3, 2, 3, 3]]]
        self.t = float(np.mean(np.linalg.norm(e, axis=2))) ** 2
        self.M = np.bincount(self.tets.ravel(), weights=np.repeat(self.vol / 4.0, 4), minlength=self.n_v)
        Lk = laplacian(self.G, self.vol, self.k, self.tets, self.n_v)
        L = laplacian(self.G, self.vol, np.ones(len(self.tets)), self.tets, self.n_v)
        self.heat = spla.splu((sp.diags(self.M) + self.t * Lk).tocsc())
        self.poisson = spla.splu((L + 1e-10 * sp.diags(self.M)).tocsc())

    def distances(self, sources):
        """(len(sources), n_v) distances from each source vertex."""
        sources = np.asarray(sources, dtype=np.int64)
        rhs = np.zeros((self.n_v, len(sources)))
        rhs[sources, np.arange(len(sources))] = 1.0
        u = self.heat.solve(rhs)                                  # (n_v, ns)
        gu = np.einsum("eik,eis->esk", self.G, u[self.tets])       # (nt, ns, 3) grad u per tet
        nrm = np.linalg.norm(gu, axis=2, keepdims=True)
        Xf = np.where(nrm > 0, -gu / np.where(nrm > 0, nrm, 1.0), 0.0) / np.sqrt(self.k)[:, None, None]
        div = np.einsum("eik,esk->eis", self.G, Xf) * self.vol[:, None, None]   # (nt, 4, ns)
        b = np.zeros((self.n_v, len(sources)))
        for c in range(4):
            np.add.at(b, self.tets[:, c], div[:, c, :])
        phi = self.poisson.solve(b)
        phi = phi - phi[sources, np.arange(len(sources))][None, :]
        return np.maximum(phi, 0.0).T


def prune_candidates(cluster_vol, ratio=PRUNE_RATIO, n=PRUNE_N):
    """Clusters to delete (§3.6.3): among those with median(vol) >= ratio * vol, the n smallest
    (ties -> lower id).  Empty clusters (vol 0) are always candidates."""
    med = np.median(cluster_vol)
    cand = np.flatnonzero(med >= ratio * cluster_vol)
    o = np.lexsort((cand, cluster_vol[cand]))
    return np.sort(cand[o][:n])


def geodesic_kmeans(scene, m, seed, max_iter=30, jump=JUMP, prune_every=PRUNE_EVERY, ratio=PRUNE_RATIO,
                    n_prune=PRUNE_N, geo=None):
    """Tet -> cluster ids (0..m'-1, m' <= m after pruning) and the centre vertices."""
    from .basis import splitmix64_uniform, weighted_pick
    X, tets = scene.X, np.asarray(scene.tets, dtype=np.int64)
    geo = geo or HeatGeodesics(X, tets, scene.E, jump)
    w = geo.M
    # kmeans++ with the geodesic distance
    centres = [weighted_pick(w, splitmix64_uniform(seed, 0))]
    D = geo.distances(centres)[0]
    for k in range(1, m):
        centres.append(weighted_pick(w * D * D, splitmix64_uniform(seed, k)))
        D = np.minimum(D, geo.distances(centres[-1:])[0])
    centres = np.array(centres, dtype=np.int64)
    bary = X[tets].mean(axis=1)
    assign = None
    for it in range(1, max_iter + 1):
        Dv = geo.distances(centres)                       # (k, n_v)
        Dt = Dv[:, tets].mean(axis=2)                     # (k, nt): mean over the four vertices
        a = np.argmin(Dt, axis=0)                         # ties -> lowest centre
        pruned = False
        cvol = np.bincount(a, weights=geo.vol, minlength=len(centres))
        if prune_every and it % prune_every == 0:
            dead = prune_candidates(cvol, ratio, n_prune)
            if len(dead):
                keep = np.setdiff1d(np.arange(len(centres)), dead)
                centres = centres[keep]
                a = np.argmin(Dt[keep], axis=0)
                cvol = np.bincount(a, weights=geo.vol, minlength=len(centres))
                pruned = True
        if assign is not None and not pruned and len(a) == len(assign) and np.array_equal(a, assign):
            break
        assign = a
        # centre update: cluster vertex nearest to the volume-weighted barycentre
        new = centres.copy()
        for i in range(len(centres)):
            sel = assign == i
            if not np.any(sel):
                continue
            bc = (geo.vol[sel, None] * bary[sel]).sum(0) / geo.vol[sel].sum()
            pv = np.unique(tets[sel])
            new[i] = pv[np.argmin(np.sum((X[pv] - bc) ** 2, axis=1))]
        centres = new
    used = np.unique(assign)
    remap = -np.ones(len(centres), dtype=np.int64)
    remap[used] = np.arange(len(used))
    return remap[assign], centres[used]
