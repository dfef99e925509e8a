"""SMS / affine basis construction (BOUNDARY precompute; SURVEY.md §8(b) `ms_basis_build`).

The basis is an INPUT to the hot path: its output (handle origins, per-vertex
(handle, phi) lists, affine weight, N_cg) is fed identically to the CUDA path
(through `ms_basis_upload`) and to the oracle.  Neither the hot path's coarse
projection B^T H B nor any solve lives here.

Steps (§3.5, §3.6, §3.7.2; readings Q15-Q17):
1. Partition tets into m clusters: seeded kmeans++ + Lloyd on volume-weighted tet
   barycentres (Euclidean stand-in for the paper's heat geodesics, NEXT-3).
2. Enforce face-connectivity of each cluster.
3. Centroid vertex c_i = cluster vertex nearest to the cluster's barycentre (Q15).
4. Subdomain T_i = cluster i + clusters sharing a vertex with it (R9/Q16).
5. Solve K u = 0 on T_i, K = L_s M^-1 L_s (Q17), u(c_i)=1, u(c_j)=0 for neighbour
   centroids, u=0 on the internal boundary and at DBC vertices.
   Clip u_pos = max(u, 0).
6. DBC weight, POU normalisation, affine weight 1-phi_DBC.
7. Handles are relabelled in lexicographic (x, y, z) order of their centroids so
   that the coarse matrix is banded in handle order.
"""
from __future__ import annotations

import dataclasses
import os

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from scipy.spatial import cKDTree


BASIS_VERSION = "v2"   # v2: counter-based kmeans++ draws (splitmix64), exact nearest-centre ties


@dataclasses.dataclass
class Basis:
    m: int
    origins: np.ndarray      # (m,3) handle origins c_i (rest positions of centroid vertices)
    vptr: np.ndarray         # (n_v+1,) int64 CSR over vertices
    handle: np.ndarray       # (nnz,) int32 handle ids (sorted within each vertex)
    phi: np.ndarray          # (nnz,) float64 weights > 0
    phi_dbc: np.ndarray      # (n_v,) DBC weight
    phi_affine: np.ndarray   # (n_v,) affine weight 1 - phi_dbc
    affine_origin: np.ndarray  # (3,) centre of mass
    n_cg: int                # 20 or 40 (hop heuristic)
    hop_radius: float
    cluster: np.ndarray      # (n_t,) cluster id (relabelled)
    centroid_vertex: np.ndarray  # (m,) int
    n_holes: int = 0         # free vertices repaired by reading B1

    def save(self, path):
        np.savez_compressed(path, **{k: getattr(self, k) for k in self.__dataclass_fields__})

    @staticmethod
    def load(path):
        z = np.load(path)
        kw = {}
        for k in Basis.__dataclass_fields__:
            v = z[k]
            kw[k] = v.item() if v.ndim == 0 else v
        kw["m"] = int(kw["m"])
        kw["n_cg"] = int(kw["n_cg"])
        kw["n_holes"] = int(kw.get("n_holes", 0))
        return Basis(**kw)


# ----------------------------------------------------------------------------- geometry

def tet_volumes(X, tets):
    """V = det[X1-X0 | X2-X0 | X3-X0] / 6, the determinant written out as a.(b x c) in a fixed
    order (the native ms_basis_build evaluates the same expression)."""
    a = X[tets[:, 1]] - X[tets[:, 0]]
    b = X[tets[:, 2]] - X[tets[:, 0]]
    c = X[tets[:, 3]] - X[tets[:, 0]]
    det = (a[:, 0] * (b[:, 1] * c[:, 2] - b[:, 2] * c[:, 1])
           - a[:, 1] * (b[:, 0] * c[:, 2] - b[:, 2] * c[:, 0])
           + a[:, 2] * (b[:, 0] * c[:, 1] - b[:, 1] * c[:, 0]))
    return det / 6.0


def tet_barycentres(X, tets):
    """((X0 + X1) + X2) + X3) / 4."""
    return (((X[tets[:, 0]] + X[tets[:, 1]]) + X[tets[:, 2]]) + X[tets[:, 3]]) / 4.0


def face_adjacency(tets):
    """Pairs (e, f) of tets sharing a triangular face."""
    nt = len(tets)
    loc = np.array([[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]])
    faces = np.sort(tets[:, loc].reshape(-1, 3), axis=1).astype(np.int64)
    owner = np.repeat(np.arange(nt), 4)
    key = (faces[:, 0] * (1 << 21) + faces[:, 1]) * (1 << 21) + faces[:, 2]
    order = np.argsort(key, kind="stable")
    ks = key[order]
    dup = np.nonzero(ks[1:] == ks[:-1])[0]
    return owner[order[dup]], owner[order[dup + 1]]


# ----------------------------------------------------------------------------- k-means

def splitmix64_uniform(seed, k):
    """k-th uniform double in [0, 1) of the counter-based SplitMix64 stream of `seed`:
    z = seed + (k+1) 0x9E3779B97F4A7C15, two xor-shift-multiply rounds, top 53 bits.
    The native ms_basis_build draws the same numbers (random draws shared by counter)."""
    M = (1 << 64) - 1
    z = (int(seed) + (int(k) + 1) * 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    z ^= z >> 31
    return (z >> 11) * (1.0 / 9007199254740992.0)


def sq_dist(P, c):
    """(dx^2 + dy^2) + dz^2 per row (fixed order, no fused multiply-add)."""
    d = P - c
    return (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]


def weighted_pick(p, u):
    """Index i with cdf[i-1] <= u cdf[n-1] < cdf[i], cdf = sequential prefix sums of p."""
    cdf = np.cumsum(p)
    t = u * cdf[-1]
    return min(int(np.searchsorted(cdf, t, side="right")), len(p) - 1)


def kmeans_pp(P, w, m, seed):
    """kmeans++ seeding ('k-means++'): first centre drawn with probability ~ w, each
    next with probability ~ w d^2 (d = distance to the nearest chosen centre); draw k uses
    splitmix64_uniform(seed, k)."""
    first = weighted_pick(w, splitmix64_uniform(seed, 0))
    C = [P[first]]
    d2 = sq_dist(P, P[first])
    for k in range(1, m):
        idx = weighted_pick(w * d2, splitmix64_uniform(seed, k))
        C.append(P[idx])
        d2 = np.minimum(d2, sq_dist(P, P[idx]))
    return np.array(C)


def nearest_centre(P, C, k=4):
    """Index of the nearest centre per point by exact squared distance (sq_dist), ties -> lowest
    centre index; cKDTree only proposes the k candidates."""
    k = min(k, len(C))
    _, cand = cKDTree(C).query(P, k=k)
    cand = np.asarray(cand).reshape(len(P), k)
    d = np.stack([sq_dist(P, C[cand[:, j]]) for j in range(k)], axis=1)
    best = d.min(axis=1, keepdims=True)
    idx = np.where(d == best, cand, np.iinfo(np.int64).max).min(axis=1)
    return idx


def lloyd(P, w, C, max_iter=100):
    """Lloyd iterations: assign to the nearest centre, move centres to the w-weighted means;
    stop at an assignment fixed point or after max_iter."""
    assign = None
    for _ in range(max_iter):
        a = nearest_centre(P, C)
        if assign is not None and np.array_equal(a, assign):
            break
        assign = a
        m = len(C)
        W = np.bincount(assign, weights=w, minlength=m)
        newC = np.stack([np.bincount(assign, weights=w * P[:, d], minlength=m) for d in range(3)], 1)
        nz = W > 0
        C = C.copy()
        C[nz] = newC[nz] / W[nz, None]
    return assign


def enforce_connectivity(assign, tets, adj_pairs, m):
    """Keep the largest face-connected component of each cluster; move the rest to the
    adjacent cluster sharing the most faces (repeat until every cluster is connected)."""
    nt = len(tets)
    ea, eb = adj_pairs
    for _ in range(20):
        same = assign[ea] == assign[eb]
        G = sp.coo_matrix((np.ones(int(same.sum())), (ea[same], eb[same])), shape=(nt, nt))
        ncomp, comp = sp.csgraph.connected_components(G, directed=False)
        # largest component per cluster
        size = np.bincount(comp, minlength=ncomp)
        comp_cluster = np.zeros(ncomp, dtype=np.int64)
        comp_cluster[comp] = assign
        order = np.lexsort((-size, comp_cluster))   # by cluster, then size desc
        keep = np.zeros(ncomp, dtype=bool)
        seen = set()
        for ci in order:
            cl = comp_cluster[ci]
            if cl not in seen:
                keep[ci] = True
                seen.add(cl)
        bad = ~keep[comp]
        if not bad.any():
            return assign
        # reassign tets of non-kept components: neighbour cluster with most shared faces
        diff = ~same
        votes = {}
        for x, y in ((ea[diff], eb[diff]), (eb[diff], ea[diff])):
            sel = bad[x]
            for e, c in zip(x[sel], assign[y[sel]]):
                key = (comp[e], int(c))
                votes[key] = votes.get(key, 0) + 1
        target = {}
        for (ci, c), v in sorted(votes.items()):
            if ci not in target or v > target[ci][1]:
                target[ci] = (c, v)
        for e in np.nonzero(bad)[0]:
            if comp[e] in target:
                assign[e] = target[comp[e]][0]
    return assign


# ----------------------------------------------------------------------------- operators

def local_laplacians(X, tets, weight):
    """Per-tet 4x4 P1 FEM Laplacian V*w*G G^T (G = shape-function gradients)."""
    D = X[tets[:, 1:]] - X[tets[:, :1]]                  # (nt,3,3) rows = edges
    vol = np.linalg.det(D) / 6.0
    Dinv = np.linalg.inv(D)                               # (nt,3,3)
    # gradients of barycentric coordinates 1..3 are the columns of D^-1 (rows edge vectors)
    g123 = np.transpose(Dinv, (0, 2, 1))                   # (nt,3,3): g_k = Dinv[:,k]
    g0 = -g123.sum(axis=1, keepdims=True)
    G = np.concatenate([g0, g123], axis=1)                # (nt,4,3)
    Kl = np.einsum("eik,ejk->eij", G, G) * (vol * weight)[:, None, None]
    return Kl, vol


def assemble_subdomain(tets_sub, Kl_sub, vol_sub, verts):
    """L_s and lumped M (volume/4) of the sub-mesh, in local vertex numbering of `verts`."""
    n = len(verts)
    gmap = {}
    loc = np.searchsorted(verts, tets_sub)
    rows = np.repeat(loc, 4, axis=1).ravel()
    cols = np.tile(loc, (1, 4)).ravel()
    L = sp.csr_matrix((Kl_sub.ravel(), (rows, cols)), shape=(n, n))
    Mdiag = np.bincount(loc.ravel(), weights=np.repeat(vol_sub / 4.0, 4), minlength=n)
    return L, Mdiag


def constrained_system(L, Mdiag, one_idx, zero_idx):
    """K = L M^-1 L with u = 1 on one_idx and u = 0 on zero_idx: returns (u with the constrained
    values, free indices, K_ff, rhs = -K_fc u_c) of the system K_ff u_f = rhs."""
    n = L.shape[0]
    K = (L @ sp.diags(1.0 / Mdiag) @ L).tocsr()
    u = np.zeros(n)
    cons = np.zeros(n, dtype=bool)
    cons[one_idx] = True
    cons[zero_idx] = True
    u[one_idx] = 1.0
    u[zero_idx] = 0.0
    cons[one_idx] = True
    free = np.nonzero(~cons)[0]
    Kff = K[free][:, free]
    rhs = -(K[free][:, np.nonzero(cons)[0]] @ u[cons])
    return u, free, Kff, rhs


def constrained_bilaplacian(L, Mdiag, one_idx, zero_idx):
    """Solve K u = 0, K = L M^-1 L, with u = 1 on one_idx and u = 0 on zero_idx (sparse LU)."""
    u, free, Kff, rhs = constrained_system(L, Mdiag, one_idx, zero_idx)
    if len(free):
        u[free] = spla.spsolve(Kff.tocsc(), rhs, permc_spec="MMD_AT_PLUS_A")
    return u


# ----------------------------------------------------------------------------- driver

_G = {}


def _handle_system(i):
    """The constrained bilaplacian of handle i on its subdomain: (verts, u, free, K_ff,
    rhs) -- the system _solve_handle solves with SuperLU."""
    g = _G
    sub_tets_mask = g["in_sub"](i)
    tsub = g["tets"][sub_tets_mask]
    verts = np.unique(tsub)
    L, Md = assemble_subdomain(tsub, g["Kl"][sub_tets_mask], g["vol"][sub_tets_mask], verts)
    # internal boundary: subdomain vertices also used by tets outside the subdomain
    inner = g["vert_tet_count"][verts] > np.bincount(np.searchsorted(verts, tsub.ravel()),
                                                       minlength=len(verts))
    zero = set(np.nonzero(inner)[0].tolist())
    for j in g["nbrs"][i]:
        if j != i:
            zero.add(int(np.searchsorted(verts, g["cv"][j])))
    if g["dbc_mask"] is not None:
        zero.update(np.nonzero(g["dbc_mask"][verts])[0].tolist())
    one = int(np.searchsorted(verts, g["cv"][i]))
    zero.discard(one)
    u, free, Kff, rhs = constrained_system(L, Md, [one], sorted(zero))
    return verts, u, free, Kff, rhs


def _solve_handle(i):
    verts, u, free, Kff, rhs = _handle_system(i)
    if len(free):
        u[free] = spla.spsolve(Kff.tocsc(), rhs, permc_spec="MMD_AT_PLUS_A")
    return verts, u


def _handle_system_csr(i):
    verts, u, free, Kff, rhs = _handle_system(i)
    Kff = Kff.tocsr()
    return i, verts, u, free, (Kff.indptr, Kff.indices, Kff.data, Kff.shape[0]), rhs


def _solve_handles_cuda(m, workers, verbose=False):
    """The m per-handle systems assembled on CPU worker processes and solved on the GPU by a dense
    fp64 Cholesky (torch.linalg.cholesky: a library factorisation, like SuperLU on the default path;
    C5's ~56 k-vertex subdomains factor in ~1.8 s each on a B200 against hours of sparse LU)."""
    import multiprocessing as mp
    import time
    import torch
    dev = torch.device("cuda")
    res = [None] * m
    t0 = time.time()
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        for n_done, (i, verts, u, free, (ip, ix, dv, nf), rhs) in enumerate(
                pool.imap_unordered(_handle_system_csr, range(m), chunksize=1)):
            if nf:
                K = torch.zeros((nf, nf), dtype=torch.float64, device=dev)
                rows = torch.repeat_interleave(torch.arange(nf, device=dev),
                                               torch.from_numpy(np.diff(ip)).to(dev))
                K[rows, torch.from_numpy(ix.astype(np.int64)).to(dev)] = torch.from_numpy(dv).to(dev)
                Lc, info = torch.linalg.cholesky_ex(K)
                del K
                if int(info) != 0:
                    raise RuntimeError(f"handle {i}: subdomain system not positive definite (info {int(info)})")
                x = torch.cholesky_solve(torch.from_numpy(rhs).to(dev)[:, None], Lc)
                del Lc
                u[free] = x[:, 0].cpu().numpy()
            res[i] = (verts, u)
            if verbose and (n_done + 1) % 64 == 0:
                print(f"    {n_done + 1}/{m} handles ({time.time() - t0:.0f}s)", flush=True)
    return res


def _solve_dbc():
    g = _G
    dbc = g["dbc"]
    cl = np.unique(g["vert_clusters_of"](dbc))
    sub = set()
    for c in cl:
        sub.update(g["nbrs"][c])
    sub_mask = np.isin(g["assign"], np.array(sorted(sub)))
    tsub = g["tets"][sub_mask]
    verts = np.unique(tsub)
    L, Md = assemble_subdomain(tsub, g["Kl"][sub_mask], g["vol"][sub_mask], verts)
    inner = g["vert_tet_count"][verts] > np.bincount(np.searchsorted(verts, tsub.ravel()),
                                                       minlength=len(verts))
    one = np.searchsorted(verts, dbc)
    zero = set(np.nonzero(inner)[0].tolist())
    zero.update(int(np.searchsorted(verts, g["cv"][c])) for c in cl)
    zero.difference_update(one.tolist())
    u = constrained_bilaplacian(L, Md, one, sorted(zero))
    out = np.zeros(len(g["X"]))
    out[verts] = np.maximum(u, 0.0)
    return out


def n_cg_from_radius(r):
    """N_cg = the closer of 20 and 40 to the mean hop radius (ties -> 20)."""
    return 20 if abs(r - 20) <= abs(r - 40) else 40


def pou_normalise(rows, uraw, u_dbc, n_v):
    """Clip and normalise: phi_i(v) = max(u_i(v), 0) / D(v) and
    phi_DBC(v) = u_DBC(v) / D(v), D(v) = sum_j max(u_j(v), 0) + u_DBC(v), for basis entries
    (rows[k] = vertex, uraw[k] = u_i(v)).  Returns (phi per entry, phi_DBC, D); entries of
    vertices with D = 0 are left 0 (coverage holes, handled by the caller)."""
    val = np.maximum(uraw, 0.0)
    denom = np.bincount(rows, weights=val, minlength=n_v) + u_dbc
    safe = np.where(denom > 0, denom, 1.0)
    phi = np.where(denom[rows] > 0, val / safe[rows], 0.0)
    phi_dbc = np.where(denom > 0, u_dbc / safe, 0.0)
    return phi, phi_dbc, denom


def hop_radius(assign, tets, cv, n_v, m):
    """Mean over partitions of the max edge-hop distance from the centroid vertex to the
    partition's vertices, BFS on mesh edges restricted to the partition (Q7)."""
    e = np.concatenate([tets[:, [a, b]] for a in range(4) for b in range(a + 1, 4)])
    A = sp.coo_matrix((np.ones(len(e)), (e[:, 0], e[:, 1])), shape=(n_v, n_v))
    A = ((A + A.T) > 0).tocsr()
    radii = []
    for i in range(m):
        pv = np.unique(tets[assign == i])
        sub = A[pv][:, pv]
        d = sp.csgraph.shortest_path(sub, unweighted=True, indices=int(np.searchsorted(pv, cv[i])))
        radii.append(np.max(d[np.isfinite(d)]))
    return float(np.mean(radii))


def scene_partition(scene, m, seed, partition, X, tets, vol, bary):
    """Step 1: the clustering of the tets (k-means or NEXT-3's heat-geodesic
    partitioner), connectivity enforcement and empty clusters dropped.  Returns (assign, m)."""
    if partition == "heat":
        from .partition import geodesic_kmeans
        assign, _ = geodesic_kmeans(scene, m, seed)
    elif partition == "euclidean":
        C0 = kmeans_pp(bary, vol, m, seed)
        assign = lloyd(bary, vol, C0)
    else:
        raise ValueError(f"unknown partition {partition!r}")
    adj = face_adjacency(tets)
    assign = enforce_connectivity(assign.copy(), tets, adj, m)
    used = np.unique(assign)
    remap = -np.ones(m, dtype=np.int64)
    remap[used] = np.arange(len(used))
    return remap[assign], len(used)


def cached_partition(scene, cache_dir=None, partition="euclidean"):
    """scene_partition cached next to the bases (the 30 min of single-threaded k-means at C5)."""
    path = cached_basis_path(scene, cache_dir, partition)[:-4] + "_partition.npz"
    if os.path.exists(path):
        z = np.load(path)
        return z["assign"].astype(np.int64), int(z["m"])
    X, tets = scene.X, scene.tets.astype(np.int64)
    assign, m = scene_partition(scene, scene.m, scene.config, partition, X, tets, tet_volumes(X, tets),
                                tet_barycentres(X, tets))
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez_compressed(path, assign=assign.astype(np.int32), m=np.array(m))
    return assign, m


def build_basis(scene, m=None, seed=None, workers=None, verbose=False, partition="euclidean",
                solver="superlu", partition_data=None) -> Basis:
    """partition: "euclidean" (step 1 below; the default of every config) or "heat" (NEXT-3: the
    paper's stiffness-weighted heat-geodesic k-means with jump penalty and pruning,
    precompute/partition.py; m is then the initial cluster count)."""
    import time
    t0 = time.time()
    X, tets = scene.X, scene.tets.astype(np.int64)
    m = scene.m if m is None else m
    n_v, n_t = len(X), len(tets)
    seed = scene.config if seed is None else seed

    vol = tet_volumes(X, tets)
    bary = tet_barycentres(X, tets)
    if partition_data is not None:   # (assign, m) from cached_partition
        assign, m = partition_data
        assign = np.asarray(assign, dtype=np.int64)
    else:
        assign, m = scene_partition(scene, m, seed, partition, X, tets, vol, bary)
    if verbose:
        print(f"  kmeans+connectivity {time.time()-t0:.1f}s", flush=True)

    # centroid vertices
    W = np.bincount(assign, weights=vol, minlength=m)
    bc = np.stack([np.bincount(assign, weights=vol * bary[:, d], minlength=m) for d in range(3)], 1) / W[:, None]
    cv = np.zeros(m, dtype=np.int64)
    for i in range(m):
        pv = np.unique(tets[assign == i])
        dd = np.sum((X[pv] - bc[i]) ** 2, axis=1)
        cv[i] = pv[np.argmin(dd)]          # argmin: ties -> lowest vertex index
    # relabel handles in lexicographic (x, y, z) order of the centroid vertex
    order = np.lexsort((X[cv, 2], X[cv, 1], X[cv, 0]))
    newid = np.empty(m, dtype=np.int64)
    newid[order] = np.arange(m)
    assign = newid[assign]
    cv = cv[order]

    # vertex -> clusters incidence and cluster vertex-adjacency
    VC = sp.coo_matrix((np.ones(4 * n_t), (tets.ravel(), np.repeat(assign, 4))), shape=(n_v, m)).tocsr()
    VC.data[:] = 1.0
    CA = (VC.T @ VC).tocsr()
    nbrs = [np.sort(CA.indices[CA.indptr[i]:CA.indptr[i + 1]]) for i in range(m)]
    vert_tet_count = np.bincount(tets.ravel(), minlength=n_v)

    Ewt = scene.E / np.median(scene.E)
    Kl, _ = local_laplacians(X, tets, Ewt)

    dbc_mask = None
    if len(scene.dbc):
        dbc_mask = np.zeros(n_v, dtype=bool)
        dbc_mask[scene.dbc] = True

    _G.clear()
    _G.update(X=X, tets=tets, assign=assign, Kl=Kl, vol=vol, cv=cv, nbrs=nbrs,
              vert_tet_count=vert_tet_count, dbc_mask=dbc_mask, dbc=np.asarray(scene.dbc, np.int64))
    _G["in_sub"] = lambda i: np.isin(assign, nbrs[i])
    _G["vert_clusters_of"] = lambda vs: np.concatenate(
        [VC.indices[VC.indptr[v]:VC.indptr[v + 1]] for v in vs])

    if workers is None:
        workers = min(os.cpu_count() or 1, 64)
    t1 = time.time()
    if solver == "cuda":
        res = _solve_handles_cuda(m, workers, verbose)
    elif workers > 1 and m > 8:
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        with ctx.Pool(workers) as pool:
            res = pool.map(_solve_handle, range(m), chunksize=max(1, m // (4 * workers)))
    else:
        res = [_solve_handle(i) for i in range(m)]
    if verbose:
        print(f"  {m} bilaplacian solves {time.time()-t1:.1f}s ({workers} workers)", flush=True)

    u_dbc = _solve_dbc() if dbc_mask is not None else np.zeros(n_v)

    # POU normalisation
    rows = np.concatenate([r[0] for r in res])
    hid = np.concatenate([np.full(len(r[0]), i, dtype=np.int64) for i, r in enumerate(res)])
    uraw = np.concatenate([r[1] for r in res])
    _, _, denom = pou_normalise(rows, uraw, u_dbc, n_v)
    free = np.ones(n_v, dtype=bool)
    if dbc_mask is not None:
        free &= ~dbc_mask
    holes = np.nonzero((denom <= 0) & free)[0]
    if len(holes):
        # Reading B1: the paper is silent on a free vertex where every clipped
        # weight vanishes; such a vertex is given to the covering handle (v in T_i) with the
        # largest unclipped u_i(v), weight 1.  POU and hence linear precision still hold.
        hole_mask = np.zeros(n_v, dtype=bool)
        hole_mask[holes] = True
        sel = np.nonzero(hole_mask[rows])[0]
        o = np.lexsort((-uraw[sel], rows[sel]))
        srt = sel[o]
        first = np.ones(len(srt), dtype=bool)
        first[1:] = rows[srt][1:] != rows[srt][:-1]
        uraw = uraw.copy()
        uraw[srt[first]] = 1.0
        if verbose:
            print(f"  coverage holes repaired: {len(holes)}")
    phi, phi_dbc, denom = pou_normalise(rows, uraw, u_dbc, n_v)
    if np.any(denom[free] <= 0):
        bad = np.nonzero((denom <= 0) & free)[0]
        raise RuntimeError(f"basis coverage hole at {len(bad)} free vertices, e.g. {bad[:5]}")
    keep = phi > 0
    rows, hid, phi = rows[keep], hid[keep], phi[keep]
    o = np.lexsort((hid, rows))
    rows, hid, phi = rows[o], hid[o], phi[o]
    vptr = np.zeros(n_v + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_v), out=vptr[1:])
    if dbc_mask is not None:
        phi_dbc[dbc_mask] = 1.0
    phi_aff = 1.0 - phi_dbc

    mass = np.bincount(tets.ravel(), weights=np.repeat(scene.rho * vol / 4.0, 4), minlength=n_v)
    com = (mass[:, None] * X).sum(0) / mass.sum()

    t2 = time.time()
    hr = hop_radius(assign, tets, cv, n_v, m)
    n_cg = n_cg_from_radius(hr)
    if verbose:
        print(f"  hop radius {hr:.2f} -> n_cg {n_cg} ({time.time()-t2:.1f}s); total {time.time()-t0:.1f}s")
    return Basis(m=m, origins=X[cv].copy(), n_holes=len(holes), vptr=vptr, handle=hid.astype(np.int32), phi=phi,
                 phi_dbc=phi_dbc, phi_affine=phi_aff, affine_origin=com, n_cg=n_cg, hop_radius=hr,
                 cluster=assign.astype(np.int32), centroid_vertex=cv)


def cached_basis_path(scene, cache_dir=None, partition="euclidean"):
    cache_dir = cache_dir or os.environ.get("MSIM_CACHE", os.path.join(os.path.dirname(__file__), "..", ".cache"))
    tag = "" if partition == "euclidean" else f"_{partition}"
    key = f"{scene.name}_{scene.n_verts}_{scene.n_tets}_{scene.m}_{BASIS_VERSION}{tag}.npz"
    return os.path.join(cache_dir, key)


def cached_basis(scene, cache_dir=None, **kw) -> Basis:
    """Build or load the basis of a scene (cache keyed by scene name, sizes, m, version and
    partitioner)."""
    path = cached_basis_path(scene, cache_dir, kw.get("partition", "euclidean"))
    os.makedirs(os.path.dirname(path), exist_ok=True)
    if os.path.exists(path):
        return Basis.load(path)
    b = build_basis(scene, **kw)
    b.save(path)
    return b
