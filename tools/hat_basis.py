"""A trilinear-hat partition-of-unity basis on a regular lattice of handles, for exercising the CUDA
path at full size while the paper's basis (precompute/basis.py: k-means + per-handle bilaplacian
solves, hours of CPU at C5) is not available.  NOT the paper's basis: phi_i = h_i^2 / sum_j h_j^2 with
h_i the trilinear hat of lattice node i (partition of unity, <= 8 handles per vertex; the squares
break the hats' linear precision, which together with the monomials [1, X - c_i] of Eq. 7 would
give B a 9-dimensional null space and a singular S), handle origins at the nodes, no DBC.
Used by tools/c5_probe.py (memory / index-width / timing probe) and, while the paper's C5 basis is
not cached, by the C5 stand-in parity cases (tests/test_gpu_fullsize.py, tests/test_gpu_newton_fullsize.py
"C5-standin-basis", oracle fixtures from tools/oracle_fixtures.py --hat): the oracle and the CUDA path
then consume the same stand-in arrays.  Bench lines use the paper's basis."""
import numpy as np

from precompute.basis import Basis


def hat_basis(scene, nodes=(16, 8, 8)):
    X = scene.X
    lo, hi = X.min(0), X.max(0)
    n = np.array(nodes)
    h = (hi - lo) / (n - 1)
    t = (X - lo) / h                                   # lattice coordinates
    c = np.minimum(np.floor(t).astype(np.int64), n - 2)
    f = t - c
    rows, hid, phi = [], [], []
    nv = len(X)
    for dx in (0, 1):
        for dy in (0, 1):
            for dz in (0, 1):
                w = ((f[:, 0] if dx else 1 - f[:, 0]) * (f[:, 1] if dy else 1 - f[:, 1])
                     * (f[:, 2] if dz else 1 - f[:, 2])) ** 2
                node = ((c[:, 0] + dx) * n[1] + (c[:, 1] + dy)) * n[2] + (c[:, 2] + dz)   # x-major = (x, y, z) order
                rows.append(np.arange(nv))
                hid.append(node)
                phi.append(w)
    rows, hid, phi = np.concatenate(rows), np.concatenate(hid), np.concatenate(phi)
    keep = phi > 1e-14
    rows, hid, phi = rows[keep], hid[keep], phi[keep]
    o = np.lexsort((hid, rows))
    rows, hid, phi = rows[o], hid[o], phi[o]
    s = np.bincount(rows, weights=phi, minlength=nv)
    phi = phi / s[rows]
    vptr = np.zeros(nv + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=nv), out=vptr[1:])
    I, J, K = np.meshgrid(np.arange(n[0]), np.arange(n[1]), np.arange(n[2]), indexing="ij")
    origins = lo + np.stack([I.ravel(), J.ravel(), K.ravel()], 1) * h
    m = int(n.prod())
    tets = np.asarray(scene.tets, dtype=np.int64)
    bc = X[tets].mean(1)
    cc = np.minimum(np.floor((bc - lo) / h).astype(np.int64), n - 2)
    cluster = ((cc[:, 0] * n[1] + cc[:, 1]) * n[2] + cc[:, 2]).astype(np.int32)
    vol = np.abs(np.linalg.det(X[tets[:, 1:]] - X[tets[:, :1]])) / 6.0
    mass = np.bincount(tets.ravel(), weights=np.repeat(vol / 4.0, 4), minlength=nv)
    com = (mass[:, None] * X).sum(0) / mass.sum()
    from scipy.spatial import cKDTree
    cv = cKDTree(X).query(origins)[1]
    return Basis(m=m, origins=origins, vptr=vptr, handle=hid.astype(np.int32), phi=phi,
                 phi_dbc=np.zeros(nv), phi_affine=np.ones(nv), affine_origin=com, n_cg=20, hop_radius=0.0,
                 cluster=cluster, centroid_vertex=cv.astype(np.int64))
