"""Multi-GPU slab partition (csrc/dist.cpp) on CPU: two `gloo` ranks take the
plan the library builds at ms_upload_mesh (ms_partition, host-only) and check that it is a valid
SPMD decomposition of the path's operations:
  * owned vertices and owned tets partition the mesh (energies counted once);
  * the local tets of a rank hold every tet incident to an owned vertex (owned rows of the
    gradient / Hessian / Galerkin terms are complete);
  * what rank r sends to q is exactly what q expects from r (same global ids, same order);
  * a halo-exchanged distributed product with the mesh operator A (assembled per tet, like the
    Hessian) over gloo point-to-point equals the global product on every owned row, and rank-
    summed owned partial dots equal the global dot (the PCG reductions).
"""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def tet_operator(X, tets, n):
    """Symmetric per-tet assembled operator (edge-length weighted graph Laplacian + identity)."""
    rows, cols, vals = [], [], []
    for a in range(4):
        for b in range(4):
            if a == b:
                continue
            w = 1.0 / (1e-3 + np.linalg.norm(X[tets[:, a]] - X[tets[:, b]], axis=1))
            rows += [tets[:, a], tets[:, a]]
            cols += [tets[:, b], tets[:, a]]
            vals += [-w, w]
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    return A + sp.identity(n, format="csr")


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from paper_2508_13386_b200 import msim
        from precompute.mesh import make_scene
        s = make_scene(2)
        X, tets, n = s.X, np.asarray(s.tets), s.n_verts
        P = msim.partition(rank, world, X, tets)
        own = P["l2g"][:P["nv_own"]]
        loc_t = P["tet_l2g"]
        # ---- partition of vertices / tets, completeness of owned rows
        owns = [None] * world
        dist.all_gather_object(owns, (own.tolist(), loc_t[:P["nt_own"]].tolist()))
        allv = np.concatenate([np.array(o[0]) for o in owns])
        allt = np.concatenate([np.array(o[1]) for o in owns])
        assert len(allv) == n and len(np.unique(allv)) == n
        assert len(allt) == len(tets) and len(np.unique(allt)) == len(tets)
        incident = np.flatnonzero(np.isin(tets, own).any(axis=1))
        assert np.array_equal(np.sort(loc_t), incident)
        # ---- halo plans agree pairwise
        plans = [None] * world
        dist.all_gather_object(plans, ({k: v.tolist() for k, v in P["send"].items()},
                                       {k: v.tolist() for k, v in P["recv"].items()}))
        for peer, ids in P["recv"].items():
            assert plans[peer][0][rank] == ids.tolist()
        # ---- distributed product with halo exchange == global product
        A = tet_operator(X, tets, n)
        rng = np.random.default_rng(5)
        xg = rng.standard_normal(n)
        x = np.full(n, np.nan)
        x[own] = xg[own]                                   # a rank starts with its owned entries
        reqs = []
        for peer, ids in P["send"].items():
            reqs.append(dist.isend(torch.from_numpy(x[ids].copy()), dst=peer))
        for peer, ids in P["recv"].items():
            buf = torch.empty(len(ids), dtype=torch.float64)
            dist.recv(buf, src=peer)
            x[ids] = buf.numpy()
        for r in reqs:
            r.wait()
        A_loc = tet_operator(X, tets[loc_t], n)           # assembled from the local tets only
        y_own = (A_loc @ np.nan_to_num(x, nan=0.0))[own]
        assert np.all(np.isfinite(x[np.unique(tets[loc_t])]))   # every local vertex received
        y_ref = (A @ xg)[own]
        assert np.abs(y_own - y_ref).max() <= 1e-12 * np.abs(y_ref).max()
        part = torch.tensor([float(xg[own] @ y_ref)], dtype=torch.float64)
        dist.all_reduce(part)
        assert abs(part.item() - xg @ (A @ xg)) <= 1e-10 * abs(xg @ (A @ xg))
        q.put((rank, "ok"))
    except BaseException as e:  # report to the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partition_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(v == "ok" for v in res.values()), res
