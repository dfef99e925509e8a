"""The world > 1 (slab-partitioned) path of the library on one GPU: W contexts, one host thread
each, exchange ghost values and reductions through the in-process hub (ms_create_hub; every
collective synchronises the caller's stream, so no kernel waits on another context).  The
partitioned timesteps must reproduce the single-context run: only the order of the rank sums
differs, so positions agree to ~1e-12 of the bounding box and the Newton iteration counts match.
The NCCL backend runs the same code with ncclAllReduce / ncclSend / ncclRecv instead of the hub.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from precompute.basis import build_basis  # noqa: E402
from precompute.mesh import make_scene, scene_small_drop  # noqa: E402


@pytest.fixture(scope="module")
def msim():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_13386_b200 import msim as m
    return m


def run_ranks(msim, s, b, world, steps, **params):
    import torch
    hub = msim.Hub(world)
    streams = [torch.cuda.Stream() for _ in range(world)]
    ctxs = [msim.context_from_scene(s, b, stream=streams[r].cuda_stream, rank=r, world=world, hub=hub, **params)
            for r in range(world)]
    stats = [[] for _ in range(world)]
    errors = []

    def work(r):
        try:
            for _ in range(steps):
                stats[r].append(ctxs[r].timestep().newton_iters)
        except Exception as e:  # noqa: BLE001
            errors.append((r, repr(e)))

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errors, errors
    x = np.zeros((s.n_verts, 3))
    v = np.zeros((s.n_verts, 3))
    owned = np.zeros(s.n_verts, dtype=int)
    for r in range(world):
        P = msim.partition(r, world, s.X, s.tets)
        own = P["l2g"][:P["nv_own"]]
        xr, vr = ctxs[r].get_state()
        x[own], v[own] = xr[own], vr[own]
        owned[own] += 1
    assert np.all(owned == 1)
    for r in range(1, world):
        assert stats[r] == stats[0]   # every rank takes the same decisions
    return x, v, stats[0]


@pytest.mark.parametrize("name,world,steps", [("drop", 2, 6), ("drop", 3, 4), ("c2", 2, 3)])
def test_partitioned_timesteps_match_single(msim, name, world, steps):
    if name == "drop":
        s = scene_small_drop(n=(10, 4, 3), m=6, drop=0.002)
    else:
        s = make_scene(2)
    b = build_basis(s, workers=1)
    ref = msim.context_from_scene(s, b)
    its = [ref.timestep().newton_iters for _ in range(steps)]
    x_ref, v_ref = ref.get_state()
    x, v, its_p = run_ranks(msim, s, b, world, steps)
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    assert its_p == its
    assert np.abs(x - x_ref).max() <= 1e-9 * diag
    assert np.abs(v - v_ref).max() <= 1e-9 * diag / s.h


def test_partitioned_two_level_refinement_matches_single(msim):
    """NEXT-4 two-level refinement on 2 ranks: restrict sums across ranks, the replicated factor
    solves, the lift and the z halo give the single-context iterates (same PCG counts)."""
    s = scene_small_drop(n=(10, 4, 3), m=6, drop=0.002)
    b = build_basis(s, workers=1)
    ref = msim.context_from_scene(s, b, refine_mode=1)
    its = [ref.timestep().newton_iters for _ in range(4)]
    x_ref, _ = ref.get_state()
    x, _, its_p = run_ranks(msim, s, b, 2, 4, refine_mode=1)
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    assert its_p == its
    assert np.abs(x - x_ref).max() <= 1e-9 * diag


@pytest.mark.parametrize("name,steps", [("drop", 6), ("c2", 3)])
def test_nccl_backend_world1_matches_single(msim, name, steps):
    """The NCCL backend itself on one GPU: a world-1 context created with an ncclUniqueId takes the
    partitioned code path (slab plan with one slab, ncclAllReduce of every rank sum, the empty
    halo group, the graph-captured distributed PCG loop and coarse stages -- the hub is not
    capturable, so only this test runs those captures).  One rank owns everything, so the sums
    have a single term and the timesteps must reproduce the plain context."""
    if name == "drop":
        s = scene_small_drop(n=(10, 4, 3), m=6, drop=0.002)
    else:
        s = make_scene(2)
    b = build_basis(s, workers=1)
    ref = msim.context_from_scene(s, b)
    its = [ref.timestep().newton_iters for _ in range(steps)]
    x_ref, v_ref = ref.get_state()
    ctx = msim.context_from_scene(s, b, rank=0, world=1, nccl_id=msim.nccl_unique_id())
    its_n = [ctx.timestep().newton_iters for _ in range(steps)]
    x, v = ctx.get_state()
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    assert its_n == its
    assert np.abs(x - x_ref).max() <= 1e-9 * diag
    assert np.abs(v - v_ref).max() <= 1e-9 * diag / s.h
