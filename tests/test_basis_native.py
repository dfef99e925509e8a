"""The native basis build (ms_basis_compute / ms_basis_build, include/msim.h; §3.5
L304-381, §3.6, §3.7.2) against the Python precompute (precompute/basis.py,
the input generator both the CUDA path and the oracle consume).

Both follow the same algorithm with the same counter-based kmeans++ draws and tie rules, so the
partition (tet -> cluster), the centroid vertices, the vertex-major (handle) lists, the hole
repairs and N_cg must be identical.  The weights come from different sparse direct solvers
(SuperLU in scipy vs the library's envelope Cholesky) of the same bilaplacian systems; they agree
to the rounding of those solves, amplified by the systems' conditioning, which grows with the
square of the stiffness contrast (the Laplacian is E-weighted, Q17): 1e-12 for the homogeneous
C1, 1e-9 for the log-normal drop scene, 1e-6 for C2 (contrast 1e4).
"""
import numpy as np
import pytest

from precompute.basis import build_basis
from precompute.mesh import make_scene, scene_small_drop


def _msim():
    try:
        from paper_2508_13386_b200 import msim
    except ImportError as e:       # the library is built by __graft_entry__.build()
        pytest.fail(f"libmsim.so missing: {e}")
    return msim


@pytest.mark.parametrize("name,tol", [("c1", 1e-12), ("drop", 1e-9), ("c2", 1e-6)])
def test_native_basis_matches_precompute(name, tol):
    msim = _msim()
    s = {"c1": lambda: make_scene(1), "c2": lambda: make_scene(2), "drop": scene_small_drop}[name]()
    b = build_basis(s, workers=1)
    info, o = msim.basis_compute(s.X, s.tets, s.E, s.rho, s.dbc, s.m, s.config)
    assert info["m"] == b.m and info["n_cg"] == b.n_cg and info["n_holes"] == b.n_holes
    assert info["hop_radius"] == b.hop_radius
    assert np.array_equal(o["cluster"], b.cluster)
    assert np.array_equal(o["centroid_vertex"], b.centroid_vertex)
    assert np.array_equal(o["origins"], b.origins)
    assert np.array_equal(o["vptr"], b.vptr) and np.array_equal(o["handle"], b.handle)
    assert np.abs(o["phi"] - b.phi).max() <= tol
    assert np.abs(o["phi_affine"] - b.phi_affine).max() <= tol
    assert np.abs(o["affine_origin"] - b.affine_origin).max() <= 1e-14 * np.abs(b.affine_origin).max()


def test_native_basis_properties_c2():
    """Partition of unity with the Dirichlet weight, zero rows at pinned vertices, linear
    precision B q_aff = (1 - phi_DBC)(A X + t)."""
    msim = _msim()
    s = make_scene(2)
    info, o = msim.basis_compute(s.X, s.tets, s.E, s.rho, s.dbc, s.m, s.config)
    nv = s.n_verts
    rows = np.repeat(np.arange(nv), np.diff(o["vptr"]))
    pou = np.bincount(rows, weights=o["phi"], minlength=nv) + (1.0 - o["phi_affine"])
    assert np.abs(pou - 1.0).max() < 1e-12
    assert np.all(np.diff(o["vptr"])[s.dbc] == 0) and np.all(o["phi_affine"][s.dbc] == 0.0)
    A = np.array([[1.1, 0.2, -0.3], [0.05, 0.9, 0.1], [-0.2, 0.3, 1.2]])
    t = np.array([0.3, -0.1, 0.2])
    c = o["origins"][o["handle"]]
    w = o["phi"][:, None] * ((s.X[rows] - c) @ A.T + (c @ A.T + t))
    field = np.zeros((nv, 3))
    np.add.at(field, rows, w)
    ref = o["phi_affine"][:, None] * (s.X @ A.T + t)
    assert np.abs(field - ref).max() < 1e-10


def test_native_basis_rejects_bad_arguments():
    msim = _msim()
    s = make_scene(1)
    with pytest.raises(msim.MsimError):
        msim.basis_compute(s.X, s.tets, s.E, s.rho, s.dbc, 0, 1)
    bad = np.array(s.tets).copy()
    bad[0, 0] = s.n_verts
    with pytest.raises(msim.MsimError):
        msim.basis_compute(s.X, bad, s.E, s.rho, s.dbc, 4, 1)


@pytest.mark.gpu
def test_ms_basis_build_context_c2():
    """ms_basis_build on a context builds and uploads the basis: its export equals the host-only
    build, and timesteps with it track those with the precompute basis (weights differ only by
    the solver rounding above)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    msim = _msim()
    s = make_scene(2)
    b = build_basis(s, workers=1)
    ctx = msim.context_from_scene(s, b)           # mesh, Dirichlet set, ground, params, basis
    ctx2 = msim.Context(0)
    ctx2.upload_mesh(s.X, s.tets, s.E, s.nu, s.rho)
    ctx2.set_dirichlet(s.dbc)
    ctx2.set_params(h=s.h, gravity=s.gravity, eps=s.eps, max_newton=s.max_newton)
    info, o = ctx2.basis_build(s.m, s.config)
    assert np.array_equal(o["cluster"], b.cluster) and np.array_equal(o["handle"], b.handle)
    assert info["n_cg"] == b.n_cg
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    for _ in range(3):
        st1, st2 = ctx.timestep(), ctx2.timestep()
        assert st1.newton_iters == st2.newton_iters
        x1, _ = ctx.get_state()
        x2, _ = ctx2.get_state()
        assert np.abs(x1 - x2).max() <= 1e-6 * diag
