"""Parity of the NEXT-4 two-level refinement (MS_REFINE_TWO_LEVEL, not in the paper,
reading N4 of DESIGN.md): PCG on H d_f = -g - H d_s with y = D^-1 r, z = y + U_s S^-1 U_s^T (r - H y), GPU against
oracle/solver.py two_level_pcg through OracleSim(refine="two_level").

* fixed iteration counts (tolerance 0, cap k): d_f to 1e-8 (the iterates are unique);
* to the default tolerance 1e-2 ||g|| and to 1e-4 ||g|| (cap 100): the iteration count (unique)
  and the direction (validity: the GPU's d meets the stopping rule measured by the oracle unless
  the cap was hit; agreement 1e-7);
* free-running timesteps with the mode on (drop scene), positions to 1e-6 of the bounding box;
* C4 (1.57 M tets, m = 512): one bootstrapped contact Newton iteration in this mode.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import ip, solver  # noqa: E402
from precompute.basis import build_basis, cached_basis  # noqa: E402
from precompute.mesh import contact_state, make_scene, random_state, scene_small_drop  # noqa: E402

TWO_LEVEL = 1


@pytest.fixture(scope="module")
def msim():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_13386_b200 import msim as m
    return m


def rel_err(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def _scene(name):
    if name == "c1":
        s = make_scene(1)
    elif name == "c2":
        s = make_scene(2)
    else:
        s = scene_small_drop(n=(6, 5, 4), m=6, drop=0.002)
    return s, build_basis(s, workers=1)


def _state(s, seed):
    x = random_state(s, 0.01, seed)
    if s.ground is not None:
        x[:, 2] = np.maximum(x[:, 2], 0.3 * s.ground["dhat"])
    rng = np.random.default_rng(seed + 1)
    xhat = s.X + 0.002 * s.a * rng.standard_normal(s.X.shape)
    return x, xhat


def _bootstrapped(msim, s, b, x, xhat, **kw):
    ctx = msim.context_from_scene(s, b, refine_mode=TWO_LEVEL, **{k: v for k, v in kw.items()})
    sim = solver.OracleSim(s, b, refine="two_level", **{k: v for k, v in kw.items()})
    ctx.set_step_state(s.X, xhat, x)
    sim.x_t, sim.xhat, sim.x = s.X.copy(), xhat, x.copy()
    info = sim.newton_iteration()
    st = ctx.newton_step()
    ds, df = ctx.get_direction()
    return ctx, sim, info, st, ds, df


@pytest.mark.parametrize("name", ["c1", "drop", "c2"])
def test_two_level_fixed_iterations(msim, name):
    s, b = _scene(name)
    x, xhat = _state(s, 51)
    for k in (1, 3, 10):
        _, _, info, st, ds, df = _bootstrapped(msim, s, b, x, xhat, refine_tol=0.0, refine_max_iter=k)
        assert st.n_cg == k == info.cg_iters
        assert rel_err(ds, info.ds) < 1e-8
        assert rel_err(df, info.df) < 1e-8, (name, k, rel_err(df, info.df))
        assert abs(st.alpha0 - info.alpha0) <= 1e-8 * info.alpha0 and st.ls_evals == info.ls_evals


@pytest.mark.parametrize("name", ["c1", "drop", "c2"])
@pytest.mark.parametrize("tol", [1e-2, 1e-4])
def test_two_level_tolerance(msim, name, tol):
    s, b = _scene(name)
    x, xhat = _state(s, 53)
    _, sim, info, st, ds, df = _bootstrapped(msim, s, b, x, xhat, refine_tol=tol)
    assert st.n_cg == info.cg_iters, (st.n_cg, info.cg_iters)
    g = ip.gradient(sim.model, x, xhat).ravel()
    H = ip.hessian(sim.model, x, xhat).tocsr()
    res = np.linalg.norm(-g - H @ (ds + df))
    if st.n_cg < 100:
        assert res <= 1.01 * tol * np.linalg.norm(g), (res / np.linalg.norm(g), st.n_cg)
    assert rel_err(ds + df, info.d) < 1e-7, rel_err(ds + df, info.d)
    assert abs(st.alpha0 - info.alpha0) <= 1e-7 * info.alpha0 and st.ls_evals == info.ls_evals


def test_two_level_timesteps_drop(msim):
    s, b = _scene("drop")
    ctx = msim.context_from_scene(s, b, refine_mode=TWO_LEVEL)
    sim = solver.OracleSim(s, b, refine="two_level")
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    for _ in range(4):
        st = ctx.timestep()
        infos = sim.timestep()
        x, _ = ctx.get_state()
        assert st.newton_iters == len(infos)
        assert st.pcg_iters == sum(i.cg_iters for i in infos)
        assert np.abs(x - sim.x).max() <= 1e-6 * diag


def test_two_level_requires_exact_coarse(msim):
    s, b = _scene("drop")
    ctx = msim.context_from_scene(s, b)
    with pytest.raises(msim.MsimError):
        ctx.set_params(refine_mode=TWO_LEVEL, coarse_mode=1)


def test_two_level_fullsize_c4(msim):
    """One bootstrapped contact Newton iteration of C4 (the bench configuration) in this mode."""
    s = make_scene(4)
    b = cached_basis(s)
    ctx = msim.context_from_scene(s, b, refine_mode=TWO_LEVEL)
    sim = solver.OracleSim(s, b, refine="two_level")
    x_t, v_t = contact_state(s)
    sim.x, sim.v = x_t.copy(), v_t
    sim.begin_step()
    ctx.set_step_state(x_t, sim.xhat, x_t)
    info = sim.newton_iteration()
    st = ctx.newton_step()
    ds, df = ctx.get_direction()
    assert st.n_cg == info.cg_iters, (st.n_cg, info.cg_iters)
    assert rel_err(ds, info.ds) < 1e-8
    assert rel_err(ds + df, info.d) < 1e-7, rel_err(ds + df, info.d)
    assert abs(st.alpha0 - info.alpha0) <= 1e-7 * info.alpha0 and st.ls_evals == info.ls_evals
