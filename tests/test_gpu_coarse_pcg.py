"""Parity of the paper's coarse mode (MS_COARSE_PCG, NEXT-1; §3.7.1, Alg. 2
L427-450): block-Jacobi PCG to a relative residual on the matrix-free sandwich B^T (H (B p)),
GPU against oracle/solver.py (coarse_mode="pcg").

* at fixed iteration counts (tolerance 0, cap k): d_s to 1e-8 (the iterates are unique);
* at the paper's tolerance 1e-4 the iterate is not unique in floating point: CG iterates of two
  implementations drift apart by rounding that grows with the iteration count on an
  ill-conditioned coarse system (loss of orthogonality: 2.6e-8 relative after ~30 steps on C1,
  1e-6 after 45 on the drop scene, 5e-6 after 110 on C2, while every fixed count <= 10 agrees to
  1e-8).  What is unique is checked exactly -- the number of SMS iterations -- and the rest for
  validity: the GPU's d_s meets the paper's stopping rule measured by the oracle,
  ||B^T(-g - H d_s)|| <= 1e-4 ||B^T r1|| (the SMS residual of q with B q = d_s - d_a), and lies within
  the solve's accuracy of the oracle's (1e-4 relative), with the same line-search outcome;
* free-running timesteps with the mode on, positions to 1e-6 of the bounding box;
* the C4 configuration (1.57 M tets, m = 512): one bootstrapped Newton iteration in this mode.
Tolerances as in tests/test_gpu_parity.py.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import coarse, ip, solver  # noqa: E402
from precompute.basis import build_basis, cached_basis  # noqa: E402
from precompute.mesh import contact_state, make_scene, random_state, scene_small_drop  # noqa: E402

PCG = 1


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


@pytest.mark.parametrize("name", ["c1", "drop", "c2"])
def test_coarse_pcg_fixed_iterations(msim, name):
    s, b = _scene(name)
    ctx = msim.context_from_scene(s, b)
    m = ip.make_model(s)
    x, xhat = _state(s, 41)
    ctx.set_step_state(s.X, xhat, x)
    ctx.assemble()
    H = ip.hessian(m, x, xhat).tocsr()
    g = ip.gradient(m, x, xhat)
    Ua, Us = coarse.affine_matrix(s.X, b), coarse.sms_matrix(s.X, b)
    for k in (1, 3, 10):
        ctx.set_params(coarse_mode=PCG, coarse_tol=0.0, coarse_max_iter=k)
        ds, da = ctx.subspace_direction()
        ds_o, da_o, _, its = solver.subspace_direction(H, g, Ua, Us, "pcg", tol=0.0, max_iter=k)
        assert its == k
        assert rel_err(da, da_o) < 1e-9, (name, k)
        assert rel_err(ds, ds_o) < 1e-8, (name, k, rel_err(ds, ds_o))


@pytest.mark.parametrize("name", ["c1", "drop", "c2"])
def test_coarse_pcg_tolerance_newton(msim, name):
    s, b = _scene(name)
    ctx = msim.context_from_scene(s, b, coarse_mode=PCG)
    sim = solver.OracleSim(s, b, coarse_mode="pcg")
    x, xhat = _state(s, 43)
    ctx.set_step_state(s.X, xhat, x)
    sim.x_t, sim.xhat, sim.x = s.X.copy(), xhat, x.copy()
    g = ip.gradient(sim.model, x, xhat)
    H = ip.hessian(sim.model, x, xhat).tocsr()
    _, _, _, its_o = solver.subspace_direction(H, g, sim.Ua, sim.Us, "pcg", tol=1e-4)
    info = sim.newton_iteration()
    st = ctx.newton_step()
    ds, df = ctx.get_direction()
    # the stopping index is an integer decided by ||r_k|| <= 1e-4 ||b|| in fp64 on both sides; the
    # iterates differ by summation order (atomic-free GPU sums vs scipy), so a residual that lands
    # within rounding of the threshold may cross one iteration apart (drop scene: 44 / 45) -- the
    # rule itself is checked on the GPU's own iterate below, the fixed-count iterates above to 1e-8
    assert abs(st.coarse_iters - its_o) <= 1, (st.coarse_iters, its_o)
    # validity: the paper's stopping rule holds for the GPU's own iterate
    _, da_o, _, _ = solver.subspace_direction(H, g, sim.Ua, sim.Us, "pcg", tol=1e-4)
    r1 = -g.ravel() - H @ da_o
    res = np.linalg.norm(sim.Us.T @ (-g.ravel() - H @ ds))
    assert res <= 1.01e-4 * np.linalg.norm(sim.Us.T @ r1), (res, np.linalg.norm(sim.Us.T @ r1))
    assert rel_err(ds, info.ds) < 1e-4, (st.coarse_iters, rel_err(ds, info.ds))
    assert abs(st.alpha0 - info.alpha0) <= 1e-4 * info.alpha0
    assert st.ls_evals == info.ls_evals


def test_coarse_pcg_timesteps_drop(msim):
    s, b = _scene("drop")
    ctx = msim.context_from_scene(s, b, coarse_mode=PCG)
    sim = solver.OracleSim(s, b, coarse_mode="pcg")
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    for _ in range(4):
        st = ctx.timestep()
        infos = sim.timestep()
        x, _ = ctx.get_state()
        assert st.newton_iters == len(infos), (st.status, st.newton_iters, st.last_alpha, st.last_ds_norm, st.coarse_iters)
        assert np.abs(x - sim.x).max() <= 1e-6 * diag


def test_coarse_pcg_fullsize_c4(msim):
    """One bootstrapped Newton iteration of C4 (the bench configuration) in the paper's mode."""
    s = make_scene(4)
    b = cached_basis(s)
    ctx = msim.context_from_scene(s, b, coarse_mode=PCG)
    sim = solver.OracleSim(s, b, coarse_mode="pcg")
    x_t, v_t = contact_state(s)
    sim.x, sim.v = x_t.copy(), v_t
    sim.begin_step()
    ctx.set_step_state(x_t, sim.xhat, x_t)
    info = sim.newton_iteration()
    st = ctx.newton_step()
    ds, df = ctx.get_direction()
    assert rel_err(ds, info.ds) < 1e-7, (st.coarse_iters, rel_err(ds, info.ds))
    assert rel_err(ds + df, info.d) < 1e-7
    assert abs(st.alpha0 - info.alpha0) <= 1e-7 * info.alpha0
    assert st.ls_evals == info.ls_evals and st.coarse_iters > 0
