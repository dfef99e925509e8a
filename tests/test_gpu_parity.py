"""GPU parity: the CUDA path (through the C-ABI) against the oracle, element by element, on the
same seeded inputs.  Tolerances (BASELINE.json north_star):
  * per-element gradient / PSD Hessian: max |gpu - oracle| <= 1e-10 * max |oracle| per element
  * PCG solution / Newton direction:    ||gpu - oracle|| <= 1e-8 ||oracle||
  * per-timestep positions:             max_v |x_gpu - x_oracle| <= 1e-6 * bbox diagonal
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import coarse, fem, ip, solver  # noqa: E402
from precompute.basis import build_basis  # noqa: E402
from precompute.mesh import make_scene, random_state, scene_small_drop  # noqa: E402


@pytest.fixture(scope="module")
def msim():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_13386_b200 import msim as m
    return m


def rel_err(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def per_element_rel(a, b):
    a = a.reshape(len(a), -1)
    b = b.reshape(len(b), -1)
    return np.max(np.abs(a - b).max(axis=1) / np.maximum(np.abs(b).max(axis=1), 1e-300))


SCENES = {}


def scene_and_basis(name):
    if name not in SCENES:
        if name == "c1":
            s = make_scene(1)
        elif name == "c2":
            s = make_scene(2)
        elif name == "drop":
            s = scene_small_drop(n=(6, 5, 4), m=6, drop=0.002)
        elif name == "drop_tiny":
            s = scene_small_drop(n=(3, 3, 2), m=3, drop=0.003)
        SCENES[name] = (s, build_basis(s, workers=1))
    return SCENES[name]


def perturbed(scene, amp, seed):
    x = random_state(scene, amp, seed)
    if scene.ground is not None:
        x[:, 2] = np.maximum(x[:, 2], 0.3 * scene.ground["dhat"])
    return x


# ----------------------------------------------------------------------------- elements
@pytest.mark.parametrize("name,amp", [("c1", 0.02), ("c2", 0.05), ("drop", 0.08)])
def test_element_parity(msim, name, amp):
    s, b = scene_and_basis(name)
    ctx = msim.context_from_scene(s, b)
    m = ip.make_model(s)
    x = perturbed(s, amp, seed=3)
    Ee, ge, He = ctx.eval_elements(x)
    E_o = fem.element_energy(x, m.tets, m.Bm, m.V, m.mu, m.lam)
    g_o = fem.element_gradient(x, m.tets, m.Bm, m.V, m.mu, m.lam)
    H_o = fem.element_hessian_psd(x, m.tets, m.Bm, m.V, m.mu, m.lam)
    assert np.all(np.isfinite(E_o))
    assert np.max(np.abs(Ee - E_o) / np.maximum(np.abs(E_o), 1e-30)) < 1e-9
    assert per_element_rel(ge, g_o) < 1e-10
    assert per_element_rel(He, H_o) < 1e-10
    # the projection is active on a good share of elements (the test exercises the clamp)
    w = np.linalg.eigvalsh(fem.element_hessian(x, m.tets, m.Bm, m.V, m.mu, m.lam))
    assert np.mean(w[:, 0] < -1e-8 * np.abs(w).max(axis=1)) > 0.1


def test_element_parity_large_strain(msim):
    s, b = scene_and_basis("c1")
    ctx = msim.context_from_scene(s, b)
    m = ip.make_model(s)
    rng = np.random.default_rng(9)
    # per-element compressions / shears up to 30 %; keep non-inverted elements only
    x = s.X + 0.03 * rng.standard_normal(s.X.shape)
    Ee, ge, He = ctx.eval_elements(x)
    E_o = fem.element_energy(x, m.tets, m.Bm, m.V, m.mu, m.lam)
    ok = np.isfinite(E_o)
    assert ok.mean() > 0.5
    assert np.array_equal(np.isfinite(Ee), ok)
    H_o = fem.element_hessian_psd(x, m.tets[ok], m.Bm[ok], m.V[ok], m.mu[ok], m.lam[ok])
    assert per_element_rel(He[ok], H_o) < 1e-10


@pytest.mark.parametrize("name,amp", [("drop", 0.08), ("c1", 0.3)])
def test_element_hessian_fallback_parity(msim, name, amp):
    """The cyclic-Jacobi fall-back of the PSD projection (k_elem_hess_eig, taken by tets with more
    than kMaxNeg negative eigenvalues or without QL convergence) forced for every indefinite
    element (MS_DEBUG_HESS_FALLBACK) and checked against the oracle's eigen-clamp (R2)."""
    s, b = scene_and_basis(name)
    ctx = msim.context_from_scene(s, b, debug_flags=1)
    m = ip.make_model(s)
    x = perturbed(s, amp, seed=11)
    E_o = fem.element_energy(x, m.tets, m.Bm, m.V, m.mu, m.lam)
    ok = np.isfinite(E_o)
    assert ok.mean() > 0.5
    _, _, He = ctx.eval_elements(x)
    H_o = fem.element_hessian_psd(x, m.tets[ok], m.Bm[ok], m.V[ok], m.mu[ok], m.lam[ok])
    assert per_element_rel(He[ok], H_o) < 1e-10
    w = np.linalg.eigvalsh(fem.element_hessian(x, m.tets[ok], m.Bm[ok], m.V[ok], m.mu[ok], m.lam[ok]))
    neg = (w < -1e-8 * np.abs(w).max(axis=1, keepdims=True)).sum(axis=1)
    assert np.mean(neg > 0) > 0.2          # the fall-back really ran on many elements
    assert neg.max() >= 3


# ----------------------------------------------------------------------------- assembly
@pytest.mark.parametrize("name", ["c1", "drop", "c2"])
def test_assembly_spmv_parity(msim, name):
    s, b = scene_and_basis(name)
    ctx = msim.context_from_scene(s, b)
    m = ip.make_model(s)
    rng = np.random.default_rng(4)
    x = perturbed(s, 0.02, seed=5)
    xhat = s.X + 0.001 * rng.standard_normal(s.X.shape)
    ctx.set_step_state(s.X, xhat, x)
    E = ctx.assemble()
    assert abs(E - ip.energy(m, x, xhat)) <= 1e-10 * abs(ip.energy(m, x, xhat))
    g = ctx.get_gradient()
    g_o = ip.gradient(m, x, xhat)
    assert np.abs(g - g_o).max() <= 1e-10 * np.abs(g_o).max()
    rp, ci, vals = ctx.export_bsr()
    H_o = ip.hessian(m, x, xhat)
    assert np.array_equal(rp, H_o.indptr) and np.array_equal(ci, H_o.indices)
    blk = H_o.data
    err = np.abs(vals - blk).max(axis=(1, 2)) / np.maximum(np.abs(blk).max(axis=(1, 2)), 1e-300)
    assert err.max() < 1e-10
    v = rng.standard_normal(3 * s.n_verts)
    y = ctx.spmv(v)
    y_o = H_o.tocsr() @ v
    assert np.abs(y - y_o).max() <= 1e-12 * np.abs(y_o).max()


# ----------------------------------------------------------------------------- basis / coarse
@pytest.mark.parametrize("name", ["c1", "c2", "drop"])
def test_basis_coarse_parity(msim, name):
    s, b = scene_and_basis(name)
    ctx = msim.context_from_scene(s, b)
    m = ip.make_model(s)
    Us, Ua = coarse.sms_matrix(s.X, b), coarse.affine_matrix(s.X, b)
    rng = np.random.default_rng(6)
    q = rng.standard_normal(12 * b.m)
    assert rel_err(ctx.basis_apply(q), Us @ q) < 1e-13
    y = rng.standard_normal(3 * s.n_verts)
    assert rel_err(ctx.basis_apply_t(y), Us.T @ y) < 1e-13
    x = perturbed(s, 0.02, seed=7)
    xhat = s.X + 0.001 * rng.standard_normal(s.X.shape)
    ctx.set_step_state(s.X, xhat, x)
    ctx.assemble()
    H = ip.hessian(m, x, xhat).tocsr()
    S, Sa = ctx.export_coarse()
    S_o = coarse.galerkin(Us, H)
    Sa_o = coarse.galerkin(Ua, H)
    assert np.abs(S - S_o).max() <= 1e-11 * np.abs(S_o).max()
    assert np.abs(Sa - Sa_o).max() <= 1e-11 * np.abs(Sa_o).max()
    ds, da = ctx.subspace_direction()
    g = ip.gradient(m, x, xhat)
    ds_o, da_o, _, _ = solver.subspace_direction(H, g, Ua, Us)
    assert rel_err(da, da_o) < 1e-9
    assert rel_err(ds, ds_o) < 1e-8


# ----------------------------------------------------------------------------- PCG
@pytest.mark.parametrize("name,iters", [("c1", 20), ("c2", 20), ("c2", 40), ("drop", 7)])
def test_pcg_parity(msim, name, iters):
    s, b = scene_and_basis(name)
    ctx = msim.context_from_scene(s, b)
    m = ip.make_model(s)
    rng = np.random.default_rng(8)
    x = perturbed(s, 0.02, seed=9)
    xhat = s.X + 0.001 * rng.standard_normal(s.X.shape)
    ctx.set_step_state(s.X, xhat, x)
    ctx.assemble()
    H = ip.hessian(m, x, xhat).tocsr()
    rhs = rng.standard_normal(3 * s.n_verts)
    rhs.reshape(-1, 3)[~m.free] = 0.0
    sol, st = ctx.pcg_solve(rhs, iters)
    sol_o = solver.pcg(H, rhs, iters)
    assert rel_err(sol, sol_o) < 1e-8
    assert st.iters == iters


def test_pcg_zero_rhs(msim):
    s, b = scene_and_basis("c1")
    ctx = msim.context_from_scene(s, b)
    ctx.assemble()
    sol, st = ctx.pcg_solve(np.zeros(3 * s.n_verts), 20)
    assert np.all(sol == 0.0) and st.rz0 == 0.0


# ----------------------------------------------------------------------------- Newton
@pytest.mark.parametrize("name", ["c1", "drop", "c2"])
def test_newton_iteration_bootstrapped(msim, name):
    """Reading R10: the oracle is bootstrapped from the GPU state before every iteration."""
    s, b = scene_and_basis(name)
    ctx = msim.context_from_scene(s, b)
    sim = solver.OracleSim(s, b)
    for step in range(2):
        ctx.begin_step()
        for it in range(4):
            x_t, xhat, x = ctx.get_step_state()
            sim.x_t, sim.xhat, sim.x = x_t, xhat, x.copy()
            info = sim.newton_iteration()
            st = ctx.newton_step()
            ds, df = ctx.get_direction()
            assert rel_err(ds, info.ds) < 1e-8, (step, it)
            assert rel_err(ds + df, info.d) < 1e-8, (step, it)
            assert abs(st.alpha0 - info.alpha0) <= 1e-10
            if st.ls_failed or info.ls_failed:
                break
            assert abs(st.alpha - info.alpha) <= 1e-10 * info.alpha
            assert st.ls_evals == info.ls_evals
            _, _, x_new = ctx.get_step_state()
            assert np.abs(x_new - sim.x).max() <= 1e-9 * np.abs(x_new - x).max() + 1e-15
            if st.converged:
                break
        ctx.end_step()


@pytest.mark.parametrize("name,steps", [("c1", 10), ("c2", 3), ("drop_tiny", 12), ("drop", 6)])
def test_timestep_free_running(msim, name, steps):
    """Free-running timesteps (reading R10): max_v |x_gpu - x_oracle| <= 1e-6 bbox diagonal.
    C1 over its full 10 steps; C2 (heterogeneous 1e9/1e5 Pa, ~56 Newton iterations per step) over
    3 here -- its full 20-step run passed on B200 in 18.5 min of oracle time
    (profiles/r01_c2_20step_parity.log; MSIM_FULL_STEPS=1 runs it)."""
    import os
    if name == "c2" and os.environ.get("MSIM_FULL_STEPS"):
        steps = 20
    s, b = scene_and_basis(name)
    ctx = msim.context_from_scene(s, b)
    sim = solver.OracleSim(s, b)
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    for k in range(steps):
        st = ctx.timestep()
        infos = sim.timestep()
        x, v = ctx.get_state()
        assert np.abs(x - sim.x).max() <= 1e-6 * diag, (k, st.newton_iters, len(infos))
        assert np.abs(v - sim.v).max() <= 1e-6 * diag / s.h


def test_free_fall_closed_form_gpu(msim):
    s = scene_small_drop(n=(3, 3, 2), m=2, drop=1.0)
    b = build_basis(s, workers=1)
    ctx = msim.context_from_scene(s, b)
    for n in range(1, 5):
        ctx.timestep()
        x, _ = ctx.get_state()
        expect = s.X[:, 2] + s.h ** 2 * s.gravity[2] * n * (n + 1) / 2
        assert np.abs(x[:, 2] - expect).max() < 1e-10
        assert np.abs(x[:, :2] - s.X[:, :2]).max() < 1e-12


def test_determinism(msim):
    s, b = scene_and_basis("drop")
    out = []
    for _ in range(2):
        ctx = msim.context_from_scene(s, b)
        for _ in range(3):
            ctx.timestep()
        out.append(ctx.get_state()[0])
    assert np.array_equal(out[0], out[1])


def test_infeasible_state_rejected(msim):
    s, b = scene_and_basis("drop_tiny")
    ctx = msim.context_from_scene(s, b)
    x = s.X.copy()
    x[0, 2] = -0.01                     # below the ground plane
    ctx.set_state(x, np.zeros_like(x))
    with pytest.raises(msim.MsimError) as e:
        ctx.timestep()
    assert e.value.code == -7
    # the failed step is abandoned cleanly: x is back at x^t, no step is in progress, and the
    # context runs again from a feasible state
    xr, _ = ctx.get_state()
    assert np.array_equal(xr, x)
    with pytest.raises(msim.MsimError) as e:
        ctx.end_step()
    assert e.value.code == -8
    ctx.set_state(s.X, np.zeros_like(s.X))
    assert ctx.timestep().newton_iters >= 1


def test_dirichlet_after_basis_rejected(msim):
    """The basis is built for one Dirichlet set: changing it afterwards is a state error, and a
    basis that does not vanish at a Dirichlet vertex is rejected at upload."""
    s, b = scene_and_basis("c1")
    ctx = msim.context_from_scene(s, b)
    with pytest.raises(msim.MsimError) as e:
        ctx.set_dirichlet(s.dbc)
    assert e.value.code == -8
    ctx2 = msim.Context(0)
    ctx2.upload_mesh(s.X, s.tets, s.E, s.nu, s.rho)
    ctx2.set_dirichlet(np.arange(20))          # more vertices than the basis was built for
    with pytest.raises(msim.MsimError) as e:
        ctx2.basis_upload(b.m, b.origins, b.vptr, b.handle, b.phi, b.phi_affine, b.affine_origin, b.n_cg)
    assert e.value.code == -1


def test_invalid_mesh_rejected(msim):
    s, _ = scene_and_basis("c1")
    ctx = msim.Context()
    bad = s.tets.copy()
    bad[0, [2, 3]] = bad[0, [3, 2]]     # negative volume
    with pytest.raises(msim.MsimError) as e:
        ctx.upload_mesh(s.X, bad, s.E, s.nu, s.rho)
    assert e.value.code == -1
    with pytest.raises(msim.MsimError):
        ctx.upload_mesh(s.X, s.tets, s.E, np.full(s.n_tets, 0.5), s.rho)


def test_state_roundtrip_pinned(msim):
    """set_state / get_state(out=...) with pinned host buffers (the bench's e2e leg) move the
    state bit-exactly and agree with the allocating get_state."""
    import torch
    s, b = scene_and_basis("drop_tiny")
    ctx = msim.context_from_scene(s, b)
    x = perturbed(s, 0.01, 3)
    v = np.random.default_rng(4).standard_normal(x.shape)
    xp = torch.zeros(x.shape, dtype=torch.float64, pin_memory=True).numpy()
    vp = torch.zeros(x.shape, dtype=torch.float64, pin_memory=True).numpy()
    xp[...] = x
    vp[...] = v
    ctx.set_state(xp, vp)
    xo = torch.zeros(x.shape, dtype=torch.float64, pin_memory=True).numpy()
    vo = torch.zeros(x.shape, dtype=torch.float64, pin_memory=True).numpy()
    ctx.get_state(out=(xo, vo))
    assert np.array_equal(xo, x) and np.array_equal(vo, v)
    xa, va = ctx.get_state()
    assert np.array_equal(xa, xo) and np.array_equal(va, vo)
    with pytest.raises(ValueError):
        ctx.get_state(out=(xo[:-1], vo))
