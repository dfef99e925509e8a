"""Pins for oracle/coarse.py and oracle/solver.py: Galerkin products vs brute force, coarse
solves vs LAPACK, the Galerkin orthogonality of the SMS stage, PCG vs direct solves, line-search
filters vs SPEC's worked examples, free fall closed form, energy monotonicity."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import coarse, ip, solver
from precompute.basis import build_basis
from precompute.mesh import make_scene, scene_small_drop

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def perturbed_c1(c1_scene, amp=0.01, seed=0):
    m = ip.make_model(c1_scene)
    rng = np.random.default_rng(seed)
    x = m.X + amp * rng.standard_normal(m.X.shape)
    x[c1_scene.dbc] = m.X[c1_scene.dbc]
    xhat = m.X + 0.001 * rng.standard_normal(m.X.shape)
    return m, x, xhat


def test_galerkin_vs_dense_bruteforce(c1_scene, c1_basis):
    m, x, xhat = perturbed_c1(c1_scene)
    H = ip.hessian(m, x, xhat)
    Us = coarse.sms_matrix(m.X, c1_basis)
    S = coarse.galerkin(Us, H)
    Hd, Ud = H.toarray(), Us.toarray()
    Sd = np.zeros((Ud.shape[1], Ud.shape[1]))
    for i in range(Ud.shape[1]):             # brute force: columns one at a time
        Sd[:, i] = Ud.T @ (Hd @ Ud[:, i])
    assert np.abs(S - Sd).max() < 1e-12 * np.abs(Sd).max()
    assert np.abs(S - S.T).max() < 1e-12 * np.abs(S).max()


def test_cholesky_solve_vs_lapack(c1_scene, c1_basis):
    m, x, xhat = perturbed_c1(c1_scene)
    H = ip.hessian(m, x, xhat)
    S = coarse.galerkin(coarse.sms_matrix(m.X, c1_basis), H)
    b = np.random.default_rng(1).standard_normal(len(S))
    q = coarse.cho_solve(coarse.cholesky(S), b)
    ref = sla.solve(S, b, assume_a="pos")
    assert np.abs(q - ref).max() < 1e-9 * np.abs(ref).max()
    assert np.abs(S @ q - b).max() < 1e-9 * np.abs(b).max()


def test_sms_galerkin_orthogonality_and_two_stage(c1_scene, c1_basis):
    """After the SMS stage B^T(-g - H d_s) = 0; the two-stage (affine then SMS) direction
    equals the one-shot Galerkin solve on U_s because span(U_a) is inside span(U_s)."""
    m, x, xhat = perturbed_c1(c1_scene)
    H = ip.hessian(m, x, xhat).tocsr()
    g = ip.gradient(m, x, xhat)
    Us, Ua = coarse.sms_matrix(m.X, c1_basis), coarse.affine_matrix(m.X, c1_basis)
    ds, da, Sa, S = solver.subspace_direction(H, g, Ua, Us)
    r = -g.ravel() - H @ ds
    assert np.abs(Us.T @ r).max() < 1e-10 * np.abs(Us.T @ g.ravel()).max()
    one_shot = Us @ np.linalg.solve(S, Us.T @ (-g.ravel()))
    assert np.abs(one_shot - ds).max() < 1e-9 * np.abs(ds).max()
    # the affine stage alone is the Galerkin solve on U_a
    assert np.abs(Ua.T @ (-g.ravel() - H @ da)).max() < 1e-10 * np.abs(Ua.T @ g.ravel()).max()


def test_zero_gradient_zero_direction(c1_scene, c1_basis):
    m = ip.make_model(c1_scene)
    H = ip.hessian(m, m.X, m.X).tocsr()
    g = np.zeros_like(m.X)
    ds, *_ = solver.subspace_direction(H, g, coarse.affine_matrix(m.X, c1_basis),
                                       coarse.sms_matrix(m.X, c1_basis))
    assert np.all(ds == 0)
    assert np.all(solver.pcg(H, np.zeros(3 * m.n), 20) == 0)


def test_pcg_exact_on_tiny_spd():
    rng = np.random.default_rng(3)
    import scipy.sparse as sp
    for n in (5, 9, 12):
        A = rng.standard_normal((n, n))
        H = sp.csr_matrix(A @ A.T + n * np.eye(n))
        b = rng.standard_normal(n)
        d = solver.pcg(H, b, n)
        ref = np.linalg.solve(H.toarray(), b)
        assert np.abs(d - ref).max() < 1e-10 * np.abs(ref).max()


def test_pcg_jacobi_one_iteration_exact_on_diagonal():
    """Fixed-count pin of the Jacobi preconditioner: on a diagonal H one PCG iteration with
    z = D^-1 r is the exact solution; with D instead of D^-1, or without preconditioning, it is
    not (the diagonal entries differ)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(5)
    diag = rng.uniform(0.5, 50.0, 40)
    H = sp.diags(diag).tocsr()
    b = rng.standard_normal(40)
    d = solver.pcg(H, b, 1)
    assert np.abs(d - b / diag).max() < 1e-13 * np.abs(b / diag).max()


def test_pcg_fixed_count_krylov_optimality():
    """CG optimality (Hestenes-Stiefel): after k iterations from 0, Jacobi-PCG returns the
    minimiser of the H-norm error over the preconditioned Krylov space
    K_k = span{z, (D^-1 H) z, ..., (D^-1 H)^{k-1} z}, z = D^-1 b.  The minimiser is formed here by
    a direct Galerkin solve on that space, independently of the recurrence."""
    import scipy.sparse as sp
    rng = np.random.default_rng(6)
    n = 30
    A = rng.standard_normal((n, n))
    Hd = A @ A.T + np.diag(rng.uniform(1.0, 100.0, n))
    H = sp.csr_matrix(Hd)
    b = rng.standard_normal(n)
    Dinv = 1.0 / np.diag(Hd)
    for k in (1, 2, 3, 5):
        K = [Dinv * b]
        for _ in range(k - 1):
            K.append(Dinv * (Hd @ K[-1]))
        V, _ = np.linalg.qr(np.array(K).T)
        ref = V @ np.linalg.solve(V.T @ Hd @ V, V.T @ b)
        d = solver.pcg(H, b, k)
        assert np.linalg.norm(d - ref) < 1e-9 * np.linalg.norm(ref), k


def _two_level_problem(n=36, nc=6, seed=16):
    """SPD H, a sparse coarse basis U and a right-hand side with U^T b = 0 (the refinement's
    residual after the SMS stage is Galerkin-orthogonal to the coarse space)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    Hd = A @ A.T + np.diag(rng.uniform(1.0, 100.0, n))
    U = rng.standard_normal((n, nc))
    U[rng.uniform(size=(n, nc)) < 0.5] = 0.0
    b = rng.standard_normal(n)
    b -= U @ np.linalg.solve(U.T @ U, U.T @ b)
    return Hd, sp.csr_matrix(Hd), sp.csr_matrix(U), U, b


def test_two_level_pcg_krylov_optimality():
    """NEXT-4: on U^T b = 0 the two-level PCG iterate after k steps minimises the H-norm error over
    K_k(P H, P b) with the symmetric balancing preconditioner
    P = Q + (I - Q H) D^-1 (I - H Q), Q = U (U^T H U)^-1 U^T, formed densely with an explicit
    inverse -- a Galerkin solve on that space, independent of the recurrence and of the oracle's
    triangular solves.  Dropping the coarse term, using S instead of S^-1 or correcting v instead
    of v - H D^-1 v changes the space."""
    Hd, H, Us, U, b = _two_level_problem()
    n = len(b)
    Q = U @ np.linalg.inv(U.T @ Hd @ U) @ U.T
    Dm = np.diag(1.0 / np.diag(Hd))
    P = Q + (np.eye(n) - Q @ Hd) @ Dm @ (np.eye(n) - Hd @ Q)
    L = coarse.cholesky(coarse.galerkin(Us, H))
    for k in (1, 2, 3, 5):
        K = [P @ b]
        for _ in range(k - 1):
            K.append(P @ (Hd @ K[-1]))
        V, _ = np.linalg.qr(np.array(K).T)
        ref = V @ np.linalg.solve(V.T @ Hd @ V, V.T @ b)
        d, it = solver.two_level_pcg(H, b, Us, L, 0.0, 1.0, k)
        assert it == k
        assert np.linalg.norm(d - ref) < 1e-9 * np.linalg.norm(ref), k


def test_two_level_pcg_stopping_rule_and_limits():
    """Stops at the FIRST k with ||b - H d_k|| <= tol ref (checked against the iterates of the
    fixed-count runs); tol 1 with ref = ||b|| stops at 0 iterations; at a tight tolerance the
    iterate is the LAPACK solution."""
    Hd, H, Us, U, b = _two_level_problem()
    L = coarse.cholesky(coarse.galerkin(Us, H))
    ref_norm = np.linalg.norm(b)
    tol = 1e-6
    d, it = solver.two_level_pcg(H, b, Us, L, tol, ref_norm, 500)
    assert np.linalg.norm(b - Hd @ d) <= tol * ref_norm
    d_prev, it_prev = solver.two_level_pcg(H, b, Us, L, 0.0, 1.0, it - 1)
    assert it_prev == it - 1 and np.linalg.norm(b - Hd @ d_prev) > tol * ref_norm
    assert solver.two_level_pcg(H, b, Us, L, 1.0, ref_norm, 500)[1] == 0
    d, _ = solver.two_level_pcg(H, b, Us, L, 1e-14, ref_norm, 500)
    ref = sla.solve(Hd, b, assume_a="pos")
    assert np.linalg.norm(d - ref) < 1e-10 * np.linalg.norm(ref)


def test_two_level_pcg_empty_coarse_space_is_jacobi():
    """With no coarse columns the preconditioner reduces to Jacobi: the iterates are those of the
    (pinned) fixed-count Jacobi-PCG."""
    import scipy.sparse as sp
    Hd, H, _, _, b = _two_level_problem()
    U0 = sp.csr_matrix((len(b), 0))
    for k in (1, 4):
        d, _ = solver.two_level_pcg(H, b, U0, np.zeros((0, 0)), 0.0, 1.0, k)
        assert np.linalg.norm(d - solver.pcg(H, b, k)) < 1e-12 * np.linalg.norm(d)


def test_pcg_converges_to_lapack_on_c1(c1_scene):
    m, x, xhat = perturbed_c1(c1_scene)
    H = ip.hessian(m, x, xhat).tocsr()
    b = np.random.default_rng(4).standard_normal(3 * m.n)
    d = solver.pcg(H, b, 3000)
    ref = sla.solve(H.toarray(), b, assume_a="pos")
    assert np.linalg.norm(d - ref) < 1e-8 * np.linalg.norm(ref)


class _GroundModel:
    def __init__(self, x):
        self.ground = dict(normal=(0.0, 0.0, 1.0), offset=0.0, dhat=1e-3, kappa=1.0)
        self.free = np.ones(len(x), dtype=bool)


def test_ccd_golden():
    g = GOLD["ccd_impact_half"]
    x = np.array([[0.0, 0.0, g["height"]]])
    d = np.array([[0.0, 0.0, g["velocity"]]])
    assert abs(solver.ccd_alpha(_GroundModel(x), x, d) - g["expected_alpha"]) < 1e-15
    d = np.array([[1.0, 0.5, 0.0]])
    assert solver.ccd_alpha(_GroundModel(x), x, d) == GOLD["ccd_parallel"]["expected_alpha"]


class _TetModel:
    def __init__(self):
        self.tets = np.array([[0, 1, 2, 3]])


def test_inversion_golden():
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float)
    m = _TetModel()
    g = GOLD["inversion_collapse"]
    # vertex 3 moves to the plane z = 0 at alpha = collapse_at: det is linear in alpha
    d = np.zeros_like(X)
    d[3, 2] = -1.0 / g["collapse_at"]
    assert abs(solver.inversion_alpha(m, X, d) - g["expected_alpha"]) < 1e-12
    assert solver.inversion_alpha(m, X, np.zeros_like(X)) == GOLD["inversion_zero_direction"]["expected_alpha"]
    assert solver.inversion_alpha(m, X, np.tile([0.3, -2.0, 5.0], (4, 1))) == 1.0


def test_det_poly_bruteforce():
    rng = np.random.default_rng(5)
    A = rng.standard_normal((20, 3, 3))
    B = rng.standard_normal((20, 3, 3))
    c = solver.det_poly(A, B)
    for t in (-1.3, 0.0, 0.4, 2.5):
        ref = np.linalg.det(A + t * B)
        val = c[0] + c[1] * t + c[2] * t ** 2 + c[3] * t ** 3
        assert np.abs(val - ref).max() < 1e-12 * (1 + np.abs(ref).max())
    # smallest positive root is a root and no sign change occurs before it
    r = solver.smallest_positive_root(c)
    for k in range(20):
        if np.isfinite(r[k]):
            assert abs(np.linalg.det(A[k] + r[k] * B[k])) < 1e-9 * (1 + np.abs(c[0][k]))
            ts = np.linspace(0, r[k], 50)[:-1]
            vals = [np.linalg.det(A[k] + t * B[k]) for t in ts]
            assert np.all(np.sign(vals) == np.sign(vals[0]))


def test_free_fall_closed_form():
    """No DBC, no contact within the horizon: IE gives x_n = x_0 + h^2 g n(n+1)/2 exactly,
    since Psi = 0 for rigid translations and the coarse space contains translations."""
    s = scene_small_drop(n=(3, 3, 2), m=2, drop=1.0)
    b = build_basis(s, workers=1)
    sim = solver.OracleSim(s, b)
    h, gz = s.h, s.gravity[2]
    for n in range(1, 5):
        infos = sim.timestep()
        expect = s.X[:, 2] + h * h * gz * n * (n + 1) / 2
        assert np.abs(sim.x[:, 2] - expect).max() < 1e-10
        assert np.abs(sim.x[:, :2] - s.X[:, :2]).max() < 1e-12
        assert infos[0].alpha == 1.0 and infos[-1].converged


def test_rest_without_gravity_one_iteration(c1_scene, c1_basis):
    import dataclasses
    s = dataclasses.replace(c1_scene, gravity=(0.0, 0.0, 0.0))
    sim = solver.OracleSim(s, c1_basis)
    infos = sim.timestep()
    assert len(infos) == 1 and infos[0].converged and infos[0].ds_norm < 1e-14
    assert np.abs(sim.x - s.X).max() < 1e-15


def test_energy_monotone_contact_steps():
    s = scene_small_drop(n=(4, 3, 2), m=3, drop=0.003)
    b = build_basis(s, workers=1)
    sim = solver.OracleSim(s, b)
    for step in range(6):
        sim.begin_step()
        e_prev = ip.energy(sim.model, sim.x, sim.xhat)
        for _ in range(30):
            info = sim.newton_iteration()
            if not info.ls_failed:
                assert info.energy < e_prev
                e_prev = info.energy
            d, _ = ip.ground_distance(sim.model, sim.x)
            assert d.min() > 0
            if info.converged or info.ls_failed:
                break
        sim.end_step()
    assert sim.x[:, 2].min() < 1e-3      # contact engaged
