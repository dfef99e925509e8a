"""Pins of the oracle's paper-faithful coarse mode (NEXT-1; §3.7.1, Alg. 2
L427-450): block-Jacobi PCG to a relative residual on the matrix-free sandwich U^T (H (U p)).

* with the tolerance 0 and enough iterations it reaches the exact (Cholesky) subspace direction;
* on a block-diagonal matrix the block-Jacobi preconditioner is exact: one iteration;
* at a fixed iteration count k it returns the minimiser of the S-norm error over the
  block-preconditioned Krylov space (formed here by a direct Galerkin solve, not the recurrence);
* the stopping rule: the returned count k is the first with ||r_k|| <= tol ||b||;
* the affine stage (one 12 x 12 block = S_a itself) converges in one iteration.
"""
import numpy as np
import scipy.sparse as sp

from oracle import coarse, ip, solver


def _c1(c1_scene):
    m = ip.make_model(c1_scene)
    rng = np.random.default_rng(31)
    x = m.X + 0.01 * rng.standard_normal(m.X.shape)
    x[~m.free] = m.X[~m.free]
    xhat = m.X + 0.002 * rng.standard_normal(m.X.shape)
    return m, x, xhat


def test_pcg_mode_reaches_exact_direction(c1_scene, c1_basis):
    m, x, xhat = _c1(c1_scene)
    H = ip.hessian(m, x, xhat).tocsr()
    g = ip.gradient(m, x, xhat)
    Ua, Us = coarse.affine_matrix(m.X, c1_basis), coarse.sms_matrix(m.X, c1_basis)
    ds_e, da_e, _, _ = solver.subspace_direction(H, g, Ua, Us)
    ds_p, da_p, ita, its = solver.subspace_direction(H, g, Ua, Us, "pcg", tol=0.0, max_iter=400)
    assert np.linalg.norm(da_p - da_e) <= 1e-12 * np.linalg.norm(da_e)
    assert np.linalg.norm(ds_p - ds_e) <= 1e-9 * np.linalg.norm(ds_e)
    # the default paper tolerance 1e-4 stops much earlier and is close, not equal
    ds_t, _, _, its_t = solver.subspace_direction(H, g, Ua, Us, "pcg", tol=1e-4)
    assert 0 < its_t < its
    assert np.linalg.norm(ds_t - ds_e) <= 1e-2 * np.linalg.norm(ds_e)


def test_affine_stage_one_iteration(c1_scene, c1_basis):
    """One 12 x 12 block: the block-Jacobi preconditioner is S_a^-1, so PCG ends after one step."""
    m, x, xhat = _c1(c1_scene)
    H = ip.hessian(m, x, xhat).tocsr()
    g = ip.gradient(m, x, xhat)
    Ua = coarse.affine_matrix(m.X, c1_basis)
    Sa = coarse.galerkin(Ua, H)
    b = Ua.T @ (-g.ravel())
    q, it, rel = solver.block_jacobi_pcg(lambda p: Ua.T @ (H @ (Ua @ p)), b,
                                         solver.galerkin_diagonal_blocks(Ua, H), 1e-12, 50)
    assert it == 1 and rel < 1e-12
    assert np.linalg.norm(q - np.linalg.solve(Sa, b)) <= 1e-12 * np.linalg.norm(q)


def _spd(rng, n):
    A = rng.standard_normal((n, n))
    return A @ A.T + n * np.diag(rng.uniform(1.0, 10.0, n))


def test_block_diagonal_is_one_iteration():
    rng = np.random.default_rng(32)
    blocks = np.array([_spd(rng, 12) for _ in range(5)])
    S = sp.block_diag(blocks).toarray()
    b = rng.standard_normal(60)
    q, it, rel = solver.block_jacobi_pcg(lambda p: S @ p, b, blocks, 1e-14, 10)
    assert it == 1
    assert np.linalg.norm(q - np.linalg.solve(S, b)) <= 1e-12 * np.linalg.norm(q)


def test_fixed_count_krylov_optimality_block_jacobi():
    rng = np.random.default_rng(33)
    n = 48
    S = _spd(rng, n)
    blocks = np.array([S[12 * i:12 * i + 12, 12 * i:12 * i + 12] for i in range(4)])
    Minv = np.zeros((n, n))
    for i in range(4):
        Minv[12 * i:12 * i + 12, 12 * i:12 * i + 12] = np.linalg.inv(blocks[i])
    b = rng.standard_normal(n)
    for k in (1, 2, 4, 7):
        K = [Minv @ b]
        for _ in range(k - 1):
            K.append(Minv @ (S @ K[-1]))
        V, _ = np.linalg.qr(np.array(K).T)
        ref = V @ np.linalg.solve(V.T @ S @ V, V.T @ b)
        q, it, _ = solver.block_jacobi_pcg(lambda p: S @ p, b, blocks, 0.0, k)
        assert it == k
        assert np.linalg.norm(q - ref) <= 1e-9 * np.linalg.norm(ref), k


def test_stopping_rule_first_crossing():
    rng = np.random.default_rng(34)
    S = _spd(rng, 60)
    blocks = np.array([S[12 * i:12 * i + 12, 12 * i:12 * i + 12] for i in range(5)])
    b = rng.standard_normal(60)
    tol = 1e-4
    q, it, rel = solver.block_jacobi_pcg(lambda p: S @ p, b, blocks, tol, 1000)
    assert rel <= tol
    assert np.linalg.norm(b - S @ q) <= 1.0001 * tol * np.linalg.norm(b)
    _, _, rel_prev = solver.block_jacobi_pcg(lambda p: S @ p, b, blocks, 0.0, it - 1)
    assert rel_prev > tol
