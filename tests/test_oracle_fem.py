"""Pins for oracle/fem.py (element energy, gradient, Hessian, PSD projection).

Each test ties the oracle to something other than itself: textbook linear elasticity,
finite differences, invariances, algebraic identities of the PSD projector, or an
independent eigen-solver written here (cyclic Jacobi)."""
import json
import os

import numpy as np
import pytest

from oracle import fem

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def one_tet(rng=None, amp=0.0):
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float) * 0.1
    if rng is not None:
        X = X + 0.02 * rng.standard_normal(X.shape)
    tets = np.array([[0, 1, 2, 3]])
    _, Bm, V = fem.rest_data(X, tets)
    if V[0] < 0:
        tets = np.array([[0, 1, 3, 2]])
        _, Bm, V = fem.rest_data(X, tets)
    return X, tets, Bm, V


def random_rotation(rng):
    Q, R = np.linalg.qr(rng.standard_normal((3, 3)))
    Q = Q * np.sign(np.diag(R))
    if np.linalg.det(Q) < 0:
        Q[:, 0] *= -1
    return Q


def test_lame_golden():
    g = GOLD["lame_textbook"]
    mu, lam = fem.lame(g["E"], g["nu"])
    assert abs(mu - g["mu"]) < 1e-9 * g["mu"] and abs(lam - g["lam"]) < 1e-9 * g["lam"]


def test_rest_stable():
    mu, lam = np.array([3.0]), np.array([7.0])
    F = np.eye(3)[None]
    assert abs(fem.psi(F, mu, lam)[0]) < 1e-15
    assert np.abs(fem.first_piola(F, mu, lam)).max() < 1e-14


def test_inverted_is_infinite():
    F = np.diag([-1.0, 1.0, 1.0])[None]
    assert np.isinf(fem.psi(F, np.array([1.0]), np.array([1.0]))[0])


@pytest.mark.parametrize("E,nu", [(1e6, 0.45), (1e5, 0.4), (2e9, 0.3)])
def test_linearisation(E, nu):
    """Small strain limit of the rest-stable form R1 (no Lame re-parameterisation):
    P(I + eps) = 2 mu sym(eps) + (lam - mu) tr(eps) I + O(eps^2).  Checked on a shear,
    a dilation and a random strain."""
    mu, lam = fem.lame(E, nu)
    mu_, lam_ = np.array([mu]), np.array([lam])
    rng = np.random.default_rng(11)
    e = 1e-7
    for eps in [np.outer([1, 0, 0], [0, 1, 0]), np.eye(3), rng.standard_normal((3, 3))]:
        F = (np.eye(3) + e * eps)[None]
        P = fem.first_piola(F, mu_, lam_)[0]
        lin = 2 * mu * e * 0.5 * (eps + eps.T) + (lam - mu) * e * np.trace(eps) * np.eye(3)
        assert np.abs(P - lin).max() < 1e-5 * np.abs(lin).max()


def test_rotation_invariance_and_frame_indifference():
    rng = np.random.default_rng(0)
    mu, lam = np.array([1.3]), np.array([4.1])
    for _ in range(20):
        F = np.eye(3) + 0.3 * rng.standard_normal((3, 3))
        if np.linalg.det(F) <= 0:
            continue
        R = random_rotation(rng)
        a = fem.psi(F[None], mu, lam)[0]
        b = fem.psi((R @ F)[None], mu, lam)[0]
        assert abs(a - b) < 1e-12 * max(1, abs(a))


def test_gradient_fd():
    rng = np.random.default_rng(1)
    for trial in range(5):
        X, tets, Bm, V = one_tet(rng)
        mu, lam = np.array([2e5]), np.array([7e5])
        x = X + 0.01 * rng.standard_normal(X.shape)
        g = fem.element_gradient(x, tets, Bm, V, mu, lam)[0]
        h = 1e-7
        fd = np.zeros(12)
        for k in range(12):
            xp, xm = x.copy(), x.copy()
            xp.flat[k] += h
            xm.flat[k] -= h
            fd[k] = (fem.element_energy(xp, tets, Bm, V, mu, lam)[0] -
                     fem.element_energy(xm, tets, Bm, V, mu, lam)[0]) / (2 * h)
        assert np.abs(fd - g).max() < 1e-6 * np.abs(g).max()


def test_hessian_fd_and_symmetry():
    rng = np.random.default_rng(2)
    for trial in range(5):
        X, tets, Bm, V = one_tet(rng)
        mu, lam = np.array([2e5]), np.array([7e5])
        x = X + 0.01 * rng.standard_normal(X.shape)
        H = fem.element_hessian(x, tets, Bm, V, mu, lam)[0]
        assert np.abs(H - H.T).max() < 1e-12 * np.abs(H).max()
        h = 1e-7
        fd = np.zeros((12, 12))
        for k in range(12):
            xp, xm = x.copy(), x.copy()
            xp.flat[k] += h
            xm.flat[k] -= h
            fd[:, k] = (fem.element_gradient(xp, tets, Bm, V, mu, lam)[0] -
                        fem.element_gradient(xm, tets, Bm, V, mu, lam)[0]) / (2 * h)
        assert np.abs(fd - H).max() < 1e-6 * np.abs(H).max()


def test_translation_null_space_and_rigid_invariance():
    rng = np.random.default_rng(3)
    X, tets, Bm, V = one_tet(rng)
    mu, lam = np.array([2e5]), np.array([7e5])
    x = X + 0.01 * rng.standard_normal(X.shape)
    H = fem.element_hessian(x, tets, Bm, V, mu, lam)[0]
    for t in np.eye(3):
        assert np.abs(H @ np.tile(t, 4)).max() < 1e-10 * np.abs(H).max()
    R = random_rotation(rng)
    e0 = fem.element_energy(x, tets, Bm, V, mu, lam)[0]
    e1 = fem.element_energy(x @ R.T + 0.3, tets, Bm, V, mu, lam)[0]
    assert abs(e0 - e1) < 1e-10 * abs(e0)


def jacobi_eig(A, tol=1e-15):
    """Independent textbook cyclic Jacobi eigen-solver (test-only)."""
    A = A.copy()
    n = len(A)
    Q = np.eye(n)
    for _ in range(50):
        off = np.sqrt(np.sum((A - np.diag(np.diag(A))) ** 2))
        if off <= tol * np.linalg.norm(A):
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                if abs(A[p, q]) <= 1e-300:
                    continue
                th = (A[q, q] - A[p, p]) / (2 * A[p, q])
                if abs(th) > 1e100:
                    t = 0.5 / th
                else:
                    t = np.sign(th) / (abs(th) + np.sqrt(th * th + 1)) if th != 0 else 1.0
                c = 1 / np.sqrt(t * t + 1)
                s = t * c
                J = np.eye(n)
                J[p, p] = J[q, q] = c
                J[p, q] = s
                J[q, p] = -s
                A = J.T @ A @ J
                Q = Q @ J
    return np.diag(A), Q


def test_psd_projection_algebra():
    rng = np.random.default_rng(4)
    for _ in range(10):
        M = rng.standard_normal((12, 12))
        H = M + M.T
        P = fem.psd_project(H)
        N = fem.psd_project(-H)
        nrm = np.abs(H).max()
        assert np.linalg.eigvalsh(P).min() > -1e-12 * nrm
        assert np.abs(P - N - H).max() < 1e-12 * nrm               # H = H+ - H-
        assert np.abs(P @ N).max() < 1e-11 * nrm ** 2              # complementary parts
        assert np.abs(fem.psd_project(P) - P).max() < 1e-12 * nrm   # idempotent
        # nearest PSD in Frobenius norm beats random PSD candidates
        for _ in range(5):
            Y = P + 0.1 * (lambda B: B @ B.T)(rng.standard_normal((12, 3)))
            assert np.linalg.norm(H - P) <= np.linalg.norm(H - Y) + 1e-12
        w, Q = jacobi_eig(H)
        Pj = Q @ np.diag(np.maximum(w, 0)) @ Q.T
        assert np.abs(Pj - P).max() < 1e-11 * nrm


def test_psd_element_reduction_equivalence():
    """12x12 clamp == Q P+(Q^T H Q) Q^T with Q an orthonormal basis of the translation
    complement (exact because H annihilates translations) -- the reading R2 the CUDA
    kernel relies on."""
    rng = np.random.default_rng(5)
    Q4 = 0.5 * np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=float)
    assert np.allclose(Q4.T @ Q4, np.eye(3)) and np.allclose(Q4.T @ np.ones(4), 0)
    Q = np.kron(Q4, np.eye(3))
    for _ in range(10):
        X, tets, Bm, V = one_tet(rng)
        mu, lam = np.array([2e5]), np.array([7e5])
        x = X + 0.03 * rng.standard_normal(X.shape)
        H = fem.element_hessian(x, tets, Bm, V, mu, lam)[0]
        P12 = fem.psd_project(H)
        P9 = Q @ fem.psd_project(Q.T @ H @ Q) @ Q.T
        assert np.abs(P12 - P9).max() < 1e-10 * np.abs(H).max()


def test_psd_identity_on_psd_input():
    rng = np.random.default_rng(6)
    B = rng.standard_normal((12, 7))
    H = B @ B.T
    assert np.abs(fem.psd_project(H) - H).max() < 1e-12 * np.abs(H).max()
