"""Pins for oracle/ip.py (barrier, mass, assembled E / g / H) and the input generators."""
import json
import os

import numpy as np
import pytest

from oracle import fem, ip
from precompute.mesh import kuhn_grid, make_scene, scene_small_drop

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_kuhn_counts_golden():
    g = GOLD["kuhn_counts"]
    for c in (1, 2):
        s = make_scene(c)
        assert [s.n_verts, s.n_tets] == g[f"C{c}"]
    X, tets, _ = kuhn_grid(4, 3, 2, 0.1)
    V = np.linalg.det(X[tets[:, 1:]] - X[tets[:, :1]]) / 6
    assert np.all(V > 0) and abs(V.sum() - 4 * 3 * 2 * 0.001) < 1e-15


def test_barrier_golden_and_c2():
    g = GOLD["barrier_half_dhat"]
    dh = g["dhat"]
    assert abs(ip.barrier(dh / 2, dh) - g["expected"]) < 1e-20
    # C2 continuity at dhat and zero beyond
    for f in (ip.barrier, ip.barrier_d1, ip.barrier_d2):
        assert f(dh, dh) == 0.0 and f(2 * dh, dh) == 0.0
        assert abs(f(dh * (1 - 1e-9), dh)) < 1e-6
    d = np.linspace(1e-6, dh * 0.999, 200)
    assert np.all(ip.barrier_d2(d, dh) > 0) and np.all(ip.barrier_d1(d, dh) < 0)
    e = 1e-10
    fd1 = (ip.barrier(d + e, dh) - ip.barrier(d - e, dh)) / (2 * e)
    fd2 = (ip.barrier_d1(d + e, dh) - ip.barrier_d1(d - e, dh)) / (2 * e)
    assert np.abs(fd1 - ip.barrier_d1(d, dh)).max() < 1e-5 * np.abs(ip.barrier_d1(d, dh)).max()
    assert np.abs(fd2 - ip.barrier_d2(d, dh)).max() < 1e-5 * np.abs(ip.barrier_d2(d, dh)).max()


def test_total_mass():
    s = make_scene(2)
    m = ip.make_model(s)
    assert abs(m.mass.sum() - 1000.0 * 40 * 10 * 10 * 0.1 ** 3) < 1e-9


def test_rest_state_no_gravity_zero_energy_and_gradient(c1_scene):
    m = ip.make_model(c1_scene)
    x = m.X.copy()
    assert ip.energy(m, x, x) == 0.0
    assert np.abs(ip.gradient(m, x, x)).max() < 1e-12


def small_model(amp=0.002, seed=0):
    s = scene_small_drop(n=(3, 2, 2), drop=0.0008)
    m = ip.make_model(s)
    rng = np.random.default_rng(seed)
    x = m.X + amp * rng.standard_normal(m.X.shape) * np.array([1.0, 1.0, 0.05])
    xhat = m.X + 0.001 * rng.standard_normal(m.X.shape)
    return s, m, x, xhat


def test_full_gradient_fd_with_barrier():
    s, m, x, xhat = small_model()
    d, _ = ip.ground_distance(m, x)
    assert np.any(d < m.ground["dhat"]) and np.all(d > 0)     # barrier active
    g = ip.gradient(m, x, xhat)
    rng = np.random.default_rng(1)
    for _ in range(5):
        v = rng.standard_normal(x.shape)
        e = 1e-8
        fd = (ip.energy(m, x + e * v, xhat) - ip.energy(m, x - e * v, xhat)) / (2 * e)
        assert abs(fd - np.sum(g * v)) < 1e-6 * np.abs(g).sum() * np.abs(v).max()


def test_energy_difference_matches_energy():
    s, m, x, xhat = small_model()
    d = 1e-4 * np.random.default_rng(3).standard_normal(x.shape)
    for a in (1.0, 0.5, 0.125):
        de = ip.energy_difference(m, x, d, a, xhat)
        ref = ip.energy(m, x + a * d, xhat) - ip.energy(m, x, xhat)
        assert abs(de - ref) < 1e-9 * max(abs(ref), 1e-12) + 1e-14 * ip.energy(m, x, xhat)


def test_hessian_matrix_free_and_fd():
    """H v == M v + h^2 (sum_e P+(H_e) v_e + kappa b'' n n^T v) evaluated element by element,
    and H == FD Hessian when no projection is active (pure small stretch, no barrier)."""
    s, m, x, xhat = small_model()
    H = ip.hessian(m, x, xhat).tocsr()
    rng = np.random.default_rng(2)
    v = rng.standard_normal(x.shape)
    He = fem.element_hessian_psd(x, m.tets, m.Bm, m.V, m.mu, m.lam)
    ve = v[m.tets].reshape(-1, 12)
    y = np.zeros_like(v)
    Hv_e = np.einsum("eij,ej->ei", He, ve)
    for a in range(4):
        np.add.at(y, m.tets[:, a], Hv_e[:, 3 * a:3 * a + 3])
    y *= m.h ** 2
    y += m.mass[:, None] * v
    d, n = ip.ground_distance(m, x)
    y += (m.h ** 2 * m.ground["kappa"] * ip.barrier_d2(d, m.ground["dhat"]) * (v @ n))[:, None] * n
    assert np.abs(H @ v.ravel() - y.ravel()).max() < 1e-12 * np.abs(y).max()

    # no projection needed: homogeneous stretch of the beam, no ground
    c1 = make_scene(1)
    m1 = ip.make_model(c1)
    m1.free[:] = True
    x1 = m1.X * np.array([1.01, 1.0, 1.0])
    H1 = ip.hessian(m1, x1, x1).toarray()
    He1 = fem.element_hessian(x1, m1.tets, m1.Bm, m1.V, m1.mu, m1.lam)
    assert min(np.linalg.eigvalsh(He1).min(axis=1)) > -1e-9 * np.abs(He1).max()
    e = 1e-7
    cols = rng.choice(3 * m1.n, 12, replace=False)
    for k in cols:
        xp, xm = x1.copy(), x1.copy()
        xp.flat[k] += e
        xm.flat[k] -= e
        fd = (ip.gradient(m1, xp, x1) - ip.gradient(m1, xm, x1)).ravel() / (2 * e)
        assert np.abs(fd - H1[:, k]).max() < 1e-5 * np.abs(H1).max()


def test_hessian_dbc_identity(c1_scene):
    m = ip.make_model(c1_scene)
    H = ip.hessian(m, m.X, m.X).toarray()
    for v in c1_scene.dbc:
        rows = H[3 * v:3 * v + 3]
        assert np.array_equal(rows[:, 3 * v:3 * v + 3], np.eye(3))
        assert np.count_nonzero(rows) == 3
        assert np.count_nonzero(H[:, 3 * v:3 * v + 3]) == 3
    assert np.abs(H - H.T).max() < 1e-12 * np.abs(H).max()
