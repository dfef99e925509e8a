"""Pins for the basis input generator (precompute/basis.py) and the oracle's explicit U_s / U_a
(oracle/coarse.py): partition of unity, linear precision, DBC compatibility, compact support
(PAPER.md L349-354, L377-381)."""
import json
import os

import numpy as np
import pytest

from oracle import coarse
from precompute.basis import build_basis
from precompute.mesh import make_scene

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.fixture(scope="module")
def c2():
    s = make_scene(2)
    return s, build_basis(s, workers=4)


def _pou(s, b):
    cnt = np.diff(b.vptr)
    return np.bincount(np.repeat(np.arange(s.n_verts), cnt), weights=b.phi, minlength=s.n_verts) + b.phi_dbc


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_pou_support_dbc(which, c1_scene, c1_basis, c2):
    s, b = (c1_scene, c1_basis) if which == "c1" else c2
    assert np.abs(_pou(s, b) - 1).max() < 1e-12
    assert np.all(b.phi > 0) and np.all(b.phi <= 1 + 1e-15)
    # DBC vertices: no SMS weight at all, phi_DBC = 1, affine weight 0
    cnt = np.diff(b.vptr)
    assert np.all(cnt[s.dbc] == 0)
    assert np.all(b.phi_dbc[s.dbc] == 1.0) and np.all(b.phi_affine[s.dbc] == 0.0)
    # compact support: handle i only on vertices of its subdomain (cluster + vertex-neighbours)
    vt = [set() for _ in range(s.n_verts)]
    for e, t in enumerate(s.tets):
        for v in t:
            vt[v].add(int(b.cluster[e]))
    clusters_of_vertex = vt
    nb = [set() for _ in range(b.m)]
    for cl in clusters_of_vertex:
        for i in cl:
            nb[i] |= cl
    rows = np.repeat(np.arange(s.n_verts), cnt)
    for v, i in zip(rows[:2000], b.handle[:2000]):
        assert clusters_of_vertex[v] & nb[i]


@pytest.mark.parametrize("which", ["c1", "c2"])
def test_linear_precision(which, c1_scene, c1_basis, c2):
    """B q_aff = (1 - phi_DBC)(A X + t) when every handle encodes the same affine map relative
    to its origin c_i: q_i rows = [A c_i + t, A] (SURVEY §8(c) pins, B rows)."""
    s, b = (c1_scene, c1_basis) if which == "c1" else c2
    Us = coarse.sms_matrix(s.X, b)
    Ua = coarse.affine_matrix(s.X, b)
    rng = np.random.default_rng(0)
    for _ in range(5):
        A = rng.standard_normal((3, 3))
        t = rng.standard_normal(3)
        field = s.X @ A.T + t
        q = np.zeros((b.m, 3, 4))
        q[:, :, 0] = b.origins @ A.T + t
        q[:, :, 1:] = A[None]
        w = (Us @ q.reshape(-1)).reshape(-1, 3)
        ref = (1 - b.phi_dbc)[:, None] * field
        assert np.abs(w - ref).max() < 1e-10 * np.abs(field).max()
        qa = np.zeros((3, 4))
        qa[:, 0] = b.affine_origin @ A.T + t
        qa[:, 1:] = A
        wa = (Ua @ qa.reshape(-1)).reshape(-1, 3)
        assert np.abs(wa - b.phi_affine[:, None] * field).max() < 1e-10 * np.abs(field).max()


def test_full_column_rank(c1_scene, c1_basis):
    Us = coarse.sms_matrix(c1_scene.X, c1_basis).toarray()
    sv = np.linalg.svd(Us, compute_uv=False)
    assert sv.min() > 1e-6 * sv.max()


def test_ncg_bins_golden():
    """precompute.basis.n_cg_from_radius on SPEC's worked cases (golden, cited in the fixture)."""
    from precompute.basis import n_cg_from_radius
    for r, expect in GOLD["ncg_bins"]["cases"]:
        assert n_cg_from_radius(r) == expect


def test_pou_arithmetic_golden():
    """precompute.basis.pou_normalise on SPEC's pou_normalize examples: the clip and
    normalisation the basis build uses, called directly."""
    from precompute.basis import pou_normalise
    g = GOLD["pou_examples"]
    phi, phi_dbc, _ = pou_normalise(np.array([0, 0]), np.array(g["u"]), np.zeros(1), 1)
    assert np.allclose(phi, g["phi"], rtol=0, atol=1e-15) and phi_dbc[0] == 0.0
    phi, phi_dbc, _ = pou_normalise(np.array([0, 0]), np.array(g["u2"]), np.array([g["u2_dbc"]]), 1)
    assert np.allclose(phi, g["phi2"], rtol=0, atol=1e-15) and abs(phi_dbc[0] - g["phi2_dbc"]) < 1e-15
    # clipping: a negative u_i contributes nothing to phi or to the denominator
    phi, _, den = pou_normalise(np.array([0, 0, 0]), np.array([0.2, -0.3, 0.6]), np.zeros(1), 1)
    assert np.allclose(phi, [0.25, 0.0, 0.75], rtol=0, atol=1e-15) and abs(den[0] - 0.8) < 1e-15
