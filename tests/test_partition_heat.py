"""Pins of the NEXT-3 partitioner (precompute/partition.py; §3.6.1-3.6.3):
the heat-method distance against closed forms (Euclidean distance on a homogeneous grid; the
1/sqrt(k) metric on a two-material bar), the jump penalty against a brute-force element scan,
the pruning rule on hand-made volumes, and the clustering's material awareness."""
import numpy as np
import pytest

from precompute.basis import build_basis
from precompute.mesh import Scene, kuhn_grid, make_scene
from precompute.partition import HeatGeodesics, element_stiffness_weights, geodesic_kmeans, prune_candidates


def test_heat_distance_homogeneous_is_euclidean():
    """Crane et al.'s heat method with t = h^2 on a homogeneous 16^3 grid: the distance from the
    centre vertex matches |x - x_c| to a few % (discretisation error of the method)."""
    X, tets, _ = kuhn_grid(16, 16, 16, 0.1)
    geo = HeatGeodesics(X, tets.astype(np.int64), np.ones(len(tets)))
    c = int(np.argmin(np.linalg.norm(X - X.mean(0), axis=1)))
    D = geo.distances([c])[0]
    R = np.linalg.norm(X - X[c], axis=1)
    sel = R > 0.25
    rel = np.abs(D[sel] - R[sel]) / R[sel]
    assert D[c] == 0.0
    assert rel.mean() < 0.04 and rel.max() < 0.15


def _two_material_bar():
    X, tets, _ = kuhn_grid(40, 4, 4, 0.1)
    tets = tets.astype(np.int64)
    xc = X[tets].mean(1)[:, 0]
    return X, tets, np.where(xc < 2.0, 1e9, 1e5)


def test_heat_distance_stiffness_metric():
    """With diffusion coefficient k the distance grows as |dx| / sqrt(k): along a bar with a stiff
    (k = 1e4 x) half the slopes differ by sqrt(1e4) = 100 (stiff regions are 'closer')."""
    X, tets, E = _two_material_bar()
    geo = HeatGeodesics(X, tets, E, jump=None)
    s0 = int(np.argmin(np.linalg.norm(X - [0.0, 0.2, 0.2], axis=1)))
    D = geo.distances([s0])[0]
    line = np.isclose(X[:, 1], 0.2) & np.isclose(X[:, 2], 0.2)
    xs, ds = X[line, 0], D[line]
    stiff = (xs > 0.3) & (xs < 1.7)
    soft = (xs > 2.3) & (xs < 3.7)
    ps = np.polyfit(xs[stiff], ds[stiff], 1)[0]
    pf = np.polyfit(xs[soft], ds[soft], 1)[0]
    assert abs(ps - 1.0 / np.sqrt(geo.k.max())) < 0.05 / np.sqrt(geo.k.max())
    assert abs(pf / ps - 100.0) < 5.0


def test_jump_penalty_bruteforce():
    """Elements with a vertex shared with an element of another material get jump * min(k); the
    others keep E / median(E) (element-by-element scan)."""
    X, tets, _ = kuhn_grid(5, 4, 3, 0.1)
    tets = tets.astype(np.int64)
    rng = np.random.default_rng(3)
    E = np.where(rng.random(len(tets)) < 0.2, 1e8, 1e6)
    k, inter = element_stiffness_weights(tets, E, jump=0.25)
    k0 = E / np.median(E)
    for e in range(len(tets)):
        expect = any(len({E[f] for f in range(len(tets)) if v in tets[f]}) > 1 for v in tets[e])
        assert inter[e] == expect, e
        assert k[e] == (0.25 * k0.min() if expect else k0[e])


def test_prune_rule():
    """§3.6.3: candidates have median >= 1.75 x volume; the n smallest are deleted."""
    vol = np.array([10.0, 1.0, 9.0, 2.0, 11.0, 5.0, 0.0, 10.0, 3.0])
    # median 5; candidates vol <= 5/1.75 = 2.857: ids 1 (1.0), 3 (2.0), 6 (0.0)
    assert list(prune_candidates(vol, 1.75, 5)) == [1, 3, 6]
    assert list(prune_candidates(vol, 1.75, 2)) == [1, 6]
    assert len(prune_candidates(np.full(7, 4.0), 1.75, 5)) == 0


def _bar_scene(m):
    X, tets, E = _two_material_bar()
    nt = len(tets)
    return Scene("bar2", 900, (40, 4, 4), 0.1, X, tets.astype(np.int32), E, np.full(nt, 0.4),
                 np.full(nt, 1000.0), np.zeros(0, np.int32), None, m=m, steps=1)


def test_geodesic_kmeans_material_aware():
    """Stiff regions get larger clusters (Fig. 'clustering'): on the two-material bar
    the stiff half holds fewer clusters than the soft half, unlike a Euclidean split."""
    s = _bar_scene(12)
    a, centres = geodesic_kmeans(s, 12, seed=1, max_iter=15)
    xc = s.X[s.tets].mean(1)[:, 0]
    n = a.max() + 1
    stiff_share = np.array([np.mean(xc[a == i] < 2.0) for i in range(n)])
    assert (stiff_share > 0.5).sum() < (stiff_share <= 0.5).sum()
    a2, _ = geodesic_kmeans(s, 12, seed=1, max_iter=15)
    assert np.array_equal(a, a2)   # deterministic


@pytest.mark.parametrize("partition", ["heat"])
def test_heat_basis_valid_c2(partition):
    """The heat-geodesic partition gives a valid basis on C2 (1e5 / 1e9 Pa cubes): partition of
    unity with the DBC weight, every free vertex covered, handles relabelled in x order."""
    s = make_scene(2)
    b = build_basis(s, workers=1, partition=partition)
    n_v = s.n_verts
    sums = np.bincount(np.repeat(np.arange(n_v), np.diff(b.vptr)), weights=b.phi, minlength=n_v) + b.phi_dbc
    assert np.abs(sums - 1.0).max() < 1e-12
    assert np.all(np.diff(b.vptr) > 0) or np.all(b.phi_dbc[np.diff(b.vptr) == 0] == 1.0)
    assert np.all(np.diff(b.origins[:, 0]) >= 0)
    assert 0 < b.m <= s.m
