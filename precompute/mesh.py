"""Seeded synthetic scene generator for the five BASELINE.json configs (C1-C5).

This module is an INPUT GENERATOR shared by the CUDA path and the oracle.  It
holds none of the method's arithmetic (no energy, Hessian, basis projection or
solver): it only lays out vertices, tetrahedra, per-tet materials, Dirichlet
vertices and the ground plane, with the recipe of SURVEY.md §8(d):

* Kuhn 6-tet split of every cube: for each axis permutation s,
  tet = (o, o+e_s1, o+e_s1+e_s2, o+(1,1,1)), reoriented to positive volume.
* Vertex id = (i*(ny+1) + j)*(nz+1) + k (x slowest, so x-slabs are contiguous);
  unused vertices (C3 lattice) are dropped keeping that order.
* Seeds: numpy default_rng(SeedSequence(c).spawn(3)) -> [materials, mask, kmeans].
* IE, h = 1/60 s, gravity (0,0,-9.8), eps = 1e-6, rho = 1000, cube edge 0.1 m.
* Ground plane n = +z, offset 0, dhat = 1e-3, kappa = 1e4 * E_lowmedian * dhat.

The paper's own scenes (Table 1) are not available; these
synthetic configs stand in for them.
"""
from __future__ import annotations

import dataclasses
import itertools

import numpy as np

H_DEFAULT = 1.0 / 60.0
GRAVITY = (0.0, 0.0, -9.8)


@dataclasses.dataclass
class Scene:
    name: str
    config: int
    dims: tuple            # (nx, ny, nz) cubes
    a: float               # cube edge [m]
    X: np.ndarray          # (n_v, 3) rest positions == initial positions [m]
    tets: np.ndarray       # (n_t, 4) int32, positive orientation
    E: np.ndarray          # (n_t,) Young's modulus [Pa]
    nu: np.ndarray         # (n_t,) Poisson ratio
    rho: np.ndarray        # (n_t,) density [kg/m^3]
    dbc: np.ndarray        # (n_d,) int32 pinned vertices
    ground: dict | None    # {normal, offset, dhat, kappa} or None
    m: int                 # number of SMS handles
    steps: int             # timesteps of the config
    h: float = H_DEFAULT
    gravity: tuple = GRAVITY
    eps: float = 1e-6
    max_newton: int = 100
    kmeans_seed: int = 0

    @property
    def n_verts(self):
        return self.X.shape[0]

    @property
    def n_tets(self):
        return self.tets.shape[0]

    def rngs(self):
        return _rngs(self.config)


def _rngs(c):
    return [np.random.default_rng(s) for s in np.random.SeedSequence(c).spawn(3)]


def kuhn_grid(nx, ny, nz, a, mask=None, origin=(0.0, 0.0, 0.0)):
    """Vertices and Kuhn tets of an nx*ny*nz cube grid (cubes with mask True).

    Returns X (n_v,3), tets (n_t,4) int32, cube_of_tet (n_t,) int64 (C-order
    cube index i*ny*nz + j*nz + k).
    """
    if mask is None:
        mask = np.ones((nx, ny, nz), dtype=bool)
    ci, cj, ck = np.nonzero(mask)                     # C-order cube list
    cube_lin = (ci * ny + cj) * nz + ck

    def vid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k

    e = np.eye(3, dtype=np.int64)
    tets = []
    cube_of = []
    for perm in itertools.permutations(range(3)):
        p1 = e[perm[0]]
        p2 = e[perm[0]] + e[perm[1]]
        corners = [np.zeros(3, np.int64), p1, p2, np.ones(3, np.int64)]
        t = np.stack([vid(ci + c[0], cj + c[1], ck + c[2]) for c in corners], axis=1)
        tets.append(t)
        cube_of.append(cube_lin)
    # interleave so that the 6 tets of one cube are adjacent: (cube, perm) order
    tets = np.stack(tets, axis=1).reshape(-1, 4)
    cube_of = np.stack(cube_of, axis=1).reshape(-1)

    gi, gj, gk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    Xfull = np.stack([gi.ravel(), gj.ravel(), gk.ravel()], axis=1).astype(np.float64) * a
    Xfull += np.asarray(origin, dtype=np.float64)

    used = np.zeros(Xfull.shape[0], dtype=bool)
    used[tets.ravel()] = True
    remap = -np.ones(Xfull.shape[0], dtype=np.int64)
    remap[used] = np.arange(int(used.sum()))
    X = Xfull[used].copy()
    tets = remap[tets]

    # positive orientation: det[x1-x0, x2-x0, x3-x0] > 0
    D = X[tets[:, 1:]] - X[tets[:, :1]]
    vol = np.linalg.det(D)
    neg = vol < 0
    tets[neg, 2], tets[neg, 3] = tets[neg, 3].copy(), tets[neg, 2].copy()
    return X, tets.astype(np.int32), cube_of


def lower_median(v):
    s = np.sort(np.asarray(v))
    return float(s[(len(s) - 1) // 2])


def make_ground(E, dhat=1e-3):
    return dict(normal=(0.0, 0.0, 1.0), offset=0.0, dhat=dhat,
                kappa=1e4 * lower_median(E) * dhat)


def scene_c1():
    """C1 cantilever beam: 10x2x2 cubes of 0.1 m, E=1e6, nu=0.45, x=0 pinned, m=8."""
    nx, ny, nz, a = 10, 2, 2, 0.1
    X, tets, cube_of = kuhn_grid(nx, ny, nz, a)
    nt = len(tets)
    dbc = np.nonzero(np.isclose(X[:, 0], 0.0))[0].astype(np.int32)
    return Scene("C1_beam", 1, (nx, ny, nz), a, X, tets, np.full(nt, 1e6), np.full(nt, 0.45),
                 np.full(nt, 1000.0), dbc, None, m=8, steps=10)


def scene_c2():
    """C2 heterogeneous bar: 40x10x10, per cube Bernoulli(0.1) E=1e9 else 1e5, nu=0.4, m=64."""
    nx, ny, nz, a = 40, 10, 10, 0.1
    r_mat, _, _ = _rngs(2)
    stiff = r_mat.random(nx * ny * nz) < 0.1
    Ecube = np.where(stiff, 1e9, 1e5)
    X, tets, cube_of = kuhn_grid(nx, ny, nz, a)
    nt = len(tets)
    dbc = np.nonzero(np.isclose(X[:, 0], 0.0))[0].astype(np.int32)
    return Scene("C2_bar", 2, (nx, ny, nz), a, X, tets, Ecube[cube_of], np.full(nt, 0.4),
                 np.full(nt, 1000.0), dbc, None, m=64, steps=20)


def c3_mask(n=60, period=30, band=17, phase=(0, 0, 0)):
    idx = np.arange(n)
    inb = [((idx + phase[d]) % period) < band for d in range(3)]
    I, J, K = np.meshgrid(inb[0], inb[1], inb[2], indexing="ij")
    cnt = I.astype(int) + J.astype(int) + K.astype(int)
    return cnt >= 2, (I, J, K)


def scene_c3(drop=0.04):
    """C3 lattice block: 60^3 with a seeded periodic strut mask, log10 E ~ U[5,8] per strut."""
    n, a = 60, 0.1
    r_mat, r_mask, _ = _rngs(3)
    phase = r_mask.integers(0, 30, size=3)
    mask, (I, J, K) = c3_mask(n, 30, 17, tuple(int(p) for p in phase))
    idx = np.arange(n)
    bi = [(idx + phase[d]) // 30 for d in range(3)]
    BI, BJ, BK = np.meshgrid(bi[0], bi[1], bi[2], indexing="ij")
    # free axis: the one coordinate not in band; joints (all 3 in band) -> x strut (axis 0)
    free = np.where(~I, 0, np.where(~J, 1, np.where(~K, 2, 0)))
    sid = np.stack([free, BI, BJ, BK], axis=-1)[mask]          # (n_cubes, 4) C-order
    uniq, inv = np.unique(sid, axis=0, return_inverse=True)
    logE = r_mat.uniform(5.0, 8.0, size=len(uniq))
    Ecube = 10.0 ** logE[inv.ravel()]
    X, tets, cube_of = kuhn_grid(n, n, n, a, mask=mask, origin=(0.0, 0.0, drop))
    # cube_of is a full-grid C-order index; map to the masked cube list order
    full_to_masked = -np.ones(n * n * n, dtype=np.int64)
    full_to_masked[np.flatnonzero(mask.ravel())] = np.arange(int(mask.sum()))
    E = Ecube[full_to_masked[cube_of]]
    nt = len(tets)
    return Scene("C3_lattice", 3, (n, n, n), a, X, tets, E, np.full(nt, 0.45), np.full(nt, 1000.0),
                 np.zeros(0, np.int32), make_ground(E), m=256, steps=30)


def scene_c4(drop=0.04, n=64, m=512):
    """C4 dense cube: 64^3, per cube ln E ~ N(ln 1e6, 1.5^2), nu=0.45, dropped on the barrier."""
    a = 0.1
    r_mat, _, _ = _rngs(4)
    Ecube = np.exp(np.log(1e6) + 1.5 * r_mat.standard_normal(n * n * n))
    X, tets, cube_of = kuhn_grid(n, n, n, a, origin=(0.0, 0.0, drop))
    E = Ecube[cube_of]
    nt = len(tets)
    return Scene("C4_cube", 4, (n, n, n), a, X, tets, E, np.full(nt, 0.45), np.full(nt, 1000.0),
                 np.zeros(0, np.int32), make_ground(E), m=m, steps=20)


def scene_c5(dims=(256, 128, 64), m=1024):
    """C5 layered slab: E = 1e5 if floor(k/8) even else 1e9, nu=0.4, bottom at z = dhat."""
    nx, ny, nz = dims
    a, dhat = 0.1, 1e-3
    X, tets, cube_of = kuhn_grid(nx, ny, nz, a, origin=(0.0, 0.0, dhat))
    k = cube_of % nz
    E = np.where((k // 8) % 2 == 0, 1e5, 1e9)
    nt = len(tets)
    return Scene("C5_slab", 5, dims, a, X, tets, E, np.full(nt, 0.4), np.full(nt, 1000.0),
                 np.zeros(0, np.int32), make_ground(E, dhat), m=m, steps=10)


def scene_small_drop(n=(6, 5, 4), m=4, drop=0.002, seed=7):
    """Small contact scene used by parity tests (not a BASELINE config): ln E ~ N(ln 1e6, 1.5)."""
    nx, ny, nz = n
    a = 0.1
    rng = np.random.default_rng(seed)
    Ecube = np.exp(np.log(1e6) + 1.5 * rng.standard_normal(nx * ny * nz))
    X, tets, cube_of = kuhn_grid(nx, ny, nz, a, origin=(0.0, 0.0, drop))
    E = Ecube[cube_of]
    nt = len(tets)
    return Scene("small_drop", 100 + seed, n, a, X, tets, E, np.full(nt, 0.45), np.full(nt, 1000.0),
                 np.zeros(0, np.int32), make_ground(E), m=m, steps=5)


SCENES = {1: scene_c1, 2: scene_c2, 3: scene_c3, 4: scene_c4, 5: scene_c5}


def make_scene(c: int) -> Scene:
    return SCENES[c]()


def contact_state(scene: Scene):
    """Deterministic contact entry state (x, v) for timed / bootstrapped Newton iterations: the
    rest shape lowered so its bottom layer sits inside the barrier band, 0.6 dhat above the
    ground, falling at 0.5 m/s (scenes without ground: rest, v = 0)."""
    x = np.array(scene.X, dtype=np.float64)
    v = np.zeros_like(x)
    if scene.ground is not None:
        x[:, 2] += 0.6 * scene.ground["dhat"] - x[:, 2].min()
        v[:, 2] = -0.5
    return x, v


def random_state(scene: Scene, amp: float, seed: int):
    """Seeded random perturbation of the rest shape (for element-level parity inputs).

    x = X + amp*a*N(0,1); DBC vertices stay at rest.  Inversions are possible for
    large amp; callers choose amp small enough (checked by the callers)."""
    rng = np.random.default_rng(seed)
    x = scene.X + amp * scene.a * rng.standard_normal(scene.X.shape)
    if len(scene.dbc):
        x[scene.dbc] = scene.X[scene.dbc]
    return x
