"""The CUDA path on a NEXT-3 basis (the paper's stiffness-weighted heat-geodesic partitioner,
precompute/partition.py; §3.6): the basis is an input, so the parity bar is the
one of tests/test_gpu_parity.py -- one bootstrapped Newton iteration of C2 (1e5 / 1e9 Pa cubes)
to 1e-8 in d_s and d, and free-running timesteps with equal Newton counts, positions to 1e-6 of
the bounding box."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import solver  # noqa: E402
from precompute.basis import build_basis  # noqa: E402
from precompute.mesh import make_scene, random_state  # noqa: E402


@pytest.fixture(scope="module")
def msim():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_13386_b200 import msim as m
    return m


@pytest.fixture(scope="module")
def c2_heat():
    s = make_scene(2)
    return s, build_basis(s, workers=1, partition="heat")


def rel_err(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def test_heat_basis_newton_iteration_c2(msim, c2_heat):
    s, b = c2_heat
    ctx = msim.context_from_scene(s, b)
    sim = solver.OracleSim(s, b)
    x = random_state(s, 0.01, 61)
    rng = np.random.default_rng(62)
    xhat = s.X + 0.002 * s.a * rng.standard_normal(s.X.shape)
    ctx.set_step_state(s.X, xhat, x)
    sim.x_t, sim.xhat, sim.x = s.X.copy(), xhat, x.copy()
    info = sim.newton_iteration()
    st = ctx.newton_step()
    ds, df = ctx.get_direction()
    assert rel_err(ds, info.ds) < 1e-8
    assert rel_err(ds + df, info.d) < 1e-8
    assert abs(st.alpha0 - info.alpha0) <= 1e-8 * info.alpha0 and st.ls_evals == info.ls_evals


def test_heat_basis_timesteps_c2(msim, c2_heat):
    s, b = c2_heat
    ctx = msim.context_from_scene(s, b)
    sim = solver.OracleSim(s, b)
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    for _ in range(2):
        st = ctx.timestep()
        infos = sim.timestep()
        x, _ = ctx.get_state()
        assert st.newton_iters == len(infos)
        assert np.abs(x - sim.x).max() <= 1e-6 * diag
