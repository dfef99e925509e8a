"""BDF2 (MS_INTEGRATOR_BDF2; NEXT-4, §3.1, reading C2) on the GPU against the
oracle's BDF2 (oracle/solver.py integrator="bdf2", pinned in tests/test_oracle_bdf2.py):
free-running timesteps -- the first an implicit-Euler step (no history), the rest BDF2 with
alpha = 4/9 -- positions to 1e-6 of the bounding box (north_star), Newton counts equal, and the
velocities, which carry the history, to the same relative accuracy."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import solver  # noqa: E402
from precompute.basis import build_basis  # noqa: E402
from precompute.mesh import make_scene, scene_small_drop  # noqa: E402

BDF2 = 1


@pytest.fixture(scope="module")
def msim():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_13386_b200 import msim as m
    return m


@pytest.mark.parametrize("name,steps", [("c1", 10), ("drop", 8), ("c2", 3)])
def test_bdf2_timesteps(msim, name, steps):
    s = {"c1": lambda: make_scene(1), "c2": lambda: make_scene(2),
         "drop": lambda: scene_small_drop(n=(6, 5, 4), m=6, drop=0.002)}[name]()
    b = build_basis(s, workers=1)
    ctx = msim.context_from_scene(s, b, integrator=BDF2)
    sim = solver.OracleSim(s, b, integrator="bdf2")
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    for k in range(steps):
        st = ctx.timestep()
        infos = sim.timestep()
        x, v = ctx.get_state()
        assert st.newton_iters == len(infos), (name, k)
        assert np.abs(x - sim.x).max() <= 1e-6 * diag, (name, k)
        vs = max(np.abs(sim.v).max(), 1e-30)
        assert np.abs(v - sim.v).max() <= 1e-5 * vs, (name, k, np.abs(v - sim.v).max() / vs)


def test_bdf2_restarts_after_set_state(msim):
    """ms_set_state starts a new trajectory: its first step is implicit Euler again."""
    s = scene_small_drop(n=(4, 3, 3), m=4, drop=0.002)
    b = build_basis(s, workers=1)
    ctx = msim.context_from_scene(s, b, integrator=BDF2)
    ie = msim.context_from_scene(s, b)
    for _ in range(3):
        ctx.timestep()
    ctx.set_state(s.X, np.zeros_like(s.X))
    ctx.timestep()
    ie.timestep()
    assert np.array_equal(ctx.get_state()[0], ie.get_state()[0])
