"""NEXT-2 on the GPU (§3.8 cubature subspace Hessian, §3.7.2 Hessian lagging; readings C3,
C4) against the oracle in the same mode (oracle/solver.py OracleSim(cubature=..., lag=...)):
free-running timesteps with both levers on, each alone, positions to 1e-6 of the bounding box
(north_star), Newton counts equal.  The cubature schemes come from precompute/cubature.py (the
input generator both sides consume).  C2 runs one step: with its 1e4 stiffness contrast inside
partitions the cubature subspace Hessian is a coarse approximation and the second step takes
76-89 lagged Newton iterations, over which the refresh decisions (a threshold on a moving
average of step sizes) amplify rounding differences into different iteration counts."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import solver  # noqa: E402
from precompute.basis import build_basis  # noqa: E402
from precompute.cubature import build_cubature  # noqa: E402
from precompute.mesh import make_scene, scene_small_drop  # noqa: E402


@pytest.fixture(scope="module")
def msim():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_13386_b200 import msim as m
    return m


@pytest.mark.parametrize("name,steps,cub,lag", [("drop", 8, 1, 1), ("c1", 6, 1, 1), ("c2", 1, 1, 1),
                                                ("drop", 6, 1, 0), ("drop", 6, 0, 1)])
def test_next2_timesteps(msim, name, steps, cub, lag):
    s = {"c1": lambda: make_scene(1), "c2": lambda: make_scene(2),
         "drop": lambda: scene_small_drop(n=(6, 5, 4), m=6, drop=0.002)}[name]()
    b = build_basis(s, workers=1)
    c = build_cubature(s, b, workers=1)
    ctx = msim.context_from_scene(s, b, cubature=c, use_cubature=cub, lag_hessian=lag)
    sim = solver.OracleSim(s, b, cubature=c if cub else None, lag=bool(lag))
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    for k in range(steps):
        st = ctx.timestep()
        infos = sim.timestep()
        x, _ = ctx.get_state()
        assert st.newton_iters == len(infos), (name, k, st.newton_iters, len(infos))
        assert np.abs(x - sim.x).max() <= 1e-6 * diag, (name, k, np.abs(x - sim.x).max() / diag)
