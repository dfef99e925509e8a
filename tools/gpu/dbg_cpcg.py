"""Debug: drop scene in the paper's coarse mode (block-Jacobi PCG): GPU against the oracle, per Newton iteration."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import solver
from precompute.basis import build_basis
from precompute.mesh import scene_small_drop
from paper_2508_13386_b200 import msim

s = scene_small_drop(n=(6, 5, 4), m=6, drop=0.002)
b = build_basis(s, workers=1)
MODE = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx = msim.context_from_scene(s, b, coarse_mode=MODE)
sim = solver.OracleSim(s, b, coarse_mode="pcg" if MODE else "exact")
diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
for step in range(1):
    ctx.begin_step()
    gpu = []
    for it in range(12):
        st = ctx.newton_step()
        gpu.append((st.coarse_iters, round(st.alpha0, 6), round(st.alpha, 6), st.ls_evals, float(st.ds_norm), bool(st.converged), bool(st.ls_failed)))
        if st.converged or st.ls_failed:
            break
    ctx.end_step()
    infos = sim.timestep()
    print("step", step, "GPU   ", gpu)
    print("step", step, "oracle", [(getattr(i, "coarse_iters", None), round(i.alpha0, 6), round(i.alpha, 6), i.ls_evals, float(i.ds_norm), bool(i.converged)) for i in infos])
    x, _ = ctx.get_state()
    print("   max|dx|/diag", np.abs(x - sim.x).max() / diag)
