"""Free-running timestep parity log (GPU against the oracle's stored trajectory).

    python tools/freerun_log.py C [out.json] [--hat]

Runs the config's timesteps from rest on cuda:0 through the C-ABI (the bench's context) and
compares, after every step, the positions with the oracle trajectory that
tools/oracle_fixtures.py traj C wrote (oracle only): max_v |x_v - x_v^o| / bbox diagonal
(north_star: <= 1e-6), the displacement-relative error ||dx - dx^o|| / ||dx^o|| and the Newton
iteration counts of both sides (SURVEY §8(c) per-timestep tolerance).  Writes one JSON object.
"""
import glob
import json
import os
import re
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from precompute.basis import BASIS_VERSION, cached_basis  # noqa: E402
from precompute.mesh import make_scene  # noqa: E402
from tools.oracle_fixtures import FIX_DIR  # noqa: E402


def main():
    hat = "--hat" in sys.argv
    sys.argv = [a for a in sys.argv if a != "--hat"]
    c = int(sys.argv[1])
    tag = f"{c}hat" if hat else f"{c}"
    files = sorted(glob.glob(os.path.join(FIX_DIR, f"traj_C{tag}_*_{BASIS_VERSION}.npz")),
                   key=lambda p: int(re.search(r"_(\d+)_v", p).group(1)))
    if not files:
        raise SystemExit(f"no oracle trajectory for C{c} under {FIX_DIR}")
    path = files[-1]
    data = np.load(path)
    xs, newton_o = data["x"], data["newton"]
    stv = int(data["stride"]) if "stride" in data else 1   # positions at vertices 0, stv, 2 stv, ...
    from paper_2508_13386_b200 import msim
    s = make_scene(c)
    if hat:
        from tools.hat_basis import hat_basis
        b = hat_basis(s)
    else:
        b = cached_basis(s)
    ctx = msim.context_from_scene(s, b)
    diag = float(np.linalg.norm(s.X.max(0) - s.X.min(0)))
    steps = []
    x_prev = s.X[::stv].copy()
    xo_prev = s.X[::stv].copy()
    t0 = time.time()
    for k in range(len(xs)):
        st = ctx.timestep()
        x, _ = ctx.get_state()
        x = x[::stv]
        err = np.linalg.norm(x - xs[k], axis=1).max() / diag
        dx, dxo = x - x_prev, xs[k] - xo_prev
        rel = float(np.linalg.norm(dx - dxo) / max(np.linalg.norm(dxo), 1e-300))
        steps.append({"step": k + 1, "max_dx_over_diag": float(err), "disp_rel": rel,
                      "newton_gpu": int(st.newton_iters), "newton_oracle": int(newton_o[k]),
                      "ls_status": int(st.status)})
        x_prev, xo_prev = x, xs[k]
    out = {"config": s.name, "basis": "stand-in (tools/hat_basis.py)" if hat else "paper (precompute/basis.py)", "n_tets": int(s.n_tets), "n_verts": int(s.n_verts), "m": int(b.m),
           "steps_compared": len(xs), "vertex_stride": stv, "steps_of_config": int(s.steps), "oracle_fixture": os.path.basename(path),
           "tolerance": "max_v |x - x_oracle| / bbox diagonal <= 1e-6 (north_star)",
           "worst_max_dx_over_diag": max(r["max_dx_over_diag"] for r in steps),
           "newton_counts_equal": all(r["newton_gpu"] == r["newton_oracle"] for r in steps),
           "gpu_seconds": time.time() - t0, "per_step": steps}
    txt = json.dumps(out, indent=1)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            f.write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
