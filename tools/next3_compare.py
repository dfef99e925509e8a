"""NEXT-3 measurement: Newton iterations per timestep of the CUDA path with the Euclidean
partitioner (the configs' default) and with the paper's stiffness-weighted heat-geodesic
partitioner (precompute/partition.py), same scene, same steps.  Prints one JSON object."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from precompute.basis import build_basis  # noqa: E402
from precompute.mesh import make_scene, scene_small_drop  # noqa: E402


def run(msim, s, b, steps):
    ctx = msim.context_from_scene(s, b)
    its, pcg = [], 0
    t = time.time()
    for _ in range(steps):
        st = ctx.timestep()
        its.append(int(st.newton_iters))
        pcg += st.pcg_iters
    return {"m": int(b.m), "n_cg": int(b.n_cg), "newton_per_step": its, "newton_total": int(sum(its)),
            "wall_s": time.time() - t}


def main():
    from paper_2508_13386_b200 import msim
    out = {}
    cases = [("C1", make_scene(1), 10), ("C2", make_scene(2), 20),
             ("drop_hetero", scene_small_drop(n=(12, 8, 6), m=16, drop=0.002), 10)]
    for name, s, steps in cases:
        row = {}
        for part in ("euclidean", "heat"):
            t = time.time()
            b = build_basis(s, workers=1, partition=part)
            r = run(msim, s, b, steps)
            r["basis_s"] = time.time() - t - r["wall_s"]
            row[part] = r
        out[name] = row
        print(name, {k: (v["m"], v["newton_total"]) for k, v in row.items()}, file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
