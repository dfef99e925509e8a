"""Oracle fixtures for the full-size GPU parity tests (test infrastructure; calls only oracle/
and precompute/, never the CUDA path).

    python tools/oracle_fixtures.py newton C      # bootstrapped Newton iterations of config C
    python tools/oracle_fixtures.py traj C [K]    # free-running timesteps 1..K of config C
    python tools/oracle_fixtures.py newton 5 --hat   # C5 on the stand-in basis of tools/hat_basis.py

compact C FILE: rewrite a full fixture in the sampled form (see compact()).

newton: from precompute.mesh.contact_state (x^t, v) the oracle runs N_ITER Newton iterations of
one timestep (Alg. 1, §3.9) and stores, per iteration, the start iterate x,
d = d_s + d_f, d_s, alpha0 (CCD / inversion filters), alpha, ls_evals, energy and ||d_s||.
traj: the oracle's own timesteps from the scene's initial state (rest, v = 0): x after every
step and the Newton iterations it took (SURVEY §8(c) per-timestep tolerance).
Files go to .cache/fixtures/ (git-ignored; they travel with the repo snapshot to the GPU box).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import solver  # noqa: E402
from precompute.basis import BASIS_VERSION, cached_basis  # noqa: E402
from precompute.mesh import contact_state, make_scene  # noqa: E402

N_ITER = 2
FIX_DIR = os.environ.get("MSIM_FIXTURES", os.path.join(ROOT, ".cache", "fixtures"))


def sample_stride(n_verts):
    """Vertex stride of the stored vectors: every vertex up to 100k vertices (C1, C2), every 4th up
    to 1M (C3, C4), every 8th beyond (C5).  Keeps the fixtures inside the repo snapshot that travels
    to the GPU box; the full-size comparisons then run on the sampled vertices (the oracle still
    computes every vertex)."""
    return 1 if n_verts <= 100_000 else (4 if n_verts <= 1_000_000 else 8)


def compact(data, n_verts, kind):
    """Sampled form of a fixture: vectors at vertices 0, stride, 2 stride, ...; for configs beyond
    1M vertices one Newton iteration and no x_t / xhat (the test recomputes them from
    precompute.mesh.contact_state and oracle.ip.predictor)."""
    st = sample_stride(n_verts)
    out = {"stride": np.array(st)}
    if kind == "newton":
        n_it = int(data["n_iter"]) if st < 8 else 1
        out["n_iter"] = np.array(n_it)
        for it in range(n_it):
            out[f"scal{it}"] = data[f"scal{it}"]
            out[f"d{it}"] = np.ascontiguousarray(data[f"d{it}"][::st])
            out[f"ds{it}"] = np.ascontiguousarray(data[f"ds{it}"][::st])
            if st < 8:
                out[f"x{it}"] = data[f"x{it}"]    # iteration starts (full: the GPU is set to them)
        if st < 8:
            out["x_t"], out["xhat"] = data["x_t"], data["xhat"]
    else:
        out["x"] = np.ascontiguousarray(data["x"][:, ::st])
        out["newton"] = data["newton"]
    return out


def fixture_path(kind, c, k=None):
    tag = f"_{k}" if k is not None else ""
    return os.path.join(FIX_DIR, f"{kind}_C{c}{tag}_{BASIS_VERSION}.npz")


def scene_basis(c, hat=False):
    s = make_scene(c)
    if hat:   # stand-in partition of unity (tools/hat_basis.py), NOT the paper's basis
        from tools.hat_basis import hat_basis
        return s, hat_basis(s)
    return s, cached_basis(s)


def newton_fixture(c, n_iter=N_ITER, verbose=True, hat=False):
    s, b = scene_basis(c, hat)
    sim = solver.OracleSim(s, b)
    sim.x, sim.v = contact_state(s)
    x_t = sim.x.copy()
    v_t = sim.v.copy()
    sim.begin_step()
    out = {"x_t": x_t, "v_t": v_t, "xhat": sim.xhat}
    for it in range(n_iter):
        x0 = sim.x.copy()
        t0 = time.time()
        info = sim.newton_iteration()
        if verbose:
            print(f"C{c} iteration {it}: alpha0={info.alpha0:.6g} alpha={info.alpha:.6g} evals={info.ls_evals} "
                  f"|ds|={info.ds_norm:.6g} ({time.time() - t0:.1f}s)", flush=True)
        out[f"x{it}"] = x0
        out[f"d{it}"] = info.d.reshape(-1, 3)
        out[f"ds{it}"] = info.ds.reshape(-1, 3)
        out[f"scal{it}"] = np.array([info.alpha0, info.alpha, info.ls_evals, info.ds_norm, info.energy,
                                     float(info.converged), float(info.ls_failed)])
        if info.converged or info.ls_failed:
            break
    out["n_iter"] = np.array(it + 1)
    return out


def traj_fixture(c, k, verbose=True, hat=False):
    s, b = scene_basis(c, hat)
    sim = solver.OracleSim(s, b)
    xs, newton = [], []
    for step in range(k):
        t0 = time.time()
        infos = sim.timestep()
        xs.append(sim.x.copy())
        newton.append(len(infos))
        if verbose:
            print(f"C{c} step {step + 1}: {len(infos)} Newton iterations, alpha={[round(i.alpha, 4) for i in infos]} "
                  f"({time.time() - t0:.1f}s)", flush=True)
    return {"x": np.array(xs), "newton": np.array(newton)}


def main():
    hat = "--hat" in sys.argv
    argv = [a for a in sys.argv if a != "--hat"]
    kind, c = argv[1], int(argv[2])
    tag = f"{c}hat" if hat else c
    os.makedirs(FIX_DIR, exist_ok=True)
    if kind == "compact":   # rewrite an existing full fixture file in the sampled form
        path = argv[3]
        full = dict(np.load(path))
        if "stride" in full:
            print("already compact", path)
            return
        data = compact(full, make_scene(c).n_verts, "traj" if "traj_" in os.path.basename(path) else "newton")
    elif kind == "newton":
        data = compact(newton_fixture(c, hat=hat), make_scene(c).n_verts, "newton")
        path = fixture_path("newton", tag)
    else:
        k = int(argv[3]) if len(argv) > 3 else make_scene(c).steps
        data = compact(traj_fixture(c, k, hat=hat), make_scene(c).n_verts, "traj")
        path = fixture_path("traj", tag, k)
    np.savez(path + ".tmp.npz", **data)
    os.replace(path + ".tmp.npz", path)
    print("wrote", path, flush=True)


if __name__ == "__main__":
    main()
