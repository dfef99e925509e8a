"""Full-size Newton-iteration and timestep parity on every BASELINE config (C1-C5), through the
C-ABI context the bench uses (context_from_scene, default parameters).

* Bootstrapped Newton iterations (reading R10): the GPU context is set to the oracle's iterate
  (x^t, xhat, x) before each iteration and runs one ms_newton_step; compared with the oracle's
  iteration from the same state (tools/oracle_fixtures.py, which calls only oracle/): the
  subspace direction d_s and the full direction d = d_s + d_f (Alg. 1, Alg. 2 P:427-450,
  P:477-484) to 1e-8 relative (north_star's PCG bar), the filtered initial step alpha0 (CCD and
  inversion filters), the accepted alpha and the number of line-search
  evaluations (backtracking, Q12) exactly / to rounding, the updated iterate, ||d_s||
  and the termination decision (R7).  The entry state (precompute.mesh.contact_state)
  puts the bottom layer inside the barrier band falling at 0.5 m/s, so the barrier, the CCD
  filter and the PSD projection are all active.
* Free-running timesteps: the GPU runs the config's own timesteps from rest and
  its positions after every step are compared with the oracle's trajectory, max_v |x_v - x_v^o|
  / bbox diagonal <= 1e-6 (north_star), Newton counts equal.  The oracle trajectories of the
  large configs take hours of CPU; they are precomputed by tools/oracle_fixtures.py and this
  test covers the steps present in the fixture (k stated in its file name).
"""
import glob
import os
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from precompute.basis import cached_basis, cached_basis_path  # noqa: E402
from oracle import ip  # noqa: E402
from precompute.mesh import contact_state, make_scene  # noqa: E402
from tools import oracle_fixtures as fx  # noqa: E402


def rel_err(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def _ctx(c, hat=False):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_13386_b200 import msim
    s = make_scene(c)
    if hat:   # C5 on the stand-in basis (tools/hat_basis.py) while the paper's basis is not cached
        from tools.hat_basis import hat_basis
        b = hat_basis(s)
    else:
        if c == 5 and not os.path.exists(cached_basis_path(s)):
            pytest.skip("C5 basis not precomputed (hours of CPU: tools/rebuild_cache.sh c5basis)")
        b = cached_basis(s)
    return s, b, msim.context_from_scene(s, b)


def _newton_fixture(c, hat=False):
    path = fx.fixture_path("newton", f"{c}hat" if hat else c)
    if c == 5 and not os.path.exists(path):
        pytest.skip("C5 oracle fixture not precomputed (tools/oracle_fixtures.py newton 5 [--hat])")
    if not os.path.exists(path):          # compute it (C1-C4: a few minutes of oracle CPU time)
        os.makedirs(fx.FIX_DIR, exist_ok=True)
        s = make_scene(c)
        np.savez(path, **fx.compact(fx.newton_fixture(c, verbose=False), s.n_verts, "newton"))
    f = dict(np.load(path))
    if "stride" not in f:                 # full vectors (fixtures written before the sampled form)
        f["stride"] = np.array(1)
    return f


@pytest.mark.parametrize("c,hat", [(1, False), (2, False), (3, False), (4, False), (5, False), (5, True)],
                         ids=["C1", "C2", "C3", "C4", "C5", "C5-standin-basis"])
def test_fullsize_newton_bootstrapped(c, hat):
    f = _newton_fixture(c, hat)
    s, b, ctx = _ctx(c, hat)
    model = ip.make_model(s)
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    st_ = int(f["stride"])                 # the directions are stored at vertices 0, st_, 2 st_, ...
    if "x_t" not in f:                    # compact large-config form: the entry state is recomputed
        x_t, v_t = contact_state(s)
        f["x_t"], f["xhat"], f["x0"] = x_t, ip.predictor(model, x_t, v_t), x_t
    for it in range(int(f["n_iter"])):
        ctx.set_step_state(f["x_t"], f["xhat"], f[f"x{it}"])
        st = ctx.newton_step()
        ds, df = ctx.get_direction()
        ds, d = ds.reshape(-1, 3)[::st_], (ds + df).reshape(-1, 3)[::st_]
        a0, alpha, evals, dsn, energy, conv, failed = f[f"scal{it}"]
        assert rel_err(ds, f[f"ds{it}"]) < 1e-8, (c, it, rel_err(ds, f[f"ds{it}"]))
        assert rel_err(d, f[f"d{it}"]) < 1e-8, (c, it, rel_err(d, f[f"d{it}"]))
        assert abs(st.alpha0 - a0) <= 1e-8 * a0, (c, it, st.alpha0, a0)
        assert abs(st.ds_norm - dsn) <= 1e-8 * dsn
        e0 = ip.energy(model, f[f"x{it}"], f["xhat"])        # E(x) at the start of the iteration
        # E is a sum of terms that cancel to first order near rest (rest-stable Psi): 1e-9
        assert abs(st.energy - e0) <= 1e-9 * abs(e0), (c, it, st.energy, e0)
        assert bool(st.ls_failed) == bool(failed)
        if not failed:
            assert st.ls_evals == int(evals), (c, it, st.ls_evals, evals)
            assert abs(st.alpha - alpha) <= 1e-8 * alpha
            _, _, x_new = ctx.get_step_state()
            x_o = f[f"x{it}"].reshape(-1, 3)[::st_] + alpha * f[f"d{it}"].reshape(-1, 3)
            assert np.abs(x_new.reshape(-1, 3)[::st_] - x_o).max() <= 1e-9 * diag
        assert bool(st.converged) == bool(conv)


def _traj_files():
    out = []
    for p in sorted(glob.glob(os.path.join(fx.FIX_DIR, f"traj_C*_{fx.BASIS_VERSION}.npz"))):
        m = re.search(r"traj_C(\d)(hat)?_(\d+)_", os.path.basename(p))
        hat = m.group(2) is not None
        out.append(pytest.param(int(m.group(1)), p, hat,
                                id=f"C{m.group(1)}{'-standin-basis' if hat else ''}x{m.group(3)}"))
    return out or [pytest.param(1, None, False, id="C1-missing")]


@pytest.mark.parametrize("c,path,hat", _traj_files())
def test_fullsize_timestep_free_running(c, path, hat):
    if path is None:                    # C1 is cheap: compute its trajectory here
        k = make_scene(1).steps
        data = fx.traj_fixture(1, k, verbose=False)
    else:
        data = dict(np.load(path))
    s, b, ctx = _ctx(c, hat)
    diag = np.linalg.norm(s.X.max(0) - s.X.min(0))
    worst = 0.0
    stv = int(data.get("stride", 1))      # positions stored at vertices 0, stv, 2 stv, ...
    for step in range(len(data["x"])):
        st = ctx.timestep()
        x, _ = ctx.get_state()
        err = np.linalg.norm(x[::stv] - data["x"][step], axis=1).max() / diag
        worst = max(worst, err)
        assert err <= 1e-6, (c, step + 1, err)
        assert st.newton_iters == int(data["newton"][step]), (c, step + 1, st.newton_iters, data["newton"][step])
