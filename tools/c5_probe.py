"""C5 full-size probe of the CUDA path (memory, index widths, time per Newton iteration) on the
trilinear-hat basis of tools/hat_basis.py (NOT the paper's basis; see there).  Prints one JSON
object: device memory in use after set-up and after the steps, Newton / PCG counts, ms per Newton
iteration and the per-phase split, and energy / gradient parity against the oracle at the
contact entry state."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402


def main(steps=2):
    import torch
    from paper_2508_13386_b200 import msim
    from precompute.mesh import contact_state, make_scene
    from tools.hat_basis import hat_basis
    from oracle import ip
    t0 = time.time()
    s = make_scene(5)
    b = hat_basis(s)
    t_setup = time.time() - t0
    free0, total = torch.cuda.mem_get_info()
    ctx = msim.context_from_scene(s, b)
    x_t, v_t = contact_state(s)
    ctx.set_state(x_t, v_t)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    out = {"n_verts": s.n_verts, "n_tets": s.n_tets, "m": b.m, "basis": "trilinear hat 16x8x8 (tools/hat_basis.py)",
           "setup_s": t_setup, "context_mem_gb": (free0 - free1) / 1e9, "total_mem_gb": total / 1e9}
    # energy / gradient parity at the contact entry state (xhat from a free predictor step)
    m = ip.make_model(s)
    xhat = ip.predictor(m, x_t, v_t)
    ctx.set_step_state(x_t, xhat, x_t)
    E = ctx.assemble()
    g = ctx.get_gradient()
    E_o = ip.energy(m, x_t, xhat)
    g_o = ip.gradient(m, x_t, xhat)
    out["energy_rel_err"] = abs(E - E_o) / abs(E_o)
    out["grad_max_rel_err"] = float(np.abs(g - g_o).max() / np.abs(g_o).max())
    ctx.set_state(x_t, v_t)
    ctx.set_profiling(True)
    newton = pcg = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    per_step = []
    for _ in range(steps):
        st = ctx.timestep()
        per_step.append(int(st.newton_iters))
        newton += st.newton_iters
        pcg += st.pcg_iters
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    ph = ctx.phase_times()
    free2, _ = torch.cuda.mem_get_info()
    out.update({"steps": steps, "newton_per_step": per_step, "pcg_iters": int(pcg),
                "ms_per_newton_profiled": ms / max(newton, 1),
                "phase_ms_per_newton": {k: v[0] / max(newton, 1) for k, v in ph.items()},
                "mem_after_steps_gb": (free0 - free2) / 1e9, "coarse": ctx.coarse_info()})
    print(json.dumps(out))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
