import sys, numpy as np
sys.path.insert(0, '.')
from paper_2508_13386_b200 import msim
from precompute.mesh import make_scene
from precompute.basis import cached_basis
from precompute.cubature import cached_cubature
c = int(sys.argv[1]); cub = int(sys.argv[2]); lag = int(sys.argv[3])
s = make_scene(c); b = cached_basis(s); cu = cached_cubature(s, b)
ctx = msim.context_from_scene(s, b, cubature=cu, use_cubature=cub, lag_hessian=lag)
for step in range(12):
    ctx.begin_step()
    for it in range(60):
        try:
            st = ctx.newton_step()
        except Exception as e:
            print('step', step, 'it', it, 'ERROR', e, flush=True); sys.exit(0)
        print(f'step {step} it {it} a0 {st.alpha0:.3g} a {st.alpha:.3g} ev {st.ls_evals} ds {st.ds_norm:.3e} E {st.energy:.6e} dE {st.delta_energy:.3e} g {st.grad_norm:.3e} fail {st.ls_failed}', flush=True)
        if st.converged or st.ls_failed: break
    ctx.end_step()
