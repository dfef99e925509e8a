"""Forms S = B^T H B a few times on C4 at a contact state (for ncu launch timing of the Galerkin
kernel, e.g. under diagnostic builds -DMSIM_GAL_SKIP_A / -DMSIM_GAL_SKIP_B)."""
import sys
sys.path.insert(0, ".")
from paper_2508_13386_b200 import msim  # noqa: E402
from precompute.basis import cached_basis  # noqa: E402
from precompute.mesh import contact_state, make_scene  # noqa: E402
from oracle import ip  # noqa: E402

s = make_scene(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
b = cached_basis(s)
ctx = msim.context_from_scene(s, b)
x_t, v_t = contact_state(s)
ctx.set_step_state(x_t, ip.predictor(ip.make_model(s), x_t, v_t), x_t)
ctx.assemble()
for _ in range(4):
    ctx.export_coarse(dense=False)
print("ok")
