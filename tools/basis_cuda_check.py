"""precompute/basis.py's solver="cuda" (dense fp64 Cholesky per handle on the GPU) against the
default sparse LU on a config whose basis is cached: same partition / handle lists, weights to the
conditioning of the two direct solves."""
import sys, time
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from precompute.basis import build_basis, cached_basis  # noqa: E402
from precompute.mesh import make_scene  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = make_scene(c)
ref = cached_basis(s)
t0 = time.time()
b = build_basis(s, solver="cuda", workers=14, verbose=True)
print(f"C{c}: cuda build {time.time() - t0:.1f}s; same handles {np.array_equal(b.handle, ref.handle)}, "
      f"same vptr {np.array_equal(b.vptr, ref.vptr)}, max |dphi| {np.abs(b.phi - ref.phi).max():.3e}, "
      f"n_cg {b.n_cg}/{ref.n_cg}", flush=True)
