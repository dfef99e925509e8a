"""Debug: S = B^T H B from W hub ranks vs one context (same state)."""
import sys, threading, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_13386_b200 import msim
from precompute.basis import build_basis
from precompute.mesh import scene_small_drop, random_state

s = scene_small_drop(n=(10, 4, 3), m=6, drop=0.002)
b = build_basis(s, workers=1)
x = random_state(s, 0.01, 3); x[:, 2] = np.maximum(x[:, 2], 0.3e-3)
xhat = s.X + 1e-3
ref = msim.context_from_scene(s, b)
ref.set_step_state(s.X, xhat, x)
E_ref = ref.assemble(); S_ref, Sa_ref = ref.export_coarse(); g_ref = ref.get_gradient()
W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
hub = msim.Hub(W)
streams = [torch.cuda.Stream() for _ in range(W)]
ctxs = [msim.context_from_scene(s, b, stream=streams[r].cuda_stream, rank=r, world=W, hub=hub) for r in range(W)]
out = [None] * W
def work(r):
    c = ctxs[r]
    c.set_step_state(s.X, xhat, x)
    E = c.assemble()
    S, Sa = c.export_coarse()
    out[r] = (E, S, Sa)
th = [threading.Thread(target=work, args=(r,)) for r in range(W)]
[t.start() for t in th]; [t.join() for t in th]
for r in range(W):
    E, S, Sa = out[r]
    print(r, "E", E, E_ref, "S err", np.abs(S - S_ref).max() / np.abs(S_ref).max(), "Sa err", np.abs(Sa - Sa_ref).max() / np.abs(Sa_ref).max())
    bad = np.argwhere(np.abs(S - S_ref) > 1e-8 * np.abs(S_ref).max())
    if len(bad):
        blk = np.unique(bad // 12, axis=0)
        print("  bad blocks", len(blk), blk[:10].tolist())
