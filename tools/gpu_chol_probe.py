"""Timing probe: dense fp64 Cholesky + solve of an n x n SPD matrix on the GPU (torch / cuSOLVER),
the size of C5's per-handle bilaplacian subdomains (n ~ 56k)."""
import sys, time
import torch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 56000
torch.manual_seed(0)
A = torch.randn(n, 64, dtype=torch.float64, device="cuda")
K = A @ A.T
K.diagonal().add_(n ** 0.5)
b = torch.randn(n, 1, dtype=torch.float64, device="cuda")
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.time()
    Lc = torch.linalg.cholesky(K)
    x = torch.cholesky_solve(b, Lc)
    torch.cuda.synchronize(); t1 = time.time()
    print(f"n={n} cholesky+solve {t1 - t0:.2f} s ({n**3 / 3 / (t1 - t0) / 1e12:.1f} TFLOP/s)", flush=True)
    del Lc
print("mem GB", torch.cuda.max_memory_allocated() / 1e9)
