"""C5's SMS basis (precompute/basis.py, the paper's construction) with the 1,024 per-handle
bilaplacian systems solved on the GPU by a dense fp64 Cholesky (solver="cuda"): the sparse-LU
default needs > 10 h of CPU at C5's ~56 k-vertex subdomains.  The partition comes from
precompute.basis.cached_partition (k-means, cached under .cache/).  Writes the basis where
cached_basis looks for it and, for the transfer back from a GPU box, a copy split into chunks of
at most 60 MiB under the directory given as argv[1] (default /tmp/c5basis).
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from precompute.basis import build_basis, cached_basis_path, cached_partition  # noqa: E402
from precompute.mesh import make_scene  # noqa: E402

CHUNK = 60 * 2 ** 20


def main():
    out_dir = sys.argv[1] if len(sys.argv) > 1 else "/tmp/c5basis"
    t0 = time.time()
    s = make_scene(5)
    part = cached_partition(s)
    print(f"partition m={part[1]} ({time.time() - t0:.0f}s)", flush=True)
    b = build_basis(s, partition_data=part, solver="cuda", workers=max(1, min(14, (os.cpu_count() or 2) - 2)),
                    verbose=True)
    path = cached_basis_path(s)
    b.save(path)
    print(f"saved {path} ({os.path.getsize(path) / 2**20:.1f} MiB, {time.time() - t0:.0f}s); n_cg={b.n_cg} "
          f"holes={b.n_holes} nnz={len(b.phi)}", flush=True)
    os.makedirs(out_dir, exist_ok=True)
    data = open(path, "rb").read()
    for k in range(0, len(data), CHUNK):
        with open(os.path.join(out_dir, f"{os.path.basename(path)}.part{k // CHUNK}"), "wb") as f:
            f.write(data[k:k + CHUNK])
    print(f"{(len(data) + CHUNK - 1) // CHUNK} chunks in {out_dir}", flush=True)


if __name__ == "__main__":
    main()
