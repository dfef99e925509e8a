"""Critical-path analysis of one dataflow Cholesky launch (chol.cu k_chol_dataflow).

Input: gpurun_out/dftask.bin written by a -DMSIM_DF_PROF build (header ntask, NT; the int4
task list; per task claim / ready / end globaltimer stamps and the CTA).  Walks back from the
last finishing task along the latest-finishing dependency and splits the path into execution,
flag latency (dependencies done -> waits satisfied) and claim latency (dependencies done before
the task was claimed).
"""
import sys
from collections import defaultdict

import numpy as np


def load(path):
    with open(path, "rb") as f:
        ntask, NT = np.frombuffer(f.read(8), dtype=np.int32)
        dag = np.frombuffer(f.read(16 * ntask), dtype=np.int32).reshape(ntask, 4)
        ts = np.frombuffer(f.read(32 * ntask), dtype=np.uint64).reshape(ntask, 4).astype(np.int64)
    return int(ntask), int(NT), dag, ts


def deps_of(dag):
    upd = {}        # (i, j, rank) -> task that applies update number `rank` to tile (i, j)
    dfl, pfl = {}, {}
    for q, (ty, i, jk, cnt) in enumerate(dag):
        j, k = jk & 0xffff, jk >> 16
        if ty == 0:
            dfl[k] = q
        elif ty == 4:
            dfl[i] = q
            pfl[(i, k)] = q
            upd[(i, i, cnt >> 16)] = q
        elif ty == 1:
            pfl[(i, k)] = q
        else:
            upd[(i, j, cnt)] = q
    deps = []
    for q, (ty, i, jk, cnt) in enumerate(dag):
        j, k = jk & 0xffff, jk >> 16
        d = []
        if ty == 0:
            if cnt:
                d.append(upd[(k, k, cnt - 1)])
        elif ty == 4:
            need, rank = cnt & 0xffff, cnt >> 16
            if need:
                d.append(upd[(i, k, need - 1)])
            if rank:
                d.append(upd[(i, i, rank - 1)])
            d.append(dfl[k])
        elif ty == 1:
            d.append(dfl[k])
            if cnt:
                d.append(upd[(i, k, cnt - 1)])
        else:
            d += [pfl[(i, k)], pfl[(j, k)]]
            if cnt:
                d.append(upd[(i, j, cnt - 1)])
        deps.append(d)
    return deps


def main(path="gpurun_out/dftask.bin"):
    ntask, NT, dag, ts = load(path)
    claim, ready, end, cta = ts[:, 0], ts[:, 1], ts[:, 2], ts[:, 3]
    t0 = claim.min()
    claim, ready, end = (claim - t0) / 1e3, (ready - t0) / 1e3, (end - t0) / 1e3
    deps = deps_of(dag)
    ddone = np.array([max((end[d] for d in ds), default=0.0) for ds in deps])
    names = {0: "D", 1: "P", 2: "U", 4: "PUD"}
    print(f"tasks {ntask}, NT {NT}, span {end.max():.1f} us, CTAs {len(set(cta.tolist()))}")
    print("type   n    exec_us   wait_us(claim->ready)   flag_lat(deps->ready)   claim_lag(deps->claim,+)")
    for ty in (0, 4, 1, 2):
        m = dag[:, 0] == ty
        if not m.any():
            continue
        ex = end[m] - ready[m]
        wt = ready[m] - claim[m]
        fl = ready[m] - np.maximum(ddone[m], claim[m])
        cl = np.maximum(0, claim[m] - ddone[m])
        print(f"{names[ty]:4s} {m.sum():6d} {ex.mean():8.2f} {wt.mean():12.2f} {fl.mean():18.2f} {cl.mean():22.2f}")
    busy = (end - claim).sum() / (end.max() * len(set(cta.tolist())))
    print(f"CTA occupancy (claim->end) {busy:.2f}, executing {(end - ready).sum() / (end.max() * len(set(cta.tolist()))):.2f}")
    # critical path
    q = int(np.argmax(end))
    acc = defaultdict(float)
    path = []
    while True:
        path.append(q)
        acc["exec_" + names[dag[q, 0]]] += end[q] - ready[q]
        if not deps[q]:
            acc["start"] += ready[q]
            break
        p = max(deps[q], key=lambda d: end[d])
        if claim[q] > end[p]:
            acc["claim_lag"] += claim[q] - end[p]
            acc["flag_lat"] += ready[q] - claim[q]
        else:
            acc["flag_lat"] += ready[q] - end[p]
        q = p
    print(f"critical path: {len(path)} tasks, " + ", ".join(f"{k} {v:.1f}" for k, v in sorted(acc.items())))
    kinds = defaultdict(int)
    for q in path:
        kinds[names[dag[q, 0]]] += 1
    print("  path task kinds:", dict(kinds))
    # the path near the middle, task by task
    mid = path[len(path) // 2: len(path) // 2 + 12]
    for q in reversed(mid):
        ty, i, jk, cnt = dag[q]
        print(f"  {names[ty]:4s} i={i:3d} j={jk & 0xffff:3d} k={jk >> 16:3d} cta={cta[q]:3d} deps_done {ddone[q]:8.1f} "
              f"claim {claim[q]:8.1f} ready {ready[q]:8.1f} end {end[q]:8.1f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
