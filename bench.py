"""Benchmark of the B200-native multilevel Newton solve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]

A "step" is one implicit-Euler timestep of config C4 (64^3 cubes x 6 = 1,572,864 tets,
274,625 vertices, m = 512 handles): predictor, Newton iterations (element gradient, PSD
Hessian, BSR assembly, S = B^T H B + Cholesky, coarse correction, N_cg Jacobi-PCG, filtered
line search) until ||d_s|| / (h n_v) < eps, velocity update -- every row of SURVEY.md §8(a).
`value` = Newton iterations / second over the timed steps (device time, CUDA events, max over
ranks); `pcg_iters_per_s` reports the PCG rate of the same run.  Inputs are larger than L2
(the BSR Hessian alone is 289 MB), so no explicit flush is done between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Newton steps/s & PCG iters/s on 1.5M-tet mesh; SpMV/assembly GB/s vs HBM peak"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured", d
    return 6650.0, "fallback", {}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, device_index):
        self.idx = device_index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if len(s) > 2 + k and s[2 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- roofline
def algorithmic_bytes(sizes, n_cg):
    """Algorithmic bytes per unit of work (SURVEY §8(d) formulas; fp64 values, int32 indices)."""
    nv, nt, nnzb = sizes["n_verts"], sizes["n_tets"], sizes["nnzb"]
    spmv = nnzb * 76 + 4 * (nv + 1) + 2 * 24 * nv
    pcg_iter = spmv + 11 * 24 * nv
    assembly = nt * (624 + 64) + nnzb * 72          # 78 unique doubles per tet + 16 slot ids + BSR write
    return {"spmv": spmv, "pcg_iter": pcg_iter, "assembly": assembly}


def load_fp64_peak(kind="dmma"):
    """FP64 peak (TFLOP/s) of the FP64 tensor cores (kind "dmma": the factorisation's tile GEMMs
    are mma.sync m8n8k4 f64) or of the scalar FMA pipe ("dfma": the Galerkin product)."""
    p = os.path.join(ROOT, "profiles", "fp64_peaks.json")
    if os.path.exists(p):
        return json.load(open(p))[kind + "_tflops"], f"measured {kind.upper()} (profiles/fp64_peaks.json)"
    return 37.2, "nominal: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz"


def load_traffic():
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of kernels captured
    with ncu --set full, committed under profiles/ (the bench itself never runs under ncu)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def phase_rooflines(phases, ab, ci, n_cg, hbm, peak_src, fp64_peak, fp64_src, traffic, jacobi=True):
    """Roofline of every phase with a defined algorithmic work unit: HBM bytes
    for the PCG iteration and the assembly, FP64 flops for the coarse factorisation and the
    Galerkin projection.  achieved = work per launch / measured average launch time."""
    out = {}

    def put(name, bound, work, unit, peak, src, kernel, per_launch_ms, n_launch_per_newton, newton):
        ach = work / (per_launch_ms * 1e-3) / (1e9 if unit == "GB/s" else 1e12)
        tr = traffic.get(kernel)
        out[name] = {"bound": bound, "kernel": kernel, "achieved": ach, "peak": peak, "unit": unit,
                     "frac": ach / peak, "peak_source": src,
                     "traffic": tr["dram_bytes"] if tr else None,
                     "work_per_launch": work, "avg_ms_per_launch": per_launch_ms,
                     "ms_per_newton": per_launch_ms * n_launch_per_newton}

    newton = max(phases["pcg"][1], 1)
    ms, n = phases["pcg"]
    if n and jacobi:   # (the two-level iteration adds restrict / triangular sweeps / lift: no HBM unit)
        put("pcg", "hbm", ab["pcg_iter"], "GB/s", hbm, peak_src, "k_pcg_spmv+k_pcg_update",
            ms / (n * n_cg), n_cg, newton)
    ms, n = phases["assembly"]
    if n:
        put("assembly", "hbm", ab["assembly"], "GB/s", hbm, peak_src, "k_assemble", ms / n, 1, newton)
    ms, n = phases["coarse_factor"]
    if n:
        put("coarse_factor", "tensor", ci["flops"], "TFLOP/s", fp64_peak, fp64_src, "k_chol_dataflow", ms / n, 1,
            newton)
    ms, n = phases["coarse_S"]
    if n and ci.get("galerkin_flops"):
        dfma, dfma_src = load_fp64_peak("dfma")
        put("coarse_S", "alu", ci["galerkin_flops"], "TFLOP/s", dfma, dfma_src, "k_galerkin_fused", ms / n, 1,
            newton)
    return out


# ----------------------------------------------------------------------------- scenes
def load_case(config, standin=False):
    from precompute.basis import cached_basis
    from precompute.mesh import make_scene
    s = make_scene(config)
    t0 = time.time()
    if standin:   # tools/hat_basis.py: a partition of unity on a handle lattice, NOT the paper's basis
        from tools.hat_basis import hat_basis
        b = hat_basis(s)
    else:
        b = cached_basis(s)
    return s, b, time.time() - t0


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


# ----------------------------------------------------------------------------- oracle (cpu)
def oracle_newton_iterations(s, b, k):
    """Times k COMPLETE Newton iterations of the oracle (as it stands) from contact_state:
    gradient, full PSD Hessian + assembly, S_a and S = B^T H B, dense Cholesky, both coarse
    stages, N_cg PCG iterations, CCD + inversion filters, every line-search evaluation and the
    update (oracle.solver.OracleSim.newton_iteration).  Returns (seconds per iteration, desc)."""
    from oracle import solver
    from precompute.mesh import contact_state
    sim = solver.OracleSim(s, b)
    sim.x, sim.v = contact_state(s)
    sim.begin_step()
    t0 = time.perf_counter()
    evals = []
    for _ in range(k):
        info = sim.newton_iteration()
        evals.append(info.ls_evals)
        if info.converged or info.ls_failed:
            break
    sec = (time.perf_counter() - t0) / len(evals)
    desc = (f"{len(evals)} complete oracle Newton iteration(s) on the full {s.name} mesh from a seeded contact "
            f"state (bottom 0.6 dhat above the ground, falling 0.5 m/s): gradient, full PSD Hessian and "
            f"assembly, S_a, S=B^T H B, Cholesky, coarse correction, {sim.n_cg} PCG iterations, CCD and "
            f"inversion filters, {sum(evals)} line-search energy evaluations, update")
    return sec, desc, len(evals)


def host_info():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "lscpu_model": model}


def threads_used():
    from oracle import fem
    return fem.n_threads()


# ----------------------------------------------------------------------------- main arms
def run_reference(args):
    """The reference arm of this tier: the oracle as it stands, on the host cores, timing
    min(K, 2) complete C4 Newton iterations (no warm-up: the oracle has no caches or JIT)."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    s, b, _ = load_case(args.config)
    k = max(1, min(args.steps, 2))
    sec, desc, done = oracle_newton_iterations(s, b, k)
    value = 1.0 / sec
    line = {"metric": METRIC, "value": value, "unit": "Newton steps/s", "impl": "reference",
            "n_gpus": world, "steps": done, "warmup": 0, "ms_per_step": 1e3 * sec,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(s, b, 1),
            "note": f"requested --steps {args.steps} --warmup {args.warmup}; the oracle times {done} "
                    "complete Newton iteration(s) so the run ends within minutes",
            "cpu_baseline": dict({"value": value, "unit": "Newton steps/s", "cores": threads_used(),
                                  "kind": "oracle", "sample": desc}, **host_info()),
            "e2e": {"value": value, "unit": "Newton steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_dict(s, b, world, partitioned=False):
    return {"workload": f"{s.name}: {s.dims[0]}x{s.dims[1]}x{s.dims[2]} cubes x6 tets = {s.n_tets} tets, "
                        f"{s.n_verts} vertices, m={b.m} handles, N_cg={b.n_cg}, IE h=1/60"
                        + (", ground barrier" if s.ground is not None else ", pinned end"),
            "n_tets": int(s.n_tets), "n_verts": int(s.n_verts), "m": int(b.m), "n_cg": int(b.n_cg),
            "parallelism": (f"slab{world}" if partitioned else f"replicas{world}") if world > 1
                           else ("slab1-nccl (diagnostic)" if partitioned else "single"),
            "l2_flush": "none: the per-step working set (BSR Hessian, staged element Hessians) exceeds the 126 MB L2"
                        if s.n_tets > 500000 else "none (small config: L2-resident, reported for completeness)"}


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2508_13386_b200 import msim
    s, b, t_basis = load_case(args.config, args.standin_basis)
    stream = torch.cuda.current_stream()
    partitioned = (world > 1 and not args.replicas) or args.nccl1
    coarse_mode = 1 if args.coarse == "pcg" else 0
    integrator = 1 if args.integrator == "bdf2" else 0
    extra = dict(coarse_mode=coarse_mode, integrator=integrator, use_cubature=int(args.cubature),
                 lag_hessian=int(args.lag), refine_mode=1 if args.refine == "two_level" else 0)
    if args.cubature:
        from precompute.cubature import cached_cubature
        extra["cubature"] = cached_cubature(s, b)
    if partitioned:
        # one problem over N GPUs: x-slab partition, NCCL halo exchange / allreduce inside the
        # library; rank 0 creates the NCCL id, broadcast over the process group
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(msim.nccl_unique_id()), dtype=torch.uint8))
        if world > 1:
            torch.distributed.broadcast(uid, src=0)
        ctx = msim.context_from_scene(s, b, device=local, stream=stream.cuda_stream, rank=rank, world=world,
                                      nccl_id=bytes(uid.cpu().numpy().tobytes()), **extra)
    else:
        ctx = msim.context_from_scene(s, b, device=local, stream=stream.cuda_stream, **extra)
    sizes = ctx.sizes()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- warm-up
    for _ in range(args.warmup):
        ctx.timestep()
    # ---- timed region (device resident, per-phase events OFF)
    launches0 = ctx.kernel_launches()
    newton = pcg = coarse_it = 0
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            st = ctx.timestep()
            newton += st.newton_iters
            pcg += st.pcg_iters
            coarse_it += st.coarse_iters
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.kernel_launches() - launches0
    # ---- second pass (not part of `value`): per-phase CUDA events for the breakdown/rooflines
    ctx.set_profiling(True)
    prof_newton = 0
    prof_pcg = 0
    for _ in range(min(args.steps, 10)):
        st = ctx.timestep()
        prof_newton += st.newton_iters
        prof_pcg += st.pcg_iters
    phases = ctx.phase_times()
    ctx.set_profiling(False)
    ms_t = torch.tensor([ms], device="cuda")
    cnt = torch.tensor([newton, pcg], device="cuda", dtype=torch.float64)
    if world > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
        # replicas: independent problems (counts add up); partitioned: one problem (same counts)
        torch.distributed.all_reduce(cnt, op=torch.distributed.ReduceOp.MAX if partitioned
                                     else torch.distributed.ReduceOp.SUM)
    ms_max = float(ms_t.item())
    newton_all, pcg_all = float(cnt[0].item()), float(cnt[1].item())

    # ---- end-to-end through the C-ABI with host buffers (H2D state, timestep, D2H state); the
    # host state lives in pinned memory (torch pin_memory, viewed as numpy)
    x_h = torch.zeros((s.n_verts, 3), dtype=torch.float64, pin_memory=True).numpy()
    v_h = torch.zeros((s.n_verts, 3), dtype=torch.float64, pin_memory=True).numpy()
    ctx.get_state(out=(x_h, v_h))
    e_newton = 0
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ctx.set_state(x_h, v_h)
        st = ctx.timestep()
        e_newton += st.newton_iters
        if partitioned:
            x_h.fill(0.0)
            v_h.fill(0.0)
        ctx.get_state(out=(x_h, v_h))
        if partitioned and world > 1:   # every rank returns its owned vertices: assemble the global state
            xv = torch.from_numpy(np.concatenate([x_h.ravel(), v_h.ravel()])).cuda()
            torch.distributed.all_reduce(xv)
            xv = xv.cpu().numpy()
            x_h[...] = xv[:x_h.size].reshape(x_h.shape)
            v_h[...] = xv[x_h.size:].reshape(v_h.shape)
    barrier()
    e_sec = time.perf_counter() - t0
    e_t = torch.tensor([e_sec], device="cuda")
    e_c = torch.tensor([float(e_newton)], device="cuda", dtype=torch.float64)
    if world > 1:
        torch.distributed.all_reduce(e_t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(e_c, op=torch.distributed.ReduceOp.MAX if partitioned
                                     else torch.distributed.ReduceOp.SUM)

    if rank == 0:
        hbm, peak_src, peaks = load_peaks()
        ab = algorithmic_bytes(sizes, b.n_cg)
        pcg_ms, pcg_n = phases["pcg"]
        pcg_iter_ms = pcg_ms / max(pcg_n * b.n_cg, 1)
        asm_ms, asm_n = phases["assembly"]
        asm_avg = asm_ms / max(asm_n, 1)
        achieved = ab["pcg_iter"] / (pcg_iter_ms * 1e-3) / 1e9
        ci = ctx.coarse_info()
        fp64_peak, fp64_src = load_fp64_peak()
        traffic = load_traffic()
        rl_phases = phase_rooflines(phases, ab, ci, b.n_cg, hbm, peak_src, fp64_peak, fp64_src, traffic,
                                    jacobi=args.refine == "jacobi")
        dominant = max(rl_phases, key=lambda k: rl_phases[k]["ms_per_newton"] if rl_phases[k]["ms_per_newton"] else 0)
        line = {
            "metric": METRIC, "value": newton_all / (ms_max * 1e-3), "unit": "Newton steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if partitioned else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_dict(s, b, world, partitioned), coarse=args.coarse, integrator=args.integrator,
                           basis="stand-in trilinear-hat partition of unity (tools/hat_basis.py)"
                           if args.standin_basis else "paper: k-means partition + bilaplacian weights",
                           cubature=bool(args.cubature), lag_hessian=bool(args.lag), refine=args.refine),
            "pcg_iters_per_s": pcg_all / (ms_max * 1e-3),
            "newton_iters": int(newton_all),
            "pcg_iters_per_newton": pcg_all / max(newton_all, 1),
            "coarse_pcg_iters_per_newton": coarse_it / max(newton, 1) if args.coarse == "pcg" else None,
            "roofline": dict(rl_phases[dominant], phase=dominant),
            "roofline_phases": rl_phases,
            "assembly_gbs": ab["assembly"] / (asm_avg * 1e-3) / 1e9 if asm_n else None,
            "phase_ms_per_newton": {k: (v[0] / max(prof_newton, 1)) for k, v in phases.items()},
            "phase_pass": f"phase times from a second profiled pass of {min(args.steps, 10)} timesteps "
                          f"({prof_newton} Newton iterations) after the timed region",
            "gpu_launches": int(launches),
            "e2e": {"value": float(e_c.item()) / float(e_t.item()), "unit": "Newton steps/s",
                    "h2d_bytes_per_step": 2 * 3 * 8 * (sizes["n_verts"] if partitioned else s.n_verts),
                    "d2h_bytes_per_step": 2 * 3 * 8 * (sizes["n_verts"] if partitioned else s.n_verts)},
            "clocks": clk.summary(),
            "basis_build_s": t_basis,
            "coarse": ci,
        }
        if not args.no_cpu_baseline:
            sec, desc, _ = oracle_newton_iterations(s, b, 1)
            line["cpu_baseline"] = dict({"value": 1.0 / sec, "unit": "Newton steps/s", "cores": threads_used(),
                                         "kind": "oracle", "sample": desc}, **host_info())
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--coarse", default="exact", choices=["exact", "pcg"],
                    help="coarse solves: exact Cholesky of S (default) or the paper's block-Jacobi PCG to 1e-4")
    ap.add_argument("--cubature", action="store_true",
                    help="NEXT-2: cubature subspace Hessian (precompute/cubature.py, cached under .cache/)")
    ap.add_argument("--lag", action="store_true", help="NEXT-2: lagged elastic Hessian for the refinement PCG")
    ap.add_argument("--integrator", default="ie", choices=["ie", "bdf2"],
                    help="time integrator: implicit Euler (default, the configs' own) or BDF2 (P:185-189)")
    ap.add_argument("--refine", default="jacobi", choices=["jacobi", "two_level"],
                    help="refinement PCG: N_cg Jacobi iterations (default, the paper's) or NEXT-4's two-level "
                         "PCG (Jacobi + SMS coarse correction every iteration) to 1e-4 ||g||")
    ap.add_argument("--standin-basis", action="store_true",
                    help="use the stand-in basis of tools/hat_basis.py (C5 while its paper basis is not cached)")
    ap.add_argument("--nccl1", action="store_true",
                    help="N=1 diagnostic: run the partitioned code path over a one-rank NCCL communicator "
                         "(cost of the distributed path's collectives and captures on one GPU)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: N independent copies of the problem instead of one slab-partitioned problem")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
