"""ctypes binding of libmsim (include/msim.h): argument marshalling only.

Every computation runs in the CUDA library; this module converts numpy arrays to pointers,
checks status codes and raises on errors.  There is no CPU fallback: if the shared library is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libmsim.so")

MS_OK, MS_WARN_LS_FAILED, MS_WARN_NEWTON_CAP = 0, 1, 2
PHASES = ["grad", "hess", "assembly", "coarse_S", "coarse_factor", "coarse_solve", "pcg", "linesearch"]


class MsimError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"msim error {code}: {msg}")
        self.code = code


class Params(C.Structure):
    _fields_ = [("h", C.c_double), ("gravity", C.c_double * 3), ("eps", C.c_double),
                ("max_newton", C.c_int32), ("n_cg", C.c_int32), ("ls_shrink", C.c_double),
                ("ls_min", C.c_double), ("filter_safety", C.c_double), ("ls_batch", C.c_int32),
                ("use_graphs", C.c_int32), ("debug_flags", C.c_int32), ("coarse_mode", C.c_int32),
                ("coarse_max_iter", C.c_int32), ("coarse_tol", C.c_double), ("use_cubature", C.c_int32),
                ("lag_hessian", C.c_int32), ("integrator", C.c_int32), ("refine_mode", C.c_int32),
                ("refine_max_iter", C.c_int32), ("refine_tol", C.c_double)]


class NewtonStats(C.Structure):
    _fields_ = [("alpha", C.c_double), ("alpha0", C.c_double), ("ds_norm", C.c_double),
                ("energy", C.c_double), ("delta_energy", C.c_double), ("grad_norm", C.c_double),
                ("ls_evals", C.c_int32), ("converged", C.c_int32), ("ls_failed", C.c_int32),
                ("n_cg", C.c_int32), ("coarse_iters", C.c_int32), ("pad_", C.c_int32)]


class StepStats(C.Structure):
    _fields_ = [("newton_iters", C.c_int32), ("pcg_iters", C.c_int32), ("ls_evals", C.c_int32),
                ("status", C.c_int32), ("coarse_iters", C.c_int32), ("pad_", C.c_int32),
                ("last_ds_norm", C.c_double), ("last_alpha", C.c_double)]


class PhaseTimes(C.Structure):
    _fields_ = [("ms", C.c_double * 8), ("count", C.c_int64 * 8)]


class CoarseInfo(C.Structure):
    _fields_ = [("n_s", C.c_int64), ("tile", C.c_int64), ("ntiles", C.c_int64), ("lower_tiles", C.c_int64),
                ("n_tasks", C.c_int64), ("critical_path", C.c_int64), ("nnzb_s", C.c_int64),
                ("critical_path_xorder", C.c_int64), ("critical_path_nd", C.c_int64),
                ("ordering", C.c_int32), ("pad_", C.c_int32), ("flops", C.c_double),
                ("flops_xorder", C.c_double), ("flops_nd", C.c_double), ("galerkin_flops", C.c_double)]


class BasisInfo(C.Structure):
    _fields_ = [("m", C.c_int32), ("n_cg", C.c_int32), ("n_holes", C.c_int32), ("pad_", C.c_int32),
                ("nnz_phi", C.c_int64), ("hop_radius", C.c_double), ("t_kmeans", C.c_double),
                ("t_connect", C.c_double), ("t_solve", C.c_double), ("t_total", C.c_double)]


class PcgStats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("rz0", C.c_double), ("rz", C.c_double)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libmsim.so not built ({LIB_PATH}); run python -m paper_2508_13386_b200.build")
    lib = C.CDLL(LIB_PATH)
    P, D, I32, I64 = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int64)
    sig = {
        "ms_version": ([], C.c_char_p),
        "ms_default_params": ([C.POINTER(Params)], None),
        "ms_create": ([C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int], C.c_int32),
        "ms_destroy": ([P], C.c_int32),
        "ms_last_error": ([P], C.c_char_p),
        "ms_upload_mesh": ([P, C.c_int64, D, C.c_int64, I32, D, D, D], C.c_int32),
        "ms_set_dirichlet": ([P, C.c_int64, I32], C.c_int32),
        "ms_set_ground": ([P, D, C.c_double, C.c_double, C.c_double], C.c_int32),
        "ms_set_params": ([P, C.POINTER(Params)], C.c_int32),
        "ms_get_params": ([P, C.POINTER(Params)], C.c_int32),
        "ms_basis_upload": ([P, C.c_int32, D, I64, I32, D, D, D, C.c_int32], C.c_int32),
        "ms_basis_build": ([P, C.c_int32, C.c_uint64, C.POINTER(BasisInfo)], C.c_int32),
        "ms_basis_export": ([P, D, I64, I32, D, D, D, I32, I32], C.c_int32),
        "ms_basis_compute": ([C.c_int64, D, C.c_int64, I32, D, D, C.c_int64, I32, C.c_int32, C.c_uint64,
                              C.POINTER(C.c_void_p), C.POINTER(BasisInfo)], C.c_int32),
        "ms_basis_copy": ([P, D, I64, I32, D, D, D, I32, I32], C.c_int32),
        "ms_basis_free": ([P], None),
        "ms_cubature_upload": ([P, C.c_int64, I32, D], C.c_int32),
        "ms_set_state": ([P, D, D], C.c_int32),
        "ms_get_state": ([P, D, D], C.c_int32),
        "ms_set_step_state": ([P, D, D, D], C.c_int32),
        "ms_get_step_state": ([P, D, D, D], C.c_int32),
        "ms_timestep": ([P, C.POINTER(StepStats)], C.c_int32),
        "ms_begin_step": ([P], C.c_int32),
        "ms_newton_step": ([P, C.POINTER(NewtonStats)], C.c_int32),
        "ms_end_step": ([P], C.c_int32),
        "ms_assemble": ([P, D], C.c_int32),
        "ms_get_gradient": ([P, D], C.c_int32),
        "ms_eval_elements": ([P, D, D, D, D], C.c_int32),
        "ms_export_bsr": ([P, I64, I32, I32, D], C.c_int32),
        "ms_spmv": ([P, D, D], C.c_int32),
        "ms_basis_apply": ([P, D, D], C.c_int32),
        "ms_basis_apply_t": ([P, D, D], C.c_int32),
        "ms_export_coarse": ([P, D, D], C.c_int32),
        "ms_subspace_direction": ([P, D, D], C.c_int32),
        "ms_get_direction": ([P, D, D], C.c_int32),
        "ms_pcg_solve": ([P, D, D, C.c_int32, C.POINTER(PcgStats)], C.c_int32),
        "ms_pcg_solve_dev": ([P, C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(PcgStats)], C.c_int32),
        "ms_set_profiling": ([P, C.c_int32], C.c_int32),
        "ms_get_phase_times": ([P, C.POINTER(PhaseTimes)], C.c_int32),
        "ms_kernel_launches": ([P], C.c_int64),
        "ms_get_sizes": ([P, I64, I64, I64, I32, I64, I64], C.c_int32),
        "ms_get_coarse_info": ([P, C.POINTER(CoarseInfo)], C.c_int32),
        "ms_nccl_unique_id": ([C.c_void_p], C.c_int32),
        "ms_hub_create": ([C.c_int32, C.POINTER(C.c_void_p)], C.c_int32),
        "ms_hub_destroy": ([C.c_void_p], C.c_int32),
        "ms_create_hub": ([C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int], C.c_int32),
        "ms_partition": ([C.c_int32, C.c_int32, C.c_int64, D, C.c_int64, I32, I32, I32, I32, I32, I32, I32],
                         C.c_int32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


lib = _load()


def _d(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _i32(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


def _i64(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int64))


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def default_params():
    p = Params()
    lib.ms_default_params(C.byref(p))
    return p


class Context:
    """One msim context (one GPU).  Methods map 1:1 onto the C-ABI entry points."""

    def __init__(self, device=0, stream=None, rank=0, world=1, nccl_id=None, hub=None):
        """world > 1: one context per rank/GPU over NCCL (nccl_id: 128 bytes from nccl_unique_id()
        on rank 0), or over an in-process Hub (one host thread per context, tests)."""
        h = C.c_void_p()
        if hub is not None:
            st = lib.ms_create_hub(C.byref(h), int(device), C.c_void_p(stream or 0), hub.h, int(rank), int(world))
        else:
            nid = None
            if nccl_id is not None:
                buf = (C.c_uint8 * 128).from_buffer_copy(bytes(nccl_id))
                nid = C.cast(buf, C.c_void_p)
            st = lib.ms_create(C.byref(h), int(device), C.c_void_p(stream or 0), nid, int(rank), int(world))
        if st != 0:
            raise MsimError(st, "ms_create failed")
        self.h = h
        self.rank, self.world = int(rank), int(world)
        self.n_verts = 0
        self.n_tets = 0
        self.m = 0

    def _chk(self, st, allow=(0,)):
        if st not in allow:
            msg = lib.ms_last_error(self.h).decode()
            raise MsimError(st, msg)
        return st

    def close(self):
        if self.h:
            lib.ms_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- setup
    def upload_mesh(self, X, tets, E, nu, rho):
        X = _f64(X, (-1, 3))
        tets = np.ascontiguousarray(tets, dtype=np.int32).reshape(-1, 4)
        E, nu, rho = _f64(E), _f64(nu), _f64(rho)
        self._chk(lib.ms_upload_mesh(self.h, len(X), _d(X), len(tets), _i32(tets), _d(E), _d(nu), _d(rho)))
        self.n_verts, self.n_tets = len(X), len(tets)

    def set_dirichlet(self, verts):
        v = np.ascontiguousarray(verts, dtype=np.int32)
        self._chk(lib.ms_set_dirichlet(self.h, len(v), _i32(v)))

    def set_ground(self, normal, offset, dhat, kappa):
        n = _f64(normal)
        self._chk(lib.ms_set_ground(self.h, _d(n), float(offset), float(dhat), float(kappa)))

    def set_params(self, **kw):
        p = Params()
        self._chk(lib.ms_get_params(self.h, C.byref(p)))
        for k, v in kw.items():
            if k == "gravity":
                for i in range(3):
                    p.gravity[i] = float(v[i])
            else:
                setattr(p, k, v)
        self._chk(lib.ms_set_params(self.h, C.byref(p)))

    def get_params(self):
        p = Params()
        self._chk(lib.ms_get_params(self.h, C.byref(p)))
        return p

    def basis_upload(self, m, origins, vptr, handle, phi, phi_affine, affine_origin, n_cg):
        o = _f64(origins, (-1, 3))
        vp = np.ascontiguousarray(vptr, dtype=np.int64)
        hd = np.ascontiguousarray(handle, dtype=np.int32)
        ph, pa, ao = _f64(phi), _f64(phi_affine), _f64(affine_origin)
        self._chk(lib.ms_basis_upload(self.h, int(m), _d(o), _i64(vp), _i32(hd), _d(ph), _d(pa), _d(ao), int(n_cg)))
        self.m = int(m)

    def basis_build(self, m, seed):
        """ms_basis_build: native basis construction + upload; returns (info dict, arrays dict)."""
        info = BasisInfo()
        self._chk(lib.ms_basis_build(self.h, int(m), C.c_uint64(int(seed)), C.byref(info)))
        self.m = int(info.m)
        out = _basis_arrays(self.n_verts, self.n_tets, info)
        self._chk(lib.ms_basis_export(self.h, _d(out["origins"]), _i64(out["vptr"]), _i32(out["handle"]),
                                      _d(out["phi"]), _d(out["phi_affine"]), _d(out["affine_origin"]),
                                      _i32(out["cluster"]), _i32(out["centroid_vertex"])))
        return {k: getattr(info, k) for k, _ in BasisInfo._fields_ if k != "pad_"}, out

    def cubature_upload(self, elements, weights):
        e = np.ascontiguousarray(elements, dtype=np.int32)
        w = _f64(weights)
        self._chk(lib.ms_cubature_upload(self.h, len(e), _i32(e), _d(w)))

    # ---------------------------------------------------------------- state
    def set_state(self, x=None, v=None):
        x = None if x is None else _f64(x, (-1, 3))
        v = None if v is None else _f64(v, (-1, 3))
        self._chk(lib.ms_set_state(self.h, _d(x), _d(v)))

    def get_state(self, out=None):
        """Global-sized arrays; with world > 1 only this rank's owned vertices are filled (rest 0).
        out = (x, v): C-contiguous float64 (n_verts, 3) arrays to fill (e.g. views of pinned host
        memory, so the device->host copies run at full PCIe rate)."""
        if out is None:
            x = np.zeros((self.n_verts, 3))
            v = np.zeros((self.n_verts, 3))
        else:
            x, v = out
            for a in (x, v):
                if a.dtype != np.float64 or a.shape != (self.n_verts, 3) or not a.flags.c_contiguous:
                    raise ValueError("get_state(out=...): C-contiguous float64 (n_verts, 3) arrays expected")
        self._chk(lib.ms_get_state(self.h, _d(x), _d(v)))
        return x, v

    def set_step_state(self, x_t, xhat, x):
        a, b, c = _f64(x_t, (-1, 3)), _f64(xhat, (-1, 3)), _f64(x, (-1, 3))
        self._chk(lib.ms_set_step_state(self.h, _d(a), _d(b), _d(c)))

    def get_step_state(self):
        a, b, c = (np.empty((self.n_verts, 3)) for _ in range(3))
        self._chk(lib.ms_get_step_state(self.h, _d(a), _d(b), _d(c)))
        return a, b, c

    # ---------------------------------------------------------------- hot path
    def timestep(self):
        s = StepStats()
        self._chk(lib.ms_timestep(self.h, C.byref(s)), allow=(0, 1, 2))
        return s

    def begin_step(self):
        self._chk(lib.ms_begin_step(self.h))

    def newton_step(self):
        s = NewtonStats()
        self._chk(lib.ms_newton_step(self.h, C.byref(s)), allow=(0, 1))
        return s

    def end_step(self):
        self._chk(lib.ms_end_step(self.h))

    # ---------------------------------------------------------------- hooks
    def assemble(self):
        e = np.zeros(1)
        self._chk(lib.ms_assemble(self.h, _d(e)))
        return float(e[0])

    def get_gradient(self):
        g = np.empty((self.n_verts, 3))
        self._chk(lib.ms_get_gradient(self.h, _d(g)))
        return g

    def eval_elements(self, x, energy=True, grad=True, hess=True):
        x = _f64(x, (-1, 3))
        Ee = np.empty(self.n_tets) if energy else None
        ge = np.empty((self.n_tets, 12)) if grad else None
        He = np.empty((self.n_tets, 12, 12)) if hess else None
        self._chk(lib.ms_eval_elements(self.h, _d(x), _d(Ee), _d(ge), _d(He)))
        return Ee, ge, He

    def export_bsr(self):
        nnzb = np.zeros(1, dtype=np.int64)
        self._chk(lib.ms_export_bsr(self.h, _i64(nnzb), None, None, None))
        rp = np.empty(self.n_verts + 1, dtype=np.int32)
        ci = np.empty(int(nnzb[0]), dtype=np.int32)
        vals = np.empty((int(nnzb[0]), 3, 3))
        self._chk(lib.ms_export_bsr(self.h, _i64(nnzb), _i32(rp), _i32(ci), _d(vals)))
        return rp, ci, vals

    def spmv(self, x):
        x = _f64(x, (-1,))
        y = np.empty_like(x)
        self._chk(lib.ms_spmv(self.h, _d(x), _d(y)))
        return y

    def basis_apply(self, q):
        q = _f64(q, (-1,))
        w = np.empty(3 * self.n_verts)
        self._chk(lib.ms_basis_apply(self.h, _d(q), _d(w)))
        return w

    def basis_apply_t(self, y):
        y = _f64(y, (-1,))
        z = np.empty(12 * self.m)
        self._chk(lib.ms_basis_apply_t(self.h, _d(y), _d(z)))
        return z

    def export_coarse(self, dense=True):
        S = np.empty((12 * self.m, 12 * self.m)) if dense else None
        Sa = np.empty((12, 12))
        self._chk(lib.ms_export_coarse(self.h, _d(S), _d(Sa)))
        return S, Sa

    def subspace_direction(self):
        ds = np.empty(3 * self.n_verts)
        da = np.empty(3 * self.n_verts)
        self._chk(lib.ms_subspace_direction(self.h, _d(ds), _d(da)))
        return ds, da

    def get_direction(self):
        ds = np.empty(3 * self.n_verts)
        df = np.empty(3 * self.n_verts)
        self._chk(lib.ms_get_direction(self.h, _d(ds), _d(df)))
        return ds, df

    def pcg_solve(self, rhs, iters):
        r = _f64(rhs, (-1,))
        sol = np.empty_like(r)
        st = PcgStats()
        self._chk(lib.ms_pcg_solve(self.h, _d(r), _d(sol), int(iters), C.byref(st)))
        return sol, st

    def pcg_solve_dev(self, rhs_ptr, sol_ptr, iters):
        st = PcgStats()
        self._chk(lib.ms_pcg_solve_dev(self.h, C.c_void_p(rhs_ptr), C.c_void_p(sol_ptr), int(iters), C.byref(st)))
        return st

    # ---------------------------------------------------------------- instrumentation
    def set_profiling(self, on):
        self._chk(lib.ms_set_profiling(self.h, 1 if on else 0))

    def phase_times(self):
        t = PhaseTimes()
        self._chk(lib.ms_get_phase_times(self.h, C.byref(t)))
        return {PHASES[i]: (t.ms[i], t.count[i]) for i in range(8)}

    def kernel_launches(self):
        return int(lib.ms_kernel_launches(self.h))

    def sizes(self):
        a = [np.zeros(1, dtype=np.int64) for _ in range(3)]
        m = np.zeros(1, dtype=np.int32)
        b = [np.zeros(1, dtype=np.int64) for _ in range(2)]
        self._chk(lib.ms_get_sizes(self.h, _i64(a[0]), _i64(a[1]), _i64(a[2]), _i32(m), _i64(b[0]), _i64(b[1])))
        return dict(n_verts=int(a[0][0]), n_tets=int(a[1][0]), nnzb=int(a[2][0]), m=int(m[0]),
                    nnz_phi=int(b[0][0]), nnzb_S=int(b[1][0]))


    def coarse_info(self):
        ci = CoarseInfo()
        self._chk(lib.ms_get_coarse_info(self.h, C.byref(ci)))
        return {k: getattr(ci, k) for k, _ in CoarseInfo._fields_ if k != "pad_"}


def _basis_arrays(nv, nt, info):
    mm, nnz = int(info.m), int(info.nnz_phi)
    return dict(origins=np.empty((mm, 3)), vptr=np.empty(nv + 1, dtype=np.int64),
                handle=np.empty(nnz, dtype=np.int32), phi=np.empty(nnz), phi_affine=np.empty(nv),
                affine_origin=np.empty(3), cluster=np.empty(nt, dtype=np.int32),
                centroid_vertex=np.empty(mm, dtype=np.int32))


def basis_compute(X, tets, E, rho, dbc, m, seed):
    """Host-only ms_basis_compute (no GPU): returns (info dict, arrays dict)."""
    X = _f64(X, (-1, 3))
    tets = np.ascontiguousarray(tets, dtype=np.int32).reshape(-1, 4)
    E, rho = _f64(E), _f64(rho)
    dbc = np.ascontiguousarray(dbc, dtype=np.int32)
    h = C.c_void_p()
    info = BasisInfo()
    st = lib.ms_basis_compute(len(X), _d(X), len(tets), _i32(tets), _d(E), _d(rho), len(dbc),
                              _i32(dbc) if len(dbc) else None, int(m), C.c_uint64(int(seed)), C.byref(h),
                              C.byref(info))
    if st != 0:
        raise MsimError(st, "ms_basis_compute failed")
    try:
        out = _basis_arrays(len(X), len(tets), info)
        st = lib.ms_basis_copy(h, _d(out["origins"]), _i64(out["vptr"]), _i32(out["handle"]), _d(out["phi"]),
                               _d(out["phi_affine"]), _d(out["affine_origin"]), _i32(out["cluster"]),
                               _i32(out["centroid_vertex"]))
        if st != 0:
            raise MsimError(st, "ms_basis_copy failed")
    finally:
        lib.ms_basis_free(h)
    return {k: getattr(info, k) for k, _ in BasisInfo._fields_ if k != "pad_"}, out


def nccl_unique_id():
    """128-byte ncclUniqueId for ms_create on every rank (call on rank 0, broadcast)."""
    buf = (C.c_uint8 * 128)()
    st = lib.ms_nccl_unique_id(buf)
    if st != 0:
        raise MsimError(st, "ms_nccl_unique_id failed")
    return bytes(buf)


def partition(rank, world, X, tets):
    """Host-only slab partition plan of `rank` (no GPU): dict with nv_own, nt_own, l2g (local ->
    global vertex; owned first), tet_l2g (owned tets first), and per peer rank the global ids
    sent to / received from it (sorted)."""
    X = _f64(X, (-1, 3))
    tets = np.ascontiguousarray(tets, dtype=np.int32).reshape(-1, 4)
    cnt = np.zeros(6, dtype=np.int32)
    st = lib.ms_partition(int(rank), int(world), len(X), _d(X), len(tets), _i32(tets), _i32(cnt),
                          None, None, None, None, None)
    if st != 0:
        raise MsimError(st, "ms_partition failed")
    nv_own, nv_loc, nt_own, nt_loc, n_send, n_recv = (int(v) for v in cnt)
    l2g = np.empty(nv_loc, dtype=np.int32)
    tl2g = np.empty(nt_loc, dtype=np.int32)
    peer = np.zeros((world, 2), dtype=np.int32)
    snd = np.empty(max(n_send, 1), dtype=np.int32)
    rcv = np.empty(max(n_recv, 1), dtype=np.int32)
    st = lib.ms_partition(int(rank), int(world), len(X), _d(X), len(tets), _i32(tets), _i32(cnt),
                          _i32(l2g), _i32(tl2g), _i32(peer), _i32(snd), _i32(rcv))
    if st != 0:
        raise MsimError(st, "ms_partition failed")
    send, recv, so, ro = {}, {}, 0, 0
    for q in range(world):
        if peer[q, 0]:
            send[q] = snd[so:so + peer[q, 0]].copy()
            so += peer[q, 0]
        if peer[q, 1]:
            recv[q] = rcv[ro:ro + peer[q, 1]].copy()
            ro += peer[q, 1]
    return dict(nv_own=nv_own, nt_own=nt_own, l2g=l2g, tet_l2g=tl2g, send=send, recv=recv)


class Hub:
    """In-process communicator for `world` contexts driven by `world` host threads."""

    def __init__(self, world):
        self.h = C.c_void_p()
        st = lib.ms_hub_create(int(world), C.byref(self.h))
        if st != 0:
            raise MsimError(st, "ms_hub_create failed")

    def __del__(self):
        try:
            if self.h:
                lib.ms_hub_destroy(self.h)
                self.h = None
        except Exception:
            pass


def context_from_scene(scene, basis, device=0, stream=None, rank=0, world=1, nccl_id=None, hub=None, cubature=None,
                       **params):
    """Create a context and upload a precompute.mesh.Scene + precompute.basis.Basis (+ optionally a
    precompute.cubature.Cubature for use_cubature)."""
    ctx = Context(device, stream, rank=rank, world=world, nccl_id=nccl_id, hub=hub)
    ctx.upload_mesh(scene.X, scene.tets, scene.E, scene.nu, scene.rho)
    if len(scene.dbc):
        ctx.set_dirichlet(scene.dbc)
    if scene.ground is not None:
        g = scene.ground
        ctx.set_ground(g["normal"], g["offset"], g["dhat"], g["kappa"])
    kw = dict(h=scene.h, gravity=scene.gravity, eps=scene.eps, max_newton=scene.max_newton)
    kw.update(params)
    ctx.set_params(**kw)
    ctx.basis_upload(basis.m, basis.origins, basis.vptr, basis.handle, basis.phi, basis.phi_affine,
                     basis.affine_origin, basis.n_cg)
    if cubature is not None:
        ctx.cubature_upload(cubature.elements, cubature.weights)
    return ctx
