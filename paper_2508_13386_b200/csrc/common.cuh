// Internal header of libmsim (B200 / sm_100a).  Not part of the C-ABI.
#pragma once

#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "msim.h"
#include "dist.h"

namespace msim {

// ---------------------------------------------------------------- error handling
struct Error {
  ms_status code;
  std::string msg;
};

#define MS_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t _e = (call);                                                                \
    if (_e != cudaSuccess)                                                                  \
      throw ::msim::Error{_e == cudaErrorMemoryAllocation ? MS_ERR_OOM : MS_ERR_CUDA,       \
                          std::string(#call) + ": " + cudaGetErrorString(_e)};              \
  } while (0)

#define MS_REQUIRE(cond, code, msg)                                                         \
  do {                                                                                      \
    if (!(cond)) throw ::msim::Error{(code), (msg)};                                        \
  } while (0)

// ---------------------------------------------------------------- device buffer
template <typename T>
struct DBuf {
  T *p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    if (count == 0) return;
    MS_CUDA(cudaMalloc((void **)&p, count * sizeof(T)));
    n = count;
    // debugging aid (MSIM_POISON=1): fresh buffers hold NaN / -1 instead of whatever the allocator
    // hands back, so a read of memory nothing wrote shows up in every run, not by allocation luck
    static const bool poison = std::getenv("MSIM_POISON") != nullptr;
    if (poison) {
      MS_CUDA(cudaMemset(p, 0xFF, count * sizeof(T)));
      MS_CUDA(cudaDeviceSynchronize());
    }
  }
  void upload(const T *h, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) MS_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T> &h, cudaStream_t s) { upload(h.data(), h.size(), s); }
  void zero(cudaStream_t s) {
    if (n) MS_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void download(T *h, size_t count, cudaStream_t s) const {
    if (count) MS_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  operator T *() const { return p; }
};

// Deterministic reduction workspace: per-CTA partials + a "last CTA" counter.
struct Reducer {
  DBuf<double> partial;       // [slots * max_blocks]
  DBuf<unsigned int> counter; // [n_counters]
};

// ---------------------------------------------------------------- tile Cholesky schedule
// staged element Hessian: 10 upper 3x3 blocks per tet, each padded to 10 doubles so every
// block starts 16-byte aligned (the assembly gathers it with 5 vector loads)
constexpr int kStageB = 10, kStageH = 10 * kStageB;
constexpr int kGalChunk = 128;   // vertices of U_i per Galerkin chunk (7-bit local index)
constexpr int kGalThreads = 2 * kGalChunk;
// shared memory of one Galerkin row CTA (galerkin.cuh): R chunk, staged entries, S accumulators
__host__ __device__ constexpr size_t galerkin_smem_doubles(int max_jup) {
  return (size_t)kGalChunk * 36 + (kGalThreads / 32) * (32 * 4 + 16) + (size_t)max_jup * 144;
}

struct CholTask {      // one trailing update A_ij -= L_ik L_jk^T (tiles)
  int32_t i, j;
};

// ---------------------------------------------------------------- context
struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string last_error;
  ms_params params;
  int64_t launches = 0;

  // ---- mesh
  int32_t nv = 0, nt = 0;           // local (owned + ghost) vertices / tets
  // ---- multi-GPU slab partition (dist.h); world == 1: everything owned
  Partition part;
  Comm *comm = nullptr;             // owned by the context (world > 1)
  int32_t nv_own = 0, nt_own = 0, nv_glob = 0;
  std::vector<int32_t> h_tets_glob; // global connectivity (world > 1: the global S pattern)
  std::vector<int32_t> h_sptr_glob, h_scol_glob;
  DBuf<int32_t> halo_send_idx, halo_recv_idx;
  DBuf<double> halo_send, halo_recv;
  // interior owned rows [int_lo, int_hi): no ghost column, so their SpMV rows need no halo and
  // run while the halo of z is in flight on halo_stream (int_lo == int_hi: no overlap)
  int32_t int_lo = 0, int_hi = 0;
  cudaStream_t halo_stream = nullptr;
  cudaEvent_t ev_z = nullptr, ev_halo = nullptr;
  // the partitioned code path: world > 1, or world == 1 with an explicit communicator (ms_create with
  // an nccl_id: one rank owning everything runs the NCCL collectives and their graph captures)
  bool dist() const { return part.world > 1 || comm != nullptr; }
  std::vector<double> h_X;          // rest positions (host copy)
  std::vector<double> h_Xg, h_Eg, h_rhog;   // global rest positions (world > 1) / per-tet E, rho
  std::vector<int32_t> h_dbc_glob;          // global Dirichlet vertex ids (ms_basis_build)
  struct BasisOutput *built_basis = nullptr;   // last ms_basis_build result (ms_basis_export)
  std::vector<int32_t> h_tets;
  DBuf<double> X;                   // (nv,3)
  DBuf<int32_t> tets;               // (nt,4)
  DBuf<double> Bm;                  // SoA [9][nt]  (Dm^-1 row-major)
  DBuf<double> vol, mu, lam;        // [nt]
  DBuf<double> mass;                // [nv]
  DBuf<uint8_t> fixed;              // [nv] 1 = Dirichlet
  std::vector<uint8_t> h_fixed;
  DBuf<int32_t> vinc_ptr, vinc;     // vertex -> (tet*4 + corner), CSR
  // BSR pattern (3x3 blocks)
  int64_t nnzb = 0;
  std::vector<int32_t> h_rowptr, h_colidx;
  DBuf<int32_t> rowptr, colidx, diag_slot, slot_row;
  DBuf<int32_t> diag_pos;           // [nv] SELL position of the diagonal block of each row
  DBuf<int32_t> cptr, contrib;      // slot -> list of (tet*16 + a*4 + b)
  DBuf<double> vals;                // SELL-32 values [npos/32][9][32] (sell.cuh)
  int64_t npos = 0;                 // SELL positions (nnzb + padding)
  DBuf<int32_t> sl_ptr, sell_col, sell_slot;
  std::vector<int64_t> h_sell_pos;  // CSR slot -> SELL position
  DBuf<double> dinv;                // [3 nv] Jacobi D^-1
  // ---- NEXT-2: cubature subspace Hessian and lagged refinement Hessian
  DBuf<double> tet_scale;           // [nt] w_e / V_e on cubature elements, 0 elsewhere
  DBuf<int32_t> cub_tets;           // local ids of the cubature elements
  int32_t n_cub = 0;
  DBuf<int32_t> cptr_c, contrib_c;  // per BSR slot: contributions of cubature elements only
  DBuf<double> vals_s;              // SELL values of the subspace Hessian when it differs from H_ref
  DBuf<double> lag_diag;            // [nv][9] alpha h^2 elastic part of the lagged diagonal blocks
  bool lag_valid = false;
  int32_t step_iter = 0, lag_last_refresh = 0, lag_refreshes = 0;
  std::vector<double> step_alphas;
  bool separate_sub() const { return params.use_cubature || params.lag_hessian; }
  const double *vals_sub() const { return separate_sub() ? vals_s.p : vals.p; }
  // ground
  bool has_ground = false;
  double gn[3] = {0, 0, 1}, goff = 0, dhat = 1e-3, kappa = 0;

  // ---- state
  DBuf<double> x, v, xt, xhat;      // (nv,3)
  DBuf<double> x_prev, v_prev;      // (nv,3) BDF2 history x^{t-1}, v^{t-1}
  bool has_history = false;         // a previous step exists (BDF2 can be used)
  double alpha = 1.0;               // IP scaling of the current step: 1 (IE) or 4/9 (BDF2), Eq. 2
  double ah2() const { return alpha * params.h * params.h; }
  DBuf<double> g, ds, da, df, d, r, rhs;   // 3nv
  DBuf<double> p, q, z, tmp;               // PCG vectors
  DBuf<double> stage_g;             // [nt*12] element gradients (unscaled by h^2)
  DBuf<double> stage_h;             // [nt*kStageH] 10 upper 3x3 blocks of P+(H_e), kStageB apart
  DBuf<int32_t> hess_work;          // [nt] tets whose reduced Hessian needs the eigen-clamp
  DBuf<unsigned int> hess_nwork;    // [1] their count
  bool step_begun = false;
  bool assembled = false;
  bool coarse_ready = false;

  // ---- basis
  int32_t m = 0;
  int32_t n_cg_basis = 20;
  int64_t nnz_phi = 0;
  DBuf<double> origins;             // (m,3)
  DBuf<int32_t> bvptr, bhandle;     // vertex-major CSR
  DBuf<double> bphi;
  DBuf<int32_t> hptr, hvert;        // handle-major CSR
  DBuf<double> hphi;
  DBuf<double> phi_aff;             // [nv]
  double aff_origin[3] = {0, 0, 0};
  // coarse S pattern: block CSR over handles (both triangles), 144 doubles per block
  int64_t nnzb_S = 0;
  std::vector<int32_t> h_sptr, h_scol;
  DBuf<int32_t> sptr, scol, srow, sT;   // sT[b]: block index of the transposed block
  DBuf<double> Sblk;                // [nnzb_S * 144]
  DBuf<double> Wphi;                // [nnz_phi * 4] phi [1, X - c] per basis entry
  DBuf<double> ga_w, gl_w;          // [|ga| * 4], [|gl| * 4]: the W rows of the Galerkin list entries,
                                    // gathered once per basis (no dependent gather in the kernel)
  // fused Galerkin (coarse.cu k_galerkin_fused): U_i lists, upper S slots, chunked entries
  DBuf<int32_t> gU_ptr, gU;         // [m+1], [sum |U_i|]
  DBuf<int32_t> ga_off;             // [sum |U_i| + 1] per (i,u) pair: range in ga_ent
  DBuf<uint32_t> ga_ent;            // Hessian row slot j of u | (basis entry p of (v, i)) << 6
  DBuf<unsigned long long> ga_mask; // per (i,u) pair: bit j set if slot j is listed
  DBuf<int32_t> gj_ptr, gj_blk;     // upper slots j >= i of row i -> S block index
  DBuf<int32_t> gl_base, gl_off;    // per (i, chunk, slot) entry ranges
  DBuf<uint32_t> gl_ent;            // u_local | (basis entry p) << 7
  int32_t gal_max_jup = 0;
  int32_t gal_parts = 4;            // CTAs per handle row (partial rows summed in a fixed order)
  DBuf<double> Spart;               // [m * gal_parts][144 gal_max_jup]
  DBuf<double> Sa;                  // 144
  DBuf<double> Ra;                  // [nv * 36]
  // dense coarse factor (tile-banded)
  int32_t nS = 0;                   // 12 m
  int32_t tile = 64;
  int32_t ntiles = 0;
  DBuf<double> Lden;                // [nS_pad * nS_pad] column-major lower factor
  int32_t nS_pad = 0;
  std::vector<std::vector<int32_t>> h_chol_panel;      // per k: tile rows i > k in struct
  DBuf<int32_t> chol_panel;
  std::vector<int64_t> h_chol_panel_off;
  std::vector<int32_t> h_perm;      // handle -> position in the nested-dissection order
  DBuf<int32_t> perm;
  DBuf<int32_t> chol_rows;          // per tile k: tile columns j < k with L_kj != 0 (flattened)
  std::vector<int64_t> h_chol_rows_off;
  double chol_flops = 0.0;          // flops of one factorisation (tile granularity)
  ms_coarse_info chol_info{};
  DBuf<int32_t> chol_rows_ptr, chol_panel_ptr, sym_tiles;
  int64_t n_sym_tiles = 0;
  DBuf<double> Uinv;                // [ntiles][64*64] U_kk = L_kk^-T (column-major)
  DBuf<int32_t> chol_dag;           // dataflow factorisation tasks (int4 each)
  DBuf<int32_t> chol_crit;          // task ids run by CTA 0 in order (the type-4 chain)
  DBuf<uint8_t> chol_cls;           // per task: 0/1 low/high-priority queue, 2 CTA 0's list
  DBuf<int32_t> chol_succ_ptr, chol_succ_mid, chol_succ;   // successors (setup.cpp dataflow_graph)
  DBuf<int32_t> chol_ndep0, chol_ndep;                     // inputs per task: pristine / live
  DBuf<int32_t> chol_queue0, chol_queue;                   // two ready queues: pristine / live
  int64_t n_crit = 0, n_pool = 0;
  bool gal_fused = false;           // Galerkin row tasks inside the factorisation launch (chol.cu)
  // ---- coarse_mode == MS_COARSE_PCG (coarse.cu): block-Jacobi PCG on the matrix-free sandwich
  std::vector<int64_t> h_bvptr;     // host copies of the (local) vertex-major basis CSR
  std::vector<int32_t> h_bhandle;
  bool cpcg_ready = false;          // diagonal-block Galerkin lists built (lazily)
  DBuf<int32_t> gd_U_ptr, gd_U, gd_ga_off, gd_gj_ptr, gd_gj_blk, gd_gl_base, gd_gl_off, gd_sT;
  DBuf<uint32_t> gd_ga_ent, gd_gl_ent;
  DBuf<unsigned long long> gd_ga_mask;
  DBuf<double> Sdiag, Sdiag_part, Minv;   // [m][144] blocks S_ii, their partial rows, S_ii^-1
  DBuf<double> cp_r, cp_z, cp_p, cp_t;    // [12m] PCG vectors (the solution goes to zs)
  DBuf<int32_t> cp_state;           // [2]: done flag, iterations
  cudaGraphExec_t cpcg_graph = nullptr;
  int64_t cpcg_graph_kernels = 0;
  int32_t coarse_iters_last = 0;
  // ---- refine_mode == MS_REFINE_TWO_LEVEL (coarse.cu): PCG with the two-level preconditioner
  DBuf<int32_t> tl_state;           // [2]: done flag, iterations
  cudaGraphExec_t tl_graph = nullptr;
  int64_t tl_graph_kernels = 0;
  int32_t refine_iters_last = 0;
  int64_t n_dag_factor = 0;         // factor tasks (the fused Galerkin tasks follow them)
  DBuf<int32_t> chol_rw_ptr, chol_rw;   // per chain task: handles whose R(i) it waits for
  int df_hi_ctas = 64;   // CTAs serving the high-priority queue
  int df_per_sm = 1;     // dataflow factorisation CTAs per SM (chol_init_attrs)
  int64_t n_dag = 0;
  DBuf<int> df_flags;               // upd[NT*NT], pfl[NT*NT], dfl[NT]
  int coop_grid = 148;
  cudaGraphExec_t factor_graph = nullptr, solve_graph = nullptr;
  int64_t factor_graph_kernels = 0, solve_graph_kernels = 0;
  DBuf<double> qa, qs, za, zs, yp;  // coarse vectors (qs/yp: permuted work space)
  DBuf<double> xsol;                // [nS_pad] permuted solution of the backward sweep
  DBuf<int32_t> flags;              // [8]: 0 = chol not SPD (S), 1 = not SPD (Sa), 2 = infeasible

  // ---- scalars / reductions
  DBuf<double> scal;                // device scalars (see SC_* in kernels)
  DBuf<double> partial;             // reduction partials
  DBuf<unsigned int> counters;
  double *h_pinned = nullptr;       // pinned host mirror of result scalars
  int max_blocks = 0;

  // ---- line search
  DBuf<double> ls_alpha;            // [ls_batch] candidate steps
  DBuf<double> ls_out;              // [ls_batch] energy differences

  // ---- graphs
  cudaGraphExec_t pcg_graph = nullptr;
  int64_t pcg_graph_kernels = 0;
  int32_t pcg_graph_iters = -1;

  // ---- profiling: (phase, start, end) event triples resolved lazily (no sync in the path)
  bool profiling = false;
  ms_phase_times ptimes{};
  struct PhaseRec { int phase; cudaEvent_t a, b; };
  std::vector<PhaseRec> prec;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  int cur_phase = -1;
};

// scalar slots in ctx.scal
enum {
  SC_RZ = 0,      // r^T z
  SC_RZ_OLD,
  SC_PQ,
  SC_ALPHA,
  SC_BETA,
  SC_ENERGY_ELEM, // sum V Psi                  \ summed across ranks together
  SC_ENERGY_VERT, // inertia + barrier          |  (k_vertex_grad writes 3 consecutive slots)
  SC_GNORM2,      //                            |
  SC_INFEAS_V,    // penetrating free vertices  |
  SC_INFEAS,      // >0 if an element is inverted at entry
  SC_DSNORM2,
  SC_ALPHA_CCD,   // \ min across ranks
  SC_ALPHA_INV,   // /
  SC_ALPHA0,
  SC_RZ0,
  SC_CG_G = 16,   // \ multi-GPU single-reduction PCG: gamma = r.z, delta = z.Hz (summed together)
  SC_CG_D,        // /
  SC_CG_GOLD,
  SC_CG_AOLD,
  SC_CP_RHO,      // coarse PCG (MS_COARSE_PCG): r.z, ||b||^2
  SC_CP_BN2,
  SC_TL_RZ,       // two-level refinement PCG (NEXT-4): r.z, r.r (summed together)
  SC_TL_RR,
  SC_CG_DI,       // multi-GPU PCG: z.Hz over the interior rows (added by the boundary launch)
  SC_COUNT = 32
};
constexpr int SC_SUM0 = SC_ENERGY_ELEM, SC_SUM_N = SC_INFEAS - SC_ENERGY_ELEM + 1;

// pinned host mirror layout
enum {
  PH_ENERGY = 0, PH_GNORM2, PH_DSNORM2, PH_ALPHA0, PH_INFEAS, PH_FLAG_S, PH_FLAG_SA,
  PH_RZ0, PH_RZ, PH_LS = 16, PH_COUNT = 128
};

// ---------------------------------------------------------------- launch helpers
constexpr int kMaxLS = 16;

inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// raise a kernel's dynamic shared-memory opt-in to the device maximum (minus its static shared
// memory); per device, so called per context on its device (create_common)
inline void set_max_dyn_smem(const void *func, int device) {
  int optin = 0;
  MS_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  cudaFuncAttributes fa;
  MS_CUDA(cudaFuncGetAttributes(&fa, func));
  MS_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes));
}

// kernels (defined in the .cu files); every launcher increments ctx.launches
void launch_elem_grad(Ctx &c);
void launch_elem_hess(Ctx &c);
void launch_eval_elements(Ctx &c, const double *x_dev, double *Ee, double *ge, double *He);
void launch_vertex_grad(Ctx &c);
void launch_assemble(Ctx &c);
void launch_assemble_sub(Ctx &c);      // the subspace Hessian (cubature / fresh) into vals_s
void launch_lag_diag(Ctx &c);          // H_lag diagonal blocks: frozen elastic part + fresh inertia / barrier
void launch_elem_hess_list(Ctx &c);    // element Hessians of the cubature elements only
void build_cubature_structures(Ctx &c, const std::vector<int32_t> &loc_elems, const std::vector<double> &w);
void launch_spmv(Ctx &c, const double *xin, double *yout, double alpha_minus_b, const double *b,
                 const int32_t *skip = nullptr, const double *vals = nullptr);
void launch_pcg(Ctx &c, const double *rhs, double *sol, int iters);
int launch_refine_two_level(Ctx &c, const double *rhs, double *sol);   // NEXT-4; returns iterations
void launch_pcg_spmv(Ctx &c, const int32_t *skip);
void launch_pcg_init(Ctx &c, const double *rhs, double *sol);   // x = 0, r = rhs, z = D^-1 r, p = q = 0   // one fused p / q update + p.q -> alpha
void pcg_reset_graph(Ctx &c);
void launch_coarse_S(Ctx &c, bool full_S = false);
// multi-GPU helpers (abi.cpp): no-ops when world == 1
void dist_sum(Ctx &c, double *dev, int64_t n);
void dist_min(Ctx &c, double *dev, int64_t n);
void halo_exchange(Ctx &c, double *vec);   // ghost entries of a 3-per-vertex vector <- owners
void launch_coarse_factor(Ctx &c);
void launch_coarse_direction(Ctx &c);
void launch_coarse_solve(Ctx &c);
void launch_basis_W(Ctx &c);
void enqueue_chol_factor(Ctx &c);
void enqueue_chol_solve(Ctx &c, const int32_t *skip = nullptr);
int64_t chol_factor_kernels(const Ctx &c);
int64_t chol_solve_kernels(const Ctx &c);
void chol_init_attrs(Ctx &c);
void coarse_init_attrs(Ctx &c);
void elem_init_attrs(Ctx &c);
void coarse_reset_graphs(Ctx &c);
void launch_lift(Ctx &c, const double *q, double *w, bool accumulate, const int32_t *skip = nullptr);
void launch_restrict(Ctx &c, const double *y, double *z, const int32_t *skip = nullptr);
void launch_filters(Ctx &c);
void launch_ls_batch(Ctx &c, int k0, int K);
void launch_update(Ctx &c, double alpha);
void launch_predictor(Ctx &c);
void launch_velocity(Ctx &c);
void launch_axpby(Ctx &c, double *y, double a, const double *x, double b, int64_t n);
void launch_dot(Ctx &c, const double *a, const double *b, int64_t n, int slot);
void launch_copy_scalars_to_host(Ctx &c);

// host-side symbolic setup (setup.cpp)
void build_mesh_structures(Ctx &c, const double *X, const int32_t *tets, const double *E,
                           const double *nu, const double *rho);
void global_s_pattern(int32_t nv, const std::vector<int32_t> &tets, int32_t m, const int64_t *vptr,
                      const int32_t *handle, std::vector<int32_t> &sptr, std::vector<int32_t> &scol);
void build_basis_structures(Ctx &c, int32_t m, const double *origins, const int64_t *vptr,
                            const int32_t *handle, const double *phi, const double *phi_aff,
                            const double aff_origin[3]);
void ensure_state_buffers(Ctx &c);
void build_coarse_pcg_structures(Ctx &c);

// profiling helpers
void phase_begin(Ctx &c, int phase);
void phase_end(Ctx &c);

}  // namespace msim
