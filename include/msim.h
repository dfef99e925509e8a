/*
 * msim.h — C-ABI of the B200-native multilevel elastodynamics Newton solve
 * (arXiv 2508.13386, "Sparse, Geometry- and Material-Aware Bases for Multilevel
 * Elastodynamic Simulation").  Library: paper_2508_13386_b200/lib/libmsim.so.
 *
 * Citations: "P:<line>" = PAPER.md line, "S:<line>" = SPEC.md line, R#/Q# = readings
 * listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Every pointer argument is a HOST pointer unless the name ends in `_dev`.  Host arrays
 *    are copied (or written) before the call returns; the caller keeps ownership.
 *  - Vectors over vertices are AoS xyz: element 3*v + c (c = x,y,z), fp64.  Indices int32.
 *  - All device work is enqueued on the CUDA stream passed to ms_create (e.g. torch's
 *    current stream), so callers and the library share ordering.  Calls that return host
 *    data synchronise that stream.
 *  - Return value: 0 OK; >0 soft warning (result valid); <0 hard error.  No C++ exception
 *    crosses the ABI.  ms_last_error() returns a message for the last non-zero status.
 *  - A context is single-GPU, single-thread (not thread-safe).
 */
#ifndef MSIM_H
#define MSIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ms_ctx ms_ctx;
typedef int32_t ms_status;

enum {
  MS_OK = 0,
  MS_WARN_LS_FAILED = 1,    /* line search fell below ls_min; iterate kept   */
  MS_WARN_NEWTON_CAP = 2,   /* max_newton iterations reached without convergence     */
  MS_ERR_ARG = -1,          /* invalid argument: index range, V<=0, E<=0, nu not in [0,.5)…  */
  MS_ERR_CUDA = -2,         /* CUDA runtime error                                             */
  MS_ERR_NCCL = -3,         /* reserved (multi-GPU)                                           */
  MS_ERR_NOT_SPD = -4,      /* coarse matrix not SPD (Cholesky pivot <= 0) (reading Q18)     */
  MS_ERR_COVERAGE = -5,     /* basis coverage hole: sum phi = 0 at a free vertex             */
  MS_ERR_OOM = -6,          /* device allocation failed                                       */
  MS_ERR_INFEASIBLE = -7,   /* inverted element or penetrating vertex at entry (E = +inf)    */
  MS_ERR_STATE = -8         /* call order violated (e.g. newton_step before begin_step)      */
};

/* Solver parameters.  Defaults (ms_default_params): h = 1/60, gravity (0,0,-9.8),
 * eps = 1e-6, max_newton = 100, n_cg = 0 (= basis heuristic), ls_shrink = 0.5,
 * ls_min = 1e-8, filter_safety = 0.9, ls_batch = 4, use_graphs = 1. */
typedef struct ms_params {
  double h;               /* timestep [s] (implicit Euler)                      */
  double gravity[3];      /* folded into the predictor xhat (reading R8)                   */
  double eps;             /* termination ||d_s||_2 / (h n_v) < eps (reading R7)     */
  int32_t max_newton;     /* Newton iteration cap per timestep                             */
  int32_t n_cg;           /* full-space Jacobi-PCG iterations; 0 = value from the basis   */
  double ls_shrink;       /* backtracking factor (reading Q12)                      */
  double ls_min;          /* smallest step tried before MS_WARN_LS_FAILED                  */
  double filter_safety;   /* CCD / inversion filter safety factor                          */
  int32_t ls_batch;       /* candidate step sizes evaluated per fused line-search pass     */
  int32_t use_graphs;     /* capture the fixed-count PCG loop in a CUDA graph              */
  int32_t debug_flags;    /* parity hooks, 0 in production: MS_DEBUG_HESS_FALLBACK routes
                             every indefinite element Hessian to the cyclic-Jacobi eigen-clamp
                             (the fall-back path of the tridiagonal-QL projection)           */
  int32_t coarse_mode;    /* MS_COARSE_EXACT (default): S = B^T H B formed and factorised
                             (reading R4); MS_COARSE_PCG: the paper's solves --
                             block-Jacobi PCG to coarse_tol on the matrix-free sandwich
                             B^T (H (B p)), 12 x 12 blocks S_ii (NEXT-1)                     */
  int32_t coarse_max_iter;/* MS_COARSE_PCG: iteration cap (default 1000)                     */
  double coarse_tol;      /* MS_COARSE_PCG: ||r||_2 <= coarse_tol ||b||_2 (default 1e-4)    */
  int32_t use_cubature;   /* NEXT-2: the subspace solves use the cubature Hessian
                             (elastic part over the ms_cubature_upload elements, weight w_e in
                             place of V_e; inertia and barrier exact); 0 = fully integrated (R3) */
  int32_t lag_hessian;    /* NEXT-2: the refinement PCG uses a lagged elastic Hessian
                             (refreshed at the first iteration of every step and when the mean of
                             the last 3 accepted step sizes < 0.2, at least 5 iterations apart;
                             inertia and barrier always fresh; reading C4)                    */
  int32_t integrator;     /* MS_INTEGRATOR_IE (default) or MS_INTEGRATOR_BDF2 (P:185-189:
                             alpha = 4/9, xhat = (4x^t - x^{t-1})/3 + (2h/9)(4v^t - v^{t-1}) +
                             alpha h^2 g, v^{t+1} = (4v^t - v^{t-1})/3 + (2h/3) a^{t+1} with
                             a^{t+1} = 9/(4h^2)(x^{t+1} - xtilde), reading C2; a step without
                             history -- the first after ms_set_state -- is implicit Euler)   */
  int32_t refine_mode;    /* full-space refinement d_f (Alg. 1): MS_REFINE_JACOBI
                             (default, reading R5: exactly n_cg Jacobi-PCG iterations) or
                             MS_REFINE_TWO_LEVEL (NEXT-4, not in the paper; reading N4): PCG with
                             y = D^-1 r, z = y + U_s S^-1 U_s^T (r - H y) (the factorised SMS
                             matrix of the Newton iteration) until ||r_k||_2 <= refine_tol ||g||_2 or
                             refine_max_iter iterations; needs MS_COARSE_EXACT                */
  int32_t refine_max_iter;/* MS_REFINE_TWO_LEVEL: iteration cap (default 100)                */
  double refine_tol;      /* MS_REFINE_TWO_LEVEL: relative residual (default 1e-2, an inexact-
                             Newton forcing term; 1e-4 needs ~100 iterations at C4)           */
} ms_params;
enum { MS_INTEGRATOR_IE = 0, MS_INTEGRATOR_BDF2 = 1 };
enum { MS_REFINE_JACOBI = 0, MS_REFINE_TWO_LEVEL = 1 };
enum { MS_COARSE_EXACT = 0, MS_COARSE_PCG = 1 };
enum { MS_DEBUG_HESS_FALLBACK = 1 };

typedef struct ms_newton_stats {
  double alpha;           /* accepted step (0 if the line search failed)                   */
  double alpha0;          /* min(1, CCD filter, inversion filter)                          */
  double ds_norm;         /* ||d_s||_2 over all 3 n_v DOFs                                  */
  double energy;          /* E(x) at the START of the iteration (Eq. 2)                    */
  double delta_energy;    /* E(x + alpha d) - E(x) of the accepted step                    */
  double grad_norm;       /* ||g||_2 at the start of the iteration                          */
  int32_t ls_evals;       /* number of candidate steps evaluated                           */
  int32_t converged;      /* termination test passed after this iteration                  */
  int32_t ls_failed;      /* 1 if no decrease down to ls_min                               */
  int32_t n_cg;           /* refinement PCG iterations performed (n_cg; MS_REFINE_TWO_LEVEL:
                             the iterations to refine_tol)                                    */
  int32_t coarse_iters;   /* MS_COARSE_PCG: SMS-stage PCG iterations (0 in exact mode)     */
  int32_t pad_;
} ms_newton_stats;

typedef struct ms_step_stats {
  int32_t newton_iters;   /* Newton iterations in this timestep                            */
  int32_t pcg_iters;      /* total full-space PCG iterations                               */
  int32_t ls_evals;       /* total line-search candidates evaluated                        */
  int32_t status;         /* MS_OK / MS_WARN_*                                              */
  int32_t coarse_iters;   /* MS_COARSE_PCG: total SMS-stage PCG iterations                 */
  int32_t pad_;
  double last_ds_norm;
  double last_alpha;
} ms_step_stats;

/* Accumulated device time (CUDA events on the library stream) per phase while profiling
 * is enabled (ms_set_profiling).  Index with the MS_PHASE_* constants. */
enum {
  MS_PHASE_GRAD = 0,      /* element energy+gradient + vertex gather   (rows a1-a2)   */
  MS_PHASE_HESS,          /* element Hessian + PSD projection          (row a3)       */
  MS_PHASE_ASSEMBLY,      /* BSR gather assembly + Jacobi diagonal     (row a4)       */
  MS_PHASE_COARSE_S,      /* B^T H B and U_a^T H U_a                   (row a5)       */
  MS_PHASE_COARSE_FACTOR, /* Cholesky of S and S_a                     (row a6)       */
  MS_PHASE_COARSE_SOLVE,  /* restrict / solve / lift / residual SpMVs  (row a7)       */
  MS_PHASE_PCG,           /* fixed-count Jacobi-PCG                    (row a8)       */
  MS_PHASE_LINESEARCH,    /* filters + batched energies + update       (row a9)       */
  MS_PHASE_COUNT
};
typedef struct ms_phase_times {
  double ms[MS_PHASE_COUNT];
  int64_t count[MS_PHASE_COUNT];
} ms_phase_times;

typedef struct ms_pcg_stats {
  int32_t iters;          /* iterations performed                                          */
  double rz0;             /* r0^T D^-1 r0                                                  */
  double rz;              /* final r^T D^-1 r                                              */
} ms_pcg_stats;

/* ---------------------------------------------------------------- lifecycle */
const char *ms_version(void);
void ms_default_params(ms_params *out);
/* Create a context on `device`, enqueuing on `cuda_stream` (a cudaStream_t; NULL = legacy
 * default stream).  Multi-GPU: one context per rank and GPU, SPMD; world > 1
 * needs nccl_id, the 128-byte ncclUniqueId that rank 0 obtained with ms_nccl_unique_id and
 * shared with the other ranks (world == 1: nccl_id may be NULL; a non-NULL id makes the single
 * rank run the partitioned path over a one-rank NCCL communicator).  Every rank then uploads the
 * full mesh and basis and makes the same calls in the same order; the context keeps an x-slab of
 * vertices (equal counts) plus one ghost layer, exchanges ghost values with its neighbours over
 * NCCL and sums energies, dot products, B^T r and S across ranks (dist.h).  State arrays
 * (ms_set_state / ms_get_state ...) stay global-sized: set reads the rank's local entries, get
 * writes its owned entries.  The parity hooks (ms_eval_elements, ms_export_bsr, ms_spmv, ...)
 * operate on the rank's local numbering. */
typedef struct ms_hub ms_hub;   /* in-process communicator (one-GPU tests of the world > 1 path) */
/* Fill out[128] with a fresh ncclUniqueId (rank 0, before ms_create). */
ms_status ms_nccl_unique_id(uint8_t out[128]);
/* In-process hub: `world` contexts created with ms_create_hub in one process (one host thread per
 * context) exchange ghost values and reductions through host memory; every collective
 * synchronises the calling stream (no device-side waiting between contexts). */
ms_status ms_hub_create(int32_t world, ms_hub **out);
ms_status ms_hub_destroy(ms_hub *hub);
ms_status ms_create_hub(ms_ctx **out, int device, void *cuda_stream, ms_hub *hub, int rank, int world);
/* Host-only (no GPU): the slab partition plan of `rank` that ms_upload_mesh builds (dist.h), for
 * tests and tooling.  counts[6] = nv_own, nv_loc, nt_own, nt_loc, n_send, n_recv; optional
 * outputs (NULL to skip): l2g[nv_loc] local -> global vertex (owned first), tet_l2g[nt_loc],
 * peer_counts[world][2] = (n_send, n_recv) per peer rank, send_global / recv_global = global
 * vertex ids concatenated by peer rank (ascending rank, ids ascending within a peer). */
ms_status ms_partition(int32_t rank, int32_t world, int64_t n_verts, const double *rest_xyz,
                       int64_t n_tets, const int32_t *tets, int32_t *counts, int32_t *l2g,
                       int32_t *tet_l2g, int32_t *peer_counts, int32_t *send_global,
                       int32_t *recv_global);
ms_status ms_create(ms_ctx **out, int device, void *cuda_stream, const uint8_t *nccl_id,
                    int rank, int world);
ms_status ms_destroy(ms_ctx *ctx);
const char *ms_last_error(ms_ctx *ctx);

/* ---------------------------------------------------------------- problem setup */
/* Tet mesh, rest positions (n_verts x 3) = initial positions, tets (n_tets x 4, positive
 * orientation), per-tet Young's modulus E [Pa], Poisson ratio nu, density rho
 * (S:22-31).  Builds the 3x3-block BSR pattern (vertex adjacency + diagonal), the
 * atomic-free assembly maps and the lumped mass m_v = sum rho V / 4 (Q9).
 * Errors: MS_ERR_ARG for out-of-range indices, V <= 0, E <= 0, nu outside [0,0.5), rho <= 0. */
ms_status ms_upload_mesh(ms_ctx *ctx, int64_t n_verts, const double *rest_xyz, int64_t n_tets,
                         const int32_t *tets, const double *E, const double *nu,
                         const double *rho);
/* Dirichlet vertices, pinned at their rest position (Q13: identity rows, g = 0).  Must precede
 * ms_basis_upload (MS_ERR_STATE afterwards): the basis is built for one Dirichlet set and has to
 * vanish at its vertices, which ms_basis_upload checks (MS_ERR_ARG otherwise). */
ms_status ms_set_dirichlet(ms_ctx *ctx, int64_t n, const int32_t *verts);
/* Ground-plane IPC barrier b(d) = -(d-dhat)^2 ln(d/dhat), d = normal.x - offset
 * (P:177); kappa is the barrier stiffness.  kappa <= 0 disables contact. */
ms_status ms_set_ground(ms_ctx *ctx, const double normal[3], double offset, double dhat,
                        double kappa);
ms_status ms_set_params(ms_ctx *ctx, const ms_params *p);
ms_status ms_get_params(ms_ctx *ctx, ms_params *p);

/* Upload the precomputed bases (Eq. 7):
 *  m handles with origins c_i (m x 3); per-vertex CSR (vptr[n_verts+1], handle[], phi[])
 *  of the SMS weights phi_i(v) > 0; the affine weight phi_a(v) = 1 - phi_DBC(v) and its
 *  origin (centre of mass); n_cg = refinement iterations from the hop heuristic.
 * The 3x12 block of vertex v and handle i is I3 kron (phi_i(v) [1, X_v - c_i]) with the 12
 * coordinates ordered [x-row(4), y-row(4), z-row(4)].  Builds the handle-major transpose,
 * the coupled-handle pattern of S = B^T H B and its Cholesky schedule.
 * Errors: MS_ERR_ARG (bad sizes / handle ids), MS_ERR_COVERAGE (sum phi + phi_DBC = 0). */
ms_status ms_basis_upload(ms_ctx *ctx, int32_t m, const double *origins, const int64_t *vptr,
                          const int32_t *handle, const double *phi, const double *phi_affine,
                          const double affine_origin[3], int32_t n_cg);

/* Build the SMS + affine bases natively on the host (C++/OpenMP) from the uploaded mesh,
 * material (E weights the Laplacian, Q17), Dirichlet set and densities, then upload them as
 * ms_basis_upload does (SURVEY §8(b) `ms_basis_build`; §3.5 L304-381 SMS basis,
 * §3.5.1 L364-381 Dirichlet weight, §3.6 L383-419 partitioning, §3.7.2 L492-495 N_cg):
 *  1. m clusters of the tets: kmeans++ seeding on volume-weighted tet barycentres with draws
 *     k = 0..m-1 of the counter-based SplitMix64 stream of `seed` (z = seed + (k+1)
 *     0x9E3779B97F4A7C15, two xor-shift-multiply rounds, u = (z >> 11) 2^-53; the pick is the
 *     first index whose sequential prefix sum exceeds u * total), Lloyd iterations with exact
 *     squared distances (ties -> lowest centre) to a fixed point or 100 rounds (Euclidean
 *     stand-in for the paper's heat geodesics, reading B2);
 *  2. face-connected clusters (largest component kept, the rest moved to the face-adjacent
 *     cluster with most shared faces); empty clusters dropped, so info->m may be < m;
 *  3. centroid vertex per cluster (nearest to the volume-weighted barycentre, Q15); handles
 *     ordered by (x, y, z) of their centroid vertex;
 *  4. per handle: K u = 0, K = L_s M^-1 L_s on the cluster + vertex-sharing clusters (R9, Q17),
 *     u(c_i) = 1, u = 0 at neighbour centroids / internal boundary / Dirichlet vertices, clip;
 *  5. Dirichlet weight, partition-of-unity normalisation, coverage-hole repair (B1), affine
 *     handle at the centre of mass with phi_a = 1 - phi_DBC (Q14); N_cg from the hop heuristic.
 * The same algorithm, draws and tie rules as precompute/basis.py: partition, centroid vertices
 * and handle lists agree exactly, weights to the rounding of the subdomain solves.
 * info may be NULL.  Errors: MS_ERR_ARG (m <= 0 or m > n_tets), MS_ERR_NOT_SPD (a subdomain
 * system is singular), MS_ERR_COVERAGE, MS_ERR_STATE (no mesh). */
typedef struct ms_basis_info {
  int32_t m;              /* handles after dropping empty clusters                         */
  int32_t n_cg;           /* refinement iterations from the hop heuristic                  */
  int32_t n_holes;        /* free vertices repaired by reading B1                           */
  int32_t pad_;
  int64_t nnz_phi;        /* (vertex, handle) entries with phi > 0                          */
  double hop_radius;      /* mean over partitions of the max hop distance                  */
  double t_kmeans, t_connect, t_solve, t_total;   /* host seconds per stage                */
} ms_basis_info;
ms_status ms_basis_build(ms_ctx *ctx, int32_t m, uint64_t seed, ms_basis_info *info);
/* Host-only form of the same construction (no GPU, no context): the global mesh as in
 * ms_upload_mesh (E and rho per tet; nu is not used) and the Dirichlet vertices.  On success *out
 * owns the result (free with ms_basis_free); read it with ms_basis_copy (sizes from info). */
typedef struct ms_basis ms_basis;
ms_status ms_basis_compute(int64_t n_verts, const double *rest_xyz, int64_t n_tets, const int32_t *tets,
                           const double *E, const double *rho, int64_t n_dbc, const int32_t *dbc, int32_t m,
                           uint64_t seed, ms_basis **out, ms_basis_info *info);
ms_status ms_basis_copy(const ms_basis *b, double *origins, int64_t *vptr, int32_t *handle, double *phi,
                        double *phi_affine, double affine_origin[3], int32_t *cluster,
                        int32_t *centroid_vertex);
void ms_basis_free(ms_basis *b);
/* Copy out the last ms_basis_build result (sizes from ms_basis_info): origins (m x 3),
 * vptr (n_verts + 1), handle / phi (nnz_phi), phi_affine (n_verts), affine_origin (3),
 * cluster (n_tets, handle id of each tet), centroid_vertex (m).  NULL pointers are skipped.
 * MS_ERR_STATE if no basis was built by this context. */
ms_status ms_basis_export(ms_ctx *ctx, double *origins, int64_t *vptr, int32_t *handle, double *phi,
                          double *phi_affine, double affine_origin[3], int32_t *cluster,
                          int32_t *centroid_vertex);

/* The cubature of the subspace Hessian (NEXT-2; §3.8, Alg. 3): n elements
 * (global tet ids, any order, no repeats) with weights w > 0 that replace the element volume in
 * the elastic-energy integral of the cubature Hessian (precompute/cubature.py fits them by
 * modal moment fitting).  Used when params.use_cubature = 1.  Errors: MS_ERR_ARG (index range,
 * w <= 0, repeats), MS_ERR_STATE (no mesh). */
ms_status ms_cubature_upload(ms_ctx *ctx, int64_t n, const int32_t *elements, const double *weights);

/* ---------------------------------------------------------------- state */
/* Set / get positions x and velocities v (n_verts x 3). */
ms_status ms_set_state(ms_ctx *ctx, const double *x, const double *v);
ms_status ms_get_state(ms_ctx *ctx, double *x, double *v);
/* Mid-step state for bootstrapped parity (reading R10): x^t, xhat and the current iterate. */
ms_status ms_set_step_state(ms_ctx *ctx, const double *x_t, const double *xhat, const double *x);
ms_status ms_get_step_state(ms_ctx *ctx, double *x_t, double *xhat, double *x);

/* ---------------------------------------------------------------- the hot path */
/* One implicit-Euler timestep: begin_step, Newton iterations until converged / cap /
 * line-search failure, end_step (Alg. 1; §3.9).  On a hard error inside the
 * Newton loop (e.g. MS_ERR_INFEASIBLE, MS_ERR_NOT_SPD) the step is abandoned: x is reset to x^t,
 * v is unchanged and no step is in progress. */
ms_status ms_timestep(ms_ctx *ctx, ms_step_stats *out);
/* xhat = x^t + h v^t + h^2 g, x = x^t (R8). */
ms_status ms_begin_step(ms_ctx *ctx);
/* One Newton iteration: gradient, PSD Hessian, BSR assembly,
 * S_a and S = B^T H B + Cholesky, coarse correction d_s (Alg. 2, R4, R6), N_cg Jacobi-PCG
 * iterations on H d_f = -g - H d_s (R5), d = d_s + d_f, CCD + inversion
 * filtered backtracking on E (Q12), x += alpha d, termination test (R7).
 * Returns MS_WARN_LS_FAILED if the line search failed (x unchanged). */
ms_status ms_newton_step(ms_ctx *ctx, ms_newton_stats *out);
/* v = (x - x^t) / h. */
ms_status ms_end_step(ms_ctx *ctx);

/* ---------------------------------------------------------------- parity hooks / pieces */
/* Evaluate energy, gradient and the assembled Hessian H at the current iterate and xhat
 * (rows a2-a4).  energy_out may be NULL. */
ms_status ms_assemble(ms_ctx *ctx, double *energy_out);
/* Gradient (3 n_verts) of the last ms_assemble / Newton iteration. */
ms_status ms_get_gradient(ms_ctx *ctx, double *g);
/* Per-element outputs at positions x (n_verts x 3): Ee[n_tets] = V_e Psi(F_e),
 * ge[n_tets x 12] = V_e G_e^T vec P, He[n_tets x 144] = P+(H_e) (row-major 12x12, vertex-
 * major xyz index 3a+c); any output pointer may be NULL. */
ms_status ms_eval_elements(ms_ctx *ctx, const double *x, double *Ee, double *ge, double *He);
/* BSR export of the assembled H: nnzb (out), rowptr[n_verts+1], colidx[nnzb], vals[9 nnzb]
 * (row-major 3x3).  Pass NULL arrays to query nnzb only. */
ms_status ms_export_bsr(ms_ctx *ctx, int64_t *nnzb, int32_t *rowptr, int32_t *colidx,
                        double *vals);
/* y = H x with the assembled H (3 n_verts vectors). */
ms_status ms_spmv(ms_ctx *ctx, const double *x, double *y);
/* w = U_s q (q: 12 m) and z = U_s^T y (y: 3 n_verts). */
ms_status ms_basis_apply(ms_ctx *ctx, const double *q, double *w);
ms_status ms_basis_apply_t(ms_ctx *ctx, const double *y, double *z);
/* Coarse matrices of the last assembly: S (12m x 12m, dense row-major; may be NULL) and
 * S_a (12 x 12; may be NULL).  Computes S, S_a from the assembled H if needed. */
ms_status ms_export_coarse(ms_ctx *ctx, double *S, double *Sa);
/* Subspace direction of the last assembly: d_s (and d_a) from Alg. 2 with exact solves. */
ms_status ms_subspace_direction(ms_ctx *ctx, double *ds, double *da);
/* Directions d_s, d_f of the last Newton iteration (3 n_verts each; either may be NULL). */
ms_status ms_get_direction(ms_ctx *ctx, double *ds, double *df);
/* Exactly `iters` Jacobi-PCG iterations on H sol = rhs from sol = 0 with the assembled H
 * (stops early only if r^T D^-1 r == 0). */
ms_status ms_pcg_solve(ms_ctx *ctx, const double *rhs, double *sol, int32_t iters,
                       ms_pcg_stats *out);
/* Same, device-resident vectors (length 3 n_verts, on the context's device/stream). */
ms_status ms_pcg_solve_dev(ms_ctx *ctx, const double *rhs_dev, double *sol_dev, int32_t iters,
                           ms_pcg_stats *out);

/* ---------------------------------------------------------------- instrumentation */
ms_status ms_set_profiling(ms_ctx *ctx, int32_t on);      /* resets the accumulators   */
ms_status ms_get_phase_times(ms_ctx *ctx, ms_phase_times *out);
/* Number of kernel launches (graph-embedded kernels included) issued by this context. */
int64_t ms_kernel_launches(ms_ctx *ctx);
/* Structure of the coarse factorisation chosen at ms_basis_upload (reading R4):
 * S is n_s x n_s (n_s = 12 m), factorised in tile x tile tiles of a dense padded array; only the
 * lower_tiles tiles of the symbolic factor are touched.  ordering: 0 = handles in centroid
 * x-order, 1 = geometric nested dissection (whichever needs fewer tile flops).  flops: flop count
 * of one factorisation at tile granularity (flops_xorder / flops_nd: both candidates); n_tasks:
 * tile tasks (factor, panel, update); critical_path: longest task chain of the tile DAG. */
typedef struct ms_coarse_info {
  int64_t n_s, tile, ntiles, lower_tiles, n_tasks, critical_path, nnzb_s;
  int64_t critical_path_xorder, critical_path_nd;
  int32_t ordering, pad_;
  double flops, flops_xorder, flops_nd;
  double galerkin_flops;   /* S = B^T H B arithmetic of one projection (fused Galerkin kernel) */
} ms_coarse_info;
ms_status ms_get_coarse_info(ms_ctx *ctx, ms_coarse_info *out);

/* Sizes: n_verts, n_tets, nnzb (BSR blocks), m (handles), nnz_phi, nnzb_S (coupled handle
 * pairs incl. diagonal) — any pointer may be NULL. */
ms_status ms_get_sizes(ms_ctx *ctx, int64_t *n_verts, int64_t *n_tets, int64_t *nnzb,
                       int32_t *m, int64_t *nnz_phi, int64_t *nnzb_S);

#ifdef __cplusplus
}
#endif
#endif /* MSIM_H */
