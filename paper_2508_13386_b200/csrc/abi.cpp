// C-ABI entry points (include/msim.h) and the host-side Newton orchestration.
//
// SURVEY §8(b) (the boundary) and §3(b) (call stack of ms_timestep).  The orchestration
// enqueues every step of one Newton iteration on the caller's stream and synchronises once
// per line-search batch (one device->host read of a few scalars).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>

#include "common.cuh"
#include "basis.h"

using namespace msim;

struct ms_ctx {
  Ctx c;
};

namespace msim {

void phase_begin(Ctx &c, int phase) {
  if (!c.profiling) return;
  if (c.ev_used + 2 > c.ev_pool.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      MS_CUDA(cudaEventCreate(&e));
      c.ev_pool.push_back(e);
    }
  }
  Ctx::PhaseRec r{phase, c.ev_pool[c.ev_used], c.ev_pool[c.ev_used + 1]};
  c.ev_used += 2;
  MS_CUDA(cudaEventRecord(r.a, c.stream));
  c.prec.push_back(r);
  c.cur_phase = phase;
}

void phase_end(Ctx &c) {
  if (!c.profiling || c.cur_phase < 0) return;
  MS_CUDA(cudaEventRecord(c.prec.back().b, c.stream));
  c.cur_phase = -1;
}

static void resolve_phases(Ctx &c) {
  if (c.prec.empty()) return;
  MS_CUDA(cudaStreamSynchronize(c.stream));
  for (auto &r : c.prec) {
    float ms = 0.f;
    MS_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    c.ptimes.ms[r.phase] += ms;
    c.ptimes.count[r.phase] += 1;
  }
  c.prec.clear();
  c.ev_used = 0;
}

static void require_mesh(Ctx &c) { MS_REQUIRE(c.nv > 0, MS_ERR_STATE, "no mesh uploaded"); }
static void require_basis(Ctx &c) { MS_REQUIRE(c.m > 0, MS_ERR_STATE, "no basis uploaded"); }

static int n_cg_of(const Ctx &c) { return c.params.n_cg > 0 ? c.params.n_cg : c.n_cg_basis; }

// NEXT-2 refresh policy of the lagged elastic Hessian (reading C4)
static bool hlag_should_update(const Ctx &c) {
  if (!c.lag_valid || c.step_iter == 0) return true;
  if (c.step_iter - c.lag_last_refresh < 5 || c.step_alphas.empty()) return false;
  const size_t n = std::min<size_t>(3, c.step_alphas.size());
  double s = 0.0;
  for (size_t k = c.step_alphas.size() - n; k < c.step_alphas.size(); ++k) s += c.step_alphas[k];
  return s / (double)n < 0.2;
}

static void enqueue_assembly(Ctx &c) {
  phase_begin(c, MS_PHASE_GRAD);
  launch_elem_grad(c);
  launch_vertex_grad(c);
  dist_sum(c, c.scal + SC_SUM0, SC_SUM_N);   // energies, |g|^2, infeasibility: over all ranks
  phase_end(c);
  // H_ref (the refinement Hessian) in vals; with NEXT-2 the subspace Hessian separately in vals_s
  const bool lag = c.params.lag_hessian != 0, cub = c.params.use_cubature != 0;
  const bool refresh = !lag || hlag_should_update(c);
  phase_begin(c, MS_PHASE_HESS);
  if (lag && !refresh && cub) launch_elem_hess_list(c);   // only the cubature elements are needed
  else launch_elem_hess(c);
  phase_end(c);
  phase_begin(c, MS_PHASE_ASSEMBLY);
  if (refresh) {
    launch_assemble(c);
    if (lag) {
      c.lag_valid = true;
      c.lag_last_refresh = c.step_iter;
      c.lag_refreshes++;
    }
  } else {
    launch_lag_diag(c);
  }
  if (c.separate_sub()) launch_assemble_sub(c);
  phase_end(c);
  c.assembled = true;
  c.coarse_ready = false;
}

static void enqueue_coarse(Ctx &c) {
  phase_begin(c, MS_PHASE_COARSE_S);
  launch_coarse_S(c);
  phase_end(c);
  phase_begin(c, MS_PHASE_COARSE_FACTOR);
  launch_coarse_factor(c);
  phase_end(c);
  phase_begin(c, MS_PHASE_COARSE_SOLVE);
  launch_coarse_direction(c);
  phase_end(c);
  c.coarse_ready = true;
}

static void fetch_scalars(Ctx &c, int K) {
  double *h = c.h_pinned;
  MS_CUDA(cudaMemcpyAsync(h, c.scal, sizeof(double) * SC_COUNT, cudaMemcpyDeviceToHost, c.stream));
  MS_CUDA(cudaMemcpyAsync(h + SC_COUNT, c.ls_out, sizeof(double) * 2 * K, cudaMemcpyDeviceToHost, c.stream));
  MS_CUDA(cudaMemcpyAsync(h + SC_COUNT + 2 * kMaxLS, c.flags, sizeof(int32_t) * 8, cudaMemcpyDeviceToHost,
                          c.stream));
  MS_CUDA(cudaStreamSynchronize(c.stream));
}

static ms_status newton_step(Ctx &c, ms_newton_stats *st) {
  require_mesh(c);
  require_basis(c);
  MS_REQUIRE(c.step_begun, MS_ERR_STATE, "ms_newton_step before ms_begin_step");
  const int n3 = 3 * c.nv;
  const int K = c.params.ls_batch;
  enqueue_assembly(c);
  enqueue_coarse(c);
  phase_begin(c, MS_PHASE_PCG);
  int ncg;
  if (c.params.refine_mode == MS_REFINE_TWO_LEVEL) {
    ncg = launch_refine_two_level(c, c.r, c.df);   // NEXT-4: to refine_tol (host-checked batches)
  } else {
    ncg = n_cg_of(c);
    launch_pcg(c, c.r, c.df, ncg);
  }
  phase_end(c);
  phase_begin(c, MS_PHASE_LINESEARCH);
  MS_CUDA(cudaMemcpyAsync(c.d, c.ds, sizeof(double) * n3, cudaMemcpyDeviceToDevice, c.stream));
  launch_axpby(c, c.d, 1.0, c.df, 1.0, n3);
  halo_exchange(c, c.d);   // multi-GPU: the line search reads d at ghost vertices
  launch_dot(c, c.ds, c.ds, 3 * (int64_t)c.nv_own, SC_DSNORM2);
  dist_sum(c, c.scal + SC_DSNORM2, 1);
  launch_filters(c);
  launch_ls_batch(c, 0, K);
  fetch_scalars(c, K);
  const double *h = c.h_pinned;
  const int32_t *fl = reinterpret_cast<const int32_t *>(h + SC_COUNT + 2 * kMaxLS);
  MS_REQUIRE(h[SC_INFEAS] == 0.0 && h[SC_INFEAS_V] == 0.0, MS_ERR_INFEASIBLE,
             "infeasible iterate: inverted element or penetrating vertex (E = +inf)");
  MS_REQUIRE(fl[0] == 0 && fl[1] == 0, MS_ERR_NOT_SPD, "coarse matrix not SPD (Cholesky pivot <= 0)");
  const double h2 = c.ah2();   // alpha h^2 (Eq. 2)
  const double energy = h2 * h[SC_ENERGY_ELEM] + h[SC_ENERGY_VERT];
  double alpha = 0.0, dE = 0.0;
  int evals = 0;
  bool failed = false, done = false;
  int k0 = 0;
  while (!done) {
    for (int k = 0; k < K; ++k) {
      const double a = h[SC_COUNT + K + k];
      const int idx = k0 + k;
      if (idx > 0 && a < c.params.ls_min) {
        failed = true;
        done = true;
        break;
      }
      evals++;
      const double de = h[SC_COUNT + k];
      if (de < 0.0) {
        alpha = a;
        dE = de;
        done = true;
        break;
      }
    }
    if (!done) {
      k0 += K;
      launch_ls_batch(c, k0, K);
      fetch_scalars(c, K);
    }
  }
  if (!failed) launch_update(c, alpha);
  phase_end(c);
  c.step_alphas.push_back(failed ? 0.0 : alpha);
  c.step_iter++;
  const double dsn = std::sqrt(h[SC_DSNORM2]);
  const bool conv = dsn / (c.params.h * c.nv_glob) < c.params.eps;   // R7: all vertices
  if (st) {
    st->alpha = failed ? 0.0 : alpha;
    st->alpha0 = h[SC_ALPHA0];
    st->ds_norm = dsn;
    st->energy = energy;
    st->delta_energy = failed ? 0.0 : dE;
    st->grad_norm = std::sqrt(h[SC_GNORM2]);
    st->ls_evals = evals;
    st->converged = conv ? 1 : 0;
    st->ls_failed = failed ? 1 : 0;
    st->n_cg = ncg;
    st->coarse_iters = c.params.coarse_mode == MS_COARSE_PCG ? c.coarse_iters_last : 0;
  }
  return failed ? MS_WARN_LS_FAILED : MS_OK;
}

static void begin_step(Ctx &c) {
  require_mesh(c);
  // error flags (pivot <= 0, infeasibility) describe one iteration: clear what an abandoned step left
  MS_CUDA(cudaMemsetAsync(c.flags, 0, sizeof(int32_t) * c.flags.n, c.stream));
  launch_predictor(c);
  c.step_begun = true;
  c.step_iter = 0;
  c.step_alphas.clear();
}

static void end_step(Ctx &c) {
  MS_REQUIRE(c.step_begun, MS_ERR_STATE, "ms_end_step before ms_begin_step");
  launch_velocity(c);
  c.step_begun = false;
}

// ---- global <-> local vertex vectors (3 per vertex); world == 1: plain copies
static void upload_global(Ctx &c, double *dev, const double *glob) {
  const size_t n3 = 3 * (size_t)c.nv;
  if (!c.dist()) {
    MS_CUDA(cudaMemcpyAsync(dev, glob, sizeof(double) * n3, cudaMemcpyHostToDevice, c.stream));
    MS_CUDA(cudaStreamSynchronize(c.stream));
    return;
  }
  std::vector<double> loc(n3);
  for (int32_t l = 0; l < c.nv; ++l)
    for (int k = 0; k < 3; ++k) loc[3 * (size_t)l + k] = glob[3 * (size_t)c.part.l2g[l] + k];
  MS_CUDA(cudaMemcpyAsync(dev, loc.data(), sizeof(double) * n3, cudaMemcpyHostToDevice, c.stream));
  MS_CUDA(cudaStreamSynchronize(c.stream));
}

// owned entries into their global positions (other entries of glob untouched)
static void download_owned(Ctx &c, const double *dev, double *glob) {
  const size_t n3 = 3 * (size_t)c.nv;
  if (!c.dist()) {
    MS_CUDA(cudaMemcpyAsync(glob, dev, sizeof(double) * n3, cudaMemcpyDeviceToHost, c.stream));
    MS_CUDA(cudaStreamSynchronize(c.stream));
    return;
  }
  std::vector<double> loc(3 * (size_t)c.nv_own);
  MS_CUDA(cudaMemcpyAsync(loc.data(), dev, sizeof(double) * loc.size(), cudaMemcpyDeviceToHost, c.stream));
  MS_CUDA(cudaStreamSynchronize(c.stream));
  for (int32_t l = 0; l < c.nv_own; ++l)
    for (int k = 0; k < 3; ++k) glob[3 * (size_t)c.part.l2g[l] + k] = loc[3 * (size_t)l + k];
}

}  // namespace msim

// ============================================================================ C-ABI
#define MS_TRY(ctx, ...)                                               \
  try {                                                                \
    __VA_ARGS__;                                                       \
  } catch (const msim::Error &err) {                                   \
    if (ctx) (ctx)->c.last_error = err.msg;                            \
    return err.code;                                                   \
  } catch (const std::bad_alloc &) {                                   \
    if (ctx) (ctx)->c.last_error = "host out of memory";               \
    return MS_ERR_OOM;                                                 \
  } catch (...) {                                                      \
    if (ctx) (ctx)->c.last_error = "unknown exception";                \
    return MS_ERR_CUDA;                                                \
  }

extern "C" {

const char *ms_version(void) { return "msim 0.1 (sm_100a, fp64)"; }

void ms_default_params(ms_params *p) {
  if (!p) return;
  p->h = 1.0 / 60.0;
  p->gravity[0] = 0.0;
  p->gravity[1] = 0.0;
  p->gravity[2] = -9.8;
  p->eps = 1e-6;
  p->max_newton = 100;
  p->n_cg = 0;
  p->ls_shrink = 0.5;
  p->ls_min = 1e-8;
  p->filter_safety = 0.9;
  p->ls_batch = 4;
  p->use_graphs = 1;
  p->debug_flags = 0;
  p->coarse_mode = MS_COARSE_EXACT;
  p->coarse_max_iter = 1000;
  p->coarse_tol = 1e-4;
  p->integrator = MS_INTEGRATOR_IE;
  p->use_cubature = 0;
  p->lag_hessian = 0;
  p->refine_mode = MS_REFINE_JACOBI;
  p->refine_max_iter = 100;
  p->refine_tol = 1e-2;
}

static ms_status create_common(ms_ctx **out, int device, void *cuda_stream, int rank, int world,
                               const uint8_t *nccl_id, msim::Hub *hub) {
  if (!out) return MS_ERR_ARG;
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return MS_ERR_ARG;
  if (world > 1 && !nccl_id && !hub) return MS_ERR_ARG;
  ms_ctx *ctx = new (std::nothrow) ms_ctx();
  if (!ctx) return MS_ERR_OOM;
  const ms_status st = [&]() -> ms_status {
    MS_TRY(ctx, {
      MS_CUDA(cudaSetDevice(device));
      ctx->c.device = device;
      ctx->c.stream = reinterpret_cast<cudaStream_t>(cuda_stream);
      ctx->c.part.rank = rank;
      ctx->c.part.world = world;
      ms_default_params(&ctx->c.params);
      MS_CUDA(cudaMallocHost((void **)&ctx->c.h_pinned, sizeof(double) * PH_COUNT));
      // per-device kernel attributes (large shared-memory opt-ins), on this context's device
      msim::elem_init_attrs(ctx->c);
      msim::coarse_init_attrs(ctx->c);
      msim::chol_init_attrs(ctx->c);
      if (world > 1 || nccl_id)
        ctx->c.comm = hub ? msim::make_hub_comm(hub, rank) : msim::make_nccl_comm(nccl_id, rank, world, device);
    });
    return MS_OK;
  }();
  if (st != MS_OK) {
    delete ctx;
    return st;
  }
  *out = ctx;
  return MS_OK;
}

ms_status ms_create(ms_ctx **out, int device, void *cuda_stream, const uint8_t *nccl_id, int rank, int world) {
  return create_common(out, device, cuda_stream, rank, world, nccl_id, nullptr);
}

ms_status ms_nccl_unique_id(uint8_t out[128]) {
  if (!out) return MS_ERR_ARG;
  try {
    msim::nccl_unique_id(out);
  } catch (...) {
    return MS_ERR_NCCL;
  }
  return MS_OK;
}

ms_status ms_partition(int32_t rank, int32_t world, int64_t nv, const double *X, int64_t nt, const int32_t *tets,
                       int32_t *counts, int32_t *l2g, int32_t *tet_l2g, int32_t *peer_counts,
                       int32_t *send_global, int32_t *recv_global) {
  if (!X || !tets || !counts || nv <= 0 || nt <= 0 || nv >= INT32_MAX || nt >= INT32_MAX) return MS_ERR_ARG;
  try {
    for (int64_t i = 0; i < 4 * nt; ++i)
      if (tets[i] < 0 || tets[i] >= nv) return MS_ERR_ARG;
    msim::Partition P;
    msim::make_partition(rank, world, (int32_t)nv, X, (int32_t)nt, tets, P);
    counts[0] = P.nv_own;
    counts[1] = P.nv_loc;
    counts[2] = P.nt_own;
    counts[3] = P.nt_loc;
    counts[4] = (int32_t)P.send_idx.size();
    counts[5] = (int32_t)P.recv_idx.size();
    if (l2g) std::copy(P.l2g.begin(), P.l2g.end(), l2g);
    if (tet_l2g) std::copy(P.tet_l2g.begin(), P.tet_l2g.end(), tet_l2g);
    if (peer_counts) {
      std::fill(peer_counts, peer_counts + 2 * (size_t)world, 0);
      for (const auto &p : P.peers) {
        peer_counts[2 * p.rank] = p.n_send;
        peer_counts[2 * p.rank + 1] = p.n_recv;
      }
    }
    if (send_global)
      for (size_t k = 0; k < P.send_idx.size(); ++k) send_global[k] = P.l2g[P.send_idx[k]];
    if (recv_global)
      for (size_t k = 0; k < P.recv_idx.size(); ++k) recv_global[k] = P.l2g[P.recv_idx[k]];
  } catch (const msim::Error &e) {
    return e.code;
  } catch (...) {
    return MS_ERR_ARG;
  }
  return MS_OK;
}

ms_status ms_hub_create(int32_t world, ms_hub **out) {
  if (!out || world < 1) return MS_ERR_ARG;
  *out = reinterpret_cast<ms_hub *>(msim::hub_create(world));
  return MS_OK;
}

ms_status ms_hub_destroy(ms_hub *hub) {
  msim::hub_destroy(reinterpret_cast<msim::Hub *>(hub));
  return MS_OK;
}

ms_status ms_create_hub(ms_ctx **out, int device, void *cuda_stream, ms_hub *hub, int rank, int world) {
  if (!hub) return MS_ERR_ARG;
  return create_common(out, device, cuda_stream, rank, world, nullptr, reinterpret_cast<msim::Hub *>(hub));
}

ms_status ms_destroy(ms_ctx *ctx) {
  if (!ctx) return MS_OK;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  pcg_reset_graph(ctx->c);
  coarse_reset_graphs(ctx->c);
  for (auto e : ctx->c.ev_pool) cudaEventDestroy(e);
  if (ctx->c.halo_stream) {
    cudaStreamSynchronize(ctx->c.halo_stream);
    cudaStreamDestroy(ctx->c.halo_stream);
    cudaEventDestroy(ctx->c.ev_z);
    cudaEventDestroy(ctx->c.ev_halo);
  }
  if (ctx->c.h_pinned) cudaFreeHost(ctx->c.h_pinned);
  delete ctx->c.comm;
  delete ctx->c.built_basis;
  delete ctx;
  return MS_OK;
}

const char *ms_last_error(ms_ctx *ctx) { return ctx ? ctx->c.last_error.c_str() : "null context"; }

ms_status ms_upload_mesh(ms_ctx *ctx, int64_t n_verts, const double *rest_xyz, int64_t n_tets,
                         const int32_t *tets, const double *E, const double *nu, const double *rho) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    MS_REQUIRE(n_verts > 0 && n_tets > 0 && rest_xyz && tets && E && nu && rho, MS_ERR_ARG, "bad mesh arguments");
    MS_REQUIRE(n_verts < INT32_MAX / 3 && n_tets < INT32_MAX / 16, MS_ERR_ARG, "mesh too large for int32 indices");
    Ctx &c = ctx->c;
    MS_CUDA(cudaSetDevice(c.device));
    c.m = 0;
    pcg_reset_graph(c);
    c.nv_glob = (int32_t)n_verts;
    c.has_history = false;
    c.h_Eg.assign(E, E + n_tets);
    c.h_rhog.assign(rho, rho + n_tets);
    c.h_dbc_glob.clear();
    if (c.dist()) c.h_Xg.assign(rest_xyz, rest_xyz + 3 * n_verts);
    if (!c.dist()) {
      c.nv = c.nv_own = (int32_t)n_verts;
      c.nt = c.nt_own = (int32_t)n_tets;
      build_mesh_structures(c, rest_xyz, tets, E, nu, rho);
    } else {
      for (int64_t i = 0; i < 4 * n_tets; ++i)
        MS_REQUIRE(tets[i] >= 0 && tets[i] < n_verts, MS_ERR_ARG, "tet vertex index out of range");
      msim::Partition &P = c.part;
      msim::make_partition(P.rank, P.world, (int32_t)n_verts, rest_xyz, (int32_t)n_tets, tets, P);
      c.h_tets_glob.assign(tets, tets + 4 * (size_t)n_tets);
      std::vector<double> X(3 * (size_t)P.nv_loc), Ev(P.nt_loc), nuv(P.nt_loc), rhov(P.nt_loc);
      for (int32_t l = 0; l < P.nv_loc; ++l)
        for (int k = 0; k < 3; ++k) X[3 * (size_t)l + k] = rest_xyz[3 * (size_t)P.l2g[l] + k];
      for (int32_t le = 0; le < P.nt_loc; ++le) {
        Ev[le] = E[P.tet_l2g[le]];
        nuv[le] = nu[P.tet_l2g[le]];
        rhov[le] = rho[P.tet_l2g[le]];
      }
      c.nv = P.nv_loc;
      c.nt = P.nt_loc;
      c.nv_own = P.nv_own;
      c.nt_own = P.nt_own;
      build_mesh_structures(c, X.data(), P.tets_loc.data(), Ev.data(), nuv.data(), rhov.data());
      c.halo_send_idx.upload(P.send_idx.empty() ? std::vector<int32_t>{0} : P.send_idx, c.stream);
      c.halo_recv_idx.upload(P.recv_idx.empty() ? std::vector<int32_t>{0} : P.recv_idx, c.stream);
      c.halo_send.alloc(3 * std::max<size_t>(P.send_idx.size(), 1));
      c.halo_recv.alloc(3 * std::max<size_t>(P.recv_idx.size(), 1));
      MS_CUDA(cudaStreamSynchronize(c.stream));
    }
  });
  return MS_OK;
}

ms_status ms_set_dirichlet(ms_ctx *ctx, int64_t n, const int32_t *verts) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    MS_REQUIRE(n == 0 || verts, MS_ERR_ARG, "null verts");
    MS_REQUIRE(c.m == 0, MS_ERR_STATE,
               "ms_set_dirichlet after ms_basis_upload: the basis was built for another Dirichlet set");
    std::fill(c.h_fixed.begin(), c.h_fixed.end(), 0);
    c.h_dbc_glob.assign(verts, verts + n);
    for (int64_t k = 0; k < n; ++k) {
      MS_REQUIRE(verts[k] >= 0 && verts[k] < c.nv_glob, MS_ERR_ARG, "Dirichlet vertex out of range");
      const int32_t l = c.dist() ? c.part.g2l[verts[k]] : verts[k];
      if (l >= 0) c.h_fixed[l] = 1;
    }
    c.fixed.upload(c.h_fixed, c.stream);
    MS_CUDA(cudaStreamSynchronize(c.stream));
  });
  return MS_OK;
}

ms_status ms_set_ground(ms_ctx *ctx, const double normal[3], double offset, double dhat, double kappa) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    MS_REQUIRE(normal != nullptr, MS_ERR_ARG, "null normal");
    const double nn = std::sqrt(normal[0] * normal[0] + normal[1] * normal[1] + normal[2] * normal[2]);
    MS_REQUIRE(std::fabs(nn - 1.0) < 1e-12, MS_ERR_ARG, "ground normal must be a unit vector");
    c.has_ground = kappa > 0.0;
    MS_REQUIRE(!c.has_ground || dhat > 0.0, MS_ERR_ARG, "dhat must be > 0");
    for (int k = 0; k < 3; ++k) c.gn[k] = normal[k];
    c.goff = offset;
    c.dhat = dhat;
    c.kappa = kappa;
  });
  return MS_OK;
}

ms_status ms_set_params(ms_ctx *ctx, const ms_params *p) {
  if (!ctx || !p) return MS_ERR_ARG;
  MS_TRY(ctx, {
    MS_REQUIRE(p->h > 0.0 && p->eps > 0.0 && p->max_newton > 0 && p->n_cg >= 0, MS_ERR_ARG, "bad params");
    MS_REQUIRE(p->ls_shrink > 0.0 && p->ls_shrink < 1.0 && p->ls_min > 0.0, MS_ERR_ARG, "bad line-search params");
    MS_REQUIRE(p->filter_safety > 0.0 && p->filter_safety <= 1.0, MS_ERR_ARG, "bad filter safety");
    MS_REQUIRE(p->ls_batch == 1 || p->ls_batch == 2 || p->ls_batch == 4 || p->ls_batch == 8, MS_ERR_ARG,
               "ls_batch must be 1, 2, 4 or 8");
    MS_REQUIRE(p->coarse_mode == MS_COARSE_EXACT || p->coarse_mode == MS_COARSE_PCG, MS_ERR_ARG, "bad coarse_mode");
    MS_REQUIRE(p->coarse_tol >= 0.0 && p->coarse_max_iter > 0, MS_ERR_ARG, "bad coarse PCG params");
    MS_REQUIRE(p->integrator == MS_INTEGRATOR_IE || p->integrator == MS_INTEGRATOR_BDF2, MS_ERR_ARG, "bad integrator");
    MS_REQUIRE(p->refine_mode == MS_REFINE_JACOBI || p->refine_mode == MS_REFINE_TWO_LEVEL, MS_ERR_ARG,
               "bad refine_mode");
    MS_REQUIRE(p->refine_mode == MS_REFINE_JACOBI || p->coarse_mode == MS_COARSE_EXACT, MS_ERR_ARG,
               "the two-level refinement needs the factorised coarse matrix (MS_COARSE_EXACT)");
    MS_REQUIRE(p->refine_tol >= 0.0 && p->refine_max_iter >= 0, MS_ERR_ARG, "bad refinement PCG params");
    if (p->integrator != ctx->c.params.integrator) ctx->c.has_history = false;
    if (p->lag_hessian != ctx->c.params.lag_hessian || p->use_cubature != ctx->c.params.use_cubature)
      ctx->c.lag_valid = false;
    if (p->n_cg != ctx->c.params.n_cg || p->use_graphs != ctx->c.params.use_graphs ||
        p->coarse_mode != ctx->c.params.coarse_mode || p->coarse_tol != ctx->c.params.coarse_tol ||
        p->coarse_max_iter != ctx->c.params.coarse_max_iter || p->refine_mode != ctx->c.params.refine_mode ||
        p->refine_tol != ctx->c.params.refine_tol || p->refine_max_iter != ctx->c.params.refine_max_iter) {
      pcg_reset_graph(ctx->c);
      coarse_reset_graphs(ctx->c);
    }
    ctx->c.params = *p;
  });
  return MS_OK;
}

ms_status ms_get_params(ms_ctx *ctx, ms_params *p) {
  if (!ctx || !p) return MS_ERR_ARG;
  *p = ctx->c.params;
  return MS_OK;
}

namespace msim {
static void basis_upload_impl(Ctx &c, int32_t m, const double *origins, const int64_t *vptr, const int32_t *handle,
                              const double *phi, const double *phi_affine, const double affine_origin[3],
                              int32_t n_cg) {
    MS_REQUIRE(n_cg > 0, MS_ERR_ARG, "n_cg must be > 0");
    if (!c.dist()) {
      build_basis_structures(c, m, origins, vptr, handle, phi, phi_affine, affine_origin);
    } else {   // local rows of the global basis + the global S pattern
      MS_REQUIRE(vptr[0] == 0, MS_ERR_ARG, "vptr[0] must be 0");
      for (int32_t v = 0; v < c.nv_glob; ++v)
        for (int64_t k = vptr[v]; k < vptr[v + 1]; ++k)
          MS_REQUIRE(handle[k] >= 0 && handle[k] < m, MS_ERR_ARG, "handle id out of range");
      global_s_pattern(c.nv_glob, c.h_tets_glob, m, vptr, handle, c.h_sptr_glob, c.h_scol_glob);
      std::vector<int64_t> lptr(c.nv + 1, 0);
      std::vector<int32_t> lh;
      std::vector<double> lphi, laff(c.nv);
      for (int32_t l = 0; l < c.nv; ++l) {
        const int32_t v = c.part.l2g[l];
        for (int64_t k = vptr[v]; k < vptr[v + 1]; ++k) {
          lh.push_back(handle[k]);
          lphi.push_back(phi[k]);
        }
        lptr[l + 1] = (int64_t)lh.size();
        laff[l] = phi_affine[v];
      }
      build_basis_structures(c, m, origins, lptr.data(), lh.data(), lphi.data(), laff.data(), affine_origin);
    }
    c.n_cg_basis = n_cg;
    pcg_reset_graph(c);
}
}  // namespace msim

ms_status ms_basis_upload(ms_ctx *ctx, int32_t m, const double *origins, const int64_t *vptr,
                          const int32_t *handle, const double *phi, const double *phi_affine,
                          const double affine_origin[3], int32_t n_cg) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    MS_REQUIRE(origins && vptr && handle && phi && phi_affine && affine_origin, MS_ERR_ARG, "null basis array");
    basis_upload_impl(c, m, origins, vptr, handle, phi, phi_affine, affine_origin, n_cg);
  });
  return MS_OK;
}

struct ms_basis {
  msim::BasisOutput b;
};

static void fill_info(const BasisOutput &b, ms_basis_info *info) {
  if (!info) return;
  info->m = b.m;
  info->n_cg = b.n_cg;
  info->n_holes = b.n_holes;
  info->pad_ = 0;
  info->nnz_phi = (int64_t)b.phi.size();
  info->hop_radius = b.hop_radius;
  info->t_kmeans = b.t_kmeans;
  info->t_connect = b.t_connect;
  info->t_solve = b.t_solve;
  info->t_total = b.t_total;
}

static void copy_basis(const BasisOutput &b, double *origins, int64_t *vptr, int32_t *handle, double *phi,
                       double *phi_affine, double affine_origin[3], int32_t *cluster, int32_t *centroid_vertex) {
  if (origins) std::copy(b.origins.begin(), b.origins.end(), origins);
  if (vptr) std::copy(b.vptr.begin(), b.vptr.end(), vptr);
  if (handle) std::copy(b.handle.begin(), b.handle.end(), handle);
  if (phi) std::copy(b.phi.begin(), b.phi.end(), phi);
  if (phi_affine) std::copy(b.phi_affine.begin(), b.phi_affine.end(), phi_affine);
  if (affine_origin) std::copy(b.affine_origin, b.affine_origin + 3, affine_origin);
  if (cluster) std::copy(b.cluster.begin(), b.cluster.end(), cluster);
  if (centroid_vertex) std::copy(b.centroid_vertex.begin(), b.centroid_vertex.end(), centroid_vertex);
}

ms_status ms_basis_compute(int64_t n_verts, const double *rest_xyz, int64_t n_tets, const int32_t *tets,
                           const double *E, const double *rho, int64_t n_dbc, const int32_t *dbc, int32_t m,
                           uint64_t seed, ms_basis **out, ms_basis_info *info) {
  if (!out) return MS_ERR_ARG;
  *out = nullptr;
  if (n_verts <= 0 || n_tets <= 0 || !rest_xyz || !tets || !E || !rho || (n_dbc > 0 && !dbc)) return MS_ERR_ARG;
  if (n_verts >= INT32_MAX / 3 || n_tets >= INT32_MAX / 16) return MS_ERR_ARG;
  for (int64_t i = 0; i < 4 * n_tets; ++i)
    if (tets[i] < 0 || tets[i] >= n_verts) return MS_ERR_ARG;
  for (int64_t k = 0; k < n_dbc; ++k)
    if (dbc[k] < 0 || dbc[k] >= n_verts) return MS_ERR_ARG;
  ms_basis *h = new (std::nothrow) ms_basis();
  if (!h) return MS_ERR_OOM;
  try {
    BasisInput in;
    in.nv = (int32_t)n_verts;
    in.nt = (int32_t)n_tets;
    in.X = rest_xyz;
    in.tets = tets;
    in.E = E;
    in.rho = rho;
    in.dbc.assign(dbc, dbc + n_dbc);
    build_basis_host(in, m, seed, h->b);
  } catch (const msim::Error &err) {
    delete h;
    return err.code;
  } catch (const std::bad_alloc &) {
    delete h;
    return MS_ERR_OOM;
  } catch (...) {
    delete h;
    return MS_ERR_ARG;
  }
  fill_info(h->b, info);
  *out = h;
  return MS_OK;
}

ms_status ms_basis_copy(const ms_basis *h, double *origins, int64_t *vptr, int32_t *handle, double *phi,
                        double *phi_affine, double affine_origin[3], int32_t *cluster, int32_t *centroid_vertex) {
  if (!h) return MS_ERR_ARG;
  copy_basis(h->b, origins, vptr, handle, phi, phi_affine, affine_origin, cluster, centroid_vertex);
  return MS_OK;
}

void ms_basis_free(ms_basis *h) { delete h; }

ms_status ms_basis_build(ms_ctx *ctx, int32_t m, uint64_t seed, ms_basis_info *info) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    BasisInput in;
    in.nv = c.nv_glob;
    in.nt = (int32_t)c.h_Eg.size();
    in.X = c.dist() ? c.h_Xg.data() : c.h_X.data();
    in.tets = c.dist() ? c.h_tets_glob.data() : c.h_tets.data();
    in.E = c.h_Eg.data();
    in.rho = c.h_rhog.data();
    in.dbc = c.h_dbc_glob;
    if (!c.built_basis) c.built_basis = new BasisOutput();
    BasisOutput &b = *c.built_basis;
    build_basis_host(in, m, seed, b);
    basis_upload_impl(c, b.m, b.origins.data(), b.vptr.data(), b.handle.data(), b.phi.data(), b.phi_affine.data(),
                      b.affine_origin, b.n_cg);
    fill_info(b, info);
  });
  return MS_OK;
}

ms_status ms_basis_export(ms_ctx *ctx, double *origins, int64_t *vptr, int32_t *handle, double *phi,
                          double *phi_affine, double affine_origin[3], int32_t *cluster,
                          int32_t *centroid_vertex) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    MS_REQUIRE(c.built_basis != nullptr, MS_ERR_STATE, "ms_basis_export before ms_basis_build");
    copy_basis(*c.built_basis, origins, vptr, handle, phi, phi_affine, affine_origin, cluster, centroid_vertex);
  });
  return MS_OK;
}

ms_status ms_cubature_upload(ms_ctx *ctx, int64_t n, const int32_t *elements, const double *weights) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    MS_REQUIRE(n >= 0 && (n == 0 || (elements && weights)), MS_ERR_ARG, "bad cubature arrays");
    const int64_t nt_glob = (int64_t)c.h_Eg.size();
    std::vector<int32_t> g2l;
    if (c.dist()) {
      g2l.assign(nt_glob, -1);
      for (int32_t le = 0; le < c.nt; ++le) g2l[c.part.tet_l2g[le]] = le;
    }
    std::vector<char> seen(nt_glob, 0);
    std::vector<int32_t> loc;
    std::vector<double> w;
    for (int64_t k = 0; k < n; ++k) {
      MS_REQUIRE(elements[k] >= 0 && elements[k] < nt_glob, MS_ERR_ARG, "cubature element out of range");
      MS_REQUIRE(weights[k] > 0.0, MS_ERR_ARG, "cubature weights must be > 0");
      MS_REQUIRE(!seen[elements[k]], MS_ERR_ARG, "repeated cubature element");
      seen[elements[k]] = 1;
      const int32_t le = c.dist() ? g2l[elements[k]] : elements[k];
      if (le < 0) continue;   // multi-GPU: not a local tet
      loc.push_back(le);
      w.push_back(weights[k]);
    }
    build_cubature_structures(c, loc, w);
    c.lag_valid = false;
  });
  return MS_OK;
}

ms_status ms_set_state(ms_ctx *ctx, const double *x, const double *v) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    if (x) upload_global(c, c.x, x);
    if (v) upload_global(c, c.v, v);
    c.step_begun = false;
    c.has_history = false;   // a new trajectory: BDF2 restarts with an implicit-Euler step
    c.assembled = false;
  });
  return MS_OK;
}

ms_status ms_get_state(ms_ctx *ctx, double *x, double *v) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    if (x) download_owned(c, c.x, x);
    if (v) download_owned(c, c.v, v);
  });
  return MS_OK;
}

ms_status ms_set_step_state(ms_ctx *ctx, const double *x_t, const double *xhat, const double *x) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    MS_REQUIRE(x_t && xhat && x, MS_ERR_ARG, "null state array");
    upload_global(c, c.xt, x_t);
    upload_global(c, c.xhat, xhat);
    upload_global(c, c.x, x);
    MS_CUDA(cudaMemsetAsync(c.flags, 0, sizeof(int32_t) * c.flags.n, c.stream));
    c.step_begun = true;
    c.assembled = false;
  });
  return MS_OK;
}

ms_status ms_get_step_state(ms_ctx *ctx, double *x_t, double *xhat, double *x) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    if (x_t) download_owned(c, c.xt, x_t);
    if (xhat) download_owned(c, c.xhat, xhat);
    if (x) download_owned(c, c.x, x);
  });
  return MS_OK;
}

ms_status ms_begin_step(ms_ctx *ctx) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, { begin_step(ctx->c); });
  return MS_OK;
}

ms_status ms_newton_step(ms_ctx *ctx, ms_newton_stats *out) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, { return newton_step(ctx->c, out); });
  return MS_ERR_CUDA;
}

ms_status ms_end_step(ms_ctx *ctx) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    end_step(ctx->c);
    MS_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
  return MS_OK;
}

ms_status ms_timestep(ms_ctx *ctx, ms_step_stats *out) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    begin_step(c);
    ms_step_stats st{};
    st.status = MS_WARN_NEWTON_CAP;
    for (int it = 0; it < c.params.max_newton; ++it) {
      ms_newton_stats ns{};
      ms_status s;
      try {
        s = newton_step(c, &ns);
      } catch (...) {
        // leave a consistent state machine: the step is abandoned at x^t (no half-finished step
        // for a later ms_newton_step / ms_end_step to continue)
        cudaMemcpyAsync(c.x, c.xt, sizeof(double) * 3 * (size_t)c.nv, cudaMemcpyDeviceToDevice, c.stream);
        c.step_begun = false;
        throw;
      }
      st.newton_iters++;
      st.pcg_iters += ns.n_cg;
      st.ls_evals += ns.ls_evals;
      st.coarse_iters += ns.coarse_iters;
      st.last_ds_norm = ns.ds_norm;
      st.last_alpha = ns.alpha;
      if (ns.converged) {
        st.status = MS_OK;
        break;
      }
      if (s == MS_WARN_LS_FAILED) {
        st.status = MS_WARN_LS_FAILED;
        break;
      }
    }
    end_step(c);
    MS_CUDA(cudaStreamSynchronize(c.stream));
    if (out) *out = st;
    return st.status;
  });
  return MS_ERR_CUDA;
}

ms_status ms_assemble(ms_ctx *ctx, double *energy_out) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    enqueue_assembly(c);
    fetch_scalars(c, 1);
    if (energy_out) {
      const double h2 = c.ah2();   // alpha h^2 (Eq. 2)
      *energy_out = (c.h_pinned[SC_INFEAS] > 0 || c.h_pinned[SC_INFEAS_V] > 0)
                        ? INFINITY
                        : h2 * c.h_pinned[SC_ENERGY_ELEM] + c.h_pinned[SC_ENERGY_VERT];
    }
  });
  return MS_OK;
}

ms_status ms_get_gradient(ms_ctx *ctx, double *g) {
  if (!ctx || !g) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    MS_REQUIRE(c.assembled, MS_ERR_STATE, "nothing assembled yet");
    c.g.download(g, 3 * (size_t)c.nv, c.stream);
    MS_CUDA(cudaStreamSynchronize(c.stream));
  });
  return MS_OK;
}

ms_status ms_eval_elements(ms_ctx *ctx, const double *x, double *Ee, double *ge, double *He) {
  if (!ctx || !x) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    const size_t n3 = 3 * (size_t)c.nv, nt = c.nt;
    DBuf<double> dx, dE, dg, dH;
    dx.upload(x, n3, c.stream);
    if (Ee) dE.alloc(nt);
    if (ge) dg.alloc(12 * nt);
    if (He) dH.alloc(144 * nt);
    launch_eval_elements(c, dx, Ee ? dE.p : nullptr, ge ? dg.p : nullptr, He ? dH.p : nullptr);
    if (Ee) dE.download(Ee, nt, c.stream);
    if (ge) dg.download(ge, 12 * nt, c.stream);
    if (He) dH.download(He, 144 * nt, c.stream);
    MS_CUDA(cudaStreamSynchronize(c.stream));
    c.assembled = false;
  });
  return MS_OK;
}

ms_status ms_export_bsr(ms_ctx *ctx, int64_t *nnzb, int32_t *rowptr, int32_t *colidx, double *vals) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    if (nnzb) *nnzb = c.nnzb;
    if (rowptr) std::memcpy(rowptr, c.h_rowptr.data(), sizeof(int32_t) * (c.nv + 1));
    if (colidx) std::memcpy(colidx, c.h_colidx.data(), sizeof(int32_t) * c.nnzb);
    if (vals) {
      MS_REQUIRE(c.assembled, MS_ERR_STATE, "nothing assembled yet");
      std::vector<double> sell((size_t)9 * c.npos);   // SELL-32 layout (sell.cuh)
      c.vals.download(sell.data(), sell.size(), c.stream);
      MS_CUDA(cudaStreamSynchronize(c.stream));
      for (int64_t s = 0; s < c.nnzb; ++s) {
        const int64_t pos = c.h_sell_pos[s], cc = pos >> 5, lane = pos & 31;
        for (int q = 0; q < 9; ++q) vals[9 * s + q] = sell[((size_t)cc * 9 + q) * 32 + lane];
      }
    }
  });
  return MS_OK;
}

ms_status ms_spmv(ms_ctx *ctx, const double *x, double *y) {
  if (!ctx || !x || !y) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    MS_REQUIRE(c.assembled, MS_ERR_STATE, "nothing assembled yet");
    const size_t n3 = 3 * (size_t)c.nv;
    MS_CUDA(cudaMemcpyAsync(c.p, x, sizeof(double) * n3, cudaMemcpyHostToDevice, c.stream));
    launch_spmv(c, c.p, c.q, 0.0, nullptr);
    c.q.download(y, n3, c.stream);
    MS_CUDA(cudaStreamSynchronize(c.stream));
  });
  return MS_OK;
}

ms_status ms_basis_apply(ms_ctx *ctx, const double *q, double *w) {
  if (!ctx || !q || !w) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_basis(c);
    MS_CUDA(cudaMemcpyAsync(c.qs, q, sizeof(double) * 12 * c.m, cudaMemcpyHostToDevice, c.stream));
    launch_lift(c, c.qs, c.tmp, false);
    c.tmp.download(w, 3 * (size_t)c.nv, c.stream);
    MS_CUDA(cudaStreamSynchronize(c.stream));
  });
  return MS_OK;
}

ms_status ms_basis_apply_t(ms_ctx *ctx, const double *y, double *z) {
  if (!ctx || !y || !z) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_basis(c);
    MS_CUDA(cudaMemcpyAsync(c.tmp, y, sizeof(double) * 3 * c.nv, cudaMemcpyHostToDevice, c.stream));
    launch_restrict(c, c.tmp, c.zs);
    c.zs.download(z, 12 * (size_t)c.m, c.stream);
    MS_CUDA(cudaStreamSynchronize(c.stream));
  });
  return MS_OK;
}

ms_status ms_export_coarse(ms_ctx *ctx, double *S, double *Sa) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_basis(c);
    MS_REQUIRE(c.assembled, MS_ERR_STATE, "nothing assembled yet");
    launch_coarse_S(c, true);
    if (S) {
      std::vector<double> blk((size_t)144 * c.nnzb_S);
      c.Sblk.download(blk.data(), blk.size(), c.stream);
      MS_CUDA(cudaStreamSynchronize(c.stream));
      const int64_t n = 12 * (int64_t)c.m;
      std::memset(S, 0, sizeof(double) * n * n);
      for (int32_t i = 0; i < c.m; ++i)
        for (int32_t k = c.h_sptr[i]; k < c.h_sptr[i + 1]; ++k) {
          const int32_t j = c.h_scol[k];
          for (int r = 0; r < 12; ++r)
            for (int cc = 0; cc < 12; ++cc) S[(12 * i + r) * n + 12 * j + cc] = blk[(size_t)144 * k + 12 * r + cc];
        }
    }
    if (Sa) c.Sa.download(Sa, 144, c.stream);
    MS_CUDA(cudaStreamSynchronize(c.stream));
  });
  return MS_OK;
}

ms_status ms_subspace_direction(ms_ctx *ctx, double *ds, double *da) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_basis(c);
    MS_REQUIRE(c.assembled, MS_ERR_STATE, "nothing assembled yet");
    enqueue_coarse(c);
    fetch_scalars(c, 1);
    const int32_t *fl = reinterpret_cast<const int32_t *>(c.h_pinned + SC_COUNT + 2 * kMaxLS);
    MS_REQUIRE(fl[0] == 0 && fl[1] == 0, MS_ERR_NOT_SPD, "coarse matrix not SPD (Cholesky pivot <= 0)");
    if (ds) c.ds.download(ds, 3 * (size_t)c.nv, c.stream);
    if (da) c.da.download(da, 3 * (size_t)c.nv, c.stream);
    MS_CUDA(cudaStreamSynchronize(c.stream));
  });
  return MS_OK;
}

ms_status ms_get_direction(ms_ctx *ctx, double *ds, double *df) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    require_mesh(c);
    if (ds) c.ds.download(ds, 3 * (size_t)c.nv, c.stream);
    if (df) c.df.download(df, 3 * (size_t)c.nv, c.stream);
    MS_CUDA(cudaStreamSynchronize(c.stream));
  });
  return MS_OK;
}

static ms_status pcg_common(ms_ctx *ctx, int32_t iters, ms_pcg_stats *out) {
  Ctx &c = ctx->c;
  launch_pcg(c, c.rhs, c.df, iters);
  fetch_scalars(c, 1);
  if (out) {
    out->iters = iters;
    out->rz0 = c.h_pinned[SC_RZ0];
    out->rz = c.h_pinned[SC_RZ];
  }
  return MS_OK;
}

ms_status ms_pcg_solve(ms_ctx *ctx, const double *rhs, double *sol, int32_t iters, ms_pcg_stats *out) {
  if (!ctx || !rhs || !sol || iters < 0) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    MS_REQUIRE(c.assembled, MS_ERR_STATE, "nothing assembled yet");
    const size_t n3 = 3 * (size_t)c.nv;
    MS_CUDA(cudaMemcpyAsync(c.rhs, rhs, sizeof(double) * n3, cudaMemcpyHostToDevice, c.stream));
    pcg_common(ctx, iters, out);
    c.df.download(sol, n3, c.stream);
    MS_CUDA(cudaStreamSynchronize(c.stream));
  });
  return MS_OK;
}

ms_status ms_pcg_solve_dev(ms_ctx *ctx, const double *rhs_dev, double *sol_dev, int32_t iters, ms_pcg_stats *out) {
  if (!ctx || !rhs_dev || !sol_dev || iters < 0) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    MS_REQUIRE(c.assembled, MS_ERR_STATE, "nothing assembled yet");
    const size_t n3 = 3 * (size_t)c.nv;
    MS_CUDA(cudaMemcpyAsync(c.rhs, rhs_dev, sizeof(double) * n3, cudaMemcpyDeviceToDevice, c.stream));
    pcg_common(ctx, iters, out);
    MS_CUDA(cudaMemcpyAsync(sol_dev, c.df, sizeof(double) * n3, cudaMemcpyDeviceToDevice, c.stream));
    MS_CUDA(cudaStreamSynchronize(c.stream));
  });
  return MS_OK;
}

ms_status ms_set_profiling(ms_ctx *ctx, int32_t on) {
  if (!ctx) return MS_ERR_ARG;
  MS_TRY(ctx, {
    Ctx &c = ctx->c;
    resolve_phases(c);
    c.profiling = on != 0;
    c.ptimes = ms_phase_times{};
  });
  return MS_OK;
}

ms_status ms_get_phase_times(ms_ctx *ctx, ms_phase_times *out) {
  if (!ctx || !out) return MS_ERR_ARG;
  MS_TRY(ctx, {
    resolve_phases(ctx->c);
    *out = ctx->c.ptimes;
  });
  return MS_OK;
}

int64_t ms_kernel_launches(ms_ctx *ctx) { return ctx ? ctx->c.launches : -1; }

ms_status ms_get_sizes(ms_ctx *ctx, int64_t *n_verts, int64_t *n_tets, int64_t *nnzb, int32_t *m,
                       int64_t *nnz_phi, int64_t *nnzb_S) {
  if (!ctx) return MS_ERR_ARG;
  const Ctx &c = ctx->c;
  if (n_verts) *n_verts = c.nv;
  if (n_tets) *n_tets = c.nt;
  if (nnzb) *nnzb = c.nnzb;
  if (m) *m = c.m;
  if (nnz_phi) *nnz_phi = c.nnz_phi;
  if (nnzb_S) *nnzb_S = c.nnzb_S;
  return MS_OK;
}

ms_status ms_get_coarse_info(ms_ctx *ctx, ms_coarse_info *out) {
  if (!ctx || !out) return MS_ERR_ARG;
  if (ctx->c.m <= 0) {
    ctx->c.last_error = "no basis uploaded";
    return MS_ERR_STATE;
  }
  *out = ctx->c.chol_info;
  return MS_OK;
}

}  // extern "C"
