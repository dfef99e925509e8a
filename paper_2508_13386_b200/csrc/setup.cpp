// Host-side symbolic setup: validation, per-tet rest data, BSR pattern and the atomic-free
// assembly maps; basis CSR (vertex- and handle-major), coarse S pattern, the fused Galerkin
// list and the S-block contribution lists; tile-envelope schedule of the coarse Cholesky.
//
// SURVEY §8(a) a4 (BSR assembly into precomputed slots), a5 (Galerkin projection), a6
// (factorisation); §8(b) ms_upload_mesh / ms_basis_upload semantics.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>

#include "common.cuh"

namespace msim {

static void rest_data(const double *X, const int32_t *t, double Bm[9], double &V) {
  double Dm[3][3];
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < 3; ++i) Dm[i][k] = X[3 * t[k + 1] + i] - X[3 * t[0] + i];
  const double det = Dm[0][0] * (Dm[1][1] * Dm[2][2] - Dm[1][2] * Dm[2][1]) -
                     Dm[0][1] * (Dm[1][0] * Dm[2][2] - Dm[1][2] * Dm[2][0]) +
                     Dm[0][2] * (Dm[1][0] * Dm[2][1] - Dm[1][1] * Dm[2][0]);
  V = det / 6.0;
  // inverse via adjugate
  double A[3][3];
  A[0][0] = Dm[1][1] * Dm[2][2] - Dm[1][2] * Dm[2][1];
  A[0][1] = Dm[0][2] * Dm[2][1] - Dm[0][1] * Dm[2][2];
  A[0][2] = Dm[0][1] * Dm[1][2] - Dm[0][2] * Dm[1][1];
  A[1][0] = Dm[1][2] * Dm[2][0] - Dm[1][0] * Dm[2][2];
  A[1][1] = Dm[0][0] * Dm[2][2] - Dm[0][2] * Dm[2][0];
  A[1][2] = Dm[0][2] * Dm[1][0] - Dm[0][0] * Dm[1][2];
  A[2][0] = Dm[1][0] * Dm[2][1] - Dm[1][1] * Dm[2][0];
  A[2][1] = Dm[0][1] * Dm[2][0] - Dm[0][0] * Dm[2][1];
  A[2][2] = Dm[0][0] * Dm[1][1] - Dm[0][1] * Dm[1][0];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Bm[3 * i + j] = A[i][j] / det;
}

void build_mesh_structures(Ctx &c, const double *X, const int32_t *tets, const double *E,
                           const double *nu, const double *rho) {
  const int32_t nv = c.nv, nt = c.nt;
  for (int64_t i = 0; i < (int64_t)nt * 4; ++i)
    MS_REQUIRE(tets[i] >= 0 && tets[i] < nv, MS_ERR_ARG, "tet vertex index out of range");
  for (int32_t e = 0; e < nt; ++e) {
    MS_REQUIRE(E[e] > 0.0, MS_ERR_ARG, "Young's modulus must be > 0");
    MS_REQUIRE(nu[e] >= 0.0 && nu[e] < 0.5, MS_ERR_ARG, "Poisson ratio must be in [0, 0.5)");
    MS_REQUIRE(rho[e] > 0.0, MS_ERR_ARG, "density must be > 0");
  }
  c.h_X.assign(X, X + 3 * (size_t)nv);
  c.h_tets.assign(tets, tets + 4 * (size_t)nt);

  std::vector<double> Bm((size_t)9 * nt), vol(nt), mu(nt), lam(nt), mass(nv, 0.0);
  for (int32_t e = 0; e < nt; ++e) {
    double b[9], V;
    rest_data(X, tets + 4 * (size_t)e, b, V);
    MS_REQUIRE(V > 0.0, MS_ERR_ARG, "tet with non-positive rest volume (orientation?)");
    for (int k = 0; k < 9; ++k) Bm[(size_t)k * nt + e] = b[k];
    vol[e] = V;
    mu[e] = E[e] / (2.0 * (1.0 + nu[e]));
    lam[e] = E[e] * nu[e] / ((1.0 + nu[e]) * (1.0 - 2.0 * nu[e]));
  }
  // lumped mass m_v = sum_e rho_e V_e / 4 in tet order (deterministic)
  for (int32_t e = 0; e < nt; ++e)
    for (int a = 0; a < 4; ++a) mass[tets[4 * (size_t)e + a]] += rho[e] * vol[e] / 4.0;

  // vertex -> (tet, corner) incidence, sorted by tet
  std::vector<int32_t> vptr(nv + 1, 0), vinc((size_t)4 * nt);
  for (int64_t i = 0; i < (int64_t)nt * 4; ++i) vptr[tets[i] + 1]++;
  for (int32_t v = 0; v < nv; ++v) vptr[v + 1] += vptr[v];
  {
    std::vector<int32_t> fill(vptr.begin(), vptr.end() - 1);
    for (int32_t e = 0; e < nt; ++e)
      for (int a = 0; a < 4; ++a) vinc[fill[tets[4 * (size_t)e + a]]++] = 4 * e + a;
  }
  for (int32_t v = 0; v < nv; ++v)
    MS_REQUIRE(vptr[v + 1] > vptr[v], MS_ERR_ARG, "vertex not referenced by any tet");

  // BSR pattern: row v = sorted unique vertices of incident tets (includes v)
  c.h_rowptr.assign(nv + 1, 0);
  std::vector<int32_t> colidx;
  colidx.reserve((size_t)nv * 16);
  std::vector<int32_t> buf;
  for (int32_t v = 0; v < nv; ++v) {
    buf.clear();
    for (int32_t k = vptr[v]; k < vptr[v + 1]; ++k) {
      const int32_t e = vinc[k] >> 2;
      for (int a = 0; a < 4; ++a) buf.push_back(tets[4 * (size_t)e + a]);
    }
    std::sort(buf.begin(), buf.end());
    buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
    colidx.insert(colidx.end(), buf.begin(), buf.end());
    MS_REQUIRE(colidx.size() < (size_t)INT32_MAX, MS_ERR_ARG, "BSR too large for int32");
    c.h_rowptr[v + 1] = (int32_t)colidx.size();
  }
  c.h_colidx = colidx;
  c.nnzb = (int64_t)colidx.size();
  std::vector<int32_t> diag(nv), slot_row(c.nnzb);
  for (int32_t v = 0; v < nv; ++v)
    for (int32_t k = c.h_rowptr[v]; k < c.h_rowptr[v + 1]; ++k) slot_row[k] = v;
  auto slot_of = [&](int32_t r, int32_t col) {
    const int32_t *b = colidx.data() + c.h_rowptr[r], *e = colidx.data() + c.h_rowptr[r + 1];
    return (int32_t)(std::lower_bound(b, e, col) - colidx.data());
  };
  for (int32_t v = 0; v < nv; ++v) diag[v] = slot_of(v, v);

  // slot -> contributions (tet*16 + a*4 + b), ordered by tet (deterministic gather order)
  std::vector<int32_t> cptr(c.nnzb + 1, 0);
  std::vector<int32_t> cslot((size_t)16 * nt);
  for (int32_t e = 0; e < nt; ++e)
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) {
        const int32_t s = slot_of(tets[4 * (size_t)e + a], tets[4 * (size_t)e + b]);
        cslot[(size_t)16 * e + 4 * a + b] = s;
        cptr[s + 1]++;
      }
  for (int64_t s = 0; s < c.nnzb; ++s) cptr[s + 1] += cptr[s];
  std::vector<int32_t> contrib((size_t)16 * nt);
  {
    std::vector<int32_t> fill(cptr.begin(), cptr.end() - 1);
    for (int64_t k = 0; k < (int64_t)16 * nt; ++k) contrib[fill[cslot[k]]++] = (int32_t)k;
  }

  // SELL-32 layout (sell.cuh): slice pointers, per-position column and slot
  const int32_t nslice = div_up(nv, 32);
  std::vector<int32_t> sl_ptr(nslice + 1, 0);
  for (int32_t sl = 0; sl < nslice; ++sl) {
    int32_t Ls = 0;
    for (int32_t r = 32 * sl; r < std::min(nv, 32 * sl + 32); ++r) Ls = std::max(Ls, c.h_rowptr[r + 1] - c.h_rowptr[r]);
    sl_ptr[sl + 1] = sl_ptr[sl] + Ls;
  }
  c.npos = (int64_t)sl_ptr[nslice] * 32;
  std::vector<int32_t> sell_col(c.npos), sell_slot(c.npos, -1);
  c.h_sell_pos.assign(c.nnzb, 0);
  for (int32_t sl = 0; sl < nslice; ++sl)
    for (int32_t l = 0; l < 32; ++l) {
      const int32_t r = 32 * sl + l;
      for (int32_t j = 0; j < sl_ptr[sl + 1] - sl_ptr[sl]; ++j) {
        const int64_t pos = (int64_t)(sl_ptr[sl] + j) * 32 + l;
        const bool real = r < nv && j < c.h_rowptr[r + 1] - c.h_rowptr[r];
        sell_col[pos] = real ? colidx[c.h_rowptr[r] + j] : std::min(r, nv - 1);
        if (real) {
          sell_slot[pos] = c.h_rowptr[r] + j;
          c.h_sell_pos[c.h_rowptr[r] + j] = pos;
        }
      }
    }

  cudaStream_t s = c.stream;
  c.sl_ptr.upload(sl_ptr, s);
  c.sell_col.upload(sell_col, s);
  c.sell_slot.upload(sell_slot, s);
  c.X.upload(X, 3 * (size_t)nv, s);
  c.tets.upload(tets, 4 * (size_t)nt, s);
  c.Bm.upload(Bm, s);
  c.vol.upload(vol, s);
  c.mu.upload(mu, s);
  c.lam.upload(lam, s);
  c.mass.upload(mass, s);
  c.vinc_ptr.upload(vptr, s);
  c.vinc.upload(vinc, s);
  c.rowptr.upload(c.h_rowptr, s);
  c.colidx.upload(c.h_colidx, s);
  c.diag_slot.upload(diag, s);
  {
    std::vector<int32_t> dpos(nv);
    for (int32_t v = 0; v < nv; ++v) dpos[v] = (int32_t)c.h_sell_pos[diag[v]];
    c.diag_pos.upload(dpos, s);
  }
  c.n_cub = 0;
  c.lag_valid = false;
  if (c.dist()) {   // interior owned rows: one contiguous run between the rows that read ghosts
    const int32_t no = c.nv_own;
    std::vector<uint8_t> touch(no, 0);
    for (int32_t r = 0; r < no; ++r)
      for (int32_t k = c.h_rowptr[r]; k < c.h_rowptr[r + 1]; ++k)
        if (c.h_colidx[k] >= no) touch[r] = 1;
    int32_t lo = 0, hi = no;
    for (int32_t r = 0; r < no / 2; ++r)
      if (touch[r]) lo = r + 1;
    for (int32_t r = no - 1; r >= no / 2; --r)
      if (touch[r]) hi = r;
    bool ok = lo < hi;
    for (int32_t r = lo; ok && r < hi; ++r) ok = !touch[r];
    c.int_lo = ok ? lo : 0;
    c.int_hi = ok ? hi : 0;
    if (!c.halo_stream) {   // created here, not lazily inside a graph capture
      MS_CUDA(cudaStreamCreateWithFlags(&c.halo_stream, cudaStreamNonBlocking));
      MS_CUDA(cudaEventCreateWithFlags(&c.ev_z, cudaEventDisableTiming));
      MS_CUDA(cudaEventCreateWithFlags(&c.ev_halo, cudaEventDisableTiming));
    }
  }
  c.slot_row.upload(slot_row, s);
  c.cptr.upload(cptr, s);
  c.contrib.upload(contrib, s);
  c.vals.alloc((size_t)9 * c.npos);
  c.h_fixed.assign(nv, 0);
  c.fixed.upload(c.h_fixed, s);
  ensure_state_buffers(c);
  MS_CUDA(cudaStreamSynchronize(s));
}

void ensure_state_buffers(Ctx &c) {
  const size_t n3 = 3 * (size_t)c.nv;
  for (DBuf<double> *b : {&c.x, &c.v, &c.xt, &c.xhat, &c.g, &c.ds, &c.da, &c.df, &c.d, &c.r, &c.rhs,
                          &c.p, &c.q, &c.z, &c.tmp, &c.dinv})
    b->alloc(n3);
  c.stage_g.alloc((size_t)12 * c.nt);
  c.stage_h.alloc((size_t)kStageH * c.nt);
  c.hess_work.alloc((size_t)c.nt);
  c.hess_nwork.alloc(1);
  c.max_blocks = std::max(div_up(c.nt, 128), div_up(c.nv, 128)) + 1024;
  c.partial.alloc((size_t)c.max_blocks * (kMaxLS + 2));
  c.counters.alloc(64);
  c.counters.zero(c.stream);
  c.scal.alloc(SC_COUNT);
  c.scal.zero(c.stream);
  c.flags.alloc(8);
  c.flags.zero(c.stream);
  c.ls_alpha.alloc(kMaxLS);
  c.ls_out.alloc(3 * kMaxLS);   // [K] energy differences, [K] steps, [K] infeasible counts (multi-GPU)
  // rest state: x = X, v = 0
  MS_CUDA(cudaMemcpyAsync(c.x, c.X, sizeof(double) * n3, cudaMemcpyDeviceToDevice, c.stream));
  c.v.zero(c.stream);
  MS_CUDA(cudaMemcpyAsync(c.xt, c.X, sizeof(double) * n3, cudaMemcpyDeviceToDevice, c.stream));
  MS_CUDA(cudaMemcpyAsync(c.xhat, c.X, sizeof(double) * n3, cudaMemcpyDeviceToDevice, c.stream));
}

// ------------------------------------------------------------------------- basis
// Global S pattern (multi-GPU): handles i, j are coupled when some vertex of supp(i) is a
// neighbour (or equal) of a vertex of supp(j) in the global mesh.
void global_s_pattern(int32_t nv, const std::vector<int32_t> &tets, int32_t m, const int64_t *vptr,
                      const int32_t *handle, std::vector<int32_t> &sptr, std::vector<int32_t> &scol) {
  const int64_t nt = (int64_t)tets.size() / 4;
  std::vector<int32_t> aptr(nv + 1, 0), adj;
  {
    std::vector<std::vector<int32_t>> nb(nv);
    for (int64_t e = 0; e < nt; ++e)
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) nb[tets[4 * e + a]].push_back(tets[4 * e + b]);
    for (int32_t v = 0; v < nv; ++v) {
      auto &l = nb[v];
      l.push_back(v);
      std::sort(l.begin(), l.end());
      l.erase(std::unique(l.begin(), l.end()), l.end());
      adj.insert(adj.end(), l.begin(), l.end());
      aptr[v + 1] = (int32_t)adj.size();
      std::vector<int32_t>().swap(l);
    }
  }
  std::vector<std::vector<int32_t>> supp(m);
  for (int32_t v = 0; v < nv; ++v)
    for (int64_t k = vptr[v]; k < vptr[v + 1]; ++k) supp[handle[k]].push_back(v);
  std::vector<int32_t> mark(m, -1), row;
  sptr.assign(1, 0);
  scol.clear();
  for (int32_t i = 0; i < m; ++i) {
    row.clear();
    for (int32_t v : supp[i])
      for (int32_t a = aptr[v]; a < aptr[v + 1]; ++a) {
        const int32_t u = adj[a];
        for (int64_t k = vptr[u]; k < vptr[u + 1]; ++k)
          if (mark[handle[k]] != i) {
            mark[handle[k]] = i;
            row.push_back(handle[k]);
          }
      }
    std::sort(row.begin(), row.end());
    scol.insert(scol.end(), row.begin(), row.end());
    sptr.push_back((int32_t)scol.size());
  }
}

// Dependency graph of the dataflow factorisation's tasks (chol.cu k_chol_dataflow): per task the
// number of inputs and its successors.  A type-4 task (P(k+1,k) U(k+1,k+1,k) D(k+1)) releases
// the readers of its panel tile P(k+1,k) before D(k+1): [succ_ptr, succ_mid) are those,
// [succ_mid, succ_ptr+1) the readers of D(k+1) and of the diagonal tile's update count.  (A
// queue task must never wait on an uncounted input: all queue CTAs could end up waiting on the
// chain while the chain waits on a queued task.)
static void dataflow_graph(const std::vector<int32_t> &dag, int NT, std::vector<int32_t> &succ_ptr,
                           std::vector<int32_t> &succ_mid, std::vector<int32_t> &succ, std::vector<int32_t> &ndep) {
  const int n = (int)(dag.size() / 4);
  std::vector<int32_t> dfl(NT, -1), pfl((size_t)NT * NT, -1);
  std::vector<std::vector<int32_t>> updt((size_t)NT * NT);
  auto put = [](std::vector<int32_t> &v, int r, int32_t q) {
    if ((int)v.size() <= r) v.resize(r + 1, -1);
    v[r] = q;
  };
  for (int q = 0; q < n; ++q) {
    const int ty = dag[4 * q], i = dag[4 * q + 1], j = dag[4 * q + 2] & 0xffff, k = dag[4 * q + 2] >> 16,
              cnt = dag[4 * q + 3];
    if (ty == 0) dfl[k] = q;
    else if (ty == 4) {
      dfl[i] = q;
      pfl[(size_t)i * NT + k] = q;
      put(updt[(size_t)i * NT + i], cnt >> 16, q);
    } else if (ty == 1) pfl[(size_t)i * NT + k] = q;
    else put(updt[(size_t)i * NT + j], cnt, q);
  }
  std::vector<std::vector<int32_t>> early(n), late(n);
  ndep.assign(n, 0);
  auto dep = [&](int q, int32_t d, bool via_panel) {
    MS_REQUIRE(d >= 0 && d < q, MS_ERR_STATE, "tile DAG: dependency missing or out of order");
    (via_panel && dag[4 * d] == 4 ? early : late)[d].push_back(q);
    ndep[q]++;
  };
  for (int q = 0; q < n; ++q) {
    const int ty = dag[4 * q], i = dag[4 * q + 1], j = dag[4 * q + 2] & 0xffff, k = dag[4 * q + 2] >> 16,
              cnt = dag[4 * q + 3];
    if (ty == 0) {
      if (cnt) dep(q, updt[(size_t)k * NT + k][cnt - 1], false);
    } else if (ty == 4) {
      if (cnt & 0xffff) dep(q, updt[(size_t)i * NT + k][(cnt & 0xffff) - 1], false);
      if (cnt >> 16) dep(q, updt[(size_t)i * NT + i][(cnt >> 16) - 1], false);
      dep(q, dfl[k], false);
    } else if (ty == 1) {
      dep(q, dfl[k], false);
      if (cnt) dep(q, updt[(size_t)i * NT + k][cnt - 1], false);
    } else {
      dep(q, pfl[(size_t)i * NT + k], true);
      if (j != i) dep(q, pfl[(size_t)j * NT + k], true);
      if (cnt) dep(q, updt[(size_t)i * NT + j][cnt - 1], false);
    }
  }
  succ_ptr.assign(n + 1, 0);
  succ_mid.assign(n, 0);
  succ.clear();
  for (int q = 0; q < n; ++q) {
    succ.insert(succ.end(), early[q].begin(), early[q].end());
    succ_mid[q] = (int32_t)succ.size();
    succ.insert(succ.end(), late[q].begin(), late[q].end());
    succ_ptr[q + 1] = (int32_t)succ.size();
  }
}

void build_basis_structures(Ctx &c, int32_t m, const double *origins, const int64_t *vptr,
                            const int32_t *handle, const double *phi, const double *phi_aff,
                            const double aff_origin[3]) {
  const int32_t nv = c.nv;
  MS_REQUIRE(m > 0, MS_ERR_ARG, "m must be > 0");
  MS_REQUIRE(vptr[0] == 0, MS_ERR_ARG, "vptr[0] must be 0");
  const int64_t nnz = vptr[nv];
  MS_REQUIRE(nnz < INT32_MAX, MS_ERR_ARG, "basis too large for int32 indices");
  for (int32_t v = 0; v < nv; ++v) {
    MS_REQUIRE(vptr[v + 1] >= vptr[v], MS_ERR_ARG, "vptr not monotone");
    double sum = 0.0;
    for (int64_t k = vptr[v]; k < vptr[v + 1]; ++k) {
      MS_REQUIRE(handle[k] >= 0 && handle[k] < m, MS_ERR_ARG, "handle id out of range");
      MS_REQUIRE(k == vptr[v] || handle[k] > handle[k - 1], MS_ERR_ARG,
                 "handles of a vertex must be strictly increasing");
      MS_REQUIRE(phi[k] > 0.0, MS_ERR_ARG, "phi entries must be > 0");
      sum += phi[k];
    }
    // pinned vertices never move: every basis column must vanish there
    MS_REQUIRE(!c.h_fixed[v] || (vptr[v + 1] == vptr[v] && phi_aff[v] == 0.0), MS_ERR_ARG,
               "basis does not vanish at a Dirichlet vertex (set the Dirichlet set before the basis)");
    // POU: sum phi + phi_DBC = 1 with phi_DBC = 1 - phi_affine; a hole is sum phi = phi_DBC = 0
    MS_REQUIRE(sum > 0.0 || c.h_fixed[v] || phi_aff[v] < 1.0, MS_ERR_COVERAGE,
               "basis coverage hole: no handle covers a free vertex");
  }
  c.m = m;
  c.nnz_phi = nnz;
  c.h_bvptr.assign(vptr, vptr + nv + 1);
  c.h_bhandle.assign(handle, handle + nnz);
  c.cpcg_ready = false;
  std::vector<int32_t> bvptr(nv + 1);
  for (int32_t v = 0; v <= nv; ++v) bvptr[v] = (int32_t)vptr[v];
  // handle-major transpose (sorted by vertex)
  std::vector<int32_t> hptr(m + 1, 0), hvert(nnz), hidx(nnz);
  std::vector<double> hphi(nnz);
  for (int64_t k = 0; k < nnz; ++k) hptr[handle[k] + 1]++;
  for (int32_t i = 0; i < m; ++i) hptr[i + 1] += hptr[i];
  {
    std::vector<int32_t> fill(hptr.begin(), hptr.end() - 1);
    for (int32_t v = 0; v < nv; ++v)
      for (int64_t k = vptr[v]; k < vptr[v + 1]; ++k) {
        const int32_t pos = fill[handle[k]]++;
        hvert[pos] = v;
        hphi[pos] = phi[k];
        hidx[pos] = (int32_t)k;
      }
  }
  if (!c.dist())   // (a rank's slab need not meet every handle's support)
    for (int32_t i = 0; i < m; ++i)
      MS_REQUIRE(hptr[i + 1] > hptr[i], MS_ERR_ARG, "handle with empty support");

  // U_i = vertices adjacent (BSR) to supp(i); J_i = handles of U_i (the S pattern row i);
  // fused Galerkin lists (coarse.cu k_galerkin_fused): per handle i, per chunk of kGalChunk
  // vertices of U_i, per upper slot j >= i of J_i the entries (u_local | p << 7) with p the
  // basis entry of (u, j).
  std::vector<int32_t> mark(nv, -1), hmark(m, -1), jslot(m, -1);
  std::vector<int32_t> sptr(1, 0), scol;
  const int32_t *rp = c.h_rowptr.data(), *ci = c.h_colidx.data();
  std::vector<int32_t> Uptr(m + 1, 0), Uall;
  for (int32_t i = 0; i < m; ++i) {
    const size_t b0 = Uall.size();
    for (int32_t k = hptr[i]; k < hptr[i + 1]; ++k) {
      const int32_t v = hvert[k];
      for (int32_t s = rp[v]; s < rp[v + 1]; ++s) {
        const int32_t u = ci[s];
        if (u >= c.nv_own) continue;   // multi-GPU: a rank projects its owned rows only
        if (mark[u] != i) {
          mark[u] = i;
          Uall.push_back(u);
        }
      }
    }
    std::sort(Uall.begin() + b0, Uall.end());   // vertex order: coalesced SELL row reads
    Uptr[i + 1] = (int32_t)Uall.size();
  }
  MS_REQUIRE(nnz < (int64_t(1) << 25), MS_ERR_ARG, "basis too large for the fused Galerkin entry encoding");
  // per (i, u) pair: the Hessian row slots j of u whose vertex v lies in supp(i): (j | p << 6)
  std::vector<int32_t> ga_off(1, 0);
  std::vector<uint32_t> ga_ent;
  std::vector<unsigned long long> ga_mask;   // bit j: slot j of row u is in the list
  ga_off.reserve(Uall.size() + 1);
  ga_mask.reserve(Uall.size());
  for (int32_t i = 0; i < m; ++i)
    for (int32_t q = Uptr[i]; q < Uptr[i + 1]; ++q) {
      const int32_t u = Uall[q];
      MS_REQUIRE(rp[u + 1] - rp[u] <= 64, MS_ERR_ARG, "Hessian row longer than 64 blocks (Galerkin encoding)");
      unsigned long long mask = 0;
      for (int32_t j = 0; j < rp[u + 1] - rp[u]; ++j) {
        const int32_t v = ci[rp[u] + j];
        const int32_t *hb = handle + vptr[v], *he = handle + vptr[v + 1];
        const int32_t *f = std::lower_bound(hb, he, i);
        if (f != he && *f == i) {
          ga_ent.push_back((uint32_t)j | ((uint32_t)(vptr[v] + (f - hb)) << 6));
          mask |= 1ull << j;
        }
      }
      ga_mask.push_back(mask);
      MS_REQUIRE(ga_ent.size() < (size_t)INT32_MAX, MS_ERR_ARG, "Galerkin pair list too large");
      ga_off.push_back((int32_t)ga_ent.size());
    }
  std::vector<int32_t> gj_ptr(m + 1, 0), gj_blk, gl_base(m + 1, 0), gl_off;
  std::vector<uint32_t> gl_ent;
  std::vector<int32_t> Jl;
  std::vector<std::vector<uint32_t>> lists;
  int32_t max_jup = 0;
  for (int32_t i = 0; i < m; ++i) {
    Jl.clear();
    if (c.dist()) {   // the global S pattern (identical on all ranks: S is summed across ranks)
      Jl.assign(c.h_scol_glob.begin() + c.h_sptr_glob[i], c.h_scol_glob.begin() + c.h_sptr_glob[i + 1]);
    } else {
      for (int32_t q = Uptr[i]; q < Uptr[i + 1]; ++q) {
        const int32_t u = Uall[q];
        for (int64_t k = vptr[u]; k < vptr[u + 1]; ++k)
          if (hmark[handle[k]] != i) {
            hmark[handle[k]] = i;
            Jl.push_back(handle[k]);
          }
      }
      std::sort(Jl.begin(), Jl.end());
    }
    const int32_t row0 = (int32_t)scol.size();
    scol.insert(scol.end(), Jl.begin(), Jl.end());
    sptr.push_back((int32_t)scol.size());
    const int32_t first_up = (int32_t)(std::lower_bound(Jl.begin(), Jl.end(), i) - Jl.begin());
    const int32_t nup = (int32_t)Jl.size() - first_up;
    max_jup = std::max(max_jup, nup);
    for (int32_t q = 0; q < nup; ++q) {
      jslot[Jl[first_up + q]] = q;
      gj_blk.push_back(row0 + first_up + q);
    }
    gj_ptr[i + 1] = (int32_t)gj_blk.size();
    const int32_t nU = Uptr[i + 1] - Uptr[i];
    const int32_t nch = (nU + kGalChunk - 1) / kGalChunk;
    gl_base[i + 1] = gl_base[i] + nch * (nup + 1);
    lists.assign(nup, {});
    for (int32_t ch = 0; ch < nch; ++ch) {
      for (auto &l : lists) l.clear();
      for (int32_t t = 0; t < kGalChunk && ch * kGalChunk + t < nU; ++t) {
        const int32_t u = Uall[Uptr[i] + ch * kGalChunk + t];
        for (int64_t k = vptr[u]; k < vptr[u + 1]; ++k)
          if (handle[k] >= i) lists[jslot[handle[k]]].push_back((uint32_t)t | ((uint32_t)k << 7));
      }
      for (int32_t q = 0; q < nup; ++q) {
        gl_off.push_back((int32_t)gl_ent.size());
        gl_ent.insert(gl_ent.end(), lists[q].begin(), lists[q].end());
      }
      gl_off.push_back((int32_t)gl_ent.size());
      MS_REQUIRE(gl_ent.size() < (size_t)INT32_MAX, MS_ERR_ARG, "coarse contribution list too large");
    }
  }
  c.h_sptr = sptr;
  c.h_scol = scol;
  c.nnzb_S = (int64_t)scol.size();
  c.gal_max_jup = max_jup;
  // Galerkin arithmetic: 36 FMA per (i,u,v) term of R, 144 per (i,j,u) term of S (upper)
  c.chol_info.galerkin_flops = 2.0 * (36.0 * (double)ga_ent.size() + 144.0 * (double)gl_ent.size());

  // ---- fill-reducing order of the handles: geometric nested dissection on the coupling graph
  // (one-sided vertex separators from recursive median bisection of the handle origins).
  std::vector<int32_t> order;
  order.reserve(m);
  {
    std::vector<char> side(m, 0);
    std::vector<int32_t> all(m);
    std::iota(all.begin(), all.end(), 0);
    struct Rec { std::vector<int32_t> h; };
    std::function<void(std::vector<int32_t> &)> nd = [&](std::vector<int32_t> &H) {
      if (H.size() <= 8) {
        order.insert(order.end(), H.begin(), H.end());
        return;
      }
      double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
      for (int32_t h : H)
        for (int d = 0; d < 3; ++d) {
          lo[d] = std::min(lo[d], origins[3 * h + d]);
          hi[d] = std::max(hi[d], origins[3 * h + d]);
        }
      int ax = 0;
      for (int d = 1; d < 3; ++d)
        if (hi[d] - lo[d] > hi[ax] - lo[ax]) ax = d;
      std::stable_sort(H.begin(), H.end(), [&](int32_t a, int32_t b) {
        return origins[3 * a + ax] < origins[3 * b + ax];
      });
      const size_t half = H.size() / 2;
      for (size_t q = 0; q < H.size(); ++q) side[H[q]] = q < half ? 1 : 2;
      std::vector<int32_t> A(H.begin(), H.begin() + half), B, Sep;
      for (size_t q = half; q < H.size(); ++q) {
        const int32_t b = H[q];
        bool touches = false;
        for (int32_t k = sptr[b]; k < sptr[b + 1] && !touches; ++k) touches = side[scol[k]] == 1;
        (touches ? Sep : B).push_back(b);
      }
      for (int32_t h : H) side[h] = 0;
      if (B.empty()) {   // no separation possible: keep as one dense block
        order.insert(order.end(), H.begin(), H.end());
        return;
      }
      nd(A);
      nd(B);
      order.insert(order.end(), Sep.begin(), Sep.end());
    };
    nd(all);
  }
  // ---- tile-level symbolic Cholesky for a handle order; the cheaper of the x-sorted order
  // (handles arrive sorted by centroid) and the nested-dissection order is kept.
  c.nS = 12 * m;
  c.tile = 64;
  c.ntiles = div_up(c.nS, c.tile);
  c.nS_pad = c.ntiles * c.tile;
  const int T = c.tile, NT = c.ntiles;
  struct Sym {
    std::vector<int32_t> perm;
    std::vector<std::vector<int32_t>> panel, rows;
    std::vector<std::vector<char>> nz;
    double flops = 0.0;
    int64_t ntask = 0;
    int32_t crit = 0;
  };
  auto symbolic = [&](const std::vector<int32_t> &ord) {
    Sym y;
    y.perm.assign(m, 0);
    for (int32_t p = 0; p < m; ++p) y.perm[ord[p]] = p;
    y.nz.assign(NT, std::vector<char>(NT, 0));
    for (int32_t t = 0; t < NT; ++t) y.nz[t][t] = 1;
    for (int32_t i = 0; i < m; ++i)
      for (int32_t k = sptr[i]; k < sptr[i + 1]; ++k) {
        const int32_t pi = y.perm[i], pj = y.perm[scol[k]];
        for (int32_t a = 12 * pi / T; a <= (12 * pi + 11) / T; ++a)
          for (int32_t b = 12 * pj / T; b <= (12 * pj + 11) / T; ++b)
            if (a >= b) y.nz[a][b] = 1;
      }
    y.panel.assign(NT, {});
    y.rows.assign(NT, {});
    for (int32_t k = 0; k < NT; ++k) {
      auto &P = y.panel[k];
      for (int32_t i = k + 1; i < NT; ++i)
        if (y.nz[i][k]) P.push_back(i);
      for (size_t a = 0; a < P.size(); ++a)
        for (size_t b = 0; b <= a; ++b) y.nz[P[a]][P[b]] = 1;
      for (int32_t i : P) y.rows[i].push_back(k);
      const double np = (double)P.size();
      y.flops += (double)T * T * T / 3.0 + np * T * T * T + np * (np + 1) * T * T * T;
      y.ntask += 1 + (int64_t)P.size() + (int64_t)(P.size() * (P.size() + 1) / 2);
    }
    // critical path of the tile DAG in tasks (D(k) -> P(i,k) -> U(i,j,k) -> ..., updates of a
    // tile applied in k order)
    std::vector<int32_t> ready((size_t)NT * NT, 0), pk(NT, 0);
    for (int32_t k = 0; k < NT; ++k) {
      const int32_t dk = ready[(size_t)k * NT + k] + 1;
      for (int32_t i : y.panel[k]) pk[i] = std::max(dk, ready[(size_t)i * NT + k]) + 1;
      const auto &P = y.panel[k];
      for (size_t a = 0; a < P.size(); ++a)
        for (size_t b = 0; b <= a; ++b) {
          int32_t &r = ready[(size_t)P[a] * NT + P[b]];
          r = std::max(r, std::max(pk[P[a]], pk[P[b]])) + 1;
        }
      y.crit = dk;
    }
    return y;
  };
  std::vector<int32_t> ident(m);
  std::iota(ident.begin(), ident.end(), 0);
  Sym sx = symbolic(ident), snd = symbolic(order);
  const char *ord_env = std::getenv("MSIM_COARSE_ORDER");   // "x" / "nd": force (diagnostics)
  Sym &best = ord_env ? (ord_env[0] == 'n' ? snd : sx) : (snd.flops < sx.flops ? snd : sx);
  c.h_perm = best.perm;
  c.chol_flops = best.flops;
  c.chol_info.n_s = c.nS;
  c.chol_info.tile = T;
  c.chol_info.ntiles = NT;
  c.chol_info.ordering = &best == &snd ? 1 : 0;
  c.chol_info.flops = best.flops;
  c.chol_info.flops_xorder = sx.flops;
  c.chol_info.flops_nd = snd.flops;
  c.chol_info.n_tasks = best.ntask;
  c.chol_info.critical_path = best.crit;
  c.chol_info.critical_path_xorder = sx.crit;
  c.chol_info.critical_path_nd = snd.crit;
  c.chol_info.nnzb_s = c.nnzb_S;
  {
    int64_t nzt = 0;
    for (int32_t i = 0; i < NT; ++i)
      for (int32_t j = 0; j <= i; ++j) nzt += best.nz[i][j];
    c.chol_info.lower_tiles = nzt;
  }
  c.h_chol_panel = best.panel;
  std::vector<int32_t> panel_flat, rows_flat, sym_tiles;
  std::vector<int32_t> panel_ptr(NT + 1, 0), rows_ptr(NT + 1, 0);
  c.h_chol_panel_off.assign(NT + 1, 0);
  c.h_chol_rows_off.assign(NT + 1, 0);
  for (int32_t k = 0; k < NT; ++k) {
    const auto &P = best.panel[k];
    panel_flat.insert(panel_flat.end(), P.begin(), P.end());
    rows_flat.insert(rows_flat.end(), best.rows[k].begin(), best.rows[k].end());
    c.h_chol_panel_off[k + 1] = (int64_t)panel_flat.size();
    c.h_chol_rows_off[k + 1] = (int64_t)rows_flat.size();
    panel_ptr[k + 1] = (int32_t)panel_flat.size();
    rows_ptr[k + 1] = (int32_t)rows_flat.size();
    for (int32_t i = k; i < NT; ++i)
      if (best.nz[i][k]) {
        sym_tiles.push_back(i);
        sym_tiles.push_back(k);
      }
  }
  c.n_sym_tiles = (int64_t)sym_tiles.size() / 2;

  // dataflow task list (chol.cu k_chol_dataflow): D(0); per k: P(.,k); U(.,k+1,k); D(k+1); U(rest,k)
  std::vector<int32_t> dag;
  {
    std::vector<int32_t> nupd((size_t)NT * NT, 0);
    auto emit = [&](int type, int i, int j, int k, int cnt) {
      dag.push_back(type);
      dag.push_back(i);
      dag.push_back(j | (k << 16));
      dag.push_back(cnt);
    };
    MS_REQUIRE(NT < 32768, MS_ERR_ARG, "coarse matrix too large for the tile DAG encoding");
    emit(0, 0, 0, 0, 0);
    for (int32_t k = 0; k < NT; ++k) {
      const auto &P = best.panel[k];
      const bool next_in = !P.empty() && P.front() == k + 1;
      if (next_in) {   // critical path first: P(k+1,k) + U(k+1,k+1,k) + D(k+1) in one task (type 4)
        const int32_t need = nupd[(size_t)(k + 1) * NT + k];
        const int32_t rank = nupd[(size_t)(k + 1) * NT + k + 1]++;
        MS_REQUIRE(need < 65536 && rank < 65536, MS_ERR_ARG, "tile DAG counter overflow");
        emit(4, k + 1, k + 1, k, need | (rank << 16));
      }
      for (int32_t i : P)
        if (!(next_in && i == k + 1)) emit(1, i, 0, k, nupd[(size_t)i * NT + k]);
      if (next_in)
        for (size_t a = 1; a < P.size(); ++a) {       // rest of column k+1
          const int32_t i = P[a];
          emit(2, i, k + 1, k, nupd[(size_t)i * NT + k + 1]++);
        }
      else if (k + 1 < NT)
        emit(0, 0, 0, k + 1, nupd[(size_t)(k + 1) * NT + k + 1]);
      for (size_t a = 0; a < P.size(); ++a)
        for (size_t b = 0; b <= a; ++b) {
          const int32_t i = P[a], j = P[b];
          if (next_in && j == k + 1) continue;
          emit(2, i, j, k, nupd[(size_t)i * NT + j]++);
        }
    }
  }
  c.n_dag = (int64_t)dag.size() / 4;
  // CTA 0 of k_chol_dataflow runs the fused diagonal chain (type 4) in order; every other task
  // is handed out through one of two ready queues (served by disjoint CTA sets) as soon as its
  // inputs exist
  std::vector<int32_t> crit, succ_ptr, succ_mid, succ, ndep;
  dataflow_graph(dag, NT, succ_ptr, succ_mid, succ, ndep);
  {
    const char *e = std::getenv("MSIM_GAL_PARTS");   // tuning / diagnostics
    c.gal_parts = e ? std::max(1, std::atoi(e)) : 4;
  }
  // ---- fused Galerkin (single GPU): the Galerkin rows of S are tasks of the same dataflow
  // launch, G(i, part) (a quarter of handle i's row, galerkin.cuh) and R(i) (sum of the parts in
  // a fixed order, scattered into the factor's tiles).  The task that first reads a tile's
  // unfactored values (the first update / panel / diagonal factor of that tile) waits for every
  // R(i) that writes into it: counted inputs for queue tasks, flag waits (rwait) for CTA 0's
  // chain.  G tasks are the only initially ready tasks, queued in handle order, so the rows of
  // the first tile columns are formed first and the factorisation starts while the rest of S is
  // still being projected.
  std::vector<int32_t> rw_ptr(1, 0), rw;
  {
    // opt-in (MSIM_GAL_FUSED=1): measured at C4 it does not pay yet -- the Galerkin rows are
    // throughput-bound (~2.2 ms of the whole GPU), so running them inside the factor launch only
    // delays the factor's own bulk updates (4.6 -> 4.7 ms for S + factor)
    const char *e = std::getenv("MSIM_GAL_FUSED");
    bool has_chain = false;
    for (int64_t q = 0; q < c.n_dag; ++q) has_chain |= dag[4 * q] == 4;
    // two CTAs per SM must still fit beside the Galerkin rows' shared memory (chol.cu)
    const bool fits = sizeof(double) * galerkin_smem_doubles(max_jup) <= 110 * 1024;
    c.gal_fused = !c.dist() && (e && e[0] == '1') && c.gal_parts > 1 && has_chain && fits;
  }
  c.n_dag_factor = c.n_dag;
  if (c.gal_fused) {
    const int64_t n0 = c.n_dag, np = c.gal_parts;
    const int64_t gid0 = n0, rid0 = n0 + (int64_t)m * np;
    // raw reader of every tile: the task that first reads its unfactored values
    std::vector<int32_t> raw((size_t)NT * NT, -1);
    for (int64_t q = 0; q < n0; ++q) {
      const int ty = dag[4 * q], i = dag[4 * q + 1], j = dag[4 * q + 2] & 0xffff, k = dag[4 * q + 2] >> 16,
                cnt = dag[4 * q + 3];
      auto mark_raw = [&](int a, int b) {
        if (raw[(size_t)a * NT + b] < 0) raw[(size_t)a * NT + b] = (int32_t)q;
      };
      if (ty == 0 && cnt == 0) mark_raw(k, k);
      if (ty == 4) {
        if ((cnt & 0xffff) == 0) mark_raw(i, k);
        if ((cnt >> 16) == 0) mark_raw(i, i);
      }
      if (ty == 1 && cnt == 0) mark_raw(i, k);
      if (ty == 2 && cnt == 0) mark_raw(i, j);
    }
    // R(i) -> raw readers of the tiles its blocks S_ij (j >= i, both triangles' lower images) hit
    std::vector<std::vector<int32_t>> rsucc(m);
    std::vector<std::vector<int32_t>> chain_wait(c.n_dag);   // type-4 raw readers: handles to wait for
    for (int32_t i = 0; i < m; ++i) {
      const int pi = 12 * c.h_perm[i];
      const int ti0 = pi / T, ti1 = (pi + 11) / T;
      std::vector<int32_t> succ_i;
      for (int32_t b = gj_ptr[i]; b < gj_ptr[i + 1]; ++b) {
        const int32_t j = scol[gj_blk[b]];
        const int pj = 12 * c.h_perm[j];
        const int tj0 = pj / T, tj1 = (pj + 11) / T;
        for (int a = ti0; a <= ti1; ++a)
          for (int bb = tj0; bb <= tj1; ++bb) {
            const int I = std::max(a, bb), J = std::min(a, bb);
            const int32_t q = raw[(size_t)I * NT + J];
            MS_REQUIRE(q >= 0, MS_ERR_STATE, "fused Galerkin: S block outside the symbolic factor");
            if (dag[4 * q] == 4) chain_wait[q].push_back(i);
            else succ_i.push_back(q);
          }
      }
      std::sort(succ_i.begin(), succ_i.end());
      succ_i.erase(std::unique(succ_i.begin(), succ_i.end()), succ_i.end());
      for (int32_t q : succ_i) ndep[q]++;
      rsucc[i] = std::move(succ_i);
    }
    // append the tasks: G(i, p) = gid0 + i np + p, R(i) = rid0 + i
    for (int32_t i = 0; i < m; ++i)
      for (int p = 0; p < np; ++p) {
        dag.push_back(5);
        dag.push_back(i);
        dag.push_back(p);
        dag.push_back(0);
      }
    for (int32_t i = 0; i < m; ++i) {
      dag.push_back(6);
      dag.push_back(i);
      dag.push_back(0);
      dag.push_back(0);
    }
    for (int32_t i = 0; i < m; ++i)
      for (int p = 0; p < np; ++p) {
        succ_mid.push_back((int32_t)succ.size());
        succ.push_back((int32_t)(rid0 + i));
        succ_ptr.push_back((int32_t)succ.size());
        ndep.push_back(0);
      }
    for (int32_t i = 0; i < m; ++i) {
      succ_mid.push_back((int32_t)succ.size());
      succ.insert(succ.end(), rsucc[i].begin(), rsucc[i].end());
      succ_ptr.push_back((int32_t)succ.size());
      ndep.push_back((int32_t)np);
    }
    (void)gid0;
    c.n_dag = (int64_t)dag.size() / 4;
    for (int64_t q = 0; q < n0; ++q)
      if (dag[4 * q] == 4) {
        auto &l = chain_wait[q];
        std::sort(l.begin(), l.end());
        l.erase(std::unique(l.begin(), l.end()), l.end());
        rw.insert(rw.end(), l.begin(), l.end());
        rw_ptr.push_back((int32_t)rw.size());
      }
  }
  std::vector<uint8_t> cls(c.n_dag, 0);
  c.n_pool = 0;
  int hi_dj = 2;   // measured best at C4 (2..4)
  {
    const char *e = std::getenv("MSIM_DF_HIDJ");
    if (e) hi_dj = std::max(1, std::atoi(e));
  }
  for (int64_t q = 0; q < c.n_dag; ++q) {
    const int ty = dag[4 * q], i = dag[4 * q + 1], j = dag[4 * q + 2] & 0xffff, k = dag[4 * q + 2] >> 16;
    // high: diagonal factors, panel tiles, and the updates of tiles that become panel tiles
    // within hi_dj steps: each band row is a chain P(i,k) -> U(i,k+1,k) -> P(i,k+1) -> ... fed by
    // the update chains of its tiles, which must not queue behind the bulk updates
    cls[q] = ty == 4 ? 2 : ty == 5 ? 0 : ty == 6 ? 1 : (ty == 0 || ty == 1 || j <= k + hi_dj) ? 1 : 0;
    if (ty == 4) crit.push_back((int32_t)q);
    else c.n_pool++;
  }
  {
    const char *e = std::getenv("MSIM_DF_HI");   // CTAs serving the high-priority queue
    c.df_hi_ctas = e ? std::max(1, std::atoi(e)) : 64;   // measured at C4 (48..80 at 2 CTAs per SM)
  }
  c.n_crit = (int64_t)crit.size();
  // queue q (0: low, 1: high) at offset q * (n_pool + 2): head, tail, entries (-1: not yet pushed)
  std::vector<int32_t> queue0((size_t)2 * (c.n_pool + 2) + 1, -1);   // + finished-task count
  queue0.back() = 0;
  for (int qq = 0; qq < 2; ++qq) {
    int32_t *Q = queue0.data() + (size_t)qq * (c.n_pool + 2);
    Q[0] = Q[1] = 0;
    for (int64_t q = 0; q < c.n_dag; ++q)
      if (cls[q] == qq && !ndep[q]) Q[2 + Q[1]++] = (int32_t)q;
  }
  if (crit.empty()) crit.push_back(0);

  cudaStream_t s = c.stream;
  c.origins.upload(origins, 3 * (size_t)m, s);
  c.bvptr.upload(bvptr, s);
  c.bhandle.upload(handle, nnz, s);
  c.bphi.upload(phi, nnz, s);
  if (c.dist()) {   // B^T restricts over the owned vertices (summed across ranks)
    std::vector<int32_t> optr(m + 1, 0), overt;
    std::vector<double> ophi;
    for (int32_t i = 0; i < m; ++i) {
      for (int32_t k = hptr[i]; k < hptr[i + 1]; ++k)
        if (hvert[k] < c.nv_own) {
          overt.push_back(hvert[k]);
          ophi.push_back(hphi[k]);
        }
      optr[i + 1] = (int32_t)overt.size();
    }
    c.hptr.upload(optr, s);
    c.hvert.upload(overt.empty() ? std::vector<int32_t>{0} : overt, s);
    c.hphi.upload(ophi.empty() ? std::vector<double>{0.0} : ophi, s);
  } else {
    c.hptr.upload(hptr, s);
    c.hvert.upload(hvert, s);
    c.hphi.upload(hphi, s);
  }
  c.phi_aff.upload(phi_aff, nv, s);
  for (int k = 0; k < 3; ++k) c.aff_origin[k] = aff_origin[k];
  c.sptr.upload(sptr, s);
  c.scol.upload(scol, s);
  {
    std::vector<int32_t> srow(scol.size()), sT(scol.size());
    for (int32_t i = 0; i < m; ++i)
      for (int32_t k = sptr[i]; k < sptr[i + 1]; ++k) {
        srow[k] = i;
        const int32_t j = scol[k];
        sT[k] = (int32_t)(std::lower_bound(scol.begin() + sptr[j], scol.begin() + sptr[j + 1], i) - scol.begin());
      }
    c.srow.upload(srow, s);
    c.sT.upload(sT, s);
  }
  c.Sblk.alloc((size_t)144 * c.nnzb_S);
  if (c.gal_parts > 1) c.Spart.alloc((size_t)m * c.gal_parts * 144 * (size_t)std::max(c.gal_max_jup, 1));
  c.gU_ptr.upload(Uptr, s);
  c.gU.upload(Uall, s);
  c.ga_off.upload(ga_off, s);
  c.ga_mask.upload(ga_mask.empty() ? std::vector<unsigned long long>{0} : ga_mask, s);
  c.ga_ent.upload(ga_ent.empty() ? std::vector<uint32_t>{0} : ga_ent, s);
  c.gj_ptr.upload(gj_ptr, s);
  c.gj_blk.upload(gj_blk, s);
  c.gl_base.upload(gl_base, s);
  c.gl_off.upload(gl_off, s);
  c.gl_ent.upload(gl_ent.empty() ? std::vector<uint32_t>{0} : gl_ent, s);
  c.Sa.alloc(144);
  c.Ra.alloc((size_t)36 * nv);
  c.Lden.alloc((size_t)c.nS_pad * c.nS_pad);
  c.perm.upload(c.h_perm, s);
  c.chol_rows.upload(rows_flat.empty() ? std::vector<int32_t>{0} : rows_flat, s);
  c.chol_rows_ptr.upload(rows_ptr, s);
  c.chol_panel_ptr.upload(panel_ptr, s);
  c.sym_tiles.upload(sym_tiles, s);
  c.chol_dag.upload(dag, s);
  c.chol_crit.upload(crit, s);
  c.chol_rw_ptr.upload(rw_ptr, s);
  c.chol_rw.upload(rw.empty() ? std::vector<int32_t>{0} : rw, s);
  c.chol_cls.upload(cls, s);
  c.chol_succ_ptr.upload(succ_ptr, s);
  c.chol_succ_mid.upload(succ_mid, s);
  c.chol_succ.upload(succ.empty() ? std::vector<int32_t>{0} : succ, s);
  c.chol_ndep0.upload(ndep, s);
  c.chol_ndep.alloc(ndep.size());
  c.chol_queue0.upload(queue0, s);
  c.chol_queue.alloc(queue0.size());
  c.df_flags.alloc((size_t)2 * NT * NT + NT + 1 + m);   // upd, pfl, dfl, chain SM, rdone[m]
  c.Uinv.alloc((size_t)NT * T * T);
  {
    int nsm = 0;
    MS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c.device));
    c.coop_grid = std::max(1, nsm);
  }
  c.chol_panel.upload(panel_flat.empty() ? std::vector<int32_t>{0} : panel_flat, s);
  c.qa.alloc(12);
  c.za.alloc(12);
  c.qs.alloc(c.nS_pad);
  c.zs.alloc(c.nS_pad);
  c.yp.alloc(c.nS_pad);
  c.xsol.alloc(c.nS_pad);
  coarse_reset_graphs(c);
  launch_basis_W(c);
  MS_CUDA(cudaStreamSynchronize(s));
}

// Cubature of the subspace Hessian (NEXT-2): per-tet scale w_e / V_e and, per BSR slot, the
// contributions (tet*16 + a*4 + b, tet order) of the cubature elements only.
void build_cubature_structures(Ctx &c, const std::vector<int32_t> &loc_elems, const std::vector<double> &w) {
  const int32_t nt = c.nt;
  std::vector<double> scale(nt, 0.0);
  std::vector<double> vol(nt);
  c.vol.download(vol.data(), nt, c.stream);
  MS_CUDA(cudaStreamSynchronize(c.stream));
  for (size_t k = 0; k < loc_elems.size(); ++k) scale[loc_elems[k]] = w[k] / vol[loc_elems[k]];
  const int32_t *tets = c.h_tets.data();
  auto slot_of = [&](int32_t r, int32_t col) {
    const int32_t *b = c.h_colidx.data() + c.h_rowptr[r], *e = c.h_colidx.data() + c.h_rowptr[r + 1];
    return (int32_t)(std::lower_bound(b, e, col) - c.h_colidx.data());
  };
  std::vector<int32_t> sorted = loc_elems;
  std::sort(sorted.begin(), sorted.end());
  std::vector<int32_t> cptr(c.nnzb + 1, 0), cslot((size_t)16 * sorted.size());
  for (size_t k = 0; k < sorted.size(); ++k) {
    const int32_t e = sorted[k];
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) {
        const int32_t sl = slot_of(tets[4 * (size_t)e + a], tets[4 * (size_t)e + b]);
        cslot[16 * k + 4 * a + b] = sl;
        cptr[sl + 1]++;
      }
  }
  for (int64_t sl = 0; sl < c.nnzb; ++sl) cptr[sl + 1] += cptr[sl];
  std::vector<int32_t> contrib(cslot.size());
  {
    std::vector<int32_t> fill(cptr.begin(), cptr.end() - 1);
    for (size_t k = 0; k < sorted.size(); ++k)
      for (int q = 0; q < 16; ++q) contrib[fill[cslot[16 * k + q]]++] = 16 * sorted[k] + q;
  }
  cudaStream_t s = c.stream;
  c.tet_scale.upload(scale, s);
  c.cub_tets.upload(sorted.empty() ? std::vector<int32_t>{0} : sorted, s);
  c.cptr_c.upload(cptr, s);
  c.contrib_c.upload(contrib.empty() ? std::vector<int32_t>{0} : contrib, s);
  c.n_cub = (int32_t)sorted.size();
  MS_CUDA(cudaStreamSynchronize(s));
}

// Lists of the diagonal-block Galerkin rows S_ii = U_i^T H U_i (the block-Jacobi preconditioner
// of the paper's coarse PCG): the same fused Galerkin kernel with U_i = supp(i) (only
// rows u in supp(i) meet W_ui != 0) and the single upper slot j = i.  Built on first use.
void build_coarse_pcg_structures(Ctx &c) {
  if (c.cpcg_ready) return;
  const int32_t m = c.m, nv = c.nv;
  const int64_t *vptr = c.h_bvptr.data();
  const int32_t *handle = c.h_bhandle.data();
  const int32_t *rp = c.h_rowptr.data(), *ci = c.h_colidx.data();
  // supp(i), owned rows, vertex order
  std::vector<int32_t> Uptr(m + 1, 0), Uall;
  {
    std::vector<std::vector<int32_t>> supp(m);
    for (int32_t v = 0; v < std::min(nv, c.nv_own); ++v)
      for (int64_t k = vptr[v]; k < vptr[v + 1]; ++k) supp[handle[k]].push_back(v);
    for (int32_t i = 0; i < m; ++i) {
      Uall.insert(Uall.end(), supp[i].begin(), supp[i].end());
      Uptr[i + 1] = (int32_t)Uall.size();
    }
  }
  std::vector<int32_t> ga_off(1, 0);
  std::vector<uint32_t> ga_ent;
  std::vector<unsigned long long> ga_mask;
  for (int32_t i = 0; i < m; ++i)
    for (int32_t q = Uptr[i]; q < Uptr[i + 1]; ++q) {
      const int32_t u = Uall[q];
      MS_REQUIRE(rp[u + 1] - rp[u] <= 64, MS_ERR_ARG, "Hessian row longer than 64 blocks (Galerkin encoding)");
      unsigned long long mask = 0;
      for (int32_t j = 0; j < rp[u + 1] - rp[u]; ++j) {
        const int32_t v = ci[rp[u] + j];
        const int32_t *hb = handle + vptr[v], *he = handle + vptr[v + 1];
        const int32_t *f = std::lower_bound(hb, he, i);
        if (f != he && *f == i) {
          ga_ent.push_back((uint32_t)j | ((uint32_t)(vptr[v] + (f - hb)) << 6));
          mask |= 1ull << j;
        }
      }
      ga_mask.push_back(mask);
      ga_off.push_back((int32_t)ga_ent.size());
    }
  std::vector<int32_t> gj_ptr(m + 1), gj_blk(m), gl_base(m + 1, 0), gl_off, sT(m);
  std::vector<uint32_t> gl_ent;
  for (int32_t i = 0; i < m; ++i) {
    gj_ptr[i] = i;
    gj_blk[i] = i;
    sT[i] = i;
    const int32_t nU = Uptr[i + 1] - Uptr[i];
    const int32_t nch = (nU + kGalChunk - 1) / kGalChunk;
    gl_base[i + 1] = gl_base[i] + nch * 2;
    for (int32_t ch = 0; ch < nch; ++ch) {
      gl_off.push_back((int32_t)gl_ent.size());
      for (int32_t t = 0; t < kGalChunk && ch * kGalChunk + t < nU; ++t) {
        const int32_t u = Uall[Uptr[i] + ch * kGalChunk + t];
        const int32_t *hb = handle + vptr[u], *he = handle + vptr[u + 1];
        const int32_t *f = std::lower_bound(hb, he, i);
        MS_REQUIRE(f != he && *f == i, MS_ERR_STATE, "diagonal Galerkin lists: vertex outside the support");
        gl_ent.push_back((uint32_t)t | ((uint32_t)(vptr[u] + (f - hb)) << 7));
      }
      gl_off.push_back((int32_t)gl_ent.size());
    }
  }
  gj_ptr[m] = m;
  cudaStream_t s = c.stream;
  c.gd_U_ptr.upload(Uptr, s);
  c.gd_U.upload(Uall.empty() ? std::vector<int32_t>{0} : Uall, s);
  c.gd_ga_off.upload(ga_off, s);
  c.gd_ga_ent.upload(ga_ent.empty() ? std::vector<uint32_t>{0} : ga_ent, s);
  c.gd_ga_mask.upload(ga_mask.empty() ? std::vector<unsigned long long>{0} : ga_mask, s);
  c.gd_gj_ptr.upload(gj_ptr, s);
  c.gd_gj_blk.upload(gj_blk, s);
  c.gd_gl_base.upload(gl_base, s);
  c.gd_gl_off.upload(gl_off.empty() ? std::vector<int32_t>{0} : gl_off, s);
  c.gd_gl_ent.upload(gl_ent.empty() ? std::vector<uint32_t>{0} : gl_ent, s);
  c.gd_sT.upload(sT, s);
  c.Sdiag.alloc((size_t)144 * m);
  c.Sdiag_part.alloc((size_t)144 * m * std::max(c.gal_parts, 1));
  c.Minv.alloc((size_t)144 * m);
  c.cp_r.alloc((size_t)12 * m);
  c.cp_z.alloc((size_t)12 * m);
  c.cp_p.alloc((size_t)12 * m);
  c.cp_t.alloc((size_t)12 * m);
  c.cp_state.alloc(2);
  MS_CUDA(cudaStreamSynchronize(s));
  c.cpcg_ready = true;
}

}  // namespace msim
