// Vertex gradient gather, atomic-free BSR assembly, 3x3-block SpMV and the fused Jacobi-PCG.
//
// SURVEY §8(a) rows a2 (g = M(x - xhat) + h^2 [sum_e g_e + kappa b'(d) n], g_DBC = 0),
// a4 (H = M + h^2 (sum_e P+(H_e) + kappa b''(d) n n^T), DBC rows/cols -> identity),
// a8 (exactly N_cg Jacobi-PCG iterations from d_f = 0, reading R5).
//
// B200 design: BSR values are stored as 9 planes [q][nnzb] so that a half-warp reading 16
// consecutive blocks of one row issues fully coalesced 128-byte loads per plane; the PCG
// direction update is fused into the SpMV (q = H z + beta q, p = z + beta p), the dot
// products are deterministic grid reductions, and the whole fixed-count loop is captured in a
// CUDA graph (no host synchronisation inside the loop).
#include "common.cuh"
#include "reduce.cuh"
#include "sell.cuh"

namespace msim {

// ------------------------------------------------------------------ barrier helpers
__device__ __forceinline__ double bar_b(double d, double dh) {
  if (d >= dh) return 0.0;
  const double t = d - dh;
  return -t * t * log(d / dh);
}
__device__ __forceinline__ double bar_d1(double d, double dh) {
  if (d >= dh) return 0.0;
  const double t = d - dh;
  return -2.0 * t * log(d / dh) - t * t / d;
}
__device__ __forceinline__ double bar_d2(double d, double dh) {
  if (d >= dh) return 0.0;
  const double t = d - dh;
  return -2.0 * log(d / dh) - 4.0 * t / d + (t * t) / (d * d);
}

struct Ground {
  int on;
  double n0, n1, n2, off, dhat, kappa;
};
static Ground ground_of(const Ctx &c) {
  return Ground{c.has_ground ? 1 : 0, c.gn[0], c.gn[1], c.gn[2], c.goff, c.dhat, c.kappa};
}

// ------------------------------------------------------------------ vertex gradient (a2)
// g_v = h^2 sum_{(e,a) in inc(v)} g_e[a] + m_v (x_v - xhat_v) + h^2 kappa b'(d_v) n ; 0 at DBC.
// Also accumulates the vertex energy terms (inertia + h^2 kappa b) over free vertices, |g|^2.
// gradient of every local vertex; energy, |g|^2 and the penetration count over the owned
// vertices [0, nv_own) only
__global__ void __launch_bounds__(256) k_vertex_grad(
    int nv, int nv_own, const int32_t *__restrict__ vptr, const int32_t *__restrict__ vinc,
    const double *__restrict__ stage_g, const double *__restrict__ x, const double *__restrict__ xhat,
    const double *__restrict__ mass, const uint8_t *__restrict__ fixed, Ground G, double h2,
    double *__restrict__ g, double *__restrict__ partial, unsigned int *__restrict__ counter,
    double *__restrict__ out /* [energy, |g|^2, infeasible] */) {
  double acc[3] = {0.0, 0.0, 0.0};
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    double ge[3] = {0.0, 0.0, 0.0};
    for (int k = vptr[v]; k < vptr[v + 1]; ++k) {
      const int code = vinc[k];
      const double *src = stage_g + (size_t)(code >> 2) * 12 + 3 * (code & 3);
      ge[0] += src[0];
      ge[1] += src[1];
      ge[2] += src[2];
    }
    double out3[3];
    const double m = mass[v];
    double r[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      r[i] = x[3 * v + i] - xhat[3 * v + i];
      out3[i] = h2 * ge[i] + m * r[i];
    }
    double e = 0.0;
    if (!fixed[v]) {
      e = 0.5 * m * (r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
      if (G.on) {
        const double d = G.n0 * x[3 * v] + G.n1 * x[3 * v + 1] + G.n2 * x[3 * v + 2] - G.off;
        if (!(d > 0.0) && v < nv_own) acc[2] += 1.0;
        const double b1 = h2 * G.kappa * bar_d1(d, G.dhat);
        out3[0] += b1 * G.n0;
        out3[1] += b1 * G.n1;
        out3[2] += b1 * G.n2;
        e += h2 * G.kappa * bar_b(d, G.dhat);
      }
    } else {
      out3[0] = out3[1] = out3[2] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) g[3 * v + i] = out3[i];
    if (v < nv_own) {
      acc[0] += e;
      acc[1] += out3[0] * out3[0] + out3[1] * out3[1] + out3[2] * out3[2];
    }
  }
  double res[3];
  if (grid_reduce<3>(acc, partial, counter, res) && threadIdx.x == 0) {
    out[0] = res[0];
    out[1] = res[1];
    out[2] = res[2];
  }
}

void launch_vertex_grad(Ctx &c) {
  const int bs = 256, nb = std::min(div_up(c.nv, bs), 148 * 8);
  const double h2 = c.ah2();   // alpha h^2 (Eq. 2)
  k_vertex_grad<<<nb, bs, 0, c.stream>>>(c.nv, c.nv_own, c.vinc_ptr, c.vinc, c.stage_g, c.x, c.xhat, c.mass,
                                         c.fixed, ground_of(c), h2, c.g, c.partial, c.counters + 1,
                                         c.scal + SC_ENERGY_VERT);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ assembly (a4)
__host__ __device__ constexpr int blk4s(int a, int b) { return a * 4 - (a * (a - 1)) / 2 + (b - a); }

#ifndef MSIM_ASM_UNROLL
#define MSIM_ASM_UNROLL 2   // two contributions' gathers in flight (measured: 0.545 -> 0.526 ms at C4)
#endif
constexpr int kAsmUnroll = MSIM_ASM_UNROLL;

// thread per SELL position (coalesced value writes); slot s = sell_slot[pos] (-1: padding)
// tet_scale (may be NULL): per-tet factor of the contributions (the cubature weight w_e / V_e);
// dinv (may be NULL): Jacobi diagonal; diag_el (may be NULL): the alpha h^2 elastic part of the
// diagonal blocks before inertia and barrier are added (the frozen part of the lagged Hessian)
__global__ void __launch_bounds__(256) k_assemble(
    int64_t npos, const int32_t *__restrict__ sell_slot, const int32_t *__restrict__ sell_col,
    const int32_t *__restrict__ cptr, const int32_t *__restrict__ contrib,
    const double *__restrict__ stage_h, const double *__restrict__ x, const double *__restrict__ mass,
    const uint8_t *__restrict__ fixed, const int32_t *__restrict__ slot_row, Ground G, double h2,
    double *__restrict__ vals, double *__restrict__ dinv, const double *__restrict__ tet_scale,
    double *__restrict__ diag_el) {
  const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= npos) return;
  const int cidx = (int)(pos >> 5), lane = (int)(pos & 31);
  const int s = sell_slot[pos];
  double acc[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q] = 0.0;
  if (s >= 0) {
    const int k1 = __ldg(&cptr[s + 1]);
#pragma unroll(kAsmUnroll)
    for (int k = __ldg(&cptr[s]); k < k1; ++k) {
      const int code = __ldg(&contrib[k]);
      const int e = code >> 4, a = (code >> 2) & 3, b = code & 3;
      const bool up = a <= b;
      const double2 *src = reinterpret_cast<const double2 *>(
          stage_h + (size_t)e * kStageH + (up ? blk4s(a, b) : blk4s(b, a)) * kStageB);
      double v[10];
#pragma unroll
      for (int h = 0; h < 5; ++h) {
        const double2 t2 = __ldg(&src[h]);
        v[2 * h] = t2.x;
        v[2 * h + 1] = t2.y;
      }
      const double sc = tet_scale ? __ldg(&tet_scale[e]) : 1.0;
#pragma unroll
      for (int q = 0; q < 9; ++q) acc[q] += sc * (up ? v[q] : v[(q % 3) * 3 + q / 3]);
    }
    const int row = slot_row[s], col = sell_col[pos];
#pragma unroll
    for (int q = 0; q < 9; ++q) acc[q] *= h2;
    if (row == col && diag_el) {
#pragma unroll
      for (int q = 0; q < 9; ++q) diag_el[9 * (size_t)row + q] = acc[q];
    }
    if (row == col) {
      const double m = mass[row];
      acc[0] += m;
      acc[4] += m;
      acc[8] += m;
      if (G.on) {
        const double d = G.n0 * x[3 * row] + G.n1 * x[3 * row + 1] + G.n2 * x[3 * row + 2] - G.off;
        const double kb = h2 * G.kappa * bar_d2(d, G.dhat);
        const double n[3] = {G.n0, G.n1, G.n2};
#pragma unroll
        for (int q = 0; q < 9; ++q) acc[q] += kb * n[q / 3] * n[q % 3];
      }
    }
    if (fixed[row] || fixed[col]) {
#pragma unroll
      for (int q = 0; q < 9; ++q) acc[q] = (row == col && (q % 4 == 0)) ? 1.0 : 0.0;
    }
    if (row == col && dinv) {
      dinv[3 * row + 0] = 1.0 / acc[0];
      dinv[3 * row + 1] = 1.0 / acc[4];
      dinv[3 * row + 2] = 1.0 / acc[8];
    }
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) vals[sell_val_index(cidx, q, lane)] = acc[q];
}

// the refinement Hessian (H, or H_lag at a refresh) into vals + dinv
void launch_assemble(Ctx &c) {
  const int bs = 256;
  const double h2 = c.ah2();   // alpha h^2 (Eq. 2)
  if (c.params.lag_hessian) c.lag_diag.alloc(9 * (size_t)c.nv);
  k_assemble<<<div_up(c.npos, bs), bs, 0, c.stream>>>(c.npos, c.sell_slot, c.sell_col, c.cptr, c.contrib,
                                                      c.stage_h, c.x, c.mass, c.fixed, c.slot_row,
                                                      ground_of(c), h2, c.vals, c.dinv, nullptr,
                                                      c.params.lag_hessian ? c.lag_diag.p : nullptr);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

// the subspace Hessian into vals_s: the cubature Hessian (contributions of the cubature elements,
// weighted w_e / V_e; NEXT-2) or, with only lagging on, the fresh fully integrated H
void launch_assemble_sub(Ctx &c) {
  const int bs = 256;
  const double h2 = c.ah2();
  c.vals_s.alloc(c.vals.n);
  const bool cub = c.params.use_cubature;
  MS_REQUIRE(!cub || c.n_cub > 0, MS_ERR_STATE, "use_cubature without ms_cubature_upload");
  k_assemble<<<div_up(c.npos, bs), bs, 0, c.stream>>>(c.npos, c.sell_slot, c.sell_col, cub ? c.cptr_c : c.cptr,
                                                      cub ? c.contrib_c : c.contrib, c.stage_h, c.x, c.mass,
                                                      c.fixed, c.slot_row, ground_of(c), h2, c.vals_s, nullptr,
                                                      cub ? c.tet_scale.p : nullptr, nullptr);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

// H_lag between refreshes: the off-diagonal blocks keep their frozen elastic values; every
// diagonal block is rebuilt as frozen elastic part + fresh inertia + fresh barrier (DBC identity)
__global__ void k_lag_diag(int nv, const int32_t *__restrict__ diag_pos, const double *__restrict__ diag_el,
                           const double *__restrict__ x, const double *__restrict__ mass,
                           const uint8_t *__restrict__ fixed, Ground G, double h2, double *__restrict__ vals,
                           double *__restrict__ dinv) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nv) return;
  double acc[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q] = diag_el[9 * (size_t)row + q];
  const double m = mass[row];
  acc[0] += m;
  acc[4] += m;
  acc[8] += m;
  if (G.on) {
    const double d = G.n0 * x[3 * row] + G.n1 * x[3 * row + 1] + G.n2 * x[3 * row + 2] - G.off;
    const double kb = h2 * G.kappa * bar_d2(d, G.dhat);
    const double n[3] = {G.n0, G.n1, G.n2};
#pragma unroll
    for (int q = 0; q < 9; ++q) acc[q] += kb * n[q / 3] * n[q % 3];
  }
  if (fixed[row]) {
#pragma unroll
    for (int q = 0; q < 9; ++q) acc[q] = (q % 4 == 0) ? 1.0 : 0.0;
  }
  dinv[3 * row + 0] = 1.0 / acc[0];
  dinv[3 * row + 1] = 1.0 / acc[4];
  dinv[3 * row + 2] = 1.0 / acc[8];
  const int pos = diag_pos[row];
#pragma unroll
  for (int q = 0; q < 9; ++q) vals[sell_val_index(pos >> 5, q, pos & 31)] = acc[q];
}

void launch_lag_diag(Ctx &c) {
  k_lag_diag<<<div_up(c.nv, 256), 256, 0, c.stream>>>(c.nv, c.diag_pos, c.lag_diag, c.x, c.mass, c.fixed,
                                                      ground_of(c), c.ah2(), c.vals, c.dinv);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ SpMV (SELL-32, thread per row)
#ifndef MSIM_SPMV_UNROLL
#define MSIM_SPMV_UNROLL 16   // = full unroll for rows of <= 16 blocks: every load of a row in flight
#endif
#ifndef MSIM_SPMV_NOLDG
#define MSIM_SPMV_LDG
#endif
constexpr int kSpmvUnroll = MSIM_SPMV_UNROLL;

// matrix values are streamed once per product: read-only path, no L1 allocation (keeps L1 for
// the x gathers)
__device__ __forceinline__ double ld_stream(const double *p) {
#ifdef MSIM_SPMV_L1ALLOC
  return __ldg(p);
#else
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#endif
}

static SellView sell_view(const Ctx &c) { return SellView{c.nv, c.sl_ptr, c.sell_col, c.vals}; }

__device__ __forceinline__ void sell_row_product(const SellView &H, int row, const double *__restrict__ xin,
                                                 double o[3]) {
  const int sl = row >> 5, lane = row & 31;
  const int c0 = __ldg(&H.sl_ptr[sl]), c1 = __ldg(&H.sl_ptr[sl + 1]);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll(kSpmvUnroll)
  for (int cc = c0; cc < c1; ++cc) {
    const int col = __ldg(&H.col[(size_t)cc * 32 + lane]);
    const double *v = H.vals + (size_t)cc * 288 + lane;
    const double x0 = xin[3 * col], x1 = xin[3 * col + 1], x2 = xin[3 * col + 2];
    a0 = fma(ld_stream(v), x0, fma(ld_stream(v + 32), x1, fma(ld_stream(v + 64), x2, a0)));
    a1 = fma(ld_stream(v + 96), x0, fma(ld_stream(v + 128), x1, fma(ld_stream(v + 160), x2, a1)));
    a2 = fma(ld_stream(v + 192), x0, fma(ld_stream(v + 224), x1, fma(ld_stream(v + 256), x2, a2)));
  }
  o[0] = a0;
  o[1] = a1;
  o[2] = a2;
}

__global__ void __launch_bounds__(256) k_spmv(SellView H, const double *__restrict__ xin,
                                              double *__restrict__ yout, const double *__restrict__ b,
                                              const int32_t *__restrict__ skip) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= H.nv || (skip && *skip)) return;
  double o[3];
  sell_row_product(H, row, xin, o);
#pragma unroll
  for (int i = 0; i < 3; ++i) yout[3 * row + i] = b ? b[3 * row + i] - o[i] : o[i];
}

// skip (device flag, may be NULL): the launch does nothing while *skip != 0 (coarse PCG batches)
void launch_spmv(Ctx &c, const double *xin, double *yout, double /*unused*/, const double *b, const int32_t *skip,
                 const double *vals) {
  SellView H = sell_view(c);
  if (vals) H.vals = vals;
  k_spmv<<<div_up(c.nv, 256), 256, 0, c.stream>>>(H, xin, yout, b, skip);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ PCG (a8)
// Scalars in scal: SC_RZ (rho), SC_PQ, SC_ALPHA, SC_BETA, SC_RZ0.
// init:   x = 0, r = rhs, z = D^-1 r, p = 0, q = 0, beta = 0, rho = r.z
// iter:   K1: p = z + beta p ; q = H z + beta q ; pq = p.q ; alpha = rho / pq
//         K2: x += alpha p ; r -= alpha q ; z = D^-1 r ; rho' = r.z ; beta = rho'/rho ; rho = rho'
// (q = H(z + beta p_old) = H z + beta H p_old, so the direction update needs no extra pass.)
constexpr int kGridCap = 148 * 8;   // persistent-style grids: a few CTAs per SM, grid-stride loops

// n3_own: the dot products cover the owned entries [0, n3_own) (multi-GPU: partial sums, the
// scalars are then derived by k_pcg_scalars after the cross-rank sum; dist = 1)
__global__ void __launch_bounds__(256) k_pcg_init(int n3, int n3_own, int dist, const double *__restrict__ rhs,
                                                  const double *__restrict__ dinv, double *__restrict__ x,
                                                  double *__restrict__ r, double *__restrict__ z,
                                                  double *__restrict__ p, double *__restrict__ q,
                                                  double *__restrict__ partial, unsigned int *counter,
                                                  double *__restrict__ scal) {
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n3; i += gridDim.x * blockDim.x) {
    const double ri = rhs[i], zi = dinv[i] * ri;
    x[i] = 0.0;
    r[i] = ri;
    z[i] = zi;
    p[i] = 0.0;
    q[i] = 0.0;
    if (i < n3_own) acc[0] = fma(ri, zi, acc[0]);
  }
  double res[1];
  if (grid_reduce<1>(acc, partial, counter, res) && threadIdx.x == 0) {
    scal[SC_RZ] = res[0];
    scal[SC_RZ0] = res[0];
    scal[SC_BETA] = 0.0;
    (void)dist;
  }
}

// thread per row (SELL-32); fused direction update and p.q partial
__global__ void __launch_bounds__(256) k_pcg_spmv(SellView H, int nv_own, int dist, const double *__restrict__ z,
                                                  double *__restrict__ p, double *__restrict__ q,
                                                  double *__restrict__ partial, unsigned int *counter,
                                                  double *__restrict__ scal, const int32_t *__restrict__ skip) {
  if (skip && *skip) return;   // uniform over the grid: no block reaches the grid reduction
  const double beta = scal[SC_BETA];
  double acc[1] = {0.0};
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row < H.nv) {
    double o[3];
    sell_row_product(H, row, z, o);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double pn = fma(beta, p[3 * row + i], z[3 * row + i]);
      const double qn = fma(beta, q[3 * row + i], o[i]);
      p[3 * row + i] = pn;
      q[3 * row + i] = qn;
      if (row < nv_own) acc[0] = fma(pn, qn, acc[0]);
    }
  }
  double res[1];
  if (grid_reduce<1>(acc, partial, counter, res) && threadIdx.x == 0) {
    const double rho = scal[SC_RZ];
    scal[SC_PQ] = res[0];
    if (!dist) scal[SC_ALPHA] = (res[0] != 0.0 && rho != 0.0) ? rho / res[0] : 0.0;
  }
}

__global__ void __launch_bounds__(256) k_pcg_update(int n3, int n3_own, int dist, const double *__restrict__ dinv,
                                                    const double *__restrict__ p, const double *__restrict__ q,
                                                    double *__restrict__ x, double *__restrict__ r,
                                                    double *__restrict__ z, double *__restrict__ partial,
                                                    unsigned int *counter, double *__restrict__ scal) {
  const double alpha = scal[SC_ALPHA];
  double acc[1] = {0.0};
  // pairs of entries through 16-byte accesses (cudaMalloc'd vectors: 16-byte aligned); an odd
  // last entry is taken by the first thread
  const int n2 = n3 >> 1;
  for (int i2 = blockIdx.x * blockDim.x + threadIdx.x; i2 < n2; i2 += gridDim.x * blockDim.x) {
    const double2 pv = reinterpret_cast<const double2 *>(p)[i2], qv = reinterpret_cast<const double2 *>(q)[i2];
    const double2 xv = reinterpret_cast<const double2 *>(x)[i2], rv = reinterpret_cast<const double2 *>(r)[i2];
    const double2 dv = reinterpret_cast<const double2 *>(dinv)[i2];
    const double r0 = fma(-alpha, qv.x, rv.x), r1 = fma(-alpha, qv.y, rv.y);
    const double z0 = dv.x * r0, z1 = dv.y * r1;
    reinterpret_cast<double2 *>(x)[i2] = make_double2(fma(alpha, pv.x, xv.x), fma(alpha, pv.y, xv.y));
    reinterpret_cast<double2 *>(r)[i2] = make_double2(r0, r1);
    reinterpret_cast<double2 *>(z)[i2] = make_double2(z0, z1);
    if (2 * i2 < n3_own) acc[0] = fma(r0, z0, acc[0]);
    if (2 * i2 + 1 < n3_own) acc[0] = fma(r1, z1, acc[0]);
  }
  if ((n3 & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int i = n3 - 1;
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    const double zi = dinv[i] * ri;
    r[i] = ri;
    z[i] = zi;
    if (i < n3_own) acc[0] = fma(ri, zi, acc[0]);
  }
  double res[1];
  if (grid_reduce<1>(acc, partial, counter, res) && threadIdx.x == 0) {
    if (dist) {
      scal[SC_RZ_OLD] = res[0];   // partial r'.z', summed across ranks before k_pcg_scalars
    } else {
      const double rho = scal[SC_RZ];
      scal[SC_BETA] = rho != 0.0 ? res[0] / rho : 0.0;
      scal[SC_RZ] = res[0];
    }
  }
}

static int grid_vec(int64_t n) { return std::min(div_up(n, 256), kGridCap); }

// multi-GPU: the PCG scalars from the rank-summed dot products (which = 0: alpha; 1: beta)
__global__ void k_pcg_scalars(double *__restrict__ scal, int which) {
  if (which == 0) {
    const double rho = scal[SC_RZ], pq = scal[SC_PQ];
    scal[SC_ALPHA] = (pq != 0.0 && rho != 0.0) ? rho / pq : 0.0;
  } else {
    const double rho = scal[SC_RZ], rn = scal[SC_RZ_OLD];
    scal[SC_BETA] = rho != 0.0 ? rn / rho : 0.0;
    scal[SC_RZ] = rn;
  }
}

// ---- multi-GPU: single-reduction PCG (Chronopoulos & Gear 1989), algebraically the same
// iterates as the recurrence above with ONE rank reduction per iteration (gamma = r.z and
// delta = z.Hz summed together):
//   w = H z; [gamma, delta] summed; beta = gamma / gamma_old; alpha = gamma / (delta - beta gamma / alpha_old)
//   (first iteration: beta = 0, alpha = gamma / delta); p = z + beta p; s = w + beta s;
//   x += alpha p; r -= alpha s; z = D^-1 r; gamma' partial = r.z (owned); halo(z)
// rows [r0, r1) then [r2, r3) (one thread each); the dot over the owned ones goes to scal[dst]
// (+ scal[SC_CG_DI] when add_int: the interior part of a split product)
__global__ void __launch_bounds__(256) k_cg_spmv(SellView H, int nv_own, int r0, int r1, int r2, int r3,
                                                 const double *__restrict__ z, double *__restrict__ w,
                                                 double *__restrict__ partial, unsigned int *counter,
                                                 double *__restrict__ scal, int dst, int add_int) {
  double acc[1] = {0.0};
  const int t = blockIdx.x * blockDim.x + threadIdx.x, n1 = r1 - r0;
  const int row = t < n1 ? r0 + t : r2 + (t - n1);
  if (row < (t < n1 ? r1 : r3)) {
    double o[3];
    sell_row_product(H, row, z, o);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      w[3 * row + i] = o[i];
      if (row < nv_own) acc[0] = fma(z[3 * row + i], o[i], acc[0]);
    }
  }
  double res[1];
  if (grid_reduce<1>(acc, partial, counter, res) && threadIdx.x == 0)
    scal[dst] = add_int ? res[0] + scal[SC_CG_DI] : res[0];
}

__global__ void k_cg_scalars(double *__restrict__ scal, int first) {
  const double g = scal[SC_CG_G], d = scal[SC_CG_D];
  double alpha, beta;
  if (first) {
    beta = 0.0;
    alpha = (g != 0.0 && d != 0.0) ? g / d : 0.0;
    scal[SC_RZ0] = g;
  } else {
    const double go = scal[SC_CG_GOLD], ao = scal[SC_CG_AOLD];
    beta = go != 0.0 ? g / go : 0.0;
    const double den = (ao != 0.0) ? d - beta * g / ao : 0.0;
    alpha = (g != 0.0 && den != 0.0) ? g / den : 0.0;
  }
  scal[SC_ALPHA] = alpha;
  scal[SC_BETA] = beta;
  scal[SC_CG_GOLD] = g;
  scal[SC_CG_AOLD] = alpha;
}

__global__ void __launch_bounds__(256) k_cg_update(int n3, int n3_own, const double *__restrict__ dinv,
                                                   const double *__restrict__ w, double *__restrict__ p,
                                                   double *__restrict__ s, double *__restrict__ x,
                                                   double *__restrict__ r, double *__restrict__ z,
                                                   double *__restrict__ partial, unsigned int *counter,
                                                   double *__restrict__ scal) {
  const double alpha = scal[SC_ALPHA], beta = scal[SC_BETA];
  double acc[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n3; i += gridDim.x * blockDim.x) {
    const double pn = fma(beta, p[i], z[i]);
    const double sn = fma(beta, s[i], w[i]);
    p[i] = pn;
    s[i] = sn;
    x[i] = fma(alpha, pn, x[i]);
    const double ri = fma(-alpha, sn, r[i]);
    const double zi = dinv[i] * ri;
    r[i] = ri;
    z[i] = zi;
    if (i < n3_own) acc[0] = fma(ri, zi, acc[0]);
  }
  double res[1];
  if (grid_reduce<1>(acc, partial, counter, res) && threadIdx.x == 0) scal[SC_CG_G] = res[0];
}

void halo_exchange_async(Ctx &c, double *vec);

static void enqueue_cg_iters_dist(Ctx &c, double *sol, int iters) {
  const int n3 = 3 * c.nv, n3o = 3 * c.nv_own, bs = 256;
  const int lo = c.int_lo, hi = c.int_hi, nv = c.nv;
  const bool split = hi > lo;   // the interior rows overlap the halo of z (previous update)
  for (int it = 0; it < iters; ++it) {
    if (split && it > 0) {
      k_cg_spmv<<<div_up(hi - lo, bs), bs, 0, c.stream>>>(sell_view(c), c.nv_own, lo, hi, nv, nv, c.z, c.tmp,
                                                         c.partial, c.counters + 3, c.scal, SC_CG_DI, 0);
      MS_CUDA(cudaStreamWaitEvent(c.stream, c.ev_halo, 0));
      // (a single slab has no boundary rows: one CTA still adds the interior part into SC_CG_D)
      k_cg_spmv<<<std::max(1, (int)div_up(lo + nv - hi, bs)), bs, 0, c.stream>>>(sell_view(c), c.nv_own, 0, lo, hi, nv, c.z, c.tmp,
                                                              c.partial, c.counters + 3, c.scal, SC_CG_D, 1);
      c.launches += 1;
    } else {
      k_cg_spmv<<<div_up(nv, bs), bs, 0, c.stream>>>(sell_view(c), c.nv_own, 0, nv, nv, nv, c.z, c.tmp, c.partial,
                                                     c.counters + 3, c.scal, SC_CG_D, 0);
    }
    dist_sum(c, c.scal + SC_CG_G, 2);   // the iteration's only reduction
    k_cg_scalars<<<1, 1, 0, c.stream>>>(c.scal, it == 0 ? 1 : 0);
    k_cg_update<<<grid_vec(n3), bs, 0, c.stream>>>(n3, n3o, c.dinv, c.tmp, c.p, c.q, sol, c.r, c.z, c.partial,
                                                   c.counters + 4, c.scal);
    if (split) halo_exchange_async(c, c.z);
    else halo_exchange(c, c.z);
    c.launches += 3;
  }
  if (split && iters > 0) MS_CUDA(cudaStreamWaitEvent(c.stream, c.ev_halo, 0));   // join (graph capture too)
}

static void enqueue_pcg_iters(Ctx &c, double *sol, int iters) {
  const int n3 = 3 * c.nv, n3o = 3 * c.nv_own, bs = 256, dist = c.dist() ? 1 : 0;
  if (dist) {
    enqueue_cg_iters_dist(c, sol, iters);
    return;
  }
  for (int it = 0; it < iters; ++it) {
    k_pcg_spmv<<<div_up(c.nv, bs), bs, 0, c.stream>>>(sell_view(c), c.nv_own, dist, c.z, c.p, c.q, c.partial,
                                                      c.counters + 3, c.scal, nullptr);
    if (dist) {
      dist_sum(c, c.scal + SC_PQ, 1);
      k_pcg_scalars<<<1, 1, 0, c.stream>>>(c.scal, 0);
    }
    k_pcg_update<<<grid_vec((n3 + 1) / 2), bs, 0, c.stream>>>(n3, n3o, dist, c.dinv, c.p, c.q, sol, c.r, c.z, c.partial,
                                                    c.counters + 4, c.scal);
    if (dist) {
      dist_sum(c, c.scal + SC_RZ_OLD, 1);
      k_pcg_scalars<<<1, 1, 0, c.stream>>>(c.scal, 1);
      halo_exchange(c, c.z);
      c.launches += 2;
    }
  }
}

void launch_pcg_init(Ctx &c, const double *rhs, double *sol) {
  const int n3 = 3 * c.nv;
  k_pcg_init<<<grid_vec(n3), 256, 0, c.stream>>>(n3, 3 * c.nv_own, c.dist() ? 1 : 0, rhs, c.dinv, sol, c.r, c.z, c.p,
                                                 c.q, c.partial, c.counters + 2, c.scal);
  c.launches++;
}

// p = z + beta p; q = H z + beta q; alpha = rho / p.q (rank-summed p.q on several GPUs)
void launch_pcg_spmv(Ctx &c, const int32_t *skip) {
  const int dist = c.dist() ? 1 : 0;
  k_pcg_spmv<<<div_up(c.nv, 256), 256, 0, c.stream>>>(sell_view(c), c.nv_own, dist, c.z, c.p, c.q, c.partial,
                                                      c.counters + 3, c.scal, skip);
  c.launches++;
  if (dist) {
    dist_sum(c, c.scal + SC_PQ, 1);
    k_pcg_scalars<<<1, 1, 0, c.stream>>>(c.scal, 0);
    c.launches++;
  }
}

// multi-GPU: the final r.z (PCG statistics) summed across ranks -- outside the iterations
static void pcg_finish_dist(Ctx &c) {
  if (!c.dist()) return;
  MS_CUDA(cudaMemcpyAsync(c.scal + SC_RZ, c.scal + SC_CG_G, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  dist_sum(c, c.scal + SC_RZ, 1);
}

void pcg_reset_graph(Ctx &c) {
  if (c.pcg_graph) cudaGraphExecDestroy(c.pcg_graph);
  c.pcg_graph = nullptr;
  c.pcg_graph_iters = -1;
}

// Runs exactly `iters` PCG iterations on H sol = rhs (sol, rhs device vectors; sol must be c.df
// when graphs are used, since the captured graph bakes in the pointer).
void launch_pcg(Ctx &c, const double *rhs, double *sol, int iters) {
  const int n3 = 3 * c.nv, bs = 256;
  k_pcg_init<<<grid_vec(n3), bs, 0, c.stream>>>(n3, 3 * c.nv_own, c.dist() ? 1 : 0, rhs, c.dinv, sol, c.r, c.z, c.p,
                                                  c.q, c.partial, c.counters + 2, c.scal);
  c.launches++;
  MS_CUDA(cudaGetLastError());
  if (c.dist()) {   // r.z stays a partial sum (summed with z.Hz in the first iteration); ghost z
    MS_CUDA(cudaMemcpyAsync(c.scal + SC_CG_G, c.scal + SC_RZ, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
    halo_exchange(c, c.z);
    if (iters <= 0) {
      dist_sum(c, c.scal + SC_RZ, 1);
      MS_CUDA(cudaMemcpyAsync(c.scal + SC_RZ0, c.scal + SC_RZ, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
    }
  }
  if (iters <= 0) return;
  // NCCL collectives are recorded into the graph too; the in-process hub synchronises on the host
  const bool graphs = c.params.use_graphs && sol == c.df.p && (!c.dist() || c.comm->capturable());
  if (!graphs) {
    enqueue_pcg_iters(c, sol, iters);
    if (!c.dist()) c.launches += 2 * (int64_t)iters;
    MS_CUDA(cudaGetLastError());
    pcg_finish_dist(c);
    return;
  }
  if (c.pcg_graph_iters != iters || !c.pcg_graph) {
    pcg_reset_graph(c);
    cudaStream_t cap;
    MS_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaStream_t saved = c.stream;
    c.stream = cap;
    cudaGraph_t graph;
    MS_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    const int64_t l0 = c.launches;
    enqueue_pcg_iters(c, sol, iters);
    const int64_t captured = c.launches - l0;   // dist: counted while enqueueing
    c.launches = l0;
    MS_CUDA(cudaStreamEndCapture(cap, &graph));
    c.stream = saved;
    MS_CUDA(cudaGraphInstantiate(&c.pcg_graph, graph, 0));
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cap);
    c.pcg_graph_iters = iters;
    c.pcg_graph_kernels = c.dist() ? captured : 2 * (int64_t)iters;
  }
  MS_CUDA(cudaGraphLaunch(c.pcg_graph, c.stream));
  c.launches += c.pcg_graph_kernels;
  pcg_finish_dist(c);
}

// ------------------------------------------------------------------ small vector kernels
__global__ void k_axpby(int64_t n, double *__restrict__ y, double a, const double *__restrict__ x, double b) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // b == 0 overwrites: y may be a fresh buffer (0 * NaN of recycled device memory would poison it)
  if (i < n) y[i] = b == 0.0 ? a * x[i] : a * x[i] + b * y[i];
}
void launch_axpby(Ctx &c, double *y, double a, const double *x, double b, int64_t n) {
  k_axpby<<<div_up(n, 256), 256, 0, c.stream>>>(n, y, a, x, b);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

__global__ void __launch_bounds__(256) k_dot(int64_t n, const double *__restrict__ a,
                                             const double *__restrict__ b, double *__restrict__ partial,
                                             unsigned int *counter, double *__restrict__ out) {
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc[0] = fma(a[i], b[i], acc[0]);
  double res[1];
  if (grid_reduce<1>(acc, partial, counter, res) && threadIdx.x == 0) *out = res[0];
}
void launch_dot(Ctx &c, const double *a, const double *b, int64_t n, int slot) {
  k_dot<<<std::min(div_up(n, 256), 1184), 256, 0, c.stream>>>(n, a, b, c.partial, c.counters + 5, c.scal + slot);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

// xhat = x^t + h v^t + h^2 g (R8); x^t = x; DBC vertices pinned at rest
__global__ void k_predictor(int nv, const double *__restrict__ X, const uint8_t *__restrict__ fixed,
                            double *__restrict__ x, const double *__restrict__ v, double *__restrict__ xt,
                            double *__restrict__ xhat, double h, double g0, double g1, double g2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const double gg[3] = {g0, g1, g2};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double xi = x[3 * i + k];
    if (fixed[i]) xi = X[3 * i + k];
    x[3 * i + k] = xi;
    xt[3 * i + k] = xi;
    xhat[3 * i + k] = xi + h * v[3 * i + k] + h * h * gg[k];
  }
}
// BDF2 predictor: xhat = (4x^t - x^{t-1})/3 + (2h/9)(4v^t - v^{t-1}) + (4/9) h^2 g
__global__ void k_predictor_bdf2(int nv, const double *__restrict__ X, const uint8_t *__restrict__ fixed,
                                 double *__restrict__ x, const double *__restrict__ v,
                                 const double *__restrict__ xp, const double *__restrict__ vp,
                                 double *__restrict__ xt, double *__restrict__ xhat, double h, double g0, double g1,
                                 double g2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const double gg[3] = {g0, g1, g2};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double xi = x[3 * i + k];
    if (fixed[i]) xi = X[3 * i + k];
    x[3 * i + k] = xi;
    xt[3 * i + k] = xi;
    xhat[3 * i + k] = (4.0 * xi - xp[3 * i + k]) / 3.0 + (2.0 * h / 9.0) * (4.0 * v[3 * i + k] - vp[3 * i + k]) +
                      (4.0 / 9.0) * h * h * gg[k];
  }
}

void launch_predictor(Ctx &c) {
  const bool bdf2 = c.params.integrator == MS_INTEGRATOR_BDF2 && c.has_history;
  c.alpha = bdf2 ? 4.0 / 9.0 : 1.0;
  if (bdf2)
    k_predictor_bdf2<<<div_up(c.nv, 256), 256, 0, c.stream>>>(c.nv, c.X, c.fixed, c.x, c.v, c.x_prev, c.v_prev, c.xt,
                                                              c.xhat, c.params.h, c.params.gravity[0],
                                                              c.params.gravity[1], c.params.gravity[2]);
  else
    k_predictor<<<div_up(c.nv, 256), 256, 0, c.stream>>>(c.nv, c.X, c.fixed, c.x, c.v, c.xt, c.xhat, c.params.h,
                                                         c.params.gravity[0], c.params.gravity[1],
                                                         c.params.gravity[2]);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

// v = (x - x^t) / h
__global__ void k_velocity(int n3, const double *__restrict__ x, const double *__restrict__ xt,
                           double *__restrict__ v, double inv_h) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n3) v[i] = (x[i] - xt[i]) * inv_h;
}

// end of a step with the BDF2 history kept: x^{t-1} <- x^t, v^{t-1} <- v^t and v^{t+1} =
//   IE step:   (x - x^t) / h
//   BDF2 step: (4v^t - v^{t-1})/3 + (2h/3) a, a = 9/(4h^2)(x - xtilde), xtilde = xhat - (4/9) h^2 g
//              (reading C2: the printed 4h^2/9 is not an acceleration)
__global__ void k_velocity_hist(int n3, int bdf2, const double *__restrict__ x, double *__restrict__ xt,
                                const double *__restrict__ xhat, double *__restrict__ v, double *__restrict__ xp,
                                double *__restrict__ vp, double h, double g0, double g1, double g2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  const double gk = (i % 3 == 0) ? g0 : (i % 3 == 1 ? g1 : g2);
  const double vt = v[i], xti = xt[i];
  double vn;
  if (bdf2) {
    const double a = 9.0 / (4.0 * h * h) * (x[i] - (xhat[i] - (4.0 / 9.0) * h * h * gk));
    vn = (4.0 * vt - vp[i]) / 3.0 + (2.0 * h / 3.0) * a;
  } else {
    vn = (x[i] - xti) / h;
  }
  xp[i] = xti;
  vp[i] = vt;
  v[i] = vn;
}

void launch_velocity(Ctx &c) {
  const int n3 = 3 * c.nv;
  if (c.params.integrator == MS_INTEGRATOR_BDF2) {
    c.x_prev.alloc(n3);
    c.v_prev.alloc(n3);
    k_velocity_hist<<<div_up(n3, 256), 256, 0, c.stream>>>(n3, c.alpha != 1.0 ? 1 : 0, c.x, c.xt, c.xhat, c.v,
                                                           c.x_prev, c.v_prev, c.params.h, c.params.gravity[0],
                                                           c.params.gravity[1], c.params.gravity[2]);
    c.has_history = true;
  } else {
    k_velocity<<<div_up(n3, 256), 256, 0, c.stream>>>(n3, c.x, c.xt, c.v, 1.0 / c.params.h);
  }
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

}  // namespace msim

namespace msim {

// ------------------------------------------------------------------ multi-GPU halo (dist.h)
__global__ void k_halo_pack(int n, const int32_t *__restrict__ idx, const double *__restrict__ vec,
                            double *__restrict__ buf) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < 3 * n) buf[t] = vec[3 * (size_t)idx[t / 3] + t % 3];
}
__global__ void k_halo_unpack(int n, const int32_t *__restrict__ idx, const double *__restrict__ buf,
                              double *__restrict__ vec) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < 3 * n) vec[3 * (size_t)idx[t / 3] + t % 3] = buf[t];
}

void halo_exchange(Ctx &c, double *vec) {
  if (!c.dist()) return;
  const int ns = (int)c.part.send_idx.size(), nr = (int)c.part.recv_idx.size();
  if (ns) k_halo_pack<<<div_up(3 * (int64_t)ns, 256), 256, 0, c.stream>>>(ns, c.halo_send_idx, vec, c.halo_send);
  c.comm->exchange(c.part.peers, c.halo_send, c.halo_recv, c.stream);
  if (nr) k_halo_unpack<<<div_up(3 * (int64_t)nr, 256), 256, 0, c.stream>>>(nr, c.halo_recv_idx, c.halo_recv, vec);
  c.launches += 2;
  MS_CUDA(cudaGetLastError());
}

// the same exchange on c.halo_stream, ordered after everything enqueued on c.stream so far; the
// caller makes c.stream wait on c.ev_halo before it reads ghost entries or writes vec again
void halo_exchange_async(Ctx &c, double *vec) {
  if (!c.dist()) return;
  MS_REQUIRE(c.halo_stream, MS_ERR_STATE, "halo stream not created");
  MS_CUDA(cudaEventRecord(c.ev_z, c.stream));
  MS_CUDA(cudaStreamWaitEvent(c.halo_stream, c.ev_z, 0));
  const int ns = (int)c.part.send_idx.size(), nr = (int)c.part.recv_idx.size();
  if (ns) k_halo_pack<<<div_up(3 * (int64_t)ns, 256), 256, 0, c.halo_stream>>>(ns, c.halo_send_idx, vec, c.halo_send);
  c.comm->exchange(c.part.peers, c.halo_send, c.halo_recv, c.halo_stream);
  if (nr) k_halo_unpack<<<div_up(3 * (int64_t)nr, 256), 256, 0, c.halo_stream>>>(nr, c.halo_recv_idx, c.halo_recv, vec);
  MS_CUDA(cudaEventRecord(c.ev_halo, c.halo_stream));
  c.launches += 2;
  MS_CUDA(cudaGetLastError());
}

void dist_sum(Ctx &c, double *dev, int64_t n) {
  if (c.dist() && n > 0) c.comm->allreduce_sum(dev, n, c.stream);
}

void dist_min(Ctx &c, double *dev, int64_t n) {
  if (c.dist() && n > 0) c.comm->allreduce_min(dev, n, c.stream);
}

}  // namespace msim
