// Subspace (coarse) levels: B lift / restrict, Galerkin products S = U_s^T H U_s and
// S_a = U_a^T H U_a, tile-envelope Cholesky of S, triangular solves, and the two-stage
// subspace direction of Alg. 2 with exact coarse solves.
//
// SURVEY §8(a) rows a5 (Galerkin projection), a6 (factorisation), a7 (coarse correction).
// PAPER.md Eq. 7 L284-298 (LBS discretisation, P_i = I3 kron [1 x y z]), L300-302 (affine
// level), L356-362 (U_s blocks), Alg. 2; readings R4 (exact solves), R6 (rhs -g).
//
// Coordinates of handle i: q_i[4c + k], c = x,y,z row, k = monomial [1, X-c_i].  The 3x12
// block of (v, i) is I3 kron w_vi^T with w_vi = phi_i(v) [1, X_v - c_i].
//
// S = B^T H B is formed by one fused kernel (one CTA per handle i, no atomics):
//   R_i(u)[(c',k'), c] = sum_{v in N(u), i in supp(v)} w_vi[k'] H_vu[c'][c]     (36 per (i,u))
//   S_ij[(c',k'), (c,k)] = sum_{u in U_i, j in supp(u)} R_i(u)[(c',k'), c] w_uj[k]   (j >= i)
// with R_i(u) held in shared memory chunk by chunk; the lists are precomputed at ms_basis_upload.
#include "common.cuh"
#include "galerkin.cuh"
#include "reduce.cuh"

namespace msim {

// ------------------------------------------------------------------ lift / restrict
// w_v[c] (+)= sum_{i in supp(v)} phi_i(v) (q_i[4c] + sum_d (X_v - c_i)[d] q_i[4c+1+d])
__global__ void k_lift(int nv, const int32_t *__restrict__ vptr, const int32_t *__restrict__ handle,
                       const double *__restrict__ phi, const double *__restrict__ X,
                       const double *__restrict__ origins, const double *__restrict__ q,
                       double *__restrict__ w, const double *__restrict__ base, const int32_t *__restrict__ skip) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv || (skip && *skip)) return;
  double o[3] = {0.0, 0.0, 0.0};
  const double xv0 = X[3 * v], xv1 = X[3 * v + 1], xv2 = X[3 * v + 2];
  for (int k = vptr[v]; k < vptr[v + 1]; ++k) {
    const int i = handle[k];
    const double f = phi[k];
    const double m1 = xv0 - origins[3 * i], m2 = xv1 - origins[3 * i + 1], m3 = xv2 - origins[3 * i + 2];
    const double *qi = q + 12 * (size_t)i;
#pragma unroll
    for (int c = 0; c < 3; ++c) o[c] += f * (qi[4 * c] + m1 * qi[4 * c + 1] + m2 * qi[4 * c + 2] + m3 * qi[4 * c + 3]);
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) w[3 * v + c] = (base ? base[3 * v + c] : 0.0) + o[c];
}

__global__ void k_lift_affine(int nv, const double *__restrict__ phi_a, const double *__restrict__ X,
                              double ox, double oy, double oz, const double *__restrict__ q,
                              double *__restrict__ w) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const double f = phi_a[v];
  const double m1 = X[3 * v] - ox, m2 = X[3 * v + 1] - oy, m3 = X[3 * v + 2] - oz;
#pragma unroll
  for (int c = 0; c < 3; ++c) w[3 * v + c] = f * (q[4 * c] + m1 * q[4 * c + 1] + m2 * q[4 * c + 2] + m3 * q[4 * c + 3]);
}

// z_i[4c + k] = sign * sum_{v in supp(i)} phi_i(v) mono_k(v, i) y_v[c]   (one CTA per handle)
__global__ void __launch_bounds__(256) k_restrict(const int32_t *__restrict__ hptr, const int32_t *__restrict__ hvert,
                                                  const double *__restrict__ hphi, const double *__restrict__ X,
                                                  const double *__restrict__ origins, const double *__restrict__ y,
                                                  double sign, double *__restrict__ z, const int32_t *__restrict__ skip) {
  __shared__ double sh[12 * 32];
  if (skip && *skip) return;
  const int i = blockIdx.x;
  const double o0 = origins[3 * i], o1 = origins[3 * i + 1], o2 = origins[3 * i + 2];
  double acc[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) acc[k] = 0.0;
  for (int k = hptr[i] + threadIdx.x; k < hptr[i + 1]; k += blockDim.x) {
    const int v = hvert[k];
    const double f = hphi[k];
    const double mono[4] = {f, f * (X[3 * v] - o0), f * (X[3 * v + 1] - o1), f * (X[3 * v + 2] - o2)};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double yc = y[3 * v + c];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) acc[4 * c + kk] = fma(mono[kk], yc, acc[4 * c + kk]);
    }
  }
  block_sum<12>(acc, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 12; ++k) z[12 * (size_t)i + k] = sign * acc[k];
  }
}

__global__ void __launch_bounds__(256) k_restrict_affine(int nv, const double *__restrict__ phi_a,
                                                         const double *__restrict__ X, double ox, double oy,
                                                         double oz, const double *__restrict__ y, double sign,
                                                         double *__restrict__ partial, unsigned int *counter,
                                                         double *__restrict__ z) {
  double acc[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) acc[k] = 0.0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    const double f = phi_a[v];
    const double mono[4] = {f, f * (X[3 * v] - ox), f * (X[3 * v + 1] - oy), f * (X[3 * v + 2] - oz)};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double yc = y[3 * v + c];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) acc[4 * c + kk] = fma(mono[kk], yc, acc[4 * c + kk]);
    }
  }
  double res[12];
  if (grid_reduce<12>(acc, partial, counter, res) && threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 12; ++k) z[k] = sign * res[k];
  }
}

void launch_lift(Ctx &c, const double *q, double *w, bool accumulate, const int32_t *skip) {
  k_lift<<<div_up(c.nv, 256), 256, 0, c.stream>>>(c.nv, c.bvptr, c.bhandle, c.bphi, c.X, c.origins, q, w,
                                                  accumulate ? w : nullptr, skip);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

void launch_restrict(Ctx &c, const double *y, double *z, const int32_t *skip) {
  k_restrict<<<c.m, 256, 0, c.stream>>>(c.hptr, c.hvert, c.hphi, c.X, c.origins, y, 1.0, z, skip);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ Galerkin products (a5)

__global__ void __launch_bounds__(kGalThreads, 2) k_galerkin_fused(GalParams G) {
  extern __shared__ double gsm[];
  galerkin_row(G, blockIdx.x / G.nparts, blockIdx.x % G.nparts, gsm);
}

__global__ void __launch_bounds__(256) k_galerkin_reduce(GalParams G) { galerkin_reduce_row(G, blockIdx.x); }

// Affine: Ra(u) = sum_{v in N(u)} w_a(v) kron H_vu  stored SoA [36][nv]
__global__ void __launch_bounds__(128) k_galerkin_Ra(int nv, HView H, const double *__restrict__ phi_a,
                                                     const double *__restrict__ X, double ox, double oy,
                                                     double oz, double *__restrict__ Ra) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nv) return;
  double acc[36];
#pragma unroll
  for (int k = 0; k < 36; ++k) acc[k] = 0.0;
  const int sl_ = u >> 5, ln_ = u & 31;
  for (int cs = H.sl_ptr[sl_]; cs < H.sl_ptr[sl_ + 1]; ++cs) {
    const int v = H.col[(size_t)cs * 32 + ln_];
    const double f = phi_a[v];
    if (f == 0.0) continue;
    const double w[4] = {f, f * (X[3 * v] - ox), f * (X[3 * v + 1] - oy), f * (X[3 * v + 2] - oz)};
    double Hvu[3][3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
#pragma unroll
      for (int cp = 0; cp < 3; ++cp) Hvu[cp][cc] = H.vals[((size_t)cs * 9 + 3 * cc + cp) * 32 + ln_];
#pragma unroll
    for (int cp = 0; cp < 3; ++cp)
#pragma unroll
      for (int kp = 0; kp < 4; ++kp)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) acc[(4 * cp + kp) * 3 + cc] = fma(w[kp], Hvu[cp][cc], acc[(4 * cp + kp) * 3 + cc]);
  }
#pragma unroll
  for (int k = 0; k < 36; ++k) Ra[(size_t)k * nv + u] = acc[k];
}

// S_a[(row), (4c + k)] = sum_u Ra(u)[l] w_a(u)[k], l = 3 row + c.  Grid: (36 entries) x chunks.
// rows u < n_use (the owned vertices) of Ra, stored [36][nv]
__global__ void __launch_bounds__(256) k_galerkin_Sa_partial(int nv, int n_use, const double *__restrict__ Ra,
                                                             const double *__restrict__ phi_a,
                                                             const double *__restrict__ X, double ox,
                                                             double oy, double oz,
                                                             double *__restrict__ part /* [36][4][chunks] */) {
  __shared__ double sh[4 * 32];
  const int l = blockIdx.x, chunk = blockIdx.y, nch = gridDim.y;
  double acc[4] = {0, 0, 0, 0};
  for (int u = chunk * blockDim.x + threadIdx.x; u < n_use; u += nch * blockDim.x) {
    const double f = phi_a[u];
    const double rv = Ra[(size_t)l * nv + u];
    const double w[4] = {f, f * (X[3 * u] - ox), f * (X[3 * u + 1] - oy), f * (X[3 * u + 2] - oz)};
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] = fma(rv, w[k], acc[k]);
  }
  block_sum<4>(acc, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) part[((size_t)l * 4 + k) * nch + chunk] = acc[k];
  }
}

__global__ void k_galerkin_Sa_final(int nch, const double *__restrict__ part, double *__restrict__ Sa) {
  const int t = threadIdx.x;  // 144 threads: (l, k)
  if (t >= 144) return;
  const int l = t / 4, k = t % 4;
  double s = 0.0;
  for (int ch = 0; ch < nch; ++ch) s += part[((size_t)l * 4 + k) * nch + ch];
  const int row = l / 3, c = l % 3;
  Sa[row * 12 + 4 * c + k] = s;
}

// the subspace Hessian (NEXT-2: the cubature Hessian; else H itself)
HView hview(const Ctx &c) { return HView{c.sl_ptr, c.sell_col, c.vals_sub()}; }

GalParams galerkin_params(const Ctx &c) {
  GalParams G;
  G.H = hview(c);
  G.gU_ptr = c.gU_ptr;
  G.gU = c.gU;
  G.ga_off = c.ga_off;
  G.ga_ent = c.ga_ent;
  G.ga_mask = c.ga_mask;
  G.gj_ptr = c.gj_ptr;
  G.gj_blk = c.gj_blk;
  G.gl_base = c.gl_base;
  G.gl_off = c.gl_off;
  G.gl_ent = c.gl_ent;
  G.W = c.Wphi;
  G.ga_w = c.ga_w;
  G.gl_w = c.gl_w;
  G.sT = c.sT;
  G.scol = c.scol;
  G.S = c.Sblk;
  G.Spart = c.Spart;
  G.nparts = c.gal_parts;
  G.pstride = 144 * c.gal_max_jup;
  return G;
}

// ------------------------------------------------------------------ dense envelope S
// Lden column-major nS_pad x nS_pad; scatter lower part of S blocks; padding -> identity.
__global__ void k_scatter_S(int64_t nblk, const int32_t *__restrict__ srow, const int32_t *__restrict__ scol,
                            const int32_t *__restrict__ perm, const double *__restrict__ S, int nSp,
                            double *__restrict__ L) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nblk * 144) return;
  const int64_t b = t / 144;
  const int e = (int)(t % 144), row = e / 12, col = e % 12;
  const int i = perm[srow[b]], j = perm[scol[b]];
  const int R = 12 * i + row, C = 12 * j + col;
  if (R >= C) L[(size_t)C * nSp + R] = S[t];
}

// z_perm[12 perm[i] + r] = z[12 i + r]  (dir = 0);  z[12 i + r] = z_perm[12 perm[i] + r]  (dir = 1)
__global__ void k_permute(int m, const int32_t *__restrict__ perm, const double *__restrict__ src,
                          double *__restrict__ dst, int dir) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 12 * m) return;
  const int i = t / 12, r = t % 12;
  if (dir == 0) dst[12 * perm[i] + r] = src[t];
  else dst[t] = src[12 * perm[i] + r];
}

__global__ void k_pad_identity(int nS, int nSp, double *__restrict__ L) {
  const int r = nS + blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nSp) L[(size_t)r * nSp + r] = 1.0;
}

// ------------------------------------------------------------------ 12x12 affine solve
// q = S_a^-1 z by Cholesky: one CTA of 144 threads, right-looking in shared memory (thread (r, c)
// updates entry (r, c)), then the two triangular sweeps by one thread (78 FMA each).  (Round 1 ran
// the whole factorisation in one thread from local memory: 17-19 us per Newton iteration.)
__global__ void __launch_bounds__(144) k_solve12(const double *__restrict__ Sa, const double *__restrict__ z,
                                                 double *__restrict__ q, int *__restrict__ flag) {
  __shared__ double A[12][13];
  const int t = threadIdx.x, r = t / 12, c = t % 12;
  A[r][c] = Sa[t];
  __syncthreads();
  for (int j = 0; j < 12; ++j) {
    if (t == 0) {
      double d = A[j][j];
      if (!(d > 0.0)) {
        *flag = 1;
        d = 1.0;
      }
      A[j][j] = sqrt(d);
    }
    __syncthreads();
    if (t > j && t < 12) A[t][j] /= A[j][j];
    __syncthreads();
    if (r > j && c > j && c <= r) A[r][c] = fma(-A[r][j], A[c][j], A[r][c]);
    __syncthreads();
  }
  if (t == 0) {
    double y[12];
    for (int i = 0; i < 12; ++i) {
      double s = z[i];
      for (int k = 0; k < i; ++k) s = fma(-A[i][k], y[k], s);
      y[i] = s / A[i][i];
    }
    for (int i = 11; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < 12; ++k) s = fma(-A[k][i], q[k], s);
      q[i] = s / A[i][i];
    }
  }
}

// W[p] = phi_p [1, X_u - c_j] for every (vertex u, handle j) basis entry p (static per basis)
__global__ void k_basis_W(int nv, const int32_t *__restrict__ vptr, const int32_t *__restrict__ handle,
                          const double *__restrict__ phi, const double *__restrict__ X,
                          const double *__restrict__ origins, double *__restrict__ W) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nv) return;
  for (int p = vptr[u]; p < vptr[u + 1]; ++p) {
    const int j = handle[p];
    const double f = phi[p];
    W[4 * (size_t)p] = f;
    W[4 * (size_t)p + 1] = f * (X[3 * u] - origins[3 * j]);
    W[4 * (size_t)p + 2] = f * (X[3 * u + 1] - origins[3 * j + 1]);
    W[4 * (size_t)p + 3] = f * (X[3 * u + 2] - origins[3 * j + 2]);
  }
}

// out[e] = W[ent[e] >> shift] (4 doubles per entry)
__global__ void k_gather_w(int64_t n, const uint32_t *__restrict__ ent, int shift, const double *__restrict__ W,
                           double *__restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const size_t p = ent[e] >> shift;
  const double4 w = *reinterpret_cast<const double4 *>(W + 4 * p);
  *reinterpret_cast<double4 *>(out + 4 * e) = w;
}

void launch_basis_W(Ctx &c) {
  c.Wphi.alloc(4 * (size_t)c.nnz_phi);
  k_basis_W<<<div_up(c.nv, 256), 256, 0, c.stream>>>(c.nv, c.bvptr, c.bhandle, c.bphi, c.X, c.origins, c.Wphi);
  c.launches++;
  // the Galerkin lists' weights in list order: phase A reads entry (u, slot) with the H row, phase
  // B entry (u, j) with its u index, both without the dependent index -> W round trip
  const int64_t na = (int64_t)c.ga_ent.n, nl = (int64_t)c.gl_ent.n;
  c.ga_w.alloc(4 * (size_t)na);
  c.gl_w.alloc(4 * (size_t)nl);
  k_gather_w<<<(unsigned)div_up(na, 256), 256, 0, c.stream>>>(na, c.ga_ent, 6, c.Wphi, c.ga_w);
  k_gather_w<<<(unsigned)div_up(nl, 256), 256, 0, c.stream>>>(nl, c.gl_ent, 7, c.Wphi, c.gl_w);
  c.launches += 2;
  MS_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ launchers
// per context, on its device (create_common): the Galerkin kernel's opt-in is raised to the
// device maximum once (never lowered: a launch uses what its basis needs)
void coarse_init_attrs(Ctx &c) {
  set_max_dyn_smem((const void *)k_galerkin_fused, c.device);
}

// ------------------------------------------------------------------ paper coarse mode (NEXT-1)
// MS_COARSE_PCG (§3.7.1, Alg. 2): the SMS stage solves
// (U_s^T H U_s) q = U_s^T r1 by PCG to ||r|| <= tol ||b|| on the matrix-free sandwich -- each
// iteration lifts (w = B p), applies H (y = H w) and restricts (t = B^T y) -- with the 12 x 12
// block-Jacobi preconditioner S_ii^-1 (blocks from the diagonal-block Galerkin rows).
// The affine stage has one 12 x 12 block, so its block-Jacobi PCG is exact after one step: it
// is the 12 x 12 Cholesky solve of the exact mode.
// Iterations run in captured batches of kCpcgBatch; every kernel of an iteration returns at once
// when the device flag state[0] says the solve has converged, so the iterates are exactly those
// of a loop stopped at the first k with ||r_k|| <= tol ||b|| (tested against oracle/solver.py).

// S_ii^-1 = L^-T L^-1 (one thread per handle, 12 x 12 in local memory; once per Newton iteration)
__global__ void k_block_inv(int m, const double *__restrict__ Sd, double *__restrict__ Minv, int *__restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double L[12][12], Li[12][12];
  for (int r = 0; r < 12; ++r)
    for (int c = 0; c < 12; ++c) {
      L[r][c] = Sd[144 * (size_t)i + 12 * r + c];
      Li[r][c] = 0.0;
    }
  for (int j = 0; j < 12; ++j) {
    double d = L[j][j];
    for (int k = 0; k < j; ++k) d -= L[j][k] * L[j][k];
    if (!(d > 0.0)) {
      *flag = 1;
      d = 1.0;
    }
    L[j][j] = sqrt(d);
    for (int r = j + 1; r < 12; ++r) {
      double s = L[r][j];
      for (int k = 0; k < j; ++k) s -= L[r][k] * L[j][k];
      L[r][j] = s / L[j][j];
    }
  }
  for (int c = 0; c < 12; ++c)
    for (int r = c; r < 12; ++r) {
      double s = r == c ? 1.0 : 0.0;
      for (int k = c; k < r; ++k) s -= L[r][k] * Li[k][c];
      Li[r][c] = s / L[r][r];
    }
  for (int a = 0; a < 12; ++a)
    for (int b = 0; b < 12; ++b) {
      double s = 0.0;
      for (int r = a > b ? a : b; r < 12; ++r) s = fma(Li[r][a], Li[r][b], s);
      Minv[144 * (size_t)i + 12 * a + b] = s;
    }
}

constexpr int kCpcgThreads = 1024;
constexpr int kCpcgBatch = 8;

// z_e = (S_ii^-1 r_i)[row] for entry e = 12 i + row
__device__ __forceinline__ double block_precond(const double *__restrict__ Minv, const double *__restrict__ r, int e) {
  const int i = e / 12, row = e - 12 * i;
  const double *Mi = Minv + 144 * (size_t)i + 12 * row, *ri = r + 12 * (size_t)i;
  double z = 0.0;
#pragma unroll
  for (int k = 0; k < 12; ++k) z = fma(Mi[k], ri[k], z);
  return z;
}

__device__ __forceinline__ double cta_sum(double v, double *sh) {
  double a[1] = {v};
  block_sum<1>(a, sh);
  if (threadIdx.x == 0) sh[32] = a[0];
  __syncthreads();
  const double out = sh[32];
  __syncthreads();
  return out;
}

// q = 0, r = b, z = M^-1 r, p = z, rho = r.z, ||b||^2; state = {done, iterations}
__global__ void __launch_bounds__(kCpcgThreads) k_cpcg_init(int n, const double *__restrict__ b,
                                                           const double *__restrict__ Minv, double *__restrict__ q,
                                                           double *__restrict__ r, double *__restrict__ z,
                                                           double *__restrict__ p, double *__restrict__ scal,
                                                           int32_t *__restrict__ state, int max_iter) {
  __shared__ double sh[33];
  double rz = 0.0, bb = 0.0;
  for (int e = threadIdx.x; e < n; e += kCpcgThreads) {
    const double zi = block_precond(Minv, b, e), bi = b[e];
    q[e] = 0.0;
    r[e] = bi;
    z[e] = zi;
    p[e] = zi;
    rz = fma(bi, zi, rz);
    bb = fma(bi, bi, bb);
  }
  rz = cta_sum(rz, sh);
  bb = cta_sum(bb, sh);
  if (threadIdx.x == 0) {
    scal[SC_CP_RHO] = rz;
    scal[SC_CP_BN2] = bb;
    state[0] = (bb == 0.0 || max_iter <= 0) ? 1 : 0;
    state[1] = 0;
  }
}

// one iteration after t = S p: alpha = rho / p.t; q += alpha p; r -= alpha t; stop at
// ||r||^2 <= tol^2 ||b||^2 or the cap; else z = M^-1 r, beta = r.z / rho, p = z + beta p
__global__ void __launch_bounds__(kCpcgThreads) k_cpcg_step(int n, const double *__restrict__ t,
                                                           const double *__restrict__ Minv, double *__restrict__ q,
                                                           double *__restrict__ r, double *__restrict__ z,
                                                           double *__restrict__ p, double *__restrict__ scal,
                                                           int32_t *__restrict__ state, double tol2, int max_iter) {
  __shared__ double sh[33];
  __shared__ int done;
  if (threadIdx.x == 0) done = state[0];
  __syncthreads();
  if (done) return;
  double pt = 0.0;
  for (int e = threadIdx.x; e < n; e += kCpcgThreads) pt = fma(p[e], t[e], pt);
  pt = cta_sum(pt, sh);
  const double rho = scal[SC_CP_RHO];
  const double alpha = (pt != 0.0 && rho != 0.0) ? rho / pt : 0.0;
  double rr = 0.0;
  for (int e = threadIdx.x; e < n; e += kCpcgThreads) {
    q[e] = fma(alpha, p[e], q[e]);
    const double re = fma(-alpha, t[e], r[e]);
    r[e] = re;
    rr = fma(re, re, rr);
  }
  rr = cta_sum(rr, sh);   // (its barriers also publish r for the block products below)
  const int it = state[1] + 1;
  if (rr <= tol2 * scal[SC_CP_BN2] || it >= max_iter) {
    if (threadIdx.x == 0) {
      state[0] = 1;
      state[1] = it;
    }
    return;
  }
  double rz = 0.0;
  for (int e = threadIdx.x; e < n; e += kCpcgThreads) {
    const double ze = block_precond(Minv, r, e);
    z[e] = ze;
    rz = fma(r[e], ze, rz);
  }
  rz = cta_sum(rz, sh);
  const double beta = rho != 0.0 ? rz / rho : 0.0;
  for (int e = threadIdx.x; e < n; e += kCpcgThreads) p[e] = fma(beta, p[e], z[e]);
  __syncthreads();
  if (threadIdx.x == 0) {
    scal[SC_CP_RHO] = rz;
    state[1] = it;
  }
}

static void enqueue_cpcg_batch(Ctx &c) {
  const int n = 12 * c.m;
  const double tol2 = c.params.coarse_tol * c.params.coarse_tol;
  for (int k = 0; k < kCpcgBatch; ++k) {
    launch_lift(c, c.cp_p, c.tmp, false, c.cp_state);      // w = B p
    launch_spmv(c, c.tmp, c.r, 0.0, nullptr, c.cp_state, c.vals_sub());  // y = H w
    launch_restrict(c, c.r, c.cp_t, c.cp_state);           // t = B^T y
    dist_sum(c, c.cp_t, n);
    k_cpcg_step<<<1, kCpcgThreads, 0, c.stream>>>(n, c.cp_t, c.Minv, c.qs, c.cp_r, c.cp_z, c.cp_p, c.scal,
                                                  c.cp_state, tol2, c.params.coarse_max_iter);
    c.launches++;
  }
}

// SMS stage of the paper's coarse mode: q (in c.qs) from b = B^T r1 (in c.zs)
static void coarse_pcg_solve(Ctx &c) {
  const int n = 12 * c.m;
  k_cpcg_init<<<1, kCpcgThreads, 0, c.stream>>>(n, c.zs, c.Minv, c.qs, c.cp_r, c.cp_z, c.cp_p, c.scal, c.cp_state,
                                                c.params.coarse_max_iter);
  c.launches++;
  const bool graphs = c.params.use_graphs && (!c.dist() || c.comm->capturable());
  int32_t *hs = reinterpret_cast<int32_t *>(c.h_pinned + PH_COUNT - 2);
  for (int batch = 0;; ++batch) {
    if (graphs) {
      if (!c.cpcg_graph) {
        cudaStream_t cap;
        MS_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        cudaStream_t saved = c.stream;
        c.stream = cap;
        cudaGraph_t graph;
        MS_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        const int64_t l0 = c.launches;
        enqueue_cpcg_batch(c);
        c.cpcg_graph_kernels = c.launches - l0;
        c.launches = l0;
        MS_CUDA(cudaStreamEndCapture(cap, &graph));
        c.stream = saved;
        MS_CUDA(cudaGraphInstantiate(&c.cpcg_graph, graph, 0));
        cudaGraphDestroy(graph);
        cudaStreamDestroy(cap);
      }
      MS_CUDA(cudaGraphLaunch(c.cpcg_graph, c.stream));
      c.launches += c.cpcg_graph_kernels;
    } else {
      enqueue_cpcg_batch(c);
    }
    MS_CUDA(cudaMemcpyAsync(hs, c.cp_state, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
    MS_CUDA(cudaStreamSynchronize(c.stream));
    if (hs[0]) break;
    MS_REQUIRE(batch < (c.params.coarse_max_iter + kCpcgBatch - 1) / kCpcgBatch + 1, MS_ERR_STATE,
               "coarse PCG did not stop");
  }
  c.coarse_iters_last = hs[1];
}

// per Newton iteration: the diagonal blocks S_ii (fused Galerkin kernel with U_i = supp(i) and
// the single slot j = i) and their inverses
static void coarse_pcg_blocks(Ctx &c) {
  build_coarse_pcg_structures(c);
  GalParams G = galerkin_params(c);
  G.gU_ptr = c.gd_U_ptr;
  G.gU = c.gd_U;
  G.ga_off = c.gd_ga_off;
  G.ga_ent = c.gd_ga_ent;
  G.ga_mask = c.gd_ga_mask;
  G.gj_ptr = c.gd_gj_ptr;
  G.gj_blk = c.gd_gj_blk;
  G.gl_base = c.gd_gl_base;
  G.gl_off = c.gd_gl_off;
  G.gl_ent = c.gd_gl_ent;
  G.ga_w = G.gl_w = nullptr;   // (diagonal-block lists: W gathered through the index)
  G.sT = c.gd_sT;
  G.S = c.Sdiag;
  G.Spart = c.Sdiag_part;
  G.pstride = 144;
  const size_t smem = sizeof(double) * galerkin_smem_doubles(1);
  k_galerkin_fused<<<c.m * G.nparts, kGalThreads, smem, c.stream>>>(G);
  c.launches++;
  if (G.nparts > 1) {
    k_galerkin_reduce<<<c.m, 256, 0, c.stream>>>(G);
    c.launches++;
  }
  dist_sum(c, c.Sdiag, 144 * (int64_t)c.m);
}

void launch_coarse_pcg_prep(Ctx &c) {
  k_block_inv<<<div_up(c.m, 128), 128, 0, c.stream>>>(c.m, c.Sdiag, c.Minv, c.flags + 0);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

// S = B^T H B into Sblk (full_S, or whenever the Galerkin rows are not fused into the factor
// launch) and S_a = U_a^T H U_a.  With c.gal_fused the rows of S are formed by the factorisation
// launch itself (chol.cu: G / R tasks write straight into the factor's tiles).
void launch_coarse_S(Ctx &c, bool full_S) {
  const bool pcg = c.params.coarse_mode == MS_COARSE_PCG;
  if (pcg && !full_S) coarse_pcg_blocks(c);
  if (full_S || (!c.gal_fused && !pcg)) {
    const size_t smem = sizeof(double) * galerkin_smem_doubles(c.gal_max_jup);
    MS_REQUIRE(smem <= 227 * 1024, MS_ERR_ARG, "coarse S row too wide for the fused Galerkin kernel");
    const GalParams G = galerkin_params(c);
    k_galerkin_fused<<<c.m * G.nparts, kGalThreads, smem, c.stream>>>(G);
    c.launches++;
    if (G.nparts > 1) {
      k_galerkin_reduce<<<c.m, 256, 0, c.stream>>>(G);
      c.launches++;
    }
  }
  const double *o = c.aff_origin;
  k_galerkin_Ra<<<div_up(c.nv, 128), 128, 0, c.stream>>>(c.nv, hview(c), c.phi_aff, c.X, o[0], o[1], o[2], c.Ra);
  const int nch = 64;
  k_galerkin_Sa_partial<<<dim3(36, nch), 256, 0, c.stream>>>(c.nv, c.nv_own, c.Ra, c.phi_aff, c.X, o[0], o[1], o[2],
                                                              c.partial);
  k_galerkin_Sa_final<<<1, 160, 0, c.stream>>>(nch, c.partial, c.Sa);
  c.launches += 3;
  // multi-GPU: each rank projected its owned rows u; S and S_a are the sums over ranks
  dist_sum(c, c.Sblk, 144 * c.nnzb_S);
  dist_sum(c, c.Sa, 144);
  MS_CUDA(cudaGetLastError());
}

void launch_scatter_S(Ctx &c) {
  k_scatter_S<<<div_up(c.nnzb_S * 144, 256), 256, 0, c.stream>>>(c.nnzb_S, c.srow, c.scol, c.perm, c.Sblk,
                                                                  c.nS_pad, c.Lden);
}

// Capture a fixed launch sequence once (pointers are fixed per basis) and replay it.
template <typename F>
static void run_captured(Ctx &c, cudaGraphExec_t &exec, F enqueue) {
  const bool graphs = c.params.use_graphs;   // (no collectives inside: replicated factor / solves)
  if (!graphs) {
    enqueue(c);
    return;
  }
  if (!exec) {
    cudaStream_t cap;
    MS_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaStream_t saved = c.stream;
    c.stream = cap;
    cudaGraph_t graph;
    MS_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    enqueue(c);
    MS_CUDA(cudaStreamEndCapture(cap, &graph));
    c.stream = saved;
    MS_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cap);
  }
  MS_CUDA(cudaGraphLaunch(exec, c.stream));
}

void coarse_reset_graphs(Ctx &c) {
  if (c.factor_graph) cudaGraphExecDestroy(c.factor_graph);
  if (c.solve_graph) cudaGraphExecDestroy(c.solve_graph);
  if (c.cpcg_graph) cudaGraphExecDestroy(c.cpcg_graph);
  if (c.tl_graph) cudaGraphExecDestroy(c.tl_graph);
  c.factor_graph = c.solve_graph = c.cpcg_graph = c.tl_graph = nullptr;
}

void launch_coarse_factor(Ctx &c) {
  if (c.params.coarse_mode == MS_COARSE_PCG) {   // the paper's mode: block-Jacobi inverses only
    launch_coarse_pcg_prep(c);
    return;
  }
  run_captured(c, c.factor_graph, enqueue_chol_factor);
  c.launches += chol_factor_kernels(c);
  MS_CUDA(cudaGetLastError());
}

void launch_coarse_solve(Ctx &c) {
  run_captured(c, c.solve_graph, [](Ctx &cc) { enqueue_chol_solve(cc); });
  c.launches += chol_solve_kernels(c);
  MS_CUDA(cudaGetLastError());
}

void launch_coarse_direction(Ctx &c) {
  const int n3 = 3 * c.nv;
  const double *o = c.aff_origin;
  // rhs = -g
  launch_axpby(c, c.rhs, -1.0, c.g, 0.0, n3);
  // affine stage: za = U_a^T(-g); qa = Sa^-1 za; da = U_a qa
  k_restrict_affine<<<std::min(div_up(c.nv_own, 256), 592), 256, 0, c.stream>>>(
      c.nv_own, c.phi_aff, c.X, o[0], o[1], o[2], c.rhs, 1.0, c.partial, c.counters + 6, c.za);
  dist_sum(c, c.za, 12);
  k_solve12<<<1, 144, 0, c.stream>>>(c.Sa, c.za, c.qa, c.flags + 1);
  k_lift_affine<<<div_up(c.nv, 256), 256, 0, c.stream>>>(c.nv, c.phi_aff, c.X, o[0], o[1], o[2], c.qa, c.da);
  c.launches += 3;
  // r1 = -g - H da
  launch_spmv(c, c.da, c.tmp, 0.0, c.rhs, nullptr, c.vals_sub());
  // SMS stage: zs = B^T r1; zs <- S^-1 zs; ds = da + B zs
  launch_restrict(c, c.tmp, c.zs);
  dist_sum(c, c.zs, 12 * (int64_t)c.m);
  const bool pcg = c.params.coarse_mode == MS_COARSE_PCG;
  if (pcg) coarse_pcg_solve(c);   // q in qs (tmp and r are its work vectors)
  else launch_coarse_solve(c);    // q in zs
  MS_CUDA(cudaMemcpyAsync(c.ds, c.da, sizeof(double) * n3, cudaMemcpyDeviceToDevice, c.stream));
  launch_lift(c, pcg ? c.qs : c.zs, c.ds, true);
  // r = -g - H ds
  launch_spmv(c, c.ds, c.r, 0.0, c.rhs, nullptr, c.vals_sub());
  MS_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ NEXT-4: two-level refinement
// PCG on H d_f = r1 from d_f = 0 with y = D^-1 r, z = y + U_s S^-1 U_s^T (r - H y) (the SMS factor of
// this Newton iteration: SpMV, restrict, the two cooperative triangular sweeps, lift; "A-DEF2",
// equal to the balancing preconditioner since U_s^T r1 = 0 after the SMS stage), stopped at the first k with
// ||r_k||^2 <= tol^2 ||g||^2 or k = refine_max_iter (reading N4; oracle/solver.py two_level_pcg).
// Host-driven batches of kTlBatch iterations, one CUDA graph; once the device flag tl_state[0] is
// set every launch of a batch returns at once, so the iterates are exactly those of a loop that
// stopped at k.  Scalars: rho = SC_RZ, beta = SC_BETA, alpha = SC_ALPHA (k_pcg_spmv's slots).
constexpr int kTlBatch = 4;

// x += alpha p; r -= alpha q; z = D^-1 r (the Jacobi part of the preconditioner)
__global__ void __launch_bounds__(256) k_tl_update(int n3, const double *__restrict__ dinv,
                                                   const double *__restrict__ p, const double *__restrict__ q,
                                                   double *__restrict__ x, double *__restrict__ r,
                                                   double *__restrict__ z, const double *__restrict__ scal,
                                                   const int32_t *__restrict__ skip) {
  if (*skip) return;
  const double alpha = scal[SC_ALPHA];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n3; i += gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    z[i] = dinv[i] * ri;
  }
}

// [r.z, r.r] over the owned entries -> scal[SC_TL_RZ], scal[SC_TL_RR] (deterministic grid sum)
__global__ void __launch_bounds__(256) k_tl_dots(int n3_own, const double *__restrict__ r,
                                                 const double *__restrict__ z, double *__restrict__ partial,
                                                 unsigned int *counter, double *__restrict__ scal,
                                                 const int32_t *__restrict__ skip) {
  if (*skip) return;
  double acc[2] = {0.0, 0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n3_own; i += gridDim.x * blockDim.x) {
    acc[0] = fma(r[i], z[i], acc[0]);
    acc[1] = fma(r[i], r[i], acc[1]);
  }
  grid_reduce<2>(acc, partial, counter, scal + SC_TL_RZ);
}

// stopping rule and beta (init: the check of r_0, rho = r_0.z_0, beta = 0)
__global__ void k_tl_decide(double *__restrict__ scal, int32_t *__restrict__ state, double tol2, int max_iter,
                            int init) {
  if (state[0]) return;
  const double rz = scal[SC_TL_RZ], rr = scal[SC_TL_RR], gg = scal[SC_GNORM2];
  if (init) {
    if (rr <= tol2 * gg || max_iter <= 0) {
      state[0] = 1;
      state[1] = 0;
      return;
    }
    scal[SC_RZ] = rz;
    scal[SC_RZ0] = rz;
    scal[SC_BETA] = 0.0;
    state[1] = 0;
    return;
  }
  const int it = state[1] + 1;
  state[1] = it;
  if (rr <= tol2 * gg || it >= max_iter) {
    state[0] = 1;
    return;
  }
  const double rho = scal[SC_RZ];
  scal[SC_BETA] = rho != 0.0 ? rz / rho : 0.0;
  scal[SC_RZ] = rz;
}

static int tl_grid(int64_t n) { return (int)std::min<int64_t>(div_up(n, 256), 148 * 8); }

// z = y + U_s S^-1 U_s^T (r - H y) with y = D^-1 r already in z, then r.z, r.r and the decision
static void enqueue_tl_precond_decide(Ctx &c, int init) {
  const int32_t *skip = c.tl_state;
  if (c.dist()) halo_exchange(c, c.z);                 // y at the ghost vertices (SpMV input)
  launch_spmv(c, c.z, c.tmp, 0.0, c.r, skip, nullptr);  // t = r - H_ref y (owned rows exact)
  launch_restrict(c, c.tmp, c.zs, skip);
  dist_sum(c, c.zs, 12 * (int64_t)c.m);
  enqueue_chol_solve(c, skip);
  c.launches += chol_solve_kernels(c);
  launch_lift(c, c.zs, c.z, true, skip);               // replicated coarse vector: ghosts exact too
  k_tl_dots<<<tl_grid(3 * (int64_t)c.nv_own), 256, 0, c.stream>>>(3 * c.nv_own, c.r, c.z, c.partial,
                                                                  c.counters + 10, c.scal, skip);
  dist_sum(c, c.scal + SC_TL_RZ, 2);
  const double tol2 = c.params.refine_tol * c.params.refine_tol;
  k_tl_decide<<<1, 1, 0, c.stream>>>(c.scal, c.tl_state, tol2, c.params.refine_max_iter, init);
  c.launches += 2;
}

static void enqueue_tl_batch(Ctx &c, double *sol) {
  const int n3 = 3 * c.nv;
  for (int k = 0; k < kTlBatch; ++k) {
    launch_pcg_spmv(c, c.tl_state);   // p = z + beta p, q = H p, alpha
    k_tl_update<<<tl_grid(n3), 256, 0, c.stream>>>(n3, c.dinv, c.p, c.q, sol, c.r, c.z, c.scal, c.tl_state);
    c.launches++;
    enqueue_tl_precond_decide(c, 0);
  }
}

int launch_refine_two_level(Ctx &c, const double *rhs, double *sol) {
  MS_REQUIRE(c.params.coarse_mode == MS_COARSE_EXACT, MS_ERR_STATE, "two-level refinement needs the coarse factor");
  if (c.tl_state.n == 0) c.tl_state.alloc(2);
  MS_CUDA(cudaMemsetAsync(c.tl_state, 0, 2 * sizeof(int32_t), c.stream));
  launch_pcg_init(c, rhs, sol);   // x = 0, r = rhs, z = D^-1 r, p = q = 0
  enqueue_tl_precond_decide(c, 1);
  const bool graphs = c.params.use_graphs && sol == c.df.p && (!c.dist() || c.comm->capturable());
  int32_t *hs = reinterpret_cast<int32_t *>(c.h_pinned + PH_COUNT - 2);
  for (int batch = 0;; ++batch) {
    if (graphs) {
      if (!c.tl_graph) {
        cudaStream_t cap;
        MS_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        cudaStream_t saved = c.stream;
        c.stream = cap;
        cudaGraph_t graph;
        MS_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        const int64_t l0 = c.launches;
        enqueue_tl_batch(c, sol);
        c.tl_graph_kernels = c.launches - l0;
        c.launches = l0;
        MS_CUDA(cudaStreamEndCapture(cap, &graph));
        c.stream = saved;
        MS_CUDA(cudaGraphInstantiate(&c.tl_graph, graph, 0));
        cudaGraphDestroy(graph);
        cudaStreamDestroy(cap);
      }
      MS_CUDA(cudaGraphLaunch(c.tl_graph, c.stream));
      c.launches += c.tl_graph_kernels;
    } else {
      enqueue_tl_batch(c, sol);
    }
    MS_CUDA(cudaMemcpyAsync(hs, c.tl_state, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
    MS_CUDA(cudaStreamSynchronize(c.stream));
    if (hs[0]) break;
    MS_REQUIRE(batch < c.params.refine_max_iter / kTlBatch + 1, MS_ERR_STATE, "two-level PCG did not stop");
  }
  MS_CUDA(cudaGetLastError());
  c.refine_iters_last = hs[1];
  return hs[1];
}

// standalone solve used by the parity hook ms_subspace_direction (same code path)
}  // namespace msim
