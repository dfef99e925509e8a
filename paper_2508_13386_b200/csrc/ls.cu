// Filtered backtracking line search.
//
// "filter for intersection with CCD (and non-inversion checks ...)
// to truncate the initial step size ... then backtracking line search on the full-space IP
// energy".  Readings Q12 (halving, strict decrease, alpha_min = 1e-8, safety 0.9; the decrease
// test is evaluated as a sum of per-element / per-vertex energy differences) and SPEC S:170,179.
//
// B200 design: the CCD (ground plane, per vertex) and inversion (per tet: smallest positive
// root of det(Ds + t dDs)) filters are min-reductions (order-independent, exact).  The
// backtracking is batched: K candidate steps alpha0 * shrink^k are evaluated in ONE pass over
// the tets and vertices (deterministic grid reductions of 2K values); the host accepts the
// first k with a strict decrease, which is identical to sequential backtracking.
#include "common.cuh"
#include "reduce.cuh"

namespace msim {

struct LSMesh {
  int32_t nt;
  const int4 *__restrict__ tets;
  const double *__restrict__ Bm;
  const double *__restrict__ vol;
  const double *__restrict__ mu;
  const double *__restrict__ lam;
};
static LSMesh lsmesh(const Ctx &c) {
  return LSMesh{c.nt, reinterpret_cast<const int4 *>(c.tets.p), c.Bm.p, c.vol.p, c.mu.p, c.lam.p};
}

__device__ __forceinline__ double det3m(const double A[3][3]) {
  return A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
         A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
}
__device__ __forceinline__ void cof3(const double F[3][3], double C[3][3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int a = (k + 1) % 3, b = (k + 2) % 3;
    C[0][k] = F[1][a] * F[2][b] - F[2][a] * F[1][b];
    C[1][k] = F[2][a] * F[0][b] - F[0][a] * F[2][b];
    C[2][k] = F[0][a] * F[1][b] - F[1][a] * F[0][b];
  }
}

__device__ __forceinline__ void edge_mats(const LSMesh &M, int e, const double *__restrict__ x,
                                          const double *__restrict__ d, double Ds[3][3], double dD[3][3],
                                          int4 &t) {
  t = __ldg(&M.tets[e]);
  const int vs[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int a = 1; a < 4; ++a)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      Ds[i][a - 1] = x[3 * vs[a] + i] - x[3 * vs[0] + i];
      dD[i][a - 1] = d[3 * vs[a] + i] - d[3 * vs[0] + i];
    }
}

__device__ __forceinline__ double cubic(double c0, double c1, double c2, double c3, double t) {
  return fma(fma(fma(c3, t, c2), t, c1), t, c0);
}

// smallest t in (0, T] with p(t) <= 0 given p(0) = c0 > 0 (inf if none)
__device__ double smallest_root(double c0, double c1, double c2, double c3, double T) {
  if (!(c0 > 0.0)) return 0.0;
  if (fabs(c1) * T + fabs(c2) * T * T + fabs(c3) * T * T * T < c0) return INFINITY;
  double pts[4];
  int n = 0;
  pts[n++] = 0.0;
  // critical points: 3 c3 t^2 + 2 c2 t + c1 = 0
  const double A = 3.0 * c3, B = 2.0 * c2, C = c1;
  double r1 = -1.0, r2 = -1.0;
  if (A != 0.0) {
    const double disc = B * B - 4.0 * A * C;
    if (disc >= 0.0) {
      const double sq = sqrt(disc);
      const double qq = -0.5 * (B + (B >= 0.0 ? sq : -sq));
      r1 = qq / A;
      r2 = qq != 0.0 ? C / qq : -1.0;
    }
  } else if (B != 0.0) {
    r1 = -C / B;
  }
  if (r1 > r2) { const double tmp = r1; r1 = r2; r2 = tmp; }
  if (r1 > 0.0 && r1 < T) pts[n++] = r1;
  if (r2 > 0.0 && r2 < T) pts[n++] = r2;
  pts[n++] = T;
  for (int s = 0; s + 1 < n; ++s) {
    double a = pts[s], b = pts[s + 1];
    if (cubic(c0, c1, c2, c3, b) <= 0.0) {
      // p(a) > 0 >= p(b), p monotone on [a,b]: bisection to full precision
      for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (a + b);
        if (mid <= a || mid >= b) break;
        if (cubic(c0, c1, c2, c3, mid) > 0.0) a = mid; else b = mid;
      }
      return b;
    }
  }
  return INFINITY;
}

// per tet: inversion filter root; per vertex: CCD time.  min-reduction -> scal[SC_ALPHA_INV/CCD]
__global__ void __launch_bounds__(256) k_filter_inv(LSMesh M, const double *__restrict__ x,
                                                    const double *__restrict__ d, double T,
                                                    double *__restrict__ partial, unsigned int *counter,
                                                    double *__restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  double tmin[1] = {INFINITY};
  if (e < M.nt) {
    double Ds[3][3], dD[3][3], cA[3][3], cB[3][3];
    int4 t;
    edge_mats(M, e, x, d, Ds, dD, t);
    cof3(Ds, cA);
    cof3(dD, cB);
    double c1 = 0.0, c2 = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        c1 = fma(cA[i][j], dD[i][j], c1);
        c2 = fma(Ds[i][j], cB[i][j], c2);
      }
    tmin[0] = smallest_root(det3m(Ds), c1, c2, det3m(dD), T);
  }
  double res[1];
  if (grid_reduce<1, 1>(tmin, partial, counter, res) && threadIdx.x == 0) *out = res[0];
}

__global__ void __launch_bounds__(256) k_filter_ccd(int nv, const double *__restrict__ x,
                                                    const double *__restrict__ d,
                                                    const uint8_t *__restrict__ fixed, double n0, double n1,
                                                    double n2, double off, int on, double *__restrict__ partial,
                                                    unsigned int *counter, double *__restrict__ out) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  double tmin[1] = {INFINITY};
  if (on && v < nv && !fixed[v]) {
    const double vel = n0 * d[3 * v] + n1 * d[3 * v + 1] + n2 * d[3 * v + 2];
    if (vel < 0.0) {
      const double dist = n0 * x[3 * v] + n1 * x[3 * v + 1] + n2 * x[3 * v + 2] - off;
      tmin[0] = dist / (-vel);
    }
  }
  double res[1];
  if (grid_reduce<1, 1>(tmin, partial, counter, res) && threadIdx.x == 0) *out = res[0];
}

// alpha0 = min(1, safety * t_ccd, safety * t_inv); candidates alpha_k = alpha0 * shrink^(k0+k)
__global__ void k_alpha0(double *__restrict__ scal, double safety) {
  const double a = fmin(1.0, fmin(safety * scal[SC_ALPHA_CCD], safety * scal[SC_ALPHA_INV]));
  scal[SC_ALPHA0] = a;
}

__device__ __forceinline__ double psi_val(const double F[3][3], double mu, double lam, bool &bad) {
  const double J = det3m(F);
  if (!(J > 0.0)) bad = true;
  double Ic = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Ic = fma(F[i][j], F[i][j], Ic);
  return 0.5 * mu * (Ic - 3.0) - mu * (J - 1.0) + 0.5 * lam * (J - 1.0) * (J - 1.0);
}

// per tet: dPsi_k = V (Psi(F + alpha_k dF) - Psi(F)); per vertex: inertia and barrier differences.
// out[k] = h^2 (sum dPsi_k + kappa sum db_k) + sum dK_k ; out[K + k] = infeasible count
// owned tets [0, nt_own) and owned vertices [0, nv_own) only; dist: raw partial sums (energy
// differences out[k], infeasible counts out[2K + k]) for the cross-rank sum, then k_ls_finalize
template <int K>
__global__ void __launch_bounds__(256) k_ls_energy(LSMesh M, int nt_own, int nv_own, int dist, const double *__restrict__ x,
                                                   const double *__restrict__ d, const double *__restrict__ xhat,
                                                   const double *__restrict__ mass,
                                                   const uint8_t *__restrict__ fixed, const double *__restrict__ scal,
                                                   int k0, double shrink, double h2, double n0, double n1,
                                                   double n2, double off, double dhat, double kappa, int on,
                                                   double *__restrict__ partial, unsigned int *counter,
                                                   double *__restrict__ out) {
  double acc[2 * K];
#pragma unroll
  for (int k = 0; k < 2 * K; ++k) acc[k] = 0.0;
  double al[K];
  {
    double a = scal[SC_ALPHA0];
    for (int k = 0; k < k0; ++k) a *= shrink;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      al[k] = a;
      a *= shrink;
    }
  }
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = gridDim.x * blockDim.x;
  for (int e = tid; e < nt_own; e += stride) {
    double Ds[3][3], dD[3][3];
    int4 t;
    edge_mats(M, e, x, d, Ds, dD, t);
    double Bm[3][3];
#pragma unroll
    for (int i = 0; i < 9; ++i) Bm[i / 3][i % 3] = __ldg(&M.Bm[(size_t)i * M.nt + e]);
    double F[3][3], dF[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        F[i][j] = Ds[i][0] * Bm[0][j] + Ds[i][1] * Bm[1][j] + Ds[i][2] * Bm[2][j];
        dF[i][j] = dD[i][0] * Bm[0][j] + dD[i][1] * Bm[1][j] + dD[i][2] * Bm[2][j];
      }
    const double V = __ldg(&M.vol[e]), mu = __ldg(&M.mu[e]), lam = __ldg(&M.lam[e]);
    bool bad0 = false;
    const double p0 = psi_val(F, mu, lam, bad0);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double Fk[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) Fk[i][j] = fma(al[k], dF[i][j], F[i][j]);
      bool bad = false;
      const double pk = psi_val(Fk, mu, lam, bad);
      acc[k] += h2 * (V * pk - V * p0);
      if (bad) acc[K + k] += 1.0;
    }
  }
  for (int v = tid; v < nv_own; v += stride) {
    if (fixed[v]) continue;
    const double m = mass[v];
    double rd = 0.0, dd = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double di = d[3 * v + i];
      rd = fma(x[3 * v + i] - xhat[3 * v + i], di, rd);
      dd = fma(di, di, dd);
    }
    double dist0 = 0.0, vel = 0.0, b0 = 0.0;
    if (on) {
      dist0 = n0 * x[3 * v] + n1 * x[3 * v + 1] + n2 * x[3 * v + 2] - off;
      vel = n0 * d[3 * v] + n1 * d[3 * v + 1] + n2 * d[3 * v + 2];
      if (dist0 < dhat) {
        const double t = dist0 - dhat;
        b0 = -t * t * log(dist0 / dhat);
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double a = al[k];
      double dv = 0.5 * m * (2.0 * a * rd + a * a * dd);
      if (on) {
        const double dist1 = dist0 + a * vel;
        if (!(dist1 > 0.0)) acc[K + k] += 1.0;
        double b1 = 0.0;
        if (dist1 < dhat && dist1 > 0.0) {
          const double t = dist1 - dhat;
          b1 = -t * t * log(dist1 / dhat);
        }
        dv += h2 * kappa * (b1 - b0);
      }
      acc[k] += dv;
    }
  }
  double res[2 * K];
  if (grid_reduce<2 * K>(acc, partial, counter, res) && threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      out[k] = dist ? res[k] : (res[K + k] > 0.0 ? INFINITY : res[k]);
      out[K + k] = al[k];
      if (dist) out[2 * K + k] = res[K + k];
    }
  }
}

__global__ void k_ls_finalize(int K, double *__restrict__ out) {
  const int k = threadIdx.x;
  if (k < K && out[2 * K + k] > 0.0) out[k] = INFINITY;
}

__global__ void k_update_x(int n3, double *__restrict__ x, const double *__restrict__ d, double alpha) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n3) x[i] = fma(alpha, d[i], x[i]);
}

void launch_filters(Ctx &c) {
  const double T = 1.0 / c.params.filter_safety;
  k_filter_inv<<<div_up(c.nt, 256), 256, 0, c.stream>>>(lsmesh(c), c.x, c.d, T, c.partial, c.counters + 7,
                                                         c.scal + SC_ALPHA_INV);
  k_filter_ccd<<<div_up(c.nv, 256), 256, 0, c.stream>>>(c.nv, c.x, c.d, c.fixed, c.gn[0], c.gn[1], c.gn[2],
                                                        c.goff, c.has_ground ? 1 : 0, c.partial,
                                                        c.counters + 8, c.scal + SC_ALPHA_CCD);
  dist_min(c, c.scal + SC_ALPHA_CCD, 2);   // SC_ALPHA_CCD, SC_ALPHA_INV
  k_alpha0<<<1, 1, 0, c.stream>>>(c.scal, c.params.filter_safety);
  c.launches += 3;
  MS_CUDA(cudaGetLastError());
}

// evaluates candidates k0 .. k0+K-1 into ls_out[0..K) (energy differences) and ls_out[K..2K) (steps)
void launch_ls_batch(Ctx &c, int k0, int K) {
  const double h2 = c.ah2();   // alpha h^2 (Eq. 2)
  const int grid = std::min(div_up(std::max(c.nt, c.nv), 256), 148 * 8);
#define LS_ARGS                                                                                       \
  lsmesh(c), c.nt_own, c.nv_own, c.dist() ? 1 : 0, c.x, c.d, c.xhat, c.mass, c.fixed, c.scal, k0, c.params.ls_shrink, h2, c.gn[0],      \
      c.gn[1], c.gn[2], c.goff, c.dhat, c.kappa, c.has_ground ? 1 : 0, c.partial, c.counters + 9, c.ls_out
  switch (K) {
    case 1: k_ls_energy<1><<<grid, 256, 0, c.stream>>>(LS_ARGS); break;
    case 2: k_ls_energy<2><<<grid, 256, 0, c.stream>>>(LS_ARGS); break;
    case 4: k_ls_energy<4><<<grid, 256, 0, c.stream>>>(LS_ARGS); break;
    case 8: k_ls_energy<8><<<grid, 256, 0, c.stream>>>(LS_ARGS); break;
    default: MS_REQUIRE(false, MS_ERR_ARG, "ls_batch must be 1, 2, 4 or 8");
  }
#undef LS_ARGS
  c.launches++;
  if (c.dist()) {
    dist_sum(c, c.ls_out, K);
    dist_sum(c, c.ls_out + 2 * K, K);
    k_ls_finalize<<<1, 32, 0, c.stream>>>(K, c.ls_out);
    c.launches++;
  }
  MS_CUDA(cudaGetLastError());
}

void launch_update(Ctx &c, double alpha) {
  const int n3 = 3 * c.nv;
  k_update_x<<<div_up(n3, 256), 256, 0, c.stream>>>(n3, c.x, c.d, alpha);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

}  // namespace msim
