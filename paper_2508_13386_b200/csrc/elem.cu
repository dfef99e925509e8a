// Element kernels: stable Neo-Hookean energy, gradient and PSD-projected 12x12 Hessian.
//
// SURVEY §8(a) rows a2 (element energy + gradient) and a3 (element Hessian + PSD projection).
// PAPER.md §3.1 L169-196 (IP energy, Newton system), L629 ("non-inverting Neo-Hookean");
// readings R1 (Psi = mu/2 (I_C-3) - mu (J-1) + lam/2 (J-1)^2, +inf for J <= 0) and R2
// (eigen-clamp of the 12x12 element Hessian).
//
// B200 design: one thread per tetrahedron, SoA per-tet data
// (coalesced), vertex positions gathered through L1/L2.  The Hessian is built directly in the
// 9-dimensional translation complement: with Q = Q4 kron I3 (Q4 = 1/2 Hadamard rows 2-4,
// orthonormal, orthogonal to (1,1,1,1)) and C = (D_ref Bm)^T Q4,
//     Q^T H_e Q = V [ mu (C^T C) kron I3 + lam g g^T + s HJ(F cof C) ],
// g = vec(cof(F) C), s = lam (J-1) - mu, HJ(A)[(b,j),(b',j')] = eps_{bb'k} eps_{jj'l} A[l][k].
// Because H_e annihilates translations, P+(H_e) = Q P+(Q^T H_e Q) Q^T exactly (pinned in
// tests/test_oracle_fem.py::test_psd_element_reduction_equivalence).  The 9x9 symmetric
// eigenproblem is solved in registers by cyclic Jacobi in the Brent-Luk parallel ordering
// (9 rounds x 4 disjoint rotations per sweep -> 4 independent angle chains for ILP).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "fastmath.cuh"
#include "reduce.cuh"
#include "eig9.cuh"

namespace msim {

struct MeshView {
  int32_t nt;
  const int4 *__restrict__ tets;
  const double *__restrict__ Bm;  // [9][nt]
  const double *__restrict__ vol;
  const double *__restrict__ mu;
  const double *__restrict__ lam;
};

static MeshView mesh_view(const Ctx &c) {
  return MeshView{c.nt, reinterpret_cast<const int4 *>(c.tets.p), c.Bm.p, c.vol.p, c.mu.p, c.lam.p};
}

struct TetKin {
  double F[3][3];
  double Bm[3][3];
  double V, mu, lam;
  int4 t;
};

__device__ __forceinline__ void load_tet_kin(const MeshView &M, const double *__restrict__ x, int e,
                                             TetKin &k) {
  k.t = __ldg(&M.tets[e]);
#pragma unroll
  for (int i = 0; i < 9; ++i) k.Bm[i / 3][i % 3] = __ldg(&M.Bm[(size_t)i * M.nt + e]);
  k.V = __ldg(&M.vol[e]);
  k.mu = __ldg(&M.mu[e]);
  k.lam = __ldg(&M.lam[e]);
  double x0[3], Ds[3][3];
  const int vs[4] = {k.t.x, k.t.y, k.t.z, k.t.w};
#pragma unroll
  for (int i = 0; i < 3; ++i) x0[i] = x[3 * vs[0] + i];
#pragma unroll
  for (int a = 1; a < 4; ++a)
#pragma unroll
    for (int i = 0; i < 3; ++i) Ds[i][a - 1] = x[3 * vs[a] + i] - x0[i];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      k.F[i][j] = Ds[i][0] * k.Bm[0][j] + Ds[i][1] * k.Bm[1][j] + Ds[i][2] * k.Bm[2][j];
}

__device__ __forceinline__ void cofactor(const double F[3][3], double C[3][3]) {
  // columns: c0 = f1 x f2, c1 = f2 x f0, c2 = f0 x f1 (f_k = column k of F)
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int a = (k + 1) % 3, b = (k + 2) % 3;
    C[0][k] = F[1][a] * F[2][b] - F[2][a] * F[1][b];
    C[1][k] = F[2][a] * F[0][b] - F[0][a] * F[2][b];
    C[2][k] = F[0][a] * F[1][b] - F[1][a] * F[0][b];
  }
}

__device__ __forceinline__ double det3(const double F[3][3]) {
  return F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) -
         F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
         F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
}

__device__ __forceinline__ double psi_snh(const double F[3][3], double J, double mu, double lam) {
  double Ic = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Ic += F[i][j] * F[i][j];
  return 0.5 * mu * (Ic - 3.0) - mu * (J - 1.0) + 0.5 * lam * (J - 1.0) * (J - 1.0);
}

// ------------------------------------------------------------------ energy + gradient (a2)
// stage_g[e*12 + 3a + i] = V_e (G_e^T vec P)_{(a,i)}; partial energy sum V_e Psi_e.
// energy and inversion count over the owned tets [0, nt_own) only (each tet is owned by one rank)
__global__ void __launch_bounds__(256) k_elem_grad(MeshView M, int nt_own, const double *__restrict__ x,
                                                   double *__restrict__ stage_g,
                                                   double *__restrict__ partial,
                                                   unsigned int *__restrict__ counter,
                                                   double *__restrict__ out_energy,
                                                   double *__restrict__ infeas,
                                                   double *__restrict__ Ee) {
  double en[2] = {0.0, 0.0};
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < M.nt; e += gridDim.x * blockDim.x) {
    TetKin k;
    load_tet_kin(M, x, e, k);
    const double J = det3(k.F);
    double cof[3][3];
    cofactor(k.F, cof);
    if (!(J > 0.0) && e < nt_own) en[1] = 1.0;
    const double s = k.lam * (J - 1.0) - k.mu;
    double P[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) P[i][j] = k.mu * k.F[i][j] + s * cof[i][j];
    // g_a (a = 1..3) = V * (P Bm^T)[:, a-1]; g_0 = -(g_1 + g_2 + g_3)
    double g[4][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double v = k.V * (P[i][0] * k.Bm[a][0] + P[i][1] * k.Bm[a][1] + P[i][2] * k.Bm[a][2]);
        g[a + 1][i] = v;
        acc += v;
      }
      g[0][i] = -acc;
    }
    double *dst = stage_g + (size_t)e * 12;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int i = 0; i < 3; ++i) dst[3 * a + i] = g[a][i];
    const double psi = psi_snh(k.F, J, k.mu, k.lam);
    if (e < nt_own) en[0] += k.V * psi;
    if (Ee) Ee[e] = (J > 0.0) ? k.V * psi : __longlong_as_double(0x7ff0000000000000ULL);
  }
  double res[2];
  if (grid_reduce<2>(en, partial, counter, res) && threadIdx.x == 0) {
    *out_energy = res[0];
    *infeas = res[1];
  }
}

// ------------------------------------------------------------------ Hessian + PSD (a3)
__host__ __device__ constexpr int sidx(int i, int j) {
  return i <= j ? i * 9 - (i * (i - 1)) / 2 + (j - i) : j * 9 - (j * (j - 1)) / 2 + (i - j);
}
__host__ __device__ constexpr int blk4(int a, int b) {  // a <= b, 10 upper blocks
  return a * 4 - (a * (a - 1)) / 2 + (b - a);
}
// Brent-Luk round-robin for n = 9: round r pairs ((r+k)%9, (r-k+9)%9), k = 1..4
// r < 0 (r = -1 - sh, sh = 0..2): the circle-method pairs (0,7),(1,6),(2,5),(3,4) shifted by sh;
// three such rounds are unrolled and the matrix is then relabelled by i -> i+3 (mod 9), so a
// sweep (3 x 3 rounds) meets every pair once with 3 rounds of code (small I-cache footprint,
// one third of the relabelling moves of a per-round shift).
__host__ __device__ constexpr int rr_pf(int sh, int k) {
  return ((k - 1 + sh) % 9) < ((8 - k + sh) % 9) ? ((k - 1 + sh) % 9) : ((8 - k + sh) % 9);
}
__host__ __device__ constexpr int rr_qf(int sh, int k) {
  return ((k - 1 + sh) % 9) < ((8 - k + sh) % 9) ? ((8 - k + sh) % 9) : ((k - 1 + sh) % 9);
}
__host__ __device__ constexpr int rr_p(int r, int k) {
  return r < 0 ? rr_pf(-1 - r, k) : (((r + k) % 9) < ((r - k + 9) % 9) ? ((r + k) % 9) : ((r - k + 9) % 9));
}
__host__ __device__ constexpr int rr_q(int r, int k) {
  return r < 0 ? rr_qf(-1 - r, k) : (((r + k) % 9) < ((r - k + 9) % 9) ? ((r - k + 9) % 9) : ((r + k) % 9));
}

template <int R>
__device__ __forceinline__ void jacobi_round(double (&a)[45], double (&v)[81]) {
  double c[4], s[4], t[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int p = rr_p(R, k + 1), q = rr_q(R, k + 1);
    const double apq = a[sidx(p, q)];
    const double dd = a[sidx(q, q)] - a[sidx(p, p)];
    // t = sgn(dd) 2 apq / (|dd| + sqrt(dd^2 + 4 apq^2))  (NR 11.1; tan of the Jacobi angle)
    const double r2 = fma(dd, dd, 4.0 * apq * apq);
    const double r = r2 > 1e-290 ? r2 * rsqrt_nr(r2) : 0.0;
    const double den = fabs(dd) + r;
    double tt = den > 0.0 ? (2.0 * apq) * rcp_nr(den) : 0.0;
    tt = dd >= 0.0 ? tt : -tt;
    t[k] = tt;
    c[k] = rsqrt_nr(fma(tt, tt, 1.0));
    s[k] = tt * c[k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int p = rr_p(R, k + 1), q = rr_q(R, k + 1);
    const double apq = a[sidx(p, q)];
    a[sidx(p, p)] = fma(-t[k], apq, a[sidx(p, p)]);
    a[sidx(q, q)] = fma(t[k], apq, a[sidx(q, q)]);
    a[sidx(p, q)] = 0.0;
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      if (r == p || r == q) continue;
      const double arp = a[sidx(r, p)], arq = a[sidx(r, q)];
      a[sidx(r, p)] = fma(c[k], arp, -s[k] * arq);
      a[sidx(r, q)] = fma(s[k], arp, c[k] * arq);
    }
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      const double vp = v[r * 9 + p], vq = v[r * 9 + q];
      v[r * 9 + p] = fma(c[k], vp, -s[k] * vq);
      v[r * 9 + q] = fma(s[k], vp, c[k] * vq);
    }
  }
}

// relabel i -> i+3 (mod 9): orbits of length 3, moved in place with one temporary each
__device__ __forceinline__ void cyclic_relabel3(double (&a)[45], double (&v)[81]) {
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = i; j < 9; ++j) {
      // visit each orbit {(i,j), (i+3,j+3), (i+6,j+6)} once, from its smallest packed index
      const int i1 = (i + 3) % 9, j1 = (j + 3) % 9, i2 = (i + 6) % 9, j2 = (j + 6) % 9;
      const int k0 = sidx(i, j), k1 = sidx(i1, j1), k2 = sidx(i2, j2);
      if (k0 < k1 && k0 < k2) {
        const double t0 = a[k0];
        a[k0] = a[k2];   // new(i,j) = old(i-3,j-3) = old(i+6,j+6)
        a[k2] = a[k1];
        a[k1] = t0;
      }
    }
#pragma unroll
  for (int r = 0; r < 9; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double t0 = v[r * 9 + k];
      v[r * 9 + k] = v[r * 9 + k + 6];
      v[r * 9 + k + 6] = v[r * 9 + k + 3];
      v[r * 9 + k + 3] = t0;
    }
}

__device__ __forceinline__ void jacobi_sweep(double (&a)[45], double (&v)[81]) {
#pragma unroll 1
  for (int rd = 0; rd < 3; ++rd) {
    jacobi_round<-1>(a, v);
    jacobi_round<-2>(a, v);
    jacobi_round<-3>(a, v);
    cyclic_relabel3(a, v);
  }
}

__device__ __forceinline__ double offdiag2(const double (&a)[45]) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = i + 1; j < 9; ++j) s = fma(a[sidx(i, j)], a[sidx(i, j)], s);
  return s;
}

// Builds the reduced 9x9 Hessian (packed symmetric) of one tet.
__device__ __forceinline__ void reduced_hessian(const TetKin &k, double (&a)[45]) {
  const double J = det3(k.F);
  double cofF[3][3];
  cofactor(k.F, cofF);
  const double s = k.lam * (J - 1.0) - k.mu;
  // C = Bm^T R0, R0 = D_ref^T Q4 = [[0,-1,-1],[-1,0,-1],[-1,-1,0]]  ->  C[a][b] = Bm[b][a] - colsum_a
  double C[3][3];
#pragma unroll
  for (int aa = 0; aa < 3; ++aa) {
    const double cs = k.Bm[0][aa] + k.Bm[1][aa] + k.Bm[2][aa];
#pragma unroll
    for (int b = 0; b < 3; ++b) C[aa][b] = k.Bm[b][aa] - cs;
  }
  double K[3][3];
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) K[b][bb] = C[0][b] * C[0][bb] + C[1][b] * C[1][bb] + C[2][b] * C[2][bb];
  double cofC[3][3];
  cofactor(C, cofC);
  double Ft[3][3], gh[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      Ft[i][j] = k.F[i][0] * cofC[0][j] + k.F[i][1] * cofC[1][j] + k.F[i][2] * cofC[2][j];
      gh[i][j] = cofF[i][0] * C[0][j] + cofF[i][1] * C[1][j] + cofF[i][2] * C[2][j];
    }
  const double Vmu = k.V * k.mu, Vlam = k.V * k.lam, Vs = k.V * s;
#pragma unroll
  for (int r = 0; r < 9; ++r)
#pragma unroll
    for (int cc = r; cc < 9; ++cc) {
      const int b = r / 3, j = r % 3, bb = cc / 3, jj = cc % 3;
      double val = Vlam * gh[j][b] * gh[jj][bb];
      if (j == jj) val += Vmu * K[b][bb];
      if (b != bb && j != jj) {
        const int kk = 3 - b - bb, l = 3 - j - jj;
        // eps_{b bb kk} * eps_{j jj l}
        const int s1 = ((bb - b + 3) % 3 == 1) ? 1 : -1;
        const int s2 = ((jj - j + 3) % 3 == 1) ? 1 : -1;
        val += (s1 * s2) * Vs * Ft[l][kk];
      }
      a[sidx(r, cc)] = val;
    }
}

// P+(Q^T H Q) in packed form (45) from the Jacobi result.
__device__ __forceinline__ void eig_clamp(double (&a)[45], double (&p9)[45]) {
  double v[81];
#pragma unroll
  for (int i = 0; i < 81; ++i) v[i] = (i / 9 == i % 9) ? 1.0 : 0.0;
  double fro2 = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = i; j < 9; ++j) fro2 += (i == j ? 1.0 : 2.0) * a[sidx(i, j)] * a[sidx(i, j)];
  // stop when ||offdiag||_F <= 1e-13 ||A||_F: the clamp then differs from the exact P+ by
  // ~1e-13 relative, three orders under the 1e-10 parity tolerance; a tighter test sits in the
  // rounding noise (~1e-15) and only adds sweeps
  const double tol2 = 1e-26 * fro2;
  for (int sweep = 0; sweep < 10; ++sweep) {
    if (2.0 * offdiag2(a) <= tol2) break;
    jacobi_sweep(a, v);
  }
  double lp[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) lp[i] = fmax(a[sidx(i, i)], 0.0);
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = i; j < 9; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int kk = 0; kk < 9; ++kk) acc = fma(lp[kk] * v[i * 9 + kk], v[j * 9 + kk], acc);
      p9[sidx(i, j)] = acc;
    }
}

// 12x12 block (a, a2) entry (i, i2) of Q P9 Q^T, Q4 = 1/2 [[1,1,1],[1,-1,-1],[-1,1,-1],[-1,-1,1]]
__host__ __device__ constexpr int q4s(int a, int b) {  // sign of Q4[a][b]
  return a == 0 ? 1 : (a == b + 1 ? 1 : -1);
}

__device__ __forceinline__ double lift_entry(const double (&p9)[45], int a, int a2, int i, int i2) {
  double acc = 0.0;
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int b2 = 0; b2 < 3; ++b2) {
      const double pv = p9[sidx(3 * b + i, 3 * b2 + i2)];
      acc += (q4s(a, b) * q4s(a2, b2) > 0) ? pv : -pv;
    }
  return 0.25 * acc;
}

// true if M + tau ||M||_F I admits a Cholesky factorisation (packed symmetric 9x9); a is
// overwritten by the factor
__device__ __forceinline__ bool psd_by_cholesky_inplace(double (&l)[45], double tau) {
  double fro2 = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = i; j < 9; ++j) fro2 += (i == j ? 1.0 : 2.0) * l[sidx(i, j)] * l[sidx(i, j)];
  const double shift = tau * fro2 * rsqrt_nr2(fro2 > 0.0 ? fro2 : 1.0);
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    double d = l[sidx(j, j)] + shift;
#pragma unroll
    for (int q = 0; q < j; ++q) d = fma(-l[sidx(j, q)], l[sidx(j, q)], d);
    ok = ok && (d > 0.0);
    const double inv = d > 0.0 ? rsqrt_nr2(d) : 0.0;
    l[sidx(j, j)] = d * inv;
#pragma unroll
    for (int i = j + 1; i < 9; ++i) {
      double s = l[sidx(i, j)];
#pragma unroll
      for (int q = 0; q < j; ++q) s = fma(-l[sidx(i, q)], l[sidx(j, q)], s);
      l[sidx(i, j)] = s * inv;
    }
  }
  return ok;
}

// dst[blk4(a,a2)*kStageB + 3 i + i2] = block (a, a2), a <= a2, of H_e = Q P9 Q^T with
// Q4 = 1/2 [[1,1,1],[1,-1,-1],[-1,1,-1],[-1,-1,1]]: for each (i, i2) the 4x4 block over (A, A2)
// is 1/4 H4 P H4^T, formed with the Hadamard pattern (42 adds)
__device__ __forceinline__ void lift_store(const double (&p9)[45], double *__restrict__ dst) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int i2 = 0; i2 < 3; ++i2) {
      double u[4][3];
#pragma unroll
      for (int b2 = 0; b2 < 3; ++b2) {
        const double P0 = p9[sidx(i, 3 * b2 + i2)], P1 = p9[sidx(3 + i, 3 * b2 + i2)],
                     P2 = p9[sidx(6 + i, 3 * b2 + i2)];
        const double t1 = P1 + P2, t2 = P1 - P2;
        u[0][b2] = P0 + t1;
        u[1][b2] = P0 - t1;
        u[2][b2] = t2 - P0;
        u[3][b2] = -t2 - P0;
      }
#pragma unroll
      for (int A = 0; A < 4; ++A) {
        const double t1 = u[A][1] + u[A][2], t2 = u[A][1] - u[A][2];
        const double w[4] = {u[A][0] + t1, u[A][0] - t1, t2 - u[A][0], -t2 - u[A][0]};
#pragma unroll
        for (int A2 = A; A2 < 4; ++A2) dst[blk4(A, A2) * kStageB + 3 * i + i2] = 0.25 * w[A2];
      }
    }
}

// stage_h[e*kStageH + blk4(a,a2)*kStageB + 3 i + i2] = P+(H_e) block (a, a2), a <= a2 (unscaled by h^2).
// Pass 1 (every tet): reduced Hessian, P+ by e9::psd_project (tridiagonal QL + inverse iteration
// on the negative eigenvalues, eig9.cuh).  A tet with more than kMaxNeg negative eigenvalues (or
// no QL convergence) goes to a work list for pass 2, the cyclic-Jacobi eigen-clamp (the list
// order depends on atomics, the per-tet result does not -> deterministic).
#ifndef MSIM_KMAXNEG
#define MSIM_KMAXNEG 4
#endif
constexpr int kMaxNeg = MSIM_KMAXNEG;

#ifndef MSIM_HESS_THREADS
#define MSIM_HESS_THREADS 128
#endif
constexpr int kHessThreads = MSIM_HESS_THREADS;
constexpr int kHessScratch = 35 + 9 * kMaxNeg;   // doubles per thread (eig9.cuh)

#ifndef MSIM_HESS_MINB
#define MSIM_HESS_MINB 2
#endif
// The projected blocks leave through shared memory: each warp writes its 32 tets' 90 doubles
// (row stride 91 against bank conflicts) and copies them to the contiguous stage_h rows of those
// tets with coalesced stores (a direct per-thread store has a 720-byte stride).
constexpr int kHessStg = kStageH + 1;

__global__ void __launch_bounds__(kHessThreads, MSIM_HESS_MINB) k_elem_hess(MeshView M, const double *__restrict__ x,
                                                            double *__restrict__ stage_h,
                                                            int32_t *__restrict__ work,
                                                            unsigned int *__restrict__ nwork, int force_fallback,
                                                            const int32_t *__restrict__ list, int nlist) {
  extern __shared__ double hsm[];   // eig9 scratch [kHessScratch][kHessThreads] / store staging
  // list (NEXT-2 cubature iterations): thread idx handles tet list[idx] instead of tet idx
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_items = list ? nlist : M.nt;
  const int e = idx < n_items ? (list ? __ldg(&list[idx]) : idx) : M.nt;
  const int lane = threadIdx.x & 31, wbase = threadIdx.x & ~31;
  bool store = false;
  double p9[45];
  if (idx < n_items) {
    TetKin k;
    load_tet_kin(M, x, e, k);
    double a[45];
    reduced_hessian(k, a);
    // already PSD (lambda_min > -1e-12 ||M||_F, Cholesky test): P+ = M to within 1e-11 relative,
    // inside the 1e-10 parity tolerance -- common near rest (free fall), skips the eigensolver
#pragma unroll
    for (int q = 0; q < 45; ++q) p9[q] = a[q];
    if (psd_by_cholesky_inplace(p9, 1e-12)) {
#pragma unroll
      for (int q = 0; q < 45; ++q) p9[q] = a[q];
      store = true;
    } else if (!force_fallback && e9::psd_project<kMaxNeg>(a, p9, hsm + threadIdx.x, kHessThreads) >= 0) {
      store = true;
    } else {
      work[atomicAdd(nwork, 1u)] = e;
    }
  }
  __syncthreads();   // the eig9 scratch is dead: reuse it for the store staging
  double *stg = hsm + (size_t)threadIdx.x * kHessStg;
  if (store) lift_store(p9, stg);
  __syncwarp();
  if (list) {   // scattered tets: each thread copies its own 100-double row
    if (store)
      for (int q = 0; q < kStageH; ++q) stage_h[(size_t)e * kStageH + q] = stg[q];
    return;
  }
  const int e0 = blockIdx.x * blockDim.x + wbase;
  const int ntet = min(32, M.nt - e0);
  double *dst = stage_h + (size_t)e0 * kStageH;
  const double *src = hsm + (size_t)wbase * kHessStg;
  // (tets of the warp that went to the Jacobi list are rewritten by k_elem_hess_eig)
  for (int idx = lane; idx < ntet * kStageH; idx += 32) dst[idx] = src[(idx / kStageH) * kHessStg + idx % kStageH];
}

__global__ void __launch_bounds__(128) k_elem_hess_eig(MeshView M, const double *__restrict__ x,
                                                       double *__restrict__ stage_h,
                                                       const int32_t *__restrict__ work,
                                                       const unsigned int *__restrict__ nwork) {
  const int n = (int)*nwork;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < n; w += gridDim.x * blockDim.x) {
    const int e = work[w];
    TetKin k;
    load_tet_kin(M, x, e, k);
    double a[45], p9[45];
    reduced_hessian(k, a);
    eig_clamp(a, p9);
    lift_store(p9, stage_h + (size_t)e * kStageH);
  }
}

// Expand staged element data to the parity-hook layout (full 12x12 row-major).
__global__ void k_expand_hess(int nt, const double *__restrict__ stage_h, double *__restrict__ He) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nt * 144) return;
  const int e = (int)(idx / 144), rc = (int)(idx % 144), r = rc / 12, cc = rc % 12;
  const int a = r / 3, i = r % 3, a2 = cc / 3, i2 = cc % 3;
  double v;
  if (a <= a2) v = stage_h[(size_t)e * kStageH + blk4(a, a2) * kStageB + 3 * i + i2];
  else v = stage_h[(size_t)e * kStageH + blk4(a2, a) * kStageB + 3 * i2 + i];
  He[idx] = v;
}

// ------------------------------------------------------------------ launchers
void launch_elem_grad_to(Ctx &c, const double *x, double *Ee) {
  const int bs = 256, nb = std::min(div_up(c.nt, bs), 148 * 8);
  k_elem_grad<<<nb, bs, 0, c.stream>>>(mesh_view(c), c.nt_own, x, c.stage_g, c.partial, c.counters + 0,
                                       c.scal + SC_ENERGY_ELEM, c.scal + SC_INFEAS, Ee);
  c.launches++;
  MS_CUDA(cudaGetLastError());
}

void launch_elem_grad(Ctx &c) { launch_elem_grad_to(c, c.x, nullptr); }

constexpr int kHessSmem = sizeof(double) * (kHessScratch > kHessStg ? kHessScratch : kHessStg) * kHessThreads;

// per context, on its device (create_common)
void elem_init_attrs(Ctx &) {
  MS_CUDA(cudaFuncSetAttribute(k_elem_hess, cudaFuncAttributeMaxDynamicSharedMemorySize, kHessSmem));
}

void launch_elem_hess_to(Ctx &c, const double *x) {
  MS_CUDA(cudaMemsetAsync(c.hess_nwork, 0, sizeof(unsigned int), c.stream));
  constexpr int smem = kHessSmem;
  k_elem_hess<<<div_up(c.nt, kHessThreads), kHessThreads, smem, c.stream>>>(
      mesh_view(c), x, c.stage_h, c.hess_work, c.hess_nwork, (c.params.debug_flags & MS_DEBUG_HESS_FALLBACK) ? 1 : 0,
      nullptr, 0);
  k_elem_hess_eig<<<148 * 2, 128, 0, c.stream>>>(mesh_view(c), x, c.stage_h, c.hess_work, c.hess_nwork);
  c.launches += 2;
  static const bool dbg = std::getenv("MSIM_DEBUG_HESS") != nullptr;   // diagnostics only
  if (dbg) {
    unsigned int nw = 0;
    MS_CUDA(cudaMemcpyAsync(&nw, c.hess_nwork, sizeof(nw), cudaMemcpyDeviceToHost, c.stream));
    MS_CUDA(cudaStreamSynchronize(c.stream));
    fprintf(stderr, "[msim] hess: %u of %d tets need the eigen-clamp (%.1f%%)\n", nw, c.nt, 100.0 * nw / c.nt);
  }
  MS_CUDA(cudaGetLastError());
}

void launch_elem_hess(Ctx &c) { launch_elem_hess_to(c, c.x); }

// NEXT-2: the element Hessians of the cubature elements only (iterations without an H_lag refresh)
void launch_elem_hess_list(Ctx &c) {
  MS_CUDA(cudaMemsetAsync(c.hess_nwork, 0, sizeof(unsigned int), c.stream));
  k_elem_hess<<<div_up(std::max(c.n_cub, 1), kHessThreads), kHessThreads, kHessSmem, c.stream>>>(
      mesh_view(c), c.x, c.stage_h, c.hess_work, c.hess_nwork, (c.params.debug_flags & MS_DEBUG_HESS_FALLBACK) ? 1 : 0,
      c.cub_tets, c.n_cub);
  k_elem_hess_eig<<<148 * 2, 128, 0, c.stream>>>(mesh_view(c), c.x, c.stage_h, c.hess_work, c.hess_nwork);
  c.launches += 2;
  MS_CUDA(cudaGetLastError());
}

void launch_eval_elements(Ctx &c, const double *x_dev, double *Ee, double *ge, double *He) {
  launch_elem_grad_to(c, x_dev, Ee);
  if (ge) MS_CUDA(cudaMemcpyAsync(ge, c.stage_g, sizeof(double) * 12 * c.nt, cudaMemcpyDeviceToDevice, c.stream));
  if (He) {
    launch_elem_hess_to(c, x_dev);
    const int64_t n = (int64_t)c.nt * 144;
    k_expand_hess<<<div_up(n, 256), 256, 0, c.stream>>>(c.nt, c.stage_h, He);
    c.launches++;
    MS_CUDA(cudaGetLastError());
  }
}

}  // namespace msim
