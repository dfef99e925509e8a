// P+(M): projection of a symmetric 9 x 9 matrix onto the PSD cone (eigenvalue clamp), the
// element-Hessian step of SURVEY §8(a) a3 (reading R2: P+(H_e) = V max(Lambda, 0) V^T),
// applied to the reduced 9 x 9 form Q^T H_e Q (elem.cu).
//
// Method (B200 design): a per-thread dense eigensolver that does O(n^2) work for
// the eigenvalues and computes eigenvectors only where they are needed:
//   1. Householder tridiagonalisation  M = Q T Q^T          (7 reflectors, in registers)
//   2. implicit QL with Wilkinson shift: eigenvalues of T     (no eigenvectors)
//   3. for every eigenvalue lambda < -thr: inverse iteration on T - lambda I (tridiagonal LU
//      with partial pivoting, 2 steps, re-orthogonalised against the previous vectors)
//   4. P+(M) = Q (T - sum_{lambda<0} lambda z z^T) Q^T  (two-sided reflector application)
// Every loop has a static trip count (data-dependent steps are predicated), so all register
// indices are static on the GPU; the rolled loops are the QL iteration count and the negative
// eigenvalues.  The reflectors and the eigenvectors live in a caller-supplied scratch (shared
// memory on the GPU) to keep the register footprint small.
// The eigenvalue clamp is unique (nearest PSD matrix in Frobenius norm), so this and any other
// accurate eigensolver (the oracle's LAPACK syevd, the Jacobi fall-back in elem.cu) agree to
// rounding: eigenvalues in [-thr, 0) (thr = 1e-14 max|lambda|) are left in place, a change of at
// most thr in the result.
//
// The header is host/device code: tests/test_eig9.py compiles it with g++ and checks it against
// numpy's eigh on random spectra (clusters, zero and repeated eigenvalues) and element Hessians.
#pragma once
#include <math.h>

#if defined(__CUDACC__)
#define E9_HD __host__ __device__ __forceinline__
#else
#define E9_HD inline
#endif

namespace e9 {

E9_HD constexpr int sx(int i, int j) {   // packed symmetric index (row-major upper)
  return i <= j ? i * 9 - (i * (i - 1)) / 2 + (j - i) : j * 9 - (j * (j - 1)) / 2 + (i - j);
}

E9_HD double sqr(double x) { return x * x; }

// reciprocal and reciprocal square root to ~1 ulp: MUFU seed + Newton on the GPU (no IEEE
// slow-path branches), plain division on the host
E9_HD double rcp(double x) {
#if defined(__CUDA_ARCH__)
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
#else
  return 1.0 / x;
#endif
}

E9_HD double rsqrt(double x) {
#if defined(__CUDA_ARCH__)
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double h = 0.5 * x * y;
    y = fma(y, fma(-h, y, 0.5), y);
  }
  return y;
#else
  return 1.0 / sqrt(x);
#endif
}

// status: >= 0 number of clamped eigenvalues; -1 more than KMAX negative eigenvalues or no
// convergence (caller falls back to another eigensolver); out is then undefined.
// scratch: 35 + 9 KMAX doubles at scratch[q * stride] (the reflectors and the eigenvectors of the
// negative eigenvalues; on the GPU a thread-minor slice of shared memory).
// The result is assembled in the tridiagonal basis, P+ = Q (T - sum lam z z^T) Q^T, so M itself
// is not needed after the reduction (M = Q T Q^T to rounding).
template <int KMAX>
E9_HD int psd_project(const double (&M)[45], double (&out)[45], double *scratch, int stride) {
  double *refl = scratch;                 // [28] reflector entries, [7] betas
  double *Zs = scratch + 35 * stride;     // [KMAX][9]
  double t[45];
#pragma unroll
  for (int q = 0; q < 45; ++q) t[q] = M[q];
  // ---------------------------------------------------------------- 1. tridiagonalisation
  // reflector k: H_k = I - beta_k v v^T on indices k+1..8, v_{k+1} = 1, v_i = t[i][k] (i >= k+2)
  double d[9], e[9], beta[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const double x0 = t[sx(k + 1, k)];
    double sig = 0.0;
#pragma unroll
    for (int i = k + 2; i < 9; ++i) sig += sqr(t[sx(i, k)]);
    double b = 0.0;
    e[k] = x0;
    if (sig > 0.0) {
      const double h2 = x0 * x0 + sig;
      const double mu = h2 * rsqrt(h2);
      const double v1 = x0 <= 0.0 ? x0 - mu : -sig * rcp(x0 + mu);
      b = 2.0 * v1 * v1 * rcp(sig + v1 * v1);
      e[k] = mu;
      const double iv = rcp(v1);
#pragma unroll
      for (int i = k + 2; i < 9; ++i) t[sx(i, k)] *= iv;
    }
    beta[k] = b;
    // A22 <- H A22 H: p = b A22 v, w = p - (b/2)(p.v) v, A22 -= v w^T + w v^T
    double v[9], p[9];
#pragma unroll
    for (int i = k + 1; i < 9; ++i) v[i] = i == k + 1 ? 1.0 : t[sx(i, k)];
    double pv = 0.0;
#pragma unroll
    for (int i = k + 1; i < 9; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = k + 1; j < 9; ++j) s = fma(t[sx(i, j)], v[j], s);
      p[i] = b * s;
      pv = fma(p[i], v[i], pv);
    }
    const double K = 0.5 * b * pv;
#pragma unroll
    for (int i = k + 1; i < 9; ++i) p[i] = fma(-K, v[i], p[i]);   // w
#pragma unroll
    for (int i = k + 1; i < 9; ++i)
#pragma unroll
      for (int j = i; j < 9; ++j) t[sx(i, j)] -= fma(v[i], p[j], p[i] * v[j]);
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) d[i] = t[sx(i, i)];
  e[7] = t[sx(8, 7)];
  e[8] = 0.0;
  {
    int q = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
#pragma unroll
      for (int i = k + 2; i < 9; ++i) refl[(q++) * stride] = t[sx(i, k)];
      refl[(28 + k) * stride] = beta[k];
    }
  }
  double d0[9], e0[8];
#pragma unroll
  for (int i = 0; i < 9; ++i) d0[i] = d[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) e0[i] = e[i];

  // ---------------------------------------------------------------- 2. implicit QL (eigenvalues)
  // Numerical Recipes tqli without eigenvectors, 0-based (e[i] couples i and i+1), with the
  // block end m found by a predicated static scan and the sweep i = m-1..l predicated on i < m.
  constexpr double kEps = 2.220446049250313e-16;
  bool conv = true;
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    bool done = false;
#pragma unroll 1
    for (int it = 0; it < 40 && !done; ++it) {
      int m = 8;
#pragma unroll
      for (int i = 7; i >= l; --i)
        if (fabs(e[i]) <= kEps * (fabs(d[i]) + fabs(d[i + 1]))) m = i;
      if (m == l) {
        done = true;
        break;
      }
      double dm = d[8];
#pragma unroll
      for (int i = l; i < 8; ++i)
        if (i == m) dm = d[i];
      double g = (d[l + 1] - d[l]) * rcp(2.0 * e[l]);
      const double g21 = g * g + 1.0;
      double r = g21 * rsqrt(g21);
      g = dm - d[l] + e[l] * rcp(g + (g >= 0.0 ? r : -r));
      double s = 1.0, c = 1.0, p = 0.0;
      bool brk = false;   // NR's underflow exit (r == 0): remaining steps skipped, sweep redone
#pragma unroll
      for (int i = 7; i >= l; --i) {
        if (i < m && !brk) {
          const double f = s * e[i], bb = c * e[i];
          const double h2 = f * f + g * g;
          if (h2 == 0.0) {
            e[i + 1] = 0.0;
            d[i + 1] -= p;
            brk = true;
          } else {
            const double ir = rsqrt(h2);
            e[i + 1] = h2 * ir;
            s = f * ir;
            c = g * ir;
            g = d[i + 1] - p;
            r = (d[i] - g) * s + 2.0 * c * bb;
            p = s * r;
            d[i + 1] = g + p;
            g = c * r - bb;
          }
        }
      }
#pragma unroll
      for (int i = l; i < 9; ++i)
        if (i == m) e[i] = 0.0;
      if (!brk) {
        d[l] -= p;
        e[l] = g;
      }
    }
    conv = conv && done;
  }
  if (!conv) return -1;

  // ---------------------------------------------------------------- 3. negative eigenpairs
  double scale = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) scale = fmax(scale, fabs(d[i]));
  const double thr = 1e-14 * scale;
  int nneg = 0;
#pragma unroll
  for (int i = 0; i < 9; ++i) nneg += d[i] < -thr ? 1 : 0;
  if (nneg > KMAX) return -1;
  // out = T - sum lam z z^T in the tridiagonal basis (nneg = 0: Q T Q^T = M to rounding)
#pragma unroll
  for (int q = 0; q < 45; ++q) out[q] = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) out[sx(i, i)] = d0[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) out[sx(i, i + 1)] = e0[i];
  const double tiny = kEps * scale;
#pragma unroll 1
  for (int found = 0; found < nneg; ++found) {
    double lam = 0.0;   // the found-th negative eigenvalue (static scan)
    {
      int cnt = 0;
#pragma unroll
      for (int i = 0; i < 9; ++i)
        if (d[i] < -thr) {
          if (cnt == found) lam = d[i];
          cnt++;
        }
    }
    // LU with partial pivoting of T0 - lam I (LAPACK dgttrf): rows i, i+1 may swap
    double dd[9], du[8], du2[7], dl[8];
    bool sw[8];
#pragma unroll
    for (int i = 0; i < 9; ++i) dd[i] = d0[i] - lam;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      du[i] = e0[i];
      dl[i] = e0[i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < 7) du2[i] = 0.0;
      sw[i] = fabs(dd[i]) < fabs(dl[i]);
      if (!sw[i]) {
        const double fact = dd[i] != 0.0 ? dl[i] * rcp(dd[i]) : 0.0;
        dl[i] = fact;
        dd[i + 1] -= fact * du[i];
      } else {
        const double fact = dd[i] * rcp(dl[i]);
        dd[i] = dl[i];
        dl[i] = fact;
        const double temp = du[i];
        du[i] = dd[i + 1];
        dd[i + 1] = temp - fact * dd[i + 1];
        if (i < 7) {
          du2[i] = du[i + 1];
          du[i + 1] = -fact * du[i + 1];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      if (fabs(dd[i]) < tiny) dd[i] = dd[i] < 0.0 ? -tiny : tiny;
      dd[i] = rcp(dd[i]);   // reciprocal pivots from here on
    }
    double x[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) x[i] = 1.0 + 0.0625 * i;   // generic start vector
#pragma unroll
    for (int iter = 0; iter < 2; ++iter) {
      // orthogonalise against the vectors already found (clusters of negative eigenvalues)
#pragma unroll 1
      for (int q = 0; q < found; ++q) {
        double z[9], h = 0.0;
#pragma unroll
        for (int i = 0; i < 9; ++i) {
          z[i] = Zs[(9 * q + i) * stride];
          h = fma(z[i], x[i], h);
        }
#pragma unroll
        for (int i = 0; i < 9; ++i) x[i] = fma(-h, z[i], x[i]);
      }
      // solve (T0 - lam I) y = x: forward (row swaps + multipliers), then back substitution
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (!sw[i]) {
          x[i + 1] -= dl[i] * x[i];
        } else {
          const double temp = x[i];
          x[i] = x[i + 1];
          x[i + 1] = temp - dl[i] * x[i];
        }
      }
      x[8] *= dd[8];
      x[7] = (x[7] - du[7] * x[8]) * dd[7];
#pragma unroll
      for (int i = 6; i >= 0; --i) x[i] = (x[i] - du[i] * x[i + 1] - du2[i] * x[i + 2]) * dd[i];
      double nrm = 0.0;
#pragma unroll
      for (int i = 0; i < 9; ++i) nrm = fma(x[i], x[i], nrm);
      const double inv = rsqrt(nrm);
#pragma unroll
      for (int i = 0; i < 9; ++i) x[i] *= inv;
    }
    // final re-orthogonalisation + normalisation
#pragma unroll 1
    for (int q = 0; q < found; ++q) {
      double z[9], h = 0.0;
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        z[i] = Zs[(9 * q + i) * stride];
        h = fma(z[i], x[i], h);
      }
#pragma unroll
      for (int i = 0; i < 9; ++i) x[i] = fma(-h, z[i], x[i]);
    }
    {
      double nrm = 0.0;
#pragma unroll
      for (int i = 0; i < 9; ++i) nrm = fma(x[i], x[i], nrm);
      const double inv = rsqrt(nrm);
#pragma unroll
      for (int i = 0; i < 9; ++i) x[i] *= inv;
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) Zs[(9 * found + i) * stride] = x[i];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const double li = lam * x[i];
#pragma unroll
      for (int j = i; j < 9; ++j) out[sx(i, j)] = fma(-li, x[j], out[sx(i, j)]);
    }
  }
  // ---------------------------------------------------------------- 4. out <- Q out Q^T
  // Q = H_0 ... H_6: apply H_6 first; H X H = X - v w^T - w v^T, p = beta X v,
  // w = p - (beta/2)(p.v) v
#pragma unroll
  for (int k = 6; k >= 0; --k) {
    double v[9];
    {
      int q = 0;
#pragma unroll
      for (int kk = 0; kk < k; ++kk) q += 7 - kk;
#pragma unroll
      for (int i = 0; i < 9; ++i) v[i] = i < k + 1 ? 0.0 : (i == k + 1 ? 1.0 : refl[(q + i - k - 2) * stride]);
    }
    const double b = refl[(28 + k) * stride];
    double p[9], pv = 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      double s2 = 0.0;
#pragma unroll
      for (int j = k + 1; j < 9; ++j) s2 = fma(out[sx(i, j)], v[j], s2);
      p[i] = b * s2;
      if (i > k) pv = fma(p[i], v[i], pv);
    }
    const double K = 0.5 * b * pv;
#pragma unroll
    for (int i = 0; i < 9; ++i)
      if (i > k) p[i] = fma(-K, v[i], p[i]);
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int j = i; j < 9; ++j)
        if (j > k) out[sx(i, j)] -= (i > k ? v[i] * p[j] : 0.0) + p[i] * v[j];
  }
  return nneg;
}

}  // namespace e9
