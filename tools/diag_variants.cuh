// Variants of the diagonal-tile step D(k) (csrc/chol_diag.cuh) for tools/bench_diag.cu.
//   V2: as chol_diag.cuh, but the reciprocal of the next pivot is formed once, by the thread
//       owning it, and published with the pivot row (the other threads load it)
//   V3: 2 x 2 block pivots (32 steps): rows i > b of the pair (a, b) = (2J, 2J+1) are updated by
//       (f_a, f_b) = (S_ia, S_ib) P^-1 with P the pair's 2 x 2 Schur block; at the end
//       L^-1 = C^-1 N with C the Cholesky factor of each 2 x 2 block
//   V4: V3 with P^-1 formed once by the thread owning the block and published with the rows
#pragma once

template <bool PUB>
__device__ __noinline__ void diag_v2(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                     int *__restrict__ flag, double *sm) {
  double *R = sm, *Li = sm + TB * LD;
  const int t = threadIdx.x, i0 = 4 * (t >> 4), c0 = 4 * (t & 15);
  double M[4][4];
  const size_t okk = tile_off(k, k, nSp);
#pragma unroll
  for (int ri = 0; ri < 4; ++ri)
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) {
      const int i = i0 + ri, c = c0 + ci;
      M[ri][ci] = c >= i ? __ldcg(&L[okk + (size_t)i * nSp + c]) : 0.0;
    }
  __syncthreads();
  if (i0 == 0) {
    *reinterpret_cast<double2 *>(&R[c0]) = make_double2(M[0][0], M[0][1]);
    *reinterpret_cast<double2 *>(&R[c0 + 2]) = make_double2(M[0][2], M[0][3]);
    if (t == 0) R[TB] = rcp_nr(M[0][0] > 0.0 ? M[0][0] : 1.0);
  }
  __syncthreads();
  for (int j = 0; j < TB - 1; ++j) {
    const double *u = R + j * LD;
    const double2 r01 = *reinterpret_cast<const double2 *>(&u[i0]);
    const double2 r23 = *reinterpret_cast<const double2 *>(&u[i0 + 2]);
    const double2 c01 = *reinterpret_cast<const double2 *>(&u[c0]);
    const double2 c23 = *reinterpret_cast<const double2 *>(&u[c0 + 2]);
    double q;
    if (PUB) q = u[TB];
    else { const double p = u[j]; q = rcp_nr(p > 0.0 ? p : 1.0); }
    const double ur[4] = {r01.x, r01.y, r23.x, r23.y};
    const double uc[4] = {c01.x, c01.y, c23.x, c23.y};
    const int jn = j + 1;
#pragma unroll
    for (int ri = 0; ri < 4; ++ri) {
      const int i = i0 + ri;
      const double f = i > j ? ur[ri] * q : 0.0;
#pragma unroll
      for (int ci = 0; ci < 4; ++ci) {
        const int c = c0 + ci;
        const double w = (c >= i || c < j) ? uc[ci] : (c == j ? 1.0 : 0.0);
        M[ri][ci] = fma(-f, w, M[ri][ci]);
      }
    }
    if (i0 == (jn & ~3)) {
      const int rs = jn & 3;
      double pv[4];
#pragma unroll
      for (int ci = 0; ci < 4; ++ci)
        pv[ci] = rs == 0 ? M[0][ci] : rs == 1 ? M[1][ci] : rs == 2 ? M[2][ci] : M[3][ci];
      *reinterpret_cast<double2 *>(&R[jn * LD + c0]) = make_double2(pv[0], pv[1]);
      *reinterpret_cast<double2 *>(&R[jn * LD + c0 + 2]) = make_double2(pv[2], pv[3]);
      if (PUB && c0 == i0) {
        const double p = rs == 0 ? pv[0] : rs == 1 ? pv[1] : rs == 2 ? pv[2] : pv[3];
        R[jn * LD + TB] = rcp_nr(p > 0.0 ? p : 1.0);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int ri = 0; ri < 4; ++ri) {
    const int i = i0 + ri;
    const double p = R[i * LD + i];
    const double r = rsqrt_nr(p > 0.0 ? p : 1.0);
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) {
      const int c = c0 + ci;
      Li[i * LD + c] = c < i ? r * M[ri][ci] : (c == i ? r : 0.0);
    }
  }
  if (t < TB && flag && !(R[t * LD + t] > 0.0)) *flag = 1;
  __syncthreads();
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
}

// 2 x 2 pivots.  Pad columns of a published row pair (a, b): R[a][TB..TB+2] = P^-1 entries
// (g_aa, g_ab, g_bb) when PUB.
template <bool PUB>
__device__ __noinline__ void diag_v3(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                     int *__restrict__ flag, double *sm) {
  double *R = sm, *Li = sm + TB * LD;
  const int t = threadIdx.x, i0 = 4 * (t >> 4), c0 = 4 * (t & 15);
  double M[4][4];
  const size_t okk = tile_off(k, k, nSp);
#pragma unroll
  for (int ri = 0; ri < 4; ++ri)
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) {
      const int i = i0 + ri, c = c0 + ci;
      M[ri][ci] = c >= i ? __ldcg(&L[okk + (size_t)i * nSp + c]) : 0.0;
    }
  __syncthreads();
  auto pinv = [](double paa, double pab, double pbb, double &gaa, double &gab, double &gbb) {
    const double det = fma(paa, pbb, -pab * pab);
    const double id = rcp_nr(det > 0.0 && paa > 0.0 ? det : 1.0);
    gaa = pbb * id;
    gab = -pab * id;
    gbb = paa * id;
  };
  if (i0 == 0) {
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      *reinterpret_cast<double2 *>(&R[rr * LD + c0]) = make_double2(M[rr][0], M[rr][1]);
      *reinterpret_cast<double2 *>(&R[rr * LD + c0 + 2]) = make_double2(M[rr][2], M[rr][3]);
    }
    if (PUB && t == 0) pinv(M[0][0], M[0][1], M[1][1], R[TB], R[TB + 1], R[TB + 2]);
  }
  __syncthreads();
  for (int J = 0; J < TB / 2 - 1; ++J) {
    const int a = 2 * J, b = a + 1;
    const double *ua = R + a * LD, *ub = R + b * LD;
    double gaa, gab, gbb;
    if (PUB) {
      gaa = ua[TB];
      gab = ua[TB + 1];
      gbb = ua[TB + 2];
    } else {
      pinv(ua[a], ua[b], ub[b], gaa, gab, gbb);
    }
    const double2 ra01 = *reinterpret_cast<const double2 *>(&ua[i0]);
    const double2 ra23 = *reinterpret_cast<const double2 *>(&ua[i0 + 2]);
    const double2 rb01 = *reinterpret_cast<const double2 *>(&ub[i0]);
    const double2 rb23 = *reinterpret_cast<const double2 *>(&ub[i0 + 2]);
    const double2 ca01 = *reinterpret_cast<const double2 *>(&ua[c0]);
    const double2 ca23 = *reinterpret_cast<const double2 *>(&ua[c0 + 2]);
    const double2 cb01 = *reinterpret_cast<const double2 *>(&ub[c0]);
    const double2 cb23 = *reinterpret_cast<const double2 *>(&ub[c0 + 2]);
    const double sa[4] = {ra01.x, ra01.y, ra23.x, ra23.y}, sb[4] = {rb01.x, rb01.y, rb23.x, rb23.y};
    const double wa[4] = {ca01.x, ca01.y, ca23.x, ca23.y}, wb[4] = {cb01.x, cb01.y, cb23.x, cb23.y};
#pragma unroll
    for (int ri = 0; ri < 4; ++ri) {
      const int i = i0 + ri;
      const bool act = i > b;
      const double fa = act ? fma(sa[ri], gaa, sb[ri] * gab) : 0.0;
      const double fb = act ? fma(sa[ri], gab, sb[ri] * gbb) : 0.0;
#pragma unroll
      for (int ci = 0; ci < 4; ++ci) {
        const int c = c0 + ci;
        const bool use = c >= i || c < a;
        const double xa = use ? wa[ci] : (c == a ? 1.0 : 0.0);
        const double xb = use ? wb[ci] : (c == b ? 1.0 : 0.0);
        M[ri][ci] = fma(-fa, xa, fma(-fb, xb, M[ri][ci]));
      }
    }
    const int an = a + 2;
    if (i0 == (an & ~3)) {   // publish rows an, an + 1 (an & 3 is 0 or 2)
      const bool hi = (an & 3) == 2;
      double pa[4], pb[4];
#pragma unroll
      for (int ci = 0; ci < 4; ++ci) {
        pa[ci] = hi ? M[2][ci] : M[0][ci];
        pb[ci] = hi ? M[3][ci] : M[1][ci];
      }
      *reinterpret_cast<double2 *>(&R[an * LD + c0]) = make_double2(pa[0], pa[1]);
      *reinterpret_cast<double2 *>(&R[an * LD + c0 + 2]) = make_double2(pa[2], pa[3]);
      *reinterpret_cast<double2 *>(&R[(an + 1) * LD + c0]) = make_double2(pb[0], pb[1]);
      *reinterpret_cast<double2 *>(&R[(an + 1) * LD + c0 + 2]) = make_double2(pb[2], pb[3]);
      if (PUB && c0 == i0) {
        const double paa = hi ? pa[2] : pa[0], pab = hi ? pa[3] : pa[1], pbb = hi ? pb[3] : pb[1];
        pinv(paa, pab, pbb, R[an * LD + TB], R[an * LD + TB + 1], R[an * LD + TB + 2]);
      }
    }
    __syncthreads();
  }
  // L^-1 = C^-1 N per 2 x 2 block: row a = r_a N_a, row b = r_b (N_b - (p_ab / p_aa) N_a)
#pragma unroll
  for (int rp = 0; rp < 2; ++rp) {
    const int a = i0 + 2 * rp, b = a + 1;
    const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
    const bool ok = paa > 0.0;
    const double ra = rsqrt_nr(ok ? paa : 1.0);
    const double m = ok ? pab * ra * ra : 0.0;
    const double s = fma(-m, pab, pbb);
    const double rb = rsqrt_nr(s > 0.0 ? s : 1.0);
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) {
      const int c = c0 + ci;
      const double na = c < a ? M[2 * rp][ci] : (c == a ? 1.0 : 0.0);
      const double nb = c < a ? M[2 * rp + 1][ci] : (c == b ? 1.0 : 0.0);
      Li[a * LD + c] = ra * na;
      Li[b * LD + c] = rb * fma(-m, na, nb);
    }
    if (c0 == i0 && flag && !(ok && s > 0.0)) *flag = 1;
  }
  __syncthreads();
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
}

// V5: scalar pivots with the j loop unrolled by 4 (row-in-block of the published row static) and
// block-type specialised threads: warps 0-2 hold strictly-upper blocks, 4-6 strictly-lower ones,
// warps 3 / 7 the rest of those plus the 16 diagonal blocks, so the per-entry choice between
// the Schur coefficient u_c and the lower coefficient (N_jc, 1, 0) is made per block, not per entry.
namespace v5 {
enum { UP = 0, LO = 1, DG = 2 };
__device__ __forceinline__ void block_of(int t, int &a, int &b, int &type) {
  if (t < 120 || (t >= 128 && t < 248)) {
    const bool up = t < 120;
    int u = up ? t : t - 128;
    a = 0;
    for (int r = 0; r < 16; ++r) {
      const int cnt = up ? 15 - r : r;
      if (u < cnt) { a = r; break; }
      u -= cnt;
    }
    b = up ? a + 1 + u : u;
    type = up ? UP : LO;
  } else {
    a = b = t < 128 ? t - 120 : t - 248 + 8;
    type = DG;
  }
}

template <int S>
__device__ __forceinline__ void step(double (&M)[4][4], int type, int a, int b, int J, const double *R, double *Rw) {
  const int j = 4 * J + S;
  const double *u = R + j * LD;
  const double2 r01 = *reinterpret_cast<const double2 *>(&u[4 * a]);
  const double2 r23 = *reinterpret_cast<const double2 *>(&u[4 * a + 2]);
  const double2 c01 = *reinterpret_cast<const double2 *>(&u[4 * b]);
  const double2 c23 = *reinterpret_cast<const double2 *>(&u[4 * b + 2]);
  const double p = u[j];
  const double q = rcp_nr(p > 0.0 ? p : 1.0);
  const double ur[4] = {r01.x, r01.y, r23.x, r23.y};
  const double uc[4] = {c01.x, c01.y, c23.x, c23.y};
  double f[4];
#pragma unroll
  for (int ri = 0; ri < 4; ++ri) f[ri] = (a > J || (a == J && ri > S)) ? ur[ri] * q : 0.0;
  // lower coefficient of column c = 4 b + ci: N_jc (c < j), 1 (c = j), 0 (c > j)
  double wl[4];
#pragma unroll
  for (int ci = 0; ci < 4; ++ci)
    wl[ci] = b < J ? uc[ci] : (b == J ? (ci < S ? uc[ci] : (ci == S ? 1.0 : 0.0)) : 0.0);
  if (type == UP) {
#pragma unroll
    for (int ri = 0; ri < 4; ++ri)
#pragma unroll
      for (int ci = 0; ci < 4; ++ci) M[ri][ci] = fma(-f[ri], uc[ci], M[ri][ci]);
  } else if (type == LO) {
#pragma unroll
    for (int ri = 0; ri < 4; ++ri)
#pragma unroll
      for (int ci = 0; ci < 4; ++ci) M[ri][ci] = fma(-f[ri], wl[ci], M[ri][ci]);
  } else {
#pragma unroll
    for (int ri = 0; ri < 4; ++ri)
#pragma unroll
      for (int ci = 0; ci < 4; ++ci) M[ri][ci] = fma(-f[ri], ci >= ri ? uc[ci] : wl[ci], M[ri][ci]);
  }
  // publish row j + 1 = 4 J + S + 1: row-in-block (S + 1) & 3 of row block J + (S == 3)
  constexpr int RS = (S + 1) & 3;
  if (a == J + (S == 3 ? 1 : 0)) {
    double *dst = Rw + (j + 1) * LD + 4 * b;
    *reinterpret_cast<double2 *>(dst) = make_double2(M[RS][0], M[RS][1]);
    *reinterpret_cast<double2 *>(dst + 2) = make_double2(M[RS][2], M[RS][3]);
  }
  __syncthreads();
}
}  // namespace v5

__device__ __noinline__ void diag_v5(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                     int *__restrict__ flag, double *sm) {
  double *R = sm, *Li = sm + TB * LD;
  const int t = threadIdx.x;
  int a, b, type;
  v5::block_of(t, a, b, type);
  const int i0 = 4 * a, c0 = 4 * b;
  double M[4][4];
  const size_t okk = tile_off(k, k, nSp);
#pragma unroll
  for (int ri = 0; ri < 4; ++ri)
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) {
      const int i = i0 + ri, c = c0 + ci;
      M[ri][ci] = c >= i ? __ldcg(&L[okk + (size_t)i * nSp + c]) : 0.0;
    }
  __syncthreads();
  if (a == 0) {
    *reinterpret_cast<double2 *>(&R[c0]) = make_double2(M[0][0], M[0][1]);
    *reinterpret_cast<double2 *>(&R[c0 + 2]) = make_double2(M[0][2], M[0][3]);
  }
  __syncthreads();
  for (int J = 0; J < 16; ++J) {
    v5::step<0>(M, type, a, b, J, R, R);
    v5::step<1>(M, type, a, b, J, R, R);
    v5::step<2>(M, type, a, b, J, R, R);
    if (J < 15) v5::step<3>(M, type, a, b, J, R, R);
  }
#pragma unroll
  for (int ri = 0; ri < 4; ++ri) {
    const int i = i0 + ri;
    const double p = R[i * LD + i];
    const double r = rsqrt_nr(p > 0.0 ? p : 1.0);
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) {
      const int c = c0 + ci;
      Li[i * LD + c] = c < i ? r * M[ri][ci] : (c == i ? r : 0.0);
    }
  }
  if (t < TB && flag && !(R[t * LD + t] > 0.0)) *flag = 1;
  __syncthreads();
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
}

// V6: V3's 2 x 2 pivots with V5's unrolling and block-type specialisation.
namespace v6 {
template <int S>
__device__ __forceinline__ void step(double (&M)[4][4], int type, int a, int b, int J, double *R) {
  const int ja = 4 * J + 2 * S, jb = ja + 1;
  const double *ua = R + ja * LD, *ub = R + jb * LD;
  const double paa = ua[ja], pab = ua[jb], pbb = ub[jb];
  const double det = fma(paa, pbb, -pab * pab);
  const double id = rcp_nr(det > 0.0 && paa > 0.0 ? det : 1.0);
  const double gaa = pbb * id, gab = -pab * id, gbb = paa * id;
  const double2 ra01 = *reinterpret_cast<const double2 *>(&ua[4 * a]);
  const double2 ra23 = *reinterpret_cast<const double2 *>(&ua[4 * a + 2]);
  const double2 rb01 = *reinterpret_cast<const double2 *>(&ub[4 * a]);
  const double2 rb23 = *reinterpret_cast<const double2 *>(&ub[4 * a + 2]);
  const double2 ca01 = *reinterpret_cast<const double2 *>(&ua[4 * b]);
  const double2 ca23 = *reinterpret_cast<const double2 *>(&ua[4 * b + 2]);
  const double2 cb01 = *reinterpret_cast<const double2 *>(&ub[4 * b]);
  const double2 cb23 = *reinterpret_cast<const double2 *>(&ub[4 * b + 2]);
  const double sa[4] = {ra01.x, ra01.y, ra23.x, ra23.y}, sb[4] = {rb01.x, rb01.y, rb23.x, rb23.y};
  const double wa[4] = {ca01.x, ca01.y, ca23.x, ca23.y}, wb[4] = {cb01.x, cb01.y, cb23.x, cb23.y};
  double fa[4], fb[4];
#pragma unroll
  for (int ri = 0; ri < 4; ++ri) {
    const bool act = a > J || (a == J && ri > 2 * S + 1);
    fa[ri] = act ? fma(sa[ri], gaa, sb[ri] * gab) : 0.0;
    fb[ri] = act ? fma(sa[ri], gab, sb[ri] * gbb) : 0.0;
  }
  double la[4], lb[4];   // lower coefficients of column 4 b + ci
#pragma unroll
  for (int ci = 0; ci < 4; ++ci) {
    if (ci < 2 * S) {
      la[ci] = b <= J ? wa[ci] : 0.0;
      lb[ci] = b <= J ? wb[ci] : 0.0;
    } else if (ci == 2 * S) {
      la[ci] = b < J ? wa[ci] : (b == J ? 1.0 : 0.0);
      lb[ci] = b < J ? wb[ci] : 0.0;
    } else if (ci == 2 * S + 1) {
      la[ci] = b < J ? wa[ci] : 0.0;
      lb[ci] = b < J ? wb[ci] : (b == J ? 1.0 : 0.0);
    } else {
      la[ci] = b < J ? wa[ci] : 0.0;
      lb[ci] = b < J ? wb[ci] : 0.0;
    }
  }
  if (type == v5::UP) {
#pragma unroll
    for (int ri = 0; ri < 4; ++ri)
#pragma unroll
      for (int ci = 0; ci < 4; ++ci) M[ri][ci] = fma(-fa[ri], wa[ci], fma(-fb[ri], wb[ci], M[ri][ci]));
  } else if (type == v5::LO) {
#pragma unroll
    for (int ri = 0; ri < 4; ++ri)
#pragma unroll
      for (int ci = 0; ci < 4; ++ci) M[ri][ci] = fma(-fa[ri], la[ci], fma(-fb[ri], lb[ci], M[ri][ci]));
  } else {
#pragma unroll
    for (int ri = 0; ri < 4; ++ri)
#pragma unroll
      for (int ci = 0; ci < 4; ++ci)
        M[ri][ci] = fma(-fa[ri], ci >= ri ? wa[ci] : la[ci], fma(-fb[ri], ci >= ri ? wb[ci] : lb[ci], M[ri][ci]));
  }
  // publish rows ja + 2, ja + 3: rows 2, 3 of block J (S = 0) or rows 0, 1 of block J + 1 (S = 1)
  constexpr int RA = S == 0 ? 2 : 0;
  if (a == J + S) {
    double *d0 = R + (ja + 2) * LD + 4 * b, *d1 = d0 + LD;
    *reinterpret_cast<double2 *>(d0) = make_double2(M[RA][0], M[RA][1]);
    *reinterpret_cast<double2 *>(d0 + 2) = make_double2(M[RA][2], M[RA][3]);
    *reinterpret_cast<double2 *>(d1) = make_double2(M[RA + 1][0], M[RA + 1][1]);
    *reinterpret_cast<double2 *>(d1 + 2) = make_double2(M[RA + 1][2], M[RA + 1][3]);
  }
  __syncthreads();
}
}  // namespace v6

__device__ __noinline__ void diag_v6(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                     int *__restrict__ flag, double *sm) {
  double *R = sm, *Li = sm + TB * LD;
  const int t = threadIdx.x;
  int a, b, type;
  v5::block_of(t, a, b, type);
  const int i0 = 4 * a, c0 = 4 * b;
  double M[4][4];
  const size_t okk = tile_off(k, k, nSp);
#pragma unroll
  for (int ri = 0; ri < 4; ++ri)
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) {
      const int i = i0 + ri, c = c0 + ci;
      M[ri][ci] = c >= i ? __ldcg(&L[okk + (size_t)i * nSp + c]) : 0.0;
    }
  __syncthreads();
  if (a == 0) {
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      *reinterpret_cast<double2 *>(&R[rr * LD + c0]) = make_double2(M[rr][0], M[rr][1]);
      *reinterpret_cast<double2 *>(&R[rr * LD + c0 + 2]) = make_double2(M[rr][2], M[rr][3]);
    }
  }
  __syncthreads();
  for (int J = 0; J < 16; ++J) {
    v6::step<0>(M, type, a, b, J, R);
    if (J < 15) v6::step<1>(M, type, a, b, J, R);
  }
#pragma unroll
  for (int rp = 0; rp < 2; ++rp) {
    const int ra_ = i0 + 2 * rp, rb_ = ra_ + 1;
    const double paa = R[ra_ * LD + ra_], pab = R[ra_ * LD + rb_], pbb = R[rb_ * LD + rb_];
    const bool ok = paa > 0.0;
    const double r1 = rsqrt_nr(ok ? paa : 1.0);
    const double m = ok ? pab * r1 * r1 : 0.0;
    const double s = fma(-m, pab, pbb);
    const double r2 = rsqrt_nr(s > 0.0 ? s : 1.0);
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) {
      const int c = c0 + ci;
      const double na = c < ra_ ? M[2 * rp][ci] : (c == ra_ ? 1.0 : 0.0);
      const double nb = c < ra_ ? M[2 * rp + 1][ci] : (c == rb_ ? 1.0 : 0.0);
      Li[ra_ * LD + c] = r1 * na;
      Li[rb_ * LD + c] = r2 * fma(-m, na, nb);
    }
    if (c0 == i0 && flag && !(ok && s > 0.0)) *flag = 1;
  }
  __syncthreads();
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
}

// V7<MODE>: timing dissection of the V1 loop (results wrong for MODE < 3):
//   0 = barrier + publish only, 1 = + pivot-row loads, 2 = + reciprocal, 3 = full step
template <int MODE>
__device__ __noinline__ void diag_v7(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                     int *__restrict__ flag, double *sm) {
  double *R = sm, *Li = sm + TB * LD;
  const int t = threadIdx.x, i0 = 4 * (t >> 4), c0 = 4 * (t & 15);
  double M[4][4];
  const size_t okk = tile_off(k, k, nSp);
#pragma unroll
  for (int ri = 0; ri < 4; ++ri)
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) {
      const int i = i0 + ri, c = c0 + ci;
      M[ri][ci] = c >= i ? __ldcg(&L[okk + (size_t)i * nSp + c]) : 0.0;
    }
  __syncthreads();
  if (i0 == 0) {
    *reinterpret_cast<double2 *>(&R[c0]) = make_double2(M[0][0], M[0][1]);
    *reinterpret_cast<double2 *>(&R[c0 + 2]) = make_double2(M[0][2], M[0][3]);
  }
  __syncthreads();
  long long t0 = clock64();
  double acc = 0.0;
  for (int j = 0; j < TB - 1; ++j) {
    const double *u = R + j * LD;
    double ur[4] = {0, 0, 0, 0}, uc[4] = {0, 0, 0, 0}, q = 1.0;
    if (MODE >= 1) {
      const double2 r01 = *reinterpret_cast<const double2 *>(&u[i0]);
      const double2 r23 = *reinterpret_cast<const double2 *>(&u[i0 + 2]);
      const double2 c01 = *reinterpret_cast<const double2 *>(&u[c0]);
      const double2 c23 = *reinterpret_cast<const double2 *>(&u[c0 + 2]);
      ur[0] = r01.x; ur[1] = r01.y; ur[2] = r23.x; ur[3] = r23.y;
      uc[0] = c01.x; uc[1] = c01.y; uc[2] = c23.x; uc[3] = c23.y;
    }
    if (MODE >= 2) {
      const double p = u[j];
      q = rcp_nr(p > 0.0 ? p : 1.0);
    }
    const int jn = j + 1;
    if (MODE >= 3) {
#pragma unroll
      for (int ri = 0; ri < 4; ++ri) {
        const int i = i0 + ri;
        const double f = i > j ? ur[ri] * q : 0.0;
#pragma unroll
        for (int ci = 0; ci < 4; ++ci) {
          const int c = c0 + ci;
          const double w = (c >= i || c < j) ? uc[ci] : (c == j ? 1.0 : 0.0);
          M[ri][ci] = fma(-f, w, M[ri][ci]);
        }
      }
    } else {
      acc += ur[0] + uc[3] * q;
    }
    if (i0 == (jn & ~3)) {
      const int rs = jn & 3;
      double pv[4];
#pragma unroll
      for (int ci = 0; ci < 4; ++ci)
        pv[ci] = rs == 0 ? M[0][ci] : rs == 1 ? M[1][ci] : rs == 2 ? M[2][ci] : M[3][ci];
      *reinterpret_cast<double2 *>(&R[jn * LD + c0]) = make_double2(pv[0] + acc, pv[1]);
      *reinterpret_cast<double2 *>(&R[jn * LD + c0 + 2]) = make_double2(pv[2], pv[3]);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (t == 0 && blockIdx.x == 0) printf("  V7<%d>: loop %lld cycles (%.0f per step)\n", MODE, t1 - t0, (t1 - t0) / 63.0);
#pragma unroll
  for (int ri = 0; ri < 4; ++ri)
#pragma unroll
    for (int ci = 0; ci < 4; ++ci) Li[(i0 + ri) * LD + c0 + ci] = M[ri][ci];
  __syncthreads();
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
}

// V8: panels of 8 pivots.  Warp w owns rows 8w..8w+7 in the m8n8k4 accumulator layout (lane l:
// row 8w + l/4, columns 8t + 2(l%4) + {0,1}, t = 0..7).  Panel P: warp P runs its 8 elimination
// steps alone (warp-synchronous, rows published to shared memory), then every warp w > P applies
// the panel as one rank-8 update on the FP64 tensor cores: M -= F W with F_ik = S_ki / p_k from the
// published rows and W the coefficient rows (upper: S_kc; lower: N_kc, 1 at c = k, 0 right of it).
__device__ __forceinline__ void dmma884v(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ long long g_v8ts[8][8][3];
#define V8TS(P_, q_) do { if (l == 0 && blockIdx.x == 0) g_v8ts[w][P_][q_] = clock64(); } while (0)
__device__ __noinline__ void diag_v8(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                     int *__restrict__ flag, double *sm, bool preloaded = false) {
  double *R = sm, *Li = sm + TB * LD;   // R[j][0..63] row j as of step j, R[j][TB] = 1 / p_j
  const int t = threadIdx.x, w = t >> 5, l = t & 31, m = l >> 2, n2 = 2 * (l & 3);
  const int i = 8 * w + m;   // this lane's row
  double M[8][2];            // M[tile][e]: column 8 tile + n2 + e
  if (preloaded) {
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? R[c * LD + i] : 0.0;
      }
  } else {
    const size_t okk = tile_off(k, k, nSp);
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? __ldcg(&L[okk + (size_t)i * nSp + c]) : 0.0;
      }
  }
  __syncthreads();   // input consumed: R is the pivot-row buffer
  for (int P = 0; P < 8; ++P) {
    V8TS(P, 0);
    if (w == P) {
      // ---- the panel's 8 steps, this warp alone
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int j = 8 * P + s;
        if (m == s) {   // publish row j (final)
#pragma unroll
          for (int tt = 0; tt < 8; ++tt)
            *reinterpret_cast<double2 *>(&R[j * LD + 8 * tt + n2]) = make_double2(M[tt][0], M[tt][1]);
        }
        __syncwarp();
        const double p = R[j * LD + j];
        const double q = rcp_nr(p > 0.0 ? p : 1.0);
        if (l == 0) R[j * LD + TB] = q;
        if (s < 7) {
          const double f = i > j ? R[j * LD + i] * q : 0.0;
#pragma unroll
          for (int tt = 0; tt < 8; ++tt) {
            const double2 u = *reinterpret_cast<const double2 *>(&R[j * LD + 8 * tt + n2]);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int c = 8 * tt + n2 + e;
              const double ue = e ? u.y : u.x;
              const double wc = (c >= i || c < j) ? ue : (c == j ? 1.0 : 0.0);
              M[tt][e] = fma(-f, wc, M[tt][e]);
            }
          }
        }
      }
    }
    V8TS(P, 1);
    __syncthreads();
    if (w > P) {
      // ---- rank-8 update with panel P on the tensor cores
      double fa[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kk = 8 * P + 4 * h + (l & 3);
        fa[h] = -R[kk * LD + i] * R[kk * LD + TB];   // -F[i][kk] (A fragment: row m, k = l & 3)
      }
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        if (tt > P && tt < w) continue;   // lower entries not yet formed: coefficient 0
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kk = 8 * P + 4 * h + (l & 3), c = 8 * tt + m;   // B fragment: k = l & 3, n = l / 4
          double b = R[kk * LD + c];
          if (tt == P) b = c < kk ? b : (c == kk ? 1.0 : 0.0);
          if (tt == w) dmma884v(d0, d1, fa[h], b);
          else dmma884v(M[tt][0], M[tt][1], fa[h], b);
        }
        if (tt == w) {   // diagonal tile: upper entries only
          if (8 * tt + n2 >= i) M[tt][0] += d0;
          if (8 * tt + n2 + 1 >= i) M[tt][1] += d1;
        }
      }
    }
    V8TS(P, 2);
  }
  // L_kk^-1 = D^-1/2 N
  {
    const double p = R[i * LD + i];
    const double r = rsqrt_nr(p > 0.0 ? p : 1.0);
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        Li[i * LD + c] = c < i ? r * M[tt][e] : (c == i ? r : 0.0);
      }
    if ((l & 3) == 0 && flag && !(p > 0.0)) *flag = 1;
  }
  __syncthreads();
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
}

// V9: V8's warp-per-panel layout with a pipelined handoff.  Warp w: rank-8 tensor-core updates
// with the panels P <= w - 2 (each released by a per-panel named barrier once complete), then the
// 8 rows of panel w - 1 one at a time as its producer publishes them (per-row named barriers:
// producer arrives, the next warp waits), then its own panel.  The critical path is the chain of
// single-warp elimination steps; panel indices are template parameters so that the position of
// each column tile against the panel is static (no per-entry selects outside the panel's tile).
namespace v9 {
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_wait(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
constexpr int kRowBar = 1;    // ids 1..8: row s of the current panel
constexpr int kPanBar = 9;    // ids 9, 10: panel P complete (P even / odd)

template <int P>
__device__ __forceinline__ void produce(double (&M)[8][2], double *R, int l) {
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * P + m;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int j = 8 * P + s;
    if (m == s) {
#pragma unroll
      for (int tt = 0; tt < 8; ++tt)
        *reinterpret_cast<double2 *>(&R[j * LD + 8 * tt + n2]) = make_double2(M[tt][0], M[tt][1]);
    }
    if (P < 7) bar_arrive(kRowBar + s, 64);
    __syncwarp();
    const double p = R[j * LD + j];
    const double q = rcp_nr(p > 0.0 ? p : 1.0);
    if (s < 7) {
      double2 uu[8];   // the pivot row and S_ji are loaded while the reciprocal forms
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) uu[tt] = *reinterpret_cast<const double2 *>(&R[j * LD + 8 * tt + n2]);
      const double sji = R[j * LD + i];
      const double f = m > s ? sji * q : 0.0;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        const double2 u = uu[tt];
        if (tt != P) {   // left of the panel: N_jc (c < j); right of it: S_jc (c > i)
          M[tt][0] = fma(-f, u.x, M[tt][0]);
          M[tt][1] = fma(-f, u.y, M[tt][1]);
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cp = n2 + e;   // column within the panel
            const double ue = e ? u.y : u.x;
            const double wc = (cp >= m || cp < s) ? ue : (cp == s ? 1.0 : 0.0);
            M[tt][e] = fma(-f, wc, M[tt][e]);
          }
        }
      }
    }
    if (l == 0) R[j * LD + TB] = q;   // 1 / p_j for the far consumers (after the loads: no aliasing stall)
  }
  if (P <= 5) bar_arrive(kPanBar + (P & 1), 32 * (7 - P));
}

// warp P + 1: the rows of panel P as they arrive (its rows are all below the panel)
template <int P>
__device__ __forceinline__ void near(double (&M)[8][2], const double *R, int l) {
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * (P + 1) + m;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int j = 8 * P + s;
    bar_wait(kRowBar + s, 64);
    const double p = R[j * LD + j];
    const double sji = R[j * LD + i];
    const double q = rcp_nr(p > 0.0 ? p : 1.0);
    const double f = sji * q;
#pragma unroll
    for (int tt = 0; tt < 8; ++tt) {
      const double2 u = *reinterpret_cast<const double2 *>(&R[j * LD + 8 * tt + n2]);
      if (tt < P || tt > P + 1) {
        M[tt][0] = fma(-f, u.x, M[tt][0]);
        M[tt][1] = fma(-f, u.y, M[tt][1]);
      } else if (tt == P) {   // panel columns (lower): N_jc, 1, 0
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cp = n2 + e;
          const double ue = e ? u.y : u.x;
          M[tt][e] = fma(-f, cp < s ? ue : (cp == s ? 1.0 : 0.0), M[tt][e]);
        }
      } else {                // own diagonal tile: upper entries only
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (n2 + e >= m) M[tt][e] = fma(-f, e ? u.y : u.x, M[tt][e]);
      }
    }
  }
}

// warp w >= P + 2: panel P as one rank-8 update on the tensor cores
__device__ __forceinline__ void far(double (&M)[8][2], const double *R, int l, int w, int P) {
  bar_wait(kPanBar + (P & 1), 32 * (7 - P));
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * w + m;
  double fa[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int kk = 8 * P + 4 * h + (l & 3);
    fa[h] = -R[kk * LD + i] * R[kk * LD + TB];
  }
#pragma unroll
  for (int tt = 0; tt < 8; ++tt) {
    if (tt > P && tt < w) continue;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = 8 * P + 4 * h + (l & 3), c = 8 * tt + m;
      double b = R[kk * LD + c];
      if (tt == P) b = c < kk ? b : (c == kk ? 1.0 : 0.0);
      if (tt == w) dmma884v(d0, d1, fa[h], b);
      else dmma884v(M[tt][0], M[tt][1], fa[h], b);
    }
    if (tt == w) {
      if (8 * tt + n2 >= i) M[tt][0] += d0;
      if (8 * tt + n2 + 1 >= i) M[tt][1] += d1;
    }
  }
}
}  // namespace v9

__device__ __noinline__ void diag_v9(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                     int *__restrict__ flag, double *sm, bool preloaded = false) {
  double *R = sm, *Li = sm + TB * LD;
  const int t = threadIdx.x, w = t >> 5, l = t & 31, m = l >> 2, n2 = 2 * (l & 3);
  const int i = 8 * w + m;
  double M[8][2];
  if (preloaded) {
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? R[c * LD + i] : 0.0;
      }
  } else {
    const size_t okk = tile_off(k, k, nSp);
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? __ldcg(&L[okk + (size_t)i * nSp + c]) : 0.0;
      }
  }
  __syncthreads();
  for (int P = 0; P + 2 <= w; ++P) v9::far(M, R, l, w, P);
  switch (w) {
    case 0: v9::produce<0>(M, R, l); break;
    case 1: v9::near<0>(M, R, l); v9::produce<1>(M, R, l); break;
    case 2: v9::near<1>(M, R, l); v9::produce<2>(M, R, l); break;
    case 3: v9::near<2>(M, R, l); v9::produce<3>(M, R, l); break;
    case 4: v9::near<3>(M, R, l); v9::produce<4>(M, R, l); break;
    case 5: v9::near<4>(M, R, l); v9::produce<5>(M, R, l); break;
    case 6: v9::near<5>(M, R, l); v9::produce<6>(M, R, l); break;
    default: v9::near<6>(M, R, l); v9::produce<7>(M, R, l); break;
  }
  __syncthreads();
  {
    const double p = R[i * LD + i];
    const double r = rsqrt_nr(p > 0.0 ? p : 1.0);
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        Li[i * LD + c] = c < i ? r * M[tt][e] : (c == i ? r : 0.0);
      }
    if ((l & 3) == 0 && flag && !(p > 0.0)) *flag = 1;
  }
  __syncthreads();
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
}

// V10: V9 with 2 x 2 block pivots in the panel chains (4 pair steps per panel).  Pair (a, b) =
// (8P + 2S, 8P + 2S + 1): G = [[p_aa, p_ab], [p_ab, p_bb]]^-1; rows below the pair get
// (f_a, f_b) = (S_ia, S_ib) G; the block leaves N_ab = N_ba = 0, so the lower coefficient rule
// (N_kc left of the pair, 1 at c = k, 0 elsewhere) reads the untouched zeros of R.
namespace v10 {
using v9::bar_arrive;
using v9::bar_wait;
__device__ __forceinline__ void pinv2(double paa, double pab, double pbb, double &gaa, double &gab, double &gbb) {
  const double det = fma(paa, pbb, -pab * pab);
  const double id = rcp_nr(det > 0.0 && paa > 0.0 ? det : 1.0);
  gaa = pbb * id;
  gab = -pab * id;
  gbb = paa * id;
}

template <int P>
__device__ __forceinline__ void produce(double (&M)[8][2], double *R, int l) {
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * P + m;
#pragma unroll
  for (int S = 0; S < 4; ++S) {
    const int a = 8 * P + 2 * S, b = a + 1;
    if ((m >> 1) == S) {   // publish rows a, b
      const int r = 8 * P + m;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt)
        *reinterpret_cast<double2 *>(&R[r * LD + 8 * tt + n2]) = make_double2(M[tt][0], M[tt][1]);
    }
    if (P < 7) bar_arrive(1 + S, 64);
    __syncwarp();
    const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
    double gaa, gab, gbb;
    if (S < 3) {
      double2 ua[8], ub[8];
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        ua[tt] = *reinterpret_cast<const double2 *>(&R[a * LD + 8 * tt + n2]);
        ub[tt] = *reinterpret_cast<const double2 *>(&R[b * LD + 8 * tt + n2]);
      }
      const double sa = R[a * LD + i], sb = R[b * LD + i];
      pinv2(paa, pab, pbb, gaa, gab, gbb);
      const bool act = m > 2 * S + 1;
      const double fa = act ? fma(sa, gaa, sb * gab) : 0.0;
      const double fb = act ? fma(sa, gab, sb * gbb) : 0.0;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        if (tt != P) {
          M[tt][0] = fma(-fa, ua[tt].x, fma(-fb, ub[tt].x, M[tt][0]));
          M[tt][1] = fma(-fa, ua[tt].y, fma(-fb, ub[tt].y, M[tt][1]));
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cp = n2 + e;
            const bool use = cp >= m || cp < 2 * S;
            const double xa = use ? (e ? ua[tt].y : ua[tt].x) : (cp == 2 * S ? 1.0 : 0.0);
            const double xb = use ? (e ? ub[tt].y : ub[tt].x) : (cp == 2 * S + 1 ? 1.0 : 0.0);
            M[tt][e] = fma(-fa, xa, fma(-fb, xb, M[tt][e]));
          }
        }
      }
    } else {
      pinv2(paa, pab, pbb, gaa, gab, gbb);
    }
    if (l == 0) {   // G for the far consumers
      R[a * LD + TB] = gaa;
      R[a * LD + TB + 1] = gab;
      R[a * LD + TB + 2] = gbb;
    }
  }
  if (P <= 5) bar_arrive(9 + (P & 1), 32 * (7 - P));
}

template <int P>
__device__ __forceinline__ void near(double (&M)[8][2], const double *R, int l) {
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * (P + 1) + m;
#pragma unroll
  for (int S = 0; S < 4; ++S) {
    const int a = 8 * P + 2 * S, b = a + 1;
    bar_wait(1 + S, 64);
    const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
    const double sa = R[a * LD + i], sb = R[b * LD + i];
    double2 ua[8], ub[8];
#pragma unroll
    for (int tt = 0; tt < 8; ++tt) {
      ua[tt] = *reinterpret_cast<const double2 *>(&R[a * LD + 8 * tt + n2]);
      ub[tt] = *reinterpret_cast<const double2 *>(&R[b * LD + 8 * tt + n2]);
    }
    double gaa, gab, gbb;
    pinv2(paa, pab, pbb, gaa, gab, gbb);
    const double fa = fma(sa, gaa, sb * gab), fb = fma(sa, gab, sb * gbb);
#pragma unroll
    for (int tt = 0; tt < 8; ++tt) {
      if (tt < P || tt > P + 1) {
        M[tt][0] = fma(-fa, ua[tt].x, fma(-fb, ub[tt].x, M[tt][0]));
        M[tt][1] = fma(-fa, ua[tt].y, fma(-fb, ub[tt].y, M[tt][1]));
      } else if (tt == P) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cp = n2 + e;
          const bool use = cp < 2 * S;
          const double xa = use ? (e ? ua[tt].y : ua[tt].x) : (cp == 2 * S ? 1.0 : 0.0);
          const double xb = use ? (e ? ub[tt].y : ub[tt].x) : (cp == 2 * S + 1 ? 1.0 : 0.0);
          M[tt][e] = fma(-fa, xa, fma(-fb, xb, M[tt][e]));
        }
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (n2 + e >= m)
            M[tt][e] = fma(-fa, e ? ua[tt].y : ua[tt].x, fma(-fb, e ? ub[tt].y : ub[tt].x, M[tt][e]));
      }
    }
  }
}

__device__ __forceinline__ void far(double (&M)[8][2], const double *R, int l, int w, int P) {
  bar_wait(9 + (P & 1), 32 * (7 - P));
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * w + m;
  double fa[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int kk = 8 * P + 4 * h + (l & 3), a = kk & ~1;   // pair (a, a + 1) holding k
    const double sa = R[a * LD + i], sb = R[(a + 1) * LD + i];
    const double gaa = R[a * LD + TB], gab = R[a * LD + TB + 1], gbb = R[a * LD + TB + 2];
    fa[h] = (kk & 1) ? -fma(sa, gab, sb * gbb) : -fma(sa, gaa, sb * gab);
  }
#pragma unroll
  for (int tt = 0; tt < 8; ++tt) {
    if (tt > P && tt < w) continue;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = 8 * P + 4 * h + (l & 3), c = 8 * tt + m;
      double b = R[kk * LD + c];
      if (tt == P) b = c < kk ? b : (c == kk ? 1.0 : 0.0);
      if (tt == w) dmma884v(d0, d1, fa[h], b);
      else dmma884v(M[tt][0], M[tt][1], fa[h], b);
    }
    if (tt == w) {
      if (8 * tt + n2 >= i) M[tt][0] += d0;
      if (8 * tt + n2 + 1 >= i) M[tt][1] += d1;
    }
  }
}
}  // namespace v10

__device__ long long g_v10ts[8][8];
#define V10TS(q_) do { if (l == 0 && blockIdx.x == 0) g_v10ts[w][q_] = clock64(); } while (0)
__device__ __noinline__ void diag_v10(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                      int *__restrict__ flag, double *sm, bool preloaded = false) {
  double *R = sm, *Li = sm + TB * LD;
  const int t = threadIdx.x, w = t >> 5, l = t & 31, m = l >> 2, n2 = 2 * (l & 3);
  const int i = 8 * w + m;
  double M[8][2];
  if (preloaded) {
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? R[c * LD + i] : 0.0;
      }
  } else {
    const size_t okk = tile_off(k, k, nSp);
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? __ldcg(&L[okk + (size_t)i * nSp + c]) : 0.0;
      }
  }
  V10TS(0);
  __syncthreads();
  V10TS(1);
  for (int P = 0; P + 2 <= w; ++P) v10::far(M, R, l, w, P);
  V10TS(2);
  if (w > 0) switch (w) {
    case 1: v10::near<0>(M, R, l); break;
    case 2: v10::near<1>(M, R, l); break;
    case 3: v10::near<2>(M, R, l); break;
    case 4: v10::near<3>(M, R, l); break;
    case 5: v10::near<4>(M, R, l); break;
    case 6: v10::near<5>(M, R, l); break;
    default: v10::near<6>(M, R, l); break;
  }
  V10TS(3);
  switch (w) {
    case 0: v10::produce<0>(M, R, l); break;
    case 1: v10::produce<1>(M, R, l); break;
    case 2: v10::produce<2>(M, R, l); break;
    case 3: v10::produce<3>(M, R, l); break;
    case 4: v10::produce<4>(M, R, l); break;
    case 5: v10::produce<5>(M, R, l); break;
    case 6: v10::produce<6>(M, R, l); break;
    default: v10::produce<7>(M, R, l); break;
  }
  V10TS(4);
  __syncthreads();
  V10TS(5);
  {
    // L^-1 = C^-1 N per 2 x 2 block (rows a = i & ~1, b = a + 1; the partner row is lane l ^ 4)
    const int a = i & ~1, b = a + 1;
    const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
    const bool ok = paa > 0.0;
    const double ra = rsqrt_nr(ok ? paa : 1.0);
    const double mm = ok ? pab * ra * ra : 0.0;
    const double sc = fma(-mm, pab, pbb);
    const double rb = rsqrt_nr(sc > 0.0 ? sc : 1.0);
    const bool is_b = i & 1;
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        const double own = c < a ? M[tt][e] : (c == i ? 1.0 : 0.0);        // N_ic
        const double na = __shfl_xor_sync(0xffffffffu, own, 4);              // partner row's N
        Li[i * LD + c] = is_b ? rb * fma(-mm, na, own) : ra * own;
      }
    if ((l & 7) == 0 && flag && !(ok && sc > 0.0)) *flag = 1;
  }
  __syncthreads();
  V10TS(6);
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
}

// V11: V10 with every warp below the panel following the producer pair by pair (rank-2 updates;
// per-pair named barrier over the producer and all followers) instead of the rank-8 tensor-core
// update at the end of each panel.
namespace v11 {
using v9::bar_arrive;
using v9::bar_wait;
using v10::pinv2;
template <int P>
__device__ __forceinline__ void produce(double (&M)[8][2], double *R, int l) {
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * P + m;
#pragma unroll
  for (int S = 0; S < 4; ++S) {
    const int a = 8 * P + 2 * S, b = a + 1;
    if ((m >> 1) == S) {
      const int r = 8 * P + m;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt)
        *reinterpret_cast<double2 *>(&R[r * LD + 8 * tt + n2]) = make_double2(M[tt][0], M[tt][1]);
    }
    if (P < 7) bar_arrive(1 + S, 32 * (8 - P));
    __syncwarp();
    if (S < 3) {
      const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
      double2 ua[8], ub[8];
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        ua[tt] = *reinterpret_cast<const double2 *>(&R[a * LD + 8 * tt + n2]);
        ub[tt] = *reinterpret_cast<const double2 *>(&R[b * LD + 8 * tt + n2]);
      }
      const double sa = R[a * LD + i], sb = R[b * LD + i];
      double gaa, gab, gbb;
      pinv2(paa, pab, pbb, gaa, gab, gbb);
      const bool act = m > 2 * S + 1;
      const double fa = act ? fma(sa, gaa, sb * gab) : 0.0;
      const double fb = act ? fma(sa, gab, sb * gbb) : 0.0;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        if (tt != P) {
          M[tt][0] = fma(-fa, ua[tt].x, fma(-fb, ub[tt].x, M[tt][0]));
          M[tt][1] = fma(-fa, ua[tt].y, fma(-fb, ub[tt].y, M[tt][1]));
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cp = n2 + e;
            const bool use = cp >= m || cp < 2 * S;
            const double xa = use ? (e ? ua[tt].y : ua[tt].x) : (cp == 2 * S ? 1.0 : 0.0);
            const double xb = use ? (e ? ub[tt].y : ub[tt].x) : (cp == 2 * S + 1 ? 1.0 : 0.0);
            M[tt][e] = fma(-fa, xa, fma(-fb, xb, M[tt][e]));
          }
        }
      }
    }
  }
}

// warp w > P: pair S of panel P
__device__ __forceinline__ void follow(double (&M)[8][2], const double *R, int l, int w, int P, int S) {
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * w + m;
  const int a = 8 * P + 2 * S, b = a + 1;
  bar_wait(1 + S, 32 * (8 - P));
  const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
  const double sa = R[a * LD + i], sb = R[b * LD + i];
  double2 ua[8], ub[8];
#pragma unroll
  for (int tt = 0; tt < 8; ++tt) {
    ua[tt] = *reinterpret_cast<const double2 *>(&R[a * LD + 8 * tt + n2]);
    ub[tt] = *reinterpret_cast<const double2 *>(&R[b * LD + 8 * tt + n2]);
  }
  double gaa, gab, gbb;
  pinv2(paa, pab, pbb, gaa, gab, gbb);
  const double fa = fma(sa, gaa, sb * gab), fb = fma(sa, gab, sb * gbb);
#pragma unroll
  for (int tt = 0; tt < 8; ++tt) {
    if (tt < P || tt > w) {
      M[tt][0] = fma(-fa, ua[tt].x, fma(-fb, ub[tt].x, M[tt][0]));
      M[tt][1] = fma(-fa, ua[tt].y, fma(-fb, ub[tt].y, M[tt][1]));
    } else if (tt == P) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cp = n2 + e;
        const bool use = cp < 2 * S;
        const double xa = use ? (e ? ua[tt].y : ua[tt].x) : (cp == 2 * S ? 1.0 : 0.0);
        const double xb = use ? (e ? ub[tt].y : ub[tt].x) : (cp == 2 * S + 1 ? 1.0 : 0.0);
        M[tt][e] = fma(-fa, xa, fma(-fb, xb, M[tt][e]));
      }
    } else if (tt == w) {
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (n2 + e >= m)
          M[tt][e] = fma(-fa, e ? ua[tt].y : ua[tt].x, fma(-fb, e ? ub[tt].y : ub[tt].x, M[tt][e]));
    }
  }
}
}  // namespace v11

__device__ __noinline__ void diag_v11(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                      int *__restrict__ flag, double *sm, bool preloaded = false) {
  double *R = sm, *Li = sm + TB * LD;
  const int t = threadIdx.x, w = t >> 5, l = t & 31, m = l >> 2, n2 = 2 * (l & 3);
  const int i = 8 * w + m;
  double M[8][2];
  if (preloaded) {
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? R[c * LD + i] : 0.0;
      }
  } else {
    const size_t okk = tile_off(k, k, nSp);
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? __ldcg(&L[okk + (size_t)i * nSp + c]) : 0.0;
      }
  }
  __syncthreads();
  for (int P = 0; P < w; ++P)
    for (int S = 0; S < 4; ++S) v11::follow(M, R, l, w, P, S);
  switch (w) {
    case 0: v11::produce<0>(M, R, l); break;
    case 1: v11::produce<1>(M, R, l); break;
    case 2: v11::produce<2>(M, R, l); break;
    case 3: v11::produce<3>(M, R, l); break;
    case 4: v11::produce<4>(M, R, l); break;
    case 5: v11::produce<5>(M, R, l); break;
    case 6: v11::produce<6>(M, R, l); break;
    default: v11::produce<7>(M, R, l); break;
  }
  __syncthreads();
  {
    const int a = i & ~1, b = a + 1;
    const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
    const bool ok = paa > 0.0;
    const double ra = rsqrt_nr(ok ? paa : 1.0);
    const double mm = ok ? pab * ra * ra : 0.0;
    const double sc = fma(-mm, pab, pbb);
    const double rb = rsqrt_nr(sc > 0.0 ? sc : 1.0);
    const bool is_b = i & 1;
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        const double own = c < a ? M[tt][e] : (c == i ? 1.0 : 0.0);
        const double na = __shfl_xor_sync(0xffffffffu, own, 4);
        Li[i * LD + c] = is_b ? rb * fma(-mm, na, own) : ra * own;
      }
    if ((l & 7) == 0 && flag && !(ok && sc > 0.0)) *flag = 1;
  }
  __syncthreads();
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
}

// V12: V10 with runtime panel / pair indices (one copy of the producer and follower code): the
// per-P template copies of V10 do not fit the instruction cache on the chain CTA (measured cold:
// 29.7 k cycles against 18.9 k warm).
namespace v12 {
using v9::bar_arrive;
using v9::bar_wait;
using v10::pinv2;

__device__ __forceinline__ void produce(double (&M)[8][2], double *R, int l, int P) {
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * P + m;
#pragma unroll 1
  for (int S = 0; S < 4; ++S) {
    const int a = 8 * P + 2 * S, b = a + 1;
    if ((m >> 1) == S) {   // publish rows a, b
      const int r = 8 * P + m;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt)
        *reinterpret_cast<double2 *>(&R[r * LD + 8 * tt + n2]) = make_double2(M[tt][0], M[tt][1]);
    }
    if (P < 7) bar_arrive(1 + S, 64);
    __syncwarp();
    const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
    double gaa, gab, gbb;
    if (S < 3) {
      double2 ua[8], ub[8];
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        ua[tt] = *reinterpret_cast<const double2 *>(&R[a * LD + 8 * tt + n2]);
        ub[tt] = *reinterpret_cast<const double2 *>(&R[b * LD + 8 * tt + n2]);
      }
      const double sa = R[a * LD + i], sb = R[b * LD + i];
      pinv2(paa, pab, pbb, gaa, gab, gbb);
      const bool act = m > 2 * S + 1;
      const double fa = act ? fma(sa, gaa, sb * gab) : 0.0;
      const double fb = act ? fma(sa, gab, sb * gbb) : 0.0;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        if (tt != P) {
          M[tt][0] = fma(-fa, ua[tt].x, fma(-fb, ub[tt].x, M[tt][0]));
          M[tt][1] = fma(-fa, ua[tt].y, fma(-fb, ub[tt].y, M[tt][1]));
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cp = n2 + e;
            const bool use = cp >= m || cp < 2 * S;
            const double xa = use ? (e ? ua[tt].y : ua[tt].x) : (cp == 2 * S ? 1.0 : 0.0);
            const double xb = use ? (e ? ub[tt].y : ub[tt].x) : (cp == 2 * S + 1 ? 1.0 : 0.0);
            M[tt][e] = fma(-fa, xa, fma(-fb, xb, M[tt][e]));
          }
        }
      }
    } else {
      pinv2(paa, pab, pbb, gaa, gab, gbb);
    }
    if (l == 0) {   // G for the far consumers
      R[a * LD + TB] = gaa;
      R[a * LD + TB + 1] = gab;
      R[a * LD + TB + 2] = gbb;
    }
  }
  if (P <= 5) bar_arrive(9 + (P & 1), 32 * (7 - P));
}

__device__ __forceinline__ void near(double (&M)[8][2], const double *R, int l, int P) {
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * (P + 1) + m;
#pragma unroll 1
  for (int S = 0; S < 4; ++S) {
    const int a = 8 * P + 2 * S, b = a + 1;
    bar_wait(1 + S, 64);
    const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
    const double sa = R[a * LD + i], sb = R[b * LD + i];
    double2 ua[8], ub[8];
#pragma unroll
    for (int tt = 0; tt < 8; ++tt) {
      ua[tt] = *reinterpret_cast<const double2 *>(&R[a * LD + 8 * tt + n2]);
      ub[tt] = *reinterpret_cast<const double2 *>(&R[b * LD + 8 * tt + n2]);
    }
    double gaa, gab, gbb;
    pinv2(paa, pab, pbb, gaa, gab, gbb);
    const double fa = fma(sa, gaa, sb * gab), fb = fma(sa, gab, sb * gbb);
#pragma unroll
    for (int tt = 0; tt < 8; ++tt) {
      if (tt < P || tt > P + 1) {
        M[tt][0] = fma(-fa, ua[tt].x, fma(-fb, ub[tt].x, M[tt][0]));
        M[tt][1] = fma(-fa, ua[tt].y, fma(-fb, ub[tt].y, M[tt][1]));
      } else if (tt == P) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cp = n2 + e;
          const bool use = cp < 2 * S;
          const double xa = use ? (e ? ua[tt].y : ua[tt].x) : (cp == 2 * S ? 1.0 : 0.0);
          const double xb = use ? (e ? ub[tt].y : ub[tt].x) : (cp == 2 * S + 1 ? 1.0 : 0.0);
          M[tt][e] = fma(-fa, xa, fma(-fb, xb, M[tt][e]));
        }
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (n2 + e >= m)
            M[tt][e] = fma(-fa, e ? ua[tt].y : ua[tt].x, fma(-fb, e ? ub[tt].y : ub[tt].x, M[tt][e]));
      }
    }
  }
}

__device__ __forceinline__ void far(double (&M)[8][2], const double *R, int l, int w, int P) {
  bar_wait(9 + (P & 1), 32 * (7 - P));
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * w + m;
  double fa[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int kk = 8 * P + 4 * h + (l & 3), a = kk & ~1;   // pair (a, a + 1) holding k
    const double sa = R[a * LD + i], sb = R[(a + 1) * LD + i];
    const double gaa = R[a * LD + TB], gab = R[a * LD + TB + 1], gbb = R[a * LD + TB + 2];
    fa[h] = (kk & 1) ? -fma(sa, gab, sb * gbb) : -fma(sa, gaa, sb * gab);
  }
#pragma unroll
  for (int tt = 0; tt < 8; ++tt) {
    if (tt > P && tt < w) continue;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = 8 * P + 4 * h + (l & 3), c = 8 * tt + m;
      double b = R[kk * LD + c];
      if (tt == P) b = c < kk ? b : (c == kk ? 1.0 : 0.0);
      if (tt == w) dmma884v(d0, d1, fa[h], b);
      else dmma884v(M[tt][0], M[tt][1], fa[h], b);
    }
    if (tt == w) {
      if (8 * tt + n2 >= i) M[tt][0] += d0;
      if (8 * tt + n2 + 1 >= i) M[tt][1] += d1;
    }
  }
}
}  // namespace v12

__device__ __noinline__ void diag_v12(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                      int *__restrict__ flag, double *sm, bool preloaded = false) {
  double *R = sm, *Li = sm + TB * LD;
  const int t = threadIdx.x, w = t >> 5, l = t & 31, m = l >> 2, n2 = 2 * (l & 3);
  const int i = 8 * w + m;
  double M[8][2];
  if (preloaded) {
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? R[c * LD + i] : 0.0;
      }
  } else {
    const size_t okk = tile_off(k, k, nSp);
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? __ldcg(&L[okk + (size_t)i * nSp + c]) : 0.0;
      }
  }
  __syncthreads();
  for (int P = 0; P + 2 <= w; ++P) v12::far(M, R, l, w, P);
  if (w > 0) v12::near(M, R, l, w - 1);
  v12::produce(M, R, l, w);
  __syncthreads();
  {
    const int a = i & ~1, b = a + 1;
    const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
    const bool ok = paa > 0.0;
    const double ra = rsqrt_nr(ok ? paa : 1.0);
    const double mm = ok ? pab * ra * ra : 0.0;
    const double sc = fma(-mm, pab, pbb);
    const double rb = rsqrt_nr(sc > 0.0 ? sc : 1.0);
    const bool is_b = i & 1;
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        const double own = c < a ? M[tt][e] : (c == i ? 1.0 : 0.0);
        const double na = __shfl_xor_sync(0xffffffffu, own, 4);
        Li[i * LD + c] = is_b ? rb * fma(-mm, na, own) : ra * own;
      }
    if ((l & 7) == 0 && flag && !(ok && sc > 0.0)) *flag = 1;
  }
  __syncthreads();
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
}

// V13: V10 with the pair loops not unrolled (panel index still static): smaller code for the
// cold instruction cache of the chain CTA.
namespace v13 {
using v9::bar_arrive;
using v9::bar_wait;
using v10::pinv2;

template <int P>
__device__ __forceinline__ void produce(double (&M)[8][2], double *R, int l) {
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * P + m;
#pragma unroll 1
  for (int S = 0; S < 4; ++S) {
    const int a = 8 * P + 2 * S, b = a + 1;
    if ((m >> 1) == S) {   // publish rows a, b
      const int r = 8 * P + m;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt)
        *reinterpret_cast<double2 *>(&R[r * LD + 8 * tt + n2]) = make_double2(M[tt][0], M[tt][1]);
    }
    if (P < 7) bar_arrive(1 + S, 64);
    __syncwarp();
    const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
    double gaa, gab, gbb;
    if (S < 3) {
      double2 ua[8], ub[8];
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        ua[tt] = *reinterpret_cast<const double2 *>(&R[a * LD + 8 * tt + n2]);
        ub[tt] = *reinterpret_cast<const double2 *>(&R[b * LD + 8 * tt + n2]);
      }
      const double sa = R[a * LD + i], sb = R[b * LD + i];
      pinv2(paa, pab, pbb, gaa, gab, gbb);
      const bool act = m > 2 * S + 1;
      const double fa = act ? fma(sa, gaa, sb * gab) : 0.0;
      const double fb = act ? fma(sa, gab, sb * gbb) : 0.0;
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        if (tt != P) {
          M[tt][0] = fma(-fa, ua[tt].x, fma(-fb, ub[tt].x, M[tt][0]));
          M[tt][1] = fma(-fa, ua[tt].y, fma(-fb, ub[tt].y, M[tt][1]));
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cp = n2 + e;
            const bool use = cp >= m || cp < 2 * S;
            const double xa = use ? (e ? ua[tt].y : ua[tt].x) : (cp == 2 * S ? 1.0 : 0.0);
            const double xb = use ? (e ? ub[tt].y : ub[tt].x) : (cp == 2 * S + 1 ? 1.0 : 0.0);
            M[tt][e] = fma(-fa, xa, fma(-fb, xb, M[tt][e]));
          }
        }
      }
    } else {
      pinv2(paa, pab, pbb, gaa, gab, gbb);
    }
    if (l == 0) {   // G for the far consumers
      R[a * LD + TB] = gaa;
      R[a * LD + TB + 1] = gab;
      R[a * LD + TB + 2] = gbb;
    }
  }
  if (P <= 5) bar_arrive(9 + (P & 1), 32 * (7 - P));
}

template <int P>
__device__ __forceinline__ void near(double (&M)[8][2], const double *R, int l) {
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * (P + 1) + m;
#pragma unroll 1
  for (int S = 0; S < 4; ++S) {
    const int a = 8 * P + 2 * S, b = a + 1;
    bar_wait(1 + S, 64);
    const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
    const double sa = R[a * LD + i], sb = R[b * LD + i];
    double2 ua[8], ub[8];
#pragma unroll
    for (int tt = 0; tt < 8; ++tt) {
      ua[tt] = *reinterpret_cast<const double2 *>(&R[a * LD + 8 * tt + n2]);
      ub[tt] = *reinterpret_cast<const double2 *>(&R[b * LD + 8 * tt + n2]);
    }
    double gaa, gab, gbb;
    pinv2(paa, pab, pbb, gaa, gab, gbb);
    const double fa = fma(sa, gaa, sb * gab), fb = fma(sa, gab, sb * gbb);
#pragma unroll
    for (int tt = 0; tt < 8; ++tt) {
      if (tt < P || tt > P + 1) {
        M[tt][0] = fma(-fa, ua[tt].x, fma(-fb, ub[tt].x, M[tt][0]));
        M[tt][1] = fma(-fa, ua[tt].y, fma(-fb, ub[tt].y, M[tt][1]));
      } else if (tt == P) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cp = n2 + e;
          const bool use = cp < 2 * S;
          const double xa = use ? (e ? ua[tt].y : ua[tt].x) : (cp == 2 * S ? 1.0 : 0.0);
          const double xb = use ? (e ? ub[tt].y : ub[tt].x) : (cp == 2 * S + 1 ? 1.0 : 0.0);
          M[tt][e] = fma(-fa, xa, fma(-fb, xb, M[tt][e]));
        }
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (n2 + e >= m)
            M[tt][e] = fma(-fa, e ? ua[tt].y : ua[tt].x, fma(-fb, e ? ub[tt].y : ub[tt].x, M[tt][e]));
      }
    }
  }
}

__device__ __forceinline__ void far(double (&M)[8][2], const double *R, int l, int w, int P) {
  bar_wait(9 + (P & 1), 32 * (7 - P));
  const int m = l >> 2, n2 = 2 * (l & 3), i = 8 * w + m;
  double fa[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int kk = 8 * P + 4 * h + (l & 3), a = kk & ~1;   // pair (a, a + 1) holding k
    const double sa = R[a * LD + i], sb = R[(a + 1) * LD + i];
    const double gaa = R[a * LD + TB], gab = R[a * LD + TB + 1], gbb = R[a * LD + TB + 2];
    fa[h] = (kk & 1) ? -fma(sa, gab, sb * gbb) : -fma(sa, gaa, sb * gab);
  }
#pragma unroll
  for (int tt = 0; tt < 8; ++tt) {
    if (tt > P && tt < w) continue;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = 8 * P + 4 * h + (l & 3), c = 8 * tt + m;
      double b = R[kk * LD + c];
      if (tt == P) b = c < kk ? b : (c == kk ? 1.0 : 0.0);
      if (tt == w) dmma884v(d0, d1, fa[h], b);
      else dmma884v(M[tt][0], M[tt][1], fa[h], b);
    }
    if (tt == w) {
      if (8 * tt + n2 >= i) M[tt][0] += d0;
      if (8 * tt + n2 + 1 >= i) M[tt][1] += d1;
    }
  }
}
}  // namespace v13

__device__ __noinline__ void diag_v13(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                      int *__restrict__ flag, double *sm, bool preloaded = false) {
  double *R = sm, *Li = sm + TB * LD;
  const int t = threadIdx.x, w = t >> 5, l = t & 31, m = l >> 2, n2 = 2 * (l & 3);
  const int i = 8 * w + m;
  double M[8][2];
  if (preloaded) {
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? R[c * LD + i] : 0.0;
      }
  } else {
    const size_t okk = tile_off(k, k, nSp);
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        M[tt][e] = c >= i ? __ldcg(&L[okk + (size_t)i * nSp + c]) : 0.0;
      }
  }
  __syncthreads();
  for (int P = 0; P + 2 <= w; ++P) v13::far(M, R, l, w, P);
  if (w > 0) switch (w) {
    case 1: v13::near<0>(M, R, l); break;
    case 2: v13::near<1>(M, R, l); break;
    case 3: v13::near<2>(M, R, l); break;
    case 4: v13::near<3>(M, R, l); break;
    case 5: v13::near<4>(M, R, l); break;
    case 6: v13::near<5>(M, R, l); break;
    default: v13::near<6>(M, R, l); break;
  }
  switch (w) {
    case 0: v13::produce<0>(M, R, l); break;
    case 1: v13::produce<1>(M, R, l); break;
    case 2: v13::produce<2>(M, R, l); break;
    case 3: v13::produce<3>(M, R, l); break;
    case 4: v13::produce<4>(M, R, l); break;
    case 5: v13::produce<5>(M, R, l); break;
    case 6: v13::produce<6>(M, R, l); break;
    default: v13::produce<7>(M, R, l); break;
  }
  __syncthreads();
  {
    // L^-1 = C^-1 N per 2 x 2 block (rows a = i & ~1, b = a + 1; the partner row is lane l ^ 4)
    const int a = i & ~1, b = a + 1;
    const double paa = R[a * LD + a], pab = R[a * LD + b], pbb = R[b * LD + b];
    const bool ok = paa > 0.0;
    const double ra = rsqrt_nr(ok ? paa : 1.0);
    const double mm = ok ? pab * ra * ra : 0.0;
    const double sc = fma(-mm, pab, pbb);
    const double rb = rsqrt_nr(sc > 0.0 ? sc : 1.0);
    const bool is_b = i & 1;
#pragma unroll
    for (int tt = 0; tt < 8; ++tt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * tt + n2 + e;
        const double own = c < a ? M[tt][e] : (c == i ? 1.0 : 0.0);        // N_ic
        const double na = __shfl_xor_sync(0xffffffffu, own, 4);              // partner row's N
        Li[i * LD + c] = is_b ? rb * fma(-mm, na, own) : ra * own;
      }
    if ((l & 7) == 0 && flag && !(ok && sc > 0.0)) *flag = 1;
  }
  __syncthreads();
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
}
