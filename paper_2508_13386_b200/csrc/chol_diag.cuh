// Diagonal-tile factorisation D(k) of the coarse tile Cholesky (chol.cu): L_kk = chol(A_kk) and
// U_kk = L_kk^-T for one 64 x 64 tile by one 256-thread CTA.  SURVEY §8(a) a6; reading R4.
// Right-looking, 16-column panels factored by one warp in registers while the other warps form
// the inverse row blocks of the finished panels on the FP64 tensor cores (timed by
// tools/bench_diag.cu; measured and dropped: a 2 x 2 recursion on 32 x 32 blocks with single-warp
// panel work, a shuffle-based panel broadcast, a scalar inverse).  Takes the tile from L
// (column-major, leading dimension nSp) or preloaded in shared memory, and writes L_kk back there
// and U_kk (row-major 64 x 64) to U + k 64^2; *flag = 1 if a pivot is not positive.
// Requires TB = 64, LD = 65 and tile_off() from the including file.
#pragma once
#ifndef DIAG_TS
#define DIAG_TS(i)
#endif
#ifndef DIAG_TS_FLUSH
#define DIAG_TS_FLUSH()
#endif
#ifndef MSIM_STORE_LKK
#define MSIM_STORE_LKK 0
#endif

// ---------------------------------------------------------------- blocked factor + inverse
// smem: A [64][LD], Li [64][LD], T [16][kTS], invd [64], broadcast scratch [16]
constexpr int kTS = 52;   // T row stride: 52 = 4 (mod 16), conflict-free m8n8k4 fragments
constexpr int kDiagSmemDoublesBlocked = 2 * TB * LD + 16 * kTS + TB + 16;

__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// inv_rowblock with the two off-diagonal products on the FP64 tensor cores (mma.sync m8n8k4,
// one 8 x 8 output tile per warp at a time):
//   T = L_{pb, 0:o} Li_{0:o, 0:o}      (16 x o; Li lower triangular: k from the tile's column)
//   Li_{pb, 0:o} = -Li_{pb,pb} T       (Li_{pb,pb} lower triangular: k up to the tile's row)
// the diagonal block inverse (threads tt < 16) runs alongside the first product on the other
// warps.  Measured on the chain: the scalar version's last row block took ~6 k cycles.
__device__ __forceinline__ void inv_rowblock_mma(int pb, const double *A, double *Li, double *T,
                                                 const double *invd, int tt, int nth, int bar_id) {
  constexpr int TS = kTS;
  const int o = 16 * pb, lane = tt & 31, gw = tt >> 5, nw = nth >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  if (tt < 16) {
    double x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      double s = r == tt ? 1.0 : 0.0, s2 = 0.0;
#pragma unroll
      for (int q = 0; q < r; q += 2) {
        s = fma(-A[(o + r) * LD + o + q], x[q], s);
        if (q + 1 < r) s2 = fma(-A[(o + r) * LD + o + q + 1], x[q + 1], s2);
      }
      x[r] = (s + s2) * invd[o + r];
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) Li[(o + r) * LD + o + tt] = x[r];
  } else if (gw >= 1) {
    for (int tile = gw - 1; tile < 4 * pb; tile += nw - 1) {
      const int ri = tile & 1, cj = tile >> 1;
      double c0 = 0.0, c1 = 0.0;
      const double *ar = A + (o + 8 * ri + lr) * LD + lk;
      const double *bc = Li + lk * LD + 8 * cj + lr;
      for (int k0 = 8 * cj; k0 < o; k0 += 4) dmma884(c0, c1, ar[k0], bc[k0 * LD]);
      T[(8 * ri + lr) * TS + 8 * cj + 2 * lk] = c0;
      T[(8 * ri + lr) * TS + 8 * cj + 2 * lk + 1] = c1;
    }
  }
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nth) : "memory");
  if (pb == 0) return;
  for (int tile = gw; tile < 4 * pb; tile += nw) {
    const int ri = tile & 1, cj = tile >> 1;
    double c0 = 0.0, c1 = 0.0;
    const double *ar = Li + (o + 8 * ri + lr) * LD + o + lk;
    const double *bc = T + lk * TS + 8 * cj + lr;
#pragma unroll
    for (int k0 = 0; k0 < 16; k0 += 4)
      if (k0 < 8 * ri + 8) dmma884(c0, c1, ar[k0], bc[k0 * TS]);
    Li[(o + 8 * ri + lr) * LD + 8 * cj + 2 * lk] = -c0;
    Li[(o + 8 * ri + lr) * LD + 8 * cj + 2 * lk + 1] = -c1;
  }
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nth) : "memory");
}

__device__ void diag_factor_blocked(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                    int *__restrict__ flag, double *sm, bool preloaded) {
  double *A = sm;              // row-major [64][LD]: the factor
  double *Li = sm + TB * LD;   // row-major [64][LD]: its inverse
  double *Tb = sm + 2 * TB * LD;
  double *invd = sm + 2 * TB * LD + 16 * kTS;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  const size_t okk = tile_off(k, k, nSp);
  if (!preloaded) {
    double v[16];
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int e = t + it * 256;
      v[it] = __ldcg(&L[okk + (size_t)(e >> 6) * nSp + (e & 63)]);
    }
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int e = t + it * 256, r = e & 63, c = e >> 6;
      A[r * LD + c] = r >= c ? v[it] : 0.0;
    }
  }
#pragma unroll
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256;
    Li[(e & 63) * LD + (e >> 6)] = 0.0;
  }
  __syncthreads();
  DIAG_TS(0);
  bool bad = false;
  for (int p = 0; p < 4; ++p) {
    const int j0 = 16 * p;
    if (w == 4) {
      // idle: warp 4 shares warp 0's scheduler and the panel is a serial chain (measured ~1%)
    } else if (w != 0) {
      // warps 1-3, 5-7: row-block p-1 of the inverse (its columns of L are final) while warp 0
      // factors panel p
      const int tt = (w < 4 ? w - 1 : w - 2) * 32 + lane;
      if (p > 0) inv_rowblock_mma(p - 1, A, Li, Tb, invd, tt, 192, 1);
    } else {
      // panel rows j0 + lane and j0 + 32 + lane, columns j0 .. j0+15
      const int ra = j0 + lane, rb = j0 + 32 + lane;
      const bool va = ra < TB, vb = rb < TB;
      double a[16], b[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        a[c] = va ? A[ra * LD + j0 + c] : 0.0;
        b[c] = vb ? A[rb * LD + j0 + c] : 0.0;
      }
      // the pivot's lane takes the rsqrt of its own (final) diagonal; the column of L is then
      // broadcast through shared memory (one store, 15 - j broadcast loads)
      // (the next pivot, a_{j+1,j+1} - l_{j+1,j}^2, is formed by its own lane from its own values,
      // off the shared-memory round trip)
      // (the next pivot's rsqrt is issued right after the column scaling, ahead of the trailing
      // FMAs, in every lane -- lane j + 1's is the one used)
      double *pc = invd + TB;   // 16-double broadcast scratch
      double piv = a[0];
      bool pos = piv > 0.0;
      double ivn = rsqrt_nr2(pos ? piv : 1.0);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (lane == j) {
          if (!pos) {
            bad = true;
            a[j] = 1.0;
          }
          invd[j0 + j] = ivn;
        }
        const double inv = __shfl_sync(0xffffffffu, ivn, j);
        const double l = a[j] * inv;   // L_jj = a_jj / sqrt(a_jj); rows above: a = 0
        a[j] = l;
        b[j] *= inv;
        if (j + 1 < 16) {
          piv = fma(-l, l, a[j + 1]);   // meaningful in lane j + 1
          pos = piv > 0.0;
          ivn = rsqrt_nr2(pos ? piv : 1.0);
        }
        if (lane < 16) pc[lane] = l;
        __syncwarp();
#pragma unroll
        for (int c = j + 1; c < 16; ++c) {
          const double lc = pc[c];
          a[c] = fma(-l, lc, a[c]);
          b[c] = fma(-b[j], lc, b[c]);
        }
        __syncwarp();
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        if (va && ra >= j0 + c) A[ra * LD + j0 + c] = a[c];
        if (vb) A[rb * LD + j0 + c] = b[c];
      }
      DIAG_TS(10 + p);   // warp 0's panel done (before waiting for the inverse warps)
    }
    __syncthreads();
    DIAG_TS(1 + 2 * p);
    // trailing update of rows/cols >= j0 + 16
    const int s0 = j0 + 16;
    for (int r = s0 + (t >> 2); r < TB; r += 64) {
      for (int c = s0 + (t & 3); c <= r; c += 8) {   // two columns, four partial sums each
        const bool two = c + 4 <= r;
        double s0a = 0.0, s1a = 0.0, s0b = 0.0, s1b = 0.0;
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          const double x0 = A[r * LD + j0 + j], x1 = A[r * LD + j0 + j + 1];
          s0a = fma(x0, A[c * LD + j0 + j], s0a);
          s1a = fma(x1, A[c * LD + j0 + j + 1], s1a);
          if (two) {
            s0b = fma(x0, A[(c + 4) * LD + j0 + j], s0b);
            s1b = fma(x1, A[(c + 4) * LD + j0 + j + 1], s1b);
          }
        }
        A[r * LD + c] -= s0a + s1a;
        if (two) A[r * LD + c + 4] -= s0b + s1b;
      }
    }
    __syncthreads();
    DIAG_TS(2 + 2 * p);
  }
  if (w == 0 && lane == 0 && bad && flag) *flag = 1;
  // store the final rows 0..47 of Li as U_kk = Li^T (row-major: U[c][r] = Li[r][c]) now: the
  // stores drain while the last row block of the inverse is formed.  L_kk itself is not stored
  // (MSIM_STORE_LKK=1 restores it): every consumer of the diagonal tile -- the panel tasks and
  // both triangular sweeps -- uses U_kk.
  double *Uk = U + (size_t)k * TB * TB;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int e = t + it * 256, r = e & 63, c = e >> 6;
#if MSIM_STORE_LKK
    if (r >= c) __stcg(&L[okk + (size_t)c * nSp + r], A[r * LD + c]);
#endif
    if (r < 48) __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
  // last row-block of the inverse (the others were formed during the panels)
  inv_rowblock_mma(3, A, Li, Tb, invd, t, 256, 1);
  DIAG_TS(9);
#pragma unroll
  for (int it = 0; it < 4; ++it) {   // rows 48..63 of Li: 16 x 64 entries
    const int e = t + it * 256, r = 48 + (e & 15), c = e >> 4;
    __stcg(&Uk[(size_t)c * TB + r], Li[r * LD + c]);
  }
  DIAG_TS_FLUSH();
}


// ---------------------------------------------------------------- dispatch
constexpr int kDiagSmemDoubles = kDiagSmemDoublesBlocked;

// preloaded: the caller has already placed the (updated) tile in sm as A [64][LD] row-major,
// lower part, zeros above the diagonal (skips the global round trip on the critical path).
__device__ __noinline__ void diag_factor(int k, int nSp, double *__restrict__ L, double *__restrict__ U,
                                         int *__restrict__ flag, double *sm, bool preloaded = false) {
  diag_factor_blocked(k, nSp, L, U, flag, sm, preloaded);
}
