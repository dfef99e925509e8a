// Coarse factorisation S = L L^T and the triangular solves (
// reading R4: exact coarse solves).
//
// Layout: S (12m x 12m, handles in the cheaper of x-sorted / nested-dissection order, chosen at
// ms_basis_upload) is held in a padded dense column-major array; only the tiles of the
// symbolic factor (64 x 64 tiles) are touched.  Right-looking tile algorithm, three launches per
// tile column k (captured once in a CUDA graph and replayed):
//   D(k): one CTA factorises the diagonal tile (blocked, 16-column panels: warp-level panel
//         factorisation in registers + block-wide trailing update) and inverts it, storing L_kk
//         and U_kk = L_kk^-T;
//   P(k): one CTA per panel tile: L_ik = A_ik U_kk (64^3 GEMM, cp.async staging, 4x4 registers);
//   U(k): one CTA per trailing tile: A_ij -= L_ik L_jk^T.
// The forward / backward solves are single cooperative launches: each CTA owns tile rows, waits
// on the solution tiles it depends on (the vectors carry their own ready pattern) and applies
// U_kk as a GEMV.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <cuda_pipeline.h>

#include "common.cuh"
#include "fastmath.cuh"

namespace msim {

constexpr int TB = 64;
constexpr int LD = TB + 1;

__device__ __forceinline__ size_t tile_off(int ti, int tj, int nSp) {
  return (size_t)(tj * TB) * nSp + (size_t)ti * TB;
}

#include "chol_diag.cuh"

__global__ void __launch_bounds__(256) k_chol_diag(int k, int nSp, double *__restrict__ L,
                                                   double *__restrict__ U, int *__restrict__ flag) {
  extern __shared__ double sm[];
  diag_factor(k, nSp, L, U, flag, sm);
}

// ------------------------------------------------------------------ 64^3 tile GEMM core
// acc[a][b] = sum_kk S1[kk*64 + tr + a] * S2[kk*64 + tc + b]
__device__ __forceinline__ void gemm64(const double *S1, const double *S2, double (&acc)[4][4], int tr, int tc) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  // thread (tr, tc) = (t & 15, t >> 4) owns rows tr + 16a and columns tc + 16b: for each a the
  // 16 lanes of a half-warp read 16 consecutive doubles (one conflict-free wavefront) and the
  // other half-warp the same addresses (broadcast); the column operand is a 2-address broadcast.
#pragma unroll 4
  for (int kk = 0; kk < TB; ++kk) {
    double x[4], y[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      x[a] = S1[kk * TB + tr + 16 * a];
      y[a] = S2[kk * TB + tc + 16 * a];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(x[a], y[b], acc[a][b]);
  }
}

// ------------------------------------------------------------------ tile GEMM of the dataflow kernel
// acc = S1^T S2 over the 64-long k dimension (S1[kk*64 + r], S2[kk*64 + c]); thread-owned elements
// idx = 0..15 at (r, c) = tile_rc(idx).  MSIM_TILE_MMA: FP64 tensor cores (mma.sync m8n8k4): warp w
// owns rows 16 (w & 3) .. +15 and columns 32 (w >> 2) .. +31 as 2 x 4 blocks of 8 x 8; otherwise
// the DFMA register-blocked gemm64.
#ifndef MSIM_TILE_MMA
#define MSIM_TILE_MMA 1
#endif

__device__ __forceinline__ void tile_rc(int idx, int &r, int &c) {
#if MSIM_TILE_MMA
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j = idx & 1, bj = (idx >> 1) & 3, bi = idx >> 3;
  r = 16 * (w & 3) + 8 * bi + (lane >> 2);
  c = 32 * (w >> 2) + 8 * bj + 2 * (lane & 3) + j;
#else
  r = (threadIdx.x & 15) + 16 * (idx >> 2);
  c = (threadIdx.x >> 4) + 16 * (idx & 3);
#endif
}

__device__ __forceinline__ void tile_gemm(const double *S1, const double *S2, double (&acc)[16]) {
#if MSIM_TILE_MMA
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r0 = 16 * (w & 3) + (lane >> 2), c0 = 32 * (w >> 2) + (lane >> 2), kl = lane & 3;
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
#pragma unroll 4
  for (int k0 = 0; k0 < TB; k0 += 4) {
    const double *s1 = S1 + (k0 + kl) * TB, *s2 = S2 + (k0 + kl) * TB;
    const double a0 = s1[r0], a1 = s1[r0 + 8];
    double b[4];
#pragma unroll
    for (int bj = 0; bj < 4; ++bj) b[bj] = s2[c0 + 8 * bj];
#pragma unroll
    for (int bi = 0; bi < 2; ++bi)
#pragma unroll
      for (int bj = 0; bj < 4; ++bj)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[(bi * 4 + bj) * 2]), "+d"(acc[(bi * 4 + bj) * 2 + 1])
                     : "d"(bi ? a1 : a0), "d"(b[bj]));
  }
#else
  double a4[4][4];
  gemm64(S1, S2, a4, threadIdx.x & 15, threadIdx.x >> 4);
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = a4[q >> 2][q & 3];
#endif
}

// stage a column-major global tile (leading dim nSp) into k-major smem S[kk*64 + r] (cp.async)
// cp.async.cg: 16-byte global -> shared copy through L2 only (L1 is not coherent across SMs, and
// the dataflow kernel reads tiles other CTAs wrote during the same launch)
__device__ __forceinline__ void cp_async_cg16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit_wait() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

__device__ __forceinline__ void stage_colmajor(double *S, const double *__restrict__ G, int ld) {
#pragma unroll
  for (int it = 0; it < (TB * TB / 2) / 256; ++it) {
    const int e2 = threadIdx.x + it * 256, kk = e2 >> 5, r2 = (e2 & 31) * 2;
    cp_async_cg16(&S[kk * TB + r2], &G[(size_t)kk * ld + r2]);
  }
}

// ------------------------------------------------------------------ P(k): L_ik = A_ik U_kk
__global__ void __launch_bounds__(256) k_chol_trsm(int k, const int32_t *__restrict__ panel, int nSp,
                                                   double *__restrict__ L, const double *__restrict__ U) {
  extern __shared__ double sm[];
  double *SA = sm, *SU = sm + TB * TB;   // SA[kk*64 + r] = A_ik[r][kk]; SU[kk*64 + c] = U[kk][c]
  const int i = panel[blockIdx.x], t = threadIdx.x;
  const size_t oik = tile_off(i, k, nSp);
  stage_colmajor(SA, L + oik, nSp);
  stage_colmajor(SU, U + (size_t)k * TB * TB, TB);   // row-major U == k-major operand
  __pipeline_commit();
  __pipeline_wait_prior(0);
  __syncthreads();
  const int tr = t & 15, tc = t >> 4;
  double acc[4][4];
  gemm64(SA, SU, acc, tr, tc);
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int a = 0; a < 4; ++a) L[oik + (size_t)(tc + 16 * b) * nSp + tr + 16 * a] = acc[a][b];
}

// ------------------------------------------------------------------ U(k): A_ij -= L_ik L_jk^T
// Look-ahead: the CTA updating tile (la, la) (la = k + 1) -- or an extra CTA if that tile gets no
// update in this step -- factorises it right away (D(k+1) runs inside U(k)).
__global__ void __launch_bounds__(256) k_chol_update(int k, const int32_t *__restrict__ tasks, int ntasks,
                                                     int la, int nSp, double *__restrict__ L,
                                                     double *__restrict__ U, int *__restrict__ flag) {
  extern __shared__ double sm[];
  if ((int)blockIdx.x >= ntasks) {
    diag_factor(la, nSp, L, U, flag, sm);
    return;
  }
  double *Si = sm, *Sj = sm + TB * TB;
  const int i = tasks[2 * blockIdx.x], j = tasks[2 * blockIdx.x + 1], t = threadIdx.x;
  stage_colmajor(Si, L + tile_off(i, k, nSp), nSp);
  stage_colmajor(Sj, L + tile_off(j, k, nSp), nSp);
  __pipeline_commit();
  const int tr = t & 15, tc = t >> 4;
  const size_t oij = tile_off(i, j, nSp);
  double old[4][4];
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int a = 0; a < 4; ++a) old[a][b] = L[oij + (size_t)(tc + 16 * b) * nSp + tr + 16 * a];
  __pipeline_wait_prior(0);
  __syncthreads();
  double acc[4][4];
  gemm64(Si, Sj, acc, tr, tc);
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r = tr + 16 * a, c = tc + 16 * b;
      if (i != j || r >= c) L[oij + (size_t)c * nSp + r] = old[a][b] - acc[a][b];
    }
  if (i == la && j == la) {
    __syncthreads();
    diag_factor(la, nSp, L, U, flag, sm);
  }
}

// ------------------------------------------------------------------ dataflow factorisation
// One cooperative launch runs the whole tile DAG: tasks are handed out in (topological) task
// order through an atomic counter to whichever CTA is free; a task waits only on tasks that
// precede it, so the earliest unfinished task is always runnable (all CTAs are co-resident).
// Tasks:
//   D(k):     wait upd[k][k] == need;         factor + invert the diagonal tile;   dfl[k] = 1
//   P(i,k):   wait dfl[k], upd[i][k] == need; L_ik = A_ik U_kk;                     pfl[i][k] = 1
//   U(i,j,k): wait pfl[i][k], pfl[j][k], upd[i][j] == rank (updates of a tile are applied in
//             step order -> deterministic);  A_ij -= L_ik L_jk^T;               upd[i][j] = rank + 1
// Tile data produced by other CTAs is read through L2 only (cp.async.cg / ld.global.cg).
#ifdef MSIM_DF_PROF   // diagnostics: global-timer stamps of the critical-path (type-4) tasks
__device__ unsigned long long g_df_prof[1024][8];
#define DF_STAMP(i, s)                                                              \
  do {                                                                              \
    if (threadIdx.x == 0) {                                                         \
      unsigned long long tt;                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                        \
      g_df_prof[(i) & 1023][s] = tt;                                                \
    }                                                                               \
  } while (0)
#else
#define DF_STAMP(i, s)
#endif

__device__ __forceinline__ void df_wait(const int *p, int val) {
  if (threadIdx.x == 0) {
    const volatile int *f = p;
    while (*f != val) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void df_signal(int *p, int val) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicExch(p, val);
  }
}

#ifndef MSIM_DF_MINB
#define MSIM_DF_MINB 2
#endif
__global__ void __launch_bounds__(256, MSIM_DF_MINB) k_chol_dataflow(int ntask, const int4 *__restrict__ tasks, int NT, int nSp,
                                                       double *__restrict__ L, double *__restrict__ U,
                                                       int *__restrict__ upd, int *__restrict__ dfl,
                                                       int *__restrict__ pfl, int *__restrict__ flag,
                                                       int *__restrict__ next) {
  extern __shared__ double sm[];
  __shared__ int s_id;
  const int t = threadIdx.x, tr = t & 15, tc = t >> 4;
  for (;;) {
    // dynamic in-order dispensing: the next unclaimed task in topological order goes to the
    // first CTA that is free (all earlier tasks are claimed by running CTAs -> no deadlock)
    if (t == 0) s_id = atomicAdd(next, 1);
    __syncthreads();
    const int id = s_id;
    __syncthreads();
    if (id >= ntask) break;
    const int4 tk = tasks[id];
    const int type = tk.x, i = tk.y, j = tk.z & 0xffff, k = tk.z >> 16, cnt = tk.w;
    if (type == 0) {
      df_wait(&upd[k * NT + k], cnt);
      diag_factor(k, nSp, L, U, flag, sm);
      df_signal(&dfl[k], 1);
    } else if (type == 4) {
      // critical-path task of step k (i = k+1): P(i,k), U(i,i,k) and D(i) in one CTA.
      // cnt = updates tile (i,k) must have seen; tk.w >> 16 unused; rank of (i,i) is upd order
      DF_STAMP(i, 0);
      // everything that does not depend on D(k) is fetched before waiting for it: A_ik (its
      // updates are done) and the diagonal tile A_ii (its earlier updates are done)
      double *SA = sm, *SU = sm + TB * TB;
      const size_t oik = tile_off(i, k, nSp), oii = tile_off(i, i, nSp);
      df_wait(&upd[i * NT + k], cnt & 0xffff);
      DF_STAMP(i, 6);
      stage_colmajor(SA, L + oik, nSp);
      asm volatile("cp.async.commit_group;\n" ::);
      df_wait(&upd[i * NT + i], cnt >> 16);
      DF_STAMP(i, 7);
      double old[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int r, c;
        tile_rc(q, r, c);
        old[q] = __ldcg(&L[oii + (size_t)c * nSp + r]);
      }
      df_wait(&dfl[k], 1);
      DF_STAMP(i, 1);
      stage_colmajor(SU, U + (size_t)k * TB * TB, TB);
      cp_async_commit_wait();
      __syncthreads();
      double acc[16];
      tile_gemm(SA, SU, acc);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int r, c;
        tile_rc(q, r, c);
        __stcg(&L[oik + (size_t)c * nSp + r], acc[q]);
      }
      df_signal(&pfl[i * NT + k], 1);             // panel tile published early for the other updates
      DF_STAMP(i, 2);
      // X = L_ik into k-major smem: SX[c*64 + r] = X[r][c]
      double *SX = sm;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int r, c;
        tile_rc(q, r, c);
        SX[c * TB + r] = acc[q];
      }
      DF_STAMP(i, 3);
      __syncthreads();
      tile_gemm(SX, SX, acc);
      __syncthreads();   // SX consumed: the updated tile goes straight into D's smem layout
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int r, c;
        tile_rc(q, r, c);
        sm[r * LD + c] = r >= c ? old[q] - acc[q] : 0.0;
      }
      DF_STAMP(i, 4);
      diag_factor(i, nSp, L, U, flag, sm, true);
      df_signal(&dfl[i], 1);
      df_signal(&upd[i * NT + i], (cnt >> 16) + 1);
      DF_STAMP(i, 5);
    } else if (type == 1) {
      df_wait(&dfl[k], 1);
      df_wait(&upd[i * NT + k], cnt);
      double *SA = sm, *SU = sm + TB * TB;
      const size_t oik = tile_off(i, k, nSp);
      stage_colmajor(SA, L + oik, nSp);
      stage_colmajor(SU, U + (size_t)k * TB * TB, TB);
      cp_async_commit_wait();
      __syncthreads();
      double acc[16];
      tile_gemm(SA, SU, acc);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int r, c;
        tile_rc(q, r, c);
        __stcg(&L[oik + (size_t)c * nSp + r], acc[q]);
      }
      df_signal(&pfl[i * NT + k], 1);
    } else {
      df_wait(&pfl[i * NT + k], 1);
      df_wait(&pfl[j * NT + k], 1);
      double *Si = sm, *Sj = sm + TB * TB;
      stage_colmajor(Si, L + tile_off(i, k, nSp), nSp);
      stage_colmajor(Sj, L + tile_off(j, k, nSp), nSp);
      df_wait(&upd[i * NT + j], cnt);
      const size_t oij = tile_off(i, j, nSp);
      double old[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int r, c;
        tile_rc(q, r, c);
        old[q] = __ldcg(&L[oij + (size_t)c * nSp + r]);
      }
      cp_async_commit_wait();
      __syncthreads();
      double acc[16];
      tile_gemm(Si, Sj, acc);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int r, c;
        tile_rc(q, r, c);
        if (i != j || r >= c) __stcg(&L[oij + (size_t)c * nSp + r], old[q] - acc[q]);
      }
      if (type == 3) {   // fused U(k+1,k+1,k) + D(k+1): the updated diagonal tile is factorised at once
        __syncthreads();
        diag_factor(i, nSp, L, U, flag, sm);
        df_signal(&dfl[i], 1);
      }
      df_signal(&upd[i * NT + j], cnt + 1);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_zero_tiles(const int32_t *__restrict__ tiles, int nSp, double *__restrict__ L) {
  const int ti = tiles[2 * blockIdx.x], tj = tiles[2 * blockIdx.x + 1];
  const size_t off = tile_off(ti, tj, nSp);
#pragma unroll
  for (int it = 0; it < 16; ++it) {
    const int e = threadIdx.x + it * 256;
    L[off + (size_t)(e >> 6) * nSp + (e & 63)] = 0.0;
  }
}

__global__ void k_pad_identity2(int nS, int nSp, double *__restrict__ L) {
  const int r = nS + blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nSp) L[(size_t)r * nSp + r] = 1.0;
}

// z_perm[12 perm[i] + r] = z[12 i + r]  (dir = 0);  z[12 i + r] = z_perm[12 perm[i] + r]  (dir = 1)
__global__ void k_permute2(int m, const int32_t *__restrict__ perm, const double *__restrict__ src,
                           double *__restrict__ dst, int dir) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 12 * m) return;
  const int i = t / 12, r = t % 12;
  if (dir == 0) dst[12 * perm[i] + r] = src[t];
  else dst[t] = src[12 * perm[i] + r];
}

// ------------------------------------------------------------------ cooperative solves
__device__ __forceinline__ void wait_flag(const int *flags, int idx) {
  if (threadIdx.x == 0) {
    const volatile int *f = flags + idx;
    while (*f == 0) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void set_flag(int *flags, int idx) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicExch(flags + idx, 1);
  }
}

// The solution vectors double as their own ready flags: they are filled with the all-ones bit
// pattern (a NaN payload arithmetic never produces) before the launch, and a consumer thread
// polls its element of tile j through L2 until it changes (one L2 round trip per dependency
// instead of flag + fence + data).
__device__ __forceinline__ double poll_ready(const double *p) {
  unsigned long long bits;
  for (;;) {
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(bits) : "l"(p));
    if (bits != ~0ull) break;
    __nanosleep(20);
  }
  return __longlong_as_double((long long)bits);
}

// forward: y_k = L_kk^-1 (b_k - sum_{j in rows(k)} L_kj y_j); tiles owned round-robin by CTAs
__global__ void __launch_bounds__(256) k_chol_fwd(int NT, const int32_t *__restrict__ rows_ptr,
                                                  const int32_t *__restrict__ rows, int nSp,
                                                  const double *__restrict__ L, const double *__restrict__ U,
                                                  const double *__restrict__ b, double *__restrict__ y) {
  __shared__ double yj[TB];
  __shared__ double part[4][TB];
  const int t = threadIdx.x, r = t & 63, q = t >> 6;
  for (int k = blockIdx.x; k < NT; k += gridDim.x) {
    // U_kk column r, rows 16q.. (U[c][r] at c*64 + r) and b_k: prefetched off the critical path
    const double *Uk = U + (size_t)k * TB * TB;
    double uv[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) uv[c] = __ldg(&Uk[(size_t)(q * 16 + c) * TB + r]);
    const double bk = t < TB ? b[k * TB + t] : 0.0;
    double acc = 0.0;
    for (int p = rows_ptr[k]; p < rows_ptr[k + 1]; ++p) {
      const int j = rows[p];
      const double *Lkj = L + tile_off(k, j, nSp) + (size_t)(q * 16) * nSp + r;
      double lv[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) lv[c] = Lkj[(size_t)c * nSp];   // prefetch before the wait
      if (t < TB) yj[t] = poll_ready(&y[j * TB + t]);
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 16; ++c) acc = fma(lv[c], yj[q * 16 + c], acc);
      __syncthreads();
    }
    part[q][r] = acc;
    __syncthreads();
    if (t < TB) yj[t] = bk - ((part[0][t] + part[1][t]) + (part[2][t] + part[3][t]));
    __syncthreads();
    // y_k[r] = sum_c Linv[r][c] v[c] = sum_c U[c][r] v[c]
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 16; ++c) s = fma(uv[c], yj[q * 16 + c], s);
    part[q][r] = s;
    __syncthreads();
    if (t < TB) __stcg(&y[k * TB + t], (part[0][t] + part[1][t]) + (part[2][t] + part[3][t]));
    __syncthreads();
  }
}

// backward: x_k = U_kk (y_k - sum_{i in panel(k)} L_ik^T x_i), tiles owned round-robin from the end
__global__ void __launch_bounds__(256) k_chol_bwd(int NT, const int32_t *__restrict__ pan_ptr,
                                                  const int32_t *__restrict__ panel, int nSp,
                                                  const double *__restrict__ L, const double *__restrict__ U,
                                                  const double *__restrict__ y, double *__restrict__ x) {
  __shared__ double xi[TB];
  __shared__ double part[4][TB];
  const int t = threadIdx.x, cidx = t >> 2, q = t & 3;
  for (int s = blockIdx.x; s < NT; s += gridDim.x) {
    const int k = NT - 1 - s;
    // x_k[r] = sum_c U[r][c] v[c] (U row-major: U[r][c] at r*64 + c); thread (r = cidx, q):
    // prefetched with y_k (y is complete: the forward launch finished)
    const double *Uk = U + (size_t)k * TB * TB + (size_t)cidx * TB;
    double uv[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) uv[c] = __ldg(&Uk[q * 16 + c]);
    const double yk = t < TB ? y[k * TB + t] : 0.0;
    double acc = 0.0;   // thread (c = cidx, q): rows 16q..16q+15 of column c
    // largest i first (ready first in the backward sweep); operand prefetched before the wait
    for (int p = pan_ptr[k + 1] - 1; p >= pan_ptr[k]; --p) {
      const int i = panel[p];
      const double *Lik = L + tile_off(i, k, nSp) + (size_t)cidx * nSp + q * 16;
      double lv[16];
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) lv[rr] = Lik[rr];
      if (t < TB) xi[t] = poll_ready(&x[i * TB + t]);
      __syncthreads();
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) acc = fma(lv[rr], xi[q * 16 + rr], acc);
      __syncthreads();
    }
    part[q][cidx] = acc;
    __syncthreads();
    if (t < TB) xi[t] = yk - ((part[0][t] + part[1][t]) + (part[2][t] + part[3][t]));
    __syncthreads();
    double sacc = 0.0;
#pragma unroll
    for (int c = 0; c < 16; ++c) sacc = fma(uv[c], xi[q * 16 + c], sacc);
    part[q][cidx] = sacc;
    __syncthreads();
    if (t < TB) __stcg(&x[k * TB + t], (part[0][t] + part[1][t]) + (part[2][t] + part[3][t]));
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host side
constexpr size_t kDiagSmem = sizeof(double) * kDiagSmemDoubles;
constexpr size_t kGemmSmem = sizeof(double) * 2 * TB * TB;
constexpr size_t kUpdSmem = kDiagSmem > kGemmSmem ? kDiagSmem : kGemmSmem;

void chol_set_attrs() {
  static bool done = false;
  if (done) return;
  MS_CUDA(cudaFuncSetAttribute(k_chol_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiagSmem));
  MS_CUDA(cudaFuncSetAttribute(k_chol_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem));
  MS_CUDA(cudaFuncSetAttribute(k_chol_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpdSmem));
  done = true;
}

void launch_scatter_S(Ctx &c);

static bool step_updates_diag(const Ctx &c, int k) {   // is tile (k+1, k+1) among the tasks of step k?
  const auto &P = c.h_chol_panel[k];
  return !P.empty() && P.front() == k + 1;
}

#ifndef MSIM_DF_PER_SM
#define MSIM_DF_PER_SM 1   // the critical-path CTA gets a whole SM (measured: 3.68 -> 3.25 ms at C4)
#endif
constexpr int kDfCtasPerSm = MSIM_DF_PER_SM;   // CTAs per SM of the dataflow factorisation

static int dataflow_grid(const Ctx &c) {
  static int per_sm = -1;
  if (per_sm < 0) {
    MS_CUDA(cudaFuncSetAttribute(k_chol_dataflow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpdSmem));
    MS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chol_dataflow, 256, kUpdSmem));
    per_sm = std::max(std::min(per_sm, kDfCtasPerSm), 1);
  }
  return (int)std::min<int64_t>(c.n_dag, (int64_t)per_sm * c.coop_grid);
}

// D(0); then for each k: P(k), U(k) with D(k+1) fused (look-ahead) -- or the single-launch
// dataflow version (default)
void enqueue_chol_factor(Ctx &c) {
  const int nSp = c.nS_pad;
  k_zero_tiles<<<(int)c.n_sym_tiles, 256, 0, c.stream>>>(c.sym_tiles, nSp, c.Lden);
  launch_scatter_S(c);
  if (nSp > c.nS) k_pad_identity2<<<div_up(nSp - c.nS, 64), 64, 0, c.stream>>>(c.nS, nSp, c.Lden);
  if (c.chol_dataflow) {
    const int NT = c.ntiles;
    MS_CUDA(cudaMemsetAsync(c.df_flags, 0, sizeof(int) * ((size_t)2 * NT * NT + NT + 1), c.stream));
    int ntask = (int)c.n_dag, NTv = NT, nSpv = nSp;
    const int4 *tk = reinterpret_cast<const int4 *>(c.chol_dag.p);
    double *Lp = c.Lden, *Up = c.Uinv;
    int *upd = c.df_flags, *pfl = c.df_flags + (size_t)NT * NT, *dfl = c.df_flags + (size_t)2 * NT * NT;
    int *fl = c.flags + 0, *nx = c.df_flags + (size_t)2 * NT * NT + NT;
    void *args[] = {&ntask, &tk, &NTv, &nSpv, &Lp, &Up, &upd, &dfl, &pfl, &fl, &nx};
    MS_CUDA(cudaLaunchCooperativeKernel((const void *)k_chol_dataflow, dim3(dataflow_grid(c)), dim3(256), args,
                                        kUpdSmem, c.stream));
#ifdef MSIM_DF_PROF
    {
      static unsigned long long h[1024][8];
      MS_CUDA(cudaStreamSynchronize(c.stream));
      MS_CUDA(cudaMemcpyFromSymbol(h, g_df_prof, sizeof(h)));
      double seg[5] = {0, 0, 0, 0, 0}, gap = 0;
      int n = 0;
      for (int i = 1; i < NT && i < 1024; ++i) {
        for (int q = 0; q < 5; ++q) seg[q] += 1e-3 * (double)(h[i][q + 1] - h[i][q]);
        if (i > 1) gap += 1e-3 * (double)(h[i][1] - h[i - 1][5]);
        n++;
      }
      double wik = 0, wii = 0, wd = 0;
      for (int i = 2; i < NT && i < 1024; ++i) {
        const double t5 = (double)h[i - 1][5];
        wik += 1e-3 * std::max(0.0, (double)h[i][6] - t5);
        wii += 1e-3 * std::max(0.0, (double)h[i][7] - std::max(t5, (double)h[i][6]));
        wd += 1e-3 * std::max(0.0, (double)h[i][1] - std::max(t5, (double)h[i][7]));
      }
      fprintf(stderr, "[msim] chol type-4 avg us: wait %.2f  P %.2f  wait-ii %.2f  U %.2f  D %.2f | ready-after-prev-D %.2f (A_ik %.2f, A_ii %.2f, D %.2f) | total %.1f us\n",
              seg[0] / n, seg[1] / n, seg[2] / n, seg[3] / n, seg[4] / n, gap / n, wik / n, wii / n, wd / n,
              1e-3 * (double)(h[NT - 1][5] - h[1][0]));
    }
#endif
    return;
  }
  k_chol_diag<<<1, 256, kDiagSmem, c.stream>>>(0, nSp, c.Lden, c.Uinv, c.flags + 0);
  for (int k = 0; k < c.ntiles; ++k) {
    const int np = (int)c.h_chol_panel[k].size();
    if (np) k_chol_trsm<<<np, 256, kGemmSmem, c.stream>>>(k, c.chol_panel + c.h_chol_panel_off[k], nSp, c.Lden, c.Uinv);
    const int nt = (int)(c.h_chol_task_off[k + 1] - c.h_chol_task_off[k]);
    const int la = k + 1 < c.ntiles ? k + 1 : -1;
    const int extra = (la >= 0 && !step_updates_diag(c, k)) ? 1 : 0;
    if (nt + extra)
      k_chol_update<<<nt + extra, 256, kUpdSmem, c.stream>>>(k, c.chol_tasks + 2 * c.h_chol_task_off[k], nt, la,
                                                             nSp, c.Lden, c.Uinv, c.flags + 0);
  }
}

int64_t chol_factor_kernels(const Ctx &c) {
  if (c.chol_dataflow) return 3 + (c.nS_pad > c.nS ? 1 : 0);
  int64_t n = 3 + (c.nS_pad > c.nS ? 1 : 0);
  for (int k = 0; k < c.ntiles; ++k) {
    const int nt = (int)(c.h_chol_task_off[k + 1] - c.h_chol_task_off[k]);
    const int extra = (k + 1 < c.ntiles && !step_updates_diag(c, k)) ? 1 : 0;
    n += (c.h_chol_panel[k].empty() ? 0 : 1) + ((nt + extra) ? 1 : 0);
  }
  return n;
}

// solve S q = z in place on c.zs (handle order)
void enqueue_chol_solve(Ctx &c) {
  const int nSp = c.nS_pad, NT = c.ntiles;
  double *b = c.qs, *y = c.yp, *xs = c.xsol;
  MS_CUDA(cudaMemsetAsync(b, 0, sizeof(double) * nSp, c.stream));
  MS_CUDA(cudaMemsetAsync(y, 0xff, sizeof(double) * nSp, c.stream));    // "not ready" pattern
  MS_CUDA(cudaMemsetAsync(xs, 0xff, sizeof(double) * nSp, c.stream));
  k_permute2<<<div_up(12 * c.m, 256), 256, 0, c.stream>>>(c.m, c.perm, c.zs, b, 0);
  const int G = std::min(NT, c.coop_grid);
  {
    int NTv = NT, nSpv = nSp;
    const int32_t *rp = c.chol_rows_ptr, *rw = c.chol_rows;
    const double *Lp = c.Lden, *Up = c.Uinv, *bp = b;
    double *yv = y;
    void *args[] = {&NTv, &rp, &rw, &nSpv, &Lp, &Up, &bp, &yv};
    MS_CUDA(cudaLaunchCooperativeKernel((const void *)k_chol_fwd, dim3(G), dim3(256), args, 0, c.stream));
  }
  {
    int NTv = NT, nSpv = nSp;
    const int32_t *pp = c.chol_panel_ptr, *pw = c.chol_panel;
    const double *Lp = c.Lden, *Up = c.Uinv, *yp = y;
    double *xv = xs;
    void *args[] = {&NTv, &pp, &pw, &nSpv, &Lp, &Up, &yp, &xv};
    MS_CUDA(cudaLaunchCooperativeKernel((const void *)k_chol_bwd, dim3(G), dim3(256), args, 0, c.stream));
  }
  k_permute2<<<div_up(12 * c.m, 256), 256, 0, c.stream>>>(c.m, c.perm, xs, c.zs, 1);
}

int64_t chol_solve_kernels(const Ctx &) { return 4; }

}  // namespace msim
