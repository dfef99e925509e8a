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
#include "galerkin.cuh"

namespace msim {

constexpr int TB = 64;
// shared-memory row strides (doubles) of the diagonal-tile layout and of the k-major staged
// tiles: 68 = 4 (mod 16), so the 8 x 4 fragments of mma.sync m8n8k4 (lanes: 8 rows x 4 k) hit 16
// distinct bank pairs per half-warp -- conflict-free (stride 65 / 64: 4-way)
constexpr int LD = TB + 4;
constexpr int SLD = TB + 4;

__device__ __forceinline__ size_t tile_off(int ti, int tj, int nSp) {
  return (size_t)(tj * TB) * nSp + (size_t)ti * TB;
}

#ifdef MSIM_CHAIN_PROF   // sub-phases of D on the chain CTA (diagnostic build only): stamps in
// shared memory (no global round trip on the panel warp), accumulated at D's end
__device__ long long g_dts[16];
__device__ __forceinline__ long long *diag_ts_buf() {
  __shared__ long long ts[16];
  return ts;
}
#define DIAG_TS(i) do { if (threadIdx.x == 0) diag_ts_buf()[i] = clock64(); } while (0)
#define DIAG_TS_FLUSH() do { if (blockIdx.x == 0 && threadIdx.x == 0) { const long long *b_ = diag_ts_buf(); \
    long long last_ = b_[0]; const int ord_[12] = {10, 1, 2, 11, 3, 4, 12, 5, 6, 13, 7, 9}; \
    for (int q_ = 0; q_ < 12; ++q_) { g_dts[ord_[q_]] += b_[ord_[q_]] - last_; last_ = b_[ord_[q_]]; } } } while (0)
#endif
#include "chol_diag.cuh"

// ------------------------------------------------------------------ tile GEMM of the dataflow kernel
// acc = S1^T S2 over the 64-long k dimension (S1[kk*SLD + r], S2[kk*SLD + c]); thread-owned elements
// idx = 0..15 at (r, c) = tile_rc(idx), on the FP64 tensor cores (mma.sync m8n8k4): warp w owns
// rows 16 (w & 3) .. +15 and columns 32 (w >> 2) .. +31 as 2 x 4 blocks of 8 x 8.

__device__ __forceinline__ void tile_rc(int idx, int &r, int &c) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j = idx & 1, bj = (idx >> 1) & 3, bi = idx >> 3;
  r = 16 * (w & 3) + 8 * bi + (lane >> 2);
  c = 32 * (w >> 2) + 8 * bj + 2 * (lane & 3) + j;
}

// LI: the second operand is a row-major inverse diagonal tile Li [64][LD] left in shared memory
// by diag_factor (S2[kk*SLD + c] = U[kk][c] = Li[c][kk]) instead of a staged k-major tile
template <bool LI = false>
__device__ __forceinline__ void tile_gemm(const double *S1, const double *S2, double (&acc)[16]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r0 = 16 * (w & 3) + (lane >> 2), c0 = 32 * (w >> 2) + (lane >> 2), kl = lane & 3;
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
#pragma unroll 4
  for (int k0 = 0; k0 < TB; k0 += 4) {
    const double *s1 = S1 + (k0 + kl) * SLD, *s2 = S2 + (k0 + kl) * SLD;
    const double a0 = s1[r0], a1 = s1[r0 + 8];
    double b[4];
#pragma unroll
    for (int bj = 0; bj < 4; ++bj) b[bj] = LI ? S2[(c0 + 8 * bj) * LD + k0 + kl] : s2[c0 + 8 * bj];
#pragma unroll
    for (int bi = 0; bi < 2; ++bi)
#pragma unroll
      for (int bj = 0; bj < 4; ++bj)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[(bi * 4 + bj) * 2]), "+d"(acc[(bi * 4 + bj) * 2 + 1])
                     : "d"(bi ? a1 : a0), "d"(b[bj]));
  }
}

// stage a column-major global tile (leading dim nSp) into k-major smem S[kk*SLD + r] (cp.async)
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
    cp_async_cg16(&S[kk * SLD + r2], &G[(size_t)kk * ld + r2]);
  }
}

// ------------------------------------------------------------------ dataflow factorisation
// One cooperative launch runs the whole tile DAG (setup.cpp builds the task list, the counted
// inputs of every task and its successors):
//   CTA 0      the critical chain T(k) = P(k+1,k) + U(k+1,k+1,k) + D(k+1), in order, waiting on
//              flags and prefetching the tiles that do not depend on D(k);
//   CTA 1      release helper: follows CTA 0's flags and hands T(k)'s successors to the queues;
//   CTAs 2..   pop ready tasks from two FIFO queues (high: D, P and updates of tiles that become
//              panel tiles within two steps; low: the bulk updates), each served by its own CTA
//              set through tickets.  A task is pushed by whoever delivers its last input; a CTA
//              that completes a task's last input keeps that task as its next one instead.
// A popped task never waits, CTA 0 waits only on earlier tasks, so the launch cannot deadlock.
// Tasks (the flags serve CTA 0's waits):
//   D(k):     factor + invert the diagonal tile;                       dfl[k] = 1
//   P(i,k):   L_ik = A_ik U_kk;                                          pfl[i][k] = 1
//   U(i,j,k): A_ij -= L_ik L_jk^T (updates of a tile are chained in step order -> deterministic);
//             upd[i][j] = rank + 1
// Tile data produced by other CTAs is read through L2 only (cp.async.cg / ld.global.cg).

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

// two flags with one poll pass, one fence and one barrier
__device__ __forceinline__ void df_wait2(const int *p1, int v1, const int *p2, int v2) {
  if (threadIdx.x == 0) {
    const volatile int *f1 = p1, *f2 = p2;
    while (*f1 != v1) __nanosleep(20);
    while (*f2 != v2) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void df_signal2(int *p1, int v1, int *p2, int v2) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicExch(p1, v1);
    atomicExch(p2, v2);
  }
}

struct DfParams {
  int NT, nSp, ncrit, npool, nhi_cta, qstride, per_sm;
  int *chain_sm;               // SM of CTA 0 + 1 (0: not yet known)
  const int4 *tasks;           // (type, i, j | k << 16, count) per task
  double *L, *U;               // tiled factor / inverse diagonal tiles
  int *upd, *dfl, *pfl, *flag; // progress flags (NT*NT, NT, NT*NT) and the pivot flag
  const int32_t *crit;         // CTA 0's tasks in order
  const uint8_t *cls;          // per task: 0/1 low/high-priority queue, 2 CTA 0's list
  const int32_t *succ_ptr, *succ_mid, *succ;
  int *ndep;                   // counted inputs still missing per task
  int *queue;                  // queue q at q * qstride: [head, tail, task ids (-1: not yet pushed)]
  int *done;                   // queue tasks finished
  // fused Galerkin rows (c.gal_fused): G(i, part) / R(i) tasks; rw_ptr == nullptr otherwise
  GalParams gal;
  const int32_t *perm;         // handle -> position of its 12 rows in the factor
  int *rdone;                  // [m] R(i) finished (chain CTA waits)
  const int32_t *rw_ptr, *rw;  // per chain task: the handles whose R(i) it waits for
};

// successors [b, e) of a finished task: one input fewer each.  A queue task whose last input
// this was is kept by the CTA as its next task if it has none yet (*keep, shared; continuation:
// the per-tile update chains U(i,j,k) -> U(i,j,k') then run back to back without a queue trip)
// or pushed to its class's queue, a FIFO served by tickets (no CAS contention: measured 60 us
// claim latency with 147 CTAs CAS-polling two shared queues).  Called right after the task's
// df_signal (CTA barrier, thread 0's fence); the second barrier orders that fence before the
// other threads' atomics.
__device__ __forceinline__ void df_release(const DfParams &P, int b, int e, int *keep) {
  if (e - b > 1) __syncthreads();
  for (int q = b + (int)threadIdx.x; q < e; q += blockDim.x) {
    const int s = P.succ[q];
    if (atomicSub(&P.ndep[s], 1) == 1) {
      const int c = P.cls[s];
      if (c < 2) {
        if (keep && atomicCAS(keep, -1, s) == -1) {
          __threadfence();   // acquire: the other producers' tiles
        } else {
          int *Q = P.queue + (size_t)c * P.qstride;
          const int slot = atomicAdd(&Q[1], 1);
          atomicExch(&Q[2 + slot], s);
        }
      }
    }
  }
}

// thread 0: ticket on queue Q: wait until the ticket's entry is pushed, or return -1 once every
// queue task has finished (kept tasks never enter a queue, so the entry may never come)
__device__ __forceinline__ int df_pop(int *Q, const int *done, int npool) {
  const int h = atomicAdd(&Q[0], 1);
  const volatile int *qe = Q + 2 + h, *dn = done;
  for (;;) {
    if (h < npool) {
      const int v = *qe;
      if (v >= 0) return v;
    }
    if (*dn >= npool) return -1;
    __nanosleep(32);
  }
}

#ifndef MSIM_DF_MINB
#define MSIM_DF_MINB 2
#endif
// -DMSIM_CHAIN_PROF: CTA 0 accumulates clock64 deltas of the phases of its chain tasks and prints
// them at the end of the launch (diagnostic build only)
#ifdef MSIM_CHAIN_PROF
#define CHAIN_TS(q) do { if (t == 0) { const long long now_ = clock64(); prof[q] += now_ - prof_last; prof_last = now_; } } while (0)
#else
#define CHAIN_TS(q)
#endif
__global__ void __launch_bounds__(256, MSIM_DF_MINB) k_chol_dataflow(const DfParams P) {
  extern __shared__ double sm[];
#ifdef MSIM_CHAIN_PROF
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0}, prof_last = clock64();
  int prof_n = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int q = 0; q < 16; ++q) g_dts[q] = 0;
#endif
  __shared__ int s_id, s_keep;
  const int t = threadIdx.x;
  if (t == 0) s_keep = -1;
  __syncthreads();
  const int NT = P.NT, nSp = P.nSp;
  double *__restrict__ L = P.L;
  double *__restrict__ U = P.U;
  int *upd = P.upd, *dfl = P.dfl, *pfl = P.pfl, *flag = P.flag;
  if (P.per_sm > 1) {
    // several CTAs per SM: the chain CTA keeps its SM to itself (a queue CTA that lands on the
    // same SM leaves at once; measured: sharing it cost more than the extra queue CTAs gained)
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (blockIdx.x == 0) {
      if (t == 0) atomicExch(P.chain_sm, (int)smid + 1);
    } else if (blockIdx.x >= 2) {
      if (t == 0) {
        const volatile int *f = P.chain_sm;
        int v;
        while ((v = *f) == 0) __nanosleep(32);
        s_id = v - 1 == (int)smid;
      }
      __syncthreads();
      if (s_id) return;
    }
  }
  if (blockIdx.x == 1) {
    // release helper: follows the chain and hands the successors of each chain task to the
    // queues as its flags appear, so that CTA 0 never spends the atomics' round trips (measured
    // ~2 us per release, twice per chain step)
    for (int q = 0; q < P.ncrit; ++q) {
      const int id = P.crit[q];
      const int4 tk = P.tasks[id];
      const int i = tk.y, k = tk.z >> 16;
      df_wait(&pfl[i * NT + k], 1);
      df_release(P, P.succ_ptr[id], P.succ_mid[id], nullptr);
      df_wait2(&dfl[i], 1, &upd[i * NT + i], (tk.w >> 16) + 1);
      df_release(P, P.succ_mid[id], P.succ_ptr[id + 1], nullptr);
      __syncthreads();
    }
    return;
  }
  int ccur = 0, my_d = -1;
  for (;;) {
    // (measured at C4: in-order dispensing from one counter left tasks 10-17 us unclaimed after
    // their inputs were done -- 1.3 of 3.0 ms on the critical path)
    int id;
    if (blockIdx.x == 0) {
      if (ccur >= P.ncrit) break;
      id = P.crit[ccur++];
    } else {
      if (t == 0) {
        if (s_keep >= 0) {
          s_id = s_keep;
          s_keep = -1;
        } else {
          const int c = blockIdx.x <= P.nhi_cta + 1 ? 1 : 0;   // CTAs 2..nhi_cta+1: high queue
          s_id = df_pop(P.queue + (size_t)c * P.qstride, P.done, P.npool);
          __threadfence();
        }
      }
      __syncthreads();
      id = s_id;
      __syncthreads();
      if (id < 0) break;
    }
    const int4 tk = P.tasks[id];
    const int type = tk.x, i = tk.y, j = tk.z & 0xffff, k = tk.z >> 16, cnt = tk.w;
    if (type == 0) {   // popped from the ready queue: its inputs are done
      (void)cnt;
      diag_factor(k, nSp, L, U, flag, sm);
      df_signal(&dfl[k], 1);
      df_release(P, P.succ_ptr[id], P.succ_ptr[id + 1], &s_keep);
    } else if (type == 4) {
      // critical-path task of step k (i = k+1): P(i,k), U(i,i,k) and D(i) in one CTA.
      // cnt = updates tile (i,k) must have seen; tk.w >> 16 unused; rank of (i,i) is upd order
      // everything that does not depend on D(k) is fetched before waiting for it: A_ik (its
      // updates are done) and the diagonal tile A_ii (its earlier updates are done)
      double *SA = sm, *SU = sm + TB * SLD;
      const size_t oik = tile_off(i, k, nSp), oii = tile_off(i, i, nSp);
      CHAIN_TS(0);   // between chain tasks
      if (P.rw_ptr)   // fused Galerkin: the rows of S this task reads unfactored
        for (int q2 = P.rw_ptr[ccur - 1]; q2 < P.rw_ptr[ccur]; ++q2) df_wait(&P.rdone[P.rw[q2]], 1);
      df_wait2(&upd[i * NT + k], cnt & 0xffff, &upd[i * NT + i], cnt >> 16);
      CHAIN_TS(1);   // waiting for the inputs' updates
      stage_colmajor(SA, L + oik, nSp);
      asm volatile("cp.async.commit_group;\n" ::);
      double old[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int r, c;
        tile_rc(q, r, c);
        old[q] = __ldcg(&L[oii + (size_t)c * nSp + r]);
      }
      // D(k) is usually this CTA's previous task: its inverse is still in shared memory
      const bool own_d = k == my_d;
      if (!own_d) df_wait(&dfl[k], 1);
      if (!own_d) stage_colmajor(SU, U + (size_t)k * TB * TB, TB);
      cp_async_commit_wait();
      __syncthreads();
      CHAIN_TS(2);   // staging A_ik, A_ii (and U_kk)
      double acc[16];
      if (own_d) tile_gemm<true>(SA, sm + TB * LD, acc);
      else tile_gemm(SA, SU, acc);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int r, c;
        tile_rc(q, r, c);
        __stcg(&L[oik + (size_t)c * nSp + r], acc[q]);
      }
      df_signal(&pfl[i * NT + k], 1);             // panel tile published early for the other updates
      CHAIN_TS(3);   // P(i,k) GEMM + stores
      // X = L_ik into k-major smem: SX[c*SLD + r] = X[r][c]
      double *SX = sm;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int r, c;
        tile_rc(q, r, c);
        SX[c * SLD + r] = acc[q];
      }
      __syncthreads();
      tile_gemm(SX, SX, acc);
      __syncthreads();   // SX consumed: the updated tile goes straight into D's smem layout
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int r, c;
        tile_rc(q, r, c);
        sm[r * LD + c] = r >= c ? old[q] - acc[q] : 0.0;
      }
      CHAIN_TS(4);   // U(i,i,k) GEMM
      diag_factor(i, nSp, L, U, flag, sm, true);
      CHAIN_TS(5);   // D(i)
      df_signal2(&dfl[i], 1, &upd[i * NT + i], (cnt >> 16) + 1);
      my_d = i;
      CHAIN_TS(6);
#ifdef MSIM_CHAIN_PROF
      ++prof_n;
#endif
    } else if (type == 5) {
      // G(i, part): a quarter of handle i's Galerkin row into its partial row (galerkin.cuh)
      galerkin_row(P.gal, i, j, sm);
      if (t == 0) __threadfence();   // the partial row before R(i) is released
      __syncthreads();
      df_release(P, P.succ_ptr[id], P.succ_ptr[id + 1], &s_keep);
    } else if (type == 6) {
      // R(i): the parts summed in a fixed order, scattered into the factor's tiles
      galerkin_reduce_to_tiles(P.gal, i, P.perm, nSp, L);
      df_signal(&P.rdone[i], 1);
      df_release(P, P.succ_ptr[id], P.succ_ptr[id + 1], &s_keep);
    } else if (type == 1) {
      double *SA = sm, *SU = sm + TB * SLD;
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
      df_release(P, P.succ_ptr[id], P.succ_ptr[id + 1], &s_keep);

    } else {
      double *Si = sm, *Sj = sm + TB * SLD;
      stage_colmajor(Si, L + tile_off(i, k, nSp), nSp);
      stage_colmajor(Sj, L + tile_off(j, k, nSp), nSp);

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
      df_signal(&upd[i * NT + j], cnt + 1);
      df_release(P, P.succ_ptr[id], P.succ_ptr[id + 1], &s_keep);

    }
    __syncthreads();
    if (t == 0 && type != 4) atomicAdd(P.done, 1);   // after this task's pushes (barrier above)
  }
#ifdef MSIM_CHAIN_PROF
  if (blockIdx.x == 0 && t == 0 && prof_n > 0)
    printf("chain tasks %d  cycles/task: gap %lld wait %lld stage %lld P %lld U %lld D %lld signal %lld\n", prof_n,
           prof[0] / prof_n, prof[1] / prof_n, prof[2] / prof_n, prof[3] / prof_n, prof[4] / prof_n, prof[5] / prof_n,
           prof[6] / prof_n);
  if (blockIdx.x == 0 && t == 0 && prof_n > 0)
    printf("D sub-phases: panel0 %lld sync %lld trail0 %lld | panel1 %lld sync %lld trail1 %lld | panel2 %lld sync %lld "
           "trail2 %lld | panel3 %lld sync %lld last %lld\n", g_dts[10] / prof_n, g_dts[1] / prof_n, g_dts[2] / prof_n,
           g_dts[11] / prof_n, g_dts[3] / prof_n, g_dts[4] / prof_n, g_dts[12] / prof_n, g_dts[5] / prof_n,
           g_dts[6] / prof_n, g_dts[13] / prof_n, g_dts[7] / prof_n, g_dts[9] / prof_n);
#endif
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
                           double *__restrict__ dst, int dir, const int32_t *__restrict__ skip) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 12 * m || (skip && *skip)) return;
  const int i = t / 12, r = t % 12;
  if (dir == 0) dst[12 * perm[i] + r] = src[t];
  else dst[t] = src[12 * perm[i] + r];
}

// solve set-up: b = permuted z (padding rows 0), y and x filled with the "not ready" pattern
__global__ void k_solve_prep(int m, int nSp, const int32_t *__restrict__ perm, const double *__restrict__ z,
                             double *__restrict__ b, double *__restrict__ y, double *__restrict__ x,
                             const int32_t *__restrict__ skip) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nSp || (skip && *skip)) return;
  const double nr = __longlong_as_double(-1ll);
  y[t] = nr;
  x[t] = nr;
  if (t < 12 * m) b[12 * perm[t / 12] + t % 12] = z[t];
  else b[t] = 0.0;
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
                                                  const double *__restrict__ b, double *__restrict__ y,
                                                  const int32_t *__restrict__ skip) {
  if (skip && *skip) return;   // uniform over the grid (two-level PCG after convergence)
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

// backward: x_k = U_kk (y_k - sum_{i in panel(k)} L_ik^T x_i), tiles owned round-robin from the end.
// Thread (r, q) reads row r, columns 16q..16q+15 of each L_ik (consecutive lanes: consecutive
// rows of a column-major tile -> coalesced) and keeps 16 column partial sums across all i; the
// rows are reduced once per tile.  (Thread-per-column reads were uncoalesced: 3.3 us per sweep
// step against 1.15 for the forward sweep, which has the coalesced pattern.)
__global__ void __launch_bounds__(256) k_chol_bwd(int NT, const int32_t *__restrict__ pan_ptr,
                                                  const int32_t *__restrict__ panel, int nSp,
                                                  const double *__restrict__ L, const double *__restrict__ U,
                                                  const double *__restrict__ y, double *__restrict__ x,
                                                  const int32_t *__restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double xi[TB];
  __shared__ double part[4][TB];
  __shared__ double red[TB][TB + 1];
  const int t = threadIdx.x, r = t & 63, q = t >> 6;
  for (int s = blockIdx.x; s < NT; s += gridDim.x) {
    const int k = NT - 1 - s;
    // x_k[r] = sum_c U[r][c] v[c] (U row-major: U[r][c] at r*64 + c): prefetched with y_k
    const double *Uk = U + (size_t)k * TB * TB + (size_t)r * TB + q * 16;
    double uv[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) uv[c] = __ldg(&Uk[c]);
    const double yk = t < TB ? y[k * TB + t] : 0.0;
    double acc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] = 0.0;
    // largest i first (ready first in the backward sweep); operand prefetched before the wait
    for (int p = pan_ptr[k + 1] - 1; p >= pan_ptr[k]; --p) {
      const int i = panel[p];
      const double *Lik = L + tile_off(i, k, nSp) + (size_t)(q * 16) * nSp + r;
      double lv[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) lv[c] = Lik[(size_t)c * nSp];
      if (t < TB) xi[t] = poll_ready(&x[i * TB + t]);
      __syncthreads();
      const double xr = xi[r];
#pragma unroll
      for (int c = 0; c < 16; ++c) acc[c] = fma(lv[c], xr, acc[c]);
      __syncthreads();
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) red[r][q * 16 + c] = acc[c];
    __syncthreads();
    {   // column sums: thread (column r, row quarter q)
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) s4[rr & 3] += red[q * 16 + rr][r];
      part[q][r] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    }
    __syncthreads();
    if (t < TB) xi[t] = yk - ((part[0][t] + part[1][t]) + (part[2][t] + part[3][t]));
    __syncthreads();
    double sacc = 0.0;
#pragma unroll
    for (int c = 0; c < 16; ++c) sacc = fma(uv[c], xi[q * 16 + c], sacc);
    part[q][r] = sacc;
    __syncthreads();
    if (t < TB) __stcg(&x[k * TB + t], (part[0][t] + part[1][t]) + (part[2][t] + part[3][t]));
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host side
constexpr size_t kDiagSmem = sizeof(double) * kDiagSmemDoubles;
constexpr size_t kGemmSmem = sizeof(double) * 2 * TB * SLD;
constexpr size_t kUpdSmem = kDiagSmem > kGemmSmem ? kDiagSmem : kGemmSmem;

#ifndef MSIM_DF_PER_SM
#define MSIM_DF_PER_SM 2   // two queue CTAs per SM, the chain CTA alone on its SM (measured at C4:
                           // 2.82 -> 2.50 ms; sharing the chain's SM made two per SM slower)
#endif
constexpr int kDfCtasPerSm = MSIM_DF_PER_SM;   // CTAs per SM of the dataflow factorisation

// Large-shared-memory opt-ins are per device: set once per context, on its device, right
// after cudaSetDevice (create_common); the occupancy-derived CTA count is kept in the context.
void chol_init_attrs(Ctx &c) {
  set_max_dyn_smem((const void *)k_chol_dataflow, c.device);
  int per_sm = 0;
  MS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chol_dataflow, 256, kUpdSmem));
  const char *e = std::getenv("MSIM_DF_PER_SM");
  c.df_per_sm = std::max(std::min(per_sm, e ? std::atoi(e) : kDfCtasPerSm), 1);
}

void launch_scatter_S(Ctx &c);



static int dataflow_grid(const Ctx &c) {
  const int per_sm = c.df_per_sm;
  // the chain CTA, the release helper, at least one CTA per queue
  return (int)std::max<int64_t>(4, (int64_t)per_sm * c.coop_grid);
}

// the whole factorisation as one cooperative dataflow launch (zeroed tiles + scattered S first)
void enqueue_chol_factor(Ctx &c) {
  const int nSp = c.nS_pad;
  k_zero_tiles<<<(int)c.n_sym_tiles, 256, 0, c.stream>>>(c.sym_tiles, nSp, c.Lden);
  launch_scatter_S(c);
  if (nSp > c.nS) k_pad_identity2<<<div_up(nSp - c.nS, 64), 64, 0, c.stream>>>(c.nS, nSp, c.Lden);
  {
    const int NT = c.ntiles;
    MS_CUDA(cudaMemsetAsync(c.df_flags, 0, sizeof(int) * c.df_flags.n, c.stream));
    MS_CUDA(cudaMemcpyAsync(c.chol_ndep.p, c.chol_ndep0.p, sizeof(int32_t) * c.chol_ndep0.n,
                            cudaMemcpyDeviceToDevice, c.stream));
    MS_CUDA(cudaMemcpyAsync(c.chol_queue.p, c.chol_queue0.p, sizeof(int32_t) * c.chol_queue0.n,
                            cudaMemcpyDeviceToDevice, c.stream));
    DfParams prm;
    prm.NT = NT;
    prm.nSp = nSp;
    prm.ncrit = (int)c.n_crit;
    prm.npool = (int)c.n_pool;
    prm.qstride = (int)c.n_pool + 2;
    prm.nhi_cta = std::max(1, std::min(c.df_hi_ctas, dataflow_grid(c) - 3));
    prm.tasks = reinterpret_cast<const int4 *>(c.chol_dag.p);
    prm.L = c.Lden;
    prm.U = c.Uinv;
    prm.upd = c.df_flags;
    prm.pfl = c.df_flags + (size_t)NT * NT;
    prm.dfl = c.df_flags + (size_t)2 * NT * NT;
    prm.flag = c.flags + 0;
    prm.crit = c.chol_crit;
    prm.cls = c.chol_cls;
    prm.succ_ptr = c.chol_succ_ptr;
    prm.succ = c.chol_succ;
    prm.succ_mid = c.chol_succ_mid;
    prm.ndep = c.chol_ndep;
    prm.queue = c.chol_queue;
    prm.done = c.chol_queue + 2 * prm.qstride;
    prm.per_sm = c.df_per_sm;
    prm.chain_sm = c.df_flags + (size_t)2 * NT * NT + NT;   // zeroed with the flags
    size_t smem = kUpdSmem;
    if (c.gal_fused) {
      prm.gal = galerkin_params(c);
      prm.perm = c.perm;
      prm.rdone = c.df_flags + (size_t)2 * NT * NT + NT + 1;
      prm.rw_ptr = c.chol_rw_ptr;
      prm.rw = c.chol_rw;
      smem = std::max(smem, sizeof(double) * galerkin_smem_doubles(c.gal_max_jup));
    } else {
      prm.perm = nullptr;
      prm.rdone = nullptr;
      prm.rw_ptr = prm.rw = nullptr;
    }
    void *args[] = {&prm};
    MS_CUDA(cudaLaunchCooperativeKernel((const void *)k_chol_dataflow, dim3(dataflow_grid(c)), dim3(256), args,
                                        smem, c.stream));
  }
}

int64_t chol_factor_kernels(const Ctx &c) { return 3 + (c.nS_pad > c.nS ? 1 : 0); }

// solve S q = z in place on c.zs (handle order); skip (device flag, may be NULL): every launch
// does nothing while *skip != 0
void enqueue_chol_solve(Ctx &c, const int32_t *skip) {
  const int nSp = c.nS_pad, NT = c.ntiles;
  double *b = c.qs, *y = c.yp, *xs = c.xsol;
  k_solve_prep<<<div_up(nSp, 256), 256, 0, c.stream>>>(c.m, nSp, c.perm, c.zs, b, y, xs, skip);
  const int G = std::min(NT, c.coop_grid);
  {
    int NTv = NT, nSpv = nSp;
    const int32_t *rp = c.chol_rows_ptr, *rw = c.chol_rows, *sk = skip;
    const double *Lp = c.Lden, *Up = c.Uinv, *bp = b;
    double *yv = y;
    void *args[] = {&NTv, &rp, &rw, &nSpv, &Lp, &Up, &bp, &yv, &sk};
    MS_CUDA(cudaLaunchCooperativeKernel((const void *)k_chol_fwd, dim3(G), dim3(256), args, 0, c.stream));
  }
  {
    int NTv = NT, nSpv = nSp;
    const int32_t *pp = c.chol_panel_ptr, *pw = c.chol_panel, *sk = skip;
    const double *Lp = c.Lden, *Up = c.Uinv, *yp = y;
    double *xv = xs;
    void *args[] = {&NTv, &pp, &pw, &nSpv, &Lp, &Up, &yp, &xv, &sk};
    MS_CUDA(cudaLaunchCooperativeKernel((const void *)k_chol_bwd, dim3(G), dim3(256), args, 0, c.stream));
  }
  k_permute2<<<div_up(12 * c.m, 256), 256, 0, c.stream>>>(c.m, c.perm, xs, c.zs, 1, skip);
}

int64_t chol_solve_kernels(const Ctx &) { return 4; }

}  // namespace msim
