// Galerkin block row of S = B^T H B (Eq. 7):
// one CTA per handle row (coarse.cu k_galerkin_fused).
#pragma once
#include "common.cuh"

namespace msim {

struct HView {                      // SELL-32 Hessian (sell.cuh)
  const int32_t *__restrict__ sl_ptr;
  const int32_t *__restrict__ col;
  const double *__restrict__ vals;
};

struct GalParams {
  HView H;
  const int32_t *gU_ptr, *gU, *ga_off;
  const uint32_t *ga_ent;
  const unsigned long long *ga_mask;
  const int32_t *gj_ptr, *gj_blk, *gl_base, *gl_off;
  const uint32_t *gl_ent;
  const double *W;
  const double *ga_w, *gl_w;        // W rows per list entry (nullable: gather through the index)
  const int32_t *sT;
  const int32_t *scol;              // S pattern columns (handle j of block b)
  double *S;                        // [nnzb_S][144] block storage
  double *Spart;                    // [m * nparts][pstride] partial rows (nparts > 1)
  int nparts, pstride;
};


GalParams galerkin_params(const Ctx &c);
HView hview(const Ctx &c);
constexpr int kGalWarps = kGalThreads / 32;


// One CTA per handle i computes the upper block row S_ij (j >= i) with R_i never leaving the
// SM.  For each chunk of kGalChunk vertices u of U_i:
//   phase A (two threads per u, even / odd Hessian row slots, summed in a fixed order):
//            R_i(u) = sum_{v in N(u), i in supp(v)} w_vi kron H_vu   -> shared Rs[u][36]
//   phase B (warp per upper slot j): S_ij += sum_{u in chunk, j in supp(u)} R_i(u) w_uj^T; the
//            warp stages 32 list entries (u, w_uj) at a time in shared memory (one round trip
//            per 32 entries); three 9-lane groups work on three entries at once.
// Every accumulator has one owner thread and a fixed summation order -> deterministic.
// R_i(u) entry l = 3 (4c'+k') + c; accumulator layout [slot][k][36] (conflict-free in l).

// Part `part` of `nparts` of handle i's row: the contiguous chunk range
// [part nch / nparts, (part + 1) nch / nparts) of U_i (vertex order, so the CTAs resident at one
// time -- consecutive handles, all parts -- work on one x-slab of the mesh and share H rows in L2).
// nparts == 1 writes S directly; otherwise the partial row goes to Spart and k_galerkin_reduce
// sums the parts in a fixed order.
__device__ __forceinline__ void galerkin_row(const GalParams &G, int i, int part, double *gsm) {
  const HView &H = G.H;
  const int32_t *__restrict__ gU_ptr = G.gU_ptr, *__restrict__ gU = G.gU, *__restrict__ ga_off = G.ga_off;
  const uint32_t *__restrict__ ga_ent = G.ga_ent;
  const unsigned long long *__restrict__ ga_mask = G.ga_mask;
  const int32_t *__restrict__ gj_ptr = G.gj_ptr, *__restrict__ gj_blk = G.gj_blk, *__restrict__ gl_base = G.gl_base;
  const int32_t *__restrict__ gl_off = G.gl_off;
  const uint32_t *__restrict__ gl_ent = G.gl_ent;
  const double *__restrict__ W = G.W;
  const int32_t *__restrict__ sT = G.sT;
  double *__restrict__ S = G.S;

  double *Rs = gsm;                                   // [kGalChunk][36]
  double *stW = Rs + kGalChunk * 36;                  // [warps][32][4]
  int *stU = reinterpret_cast<int *>(stW + kGalWarps * 32 * 4);   // [warps][32]
  double *Sacc = stW + kGalWarps * 32 * 4 + kGalWarps * 16;       // [nup][4][36]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ul_a = t & (kGalChunk - 1), half = t / kGalChunk;
  const int u0 = gU_ptr[i], nU = gU_ptr[i + 1] - u0;
  const int j0 = gj_ptr[i], nup = gj_ptr[i + 1] - j0;
  for (int e = t; e < nup * 144; e += kGalThreads) Sacc[e] = 0.0;
  const int nch = (nU + kGalChunk - 1) / kGalChunk;
  const int ch0 = (int)((int64_t)part * nch / G.nparts), ch1 = (int)((int64_t)(part + 1) * nch / G.nparts);
  const int *off = gl_off + gl_base[i];
  double *myW = stW + warp * 128;
  int *myU = stU + warp * 32;
  for (int ch = ch0; ch < ch1; ++ch) {
    // ---- phase A
    double acc[36];
#pragma unroll
    for (int k = 0; k < 36; ++k) acc[k] = 0.0;
    const int uq = ch * kGalChunk + ul_a;
#ifdef MSIM_GAL_SKIP_A   // timing diagnostics only (wrong results): phase B alone
    if (false) {
#else
    if (uq < nU) {
#endif
      // slot-synchronous walk of row u: lanes of a warp (consecutive u of one SELL slice) read
      // the same slot j together (coalesced value planes); the two halves take even / odd slots
      const int q = u0 + uq;
      const int u = __ldg(&gU[q]);
      const int ln_ = u & 31;
      const int base = __ldg(&H.sl_ptr[u >> 5]), len = __ldg(&H.sl_ptr[(u >> 5) + 1]) - base;
      const unsigned long long mask = __ldg(&ga_mask[q]);
      const int e0 = __ldg(&ga_off[q]);
#pragma unroll 2
      for (int j = half; j < len; j += 2) {
        if (!((mask >> j) & 1ull)) continue;
        const int ea = e0 + __popcll(mask & ((1ull << j) - 1ull));
        const size_t cs = (size_t)base + j;
        const double *wp = G.ga_w ? G.ga_w + 4 * (size_t)ea : W + 4 * (size_t)(__ldg(&ga_ent[ea]) >> 6);
        const double2 w01 = __ldg(reinterpret_cast<const double2 *>(wp));
        const double2 w23 = __ldg(reinterpret_cast<const double2 *>(wp + 2));
        const double w[4] = {w01.x, w01.y, w23.x, w23.y};
        // H_vu[c'][c] = H_uv[c][c'] = vals plane 3c + c'
        double Hvu[3][3];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
#pragma unroll
          for (int cp = 0; cp < 3; ++cp) Hvu[cp][cc] = __ldg(&H.vals[(cs * 9 + 3 * cc + cp) * 32 + ln_]);
#pragma unroll
        for (int cp = 0; cp < 3; ++cp)
#pragma unroll
          for (int kp = 0; kp < 4; ++kp)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc)
              acc[(4 * cp + kp) * 3 + cc] = fma(w[kp], Hvu[cp][cc], acc[(4 * cp + kp) * 3 + cc]);
      }
    }
    __syncthreads();   // previous chunk's phase B is done with Rs
    if (half == 0) {
#pragma unroll
      for (int k = 0; k < 36; ++k) Rs[ul_a * 36 + k] = acc[k];
    }
    __syncthreads();
    if (half == 1) {
#pragma unroll
      for (int k = 0; k < 36; ++k) Rs[ul_a * 36 + k] += acc[k];
    }
    __syncthreads();
    // ---- phase B: three groups of 9 lanes per warp take every third staged entry; lane g of
    // a group owns R entries 4g..4g+3 x the 4 monomials k (16 accumulators); the groups are
    // summed in a fixed order at the end of the slot
    const int *o = off + ch * (nup + 1);
    const int grp = lane / 9, g = lane - 9 * grp;   // grp 3: lanes 27..31 idle in the FMA loop
#ifdef MSIM_GAL_SKIP_B   // timing diagnostics only (wrong results): phase A alone
    for (int q = nup; q < nup; q += kGalWarps) {
#else
    for (int q = warp; q < nup; q += kGalWarps) {
#endif
      double a[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int k = 0; k < 4; ++k) a[r][k] = 0.0;
      const int e1 = __ldg(&o[q + 1]);
      // the list entries of batch b+1 (index, then the gathered w_uj) are loaded while batch b
      // is multiplied: two dependent global round trips per batch otherwise stall the warp
      uint32_t en_n = 0;
      double2 w01_n = make_double2(0.0, 0.0), w23_n = w01_n;
      int eb = __ldg(&o[q]);
      if (eb + lane < e1) {
        en_n = __ldg(&gl_ent[eb + lane]);
        const double *wp = G.gl_w ? G.gl_w + 4 * (size_t)(eb + lane) : W + 4 * (size_t)(en_n >> 7);
        w01_n = __ldg(reinterpret_cast<const double2 *>(wp));
        w23_n = __ldg(reinterpret_cast<const double2 *>(wp + 2));
      }
      for (; eb < e1; eb += 32) {
        const int n = min(32, e1 - eb);
        __syncwarp();
        if (lane < n) {
          reinterpret_cast<double2 *>(myW)[2 * lane] = w01_n;
          reinterpret_cast<double2 *>(myW)[2 * lane + 1] = w23_n;
          myU[lane] = (int)(en_n & (kGalChunk - 1)) * 36;
        }
        __syncwarp();
        if (eb + 32 + lane < e1) {
          en_n = __ldg(&gl_ent[eb + 32 + lane]);
          const double *wp = G.gl_w ? G.gl_w + 4 * (size_t)(eb + 32 + lane) : W + 4 * (size_t)(en_n >> 7);
          w01_n = __ldg(reinterpret_cast<const double2 *>(wp));
          w23_n = __ldg(reinterpret_cast<const double2 *>(wp + 2));
        }
        if (grp < 3) {
#pragma unroll 2
          for (int k = grp; k < n; k += 3) {
            const double2 w01 = reinterpret_cast<const double2 *>(myW)[2 * k];
            const double2 w23 = reinterpret_cast<const double2 *>(myW)[2 * k + 1];
            const double *rr = Rs + myU[k] + 4 * g;
            const double2 r01 = reinterpret_cast<const double2 *>(rr)[0];
            const double2 r23 = reinterpret_cast<const double2 *>(rr)[1];
            const double rv[4] = {r01.x, r01.y, r23.x, r23.y}, wv[4] = {w01.x, w01.y, w23.x, w23.y};
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int k2 = 0; k2 < 4; ++k2) a[r][k2] = fma(rv[r], wv[k2], a[r][k2]);
          }
        }
      }
      // a (group 0) + a (group 1) + a (group 2), then add to the slot accumulator
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double v1 = __shfl_down_sync(0xffffffffu, a[r][k], 9);
          const double v2 = __shfl_down_sync(0xffffffffu, a[r][k], 18);
          a[r][k] = (a[r][k] + v1) + v2;
        }
      if (grp == 0) {
        double *sa = Sacc + q * 144;
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int k = 0; k < 4; ++k) sa[k * 36 + 4 * g + r] += a[r][k];
      }
    }
  }
  __syncthreads();
  if (G.nparts > 1) {
    double *dst = G.Spart + (size_t)(i * G.nparts + part) * G.pstride;
    for (int e = t; e < nup * 144; e += kGalThreads) dst[e] = Sacc[e];
    __syncthreads();
    return;
  }
  // ---- write S_ij (row-major 12x12: row 4c'+k', column 4c+k) and its transpose S_ji
  for (int e = t; e < nup * 144; e += kGalThreads) {
    const int q = e / 144, r = e % 144, k = r / 36, l = r % 36;
    const int row = l / 3, cc = l % 3;
    const int b = __ldg(&gj_blk[j0 + q]);
    const double val = Sacc[e];
    S[144 * (size_t)b + row * 12 + 4 * cc + k] = val;
    const int bt = __ldg(&sT[b]);
    if (bt != b) S[144 * (size_t)bt + (4 * cc + k) * 12 + row] = val;
  }
  __syncthreads();
}

// S_i. = sum of the parts (fixed order), written as S_ij and its transpose S_ji
__device__ __forceinline__ void galerkin_reduce_row(const GalParams &G, int i) {
  const int j0 = G.gj_ptr[i], nup = G.gj_ptr[i + 1] - j0;
  const double *src = G.Spart + (size_t)i * G.nparts * G.pstride;
  for (int e = threadIdx.x; e < nup * 144; e += blockDim.x) {
    double val = src[e];
    for (int p = 1; p < G.nparts; ++p) val += src[(size_t)p * G.pstride + e];
    const int q = e / 144, r = e % 144, k = r / 36, l = r % 36;
    const int row = l / 3, cc = l % 3;
    const int b = __ldg(&G.gj_blk[j0 + q]);
    G.S[144 * (size_t)b + row * 12 + 4 * cc + k] = val;
    const int bt = __ldg(&G.sT[b]);
    if (bt != b) G.S[144 * (size_t)bt + (4 * cc + k) * 12 + row] = val;
  }
}

// Fused form (chol.cu task R(i)): the parts of handle i's row summed in the same fixed order,
// scattered straight into the lower triangle of the padded dense factor array L (column-major,
// handle i at rows 12 perm[i] ..): block S_ij (j >= i) lands at (12 perm[i] + row, 12 perm[j] + col)
// if that is in the lower triangle, else (its transposed image) at the mirrored position; of the
// diagonal block only the lower triangle is written (as k_scatter_S does).
__device__ __forceinline__ void galerkin_reduce_to_tiles(const GalParams &G, int i, const int32_t *__restrict__ perm,
                                                         int nSp, double *__restrict__ L) {
  const int j0 = G.gj_ptr[i], nup = G.gj_ptr[i + 1] - j0;
  const double *src = G.Spart + (size_t)i * G.nparts * G.pstride;
  const int pi = 12 * perm[i];
  for (int e = threadIdx.x; e < nup * 144; e += blockDim.x) {
    double val = __ldcg(&src[e]);
    for (int p = 1; p < G.nparts; ++p) val += __ldcg(&src[(size_t)p * G.pstride + e]);
    const int q = e / 144, r = e % 144, k = r / 36, l = r % 36;
    const int row = l / 3, cc = l % 3;
    const int j = __ldg(&G.scol[__ldg(&G.gj_blk[j0 + q])]);
    const int R = pi + row, C = 12 * perm[j] + 4 * cc + k;
    if (R >= C) L[(size_t)C * nSp + R] = val;
    else if (j != i) L[(size_t)R * nSp + C] = val;
  }
}

}  // namespace msim
