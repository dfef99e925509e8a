// cycles of the single-warp 32x32 kernels of chol_diag.cuh (one warp, warm loop)
#include <cstdio>
#include <cuda_runtime.h>
#include "fastmath.cuh"
namespace msim {
constexpr int TB = 64;
constexpr int LD = TB + 1;
__device__ __forceinline__ size_t tile_off(int ti, int tj, int nSp) { return (size_t)(tj * TB) * nSp + (size_t)ti * TB; }
#include "chol_diag.cuh"
}
using namespace msim;
__global__ void kw(long long *out, int reps) {
  __shared__ double A[64 * LD], Li[64 * LD], invd[64], col[64];
  const int lane = threadIdx.x;
  long long t1 = 0, t2 = 0, t3 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = lane; e < 64 * LD; e += 32) { int r = e / LD, c = e % LD; A[e] = (r == c) ? 40.0 : 1.0 / (1 + r + c); Li[e] = 0; }
    for (int e = lane; e < 64; e += 32) { col[e] = 0; invd[e] = 0; }
    __syncwarp();
    long long a = clock64();
    warp_potrf32(A, LD, invd, col, lane);
    __syncwarp();
    long long b = clock64();
    warp_trsm32(A, A + 32 * LD, LD, invd, lane);
    __syncwarp();
    long long c = clock64();
    warp_trinv32(A, LD, invd, Li, lane);
    __syncwarp();
    long long d = clock64();
    t1 += b - a; t2 += c - b; t3 += d - c;
  }
  if (lane == 0) { out[0] = t1 / reps; out[1] = t2 / reps; out[2] = t3 / reps; }
}
int main() {
  long long *d; cudaMalloc(&d, 64); kw<<<1, 32>>>(d, 2); kw<<<1, 32>>>(d, 10);
  long long h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("potrf32 %lld  trsm32 %lld  trinv32 %lld cycles\n", h[0], h[1], h[2]);
}
