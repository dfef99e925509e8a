#include <cstdio>
__global__ void k(double *o, long long *c, int n) {
  double a = o[threadIdx.x], b = 1.0000001, x = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { a = fma(a, b, x); a = fma(a, b, x); a = fma(a, b, x); a = fma(a, b, x); }
  long long t1 = clock64();
  // independent: 8 chains
  double r[8]; for (int q = 0; q < 8; ++q) r[q] = o[q];
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = fma(r[q], b, x);
  }
  long long t3 = clock64();
  double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(y + 1.0));
  long long t5 = clock64();
  double s = 0; for (int q = 0; q < 8; ++q) s += r[q];
  o[threadIdx.x] = a + s + y;
  if (threadIdx.x == 0) { c[0] = (t1 - t0) / (4 * n); c[1] = (t3 - t2) / (8 * n); c[2] = (t5 - t4) / n; }
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 64); cudaMemset(o, 0, 8192);
  long long h[3];
  for (int w : {32, 128, 1024}) {
    k<<<1, w>>>(o, c, 1000); k<<<1, w>>>(o, c, 10000);
    cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("threads %4d: dependent DFMA latency %lld cyc; 8-chain DFMA %lld cyc/instr/warp-thread; rsqrt+dadd chain %lld\n", w, h[0], h[1], h[2]);
  }
}
