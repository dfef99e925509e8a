// FP64 tensor-core (mma.sync m8n8k4 f64) vs DFMA throughput on this GPU: cycles per instruction
// per SM with many warps, and achieved TFLOP/s.
#include <cstdio>
__global__ void kdmma(double *o, int n) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  double c[8][2];
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kdfma(double *o, int n) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  double c[8];
  for (int q = 0; q < 8; ++q) c[q] = q;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = fma(a, b, c[q]);
  }
  double s = 0; for (int q = 0; q < 8; ++q) s += c[q];
  o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double *o; cudaMalloc(&o, 8 << 22);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const int n = 4096, blocks = 148 * 4, threads = 256;
  kdmma<<<blocks, threads>>>(o, 16); cudaEventRecord(e0); kdmma<<<blocks, threads>>>(o, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * 8.0 * n * (blocks * threads / 32);
  printf("DMMA m8n8k4: %.1f TFLOP/s\n", fl / ms / 1e9);
  kdfma<<<blocks, threads>>>(o, 16); cudaEventRecord(e0); kdfma<<<blocks, threads>>>(o, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 2.0 * 8.0 * n * blocks * threads;
  printf("DFMA: %.1f TFLOP/s\n", fl / ms / 1e9);
}
