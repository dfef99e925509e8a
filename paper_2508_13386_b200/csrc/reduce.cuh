// Deterministic block reductions: per-CTA partials written to a buffer,
// the last CTA to finish (threadfence + atomic ticket) sums them in a fixed order.
// The result is independent of CTA scheduling: bit-identical reruns.
#pragma once
#include <cuda_runtime.h>

namespace msim {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// Sum NV per-thread values over the block; result valid in thread 0.  smem: NV*32 doubles.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = warp_sum(v[k]);
    if (lane == 0) sh[k * 32 + wid] = s;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = lane < nw ? sh[k * 32 + lane] : 0.0;
      v[k] = warp_sum(s);
    }
  }
  __syncthreads();
}

// Grid-wide deterministic sum of NV values.  partial: [NV][gridDim.x]; out: [NV].
// op: 0 = sum, 1 = min.  Every thread of every block must call this.
template <int NV, int OP = 0>
__device__ __forceinline__ bool grid_reduce(double (&v)[NV], double *partial, unsigned int *counter,
                                            double *out) {
  __shared__ double sh[NV * 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = OP == 0 ? warp_sum(v[k]) : warp_min(v[k]);
    if (lane == 0) sh[k * 32 + wid] = s;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = lane < nw ? sh[k * 32 + lane] : (OP == 0 ? 0.0 : 1e300);
      s = OP == 0 ? warp_sum(s) : warp_min(s);
      if (lane == 0) partial[(size_t)k * gridDim.x + blockIdx.x] = s;
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  // last block: fixed-order strided accumulation (4 independent chains for memory-level
  // parallelism) + fixed tree
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double init = OP == 0 ? 0.0 : 1e300;
    double s4[4] = {init, init, init, init};
    const double *pk = partial + (size_t)k * gridDim.x;
    const int G = (int)gridDim.x, step = blockDim.x;
    int b = threadIdx.x;
    for (; b + 3 * step < G; b += 4 * step) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double pv = __ldcg(&pk[b + u * step]);
        s4[u] = OP == 0 ? s4[u] + pv : fmin(s4[u], pv);
      }
    }
    for (; b < G; b += step) {
      const double pv = __ldcg(&pk[b]);
      s4[0] = OP == 0 ? s4[0] + pv : fmin(s4[0], pv);
    }
    double s = OP == 0 ? (s4[0] + s4[1]) + (s4[2] + s4[3]) : fmin(fmin(s4[0], s4[1]), fmin(s4[2], s4[3]));
    s = OP == 0 ? warp_sum(s) : warp_min(s);
    if (lane == 0) sh[k * 32 + wid] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = OP == 0 ? 0.0 : 1e300;
      for (int w = 0; w < nw; ++w) s = OP == 0 ? s + sh[k * 32 + w] : fmin(s, sh[k * 32 + w]);
      out[k] = s;
    }
    *counter = 0u;
  }
  return true;
}

}  // namespace msim
