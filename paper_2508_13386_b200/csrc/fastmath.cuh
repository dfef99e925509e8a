// Branch-free fp64 reciprocal / reciprocal square root: MUFU seed + Newton steps (no slow-path
// subroutine calls, no divergence).  Relative error ~1 ulp for normal, finite, positive inputs.
#pragma once

namespace msim {

__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double h = 0.5 * x * y;
    y = fma(y, fma(-h, y, 0.5), y);   // y += y (0.5 - 0.5 x y^2)
  }
  return y;
}

// two Newton steps: enough from the MUFU seed for ~1-2 ulp
__device__ __forceinline__ double rsqrt_nr2(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double h = 0.5 * x * y;
    y = fma(y, fma(-h, y, 0.5), y);
  }
  return y;
}

}  // namespace msim
