// debug_kernels.cuh — elementwise test-hook kernels of srmdp_debug.h
// (non-template: included by srmdp.cu only).
#pragma once
#include "problem.cuh"

namespace srk {

__global__ void detmath_kernel(const int op, const int64_t n, const double* __restrict__ in,
                               double* __restrict__ o0, double* __restrict__ o1, const double* __restrict__ det) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  DetTabs T;
  T.logt = reinterpret_cast<const double2*>(det);
  T.sct = reinterpret_cast<const double2*>(det + 256);
  T.stride = 1;
  if (op == 0) {
    o0[t] = dm_log(in[t], T);
  } else if (op == 2) {
    o0[t] = dsqrt_inrange(in[t]);   // Box-Muller's sqrt (in-range inputs only)
  } else if (op == 3) {
    o0[t] = inv_minus_one<true>(in[t]);   // the start point's 1/p - 1 (2^-1000 <= p < 1 only)
  } else {
    double s, c;
    dm_sincospi2(in[t], T, s, c);
    o0[t] = s;
    o1[t] = c;
  }
}

__global__ void philox_kernel(const int64_t n, const uint32_t* __restrict__ ctr, const uint32_t k0,
                              const uint32_t k1, uint32_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const U4 o = philox4x32_10(U4{ctr[4 * t], ctr[4 * t + 1], ctr[4 * t + 2], ctr[4 * t + 3]}, k0, k1);
  out[4 * t] = o.x;
  out[4 * t + 1] = o.y;
  out[4 * t + 2] = o.z;
  out[4 * t + 3] = o.w;
}

}  // namespace srk
