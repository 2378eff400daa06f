// aux_kernels.cuh — evaluation kernel (srmdp_eval) and the test-hook kernels
// of srmdp_debug.h. They inline the same __device__ functions as the step
// kernel (problem.cuh, detmath.cuh, eval_block).
#pragma once
#include "step_kernel.cuh"

namespace srk {

// y_i^(M), z_i^(M) at n points (truncated); i == N: g.
template <int D, int Q>
__global__ void eval_kernel(const DevProblem P, const int i, const int64_t n, const double* __restrict__ xs,
                            double* __restrict__ ys, double* __restrict__ zs) {
  using KC = KCfg<D, Q>;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double x[D];
#pragma unroll
  for (int l = 0; l < D; ++l) x[l] = xs[t * D + l];
  if (i == P.N) {
    ys[t] = g_eval<D>(P, x);
    return;
  }
  const double* cen = P.tabs + 2 * (P.C + 1);   // read through L1 (no draws here)
  uint32_t kn = 0;
  double a[D + 1];
  a[0] = 1.0;
#pragma unroll
  for (int l = 0; l < D; ++l) {
    const int c = P.equi ? locate_g<true>(P, P.tabs + (P.C + 1), x[l]) : locate_g<false>(P, P.tabs + (P.C + 1), x[l]);
    kn = kn * (uint32_t)P.C + (uint32_t)c;
    a[1 + l] = x[l] - __ldg(cen + c);
  }
  SRK_CHECK(kn < (uint64_t)P.K && i < P.N, "eval cell");
  const double* blk = P.table + ((size_t)i * (size_t)P.K_pad + kn) * (size_t)KC::NBP;
  double v = 0.0;
#pragma unroll
  for (int p = 0; p <= D; ++p) v = fma(__ldg(blk + p), a[p], v);
  ys[t] = trunc_L(v, P.C_y);
  if (zs) {
    for (int l = 0; l < Q; ++l) {
      double w = 0.0;
#pragma unroll
      for (int p = 0; p <= D; ++p) w = fma(__ldg(blk + KC::NH + l * KC::N1 + p), a[p], w);
      zs[t * Q + l] = trunc_L(w, P.C_z);
    }
  }
}

// Path trace (srmdp_debug_trace): start point, increments, Euler states and
// located cells of paths m0 .. m0+n-1 of cloud (i,k).
template <int D, int Q>
__global__ void trace_kernel(const DevProblem P, const int i, const uint32_t k, const int64_t m0, const int64_t n,
                             double* __restrict__ xs, int64_t* __restrict__ cells, double* __restrict__ dws) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint32_t m = (uint32_t)(m0 + t);
  const Grid G = make_grid(P.tabs, P.C);
  int cc[D];
  {
    uint32_t r = k;
#pragma unroll
    for (int l = D - 1; l >= 0; --l) { cc[l] = (int)(r % (uint32_t)P.C); r /= (uint32_t)P.C; }
  }
  const int steps = P.N - i;
  double X[D];
  if (P.equi) start_point<D, true>(P, G, cc, i, k, m, X);
  else start_point<D, false>(P, G, cc, i, k, m, X);
  double* xo = xs + t * (int64_t)(steps + 1) * D;
  int64_t* co = cells + t * (int64_t)(steps + 1);
  double* wo = dws + t * (int64_t)steps * Q;
  auto put = [&](int s, const double (&v)[D]) {
    uint32_t kn = 0;
#pragma unroll
    for (int l = 0; l < D; ++l) {
      xo[s * D + l] = v[l];
      kn = kn * (uint32_t)P.C + (uint32_t)(P.equi ? locate_g<true>(P, G.edge, v[l]) : locate_g<false>(P, G.edge, v[l]));
    }
    co[s] = kn;
  };
  put(0, X);
  for (int j = i; j < P.N; ++j) {
    double dW[Q], Xn[D];
    brownian<Q>(P, G, i, j, k, m, dW);
    euler<D, Q>(P, (double)j * P.dt, X, dW, Xn);
#pragma unroll
    for (int l = 0; l < Q; ++l) wo[(j - i) * Q + l] = dW[l];
    put(j - i + 1, Xn);
#pragma unroll
    for (int l = 0; l < D; ++l) X[l] = Xn[l];
  }
}

}  // namespace srk
