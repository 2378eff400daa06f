// inst.cuh — launch wrappers for one (D, Q) (see ops.h). Included only by the
// inst_*.cu instantiation units.
#pragma once
#include "aux_kernels.cuh"
#include "ops.h"

using namespace srk;

template <int D, int Q, bool EQ, int DK = -1, bool XW = false>
static cudaError_t prepare_impl(int C, size_t* smem, int* ctas) {
  *smem = SmemLayout<D, Q>::bytes(C);
  cudaError_t e = cudaFuncSetAttribute(step_kernel<D, Q, EQ, false, DK, XW>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem);
  if (e != cudaSuccess) return e;
  return fit_carveout((const void*)step_kernel<D, Q, EQ, false, DK, XW>, *smem, step_threads(D), ctas);
}
template <int D, int Q, bool EQ, int DK = -1, bool XW = false>
static void step_impl(const DevProblem& P, int i, int64_t kb, int64_t nk, int grid, size_t smem, cudaStream_t s) {
  step_kernel<D, Q, EQ, false, DK, XW><<<grid, step_threads(D), smem, s>>>(P, i, kb, nk);
}
template <int D, int Q>
static void step_dump_impl(const DevProblem& P, int i, int64_t kb, int64_t nk, int grid, size_t smem, cudaStream_t s) {
  // same code as step_kernel<D, Q, false, false, DYN_BM> plus the dump stores; same shared memory
  if (cudaFuncSetAttribute(step_kernel<D, Q, false, true, DYN_BM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return;   // the launch below then fails and cudaGetLastError reports it
  step_kernel<D, Q, false, true, DYN_BM><<<grid, step_threads(D), smem, s>>>(P, i, kb, nk);
}
template <int D, int Q>
static void eval_impl(const DevProblem& P, int i, int64_t n, const double* x, double* y, double* z, cudaStream_t s) {
  const int bs = 128;
  eval_kernel<D, Q><<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(P, i, n, x, y, z);
}
template <int D, int Q>
static void trace_impl(const DevProblem& P, int i, uint32_t k, int64_t m0, int64_t n, double* x, int64_t* c,
                       double* w, cudaStream_t s) {
  const int bs = 64;
  trace_kernel<D, Q><<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(P, i, k, m0, n, x, c, w);
}

template <int D, int Q>
Ops make_ops() {
  // the cell-dump debug variant is compiled for the benchmark dimensions the
  // parity suite checks (d = 1, 2, 4, 6, 11, 19)
  constexpr bool dump = (D == Q) && (D == 1 || D == 2 || D == 4 || D == 6 || D == 11 || D == 19);
  void (*sd)(const DevProblem&, int, int64_t, int64_t, int, size_t, cudaStream_t) = nullptr;
  if constexpr (dump) sd = step_dump_impl<D, Q>;
  // BM-specialised kernel for the q = d benchmark dynamics (X = W)
  cudaError_t (*pb)(int, size_t*, int*) = nullptr, (*pbx)(int, size_t*, int*) = nullptr;
  void (*sb)(const DevProblem&, int, int64_t, int64_t, int, size_t, cudaStream_t) = nullptr;
  void (*sbx)(const DevProblem&, int, int64_t, int64_t, int, size_t, cudaStream_t) = nullptr;
  if constexpr (D == Q) {
    pb = prepare_impl<D, Q, false, DYN_BM>;
    sb = step_impl<D, Q, false, DYN_BM>;
    pbx = prepare_impl<D, Q, false, DYN_BM, true>;
    sbx = step_impl<D, Q, false, DYN_BM, true>;
  }
  if constexpr (D <= 8)
    return Ops{D, Q, prepare_impl<D, Q, false>, step_impl<D, Q, false>, prepare_impl<D, Q, true>, step_impl<D, Q, true>,
               eval_impl<D, Q>, trace_impl<D, Q>, sd, pb, sb, pbx, sbx};
  else
    return Ops{D, Q, prepare_impl<D, Q, false>, step_impl<D, Q, false>, nullptr, nullptr, eval_impl<D, Q>,
               trace_impl<D, Q>, sd, pb, sb, pbx, sbx};
}
