// ops.h — per-(d,q) launch wrappers of the step / eval / trace kernels.
// make_ops<D,Q>() is defined in inst.cuh and explicitly instantiated in the
// inst_*.cu translation units, which nvcc compiles in parallel.
#pragma once
#include <cuda_runtime.h>

#include "problem.cuh"

struct Ops {
  int D, Q;
  cudaError_t (*prepare)(int C, size_t* smem, int* ctas);     // equal-size grid
  void (*step)(const srk::DevProblem&, int, int64_t, int64_t, int, size_t, cudaStream_t);
  cudaError_t (*prepare_eq)(int C, size_t* smem, int* ctas);  // equal-probability
  void (*step_eq)(const srk::DevProblem&, int, int64_t, int64_t, int, size_t, cudaStream_t);   // (nullptr: d > 8)
  void (*eval)(const srk::DevProblem&, int, int64_t, const double*, double*, double*, cudaStream_t);
  void (*trace)(const srk::DevProblem&, int, uint32_t, int64_t, int64_t, double*, int64_t*, double*, cudaStream_t);
};

template <int D, int Q>
Ops make_ops();
