// ops.h — per-(d,q) launch wrappers of the step / eval / trace kernels.
// make_ops<D,Q>() is defined in inst.cuh and explicitly instantiated in the
// inst_*.cu translation units, which nvcc compiles in parallel.
#pragma once
#include <cuda_runtime.h>

#include "problem.cuh"

#include <cmath>

// Smallest shared-memory carveout that still holds the resident CTAs: the
// rest of the SM's 256 KB L1/shared array stays L1 for the gathered hot
// lines (left to itself the driver picks 132 KB for 3 x 31 KB at d = 6).
#ifndef SRMDP_CARVEOUT_FIT
#define SRMDP_CARVEOUT_FIT 1
#endif
static inline cudaError_t fit_carveout(const void* f, size_t smem, int threads, int* ctas) {
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas, f, threads, smem);
  if (e != cudaSuccess || *ctas < 1 || !SRMDP_CARVEOUT_FIT) return e;
  int dev = 0, maxsm = 0, reserved = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  if (maxsm <= 0) return cudaSuccess;
  int pct = (int)std::ceil(100.0 * (double)(*ctas) * (double)(smem + reserved) / (double)maxsm);
  pct = pct < 0 ? 0 : (pct > 100 ? 100 : pct);
  return cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

struct Ops {
  int D, Q;
  cudaError_t (*prepare)(int C, size_t* smem, int* ctas);     // equal-size grid
  void (*step)(const srk::DevProblem&, int, int64_t, int64_t, int, size_t, cudaStream_t);
  cudaError_t (*prepare_eq)(int C, size_t* smem, int* ctas);  // equal-probability
  void (*step_eq)(const srk::DevProblem&, int, int64_t, int64_t, int, size_t, cudaStream_t);   // (nullptr: d > 8)
  void (*eval)(const srk::DevProblem&, int, int64_t, const double*, double*, double*, cudaStream_t);
  void (*trace)(const srk::DevProblem&, int, uint32_t, int64_t, int64_t, double*, int64_t*, double*, cudaStream_t);
  // debug variant of `step_bm` that dumps located cells / states (srmdp_debug_step_dump)
  void (*step_dump)(const srk::DevProblem&, int, int64_t, int64_t, int, size_t, cudaStream_t);
  // the equal-size-grid kernel with the dynamics fixed to BM (X = W, the §5.1 benchmark)
  cudaError_t (*prepare_bm)(int C, size_t* smem, int* ctas);
  void (*step_bm)(const srk::DevProblem&, int, int64_t, int64_t, int, size_t, cudaStream_t);
  // the same with the in-kernel exchange flags (fused P2P / NVLS exchange)
  cudaError_t (*prepare_bm_xw)(int C, size_t* smem, int* ctas);
  void (*step_bm_xw)(const srk::DevProblem&, int, int64_t, int64_t, int, size_t, cudaStream_t);
};

template <int D, int Q>
Ops make_ops();
