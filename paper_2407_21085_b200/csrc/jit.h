// jit.h — NVRTC builds of the step / eval / trace kernels for user problems
// (srmdp.h, SRMDP_*_USER) and for (d, q) pairs outside the compiled set.
#pragma once
#include <cuda_runtime.h>

#include <string>

struct JitKernels {
  int d = 0, q = 0;
  cudaKernel_t step[2] = {nullptr, nullptr};   // [equal-size grid, equal-probability grid]
  cudaKernel_t eval = nullptr;
  cudaKernel_t trace = nullptr;
};

// Compile (or fetch from the process-wide cache) the kernels of one (d, q)
// with the given user source; user_* select which srmdp_user_* functions the
// kernels call. Returns nullptr with a message (incl. the NVRTC log) in err.
const JitKernels* jit_kernels(int d, int q, bool user_dyn, bool user_f, bool user_g, const std::string& user_src,
                              std::string& err);

// NVRTC compile only (no GPU, nothing loaded): srmdp_jit_check.
bool jit_compile_check(int d, int q, bool user_dyn, bool user_f, bool user_g, const std::string& user_src,
                       std::string& err, size_t* cubin_bytes);
