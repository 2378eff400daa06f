/*
 * srmdp_debug.h — test hooks of the SRMDP library (same .so as srmdp.h).
 *
 * They run the product's own __device__ functions (the ones the step kernel
 * inlines) on the GPU and return their raw results, so tests can compare
 * path states and transcendental bits with the CPU oracle element by element
 * (docs/streams.md, docs/detmath.md). Host pointers; blocking; status codes
 * as in srmdp.h. Not part of the hot path.
 */
#ifndef SRMDP_DEBUG_H
#define SRMDP_DEBUG_H

#include "srmdp.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Path trace of cloud (i,k), paths m = m0 .. m0+n-1 (docs/streams.md §2-7):
 * x[n][N-i+1][d] = x_i .. x_N, cell[n][N-i+1] = located cells, dW[n][N-i][q].
 * Uses the start-point sampler, Box-Muller, Euler and locate of the step kernel. */
srmdp_status srmdp_debug_trace(const srmdp_t* h, int i, int64_t k, int64_t m0, int64_t n,
                               double* x, int64_t* cell, double* dW);

/* Re-run step i of the sweep with the cell-dump variant of the step kernel
 * (same code as the product kernel plus stores; compiled for the static
 * BM-dynamics (X = W) kernels of d = q in {1, 2, 4, 6, 11, 19}, equal-size
 * grid -- the kernels the §5.1 benchmark runs): for the first dump_m paths
 * of every cell of this rank's range, cell[kl][m][s] = located cell of
 * X_{i+1+s} (s = 0 .. N-i-2) and x[kl][m][s][d] = X_{i+1+s} (s = 0 .. N-i-1),
 * kl = k - k_begin. Needs slices i+1 .. N-1 present; rewrites slice i with the
 * same values a solve gives. srmdp_stats then holds this step's event counts
 * (lp0_fallbacks, exact_z_evals, exact_z_i). SRMDP_E_UNSUPPORTED for other (d, q) / NVRTC
 * builds / the equal-probability grid. */
srmdp_status srmdp_debug_step_dump(srmdp_t* h, int i, int dump_m, uint32_t* cell, double* x);

/* Elementwise device detmath (docs/detmath.md): op 0 = dm_log(in) -> out0;
 * op 1 = dm_sincospi2(in) -> (out0 = sin, out1 = cos); op 2 = the path's
 * correctly rounded sqrt (dsqrt_inrange, valid for 2^-970 <= in < 2^1023) -> out0;
 * op 3 = the start point's 1/p - 1 by the range-proved reciprocal
 * (inv_minus_one<true>, valid for 2^-1000 <= in < 1) -> out0. */
srmdp_status srmdp_debug_detmath(int op, size_t n, const double* in, double* out0, double* out1);

/* Philox4x32-10 on the device: ctr[n][4], key[2] -> out[n][4]. */
srmdp_status srmdp_debug_philox(size_t n, const uint32_t* ctr, const uint32_t key[2], uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
