// fp64_peak.cu — measured FP64 (DFMA) throughput of this B200, the roofline
// denominator of the ALU-bound SRMDP step kernel (MEASURED_PEAKS.json has no
// FP64 entry). 8 independent DFMA chains per thread, full occupancy, timed
// with CUDA events: burst (one ~50 ms launch after warm-up) and sustained
// (back-to-back launches for ~4 s). Prints one JSON line.
#include <cuda_runtime.h>

#include <cstdio>

__global__ void __launch_bounds__(256) dfma_chains(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
  double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 12345.678) out[blockIdx.x] = s;   // keep the chains alive
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dfma_chains, 256, 0);
  const int grid = per_sm * p.multiProcessorCount;
  double* out;
  cudaMalloc(&out, grid * sizeof(double));
  const int iters = 2000;
  const double flops_per_launch = 2.0 * 8 * 16 * (double)iters * 256 * grid;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dfma_chains<<<grid, 256>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e0);
  dfma_chains<<<grid, 256>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double burst = flops_per_launch / (ms * 1e-3) / 1e12;
  // sustained: ~4 s of back-to-back launches
  int n = (int)(4000.0 / ms) + 1;
  cudaEventRecord(e0);
  for (int t = 0; t < n; ++t) dfma_chains<<<grid, 256>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms2 = 0;
  cudaEventElapsedTime(&ms2, e0, e1);
  const double sustained = n * flops_per_launch / (ms2 * 1e-3) / 1e12;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"fp64_tflops_burst\": %.3f, \"fp64_tflops_sustained\": %.3f, \"sms\": %d, \"ctas_per_sm\": %d, "
         "\"burst_ms\": %.3f, \"sustained_launches\": %d, \"attr_clock_mhz\": %.0f, \"err\": \"%s\"}\n",
         burst, sustained, p.multiProcessorCount, per_sm, ms, n, clk / 1000.0, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
