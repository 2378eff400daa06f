// gather_bw.cu — the coefficient-gather ceiling of the SRMDP step kernel
// ("measure L2 gather GB/s with a random-block-gather
// microbenchmark"). Every thread repeatedly reads one 128-byte hot line of a
// 64-double block chosen per lane from a table of K blocks (cfg4: K = 15625,
// 512 B stride, 8 MB: L2-resident), as the step kernel's per-lane gather does:
//  - "random":   every lane an independent uniformly random block (worst case)
//  - "local":    lanes of a warp share a start block and hop to a random
//                neighbour (|dk| <= 1 in 3 of 6 coordinates of a 5^6 grid)
//                with probability 0.26, as paths do around their start cell
// with 128-bit (8 x LDG.128) and 256-bit (4 x LDG.256) loads. Occupancy as the
// step kernel (256 threads, 3 CTAs/SM, persistent). Prints one JSON line with
// lines/s and GB/s per variant.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <bool W256, bool LOCAL>
__global__ void __launch_bounds__(256, 3) gather(const double* __restrict__ tab, int K, int iters, double* out) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t k = hash32(LOCAL ? (tid >> 5) : tid) % (uint32_t)K;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t h = hash32(tid * 2654435761u + it);
    uint32_t kk;
    if (LOCAL) {
      // neighbour of the warp's cell with prob. 0.26 (5^6 grid, one coordinate +-1)
      int c[6];
      uint32_t r = k;
      for (int l = 5; l >= 0; --l) { c[l] = r % 5; r /= 5; }
      if ((h & 1023) < 266) {
        const int l = (h >> 10) % 6;
        c[l] = min(4, max(0, c[l] + (((h >> 13) & 1) ? 1 : -1)));
      }
      kk = 0;
      for (int l = 0; l < 6; ++l) kk = kk * 5 + c[l];
    } else {
      kk = h % (uint32_t)K;
    }
    const double* b = tab + (size_t)kk * 64;
    if (W256) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double v0, v1, v2, v3;
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v0), "=d"(v1), "=d"(v2), "=d"(v3) : "l"(b + 4 * u));
        acc += (v0 + v1) + (v2 + v3);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(b) + u);
        acc += v.x + v.y;
      }
    }
  }
  if (acc == 1234.5) out[tid] = acc;
}

template <bool W256, bool LOCAL>
static double run(const double* tab, int K, int grid, double* out, const char* name, bool last) {
  const int iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) gather<W256, LOCAL><<<grid, 256>>>(tab, K, iters, out);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) gather<W256, LOCAL><<<grid, 256>>>(tab, K, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double lines = (double)grid * 256 * iters * reps;
  const double ls = lines / (ms * 1e-3);
  printf("\"%s\": {\"lines_per_s\": %.4e, \"GB_per_s\": %.1f}%s", name, ls, ls * 128 / 1e9, last ? "" : ", ");
  return ls;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int K = 15625;
  double* tab;
  double* out;
  cudaMalloc(&tab, (size_t)K * 64 * sizeof(double));
  cudaMemset(tab, 0, (size_t)K * 64 * sizeof(double));
  const int grid = 3 * p.multiProcessorCount;
  cudaMalloc(&out, (size_t)grid * 256 * sizeof(double));
  printf("{\"device\": \"%s\", \"sms\": %d, \"K\": %d, \"block_bytes\": 512, \"line_bytes\": 128, ", p.name,
         p.multiProcessorCount, K);
  run<false, false>(tab, K, grid, out, "random_ldg128", false);
  run<true, false>(tab, K, grid, out, "random_ldg256", false);
  run<false, true>(tab, K, grid, out, "local_ldg128", false);
  run<true, true>(tab, K, grid, out, "local_ldg256", true);
  printf("}\n");
  return 0;
}
