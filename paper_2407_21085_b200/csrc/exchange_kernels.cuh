// exchange_kernels.cuh — cross-GPU completion flags of the fused exchange
// (SRMDP_FLAG_P2P_EXCHANGE, srmdp.cu). The step kernel's epilogue stores each
// coefficient block into every rank's table (peer pointers opened through
// CUDA IPC); these kernels order those stores against the next step's reads.
//
// flags: every rank owns a uint32 array [N + 1][world] (IPC-shared). Slot i
// (0 <= i < N) says "rank r has written all its blocks of slice i into my
// table"; slot N is the entry barrier of a solve (no rank writes into a peer's
// table before that peer has entered the same solve). Values are the solve
// epoch, so flags never need resetting. Release / acquire at system scope.
// Non-template: included by srmdp.cu only.
#pragma once
#include "detmath.cuh"

namespace srk {

constexpr int kMaxRanks = 8;

struct FlagPtrs {
  unsigned* f[kMaxRanks];   // every rank's flag array (own included), as mapped here
};

__global__ void epoch_kernel(unsigned* epoch) { *epoch = *epoch + 1u; }

// After the step kernel of slice `slot` (same stream): make this rank's
// stores to the peers' tables visible, then publish the epoch in every
// rank's flag array at [slot][rank].
__global__ void exchange_signal_kernel(const FlagPtrs F, int world, int rank, int slot, const unsigned* epoch) {
  const int r = threadIdx.x;
  if (r >= world) return;
  __threadfence_system();
  const unsigned e = *epoch;
  unsigned* p = F.f[r] + (size_t)slot * world + rank;
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(e) : "memory");
}

// NVLS variant: one multimem release store through the multicast mapping of
// the flag arrays publishes the epoch at [slot][rank] in every rank's flags.
__global__ void exchange_signal_mc_kernel(unsigned* mc_flags, int world, int rank, int slot, const unsigned* epoch) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  asm volatile("fence.proxy.alias;" ::: "memory");
  const unsigned e = *epoch;
  unsigned* p = mc_flags + (size_t)slot * world + rank;
  asm volatile("multimem.st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(e) : "memory");
}

// Before anything reads slice `slot` (or, for the entry slot, before the
// first peer store): wait until every rank has published this epoch. The spin
// is bounded (timeout_ns of %globaltimer): a rank that never signals (died,
// failed collective) sets err = 1 + slot instead of hanging this stream; the
// host turns it into SRMDP_E_NCCL at srmdp_wait and the table is invalid.
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void exchange_wait_kernel(const unsigned* own, int world, int slot, const unsigned* epoch, unsigned* err,
                                     uint64_t timeout_ns) {
  const int r = threadIdx.x;
  if (r >= world) return;
  const unsigned e = *epoch;
  const unsigned* p = own + (size_t)slot * world + r;
  const uint64_t t0 = global_ns();
  unsigned v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if ((int)(v - e) >= 0) break;
    if (*(volatile unsigned*)err || global_ns() - t0 > timeout_ns) {   // give up (once one wait failed, all do)
      atomicCAS(err, 0u, 1u + (unsigned)slot);
      break;
    }
    __nanosleep(200);
  }
  __threadfence_system();
}

}  // namespace srk
