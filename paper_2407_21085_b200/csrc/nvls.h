// nvls.h — NVLS multicast mapping of the coefficient table (the fused
// exchange's multicast epilogue, SRMDP_FLAG_NVLS_EXCHANGE).
//
// Every rank's [table | flags] is one physical allocation (cuMemCreate) bound
// to one multicast object that spans the ranks' GPUs (NVSwitch). The step
// kernel's epilogue stores each finished block once, with multimem.st through
// the multicast address, and the switch writes it into every rank's table;
// kernels read their own copy through the unicast address. Driver entry points
// are resolved at run time (cudaGetDriverEntryPoint): the library does not
// link libcuda, so it still loads on machines without a driver.
#pragma once
#include <cstddef>
#include <functional>
#include <string>

struct NvlsTable {
  void* uc = nullptr;        // unicast mapping (this rank's copy)
  void* mc = nullptr;        // multicast mapping (stores reach every rank)
  size_t bytes = 0;          // mapped size (multiple of the multicast granularity)
  unsigned long long phys = 0, mcobj = 0;   // CUmemGenericAllocationHandle
  int device = 0;
  bool bound = false;
};

// Collective over `world` ranks. `barrier` must block until every rank has
// reached it (the handle's NCCL communicator); `key` names the rendezvous of
// the multicast handle (rank 0 creates it and passes the file descriptor to
// the others over a Unix-domain socket in the abstract namespace).
// Returns false with `err` set on any failure (e.g. no NVLS on this system).
bool nvls_create(int device, size_t bytes, int world, int rank, const std::string& key,
                 const std::function<bool()>& barrier, NvlsTable* out, std::string& err);
void nvls_destroy(NvlsTable* t);
