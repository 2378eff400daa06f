// nvls.cu — NVLS multicast mapping of the coefficient table (see nvls.h).
#include "nvls.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <cstring>

namespace {

struct Drv {
  bool ok = false;
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long) = nullptr;
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long) = nullptr;
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
};

Drv& drv() {
  static Drv d;
  static bool tried = false;
  if (tried) return d;
  tried = true;
  bool ok = true;
  auto get = [&](const char* name, void** fn) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
        !*fn)
      ok = false;
  };
  get("cuDeviceGet", (void**)&d.DeviceGet);
  get("cuDeviceGetAttribute", (void**)&d.DeviceGetAttribute);
  get("cuMulticastGetGranularity", (void**)&d.MulticastGetGranularity);
  get("cuMulticastCreate", (void**)&d.MulticastCreate);
  get("cuMulticastAddDevice", (void**)&d.MulticastAddDevice);
  get("cuMulticastBindMem", (void**)&d.MulticastBindMem);
  get("cuMulticastUnbind", (void**)&d.MulticastUnbind);
  get("cuMemCreate", (void**)&d.MemCreate);
  get("cuMemRelease", (void**)&d.MemRelease);
  get("cuMemAddressReserve", (void**)&d.MemAddressReserve);
  get("cuMemAddressFree", (void**)&d.MemAddressFree);
  get("cuMemMap", (void**)&d.MemMap);
  get("cuMemUnmap", (void**)&d.MemUnmap);
  get("cuMemSetAccess", (void**)&d.MemSetAccess);
  get("cuMemExportToShareableHandle", (void**)&d.MemExportToShareableHandle);
  get("cuMemImportFromShareableHandle", (void**)&d.MemImportFromShareableHandle);
  get("cuGetErrorString", (void**)&d.GetErrorString);
  d.ok = ok;
  return d;
}

bool fail(std::string& err, const char* what, CUresult r) {
  const char* s = nullptr;
  if (drv().GetErrorString) drv().GetErrorString(r, &s);
  err = std::string("NVLS ") + what + ": " + (s ? s : "error");
  return false;
}

// Abstract-namespace Unix socket address of the rendezvous `key`.
socklen_t sock_addr(const std::string& key, sockaddr_un* a) {
  memset(a, 0, sizeof(*a));
  a->sun_family = AF_UNIX;
  const std::string name = "srmdp-nvls-" + key;
  const size_t n = name.size() < sizeof(a->sun_path) - 2 ? name.size() : sizeof(a->sun_path) - 2;
  memcpy(a->sun_path + 1, name.data(), n);   // sun_path[0] = 0: abstract namespace
  return (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
}

bool send_fd(int sock, int fd) {
  char byte = 0;
  iovec iov{&byte, 1};
  char ctl[CMSG_SPACE(sizeof(int))];
  memset(ctl, 0, sizeof(ctl));
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctl;
  m.msg_controllen = sizeof(ctl);
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int));
  memcpy(CMSG_DATA(c), &fd, sizeof(int));
  return sendmsg(sock, &m, 0) == 1;
}

int recv_fd(int sock) {
  char byte = 0;
  iovec iov{&byte, 1};
  char ctl[CMSG_SPACE(sizeof(int))];
  msghdr m{};
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = ctl;
  m.msg_controllen = sizeof(ctl);
  if (recvmsg(sock, &m, 0) != 1) return -1;
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  if (!c || c->cmsg_type != SCM_RIGHTS) return -1;
  int fd = -1;
  memcpy(&fd, CMSG_DATA(c), sizeof(int));
  return fd;
}

}  // namespace

bool nvls_create(int device, size_t bytes, int world, int rank, const std::string& key,
                 const std::function<bool()>& barrier, NvlsTable* out, std::string& err) {
  Drv& d = drv();
  if (!d.ok) { err = "NVLS: driver entry points unavailable"; return false; }
  NvlsTable t;
  t.device = device;
  CUdevice dev;
  CUresult r = d.DeviceGet(&dev, device);
  if (r != CUDA_SUCCESS) return fail(err, "cuDeviceGet", r);
  int mc_ok = 0;
  d.DeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  if (!mc_ok) { err = "NVLS: multicast not supported on this GPU / system (no NVSwitch NVLS)"; return false; }
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.numDevices = (unsigned)world;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes;
  size_t gran = 0;
  if ((r = d.MulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED)) != CUDA_SUCCESS)
    return fail(err, "cuMulticastGetGranularity", r);
  t.bytes = (bytes + gran - 1) / gran * gran;
  mp.size = t.bytes;

  // physical memory of this rank's replica
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle ph = 0, mc = 0;
  if ((r = d.MemCreate(&ph, t.bytes, &ap, 0)) != CUDA_SUCCESS) return fail(err, "cuMemCreate", r);
  t.phys = ph;

  // the multicast object: rank 0 creates it; the others receive its handle
  if (rank == 0) {
    if ((r = d.MulticastCreate(&mc, &mp)) != CUDA_SUCCESS) { nvls_destroy(&t); return fail(err, "cuMulticastCreate", r); }
    t.mcobj = mc;
  }
  if (world > 1) {
    sockaddr_un a;
    const socklen_t al = sock_addr(key, &a);
    int fd = -1, lsock = -1;
    if (rank == 0) {
      if ((r = d.MemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0)) != CUDA_SUCCESS) {
        nvls_destroy(&t);
        return fail(err, "cuMemExportToShareableHandle", r);
      }
      lsock = socket(AF_UNIX, SOCK_STREAM, 0);
      if (lsock < 0 || bind(lsock, (sockaddr*)&a, al) != 0 || listen(lsock, world) != 0) {
        if (lsock >= 0) close(lsock);
        close(fd);
        nvls_destroy(&t);
        err = "NVLS: rendezvous socket";
        return false;
      }
    }
    if (!barrier()) { err = "NVLS: barrier (listen)"; nvls_destroy(&t); return false; }
    bool ok = true;
    if (rank == 0) {
      for (int n = 1; n < world && ok; ++n) {
        const int s = accept(lsock, nullptr, nullptr);
        ok = s >= 0 && send_fd(s, fd);
        if (s >= 0) close(s);
      }
      close(lsock);
      close(fd);
    } else {
      const int s = socket(AF_UNIX, SOCK_STREAM, 0);
      int tries = 0;
      while (s >= 0 && connect(s, (sockaddr*)&a, al) != 0 && ++tries < 200) usleep(10000);
      fd = (s >= 0 && tries < 200) ? recv_fd(s) : -1;
      if (s >= 0) close(s);
      ok = fd >= 0;
      if (ok) {
        r = d.MemImportFromShareableHandle(&mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
        close(fd);
        ok = r == CUDA_SUCCESS;
        if (ok) t.mcobj = mc;
      }
    }
    if (!ok) { nvls_destroy(&t); err = "NVLS: multicast handle exchange failed"; return false; }
  }
  // every device joins before any memory is bound
  if ((r = d.MulticastAddDevice(mc, dev)) != CUDA_SUCCESS) { nvls_destroy(&t); return fail(err, "cuMulticastAddDevice", r); }
  if (world > 1 && !barrier()) { nvls_destroy(&t); err = "NVLS: barrier (add device)"; return false; }
  if ((r = d.MulticastBindMem(mc, 0, ph, 0, t.bytes, 0)) != CUDA_SUCCESS) {
    nvls_destroy(&t);
    return fail(err, "cuMulticastBindMem", r);
  }
  t.bound = true;
  CUmemAccessDesc ad;
  memset(&ad, 0, sizeof(ad));
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = device;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mcp = 0;
  if ((r = d.MemAddressReserve(&uc, t.bytes, gran, 0, 0)) != CUDA_SUCCESS) { nvls_destroy(&t); return fail(err, "reserve", r); }
  t.uc = (void*)uc;
  if ((r = d.MemMap(uc, t.bytes, 0, ph, 0)) != CUDA_SUCCESS || (r = d.MemSetAccess(uc, t.bytes, &ad, 1)) != CUDA_SUCCESS) {
    nvls_destroy(&t);
    return fail(err, "unicast map", r);
  }
  if ((r = d.MemAddressReserve(&mcp, t.bytes, gran, 0, 0)) != CUDA_SUCCESS) { nvls_destroy(&t); return fail(err, "reserve", r); }
  t.mc = (void*)mcp;
  if ((r = d.MemMap(mcp, t.bytes, 0, mc, 0)) != CUDA_SUCCESS || (r = d.MemSetAccess(mcp, t.bytes, &ad, 1)) != CUDA_SUCCESS) {
    nvls_destroy(&t);
    return fail(err, "multicast map", r);
  }
  if (world > 1 && !barrier()) { nvls_destroy(&t); err = "NVLS: barrier (mapped)"; return false; }
  *out = t;
  return true;
}

void nvls_destroy(NvlsTable* t) {
  Drv& d = drv();
  if (!d.ok || !t) return;
  if (t->mc) {
    d.MemUnmap((CUdeviceptr)t->mc, t->bytes);
    d.MemAddressFree((CUdeviceptr)t->mc, t->bytes);
  }
  if (t->uc) {
    d.MemUnmap((CUdeviceptr)t->uc, t->bytes);
    d.MemAddressFree((CUdeviceptr)t->uc, t->bytes);
  }
  if (t->bound && t->mcobj) {
    CUdevice dev;
    if (d.DeviceGet(&dev, t->device) == CUDA_SUCCESS) d.MulticastUnbind(t->mcobj, dev, 0, t->bytes);
  }
  if (t->phys) d.MemRelease(t->phys);
  if (t->mcobj) d.MemRelease(t->mcobj);
  *t = NvlsTable();
}
