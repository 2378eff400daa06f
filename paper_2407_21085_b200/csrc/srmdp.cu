// srmdp.cu — host orchestrator and C ABI (include/srmdp.h, include/srmdp_debug.h)
// of the B200-native SRMDP backward sweep (arXiv 2407.21085, Alg. srmdp
// P:332-365).
//
// One process per GPU. Each rank owns a contiguous cell range; per time point
// i = N-1 .. 0 it launches the fused step kernel (step_kernel.cuh) on its
// cells and all-gathers slice i in place over NCCL (NVLink/NVSwitch), so every
// rank holds the full replicated coefficient table for the next step. The N
// launches (+ collectives) are captured once into a CUDA graph and replayed.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing without a tool attached

#include <chrono>
#include <algorithm>
#include <climits>
#include <cmath>
#include <map>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/srmdp.h"
#include "../../include/srmdp_debug.h"
#include "aux_kernels.cuh"
#include "debug_kernels.cuh"
#include "exchange_kernels.cuh"
#include "jit.h"
#include "nvls.h"
#include "ops.h"

using namespace srk;

// ------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------
static thread_local std::string g_create_err = "no error";


// ------------------------------------------------------------------------
// NCCL, loaded at run time (libnccl.so.2 is already mapped when torch is)
// ------------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string err;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = nullptr;
  const char* env = getenv("SRMDP_NCCL_LIB");
  if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
    return api;
  }
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
  api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
  api.CommAbort = (decltype(api.CommAbort))dlsym(h, "ncclCommAbort");
  api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  api.ok = api.GetUniqueId && api.CommInitRank && api.AllGather && api.CommDestroy && api.GetErrorString &&
           api.CommAbort && api.CommGetAsyncError;
  if (!api.ok) api.err = "libnccl.so.2 lacks a required symbol";
  return api;
}

// ------------------------------------------------------------------------
// host math of the grid (docs/streams.md §5, docs/detmath.md dm_exp,
// docs/layout.md). Compiled with -ffp-contract=off: each op one rounding.
// ------------------------------------------------------------------------
static double host_dm_exp(double x) {
  static const double E[15] = {
      0x1p+0, 0x1p+0, 0x1p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5,
      0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
      0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22,
      0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33,
      0x1.93974a8c07c9dp-37};
  if (x != x) return x;
  if (x > 709.782712893384) return INFINITY;
  if (x < -745.1332191019412) return 0.0;
  const double kf = std::rint(x * 0x1.71547652b82fep+0);
  const double r = (x - (kf * 0x1.62e42fee00000p-1)) - (kf * 0x1.a39ef35793c76p-33);
  double p = E[14];
  for (int j = 13; j >= 0; --j) p = std::fma(p, r, E[j]);
  return std::ldexp(p, (int)kf);
}

// Reference functions of docs/detmath.md (table builders only).
static double host_dm_log_series(double x) {
  static const double LG[11] = {0.0,
      0x1.5555555555555p-1, 0x1.999999999999ap-2, 0x1.2492492492492p-2, 0x1.c71c71c71c71cp-3,
      0x1.745d1745d1746p-3, 0x1.3b13b13b13b14p-3, 0x1.1111111111111p-3, 0x1.e1e1e1e1e1e1ep-4,
      0x1.af286bca1af28p-4, 0x1.8618618618618p-4};
  if (x != x || x < 0.0) return NAN;
  if (x == 0.0) return -INFINITY;
  if (std::isinf(x)) return INFINITY;
  int k = 0;
  if (x < 0x1p-1022) { x = x * 0x1p54; k = -54; }
  uint64_t b;
  memcpy(&b, &x, 8);
  k = k + (int)(b >> 52) - 1023;
  const uint64_t mb = (b & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
  double m;
  memcpy(&m, &mb, 8);
  if (m > 0x1.6a09e667f3bcdp+0) { m = m * 0.5; k = k + 1; }
  const double f = m - 1.0;
  const double s = f / (2.0 + f);
  const double z = s * s;
  double P = LG[10];
  for (int j = 9; j >= 1; --j) P = std::fma(P, z, LG[j]);
  const double R = z * P;
  const double t = s * R;
  const double lm = (2.0 * s) + t;
  const double hi = (double)k * 0x1.62e42fee00000p-1;
  const double lo = (double)k * 0x1.a39ef35793c76p-33;
  return hi + (lm + lo);
}

static void host_dm_sincospi2_series(double u, double* sn_out, double* cs_out) {
  static const double S[9] = {
      0x1.921fb54442d18p+0, -0x1.4abbce625be53p-1, 0x1.466bc6775aae2p-4, -0x1.32d2cce62bd86p-8,
      0x1.50783487ee782p-13, -0x1.e3074fde8871fp-19, 0x1.e8f434d018d63p-25, -0x1.6fadb9f155744p-31,
      0x1.aaec32af93359p-38};
  static const double Cc[10] = {
      0x1.0000000000000p+0, -0x1.3bd3cc9be45dep+0, 0x1.03c1f081b5ac4p-2, -0x1.55d3c7e3cbffap-6,
      0x1.e1f506891babbp-11, -0x1.a6d1f2a204a8cp-16, 0x1.f9d38a3763cc3p-22, -0x1.b6e24f44b128fp-28,
      0x1.20c62c2f2d7f5p-34, -0x1.2a0c591af8314p-41};
  const double v = 4.0 * u;
  const double n = std::rint(v);
  const double f = v - n;
  const double f2 = f * f;
  double ps = S[8];
  for (int j = 7; j >= 0; --j) ps = std::fma(ps, f2, S[j]);
  const double sn = f * ps;
  double pc = Cc[9];
  for (int j = 8; j >= 0; --j) pc = std::fma(pc, f2, Cc[j]);
  const double cs = pc;
  switch (((int)n) & 3) {
    case 0: *sn_out = sn; *cs_out = cs; break;
    case 1: *sn_out = cs; *cs_out = -sn; break;
    case 2: *sn_out = -sn; *cs_out = -cs; break;
    default: *sn_out = -cs; *cs_out = sn; break;
  }
}

// LOGT (128 x (INVC, LT)) and SCT (128 x (sin, cos)) of docs/detmath.md
static void det_tables(double* out /* 512 */) {
  for (int j = 0; j < 128; ++j) {
    double invc = 1.0, lt = 0.0;
    if (j != 0 && j != 127) {
      double c = 1.0 + (((double)j + 0.5) / 128.0);
      if (j >= 53) c = c * 0.5;
      invc = 1.0 / c;
      lt = -host_dm_log_series(invc);
    }
    out[2 * j] = invc;
    out[2 * j + 1] = lt;
    host_dm_sincospi2_series((double)j / 128.0, &out[256 + 2 * j], &out[256 + 2 * j + 1]);
  }
}

// dm_log (path function of docs/detmath.md) on the host, from the tables.
static double host_dm_log(double x, const double* det) {
  if (x != x || x < 0.0) return NAN;
  if (x == 0.0) return -INFINITY;
  if (std::isinf(x)) return INFINITY;
  static const double A[10] = {0.0, 0.0,
      -0x1.0000000000000p-1, 0x1.5555555555555p-2, -0x1.0000000000000p-2, 0x1.999999999999ap-3,
      -0x1.5555555555555p-3, 0x1.2492492492492p-3, -0x1.0000000000000p-3, 0x1.c71c71c71c71cp-4};
  int k = 0;
  if (x < 0x1p-1022) { x = x * 0x1p54; k = -54; }
  uint64_t b;
  memcpy(&b, &x, 8);
  k = k + (int)(b >> 52) - 1023;
  const uint64_t mb = b & 0x000fffffffffffffull;
  const int j = (int)(mb >> 45);
  const uint64_t m1 = mb | 0x3ff0000000000000ull;
  double m;
  memcpy(&m, &m1, 8);
  if (j >= 53) { m = m * 0.5; k = k + 1; }
  const double r = std::fma(m, det[2 * j], -1.0);
  const double r2 = r * r;
  double p = A[9];
  for (int n = 8; n >= 2; --n) p = std::fma(p, r, A[n]);
  const double l1 = std::fma(r2, p, r);
  const double kd = (double)k;
  return ((kd * 0x1.62e42fee00000p-1) + det[2 * j + 1]) + (l1 + (kd * 0x1.a39ef35793c76p-33));
}

// F_nu(x) = 1/(1+exp(-mu x))
static double host_F(double mu, double x) {
  if (x == -INFINITY) return 0.0;
  if (x == INFINITY) return 1.0;
  return 1.0 / (1.0 + host_dm_exp(-(mu * x)));
}

// tabs = [F(e_c), c=0..C | e_c, c=0..C | r_c, c=0..C-1 | pad | LOGT | SCT] (problem.cuh)
// equi: equal-probability breakpoints e_c = -(1/mu) dm_log(C/c - 1) (docs/streams.md §5)
static std::vector<double> grid_tables(int C, double L, double mu, bool equi) {
  std::vector<double> t(tabs_len(C), 0.0);
  double* det = t.data() + tabs_det_off(C);
  det_tables(det);
  const double delta = (2.0 * L) / (double)C;
  for (int c = 0; c <= C; ++c) {
    double e;
    if (c == 0) e = -INFINITY;
    else if (c == C) e = INFINITY;
    else if (equi) e = (-(1.0 / mu)) * host_dm_log(((double)C / (double)c) - 1.0, det);
    else e = (-L) + ((double)c * delta);
    t[C + 1 + c] = e;
    t[c] = host_F(mu, e);
  }
  const double* edge = t.data() + C + 1;
  for (int c = 0; c < C; ++c) {   // the certain-membership band and the clamp below e_{c+1} (problem.cuh)
    const double lo = edge[c], hi = edge[c + 1];
    const double m = 0x1p-40 * (std::fabs(L) + std::fabs(std::isfinite(lo) ? lo : 0.0) +
                                std::fabs(std::isfinite(hi) ? hi : 0.0) + 1.0);
    t[3 * C + 2 + c] = std::isfinite(lo) ? lo + m : lo;
    t[4 * C + 2 + c] = std::isfinite(hi) ? hi - m : hi;
    t[5 * C + 2 + c] = std::nextafter(hi, -INFINITY);
  }
  for (int c = 0; c < C; ++c) {
    double r;
    if (C == 1) r = 0.0;
    else if (equi) r = (c == 0) ? edge[1] : (c == C - 1) ? edge[C - 1] : (edge[c] + edge[c + 1]) * 0.5;
    else if (c == 0) r = (-L) + (1.0 * delta);
    else if (c == C - 1) r = (-L) + ((double)(C - 1) * delta);
    else r = (-L) + (((double)c + 0.5) * delta);
    t[2 * (C + 1) + c] = r;
  }
  return t;
}

// ------------------------------------------------------------------------
// per-(d,q) kernel dispatch: the launch wrappers are instantiated in the
// inst_*.cu translation units (compiled in parallel), see ops.h
// ------------------------------------------------------------------------
// Compiled (d, q) set: d = q = 1..8 and the paper's high-d rows 11..19
// (PAPER.md table:LP1d11 .. table:LP1d15_19), plus small d != q for AFFINE.
static const Ops kOps[] = {
    make_ops<1, 1>(),   make_ops<2, 2>(),   make_ops<3, 3>(),   make_ops<4, 4>(),
    make_ops<5, 5>(),   make_ops<6, 6>(),   make_ops<7, 7>(),   make_ops<8, 8>(),
    make_ops<11, 11>(), make_ops<12, 12>(), make_ops<13, 13>(), make_ops<14, 14>(),
    make_ops<15, 15>(), make_ops<16, 16>(), make_ops<17, 17>(), make_ops<18, 18>(),
    make_ops<19, 19>(), make_ops<1, 2>(),   make_ops<2, 1>(),   make_ops<2, 3>(),
    make_ops<3, 2>(),
};

static const Ops* find_ops(int d, int q) {
  for (const Ops& o : kOps)
    if (o.D == d && o.Q == q) return &o;
  return nullptr;
}

// ------------------------------------------------------------------------
// the handle
// ------------------------------------------------------------------------
struct srmdp {
  srmdp_config cfg{};
  std::vector<double> params;  // [dyn | theta | g]
  std::vector<double> tabs;    // host copy of the grid tables
  int d = 0, q = 0, N = 0, C = 0, B = 0, B_pad = 0;
  int64_t K = 0, K_pad = 0, chunk = 0, k_begin = 0, k_end = 0, M = 0;
  double C_y = 0, C_z = 0;
  bool smallness_ok = true;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  double* d_table = nullptr;
  double* d_replica = nullptr;       // P2P_SELF_PEER test mode: the table the kernels read
  double* d_params = nullptr;
  double* d_tabs = nullptr;
  double* d_scratch = nullptr;
  unsigned long long* d_counters = nullptr;   // [lp0 fallbacks, exact z evals, exact z_i]
  double* d_io = nullptr;
  size_t io_cap = 0;
  DevProblem dp{};
  const Ops* ops = nullptr;          // static kernels of (d, q), or
  const JitKernels* jit = nullptr;   // the NVRTC build (user problem / other (d, q))
  std::string user_src;
  int grid = 0, ctas = 0, sms = 0;
  size_t smem = 0;
  cudaGraphExec_t graph = nullptr;
  ncclComm_t comm = nullptr;
  bool solved = false;
  // fused exchange (SRMDP_FLAG_P2P_EXCHANGE)
  bool p2p = false;
  bool nvls = false;                 // SRMDP_FLAG_NVLS_EXCHANGE: table bound to a multicast object
  NvlsTable nv;
  unsigned* mc_flags = nullptr;      // multicast mapping of the flag arrays
  void* ipc_base = nullptr;          // cudaMalloc'd [table | flags], IPC-exported
  size_t ipc_bytes = 0;
  unsigned* d_flags = nullptr;       // own flags [N+1][world]
  unsigned* d_epoch = nullptr;
  unsigned* d_xerr = nullptr;        // 1 + slot of a timed-out flag wait, else 0
  unsigned* d_xw_counter = nullptr;  // CTAs done in the current step launch (in-kernel exchange)
  uint64_t xchg_timeout_ns = 0;
  FlagPtrs fptr{};
  std::vector<void*> opened;         // peers' bases opened through IPC
  int launches_per_solve = 0;
  int valid_from = 0;          // slices valid_from .. N-1 are present (N: none)
  int graph_launches = 0;
  bool pending = false;
  std::chrono::steady_clock::time_point t_submit;
  nvtxRangeId_t nvtx_solve = 0;
  int last_hi = 0, last_lo = 0;
  std::vector<double> step_ms, xchg_ms;
  std::vector<cudaEvent_t> ev;       // [2N] step kernels, then [2N] exchanges
  srmdp_stats_t st{};
  mutable std::string err = "no error";
};

static srmdp_status cuda_fail(const srmdp_t* h, cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  if (h) h->err = m; else g_create_err = m;
  return (e == cudaErrorMemoryAllocation) ? SRMDP_E_NOMEM : SRMDP_E_CUDA;
}

// Device memory of the handles comes from one process-wide stream-ordered
// pool per device that keeps its pages (release threshold = max): creating and
// destroying handles (one solve per request in a serving loop, the e2e bench)
// reuses memory instead of cudaMalloc / cudaFree, whose unmapping of the
// 240 MB cfg4 table took up to ~0.4 s (tools/e2e_breakdown.py).
static cudaError_t device_pool(int dev, cudaMemPool_t* out) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lock(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) { *out = it->second; return cudaSuccess; }
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool;
  cudaError_t e = cudaMemPoolCreate(&pool, &props);
  if (e != cudaSuccess) return e;
  uint64_t keep = ~0ull;
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  if (e != cudaSuccess) return e;
  pools[dev] = pool;
  *out = pool;
  return cudaSuccess;
}

// IPC-exportable allocations of the fused exchange ([table | flags],
// cudaMalloc: pool memory cannot be exported with cudaIpcGetMemHandle) are
// kept the same way: freed blocks are cached per (device, size) and reused.
static std::mutex g_ipc_mu;
static std::multimap<std::pair<int, size_t>, void*> g_ipc_free;

static cudaError_t ipc_alloc(int dev, void** p, size_t bytes) {
  {
    std::lock_guard<std::mutex> lock(g_ipc_mu);
    auto it = g_ipc_free.find({dev, bytes});
    if (it != g_ipc_free.end()) {
      *p = it->second;
      g_ipc_free.erase(it);
      return cudaSuccess;
    }
  }
  return cudaMalloc(p, bytes);
}

static void ipc_release(int dev, void* p, size_t bytes) {
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  g_ipc_free.insert({{dev, bytes}, p});
}

template <typename T>
static cudaError_t dalloc(const srmdp_t* h, T** p, size_t bytes) {
  cudaMemPool_t pool;
  cudaError_t e = device_pool(h->cfg.device, &pool);
  if (e != cudaSuccess) return e;
  return cudaMallocFromPoolAsync((void**)p, bytes < 16 ? 16 : bytes, pool, h->stream);
}

static void dfree(const srmdp_t* h, void* p) {
  if (p) cudaFreeAsync(p, h->stream);
}

#define CK(h, call, what)                                  \
  do {                                                     \
    cudaError_t _e = (call);                               \
    if (_e != cudaSuccess) return cuda_fail((h), _e, what); \
  } while (0)

// A failed collective leaves the communicator unusable (peers may be blocked
// in the same collective): abort it so no rank hangs, drop the table.
static srmdp_status nccl_fail(srmdp_t* h, const char* what, ncclResult_t r) {
  h->err = std::string(what) + ": " + nccl().GetErrorString(r) + " (communicator aborted; recreate the handle)";
  if (h->comm) {
    nccl().CommAbort(h->comm);
    h->comm = nullptr;
  }
  h->valid_from = h->N;
  h->solved = false;
  return SRMDP_E_NCCL;
}

extern "C" srmdp_status srmdp_shard_plan(int64_t K, int world, int rank, int64_t out[4]) {
  if (K < 1 || world < 1 || rank < 0 || rank >= world || !out) return SRMDP_E_ARG;
  const int64_t chunk = (K + world - 1) / world;
  const int64_t K_pad = chunk * world;
  int64_t b = (int64_t)rank * chunk, e = b + chunk;
  if (b > K) b = K;
  if (e > K) e = K;
  out[0] = b;
  out[1] = e;
  out[2] = chunk;
  out[3] = K_pad;
  return SRMDP_OK;
}

static int expected_params(int which, int kind, int d, int q) {
  if (which == 0)
    return (kind == SRMDP_DYN_BM || kind == SRMDP_DYN_USER) ? 0
           : (kind == SRMDP_DYN_GBM || kind == SRMDP_DYN_GBM_EXACT) ? 2 * d
                                                                    : d + d * d + d * q;
  if (which == 1) return kind == SRMDP_F_LINEAR ? 2 + q : 0;
  return kind == SRMDP_G_AFFINE ? 1 + d : 0;
}

static bool uses_user(const srmdp_config* c) {
  return c->dyn.kind == SRMDP_DYN_USER || c->driver.kind == SRMDP_F_USER || c->terminal.kind == SRMDP_G_USER;
}

// NVRTC build needed: a user problem, a (d, q) outside the compiled set, the
// equal-probability grid above d = 8, or forced (SRMDP_FLAG_JIT).
static bool needs_jit(const srmdp_config* c) {
  const Ops* o = find_ops(c->d, c->q);
  return uses_user(c) || !o || (c->grid == 1 && !o->step_eq) || (c->flags & SRMDP_FLAG_JIT);
}

static srmdp_status validate(const srmdp_config* c, std::string& err) {
  auto bad = [&](srmdp_status s, const char* m) { err = m; return s; };
  if (!c) return bad(SRMDP_E_ARG, "cfg is NULL");
  if (c->d < 1 || c->q < 1) return bad(SRMDP_E_ARG, "d and q must be >= 1");
  if (c->N < 1) return bad(SRMDP_E_ARG, "N must be >= 1");
  if (!(c->T > 0)) return bad(SRMDP_E_ARG, "T must be > 0");
  if (c->cells_per_dim < 1) return bad(SRMDP_E_ARG, "cells_per_dim must be >= 1");
  if (!(c->L > 0)) return bad(SRMDP_E_ARG, "L must be > 0");
  if (!(c->mu > 0)) return bad(SRMDP_E_ARG, "mu must be > 0");
  if (c->M < c->d + 1) return bad(SRMDP_E_PRECOND, "M < d+1: the LP1 OLS needs M >= d+1 (P:312)");
  if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return bad(SRMDP_E_ARG, "bad rank/world");
  const bool loopback = c->flags & SRMDP_FLAG_LOOPBACK;
  if (((c->world > 1 && !loopback) || (c->flags & SRMDP_FLAG_FORCE_NCCL)) && !c->nccl_unique_id)
    return bad(SRMDP_E_ARG, "the NCCL exchange needs nccl_unique_id");
  if (loopback && (c->flags & SRMDP_FLAG_FORCE_NCCL)) return bad(SRMDP_E_ARG, "LOOPBACK and FORCE_NCCL exclude each other");
  if ((c->flags & SRMDP_FLAG_P2P_EXCHANGE) && (loopback || c->world > kMaxRanks))
    return bad(SRMDP_E_ARG, "P2P_EXCHANGE needs world <= 8 and excludes LOOPBACK");
  if ((c->flags & SRMDP_FLAG_P2P_SELF_PEER) && (!(c->flags & SRMDP_FLAG_P2P_EXCHANGE) || c->world != 1))
    return bad(SRMDP_E_ARG, "P2P_SELF_PEER is a world == 1 test mode of P2P_EXCHANGE");
  if ((c->flags & SRMDP_FLAG_NVLS_EXCHANGE) &&
      (loopback || (c->flags & SRMDP_FLAG_P2P_EXCHANGE) || c->world > kMaxRanks))
    return bad(SRMDP_E_ARG, "NVLS_EXCHANGE needs world <= 8 and excludes LOOPBACK and P2P_EXCHANGE");
  if (c->dyn.kind < 0 || c->dyn.kind > 4 || c->driver.kind < 0 || c->driver.kind > 3 || c->terminal.kind < 0 ||
      c->terminal.kind > 2)
    return bad(SRMDP_E_ARG, "unknown problem family kind");
  if (uses_user(c) && !c->user_src) return bad(SRMDP_E_ARG, "a *_USER kind needs user_src");
  if (c->n_user_params < 0 || (c->n_user_params > 0 && !c->user_params))
    return bad(SRMDP_E_ARG, "user_params must hold n_user_params doubles");
  if ((c->dyn.kind == SRMDP_DYN_BM || c->dyn.kind == SRMDP_DYN_GBM || c->dyn.kind == SRMDP_DYN_GBM_EXACT) &&
      c->q != c->d)
    return bad(SRMDP_E_ARG, "BM and GBM dynamics need q == d");
  const srmdp_fn* fns[3] = {&c->dyn, &c->driver, &c->terminal};
  for (int w = 0; w < 3; ++w) {
    const int need = expected_params(w, fns[w]->kind, c->d, c->q);
    if (fns[w]->n_params != need || (need > 0 && !fns[w]->params))
      return bad(SRMDP_E_ARG, "parameter count does not match the family layout (srmdp.h)");
  }
  if (c->N >= (1 << 24)) return bad(SRMDP_E_UNSUPPORTED, "N >= 2^24 (Philox counter layout)");
  if (c->M >= (int64_t)1 << 32) return bad(SRMDP_E_UNSUPPORTED, "M >= 2^32 (Philox counter layout)");
  if (c->cells_per_dim > 2048) return bad(SRMDP_E_UNSUPPORTED, "cells_per_dim > 2048");
  double K = 1;
  for (int l = 0; l < c->d; ++l) K *= c->cells_per_dim;
  if (K >= 4294967296.0) return bad(SRMDP_E_UNSUPPORTED, "K = C^d >= 2^32 (Philox counter layout)");
  if (c->d > 32 || c->q > 32) return bad(SRMDP_E_UNSUPPORTED, "d, q <= 32");
  if (c->grid != 0 && c->grid != 1) return bad(SRMDP_E_ARG, "grid must be 0 (equal-size) or 1 (equal-probability)");
  return SRMDP_OK;
}

// Prop. bound (eq. prop:bound).
static void bounds(double C_g, double C_f, double L_f, int q, double T, int N, double* cy, double* cz, bool* ok) {
  const double dt = T / (double)N;
  const double Lf2 = L_f * L_f;
  const double a = Lf2 > 1.0 ? Lf2 : 1.0;
  const double Tv = T > 1.0 ? T : 1.0;
  *cy = std::exp(T / 4.0 + 6.0 * q * a * Tv) * (C_g + T * C_f / (2.0 * std::sqrt((double)q)));
  *cz = *cy / std::sqrt(dt);
  *ok = dt * Lf2 <= 1.0 / (12.0 * q);
}

// Inside stream capture an event must be an external record node to time
// the captured kernel; outside capture a plain record.
static cudaError_t record_event(srmdp_t* h, cudaEvent_t e) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t r = cudaStreamIsCapturing(h->stream, &cs);
  if (r != cudaSuccess) return r;
  return (cs == cudaStreamCaptureStatusActive) ? cudaEventRecordWithFlags(e, h->stream, cudaEventRecordExternal)
                                               : cudaEventRecord(e, h->stream);
}

// Step-kernel attributes and residency: the static instantiation or the NVRTC
// build (sized with the same step_smem_bytes formula).
// The static kernel of this problem: the BM-specialised one for X = W on the
// equal-size grid (the §5.1 benchmark), else the runtime-dynamics kernel.
static bool use_bm_kernel(const srmdp_t* h) {
  // the BM kernels compile only the range-proved start-point reciprocal (SRMDP_BM_FAST_ONLY)
  return !h->jit && !h->cfg.grid && h->cfg.dyn.kind == SRMDP_DYN_BM && h->ops->step_bm &&
         (!SRMDP_BM_FAST_ONLY || h->dp.rcp_fast);
}

// Fused exchanges on the BM kernels, opt-in (SRMDP_FLAG_INKERNEL_FLAGS): the
// flags in the step kernel itself (wait after the table-free head of the
// first round, publish from the last CTA) instead of a signal and a wait
// kernel per step. Measured on one GPU (cfg4): the step kernels are 1.4%
// slower with the head / tail split compiled in, against 0.35 ms per solve
// for the separate flag kernels -- so the separate kernels are the default.
static bool use_xw(const srmdp_t* h) {
  return (h->p2p || h->nvls) && use_bm_kernel(h) && h->ops->step_bm_xw && (h->cfg.flags & SRMDP_FLAG_INKERNEL_FLAGS);
}

static cudaError_t prepare_step(srmdp_t* h) {
  if (use_xw(h)) return h->ops->prepare_bm_xw(h->C, &h->smem, &h->ctas);
  if (use_bm_kernel(h)) return h->ops->prepare_bm(h->C, &h->smem, &h->ctas);
  if (!h->jit) return (h->cfg.grid ? h->ops->prepare_eq : h->ops->prepare)(h->C, &h->smem, &h->ctas);
  const void* k = (const void*)h->jit->step[h->cfg.grid ? 1 : 0];
  h->smem = step_smem_bytes(h->d, h->q, h->C);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->smem);
  if (e != cudaSuccess) return e;
  return fit_carveout(k, h->smem, step_threads(h->d), &h->ctas);
}

static void launch_step(srmdp_t* h, int i, int64_t kb, int64_t nk) {
  if (use_xw(h)) {
    h->ops->step_bm_xw(h->dp, i, kb, nk, h->grid, h->smem, h->stream);
    return;
  }
  if (use_bm_kernel(h)) {
    h->ops->step_bm(h->dp, i, kb, nk, h->grid, h->smem, h->stream);
    return;
  }
  if (!h->jit) {
    (h->cfg.grid ? h->ops->step_eq : h->ops->step)(h->dp, i, kb, nk, h->grid, h->smem, h->stream);
    return;
  }
  void* args[] = {&h->dp, &i, &kb, &nk};
  cudaLaunchKernel((const void*)h->jit->step[h->cfg.grid ? 1 : 0], dim3(h->grid), dim3(step_threads(h->d)), args, h->smem,
                   h->stream);   // errors surface through cudaGetLastError below
}

static srmdp_status enqueue_sweep(srmdp_t* h, int i_hi, int i_lo) {
  const bool timed = h->cfg.flags & SRMDP_FLAG_TIME_KERNELS;
  CK(h, cudaMemsetAsync(h->d_counters, 0, 3 * sizeof(unsigned long long), h->stream), "memset");
  const int64_t nk = h->k_end - h->k_begin;
  const bool loopback = h->cfg.flags & SRMDP_FLAG_LOOPBACK;
  h->launches_per_solve = 0;
  const bool xw = use_xw(h);
  h->dp.xw_wait_below = i_hi;   // the sweep's first step reads slices of an earlier sweep: no wait
  if (h->p2p || h->nvls) {
    // new epoch; entry barrier: no rank stores into a peer's table before
    // that peer has entered this sweep (slot N)
    epoch_kernel<<<1, 1, 0, h->stream>>>(h->d_epoch);
    if (h->nvls) exchange_signal_mc_kernel<<<1, 32, 0, h->stream>>>(h->mc_flags, h->cfg.world, h->cfg.rank, h->N, h->d_epoch);
    else exchange_signal_kernel<<<1, kMaxRanks, 0, h->stream>>>(h->fptr, h->cfg.world, h->cfg.rank, h->N, h->d_epoch);
    exchange_wait_kernel<<<1, kMaxRanks, 0, h->stream>>>(h->d_flags, h->cfg.world, h->N, h->d_epoch, h->d_xerr,
                                                         h->xchg_timeout_ns);
    CK(h, cudaGetLastError(), "exchange entry barrier");
  }
  for (int i = i_hi; i >= i_lo; --i) {
    char rname[48];
    snprintf(rname, sizeof(rname), "srmdp step i=%d", i);
    nvtxRangePushA(rname);   // per time step (launch + exchange); inside graph capture it tags the nodes
    struct Pop { ~Pop() { nvtxRangePop(); } } pop_at_scope_end;
    if (timed) CK(h, record_event(h, h->ev[2 * i]), "event");
    if (loopback) {
      for (int r = 0; r < h->cfg.world; ++r) {   // shards in sequence on one table
        int64_t plan[4];
        srmdp_shard_plan(h->K, h->cfg.world, r, plan);
        if (plan[1] > plan[0]) {
          launch_step(h, i, plan[0], plan[1] - plan[0]);
          ++h->launches_per_solve;
        }
      }
    } else if (nk > 0) {
      launch_step(h, i, h->k_begin, nk);
      ++h->launches_per_solve;
    }
    CK(h, cudaGetLastError(), "step kernel launch");
    if (timed) CK(h, record_event(h, h->ev[2 * i + 1]), "event");
    const bool xchg = (h->p2p || h->nvls || h->comm) && !(xw && i != i_lo);
    if (timed && xchg) CK(h, record_event(h, h->ev[2 * h->N + 2 * i]), "event");
    if (xw) {
      // the step kernels wait / publish themselves; the sweep's last slice is
      // complete everywhere once every rank's last CTA has published it
      if (i == i_lo) {
        exchange_wait_kernel<<<1, kMaxRanks, 0, h->stream>>>(h->d_flags, h->cfg.world, i, h->d_epoch, h->d_xerr,
                                                             h->xchg_timeout_ns);
        CK(h, cudaGetLastError(), "exchange flags");
      }
    } else if (h->p2p || h->nvls) {
      // blocks of slice i are in every table once all ranks have signalled
      if (h->nvls) exchange_signal_mc_kernel<<<1, 32, 0, h->stream>>>(h->mc_flags, h->cfg.world, h->cfg.rank, i, h->d_epoch);
      else exchange_signal_kernel<<<1, kMaxRanks, 0, h->stream>>>(h->fptr, h->cfg.world, h->cfg.rank, i, h->d_epoch);
      exchange_wait_kernel<<<1, kMaxRanks, 0, h->stream>>>(h->d_flags, h->cfg.world, i, h->d_epoch, h->d_xerr,
                                                           h->xchg_timeout_ns);
      CK(h, cudaGetLastError(), "exchange flags");
    } else if (h->comm) {
      double* slice = h->d_table + (size_t)i * h->K_pad * h->B_pad;
      const size_t cnt = (size_t)h->chunk * h->B_pad;
      ncclResult_t r = nccl().AllGather(slice + (size_t)h->cfg.rank * cnt, slice, cnt, ncclDouble, h->comm, h->stream);
      if (r != ncclSuccess) return nccl_fail(h, "ncclAllGather", r);
    }
    if (timed && xchg) CK(h, record_event(h, h->ev[2 * h->N + 2 * i + 1]), "event");
  }
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_create(const srmdp_config* cfg, srmdp_t** out) {
  if (!out) { g_create_err = "out is NULL"; return SRMDP_E_ARG; }
  *out = nullptr;
  std::string verr;
  srmdp_status vs = validate(cfg, verr);
  if (vs != SRMDP_OK) { g_create_err = verr; return vs; }
  srmdp_t* h = new srmdp();
  h->cfg = *cfg;
  h->d = cfg->d; h->q = cfg->q; h->N = cfg->N; h->C = cfg->cells_per_dim; h->M = cfg->M;
  h->K = 1;
  for (int l = 0; l < h->d; ++l) h->K *= h->C;
  h->B = (h->q + 1) * (h->d + 1);
  h->B_pad = block_stride(h->d, h->q);
  int64_t plan[4];
  srmdp_shard_plan(h->K, cfg->world, (cfg->flags & SRMDP_FLAG_LOOPBACK) ? 0 : cfg->rank, plan);
  h->k_begin = plan[0]; h->k_end = plan[1]; h->chunk = plan[2]; h->K_pad = plan[3];
  if (cfg->flags & SRMDP_FLAG_LOOPBACK) { h->k_begin = 0; h->k_end = h->K; }
  h->ops = find_ops(h->d, h->q);
  if (needs_jit(cfg)) {
    h->user_src = cfg->user_src ? cfg->user_src : "";
    std::string jerr;
    h->jit = jit_kernels(h->d, h->q, cfg->dyn.kind == SRMDP_DYN_USER, cfg->driver.kind == SRMDP_F_USER,
                         cfg->terminal.kind == SRMDP_G_USER, h->user_src, jerr);
    if (!h->jit) {
      g_create_err = jerr;
      delete h;
      return SRMDP_E_JIT;
    }
    h->ops = nullptr;
  }
  h->cfg.user_src = nullptr;
  // truncation constants: override, else eq. prop:bound (reading R5)
  double by, bz;
  bool ok;
  bounds(cfg->C_g, cfg->C_f, cfg->L_f, h->q, cfg->T, h->N, &by, &bz, &ok);
  h->smallness_ok = ok;
  h->C_y = std::isnan(cfg->C_y_override) ? by : cfg->C_y_override;
  h->C_z = std::isnan(cfg->C_z_override) ? bz : cfg->C_z_override;
  // deep-copy parameters: [dyn | theta | g | user]
  const int nd = cfg->dyn.n_params, nf = cfg->driver.n_params, ng = cfg->terminal.n_params;
  const int nu = cfg->n_user_params;
  h->params.assign(nd + (nf > 2 ? nf - 2 : 0) + ng + nu + 1, 0.0);
  for (int t = 0; t < nd; ++t) h->params[t] = cfg->dyn.params[t];
  for (int t = 2; t < nf; ++t) h->params[nd + t - 2] = cfg->driver.params[t];
  const int goff = nd + (nf > 2 ? nf - 2 : 0);
  for (int t = 0; t < ng; ++t) h->params[goff + t] = cfg->terminal.params[t];
  const int uoff = goff + ng;
  for (int t = 0; t < nu; ++t) h->params[uoff + t] = cfg->user_params[t];
  h->cfg.dyn.params = h->cfg.driver.params = h->cfg.terminal.params = nullptr;
  h->cfg.user_params = nullptr;
  h->cfg.nccl_unique_id = nullptr;

  auto fail = [&](srmdp_status s) {
    g_create_err = h->err;
    srmdp_destroy(h);
    return s;
  };
  cudaError_t e = cudaSetDevice(cfg->device);
  if (e != cudaSuccess) { cuda_fail(h, e, "cudaSetDevice"); return fail(SRMDP_E_CUDA); }
  if (cfg->stream) {
    h->stream = (cudaStream_t)cfg->stream;
  } else {
    e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { cuda_fail(h, e, "cudaStreamCreate"); return fail(SRMDP_E_CUDA); }
    h->own_stream = true;
  }
  e = cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, cfg->device);
  if (e != cudaSuccess) { cuda_fail(h, e, "device attribute"); return fail(SRMDP_E_CUDA); }

  const size_t table_bytes = (size_t)h->N * h->K_pad * h->B_pad * sizeof(double);
  std::vector<double> tabs = grid_tables(h->C, cfg->L, cfg->mu, cfg->grid != 0);
  {   // the smallest start-point p of the grid is Fe[c] + U (Fe[c+1] - Fe[c]) >= 2^-53 min_c(Fe[c+1] - Fe[c])
      // for the leftmost cell (Fe[0] = 0), >= Fe[1] for the others: the fast 1/p is exact above 2^-1000
      // (decided before prepare_step: the BM kernels need it)
    double mind = 1.0;
    for (int c = 0; c < h->C; ++c) mind = std::min(mind, tabs[c + 1] - tabs[c]);
    h->dp.rcp_fast = (mind > 0x1p-946) ? 1 : 0;
  }
  h->p2p = cfg->flags & SRMDP_FLAG_P2P_EXCHANGE;
  h->nvls = cfg->flags & SRMDP_FLAG_NVLS_EXCHANGE;
  {   // bounded flag waits of the fused exchange (exchange_wait_kernel)
    const char* t = getenv("SRMDP_EXCHANGE_TIMEOUT_S");
    const double sec = (t && atof(t) > 0) ? atof(t) : 60.0;
    h->xchg_timeout_ns = (uint64_t)(sec * 1e9);
  }
  const size_t flags_off = (table_bytes + 255) & ~(size_t)255;
  const size_t flags_bytes = (size_t)(h->N + 1) * cfg->world * sizeof(unsigned);
  if (h->p2p) {   // IPC-exportable allocation: [table | flags]
    h->ipc_bytes = flags_off + flags_bytes;
    if ((e = ipc_alloc(cfg->device, &h->ipc_base, h->ipc_bytes)) != cudaSuccess ||
        (e = cudaMemsetAsync((char*)h->ipc_base + flags_off, 0, flags_bytes, h->stream)) != cudaSuccess ||
        (e = dalloc(h, &h->d_epoch, sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMemsetAsync(h->d_epoch, 0, sizeof(unsigned), h->stream)) != cudaSuccess ||
        (e = dalloc(h, &h->d_xerr, sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMemsetAsync(h->d_xerr, 0, sizeof(unsigned), h->stream)) != cudaSuccess) {
      cuda_fail(h, e, "p2p table alloc");
      return fail(SRMDP_E_NOMEM);
    }
    h->d_table = (double*)h->ipc_base;
    h->d_flags = (unsigned*)((char*)h->ipc_base + flags_off);
    h->fptr.f[cfg->rank] = h->d_flags;
  } else if (h->nvls) {   // the table comes from nvls_create below (after the communicator exists)
    if ((e = dalloc(h, &h->d_epoch, sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMemsetAsync(h->d_epoch, 0, sizeof(unsigned), h->stream)) != cudaSuccess ||
        (e = dalloc(h, &h->d_xerr, sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMemsetAsync(h->d_xerr, 0, sizeof(unsigned), h->stream)) != cudaSuccess) {
      cuda_fail(h, e, "nvls flag alloc");
      return fail(SRMDP_E_NOMEM);
    }
  } else if ((e = dalloc(h, &h->d_table, table_bytes)) != cudaSuccess) {
    cuda_fail(h, e, "table alloc");
    return fail(SRMDP_E_NOMEM);
  }
  if ((e = dalloc(h, &h->d_params, h->params.size() * sizeof(double))) != cudaSuccess ||
      (e = dalloc(h, &h->d_tabs, tabs.size() * sizeof(double))) != cudaSuccess ||
      (e = dalloc(h, &h->d_counters, 3 * sizeof(unsigned long long))) != cudaSuccess) {
    cuda_fail(h, e, "alloc");
    return fail(SRMDP_E_NOMEM);
  }
  if ((e = cudaMemcpyAsync(h->d_params, h->params.data(), h->params.size() * sizeof(double), cudaMemcpyHostToDevice,
                           h->stream)) != cudaSuccess ||
      (e = cudaMemcpyAsync(h->d_tabs, tabs.data(), tabs.size() * sizeof(double), cudaMemcpyHostToDevice,
                           h->stream)) != cudaSuccess ||
      (e = cudaStreamSynchronize(h->stream)) != cudaSuccess) {   // pageable sources: complete before return
    cuda_fail(h, e, "upload");
    return fail(SRMDP_E_CUDA);
  }
  h->tabs = tabs;

  // launch configuration: persistent CTAs; the pass-2 records go to a per-CTA
  // global scratch so shared memory stays small and the L1 keeps room for the
  // gathered coefficient lines (3 x 256 threads per SM at d <= 8, 4 x 128 above)
  e = prepare_step(h);
  if (e != cudaSuccess || h->ctas < 1) {
    if (e == cudaSuccess) h->err = "step kernel does not fit on an SM";
    else cuda_fail(h, e, "kernel attributes");
    return fail(SRMDP_E_UNSUPPORTED);
  }
  const int64_t nk = (cfg->flags & SRMDP_FLAG_LOOPBACK) ? h->chunk : h->k_end - h->k_begin;
  const int64_t full = (int64_t)h->ctas * h->sms;
  h->grid = (int)(nk < full ? (nk > 0 ? nk : 1) : full);
  if ((e = dalloc(h, &h->d_scratch, (size_t)h->grid * h->M * scratch_stride(h->d) * sizeof(double))) != cudaSuccess) {
    cuda_fail(h, e, "scratch alloc");
    return fail(SRMDP_E_NOMEM);
  }

  DevProblem& P = h->dp;
  P.d = h->d; P.q = h->q; P.N = h->N; P.C = h->C; P.B = h->B; P.B_pad = h->B_pad;
  P.dyn = cfg->dyn.kind; P.fk = cfg->driver.kind; P.gk = cfg->terminal.kind;
  P.nbd = (h->d + 1) / 2; P.nbq = (h->q + 1) / 2;
  P.lp0 = cfg->lp0 ? 1 : 0;
  P.equi = cfg->grid ? 1 : 0;
  P.K = h->K; P.K_pad = h->K_pad; P.M = h->M;
  P.T = cfg->T;
  P.dt = cfg->T / (double)h->N;
  P.sdt = std::sqrt(P.dt);
  P.L = cfg->L;
  P.inv_delta = (double)h->C / (2.0 * cfg->L);
  P.delta = (2.0 * cfg->L) / (double)h->C;     // as grid_tables (centers)
  P.half_delta = P.delta * 0.5;

  P.neg_inv_mu = -(1.0 / cfg->mu);
  P.C_y = h->C_y; P.C_z = h->C_z;
  P.f_a = (cfg->driver.kind == SRMDP_F_LINEAR) ? cfg->driver.params[0] : 0.0;
  P.f_c = (cfg->driver.kind == SRMDP_F_LINEAR) ? cfg->driver.params[1] : 0.0;
  P.f_cq = (2.0 + (double)h->q) / (2.0 * (double)h->q);
  P.key0 = (uint32_t)(cfg->seed & 0xffffffffu);
  P.key1 = (uint32_t)(cfg->seed >> 32);
  for (int r = 0; r < 10; ++r) {   // Philox round keys (docs/streams.md §1)
    P.rkey.k0[r] = P.key0 + (uint32_t)r * 0x9E3779B9u;
    P.rkey.k1[r] = P.key1 + (uint32_t)r * 0xBB67AE85u;
  }
  P.inv_dt = 1.0 / P.dt;
  P.C_z_safe = h->C_z * (1.0 - 0x1p-40);
  P.dyn_params = h->d_params;
  P.theta = h->d_params + nd;
  P.g_params = h->d_params + goff;
  P.user_params = h->d_params + uoff;
  P.tabs = h->d_tabs;
  P.table = h->d_table;
  if (cfg->flags & SRMDP_FLAG_P2P_SELF_PEER) {
    // test mode of the fused exchange on one GPU: the kernels read and store
    // into a replica, and the epilogue's peer-store loop (n_peers = 1) writes
    // every block into the handle's own IPC table, which srmdp_coeffs reads --
    // so that table holds only what the peer stores delivered
    if ((e = dalloc(h, &h->d_replica, table_bytes)) != cudaSuccess) {
      cuda_fail(h, e, "replica alloc");
      return fail(SRMDP_E_NOMEM);
    }
    P.table = h->d_replica;
    P.peer_table[0] = h->d_table;
    P.n_peers = 1;
  }
  P.by_scratch = h->d_scratch;
  P.counters = h->d_counters;

  if (cfg->flags & SRMDP_FLAG_TIME_KERNELS) {
    h->ev.resize(4 * h->N);
    for (auto& x : h->ev) cudaEventCreate(&x);
  }
  if ((cfg->world > 1 && !(cfg->flags & SRMDP_FLAG_LOOPBACK)) || (cfg->flags & SRMDP_FLAG_FORCE_NCCL)) {
    NcclApi& api = nccl();
    if (!api.ok) { h->err = api.err; return fail(SRMDP_E_NCCL); }
    ncclUniqueId id;
    memcpy(&id, cfg->nccl_unique_id, sizeof(id));
    ncclResult_t r = api.CommInitRank(&h->comm, cfg->world, id, cfg->rank);
    if (r != ncclSuccess) { h->err = std::string("ncclCommInitRank: ") + api.GetErrorString(r); return fail(SRMDP_E_NCCL); }
  }
  if (h->nvls) {
    // [table | flags] bound to a multicast object over the ranks' GPUs (nvls.h);
    // the communicator serves as the rendezvous barrier
    char* bar = nullptr;
    if ((e = dalloc(h, &bar, 16 * cfg->world)) != cudaSuccess) { cuda_fail(h, e, "nvls barrier"); return fail(SRMDP_E_NOMEM); }
    auto barrier = [&]() -> bool {
      if (!h->comm) return true;
      if (nccl().AllGather(bar, bar, 16, ncclChar, h->comm, h->stream) != ncclSuccess) return false;
      return cudaStreamSynchronize(h->stream) == cudaSuccess;
    };
    std::string key;
    if (cfg->world > 1) {
      uint64_t kh = 0xcbf29ce484222325ull;
      const unsigned char* u = (const unsigned char*)cfg->nccl_unique_id;
      for (int t = 0; t < 128; ++t) { kh ^= u[t]; kh *= 0x100000001b3ull; }
      char buf[32];
      snprintf(buf, sizeof(buf), "%016llx", (unsigned long long)kh);
      key = buf;
    }
    std::string nerr;
    const bool ok = nvls_create(cfg->device, flags_off + flags_bytes, cfg->world, cfg->rank, key, barrier, &h->nv, nerr);
    if (ok) {
      h->d_table = (double*)h->nv.uc;
      h->d_flags = (unsigned*)((char*)h->nv.uc + flags_off);
      h->mc_flags = (unsigned*)((char*)h->nv.mc + flags_off);
      e = cudaMemsetAsync(h->d_flags, 0, flags_bytes, h->stream);
    }
    const bool ok2 = ok && e == cudaSuccess && barrier();   // every rank's flags zeroed before anyone signals
    dfree(h, bar);
    if (!ok2) { h->err = ok ? "nvls flag init" : nerr; return fail(ok ? SRMDP_E_CUDA : SRMDP_E_UNSUPPORTED); }
    h->dp.table = h->d_table;
    h->dp.mc_table = (double*)h->nv.mc;
  }
  if (h->p2p && cfg->world > 1) {
    // exchange the IPC handles of [table | flags] over the communicator, open the peers'
    if (!h->comm) { h->err = "P2P_EXCHANGE with world > 1 needs nccl_unique_id"; return fail(SRMDP_E_ARG); }
    cudaIpcMemHandle_t mine;
    if ((e = cudaIpcGetMemHandle(&mine, h->ipc_base)) != cudaSuccess) { cuda_fail(h, e, "ipc handle"); return fail(SRMDP_E_CUDA); }
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    std::vector<cudaIpcMemHandle_t> all(cfg->world);
    char* dbuf = nullptr;
    if ((e = dalloc(h, &dbuf, hb * (cfg->world + 1))) != cudaSuccess ||
        (e = cudaMemcpyAsync(dbuf, &mine, hb, cudaMemcpyHostToDevice, h->stream)) != cudaSuccess) {
      cuda_fail(h, e, "ipc exchange");
      return fail(SRMDP_E_CUDA);
    }
    ncclResult_t r = nccl().AllGather(dbuf, dbuf + hb, hb, ncclChar, h->comm, h->stream);
    if (r != ncclSuccess) { h->err = std::string("ncclAllGather (ipc handles): ") + nccl().GetErrorString(r); return fail(SRMDP_E_NCCL); }
    e = cudaMemcpyAsync(all.data(), dbuf + hb, hb * cfg->world, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    dfree(h, dbuf);
    if (e != cudaSuccess) { cuda_fail(h, e, "ipc exchange"); return fail(SRMDP_E_CUDA); }
    int np = 0;
    for (int r2 = 0; r2 < cfg->world; ++r2) {
      if (r2 == cfg->rank) continue;
      void* base = nullptr;
      if ((e = cudaIpcOpenMemHandle(&base, all[r2], cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess) {
        cuda_fail(h, e, "cudaIpcOpenMemHandle (peers must share an NVLink domain)");
        return fail(SRMDP_E_CUDA);
      }
      h->opened.push_back(base);
      h->dp.peer_table[np++] = (double*)base;
      h->fptr.f[r2] = (unsigned*)((char*)base + flags_off);
    }
    h->dp.n_peers = np;
  }
  if (h->p2p || h->nvls) {   // in-kernel exchange flags (use_xw)
    if ((e = dalloc(h, &h->d_xw_counter, sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMemsetAsync(h->d_xw_counter, 0, sizeof(unsigned), h->stream)) != cudaSuccess ||
        (e = cudaStreamSynchronize(h->stream)) != cudaSuccess) {
      cuda_fail(h, e, "exchange counter");
      return fail(SRMDP_E_NOMEM);
    }
    DevProblem& Q = h->dp;
    Q.xw_counter = h->d_xw_counter;
    Q.xw_own = h->d_flags;
    for (int r = 0; r < cfg->world && r <= kMaxPeers; ++r) Q.xw_flags[r] = h->fptr.f[r];
    Q.xw_mc = h->nvls ? h->mc_flags : nullptr;
    Q.xw_epoch = h->d_epoch;
    Q.xw_err = h->d_xerr;
    Q.xw_world = cfg->world;
    Q.xw_rank = cfg->rank;
  }
  h->valid_from = h->N;
  h->st.path_steps = (uint64_t)h->K * (uint64_t)h->M * (uint64_t)h->N * (uint64_t)(h->N + 1) / 2;
  h->st.rank_path_steps = (uint64_t)(h->k_end - h->k_begin) * (uint64_t)h->M * (uint64_t)h->N * (uint64_t)(h->N + 1) / 2;
  *out = h;
  return SRMDP_OK;
}

static srmdp_status finish_solve(srmdp_t* h, std::chrono::steady_clock::time_point t0);

extern "C" srmdp_status srmdp_solve_async(srmdp_t* h) {
  if (!h) return SRMDP_E_ARG;
  h->t_submit = std::chrono::steady_clock::now();
  h->nvtx_solve = nvtxRangeStartA("srmdp_solve");
  CK(h, cudaSetDevice(h->cfg.device), "cudaSetDevice");
  const bool use_graph = !(h->cfg.flags & SRMDP_FLAG_NO_GRAPH);
  if (use_graph) {
    if (!h->graph) {
      CK(h, cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
      srmdp_status s = enqueue_sweep(h, h->N - 1, 0);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(h->stream, &g);
      if (s != SRMDP_OK) { if (g) cudaGraphDestroy(g); return s; }
      if (e != cudaSuccess) return cuda_fail(h, e, "end capture");
      e = cudaGraphInstantiate(&h->graph, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(h, e, "graph instantiate");
      h->graph_launches = h->launches_per_solve;
    }
    CK(h, cudaGraphLaunch(h->graph, h->stream), "graph launch");
    h->launches_per_solve = h->graph_launches;
  } else {
    srmdp_status s = enqueue_sweep(h, h->N - 1, 0);
    if (s != SRMDP_OK) return s;
  }
  h->last_hi = h->N - 1;
  h->last_lo = 0;
  h->pending = true;
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_wait(srmdp_t* h) {
  if (!h) return SRMDP_E_ARG;
  if (!h->pending) return SRMDP_OK;
  h->pending = false;
  return finish_solve(h, h->t_submit);
}

extern "C" srmdp_status srmdp_solve(srmdp_t* h) {
  srmdp_status s = srmdp_solve_async(h);
  if (s != SRMDP_OK) return s;
  return srmdp_wait(h);
}

static srmdp_status finish_solve(srmdp_t* h, std::chrono::steady_clock::time_point t0) {
  cudaError_t se = cudaStreamSynchronize(h->stream);
  if (h->comm) {   // errors a collective raised after it was enqueued (e.g. a peer failed)
    ncclResult_t ae = ncclSuccess;
    if (nccl().CommGetAsyncError(h->comm, &ae) != ncclSuccess || ae != ncclSuccess) return nccl_fail(h, "NCCL", ae);
  }
  if (se != cudaSuccess) return cuda_fail(h, se, "solve");
  unsigned long long cnt[3] = {0, 0, 0};
  CK(h, cudaMemcpy(cnt, h->d_counters, sizeof(cnt), cudaMemcpyDeviceToHost), "event counters");
  if (h->p2p || h->nvls) {
    unsigned xerr = 0;
    CK(h, cudaMemcpy(&xerr, h->d_xerr, sizeof(xerr), cudaMemcpyDeviceToHost), "exchange status");
    if (xerr) {
      cudaMemset(h->d_xerr, 0, sizeof(unsigned));
      h->valid_from = h->N;
      h->solved = false;
      h->err = "fused exchange: a peer rank did not publish slot " + std::to_string(xerr - 1) +
               " within the timeout (SRMDP_EXCHANGE_TIMEOUT_S); the table is invalid";
      return SRMDP_E_NCCL;
    }
  }
  h->st.lp0_fallbacks = cnt[0];
  h->st.exact_z_evals = cnt[1];
  h->st.exact_z_i = cnt[2];
  h->st.kernel_launches = h->launches_per_solve;
  if (h->cfg.flags & SRMDP_FLAG_TIME_KERNELS) {
    double tot = 0, xt = 0;
    h->step_ms.assign(h->N, 0.0);
    h->xchg_ms.assign(h->N, 0.0);
    for (int i = h->last_lo; i <= h->last_hi; ++i) {
      float ms = 0;
      CK(h, cudaEventElapsedTime(&ms, h->ev[2 * i], h->ev[2 * i + 1]), "event time");
      h->step_ms[i] = ms;
      tot += ms;
      if ((h->p2p || h->nvls || h->comm) && !(use_xw(h) && i != h->last_lo)) {   // the events enqueue_sweep recorded
        CK(h, cudaEventElapsedTime(&ms, h->ev[2 * h->N + 2 * i], h->ev[2 * h->N + 2 * i + 1]), "event time");
        h->xchg_ms[i] = ms;
        xt += ms;
      }
    }
    h->st.kernel_ms = tot;
    h->st.gather_ms = xt;
  }
  h->valid_from = h->last_lo;
  h->solved = (h->valid_from == 0);
  if (h->nvtx_solve) { nvtxRangeEnd(h->nvtx_solve); h->nvtx_solve = 0; }
  h->st.solve_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return SRMDP_OK;
}

static void centers_host(const srmdp_t* h, int64_t k, double* r) {
  if (h->cfg.grid) {                 // equal-probability grid: from the host copy of the tables
    int64_t rem = k;
    for (int l = h->d - 1; l >= 0; --l) {
      r[l] = h->tabs[2 * (h->C + 1) + (int)(rem % h->C)];
      rem /= h->C;
    }
    return;
  }
  const double L = h->cfg.L;
  const int C = h->C;
  const double delta = (2.0 * L) / (double)C;
  int64_t rem = k;
  for (int l = h->d - 1; l >= 0; --l) {
    const int c = (int)(rem % C);
    rem /= C;
    if (C == 1) r[l] = 0.0;
    else if (c == 0) r[l] = (-L) + (1.0 * delta);
    else if (c == C - 1) r[l] = (-L) + ((double)(C - 1) * delta);
    else r[l] = (-L) + (((double)c + 0.5) * delta);
  }
}

extern "C" srmdp_status srmdp_coeffs(const srmdp_t* h, int i, int basis, double* out, size_t out_len) {
  if (!h) return SRMDP_E_ARG;
  if (i < h->valid_from && i >= 0) { h->err = "coeffs: slice not computed (solve first)"; return SRMDP_E_STATE; }
  if (i < 0 || i >= h->N || (basis != 0 && basis != 1) || !out || out_len != (size_t)h->K * h->B) {
    h->err = "coeffs: bad i / basis / out_len (must be K*B)";
    return SRMDP_E_ARG;
  }
  CK(h, cudaSetDevice(h->cfg.device), "cudaSetDevice");
  const double* src = h->d_table + (size_t)i * h->K_pad * h->B_pad;
  // device block [Y | W | S | pad | Z_1..Z_q | pad] -> host [Y | Z_1..Z_q]
  const size_t n1 = (size_t)(h->d + 1), hot = (size_t)hot_len(h->d);
  CK(h, cudaMemcpy2DAsync(out, h->B * sizeof(double), src, h->B_pad * sizeof(double), n1 * sizeof(double),
                          (size_t)h->K, cudaMemcpyDeviceToHost, h->stream),
     "coeffs copy");
  CK(h, cudaMemcpy2DAsync(out + n1, h->B * sizeof(double), src + hot, h->B_pad * sizeof(double),
                          (h->B - n1) * sizeof(double), (size_t)h->K, cudaMemcpyDeviceToHost, h->stream),
     "coeffs copy");
  CK(h, cudaStreamSynchronize(h->stream), "coeffs copy");
  if (basis == 0) {  // raw alpha of P:718: alpha_0 = beta_0 - sum_j beta_j r_j
    std::vector<double> r(h->d);
    const int n1 = h->d + 1;
    for (int64_t k = 0; k < h->K; ++k) {
      centers_host(h, k, r.data());
      for (int o = 0; o <= h->q; ++o) {
        double* b = out + (size_t)k * h->B + (size_t)o * n1;
        double s = b[0];
        for (int j = 0; j < h->d; ++j) s -= b[1 + j] * r[j];
        b[0] = s;
      }
    }
  }
  return SRMDP_OK;
}

static srmdp_status ensure_io(const srmdp_t* hc, size_t bytes) {
  srmdp_t* h = const_cast<srmdp_t*>(hc);
  if (h->io_cap >= bytes) return SRMDP_OK;
  dfree(h, h->d_io);
  h->d_io = nullptr;
  h->io_cap = 0;
  CK(h, dalloc(h, &h->d_io, bytes), "io alloc");
  h->io_cap = bytes;
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_eval(const srmdp_t* h, int i, size_t n, const double* x, double* y, double* z) {
  if (!h) return SRMDP_E_ARG;
  if (i < 0 || i > h->N || (n > 0 && (!x || !y)) || (i == h->N && z)) {
    h->err = "eval: bad i, NULL buffer, or z requested at i == N";
    return SRMDP_E_ARG;
  }
  if (i < h->N && i < h->valid_from) { h->err = "eval: slice not computed (solve first)"; return SRMDP_E_STATE; }
  if (n == 0) return SRMDP_OK;
  CK(h, cudaSetDevice(h->cfg.device), "cudaSetDevice");
  const size_t nx = n * h->d, nz = z ? n * h->q : 0;
  srmdp_status s = ensure_io(h, (nx + n + nz) * sizeof(double));
  if (s != SRMDP_OK) return s;
  double* dx = h->d_io;
  double* dy = dx + nx;
  double* dz = z ? dy + n : nullptr;
  CK(h, cudaMemcpyAsync(dx, x, nx * sizeof(double), cudaMemcpyHostToDevice, h->stream), "eval h2d");
  if (h->jit) {
    const int bs = 128;
    int ii = i;
    int64_t nn = (int64_t)n;
    void* args[] = {const_cast<DevProblem*>(&h->dp), &ii, &nn, &dx, &dy, &dz};
    CK(h, cudaLaunchKernel((const void*)h->jit->eval, dim3((unsigned)((n + bs - 1) / bs)), dim3(bs), args, 0, h->stream),
       "eval kernel");
  } else {
    h->ops->eval(h->dp, i, (int64_t)n, dx, dy, dz, h->stream);
  }
  CK(h, cudaGetLastError(), "eval kernel");
  CK(h, cudaMemcpyAsync(y, dy, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream), "eval d2h");
  if (z) CK(h, cudaMemcpyAsync(z, dz, nz * sizeof(double), cudaMemcpyDeviceToHost, h->stream), "eval d2h");
  CK(h, cudaStreamSynchronize(h->stream), "eval");
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_reseed(srmdp_t* h, uint64_t seed) {
  if (!h) return SRMDP_E_ARG;
  h->cfg.seed = seed;
  DevProblem& P = h->dp;
  P.key0 = (uint32_t)(seed & 0xffffffffu);
  P.key1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    P.rkey.k0[r] = P.key0 + (uint32_t)r * 0x9E3779B9u;
    P.rkey.k1[r] = P.key1 + (uint32_t)r * 0xBB67AE85u;
  }
  if (h->graph) {               // kernel parameters are baked into the graph: re-capture
    cudaSetDevice(h->cfg.device);
    cudaGraphExecDestroy(h->graph);
    h->graph = nullptr;
  }
  h->solved = false;
  h->valid_from = h->N;
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_solve_steps(srmdp_t* h, int i_hi, int i_lo) {
  if (!h) return SRMDP_E_ARG;
  if (i_hi < i_lo || i_lo < 0 || i_hi >= h->N) { h->err = "solve_steps: need N > i_hi >= i_lo >= 0"; return SRMDP_E_ARG; }
  if (i_hi != h->N - 1 && i_hi != h->valid_from - 1) {
    h->err = "solve_steps: i_hi must be N-1 or one below the lowest present slice";
    return SRMDP_E_STATE;
  }
  auto t0 = std::chrono::steady_clock::now();
  CK(h, cudaSetDevice(h->cfg.device), "cudaSetDevice");
  srmdp_status s = enqueue_sweep(h, i_hi, i_lo);
  if (s != SRMDP_OK) return s;
  h->last_hi = i_hi;
  h->last_lo = i_lo;
  return finish_solve(h, t0);
}

// Checkpoint file (srmdp.h): header v2 identifies the problem completely --
// every input of the sweep's arithmetic -- so a slice set can only be loaded
// into a handle that would have computed the same slices.
struct SrmdHeader {
  char magic[4];
  int32_t version, d, q, N, B_pad, hot, i_lo;
  int32_t lp0, grid, dyn, fk, gk, C;
  int64_t K, M;
  uint64_t seed;
  double T, L, mu, C_y, C_z;
  uint64_t problem_hash;   // FNV-1a over the parameter arrays and the user source
};

static uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = (const unsigned char*)p;
  for (size_t t = 0; t < n; ++t) { h ^= b[t]; h *= 0x100000001b3ull; }
  return h;
}

static SrmdHeader make_header(const srmdp_t* h) {
  SrmdHeader hd;
  memset(&hd, 0, sizeof(hd));   // padding bytes too: the header is compared field by field, written as bytes
  memcpy(hd.magic, "SRMD", 4);
  hd.version = 2;
  hd.d = h->d; hd.q = h->q; hd.N = h->N; hd.B_pad = h->B_pad; hd.hot = hot_len(h->d); hd.i_lo = h->valid_from;
  hd.lp0 = h->cfg.lp0 ? 1 : 0; hd.grid = h->cfg.grid; hd.dyn = h->cfg.dyn.kind; hd.fk = h->cfg.driver.kind;
  hd.gk = h->cfg.terminal.kind; hd.C = h->C;
  hd.K = h->K; hd.M = h->M; hd.seed = h->cfg.seed;
  hd.T = h->cfg.T; hd.L = h->cfg.L; hd.mu = h->cfg.mu; hd.C_y = h->C_y; hd.C_z = h->C_z;
  uint64_t ph = 0xcbf29ce484222325ull;
  ph = fnv1a(ph, h->params.data(), h->params.size() * sizeof(double));
  ph = fnv1a(ph, h->user_src.data(), h->user_src.size());
  hd.problem_hash = ph;
  return hd;
}

// One slice at a time through a pinned staging buffer, on the handle's stream
// (ordered with the solves that produce / consume the table).
extern "C" srmdp_status srmdp_table_save(const srmdp_t* h, const char* path) {
  if (!h || !path) return SRMDP_E_ARG;
  if (h->valid_from >= h->N) { h->err = "table_save: no slice present"; return SRMDP_E_STATE; }
  CK(h, cudaSetDevice(h->cfg.device), "cudaSetDevice");
  CK(h, cudaStreamSynchronize(h->stream), "table_save: pending work");   // e.g. after srmdp_solve_async
  const size_t n = (size_t)h->K * h->B_pad;
  double* buf = nullptr;
  CK(h, cudaMallocHost(&buf, n * sizeof(double)), "table_save: pinned buffer");
  FILE* f = fopen(path, "wb");
  if (!f) { cudaFreeHost(buf); h->err = std::string("table_save: cannot open ") + path; return SRMDP_E_ARG; }
  const SrmdHeader hd = make_header(h);
  bool ok = fwrite(&hd, sizeof(hd), 1, f) == 1;
  cudaError_t e = cudaSuccess;
  for (int i = h->valid_from; ok && i < h->N; ++i) {
    e = cudaMemcpyAsync(buf, h->d_table + (size_t)i * h->K_pad * h->B_pad, n * sizeof(double), cudaMemcpyDeviceToHost,
                        h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) break;
    ok = fwrite(buf, sizeof(double), n, f) == n;
  }
  ok = (fclose(f) == 0) && ok;
  cudaFreeHost(buf);
  if (e != cudaSuccess) return cuda_fail(h, e, "table_save copy");
  if (!ok) { h->err = "table_save: write failed"; return SRMDP_E_ARG; }
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_table_load(srmdp_t* h, const char* path) {
  if (!h || !path) return SRMDP_E_ARG;
  if (h->d_replica) { h->err = "table_load: not in the P2P_SELF_PEER test mode"; return SRMDP_E_UNSUPPORTED; }
  FILE* f = fopen(path, "rb");
  if (!f) { h->err = std::string("table_load: cannot open ") + path; return SRMDP_E_ARG; }
  SrmdHeader hd;
  if (fread(&hd, sizeof(hd), 1, f) != 1 || memcmp(hd.magic, "SRMD", 4) != 0 || hd.version != 2) {
    fclose(f);
    h->err = "table_load: not an SRMD v2 file";
    return SRMDP_E_ARG;
  }
  SrmdHeader mine = make_header(h);
  mine.i_lo = hd.i_lo;
  if (memcmp(&mine, &hd, sizeof(hd)) != 0 || hd.i_lo < 0 || hd.i_lo >= h->N) {
    fclose(f);
    h->err = "table_load: file does not match this problem (d, q, N, cells, M, T, L, mu, C_y, C_z, basis, grid, "
             "families, parameters, user source, seed)";
    return SRMDP_E_ARG;
  }
  CK(h, cudaSetDevice(h->cfg.device), "cudaSetDevice");
  CK(h, cudaStreamSynchronize(h->stream), "table_load: pending work");
  const size_t n = (size_t)h->K * h->B_pad;
  double* buf = nullptr;
  cudaError_t e = cudaMallocHost(&buf, n * sizeof(double));
  if (e != cudaSuccess) { fclose(f); return cuda_fail(h, e, "table_load: pinned buffer"); }
  srmdp_status st = SRMDP_OK;
  for (int i = hd.i_lo; i < h->N; ++i) {
    if (fread(buf, sizeof(double), n, f) != n) {
      h->err = "table_load: truncated file";
      st = SRMDP_E_ARG;
      break;
    }
    e = cudaMemcpyAsync(h->d_table + (size_t)i * h->K_pad * h->B_pad, buf, n * sizeof(double), cudaMemcpyHostToDevice,
                        h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);   // buf is reused for the next slice
    if (e != cudaSuccess) { st = cuda_fail(h, e, "table_load copy"); break; }
  }
  fclose(f);
  cudaFreeHost(buf);
  if (st != SRMDP_OK) {   // the table may be partly overwritten: nothing is present any more
    h->valid_from = h->N;
    h->solved = false;
    return st;
  }
  h->valid_from = hd.i_lo;
  h->solved = (hd.i_lo == 0);
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_step_ms(const srmdp_t* h, double* out, int n) {
  if (!h || !out || n != h->N) return SRMDP_E_ARG;
  for (int i = 0; i < n; ++i) out[i] = (i < (int)h->step_ms.size()) ? h->step_ms[i] : 0.0;
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_exchange_ms(const srmdp_t* h, double* out, int n) {
  if (!h || !out || n != h->N) return SRMDP_E_ARG;
  for (int i = 0; i < n; ++i) out[i] = (i < (int)h->xchg_ms.size()) ? h->xchg_ms[i] : 0.0;
  return SRMDP_OK;
}

extern "C" void srmdp_destroy(srmdp_t* h) {
  if (!h) return;
  cudaSetDevice(h->cfg.device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->graph) cudaGraphExecDestroy(h->graph);
  for (auto& e : h->ev) cudaEventDestroy(e);
  if (h->comm && nccl().ok) nccl().CommDestroy(h->comm);
  for (void* b : h->opened) cudaIpcCloseMemHandle(b);
  if (h->ipc_base) {
    if (h->stream) cudaStreamSynchronize(h->stream);
    ipc_release(h->cfg.device, h->ipc_base, h->ipc_bytes);
    h->d_table = nullptr;
  }
  if (h->nvls) {
    if (h->stream) cudaStreamSynchronize(h->stream);
    nvls_destroy(&h->nv);
    h->d_table = nullptr;
  }
  if (h->stream) {
    dfree(h, h->d_epoch);
    dfree(h, h->d_xerr);
    dfree(h, h->d_xw_counter);
    dfree(h, h->d_replica);
    dfree(h, h->d_table);
    dfree(h, h->d_params);
    dfree(h, h->d_tabs);
    dfree(h, h->d_scratch);
    dfree(h, h->d_counters);
    dfree(h, h->d_io);
    cudaStreamSynchronize(h->stream);
  }
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

extern "C" const char* srmdp_last_error(const srmdp_t* h) { return h ? h->err.c_str() : g_create_err.c_str(); }

extern "C" srmdp_status srmdp_nccl_unique_id(void* out128) {
  if (!out128) return SRMDP_E_ARG;
  NcclApi& api = nccl();
  if (!api.ok) { g_create_err = api.err; return SRMDP_E_NCCL; }
  ncclUniqueId id;
  ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) { g_create_err = std::string("ncclGetUniqueId: ") + api.GetErrorString(r); return SRMDP_E_NCCL; }
  memcpy(out128, &id, sizeof(id));
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_stats(const srmdp_t* h, srmdp_stats_t* out) {
  if (!h || !out) return SRMDP_E_ARG;
  srmdp_stats_t s = h->st;
  s.smallness_violated = h->smallness_ok ? 0 : 1;
  s.C_y = h->C_y;
  s.C_z = h->C_z;
  s.K = h->K; s.K_pad = h->K_pad; s.chunk = h->chunk; s.k_begin = h->k_begin; s.k_end = h->k_end;
  s.B = h->B; s.B_pad = h->B_pad;
  s.grid = h->grid; s.block = step_threads(h->d); s.smem_bytes = (int)h->smem; s.ctas_per_sm = h->ctas;
  *out = s;
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_jit_check(int d, int q, int dyn_kind, int f_kind, int g_kind, const char* user_src,
                                        char* log, size_t log_len) {
  if (d < 1 || q < 1 || d > 32 || q > 32) return SRMDP_E_ARG;
  std::string err;
  size_t bytes = 0;
  const bool ok = jit_compile_check(d, q, dyn_kind == SRMDP_DYN_USER, f_kind == SRMDP_F_USER, g_kind == SRMDP_G_USER,
                                    user_src ? user_src : "", err, &bytes);
  if (ok) err = "ok: " + std::to_string(bytes) + " bytes of sm_100a CUBIN";
  if (log && log_len) {
    const size_t n = err.size() < log_len - 1 ? err.size() : log_len - 1;
    memcpy(log, err.data(), n);
    log[n] = '\0';
  }
  return ok ? SRMDP_OK : SRMDP_E_JIT;
}

extern "C" srmdp_status srmdp_plan(int d, int q, int N, double mu, int lp0, double c_delta, double c_M,
                                   double mem_bytes, srmdp_plan_t* out) {
  if (!out || d < 1 || q < 1 || d > 32 || q > 32 || N < 1 || !(mu > 0) || mem_bytes < 0) return SRMDP_E_ARG;
  const double cd = c_delta > 0 ? c_delta : 1.0, cm = c_M > 0 ? c_M : 1.0;
  srmdp_plan_t p{};
  p.L = std::log((double)N) / mu;
  p.delta = cd * std::pow((double)N, lp0 ? -0.5 : -0.25);
  const double cpd = std::ceil(2.0 * p.L / p.delta);
  p.cells_per_dim = (p.L > 0 && cpd >= 1) ? (int)std::min(cpd, 2048.0) : 1;
  double K = 1;
  for (int l = 0; l < d; ++l) K *= p.cells_per_dim;
  p.K = K < 9.2e18 ? (int64_t)K : INT64_MAX;
  const double M = std::ceil(cm * (lp0 ? 1.0 : (double)(d + 1)) * (double)N * (double)N);
  p.M = (int64_t)std::max(M, (double)(d + 1));
  p.B = (q + 1) * (d + 1);
  p.B_pad = block_stride(d, q);
  p.table_bytes = (double)N * K * (double)p.B_pad * 8.0;
  p.path_steps = K * (double)p.M * (double)N * (double)(N + 1) / 2.0;
  p.path_starts = K * (double)p.M * (double)N;
  p.fits = (mem_bytes == 0 || p.table_bytes <= mem_bytes) ? 1 : 0;
  *out = p;
  return SRMDP_OK;
}

extern "C" const char* srmdp_build_info(void) {
  static std::string info;
  if (info.empty()) {
    info = "srmdp ABI " + std::to_string(SRMDP_ABI_VERSION) + "; sm_100a fp64; (d,q) =";
    for (const Ops& o : kOps) info += " (" + std::to_string(o.D) + "," + std::to_string(o.Q) + ")";
    info += "; NVRTC: user problems and any other d, q <= 32";
  }
  return info.c_str();
}

// ------------------------------------------------------------------------
// test hooks (include/srmdp_debug.h)
// ------------------------------------------------------------------------
extern "C" srmdp_status srmdp_debug_trace(const srmdp_t* h, int i, int64_t k, int64_t m0, int64_t n, double* x,
                                          int64_t* cell, double* dW) {
  if (!h || i < 0 || i >= h->N || k < 0 || k >= h->K || m0 < 0 || n < 1 || !x || !cell || !dW) return SRMDP_E_ARG;
  CK(h, cudaSetDevice(h->cfg.device), "cudaSetDevice");
  const int steps = h->N - i;
  const size_t nx = (size_t)n * (steps + 1) * h->d, nc = (size_t)n * (steps + 1), nw = (size_t)n * steps * h->q;
  srmdp_status s = ensure_io(h, (nx + nc + nw) * sizeof(double));
  if (s != SRMDP_OK) return s;
  double* dx = h->d_io;
  int64_t* dc = reinterpret_cast<int64_t*>(dx + nx);
  double* dw = dx + nx + nc;
  if (h->jit) {
    const int bs = 64;
    int ii = i;
    uint32_t kk = (uint32_t)k;
    void* args[] = {const_cast<DevProblem*>(&h->dp), &ii, &kk, &m0, &n, &dx, &dc, &dw};
    CK(h, cudaLaunchKernel((const void*)h->jit->trace, dim3((unsigned)((n + bs - 1) / bs)), dim3(bs), args, 0, h->stream),
       "trace kernel");
  } else {
    h->ops->trace(h->dp, i, (uint32_t)k, m0, n, dx, dc, dw, h->stream);
  }
  CK(h, cudaGetLastError(), "trace kernel");
  CK(h, cudaMemcpyAsync(x, dx, nx * sizeof(double), cudaMemcpyDeviceToHost, h->stream), "trace d2h");
  CK(h, cudaMemcpyAsync(cell, dc, nc * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream), "trace d2h");
  CK(h, cudaMemcpyAsync(dW, dw, nw * sizeof(double), cudaMemcpyDeviceToHost, h->stream), "trace d2h");
  CK(h, cudaStreamSynchronize(h->stream), "trace");
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_debug_step_dump(srmdp_t* h, int i, int dump_m, uint32_t* cell, double* x) {
  if (!h || i < 0 || i >= h->N || dump_m < 1 || dump_m > h->M || !cell || !x) return SRMDP_E_ARG;
  if (!use_bm_kernel(h) || !h->ops->step_dump || (h->cfg.flags & SRMDP_FLAG_LOOPBACK)) {
    h->err = "step_dump: only the static BM (X = W) equal-size kernels of d = q in {1, 2, 4, 6, 11, 19}";
    return SRMDP_E_UNSUPPORTED;
  }
  if (h->valid_from > i + 1) { h->err = "step_dump: slices i+1 .. N-1 must be present"; return SRMDP_E_STATE; }
  CK(h, cudaSetDevice(h->cfg.device), "cudaSetDevice");
  const int64_t nk = h->k_end - h->k_begin;
  const int steps = h->N - i;
  const size_t nc = (size_t)nk * dump_m * (size_t)(steps > 1 ? steps - 1 : 0);
  const size_t nx = (size_t)nk * dump_m * (size_t)steps * h->d;
  srmdp_status s = ensure_io(h, (nx + nc / 2 + 2) * sizeof(double));
  if (s != SRMDP_OK) return s;
  DevProblem P = h->dp;
  P.dump_m = dump_m;
  P.dump_x = h->d_io;
  P.dump_cell = reinterpret_cast<uint32_t*>(h->d_io + nx);
  CK(h, cudaMemsetAsync(h->d_counters, 0, 3 * sizeof(unsigned long long), h->stream), "memset");
  if (nk > 0) h->ops->step_dump(P, i, h->k_begin, nk, h->grid, h->smem, h->stream);
  CK(h, cudaGetLastError(), "step dump kernel");
  CK(h, cudaMemcpyAsync(x, P.dump_x, nx * sizeof(double), cudaMemcpyDeviceToHost, h->stream), "dump d2h");
  if (nc) CK(h, cudaMemcpyAsync(cell, P.dump_cell, nc * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream), "dump d2h");
  CK(h, cudaStreamSynchronize(h->stream), "step dump");
  unsigned long long cnt[3] = {0, 0, 0};
  CK(h, cudaMemcpy(cnt, h->d_counters, sizeof(cnt), cudaMemcpyDeviceToHost), "event counters");
  h->st.lp0_fallbacks = cnt[0];    // of this one step
  h->st.exact_z_evals = cnt[1];
  h->st.exact_z_i = cnt[2];
  if (h->valid_from == i + 1) h->valid_from = i;
  h->solved = (h->valid_from == 0);
  return SRMDP_OK;
}

extern "C" srmdp_status srmdp_debug_detmath(int op, size_t n, const double* in, double* out0, double* out1) {
  if (op < 0 || op > 3 || !in || !out0 || (op == 1 && !out1)) return SRMDP_E_ARG;
  if (n == 0) return SRMDP_OK;
  double* d = nullptr;
  cudaError_t e = cudaMalloc(&d, (3 * n + 512) * sizeof(double));
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "detmath alloc");
  std::vector<double> det(512);
  det_tables(det.data());
  double* dt = d;                 // tables first: 16-byte aligned double2 rows
  double* din = d + 512;
  cudaMemcpy(dt, det.data(), 512 * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(din, in, n * sizeof(double), cudaMemcpyHostToDevice);
  detmath_kernel<<<(unsigned)((n + 255) / 256), 256>>>(op, (int64_t)n, din, din + n, din + 2 * n, dt);
  e = cudaDeviceSynchronize();
  if (e == cudaSuccess) {
    cudaMemcpy(out0, din + n, n * sizeof(double), cudaMemcpyDeviceToHost);
    if (op == 1) cudaMemcpy(out1, din + 2 * n, n * sizeof(double), cudaMemcpyDeviceToHost);
  }
  cudaFree(d);
  return e == cudaSuccess ? SRMDP_OK : cuda_fail(nullptr, e, "detmath kernel");
}

extern "C" srmdp_status srmdp_debug_philox(size_t n, const uint32_t* ctr, const uint32_t key[2], uint32_t* out) {
  if (!ctr || !key || !out) return SRMDP_E_ARG;
  if (n == 0) return SRMDP_OK;
  uint32_t* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 8 * n * sizeof(uint32_t));
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "philox alloc");
  cudaMemcpy(d, ctr, 4 * n * sizeof(uint32_t), cudaMemcpyHostToDevice);
  philox_kernel<<<(unsigned)((n + 255) / 256), 256>>>((int64_t)n, d, key[0], key[1], d + 4 * n);
  e = cudaDeviceSynchronize();
  if (e == cudaSuccess) cudaMemcpy(out, d + 4 * n, 4 * n * sizeof(uint32_t), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? SRMDP_OK : cuda_fail(nullptr, e, "philox kernel");
}
