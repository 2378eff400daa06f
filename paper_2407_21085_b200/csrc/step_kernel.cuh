// step_kernel.cuh — the fused SRMDP time-step kernel (one launch per t_i).
//
// For every owned hypercube H_k (one persistent CTA walks cells k = blockIdx,
// blockIdx + gridDim, ...), Alg. srmdp at time i:
//  pass 1  each thread simulates one path per round (M/256 rounds):
//          conditional-logistic start point, Euler chain to T
//           with locate + gather of the fitted block of the cell
//          the path lands in, truncated evaluation (eq. TL) and
//          the multistep response S_{Y,i+1} (eq. PsiM). The design
//          row (1, x_i - r_k) and the Z responses S_{Y,i+1} dW_i / dt go to a
//          shared-memory row tile, folded into the Gram matrix and Z
//          right-hand sides in a fixed order (FP64 MMA for d >= 4, owner-
//          compute threads below); (B, Y1, x_i - r_k) go to a per-CTA scratch.
//  solve   Cholesky of the (d+1)^2 Gram (thread 0), q triangular solves
//          -> beta^Z (same OLS minimiser as the paper's QR).
//  pass 2  S_{Y,i} = S_{Y,i+1} + f_i(x_i, y_{i+1}(x_{i+1}), z_i(x_i)) dt with
//          the fresh z_i of this cell from the scratch records,
//          warp-shuffle + fixed-order block reduction of the Y right-hand
//          side, solve -> beta^Y.
//  store   [beta^Y | beta^Z_1..q] into table[i][k] (docs/layout.md).
// Reduction orders depend only on (M, thread count), never on the number of
// ranks, so tables are bit-identical for every world size.
#pragma once
#include "problem.cuh"

namespace srk {

// Threads per CTA = paths per round. d > 8: 128-thread CTAs, 4 per SM (the
// same 16 warps per SM at 128 registers as 2 x 256, in finer units: fewer
// warps wait at each round's barriers; cfg5 +5.5%). d <= 8: 256 x 3 (128 x 6
// measured -1.1% at cfg4).
#ifndef SRMDP_THREADS
#define SRMDP_THREADS 256
#endif
#ifndef SRMDP_THREADS_HI
#define SRMDP_THREADS_HI 128
#endif
__host__ __device__ constexpr int step_threads(int d) { return d > 8 ? SRMDP_THREADS_HI : SRMDP_THREADS; }

// Kernel variants (A/B builds: build.py -DNAME=VALUE)
#ifndef SRMDP_LDG256
#define SRMDP_LDG256 1    // 256-bit hot-line loads
#endif
#ifndef SRMDP_J_UNROLL
#define SRMDP_J_UNROLL 2   // d <= 8: path-step loop unrolled by 2, X_{j+1} / X_{j+2} swap roles without register moves (+0.9% at d = 6; at d = 19 the doubled body costs 15% in instruction-cache misses, so 1 there)
#endif
constexpr int kJUnroll = SRMDP_J_UNROLL;
#ifndef SRMDP_LOCATE_MAGIC
#define SRMDP_LOCATE_MAGIC 0
#endif
// Pass-2 record scratch accesses: plain, or streaming (evict-first: the
// records are touched twice and should not push the gathered slices out of L2)
// (measured: d = 19 +2.6%, where the slices exceed L2; d = 6 -1.5%: 2 = only d > 8)
#ifndef SRMDP_RECORD_CS
#define SRMDP_RECORD_CS 2
#endif
template <int D>
__device__ __forceinline__ void rec_st(double* p, double v) {
  if constexpr (SRMDP_RECORD_CS == 1 || (SRMDP_RECORD_CS == 2 && D > 8)) __stcs(p, v);
  else *p = v;
}
template <int D>
__device__ __forceinline__ double rec_ld(const double* p) {
  if constexpr (SRMDP_RECORD_CS == 1 || (SRMDP_RECORD_CS == 2 && D > 8)) return __ldcs(p);
  else return *p;
}

#ifndef SRMDP_RNG_AHEAD
#define SRMDP_RNG_AHEAD 0
#endif
#ifndef SRMDP_BM_FAST_ONLY
#define SRMDP_BM_FAST_ONLY 0   // 1: BM kernels compile only the range-proved start point (launched only when rcp_fast; measured neutral)
#endif
#ifndef SRMDP_MMA_REUSE
#define SRMDP_MMA_REUSE 0
#endif
#ifndef SRMDP_MMA_ACC2
#define SRMDP_MMA_ACC2 0   // measured: two DMMA chains ±0% at d = 6, -1.5% at d = 19
#endif
#ifndef SRMDP_PASS2_UNROLL
#define SRMDP_PASS2_UNROLL 0   // 0: the compiler's choice; n: records of several paths in flight per thread (pass 2 is latency-bound on the scratch reads)
#endif
constexpr int kPass2Unroll = SRMDP_PASS2_UNROLL;
#ifndef SRMDP_PREFETCH
#define SRMDP_PREFETCH 0  // prefetch of the next hot line, d <= 8 (0 none, 1 L1, 2 L2): measured -1.2% at d = 6 with the 256-bit loads
#endif
#ifndef SRMDP_PREFETCH_HD
#define SRMDP_PREFETCH_HD 0   // d > 8: L1 prefetch measured -3% at d = 19 (4.34e9 vs 4.48e9), L2 -6%
#endif

// Row stride (doubles) of the shared-memory row tile [1 | x - r_k | S dW/dt]:
// odd (spreads banks). Dynamic shared memory of the step kernel for (d, q, C):
// the grid tables then the row tile (the solve arrays alias the tile). Plain
// functions so the host sizes NVRTC-built kernels with the same formula.
__host__ __device__ constexpr int row_stride(int d, int q) { return (1 + d + q) | 1; }
// (+8 doubles: the MMA fragment loads of the last row read up to 7 padding
// columns past the tile; they only feed discarded outputs)
__host__ __device__ constexpr size_t step_smem_bytes(int d, int q, int C) {
  return sizeof(double) * (size_t)((smem_tabs_len(d, C) + step_threads(d) * row_stride(d, q) + 8 + 1) & ~1);
}

template <int D, int Q>
struct KCfg {
  static constexpr int kThreads = step_threads(D);
  static constexpr int N1 = D + 1;
  static constexpr int NB = (Q + 1) * N1;           // B
  static constexpr int NH = hot_len(D);             // hot part [Y | W | S | pad]
  static constexpr int NBP = block_stride(D, Q);    // device block stride (doubles)
  static constexpr int NG = N1 * (N1 + 1) / 2;      // Gram entries (upper, incl. diag)
  static constexpr int NZ = Q * N1;                 // Z right-hand-side entries
  static constexpr int E = NG + NZ;
  static constexpr int ROWS = kThreads;            // rows (paths) per round: one path per thread
  // resident CTAs per SM (launch bounds): 3 x 256 threads (<= 85 registers) up
  // to d = 8; the high-d kernels keep their d-long state in 128 registers at
  // 4 x 128 threads per SM
#ifndef SRMDP_CTAS_LO
#define SRMDP_CTAS_LO 3
#endif
#ifndef SRMDP_CTAS_HI
#define SRMDP_CTAS_HI 4
#endif
  static constexpr int CTAS = (D > 8) ? SRMDP_CTAS_HI : SRMDP_CTAS_LO;
  static constexpr int S = (E <= kThreads) ? (kThreads / E) : 1;  // row slices per entry
  static constexpr int PAIRS = E * S;
  static constexpr int NACC = (PAIRS + kThreads - 1) / kThreads;
  // Gram / Z right-hand sides by FP64 tensor-core MMA (mma.sync m8n8k4 f64):
  // C = V^T V over the rows V = [1 | x - r_k | S dW/dt] of a round
#ifndef SRMDP_MMA_MIN_D
#define SRMDP_MMA_MIN_D 4
#endif
  // FP64 MMA Gram: 4x fewer shared-memory wavefronts than the owner-compute
  // fold (the L1 data pipe is the busiest unit once the gather uses 256-bit
  // loads); measured d=19 +12%, d=6 +2.8% (scalar won at d=6 before LDG.256)
  static constexpr bool USE_MMA = (D >= SRMDP_MMA_MIN_D);
  static constexpr int NCOL = 1 + D + Q;            // used columns of a row
  static constexpr int PB = (N1 + 7) / 8;           // 8-row blocks of C (p <= d)
  static constexpr int QB = (NCOL + 7) / 8;         // 8-column blocks of C
  static constexpr int TILES = PB * QB - PB * (PB - 1) / 2;   // blocks with qb >= pb
  static constexpr int NW = kThreads / 32;
  // row slices per 8x8 tile: the smallest split that gives every warp the
  // same number of (tile, slice) items (d = 8, 11: 5 tiles -> 40 items;
  // d = 19: 12 tiles -> 24 items), so no warp idles at the barrier after the
  // fold; the old rule split only when there were fewer tiles than warps
#ifndef SRMDP_KSPLIT_BALANCE
#define SRMDP_KSPLIT_BALANCE 1
#endif
  static constexpr int KSPLIT_OLD = (TILES >= NW) ? 1 : (NW / TILES >= 8 ? 8 : (NW / TILES >= 4 ? 4 : (NW / TILES >= 2 ? 2 : 1)));
  static constexpr int KSPLIT_BAL = (TILES % NW == 0) ? 1 : ((2 * TILES) % NW == 0 ? 2 : ((4 * TILES) % NW == 0 ? 4 : 8));
  // (the balanced split only where its partials fit the row tile beside the solve arrays, SmemLayout)
  static constexpr int SOLVE_LEN = N1 * N1 + 2 * NZ + 2 * N1 + (kThreads / 32) * N1 + 2 + N1 + 2;
  static constexpr bool BAL_FITS = TILES * KSPLIT_BAL * 64 + SOLVE_LEN + 2 <= ROWS * row_stride(D, Q);
  static constexpr int KSPLIT = (SRMDP_KSPLIT_BALANCE && BAL_FITS) ? KSPLIT_BAL : KSPLIT_OLD;
  static constexpr int ITEMS = TILES * KSPLIT;      // (tile, row slice) work items
  // Fragment-reusing fold (SRMDP_MMA_REUSE): warp w takes one tile row pb
  // (all QB - pb tiles of it) over a row slice, so each 8-column fragment is
  // loaded once per k-step for every tile of the row (QB - pb loads for QB - pb
  // DMMA instead of 2 per DMMA). Warps per tile row in proportion to its
  // tiles (largest remainder, at least one each).
  __host__ __device__ static constexpr int GT(int p) { return QB - p; }
  __host__ __device__ static constexpr int GW(int p) {               // warps of tile row p
    int n[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int used = 0;
    for (int g = 0; g < PB; ++g) { n[g] = (NW * GT(g)) / TILES; if (n[g] < 1) n[g] = 1; used += n[g]; }
    while (used < NW) {                          // largest remainder NW*GT/TILES - n
      int best = 0, bv = -1000000;
      for (int g = 0; g < PB; ++g) { const int r = NW * GT(g) - n[g] * TILES; if (r > bv) { bv = r; best = g; } }
      ++n[best]; ++used;
    }
    return n[p];
  }
  __host__ __device__ static constexpr int GW0(int p) { int f = 0; for (int g = 0; g < p; ++g) f += GW(g); return f; }        // first warp
  __host__ __device__ static constexpr int GSLOT(int p) { int f = 0; for (int g = 0; g < p; ++g) f += GT(g) * GW(g); return f; }  // first partial slot
  static constexpr int RSLOTS = GSLOT(PB);       // (tile, slice) partials of the reuse fold
  static constexpr int NI = (ITEMS + NW - 1) / NW;  // items per warp
  // odd row stride (spreads banks); MMA fragment loads of the padding columns
  // (>= NCOL) read neighbouring smem and only feed discarded outputs
  static constexpr int ROW = row_stride(D, Q);
  static constexpr bool UNROLL_GATHER = (NB <= 128);
};

// Shared-memory carve-up (in doubles), shared by host sizing and the kernel.
template <int D, int Q>
struct SmemLayout {
  // The solve-phase arrays (Gram/L, R_Z, beta, R_Y, warp partials, flag) alias
  // the row tile behind the reduction scratch `red`: they are only live after
  // the last round of pass 1 and die before the next cell's pass 1. Keeps a
  // d = 6 CTA at 31 KB, so 3 CTAs/SM fit a 100 KB shared-memory carveout and
  // L1 keeps the rest for the coefficient hot lines (fit_carveout, ops.h).
  using KC = KCfg<D, Q>;
  static constexpr int kThreads = KC::kThreads;
  static constexpr int MMA_RED = (SRMDP_MMA_REUSE ? KC::RSLOTS : KC::ITEMS) * 64;
  static constexpr int RED = (((KC::USE_MMA ? MMA_RED : KC::PAIRS) > kThreads
                                   ? (KC::USE_MMA ? MMA_RED : KC::PAIRS)
                                   : kThreads) + 1) & ~1;
  static constexpr int SOLVE = KC::SOLVE_LEN;
  static_assert(RED + SOLVE <= KC::ROWS * KC::ROW, "solve arrays must fit in the row tile");
  static_assert(!KC::USE_MMA || MMA_RED <= RED, "MMA tile partials must fit the reduction scratch");
  static_assert(!KC::USE_MMA || 8 * (KC::QB - 1) + 7 < KC::ROW + 8, "MMA fragment columns stay within a row + padding");
  __host__ __device__ static int tabs(int C) { return smem_tabs_len(D, C); }
  __host__ __device__ static int rows(int C) { return tabs(C); }
  __host__ __device__ static int L(int C) { return rows(C) + RED; }
  __host__ __device__ static int RZ(int C) { return L(C) + KC::N1 * KC::N1; }
  __host__ __device__ static int BZ(int C) { return RZ(C) + KC::NZ; }
  __host__ __device__ static int BY(int C) { return BZ(C) + KC::NZ; }
  __host__ __device__ static int RY(int C) { return BY(C) + KC::N1; }
  __host__ __device__ static int warp(int C) { return RY(C) + KC::N1; }
  __host__ __device__ static int flag(int C) { return warp(C) + (kThreads / 32) * KC::N1; }
  __host__ __device__ static int W(int C) { return flag(C) + 2; }   // W (d+1) then S
  __host__ __device__ static size_t bytes(int C) { return step_smem_bytes(D, Q, C); }
};

// Warp-aggregated event count (one atomic per warp and event site); only
// executed where the event happens, so the certified fast paths pay nothing.
__device__ __forceinline__ void count_event(unsigned long long* c) {
  const unsigned mask = __activemask();
  if ((int)(threadIdx.x & 31) == __ffs(mask) - 1) atomicAdd(c, (unsigned long long)__popc(mask));
}

// Exact evaluation of the q Z blocks: zlin = sum_l w_l T_{C_z}(beta^{Z_l} . a).
template <int D, int Q>
__device__ __forceinline__ double zlin_exact(const DevProblem& P, const double* __restrict__ blk, const double (&a)[D + 1]) {
  using KC = KCfg<D, Q>;
  double zl = 0.0;
#pragma unroll 1
  for (int l = 0; l < Q; ++l) {
    const double* bz = blk + KC::NH + l * KC::N1;
    double v = 0.0;
#pragma unroll
    for (int p = 0; p <= D; ++p) v = fma(__ldg(bz + p), a[p], v);
    zl = fma(zweight(P, l), trunc_L(v, P.C_z), zl);
  }
  return zl;
}

// Evaluate the fitted block of a cell at centered coordinates a = (1, x - r):
// y = T_{C_y}(beta^Y . a), zlin = sum_l w_l T_{C_z}(beta^{Z_l} . a).
// Fast path (one 128-byte line for d <= 6): when S * max(1, max_p |a_p|) is
// below C_z no component can be truncated, so zlin = W . a (same value up to
// rounding order, reading R23); otherwise the exact per-component path.
// Counting the exact path-step evaluations (srmdp_stats.exact_z_evals) is
// compiled into the DUMP (debug) kernels only: even never executed, the
// counting branch in the d = 19 product kernel cost 7% (register allocation
// of the hot loop; measured: atomic 4.72e9, register count 4.33e9, none
// 5.05e9 path-steps/s at cfg5). 1 = a warp-aggregated atomic inside the exact
// branch, 2 = a per-thread register count flushed once per path.
#ifndef SRMDP_GATHER_EL
#define SRMDP_GATHER_EL 0   // experiment (d > 8): L2 evict_last fraction of the hot-line loads, in tenths
#endif
#ifndef SRMDP_COUNT_EXACT
#define SRMDP_COUNT_EXACT 1
#endif
template <int D, int Q, bool COUNT>
__device__ __forceinline__ void eval_block(const DevProblem& P, const double* __restrict__ blk,
                                           const double (&a)[D + 1], double& y, double& zlin, int& nexact) {
  using KC = KCfg<D, Q>;
  constexpr int NHOT = 2 * KC::N1 + 1;
  double yv = 0.0, wv = 0.0, S = 0.0;
#if SRMDP_LDG256
  // 256-bit loads (LDG.E.ENL2.256, sm_100): half the L1 wavefronts of 128-bit
  // loads for the divergent per-lane gather; blocks are 128-byte aligned
#pragma unroll
  for (int u = 0; u < (NHOT + 3) / 4; ++u) {
    double v[4];
#if SRMDP_GATHER_EL
    if constexpr (D > 8) {
      // experiment: L2 evict_last policy on the hot lines (a fraction of them)
      uint64_t pol;
      asm("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(pol) : "f"(SRMDP_GATHER_EL / 10.0f));
      asm("ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
          : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(blk + 4 * u), "l"(pol));
    } else
#endif
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(blk + 4 * u));
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int e = 4 * u + h;
      const double c = v[h];
      if (e < KC::N1) yv = fma(c, a[e], yv);
      else if (e < 2 * KC::N1) wv = fma(c, a[e - KC::N1], wv);
      else if (e == 2 * KC::N1) S = c;
    }
  }
#else
  const double2* b2 = reinterpret_cast<const double2*>(blk);
#pragma unroll
  for (int u = 0; u < (NHOT + 1) / 2; ++u) {
    const double2 v = __ldg(b2 + u);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = 2 * u + h;
      const double c = h ? v.y : v.x;
      if (e < KC::N1) yv = fma(c, a[e], yv);
      else if (e < 2 * KC::N1) wv = fma(c, a[e - KC::N1], wv);
      else if (e == 2 * KC::N1) S = c;
    }
  }
#endif
  y = trunc_L(yv, P.C_y);
  // conservative max(1, max_p |a_p|) from the high words (integer pipe)
  int hm = 0x3ff00000;
#pragma unroll
  for (int p = 1; p <= D; ++p) hm = max(hm, __double2hiint(a[p]) & 0x7fffffff);
  const double amax = __hiloint2double(hm, 0xffffffff);
  if (S * amax <= P.C_z_safe) {
    zlin = wv;
  } else {
    zlin = zlin_exact<D, Q>(P, blk, a);
    if constexpr (COUNT) {
#if SRMDP_COUNT_EXACT == 1
      count_event(P.counters + 1);
#elif SRMDP_COUNT_EXACT == 2
      ++nexact;
#endif
    }
  }
}

// Prefetch of a coefficient block's hot part (every 128-byte line it spans)
// into L1 (mode 1) or L2 (mode 2), issued before the next step's increments.
template <int NHOT, int MODE>
__device__ __forceinline__ void prefetch_block(const double* blk) {
  if constexpr (MODE == 1) {
#pragma unroll
    for (int off = 0; off < NHOT * 8; off += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"((const char*)blk + off));
  } else if constexpr (MODE == 2) {
#pragma unroll
    for (int off = 0; off < NHOT * 8; off += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)blk + off));
  }
}

// One path of cloud (i,k), pass 1 (path m of this thread, shared-memory row
// `row`). The design row (1, x_i - r_k) and dW_i are written to the row as soon
// as they exist, so they do not stay in registers across the Euler chain.
// Returns B = S_{Y,i+1}(x_i) = g(x_N) + sum_{j>i} f_j dt (eq. PsiM) and
// Y1 = y_{i+1}(x_{i+1}). Software pipeline per step: the cell of X_{j+1} is
// located, the increments and Euler step of X_{j+2} are computed (FP64-heavy,
// independent of the gather) while its 128-byte hot line is loaded with four
// 256-bit loads, then the block is evaluated. The per-lane gather is
// divergent (up to 32 lines per warp instruction), so the L1 data pipe, not
// latency, is what it costs: 256-bit instead of 128-bit loads gained 7%, an
// explicit L1 prefetch now loses 1%. (Two paths per thread for ILP measured
// slower: 2.43e10 vs 2.65e10.)
// The table-free head of a path: start point x_i (row: 1, x_i - r_k), the
// increments dW_i (row) and X_{i+1} = Euler(x_i, dW_i) into Xn.
template <int D, int Q, bool EQ, int DK>
__device__ __forceinline__ void simulate_head(const DevProblem& P, const Grid& G, const int (&cc)[D], int i,
                                              uint32_t k, uint32_t m, double* row, double (&Xn)[D]) {
#ifdef SRMDP_EXPERIMENT_START_CENTER   // timing experiment only (wrong results): no start-point sampling
#pragma unroll
  for (int l = 0; l < D; ++l)   // a point inside the cell: the centre, or +-0.8 for the two-cell grid (centres 0)
    Xn[l] = (P.C == 2 ? (cc[l] == 0 ? -0.8 : 0.8) : G.cen[cc[l]]) + 1e-3 * (double)(m & 7);
#else
  start_point<D, EQ, (DK == DYN_BM && SRMDP_BM_FAST_ONLY) ? 1 : 0>(P, G, cc, i, k, m, Xn);
#endif
  row[0] = 1.0;
#pragma unroll
  for (int l = 0; l < D; ++l) row[1 + l] = Xn[l] - G.cen[cc[l]];
  {
    double dW[Q], X1[D];
    brownian<Q>(P, G, i, i, k, m, dW);
#pragma unroll
    for (int l = 0; l < Q; ++l) row[1 + D + l] = dW[l];
    euler<D, Q, DK>(P, (double)i * P.dt, Xn, dW, X1);
#pragma unroll
    for (int l = 0; l < D; ++l) Xn[l] = X1[l];
  }
}

// The rest of the path from X_{i+1} (the first gather reads slice i+1).
template <int D, int Q, bool EQ, bool DUMP, int DK>
__device__ __forceinline__ void simulate_tail(const DevProblem& P, const Grid& G, int i, uint32_t k, uint32_t m,
                                              double (&Xn)[D], double& Bout, double& Y1out, int64_t kl) {
  using KC = KCfg<D, Q>;
  double acc = 0.0, zlin = 0.0, Y1 = 0.0, yv = 0.0;
  int nexact = 0;
  const int N = P.N;
#ifndef SRMDP_J_UNROLL_HD
#define SRMDP_J_UNROLL_HD 1
#endif
  constexpr int JU = (D <= 8) ? kJUnroll : SRMDP_J_UNROLL_HD;
  // RNG one step ahead (SRMDP_RNG_AHEAD, phase-ordered Brownian only): the
  // Philox words of step j+2 are drawn while step j+1's are transformed
  constexpr bool AHEAD = SRMDP_RNG_AHEAD && ((Q + 1) / 2 <= SRMDP_PHASE_MAX);
  U4 onx[(Q + 1) / 2];
  if constexpr (AHEAD) {
    if (i + 1 < N) brownian_words<Q>(P, i, i + 1, k, m, onx);
  }
#pragma unroll JU
  for (int j = i; j < N; ++j) {
    // Xn = X_{j+1}
    double zn = 0.0;
    if (j + 1 < N) {
      int c[D];
      uint32_t kn = 0;
#if SRMDP_LOCATE_MAGIC
      if constexpr (!EQ) {
        // floor((x + L) / delta) without a conversion instruction: rounded
        // down, t + 1.5*2^52 is 1.5*2^52 + floor(t) exactly for |t| < 2^51, so
        // the low word is floor(t) whenever the high word shows |t| < 2^31
        // (else -- NaN, inf, huge x -- every coordinate takes locate1); the
        // same cells as locate1 (docs/streams.md §6) for every input
        unsigned bad = 0;
#pragma unroll
        for (int l = 0; l < D; ++l) {
          const double t = __dmul_rn(__dadd_rn(Xn[l], P.L), P.inv_delta);
          const double r = __dadd_rd(t, 0x1.8p52);
          bad |= (unsigned)(__double2hiint(r) - 0x4337ffff) > 1u ? 1u : 0u;
          c[l] = min(max(__double2loint(r), 0), P.C - 1);
        }
        if (bad) {
#pragma unroll
          for (int l = 0; l < D; ++l) c[l] = locate1(Xn[l], P.L, P.inv_delta, P.C);
        }
#pragma unroll
        for (int l = 0; l < D; ++l) kn = kn * (uint32_t)P.C + (uint32_t)c[l];
      } else
#endif
      {
#pragma unroll
        for (int l = 0; l < D; ++l) {
          c[l] = locate_g<EQ>(P, G.edge, Xn[l]);
          kn = kn * (uint32_t)P.C + (uint32_t)c[l];
        }
      }
#ifdef SRMDP_EXPERIMENT_GATHER_SELF   // timing experiment only (wrong results): every gather hits the start cell
      kn = k;
#endif
      if constexpr (DUMP) {   // debug build (srmdp_debug_step_dump): the cell and state this loop located
        if ((int64_t)m < P.dump_m) {
          const int64_t s = (kl * P.dump_m + m) * (int64_t)(N - i);
          SRK_CHECK(j - i < N - i - 1, "dump index");
          P.dump_cell[(kl * P.dump_m + m) * (int64_t)(N - i - 1) + (j - i)] = kn;
#pragma unroll
          for (int l = 0; l < D; ++l) P.dump_x[(s + (j - i)) * D + l] = Xn[l];
        }
      }
      SRK_CHECK(kn < (uint64_t)P.K && j + 1 < P.N, "gathered cell / slice");
      const double* blk = P.table + ((size_t)(j + 1) * (size_t)P.K_pad + kn) * (size_t)KC::NBP;
      prefetch_block<2 * KC::N1 + 1, (D > 8 ? SRMDP_PREFETCH_HD : SRMDP_PREFETCH)>(blk);
      double Xnn[D];
      {
        double dW[Q];
        if constexpr (AHEAD) {
          U4 ocur[(Q + 1) / 2];
#pragma unroll
          for (int b = 0; b < (Q + 1) / 2; ++b) ocur[b] = onx[b];
          if (j + 2 < N) brownian_words<Q>(P, i, j + 2, k, m, onx);
          brownian_transform<Q>(P, G, ocur, dW);
        } else {
          brownian<Q>(P, G, i, j + 1, k, m, dW);   // increments of step j+1
        }
        euler<D, Q, DK>(P, (double)(j + 1) * P.dt, Xn, dW, Xnn);
      }
      double a[D + 1];
      a[0] = 1.0;
#pragma unroll
      for (int l = 0; l < D; ++l) a[1 + l] = Xn[l] - center_of<EQ>(P, G, c[l]);
      eval_block<D, Q, DUMP>(P, blk, a, yv, zn, nexact);   // y_{j+1}(x_{j+1}), z_{j+1}(x_{j+1})
#pragma unroll
      for (int l = 0; l < D; ++l) Xn[l] = Xnn[l];
    } else {
      yv = g_eval<D>(P, Xn);                     // y_N := g
      if constexpr (DUMP) {
        if ((int64_t)m < P.dump_m) {
          const int64_t s = (kl * P.dump_m + m) * (int64_t)(N - i);
#pragma unroll
          for (int l = 0; l < D; ++l) P.dump_x[(s + (j - i)) * D + l] = Xn[l];
        }
      }
    }
    if (j == i) {
      Y1 = yv;
    } else {
      const double fdt = f_eval(P, yv, zlin) * P.dt;   // f_j(x_j, y_{j+1}(x_{j+1}), z_j(x_j)) dt
      acc = acc + fdt;
    }
    zlin = zn;
  }
  Bout = yv + acc;                                 // g(x_N) + sum
  Y1out = Y1;
#if SRMDP_COUNT_EXACT == 2
  if constexpr (DUMP) {   // one warp-aggregated atomic per path round
    const unsigned mask = __activemask();
    const unsigned tot = __reduce_add_sync(mask, (unsigned)nexact);
    if (tot && (int)(threadIdx.x & 31) == __ffs(mask) - 1) atomicAdd(P.counters + 1, (unsigned long long)tot);
  }
#endif
}

template <int D, int Q, bool EQ, bool DUMP, int DK>
__device__ __forceinline__ void simulate_path(const DevProblem& P, const Grid& G, const int (&cc)[D], int i,
                                              uint32_t k, uint32_t m, double* row, double& Bout, double& Y1out,
                                              int64_t kl) {
  double Xn[D];
  simulate_head<D, Q, EQ, DK>(P, G, cc, i, k, m, row, Xn);
  simulate_tail<D, Q, EQ, DUMP, DK>(P, G, i, k, m, Xn, Bout, Y1out, kl);
}

#if SRMDP_USER_F
// Pass 1 of one path for a user driver f(t, x, y, z) that reads the whole
// truncated z vector, t and x (srmdp.h, SRMDP_F_USER): the plain order of
// Alg. SRMDP -- per step the increments, the Euler step, then
// y_{j+1}, z_{j+1} at x_{j+1} from the full block, f_j(x_j, y_{j+1}, z_j(x_j)).
template <int D, int Q, bool EQ>
__device__ __forceinline__ void simulate_path_user(const DevProblem& P, const Grid& G, const int (&cc)[D], int i,
                                                   uint32_t k, uint32_t m, double* row, double& Bout, double& Y1out) {
  using KC = KCfg<D, Q>;
  double X[D];
  start_point<D, EQ>(P, G, cc, i, k, m, X);
  row[0] = 1.0;
#pragma unroll
  for (int l = 0; l < D; ++l) row[1 + l] = X[l] - G.cen[cc[l]];
  double zc[Q];
#pragma unroll
  for (int l = 0; l < Q; ++l) zc[l] = 0.0;
  double acc = 0.0, Y1 = 0.0, yv = 0.0;
  const int N = P.N;
#pragma unroll 1
  for (int j = i; j < N; ++j) {
    const double tj = (double)j * P.dt;
    double dW[Q], Xn[D], zn[Q];
    brownian<Q>(P, G, i, j, k, m, dW);
    if (j == i) {
#pragma unroll
      for (int l = 0; l < Q; ++l) row[1 + D + l] = dW[l];
    }
    euler<D, Q>(P, tj, X, dW, Xn);
    if (j + 1 < N) {
      uint32_t kn = 0;
      double a[D + 1];
      a[0] = 1.0;
#pragma unroll
      for (int l = 0; l < D; ++l) {
        const int c = locate_g<EQ>(P, G.edge, Xn[l]);
        kn = kn * (uint32_t)P.C + (uint32_t)c;
        a[1 + l] = Xn[l] - G.cen[c];
      }
      SRK_CHECK(kn < (uint64_t)P.K && j + 1 < P.N, "gathered cell / slice (user driver)");
      const double* blk = P.table + ((size_t)(j + 1) * (size_t)P.K_pad + kn) * (size_t)KC::NBP;
      double v = 0.0;
#pragma unroll
      for (int p = 0; p <= D; ++p) v = fma(__ldg(blk + p), a[p], v);
      yv = trunc_L(v, P.C_y);
#pragma unroll 1
      for (int l = 0; l < Q; ++l) {
        double w = 0.0;
#pragma unroll
        for (int p = 0; p <= D; ++p) w = fma(__ldg(blk + KC::NH + l * KC::N1 + p), a[p], w);
        zn[l] = trunc_L(w, P.C_z);
      }
    } else {
      yv = g_eval<D>(P, Xn);                       // y_N := g
#pragma unroll
      for (int l = 0; l < Q; ++l) zn[l] = 0.0;
    }
    if (j == i) Y1 = yv;
    else acc = acc + f_user<D, Q>(P, tj, X, yv, zc) * P.dt;   // f_j(x_j, y_{j+1}(x_{j+1}), z_j(x_j)) dt
#pragma unroll
    for (int l = 0; l < Q; ++l) zc[l] = zn[l];
#pragma unroll
    for (int l = 0; l < D; ++l) X[l] = Xn[l];
  }
  Bout = yv + acc;
  Y1out = Y1;
}
#endif

// Cholesky of the symmetric n x n matrix in A (full storage), lower factor in
// place. Returns 1 iff positive definite with min diag(L) >= 1e-10 max diag(L)
// (= QR's |R_jj| test, reading R15).
template <int N1>
__device__ int cholesky_inplace(double* A) {
  double mx = 0.0, mn = 1e300;
  for (int j = 0; j < N1; ++j) {
    double s = A[j * N1 + j];
    for (int kk = 0; kk < j; ++kk) s = s - A[j * N1 + kk] * A[j * N1 + kk];
    if (!(s > 0.0)) return 0;
    const double ljj = sqrt(s);
    A[j * N1 + j] = ljj;
    mx = fmax(mx, ljj);
    mn = fmin(mn, ljj);
    for (int r = j + 1; r < N1; ++r) {
      double t = A[r * N1 + j];
      for (int kk = 0; kk < j; ++kk) t = t - A[r * N1 + kk] * A[j * N1 + kk];
      A[r * N1 + j] = t / ljj;
    }
  }
  return (mn >= 1e-10 * mx) ? 1 : 0;
}

// The same factorization by one warp (for d > 8): column j's entries
// t_r = A[r][j] - sum_{k<j} L[r][k] L[j][k] (k ascending, exactly the serial
// order) are computed by lanes r = j.. in parallel; bit-identical result.
template <int N1>
__device__ int cholesky_warp(double* A, int lane) {
  double mx = 0.0, mn = 1e300;
  for (int j = 0; j < N1; ++j) {
    double tj = 0.0;
    for (int r = j + lane; r < N1; r += 32) {
      double t = A[r * N1 + j];
      for (int kk = 0; kk < j; ++kk) t = t - A[r * N1 + kk] * A[j * N1 + kk];
      if (r == j) tj = t;
      else A[r * N1 + j] = t;            // column j below the diagonal: not read by column j itself
    }
    const double s = __shfl_sync(0xffffffffu, tj, 0);   // lane 0 owns r = j
    if (!(s > 0.0)) return 0;
    const double ljj = sqrt(s);
    mx = fmax(mx, ljj);
    mn = fmin(mn, ljj);
    __syncwarp();
    for (int r = j + lane; r < N1; r += 32) A[r * N1 + j] = (r == j) ? ljj : A[r * N1 + j] / ljj;
    __syncwarp();
  }
  return (mn >= 1e-10 * mx) ? 1 : 0;
}

// Solve L L^T b = r (L lower in full storage).
template <int N1>
__device__ void chol_solve(const double* L, const double* r, double* b) {
  double y[N1];
  for (int p = 0; p < N1; ++p) {
    double s = r[p];
    for (int kk = 0; kk < p; ++kk) s = s - L[p * N1 + kk] * y[kk];
    y[p] = s / L[p * N1 + p];
  }
  for (int p = N1 - 1; p >= 0; --p) {
    double s = y[p];
    for (int kk = p + 1; kk < N1; ++kk) s = s - L[kk * N1 + p] * b[kk];
    b[p] = s / L[p * N1 + p];
  }
}

// The same solve by one warp for NR right-hand sides at once (d > 8):
// forward substitution as a wavefront -- lane q keeps row q's running sums
// r_q - sum_{k<p} L[q][k] y_k for every right-hand side, subtracting in
// increasing k exactly as chol_solve (bit-identical y); backward substitution
// likewise, subtracting L[k][q] b_k for k from N1-1 down (summation order
// differs from chol_solve at rounding level). N1 shuffle steps with NR
// independent chains instead of an N1^2 serial chain per thread. Right-hand
// side j is r + j*rs, its solution b + j*rs (j < nr <= NR).
template <int N1, int NR>
__device__ void chol_solve_warp(const double* L, const double* r, double* b, int rs, int nr, int lane) {
  constexpr int R = (N1 + 31) / 32;
  double s[NR][R], y[NR][R];
#pragma unroll
  for (int j = 0; j < NR; ++j)
#pragma unroll
    for (int t = 0; t < R; ++t) {
      s[j][t] = (j < nr && lane + 32 * t < N1) ? r[j * rs + lane + 32 * t] : 0.0;
      y[j][t] = 0.0;
    }
  for (int p = 0; p < N1; ++p) {
    const double inv_owner = L[p * N1 + p];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      double v = 0.0;
#pragma unroll
      for (int t = 0; t < R; ++t)
        if (lane + 32 * t == p) { v = s[j][t] / inv_owner; y[j][t] = v; }
      const double yp = __shfl_sync(0xffffffffu, v, p & 31);
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int q = lane + 32 * t;
        if (q > p && q < N1) s[j][t] = s[j][t] - L[q * N1 + p] * yp;
      }
    }
  }
  for (int p = N1 - 1; p >= 0; --p) {
    const double lpp = L[p * N1 + p];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      double v = 0.0;
#pragma unroll
      for (int t = 0; t < R; ++t)
        if (lane + 32 * t == p) {
          v = y[j][t] / lpp;
          if (j < nr) b[j * rs + p] = v;
        }
      const double bp = __shfl_sync(0xffffffffu, v, p & 31);
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int q = lane + 32 * t;
        if (q < p) y[j][t] = y[j][t] - L[p * N1 + q] * bp;
      }
    }
  }
}

#ifndef SRMDP_WARP_SOLVE
#define SRMDP_WARP_SOLVE 0   // measured at d = 19: -1.5% (more code; the per-thread solves already run the q right-hand sides in parallel)
#endif

// EQ: equal-probability strata (binary-search locate) — a template parameter so
// the equal-size grid's hot loop carries no grid branch (a runtime branch cost 4%).
// DUMP: debug variant (srmdp_debug_step_dump) that also writes the located
// cells and states of the first dump_m paths of every cell; otherwise the
// same code.
// In-kernel exchange (XW): wait until every rank has published slice i+1
// (flags [i+1][*] at this solve's epoch; acquire at system scope) -- one
// thread per CTA, after the table-free head of the first round, so the start
// points overlap the other ranks' last stores -- and, in the last CTA of the
// launch, publish slice i (release at system scope, after every CTA's
// stores and fence). Bounded like exchange_wait_kernel.
__device__ __forceinline__ void xw_wait(const DevProblem& P, int slot) {
  unsigned e;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(e) : "l"(P.xw_epoch) : "memory");
  for (int r = 0; r < P.xw_world; ++r) {
    const unsigned* p = P.xw_own + (size_t)slot * P.xw_world + r;
    unsigned v;
    for (int n = 0;; ++n) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
      if ((int)(v - e) >= 0) break;
      if (n > (1 << 28) || *(volatile unsigned*)P.xw_err) {   // ~minutes, or another wait already failed
        atomicCAS(P.xw_err, 0u, 1u + (unsigned)slot);
        return;
      }
      __nanosleep(200);
    }
  }
}

__device__ __forceinline__ void xw_signal(const DevProblem& P, int slot) {
  __threadfence_system();
  const unsigned e = *P.xw_epoch;
  if (P.xw_mc) {
    asm volatile("fence.proxy.alias;" ::: "memory");
    unsigned* p = P.xw_mc + (size_t)slot * P.xw_world + P.xw_rank;
    asm volatile("multimem.st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(e) : "memory");
  } else {
    for (int r = 0; r < P.xw_world; ++r) {
      unsigned* p = P.xw_flags[r] + (size_t)slot * P.xw_world + P.xw_rank;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(e) : "memory");
    }
  }
}

// DK: dynamics family fixed at compile time (-1 = runtime, see euler()).
// XW: in-kernel exchange flags (above) instead of separate signal / wait kernels.
template <int D, int Q, bool EQ, bool DUMP = false, int DK = -1, bool XW = false>
__global__ void __launch_bounds__(step_threads(D), KCfg<D, Q>::CTAS)
step_kernel(const DevProblem P, const int i, const int64_t k_begin, const int64_t nk) {
  using KC = KCfg<D, Q>;
  constexpr int kThreads = KC::kThreads;
  using SL = SmemLayout<D, Q>;
  extern __shared__ double sm[];
  const int C = P.C;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, gid = (tid & 31) >> 2, tig = tid & 3;   // MMA fragment coordinates
  constexpr int TC = tab_copies(D);
  const Grid G = make_grid_smem<TC>(sm, C);
  double* sRows = sm + SL::rows(C);
  double* sL = sm + SL::L(C);
  double* sRZ = sm + SL::RZ(C);
  double* sBZ = sm + SL::BZ(C);
  double* sBY = sm + SL::BY(C);
  double* sRY = sm + SL::RY(C);
  double* sWarp = sm + SL::warp(C);
  int* sFlag = reinterpret_cast<int*>(sm + SL::flag(C));
  double* sW = sm + SL::W(C);                 // certificate of the fresh Z: W[d+1], S
  double* sS = sW + KC::N1;
  constexpr int SB = scratch_stride(D);
  double* BYs = P.by_scratch + (size_t)blockIdx.x * (size_t)P.M * SB;   // this CTA's pass-2 records

#if SRMDP_BOUNDS_CHECK
  {   // the carve-up (tables, row tile + MMA padding, solve arrays) fits the launch's dynamic shared memory
    unsigned dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    SRK_CHECK((size_t)(SL::rows(C) + KC::ROWS * KC::ROW + 8) * 8 <= dyn, "row tile in shared memory");
    SRK_CHECK((size_t)(SL::W(C) + KC::N1 + 1) * 8 <= dyn, "solve arrays in shared memory");
    SRK_CHECK((size_t)(SL::rows(C) + SL::RED) <= (size_t)SL::L(C), "reduction scratch");
    SRK_CHECK(k_begin >= 0 && k_begin + nk <= P.K, "cell range");
  }
#endif
  {   // grid tables, then the detmath tables replicated entry by entry (DetTabs)
    const int off = tabs_det_off(C);
    for (int t = tid; t < off; t += kThreads) sm[t] = P.tabs[t];
    const double2* src = reinterpret_cast<const double2*>(P.tabs + off);
    double2* dst = reinterpret_cast<double2*>(sm + off);
    for (int t = tid; t < 256 * TC; t += kThreads) dst[t] = src[t / TC];
  }

  // Owner-compute assignment (scalar reduction path): pair idx -> (entry e, row slice s).
  int cA[KC::NACC], cB[KC::NACC], rlo[KC::NACC], rhi[KC::NACC];
#pragma unroll
  for (int n = 0; n < KC::NACC; ++n) {
    const int idx = tid + n * kThreads;
    if (idx < KC::PAIRS) {
      const int e = idx % KC::E, s = idx / KC::E;
      if (e < KC::NG) {               // Gram (p <= q), row-major upper enumeration
        int p = 0, rem = e;
        while (rem >= KC::N1 - p) { rem -= KC::N1 - p; ++p; }
        cA[n] = p;
        cB[n] = p + rem;
      } else {                        // Z RHS: (l, p) -> a'_p * R_l
        const int z = e - KC::NG;
        cA[n] = z % KC::N1;
        cB[n] = 1 + D + z / KC::N1;
      }
      rlo[n] = (s * KC::ROWS) / KC::S;
      rhi[n] = ((s + 1) * KC::ROWS) / KC::S;
    } else {
      cA[n] = cB[n] = 0;
      rlo[n] = rhi[n] = 0;
    }
  }
  __syncthreads();

  const int64_t M = P.M;
  const double dt = P.dt;
  for (int64_t kl = blockIdx.x; kl < nk; kl += gridDim.x) {
    const uint32_t k = (uint32_t)(k_begin + kl);
    int cc[D];
    {
      uint32_t r = k;
#pragma unroll
      for (int l = D - 1; l >= 0; --l) { cc[l] = (int)(r % (uint32_t)C); r /= (uint32_t)C; }
    }

    // ---------------- pass 1: paths, Gram and Z right-hand sides ----------
    double acc[KC::NACC];
#pragma unroll
    for (int n = 0; n < KC::NACC; ++n) acc[n] = 0.0;
    constexpr int NMACC = SRMDP_MMA_REUSE ? KC::QB : KC::NI;
    double macc[NMACC][2];
#pragma unroll
    for (int it = 0; it < NMACC; ++it) macc[it][0] = macc[it][1] = 0.0;
    for (int64_t m0 = 0; m0 < M; m0 += KC::ROWS) {
      const int nrows = (int)((M - m0) < KC::ROWS ? (M - m0) : KC::ROWS);
      const int64_t m = m0 + tid;
      // XW: the table-free head of every path first, and in the first round
      // of this CTA's first cell a wait for slice i+1's flags before the rest
      // (measured: splitting every round costs less than a separate first round)
      double Xh[D];
      if constexpr (XW) {
        if (m < M) simulate_head<D, Q, EQ, DK>(P, G, cc, i, k, (uint32_t)m, sRows + tid * KC::ROW, Xh);
        if (kl == (int64_t)blockIdx.x && m0 == 0 && i < P.xw_wait_below) {
          if (tid == 0) xw_wait(P, i + 1);
          __syncthreads();
        }
      }
      if (m < M) {
        double* row = sRows + tid * KC::ROW;
        double Bv, Y1;
#if SRMDP_USER_F
        simulate_path_user<D, Q, EQ>(P, G, cc, i, k, (uint32_t)m, row, Bv, Y1);
#else
        if constexpr (XW) simulate_tail<D, Q, EQ, DUMP, DK>(P, G, i, k, (uint32_t)m, Xh, Bv, Y1, kl);
        else simulate_path<D, Q, EQ, DUMP, DK>(P, G, cc, i, k, (uint32_t)m, row, Bv, Y1, kl);
#endif
        const double sc = Bv * P.inv_dt;
#pragma unroll
        for (int l = 0; l < Q; ++l) row[1 + D + l] = row[1 + D + l] * sc;   // S_{Z,i} = S_{Y,i+1} dW_i / dt
        SRK_CHECK(blockIdx.x < gridDim.x && m < M, "pass-2 record");
        rec_st<D>(BYs + m, Bv);                       // scratch is field-major (coalesced)
        rec_st<D>(BYs + M + m, Y1);
        if constexpr (store_design(D)) {
#pragma unroll
          for (int l = 0; l < D; ++l) rec_st<D>(BYs + (2 + l) * M + m, row[1 + l]);
        }
      }
      __syncthreads();
#ifdef SRMDP_EXPERIMENT_NO_FOLD   // timing experiment only (wrong results): no Gram / Z fold
      if (false) {
      } else
#endif
      if constexpr (KC::USE_MMA && SRMDP_MMA_REUSE) {
        // fragment-reusing fold: this warp's tile row pb over its row slice
        int pb = 0;
#pragma unroll
        for (int g = 1; g < KC::PB; ++g) pb += (warp >= KC::GW0(g)) ? 1 : 0;
        int nw = 0, w0 = 0, nt = 0;
#pragma unroll
        for (int g = 0; g < KC::PB; ++g)
          if (g == pb) { nw = KC::GW(g); w0 = KC::GW0(g); nt = KC::GT(g); }
        const int sl = warp - w0;
        const int rlo_ = 4 * ((sl * (kThreads / 4)) / nw), rhi_ = 4 * (((sl + 1) * (kThreads / 4)) / nw);
        const int rend = rhi_ < nrows ? rhi_ : nrows;
        const double* pf = sRows + 8 * pb + gid;    // fragment t: columns 8 (pb + t) .. + 7
        for (int r0 = rlo_; r0 < rend; r0 += 4) {
          const int rr = r0 + tig;
          const bool in = rr < rend;                 // ragged last k-step: rows >= nrows are 0
          double f[KC::QB];
#pragma unroll
          for (int t = 0; t < KC::QB; ++t) f[t] = (t < nt && in) ? pf[rr * KC::ROW + 8 * t] : 0.0;
#pragma unroll
          for (int t = 0; t < KC::QB; ++t)
            if (t < nt)
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(macc[t][0]), "+d"(macc[t][1]) : "d"(f[0]), "d"(f[t]));
        }
      } else if constexpr (KC::USE_MMA) {
        // C += V^T V on the tensor cores: A(8x4) = V[r0..r0+3][p0..p0+7]^T,
        // B(4x8) = V[r0..r0+3][q0..q0+7]; rows >= nrows contribute 0
#pragma unroll
        for (int it = 0; it < KC::NI; ++it) {
          const int item = warp + it * KC::NW;
          if (item < KC::ITEMS) {
            const int t = item / KC::KSPLIT, sl = item % KC::KSPLIT;
            int pb = 0, tt = t;
            while (tt >= KC::QB - pb) { tt -= KC::QB - pb; ++pb; }
            const int qb = pb + tt;
            const int rlo_ = (sl * kThreads) / KC::KSPLIT, rhi_ = ((sl + 1) * kThreads) / KC::KSPLIT;
            const double* pa = sRows + 8 * pb + gid;
            const double* pbp = sRows + 8 * qb + gid;
            double c0 = macc[it][0], c1 = macc[it][1];
            const int rend = rhi_ < nrows ? rhi_ : nrows;
            int r0 = rlo_;
#if SRMDP_MMA_ACC2
            // two independent accumulator chains (even / odd k-steps of 4
            // rows): DMMA issues back to back instead of waiting for its own
            // previous result; summed in a fixed order below
            double e0 = 0.0, e1 = 0.0;
#pragma unroll 2
            for (; r0 + 8 <= rend; r0 += 8) {
              const double av = pa[(r0 + tig) * KC::ROW];
              const double bv = pbp[(r0 + tig) * KC::ROW];
              const double av2 = pa[(r0 + 4 + tig) * KC::ROW];
              const double bv2 = pbp[(r0 + 4 + tig) * KC::ROW];
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(c0), "+d"(c1) : "d"(av), "d"(bv));
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(e0), "+d"(e1) : "d"(av2), "d"(bv2));
            }
            c0 = c0 + e0;
            c1 = c1 + e1;
#endif
#pragma unroll 4
            for (; r0 + 4 <= rend; r0 += 4) {        // full k-steps: no predicates
              const double av = pa[(r0 + tig) * KC::ROW];
              const double bv = pbp[(r0 + tig) * KC::ROW];
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(c0), "+d"(c1) : "d"(av), "d"(bv));
            }
            if (r0 < rend) {                          // ragged last k-step: rows >= nrows are 0
              const int rr = r0 + tig;
              const double av = (rr < rend) ? pa[rr * KC::ROW] : 0.0;
              const double bv = (rr < rend) ? pbp[rr * KC::ROW] : 0.0;
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(c0), "+d"(c1) : "d"(av), "d"(bv));
            }
            macc[it][0] = c0;
            macc[it][1] = c1;
          }
        }
      } else {
#pragma unroll
        for (int n = 0; n < KC::NACC; ++n) {
          const int hi = rhi[n] < nrows ? rhi[n] : nrows;
          double a = acc[n];
          for (int r = rlo[n]; r < hi; ++r) a = fma(sRows[r * KC::ROW + cA[n]], sRows[r * KC::ROW + cB[n]], a);
          acc[n] = a;
        }
      }
      __syncthreads();
    }
    if constexpr (KC::USE_MMA && SRMDP_MMA_REUSE) {
      // partials -> shared memory [slot][8][8], slot = GSLOT(pb) + t * GW(pb) + slice;
      // then a fixed-order sum over the slices of each tile
      double* red = sRows;
      {
        int pb = 0;
#pragma unroll
        for (int g = 1; g < KC::PB; ++g) pb += (warp >= KC::GW0(g)) ? 1 : 0;
#pragma unroll
        for (int g = 0; g < KC::PB; ++g)
          if (g == pb) {
            const int sl = warp - KC::GW0(g);
#pragma unroll
            for (int t = 0; t < KC::QB; ++t)
              if (t < KC::GT(g)) {
                const int slot = KC::GSLOT(g) + t * KC::GW(g) + sl;
                red[slot * 64 + gid * 8 + 2 * tig] = macc[t][0];
                red[slot * 64 + gid * 8 + 2 * tig + 1] = macc[t][1];
              }
          }
      }
      __syncthreads();
      for (int e = tid; e < KC::N1 * KC::NCOL; e += kThreads) {
        const int p = e / KC::NCOL, q2 = e % KC::NCOL;
        if (q2 < p) continue;                       // Gram: upper half only
        const int pb = p / 8, t = q2 / 8 - pb;
        int nw = 0, s0 = 0;
#pragma unroll
        for (int g = 0; g < KC::PB; ++g)
          if (g == pb) { nw = KC::GW(g); s0 = KC::GSLOT(g) + t * KC::GW(g); }
        double v = red[s0 * 64 + (p % 8) * 8 + (q2 % 8)];
        for (int sl = 1; sl < nw; ++sl) v = v + red[(s0 + sl) * 64 + (p % 8) * 8 + (q2 % 8)];
        if (q2 < KC::N1) {
          sL[p * KC::N1 + q2] = v;
          sL[q2 * KC::N1 + p] = v;
        } else {
          sRZ[(q2 - KC::N1) * KC::N1 + p] = v;      // [l][p]
        }
      }
    } else if constexpr (KC::USE_MMA) {
      // tile partials -> shared memory [item][8][8], then fixed-order sum over row slices
      double* red = sRows;
#pragma unroll
      for (int it = 0; it < KC::NI; ++it) {
        const int item = warp + it * KC::NW;
        if (item < KC::ITEMS) {
          red[item * 64 + gid * 8 + 2 * tig] = macc[it][0];
          red[item * 64 + gid * 8 + 2 * tig + 1] = macc[it][1];
        }
      }
      __syncthreads();
      for (int e = tid; e < KC::N1 * KC::NCOL; e += kThreads) {
        const int p = e / KC::NCOL, q2 = e % KC::NCOL;
        if (q2 < p) continue;                       // Gram: upper half only
        const int pb = p / 8, qb = q2 / 8;
        const int t = pb * KC::QB - pb * (pb - 1) / 2 + (qb - pb);
        double v = red[(t * KC::KSPLIT) * 64 + (p % 8) * 8 + (q2 % 8)];
        for (int sl = 1; sl < KC::KSPLIT; ++sl) v = v + red[(t * KC::KSPLIT + sl) * 64 + (p % 8) * 8 + (q2 % 8)];
        if (q2 < KC::N1) {
          sL[p * KC::N1 + q2] = v;
          sL[q2 * KC::N1 + p] = v;
        } else {
          sRZ[(q2 - KC::N1) * KC::N1 + p] = v;      // [l][p]
        }
      }
    } else {
    // fixed-order combination of the row-slice partials
    double* red = sRows;
#pragma unroll
    for (int n = 0; n < KC::NACC; ++n) {
      const int idx = tid + n * kThreads;
      if (idx < KC::PAIRS) red[(idx % KC::E) * KC::S + idx / KC::E] = acc[n];
    }
    __syncthreads();
    for (int e = tid; e < KC::E; e += kThreads) {
      double v = red[e * KC::S];
      for (int s = 1; s < KC::S; ++s) v = v + red[e * KC::S + s];
      if (e < KC::NG) {
        int p = 0, rem = e;
        while (rem >= KC::N1 - p) { rem -= KC::N1 - p; ++p; }
        const int q2 = p + rem;
        sL[p * KC::N1 + q2] = v;
        sL[q2 * KC::N1 + p] = v;
      } else {
        const int z = e - KC::NG;
        sRZ[(z / KC::N1) * KC::N1 + z % KC::N1] = v;   // [l][p]
      }
    }
    }
    __syncthreads();
    if constexpr (KC::N1 > 9) {
      if (tid < 32) {
        const int okw = P.lp0 ? 0 : cholesky_warp<KC::N1>(sL, tid);
        if (tid == 0) sFlag[0] = okw;
      }
    } else {
      if (tid == 0) sFlag[0] = P.lp0 ? 0 : cholesky_inplace<KC::N1>(sL);   // LP0: means below
    }
    __syncthreads();
    const int ok = sFlag[0];
    // ---------------- solve Z ---------------------------------
    if (KC::N1 > 9 && SRMDP_WARP_SOLVE && ok) {      // d > 8: each warp solves ceil(q/8) right-hand sides at once
      // warp w solves right-hand sides w*NRW .. w*NRW + NRW-1 together
      constexpr int NRW = (Q + KC::NW - 1) / KC::NW;
      const int l0 = warp * NRW, nr = (Q - l0 < NRW) ? (Q - l0) : NRW;
      if (nr > 0) chol_solve_warp<KC::N1, NRW>(sL, sRZ + l0 * KC::N1, sBZ + l0 * KC::N1, KC::N1, nr, tid & 31);
    } else {
      for (int l = tid; l < Q; l += kThreads) {
        if (ok) {
          chol_solve<KC::N1>(sL, sRZ + l * KC::N1, sBZ + l * KC::N1);
        } else {                                   // LP0 fallback: mean
          sBZ[l * KC::N1] = sRZ[l * KC::N1] / (double)M;
          for (int p = 1; p < KC::N1; ++p) sBZ[l * KC::N1 + p] = 0.0;
        }
      }
    }
    __syncthreads();

    // certificate of the fresh Z blocks: W = sum_l w_l beta^{Z_l}, S = max_l ||beta^{Z_l}||_1
    // (stored in the hot line; also used for z_i in pass 2)
    if (tid < KC::N1) {
      double wsum = 0.0;
      for (int l = 0; l < Q; ++l) wsum = fma(zweight(P, l), sBZ[l * KC::N1 + tid], wsum);
      sW[tid] = wsum;
    } else if (tid >= kThreads - 32) {
      // S by the last warp: lane l sums |beta^{Z_l}| (p ascending), then a
      // max-reduction (fmax is exact and order-free: the serial result)
      const int lane = tid & 31;
      double smax = 0.0;
      for (int l = lane; l < Q; l += 32) {
        double t = 0.0;
        for (int p = 0; p < KC::N1; ++p) t += fabs(sBZ[l * KC::N1 + p]);
        smax = fmax(smax, t);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, off));
      if (lane == 0) sS[0] = smax;
    }
    __syncthreads();

    // ---------------- pass 2: Y responses with the fresh z_i ---
#ifdef SRMDP_EXPERIMENT_NO_PASS2   // timing experiment only (wrong results): no pass 2 loop
    const int64_t M2 = 0;
#else
    const int64_t M2 = M;
#endif
    double ry[KC::N1];
#pragma unroll
    for (int p = 0; p < KC::N1; ++p) ry[p] = 0.0;
#if SRMDP_PASS2_UNROLL > 0
#pragma unroll kPass2Unroll
#endif
    for (int64_t m = tid; m < M2; m += kThreads) {
      double a[KC::N1];
      a[0] = 1.0;
      if constexpr (store_design(D)) {
#pragma unroll
        for (int l = 0; l < D; ++l) a[1 + l] = rec_ld<D>(BYs + (2 + l) * M + m);
      } else {
        double x[D];
        start_point<D, EQ>(P, G, cc, i, k, (uint32_t)m, x);
#pragma unroll
        for (int l = 0; l < D; ++l) a[1 + l] = x[l] - G.cen[cc[l]];
      }
#if SRMDP_USER_F
      // user driver: f(t_i, x_i, Y1, z_i(x_i)) with the full truncated z_i of
      // the fresh blocks; x_i regenerated exactly (same bits as pass 1)
      double xi[D], zi[Q];
      start_point<D, EQ>(P, G, cc, i, k, (uint32_t)m, xi);
      for (int l = 0; l < Q; ++l) {
        double v = 0.0;
#pragma unroll
        for (int p = 0; p < KC::N1; ++p) v = fma(sBZ[l * KC::N1 + p], a[p], v);
        zi[l] = trunc_L(v, P.C_z);
      }
      const double Sm = BYs[m] + f_user<D, Q>(P, (double)i * dt, xi, BYs[M + m], zi) * dt;
#else
      // z_i(x_i) through the certificate of the fresh blocks (as eval_block)
      double zl = 0.0;
      int hm = 0x3ff00000;
#pragma unroll
      for (int p = 1; p <= D; ++p) hm = max(hm, __double2hiint(a[p]) & 0x7fffffff);
      if (sS[0] * __hiloint2double(hm, 0xffffffff) <= P.C_z_safe) {
#pragma unroll
        for (int p = 0; p < KC::N1; ++p) zl = fma(sW[p], a[p], zl);
      } else {
        for (int l = 0; l < Q; ++l) {
          double v = 0.0;
#pragma unroll
          for (int p = 0; p < KC::N1; ++p) v = fma(sBZ[l * KC::N1 + p], a[p], v);
          zl = fma(zweight(P, l), trunc_L(v, P.C_z), zl);
        }
        count_event(P.counters + 2);
      }
      const double Sm = rec_ld<D>(BYs + m) + f_eval(P, rec_ld<D>(BYs + M + m), zl) * dt;
#endif
#pragma unroll
      for (int p = 0; p < KC::N1; ++p) ry[p] = fma(a[p], Sm, ry[p]);
    }
#pragma unroll
    for (int p = 0; p < KC::N1; ++p) {
      double v = ry[p];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v = v + __shfl_down_sync(0xffffffffu, v, off);
      if ((tid & 31) == 0) sWarp[(tid >> 5) * KC::N1 + p] = v;
    }
    __syncthreads();
    if (tid < KC::N1) {
      double v = sWarp[tid];
      for (int w = 1; w < kThreads / 32; ++w) v = v + sWarp[w * KC::N1 + tid];
      sRY[tid] = v;
    }
    __syncthreads();
    if (KC::N1 > 9 && SRMDP_WARP_SOLVE && ok) {
      if (tid < 32) chol_solve_warp<KC::N1, 1>(sL, sRY, sBY, 0, 1, tid);
    } else if (tid == 0) {
      if (ok) {
        chol_solve<KC::N1>(sL, sRY, sBY);
      } else {
        sBY[0] = sRY[0] / (double)M;               // eq. lp0:explicit
        for (int p = 1; p < KC::N1; ++p) sBY[p] = 0.0;
        if (!P.lp0) atomicAdd(P.counters, 1ull);   // rank-deficient LP1 fallback (R15)
      }
    }
    __syncthreads();
    SRK_CHECK(i >= 0 && i < P.N && (int64_t)k < P.K, "epilogue block");
    double* dst = P.table + ((size_t)i * (size_t)P.K_pad + k) * (size_t)KC::NBP;
    for (int b = tid; b < KC::NBP; b += kThreads) {
      double v = 0.0;
      if (b < KC::N1) v = sBY[b];
      else if (b < 2 * KC::N1) v = sW[b - KC::N1];
      else if (b == 2 * KC::N1) v = sS[0];
      else if (b >= KC::NH && b < KC::NH + KC::NZ) v = sBZ[b - KC::NH];
      if (P.mc_table) {
        // NVLS exchange: one multimem store through the multicast mapping;
        // NVSwitch writes it into every rank's replica (this one included)
        asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(P.mc_table + (dst - P.table) + b), "d"(v)
                     : "memory");
      } else {
        dst[b] = v;
      }
      // fused exchange: the same block into every peer's replica (NVLink
      // stores, coalesced per block); made visible by exchange_signal_kernel
      for (int r = 0; r < P.n_peers; ++r) P.peer_table[r][(dst - P.table) + b] = v;
    }
    if (P.mc_table) asm volatile("fence.proxy.alias;" ::: "memory");   // multicast alias vs the unicast reads
    if (P.n_peers || P.mc_table) __threadfence_system();   // ordered before the signal kernel's release
    __syncthreads();
  }
  if constexpr (XW) {
    // the last CTA of the launch publishes slice i to every rank
    if (tid == 0) {
      __threadfence_system();
      const unsigned prev = atomicAdd(P.xw_counter, 1u);
      if (prev == gridDim.x - 1) {
        *P.xw_counter = 0u;                  // every CTA has counted: reset for the next launch
        xw_signal(P, i);
      }
    }
  }
}

}  // namespace srk
