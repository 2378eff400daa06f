/*
 * srmdp.h — C ABI of the B200-native SRMDP hot path.
 *
 * Stratified Regression MDP (SRMDP) of Gobet, Lopez-Salas, Turkedjiev,
 * Vazquez, arXiv 2407.21085 ("PAPER.md"; P:n = line n). The library computes
 * the backward sweep of Alg. srmdp: for i = N-1 .. 0 and every
 * hypercube H_k independently, M start points drawn from the conditional
 * logistic law nu_k (Alg. stratify), Euler paths to T,
 * MDP responses (eq. PsiM) reading the already-fitted affine (LP1,
 * P:204-209) coefficients of later times, the per-cell Gram matrix and Z / Y
 * right-hand sides, their least-squares solution (OLS), truncation
 * at evaluation (eq. TL). Everything runs in fp64 CUDA kernels for
 * sm_100a; there is no CPU fallback.
 *
 * Conventions (all entry points):
 *  - Return an srmdp_status; 0 = OK, negative = error. No exception or exit()
 *    crosses the ABI. srmdp_last_error() returns a human-readable message.
 *  - Host pointers only (the library owns its device memory). Caller owns
 *    every buffer it passes; configuration arrays are deep-copied by create.
 *  - create / solve / destroy are collective over `world` ranks (one process
 *    per GPU, SPMD); coeffs / eval are rank-local (the table is replicated).
 *  - A handle is not thread-safe; distinct handles are independent.
 *  - Random numbers: counter-based Philox4x32-10 keyed by `seed`
 *    (docs/streams.md); results are a deterministic function of the config,
 *    bit-identical for every `world`.
 */
#ifndef SRMDP_H
#define SRMDP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRMDP_ABI_VERSION 3   /* 2: srmdp_config gained user_src / user_params / n_user_params;
                                 3: srmdp_stats_t gained exact_z_evals / exact_z_i / gather_ms */

typedef struct srmdp srmdp_t; /* opaque: device table, streams, graph, NCCL comm */

typedef enum {
  SRMDP_OK = 0,
  SRMDP_E_ARG = -1,         /* invalid argument (d=0, N<1, L<=0, mu<=0, T<=0, size mismatch, ...) */
  SRMDP_E_PRECOND = -2,     /* M < d+1: OLS needs M >= dim L_Y (reading R14) */
  SRMDP_E_STATE = -3,       /* coeffs/eval before a successful solve */
  SRMDP_E_CUDA = -4,        /* CUDA runtime error (message has the CUDA string) */
  SRMDP_E_NCCL = -5,        /* NCCL error / library not loadable for world > 1 */
  SRMDP_E_NOMEM = -6,       /* device allocation failed */
  SRMDP_E_UNSUPPORTED = -7, /* outside the counter / size limits (d, q <= 32, ...) */
  SRMDP_E_JIT = -8          /* the user-problem / (d,q) NVRTC build failed (message has the log) */
} srmdp_status;

/* Closed-form problem families (no host callbacks: they cannot run on the
 * device). Parameter layouts, op order frozen by docs/streams.md §7:
 *  dyn    BM     (q = d): X = W, paper §5.1               params: none
 *         GBM    (q = d): b = mu o x, sigma = diag(s o x)           params: mu[d], s[d]
 *         AFFINE        : b = b0 + B1 x, sigma = S0 (constant)      params: b0[d], B1[d*d], S0[d*q]
 *         GBM_EXACT (q = d): as GBM, exact transition x e^{(mu-s^2/2)dt + s dW}
 *                           (Alg. "SDE dynamics")        params: mu[d], s[d]
 *  driver ZERO          : f = 0                                     params: none
 *         LINEAR        : f = a y + theta.z + c                     params: a, c, theta[q]
 *         PAPER         : f = (sum_k z_k)(y - (2+q)/(2q))   params: none
 *  terminal AFFINE      : g = a + w.x                               params: a, w[d]
 *         PAPER         : g = omega/(1+omega), omega = e^{T+sum x} params: none */
typedef enum { SRMDP_DYN_BM = 0, SRMDP_DYN_GBM = 1, SRMDP_DYN_AFFINE = 2, SRMDP_DYN_GBM_EXACT = 3,
               SRMDP_DYN_USER = 4 } srmdp_dyn_kind;
typedef enum { SRMDP_F_ZERO = 0, SRMDP_F_LINEAR = 1, SRMDP_F_PAPER = 2, SRMDP_F_USER = 3 } srmdp_f_kind;
typedef enum { SRMDP_G_AFFINE = 0, SRMDP_G_PAPER = 1, SRMDP_G_USER = 2 } srmdp_g_kind;

/* User problems (b, sigma, f, g given as code). A *_USER
 * kind takes n_params = 0 in its srmdp_fn; the functions come from
 * srmdp_config.user_src, CUDA C++ device code that srmdp_create compiles with
 * NVRTC for sm_100a together with the step, eval and trace kernels (one
 * module per distinct (source, d, q, kinds), cached for the process; the
 * compile takes ~2 s). The source sees SRMDP_D, SRMDP_Q (the problem's d, q)
 * and SRMDP_USER_FN (the function qualifiers) and defines, for the kinds
 * selected:
 *
 *   SRMDP_USER_FN void   srmdp_user_b    (const double* p, double t, const double* x, double* b);    b[d]
 *   SRMDP_USER_FN void   srmdp_user_sigma(const double* p, double t, const double* x, double* s);    s[d*q], row-major
 *   SRMDP_USER_FN double srmdp_user_f    (const double* p, double t, const double* x, double y,
 *                                         const double* z);                                          z[q]
 *   SRMDP_USER_FN double srmdp_user_g    (const double* p, const double* x);
 *
 * p = user_params (device copy). t = t_j = j*dt. Euler (indices
 * t_j, X_j, dW_j): x'_l = x_l + ((b_l dt) + sw_l), sw_l = s_l0 dW_0 + ... +
 * s_l,q-1 dW_{q-1} in that order. f_j(x_j, y_{j+1}(x_{j+1}), z_j(x_j)) as
 * P:357 with the full truncated z vector; g at t_N. The module is compiled
 * with --fmad=false: each + - * / written in the source is one IEEE rounding
 * (as C with -ffp-contract=off), so b and sigma built from those and sqrt
 * give path states that a C implementation reproduces bit for bit; vendor
 * transcendentals (exp, log, ...) do not. NVRTC is loaded at run time
 * (libnvrtc.so.12); without it a user problem fails with SRMDP_E_JIT.
 * The same NVRTC build serves (d, q) pairs outside the compiled set
 * (srmdp_build_info) for the closed-form families. */

typedef struct {
  int kind;             /* one of the enums above */
  int n_params;         /* must equal the layout's length */
  const double* params; /* host array, copied at create */
} srmdp_fn;

/* Flags */
#define SRMDP_FLAG_NO_GRAPH     1 /* launch step kernels directly instead of replaying a CUDA graph */
#define SRMDP_FLAG_TIME_KERNELS 2 /* record CUDA events around every step kernel (srmdp_stats.kernel_ms) */
#define SRMDP_FLAG_FORCE_NCCL   4 /* use the NCCL exchange even for world == 1 (tests the collective path
                                     on one GPU; needs nccl_unique_id) */
#define SRMDP_FLAG_LOOPBACK     8 /* emulate `world` ranks in this process: each step launches the world
                                     shards one after another on the same table, no NCCL (tests sharding
                                     and padding on one GPU; `rank` is ignored) */
#define SRMDP_FLAG_JIT         16 /* build the kernels with NVRTC even when (d, q) is compiled in */
#define SRMDP_FLAG_P2P_EXCHANGE 32 /* fused exchange instead of ncclAllGather: every step kernel's
                                     epilogue stores each block into all ranks' tables over NVLink
                                     (CUDA IPC mappings, world <= 8, one node); per-slice release /
                                     acquire flags at system scope order the stores against the next
                                     step's reads. NCCL is still used once, at create, to exchange
                                     the IPC handles (world > 1). */
#define SRMDP_FLAG_NVLS_EXCHANGE 128 /* fused exchange through NVLS multicast: every
                                     rank's [table | flags] is bound to one multicast object over the
                                     ranks' GPUs (NVSwitch); the step kernel's epilogue stores each block
                                     once with multimem.st and the switch writes it into every replica;
                                     per-slice flags as P2P_EXCHANGE, published with one multimem release
                                     store. world <= 8; NCCL serves as the rendezvous barrier (world > 1)
                                     and the multicast handle reaches the other ranks as a file descriptor
                                     over a Unix socket. SRMDP_E_UNSUPPORTED where the GPU / system has no
                                     multicast. At world == 1 the multicast object spans this GPU alone. */
#define SRMDP_FLAG_INKERNEL_FLAGS 256 /* fused exchanges on the BM (X = W) kernels: instead of a signal and a
                                     wait kernel after every step, the step kernel itself waits for slice
                                     i+1 after the table-free head (start points, first increments) of
                                     its first round -- overlapping the peers' last stores -- and its last
                                     CTA publishes slice i. Opt-in: on one GPU the kernel is 1.4% slower
                                     with the head / tail split compiled in, the separate kernels cost 0.35 ms
                                     per cfg4 solve */
#define SRMDP_FLAG_P2P_SELF_PEER 64 /* test mode of P2P_EXCHANGE at world == 1: the kernels read and store
                                     a second table on this GPU and the epilogue's peer-store loop
                                     (n_peers = 1) writes every block into the handle's own table, the
                                     one srmdp_coeffs reads: that table then holds exactly what the
                                     peer stores delivered (no table_load in this mode) */

typedef struct {
  int d, q, N;          /* state dim, Brownian dim, time steps */
  double T;             /* horizon; dt = T/N */
  srmdp_fn dyn, driver, terminal;
  int cells_per_dim;    /* #C; K = #C^d hypercubes; breakpoints -L + j*2L/#C, outer cells infinite */
  double L;             /* half-width of the uniformly stratified box [-L, L]^d */
  double mu;            /* logistic parameter of nu (A_nu) — north_star's "nu" */
  int64_t M;            /* simulations per hypercube and time step; M >= d+1 */
  double C_g, C_f, L_f; /* bounds of (A_g), (A_f) -> C_y, C_z by eq. prop:bound */
  double C_y_override;  /* NaN: use the bound; +INFINITY: no truncation; else this value */
  double C_z_override;  /* same, for C_z */
  uint64_t seed;        /* Philox key (docs/streams.md §2) */
  int rank, world;      /* SPMD position; world == 1: no NCCL */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId from srmdp_nccl_unique_id (world > 1) */
  int device;           /* CUDA device ordinal of this rank */
  void* stream;         /* cudaStream_t to run on; NULL = a library-owned stream */
  int flags;            /* SRMDP_FLAG_* */
  int lp0;              /* 0: LP1 affine local basis (the hot path); nonzero: LP0
                           piecewise-constant basis (eq. lp0:explicit P:700-707):
                           every coefficient block is (mean, 0, ..., 0) */
  int grid;             /* 0: equal-size cells, breakpoints -L + j*2L/#C (default);
                           1: equal-probability cells under nu, breakpoints F^{-1}(j/#C)
                           ((A_Strat.) example ii; L unused) */
  const char* user_src;        /* user problem source (see above), or NULL; copied at create */
  const double* user_params;   /* host array of n_user_params doubles, copied at create */
  int n_user_params;
} srmdp_config;

/* Validate, compute C_y/C_z, build the per-dimension breakpoint/F tables,
 * allocate the N x K_pad x B_pad fp64 table (docs/layout.md), init NCCL.
 * Collective. On error *out is NULL and srmdp_last_error(NULL) explains. */
srmdp_status srmdp_create(const srmdp_config* cfg, srmdp_t** out);

/* Run the whole backward sweep i = N-1 .. 0 (Alg. srmdp), one fused
 * step kernel per time point on this rank's cells, then an in-place
 * ncclAllGather of slice i (world > 1). Collective; blocks until done. */
srmdp_status srmdp_solve(srmdp_t* h);

/* srmdp_solve split in two: srmdp_solve_async enqueues the whole sweep on the
 * handle's stream (one CUDA-graph launch) and returns; srmdp_wait
 * synchronizes that stream and finalizes srmdp_stats. Lets a caller bracket
 * the device work with its own CUDA events without host gaps. */
srmdp_status srmdp_solve_async(srmdp_t* h);
srmdp_status srmdp_wait(srmdp_t* h);

/* Copy the coefficients of time i (0 <= i < N) to host `out`, K x B doubles,
 * B = (q+1)(d+1), per cell [Y | Z_1 .. Z_q] each (d+1) long (docs/layout.md).
 * basis 1: centered beta (native); basis 0: the paper's raw alpha.
 * out_len must be exactly K*B. Coefficients are raw (truncation applies at
 * evaluation). */
srmdp_status srmdp_coeffs(const srmdp_t* h, int i, int basis, double* out, size_t out_len);

/* Evaluate the truncated approximations at time i on n host points x (n x d,
 * row-major): y[n] = T_{C_y}(y_i^(M)(x)), z[n x q] = T_{C_z}(z_i^(M)(x)) (may be
 * NULL). i == N gives y = g(x) and requires z == NULL. */
srmdp_status srmdp_eval(const srmdp_t* h, int i, size_t n, const double* x, double* y, double* z);

/* Checkpoint / resume. The sweep state after steps N-1 .. i is exactly the
 * table slices i .. N-1 (the Philox clouds are stateless), so a solve can be
 * split and resumed bit-identically (also on another `world`):
 *  srmdp_solve_steps runs steps i_hi down to i_lo (inclusive) with direct
 *    launches; i_hi must be N-1 or one below the lowest slice already present
 *    (solved or loaded). Collective.
 *  srmdp_table_save writes the present slices to a file (the library's own
 *    checkpoint format, SURVEY §5 "checkpoint / resume"): a 128-byte header --
 *    magic "SRMD", int32 {version = 2, d, q, N, B_pad, hot_len, i_lo, lp0, grid,
 *    dyn kind, f kind, g kind, cells_per_dim}, int64 {K, M}, uint64 seed,
 *    double {T, L, mu, C_y, C_z}, uint64 FNV-1a hash of the parameter arrays
 *    and the user source -- then (N - i_lo) x K x B_pad little-endian doubles,
 *    slices i_lo .. N-1 in the device block layout of docs/layout.md
 *    (rank-local; call on one rank).
 *  srmdp_table_load reads such a file into a handle whose header matches in
 *    every field but i_lo (the same problem, clouds and basis: anything else is
 *    SRMDP_E_ARG); collective (every rank loads). Copies go through a pinned
 *    buffer on the handle's stream. */
srmdp_status srmdp_solve_steps(srmdp_t* h, int i_hi, int i_lo);
srmdp_status srmdp_table_save(const srmdp_t* h, const char* path);
srmdp_status srmdp_table_load(srmdp_t* h, const char* path);

/* Per-step kernel durations of the last solve in ms, out[i] for step i
 * (needs SRMDP_FLAG_TIME_KERNELS; steps not run in the last call are 0). */
srmdp_status srmdp_step_ms(const srmdp_t* h, double* out, int n);
/* Per-step exchange durations (the ncclAllGather of slice i, or the fused
 * exchange's flag wait) of the last solve in ms, out[i] for step i; same
 * conditions as srmdp_step_ms, 0 where no exchange ran. */
srmdp_status srmdp_exchange_ms(const srmdp_t* h, double* out, int n);

/* Replace the Philox key (docs/streams.md §2) for the next srmdp_solve: a new,
 * independent set of clouds on the same problem (independent runs, e.g. the
 * MSE indicators of eq. mse). Collective (same seed on all ranks). */
srmdp_status srmdp_reseed(srmdp_t* h, uint64_t seed);

void srmdp_destroy(srmdp_t* h);

/* Per-handle message of the last failing call; NULL handle: this thread's
 * last create error. Never NULL. */
const char* srmdp_last_error(const srmdp_t* h);

/* Rank 0 calls this and broadcasts the 128 bytes (e.g. torch.distributed). */
srmdp_status srmdp_nccl_unique_id(void* out128);

typedef struct {
  double solve_ms;       /* host wall time of the last srmdp_solve */
  double kernel_ms;      /* sum of step-kernel durations (needs SRMDP_FLAG_TIME_KERNELS) */
  int kernel_launches;   /* step kernels in the last solve (= N) */
  uint64_t path_steps;   /* K * M * N(N+1)/2 over all ranks */
  uint64_t rank_path_steps; /* this rank's share */
  uint64_t lp0_fallbacks;   /* rank-deficient (i,k) regressions (reading R15) */
  int smallness_violated;   /* (T/N) L_f^2 > 1/(12 q): warning only */
  double C_y, C_z;          /* truncation constants in use */
  int64_t K, K_pad, chunk, k_begin, k_end; /* sharding (docs/layout.md) */
  int B, B_pad;
  int grid, block, smem_bytes, ctas_per_sm; /* launch configuration of the step kernel */
  /* ABI 3: */
  uint64_t exact_z_evals;   /* path-step evaluations where the certificate (reading R23) could not rule
                               out truncation and z was truncated per component (eq. TL);
                               counted by the debug kernel of srmdp_debug_step_dump only (the step it
                               re-ran), 0 after srmdp_solve -- the count costs the d = 19 product
                               kernel 7% even when never taken */
  uint64_t exact_z_i;       /* the same for z_i(x_i) in the Y response (pass 2), every solve */
  double gather_ms;         /* sum of the per-step exchange durations (ncclAllGather or the fused
                               flag wait) of the last solve, device-timed (needs SRMDP_FLAG_TIME_KERNELS;
                               0 for world == 1 without FORCE_NCCL / P2P_EXCHANGE) */
} srmdp_stats_t;

srmdp_status srmdp_stats(const srmdp_t* h, srmdp_stats_t* out);

/* Pure host helper (no GPU): the contiguous cell range of `rank` among
 * `world` ranks (docs/layout.md): out[0] = k_begin, out[1] = k_end,
 * out[2] = chunk, out[3] = K_pad. */
srmdp_status srmdp_shard_plan(int64_t K, int world, int rank, int64_t out[4]);

/* NVRTC build of the kernels for a user problem (or a (d, q) outside the
 * compiled set) without a GPU and without loading anything: checks user_src
 * before srmdp_create. Kinds as in srmdp_config (user_src may be NULL when no
 * *_USER kind is given). log (may be NULL) receives the NVRTC log or the
 * error, NUL-terminated and truncated to log_len bytes. SRMDP_OK or
 * SRMDP_E_JIT (SRMDP_E_ARG for d, q outside 1..32). */
srmdp_status srmdp_jit_check(int d, int q, int dyn_kind, int f_kind, int g_kind, const char* user_src, char* log,
                             size_t log_len);

/* Parameter planner of the paper's complexity analysis (§4.3) --
 * pure host arithmetic, no GPU. For a target of O(1/N) total error:
 *   L = log(N)/mu                         (nu(R^d \ [-L,L]^d) <= 2d e^{-mu L} = O(1/N))
 *   delta = c_delta N^{-1/4} (LP1) or c_delta N^{-1/2} (LP0)   (squared bias delta^4 resp. delta^2)
 *   cells_per_dim = max(1, ceil(2L / delta)),  K = cells_per_dim^d     (K = O(N^{d/4}) resp. O(N^{d/2}))
 *   M = ceil(c_M (d+1) N^2) (LP1) or ceil(c_M N^2) (LP0)   (statistical error O(N K' log M / M))
 * and reports what that costs on this implementation: the replicated
 * coefficient table N K B_pad 8 bytes (docs/layout.md), path-steps
 * K M N(N+1)/2 and path-starts K M N per solve (the computational cost
 * O(N^{4+d/4}) resp. O(N^{4+d/2})), and whether the table fits
 * `mem_bytes` (e.g. 180e9 per B200; 0 = no check). c_delta, c_M <= 0 mean 1. */
typedef struct {
  double L, delta;
  int cells_per_dim;
  int64_t K, M;
  int B, B_pad;
  double table_bytes;       /* N * K * B_pad * 8 */
  double path_steps, path_starts;
  int fits;                 /* table_bytes <= mem_bytes (1 when mem_bytes == 0) */
} srmdp_plan_t;
srmdp_status srmdp_plan(int d, int q, int N, double mu, int lp0, double c_delta, double c_M, double mem_bytes,
                        srmdp_plan_t* out);

/* Library version / build info string (ABI version, arch, compiled (d,q)). */
const char* srmdp_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* SRMDP_H */
