/*
 * srmdp_oracle.h — CPU ORACLE for the SRMDP hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the plain, slow, obviously-correct reference of what the CUDA path
 * computes: Algorithm SRMDP of Gobet, Lopez-Salas, Turkedjiev, Vazquez,
 * arXiv 2407.21085, followed step by step in the paper's
 * order, in fp64, with Householder-QR OLS (Golub-Van Loan 5.3.2).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load it. The product path (paper_2407_21085_b200/) never includes,
 * links or calls anything here, and this file includes nothing from it: the
 * two implementations share only the written specs in docs/ (streams, detmath, layout).
 *
 * Parity status per function: see the header comment of srmdp_oracle.c.
 */
#ifndef SRMDP_ORACLE_H
#define SRMDP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_DYN_BM = 0, OR_DYN_GBM = 1, OR_DYN_AFFINE = 2, OR_DYN_GBM_EXACT = 3, OR_DYN_USER = 4 };
enum { OR_F_ZERO = 0, OR_F_LINEAR = 1, OR_F_PAPER = 2, OR_F_USER = 3 };
enum { OR_G_AFFINE = 0, OR_G_PAPER = 1, OR_G_USER = 2 };

/* User problem functions (OR_*_USER kinds): the caller's C code for b, sigma,
 * f, g (include/srmdp.h "User problems" states their meaning); p = user_params. */
typedef void (*or_user_vec_fn)(const double* p, double t, const double* x, double* out);
typedef double (*or_user_f_fn)(const double* p, double t, const double* x, double y, const double* z);
typedef double (*or_user_g_fn)(const double* p, const double* x);

typedef struct {
  int d, q, N;
  double T;
  int dyn_kind;           /* OR_DYN_* : b, sigma */
  const double* dyn_params;
  int f_kind;             /* OR_F_*   : driver f */
  const double* f_params;
  int g_kind;             /* OR_G_*   : terminal g */
  const double* g_params;
  int C;                  /* cells per dimension (#C); K = C^d */
  double L;               /* interior grid [-L, L]^d */
  double mu;              /* logistic parameter (A_nu) */
  int64_t M;              /* paths per cloud */
  double C_y, C_z;        /* truncation bounds (INFINITY = none) */
  uint64_t seed;          /* Philox key, docs/streams.md */
  int lp0;                /* LP0 piecewise-constant basis (eq. lp0:explicit P:700-707) */
  int grid;               /* 0: equal-size cells on [-L,L]; 1: equal-probability cells under nu */
  or_user_vec_fn user_b;      /* b(t, x) -> b[d]          (OR_DYN_USER) */
  or_user_vec_fn user_sigma;  /* sigma(t, x) -> s[d*q]    (OR_DYN_USER), row-major */
  or_user_f_fn user_f;        /* f(t, x, y, z)            (OR_F_USER) */
  or_user_g_fn user_g;        /* g(x)                     (OR_G_USER) */
  const double* user_params;
} or_problem;

/* --- primitives (docs/streams.md, docs/detmath.md) --- */
void   or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double or_u01(uint64_t w);
double or_dm_log(double x);                              /* path function (table-driven) */
double or_dm_log_series(double x);                       /* reference function */
double or_dm_exp(double x);
void   or_dm_sincospi2(double u, double* s, double* c);  /* path function (table-driven) */
void   or_dm_sincospi2_series(double u, double* s, double* c);
void   or_init_tables(void);
double or_F(double mu, double x);
double or_inv_cdf_cond(double mu, double lo, double hi, double U);
int    or_locate1(double x, int C, double L);
int64_t or_locate(const or_problem* p, const double* x);
void   or_cell_center(const or_problem* p, int64_t k, double* r);
int64_t or_num_cells(const or_problem* p);

/* --- problem functions --- */
double or_g(const or_problem* p, const double* x);
double or_f(const or_problem* p, double t, const double* x, double y, const double* z);
void   or_euler(const or_problem* p, double t, const double* x, const double* dW, double* xn);

/* Prop. bound and Lemma cor:as2. Returns 1 iff the
 * smallness condition (T/N) L_f^2 <= 1/(12 q) holds. */
int    or_bounds(double C_g, double C_f, double L_f, int q, double T, int N,
                 double* C_y, double* C_z, double* C_star);

/* --- clouds (Def. clouds) --- */
void   or_start_point(const or_problem* p, int i, int64_t k, int64_t m, double* x);
void   or_brownian(const or_problem* p, int i, int j, int64_t k, int64_t m, double* dW);
/* Trace of one path of cloud (i,k), path m: x[(N-i+1)*d] = x_i..x_N,
 * cell[N-i+1] = located cells of x_i..x_N, dW[(N-i)*q]. */
void   or_trace_path(const or_problem* p, int i, int64_t k, int64_t m,
                     double* x, int64_t* cell, double* dW);

/* --- OLS by Householder QR. A is M x n row-major (overwritten),
 * S is M x nrhs row-major (overwritten), beta is n x nrhs row-major.
 * Returns 1 if full rank (min|R_jj| >= 1e-10 max|R_jj|), else 0 and beta
 * is left untouched. */
int    or_ols_qr(double* A, int64_t M, int n, double* S, int nrhs, double* beta);

/* --- SRMDP (Alg. srmdp) ---
 * table: N * K * B doubles, B = (q+1)(d+1), layout docs/layout.md (unpadded).
 * or_step computes table[i][k] for k in [k_begin, k_end) with stride k_stride,
 * reading table[j][*] for j > i. Returns the number of LP0 fallbacks. */
int64_t or_step(const or_problem* p, double* table, int i,
                int64_t k_begin, int64_t k_end, int64_t k_stride);
/* Same for an explicit list of cells (used to evaluate only visited cells). */
int64_t or_step_cells(const or_problem* p, double* table, int i, const int64_t* cells, int64_t n);
int64_t or_solve(const or_problem* p, double* table);
/* Evaluate the truncated approximations at time i (i == N: g, z ignored). */
void   or_eval(const or_problem* p, const double* table, int i, int64_t n,
               const double* x, double* y, double* z);
int    or_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
