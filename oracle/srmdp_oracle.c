/*
 * srmdp_oracle.c — CPU ORACLE of the SRMDP backward sweep. TEST INFRASTRUCTURE:
 * only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / reference
 * leg) may load this. It shares no code with paper_2407_21085_b200/ (the CUDA
 * product); both follow the written specs docs/streams.md, docs/detmath.md,
 * docs/layout.md and the paper.
 *
 * Paper: Gobet, Lopez-Salas, Turkedjiev, Vazquez, "Stratified regression
 * Monte-Carlo scheme for semilinear PDEs and BSDEs with large scale
 * parallelization on GPUs", arXiv 2407.21085. P:n = line n of PAPER.md.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared (no -ffast-math),
 * so every a*b+c below is two roundings unless written fma().
 *
 * Pins (tests/test_oracle_*.py, all `-m "not gpu"`):
 *   philox            Random123/cuRAND known-answer vectors
 *   or_u01            exact extremes 2^-53, 1-2^-53
 *   dm_log/exp/sincos mpmath at <= 3 ulp (path and reference/series versions)
 *   F, inv_cdf_cond   closed forms (F(ln 3)=0.75, medians), KS vs analytic CDF
 *   locate            SPEC-style examples, membership of every sample
 *   euler             closed-form random walk / ODE examples
 *   or_ols_qr         numpy.linalg.lstsq (LAPACK), exact affine recovery
 *   or_bounds         C_y = e^{6.25} example, C_z sqrt(dt) = C_y
 *   or_step/or_solve  deterministic bookkeeping closed form (affine y to rounding),
 *                     linear BS-type exact discrete solution (mean over seeds),
 *                     benchmark d=1 vs Gauss-Hermite discrete MDP, nested MC
 *   or_eval           truncation binding with small C_y
 * parity unpinned: none of the functions above is unpinned; the finite-M value
 * of the nonlinear benchmark solve is pinned only statistically.
 */
#include "srmdp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (docs/streams.md §1)                                   */
/* ------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; r++) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* docs/streams.md §3: u = (2*(w>>12)+1) * 2^-53, exact. */
double or_u01(uint64_t w) {
  return (double)(2u * (w >> 12) + 1u) * 0x1p-53;
}

static void draw_block(const or_problem* p, uint32_t c0, int64_t m, int64_t k, int i,
                       int domain, double* ua, double* ub) {
  uint32_t ctr[4] = {c0, (uint32_t)m, (uint32_t)k, (uint32_t)i | ((uint32_t)domain << 24)};
  uint32_t key[2] = {(uint32_t)(p->seed & 0xffffffffu), (uint32_t)(p->seed >> 32)};
  uint32_t o[4];
  or_philox4x32_10(ctr, key, o);
  uint64_t wa = ((uint64_t)o[1] << 32) | o[0];
  uint64_t wb = ((uint64_t)o[3] << 32) | o[2];
  *ua = or_u01(wa);
  *ub = or_u01(wb);
}

/* ------------------------------------------------------------------ */
/* detmath (docs/detmath.md)                                           */
/* ------------------------------------------------------------------ */
static const double LN2_HI = 0x1.62e42fee00000p-1;
static const double LN2_LO = 0x1.a39ef35793c76p-33;

double or_dm_log_series(double x) {
  static const double LG[11] = {0.0,
      0x1.5555555555555p-1, 0x1.999999999999ap-2, 0x1.2492492492492p-2,
      0x1.c71c71c71c71cp-3, 0x1.745d1745d1746p-3, 0x1.3b13b13b13b14p-3,
      0x1.1111111111111p-3, 0x1.e1e1e1e1e1e1ep-4, 0x1.af286bca1af28p-4,
      0x1.8618618618618p-4};
  if (x != x || x < 0.0) return NAN;
  if (x == 0.0) return -INFINITY;
  if (isinf(x)) return INFINITY;
  int k = 0;
  if (x < 0x1p-1022) { x = x * 0x1p54; k = -54; }
  uint64_t b;
  memcpy(&b, &x, 8);
  k = k + (int)(b >> 52) - 1023;
  uint64_t mb = (b & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
  double m;
  memcpy(&m, &mb, 8);
  if (m > 0x1.6a09e667f3bcdp+0) { m = m * 0.5; k = k + 1; }
  double f = m - 1.0;
  double s = f / (2.0 + f);
  double z = s * s;
  double P = LG[10];
  for (int j = 9; j >= 1; j--) P = fma(P, z, LG[j]);
  double R = z * P;
  double t = s * R;
  double lm = (2.0 * s) + t;
  double hi = (double)k * LN2_HI;
  double lo = (double)k * LN2_LO;
  return hi + (lm + lo);
}

double or_dm_exp(double x) {
  static const double E[15] = {
      0x1p+0, 0x1p+0, 0x1p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5,
      0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
      0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22,
      0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33,
      0x1.93974a8c07c9dp-37};
  if (x != x) return NAN;
  if (x > 709.782712893384) return INFINITY;
  if (x < -745.1332191019412) return 0.0;
  double kf = rint(x * 0x1.71547652b82fep+0);
  double r = (x - (kf * LN2_HI)) - (kf * LN2_LO);
  double P = E[14];
  for (int j = 13; j >= 0; j--) P = fma(P, r, E[j]);
  return ldexp(P, (int)kf);
}

void or_dm_sincospi2_series(double u, double* s, double* c) {
  static const double S[9] = {
      0x1.921fb54442d18p+0, -0x1.4abbce625be53p-1, 0x1.466bc6775aae2p-4,
      -0x1.32d2cce62bd86p-8, 0x1.50783487ee782p-13, -0x1.e3074fde8871fp-19,
      0x1.e8f434d018d63p-25, -0x1.6fadb9f155744p-31, 0x1.aaec32af93359p-38};
  static const double Cc[10] = {
      0x1.0000000000000p+0, -0x1.3bd3cc9be45dep+0, 0x1.03c1f081b5ac4p-2,
      -0x1.55d3c7e3cbffap-6, 0x1.e1f506891babbp-11, -0x1.a6d1f2a204a8cp-16,
      0x1.f9d38a3763cc3p-22, -0x1.b6e24f44b128fp-28, 0x1.20c62c2f2d7f5p-34,
      -0x1.2a0c591af8314p-41};
  double v = 4.0 * u;
  double n = rint(v);
  double f = v - n;
  double f2 = f * f;
  double ps = S[8];
  for (int j = 7; j >= 0; j--) ps = fma(ps, f2, S[j]);
  double sn = f * ps;
  double pc = Cc[9];
  for (int j = 8; j >= 0; j--) pc = fma(pc, f2, Cc[j]);
  double cs = pc;
  int q = ((int)n) & 3;
  switch (q) {
    case 0: *s = sn; *c = cs; break;
    case 1: *s = cs; *c = -sn; break;
    case 2: *s = -sn; *c = -cs; break;
    default: *s = -cs; *c = sn; break;
  }
}

/* Tables of docs/detmath.md, built once from the reference functions. */
static double LOGT_INVC[128], LOGT_LT[128], SCT_S[128], SCT_C[128];
static pthread_once_t tables_once = PTHREAD_ONCE_INIT;

static void build_tables(void) {
  for (int j = 0; j < 128; j++) {
    if (j == 0 || j == 127) {
      LOGT_INVC[j] = 1.0;
      LOGT_LT[j] = 0.0;
    } else {
      double c = 1.0 + (((double)j + 0.5) / 128.0);
      if (j >= 53) c = c * 0.5;
      LOGT_INVC[j] = 1.0 / c;
      LOGT_LT[j] = -or_dm_log_series(LOGT_INVC[j]);
    }
    or_dm_sincospi2_series((double)j / 128.0, &SCT_S[j], &SCT_C[j]);
  }
}

void or_init_tables(void) { pthread_once(&tables_once, build_tables); }

/* dm_log (path function, docs/detmath.md): table-driven, division-free. */
double or_dm_log(double x) {
  static const double A[10] = {0.0, 0.0,
      -0x1.0000000000000p-1, 0x1.5555555555555p-2, -0x1.0000000000000p-2, 0x1.999999999999ap-3,
      -0x1.5555555555555p-3, 0x1.2492492492492p-3, -0x1.0000000000000p-3, 0x1.c71c71c71c71cp-4};
  or_init_tables();
  if (x != x || x < 0.0) return NAN;
  if (x == 0.0) return -INFINITY;
  if (isinf(x)) return INFINITY;
  int k = 0;
  if (x < 0x1p-1022) { x = x * 0x1p54; k = -54; }
  uint64_t b;
  memcpy(&b, &x, 8);
  k = k + (int)(b >> 52) - 1023;
  uint64_t mb = b & 0x000fffffffffffffull;
  int j = (int)(mb >> 45);
  uint64_t m1 = mb | 0x3ff0000000000000ull;
  double m;
  memcpy(&m, &m1, 8);
  if (j >= 53) { m = m * 0.5; k = k + 1; }
  double r = fma(m, LOGT_INVC[j], -1.0);
  double r2 = r * r;
  double p = A[9];
  for (int n = 8; n >= 2; n--) p = fma(p, r, A[n]);
  double l1 = fma(r2, p, r);
  double kd = (double)k;
  return ((kd * LN2_HI) + LOGT_LT[j]) + (l1 + (kd * LN2_LO));
}

/* dm_sincospi2 (path function, docs/detmath.md): (sin 2 pi u, cos 2 pi u), 0 <= u < 1. */
void or_dm_sincospi2(double u, double* s, double* c) {
  static const double Pk[5] = {0x1.921fb54442d18p-5, -0x1.4abbce625be53p-16, 0x1.466bc6775aae2p-29,
                               -0x1.32d2cce62bd86p-43, 0x1.50783487ee782p-58};
  static const double Qk[5] = {0x1.0000000000000p+0, -0x1.3bd3cc9be45dep-10, 0x1.03c1f081b5ac4p-22,
                               -0x1.55d3c7e3cbffap-36, 0x1.e1f506891babbp-51};
  or_init_tables();
  double t = u * 128.0;
  int j = (int)floor(t);
  double g = t - (double)j;
  double g2 = g * g;
  double ps = Pk[4];
  for (int k = 3; k >= 0; k--) ps = fma(ps, g2, Pk[k]);
  double sg = g * ps;
  double pc = Qk[4];
  for (int k = 3; k >= 0; k--) pc = fma(pc, g2, Qk[k]);
  double cg = pc;
  double Sj = SCT_S[j], Cj = SCT_C[j];
  *s = fma(Sj, cg, Cj * sg);
  *c = fma(Cj, cg, -(Sj * sg));
}

/* ------------------------------------------------------------------ */
/* Stratification: (A_nu) P:216-229, Alg. stratify,           */
/* (A_Strat.) P:188-197. docs/streams.md §5-6, docs/layout.md.          */
/* ------------------------------------------------------------------ */

/* F_nu(x) = 1/(1+exp(-mu x)). */
double or_F(double mu, double x) {
  if (x == -INFINITY) return 0.0;
  if (x == INFINITY) return 1.0;
  return 1.0 / (1.0 + or_dm_exp(-(mu * x)));
}

static double edge(int c, int C, double L) {
  /* e_c = -L + c*delta, e_0 = -inf, e_C = +inf (outer strata infinite). */
  if (c <= 0) return -INFINITY;
  if (c >= C) return INFINITY;
  double delta = (2.0 * L) / (double)C;
  return (-L) + ((double)c * delta);
}

/* Breakpoint c of the problem's grid (docs/streams.md §5/§6b). Equal-probability
 * strata ((A_Strat.) example ii): e_c = F^{-1}(c/C) = -(1/mu) log(C/c - 1). */
static double edge_p(const or_problem* p, int c) {
  if (p->grid == 0) return edge(c, p->C, p->L);
  if (c <= 0) return -INFINITY;
  if (c >= p->C) return INFINITY;
  return (-(1.0 / p->mu)) * or_dm_log(((double)p->C / (double)c) - 1.0);
}

/* Locate one coordinate: docs/streams.md §6. */
int or_locate1(double x, int C, double L) {
  double inv_delta = (double)C / (2.0 * L);
  double t = floor((x + L) * inv_delta);
  t = fmax(t, 0.0);
  t = fmin(t, (double)(C - 1));
  return (int)t;
}

int64_t or_num_cells(const or_problem* p) {
  int64_t K = 1;
  for (int l = 0; l < p->d; l++) K *= p->C;
  return K;
}

/* Cell of one coordinate on the problem's grid: uniform grid as or_locate1;
 * equal-probability grid: the number of breakpoints e_1..e_{C-1} <= x. */
static int locate1_p(const or_problem* p, double x) {
  if (p->grid == 0) return or_locate1(x, p->C, p->L);
  int c = 0;
  for (int l = 1; l < p->C; l++)
    if (x >= edge_p(p, l)) c = l;
  return c;
}

int64_t or_locate(const or_problem* p, const double* x) {
  int64_t k = 0;
  for (int l = 0; l < p->d; l++) k = k * p->C + locate1_p(p, x[l]);
  return k;
}

static void cell_coords(const or_problem* p, int64_t k, int* c) {
  for (int l = p->d - 1; l >= 0; l--) { c[l] = (int)(k % p->C); k /= p->C; }
}

void or_cell_center(const or_problem* p, int64_t k, double* r) {
  int c[64];
  cell_coords(p, k, c);
  int C = p->C;
  double delta = (2.0 * p->L) / (double)C;
  for (int l = 0; l < p->d; l++) {
    if (p->grid != 0) {   /* equal-probability grid: midpoints, finite edge for outer cells */
      if (C == 1) r[l] = 0.0;
      else if (c[l] == 0) r[l] = edge_p(p, 1);
      else if (c[l] == C - 1) r[l] = edge_p(p, C - 1);
      else r[l] = (edge_p(p, c[l]) + edge_p(p, c[l] + 1)) * 0.5;
      continue;
    }
    if (C == 1) r[l] = 0.0;
    else if (c[l] == 0) r[l] = (-p->L) + (1.0 * delta);
    else if (c[l] == C - 1) r[l] = (-p->L) + ((double)(C - 1) * delta);
    else r[l] = (-p->L) + (((double)c[l] + 0.5) * delta);
  }
}

/* F^{-1}_{nu,[lo,hi)}(U) = -(1/mu) log(1/(F(lo)+U(F(hi)-F(lo))) - 1). */
double or_inv_cdf_cond(double mu, double lo, double hi, double U) {
  double Fa = or_F(mu, lo), Fb = or_F(mu, hi);
  double dF = Fb - Fa;
  double pr = Fa + (U * dF);
  if (pr >= 1.0) pr = 0x1.fffffffffffffp-1;
  if (pr <= 0.0) pr = 0x1p-1022;
  double w = (1.0 / pr) - 1.0;
  double neg_inv_mu = -(1.0 / mu);
  return neg_inv_mu * or_dm_log(w);
}

/* One start-point coordinate in cell c of a dimension, with the membership
 * fix-up of docs/streams.md §5 (reading R7). */
static double sample_coord(const or_problem* p, int c, double U) {
  double lo = edge_p(p, c), hi = edge_p(p, c + 1);
  double x = or_inv_cdf_cond(p->mu, lo, hi, U);
  if (isfinite(lo) && x < lo) x = lo;
  if (isfinite(hi) && x >= hi) x = nextafter(hi, -INFINITY);
  int n = 0;
  while (locate1_p(p, x) < c && n < 4096) { x = nextafter(x, INFINITY); n++; }
  while (locate1_p(p, x) > c && n < 4096) { x = nextafter(x, -INFINITY); n++; }
  return x;
}

/* X^{i,nu_k}_i ~ nu_k by Alg. stratify; Philox blocks c0 = 0..ceil(d/2)-1. */
void or_start_point(const or_problem* p, int i, int64_t k, int64_t m, double* x) {
  int c[64];
  cell_coords(p, k, c);
  int nb = (p->d + 1) / 2;
  for (int b = 0; b < nb; b++) {
    double ua, ub;
    draw_block(p, (uint32_t)b, m, k, i, 0, &ua, &ub);
    x[2 * b] = sample_coord(p, c[2 * b], ua);
    if (2 * b + 1 < p->d) x[2 * b + 1] = sample_coord(p, c[2 * b + 1], ub);
  }
}

/* dW_j of path m of cloud (i,k): Box-Muller, docs/streams.md §4. */
void or_brownian(const or_problem* p, int i, int j, int64_t k, int64_t m, double* dW) {
  double dt = p->T / (double)p->N;
  double sdt = sqrt(dt);
  int nbd = (p->d + 1) / 2, nbq = (p->q + 1) / 2;
  for (int b = 0; b < nbq; b++) {
    double ua, ub, s, c;
    draw_block(p, (uint32_t)(nbd + (j - i) * nbq + b), m, k, i, 0, &ua, &ub);
    double rho = sqrt((-2.0) * or_dm_log(ua));
    or_dm_sincospi2(ub, &s, &c);
    double n0 = rho * c, n1 = rho * s;
    dW[2 * b] = sdt * n0;
    if (2 * b + 1 < p->q) dW[2 * b + 1] = sdt * n1;
  }
}

/* ------------------------------------------------------------------ */
/* Problem functions: P:909-921 (benchmark), eq. fbsde P:25-38.          */
/* ------------------------------------------------------------------ */

/* Euler dynamics, Alg. Euler P:161-164 (indices t_j, X_j, dW_j: reading R1),
 * op order frozen by docs/streams.md §7. */
void or_euler(const or_problem* p, double t, const double* x, const double* dW, double* xn) {
  (void)t;
  double dt = p->T / (double)p->N;
  int d = p->d, q = p->q;
  if (p->dyn_kind == OR_DYN_BM) {
    for (int l = 0; l < d; l++) xn[l] = x[l] + dW[l];
  } else if (p->dyn_kind == OR_DYN_USER) {
    /* user b(t_j, X_j), sigma(t_j, X_j): X + (b dt + sigma dW), sigma dW summed
     * over p = 0..q-1 in order (srmdp.h "User problems"). */
    double b[64], sg[64 * 64];
    p->user_b(p->user_params, t, x, b);
    p->user_sigma(p->user_params, t, x, sg);
    for (int l = 0; l < d; l++) {
      double sw = sg[l * q + 0] * dW[0];
      for (int pp = 1; pp < q; pp++) sw = sw + (sg[l * q + pp] * dW[pp]);
      xn[l] = x[l] + ((b[l] * dt) + sw);
    }
  } else if (p->dyn_kind == OR_DYN_GBM_EXACT) {
    /* Alg. "SDE dynamics": exact transition of dX = mu X dt + s X dW. */
    const double* mu = p->dyn_params;
    const double* s = p->dyn_params + d;
    for (int l = 0; l < d; l++) {
      double a = mu[l] - (0.5 * (s[l] * s[l]));
      xn[l] = x[l] * or_dm_exp((a * dt) + (s[l] * dW[l]));
    }
  } else if (p->dyn_kind == OR_DYN_GBM) {
    const double* mu = p->dyn_params;
    const double* s = p->dyn_params + d;
    for (int l = 0; l < d; l++) {
      double a = (mu[l] * x[l]) * dt;
      double b = (s[l] * x[l]) * dW[l];
      xn[l] = x[l] + (a + b);
    }
  } else {
    const double* b0 = p->dyn_params;
    const double* B1 = p->dyn_params + d;
    const double* S0 = p->dyn_params + d + d * d;
    for (int l = 0; l < d; l++) {
      double b = b0[l];
      for (int kk = 0; kk < d; kk++) b = b + (B1[l * d + kk] * x[kk]);
      double sw = S0[l * q + 0] * dW[0];
      for (int pp = 1; pp < q; pp++) sw = sw + (S0[l * q + pp] * dW[pp]);
      xn[l] = x[l] + ((b * dt) + sw);
    }
  }
}

/* Terminal condition g. PAPER: g = omega/(1+omega), omega = exp(T + sum x)
 * (P:914), written 1/(1+exp(-(T+sum x))) (reading R22: same value, no overflow). */
double or_g(const or_problem* p, const double* x) {
  double s = 0.0;
  if (p->g_kind == OR_G_USER) return p->user_g(p->user_params, x);
  if (p->g_kind == OR_G_AFFINE) {
    s = p->g_params[0];
    for (int l = 0; l < p->d; l++) s = s + p->g_params[1 + l] * x[l];
    return s;
  }
  s = p->T;
  for (int l = 0; l < p->d; l++) s = s + x[l];
  return 1.0 / (1.0 + exp(-s));
}

/* Driver f_j(x, y, z) = f(t_j, x, y, z) (reading R17).
 * PAPER: (sum_k z_k)(y - (2+q)/(2q)). LINEAR: a y + theta.z + c. */
double or_f(const or_problem* p, double t, const double* x, double y, const double* z) {
  if (p->f_kind == OR_F_USER) return p->user_f(p->user_params, t, x, y, z);
  if (p->f_kind == OR_F_ZERO) return 0.0;
  if (p->f_kind == OR_F_LINEAR) {
    double v = p->f_params[0] * y;
    for (int l = 0; l < p->q; l++) v = v + p->f_params[2 + l] * z[l];
    return v + p->f_params[1];
  }
  double sz = 0.0;
  for (int l = 0; l < p->q; l++) sz = sz + z[l];
  double c = (2.0 + (double)p->q) / (2.0 * (double)p->q);
  return sz * (y - c);
}

/* Truncation T_L (eq. TL): -L v x ^ L. */
static double trunc_L(double v, double Lb) {
  if (v < -Lb) return -Lb;
  if (v > Lb) return Lb;
  return v;
}

/* Prop. bound (eq. prop:bound) and C_* of Lemma P:379-383. */
int or_bounds(double C_g, double C_f, double L_f, int q, double T, int N,
              double* C_y, double* C_z, double* C_star) {
  double dt = T / (double)N;
  double Lf2 = L_f * L_f;
  double a = (Lf2 > 1.0 ? Lf2 : 1.0);
  double Tv = (T > 1.0 ? T : 1.0);
  double cy = exp(T / 4.0 + 6.0 * (double)q * a * Tv) * (C_g + T * C_f / (2.0 * sqrt((double)q)));
  *C_y = cy;
  *C_z = cy / sqrt(dt);
  *C_star = C_g + T * (L_f * cy * (1.0 + sqrt((double)q) / sqrt(dt)) + C_f);
  return (dt * Lf2 <= 1.0 / (12.0 * (double)q)) ? 1 : 0;
}

/* ------------------------------------------------------------------ */
/* Evaluation of the fitted, truncated functions. */
/* ------------------------------------------------------------------ */
static void eval_block(const or_problem* p, const double* blk, int64_t cell,
                       const double* x, double* y, double* z) {
  int d = p->d;
  double r[64], a[65];
  or_cell_center(p, cell, r);
  a[0] = 1.0;
  for (int l = 0; l < d; l++) a[l + 1] = x[l] - r[l];
  double v = 0.0;
  for (int j = 0; j <= d; j++) v = v + blk[j] * a[j];
  *y = trunc_L(v, p->C_y);
  if (z) {
    for (int l = 0; l < p->q; l++) {
      const double* bz = blk + (size_t)(1 + l) * (d + 1);
      double w = 0.0;
      for (int j = 0; j <= d; j++) w = w + bz[j] * a[j];
      z[l] = trunc_L(w, p->C_z);
    }
  }
}

void or_eval(const or_problem* p, const double* table, int i, int64_t n,
             const double* x, double* y, double* z) {
  int d = p->d, q = p->q;
  int64_t K = or_num_cells(p);
  size_t B = (size_t)(q + 1) * (d + 1);
  for (int64_t t = 0; t < n; t++) {
    const double* xt = x + t * d;
    if (i == p->N) { y[t] = or_g(p, xt); continue; }   /* y_N := g */
    int64_t c = or_locate(p, xt);
    eval_block(p, table + ((size_t)i * K + c) * B, c, xt, &y[t], z ? z + t * q : NULL);
  }
}

/* ------------------------------------------------------------------ */
/* Trace of one simulated path (for bit-exact path-state parity).        */
/* ------------------------------------------------------------------ */
void or_trace_path(const or_problem* p, int i, int64_t k, int64_t m,
                   double* x, int64_t* cell, double* dW) {
  int d = p->d, q = p->q, N = p->N;
  double dt = p->T / (double)N;
  or_start_point(p, i, k, m, x);
  cell[0] = or_locate(p, x);
  for (int j = i; j < N; j++) {
    double* xj = x + (size_t)(j - i) * d;
    double* xn = xj + d;
    double* w = dW + (size_t)(j - i) * q;
    or_brownian(p, i, j, k, m, w);
    or_euler(p, (double)j * dt, xj, w, xn);
    cell[j - i + 1] = or_locate(p, xn);
  }
}

/* ------------------------------------------------------------------ */
/* Householder QR least squares (Golub-Van Loan Alg. 5.3.2). */
/* ------------------------------------------------------------------ */
int or_ols_qr(double* A, int64_t M, int n, double* S, int nrhs, double* beta) {
  if (M < n) return 0;                               /* rank < n: P:712 needs M >= d+1 */
  double* v = (double*)malloc(sizeof(double) * (size_t)M);
  double rdiag[128];
  for (int j = 0; j < n; j++) {
    /* Householder vector for column j, rows j..M-1. */
    double nrm = 0.0;
    for (int64_t r = j; r < M; r++) nrm = nrm + A[r * n + j] * A[r * n + j];
    nrm = sqrt(nrm);
    double x0 = A[(int64_t)j * n + j];
    double alpha = (x0 > 0.0) ? -nrm : nrm;       /* R_jj = alpha */
    rdiag[j] = alpha;
    double vnorm2 = 0.0;
    for (int64_t r = j; r < M; r++) v[r] = A[r * n + j];
    v[j] = x0 - alpha;
    for (int64_t r = j; r < M; r++) vnorm2 = vnorm2 + v[r] * v[r];
    if (vnorm2 == 0.0) continue;                     /* column already reduced */
    /* Apply H = I - 2 v v^T / (v^T v) to A[j:, j:] and S[j:, :]. */
    for (int c = j; c < n; c++) {
      double dot = 0.0;
      for (int64_t r = j; r < M; r++) dot = dot + v[r] * A[r * n + c];
      double sc = 2.0 * dot / vnorm2;
      for (int64_t r = j; r < M; r++) A[r * n + c] = A[r * n + c] - sc * v[r];
    }
    for (int c = 0; c < nrhs; c++) {
      double dot = 0.0;
      for (int64_t r = j; r < M; r++) dot = dot + v[r] * S[r * nrhs + c];
      double sc = 2.0 * dot / vnorm2;
      for (int64_t r = j; r < M; r++) S[r * nrhs + c] = S[r * nrhs + c] - sc * v[r];
    }
  }
  free(v);
  double mx = 0.0, mn = INFINITY;
  for (int j = 0; j < n; j++) {
    double a = fabs(rdiag[j]);
    if (a > mx) mx = a;
    if (a < mn) mn = a;
  }
  if (!(mn >= 1e-10 * mx) || mx == 0.0) return 0;
  /* Back substitution R beta = (Q^T S)[0:n] (eq. lp1:explicit). */
  for (int c = 0; c < nrhs; c++) {
    for (int j = n - 1; j >= 0; j--) {
      double s = S[(int64_t)j * nrhs + c];
      for (int jj = j + 1; jj < n; jj++) s = s - A[(int64_t)j * n + jj] * beta[jj * nrhs + c];
      beta[j * nrhs + c] = s / A[(int64_t)j * n + j];
    }
  }
  return 1;
}

/* ------------------------------------------------------------------ */
/* Alg. SRMDP, one time step i (eq. PsiM).           */
/* ------------------------------------------------------------------ */
static int64_t step_cell(const or_problem* p, double* table, int i, int64_t k) {
  const int d = p->d, q = p->q, N = p->N, n = d + 1;
  const int64_t M = p->M, K = or_num_cells(p);
  const size_t B = (size_t)(q + 1) * (d + 1);
  const double dt = p->T / (double)N;
  double r[64], x[64], X[64], Xn[64], dW[64], dWi[64], zcur[64], zv[64];
  or_cell_center(p, k, r);

  double* A = (double*)malloc(sizeof(double) * (size_t)M * n);   /* design */
  double* A2 = (double*)malloc(sizeof(double) * (size_t)M * n);
  double* SZ = (double*)malloc(sizeof(double) * (size_t)M * q);  /* Z responses */
  double* SY = (double*)malloc(sizeof(double) * (size_t)M);      /* Y responses */
  double* Bm = (double*)malloc(sizeof(double) * (size_t)M);      /* S_{Y,i+1} */
  double* Y1 = (double*)malloc(sizeof(double) * (size_t)M);      /* y_{i+1}(x_{i+1}) */
  double* Xi = (double*)malloc(sizeof(double) * (size_t)M * d);  /* x_i^m */

  for (int64_t m = 0; m < M; m++) {
    /* Cloud C_{i,k}: start point ~ nu_k, then the Euler chain. */
    or_start_point(p, i, k, m, x);
    for (int l = 0; l < d; l++) { X[l] = x[l]; Xi[m * d + l] = x[l]; }
    A[m * n + 0] = 1.0;
    for (int l = 0; l < d; l++) A[m * n + 1 + l] = x[l] - r[l];
    double acc = 0.0, y1 = 0.0, gN = 0.0;
    for (int j = i; j < N; j++) {
      double tj = (double)j * dt;
      or_brownian(p, i, j, k, m, dW);
      or_euler(p, tj, X, dW, Xn);
      double yv;
      if (j + 1 < N) {
        /* y^{(M)}_{j+1}(x_{j+1}), z^{(M)}_{j+1}(x_{j+1}) from the fitted table. */
        int64_t c = or_locate(p, Xn);
        eval_block(p, table + ((size_t)(j + 1) * K + c) * B, c, Xn, &yv, zv);
      } else {
        yv = or_g(p, Xn);           /* y_N := g */
        gN = yv;
      }
      if (j == i) {
        y1 = yv;
        for (int l = 0; l < q; l++) dWi[l] = dW[l];
      } else {
        /* f_j(x_j, y_{j+1}(x_{j+1}), z_j(x_j)) dt, j = i+1..N-1 (eq. PsiM). */
        double fdt = or_f(p, tj, X, yv, zcur) * dt;
        acc = acc + fdt;
      }
      for (int l = 0; l < q; l++) zcur[l] = zv[l];
      for (int l = 0; l < d; l++) X[l] = Xn[l];
    }
    double Bv = gN + acc;          /* S_{Y,i+1}(x_i) */
    Bm[m] = Bv;
    Y1[m] = y1;
    for (int l = 0; l < q; l++) SZ[m * q + l] = (Bv * dWi[l]) / dt;   /* S_{Z,i} = S_{Y,i+1} w / dt */
  }

  int64_t fallbacks = 0;
  double* blk = table + ((size_t)i * K + k) * B;
  double betaZ[64 * 65], betaY[65];
  double* SZ0 = (double*)malloc(sizeof(double) * (size_t)M * q);
  memcpy(SZ0, SZ, sizeof(double) * (size_t)M * q);
  memcpy(A2, A, sizeof(double) * (size_t)M * n);
  /* Z first: OLS(S_Z, L_Z,k, nu_{i,k,M}). LP0: the OLS on the
   * constant basis is the mean (eq. lp0:explicit). */
  int ok = p->lp0 ? 0 : or_ols_qr(A2, M, n, SZ, q, betaZ);
  if (ok) {
    for (int l = 0; l < q; l++)
      for (int j = 0; j < n; j++) blk[(size_t)(1 + l) * n + j] = betaZ[j * q + l];
  } else {
    /* LP0 basis, or rank-deficient LP1 design: LP0 fallback (eq. lp0:explicit
     * P:700-707, reading R15) = mean of the responses (fallbacks counted). */
    fallbacks = p->lp0 ? 0 : 1;
    for (int l = 0; l < q; l++) {
      double s = 0.0;
      for (int64_t m = 0; m < M; m++) s = s + SZ0[m * q + l];
      blk[(size_t)(1 + l) * n + 0] = s / (double)M;
      for (int j = 1; j < n; j++) blk[(size_t)(1 + l) * n + j] = 0.0;
    }
  }
  free(SZ0);
  /* z^{(M)}_i|_{H_k} := T_{C_z}(psi_Z). Y responses:
   * S_{Y,i} = S_{Y,i+1} + f_i(x_i, y_{i+1}(x_{i+1}), z_i(x_i)) dt. */
  for (int64_t m = 0; m < M; m++) {
    double zi[64], a[65];
    const double* xm = Xi + m * d;
    a[0] = 1.0;
    for (int l = 0; l < d; l++) a[l + 1] = xm[l] - r[l];
    for (int l = 0; l < q; l++) {
      const double* bz = blk + (size_t)(1 + l) * n;
      double w = 0.0;
      for (int j = 0; j <= d; j++) w = w + bz[j] * a[j];
      zi[l] = trunc_L(w, p->C_z);
    }
    double fdt = or_f(p, (double)i * dt, xm, Y1[m], zi) * dt;
    SY[m] = Bm[m] + fdt;
  }
  if (ok) {
    memcpy(A2, A, sizeof(double) * (size_t)M * n);
    /* OLS(S_Y, L_Y,k, nu_{i,k,M}); same design, same rank. */
    ok = or_ols_qr(A2, M, n, SY, 1, betaY);
    for (int j = 0; j < n; j++) blk[j] = betaY[j];
  } else {
    double s = 0.0;
    for (int64_t m = 0; m < M; m++) s = s + SY[m];
    blk[0] = s / (double)M;
    for (int j = 1; j < n; j++) blk[j] = 0.0;
  }
  for (size_t b = (size_t)(q + 1) * n; b < B; b++) blk[b] = 0.0;

  free(A); free(A2); free(SZ); free(SY); free(Bm); free(Y1); free(Xi);
  return fallbacks;
}

int64_t or_step(const or_problem* p, double* table, int i,
                int64_t k_begin, int64_t k_end, int64_t k_stride) {
  int64_t fb = 0;
  or_init_tables();
  if (k_stride < 1) k_stride = 1;
  int64_t cnt = (k_end > k_begin) ? (k_end - k_begin + k_stride - 1) / k_stride : 0;
#pragma omp parallel for schedule(static) reduction(+ : fb)
  for (int64_t t = 0; t < cnt; t++) fb += step_cell(p, table, i, k_begin + t * k_stride);
  return fb;
}

int64_t or_step_cells(const or_problem* p, double* table, int i, const int64_t* cells, int64_t n) {
  int64_t fb = 0;
  or_init_tables();
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : fb)
  for (int64_t t = 0; t < n; t++) fb += step_cell(p, table, i, cells[t]);
  return fb;
}

/* Backward iteration i = N-1 .. 0. */
int64_t or_solve(const or_problem* p, double* table) {
  int64_t K = or_num_cells(p), fb = 0;
  for (int i = p->N - 1; i >= 0; i--) fb += or_step(p, table, i, 0, K, 1);
  return fb;
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
