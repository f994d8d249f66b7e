/*
 * pdmg_oracle.c -- plain-C restatement of the reference multigrid path.  TEST INFRASTRUCTURE ONLY
 * (see pdmg_oracle.h): the checker for the CUDA path and the CPU baseline, never the product.
 *
 * Floating-point operation order follows the reference line by line so that results are
 * bit-identical to the reference's own grid.cpp/smoother.cpp (built under oracle/_ref).
 * Compile with -ffp-contract=off (no FMA contraction), as the reference's x86-64 -O2 build has.
 */
#include "pdmg_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#undef I /* use _Complex_I explicitly; I is a coordinate name below */

static __thread char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

/* ------------------------------------------------------------------------------------------ */
/* std::mt19937 + std::uniform_real_distribution<double> (libstdc++), restated.                 */
/* tools/pdmg.cpp:137-147: per node draw re then im.                                            */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  uint32_t mt[624];
  int idx;
} mt19937;

static void mt_seed(mt19937* s, uint32_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 624; ++i) s->mt[i] = 1812433253u * (s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) + (uint32_t)i;
  s->idx = 624;
}

static uint32_t mt_next(mt19937* s) {
  if (s->idx >= 624) {
    for (int i = 0; i < 624; ++i) {
      uint32_t y = (s->mt[i] & 0x80000000u) | (s->mt[(i + 1) % 624] & 0x7fffffffu);
      uint32_t v = s->mt[(i + 397) % 624] ^ (y >> 1);
      if (y & 1u) v ^= 0x9908b0dfu;
      s->mt[i] = v;
    }
    s->idx = 0;
  }
  uint32_t y = s->mt[s->idx++];
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

/* generate_canonical<double, 53>: two 32-bit draws, sum = g0 + g1 * 2^32, divided by 2^64. */
static double canonical53(mt19937* s) {
  double sum = 0.0, tmp = 1.0;
  for (int k = 0; k < 2; ++k) {
    sum += (double)mt_next(s) * tmp;
    tmp *= 4294967296.0;
  }
  double r = sum / tmp;
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return r;
}

static double uniform(mt19937* s, double lo, double hi) { return canonical53(s) * (hi - lo) + lo; }

void orc_random_complex(uint32_t seed, double lo, double hi, int64_t count, double* out) {
  mt19937 s;
  mt_seed(&s, seed);
  for (int64_t k = 0; k < count; ++k) {
    const double re = uniform(&s, lo, hi);
    const double im = uniform(&s, lo, hi);
    out[2 * k] = re;
    out[2 * k + 1] = im;
  }
}

void orc_random_real(uint32_t seed, double lo, double hi, int64_t count, double* out) {
  mt19937 s;
  mt_seed(&s, seed);
  for (int64_t k = 0; k < count; ++k) out[k] = uniform(&s, lo, hi);
}

/* principal value of alpha^p for real alpha != 0 (alpha < 0: |alpha|^p e^{i pi p}) */
static orc_cplx real_pow_c(double alpha, double p) {
  if (alpha > 0.0) return pow(alpha, p);
  return pow(-alpha, p) * cexp(_Complex_I * (M_PI * p));
}

void orc_circulant_shifts(double alpha, int nt, double dt, int j0, int count, double* out) {
  const orc_cplx g = real_pow_c(alpha, 1.0 / nt);
  for (int q = 0; q < count; ++q) {
    const int j = j0 + q;
    const double ang = 2.0 * M_PI * (double)j / (double)nt;
    const orc_cplx z = g * cexp(_Complex_I * ang);
    const orc_cplx lam = ((orc_cplx)1.0 - z) / dt;
    out[2 * q] = creal(lam);
    out[2 * q + 1] = cimag(lam);
  }
}

/* ------------------------------------------------------------------------------------------ */
/* Core grid operators: proj/src/grid.cpp                                                       */
/* ------------------------------------------------------------------------------------------ */
#define ROW(p, j, m) ((p) + (size_t)((j)-1) * (size_t)(m)-1) /* grid.hpp:72-73: p[i] = node (i,j) */

double orc_norm(int n, const orc_cplx* v) { /* grid.cpp:7-11 */
  const long N = (long)(n - 1) * (n - 1);
  double s = 0.0;
  for (long k = 0; k < N; ++k) s += creal(v[k]) * creal(v[k]) + cimag(v[k]) * cimag(v[k]);
  return sqrt(s);
}

void orc_apply_stencil(int n, const orc_cplx w[9], double scale, const orc_cplx* u, orc_cplx* out) {
  const int m = n - 1; /* grid.cpp:30-58 */
  for (int j = 1; j <= m; ++j) {
    const orc_cplx* rm = (j > 1) ? ROW(u, j - 1, m) : NULL;
    const orc_cplx* rc = ROW(u, j, m);
    const orc_cplx* rp = (j < m) ? ROW(u, j + 1, m) : NULL;
    orc_cplx* o = ROW(out, j, m);
    for (int i = 1; i <= m; ++i) {
      orc_cplx acc = 0.0;
      const int left = i > 1, right = i < m;
      if (rm) {
        if (left) acc += w[0] * rm[i - 1];
        acc += w[1] * rm[i];
        if (right) acc += w[2] * rm[i + 1];
      }
      if (left) acc += w[3] * rc[i - 1];
      acc += w[4] * rc[i];
      if (right) acc += w[5] * rc[i + 1];
      if (rp) {
        if (left) acc += w[6] * rp[i - 1];
        acc += w[7] * rp[i];
        if (right) acc += w[8] * rp[i + 1];
      }
      o[i] = scale * acc;
    }
  }
}

void orc_apply_shifted_laplacian(int n, orc_cplx lambda, const orc_cplx* u, orc_cplx* out) {
  const int m = n - 1; /* grid.cpp:69-90 */
  const double h = 1.0 / n;
  const double inv_h2 = 1.0 / (h * h);
  const orc_cplx diag = (orc_cplx)4.0 + lambda * (h * h);
  for (int j = 1; j <= m; ++j) {
    const orc_cplx* rm = (j > 1) ? ROW(u, j - 1, m) : NULL;
    const orc_cplx* rc = ROW(u, j, m);
    const orc_cplx* rp = (j < m) ? ROW(u, j + 1, m) : NULL;
    orc_cplx* o = ROW(out, j, m);
    for (int i = 1; i <= m; ++i) {
      orc_cplx acc = diag * rc[i];
      if (i > 1) acc -= rc[i - 1];
      if (i < m) acc -= rc[i + 1];
      if (rm) acc -= rm[i];
      if (rp) acc -= rp[i];
      o[i] = inv_h2 * acc;
    }
  }
}

void orc_residual(int n, orc_cplx lambda, const orc_cplx* b, const orc_cplx* u, orc_cplx* r) {
  orc_apply_shifted_laplacian(n, lambda, u, r); /* grid.cpp:92-100 */
  const long N = (long)(n - 1) * (n - 1);
  for (long k = 0; k < N; ++k) r[k] = b[k] - r[k];
}

void orc_restrict_fw(int n_fine, const orc_cplx* fine, orc_cplx* coarse) {
  const int mf = n_fine - 1, mc = n_fine / 2 - 1; /* grid.cpp:102-121 */
  for (int J = 1; J <= mc; ++J) {
    const orc_cplx* rm = ROW(fine, 2 * J - 1, mf);
    const orc_cplx* rc = ROW(fine, 2 * J, mf);
    const orc_cplx* rp = ROW(fine, 2 * J + 1, mf);
    orc_cplx* o = ROW(coarse, J, mc);
    for (int I = 1; I <= mc; ++I) {
      const int i = 2 * I;
      const orc_cplx sum = rm[i - 1] + 2.0 * rm[i] + rm[i + 1] + 2.0 * rc[i - 1] + 4.0 * rc[i] +
                           2.0 * rc[i + 1] + rp[i - 1] + 2.0 * rp[i] + rp[i + 1];
      o[I] = sum * (1.0 / 16.0);
    }
  }
}

static orc_cplx cval(const orc_cplx* c, int mc, int I, int J) {
  if (I < 1 || I > mc || J < 1 || J > mc) return 0.0;
  return c[(size_t)(J - 1) * mc + (I - 1)];
}

void orc_prolong_bilinear(int n_coarse, const orc_cplx* coarse, orc_cplx* fine) {
  const int mc = n_coarse - 1, mf = 2 * n_coarse - 1; /* grid.cpp:123-153 */
  for (int j = 1; j <= mf; ++j) {
    orc_cplx* o = ROW(fine, j, mf);
    const int J = j / 2;
    const int jeven = (j % 2 == 0);
    for (int i = 1; i <= mf; ++i) {
      const int Ii = i / 2;
      const int ieven = (i % 2 == 0);
      if (ieven && jeven)
        o[i] = cval(coarse, mc, Ii, J);
      else if (!ieven && jeven)
        o[i] = 0.5 * (cval(coarse, mc, Ii, J) + cval(coarse, mc, Ii + 1, J));
      else if (ieven && !jeven)
        o[i] = 0.5 * (cval(coarse, mc, Ii, J) + cval(coarse, mc, Ii, J + 1));
      else
        o[i] = 0.25 * (cval(coarse, mc, Ii, J) + cval(coarse, mc, Ii + 1, J) + cval(coarse, mc, Ii, J + 1) +
                       cval(coarse, mc, Ii + 1, J + 1));
    }
  }
}

/* ------------------------------------------------------------------------------------------ */
/* Smoothers: proj/src/smoother.cpp                                                             */
/* ------------------------------------------------------------------------------------------ */
static int checked_inverse(orc_cplx z, const char* what, orc_cplx* out) { /* smoother.cpp:8-15 */
  if (cabs(z) <= 1e-12)
    return fail(ORC_SINGULAR, "vanka_coeffs: patch eigenvalue %s is singular for this shift", what);
  *out = (orc_cplx)1.0 / z;
  return ORC_OK;
}

int orc_vanka_coeffs(orc_cplx eta, orc_cplx* a, orc_cplx* b, orc_cplx* c) { /* smoother.cpp:18-29 */
  orc_cplx i2, i4, i6;
  int st;
  if ((st = checked_inverse((orc_cplx)2.0 + eta, "2+eta", &i2))) return st;
  if ((st = checked_inverse((orc_cplx)4.0 + eta, "4+eta", &i4))) return st;
  if ((st = checked_inverse((orc_cplx)6.0 + eta, "6+eta", &i6))) return st;
  *a = 0.25 * (i2 + 2.0 * i4 + i6);
  *b = 0.25 * (i2 - i6);
  *c = 0.25 * (i2 - 2.0 * i4 + i6);
  return ORC_OK;
}

int orc_vanka_stencil(orc_cplx lambda, double h, orc_cplx w[9], double* scale) { /* :31-40 */
  orc_cplx a, b, c;
  const int st = orc_vanka_coeffs(lambda * (h * h), &a, &b, &c);
  if (st) return st;
  const orc_cplx tb = 2.0 * b;
  w[0] = c; w[1] = tb; w[2] = c;
  w[3] = tb; w[4] = 4.0 * a; w[5] = tb;
  w[6] = c; w[7] = tb; w[8] = c;
  *scale = h * h / 4.0;
  return ORC_OK;
}

int orc_jacobi_weight(orc_cplx eta, double h, orc_cplx* w) { /* smoother.cpp:42-47 */
  const orc_cplx d = (orc_cplx)4.0 + eta;
  if (cabs(d) <= 1e-12) return fail(ORC_SINGULAR, "jacobi_weight: 4+eta is singular for this shift");
  *w = (orc_cplx)(h * h) / d;
  return ORC_OK;
}

int orc_apply_smoother(int n, orc_cplx lambda, int kind, double omega, const orc_cplx* u,
                       const orc_cplx* b, orc_cplx* out) { /* smoother.cpp:49-67 */
  const double h = 1.0 / n;
  const long N = (long)(n - 1) * (n - 1);
  orc_cplx* r = (orc_cplx*)malloc(sizeof(orc_cplx) * (size_t)N);
  int st = ORC_OK;
  orc_residual(n, lambda, b, u, r);
  if (kind == ORC_JACOBI) {
    orc_cplx jw;
    if ((st = orc_jacobi_weight(lambda * (h * h), h, &jw))) goto done;
    const orc_cplx w = omega * jw;
    for (long k = 0; k < N; ++k) out[k] = u[k] + w * r[k];
  } else {
    orc_cplx w[9];
    double scale;
    if ((st = orc_vanka_stencil(lambda, h, w, &scale))) goto done;
    orc_apply_stencil(n, w, scale, r, out); /* out holds mr */
    const orc_cplx om = omega;              /* mr *= cplx(omega, 0) */
    for (long k = 0; k < N; ++k) out[k] = u[k] + out[k] * om;
  }
done:
  free(r);
  return st;
}

/* ------------------------------------------------------------------------------------------ */
/* Dense operator / patch-sum Vanka / partial-pivot LU: proj/src/dense.cpp (Eigen restated)     */
/* ------------------------------------------------------------------------------------------ */
int orc_dense_operator(int n, orc_cplx lambda, orc_cplx* A) { /* dense.cpp:18-39 */
  if (n > 128) return fail(ORC_CONFIG, "dense_shifted_operator: dense assembly refused for n = %d (limit 128)", n);
  const int m = n - 1;
  const double h = 1.0 / n, inv_h2 = 1.0 / (h * h);
  const orc_cplx diag = ((orc_cplx)4.0 + lambda * (h * h)) * inv_h2;
  const orc_cplx off = -inv_h2;
  const long N = (long)m * m;
  memset(A, 0, sizeof(orc_cplx) * (size_t)(N * N));
#define IDX(i, j) ((long)((j)-1) * m + ((i)-1))
  for (int j = 1; j <= m; ++j)
    for (int i = 1; i <= m; ++i) {
      const long r = IDX(i, j);
      A[r * N + r] = diag;
      if (i > 1) A[r * N + IDX(i - 1, j)] = off;
      if (i < m) A[r * N + IDX(i + 1, j)] = off;
      if (j > 1) A[r * N + IDX(i, j - 1)] = off;
      if (j < m) A[r * N + IDX(i, j + 1)] = off;
    }
  return ORC_OK;
}

/* Inverse of a 4x4 complex matrix by Gauss-Jordan with partial pivoting. */
static void inv4(orc_cplx a[4][4], orc_cplx inv[4][4]) {
  orc_cplx t[4][8];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 8; ++c) t[r][c] = c < 4 ? a[r][c] : (c - 4 == r ? 1.0 : 0.0);
  for (int k = 0; k < 4; ++k) {
    int p = k;
    for (int r = k + 1; r < 4; ++r)
      if (cabs(t[r][k]) > cabs(t[p][k])) p = r;
    for (int c = 0; c < 8; ++c) {
      orc_cplx s = t[k][c];
      t[k][c] = t[p][c];
      t[p][c] = s;
    }
    const orc_cplx piv = t[k][k];
    for (int c = 0; c < 8; ++c) t[k][c] /= piv;
    for (int r = 0; r < 4; ++r)
      if (r != k) {
        const orc_cplx f = t[r][k];
        for (int c = 0; c < 8; ++c) t[r][c] -= f * t[k][c];
      }
  }
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) inv[r][c] = t[r][c + 4];
}

int orc_dense_vanka(int n, orc_cplx lambda, orc_cplx* M) { /* dense.cpp:41-80 */
  if (n > 128) return fail(ORC_CONFIG, "dense_vanka_preconditioner: dense assembly refused for n = %d (limit 128)", n);
  const int m = n - 1;
  const double h = 1.0 / n, inv_h2 = 1.0 / (h * h);
  const long N = (long)m * m;
  const orc_cplx d = ((orc_cplx)4.0 + lambda * (h * h)) * inv_h2, o = -inv_h2;
  /* patch nodes SW, SE, NW, NE; 4-cycle edges SW-SE, SW-NW, SE-NE, NW-NE (dense.cpp:41-54) */
  orc_cplx L[4][4] = {{d, o, o, 0}, {o, d, 0, o}, {o, 0, d, o}, {0, o, o, d}}, Li[4][4];
  inv4(L, Li);
  memset(M, 0, sizeof(orc_cplx) * (size_t)(N * N));
  for (int j = 0; j <= m; ++j)
    for (int i = 0; i <= m; ++i) {
      const int pi[4] = {i, i + 1, i, i + 1}, pj[4] = {j, j, j + 1, j + 1};
      for (int r = 0; r < 4; ++r) {
        if (pi[r] < 1 || pi[r] > m || pj[r] < 1 || pj[r] > m) continue;
        for (int c = 0; c < 4; ++c) {
          if (pi[c] < 1 || pi[c] > m || pj[c] < 1 || pj[c] > m) continue;
          M[IDX(pi[r], pj[r]) * N + IDX(pi[c], pj[c])] += 0.25 * Li[r][c];
        }
      }
    }
#undef IDX
  return ORC_OK;
}

int orc_dense_factor(int n, orc_cplx lambda, orc_dense* d) { /* dense.cpp:82-88 */
  const int m = n - 1;
  const int N = m * m;
  d->N = N;
  d->lu = (orc_cplx*)malloc(sizeof(orc_cplx) * (size_t)N * N);
  d->piv = (int*)malloc(sizeof(int) * (size_t)N);
  int st = orc_dense_operator(n, lambda, d->lu);
  if (st) return st;
  double fro = 0.0;
  for (long k = 0; k < (long)N * N; ++k) fro += creal(d->lu[k]) * creal(d->lu[k]) + cimag(d->lu[k]) * cimag(d->lu[k]);
  fro = sqrt(fro);
  orc_cplx* a = d->lu;
  double min_pivot = INFINITY;
  /* A is banded (lower bandwidth m, upper m; with partial pivoting U's bandwidth grows to 2m): the loops
   * below skip only entries that are exactly zero, so the factors and pivots are those of the dense
   * elimination, operation for operation. */
  for (int k = 0; k < N; ++k) {
    const int rmax = k + m < N - 1 ? k + m : N - 1, cmax = k + 2 * m < N - 1 ? k + 2 * m : N - 1;
    int p = k;
    double best = cabs(a[(long)k * N + k]);
    for (int r = k + 1; r <= rmax; ++r) {
      const double v = cabs(a[(long)r * N + k]);
      if (v > best) best = v, p = r;
    }
    d->piv[k] = p;
    if (p != k)
      for (int c = 0; c < N; ++c) {
        orc_cplx s = a[(long)k * N + c];
        a[(long)k * N + c] = a[(long)p * N + c];
        a[(long)p * N + c] = s;
      }
    const orc_cplx piv = a[(long)k * N + k];
    if (cabs(piv) < min_pivot) min_pivot = cabs(piv);
    if (piv == 0.0) continue;
    for (int r = k + 1; r <= rmax; ++r) {
      const orc_cplx f = a[(long)r * N + k] / piv;
      a[(long)r * N + k] = f;
      for (int c = k + 1; c <= cmax; ++c) a[(long)r * N + c] -= f * a[(long)k * N + c];
    }
  }
  d->singular = !(min_pivot > 1e-14 * fro);
  return ORC_OK;
}

int orc_dense_solve(const orc_dense* d, const orc_cplx* b, orc_cplx* x) { /* dense.cpp:90-100 */
  const int N = d->N;
  if (d->singular) {
    int m = 1;
    while (m * m < N) ++m;
    return fail(ORC_SINGULAR, "DenseShiftedSolver: operator is singular on grid n = %d", m + 1);
  }
  for (int k = 0; k < N; ++k) x[k] = b[k];
  for (int k = 0; k < N; ++k) {
    const int p = d->piv[k];
    if (p != k) {
      orc_cplx s = x[k];
      x[k] = x[p];
      x[p] = s;
    }
  }
  for (int r = 0; r < N; ++r)
    for (int c = 0; c < r; ++c) x[r] -= d->lu[(long)r * N + c] * x[c];
  for (int r = N - 1; r >= 0; --r) {
    for (int c = r + 1; c < N; ++c) x[r] -= d->lu[(long)r * N + c] * x[c];
    x[r] /= d->lu[(long)r * N + r];
  }
  return ORC_OK;
}

void orc_dense_free(orc_dense* d) {
  free(d->lu);
  free(d->piv);
  d->lu = NULL;
  d->piv = NULL;
}

/* ------------------------------------------------------------------------------------------ */
/* Multigrid: proj/src/multigrid.cpp                                                            */
/* ------------------------------------------------------------------------------------------ */
static int validate(const orc_config* c) { /* multigrid.hpp:25-31 */
  if (c->nu1 < 0 || c->nu2 < 0) return fail(ORC_CONFIG, "MultigridConfig: negative smoothing counts");
  if (c->nu1 + c->nu2 == 0) return fail(ORC_CONFIG, "MultigridConfig: nu1 + nu2 must be positive");
  if (c->coarsest_n < 2) return fail(ORC_CONFIG, "MultigridConfig: coarsest_n must be >= 2");
  if (!(c->tol > 0.0)) return fail(ORC_CONFIG, "MultigridConfig: tol must be positive");
  if (c->max_iter < 1) return fail(ORC_CONFIG, "MultigridConfig: max_iter must be >= 1");
  return ORC_OK;
}

int orc_mg_levels(int n, const orc_config* cfg, int* lv) { /* multigrid.cpp:24-44 */
  int st = validate(cfg);
  if (st) return st;
  if (n < 2) return fail(ORC_CONFIG, "Grid2D: need at least 2 subdivisions per side, got %d", n);
  if (n < cfg->coarsest_n)
    return fail(ORC_CONFIG, "MultigridHierarchy: fine grid n = %d is finer than coarsest_n = %d allows", n,
                cfg->coarsest_n);
  int L = 0, g = n;
  lv[L++] = g;
  while (g > cfg->coarsest_n) {
    if (!(g % 2 == 0 && g >= 4))
      return fail(ORC_CONFIG, "MultigridHierarchy: grid n = %d cannot be coarsened to reach coarsest_n = %d", g,
                  cfg->coarsest_n);
    g /= 2;
    lv[L++] = g;
  }
  if (g != cfg->coarsest_n)
    return fail(ORC_CONFIG, "MultigridHierarchy: coarsening from n = %d reaches n = %d, not coarsest_n = %d", n, g,
                cfg->coarsest_n);
  return -L; /* negative level count on success */
}

typedef struct {
  int L;
  int ln[32];
  orc_cplx lambda;
  orc_config cfg;
  orc_dense coarse;
} hier;

static int hier_init(hier* H, int n, orc_cplx lambda, const orc_config* cfg) {
  memset(H, 0, sizeof *H);
  int r = orc_mg_levels(n, cfg, H->ln);
  if (r > 0) return r;
  H->L = -r;
  H->lambda = lambda;
  H->cfg = *cfg;
  for (int l = 0; l + 1 < H->L; ++l) { /* multigrid.cpp:47-58 */
    const double h = 1.0 / H->ln[l];
    orc_cplx a, b, c;
    int st = cfg->smoother == ORC_VANKA ? orc_vanka_coeffs(lambda * (h * h), &a, &b, &c)
                                        : orc_jacobi_weight(lambda * (h * h), h, &a);
    if (st) {
      char inner[512];
      snprintf(inner, sizeof inner, "%s", g_err);
      return fail(st, "level %d (n = %d): %s", l, H->ln[l], inner);
    }
  }
  return orc_dense_factor(H->ln[H->L - 1], lambda, &H->coarse);
}

static void hier_free(hier* H) { orc_dense_free(&H->coarse); }

static int cycle_on_level(const hier* H, int l, orc_cplx* u, const orc_cplx* b) { /* :63-77 */
  const int n = H->ln[l];
  const long N = (long)(n - 1) * (n - 1);
  if (l + 1 == H->L) return orc_dense_solve(&H->coarse, b, u);
  const int nc = H->ln[l + 1];
  const long Nc = (long)(nc - 1) * (nc - 1);
  orc_cplx* tmp = (orc_cplx*)malloc(sizeof(orc_cplx) * (size_t)N);
  orc_cplx* rc = (orc_cplx*)calloc((size_t)Nc, sizeof(orc_cplx));
  orc_cplx* ec = (orc_cplx*)calloc((size_t)Nc, sizeof(orc_cplx));
  int st = ORC_OK;
  for (int k = 0; k < H->cfg.nu1; ++k) {
    if ((st = orc_apply_smoother(n, H->lambda, H->cfg.smoother, H->cfg.omega, u, b, tmp))) goto done;
    memcpy(u, tmp, sizeof(orc_cplx) * (size_t)N);
  }
  orc_residual(n, H->lambda, b, u, tmp);
  orc_restrict_fw(n, tmp, rc);
  const int gamma = H->cfg.cycle == ORC_CYCLE_W ? 2 : 1;
  for (int g = 0; g < gamma; ++g)
    if ((st = cycle_on_level(H, l + 1, ec, rc))) goto done;
  orc_prolong_bilinear(nc, ec, tmp);
  for (long k = 0; k < N; ++k) u[k] += tmp[k];
  for (int k = 0; k < H->cfg.nu2; ++k) {
    if ((st = orc_apply_smoother(n, H->lambda, H->cfg.smoother, H->cfg.omega, u, b, tmp))) goto done;
    memcpy(u, tmp, sizeof(orc_cplx) * (size_t)N);
  }
done:
  free(tmp);
  free(rc);
  free(ec);
  return st;
}

int orc_mg_cycle(int n, orc_cplx lambda, const orc_config* cfg, orc_cplx* u, const orc_cplx* b) {
  hier H;
  int st = hier_init(&H, n, lambda, cfg);
  if (!st) st = cycle_on_level(&H, 0, u, b);
  hier_free(&H);
  return st;
}

double orc_measured_rate(const double* hist, int iters) { /* multigrid.cpp:9-21 */
  if (iters <= 0) return 0.0;
  int count = iters - 1 < 5 ? iters - 1 : 5;
  if (count == 0) count = 1;
  double log_sum = 0.0;
  for (int k = iters - count + 1; k <= iters; ++k) {
    if (hist[k] == 0.0) return 0.0;
    if (hist[k - 1] == 0.0) return 0.0;
    log_sum += log(hist[k] / hist[k - 1]);
  }
  return exp(log_sum / count);
}

static int solve_h(const hier* H, const orc_cplx* b, orc_cplx* u, double* hist, int* iters, int* conv,
                   double* rate) { /* multigrid.cpp:85-110 */
  const int n = H->ln[0];
  const long N = (long)(n - 1) * (n - 1);
  memset(u, 0, sizeof(orc_cplx) * (size_t)N);
  const double r0 = orc_norm(n, b);
  hist[0] = r0;
  *iters = 0;
  *conv = 0;
  int st = ORC_OK;
  if (r0 == 0.0 || H->cfg.tol >= 1.0) {
    *conv = 1;
  } else {
    orc_cplx* r = (orc_cplx*)malloc(sizeof(orc_cplx) * (size_t)N);
    for (int k = 1; k <= H->cfg.max_iter; ++k) {
      if ((st = cycle_on_level(H, 0, u, b))) break;
      orc_residual(n, H->lambda, b, u, r);
      const double rk = orc_norm(n, r);
      hist[k] = rk;
      *iters = k;
      if (rk <= H->cfg.tol * r0) {
        *conv = 1;
        break;
      }
    }
    free(r);
  }
  *rate = orc_measured_rate(hist, *iters);
  return st;
}

int orc_mg_solve(int n, orc_cplx lambda, const orc_config* cfg, const orc_cplx* b, orc_cplx* u, double* hist,
                 int* iterations, int* converged, double* rate) {
  hier H;
  int st = hier_init(&H, n, lambda, cfg);
  if (!st) st = solve_h(&H, b, u, hist, iterations, converged, rate);
  hier_free(&H);
  return st;
}

/* Thread pool over contiguous shift chunks: paradiag.cpp:217-236. */
typedef struct {
  int n, b0, b1;
  const orc_cplx* lambdas;
  const orc_config* cfg;
  const orc_cplx *b;
  orc_cplx* u;
  double *hist, *rates;
  int *iters, *conv;
  int status;
  char err[512];
} chunk_job;

static void* run_chunk(void* p) {
  chunk_job* J = (chunk_job*)p;
  const long N = (long)(J->n - 1) * (J->n - 1);
  const int H = J->cfg->max_iter + 1;
  J->status = ORC_OK;
  for (int s = J->b0; s < J->b1; ++s) {
    const int st = orc_mg_solve(J->n, J->lambdas[s], J->cfg, J->b + (size_t)s * N, J->u + (size_t)s * N,
                                J->hist + (size_t)s * H, J->iters + s, J->conv + s, J->rates + s);
    if (st) {
      J->status = st;
      snprintf(J->err, sizeof J->err, "%s", g_err);
      break;
    }
  }
  return NULL;
}

int orc_mg_solve_batch(int n, int count, const orc_cplx* lambdas, const orc_config* cfg, const orc_cplx* b,
                       orc_cplx* u, double* hist, int* iters, int* conv, double* rates, int threads) {
  if (threads < 1) return fail(ORC_CONFIG, "paradiag_solve: threads must be >= 1");
  const int nw = threads < count ? threads : count;
  if (nw <= 0) return ORC_OK;
  const int chunk = (count + nw - 1) / nw;
  chunk_job* jobs = (chunk_job*)calloc((size_t)nw, sizeof(chunk_job));
  pthread_t* th = (pthread_t*)calloc((size_t)nw, sizeof(pthread_t));
  for (int t = 0; t < nw; ++t) {
    chunk_job* J = &jobs[t];
    J->n = n;
    J->b0 = t * chunk < count ? t * chunk : count;
    J->b1 = J->b0 + chunk < count ? J->b0 + chunk : count;
    J->lambdas = lambdas;
    J->cfg = cfg;
    J->b = b;
    J->u = u;
    J->hist = hist;
    J->rates = rates;
    J->iters = iters;
    J->conv = conv;
    if (nw == 1)
      run_chunk(J);
    else
      pthread_create(&th[t], NULL, run_chunk, J);
  }
  if (nw > 1)
    for (int t = 0; t < nw; ++t) pthread_join(th[t], NULL);
  int st = ORC_OK;
  for (int t = 0; t < nw && !st; ++t)
    if (jobs[t].status) st = fail(jobs[t].status, "%s", jobs[t].err);
  free(jobs);
  free(th);
  return st;
}

/* ------------------------------------------------------------------------------------------ */
/* ParaDIAG with the alpha-circulant time matrix (restated; the reference only has the alpha<0  */
/* closed form, paradiag.cpp:84-108, and the three-step driver, paradiag.cpp:185-248).          */
/* ------------------------------------------------------------------------------------------ */
double orc_all_at_once_residual_norm(int n, int nt, double alpha, double dt, const orc_cplx* u, const orc_cplx* f) {
  const long N = (long)(n - 1) * (n - 1);
  orc_cplx* y = (orc_cplx*)malloc(sizeof(orc_cplx) * (size_t)N);
  double s = 0.0;
  for (int t = 0; t < nt; ++t) { /* all_at_once_apply (paradiag.cpp:141-161), B = C_alpha */
    orc_apply_shifted_laplacian(n, 0.0, u + (size_t)t * N, y);
    /* nonzeros of row t in ascending column order */
    int cols[2];
    double vals[2];
    int nnz = 0;
    if (t == 0) {
      cols[nnz] = 0, vals[nnz++] = 1.0 / dt;
      if (nt - 1 > 0) cols[nnz] = nt - 1, vals[nnz++] = -alpha / dt;
    } else {
      cols[nnz] = t - 1, vals[nnz++] = -1.0 / dt;
      cols[nnz] = t, vals[nnz++] = 1.0 / dt;
    }
    for (int q = 0; q < nnz; ++q) {
      const orc_cplx w = vals[q];
      const orc_cplx* uj = u + (size_t)cols[q] * N;
      for (long k = 0; k < N; ++k) y[k] += w * uj[k];
    }
    double ss = 0.0;
    for (long k = 0; k < N; ++k) {
      const orc_cplx r = f[(size_t)t * N + k] - y[k];
      ss += creal(r) * creal(r) + cimag(r) * cimag(r);
    }
    const double nr = sqrt(ss);
    s += nr * nr;
  }
  free(y);
  return sqrt(s);
}

int orc_paradiag_circulant(int n, int nt, double alpha, double dt, const orc_config* cfg, const orc_cplx* f,
                           orc_cplx* u, int* iters, int* conv, double* relres, int threads) {
  if (nt < 2) return fail(ORC_CONFIG, "TimeDiscretization: need n >= 2 time steps");
  if (!(dt > 0.0)) return fail(ORC_CONFIG, "TimeDiscretization: tau must be positive");
  if (!(alpha != 0.0) || alpha != alpha) return fail(ORC_CONFIG, "alpha-circulant: alpha must be nonzero");
  const long N = (long)(n - 1) * (n - 1);
  orc_cplx* tw = (orc_cplx*)malloc(sizeof(orc_cplx) * (size_t)nt);
  for (int q = 0; q < nt; ++q) tw[q] = cexp(_Complex_I * (2.0 * M_PI * (double)q / (double)nt));
  orc_cplx* g = (orc_cplx*)calloc((size_t)nt * N, sizeof(orc_cplx));
  orc_cplx* w = (orc_cplx*)calloc((size_t)nt * N, sizeof(orc_cplx));
  orc_cplx* sc = (orc_cplx*)malloc(sizeof(orc_cplx) * (size_t)nt);
  for (int t = 0; t < nt; ++t) sc[t] = real_pow_c(alpha, (double)t / nt);
  /* step 1: g_k = (1/nt) sum_t alpha^(t/nt) f_t e^{+2 pi i t k / nt} */
  for (int k = 0; k < nt; ++k) {
    orc_cplx* gk = g + (size_t)k * N;
    for (int t = 0; t < nt; ++t) {
      const orc_cplx c = sc[t] * tw[(long)t * k % nt];
      const orc_cplx* ft = f + (size_t)t * N;
      for (long p = 0; p < N; ++p) gk[p] += c * ft[p];
    }
    for (long p = 0; p < N; ++p) gk[p] *= 1.0 / nt;
  }
  /* step 2: shifted solves */
  orc_cplx* lam = (orc_cplx*)malloc(sizeof(orc_cplx) * (size_t)nt);
  orc_circulant_shifts(alpha, nt, dt, 0, nt, (double*)lam);
  double* hist = (double*)malloc(sizeof(double) * (size_t)nt * (cfg->max_iter + 1));
  double* rates = (double*)malloc(sizeof(double) * (size_t)nt);
  int st = orc_mg_solve_batch(n, nt, lam, cfg, g, w, hist, iters, conv, rates, threads);
  if (!st) {
    /* step 3: u_t = alpha^(-t/nt) sum_k w_k e^{-2 pi i t k / nt} */
    for (int t = 0; t < nt; ++t) {
      orc_cplx* ut = u + (size_t)t * N;
      memset(ut, 0, sizeof(orc_cplx) * (size_t)N);
      for (int k = 0; k < nt; ++k) {
        const orc_cplx c = conj(tw[(long)t * k % nt]);
        const orc_cplx* wk = w + (size_t)k * N;
        for (long p = 0; p < N; ++p) ut[p] += c * wk[p];
      }
      const orc_cplx s = (orc_cplx)1.0 / sc[t];
      for (long p = 0; p < N; ++p) ut[p] *= s;
    }
    double fn = 0.0;
    for (int t = 0; t < nt; ++t) {
      const double q = orc_norm(n, f + (size_t)t * N);
      fn += q * q;
    }
    fn = sqrt(fn);
    const double rn = orc_all_at_once_residual_norm(n, nt, alpha, dt, u, f);
    *relres = fn > 0.0 ? rn / fn : rn;
  }
  free(tw), free(g), free(w), free(sc), free(lam), free(hist), free(rates);
  return st;
}
