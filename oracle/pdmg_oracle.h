/*
 * pdmg_oracle.h -- CPU restatement of the reference solver path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity oracle for the B200 implementation.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it, and only as the checker or
 * the CPU baseline -- never as the product path.  The product (paper_2203_11154_b200) fails
 * loudly when its CUDA library is missing; it never falls back to this file.
 *
 * Every function restates the reference (He & Liu, arXiv 2203.11154; artifact `pdmg`) in plain C99
 * with the same floating-point operation order, so its outputs are bit-identical to the
 * reference's own grid.cpp / smoother.cpp compiled under oracle/_ref (checked in
 * tests/test_oracle.py against tests/golden/, which were produced by that build).
 *
 * Layout (reference proj/include/pdmg/grid.hpp:54-91): interior nodes only, m = n-1 per side,
 * row-major with x fastest; node (i,j), 1 <= i,j <= m, lives at index (j-1)*m + (i-1).
 */
#ifndef PDMG_ORACLE_H
#define PDMG_ORACLE_H

#include <complex.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double _Complex orc_cplx;

enum { ORC_OK = 0, ORC_CONFIG = 1, ORC_SINGULAR = 2 };
enum { ORC_CYCLE_V = 0, ORC_CYCLE_W = 1 };
enum { ORC_VANKA = 0, ORC_JACOBI = 1 };

/* MultigridConfig, proj/include/pdmg/multigrid.hpp:14-32 (smoother fields from smoother.hpp:30-38). */
typedef struct {
  int cycle, nu1, nu2, coarsest_n, max_iter, smoother;
  double tol, omega;
} orc_config;

/* Last error message (thread-local). */
const char* orc_last_error(void);

/* ---- inputs: tools/pdmg.cpp:137-147 (random_rhs), tests/support/helpers.hpp:16-28 ---- */
/* Fills `count` complex values from std::mt19937(seed) + uniform_real_distribution<double>(lo,hi),
 * drawing re then im.  Restates libstdc++'s generate_canonical<double,53> over mt19937. */
void orc_random_complex(uint32_t seed, double lo, double hi, int64_t count, double* out_re_im);
/* Real draws (one per value), same engine/distribution. */
void orc_random_real(uint32_t seed, double lo, double hi, int64_t count, double* out);
/* BASELINE.json shift family lambda_j = (1 - alpha^(1/nt) e^(2 pi i j/nt))/dt, j = j0 .. j0+count-1. */
void orc_circulant_shifts(double alpha, int nt, double dt, int j0, int count, double* out_re_im);

/* ---- core grid (proj/src/grid.cpp) ---- */
double orc_norm(int n, const orc_cplx* v);                                                  /* :7-11 */
void orc_apply_stencil(int n, const orc_cplx w[9], double scale, const orc_cplx* u, orc_cplx* out); /* :30-58 */
void orc_apply_shifted_laplacian(int n, orc_cplx lambda, const orc_cplx* u, orc_cplx* out); /* :69-90 */
void orc_residual(int n, orc_cplx lambda, const orc_cplx* b, const orc_cplx* u, orc_cplx* r); /* :92-100 */
void orc_restrict_fw(int n_fine, const orc_cplx* fine, orc_cplx* coarse);                   /* :102-121 */
void orc_prolong_bilinear(int n_coarse, const orc_cplx* coarse, orc_cplx* fine);           /* :123-153 */

/* ---- smoothers (proj/src/smoother.cpp) ---- */
int orc_vanka_coeffs(orc_cplx eta, orc_cplx* a, orc_cplx* b, orc_cplx* c);               /* :18-29 */
int orc_vanka_stencil(orc_cplx lambda, double h, orc_cplx w[9], double* scale);          /* :31-40 */
int orc_jacobi_weight(orc_cplx eta, double h, orc_cplx* w);                               /* :42-47 */
int orc_apply_smoother(int n, orc_cplx lambda, int kind, double omega, const orc_cplx* u,
                       const orc_cplx* b, orc_cplx* out);                                  /* :49-67 */

/* ---- dense coarse solver (proj/src/dense.cpp:18-39, 82-100) without Eigen ---- */
typedef struct {
  int N;
  orc_cplx* lu; /* N*N row-major, L unit-lower + U */
  int* piv;
  int singular;
} orc_dense;
int orc_dense_factor(int n, orc_cplx lambda, orc_dense* d);
int orc_dense_solve(const orc_dense* d, const orc_cplx* b, orc_cplx* x);
void orc_dense_free(orc_dense* d);
/* Dense A + lambda I (N x N row-major) and dense patch-sum Vanka M (dense.cpp:56-80). */
int orc_dense_operator(int n, orc_cplx lambda, orc_cplx* A);
int orc_dense_vanka(int n, orc_cplx lambda, orc_cplx* M);

/* ---- multigrid (proj/src/multigrid.cpp) ---- */
int orc_mg_levels(int n, const orc_config* cfg, int* levels_n /* >= 32 */);
/* One cycle in place (multigrid.cpp:63-83). */
int orc_mg_cycle(int n, orc_cplx lambda, const orc_config* cfg, orc_cplx* u, const orc_cplx* b);
/* Full solve from u = 0 (multigrid.cpp:85-110).  hist has room for max_iter+1 entries. */
int orc_mg_solve(int n, orc_cplx lambda, const orc_config* cfg, const orc_cplx* b, orc_cplx* u,
                 double* hist, int* iterations, int* converged, double* rate);
double orc_measured_rate(const double* hist, int iterations); /* multigrid.cpp:9-21 */

/* Batch over shifts with a thread pool of contiguous chunks (paradiag.cpp:217-236).
 * b, u: count * m*m complex each (shift-major).  hist: count * (max_iter+1). */
int orc_mg_solve_batch(int n, int count, const orc_cplx* lambdas, const orc_config* cfg,
                       const orc_cplx* b, orc_cplx* u, double* hist, int* iterations,
                       int* converged, double* rates, int threads);

/* ---- ParaDIAG with the alpha-circulant time matrix (restated) ----
 * C_alpha = (1/dt)(I - Sigma_alpha), Sigma_alpha = down-shift with corner alpha at (0, nt-1).  alpha > 0 is
 * the BASELINE circulant preconditioner; alpha = -1/beta < 0 is the reference's BackwardHeatQBV matrix
 * (paradiag.cpp:180-188), diagonalized with the principal root |alpha|^(1/nt) e^(i pi/nt) (paradiag.cpp:209-213).
 * Solves (C_alpha (x) I + I (x) A) U = F: g = ifft_t(alpha^(t/nt) f), nt shifted MG solves,
 * U = alpha^(-t/nt) fft_k(w).  f, u: nt * m*m complex (time-major). */
int orc_paradiag_circulant(int n, int nt, double alpha, double dt, const orc_config* cfg,
                           const orc_cplx* f, orc_cplx* u, int* iterations, int* converged,
                           double* relres, int threads);
/* r = F - (C_alpha (x) I + I (x) A) U, returns ||r|| (paradiag.cpp:141-183 with B = C_alpha). */
double orc_all_at_once_residual_norm(int n, int nt, double alpha, double dt, const orc_cplx* u,
                                     const orc_cplx* f);

#ifdef __cplusplus
}
#endif
#endif
