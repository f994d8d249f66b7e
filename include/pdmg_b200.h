/*
 * pdmg_b200.h -- C ABI of the B200-native batched shifted-Laplacian multigrid (libpdmg_b200.so).
 *
 * Drop-in boundary for the reference `pdmg` solver path (He & Liu, arXiv 2203.11154).  The reference
 * exposes this path as C++ in namespace pdmg, linked statically (proj/src/CMakeLists.txt:1-12); it has
 * no FFI.  Each entry point below replaces the reference interface cited beside it; the C++ facade
 * include/pdmg_b200.hpp restores the reference's class shapes and exception types on top of it.
 *
 * Conventions
 *  - Plain C types only.  pdmg_c128 is layout-compatible with std::complex<double> and double2.
 *  - Host grid arrays use the reference layout (proj/include/pdmg/grid.hpp:54-91): per shift, the
 *    (n-1)x(n-1) interior nodes, row-major with x fastest; shifts are stacked shift-major.
 *  - Status codes mirror proj/include/pdmg/errors.hpp:10-28: 0 OK, 1 ConfigError, 2
 *    SingularOperatorError, 3 runtime (CUDA) error.  pdmg_last_error() returns the message of the
 *    last failing call on the calling thread (same text as the reference's exception what()).
 *  - Non-convergence is data (converged[] = 0), never an error (proj/src/multigrid.cpp:93-106).
 *  - Every solve runs on the GPU; there is no CPU fallback.  A missing/unusable GPU is status 3.
 */
#ifndef PDMG_B200_H
#define PDMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDMG_B200_ABI_VERSION 2

typedef struct {
  double re, im;
} pdmg_c128;

enum {
  PDMG_OK = 0,
  PDMG_ERR_CONFIG = 1,   /* pdmg::ConfigError           (errors.hpp:12-15) */
  PDMG_ERR_SINGULAR = 2, /* pdmg::SingularOperatorError (errors.hpp:20-23) */
  PDMG_ERR_RUNTIME = 3   /* CUDA / device failure                          */
};
enum { PDMG_CYCLE_V = 0, PDMG_CYCLE_W = 1 };              /* pdmg::CycleKind    (multigrid.hpp:12) */
enum { PDMG_SMOOTHER_VANKA = 0, PDMG_SMOOTHER_JACOBI = 1 }; /* pdmg::SmootherKind (smoother.hpp:28) */
enum { PDMG_PREC_C128 = 0, PDMG_PREC_C64 = 1 };

/* pdmg::MultigridConfig (proj/include/pdmg/multigrid.hpp:14-32) with its SmootherConfig
 * (proj/include/pdmg/smoother.hpp:30-38) flattened in. */
typedef struct {
  int32_t cycle;      /* PDMG_CYCLE_V / PDMG_CYCLE_W                 */
  int32_t nu1, nu2;   /* pre / post smoothing sweeps                 */
  int32_t coarsest_n; /* coarsest level mesh width 1/coarsest_n      */
  double tol;         /* relative residual reduction target          */
  int32_t max_iter;
  int32_t smoother;   /* PDMG_SMOOTHER_VANKA / PDMG_SMOOTHER_JACOBI  */
  double omega;       /* real relaxation weight (smoother.hpp:34)    */
} pdmg_mg_config;

/* Reference defaults: W(1,0), coarsest_n 8, tol 1e-8, max_iter 200, Vanka omega 24/25
 * (multigrid.hpp:14-23, smoother.hpp:32-36). */
void pdmg_mg_config_default(pdmg_mg_config* cfg);

/* A batch of hierarchies sharing one fine grid and config, one per shift.  Replaces constructing one
 * pdmg::MultigridHierarchy(Grid2D(n), Shift{lambda_j}, cfg) per shift (multigrid.hpp:52,
 * multigrid.cpp:24-61) inside paradiag_solve's loop (paradiag.cpp:207-236). */
typedef struct {
  int32_t n;                /* Grid2D.n of the finest grid (h = 1/n)       */
  int32_t n_shifts;         /* >= 1                                        */
  const pdmg_c128* lambdas; /* host [n_shifts]: Shift.lambda (grid.hpp:44) */
  pdmg_mg_config cfg;
  int32_t precision;        /* PDMG_PREC_C128 (the reference's type)       */
  int32_t device;           /* CUDA device ordinal (when n_devices == 0)   */
  /* Optional device list: the reference's `threads` argument of paradiag_solve (paradiag.cpp:207-236) becomes a
   * list of devices.  Shard p = shifts [p*chunk, min(S, (p+1)*chunk)), chunk = ceil(S / n_devices), runs on
   * devices[p] in its own engine; every call runs the shards concurrently (one host thread each).  A device may
   * repeat.  NULL / 0: a single engine on `device`. */
  const int32_t* devices;
  int32_t n_devices;
} pdmg_batch_desc;

typedef struct pdmg_ctx pdmg_ctx;

/* Per-shift outputs of MultigridHierarchy::solve (pdmg::SolveReport, multigrid.hpp:34-44).  Any pointer
 * may be NULL.  residual_history is [n_shifts][max_iter+1]; entries past iterations[s] are 0. */
typedef struct {
  int32_t* iterations;
  uint8_t* converged;
  double* residual_history;
  double* rate;
  double seconds; /* wall time of the call (SolveReport.seconds) */
} pdmg_solve_report;

const char* pdmg_last_error(void);
int pdmg_abi_version(void);

/* Builds the hierarchy for every shift: validates cfg (multigrid.hpp:25-31), the level list
 * (multigrid.cpp:27-44), the smoother on every non-coarsest level (multigrid.cpp:47-58, throws
 * "level l (n = N): ..."), factors each coarsest operator (dense.cpp:82-88) and allocates device
 * storage.  Config and singular-smoother errors are reported before any CUDA call. */
int pdmg_create(const pdmg_batch_desc* desc, pdmg_ctx** out);
void pdmg_destroy(pdmg_ctx* ctx);
int pdmg_num_levels(const pdmg_ctx* ctx);           /* MultigridHierarchy::num_levels */
int pdmg_level_n(const pdmg_ctx* ctx, int level);   /* level_grid(level).n             */
int pdmg_num_shifts(const pdmg_ctx* ctx);
/* 1 if shift s's coarsest operator is singular (DenseShiftedSolver::singular, dense.hpp:40). */
int pdmg_coarse_singular(const pdmg_ctx* ctx, int shift);

/* MultigridHierarchy::solve for all shifts from u = 0 (multigrid.cpp:85-110): b, u host arrays of
 * n_shifts*(n-1)^2.  A singular coarsest operator fails with status 2 (dense.cpp:90-94). */
int pdmg_solve(pdmg_ctx* ctx, const pdmg_c128* b, pdmg_c128* u, pdmg_solve_report* report);
/* Same with b, u already resident in device memory of ctx's device (compact layout as above). */
int pdmg_solve_device(pdmg_ctx* ctx, const void* d_b, void* d_u, pdmg_solve_report* report);

/* Device-resident solve of a context sharded over devices: d_b[p], d_u[p] hold shard p's shifts (compact layout) in
 * the memory of shard p's device (pdmg_part_range).  For a single-device context this is pdmg_solve_device. */
int pdmg_solve_device_shards(pdmg_ctx* ctx, const void* const* d_b, void* const* d_u, pdmg_solve_report* report);
int pdmg_num_parts(const pdmg_ctx* ctx);
/* Shard `part`: its first shift, shift count and device. */
int pdmg_part_range(const pdmg_ctx* ctx, int part, int32_t* shift0, int32_t* count, int32_t* device);

/* MultigridHierarchy::cycle: one cycle applied in place to every shift's u (multigrid.cpp:79-83). */
int pdmg_cycle(pdmg_ctx* ctx, pdmg_c128* u, const pdmg_c128* b);

/* Level operators, batched over all shifts of ctx at hierarchy level `level` (0 = finest).  They use
 * ctx's level buffers as scratch.  Host arrays are n_shifts * (level_n-1)^2. */
int pdmg_apply_smoother(pdmg_ctx* ctx, int level, const pdmg_c128* u, const pdmg_c128* b,
                        pdmg_c128* out);                                   /* smoother.cpp:49-67 */
int pdmg_residual(pdmg_ctx* ctx, int level, const pdmg_c128* b, const pdmg_c128* u,
                  pdmg_c128* r);                                           /* grid.cpp:92-100    */
int pdmg_restrict_full_weighting(pdmg_ctx* ctx, int level, const pdmg_c128* fine,
                                 pdmg_c128* coarse);                       /* grid.cpp:102-121   */
int pdmg_prolong_bilinear(pdmg_ctx* ctx, int level, const pdmg_c128* coarse,
                          pdmg_c128* fine);                                /* grid.cpp:123-153   */
int pdmg_norm(pdmg_ctx* ctx, int level, const pdmg_c128* v, double* norms); /* grid.cpp:7-11    */
int pdmg_coarse_solve(pdmg_ctx* ctx, const pdmg_c128* b, pdmg_c128* u);      /* dense.cpp:90-100 */

/* ParaDIAG with the alpha-circulant backward-Euler time matrix C_alpha = (1/dt)(I - Sigma_alpha), Sigma_alpha the
 * down-shift with corner alpha (restated; the reference's three-step driver is paradiag.cpp:185-248 and its
 * closed-form alpha-circulant diagonalization, for alpha < 0 only, paradiag.cpp:84-108):
 *   step 1  g = ifft_t(alpha^(t/nt) f)                                  (kron_time_solve, paradiag.cpp:135-139)
 *   step 2  (A + lambda_k I) w_k = g_k, lambda_k = (1 - alpha^(1/nt) e^(2 pi i k/nt))/dt  (paradiag.cpp:207-236)
 *   step 3  u = alpha^(-t/nt) fft_k(w)                                  (kron_time_apply, paradiag.cpp:129-133)
 *   relres  = ||f - (C_alpha (x) I + I (x) A) u|| / ||f||               (paradiag.cpp:243-245)
 * f, u: [nt][(n-1)^2] time slices in the reference layout.  report arrays are per time slot k. */
typedef struct pdmg_paradiag pdmg_paradiag;
int pdmg_paradiag_create(int32_t n, int32_t nt, double alpha, double dt, const pdmg_mg_config* cfg, int32_t device,
                         pdmg_paradiag** out);
/* The same with the time slices (and their shift slots) sharded over a device list -- the reference's `threads`
 * argument of paradiag_solve (paradiag.cpp:207-236): shard p holds slices [p*chunk, min(nt, (p+1)*chunk)),
 * chunk = ceil(nt / n_devices), on devices[p].  Both time transforms gather their time columns from every shard
 * and scatter the results to the owners through NVLink peer pointers inside the transform kernel (no separate
 * all-to-all); peer access between distinct devices is enabled at creation (status 3 if unavailable). */
int pdmg_paradiag_create_multi(int32_t n, int32_t nt, double alpha, double dt, const pdmg_mg_config* cfg,
                               const int32_t* devices, int32_t n_devices, pdmg_paradiag** out);
/* General diagonalizable time matrix (HeatBVM: diagonalize_time_matrix, paradiag.cpp:71-82): B = V diag(lambdas)
 * V^{-1} supplied by the caller (host, nt x nt row-major; B real).  The time transforms g = (V^{-1} (x) I) f and
 * u = (V (x) I) w are hand-written complex fp64 GEMM kernels over the time index (k_time_gemm), sharded like the
 * circulant scheme; relres = ||f - (B (x) I + I (x) A) u|| / ||f||. */
int pdmg_paradiag_create_general(int32_t n, int32_t nt, const pdmg_c128* lambdas, const pdmg_c128* V,
                                 const pdmg_c128* Vinv, const double* B, const pdmg_mg_config* cfg,
                                 const int32_t* devices, int32_t n_devices, pdmg_paradiag** out);
int pdmg_paradiag_num_parts(const pdmg_paradiag* p);
/* Shard `part`: first time slice, slice count, device. */
int pdmg_paradiag_part_range(const pdmg_paradiag* p, int part, int32_t* t0, int32_t* count, int32_t* device);
/* Rank mode: one process per GPU (torchrun).  This process owns time slices [rank*chunk, ...) of `nranks` contiguous
 * chunks on `device`; the other ranks' slice buffers are opened from their CUDA IPC handles, so the transform kernels
 * gather / scatter across processes through NVLink peer memory -- the all-to-all stays inside the transforms.
 *   pdmg_paradiag_ipc_handles(p, h)      h: 4 x 64 bytes (cudaIpcMemHandle_t of f, g, w, u)
 *   pdmg_paradiag_open_peers(p, all)     all: [nranks][4 x 64 bytes], every rank's handles (own entry ignored)
 *   pdmg_paradiag_rank_buffer(p, which)  this rank's device buffers: 0 = f (input slices), 3 = u (output slices)
 *   pdmg_paradiag_rank_phase(p, k, ...)  k = 1 step-1 transform, 2 shifted solves (report: this rank's slots at
 *                                        their global indices), 3 step-3 transform, 4 residual sums
 *                                        {||r||^2, ||f||^2} of this rank's slices; the caller barriers all ranks
 *                                        between phases (each returns once its GPU work is complete). */
int pdmg_paradiag_create_rank(int32_t n, int32_t nt, double alpha, double dt, const pdmg_mg_config* cfg, int32_t rank,
                              int32_t nranks, int32_t device, pdmg_paradiag** out);
int pdmg_paradiag_ipc_handles(pdmg_paradiag* p, void* handles);
int pdmg_paradiag_open_peers(pdmg_paradiag* p, const void* all_handles);
int pdmg_paradiag_rank_phase(pdmg_paradiag* p, int32_t phase, pdmg_solve_report* report, double* sums);
void* pdmg_paradiag_rank_buffer(pdmg_paradiag* p, int32_t which);
/* Device-resident run of a sharded solver: d_f[p], d_u[p] = shard p's slices in its device's memory. */
int pdmg_paradiag_run_shards(pdmg_paradiag* p, const void* const* d_f, void* const* d_u, pdmg_solve_report* report,
                             double* relres);
void pdmg_paradiag_destroy(pdmg_paradiag* p);
pdmg_ctx* pdmg_paradiag_solver(pdmg_paradiag* p); /* shard 0's batched solver (stats, levels, stream) */
int pdmg_paradiag_run(pdmg_paradiag* p, const pdmg_c128* f, pdmg_c128* u, pdmg_solve_report* report,
                      double* relres);
int pdmg_paradiag_run_device(pdmg_paradiag* p, const void* d_f, void* d_u, pdmg_solve_report* report,
                             double* relres);
/* One-shot convenience (paradiag_solve, paradiag.hpp:112-113). */
int pdmg_paradiag_circulant(int32_t n, int32_t nt, double alpha, double dt, const pdmg_mg_config* cfg,
                            int32_t device, const pdmg_c128* f, pdmg_c128* u, pdmg_solve_report* report,
                            double* relres);
/* One-shot general-scheme solve on one device (pdmg_paradiag_create_general + run + destroy). */
int pdmg_paradiag_general(int32_t n, int32_t nt, const pdmg_c128* lambdas, const pdmg_c128* V, const pdmg_c128* Vinv,
                          const double* B, const pdmg_mg_config* cfg, int32_t device, const pdmg_c128* f,
                          pdmg_c128* u, pdmg_solve_report* report, double* relres);
/* Y = (M (x) I) X for device arrays [nt][npts] (kron_time_apply, paradiag.cpp:129-133); M host nt x nt. */
int pdmg_time_transform(int32_t device, int32_t nt, int64_t npts, const pdmg_c128* M, const void* d_in, void* d_out,
                        void* stream);
/* Building blocks of the multi-GPU driver (time slices sharded over ranks, NCCL all-to-all between):
 * alpha-scaled DFT over the full time axis of npts points laid out [nt][npts] (step 1 or 3 above), and
 * the all-at-once residual of local slices [t0, t0+ntl) given the slice before t0 (u_{nt-1} if t0 == 0):
 * sums = {||r||^2, ||f||^2} over the local slices.  stream: a cudaStream_t (NULL = default stream). */
int pdmg_time_dft(int32_t device, int32_t nt, int64_t npts, double alpha, int32_t step, const void* d_in,
                  void* d_out, void* stream);
int pdmg_aao_residual(int32_t device, int32_t n, int32_t ntl, int32_t t0, double alpha, double dt, const void* d_u,
                      const void* d_u_prev, const void* d_f, double* sums, void* stream);

/* ---- Local Fourier analysis (proj/include/pdmg/lfa.hpp, proj/src/lfa.cpp) ----------------------------------------
 * Symbols of the shifted operator, the Vanka / Jacobi preconditioner, the smoother error and the transfer operators;
 * smoothing factors over the sampled high-frequency region (first maximizer in the reference's sampling order);
 * the shift-splitting bound; the two-grid model rho(omega, nu); the damping optimization (coarse scan of
 * [0.1, 1.9] by 0.01, golden-section refinement to 1e-4).  The per-frequency work runs on `device`: one thread per
 * (omega, base frequency) for the 4 x 4 two-grid spectral radii. */
typedef struct {
  int32_t samples_per_dim; /* even, >= 16 (LFAConfig, lfa.hpp:21-31)          */
  double coarse_skip_tol;  /* two-grid bases with |coarse symbol| <= this skipped */
} pdmg_lfa_config;
enum { PDMG_LFA_OPERATOR = 0, PDMG_LFA_VANKA = 1, PDMG_LFA_PRECONDITIONER = 2, PDMG_LFA_SMOOTHER_ERROR = 3,
       PDMG_LFA_TRANSFER = 4 };
enum { PDMG_LFA_TWO_GRID_RHO = 0, PDMG_LFA_SMOOTHING_MU = 1 }; /* OmegaObjective (lfa.hpp:100-103) */
void pdmg_lfa_config_default(pdmg_lfa_config* cfg); /* {64, 1e-8} */
/* symbol_shifted_laplacian / symbol_vanka / symbol_preconditioner / symbol_smoother_error / symbol_transfer
 * (lfa.hpp:33-53) at (t1, t2) for Shift{lambda} on mesh width h; `smoother` and `omega` where they apply. */
int pdmg_lfa_symbol(int32_t which, double t1, double t2, pdmg_c128 lambda, double h, int32_t smoother, double omega,
                    pdmg_c128* out);
/* smoothing_factor (lfa.hpp:62-63): mu and its first sampled maximizer argmax[2] (may be NULL). */
int pdmg_lfa_smoothing_factor(pdmg_c128 lambda, double h, int32_t smoother, double omega, const pdmg_lfa_config* lfa,
                              int32_t device, double* mu, double* argmax);
/* smoothing_factor_bound (lfa.hpp:69-75): phi[0] = phi_base, phi[1] = phi_shift (Vanka). */
int pdmg_lfa_smoothing_bound(pdmg_c128 lambda, double h, double omega, const pdmg_lfa_config* lfa, int32_t device,
                             double* phi);
/* TwoGridModel (lfa.hpp:77-96), symbol caches in device memory. */
typedef struct pdmg_lfa_model pdmg_lfa_model;
int pdmg_lfa_model_create(pdmg_c128 lambda, double h, int32_t smoother, const pdmg_lfa_config* lfa, int32_t device,
                          pdmg_lfa_model** out);
void pdmg_lfa_model_destroy(pdmg_lfa_model* model);
int pdmg_lfa_model_skipped(const pdmg_lfa_model* model);
/* rho[k] = TwoGridModel::rho(omegas[k], nu) for k < count (one launch for the whole batch). */
int pdmg_lfa_model_rho(pdmg_lfa_model* model, int32_t count, const double* omegas, int32_t nu, double* rho);
/* TwoGridModel::smoothing(omega): mu and argmax[2] (may be NULL). */
int pdmg_lfa_model_smoothing(pdmg_lfa_model* model, double omega, double* mu, double* argmax);
/* optimize_omega(model, objective, nu) (lfa.hpp:112-113). */
int pdmg_lfa_optimize_omega(pdmg_lfa_model* model, int32_t objective, int32_t nu, double* omega, double* value);
/* optimize_omega(shift, h, kind, SmoothingMu) without a two-grid model (lfa.cpp:231-246). */
int pdmg_lfa_optimize_omega_smoothing(pdmg_c128 lambda, double h, int32_t smoother, const pdmg_lfa_config* lfa,
                                      int32_t device, double* omega, double* value);

/* Host helpers (no GPU needed). */
/* tools/pdmg.cpp:137-147 random_rhs: std::mt19937(seed), uniform_real_distribution<double>(lo,hi),
 * re then im per node; `count` complex values. */
void pdmg_random_rhs(uint32_t seed, double lo, double hi, int64_t count, pdmg_c128* out);
/* lambda_j = (1 - alpha^(1/nt) e^(2 pi i j/nt))/dt for j = j0 .. j0+count-1 (BASELINE.json shifts). */
void pdmg_circulant_shifts(double alpha, int32_t nt, double dt, int32_t j0, int32_t count, pdmg_c128* out);
/* Pinned host memory for fast host<->device staging. */
void* pdmg_host_alloc(size_t bytes);
void pdmg_host_free(void* p);

/* Instrumentation.  When profiling is on, every kernel launch is bracketed by CUDA events on ctx's
 * stream and attributed to a kernel class; stats accumulate until reset. */
void* pdmg_stream(pdmg_ctx* ctx); /* the cudaStream_t all of ctx's work runs on */
/* Solve strategy: 0 auto (default), 1 batched level passes (one launch per fused operator and level,
 * over all shifts), 2 one CTA per shift running the whole solve loop in one launch (small grids). */
int pdmg_set_solve_path(pdmg_ctx* ctx, int path);
int pdmg_set_profiling(pdmg_ctx* ctx, int on);
void pdmg_reset_stats(pdmg_ctx* ctx);
int64_t pdmg_launch_count(const pdmg_ctx* ctx); /* kernels launched since the last reset */
/* Kernel class i: name, launches, total device ms, total algorithmic DRAM bytes.  Returns 0 while i is
 * valid, 1 past the end. */
int pdmg_kernel_stats(const pdmg_ctx* ctx, int i, char* name, size_t name_len, int64_t* launches,
                      double* total_ms, double* algo_bytes);
/* Kernel class i, SURVEY 8(d) accounting: unit_bytes = 48 B (c128; 24 B c64) per grid-point smoother update
 * the class performed plus its fused transfer bytes (the bytes moved, for passes without a smoother update),
 * and the number of smoother updates.  A fused two-sweep pass counts two updates per point while moving
 * the bytes of one (pdmg_kernel_stats).  Returns 0 while i is valid, 1 past the end. */
int pdmg_kernel_updates(const pdmg_ctx* ctx, int i, double* unit_bytes, double* updates);
/* Grid-point smoother updates performed by the last solve (sum over shifts and cycles). */
double pdmg_last_updates(const pdmg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* PDMG_B200_H */
