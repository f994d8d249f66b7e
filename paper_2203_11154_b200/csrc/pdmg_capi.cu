// pdmg_capi.cu -- host orchestration (C++) and the extern "C" boundary of libpdmg_b200.so.
//
// Mirrors the reference solver path (proj/src/multigrid.cpp, proj/src/paradiag.cpp) for a BATCH of
// shifts: one pdmg_ctx holds, for every shift, what one pdmg::MultigridHierarchy holds (level list,
// per-level smoother coefficients, coarsest factorization) plus device storage for all levels.  Every
// cycle is a short sequence of batched k_level launches (pdmg_kernels.cuh) over all still-active
// shifts; convergence is decided on the device per shift (k_finalize) exactly as in
// MultigridHierarchy::solve, so per-shift cycle counts match the reference.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pdmg_b200.h"
#include "pdmg_kernels.cuh"
#include "pdmg_march2ws.cuh"

using cplx = std::complex<double>;

namespace pdmg_b200 {

// ---------------------------------------------------------------------------------------------
// Error taxonomy (proj/include/pdmg/errors.hpp:10-28) carried through the C ABI as status codes.
// ---------------------------------------------------------------------------------------------
struct ConfigError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct SingularOperatorError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

thread_local std::string g_last_error;

#define CK(x)                                                                                        \
  do {                                                                                               \
    cudaError_t e_ = (x);                                                                            \
    if (e_ != cudaSuccess)                                                                           \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" +          \
                      std::to_string(__LINE__) + ")");                                               \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PDMG_OK;
  } catch (const ConfigError& e) {
    g_last_error = e.what();
    return PDMG_ERR_CONFIG;
  } catch (const SingularOperatorError& e) {
    g_last_error = e.what();
    return PDMG_ERR_SINGULAR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PDMG_ERR_RUNTIME;
  }
}

// ---------------------------------------------------------------------------------------------
// Host-side setup math (fp64), restating the reference formulas.
// ---------------------------------------------------------------------------------------------
constexpr double kSingularTol = 1e-12;  // smoother.cpp:6

cplx checked_inverse(cplx z, const char* what) {  // smoother.cpp:8-15
  if (std::abs(z) <= kSingularTol)
    throw SingularOperatorError(std::string("vanka_coeffs: patch eigenvalue ") + what + " is singular for this shift");
  return cplx(1.0, 0.0) / z;
}

struct Vanka {
  cplx a, b, c;
};
Vanka vanka_coeffs(cplx eta) {  // smoother.cpp:18-29
  const cplx i2 = checked_inverse(cplx(2.0, 0.0) + eta, "2+eta");
  const cplx i4 = checked_inverse(cplx(4.0, 0.0) + eta, "4+eta");
  const cplx i6 = checked_inverse(cplx(6.0, 0.0) + eta, "6+eta");
  return {0.25 * (i2 + 2.0 * i4 + i6), 0.25 * (i2 - i6), 0.25 * (i2 - 2.0 * i4 + i6)};
}
cplx jacobi_weight(cplx eta, double h) {  // smoother.cpp:42-47
  const cplx d = cplx(4.0, 0.0) + eta;
  if (std::abs(d) <= kSingularTol) throw SingularOperatorError("jacobi_weight: 4+eta is singular for this shift");
  return cplx(h * h, 0.0) / d;
}

// Dense A + lambda I on the coarsest grid (dense.cpp:18-39), partial-pivot LU with the reference's
// singularity rule min|U_ii| > 1e-14 ||A||_F (dense.cpp:82-88), then A^{-1} for the batched kernel.
struct CoarseFactor {
  bool singular = false;
  std::vector<cplx> inv;  // N x N row-major
};
CoarseFactor factor_coarse(int n, cplx lambda) {
  if (n > 128)
    throw ConfigError("dense_shifted_operator: dense assembly refused for n = " + std::to_string(n) + " (limit 128)");
  const int m = n - 1, N = m * m;
  const double h = 1.0 / n, inv_h2 = 1.0 / (h * h);
  const cplx diag = (cplx(4.0, 0.0) + lambda * (h * h)) * inv_h2, off(-inv_h2, 0.0);
  std::vector<cplx> A(static_cast<size_t>(N) * N, cplx(0.0, 0.0));
  auto idx = [m](int i, int j) { return (j - 1) * m + (i - 1); };
  for (int j = 1; j <= m; ++j)
    for (int i = 1; i <= m; ++i) {
      const int r = idx(i, j);
      A[(size_t)r * N + r] = diag;
      if (i > 1) A[(size_t)r * N + idx(i - 1, j)] = off;
      if (i < m) A[(size_t)r * N + idx(i + 1, j)] = off;
      if (j > 1) A[(size_t)r * N + idx(i, j - 1)] = off;
      if (j < m) A[(size_t)r * N + idx(i, j + 1)] = off;
    }
  double fro = 0.0;
  for (const cplx& z : A) fro += std::norm(z);
  fro = std::sqrt(fro);
  std::vector<int> piv(N);
  double min_pivot = INFINITY;
  for (int k = 0; k < N; ++k) {
    int p = k;
    double best = std::abs(A[(size_t)k * N + k]);
    for (int r = k + 1; r < N; ++r)
      if (std::abs(A[(size_t)r * N + k]) > best) best = std::abs(A[(size_t)r * N + k]), p = r;
    piv[k] = p;
    if (p != k)
      for (int c = 0; c < N; ++c) std::swap(A[(size_t)k * N + c], A[(size_t)p * N + c]);
    const cplx pv = A[(size_t)k * N + k];
    min_pivot = std::min(min_pivot, std::abs(pv));
    if (pv == cplx(0.0, 0.0)) continue;
    for (int r = k + 1; r < N; ++r) {
      const cplx f = A[(size_t)r * N + k] / pv;
      A[(size_t)r * N + k] = f;
      for (int c = k + 1; c < N; ++c) A[(size_t)r * N + c] -= f * A[(size_t)k * N + c];
    }
  }
  CoarseFactor cf;
  cf.singular = !(min_pivot > 1e-14 * fro);
  cf.inv.assign(static_cast<size_t>(N) * N, cplx(0.0, 0.0));
  if (cf.singular) return cf;
  std::vector<cplx> x(N);
  for (int col = 0; col < N; ++col) {
    std::fill(x.begin(), x.end(), cplx(0.0, 0.0));
    x[col] = 1.0;
    for (int k = 0; k < N; ++k)
      if (piv[k] != k) std::swap(x[k], x[piv[k]]);
    for (int r = 0; r < N; ++r)
      for (int c = 0; c < r; ++c) x[r] -= A[(size_t)r * N + c] * x[c];
    for (int r = N - 1; r >= 0; --r) {
      for (int c = r + 1; c < N; ++c) x[r] -= A[(size_t)r * N + c] * x[c];
      x[r] /= A[(size_t)r * N + r];
    }
    for (int r = 0; r < N; ++r) cf.inv[(size_t)r * N + col] = x[r];
  }
  return cf;
}

void validate(const pdmg_mg_config& c) {  // multigrid.hpp:25-31
  if (c.nu1 < 0 || c.nu2 < 0) throw ConfigError("MultigridConfig: negative smoothing counts");
  if (c.nu1 + c.nu2 == 0) throw ConfigError("MultigridConfig: nu1 + nu2 must be positive");
  if (c.coarsest_n < 2) throw ConfigError("MultigridConfig: coarsest_n must be >= 2");
  if (!(c.tol > 0.0)) throw ConfigError("MultigridConfig: tol must be positive");
  if (c.max_iter < 1) throw ConfigError("MultigridConfig: max_iter must be >= 1");
  if (c.cycle != PDMG_CYCLE_V && c.cycle != PDMG_CYCLE_W) throw ConfigError("MultigridConfig: unknown cycle kind");
  if (c.smoother != PDMG_SMOOTHER_VANKA && c.smoother != PDMG_SMOOTHER_JACOBI)
    throw ConfigError("SmootherConfig: unknown smoother kind");
}

std::vector<int> level_list(int n, const pdmg_mg_config& c) {  // multigrid.cpp:27-44
  if (n < 2) throw ConfigError("Grid2D: need at least 2 subdivisions per side, got " + std::to_string(n));
  validate(c);
  if (n < c.coarsest_n)
    throw ConfigError("MultigridHierarchy: fine grid n = " + std::to_string(n) + " is finer than coarsest_n = " +
                      std::to_string(c.coarsest_n) + " allows");
  std::vector<int> lv{n};
  int g = n;
  while (g > c.coarsest_n) {
    if (!(g % 2 == 0 && g >= 4))
      throw ConfigError("MultigridHierarchy: grid n = " + std::to_string(g) + " cannot be coarsened to reach coarsest_n = " +
                        std::to_string(c.coarsest_n));
    g /= 2;
    lv.push_back(g);
  }
  if (g != c.coarsest_n)
    throw ConfigError("MultigridHierarchy: coarsening from n = " + std::to_string(n) + " reaches n = " + std::to_string(g) +
                      ", not coarsest_n = " + std::to_string(c.coarsest_n));
  return lv;
}

// ---------------------------------------------------------------------------------------------
// Kernel variant table: flags -> instantiation of k_level.
// ---------------------------------------------------------------------------------------------
struct Variant {
  bool loadu, prolong, sweep;
  int post;
  bool store, jacobi;
  int key() const {
    return (loadu ? 1 : 0) | (prolong ? 2 : 0) | (sweep ? 4 : 0) | (post << 3) | (store ? 32 : 0) | (jacobi ? 64 : 0);
  }
  std::string name() const {
    std::string s;
    if (prolong) s += loadu ? "prolong+" : "prolong0+";
    else if (!loadu) s += "zero+";
    if (sweep) s += jacobi ? "jacobi" : "vanka";
    else if (!prolong) s += "pass";
    else s.pop_back();
    if (post == POST_NORM) s += "+norm";
    if (post == POST_RESTRICT) s += "+restrict";
    if (post == POST_RESID) s += "+resid";
    return s;
  }
};

template <class T>
struct KernelEntry {
  void (*fn)(LevelArgs<T>) = nullptr;
  size_t smem = 0;
};

template <class T>
struct KernelTable {
  KernelEntry<T> e[128];
  template <bool LU, bool PR, bool SW, int PO, bool ST, bool JA>
  void reg() {
    const int k = (LU ? 1 : 0) | (PR ? 2 : 0) | (SW ? 4 : 0) | (PO << 3) | (ST ? 32 : 0) | (JA ? 64 : 0);
    e[k].fn = &k_level<T, LU, PR, SW, PO, ST, JA>;
    e[k].smem = LevelShape<T, LU || PR, SW, PO, PR>::bytes;
  }
  template <bool LU, bool PR, int PO, bool JA>
  void reg_sweep() {
    reg<LU, PR, true, PO, true, JA>();
  }
  template <bool LU, bool PR, int PO>
  void reg_sweep2() {
    reg_sweep<LU, PR, PO, false>();
    reg_sweep<LU, PR, PO, true>();
  }
  template <int PO>
  void reg_sweep4() {
    reg_sweep2<false, false, PO>();
    reg_sweep2<true, false, PO>();
    reg_sweep2<false, true, PO>();
    reg_sweep2<true, true, PO>();
  }
  KernelTable() {
    reg_sweep4<POST_NONE>();
    reg_sweep4<POST_NORM>();
    // restriction follows pre-smoothing only, which never prolongates
    reg_sweep2<false, false, POST_RESTRICT>();
    reg_sweep2<true, false, POST_RESTRICT>();
    // prolongate-and-correct without a sweep (nu2 == 0)
    reg<false, true, false, POST_NONE, true, false>();
    reg<true, true, false, POST_NONE, true, false>();
    reg<false, true, false, POST_NORM, true, false>();
    reg<true, true, false, POST_NORM, true, false>();
    // residual passes without a sweep (nu1 == 0, convergence norm, level operators)
    reg<false, false, false, POST_NORM, false, false>();
    reg<true, false, false, POST_NORM, false, false>();
    reg<false, false, false, POST_RESTRICT, false, false>();
    reg<true, false, false, POST_RESTRICT, false, false>();
    reg<true, false, false, POST_RESID, false, false>();
  }
  const KernelEntry<T>& get(const Variant& v) const {
    const KernelEntry<T>& k = e[v.key()];
    if (!k.fn) throw std::logic_error("pdmg_b200: no kernel instantiated for variant " + v.name());
    return k;
  }
};

template <class T>
struct MarchTable {
  void (*e[128])(MarchArgs<T>) = {};
  static int key(bool lu, bool pr, int post, bool ja, int lc, bool nin = false) {
    return (lu ? 1 : 0) | (pr ? 2 : 0) | (post << 2) | (ja ? 16 : 0) | (lc == 2 ? 32 : 0) | (nin ? 64 : 0);
  }
  template <bool LU, bool PR, int PO, bool JA>
  void reg() {
    e[key(LU, PR, PO, JA, 1)] = &k_march<T, LU, PR, PO, JA, 1>;
    e[key(LU, PR, PO, JA, 2)] = &k_march<T, LU, PR, PO, JA, 2>;
  }
  template <int PO, bool JA>
  void reg4() {
    reg<false, false, PO, JA>();
    reg<true, false, PO, JA>();
    if constexpr (PO != POST_RESTRICT) {
      reg<false, true, PO, JA>();
      reg<true, true, PO, JA>();
    }
  }
  template <bool LU, int PO, bool JA>
  void reg_nin() {  // first fine sweep of a cycle that also yields the previous iterate's residual norm
    e[key(LU, false, PO, JA, 2, true)] = &k_march<T, LU, false, PO, JA, 2, true>;
  }
  MarchTable() {
    reg_nin<false, POST_RESTRICT, false>();
    reg_nin<true, POST_RESTRICT, false>();
    reg_nin<false, POST_RESTRICT, true>();
    reg_nin<true, POST_RESTRICT, true>();
    reg4<POST_NONE, false>();
    reg4<POST_NONE, true>();
    reg4<POST_NORM, false>();
    reg4<POST_NORM, true>();
    reg4<POST_RESTRICT, false>();
    reg4<POST_RESTRICT, true>();
  }
};

// two-sweep fused Vanka passes (k_march2): key = loadu | prolong << 1 | post << 2
template <class T>
struct March2Table {
  void (*e[64])(MarchArgs<T>, CoefPack) = {};
  static int key(bool lu, bool pr, int post, bool nin = false, bool mid = false) {
    return (lu ? 1 : 0) | (pr ? 2 : 0) | (post << 2) | (nin ? 16 : 0) | (mid ? 32 : 0);
  }
  void (*ws[64])(MarchArgs<T>, CoefPack) = {};  // warp-specialised pair kernels (k_march2ws), same keys
  size_t smem[64] = {};
  template <bool LU, bool PR, int PO, bool NI = false, bool MID = false>
  void reg() {
    if constexpr (!MID) ws[key(LU, PR, PO, NI)] = &k_march2ws<T, LU, PR, PO, NI>;
    e[key(LU, PR, PO, NI, MID)] = &k_march2<T, LU, PR, PO, NI, MID>;
    smem[key(LU, PR, PO, NI, MID)] = march2_smem<T>(LU);
    if (march2_smem<T>(LU) > 0)
      CK(cudaFuncSetAttribute(&k_march2<T, LU, PR, PO, NI, MID>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)march2_smem<T>(LU)));
  }
  March2Table() {
    reg<false, false, POST_NONE>();
    reg<true, false, POST_NONE>();
    reg<false, false, POST_RESTRICT>();
    reg<true, false, POST_RESTRICT>();
    reg<false, false, POST_NORM>();
    reg<true, false, POST_NORM>();
    reg<false, true, POST_NONE>();
    reg<true, true, POST_NONE>();
    reg<false, true, POST_NORM>();
    reg<true, true, POST_NORM>();
    reg<false, false, POST_RESTRICT, true>();
    reg<true, false, POST_RESTRICT, true>();
    reg<false, false, POST_NONE, true>();
    reg<true, false, POST_NONE, true>();
    reg<true, true, POST_RESTRICT, false, true>();  // V(1,1) cross-cycle fusion
    reg1<false>();
    reg1<true>();
  }
  // one-sweep passes (k_march2<..., TWO = false>), same keys
  void (*e1[64])(MarchArgs<T>, CoefPack) = {};
  template <bool LU>
  void reg1() {
    e1[key(LU, false, POST_NONE)] = &k_march2<T, LU, false, POST_NONE, false, false, false>;
    e1[key(LU, false, POST_RESTRICT)] = &k_march2<T, LU, false, POST_RESTRICT, false, false, false>;
    e1[key(LU, false, POST_NORM)] = &k_march2<T, LU, false, POST_NORM, false, false, false>;
    e1[key(LU, true, POST_NONE)] = &k_march2<T, LU, true, POST_NONE, false, false, false>;
    e1[key(LU, true, POST_NORM)] = &k_march2<T, LU, true, POST_NORM, false, false, false>;
    e1[key(LU, false, POST_RESTRICT, true)] = &k_march2<T, LU, false, POST_RESTRICT, true, false, false>;
    e1[key(LU, false, POST_NONE, true)] = &k_march2<T, LU, false, POST_NONE, true, false, false>;
  }
};

// ---------------------------------------------------------------------------------------------
// Engine: one batch of shifts on one device.
// ---------------------------------------------------------------------------------------------
struct Stat {
  int64_t launches = 0;
  double ms = 0.0, bytes = 0.0;  // bytes: the minimum DRAM traffic of the fused pass (what it must move)
  double ubytes = 0.0;           // SURVEY 8(d) algorithmic bytes: 48 B (c128) per smoother update + transfers
  double updates = 0.0;          // grid-point smoother updates
};

// Precision-independent part of an engine (what the C ABI needs without knowing the storage type).
struct EngineBase {
  int device = 0;
  cudaStream_t stream = nullptr;
  int S = 0;
  pdmg_mg_config cfg{};
  std::vector<int> ln;
  std::vector<cplx> lambdas;
  std::vector<uint8_t> coarse_singular;
  bool any_singular = false;
  bool profiling = false;
  int64_t launches = 0;
  std::map<std::string, Stat> stats;
  double last_updates = 0.0;
  int solve_path = 0;  // 0 auto, 1 batched level passes, 2 one CTA per shift (small grids)

  virtual ~EngineBase() = default;
  virtual void setup_host(const pdmg_batch_desc& d) = 0;
  virtual void setup_device(int dev) = 0;
  virtual void solve_host(const pdmg_c128* b, pdmg_c128* u, pdmg_solve_report* rep) = 0;
  virtual void solve_device(const double2* d_b, double2* d_u, pdmg_solve_report* rep) = 0;
  virtual void cycle_host(pdmg_c128* u, const pdmg_c128* b) = 0;
  virtual void op_smooth(int l, const pdmg_c128* u, const pdmg_c128* b, pdmg_c128* out) = 0;
  virtual void op_residual(int l, const pdmg_c128* b, const pdmg_c128* u, pdmg_c128* r) = 0;
  virtual void op_restrict(int l, const pdmg_c128* fine, pdmg_c128* coarse) = 0;
  virtual void op_prolong(int l, const pdmg_c128* coarse, pdmg_c128* fine) = 0;
  virtual void op_norm(int l, const pdmg_c128* v, double* norms) = 0;
  virtual void op_coarse_solve(const pdmg_c128* b, pdmg_c128* u) = 0;
};

template <class T>
struct Engine : EngineBase {
  using V = typename vec2<T>::type;
  struct Level {
    int n = 0, m = 0;
    int64_t ss = 0;  // shift stride (elements)
    size_t elems = 0;
    V* u[3] = {nullptr, nullptr, nullptr};  // u[2]: level 0 only, V(1,1) cross-cycle fusion
    V* b = nullptr;
    int ntx = 0, nty = 0, ntiles = 0, H = 0;
    LevelCoef* coef = nullptr;
    std::vector<LevelCoef> hcoef;  // host copy (kernel-parameter coefficient packs)
    int cur = 0;
    bool uzero = false;
  };

  std::vector<Level> lv;
  double2* d_ainv = nullptr;
  int coarse_N = 0;
  int last_partials = 0;  // partial sums written by the last level pass (tiles or warp tasks per shift)
  int *d_active = nullptr, *d_iters = nullptr, *d_conv = nullptr, *d_nactive = nullptr, *d_parity = nullptr;
  int* d_ones = nullptr;
  double *d_r0 = nullptr, *d_hist = nullptr, *d_partial = nullptr, *d_norms = nullptr;
  double2* d_stage = nullptr;  // compact complex128 host-I/O staging
  size_t stage_elems = 0;
  // mapped pinned results, written by k_copy_words: [hist S*H doubles][iters S][conv S][nactive 2]
  char* h_map = nullptr;
  char* d_map = nullptr;
  size_t map_hist() const { return 0; }
  size_t map_iters() const { return sizeof(double) * (size_t)S * (cfg.max_iter + 1); }
  size_t map_conv() const { return map_iters() + sizeof(int) * S; }
  size_t map_nact() const { return map_conv() + sizeof(int) * S; }
  void to_host(const void* dsrc, size_t map_off, size_t bytes) {
    const int64_t w = (int64_t)(bytes / 4);
    const int blocks = (int)std::min<int64_t>((w + 255) / 256, 148);
    k_copy_words<<<std::max(blocks, 1), 256, 0, stream>>>((const uint32_t*)dsrc, (uint32_t*)(d_map + map_off), w);
  }
  cudaEvent_t ev_nactive[2] = {nullptr, nullptr};
  int n_active_host = 0;
  const KernelTable<T>* table = nullptr;
  // instrumentation
  struct Pending {
    std::string cls;
    cudaEvent_t e0, e1;
    double bytes, ubytes, updates;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  int march_min_n = 64;  // levels with n >= this use the warp-marching sweep kernel (0 = never)
  int level_h_min_n = 512;  // levels with n >= this use 128-row strips in k_level (else 64)
  int tail_max_n = 64;      // levels with n <= this run as one per-shift CTA cycle (k_small_cycle); 0 = off
  int march_hs = 0;       // strip height override (0 = automatic)
  int march_lc = 2;       // columns per lane of the marcher (1 or 2)

  static const MarchTable<T>& marches() {
    static MarchTable<T> t;
    return t;
  }
  static const March2Table<T>& marches2() {
    static March2Table<T> t;
    return t;
  }
  int march2_min_n = 64;  // levels with n >= this run Vanka sweep pairs as one k_march2 pass (0 = never)
  int march2_hs = 0;      // strip height override (0 = automatic)
  // per-level strip heights (tuning: PDMG_MARCH2_HS_R / _P = "n:H,n:H,..." for the non-prolongating /
  // prolongating passes; levels not listed use march2_hs_default)
  std::vector<std::pair<int, int>> march2_hs_r, march2_hs_p;
  int march2_prolong_b = 0;  // prolongating passes may use loop shape (b) on levels with n >= march2_loopb_min_n
  static int march2_ha(int post, bool two) {  // = k_march2's hA
    return ((two ? 4 : 2) + (post == POST_RESTRICT ? 2 : post == POST_NORM ? 1 : 0) + 1) & ~1;
  }
  int march2_tasks(int n, int post, bool two, bool prolong) const {  // warp tasks per shift of a k_march2 pass
    const int wout = 64 - 2 * march2_ha(post, two), hs = march2_hs_for(n, prolong);
    return ((n + wout - 1) / wout) * ((n + hs - 1) / hs);
  }
  int march2_hs_for(int n, bool prolong) const {
    if (march2_hs > 0) return march2_hs;
    for (auto& e : prolong ? march2_hs_p : march2_hs_r)
      if (e.first == n) return e.second;
    return n >= 512 ? 128 : n >= 256 ? 64 : 32;  // measured at C3 (DESIGN 3.2b)
  }
  bool march2_pre = true, march2_post = true;  // fuse the pre- / post-smoothing sweep pairs
  int march2_loopb_min_n = 128;  // (prolongating passes: shape (a), see march2_prolong_b)
  bool march2_ws = false;  // run the pair passes as warp-specialised producer/consumer warp pairs (k_march2ws)
  bool norm_next = true;  // fine-level convergence norm from the next cycle's first pass (see solve_device)
  double pred_final = 0.5;  // predicted-last-norm threshold (solve_device; 0 = off, PDMG_PRED_FINAL)
  // V(1,1): fuse cycle k's fine post-sweep with cycle k+1's pre-sweep (solve_xfuse).  Off by default:
  // measured on B200 the fused pass costs what the two single-sweep passes cost (C3 at V(1,1): 1621 vs
  // 807 + 821 us; C4 with 256 shifts: 6.38 vs 6.75 ms; C5 9.75 vs 9.08 ms per step) -- the passes are
  // issue/latency-bound, so halving the fine-level bytes does not pay.  PDMG_XFUSE=1 enables it.
  bool xfuse = false;
  // (level sizes from `ln`: also called while the levels are being allocated)
  bool use_xfuse() const {
    return xfuse && norm_next && cfg.nu1 == 1 && cfg.nu2 == 1 && cfg.smoother == PDMG_SMOOTHER_VANKA &&
           ln.size() >= 3 && march2_min_n > 0 && ln[0] >= march2_min_n && march_min_n > 0 && ln[0] >= march_min_n &&
           march_lc == 2 && ln[1] > 4;
  }
  int nin_k = -1;         // cycle_level: the first fine pass computes the norm of iterate nin_k (>= 0)
  // the first fine pass of a cycle must be a marching sweep that can also form ||b - L u_in||: the single
  // sweep + restriction (nu1 = 1) or a fused pair (even nu1)
  bool use_norm_next() const {
    if (!norm_next || lv.size() < 2) return false;
    if (cfg.nu1 == 1) return march_min_n > 0 && lv[0].n >= march_min_n && march_lc == 2;
    return march2_pre && use_march2(0) && cfg.nu1 >= 2 && cfg.nu1 % 2 == 0;
  }
  bool use_march2(int l) const {
    return march2_min_n > 0 && lv[l].n >= march2_min_n && cfg.smoother == PDMG_SMOOTHER_VANKA;
  }
  std::unique_ptr<CoefPack> cpack{new CoefPack()};
  // coefficients of engine shifts [c0, c0 + cnt) (RangeView: engine shift s = global shift s_base + s)
  void fill_pack(const Level& Lv, int c0, int cnt) {
    cpack->inv_h2 = Lv.hcoef.empty() ? 0.0 : Lv.hcoef[0].inv_h2;
    cpack->shift0 = c0;
    for (int i = 0; i < cnt; ++i) {
      const LevelCoef& c = Lv.hcoef[s_base + c0 + i];
      cpack->c[i] = CoefU{c.dd, c.k0, c.k1, c.k2};
    }
  }
  // two consecutive Vanka sweeps u[cur] -> u[cur^1] (+ prolongation of ec before, + restriction/norm after)
  // two = false: ONE Vanka sweep through the same kernel (k_march2<..., TWO = false>)
  void level_pass2(int l, bool loadu, bool prolong, int post, const V* uin, V* uout, const V* b, const V* ec, V* bc,
                   const int* active, int n_act, bool norm_in = false, V* umid = nullptr, bool two = true) {
    const Level& Lv = lv[l];
    MarchArgs<T> ma{};
    ma.u_in = uin, ma.u_out = uout, ma.b = b, ma.ec = ec, ma.bc = bc, ma.partial = d_partial, ma.u_mid = umid;
    ma.coef = Lv.coef, ma.active = active, ma.n = Lv.n;
    ma.nc = (l + 1 < (int)lv.size()) ? lv[l + 1].n : Lv.n / 2;
    ma.ss = Lv.ss, ma.ssc = (l + 1 < (int)lv.size()) ? lv[l + 1].ss : 0;
    const int wout = 64 - 2 * march2_ha(post, two);
    ma.Hs = march2_hs_for(Lv.n, prolong);
    // loop shape (a) for prolongating passes unless march2_prolong_b (measured, DESIGN 3.2b)
    ma.loop_a = Lv.n < march2_loopb_min_n || (prolong && !march2_prolong_b);
    ma.ntx = (Lv.n + wout - 1) / wout;
    ma.ntasks = ma.ntx * ((Lv.n + ma.Hs - 1) / ma.Hs);
    if (ma.ntasks != march2_tasks(Lv.n, post, two, prolong)) throw std::logic_error("pdmg_b200: march2 task count");
    const int key2 = March2Table<T>::key(loadu, prolong, post, norm_in, umid != nullptr);
    const bool ws = two && march2_ws && umid == nullptr;
    auto fn = !two ? marches2().e1[key2] : ws ? marches2().ws[key2] : marches2().e[key2];
    const size_t smem2 = ws || !two ? 0 : marches2().smem[key2];
    if (!fn) throw std::logic_error("pdmg_b200: no two-sweep kernel for this variant");
    const double S_ = sizeof(V), pts = (double)n_act * Lv.m * Lv.m;
    const double bpp = (loadu ? S_ : 0) + S_ + (prolong ? S_ / 4 : 0) + S_ + (post == POST_RESTRICT ? S_ / 4 : 0) +
                       (umid ? S_ : 0);
    std::string cls = "L" + std::to_string(l) + ":" + (prolong ? (loadu ? "prolong+" : "prolong0+") : (loadu ? "" : "zero+")) +
                      (two ? "vanka2" : "vanka") + (post == POST_NORM ? "+norm" : post == POST_RESTRICT ? "+restrict" : "") +
                      (norm_in ? "+norm_in" : "") + (umid ? "+mid" : "");
    const int per_cta = ws ? WS_PAIRS : MARCH_WARPS;
    const double ubpp = (two ? 2 : 1) * 3 * S_ + (prolong ? S_ / 4 : 0) + (post == POST_RESTRICT ? S_ / 4 : 0) + (umid ? S_ : 0);
    timed(cls, pts * bpp, [&] {
      for (int c0 = 0; c0 < S; c0 += COEF_MAX) {  // one launch per COEF_MAX shifts (coefficients as parameters)
        const int cnt = std::min(COEF_MAX, S - c0);
        fill_pack(Lv, c0, cnt);
        dim3 grid((ma.ntasks + per_cta - 1) / per_cta, cnt);
        fn<<<grid, ws ? WS_THREADS : 32 * MARCH_WARPS, smem2, stream>>>(ma, *cpack);
      }
    }, pts * ubpp, (two ? 2 : 1) * pts);
    last_partials = ma.ntasks;
  }
  // measured on B200 (C3, C4): the marcher wins for sweep+norm and sweep+restrict, the ring
  // kernel for the plain and prolongating sweeps; PDMG_MARCH_ALL=1 routes every sweep variant to the marcher
  bool march_all = false;
  // single Vanka sweeps on levels with n >= march2_min_n through k_march2<TWO = false> (PDMG_MARCH1=0: the
  // older k_level / k_march kernels)
  bool march1 = true;
  bool resid_norm_kernel = true;  // residual-only norm passes through k_resid_norm (PDMG_RESID_NORM=0: k_level)
  bool use_march1(int l, const Variant& v) const {
    return march1 && march2_min_n > 0 && lv[l].n >= march2_min_n && v.sweep && v.store && !v.jacobi &&
           v.post != POST_RESID && marches2().e1[March2Table<T>::key(v.loadu, v.prolong, v.post)] != nullptr;
  }
  bool use_march(int l, const Variant& v) const {
    if (!(march_min_n > 0 && lv[l].n >= march_min_n && v.sweep && v.store && v.post != POST_RESID)) return false;
    if (march_all) return true;
    return !v.prolong && (v.post == POST_NORM || v.post == POST_RESTRICT);
  }
  int march_hs_for(int n) const { return march_hs > 0 ? march_hs : (n >= 512 ? 128 : 64); }
  int march_tasks(int l, int post) const {
    const int hA = (post == POST_RESTRICT ? 1 : post == POST_NONE ? -1 : 0) + 3;
    const int wout = 32 - 2 * hA, n = lv[l].n, hs = march_hs_for(n);  // LC = 1 (most tasks): sizing bound
    return ((n + wout - 1) / wout) * ((n + hs - 1) / hs);
  }

  bool use_small_path() const {
    if (solve_path == 1) return false;
    if (solve_path == 2) return true;
    return lv[0].n <= 128 && lv.size() <= MAX_LEVELS;  // BASELINE configs 1-2: launch/sync latency bound
  }

  static const KernelTable<T>& kernels() {
    static KernelTable<T> t;
    return t;
  }

  ~Engine() {
    if (device >= 0) cudaSetDevice(device);
    for (auto& L : lv) {
      if (!borrow) {
        cudaFree(L.u[0]);
        cudaFree(L.u[1]);
        cudaFree(L.u[2]);
        cudaFree(L.b);
      }
      cudaFree(L.coef);
    }
    cudaFree(d_ainv);
    cudaFree(d_active);
    cudaFree(d_iters);
    cudaFree(d_conv);
    cudaFree(d_nactive);
    cudaFree(d_parity);
    cudaFree(d_ones);
    cudaFree(d_r0);
    cudaFree(d_hist);
    cudaFree(d_partial);
    cudaFree(d_norms);
    cudaFree(d_stage);
    if (h_map) cudaFreeHost(h_map);
    for (auto e : ev_nactive)
      if (e) cudaEventDestroy(e);
    for (auto& p : pending) {
      cudaEventDestroy(p.e0);
      cudaEventDestroy(p.e1);
    }
    for (auto e : event_pool) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (stream) cudaStreamDestroy(stream);
  }

  // ---- construction: host validation first (no CUDA), then device allocation ----------------
  void setup_host(const pdmg_batch_desc& d) override {
    desc_ = d;
    desc_.lambdas = nullptr;  // (the engine keeps its own copy in `lambdas`)
    if (d.n_shifts < 1) throw ConfigError("pdmg_create: n_shifts must be >= 1");
    if (d.n_shifts > 65535) throw ConfigError("pdmg_create: n_shifts must be <= 65535 per context");
    if (!d.lambdas) throw ConfigError("pdmg_create: lambdas is NULL");
    cfg = d.cfg;
    ln = level_list(d.n, cfg);
    S = d.n_shifts;
    lambdas.resize(S);
    for (int s = 0; s < S; ++s) lambdas[s] = cplx(d.lambdas[s].re, d.lambdas[s].im);
    // smoother validity on every non-coarsest level (multigrid.cpp:47-58), in shift order
    for (int s = 0; s < S; ++s)
      for (size_t l = 0; l + 1 < ln.size(); ++l) {
        const double h = 1.0 / ln[l];
        try {
          if (cfg.smoother == PDMG_SMOOTHER_VANKA) (void)vanka_coeffs(lambdas[s] * (h * h));
          else (void)jacobi_weight(lambdas[s] * (h * h), h);
        } catch (const SingularOperatorError& e) {
          throw SingularOperatorError("level " + std::to_string(l) + " (n = " + std::to_string(ln[l]) + "): " + e.what());
        }
      }
    if (ln.back() > 128)
      throw ConfigError("dense_shifted_operator: dense assembly refused for n = " + std::to_string(ln.back()) +
                        " (limit 128)");
  }

  void setup_device(int dev) override {
    device = dev;
    if (const char* e = std::getenv("PDMG_MARCH_MIN_N")) march_min_n = std::atoi(e);
    if (const char* e = std::getenv("PDMG_LEVEL_H_MIN_N")) level_h_min_n = std::atoi(e);
    if (const char* e = std::getenv("PDMG_TAIL_MAX_N")) tail_max_n = std::atoi(e);
    if (const char* e = std::getenv("PDMG_IO_CHUNKS")) io_chunks = std::atoi(e);
    if (const char* e = std::getenv("PDMG_IO_MODE")) io_mode = std::atoi(e);
    if (const char* e = std::getenv("PDMG_SMALL_THREADS")) small_threads_env = std::atoi(e);
    if (const char* e = std::getenv("PDMG_MARCH2_MIN_N")) march2_min_n = std::atoi(e);
    if (const char* e = std::getenv("PDMG_MARCH2_HS")) march2_hs = std::atoi(e);
    auto parse_hs = [](const char* e, std::vector<std::pair<int, int>>& out) {
      out.clear();
      for (const char* q = e; *q;) {
        int n = 0, h = 0;
        if (std::sscanf(q, "%d:%d", &n, &h) == 2 && n > 0 && h > 0) out.emplace_back(n, h);
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
    };
    if (const char* e = std::getenv("PDMG_MARCH2_HS_R")) parse_hs(e, march2_hs_r);
    if (const char* e = std::getenv("PDMG_MARCH2_HS_P")) parse_hs(e, march2_hs_p);
    if (const char* e = std::getenv("PDMG_MARCH2_PROLONG_B")) march2_prolong_b = std::atoi(e);
    if (const char* e = std::getenv("PDMG_MARCH2_PRE")) march2_pre = std::atoi(e) != 0;
    if (const char* e = std::getenv("PDMG_MARCH2_POST")) march2_post = std::atoi(e) != 0;
    if (const char* e = std::getenv("PDMG_NORM_NEXT")) norm_next = std::atoi(e) != 0;
    if (const char* e = std::getenv("PDMG_XFUSE")) xfuse = std::atoi(e) != 0;
    if (const char* e = std::getenv("PDMG_MARCH2_LOOPB_MIN_N")) march2_loopb_min_n = std::atoi(e);
    if (const char* e = std::getenv("PDMG_MARCH2_WS")) march2_ws = std::atoi(e) != 0;
    if (const char* e = std::getenv("PDMG_MARCH_HS")) march_hs = std::atoi(e);
    if (const char* e = std::getenv("PDMG_MARCH_ALL")) march_all = std::atoi(e) != 0;
    if (const char* e = std::getenv("PDMG_MARCH1")) march1 = std::atoi(e) != 0;
    if (const char* e = std::getenv("PDMG_PRED_FINAL")) pred_final = std::atof(e);
    if (const char* e = std::getenv("PDMG_RESID_NORM")) resid_norm_kernel = std::atoi(e) != 0;
    if (const char* e = std::getenv("PDMG_MARCH_LC")) march_lc = std::atoi(e) == 1 ? 1 : 2;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (dev < 0 || dev >= ndev) throw CudaError("pdmg_create: CUDA device " + std::to_string(dev) + " not available");
    CK(cudaSetDevice(dev));
    CK(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, stream_priority));
    table = &kernels();
    const int L = (int)ln.size();
    lv.resize(L);
    for (int l = 0; l < L; ++l) {
      Level& Lv = lv[l];
      Lv.n = ln[l];
      Lv.m = Lv.n - 1;
      Lv.ss = (int64_t)(Lv.n + 1) * Lv.n;
      Lv.elems = (size_t)Lv.ss * S + Lv.n + 2;  // + guard so the last shift's ghost reads stay in bounds
      if (borrow) {
        // the parent's arrays are zeroed (ghost rings included); past the last shift of a middle range the
        // guard reads land in the next range's first shift, exactly as they do inside the parent
        const Level& P = borrow->lv[l];
        const int64_t off = (int64_t)borrow_s0 * Lv.ss;
        Lv.u[0] = P.u[0] + off, Lv.u[1] = P.u[1] + off, Lv.b = P.b + off;
        Lv.u[2] = P.u[2] ? P.u[2] + off : nullptr;
        if (borrow_s0 + S < borrow->S) Lv.elems = (size_t)Lv.ss * S;
      } else {
        for (V** p : {&Lv.u[0], &Lv.u[1], &Lv.b}) {
          CK(cudaMalloc(p, Lv.elems * sizeof(V)));
          CK(cudaMemsetAsync(*p, 0, Lv.elems * sizeof(V), stream));
        }
        if (l == 0 && use_xfuse()) {
          CK(cudaMalloc(&Lv.u[2], Lv.elems * sizeof(V)));
          CK(cudaMemsetAsync(Lv.u[2], 0, Lv.elems * sizeof(V), stream));
        }
      }
      Lv.H = std::min(Lv.n >= level_h_min_n ? 128 : 64, Lv.n + (Lv.n & 1));
      Lv.ntx = (Lv.n + TILE_W - 1) / TILE_W;
      Lv.nty = (Lv.n + Lv.H - 1) / Lv.H;
      Lv.ntiles = Lv.ntx * Lv.nty;
      // coefficients (multigrid.cpp:47-58 per level; smoother.cpp:31-40 stencil; grid.cpp:73 diagonal)
      std::vector<LevelCoef> hc(S);
      const double h = 1.0 / Lv.n;
      for (int s = 0; s < S; ++s) {
        const cplx eta = lambdas[s] * (h * h);
        const cplx dd = cplx(4.0, 0.0) + eta;
        cplx k0(0, 0), k1(0, 0), k2(0, 0);
        if (l + 1 < L) {
          if (cfg.smoother == PDMG_SMOOTHER_VANKA) {
            const Vanka v = vanka_coeffs(eta);
            const double sc = cfg.omega * (h * h / 4.0);
            k0 = sc * (4.0 * v.a);
            k1 = sc * (2.0 * v.b);
            k2 = sc * v.c;
          } else {
            k0 = cfg.omega * jacobi_weight(eta, h);
          }
        }
        LevelCoef& c = hc[s];
        c.d = make_double2(dd.real(), dd.imag());
        c.dd = make_double2(dd.real() / (h * h), dd.imag() / (h * h));
        c.k0 = make_double2(k0.real(), k0.imag());
        c.k1 = make_double2(k1.real(), k1.imag());
        c.k2 = make_double2(k2.real(), k2.imag());
        c.inv_h2 = 1.0 / (h * h);
        c.pad_ = 0;
      }
      Lv.hcoef = hc;
      CK(cudaMalloc(&Lv.coef, sizeof(LevelCoef) * S));
      CK(cudaMemcpyAsync(Lv.coef, hc.data(), sizeof(LevelCoef) * S, cudaMemcpyHostToDevice, stream));
    }
    // coarsest factorizations (dense.cpp:82-88), one per shift
    const int nc = ln.back(), mc = nc - 1;
    coarse_N = mc * mc;
    coarse_singular.assign(S, 0);
    std::vector<double2> hinv((size_t)S * coarse_N * coarse_N);
    for (int s = 0; s < S; ++s) {
      CoarseFactor cf = factor_coarse(nc, lambdas[s]);
      coarse_singular[s] = cf.singular;
      any_singular |= cf.singular;
      for (size_t q = 0; q < cf.inv.size(); ++q) {
        hinv[(size_t)s * coarse_N * coarse_N + q] = make_double2(cf.inv[q].real(), cf.inv[q].imag());
      }
    }
    CK(cudaMalloc(&d_ainv, sizeof(double2) * hinv.size()));
    CK(cudaMemcpyAsync(d_ainv, hinv.data(), sizeof(double2) * hinv.size(), cudaMemcpyHostToDevice, stream));
    // solve state
    int maxtiles = 1;
    for (size_t l = 0; l < lv.size(); ++l) {
      maxtiles = std::max(maxtiles, lv[l].ntiles);
      for (int post : {POST_NONE, POST_NORM, POST_RESTRICT}) {
        maxtiles = std::max(maxtiles, march_tasks((int)l, post));
        for (int two = 0; two < 2; ++two)
          for (int pr = 0; pr < 2; ++pr) maxtiles = std::max(maxtiles, march2_tasks(lv[l].n, post, two != 0, pr != 0));
      }
      maxtiles = std::max(maxtiles, (lv[l].n - 1 + RN_ROWS - 1) / RN_ROWS);  // k_resid_norm
    }
    CK(cudaMalloc(&d_active, sizeof(int) * S));
    CK(cudaMalloc(&d_iters, sizeof(int) * S));
    CK(cudaMalloc(&d_conv, sizeof(int) * S));
    CK(cudaMalloc(&d_nactive, 6 * sizeof(int)));  // [n_active slot 0, 1][pred slot 0, 1 (8 B each)]
    CK(cudaMalloc(&d_parity, sizeof(int) * (cfg.max_iter + 1)));
    CK(cudaMalloc(&d_ones, sizeof(int) * S));
    CK(cudaMalloc(&d_r0, sizeof(double) * S));
    CK(cudaMalloc(&d_hist, sizeof(double) * S * (size_t)(cfg.max_iter + 1)));
    CK(cudaMalloc(&d_partial, sizeof(double) * S * (size_t)maxtiles));
    CK(cudaMalloc(&d_norms, sizeof(double) * S));
    std::vector<int> ones(S, 1);
    CK(cudaMemcpyAsync(d_ones, ones.data(), sizeof(int) * S, cudaMemcpyHostToDevice, stream));
    CK(cudaHostAlloc((void**)&h_map, map_nact() + 6 * sizeof(int), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&d_map, h_map, 0));
    CK(cudaEventCreateWithFlags(&ev_nactive[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_nactive[1], cudaEventDisableTiming));
    for (auto& kv : table->e)
      if (kv.fn) CK(cudaFuncSetAttribute(kv.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kv.smem));
    CK(cudaStreamSynchronize(stream));
  }

  // ---- instrumentation ---------------------------------------------------------------------
  cudaEvent_t get_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  // ubytes < 0: the pass performs no smoother update, its algorithmic bytes are the bytes it moves
  template <class F>
  void timed(const std::string& cls, double bytes, F&& launch, double ubytes = -1.0, double updates = 0.0) {
    ++launches;
    if (!profiling) {
      launch();
      return;
    }
    Pending p{cls, get_event(), get_event(), bytes, ubytes < 0 ? bytes : ubytes, updates};
    CK(cudaEventRecord(p.e0, stream));
    launch();
    CK(cudaEventRecord(p.e1, stream));
    pending.push_back(p);
  }
  void drain_stats() {
    if (pending.empty()) return;
    CK(cudaStreamSynchronize(stream));
    for (auto& p : pending) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, p.e0, p.e1));
      Stat& st = stats[p.cls];
      st.launches += 1;
      st.ms += ms;
      st.bytes += p.bytes;
      st.ubytes += p.ubytes;
      st.updates += p.updates;
      event_pool.push_back(p.e0);
      event_pool.push_back(p.e1);
    }
    pending.clear();
  }

  // ---- kernel launch ------------------------------------------------------------------------
  void level_pass(int l, const Variant& v, const V* uin, V* uout, const V* b, const V* ec, V* bc, const int* active,
                  int n_act, bool norm_in = false) {
    const Level& Lv = lv[l];
    LevelArgs<T> a{};
    a.u_in = uin;
    a.u_out = uout;
    a.b = b;
    a.ec = ec;
    a.bc = bc;
    a.partial = d_partial;
    a.coef = Lv.coef;
    a.active = active;
    a.n = Lv.n;
    a.nc = (l + 1 < (int)lv.size()) ? lv[l + 1].n : Lv.n / 2;
    a.ss = Lv.ss;
    a.ssc = (l + 1 < (int)lv.size()) ? lv[l + 1].ss : 0;
    a.ntx = Lv.ntx;
    a.ntiles = Lv.ntiles;
    a.H = Lv.H;
    const double pts = (double)n_act * Lv.m * Lv.m, S_ = sizeof(V);
    double bpp = 0;  // algorithmic DRAM bytes per point
    if (v.loadu) bpp += S_;
    if (v.sweep || v.post != POST_NONE) bpp += S_;  // b
    if (v.prolong) bpp += S_ / 4;
    if (v.store || v.post == POST_RESID) bpp += S_;
    if (v.post == POST_RESTRICT) bpp += S_ / 4;
    const std::string cls = "L" + std::to_string(l) + ":" + v.name() + (norm_in ? "+norm_in" : "");
    // a smoother update is 3 S (u in, b in, u out) whatever the pass actually moves
    const double ubpp = v.sweep ? 3 * S_ + (v.prolong ? S_ / 4 : 0) + (v.post == POST_RESTRICT ? S_ / 4 : 0) : -1.0;
    const double ub = ubpp < 0 ? -1.0 : pts * ubpp, nupd = v.sweep ? pts : 0.0;
    if (resid_norm_kernel && v.loadu && !v.prolong && !v.sweep && !v.store && v.post == POST_NORM && !norm_in) {
      const int ntiles = (Lv.m + RN_ROWS - 1) / RN_ROWS;
      dim3 grid(ntiles, S);
      timed(cls, pts * bpp, [&] {
        k_resid_norm<T><<<grid, RN_THREADS, 0, stream>>>(uin, b, Lv.coef, active, Lv.n, Lv.ss, d_partial);
      }, ub, nupd);
      last_partials = ntiles;
      return;
    }
    if (use_march1(l, v)) {
      level_pass2(l, v.loadu, v.prolong, v.post, uin, uout, b, ec, bc, active, n_act, norm_in, nullptr, false);
      return;
    }
    if (norm_in && !use_march(l, v)) throw std::logic_error("pdmg_b200: norm_in needs the marching kernel");
    if (use_march(l, v)) {
      MarchArgs<T> ma{};
      ma.u_in = uin, ma.u_out = uout, ma.b = b, ma.ec = ec, ma.bc = bc, ma.partial = d_partial;
      ma.coef = Lv.coef, ma.active = active, ma.n = a.n, ma.nc = a.nc, ma.ss = a.ss, ma.ssc = a.ssc;
      const int hA = (v.post == POST_RESTRICT ? 4 : v.post == POST_NORM ? 3 : 2);
      const int wout = 32 * march_lc - 2 * hA;
      ma.Hs = march_hs_for(Lv.n);
      ma.ntx = (Lv.n + wout - 1) / wout;
      ma.ntasks = ma.ntx * ((Lv.n + ma.Hs - 1) / ma.Hs);
      auto fn = marches().e[MarchTable<T>::key(v.loadu, v.prolong, v.post, v.jacobi, march_lc, norm_in)];
      if (!fn) throw std::logic_error("pdmg_b200: no march kernel for variant " + v.name());
      dim3 grid((ma.ntasks + MARCH_WARPS - 1) / MARCH_WARPS, S);
      timed(cls, pts * bpp, [&] { fn<<<grid, 32 * MARCH_WARPS, 0, stream>>>(ma); }, ub, nupd);
      last_partials = ma.ntasks;
      return;
    }
    const KernelEntry<T>& k = table->get(v);
    dim3 grid(Lv.ntiles, S);
    timed(cls, pts * bpp, [&] { k.fn<<<grid, NTHREADS, k.smem, stream>>>(a); }, ub, nupd);
    last_partials = Lv.ntiles;
  }

  void coarse_solve(const V* b, V* u, const int* active) {
    const Level& Lv = lv.back();
    const int thr = std::min(1024, std::max(32, ((coarse_N + 31) / 32) * 32));
    const double bytes = (double)S * coarse_N * (coarse_N + 2) * sizeof(V);
    timed("coarse_solve", bytes, [&] {
      k_coarse_solve<T><<<S, thr, coarse_N * sizeof(double2), stream>>>(b, u, d_ainv, active, Lv.n, Lv.ss);
    });
  }

  // ---- one cycle on level l (multigrid.cpp:63-77) -------------------------------------------
  // zero: u on this level is known to be zero on entry (ec = 0 before recursing, multigrid.cpp:72;
  // u = 0 before the first fine cycle, multigrid.cpp:90).  fuse_norm: leave ||b - L u||^2 partials of
  // the updated fine iterate in d_partial (returns whether it did).
  // first level of the coarse tail (levels with n <= tail_max_n below the finest), or -1
  int tail_level() const {
    if (tail_max_n <= 0 || (int)lv.size() > MAX_LEVELS) return -1;
    for (int l = 1; l < (int)lv.size(); ++l)
      if (lv[l].n <= tail_max_n) return l;
    return -1;
  }
  // Block size of the one-CTA-per-shift kernels (64 registers/thread: 1024 threads fill an SM's register
  // file).  Smaller blocks once S exceeds the SM count keep every shift resident in a single wave.
  int small_threads_env = 0;
  int small_threads() const {
    if (small_threads_env > 0) return small_threads_env;
    int sms = 148;
    return S <= sms ? SMALL_THREADS : S <= 2 * sms ? SMALL_THREADS / 2 : SMALL_THREADS / 4;
  }
  void tail_cycle(int l, const int* active, bool zero) {
    SmallArgs<T> sa{};
    for (size_t q = l; q < lv.size(); ++q)
      sa.lv[q - l] = SmallLevel<T>{lv[q].u[0], lv[q].u[1], lv[q].b, lv[q].coef, lv[q].n, lv[q].ss};
    sa.L = (int)lv.size() - l;
    sa.nu1 = cfg.nu1, sa.nu2 = cfg.nu2, sa.gamma = cfg.cycle == PDMG_CYCLE_W ? 2 : 1;
    sa.jacobi = cfg.smoother == PDMG_SMOOTHER_JACOBI, sa.max_iter = cfg.max_iter, sa.tol = cfg.tol;
    sa.ainv = d_ainv, sa.coarse_N = coarse_N, sa.active = active, sa.tail_zero = zero ? 1 : 0;
    timed("coarse_tail", 0.0,
          [&] { k_small_cycle<T><<<S, small_threads(), coarse_N * sizeof(double2), stream>>>(sa); });
    for (size_t q = l; q < lv.size(); ++q) lv[q].cur = 0, lv[q].uzero = false;
  }

  bool cycle_level(int l, bool zero, const int* active, int n_act, bool want_norm) {
    Level& Lv = lv[l];
    const int L = (int)lv.size();
    const bool jac = cfg.smoother == PDMG_SMOOTHER_JACOBI;
    if (l > 0 && l == tail_level()) {  // the whole coarse tail in one launch (each visit of a W-cycle)
      tail_cycle(l, active, zero);
      return false;
    }
    if (l + 1 == L) {
      coarse_solve(Lv.b, Lv.u[Lv.cur], active);
      Lv.uzero = false;
      return false;
    }
    Level& Lc = lv[l + 1];
    if (zero) Lv.uzero = true;
    const bool pair = use_march2(l) && march2_pre;
    for (int k = 0; k < cfg.nu1; ++k) {
      const bool last = k == cfg.nu1 - 1;
      if (pair && (cfg.nu1 - k) % 2 == 0) {  // sweeps k, k+1 as one pass (the pairs end at the last sweep)
        const bool nin = l == 0 && k == 0 && nin_k >= 0;
        level_pass2(l, !Lv.uzero, false, k + 2 == cfg.nu1 ? POST_RESTRICT : POST_NONE, Lv.u[Lv.cur], Lv.u[Lv.cur ^ 1],
                    Lv.b, nullptr, Lc.b, active, n_act, nin);
        if (nin) {  // convergence bookkeeping of the previous iterate (still in u[cur]) before the rest runs
          finalize(nin_k, last_partials, false, Lv.cur);
          nin_k = -1;
        }
        Lv.cur ^= 1;
        Lv.uzero = false;
        ++k;
        continue;
      }
      Variant v{!Lv.uzero, false, true, last ? POST_RESTRICT : POST_NONE, true, jac};
      const bool nin = l == 0 && k == 0 && nin_k >= 0;  // (only with nu1 == 1: see use_norm_next)
      level_pass(l, v, Lv.u[Lv.cur], Lv.u[Lv.cur ^ 1], Lv.b, nullptr, Lc.b, active, n_act, nin);
      if (nin) {
        finalize(nin_k, last_partials, false, Lv.cur);
        nin_k = -1;
      }
      Lv.cur ^= 1;
      Lv.uzero = false;
    }
    if (cfg.nu1 == 0) {
      Variant v{!Lv.uzero, false, false, POST_RESTRICT, false, false};
      level_pass(l, v, Lv.u[Lv.cur], nullptr, Lv.b, nullptr, Lc.b, active, n_act);
    }
    const int gamma = cfg.cycle == PDMG_CYCLE_W ? 2 : 1;
    for (int g = 0; g < gamma; ++g) cycle_level(l + 1, g == 0, active, n_act, false);
    const V* ec = Lc.u[Lc.cur];
    bool normed = false;
    if (cfg.nu2 > 0) {
      for (int k = 0; k < cfg.nu2; ++k) {
        const bool last = k == cfg.nu2 - 1;
        if (use_march2(l) && march2_post && k + 1 < cfg.nu2) {  // sweeps k, k+1 as one pass (pairs from the first, prolongating, sweep)
          const int post2 = (k + 2 == cfg.nu2 && want_norm) ? POST_NORM : POST_NONE;
          level_pass2(l, k == 0 ? !Lv.uzero : true, k == 0, post2, Lv.u[Lv.cur], Lv.u[Lv.cur ^ 1], Lv.b,
                      k == 0 ? ec : nullptr, nullptr, active, n_act);
          Lv.cur ^= 1;
          Lv.uzero = false;
          normed = post2 == POST_NORM;
          ++k;
          continue;
        }
        const int post = (last && want_norm) ? POST_NORM : POST_NONE;
        Variant v{k == 0 ? !Lv.uzero : true, k == 0, true, post, true, jac};
        level_pass(l, v, Lv.u[Lv.cur], Lv.u[Lv.cur ^ 1], Lv.b, k == 0 ? ec : nullptr, nullptr, active, n_act);
        Lv.cur ^= 1;
        Lv.uzero = false;
        normed = post == POST_NORM;
      }
    } else {
      Variant v{!Lv.uzero, true, false, want_norm ? POST_NORM : POST_NONE, true, false};
      level_pass(l, v, Lv.u[Lv.cur], Lv.u[Lv.cur ^ 1], Lv.b, ec, nullptr, active, n_act);
      Lv.cur ^= 1;
      Lv.uzero = false;
      normed = want_norm;
    }
    return normed;
  }

  // Convergence bookkeeping of cycle k (k_finalize); the active count lands in pinned slot k % 2.  With
  // wait = false the host does not block: the solve loop enqueues cycle k+1 before reading cycle k's count
  // (converged shifts are frozen on the device, so a speculative extra cycle leaves them untouched).
  void finalize(int k, int ntiles, bool wait = true, int cur = 0) {
    const int slot = k & 1;
    unsigned long long* d_pred = reinterpret_cast<unsigned long long*>(d_nactive + 2) + slot;
    CK(cudaMemsetAsync(d_nactive + slot, 0, sizeof(int), stream));
    CK(cudaMemsetAsync(d_pred, 0, sizeof(unsigned long long), stream));
    SolveState st{d_active, d_iters, d_conv, d_r0, d_hist, d_nactive + slot, S, cfg.max_iter, cfg.tol, d_parity, cur,
                  d_pred};
    const int threads = 256, blocks = (S * 32 + threads - 1) / threads;
    timed("finalize", 0.0, [&] { k_finalize<<<blocks, threads, 0, stream>>>(d_partial, ntiles, k, st); });
    to_host(d_nactive, map_nact(), 6 * sizeof(int));  // both slots' counts and predictions (24 B, one launch)
    CK(cudaEventRecord(ev_nactive[slot], stream));
    if (wait) n_active_host = read_nactive(k);
  }
  int read_nactive(int k) {
    CK(cudaEventSynchronize(ev_nactive[k & 1]));
    return ((volatile int*)(h_map + map_nact()))[k & 1];
  }
  // after read_nactive(k): max over the still-active shifts of the predicted r_{k+1} / (tol r0)
  double read_pred(int k) {
    const unsigned long long v = ((volatile unsigned long long*)(h_map + map_nact() + 2 * sizeof(int)))[k & 1];
    double q;
    std::memcpy(&q, &v, sizeof(q));
    return q;
  }

  void unpack(const double2* src, V* dst, int l) {
    const Level& Lv = lv[l];
    const int64_t total = (int64_t)S * Lv.m * Lv.m;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    timed("unpack", (double)total * 2 * sizeof(V),
          [&] { k_unpack<T><<<blocks, 256, 0, stream>>>(src, dst, Lv.n, Lv.ss, total); });
  }
  void pack(const V* b0, const V* b1, const int* iters, const int* parity, double2* dst, int l,
            const V* b2 = nullptr) {
    const Level& Lv = lv[l];
    const int64_t total = (int64_t)S * Lv.m * Lv.m;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    timed("pack", (double)total * 2 * sizeof(V),
          [&] { k_pack<T><<<blocks, 256, 0, stream>>>(b0, b1, b2 ? b2 : b0, iters, parity, dst, Lv.n, Lv.ss, total); });
  }

  // ---- MultigridHierarchy::solve for all shifts (multigrid.cpp:85-110) -----------------------
  void solve_device(const double2* d_b, double2* d_u, pdmg_solve_report* rep) override {
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaSetDevice(device));
    Level& F = lv[0];
    const int H = cfg.max_iter + 1;
    unpack(d_b, F.b, 0);
    CK(cudaMemsetAsync(F.u[0], 0, F.elems * sizeof(V), stream));
    F.cur = 0;
    CK(cudaMemcpyAsync(d_active, d_ones, sizeof(int) * S, cudaMemcpyDeviceToDevice, stream));
    CK(cudaMemsetAsync(d_iters, 0, sizeof(int) * S, stream));
    CK(cudaMemsetAsync(d_conv, 0, sizeof(int) * S, stream));
    CK(cudaMemsetAsync(d_hist, 0, sizeof(double) * S * (size_t)H, stream));
    if (use_small_path()) {
      if (any_singular) {
        // the reference throws at the first coarse solve, i.e. only for shifts that run a cycle
        std::vector<double> nb(S);
        level_pass(0, Variant{false, false, false, POST_NORM, false, false}, nullptr, nullptr, F.b, nullptr, nullptr,
                   nullptr, S);
        finalize(0, last_partials);
        std::vector<int> act(S);
        CK(cudaMemcpy(act.data(), d_active, sizeof(int) * S, cudaMemcpyDeviceToHost));
        for (int s = 0; s < S; ++s)
          if (act[s] && coarse_singular[s_base + s])
            throw SingularOperatorError("DenseShiftedSolver: operator is singular on grid n = " +
                                        std::to_string(lv.back().n));
      }
      SmallArgs<T> sa{};
      for (size_t l = 0; l < lv.size(); ++l)
        sa.lv[l] = SmallLevel<T>{lv[l].u[0], lv[l].u[1], lv[l].b, lv[l].coef, lv[l].n, lv[l].ss};
      sa.L = (int)lv.size();
      sa.nu1 = cfg.nu1, sa.nu2 = cfg.nu2, sa.gamma = cfg.cycle == PDMG_CYCLE_W ? 2 : 1;
      sa.jacobi = cfg.smoother == PDMG_SMOOTHER_JACOBI, sa.max_iter = cfg.max_iter, sa.tol = cfg.tol;
      sa.ainv = d_ainv, sa.coarse_N = coarse_N;
      sa.iterations = d_iters, sa.converged = d_conv, sa.r0 = d_r0, sa.hist = d_hist, sa.n_active = d_nactive;  // unused
      const double per_shift_bytes = 0.0;
      (void)per_shift_bytes;
      timed("small_solve", 0.0, [&] {
        k_small_solve<T><<<S, small_threads(), coarse_N * sizeof(double2), stream>>>(sa);
      });
      CK(cudaGetLastError());
      CK(cudaMemsetAsync(d_parity, 0, sizeof(int) * H, stream));
      pack(F.u[0], F.u[1], d_iters, d_parity, d_u, 0);
      finish_report(rep, t0, H);
      return;
    }
    if (use_xfuse() && !any_singular && !use_small_path()) {
      solve_xfuse();
      pack(F.u[0], F.u[1], d_iters, d_parity, d_u, 0, F.u[2]);
      finish_report(rep, t0, H);
      return;
    }
    if (use_norm_next() && !any_singular) {
      // The residual norm of iterate k-1 (multigrid.cpp:91, 96-105) is the first fine sweep's residual in
      // cycle k: that pass leaves its partials, k_finalize(k-1) runs right after it (freezing converged
      // shifts, whose iterate stays in the other buffer) and the rest of cycle k runs for the active ones.
      // The host reads count(k-1) once cycle k is enqueued, so it enqueues cycle k+1 while the GPU is
      // still in cycle k.  After max_iter cycles one norm pass closes the history.
      // Predicted last norm: when every active shift's predicted r_{k-1} (from finalize(k-2): the last
      // ratio times the last contraction) is below pred_final * tol * r0, iterate k-1's norm is formed by
      // a residual-only pass instead of cycle k's first (fused, two-sweep) pass, which would otherwise be
      // spent only to find that every shift has converged.  Mispredicted, cycle k runs without norm_in.
      int n_act = S, k = 1;
      double pred = 1e300;
      for (; k <= cfg.max_iter; ++k) {
        if (pred_final > 0 && k >= 4 && pred <= pred_final) {
          level_pass(0, Variant{true, false, false, POST_NORM, false, false}, F.u[F.cur], nullptr, F.b, nullptr,
                     nullptr, d_active, n_act);
          finalize(k - 1, last_partials, true, F.cur);
          n_act = n_active_host;
          if (n_act == 0) break;
          pred = read_pred(k - 1);
          nin_k = -1;
          cycle_level(0, false, d_active, n_act, false);
          continue;
        }
        nin_k = k - 1;
        const bool normed = cycle_level(0, k == 1, d_active, n_act, false);
        (void)normed;
        n_act = read_nactive(k - 1);
        if (n_act == 0) break;
        pred = read_pred(k - 1);
      }
      if (k > cfg.max_iter) {
        level_pass(0, Variant{true, false, false, POST_NORM, false, false}, F.u[F.cur], nullptr, F.b, nullptr,
                   nullptr, d_active, n_act);
        finalize(cfg.max_iter, last_partials, true, F.cur);
      }
      pack(F.u[0], F.u[1], d_iters, d_parity, d_u, 0);
      finish_report(rep, t0, H);
      return;
    }
    // r0 = ||b|| (multigrid.cpp:91): residual of the zero guess
    level_pass(0, Variant{false, false, false, POST_NORM, false, false}, nullptr, nullptr, F.b, nullptr, nullptr,
               nullptr, S);
    finalize(0, last_partials);
    if (any_singular && n_active_host > 0) {
      std::vector<int> act(S);
      CK(cudaMemcpy(act.data(), d_active, sizeof(int) * S, cudaMemcpyDeviceToHost));
      for (int s = 0; s < S; ++s)
        if (act[s] && coarse_singular[s_base + s])
          throw SingularOperatorError("DenseShiftedSolver: operator is singular on grid n = " + std::to_string(lv.back().n));
    }
    // cycles are enqueued one ahead of the host's convergence check (pipelined: the GPU never idles on it)
    int n_act = n_active_host;
    for (int k = 1; k <= cfg.max_iter && n_act > 0; ++k) {
      const bool normed = cycle_level(0, k == 1, d_active, n_act, true);
      if (!normed)
        level_pass(0, Variant{true, false, false, POST_NORM, false, false}, F.u[F.cur], nullptr, F.b, nullptr, nullptr,
                   d_active, n_act);
      finalize(k, last_partials, false, F.cur);  // records parity[k] = F.cur on the device
      if (k >= 2 || k == cfg.max_iter) n_act = read_nactive(k == cfg.max_iter ? k : k - 1);
      if (k == 1 && cfg.max_iter > 1) continue;  // cycle 2 is enqueued before cycle 1's count is read
    }
    pack(F.u[0], F.u[1], d_iters, d_parity, d_u, 0);
    finish_report(rep, t0, H);
  }

  // V(1,1) with the fine level fused across cycles: after cycle 1's pre-sweep, every fine pass is
  //   [u_in + P e_c -> post-sweep of cycle k -> u_k (stored to a third buffer) -> pre-sweep of cycle k+1
  //    -> residual -> restriction]
  // one k_march2<MID> pass: 4.5 S of HBM traffic per fine point and cycle instead of 6.5 S for the two
  // single-sweep passes.  Its partials are ||b - L u_k||^2 (the second sweep's residual), so k_finalize(k)
  // runs right after it; shifts converged at k are frozen with u_k in buffer X, the rest continue from the
  // pre-smoothed iterate in Y.  The buffers rotate over three (pass input, u_k, pre-smoothed), parity[k]
  // records X for k_pack.  Host pipelining as in the norm-next loop: count(k-1) is read once cycle k is
  // enqueued.  At max_iter the last post-sweep runs alone with the norm.  Every point gets exactly the
  // arithmetic of the unfused cycle (same sweeps, same residual formula), so iterates and histories match.
  void solve_xfuse() {
    Level& F = lv[0];
    Level& Lc = lv[1];
    const int gamma = cfg.cycle == PDMG_CYCLE_W ? 2 : 1;
    int n_act = S;
    // cycle 1's pre-sweep from the zero guess + restriction; its input residual is b, i.e. r0 (finalize(0))
    level_pass(0, Variant{false, false, true, POST_RESTRICT, true, false}, F.u[0], F.u[1], F.b, nullptr, Lc.b,
               d_active, n_act, true);
    finalize(0, last_partials, false, 0);
    F.cur = 1;
    F.uzero = false;
    for (int k = 1;; ++k) {
      for (int g = 0; g < gamma; ++g) cycle_level(1, g == 0, d_active, n_act, false);
      const V* ec = Lc.u[Lc.cur];
      if (k == cfg.max_iter) {
        const int w = (F.cur + 1) % 3;
        level_pass(0, Variant{true, true, true, POST_NORM, true, false}, F.u[F.cur], F.u[w], F.b, ec, nullptr,
                   d_active, n_act);
        finalize(k, last_partials, true, w);
        F.cur = w;
        break;
      }
      const int X = (F.cur + 1) % 3, Y = (F.cur + 2) % 3;
      level_pass2(0, true, true, POST_RESTRICT, F.u[F.cur], F.u[Y], F.b, ec, Lc.b, d_active, n_act, false, F.u[X]);
      finalize(k, last_partials, false, X);
      F.cur = Y;
      n_act = read_nactive(k - 1);
      if (n_act == 0) break;
    }
    F.cur = 0;  // (level state for the op-level entry points)
  }

  // Copy the per-shift report back; counts the smoother updates performed (sum over shifts of cycles).
  void finish_report(pdmg_solve_report* rep, std::chrono::steady_clock::time_point t0, int H) {
    to_host(d_iters, map_iters(), sizeof(int) * S);
    to_host(d_conv, map_conv(), sizeof(int) * S);
    const bool need_hist = rep && (rep->residual_history || rep->rate);
    if (need_hist) to_host(d_hist, map_hist(), sizeof(double) * S * (size_t)H);
    CK(cudaStreamSynchronize(stream));
    CK(cudaGetLastError());
    const int* it = (const int*)(h_map + map_iters());
    const int* cv = (const int*)(h_map + map_conv());
    const double* hist = (const double*)(h_map + map_hist());
    drain_stats();
    // updates per cycle per shift: (nu1+nu2) * sum_l m_l^2 * gamma^l over non-coarsest levels
    double per_cycle = 0.0, visits = 1.0;
    for (size_t l = 0; l + 1 < lv.size(); ++l) {
      per_cycle += (cfg.nu1 + cfg.nu2) * (double)lv[l].m * lv[l].m * visits;
      if (cfg.cycle == PDMG_CYCLE_W) visits *= 2;
    }
    double cycles_done = 0.0;
    for (int s = 0; s < S; ++s) cycles_done += it[s];
    last_updates = per_cycle * cycles_done;
    if (rep) {
      for (int s = 0; s < S; ++s) {
        if (rep->iterations) rep->iterations[s] = it[s];
        if (rep->converged) rep->converged[s] = (uint8_t)cv[s];
        if (rep->residual_history)
          std::memcpy(rep->residual_history + (size_t)s * H, hist + (size_t)s * H, sizeof(double) * H);
        if (rep->rate) rep->rate[s] = measured_rate(hist + (size_t)s * H, it[s]);
      }
      rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  }

  static double measured_rate(const double* hist, int iters) {  // multigrid.cpp:9-21
    if (iters <= 0) return 0.0;
    int count = std::min(5, iters - 1);
    if (count == 0) count = 1;
    double log_sum = 0.0;
    for (int k = iters - count + 1; k <= iters; ++k) {
      if (hist[k] == 0.0) return 0.0;
      if (hist[k - 1] == 0.0) return 0.0;
      log_sum += std::log(hist[k] / hist[k - 1]);
    }
    return std::exp(log_sum / count);
  }

  // ---- host I/O staging --------------------------------------------------------------------
  double2* stage(size_t elems) {
    if (elems > stage_elems) {
      cudaFree(d_stage);
      d_stage = nullptr;
      CK(cudaMalloc(&d_stage, elems * sizeof(double2)));
      stage_elems = elems;
    }
    return d_stage;
  }
  size_t compact_elems(int l) const { return (size_t)S * lv[l].m * lv[l].m; }
  void h2d(const pdmg_c128* src, double2* dst, size_t elems) {
    CK(cudaMemcpyAsync(dst, src, elems * sizeof(double2), cudaMemcpyHostToDevice, stream));
  }
  void d2h(const double2* src, pdmg_c128* dst, size_t elems) {
    CK(cudaMemcpyAsync(dst, src, elems * sizeof(double2), cudaMemcpyDeviceToHost, stream));
  }
  void check_level(int l, int need_coarser) const {
    if (l < 0 || l + need_coarser >= (int)lv.size())
      throw ConfigError("level index " + std::to_string(l) + " out of range for a " + std::to_string(lv.size()) +
                        "-level hierarchy");
  }

  // ---- shift sub-range view: the engine's per-shift arrays offset to shifts [s0, s0 + cnt) ---------------
  int s_base = 0;  // offset of the current view into coarse_singular
  struct RangeView {
    Engine& e;
    int S0;
    std::vector<std::array<V*, 4>> saved_lv;
    std::vector<LevelCoef*> saved_coef;
    std::vector<size_t> saved_elems;
    double2* ainv;
    int *act, *it, *cv, *ones;
    double *r0, *hist;
    RangeView(Engine& en, int s0, int cnt) : e(en), S0(en.S) {
      for (auto& L : e.lv) {
        saved_lv.push_back({L.u[0], L.u[1], L.b, L.u[2]});
        saved_coef.push_back(L.coef);
        saved_elems.push_back(L.elems);
        L.u[0] += s0 * L.ss, L.u[1] += s0 * L.ss, L.b += s0 * L.ss, L.coef += s0;
        if (L.u[2]) L.u[2] += s0 * L.ss;
        L.elems = (size_t)L.ss * cnt + (s0 + cnt == en.S ? L.n + 2 : 0);
      }
      ainv = e.d_ainv, act = e.d_active, it = e.d_iters, cv = e.d_conv, ones = e.d_ones, r0 = e.d_r0, hist = e.d_hist;
      e.d_ainv += (int64_t)s0 * e.coarse_N * e.coarse_N;
      e.d_active += s0, e.d_iters += s0, e.d_conv += s0, e.d_ones += s0, e.d_r0 += s0;
      e.d_hist += (int64_t)s0 * (e.cfg.max_iter + 1);
      e.S = cnt;
      e.s_base = s0;
    }
    ~RangeView() {
      for (size_t l = 0; l < e.lv.size(); ++l) {
        e.lv[l].u[0] = saved_lv[l][0], e.lv[l].u[1] = saved_lv[l][1], e.lv[l].b = saved_lv[l][2];
        e.lv[l].u[2] = saved_lv[l][3];
        e.lv[l].coef = saved_coef[l], e.lv[l].elems = saved_elems[l];
      }
      e.d_ainv = ainv, e.d_active = act, e.d_iters = it, e.d_conv = cv, e.d_ones = ones, e.d_r0 = r0, e.d_hist = hist;
      e.S = S0;
      e.s_base = 0;
    }
  };

  cudaStream_t copy_stream = nullptr;
  int io_chunks = 0;  // 0 = automatic
  int io_mode = 1;    // 1: chunks solve concurrently on sub-engines (own streams, priorities); 0: one stream
  int stream_priority = 0;
  // sub-engine of a concurrent host solve: its level arrays are the shift range [borrow_s0, borrow_s0 + S)
  // of the parent engine's (a contiguous block of the shift-major storage), not allocations of its own
  Engine* borrow = nullptr;
  int borrow_s0 = 0;
  // Sub-engines of the concurrent host-buffer pipeline: shifts [sub_lo[c], sub_lo[c+1]) on their own stream,
  // chunk c at stream priority greatest + c, so chunks finish in order while later chunks fill the SMs the
  // earlier ones leave idle (coarse levels, convergence bookkeeping, tails of the large passes).
  std::vector<std::unique_ptr<Engine<T>>> subs;
  std::vector<int> sub_lo;
  pdmg_batch_desc desc_{};
  bool build_subs(const std::vector<int>& lo) {
    if (subs.size() + 1 == lo.size() && sub_lo == lo) {
      for (auto& e : subs) e->solve_path = solve_path;
      return true;
    }
    subs.clear();
    sub_lo.clear();
    // memory: each sub-engine works in its shift range of this engine's level arrays (borrow); it only
    // allocates its coefficient tables, coarse factors and bookkeeping
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    for (size_t c = 0; c + 1 < lo.size(); ++c) {
      auto e = std::make_unique<Engine<T>>();
      pdmg_batch_desc d = desc_;
      std::vector<pdmg_c128> lam(lo[c + 1] - lo[c]);
      for (int s = lo[c]; s < lo[c + 1]; ++s) lam[s - lo[c]] = pdmg_c128{lambdas[s].real(), lambdas[s].imag()};
      d.n_shifts = lo[c + 1] - lo[c];
      d.lambdas = lam.data();
      e->device = -1;
      e->setup_host(d);
      e->stream_priority = std::min(greatest + (int)c, least);
      e->borrow = this;
      e->borrow_s0 = lo[c];
      e->setup_device(device);
      e->io_chunks = 1;
      e->solve_path = solve_path;
      subs.push_back(std::move(e));
    }
    sub_lo = lo;
    return true;
  }

  // Host-buffer solve.  Large batches are pipelined over chunks of shifts: H2D of later chunks and D2H of
  // earlier ones run on a copy stream while the current chunk solves (results are identical: every shift's
  // solve is independent and its kernels see the same data).
  void solve_host(const pdmg_c128* b, pdmg_c128* u, pdmg_solve_report* rep) override {
    CK(cudaSetDevice(device));
    const size_t N = compact_elems(0);
    const int64_t per = (int64_t)lv[0].m * lv[0].m;
    double2* st = stage(2 * N);
    // automatic: three chunks of S/4, S/2, S/4 shifts.  Each chunk solve carries a fixed ~3 ms of
    // coarse-level latency (C3 on B200: t(S) ~ 2.9 ms + 0.148 ms * S), so few chunks with short end
    // chunks minimise exposed copy + overhead: 62 ms (4 equal) -> ~55 ms for C3 (serial: 78 ms).
    const bool auto_split = io_chunks <= 0;
    int nch = io_chunks > 0 ? io_chunks : (N * sizeof(double2) >= ((size_t)256 << 20) && S >= 8 ? 3 : 1);
    nch = std::max(1, std::min(nch, S));
    auto pinned = [](const void* p) {
      cudaPointerAttributes a{};
      if (cudaPointerGetAttributes(&a, p) != cudaSuccess) return (cudaGetLastError(), false);
      return a.type == cudaMemoryTypeHost;
    };
    if (nch > 1 && !(pinned(b) && pinned(u))) nch = 1;  // pageable copies are host-synchronous: no overlap
    if (nch == 1) {
      h2d(b, st, N);
      solve_device(st, st + N, rep);
      d2h(st + N, u, N);
      CK(cudaStreamSynchronize(stream));
      return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    if (!copy_stream) CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    if (io_mode == 1 && solve_concurrent(b, u, rep, st, N, per)) {
      if (rep) rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      return;
    }
    std::vector<cudaEvent_t> in(nch), done(nch);
    for (int c = 0; c < nch; ++c) {
      CK(cudaEventCreateWithFlags(&in[c], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&done[c], cudaEventDisableTiming));
    }
    auto bound = [&](int c) {
      if (auto_split && nch == 3) return c == 0 ? 0 : c == 1 ? S / 4 : c == 2 ? S - S / 4 : S;
      return (int)((int64_t)S * c / nch);
    };
    auto range = [&](int c) { return std::make_pair(bound(c), bound(c + 1)); };
    for (int c = 0; c < nch; ++c) {
      const auto [s0, s1] = range(c);
      CK(cudaMemcpyAsync(st + s0 * per, b + s0 * per, sizeof(double2) * per * (s1 - s0), cudaMemcpyHostToDevice,
                         copy_stream));
      CK(cudaEventRecord(in[c], copy_stream));
    }
    const int H = cfg.max_iter + 1;
    double upd = 0.0;
    for (int c = 0; c < nch; ++c) {
      const auto [s0, s1] = range(c);
      CK(cudaStreamWaitEvent(stream, in[c], 0));
      pdmg_solve_report rc{};
      if (rep) {
        rc.iterations = rep->iterations ? rep->iterations + s0 : nullptr;
        rc.converged = rep->converged ? rep->converged + s0 : nullptr;
        rc.residual_history = rep->residual_history ? rep->residual_history + (int64_t)s0 * H : nullptr;
        rc.rate = rep->rate ? rep->rate + s0 : nullptr;
      }
      {
        RangeView view(*this, s0, s1 - s0);
        solve_device(st + s0 * per, st + N + s0 * per, rep ? &rc : nullptr);
      }
      upd += last_updates;
      CK(cudaEventRecord(done[c], stream));
      CK(cudaStreamWaitEvent(copy_stream, done[c], 0));
      CK(cudaMemcpyAsync(u + s0 * per, st + N + s0 * per, sizeof(double2) * per * (s1 - s0), cudaMemcpyDeviceToHost,
                         copy_stream));
    }
    CK(cudaStreamSynchronize(copy_stream));
    for (int c = 0; c < nch; ++c) cudaEventDestroy(in[c]), cudaEventDestroy(done[c]);
    last_updates = upd;
    if (rep) rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }

  // Concurrent host pipeline: all H2D copies queue on the copy stream in chunk order; chunk c's host thread
  // waits for its copy, solves on its sub-engine's stream and queues its own D2H there.  Every shift's solve
  // is independent, so the results are bitwise those of one batch (test_chunked_host_solve_matches).
  bool solve_concurrent(const pdmg_c128* b, pdmg_c128* u, pdmg_solve_report* rep, double2* st, size_t N, int64_t per) {
    // automatic: six chunks weighted 1,2,2,2,2,1 -- half-size first and last chunks shorten the exposed fill
    // (first H2D) and drain (last D2H); measured on B200 (C3): 45.9 ms vs 47.4 (1,2,2,2,1), 48.1 (8 equal),
    // 49.4 (1,3,3,1) and 51.4 for the one-stream three-chunk pipeline (io_mode 0)
    int nch = io_chunks > 0 ? io_chunks : 6;
    nch = std::max(2, std::min(nch, S));
    std::vector<int> lo(nch + 1);
    if (io_chunks <= 0 && nch == 6) {
      static const int wt[6] = {1, 2, 2, 2, 2, 1};
      int acc = 0;
      for (int c = 0; c < 6; ++c) acc += wt[c], lo[c + 1] = (int)((int64_t)S * acc / 10);
    } else {
      for (int c = 0; c <= nch; ++c) lo[c] = (int)((int64_t)S * c / nch);
    }
    if (const char* e = std::getenv("PDMG_IO_LAYOUT")) {  // chunk sizes in parts, e.g. "1,2,2,2,1" (tuning)
      std::vector<double> w;
      for (const char* q = e; *q;) {
        char* end = nullptr;
        w.push_back(std::strtod(q, &end));
        q = (*end == ',') ? end + 1 : end;
        if (end == q && *q) break;
      }
      double tw = 0;
      for (double x : w) tw += x;
      lo.assign(w.size() + 1, 0);
      double acc = 0;
      for (size_t c = 0; c < w.size(); ++c) acc += w[c], lo[c + 1] = (int)std::lround(S * acc / tw);
      lo.back() = S;
      nch = (int)w.size();
    }
    for (int c = 0; c < nch; ++c)
      if (lo[c + 1] <= lo[c]) return false;
    if (!build_subs(lo)) return false;
    std::vector<cudaEvent_t> in(nch);
    static const bool dbg = std::getenv("PDMG_IO_DEBUG") != nullptr;
    auto tevent = [&](cudaStream_t st_) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      CK(cudaEventRecord(e, st_));
      return e;
    };
    std::vector<cudaEvent_t> t_in(nch), t_sol(nch), t_out(nch);
    cudaEvent_t t_start = dbg ? tevent(copy_stream) : nullptr;
    for (int c = 0; c < nch; ++c) {
      CK(cudaEventCreateWithFlags(&in[c], dbg ? 0 : cudaEventDisableTiming));
      CK(cudaMemcpyAsync(st + lo[c] * per, b + lo[c] * per, sizeof(double2) * per * (lo[c + 1] - lo[c]),
                         cudaMemcpyHostToDevice, copy_stream));
      CK(cudaEventRecord(in[c], copy_stream));
    }
    const int H = cfg.max_iter + 1;
    std::vector<std::exception_ptr> err(nch);
    std::vector<std::thread> th;
    for (int c = 0; c < nch; ++c) {
      th.emplace_back([&, c] {
        try {
          Engine<T>& e = *subs[c];
          CK(cudaSetDevice(device));
          const int s0 = lo[c], cnt = lo[c + 1] - lo[c];
          CK(cudaStreamWaitEvent(e.stream, in[c], 0));
          pdmg_solve_report rc{};
          if (rep) {
            rc.iterations = rep->iterations ? rep->iterations + s0 : nullptr;
            rc.converged = rep->converged ? rep->converged + s0 : nullptr;
            rc.residual_history = rep->residual_history ? rep->residual_history + (int64_t)s0 * H : nullptr;
            rc.rate = rep->rate ? rep->rate + s0 : nullptr;
          }
          e.solve_device(st + s0 * per, st + N + s0 * per, rep ? &rc : nullptr);
          if (dbg) t_sol[c] = tevent(e.stream);
          CK(cudaMemcpyAsync(u + s0 * per, st + N + s0 * per, sizeof(double2) * per * cnt, cudaMemcpyDeviceToHost,
                             e.stream));
          if (dbg) t_out[c] = tevent(e.stream);
          CK(cudaStreamSynchronize(e.stream));
        } catch (...) {
          err[c] = std::current_exception();
        }
      });
    }
    for (auto& t : th) t.join();
    if (dbg) {
      for (int c = 0; c < nch; ++c) {
        float a = 0, b2 = 0, c2 = 0;
        cudaEventElapsedTime(&a, t_start, in[c]);
        if (t_sol[c]) cudaEventElapsedTime(&b2, t_start, t_sol[c]);
        if (t_out[c]) cudaEventElapsedTime(&c2, t_start, t_out[c]);
        std::fprintf(stderr, "pdmg io chunk %d [%d,%d): in %.2f solved %.2f out %.2f ms\n", c, lo[c], lo[c + 1], a, b2, c2);
        if (t_sol[c]) cudaEventDestroy(t_sol[c]);
        if (t_out[c]) cudaEventDestroy(t_out[c]);
      }
      cudaEventDestroy(t_start);
    }
    for (int c = 0; c < nch; ++c) cudaEventDestroy(in[c]);
    for (auto& x : err)
      if (x) std::rethrow_exception(x);
    double upd = 0.0;
    for (auto& e : subs) upd += e->last_updates, launches += e->launches, e->launches = 0;
    last_updates = upd;
    return true;
  }

  void cycle_host(pdmg_c128* u, const pdmg_c128* b) override {
    CK(cudaSetDevice(device));
    if (any_singular)
      throw SingularOperatorError("DenseShiftedSolver: operator is singular on grid n = " + std::to_string(lv.back().n));
    Level& F = lv[0];
    const size_t N = compact_elems(0);
    double2* st = stage(2 * N);
    h2d(b, st, N);
    h2d(u, st + N, N);
    unpack(st, F.b, 0);
    F.cur = 0;
    unpack(st + N, F.u[0], 0);
    cycle_level(0, false, nullptr, S, false);
    pack(F.u[F.cur], F.u[F.cur], nullptr, nullptr, st + N, 0);
    d2h(st + N, u, N);
    CK(cudaStreamSynchronize(stream));
    CK(cudaGetLastError());
    drain_stats();
  }

  // level operators ----------------------------------------------------------------------------
  void op_smooth(int l, const pdmg_c128* u, const pdmg_c128* b, pdmg_c128* out) override {
    check_level(l, 1);
    CK(cudaSetDevice(device));
    Level& Lv = lv[l];
    const size_t N = compact_elems(l);
    double2* st = stage(2 * N);
    h2d(u, st, N);
    h2d(b, st + N, N);
    unpack(st, Lv.u[0], l);
    unpack(st + N, Lv.b, l);
    level_pass(l, Variant{true, false, true, POST_NONE, true, cfg.smoother == PDMG_SMOOTHER_JACOBI}, Lv.u[0], Lv.u[1],
               Lv.b, nullptr, nullptr, nullptr, S);
    pack(Lv.u[1], Lv.u[1], nullptr, nullptr, st, l);
    d2h(st, out, N);
    finish();
  }
  void op_residual(int l, const pdmg_c128* b, const pdmg_c128* u, pdmg_c128* r) override {
    check_level(l, 0);
    CK(cudaSetDevice(device));
    Level& Lv = lv[l];
    const size_t N = compact_elems(l);
    double2* st = stage(2 * N);
    h2d(u, st, N);
    h2d(b, st + N, N);
    unpack(st, Lv.u[0], l);
    unpack(st + N, Lv.b, l);
    level_pass(l, Variant{true, false, false, POST_RESID, false, false}, Lv.u[0], Lv.u[1], Lv.b, nullptr, nullptr,
               nullptr, S);
    pack(Lv.u[1], Lv.u[1], nullptr, nullptr, st, l);
    d2h(st, r, N);
    finish();
  }
  void op_restrict(int l, const pdmg_c128* fine, pdmg_c128* coarse) override {
    check_level(l, 1);
    CK(cudaSetDevice(device));
    Level &Lv = lv[l], &Lc = lv[l + 1];
    const size_t N = compact_elems(l), Nc = compact_elems(l + 1);
    double2* st = stage(N + Nc);
    h2d(fine, st, N);
    unpack(st, Lv.b, l);
    level_pass(l, Variant{false, false, false, POST_RESTRICT, false, false}, nullptr, nullptr, Lv.b, nullptr, Lc.b,
               nullptr, S);
    pack(Lc.b, Lc.b, nullptr, nullptr, st + N, l + 1);
    d2h(st + N, coarse, Nc);
    finish();
  }
  void op_prolong(int l, const pdmg_c128* coarse, pdmg_c128* fine) override {
    check_level(l, 1);
    CK(cudaSetDevice(device));
    Level &Lv = lv[l], &Lc = lv[l + 1];
    const size_t N = compact_elems(l), Nc = compact_elems(l + 1);
    double2* st = stage(N + Nc);
    h2d(coarse, st + N, Nc);
    unpack(st + N, Lc.u[0], l + 1);
    level_pass(l, Variant{false, true, false, POST_NONE, true, false}, nullptr, Lv.u[1], Lv.b, Lc.u[0], nullptr,
               nullptr, S);
    pack(Lv.u[1], Lv.u[1], nullptr, nullptr, st, l);
    d2h(st, fine, N);
    finish();
  }
  void op_norm(int l, const pdmg_c128* v, double* norms) override {
    check_level(l, 0);
    CK(cudaSetDevice(device));
    Level& Lv = lv[l];
    const size_t N = compact_elems(l);
    double2* st = stage(N);
    h2d(v, st, N);
    unpack(st, Lv.b, l);
    level_pass(l, Variant{false, false, false, POST_NORM, false, false}, nullptr, nullptr, Lv.b, nullptr, nullptr,
               nullptr, S);
    const int threads = 256, blocks = (S * 32 + threads - 1) / threads;
    timed("sum_partials", 0.0,
          [&] { k_sum_partials<<<blocks, threads, 0, stream>>>(d_partial, last_partials, S, d_norms); });
    CK(cudaMemcpyAsync(norms, d_norms, sizeof(double) * S, cudaMemcpyDeviceToHost, stream));
    finish();
  }
  void op_coarse_solve(const pdmg_c128* b, pdmg_c128* u) override {
    CK(cudaSetDevice(device));
    if (any_singular)
      throw SingularOperatorError("DenseShiftedSolver: operator is singular on grid n = " + std::to_string(lv.back().n));
    const int l = (int)lv.size() - 1;
    Level& Lv = lv[l];
    const size_t N = compact_elems(l);
    double2* st = stage(2 * N);
    h2d(b, st, N);
    unpack(st, Lv.b, l);
    coarse_solve(Lv.b, Lv.u[0], nullptr);
    pack(Lv.u[0], Lv.u[0], nullptr, nullptr, st + N, l);
    d2h(st + N, u, N);
    finish();
  }
  void finish() {
    CK(cudaStreamSynchronize(stream));
    CK(cudaGetLastError());
    drain_stats();
  }
};


// ---------------------------------------------------------------------------------------------
// ParaDIAG time direction (alpha-circulant backward Euler), restated: paradiag.cpp:185-248 three-step
// driver with B = C_alpha = (1/dt)(I - Sigma_alpha), diagonalized by an alpha-scaled DFT over time.
// ---------------------------------------------------------------------------------------------
struct DftTables {
  double2* tw = nullptr;  // e^{dir 2 pi i q/nt}
  double2* pre = nullptr;
  double2* post = nullptr;
  int nt = 0, log2nt = -1;
  ~DftTables() {
    cudaFree(tw);
    cudaFree(pre);
    cudaFree(post);
  }
};

// principal value of alpha^p for real alpha != 0 (alpha < 0: |alpha|^p e^{i pi p}, paradiag.cpp:209-213)
cplx real_pow_c(double alpha, double p) {
  if (alpha > 0.0) return cplx(std::pow(alpha, p), 0.0);
  return std::polar(std::pow(-alpha, p), M_PI * p);
}

// step 1: pre = alpha^(t/nt), dir +1, post = 1/nt;  step 3: pre = 1, dir -1, post = alpha^(-t/nt)
std::unique_ptr<DftTables> make_dft_tables(int nt, double alpha, int step, cudaStream_t st) {
  if (nt < 1) throw ConfigError("time DFT: nt must be >= 1");
  auto T = std::make_unique<DftTables>();
  T->nt = nt;
  T->log2nt = ((nt & (nt - 1)) == 0) ? __builtin_ctz((unsigned)nt) : -1;
  std::vector<double2> tw(nt), pre(nt), post(nt);
  const double dir = step == 1 ? 1.0 : -1.0;
  for (int q = 0; q < nt; ++q) {
    const cplx z = std::polar(1.0, dir * 2.0 * M_PI * (double)q / (double)nt);
    tw[q] = make_double2(z.real(), z.imag());
    const cplx sc = real_pow_c(alpha, (double)q / (double)nt);
    const cplx pr = step == 1 ? sc : cplx(1.0, 0.0);
    const cplx po = step == 1 ? cplx(1.0 / nt, 0.0) : cplx(1.0, 0.0) / sc;
    pre[q] = make_double2(pr.real(), pr.imag());
    post[q] = make_double2(po.real(), po.imag());
  }
  CK(cudaMalloc(&T->tw, sizeof(double2) * nt));
  CK(cudaMalloc(&T->pre, sizeof(double2) * nt));
  CK(cudaMalloc(&T->post, sizeof(double2) * nt));
  CK(cudaMemcpyAsync(T->tw, tw.data(), sizeof(double2) * nt, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(T->pre, pre.data(), sizeof(double2) * nt, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(T->post, post.data(), sizeof(double2) * nt, cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  return T;
}

int dft_points_per_cta(int nt) { return std::max(1, std::min(64, 4096 / nt)); }

void launch_time_dft(const DftTables& T, const double2* in, double2* out, int64_t npts, cudaStream_t st) {
  const int P = dft_points_per_cta(T.nt);
  const size_t smem = (size_t)T.nt * P * sizeof(double2);
  static bool attr_set = false;
  if (!attr_set) {
    CK(cudaFuncSetAttribute(k_time_dft, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    attr_set = true;
  }
  const int64_t blocks = (npts + P - 1) / P;
  if (blocks > 0)
    k_time_dft<<<(unsigned)blocks, DFT_THREADS, smem, st>>>(in, out, T.nt, T.log2nt, (int)npts, P, T.tw, T.pre, T.post);
  CK(cudaGetLastError());
}

struct Paradiag {
  int n = 0, nt = 0;
  double alpha = 0, dt = 0;
  int device = 0;
  std::unique_ptr<Engine<double>> eng;
  std::unique_ptr<DftTables> t1, t3;
  double2 *d_f = nullptr, *d_g = nullptr, *d_w = nullptr, *d_u = nullptr;
  double* d_partial = nullptr;
  int res_blocks = 0;
  int64_t npts = 0;

  ~Paradiag() {
    if (eng) cudaSetDevice(device);
    cudaFree(d_f);
    cudaFree(d_g);
    cudaFree(d_w);
    cudaFree(d_u);
    cudaFree(d_partial);
  }

  void setup(int n_, int nt_, double alpha_, double dt_, const pdmg_mg_config& cfg, int dev) {
    if (nt_ < 2) throw ConfigError("TimeDiscretization: need n >= 2 time steps");
    if (!(dt_ > 0.0)) throw ConfigError("TimeDiscretization: tau must be positive");
    if (!(alpha_ != 0.0)) throw ConfigError("alpha-circulant: alpha must be nonzero");
    n = n_, nt = nt_, alpha = alpha_, dt = dt_, device = dev;
    std::vector<pdmg_c128> lam(nt);
    pdmg_circulant_shifts(alpha, nt, dt, 0, nt, lam.data());
    pdmg_batch_desc d{n, nt, lam.data(), cfg, PDMG_PREC_C128, dev};
    eng = std::make_unique<Engine<double>>();
    eng->device = -1;
    eng->setup_host(d);
    eng->setup_device(dev);
    npts = (int64_t)(n - 1) * (n - 1);
    const size_t bytes = sizeof(double2) * (size_t)nt * npts;
    for (double2** p : {&d_f, &d_g, &d_w, &d_u}) CK(cudaMalloc(p, bytes));
    t1 = make_dft_tables(nt, alpha, 1, eng->stream);
    t3 = make_dft_tables(nt, alpha, 3, eng->stream);
    res_blocks = 148 * 8;
    CK(cudaMalloc(&d_partial, sizeof(double) * 2 * res_blocks));
  }

  // f, u: device [nt][npts]; returns relres = ||f - K u|| / ||f|| (paradiag.cpp:243-245)
  void run_device(const double2* f, double2* u, pdmg_solve_report* rep, double* relres) {
    CK(cudaSetDevice(device));
    cudaStream_t st = eng->stream;
    eng->timed("time_dft", 2.0 * sizeof(double2) * nt * npts, [&] { launch_time_dft(*t1, f, d_g, npts, st); });
    eng->solve_device(d_g, d_w, rep);  // step 2: the nt shifted solves (paradiag.cpp:207-236)
    eng->timed("time_dft", 2.0 * sizeof(double2) * nt * npts, [&] { launch_time_dft(*t3, d_w, u, npts, st); });
    if (relres) {
      eng->timed("aao_residual", 3.0 * sizeof(double2) * nt * npts, [&] {
        k_aao_residual<<<res_blocks, 256, 0, st>>>(u, u + (int64_t)(nt - 1) * npts, f, n, nt, 0, alpha, dt, d_partial);
      });
      std::vector<double> part(2 * res_blocks);
      CK(cudaMemcpyAsync(part.data(), d_partial, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      double rr = 0.0, ff = 0.0;
      for (int b = 0; b < res_blocks; ++b) rr += part[2 * b], ff += part[2 * b + 1];
      *relres = ff > 0.0 ? std::sqrt(rr) / std::sqrt(ff) : std::sqrt(rr);
    }
    CK(cudaStreamSynchronize(st));
    eng->drain_stats();
  }

  void run_host(const pdmg_c128* f, pdmg_c128* u, pdmg_solve_report* rep, double* relres) {
    CK(cudaSetDevice(device));
    const size_t bytes = sizeof(double2) * (size_t)nt * npts;
    CK(cudaMemcpyAsync(d_f, f, bytes, cudaMemcpyHostToDevice, eng->stream));
    run_device(d_f, d_u, rep, relres);
    CK(cudaMemcpyAsync(u, d_u, bytes, cudaMemcpyDeviceToHost, eng->stream));
    CK(cudaStreamSynchronize(eng->stream));
  }
};

}  // namespace pdmg_b200

using namespace pdmg_b200;

namespace pdmg_b200 {

// cuBLAS handle per device (created on first use); plain library ZGEMMs for the dense time transforms
cublasHandle_t cublas_for(int device) {
  static std::map<int, cublasHandle_t> handles;
  auto it = handles.find(device);
  if (it != handles.end()) return it->second;
  cublasHandle_t h;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasCreate failed");
  handles[device] = h;
  return h;
}

// Y[nt][npts] = M[nt][nt] X[nt][npts] (row-major, time slowest): column-major Y^T = X^T M^T, i.e.
// ZGEMM(N, N, npts, nt, nt, X, M-as-column-major(=M^T)).
void time_gemm(int device, cudaStream_t st, int nt, int64_t npts, const double2* dM, const double2* dX, double2* dY) {
  cublasHandle_t h = cublas_for(device);
  if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasSetStream failed");
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  const cublasStatus_t s =
      cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)npts, nt, nt, &one, reinterpret_cast<const cuDoubleComplex*>(dX),
                  (int)npts, reinterpret_cast<const cuDoubleComplex*>(dM), nt, &zero,
                  reinterpret_cast<cuDoubleComplex*>(dY), (int)npts);
  if (s != CUBLAS_STATUS_SUCCESS) throw CudaError("cublasZgemm failed (" + std::to_string((int)s) + ")");
}

// paradiag_solve with a general diagonalization B = V diag(lambda) V^{-1} supplied by the caller
// (diagonalize_time_matrix, paradiag.cpp:71-82): g = (V^{-1} (x) I) f, batched shifted solves,
// u = (V (x) I) w, relres = ||f - (B (x) I + I (x) A) u|| / ||f|| (paradiag.cpp:185-248).
void paradiag_general(int n, int nt, const pdmg_c128* lambdas, const pdmg_c128* V, const pdmg_c128* Vinv,
                      const double* B, const pdmg_mg_config& cfg, int device, const pdmg_c128* f, pdmg_c128* u,
                      pdmg_solve_report* rep, double* relres) {
  pdmg_batch_desc d{n, nt, lambdas, cfg, PDMG_PREC_C128, device};
  Engine<double> eng;
  eng.device = -1;
  eng.setup_host(d);
  eng.setup_device(device);
  cudaStream_t st = eng.stream;
  const int64_t npts = (int64_t)(n - 1) * (n - 1);
  const size_t bytes = sizeof(double2) * (size_t)nt * npts;
  double2 *d_f = nullptr, *d_g = nullptr, *d_w = nullptr, *d_u = nullptr, *d_V = nullptr, *d_Vi = nullptr,
          *d_B = nullptr;
  double* d_part = nullptr;
  const int blocks = 148 * 8;
  auto cleanup = [&] {
    cudaFree(d_f), cudaFree(d_g), cudaFree(d_w), cudaFree(d_u), cudaFree(d_V), cudaFree(d_Vi), cudaFree(d_B);
    cudaFree(d_part);
  };
  try {
    for (double2** p : {&d_f, &d_g, &d_w, &d_u}) CK(cudaMalloc(p, bytes));
    for (double2** p : {&d_V, &d_Vi, &d_B}) CK(cudaMalloc(p, sizeof(double2) * nt * nt));
    CK(cudaMalloc(&d_part, sizeof(double) * 2 * blocks));
    std::vector<double2> Bc((size_t)nt * nt);
    for (size_t q = 0; q < Bc.size(); ++q) Bc[q] = make_double2(B[q], 0.0);
    CK(cudaMemcpyAsync(d_V, V, sizeof(double2) * nt * nt, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_Vi, Vinv, sizeof(double2) * nt * nt, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_B, Bc.data(), sizeof(double2) * nt * nt, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_f, f, bytes, cudaMemcpyHostToDevice, st));
    time_gemm(device, st, nt, npts, d_Vi, d_f, d_g);  // step 1 (kron_time_solve, paradiag.cpp:135-139)
    eng.solve_device(d_g, d_w, rep);                   // step 2 (paradiag.cpp:207-236)
    time_gemm(device, st, nt, npts, d_V, d_w, d_u);   // step 3 (kron_time_apply, paradiag.cpp:129-133)
    if (relres) {
      time_gemm(device, st, nt, npts, d_B, d_u, d_g);  // (B (x) I) u
      k_aao_residual_dense<<<blocks, 256, 0, st>>>(d_u, d_g, d_f, n, nt, d_part);
      CK(cudaGetLastError());
      std::vector<double> part(2 * blocks);
      CK(cudaMemcpyAsync(part.data(), d_part, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      double rr = 0.0, ff = 0.0;
      for (int b = 0; b < blocks; ++b) rr += part[2 * b], ff += part[2 * b + 1];
      *relres = ff > 0.0 ? std::sqrt(rr) / std::sqrt(ff) : std::sqrt(rr);
    }
    CK(cudaMemcpyAsync(u, d_u, bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

}  // namespace pdmg_b200

struct pdmg_ctx {
  std::unique_ptr<EngineBase> e;
};

// ---------------------------------------------------------------------------------------------
// extern "C" boundary
// ---------------------------------------------------------------------------------------------
extern "C" {

const char* pdmg_last_error(void) { return g_last_error.c_str(); }
int pdmg_abi_version(void) { return PDMG_B200_ABI_VERSION; }

void pdmg_mg_config_default(pdmg_mg_config* c) {
  c->cycle = PDMG_CYCLE_W;
  c->nu1 = 1;
  c->nu2 = 0;
  c->coarsest_n = 8;
  c->tol = 1e-8;
  c->max_iter = 200;
  c->smoother = PDMG_SMOOTHER_VANKA;
  c->omega = 24.0 / 25.0;
}

int pdmg_create(const pdmg_batch_desc* d, pdmg_ctx** out) {
  return guarded([&] {
    if (!d || !out) throw ConfigError("pdmg_create: NULL argument");
    *out = nullptr;
    std::unique_ptr<EngineBase> e;
    if (d->precision == PDMG_PREC_C128)
      e = std::make_unique<Engine<double>>();
    else if (d->precision == PDMG_PREC_C64)
      e = std::make_unique<Engine<float>>();
    else
      throw ConfigError("pdmg_create: unknown precision " + std::to_string(d->precision));
    e->device = -1;
    e->setup_host(*d);  // all ConfigError / SingularOperatorError paths run before any CUDA call
    e->setup_device(d->device);
    auto* c = new pdmg_ctx;
    c->e = std::move(e);
    *out = c;
  });
}

void pdmg_destroy(pdmg_ctx* c) { delete c; }
int pdmg_num_levels(const pdmg_ctx* c) { return c ? (int)c->e->ln.size() : 0; }
int pdmg_level_n(const pdmg_ctx* c, int l) {
  return (c && l >= 0 && l < (int)c->e->ln.size()) ? c->e->ln[l] : -1;
}
int pdmg_num_shifts(const pdmg_ctx* c) { return c ? c->e->S : 0; }
int pdmg_coarse_singular(const pdmg_ctx* c, int s) {
  return (c && s >= 0 && s < c->e->S) ? (int)c->e->coarse_singular[s] : -1;
}

#define NEED_CTX(c) \
  if (!(c)) throw ConfigError("NULL pdmg_ctx")

int pdmg_solve(pdmg_ctx* c, const pdmg_c128* b, pdmg_c128* u, pdmg_solve_report* rep) {
  return guarded([&] {
    NEED_CTX(c);
    if (!b || !u) throw ConfigError("pdmg_solve: NULL b or u");
    c->e->solve_host(b, u, rep);
  });
}
int pdmg_solve_device(pdmg_ctx* c, const void* d_b, void* d_u, pdmg_solve_report* rep) {
  return guarded([&] {
    NEED_CTX(c);
    if (!d_b || !d_u) throw ConfigError("pdmg_solve_device: NULL b or u");
    c->e->solve_device(static_cast<const double2*>(d_b), static_cast<double2*>(d_u), rep);
  });
}
int pdmg_cycle(pdmg_ctx* c, pdmg_c128* u, const pdmg_c128* b) {
  return guarded([&] {
    NEED_CTX(c);
    c->e->cycle_host(u, b);
  });
}
int pdmg_apply_smoother(pdmg_ctx* c, int l, const pdmg_c128* u, const pdmg_c128* b, pdmg_c128* out) {
  return guarded([&] {
    NEED_CTX(c);
    c->e->op_smooth(l, u, b, out);
  });
}
int pdmg_residual(pdmg_ctx* c, int l, const pdmg_c128* b, const pdmg_c128* u, pdmg_c128* r) {
  return guarded([&] {
    NEED_CTX(c);
    c->e->op_residual(l, b, u, r);
  });
}
int pdmg_restrict_full_weighting(pdmg_ctx* c, int l, const pdmg_c128* f, pdmg_c128* co) {
  return guarded([&] {
    NEED_CTX(c);
    c->e->op_restrict(l, f, co);
  });
}
int pdmg_prolong_bilinear(pdmg_ctx* c, int l, const pdmg_c128* co, pdmg_c128* f) {
  return guarded([&] {
    NEED_CTX(c);
    c->e->op_prolong(l, co, f);
  });
}
int pdmg_norm(pdmg_ctx* c, int l, const pdmg_c128* v, double* norms) {
  return guarded([&] {
    NEED_CTX(c);
    c->e->op_norm(l, v, norms);
  });
}
int pdmg_coarse_solve(pdmg_ctx* c, const pdmg_c128* b, pdmg_c128* u) {
  return guarded([&] {
    NEED_CTX(c);
    c->e->op_coarse_solve(b, u);
  });
}

void pdmg_random_rhs(uint32_t seed, double lo, double hi, int64_t count, pdmg_c128* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (int64_t k = 0; k < count; ++k) {
    const double re = dist(rng), im = dist(rng);
    out[k].re = re;
    out[k].im = im;
  }
}

void pdmg_circulant_shifts(double alpha, int32_t nt, double dt, int32_t j0, int32_t count, pdmg_c128* out) {
  const cplx g = real_pow_c(alpha, 1.0 / nt);
  for (int q = 0; q < count; ++q) {
    const double ang = 2.0 * M_PI * (double)(j0 + q) / (double)nt;
    const cplx lam = (cplx(1.0, 0.0) - g * std::exp(cplx(0.0, ang))) / dt;
    out[q].re = lam.real();
    out[q].im = lam.imag();
  }
}

void* pdmg_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
  return p;
}
void pdmg_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

void* pdmg_stream(pdmg_ctx* c) { return c ? (void*)c->e->stream : nullptr; }
int pdmg_set_solve_path(pdmg_ctx* c, int path) {
  if (!c || path < 0 || path > 2) return PDMG_ERR_CONFIG;
  c->e->solve_path = path;
  return PDMG_OK;
}
int pdmg_set_profiling(pdmg_ctx* c, int on) {
  if (!c) return PDMG_ERR_CONFIG;
  c->e->profiling = on != 0;
  return PDMG_OK;
}
void pdmg_reset_stats(pdmg_ctx* c) {
  if (!c) return;
  c->e->stats.clear();
  c->e->launches = 0;
}
int64_t pdmg_launch_count(const pdmg_ctx* c) { return c ? c->e->launches : 0; }
int pdmg_kernel_updates(const pdmg_ctx* c, int i, double* unit_bytes, double* updates) {
  if (!c || i < 0 || i >= (int)c->e->stats.size()) return 1;
  auto it = c->e->stats.begin();
  std::advance(it, i);
  if (unit_bytes) *unit_bytes = it->second.ubytes;
  if (updates) *updates = it->second.updates;
  return 0;
}
int pdmg_kernel_stats(const pdmg_ctx* c, int i, char* name, size_t name_len, int64_t* launches, double* total_ms,
                      double* algo_bytes) {
  if (!c || i < 0 || i >= (int)c->e->stats.size()) return 1;
  auto it = c->e->stats.begin();
  std::advance(it, i);
  if (name && name_len) {
    std::strncpy(name, it->first.c_str(), name_len - 1);
    name[name_len - 1] = 0;
  }
  if (launches) *launches = it->second.launches;
  if (total_ms) *total_ms = it->second.ms;
  if (algo_bytes) *algo_bytes = it->second.bytes;
  return 0;
}
double pdmg_last_updates(const pdmg_ctx* c) { return c ? c->e->last_updates : 0.0; }

struct pdmg_paradiag {
  Paradiag p;
  pdmg_ctx* solver = nullptr;  // non-owning view of p.eng for the stats API
};

int pdmg_paradiag_create(int32_t n, int32_t nt, double alpha, double dt, const pdmg_mg_config* cfg, int32_t device,
                         pdmg_paradiag** out) {
  return guarded([&] {
    if (!cfg || !out) throw ConfigError("pdmg_paradiag_create: NULL argument");
    *out = nullptr;
    auto* P = new pdmg_paradiag;
    try {
      P->p.setup(n, nt, alpha, dt, *cfg, device);
    } catch (...) {
      delete P;
      throw;
    }
    P->solver = new pdmg_ctx;
    P->solver->e.reset(P->p.eng.get());
    *out = P;
  });
}
void pdmg_paradiag_destroy(pdmg_paradiag* P) {
  if (!P) return;
  if (P->solver) {
    P->solver->e.release();
    delete P->solver;
  }
  delete P;
}
pdmg_ctx* pdmg_paradiag_solver(pdmg_paradiag* P) { return P ? P->solver : nullptr; }
int pdmg_paradiag_run(pdmg_paradiag* P, const pdmg_c128* f, pdmg_c128* u, pdmg_solve_report* rep, double* relres) {
  return guarded([&] {
    if (!P || !f || !u) throw ConfigError("pdmg_paradiag_run: NULL argument");
    P->p.run_host(f, u, rep, relres);
  });
}
int pdmg_paradiag_run_device(pdmg_paradiag* P, const void* d_f, void* d_u, pdmg_solve_report* rep, double* relres) {
  return guarded([&] {
    if (!P || !d_f || !d_u) throw ConfigError("pdmg_paradiag_run_device: NULL argument");
    P->p.run_device(static_cast<const double2*>(d_f), static_cast<double2*>(d_u), rep, relres);
  });
}

int pdmg_paradiag_circulant(int32_t n, int32_t nt, double alpha, double dt, const pdmg_mg_config* cfg, int32_t device,
                            const pdmg_c128* f, pdmg_c128* u, pdmg_solve_report* rep, double* relres) {
  pdmg_paradiag* P = nullptr;
  int st = pdmg_paradiag_create(n, nt, alpha, dt, cfg, device, &P);
  if (st) return st;
  st = pdmg_paradiag_run(P, f, u, rep, relres);
  pdmg_paradiag_destroy(P);
  return st;
}

int pdmg_paradiag_general(int32_t n, int32_t nt, const pdmg_c128* lambdas, const pdmg_c128* V, const pdmg_c128* Vinv,
                          const double* B, const pdmg_mg_config* cfg, int32_t device, const pdmg_c128* f, pdmg_c128* u,
                          pdmg_solve_report* report, double* relres) {
  return guarded([&] {
    if (!lambdas || !V || !Vinv || !B || !cfg || !f || !u) throw ConfigError("pdmg_paradiag_general: NULL argument");
    if (nt < 1) throw ConfigError("paradiag_solve: empty right-hand side");
    paradiag_general(n, nt, lambdas, V, Vinv, B, *cfg, device, f, u, report, relres);
  });
}

int pdmg_time_transform(int32_t device, int32_t nt, int64_t npts, const pdmg_c128* M, const void* d_in, void* d_out,
                        void* stream) {
  return guarded([&] {
    if (!M || !d_in || !d_out) throw ConfigError("pdmg_time_transform: NULL argument");
    CK(cudaSetDevice(device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double2* dM = nullptr;
    CK(cudaMalloc(&dM, sizeof(double2) * nt * nt));
    CK(cudaMemcpyAsync(dM, M, sizeof(double2) * nt * nt, cudaMemcpyHostToDevice, st));
    try {
      time_gemm(device, st, nt, npts, dM, static_cast<const double2*>(d_in), static_cast<double2*>(d_out));
      CK(cudaStreamSynchronize(st));
    } catch (...) {
      cudaFree(dM);
      throw;
    }
    cudaFree(dM);
  });
}

int pdmg_time_dft(int32_t device, int32_t nt, int64_t npts, double alpha, int32_t step, const void* d_in, void* d_out,
                  void* stream) {
  return guarded([&] {
    if (step != 1 && step != 3) throw ConfigError("pdmg_time_dft: step must be 1 (forward transform) or 3 (back)");
    if (!(alpha != 0.0)) throw ConfigError("alpha-circulant: alpha must be nonzero");
    CK(cudaSetDevice(device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto T = make_dft_tables(nt, alpha, step, st);
    launch_time_dft(*T, static_cast<const double2*>(d_in), static_cast<double2*>(d_out), npts, st);
    CK(cudaStreamSynchronize(st));
  });
}

int pdmg_aao_residual(int32_t device, int32_t n, int32_t ntl, int32_t t0, double alpha, double dt, const void* d_u,
                      const void* d_u_prev, const void* d_f, double* sums, void* stream) {
  return guarded([&] {
    if (!sums) throw ConfigError("pdmg_aao_residual: NULL sums");
    CK(cudaSetDevice(device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int blocks = 148 * 8;
    double* part = nullptr;
    CK(cudaMalloc(&part, sizeof(double) * 2 * blocks));
    k_aao_residual<<<blocks, 256, 0, st>>>(static_cast<const double2*>(d_u), static_cast<const double2*>(d_u_prev),
                                           static_cast<const double2*>(d_f), n, ntl, t0, alpha, dt, part);
    std::vector<double> h(2 * blocks);
    CK(cudaMemcpyAsync(h.data(), part, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFree(part);
    sums[0] = sums[1] = 0.0;
    for (int b = 0; b < blocks; ++b) sums[0] += h[2 * b], sums[1] += h[2 * b + 1];
  });
}

}  // extern "C"
