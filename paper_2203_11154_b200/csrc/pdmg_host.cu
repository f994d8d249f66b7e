// pdmg_host.cu -- host setup math of libpdmg_b200.so (restating the reference formulas in fp64).
#include "pdmg_host.h"

namespace pdmg_b200 {

thread_local std::string g_last_error;

// ---------------------------------------------------------------------------------------------
// Host-side setup math (fp64), restating the reference formulas.
// ---------------------------------------------------------------------------------------------

cplx checked_inverse(cplx z, const char* what) {  // smoother.cpp:8-15
  if (std::abs(z) <= kSingularTol)
    throw SingularOperatorError(std::string("vanka_coeffs: patch eigenvalue ") + what + " is singular for this shift");
  return cplx(1.0, 0.0) / z;
}

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
  // A is banded (lower bandwidth m; with partial pivoting U's upper bandwidth grows to 2m): the loops skip
  // only exact zeros, so factors and pivots are those of the dense elimination (dense.cpp:82-88)
  for (int k = 0; k < N; ++k) {
    const int rmax = std::min(N - 1, k + m), cmax = std::min(N - 1, k + 2 * m);
    int p = k;
    double best = std::abs(A[(size_t)k * N + k]);
    for (int r = k + 1; r <= rmax; ++r)
      if (std::abs(A[(size_t)r * N + k]) > best) best = std::abs(A[(size_t)r * N + k]), p = r;
    piv[k] = p;
    if (p != k)
      for (int c = 0; c < N; ++c) std::swap(A[(size_t)k * N + c], A[(size_t)p * N + c]);
    const cplx pv = A[(size_t)k * N + k];
    min_pivot = std::min(min_pivot, std::abs(pv));
    if (pv == cplx(0.0, 0.0)) continue;
    for (int r = k + 1; r <= rmax; ++r) {
      const cplx f = A[(size_t)r * N + k] / pv;
      A[(size_t)r * N + k] = f;
      for (int c = k + 1; c <= cmax; ++c) A[(size_t)r * N + c] -= f * A[(size_t)k * N + c];
    }
  }
  CoarseFactor cf;
  cf.singular = !(min_pivot > 1e-14 * fro);
  cf.inv.assign(static_cast<size_t>(N) * N, cplx(0.0, 0.0));
  if (cf.singular) return cf;
  // A^{-1} column by column; L rows (row swaps applied to the stored multipliers) and U rows are sparse:
  // loop over each row's nonzero span only
  std::vector<int> lfirst(N), ulast(N);
  for (int r = 0; r < N; ++r) {
    int c = 0;
    while (c < r && A[(size_t)r * N + c] == cplx(0.0, 0.0)) ++c;
    lfirst[r] = c;
    int e = N - 1;
    while (e > r && A[(size_t)r * N + e] == cplx(0.0, 0.0)) --e;
    ulast[r] = e;
  }
  std::vector<cplx> x(N);
  for (int col = 0; col < N; ++col) {
    std::fill(x.begin(), x.end(), cplx(0.0, 0.0));
    x[col] = 1.0;
    for (int k = 0; k < N; ++k)
      if (piv[k] != k) std::swap(x[k], x[piv[k]]);
    int first = 0;
    while (first < N && x[first] == cplx(0.0, 0.0)) ++first;
    for (int r = first; r < N; ++r)
      for (int c = std::max(lfirst[r], first); c < r; ++c) x[r] -= A[(size_t)r * N + c] * x[c];
    for (int r = N - 1; r >= 0; --r) {
      for (int c = r + 1; c <= ulast[r]; ++c) x[r] -= A[(size_t)r * N + c] * x[c];
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

cplx real_pow_c(double alpha, double p) {
  if (alpha > 0.0) return cplx(std::pow(alpha, p), 0.0);
  return std::polar(std::pow(-alpha, p), M_PI * p);
}

std::unique_ptr<EngineBase> make_engine(int precision) {
  if (precision == PDMG_PREC_C128) return make_engine_c128();
  if (precision == PDMG_PREC_C64) return make_engine_c64();
  throw ConfigError("pdmg_create: unknown precision " + std::to_string(precision));
}

}  // namespace pdmg_b200
