// pdmg_b200.hpp -- header-only C++ facade over the C ABI (pdmg_b200.h), restoring the reference's
// pdmg:: class shapes and exception types so reference call sites port with a namespace change:
//
//   reference (proj/include/pdmg/...)                       this facade
//   Grid2D, Shift                 (grid.hpp:16-52)          pdmg_b200::Grid2D, Shift
//   SmootherConfig                (smoother.hpp:30-38)      pdmg_b200::SmootherConfig
//   MultigridConfig, SolveReport  (multigrid.hpp:14-44)     pdmg_b200::MultigridConfig, SolveReport
//   MultigridHierarchy            (multigrid.hpp:50-78)     pdmg_b200::BatchedMultigridHierarchy (n shifts)
//   multigrid_solve               (multigrid.hpp:82-83)     pdmg_b200::multigrid_solve
//   ConfigError, SingularOperatorError (errors.hpp:12-23)   same names, same std:: bases
//
// Grid functions are std::vector<std::complex<double>> in the reference layout (interior nodes, x
// fastest), stacked shift-major for batches.
#pragma once

#include <complex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pdmg_b200.h"

namespace pdmg_b200 {

using cplx = std::complex<double>;
static_assert(sizeof(cplx) == sizeof(pdmg_c128), "std::complex<double> must match pdmg_c128");

class ConfigError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class SingularOperatorError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int status) {
  if (status == PDMG_OK) return;
  const std::string msg = pdmg_last_error();
  if (status == PDMG_ERR_CONFIG) throw ConfigError(msg);
  if (status == PDMG_ERR_SINGULAR) throw SingularOperatorError(msg);
  throw DeviceError(msg);
}

struct Grid2D {
  int n = 0;
  Grid2D() = default;
  explicit Grid2D(int subdivisions) : n(subdivisions) {
    if (n < 2) throw ConfigError("Grid2D: need at least 2 subdivisions per side, got " + std::to_string(n));
  }
  double h() const { return 1.0 / n; }
  int interior_per_side() const { return n - 1; }
  long size() const { return static_cast<long>(n - 1) * (n - 1); }
};

struct Shift {
  cplx lambda{0.0, 0.0};
  int index = 0;
};

enum class CycleKind { V = PDMG_CYCLE_V, W = PDMG_CYCLE_W };
enum class SmootherKind { Vanka = PDMG_SMOOTHER_VANKA, Jacobi = PDMG_SMOOTHER_JACOBI };

struct SmootherConfig {
  SmootherKind kind = SmootherKind::Vanka;
  double omega = 24.0 / 25.0;
  static SmootherConfig vanka(double w = 24.0 / 25.0) { return {SmootherKind::Vanka, w}; }
  static SmootherConfig jacobi(double w = 4.0 / 5.0) { return {SmootherKind::Jacobi, w}; }
};

struct MultigridConfig {
  CycleKind cycle = CycleKind::W;
  int nu1 = 1;
  int nu2 = 0;
  int coarsest_n = 8;
  double tol = 1e-8;
  int max_iter = 200;
  SmootherConfig smoother{};

  pdmg_mg_config c() const {
    return pdmg_mg_config{static_cast<int32_t>(cycle), nu1, nu2, coarsest_n, tol, max_iter,
                          static_cast<int32_t>(smoother.kind), smoother.omega};
  }
};

struct SolveReport {
  bool converged = false;
  int iterations = 0;
  std::vector<double> residual_history;
  double rate = 0.0;
  double seconds = 0.0;
};

// One hierarchy per shift on a shared fine grid, all advanced together on one GPU.
class BatchedMultigridHierarchy {
 public:
  BatchedMultigridHierarchy(Grid2D fine, const std::vector<Shift>& shifts, const MultigridConfig& cfg, int device = 0)
      : BatchedMultigridHierarchy(fine, shifts, cfg, std::vector<int>{}, device) {}
  // Shifts sharded over `devices` (the reference's `threads` argument of paradiag_solve, paradiag.cpp:207-236):
  // contiguous chunks of ceil(S / devices.size()), one engine and host thread per device.
  BatchedMultigridHierarchy(Grid2D fine, const std::vector<Shift>& shifts, const MultigridConfig& cfg,
                            const std::vector<int>& devices, int device = 0)
      : grid_(fine), cfg_(cfg), S_(static_cast<int>(shifts.size())) {
    std::vector<pdmg_c128> lam(shifts.size());
    for (size_t s = 0; s < shifts.size(); ++s) lam[s] = {shifts[s].lambda.real(), shifts[s].lambda.imag()};
    std::vector<int32_t> devs(devices.begin(), devices.end());
    pdmg_batch_desc d{fine.n, S_, lam.data(), cfg.c(), PDMG_PREC_C128, device,
                      devs.empty() ? nullptr : devs.data(), static_cast<int32_t>(devs.size())};
    check(pdmg_create(&d, &ctx_));
  }
  ~BatchedMultigridHierarchy() { pdmg_destroy(ctx_); }
  BatchedMultigridHierarchy(const BatchedMultigridHierarchy&) = delete;
  BatchedMultigridHierarchy& operator=(const BatchedMultigridHierarchy&) = delete;

  int num_levels() const { return pdmg_num_levels(ctx_); }
  Grid2D level_grid(int ell) const { return Grid2D(pdmg_level_n(ctx_, ell)); }
  int num_shifts() const { return S_; }

  // MultigridHierarchy::solve for every shift (multigrid.cpp:85-110); u is overwritten.
  std::vector<SolveReport> solve(std::vector<cplx>& u, const std::vector<cplx>& b) const {
    const size_t N = static_cast<size_t>(S_) * grid_.size();
    if (b.size() != N) throw ConfigError("MultigridHierarchy::solve: grid mismatch");
    u.resize(N);
    const int H = cfg_.max_iter + 1;
    std::vector<int32_t> it(S_);
    std::vector<uint8_t> cv(S_);
    std::vector<double> hist(static_cast<size_t>(S_) * H), rate(S_);
    pdmg_solve_report rep{it.data(), cv.data(), hist.data(), rate.data(), 0.0};
    check(pdmg_solve(ctx_, reinterpret_cast<const pdmg_c128*>(b.data()), reinterpret_cast<pdmg_c128*>(u.data()),
                     &rep));
    std::vector<SolveReport> out(S_);
    for (int s = 0; s < S_; ++s) {
      out[s].converged = cv[s] != 0;
      out[s].iterations = it[s];
      out[s].residual_history.assign(hist.begin() + static_cast<long>(s) * H,
                                     hist.begin() + static_cast<long>(s) * H + it[s] + 1);
      out[s].rate = rate[s];
      out[s].seconds = rep.seconds;
    }
    return out;
  }

  // MultigridHierarchy::cycle (multigrid.cpp:79-83), in place for every shift.
  void cycle(std::vector<cplx>& u, const std::vector<cplx>& b) const {
    check(pdmg_cycle(ctx_, reinterpret_cast<pdmg_c128*>(u.data()), reinterpret_cast<const pdmg_c128*>(b.data())));
  }

  int num_parts() const { return pdmg_num_parts(ctx_); }
  pdmg_ctx* handle() const { return ctx_; }

 private:
  Grid2D grid_;
  MultigridConfig cfg_;
  int S_;
  pdmg_ctx* ctx_ = nullptr;
};

// multigrid.cpp:112-118 convenience driver for one shift.
inline std::pair<std::vector<cplx>, SolveReport> multigrid_solve(const std::vector<cplx>& b, Grid2D g,
                                                                  const Shift& shift, const MultigridConfig& cfg,
                                                                  int device = 0) {
  BatchedMultigridHierarchy mg(g, {shift}, cfg, device);
  std::vector<cplx> u;
  auto reps = mg.solve(u, b);
  return {std::move(u), reps[0]};
}

// tools/pdmg.cpp:137-147
inline std::vector<cplx> random_rhs(Grid2D g, unsigned seed) {
  std::vector<cplx> b(static_cast<size_t>(g.size()));
  pdmg_random_rhs(seed, -1.0, 1.0, g.size(), reinterpret_cast<pdmg_c128*>(b.data()));
  return b;
}

// ---- ParaDIAG (proj/include/pdmg/paradiag.hpp:95-113) -------------------------------------------------------------
// ParadiagResult without the Eigen members: u (time slices stacked, reference layout), the per-slot shifts and
// reports (in the order of the time matrix's eigenvalues), all_converged, relative_residual, seconds.
struct ParadiagResult {
  std::vector<cplx> u;
  std::vector<Shift> shifts;
  std::vector<SolveReport> reports;
  bool all_converged = false;
  double relative_residual = 0.0;
  double seconds = 0.0;
};

namespace detail {
inline ParadiagResult run_paradiag(pdmg_paradiag* p, const std::vector<cplx>& f, long slices, int max_iter) {
  ParadiagResult r;
  r.u.resize(f.size());
  const int H = max_iter + 1;
  std::vector<int32_t> it(slices);
  std::vector<uint8_t> cv(slices);
  std::vector<double> hist(static_cast<size_t>(slices) * H), rate(slices);
  pdmg_solve_report rep{it.data(), cv.data(), hist.data(), rate.data(), 0.0};
  const int st = pdmg_paradiag_run(p, reinterpret_cast<const pdmg_c128*>(f.data()),
                                   reinterpret_cast<pdmg_c128*>(r.u.data()), &rep, &r.relative_residual);
  pdmg_paradiag_destroy(p);
  check(st);
  r.reports.resize(slices);
  r.all_converged = true;
  for (long s = 0; s < slices; ++s) {
    SolveReport& q = r.reports[s];
    q.converged = cv[s] != 0, q.iterations = it[s], q.rate = rate[s], q.seconds = rep.seconds;
    q.residual_history.assign(hist.begin() + s * H, hist.begin() + s * H + it[s] + 1);
    r.all_converged = r.all_converged && q.converged;
  }
  r.seconds = rep.seconds;
  return r;
}
}  // namespace detail

// paradiag_solve (paradiag.cpp:185-248) for the alpha-circulant time matrix C_alpha = (1/tau)(I - Sigma_alpha):
// the BASELINE preconditioner (alpha > 0) or, with alpha = -1/beta, the reference's BackwardHeatQBV (whose reports
// this returns in the reference's eigenvalue order, paradiag.cpp:84-108).  f: `slices` time slices of the fine grid
// stacked; devices: the reference's `threads` (time slices sharded over the devices, transforms through peer memory).
inline ParadiagResult paradiag_solve_circulant(const std::vector<cplx>& f, Grid2D g, int slices, double alpha,
                                               double tau, const MultigridConfig& cfg,
                                               const std::vector<int>& devices = {0}) {
  if (slices < 1 || f.size() != static_cast<size_t>(slices) * g.size())
    throw ConfigError("paradiag_solve: expected " + std::to_string(slices) + " time slices");
  const pdmg_mg_config c = cfg.c();
  std::vector<int32_t> devs(devices.begin(), devices.end());
  pdmg_paradiag* p = nullptr;
  check(pdmg_paradiag_create_multi(g.n, slices, alpha, tau, &c, devs.data(), static_cast<int32_t>(devs.size()), &p));
  ParadiagResult r = detail::run_paradiag(p, f, slices, cfg.max_iter);
  std::vector<pdmg_c128> lam(slices);
  pdmg_circulant_shifts(alpha, slices, tau, 0, slices, lam.data());
  r.shifts.resize(slices);
  for (int k = 0; k < slices; ++k) r.shifts[k] = Shift{cplx(lam[k].re, lam[k].im), k};
  if (alpha < 0) {  // QBV: reference index k is circulant slot (m - k) mod m
    std::vector<SolveReport> reps(slices);
    std::vector<Shift> sh(slices);
    for (int k = 0; k < slices; ++k) {
      const int q = (slices - k) % slices;
      reps[k] = r.reports[q], sh[k] = Shift{r.shifts[q].lambda, k};
    }
    r.reports.swap(reps), r.shifts.swap(sh);
  }
  return r;
}

// paradiag_solve with a general diagonalization B = V diag(lambdas) V^{-1} supplied by the caller (HeatBVM:
// diagonalize_time_matrix, paradiag.cpp:71-82); V, Vinv complex and B real, nt x nt row-major.
inline ParadiagResult paradiag_solve_general(const std::vector<cplx>& f, Grid2D g, const std::vector<cplx>& lambdas,
                                             const std::vector<cplx>& V, const std::vector<cplx>& Vinv,
                                             const std::vector<double>& B, const MultigridConfig& cfg,
                                             const std::vector<int>& devices = {0}) {
  const int nt = static_cast<int>(lambdas.size());
  if (nt < 1 || f.size() != static_cast<size_t>(nt) * g.size() || V.size() != static_cast<size_t>(nt) * nt ||
      Vinv.size() != V.size() || B.size() != V.size())
    throw ConfigError("paradiag_solve: inconsistent time-matrix or right-hand-side sizes");
  const pdmg_mg_config c = cfg.c();
  std::vector<int32_t> devs(devices.begin(), devices.end());
  pdmg_paradiag* p = nullptr;
  check(pdmg_paradiag_create_general(g.n, nt, reinterpret_cast<const pdmg_c128*>(lambdas.data()),
                                     reinterpret_cast<const pdmg_c128*>(V.data()),
                                     reinterpret_cast<const pdmg_c128*>(Vinv.data()), B.data(), &c, devs.data(),
                                     static_cast<int32_t>(devs.size()), &p));
  ParadiagResult r = detail::run_paradiag(p, f, nt, cfg.max_iter);
  r.shifts.resize(nt);
  for (int k = 0; k < nt; ++k) r.shifts[k] = Shift{lambdas[k], k};
  return r;
}

}  // namespace pdmg_b200
