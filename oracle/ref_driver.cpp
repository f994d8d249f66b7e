// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.  Builds oracle/_ref/libpdmg_ref.so from the
// reference's OWN, UNMODIFIED sources proj/src/grid.cpp + proj/src/smoother.cpp (compiled where they
// lie under /root/reference by oracle/Makefile; nothing is copied).  The reference's multigrid.cpp,
// dense.cpp and paradiag.cpp need Eigen, which is absent, so the driver below restates
// MultigridHierarchy (proj/src/multigrid.cpp:9-118) and the thread pool (proj/src/paradiag.cpp:217-236)
// over the reference's pdmg::GridFunction, and uses the oracle's partial-pivot LU for the coarsest
// level in place of Eigen::PartialPivLU (proj/src/dense.cpp:82-100).
//
// Used to (1) pin oracle/pdmg_oracle.c bit-for-bit against the reference operators and (2) generate
// tests/golden/ fixtures, and (3) as bench.py's CPU baseline (kind "reference").
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "pdmg/grid.hpp"
#include "pdmg/smoother.hpp"

extern "C" {
#include "pdmg_oracle.h"
}

using namespace pdmg;

namespace {
thread_local std::string g_err;

struct Cfg {  // MultigridConfig, proj/include/pdmg/multigrid.hpp:14-32
  int cycle, nu1, nu2, coarsest_n, max_iter, smoother;
  double tol, omega;
};

GridFunction load(const Grid2D& g, const double* p) {
  GridFunction f(g);
  std::memcpy(f.data(), p, sizeof(cplx) * static_cast<size_t>(g.size()));
  return f;
}
void store(const GridFunction& f, double* p) {
  std::memcpy(p, f.data(), sizeof(cplx) * static_cast<size_t>(f.size()));
}

class Coarse {  // DenseShiftedSolver, restated without Eigen
 public:
  Coarse(Grid2D g, cplx lambda) : g_(g) {
    orc_dense_factor(g.n, orc_cplx_from(lambda), &d_);
  }
  ~Coarse() { orc_dense_free(&d_); }
  GridFunction solve(const GridFunction& b) const {
    if (d_.singular)
      throw SingularOperatorError("DenseShiftedSolver: operator is singular on grid n = " + std::to_string(g_.n));
    GridFunction x(g_);
    orc_dense_solve(&d_, reinterpret_cast<const orc_cplx*>(b.data()), reinterpret_cast<orc_cplx*>(x.data()));
    return x;
  }

 private:
  static orc_cplx orc_cplx_from(cplx z) {
    orc_cplx r;
    std::memcpy(&r, &z, sizeof r);
    return r;
  }
  Grid2D g_;
  orc_dense d_{};
};

class Hierarchy {  // MultigridHierarchy, proj/src/multigrid.cpp:24-110
 public:
  Hierarchy(Grid2D fine, const Shift& s, const Cfg& c) : shift_(s), cfg_(c) {
    if (cfg_.nu1 < 0 || cfg_.nu2 < 0) throw ConfigError("MultigridConfig: negative smoothing counts");
    if (cfg_.nu1 + cfg_.nu2 == 0) throw ConfigError("MultigridConfig: nu1 + nu2 must be positive");
    if (cfg_.coarsest_n < 2) throw ConfigError("MultigridConfig: coarsest_n must be >= 2");
    if (!(cfg_.tol > 0.0)) throw ConfigError("MultigridConfig: tol must be positive");
    if (cfg_.max_iter < 1) throw ConfigError("MultigridConfig: max_iter must be >= 1");
    if (fine.n < cfg_.coarsest_n)
      throw ConfigError("MultigridHierarchy: fine grid n = " + std::to_string(fine.n) +
                        " is finer than coarsest_n = " + std::to_string(cfg_.coarsest_n) + " allows");
    Grid2D g = fine;
    levels_.push_back(g);
    while (g.n > cfg_.coarsest_n) {
      if (!g.coarsenable())
        throw ConfigError("MultigridHierarchy: grid n = " + std::to_string(g.n) +
                          " cannot be coarsened to reach coarsest_n = " + std::to_string(cfg_.coarsest_n));
      g = g.coarse();
      levels_.push_back(g);
    }
    if (g.n != cfg_.coarsest_n)
      throw ConfigError("MultigridHierarchy: coarsening from n = " + std::to_string(fine.n) + " reaches n = " +
                        std::to_string(g.n) + ", not coarsest_n = " + std::to_string(cfg_.coarsest_n));
    sm_ = cfg_.smoother == 0 ? SmootherConfig::vanka(cfg_.omega) : SmootherConfig::jacobi(cfg_.omega);
    for (size_t l = 0; l + 1 < levels_.size(); ++l) {
      const double h = levels_[l].h();
      try {
        if (sm_.kind == SmootherKind::Vanka)
          (void)vanka_coeffs(shift_.eta(h));
        else
          (void)jacobi_weight(shift_.eta(h), h);
      } catch (const SingularOperatorError& e) {
        throw SingularOperatorError("level " + std::to_string(l) + " (n = " + std::to_string(levels_[l].n) +
                                    "): " + e.what());
      }
    }
    coarse_ = std::make_unique<Coarse>(levels_.back(), shift_.lambda);
  }

  void cycle_on_level(size_t l, GridFunction& u, const GridFunction& b) const {
    if (l + 1 == levels_.size()) {
      u = coarse_->solve(b);
      return;
    }
    for (int k = 0; k < cfg_.nu1; ++k) u = apply_smoother(u, b, shift_, sm_);
    GridFunction rc = restrict_full_weighting(residual(b, u, shift_));
    GridFunction ec(levels_[l + 1]);
    const int gamma = cfg_.cycle == 1 ? 2 : 1;
    for (int g = 0; g < gamma; ++g) cycle_on_level(l + 1, ec, rc);
    u += prolong_bilinear(ec);
    for (int k = 0; k < cfg_.nu2; ++k) u = apply_smoother(u, b, shift_, sm_);
  }

  int solve(GridFunction& u, const GridFunction& b, double* hist, int* iters, int* conv, double* rate) const {
    u = GridFunction(levels_[0]);
    const double r0 = b.norm();
    int nh = 0;
    hist[nh++] = r0;
    *iters = 0;
    *conv = 0;
    if (r0 == 0.0 || cfg_.tol >= 1.0) {
      *conv = 1;
    } else {
      for (int k = 1; k <= cfg_.max_iter; ++k) {
        cycle_on_level(0, u, b);
        const double r = residual(b, u, shift_).norm();
        hist[nh++] = r;
        *iters = k;
        if (r <= cfg_.tol * r0) {
          *conv = 1;
          break;
        }
      }
    }
    *rate = orc_measured_rate(hist, *iters);
    return 0;
  }

 private:
  std::vector<Grid2D> levels_;
  Shift shift_;
  Cfg cfg_;
  SmootherConfig sm_;
  std::unique_ptr<Coarse> coarse_;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const SingularOperatorError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// tools/pdmg.cpp:137-147 with the real std::mt19937 / std::uniform_real_distribution.
void ref_random_complex(uint32_t seed, double lo, double hi, int64_t count, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (int64_t k = 0; k < count; ++k) {
    const double re = dist(rng), im = dist(rng);
    out[2 * k] = re;
    out[2 * k + 1] = im;
  }
}

int ref_vanka_coeffs(double er, double ei, double* abc) {
  return guarded([&] {
    const VankaCoeffs k = vanka_coeffs(cplx(er, ei));
    const cplx v[3] = {k.a, k.b, k.c};
    std::memcpy(abc, v, sizeof v);
  });
}

int ref_apply_smoother(int n, double lr, double li, int kind, double omega, const double* u, const double* b,
                       double* out) {
  return guarded([&] {
    const Grid2D g(n);
    const SmootherConfig c = kind == 0 ? SmootherConfig::vanka(omega) : SmootherConfig::jacobi(omega);
    store(apply_smoother(load(g, u), load(g, b), Shift{cplx(lr, li), 0, ShiftKind::User}, c), out);
  });
}

int ref_residual(int n, double lr, double li, const double* b, const double* u, double* r) {
  return guarded([&] {
    const Grid2D g(n);
    store(residual(load(g, b), load(g, u), Shift{cplx(lr, li), 0, ShiftKind::User}), r);
  });
}

int ref_apply_stencil(int n, const double* w9, double scale, const double* u, double* out) {
  return guarded([&] {
    const Grid2D g(n);
    Stencil3x3 s;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) s.w[r][c] = cplx(w9[2 * (3 * r + c)], w9[2 * (3 * r + c) + 1]);
    s.scale = scale;
    store(apply_stencil(s, load(g, u)), out);
  });
}

int ref_restrict(int n_fine, const double* fine, double* coarse) {
  return guarded([&] { store(restrict_full_weighting(load(Grid2D(n_fine), fine)), coarse); });
}

int ref_prolong(int n_coarse, const double* coarse, double* fine) {
  return guarded([&] { store(prolong_bilinear(load(Grid2D(n_coarse), coarse)), fine); });
}

int ref_mg_solve(int n, double lr, double li, const int* ci, const double* cd, const double* b, double* u,
                 double* hist, int* iters, int* conv, double* rate) {
  return guarded([&] {
    const Cfg c{ci[0], ci[1], ci[2], ci[3], ci[4], ci[5], cd[0], cd[1]};
    const Grid2D g(n);
    Hierarchy H(g, Shift{cplx(lr, li), 0, ShiftKind::User}, c);
    GridFunction uu(g);
    H.solve(uu, load(g, b), hist, iters, conv, rate);
    store(uu, u);
  });
}

// Batch over shifts on `threads` std::threads with contiguous chunks (paradiag.cpp:217-236).
int ref_mg_solve_batch(int n, int count, const double* lambdas, const int* ci, const double* cd, const double* b,
                       double* u, double* hist, int* iters, int* conv, double* rates, int threads) {
  return guarded([&] {
    if (threads < 1) throw ConfigError("paradiag_solve: threads must be >= 1");
    const Cfg c{ci[0], ci[1], ci[2], ci[3], ci[4], ci[5], cd[0], cd[1]};
    const Grid2D g(n);
    const long N = g.size();
    const int H = c.max_iter + 1;
    auto run_range = [&](int b0, int b1) {
      for (int s = b0; s < b1; ++s) {
        Hierarchy mg(g, Shift{cplx(lambdas[2 * s], lambdas[2 * s + 1]), s, ShiftKind::User}, c);
        GridFunction uu(g);
        mg.solve(uu, load(g, b + 2 * N * s), hist + static_cast<size_t>(H) * s, iters + s, conv + s, rates + s);
        store(uu, u + 2 * N * s);
      }
    };
    const int nw = std::min(threads, count);
    if (nw <= 1) {
      run_range(0, count);
      return;
    }
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errors(static_cast<size_t>(nw));
    const int chunk = (count + nw - 1) / nw;
    for (int t = 0; t < nw; ++t) {
      const int b0 = std::min(count, t * chunk), b1 = std::min(count, b0 + chunk);
      pool.emplace_back([&, t, b0, b1] {
        try {
          run_range(b0, b1);
        } catch (...) {
          errors[static_cast<size_t>(t)] = std::current_exception();
        }
      });
    }
    for (std::thread& th : pool) th.join();
    for (const std::exception_ptr& e : errors)
      if (e) std::rethrow_exception(e);
  });
}

}  // extern "C"
