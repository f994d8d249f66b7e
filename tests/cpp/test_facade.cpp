// C++ facade test (reads like the reference's doctest suites, proj/tests/test_multigrid.cpp):
// builds against include/pdmg_b200.hpp + libpdmg_b200.so; run on a GPU by tests/test_gpu_facade.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "pdmg_b200.hpp"

using namespace pdmg_b200;

#define CHECK(c)                                                        \
  do {                                                                  \
    if (!(c)) {                                                         \
      std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
      std::exit(1);                                                     \
    }                                                                   \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::string(argv[1]) == "--gpu";
  // configuration errors surface as the reference exception types, with no GPU needed
  bool threw = false;
  try {
    MultigridConfig c;
    c.coarsest_n = 5;
    BatchedMultigridHierarchy bad(Grid2D(64), {Shift{}}, c);
  } catch (const ConfigError& e) {
    threw = std::string(e.what()).find("not coarsest_n = 5") != std::string::npos;
  }
  CHECK(threw);
  threw = false;
  try {
    BatchedMultigridHierarchy bad(Grid2D(64), {Shift{cplx(-2.0 * 64 * 64, 0.0)}}, MultigridConfig{});
  } catch (const SingularOperatorError& e) {
    threw = std::string(e.what()).find("level 0 (n = 64)") != std::string::npos;
  }
  CHECK(threw);
  if (!gpu) {
    std::puts("facade (host checks) ok");
    return 0;
  }
  // BASELINE config 1 through the facade: 11 V(1,1) cycles to 1e-10
  MultigridConfig cfg;
  cfg.cycle = CycleKind::V;
  cfg.nu1 = 1;
  cfg.nu2 = 1;
  cfg.coarsest_n = 4;
  cfg.tol = 1e-10;
  pdmg_c128 lam;
  pdmg_circulant_shifts(0.01, 32, 1.0 / 32, 3, 1, &lam);
  const Grid2D g(64);
  auto [u, rep] = multigrid_solve(random_rhs(g, 0), g, Shift{cplx(lam.re, lam.im)}, cfg);
  CHECK(rep.converged);
  CHECK(rep.iterations == 11);
  CHECK(rep.residual_history.size() == 12);
  CHECK(rep.residual_history.back() <= 1e-10 * rep.residual_history.front());
  // W(1,0) README row (proj/README.md:37-41): 14 cycles, rate ~0.273
  auto [u2, rep2] = multigrid_solve(random_rhs(g, 123), g, Shift{}, MultigridConfig{});
  CHECK(rep2.iterations == 14);
  CHECK(std::abs(rep2.rate - 0.273) < 1e-3);
  // paradiag_solve through the facade: BASELINE's alpha-circulant preconditioner on one device and sharded over the
  // device list {0, 0} (bitwise the same u), and the QBV scheme (alpha = -1/beta) in the reference's order
  const Grid2D g32(32);
  const int nt = 8;
  std::vector<cplx> f(static_cast<size_t>(nt) * g32.size());
  pdmg_random_rhs(4, -1.0, 1.0, (int64_t)f.size(), reinterpret_cast<pdmg_c128*>(f.data()));
  const ParadiagResult p1 = paradiag_solve_circulant(f, g32, nt, 0.01, 1.0 / nt, cfg);
  const ParadiagResult p2 = paradiag_solve_circulant(f, g32, nt, 0.01, 1.0 / nt, cfg, {0, 0});
  CHECK(p1.all_converged && p1.relative_residual < 1e-8 && p1.u == p2.u);
  const ParadiagResult q = paradiag_solve_circulant(f, g32, nt, -100.0, 1.0 / nt, cfg);
  CHECK(q.all_converged && q.reports.size() == (size_t)nt);
  // slot k holds (1 - gamma zeta^{-k}) / tau with gamma = 100^{1/nt} e^{i pi / nt}
  const double pi = 3.14159265358979323846;
  const cplx lam1 = (1.0 - std::polar(std::pow(100.0, 1.0 / nt), pi / nt - 2.0 * pi / nt)) * (double)nt;
  CHECK(std::abs(q.shifts[1].lambda - lam1) <= 1e-12 * std::abs(lam1));
  std::printf("facade ok: C1 %d cycles, W(1,0) %d cycles rate %.4f; paradiag relres %.2e\n", rep.iterations,
              rep2.iterations, rep2.rate, p1.relative_residual);
  return 0;
}
