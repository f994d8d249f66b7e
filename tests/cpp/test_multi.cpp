// Multi-device / multi-thread use of the C ABI through the C++ facade (the reference's solver is reentrant:
// distinct hierarchies solve concurrently from distinct threads; paradiag_solve spreads shifts over `threads`,
// proj/src/paradiag.cpp:207-236).  Checks, against one single-device context solving every shift:
//   1. two contexts driven concurrently from two host threads reproduce their shifts bitwise;
//   2. one context sharded over a device list (here {0, 0}: two shards on one GPU, each with its own engine and
//      stream) reproduces every shift bitwise, with the reference's contiguous ceil(S / P) chunking.
// Run on a GPU by tests/test_facade.py.
#include <cstdio>
#include <cstdlib>
#include <thread>

#include "pdmg_b200.hpp"

using namespace pdmg_b200;

#define CHECK(c)                                                          \
  do {                                                                    \
    if (!(c)) {                                                           \
      std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
      std::exit(1);                                                       \
    }                                                                     \
  } while (0)

int main() {
  const Grid2D g(128);
  const int S = 9;
  MultigridConfig cfg;
  cfg.cycle = CycleKind::V, cfg.nu1 = 1, cfg.nu2 = 1, cfg.coarsest_n = 4, cfg.tol = 1e-10;
  std::vector<pdmg_c128> lam(S);
  pdmg_circulant_shifts(0.01, 32, 1.0 / 32, 0, S, lam.data());
  std::vector<Shift> shifts(S);
  for (int s = 0; s < S; ++s) shifts[s] = Shift{cplx(lam[s].re, lam[s].im), s};
  const long N = g.size();
  std::vector<cplx> b(static_cast<size_t>(S) * N);
  pdmg_random_rhs(1, -1.0, 1.0, S * N, reinterpret_cast<pdmg_c128*>(b.data()));

  BatchedMultigridHierarchy all(g, shifts, cfg);
  std::vector<cplx> u_ref;
  const auto rep_ref = all.solve(u_ref, b);

  // 1. two contexts, two threads: shifts [0, 4) and [4, 9)
  std::vector<Shift> sa(shifts.begin(), shifts.begin() + 4), sb(shifts.begin() + 4, shifts.end());
  std::vector<cplx> ba(b.begin(), b.begin() + 4 * N), bb(b.begin() + 4 * N, b.end()), ua, ub;
  std::vector<SolveReport> ra, rb;
  {
    BatchedMultigridHierarchy ha(g, sa, cfg), hb(g, sb, cfg);
    std::thread t1([&] { ra = ha.solve(ua, ba); });
    std::thread t2([&] { rb = hb.solve(ub, bb); });
    t1.join();
    t2.join();
  }
  for (int s = 0; s < S; ++s) {
    const SolveReport& r = s < 4 ? ra[s] : rb[s - 4];
    CHECK(r.iterations == rep_ref[s].iterations);
    CHECK(r.residual_history == rep_ref[s].residual_history);
    const cplx* u = s < 4 ? ua.data() + s * N : ub.data() + (s - 4) * N;
    for (long q = 0; q < N; ++q) CHECK(u[q] == u_ref[s * N + q]);
  }

  // 2. one context over the device list {0, 0}: shards [0, 5) and [5, 9)
  BatchedMultigridHierarchy sharded(g, shifts, cfg, std::vector<int>{0, 0});
  CHECK(sharded.num_parts() == 2);
  int32_t s0 = -1, cnt = -1, dev = -1;
  CHECK(pdmg_part_range(sharded.handle(), 1, &s0, &cnt, &dev) == PDMG_OK);
  CHECK(s0 == 5 && cnt == 4 && dev == 0);
  std::vector<cplx> us;
  const auto rs = sharded.solve(us, b);
  for (int s = 0; s < S; ++s) {
    CHECK(rs[s].iterations == rep_ref[s].iterations);
    CHECK(rs[s].converged == rep_ref[s].converged);
    CHECK(rs[s].residual_history == rep_ref[s].residual_history);
  }
  CHECK(us == u_ref);
  std::printf("multi ok: 2 threads x 2 contexts and a 2-shard context reproduce %d shifts bitwise\n", S);
  return 0;
}
