// pdmg_multi.cu -- a batch of shifts sharded over a list of devices behind one pdmg_ctx.
//
// The reference's parallel resource is an argument of the solver: paradiag_solve(f, td, cfg, threads) splits the
// shifts into contiguous chunks of ceil(S / threads) and runs each chunk on its own std::thread
// (proj/src/paradiag.cpp:207-236).  Here the resource is a device list: shard p = shifts
// [p * chunk, min(S, (p + 1) * chunk)) lives on devices[p] in its own engine (its own streams and level storage),
// and every call runs the shards concurrently, one host thread per shard.  The shifts are independent, so there is
// no data exchange between devices and every shard's results are bitwise those of a single-device solve of the
// same shifts.  A device may appear more than once (shards then share it, each on its own stream).
#include <thread>

#include "pdmg_host.h"

namespace pdmg_b200 {

struct MultiEngine : EngineBase {
  std::vector<std::unique_ptr<EngineBase>> parts;
  std::vector<int> lo;    // shard p = shifts [lo[p], lo[p + 1])
  std::vector<int> devs;  // devices[p]
  int64_t per0 = 0;       // interior points per shift on the finest level

  void setup_host(const pdmg_batch_desc& d) override {
    if (d.n_devices < 1 || !d.devices) throw ConfigError("pdmg_create: empty device list");
    if (d.n_shifts < 1) throw ConfigError("pdmg_create: n_shifts must be >= 1");
    if (!d.lambdas) throw ConfigError("pdmg_create: lambdas is NULL");
    cfg = d.cfg;
    ln = level_list(d.n, cfg);
    S = d.n_shifts;
    per0 = (int64_t)(d.n - 1) * (d.n - 1);
    const int nw = std::min(d.n_devices, S);
    const int chunk = (S + nw - 1) / nw;  // paradiag.cpp:222
    lo.clear();
    devs.clear();
    for (int t = 0; t < nw; ++t) {
      const int b0 = t * chunk, b1 = std::min(S, b0 + chunk);
      if (b0 >= b1) break;
      lo.push_back(b0);
      devs.push_back(d.devices[t]);
    }
    lo.push_back(S);
    lambdas.resize(S);
    for (int s = 0; s < S; ++s) lambdas[s] = cplx(d.lambdas[s].re, d.lambdas[s].im);
    // shard by shard in shift order, so the first failing shift (in the reference's order) is the one reported
    for (size_t p = 0; p + 1 < lo.size(); ++p) {
      pdmg_batch_desc dp = d;
      dp.n_shifts = lo[p + 1] - lo[p];
      dp.lambdas = d.lambdas + lo[p];
      dp.devices = nullptr;
      dp.n_devices = 0;
      dp.device = devs[p];
      auto e = make_engine(d.precision);
      e->device = -1;
      e->setup_host(dp);
      parts.push_back(std::move(e));
    }
    coarse_singular.clear();
    for (auto& e : parts) coarse_singular.insert(coarse_singular.end(), e->coarse_singular.begin(), e->coarse_singular.end());
    for (uint8_t c : coarse_singular) any_singular |= c != 0;
  }

  // Runs f(p, part) for every shard on its own host thread; rethrows the first shard's exception in shard order
  // (paradiag.cpp:221-235).
  template <class F>
  void each(F&& f) {
    std::vector<std::exception_ptr> err(parts.size());
    std::vector<std::thread> th;
    for (size_t p = 0; p < parts.size(); ++p)
      th.emplace_back([&, p] {
        try {
          CK(cudaSetDevice(devs[p]));
          f(p, *parts[p]);
        } catch (...) {
          err[p] = std::current_exception();
        }
      });
    for (auto& t : th) t.join();
    for (auto& x : err)
      if (x) std::rethrow_exception(x);
  }

  void setup_device(int) override {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    for (int d : devs)
      if (d < 0 || d >= ndev) throw CudaError("pdmg_create: CUDA device " + std::to_string(d) + " not available");
    each([&](size_t p, EngineBase& e) { e.setup_device(devs[p]); });
    device = devs[0];
    stream = parts[0]->stream;
  }

  void sync_flags() {
    for (auto& e : parts) e->solve_path = solve_path, e->profiling = profiling;
  }
  void gather_stats() {
    double upd = 0.0;
    for (auto& e : parts) {
      upd += e->last_updates;
      launches += e->launches;
      e->launches = 0;
      for (auto& kv : e->stats) {
        Stat& st = stats[kv.first];
        st.launches += kv.second.launches;
        st.ms += kv.second.ms;
        st.bytes += kv.second.bytes;
        st.ubytes += kv.second.ubytes;
        st.updates += kv.second.updates;
      }
      e->stats.clear();
    }
    last_updates = upd;
  }
  // report arrays of shard p (offsets into the caller's per-shift arrays)
  pdmg_solve_report sub_report(const pdmg_solve_report* rep, size_t p) const {
    pdmg_solve_report rc{};
    if (!rep) return rc;
    const int s0 = lo[p];
    const int64_t H = cfg.max_iter + 1;
    rc.iterations = rep->iterations ? rep->iterations + s0 : nullptr;
    rc.converged = rep->converged ? rep->converged + s0 : nullptr;
    rc.residual_history = rep->residual_history ? rep->residual_history + s0 * H : nullptr;
    rc.rate = rep->rate ? rep->rate + s0 : nullptr;
    return rc;
  }

  void solve_host(const pdmg_c128* b, pdmg_c128* u, pdmg_solve_report* rep) override {
    const auto t0 = std::chrono::steady_clock::now();
    sync_flags();
    each([&](size_t p, EngineBase& e) {
      pdmg_solve_report rc = sub_report(rep, p);
      e.solve_host(b + lo[p] * per0, u + lo[p] * per0, rep ? &rc : nullptr);
    });
    gather_stats();
    if (rep) rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  void solve_device(const double2* d_b, double2* d_u, pdmg_solve_report* rep) override {
    if (parts.size() != 1)
      throw ConfigError("pdmg_solve_device: the context spans " + std::to_string(parts.size()) +
                        " devices; pass per-shard device buffers to pdmg_solve_device_shards");
    sync_flags();
    parts[0]->solve_device(d_b, d_u, rep);
    gather_stats();
  }
  void solve_device_shards(const void* const* d_b, void* const* d_u, pdmg_solve_report* rep) override {
    const auto t0 = std::chrono::steady_clock::now();
    sync_flags();
    each([&](size_t p, EngineBase& e) {
      pdmg_solve_report rc = sub_report(rep, p);
      e.solve_device(static_cast<const double2*>(d_b[p]), static_cast<double2*>(d_u[p]), rep ? &rc : nullptr);
    });
    gather_stats();
    if (rep) rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  int num_parts() const override { return (int)parts.size(); }
  void part_range(int p, int* s0, int* count, int* dev) const override {
    if (p < 0 || p >= (int)parts.size()) throw ConfigError("pdmg_part_range: shard index out of range");
    if (s0) *s0 = lo[p];
    if (count) *count = lo[p + 1] - lo[p];
    if (dev) *dev = devs[p];
  }

  // level-shaped host arrays of shard p at level l
  int64_t per(int l) const { return (int64_t)(ln[l] - 1) * (ln[l] - 1); }
  void cycle_host(pdmg_c128* u, const pdmg_c128* b) override {
    sync_flags();
    each([&](size_t p, EngineBase& e) { e.cycle_host(u + lo[p] * per0, b + lo[p] * per0); });
    gather_stats();
  }
  void check_level(int l, int need_coarser) const {
    if (l < 0 || l + need_coarser >= (int)ln.size())
      throw ConfigError("level index " + std::to_string(l) + " out of range for a " + std::to_string(ln.size()) +
                        "-level hierarchy");
  }
  void op_smooth(int l, const pdmg_c128* u, const pdmg_c128* b, pdmg_c128* out) override {
    check_level(l, 1);
    each([&](size_t p, EngineBase& e) {
      const int64_t o = lo[p] * per(l);
      e.op_smooth(l, u + o, b + o, out + o);
    });
    gather_stats();
  }
  void op_residual(int l, const pdmg_c128* b, const pdmg_c128* u, pdmg_c128* r) override {
    check_level(l, 0);
    each([&](size_t p, EngineBase& e) {
      const int64_t o = lo[p] * per(l);
      e.op_residual(l, b + o, u + o, r + o);
    });
    gather_stats();
  }
  void op_restrict(int l, const pdmg_c128* fine, pdmg_c128* coarse) override {
    check_level(l, 1);
    each([&](size_t p, EngineBase& e) { e.op_restrict(l, fine + lo[p] * per(l), coarse + lo[p] * per(l + 1)); });
    gather_stats();
  }
  void op_prolong(int l, const pdmg_c128* coarse, pdmg_c128* fine) override {
    check_level(l, 1);
    each([&](size_t p, EngineBase& e) { e.op_prolong(l, coarse + lo[p] * per(l + 1), fine + lo[p] * per(l)); });
    gather_stats();
  }
  void op_norm(int l, const pdmg_c128* v, double* norms) override {
    check_level(l, 0);
    each([&](size_t p, EngineBase& e) { e.op_norm(l, v + lo[p] * per(l), norms + lo[p]); });
    gather_stats();
  }
  void op_coarse_solve(const pdmg_c128* b, pdmg_c128* u) override {
    const int l = (int)ln.size() - 1;
    each([&](size_t p, EngineBase& e) { e.op_coarse_solve(b + lo[p] * per(l), u + lo[p] * per(l)); });
    gather_stats();
  }
};

std::unique_ptr<EngineBase> create_engine(const pdmg_batch_desc& d) {
  std::unique_ptr<EngineBase> e;
  if (d.n_devices > 0 || d.devices) {
    e = std::make_unique<MultiEngine>();
  } else {
    e = make_engine(d.precision);
  }
  e->device = -1;
  e->setup_host(d);  // all ConfigError / SingularOperatorError paths run before any CUDA call
  e->setup_device(d.device);
  return e;
}

}  // namespace pdmg_b200
