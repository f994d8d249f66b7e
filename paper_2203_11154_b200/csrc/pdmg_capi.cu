// pdmg_capi.cu -- the extern "C" boundary of libpdmg_b200.so (include/pdmg_b200.h).
#include <random>

#include "pdmg_host.h"
#include "pdmg_paradiag.h"

using namespace pdmg_b200;

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
    auto e = create_engine(*d);
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
int pdmg_solve_device_shards(pdmg_ctx* c, const void* const* d_b, void* const* d_u, pdmg_solve_report* rep) {
  return guarded([&] {
    NEED_CTX(c);
    if (!d_b || !d_u) throw ConfigError("pdmg_solve_device_shards: NULL buffer list");
    for (int p = 0; p < c->e->num_parts(); ++p)
      if (!d_b[p] || !d_u[p]) throw ConfigError("pdmg_solve_device_shards: NULL b or u for shard " + std::to_string(p));
    c->e->solve_device_shards(d_b, d_u, rep);
  });
}
int pdmg_num_parts(const pdmg_ctx* c) { return c ? c->e->num_parts() : 0; }
int pdmg_part_range(const pdmg_ctx* c, int part, int32_t* shift0, int32_t* count, int32_t* device) {
  return guarded([&] {
    NEED_CTX(c);
    c->e->part_range(part, shift0, count, device);
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

}  // extern "C"
struct pdmg_paradiag {
  Paradiag p;
  pdmg_ctx* solver = nullptr;  // non-owning view of shard 0's engine for the stats API
};
extern "C" {

}  // extern "C"

static std::vector<int> device_list(int32_t device, const int32_t* devices, int32_t n_devices) {
  if (n_devices < 0 || (n_devices > 0 && !devices)) throw ConfigError("ParaDIAG: bad device list");
  if (n_devices == 0) return {device};
  return std::vector<int>(devices, devices + n_devices);
}

template <class F>
static int paradiag_make(pdmg_paradiag** out, F&& setup) {
  return guarded([&] {
    if (!out) throw ConfigError("pdmg_paradiag_create: NULL argument");
    *out = nullptr;
    auto* P = new pdmg_paradiag;
    try {
      setup(P->p);
    } catch (...) {
      delete P;
      throw;
    }
    P->solver = new pdmg_ctx;
    P->solver->e.reset(P->p.solver());
    *out = P;
  });
}

extern "C" {

int pdmg_paradiag_create(int32_t n, int32_t nt, double alpha, double dt, const pdmg_mg_config* cfg, int32_t device,
                         pdmg_paradiag** out) {
  return pdmg_paradiag_create_multi(n, nt, alpha, dt, cfg, &device, 1, out);
}
int pdmg_paradiag_create_multi(int32_t n, int32_t nt, double alpha, double dt, const pdmg_mg_config* cfg,
                               const int32_t* devices, int32_t n_devices, pdmg_paradiag** out) {
  return paradiag_make(out, [&](Paradiag& p) {
    if (!cfg) throw ConfigError("pdmg_paradiag_create: NULL argument");
    p.setup_circulant(n, nt, alpha, dt, *cfg, device_list(0, devices, n_devices));
  });
}
int pdmg_paradiag_create_general(int32_t n, int32_t nt, const pdmg_c128* lambdas, const pdmg_c128* V,
                                 const pdmg_c128* Vinv, const double* B, const pdmg_mg_config* cfg,
                                 const int32_t* devices, int32_t n_devices, pdmg_paradiag** out) {
  return paradiag_make(out, [&](Paradiag& p) {
    if (!lambdas || !V || !Vinv || !B || !cfg) throw ConfigError("pdmg_paradiag_create_general: NULL argument");
    p.setup_general(n, nt, lambdas, V, Vinv, B, *cfg, device_list(0, devices, n_devices));
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
int pdmg_paradiag_num_parts(const pdmg_paradiag* P) { return P ? (int)P->p.sh.size() : 0; }
int pdmg_paradiag_part_range(const pdmg_paradiag* P, int part, int32_t* t0, int32_t* count, int32_t* device) {
  return guarded([&] {
    if (!P || part < 0 || part >= (int)P->p.sh.size()) throw ConfigError("pdmg_paradiag_part_range: bad shard");
    const PdShard& s = *P->p.sh[part];
    if (t0) *t0 = s.t0;
    if (count) *count = s.cnt;
    if (device) *device = s.device;
  });
}
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
int pdmg_paradiag_run_shards(pdmg_paradiag* P, const void* const* d_f, void* const* d_u, pdmg_solve_report* rep,
                             double* relres) {
  return guarded([&] {
    if (!P || !d_f || !d_u) throw ConfigError("pdmg_paradiag_run_shards: NULL argument");
    for (size_t q = 0; q < P->p.sh.size(); ++q)
      if (!d_f[q] || !d_u[q]) throw ConfigError("pdmg_paradiag_run_shards: NULL buffer for shard " + std::to_string(q));
    P->p.run_shards(reinterpret_cast<const double2* const*>(d_f), reinterpret_cast<double2* const*>(d_u), rep, relres);
  });
}

int pdmg_paradiag_create_rank(int32_t n, int32_t nt, double alpha, double dt, const pdmg_mg_config* cfg, int32_t rank,
                              int32_t nranks, int32_t device, pdmg_paradiag** out) {
  return paradiag_make(out, [&](Paradiag& p) {
    if (!cfg) throw ConfigError("pdmg_paradiag_create_rank: NULL argument");
    p.setup_rank(n, nt, alpha, dt, *cfg, rank, nranks, device);
  });
}
int pdmg_paradiag_ipc_handles(pdmg_paradiag* P, void* handles) {
  return guarded([&] {
    if (!P || !handles) throw ConfigError("pdmg_paradiag_ipc_handles: NULL argument");
    P->p.ipc_handles(handles);
  });
}
int pdmg_paradiag_open_peers(pdmg_paradiag* P, const void* all_handles) {
  return guarded([&] {
    if (!P || !all_handles) throw ConfigError("pdmg_paradiag_open_peers: NULL argument");
    P->p.open_peers(all_handles);
  });
}
int pdmg_paradiag_rank_phase(pdmg_paradiag* P, int32_t phase, pdmg_solve_report* report, double* sums) {
  return guarded([&] {
    if (!P) throw ConfigError("pdmg_paradiag_rank_phase: NULL argument");
    P->p.rank_phase(phase, report, sums);
  });
}
void* pdmg_paradiag_rank_buffer(pdmg_paradiag* P, int32_t which) {
  if (!P || P->p.local < 0 || which < 0 || which > 3) return nullptr;
  const PdShard& s = *P->p.sh[P->p.local];
  return which == 0 ? (void*)s.f : which == 1 ? (void*)s.g : which == 2 ? (void*)s.w : (void*)s.u;
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
  if (!f || !u) {
    g_last_error = "pdmg_paradiag_general: NULL argument";
    return PDMG_ERR_CONFIG;
  }
  pdmg_paradiag* P = nullptr;
  int st = pdmg_paradiag_create_general(n, nt, lambdas, V, Vinv, B, cfg, &device, 1, &P);
  if (st) return st;
  st = pdmg_paradiag_run(P, f, u, report, relres);
  pdmg_paradiag_destroy(P);
  return st;
}

int pdmg_time_transform(int32_t device, int32_t nt, int64_t npts, const pdmg_c128* M, const void* d_in, void* d_out,
                        void* stream) {
  return guarded([&] {
    if (!M || !d_in || !d_out) throw ConfigError("pdmg_time_transform: NULL argument");
    if (nt < 1 || npts < 0) throw ConfigError("pdmg_time_transform: bad sizes");
    CK(cudaSetDevice(device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double2* dM = nullptr;
    CK(cudaMalloc(&dM, sizeof(double2) * nt * nt));
    try {
      CK(cudaMemcpyAsync(dM, M, sizeof(double2) * nt * nt, cudaMemcpyHostToDevice, st));
      time_transform(device, st, nt, npts, dM, static_cast<const double2*>(d_in), static_cast<double2*>(d_out));
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
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    time_dft(device, nt, npts, alpha, step, static_cast<const double2*>(d_in), static_cast<double2*>(d_out), st);
    CK(cudaStreamSynchronize(st));
  });
}

int pdmg_aao_residual(int32_t device, int32_t n, int32_t ntl, int32_t t0, double alpha, double dt, const void* d_u,
                      const void* d_u_prev, const void* d_f, double* sums, void* stream) {
  return guarded([&] {
    if (!sums) throw ConfigError("pdmg_aao_residual: NULL sums");
    aao_residual_sums(device, n, ntl, t0, alpha, dt, static_cast<const double2*>(d_u),
                      static_cast<const double2*>(d_u_prev), static_cast<const double2*>(d_f), sums,
                      static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
