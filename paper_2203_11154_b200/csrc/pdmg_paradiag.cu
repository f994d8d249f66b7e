// pdmg_paradiag.cu -- ParaDIAG on the GPU (restating proj/src/paradiag.cpp:185-248), on one device or with the
// time slices sharded over a device list (see pdmg_paradiag.h).
#include <condition_variable>
#include <mutex>
#include <set>
#include <thread>
#include <tuple>

#include "pdmg_paradiag.h"
#include "pdmg_time_kernels.cuh"

namespace pdmg_b200 {

namespace {

constexpr int DFT_SMEM_MAX = 96 * 1024;
int dft_points_per_cta(int nt) { return std::max(1, std::min(64, 4096 / nt)); }

// k_time_dft's shared-memory opt-in, once per device (function attributes are per device context)
void dft_attr(int device) {
  static std::mutex mu;
  static std::set<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(device)) return;
  CK(cudaFuncSetAttribute(k_time_dft, cudaFuncAttributeMaxDynamicSharedMemorySize, DFT_SMEM_MAX));
  done.insert(device);
}

RowTab rowtab(const std::vector<double2*>& p, int rows, int64_t ld) {
  if (p.size() > (size_t)MAX_SHARDS) throw ConfigError("ParaDIAG: at most 16 device shards");
  RowTab T{};
  for (size_t s = 0; s < p.size(); ++s) T.p[s] = p[s];
  T.rows = rows;
  T.ld = ld;
  return T;
}

void launch_dft(const DftTables& T, const RowTab& in, const RowTab& out, int64_t pt0, int64_t pt1, cudaStream_t st) {
  const int P = dft_points_per_cta(T.nt);
  // data + (radix-2 path) the nt/2 twiddles
  const size_t smem = (size_t)T.nt * P * sizeof(double2) + (T.log2nt >= 0 ? (size_t)(T.nt / 2) * sizeof(double2) : 0);
  const int64_t blocks = (pt1 - pt0 + P - 1) / P;
  if (blocks > 0)
    k_time_dft<<<(unsigned)blocks, DFT_THREADS, smem, st>>>(in, out, T.nt, T.log2nt, pt0, pt1, P, T.tw, T.pre, T.post);
  CK(cudaGetLastError());
}

void launch_gemm(const double2* M, int nt, const RowTab& X, const RowTab& Y, int r0, int r1, int yoff, int64_t pt0,
                 int64_t pt1, cudaStream_t st) {
  if (r1 <= r0 || pt1 <= pt0) return;
  dim3 grid((unsigned)((pt1 - pt0 + GM_BN - 1) / GM_BN), (unsigned)((r1 - r0 + GM_BM - 1) / GM_BM));
  k_time_gemm<<<grid, GM_THREADS, 0, st>>>(M, nt, X, Y, r0, r1, yoff, pt0, pt1);
  CK(cudaGetLastError());
}

double2* upload(const std::vector<double2>& h, cudaStream_t st) {
  double2* d = nullptr;
  CK(cudaMalloc(&d, sizeof(double2) * h.size()));
  CK(cudaMemcpyAsync(d, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice, st));
  return d;
}

// A reusable barrier for the shard threads of one call (C++17: no std::barrier).  A shard that fails breaks it,
// so the others stop at their next phase instead of waiting forever.
struct BarrierBroken {};
class Barrier {
 public:
  explicit Barrier(int n) : n_(n) {}
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    if (broken_) throw BarrierBroken{};
    const int gen = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(lk, [&] { return gen != gen_ || broken_; });
      if (broken_) throw BarrierBroken{};
    }
  }
  void fail() {
    std::lock_guard<std::mutex> lk(mu_);
    broken_ = true;
    cv_.notify_all();
  }

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  int n_, count_ = 0, gen_ = 0;
  bool broken_ = false;
};

void enable_peers(const std::vector<int>& devs) {
  for (int a : devs)
    for (int b : devs) {
      if (a == b) continue;
      int can = 0;
      CK(cudaDeviceCanAccessPeer(&can, a, b));
      if (!can)
        throw CudaError("ParaDIAG: device " + std::to_string(a) + " cannot access device " + std::to_string(b) +
                        " (peer access over NVLink is required for sharded time transforms)");
      CK(cudaSetDevice(a));
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
      else CK(e);
    }
}

}  // namespace

void check_dft_size(int nt) {
  const bool pow2 = nt > 0 && (nt & (nt - 1)) == 0;  // (the radix-2 path also holds nt/2 twiddles)
  if ((size_t)nt * dft_points_per_cta(nt) * sizeof(double2) + (pow2 ? (size_t)(nt / 2) * sizeof(double2) : 0) > (size_t)DFT_SMEM_MAX)
    throw ConfigError("time DFT: nt = " + std::to_string(nt) + " needs more than " + std::to_string(DFT_SMEM_MAX) +
                      " B of shared memory per transform (nt <= 6144)");
}

std::unique_ptr<DftTables> make_dft_tables(int nt, double alpha, int step, cudaStream_t st) {
  if (nt < 1) throw ConfigError("time DFT: nt must be >= 1");
  check_dft_size(nt);
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
  T->tw = upload(tw, st);
  T->pre = upload(pre, st);
  T->post = upload(post, st);
  CK(cudaStreamSynchronize(st));
  return T;
}

PdShard::~PdShard() {
  if (remote) {  // another rank's buffers, opened over IPC
    for (double2* p : {f, g, w, u})
      if (p) cudaIpcCloseMemHandle(p);
    return;
  }
  cudaSetDevice(device);
  for (double2* p : {f, g, w, u, y, V, Vi, B}) cudaFree(p);
  cudaFree(partial);
  if (h_partial) cudaFreeHost(h_partial);
  for (cudaEvent_t e : ev)
    if (e) cudaEventDestroy(e);
  t1.reset();
  t3.reset();
  eng.reset();
}

// Shards: contiguous time slices of ceil(nt / P) (paradiag.cpp:222), each with the engine of its shift slots and
// the spatial points it transforms (npts split evenly).
void Paradiag::setup_shards(int n_, int nt_, const std::vector<pdmg_c128>& lam, const pdmg_mg_config& cfg,
                            const std::vector<int>& devices) {
  n = n_, nt = nt_;
  npts = (int64_t)(n - 1) * (n - 1);
  std::vector<int> devs = devices.empty() ? std::vector<int>{0} : devices;
  const int nw = std::min((int)devs.size(), nt);
  const int chunk = (nt + nw - 1) / nw;
  std::vector<int> used;
  for (int t = 0; t < nw; ++t) {
    const int b0 = t * chunk, b1 = std::min(nt, b0 + chunk);
    if (b0 >= b1) break;
    auto s = std::make_unique<PdShard>();
    s->device = devs[t], s->t0 = b0, s->cnt = b1 - b0;
    pdmg_batch_desc d{n, s->cnt, lam.data() + b0, cfg, PDMG_PREC_C128, s->device};
    s->eng = make_engine_c128();
    s->eng->device = -1;
    s->eng->setup_host(d);  // config / singular-smoother errors in slot order, before any CUDA call
    sh.push_back(std::move(s));
    used.push_back(devs[t]);
  }
  if (sh.size() > (size_t)MAX_SHARDS) throw ConfigError("ParaDIAG: at most 16 device shards");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  for (int d : used)
    if (d < 0 || d >= ndev) throw CudaError("ParaDIAG: CUDA device " + std::to_string(d) + " not available");
  std::vector<int> uniq(used);
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  enable_peers(uniq);
  const int P = (int)sh.size();
  for (int p = 0; p < P; ++p) {
    PdShard& s = *sh[p];
    s.pt0 = npts * p / P, s.pt1 = npts * (p + 1) / P;
    s.eng->setup_device(s.device);
    CK(cudaSetDevice(s.device));
    const size_t bytes = sizeof(double2) * (size_t)s.cnt * npts;
    for (double2** q : {&s.f, &s.g, &s.w, &s.u}) CK(cudaMalloc(q, bytes));
    CK(cudaMalloc(&s.partial, sizeof(double) * 2 * res_blocks));
    CK(cudaMallocHost(&s.h_partial, sizeof(double) * 2 * res_blocks));
    for (auto& e : s.ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
}

void Paradiag::setup_circulant(int n_, int nt_, double alpha_, double dt_, const pdmg_mg_config& cfg,
                               const std::vector<int>& devices) {
  if (nt_ < 2) throw ConfigError("TimeDiscretization: need n >= 2 time steps");
  if (!(dt_ > 0.0)) throw ConfigError("TimeDiscretization: tau must be positive");
  if (!(alpha_ != 0.0)) throw ConfigError("alpha-circulant: alpha must be nonzero");
  check_dft_size(nt_);
  general = false, alpha = alpha_, dt = dt_;
  std::vector<pdmg_c128> lam(nt_);
  pdmg_circulant_shifts(alpha, nt_, dt, 0, nt_, lam.data());
  setup_shards(n_, nt_, lam, cfg, devices);
  for (auto& s : sh) {
    CK(cudaSetDevice(s->device));
    dft_attr(s->device);
    s->t1 = make_dft_tables(nt, alpha, 1, s->eng->stream);
    s->t3 = make_dft_tables(nt, alpha, 3, s->eng->stream);
  }
}

void Paradiag::setup_general(int n_, int nt_, const pdmg_c128* lambdas, const pdmg_c128* V, const pdmg_c128* Vinv,
                             const double* B, const pdmg_mg_config& cfg, const std::vector<int>& devices) {
  if (nt_ < 1) throw ConfigError("paradiag_solve: empty right-hand side");
  general = true;
  std::vector<pdmg_c128> lam(lambdas, lambdas + nt_);
  setup_shards(n_, nt_, lam, cfg, devices);
  std::vector<double2> hV((size_t)nt * nt), hVi((size_t)nt * nt), hB((size_t)nt * nt);
  for (size_t q = 0; q < hV.size(); ++q) {
    hV[q] = make_double2(V[q].re, V[q].im);
    hVi[q] = make_double2(Vinv[q].re, Vinv[q].im);
    hB[q] = make_double2(B[q], 0.0);
  }
  for (auto& s : sh) {
    CK(cudaSetDevice(s->device));
    cudaStream_t st = s->eng->stream;
    s->V = upload(hV, st), s->Vi = upload(hVi, st), s->B = upload(hB, st);
    CK(cudaMalloc(&s->y, sizeof(double2) * (size_t)s->cnt * npts));
    CK(cudaStreamSynchronize(st));
  }
}

// One host thread per shard; the cross-device order of the phases is carried by events, recorded before a host
// barrier and waited on after it:
//   [input ready] -> step 1 transform (gather f columns from every shard, scatter g rows to their owners)
//   -> [g ready everywhere] -> the shard's shifted solves -> [w ready everywhere] -> step 3 transform
//   -> [u ready everywhere] -> all-at-once residual of the shard's slices (the slice before t0 read from its
//   owner) -> host sums of the partials.
// Step k of one ParaDIAG run on shard p (tables: row tables of f, g, w, u over all shards), enqueued on the shard's
// stream: 1 = step-1 transform, 2 = the shard's shifted solves, 3 = step-3 transform, 4 = the all-at-once residual of
// the shard's slices (partials to s.h_partial).  Cross-shard ordering is the caller's (events + barriers, or a
// process barrier in rank mode).
void Paradiag::phase(int p, int k, const RowTab (&T)[4], pdmg_solve_report* rep) {
  PdShard& s = *sh[p];
  EngineBase& E = *s.eng;
  cudaStream_t st = E.stream;
  const double slice_bytes = sizeof(double2) * (double)npts;
  const int P = (int)sh.size();
  if (k == 1 || k == 3) {  // g = (V^{-1} (x) I) f (kron_time_solve, paradiag.cpp:135-139); u = (V (x) I) w (:129-133)
    const RowTab &in = T[k == 1 ? 0 : 2], &out = T[k == 1 ? 1 : 3];
    E.timed(general ? "time_gemm" : "time_dft", 2.0 * slice_bytes * nt * (double)(s.pt1 - s.pt0) / npts, [&] {
      if (general) launch_gemm(k == 1 ? s.Vi : s.V, nt, in, out, 0, nt, 0, s.pt0, s.pt1, st);
      else launch_dft(k == 1 ? *s.t1 : *s.t3, in, out, s.pt0, s.pt1, st);
    });
  } else if (k == 2) {  // the shard's shifted solves (paradiag.cpp:207-236)
    pdmg_solve_report rc{};
    if (rep) {
      const int64_t Hn = E.cfg.max_iter + 1;
      rc.iterations = rep->iterations ? rep->iterations + s.t0 : nullptr;
      rc.converged = rep->converged ? rep->converged + s.t0 : nullptr;
      rc.residual_history = rep->residual_history ? rep->residual_history + s.t0 * Hn : nullptr;
      rc.rate = rep->rate ? rep->rate + s.t0 : nullptr;
    }
    E.solve_device(s.g, s.w, rep ? &rc : nullptr);
  } else {  // relres = ||f - K u|| / ||f|| (paradiag.cpp:243-245)
    double2* up = T[3].p[p];
    const double2* fp = T[0].p[p];
    E.timed("aao_residual", 3.0 * slice_bytes * s.cnt, [&] {
      if (general) {
        const RowTab Ty = rowtab({s.y}, s.cnt, npts);
        launch_gemm(s.B, nt, T[3], Ty, s.t0, s.t0 + s.cnt, s.t0, 0, npts, st);  // (B (x) I) u on the shard's rows
        k_aao_residual_dense<<<res_blocks, 256, 0, st>>>(up, s.y, fp, n, s.cnt, s.partial);
      } else {
        const int q = (p + P - 1) % P;  // owner of slice t0 - 1 (slice nt - 1 for t0 = 0)
        const double2* prev = T[3].p[q] + (int64_t)(sh[q]->cnt - 1) * npts;
        k_aao_residual<<<res_blocks, 256, 0, st>>>(up, prev, fp, n, s.cnt, s.t0, alpha, dt, s.partial);
      }
      CK(cudaGetLastError());
    });
    CK(cudaMemcpyAsync(s.h_partial, s.partial, sizeof(double) * 2 * res_blocks, cudaMemcpyDeviceToHost, st));
  }
}

// One host thread per shard; the cross-device order of the phases is carried by events, recorded before a host
// barrier and waited on after it:
//   [input ready] -> step 1 transform (gather f columns from every shard, scatter g rows to their owners)
//   -> [g ready everywhere] -> the shard's shifted solves -> [w ready everywhere] -> step 3 transform
//   -> [u ready everywhere] -> all-at-once residual of the shard's slices (the slice before t0 read from its
//   owner) -> host sums of the partials.
void Paradiag::run_impl(const double2* const* f, double2* const* u, pdmg_solve_report* rep, double* relres,
                        const pdmg_c128* hf, pdmg_c128* hu) {
  if (local >= 0) throw ConfigError("ParaDIAG: a per-rank solver runs through pdmg_paradiag_rank_phase");
  const int P = (int)sh.size();
  std::vector<double2*> fp(P), gp(P), wp(P), up(P);
  for (int p = 0; p < P; ++p) {
    fp[p] = const_cast<double2*>(f ? f[p] : sh[p]->f);
    up[p] = u ? u[p] : sh[p]->u;
    gp[p] = sh[p]->g, wp[p] = sh[p]->w;
  }
  const int rows = sh[0]->cnt;
  const RowTab T[4] = {rowtab(fp, rows, npts), rowtab(gp, rows, npts), rowtab(wp, rows, npts), rowtab(up, rows, npts)};
  Barrier bar(P);
  std::vector<std::exception_ptr> err(P);
  std::vector<double> sums(2 * P, 0.0);
  auto body = [&](int p) {
    PdShard& s = *sh[p];
    EngineBase& E = *s.eng;
    cudaStream_t st = E.stream;
    CK(cudaSetDevice(s.device));
    const double slice_bytes = sizeof(double2) * (double)npts;
    if (hf) CK(cudaMemcpyAsync(fp[p], hf + (int64_t)s.t0 * npts, slice_bytes * s.cnt, cudaMemcpyHostToDevice, st));
    for (int k = 1; k <= 4; ++k) {
      CK(cudaEventRecord(s.ev[k - 1], st));
      bar.wait();
      for (auto& o : sh) CK(cudaStreamWaitEvent(st, o->ev[k - 1], 0));
      if (k == 4) {
        if (hu) CK(cudaMemcpyAsync(hu + (int64_t)s.t0 * npts, up[p], slice_bytes * s.cnt, cudaMemcpyDeviceToHost, st));
        if (!relres) break;
      }
      phase(p, k, T, rep);
    }
    CK(cudaStreamSynchronize(st));
    if (relres)
      for (int b = 0; b < res_blocks; ++b) sums[2 * p] += s.h_partial[2 * b], sums[2 * p + 1] += s.h_partial[2 * b + 1];
    E.drain_stats();
  };
  std::vector<std::thread> th;
  for (int p = 0; p < P; ++p)
    th.emplace_back([&, p] {
      try {
        body(p);
      } catch (const BarrierBroken&) {  // another shard failed
        cudaStreamSynchronize(sh[p]->eng->stream);
      } catch (...) {
        err[p] = std::current_exception();
        bar.fail();
        cudaStreamSynchronize(sh[p]->eng->stream);
      }
    });
  for (auto& t : th) t.join();
  for (auto& x : err)
    if (x) std::rethrow_exception(x);
  if (relres) {
    double rr = 0.0, ff = 0.0;
    for (int p = 0; p < P; ++p) rr += sums[2 * p], ff += sums[2 * p + 1];
    *relres = ff > 0.0 ? std::sqrt(rr) / std::sqrt(ff) : std::sqrt(rr);
  }
}

// ---- rank mode: one process per GPU, the other shards' buffers opened over CUDA IPC ---------------------------------
void Paradiag::setup_rank(int n_, int nt_, double alpha_, double dt_, const pdmg_mg_config& cfg, int rank,
                          int nranks, int device) {
  if (nt_ < 2) throw ConfigError("TimeDiscretization: need n >= 2 time steps");
  if (!(dt_ > 0.0)) throw ConfigError("TimeDiscretization: tau must be positive");
  if (!(alpha_ != 0.0)) throw ConfigError("alpha-circulant: alpha must be nonzero");
  if (nranks < 1 || nranks > MAX_SHARDS || rank < 0 || rank >= nranks)
    throw ConfigError("ParaDIAG: rank " + std::to_string(rank) + " of " + std::to_string(nranks) + " (1..16 ranks)");
  const int chunk = (nt_ + nranks - 1) / nranks;
  if ((int64_t)(nranks - 1) * chunk >= nt_)
    throw ConfigError("ParaDIAG: " + std::to_string(nt_) + " time steps leave a rank without slices at " +
                      std::to_string(nranks) + " ranks");
  check_dft_size(nt_);
  general = false, alpha = alpha_, dt = dt_;
  n = n_, nt = nt_;
  npts = (int64_t)(n - 1) * (n - 1);
  local = rank;
  std::vector<pdmg_c128> lam(nt);
  pdmg_circulant_shifts(alpha, nt, dt, 0, nt, lam.data());
  for (int t = 0; t < nranks; ++t) {
    auto s = std::make_unique<PdShard>();
    s->t0 = t * chunk, s->cnt = std::min(nt, s->t0 + chunk) - s->t0;
    s->pt0 = npts * t / nranks, s->pt1 = npts * (t + 1) / nranks;
    s->remote = t != rank;
    s->device = t == rank ? device : -1;
    sh.push_back(std::move(s));
  }
  PdShard& s = *sh[rank];
  pdmg_batch_desc d{n, s.cnt, lam.data() + s.t0, cfg, PDMG_PREC_C128, device};
  s.eng = make_engine_c128();
  s.eng->device = -1;
  s.eng->setup_host(d);
  s.eng->setup_device(device);
  CK(cudaSetDevice(device));
  const size_t bytes = sizeof(double2) * (size_t)s.cnt * npts;
  for (double2** q : {&s.f, &s.g, &s.w, &s.u}) CK(cudaMalloc(q, bytes));
  CK(cudaMalloc(&s.partial, sizeof(double) * 2 * res_blocks));
  CK(cudaMallocHost(&s.h_partial, sizeof(double) * 2 * res_blocks));
  for (auto& e : s.ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  dft_attr(device);
  s.t1 = make_dft_tables(nt, alpha, 1, s.eng->stream);
  s.t3 = make_dft_tables(nt, alpha, 3, s.eng->stream);
}

void Paradiag::ipc_handles(void* out) const {
  if (local < 0) throw ConfigError("pdmg_paradiag_ipc_handles: not a per-rank solver");
  const PdShard& s = *sh[local];
  CK(cudaSetDevice(s.device));
  cudaIpcMemHandle_t h[4];
  const double2* bufs[4] = {s.f, s.g, s.w, s.u};
  for (int k = 0; k < 4; ++k) CK(cudaIpcGetMemHandle(&h[k], const_cast<double2*>(bufs[k])));
  std::memcpy(out, h, sizeof(h));
}

void Paradiag::open_peers(const void* all) {
  if (local < 0) throw ConfigError("pdmg_paradiag_open_peers: not a per-rank solver");
  CK(cudaSetDevice(sh[local]->device));
  const auto* h = static_cast<const cudaIpcMemHandle_t*>(all);
  for (size_t p = 0; p < sh.size(); ++p) {
    if ((int)p == local) continue;
    PdShard& s = *sh[p];
    double2** bufs[4] = {&s.f, &s.g, &s.w, &s.u};
    for (int k = 0; k < 4; ++k) {
      if (*bufs[k]) CK(cudaIpcCloseMemHandle(*bufs[k]));
      void* ptr = nullptr;
      CK(cudaIpcOpenMemHandle(&ptr, h[p * 4 + k], cudaIpcMemLazyEnablePeerAccess));
      *bufs[k] = static_cast<double2*>(ptr);
    }
  }
  peers_open = true;
}

void Paradiag::rank_phase(int k, pdmg_solve_report* rep, double* sums) {
  if (local < 0) throw ConfigError("pdmg_paradiag_rank_phase: not a per-rank solver");
  if (!peers_open && sh.size() > 1) throw ConfigError("pdmg_paradiag_rank_phase: peers not opened");
  if (k < 1 || k > 4) throw ConfigError("pdmg_paradiag_rank_phase: phase must be 1..4");
  const int P = (int)sh.size();
  std::vector<double2*> fp(P), gp(P), wp(P), up(P);
  for (int p = 0; p < P; ++p) fp[p] = sh[p]->f, gp[p] = sh[p]->g, wp[p] = sh[p]->w, up[p] = sh[p]->u;
  const int rows = sh[0]->cnt;
  const RowTab T[4] = {rowtab(fp, rows, npts), rowtab(gp, rows, npts), rowtab(wp, rows, npts), rowtab(up, rows, npts)};
  PdShard& s = *sh[local];
  CK(cudaSetDevice(s.device));
  phase(local, k, T, rep);
  CK(cudaStreamSynchronize(s.eng->stream));  // this rank's part of the phase is complete (peer writes included)
  if (k == 4 && sums) {
    sums[0] = sums[1] = 0.0;
    for (int b = 0; b < res_blocks; ++b) sums[0] += s.h_partial[2 * b], sums[1] += s.h_partial[2 * b + 1];
  }
  s.eng->drain_stats();
}

void Paradiag::run_shards(const double2* const* f, double2* const* u, pdmg_solve_report* rep, double* relres) {
  const auto t0 = std::chrono::steady_clock::now();
  run_impl(f, u, rep, relres, nullptr, nullptr);
  if (rep) rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void Paradiag::run_device(const double2* f, double2* u, pdmg_solve_report* rep, double* relres) {
  if (sh.size() != 1)
    throw ConfigError("pdmg_paradiag_run_device: the solver spans " + std::to_string(sh.size()) +
                      " devices; pass per-shard buffers to pdmg_paradiag_run_shards");
  run_shards(&f, &u, rep, relres);
}

void Paradiag::run_host(const pdmg_c128* f, pdmg_c128* u, pdmg_solve_report* rep, double* relres) {
  const auto t0 = std::chrono::steady_clock::now();
  run_impl(nullptr, nullptr, rep, relres, f, u);
  if (rep) rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- single-device building blocks of the multi-process driver (paradiag_dist.py) ---------------------------------
void aao_residual_sums(int device, int n, int ntl, int t0, double alpha, double dt, const double2* u,
                       const double2* u_prev, const double2* f, double* sums, cudaStream_t st) {
  CK(cudaSetDevice(device));
  constexpr int blocks = 148 * 8;
  // per-thread cached device/pinned partial buffers (no allocation per call)
  struct Buf {
    int dev = -1;
    double *d = nullptr, *h = nullptr;
  };
  thread_local std::vector<Buf> bufs;
  Buf* b = nullptr;
  for (auto& x : bufs)
    if (x.dev == device) b = &x;
  if (!b) {
    bufs.push_back(Buf{device});
    b = &bufs.back();
    CK(cudaMalloc(&b->d, sizeof(double) * 2 * blocks));
    CK(cudaMallocHost(&b->h, sizeof(double) * 2 * blocks));
  }
  k_aao_residual<<<blocks, 256, 0, st>>>(u, u_prev, f, n, ntl, t0, alpha, dt, b->d);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(b->h, b->d, sizeof(double) * 2 * blocks, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  sums[0] = sums[1] = 0.0;
  for (int q = 0; q < blocks; ++q) sums[0] += b->h[2 * q], sums[1] += b->h[2 * q + 1];
}

void time_transform(int device, cudaStream_t st, int nt, int64_t npts, const double2* dM, const double2* dX,
                    double2* dY) {
  CK(cudaSetDevice(device));
  const RowTab X = rowtab({const_cast<double2*>(dX)}, nt, npts), Y = rowtab({dY}, nt, npts);
  launch_gemm(dM, nt, X, Y, 0, nt, 0, 0, npts, st);
}

void time_dft(int device, int nt, int64_t npts, double alpha, int step, const double2* in, double2* out,
              cudaStream_t st) {
  CK(cudaSetDevice(device));
  dft_attr(device);
  // tables cached per (device, nt, alpha, step)
  struct Key {
    int dev, nt, step;
    double alpha;
    bool operator<(const Key& o) const {
      return std::tie(dev, nt, step, alpha) < std::tie(o.dev, o.nt, o.step, o.alpha);
    }
  };
  static std::mutex mu;
  static std::map<Key, std::unique_ptr<DftTables>> cache;
  const DftTables* T = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto& e = cache[Key{device, nt, step, alpha}];
    if (!e) e = make_dft_tables(nt, alpha, step, st);
    T = e.get();
  }
  launch_dft(*T, rowtab({const_cast<double2*>(in)}, nt, npts), rowtab({out}, nt, npts), 0, npts, st);
}

}  // namespace pdmg_b200
