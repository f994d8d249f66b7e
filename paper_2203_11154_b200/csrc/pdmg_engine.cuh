// pdmg_engine.cuh -- the batched multigrid engine (host orchestration of the sm_100a kernels in
// pdmg_kernels.cuh) for one batch of shifts on one device, templated on the storage type T (double:
// complex128, float: complex64).  Mirrors the reference solver path (proj/src/multigrid.cpp) for a BATCH of
// shifts: one engine holds, for every shift, what one pdmg::MultigridHierarchy holds (level list,
// per-level smoother coefficients, coarsest factorization) plus device storage for all levels.  Every
// cycle is a short sequence of batched level passes over all still-active shifts; convergence is decided
// on the device per shift (k_finalize) exactly as in MultigridHierarchy::solve, so per-shift cycle counts
// match the reference.
#pragma once
#include <array>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "pdmg_host.h"
#include "pdmg_kernels.cuh"
#include "pdmg_march2_table.h"

// compile the hot marching passes with the level's n as a constant (n = 256, 512, 1024; complex128)
#ifndef PDMG_MARCH2_NF
#define PDMG_MARCH2_NF 1
#endif

namespace pdmg_b200 {

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

// fused Vanka passes (k_march2): key = loadu | prolong << 1 | post << 2 | norm_in << 4.  The kernels are instantiated
// in their own translation units (pdmg_march2_units.cuh); the table is filled through pdmg_march2_table.h.
template <class T>
struct March2Table {
  using Fn = March2Fn<T>;
  Fn e[32] = {};   // two sweeps per pass
  Fn e1[32] = {};  // one sweep per pass (k_march2<..., TWO = false>)
  // the hot variants with the level's n compiled in (NF): [n = 256, 512, 1024, 128][key]
  Fn eN[4][32] = {}, e1N[4][32] = {};
  static int nf_slot(int n) { return n == 256 ? 0 : n == 512 ? 1 : n == 1024 ? 2 : n == 128 ? 3 : -1; }
  static int key(bool lu, bool pr, int post, bool nin = false) { return march2_key(lu, pr, post, nin); }
  March2Table() {
    march2_fill_two(e);
    march2_fill_one(e1);
#if PDMG_MARCH2_NF
    march2_fill_hot_256(eN[0], e1N[0]);
    march2_fill_hot_512(eN[1], e1N[1]);
    march2_fill_hot_1024(eN[2], e1N[2]);
    march2_fill_hot_128(eN[3], e1N[3]);
#endif
  }
};


template <class T>
struct Engine : EngineBase {
  using V = typename vec2<T>::type;
  struct Level {
    int n = 0, m = 0;
    int64_t ss = 0;  // shift stride (elements)
    size_t elems = 0;
    int64_t alloc_left = 0;  // elements from this view's start to the end of the allocation (bounds checks)
    V* u[2] = {nullptr, nullptr};
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
  // rolling host solve (solve_rolling): per-shift cycle counters and final-buffer indices, the identity table k_pack
  // reads them through, the round's active flags in mapped memory (two slots of S ints after the counts)
  int *d_kcur = nullptr, *d_fbuf = nullptr, *d_ident = nullptr;
  bool rolling = false;
  int roll_slot = 0;
  cudaStream_t out_stream = nullptr;
  size_t map_flags() const { return map_nact() + 8 * sizeof(int); }
  int n_active_host = 0;
  const KernelTable<T>* table = nullptr;
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
  // strips across a row of a k_march2 pass: 64 columns each, WOUT = 64 - 2 hA apart, the last one ending at the
  // domain edge (k_march2's sA)
  static int march2_ntx(int n, int ha) {
    const int wout = 64 - 2 * ha;
    return n <= 64 ? 1 : 1 + (n - 64 + wout - 1) / wout;
  }
  int march2_tasks(int n, int post, bool two, bool prolong) const {  // warp tasks per shift of a k_march2 pass
    const int hs = march2_hs_for(n, prolong, post, two);
    return march2_ntx(n, march2_ha(post, two)) * ((n + hs - 1) / hs);
  }
  static constexpr int kMinStrip = 16;  // smallest strip height the wave model may pick (partial-buffer sizing)
  int sm_count = 148;
  // Strip height of a k_march2 pass.  The measured defaults (128 rows for n >= 512, 64 for n = 256, 32 below;
  // DESIGN 3.2b, at C3's 256 shifts) unless a wave model of the launch finds a clearly shorter pass: a warp marches
  // Hs + 2 hA rows, CTAs of MARCH_WARPS strips run in waves of (SMs x resident CTAs), and the pass takes about
  // waves x (Hs + 2 hA) row steps.  Small batches (strong scaling: 32 shifts per GPU) leave the default's last wave
  // nearly empty; shorter strips fill it (C3 with 32 shifts: n = 512 passes at Hs = 96 instead of 128).
  int march2_hs_for(int n, bool prolong, int post = POST_NONE, bool two = true) const {
    if (march2_hs > 0) return march2_hs;
    for (auto& e : prolong ? march2_hs_p : march2_hs_r)
      if (e.first == n) return e.second;
    const int def = n >= 512 ? 128 : n >= 256 ? 64 : 32;
    const int ha = march2_ha(post, two), ntx = march2_ntx(n, ha);
    const int wpc = two ? m2_wpc : m1_wpc;
    const int64_t slots = (int64_t)sm_count * (march2_warps_per_sm(two) / wpc);
    auto cost = [&](int hs) {
      const int64_t ctas = (int64_t)((ntx * ((n + hs - 1) / hs) + wpc - 1) / wpc) * S;
      return (double)((ctas + slots - 1) / slots) * (hs + 2 * ha);
    };
    int best = def;
    double bc = 0.95 * cost(def);  // the default keeps a 5% preference (it is the measured optimum at C3)
    for (int hs = kMinStrip; hs <= 256 && hs <= n + (n & 1); hs += 8) {
      const double c = cost(hs);
      if (c < bc) best = hs, bc = c;
    }
    return best;
  }
  int m2_wpc = 4, m1_wpc = 4;  // warps per CTA of the two-sweep / one-sweep marching passes (PDMG_M2_WPC, PDMG_M1_WPC)
  bool march2_pre = true, march2_post = true;  // fuse the pre- / post-smoothing sweep pairs
  int march2_loopb_min_n = 128;  // (prolongating passes: shape (a), see march2_prolong_b)
  bool norm_next = true;  // fine-level convergence norm from the next cycle's first pass (see solve_device)
  double pred_final = 0.5;  // predicted-last-norm threshold (solve_device; 0 = off, PDMG_PRED_FINAL)
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
                   const int* active, int n_act, bool norm_in = false, bool two = true) {
    const Level& Lv = lv[l];
    MarchArgs<T> ma{};
    ma.u_in = uin, ma.u_out = uout, ma.b = b, ma.ec = ec, ma.bc = bc, ma.partial = d_partial;
    ma.coef = Lv.coef, ma.active = active, ma.n = Lv.n;
    ma.nc = (l + 1 < (int)lv.size()) ? lv[l + 1].n : Lv.n / 2;
    ma.ss = Lv.ss, ma.ssc = (l + 1 < (int)lv.size()) ? lv[l + 1].ss : 0;
    ma.elems = Lv.alloc_left, ma.elems_c = (l + 1 < (int)lv.size()) ? lv[l + 1].alloc_left : 0;
    ma.Hs = march2_hs_for(Lv.n, prolong, post, two);
    // loop shape (a) for prolongating passes unless march2_prolong_b (measured, DESIGN 3.2b)
    ma.loop_a = Lv.n < march2_loopb_min_n || (prolong && !march2_prolong_b);
    ma.ntx = march2_ntx(Lv.n, march2_ha(post, two));
    ma.ntasks = ma.ntx * ((Lv.n + ma.Hs - 1) / ma.Hs);
    if (ma.ntasks != march2_tasks(Lv.n, post, two, prolong)) throw std::logic_error("pdmg_b200: march2 task count");
    const int key2 = March2Table<T>::key(loadu, prolong, post, norm_in);
    auto fn = two ? marches2().e[key2] : marches2().e1[key2];
    if (const int sl = March2Table<T>::nf_slot(Lv.n); sl >= 0) {
      auto fnN = two ? marches2().eN[sl][key2] : marches2().e1N[sl][key2];
      if (fnN) fn = fnN;
    }
    if (!fn) throw std::logic_error("pdmg_b200: no two-sweep kernel for this variant");
    const double S_ = sizeof(V), pts = (double)n_act * Lv.m * Lv.m;
    const double bpp = (loadu ? S_ : 0) + S_ + (prolong ? S_ / 4 : 0) + S_ + (post == POST_RESTRICT ? S_ / 4 : 0);
    std::string cls = "L" + std::to_string(l) + ":" + (prolong ? (loadu ? "prolong+" : "prolong0+") : (loadu ? "" : "zero+")) +
                      (two ? "vanka2" : "vanka") + (post == POST_NORM ? "+norm" : post == POST_RESTRICT ? "+restrict" : "") +
                      (norm_in ? "+norm_in" : "");
    const double ubpp = (two ? 2 : 1) * 3 * S_ + (prolong ? S_ / 4 : 0) + (post == POST_RESTRICT ? S_ / 4 : 0);
    timed(cls, pts * bpp, [&] {
      for (int c0 = 0; c0 < S; c0 += COEF_MAX) {  // one launch per COEF_MAX shifts (coefficients as parameters)
        const int cnt = std::min(COEF_MAX, S - c0);
        fill_pack(Lv, c0, cnt);
        const int wpc = two ? m2_wpc : m1_wpc;
        dim3 grid((ma.ntasks + wpc - 1) / wpc, cnt);
        fn<<<grid, 32 * wpc, (size_t)wpc * M2_SMEM_PER_WARP, stream>>>(ma, *cpack);
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
    cudaFree(d_kcur);
    cudaFree(d_fbuf);
    cudaFree(d_ident);
    if (out_stream) cudaStreamDestroy(out_stream);
    cudaFree(d_ones);
    cudaFree(d_r0);
    cudaFree(d_hist);
    cudaFree(d_partial);
    cudaFree(d_norms);
    cudaFree(d_stage);
    if (h_map) cudaFreeHost(h_map);
    for (auto e : ev_nactive)
      if (e) cudaEventDestroy(e);
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
    if (const char* e = std::getenv("PDMG_TAIL_MAX_N")) tail_max_n = std::atoi(e);
    if (const char* e = std::getenv("PDMG_MARCH2_MIN_N")) march2_min_n = std::atoi(e);  // (tuning)
    if (const char* e = std::getenv("PDMG_MARCH_MIN_N")) march_min_n = std::atoi(e);    // (tuning)
    if (const char* e = std::getenv("PDMG_IO_CHUNKS")) io_chunks = std::atoi(e);
    if (const char* e = std::getenv("PDMG_IO_MODE")) io_mode = std::atoi(e);
    if (const char* e = std::getenv("PDMG_ROLL_LANES")) roll_lanes = std::atoi(e);
    if (const char* e = std::getenv("PDMG_ROLL_PIECE")) roll_piece = std::atoi(e);
    if (const char* e = std::getenv("PDMG_SMALL_THREADS")) small_threads_env = std::atoi(e);
    if (const char* e = std::getenv("PDMG_SMALL_CLUSTER")) small_cluster = std::atoi(e);
    if (const char* e = std::getenv("PDMG_SMALL_CLUSTER_NODES")) small_cluster_min_nodes = std::atoi(e);
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
    if (const char* e = std::getenv("PDMG_MARCH1")) march1 = std::atoi(e) != 0;
    if (const char* e = std::getenv("PDMG_M2_WPC")) m2_wpc = std::max(1, std::min(8, std::atoi(e)));
    if (const char* e = std::getenv("PDMG_M1_WPC")) m1_wpc = std::max(1, std::min(8, std::atoi(e)));
    if (const char* e = std::getenv("PDMG_PRED_FINAL")) pred_final = std::atof(e);
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (dev < 0 || dev >= ndev) throw CudaError("pdmg_create: CUDA device " + std::to_string(dev) + " not available");
    CK(cudaSetDevice(dev));
    CK(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, stream_priority));
    CK(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));
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
        // Invariant every kernel keeps (the concurrent chunks run on these overlapping views at the same time): a
        // pass writes only cells of its own shifts [s * ss, (s + 1) * ss), and any cell it reads outside them (halo
        // or guard reads past the last shift, here the next chunk's first shift) only reaches results that are
        // masked to its own interior.  tests/test_gpu_parity.py::test_chunked_host_solve_marching_passes checks
        // the chunked results bitwise against one batch; PDMG_BOUNDS_CHECK builds assert the allocation bounds.
        if (borrow_s0 + S < borrow->S) Lv.elems = (size_t)Lv.ss * S;
        Lv.alloc_left = P.alloc_left - off;
      } else {
        Lv.alloc_left = (int64_t)Lv.elems;
        for (V** p : {&Lv.u[0], &Lv.u[1], &Lv.b}) {
          CK(cudaMalloc(p, Lv.elems * sizeof(V)));
          CK(cudaMemsetAsync(*p, 0, Lv.elems * sizeof(V), stream));
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
    // the coarse-solve kernels stage the coarsest right-hand side (coarse_N complex values) in dynamic shared
    // memory: opt in above the 48 KB default, and refuse grids whose coarsest level cannot fit (the reference
    // accepts coarsest_n up to 128, dense.cpp:9-15; 16 B per unknown caps it at 119 here)
    {
      int optin = 0;
      CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      const size_t need = (size_t)coarse_N * sizeof(double2), static_red = 33 * sizeof(double);
      if (need + static_red > (size_t)optin)
        throw ConfigError("MultigridHierarchy: coarsest grid n = " + std::to_string(nc) + " needs " +
                          std::to_string(need) + " B of shared memory for the batched direct solve (device limit " +
                          std::to_string(optin - (int)static_red) + " B; coarsest_n <= 119)");
      const int sm = (int)std::max<size_t>(need, 1);
      CK(cudaFuncSetAttribute(k_coarse_solve<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(cudaFuncSetAttribute(k_small_cycle<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(cudaFuncSetAttribute(k_small_solve<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    }
    CK(cudaMalloc(&d_ainv, sizeof(double2) * hinv.size()));
    CK(cudaMemcpyAsync(d_ainv, hinv.data(), sizeof(double2) * hinv.size(), cudaMemcpyHostToDevice, stream));
    // solve state
    int maxtiles = 1;
    for (size_t l = 0; l < lv.size(); ++l) {
      maxtiles = std::max(maxtiles, lv[l].ntiles);
      for (int post : {POST_NONE, POST_NORM, POST_RESTRICT}) {
        maxtiles = std::max(maxtiles, march_tasks((int)l, post));
        for (int two = 0; two < 2; ++two) {  // (any strip height the wave model may pick, any batch size)
          const int n = lv[l].n;
          maxtiles = std::max(maxtiles, march2_ntx(n, march2_ha(post, two != 0)) * ((n + kMinStrip - 1) / kMinStrip));
          for (int pr = 0; pr < 2; ++pr) maxtiles = std::max(maxtiles, march2_tasks(n, post, two != 0, pr != 0));
        }
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
    CK(cudaMalloc(&d_kcur, sizeof(int) * S));
    CK(cudaMalloc(&d_fbuf, sizeof(int) * S));
    CK(cudaMalloc(&d_ident, sizeof(int) * 2));
    const int ident[2] = {0, 1};
    CK(cudaMemcpyAsync(d_ident, ident, sizeof(ident), cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));  // (ident is a stack array)
    CK(cudaHostAlloc((void**)&h_map, map_flags() + 2 * sizeof(int) * (size_t)S, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&d_map, h_map, 0));
    CK(cudaEventCreateWithFlags(&ev_nactive[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_nactive[1], cudaEventDisableTiming));
    for (auto& kv : table->e)
      if (kv.fn) CK(cudaFuncSetAttribute(kv.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kv.smem));
    {  // the b-row rings of the fused Vanka passes: up to 8 warps per CTA (m2_wpc / m1_wpc)
      const March2Table<T>& mt = marches2();
      auto opt_in = [&](const typename March2Table<T>::Fn* f, int cnt) {
        for (int i = 0; i < cnt; ++i)
          if (f[i]) CK(cudaFuncSetAttribute(f[i], cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * M2_SMEM_PER_WARP));
      };
      opt_in(mt.e, 32), opt_in(mt.e1, 32);
      for (int q = 0; q < 4; ++q) opt_in(mt.eN[q], 32), opt_in(mt.e1N[q], 32);
    }
    CK(cudaStreamSynchronize(stream));
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
      level_pass2(l, v.loadu, v.prolong, v.post, uin, uout, b, ec, bc, active, n_act, norm_in, false);
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
  // (count: the CTAs that do work -- the batch, or the active shifts of a rolling round, whose other CTAs exit)
  int small_threads(int count = 0) const {
    if (small_threads_env > 0) return small_threads_env;
    if (count <= 0) count = S;
    return count <= sm_count ? SMALL_THREADS : count <= 2 * sm_count ? SMALL_THREADS / 2 : SMALL_THREADS / 4;
  }
  // Thread-block cluster size of a one-CTA-per-shift launch: when the shifts that do work are fewer than the SMs, a
  // cluster of 2, 4 or 8 full-size CTAs shares each shift (SmallSolver), as many as still fit one CTA per SM.
  int small_cluster = 8;  // largest cluster size (PDMG_SMALL_CLUSTER; 0 or 1: always one CTA per shift)
  int small_cluster_min_nodes = 8192;  // (PDMG_SMALL_CLUSTER_NODES) top-level nodes from which a cluster pays
  int small_cluster_size(int count, int threads, int top_n) const {
    if (small_cluster <= 1 || threads != SMALL_THREADS) return 1;
    if ((top_n - 1) * (top_n - 1) < small_cluster_min_nodes) return 1;
    if (count <= 0) count = S;
    // (clusters of 8 need 8 free SMs of one GPC each: only when they fill at most half the GPU -- 16 clusters of 8
    // measured no faster than single CTAs, 16 clusters of 4 1.5x faster;
    // and 36 clusters of 4 -- 144 of 148 SMs -- do not all fit their GPCs at once: 2.0 vs 1.7 ms)
    for (int c : {8, 4, 2})
      if (c <= small_cluster && (int64_t)count * c <= (c == 8 ? sm_count / 2 : c == 4 ? sm_count * 7 / 8 : sm_count)) return c;
    return 1;
  }
  template <class K>
  void launch_small(K kernel, int threads, int csize, size_t smem, const SmallArgs<T>& sa) {
    if (csize <= 1) {
      kernel<<<S, threads, smem, stream>>>(sa);
      return;
    }
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)S * csize), lc.blockDim = dim3(threads), lc.dynamicSmemBytes = smem, lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
    lc.attrs = at, lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, kernel, sa));
  }
  void tail_cycle(int l, const int* active, bool zero, int n_act = 0) {
    SmallArgs<T> sa{};
    for (size_t q = l; q < lv.size(); ++q)
      sa.lv[q - l] = SmallLevel<T>{lv[q].u[0], lv[q].u[1], lv[q].b, lv[q].coef, lv[q].n, lv[q].ss};
    sa.L = (int)lv.size() - l;
    sa.nu1 = cfg.nu1, sa.nu2 = cfg.nu2, sa.gamma = cfg.cycle == PDMG_CYCLE_W ? 2 : 1;
    sa.jacobi = cfg.smoother == PDMG_SMOOTHER_JACOBI, sa.max_iter = cfg.max_iter, sa.tol = cfg.tol;
    sa.ainv = d_ainv, sa.coarse_N = coarse_N, sa.active = active, sa.tail_zero = zero ? 1 : 0;
    const int cnt = (rolling || active == nullptr) ? n_act : 0, thr = small_threads(cnt);
    timed("coarse_tail", 0.0, [&] {
      launch_small(k_small_cycle<T>, thr, small_cluster_size(cnt, thr, lv[l].n), coarse_N * sizeof(double2), sa);
    });
    for (size_t q = l; q < lv.size(); ++q) lv[q].cur = 0, lv[q].uzero = false;
  }

  bool cycle_level(int l, bool zero, const int* active, int n_act, bool want_norm) {
    Level& Lv = lv[l];
    const int L = (int)lv.size();
    const bool jac = cfg.smoother == PDMG_SMOOTHER_JACOBI;
    if (l > 0 && l == tail_level()) {  // the whole coarse tail in one launch (each visit of a W-cycle)
      tail_cycle(l, active, zero, n_act);
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
    if (rolling) {  // per-shift counters; the round's active flags go to the host (slot roll_slot)
      const int slot = roll_slot;
      CK(cudaMemsetAsync(d_nactive + slot, 0, sizeof(int), stream));
      SolveState st{d_active, d_iters, d_conv, d_r0, d_hist, d_nactive + slot, S, cfg.max_iter, cfg.tol, nullptr, cur, nullptr};
      const int threads = 256, blocks = (S * 32 + threads - 1) / threads;
      timed("finalize", 0.0, [&] { k_finalize_roll<<<blocks, threads, 0, stream>>>(d_partial, ntiles, st, d_kcur, d_fbuf); });
      to_host(d_active, map_flags() + sizeof(int) * (size_t)S * slot, sizeof(int) * (size_t)S);
      CK(cudaEventRecord(ev_nactive[slot], stream));
      return;
    }
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
  void pack(const V* b0, const V* b1, const int* iters, const int* parity, double2* dst, int l) {
    const Level& Lv = lv[l];
    const int64_t total = (int64_t)S * Lv.m * Lv.m;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    timed("pack", (double)total * 2 * sizeof(V),
          [&] { k_pack<T><<<blocks, 256, 0, stream>>>(b0, b1, iters, parity, dst, Lv.n, Lv.ss, total); });
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
        launch_small(k_small_solve<T>, small_threads(), small_cluster_size(S, small_threads(), lv[0].n), coarse_N * sizeof(double2), sa);
      });
      CK(cudaGetLastError());
      CK(cudaMemsetAsync(d_parity, 0, sizeof(int) * H, stream));
      pack(F.u[0], F.u[1], d_iters, d_parity, d_u, 0);
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

  // Copy the per-shift report back; counts the smoother updates performed (sum over shifts of cycles).
  // own: only the shifts with own[s] != 0 are this engine's (a lane of the rolling solve)
  void finish_report(pdmg_solve_report* rep, std::chrono::steady_clock::time_point t0, int H,
                     const std::vector<char>* own = nullptr) {
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
    for (int s = 0; s < S; ++s)
      if (!own || (*own)[s]) cycles_done += it[s];
    last_updates = per_cycle * cycles_done;
    if (rep) {
      for (int s = 0; s < S; ++s) {
        if (own && !(*own)[s]) continue;
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
    std::vector<std::array<V*, 3>> saved_lv;
    std::vector<LevelCoef*> saved_coef;
    std::vector<size_t> saved_elems;
    std::vector<int64_t> saved_left;
    double2* ainv;
    int *act, *it, *cv, *ones;
    double *r0, *hist;
    RangeView(Engine& en, int s0, int cnt) : e(en), S0(en.S) {
      for (auto& L : e.lv) {
        saved_lv.push_back({L.u[0], L.u[1], L.b});
        saved_coef.push_back(L.coef);
        saved_elems.push_back(L.elems);
        L.u[0] += s0 * L.ss, L.u[1] += s0 * L.ss, L.b += s0 * L.ss, L.coef += s0;
        saved_left.push_back(L.alloc_left);
        L.alloc_left -= (int64_t)s0 * L.ss;
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
        e.lv[l].coef = saved_coef[l], e.lv[l].elems = saved_elems[l], e.lv[l].alloc_left = saved_left[l];
      }
      e.d_ainv = ainv, e.d_active = act, e.d_iters = it, e.d_conv = cv, e.d_ones = ones, e.d_r0 = r0, e.d_hist = hist;
      e.S = S0;
      e.s_base = 0;
    }
  };

  cudaStream_t copy_stream = nullptr;
  int io_chunks = 0;  // 0 = automatic
  int io_mode = 2;    // 2: rolling batch (solve_rolling); 1: chunks solve concurrently on sub-engines (own streams,
                      // priorities); 0: chunks on one stream (PDMG_IO_MODE)
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
      for (auto& e : subs) e->solve_path = solve_path, e->profiling = profiling;
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
      e->profiling = profiling;
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
    if (io_mode == 2 && io_chunks <= 0 && roll_piece > 0) nch = std::max(nch, 2);
    nch = std::max(1, std::min(nch, S));
    auto pinned = [](const void* p) {
      cudaPointerAttributes a{};
      if (cudaPointerGetAttributes(&a, p) != cudaSuccess) return (cudaGetLastError(), false);
      return a.type == cudaMemoryTypeHost;
    };
    // pageable caller buffers (a std::vector through the C++ facade): the chunked pipeline through the library's
    // pinned bounce buffers (a pageable cudaMemcpy is host-synchronous and would serialize it; page-locking the
    // caller's 2 GB per call measured 2.7x slower than this at C3).  PDMG_PAGEABLE=0: plain copies.
    bool staged = false;
    if (nch > 1 && !(pinned(b) && pinned(u))) {
      static const bool stage_on = [] {
        const char* e = std::getenv("PDMG_PAGEABLE");
        return !(e && std::atoi(e) == 0);
      }();
      if (stage_on && io_mode >= 1) staged = true;
      else nch = 1;
    }
    if (nch == 1) {
      h2d(b, st, N);
      solve_device(st, st + N, rep);
      d2h(st + N, u, N);
      CK(cudaStreamSynchronize(stream));
      return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    if (!copy_stream) CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    if (io_mode == 2 && io_chunks <= 0 && solve_rolling(b, u, rep, st, N, per, staged)) {
      if (rep) rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      return;
    }
    if (io_mode >= 1 && solve_concurrent(b, u, rep, st, N, per, staged)) {
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
  // Pageable host buffers go through pinned bounce buffers (the library's own): multi-threaded host copies into
  // a ring of pinned pieces, each piece's DMA queued as soon as it is filled; the output the same way back.
  static constexpr size_t kStagePiece = (size_t)32 << 20;  // bytes per bounce piece
  static constexpr int kStageRing = 4;                      // input pieces in flight
  struct Bounce {
    void* buf[kStageRing] = {};
    cudaEvent_t ev[kStageRing] = {};
    int n = 0;
    void ensure(int count) {
      for (; n < count; ++n) {
        CK(cudaMallocHost(&buf[n], kStagePiece));
        CK(cudaEventCreateWithFlags(&ev[n], cudaEventDisableTiming));
      }
    }
    ~Bounce() {
      for (int i = 0; i < n; ++i) cudaFreeHost(buf[i]), cudaEventDestroy(ev[i]);
    }
  };
  std::unique_ptr<Bounce> bounce_in, bounce_out;
  // Host copies of the bounce pipeline run on one persistent pool of worker threads shared by the input and all
  // output streams (no per-piece thread creation, no oversubscription of the host cores).
  // Host copy of a bounce-pipeline slice with non-temporal stores (AVX2, checked at run time): the destination is
  // either a pinned piece the DMA engine reads next or the caller's result buffer, neither of which is wanted in the
  // cache, and a plain memcpy of a 2 MB slice pays a read-for-ownership of every destination line.
#if defined(__x86_64__)
  __attribute__((target("avx2"))) static void stream_copy_avx2(void* dst, const void* src, size_t len) {
    char* d = (char*)dst;
    const char* q = (const char*)src;
    const size_t head = (32 - ((uintptr_t)d & 31)) & 31;
    if (head >= len) {
      std::memcpy(d, q, len);
      return;
    }
    std::memcpy(d, q, head);
    d += head, q += head, len -= head;
    size_t i = 0;
    for (; i + 128 <= len; i += 128) {
      const __m256i a = _mm256_loadu_si256((const __m256i*)(q + i)), b = _mm256_loadu_si256((const __m256i*)(q + i + 32));
      const __m256i c = _mm256_loadu_si256((const __m256i*)(q + i + 64)), e = _mm256_loadu_si256((const __m256i*)(q + i + 96));
      _mm256_stream_si256((__m256i*)(d + i), a), _mm256_stream_si256((__m256i*)(d + i + 32), b);
      _mm256_stream_si256((__m256i*)(d + i + 64), c), _mm256_stream_si256((__m256i*)(d + i + 96), e);
    }
    _mm_sfence();
    std::memcpy(d + i, q + i, len - i);
  }
#endif
  static void stream_copy(void* dst, const void* src, size_t len) {
#if defined(__x86_64__)
    static const bool avx2 = __builtin_cpu_supports("avx2") && !std::getenv("PDMG_NO_STREAM_COPY");
    if (avx2 && len >= 4096) {
      stream_copy_avx2(dst, src, len);
      return;
    }
#endif
    std::memcpy(dst, src, len);
  }
  struct CopyPool {
    std::mutex mu;
    std::condition_variable cv;
    struct Task {
      void* dst;
      const void* src;
      size_t len;
      std::atomic<int>* left;
    };
    std::vector<Task> q;
    std::vector<std::thread> th;
    bool stop = false;
    explicit CopyPool(int n) {
      for (int i = 0; i < n; ++i)
        th.emplace_back([this] {
          for (;;) {
            Task t;
            {
              std::unique_lock<std::mutex> lk(mu);
              cv.wait(lk, [&] { return stop || !q.empty(); });
              if (stop && q.empty()) return;
              t = q.back();
              q.pop_back();
            }
            stream_copy(t.dst, t.src, t.len);
            t.left->fetch_sub(1, std::memory_order_acq_rel);
          }
        });
    }
    ~CopyPool() {
      {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
      }
      cv.notify_all();
      for (auto& x : th) x.join();
    }
    static CopyPool& get() {
      static CopyPool pool([] {
        if (const char* e = std::getenv("PDMG_COPY_THREADS")) return std::max(1, std::atoi(e));
        return std::max(1, std::min(12, (int)std::thread::hardware_concurrency() * 3 / 4));  // (8 -> 12 of 16: ~8 % faster)
      }());
      return pool;
    }
  };
  static void parallel_memcpy(void* dst, const void* src, size_t bytes) {
    constexpr size_t slice = (size_t)2 << 20;
    if (bytes <= slice) {
      std::memcpy(dst, src, bytes);
      return;
    }
    CopyPool& P = CopyPool::get();
    std::atomic<int> left{0};
    {
      std::lock_guard<std::mutex> lk(P.mu);
      for (size_t o = 0; o < bytes; o += slice) {
        P.q.push_back({(char*)dst + o, (const char*)src + o, std::min(slice, bytes - o), &left});
        left.fetch_add(1, std::memory_order_relaxed);
      }
    }
    P.cv.notify_all();
    while (left.load(std::memory_order_acquire) > 0) std::this_thread::yield();
  }
  // host -> device through the input ring (on `st_`); returns after the last piece's DMA is queued
  void staged_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st_) {
    Bounce& B = *bounce_in;
    static thread_local int slot = 0;
    for (size_t o = 0; o < bytes; o += kStagePiece) {
      const size_t len = std::min(kStagePiece, bytes - o);
      const int k = slot++ % kStageRing;
      CK(cudaEventSynchronize(B.ev[k]));  // the piece's previous DMA has drained
      parallel_memcpy(B.buf[k], (const char*)src + o, len);
      CK(cudaMemcpyAsync((char*)dst + o, B.buf[k], len, cudaMemcpyHostToDevice, st_));
      CK(cudaEventRecord(B.ev[k], st_));
    }
  }
  // device -> host through two pinned pieces owned by the calling sub-engine (double-buffered)
  void staged_d2h(void* dst, const void* src, size_t bytes, cudaStream_t st_, Bounce& B) {
    int k = 0;
    size_t pend_o = 0, pend_len = 0;
    int pend_k = -1;
    for (size_t o = 0; o < bytes; o += kStagePiece) {
      const size_t len = std::min(kStagePiece, bytes - o);
      CK(cudaMemcpyAsync(B.buf[k], (const char*)src + o, len, cudaMemcpyDeviceToHost, st_));
      CK(cudaEventRecord(B.ev[k], st_));
      if (pend_k >= 0) {  // drain the previous piece while this one transfers
        CK(cudaEventSynchronize(B.ev[pend_k]));
        parallel_memcpy((char*)dst + pend_o, B.buf[pend_k], pend_len);
      }
      pend_k = k, pend_o = o, pend_len = len;
      k ^= 1;
    }
    if (pend_k >= 0) {
      CK(cudaEventSynchronize(B.ev[pend_k]));
      parallel_memcpy((char*)dst + pend_o, B.buf[pend_k], pend_len);
    }
  }

  // Rolling host solve: shifts join the batch as their right-hand sides arrive (pieces of ~32 MB on the copy
  // stream) and leave it as they converge (packed and copied back on an output stream while the others keep
  // cycling).  Every round is one multigrid cycle over the shifts active at that moment; each shift carries its own
  // cycle counter (k_finalize_roll), so its iterates, history and cycle count are those of the batch solve.
  // Compared with solving chunks on sub-engines, the GPU always works on everything that has arrived and results
  // start flowing back after the first shifts' last cycle instead of after a whole chunk.  The pieces are dealt
  // round-robin to `roll_lanes` lanes -- this engine and lane engines that work in the same level arrays (disjoint
  // shifts) on their own streams and host threads -- so that one lane's latency-bound coarse levels overlap the
  // other's fine-level passes.  Needs the norm-next scheme (the first fine pass of a round forms the convergence
  // norm); otherwise the chunked pipelines below run.
  int roll_lanes = 2;      // PDMG_ROLL_LANES
  int roll_piece = 0;      // shifts per piece (0 = ~32 MB); > 0 also takes small batches through the rolling solve (tests)
  std::vector<std::unique_ptr<Engine<T>>> lanes;
  struct RollShared {
    const pdmg_c128* b;
    pdmg_c128* u;
    pdmg_solve_report* rep;
    double2* st;
    size_t N;
    int64_t per;
    bool staged;
    std::vector<int> plo;  // piece p = shifts [plo[p], plo[p + 1])
    std::vector<cudaEvent_t> in;
    std::mutex mu;
    std::condition_variable cv;
    int in_ready = 0;
    std::exception_ptr in_err;
    std::chrono::steady_clock::time_point t0;
  };
  bool build_lanes(int nl) {
    if ((int)lanes.size() + 1 == nl) {
      for (auto& e : lanes) e->solve_path = solve_path, e->profiling = profiling;
      return true;
    }
    lanes.clear();
    std::vector<pdmg_c128> lam(S);
    for (int s = 0; s < S; ++s) lam[s] = pdmg_c128{lambdas[s].real(), lambdas[s].imag()};
    for (int l = 1; l < nl; ++l) {
      auto e = std::make_unique<Engine<T>>();
      pdmg_batch_desc d = desc_;
      d.n_shifts = S;
      d.lambdas = lam.data();
      e->device = -1;
      e->setup_host(d);
      e->borrow = this;
      e->borrow_s0 = 0;
      e->setup_device(device);
      e->solve_path = solve_path;
      e->profiling = profiling;
      lanes.push_back(std::move(e));
    }
    return true;
  }

  bool solve_rolling(const pdmg_c128* b, pdmg_c128* u, pdmg_solve_report* rep, double2* st, size_t N, int64_t per,
                     bool staged) {
    if (!use_norm_next() || any_singular || use_small_path() || cfg.max_iter < 1) return false;
    RollShared sh;
    sh.b = b, sh.u = u, sh.rep = rep, sh.st = st, sh.N = N, sh.per = per, sh.staged = staged;
    sh.t0 = std::chrono::steady_clock::now();
    // pieces of whole shifts, ~32 MB each (C3: 8 shifts)
    const int pshift = roll_piece > 0 ? std::min(roll_piece, S)
                                      : (int)std::max<int64_t>(1, std::min<int64_t>(S, (int64_t)(kStagePiece / (per * sizeof(double2)))));
    for (int s = 0; s < S; s += pshift) sh.plo.push_back(s);
    const int np = (int)sh.plo.size();
    sh.plo.push_back(S);
    const int nl = std::max(1, std::min(std::min(roll_lanes, 4), np));
    if (!build_lanes(nl)) return false;
    sh.in.resize(np);
    for (auto& e : sh.in) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    // ---- input: all pieces queue on the copy stream (pageable: through the pinned bounce ring, on a thread) ----
    std::thread in_thread;
    if (staged) {
      if (!bounce_in) bounce_in = std::make_unique<Bounce>();
      bounce_in->ensure(kStageRing);
      in_thread = std::thread([&] {
        try {
          CK(cudaSetDevice(device));
          for (int p = 0; p < np; ++p) {
            staged_h2d(st + sh.plo[p] * per, b + sh.plo[p] * per, sizeof(double2) * per * (sh.plo[p + 1] - sh.plo[p]),
                       copy_stream);
            CK(cudaEventRecord(sh.in[p], copy_stream));
            std::lock_guard<std::mutex> lk(sh.mu);
            sh.in_ready = p + 1;
            sh.cv.notify_all();
          }
        } catch (...) {
          std::lock_guard<std::mutex> lk(sh.mu);
          sh.in_err = std::current_exception();
          sh.in_ready = np;
          sh.cv.notify_all();
        }
      });
    } else {
      for (int p = 0; p < np; ++p) {
        CK(cudaMemcpyAsync(st + sh.plo[p] * per, b + sh.plo[p] * per, sizeof(double2) * per * (sh.plo[p + 1] - sh.plo[p]),
                           cudaMemcpyHostToDevice, copy_stream));
        CK(cudaEventRecord(sh.in[p], copy_stream));
      }
      sh.in_ready = np;
    }
    std::vector<std::exception_ptr> err(nl);
    std::vector<std::thread> th;
    for (int l = 1; l < nl; ++l)
      th.emplace_back([&, l] {
        try {
          CK(cudaSetDevice(device));
          lanes[l - 1]->roll_lane(sh, l, nl);
        } catch (...) {
          err[l] = std::current_exception();
        }
      });
    try {
      roll_lane(sh, 0, nl);
    } catch (...) {
      err[0] = std::current_exception();
    }
    for (auto& t : th) t.join();
    if (in_thread.joinable()) in_thread.join();
    cudaStreamSynchronize(copy_stream);
    for (auto e : sh.in) cudaEventDestroy(e);
    for (auto& x : err)
      if (x) std::rethrow_exception(x);
    if (sh.in_err) std::rethrow_exception(sh.in_err);
    for (auto& e : lanes) {  // (each lane drained its own events at the end of its solve)
      last_updates += e->last_updates, launches += e->launches, e->launches = 0;
      for (auto& kv : e->stats) {
        Stat& q = stats[kv.first];
        q.launches += kv.second.launches, q.ms += kv.second.ms, q.bytes += kv.second.bytes;
        q.ubytes += kv.second.ubytes, q.updates += kv.second.updates;
      }
      e->stats.clear();
    }
    return true;
  }

  // One lane of the rolling solve: pieces lane, lane + nl, ... of sh (this engine's streams; the level arrays may be
  // a parent's, shared with the other lanes, which touch other shifts).
  void roll_lane(RollShared& sh, int lane, int nl) {
    Level& F = lv[0];
    const int H = cfg.max_iter + 1;
    const int64_t per = sh.per;
    const size_t N = sh.N;
    double2* st = sh.st;
    const bool staged = sh.staged;
    const int np = (int)sh.in.size();
    static const bool dbg = std::getenv("PDMG_IO_DEBUG") != nullptr;
    if (!out_stream) CK(cudaStreamCreateWithFlags(&out_stream, cudaStreamNonBlocking));
    std::vector<int> mine;  // this lane's pieces, in arrival order
    for (int p = lane; p < np; p += nl) mine.push_back(p);
    const int nm = (int)mine.size();
    int n_mine = 0;
    for (int p : mine) n_mine += sh.plo[p + 1] - sh.plo[p];
    // ---- output: finished runs of shifts are packed on the output stream; pinned destinations are copied there,
    // pageable ones by an output thread through two pinned bounce pieces ----
    struct OutItem {
      int s0, s1;
      cudaEvent_t packed;
    };
    std::mutex out_mu;
    std::condition_variable out_cv;
    std::vector<OutItem> out_q;
    bool out_stop = false;
    std::exception_ptr out_err;
    std::thread out_thread;
    if (staged) {
      if (!bounce_out) bounce_out = std::make_unique<Bounce>();
      bounce_out->ensure(2);
      out_thread = std::thread([&] {
        try {
          CK(cudaSetDevice(device));
          cudaStream_t ds;
          CK(cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking));
          for (size_t next = 0;;) {
            OutItem it;
            {
              std::unique_lock<std::mutex> lk(out_mu);
              out_cv.wait(lk, [&] { return out_stop || next < out_q.size(); });
              if (next >= out_q.size()) break;
              it = out_q[next++];
            }
            CK(cudaStreamWaitEvent(ds, it.packed, 0));
            staged_d2h(sh.u + it.s0 * per, st + N + it.s0 * per, sizeof(double2) * per * (it.s1 - it.s0), ds, *bounce_out);
          }
          CK(cudaStreamSynchronize(ds));
          cudaStreamDestroy(ds);
        } catch (...) {
          out_err = std::current_exception();
        }
      });
    }
    std::vector<cudaEvent_t> packed_events;
    auto emit = [&](int s0, int s1, cudaEvent_t after) {
      CK(cudaStreamWaitEvent(out_stream, after, 0));
      const int64_t total = (int64_t)(s1 - s0) * per;
      const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
      k_pack<T><<<blocks, 256, 0, out_stream>>>(F.u[0] + (int64_t)s0 * F.ss, F.u[1] + (int64_t)s0 * F.ss, d_fbuf + s0,
                                                 d_ident, st + N + s0 * per, F.n, F.ss, total);
      ++launches;
      if (!staged) {
        CK(cudaMemcpyAsync(sh.u + s0 * per, st + N + s0 * per, sizeof(double2) * total, cudaMemcpyDeviceToHost, out_stream));
      } else {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventRecord(e, out_stream));
        packed_events.push_back(e);
        std::lock_guard<std::mutex> lk(out_mu);
        out_q.push_back({s0, s1, e});
        out_cv.notify_all();
      }
    };
    // ---- the rounds ----
    CK(cudaMemsetAsync(d_active, 0, sizeof(int) * S, stream));
    CK(cudaMemsetAsync(d_iters, 0, sizeof(int) * S, stream));
    CK(cudaMemsetAsync(d_conv, 0, sizeof(int) * S, stream));
    CK(cudaMemsetAsync(d_hist, 0, sizeof(double) * S * (size_t)H, stream));
    F.cur = 0;
    enum : char { WAITING = 0, ACTIVE = 1, DONE = 2 };
    std::vector<char> state(S, WAITING);
    int admitted = 0, n_active = 0, n_done = 0, round = 0;
    std::exception_ptr err;
    rolling = true;
    try {
      while (n_done < n_mine) {
        // admit the pieces whose copies have landed; with nothing active, wait for the next one (admitting pieces
        // ahead of their copy, with the stream waiting for them, measured no faster)
        for (; admitted < nm;) {
          const int p = mine[admitted];
          {
            std::unique_lock<std::mutex> lk(sh.mu);
            if (sh.in_ready <= p) {
              if (n_active > 0) break;
              sh.cv.wait(lk, [&] { return sh.in_ready > p; });
            }
            if (sh.in_err) std::rethrow_exception(sh.in_err);
          }
          if (n_active > 0 && cudaEventQuery(sh.in[p]) != cudaSuccess) {
            (void)cudaGetLastError();
            break;
          }
          const int s0 = sh.plo[p], s1 = sh.plo[p + 1];
          CK(cudaStreamWaitEvent(stream, sh.in[p], 0));
          {
            const int64_t total = (int64_t)(s1 - s0) * per;
            const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
            timed("unpack", (double)total * 2 * sizeof(V), [&] {
              k_unpack<T><<<blocks, 256, 0, stream>>>(st + s0 * per, F.b + (int64_t)s0 * F.ss, F.n, F.ss, total);
            });
          }
          CK(cudaMemsetAsync(F.u[F.cur] + (int64_t)s0 * F.ss, 0, sizeof(V) * (size_t)F.ss * (s1 - s0), stream));
          k_admit<<<1, 256, 0, stream>>>(d_active, d_kcur, s0, s1);
          ++launches;
          for (int s = s0; s < s1; ++s) state[s] = ACTIVE;
          n_active += s1 - s0;
          ++admitted;
        }
        // one cycle over the active shifts; its first fine pass forms their convergence norms and k_finalize_roll
        // retires the shifts that are done before the rest of the cycle runs
        roll_slot = round & 1;
        nin_k = 0;
        F.uzero = false;
        cycle_level(0, false, d_active, n_active, false);
        // flags of this round (the GPU is still in the previous round's tail or this round's first pass)
        CK(cudaEventSynchronize(ev_nactive[roll_slot]));
        const volatile int* fl = (const volatile int*)(h_map + map_flags() + sizeof(int) * (size_t)S * roll_slot);
        for (int s = 0; s < S;) {
          if (!(state[s] == ACTIVE && fl[s] == 0)) {
            ++s;
            continue;
          }
          int e = s;
          while (e < S && state[e] == ACTIVE && fl[e] == 0) state[e++] = DONE;
          emit(s, e, ev_nactive[roll_slot]);
          n_done += e - s, n_active -= e - s;
          s = e;
        }
        if (dbg)
          std::fprintf(stderr, "pdmg rolling lane %d round %d: %.2f ms admitted %d/%d active %d done %d\n", lane, round,
                       std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - sh.t0).count(),
                       admitted, nm, n_active, n_done);
        ++round;
      }
    } catch (...) {
      err = std::current_exception();
    }
    rolling = false;
    nin_k = -1;
    if (out_thread.joinable()) {
      {
        std::lock_guard<std::mutex> lk(out_mu);
        out_stop = true;
      }
      out_cv.notify_all();
      out_thread.join();
    }
    if (!err) {
      try {
        finish_report(sh.rep, sh.t0, H, &state);
        CK(cudaStreamSynchronize(out_stream));
      } catch (...) {
        err = std::current_exception();
      }
    } else {
      cudaStreamSynchronize(stream), cudaStreamSynchronize(out_stream);
    }
    for (auto e : packed_events) cudaEventDestroy(e);
    if (err) std::rethrow_exception(err);
    if (out_err) std::rethrow_exception(out_err);
  }

  bool solve_concurrent(const pdmg_c128* b, pdmg_c128* u, pdmg_solve_report* rep, double2* st, size_t N, int64_t per,
                        bool staged = false) {
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
    for (int c = 0; c < nch; ++c) CK(cudaEventCreateWithFlags(&in[c], dbg ? 0 : cudaEventDisableTiming));
    // staged input: an input thread fills the bounce ring chunk by chunk; chunk c's solve waits (on the host) until
    // in[c] is recorded, then (on its stream) for the copy itself
    std::mutex in_mu;
    std::condition_variable in_cv;
    int in_ready = 0;
    std::exception_ptr in_err;
    std::thread in_thread;
    if (staged) {
      if (!bounce_in) bounce_in = std::make_unique<Bounce>();
      bounce_in->ensure(kStageRing);
      for (auto& e : subs) {
        if (!e->bounce_out) e->bounce_out = std::make_unique<Bounce>();
        e->bounce_out->ensure(2);
      }
      in_thread = std::thread([&] {
        try {
          CK(cudaSetDevice(device));
          for (int c = 0; c < nch; ++c) {
            staged_h2d(st + lo[c] * per, b + lo[c] * per, sizeof(double2) * per * (lo[c + 1] - lo[c]), copy_stream);
            CK(cudaEventRecord(in[c], copy_stream));
            std::lock_guard<std::mutex> lk(in_mu);
            in_ready = c + 1;
            in_cv.notify_all();
          }
        } catch (...) {
          std::lock_guard<std::mutex> lk(in_mu);
          in_err = std::current_exception();
          in_ready = nch;
          in_cv.notify_all();
        }
      });
    } else {
      for (int c = 0; c < nch; ++c) {
        CK(cudaMemcpyAsync(st + lo[c] * per, b + lo[c] * per, sizeof(double2) * per * (lo[c + 1] - lo[c]),
                           cudaMemcpyHostToDevice, copy_stream));
        CK(cudaEventRecord(in[c], copy_stream));
      }
      in_ready = nch;
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
          {
            std::unique_lock<std::mutex> lk(in_mu);
            in_cv.wait(lk, [&] { return in_ready > c; });
            if (in_err) return;
          }
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
          if (staged) {
            staged_d2h(u + s0 * per, st + N + s0 * per, sizeof(double2) * per * cnt, e.stream, *e.bounce_out);
          } else {
            CK(cudaMemcpyAsync(u + s0 * per, st + N + s0 * per, sizeof(double2) * per * cnt, cudaMemcpyDeviceToHost,
                               e.stream));
          }
          if (dbg) t_out[c] = tevent(e.stream);
          CK(cudaStreamSynchronize(e.stream));
        } catch (...) {
          err[c] = std::current_exception();
        }
      });
    }
    for (auto& t : th) t.join();
    if (in_thread.joinable()) in_thread.join();
    if (in_err) std::rethrow_exception(in_err);
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
    for (auto& e : subs) {
      upd += e->last_updates, launches += e->launches, e->launches = 0;
      for (auto& kv : e->stats) {  // (each sub-engine drained its own events at the end of its solve)
        Stat& st = stats[kv.first];
        st.launches += kv.second.launches, st.ms += kv.second.ms, st.bytes += kv.second.bytes;
        st.ubytes += kv.second.ubytes, st.updates += kv.second.updates;
      }
      e->stats.clear();
    }
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


}  // namespace pdmg_b200
