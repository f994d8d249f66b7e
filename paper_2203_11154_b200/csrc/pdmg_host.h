// pdmg_host.h -- host side of libpdmg_b200.so (C++): error taxonomy, setup math restating the reference
// formulas, and the precision-independent engine interface the C ABI (pdmg_capi.cu), the multi-device
// engine (pdmg_multi.cu) and the ParaDIAG driver (pdmg_paradiag.cu) program against.  The batched
// multigrid engine itself is pdmg_engine.cuh, instantiated per storage precision in pdmg_engine_c128.cu /
// pdmg_engine_c64.cu.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pdmg_b200.h"

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

extern thread_local std::string g_last_error;

#define CK(x)                                                                                        \
  do {                                                                                               \
    cudaError_t e_ = (x);                                                                            \
    if (e_ != cudaSuccess)                                                                           \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" +          \
                      std::to_string(__LINE__) + ")");                                               \
  } while (0)

template <class F>
inline int guarded(F&& f) {
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
// Host-side setup math (fp64), restating the reference formulas (definitions in pdmg_host.cu).
// ---------------------------------------------------------------------------------------------
constexpr double kSingularTol = 1e-12;  // smoother.cpp:6
cplx checked_inverse(cplx z, const char* what);  // smoother.cpp:8-15
struct Vanka {
  cplx a, b, c;
};
Vanka vanka_coeffs(cplx eta);               // smoother.cpp:18-29
cplx jacobi_weight(cplx eta, double h);     // smoother.cpp:42-47
// Dense A + lambda I on the coarsest grid (dense.cpp:18-39), partial-pivot LU with the reference's
// singularity rule min|U_ii| > 1e-14 ||A||_F (dense.cpp:82-88), then A^{-1} for the batched kernel.
struct CoarseFactor {
  bool singular = false;
  std::vector<cplx> inv;  // N x N row-major
};
CoarseFactor factor_coarse(int n, cplx lambda);
void validate(const pdmg_mg_config& c);                        // multigrid.hpp:25-31
std::vector<int> level_list(int n, const pdmg_mg_config& c);   // multigrid.cpp:27-44
cplx real_pow_c(double alpha, double p);  // principal alpha^p for real alpha != 0 (paradiag.cpp:209-213)

// ---------------------------------------------------------------------------------------------
// Engine interface: one batch of shifts (one device, or a list of devices: pdmg_multi.cu).
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

  // instrumentation: with profiling on, every launch is bracketed by CUDA events on `stream` and attributed
  // to a kernel class (drained into `stats` at the end of a call)
  struct Pending {
    std::string cls;
    cudaEvent_t e0, e1;
    double bytes, ubytes, updates;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
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


  virtual ~EngineBase() {
    for (auto& p : pending) {
      cudaEventDestroy(p.e0);
      cudaEventDestroy(p.e1);
    }
    for (auto e : event_pool) cudaEventDestroy(e);
  }
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
  // device shards (a single-device engine is one shard holding every shift)
  virtual void solve_device_shards(const void* const* d_b, void* const* d_u, pdmg_solve_report* rep) {
    solve_device(static_cast<const double2*>(d_b[0]), static_cast<double2*>(d_u[0]), rep);
  }
  virtual int num_parts() const { return 1; }
  virtual void part_range(int p, int* s0, int* count, int* dev) const {
    if (p != 0) throw ConfigError("pdmg_part_range: shard index out of range");
    if (s0) *s0 = 0;
    if (count) *count = S;
    if (dev) *dev = device;
  }
};

// factories (pdmg_engine_c128.cu, pdmg_engine_c64.cu, pdmg_multi.cu)
std::unique_ptr<EngineBase> make_engine_c128();
std::unique_ptr<EngineBase> make_engine_c64();
std::unique_ptr<EngineBase> make_engine(int precision);  // throws ConfigError on an unknown precision
// pdmg_create's engine: single-device, or sharded over desc.devices (one engine per device, contiguous shift
// ranges, paradiag.cpp:217-236)
std::unique_ptr<EngineBase> create_engine(const pdmg_batch_desc& d);

}  // namespace pdmg_b200
