// pdmg_paradiag.h -- ParaDIAG drivers on the GPU (pdmg_paradiag.cu), restating proj/src/paradiag.cpp:185-248.
//
// The all-at-once system (B (x) I + I (x) A) U = F is solved in three steps: g = (V^{-1} (x) I) f, the batched
// shifted solves (A + lambda_k I) w_k = g_k, u = (V (x) I) w, then relres = ||F - K U|| / ||F||.  The time slices
// (and the shift slots, one per slice) may be sharded over several devices of one process -- the reference's
// `threads` argument (paradiag.cpp:217-236) becomes a device list -- in which case both time transforms gather
// their time columns from every shard and scatter the results to the owners through NVLink peer pointers inside
// the transform kernel itself (pdmg_time_kernels.cuh RowTab): no separate all-to-all.
#pragma once
#include "pdmg_host.h"

namespace pdmg_b200 {

struct RowTab;  // pdmg_time_kernels.cuh

// alpha-scaled DFT tables over the time index (device arrays of one device)
struct DftTables {
  double2* tw = nullptr;  // e^{dir 2 pi i q/nt}
  double2* pre = nullptr;
  double2* post = nullptr;
  int nt = 0, log2nt = -1;
  ~DftTables() {
    cudaFree(tw);
    cudaFree(pre);
    cudaFree(post);
  }
};
// step 1: pre = alpha^(t/nt), dir +1, post = 1/nt;  step 3: pre = 1, dir -1, post = alpha^(-t/nt)
std::unique_ptr<DftTables> make_dft_tables(int nt, double alpha, int step, cudaStream_t st);
// throws ConfigError when nt exceeds what one CTA's shared memory can transform
void check_dft_size(int nt);

struct PdShard {
  int device = 0, t0 = 0, cnt = 0;   // time slices / shift slots [t0, t0 + cnt)
  int64_t pt0 = 0, pt1 = 0;          // spatial points this shard transforms
  std::unique_ptr<EngineBase> eng;   // the shard's shifted solves
  double2 *f = nullptr, *g = nullptr, *w = nullptr, *u = nullptr, *y = nullptr;  // cnt slices each
  double* partial = nullptr;         // residual partial sums [res_blocks][2]
  double* h_partial = nullptr;       // pinned host copy
  std::unique_ptr<DftTables> t1, t3; // circulant scheme
  double2 *V = nullptr, *Vi = nullptr, *B = nullptr;  // general scheme (nt x nt, this device)
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // input ready, g ready, w ready, u ready
  bool remote = false;  // rank mode: another process's shard (buffers opened over CUDA IPC, no engine)
  ~PdShard();
};

struct Paradiag {
  int n = 0, nt = 0;
  bool general = false;
  double alpha = 0, dt = 0;  // circulant scheme
  int64_t npts = 0;
  int res_blocks = 148 * 8;
  std::vector<std::unique_ptr<PdShard>> sh;

  // alpha-circulant C_alpha = (1/dt)(I - Sigma_alpha), diagonalized by the alpha-scaled DFT (BASELINE formula; with
  // alpha = -1/beta the reference's BackwardHeatQBV, paradiag.cpp:84-108)
  void setup_circulant(int n_, int nt_, double alpha_, double dt_, const pdmg_mg_config& cfg,
                       const std::vector<int>& devices);
  // general diagonalizable B = V diag(lambdas) V^{-1} (diagonalize_time_matrix, paradiag.cpp:71-82)
  void setup_general(int n_, int nt_, const pdmg_c128* lambdas, const pdmg_c128* V, const pdmg_c128* Vinv,
                     const double* B, const pdmg_mg_config& cfg, const std::vector<int>& devices);
  // f[s], u[s]: shard s's time slices [t0, t0 + cnt) x npts in its device's memory
  void run_shards(const double2* const* f, double2* const* u, pdmg_solve_report* rep, double* relres);
  void run_device(const double2* f, double2* u, pdmg_solve_report* rep, double* relres);  // one shard
  void run_host(const pdmg_c128* f, pdmg_c128* u, pdmg_solve_report* rep, double* relres);
  EngineBase* solver() { return sh.empty() ? nullptr : sh[local >= 0 ? local : 0]->eng.get(); }

  // Rank mode (one process per GPU): this process owns shard `rank` of `nranks`; the other shards' f, g, w, u are
  // opened from their CUDA IPC handles, so the transform kernels gather / scatter across processes through NVLink
  // peer memory exactly as across the devices of one process.  The caller runs the four phases with a process
  // barrier between them (each phase returns once its GPU work, peer writes included, is complete).
  int local = -1;
  bool peers_open = false;
  void setup_rank(int n_, int nt_, double alpha_, double dt_, const pdmg_mg_config& cfg, int rank, int nranks,
                  int device);
  void ipc_handles(void* out) const;  // 4 cudaIpcMemHandle_t: f, g, w, u
  void open_peers(const void* all);   // [nranks][4] handles
  void rank_phase(int k, pdmg_solve_report* rep, double* sums);

 private:
  void phase(int p, int k, const RowTab (&T)[4], pdmg_solve_report* rep);
  void setup_shards(int n_, int nt_, const std::vector<pdmg_c128>& lam, const pdmg_mg_config& cfg,
                    const std::vector<int>& devices);
  void run_impl(const double2* const* f, double2* const* u, pdmg_solve_report* rep, double* relres,
                const pdmg_c128* hf, pdmg_c128* hu);
};

// all-at-once residual sums {||r||^2, ||f||^2} of local slices [t0, t0 + ntl) (paradiag.cpp:141-183)
void aao_residual_sums(int device, int n, int ntl, int t0, double alpha, double dt, const double2* u,
                       const double2* u_prev, const double2* f, double* sums, cudaStream_t st);
// Y = (M (x) I) X for device arrays [nt][npts] of one device (kron_time_apply, paradiag.cpp:129-133)
void time_transform(int device, cudaStream_t st, int nt, int64_t npts, const double2* dM, const double2* dX,
                    double2* dY);
// alpha-scaled time DFT of device arrays [nt][npts] of one device (tables cached per device)
void time_dft(int device, int nt, int64_t npts, double alpha, int step, const double2* in, double2* out,
              cudaStream_t st);

}  // namespace pdmg_b200
