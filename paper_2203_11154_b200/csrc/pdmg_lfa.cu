// pdmg_lfa.cu -- local Fourier analysis of the shifted Laplacian with the Vanka / Jacobi smoother on the GPU
// (restating proj/src/lfa.cpp:68-248, proj/include/pdmg/lfa.hpp).
//
// The analysis samples the low-frequency quadrant [-pi/2, pi/2)^2 with samples_per_dim^2 base frequencies; every
// base carries its four harmonics theta + pi (s1, s2).  Per sampled frequency the symbols are closed forms
// (cheap), and the two-grid factor needs, per base and per damping omega, the spectral radius of a 4 x 4 complex
// error matrix E = diag((1 - omega M L)^nu) (I - R R^T L / L_c) -- the only expensive part, and embarrassingly
// parallel: one thread per (omega, base).  The damping optimization evaluates its whole coarse omega scan
// (0.1 : 0.01 : 1.9) in one launch and the golden-section refinement one omega per launch.  Maxima over the
// sampled frequencies are formed on the host in the reference's deterministic order (first maximizer wins,
// ties within 1e-12, lfa.cpp:16-60), so the reported argmax matches the reference's.
#include <functional>
#include <mutex>

#include "pdmg_host.h"
#include "pdmg_kernels.cuh"

namespace pdmg_b200 {

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kArgmaxTieTol = 1e-12;  // lfa.cpp:15

struct LfaSetup {  // per (shift, h, smoother): what every symbol evaluation needs
  double2 lam;     // lambda
  double2 va, vb, vc;  // Vanka coefficients a, b, c (smoother.cpp:18-29)
  double2 jw;          // Jacobi weight h^2 / (4 + eta)
  double h;
  int jacobi;
};

__host__ __device__ inline double2 c_mul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ inline double2 c_div(double2 a, double2 b) {  // (Smith's algorithm)
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  }
  const double r = b.x / b.y, d = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}
__host__ __device__ inline double c_abs(double2 a) { return hypot(a.x, a.y); }

// symbol_shifted_laplacian (lfa.cpp:68-71): (4 - 2 cos t1 - 2 cos t2 + eta(h)) / h^2, eta(h) = lambda h^2 -- of the
// mesh width it is evaluated on (the coarse symbol uses 2h and lambda (2h)^2)
__host__ __device__ inline double2 sym_L(double t1, double t2, double2 lambda, double h) {
  const double s = 4.0 - 2.0 * cos(t1) - 2.0 * cos(t2), h2 = h * h;
  return make_double2((s + lambda.x * h2) / h2, (lambda.y * h2) / h2);
}
// symbol_vanka (lfa.cpp:73-77): h^2 (a + b (cos t1 + cos t2) + c cos t1 cos t2)
__host__ __device__ inline double2 sym_vanka(double t1, double t2, const LfaSetup& S) {
  const double c1 = cos(t1), c2 = cos(t2), s = c1 + c2, p = c1 * c2;
  const double h2 = S.h * S.h;
  return make_double2(h2 * (S.va.x + S.vb.x * s + S.vc.x * p), h2 * (S.va.y + S.vb.y * s + S.vc.y * p));
}
__host__ __device__ inline double2 sym_M(double t1, double t2, const LfaSetup& S) {  // lfa.cpp:79-82
  return S.jacobi ? S.jw : sym_vanka(t1, t2, S);
}
__host__ __device__ inline double sym_R(double t1, double t2) {  // lfa.cpp:89-91
  return 0.25 * (1.0 + cos(t1)) * (1.0 + cos(t2));
}

// Eigenvalue moduli of a complex 4 x 4 matrix (Hessenberg reduction by Givens similarities, then single-shift
// QR with Wilkinson shifts and deflation): the spectral radius of the two-grid error symbol (the reference uses
// Eigen::ComplexEigenSolver, lfa.cpp:39-45).
__host__ __device__ inline void givens(double2 a, double2 b, double& c, double2& s) {
  const double aa = c_abs(a), r = hypot(aa, c_abs(b));
  if (r == 0.0) {
    c = 1.0, s = make_double2(0.0, 0.0);
  } else if (aa == 0.0) {
    c = 0.0, s = make_double2(b.x / r, -b.y / r);  // conj(b)/r: maps (0, b) to (|b|, 0)
  } else {
    const double2 ph = make_double2(a.x / aa, a.y / aa);
    c = aa / r;
    s = c_mul(ph, make_double2(b.x / r, -b.y / r));
  }
}
// rows k, k+1 <- G [row k; row k+1], G = [c s; -conj(s) c], columns [j0, j1)
__host__ __device__ inline void rot_rows(double2 (&H)[4][4], int k, double c, double2 s, int j0, int j1) {
  for (int j = j0; j < j1; ++j) {
    const double2 x = H[k][j], y = H[k + 1][j];
    const double2 sy = c_mul(s, y), sx = c_mul(make_double2(s.x, -s.y), x);
    H[k][j] = make_double2(c * x.x + sy.x, c * x.y + sy.y);
    H[k + 1][j] = make_double2(c * y.x - sx.x, c * y.y - sx.y);
  }
}
// columns k, k+1 <- [col k, col k+1] G^H, rows [i0, i1)
__host__ __device__ inline void rot_cols(double2 (&H)[4][4], int k, double c, double2 s, int i0, int i1) {
  for (int i = i0; i < i1; ++i) {
    const double2 x = H[i][k], y = H[i][k + 1];
    const double2 ys = c_mul(y, make_double2(s.x, -s.y)), xs = c_mul(x, s);
    H[i][k] = make_double2(c * x.x + ys.x, c * x.y + ys.y);
    H[i][k + 1] = make_double2(c * y.x - xs.x, c * y.y - xs.y);
  }
}
__host__ __device__ inline double spectral_radius4(double2 (&H)[4][4]) {
  constexpr int n = 4;
  // Hessenberg: zero H[3][0], H[2][0] (rows 2,3 then 1,2), then H[3][1]
  const int zr[3][2] = {{3, 0}, {2, 0}, {3, 1}};
  for (auto& z : zr) {
    const int i = z[0], k = z[1];
    double c;
    double2 s;
    givens(H[i - 1][k], H[i][k], c, s);
    rot_rows(H, i - 1, c, s, 0, n);
    rot_cols(H, i - 1, c, s, 0, n);
    H[i][k] = make_double2(0.0, 0.0);
  }
  double norm = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) norm = fmax(norm, c_abs(H[i][j]));
  double rho = 0.0;
  int hi = n - 1, iter = 0;
  while (hi >= 0) {
    if (hi == 0) {
      rho = fmax(rho, c_abs(H[0][0]));
      break;
    }
    int l = hi;
    for (; l > 0; --l) {
      const double sub = c_abs(H[l][l - 1]);
      if (sub <= 2.220446049250313e-16 * (c_abs(H[l - 1][l - 1]) + c_abs(H[l][l])) || sub <= 1e-300 * norm + 1e-300) {
        H[l][l - 1] = make_double2(0.0, 0.0);
        break;
      }
    }
    if (l == hi) {  // H[hi][hi] deflated
      rho = fmax(rho, c_abs(H[hi][hi]));
      --hi;
      iter = 0;
      continue;
    }
    if (++iter > 60) {  // not converged: fall back to the Gershgorin bound of the active block
      for (int i = l; i <= hi; ++i) {
        double r = 0.0;
        for (int j = l; j <= hi; ++j) r += c_abs(H[i][j]);
        rho = fmax(rho, r);
      }
      break;
    }
    // Wilkinson shift: the eigenvalue of the trailing 2 x 2 block closer to H[hi][hi]
    const double2 a = H[hi - 1][hi - 1], b = H[hi - 1][hi], cc = H[hi][hi - 1], d = H[hi][hi];
    const double2 half = make_double2(0.5 * (a.x - d.x), 0.5 * (a.y - d.y));
    double2 disc = c_mul(half, half);
    const double2 bc = c_mul(b, cc);
    disc.x += bc.x, disc.y += bc.y;
    const double r = c_abs(disc);
    double2 sq = make_double2(sqrt(0.5 * (r + disc.x)), 0.0);  // principal complex sqrt
    sq.y = disc.y >= 0 ? sqrt(fmax(0.0, 0.5 * (r - disc.x))) : -sqrt(fmax(0.0, 0.5 * (r - disc.x)));
    const double2 m = make_double2(0.5 * (a.x + d.x), 0.5 * (a.y + d.y));
    const double2 e1 = make_double2(m.x + sq.x, m.y + sq.y), e2 = make_double2(m.x - sq.x, m.y - sq.y);
    double2 mu = c_abs(make_double2(e1.x - d.x, e1.y - d.y)) < c_abs(make_double2(e2.x - d.x, e2.y - d.y)) ? e1 : e2;
    if (iter % 11 == 10) mu = make_double2(d.x + c_abs(cc), d.y);  // exceptional shift
    // explicit shifted QR step on the active block [l, hi]
    for (int i = l; i <= hi; ++i) H[i][i].x -= mu.x, H[i][i].y -= mu.y;
    double cs[3];
    double2 sn[3];
    for (int k = l; k < hi; ++k) {
      givens(H[k][k], H[k + 1][k], cs[k - l], sn[k - l]);
      rot_rows(H, k, cs[k - l], sn[k - l], k, hi + 1);
      H[k + 1][k] = make_double2(0.0, 0.0);
    }
    for (int k = l; k < hi; ++k) rot_cols(H, k, cs[k - l], sn[k - l], l, (k + 2 < hi ? k + 2 : hi) + 1);
    for (int i = l; i <= hi; ++i) H[i][i].x += mu.x, H[i][i].y += mu.y;
  }
  return rho;
}

// ---- kernels ---------------------------------------------------------------------------------------------------
// The sampled high-frequency region in the reference's order (lfa.cpp:31-37): theta1 outer, theta2 inner,
// harmonic shifts (1,0), (0,1), (1,1) innermost; q = (i1 * n + i2) * 3 + s.
__device__ inline void high_freq(int q, int n, double& t1, double& t2) {
  const int s = q % 3, b = q / 3, i2 = b % n, i1 = b / n;
  const double step = kPi / n;
  t1 = -0.5 * kPi + i1 * step + (s != 1 ? kPi : 0.0);
  t2 = -0.5 * kPi + i2 * step + (s != 0 ? kPi : 0.0);
}

// |1 - omega M L| at every sampled high frequency (smoothing_factor, lfa.cpp:93-100)
__global__ void k_lfa_smoothing(LfaSetup S, int n, double omega, double* __restrict__ val) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= 3 * n * n) return;
  double t1, t2;
  high_freq(q, n, t1, t2);
  const double2 ml = c_mul(sym_M(t1, t2, S), sym_L(t1, t2, S.lam, S.h));
  val[q] = c_abs(make_double2(1.0 - omega * ml.x, -omega * ml.y));
}

// smoothing_factor_bound (lfa.cpp:102-115): per point |1 - omega M0 A0| (unshifted) and |omega lambda M|
__global__ void k_lfa_bound(LfaSetup S, LfaSetup S0, double2 lambda, int n, double omega, double* __restrict__ val) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= 3 * n * n) return;
  double t1, t2;
  high_freq(q, n, t1, t2);
  const double2 b = c_mul(sym_vanka(t1, t2, S0), sym_L(t1, t2, make_double2(0.0, 0.0), S.h));
  val[2 * q] = c_abs(make_double2(1.0 - omega * b.x, -omega * b.y));
  const double2 lm = c_mul(lambda, sym_vanka(t1, t2, S));
  val[2 * q + 1] = c_abs(make_double2(omega * lm.x, omega * lm.y));
}

// TwoGridModel construction (lfa.cpp:117-153): per base, M L at the four harmonics, the coarse-grid correction
// symbol I - R R^T L / L_c (rank-one update of I), and the skip flag |L_c| <= coarse_skip_tol.
struct LfaBase {
  double2 ml[4];
  double2 u[4];  // cgc(r, c) = delta_rc - u[r] * v[c]
  double2 v[4];
  int skip;
};
__global__ void k_lfa_model(LfaSetup S, int n, double skip_tol, LfaBase* __restrict__ bases,
                            double2* __restrict__ high_ml) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n * n) return;
  const int i1 = b / n, i2 = b % n;
  const double step = kPi / n;
  const double t1 = -0.5 * kPi + i1 * step, t2 = -0.5 * kPi + i2 * step;
  const double th1[4] = {t1, t1 + kPi, t1, t1 + kPi}, th2[4] = {t2, t2, t2 + kPi, t2 + kPi};
  LfaBase e;
  const double2 Lc = sym_L(2.0 * t1, 2.0 * t2, S.lam, 2.0 * S.h);  // re-discretized coarse symbol (mesh 2h)
  for (int k = 0; k < 4; ++k) {
    const double2 L = sym_L(th1[k], th2[k], S.lam, S.h);
    e.ml[k] = c_mul(sym_M(th1[k], th2[k], S), L);
    const double R = sym_R(th1[k], th2[k]);
    e.u[k] = make_double2(R, 0.0);
    e.v[k] = c_div(make_double2(R * L.x, R * L.y), Lc);
    if (k > 0) high_ml[3 * b + k - 1] = e.ml[k];
  }
  e.skip = c_abs(Lc) <= skip_tol;
  bases[b] = e;
}

// rho(omega_w, nu) = max over the non-skipped bases of the spectral radius of
// E = diag((1 - omega ml)^nu) (I - u v^T) (lfa.cpp:155-167); one thread per (base, omega).
__global__ void k_lfa_rho(const LfaBase* __restrict__ bases, int nb, const double* __restrict__ omegas, int nu,
                          unsigned long long* __restrict__ rho_bits) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int w = blockIdx.y;
  double r = 0.0;
  if (b < nb && !bases[b].skip) {
    const LfaBase& e = bases[b];
    const double om = omegas[w];
    double2 E[4][4];
    for (int i = 0; i < 4; ++i) {
      const double2 z = make_double2(1.0 - om * e.ml[i].x, -om * e.ml[i].y);
      double2 s = make_double2(1.0, 0.0);
      for (int k = 0; k < nu; ++k) s = c_mul(s, z);  // ipow (lfa.cpp:47-51)
      for (int j = 0; j < 4; ++j) {
        double2 g = c_mul(e.u[i], e.v[j]);
        g = make_double2((i == j ? 1.0 : 0.0) - g.x, -g.y);
        E[i][j] = c_mul(s, g);
      }
    }
    r = spectral_radius4(E);
  }
  // max over the bases of this omega: warp reduction, then one atomic per warp (r >= 0, so the IEEE bit pattern
  // orders like the value)
  for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
  if ((threadIdx.x & 31) == 0 && r > 0.0) atomicMax(rho_bits + w, (unsigned long long)__double_as_longlong(r));
}

// |1 - omega ml| over the cached high-frequency symbols (TwoGridModel::smoothing, lfa.cpp:169-174)
__global__ void k_lfa_model_smoothing(const double2* __restrict__ high_ml, int count, double omega,
                                      double* __restrict__ val) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < count) val[q] = c_abs(make_double2(1.0 - omega * high_ml[q].x, -omega * high_ml[q].y));
}

// max |1 - omega_w ml| over every high frequency, for a batch of omegas (smoothing objective)
__global__ void k_lfa_mu_batch(const double2* __restrict__ high_ml, int count, const double* __restrict__ omegas,
                               unsigned long long* __restrict__ mu_bits) {
  const int w = blockIdx.y;
  double r = 0.0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < count; q += gridDim.x * blockDim.x)
    r = fmax(r, c_abs(make_double2(1.0 - omegas[w] * high_ml[q].x, -omegas[w] * high_ml[q].y)));
  for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
  if ((threadIdx.x & 31) == 0 && r > 0.0) atomicMax(mu_bits + w, (unsigned long long)__double_as_longlong(r));
}

__global__ void k_lfa_high_ml(LfaSetup S, int n, double2* __restrict__ high_ml) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= 3 * n * n) return;
  double t1, t2;
  high_freq(q, n, t1, t2);
  high_ml[q] = c_mul(sym_M(t1, t2, S), sym_L(t1, t2, S.lam, S.h));
}

void validate_lfa(const pdmg_lfa_config& c) {  // lfa.hpp:25-30
  if (c.samples_per_dim < 16 || c.samples_per_dim % 2 != 0)
    throw ConfigError("LFAConfig: samples_per_dim must be even and >= 16");
  if (!(c.coarse_skip_tol > 0.0)) throw ConfigError("LFAConfig: coarse_skip_tol must be positive");
}

LfaSetup make_setup(pdmg_c128 lambda, double h, int smoother) {
  if (smoother != PDMG_SMOOTHER_VANKA && smoother != PDMG_SMOOTHER_JACOBI)
    throw ConfigError("SmootherConfig: unknown smoother kind");
  const cplx eta = cplx(lambda.re, lambda.im) * (h * h);  // Shift::eta (grid.hpp:44-52)
  LfaSetup S{};
  S.lam = make_double2(lambda.re, lambda.im);
  S.h = h;
  S.jacobi = smoother == PDMG_SMOOTHER_JACOBI;
  if (S.jacobi) {
    const cplx w = jacobi_weight(eta, h);
    S.jw = make_double2(w.real(), w.imag());
  } else {
    const Vanka v = vanka_coeffs(eta);
    S.va = make_double2(v.a.real(), v.a.imag());
    S.vb = make_double2(v.b.real(), v.b.imag());
    S.vc = make_double2(v.c.real(), v.c.imag());
  }
  return S;
}

// MaxTracker (lfa.cpp:53-62) over values in the sampled order
void first_max(const std::vector<double>& v, int n, double* mu, double* arg) {
  double best = -1.0;
  size_t at = 0;
  for (size_t q = 0; q < v.size(); ++q)
    if (v[q] > best + kArgmaxTieTol) best = v[q], at = q;
  *mu = best;
  if (arg) {
    const int s = (int)(at % 3), b = (int)(at / 3), i2 = b % n, i1 = b / n;
    const double step = kPi / n;
    arg[0] = -0.5 * kPi + i1 * step + (s != 1 ? kPi : 0.0);
    arg[1] = -0.5 * kPi + i2 * step + (s != 0 ? kPi : 0.0);
  }
}

struct DevBuf {  // a device allocation freed on scope exit
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { CK(cudaMalloc(&p, bytes)); }
  ~DevBuf() { cudaFree(p); }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// minimize_scalar (lfa.cpp:183-219): coarse scan of [0.1, 1.9] step 0.01 (one batched evaluation), then a
// golden-section refinement of the winning bracket to width 1e-4 (sequential evaluations)
template <class Batch>
void minimize_scalar(Batch&& f, double* omega, double* value) {
  constexpr double lo = 0.1, hi = 1.9, step = 0.01;
  const int nsteps = (int)std::lround((hi - lo) / step);
  std::vector<double> ws(nsteps + 1);
  for (int k = 0; k <= nsteps; ++k) ws[k] = lo + k * step;
  ws[0] = lo;
  const std::vector<double> vs = f(ws);
  double best_w = lo, best_v = vs[0];
  for (int k = 1; k <= nsteps; ++k)
    if (vs[k] < best_v) best_v = vs[k], best_w = ws[k];
  auto f1 = [&](double w) { return f(std::vector<double>{w})[0]; };
  double a = std::max(lo, best_w - step), b = std::min(hi, best_w + step);
  const double invphi = (std::sqrt(5.0) - 1.0) / 2.0;
  double x1 = b - invphi * (b - a), x2 = a + invphi * (b - a);
  double v1 = f1(x1), v2 = f1(x2);
  while (b - a > 1e-4) {
    if (v1 <= v2) {
      b = x2, x2 = x1, v2 = v1;
      x1 = b - invphi * (b - a);
      v1 = f1(x1);
    } else {
      a = x1, x1 = x2, v1 = v2;
      x2 = a + invphi * (b - a);
      v2 = f1(x2);
    }
  }
  const double w = 0.5 * (a + b);
  *omega = w;
  *value = f1(w);
}

std::vector<double> max_batch(const std::vector<double>& ws, int count, int grid_x, int threads,
                              const std::function<void(const double*, unsigned long long*, dim3)>& launch) {
  DevBuf dw(sizeof(double) * ws.size()), dm(sizeof(unsigned long long) * ws.size());
  CK(cudaMemcpy(dw.p, ws.data(), sizeof(double) * ws.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dm.p, 0, sizeof(unsigned long long) * ws.size()));
  launch(dw.as<double>(), dm.as<unsigned long long>(), dim3(grid_x, (unsigned)ws.size()));
  CK(cudaGetLastError());
  std::vector<unsigned long long> bits(ws.size());
  CK(cudaMemcpy(bits.data(), dm.p, sizeof(unsigned long long) * bits.size(), cudaMemcpyDeviceToHost));
  std::vector<double> out(ws.size());
  for (size_t k = 0; k < ws.size(); ++k) std::memcpy(&out[k], &bits[k], sizeof(double));
  (void)count, (void)threads;
  return out;
}

}  // namespace

// TwoGridModel (lfa.hpp:70-96) with its symbol caches in device memory
struct LfaModel {
  int device = 0, n = 0, skipped = 0, smoother = 0;
  LfaSetup S{};
  LfaBase* bases = nullptr;
  double2* high_ml = nullptr;
  ~LfaModel() {
    cudaSetDevice(device);
    cudaFree(bases);
    cudaFree(high_ml);
  }
  std::vector<double> rho(const std::vector<double>& ws, int nu) const {
    if (nu < 1) throw ConfigError("TwoGridModel::rho: nu must be >= 1");
    CK(cudaSetDevice(device));
    const int nb = n * n, threads = 128;
    return max_batch(ws, nb, (nb + threads - 1) / threads, threads,
                     [&](const double* w, unsigned long long* m, dim3 g) {
                       k_lfa_rho<<<g, threads>>>(bases, nb, w, nu, m);
                     });
  }
  std::vector<double> mu(const std::vector<double>& ws) const {
    CK(cudaSetDevice(device));
    const int cnt = 3 * n * n, threads = 256;
    return max_batch(ws, cnt, std::min(148, (cnt + threads - 1) / threads), threads,
                     [&](const double* w, unsigned long long* m, dim3 g) {
                       k_lfa_mu_batch<<<g, threads>>>(high_ml, cnt, w, m);
                     });
  }
  void smoothing(double omega, double* mu_out, double* arg) const {
    CK(cudaSetDevice(device));
    const int cnt = 3 * n * n;
    DevBuf dv(sizeof(double) * cnt);
    k_lfa_model_smoothing<<<(cnt + 255) / 256, 256>>>(high_ml, cnt, omega, dv.as<double>());
    CK(cudaGetLastError());
    std::vector<double> v(cnt);
    CK(cudaMemcpy(v.data(), dv.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
    first_max(v, n, mu_out, arg);
  }
};

}  // namespace pdmg_b200

using namespace pdmg_b200;

struct pdmg_lfa_model {
  LfaModel m;
};

extern "C" {

void pdmg_lfa_config_default(pdmg_lfa_config* c) {
  c->samples_per_dim = 64;
  c->coarse_skip_tol = 1e-8;
}

int pdmg_lfa_symbol(int32_t which, double t1, double t2, pdmg_c128 lambda, double h, int32_t smoother, double omega,
                    pdmg_c128* out) {
  return guarded([&] {
    if (!out) throw ConfigError("pdmg_lfa_symbol: NULL out");
    double2 v = make_double2(0.0, 0.0);
    if (which == PDMG_LFA_TRANSFER) {
      v = make_double2(sym_R(t1, t2), 0.0);
    } else {
      const LfaSetup S = make_setup(lambda, h, which == PDMG_LFA_VANKA ? PDMG_SMOOTHER_VANKA : smoother);
      const double2 L = sym_L(t1, t2, S.lam, h);
      if (which == PDMG_LFA_OPERATOR) v = L;
      else if (which == PDMG_LFA_VANKA) v = sym_vanka(t1, t2, S);
      else if (which == PDMG_LFA_PRECONDITIONER) v = sym_M(t1, t2, S);
      else if (which == PDMG_LFA_SMOOTHER_ERROR) {
        const double2 ml = c_mul(sym_M(t1, t2, S), L);
        v = make_double2(1.0 - omega * ml.x, -omega * ml.y);
      } else {
        throw ConfigError("pdmg_lfa_symbol: unknown symbol " + std::to_string(which));
      }
    }
    *out = pdmg_c128{v.x, v.y};
  });
}

int pdmg_lfa_smoothing_factor(pdmg_c128 lambda, double h, int32_t smoother, double omega, const pdmg_lfa_config* lfa,
                              int32_t device, double* mu, double* argmax) {
  return guarded([&] {
    if (!lfa || !mu) throw ConfigError("pdmg_lfa_smoothing_factor: NULL argument");
    validate_lfa(*lfa);
    const LfaSetup S = make_setup(lambda, h, smoother);
    CK(cudaSetDevice(device));
    const int n = lfa->samples_per_dim, cnt = 3 * n * n;
    DevBuf dv(sizeof(double) * cnt);
    k_lfa_smoothing<<<(cnt + 255) / 256, 256>>>(S, n, omega, dv.as<double>());
    CK(cudaGetLastError());
    std::vector<double> v(cnt);
    CK(cudaMemcpy(v.data(), dv.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
    first_max(v, n, mu, argmax);
  });
}

int pdmg_lfa_smoothing_bound(pdmg_c128 lambda, double h, double omega, const pdmg_lfa_config* lfa, int32_t device,
                             double* phi) {
  return guarded([&] {
    if (!lfa || !phi) throw ConfigError("pdmg_lfa_smoothing_bound: NULL argument");
    validate_lfa(*lfa);
    const LfaSetup S = make_setup(lambda, h, PDMG_SMOOTHER_VANKA);
    const LfaSetup S0 = make_setup(pdmg_c128{0.0, 0.0}, h, PDMG_SMOOTHER_VANKA);
    CK(cudaSetDevice(device));
    const int n = lfa->samples_per_dim, cnt = 3 * n * n;
    DevBuf dv(sizeof(double) * 2 * cnt);
    k_lfa_bound<<<(cnt + 255) / 256, 256>>>(S, S0, make_double2(lambda.re, lambda.im), n, omega, dv.as<double>());
    CK(cudaGetLastError());
    std::vector<double> v(2 * cnt);
    CK(cudaMemcpy(v.data(), dv.p, sizeof(double) * v.size(), cudaMemcpyDeviceToHost));
    phi[0] = phi[1] = 0.0;
    for (int q = 0; q < cnt; ++q) phi[0] = std::max(phi[0], v[2 * q]), phi[1] = std::max(phi[1], v[2 * q + 1]);
  });
}

int pdmg_lfa_model_create(pdmg_c128 lambda, double h, int32_t smoother, const pdmg_lfa_config* lfa, int32_t device,
                          pdmg_lfa_model** out) {
  return guarded([&] {
    if (!lfa || !out) throw ConfigError("pdmg_lfa_model_create: NULL argument");
    *out = nullptr;
    validate_lfa(*lfa);
    auto P = std::make_unique<pdmg_lfa_model>();
    LfaModel& M = P->m;
    M.S = make_setup(lambda, h, smoother);
    M.n = lfa->samples_per_dim, M.device = device, M.smoother = smoother;
    CK(cudaSetDevice(device));
    const int nb = M.n * M.n;
    CK(cudaMalloc(&M.bases, sizeof(LfaBase) * nb));
    CK(cudaMalloc(&M.high_ml, sizeof(double2) * 3 * nb));
    k_lfa_model<<<(nb + 127) / 128, 128>>>(M.S, M.n, lfa->coarse_skip_tol, M.bases, M.high_ml);
    CK(cudaGetLastError());
    std::vector<LfaBase> hb(nb);
    CK(cudaMemcpy(hb.data(), M.bases, sizeof(LfaBase) * nb, cudaMemcpyDeviceToHost));
    for (const LfaBase& e : hb) M.skipped += e.skip;
    if (M.skipped == nb) throw ConfigError("TwoGridModel: every sampled base frequency was skipped as singular");
    *out = P.release();
  });
}
void pdmg_lfa_model_destroy(pdmg_lfa_model* m) { delete m; }
int pdmg_lfa_model_skipped(const pdmg_lfa_model* m) { return m ? m->m.skipped : -1; }
int pdmg_lfa_model_rho(pdmg_lfa_model* m, int32_t count, const double* omegas, int32_t nu, double* rho) {
  return guarded([&] {
    if (!m || !omegas || !rho || count < 1) throw ConfigError("pdmg_lfa_model_rho: bad argument");
    const auto r = m->m.rho(std::vector<double>(omegas, omegas + count), nu);
    std::copy(r.begin(), r.end(), rho);
  });
}
int pdmg_lfa_model_smoothing(pdmg_lfa_model* m, double omega, double* mu, double* argmax) {
  return guarded([&] {
    if (!m || !mu) throw ConfigError("pdmg_lfa_model_smoothing: NULL argument");
    m->m.smoothing(omega, mu, argmax);
  });
}
int pdmg_lfa_optimize_omega(pdmg_lfa_model* m, int32_t objective, int32_t nu, double* omega, double* value) {
  return guarded([&] {
    if (!m || !omega || !value) throw ConfigError("pdmg_lfa_optimize_omega: NULL argument");
    if (objective == PDMG_LFA_TWO_GRID_RHO)
      minimize_scalar([&](const std::vector<double>& ws) { return m->m.rho(ws, nu); }, omega, value);
    else if (objective == PDMG_LFA_SMOOTHING_MU)
      minimize_scalar([&](const std::vector<double>& ws) { return m->m.mu(ws); }, omega, value);
    else
      throw ConfigError("pdmg_lfa_optimize_omega: unknown objective");
  });
}
int pdmg_lfa_optimize_omega_smoothing(pdmg_c128 lambda, double h, int32_t smoother, const pdmg_lfa_config* lfa,
                                      int32_t device, double* omega, double* value) {
  return guarded([&] {
    if (!lfa || !omega || !value) throw ConfigError("pdmg_lfa_optimize_omega_smoothing: NULL argument");
    validate_lfa(*lfa);
    LfaModel M;  // smoothing objective: only the high-frequency symbol cache (lfa.cpp:231-246)
    M.S = make_setup(lambda, h, smoother);
    M.n = lfa->samples_per_dim, M.device = device;
    CK(cudaSetDevice(device));
    const int cnt = 3 * M.n * M.n;
    CK(cudaMalloc(&M.high_ml, sizeof(double2) * cnt));
    k_lfa_high_ml<<<(cnt + 255) / 256, 256>>>(M.S, M.n, M.high_ml);
    CK(cudaGetLastError());
    minimize_scalar([&](const std::vector<double>& ws) { return M.mu(ws); }, omega, value);
  });
}

}  // extern "C"
