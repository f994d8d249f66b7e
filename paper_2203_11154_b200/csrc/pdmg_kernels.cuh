// pdmg_kernels.cuh -- sm_100a kernels for the batched complex-shifted-Laplacian multigrid.
//
// Device layout: every level of every shift is stored with an explicit
// zero ghost ring.  For subdivision count n (h = 1/n, m = n-1 interior per side) a shift's block is
// (n+1) rows x pitch n elements; interior node (i,j), 1 <= i,j <= m, lives at j*n + i.  Row 0, row n and
// column 0 are ghosts (column n of row j aliases column 0 of row j+1), so neighbours of boundary nodes
// read zeros -- the homogeneous Dirichlet truncation of grid.cpp:30-58/69-90.  Kernels never write
// ghosts.  Shifts are stacked with stride (n+1)*n; all arrays are double2 (c128) or float2 (c64).
//
// One templated "level pass" kernel (k_level) implements every grid operator on the path, fused:
//   stage A  u_in  = [u] (+ P e_c)                    (load, zero guess, or prolongate-and-correct)
//   stage B  r     = b - (A + lambda I) u_in           (grid.cpp:92-100)
//   stage C  u_out = u_in + omega M r                  (smoother.cpp:49-67; Vanka 9-pt or Jacobi)
//   stage D  r2    = b - (A + lambda I) u_out          (residual of the new iterate)
//   stage E  b_c   = R r2  or  partial ||r2||^2        (grid.cpp:102-121, grid.cpp:7-11)
// A CTA owns a TILE_W-column x H-row output tile of one shift and marches down it in CHUNK-row steps;
// each stage keeps a RING-row circular buffer in shared memory (wide enough for its halo), so global
// memory is read ~once per pass: u, b, e_c in; u_out, b_c out.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <type_traits>

namespace pdmg_b200 {

template <class T>
struct vec2;
template <>
struct vec2<double> {
  using type = double2;
};
template <>
struct vec2<float> {
  using type = float2;
};

template <class V>
__device__ __forceinline__ V cz() {
  V r;
  r.x = 0;
  r.y = 0;
  return r;
}
template <class V>
__device__ __forceinline__ V cadd(V a, V b) {
  a.x += b.x;
  a.y += b.y;
  return a;
}
template <class V>
__device__ __forceinline__ V csub(V a, V b) {
  a.x -= b.x;
  a.y -= b.y;
  return a;
}
template <class V>
__device__ __forceinline__ V cmul(V a, V b) {
  V r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}
template <class V, class S>
__device__ __forceinline__ V cscale(S s, V a) {
  a.x *= s;
  a.y *= s;
  return a;
}

// Storage type T (double: complex128, float: complex64); all arithmetic is fp64.  For complex64 the
// fp32 values are widened on load, so the residual b - (A + lambda I) u of the *stored* iterate is
// formed exactly (an fp32-arithmetic residual floors at 1.2e-5 > the 1e-5 target).
__device__ __forceinline__ double2 ld2(double2 v) { return v; }
__device__ __forceinline__ double2 ld2(float2 v) { return make_double2((double)v.x, (double)v.y); }
template <class V>
__device__ __forceinline__ V st2(double2 v);
template <>
__device__ __forceinline__ double2 st2<double2>(double2 v) {
  return v;
}
template <>
__device__ __forceinline__ float2 st2<float2>(double2 v) {
  return make_float2((float)v.x, (float)v.y);
}

__device__ __forceinline__ double2 csel(bool c, double2 a) { return c ? a : make_double2(0.0, 0.0); }
// b - (1/h^2)((4+eta) u_c - (u_w + u_e + u_s + u_n)) with dd = (4+eta)/h^2 folded into FMAs
#ifndef PDMG_RES5_TREE
#define PDMG_RES5_TREE 0
#endif
__device__ __forceinline__ double2 res5(double2 b, double ih2, double2 dd, double2 uc, double2 uw, double2 ue,
                                        double2 us, double2 un) {
  const double sx = (uw.x + ue.x) + (us.x + un.x), sy = (uw.y + ue.y) + (us.y + un.y);
#if PDMG_RES5_TREE
  // the centre term and the neighbour sum as independent chains (dependency depth 3 instead of 5)
  double tx = fma(-dd.x, uc.x, b.x), ty = fma(-dd.x, uc.y, b.y);
  tx = fma(dd.y, uc.y, tx);
  ty = fma(-dd.y, uc.x, ty);
  return make_double2(fma(ih2, sx, tx), fma(ih2, sy, ty));
#else
  double rx = fma(ih2, sx, b.x), ry = fma(ih2, sy, b.y);
  rx = fma(-dd.x, uc.x, rx);
  rx = fma(dd.y, uc.y, rx);
  ry = fma(-dd.x, uc.y, ry);
  ry = fma(-dd.y, uc.x, ry);
  return make_double2(rx, ry);
#endif
}
// k0 rc + k1 e1 + k2 e2 (complex), as one FMA chain per component
__device__ __forceinline__ double2 cdot3(double2 k0, double2 rc, double2 k1, double2 e1, double2 k2, double2 e2) {
  double x = k0.x * rc.x;
  x = fma(-k0.y, rc.y, x);
  x = fma(k1.x, e1.x, x);
  x = fma(-k1.y, e1.y, x);
  x = fma(k2.x, e2.x, x);
  x = fma(-k2.y, e2.y, x);
  double y = k0.x * rc.y;
  y = fma(k0.y, rc.x, y);
  y = fma(k1.x, e1.y, y);
  y = fma(k1.y, e1.x, y);
  y = fma(k2.x, e2.y, y);
  y = fma(k2.y, e2.x, y);
  return make_double2(x, y);
}

// k0 x + k1 y (complex), one FMA chain per component (PDMG_CMAD_TREE: two chains of two per component)
#ifndef PDMG_CMAD_TREE
#define PDMG_CMAD_TREE 0
#endif
__device__ __forceinline__ double2 cmad2(double2 k0, double2 x, double2 k1, double2 y) {
#if PDMG_CMAD_TREE
  const double ra = fma(-k0.y, x.y, k0.x * x.x), rb = fma(-k1.y, y.y, k1.x * y.x);
  const double ia = fma(k0.y, x.x, k0.x * x.y), ib = fma(k1.y, y.x, k1.x * y.y);
  return make_double2(ra + rb, ia + ib);
#endif
  double re = k0.x * x.x;
  re = fma(-k0.y, x.y, re);
  re = fma(k1.x, y.x, re);
  re = fma(-k1.y, y.y, re);
  double im = k0.x * x.y;
  im = fma(k0.y, x.x, im);
  im = fma(k1.x, y.y, im);
  im = fma(k1.y, y.x, im);
  return make_double2(re, im);
}

// a + k0 x + k1 y (complex): the accumulator starts the FMA chains
__device__ __forceinline__ double2 cmad2_acc(double2 a, double2 k0, double2 x, double2 k1, double2 y) {
  double re = fma(k0.x, x.x, a.x);
  re = fma(-k0.y, x.y, re);
  re = fma(k1.x, y.x, re);
  re = fma(-k1.y, y.y, re);
  double im = fma(k0.x, x.y, a.y);
  im = fma(k0.y, x.x, im);
  im = fma(k1.x, y.y, im);
  im = fma(k1.y, y.x, im);
  return make_double2(re, im);
}

// Per (level, shift) operator coefficients, precomputed on the host in fp64 (multigrid.cpp:47-58).
struct LevelCoef {
  double2 d;      // 4 + eta, eta = lambda h^2              (grid.cpp:73)
  double2 dd;     // (4 + eta) / h^2
  double2 k0;     // Vanka: omega*(h^2/4)*4a ; Jacobi: omega*h^2/(4+eta)
  double2 k1;     // Vanka: omega*(h^2/4)*2b
  double2 k2;     // Vanka: omega*(h^2/4)*c
  double inv_h2;  // 1/h^2
  double pad_;
};

// The per-shift operator coefficients of one level, passed to the marching kernels as a __grid_constant__
// kernel parameter: indexed by blockIdx.y (CTA-uniform) they load into uniform registers (LDCU) and feed
// the FP64 instructions as uniform operands, which frees 18 vector registers per thread in kernels whose
// occupancy is register-bound.  A launch covers at most COEF_MAX shifts (16 KB of parameters).
struct CoefU {
  double2 dd, k0, k1, k2;  // as in LevelCoef
};
constexpr int COEF_MAX = 256;
struct CoefPack {
  double inv_h2;
  int shift0;  // global shift of blockIdx.y == 0
  int pad_;
  CoefU c[COEF_MAX];
};
__device__ __forceinline__ LevelCoef coef_of(const CoefPack& cp) {
  LevelCoef cf;
  const CoefU& u = cp.c[blockIdx.y];
  cf.d = make_double2(0.0, 0.0);
  cf.dd = u.dd, cf.k0 = u.k0, cf.k1 = u.k1, cf.k2 = u.k2;
  cf.inv_h2 = cp.inv_h2;
  cf.pad_ = 0.0;
  return cf;
}

enum : int { POST_NONE = 0, POST_NORM = 1, POST_RESTRICT = 2, POST_RESID = 3 };

#ifndef PDMG_CHUNK
#define PDMG_CHUNK 16
#endif
#ifndef PDMG_RPT
#define PDMG_RPT 4
#endif
constexpr int TILE_W = 64;          // output columns per CTA
constexpr int CHUNK = PDMG_CHUNK;   // rows each stage advances per step
constexpr int RING = CHUNK + 2;     // rows of the r / delta rings (a stage reads its producer's rows -1..CHUNK)
constexpr int RING_R = CHUNK + 4;   // ... when the restriction (which looks 2 more rows back) consumes them
constexpr int ARING = 2 * CHUNK + 2;  // rows of the u_in ring: the rows in use + the next chunk landing (TMA)
constexpr int RPT = PDMG_RPT;       // rows per stencil task (register-blocked along the column)
constexpr int RGROUPS = CHUNK / RPT;
constexpr int NTHREADS = 288;       // 9 warps >= (TILE_W + 2*hB) * RGROUPS tasks for every variant
constexpr int CB_ROWS = CHUNK / 2 + 2, CB_COLS = 40;  // coarse block for prolongation
constexpr int VX_W = TILE_W + 2;           // restriction exchange row width

template <class T>
struct LevelArgs {
  using V = typename vec2<T>::type;
  const V* u_in;             // level u (LOADU)
  V* u_out;                  // level u output (STORE) or residual output (POST_RESID)
  const V* b;                // level rhs
  const V* ec;               // coarse correction (PROLONG), coarse layout
  V* bc;                     // coarse rhs output (POST_RESTRICT), coarse layout
  double* partial;           // [shift][tile] partial sums of |r2|^2 (POST_NORM)
  const LevelCoef* coef;     // [shift] at this level
  const int* active;         // [shift] convergence mask, or nullptr
  int n, nc;                 // fine / coarse subdivisions
  int64_t ss, ssc;           // shift strides (elements)
  int ntx, ntiles, H;        // tiles across, tiles per shift, strip height (even)
};

__device__ __forceinline__ int floordiv2(int a) { return a >> 1; }  // arithmetic shift = floor(a/2)

// ---- TMA bulk copies (cp.async.bulk, 1-D) completing on an mbarrier ------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gsrc, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Halo widths and shared-memory footprint of a k_level instantiation.  Rings fed by TMA (u_in, b, e_c)
// hold the storage type; r, delta and the restriction sums hold fp64.  With 8-byte elements the TMA-fed
// buffers start at an even column (16-byte aligned segments), so their halos are rounded up to even.
template <class T, bool USE_A, bool SWEEP, int POST, bool PROLONG>
struct LevelShape {
  using V = typename vec2<T>::type;
  static constexpr bool HASD = POST != POST_NONE;
  static constexpr int hD = POST == POST_RESTRICT ? 1 : 0;
  static constexpr int hC = HASD ? hD + 1 : 0;
  static constexpr int hA = SWEEP ? hC + 2 : hC;
  static constexpr int hB = hA - 1;
  static constexpr bool EVEN = sizeof(V) == 8;
  static constexpr int hAs = EVEN ? (hA + 1) / 2 * 2 : hA;  // storage halo of the u ring
  static constexpr int hBs = EVEN ? (hB + 1) / 2 * 2 : hB;  // storage halo of the b buffer
  static constexpr int WA = TILE_W + 2 * hAs, WBb = TILE_W + 2 * hBs;
  static constexpr int WB = TILE_W + 2 * hB, WC = TILE_W + 2 * hC;
  static constexpr int RR = POST == POST_RESTRICT ? RING_R : RING;  // rows of the r / delta rings
  static constexpr size_t bytes_v = sizeof(V) * ((size_t)(USE_A ? ARING * WA : 0) + (SWEEP ? CHUNK * WBb : 0) +
                                                 (PROLONG ? CB_ROWS * CB_COLS : 0));
  static constexpr size_t bytes_d = sizeof(double2) * ((size_t)(SWEEP ? RR * WB : 0) + (SWEEP && HASD ? RR * WC : 0) +
                                                       (POST == POST_RESTRICT ? 2 * RGROUPS * VX_W : 0));
  static constexpr size_t bytes = 32 + bytes_v + bytes_d + 16 * sizeof(double);
  // CTAs per SM the shared memory allows (227 KB usable); used as the register budget hint
  static constexpr int min_blocks = bytes <= 75 * 1024 ? 3 : 2;
  static_assert(!SWEEP || WB * RGROUPS <= NTHREADS, "stage-B tasks exceed the CTA");
  static_assert(bytes <= 113 * 1024, "two CTAs per SM must fit");
};

// Stage row ranges: stage x (A=0, B=1, C=2, D=3) handles, in step t, rows [base - x + CHUNK t, +CHUNK)
// clipped to [r0 - h_x, r0 + H + h_x), where base = r0 - hA.  Consecutive stages lag one row, so a
// stage only ever reads rows its producer finished in this step or the previous one.  The inputs of
// step t+1 (u rows, b rows, coarse block) stream in by TMA while step t computes.  Ring slots outside
// the interior may hold stale data: every stage masks by interior(), and the one-node ghost ring that
// the 5-point operator reads is zero in global memory (and copied).
template <class T, bool LOADU, bool PROLONG, bool SWEEP, int POST, bool STORE, bool JACOBI>
__global__ void __launch_bounds__(NTHREADS, (LevelShape<T, LOADU || PROLONG, SWEEP, POST, PROLONG>::min_blocks))
    k_level(LevelArgs<T> a) {
  using V = typename vec2<T>::type;
  constexpr bool USE_A = LOADU || PROLONG;  // otherwise u_in == 0
  using SH = LevelShape<T, USE_A, SWEEP, POST, PROLONG>;
  constexpr bool HASD = SH::HASD;
  using D2 = double2;
  constexpr int hA = SH::hA, hB = SH::hB, hC = SH::hC, hD = SH::hD, hAs = SH::hAs, hBs = SH::hBs;
  constexpr int WA = SH::WA, WB = SH::WB, WBb = SH::WBb, WC = SH::WC, RR = SH::RR;
  constexpr int xD = SWEEP ? 3 : 1;  // stage index of D
  constexpr int VB = (int)sizeof(V);
  constexpr int ALN = SH::EVEN ? 2 : 1;  // TMA segment alignment in elements

  const int shift = blockIdx.y;
  if (a.active != nullptr && a.active[shift] == 0) return;  // converged shifts are frozen
  const int tile = blockIdx.x;
  const int tx = tile % a.ntx, ty = tile / a.ntx;
  const int n = a.n, m = n - 1, H = a.H;
  const int c0 = tx * TILE_W, r0 = ty * H;
  const int tid = threadIdx.x;
  const int64_t sbase = (int64_t)shift * a.ss;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);  // [2] chunk barriers
  D2* dm_ = reinterpret_cast<D2*>(smem_raw + 32);  // fp64 buffers first (16-B aligned)
  D2* RB = dm_;  // r = b - L u_in: RR x WB
  if constexpr (SWEEP) dm_ += RR * WB;
  D2* RC = dm_;  // delta = omega M r: RR x WC
  if constexpr (SWEEP && HASD) dm_ += RR * WC;
  D2* VX = dm_;  // vertical 1-2-1 sums exchanged for the restriction: [2*RGROUPS][VX_W]
  if constexpr (POST == POST_RESTRICT) dm_ += 2 * RGROUPS * VX_W;
  double* red = reinterpret_cast<double*>(dm_);
  V* sm = reinterpret_cast<V*>(red + 16);
  V* RA = sm;  // u_in (+ P e_c): ARING x WA, local col 0 = storage col c0 - hAs
  if constexpr (USE_A) sm += ARING * WA;
  V* Bb = sm;  // b rows of the current B step: CHUNK x WBb, local col 0 = storage col c0 - hBs
  if constexpr (SWEEP) sm += CHUNK * WBb;
  V* CB = sm;  // coarse block for the prolongation
  if constexpr (PROLONG) sm += CB_ROWS * CB_COLS;

  const LevelCoef cf = a.coef[shift];
  const V* __restrict__ uin = a.u_in + sbase;
  const V* __restrict__ bb = a.b + sbase;
  V* __restrict__ uout = a.u_out + sbase;
  const V* __restrict__ ecs = a.ec + (int64_t)shift * a.ssc;
  const int nc = a.nc;
  const int base = r0 - hA;
  const int n_iter = (H + 2 * hA + CHUNK - 1) / CHUNK;

  auto row_in = [&](int row) { return (unsigned)(row - 1) < (unsigned)m; };
  // ring slot of a row (rows are > -NR); the callers step it incrementally
  auto slot = [](int row, int NR) { return (row + 4 * NR) % NR; };

  // ---- TMA issue of a step's inputs: warp 0, one bulk copy per row segment --------------------
  auto issue = [&](int t, bool do_a, bool do_b) {
    if (tid >= 32) return;
    const int lane = tid;
    unsigned bytes = 0;
    // u rows of step t: storage rows [k0, k0+CHUNK) clipped to [0, n], cols [c0-hA, c0+W+hA) clipped to [0, n]
    const int k0 = base + CHUNK * t;
    const int ar_lo = max(k0, 0), ar_hi = min(min(k0 + CHUNK, r0 + H + hA), n + 1);
    const int ac_lo = max(c0 - hA, 0) / ALN * ALN, ac_hi = (min(c0 + TILE_W + hA, n + 1) + ALN - 1) / ALN * ALN;
    const int kb0 = base - 1 + CHUNK * t;
    const int br_lo = max(max(kb0, r0 - hB), 1), br_hi = min(min(kb0 + CHUNK, r0 + H + hB), m + 1);
    const int bc_lo = max(c0 - hB, 1) / ALN * ALN, bc_hi = (min(c0 + TILE_W + hB, m + 1) + ALN - 1) / ALN * ALN;
    const int J0 = floordiv2(k0), I0 = floordiv2(c0 - hA) / ALN * ALN;
    const int er_lo = max(J0, 0), er_hi = min(J0 + CB_ROWS, nc + 1);
    const int ec_lo = max(I0, 0), ec_hi = (min(I0 + CB_COLS, nc + 1) + ALN - 1) / ALN * ALN;
    // One arrival per step and barrier phase, carrying the byte count of ALL of the step's copies (the
    // b rows of a sweep are issued later, after stage B has consumed the previous ones).
    const bool arrive = USE_A ? do_a : do_b;
    if (arrive) {
      if constexpr (LOADU) bytes += (unsigned)(max(ar_hi - ar_lo, 0) * max(ac_hi - ac_lo, 0) * VB);
      if constexpr (PROLONG) bytes += (unsigned)(max(er_hi - er_lo, 0) * max(ec_hi - ec_lo, 0) * VB);
      if constexpr (SWEEP) bytes += (unsigned)(max(br_hi - br_lo, 0) * max(bc_hi - bc_lo, 0) * VB);
      if (lane == 0) mbar_arrive_expect_tx(&bar[t & 1], bytes);
    }
    __syncwarp();
    if (do_a && USE_A) {
      if constexpr (LOADU) {
        if (ac_hi > ac_lo)
          for (int row = ar_lo + lane; row < ar_hi; row += 32)
            tma_load_1d(RA + slot(row, ARING) * WA + (ac_lo - (c0 - hAs)), uin + (int64_t)row * n + ac_lo,
                        (unsigned)((ac_hi - ac_lo) * VB), &bar[t & 1]);
      }
      if constexpr (PROLONG) {
        if (ec_hi > ec_lo)
          for (int J = er_lo + lane; J < er_hi; J += 32)
            tma_load_1d(CB + (J - J0) * CB_COLS + (ec_lo - I0), ecs + (int64_t)J * nc + ec_lo,
                        (unsigned)((ec_hi - ec_lo) * VB), &bar[t & 1]);
      }
    }
    if (do_b && SWEEP) {
      if (bc_hi > bc_lo)
        for (int row = br_lo + lane; row < br_hi; row += 32)
          tma_load_1d(Bb + (row - kb0) * WBb + (bc_lo - (c0 - hBs)), bb + (int64_t)row * n + bc_lo,
                      (unsigned)((bc_hi - bc_lo) * VB), &bar[t & 1]);
    }
  };

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // b - (A + lambda I) u at an interior node (grid.cpp:69-100 order: d*u_c - W - E - S - N)
  auto apply_res = [&](D2 bv, D2 uc, D2 uw, D2 ue, D2 us, D2 un) {
    return res5(bv, cf.inv_h2, cf.dd, uc, uw, ue, us, un);
  };

  // fixed per-thread task geometry
  const int rg = tid / (SWEEP ? WB : 1);  // (recomputed per stage below where widths differ)
  (void)rg;

  double nacc = 0.0;
  issue(0, true, true);

  for (int t = 0; t < n_iter; ++t) {
    if (USE_A || SWEEP) mbar_wait(&bar[t & 1], (unsigned)((t >> 1) & 1));
    __syncthreads();
    // ---------------- stage A: u_in = [u] + P e_c (in place on the landed rows) -----------------
    if constexpr (PROLONG) {  // u += prolong_bilinear(e_c) (grid.cpp:123-153, multigrid.cpp:75)
      // one thread per coarse cell (I, J): its 2x2 fine block (2I..2I+1, 2J..2J+1) needs e(I..I+1, J..J+1)
      const int k0 = base + CHUNK * t;
      const int J0 = floordiv2(k0), I0 = floordiv2(c0 - hA) / ALN * ALN;
      const int rhi = min(k0 + CHUNK, r0 + H + hA);
      const int clo = c0 - hAs, chi = clo + WA;
      const int Jb = floordiv2(k0), Ib = floordiv2(clo);
      const int nJ = floordiv2(rhi - 1) - Jb + 1, nI = floordiv2(chi - 1) - Ib + 1;
      for (int q = tid; q < nJ * nI; q += NTHREADS) {
        const int jl = q / nI, il = q - jl * nI;
        const int J = Jb + jl, I = Ib + il;
        const V* e0 = CB + (J - J0) * CB_COLS + (I - I0);
        const D2 e00 = ld2(e0[0]), e10 = ld2(e0[1]), e01 = ld2(e0[CB_COLS]), e11 = ld2(e0[CB_COLS + 1]);
        const D2 pv[2][2] = {{e00, cscale(0.5, cadd(e00, e10))},
                             {cscale(0.5, cadd(e00, e01)), cscale(0.25, cadd(cadd(cadd(e00, e10), e01), e11))}};
#pragma unroll
        for (int dy = 0; dy < 2; ++dy) {
          const int row = 2 * J + dy;
          if (row < k0 || row >= rhi) continue;
          V* rowp = RA + slot(row, ARING) * WA - clo;
          const bool rin = row_in(row);
#pragma unroll
          for (int dx = 0; dx < 2; ++dx) {
            const int col = 2 * I + dx;
            if (col < clo || col >= chi) continue;
            D2 v = cz<D2>();
            if (rin && (unsigned)(col - 1) < (unsigned)m) {
              v = pv[dy][dx];
              if constexpr (LOADU) v = cadd(ld2(rowp[col]), v);
            }
            const V vs = st2<V>(v);
            rowp[col] = vs;  // non-interior nodes become exact zeros (the ghost ring the stencil reads)
            if constexpr (!SWEEP && STORE) {
              if (row >= r0 && row < r0 + H && rin && col >= c0 && col < c0 + TILE_W && (unsigned)(col - 1) < (unsigned)m)
                uout[(int64_t)row * n + col] = vs;
            }
          }
        }
      }
      __syncthreads();
    }
    if constexpr (SWEEP) {
      if (t + 1 < n_iter) issue(t + 1, true, false);  // lands in ring rows no stage of step t touches
      // -------------- stage B: r = b - (A + lambda I) u_in  (grid.cpp:69-100) ---------------------
      const int gB = tid / WB;
      const int kbg = base - 1 + CHUNK * t + RPT * gB;
      if (tid < WB * RGROUPS && kbg + RPT > r0 - hB && kbg < r0 + H + hB) {
        // rows outside the stage range are computed too (from stale ring rows) and written to ring slots no
        // later stage reads; only the interior mask (Dirichlet zeros) must be exact.  Task groups entirely
        // outside the range (first/last step of a strip) are skipped.
        const int g = gB, ci = tid - g * WB;
        const int kb = kbg, col = c0 - hB + ci;
        const bool cin = (unsigned)(col - 1) < (unsigned)m;
        int sa = slot(kb - 1, ARING), sb = slot(kb, RR);
        const V* ap = RA + ci + (hAs - hB);  // local col of `col` in the A ring
        const V* bbp = Bb + ci + (hBs - hB) + RPT * g * WBb;  // ... and in the b buffer
        D2* bp = RB + ci;
        D2 am, ac, an;
        if constexpr (USE_A) {
          am = ld2(ap[sa * WA]);
          sa = sa + 1 == ARING ? 0 : sa + 1;
          ac = ld2(ap[sa * WA]);
        }
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int row = kb + i;
          const int sn = sa + 1 == ARING ? 0 : sa + 1;
          const D2 bv = ld2(bbp[i * WBb]);
          D2 r;
          if constexpr (USE_A) {
            an = ld2(ap[sn * WA]);
            const V* arow = ap + sa * WA;
            r = apply_res(bv, ac, ld2(arow[-1]), ld2(arow[1]), am, an);
            am = ac, ac = an;
          } else {
            r = bv;  // zero initial guess: r = b
          }
          bp[sb * WB] = csel(cin && row_in(row), r);
          sa = sn;
          sb = sb + 1 == RR ? 0 : sb + 1;
        }
      }
      __syncthreads();
      if (t + 1 < n_iter) issue(t + 1, false, true);
      // -------------- stage C: delta = omega M r; u_out = u_in + delta  (smoother.cpp:49-67) -------
      const int gC = tid / WC;
      const int kcg = base - 2 + CHUNK * t + RPT * gC;
      if (tid < WC * RGROUPS && kcg + RPT > r0 - hC && kcg < r0 + H + hC) {
        const int g = gC, ci = tid - g * WC;
        const int kc = kcg, col = c0 - hC + ci;
        const bool cin = (unsigned)(col - 1) < (unsigned)m;
        const bool cout = cin && col >= c0 && col < c0 + TILE_W;
        const D2* rpc = RB + (ci + (hB - hC));  // local col of `col` in the r ring
        int s = slot(kc - 1, RR);
        // rolling 3-row window over the column: r and the horizontal pair sum r(col-1)+r(col+1)
        D2 rm, rc, rn, sm_, sc, sn_;
        {
          const D2* q = rpc + s * WB;
          rm = q[0];
          if constexpr (!JACOBI) sm_ = cadd(q[-1], q[1]);
          s = s + 1 == RR ? 0 : s + 1;
          q = rpc + s * WB;
          rc = q[0];
          if constexpr (!JACOBI) sc = cadd(q[-1], q[1]);
        }
        int sa = slot(kc, ARING), sd = slot(kc, RR);
        V* outp = uout + (int64_t)kc * n + col;
        const int olo = max(r0, 1), ohi = min(r0 + H, m + 1);  // stored output rows
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int row = kc + i;
          s = s + 1 == RR ? 0 : s + 1;
          {
            const D2* q = rpc + s * WB;
            rn = q[0];
            if constexpr (!JACOBI) sn_ = cadd(q[-1], q[1]);
          }
          const bool inn = cin && row_in(row);
          D2 dl;
          if constexpr (JACOBI) {
            dl = cmul(cf.k0, rc);
          } else {  // (h^2/4)[c,2b,c;2b,4a,2b;c,2b,c] r with omega folded in (smoother.cpp:31-40)
            const D2 e1 = cadd(cadd(sc, rm), rn);
            const D2 e2 = cadd(sm_, sn_);
            dl = cdot3(cf.k0, rc, cf.k1, e1, cf.k2, e2);
          }
          dl = csel(inn, dl);
          if constexpr (STORE) {
            D2 ui = cz<D2>();
            if constexpr (USE_A) ui = ld2(RA[sa * WA + ci + (hAs - hC)]);
            const V us = st2<V>(cadd(ui, dl));
            if (cout && row >= olo && row < ohi) *outp = us;
            // with fp32 storage, continue with the correction the stored iterate actually received, so
            // the residual formed next is that of the stored u (exact: a difference of two floats)
            if constexpr (SH::EVEN) dl = csel(inn, csub(ld2(us), ui));
          }
          if constexpr (HASD) RC[sd * WC + ci] = dl;
          rm = rc, sm_ = sc, rc = rn, sc = sn_;
          sa = sa + 1 == ARING ? 0 : sa + 1;
          sd = sd + 1 == RR ? 0 : sd + 1;
          outp += n;
        }
      }
      if constexpr (HASD) __syncthreads();
    }
    // -------------- stage D: r2 = b - (A + lambda I) u_out ---------------------------------------------
    // after a sweep r2 = r - (A + lambda I) delta (exact algebra; b is not read again); without a sweep
    // u_out = u_in (ring A, or zero) and b comes from global memory.
    if constexpr (POST == POST_NORM || POST == POST_RESID || POST == POST_RESTRICT) {
      constexpr int WU = SWEEP ? WC : WA;  // width of the ring holding u_out (or delta)
      constexpr int NRU = SWEEP ? RR : ARING;
      using UT = typename std::conditional<SWEEP, D2, V>::type;
      const UT* U;
      if constexpr (SWEEP) U = RC;
      else U = RA;
      constexpr int hU = SWEEP ? hC : hAs;
      // r2 down one column over rows [k, k+nr): rolls a 3-row window of U
      auto r2_column = [&](int k, int col, int nr, auto&& consume) {
        const int lc = col - (c0 - hU);
        const UT* up = U + lc;
        int s = slot(k - 1, NRU);
        int srb = slot(k, RR);
        const bool cin = (unsigned)(col - 1) < (unsigned)m;
        D2 um = cz<D2>(), uc = cz<D2>(), un = cz<D2>();
        if constexpr (USE_A || SWEEP) {
          um = ld2(up[s * WU]);
          s = s + 1 == NRU ? 0 : s + 1;
          uc = ld2(up[s * WU]);
        }
        const V* bg = bb + (int64_t)k * n + col;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
          if (i >= nr) break;
          const int row = k + i;
          const int sn = s + 1 == NRU ? 0 : s + 1;
          if constexpr (USE_A || SWEEP) un = ld2(up[sn * WU]);
          const bool inn = cin && row_in(row);
          D2 rb;
          if constexpr (SWEEP) rb = RB[srb * WB + (col - (c0 - hB))];
          else rb = inn ? ld2(bg[0]) : cz<D2>();
          D2 r2 = rb;
          if constexpr (USE_A || SWEEP) {
            const UT* urow = up + s * WU;
            r2 = apply_res(rb, uc, ld2(urow[-1]), ld2(urow[1]), um, un);
          }
          r2 = csel(inn, r2);
          consume(i, row, r2);
          um = uc, uc = un;
          s = sn;
          srb = srb + 1 == RR ? 0 : srb + 1;
          bg += n;
        }
      };
      if constexpr (POST == POST_NORM || POST == POST_RESID) {
        const int gD = tid / TILE_W;
        const int kdg = base - xD + CHUNK * t + RPT * gD;
        if (tid < TILE_W * RGROUPS && kdg + RPT > r0 && kdg < r0 + H) {
          const int g = gD, ci = tid - g * TILE_W;
          const int kd = kdg, col = c0 + ci;
          if (col <= m) {
            r2_column(kd, col, RPT, [&](int, int row, D2 r2) {
              if (row >= r0 && row < r0 + H && row_in(row) && col >= 1) {
                if constexpr (POST == POST_NORM) nacc += r2.x * r2.x + r2.y * r2.y;
                if constexpr (POST == POST_RESID) uout[(int64_t)row * n + col] = st2<V>(r2);
              }
            });
          }
        }
      } else {
        // ------------ restriction b_c(I,J) = (1/16)[1 2 1;2 4 2;1 2 1] r2 around (2I,2J) (grid.cpp:102-121)
        // coarse rows J of this step are those whose fine rows 2J-1..2J+1 completed in it.
        const int kcur = min(base - xD + CHUNK * (t + 1), r0 + H + hD);
        const int kprev = min(base - xD + CHUNK * t, r0 + H + hD);
        const int mc = nc - 1;
        int jlo = max(r0 >> 1, 1);
        if (t > 0) jlo = max(jlo, floordiv2(kprev - 2) + 1);
        const int jhi = min(min(floordiv2(kcur - 2), ((r0 + H) >> 1) - 1), mc);
        const int nj = jhi - jlo + 1;
        // phase 1: per fine column f, vertical 1-2-1 sums of r2 for coarse rows (jlo+2g, jlo+2g+1)
        if (tid < VX_W * RGROUPS) {
          const int g = tid / VX_W, f = tid - g * VX_W;
          const int Ja = jlo + 2 * g;
          if (2 * g < nj) {
            const int col = c0 - 1 + f;
            const int nr = 2 * g + 1 < nj ? 5 : 3;
            D2 acc_a = cz<D2>(), acc_b = cz<D2>();
            r2_column(2 * Ja - 1, col, nr, [&](int i, int, D2 r2) {
              if (i <= 2) acc_a = cadd(acc_a, i == 1 ? cscale(2.0, r2) : r2);
              if (i >= 2) acc_b = cadd(acc_b, i == 3 ? cscale(2.0, r2) : r2);
            });
            VX[(2 * g) * VX_W + f] = acc_a;
            VX[(2 * g + 1) * VX_W + f] = acc_b;
          }
        }
        __syncthreads();
        // phase 2: horizontal 1-2-1 of the column sums, one coarse node per thread
        V* __restrict__ bco = a.bc + (int64_t)shift * a.ssc;
        if (tid < nj * (TILE_W / 2)) {
          const int jr = tid / (TILE_W / 2), il = tid - jr * (TILE_W / 2);
          const int I = (c0 >> 1) + il, J = jlo + jr;
          if (I >= 1 && I <= mc) {
            const D2* v = VX + jr * VX_W + 2 * il;  // fine col 2I - 1 is local f = 2*il
            const D2 s = cadd(cadd(v[0], cscale(2.0, v[1])), v[2]);
            bco[(int64_t)J * nc + I] = st2<V>(cscale(1.0 / 16.0, s));
          }
        }
      }
    }
    if constexpr (!SWEEP) {  // D read u_in rows further back: refill only after they are done
      if (USE_A && t + 1 < n_iter) {
        __syncthreads();
        issue(t + 1, true, false);
      }
    }
  }

  if constexpr (POST == POST_NORM) {
    // deterministic block reduction: warp tree, then warp 0 over the per-warp sums
    for (int o = 16; o > 0; o >>= 1) nacc += __shfl_xor_sync(0xffffffffu, nacc, o);
    if ((tid & 31) == 0) red[tid >> 5] = nacc;
    __syncthreads();
    if (tid < 32) {
      double v = tid < NTHREADS / 32 ? red[tid] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (tid == 0) a.partial[(int64_t)shift * a.ntiles + tile] = v;
    }
  }
}

// Per-shift convergence bookkeeping after a cycle (multigrid.cpp:96-105): one warp per shift sums the
// tile partials in a fixed order, records the residual history and freezes converged shifts.
struct SolveState {
  int* active;       // [S]
  int* iterations;   // [S]
  int* converged;    // [S]
  double* r0;        // [S]
  double* hist;      // [S][max_iter+1]
  int* n_active;     // scalar
  int S, max_iter;
  double tol;
  int* parity;       // [max_iter+1]: which u buffer holds the iterate after cycle k (written by k_finalize)
  int cur;
  // max over the shifts still active after cycle k of the predicted next residual ratio
  // (r_k / r0) (r_k / r_{k-1}) / tol, as double bits (atomicMax; k >= 2): the host's cue that the next
  // iterate is likely the last one (solve_device)
  unsigned long long* pred;
};

static __global__ void k_finalize(const double* __restrict__ partial, int ntiles, int k, SolveState st) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0 && st.parity) st.parity[k] = st.cur;
  if (warp >= st.S) return;
  const int s = warp;
  if (st.active[s] == 0) return;
  double acc = 0.0;
  for (int t = lane; t < ntiles; t += 32) acc += partial[(int64_t)s * ntiles + t];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane != 0) return;
  const double r = sqrt(acc);
  const int H = st.max_iter + 1;
  int act = 1;
  if (k == 0) {
    st.r0[s] = r;
    st.hist[(int64_t)s * H] = r;
    st.iterations[s] = 0;
    if (r == 0.0 || st.tol >= 1.0) {
      st.converged[s] = 1;
      act = 0;
    }
  } else {
    st.hist[(int64_t)s * H + k] = r;
    st.iterations[s] = k;
    if (r <= st.tol * st.r0[s]) {
      st.converged[s] = 1;
      act = 0;
    } else if (k >= st.max_iter) {
      act = 0;
    }
  }
  st.active[s] = act;
  if (act) atomicAdd(st.n_active, 1);
  if (act && st.pred) {
    const double q = k >= 2 ? (r / st.r0[s]) * (r / st.hist[(int64_t)s * H + k - 1]) / st.tol : 1e300;
    atomicMax(st.pred, (unsigned long long)__double_as_longlong(q));
  }
}

// ---- rolling host solve (Engine::solve_rolling) -------------------------------------------------------------------
// Shifts join the batch as their right-hand sides arrive from the host and leave it as they converge, so every shift
// carries its own cycle counter: kcur[s] = cycles completed = index of the iterate whose residual norm the coming
// round's first fine pass forms (norm-next).  k_admit starts shifts [s0, s1); k_finalize_roll is k_finalize with the
// per-shift counter: it also records, for a shift that stops, which u buffer holds its final iterate (fbuf[s] = the
// buffer the first pass read).
static __global__ void k_admit(int* __restrict__ active, int* __restrict__ kcur, int s0, int s1) {
  for (int s = s0 + blockIdx.x * blockDim.x + threadIdx.x; s < s1; s += gridDim.x * blockDim.x) active[s] = 1, kcur[s] = 0;
}
static __global__ void k_finalize_roll(const double* __restrict__ partial, int ntiles, SolveState st,
                                       int* __restrict__ kcur, int* __restrict__ fbuf) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= st.S) return;
  const int s = warp;
  if (st.active[s] == 0) return;
  double acc = 0.0;
  for (int t = lane; t < ntiles; t += 32) acc += partial[(int64_t)s * ntiles + t];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane != 0) return;
  const double r = sqrt(acc);
  const int H = st.max_iter + 1, k = kcur[s];
  int act = 1;
  st.hist[(int64_t)s * H + k] = r;
  st.iterations[s] = k;
  if (k == 0) {  // multigrid.cpp:91-94
    st.r0[s] = r;
    if (r == 0.0 || st.tol >= 1.0) st.converged[s] = 1, act = 0;
  } else if (r <= st.tol * st.r0[s]) {  // multigrid.cpp:96-105
    st.converged[s] = 1, act = 0;
  } else if (k >= st.max_iter) {
    act = 0;
  }
  st.active[s] = act;
  if (act) {
    kcur[s] = k + 1;
    atomicAdd(st.n_active, 1);
  } else {
    fbuf[s] = st.cur;
  }
}

// Device -> mapped pinned host words, written by SMs over PCIe: small result copies that never queue
// behind bulk transfers on the copy engines (the chunked host solve keeps those busy).
static __global__ void k_copy_words(const uint32_t* __restrict__ src, volatile uint32_t* dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Residual-only norm pass ||b - (A + lambda I) u||^2 (multigrid.cpp:91, 96-105) for the convergence
// test outside a smoothing pass (predicted last norm, the max_iter closing norm).  HBM-bound: u and b are
// each read once (the neighbour rows and columns are L1 hits); one CTA per (RN_ROWS-row block, shift),
// each thread two adjacent columns per row, so a row is one coalesced 1 KB-per-warp sweep; the partial
// layout is k_finalize's [shift][tile].  The ghost ring reads as zero (homogeneous Dirichlet).
constexpr int RN_ROWS = 16, RN_THREADS = 256;
template <class T>
__global__ void __launch_bounds__(RN_THREADS) k_resid_norm(const typename vec2<T>::type* __restrict__ u,
                                                            const typename vec2<T>::type* __restrict__ b,
                                                            const LevelCoef* __restrict__ coef,
                                                            const int* __restrict__ active, int n, int64_t ss,
                                                            double* __restrict__ partial) {
  __shared__ double red[RN_THREADS / 32];
  const int shift = blockIdx.y, tile = blockIdx.x, ntiles = gridDim.x;
  if (active != nullptr && active[shift] == 0) return;
  const int m = n - 1;
  const LevelCoef cf = coef[shift];
  const auto* us = u + (int64_t)shift * ss;
  const auto* bs = b + (int64_t)shift * ss;
  const int j0 = 1 + tile * RN_ROWS, j1 = min(j0 + RN_ROWS, m + 1);
  double acc = 0.0;
  for (int j = j0; j < j1; ++j) {
    for (int i = 1 + threadIdx.x; i <= m; i += RN_THREADS) {
      const int64_t p = (int64_t)j * n + i;
      const double2 r = res5(ld2(bs[p]), cf.inv_h2, cf.dd, ld2(us[p]), ld2(us[p - 1]), ld2(us[p + 1]), ld2(us[p - n]),
                             ld2(us[p + n]));
      acc += r.x * r.x + r.y * r.y;
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < RN_THREADS / 32; ++w) t += red[w];
    partial[(int64_t)shift * ntiles + tile] = t;
  }
}

// Per-shift norms (op-level pdmg_norm): sum partials -> sqrt.
static __global__ void k_sum_partials(const double* __restrict__ partial, int ntiles, int S, double* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= S) return;
  double acc = 0.0;
  for (int t = lane; t < ntiles; t += 32) acc += partial[(int64_t)warp * ntiles + t];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[warp] = sqrt(acc);
}

// Coarsest-level direct solve u = A^{-1} b per shift (replaces Eigen PartialPivLU::solve,
// dense.cpp:90-100): one CTA per shift, one thread per unknown, A^{-1} precomputed in fp64 on the host.
template <class T>
__global__ void k_coarse_solve(const typename vec2<T>::type* __restrict__ b, typename vec2<T>::type* __restrict__ u,
                               const double2* __restrict__ ainv, const int* __restrict__ active, int n, int64_t ss) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sb = reinterpret_cast<double2*>(smem_raw);
  const int s = blockIdx.x;
  if (active != nullptr && active[s] == 0) return;
  const int m = n - 1, N = m * m;
  const typename vec2<T>::type* bs = b + (int64_t)s * ss;
  for (int q = threadIdx.x; q < N; q += blockDim.x) sb[q] = ld2(bs[(int64_t)(q / m + 1) * n + (q % m + 1)]);
  __syncthreads();
  const double2* A = ainv + (int64_t)s * N * N;
  typename vec2<T>::type* us = u + (int64_t)s * ss;
  for (int r = threadIdx.x; r < N; r += blockDim.x) {
    double2 acc = cz<double2>();
    for (int c = 0; c < N; ++c) acc = cadd(acc, cmul(A[(int64_t)r * N + c], sb[c]));
    us[(int64_t)(r / m + 1) * n + (r % m + 1)] = st2<typename vec2<T>::type>(acc);
  }
}

// Compact complex128 (reference layout, [S][m][m]) <-> ghosted level storage of type T.
template <class T>
__global__ void k_unpack(const double2* __restrict__ src, typename vec2<T>::type* __restrict__ dst, int n, int64_t ss,
                         int64_t total) {
  const int m = n - 1;
  const int64_t N = (int64_t)m * m;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = q / N, p = q % N;
    const int j = (int)(p / m) + 1, i = (int)(p % m) + 1;
    dst[s * ss + (int64_t)j * n + i] = st2<typename vec2<T>::type>(src[q]);
  }
}

// Gather u out of the buffer each shift finished in: sel = parity[iterations[s]].
template <class T>
__global__ void k_pack(const typename vec2<T>::type* __restrict__ buf0, const typename vec2<T>::type* __restrict__ buf1,
                       const int* __restrict__ iters,
                       const int* __restrict__ parity, double2* __restrict__ dst, int n, int64_t ss, int64_t total) {
  const int m = n - 1;
  const int64_t N = (int64_t)m * m;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = q / N, p = q % N;
    const int j = (int)(p / m) + 1, i = (int)(p % m) + 1;
    const int sel = (iters == nullptr) ? 0 : parity[iters[s]];
    const typename vec2<T>::type* src = sel == 0 ? buf0 : buf1;
    dst[q] = ld2(src[s * ss + (int64_t)j * n + i]);
  }
}

}  // namespace pdmg_b200


// ===================================================================================================
// Small-grid path: one CTA runs the WHOLE solve of one shift (multigrid.cpp:85-110 loop, V or W cycles,
// convergence test) in a single launch.  For grids whose per-level passes are far too small to fill the
// GPU (BASELINE configs 1-2: one 63x63 system, 32 127x127 systems) the batched path is launch- and
// sync-latency bound; here every operator is a block-wide pass over the (L2/L1-resident) level arrays
// separated by __syncthreads, and the host is not involved until the solve ends.
// Level arrays use the same ghosted layout; u lives in u[0] (updated in place), u[1] holds r.
// ===================================================================================================
namespace pdmg_b200 {

constexpr int SMALL_THREADS = 1024;
constexpr int MAX_LEVELS = 16;

template <class T>
struct SmallLevel {
  using V = typename vec2<T>::type;
  V* u;   // u (level 0: the iterate; coarser: the correction e)
  V* r;   // residual scratch
  V* b;   // rhs (level 0: user rhs; coarser: restricted residual)
  const LevelCoef* coef;
  int n;
  int64_t ss;
};

template <class T>
struct SmallArgs {
  SmallLevel<T> lv[MAX_LEVELS];
  int L;
  int nu1, nu2, gamma, jacobi, max_iter;
  double tol;
  const double2* ainv;  // [S][N][N] coarsest inverse (fp64)
  int coarse_N;
  int* iterations;
  int* converged;
  double* r0;
  double* hist;
  int* n_active;
  const int* active;  // tail mode: convergence mask of the batched solve (nullptr = all)
  int tail_zero;      // tail mode: u of the tail's top level starts at zero (first visit of the cycle)
};

template <class T>
struct SmallSolver {
  using V = typename vec2<T>::type;
  const SmallArgs<T>& a;
  int s;
  double* red;  // [33] block reduction scratch (shared)
  double2* cb;  // coarsest rhs staging (shared, coarse_N)
  // A shift may be worked on by a thread-block CLUSTER of csize CTAs (small batches: BASELINE configs 1-2, the coarse
  // tail of a strong-scaling share or of a rolling round -- fewer shifts than SMs).  The passes stride over the
  // cluster's threads, a pass ends with a cluster barrier (release / acquire at cluster scope: the level arrays live
  // in global memory and the next pass reads nodes another CTA wrote), block reductions are combined over distributed
  // shared memory, and the coarsest solve runs on the cluster's first CTA.  csize = 1 is the one-CTA form.
  int crank = 0, csize = 1;
  int tid = 0, nthr = 0;  // this thread's rank among, and the number of, the threads that share the shift
  __device__ __forceinline__ void sync() const {
    if (csize > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
  }

  __device__ __forceinline__ V* ptr(V* base, int l) const { return base + (int64_t)s * a.lv[l].ss; }
  // Block-wide passes walk the m x m interior as rows of W = 2^lw >= m slots (node index = slot >> lw, slot & (W - 1)):
  // shifts and masks instead of a division by m per node and pass (the passes are instruction-bound: 55 % of what
  // they issued was index arithmetic); the W - m slots past a row's end idle.
  __device__ __forceinline__ static int row_bits(int m) { return m > 1 ? 32 - __clz(m - 1) : 0; }
  __device__ __forceinline__ LevelCoef coef(int l) const { return a.lv[l].coef[s]; }

  // r = b - (A + lambda I) u on level l (grid.cpp:69-100); returns the block-reduced ||r||^2 if wanted
  __device__ double residual(int l, bool zero_u, bool want_norm) const {
    const SmallLevel<T>& L = a.lv[l];
    const int n = L.n, m = n - 1;
    const LevelCoef cf = coef(l);
    const V* u = ptr(L.u, l);
    const V* b = ptr(L.b, l);
    V* r = ptr(L.r, l);
    double acc2 = 0.0;
    const int lw = row_bits(m);
    for (int q = tid; q < (m << lw); q += nthr) {
      const int j = (q >> lw) + 1, i = (q & ((1 << lw) - 1)) + 1;
      if (i > m) continue;
      const int p = j * n + i;
      double2 rv = ld2(b[p]);
      if (!zero_u) {
        double2 acc = cmul(cf.d, ld2(u[p]));
        acc = csub(acc, ld2(u[p - 1]));
        acc = csub(acc, ld2(u[p + 1]));
        acc = csub(acc, ld2(u[p - n]));
        acc = csub(acc, ld2(u[p + n]));
        rv = csub(rv, cscale(cf.inv_h2, acc));
      }
      r[p] = st2<V>(rv);
      if (want_norm) acc2 += rv.x * rv.x + rv.y * rv.y;
    }
    if (!want_norm) {
      sync();
      return 0.0;
    }
    for (int o = 16; o > 0; o >>= 1) acc2 += __shfl_xor_sync(0xffffffffu, acc2, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc2;
    __syncthreads();
    double tot = 0.0;
    if (threadIdx.x < 32) {
      tot = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      if (threadIdx.x == 0) red[32] = tot;
    }
    sync();  // (also ends the pass: r is complete)
    if (csize > 1) {  // the CTAs' partial sums, in rank order, over distributed shared memory
      tot = 0.0;
      for (int q = 0; q < csize; ++q) tot += *cooperative_groups::this_cluster().map_shared_rank(&red[32], q);
    } else {
      tot = red[32];
    }
    sync();
    return tot;
  }

  // u += omega M r (Vanka 9-point or Jacobi), in place; u := omega M r when zero_u (smoother.cpp:49-67)
  __device__ void correct(int l, bool zero_u) const {
    const SmallLevel<T>& L = a.lv[l];
    const int n = L.n, m = n - 1;
    const LevelCoef cf = coef(l);
    V* u = ptr(L.u, l);
    const V* r = ptr(L.r, l);
    const int lw = row_bits(m);
    for (int q = tid; q < (m << lw); q += nthr) {
      const int j = (q >> lw) + 1, i = (q & ((1 << lw) - 1)) + 1;
      if (i > m) continue;
      const int p = j * n + i;
      double2 dl;
      if (a.jacobi) {
        dl = cmul(cf.k0, ld2(r[p]));
      } else {
        const double2 e1 = cadd(cadd(cadd(ld2(r[p - n]), ld2(r[p - 1])), ld2(r[p + 1])), ld2(r[p + n]));
        const double2 e2 =
            cadd(cadd(cadd(ld2(r[p - n - 1]), ld2(r[p - n + 1])), ld2(r[p + n - 1])), ld2(r[p + n + 1]));
        dl = cadd(cadd(cmul(cf.k0, ld2(r[p])), cmul(cf.k1, e1)), cmul(cf.k2, e2));
      }
      u[p] = st2<V>(zero_u ? dl : cadd(ld2(u[p]), dl));
    }
    sync();
  }

  // b_{l+1} = R r_l (grid.cpp:102-121) and e_{l+1} = 0
  __device__ void restrict_to(int l) const {
    const SmallLevel<T>& F = a.lv[l];
    const SmallLevel<T>& Cc = a.lv[l + 1];
    const int nf = F.n, nc = Cc.n, mc = nc - 1;
    const V* r = ptr(F.r, l);
    V* bc = ptr(Cc.b, l + 1);
    const int lw = row_bits(mc);
    for (int q = tid; q < (mc << lw); q += nthr) {
      const int J = (q >> lw) + 1, I = (q & ((1 << lw) - 1)) + 1;
      if (I > mc) continue;
      const int c = (2 * J) * nf + 2 * I;
      double2 sum = ld2(r[c - nf - 1]);
      sum = cadd(sum, cscale(2.0, ld2(r[c - nf])));
      sum = cadd(sum, ld2(r[c - nf + 1]));
      sum = cadd(sum, cscale(2.0, ld2(r[c - 1])));
      sum = cadd(sum, cscale(4.0, ld2(r[c])));
      sum = cadd(sum, cscale(2.0, ld2(r[c + 1])));
      sum = cadd(sum, ld2(r[c + nf - 1]));
      sum = cadd(sum, cscale(2.0, ld2(r[c + nf])));
      sum = cadd(sum, ld2(r[c + nf + 1]));
      bc[J * nc + I] = st2<V>(cscale(1.0 / 16.0, sum));
    }
    sync();
  }

  // u_l += P e_{l+1} (grid.cpp:123-153); u_l := P e when zero_u
  __device__ void prolong_add(int l, bool zero_u) const {
    const SmallLevel<T>& F = a.lv[l];
    const SmallLevel<T>& Cc = a.lv[l + 1];
    const int nf = F.n, mf = nf - 1, nc = Cc.n;
    V* u = ptr(F.u, l);
    const V* e = ptr(Cc.u, l + 1);
    const int lw = row_bits(mf);
    for (int q = tid; q < (mf << lw); q += nthr) {
      const int j = (q >> lw) + 1, i = (q & ((1 << lw) - 1)) + 1;
      if (i > mf) continue;
      const V* e0 = e + (j >> 1) * nc + (i >> 1);
      double2 pv;
      if (!(i & 1) && !(j & 1)) pv = ld2(e0[0]);
      else if ((i & 1) && !(j & 1)) pv = cscale(0.5, cadd(ld2(e0[0]), ld2(e0[1])));
      else if (!(i & 1) && (j & 1)) pv = cscale(0.5, cadd(ld2(e0[0]), ld2(e0[nc])));
      else pv = cscale(0.25, cadd(cadd(cadd(ld2(e0[0]), ld2(e0[1])), ld2(e0[nc])), ld2(e0[nc + 1])));
      const int p = j * nf + i;
      u[p] = st2<V>(zero_u ? pv : cadd(ld2(u[p]), pv));
    }
    sync();
  }

  __device__ void coarse_solve(int l) const {
    const SmallLevel<T>& L = a.lv[l];
    const int n = L.n, m = n - 1, N = a.coarse_N;
    const V* b = ptr(L.b, l);
    V* u = ptr(L.u, l);
    if (crank == 0) {  // (the staged right-hand side lives in this CTA's shared memory)
      for (int q = threadIdx.x; q < N; q += blockDim.x) cb[q] = ld2(b[(int64_t)(q / m + 1) * n + (q % m + 1)]);
      __syncthreads();
      const double2* A = a.ainv + (int64_t)s * N * N;
      for (int rr = threadIdx.x; rr < N; rr += blockDim.x) {
        double2 acc = cz<double2>();
        for (int c = 0; c < N; ++c) acc = cadd(acc, cmul(A[(int64_t)rr * N + c], cb[c]));
        u[(int64_t)(rr / m + 1) * n + (rr % m + 1)] = st2<V>(acc);
      }
    }
    sync();
  }

  // cycle_on_level (multigrid.cpp:63-77) as an explicit state machine (no device recursion): st[l] counts
  // the gamma sub-cycles started from level l; z[l] says u_l is still the zero guess.
  __device__ void cycle(bool zero0) const {
    int st[MAX_LEVELS];
    bool z[MAX_LEVELS];
    int l = 0;
    st[0] = 0;
    z[0] = zero0;
    while (l >= 0) {
      if (l + 1 == a.L) {  // coarsest: u = A^{-1} b (multigrid.cpp:64-68)
        coarse_solve(l);
        --l;
        continue;
      }
      if (st[l] == 0) {
        for (int k = 0; k < a.nu1; ++k) {
          residual(l, z[l], false);
          correct(l, z[l]);
          z[l] = false;
        }
        residual(l, z[l], false);
        restrict_to(l);  // rc = R(b - L u); ec = 0 (multigrid.cpp:71-72)
        st[l] = 1;
        st[l + 1] = 0;
        z[l + 1] = true;
        ++l;
        continue;
      }
      if (st[l] < a.gamma) {  // W-cycle: second recursion from the current ec (multigrid.cpp:73-74)
        ++st[l];
        st[l + 1] = 0;
        z[l + 1] = false;
        ++l;
        continue;
      }
      prolong_add(l, z[l]);  // u += P ec (multigrid.cpp:75)
      z[l] = false;
      for (int k = 0; k < a.nu2; ++k) {
        residual(l, false, false);
        correct(l, false);
      }
      --l;
    }
  }
};

// Coarse tail of a batched cycle: one CTA per shift runs cycle_on_level from the first tail level down
// (multigrid.cpp:63-77) entirely in one launch; the tail's top-level u (the correction) starts at zero and
// is left in lv[0].u for the prolongation by the level above.
template <class T>
__global__ void __launch_bounds__(SMALL_THREADS, 1) k_small_cycle(SmallArgs<T> a) {
  using V = typename vec2<T>::type;
  __shared__ double red[33];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int csize = (int)cooperative_groups::this_cluster().num_blocks();
  const int crank = (int)cooperative_groups::this_cluster().block_rank(), s = (int)blockIdx.x / csize;
  if (a.active != nullptr && a.active[s] == 0) return;  // (the whole cluster)
  SmallSolver<T> S{a, s, red, reinterpret_cast<double2*>(smem_raw), crank, csize,
                   crank * (int)blockDim.x + (int)threadIdx.x, csize * (int)blockDim.x};
  S.cycle(a.tail_zero != 0);
}

template <class T>
__global__ void __launch_bounds__(SMALL_THREADS, 1) k_small_solve(SmallArgs<T> a) {
  using V = typename vec2<T>::type;
  __shared__ double red[33];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int csize = (int)cooperative_groups::this_cluster().num_blocks();
  const int crank = (int)cooperative_groups::this_cluster().block_rank(), s = (int)blockIdx.x / csize;
  SmallSolver<T> S{a, s, red, reinterpret_cast<double2*>(smem_raw), crank, csize,
                   crank * (int)blockDim.x + (int)threadIdx.x, csize * (int)blockDim.x};
  const bool lead = crank == 0 && threadIdx.x == 0;
  const int H = a.max_iter + 1;
  // u = 0 (multigrid.cpp:90), r0 = ||b|| (:91)
  const double r0 = sqrt(S.residual(0, true, true));
  if (lead) {
    a.r0[s] = r0;
    a.hist[(int64_t)s * H] = r0;
    a.iterations[s] = 0;
    a.converged[s] = (r0 == 0.0 || a.tol >= 1.0) ? 1 : 0;
  }
  {
    const SmallLevel<T>& L0 = a.lv[0];
    V* u = S.ptr(L0.u, 0);
    const int n = L0.n, m = n - 1;
    for (int q = S.tid; q < m * m; q += S.nthr) u[(int64_t)(q / m + 1) * n + (q % m + 1)] = st2<V>(cz<double2>());
    S.sync();
  }
  if (r0 == 0.0 || a.tol >= 1.0) return;
  for (int k = 1; k <= a.max_iter; ++k) {
    S.cycle(k == 1);
    const double rk = sqrt(S.residual(0, false, true));
    if (lead) {
      a.hist[(int64_t)s * H + k] = rk;
      a.iterations[s] = k;
    }
    if (rk <= a.tol * r0) {
      if (lead) a.converged[s] = 1;
      break;
    }
  }
}

}  // namespace pdmg_b200

// ===================================================================================================
// k_march: warp-marching fused sweep for the large levels (the dominant kernels of every cycle).
// Each warp owns a 64-column strip (2 columns per lane) of one shift, H_s rows tall, and marches down it
// one row per step.  Every stage (u_in -> r -> delta/u_out -> r2 -> restriction or norm) keeps a 3-row
// register window per column; horizontal neighbours come from warp shuffles (lane l holds columns
// c0 + 2l, c0 + 2l + 1).  No shared memory and no CTA barriers: warps are independent, so latency is hidden
// by the other warps and the loads prefetched one row ahead.  Each stage's valid columns shrink by one
// per stage; a warp stores only its middle 64 - 2 hA columns (neighbouring strips overlap by 2 hA).
// Stage lags: at step j the warp loads u row j, computes r at j-1, delta/u_out at j-2, r2 at j-3 and the
// coarse row whose fine rows end at j-3.
// ===================================================================================================
namespace pdmg_b200 {

constexpr int MARCH_WARPS = 4;  // warps per CTA (independent)
// Register caps of the marching passes (k_march2).  The caps, not the CTA shape, set the warps resident per SM
// (registers are allocated in units of 16 per thread: 8 warps for the two-sweep passes at cap 232 -- 198-218 used --
// and 12 for the one-sweep passes at cap 168).  Lower caps for 9 or 10 warps were measured slower (DESIGN 3.2d).
// The host picks the CTA size (Engine::m2_wpc / m1_wpc, 4 warps).
#ifndef PDMG_M2_MAXNREG
#define PDMG_M2_MAXNREG 232
#endif
#ifndef PDMG_M1_MAXNREG
#define PDMG_M1_MAXNREG 168
#endif
constexpr int M2_MAXNREG = PDMG_M2_MAXNREG, M1_MAXNREG = PDMG_M1_MAXNREG;
constexpr int M2_RING = 8;  // slots of the per-warp b-row ring of k_march2 (rows j-1 .. j-5 live); 8 KB per warp
constexpr int M2_SMEM_PER_WARP = M2_RING * 2 * 32 * 16;
__host__ __device__ constexpr int march2_maxnreg(bool two) { return two ? M2_MAXNREG : M1_MAXNREG; }
// warps of a marching pass resident per SM (registers are allocated per warp in units of 8 per thread)
__host__ __device__ constexpr int march2_warps_per_sm(bool two) {
  return 65536 / (32 * ((march2_maxnreg(two) + 7) / 8 * 8)) > 64 ? 64 : 65536 / (32 * ((march2_maxnreg(two) + 7) / 8 * 8));
}

__device__ __forceinline__ double2 shfl_up2(double2 v) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ double2 shfl_dn2(double2 v) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}

template <class T>
struct MarchArgs {
  using V = typename vec2<T>::type;
  const V* u_in;
  V* u_out;
  const V* b;
  const V* ec;
  V* bc;
  double* partial;
  const LevelCoef* coef;
  const int* active;
  int n, nc;
  int64_t ss, ssc;
  int ntx, ntasks, Hs;  // strips across, warp tasks per shift, strip height
  int64_t elems, elems_c;  // elements from u_in / b / u_out (and ec / bc) to the end of their allocations
                           // (PDMG_BOUNDS_CHECK builds assert every k_march2 access against them)
  int loop_a;           // k_march2 loop shape (see there)
};

template <class T, bool LOADU, bool PROLONG, int POST, bool JACOBI, int LC, bool NORM_IN = false>
#ifndef PDMG_MARCH_MINB
#define PDMG_MARCH_MINB 3
#endif
__global__ void __launch_bounds__(32 * MARCH_WARPS, PDMG_MARCH_MINB) k_march(MarchArgs<T> a) {
  using V = typename vec2<T>::type;
  using D2 = double2;
  constexpr bool EVEN = sizeof(V) == 8;
  constexpr bool HASD = POST != POST_NONE;
  constexpr int hD = POST == POST_RESTRICT ? 1 : 0;
  constexpr int hC = HASD ? hD + 1 : 0;
  constexpr int hA = hC + 2;
  constexpr int WOUT = 32 * LC - 2 * hA;  // stored columns per warp
  const int shift = blockIdx.y;
  if (a.active != nullptr && a.active[shift] == 0) return;
  const int task = blockIdx.x * MARCH_WARPS + __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // warp-uniform (see k_march2)
  if (task >= a.ntasks) return;
  const int lane = threadIdx.x & 31;
  const int tx = task % a.ntx, ty = task / a.ntx;
  const int n = a.n, m = n - 1, Hs = a.Hs, nc = a.nc;
  const int x0 = tx * WOUT, r0 = ty * Hs;
  const int64_t sbase = (int64_t)shift * a.ss;
  const V* __restrict__ uin = a.u_in + sbase;
  const V* __restrict__ bb = a.b + sbase;
  V* __restrict__ uout = a.u_out + sbase;
  const V* __restrict__ ecs = a.ec + (int64_t)shift * a.ssc;
  const LevelCoef cf = a.coef[shift];

  const int cA = x0 - hA + LC * lane;  // storage column of this lane's first column
  bool cin[LC], cst[LC];
#pragma unroll
  for (int k = 0; k < LC; ++k) {
    const int c = cA + k;
    cin[k] = (unsigned)(c - 1) < (unsigned)m;
    cst[k] = cin[k] && c >= x0 && c < x0 + WOUT;
  }
  const int rlo = r0 - hA, rhi = r0 + Hs + hA;  // rows loaded
  const int olo = max(r0, 1), ohi = min(r0 + Hs, m + 1);
  auto row_in = [&](int row) { return (unsigned)(row - 1) < (unsigned)m; };

  // prolongation: a 2-coarse-row register window of e(Ie .. Ie+LC, J), Ie = floor(cA / 2), refilled once per
  // coarse row (rows are loaded in increasing order), instead of 2-4 coarse loads per fine row
  constexpr int NE = LC + 1;
  D2 E0[NE], E1[NE];
  int wJ = -1000;
  const int Ie = cA >> 1;
  auto load_crow = [&](int J, D2* out) {
#pragma unroll
    for (int q = 0; q < NE; ++q) {
      const int I = Ie + q;
      out[q] = ((unsigned)J <= (unsigned)nc && (unsigned)I <= (unsigned)nc) ? ld2(ecs[(int64_t)J * nc + I]) : cz<D2>();
    }
  };
  // u_in row `row` (out: the raw load, consumed a step later) and its prolongation term (pout, from the
  // register window: computed now so neither the u nor the coarse loads are waited on in this step)
  auto load_u = [&](int row, D2* out, D2* pout) {
#pragma unroll
    for (int k = 0; k < LC; ++k) out[k] = pout[k] = cz<D2>();
    if constexpr (PROLONG) {
      const int J = row >> 1;
      if (J == wJ + 1) {
#pragma unroll
        for (int q = 0; q < NE; ++q) E0[q] = E1[q];
        load_crow(J + 1, E1);
        wJ = J;
      } else if (J != wJ) {
        load_crow(J, E0);
        load_crow(J + 1, E1);
        wJ = J;
      }
    }
    if (!row_in(row)) return;
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      if (!cin[k]) continue;
      const int c = cA + k;
      if constexpr (LOADU) out[k] = ld2(uin[(int64_t)row * n + c]);
      if constexpr (PROLONG) {  // u += prolong_bilinear(e_c) (grid.cpp:123-153)
        const int q = (c >> 1) - Ie;  // 0 .. LC-1 (runtime for odd cA): select, no local-memory indexing
        D2 a0 = E0[0], a1 = E0[1], b0 = E1[0], b1 = E1[1];
#pragma unroll
        for (int z = 1; z < LC; ++z)
          if (q == z) a0 = E0[z], a1 = E0[z + 1], b0 = E1[z], b1 = E1[z + 1];
        // row parity is warp-uniform: even rows never wait on the coarse row (E1) just issued
        D2 p;
        if (row & 1) p = (c & 1) ? cscale(0.25, cadd(cadd(cadd(a0, a1), b0), b1)) : cscale(0.5, cadd(a0, b0));
        else p = (c & 1) ? cscale(0.5, cadd(a0, a1)) : a0;
        pout[k] = p;
      }
    }
  };
  auto load_b = [&](int row, D2* out) {
#pragma unroll
    for (int k = 0; k < LC; ++k)
      out[k] = (row_in(row) && cin[k]) ? ld2(bb[(int64_t)row * n + cA + k]) : cz<D2>();
  };
  // horizontal neighbours of a row held as x[LC]: west of column k and east of column k
  auto west = [&](const D2* x, int k, const D2& wl) { return k == 0 ? wl : x[k - 1]; };
  auto east = [&](const D2* x, int k, const D2& er) { return k == LC - 1 ? er : x[k + 1]; };

  D2 U[3][LC], R[3][LC], S[3][LC], Dl[3][LC];
  D2 Vp[LC], R2c[LC];  // restriction: partial vertical 1-2-1 sum of the coarse row in progress, last r2
  D2 Bc[LC], Un[LC], Pn[LC], Bn[LC];
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int k = 0; k < LC; ++k) U[q][k] = R[q][k] = S[q][k] = Dl[q][k] = cz<D2>();
#pragma unroll
  for (int k = 0; k < LC; ++k) Vp[k] = R2c[k] = cz<D2>();
  double nacc = 0.0;
  load_u(rlo, Un, Pn);
  load_b(rlo - 1, Bn);

  for (int j = rlo; j < rhi; ++j) {
    // ---- stage A: u row j (prefetched), prefetch row j+1 --------------------------------------------
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      U[0][k] = U[1][k];
      U[1][k] = U[2][k];
      U[2][k] = PROLONG ? cadd(Un[k], Pn[k]) : Un[k];
      Bc[k] = Bn[k];
    }
    if (j + 1 < rhi) {
      load_u(j + 1, Un, Pn);
      load_b(j, Bn);
    }
    // ---- stage B: r at row j-1 = b - (A + lambda I) u  ---------------------------------------------
    {
      const int row = j - 1;
      const bool rin = row_in(row);
      const D2 wl = shfl_up2(U[1][LC - 1]), er = shfl_dn2(U[1][0]);
      D2 rn[LC];
#pragma unroll
      for (int k = 0; k < LC; ++k)
        rn[k] = csel(rin && cin[k], res5(Bc[k], cf.inv_h2, cf.dd, U[1][k], west(U[1], k, wl), east(U[1], k, er),
                                         U[0][k], U[2][k]));
      if constexpr (NORM_IN) {  // ||b - L u_in||^2 of the owned rows/columns (the previous iterate's residual)
        if (row >= olo && row < ohi) {
#pragma unroll
          for (int k = 0; k < LC; ++k)
            if (cst[k]) nacc += rn[k].x * rn[k].x + rn[k].y * rn[k].y;
        }
      }
      D2 sn[LC];
      if constexpr (!JACOBI) {
        const D2 rwl = shfl_up2(rn[LC - 1]), rer = shfl_dn2(rn[0]);
#pragma unroll
        for (int k = 0; k < LC; ++k) sn[k] = cadd(west(rn, k, rwl), east(rn, k, rer));
      }
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        R[0][k] = R[1][k];
        R[1][k] = R[2][k];
        R[2][k] = rn[k];
        if constexpr (!JACOBI) {
          S[0][k] = S[1][k];
          S[1][k] = S[2][k];
          S[2][k] = sn[k];
        }
      }
    }
    // ---- stage C: delta, u_out at row j-2 (u_in at row j-2 is U[0]) ------------------------------------
    {
      const int row = j - 2;
      const bool rin = row_in(row);
      const bool rst = row >= olo && row < ohi;
      D2 dn[LC];
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        D2 dl;
        if constexpr (JACOBI) {
          dl = cmul(cf.k0, R[1][k]);
        } else {  // (h^2/4)[c,2b,c;2b,4a,2b;c,2b,c] r with omega folded in (smoother.cpp:31-40)
          const D2 e1 = cadd(cadd(S[1][k], R[0][k]), R[2][k]);
          const D2 e2 = cadd(S[0][k], S[2][k]);
          dl = cdot3(cf.k0, R[1][k], cf.k1, e1, cf.k2, e2);
        }
        const bool inn = rin && cin[k];
        dl = csel(inn, dl);
        const D2 ui = U[0][k];
        const V us = st2<V>(cadd(ui, dl));
        if (rst && cst[k]) uout[(int64_t)row * n + cA + k] = us;
        if constexpr (EVEN) dl = csel(inn, csub(ld2(us), ui));
        dn[k] = dl;
      }
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        Dl[0][k] = Dl[1][k];
        Dl[1][k] = Dl[2][k];
        Dl[2][k] = dn[k];
      }
    }
    if constexpr (HASD) {
      // ---- stage D: r2 at row j-3 = r - (A + lambda I) delta  (r at j-3 is R[0]) -----------------------
      const int row = j - 3;
      const bool rin = row_in(row);
      const D2 wl = shfl_up2(Dl[1][LC - 1]), er = shfl_dn2(Dl[1][0]);
      D2 r2[LC];
#pragma unroll
      for (int k = 0; k < LC; ++k)
        r2[k] = csel(rin && cin[k], res5(R[0][k], cf.inv_h2, cf.dd, Dl[1][k], west(Dl[1], k, wl),
                                         east(Dl[1], k, er), Dl[0][k], Dl[2][k]));
      if constexpr (POST == POST_NORM) {
        if (row >= olo && row < ohi) {
#pragma unroll
          for (int k = 0; k < LC; ++k)
            if (cst[k]) nacc += r2[k].x * r2[k].x + r2[k].y * r2[k].y;
        }
      }
      if constexpr (POST == POST_RESTRICT) {
        // ---- stage E: coarse row J, fine rows 2J-1, 2J, 2J+1 (grid.cpp:102-121) --------------------------
        // vertical 1-2-1 accumulated as rows arrive: odd row 2J-1 opens J (and closes J-1), even row 2J adds 2x
        if (row & 1) {
          D2 v[LC];
#pragma unroll
          for (int k = 0; k < LC; ++k) {
            v[k] = cadd(Vp[k], r2[k]);  // closes coarse row (row-1)/2 = J
            Vp[k] = r2[k];              // opens coarse row J+1 with its first fine row
          }
          const int J = (row - 1) >> 1;
          if (row >= r0 + 1 && row <= r0 + Hs && J >= 1 && J <= nc - 1) {
            const D2 vwl = shfl_up2(v[LC - 1]), ver = shfl_dn2(v[0]);
#pragma unroll
            for (int k = 0; k < LC; ++k) {
              const int c = cA + k;
              if (!(c & 1) && c >= x0 && c < x0 + WOUT) {
                const int I = c >> 1;
                if (I >= 1 && I <= nc - 1) {
                  const D2 s = cadd(cadd(west(v, k, vwl), cscale(2.0, v[k])), east(v, k, ver));
                  a.bc[(int64_t)shift * a.ssc + (int64_t)J * nc + I] = st2<V>(cscale(1.0 / 16.0, s));
                }
              }
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < LC; ++k) Vp[k] = cadd(Vp[k], cscale(2.0, r2[k]));
        }
      }
    }
  }
  if constexpr (POST == POST_NORM || NORM_IN) {
    for (int o = 16; o > 0; o >>= 1) nacc += __shfl_xor_sync(0xffffffffu, nacc, o);
    if (lane == 0) a.partial[(int64_t)shift * a.ntasks + task] = nacc;
  }
}

// ===================================================================================================
// k_march2: TWO fused Vanka sweeps per pass (temporal blocking) for the large levels.  A V(nu1, nu2) cycle
// with nu >= 2 runs its last two pre-sweeps (+ residual + restriction) and its first two post-sweeps
// (prolongation + sweeps [+ norm]) as one pass each, so the fine level is streamed twice per cycle instead
// of four times.  Every point gets exactly the arithmetic of two consecutive single sweeps (the second
// sweep's residual is b - L u1 of the first sweep's stored iterate, fp32-rounded for complex64); only the
// halo (hA = 4 + hC columns/rows per side) is computed redundantly by neighbouring strips.
// The Vanka correction delta_t = k0 r_t + k1 (s_t + r_{t-1} + r_{t+1}) + k2 (s_{t-1} + s_{t+1}), s = the
// horizontal neighbour sum of r, is accumulated row by row: c_t = k1 r_t + k2 s_t, d_t = k0 r_t + k1 s_t,
// delta_t = c_{t-1} + d_t + c_{t+1}, so a sweep keeps 2 complex per column in registers instead of 6.
// Stage lags at step j: load u0 row j; r at j-1 -> delta1/u1 at j-2; r' at j-3 -> delta2/u2 at j-4 (stored);
// r2 = b - L u2 at j-5 -> restriction or norm.  b rows j-3 and j-5 are re-read (L1 hits).
// The row loop is unrolled by 3 with the 3-row windows addressed as rings (no register rotation), and
// steps whose rows and columns are all interior run a copy without Dirichlet masking.
// Input rows (u_in and b, 64 columns) reach shared memory by TMA bulk copies issued M2_D rows ahead into a
// per-warp ring of M2_NS slots (one mbarrier each): M2_D rows of both arrays in flight per warp keep
// enough bytes moving to saturate HBM at 8 warps/SM, without spending registers on prefetch.  b rows stay
// in the ring until the second sweep (row j-3) and the post-residual (row j-5) have read them.
// ===================================================================================================
// A lane's two adjacent columns of one row as ONE access (32 B for complex128: LDG.E.256 / STG.E.256, sm_100+;
// 16 B for complex64).  Per-column 16-B accesses at a 32-B lane stride touch every 128-B line of the row twice: 16
// L1 wavefronts per row instead of 8, and the LSU data pipe is the busiest unit of the marching passes (ncu:
// l1tex__data_pipe_lsu_wavefronts 69 %).  The address must be 32-B (16-B) aligned: even column, even n.
struct alignas(32) PairC128 {
  double2 a, b;
};
struct alignas(16) PairC64 {
  float2 a, b;
};
__device__ __forceinline__ void ldpair(const double2* p, double2& a, double2& b) {
  const PairC128 v = *reinterpret_cast<const PairC128*>(p);
  a = v.a, b = v.b;
}
__device__ __forceinline__ void ldpair(const float2* p, double2& a, double2& b) {
  const PairC64 v = *reinterpret_cast<const PairC64*>(p);
  a = ld2(v.a), b = ld2(v.b);
}
__device__ __forceinline__ void ldpair_raw(const double2* p, double2& a, double2& b) { ldpair(p, a, b); }
__device__ __forceinline__ void ldpair_raw(const float2* p, float2& a, float2& b) {
  const PairC64 v = *reinterpret_cast<const PairC64*>(p);
  a = v.a, b = v.b;
}
__device__ __forceinline__ void stpair(double2* p, double2 a, double2 b) {
  PairC128 v;
  v.a = a, v.b = b;
  *reinterpret_cast<PairC128*>(p) = v;
}
__device__ __forceinline__ void stpair(float2* p, float2 a, float2 b) {
  PairC64 v;
  v.a = a, v.b = b;
  *reinterpret_cast<PairC64*>(p) = v;
}
// (PDMG_M2_PF_LANES: a lane's hint covers its own 32 B; with 2 / 4 only every 2nd / 4th lane issues one -- 64 / 128 B
// apart -- which cuts the hints' L1 wavefronts if the prefetch granularity is a 64 / 128 B line)
#ifndef PDMG_M2_PF_LANES
#define PDMG_M2_PF_LANES 1
#endif
__device__ __forceinline__ void l2_prefetch(const void* p) {
  if (PDMG_M2_PF_LANES == 1 || (threadIdx.x & (PDMG_M2_PF_LANES - 1)) == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
template <int X>
struct IC {
  static constexpr int value = X;
};
// (measured and removed, DESIGN 3.2b: input rows through a TMA ring in shared memory, L2 bulk prefetch,
// register prefetch two rows ahead, warp-specialised sweep pairs, V(1,1) cross-cycle fusion -- all slower
// than or as fast as this one-row register prefetch)
// NORM_IN: also leave the partial sums of ||b - L u_in||^2 (the first sweep's residual, i.e. the residual of
// the previous cycle's iterate) in a.partial -- the fine-level convergence norm, read one pass later.
// TWO = false: ONE Vanka sweep per pass with the same machinery (the single-sweep passes of V(1,1) and odd
// nu): u1 at row j-2 is the stored iterate and the post stage reads r2 = b - L u1 at row j-3.
// Debug builds (-DPDMG_BOUNDS_CHECK=1, compute-sanitizer being closed on this pool): every global access of the
// marching pass is checked against its allocation and traps with the offending index.
#ifndef PDMG_BOUNDS_CHECK
#define PDMG_BOUNDS_CHECK 0
#endif
__device__ __forceinline__ void bounds_check(int64_t idx, int64_t lim, int what) {
#if PDMG_BOUNDS_CHECK
  if (idx < 0 || idx >= lim) {
    printf("pdmg bounds check: access %d index %lld outside [0, %lld) block (%d,%d) thread %d\n", what,
           (long long)idx, (long long)lim, blockIdx.x, blockIdx.y, threadIdx.x);
    __trap();
  }
#endif
}
// NF > 0: the level's subdivision count n as a compile-time constant (row offsets become immediates)
template <class T, bool LOADU, bool PROLONG, int POST, bool NORM_IN = false, bool TWO = true, int NF = 0>
__global__ void __maxnreg__(march2_maxnreg(TWO))
    k_march2(const __grid_constant__ MarchArgs<T> a, const __grid_constant__ CoefPack cp) {
  using V = typename vec2<T>::type;
  using D2 = double2;
  constexpr int LC = 2;
  constexpr bool EVEN = sizeof(V) == 8;
  constexpr bool HASD = POST != POST_NONE;
  // paired 32-B / 16-B accesses (ldpair / stpair) where n is a compile-time even constant: the strips start at
  // even columns and the level arrays are 256-B aligned with even row pitch and shift stride
  constexpr bool PAIR = NF > 0 && (NF % 2) == 0;
#ifndef PDMG_M2_PAIR_U
#define PDMG_M2_PAIR_U 0
#endif
#ifndef PDMG_M2_PAIR_B
#define PDMG_M2_PAIR_B 0
#endif
#ifndef PDMG_M2_PAIR_ST
#define PDMG_M2_PAIR_ST 1
#endif
  constexpr bool PAIR_U = PAIR && PDMG_M2_PAIR_U, PAIR_B = PAIR && PDMG_M2_PAIR_B, PAIR_ST = PAIR && PDMG_M2_PAIR_ST;
  static_assert(!(PROLONG && POST == POST_RESTRICT), "prolongation and restriction never share a pass");
  constexpr int hD = POST == POST_RESTRICT ? 1 : 0;
  constexpr int hC = HASD ? hD + 1 : 0;
  // 2 halo columns/rows per sweep (residual + Vanka patch) + the post stage, rounded up to even (strips
  // start at even columns)
  constexpr int hA = (hC + (TWO ? 4 : 2) + 1) & ~1;
  constexpr int WOUT = 32 * LC - 2 * hA;
  // L2 prefetch distance in rows (0 = none).  Measured at C3 (DESIGN 3.2b): 2 rows ahead speeds up every
  // marching pass
#ifndef PDMG_M2_PF
#define PDMG_M2_PF 2
#endif
  constexpr int M2_PF = PDMG_M2_PF;
  // L2 prefetch of the coarse-correction row M2_CPF coarse rows ahead (prolongating passes; 0 = none)
#ifndef PDMG_M2_CPF
#define PDMG_M2_CPF 2
#endif
  constexpr int M2_CPF = PDMG_M2_CPF;
  const int shift = cp.shift0 + blockIdx.y;
  if (a.active != nullptr && a.active[shift] == 0) return;
  // the warp index broadcast from lane 0, so the compiler knows that the task and everything derived from it
  // (row ranges, loop bounds, row parity) is warp-uniform: uniform branches, no divergence guards (BRA.DIV)
  // around the shuffles and no register moves into their fixed operands
  const int task = blockIdx.x * (blockDim.x >> 5) + __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  if (task >= a.ntasks) return;
  const int lane = threadIdx.x & 31;
  const int tx = task % a.ntx, ty = task / a.ntx;
  const int n = NF ? NF : a.n, m = n - 1, Hs = a.Hs, nc = NF ? NF / 2 : a.nc;
  // Strip tx covers the 64 columns from sA = min(tx * WOUT, n - 64): the first strip starts at the ghost column 0
  // and the last one ends at the domain edge (no lanes spent beyond it), the others sit WOUT apart.  It stores
  // columns [xlo, xhi): its 64 columns less hA on each side, up to the domain edge for the first and last strips.
  // ntx = 1 + ceil((n - 64) / WOUT) strips cover a row (Engine::march2_ntx): 9 instead of 10 for the prolongating
  // pair at n = 512.
  const int r0 = ty * Hs;
  const int sA = min(tx * WOUT, max(((n + 1) & ~1) - 32 * LC, 0));
  const int xlo = tx == 0 ? 0 : tx * WOUT + hA, xhi = tx == a.ntx - 1 ? n + 1 : (tx + 1) * WOUT + hA;
  const int64_t sbase = (int64_t)shift * (NF ? (int64_t)(NF + 1) * NF : a.ss);
  const int cA = sA + LC * lane;
  V* __restrict__ uout = a.u_out + sbase + cA;  // per-lane column pointer (row 0)
  const V* __restrict__ ecs = a.ec + (int64_t)shift * (NF ? (int64_t)(NF / 2 + 1) * (NF / 2) : a.ssc);
  const LevelCoef cf = coef_of(cp);

  bool cin[LC], cst[LC];
#pragma unroll
  for (int k = 0; k < LC; ++k) {
    const int c = cA + k;
    cin[k] = (unsigned)(c - 1) < (unsigned)m;
    cst[k] = cin[k] && c >= xlo && c < xhi;
  }
  // rows marched: the strip and its halo, clamped to the domain (rows above row 0 are zero, as the windows start;
  // past row m + 5 nothing is stored or restricted any more)
  const int rlo = max(r0 - hA, 0), rhi = min(r0 + Hs + hA, m + 6);
  const int olo = max(r0, 1), ohi = min(r0 + Hs, m + 1);
  auto row_in = [&](int row) __attribute__((always_inline)) { return (unsigned)(row - 1) < (unsigned)m; };
  // rows before rlo are never loaded: they read as zero (they only reach halo rows, which are not stored)
  auto row_ok = [&](int row) __attribute__((always_inline)) { return row_in(row) && row >= rlo; };
  const V* __restrict__ uin = a.u_in + sbase + cA;  // per-lane column pointers
  const V* __restrict__ bb = a.b + sbase + cA;
  // warp-uniform: every column of the strip (and its coarse prolongation columns) is interior
  const bool col_int = (sA >= 1) && (sA + 32 * LC + 1 <= m - 1);
  // steps j in [jlo_int, jhi_int] touch only interior rows (loads j-5 .. j+1, coarse rows up to (j+1)/2+1)
  const int jlo_int = max(6, rlo + 5), jhi_int = m - 3;  // (register path: loads reach j+1 and j-4)
  // (one sweep: the b rows read are j-1 and j-3 only)
  constexpr bool NEED_B3 = TWO || HASD, NEED_B5 = TWO && HASD;
  // The b rows j-3 and j-5 (second sweep, closing residual) come back from a per-warp ring in shared memory that each
  // lane fills with its own two columns when row j-1 is first used: lane-private slots, so no synchronisation and no
  // bank conflicts, 4 L1 wavefronts per 16-B access instead of the 8 of a strided global re-read, and no prefetch
  // registers (and their copies) for the re-read rows.  M2_RING slots x 2 columns x 32 lanes x 16 B = 8 KB per warp.
#ifndef PDMG_M2_BRING
#define PDMG_M2_BRING 1
#endif
  // (measured: the ring pays in the passes with a post stage -- C3 L0 vanka2+restrict 962 -> 905 us, C5 L0
  // vanka+restrict 180 -> 167 us -- and costs in the prolongating pair, which re-reads one row and has no post
  // stage -- C3 L0 prolong+vanka2 712 -> 755 us; PDMG_M2_BRING = 2 rings every variant that re-reads, 0 none)
  constexpr bool BRING = PDMG_M2_BRING == 2 ? NEED_B3 : PDMG_M2_BRING == 1 ? HASD : false;
  extern __shared__ __align__(16) unsigned char m2_smem[];
  D2* const ring = reinterpret_cast<D2*>(m2_smem) + ((threadIdx.x >> 5) * M2_RING * LC) * 32 + (threadIdx.x & 31);
  auto ring_at = [&](int row, int k) __attribute__((always_inline)) -> D2& {
    return ring[((row & (M2_RING - 1)) * LC + k) * 32];
  };

  const int Ie = cA >> 1;
  // the last strip ends at column m = n - 1 (even n): lane 31's east neighbour is the ghost column n, which no lane
  // holds -- its shuffled value is replaced by zero (masked steps only: an edge strip never runs unmasked ones)
  const bool east_ghost = tx == a.ntx - 1 && lane == 31;
  const bool codd = (cA & 1) != 0;  // warp-uniform (strips start at sA, lanes step by 2)
  // (masked pair loads fetch both columns when either is interior and zero the other: a column outside the domain
  // lies inside the allocation -- the neighbouring row or the tail guard)
  // Mask modes of a step (MK): 0 = every row and column the step touches is interior (nothing masked); 1 = rows and
  // columns masked to the domain (loads predicated); 2 = interior rows of a strip at the left or right domain edge:
  // loads unpredicated (the columns outside the domain lie inside the allocation and hold finite values) and only
  // the residuals, corrections and prolongation forced to zero outside the interior columns -- the ghost column
  // then shields the interior from whatever the lanes beyond it compute.
  // The prefetched rows stay in the STORAGE type (V) until the step that consumes them: widening a complex64 value
  // where it is loaded made the conversion wait for the load it was meant to run ahead of (ncu: 39 % of the c64
  // pass's stall samples sat on those F2F instructions).
  auto gpair = [&](const V* __restrict__ base, int row, V* out, auto MK, int what) __attribute__((always_inline)) {
    constexpr bool MASK = decltype(MK)::value == 1;
    out[0] = out[1] = cz<V>();
    if (!MASK || (row_ok(row) && (cin[0] || cin[1]))) {
      bounds_check(sbase + cA + (int64_t)row * n + 1, a.elems, what);
      bounds_check(sbase + cA + (int64_t)row * n, a.elems, what);
      ldpair_raw(base + (int64_t)row * n, out[0], out[1]);
      if constexpr (MASK) {
        if (!cin[0]) out[0] = cz<V>();
        if (!cin[1]) out[1] = cz<V>();
      }
    }
  };
  auto gread_u = [&](int row, V* out, auto MK) __attribute__((always_inline)) {
    constexpr bool MASK = decltype(MK)::value == 1;
    if constexpr (PAIR_U && LOADU) {
      gpair(uin, row, out, MK, 0);
      return;
    }
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      out[k] = cz<V>();
      if constexpr (LOADU) {
        if (!MASK || (row_ok(row) && cin[k])) {
          bounds_check(sbase + cA + (int64_t)row * n + k, a.elems, 0);
          out[k] = uin[(int64_t)row * n + k];
        }
      }
    }
  };
  auto gload_b = [&](int row, V* out, auto MK) __attribute__((always_inline)) {
    constexpr bool MASK = decltype(MK)::value == 1;
    if constexpr (PAIR_B) {
      gpair(bb, row, out, MK, 1);
      return;
    }
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      if constexpr (MASK) {
        out[k] = cz<V>();
        if (row_ok(row) && cin[k]) {
          bounds_check(sbase + cA + (int64_t)row * n + k, a.elems, 1);
          out[k] = bb[(int64_t)row * n + k];
        }
      } else {
        bounds_check(sbase + cA + (int64_t)row * n + k, a.elems, 2);
        out[k] = bb[(int64_t)row * n + k];
      }
    }
  };
  // prolong_bilinear (grid.cpp:123-153) onto fine row `row` from the coarse values a0 = e(J, Ie),
  // a1 = e(J, Ie+1), b0 = e(J+1, Ie), b1 = e(J+1, Ie+1): even/odd fine column and row (both warp-uniform)
  auto prolong_of = [&](int row, const D2& a0, const D2& a1, const D2& b0, const D2& b1, D2* pout, auto MK)
                        __attribute__((always_inline)) {
    constexpr bool MASK = decltype(MK)::value != 0;
    const bool rin = decltype(MK)::value != 1 || row_ok(row);
    D2 p[LC];
    if (row & 1) {
      const D2 q4 = cscale(0.25, cadd(cadd(cadd(a0, a1), b0), b1));
      p[0] = codd ? q4 : cscale(0.5, cadd(a0, b0));
      p[1] = codd ? cscale(0.5, cadd(a1, b1)) : q4;
    } else {
      const D2 q2 = cscale(0.5, cadd(a0, a1));
      p[0] = codd ? q2 : a0;
      p[1] = codd ? a1 : q2;
    }
#pragma unroll
    for (int k = 0; k < LC; ++k) pout[k] = MASK ? csel(rin && cin[k], p[k]) : p[k];
  };
  // the four coarse values of fine row `row` -- e(J, Ie), e(J, Ie+1), e(J+1, Ie), e(J+1, Ie+1), J = row >> 1 --
  // are loaded unconditionally (indices clamped into the array; out-of-domain points are masked when the
  // prolongation is formed) one step before the row is consumed: no window rotation, no branch around the
  // loads, so no register copy waits on a load that was just issued (DESIGN 3.2b)
  V Cq[4];  // (storage type: widened where the prolongation is formed, one step after the loads)
  auto load_coarse = [&](int row, auto MK) __attribute__((always_inline)) {
    constexpr bool MASK = decltype(MK)::value == 1;
    int J = row >> 1, I = Ie;
    if constexpr (MASK) J = min(max(J, 0), nc - 1), I = min(max(I, 0), nc - 1);
    const V* p0 = ecs + (int64_t)J * nc + I;
    bounds_check((p0 - a.ec) + nc + 1, a.elems_c, 3);
    bounds_check(p0 - a.ec, a.elems_c, 3);
    Cq[0] = p0[0], Cq[1] = p0[1], Cq[2] = p0[nc], Cq[3] = p0[nc + 1];
  };
  auto west = [&](const D2* x, int k, const D2& wl) __attribute__((always_inline)) { return k == 0 ? wl : x[k - 1]; };
  auto east = [&](const D2* x, int k, const D2& er) __attribute__((always_inline)) { return k == LC - 1 ? er : x[k + 1]; };
  // residual b - L u at the centre row c of a window (rows above/below: lo, hi), masked to the domain
  auto resid = [&](const D2* lo, const D2* c, const D2* hi, const D2* bw, bool inside, D2* r, auto MK) __attribute__((always_inline)) {
    constexpr bool MASK = decltype(MK)::value != 0;
    if constexpr (decltype(MK)::value == 2) inside = true;
    const D2 wl = shfl_up2(c[LC - 1]);
    D2 er = shfl_dn2(c[0]);
    if constexpr (MASK) er = csel(!east_ghost, er);
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      const D2 v = res5(bw[k], cf.inv_h2, cf.dd, c[k], west(c, k, wl), east(c, k, er), lo[k], hi[k]);
      r[k] = MASK ? csel(inside && cin[k], v) : v;
    }
  };
  // one Vanka sweep's row update: r_t arrives, delta_{t-1} leaves (masked to the domain at row t-1)
  auto vanka_row = [&](const D2* r, D2* P, D2* C, bool din, D2* dl, auto MK) __attribute__((always_inline)) {
    constexpr bool MASK = decltype(MK)::value != 0;
    if constexpr (decltype(MK)::value == 2) din = true;
    const D2 rwl = shfl_up2(r[LC - 1]);
    D2 rer = shfl_dn2(r[0]);
    if constexpr (MASK) rer = csel(!east_ghost, rer);
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      const D2 s = cadd(west(r, k, rwl), east(r, k, rer));
      const D2 c = cmad2(cf.k1, r[k], cf.k2, s);
      const D2 v = cadd(P[k], c);
      dl[k] = MASK ? csel(din && cin[k], v) : v;
      P[k] = cmad2_acc(C[k], cf.k0, r[k], cf.k1, s);  // C + d, d = k0 r + k1 s, as one FMA chain per component
      C[k] = c;
    }
  };

  D2 U0[3][LC], U1[3][LC], U2[3][LC];
  D2 P1[LC], C1[LC], P2[LC], C2[LC], Vp[LC];
  // rows prefetched one step ahead (indexing these by window phase, so a step reads one slot and loads the
  // next, was measured to make ptxas keep three copies live and spill)
  V Unx[LC], Bn[LC], B3n[LC], B5n[LC];
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int k = 0; k < LC; ++k) U0[q][k] = U1[q][k] = U2[q][k] = cz<D2>();
#pragma unroll
  for (int k = 0; k < LC; ++k) P1[k] = C1[k] = P2[k] = C2[k] = Vp[k] = cz<D2>();
  double nacc = 0.0;
  gread_u(rlo, Unx, IC<1>{});
  gload_b(rlo - 1, Bn, IC<1>{});
  if constexpr (BRING) {  // rows before rlo read as zero
#pragma unroll
    for (int q = 0; q < M2_RING; ++q)
#pragma unroll
      for (int k = 0; k < LC; ++k) ring_at(q, k) = cz<D2>();
  } else {
    if constexpr (NEED_B3) gload_b(rlo - 3, B3n, IC<1>{});
    if constexpr (NEED_B5) gload_b(rlo - 5, B5n, IC<1>{});
  }
  if constexpr (PROLONG) load_coarse(rlo, IC<1>{});

  // one step at row j; window slot of (oldest, middle, newest) row = ((PH + 0, 1, 2) % 3)
  auto step = [&](int j, auto PH, auto MK) __attribute__((always_inline)) {
    constexpr int ph = decltype(PH)::value;
    constexpr int so = ph % 3, sm = (ph + 1) % 3, sn = (ph + 2) % 3;
    // ---- loads: u0 row j (prefetched last step), prefetch u0 row j+1 and b row j; b rows j-3, j-5 ----
    D2 B3[LC], B5[LC], Bc[LC], Un[LC];
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      Un[k] = ld2(Unx[k]);
      Bc[k] = ld2(Bn[k]);
      if constexpr (BRING) {
        ring_at(j - 1, k) = Bc[k];
        if constexpr (NEED_B3) B3[k] = ring_at(j - 3, k);
        if constexpr (NEED_B5) B5[k] = ring_at(j - 5, k);
      } else {
        if constexpr (NEED_B3) B3[k] = ld2(B3n[k]);
        if constexpr (NEED_B5) B5[k] = ld2(B5n[k]);
      }
    }
    if constexpr (PROLONG) {  // u row j += P e_c (coarse values loaded last step)
      D2 Pc[LC];
      prolong_of(j, ld2(Cq[0]), ld2(Cq[1]), ld2(Cq[2]), ld2(Cq[3]), Pc, MK);
#pragma unroll
      for (int k = 0; k < LC; ++k) Un[k] = cadd(Un[k], Pc[k]);
    }
    if (j + 1 < rhi) {
      if constexpr (M2_PF > 0) {  // L2 prefetch of the rows M2_PF steps ahead (one hint per lane)
        if constexpr (LOADU) l2_prefetch(uin + (int64_t)min(j + 1 + M2_PF, n) * n);
        l2_prefetch(bb + (int64_t)min(j + M2_PF, n) * n);
      }
      gread_u(j + 1, Unx, MK);
      gload_b(j, Bn, MK);
      if constexpr (PROLONG) {
        // coarse rows J, J + 1 serve the fine rows 2J and 2J + 1: loaded once per pair, when the even row is next
        // (j is warp-uniform, so this is a uniform branch; the values stay in Cq for two steps)
#ifndef PDMG_M2_COARSE_PAIR
#define PDMG_M2_COARSE_PAIR 1
#endif
        if (!PDMG_M2_COARSE_PAIR || ((j + 1) & 1) == 0) {
          if constexpr (M2_CPF > 0) l2_prefetch(ecs + (int64_t)min((j + 1 + 2 * M2_CPF) >> 1, nc) * nc + Ie);
          load_coarse(j + 1, MK);
        }
      }
      if constexpr (!BRING) {
        if constexpr (NEED_B3) gload_b(j - 2, B3n, MK);
        if constexpr (NEED_B5) gload_b(j - 4, B5n, MK);
      }
    }
#pragma unroll
    for (int k = 0; k < LC; ++k) U0[sn][k] = Un[k];
    // ---- sweep 1: r at j-1, delta1 / u1 at j-2 ------------------------------------------------------
    {
      D2 r[LC], dl[LC];
      resid(U0[so], U0[sm], U0[sn], Bc, row_in(j - 1), r, MK);
      if constexpr (NORM_IN) {
        if (j - 1 >= olo && j - 1 < ohi) {
#pragma unroll
          for (int k = 0; k < LC; ++k)
            if (cst[k]) nacc += r[k].x * r[k].x + r[k].y * r[k].y;
        }
      }
      vanka_row(r, P1, C1, row_in(j - 2), dl, MK);
      const bool rst1 = !TWO && j - 2 >= olo && j - 2 < ohi;
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        D2 u1 = cadd(U0[so][k], dl[k]);
        if constexpr (EVEN) u1 = ld2(st2<V>(u1));  // the iterate the unfused sweep would have stored
        U1[sn][k] = u1;
        if constexpr (!TWO && !PAIR_ST) {
          if (rst1 && cst[k]) {
            bounds_check(sbase + cA + (int64_t)(j - 2) * n + k, a.elems, 4);
            uout[(int64_t)(j - 2) * n + k] = st2<V>(u1);
          }
        }
      }
      if constexpr (!TWO && PAIR_ST) {
        // (a pair with one column on the boundary stores that column's zero: masked steps keep the iterate zero
        // outside the domain, and column 0 / n is the zero ghost)
        if (rst1 && (cst[0] || cst[1])) {
          bounds_check(sbase + cA + (int64_t)(j - 2) * n + 1, a.elems, 4);
          stpair(uout + (int64_t)(j - 2) * n, st2<V>(U1[sn][0]), st2<V>(U1[sn][1]));
        }
      }
    }
    // ---- sweep 2: r' = b - L u1 at j-3, delta2 / u2 at j-4 (stored) ----------------------------------
    if constexpr (TWO) {
      D2 r[LC], dl[LC];
      resid(U1[so], U1[sm], U1[sn], B3, row_in(j - 3), r, MK);
      const int row = j - 4;
      vanka_row(r, P2, C2, row_in(row), dl, MK);
      const bool rst = row >= olo && row < ohi;
      V usp[LC];
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        const V us = st2<V>(cadd(U1[so][k], dl[k]));
        usp[k] = us;
        if constexpr (!PAIR_ST) {
          if (rst && cst[k]) {
            bounds_check(sbase + cA + (int64_t)row * n + k, a.elems, 5);
            uout[(int64_t)row * n + k] = us;
          }
        }
        U2[sn][k] = ld2(us);
      }
      if constexpr (PAIR_ST) {
        if (rst && (cst[0] || cst[1])) {
          bounds_check(sbase + cA + (int64_t)row * n + 1, a.elems, 5);
          stpair(uout + (int64_t)row * n, usp[0], usp[1]);
        }
      }
    }
    if constexpr (HASD) {
      // ---- r2 = b - L u2 at j-5 (one sweep: b - L u1 at j-3): norm or restriction (grid.cpp:102-121) ----
      const int row = TWO ? j - 5 : j - 3;
      D2 r2[LC];
      if constexpr (TWO) resid(U2[so], U2[sm], U2[sn], B5, row_in(row), r2, MK);
      else resid(U1[so], U1[sm], U1[sn], B3, row_in(row), r2, MK);
      if constexpr (POST == POST_NORM) {
        if (row >= olo && row < ohi) {
#pragma unroll
          for (int k = 0; k < LC; ++k)
            if (cst[k]) nacc += r2[k].x * r2[k].x + r2[k].y * r2[k].y;
        }
      }
      if constexpr (POST == POST_RESTRICT) {
        if (row & 1) {
          D2 v[LC];
#pragma unroll
          for (int k = 0; k < LC; ++k) {
            v[k] = cadd(Vp[k], r2[k]);
            Vp[k] = r2[k];
          }
          const int J = (row - 1) >> 1;
          // (shuffles outside the task-dependent test: no divergence check around them)
          const D2 vwl = shfl_up2(v[LC - 1]);
          D2 ver = shfl_dn2(v[0]);
          if constexpr (decltype(MK)::value != 0) ver = csel(!east_ghost, ver);
          if (row >= r0 + 1 && row <= r0 + Hs && J >= 1 && J <= nc - 1) {
#pragma unroll
            for (int k = 0; k < LC; ++k) {
              const int c = cA + k;
              if (!(c & 1) && c >= xlo && c < xhi) {
                const int I = c >> 1;
                if (I >= 1 && I <= nc - 1) {
                  const D2 s = cadd(cadd(west(v, k, vwl), cscale(2.0, v[k])), east(v, k, ver));
                  bounds_check((int64_t)shift * a.ssc + (int64_t)J * nc + I, a.elems_c, 6);
                  a.bc[(int64_t)shift * a.ssc + (int64_t)J * nc + I] = st2<V>(cscale(1.0 / 16.0, s));
                }
              }
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < LC; ++k) Vp[k] = make_double2(fma(2.0, r2[k].x, Vp[k].x), fma(2.0, r2[k].y, Vp[k].y));
        }
      }
    }
  };
  // Two loop shapes (measured per variant on B200, the prolongating passes prefer the first):
  //  (a) every step unrolled by 3 over the window phases, each with a masked and an unmasked copy;
  //  (b) boundary steps one at a time in window phase 0 followed by a register rotation, interior steps
  //      unmasked and unrolled by 3 -- only unmasked copies in the hot loop (smaller code).
  // (prolongating passes with a post stage: shape (a) only -- both shapes in one function spill)
  // Kernels with n compiled in (the hot variants) also fix the loop shape -- (a) for the prolongating passes, (b)
  // for the others, as measured -- and give edge strips their own interior copy (mask mode 2); the generic kernels
  // choose the shape at run time (a.loop_a) and run edge strips fully masked, to keep their code size down.
#ifndef PDMG_M2_EDGE_MODE
#define PDMG_M2_EDGE_MODE 2
#endif
#ifndef PDMG_M2_EDGE_UNROLL
#define PDMG_M2_EDGE_UNROLL 1
#endif
#ifndef PDMG_M2_PROLONG_B
#define PDMG_M2_PROLONG_B 1
#endif
  using MEdge = IC<(NF > 0 ? PDMG_M2_EDGE_MODE : 1)>;
  auto run_a = [&]() __attribute__((always_inline)) {
    auto run = [&](auto MI) __attribute__((always_inline)) {  // MI: mask mode of the steps with interior rows
      auto step_any = [&](int j, auto PH) __attribute__((always_inline)) {
        if (j >= jlo_int && j <= jhi_int) step(j, PH, MI);
        else step(j, PH, IC<1>{});
      };
      int j = rlo;
      for (; j + 2 < rhi; j += 3) {
        step_any(j, IC<0>{});
        step_any(j + 1, IC<1>{});
        step_any(j + 2, IC<2>{});
      }
      if (j < rhi) step_any(j, IC<0>{});
      if (j + 1 < rhi) step_any(j + 1, IC<1>{});
    };
    if constexpr (NF > 0) {
      if (col_int) run(IC<0>{});
      else run(MEdge{});
    } else {
      // generic kernels: ONE copy of the loop for interior and edge strips (two copies of this 29 KB loop live on
      // an SM at once overflow the 32 KB instruction cache: measured 93 -> 132 us per L2 pass at C3)
      auto step_any = [&](int j, auto PH) __attribute__((always_inline)) {
        if (col_int && j >= jlo_int && j <= jhi_int) step(j, PH, IC<0>{});
        else step(j, PH, IC<1>{});
      };
      int j = rlo;
      for (; j + 2 < rhi; j += 3) {
        step_any(j, IC<0>{});
        step_any(j + 1, IC<1>{});
        step_any(j + 2, IC<2>{});
      }
      if (j < rhi) step_any(j, IC<0>{});
      if (j + 1 < rhi) step_any(j + 1, IC<1>{});
    }
  };
  auto run_b = [&]() __attribute__((always_inline)) {
    auto rotate = [&]() __attribute__((always_inline)) {
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        U0[0][k] = U0[1][k], U0[1][k] = U0[2][k];
        U1[0][k] = U1[1][k], U1[1][k] = U1[2][k];
        U2[0][k] = U2[1][k], U2[1][k] = U2[2][k];
      }
    };
    // steps with interior rows: [jm_lo, jm_end) (generic kernels: none for an edge strip, which runs fully masked)
    const int jm_lo = (NF > 0 || col_int) ? max(rlo, jlo_int) : rhi;
    const int jm_end = (NF > 0 || col_int) ? max(jm_lo, min(jhi_int + 1, rhi)) : rhi;
    int j = rlo;
    for (; j < jm_lo; ++j) {  // leading boundary steps
      step(j, IC<0>{}, IC<1>{});
      rotate();
    }
    auto mid = [&](auto MI) __attribute__((always_inline)) {
      // (edge strips one step at a time unless PDMG_M2_EDGE_UNROLL: the interior strips' unrolled loop and the edge
      // strips' loop are live on an SM at the same time, and together they should fit the 32 KB instruction cache)
      if constexpr (decltype(MI)::value == 0 || PDMG_M2_EDGE_UNROLL) {
        for (; j + 2 < jm_end; j += 3) {
          step(j, IC<0>{}, MI);
          step(j + 1, IC<1>{}, MI);
          step(j + 2, IC<2>{}, MI);
        }
      }
      for (; j < jm_end; ++j) {
        step(j, IC<0>{}, MI);
        rotate();
      }
    };
    if constexpr (NF > 0) {
      if (col_int) mid(IC<0>{});
      else mid(MEdge{});
    } else {
      mid(IC<0>{});
    }
    for (; j < rhi; ++j) {  // trailing boundary steps
      step(j, IC<0>{}, IC<1>{});
      rotate();
    }
  };
  if constexpr (NF > 0) {
    if constexpr (PROLONG && !(PDMG_M2_PROLONG_B)) run_a();
    else run_b();
  } else {
    if (a.loop_a || (PROLONG && POST != POST_NONE)) run_a();
    else run_b();
  }
  if constexpr (POST == POST_NORM || NORM_IN) {
    for (int o = 16; o > 0; o >>= 1) nacc += __shfl_xor_sync(0xffffffffu, nacc, o);
    if (lane == 0) a.partial[(int64_t)shift * a.ntasks + task] = nacc;
  }
}

}  // namespace pdmg_b200
