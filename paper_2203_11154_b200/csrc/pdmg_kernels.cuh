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
#include <cuda_runtime.h>
#include <stdint.h>

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

// Per (level, shift) operator coefficients, precomputed on the host in fp64 (multigrid.cpp:47-58).
template <class T>
struct LevelCoef {
  typename vec2<T>::type d;  // 4 + eta, eta = lambda h^2              (grid.cpp:73)
  typename vec2<T>::type k0; // Vanka: omega*(h^2/4)*4a ; Jacobi: omega*h^2/(4+eta)
  typename vec2<T>::type k1; // Vanka: omega*(h^2/4)*2b
  typename vec2<T>::type k2; // Vanka: omega*(h^2/4)*c
  T inv_h2;                  // 1/h^2
  T pad_;
};

enum : int { POST_NONE = 0, POST_NORM = 1, POST_RESTRICT = 2, POST_RESID = 3 };

constexpr int TILE_W = 64;    // output columns per CTA
constexpr int CHUNK = 16;     // rows each stage advances per step
constexpr int RING = 18;      // rows of the r / delta rings (= CHUNK + 2: a stage reads its producer's rows -1..CHUNK)
constexpr int RING_R = 20;    // ... when the restriction (which looks 2 more rows back) consumes them
constexpr int ARING = 34;     // rows of the u_in ring: the 18 rows in use + the next chunk landing (cp.async)
constexpr int RPT = 4;        // rows per stencil task (register-blocked along the column)
constexpr int RGROUPS = CHUNK / RPT;
constexpr int NTHREADS = 288; // 9 warps >= (TILE_W + 2*hB) * RGROUPS tasks for every variant
constexpr int CB_ROWS = 10, CB_COLS = 40;  // coarse block for prolongation (CHUNK/2 + 2 rows, (TILE_W+8)/2 + 4 cols)

template <class T>
struct LevelArgs {
  using V = typename vec2<T>::type;
  const V* u_in;             // level u (LOADU)
  V* u_out;                  // level u output (STORE) or residual output (POST_RESID)
  const V* b;                // level rhs
  const V* ec;               // coarse correction (PROLONG), coarse layout
  V* bc;                     // coarse rhs output (POST_RESTRICT), coarse layout
  double* partial;           // [shift][tile] partial sums of |r2|^2 (POST_NORM)
  const LevelCoef<T>* coef;  // [shift] at this level
  const int* active;         // [shift] convergence mask, or nullptr
  int n, nc;                 // fine / coarse subdivisions
  int64_t ss, ssc;           // shift strides (elements)
  int ntx, ntiles, H;        // tiles across, tiles per shift, strip height (even)
};

__device__ __forceinline__ int floordiv2(int a) { return a >> 1; }  // arithmetic shift = floor(a/2)

// 16-byte global->shared async copy; src_bytes = 0 zero-fills (used for every non-interior node, which
// is how the homogeneous Dirichlet boundary enters the stencil stages).
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int nbytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Circular row buffer: rows map to slots row mod NROWS (rows are >= -NROWS).
template <class T, int HALO, int NROWS>
struct Ring {
  using V = typename vec2<T>::type;
  static constexpr int WIDTH = TILE_W + 2 * HALO;
  V* p;
  int c_lo;  // storage column of local column 0
  __device__ __forceinline__ V* row_ptr(int row) const { return p + ((row + NROWS) % NROWS) * WIDTH - c_lo; }
  __device__ __forceinline__ V& at(int row, int col) const { return row_ptr(row)[col]; }
};

// Halo widths and shared-memory footprint of a k_level instantiation.
template <class T, bool USE_A, bool SWEEP, int POST, bool PROLONG>
struct LevelShape {
  static constexpr bool HASD = POST != POST_NONE;
  static constexpr int hD = POST == POST_RESTRICT ? 1 : 0;
  static constexpr int hC = HASD ? hD + 1 : 0;
  static constexpr int hA = SWEEP ? hC + 2 : hC;
  static constexpr int hB = hA - 1;
  static constexpr int WA = TILE_W + 2 * hA, WB = TILE_W + 2 * hB, WC = TILE_W + 2 * hC;
  static constexpr int RR = POST == POST_RESTRICT ? RING_R : RING;  // rows of the r / delta rings
  static constexpr size_t elems = (size_t)(USE_A ? ARING * WA : 0) + (SWEEP ? (CHUNK + RR) * WB : 0) +
                                  (SWEEP && HASD ? RR * WC : 0) + (PROLONG ? CB_ROWS * CB_COLS : 0);
  static constexpr size_t bytes = elems * sizeof(typename vec2<T>::type) + 16 * sizeof(double);
  // CTAs per SM the shared memory allows (227 KB usable); used as the register budget hint
  static constexpr int min_blocks = bytes <= 75 * 1024 ? 3 : 2;
  static_assert(!SWEEP || WB * RGROUPS <= NTHREADS, "stage-B tasks exceed the CTA");
  static_assert(bytes <= 113 * 1024, "two CTAs per SM must fit");
};

// Stage row ranges: stage x (A=0, B=1, C=2, D=3) handles, in step t, rows [base - x + CHUNK t, +CHUNK)
// clipped to [r0 - h_x, r0 + H + h_x), where base = r0 - hA.  Consecutive stages lag one row, so a
// stage only ever reads rows its producer finished in this step or the previous one.  The inputs of
// step t+1 (u rows, b rows, coarse block) are copied asynchronously while step t computes.
template <class T, bool LOADU, bool PROLONG, bool SWEEP, int POST, bool STORE, bool JACOBI>
__global__ void __launch_bounds__(NTHREADS, (LevelShape<T, LOADU || PROLONG || !SWEEP, SWEEP, POST, PROLONG>::min_blocks))
    k_level(LevelArgs<T> a) {
  using V = typename vec2<T>::type;
  constexpr bool USE_A = LOADU || PROLONG || !SWEEP;
  using SH = LevelShape<T, USE_A, SWEEP, POST, PROLONG>;
  constexpr bool HASD = SH::HASD;
  constexpr int hA = SH::hA, hB = SH::hB, hC = SH::hC, hD = SH::hD;
  constexpr int WA = SH::WA, WB = SH::WB, WC = SH::WC, RR = SH::RR;
  constexpr int xD = SWEEP ? 3 : 1;  // stage index of D

  const int shift = blockIdx.y;
  if (a.active != nullptr && a.active[shift] == 0) return;  // converged shifts are frozen
  const int tile = blockIdx.x;
  const int tx = tile % a.ntx, ty = tile / a.ntx;
  const int n = a.n, m = n - 1, H = a.H;
  const int c0 = tx * TILE_W, r0 = ty * H;
  const int tid = threadIdx.x;
  const int64_t sbase = (int64_t)shift * a.ss;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* sm = reinterpret_cast<V*>(smem_raw);
  Ring<T, hA, ARING> RA{sm, c0 - hA};  // u_in (+ P e_c)
  if constexpr (USE_A) sm += ARING * WA;
  V* Bb = sm;                           // b rows of the current B step, [CHUNK][WB]
  if constexpr (SWEEP) sm += CHUNK * WB;
  Ring<T, hB, RR> RB{sm, c0 - hB};     // r = b - L u_in
  if constexpr (SWEEP) sm += RR * WB;
  Ring<T, hC, RR> RC{sm, c0 - hC};     // delta = omega M r
  if constexpr (SWEEP && HASD) sm += RR * WC;
  V* CB = sm;                           // coarse block for the prolongation
  if constexpr (PROLONG) sm += CB_ROWS * CB_COLS;
  double* red = reinterpret_cast<double*>(sm);

  const LevelCoef<T> cf = a.coef[shift];
  const V* __restrict__ uin = a.u_in + sbase;
  const V* __restrict__ bb = a.b + sbase;
  V* __restrict__ uout = a.u_out + sbase;
  const V* __restrict__ ecs = a.ec + (int64_t)shift * a.ssc;
  const int nc = a.nc;

  auto interior = [&](int row, int col) { return (unsigned)(row - 1) < (unsigned)m && (unsigned)(col - 1) < (unsigned)m; };
  auto in_out = [&](int row, int col) {
    return row >= r0 && row < r0 + H && col >= c0 && col < c0 + TILE_W && interior(row, col);
  };
  const int base = r0 - hA;
  const int n_iter = (H + 2 * hA + CHUNK - 1) / CHUNK;

  // ---- asynchronous staging of a step's inputs ------------------------------------------------
  auto issue_A = [&](int t) {  // u rows of step t (zero outside the interior) and the coarse block
    if constexpr (USE_A) {
      const int k0 = base + CHUNK * t;
      for (int q = tid; q < CHUNK * WA; q += NTHREADS) {
        const int row = k0 + q / WA, col = c0 - hA + q % WA;
        if (row >= r0 + H + hA) break;
        V* dst = &RA.at(row, col);
        if constexpr (LOADU) {
          const bool ok = interior(row, col);
          cp_async16(dst, ok ? (const void*)(uin + (int64_t)row * n + col) : (const void*)uin, ok);
        } else {
          *dst = cz<V>();
        }
      }
      if constexpr (PROLONG) {
        const int J0 = floordiv2(k0), I0 = floordiv2(c0 - hA);
        for (int q = tid; q < CB_ROWS * CB_COLS; q += NTHREADS) {
          const int J = J0 + q / CB_COLS, I = I0 + q % CB_COLS;
          const bool ok = (unsigned)J <= (unsigned)nc && (unsigned)I <= (unsigned)nc;
          cp_async16(CB + q, ok ? (const void*)(ecs + (int64_t)J * nc + I) : (const void*)ecs, ok);
        }
      }
    }
  };
  auto issue_B = [&](int t) {  // b rows consumed by stage B in step t
    if constexpr (SWEEP) {
      const int k0 = base - 1 + CHUNK * t;
      for (int q = tid; q < CHUNK * WB; q += NTHREADS) {
        const int row = k0 + q / WB, col = c0 - hB + q % WB;
        const bool ok = row >= r0 - hB && row < r0 + H + hB && interior(row, col);
        cp_async16(Bb + q, ok ? (const void*)(bb + (int64_t)row * n + col) : (const void*)bb, ok);
      }
    }
  };
  // b - (A + lambda I) u at an interior node from ring values (grid.cpp:69-100: d*u_c - W - E - S - N)
  auto apply_res = [&](V bv, V uc, V uw, V ue, V us, V un) {
    V acc = cmul(cf.d, uc);
    acc = csub(acc, uw);
    acc = csub(acc, ue);
    acc = csub(acc, us);
    acc = csub(acc, un);
    return csub(bv, cscale(cf.inv_h2, acc));
  };

  double nacc = 0.0;
  issue_A(0);
  issue_B(0);
  cp_async_commit();

  for (int t = 0; t < n_iter; ++t) {
    cp_async_wait_all();
    __syncthreads();
    // ---------------- stage A: u_in = [u] + P e_c (in place on the landed rows) -----------------
    if constexpr (PROLONG) {  // u += prolong_bilinear(e_c) (grid.cpp:123-153, multigrid.cpp:75)
      const int k0 = base + CHUNK * t;
      const int J0 = floordiv2(k0), I0 = floordiv2(c0 - hA);
      for (int q = tid; q < CHUNK * WA; q += NTHREADS) {
        const int row = k0 + q / WA, col = c0 - hA + q % WA;
        if (row >= r0 + H + hA) break;
        V& slot = RA.at(row, col);
        V v = cz<V>();
        if (interior(row, col)) {
          const V* e0 = CB + (floordiv2(row) - J0) * CB_COLS + (floordiv2(col) - I0);
          V p;
          if (!(col & 1) && !(row & 1)) {
            p = e0[0];
          } else if ((col & 1) && !(row & 1)) {
            p = cscale((T)0.5, cadd(e0[0], e0[1]));
          } else if (!(col & 1) && (row & 1)) {
            p = cscale((T)0.5, cadd(e0[0], e0[CB_COLS]));
          } else {
            p = cscale((T)0.25, cadd(cadd(cadd(e0[0], e0[1]), e0[CB_COLS]), e0[CB_COLS + 1]));
          }
          v = p;
          if constexpr (LOADU) v = cadd(slot, p);
        }
        slot = v;
        if constexpr (!SWEEP && STORE) {
          if (in_out(row, col)) uout[(int64_t)row * n + col] = v;
        }
      }
      __syncthreads();
    }
    if constexpr (SWEEP) {
      if (t + 1 < n_iter) issue_A(t + 1);  // lands in ring rows no stage of step t touches
      cp_async_commit();
    }
    if constexpr (SWEEP) {
      // -------------- stage B: r = b - (A + lambda I) u_in  (grid.cpp:69-100) ---------------------
      {
        const int q = tid;
        if (q < WB * RGROUPS) {
          const int ci = q % WB, rg = q / WB;
          const int kb = base - 1 + CHUNK * t + RPT * rg, col = c0 - hB + ci;
          V am, ac, ap;  // rolling window of u_in down the column
          if constexpr (USE_A) {
            am = RA.at(kb - 1, col);
            ac = RA.at(kb, col);
          }
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            const int row = kb + i;
            if constexpr (USE_A) ap = RA.at(row + 1, col);
            if (row >= r0 - hB && row < r0 + H + hB) {
              V r = cz<V>();
              if (interior(row, col)) {
                const V bv = Bb[(RPT * rg + i) * WB + ci];
                if constexpr (USE_A) {
                  const V* rp = RA.row_ptr(row);
                  r = apply_res(bv, ac, rp[col - 1], rp[col + 1], am, ap);
                } else {
                  r = bv;  // zero initial guess: r = b
                }
              }
              RB.at(row, col) = r;
            }
            if constexpr (USE_A) am = ac, ac = ap;
          }
        }
      }
      __syncthreads();
      if (t + 1 < n_iter) issue_B(t + 1);
      cp_async_commit();
      // -------------- stage C: delta = omega M r; u_out = u_in + delta  (smoother.cpp:49-67) -------
      {
        const int q = tid;
        if (q < WC * RGROUPS) {
          const int ci = q % WC, rg = q / WC;
          const int kc = base - 2 + CHUNK * t + RPT * rg, col = c0 - hC + ci;
          // rolling 3-row window over the column: r and the horizontal pair sum r(col-1)+r(col+1)
          V rm, rc, rp, sm_, sc, sp;
          auto fetch = [&](int row, V& r_, V& s_) {
            const V* q_ = RB.row_ptr(row);
            r_ = q_[col];
            if constexpr (!JACOBI) s_ = cadd(q_[col - 1], q_[col + 1]);
          };
          fetch(kc - 1, rm, sm_);
          fetch(kc, rc, sc);
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            const int row = kc + i;
            fetch(row + 1, rp, sp);
            if (row >= r0 - hC && row < r0 + H + hC) {
              V dl = cz<V>();
              if (interior(row, col)) {
                if constexpr (JACOBI) {
                  dl = cmul(cf.k0, rc);
                } else {  // (h^2/4)[c,2b,c;2b,4a,2b;c,2b,c] r with omega folded in (smoother.cpp:31-40)
                  const V e1 = cadd(cadd(sc, rm), rp);
                  const V e2 = cadd(sm_, sp);
                  dl = cadd(cadd(cmul(cf.k0, rc), cmul(cf.k1, e1)), cmul(cf.k2, e2));
                }
              }
              if constexpr (HASD) RC.at(row, col) = dl;
              if constexpr (STORE) {
                if (in_out(row, col)) {
                  V uo = dl;
                  if constexpr (USE_A) uo = cadd(RA.at(row, col), dl);
                  uout[(int64_t)row * n + col] = uo;
                }
              }
            }
            rm = rc, sm_ = sc, rc = rp, sc = sp;
          }
        }
      }
      if constexpr (HASD) __syncthreads();
    }
    // -------------- stage D: r2 = b - (A + lambda I) u_out ---------------------------------------------
    // after a sweep r2 = r - (A + lambda I) delta (exact algebra; b is not read again)
    auto Urow = [&](int row) -> const V* {
      if constexpr (SWEEP) return RC.row_ptr(row);
      else return RA.row_ptr(row);
    };
    auto r2_at = [&](int row, int col, V uc, V um, V up) {  // uc/um/up: u_out (or delta) at rows row, row-1, row+1
      const V* rp = Urow(row);
      V rb;
      if constexpr (SWEEP) rb = RB.at(row, col);
      else rb = bb[(int64_t)row * n + col];
      return apply_res(rb, uc, rp[col - 1], rp[col + 1], um, up);
    };
    if constexpr (POST == POST_NORM || POST == POST_RESID) {
      const int q = tid;
      if (q < TILE_W * RGROUPS) {
        const int ci = q % TILE_W, rg = q / TILE_W;
        const int kd = base - xD + CHUNK * t + RPT * rg, col = c0 + ci;
        V dm = Urow(kd - 1)[col], dc = Urow(kd)[col], dp;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int row = kd + i;
          dp = Urow(row + 1)[col];
          if (in_out(row, col)) {
            const V r2 = r2_at(row, col, dc, dm, dp);
            if constexpr (POST == POST_NORM) nacc += (double)r2.x * (double)r2.x + (double)r2.y * (double)r2.y;
            if constexpr (POST == POST_RESID) uout[(int64_t)row * n + col] = r2;
          }
          dm = dc, dc = dp;
        }
      }
    }
    if constexpr (POST == POST_RESTRICT) {
      // ------------ stage D+E: b_c(I,J) = (1/16)[1 2 1;2 4 2;1 2 1] r2 around (2I,2J)  (grid.cpp:102-121)
      // one coarse node per thread; r2 is formed on the 3x3 fine block in registers (no r2 ring).
      const int kcur = min(base - xD + CHUNK * (t + 1), r0 + H + hD);
      const int kprev = min(base - xD + CHUNK * t, r0 + H + hD);
      const int mc = nc - 1;
      int jlo = max(r0 >> 1, 1);
      if (t > 0) jlo = max(jlo, floordiv2(kprev - 2) + 1);
      const int jhi = min(min(floordiv2(kcur - 2), ((r0 + H) >> 1) - 1), mc);
      V* __restrict__ bco = a.bc + (int64_t)shift * a.ssc;
      const int q = tid;
      if (q < (jhi - jlo + 1) * (TILE_W / 2)) {
        const int J = jlo + q / (TILE_W / 2);
        const int I = (c0 >> 1) + q % (TILE_W / 2);
        if (I >= 1 && I <= mc) {
          const int i = 2 * I, j = 2 * J;
          V s = cz<V>();
          V u_m[3], u_c[3], u_p[3];  // u (or delta) at rows j-2.., cols i-1..i+1, rolled down
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            u_m[c] = Urow(j - 2)[i - 1 + c];
            u_c[c] = Urow(j - 1)[i - 1 + c];
          }
#pragma unroll
          for (int rr = 0; rr < 3; ++rr) {
            const int row = j - 1 + rr;
#pragma unroll
            for (int c = 0; c < 3; ++c) u_p[c] = Urow(row + 1)[i - 1 + c];
            const T wr = rr == 1 ? (T)2 : (T)1;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const V r2 = r2_at(row, i - 1 + c, u_c[c], u_m[c], u_p[c]);
              const T w = wr * (c == 1 ? (T)2 : (T)1);
              s = cadd(s, cscale(w, r2));
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) u_m[c] = u_c[c], u_c[c] = u_p[c];
          }
          bco[(int64_t)J * nc + I] = cscale((T)(1.0 / 16.0), s);
        }
      }
    }
    if constexpr (!SWEEP) {  // D/E read u_in rows further back: refill only after they are done
      if (t + 1 < n_iter) {
        __syncthreads();
        issue_A(t + 1);
      }
      cp_async_commit();
    }
  }
  cp_async_wait_all();

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
};

__global__ void k_finalize(const double* __restrict__ partial, int ntiles, int k, SolveState st) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
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
}

// Per-shift norms (op-level pdmg_norm): sum partials -> sqrt.
__global__ void k_sum_partials(const double* __restrict__ partial, int ntiles, int S, double* out) {
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
                               const typename vec2<T>::type* __restrict__ ainv, const int* __restrict__ active,
                               int n, int64_t ss) {
  using V = typename vec2<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* sb = reinterpret_cast<V*>(smem_raw);
  const int s = blockIdx.x;
  if (active != nullptr && active[s] == 0) return;
  const int m = n - 1, N = m * m;
  const V* bs = b + (int64_t)s * ss;
  for (int q = threadIdx.x; q < N; q += blockDim.x) sb[q] = bs[(int64_t)(q / m + 1) * n + (q % m + 1)];
  __syncthreads();
  const V* A = ainv + (int64_t)s * N * N;
  V* us = u + (int64_t)s * ss;
  for (int r = threadIdx.x; r < N; r += blockDim.x) {
    V acc = cz<V>();
    for (int c = 0; c < N; ++c) acc = cadd(acc, cmul(A[(int64_t)r * N + c], sb[c]));
    us[(int64_t)(r / m + 1) * n + (r % m + 1)] = acc;
  }
}

// Compact (reference layout, [S][m][m]) <-> ghosted level storage.
template <class T>
__global__ void k_unpack(const typename vec2<T>::type* __restrict__ src, typename vec2<T>::type* __restrict__ dst,
                         int n, int64_t ss, int64_t total) {
  const int m = n - 1;
  const int64_t N = (int64_t)m * m;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = q / N, p = q % N;
    const int j = (int)(p / m) + 1, i = (int)(p % m) + 1;
    dst[s * ss + (int64_t)j * n + i] = src[q];
  }
}

// Gather u out of the double buffer each shift finished in: sel = parity[iterations[s]].
template <class T>
__global__ void k_pack(const typename vec2<T>::type* __restrict__ buf0, const typename vec2<T>::type* __restrict__ buf1,
                       const int* __restrict__ iters, const int* __restrict__ parity, typename vec2<T>::type* __restrict__ dst,
                       int n, int64_t ss, int64_t total) {
  const int m = n - 1;
  const int64_t N = (int64_t)m * m;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = q / N, p = q % N;
    const int j = (int)(p / m) + 1, i = (int)(p % m) + 1;
    const int sel = (iters == nullptr) ? 0 : parity[iters[s]];
    const typename vec2<T>::type* src = sel ? buf1 : buf0;
    dst[q] = src[s * ss + (int64_t)j * n + i];
  }
}

}  // namespace pdmg_b200
