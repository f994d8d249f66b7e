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

constexpr int TILE_W = 64;   // output columns per CTA
constexpr int CHUNK = 8;     // rows advanced per step
constexpr int RING = 16;     // rows held per stage ring (>= CHUNK + 2)
constexpr int NTHREADS = 256;

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

template <class T, int HALO>
struct Ring {
  using V = typename vec2<T>::type;
  static constexpr int WIDTH = TILE_W + 2 * HALO;
  V* p;
  int c_lo;  // storage column of local column 0
  __device__ __forceinline__ V& at(int row, int col) const { return p[(row & (RING - 1)) * WIDTH + (col - c_lo)]; }
};

// Shared-memory footprint (bytes) of a k_level instantiation.
template <class T, bool SWEEP, int POST>
struct LevelSmem {
  static constexpr bool HASD = POST != POST_NONE;
  static constexpr int hD = POST == POST_RESTRICT ? 1 : 0;
  static constexpr int hC = HASD ? hD + 1 : 0;
  static constexpr int hA = SWEEP ? hC + 2 : hC;
  static constexpr int hB = hA - 1;
  static constexpr int WA = TILE_W + 2 * hA, WB = TILE_W + 2 * hB, WC = TILE_W + 2 * hC, WD = TILE_W + 2 * hD;
  static constexpr size_t elems = (size_t)RING * (WA + (SWEEP ? WB : 0) + (SWEEP && HASD ? WB + WC : 0) +
                                                  (POST == POST_RESTRICT ? WD : 0));
  static constexpr size_t bytes = elems * sizeof(typename vec2<T>::type) + 64 * sizeof(double);
};

template <class T, bool LOADU, bool PROLONG, bool SWEEP, int POST, bool STORE, bool JACOBI>
__global__ void __launch_bounds__(NTHREADS) k_level(LevelArgs<T> a) {
  using V = typename vec2<T>::type;
  using SM = LevelSmem<T, SWEEP, POST>;
  constexpr bool HASD = SM::HASD;
  constexpr int hA = SM::hA, hB = SM::hB, hC = SM::hC, hD = SM::hD;
  constexpr int xD = SWEEP ? 3 : 1;  // stage index of D (A = 0, B = 1, C = 2)

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
  Ring<T, hA> RA{sm, c0 - hA};
  sm += RING * SM::WA;
  Ring<T, hB> RB{sm, c0 - hB};   // r = b - L u_in
  Ring<T, hB> RBb{sm, c0 - hB};  // b (kept for stage D)
  Ring<T, hC> RC{sm, c0 - hC};   // u_out
  if constexpr (SWEEP) {
    RB.p = sm;
    sm += RING * SM::WB;
    if constexpr (HASD) {
      RBb.p = sm;
      sm += RING * SM::WB;
      RC.p = sm;
      sm += RING * SM::WC;
    }
  }
  Ring<T, hD> RD{sm, c0 - hD};
  if constexpr (POST == POST_RESTRICT) sm += RING * SM::WD;
  double* red = reinterpret_cast<double*>(sm);

  LevelCoef<T> cf = a.coef[shift];
  const V* __restrict__ uin = a.u_in + sbase;
  const V* __restrict__ bb = a.b + sbase;
  V* __restrict__ uout = a.u_out + sbase;

  auto interior = [&](int row, int col) { return (unsigned)(row - 1) < (unsigned)m && (unsigned)(col - 1) < (unsigned)m; };
  auto in_out = [&](int row, int col) {
    return row >= r0 && row < r0 + H && col >= c0 && col < c0 + TILE_W && interior(row, col);
  };
  // b - (A + lambda I) u at (row, col) from a ring (grid.cpp:69-100 order: d*u_c - W - E - S - N).
  auto resid = [&](const auto& R, V bv, int row, int col) {
    V acc = cmul(cf.d, R.at(row, col));
    acc = csub(acc, R.at(row, col - 1));
    acc = csub(acc, R.at(row, col + 1));
    acc = csub(acc, R.at(row - 1, col));
    acc = csub(acc, R.at(row + 1, col));
    return csub(bv, cscale(cf.inv_h2, acc));
  };

  double nacc = 0.0;
  const int base = r0 - hA;
  const int n_iter = (H + 2 * hA + CHUNK - 1) / CHUNK;

  for (int t = 0; t < n_iter; ++t) {
    // ---------------- stage A: u_in --------------------------------------------------------
    {
      const int k0 = base + CHUNK * t;
      const int kend = min(k0 + CHUNK, r0 + H + hA);
      for (int idx = tid; idx < CHUNK * SM::WA; idx += NTHREADS) {
        const int row = k0 + idx / SM::WA;
        if (row >= kend) break;
        const int col = RA.c_lo + idx % SM::WA;
        V v = cz<V>();
        if (interior(row, col)) {
          if constexpr (LOADU) v = uin[(int64_t)row * n + col];
          if constexpr (PROLONG) {  // u += prolong_bilinear(e_c) (grid.cpp:123-153, multigrid.cpp:75)
            const V* __restrict__ e = a.ec + (int64_t)shift * a.ssc;
            const int nc = a.nc, I = col >> 1, J = row >> 1;
            const V* e0 = e + (int64_t)J * nc + I;
            V p;
            if (!(col & 1) && !(row & 1)) {
              p = e0[0];
            } else if ((col & 1) && !(row & 1)) {
              p = cscale((T)0.5, cadd(e0[0], e0[1]));
            } else if (!(col & 1) && (row & 1)) {
              p = cscale((T)0.5, cadd(e0[0], e0[nc]));
            } else {
              p = cscale((T)0.25, cadd(cadd(cadd(e0[0], e0[1]), e0[nc]), e0[nc + 1]));
            }
            v = cadd(v, p);
          }
        }
        RA.at(row, col) = v;
        if constexpr (!SWEEP && STORE) {
          if (in_out(row, col)) uout[(int64_t)row * n + col] = v;
        }
      }
    }
    __syncthreads();
    if constexpr (SWEEP) {
      // -------------- stage B: r = b - L u_in ---------------------------------------------
      {
        const int k0 = base + CHUNK * t - 1;
        const int klo = r0 - hB, khi = r0 + H + hB;
        for (int idx = tid; idx < CHUNK * SM::WB; idx += NTHREADS) {
          const int row = k0 + idx / SM::WB;
          if (row >= khi) break;
          if (row < klo) continue;
          const int col = RB.c_lo + idx % SM::WB;
          V r = cz<V>(), bv = cz<V>();
          if (interior(row, col)) {
            bv = bb[(int64_t)row * n + col];
            r = resid(RA, bv, row, col);
          }
          RB.at(row, col) = r;
          if constexpr (HASD) RBb.at(row, col) = bv;
        }
      }
      __syncthreads();
      // -------------- stage C: u_out = u_in + omega M r ----------------------------------
      {
        const int k0 = base + CHUNK * t - 2;
        const int klo = r0 - hC, khi = r0 + H + hC;
        constexpr int WCC = TILE_W + 2 * hC;
        for (int idx = tid; idx < CHUNK * WCC; idx += NTHREADS) {
          const int row = k0 + idx / WCC;
          if (row >= khi) break;
          if (row < klo) continue;
          const int col = c0 - hC + idx % WCC;
          V uo = cz<V>();
          if (interior(row, col)) {
            V mr;
            if constexpr (JACOBI) {
              mr = cmul(cf.k0, RB.at(row, col));
            } else {  // (h^2/4)[c,2b,c;2b,4a,2b;c,2b,c] r, omega folded into k (smoother.cpp:31-40, 62-64)
              const V e1 = cadd(cadd(cadd(RB.at(row - 1, col), RB.at(row, col - 1)), RB.at(row, col + 1)),
                                RB.at(row + 1, col));
              const V e2 = cadd(cadd(cadd(RB.at(row - 1, col - 1), RB.at(row - 1, col + 1)), RB.at(row + 1, col - 1)),
                                RB.at(row + 1, col + 1));
              mr = cadd(cadd(cmul(cf.k0, RB.at(row, col)), cmul(cf.k1, e1)), cmul(cf.k2, e2));
            }
            uo = cadd(RA.at(row, col), mr);
          }
          if constexpr (HASD) RC.at(row, col) = uo;
          if constexpr (STORE) {
            if (in_out(row, col)) uout[(int64_t)row * n + col] = uo;
          }
        }
      }
      __syncthreads();
    }
    if constexpr (HASD) {
      // -------------- stage D: r2 = b - L u_out ---------------------------------------------
      {
        const int k0 = base + CHUNK * t - xD;
        const int klo = r0 - hD, khi = r0 + H + hD;
        constexpr int WDD = TILE_W + 2 * hD;
        for (int idx = tid; idx < CHUNK * WDD; idx += NTHREADS) {
          const int row = k0 + idx / WDD;
          if (row >= khi) break;
          if (row < klo) continue;
          const int col = c0 - hD + idx % WDD;
          V r2 = cz<V>();
          if (interior(row, col)) {
            V bv;
            if constexpr (SWEEP) bv = RBb.at(row, col);
            else bv = bb[(int64_t)row * n + col];
            if constexpr (SWEEP) r2 = resid(RC, bv, row, col);
            else r2 = resid(RA, bv, row, col);
          }
          if constexpr (POST == POST_RESTRICT) RD.at(row, col) = r2;
          if constexpr (POST == POST_NORM) {
            if (in_out(row, col)) nacc += (double)r2.x * (double)r2.x + (double)r2.y * (double)r2.y;
          }
          if constexpr (POST == POST_RESID) {
            if (in_out(row, col)) uout[(int64_t)row * n + col] = r2;
          }
        }
      }
      if constexpr (POST == POST_RESTRICT) {
        __syncthreads();
        // ------------ stage E: b_c(I,J) = (1/16)[1 2 1;2 4 2;1 2 1] r2 at (2I,2J) -------------
        const int kcur = min(base - xD + CHUNK * (t + 1), r0 + H + hD);
        const int kprev = min(base - xD + CHUNK * t, r0 + H + hD);
        const int mc = a.nc - 1;
        int jlo = max(r0 >> 1, 1);
        if (t > 0) jlo = max(jlo, floordiv2(kprev - 2) + 1);
        const int jhi = min(min(floordiv2(kcur - 2), ((r0 + H) >> 1) - 1), mc);
        const int nj = jhi - jlo + 1;
        V* __restrict__ bco = a.bc + (int64_t)shift * a.ssc;
        for (int idx = tid; idx < nj * (TILE_W / 2); idx += NTHREADS) {
          const int J = jlo + idx / (TILE_W / 2);
          const int I = (c0 >> 1) + idx % (TILE_W / 2);
          if (I < 1 || I > mc) continue;
          const int i = 2 * I, j = 2 * J;
          V s = RD.at(j - 1, i - 1);
          s = cadd(s, cscale((T)2, RD.at(j - 1, i)));
          s = cadd(s, RD.at(j - 1, i + 1));
          s = cadd(s, cscale((T)2, RD.at(j, i - 1)));
          s = cadd(s, cscale((T)4, RD.at(j, i)));
          s = cadd(s, cscale((T)2, RD.at(j, i + 1)));
          s = cadd(s, RD.at(j + 1, i - 1));
          s = cadd(s, cscale((T)2, RD.at(j + 1, i)));
          s = cadd(s, RD.at(j + 1, i + 1));
          bco[(int64_t)J * a.nc + I] = cscale((T)(1.0 / 16.0), s);
        }
      }
    }
    __syncthreads();
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
