// pdmg_time_kernels.cuh -- sm_100a kernels of the ParaDIAG time direction (time DFT, dense time transform,
// all-at-once residuals).
//
// Layout: the all-at-once vectors are [nt][npts] time slices of the reference layout (paradiag.cpp:30-43 packs time
// slices as the rows of a dense matrix).  With the time slices sharded over devices, row r lives on shard
// r / rows at slot r % rows; a RowTab carries the shards' base pointers -- local or NVLink peer pointers -- so one
// kernel gathers the time column of its spatial points from every device, transforms it and scatters the
// result rows to their owners: the all-to-all of the time-direction transform is fused into the transform itself.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pdmg_kernels.cuh"

namespace pdmg_b200 {

constexpr int MAX_SHARDS = 16;
struct RowTab {
  double2* p[MAX_SHARDS];  // shard base pointers (device memory of the shard's GPU; peer-mapped if remote)
  int rows;                // rows per shard (the last shard may hold fewer)
  int64_t ld;              // elements per row
};
__device__ __forceinline__ double2* row_ptr(const RowTab& T, int r) {
  if (r < T.rows) return T.p[0] + (int64_t)r * T.ld;  // first (or only) shard: no division
  const int s = r / T.rows;
  return T.p[s] + (int64_t)(r - s * T.rows) * T.ld;
}

// ===================================================================================================
// alpha-scaled DFT over the time index (the alpha-circulant diagonalization; restated, DESIGN.md row P3):
//   step 1:  g_k = (1/nt) sum_t alpha^(t/nt) f_t e^{+2 pi i t k / nt}      (dir = +1, pre-scale, 1/nt)
//   step 3:  u_t = alpha^(-t/nt) sum_k w_k e^{-2 pi i t k / nt}           (dir = -1, post-scale)
// A CTA transforms P spatial points of [pt0, pt1): loads the nt rows (P contiguous complex each), runs an in-place
// radix-2 DIT FFT in shared memory when nt is a power of two (direct O(nt^2) DFT otherwise), writes rows k.
// tw[q] = e^{dir 2 pi i q / nt}; pre[t] multiplies the input, post[k] the output (complex: alpha^(t/nt) is
// complex for the QBV scheme's alpha < 0).
// ===================================================================================================
constexpr int DFT_THREADS = 256;

__global__ void __launch_bounds__(DFT_THREADS) k_time_dft(const RowTab in, const RowTab out, int nt, int log2nt,
                                                          int64_t pt0, int64_t pt1, int P,
                                                          const double2* __restrict__ tw,
                                                          const double2* __restrict__ pre,
                                                          const double2* __restrict__ post) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);  // [nt][P]
  const int64_t p0 = pt0 + (int64_t)blockIdx.x * P;
  const int np = (int)min((int64_t)P, pt1 - p0);
  const int tid = threadIdx.x;
  // (radix-2 path: nt and P are powers of two, so the index splits are shifts and masks, not divisions)
  const int lp = log2nt >= 0 ? 31 - __clz(P) : 0;
  // radix-2 path: the nt/2 twiddles the butterflies use sit in shared memory behind the data (a global load per
  // butterfly, even an L1 hit, stalled every one of them: 56 % of the kernel's stall samples)
  double2* stw = buf + (size_t)nt * P;
  if (log2nt >= 0)
    for (int q = tid; q < (nt >> 1); q += blockDim.x) stw[q] = tw[q];
  // load (bit-reversed time order for the radix-2 path), with the pre-scaling
#pragma unroll 4
  for (int q = tid; q < nt * P; q += blockDim.x) {
    const int t = log2nt >= 0 ? q >> lp : q / P, pl = q - t * P;
    double2 v = make_double2(0.0, 0.0);
    if (pl < np) v = cmul(pre[t], row_ptr(in, t)[p0 + pl]);
    const int dst = log2nt >= 0 ? (int)(__brev((unsigned)t) >> (32 - log2nt)) : t;
    buf[dst * P + pl] = v;
  }
  __syncthreads();
  if (log2nt >= 0) {
    // Two radix-2 stages per pass over shared memory (a thread carries four elements through both: the same
    // butterflies in the same order, half the shared-memory traffic and barriers); a last single stage if log2 nt
    // is odd.
    auto cmulw = [](double2 w, double2 b) { return make_double2(w.x * b.x - w.y * b.y, w.x * b.y + w.y * b.x); };
    int lh = 0;
    for (; lh + 1 < log2nt; lh += 2) {
      const int h = 1 << lh, t1 = nt >> (lh + 1), t2 = nt >> (lh + 2);
      for (int q = tid; q < (nt >> 2) * P; q += blockDim.x) {
        const int bf = q >> lp, pl = q & (P - 1);
        const int grp = bf >> lh, jj = bf & (h - 1);
        const int i0 = (grp * 4 * h + jj) * P + pl, st = h * P;
        const double2 w1 = stw[jj * t1], w2 = stw[jj * t2], w3 = stw[(jj + h) * t2];
        const double2 a = buf[i0], b = buf[i0 + st], c = buf[i0 + 2 * st], d = buf[i0 + 3 * st];
        const double2 wb = cmulw(w1, b), wd = cmulw(w1, d);
        const double2 a1 = make_double2(a.x + wb.x, a.y + wb.y), b1 = make_double2(a.x - wb.x, a.y - wb.y);
        const double2 c1 = make_double2(c.x + wd.x, c.y + wd.y), d1 = make_double2(c.x - wd.x, c.y - wd.y);
        const double2 wc = cmulw(w2, c1), we = cmulw(w3, d1);
        buf[i0] = make_double2(a1.x + wc.x, a1.y + wc.y);
        buf[i0 + 2 * st] = make_double2(a1.x - wc.x, a1.y - wc.y);
        buf[i0 + st] = make_double2(b1.x + we.x, b1.y + we.y);
        buf[i0 + 3 * st] = make_double2(b1.x - we.x, b1.y - we.y);
      }
      __syncthreads();
    }
    for (; lh < log2nt; ++lh) {
      const int half = 1 << lh, len = half << 1, tstep = nt >> (lh + 1);
      for (int q = tid; q < (nt >> 1) * P; q += blockDim.x) {
        const int bf = q >> lp, pl = q & (P - 1);
        const int grp = bf >> lh, jj = bf & (half - 1);
        const int i0 = grp * len + jj, i1 = i0 + half;
        const double2 w = stw[jj * tstep];
        const double2 a = buf[i0 * P + pl], b = buf[i1 * P + pl];
        const double2 wb = cmulw(w, b);
        buf[i0 * P + pl] = make_double2(a.x + wb.x, a.y + wb.y);
        buf[i1 * P + pl] = make_double2(a.x - wb.x, a.y - wb.y);
      }
      __syncthreads();
    }
#pragma unroll 4
    for (int q = tid; q < nt * P; q += blockDim.x) {
      const int k = q >> lp, pl = q & (P - 1);
      if (pl < np) row_ptr(out, k)[p0 + pl] = cmul(post[k], buf[k * P + pl]);
    }
  } else {
    for (int q = tid; q < nt * P; q += blockDim.x) {
      const int k = q / P, pl = q - k * P;
      if (pl >= np) continue;
      double2 acc = make_double2(0.0, 0.0);
      int idx = 0;  // (t * k) mod nt
      for (int t = 0; t < nt; ++t) {
        const double2 w = tw[idx], v = buf[t * P + pl];
        acc.x += w.x * v.x - w.y * v.y;
        acc.y += w.x * v.y + w.y * v.x;
        idx += k;
        if (idx >= nt) idx -= nt;
      }
      row_ptr(out, k)[p0 + pl] = cmul(post[k], acc);
    }
  }
}

// ===================================================================================================
// Dense time transform Y = (M (x) I) X over the time index (kron_time_apply / kron_time_solve,
// paradiag.cpp:129-139: the reference packs the slices as matrix rows and multiplies by V or solves with V's LU;
// here V^{-1} is formed once on the host and both directions are the same product).  Output rows [r0, r1) x
// points [pt0, pt1): Y[t][p] = sum_k M[t][k] X[k][p], complex fp64, output row t stored as row t - yoff of Y.  A CTA computes a GM_BM x GM_BN tile through
// shared-memory K panels of GM_BK; each thread holds GM_TM x GM_TN complex accumulators.  FP64 FMA-bound for
// nt >= 32 (8 nt flops per 32 B of X and Y); not a tensor-core shape (fp64, complex, K = nt small).
// ===================================================================================================
constexpr int GM_BM = 32, GM_BN = 64, GM_BK = 16, GM_TM = 4, GM_TN = 2, GM_THREADS = 256;
static_assert((GM_BM / GM_TM) * (GM_BN / GM_TN) == GM_THREADS, "thread tile layout");

__global__ void __launch_bounds__(GM_THREADS) k_time_gemm(const double2* __restrict__ M, int nt, const RowTab X,
                                                          const RowTab Y, int r0, int r1, int yoff, int64_t pt0,
                                                          int64_t pt1) {
  __shared__ double2 sM[GM_BK][GM_BM + 1];  // transposed panel: sM[k][t]
  __shared__ double2 sX[GM_BK][GM_BN];
  const int tid = threadIdx.x;
  const int tx = tid % (GM_BN / GM_TN), ty = tid / (GM_BN / GM_TN);
  const int tb = r0 + blockIdx.y * GM_BM;
  const int64_t pb = pt0 + (int64_t)blockIdx.x * GM_BN;
  double2 acc[GM_TM][GM_TN];
#pragma unroll
  for (int i = 0; i < GM_TM; ++i)
#pragma unroll
    for (int j = 0; j < GM_TN; ++j) acc[i][j] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < nt; k0 += GM_BK) {
    for (int q = tid; q < GM_BM * GM_BK; q += GM_THREADS) {  // M panel rows tb.., columns k0..
      const int i = q / GM_BK, kk = q - i * GM_BK;
      const int t = tb + i, k = k0 + kk;
      sM[kk][i] = (t < r1 && k < nt) ? M[(int64_t)t * nt + k] : make_double2(0.0, 0.0);
    }
    for (int q = tid; q < GM_BK * GM_BN; q += GM_THREADS) {  // X panel rows k0.., points pb..
      const int kk = q / GM_BN, j = q - kk * GM_BN;
      const int k = k0 + kk;
      const int64_t p = pb + j;
      sX[kk][j] = (k < nt && p < pt1) ? row_ptr(X, k)[p] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < GM_BK; ++kk) {
      double2 a[GM_TM], b[GM_TN];
#pragma unroll
      for (int i = 0; i < GM_TM; ++i) a[i] = sM[kk][ty * GM_TM + i];
#pragma unroll
      for (int j = 0; j < GM_TN; ++j) b[j] = sX[kk][tx + j * (GM_BN / GM_TN)];
#pragma unroll
      for (int i = 0; i < GM_TM; ++i)
#pragma unroll
        for (int j = 0; j < GM_TN; ++j) {
          acc[i][j].x = fma(a[i].x, b[j].x, fma(-a[i].y, b[j].y, acc[i][j].x));
          acc[i][j].y = fma(a[i].x, b[j].y, fma(a[i].y, b[j].x, acc[i][j].y));
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < GM_TM; ++i) {
    const int t = tb + ty * GM_TM + i;
    if (t >= r1) continue;
    double2* yr = row_ptr(Y, t - yoff);
#pragma unroll
    for (int j = 0; j < GM_TN; ++j) {
      const int64_t p = pb + tx + j * (GM_BN / GM_TN);
      if (p < pt1) yr[p] = acc[i][j];
    }
  }
}

// ===================================================================================================
// All-at-once residual r_t = f_t - ((C_alpha (x) I + I (x) A) u)_t over the local time slices [t0, t0+ntl) of a
// global nt (paradiag.cpp:141-183 with B = C_alpha): C_alpha row t couples u_t and u_{t-1} (1/dt, -1/dt), row 0
// couples u_0 and alpha u_{nt-1}.  u_prev is the slice before t0 (u_{nt-1} when t0 == 0; a peer pointer when it
// lives on another device).  Per-block partial sums of |r|^2 and |f|^2 (fixed order, deterministic).
// ===================================================================================================
__device__ __forceinline__ void block_sums2(double rr, double ff, double* __restrict__ partial) {
  __shared__ double red[2][32];
  for (int o = 16; o > 0; o >>= 1) {
    rr += __shfl_xor_sync(0xffffffffu, rr, o);
    ff += __shfl_xor_sync(0xffffffffu, ff, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[0][w] = rr, red[1][w] = ff;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    double a = l < nw ? red[0][l] : 0.0, b = l < nw ? red[1][l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (l == 0) partial[2 * blockIdx.x] = a, partial[2 * blockIdx.x + 1] = b;
  }
}

// unshifted 5-point A u at interior point p = (i, j) of a compact m x m slice (grid.cpp:69-90), times h^2
__device__ __forceinline__ double2 lap5_h2(const double2* __restrict__ ut, int p, int i, int j, int m) {
  const double2 c = ut[p];
  double ax = 4.0 * c.x, ay = 4.0 * c.y;
  if (i > 0) ax -= ut[p - 1].x, ay -= ut[p - 1].y;
  if (i < m - 1) ax -= ut[p + 1].x, ay -= ut[p + 1].y;
  if (j > 0) ax -= ut[p - m].x, ay -= ut[p - m].y;
  if (j < m - 1) ax -= ut[p + m].x, ay -= ut[p + m].y;
  return make_double2(ax, ay);
}

__global__ void k_aao_residual(const double2* __restrict__ u, const double2* __restrict__ u_prev,
                               const double2* __restrict__ f, int n, int ntl, int t0, double alpha, double dt,
                               double* __restrict__ partial) {
  const int m = n - 1, npts = m * m;
  const double h = 1.0 / n, inv_h2 = 1.0 / (h * h), idt = 1.0 / dt;
  double rr = 0.0, ff = 0.0;
  const int64_t total = (int64_t)ntl * npts;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int tl = (int)(q / npts), p = (int)(q - (int64_t)tl * npts);
    const int j = p / m, i = p - j * m;  // 0-based interior coords
    const double2* ut = u + (int64_t)tl * npts;
    const double2 c = ut[p];
    double2 a = lap5_h2(ut, p, i, j, m);
    double ax = a.x * inv_h2, ay = a.y * inv_h2;
    const double2 pv = tl > 0 ? u[(int64_t)(tl - 1) * npts + p] : u_prev[p];
    const double wp = (t0 + tl == 0) ? -alpha * idt : -idt;
    ax += idt * c.x + wp * pv.x;
    ay += idt * c.y + wp * pv.y;
    const double2 fv = f[(int64_t)tl * npts + p];
    const double rx = fv.x - ax, ry = fv.y - ay;
    rr += rx * rx + ry * ry;
    ff += fv.x * fv.x + fv.y * fv.y;
  }
  block_sums2(rr, ff, partial);
}

// General (dense) time matrix B (HeatBVM, paradiag.cpp:46-82): r = f - Y - (I (x) A) u over local slices, with
// Y = (B (x) I) u restricted to those slices precomputed by k_time_gemm.
__global__ void k_aao_residual_dense(const double2* __restrict__ u, const double2* __restrict__ y,
                                     const double2* __restrict__ f, int n, int ntl, double* __restrict__ partial) {
  const int m = n - 1, npts = m * m;
  const double h = 1.0 / n, inv_h2 = 1.0 / (h * h);
  double rr = 0.0, ff = 0.0;
  const int64_t total = (int64_t)ntl * npts;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(q / npts), p = (int)(q - (int64_t)t * npts);
    const int j = p / m, i = p - j * m;
    const double2 a = lap5_h2(u + (int64_t)t * npts, p, i, j, m);
    const double2 yv = y[q], fv = f[q];
    const double rx = fv.x - (inv_h2 * a.x + yv.x), ry = fv.y - (inv_h2 * a.y + yv.y);
    rr += rx * rx + ry * ry;
    ff += fv.x * fv.x + fv.y * fv.y;
  }
  block_sums2(rr, ff, partial);
}

}  // namespace pdmg_b200
