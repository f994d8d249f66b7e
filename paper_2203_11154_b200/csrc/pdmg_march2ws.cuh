// pdmg_march2ws.cuh -- warp-specialised two-sweep Vanka pass (k_march2ws).
//
// Same arithmetic, lags and halos as k_march2 (pdmg_kernels.cuh), split over a PAIR of warps that share one
// 64-column strip:
//   warp A (producer): loads u_in / b rows, prolongate-and-correct, r = b - L u0 (+ ||r||^2 for NORM_IN),
//                      delta1 and u1 = u0 + delta1, and hands each u1 row to warp B through a shared-memory
//                      ring of WS_R rows (full/empty mbarriers, one arrival per lane);
//   warp B (consumer): r' = b - L u1, delta2, u2 = u1 + delta2 (stored), r2 = b - L u2 -> restriction / norm.
// Each warp carries only its own sweep's register windows (~half of k_march2's 244 registers), so twice as
// many warps are resident per SM: the k_march2 pass is issue/latency-bound (FP64 pipe 33 %, 8 warps/SM),
// and the extra warps hide the FP64 dependency chains and load latency.  Per step the hand-off costs each
// warp two 16-byte shared stores or loads per lane and one mbarrier arrive + wait.
#pragma once
#include "pdmg_kernels.cuh"

namespace pdmg_b200 {

#ifndef PDMG_WS_MINB
#define PDMG_WS_MINB 3
#endif
#ifndef PDMG_WS_PAIRS
#define PDMG_WS_PAIRS 2
#endif
constexpr int WS_R = 8;                 // u1 rows in flight between the two warps of a pair
constexpr int WS_PAIRS = PDMG_WS_PAIRS;  // warp pairs (strips) per CTA
constexpr int WS_THREADS = 64 * WS_PAIRS;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <class T, bool LOADU, bool PROLONG, int POST, bool NORM_IN = false>
__global__ void __launch_bounds__(WS_THREADS, PDMG_WS_MINB) k_march2ws(const __grid_constant__ MarchArgs<T> a, const __grid_constant__ CoefPack cp) {
  using V = typename vec2<T>::type;
  using D2 = double2;
  constexpr int LC = 2;
  constexpr bool EVEN = sizeof(V) == 8;
  constexpr bool HASD = POST != POST_NONE;
  constexpr int hD = POST == POST_RESTRICT ? 1 : 0;
  constexpr int hC = HASD ? hD + 1 : 0;
  constexpr int hA = (hC + 5) & ~1;  // = k_march2
  constexpr int WOUT = 32 * LC - 2 * hA;

  __shared__ __align__(16) D2 ring[WS_PAIRS][WS_R][32 * LC];
  __shared__ __align__(8) uint64_t bfull[WS_PAIRS][WS_R], bempty[WS_PAIRS][WS_R];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = wid >> 1;
  const bool producer = (wid & 1) == 0;
  if (threadIdx.x < WS_PAIRS * WS_R) {
    mbar_init(&bfull[0][0] + threadIdx.x, 32);
    mbar_init(&bempty[0][0] + threadIdx.x, 32);
  }
  __syncthreads();

  const int shift = cp.shift0 + blockIdx.y;
  if (a.active != nullptr && a.active[shift] == 0) return;
  const int task = blockIdx.x * WS_PAIRS + pair;
  if (task >= a.ntasks) return;  // both warps of the pair leave together
  const int tx = task % a.ntx, ty = task / a.ntx;
  const int n = a.n, m = n - 1, Hs = a.Hs, nc = a.nc;
  const int x0 = tx * WOUT, r0 = ty * Hs;
  const int64_t sbase = (int64_t)shift * a.ss;
  const int cA = x0 - hA + LC * lane;
  const LevelCoef cf = coef_of(cp);
  bool cin[LC], cst[LC];
#pragma unroll
  for (int k = 0; k < LC; ++k) {
    const int c = cA + k;
    cin[k] = (unsigned)(c - 1) < (unsigned)m;
    cst[k] = cin[k] && c >= x0 && c < x0 + WOUT;
  }
  const int rlo = r0 - hA, rhi = r0 + Hs + hA;
  const int olo = max(r0, 1), ohi = min(r0 + Hs, m + 1);
  auto row_in = [&](int row) __attribute__((always_inline)) { return (unsigned)(row - 1) < (unsigned)m; };
  auto row_ok = [&](int row) __attribute__((always_inline)) { return row_in(row) && row >= rlo; };
  const V* __restrict__ bb = a.b + sbase + cA;
  const bool col_int = (x0 - hA >= 1) && (x0 - hA + 32 * LC + 1 <= m - 1);
  const int jlo_int = max(6, rlo + 5), jhi_int = m - 3;
  D2* myring = &ring[pair][0][0];
  uint64_t* fullb = &bfull[pair][0];
  uint64_t* emptyb = &bempty[pair][0];

  auto gload_b = [&](int row, D2* out, auto MK) __attribute__((always_inline)) {
    constexpr bool MASK = decltype(MK)::value;
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      if constexpr (MASK)
        out[k] = (row_ok(row) && cin[k]) ? ld2(bb[(int64_t)row * n + k]) : cz<D2>();
      else
        out[k] = ld2(bb[(int64_t)row * n + k]);
    }
  };
  auto west = [&](const D2* x, int k, const D2& wl) __attribute__((always_inline)) { return k == 0 ? wl : x[k - 1]; };
  auto east = [&](const D2* x, int k, const D2& er) __attribute__((always_inline)) { return k == LC - 1 ? er : x[k + 1]; };
  auto resid = [&](const D2* lo, const D2* c, const D2* hi, const D2* bw, bool inside, D2* r, auto MK) __attribute__((always_inline)) {
    constexpr bool MASK = decltype(MK)::value;
    const D2 wl = shfl_up2(c[LC - 1]), er = shfl_dn2(c[0]);
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      const D2 v = res5(bw[k], cf.inv_h2, cf.dd, c[k], west(c, k, wl), east(c, k, er), lo[k], hi[k]);
      r[k] = MASK ? csel(inside && cin[k], v) : v;
    }
  };
  auto vanka_row = [&](const D2* r, D2* P, D2* C, bool din, D2* dl, auto MK) __attribute__((always_inline)) {
    constexpr bool MASK = decltype(MK)::value;
    const D2 rwl = shfl_up2(r[LC - 1]), rer = shfl_dn2(r[0]);
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      const D2 s = cadd(west(r, k, rwl), east(r, k, rer));
      const D2 c = cmad2(cf.k1, r[k], cf.k2, s);
      const D2 d = cmad2(cf.k0, r[k], cf.k1, s);
      const D2 v = cadd(P[k], c);
      dl[k] = MASK ? csel(din && cin[k], v) : v;
      P[k] = cadd(C[k], d);
      C[k] = c;
    }
  };
  // Loop shape: boundary steps one at a time (masked, window phase 0, then a register rotation) and the
  // interior steps unmasked and unrolled by 3 over the window phases, so the hot loop is only the three
  // unmasked step copies (instruction-cache footprint: the pass is fetch-bound with larger loop bodies).
  const int jm_lo = col_int ? max(rlo, jlo_int) : rhi;
  const int jm_end = col_int ? max(jm_lo, min(jhi_int + 1, rhi)) : rhi;
#define WS_LOOP(STEP, ROT)                                   \
  {                                                          \
    int j = rlo;                                             \
    for (; j < jm_lo; ++j) {                                 \
      STEP(j, IC<0>{}, IC<1>{});                             \
      ROT();                                                 \
    }                                                        \
    for (; j + 2 < jm_end; j += 3) {                         \
      STEP(j, IC<0>{}, IC<0>{});                             \
      STEP(j + 1, IC<1>{}, IC<0>{});                         \
      STEP(j + 2, IC<2>{}, IC<0>{});                         \
    }                                                        \
    for (; j < rhi; ++j) {                                   \
      if (j < jm_end) STEP(j, IC<0>{}, IC<0>{});             \
      else STEP(j, IC<0>{}, IC<1>{});                        \
      ROT();                                                 \
    }                                                        \
  }
  double nacc = 0.0;
  int q = 0;
  unsigned ph = 0;
  auto adv = [&]() __attribute__((always_inline)) {
    if (++q == WS_R) q = 0, ph ^= 1u;
  };

  if (producer) {
    // ================= warp A: u0 -> r -> delta1 -> u1 (ring) =================================================
    const V* __restrict__ uin = a.u_in + sbase + cA;
    const V* __restrict__ ecs = a.ec + (int64_t)shift * a.ssc;
    D2 Eo0 = cz<D2>(), Eo1 = cz<D2>(), Eo2 = cz<D2>(), Ex0 = cz<D2>(), Ex1 = cz<D2>(), Ex2 = cz<D2>();
    int wJ = -1000;
    const int Ie = cA >> 1;
    const bool codd = (cA & 1) != 0;
    auto load_crow = [&](int J, D2& o, D2& x, auto MK) __attribute__((always_inline)) {
      constexpr bool MASK = decltype(MK)::value;
      const bool jok = (unsigned)J <= (unsigned)nc;
      if constexpr (MASK)
        o = (jok && (unsigned)Ie <= (unsigned)nc) ? ld2(ecs[(int64_t)J * nc + Ie]) : cz<D2>();
      else
        o = ld2(ecs[(int64_t)J * nc + Ie]);
      if (lane == 31) x = (jok && (unsigned)(Ie + 1) <= (unsigned)nc) ? ld2(ecs[(int64_t)J * nc + Ie + 1]) : cz<D2>();
    };
    auto gread_u = [&](int row, D2* out, auto MK) __attribute__((always_inline)) {
      constexpr bool MASK = decltype(MK)::value;
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        out[k] = cz<D2>();
        if constexpr (LOADU) {
          if (!MASK || (row_ok(row) && cin[k])) out[k] = ld2(uin[(int64_t)row * n + k]);
        }
      }
    };
    auto prolong_row = [&](int row, D2* pout, auto MK) __attribute__((always_inline)) {
      constexpr bool MASK = decltype(MK)::value;
      const int J = row >> 1;
      if (J == wJ + 1) {
        Eo0 = Eo1, Eo1 = Eo2, Ex0 = Ex1, Ex1 = Ex2;
        load_crow(J + 2, Eo2, Ex2, MK);
        wJ = J;
      } else if (J != wJ) {
        load_crow(J, Eo0, Ex0, IC<1>{});
        load_crow(J + 1, Eo1, Ex1, IC<1>{});
        load_crow(J + 2, Eo2, Ex2, IC<1>{});
        wJ = J;
      }
      const D2 a0 = Eo0, b0 = Eo1;
      D2 a1 = shfl_dn2(Eo0), b1 = shfl_dn2(Eo1);
      if (lane == 31) a1 = Ex0, b1 = Ex1;
      const bool rin = !MASK || row_ok(row);
      D2 p[LC];
      if (row & 1) {  // prolong_bilinear (grid.cpp:123-153)
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

    D2 U0[3][LC], P1[LC], C1[LC], Pn[LC], Unx[LC], Bn[LC];
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      U0[0][k] = U0[1][k] = U0[2][k] = P1[k] = C1[k] = Pn[k] = cz<D2>();
    }
    gread_u(rlo, Unx, IC<1>{});
    gload_b(rlo - 1, Bn, IC<1>{});
    if constexpr (PROLONG) prolong_row(rlo, Pn, IC<1>{});
    int i = 0;  // steps done
    auto stepA = [&](int j, auto PH, auto MK) __attribute__((always_inline)) {
      constexpr int ph3 = decltype(PH)::value;
      constexpr int so = ph3 % 3, sm = (ph3 + 1) % 3, sn = (ph3 + 2) % 3;
      D2 Bc[LC];
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        U0[sn][k] = PROLONG ? cadd(Unx[k], Pn[k]) : Unx[k];
        Bc[k] = Bn[k];
      }
      if (!decltype(MK)::value || j + 1 < rhi) {  // (interior steps: row j+1 <= m-2 is always loadable)
        gread_u(j + 1, Unx, MK);
        if constexpr (PROLONG) prolong_row(j + 1, Pn, MK);
        gload_b(j, Bn, MK);
      }
      D2 r[LC], dl[LC], u1[LC];
      resid(U0[so], U0[sm], U0[sn], Bc, row_in(j - 1), r, MK);
      if constexpr (NORM_IN) {
        if (j - 1 >= olo && j - 1 < ohi) {
#pragma unroll
          for (int k = 0; k < LC; ++k)
            if (cst[k]) nacc += r[k].x * r[k].x + r[k].y * r[k].y;
        }
      }
      vanka_row(r, P1, C1, row_in(j - 2), dl, MK);
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        u1[k] = cadd(U0[so][k], dl[k]);
        if constexpr (EVEN) u1[k] = ld2(st2<V>(u1[k]));  // the iterate the unfused sweep would have stored
      }
      // hand u1 row j-2 to warp B
      if (i >= WS_R) mbar_wait(&emptyb[q], ph ^ 1u);
      D2* slot = myring + q * (32 * LC) + LC * lane;
#pragma unroll
      for (int k = 0; k < LC; ++k) slot[k] = u1[k];
      mbar_arrive(&fullb[q]);
      adv();
      ++i;
    };
    auto rotA = [&]() __attribute__((always_inline)) {
#pragma unroll
      for (int k = 0; k < LC; ++k) U0[0][k] = U0[1][k], U0[1][k] = U0[2][k];
    };
    WS_LOOP(stepA, rotA);
  } else {
    // ================= warp B: u1 (ring) -> r' -> delta2 -> u2 (stored) -> r2 -> restriction / norm ============
    V* __restrict__ uout = a.u_out + sbase + cA;
    D2 U1[3][LC], U2[3][LC], P2[LC], C2[LC], Vp[LC], B3n[LC], B5n[LC];
#pragma unroll
    for (int k = 0; k < LC; ++k) {
      U1[0][k] = U1[1][k] = U1[2][k] = U2[0][k] = U2[1][k] = U2[2][k] = cz<D2>();
      P2[k] = C2[k] = Vp[k] = cz<D2>();
    }
    gload_b(rlo - 3, B3n, IC<1>{});
    if constexpr (HASD) gload_b(rlo - 5, B5n, IC<1>{});
    auto stepB = [&](int j, auto PH, auto MK) __attribute__((always_inline)) {
      constexpr int ph3 = decltype(PH)::value;
      constexpr int so = ph3 % 3, sm = (ph3 + 1) % 3, sn = (ph3 + 2) % 3;
      D2 B3[LC], B5[LC];
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        B3[k] = B3n[k];
        if constexpr (HASD) B5[k] = B5n[k];
      }
      if (!decltype(MK)::value || j + 1 < rhi) {
        gload_b(j - 2, B3n, MK);
        if constexpr (HASD) gload_b(j - 4, B5n, MK);
      }
      mbar_wait(&fullb[q], ph);
      const D2* slot = myring + q * (32 * LC) + LC * lane;
#pragma unroll
      for (int k = 0; k < LC; ++k) U1[sn][k] = slot[k];
      mbar_arrive(&emptyb[q]);
      adv();
      {
        D2 r[LC], dl[LC];
        resid(U1[so], U1[sm], U1[sn], B3, row_in(j - 3), r, MK);
        const int row = j - 4;
        vanka_row(r, P2, C2, row_in(row), dl, MK);
        const bool rst = row >= olo && row < ohi;
#pragma unroll
        for (int k = 0; k < LC; ++k) {
          const V us = st2<V>(cadd(U1[so][k], dl[k]));
          if (rst && cst[k]) uout[(int64_t)row * n + k] = us;
          U2[sn][k] = ld2(us);
        }
      }
      if constexpr (HASD) {
        const int row = j - 5;
        D2 r2[LC];
        resid(U2[so], U2[sm], U2[sn], B5, row_in(row), r2, MK);
        if constexpr (POST == POST_NORM) {
          if (row >= olo && row < ohi) {
#pragma unroll
            for (int k = 0; k < LC; ++k)
              if (cst[k]) nacc += r2[k].x * r2[k].x + r2[k].y * r2[k].y;
          }
        }
        if constexpr (POST == POST_RESTRICT) {  // full weighting (grid.cpp:102-121)
          if (row & 1) {
            D2 v[LC];
#pragma unroll
            for (int k = 0; k < LC; ++k) {
              v[k] = cadd(Vp[k], r2[k]);
              Vp[k] = r2[k];
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
    };
    auto rotB = [&]() __attribute__((always_inline)) {
#pragma unroll
      for (int k = 0; k < LC; ++k) {
        U1[0][k] = U1[1][k], U1[1][k] = U1[2][k];
        U2[0][k] = U2[1][k], U2[1][k] = U2[2][k];
      }
    };
    WS_LOOP(stepB, rotB);
  }
  if constexpr (POST == POST_NORM || NORM_IN) {
    constexpr bool MINE_IS_A = NORM_IN;  // the pass's single norm: sweep 1's input residual (A) or r2 (B)
    if (producer == MINE_IS_A) {
      for (int o = 16; o > 0; o >>= 1) nacc += __shfl_xor_sync(0xffffffffu, nacc, o);
      if (lane == 0) a.partial[(int64_t)shift * a.ntasks + task] = nacc;
    }
  }
}

#undef WS_LOOP
}  // namespace pdmg_b200
