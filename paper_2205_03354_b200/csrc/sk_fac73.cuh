// Composed 73-point apply in FACTORED form, v2 (3D, periodic, sm_100a).
//
//   v = B u,  B = compose(L4, L4)   (stencil.cpp:75-87; L4 = laplacian(3, 4),
//                                    the 13-point fourth-order Laplacian,
//                                    generators.cpp:94-108)
//   w = L4 u ;  v = L4 w           (two fused radius-2 passes)
//
// On a periodic grid B u = L4 (L4 u) exactly in rational arithmetic: the
// same operator as the literal 73-weight kernel (stream3d_kernel, R = 4) up to
// rounding, with ~30 instead of ~49 fp64 operations per point and, more
// important on this chip, about half the shared-memory traffic per point
// (the literal kernel reads a 10 x 10 window per 2 x 2 points and is
// shared-bandwidth-bound).
//
// Layout: one CTA of 8 warps per SM (tile 64 x 16, warp = row pair, lane =
// 2 x 2 points; the 5-plane u and w queues take ~100 registers), streamed along z over the
// balanced rotated unit ranges of sk_stream3d.cuh (seg_of). u planes land
// through the 16-byte cp.async ring of PlaneLoader (radius-4 halo, periodic
// wrap); each thread signals its copies on the stage's FULL mbarrier
// (cp.async.mbarrier.arrive.noinc), so there is no CTA barrier for data.
// Per input plane k (all roles static: the loop is unrolled by 5):
//   w(k-2) at the thread's 4 core points: z-neighbours from a 5-plane
//          register queue of own u, in-plane neighbours from stage k-2;
//          at the thread's (at most one) x-pair of the 2-wide w border:
//          the same with a 5-plane register queue of that pair's u. No other
//          stage than k-2 and k is read, so only three stages are live.
//          w goes to a 4-slot ring (tile + border).
//   v(k-4) at the 4 core points: z from a 5-plane register queue of own w,
//          in-plane from the w slot of plane k-4 -> 128-bit stores.
// Synchronisation: a split-phase step barrier (per-warp mbarrier arrival
// after the w writes, wait one step later before the next w write / stage
// refill). Four w slots make the v reads (after the arrival) safe: a slot is
// rewritten only after every warp has passed the step that read it.
#pragma once

#include <type_traits>

#include "sk_stream3d.cuh"

namespace sk {

#ifndef SK_F2_TY
// 64 x 16 tiles, 8 stages, one 8-warp CTA per SM (212 registers, no spills):
// 90.2 us at 256^3 against 99.4 us for the literal kernel. 64 x 32 tiles with
// 16 warps need <= 128 registers and spill the 5-plane queues (179 us).
// (Border pairs reading their z-neighbours from 5 live stages instead of a
// register queue: 166 registers, 12 warps/SM with 64 x 24 tiles, 94.4 vs
// 93.6 us -- the kernel is bound by its shared traffic; experiment removed.)
#define SK_F2_TY 16
#define SK_F2_S 8
#endif
using CfgF2 = Cfg3<4, 64, SK_F2_TY, 2, 2, SK_F2_S, 1>;

struct L4W {
  double a0, a1, a2;  // centre (3 axes), axis +-1, axis +-2 weights of L4, scaled by h^-2
};

template <class C>
struct F2Smem {
  static constexpr int WSLOTS = 4;
  static constexpr int WP = C::TX + 4;   // w slot pitch: x in [-2, TX+2) at column x + 2
  static constexpr int WROWS = C::TY + 4;  // y in [-2, TY+2)
  static constexpr int WPLANE = WROWS * WP;
  static constexpr int NB = 2 * (C::TX + 4) + 2 * C::TY;  // w border x-pairs
  static constexpr int BAR_OFS = 0;                        // S full + 3 step barriers (first 128 B)
  static constexpr int BYTES = C::RING_OFS + (C::STAGES * C::PLANE + WSLOTS * WPLANE) * 8;
  static_assert(NB <= C::THREADS, "one w border pair per thread at most");
  static_assert((C::STAGES + 3) * 8 <= C::RING_OFS, "barriers before the ring");
  static_assert(WP % 2 == 0, "16-byte w rows");
};

// L4 at a pair of points (x, x+1) of one row: centre pair c, left pair
// (x-2, x-1), right pair (x+2, x+3), the pairs of rows y-1, y+1, y-2, y+2 and
// the z-neighbour pairs; s_d = ((x +- d) + (y +- d)) + (z +- d).
__device__ __forceinline__ double2 l4_pair(const L4W& lw, double2 c, double2 l, double2 r, double2 ym1, double2 yp1,
                                           double2 ym2, double2 yp2, double2 zm1, double2 zp1, double2 zm2,
                                           double2 zp2) {
  const double s1a = ((l.y + c.y) + (ym1.x + yp1.x)) + (zm1.x + zp1.x);
  const double s2a = ((l.x + r.x) + (ym2.x + yp2.x)) + (zm2.x + zp2.x);
  const double s1b = ((c.x + r.x) + (ym1.y + yp1.y)) + (zm1.y + zp1.y);
  const double s2b = ((l.y + r.y) + (ym2.y + yp2.y)) + (zm2.y + zp2.y);
  return make_double2(fma(lw.a2, s2a, fma(lw.a1, s1a, lw.a0 * c.x)), fma(lw.a2, s2b, fma(lw.a1, s1b, lw.a0 * c.y)));
}

// PQ (matrix-free CG on the ghost-padded p, sk_cg.cu): q = A p with p.q
// reduced in the store epilogue from the register queue (u(k-4) is p at the
// output point) and alpha published by the last CTA; the separate p.q pass
// disappears. A no-op once the solver has stopped.
template <class C, bool PQ = false>
__global__ void __launch_bounds__(C::THREADS, 1) fac73v2_kernel(const Args3D a, const L4W lw) {
  constexpr int R = 4, S = C::STAGES, P = C::PITCH, PLANE = C::PLANE;
  if constexpr (PQ) {
    if (a.cg->status != kCgRunning) return;
  }
  double pq = 0.0;
  (void)pq;
  static_assert(C::R == 4 && C::PX == 2 && C::PY == 2 && C::TX == 64, "layout: warp = row pair");
  using SM = F2Smem<C>;
  constexpr int WP = SM::WP, WPLANE = SM::WPLANE, WS = SM::WSLOTS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + SM::BAR_OFS);
  uint64_t* stepbar = full + S;
  double* ring = reinterpret_cast<double*>(smem_raw + C::RING_OFS);
  double* wring = ring + S * PLANE;

  const int units = a.tiles_x * a.tiles_y * int(a.nz);
  const int G = gridDim.x, b = blockIdx.x;
  const int per = units / G, rem = units % G;
  const int ubeg = b * per + (b < rem ? b : rem);
  const int uend = ubeg + per + (b < rem ? 1 : 0);
  const int lane = threadIdx.x % 32, ty = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&full[i], C::THREADS);
    for (int i = 0; i < 3; ++i) mbar_init(&stepbar[i], C::THREADS / 32);
    fence_mbar_init();
  }
  __syncthreads();
  LoadCursor<C, false> lc;
  lc.u = ubeg;
  lc.uend = uend;
  if (ubeg < uend) lc.start(a, ring);
  int s_load = 0;
  auto issue = [&]() {  // next plane into stage s_load; this thread's arrival on its FULL barrier
    if (lc.u < lc.uend) {
      lc.issue_next(ring, s_load, a);
      cp_async_arrive_noinc(&full[s_load]);
    }
    s_load = s_load + 1 == S ? 0 : s_load + 1;
  };
  constexpr int LIVE = 3;  // stages read per step: k-2 .. k
  for (int k = 0; k < S - LIVE; ++k) issue();  // lookahead S - LIVE planes

  const int cofs = (2 * ty + R) * P + 2 * lane + R;    // own point (row 0, col 0) in a u stage
  const int wofs = (2 * ty + 2) * WP + 2 * lane + 2;   // ... in a w slot
  // this thread's w border pair (x even): u stage offset of its left point, w slot offset
  int b_r = -1, b_w = 0;
  {
    int i = threadIdx.x, x = 0, y = 0;
    if (i < SM::NB) {
      constexpr int RW = (C::TX + 4) / 2;  // pairs per border row
      if (i < 2 * RW) {
        y = i / RW - 2;
        x = 2 * (i % RW) - 2;
      } else if ((i -= 2 * RW) < 2 * RW) {
        y = C::TY + i / RW;
        x = 2 * (i % RW) - 2;
      } else {
        i -= 2 * RW;
        y = i / 2;
        x = (i % 2) ? C::TX : -2;
      }
      b_r = (y + R) * P + x + R;
      b_w = (y + 2) * WP + x + 2;
    }
  }
  const bool has_b = b_r >= 0;
  if (!has_b) b_r = cofs;  // harmless in-range offset (loads unused)

  double2 U[5][2], W[5][2];  // own u / w of plane j in [j % 5]: row 0 pair, row 1 pair
  double2 UB[5];             // the border pair's u of plane j
  int s_k = 0;               // stage of u plane k
  uint32_t fph = 0;          // parity of the current use of stage s_k
  int w_slot = 0;            // w slot of plane k-2 (written this step); plane k-4: w_slot - 2 (mod 4)
  int sb = 0;                // step barrier t % 3
  uint32_t sph = 0;          // (t / 3) & 1
  bool started = false;      // t > 0

  for (int u = ubeg; u < uend;) {
    const Seg sg = seg_of<C>(a, u, uend);
    u += sg.len;
    const int64_t gx0 = sg.x0 + 2 * lane, gy0 = sg.y0 + 2 * ty;
    const bool row0 = gy0 < a.ny, row1 = gy0 + 1 < a.ny;
    const bool vec_ok = !(a.nx & 1) && gx0 + 2 <= a.nx;  // 16-byte stores: even rows (a padded input may be odd)
    double* outp = a.v + int64_t(sg.z0) * a.nx * a.ny + gy0 * a.nx + gx0;
    const int np = sg.len + 2 * R;

    auto step = [&](auto kk_t, int k) {
      constexpr int K = decltype(kk_t)::value;  // k % 5
      constexpr int J0 = K, J1 = (K + 4) % 5, J2 = (K + 3) % 5, J3 = (K + 2) % 5, J4 = (K + 1) % 5;  // k .. k-4
      mbar_wait(&full[s_k], fph);  // u plane k landed (every thread's copies)
      sk_jitter(50);
      {
        const double* cn = ring + s_k * PLANE;
        U[J0][0] = ld2(cn + cofs);
        U[J0][1] = ld2(cn + cofs + P);
        UB[J0] = ld2(cn + b_r);
      }
      const int s_k2 = s_k >= 2 ? s_k - 2 : s_k - 2 + S;  // stage of plane k-2
      // all warps past step t-1: the stage of plane k-3 and the w slot written below are free
      if (started) mbar_wait(&stepbar[sb == 0 ? 2 : sb - 1], sb == 0 ? sph ^ 1u : sph);
      sk_jitter(51);
      issue();  // plane k + S - LIVE into the stage of plane k - LIVE (last read at step t-1)
      double* wsl = wring + w_slot * WPLANE;
      if (k >= 4) {  // w(k-2)
        const double* rc = ring + s_k2 * PLANE;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double* c = rc + cofs + q * P;
          const double2 l = ld2(c - 2), r = ld2(c + 2);
          const double2 ym1 = q == 0 ? ld2(c - P) : U[J2][0];
          const double2 yp1 = q == 0 ? U[J2][1] : ld2(c + P);
          const double2 ym2 = ld2(c - 2 * P), yp2 = ld2(c + 2 * P);
          W[J2][q] = l4_pair(lw, U[J2][q], l, r, ym1, yp1, ym2, yp2, U[J3][q], U[J1][q], U[J4][q], U[J0][q]);
        }
        *reinterpret_cast<double2*>(wsl + wofs) = W[J2][0];
        *reinterpret_cast<double2*>(wsl + wofs + WP) = W[J2][1];
        if (has_b) {
          const double* c = rc + b_r;
          const double2 wb = l4_pair(lw, UB[J2], ld2(c - 2), ld2(c + 2), ld2(c - P), ld2(c + P), ld2(c - 2 * P),
                                     ld2(c + 2 * P), UB[J3], UB[J1], UB[J4], UB[J0]);
          *reinterpret_cast<double2*>(wsl + b_w) = wb;
        }
      }
      sk_jitter(52);
      __syncwarp();
      if (lane == 0) mbar_arrive(&stepbar[sb]);  // this warp's w of plane k-2 is in the slot
      started = true;
      if (++sb == 3) {
        sb = 0;
        sph ^= 1u;
      }
      if (k >= 8) {  // v(k-4) = L4 w(k-4): written two steps ago (this warp waited for that step's arrivals)
        const double* wr = wring + (w_slot >= 2 ? w_slot - 2 : w_slot + 2) * WPLANE;
        double2 o[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double* c = wr + wofs + q * WP;
          const double2 l = ld2(c - 2), r = ld2(c + 2);
          const double2 ym1 = q == 0 ? ld2(c - WP) : W[J4][0];
          const double2 yp1 = q == 0 ? W[J4][1] : ld2(c + WP);
          const double2 ym2 = ld2(c - 2 * WP), yp2 = ld2(c + 2 * WP);
          // centre w(k-4) (J4); z-1 w(k-5) (J0), z+1 w(k-3) (J3), z-2 w(k-6) (J1), z+2 w(k-2) (J2)
          o[q] = l4_pair(lw, W[J4][q], l, r, ym1, yp1, ym2, yp2, W[J0][q], W[J3][q], W[J1][q], W[J2][q]);
        }
        if (vec_ok) {
          if (row0) store_f64x2<Mode::Apply>(outp, o[0].x, o[0].y);
          if (row1) store_f64x2<Mode::Apply>(outp + a.nx, o[1].x, o[1].y);
        } else if (gx0 < a.nx) {  // odd rows (ghost-padded input): scalar stores
          const bool x1 = gx0 + 1 < a.nx;
          if (row0) {
            outp[0] = o[0].x;
            if (x1) outp[1] = o[0].y;
          }
          if (row1) {
            outp[a.nx] = o[1].x;
            if (x1) outp[a.nx + 1] = o[1].y;
          }
        }
        if constexpr (PQ) {  // p at the output points: the centre of u plane k-4 (J4)
          const bool x0ok = gx0 < a.nx, x1ok = gx0 + 1 < a.nx;
          if (row0) {
            if (x0ok) pq = fma(U[J4][0].x, o[0].x, pq);
            if (x1ok) pq = fma(U[J4][0].y, o[0].y, pq);
          }
          if (row1) {
            if (x0ok) pq = fma(U[J4][1].x, o[1].x, pq);
            if (x1ok) pq = fma(U[J4][1].y, o[1].y, pq);
          }
        }
        outp += a.nx * a.ny;
      }
      if (++s_k == S) {
        s_k = 0;
        fph ^= 1u;
      }
      w_slot = w_slot + 1 == WS ? 0 : w_slot + 1;
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    using I4 = std::integral_constant<int, 4>;
#pragma unroll 1
    for (int k = 0; k < np; k += 5) {
      step(I0{}, k);
      if (k + 1 < np) step(I1{}, k + 1);
      if (k + 2 < np) step(I2{}, k + 2);
      if (k + 3 < np) step(I3{}, k + 3);
      if (k + 4 < np) step(I4{}, k + 4);
    }
  }
  cp_async_wait_all();
  if constexpr (PQ) {
    __shared__ double sh[32];
    pq = block_sum<C::THREADS>(pq, sh);
    if (threadIdx.x == 0) a.cg_partials[blockIdx.x] = pq;
    if (last_block(&a.cg->counter[0])) {
      const double t = reduce_partials<C::THREADS>(a.cg_partials, gridDim.x, sh);
      if (threadIdx.x == 0) cg_publish_pq(a.cg, t);
    }
  }
}

}  // namespace sk
