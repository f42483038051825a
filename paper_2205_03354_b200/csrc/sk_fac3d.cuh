// Composed 73-point apply in FACTORED form (3D, periodic, sm_100a):
//
//   v = B u,  B = compose(L4, L4)   (stencil.cpp:75-87; laplacian(3, 4) is the
//                                    13-point fourth-order Laplacian,
//                                    generators.cpp:94-108)
//   w = L4 u ;  v = L4 w           (two fused radius-2 passes)
//
// On a periodic grid B u = L4 (L4 u) exactly in rational arithmetic, so this
// is the same operator as the literal 73-weight kernel (stream3d_kernel, R =
// 4) up to rounding: 2 x 13 instead of ~73 fp64 operations per point. The
// literal kernel is fp64-issue-bound at ~37% of the HBM roofline; this one
// moves the same 16 bytes per point with ~2.5x less arithmetic (see Status).
//
// Streaming along z per CTA over the balanced, rotated unit ranges of
// sk_stream3d.cuh (seg_of), input planes through the cp.async ring of
// PlaneLoader (tile + radius-4 halo, periodic wrap). Thread = 2 x 2 points of
// a 64 x TY tile (warp = row pair). Per input plane k:
//   w(k-2): own points from a 5-plane register queue of u (z +-1, +-2),
//           x- and y-neighbours from the ring (128-bit loads); the tile's 2-wide w border
//           (68 x (TY+4) minus the core) point-per-thread from the ring;
//           stored to a 3-slot w ring (read two planes later);
//   v(k-4): the same pattern on w (register queue + w ring) -> 128-bit stores.
// One __syncthreads per plane; the plane loop is unrolled by 5 so every
// queue role is static.
//
// Status: OPT-IN (SK_F73=1). Correct (tests/test_gpu_fac73.py) but measured
// at 113 us for 256^3 against 110.7 us for the literal 73-weight kernel: with
// 8 warps per SM (177 registers, 157 KB of ring + w slots) the kernel is
// latency-bound (ncu: issue 33%, fp64 pipe 22%, stalls wait 27% / short
// scoreboard 21%), so the 2.5x cut in arithmetic does not show. Tried: x
// neighbours by shuffles (133 us), 64x8 tiles at 2 CTAs/SM (125 us), own u
// re-read from the ring (126 us).
#pragma once

#include <type_traits>

#include "sk_stream3d.cuh"

namespace sk {

#ifndef SK_F73_TY
#define SK_F73_TY 16
#define SK_F73_S 8
#define SK_F73_MINB 1
#endif
#ifndef SK_F73_UREG
#define SK_F73_UREG 1  // 0: own u re-read from the ring (fewer registers; measured 126 vs 113 us)
#endif
using CfgFac73 = Cfg3<4, 64, SK_F73_TY, 2, 2, SK_F73_S, SK_F73_MINB>;

template <class C>
struct FacSmem {
  static constexpr int WP = C::TX + 8;                 // w slot pitch: x in [-2, TX+2) at column x + 2
  static constexpr int WROWS = C::TY + 4;              // y in [-2, TY+2)
  static constexpr int WPLANE = WROWS * WP;
  static constexpr int TAB = C::STAGES * C::PLANE + 3 * WPLANE;  // fallback loader's table (doubles from the ring)
  static constexpr int NB = 2 * (C::TX + 4) + 2 * C::TY;         // w border point PAIRS (x-aligned)
  static constexpr int BPT = (NB + C::THREADS - 1) / C::THREADS;  // border pairs per thread
  static constexpr int BYTES = C::RING_OFS + TAB * 8;
  static constexpr int BYTES_FB = BYTES + C::TABLE_BYTES;
};

// L4 at own points: a0 x + a1 s1 + a2 s2, s_d = ((x-d + x+d) + (y-d + y+d)) + (z-d + z+d)
struct L4W {
  double a0, a1, a2;
};

template <class C, bool FB>
__global__ void __launch_bounds__(C::THREADS, C::MIN_BLOCKS) fac73_kernel(const Args3D a, const L4W lw) {
  constexpr int R = 4, S = C::STAGES, P = C::PITCH, PLANE = C::PLANE;
  static_assert(C::R == 4 && C::PX == 2 && C::PY == 2 && C::TX == 64, "factored 73-point layout: warp = row pair");
  using SM = FacSmem<C>;
  constexpr int WP = SM::WP, WPLANE = SM::WPLANE;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw + C::RING_OFS);
  double* wring = ring + S * PLANE;

  const int units = a.tiles_x * a.tiles_y * int(a.nz);
  const int G = gridDim.x, b = blockIdx.x;
  const int per = units / G, rem = units % G;
  const int ubeg = b * per + (b < rem ? b : rem);
  const int uend = ubeg + per + (b < rem ? 1 : 0);
  LoadCursor<C, FB, SM::TAB> lc;
  lc.u = ubeg;
  lc.uend = uend;
  if (ubeg < uend) lc.start(a, ring);
  int s_load = 0;
#pragma unroll 1
  for (int k = 0; k < S - 5; ++k) {  // lookahead S - 5 planes (the ring holds planes k-4 .. k)
    lc.issue_next(ring, s_load, a);
    s_load = s_load + 1 == S ? 0 : s_load + 1;
  }

  const int lane = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int cofs = (2 * ty + R) * P + 2 * lane + R;  // own point (row 0, col 0) in a ring stage
  const int wofs = (2 * ty + 2) * WP + 2 * lane + 2;  // ... in a w slot
  // this thread's w border pairs (x even, two adjacent points): ring offset
  // of the left point, w slot offset
  int b_r[SM::BPT], b_w[SM::BPT];
#pragma unroll
  for (int j = 0; j < SM::BPT; ++j) {
    int i = threadIdx.x + j * C::THREADS, x = 0, y = 0;
    b_r[j] = -1;
    b_w[j] = 0;
    if (i < SM::NB) {
      constexpr int RW = (C::TX + 4) / 2;  // pairs per border row
      if (i < 2 * RW) {  // rows -2, -1
        y = i / RW - 2;
        x = 2 * (i % RW) - 2;
      } else if ((i -= 2 * RW) < 2 * RW) {  // rows TY, TY+1
        y = C::TY + i / RW;
        x = 2 * (i % RW) - 2;
      } else {  // pairs x = -2, -1 and TX, TX+1 of rows 0 .. TY-1
        i -= 2 * RW;
        y = i / 2;
        x = (i % 2) ? C::TX : -2;
      }
      b_r[j] = (y + R) * P + x + R;
      b_w[j] = (y + 2) * WP + x + 2;
    }
  }

#if SK_F73_UREG
  double U[5][4];  // own u of plane j in U[j % 5] (else re-read from the ring)
#endif
  double W[5][4];  // own w of plane j in W[j % 5]
  int s_k = 0;              // ring stage of u plane k
  int w_slot = 0;           // w slot written this plane; read: the one written two planes ago
  for (int u = ubeg; u < uend;) {
    const Seg sg = seg_of<C>(a, u, uend);
    u += sg.len;
    const int64_t gx0 = sg.x0 + 2 * lane, gy0 = sg.y0 + 2 * ty;
    const bool row0 = gy0 < a.ny, row1 = gy0 + 1 < a.ny;
    const bool vec_ok = gx0 + 2 <= a.nx;
    double* outp = a.v + int64_t(sg.z0) * a.nx * a.ny + gy0 * a.nx + gx0;
    const int np = sg.len + 2 * R;

    auto step = [&](auto kk_t, int k) {
      constexpr int K = decltype(kk_t)::value;  // k % 5
      constexpr int J0 = K, J1 = (K + 4) % 5, J2 = (K + 3) % 5, J3 = (K + 2) % 5, J4 = (K + 1) % 5;  // planes k .. k-4
      cp_async_wait_group<S - 6>();  // u plane k landed (this thread's copies) ...
      __syncthreads();               // ... everyone's; stage of plane k-5 free, w slot of plane k-3 complete
      lc.issue_next(ring, s_load, a);
      s_load = s_load + 1 == S ? 0 : s_load + 1;
      auto st = [&](int back) { return s_k >= back ? s_k - back : s_k - back + S; };
#if SK_F73_UREG
      {
        const double* cn = ring + s_k * PLANE + cofs;
        const double2 r0 = ld2(cn), r1 = ld2(cn + P);
        U[J0][0] = r0.x; U[J0][1] = r0.y; U[J0][2] = r1.x; U[J0][3] = r1.y;
      }
#endif
      double* wsl = wring + w_slot * WPLANE;                                  // w(k-2)
      const double* wrd = wring + (w_slot == 2 ? 0 : w_slot + 1) * WPLANE;  // w(k-4)

      // L4 at own points of plane X (z-neighbours Xm1, Xp1, Xm2, Xp2), in-plane
      // values from `src` (row pitch pitch, own point at ofs): edge lanes and
      // the rows above / below come from there
      auto l4_own = [&](const double* X, const double* Xm1, const double* Xp1, const double* Xm2,
                        const double* Xp2, const double* src, int pitch, int ofs, double* out) {
        // x-neighbours from `src` too (128-bit loads of the pairs x-2, x-1 and
        // x+2, x+3: fewer instructions than four 64-bit shuffles per row)
        const double* sp = src + ofs;
        double l0[2], l1[2], r0[2], r1[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double2 lp = ld2(sp + q * pitch - 2), rp = ld2(sp + q * pitch + 2);
          l0[q] = lp.x; l1[q] = lp.y; r0[q] = rp.x; r1[q] = rp.y;
        }
        const double2 ym2 = ld2(sp - 2 * pitch), ym1 = ld2(sp - pitch);
        const double2 yp2 = ld2(sp + 2 * pitch), yp3 = ld2(sp + 3 * pitch);
        // per point (q = row, c = column): x-1, x+1, x-2, x+2, y-1, y+1, y-2, y+2
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int i = 2 * q + c;
            const double xm1 = c == 0 ? l1[q] : X[2 * q];
            const double xp1 = c == 0 ? X[2 * q + 1] : r0[q];
            const double xm2 = c == 0 ? l0[q] : l1[q];
            const double xp2 = c == 0 ? r0[q] : r1[q];
            const double rowm1 = q == 0 ? (c == 0 ? ym1.x : ym1.y) : X[c];
            const double rowp1 = q == 0 ? X[2 + c] : (c == 0 ? yp2.x : yp2.y);
            const double rowm2 = q == 0 ? (c == 0 ? ym2.x : ym2.y) : (c == 0 ? ym1.x : ym1.y);
            const double rowp2 = q == 0 ? (c == 0 ? yp2.x : yp2.y) : (c == 0 ? yp3.x : yp3.y);
            const double s1 = ((xm1 + xp1) + (rowm1 + rowp1)) + (Xm1[i] + Xp1[i]);
            const double s2 = ((xm2 + xp2) + (rowm2 + rowp2)) + (Xm2[i] + Xp2[i]);
            out[i] = fma(lw.a2, s2, fma(lw.a1, s1, lw.a0 * X[i]));
          }
      };

      if (k >= 4) {  // w(k-2) on the core and the 2-wide border
        const double* rc = ring + st(2) * PLANE;
#if SK_F73_UREG
        l4_own(U[J2], U[J3], U[J1], U[J4], U[J0], rc, P, cofs, W[J2]);
#else
        // own u of planes k-4 .. k from the ring (it holds them for the border anyway)
        double uq[5][4];
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          const double* cn = ring + st(d) * PLANE + cofs;
          const double2 r0 = ld2(cn), r1 = ld2(cn + P);
          uq[d][0] = r0.x; uq[d][1] = r0.y; uq[d][2] = r1.x; uq[d][3] = r1.y;
        }
        l4_own(uq[2], uq[3], uq[1], uq[4], uq[0], rc, P, cofs, W[J2]);
#endif
        *reinterpret_cast<double2*>(wsl + wofs) = make_double2(W[J2][0], W[J2][1]);
        *reinterpret_cast<double2*>(wsl + wofs + WP) = make_double2(W[J2][2], W[J2][3]);
        const double* rm1 = ring + st(3) * PLANE;
        const double* rp1 = ring + st(1) * PLANE;
        const double* rm2 = ring + st(4) * PLANE;
        const double* rp2 = ring + s_k * PLANE;
#pragma unroll
        for (int j = 0; j < SM::BPT; ++j) {
          if (b_r[j] >= 0) {
            const int o = b_r[j];
            const double* c = rc + o;
            const double2 x0 = ld2(c), xl = ld2(c - 2), xr = ld2(c + 2);
            const double2 ym1 = ld2(c - P), yp1 = ld2(c + P), ym2 = ld2(c - 2 * P), yp2 = ld2(c + 2 * P);
            const double2 zm1 = ld2(rm1 + o), zp1 = ld2(rp1 + o), zm2 = ld2(rm2 + o), zp2 = ld2(rp2 + o);
            const double s1a = ((xl.y + x0.y) + (ym1.x + yp1.x)) + (zm1.x + zp1.x);
            const double s2a = ((xl.x + xr.x) + (ym2.x + yp2.x)) + (zm2.x + zp2.x);
            const double s1b = ((x0.x + xr.x) + (ym1.y + yp1.y)) + (zm1.y + zp1.y);
            const double s2b = ((xl.y + xr.y) + (ym2.y + yp2.y)) + (zm2.y + zp2.y);
            *reinterpret_cast<double2*>(wsl + b_w[j]) =
                make_double2(fma(lw.a2, s2a, fma(lw.a1, s1a, lw.a0 * x0.x)),
                             fma(lw.a2, s2b, fma(lw.a1, s1b, lw.a0 * x0.y)));
          }
        }
      }
      if (k >= 8) {  // v(k-4) = L4 w(k-4)
        double o[4];
        // centre w(k-4); z-1 w(k-5) (slot J0), z+1 w(k-3), z-2 w(k-6) (slot J1), z+2 w(k-2)
        l4_own(W[J4], W[J0], W[J3], W[J1], W[J2], wrd, WP, wofs, o);
        if (vec_ok) {
          if (row0) store_f64x2<Mode::Apply>(outp, o[0], o[1]);
          if (row1) store_f64x2<Mode::Apply>(outp + a.nx, o[2], o[3]);
        } else {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            if (row0 && gx0 + i < a.nx) outp[i] = o[i];
            if (row1 && gx0 + i < a.nx) outp[a.nx + i] = o[2 + i];
          }
        }
        outp += a.nx * a.ny;
      }
      s_k = s_k + 1 == S ? 0 : s_k + 1;
      w_slot = w_slot == 2 ? 0 : w_slot + 1;
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
}

}  // namespace sk
