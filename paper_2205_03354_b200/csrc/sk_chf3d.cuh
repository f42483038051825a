// Fused explicit Cahn-Hilliard step in FACTORED form (3D, sm_100a):
//
//   mu = f'(c) - kappa L c          (chemical potential, 7-point L)
//   c' = c + dt M L mu              (= c + dt M (L f'(c) - kappa L(L c)))
//
// L(L c) is exactly the composed 25-point operator B c (B = compose(L, L),
// stencil.cpp:75-87), so this is the same step as the composed kernel in
// sk_stream3d.cuh up to rounding, with ~19 instead of ~37 fp64 operations per
// point. It is the north-star form Delta(u^3 - u - eps^2 Delta u) fused into
// one pass.
//
// Streaming along z (per CTA: one 64 x 16 column tile over a z-range, the
// unit schedule of sk_stream3d.cuh). Each warp owns a row pair of the tile,
// each lane 2 x 2 points, and keeps its own points of c (planes k, k-1, k-2)
// and mu (planes k-1, k-2, k-3) in registers:
//   step k : c-plane k has landed (multistage cp.async ring, S stages)
//            -> own c of plane k: two 128-bit shared loads
//            -> mu of plane k-1: x-neighbours by warp shuffles (edge lanes
//               read the halo), y-neighbours from the ring (the rows of the
//               adjacent warps), z-neighbours from registers; written to a
//               3-slot mu ring. The tile's 1-point mu border (the rows above
//               and below, the side columns) is computed point-per-lane by
//               21 lanes of every warp (balanced critical path).
//            -> output plane k-2: L mu the same way (shuffles, mu ring rows,
//               registers) + c of plane k-2 (register); 128-bit stores.
// Shared-memory traffic per point is ~1/2 of a window-load design (the
// kernel was bound by shared wavefronts: ncu, profiles/). One __syncthreads
// per plane orders everything (mu slot of plane k-1 is written at step k and
// read at step k+1; c stage k-3 is refilled at step k). The step loop is
// unrolled by 3 so every register / slot role is static.
#pragma once

#include <type_traits>

#include "sk_stream3d.cuh"

namespace sk {

// plain 128-bit shared load: unlike the volatile-asm lds128 the compiler may
// hoist it across independent work
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }

template <class C>
struct ChfSmem {
  static constexpr int MP = C::TX + 4;              // mu ring pitch: x in [-1, TX] at column x + 2
  static constexpr int MU_ROWS = C::TY + 2;         // y in [-1, TY]
  static constexpr int MU_PLANE = MU_ROWS * MP;
  static constexpr int BYTES = C::RING_OFS + (C::STAGES * C::PLANE + 3 * MU_PLANE) * 8;
  static constexpr int WARPS = C::THREADS / 32;
  static constexpr int BORDER_ROWS = 2 * (C::TX + 2);                     // mu rows -1 and TY, x in [-1, TX]
  static constexpr int ROWS_PER_WARP = (BORDER_ROWS + WARPS - 1) / WARPS;  // + 4 side points per warp
  static_assert(ROWS_PER_WARP + 4 <= 32, "border points per warp");
};

// V = 0: the step. V = 1 (profiling only): same pipeline, loads and stores,
// no stencil arithmetic (the data-movement ceiling of this design).
template <class C, int V = 0>
__global__ void __launch_bounds__(C::THREADS, C::MIN_BLOCKS) chf3d_kernel(const Args3D a) {
  constexpr int R = 2, S = C::STAGES, P = C::PITCH;
  static_assert(C::R == 2 && C::PX == 2 && C::PY == 2 && C::TX == 64, "factored CH kernel layout: warp = row pair");
  using SM = ChfSmem<C>;
  constexpr int MP = SM::MP;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw + C::RING_OFS);
  double* mu_ring = ring + S * C::PLANE;

  // static balanced schedule: a contiguous range of (z-chunk, tile, z) units
  // per CTA (measured faster than the dynamic item queue for this
  // issue-bound kernel: no per-item pipeline re-priming)
  const int units = a.tiles_x * a.tiles_y * int(a.nz);
  const int G = gridDim.x, b = blockIdx.x;
  const int per = units / G, rem = units % G;
  const int ubeg = b * per + (b < rem ? b : rem);
  const int uend = ubeg + per + (b < rem ? 1 : 0);
  LoadCursor<C> lc;
  lc.u = ubeg;
  lc.uend = uend;
  if (ubeg < uend) lc.start(a, ring);
  int s_load = 0;
#pragma unroll 1
  for (int k = 0; k < S - 3; ++k) {
    lc.issue_next(ring, s_load, a);
    s_load = s_load + 1 == S ? 0 : s_load + 1;
  }

  const int lane = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int cofs = (2 * ty + R) * P + 2 * lane + R;  // own point (row 0, column 0) in a c stage
  const int mofs = (2 * ty + 1) * MP + 2 * lane + 2;  // own point in a mu slot
  const int64_t plane_sz = a.nx * a.ny;
  // one border point of the mu tile per lane (lanes < ROWS_PER_WARP: the
  // rows above / below the tile, contiguous; the next 4 lanes: the side
  // columns of this warp's row pair)
  int ex_c = 0, ex_m = 0;
  bool has_ex = false;
  {
    int rx = 0, ry = 0;
    if (lane < SM::ROWS_PER_WARP) {
      const int i = ty * SM::ROWS_PER_WARP + lane;
      has_ex = i < SM::BORDER_ROWS;
      rx = (i < C::TX + 2 ? i : i - (C::TX + 2)) - 1;
      ry = i < C::TX + 2 ? -1 : C::TY;
    } else if (lane < SM::ROWS_PER_WARP + 4) {
      const int sidx = lane - SM::ROWS_PER_WARP;
      has_ex = true;
      rx = sidx < 2 ? -1 : C::TX;
      ry = 2 * ty + (sidx & 1);
    }
    ex_c = (ry + R) * P + rx + R;
    ex_m = (ry + 1) * MP + rx + 2;
  }

  double Cz[3][4], M[3][4];  // own c of plane j in Cz[j % 3], own mu of plane j in M[j % 3]; point 2 * row + col
  int s_k = 0;               // stage of c-plane k
  for (int u = ubeg; u < uend; ) {
    const Seg sg = seg_of<C>(a, u, uend);
    u += sg.len;
    const int64_t gx0 = sg.x0 + 2 * lane, gy0 = sg.y0 + 2 * ty;
    const bool row0 = gy0 < a.ny, row1 = gy0 + 1 < a.ny;
    const bool vec_ok = a.bulk_ok && gx0 + 2 <= a.nx;
    double* outp = a.v + int64_t(sg.z0) * plane_sz + gy0 * a.nx + gx0;
    const int np = sg.len + 2 * R;

    // one step: plane k landed; DO_MU: mu of plane k-1; DO_OUT: output plane k-2
    auto step = [&](auto kk_t, auto mu_t, auto out_t) {
      constexpr int K = decltype(kk_t)::value;  // k % 3
      constexpr bool DO_MU = decltype(mu_t)::value, DO_OUT = decltype(out_t)::value;
      constexpr int C0 = K, C1 = (K + 2) % 3, C2 = (K + 1) % 3;  // c of planes k, k-1, k-2
      constexpr int M1 = (K + 2) % 3, M2 = (K + 1) % 3, M3 = K;  // mu of planes k-1, k-2, k-3
      cp_async_wait_group<S - 4>();
      __syncthreads();
      lc.issue_next(ring, s_load, a);
      s_load = s_load + 1 == S ? 0 : s_load + 1;
      const int s_k1 = s_k == 0 ? S - 1 : s_k - 1;   // stage of plane k-1
      const int s_k2 = s_k1 == 0 ? S - 1 : s_k1 - 1;  // stage of plane k-2
      {
        const double* cn = ring + s_k * C::PLANE + cofs;
        const double2 r0 = ld2(cn), r1 = ld2(cn + P);
        Cz[C0][0] = r0.x; Cz[C0][1] = r0.y; Cz[C0][2] = r1.x; Cz[C0][3] = r1.y;
      }
      if constexpr (DO_MU && V == 1) {
#pragma unroll
        for (int i = 0; i < 4; ++i) M[M1][i] = Cz[C1][i];
      } else if constexpr (DO_MU) {
        const double* cb = ring + s_k1 * C::PLANE + cofs;  // c, plane k-1
        const double* c1 = Cz[C1];
        const double* zp = Cz[C0];
        const double* zm = Cz[C2];
        double lf0 = __shfl_up_sync(0xffffffffu, c1[1], 1), lf1 = __shfl_up_sync(0xffffffffu, c1[3], 1);
        double rt0 = __shfl_down_sync(0xffffffffu, c1[0], 1), rt1 = __shfl_down_sync(0xffffffffu, c1[2], 1);
        if (lane == 0) { lf0 = cb[-1]; lf1 = cb[P - 1]; }
        if (lane == 31) { rt0 = cb[2]; rt1 = cb[P + 2]; }
        const double2 up = ld2(cb - P), dn = ld2(cb + 2 * P);
        // 6-neighbour sums: ((z-1 + z+1) + (left + right)) + (up + down)
        const double s00 = ((zm[0] + zp[0]) + (lf0 + c1[1])) + (up.x + c1[2]);
        const double s01 = ((zm[1] + zp[1]) + (c1[0] + rt0)) + (up.y + c1[3]);
        const double s10 = ((zm[2] + zp[2]) + (lf1 + c1[3])) + (c1[0] + dn.x);
        const double s11 = ((zm[3] + zp[3]) + (c1[2] + rt1)) + (c1[1] + dn.y);
        double* m1 = M[M1];
        m1[0] = fma(a.kl1, s00, fma(a.kl0, c1[0], poly3(c1[0], a.chem)));
        m1[1] = fma(a.kl1, s01, fma(a.kl0, c1[1], poly3(c1[1], a.chem)));
        m1[2] = fma(a.kl1, s10, fma(a.kl0, c1[2], poly3(c1[2], a.chem)));
        m1[3] = fma(a.kl1, s11, fma(a.kl0, c1[3], poly3(c1[3], a.chem)));
        double* mb = mu_ring + M1 * SM::MU_PLANE + mofs;  // slot of plane k-1
        *reinterpret_cast<double2*>(mb) = make_double2(m1[0], m1[1]);
        *reinterpret_cast<double2*>(mb + MP) = make_double2(m1[2], m1[3]);
        if (has_ex) {  // one border point of the mu tile
          const double* rb = ring + s_k1 * C::PLANE + ex_c;
          const double cc = rb[0];
          const double sr = ((ring[s_k2 * C::PLANE + ex_c] + ring[s_k * C::PLANE + ex_c]) + (rb[-1] + rb[1])) +
                            (rb[-P] + rb[P]);
          mu_ring[M1 * SM::MU_PLANE + ex_m] = fma(a.kl1, sr, fma(a.kl0, cc, poly3(cc, a.chem)));
        }
      }
      if constexpr (DO_OUT) {  // output plane k-2
        const double* c2 = Cz[C2];
        double o[4];
        if constexpr (V == 1) {
#pragma unroll
          for (int i = 0; i < 4; ++i) o[i] = c2[i];
        } else {
          const double* m1 = M[M1];
          const double* m2 = M[M2];
          const double* m3 = M[M3];
          const double* mb = mu_ring + M2 * SM::MU_PLANE + mofs;  // slot of plane k-2
          double lf0 = __shfl_up_sync(0xffffffffu, m2[1], 1), lf1 = __shfl_up_sync(0xffffffffu, m2[3], 1);
          double rt0 = __shfl_down_sync(0xffffffffu, m2[0], 1), rt1 = __shfl_down_sync(0xffffffffu, m2[2], 1);
          if (lane == 0) { lf0 = mb[-1]; lf1 = mb[MP - 1]; }
          if (lane == 31) { rt0 = mb[2]; rt1 = mb[MP + 2]; }
          const double2 up = ld2(mb - MP), dn = ld2(mb + 2 * MP);
          const double s00 = ((m3[0] + m1[0]) + (lf0 + m2[1])) + (up.x + m2[2]);
          const double s01 = ((m3[1] + m1[1]) + (m2[0] + rt0)) + (up.y + m2[3]);
          const double s10 = ((m3[2] + m1[2]) + (lf1 + m2[3])) + (m2[0] + dn.x);
          const double s11 = ((m3[3] + m1[3]) + (m2[2] + rt1)) + (m2[1] + dn.y);
          o[0] = fma(a.wl1, s00, fma(a.wl0, m2[0], c2[0]));
          o[1] = fma(a.wl1, s01, fma(a.wl0, m2[1], c2[1]));
          o[2] = fma(a.wl1, s10, fma(a.wl0, m2[2], c2[2]));
          o[3] = fma(a.wl1, s11, fma(a.wl0, m2[3], c2[3]));
        }
        if (vec_ok) {
          if (row0) store_f64x2<Mode::CahnHilliard>(outp, o[0], o[1]);
          if (row1) store_f64x2<Mode::CahnHilliard>(outp + a.nx, o[2], o[3]);
        } else {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            if (row0 && gx0 + i < a.nx) outp[i] = o[i];
            if (row1 && gx0 + i < a.nx) outp[a.nx + i] = o[2 + i];
          }
        }
        outp += plane_sz;
      }
      s_k = s_k + 1 == S ? 0 : s_k + 1;
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using T = std::true_type;
    using F = std::false_type;
    // prologue (np >= 5 always: len >= 1): k = 0..3
    step(I0{}, F{}, F{});
    step(I1{}, F{}, F{});
    step(I2{}, T{}, F{});
    step(I0{}, T{}, F{});
    // steady state: k = kb + ph, kb = 4 (mod 3 = 1)
#pragma unroll 1
    for (int kb = 4; kb < np; kb += 3) {
      step(I1{}, T{}, T{});
      if (kb + 1 < np) step(I2{}, T{}, T{});
      if (kb + 2 < np) step(I0{}, T{}, T{});
    }
  }
  cp_async_wait_all();
}

}  // namespace sk
