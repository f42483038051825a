// Fused explicit Cahn-Hilliard step in FACTORED form (3D, sm_100a):
//
//   mu = f'(c) - kappa L c          (chemical potential, 7-point L)
//   c' = c + dt M L mu              (= c + dt M (L f'(c) - kappa L(L c)))
//
// L(L c) is exactly the composed 25-point operator B c (B = compose(L, L),
// stencil.cpp:75-87), so this is the same step as the composed kernel in
// sk_stream3d.cuh up to rounding, with ~19 instead of ~37 fp64 operations per
// point and a handful of registers. It is the north-star form
// Delta(u^3 - u - eps^2 Delta u) fused into one pass.
//
// Streaming along z (per CTA: one TX x TY column tile over a z-range, the
// persistent balanced unit order of sk_stream3d.cuh):
//   step k : c-plane k has landed (multistage cp.async ring, S stages)
//            -> mu of plane k-1 on the tile + a 1-point ring (c planes
//               k-2, k-1, k), own points from 128-bit loads, ring points by
//               a few threads; written to a 2-slot mu ring in shared memory
//            -> output plane k-2: L mu from the mu ring (in-plane) and the
//               thread's own mu of planes k-3, k-1 (registers), + c of
//               plane k-2 (register), streamed out with 128-bit stores.
// One __syncthreads per plane orders everything (mu slot written at step k is
// read at step k+1; c stage k-3 is refilled at step k).
#pragma once

#include <type_traits>

#include "sk_stream3d.cuh"

namespace sk {

template <class C>
struct ChfSmem {
  static constexpr int MU_ROWS = C::TY + 2;          // y in [-1, TY]
  static constexpr int MU_PLANE = MU_ROWS * C::PITCH;  // x at column x + 2 (interior 16B aligned)
  static constexpr int BYTES = 128 + (C::STAGES * C::PLANE + 2 * MU_PLANE) * 8;
  static constexpr int RING_PTS = 2 * (C::TX + 2) + 2 * C::TY;  // the 1-point border
};

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MIN_BLOCKS) chf3d_kernel(const Args3D a) {
  constexpr int R = 2, S = C::STAGES, P = C::PITCH;
  static_assert(C::R == 2 && C::PX == 2 && C::PY == 2, "factored CH kernel layout");
  using SM = ChfSmem<C>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw + 128);
  double* mu_ring = ring + S * C::PLANE;

  const int64_t units = int64_t(a.tiles_x) * a.tiles_y * a.nz;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t per = units / G, rem = units % G;
  const int64_t ubeg = b * per + (b < rem ? b : rem);
  const int64_t uend = ubeg + per + (b < rem ? 1 : 0);

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

  const int tx = threadIdx.x % (C::TX / 2), ty = threadIdx.x / (C::TX / 2);
  const int cofs = (2 * ty + R) * P + 2 * tx + R;  // own point (x, y) in a c buffer
  const int mofs = (2 * ty + 1) * P + 2 * tx + 2;  // own point in a mu buffer
  const int64_t plane_sz = a.nx * a.ny;
  // ring point handled by this thread (if any): its coordinates in tile space
  int rx = 0, ry = 0;
  // border points on the first RING_PTS threads (consecutive lanes on
  // consecutive shared-memory words; measured faster than spreading them)
  const int ring_i = threadIdx.x;
  const bool has_ring = ring_i < SM::RING_PTS;
  {
    const int i = ring_i;
    if (i < C::TX + 2) { rx = i - 1; ry = -1; }
    else if (i < 2 * (C::TX + 2)) { rx = i - (C::TX + 2) - 1; ry = C::TY; }
    else if (i < 2 * (C::TX + 2) + C::TY) { rx = -1; ry = i - 2 * (C::TX + 2); }
    else { rx = C::TX; ry = i - 2 * (C::TX + 2) - C::TY; }
  }
  const int ring_c = (ry + R) * P + rx + R;
  const int ring_m = (ry + 1) * P + rx + 2;

  // Register roles are static: mu of plane j lives in M[j % 3], own c of
  // plane j in Cc[j % 2]; the steady-state loop is unrolled by 6 (lcm) so no
  // register is ever copied. Shared-memory stage indices rotate at run time.
  double M[3][4], Cc[2][4];
  int s_k = 0;  // stage of c-plane k
  for (int64_t u = ubeg; u < uend;) {
    const Seg sg = seg_of<C>(a, u, uend);
    const int64_t gx0 = sg.x0 + 2 * tx, gy0 = sg.y0 + 2 * ty;
    const bool row0 = gy0 < a.ny, row1 = gy0 + 1 < a.ny;
    const bool vec_ok = a.bulk_ok && gx0 + 2 <= a.nx;
    double* outp = a.v + sg.z0 * plane_sz + gy0 * a.nx + gx0;
    const int np = int(sg.len) + 2 * R;

    // one step: plane k landed; DO_MU: mu of plane k-1; DO_OUT: output plane k-2
    auto step = [&](auto k3_t, auto k2_t, auto mu_t, auto out_t, int k) {
      constexpr int K3 = decltype(k3_t)::value, K2 = decltype(k2_t)::value;
      constexpr bool DO_MU = decltype(mu_t)::value, DO_OUT = decltype(out_t)::value;
      constexpr int I_M1 = (K3 + 2) % 3, I_M2 = (K3 + 1) % 3, I_M3 = K3;  // planes k-1, k-2, k-3
      constexpr int I_C1 = (K2 + 1) % 2, I_C2 = K2;                      // planes k-1, k-2
      cp_async_wait_group<S - 4>();
      __syncthreads();
      lc.issue_next(ring, s_load, a);
      s_load = s_load + 1 == S ? 0 : s_load + 1;
      const int s_k1 = s_k == 0 ? S - 1 : s_k - 1;   // stage of plane k-1
      const int s_k2 = s_k1 == 0 ? S - 1 : s_k1 - 1;  // stage of plane k-2
      if constexpr (DO_MU) {
        const double* cb = ring + s_k1 * C::PLANE + cofs;  // c, plane k-1 (in-plane window)
        const double* cn = ring + s_k * C::PLANE + cofs;   // c, plane k (z+1 centres)
        double* mb = mu_ring + ((k - 1) & 1) * SM::MU_PLANE + mofs;
        const double2 up = lds128(cb - P), dn = lds128(cb + 2 * P);
        const double2 l0 = lds128(cb - 2), o0 = lds128(cb), r0 = lds128(cb + 2);
        const double2 l1 = lds128(cb + P - 2), o1 = lds128(cb + P), r1 = lds128(cb + P + 2);
        const double2 z0n = lds128(cn), z1n = lds128(cn + P);
        double* c1 = Cc[I_C1];
        const double* c2 = Cc[I_C2];
        double* m1 = M[I_M1];
        c1[0] = o0.x; c1[1] = o0.y; c1[2] = o1.x; c1[3] = o1.y;
        // 6-neighbour sums (z-1 from the register copy of plane k-2)
        double s6[4];
        s6[0] = ((c2[0] + z0n.x) + (l0.y + o0.y)) + (up.x + o1.x);
        s6[1] = ((c2[1] + z0n.y) + (o0.x + r0.x)) + (up.y + o1.y);
        s6[2] = ((c2[2] + z1n.x) + (l1.y + o1.y)) + (o0.x + dn.x);
        s6[3] = ((c2[3] + z1n.y) + (o1.x + r1.x)) + (o0.y + dn.y);
#pragma unroll
        for (int i = 0; i < 4; ++i) m1[i] = fma(a.kl1, s6[i], fma(a.kl0, c1[i], poly3(c1[i], a.chem)));
        *reinterpret_cast<double2*>(mb) = make_double2(m1[0], m1[1]);
        *reinterpret_cast<double2*>(mb + P) = make_double2(m1[2], m1[3]);
        if (has_ring) {  // one border point of the mu tile
          const double* rb = ring + s_k1 * C::PLANE + ring_c;
          const double cc = rb[0];
          const double sr = ((ring[s_k2 * C::PLANE + ring_c] + ring[s_k * C::PLANE + ring_c]) + (rb[-1] + rb[1])) +
                            (rb[-P] + rb[P]);
          mu_ring[((k - 1) & 1) * SM::MU_PLANE + ring_m] = fma(a.kl1, sr, fma(a.kl0, cc, poly3(cc, a.chem)));
        }
      } else if (K2 == 0 && K3 == 0) {  // k == 0: step 2 needs c of plane 0 (its z-1 centres)
        const double* cb = ring + s_k * C::PLANE + cofs;
        const double2 o0 = lds128(cb), o1 = lds128(cb + P);
        Cc[0][0] = o0.x; Cc[0][1] = o0.y; Cc[0][2] = o1.x; Cc[0][3] = o1.y;
      }
      if constexpr (DO_OUT) {  // output plane k-2
        const double* mb = mu_ring + (k & 1) * SM::MU_PLANE + mofs;  // slot of plane k-2
        const double2 up = lds128(mb - P), dn = lds128(mb + 2 * P);
        const double2 l0 = lds128(mb - 2), r0 = lds128(mb + 2);
        const double2 l1 = lds128(mb + P - 2), r1 = lds128(mb + P + 2);
        const double* m1 = M[I_M1];
        const double* m2 = M[I_M2];
        const double* m3 = M[I_M3];
        const double* c2 = Cc[I_C2];
        double s6[4], o[4];
        s6[0] = ((m3[0] + m1[0]) + (l0.y + m2[1])) + (up.x + m2[2]);
        s6[1] = ((m3[1] + m1[1]) + (m2[0] + r0.x)) + (up.y + m2[3]);
        s6[2] = ((m3[2] + m1[2]) + (l1.y + m2[3])) + (m2[0] + dn.x);
        s6[3] = ((m3[3] + m1[3]) + (m2[2] + r1.x)) + (m2[1] + dn.y);
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = fma(a.wl1, s6[i], fma(a.wl0, m2[i], c2[i]));
        if (vec_ok) {
          if (row0) store_f64x2<Mode::CahnHilliard>(outp, o[0], o[1]);
          if (row1) store_f64x2<Mode::CahnHilliard>(outp + a.nx, o[2], o[3]);
        } else {
          if (row0 && gx0 < a.nx) outp[0] = o[0];
          if (row0 && gx0 + 1 < a.nx) outp[1] = o[1];
          if (row1 && gx0 < a.nx) outp[a.nx] = o[2];
          if (row1 && gx0 + 1 < a.nx) outp[a.nx + 1] = o[3];
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
    step(I0{}, I0{}, F{}, F{}, 0);
    step(I1{}, I1{}, F{}, F{}, 1);
    step(I2{}, I0{}, T{}, F{}, 2);
    step(I0{}, I1{}, T{}, F{}, 3);
    // steady state: k = kb + ph, kb = 4 (mod 6): k % 3 = (1 + ph) % 3, k % 2 = ph % 2
#pragma unroll 1
    for (int kb = 4; kb < np; kb += 6) {
      step(I1{}, I0{}, T{}, T{}, kb);
      if (kb + 1 < np) step(I2{}, I1{}, T{}, T{}, kb + 1);
      if (kb + 2 < np) step(I0{}, I0{}, T{}, T{}, kb + 2);
      if (kb + 3 < np) step(I1{}, I1{}, T{}, T{}, kb + 3);
      if (kb + 4 < np) step(I2{}, I0{}, T{}, T{}, kb + 4);
      if (kb + 5 < np) step(I0{}, I1{}, T{}, T{}, kb + 5);
    }
    u += sg.len;
  }
  cp_async_wait_all();
}

}  // namespace sk
