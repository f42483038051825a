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
// unit schedule of sk_stream3d.cuh):
//   step k : c-plane k has landed (multistage cp.async ring, S stages)
//            -> mu of plane k-1 on the tile + a 1-point ring (c planes
//               k-2, k-1, k), own points from 128-bit loads, ring points by
//               a few threads; written to a 2-slot mu ring in shared memory
//            -> output plane k-2: L mu from the mu ring (in-plane) and the
//               thread's own mu of planes k-3, k-1 (registers), + c of
//               plane k-2 (register), streamed out with 128-bit stores.
// One __syncthreads per plane orders everything (mu slot written at step k is
// read at step k+1; c stage k-3 is refilled at step k). Each thread owns
// 2 rows x PX columns; register roles are static (mu of plane j in M[j % 3],
// own c of plane j in Cc[j % 2], loop unrolled by 6), so no register moves.
#pragma once

#include <type_traits>

#include "sk_stream3d.cuh"

namespace sk {

template <class C>
struct ChfSmem {
  static constexpr int MU_ROWS = C::TY + 2;            // y in [-1, TY]
  static constexpr int MU_PLANE = MU_ROWS * C::PITCH;  // x at column x + 2 (interior 16B aligned)
  static constexpr int BYTES = 128 + (C::STAGES * C::PLANE + 2 * MU_PLANE) * 8;
  static constexpr int RING_PTS = 2 * (C::TX + 2) + 2 * C::TY;  // the 1-point border
  static constexpr int RING_PER_THREAD = (RING_PTS + C::THREADS - 1) / C::THREADS;
};

// V = 0: the step. V = 1 (profiling only): same pipeline, loads and stores,
// no stencil arithmetic (the data-movement ceiling of this design).
template <class C, int V = 0>
__global__ void __launch_bounds__(C::THREADS, C::MIN_BLOCKS) chf3d_kernel(const Args3D a) {
  constexpr int R = 2, S = C::STAGES, P = C::PITCH, PX = C::PX, NP = 2 * PX;
  constexpr int W = PX + 4;  // in-row window x-2 .. x+PX+1
  static_assert(C::R == 2 && C::PY == 2 && (PX == 2 || PX == 4), "factored CH kernel layout");
  using SM = ChfSmem<C>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw + 128);
  double* mu_ring = ring + S * C::PLANE;

  // static balanced schedule: a contiguous range of (z-chunk, tile, z) units
  // per CTA (measured faster than the dynamic item queue for this
  // issue-bound kernel: no per-item pipeline re-priming)
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

  const int tx = threadIdx.x % (C::TX / PX), ty = threadIdx.x / (C::TX / PX);
  const int cofs = (2 * ty + R) * P + PX * tx + R;  // own point (x, y) in a c buffer
  const int mofs = (2 * ty + 1) * P + PX * tx + 2;  // own point in a mu buffer
  const int64_t plane_sz = a.nx * a.ny;
  // border points of the mu tile: point i on thread i % THREADS
  int ring_c[SM::RING_PER_THREAD], ring_m[SM::RING_PER_THREAD];
  bool has_ring[SM::RING_PER_THREAD];
#pragma unroll
  for (int q = 0; q < SM::RING_PER_THREAD; ++q) {
    const int i = threadIdx.x + q * C::THREADS;
    int rx, ry;
    if (i < C::TX + 2) { rx = i - 1; ry = -1; }
    else if (i < 2 * (C::TX + 2)) { rx = i - (C::TX + 2) - 1; ry = C::TY; }
    else if (i < 2 * (C::TX + 2) + C::TY) { rx = -1; ry = i - 2 * (C::TX + 2); }
    else { rx = C::TX; ry = i - 2 * (C::TX + 2) - C::TY; }
    has_ring[q] = i < SM::RING_PTS;
    ring_c[q] = (ry + R) * P + rx + R;
    ring_m[q] = (ry + 1) * P + rx + 2;
  }

  double M[3][NP], Cc[2][NP];  // own points: j * PX + i (row j, column i)
  int s_k = 0;                 // stage of c-plane k
  for (int64_t u = ubeg; u < uend; ) {
    const Seg sg = seg_of<C>(a, u, uend);
    u += sg.len;
    const int64_t gx0 = sg.x0 + PX * tx, gy0 = sg.y0 + 2 * ty;
    const bool row0 = gy0 < a.ny, row1 = gy0 + 1 < a.ny;
    const bool vec_ok = a.bulk_ok && gx0 + PX <= a.nx;
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
      if constexpr (DO_MU && V == 1) {
        const double* cb = ring + s_k1 * C::PLANE + cofs;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int m = 0; m < PX; m += 2) {
            const double2 o = lds128(cb + j * P + m);
            Cc[I_C1][j * PX + m] = M[I_M1][j * PX + m] = o.x;
            Cc[I_C1][j * PX + m + 1] = M[I_M1][j * PX + m + 1] = o.y;
          }
      } else if constexpr (DO_MU) {
        const double* cb = ring + s_k1 * C::PLANE + cofs;  // c, plane k-1 (in-plane window)
        const double* cn = ring + s_k * C::PLANE + cofs;   // c, plane k (z+1 centres)
        double* mb = mu_ring + ((k - 1) & 1) * SM::MU_PLANE + mofs;
        double w0[W], w1[W], up[PX], dn[PX], z0[PX], z1[PX];
#pragma unroll
        for (int m = 0; m < W; m += 2) {
          const double2 a0 = lds128(cb + m - 2), a1 = lds128(cb + P + m - 2);
          w0[m] = a0.x; w0[m + 1] = a0.y; w1[m] = a1.x; w1[m + 1] = a1.y;
        }
#pragma unroll
        for (int m = 0; m < PX; m += 2) {
          const double2 u2 = lds128(cb - P + m), d2 = lds128(cb + 2 * P + m);
          const double2 za = lds128(cn + m), zb = lds128(cn + P + m);
          up[m] = u2.x; up[m + 1] = u2.y; dn[m] = d2.x; dn[m + 1] = d2.y;
          z0[m] = za.x; z0[m + 1] = za.y; z1[m] = zb.x; z1[m + 1] = zb.y;
        }
        double* c1 = Cc[I_C1];
        const double* c2 = Cc[I_C2];
        double* m1 = M[I_M1];
#pragma unroll
        for (int i = 0; i < PX; ++i) {
          c1[i] = w0[i + 2];
          c1[PX + i] = w1[i + 2];
          // 6-neighbour sums: ((z-1 + z+1) + (left + right)) + (up + down)
          const double s0 = ((c2[i] + z0[i]) + (w0[i + 1] + w0[i + 3])) + (up[i] + w1[i + 2]);
          const double s1 = ((c2[PX + i] + z1[i]) + (w1[i + 1] + w1[i + 3])) + (w0[i + 2] + dn[i]);
          m1[i] = fma(a.kl1, s0, fma(a.kl0, c1[i], poly3(c1[i], a.chem)));
          m1[PX + i] = fma(a.kl1, s1, fma(a.kl0, c1[PX + i], poly3(c1[PX + i], a.chem)));
        }
#pragma unroll
        for (int m = 0; m < PX; m += 2) {
          *reinterpret_cast<double2*>(mb + m) = make_double2(m1[m], m1[m + 1]);
          *reinterpret_cast<double2*>(mb + P + m) = make_double2(m1[PX + m], m1[PX + m + 1]);
        }
#pragma unroll
        for (int q = 0; q < SM::RING_PER_THREAD; ++q) {
          if (has_ring[q]) {  // one border point of the mu tile
            const double* rb = ring + s_k1 * C::PLANE + ring_c[q];
            const double cc = rb[0];
            const double sr = ((ring[s_k2 * C::PLANE + ring_c[q]] + ring[s_k * C::PLANE + ring_c[q]]) +
                               (rb[-1] + rb[1])) + (rb[-P] + rb[P]);
            mu_ring[((k - 1) & 1) * SM::MU_PLANE + ring_m[q]] = fma(a.kl1, sr, fma(a.kl0, cc, poly3(cc, a.chem)));
          }
        }
      } else if (K2 == 0 && K3 == 0) {  // k == 0: step 2 needs c of plane 0 (its z-1 centres)
        const double* cb = ring + s_k * C::PLANE + cofs;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int m = 0; m < PX; m += 2) {
            const double2 o = lds128(cb + j * P + m);
            Cc[0][j * PX + m] = o.x;
            Cc[0][j * PX + m + 1] = o.y;
          }
      }
      if constexpr (DO_OUT) {  // output plane k-2
        const double* m1 = M[I_M1];
        const double* m2 = M[I_M2];
        const double* m3 = M[I_M3];
        const double* c2 = Cc[I_C2];
        double o[NP];
        if constexpr (V == 1) {
#pragma unroll
          for (int i = 0; i < NP; ++i) o[i] = c2[i];
        } else {
          const double* mb = mu_ring + (k & 1) * SM::MU_PLANE + mofs;  // slot of plane k-2
          double mu[PX], md[PX];
#pragma unroll
          for (int m = 0; m < PX; m += 2) {
            const double2 u2 = lds128(mb - P + m), d2 = lds128(mb + 2 * P + m);
            mu[m] = u2.x; mu[m + 1] = u2.y; md[m] = d2.x; md[m + 1] = d2.y;
          }
          const double l0 = lds128(mb - 2).y, r0 = lds128(mb + PX).x;
          const double l1 = lds128(mb + P - 2).y, r1 = lds128(mb + P + PX).x;
#pragma unroll
          for (int i = 0; i < PX; ++i) {
            const double lf0 = i > 0 ? m2[i - 1] : l0, rt0 = i < PX - 1 ? m2[i + 1] : r0;
            const double lf1 = i > 0 ? m2[PX + i - 1] : l1, rt1 = i < PX - 1 ? m2[PX + i + 1] : r1;
            const double s0 = ((m3[i] + m1[i]) + (lf0 + rt0)) + (mu[i] + m2[PX + i]);
            const double s1 = ((m3[PX + i] + m1[PX + i]) + (lf1 + rt1)) + (m2[i] + md[i]);
            o[i] = fma(a.wl1, s0, fma(a.wl0, m2[i], c2[i]));
            o[PX + i] = fma(a.wl1, s1, fma(a.wl0, m2[PX + i], c2[PX + i]));
          }
        }
        if (vec_ok) {
#pragma unroll
          for (int m = 0; m < PX; m += 2) {
            if (row0) store_f64x2<Mode::CahnHilliard>(outp + m, o[m], o[m + 1]);
            if (row1) store_f64x2<Mode::CahnHilliard>(outp + a.nx + m, o[PX + m], o[PX + m + 1]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < PX; ++i) {
            if (row0 && gx0 + i < a.nx) outp[i] = o[i];
            if (row1 && gx0 + i < a.nx) outp[a.nx + i] = o[PX + i];
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
  }
  cp_async_wait_all();
}

}  // namespace sk
