// TWO fused explicit Cahn-Hilliard steps per launch (temporal blocking, 3D,
// sm_100a), factored form as in sk_chf3d.cuh:
//
//   mu0 = f'(c0) - kappa L c0 ;  c1 = c0 + dt M L mu0
//   mu1 = f'(c1) - kappa L c1 ;  c2 = c1 + dt M L mu1
//
// Each launch reads c0 once and writes c2 once, so a step moves 8 instead of
// 16 bytes per point through HBM; the price is redundant arithmetic on a
// 4-point halo (radius 1 per stage, four stages).
//
// Tile: a FRAME of 64 x FY loaded points (TMA box from the ghost-padded field,
// 4-wide ghost frame), a core of 56 x (FY - 8) outputs. Warp w owns frame rows
// A w .. A w + A - 1, lane l columns 2l, 2l+1 (2A points). EVERY stage is
// evaluated on the whole frame, with no border special cases: x-neighbours
// come from warp shuffles (the outermost lanes get garbage), y-neighbours from
// the adjacent warps' published edge rows (top and bottom row of every stage
// in shared memory), z-neighbours from per-thread register queues (c0 from the
// ring). A wrong value at the frame edge moves one point inward per stage, so
// after the four stages the 56 x (FY - 8) core is exact. Operation order per
// point is exactly that of chf3d_kernel: two launches' results are
// bit-identical to single steps (tests/test_gpu_ch2step.py).
//
// Pipeline along z (per segment of `len` output planes, np = len + 8 input
// planes; iteration k: c0 plane k has landed):
//   mu0(k-1) [k >= 2]   c1(k-2) [k >= 4]   mu1(k-3) [k >= 6]   c2(k-4) [k >= 8]
// Each stage reads its input plane's neighbours published in iteration k-1,
// so one __syncthreads per plane orders everything (edge slots double
// buffered by iteration parity; c ring stage of plane k-3 is refilled at k).
//
// Status: OPT-IN (SK_CH_2STEP=1). Measured on B200 at 256^3: 97.9 us/step
// (A = 4, FY = 32) and 127 us/step (A = 2) against 62.6 us for the
// single-step kernel. The halo-4 frame computes 1.72 frame points per output
// (1.5x the fp64 work per step of the single-step kernel, whose halo is 1),
// and the kernel is issue/latency-bound (ncu: fp64 pipe 28%, issue 30%,
// stalls wait 29% / barrier 16%, 255 registers at 8 warps per SM), so the
// halved HBM traffic does not pay on this chip's fp64 rate.
#pragma once

#include "sk_chf3d.cuh"

namespace sk {

#ifndef SK_CH2_FY
#define SK_CH2_FY 32
#endif
#ifndef SK_CH2_S
#define SK_CH2_S 8
#endif
#ifndef SK_CH2_A
#define SK_CH2_A 4
#endif

template <int FY_, int A_>
struct Chf2Cfg {
  static constexpr int H = 4;                     // frame halo: 2 steps x (1 + 1)
  static constexpr int FX = 64, FY = FY_;         // frame per tile plane
  static constexpr int TX = FX - 2 * H, TY = FY - 2 * H;  // core (outputs): 56 x (FY - 8)
  static constexpr int R = H, MIN_BLOCKS = 1;     // for persistent_grid / seg_of
  static constexpr int A = A_, NP = 2 * A;       // rows per warp, points per lane
  static constexpr int WARPS = FY / A, THREADS = WARPS * 32;
  static constexpr int S = SK_CH2_S;              // c ring stages (lookahead S - 3 planes)
  static constexpr int PLANE = FX * FY;           // doubles
  static constexpr int EDGE = 2 * FX;             // a warp's published rows (top, bottom)
  static constexpr int SLOT = WARPS * EDGE;       // one stage's edge rows of one plane
  static constexpr int RING_OFS = 128;            // stage barriers in the first 128 bytes
  static constexpr int BYTES = RING_OFS + (S * PLANE + 2 * 3 * SLOT) * 8;
  static_assert(FY % A == 0 && A >= 2 && S * 8 <= 128 && (PLANE * 8) % 128 == 0, "frame layout");
  static_assert(BYTES <= 227 * 1024, "shared memory");
};
using CfgChf3D2 = Chf2Cfg<SK_CH2_FY, SK_CH2_A>;

// TMA producer (thread 0): one box per input plane, walking the CTA's unit
// range (segments of len output planes need len + 8 input planes).
template <class C>
struct Tma2Cursor {
  int u, uend, lp, np, x0, y0, z;
  __device__ __forceinline__ void start(const Args3D& a) {
    const Seg sg = seg_of<C>(a, u, uend);
    x0 = sg.x0 + kPadL - C::H;
    y0 = sg.y0 + kPadT - C::H;
    z = sg.z0 - C::H < 0 ? sg.z0 - C::H + int(a.nz) : sg.z0 - C::H;
    lp = 0;
    np = sg.len + 2 * C::H;
  }
  __device__ __forceinline__ void issue(double* ring, uint64_t* bars, int stage, const Args3D& a,
                                        const CUtensorMap* tm) {
    if (u < uend) {
      mbar_arrive_expect_tx(&bars[stage], C::PLANE * 8);
      tma_load_3d_hint<SK_TMA_HINT>(ring + stage * C::PLANE, tm, x0, y0, z, &bars[stage]);
      z = z + 1 == a.nz ? 0 : z + 1;
      if (++lp == np) {
        u += np - 2 * C::H;
        if (u < uend) start(a);
      }
    }
  }
};

// 6-neighbour sums of the 2A own points of plane X (rows r = 0..A-1, columns
// 0, 1 -> index 2r + col): (((left + right) + (up + down)) + z-1) + z+1, the
// order of chf3d_kernel. up / dn: the rows above and below this warp's rows.
// The z+1 plane (computed in the same iteration) enters last, so the in-plane
// parts of all four stages are independent work.
template <int A>
__device__ __forceinline__ void nb_sums(const double* X, const double* Xm, const double* Xp, double2 up,
                                        double2 dn, double* s) {
#pragma unroll
  for (int r = 0; r < A; ++r) {
    const double lf = __shfl_up_sync(0xffffffffu, X[2 * r + 1], 1);
    const double rt = __shfl_down_sync(0xffffffffu, X[2 * r], 1);
    const double u0 = r == 0 ? up.x : X[2 * r - 2], u1 = r == 0 ? up.y : X[2 * r - 1];
    const double d0 = r == A - 1 ? dn.x : X[2 * r + 2], d1 = r == A - 1 ? dn.y : X[2 * r + 3];
    s[2 * r] = (((lf + X[2 * r + 1]) + (u0 + d0)) + Xm[2 * r]) + Xp[2 * r];
    s[2 * r + 1] = (((X[2 * r] + rt) + (u1 + d1)) + Xm[2 * r + 1]) + Xp[2 * r + 1];
  }
}

// OUT 1: c2 into the interior of a ghost-padded field (kPadT >= 4 rows) plus
// its periodic images in the 4-wide ghost frame; OUT 0: plain field.
template <class C, int OUT>
__global__ void __launch_bounds__(C::THREADS, 1)
    chf3d2_kernel(const __grid_constant__ Args3D a, const __grid_constant__ CUtensorMap tmap) {
  constexpr int S = C::S, FX = C::FX, FY = C::FY, PLANE = C::PLANE, H = C::H, A = C::A, NP = C::NP;
  static_assert(kPadT >= H, "2-step boxes need a 4-row ghost frame");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  double* ring = reinterpret_cast<double*>(smem_raw + C::RING_OFS);
  double* pub = ring + S * PLANE;  // [parity][stage 0: mu0, 1: c1, 2: mu1][SLOT]

  const int units = a.tiles_x * a.tiles_y * int(a.nz);
  const int G = gridDim.x, b = blockIdx.x;
  const int per = units / G, rem = units % G;
  const int ubeg = b * per + (b < rem ? b : rem);
  const int uend = ubeg + per + (b < rem ? 1 : 0);

  Tma2Cursor<C> tc;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // programmatic dependent launch: the previous launch wrote our input
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    tc.u = ubeg;
    tc.uend = uend;
    if (ubeg < uend) tc.start(a);
    for (int k = 0; k < S - 3; ++k) tc.issue(ring, bars, k, a, &tmap);
  }
  int s_load = S - 3;

  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  const int own = A * w * FX + 2 * lane;                                    // row 0 of own points in a ring stage
  const int rup = (w == 0 ? 0 : A * w - 1) * FX + 2 * lane;                 // row above (clamped: garbage row)
  const int rdn = (w == C::WARPS - 1 ? FY - 1 : A * w + A) * FX + 2 * lane;  // row below
  const int pme = w * C::EDGE + 2 * lane;                                   // own edge rows in a slot
  const int pup = (w == 0 ? 0 : (w - 1) * C::EDGE + FX) + 2 * lane;         // bottom row of warp w-1
  const int pdn = (w == C::WARPS - 1 ? w * C::EDGE : (w + 1) * C::EDGE) + 2 * lane;  // top row of warp w+1
  const bool out_warp = A * w + A > H && A * w < FY - H;  // warps holding core rows
  const bool out_lane = out_warp && lane >= H / 2 && lane < (FX - H) / 2;
  const int64_t opx = OUT ? a.nx + 2 * kPadL : a.nx, opp = opx * (OUT ? a.ny + 2 * kPadT : a.ny);

  // queues: plane j of each field in slot j % 3
  double m0q[3][NP], c1q[3][NP], m1q[3][NP];  // c0's own points are re-read from the ring
  int s_k = 0;       // ring stage of c0 plane k
  uint32_t ph = 0;   // its mbarrier parity
  for (int u = ubeg; u < uend;) {
    const Seg sg = seg_of<C>(a, u, uend);
    u += sg.len;
    const int np = sg.len + 2 * H;
    const int gx = sg.x0 + 2 * lane - H;   // global x of own column 0
    const int gy = sg.y0 + A * w - H;      // global y of own row 0
    bool st_ok[A];
#pragma unroll
    for (int r = 0; r < A; ++r)
      st_ok[r] = out_lane && gx < a.nx && gy + r >= sg.y0 && gy + r < sg.y0 + C::TY && gy + r < a.ny;
    double* outp = a.v + int64_t(sg.z0) * opp + int64_t(gy + (OUT ? kPadT : 0)) * opx + gx + (OUT ? kPadL : 0);
    const int64_t gdx = OUT ? (gx < 4 ? a.nx : (gx >= a.nx - 4 ? -a.nx : 0)) : 0;
    int64_t gdy[A];
#pragma unroll
    for (int r = 0; r < A; ++r) gdy[r] = OUT ? (gy + r < 4 ? a.ny : (gy + r >= a.ny - 4 ? -a.ny : 0)) * opx : 0;

    auto step = [&](auto kk_t, int k) {
      constexpr int K = decltype(kk_t)::value;  // k % 3
      constexpr int J0 = K, J1 = (K + 2) % 3, J2 = (K + 1) % 3;  // slots of planes k, k-1, k-2 (mod 3)
      mbar_wait(&bars[s_k], ph);  // c0 plane k landed
      __syncthreads();            // ... and every read of iteration k-1 is done
      if (threadIdx.x == 0) {
        fence_proxy_async_smem();
        tc.issue(ring, bars, s_load, a, &tmap);  // plane k + S - 3 into the stage of plane k - 3
      }
      s_load = s_load + 1 == S ? 0 : s_load + 1;
      const int s_k1 = s_k == 0 ? S - 1 : s_k - 1, s_k2 = s_k1 == 0 ? S - 1 : s_k1 - 1;
      const double* rk = ring + s_k * PLANE;
      const double* rk1 = ring + s_k1 * PLANE;
      const double* rk2 = ring + s_k2 * PLANE;
      double* pw = pub + (k & 1) * 3 * C::SLOT;         // publish (this iteration)
      const double* pr = pub + (~k & 1) * 3 * C::SLOT;  // read (iteration k-1)
#pragma unroll
      double cn[NP], cm1[NP], cm2[NP];  // own c0 of planes k, k-1, k-2
      auto ld_own = [&](const double* st, double* x) {
#pragma unroll
        for (int r = 0; r < A; ++r) {
          const double2 v = ld2(st + own + r * FX);
          x[2 * r] = v.x;
          x[2 * r + 1] = v.y;
        }
      };
      if (k >= 2) {
        ld_own(rk, cn);
        ld_own(rk1, cm1);
        ld_own(rk2, cm2);
      }
      auto publish = [&](double* slot, const double* x) {
        *reinterpret_cast<double2*>(slot + pme) = make_double2(x[0], x[1]);
        *reinterpret_cast<double2*>(slot + pme + FX) = make_double2(x[NP - 2], x[NP - 1]);
      };
      double s[NP];
      if (k >= 2) {  // mu0(k-1) from c0(k-2), c0(k-1), c0(k)
        const double* x = cm1;
        nb_sums<A>(x, cm2, cn, ld2(rk1 + rup), ld2(rk1 + rdn), s);
        double* m = m0q[J1];
#pragma unroll
        for (int i = 0; i < NP; ++i) m[i] = fma(a.kl1, s[i], fma(a.kl0, x[i], poly3(x[i], a.chem)));
        publish(pw, m);
      }
      if (k >= 4) {  // c1(k-2) = c0(k-2) + dt M L mu0(k-2)
        const double* x = m0q[J2];
        nb_sums<A>(x, m0q[J0], m0q[J1], ld2(pr + pup), ld2(pr + pdn), s);
        double* c = c1q[J2];
        const double* base = cm2;
#pragma unroll
        for (int i = 0; i < NP; ++i) c[i] = fma(a.wl1, s[i], fma(a.wl0, x[i], base[i]));
        publish(pw + C::SLOT, c);
      }
      if (k >= 6) {  // mu1(k-3) from c1(k-4), c1(k-3), c1(k-2)
        const double* x = c1q[J0];
        nb_sums<A>(x, c1q[J1], c1q[J2], ld2(pr + C::SLOT + pup), ld2(pr + C::SLOT + pdn), s);
        double* m = m1q[J0];
#pragma unroll
        for (int i = 0; i < NP; ++i) m[i] = fma(a.kl1, s[i], fma(a.kl0, x[i], poly3(x[i], a.chem)));
        publish(pw + 2 * C::SLOT, m);
      }
      if (k >= 8 && out_warp) {  // c2(k-4) = c1(k-4) + dt M L mu1(k-4) (core rows only)
        const double* x = m1q[J1];
        nb_sums<A>(x, m1q[J2], m1q[J0], ld2(pr + 2 * C::SLOT + pup), ld2(pr + 2 * C::SLOT + pdn), s);
        const double* base = c1q[J1];
        double o[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) o[i] = fma(a.wl1, s[i], fma(a.wl0, x[i], base[i]));
#pragma unroll
        for (int r = 0; r < A; ++r) {
          if (st_ok[r]) {
            double* p = outp + r * opx;
            store_f64x2<Mode::CahnHilliard>(p, o[2 * r], o[2 * r + 1]);
            if constexpr (OUT == 1) {
              if (gdx) store_f64x2<Mode::CahnHilliard>(p + gdx, o[2 * r], o[2 * r + 1]);
              if (gdy[r]) {
                store_f64x2<Mode::CahnHilliard>(p + gdy[r], o[2 * r], o[2 * r + 1]);
                if (gdx) store_f64x2<Mode::CahnHilliard>(p + gdy[r] + gdx, o[2 * r], o[2 * r + 1]);
              }
            }
          }
        }
        outp += opp;
      }
      s_k = s_k + 1 == S ? 0 : s_k + 1;
      if (s_k == 0) ph ^= 1u;
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
#pragma unroll 1
    for (int k = 0; k < np; k += 3) {
      step(I0{}, k);
      if (k + 1 < np) step(I1{}, k + 1);
      if (k + 2 < np) step(I2{}, k + 2);
    }
  }
  asm volatile("griddepcontrol.launch_dependents;");
}

}  // namespace sk
