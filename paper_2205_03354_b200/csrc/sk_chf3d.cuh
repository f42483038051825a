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
// kernel was bound by shared wavefronts: ncu, profiles/). Stages complete on
// FULL mbarriers (TMA bytes, or every thread's cp.async arrivals); a
// split-phase step barrier orders the rest (mu slot of plane k-1 is written
// at step k and read at step k+1; c stage k-3 is refilled at step k; see the
// comment at `stepbar`). The step loop is unrolled by 3 so every register /
// slot role is static.
#pragma once

#include <cuda.h>

#include <type_traits>

#include "sk_stream3d.cuh"

namespace sk {


// Ghost-padded field of the TMA path: row pitch nx + 2 kPadL, kPadT ghost
// rows above and below; interior x at column x + kPadL (128 B-aligned rows
// and tiles, so the interior stores are whole lines), ghosts x = -2, -1 and
// nx, nx + 1 at columns kPadL - 2 .. and kPadL + nx ... (images: 4 columns, 2 rows)
#ifndef SK_PADL
#define SK_PADL 16
#endif
constexpr int kPadL = SK_PADL, kPadT = 2;  // ghost rows above and below (the radius-2 periodic images)
// L2 policy of the TMA loads: evict_last keeps tile halos for the
// y-neighbour tile's CTA (measured +0.5%; evict_first: -19%)
#ifndef SK_TMA_HINT
#define SK_TMA_HINT 1
#endif
#ifndef SK_MU_SLOTS
#define SK_MU_SLOTS 3
#endif
#ifndef SK_TMA_SPLIT
#define SK_TMA_SPLIT 1
#endif
constexpr int kTmaSplit = SK_TMA_SPLIT;  // TMA boxes per plane

// LD 0: cp.async ring over the caller's field (periodic wrap per chunk,
// 128 B-aligned pitch C::PITCH). LD 1: one TMA box per plane from a
// ghost-padded field (kPadL / kPadT below, see OUT 1) into dense stages of
// pitch C::WIDTH; no wrap logic, no per-thread copy instructions.
template <class C, int LD = 0, bool FB = false>
struct ChfSmem {
  // LD 1 boxes start XO = 4 columns left of the tile and are 72 wide: whole
  // 32 B sectors from the 128 B-aligned padded rows, and a 576 B pitch whose
  // row pairs are 128 B multiples (the box may be split along y)
  static constexpr int XO = LD ? 2 * C::R : C::R;            // column of tile x = 0 in a stage
  static constexpr int P = LD ? C::TX + 4 * C::R : C::PITCH;  // c stage pitch
  static constexpr int PLANE = C::ROWS * P;
  static constexpr int RING_OFS = LD ? 128 : C::RING_OFS;  // LD 1: stage barriers in the first 128 B
  static constexpr uint32_t STAGE_BYTES = PLANE * 8;
  static constexpr int MP = C::TX + 4;              // mu ring pitch: x in [-1, TX] at column x + 2
  static constexpr int MU_ROWS = C::TY + 2;         // y in [-1, TY]
  static constexpr int MU_PLANE = MU_ROWS * MP;
  // 3: slot = plane % 3 (static roles); 4 (TMA path): rotating slots, which
  // lets the step barrier's wait move after the mu write (more slack)
  static constexpr int MU_SLOTS = LD ? SK_MU_SLOTS : 3;
  // LD 0 with the 8-byte fallback loader (FB): its boundary-map table after the mu ring
  static constexpr int TAB = C::STAGES * PLANE + MU_SLOTS * MU_PLANE;  // doubles from the ring
  static constexpr int BYTES = RING_OFS + TAB * 8 + (FB ? C::TABLE_BYTES : 0);
  static constexpr int WARPS = C::THREADS / 32;
  static constexpr int BORDER_ROWS = 2 * (C::TX + 2);                     // mu rows -1 and TY, x in [-1, TX]
  static constexpr int ROWS_PER_WARP = (BORDER_ROWS + WARPS - 1) / WARPS;  // + 4 side points per warp
  static_assert(ROWS_PER_WARP + 4 <= 32, "border points per warp");
  static_assert(!LD || STAGE_BYTES % 128 == 0, "TMA stage alignment");
  static_assert((C::STAGES + 3) * 8 <= (LD ? 128 : C::RING_OFS), "full + step barriers before the ring");
  static_assert(!LD || (C::ROWS % kTmaSplit == 0 && (C::ROWS / kTmaSplit) * P * 8 % 128 == 0), "TMA box split");
};

// TMA producer (thread 0): walks the CTA's unit range one plane ahead of
// the consumers' needs, like LoadCursor, issuing one box per plane.
template <class C>
struct TmaCursor {
  int u, uend, lp, np, x0, y0, z;
  __device__ __forceinline__ void start(const Args3D& a) {
    const Seg sg = seg_of<C>(a, u, uend);
    x0 = sg.x0 + kPadL - ChfSmem<C, 1>::XO;  // padded coordinates of the box origin
    y0 = sg.y0 + kPadT - C::R;
    z = sg.z0 - C::R < 0 ? sg.z0 - C::R + int(a.nz) : sg.z0 - C::R;
    lp = 0;
    np = sg.len + 2 * C::R;
  }
  __device__ __forceinline__ void issue_next(double* ring, uint64_t* bars, int stage, const Args3D& a,
                                             const CUtensorMap* tm) {
    using SM = ChfSmem<C, 1>;
    if (u < uend) {
      mbar_arrive_expect_tx(&bars[stage], SM::STAGE_BYTES);
#pragma unroll
      for (int q = 0; q < kTmaSplit; ++q)  // the box: C::ROWS / kTmaSplit rows
        tma_load_3d_hint<SK_TMA_HINT>(ring + stage * SM::PLANE + q * (C::ROWS / kTmaSplit) * SM::P, tm, x0,
                                      y0 + q * (C::ROWS / kTmaSplit), z, &bars[stage]);
      z = z + 1 == a.nz ? 0 : z + 1;
      if (++lp == np) {
        u += np - 2 * C::R;
        if (u < uend) start(a);
      }
    }
  }
};

// V = 0: the step. V = 1 (profiling only): same pipeline, loads and stores,
// no stencil arithmetic (the data-movement ceiling of this design).
// OUT 0: write c' to a.v (nx x ny x nz). OUT 1: write c' into the interior of
// a ghost-padded field at a.v and its periodic images into the 2-wide ghost
// frame (the next step's TMA boxes then never wrap). LD 1 / OUT 1 need whole
// tiles (nx % TX == 0, ny % TY == 0). OUT 2 (z-slabs): OUT 0, and the points
// of output planes 0, 1 / nz-2, nz-1 are stored a second time at a.peer_lo /
// a.peer_hi, the z-neighbours' ghost planes (peer memory over NVLink): the
// halo exchange rides on the step's own stores.
template <class C, int V = 0, int LD = 0, int OUT = 0, bool FB = false>
__global__ void __launch_bounds__(C::THREADS, C::MIN_BLOCKS)
    chf3d_kernel(const __grid_constant__ Args3D a, const __grid_constant__ CUtensorMap tmap) {
  constexpr int R = 2, S = C::STAGES;
  static_assert(C::R == 2 && C::PX == 2 && C::PY == 2 && C::TX == 64, "factored CH kernel layout: warp = row pair");
  using SM = ChfSmem<C, LD, FB>;
  constexpr int P = SM::P, PLANE = SM::PLANE, MP = SM::MP;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw + SM::RING_OFS);
  double* mu_ring = ring + S * PLANE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);  // LD 1: one full-barrier per stage

  // static balanced schedule: a contiguous range of (z-chunk, tile, z) units
  // per CTA (measured faster than a dynamic item queue for this kernel)
  const int units = a.tiles_x * a.tiles_y * int(a.nz);
  const int G = gridDim.x, b = blockIdx.x;
  const int per = units / G, rem = units % G;
  const int ubeg = b * per + (b < rem ? b : rem);
  const int uend = ubeg + per + (b < rem ? 1 : 0);
  LoadCursor<C, FB, SM::TAB> lc;
  TmaCursor<C> tc;
  int s_load = 0;
  // programmatic dependent launch: wait for the previous step (which wrote
  // our input) before the first load; the next step is released at the end
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // FULL barrier per stage: TMA (LD 1) completes its bytes on it; with
  // cp.async (LD 0) every thread's copies arrive on it (arrive.noinc), so the
  // data needs no CTA barrier either. Then three step barriers (below).
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&bars[i], LD ? 1 : C::THREADS);
    for (int i = 0; i < 3; ++i) mbar_init(&bars[S + i], C::THREADS / 32);  // step barriers: one arrival per warp
    fence_mbar_init();
  }
  __syncthreads();
  // LD 0: issue the next plane into stage `st` (this thread's copies) and arm its FULL barrier
  auto cp_issue = [&](int st) {
    if (lc.u < lc.uend) {
      lc.issue_next(ring, st, a);
      cp_async_arrive_noinc(&bars[st]);
    }
  };
  if constexpr (LD == 0) {
    lc.u = ubeg;
    lc.uend = uend;
    if (ubeg < uend) lc.start(a, ring);
#pragma unroll 1
    for (int k = 0; k < S - 3; ++k) {
      cp_issue(s_load);
      s_load = s_load + 1 == S ? 0 : s_load + 1;
    }
  } else {
    if (threadIdx.x == 0) {  // the producer
      tc.u = ubeg;
      tc.uend = uend;
      if (ubeg < uend) tc.start(a);
      for (int k = 0; k < S - 3; ++k) tc.issue_next(ring, bars, k, a, &tmap);
    }
    s_load = S - 3;
  }

  const int lane = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int cofs = (2 * ty + R) * P + 2 * lane + SM::XO;  // own point (row 0, column 0) in a c stage
  const int mofs = (2 * ty + 1) * MP + 2 * lane + 2;  // own point in a mu slot
  const int64_t opx = OUT == 1 ? a.nx + 2 * kPadL : a.nx, opp = opx * (OUT == 1 ? a.ny + 2 * kPadT : a.ny);  // output pitches
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
    ex_c = (ry + R) * P + rx + SM::XO;
    ex_m = (ry + 1) * MP + rx + 2;
  }

  double Cz[3][4], M[3][4];  // own c of plane j in Cz[j % 3], own mu of plane j in M[j % 3]; point 2 * row + col
  int s_k = 0;               // stage of c-plane k
  uint32_t ph = 0;           // LD 1: parity of the current use of stage s_k
  int ms = 0;                // MU_SLOTS 4: mu slot of plane k-1 (plane k-2: ms - 1 mod 4)
  constexpr bool kLateWait = SM::MU_SLOTS >= 4;
  // LD 1: split-phase step barrier instead of __syncthreads. Every warp
  // arrives on step barrier t % 3 once its mu slot and border points of step
  // t are written (its reads of the c stages of step t are done by then),
  // and waits for step t-1's barrier after loading its own c of step t,
  // before it overwrites the mu slot its neighbours read in step t-2: the
  // output of step t-1 (computed after that arrival) is the slack, so warps
  // drift instead of idling at a full-CTA barrier. Three rotating barriers
  // (the mu ring's three slots) keep every reuse ordered transitively.
  uint64_t* stepbar = bars + S;
  int sb = 0;                // t % 3
  uint32_t sph = 0;          // (t / 3) & 1
  bool started = false;      // t > 0
  for (int u = ubeg; u < uend; ) {
    const Seg sg = seg_of<C>(a, u, uend);
    u += sg.len;
    const int64_t gx0 = sg.x0 + 2 * lane, gy0 = sg.y0 + 2 * ty;
    const bool row0 = gy0 < a.ny, row1 = gy0 + 1 < a.ny;
    const bool vec_ok = a.bulk_ok && gx0 + 2 <= a.nx;
    double* outp = a.v + int64_t(sg.z0) * opp + (gy0 + (OUT == 1 ? kPadT : 0)) * opx + gx0 + (OUT == 1 ? kPadL : 0);
    // OUT 1: periodic images in the ghost frame: columns 0..3 and nx-4..nx-1
    // (whole 32 B sectors: no partial-sector writes), rows 0..g-1 and ny-g..ny-1
    // (g = a.ghost = 2)
    const int64_t gdx_ = OUT == 1 ? (gx0 < 4 ? a.nx : (gx0 >= a.nx - 4 ? -a.nx : 0)) : 0;
    const int64_t gdy_ = OUT == 1 ? (gy0 < a.ghost ? a.ny : (gy0 >= a.ny - a.ghost ? -a.ny : 0)) * opx : 0;
    const int64_t gdx = gdx_, gdy = gdy_;
    const int np = sg.len + 2 * R;
    int zo = sg.z0;  // OUT 2: the output plane the next store goes to
    (void)zo;

    // one step: plane k landed; DO_MU: mu of plane k-1; DO_OUT: output plane k-2
    auto step = [&](auto kk_t, auto mu_t, auto out_t) {
      constexpr int K = decltype(kk_t)::value;  // k % 3
      constexpr bool DO_MU = decltype(mu_t)::value, DO_OUT = decltype(out_t)::value;
      constexpr int C0 = K, C1 = (K + 2) % 3, C2 = (K + 1) % 3;  // c of planes k, k-1, k-2
      constexpr int M1 = (K + 2) % 3, M2 = (K + 1) % 3, M3 = K;  // mu of planes k-1, k-2, k-3
      (void)M2;
      (void)M3;
      const int s_iss = s_load;  // the stage refilled in this step (plane k-3's)
      mbar_wait(&bars[s_k], ph);  // plane k landed
      sk_jitter(10);
      s_load = s_load + 1 == S ? 0 : s_load + 1;
      const int s_k1 = s_k == 0 ? S - 1 : s_k - 1;   // stage of plane k-1
      const int s_k2 = s_k1 == 0 ? S - 1 : s_k1 - 1;  // stage of plane k-2
      {
        const double* cn = ring + s_k * PLANE + cofs;
        const double2 r0 = ld2(cn), r1 = ld2(cn + P);
        Cz[C0][0] = r0.x; Cz[C0][1] = r0.y; Cz[C0][2] = r1.x; Cz[C0][3] = r1.y;
      }
      // neighbour values of the output's mu plane (k-2), issued first: they
      // only depend on the previous step's mu slot and the own mu registers
      double olf0 = 0, olf1 = 0, ort0 = 0, ort1 = 0;
      double2 oup = make_double2(0, 0), odn = make_double2(0, 0);
      auto out_neighbours = [&]() {
        const double* m2 = M[M2];
        const double* mb = mu_ring + (SM::MU_SLOTS == 3 ? M2 : (ms == 0 ? SM::MU_SLOTS - 1 : ms - 1)) * SM::MU_PLANE + mofs;  // plane k-2
        olf0 = __shfl_up_sync(0xffffffffu, m2[1], 1);
        olf1 = __shfl_up_sync(0xffffffffu, m2[3], 1);
        ort0 = __shfl_down_sync(0xffffffffu, m2[0], 1);
        ort1 = __shfl_down_sync(0xffffffffu, m2[2], 1);
        if (lane == 0) { olf0 = mb[-1]; olf1 = mb[MP - 1]; }
        if (lane == 31) { ort0 = mb[2]; ort1 = mb[MP + 2]; }
        oup = ld2(mb - MP);
        odn = ld2(mb + 2 * MP);
      };
      if constexpr (!kLateWait) {  // all warps past step t-1: the mu slot written below is free
        sk_jitter(11);
#ifndef SK_RACE_SELFTEST_DROP_STEP_WAIT  // tools/race_jitter.py: proves the detector sees a missing wait
        if (started) mbar_wait(&stepbar[sb == 0 ? 2 : sb - 1], sb == 0 ? sph ^ 1u : sph);
#endif
      }
      if constexpr (LD == 0) cp_issue(s_iss);  // stage of plane k-3 is free (last read at step t-1)
      if constexpr (DO_MU && V == 1) {
#pragma unroll
        for (int i = 0; i < 4; ++i) M[M1][i] = Cz[C1][i];
      } else if constexpr (DO_MU) {
        const double* cb = ring + s_k1 * PLANE + cofs;  // c, plane k-1
        const double* c1 = Cz[C1];
        const double* zp = Cz[C0];
        const double* zm = Cz[C2];
        double lf0 = __shfl_up_sync(0xffffffffu, c1[1], 1), lf1 = __shfl_up_sync(0xffffffffu, c1[3], 1);
        double rt0 = __shfl_down_sync(0xffffffffu, c1[0], 1), rt1 = __shfl_down_sync(0xffffffffu, c1[2], 1);
        if (lane == 0) { lf0 = cb[-1]; lf1 = cb[P - 1]; }
        if (lane == 31) { rt0 = cb[2]; rt1 = cb[P + 2]; }
        const double2 up = ld2(cb - P), dn = ld2(cb + 2 * P);
        // 6-neighbour sums: (((left + right) + (up + down)) + z-1) + z+1 (the
        // plane that arrived last enters last: short dependency chains)
        const double s00 = (((lf0 + c1[1]) + (up.x + c1[2])) + zm[0]) + zp[0];
        const double s01 = (((c1[0] + rt0) + (up.y + c1[3])) + zm[1]) + zp[1];
        const double s10 = (((lf1 + c1[3]) + (c1[0] + dn.x)) + zm[2]) + zp[2];
        const double s11 = (((c1[2] + rt1) + (c1[1] + dn.y)) + zm[3]) + zp[3];
        double* m1 = M[M1];
        m1[0] = fma(a.kl1, s00, fma(a.kl0, c1[0], poly3(c1[0], a.chem)));
        m1[1] = fma(a.kl1, s01, fma(a.kl0, c1[1], poly3(c1[1], a.chem)));
        m1[2] = fma(a.kl1, s10, fma(a.kl0, c1[2], poly3(c1[2], a.chem)));
        m1[3] = fma(a.kl1, s11, fma(a.kl0, c1[3], poly3(c1[3], a.chem)));
        double* mb = mu_ring + (SM::MU_SLOTS == 3 ? M1 : ms) * SM::MU_PLANE + mofs;  // plane k-1
        *reinterpret_cast<double2*>(mb) = make_double2(m1[0], m1[1]);
        *reinterpret_cast<double2*>(mb + MP) = make_double2(m1[2], m1[3]);
      }
      auto border_mu = [&]() {
        if constexpr (DO_MU && V == 0) {
          if (has_ex) {  // one border point of the mu tile (needed from the next step on)
            const double* rb = ring + s_k1 * PLANE + ex_c;
            const double cc = rb[0];
            const double sr =
                (((rb[-1] + rb[1]) + (rb[-P] + rb[P])) + ring[s_k2 * PLANE + ex_c]) + ring[s_k * PLANE + ex_c];
            mu_ring[(SM::MU_SLOTS == 3 ? M1 : ms) * SM::MU_PLANE + ex_m] =
                fma(a.kl1, sr, fma(a.kl0, cc, poly3(cc, a.chem)));
          }
        }
      };
      {
        border_mu();
        sk_jitter(12);
        __syncwarp();
        if (lane == 0) mbar_arrive(&stepbar[sb]);  // this warp is done with step t's stages and mu slot
        if constexpr (kLateWait) {  // 4 mu slots: the slot written above was last read in step t-3
          if (started) mbar_wait(&stepbar[sb == 0 ? 2 : sb - 1], sb == 0 ? sph ^ 1u : sph);
        }
        if constexpr (LD == 1) {
          if (threadIdx.x == 0) {  // stage of plane k-3 is free (last read at step t-1)
            sk_jitter(13);
            tma_war_fence();
            tc.issue_next(ring, bars, s_iss, a, &tmap);
          }
        }
        if constexpr (DO_OUT && V == 0) out_neighbours();
        started = true;
        if (++sb == 3) {
          sb = 0;
          sph ^= 1u;
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
          const double s00 = (((olf0 + m2[1]) + (oup.x + m2[2])) + m3[0]) + m1[0];
          const double s01 = (((m2[0] + ort0) + (oup.y + m2[3])) + m3[1]) + m1[1];
          const double s10 = (((olf1 + m2[3]) + (m2[0] + odn.x)) + m3[2]) + m1[2];
          const double s11 = (((m2[2] + ort1) + (m2[1] + odn.y)) + m3[3]) + m1[3];
          o[0] = fma(a.wl1, s00, fma(a.wl0, m2[0], c2[0]));
          o[1] = fma(a.wl1, s01, fma(a.wl0, m2[1], c2[1]));
          o[2] = fma(a.wl1, s10, fma(a.wl0, m2[2], c2[2]));
          o[3] = fma(a.wl1, s11, fma(a.wl0, m2[3], c2[3]));
        }
        if constexpr (OUT == 1) {  // whole tiles: every point exists
          store_f64x2<Mode::CahnHilliard>(outp, o[0], o[1]);
          store_f64x2<Mode::CahnHilliard>(outp + opx, o[2], o[3]);
          if (gdx) {
            store_f64x2<Mode::CahnHilliard>(outp + gdx, o[0], o[1]);
            store_f64x2<Mode::CahnHilliard>(outp + gdx + opx, o[2], o[3]);
          }
          if (gdy) {
            store_f64x2<Mode::CahnHilliard>(outp + gdy, o[0], o[1]);
            store_f64x2<Mode::CahnHilliard>(outp + gdy + opx, o[2], o[3]);
            if (gdx) {
              store_f64x2<Mode::CahnHilliard>(outp + gdx + gdy, o[0], o[1]);
              store_f64x2<Mode::CahnHilliard>(outp + gdx + gdy + opx, o[2], o[3]);
            }
          }
        } else {
          double* dsts[2] = {outp, nullptr};
          if constexpr (OUT == 2) {  // the neighbours' ghost planes: the same point again
            double* pb = zo < 2 ? a.peer_lo : (zo >= a.nz - 2 ? a.peer_hi : nullptr);
            if (pb) dsts[1] = pb + (zo < 2 ? zo : zo - (a.nz - 2)) * opp + (gy0 * a.nx + gx0);
            ++zo;
          }
#pragma unroll
          for (int d = 0; d < (OUT == 2 ? 2 : 1); ++d) {
            double* op = dsts[d];
            if (!op) continue;
            if (vec_ok) {
              if (row0) store_f64x2<Mode::CahnHilliard>(op, o[0], o[1]);
              if (row1) store_f64x2<Mode::CahnHilliard>(op + a.nx, o[2], o[3]);
            } else {
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                if (row0 && gx0 + i < a.nx) op[i] = o[i];
                if (row1 && gx0 + i < a.nx) op[a.nx + i] = o[2 + i];
              }
            }
          }
        }
        outp += opp;
      }
      if (++s_k == S) {
        s_k = 0;
        ph ^= 1u;
      }
      if constexpr (SM::MU_SLOTS != 3) ms = ms + 1 == SM::MU_SLOTS ? 0 : ms + 1;
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
  asm volatile("griddepcontrol.launch_dependents;");
  cp_async_wait_all();
}

}  // namespace sk
