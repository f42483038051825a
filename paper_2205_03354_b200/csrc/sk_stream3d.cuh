// 3D streaming stencil kernel (sm_100a): composed 25/73-point apply and the
// fused explicit Cahn-Hilliard step.
//
// Work decomposition: the grid is cut into TX x TY column tiles; the unit of
// work is one OUTPUT PLANE of one tile. The tiles*nz units are split into
// gridDim.x contiguous, equal ranges (MIN_BLOCKS persistent CTAs per SM: a
// single balanced wave); a range walks z inside a tile and may continue into
// the next tile (a new "segment", whose first 2R planes re-prime the
// pipeline). With Args3D::zrot the tile columns are rotated in z so that all
// CTAs stream the same planes at the same time (seg_of).
//
// Pipeline: every thread issues its share of each input plane ((TY+2R) x
// (TX+2R) doubles, periodic wrap or boundary map: PlaneLoader) as cp.async
// into a STAGES-deep shared-memory ring, STAGES-1 planes ahead; one barrier
// per plane. Each thread owns PX x PY points and, per input plane:
//   1. loads the (PY+2R) rows of its window as 128-bit shared loads,
//   2. accumulates in-plane ORBIT SUMS (centre, A1 = 4 axis neighbours at 1,
//      D11 = 4 diagonals, A2, and for R=4 D21, D22, A3, A4) — the first member
//      of each sum is assigned, the rest added, so there are no zero-inits,
//   3. forms the R+1 slice sums S_d = sum over orbits with |dz| = d of w * sum,
//   4. pushes them into a register queue of 2R+1 output planes (slot of an
//      output is fixed; the rotation is static because the plane loop is
//      unrolled by 2R+1), the deepest slot being ASSIGNED.
// An output plane completes R planes after its own input plane; it is stored
// with 128-bit streaming stores.
//
// Cahn-Hilliard mode adds, on the same loaded values, g = f'(c) as a cubic
// polynomial (3 FMA; f'(c) = 2 rho (c-a)(c-b)(2c-a-b) expanded on the host)
// and the 7-point Laplacian of g (S0 += wl0 g + wl1 sum_A1 g, S1 += wl1 g),
// with B, L weights pre-scaled by -dt M kappa and dt M; output = c + queue.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "sk_cgstate.cuh"
#include "sk_common.cuh"
#include "sk_stencil_kernels.cuh"

namespace sk {

template <int R_, int TX_, int TY_, int PX_, int PY_, int STAGES_, int MINB_>
struct Cfg3 {
  static constexpr int R = R_, TX = TX_, TY = TY_, PX = PX_, PY = PY_, STAGES = STAGES_, MIN_BLOCKS = MINB_;
  static constexpr int WIDTH = TX + 2 * R;  // loaded columns x0-R .. x0+TX+R-1
  static constexpr int ROWS = TY + 2 * R;
  // Row pitch a multiple of 128 B and column 0 at byte 128 - 8R (mod 128):
  // with x0 % 16 == 0 and nx % 16 == 0 every 128-byte global line of a row
  // lands in ONE 128-byte shared line, so a 16-byte cp.async warp costs 4
  // shared wavefronts instead of ~15 (measured, ncu source page).
  static constexpr int PITCH = (WIDTH + 15) / 16 * 16;
  static constexpr int RING_OFS = 128 + (128 - (8 * R) % 128) % 128;  // bytes from smem base
  static constexpr int PLANE = ROWS * PITCH;  // doubles
  static constexpr int CONSUMERS = (TX / PX) * (TY / PY);
  static_assert(CONSUMERS % 32 == 0, "consumer threads must be whole warps");
  static_assert(PX % 2 == 0 && R % 2 == 0, "128-bit row loads need even PX and R");
  static constexpr int THREADS = CONSUMERS;
  static constexpr int TABLE_BYTES = ROWS * WIDTH * 8;  // boundary map of the 8-byte fallback loader
  static constexpr int SMEM_BYTES = RING_OFS + STAGES * PLANE * 8 + TABLE_BYTES;
  static constexpr int Q = 2 * R + 1;
};

struct Args3D {
  const double* __restrict__ u;
  double* __restrict__ v;
  int64_t nx, ny, nz;
  int tiles_x, tiles_y;
  double w[8];       // orbit weights (pre-scaled)
  double wl0, wl1;   // CH: 7-point Laplacian (pre-scaled by dt M)
  double kl0, kl1;   // factored CH: 7-point Laplacian pre-scaled by -kappa (mu = f' - kappa L c)
  Poly3 chem;        // CH: f'
  int bulk_ok;       // even nx, tiles fit, aligned, nx*ny < 2^31: 16-byte copies, int32 offsets
  int bc[3];         // boundary kind per axis (nx, ny, nz are unknown counts); bulk path: periodic only
  int z_ghosted;     // slab mode: planes -R..-1 and nz..nz+R-1 exist in memory around u (no z wrap)
  CgState* cg;       // PQ kernels (matrix-free CG, sk_cg.cu): q = A p fused with p.q -> alpha
  double* cg_partials;
  int zchunk;        // unit order (z-chunk, tile [y fastest], z): concurrent CTAs stay close in z
  int ghost;         // chf3d OUT 1: ghost rows written on each side (2)
  int zrot;          // periodic z, zchunk = nz: every tile column is rotated so CTA range starts sit at
                     // the same planes in every column (seg_of): neighbour tiles are streamed in phase
  int64_t in_pitch;  // != 0: u is a ghost-padded field (row pitch in_pitch, plane pitch in_plane, u at the
  int64_t in_plane;  // interior origin, every halo point present): 16-byte loads without wrap (matrix-free CG)
  double* peer_lo;   // chf3d OUT 2 (slab step with fused halo stores): output planes 0, 1 also go here,
  double* peer_hi;   // planes nz-2, nz-1 here (the z-neighbours' ghost planes; either may be null)
};

// Host: tiles, persistent grid (min_blocks CTAs per SM, each a balanced
// contiguous unit range) and the z-chunk of the unit order. Returns 0 when the
// unit count does not fit the kernels' 32-bit unit cursor (> 2^31 tile-planes,
// i.e. > 2^41 points: beyond any device memory).
template <class C>
inline int64_t persistent_grid(Args3D& a, int num_sms, bool lockstep) {
  a.tiles_x = int((a.nx + C::TX - 1) / C::TX);
  a.tiles_y = int((a.ny + C::TY - 1) / C::TY);
  if (a.nx * a.ny >= (int64_t(1) << 31)) a.bulk_ok = 0;  // int32 in-plane offsets
  const int64_t tiles = int64_t(a.tiles_x) * a.tiles_y;
  const int64_t units = tiles * a.nz;
  if (units >= (int64_t(1) << 31) || a.nz >= (int64_t(1) << 31)) return 0;
  const int64_t slots = int64_t(num_sms) * C::MIN_BLOCKS;
  int64_t grid = slots < units ? slots : units;
  if (lockstep) {
    // lockstep: one CTA per (tile, z-chunk) with the most z-chunks
    // that still fit one wave; every CTA starts at a chunk top, so the tiles
    // around a halo are read at the same z at about the same time and the
    // halo rows come from L2 instead of HBM.
    for (int64_t k = a.nz; k >= 1; --k)
      if (a.nz % k == 0 && tiles * k <= slots && a.nz / k >= 2 * C::R + 1) {
        a.zchunk = int(a.nz / k);
        return tiles * k;
      }
  }
  if (a.zrot) {  // rotated columns (seg_of): whole columns are the items
    a.zchunk = int(a.nz);
    return grid;
  }
  // balanced: the smallest z-chunk divisor covering one CTA's equal share
  const int64_t share = (units + grid - 1) / grid;
  a.zchunk = int(a.nz);
  for (int64_t d = 1; d <= a.nz; ++d)
    if (a.nz % d == 0 && d >= share) {
      a.zchunk = int(d);
      break;
    }
  return grid;
}

// Unit u -> segment (tile, first plane z0, planes left in this item).
struct Seg {
  int x0, y0, z0, len;
};
template <class C>
__device__ __forceinline__ Seg seg_of(const Args3D& a, int u, int uend) {
  const int item = u / a.zchunk, k = u - item * a.zchunk;
  if (a.zrot) {
    // Column `item` (zchunk = nz) is walked from plane -r (mod nz), r = the
    // offset of the first CTA range that starts inside it, so every range
    // start maps to plane 0 + m * (units / G) in EVERY column: at any moment
    // all CTAs stream the same planes of their columns and a tile's halo
    // rows are read by its neighbours while they sit in L2. Balance is
    // unchanged (same contiguous ranges); a segment ends at the z wrap.
    const int nz = int(a.nz), T = item * nz, G = gridDim.x;
    const int units = a.tiles_x * a.tiles_y * nz, per = units / G, rem = units % G;
    int b = (T + per) / (per + 1);  // first range start >= T: ceil(T / (per + 1)) ...
    int ub = b * (per + 1);
    if (b > rem) {                  // ... or past the longer ranges
      b = (T - rem + per - 1) / per;
      ub = b * per + rem;
    }
    const int r = (ub - T) % nz;
    const int z = (k - r) % nz;
    const int tile = item;
    const int ty = tile % a.tiles_y;
    Seg s;
    s.z0 = z < 0 ? z + nz : z;
    s.len = nz - k < uend - u ? nz - k : uend - u;
    if (s.len > nz - s.z0) s.len = nz - s.z0;  // segments stop at the z wrap (output planes stay contiguous)
    s.y0 = ty * C::TY;
    s.x0 = ((tile - ty) / a.tiles_y) * C::TX;
    return s;
  }
  const int tiles = a.tiles_x * a.tiles_y;
  const int zc = item / tiles, tile = item - zc * tiles;
  const int ty = tile % a.tiles_y;  // y fastest: y-neighbour tiles run concurrently
  Seg s;
  s.z0 = zc * a.zchunk + k;
  s.len = a.zchunk - k < uend - u ? a.zchunk - k : uend - u;
  s.y0 = ty * C::TY;
  s.x0 = ((tile - ty) / a.tiles_y) * C::TX;
  return s;
}

// orbit-sum index of in-plane offset (|dx|, |dy|) at radius R; -1: not used
template <int R>
__host__ __device__ constexpr int kind_of(int ax, int ay) {
  const int a = ax > ay ? ax : ay, b = ax > ay ? ay : ax;
  if (a == 0) return 0;
  if (a == 1 && b == 0) return 1;
  if (a == 1 && b == 1) return 2;
  if (a == 2 && b == 0) return 3;
  if (R >= 4) {
    if (a == 2 && b == 1) return 4;
    if (a == 2 && b == 2) return 5;
    if (a == 3 && b == 0) return 6;
    if (a == 4 && b == 0) return 7;
  }
  return -1;
}
template <int R>
__host__ __device__ constexpr int num_kinds() { return R >= 4 ? 8 : 4; }

// Every thread of the CTA issues its share of one plane buffer as 16-byte
// cp.async (LDGSTS, lane-parallel, deep memory-level parallelism); periodic
// wrap per pair (pairs never straddle the wrap: nx, x0 and R are even).
// Fallback (odd nx, tiny or unaligned grids): 8-byte copies, modulo wrap.
// A thread's share of a plane buffer is the same set of (row, pair) slots for
// every plane of a segment: the wrapped source pointers are computed once per
// segment and advanced by one plane per issue, the shared-memory addresses
// are precomputed, so a 16-byte pair costs an add, a 64-bit add and an LDGSTS.
// FB: the 8-byte fallback loader (kernels are instantiated for both and
// launched with FB = !bulk_ok, so the 16-byte path carries no fallback code).
// TAB: offset of the fallback's boundary-map table from the ring (doubles;
// the stream kernels keep it right after the ring).
template <class C, bool FB, int TAB = C::STAGES * C::PLANE>
struct PlaneLoader {
  static constexpr int HP = C::WIDTH / 2;  // 16-byte chunks per row
  static constexpr int NP = (C::ROWS * HP + C::THREADS - 1) / C::THREADS;
  const double* plane;  // the next plane to load
  int off[NP];          // wrapped in-plane source offset of each of this thread's chunks (elements)
  uint32_t dst[NP];     // its shared address in stage 0 (bytes)
  int x0, y0;           // tile origin (8-byte fallback)

  __device__ __forceinline__ static bool used(int k) {
    return k + 1 < NP || int(threadIdx.x) + k * C::THREADS < C::ROWS * HP;
  }
  // 8-byte fallback: the tile's boundary map (it depends on x0, y0 only) is
  // tabulated once per segment at ring + TAB: entry i = (source, shared
  // offset), source = in-plane offset o >= 0 (copy), -1 (boundary zero) or
  // -2 - o (odd reflection: negated copy). Each thread writes and reads only
  // its own entries (i = tid mod THREADS): no barrier.
  static constexpr int NT = C::ROWS * C::WIDTH;
  __device__ __forceinline__ static int2* table(const double* ring) {
    return reinterpret_cast<int2*>(const_cast<double*>(ring) + TAB);
  }
  __device__ __forceinline__ static bool tabulated(const Args3D& a) { return a.nx * a.ny < (int64_t(1) << 29); }
  // first plane to load: gz (already wrapped)
  __device__ __forceinline__ void setup(const Args3D& a, const double* ring, int x0_, int y0_, int gz) {
    constexpr int R = C::R;
    x0 = x0_;
    y0 = y0_;
    plane = a.u + int64_t(gz) * (a.in_pitch ? a.in_plane : a.nx * a.ny);
    if constexpr (!FB) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const int i = threadIdx.x + k * C::THREADS;
        off[k] = 0;
        dst[k] = smem_u32(ring);
        if (used(k)) {
          const int r = i / HP, c = 2 * (i - r * HP);
          if (a.in_pitch) {  // ghost-padded input: the halo exists around the field
            off[k] = int((y0 - R + r) * a.in_pitch + (x0 - R + c));
          } else {
            const int64_t gy = wrap1(y0 - R + r, a.ny), gx = wrap1(x0 - R + c, a.nx);
            off[k] = int(gy * a.nx + gx);  // bulk path: nx * ny < 2^31
          }
          dst[k] = smem_u32(ring + r * C::PITCH + c);
        }
      }
    } else if (tabulated(a)) {
      int2* t = table(ring);
      for (int i = threadIdx.x; i < NT; i += C::THREADS) {
        const int r = i / C::WIDTH, c = i - r * C::WIDTH;
        double f = 1.0;
        const int64_t gy = bc_map(y0 - R + r, a.ny, a.bc[1], f), gx = bc_map(x0 - R + c, a.nx, a.bc[0], f);
        const int o = int(gy * a.nx + gx);
        t[i] = make_int2(f == 1.0 ? o : (f == 0.0 ? -1 : -2 - o), r * C::PITCH + c);
      }
    }
  }

  // load plane `plane` (z = gz) into stage `stage`, then step to the next
  // plane (back to z = 0 after the last one: periodic z)
  __device__ __forceinline__ void issue(double* ring, int stage, const Args3D& a, int gz, int gze) {
    constexpr int R = C::R;
    if constexpr (!FB) {
      const uint32_t soff = uint32_t(stage) * (C::PLANE * 8);
#pragma unroll
      for (int k = 0; k < NP; ++k)
        if (used(k))
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst[k] + soff), "l"(plane + off[k])
                       : "memory");
    } else {  // fallback: 8-byte copies, any boundary kind (odd nx, tiny, unaligned or non-periodic grids)
      double* buf = ring + stage * C::PLANE;
      double fz = 1.0;
      const int64_t pz = a.z_ghosted ? gze : bc_map(gze, a.nz, a.bc[2], fz);  // gze: the unwrapped plane index
      const double* src = a.u + pz * a.nx * a.ny;
      if (fz == 1.0 && tabulated(a)) {
        const int2* t = table(ring);
        for (int i = threadIdx.x; i < NT; i += C::THREADS) {
          const int2 e = t[i];
          if (e.x >= 0)
            cp_async8(buf + e.y, src + e.x);
          else
            buf[e.y] = e.x == -1 ? 0.0 : -__ldg(src + (-2 - e.x));  // boundary zero / odd reflection
        }
      } else {  // planes mirrored in z (or huge planes): map every element
        for (int i = threadIdx.x; i < C::ROWS * C::WIDTH; i += C::THREADS) {
          const int r = i / C::WIDTH, c = i - r * C::WIDTH;
          double f = fz;
          const int64_t gy = bc_map(y0 - R + r, a.ny, a.bc[1], f), gx = bc_map(x0 - R + c, a.nx, a.bc[0], f);
          double* d = buf + r * C::PITCH + c;
          if (f == 1.0)
            cp_async8(d, src + gy * a.nx + gx);
          else
            *d = f == 0.0 ? 0.0 : f * __ldg(src + gy * a.nx + gx);  // boundary zero / odd reflection
        }
      }
    }
    plane = (!a.z_ghosted && gz + 1 == a.nz) ? a.u : plane + (a.in_pitch ? a.in_plane : a.nx * a.ny);
  }
};

__device__ __forceinline__ double2 lds128(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}

// Per-plane evaluation for one thread: slice sums sl[d][pt], d = 0..R, and
// (CH) the centre values of the plane at the owned points.
template <Mode M, class C>
__device__ __forceinline__ void plane_slices(const double* base, const Args3D& a, double (&sl)[C::R + 1][C::PX * C::PY],
                                             double (&cen)[C::PX * C::PY]) {
  constexpr int R = C::R, PX = C::PX, PY = C::PY, NK = num_kinds<R>();
  constexpr int W = PX + 2 * R;  // window width per row
  double sums[PY][PX][NK];
  double gc[PY][PX], ga1[PY][PX];  // CH: g at the point, sum of g over A1
#pragma unroll
  for (int r = -R; r < PY + R; ++r) {
    // which columns of this row does any owned point need?
    double row[W];
    double grow[W];
#pragma unroll
    for (int k = 0; k < W; k += 2) {
      bool need = false;
#pragma unroll
      for (int j = 0; j < PY; ++j)
#pragma unroll
        for (int i = 0; i < PX; ++i)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int dx = k + e - R - i, dy = r - j;
            const int ax = dx < 0 ? -dx : dx, ay = dy < 0 ? -dy : dy;
            if (ax <= R && ay <= R && kind_of<R>(ax, ay) >= 0) need = true;
          }
      if (need) {
        const double2 v = lds128(base + r * C::PITCH + k - R);
        row[k] = v.x;
        row[k + 1] = v.y;
      } else {
        row[k] = row[k + 1] = 0.0;
      }
    }
    if (M == Mode::CahnHilliard) {
#pragma unroll
      for (int k = 0; k < W; ++k) {
        bool need = false;
#pragma unroll
        for (int j = 0; j < PY; ++j)
#pragma unroll
          for (int i = 0; i < PX; ++i) {
            const int dx = k - R - i, dy = r - j;
            const int ax = dx < 0 ? -dx : dx, ay = dy < 0 ? -dy : dy;
            if (ax + ay <= 1) need = true;
          }
        grow[k] = need ? poly3(row[k], a.chem) : 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      const int dy = r - j, ay = dy < 0 ? -dy : dy;
      if (ay > R) continue;
#pragma unroll
      for (int i = 0; i < PX; ++i) {
#pragma unroll
        for (int dx = -R; dx <= R; ++dx) {
          const int ax = dx < 0 ? -dx : dx;
          const int kd = kind_of<R>(ax, ay);
          if (kd < 0) continue;
          const double v = row[i + dx + R];
          // first member of orbit (a, b), a >= b, in (dy, dx) scan order is (-a, -b)
          const int oa = ax > ay ? ax : ay, ob = ax > ay ? ay : ax;
          const bool first = (dy == -oa && dx == -ob);
          if (first) sums[j][i][kd] = v;
          else sums[j][i][kd] += v;
          if (M == Mode::CahnHilliard) {
            if (kd == 0) gc[j][i] = grow[i + dx + R];
            if (kd == 1) {
              if (first) ga1[j][i] = grow[i + dx + R];
              else ga1[j][i] += grow[i + dx + R];
            }
          }
        }
      }
    }
  }
  const double* w = a.w;
#pragma unroll
  for (int j = 0; j < PY; ++j)
#pragma unroll
    for (int i = 0; i < PX; ++i) {
      const double* s = sums[j][i];
      const int pt = j * PX + i;
      cen[pt] = s[0];
      if constexpr (R == 2) {
        sl[0][pt] = fma(w[3], s[3], fma(w[2], s[2], fma(w[1], s[1], w[0] * s[0])));
        sl[1][pt] = fma(w[2], s[1], w[1] * s[0]);
        sl[2][pt] = w[3] * s[0];
      } else {
        sl[0][pt] = fma(w[7], s[7], fma(w[6], s[6], fma(w[5], s[5], fma(w[4], s[4], fma(w[3], s[3],
                        fma(w[2], s[2], fma(w[1], s[1], w[0] * s[0])))))));
        sl[1][pt] = fma(w[4], s[3], fma(w[2], s[1], w[1] * s[0]));
        sl[2][pt] = fma(w[5], s[3], fma(w[4], s[1], w[3] * s[0]));
        sl[3][pt] = w[6] * s[0];
        sl[4][pt] = w[7] * s[0];
      }
      if (M == Mode::CahnHilliard) {
        sl[0][pt] = fma(a.wl1, ga1[j][i], fma(a.wl0, gc[j][i], sl[0][pt]));
        sl[1][pt] = fma(a.wl1, gc[j][i], sl[1][pt]);
      }
    }
}

#ifndef SK_A25_TY
#define SK_A25_TY 8  // 64x8 tiles, 4 CTAs/SM (measured 59.5 us at 256^3; 64x16 x2: 60.7 us)
#define SK_A25_S 6
#define SK_A25_MINB 4
#endif
using Cfg3R2 = Cfg3<2, 64, SK_A25_TY, 2, 2, SK_A25_S, SK_A25_MINB>;    // 25-point apply
#ifndef SK_CH3_TY  // experiments: -DSK_CH3_TY=.. -DSK_CH3_S=.. -DSK_CH3_MINB=..
#define SK_CH3_TY 8
#define SK_CH3_S 8
#define SK_CH3_MINB 2  // 64x8 tiles, 2 CTAs/SM, 198 registers, no spills (64x16 x2 spilled: 96 us; x1: 82 us; this: 71 us)
#endif
using Cfg3CH = Cfg3<2, 64, SK_CH3_TY, 2, 2, SK_CH3_S, SK_CH3_MINB>;    // 3D CH (7-point L f' + 25-point B)
#ifndef SK_A73_TY
#define SK_A73_TY 16
#define SK_A73_PX 2
#define SK_A73_PY 2
#define SK_A73_S 8
#define SK_A73_MINB 1
#endif
using Cfg3R4 = Cfg3<4, 64, SK_A73_TY, SK_A73_PX, SK_A73_PY, SK_A73_S, SK_A73_MINB>;    // 73-point apply
// 73-point apply on the 16-byte (periodic) path: 64x8 tiles, 10 stages, 2
// CTAs/SM — with the rotated-column schedule the extra halo rows come from
// L2, and two independent CTAs per SM hide each other's barrier: 108.6 ->
// 96.9 us at 256^3. The boundary-mapped loader (clamped / simply supported)
// keeps 64x16 x 1 CTA (its per-segment table favours big tiles: 204 vs 241 us).
#ifndef SK_A73P_TY
#define SK_A73P_TY 8
#define SK_A73P_S 10
#define SK_A73P_MINB 2
#endif
using Cfg3R4P = Cfg3<4, 64, SK_A73P_TY, 2, 2, SK_A73P_S, SK_A73P_MINB>;
#ifndef SK_CHP_TY  // cp.async path (first step of a chunk, remainders, grids without whole TMA tiles):
#define SK_CHP_TY 16  // 64x16 tiles, 2 CTAs/SM + rotated columns: 68.3 -> 65.2 us/step at 256^3
#define SK_CHP_S 6
#define SK_CHP_MINB 2
#endif
using CfgChf3 = Cfg3<2, 64, SK_CHP_TY, 2, 2, SK_CHP_S, SK_CHP_MINB>;   // factored 3D CH (sk_chf3d.cuh), cp.async loads
#ifndef SK_CHT_TY
// 64x16 tiles, 7 stages, 2 CTAs/SM (with the rotated-column schedule the
// halo rows come from L2, so smaller tiles cost little and two CTAs hide
// each other's per-plane barrier): 58.6 us/step at 256^3, against 61.6 for
// 64x32 x 8 stages x 1 CTA, 58.9 for 6 stages, 77.8 for 4
#define SK_CHT_TY 16
#define SK_CHT_S 7
#define SK_CHT_MINB 2
#endif
using CfgChf3T = Cfg3<2, 64, SK_CHT_TY, 2, 2, SK_CHT_S, SK_CHT_MINB>;  // factored 3D CH, TMA loads from ghost-padded fields

// Load cursor: walks the block's segment/plane sequence S-1 planes ahead of
// the compute loop. The per-segment setup (64-bit divisions, wrapped source
// offsets) is out of line so the unrolled plane loop stays lean.
template <class C, bool FB, int TAB = C::STAGES * C::PLANE>
struct LoadCursor {
  int u, uend, lz, lze, lp, np;  // lz: wrapped plane index, lze: unwrapped (non-periodic z)
  PlaneLoader<C, FB, TAB> ld;
  __device__ __forceinline__ void start(const Args3D& a, const double* ring) {
    const Seg seg = seg_of<C>(a, u, uend);
    lze = seg.z0 - C::R;
    lz = (lze < 0 && !a.z_ghosted) ? lze + int(a.nz) : lze;
    ld.setup(a, ring, seg.x0, seg.y0, lz);
    lp = 0;
    np = seg.len + 2 * C::R;
  }
  __device__ __forceinline__ void issue_next(double* ring, int stage, const Args3D& a) {
    if (u < uend) {
      ld.issue(ring, stage, a, lz, lze);
      lz = (lz + 1 == a.nz && !a.z_ghosted) ? 0 : lz + 1;
      ++lze;
      if (++lp == np) {
        u += np - 2 * C::R;
        if (u < uend) start(a, ring);
      }
    }
    cp_async_commit();
  }
};

// PQ (Apply only): one matrix-free CG iteration's q = A p (sk_cg.cu) with the
// p.q reduction in the store epilogue (p re-read from L2 at the output point)
// and alpha = rho / p.q (or "not positive definite") published by the last
// CTA: the separate p.q pass (16 B per unknown) disappears. A no-op once the
// solver has stopped, like the other kernels of the iteration graph.
template <Mode M, class C, bool FB, bool PQ = false>
__global__ void __launch_bounds__(C::THREADS, C::MIN_BLOCKS) stream3d_kernel(const Args3D a) {
  constexpr int R = C::R, Q = C::Q, S = C::STAGES, PX = C::PX, PY = C::PY;
  constexpr int NPT = PX * PY;
  if constexpr (PQ) {
    if (a.cg->status != kCgRunning) return;
  }
  double pq = 0.0;
  (void)pq;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw + C::RING_OFS);

  // balanced contiguous range of units (see seg_of for the unit order)
  const int units = a.tiles_x * a.tiles_y * int(a.nz);
  const int G = gridDim.x, b = blockIdx.x;
  const int per = units / G, rem = units % G;
  const int ubeg = b * per + (b < rem ? b : rem);
  const int uend = ubeg + per + (b < rem ? 1 : 0);

  LoadCursor<C, FB> lc;
  lc.u = ubeg;
  lc.uend = uend;
  if (ubeg < uend) lc.start(a, ring);
  int s_load = 0;  // stage the load cursor fills next
#pragma unroll 1
  for (int k = 0; k < S - 1; ++k) {
    lc.issue_next(ring, s_load, a);
    s_load = s_load + 1 == S ? 0 : s_load + 1;
  }

  const int tx = threadIdx.x % (C::TX / PX), ty = threadIdx.x / (C::TX / PX);
  const int lofs = (ty * PY + R) * C::PITCH + tx * PX + R;  // first owned point in a plane buffer
  const int64_t plane_sz = a.nx * a.ny;
  int s_comp = 0;  // stage of the plane being computed
  double q[Q][NPT];
  double cen[Q][NPT];
  (void)cen;
  for (int u = ubeg; u < uend;) {
    const Seg sg = seg_of<C>(a, u, uend);
    const int64_t gx0 = sg.x0 + tx * PX, gy0 = sg.y0 + ty * PY;
    bool row_ok[PY];
#pragma unroll
    for (int j = 0; j < PY; ++j) row_ok[j] = gy0 + j < a.ny;
    const bool vec_ok = a.bulk_ok && !(a.nx & 1) && gx0 + PX <= a.nx;  // 16-byte stores need even rows (padded input may be odd)
    double* outp = a.v + int64_t(sg.z0) * plane_sz + gy0 * a.nx + gx0;  // output plane z0, first owned point
    const int np = int(sg.len) + 2 * R;
    for (int pb = 0; pb < np; pb += Q) {
#pragma unroll
      for (int st = 0; st < Q; ++st) {
        const int p = pb + st;
        if (p < np) {
          cp_async_wait_group<S - 2>();  // this thread's copies of the plane have landed
          sk_jitter(20);
          __syncthreads();               // ... everyone's, and the previous plane is fully consumed
          lc.issue_next(ring, s_load, a);
          s_load = s_load + 1 == S ? 0 : s_load + 1;
          double sl[R + 1][NPT];
          double cz[NPT];
          plane_slices<M, C>(ring + s_comp * C::PLANE + lofs, a, sl, cz);
          s_comp = s_comp + 1 == S ? 0 : s_comp + 1;
          // input plane p feeds output o = p - R - dz at queue slot (st + t) % Q, t = R - dz;
          // t = 2R is the deepest (first) contribution of an output: assign
#pragma unroll
          for (int t = 0; t < Q; ++t) {
            const int d = t < R ? R - t : t - R;
            const int slot = (st + t) % Q;
#pragma unroll
            for (int i = 0; i < NPT; ++i) {
              if (t == 2 * R) q[slot][i] = sl[d][i];
              else q[slot][i] += sl[d][i];
            }
          }
          if (M == Mode::CahnHilliard) {
#pragma unroll
            for (int i = 0; i < NPT; ++i) cen[st][i] = cz[i];
          }
          if (p >= 2 * R) {  // output plane p - 2R is complete
            const int slot0 = st % Q;
#pragma unroll
            for (int j = 0; j < PY; ++j) {
              if (!row_ok[j]) continue;
              double val[PX];
#pragma unroll
              for (int i = 0; i < PX; ++i) {
                val[i] = q[slot0][j * PX + i];
                if (M == Mode::CahnHilliard) val[i] += cen[(st + R + 1) % Q][j * PX + i];
              }
              double* dst = outp + j * a.nx;
              if (vec_ok) {
#pragma unroll
                for (int i = 0; i < PX; i += 2) store_f64x2<M>(dst + i, val[i], val[i + 1]);
              } else {
#pragma unroll
                for (int i = 0; i < PX; ++i)
                  if (gx0 + i < a.nx) dst[i] = val[i];
              }
              if constexpr (PQ) {
                const double* pp = a.u + (dst - a.v);
#pragma unroll
                for (int i = 0; i < PX; ++i)
                  if (gx0 + i < a.nx) pq = fma(__ldg(pp + i), val[i], pq);
              }
            }
            outp += plane_sz;
          }
        }
      }
    }
    u += sg.len;
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
