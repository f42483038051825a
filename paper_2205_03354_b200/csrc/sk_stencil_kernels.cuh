// Matrix-free composed-stencil kernels for sm_100a (device code).
//
// Both the plain composed apply (v = S u) and the fused explicit
// Cahn-Hilliard step (c' = c + dt M (L f'(c) - kappa B c)) share one
// formulation: a symmetric stencil is a set of ORBITS (all signed axis
// permutations of a representative offset, one weight each), and the stencil
// is evaluated plane by plane along the slowest axis ("streaming axis"):
//
//   out(z) = sum_{dz=-R..R} S_|dz|(z + dz),   S_d = in-plane slice at |dz| = d
//
// Each input plane is read from shared memory ONCE per thread; its R+1 slice
// sums are pushed into a register queue of 2R+1 output planes (2.5D
// blocking). Orbit sums (A_k = 4 axis points at distance k, D_ab = diagonal
// families) are formed with adds and multiplied once per orbit, so the fp64
// op count per point is ~13 (2D 13-pt), ~21 (3D 25-pt), ~49 (3D 73-pt)
// instead of one FMA per stencil entry.
//
// Data movement: tiles (+ radius-R halo) land in shared memory through the
// TMA bulk-copy engine (cp.async.bulk, SASS UBLKCP) one row segment per copy,
// periodic wrap handled by splitting a row into <= 2 contiguous pieces, with
// mbarrier transaction counts. 3D kernels run a warp-specialised ring: one
// producer warp streams planes ahead of 8 consumer warps.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "sk_common.cuh"

namespace sk {

// Orbit layouts (index -> representative offset, sorted |o| descending):
//   2D (class 1, radius 2): 0:(0,0) 1:(1,0) 2:(1,1) 3:(2,0)
//   3D (class 2, radius 2): 0:(0,0,0) 1:(1,0,0) 2:(1,1,0) 3:(2,0,0)
//   3D (class 3, radius 4): 0:(000) 1:(100) 2:(110) 3:(200) 4:(210) 5:(220) 6:(300) 7:(400)
struct OrbitW {
  double w[8];
};

struct ChemParams {  // f'(c) = 2 rho (c - ca)(c - cb)(2c - ca - cb), cahn_hilliard.cpp:70-73
  double rho_w, c_alpha, c_beta;
};

// Reference evaluation order, no contraction: bit-identical to f_chem_prime.
__device__ __forceinline__ double chem_prime(double c, const ChemParams& p) {
  const double a = __dsub_rn(c, p.c_alpha);
  const double b = __dsub_rn(c, p.c_beta);
  const double t = __dsub_rn(__dsub_rn(__dmul_rn(2.0, c), p.c_alpha), p.c_beta);
  return __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, p.rho_w), a), b), t);
}

enum class Mode { Apply = 0, CahnHilliard = 1 };

// Apply outputs are never re-read by the next launch (config 1 ping-pongs
// outputs from a fixed input): stream them past L2 (evict-first) so the input
// stays resident. CH outputs are the next step's input: keep normal policy.
template <Mode M>
__device__ __forceinline__ void store_f64x2(double* p, double a, double b) {
  if constexpr (M == Mode::Apply) {
    st_cs_f64x2(p, a, b);
  } else {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
  }
}

// =========================================================================
// 2D: full tile (TX x TY outputs + radius-2 halo) per CTA, x fastest.
// Thread (tx, ty) owns PX consecutive x points and PY consecutive rows and
// walks the PY+4 input rows of its strip with a register queue.
// =========================================================================
template <int TX, int TY, int PX, int PY>
struct Tile2D {
  static constexpr int R = 2;
  static constexpr int PITCH = TX + 2 * R;
  static constexpr int ROWS = TY + 2 * R;
  static constexpr int THREADS = (TX / PX) * (TY / PY);
  static constexpr int SMEM_BYTES = ROWS * PITCH * 8 + 16;
};

struct Apply2DArgs {
  const double* __restrict__ u;
  double* __restrict__ v;
  int64_t nx, ny;
  OrbitW w;      // scaled orbit weights of the composed stencil (Apply) or B' (CH)
  double wl0, wl1;  // CH: scaled 5-point Laplacian weights (center, axis)
  ChemParams chem;
  int bulk_ok;   // 1: nx even and >= TX+4 -> TMA bulk row copies
};

template <int TX, int TY, int PX, int PY>
__device__ __forceinline__ void load_tile_2d(double* tile, uint64_t* bar, const Apply2DArgs& a, int64_t x0,
                                             int64_t y0) {
  using T = Tile2D<TX, TY, PX, PY>;
  constexpr int R = T::R;
  const int tid = threadIdx.x;
  if (a.bulk_ok) {
    if (tid < 32) {
      if (tid == 0) mbar_arrive_expect_tx(bar, T::ROWS * T::PITCH * 8);
      __syncwarp();
      const int64_t xs = x0 - R;  // may be -R or run past nx: split into <= 2 pieces
      for (int r = tid; r < T::ROWS; r += 32) {
        int64_t gy = y0 - R + r;
        gy = wrap_idx(gy, a.ny);
        const double* row = a.u + gy * a.nx;
        double* dst = tile + r * T::PITCH;
        if (xs < 0) {
          bulk_g2s(dst, row + (a.nx + xs), uint32_t(-xs) * 8, bar);
          bulk_g2s(dst - xs, row, uint32_t(T::PITCH + xs) * 8, bar);
        } else if (xs + T::PITCH > a.nx) {
          const uint32_t first = uint32_t(a.nx - xs);
          bulk_g2s(dst, row + xs, first * 8, bar);
          bulk_g2s(dst + first, row, uint32_t(T::PITCH - first) * 8, bar);
        } else {
          bulk_g2s(dst, row + xs, T::PITCH * 8, bar);
        }
      }
    }
    mbar_wait(bar, 0);
  } else {
    for (int i = tid; i < T::ROWS * T::PITCH; i += T::THREADS) {
      const int r = i / T::PITCH, c = i % T::PITCH;
      const int64_t gy = wrap_idx(y0 - R + r, a.ny), gx = wrap_idx(x0 - R + c, a.nx);
      tile[i] = __ldg(a.u + gy * a.nx + gx);
    }
    __syncthreads();
  }
}

template <Mode M, int TX, int TY, int PX, int PY>
__global__ void __launch_bounds__(Tile2D<TX, TY, PX, PY>::THREADS)
    stencil2d_kernel(const Apply2DArgs a) {
  using T = Tile2D<TX, TY, PX, PY>;
  constexpr int R = T::R;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double* tile = reinterpret_cast<double*>(smem_raw + 16);

  const int64_t x0 = int64_t(blockIdx.x) * TX, y0 = int64_t(blockIdx.y) * TY;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  load_tile_2d<TX, TY, PX, PY>(tile, bar, a, x0, y0);

  const int tx = threadIdx.x % (TX / PX), ty = threadIdx.x / (TX / PX);
  const int lx = tx * PX + R;  // tile column of the first owned point
  const int ly = ty * PY;      // tile row of the first owned output (input row ly + R)

  double acc[PY][PX];
#pragma unroll
  for (int j = 0; j < PY; ++j)
#pragma unroll
    for (int i = 0; i < PX; ++i) acc[j][i] = 0.0;

  // walk input rows ly .. ly + PY + 2R - 1 (tile rows); input row k feeds
  // outputs j with |k - R - j| <= R via slice S_|k-R-j|
#pragma unroll
  for (int k = 0; k < PY + 2 * R; ++k) {
    const double* row = tile + (ly + k) * T::PITCH + lx;
    double u[PX + 2 * R];  // x - R .. x + PX - 1 + R
#pragma unroll
    for (int i = 0; i < PX + 2 * R; ++i) u[i] = row[i - R];
    // which slices of this row are needed by some owned output
    bool need0 = false, need1 = false, need2 = false;
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      const int d = k - R - j;
      need0 |= d == 0;
      need1 |= d == 1 || d == -1;
      need2 |= d == 2 || d == -2;
    }
#pragma unroll
    for (int i = 0; i < PX; ++i) {
      const double c = u[i + R];
      const double p1 = u[i + R - 1] + u[i + R + 1];
      double s0 = 0, s1 = 0, s2 = 0;
      if (need0) {
        const double p2 = u[i + R - 2] + u[i + R + 2];
        s0 = fma(a.w.w[3], p2, fma(a.w.w[1], p1, a.w.w[0] * c));
      }
      if (need1) s1 = fma(a.w.w[2], p1, a.w.w[1] * c);
      if (need2) s2 = a.w.w[3] * c;
      if (M == Mode::CahnHilliard) {
        // L f'(c): 5-point on g = f'(c); g at this row's point (for |d| = 1)
        // and the row neighbours (for d = 0). Vertical neighbours arrive as
        // the g-centre of adjacent rows through the |d| = 1 slice.
        const double g = chem_prime(c, a.chem);
        if (need0) {
          const double gp = chem_prime(u[i + R - 1], a.chem) + chem_prime(u[i + R + 1], a.chem);
          s0 = fma(a.wl1, gp, fma(a.wl0, g, s0));
        }
        if (need1) s1 = fma(a.wl1, g, s1);
      }
#pragma unroll
      for (int j = 0; j < PY; ++j) {
        const int d = k - R - j;
        if (d == 0) acc[j][i] += s0;
        if (d == 1 || d == -1) acc[j][i] += s1;
        if (d == 2 || d == -2) acc[j][i] += s2;
      }
    }
  }

  const int64_t gx = x0 + tx * PX;
#pragma unroll
  for (int j = 0; j < PY; ++j) {
    const int64_t gy = y0 + ly + j;
    if (gy >= a.ny) continue;
    double* out = a.v + gy * a.nx + gx;
    double val[PX];
#pragma unroll
    for (int i = 0; i < PX; ++i) {
      val[i] = acc[j][i];
      if (M == Mode::CahnHilliard) val[i] += tile[(ly + j + R) * T::PITCH + lx + i];
    }
    if (a.bulk_ok && PX % 2 == 0 && gx + PX <= a.nx) {
#pragma unroll
      for (int i = 0; i < PX; i += 2) store_f64x2<M>(out + i, val[i], val[i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < PX; ++i)
        if (gx + i < a.nx) out[i] = val[i];
    }
  }
}

// =========================================================================
// 3D: warp-specialised streaming along z. CTA = TX x TY column of the grid
// over a chunk of CZ output planes; ring of STAGES plane buffers
// ((TY+2R) x (TX+2R) doubles each) filled by one producer warp with TMA bulk
// row copies; 8 consumer warps, each thread PX x PY points, register queue of
// 2R+1 output planes rotated by loop unrolling (no register moves).
// =========================================================================
template <int R_, int TX_, int TY_, int PX_, int PY_, int STAGES_>
struct Cfg3D {
  static constexpr int R = R_, TX = TX_, TY = TY_, PX = PX_, PY = PY_, STAGES = STAGES_;
  static constexpr int PITCH = TX + 2 * R;
  static constexpr int ROWS = TY + 2 * R;
  static constexpr int PLANE = ROWS * PITCH;  // doubles
  static constexpr int CONSUMERS = (TX / PX) * (TY / PY);
  static_assert(CONSUMERS % 32 == 0, "consumer threads must be whole warps");
  static constexpr int CONSUMER_WARPS = CONSUMERS / 32;
  static constexpr int THREADS = CONSUMERS + 32;
  static constexpr int BAR_BYTES = 2 * STAGES * 8;
  static constexpr int SMEM_BYTES = 128 + STAGES * PLANE * 8;
  static constexpr int Q = 2 * R + 1;
};

struct Apply3DArgs {
  const double* __restrict__ u;
  double* __restrict__ v;
  int64_t nx, ny, nz;
  int cz;        // output planes per CTA
  int tiles_x;   // CTAs along x
  OrbitW w;
  double wl0, wl1;
  ChemParams chem;
  int bulk_ok;
};

template <class C>
__device__ __forceinline__ void produce_plane_3d(double* buf, uint64_t* full, const Apply3DArgs& a, int64_t x0,
                                                 int64_t y0, int64_t gz, int lane) {
  constexpr int R = C::R;
  const double* plane = a.u + gz * a.nx * a.ny;
  if (a.bulk_ok) {
    if (lane == 0) mbar_arrive_expect_tx(full, C::PLANE * 8);
    __syncwarp();
    const int64_t xs = x0 - R;
    for (int r = lane; r < C::ROWS; r += 32) {
      const int64_t gy = wrap_idx(y0 - R + r, a.ny);
      const double* row = plane + gy * a.nx;
      double* dst = buf + r * C::PITCH;
      if (xs < 0) {
        bulk_g2s(dst, row + (a.nx + xs), uint32_t(-xs) * 8, full);
        bulk_g2s(dst - xs, row, uint32_t(C::PITCH + xs) * 8, full);
      } else if (xs + C::PITCH > a.nx) {
        const uint32_t first = uint32_t(a.nx - xs);
        bulk_g2s(dst, row + xs, first * 8, full);
        bulk_g2s(dst + first, row, uint32_t(C::PITCH - first) * 8, full);
      } else {
        bulk_g2s(dst, row + xs, C::PITCH * 8, full);
      }
    }
  } else {
    for (int i = lane; i < C::PLANE; i += 32) {
      const int r = i / C::PITCH, c = i % C::PITCH;
      const int64_t gy = wrap_idx(y0 - R + r, a.ny), gx = wrap_idx(x0 - R + c, a.nx);
      buf[i] = __ldg(plane + gy * a.nx + gx);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(full);
  }
}

// In-plane orbit sums at tile position (ly, lx) for the point set of one
// thread. Slices per radius:
//   R=2 (25-pt): S0 = w0 c + w1 A1 + w2 D11 + w3 A2 ; S1 = w1 c + w2 A1 ; S2 = w3 c
//   R=4 (73-pt): S0 = w0 c + w1 A1 + w2 D11 + w3 A2 + w4 D21 + w5 D22 + w6 A3 + w7 A4
//                S1 = w1 c + w2 A1 + w4 A2 ; S2 = w3 c + w4 A1 + w5 A2 ; S3 = w6 c ; S4 = w7 c
template <int R>
__device__ __forceinline__ void slices_3d(const double* __restrict__ buf, int pitch, int ly, int lx, const OrbitW& w,
                                          double* s) {
  auto at = [&](int dy, int dx) { return buf[(ly + dy) * pitch + lx + dx]; };
  const double c = at(0, 0);
  const double a1 = (at(0, -1) + at(0, 1)) + (at(-1, 0) + at(1, 0));
  if constexpr (R == 2) {
    const double d11 = (at(-1, -1) + at(-1, 1)) + (at(1, -1) + at(1, 1));
    const double a2 = (at(0, -2) + at(0, 2)) + (at(-2, 0) + at(2, 0));
    s[0] = fma(w.w[3], a2, fma(w.w[2], d11, fma(w.w[1], a1, w.w[0] * c)));
    s[1] = fma(w.w[2], a1, w.w[1] * c);
    s[2] = w.w[3] * c;
  } else {
    const double d11 = (at(-1, -1) + at(-1, 1)) + (at(1, -1) + at(1, 1));
    const double a2 = (at(0, -2) + at(0, 2)) + (at(-2, 0) + at(2, 0));
    const double d21 = ((at(-1, -2) + at(-1, 2)) + (at(1, -2) + at(1, 2))) +
                       ((at(-2, -1) + at(-2, 1)) + (at(2, -1) + at(2, 1)));
    const double d22 = (at(-2, -2) + at(-2, 2)) + (at(2, -2) + at(2, 2));
    const double a3 = (at(0, -3) + at(0, 3)) + (at(-3, 0) + at(3, 0));
    const double a4 = (at(0, -4) + at(0, 4)) + (at(-4, 0) + at(4, 0));
    s[0] = fma(w.w[7], a4,
               fma(w.w[6], a3,
                   fma(w.w[5], d22, fma(w.w[4], d21, fma(w.w[3], a2, fma(w.w[2], d11, fma(w.w[1], a1, w.w[0] * c)))))));
    s[1] = fma(w.w[4], a2, fma(w.w[2], a1, w.w[1] * c));
    s[2] = fma(w.w[5], a2, fma(w.w[4], a1, w.w[3] * c));
    s[3] = w.w[6] * c;
    s[4] = w.w[7] * c;
  }
}

template <Mode M, class C>
__global__ void __launch_bounds__(C::THREADS) stencil3d_kernel(const Apply3DArgs a) {
  constexpr int R = C::R, Q = C::Q, S = C::STAGES;
  constexpr int NPT = C::PX * C::PY;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + S;
  double* ring = reinterpret_cast<double*>(smem_raw + 128);

  const int tile = blockIdx.x;
  const int64_t x0 = int64_t(tile % a.tiles_x) * C::TX;
  const int64_t y0 = int64_t(tile / a.tiles_x) * C::TY;
  const int64_t z0 = int64_t(blockIdx.y) * a.cz;
  const int cz = int(a.nz - z0 < int64_t(a.cz) ? a.nz - z0 : int64_t(a.cz));
  const int np = cz + 2 * R;  // input planes z0-R .. z0+cz-1+R

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::CONSUMER_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == C::CONSUMER_WARPS) {  // ---- producer warp ----
    for (int p = 0; p < np; ++p) {
      const int s = p % S;
      if (p >= S) mbar_wait(&empty[s], ((p / S) - 1) & 1);
      const int64_t gz = wrap_idx(z0 - R + p, a.nz);
      produce_plane_3d<C>(ring + s * C::PLANE, &full[s], a, x0, y0, gz, lane);
    }
    return;
  }

  // ---- consumer warps ----
  const int tx = threadIdx.x % (C::TX / C::PX), ty = threadIdx.x / (C::TX / C::PX);
  const int lx0 = tx * C::PX + R, ly0 = ty * C::PY + R;
  const int64_t gx0 = x0 + tx * C::PX;

  double q[Q][NPT];
#pragma unroll
  for (int t = 0; t < Q; ++t)
#pragma unroll
    for (int i = 0; i < NPT; ++i) q[t][i] = 0.0;
  double cen[Q][NPT];  // CH: centre values of input planes, slot = plane % Q
  (void)cen;

  // process planes in groups of Q so the queue rotation is static
  for (int pb = 0; pb < np; pb += Q) {
#pragma unroll
    for (int st = 0; st < Q; ++st) {
      const int p = pb + st;
      if (p < np) {
        const int s = p % S;
        mbar_wait(&full[s], (p / S) & 1);
        const double* buf = ring + s * C::PLANE;
        double sl[R + 1][NPT];
#pragma unroll
        for (int j = 0; j < C::PY; ++j)
#pragma unroll
          for (int i = 0; i < C::PX; ++i) {
            double sv[R + 1];
            slices_3d<R>(buf, C::PITCH, ly0 + j, lx0 + i, a.w, sv);
            if (M == Mode::CahnHilliard) {
              // L f'(c) with the 7-point Laplacian: in-plane part at d=0, centre at |d|=1
              auto at = [&](int dy, int dx) { return buf[(ly0 + j + dy) * C::PITCH + lx0 + i + dx]; };
              const double g = chem_prime(at(0, 0), a.chem);
              const double ga = (chem_prime(at(0, -1), a.chem) + chem_prime(at(0, 1), a.chem)) +
                                (chem_prime(at(-1, 0), a.chem) + chem_prime(at(1, 0), a.chem));
              sv[0] = fma(a.wl1, ga, fma(a.wl0, g, sv[0]));
              sv[1] = fma(a.wl1, g, sv[1]);
            }
#pragma unroll
            for (int d = 0; d <= R; ++d) sl[d][j * C::PX + i] = sv[d];
          }
        // centre values needed by the CH update of the output plane p - R
        double cz_now[NPT];
        if (M == Mode::CahnHilliard) {
#pragma unroll
          for (int j = 0; j < C::PY; ++j)
#pragma unroll
            for (int i = 0; i < C::PX; ++i) cz_now[j * C::PX + i] = buf[(ly0 + j) * C::PITCH + lx0 + i];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        // push: input plane p feeds output o = p - R - dz, queue slot t = R - dz
#pragma unroll
        for (int t = 0; t < Q; ++t) {
          const int d = t < R ? R - t : t - R;
          const int slot = (st + t) % Q;
#pragma unroll
          for (int i = 0; i < NPT; ++i) q[slot][i] += sl[d][i];
        }
        if (M == Mode::CahnHilliard) {
          // input plane p is output plane p - R: keep its centre values until complete
#pragma unroll
          for (int i = 0; i < NPT; ++i) cen[st][i] = cz_now[i];
        }
        // output o = p - 2R (queue slot t = 0) is complete
        const int o = p - 2 * R;
        const int slot0 = st % Q;
        if (o >= 0) {
          const int64_t gz = z0 + o;
          double* outp = a.v + (gz * a.ny) * a.nx;
#pragma unroll
          for (int j = 0; j < C::PY; ++j) {
            const int64_t gy = y0 + ty * C::PY + j;
            if (gy >= a.ny) continue;
            double val[C::PX];
#pragma unroll
            for (int i = 0; i < C::PX; ++i) {
              val[i] = q[slot0][j * C::PX + i];
              if (M == Mode::CahnHilliard) val[i] += cen[(st + R + 1) % Q][j * C::PX + i];
            }
            double* dst = outp + gy * a.nx + gx0;
            if (a.bulk_ok && C::PX % 2 == 0 && gx0 + C::PX <= a.nx) {
#pragma unroll
              for (int i = 0; i < C::PX; i += 2) store_f64x2<M>(dst + i, val[i], val[i + 1]);
            } else {
#pragma unroll
              for (int i = 0; i < C::PX; ++i)
                if (gx0 + i < a.nx) dst[i] = val[i];
            }
          }
        }
#pragma unroll
        for (int i = 0; i < NPT; ++i) q[slot0][i] = 0.0;
      }
    }
  }
}

// =========================================================================
// Generic fallback: any stencil (dim 1..3, any offsets, any boundary kind),
// one thread per unknown, entries read through the read-only cache. Row
// semantics follow assemble (grid.cpp:89-138): periodic wrap, odd (simply
// supported) or even (clamped) reflection, boundary ghosts dropped.
// =========================================================================
struct GenericArgs {
  const double* __restrict__ u;
  double* __restrict__ v;
  const int* __restrict__ off;     // nent * 3 (unused axes 0)
  const double* __restrict__ coeff;  // nent
  int nent;
  int dim;
  int64_t n[3], un[3];
  int bc[3];
  double scale;  // pow_int(h, h_power)
  int64_t rows;
};

static __global__ void stencil_generic_kernel(const GenericArgs a) {
  const int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= a.rows) return;
  int64_t idx[3];
  int64_t rem = row;
  for (int d = 0; d < 3; ++d) {
    idx[d] = rem % a.un[d];
    rem /= a.un[d];
  }
  double acc = 0.0;
  for (int e = 0; e < a.nent; ++e) {
    double val = __ldg(a.coeff + e) * a.scale;
    int64_t col = 0, stride = 1;
    bool dropped = false;
    for (int d = 0; d < a.dim; ++d) {
      const int o = __ldg(a.off + 3 * e + d);
      int64_t comp;
      if (a.bc[d] == SK_BC_PERIODIC) {
        comp = wrap_idx(idx[d] + o, a.n[d]);
      } else {
        int64_t gi = idx[d] + 1 + o;
        if (gi < 0) {
          gi = -gi;
          if (a.bc[d] == SK_BC_SIMPLY_SUPPORTED) val = -val;
        } else if (gi > a.n[d] - 1) {
          gi = 2 * (a.n[d] - 1) - gi;
          if (a.bc[d] == SK_BC_SIMPLY_SUPPORTED) val = -val;
        }
        if (gi == 0 || gi == a.n[d] - 1) {
          dropped = true;
          break;
        }
        comp = gi - 1;
      }
      col += stride * comp;
      stride *= a.un[d];
    }
    if (!dropped) acc = fma(val, __ldg(a.u + col), acc);
  }
  a.v[row] = acc;
}

}  // namespace sk
