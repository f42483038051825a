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
// Data movement: tiles (+ radius-R halo) land in shared memory through
// all-thread 16-byte cp.async (LDGSTS) on periodic grids with aligned rows;
// otherwise (odd widths, non-periodic boundaries) element-wise with the
// boundary map of assemble (bc_map: wrap, even / odd reflection, zero
// boundary points). The 3D kernels (sk_stream3d.cuh) stream planes through a
// multistage shared ring with one barrier per plane; the headline factored
// CH kernel (sk_chf3d.cuh) uses TMA boxes from ghost-padded fields.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "sk_cgstate.cuh"
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

// f'(c) expanded on the host into a cubic, evaluated with 3 FMAs:
//   2 rho (c-a)(c-b)(2c-a-b) = 4rho c^3 - 6rho(a+b) c^2 + 2rho((a+b)^2 + 2ab) c - 2rho ab(a+b)
// (for rho = 1/4, a = -1, b = 1 exactly c^3 - c).
struct Poly3 {
  double k3, k2, k1, k0;
};

__device__ __forceinline__ double poly3(double c, const Poly3& p) {
  return fma(fma(fma(p.k3, c, p.k2), c, p.k1), c, p.k0);
}

// CgApply: one matrix-free CG iteration's first half (sk_cg.cu, fused2d):
// p' = r + beta p formed on the tile load (the bit-exact xpby of
// linalg.cpp:57, deferred from the previous iteration), q = A p', and the
// p'.q partials reduced to alpha by the last CTA. p itself is not written:
// the update kernel that follows recomputes p' and stores it.
enum class Mode { Apply = 0, CahnHilliard = 1, CgApply = 2 };

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
  static constexpr int SMEM_BYTES_CG = 2 * ROWS * PITCH * 8 + 16;  // + the r tile
};

struct Apply2DArgs {
  const double* __restrict__ u;
  double* __restrict__ v;
  int64_t nx, ny;
  OrbitW w;      // scaled orbit weights of the composed stencil (Apply) or B' (CH)
  double wl0, wl1;  // CH: scaled 5-point Laplacian weights (center, axis)
  Poly3 chem;
  int bulk_ok;   // 1: nx even and >= TX+4, periodic -> 16-byte cp.async rows
  int bc[2];     // boundary kind per axis (nx, ny are unknown counts)
  int input_stable;  // Apply: u is not written by the preceding kernel (early loads under PDL)
  // CgApply: u = p (previous direction), v = q
  const double* __restrict__ r;
  CgState* st;
  double* partials;  // one per CTA
};

// NC: p and r are read-only for the whole kernel (ld.global.nc allowed); the
// cooperative CG kernel, which rewrites them between its grid barriers, loads
// them coherently (cp.async and ld.global.cg are ordered by the barrier's
// acquire; the non-coherent read-only path is not).
template <Mode M, int TX, int TY, int PX, int PY, bool NC = true>
__device__ __forceinline__ void load_tile_2d(double* tile, const Apply2DArgs& a, int64_t x0, int64_t y0,
                                             double beta) {
  using T = Tile2D<TX, TY, PX, PY>;
  constexpr int R = T::R;
  const int tid = threadIdx.x;
  // tile wholly inside the grid: no boundary map
  const bool inner = x0 >= R && x0 + TX + R <= a.nx && y0 >= R && y0 + TY + R <= a.ny;
  if constexpr (M == Mode::CgApply) {
    if (inner) {  // both tiles by 8-byte cp.async, then p' in place (each thread its own points)
      double* rt = tile + T::ROWS * T::PITCH;
      const int64_t base = (y0 - R) * a.nx + (x0 - R);
      for (int i = tid; i < T::ROWS * T::PITCH; i += T::THREADS) {
        const int r = i / T::PITCH, c = i - r * T::PITCH;
        const int64_t g = base + r * a.nx + c;
        cp_async8(tile + i, a.u + g);
        cp_async8(rt + i, a.r + g);
      }
      cp_async_wait_all();
      for (int i = tid; i < T::ROWS * T::PITCH; i += T::THREADS) tile[i] = __dadd_rn(rt[i], __dmul_rn(beta, tile[i]));
      __syncthreads();
      return;
    }
    for (int i = tid; i < T::ROWS * T::PITCH; i += T::THREADS) {
      const int r = i / T::PITCH, c = i % T::PITCH;
      double f = 1.0;
      const int64_t gy = bc_map(y0 - R + r, a.ny, a.bc[1], f), gx = bc_map(x0 - R + c, a.nx, a.bc[0], f);
      const int64_t g = gy * a.nx + gx;
      double v = 0.0;  // boundary zero (g may lie outside the field then)
      if (f != 0.0) {
        const double rv = NC ? __ldg(a.r + g) : __ldcg(a.r + g), pv = NC ? __ldg(a.u + g) : __ldcg(a.u + g);
        v = f * __dadd_rn(rv, __dmul_rn(beta, pv));
      }
      tile[i] = v;
    }
    __syncthreads();
  } else if (a.bulk_ok) {
    // every thread issues 16-byte cp.async (LDGSTS) pairs of the haloed tile
    constexpr int HP = T::PITCH / 2;
    for (int i = tid; i < T::ROWS * HP; i += T::THREADS) {
      const int r = i / HP, c = 2 * (i - r * HP);
      const int64_t gy = wrap1(y0 - R + r, a.ny), gx = wrap1(x0 - R + c, a.nx);
      cp_async16(tile + r * T::PITCH + c, a.u + gy * a.nx + gx);
    }
    cp_async_wait_all();
    sk_jitter(30);
    __syncthreads();
  } else if (inner) {  // 8-byte cp.async (rows need not be 16-byte aligned)
    const int64_t base = (y0 - R) * a.nx + (x0 - R);
    for (int i = tid; i < T::ROWS * T::PITCH; i += T::THREADS) {
      const int r = i / T::PITCH, c = i - r * T::PITCH;
      cp_async8(tile + i, a.u + base + r * a.nx + c);
    }
    cp_async_wait_all();
    sk_jitter(30);
    __syncthreads();
  } else {
    for (int i = tid; i < T::ROWS * T::PITCH; i += T::THREADS) {  // any boundary kind
      const int r = i / T::PITCH, c = i % T::PITCH;
      double f = 1.0;
      const int64_t gy = bc_map(y0 - R + r, a.ny, a.bc[1], f), gx = bc_map(x0 - R + c, a.nx, a.bc[0], f);
      tile[i] = f == 0.0 ? 0.0 : f * __ldg(a.u + gy * a.nx + gx);
    }
    __syncthreads();
  }
}

// One tile: load (+ halo), evaluate, store. CgApply: returns this thread's
// p'.q partial (p' = r + beta p). The caller orders the tile buffer's reuse.
template <Mode M, int TX, int TY, int PX, int PY, bool NC = true>
__device__ __forceinline__ double stencil2d_tile(double* tile, const Apply2DArgs& a, int64_t x0, int64_t y0,
                                                 double beta) {
  using T = Tile2D<TX, TY, PX, PY>;
  constexpr int R = T::R;
  load_tile_2d<M, TX, TY, PX, PY, NC>(tile, a, x0, y0, beta);

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
        const double g = poly3(c, a.chem);
        if (need0) {
          const double gp = poly3(u[i + R - 1], a.chem) + poly3(u[i + R + 1], a.chem);
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
  if constexpr (M == Mode::Apply) asm volatile("griddepcontrol.wait;" ::: "memory");
  double pq = 0.0;
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
    if constexpr (M == Mode::CgApply) {
#pragma unroll
      for (int i = 0; i < PX; ++i) {
        if (gx + i < a.nx) {
          const double p = tile[(ly + j + R) * T::PITCH + lx + i];
          out[i] = val[i];
          pq = fma(p, val[i], pq);
        }
      }
    } else if (a.bulk_ok && PX % 2 == 0 && gx + PX <= a.nx) {
#pragma unroll
      for (int i = 0; i < PX; i += 2) store_f64x2<M>(out + i, val[i], val[i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < PX; ++i)
        if (gx + i < a.nx) out[i] = val[i];
    }
  }
  return pq;
}

template <Mode M, int TX, int TY, int PX, int PY>
__global__ void __launch_bounds__(Tile2D<TX, TY, PX, PY>::THREADS)
    stencil2d_kernel(const Apply2DArgs a) {
  using T = Tile2D<TX, TY, PX, PY>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* tile = reinterpret_cast<double*>(smem_raw + 16);

  const int64_t x0 = int64_t(blockIdx.x) * TX, y0 = int64_t(blockIdx.y) * TY;
  // Programmatic dependent launch (launch_2d): the next kernel of the stream
  // may start its CTAs now; this one waits for its predecessor before the
  // first access that can conflict with it: the first load, except for an
  // Apply whose input no predecessor writes (the repeated apply of config 1),
  // which loads and computes first and waits before overwriting its output
  // (in stencil2d_tile). Without the launch attribute both are no-ops.
  asm volatile("griddepcontrol.launch_dependents;");
  if (M != Mode::Apply || !a.input_stable) asm volatile("griddepcontrol.wait;" ::: "memory");
  double beta = 0.0;
  if constexpr (M == Mode::CgApply) {
    if (a.st->status != kCgRunning) return;  // uniform: set by the previous iteration
    beta = a.st->beta;
  }
  __syncthreads();
  double pq = stencil2d_tile<M, TX, TY, PX, PY>(tile, a, x0, y0, beta);
  if constexpr (M == Mode::CgApply) {
    __shared__ double red[32];
    const unsigned cta = blockIdx.y * gridDim.x + blockIdx.x, nctas = gridDim.x * gridDim.y;
    pq = block_sum<T::THREADS>(pq, red);
    if (threadIdx.x == 0) a.partials[cta] = pq;
    if (last_block(&a.st->counter[0], nctas)) {
      pq = reduce_partials<T::THREADS>(a.partials, int(nctas), red);
      if (threadIdx.x == 0) cg_publish_pq(a.st, pq);
    }
  }
}

// =========================================================================
// Generic fallback: any stencil (dim 1..3, any offsets, any boundary kind),
// one thread per unknown. Row semantics follow assemble (grid.cpp:89-138):
// periodic wrap, odd (simply supported) or even (clamped) reflection,
// boundary ghosts dropped. Launched over (x blocks, y, z), so the point's
// index needs no division; every entry's linear offset and weight sit in
// shared memory, and a point whose whole support lies inside the grid
// (no wrap, no reflection) sums u[row + delta_e] directly. Entries are summed
// in stencil order on both paths (the same bits as the boundary logic).
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
  int lo[3], hi[3];  // the stencil's support per axis
};

static __global__ void __launch_bounds__(256) stencil_generic_kernel(const GenericArgs a) {
  extern __shared__ __align__(16) unsigned char gen_smem[];
  int64_t* delta = reinterpret_cast<int64_t*>(gen_smem);  // linear offset of each entry
  double* wv = reinterpret_cast<double*>(delta + a.nent);  // its weight (coeff * h^power)
  for (int e = threadIdx.x; e < a.nent; e += blockDim.x) {
    int64_t dl = 0, stride = 1;
    for (int d = 0; d < a.dim; ++d) {
      dl += stride * __ldg(a.off + 3 * e + d);
      stride *= a.un[d];
    }
    delta[e] = dl;
    wv[e] = __ldg(a.coeff + e) * a.scale;
  }
  __syncthreads();
  const int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= a.un[0]) return;
  const int64_t idx[3] = {x, int64_t(blockIdx.y), int64_t(blockIdx.z)};
  const int64_t row = x + a.un[0] * (idx[1] + a.un[1] * idx[2]);
  bool inner = true;
  for (int d = 0; d < a.dim; ++d) inner = inner && idx[d] + a.lo[d] >= 0 && idx[d] + a.hi[d] <= a.un[d] - 1;
  double acc = 0.0;
  if (inner) {
    for (int e = 0; e < a.nent; ++e) acc = fma(wv[e], __ldg(a.u + row + delta[e]), acc);
    a.v[row] = acc;
    return;
  }
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
