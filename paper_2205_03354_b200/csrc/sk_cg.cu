// Conjugate gradients on the device, control flow of linalg.cpp:15-72.
//
// Per iteration three kernels (captured in a CUDA graph of `check_every`
// iterations; all scalars stay on the device, the host polls a status word
// once per graph):
//   K1  q = M p (CSR, reference rounding) fused with the p.q partials; the
//       last CTA forms pq, flags "not positive definite" (linalg.cpp:50-51)
//       or sets alpha = rho / pq.
//   K2  x += alpha p ; r -= alpha q (bit-exact axpy) fused with r.r
//       partials; the last CTA sets rho_next, beta, counts the iteration and
//       raises CHECK when sqrt(rho) <= tol ||b|| (linalg.cpp:31) or stops at
//       max_iter.
//   K3  p = r + beta p (bit-exact xpby).
// Matrix-free operators replace K1 by the stencil apply + a p.q pass; on a
// 2D 13-point class stencil the iteration is two kernels instead (fused2d):
// the apply forms p' = r + beta p while loading its tile, writes q = A p' and
// reduces alpha; K2 recomputes p' (same bits), stores it and updates x, r.
// Kernels of a graph become no-ops once the status leaves RUNNING, so the
// iteration count is exact. The rare true-residual check / restart
// (linalg.cpp:32-47) and the final acceptance test (:59-66) run outside the
// graph.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "sk_internal.hpp"
#include "sk_cgstate.cuh"
#include "sk_sell.cuh"
#include "sk_stencil_kernels.cuh"

namespace sk {

namespace {

constexpr int kT = 256;
enum : int { kRunning = kCgRunning, kCheck = kCgCheck, kNotPD = kCgNotPD, kMaxIter = kCgMaxIter };
constexpr int64_t kCoopMaxRows = 131072;  // k_cg2d_coop up to this many unknowns (measured crossover)
constexpr int kLoopUnroll = 4;  // CG iterations per round of the device-side while loop

// Row i of M times x from the SELL-32 copy (sk_sell.cuh): reference order and rounding.
template <class IDX>
__device__ __forceinline__ double row_dot(const int64_t* __restrict__ sp, const int32_t* __restrict__ len,
                                          const IDX* __restrict__ col, const double* __restrict__ val,
                                          const double* __restrict__ x, int64_t i) {
  return sell_row_dot(i, sp, len, col, val, x);
}

template <class IDX>
__global__ void __launch_bounds__(kT) k1_spmv_pq(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ len,
                                                 const IDX* __restrict__ col, const double* __restrict__ val,
                                                 const double* __restrict__ p, double* __restrict__ q, CgState* st,
                                                 double* partials) {
  if (st->status != kRunning) return;
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) {
    const double qi = row_dot(rp, len, col, val, p, i);
    q[i] = qi;
    acc = fma(p[i], qi, acc);
  }
  acc = block_sum<kT>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  if (last_block(&st->counter[0])) {
    const double pq = reduce_partials<kT>(partials, gridDim.x, sh);
    if (threadIdx.x == 0) cg_publish_pq(st, pq);
  }
}

// FUSED (2D fused path, which has no K3): K3 of the previous iteration is
// deferred to here, p' = r + beta p (the same bits the apply formed) stored
// before the updates use it, and the last CTA publishes the device-side while
// loop's condition (COND). The new beta is written after every CTA has read
// the old one (last_block orders it).
template <bool COND, bool FUSED>
__global__ void __launch_bounds__(kT) k2_update_rr(int64_t n, double* __restrict__ p, const double* __restrict__ q,
                                                   double* __restrict__ x, double* __restrict__ r, CgState* st,
                                                   double* partials, cudaGraphConditionalHandle cond) {
  if (st->status != kRunning) {
    if constexpr (COND) {
      if (blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0u);
    }
    return;
  }
  __shared__ double sh[32];
  const double alpha = st->alpha, nalpha = -alpha;
  const double beta = FUSED ? st->beta : 0.0;
  double acc = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) {
    double pi = p[i];
    if constexpr (FUSED) {
      pi = __dadd_rn(r[i], __dmul_rn(beta, pi));  // xpby(r, beta, p)
      p[i] = pi;
    }
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, pi));               // axpy(alpha, p, x)
    const double ri = __dadd_rn(r[i], __dmul_rn(nalpha, q[i]));  // axpy(-alpha, q, r)
    r[i] = ri;
    acc = fma(ri, ri, acc);
  }
  acc = block_sum<kT>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  if (last_block(&st->counter[1])) {
    const double rho_next = reduce_partials<kT>(partials, gridDim.x, sh);
    if (threadIdx.x == 0) {
      st->beta = rho_next / st->rho;
      st->rho = rho_next;
      st->it += 1;
      if (st->it >= st->max_iter) st->status = kMaxIter;
      else if (sqrt(rho_next) <= st->target) st->status = kCheck;
      if constexpr (COND) cudaGraphSetConditional(cond, st->status == kRunning ? 1u : 0u);
    }
  }
}

// COND: the body of a device-side while loop (conditional graph node): the
// first thread publishes "keep iterating" for the next round.
template <bool COND>
__global__ void k3_xpby(int64_t n, const double* __restrict__ r, double* __restrict__ p, const CgState* st,
                        cudaGraphConditionalHandle cond) {
  if constexpr (COND) {
    if (blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, st->status == kRunning ? 1u : 0u);
  }
  if (st->status != kRunning) return;
  const double beta = st->beta;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));
}

// Ghost-padded copy of p for the radius-4 matrix-free apply on non-periodic
// grids (launch_apply_padded): every interior point is written at its padded
// position and at each of its ghost images (assemble's boundary handling,
// grid.cpp:104-122: even reflection about the boundary point for clamped,
// odd for simply supported, wrap for periodic axes); the boundary points
// (padded -1 and un) stay 0 from the initial memset. Per axis a point x has
// the image -x-2 when x < R and 2un-x when x >= un-R (periodic: x+un / x-un).
struct PadLayout {
  int pad = 0;         // frame width (>= R + 1, even)
  int padx = 0;        // frame width before x = 0 (>= pad): 16 puts every interior row on a 128-byte boundary
  int64_t px = 0, py = 0, plane = 0;  // row and plane pitch (elements)
  int64_t un[3] = {0, 0, 0};
  int bc[3] = {0, 0, 0};
  int R = 4;
  __host__ __device__ int64_t at(int64_t x, int64_t y, int64_t z) const {
    return (z + pad) * plane + (y + pad) * px + (x + padx);
  }
};

__device__ __forceinline__ int pad_images(const PadLayout& L, int a, int64_t x, int64_t* pos, double* sgn) {
  pos[0] = x;
  sgn[0] = 1.0;
  int n = 1;
  const int64_t un = L.un[a];
  if (L.bc[a] == SK_BC_PERIODIC) {
    if (x < L.R) { pos[n] = x + un; sgn[n++] = 1.0; }
    if (x >= un - L.R) { pos[n] = x - un; sgn[n++] = 1.0; }
  } else {
    const double s = L.bc[a] == SK_BC_SIMPLY_SUPPORTED ? -1.0 : 1.0;
    if (x < L.R) { pos[n] = -x - 2; sgn[n++] = s; }
    if (x >= un - L.R) { pos[n] = 2 * un - x; sgn[n++] = s; }
  }
  return n;
}

// one interior point (x, y, z) with value v: its padded position and images
__device__ __forceinline__ void pad_store(const PadLayout& L, double* __restrict__ pp, int64_t x, int64_t y,
                                          int64_t z, bool row_edge, double v) {
  if (!row_edge) {  // a row away from the y / z faces: images along x only
    pp[L.at(x, y, z)] = v;
    if (x >= L.R && x < L.un[0] - L.R) return;
    int64_t px[3];
    double sx[3];
    const int nx = pad_images(L, 0, x, px, sx);
    for (int a = 1; a < nx; ++a) pp[L.at(px[a], y, z)] = sx[a] * v;
    return;
  }
  int64_t px[3], py[3], pz[3];
  double sx[3], sy[3], sz[3];
  const int nx = pad_images(L, 0, x, px, sx), ny = pad_images(L, 1, y, py, sy), nz = pad_images(L, 2, z, pz, sz);
  for (int c = 0; c < nz; ++c)
    for (int b = 0; b < ny; ++b)
      for (int a = 0; a < nx; ++a) pp[L.at(px[a], py[b], pz[c])] = (sx[a] * sy[b] * sz[c]) * v;
}

// Row-mapped launches (block = one x-row of the interior, no per-element
// division): grid-stride over rows, threads over x.
__device__ __forceinline__ bool pad_row(const PadLayout& L, int64_t row, int64_t& y, int64_t& z) {
  z = row / L.un[1];
  y = row - z * L.un[1];
  return y < L.R || z < L.R || y >= L.un[1] - L.R || z >= L.un[2] - L.R;
}

// Warp per interior x-row (grid-stride over rows), 8 points per lane with
// all loads issued before the stores: the row's padded position and images.
constexpr int kPadPts = 8;

__global__ void __launch_bounds__(256) k_pad_fill(const double* __restrict__ p, double* __restrict__ pp,
                                                  const PadLayout L) {
  const int64_t rows = L.un[1] * L.un[2];
  const int lane = threadIdx.x % 32;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  for (int64_t row = int64_t(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32; row < rows; row += warps) {
    int64_t y, z;
    const bool edge = pad_row(L, row, y, z);
    const double* pr = p + row * L.un[0];
    for (int64_t x0 = 0; x0 < L.un[0]; x0 += 32 * kPadPts) {
      double v[kPadPts];
#pragma unroll
      for (int j = 0; j < kPadPts; ++j) {
        const int64_t x = x0 + lane + 32 * j;
        v[j] = x < L.un[0] ? pr[x] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < kPadPts; ++j) {
        const int64_t x = x0 + lane + 32 * j;
        if (x < L.un[0]) pad_store(L, pp, x, y, z, edge, v[j]);
      }
    }
  }
}

// K3 for the padded operator: p = r + beta p (bit-exact xpby) into p and its padded copy
template <bool COND>
__global__ void __launch_bounds__(256) k3_xpby_pad(const double* __restrict__ r, double* __restrict__ p,
                                                   double* __restrict__ pp, const PadLayout L, const CgState* st,
                                                   cudaGraphConditionalHandle cond) {
  if constexpr (COND) {
    if (blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, st->status == kRunning ? 1u : 0u);
  }
  if (st->status != kRunning) return;
  const double beta = st->beta;
  const int64_t rows = L.un[1] * L.un[2];
  const int lane = threadIdx.x % 32;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  for (int64_t row = int64_t(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32; row < rows; row += warps) {
    int64_t y, z;
    const bool edge = pad_row(L, row, y, z);
    const int64_t base = row * L.un[0];
    for (int64_t x0 = 0; x0 < L.un[0]; x0 += 32 * kPadPts) {
      double rv[kPadPts], pv[kPadPts];
#pragma unroll
      for (int j = 0; j < kPadPts; ++j) {
        const int64_t x = x0 + lane + 32 * j;
        rv[j] = x < L.un[0] ? r[base + x] : 0.0;
        pv[j] = x < L.un[0] ? p[base + x] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < kPadPts; ++j) {
        const int64_t x = x0 + lane + 32 * j;
        if (x < L.un[0]) {
          const double pi = __dadd_rn(rv[j], __dmul_rn(beta, pv[j]));
          p[base + x] = pi;
          pad_store(L, pp, x, y, z, edge, pi);
        }
      }
    }
  }
}

// q = M x ; out = sum (b - q)^2   (linalg.cpp:33-39, :59-61)
template <class IDX>
__global__ void __launch_bounds__(kT) k_true_residual(int64_t n, const int64_t* __restrict__ rp,
                                                      const int32_t* __restrict__ len, const IDX* __restrict__ col,
                                                      const double* __restrict__ val, const double* __restrict__ x,
                                                      const double* __restrict__ b, double* __restrict__ q, CgState* st,
                                                      double* partials) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) {
    const double qi = row_dot(rp, len, col, val, x, i);
    q[i] = qi;
    const double d = __dsub_rn(b[i], qi);
    acc = fma(d, d, acc);
  }
  acc = block_sum<kT>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  if (last_block(&st->counter[2])) {
    const double t = reduce_partials<kT>(partials, gridDim.x, sh);
    if (threadIdx.x == 0) st->scalar_out = t;
  }
}

// restart: r = b - q ; p = r ; rho = r.r   (linalg.cpp:43-46)
// (beta = 0: the fused path's deferred p' = r + 0 p is then r)
__global__ void __launch_bounds__(kT) k_restart(int64_t n, const double* __restrict__ b, const double* __restrict__ q,
                                                double* __restrict__ r, double* __restrict__ p, CgState* st,
                                                double* partials) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) {
    const double ri = __dsub_rn(b[i], q[i]);
    r[i] = ri;
    p[i] = ri;
    acc = fma(ri, ri, acc);
  }
  acc = block_sum<kT>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  if (last_block(&st->counter[3])) {
    const double t = reduce_partials<kT>(partials, gridDim.x, sh);
    if (threadIdx.x == 0) {
      st->rho = t;
      st->beta = 0.0;
      st->status = kRunning;
    }
  }
}

// op 0: sum a*a ; 1: sum a  -> st->scalar_out (uses counter[2])
template <int OP>
__global__ void __launch_bounds__(kT) k_reduce(int64_t n, const double* __restrict__ a, CgState* st, double* partials) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT)
    acc = OP == 0 ? fma(a[i], a[i], acc) : acc + a[i];
  acc = block_sum<kT>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  if (last_block(&st->counter[2])) {
    const double t = reduce_partials<kT>(partials, gridDim.x, sh);
    if (threadIdx.x == 0) st->scalar_out = t;
  }
}

__global__ void k_shift(int64_t n, double* __restrict__ x, double mean) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    x[i] -= mean;
}

// matrix-free operator: K1 split into the stencil apply q = A p and this p.q pass
__global__ void __launch_bounds__(kT) k_pq(int64_t n, const double* __restrict__ p, const double* __restrict__ q,
                                           CgState* st, double* partials) {
  if (st->status != kRunning) return;
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT)
    acc = fma(p[i], q[i], acc);
  acc = block_sum<kT>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  if (last_block(&st->counter[0])) {
    const double pq = reduce_partials<kT>(partials, gridDim.x, sh);
    if (threadIdx.x == 0) cg_publish_pq(st, pq);
  }
}

// sum (b - q)^2 with q = A x already applied (matrix-free true residual)
__global__ void __launch_bounds__(kT) k_resid(int64_t n, const double* __restrict__ b, const double* __restrict__ q,
                                              CgState* st, double* partials) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) {
    const double d = __dsub_rn(b[i], q[i]);
    acc = fma(d, d, acc);
  }
  acc = block_sum<kT>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  if (last_block(&st->counter[2])) {
    const double t = reduce_partials<kT>(partials, gridDim.x, sh);
    if (threadIdx.x == 0) st->scalar_out = t;
  }
}

// Whole CG iterations in one cooperative launch (2D class-1 stencil operator):
// phase A = the fused apply over the tiles (q = A p', p' = r + beta p, p'.q
// partials), grid barrier, every CTA sums the partials in the same order
// (identical alpha everywhere), phase B = the fused update (p = p', x, r,
// r.r partials), grid barrier, beta and the stopping rule. Runs while the
// status is RUNNING; CTA 0 publishes the scalars at exit. The recurrence is
// the fused2d graph path's (same kernels' arithmetic, same reduction order
// per CTA); L2-resident systems lose the launch and tail gaps of two kernels
// per iteration.
using CoopTile = Tile2D<64, 32, 2, 4>;

struct Coop2DArgs {
  Apply2DArgs a;  // u = p, v = q, r
  double* x;
  double* p;
  double* r;
  double* part_a;
  double* part_b;
  int64_t n;
  int tiles_x, tiles;
};

template <int THREADS>
__device__ __forceinline__ double block_broadcast_sum(const double* partials, int count, double* red, double* slot) {
  const double v = reduce_partials<THREADS>(partials, count, red);
  if (threadIdx.x == 0) *slot = v;
  __syncthreads();
  return *slot;
}

__global__ void __launch_bounds__(CoopTile::THREADS, 4) k_cg2d_coop(const Coop2DArgs c, CgState* st) {
  namespace cg = cooperative_groups;
  constexpr int T = CoopTile::THREADS;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* tile = reinterpret_cast<double*>(smem_raw + 16);
  __shared__ double red[32];
  __shared__ double bcast;
  double rho = st->rho, beta = st->beta, alpha = st->alpha, pq = st->pq;
  const double target = st->target;
  int64_t it = st->it;
  const int64_t max_iter = st->max_iter;
  int status = st->status;
  const int G = gridDim.x;
  while (status == kRunning) {
    double acc = 0.0;
    for (int t = blockIdx.x; t < c.tiles; t += G) {
      __syncthreads();  // the previous tile is consumed
      const int ty = t / c.tiles_x, tx = t - ty * c.tiles_x;
      acc += stencil2d_tile<Mode::CgApply, 64, 32, 2, 4, false>(tile, c.a, int64_t(tx) * 64, int64_t(ty) * 32, beta);
    }
    acc = block_sum<T>(acc, red);
    if (threadIdx.x == 0) c.part_a[blockIdx.x] = acc;
    sk_jitter(40);
    grid.sync();
    pq = block_broadcast_sum<T>(c.part_a, G, red, &bcast);
    if (pq <= 0) {  // linalg.cpp:50-51
      status = kNotPD;
      break;
    }
    alpha = rho / pq;
    const double nalpha = -alpha;
    acc = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * T + threadIdx.x; i < c.n; i += int64_t(G) * T) {
      const double pi = __dadd_rn(c.r[i], __dmul_rn(beta, c.p[i]));  // xpby(r, beta, p)
      c.p[i] = pi;
      c.x[i] = __dadd_rn(c.x[i], __dmul_rn(alpha, pi));                 // axpy(alpha, p, x)
      const double ri = __dadd_rn(c.r[i], __dmul_rn(nalpha, c.a.v[i]));  // axpy(-alpha, q, r)
      c.r[i] = ri;
      acc = fma(ri, ri, acc);
    }
    acc = block_sum<T>(acc, red);
    if (threadIdx.x == 0) c.part_b[blockIdx.x] = acc;
    sk_jitter(40);
    grid.sync();
    const double rho_next = block_broadcast_sum<T>(c.part_b, G, red, &bcast);
    beta = rho_next / rho;
    rho = rho_next;
    ++it;
    if (it >= max_iter) status = kMaxIter;
    else if (sqrt(rho_next) <= target) status = kCheck;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->rho = rho;
    st->beta = beta;
    st->alpha = alpha;
    st->pq = pq;
    st->it = it;
    st->status = status;
  }
}

// Co-resident grid for k_cg2d_coop (0: cooperative launch unavailable):
// every SM's resident CTAs, no more than the tiles / rows need.
int coop_grid_size(int tiles, int64_t n) {
  int dev = 0, coop = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (!coop || sms <= 0) return 0;
  if (cudaFuncSetAttribute(k_cg2d_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, CoopTile::SMEM_BYTES_CG) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg2d_coop, CoopTile::THREADS,
                                                    CoopTile::SMEM_BYTES_CG) != cudaSuccess ||
      per_sm <= 0) {
    cudaGetLastError();
    return 0;
  }
  const int64_t need = std::max<int64_t>(tiles, (n + CoopTile::THREADS - 1) / CoopTile::THREADS);
  return int(std::min<int64_t>(int64_t(per_sm) * sms, need));
}

}  // namespace

// A CG workspace (r, p, q, partials, device state) plus the captured graph of
// `check_every` iterations for one solution pointer x. Reused across solves
// (the IMEX stepper solves one system per time step).
struct CgPlan {
  CgOperator op;
  int64_t n = 0;
  int grid = 0;
  int check_every = 64;
  char* ws = nullptr;
  CgState* st = nullptr;  // device
  double* partials = nullptr;
  double *r = nullptr, *p = nullptr, *q = nullptr;
  // fused2d: 2D class-1 stencil operator; each iteration is two kernels,
  // [q = A (r + beta p) ; alpha] and [p = r + beta p ; x, r update ; beta]
  bool fused2d = false;
  // coop: fused2d iterations run by k_cg2d_coop (one cooperative launch per
  // round of iterations) instead of the iteration graph
  bool coop = false;
  int coop_grid = 0;
  double* part_b = nullptr;
  cudaGraphExec_t exec = nullptr;
  const double* graph_x = nullptr;
  bool device_loop = false;  // exec = while(status == running) { iteration } on the device
  bool pq_fused = false;     // 3D streaming stencil: the apply reduces p.q itself
  // padded: radius-4 3D stencil on a non-periodic grid; K3 also writes a
  // ghost-padded copy of p (ppad, layout pl) and the apply reads it with the
  // 16-byte loader instead of the 8-byte boundary-map loader (config 5,
  // 255^3: apply 215 -> 130 us, iteration 455 -> 415 us; p.q stays a separate
  // pass: in the apply's epilogue it measured 511 us per iteration)
  bool padded = false;
  PadLayout pl;
  double* ppad = nullptr;
  int kpi = 0;  // kernels one iteration launches (counted while capturing)
  int kernels_per_iteration() const { return kpi ? kpi : (fused2d ? 2 : ((op.m || pq_fused) ? 3 : 4)); }

  ~CgPlan() {
    if (exec) cudaGraphExecDestroy(exec);
    if (ws) cudaFree(ws);
    if (ppad) cudaFree(ppad);
  }
  // warp per row, 8 warps per block, 8 blocks per SM resident
  unsigned pad_grid() const { return unsigned(std::min<int64_t>((pl.un[1] * pl.un[2] + 7) / 8, int64_t(kNumSMs) * 8)); }
  // after p was set outside the iteration (x0 = 0 start, restart)
  int refresh_pad(cudaStream_t stream) {
    if (!padded) return SK_OK;
    k_pad_fill<<<pad_grid(), 256, 0, stream>>>(p, ppad, pl);
    SK_LAUNCH_CHECK("k_pad_fill");
    return SK_OK;
  }

  // q = A p (+ p.q, alpha)
  int launch_q(cudaStream_t stream) {
    if (op.m) {
      const sk_csr* m = op.m;
      if (m->index_bits == 32)
        k1_spmv_pq<int32_t><<<grid, kT, 0, stream>>>(n, m->sell_ptr, m->sell_len,
                                                      static_cast<const int32_t*>(m->sell_col), m->sell_val, p, q,
                                                      st, partials);
      else
        k1_spmv_pq<int64_t><<<grid, kT, 0, stream>>>(n, m->sell_ptr, m->sell_len,
                                                      static_cast<const int64_t*>(m->sell_col), m->sell_val, p, q,
                                                      st, partials);
      SK_LAUNCH_CHECK("k1_spmv_pq");
      return SK_OK;
    }
    const int f = launch_apply_pq(op.s, op.g, p, q, st, partials, stream);  // fused p.q (3D streaming stencils)
    if (f != kApplyPqUnsupported) return f;
    if (padded) {
      if (option(SK_OPT_CG_PQ)) {  // fused p.q (factored 73-point apply on the padded p)
        const int e = launch_apply_padded(op.s, op.g, ppad + pl.at(0, 0, 0), pl.px, pl.plane, q, stream, st, partials);
        if (e != kApplyPqUnsupported) return e;
      }
      if (int e = launch_apply_padded(op.s, op.g, ppad + pl.at(0, 0, 0), pl.px, pl.plane, q, stream)) return e;
    } else if (int e = launch_apply(op.s, op.g, p, q, stream)) {
      return e;
    }
    k_pq<<<grid, kT, 0, stream>>>(n, p, q, st, partials);
    SK_LAUNCH_CHECK("k_pq");
    return SK_OK;
  }
  int true_residual(const double* x, const double* b, double* out, cudaStream_t stream) {
    if (op.m) {
      const sk_csr* m = op.m;
      if (m->index_bits == 32)
        k_true_residual<int32_t><<<grid, kT, 0, stream>>>(n, m->sell_ptr, m->sell_len,
                                                           static_cast<const int32_t*>(m->sell_col), m->sell_val, x, b,
                                                           q, st, partials);
      else
        k_true_residual<int64_t><<<grid, kT, 0, stream>>>(n, m->sell_ptr, m->sell_len,
                                                           static_cast<const int64_t*>(m->sell_col), m->sell_val, x, b,
                                                           q, st, partials);
      SK_LAUNCH_CHECK("k_true_residual");
    } else {
      if (int e = launch_apply(op.s, op.g, x, q, stream)) return e;
      k_resid<<<grid, kT, 0, stream>>>(n, b, q, st, partials);
      SK_LAUNCH_CHECK("k_resid");
    }
    SK_CUDA_TRY(cudaMemcpyAsync(out, &st->scalar_out, sizeof(double), cudaMemcpyDeviceToHost, stream));
    SK_CUDA_TRY(cudaStreamSynchronize(stream));
    *out = std::sqrt(*out);
    return SK_OK;
  }
  template <int OP>
  int reduce(const double* a, double* out, cudaStream_t stream) {
    k_reduce<OP><<<grid, kT, 0, stream>>>(n, a, st, partials);
    SK_LAUNCH_CHECK("k_reduce");
    SK_CUDA_TRY(cudaMemcpyAsync(out, &st->scalar_out, sizeof(double), cudaMemcpyDeviceToHost, stream));
    SK_CUDA_TRY(cudaStreamSynchronize(stream));
    return SK_OK;
  }
  // The iteration graph updating x: a device-side while loop over one
  // iteration (conditional node; one launch runs until the status leaves
  // RUNNING), or, where conditional nodes are unavailable, check_every
  // unrolled iterations whose kernels become no-ops after convergence.
  int ensure_graph(double* x, cudaStream_t stream) {
    if (exec && graph_x == x) return SK_OK;
    if (exec) {
      cudaGraphExecDestroy(exec);
      exec = nullptr;
    }
    cudaStream_t cap = stream ? stream : capture_stream();
    if (option(SK_OPT_CG_DEVICE_LOOP) && build_loop_graph(x, cap) == SK_OK) {
      device_loop = true;
      graph_x = x;
      return SK_OK;
    }
    cudaGetLastError();  // clear a failed attempt
    device_loop = false;
    SK_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    int st_ = SK_OK;
    const int64_t l0 = g_launches.load();
    for (int k = 0; k < check_every && st_ == SK_OK; ++k) st_ = iteration(x, cap, false, 0);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(cap, &graph);
    const int64_t captured = g_launches.load() - l0;
    if (st_ == SK_OK && check_every > 0) kpi = int(captured / check_every);
    g_launches -= captured;  // capture does not execute
    if (st_ != SK_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st_;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    graph_x = x;
    return SK_OK;
  }
  int launch_coop(double* x, cudaStream_t stream) {
    Coop2DArgs c{};
    cg_apply_2d_args(op.s, op.g, p, r, q, &c.a);
    c.x = x;
    c.p = p;
    c.r = r;
    c.part_a = partials;
    c.part_b = part_b;
    c.n = n;
    c.tiles_x = int((op.g.un[0] + 63) / 64);
    c.tiles = cg_apply_2d_ctas(op.s, op.g);
    CgState* stp = st;
    void* args[] = {&c, &stp};
    SK_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_cg2d_coop), dim3(unsigned(coop_grid)),
                                            dim3(CoopTile::THREADS), args, CoopTile::SMEM_BYTES_CG, stream));
    SK_LAUNCH_CHECK("k_cg2d_coop");
    return SK_OK;
  }
  int iteration(double* x, cudaStream_t cap, bool cond, cudaGraphConditionalHandle h) {
    if (fused2d) {
      if (int e = launch_cg_apply_2d(op.s, op.g, p, r, q, st, partials, cap)) return e;
      if (cond)
        k2_update_rr<true, true><<<grid, kT, 0, cap>>>(n, p, q, x, r, st, partials, h);
      else
        k2_update_rr<false, true><<<grid, kT, 0, cap>>>(n, p, q, x, r, st, partials, h);
      SK_LAUNCH_CHECK("k2_update_rr");
      return SK_OK;
    }
    if (int e = launch_q(cap)) return e;
    k2_update_rr<false, false><<<grid, kT, 0, cap>>>(n, p, q, x, r, st, partials, h);
    SK_LAUNCH_CHECK("k2_update_rr");
    if (padded) {
      if (cond)
        k3_xpby_pad<true><<<pad_grid(), 256, 0, cap>>>(r, p, ppad, pl, st, h);
      else
        k3_xpby_pad<false><<<pad_grid(), 256, 0, cap>>>(r, p, ppad, pl, st, h);
    } else if (cond) {
      k3_xpby<true><<<grid, kT, 0, cap>>>(n, r, p, st, h);
    } else {
      k3_xpby<false><<<grid, kT, 0, cap>>>(n, r, p, st, h);
    }
    SK_LAUNCH_CHECK("k3_xpby");
    return SK_OK;
  }
  int build_loop_graph(double* x, cudaStream_t cap) {
    cudaGraph_t graph = nullptr;
    if (cudaGraphCreate(&graph, 0) != cudaSuccess) return SK_ERR_CUDA;
    struct G {
      cudaGraph_t g;
      ~G() { cudaGraphDestroy(g); }
    } guard{graph};
    cudaGraphConditionalHandle h;
    if (cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault) != cudaSuccess) return SK_ERR_CUDA;
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    if (cudaGraphAddNode(&node, graph, nullptr, 0, &cp) != cudaSuccess) return SK_ERR_CUDA;
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if (cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
        cudaSuccess)
      return SK_ERR_CUDA;
    // body: kLoopUnroll iterations (no-ops once the status leaves RUNNING),
    // the last one publishing the loop condition
    int st_ = SK_OK;
    const int64_t l0 = g_launches.load();
    for (int k = 0; k < kLoopUnroll && st_ == SK_OK; ++k) st_ = iteration(x, cap, k + 1 == kLoopUnroll, h);
    cudaGraph_t out = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cap, &out);
    const int64_t captured = g_launches.load() - l0;
    if (st_ == SK_OK) kpi = int(captured / kLoopUnroll);
    g_launches -= captured;  // capture does not execute
    if (st_ != SK_OK || e != cudaSuccess) return SK_ERR_CUDA;
    if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
      exec = nullptr;
      return SK_ERR_CUDA;
    }
    return SK_OK;
  }
};

int cg_plan_create(const CgOperator& op, int check_every, cudaStream_t stream, CgPlan** out) {
  *out = nullptr;
  auto* pl = new CgPlan;
  pl->op = op;
  pl->n = op.n;
  pl->check_every = check_every > 0 ? check_every : 64;
  const int64_t g = (op.n + kT - 1) / kT;
  pl->grid = int(g > int64_t(kNumSMs) * 8 ? int64_t(kNumSMs) * 8 : (g > 0 ? g : 1));
  int partials = pl->grid;
  if (op.s) {
    pl->pq_fused = apply_pq_supported(op.s, op.g);
    partials = std::max(partials, kNumSMs * 4);  // the 3D streaming apply's persistent grid (fused p.q)
    const int ctas = cg_apply_2d_ctas(op.s, op.g);
    if (ctas > 0 && option(SK_OPT_CG_FUSED)) {
      pl->fused2d = true;
      partials = std::max(partials, ctas);
      // cooperative kernel for small systems only: measured (tools/cg_fused_timing.py,
      // config 2's operator) 14.5 vs 16-21 us/iteration at 65k unknowns, but
      // slower than the two-kernel graph from 261k up (fewer resident CTAs
      // per phase). SK_OPT_CG_COOP 1 / 0 forces it on / off.
      const int coop = option(SK_OPT_CG_COOP);
      const bool want = coop >= 0 ? coop == 1 : op.n <= kCoopMaxRows;
      if (want) pl->coop_grid = coop_grid_size(ctas, op.n);
      pl->coop = pl->coop_grid > 0;
    }
  }
  if (op.s && apply_padded_supported(op.s, op.g) && option(SK_OPT_CG_PADDED)) {
    bool per = true;
    for (int a = 0; a < 3; ++a) per &= op.g.bc[a] == SK_BC_PERIODIC;
    PadLayout& L = pl->pl;
    L.pad = 6;  // >= R + 1 (boundary + 4 ghosts), even: 16-byte aligned rows
    L.R = 4;
    for (int a = 0; a < 3; ++a) {
      L.un[a] = op.g.un[a];
      L.bc[a] = op.g.bc[a];
    }
    // interior rows start 128-byte aligned (whole-line stores from the p update;
    // the apply's 16-byte tile loads stay aligned): 16 columns before x = 0,
    // >= pad after the last, the pitch a multiple of 16
    L.padx = 16;
    L.px = (L.padx + op.g.un[0] + L.pad + 15) / 16 * 16;
    L.py = op.g.un[1] + 2 * L.pad;
    L.plane = L.px * L.py;
    const size_t elems = size_t(L.plane) * size_t(op.g.un[2] + 2 * L.pad);
    // the 8-byte boundary-map loader is the slow case; periodic grids already take the 16-byte path
    if (!per && op.g.un[0] >= 4 && op.g.un[1] >= 4 && op.g.un[2] >= 4 && L.plane * (op.g.un[2] + 8) < (int64_t(1) << 31)) {
      if (cudaMalloc(reinterpret_cast<void**>(&pl->ppad), elems * sizeof(double)) != cudaSuccess) {
        delete pl;
        return fail(SK_ERR_OUT_OF_MEMORY, "cg padded p");
      }
      if (cudaMemsetAsync(pl->ppad, 0, elems * sizeof(double), stream) != cudaSuccess) {
        delete pl;
        return fail(SK_ERR_CUDA, "cg padded p init");
      }
      pl->padded = true;
    }
  }
  if (op.m) {
    if (int e = csr_build_sell(const_cast<sk_csr*>(op.m), stream)) {  // before any graph capture
      delete pl;
      return e;
    }
  }
  const size_t vec = sizeof(double) * size_t(op.n > 0 ? op.n : 1);
  const size_t ws_bytes =
      3 * vec + sizeof(double) * (size_t(partials) + size_t(pl->coop_grid)) + sizeof(CgState) + 256;
  if (cudaMalloc(reinterpret_cast<void**>(&pl->ws), ws_bytes) != cudaSuccess) {
    delete pl;
    return fail(SK_ERR_OUT_OF_MEMORY, "cg workspace");
  }
  pl->r = reinterpret_cast<double*>(pl->ws);
  pl->p = pl->r + op.n;
  pl->q = pl->p + op.n;
  pl->partials = pl->q + op.n;
  pl->part_b = pl->partials + partials;
  pl->st = reinterpret_cast<CgState*>((reinterpret_cast<uintptr_t>(pl->part_b + pl->coop_grid) + 127) &
                                      ~uintptr_t(127));
  *out = pl;
  return SK_OK;
}

void cg_plan_destroy(CgPlan* p) { delete p; }

int cg_plan_solve(CgPlan* s, const double* b, double* x, const sk_solve_options* o, sk_solve_report* rep,
                  cudaStream_t stream) {
  const int64_t n = s->n;
  sk_solve_options opts{1e-10, 0, 0, 0, 0, 0};
  if (o) opts = *o;
  const int64_t max_iter = opts.max_iter > 0 ? opts.max_iter : 10 * n;  // linalg.cpp:20
  sk_solve_report report{0, 0, 0.0, 0.0};
  if (rep) *rep = report;
  if (n == 0) return SK_OK;
  const size_t vec = sizeof(double) * size_t(n);

  SK_CUDA_TRY(cudaMemsetAsync(s->st, 0, sizeof(CgState), stream));
  double bb = 0;
  if (int e = s->reduce<0>(b, &bb, stream)) return e;
  const double bnorm = std::sqrt(bb);  // :23
  if (bnorm == 0.0) {                  // :24
    SK_CUDA_TRY(cudaMemsetAsync(x, 0, vec, stream));
    return SK_OK;
  }
  double rho0 = bb;
  if (opts.use_initial_guess) {
    // extension: r = b - M x0, p = r (the restart kernel computes exactly that)
    double dummy = 0;
    if (int e = s->true_residual(x, b, &dummy, stream)) return e;
    k_restart<<<s->grid, kT, 0, stream>>>(n, b, s->q, s->r, s->p, s->st, s->partials);
    SK_LAUNCH_CHECK("k_restart");
    if (int e = s->refresh_pad(stream)) return e;
    SK_CUDA_TRY(cudaMemcpyAsync(&rho0, &s->st->rho, sizeof(double), cudaMemcpyDeviceToHost, stream));
    SK_CUDA_TRY(cudaStreamSynchronize(stream));
  } else {
    // x = 0, r = p = b (linalg.cpp:22)
    SK_CUDA_TRY(cudaMemsetAsync(x, 0, vec, stream));
    SK_CUDA_TRY(cudaMemcpyAsync(s->r, b, vec, cudaMemcpyDeviceToDevice, stream));
    SK_CUDA_TRY(cudaMemcpyAsync(s->p, b, vec, cudaMemcpyDeviceToDevice, stream));
    if (int e = s->refresh_pad(stream)) return e;
  }
  const double target = opts.rel_tol * bnorm;
  CgState h{};
  h.rho = rho0;  // rho = r.r (:27)
  h.target = target;
  h.it = 0;
  h.max_iter = max_iter;
  h.status = kRunning;
  SK_CUDA_TRY(cudaMemcpyAsync(s->st, &h, sizeof(CgState), cudaMemcpyHostToDevice, stream));
  if (!s->coop)
    if (int e = s->ensure_graph(x, stream)) return e;

  int64_t restarts = 0;
  double rho = rho0;
  int64_t it = 0;
  int status = kRunning;
  for (;;) {
    if (it >= max_iter) break;
    if (std::sqrt(rho) <= target) {
      if (opts.accept_recurrence) break;  // extension: report the true residual instead
      // recurrence says converged; accept only if the true residual agrees (:31-47)
      double true_res = 0;
      if (int e = s->true_residual(x, b, &true_res, stream)) return e;
      if (true_res <= target) break;
      k_restart<<<s->grid, kT, 0, stream>>>(n, b, s->q, s->r, s->p, s->st, s->partials);
      SK_LAUNCH_CHECK("k_restart");
      if (int e = s->refresh_pad(stream)) return e;
      restarts++;
    }
    if (s->coop) {
      if (int e = s->launch_coop(x, stream)) return e;
    } else {
      SK_CUDA_TRY(cudaGraphLaunch(s->exec, stream));
    }
    SK_CUDA_TRY(cudaMemcpyAsync(&h, s->st, sizeof(CgState), cudaMemcpyDeviceToHost, stream));
    SK_CUDA_TRY(cudaStreamSynchronize(stream));
    // launched kernels: whole loop bodies up to the round that stopped
    const int64_t rounds = (h.it - it + kLoopUnroll) / kLoopUnroll;
    if (s->coop)
      g_launches += 1;
    else
      g_launches += int64_t(s->kernels_per_iteration()) *
                    (s->device_loop ? rounds * kLoopUnroll : int64_t(s->check_every));
    it = h.it;
    rho = h.rho;
    status = h.status;
    if (status == kNotPD) {
      report.iterations = it;
      report.restarts = restarts;
      if (rep) *rep = report;
      return fail(SK_ERR_NO_CONVERGENCE, "matrix is not positive definite on the Krylov space");
    }
    if (status == kMaxIter) break;
    if (status == kCheck) {
      h.status = kRunning;  // the check itself runs at the loop top
      SK_CUDA_TRY(cudaMemcpyAsync(&s->st->status, &h.status, sizeof(int), cudaMemcpyHostToDevice, stream));
    }
  }
  // final acceptance on the true residual (:59-66)
  double res = 0;
  if (int e = s->true_residual(x, b, &res, stream)) return e;
  report.iterations = it;
  report.restarts = restarts;
  report.true_rel_residual = res / bnorm;
  report.recurrence_rel_residual = std::sqrt(rho) / bnorm;
  if (rep) *rep = report;
  const bool converged = opts.accept_recurrence ? std::sqrt(rho) <= target : res <= target;
  if (!converged)
    return fail(SK_ERR_NO_CONVERGENCE, "cg stalled after " + std::to_string(it) + " iterations at relative residual " +
                                           std::to_string(res / bnorm));
  if (opts.deflate_mean) {  // :67-70
    double sum = 0;
    if (int e = s->reduce<1>(x, &sum, stream)) return e;
    const double mean = sum / double(n);
    k_shift<<<s->grid, kT, 0, stream>>>(n, x, mean);
    SK_LAUNCH_CHECK("k_shift");
    SK_CUDA_TRY(cudaStreamSynchronize(stream));
  }
  return SK_OK;
}

int cg_solve(const sk_csr* m, const double* b, double* x, const sk_solve_options* o, sk_solve_report* rep,
             cudaStream_t stream) {
  if (m->rows != m->cols) return fail(SK_ERR_SHAPE_MISMATCH, "cg_solve needs a square matrix");
  if (rep) *rep = sk_solve_report{0, 0, 0.0, 0.0};
  if (m->rows == 0) return SK_OK;
  // one cached plan per host thread: repeated solves on the same matrix reuse
  // the workspace and the captured iteration graph (matrix uids are unique)
  struct Cache {
    uint64_t uid = 0;
    int check_every = -1;
    uint64_t epoch = 0;
    CgPlan* plan = nullptr;
    ~Cache() { cg_plan_destroy(plan); }
  };
  thread_local Cache cache;
  const int ce = o ? o->check_every : 0;
  if (!cache.plan || cache.uid != m->uid || cache.check_every != ce || cache.epoch != option_epoch()) {
    if (cache.plan) {
      cudaDeviceSynchronize();  // the old workspace may still be in use by queued work
      cg_plan_destroy(cache.plan);
      cache.plan = nullptr;
    }
    CgOperator op;
    op.m = m;
    op.n = m->rows;
    if (int e = cg_plan_create(op, ce, stream, &cache.plan)) return e;
    cache.uid = m->uid;
    cache.check_every = ce;
    cache.epoch = option_epoch();
  }
  return cg_plan_solve(cache.plan, b, x, o, rep, stream);
}

// Matrix-free CG: the operator is the composed stencil applied by the
// streaming kernels on the grid's boundary kind (equal to assemble(s, g) in
// exact arithmetic; per-row sums in orbit order instead of column order).
int cg_solve_stencil(const sk_stencil* s, const GridInfo& g, const double* b, double* x, const sk_solve_options* o,
                     sk_solve_report* rep, cudaStream_t stream) {
  if (rep) *rep = sk_solve_report{0, 0, 0.0, 0.0};
  if (g.rows == 0) return SK_OK;
  struct Cache {
    uint64_t uid = 0;
    GridInfo g{};
    int check_every = -1;
    uint64_t epoch = 0;
    CgPlan* plan = nullptr;
    ~Cache() { cg_plan_destroy(plan); }
  };
  thread_local Cache cache;
  const int ce = o ? o->check_every : 0;
  bool hit = cache.plan && cache.uid == s->uid && cache.check_every == ce && cache.g.dim == g.dim &&
             cache.g.h == g.h && cache.epoch == option_epoch();
  for (int a = 0; a < 3 && hit; ++a) hit = cache.g.n[a] == g.n[a] && cache.g.bc[a] == g.bc[a];
  if (!hit) {
    if (cache.plan) {
      cudaDeviceSynchronize();
      cg_plan_destroy(cache.plan);
      cache.plan = nullptr;
    }
    CgOperator op;
    op.s = s;
    op.g = g;
    op.n = g.rows;
    if (int e = cg_plan_create(op, ce, stream, &cache.plan)) return e;
    cache.uid = s->uid;
    cache.g = g;
    cache.check_every = ce;
    cache.epoch = option_epoch();
  }
  return cg_plan_solve(cache.plan, b, x, o, rep, stream);
}

}  // namespace sk

using namespace sk;

extern "C" {

int sk_cg_solve_stencil(const sk_stencil* s, const sk_grid_desc* gd, const double* b, double* x,
                        const sk_solve_options* o, sk_solve_report* rep, void* stream) {
  if (!s) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  if (s->dim != g.dim) return fail(SK_ERR_DIM_MISMATCH, "stencil/grid dimension mismatch");
  if (int st = check_width(s, g)) return st;
  if (g.rows > 0 && (!b || !x)) return fail(SK_ERR_INVALID_ARGUMENT, "null vector");
  return cg_solve_stencil(s, g, b, x, o, rep, as_stream(stream));
}

int sk_cg_solve(const sk_csr* m, const double* b, double* x, const sk_solve_options* o, sk_solve_report* rep,
                void* stream) {
  if (!m) return fail(SK_ERR_INVALID_ARGUMENT, "null matrix");
  if (m->rows > 0 && (!b || !x)) return fail(SK_ERR_INVALID_ARGUMENT, "null vector");
  return cg_solve(m, b, x, o, rep, as_stream(stream));
}

int sk_cg_solve_host(const sk_csr* m, const double* b_host, double* x_host, const sk_solve_options* o,
                     sk_solve_report* rep) {
  if (!m) return fail(SK_ERR_INVALID_ARGUMENT, "null matrix");
  if (m->rows != m->cols) return fail(SK_ERR_SHAPE_MISMATCH, "cg_solve needs a square matrix");
  if (m->rows == 0) return SK_OK;
  // the last iterate is returned even on NoConvergence
  int solve_status = SK_OK;
  std::string msg;
  int st = host_roundtrip(b_host, size_t(m->rows), x_host, size_t(m->rows),
                          [&](const double* b, double* x, cudaStream_t s) {
                            if (o && o->use_initial_guess)
                              SK_CUDA_TRY(cudaMemcpyAsync(x, x_host, sizeof(double) * size_t(m->rows),
                                                          cudaMemcpyHostToDevice, s));
                            solve_status = cg_solve(m, b, x, o, rep, s);
                            if (solve_status != SK_OK && solve_status != SK_ERR_NO_CONVERGENCE) return solve_status;
                            if (solve_status != SK_OK) msg = sk_last_error();
                            return int(SK_OK);
                          });
  if (st != SK_OK) return st;
  if (solve_status != SK_OK) return fail(solve_status, msg.substr(msg.find(": ") + 2));
  return SK_OK;
}

}  // extern "C"
