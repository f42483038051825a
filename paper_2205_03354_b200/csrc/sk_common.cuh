// Shared plumbing for the sm_100a stencil library: status/error handling,
// launch accounting, PTX wrappers for the bulk-copy + mbarrier pipeline.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>

#include "sk_cuda.h"

namespace sk {

// ---- errors ---------------------------------------------------------------
void set_error(int status, const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
extern std::atomic<int64_t> g_launches;
// sk_set_option state: current value, and a counter bumped on every change
// (cached graphs / plans record it and rebuild when it moves)
int option(int id);
uint64_t option_epoch();

#define SK_CUDA_TRY(expr)                                        \
  do {                                                           \
    cudaError_t sk_e_ = (expr);                                  \
    if (sk_e_ != cudaSuccess) return ::sk::cuda_fail(sk_e_, #expr); \
  } while (0)

// After a kernel launch: count it and surface launch-configuration errors.
#define SK_LAUNCH_CHECK(name)                                          \
  do {                                                                 \
    ::sk::g_launches.fetch_add(1, std::memory_order_relaxed);          \
    cudaError_t sk_e_ = cudaGetLastError();                            \
    if (sk_e_ != cudaSuccess) return ::sk::cuda_fail(sk_e_, name);     \
  } while (0)

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// ---- grid helpers ----------------------------------------------------------
struct GridInfo {
  int dim;
  int64_t n[3];   // points per axis incl. boundary
  int64_t un[3];  // unknowns per axis (grid.cpp:27-29)
  int bc[3];
  double h;
  int64_t rows;
};
int grid_info(const sk_grid_desc* g, GridInfo* out);  // validates like GridSpec::validate
double pow_int(double base, int exp);                  // grid.cpp:10-15, bit-identical

constexpr int kNumSMs = 148;

// ---- device helpers --------------------------------------------------------
// Race amplification (test builds only, -DSK_RACE_JITTER, tools/race_jitter.py):
// a pseudo-random sleep of up to ~1 us for one thread in four at every
// synchronisation point of the kernels, so a missing barrier / fence /
// mbarrier wait shows up as a changed result instead of hiding behind lucky
// timing. Compiles to nothing in the product build.
#ifdef SK_RACE_JITTER
__device__ __forceinline__ void sk_jitter(unsigned site) {
  unsigned t;
  asm volatile("mov.u32 %0, %%clock;" : "=r"(t));
  unsigned h = t ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu) ^ (site * 0xC2B2AE35u);
  h ^= h >> 13;
  h *= 0x5BD1E995u;
  h ^= h >> 15;
  if ((h & 3u) == 0u) __nanosleep((h >> 16) & 1023u);
}
#else
__device__ __forceinline__ void sk_jitter(unsigned) {}
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// one of the barrier's expected arrivals, triggered when all of this thread's
// prior cp.async copies have landed (the pending count is not incremented)
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// plain arrival (release, CTA scope): count one of the barrier's expected arrivals
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 3D tiled tensor copy global -> shared (TMA engine, SASS UTMALDG): the box of
// the tensor map at element coordinates (x, y, z) lands densely at dst
// (128-byte aligned), completing its bytes on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst_smem, const void* tmap, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst_smem)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// the same with an L2 eviction-priority hint (createpolicy.fractional)
template <int HINT>  // 0 evict_normal (no hint), 1 evict_last, 2 evict_first
__device__ __forceinline__ void tma_load_3d_hint(void* dst_smem, const void* tmap, int x, int y, int z, uint64_t* bar) {
  if constexpr (HINT == 0) {
    tma_load_3d(dst_smem, tmap, x, y, z, bar);
  } else {
    uint64_t pol;
    if constexpr (HINT == 1)
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
        "{%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst_smem)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
  }
}

// order this thread's prior generic-proxy shared accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Before a TMA refill of a ring slot that generic loads read earlier (WAR).
// The reads are ordered before the refill by the mbarrier that frees the slot
// (every reader arrives, release; the producer waits, acquire) -- the usual
// TMA-pipeline hand-off. An explicit proxy fence (-DSK_TMA_WAR_FENCE=1)
// compiles to MEMBAR.ALL.CTA, which also waits for the producer thread's
// outstanding global stores: measured 55.3 vs 54.9 us per 256^3 CH step.
#ifndef SK_TMA_WAR_FENCE
#define SK_TMA_WAR_FENCE 0
#endif
__device__ __forceinline__ void tma_war_fence() {
#if SK_TMA_WAR_FENCE
  fence_proxy_async_smem();
#endif
}

// Per-thread asynchronous global->shared copies (LDGSTS), L1-bypassing.
__device__ __forceinline__ void cp_async16(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// i in [-n, 2n): periodic wrap without a 64-bit division
__device__ __forceinline__ int64_t wrap1(int64_t i, int64_t n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// Streaming 128-bit global store of two doubles (outputs are not re-read).
__device__ __forceinline__ void st_cs_f64x2(double* p, double a, double b) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction (fixed tree): result valid in thread 0.
template <int THREADS>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  static_assert(THREADS % 32 == 0 && THREADS <= 1024, "block size");
  v = warp_sum(v);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  sk_jitter(1);
  __syncthreads();  // sh may be reused back to back
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < THREADS / 32 ? sh[lane] : 0.0;
    v = warp_sum(v);
  }
  return v;
}

// "Last block done" ticket: returns true in every thread of the CTA that
// finishes last; that CTA then combines the per-CTA partials in index order,
// so the two-level reduction is deterministic for a given grid size.
__device__ __forceinline__ bool last_block(unsigned* counter, unsigned nblocks) {
  __shared__ bool is_last;
  sk_jitter(2);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned ticket = atomicAdd(counter, 1u);
    is_last = ticket == nblocks - 1;
    if (is_last) *counter = 0;  // reset for the next launch
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}
__device__ __forceinline__ bool last_block(unsigned* counter) { return last_block(counter, gridDim.x); }

// Sum the per-CTA partials in a fixed order (called by the last CTA only).
template <int THREADS>
__device__ __forceinline__ double reduce_partials(const double* partials, int count, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < count; i += THREADS) v += __ldcg(partials + i);
  return block_sum<THREADS>(v, sh);
}

// plain 128-bit shared load: unlike a volatile-asm ld.shared the compiler may
// hoist it across independent work
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// Extended unknown index i along an axis with `un` unknowns -> the unknown it
// reads and a factor (assemble's boundary handling, grid.cpp:104-120):
// periodic wraps; simply supported reflects oddly about the boundary point
// (factor -1), clamped evenly (factor +1); the boundary points themselves are
// zero (factor 0). Indices beyond one reflection (partial-tile padding,
// never an output's neighbour) read as zero.
__device__ __forceinline__ int64_t bc_map(int64_t i, int64_t un, int bc, double& factor) {
  if (i >= 0 && i < un) return i;
  if (bc == SK_BC_PERIODIC) {
    i %= un;
    return i < 0 ? i + un : i;
  }
  int64_t gi = i + 1;  // grid index; boundary points 0 and un + 1
  const int64_t last = un + 1;
  if (gi == 0 || gi == last) {
    factor = 0.0;
    return 0;
  }
  gi = gi < 0 ? -gi : 2 * last - gi;
  if (gi < 1 || gi > un) {  // beyond one reflection: only partial-tile padding reads it
    factor = 0.0;
    return 0;
  }
  if (bc == SK_BC_SIMPLY_SUPPORTED) factor = -factor;
  return gi - 1;
}

__device__ __forceinline__ int64_t wrap_idx(int64_t i, int64_t n) {
  i %= n;
  return i < 0 ? i + n : i;
}

}  // namespace sk
