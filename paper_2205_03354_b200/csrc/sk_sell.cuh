// SELL-32 row evaluation shared by the SpMV and the CG kernels.
//
// Layout (built from the CSR by csr_build_sell): rows are grouped in slices
// of 32; slice s stores entry k of its row (32 s + lane) at
// sell_ptr[s] + 32 k + lane. One thread per row walks k = 0..len-1, so the
// 32 lanes of a warp read 32 consecutive values (and indices) per step —
// coalesced — while each row is still accumulated sequentially in column
// order with separate multiply and add: bit-identical to the reference's
// serial csr_matvec (kernels.cpp:13-15). Matrix data is streamed past L1
// (no_allocate) so L1 keeps the x gathers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sk {

__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int64_t ld_stream_idx(const int64_t* p) {
  int64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int64_t ld_stream_idx(const int32_t* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <class IDX>
__device__ __forceinline__ double sell_row_dot(int64_t i, const int64_t* __restrict__ sp, const int32_t* __restrict__ len,
                                               const IDX* __restrict__ col, const double* __restrict__ val,
                                               const double* __restrict__ x) {
  int64_t k0 = __ldg(sp + (i >> 5)) + (i & 31);
  const int L = __ldg(len + i);
  double acc = 0.0;
#pragma unroll 4
  for (int k = 0; k < L; ++k, k0 += 32) {
    const double v = ld_stream_f64(val + k0);
    const int64_t c = ld_stream_idx(col + k0);
    acc = __dadd_rn(acc, __dmul_rn(v, __ldg(x + c)));
  }
  return acc;
}

}  // namespace sk
