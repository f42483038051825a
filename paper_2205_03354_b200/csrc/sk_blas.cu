// BLAS-1 kernels of the reference (kernels.cpp:19-60) on the device.
//
// axpy / xpby round exactly like the reference's Release build (separate
// multiply and add, no contraction), so they are bit-identical to
// kernels::serial::axpy / xpby (test_kernels.cpp:37-47). Reductions are
// deterministic two-level trees (per-CTA partials combined in index order by
// the last CTA); like the reference's OpenMP reductions they agree with the
// serial sum to rounding (test_kernels.cpp:49-60).
#include <cuda_runtime.h>

#include <cfloat>

#include "sk_common.cuh"

namespace sk {

namespace {

constexpr int kThreads = 256;

int reduce_grid(int64_t n) {
  const int64_t per = int64_t(kThreads) * 4;
  int64_t g = (n + per - 1) / per;
  if (g > int64_t(kNumSMs) * 8) g = int64_t(kNumSMs) * 8;
  return g < 1 ? 1 : int(g);
}

// op 0: sum a*b, 1: sum a, 2: sum a*a
template <int OP>
__global__ void __launch_bounds__(kThreads)
    reduce_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double* partials,
                  unsigned* counter, double* out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kThreads + threadIdx.x; i < n; i += int64_t(gridDim.x) * kThreads) {
    const double x = a[i];
    if (OP == 0) acc = fma(x, b[i], acc);
    if (OP == 1) acc += x;
    if (OP == 2) acc = fma(x, x, acc);
  }
  acc = block_sum<kThreads>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  if (last_block(counter)) {
    const double t = reduce_partials<kThreads>(partials, gridDim.x, sh);
    if (threadIdx.x == 0) *out = t;
  }
}

__global__ void __launch_bounds__(kThreads)
    minmax_kernel(int64_t n, const double* __restrict__ a, double* partials, unsigned* counter, double* out) {
  __shared__ double smin[32], smax[32];
  double lo = DBL_MAX, hi = -DBL_MAX;
  for (int64_t i = int64_t(blockIdx.x) * kThreads + threadIdx.x; i < n; i += int64_t(gridDim.x) * kThreads) {
    const double x = a[i];
    lo = fmin(lo, x);
    hi = fmax(hi, x);
  }
  auto block_minmax = [&](double& l, double& h) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      l = fmin(l, __shfl_xor_sync(0xffffffffu, l, o));
      h = fmax(h, __shfl_xor_sync(0xffffffffu, h, o));
    }
    __syncthreads();
    if (threadIdx.x % 32 == 0) {
      smin[threadIdx.x / 32] = l;
      smax[threadIdx.x / 32] = h;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      l = threadIdx.x < kThreads / 32 ? smin[threadIdx.x] : DBL_MAX;
      h = threadIdx.x < kThreads / 32 ? smax[threadIdx.x] : -DBL_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        l = fmin(l, __shfl_xor_sync(0xffffffffu, l, o));
        h = fmax(h, __shfl_xor_sync(0xffffffffu, h, o));
      }
    }
  };
  block_minmax(lo, hi);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = lo;
    partials[2 * blockIdx.x + 1] = hi;
  }
  if (last_block(counter)) {
    double l = DBL_MAX, h = -DBL_MAX;
    for (int i = threadIdx.x; i < int(gridDim.x); i += kThreads) {
      l = fmin(l, __ldcg(partials + 2 * i));
      h = fmax(h, __ldcg(partials + 2 * i + 1));
    }
    block_minmax(l, h);
    if (threadIdx.x == 0) {
      out[0] = l;
      out[1] = h;
    }
  }
}

// y[i] += a * x[i]   (kernels.cpp:29-33), no contraction
__global__ void axpy_kernel(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = __dadd_rn(y[i], __dmul_rn(a, x[i]));
}

// y[i] = x[i] + b * y[i]   (kernels.cpp:35-40), no contraction
__global__ void xpby_kernel(int64_t n, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = __dadd_rn(x[i], __dmul_rn(b, y[i]));
}

// Scratch for one host-visible reduction: partials, ticket, result.
struct Scratch {
  double* partials = nullptr;
  unsigned* counter = nullptr;
  double* out = nullptr;
  cudaStream_t stream = nullptr;
  ~Scratch() {
    if (partials) cudaFreeAsync(partials, stream);
  }
};

int make_scratch(Scratch& s, int grid, cudaStream_t stream) {
  s.stream = stream;
  const size_t pbytes = sizeof(double) * size_t(2 * grid);
  const size_t total = pbytes + 4 * sizeof(double) + 64;
  SK_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&s.partials), total, stream));
  s.out = s.partials + 2 * grid;
  s.counter = reinterpret_cast<unsigned*>(s.out + 4);
  SK_CUDA_TRY(cudaMemsetAsync(s.counter, 0, sizeof(unsigned), stream));
  return SK_OK;
}

template <int OP>
int host_reduce(int64_t n, const double* a, const double* b, double* out_host, cudaStream_t stream) {
  if (n < 0 || !out_host) return fail(SK_ERR_INVALID_ARGUMENT, "bad reduction arguments");
  if (n == 0) {
    *out_host = 0.0;
    return SK_OK;
  }
  if (!a || (OP == 0 && !b)) return fail(SK_ERR_INVALID_ARGUMENT, "null vector");
  const int grid = reduce_grid(n);
  Scratch s;
  if (int st = make_scratch(s, grid, stream)) return st;
  reduce_kernel<OP><<<grid, kThreads, 0, stream>>>(n, a, b, s.partials, s.counter, s.out);
  SK_LAUNCH_CHECK("reduce_kernel");
  SK_CUDA_TRY(cudaMemcpyAsync(out_host, s.out, sizeof(double), cudaMemcpyDeviceToHost, stream));
  SK_CUDA_TRY(cudaStreamSynchronize(stream));
  return SK_OK;
}

int elementwise_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > int64_t(kNumSMs) * 16) g = int64_t(kNumSMs) * 16;
  return g < 1 ? 1 : int(g);
}

}  // namespace

}  // namespace sk

using namespace sk;

extern "C" {

int sk_dot(int64_t n, const double* a, const double* b, double* out, void* stream) {
  return host_reduce<0>(n, a, b, out, as_stream(stream));
}

int sk_sum(int64_t n, const double* a, double* out, void* stream) {
  return host_reduce<1>(n, a, nullptr, out, as_stream(stream));
}

int sk_nrm2(int64_t n, const double* a, double* out, void* stream) {
  int st = host_reduce<2>(n, a, nullptr, out, as_stream(stream));
  if (st == SK_OK) *out = std::sqrt(*out);
  return st;
}

int sk_minmax(int64_t n, const double* a, double* lo, double* hi, void* stream_p) {
  // kernels.cpp:50-60 reads a[0] unconditionally: an empty span is undefined
  // there; here it is an error.
  if (n <= 0 || !a || !lo || !hi) return fail(SK_ERR_INVALID_ARGUMENT, "minmax needs a non-empty vector");
  cudaStream_t stream = as_stream(stream_p);
  const int grid = reduce_grid(n);
  Scratch s;
  if (int st = make_scratch(s, grid, stream)) return st;
  minmax_kernel<<<grid, kThreads, 0, stream>>>(n, a, s.partials, s.counter, s.out);
  SK_LAUNCH_CHECK("minmax_kernel");
  double r[2];
  SK_CUDA_TRY(cudaMemcpyAsync(r, s.out, 2 * sizeof(double), cudaMemcpyDeviceToHost, stream));
  SK_CUDA_TRY(cudaStreamSynchronize(stream));
  *lo = r[0];
  *hi = r[1];
  return SK_OK;
}

int sk_axpy(int64_t n, double a, const double* x, double* y, void* stream) {
  if (n < 0 || (n > 0 && (!x || !y))) return fail(SK_ERR_INVALID_ARGUMENT, "bad axpy arguments");
  if (n == 0) return SK_OK;
  axpy_kernel<<<elementwise_grid(n), 256, 0, as_stream(stream)>>>(n, a, x, y);
  SK_LAUNCH_CHECK("axpy_kernel");
  return SK_OK;
}

int sk_xpby(int64_t n, const double* x, double b, double* y, void* stream) {
  if (n < 0 || (n > 0 && (!x || !y))) return fail(SK_ERR_INVALID_ARGUMENT, "bad xpby arguments");
  if (n == 0) return SK_OK;
  xpby_kernel<<<elementwise_grid(n), 256, 0, as_stream(stream)>>>(n, x, b, y);
  SK_LAUNCH_CHECK("xpby_kernel");
  return SK_OK;
}

}  // extern "C"
