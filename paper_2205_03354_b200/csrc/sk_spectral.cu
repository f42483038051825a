// Spectral tools on the device:
//
//   power_iteration   linalg.cpp:74-106   spectral radius of an assembled
//                     operator; the whole loop (SpMV + Rayleigh quotient +
//                     normalisation + the geometric-tail stopping rule) runs
//                     as a device-side while loop (conditional graph node)
//   periodic_spectrum linalg.cpp:149-222  every Fourier mode's eigenvalue of a
//                     stencil on an all-periodic grid, spectral radius,
//                     condition estimate, and the continuous-torus symbol
//                     maximum (grid sampling on the device, the
//                     golden-section polish of refine_symbol_max, :110-147,
//                     on the host with the reference's libm evaluation).
#include <cuda_runtime.h>

#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdlib>
#include <random>
#include <vector>

#include "sk_internal.hpp"
#include "sk_sell.cuh"

namespace sk {
namespace {

constexpr int kT = 256;
enum : int { kPiRunning = 0, kPiDone = 1, kPiZero = 2, kPiMaxIter = 3 };

struct PiState {
  double lambda, prev, prev_delta, wn, result, tol;
  int64_t it, max_iter;
  int status;
  unsigned counter[2];
};

// w = M v (reference row order and rounding), partials of v.w and w.w; the
// last CTA applies one iteration of the stopping rule (linalg.cpp:85-103)
template <class IDX>
__global__ void __launch_bounds__(kT) k_pi_spmv(int64_t n, const int64_t* __restrict__ sp,
                                                const int32_t* __restrict__ len, const IDX* __restrict__ col,
                                                const double* __restrict__ val, const double* __restrict__ v,
                                                double* __restrict__ w, PiState* st, double2* partials) {
  if (st->status != kPiRunning) return;
  __shared__ double sh[32];
  double vw = 0.0, ww = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) {
    const double wi = sell_row_dot(i, sp, len, col, val, v);
    w[i] = wi;
    vw = fma(v[i], wi, vw);
    ww = fma(wi, wi, ww);
  }
  vw = block_sum<kT>(vw, sh);
  ww = block_sum<kT>(ww, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = make_double2(vw, ww);
  if (last_block(&st->counter[0])) {
    // fixed-order final reduction (deterministic)
    double a = 0.0, b = 0.0;
    for (int k = threadIdx.x; k < int(gridDim.x); k += kT) {
      const double2 pk = __ldcg(&partials[k]);
      a += pk.x;
      b += pk.y;
    }
    a = block_sum<kT>(a, sh);
    b = block_sum<kT>(b, sh);
    if (threadIdx.x == 0) {
      const double lambda = a;  // Rayleigh quotient, |v| = 1
      const double wn = sqrt(b);
      const int64_t it = st->it;
      st->lambda = lambda;
      st->wn = wn;
      if (wn == 0.0) {  // hit the kernel exactly
        st->status = kPiZero;
        st->result = 0.0;
        return;
      }
      bool done = false;
      if (it > 0) {
        const double delta = fabs(lambda - st->prev);
        if (it > 1 && st->prev_delta > 0 && delta < st->prev_delta) {
          const double r = delta / st->prev_delta;  // geometric tail estimate
          const double tail = delta * r / (1.0 - r);
          if (tail <= 0.25 * st->tol * fabs(lambda)) done = true;
        }
        if (delta == 0.0) done = true;
      }
      if (done) {
        st->status = kPiDone;
        st->result = fabs(lambda);
      }
      st->prev_delta = it > 0 ? fabs(lambda - st->prev) : 0.0;
      st->prev = lambda;
      st->it = it + 1;
      if (!done && st->it >= st->max_iter) st->status = kPiMaxIter;
    }
  }
}

// v = w / wn ; publishes "keep iterating" for the device loop
template <bool COND>
__global__ void k_pi_scale(int64_t n, const double* __restrict__ w, double* __restrict__ v, const PiState* st,
                           cudaGraphConditionalHandle cond) {
  if constexpr (COND) {
    if (blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, st->status == kPiRunning ? 1u : 0u);
  }
  const double wn = st->wn;
  if (wn == 0.0) return;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    v[i] = __ddiv_rn(w[i], wn);
}

__global__ void k_div(int64_t n, double* __restrict__ v, const double* nv) {
  const double d = *nv;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    v[i] = __ddiv_rn(v[i], d);
}

__global__ void k_sumsq_sqrt(int64_t n, const double* __restrict__ v, double* partials, unsigned* counter,
                             double* out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT)
    acc = fma(v[i], v[i], acc);
  acc = block_sum<kT>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  if (last_block(counter)) {
    const double t = reduce_partials<kT>(partials, gridDim.x, sh);
    if (threadIdx.x == 0) *out = sqrt(t);
  }
}

// ---- periodic spectrum ----
struct SpecArgs {
  int dim, nent;
  int64_t n[3];
  const int* off;       // nent * 3
  const double* coeff;  // nent: Rational::to_double
  double shift, scale;  // affine_shift, affine_scale * pow_int(h, h_power)
};

// symbol_nd (stability.cpp:45-55) in entry order: acc += coeff * (cos phase, sin phase)
__device__ __forceinline__ void symbol_dev(const SpecArgs& a, const double* theta, double& re, double& im) {
  re = 0.0;
  im = 0.0;
  for (int e = 0; e < a.nent; ++e) {
    double phase = 0.0;
    for (int ax = 0; ax < a.dim; ++ax) phase = __dadd_rn(phase, __dmul_rn(theta[ax], double(a.off[e * 3 + ax])));
    // sin odd / cos even exactly (as libm's are), so symmetric stencils'
    // imaginary parts cancel exactly as in the reference
    double s, c;
    sincos(fabs(phase), &s, &c);
    s = copysign(s, phase);
    re = __dadd_rn(re, __dmul_rn(a.coeff[e], c));
    im = __dadd_rn(im, __dmul_rn(a.coeff[e], s));
  }
}

__device__ __forceinline__ double two_pi_frac(int64_t k, int64_t na) {
  return __ddiv_rn(__dmul_rn(2.0 * 3.141592653589793, double(k)), double(na));
}

// eigenvalue of every mode (:172-181) and |ev|
__global__ void k_eigen(int64_t modes, SpecArgs a, double2* __restrict__ ev, double* __restrict__ mag) {
  for (int64_t m = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; m < modes; m += int64_t(gridDim.x) * blockDim.x) {
    int64_t rem = m;
    double theta[3] = {0, 0, 0};
    for (int ax = 0; ax < a.dim; ++ax) {
      theta[ax] = two_pi_frac(rem % a.n[ax], a.n[ax]);
      rem /= a.n[ax];
    }
    double re, im;
    symbol_dev(a, theta, re, im);
    const double er = __dadd_rn(a.shift, __dmul_rn(a.scale, re)), ei = __dmul_rn(a.scale, im);
    ev[m] = make_double2(er, ei);
    mag[m] = hypot(er, ei);
  }
}

// max of mag, then min of mag over mag > thr  (order-free: exact)
__global__ void k_maxmin(int64_t n, const double* __restrict__ mag, double thr, int mode, double* partials,
                         unsigned* counter, double* out) {
  __shared__ double sh[32];
  double acc = mode == 0 ? 0.0 : INFINITY;
  for (int64_t i = int64_t(blockIdx.x) * kT + threadIdx.x; i < n; i += int64_t(gridDim.x) * kT) {
    const double v = mag[i];
    if (mode == 0) acc = fmax(acc, v);
    else if (v > thr) acc = fmin(acc, v);
  }
  // block reduction of max / min
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_down_sync(0xffffffffu, acc, o);
    acc = mode == 0 ? fmax(acc, t) : fmin(acc, t);
  }
  if (threadIdx.x % 32 == 0) sh[threadIdx.x / 32] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = sh[0];
    for (int w = 1; w < kT / 32; ++w) b = mode == 0 ? fmax(b, sh[w]) : fmin(b, sh[w]);
    partials[blockIdx.x] = b;
  }
  if (last_block(counter) && threadIdx.x == 0) {
    double b = __ldcg(&partials[0]);
    for (int k = 1; k < int(gridDim.x); ++k) b = mode == 0 ? fmax(b, __ldcg(&partials[k])) : fmin(b, __ldcg(&partials[k]));
    *out = b;
  }
}

// continuous-torus sampling (:190-216): per sample |shift + scale * Re symbol|;
// the best value, ties to the lexicographically smallest theta
struct Best {
  double v;
  int64_t key;  // theta order: axis 0 most significant
};
__device__ __forceinline__ bool better(const Best& a, const Best& b) {
  return a.v > b.v || (a.v == b.v && a.key < b.key);
}

__global__ void k_sample(int64_t total, int S, SpecArgs a, Best* partials, unsigned* counter, Best* out) {
  __shared__ Best sh[kT];
  Best best{-1.0, INT64_MAX};
  for (int64_t k = blockIdx.x * int64_t(kT) + threadIdx.x; k < total; k += int64_t(gridDim.x) * kT) {
    int64_t rem = k, key = 0;
    double theta[3] = {0, 0, 0};
    int64_t idx[3] = {0, 0, 0};
    for (int ax = 0; ax < a.dim; ++ax) {
      idx[ax] = rem % S;
      theta[ax] = two_pi_frac(idx[ax], S);
      rem /= S;
    }
    for (int ax = 0; ax < a.dim; ++ax) key = key * S + idx[ax];
    double re, im;
    symbol_dev(a, theta, re, im);
    const Best c{fabs(__dadd_rn(a.shift, __dmul_rn(a.scale, re))), key};
    if (better(c, best)) best = c;
  }
  sh[threadIdx.x] = best;
  __syncthreads();
  for (int s = kT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s && better(sh[threadIdx.x + s], sh[threadIdx.x])) sh[threadIdx.x] = sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
  if (last_block(counter) && threadIdx.x == 0) {
    auto ld = [&](int k) { return Best{__ldcg(&partials[k].v), (int64_t)__ldcg((const long long*)&partials[k].key)}; };
    Best b = ld(0);
    for (int k = 1; k < int(gridDim.x); ++k)
      if (better(ld(k), b)) b = ld(k);
    *out = b;
  }
}

int grid_for(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, int64_t(num_sms()) * 8))); }

// ---- host: symbol_nd and refine_symbol_max (the reference's libm evaluation) ----
std::complex<double> symbol_host(const sk_stencil* s, const std::vector<double>& theta) {
  std::complex<double> acc(0, 0);
  for (int e = 0; e < s->nent; ++e) {
    double phase = 0;
    for (size_t a = 0; a < theta.size(); ++a) phase += theta[a] * s->off[size_t(e) * 3 + a];
    acc += s->coeff[size_t(e)] * std::complex<double>(std::cos(phase), std::sin(phase));
  }
  return acc;
}

double refine_symbol_max(const sk_stencil* s, std::vector<double> theta, double best, double shift,
                         double scale_total) {  // linalg.cpp:110-147
  constexpr double inv_phi = 0.6180339887498949;
  auto value = [&](const std::vector<double>& th) { return std::abs(shift + scale_total * symbol_host(s, th).real()); };
  const double two_pi = 2 * 3.141592653589793;  // 2 * std::numbers::pi
  double window = two_pi / 64;
  for (int sweep = 0; sweep < 4; ++sweep) {
    for (size_t a = 0; a < theta.size(); ++a) {
      double lo = theta[a] - window, hi = theta[a] + window;
      auto f = [&](double t) {
        std::vector<double> th = theta;
        th[a] = t;
        return -value(th);
      };
      double x1 = hi - inv_phi * (hi - lo), x2 = lo + inv_phi * (hi - lo);
      double f1 = f(x1), f2 = f(x2);
      while (hi - lo > 1e-12) {
        if (f1 < f2) {
          hi = x2;
          x2 = x1;
          f2 = f1;
          x1 = hi - inv_phi * (hi - lo);
          f1 = f(x1);
        } else {
          lo = x1;
          x1 = x2;
          f1 = f2;
          x2 = lo + inv_phi * (hi - lo);
          f2 = f(x2);
        }
      }
      theta[a] = 0.5 * (lo + hi);
    }
    window /= 16;
  }
  return std::max(best, value(theta));
}

}  // namespace
}  // namespace sk

using namespace sk;

extern "C" {

int sk_power_iteration(const sk_csr* m, double tol, uint64_t seed, int64_t max_iter, double* out,
                       int64_t* iterations, void* stream_p) {
  if (!m || !out) return fail(SK_ERR_INVALID_ARGUMENT, "null matrix/output");
  if (m->rows != m->cols) return fail(SK_ERR_SHAPE_MISMATCH, "power iteration needs a square matrix");
  if (iterations) *iterations = 0;
  const int64_t n = m->rows;
  cudaStream_t st = as_stream(stream_p);
  if (int e = csr_build_sell(const_cast<sk_csr*>(m), st)) return e;
  // v: mt19937_64(seed) uniform(-1, 1) in order (linalg.cpp:77-79), on the host
  std::vector<double> v0(size_t(std::max<int64_t>(n, 1)));
  {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> unit(-1.0, 1.0);
    for (int64_t i = 0; i < n; ++i) v0[size_t(i)] = unit(rng);
  }
  const int grid = grid_for(n);
  char* ws = nullptr;
  const size_t vec = sizeof(double) * size_t(std::max<int64_t>(n, 1));
  const size_t bytes = 2 * vec + sizeof(double2) * size_t(grid) + sizeof(PiState) + 512;
  SK_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&ws), bytes));
  struct Free {
    char* p;
    ~Free() { cudaFree(p); }
  } guard{ws};
  double* v = reinterpret_cast<double*>(ws);
  double* w = v + std::max<int64_t>(n, 1);
  auto* partials = reinterpret_cast<double2*>(w + std::max<int64_t>(n, 1));
  auto* ps = reinterpret_cast<PiState*>((reinterpret_cast<uintptr_t>(partials + grid) + 127) & ~uintptr_t(127));
  double* scratch = reinterpret_cast<double*>(ps + 1);
  SK_CUDA_TRY(cudaMemcpyAsync(v, v0.data(), sizeof(double) * size_t(n), cudaMemcpyHostToDevice, st));
  SK_CUDA_TRY(cudaMemsetAsync(ps, 0, sizeof(PiState) + 64, st));
  // v /= nrm2(v)   (:80-81)
  k_sumsq_sqrt<<<grid, kT, 0, st>>>(n, v, reinterpret_cast<double*>(partials), &ps->counter[1], scratch);
  k_div<<<grid, kT, 0, st>>>(n, v, scratch);
  g_launches += 2;
  PiState h{};
  h.tol = tol;
  h.max_iter = max_iter;
  h.status = max_iter > 0 ? kPiRunning : kPiMaxIter;
  SK_CUDA_TRY(cudaMemcpyAsync(ps, &h, offsetof(PiState, counter), cudaMemcpyHostToDevice, st));

  // device loop: while (running) { w = M v + stopping rule ; v = w / |w| }
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  SK_CUDA_TRY(cudaGraphCreate(&graph, 0));
  struct G {
    cudaGraph_t g;
    cudaGraphExec_t* e;
    ~G() {
      if (*e) cudaGraphExecDestroy(*e);
      cudaGraphDestroy(g);
    }
  } gguard{graph, &exec};
  cudaGraphConditionalHandle hc;
  SK_CUDA_TRY(cudaGraphConditionalHandleCreate(&hc, graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  SK_CUDA_TRY(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
  cudaStream_t cap = st ? st : capture_stream();
  SK_CUDA_TRY(cudaStreamBeginCaptureToGraph(cap, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal));
  if (m->index_bits == 32)
    k_pi_spmv<int32_t><<<grid, kT, 0, cap>>>(n, m->sell_ptr, m->sell_len, static_cast<const int32_t*>(m->sell_col),
                                             m->sell_val, v, w, ps, partials);
  else
    k_pi_spmv<int64_t><<<grid, kT, 0, cap>>>(n, m->sell_ptr, m->sell_len, static_cast<const int64_t*>(m->sell_col),
                                             m->sell_val, v, w, ps, partials);
  k_pi_scale<true><<<grid, kT, 0, cap>>>(n, w, v, ps, hc);
  cudaGraph_t body = nullptr;
  SK_CUDA_TRY(cudaStreamEndCapture(cap, &body));
  SK_CUDA_TRY(cudaGraphInstantiate(&exec, graph, 0));
  SK_CUDA_TRY(cudaGraphLaunch(exec, st));
  SK_CUDA_TRY(cudaMemcpyAsync(&h, ps, sizeof(PiState), cudaMemcpyDeviceToHost, st));
  SK_CUDA_TRY(cudaStreamSynchronize(st));
  g_launches += 2 * (h.it + 1);
  if (iterations) *iterations = h.it;
  if (h.status == kPiDone || h.status == kPiZero) {
    *out = h.result;
    return SK_OK;
  }
  return fail(SK_ERR_NO_CONVERGENCE, "power iteration did not settle within iteration budget");
}

int sk_periodic_spectrum(const sk_stencil* s, const sk_grid_desc* gd, double affine_shift, double affine_scale,
                         double* eigen_host, double* spectral_radius, double* symbol_radius,
                         double* condition_estimate) {
  if (!s) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  if (s->dim != g.dim) return fail(SK_ERR_DIM_MISMATCH, "stencil/grid dimension mismatch");
  for (int a = 0; a < g.dim; ++a)
    if (g.bc[a] != SK_BC_PERIODIC) return fail(SK_ERR_NON_PERIODIC, "analytic spectrum needs all axes periodic");
  cudaStream_t st = host_stream();
  const int64_t modes = g.rows;
  SpecArgs a{};
  a.dim = g.dim;
  a.nent = s->nent;
  for (int i = 0; i < 3; ++i) a.n[i] = g.n[i];
  a.off = s->d_off;
  a.coeff = s->d_coeff;
  a.shift = affine_shift;
  a.scale = affine_scale * pow_int(g.h, s->h_power);  // scale_total (:158)
  const int grid = grid_for(modes);
  const int S = g.dim == 1 ? 4096 : (g.dim == 2 ? 512 : 96);
  int64_t total = 1;
  for (int i = 0; i < g.dim; ++i) total *= S;
  const int sgrid = grid_for(total);
  AsyncBuf buf(st);
  const size_t bytes = size_t(modes) * (sizeof(double2) + sizeof(double)) +
                       size_t(std::max(grid, sgrid)) * sizeof(Best) + 256;
  SK_CUDA_TRY(buf.alloc(bytes));
  auto* ev = reinterpret_cast<double2*>(buf.p);
  auto* mag = reinterpret_cast<double*>(ev + modes);
  auto* partials = reinterpret_cast<Best*>(mag + modes);
  auto* misc = reinterpret_cast<char*>(partials + std::max(grid, sgrid));
  auto* counters = reinterpret_cast<unsigned*>(misc);  // 3 counters
  auto* res = reinterpret_cast<double*>(misc + 64);     // rho, min_nonzero
  auto* best = reinterpret_cast<Best*>(misc + 128);
  SK_CUDA_TRY(cudaMemsetAsync(counters, 0, 64, st));
  k_eigen<<<grid, kT, 0, st>>>(modes, a, ev, mag);
  k_maxmin<<<grid, kT, 0, st>>>(modes, mag, 0.0, 0, reinterpret_cast<double*>(partials), &counters[0], &res[0]);
  double rho = 0;
  SK_CUDA_TRY(cudaMemcpyAsync(&rho, &res[0], sizeof(double), cudaMemcpyDeviceToHost, st));
  SK_CUDA_TRY(cudaStreamSynchronize(st));
  k_maxmin<<<grid, kT, 0, st>>>(modes, mag, 1e-12 * rho, 1, reinterpret_cast<double*>(partials), &counters[1],
                                &res[1]);
  k_sample<<<sgrid, kT, 0, st>>>(total, S, a, partials, &counters[2], best);
  g_launches += 4;
  double minnz = 0;
  Best hb{};
  SK_CUDA_TRY(cudaMemcpyAsync(&minnz, &res[1], sizeof(double), cudaMemcpyDeviceToHost, st));
  SK_CUDA_TRY(cudaMemcpyAsync(&hb, best, sizeof(Best), cudaMemcpyDeviceToHost, st));
  if (eigen_host)
    SK_CUDA_TRY(cudaMemcpyAsync(eigen_host, ev, sizeof(double2) * size_t(modes), cudaMemcpyDeviceToHost, st));
  SK_CUDA_TRY(cudaStreamSynchronize(st));
  if (!(minnz < INFINITY)) minnz = 0;
  if (spectral_radius) *spectral_radius = rho;
  if (condition_estimate) *condition_estimate = minnz > 0 ? rho / minnz : 0;
  if (symbol_radius) {
    // best theta of the device sampling, re-evaluated and polished on the host
    std::vector<double> theta(size_t(g.dim));
    const double two_pi = 2 * 3.141592653589793;  // 2 * std::numbers::pi
    int64_t key = hb.key;
    for (int ax = g.dim - 1; ax >= 0; --ax) {
      theta[size_t(ax)] = two_pi * static_cast<double>(key % S) / S;
      key /= S;
    }
    const double best_host = std::abs(affine_shift + a.scale * symbol_host(s, theta).real());
    *symbol_radius = refine_symbol_max(s, theta, best_host, affine_shift, a.scale);
  }
  return SK_OK;
}

}  // extern "C"
