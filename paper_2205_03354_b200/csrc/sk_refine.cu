// Iterative refinement for the composed-stencil BVP (configs 2 / 5): the
// residual of the EXACT composed operator, and a refinement loop around the
// device CG.
//
// Why (measured): the 73-point composed weights
// (compose(laplacian(3,4), itself), stencil.cpp:75-87) are non-dyadic
// rationals; their doubles (Rational::to_double truncation, grid.cpp:77-81)
// sum to -2.6e-15 instead of 0. At h = 1/256 that is a zeroth-order term of
// -2.6e-15 h^-4 = -1.1e-5 in the assembled operator, which moves the
// manufactured solution by ~5e-9 — the size of the 4th-order discretisation
// error there, so the reference's own matrix shows order 3.38 on the
// 128 -> 256 pair. The true residual of ANY fp64 iterate also bottoms out
// near 1e-7 |b| (eps |A| |x|), so CG cannot see the difference.
//
// Refinement: x_0 = CG(A_fl, b); r_k = b - A_exact x_k evaluated in
// double-double (error-free products, compensated sums, weights
// coeff + coeff_lo); d_k = CG(A_fl, r_k) to a modest tolerance; x_{k+1} =
// x_k + d_k. A_fl^{-1} A_exact = I + O(1e-8) on the smooth modes, so each
// step contracts the error by the inner tolerance; the loop stops when the
// correction is below fp64 resolution of x.
#include <cuda_runtime.h>

#include <array>
#include <cmath>
#include <map>
#include <vector>

#include "sk_internal.hpp"

namespace sk {
namespace {

struct RefineArgs {
  const double* __restrict__ x;
  const double* __restrict__ b;
  double* __restrict__ r;
  const int* __restrict__ off;
  const double* __restrict__ hi;
  const double* __restrict__ lo;  // may be null (no correction)
  int nent, dim;
  int64_t n[3], un[3];
  int bc[3];
  double scale;  // pow_int(h, h_power)
  int64_t rows;
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

// r = b - A x in double-double: each term w x with w = (hi + lo) * scale is
// split exactly (fma), the running sum carries its rounding errors.
__global__ void residual_dd_kernel(const RefineArgs a) {
  const int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= a.rows) return;
  int64_t idx[3];
  int64_t rem = row;
  for (int d = 0; d < 3; ++d) {
    idx[d] = rem % a.un[d];
    rem /= a.un[d];
  }
  double s_hi = 0.0, s_lo = 0.0;
  for (int e = 0; e < a.nent; ++e) {
    // weight (hi + lo) * scale as a double-double
    const double h0 = __ldg(a.hi + e);
    double w_hi = h0 * a.scale;
    double w_lo = fma(h0, a.scale, -w_hi);
    if (a.lo) w_lo = fma(__ldg(a.lo + e), a.scale, w_lo);
    int64_t col = 0, stride = 1;
    bool dropped = false;
    double sign = 1.0;
    for (int d = 0; d < a.dim; ++d) {  // grid.cpp:104-122 (and the clamped even reflection)
      const int o = __ldg(a.off + 3 * e + d);
      int64_t comp;
      if (a.bc[d] == SK_BC_PERIODIC) {
        comp = wrap_idx(idx[d] + o, a.n[d]);
      } else {
        int64_t gi = idx[d] + 1 + o;
        if (gi < 0) {
          gi = -gi;
          if (a.bc[d] == SK_BC_SIMPLY_SUPPORTED) sign = -sign;
        } else if (gi > a.n[d] - 1) {
          gi = 2 * (a.n[d] - 1) - gi;
          if (a.bc[d] == SK_BC_SIMPLY_SUPPORTED) sign = -sign;
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
    if (dropped) continue;
    const double xv = sign * __ldg(a.x + col);
    const double p_hi = w_hi * xv;
    const double p_lo = fma(w_hi, xv, -p_hi) + w_lo * xv;
    double t, err;
    two_sum(s_hi, p_hi, t, err);
    s_hi = t;
    s_lo += err + p_lo;
  }
  // r = b - (s_hi + s_lo)
  double t, err;
  two_sum(__ldg(a.b + row), -s_hi, t, err);
  a.r[row] = t + (err - s_lo);
}

}  // namespace

int residual_refined(const sk_stencil* s, const GridInfo& g, const double* b, const double* x, double* r,
                     cudaStream_t stream) {
  if (g.rows == 0) return SK_OK;
  RefineArgs a{};
  a.x = x;
  a.b = b;
  a.r = r;
  a.off = s->d_off;
  a.hi = s->d_coeff;
  a.lo = s->d_coeff_lo;
  a.nent = s->nent;
  a.dim = g.dim;
  for (int d = 0; d < 3; ++d) {
    a.n[d] = g.n[d];
    a.un[d] = g.un[d];
    a.bc[d] = g.bc[d];
  }
  a.scale = pow_int(g.h, s->h_power);
  a.rows = g.rows;
  residual_dd_kernel<<<unsigned((g.rows + 255) / 256), 256, 0, stream>>>(a);
  SK_LAUNCH_CHECK("residual_dd_kernel");
  return SK_OK;
}

int cg_solve_stencil(const sk_stencil* s, const GridInfo& g, const double* b, double* x, const sk_solve_options* o,
                     sk_solve_report* rep, cudaStream_t stream);

}  // namespace sk

using namespace sk;

extern "C" {

int sk_stencil_create_exact(int dim, int nent, const int32_t* offsets, const double* coeff, const double* coeff_lo,
                            int h_power, sk_stencil** out) {
  if (int st = sk_stencil_create(dim, nent, offsets, coeff, h_power, out)) return st;
  if (!coeff_lo) return SK_OK;
  sk_stencil* s = *out;
  std::map<std::array<int, 3>, double> lo;
  for (int e = 0; e < nent; ++e) {
    std::array<int, 3> o{0, 0, 0};
    for (int a = 0; a < dim; ++a) o[a] = offsets[e * dim + a];
    lo[o] = coeff_lo[e];
  }
  s->coeff_lo.assign(size_t(s->nent), 0.0);  // canonical (sorted) entry order, like s->coeff
  for (int e = 0; e < s->nent; ++e) {
    const std::array<int, 3> o{s->off[3 * e], s->off[3 * e + 1], s->off[3 * e + 2]};
    auto it = lo.find(o);
    if (it != lo.end()) s->coeff_lo[size_t(e)] = it->second;
  }
  cudaError_t err = cudaMalloc(&s->d_coeff_lo, sizeof(double) * s->coeff_lo.size());
  if (err == cudaSuccess)
    err = cudaMemcpy(s->d_coeff_lo, s->coeff_lo.data(), sizeof(double) * s->coeff_lo.size(), cudaMemcpyHostToDevice);
  if (err != cudaSuccess) {
    sk_stencil_destroy(s);
    *out = nullptr;
    return cuda_fail(err, "sk_stencil_create_exact upload");
  }
  return SK_OK;
}

int sk_residual_refined(const sk_stencil* s, const sk_grid_desc* gd, const double* b, const double* x, double* r,
                        void* stream) {
  if (!s) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  if (s->dim != g.dim) return fail(SK_ERR_DIM_MISMATCH, "stencil/grid dimension mismatch");
  if (int st = check_width(s, g)) return st;
  if (g.rows > 0 && (!b || !x || !r)) return fail(SK_ERR_INVALID_ARGUMENT, "null vector");
  return residual_refined(s, g, b, x, r, as_stream(stream));
}

int sk_cg_solve_stencil_refined(const sk_stencil* s, const sk_grid_desc* gd, const double* b, double* x,
                                const sk_solve_options* o, double inner_rel_tol, int max_refinements,
                                sk_refine_report* rep, void* stream_p) {
  if (!s) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  if (s->dim != g.dim) return fail(SK_ERR_DIM_MISMATCH, "stencil/grid dimension mismatch");
  if (int st = check_width(s, g)) return st;
  if (g.rows > 0 && (!b || !x)) return fail(SK_ERR_INVALID_ARGUMENT, "null vector");
  if (max_refinements < 0 || !(inner_rel_tol > 0)) return fail(SK_ERR_INVALID_ARGUMENT, "bad refinement settings");
  cudaStream_t stream = as_stream(stream_p);
  sk_refine_report out{};
  const int64_t n = g.rows;
  if (n == 0) {
    if (rep) *rep = out;
    return SK_OK;
  }
  sk_solve_options base = o ? *o : sk_solve_options{1e-10, 0, 0, 0, 0, 0};
  // the first solve only provides the starting iterate (the refinement makes it
  // exact): stop on the recurrence, the fp64 true residual cannot reach the
  // tolerance at config sizes
  base.accept_recurrence = 1;
  sk_solve_report r0{};
  if (int st = cg_solve_stencil(s, g, b, x, &base, &r0, stream)) return st;
  out.iterations = r0.iterations;
  out.initial_true_rel_residual = r0.true_rel_residual;
  double* work = nullptr;
  SK_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&work), sizeof(double) * size_t(2 * n), stream));
  double* res = work;
  double* d = work + n;
  double bn = 0, xn = 0, dn = 0, rn = 0;
  int st = sk_nrm2(n, b, &bn, stream);
  sk_solve_options inner = base;
  inner.rel_tol = inner_rel_tol;
  inner.accept_recurrence = 1;
  inner.use_initial_guess = 0;
  inner.deflate_mean = 0;
  for (int k = 0; k < max_refinements && st == SK_OK; ++k) {
    st = residual_refined(s, g, b, x, res, stream);
    if (st == SK_OK) st = sk_nrm2(n, res, &rn, stream);
    if (st != SK_OK) break;
    out.refined_rel_residual = bn > 0 ? rn / bn : rn;
    if (rn == 0.0) break;
    sk_solve_report ri{};
    st = cg_solve_stencil(s, g, res, d, &inner, &ri, stream);
    if (st != SK_OK) break;
    out.iterations += ri.iterations;
    st = sk_axpy(n, 1.0, d, x, stream);
    if (st == SK_OK) st = sk_nrm2(n, d, &dn, stream);
    if (st == SK_OK) st = sk_nrm2(n, x, &xn, stream);
    if (st != SK_OK) break;
    out.refinements = k + 1;
    out.last_correction_rel = xn > 0 ? dn / xn : dn;
    if (out.last_correction_rel <= 1e-15) break;  // below fp64 resolution of x
  }
  if (st == SK_OK) {  // the final refined residual
    st = residual_refined(s, g, b, x, res, stream);
    if (st == SK_OK) st = sk_nrm2(n, res, &rn, stream);
    out.refined_rel_residual = bn > 0 ? rn / bn : rn;
  }
  cudaFreeAsync(work, stream);
  if (rep) *rep = out;
  return st;
}

}  // extern "C"
