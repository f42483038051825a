// IMEX Cahn-Hilliard stepping on the device: the reference's own CH path
// (SURVEY.md §8(f) 1), CahnHilliardStepper (cahn_hilliard.cpp:121-189):
//
//   chem = L f'(c)                                  (:146-152)
//   order 1: (I + dt M kappa B) c' = c + dt M chem  (:159-164)
//   order 2: (I + dt M kappa B / 2) c' = c - dt M kappa / 2 B c
//                                      + dt M (3/2 chem - 1/2 chem_prev)   (:166-178)
//   c' = cg_solve(implicit, rhs)                    (:180)
//
// with L = assemble(laplacian(d, 2)), B = assemble(compose(L, L)) built on the
// GPU (bit-identical CSR), the implicit matrix identity_plus_scaled(B, factor)
// (linalg.cpp:224-251) built on the GPU and cached per (factor, order) like
// ensure_implicit_matrix (:131-137), and the device CG (sk_cg.cu). Everything
// before the solve is bit-identical to the reference (sequential per-row sums
// with separately rounded multiply and add, the reference's f_chem_prime
// expression); the solve matches to its tolerance.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <utility>
#include <vector>

#include "sk_internal.hpp"

struct sk_ch_imex {
  sk::GridInfo g{};
  sk_grid_desc desc{};
  sk_ch_params p{};
  sk_solve_options opts{};
  sk_stencil* lap = nullptr;
  sk_stencil* bilap = nullptr;
  sk_csr* L = nullptr;
  sk_csr* B = nullptr;
  sk_csr* A = nullptr;  // identity_plus_scaled(B, a_factor)
  // matrix-free CG operator: the stencil of A (same weights as A's CSR
  // values, applied by the streaming stencil kernels: no matrix traffic)
  bool matrix_free = false;
  sk_stencil* a_st = nullptr;
  sk::CgPlan* plan = nullptr;
  double a_factor = 0.0;
  int a_order = 0;
  double* chem = nullptr;  // L f'(c) of this step
  double* prev = nullptr;  // ... of the previous order-2 step (prev_explicit_)
  double* rhs = nullptr;
  double* bc = nullptr;    // B c (order 2)
  bool have_prev = false;
  double prev_dt = 0.0;
  ~sk_ch_imex() {
    sk::cg_plan_destroy(plan);
    sk_stencil_destroy(a_st);
    sk_csr_destroy(A);
    sk_csr_destroy(B);
    sk_csr_destroy(L);
    sk_stencil_destroy(lap);
    sk_stencil_destroy(bilap);
    for (double* q : {chem, prev, rhs, bc})
      if (q) cudaFree(q);
  }
};

namespace sk {
namespace {

constexpr int kT = 256;

// f_chem_prime (cahn_hilliard.cpp:70-73), same operation order, no contraction
__device__ __forceinline__ double fprime_ref(double c, double rho, double ca, double cb) {
  const double a = __dadd_rn(c, -ca), b = __dadd_rn(c, -cb);
  const double t = __dmul_rn(__dmul_rn(__dmul_rn(2.0, rho), a), b);
  return __dmul_rn(t, __dadd_rn(__dadd_rn(__dmul_rn(2.0, c), -ca), -cb));
}

// chem_i = sum_k L_ik f'(c_col[k]) in column order (kernels.cpp:8-17 on w = f'(c))
template <class Idx>
__global__ void k_chem(int64_t rows, const int64_t* __restrict__ rp, const Idx* __restrict__ col,
                       const double* __restrict__ val, const double* __restrict__ c, double rho, double ca,
                       double cb, double* __restrict__ chem) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < rows; i += int64_t(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      acc = __dadd_rn(acc, __dmul_rn(val[k], fprime_ref(c[int64_t(col[k])], rho, ca, cb)));
    chem[i] = acc;
  }
}

// order 1 (:162-164): rhs = c + (dt M) chem
__global__ void k_rhs1(int64_t n, const double* __restrict__ c, const double* __restrict__ chem, double dtm,
                       double* __restrict__ rhs) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    rhs[i] = __dadd_rn(c[i], __dmul_rn(dtm, chem[i]));
}

// order 2 (:170-177): rhs = (c - half Bc) + (dt M) (1.5 chem - 0.5 prev)
__global__ void k_rhs2(int64_t n, const double* __restrict__ c, const double* __restrict__ bc,
                       const double* __restrict__ chem, const double* __restrict__ prev, double half, double dtm,
                       double* __restrict__ rhs) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double lin = __dadd_rn(c[i], -__dmul_rn(half, bc[i]));
    const double ex = __dmul_rn(dtm, __dadd_rn(__dmul_rn(1.5, chem[i]), -__dmul_rn(0.5, prev[i])));
    rhs[i] = __dadd_rn(lin, ex);
  }
}

// identity_plus_scaled (linalg.cpp:224-251): per row, v = alpha b (+1 on the
// diagonal), exact zeros dropped, a missing diagonal inserted as 1.0, columns
// kept sorted. Pass 1 counts, pass 2 writes.
template <class Idx>
__global__ void k_ips_count(int64_t rows, const int64_t* __restrict__ rp, const Idx* __restrict__ col,
                            const double* __restrict__ val, double alpha, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < rows; i += int64_t(gridDim.x) * blockDim.x) {
    int64_t n = 0;
    bool diag = false;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      double v = __dmul_rn(alpha, val[k]);
      if (int64_t(col[k]) == i) {
        v = __dadd_rn(v, 1.0);
        diag = true;
      }
      n += v != 0.0;
    }
    cnt[i] = n + (diag ? 0 : 1);
  }
}

template <class Idx>
__global__ void k_ips_fill(int64_t rows, const int64_t* __restrict__ rp, const Idx* __restrict__ col,
                           const double* __restrict__ val, double alpha, const int64_t* __restrict__ orp,
                           Idx* __restrict__ ocol, double* __restrict__ oval) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < rows; i += int64_t(gridDim.x) * blockDim.x) {
    int64_t o = orp[i];
    bool diag = false, placed = false;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t j = int64_t(col[k]);
      if (!placed && j > i) {  // missing diagonal goes before the first larger column
        if (!diag) {
          ocol[o] = Idx(i);
          oval[o++] = 1.0;
        }
        placed = true;
      }
      double v = __dmul_rn(alpha, val[k]);
      if (j == i) {
        v = __dadd_rn(v, 1.0);
        diag = placed = true;
      }
      if (v != 0.0) {
        ocol[o] = Idx(j);
        oval[o++] = v;
      }
    }
    if (!diag && !placed) {
      ocol[o] = Idx(i);
      oval[o] = 1.0;
    }
  }
}

int grid_for(int64_t n) { return int(std::min<int64_t>((n + kT - 1) / kT, int64_t(num_sms()) * 8)); }

template <class Idx>
int ips_build(const sk_csr* b, double alpha, sk_csr** out, cudaStream_t s, bool sell) {
  const int64_t rows = b->rows;
  const Idx* col = static_cast<const Idx*>(b->col);
  int64_t* cnt = nullptr;
  SK_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&cnt), sizeof(int64_t) * size_t(rows + 1), s));
  k_ips_count<Idx><<<grid_for(rows), kT, 0, s>>>(rows, b->row_ptr, col, b->val, alpha, cnt);
  SK_LAUNCH_CHECK("k_ips_count");
  auto* m = new sk_csr;
  m->rows = rows;
  m->cols = b->cols;
  m->index_bits = b->index_bits;
  int st = SK_OK;
  if (cudaMalloc(reinterpret_cast<void**>(&m->row_ptr), sizeof(int64_t) * size_t(rows + 1)) != cudaSuccess)
    st = fail(SK_ERR_OUT_OF_MEMORY, "implicit matrix row_ptr");
  size_t tmp_bytes = 0;
  void* tmp = nullptr;
  if (st == SK_OK) {
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, m->row_ptr, rows + 1, s);
    if (cudaMallocAsync(&tmp, tmp_bytes, s) != cudaSuccess) st = fail(SK_ERR_OUT_OF_MEMORY, "scan scratch");
  }
  if (st == SK_OK) {
    // cnt[rows] is the scan's last input: zero it so row_ptr[rows] = nnz
    cudaMemsetAsync(cnt + rows, 0, sizeof(int64_t), s);
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, m->row_ptr, rows + 1, s);
    cudaMemcpyAsync(&m->nnz, m->row_ptr + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) st = fail(SK_ERR_CUDA, "implicit matrix scan");
  }
  if (tmp) cudaFreeAsync(tmp, s);
  cudaFreeAsync(cnt, s);
  if (st == SK_OK &&
      (cudaMalloc(&m->col, sizeof(Idx) * size_t(std::max<int64_t>(m->nnz, 1))) != cudaSuccess ||
       cudaMalloc(reinterpret_cast<void**>(&m->val), sizeof(double) * size_t(std::max<int64_t>(m->nnz, 1))) !=
           cudaSuccess))
    st = fail(SK_ERR_OUT_OF_MEMORY, "implicit matrix entries");
  if (st == SK_OK) {
    k_ips_fill<Idx><<<grid_for(rows), kT, 0, s>>>(rows, b->row_ptr, col, b->val, alpha, m->row_ptr,
                                                  static_cast<Idx*>(m->col), m->val);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) st = cuda_fail(e, "k_ips_fill");
  }
  if (st == SK_OK && sell) st = csr_build_sell(m, s);
  if (st != SK_OK) {
    delete m;
    return st;
  }
  *out = m;
  return SK_OK;
}

// sell: also build the SELL copy the CSR CG operator reads
int identity_plus_scaled(const sk_csr* b, double alpha, sk_csr** out, cudaStream_t s, bool sell) {
  if (b->rows != b->cols) return fail(SK_ERR_SHAPE_MISMATCH, "needs a square matrix");
  return b->index_bits == 32 ? ips_build<int32_t>(b, alpha, out, s, sell) : ips_build<int64_t>(b, alpha, out, s, sell);
}

// laplacian(dim, 2) (generators.cpp:94-108) and compose(L, L) (stencil.cpp:75-87):
// integer coefficients, exactly representable; entries in lexicographic order.
void lap_entries(int dim, std::vector<int32_t>& off, std::vector<double>& co) {
  off.clear();
  co.clear();
  // offsets sorted lexicographically (axis 0 slowest) like Stencil's std::map
  std::vector<std::vector<int>> pts;
  for (int a = dim - 1; a >= 0; --a) {
    std::vector<int> p(size_t(dim), 0);
    p[size_t(a)] = -1;
    pts.push_back(p);
  }
  std::vector<int> zero(size_t(dim), 0);
  pts.push_back(zero);
  for (int a = 0; a < dim; ++a) {
    std::vector<int> p(size_t(dim), 0);
    p[size_t(a)] = 1;
    pts.push_back(p);
  }
  std::sort(pts.begin(), pts.end());
  for (const auto& p : pts) {
    bool centre = true;
    for (int v : p) centre &= v == 0;
    for (int v : p) off.push_back(v);
    co.push_back(centre ? -2.0 * dim : 1.0);
  }
}

void compose_entries(int dim, const std::vector<int32_t>& lo, const std::vector<double>& lc,
                     std::vector<int32_t>& off, std::vector<double>& co) {
  std::vector<std::pair<std::vector<int>, double>> acc;
  const size_t n = lc.size();
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < n; ++j) {
      std::vector<int> p(static_cast<size_t>(dim));
      for (int a = 0; a < dim; ++a) p[size_t(a)] = lo[i * size_t(dim) + size_t(a)] + lo[j * size_t(dim) + size_t(a)];
      bool found = false;
      for (auto& e : acc)
        if (e.first == p) {
          e.second += lc[i] * lc[j];  // integers: exact in any order
          found = true;
        }
      if (!found) acc.push_back({p, lc[i] * lc[j]});
    }
  std::sort(acc.begin(), acc.end());
  off.clear();
  co.clear();
  for (const auto& e : acc) {
    if (e.second == 0.0) continue;
    for (int v : e.first) off.push_back(v);
    co.push_back(e.second);
  }
}

}  // namespace
}  // namespace sk

using namespace sk;

extern "C" {

int sk_ch_imex_create(const sk_grid_desc* gd, const sk_ch_params* p, const sk_solve_options* o,
                      sk_ch_imex** out) {
  if (!out || !p) return fail(SK_ERR_INVALID_ARGUMENT, "null params/output");
  *out = nullptr;
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  for (int a = 0; a < g.dim; ++a)  // require_periodic (cahn_hilliard.cpp:12-16)
    if (g.bc[a] != SK_BC_PERIODIC) return fail(SK_ERR_NON_PERIODIC, "Cahn-Hilliard runs on periodic grids");
  auto* s = new sk_ch_imex;
  s->g = g;
  s->desc = *gd;
  s->p = *p;
  if (o) {
    s->opts = *o;
  } else {  // the stepper's default SolveOptions{.rel_tol = 1e-12} (cahn_hilliard.hpp:51-52)
    s->opts = sk_solve_options{};
    s->opts.rel_tol = 1e-12;
  }
  std::vector<int32_t> lo, bo;
  std::vector<double> lc, bcf;
  lap_entries(g.dim, lo, lc);
  compose_entries(g.dim, lo, lc, bo, bcf);
  int st = sk_stencil_create(g.dim, int(lc.size()), lo.data(), lc.data(), -2, &s->lap);
  if (st == SK_OK) st = sk_stencil_create(g.dim, int(bcf.size()), bo.data(), bcf.data(), -4, &s->bilap);
  cudaStream_t hs = host_stream();
  if (st == SK_OK) st = sk_csr_assemble(s->lap, gd, 64, &s->L, hs);
  if (st == SK_OK) st = sk_csr_assemble(s->bilap, gd, 64, &s->B, hs);
  const size_t bytes = sizeof(double) * size_t(std::max<int64_t>(g.rows, 1));
  for (double** q : {&s->chem, &s->prev, &s->rhs, &s->bc})
    if (st == SK_OK && cudaMalloc(reinterpret_cast<void**>(q), bytes) != cudaSuccess)
      st = fail(SK_ERR_OUT_OF_MEMORY, "IMEX work vectors");
  if (st == SK_OK) st = csr_build_sell(s->B, hs);
  // matrix-free implicit operator on the kernels' symmetric radius-2 classes
  // (grid at least the stencil width: no wrapped duplicates) unless
  // SK_OPT_IMEX_MATRIX_FREE = 0 (CSR SpMV, bit-identical products)
  if (st == SK_OK) {
    bool wide = true;
    for (int a = 0; a < g.dim; ++a) wide &= g.n[a] >= 5;
    s->matrix_free = wide && (s->bilap->kclass == 1 || s->bilap->kclass == 2) && option(SK_OPT_IMEX_MATRIX_FREE);
  }
  if (st == SK_OK && cudaStreamSynchronize(hs) != cudaSuccess) st = fail(SK_ERR_CUDA, "IMEX setup");
  if (st != SK_OK) {
    delete s;
    return st;
  }
  *out = s;
  return SK_OK;
}

int sk_ch_imex_destroy(sk_ch_imex* s) {
  delete s;
  return SK_OK;
}

int sk_ch_imex_reset_history(sk_ch_imex* s) {
  if (!s) return fail(SK_ERR_INVALID_ARGUMENT, "null stepper");
  s->have_prev = false;
  s->prev_dt = 0.0;
  return SK_OK;
}

int sk_ch_imex_step(sk_ch_imex* s, double* c, double dt, int order, int64_t nsteps, sk_solve_report* last,
                    int64_t* cg_iterations, void* stream_p) {
  if (!s) return fail(SK_ERR_INVALID_ARGUMENT, "null stepper");
  if (order != 1 && order != 2) return fail(SK_ERR_INVALID_ARGUMENT, "IMEX order must be 1 or 2");
  if (!(dt > 0)) return fail(SK_ERR_INVALID_ARGUMENT, "dt must be positive");
  if (nsteps < 0) return fail(SK_ERR_INVALID_ARGUMENT, "nsteps must be >= 0");
  if (!c && s->g.rows > 0) return fail(SK_ERR_INVALID_ARGUMENT, "null field");
  if (cg_iterations) *cg_iterations = 0;
  cudaStream_t st = as_stream(stream_p);
  const int64_t n = s->g.rows;
  const int grid = grid_for(n);
  const double M = s->p.mobility, kappa = s->p.kappa;
  for (int64_t k = 0; k < nsteps; ++k) {
    // explicit chemistry (:146-152)
    if (s->L->index_bits == 32)
      k_chem<int32_t><<<grid, kT, 0, st>>>(n, s->L->row_ptr, static_cast<const int32_t*>(s->L->col), s->L->val, c,
                                           s->p.rho_w, s->p.c_alpha, s->p.c_beta, s->chem);
    else
      k_chem<int64_t><<<grid, kT, 0, st>>>(n, s->L->row_ptr, static_cast<const int64_t*>(s->L->col), s->L->val, c,
                                           s->p.rho_w, s->p.c_alpha, s->p.c_beta, s->chem);
    SK_LAUNCH_CHECK("k_chem");
    // AB2 needs a same-dt history (:155-157)
    const int eff = (order == 2 && s->have_prev && s->prev_dt == dt) ? 2 : 1;
    // ensure_implicit_matrix (:131-137)
    const double factor = dt * M * kappa * (eff == 2 ? 0.5 : 1.0);
    if (!s->A || s->a_factor != factor || s->a_order != eff) {
      cg_plan_destroy(s->plan);
      s->plan = nullptr;
      sk_csr_destroy(s->A);
      s->A = nullptr;
      sk_stencil_destroy(s->a_st);
      s->a_st = nullptr;
      if (int e = identity_plus_scaled(s->B, factor, &s->A, st, !s->matrix_free)) return e;
      CgOperator op;
      op.n = n;
      if (s->matrix_free) {
        // A's weights exactly as identity_plus_scaled forms its values:
        // alpha * (coeff * pow_int(h, h_power)) (+ 1.0 on the centre), h_power 0
        const sk_stencil* b = s->bilap;
        const double scale = pow_int(s->g.h, b->h_power);
        std::vector<int32_t> off(size_t(b->nent) * size_t(s->g.dim));
        std::vector<double> co(size_t(b->nent));
        for (int e = 0; e < b->nent; ++e) {
          bool centre = true;
          for (int a = 0; a < s->g.dim; ++a) {
            off[size_t(e) * size_t(s->g.dim) + size_t(a)] = b->off[size_t(e) * 3 + size_t(a)];
            centre &= b->off[size_t(e) * 3 + size_t(a)] == 0;
          }
          double v = factor * (b->coeff[size_t(e)] * scale);
          if (centre) v += 1.0;
          co[size_t(e)] = v;
        }
        if (int e = sk_stencil_create(s->g.dim, b->nent, off.data(), co.data(), 0, &s->a_st)) return e;
        op.s = s->a_st;
        op.g = s->g;
      } else {
        op.m = s->A;
      }
      if (int e = cg_plan_create(op, s->opts.check_every, st, &s->plan)) return e;
      s->a_factor = factor;
      s->a_order = eff;
    }
    const double dtm = dt * M;
    if (eff == 1) {
      k_rhs1<<<grid, kT, 0, st>>>(n, c, s->chem, dtm, s->rhs);
      SK_LAUNCH_CHECK("k_rhs1");
    } else {
      if (int e = sk_csr_matvec(s->B, c, s->bc, st)) return e;
      const double half = 0.5 * dt * M * kappa;
      k_rhs2<<<grid, kT, 0, st>>>(n, c, s->bc, s->chem, s->prev, half, dtm, s->rhs);
      SK_LAUNCH_CHECK("k_rhs2");
    }
    sk_solve_report rep{};
    sk_solve_options o = s->opts;
    o.use_initial_guess = 0;  // cg_solve starts from x0 = 0 (linalg.cpp:22)
    if (int e = cg_plan_solve(s->plan, s->rhs, c, &o, &rep, st)) return e;
    if (last) *last = rep;
    if (cg_iterations) *cg_iterations += rep.iterations;
    if (order == 2) {  // (:183-188)
      std::swap(s->prev, s->chem);
      s->have_prev = true;
      s->prev_dt = dt;
    } else {
      s->have_prev = false;
    }
  }
  return SK_OK;
}

int sk_ch_imex_matrix(const sk_ch_imex* s, int which, const sk_csr** out) {
  if (!s || !out) return fail(SK_ERR_INVALID_ARGUMENT, "null stepper/output");
  *out = which == 0 ? s->L : which == 1 ? s->B : s->A;
  if (!*out) return fail(SK_ERR_INVALID_ARGUMENT, "implicit matrix not built yet");
  return SK_OK;
}

// ch_init (cahn_hilliard.cpp:20-63): the trigonometric initial condition,
// evaluated on the host with the same libm expressions (bit-identical).
int sk_ch_init_host(const sk_grid_desc* gd, double c0, double eps, double* out) {
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  for (int a = 0; a < g.dim; ++a)
    if (g.bc[a] != SK_BC_PERIODIC) return fail(SK_ERR_NON_PERIODIC, "Cahn-Hilliard runs on periodic grids");
  if (g.dim != 2 && g.dim != 3) return fail(SK_ERR_INVALID_ARGUMENT, "initial condition is defined for 2D and 3D");
  if (!out) return fail(SK_ERR_INVALID_ARGUMENT, "null output");
  const double h = g.h;
  auto coord = [h](int64_t i) { return 0.0 + double(int(i)) * h; };  // GridSpec::coordinate, origin 0
  const int64_t nx = g.n[0], ny = g.n[1];
  if (g.dim == 2) {
    for (int64_t j = 0; j < ny; ++j) {
      const double y = coord(j);
      for (int64_t i = 0; i < nx; ++i) {
        const double x = coord(i);
        const double c2 = std::cos(0.13 * x) * std::cos(0.087 * y);
        out[j * nx + i] = c0 + eps * (std::cos(0.105 * x) * std::cos(0.11 * y) + c2 * c2 +
                                      std::cos(0.025 * x - 0.15 * y) * std::cos(0.07 * x - 0.02 * y));
      }
    }
  } else {
    const int64_t nz = g.n[2];
    for (int64_t k = 0; k < nz; ++k) {
      const double z = coord(k);
      for (int64_t j = 0; j < ny; ++j) {
        const double y = coord(j);
        for (int64_t i = 0; i < nx; ++i) {
          const double x = coord(i);
          const double c2 = std::cos(0.13 * x) * std::cos(0.087 * y) * std::cos(0.1 * z);
          out[(k * ny + j) * nx + i] =
              c0 + eps * (std::cos(0.105 * x) * std::cos(0.11 * y) * std::cos(0.11 * z) + c2 * c2 +
                          std::cos(0.025 * x - 0.15 * y - 0.1 * z) * std::cos(0.07 * x - 0.02 * y + 0.01 * z));
        }
      }
    }
  }
  return SK_OK;
}

}  // extern "C"
