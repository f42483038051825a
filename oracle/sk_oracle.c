/* ORACLE TEST INFRASTRUCTURE — never linked into or called by the product.
 *
 * Plain-C restatement of the reference's hot-path algorithms (reference:
 * /root/reference/proj). Built with -ffp-contract=off so every multiply-add
 * rounds twice, as the reference's CMake Release build does (no -march, so
 * no FMA); the CSR assembly and csr_matvec below are therefore bit-identical
 * to the reference (checked by tests/test_oracle.py against
 * oracle/_ref/libstencilkit_ref.so and the committed golden fixtures).
 */
#include "sk_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

/* ---- grid (grid.cpp:10-40) ------------------------------------------- */

static double pow_int(double base, int exp) { /* grid.cpp:10-15 */
  if (exp < 0) return 1.0 / pow_int(base, -exp);
  double r = 1.0;
  for (int k = 0; k < exp; ++k) r *= base;
  return r;
}

static int64_t unknowns(int bc, int64_t n) { return bc == 0 ? n : n - 2; } /* grid.cpp:27-29 */

int sko_threads(void) { return omp_get_max_threads(); }

/* ---- assembly (grid.cpp:62-158) --------------------------------------- */

typedef struct {
  int64_t col;
  double val;
} pair_t;

static int pair_cmp(const void* pa, const void* pb) { /* std::pair<int64,double> operator< */
  const pair_t* a = (const pair_t*)pa;
  const pair_t* b = (const pair_t*)pb;
  if (a->col != b->col) return a->col < b->col ? -1 : 1;
  if (a->val < b->val) return -1;
  if (a->val > b->val) return 1;
  return 0;
}

/* One row of grid.cpp:89-138: wrap / reflect each entry, sort (col, val),
 * merge equal columns summing in sorted order, drop exact zeros. `buf` holds
 * nent pairs. Returns the row's entry count; results in buf[0..count). */
static int assemble_one(int dim, int nent, const int* off, const double* wval, const int64_t* n, const int64_t* un,
                        const int* bc, int64_t row, pair_t* buf) {
  int64_t idx[3] = {0, 0, 0};
  int64_t rem = row;
  for (int a = 0; a < dim; ++a) { /* x fastest, :93-96 */
    idx[a] = rem % un[a];
    rem /= un[a];
  }
  int cnt = 0;
  for (int e = 0; e < nent; ++e) {
    double val = wval[e];
    int64_t col = 0, stride = 1;
    int dropped = 0;
    for (int a = 0; a < dim && !dropped; ++a) {
      const int64_t na = n[a];
      int64_t comp;
      if (bc[a] == 0) {
        comp = ((idx[a] + off[e * dim + a]) % na + na) % na; /* :106-107 */
      } else {
        int64_t gi = idx[a] + 1 + off[e * dim + a]; /* :109-116, clamped keeps the sign */
        if (gi < 0) {
          gi = -gi;
          if (bc[a] == 1) val = -val;
        } else if (gi > na - 1) {
          gi = 2 * (na - 1) - gi;
          if (bc[a] == 1) val = -val;
        }
        if (gi == 0 || gi == na - 1) { /* :117-120 */
          dropped = 1;
          break;
        }
        comp = gi - 1;
      }
      col += stride * comp;
      stride *= un[a];
    }
    if (!dropped) {
      buf[cnt].col = col;
      buf[cnt].val = val;
      ++cnt;
    }
  }
  qsort(buf, (size_t)cnt, sizeof(pair_t), pair_cmp); /* :128 */
  int w = 0;
  for (int r = 0; r < cnt;) { /* :130-137 */
    const int64_t c = buf[r].col;
    double v = 0;
    while (r < cnt && buf[r].col == c) v += buf[r++].val;
    if (v != 0.0) {
      buf[w].col = c;
      buf[w].val = v;
      ++w;
    }
  }
  return w;
}

/* Width checks (grid.cpp:66-75). Returns 0 or Errc+1 (StencilWiderThanGrid = 11). */
static int check_width(int dim, int nent, const int* off, const int64_t* n, const int* bc) {
  for (int a = 0; a < dim; ++a) {
    int lo = off[a], hi = off[a];
    for (int e = 1; e < nent; ++e) {
      if (off[e * dim + a] < lo) lo = off[e * dim + a];
      if (off[e * dim + a] > hi) hi = off[e * dim + a];
    }
    if (bc[a] == 0) {
      if (hi - lo > n[a] - 1) return 11;
    } else {
      const int m = abs(lo) > abs(hi) ? abs(lo) : abs(hi);
      if (m > n[a] - 2) return 11;
    }
  }
  return 0;
}

static int setup(int dim, int nent, const int* off, const double* coeff, int h_power, const int64_t* n, double h,
                 const int* bc, int64_t* un, double* wval, int64_t* rows) {
  if (dim < 1 || dim > 3) return 18;
  for (int a = 0; a < dim; ++a)
    if (n[a] < 3) return 18;
  if (!(h > 0)) return 18;
  int st = check_width(dim, nent, off, n, bc);
  if (st) return st;
  const double scale = pow_int(h, h_power); /* :77 */
  for (int e = 0; e < nent; ++e) wval[e] = coeff[e] * scale; /* :80 */
  *rows = 1;
  for (int a = 0; a < dim; ++a) {
    un[a] = unknowns(bc[a], n[a]);
    *rows *= un[a];
  }
  return 0;
}

int sko_assemble(int dim, int nent, const int* off, const double* coeff, int h_power, const int64_t* n, double h,
                 const int* bc, sko_csr* out) {
  int64_t un[3] = {1, 1, 1}, rows = 0;
  double* wval = (double*)malloc(sizeof(double) * (size_t)nent);
  int st = setup(dim, nent, off, coeff, h_power, n, h, bc, un, wval, &rows);
  if (st) {
    free(wval);
    return st;
  }
  out->rows = out->cols = rows;
  out->row_ptr = (int64_t*)calloc((size_t)rows + 1, sizeof(int64_t));
  int64_t* counts = out->row_ptr + 1;
#pragma omp parallel
  {
    pair_t* buf = (pair_t*)malloc(sizeof(pair_t) * (size_t)nent);
#pragma omp for schedule(static)
    for (int64_t r = 0; r < rows; ++r) counts[r] = assemble_one(dim, nent, off, wval, n, un, bc, r, buf);
    free(buf);
  }
  for (int64_t r = 0; r < rows; ++r) out->row_ptr[r + 1] += out->row_ptr[r]; /* :141-144 */
  out->nnz = out->row_ptr[rows];
  out->col_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(out->nnz > 0 ? out->nnz : 1));
  out->values = (double*)malloc(sizeof(double) * (size_t)(out->nnz > 0 ? out->nnz : 1));
#pragma omp parallel
  {
    pair_t* buf = (pair_t*)malloc(sizeof(pair_t) * (size_t)nent);
#pragma omp for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
      const int cnt = assemble_one(dim, nent, off, wval, n, un, bc, r, buf);
      int64_t k = out->row_ptr[r];
      for (int i = 0; i < cnt; ++i, ++k) {
        out->col_idx[k] = buf[i].col;
        out->values[k] = buf[i].val;
      }
    }
    free(buf);
  }
  free(wval);
  return 0;
}

int sko_assemble_row(int dim, int nent, const int* off, const double* coeff, int h_power, const int64_t* n, double h,
                     const int* bc, int64_t row, int64_t* cols, double* vals) {
  int64_t un[3] = {1, 1, 1}, rows = 0;
  double* wval = (double*)malloc(sizeof(double) * (size_t)nent);
  int st = setup(dim, nent, off, coeff, h_power, n, h, bc, un, wval, &rows);
  if (st) {
    free(wval);
    return -st;
  }
  pair_t* buf = (pair_t*)malloc(sizeof(pair_t) * (size_t)nent);
  const int cnt = assemble_one(dim, nent, off, wval, n, un, bc, row, buf);
  for (int i = 0; i < cnt; ++i) {
    cols[i] = buf[i].col;
    vals[i] = buf[i].val;
  }
  free(buf);
  free(wval);
  return cnt;
}

void sko_csr_free(sko_csr* m) {
  free(m->row_ptr);
  free(m->col_idx);
  free(m->values);
  m->row_ptr = m->col_idx = NULL;
  m->values = NULL;
}

/* ---- kernels (kernels.cpp:8-60): per-row sequential, no contraction ---- */

void sko_csr_matvec(const sko_csr* m, const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m->rows; ++i) {
    double acc = 0;
    for (int64_t k = m->row_ptr[i]; k < m->row_ptr[i + 1]; ++k) acc += m->values[k] * x[m->col_idx[k]];
    y[i] = acc;
  }
}

double sko_dot(int64_t n, const double* a, const double* b) { /* serial twin, kernels.cpp:64-68 */
  double acc = 0;
  for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

double sko_nrm2(int64_t n, const double* a) { return sqrt(sko_dot(n, a, a)); }

double sko_sum(int64_t n, const double* a) {
  double acc = 0;
  for (int64_t i = 0; i < n; ++i) acc += a[i];
  return acc;
}

void sko_minmax(int64_t n, const double* a, double* lo, double* hi) {
  *lo = *hi = a[0];
  for (int64_t i = 0; i < n; ++i) {
    if (a[i] < *lo) *lo = a[i];
    if (a[i] > *hi) *hi = a[i];
  }
}

void sko_axpy(int64_t n, double a, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] += a * x[i];
}

void sko_xpby(int64_t n, const double* x, double b, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = x[i] + b * y[i];
}

/* ---- cg_solve (linalg.cpp:15-72) --------------------------------------
 * Returns 0, or 13 (NoConvergence, Errc+1) on a non-PD Krylov space or a
 * stalled true residual; x holds the last iterate either way. */
int sko_cg_solve(const sko_csr* m, const double* b, double* x, double rel_tol, int64_t max_iter_in, int deflate_mean,
                 int64_t* iterations, double* true_rel_residual) {
  const int64_t n = m->rows;
  const int64_t max_iter = max_iter_in > 0 ? max_iter_in : 10 * n; /* :20 */
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  double* p = (double*)malloc(sizeof(double) * (size_t)n);
  double* q = (double*)malloc(sizeof(double) * (size_t)n);
  memset(x, 0, sizeof(double) * (size_t)n);
  memcpy(r, b, sizeof(double) * (size_t)n);
  memcpy(p, b, sizeof(double) * (size_t)n);
  const double bnorm = sko_nrm2(n, r);
  int st = 0;
  int64_t it = 0;
  if (bnorm == 0.0) {
    if (true_rel_residual) *true_rel_residual = 0;
    goto done;
  }
  const double target = rel_tol * bnorm;
  double rho = sko_dot(n, r, r);
  for (; it < max_iter; ++it) {
    if (sqrt(rho) <= target) { /* :31-47 */
      sko_csr_matvec(m, x, q);
      double tr = 0;
      for (int64_t i = 0; i < n; ++i) {
        const double d = b[i] - q[i];
        tr += d * d;
      }
      if (sqrt(tr) <= target) break;
      for (int64_t i = 0; i < n; ++i) r[i] = b[i] - q[i];
      memcpy(p, r, sizeof(double) * (size_t)n);
      rho = sko_dot(n, r, r);
    }
    sko_csr_matvec(m, p, q); /* :48 */
    const double pq = sko_dot(n, p, q);
    if (pq <= 0) { /* :50-51 */
      st = 13;
      goto done;
    }
    const double alpha = rho / pq;
    sko_axpy(n, alpha, p, x);
    sko_axpy(n, -alpha, q, r);
    const double rho_next = sko_dot(n, r, r);
    sko_xpby(n, r, rho_next / rho, p);
    rho = rho_next;
  }
  {
    sko_csr_matvec(m, x, q); /* :59-66 */
    double res = 0;
    for (int64_t i = 0; i < n; ++i) res += (b[i] - q[i]) * (b[i] - q[i]);
    res = sqrt(res);
    if (true_rel_residual) *true_rel_residual = res / bnorm;
    if (res > target) {
      st = 13;
      goto done;
    }
  }
  if (deflate_mean) { /* :67-70 */
    const double mean = sko_sum(n, x) / (double)n;
    for (int64_t i = 0; i < n; ++i) x[i] -= mean;
  }
done:
  if (iterations) *iterations = it;
  free(r);
  free(p);
  free(q);
  return st;
}

/* ---- matrix-free apply, entry order (the assemble+apply of grid.cpp:166-172
 * without the per-row sort: a second, independent restatement) ----------- */
void sko_apply_direct(int dim, int nent, const int* off, const double* coeff, int h_power, const int64_t* n, double h,
                      const int* bc, const double* u, double* v) {
  int64_t un[3] = {1, 1, 1}, rows = 0;
  double* wval = (double*)malloc(sizeof(double) * (size_t)nent);
  if (setup(dim, nent, off, coeff, h_power, n, h, bc, un, wval, &rows)) {
    free(wval);
    return;
  }
#pragma omp parallel
  {
    pair_t* buf = (pair_t*)malloc(sizeof(pair_t) * (size_t)nent);
#pragma omp for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
      const int cnt = assemble_one(dim, nent, off, wval, n, un, bc, r, buf);
      double acc = 0;
      for (int i = 0; i < cnt; ++i) acc += buf[i].val * u[buf[i].col];
      v[r] = acc;
    }
    free(buf);
  }
  free(wval);
}

/* ---- Cahn-Hilliard ------------------------------------------------------ */

/* laplacian(dim, 2) (generators.cpp:94-108): centre -2*dim, axis +-1: 1;
 * compose(lap, lap) (stencil.cpp:75-87): offsets add, coefficients multiply.
 * Integer coefficients, exact in double. Entries in lexicographic order. */
static int lap_entries(int dim, int* off, double* coeff) {
  int k = 0;
  for (int a = 0; a < dim; ++a) /* gather all offsets, then sort below */
    for (int s = -1; s <= 1; s += 2) {
      for (int b = 0; b < dim; ++b) off[k * dim + b] = (b == a) ? s : 0;
      coeff[k++] = 1.0;
    }
  for (int b = 0; b < dim; ++b) off[k * dim + b] = 0;
  coeff[k++] = -2.0 * dim;
  return k;
}

static int compose_entries(int dim, int na, const int* oa, const double* ca, int* out_off, double* out_c) {
  int k = 0;
  for (int i = 0; i < na; ++i)
    for (int j = 0; j < na; ++j) {
      int o[3] = {0, 0, 0};
      for (int b = 0; b < dim; ++b) o[b] = oa[i * dim + b] + oa[j * dim + b];
      int f = -1;
      for (int t = 0; t < k && f < 0; ++t) {
        int same = 1;
        for (int b = 0; b < dim; ++b) same &= out_off[t * dim + b] == o[b];
        if (same) f = t;
      }
      if (f < 0) {
        f = k++;
        for (int b = 0; b < dim; ++b) out_off[f * dim + b] = o[b];
        out_c[f] = 0;
      }
      out_c[f] += ca[i] * ca[j];
    }
  int w = 0; /* canonical form drops zeros (stencil.cpp:15-25) */
  for (int t = 0; t < k; ++t)
    if (out_c[t] != 0) {
      for (int b = 0; b < dim; ++b) out_off[w * dim + b] = out_off[t * dim + b];
      out_c[w++] = out_c[t];
    }
  return w;
}

static double f_chem_prime(double c, double rho_w, double ca, double cb) { /* cahn_hilliard.cpp:70-73 */
  const double a = c - ca, b = c - cb;
  return 2.0 * rho_w * a * b * (2.0 * c - ca - cb);
}

/* Explicit forward Euler, the restatement of SURVEY.md Appendix A:
 * w = f'(c); a = L w; b = B c; c += dt * M * (a - kappa * b). */
int sko_ch_explicit(int dim, int64_t n, double h, double mobility, double kappa, double rho_w, double c_alpha,
                    double c_beta, double dt, int64_t nsteps, double* c) {
  const int64_t nn[3] = {n, n, n};
  return sko_ch_explicit_dims(dim, nn, h, mobility, kappa, rho_w, c_alpha, c_beta, dt, nsteps, c);
}

/* the same on an n[0] x n[1] (x n[2]) periodic grid */
int sko_ch_explicit_dims(int dim, const int64_t* ndims, double h, double mobility, double kappa, double rho_w,
                         double c_alpha, double c_beta, double dt, int64_t nsteps, double* c) {
  int lo[3 * 7] = {0}, bo[3 * 49] = {0};
  double lc[7], bcf[49];
  const int nl = lap_entries(dim, lo, lc);
  const int nb = compose_entries(dim, nl, lo, lc, bo, bcf);
  const int64_t nn[3] = {ndims[0], dim > 1 ? ndims[1] : 1, dim > 2 ? ndims[2] : 1};
  const int bcs[3] = {0, 0, 0};
  sko_csr L, B;
  int st = sko_assemble(dim, nl, lo, lc, -2, nn, h, bcs, &L);
  if (st) return st;
  st = sko_assemble(dim, nb, bo, bcf, -4, nn, h, bcs, &B);
  if (st) {
    sko_csr_free(&L);
    return st;
  }
  const int64_t rows = L.rows;
  double* w = (double*)malloc(sizeof(double) * (size_t)rows);
  double* la = (double*)malloc(sizeof(double) * (size_t)rows);
  double* lb = (double*)malloc(sizeof(double) * (size_t)rows);
  for (int64_t k = 0; k < nsteps; ++k) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) w[i] = f_chem_prime(c[i], rho_w, c_alpha, c_beta);
    sko_csr_matvec(&L, w, la);
    sko_csr_matvec(&B, c, lb);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; ++i) c[i] += dt * mobility * (la[i] - kappa * lb[i]);
  }
  free(w);
  free(la);
  free(lb);
  sko_csr_free(&L);
  sko_csr_free(&B);
  return 0;
}

/* identity_plus_scaled (linalg.cpp:224-251): v = alpha b (+1 on the diagonal),
 * exact zeros dropped, a missing diagonal inserted as 1.0, columns sorted. */
int sko_identity_plus_scaled(const sko_csr* m, double alpha, sko_csr* out) {
  const int64_t rows = m->rows;
  out->rows = rows;
  out->cols = m->cols;
  out->row_ptr = (int64_t*)calloc((size_t)rows + 1, sizeof(int64_t));
  out->col_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m->nnz + rows + 1));
  out->values = (double*)malloc(sizeof(double) * (size_t)(m->nnz + rows + 1));
  if (!out->row_ptr || !out->col_idx || !out->values) return 1;
  int64_t o = 0;
  for (int64_t i = 0; i < rows; ++i) {
    int diag = 0, placed = 0;
    for (int64_t k = m->row_ptr[i]; k < m->row_ptr[i + 1]; ++k) {
      const int64_t j = m->col_idx[k];
      if (!placed && j > i) { /* the sorted position of an inserted diagonal */
        if (!diag) {
          out->col_idx[o] = i;
          out->values[o++] = 1.0;
        }
        placed = 1;
      }
      double v = alpha * m->values[k];
      if (j == i) {
        v += 1.0;
        diag = placed = 1;
      }
      if (v != 0.0) {
        out->col_idx[o] = j;
        out->values[o++] = v;
      }
    }
    if (!diag && !placed) {
      out->col_idx[o] = i;
      out->values[o++] = 1.0;
    }
    out->row_ptr[i + 1] = o;
  }
  out->nnz = o;
  return 0;
}

/* IMEX stepping (cahn_hilliard.cpp:121-189) on ONE fresh stepper over a
 * sequence of legs (dt, order, steps): L, B assembled (:126-128); per step
 * chem = L f'(c) (:146-152); AB2 only with a same-dt history (:155-157),
 * the history kept by order-2 steps and dropped by order-1 steps (:183-188);
 * implicit matrix per (factor, order) (:131-137); rhs (:159-178);
 * c = cg_solve(implicit, rhs, rel_tol) from x0 = 0 (:180). */
int sko_ch_imex_seq(int dim, int64_t n, double h, double mobility, double kappa, double rho_w, double c_alpha,
                    double c_beta, double rel_tol, int nlegs, const double* dts, const int* orders,
                    const int64_t* steps, double* c) {
  int lo[3 * 7] = {0}, bo[3 * 49] = {0};
  double lc[7], bcf[49];
  const int nl = lap_entries(dim, lo, lc);
  const int nb = compose_entries(dim, nl, lo, lc, bo, bcf);
  const int64_t nn[3] = {n, n, n};
  const int bcs[3] = {0, 0, 0};
  sko_csr L, B, A;
  int st = sko_assemble(dim, nl, lo, lc, -2, nn, h, bcs, &L);
  if (st) return st;
  st = sko_assemble(dim, nb, bo, bcf, -4, nn, h, bcs, &B);
  if (st) {
    sko_csr_free(&L);
    return st;
  }
  const int64_t rows = L.rows;
  double* w = (double*)malloc(sizeof(double) * (size_t)rows);
  double* chem = (double*)malloc(sizeof(double) * (size_t)rows);
  double* prev = (double*)malloc(sizeof(double) * (size_t)rows);
  double* rhs = (double*)malloc(sizeof(double) * (size_t)rows);
  double* bc = (double*)malloc(sizeof(double) * (size_t)rows);
  int have_prev = 0, a_order = 0;
  double a_factor = 0.0, prev_dt = 0.0;
  A.row_ptr = NULL;
  for (int leg = 0; leg < nlegs && st == 0; ++leg) {
    const double dt = dts[leg];
    const int order = orders[leg];
    for (int64_t k = 0; k < steps[leg] && st == 0; ++k) {
      for (int64_t i = 0; i < rows; ++i) w[i] = f_chem_prime(c[i], rho_w, c_alpha, c_beta);
      sko_csr_matvec(&L, w, chem);
      const int eff = (order == 2 && have_prev && prev_dt == dt) ? 2 : 1;
      const double factor = dt * mobility * kappa * (eff == 2 ? 0.5 : 1.0);
      if (!A.row_ptr || factor != a_factor || eff != a_order) {
        if (A.row_ptr) sko_csr_free(&A);
        sko_identity_plus_scaled(&B, factor, &A);
        a_factor = factor;
        a_order = eff;
      }
      if (eff == 1) {
        for (int64_t i = 0; i < rows; ++i) rhs[i] = c[i] + dt * mobility * chem[i];
      } else {
        sko_csr_matvec(&B, c, bc);
        const double half = 0.5 * dt * mobility * kappa;
        for (int64_t i = 0; i < rows; ++i)
          rhs[i] = c[i] - half * bc[i] + dt * mobility * (1.5 * chem[i] - 0.5 * prev[i]);
      }
      int64_t it = 0;
      double res = 0;
      st = sko_cg_solve(&A, rhs, c, rel_tol, 0, 0, &it, &res);
      if (order == 2) {
        double* t = prev;
        prev = chem;
        chem = t;
        have_prev = 1;
        prev_dt = dt;
      } else {
        have_prev = 0;
      }
    }
  }
  if (A.row_ptr) sko_csr_free(&A);
  free(w);
  free(chem);
  free(prev);
  free(rhs);
  free(bc);
  sko_csr_free(&L);
  sko_csr_free(&B);
  return st;
}

int sko_ch_imex(int dim, int64_t n, double h, double mobility, double kappa, double rho_w, double c_alpha,
                double c_beta, double rel_tol, double dt, int order, int64_t nsteps, double* c) {
  return sko_ch_imex_seq(dim, n, h, mobility, kappa, rho_w, c_alpha, c_beta, rel_tol, 1, &dt, &order, &nsteps, c);
}

/* csr_matmul (linalg.cpp:253-283): out = b * a, dense accumulator per row,
 * columns recorded on first touch (acc == 0), sorted, exact zeros dropped */
static int cmp_i64(const void* x, const void* y) {
  const int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return (a > b) - (a < b);
}
int sko_csr_matmul(const sko_csr* b, const sko_csr* a, sko_csr* out) {
  out->rows = b->rows;
  out->cols = a->cols;
  out->row_ptr = (int64_t*)calloc((size_t)b->rows + 1, sizeof(int64_t));
  double* acc = (double*)calloc((size_t)(a->cols > 0 ? a->cols : 1), sizeof(double));
  int64_t cap = 1024, nnz = 0;
  out->col_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
  out->values = (double*)malloc(sizeof(double) * (size_t)cap);
  int64_t tcap = 1024;
  int64_t* touched = (int64_t*)malloc(sizeof(int64_t) * (size_t)tcap);
  for (int64_t i = 0; i < b->rows; ++i) {
    int64_t nt = 0;
    for (int64_t kb = b->row_ptr[i]; kb < b->row_ptr[i + 1]; ++kb) {
      const int64_t j = b->col_idx[kb];
      const double vb = b->values[kb];
      for (int64_t ka = a->row_ptr[j]; ka < a->row_ptr[j + 1]; ++ka) {
        const int64_t c = a->col_idx[ka];
        if (acc[c] == 0.0) {
          if (nt == tcap) touched = (int64_t*)realloc(touched, sizeof(int64_t) * (size_t)(tcap *= 2));
          touched[nt++] = c;
        }
        acc[c] += vb * a->values[ka];
      }
    }
    qsort(touched, (size_t)nt, sizeof(int64_t), cmp_i64);
    for (int64_t t = 0; t < nt; ++t) {
      const int64_t c = touched[t];
      if (acc[c] != 0.0) {
        if (nnz == cap) {
          cap *= 2;
          out->col_idx = (int64_t*)realloc(out->col_idx, sizeof(int64_t) * (size_t)cap);
          out->values = (double*)realloc(out->values, sizeof(double) * (size_t)cap);
        }
        out->col_idx[nnz] = c;
        out->values[nnz++] = acc[c];
      }
      acc[c] = 0.0;
    }
    out->row_ptr[i + 1] = nnz;
  }
  out->nnz = nnz;
  free(acc);
  free(touched);
  return 0;
}

/* power_iteration (linalg.cpp:74-106), serial reductions */
int sko_power_iteration(const sko_csr* m, double tol, uint64_t seed, int64_t max_iter, double* out,
                        int64_t* iterations) {
  const int64_t n = m->rows;
  double* v = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double* w = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  sko_uniform(seed, n, -1.0, 1.0, v);
  const double nv = sko_nrm2(n, v);
  for (int64_t i = 0; i < n; ++i) v[i] /= nv;
  double lambda = 0, prev = 0, prev_delta = 0;
  int st = 1;
  *out = 0;
  for (int64_t it = 0; it < max_iter; ++it) {
    if (iterations) *iterations = it + 1;
    sko_csr_matvec(m, v, w);
    lambda = sko_dot(n, v, w);
    const double wn = sko_nrm2(n, w);
    if (wn == 0.0) {
      st = 0;
      break;
    }
    for (int64_t i = 0; i < n; ++i) v[i] = w[i] / wn;
    if (it > 0) {
      const double delta = fabs(lambda - prev);
      if (it > 1 && prev_delta > 0 && delta < prev_delta) {
        const double r = delta / prev_delta;
        const double tail = delta * r / (1.0 - r);
        if (tail <= 0.25 * tol * fabs(lambda)) {
          *out = fabs(lambda);
          st = 0;
          break;
        }
      }
      if (delta == 0.0) {
        *out = fabs(lambda);
        st = 0;
        break;
      }
    }
    prev_delta = it > 0 ? fabs(lambda - prev) : 0;
    prev = lambda;
  }
  free(v);
  free(w);
  return st;
}

/* periodic_spectrum eigenvalues (linalg.cpp:160-181) and the radius /
 * condition reductions (:183-193); eig: 2 doubles per mode */
void sko_periodic_eigen(int dim, int nent, const int* off, const double* coeff, int h_power, const int64_t* n,
                        double h, double shift, double scale, double* eig, double* rho_out, double* cond_out) {
  const double two_pi = 2 * 3.141592653589793;
  const double scale_total = scale * pow_int(h, h_power);
  int64_t modes = 1;
  for (int a = 0; a < dim; ++a) modes *= n[a];
  double rho = 0, min_nz = 0;
  for (int64_t m = 0; m < modes; ++m) {
    int64_t rem = m;
    double theta[3];
    for (int a = 0; a < dim; ++a) {
      theta[a] = two_pi * (double)(rem % n[a]) / (double)n[a];
      rem /= n[a];
    }
    double re = 0, im = 0;
    for (int e = 0; e < nent; ++e) {
      double phase = 0;
      for (int a = 0; a < dim; ++a) phase += theta[a] * off[e * dim + a];
      re += coeff[e] * cos(phase);
      im += coeff[e] * sin(phase);
    }
    eig[2 * m] = shift + scale_total * re;
    eig[2 * m + 1] = scale_total * im;
    const double mag = hypot(eig[2 * m], eig[2 * m + 1]);
    if (mag > rho) rho = mag;
  }
  for (int64_t m = 0; m < modes; ++m) {
    const double mag = hypot(eig[2 * m], eig[2 * m + 1]);
    if (mag > 1e-12 * rho && (min_nz == 0 || mag < min_nz)) min_nz = mag;
  }
  *rho_out = rho;
  *cond_out = min_nz > 0 ? rho / min_nz : 0;
}

/* ch_init (cahn_hilliard.cpp:20-63), origin 0 */
void sko_ch_init(int dim, int64_t n, double h, double c0, double eps, double* out) {
  if (dim == 2) {
    for (int64_t j = 0; j < n; ++j) {
      const double y = 0.0 + (int)j * h;
      for (int64_t i = 0; i < n; ++i) {
        const double x = 0.0 + (int)i * h;
        const double c2 = cos(0.13 * x) * cos(0.087 * y);
        out[j * n + i] = c0 + eps * (cos(0.105 * x) * cos(0.11 * y) + c2 * c2 +
                                     cos(0.025 * x - 0.15 * y) * cos(0.07 * x - 0.02 * y));
      }
    }
  } else {
    for (int64_t k = 0; k < n; ++k) {
      const double z = 0.0 + (int)k * h;
      for (int64_t j = 0; j < n; ++j) {
        const double y = 0.0 + (int)j * h;
        for (int64_t i = 0; i < n; ++i) {
          const double x = 0.0 + (int)i * h;
          const double c2 = cos(0.13 * x) * cos(0.087 * y) * cos(0.1 * z);
          out[(k * n + j) * n + i] =
              c0 + eps * (cos(0.105 * x) * cos(0.11 * y) * cos(0.11 * z) + c2 * c2 +
                          cos(0.025 * x - 0.15 * y - 0.1 * z) * cos(0.07 * x - 0.02 * y + 0.01 * z));
        }
      }
    }
  }
}

/* free_energy, serial form (cahn_hilliard.cpp:77-107,116-119) */
double sko_free_energy(int dim, int64_t n, double h, double kappa, double rho_w, double c_alpha, double c_beta,
                       const double* c) {
  const double inv_2h = 0.5 / h;
  int64_t stride[3], count = 1;
  for (int a = 0; a < dim; ++a) {
    stride[a] = count;
    count *= n;
  }
  double total = 0;
  for (int64_t idx = 0; idx < count; ++idx) {
    const double a0 = c[idx] - c_alpha, b0 = c[idx] - c_beta;
    double cell = rho_w * a0 * a0 * b0 * b0; /* f_chem :65-68 */
    int64_t rem = idx;
    for (int a = 0; a < dim; ++a) {
      const int64_t ia = rem % n;
      rem /= n;
      const int64_t up = idx + stride[a] * ((ia + 1 == n) ? 1 - n : 1);
      const int64_t dn = idx - stride[a] * ((ia == 0) ? 1 - n : 1);
      const double grad = (c[up] - c[dn]) * inv_2h;
      cell += 0.5 * kappa * grad * grad;
    }
    total += cell;
  }
  return total * pow_int(h, dim);
}

/* ---- clamped biharmonic manufactured problem (BASELINE configs 2 and 5) --
 * u = prod_i a(x_i), a(x) = sin^2(pi x); a'' = 2 pi^2 cos(2 pi x),
 * a'''' = -8 pi^4 cos(2 pi x); f = Delta^2 u = sum_i a''''_i prod_{j!=i} a_j
 * + 2 sum_{i<j} a''_i a''_j prod_{k!=i,j} a_k. Unknowns at x = (i+1) h,
 * h = 1/intervals (experiments.cpp:105-124 layout). */
void sko_biharmonic_clamped(int dim, int64_t intervals, double* f, double* u_exact) {
  const double pi = 3.14159265358979323846;
  const double h = 1.0 / (double)intervals;
  const int64_t m = intervals - 1;
  int64_t count = 1;
  for (int a = 0; a < dim; ++a) count *= m;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < count; ++r) {
    double av[3], a2[3], a4[3];
    int64_t rem = r;
    for (int d = 0; d < dim; ++d) {
      const double x = (double)(rem % m + 1) * h;
      rem /= m;
      const double s = sin(pi * x), cs = cos(2.0 * pi * x);
      av[d] = s * s;
      a2[d] = 2.0 * pi * pi * cs;
      a4[d] = -8.0 * pi * pi * pi * pi * cs;
    }
    double u = 1.0, fv = 0.0;
    for (int d = 0; d < dim; ++d) u *= av[d];
    for (int i = 0; i < dim; ++i) {
      double t = a4[i];
      for (int j = 0; j < dim; ++j)
        if (j != i) t *= av[j];
      fv += t;
    }
    for (int i = 0; i < dim; ++i)
      for (int j = i + 1; j < dim; ++j) {
        double t = 2.0 * a2[i] * a2[j];
        for (int k = 0; k < dim; ++k)
          if (k != i && k != j) t *= av[k];
        fv += t;
      }
    f[r] = fv;
    if (u_exact) u_exact[r] = u;
  }
}

/* fit_loglog (experiments.cpp:16-42). Returns 0 or 18 (InvalidArgument). */
int sko_fit_loglog(int count, const double* h, const double* err, double* slope, double* coeff, double* resid) {
  if (count < 3) return 18;
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  const double n = (double)count;
  for (int i = 0; i < count; ++i) {
    if (!(h[i] > 0) || !(err[i] > 0)) return 18;
    const double lx = log(h[i]), ly = log(err[i]);
    sx += lx;
    sy += ly;
    sxx += lx * lx;
    sxy += lx * ly;
  }
  *slope = (n * sxy - sx * sy) / (n * sxx - sx * sx);
  const double intercept = (sy - *slope * sx) / n;
  *coeff = exp(intercept);
  double rss = 0;
  for (int i = 0; i < count; ++i) {
    const double r = log(err[i]) - (*slope * log(h[i]) + intercept);
    rss += r * r;
  }
  *resid = sqrt(rss / n);
  return 0;
}

/* std::mt19937_64 (the published MT19937-64 recurrence) + libstdc++'s
 * uniform_real_distribution<double>: generate_canonical draws one 64-bit word,
 * r = word / 2^64 (nudged below 1), value = r * (hi - lo) + lo. */
void sko_uniform(uint64_t seed, int64_t count, double lo, double hi, double* out) {
  enum { NN = 312, MM = 156 };
  const uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL, UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  uint64_t mt[NN];
  int mti;
  mt[0] = seed;
  for (mti = 1; mti < NN; mti++) mt[mti] = 6364136223846793005ULL * (mt[mti - 1] ^ (mt[mti - 1] >> 62)) + (uint64_t)mti;
  for (int64_t k = 0; k < count; ++k) {
    if (mti >= NN) {
      int i;
      uint64_t x;
      for (i = 0; i < NN - MM; i++) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + MM] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
      }
      for (; i < NN - 1; i++) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + (MM - NN)] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
      }
      x = (mt[NN - 1] & UM) | (mt[0] & LM);
      mt[NN - 1] = mt[MM - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
      mti = 0;
    }
    uint64_t y = mt[mti++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    double r = (double)y / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    out[k] = r * (hi - lo) + lo;
  }
}
