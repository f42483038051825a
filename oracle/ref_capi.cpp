// ORACLE TEST INFRASTRUCTURE — never linked into the product.
//
// A C-ABI over the UNMODIFIED reference library (`/root/reference/proj/src`,
// compiled by oracle/Makefile into oracle/_ref/libstencilkit_ref.so) so the
// Python tests and bench.py's CPU-baseline leg can call the reference's own
// code path. Everything here calls reference APIs only; the two pieces the
// reference does not have are restated explicitly and marked EXTENSION:
//   * clamped (even-reflection) assembly — grid.cpp:62-158 with the sign flip
//     of :111/:115 removed;
//   * the explicit forward-Euler Cahn-Hilliard step built from the stepper's
//     own pieces (cahn_hilliard.cpp:126-128 matrices, :148-152 chemistry).
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "stencilkit/cahn_hilliard.hpp"
#include "stencilkit/experiments.hpp"
#include "stencilkit/generators.hpp"
#include "stencilkit/grid.hpp"
#include "stencilkit/kernels.hpp"
#include "stencilkit/linalg.hpp"
#include "stencilkit/runtime.hpp"

using namespace stencilkit;

namespace {

thread_local std::string g_err;

int fail(const Error& e) {
  g_err = e.what();
  return static_cast<int>(e.code()) + 1;
}
int fail_std(const std::exception& e) {
  g_err = e.what();
  return 1000;
}

// kind: 0 identity, 1 laplacian(dim, acc), 2 compose(lap, lap),
//       3 make({deriv=acc... }) is not needed on the hot path.
Stencil build_stencil(int dim, int acc, int kind) {
  if (kind == 0) return Stencil::identity(dim);
  Stencil lap = laplacian(dim, acc);
  if (kind == 1) return lap;
  if (kind == 2) return compose(lap, lap);
  if (kind == 3) return scale(lap, Rational(-1));
  if (kind == 4) return scale(compose(lap, lap), Rational(1));
  throw Error(Errc::invalid_argument, "unknown stencil kind");
}

GridSpec build_grid(int dim, const int* n, double h, const int* bc) {
  GridSpec g;
  g.dim = dim;
  g.h = h;
  for (int a = 0; a < dim; ++a) {
    g.n.push_back(n[a]);
    g.origin.push_back(0.0);
    // 2 (clamped) is an EXTENSION; the reference grid sees simply_supported
    g.bc.push_back(bc[a] == 0 ? BoundaryKind::periodic : BoundaryKind::simply_supported);
  }
  return g;
}

// EXTENSION: grid.cpp:62-158 restated with even reflection (clamped plate:
// u = 0 on the boundary, ghost u_{-k} = u_{k} so du/dn = 0). Identical to the
// reference loop except that the reflected value keeps its sign.
CsrMatrix assemble_mixed(const Stencil& s, const GridSpec& g, const int* bc) {
  bool any_clamped = false;
  for (int a = 0; a < g.dim; ++a) any_clamped |= bc[a] == 2;
  if (!any_clamped) return assemble(s, g);

  g.validate();
  if (s.dim() != g.dim) throw Error(Errc::dim_mismatch, "stencil/grid dimension mismatch");
  for (int a = 0; a < g.dim; ++a) {
    auto [lo, hi] = s.support(a);
    if (g.bc[a] == BoundaryKind::periodic) {
      if (hi - lo > g.n[a] - 1)
        throw Error(Errc::stencil_wider_than_grid, "periodic axis narrower than stencil support");
    } else if (std::max(std::abs(lo), std::abs(hi)) > g.n[a] - 2) {
      throw Error(Errc::stencil_wider_than_grid, "reflected ghost would leave the grid");
    }
  }
  const double scale_h = pow_int(g.h, s.h_power());
  struct Flat {
    std::vector<int> off;
    double value;
  };
  std::vector<Flat> entries;
  for (const auto& [off, coeff] : s.entries())
    entries.push_back({std::vector<int>(off.begin(), off.end()), coeff.to_double() * scale_h});
  std::vector<int> un(static_cast<size_t>(g.dim));
  for (int a = 0; a < g.dim; ++a) un[static_cast<size_t>(a)] = g.unknowns_per_axis(a);
  const std::int64_t rows = g.unknown_count();
  std::vector<std::vector<std::pair<std::int64_t, double>>> row_entries(static_cast<size_t>(rows));
#pragma omp parallel for schedule(static)
  for (std::int64_t row = 0; row < rows; ++row) {
    std::vector<int> idx(static_cast<size_t>(g.dim));
    std::int64_t rem = row;
    for (int a = 0; a < g.dim; ++a) {
      idx[static_cast<size_t>(a)] = static_cast<int>(rem % un[static_cast<size_t>(a)]);
      rem /= un[static_cast<size_t>(a)];
    }
    auto& out = row_entries[static_cast<size_t>(row)];
    for (const auto& e : entries) {
      double val = e.value;
      std::int64_t col = 0, stride = 1;
      bool dropped = false;
      for (int a = 0; a < g.dim && !dropped; ++a) {
        const int na = g.n[static_cast<size_t>(a)];
        int comp;
        if (bc[a] == 0) {
          comp = ((idx[static_cast<size_t>(a)] + e.off[static_cast<size_t>(a)]) % na + na) % na;
        } else {
          int gi = idx[static_cast<size_t>(a)] + 1 + e.off[static_cast<size_t>(a)];
          const bool odd = bc[a] == 1;
          if (gi < 0) {
            gi = -gi;
            if (odd) val = -val;
          } else if (gi > na - 1) {
            gi = 2 * (na - 1) - gi;
            if (odd) val = -val;
          }
          if (gi == 0 || gi == na - 1) {
            dropped = true;
            break;
          }
          comp = gi - 1;
        }
        col += stride * comp;
        stride *= un[static_cast<size_t>(a)];
      }
      if (!dropped) out.emplace_back(col, val);
    }
    std::sort(out.begin(), out.end());
    size_t w = 0;
    for (size_t r = 0; r < out.size();) {
      std::int64_t c = out[r].first;
      double v = 0;
      while (r < out.size() && out[r].first == c) v += out[r++].second;
      if (v != 0.0) out[w++] = {c, v};
    }
    out.resize(w);
  }
  CsrMatrix m;
  m.rows = m.cols = rows;
  m.row_ptr.resize(static_cast<size_t>(rows) + 1, 0);
  for (std::int64_t i = 0; i < rows; ++i)
    m.row_ptr[static_cast<size_t>(i) + 1] =
        m.row_ptr[static_cast<size_t>(i)] + static_cast<std::int64_t>(row_entries[static_cast<size_t>(i)].size());
  m.col_idx.resize(static_cast<size_t>(m.row_ptr.back()));
  m.values.resize(static_cast<size_t>(m.row_ptr.back()));
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < rows; ++i) {
    std::int64_t k = m.row_ptr[static_cast<size_t>(i)];
    for (const auto& [c, v] : row_entries[static_cast<size_t>(i)]) {
      m.col_idx[static_cast<size_t>(k)] = c;
      m.values[static_cast<size_t>(k)] = v;
      ++k;
    }
  }
  return m;
}

CahnHilliardParams ch_params(double mobility, double kappa, double rho_w, double c_alpha, double c_beta) {
  CahnHilliardParams p;
  p.mobility = mobility;
  p.kappa = kappa;
  p.rho_w = rho_w;
  p.c_alpha = c_alpha;
  p.c_beta = c_beta;
  return p;
}

}  // namespace

extern "C" {

const char* skref_last_error() { return g_err.c_str(); }
int skref_threads() { return thread_count(); }
void skref_set_threads(int t) { set_thread_count(t); }

// Reference stencil entries in std::map order. coeff_d = Rational::to_double
// (rational.hpp:32); num/den exact (must fit int64).
int skref_stencil(int dim, int acc, int kind, int cap, int* nent, int* offsets, double* coeff_d,
                  long long* num, long long* den, int* h_power) {
  try {
    Stencil s = build_stencil(dim, acc, kind);
    *nent = static_cast<int>(s.entries().size());
    *h_power = s.h_power();
    if (*nent > cap) return 0;
    int k = 0;
    for (const auto& [off, c] : s.entries()) {
      for (int a = 0; a < dim; ++a) offsets[k * dim + a] = off[static_cast<size_t>(a)];
      coeff_d[k] = c.to_double();
      num[k] = std::stoll(c.num().get_str());
      den[k] = std::stoll(c.den().get_str());
      ++k;
    }
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

// bc per axis: 0 periodic, 1 simply supported (reference), 2 clamped (EXTENSION)
int skref_assemble(int dim, int acc, int kind, const int* n, double h, const int* bc, void** out) {
  try {
    Stencil s = build_stencil(dim, acc, kind);
    GridSpec g = build_grid(dim, n, h, bc);
    *out = new CsrMatrix(assemble_mixed(s, g, bc));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

// Assemble from explicit stencil entries (used for the random-stencil
// compose-before-assemble checks): offsets[nent*dim], exact num/den.
int skref_assemble_entries(int dim, int nent, const int* offsets, const long long* num,
                           const long long* den, int h_power, const int* n, double h, const int* bc,
                           void** out) {
  try {
    std::map<Offset, Rational> e;
    for (int k = 0; k < nent; ++k) {
      Offset o(static_cast<size_t>(dim));
      for (int a = 0; a < dim; ++a) o[static_cast<size_t>(a)] = offsets[k * dim + a];
      e[o] += Rational(static_cast<long>(num[k]), static_cast<long>(den[k]));
    }
    Stencil s(dim, h_power, std::move(e));
    GridSpec g = build_grid(dim, n, h, bc);
    *out = new CsrMatrix(assemble_mixed(s, g, bc));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

long long skref_csr_rows(void* m) { return static_cast<CsrMatrix*>(m)->rows; }
long long skref_csr_nnz(void* m) { return static_cast<CsrMatrix*>(m)->nnz(); }
void skref_csr_copy(void* mp, long long* row_ptr, long long* col_idx, double* values) {
  auto* m = static_cast<CsrMatrix*>(mp);
  std::memcpy(row_ptr, m->row_ptr.data(), m->row_ptr.size() * sizeof(long long));
  std::memcpy(col_idx, m->col_idx.data(), m->col_idx.size() * sizeof(long long));
  std::memcpy(values, m->values.data(), m->values.size() * sizeof(double));
}
void skref_csr_free(void* m) { delete static_cast<CsrMatrix*>(m); }

void skref_csr_matvec(void* mp, const double* x, double* y, int serial) {
  auto* m = static_cast<CsrMatrix*>(mp);
  std::span<const double> xs(x, static_cast<size_t>(m->cols));
  std::span<double> ys(y, static_cast<size_t>(m->rows));
  if (serial)
    kernels::serial::csr_matvec(*m, xs, ys);
  else
    kernels::csr_matvec(*m, xs, ys);
}

double skref_dot(long long n, const double* a, const double* b, int serial) {
  std::span<const double> as(a, static_cast<size_t>(n)), bs(b, static_cast<size_t>(n));
  return serial ? kernels::serial::dot(as, bs) : kernels::dot(as, bs);
}
double skref_nrm2(long long n, const double* a, int serial) {
  std::span<const double> as(a, static_cast<size_t>(n));
  return serial ? kernels::serial::nrm2(as) : kernels::nrm2(as);
}
double skref_sum(long long n, const double* a, int serial) {
  std::span<const double> as(a, static_cast<size_t>(n));
  return serial ? kernels::serial::sum(as) : kernels::sum(as);
}
void skref_minmax(long long n, const double* a, double* lo, double* hi, int serial) {
  std::span<const double> as(a, static_cast<size_t>(n));
  if (serial)
    kernels::serial::minmax(as, *lo, *hi);
  else
    kernels::minmax(as, *lo, *hi);
}
void skref_axpy(long long n, double alpha, const double* x, double* y, int serial) {
  std::span<const double> xs(x, static_cast<size_t>(n));
  std::span<double> ys(y, static_cast<size_t>(n));
  if (serial)
    kernels::serial::axpy(alpha, xs, ys);
  else
    kernels::axpy(alpha, xs, ys);
}
void skref_xpby(long long n, const double* x, double beta, double* y, int serial) {
  std::span<const double> xs(x, static_cast<size_t>(n));
  std::span<double> ys(y, static_cast<size_t>(n));
  if (serial)
    kernels::serial::xpby(xs, beta, ys);
  else
    kernels::xpby(xs, beta, ys);
}

// Reference cg_solve (linalg.cpp:15-72). Returns 0 or Errc+1.
int skref_cg_solve(void* mp, const double* b, double* x, double rel_tol, long long max_iter,
                   int deflate_mean) {
  try {
    auto* m = static_cast<CsrMatrix*>(mp);
    SolveOptions o;
    o.rel_tol = rel_tol;
    o.max_iter = max_iter;
    o.deflate_mean = deflate_mean != 0;
    std::vector<double> r = cg_solve(*m, std::span<const double>(b, static_cast<size_t>(m->rows)), o);
    std::memcpy(x, r.data(), r.size() * sizeof(double));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

// EXTENSION: explicit forward-Euler CH on a periodic grid, from the stepper's
// own matrices (cahn_hilliard.cpp:126-128) and chemistry (:148-152):
//   w = f_chem_prime(c); a = L w; b = B c; c += dt * M * (a - kappa * b)
// The matrices are built once per handle so timing loops can exclude them.
struct ChExplicit {
  CsrMatrix lap, bilap;
  CahnHilliardParams p;
  std::vector<double> w, a, b;
};

int skref_ch_create(int dim, int n, double h, double mobility, double kappa, double rho_w,
                    double c_alpha, double c_beta, void** out) {
  try {
    GridSpec g = make_periodic_grid(dim, n, h);
    auto* s = new ChExplicit;
    Stencil lap = laplacian(dim, 2);
    s->lap = assemble(lap, g);
    s->bilap = assemble(compose(lap, lap), g);
    s->p = ch_params(mobility, kappa, rho_w, c_alpha, c_beta);
    const size_t rows = static_cast<size_t>(s->lap.rows);
    s->w.resize(rows);
    s->a.resize(rows);
    s->b.resize(rows);
    *out = s;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

void skref_ch_steps(void* sp, double dt, long long nsteps, double* c) {
  auto* s = static_cast<ChExplicit*>(sp);
  const std::int64_t n = s->lap.rows;
  std::span<const double> cs(c, static_cast<size_t>(n));
  const double mob = s->p.mobility, kappa = s->p.kappa;
  for (long long k = 0; k < nsteps; ++k) {
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < n; ++i) s->w[static_cast<size_t>(i)] = f_chem_prime(c[i], s->p);
    kernels::csr_matvec(s->lap, s->w, s->a);
    kernels::csr_matvec(s->bilap, cs, s->b);
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < n; ++i)
      c[i] += dt * mob * (s->a[static_cast<size_t>(i)] - kappa * s->b[static_cast<size_t>(i)]);
  }
}

void skref_ch_free(void* s) { delete static_cast<ChExplicit*>(s); }

// The reference IMEX stepper itself (cahn_hilliard.cpp:121-189): one
// CahnHilliardStepper per handle, so the AB2 history and the implicit-matrix
// cache persist across calls exactly as in the reference.
struct ImexHandle {
  GridSpec grid;
  CahnHilliardStepper stepper;
  ImexHandle(const GridSpec& g, const CahnHilliardParams& p, double rel_tol)
      : grid(g), stepper(g, p, SolveOptions{.rel_tol = rel_tol}) {}
};

int skref_imex_create(int dim, int n, double h, double mobility, double kappa, double rho_w,
                      double c_alpha, double c_beta, double rel_tol, void** out) {
  try {
    GridSpec g = make_periodic_grid(dim, n, h);
    *out = new ImexHandle(g, ch_params(mobility, kappa, rho_w, c_alpha, c_beta), rel_tol);
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

int skref_imex_steps(void* hp, double dt, int order, long long nsteps, double* c) {
  try {
    auto* hd = static_cast<ImexHandle*>(hp);
    CahnHilliardState st;
    st.grid = hd->grid;
    st.c.assign(c, c + hd->grid.unknown_count());
    for (long long k = 0; k < nsteps; ++k) hd->stepper.step(st, dt, order);
    std::memcpy(c, st.c.data(), st.c.size() * sizeof(double));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

void skref_imex_free(void* h) { delete static_cast<ImexHandle*>(h); }

// ch_init (cahn_hilliard.cpp:20-63) with the given c0 / eps_ic
int skref_ch_init(int dim, int n, double h, double c0, double eps_ic, double* out) {
  try {
    CahnHilliardParams p;
    p.c0 = c0;
    p.eps_ic = eps_ic;
    CahnHilliardState st = ch_init(make_periodic_grid(dim, n, h), p);
    std::memcpy(out, st.c.data(), st.c.size() * sizeof(double));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

// csr_matmul (linalg.cpp:253-283) of two assembled handles: b * a
void* skref_csr_matmul(void* b, void* a) {
  return new CsrMatrix(csr_matmul(*static_cast<CsrMatrix*>(b), *static_cast<CsrMatrix*>(a)));
}

// identity_plus_scaled (linalg.cpp:224-251) on an assembled operator
void* skref_identity_plus_scaled(void* mp, double alpha) {
  return new CsrMatrix(identity_plus_scaled(*static_cast<CsrMatrix*>(mp), alpha));
}

// power_iteration (linalg.cpp:74-106) on an assembled handle
int skref_power_iteration(void* mp, double tol, unsigned long long seed, long long max_iter, double* out) {
  try {
    *out = power_iteration(*static_cast<CsrMatrix*>(mp), tol, seed, max_iter);
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// periodic_spectrum (linalg.cpp:149-222) of build_stencil(dim, acc, kind)
int skref_periodic_spectrum(int dim, int acc, int kind, const int* n, double h, double shift, double scale,
                            double* eig, double* rho, double* sym, double* cond) {
  try {
    GridSpec g = make_periodic_grid(dim, n[0], h);
    for (int a = 0; a < dim; ++a) g.n[static_cast<size_t>(a)] = n[a];
    SpectrumReport r = periodic_spectrum(build_stencil(dim, acc, kind), g, shift, scale);
    for (size_t i = 0; i < r.eigenvalues.size(); ++i) {
      eig[2 * i] = r.eigenvalues[i].real();
      eig[2 * i + 1] = r.eigenvalues[i].imag();
    }
    *rho = r.spectral_radius;
    *sym = r.symbol_radius;
    *cond = r.condition_estimate;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

double skref_free_energy(int dim, int n, double h, double kappa, double rho_w, double c_alpha,
                         double c_beta, const double* c, int serial) {
  CahnHilliardState st;
  st.grid = make_periodic_grid(dim, n, h);
  st.c.assign(c, c + st.grid.unknown_count());
  CahnHilliardParams p = ch_params(1.0, kappa, rho_w, c_alpha, c_beta);
  return serial ? free_energy_serial(st, p) : free_energy(st, p);
}

double skref_f_chem_prime(double c, double rho_w, double c_alpha, double c_beta) {
  return f_chem_prime(c, ch_params(1.0, 1.0, rho_w, c_alpha, c_beta));
}

// std::mt19937_64(seed) + uniform_real_distribution<double>(lo, hi), drawn in
// order (linalg.cpp:77-78, bench_kernels.cpp:42-43, test_kernels.cpp:15-19).
void skref_uniform(unsigned long long seed, long long n, double lo, double hi, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(lo, hi);
  for (long long i = 0; i < n; ++i) out[i] = unit(rng);
}

// fit_loglog (experiments.cpp:16-42)
int skref_fit_loglog(int n, const double* h, const double* err, double* slope, double* coeff,
                     double* resid) {
  try {
    std::vector<std::pair<double, double>> s;
    for (int i = 0; i < n; ++i) s.emplace_back(h[i], err[i]);
    ConvergenceFit f = fit_loglog(std::move(s));
    *slope = f.slope;
    *coeff = f.coefficient;
    *resid = f.fit_residual;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// biharmonic_solve (experiments.cpp:99-143) — simply supported, sin*sin.
int skref_biharmonic_solve(int nlad, const int* ladder, double rel_tol, double* slope, double* coeff,
                           double* residuals) {
  try {
    std::vector<int> lad(ladder, ladder + nlad);
    BiharmonicResult r = biharmonic_solve(lad, rel_tol);
    *slope = r.fit.slope;
    *coeff = r.fit.coefficient;
    for (int i = 0; i < nlad; ++i) residuals[i] = r.residuals[static_cast<size_t>(i)];
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

}  // extern "C"
