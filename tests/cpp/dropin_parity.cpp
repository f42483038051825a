// Drop-in parity: the reference library's own C++ API against
// stencilkit::cuda (include/stencilkit/cuda.hpp) on identical inputs.
//
// Built by `make -C oracle _ref/dropin_parity` against the UNMODIFIED
// reference headers and library (oracle/_ref/libstencilkit_ref.so) and the
// product library (libsk_cuda.so); run on a GPU by tests/test_gpu_dropin.py.
// This is the integration a reference maintainer would do: swap
// stencilkit::assemble / kernels::csr_matvec / cg_solve for the
// stencilkit::cuda versions and get the same CsrMatrix and the same numbers.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "stencilkit/cahn_hilliard.hpp"
#include "stencilkit/cuda.hpp"
#include "stencilkit/generators.hpp"
#include "stencilkit/grid.hpp"
#include "stencilkit/kernels.hpp"
#include "stencilkit/linalg.hpp"

using namespace stencilkit;

static int failures = 0;
#define EXPECT(cond, what)                                   \
  do {                                                       \
    if (!(cond)) {                                           \
      std::printf("FAIL: %s (%s:%d)\n", what, __FILE__, __LINE__); \
      ++failures;                                            \
    } else {                                                 \
      std::printf("ok: %s\n", what);                         \
    }                                                        \
  } while (0)

static std::vector<double> uniform(std::uint64_t seed, std::size_t n) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(-1.0, 1.0);
  std::vector<double> v(n);
  for (auto& x : v) x = unit(rng);
  return v;
}

static GridSpec ss_grid(int dim, int intervals) {
  GridSpec g;
  g.dim = dim;
  g.n.assign(static_cast<size_t>(dim), intervals + 1);
  g.h = 1.0 / intervals;
  g.origin.assign(static_cast<size_t>(dim), 0.0);
  g.bc.assign(static_cast<size_t>(dim), BoundaryKind::simply_supported);
  return g;
}

static bool same_csr(const CsrMatrix& a, const CsrMatrix& b) {
  return a.rows == b.rows && a.cols == b.cols && a.row_ptr == b.row_ptr && a.col_idx == b.col_idx &&
         a.values == b.values;
}

int main() {
  if (sk_device_init(0) != SK_OK) {
    std::printf("no device: %s\n", sk_last_error());
    return 2;
  }
  const Stencil lap2 = laplacian(2, 2), bilap2 = compose(lap2, lap2);
  const Stencil lap3_4 = laplacian(3, 4), bilap3_4 = compose(lap3_4, lap3_4);

  // assemble: periodic 13-point (test_kernels.cpp:26-35 grid) and simply-supported 73-point
  {
    const GridSpec g = make_periodic_grid(2, 37, 1.0);
    EXPECT(same_csr(assemble(bilap2, g), cuda::assemble(bilap2, g)), "assemble 13-pt periodic 37^2 bit-identical");
    const GridSpec g3 = ss_grid(3, 20);
    EXPECT(same_csr(assemble(bilap3_4, g3), cuda::assemble(bilap3_4, g3)), "assemble 73-pt simply supported 19^3");
  }
  // csr_matvec: bit-identical to the reference's serial kernel
  {
    const GridSpec g = make_periodic_grid(2, 64, 1.0 / 64);
    const CsrMatrix m = assemble(bilap2, g);
    const std::vector<double> x = uniform(99, static_cast<size_t>(m.rows));
    std::vector<double> y_ref(x.size()), y_gpu(x.size());
    kernels::serial::csr_matvec(m, x, y_ref);
    cuda::kernels::csr_matvec(m, x, y_gpu);
    EXPECT(y_ref == y_gpu, "csr_matvec bit-identical to kernels::serial::csr_matvec");
    const std::vector<double> v = cuda::composed_apply(bilap2, g, x);
    double err = 0, mx = 0;
    for (size_t i = 0; i < v.size(); ++i) {
      err = std::max(err, std::abs(v[i] - y_ref[i]));
      mx = std::max(mx, std::abs(y_ref[i]));
    }
    EXPECT(err <= 1e-12 * mx, "matrix-free composed_apply within 1e-12 of assemble+csr_matvec");
    bool threw = false;
    try {
      cuda::apply(m, std::vector<double>(x.size() + 1));
    } catch (const Error& e) {
      threw = e.code() == Errc::shape_mismatch;
    }
    EXPECT(threw, "apply throws ShapeMismatch on a length mismatch (grid.cpp:167-168)");
  }
  // cg_solve: reference simply-supported biharmonic problem (experiments.cpp:99-126)
  {
    const GridSpec g = ss_grid(2, 32);
    const CsrMatrix m = assemble(bilap2, g);
    std::vector<double> b(static_cast<size_t>(m.rows));
    const int nu = g.unknowns_per_axis(0);
    for (std::int64_t r = 0; r < m.rows; ++r) {
      const double x = g.coordinate(0, static_cast<int>(r % nu)), y = g.coordinate(1, static_cast<int>(r / nu));
      b[static_cast<size_t>(r)] = 4.0 * std::pow(M_PI, 4) * std::sin(M_PI * x) * std::sin(M_PI * y);
    }
    const std::vector<double> x_ref = cg_solve(m, b, {.rel_tol = 1e-10});
    const std::vector<double> x_gpu = cuda::cg_solve(m, b, {.rel_tol = 1e-10});
    double d = 0, n = 0;
    for (size_t i = 0; i < b.size(); ++i) {
      d += (x_ref[i] - x_gpu[i]) * (x_ref[i] - x_gpu[i]);
      n += x_ref[i] * x_ref[i];
    }
    EXPECT(std::sqrt(d) <= 1e-8 * std::sqrt(n), "cg_solve within 1e-8 of the reference");
    bool threw = false;
    try {
      const CsrMatrix neg = assemble(lap2, make_periodic_grid(2, 8, 1.0));  // negative semi-definite
      cuda::cg_solve(neg, uniform(1, 64));
    } catch (const Error& e) {
      threw = e.code() == Errc::no_convergence;
    }
    EXPECT(threw, "cg_solve throws NoConvergence on a non-PD matrix (linalg.cpp:50-51)");
  }
  // free_energy and the explicit CH step from the stepper's own matrices
  {
    CahnHilliardParams p;
    p.kappa = 1e-4;
    p.mobility = 1.0;
    p.rho_w = 0.25;
    p.c_alpha = -1.0;
    p.c_beta = 1.0;
    const int n = 64;
    const double h = 1.0 / n, dt = 0.25 * std::pow(h, 4) / (64.0 * p.kappa);
    CahnHilliardState s;
    s.grid = make_periodic_grid(2, n, h);
    s.c = uniform(1, static_cast<size_t>(n) * n);
    for (auto& v : s.c) v *= 0.05;
    const double e_ref = free_energy(s, p), e_gpu = cuda::free_energy(s, p);
    EXPECT(std::abs(e_ref - e_gpu) <= 1e-12 * std::abs(e_ref), "free_energy within 1e-12");
    CahnHilliardStepper st(s.grid, p);  // reference L and B (cahn_hilliard.cpp:126-128)
    std::vector<double> c = s.c, w(c.size()), a(c.size()), bb(c.size());
    for (int k = 0; k < 40; ++k) {
      for (size_t i = 0; i < c.size(); ++i) w[i] = f_chem_prime(c[i], p);
      kernels::csr_matvec(st.laplacian_matrix(), w, a);
      kernels::csr_matvec(st.bilaplacian_matrix(), c, bb);
      for (size_t i = 0; i < c.size(); ++i) c[i] += dt * p.mobility * (a[i] - p.kappa * bb[i]);
    }
    for (int form : {SK_CH_FACTORED, SK_CH_COMPOSED}) {
      CahnHilliardState g = s;
      cuda::CahnHilliardExplicit(g.grid, p, form).step(g, dt, 40);
      double d = 0, nn = 0;
      for (size_t i = 0; i < c.size(); ++i) {
        d += (g.c[i] - c[i]) * (g.c[i] - c[i]);
        nn += c[i] * c[i];
      }
      EXPECT(std::sqrt(d) <= 1e-9 * std::sqrt(nn),
             form == SK_CH_FACTORED ? "explicit CH (factored kernel) within 1e-9 after 40 steps"
                                    : "explicit CH (composed kernel) within 1e-9 after 40 steps");
    }
  }
  {  // the multi-GPU slab stepper (one rank: its ghosts are its own) against
     // the single-domain drop-in stepper, bit for bit
    CahnHilliardParams p;
    p.kappa = 0.02 * 0.02;
    const int n = 32;
    const double h = 1.0 / n, dt = 0.2 * h * h * h * h / (144 * p.kappa);
    CahnHilliardState s;
    s.grid = make_periodic_grid(3, n, h);
    s.c = uniform(3, static_cast<size_t>(n) * n * n);
    for (auto& v : s.c) v *= 0.05;
    const size_t plane = static_cast<size_t>(n) * n;
    std::vector<double> ghosted((n + 4) * plane);
    for (int k = -2; k < n + 2; ++k)
      std::copy_n(s.c.begin() + ((k + n) % n) * plane, plane, ghosted.begin() + (k + 2) * plane);
    cuda::SlabStepper slab(s.grid, p);
    slab.connect_self();
    slab.load(ghosted);
    for (int k = 0; k < 6; ++k) slab.step(dt);
    CahnHilliardState g = s;
    cuda::CahnHilliardExplicit(g.grid, p).step(g, dt, 6);
    EXPECT(slab.interior() == g.c, "SlabStepper (fused peer halo stores, 1 rank) bit-identical to the explicit stepper");
  }
  {  // IMEX: the reference CahnHilliardStepper vs the drop-in, same calls
    CahnHilliardParams p;  // the reference's benchmark parameters
    const GridSpec grid = make_periodic_grid(2, 40, 1.0);
    CahnHilliardState r = ch_init(grid, p), g = cuda::ch_init(grid, p);
    EXPECT(r.c == g.c, "ch_init bit-identical");
    CahnHilliardStepper rs(grid, p);
    cuda::CahnHilliardStepper gs(grid, p);
    const int orders[6] = {1, 2, 2, 2, 1, 2};
    for (int k = 0; k < 6; ++k) {
      rs.step(r, 0.05, orders[k]);
      cuda::imex_step(gs, g, 0.05, orders[k]);
    }
    double d = 0, nn = 0;
    for (size_t i = 0; i < r.c.size(); ++i) {
      d += (g.c[i] - r.c[i]) * (g.c[i] - r.c[i]);
      nn += r.c[i] * r.c[i];
    }
    EXPECT(std::sqrt(d) <= 1e-9 * std::sqrt(nn) && g.t == r.t, "IMEX stepper (orders 1/2, AB2 history) within 1e-9");
  }
  {  // spectral tools: the reference's own known answers (test_linalg.cpp:74-145)
    const Stencil bil = compose(laplacian(2, 2), laplacian(2, 2));  // builtin "bilaplacian-2d"
    const GridSpec g20 = make_periodic_grid(2, 20, 10.0);
    const double rho = cuda::power_iteration(assemble(bil, g20), 1e-8);
    const SpectrumReport r = periodic_spectrum(bil, g20), c = cuda::periodic_spectrum(bil, g20);
    EXPECT(std::abs(rho - r.spectral_radius) <= 1e-6 * r.spectral_radius, "power_iteration within 1e-6");
    EXPECT(c.spectral_radius == r.spectral_radius && c.symbol_radius == r.symbol_radius,
           "periodic_spectrum radii identical to the reference");
    const SpectrumReport t = cuda::periodic_spectrum(bil, make_periodic_grid(2, 50, 4.0), 1.0, 1.0);
    EXPECT(t.symbol_radius == 1.25 && t.spectral_radius == 1.25 && t.condition_estimate == 1.25,
           "time-stepping table row h=4 exact");
  }
  {  // csr_matmul: bit-identical to the reference's product
    const GridSpec g = make_periodic_grid(2, 33, 0.25);
    const CsrMatrix a = assemble(laplacian(2, 4), g), b = assemble(compose(laplacian(2, 2), laplacian(2, 2)), g);
    const CsrMatrix r = csr_matmul(b, a), c = cuda::csr_matmul(b, a);
    EXPECT(r.row_ptr == c.row_ptr && r.col_idx == c.col_idx && r.values == c.values, "csr_matmul bit-identical");
  }
  {  // exact-operator refinement (configs 2 / 5): the 73-point composition's Rational
     // coefficients reach the device as double + exact residue; the refined
     // solve agrees with the plain one where the weight rounding is negligible
    const Stencil bih = compose(laplacian(3, 4), laplacian(3, 4));
    const int N = 16;
    const GridSpec g = ss_grid(3, N);
    std::vector<double> b(static_cast<size_t>(g.unknown_count()));
    for (size_t i = 0; i < b.size(); ++i) b[i] = std::sin(0.01 * double(i)) + 1.0;
    sk_refine_report rep{};
    const std::vector<double> xr = cuda::cg_solve_refined(bih, g, b, SolveOptions{1e-10, 0, false}, true, 1e-6, 4, &rep);
    const std::vector<double> x0 = cuda::cg_solve(cuda::DeviceCsr(bih, g, true), b, SolveOptions{1e-9, 0, false});
    double d = 0, nn = 0;
    for (size_t i = 0; i < b.size(); ++i) {
      d += (xr[i] - x0[i]) * (xr[i] - x0[i]);
      nn += x0[i] * x0[i];
    }
    EXPECT(rep.refinements >= 1 && rep.last_correction_rel <= 1e-13, "refinement converged to fp64 resolution");
    EXPECT(std::sqrt(d) <= 1e-7 * std::sqrt(nn), "refined solve agrees with cg_solve (clamped 73-point, 15^3)");
    EXPECT(cuda::rational_residue(Rational(1607, 24), Rational(1607, 24).to_double()) != 0.0 &&
               cuda::rational_residue(Rational(20), 20.0) == 0.0,
           "exact residues of non-dyadic / integer weights");
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
