// stencilkit/cuda.hpp — drop-in B200 (sm_100a) replacements for the
// data-parallel half of the reference library, same names and argument
// types, in namespace stencilkit::cuda.
//
// Header-only C++ over the C-ABI in sk_cuda.h; include it next to the
// reference's own headers (it uses stencilkit::Stencil, GridSpec, CsrMatrix,
// SolveOptions, CahnHilliardParams/State and throws stencilkit::Error with
// the same Errc) and link libsk_cuda.so. Replaces:
//   assemble      grid.cpp:62-158        (GPU assembly, bit-identical CSR)
//   apply         grid.cpp:166-172       (shape check + device SpMV)
//   csr_matvec / dot / nrm2 / axpy / xpby / sum / minmax   kernels.cpp:8-60
//   cg_solve      linalg.cpp:15-72       (same contract, device loop)
//   free_energy   cahn_hilliard.cpp:111-114
// and adds what the reference lacks: composed_apply (matrix-free v = S u)
// and CahnHilliardExplicit (fused explicit step, BASELINE configs 3/4).
//
// Host-span overloads copy to and from the device on every call (the
// reference's calling convention); DeviceCsr / DeviceField keep data resident
// for loops.
#ifndef STENCILKIT_CUDA_HPP
#define STENCILKIT_CUDA_HPP

#include <sk_cuda.h>

#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "stencilkit/cahn_hilliard.hpp"
#include "stencilkit/grid.hpp"
#include "stencilkit/linalg.hpp"
#include "stencilkit/stencil.hpp"

namespace stencilkit::cuda {

/// Status -> exception: Errc-valued codes rethrow stencilkit::Error (error.hpp:33-41).
inline void check(int status) {
  if (status == SK_OK) return;
  const std::string msg = sk_last_error();
  if (status >= 1 && status <= SK_ERR_INVALID_ARGUMENT) throw Error(static_cast<Errc>(status - 1), msg);
  throw std::runtime_error("stencilkit::cuda: " + msg);
}

/// GridSpec -> descriptor. `clamped` selects even reflection on the
/// non-periodic axes (the reference only has simply_supported, grid.hpp:17).
inline sk_grid_desc grid_desc(const GridSpec& g, bool clamped = false) {
  g.validate();
  sk_grid_desc d{};
  d.dim = g.dim;
  d.h = g.h;
  for (int a = 0; a < 3; ++a) {
    d.n[a] = a < g.dim ? g.n[static_cast<size_t>(a)] : 1;
    d.bc[a] = a < g.dim && g.bc[static_cast<size_t>(a)] != BoundaryKind::periodic
                  ? (clamped ? SK_BC_CLAMPED : SK_BC_SIMPLY_SUPPORTED)
                  : SK_BC_PERIODIC;
  }
  return d;
}

/// q - hi exactly, rounded once (hi = q.to_double()): the exact-weight
/// correction of sk_stencil_create_exact. 0 when hi is outside the range a
/// long-denominator Rational represents exactly (|hi| < 2^-10: not a composed
/// FD weight of the configs).
inline double rational_residue(const Rational& q, double hi) {
  if (hi == 0.0) return q.to_double();
  int e = 0;
  const double f = std::frexp(hi, &e);  // hi = f 2^e, f in [0.5, 1)
  const long m = static_cast<long>(std::ldexp(f, 53));
  const int sh = 53 - e;
  if (sh < 0 || sh > 62) return 0.0;
  return (q - Rational(m, 1L << sh)).to_double();
}

/// A composed stencil uploaded for the device: offsets in the Stencil's map
/// order, coefficients as Rational::to_double() (rational.hpp:32), plus their
/// exact-weight corrections (used only by the refined residual / solver).
class DeviceStencil {
 public:
  explicit DeviceStencil(const Stencil& s) {
    std::vector<int32_t> off;
    std::vector<double> coeff, lo;
    for (const auto& [o, c] : s.entries()) {
      off.insert(off.end(), o.begin(), o.end());
      coeff.push_back(c.to_double());
      lo.push_back(rational_residue(c, coeff.back()));
    }
    sk_stencil* h = nullptr;
    check(sk_stencil_create_exact(s.dim(), static_cast<int>(coeff.size()), off.data(), coeff.data(), lo.data(),
                                  s.h_power(), &h));
    h_.reset(h);
  }
  sk_stencil* get() const { return h_.get(); }

 private:
  struct Del {
    void operator()(sk_stencil* p) const { sk_stencil_destroy(p); }
  };
  std::unique_ptr<sk_stencil, Del> h_;
};

/// Device-resident CSR (upload a reference CsrMatrix or assemble on the GPU).
class DeviceCsr {
 public:
  explicit DeviceCsr(const CsrMatrix& m, int index_bits = 64) {
    sk_csr* h = nullptr;
    check(sk_csr_upload(m.rows, m.cols, m.nnz(), m.row_ptr.data(), m.col_idx.data(), m.values.data(), index_bits, &h));
    h_.reset(h);
  }
  DeviceCsr(const Stencil& s, const GridSpec& g, bool clamped = false, int index_bits = 64) {
    const DeviceStencil ds(s);
    const sk_grid_desc d = grid_desc(g, clamped);
    sk_csr* h = nullptr;
    check(sk_csr_assemble(ds.get(), &d, index_bits, &h, nullptr));
    h_.reset(h);
  }
  /// adopt a handle returned by the C-ABI (e.g. sk_csr_matmul)
  explicit DeviceCsr(sk_csr* adopt) { h_.reset(adopt); }
  sk_csr* get() const { return h_.get(); }
  std::int64_t rows() const {
    int64_t r = 0;
    check(sk_csr_info(get(), &r, nullptr, nullptr, nullptr));
    return r;
  }
  CsrMatrix download() const {
    int64_t rows = 0, cols = 0, nnz = 0;
    int bits = 0;
    check(sk_csr_info(get(), &rows, &cols, &nnz, &bits));
    CsrMatrix m;
    m.rows = rows;
    m.cols = cols;
    m.row_ptr.resize(static_cast<size_t>(rows) + 1);
    m.col_idx.resize(static_cast<size_t>(nnz));
    m.values.resize(static_cast<size_t>(nnz));
    check(sk_csr_download(get(), reinterpret_cast<int64_t*>(m.row_ptr.data()),
                          reinterpret_cast<int64_t*>(m.col_idx.data()), m.values.data()));
    return m;
  }

 private:
  struct Del {
    void operator()(sk_csr* p) const { sk_csr_destroy(p); }
  };
  std::unique_ptr<sk_csr, Del> h_;
};

/// assemble (grid.cpp:62-158) on the GPU: identical row_ptr, col_idx, values.
inline CsrMatrix assemble(const Stencil& s, const GridSpec& g, bool clamped = false) {
  return DeviceCsr(s, g, clamped).download();
}

/// apply (grid.cpp:166-172).
inline std::vector<double> apply(const DeviceCsr& m, std::span<const double> x) {
  int64_t rows = 0, cols = 0;
  check(sk_csr_info(m.get(), &rows, &cols, nullptr, nullptr));
  if (static_cast<int64_t>(x.size()) != cols)
    throw Error(Errc::shape_mismatch, "vector length does not match matrix columns");
  std::vector<double> y(static_cast<size_t>(rows));
  check(sk_csr_matvec_host(m.get(), x.data(), y.data()));
  return y;
}
inline std::vector<double> apply(const CsrMatrix& m, std::span<const double> x) {
  return cuda::apply(DeviceCsr(m), x);
}

namespace kernels {
/// csr_matvec (kernels.cpp:8-17): bit-identical to kernels::serial::csr_matvec.
inline void csr_matvec(const CsrMatrix& m, std::span<const double> x, std::span<double> y) {
  const DeviceCsr d(m);
  check(sk_csr_matvec_host(d.get(), x.data(), y.data()));
}
inline double dot(std::span<const double> a, std::span<const double> b);
inline double nrm2(std::span<const double> a);
inline double sum(std::span<const double> a);
}  // namespace kernels

/// A device field (fp64 vector) for resident loops.
class DeviceField {
 public:
  explicit DeviceField(std::size_t n) : n_(n) {
    void* p = nullptr;
    check(sk_device_alloc(n * sizeof(double), &p));
    p_.reset(static_cast<double*>(p));
  }
  explicit DeviceField(std::span<const double> h) : DeviceField(h.size()) { upload(h); }
  void upload(std::span<const double> h) {
    check(sk_memcpy_h2d(p_.get(), h.data(), n_ * sizeof(double), nullptr));
    check(sk_stream_sync(nullptr));
  }
  void download(std::span<double> h) const { check(sk_memcpy_d2h(h.data(), p_.get(), n_ * sizeof(double), nullptr)); }
  double* data() const { return p_.get(); }
  std::size_t size() const { return n_; }

 private:
  struct Del {
    void operator()(double* p) const { sk_device_free(p); }
  };
  std::size_t n_;
  std::unique_ptr<double, Del> p_;
};

inline double kernels::dot(std::span<const double> a, std::span<const double> b) {
  const DeviceField da(a), db(b);
  double r = 0;
  check(sk_dot(static_cast<int64_t>(a.size()), da.data(), db.data(), &r, nullptr));
  return r;
}
inline double kernels::nrm2(std::span<const double> a) {
  const DeviceField da(a);
  double r = 0;
  check(sk_nrm2(static_cast<int64_t>(a.size()), da.data(), &r, nullptr));
  return r;
}
inline double kernels::sum(std::span<const double> a) {
  const DeviceField da(a);
  double r = 0;
  check(sk_sum(static_cast<int64_t>(a.size()), da.data(), &r, nullptr));
  return r;
}

/// cg_solve (linalg.cpp:15-72): same contract — true residual re-checked,
/// throws Error(no_convergence) on a non-PD Krylov space or a stalled solve.
inline std::vector<double> cg_solve(const DeviceCsr& m, std::span<const double> b, const SolveOptions& opts = {},
                                    sk_solve_report* report = nullptr) {
  int64_t rows = 0, cols = 0;
  check(sk_csr_info(m.get(), &rows, &cols, nullptr, nullptr));
  if (rows != cols) throw Error(Errc::shape_mismatch, "cg_solve needs a square matrix");
  if (static_cast<int64_t>(b.size()) != rows) throw Error(Errc::shape_mismatch, "rhs length does not match matrix");
  const sk_solve_options o{opts.rel_tol, opts.max_iter, opts.deflate_mean ? 1 : 0, 0, 0, 0};
  std::vector<double> x(b.size());
  check(sk_cg_solve_host(m.get(), b.data(), x.data(), &o, report));
  return x;
}
inline std::vector<double> cg_solve(const CsrMatrix& m, std::span<const double> b, const SolveOptions& opts = {}) {
  return cg_solve(DeviceCsr(m), b, opts);
}

/// Matrix-free composed apply: v = S u, equal to apply(assemble(s, g), u).
inline std::vector<double> composed_apply(const Stencil& s, const GridSpec& g, std::span<const double> u,
                                          bool clamped = false) {
  const DeviceStencil ds(s);
  const sk_grid_desc d = grid_desc(g, clamped);
  if (static_cast<int64_t>(u.size()) != g.unknown_count())
    throw Error(Errc::shape_mismatch, "field length does not match the grid");
  std::vector<double> v(u.size());
  check(sk_composed_apply_host(ds.get(), &d, u.data(), v.data()));
  return v;
}

/// Matrix-free CG on the composed operator, then iterative refinement against
/// the EXACT rational operator (double-double residual): the solution of the
/// exact discrete system instead of the fp64-weight matrix (BVP configs 2/5;
/// experiments.cpp:99-143 is the driver it serves). opts.rel_tol is the first
/// solve's recurrence tolerance (the fp64 true-residual floor makes the
/// reference's acceptance unattainable at config sizes).
inline std::vector<double> cg_solve_refined(const Stencil& s, const GridSpec& g, std::span<const double> b,
                                            const SolveOptions& opts = {}, bool clamped = false,
                                            double inner_rel_tol = 1e-6, int max_refinements = 4,
                                            sk_refine_report* report = nullptr) {
  const DeviceStencil ds(s);
  const sk_grid_desc d = grid_desc(g, clamped);
  if (static_cast<int64_t>(b.size()) != g.unknown_count())
    throw Error(Errc::shape_mismatch, "rhs length does not match the grid");
  const sk_solve_options o{opts.rel_tol, opts.max_iter, opts.deflate_mean ? 1 : 0, 0, 1, 0};
  const DeviceField db(b);
  DeviceField dx(b.size());
  check(sk_cg_solve_stencil_refined(ds.get(), &d, db.data(), dx.data(), &o, inner_rel_tol, max_refinements, report,
                                    nullptr));
  std::vector<double> x(b.size());
  dx.download(x);
  check(sk_stream_sync(nullptr));
  return x;
}

inline sk_ch_params ch_params(const CahnHilliardParams& p, int formulation = SK_CH_FACTORED) {
  return sk_ch_params{p.kappa, p.mobility, p.rho_w, p.c_alpha, p.c_beta, formulation};
}

/// Explicit forward-Euler Cahn-Hilliard stepper, fused into one kernel per
/// step: c <- c + dt M (L f'(c) - kappa B c), L = laplacian(d, 2),
/// B = compose(L, L) — the matrices of CahnHilliardStepper (cahn_hilliard.cpp:126-128).
class CahnHilliardExplicit {
 public:
  CahnHilliardExplicit(const GridSpec& grid, const CahnHilliardParams& p, int formulation = SK_CH_FACTORED)
      : grid_(grid), desc_(grid_desc(grid)), params_(ch_params(p, formulation)),
        lap_(laplacian_of(grid)), bilap_(compose(laplacian_of(grid), laplacian_of(grid))) {}
  void step(CahnHilliardState& s, double dt, std::int64_t nsteps = 1) {
    if (static_cast<int64_t>(s.c.size()) != grid_.unknown_count())
      throw Error(Errc::shape_mismatch, "state does not match the stepper grid");
    check(sk_ch_explicit_host(lap_.get(), bilap_.get(), &desc_, &params_, dt, nsteps, s.c.data()));
    s.t += dt * static_cast<double>(nsteps);
  }

 private:
  static Stencil laplacian_of(const GridSpec& g);
  GridSpec grid_;
  sk_grid_desc desc_;
  sk_ch_params params_;
  DeviceStencil lap_, bilap_;
};

}  // namespace stencilkit::cuda

#include "stencilkit/generators.hpp"

inline stencilkit::Stencil stencilkit::cuda::CahnHilliardExplicit::laplacian_of(const GridSpec& g) {
  return laplacian(g.dim, 2);
}

namespace stencilkit::cuda {
/// One rank's z-slab of a periodic 3D explicit Cahn-Hilliard run across GPUs
/// (one process per GPU). `slab` is the local grid (n[2] =
/// this rank's interior planes, the same on every rank, >= 4; n[0], n[1] the
/// full x / y extents). Its two
/// ghosted buffers (n[2] + 4 planes) come from sk_device_alloc, so they are
/// IPC-exportable: handles() gives their 64-byte handles for the caller's
/// communicator (MPI_Allgather, ...), connect() maps the z-neighbours'
/// (connect_self() for a single rank), and step() runs one fused step whose
/// store epilogue also writes the two boundary planes into the neighbours'
/// ghost planes (NVLink peer stores; sk_ch_explicit_slab_peer). After each
/// step the caller puts a barrier between the ranks (the stream is
/// synchronised inside step()).
class SlabStepper {
 public:
  using Handle = std::array<unsigned char, 64>;
  SlabStepper(const GridSpec& slab, const CahnHilliardParams& p)
      : desc_(grid_desc(slab)), params_(ch_params(p, SK_CH_FACTORED)), plane_(slab.n[0] * slab.n[1]),
        nz_(slab.n[2]), lap_(laplacian_of(slab)), bilap_(compose(laplacian_of(slab), laplacian_of(slab))) {
    if (slab.dim != 3 || nz_ < 4) throw Error(Errc::invalid_argument, "a 3D slab of at least 4 planes");
    for (auto& b : buf_) {
      void* q = nullptr;
      const int st = sk_device_alloc(bytes(), &q);
      if (st != SK_OK) {
        for (double* d : buf_) sk_device_free(d);
        check(st);
      }
      b = static_cast<double*>(q);
    }
  }
  ~SlabStepper() {
    for (double* q : opened_) sk_ipc_close_handle(q);
    for (double* b : buf_) sk_device_free(b);
  }
  SlabStepper(const SlabStepper&) = delete;
  SlabStepper& operator=(const SlabStepper&) = delete;

  std::array<Handle, 2> handles() const {
    std::array<Handle, 2> h{};
    for (int i = 0; i < 2; ++i) check(sk_ipc_get_handle(buf_[i], h[i].data()));
    return h;
  }
  void connect(const std::array<Handle, 2>& lower, const std::array<Handle, 2>& upper) {
    for (int i = 0; i < 2; ++i) {
      lower_[i] = open(lower[i]);
      upper_[i] = open(upper[i]);
    }
  }
  void connect_self() {  // a single rank: the ghosts are its own
    for (int i = 0; i < 2; ++i) lower_[i] = upper_[i] = buf_[i];
  }
  /// this rank's interior planes and the two ghost planes on each side (z-major)
  void load(std::span<const double> ghosted) {
    if (static_cast<std::int64_t>(ghosted.size()) != (nz_ + 4) * plane_)
      throw Error(Errc::shape_mismatch, "ghosted slab size");
    check(sk_memcpy_h2d(buf_[cur_], ghosted.data(), bytes(), nullptr));
    check(sk_stream_sync(nullptr));
  }
  void step(double dt) {
    const int nxt = 1 - cur_;
    double* peer_lo = lower_[nxt] + (2 + nz_) * plane_;  // the lower neighbour's upper ghost planes
    double* peer_hi = upper_[nxt];                       // the upper neighbour's lower ghost planes
    check(sk_ch_explicit_slab_peer(lap_.get(), bilap_.get(), &desc_, &params_, dt, buf_[cur_],
                                   buf_[nxt] + 2 * plane_, peer_lo, peer_hi, nullptr));
    check(sk_stream_sync(nullptr));
    cur_ = nxt;
  }
  std::vector<double> interior() const {
    std::vector<double> out(static_cast<size_t>(nz_ * plane_));
    check(sk_memcpy_d2h(out.data(), buf_[cur_] + 2 * plane_, out.size() * sizeof(double), nullptr));
    return out;
  }

 private:
  static Stencil laplacian_of(const GridSpec& g);
  size_t bytes() const { return static_cast<size_t>((nz_ + 4) * plane_) * sizeof(double); }
  double* open(const Handle& h) {
    void* p = nullptr;
    check(sk_ipc_open_handle(h.data(), &p));
    opened_.push_back(static_cast<double*>(p));
    return static_cast<double*>(p);
  }
  sk_grid_desc desc_;
  sk_ch_params params_;
  std::int64_t plane_, nz_;
  DeviceStencil lap_, bilap_;
  double* buf_[2] = {nullptr, nullptr};
  double* lower_[2] = {nullptr, nullptr};
  double* upper_[2] = {nullptr, nullptr};
  std::vector<double*> opened_;
  int cur_ = 0;
};
}  // namespace stencilkit::cuda

inline stencilkit::Stencil stencilkit::cuda::SlabStepper::laplacian_of(const GridSpec& g) {
  return laplacian(g.dim, 2);
}

namespace stencilkit::cuda {
/// free_energy (cahn_hilliard.cpp:77-114) with a device reduction.
inline double free_energy(const CahnHilliardState& s, const CahnHilliardParams& p) {
  const sk_grid_desc d = grid_desc(s.grid);
  const sk_ch_params cp = ch_params(p);
  const DeviceField c(s.c);
  double e = 0;
  check(sk_free_energy(&d, &cp, c.data(), &e, nullptr));
  return e;
}
}  // namespace stencilkit::cuda

namespace stencilkit::cuda {
/// IMEX stepper (cahn_hilliard.hpp:47-68 / cahn_hilliard.cpp:121-189) on the
/// device: same constructor arguments and step(state, dt, order) contract
/// (AB2 history and implicit-matrix cache kept between calls; errors thrown
/// as stencilkit::Error). The field is copied in and out per call; use
/// step_device for a device-resident field.
class CahnHilliardStepper {
 public:
  CahnHilliardStepper(const GridSpec& grid, const CahnHilliardParams& p, SolveOptions solve = {.rel_tol = 1e-12})
      : grid_(grid), desc_(grid_desc(grid)), params_(ch_params(p)) {
    const sk_solve_options o{solve.rel_tol, solve.max_iter, solve.deflate_mean ? 1 : 0, 0, 0, 0};
    sk_ch_imex* h = nullptr;
    check(sk_ch_imex_create(&desc_, &params_, &o, &h));
    h_.reset(h);
  }
  void step(CahnHilliardState& s, double dt, int order) {
    if (static_cast<int64_t>(s.c.size()) != grid_.unknown_count())
      throw Error(Errc::shape_mismatch, "state does not match the stepper grid");
    DeviceField c(s.c);
    check(sk_ch_imex_step(h_.get(), c.data(), dt, order, 1, nullptr, nullptr, nullptr));
    c.download(s.c);
    s.t += dt;
  }
  /// nsteps steps of a device-resident field (caller-owned device pointer)
  void step_device(double* c_dev, double dt, int order, std::int64_t nsteps = 1, void* stream = nullptr) {
    check(sk_ch_imex_step(h_.get(), c_dev, dt, order, nsteps, nullptr, nullptr, stream));
  }

 private:
  struct Del {
    void operator()(sk_ch_imex* h) const { sk_ch_imex_destroy(h); }
  };
  GridSpec grid_;
  sk_grid_desc desc_;
  sk_ch_params params_;
  std::unique_ptr<sk_ch_imex, Del> h_;
};

inline void imex_step(CahnHilliardStepper& stepper, CahnHilliardState& s, double dt, int order) {
  stepper.step(s, dt, order);
}

/// csr_matmul (linalg.cpp:253-283) on the device: b * a, bit-identical values.
inline CsrMatrix csr_matmul(const CsrMatrix& b, const CsrMatrix& a) {
  if (b.cols != a.rows) throw Error(Errc::shape_mismatch, "inner dimensions do not match");
  const DeviceCsr db(b), da(a);
  sk_csr* out = nullptr;
  check(sk_csr_matmul(db.get(), da.get(), &out, nullptr));
  const DeviceCsr prod(out);
  return prod.download();
}

/// power_iteration (linalg.cpp:74-106): the loop runs on the device.
inline double power_iteration(const DeviceCsr& m, double tol, std::uint64_t seed = 20240801,
                              std::int64_t max_iter = 2'000'000) {
  double out = 0;
  check(sk_power_iteration(m.get(), tol, seed, max_iter, &out, nullptr, nullptr));
  return out;
}
inline double power_iteration(const CsrMatrix& m, double tol, std::uint64_t seed = 20240801,
                              std::int64_t max_iter = 2'000'000) {
  return power_iteration(DeviceCsr(m), tol, seed, max_iter);
}

/// periodic_spectrum (linalg.cpp:149-222): modes and sampling on the device.
inline SpectrumReport periodic_spectrum(const Stencil& s, const GridSpec& g, double affine_shift = 0.0,
                                        double affine_scale = 1.0) {
  const DeviceStencil ds(s);
  const sk_grid_desc d = grid_desc(g);
  SpectrumReport rep;
  rep.eigenvalues.resize(static_cast<size_t>(g.unknown_count()));
  check(sk_periodic_spectrum(ds.get(), &d, affine_shift, affine_scale, reinterpret_cast<double*>(rep.eigenvalues.data()),
                             &rep.spectral_radius, &rep.symbol_radius, &rep.condition_estimate));
  return rep;
}

/// ch_init (cahn_hilliard.cpp:20-63), bit-identical (origin 0 grids).
inline CahnHilliardState ch_init(const GridSpec& grid, const CahnHilliardParams& p) {
  CahnHilliardState s;
  s.grid = grid;
  s.c.resize(static_cast<size_t>(grid.unknown_count()));
  const sk_grid_desc d = grid_desc(grid);
  check(sk_ch_init_host(&d, p.c0, p.eps_ic, s.c.data()));
  return s;
}
}  // namespace stencilkit::cuda

#endif  // STENCILKIT_CUDA_HPP
