/* sk_cuda.h — C-ABI of the B200 (sm_100a) stencil-composition hot path.
 *
 * The drop-in boundary for the data-parallel half of the reference library
 * `stencilkit` (/root/reference/proj). Everything is `extern "C"`, plain
 * pointers and sizes; no C++ or torch types cross it. The reference-facing
 * C++ wrapper is include/stencilkit/cuda.hpp (same names and argument meaning
 * as the reference functions it replaces); INTEGRATION.md shows the binding.
 *
 * Conventions (mirroring the reference):
 *  - Every entry point returns an int status: SK_OK (0) or SK_ERR_<Errc>+...,
 *    the reference `stencilkit::Errc` ordinal + 1 (error.hpp:9-28), or one of
 *    the CUDA-side codes >= 100. sk_last_error() returns the thread-local
 *    message of the most recent failure (the reference's Error::what()).
 *  - Device pointers are caller-owned unless created by an *_create call;
 *    opaque handles are freed by the matching *_destroy.
 *  - `stream` may be NULL (legacy default stream) or any cudaStream_t.
 *  - Functions named *_host take HOST buffers and copy in/out inside the call
 *    (the reference's std::span signatures); the others take DEVICE pointers.
 *  - Grids are lexicographic with x fastest (grid.cpp:93-96); on a periodic
 *    axis every point is an unknown, on a simply-supported or clamped axis
 *    only the n-2 interior points are (grid.hpp:27-29).
 *  - All arithmetic is fp64; CSR indices are int64 (reference layout,
 *    grid.hpp:39-46) or int32 (compact, opt-in).
 *  - Weights reach the device as coeff.to_double() * pow_int(h, h_power), the
 *    exact expression of grid.cpp:77-81.
 */
#ifndef SK_CUDA_H
#define SK_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: reference Errc ordinal + 1 (error.hpp:9-28) ---------- */
enum sk_status {
  SK_OK = 0,
  SK_ERR_ZERO_SCALE = 1,
  SK_ERR_DIM_MISMATCH = 2,
  SK_ERR_POWER_MISMATCH = 3,
  SK_ERR_EMPTY_STENCIL = 4,
  SK_ERR_TRUNCATION_TOO_SMALL = 5,
  SK_ERR_NOT_NORMALIZED = 6,
  SK_ERR_ACCURACY_EXCEEDS_TRUNCATION = 7,
  SK_ERR_MIXED_LEADING_ORDER = 8,
  SK_ERR_SINGULAR_SYSTEM = 9,
  SK_ERR_UNSUPPORTED_ACCURACY = 10,
  SK_ERR_STENCIL_WIDER_THAN_GRID = 11,
  SK_ERR_SHAPE_MISMATCH = 12,
  SK_ERR_NO_CONVERGENCE = 13,
  SK_ERR_NOT_DISSIPATIVE = 14,
  SK_ERR_UNSTABLE_FOR_ALL_DT = 15,
  SK_ERR_NON_PERIODIC = 16,
  SK_ERR_ZERO_DENOMINATOR = 17,
  SK_ERR_INVALID_ARGUMENT = 18,
  /* device-side failures (no reference equivalent) */
  SK_ERR_CUDA = 100,
  SK_ERR_OUT_OF_MEMORY = 101,
  SK_ERR_NO_DEVICE = 102
};

/* Boundary kind per axis. periodic and simply_supported are the reference's
 * BoundaryKind (grid.hpp:17); clamped (u = du/dn = 0, ghosts by even
 * reflection) is the extension BASELINE.json configs 2 and 5 require. */
enum sk_bc { SK_BC_PERIODIC = 0, SK_BC_SIMPLY_SUPPORTED = 1, SK_BC_CLAMPED = 2 };

/* GridSpec (grid.hpp:22-34): n = points per axis INCLUDING boundary points. */
typedef struct sk_grid_desc {
  int dim;       /* 1..3 */
  int64_t n[3];  /* points per axis, boundary included; unused axes ignored */
  double h;      /* uniform spacing */
  int bc[3];     /* enum sk_bc per axis */
} sk_grid_desc;

/* CahnHilliardParams (cahn_hilliard.hpp:14-22), chemistry f'(c) =
 * 2 rho_w (c - c_alpha)(c - c_beta)(2c - c_alpha - c_beta) (cahn_hilliard.cpp:70-73). */
typedef struct sk_ch_params {
  double kappa;
  double mobility;
  double rho_w;
  double c_alpha;
  double c_beta;
  /* SK_CH_FACTORED (default): c' = c + dt M L(f'(c) - kappa L c), the
   * composition applied as two 5/7-point passes inside one kernel;
   * SK_CH_COMPOSED: the literal composed 13/25-point B = compose(L, L).
   * Identical in exact arithmetic, both parity-tested against the oracle. */
  int formulation;
} sk_ch_params;

enum sk_ch_formulation { SK_CH_FACTORED = 0, SK_CH_COMPOSED = 1 };

/* SolveOptions (linalg.hpp:13-17) */
typedef struct sk_solve_options {
  double rel_tol;      /* default 1e-10 */
  int64_t max_iter;    /* <= 0: 10 * rows, as linalg.cpp:20 */
  int deflate_mean;    /* nonzero: subtract the mean of x on return */
  int check_every;     /* device iterations between host status polls (0: 64) */
  /* Extensions (0 = reference behaviour):
   * accept_recurrence: stop when the recurrence residual sqrt(r.r) <= tol ||b||
   *   and report the true residual instead of requiring it (SURVEY.md §7.3:
   *   the fp64 true-residual floor of the biharmonic exceeds 1e-10 at config
   *   sizes, so the reference criterion cannot terminate there);
   * use_initial_guess: start from the x passed in (nested iteration) instead
   *   of x0 = 0 (linalg.cpp:22). */
  int accept_recurrence;
  int use_initial_guess;
} sk_solve_options;

typedef struct sk_solve_report {
  int64_t iterations;        /* CG iterations executed (linalg.cpp loop counter) */
  int64_t restarts;          /* true-residual restarts (linalg.cpp:42-46) */
  double true_rel_residual;  /* ||b - M x|| / ||b|| at return */
  double recurrence_rel_residual; /* sqrt(rho) / ||b|| at return */
} sk_solve_report;

typedef struct sk_stencil sk_stencil; /* device-ready composed stencil */
typedef struct sk_csr sk_csr;         /* device-resident CSR matrix */

/* ---- library ------------------------------------------------------------ */
const char* sk_last_error(void);
const char* sk_status_name(int status);
int sk_version(void);
/* Select the device for this thread and create its context. */
int sk_device_init(int device);
/* Device allocation helpers for callers without their own allocator. */
int sk_device_alloc(size_t bytes, void** out);
int sk_device_free(void* p);
int sk_memcpy_h2d(void* dst_dev, const void* src_host, size_t bytes, void* stream);
int sk_memcpy_d2h(void* dst_host, const void* src_dev, size_t bytes, void* stream);
int sk_stream_sync(void* stream);
/* CUDA IPC for buffers from sk_device_alloc (the slab neighbours' buffers in
 * another process, on this or a peer GPU over NVLink): the 64-byte handle of
 * an allocation's base pointer; open maps a handle from another process
 * (peer access enabled lazily); close unmaps it. */
int sk_ipc_get_handle(const void* base_dev, unsigned char handle_out[64]);
int sk_ipc_open_handle(const unsigned char handle[64], void** base_dev_out);
int sk_ipc_close_handle(void* base_dev);
/* A non-blocking stream for callers without their own CUDA runtime. */
int sk_stream_create(void** out);
int sk_stream_destroy(void* stream);
/* Host-side seeded input: std::mt19937_64(seed) + uniform_real_distribution<double>(lo, hi),
 * drawn in order — the generator the reference uses (linalg.cpp:77-78). */
int sk_fill_uniform_host(uint64_t seed, int64_t count, double lo, double hi, double* out);
/* Number of kernel launches this library has issued (monotone counter). */
int64_t sk_launch_count(void);
/* Page-lock a caller host buffer so *_host calls copy at full PCIe/C2C rate. */
int sk_host_register(void* host_ptr, size_t bytes);
int sk_host_unregister(void* host_ptr);
/* CUDA events for device-side timing on the launching stream. */
int sk_event_create(void** ev);
int sk_event_destroy(void* ev);
int sk_event_record(void* ev, void* stream);
int sk_event_elapsed_ms(void* start, void* end, float* ms); /* waits for `end` */
/* Evict L2 by writing a buffer larger than it (timing hygiene). */
int sk_l2_flush(void* stream);

/* ---- execution options ----------------------------------------------------
 * Process-wide switches between alternative device paths that compute the
 * same result (kept for parity tests and A/B timing). They are set only
 * through this call — the library never reads the environment — and every
 * cached graph or plan is rebuilt after a change. Defaults are the measured
 * fastest paths. Unknown options or values:
 * SK_ERR_INVALID_ARGUMENT. */
enum sk_option {
  SK_OPT_PDL = 0,              /* programmatic dependent launch between chained kernels: 1 */
  SK_OPT_CH_PADDED = 1,        /* 3D factored CH runs >= 2 steps through ghost-padded TMA buffers: 1 */
  SK_OPT_CG_DEVICE_LOOP = 2,   /* CG iterations in a device-side while loop (0: unrolled graph chunks): 1 */
  SK_OPT_CG_FUSED = 3,         /* 2D matrix-free CG: two-kernel fused iteration: 1 */
  SK_OPT_CG_COOP = 4,          /* 2D matrix-free CG, one cooperative kernel per iteration: -1 auto, 0, 1 */
  SK_OPT_CG_PQ = 5,            /* 3D radius-2 matrix-free CG: p.q reduced in the apply epilogue: 1 */
  SK_OPT_IMEX_MATRIX_FREE = 6, /* IMEX implicit operator applied matrix-free (0: CSR SpMV): 1 */
  SK_OPT_APPLY73_FACTORED = 7, /* periodic 73-point apply as L4(L4 u) (0: literal 73 weights): 1 */
  SK_OPT_CG_PADDED = 8,        /* radius-4 matrix-free CG off periodic grids: ghost-padded p (16-byte loads): 1 */
  SK_OPT_CH_HOST_PIPELINE = 9, /* sk_ch_explicit_host (3D, pinned host field): upload / steps / download overlapped: 1 */
  SK_OPT_COUNT = 10
};
int sk_set_option(int option, int value);
int sk_get_option(int option, int* value);

/* ---- stencil (host composition result -> device) ------------------------
 * Replaces handing a `stencilkit::Stencil` (stencil.hpp:19-42) to assemble().
 * offsets: nent*dim ints (entry-major), coeff: the exact coefficients as
 * doubles (Rational::to_double, rational.hpp:32), h_power: Stencil::h_power(). */
int sk_stencil_create(int dim, int nent, const int32_t* offsets, const double* coeff, int h_power,
                      sk_stencil** out);
int sk_stencil_destroy(sk_stencil* s);
/* Which kernel the stencil maps to: 0 generic (any offsets), 1 symmetric 2D
 * radius<=2 (5/13-point), 2 symmetric 3D radius<=2 (7/25-point), 3 symmetric
 * 3D radius<=4 (73-point family). */
int sk_stencil_kernel_class(const sk_stencil* s);

/* ---- matrix-free composed apply (no reference symbol; equals
 * apply(assemble(s, g), u), grid.cpp:166-172) ---------------------------- */
int sk_composed_apply(const sk_stencil* s, const sk_grid_desc* g, const double* u_dev, double* v_dev,
                      void* stream);
/* `repeats` applications of s to the same u, outputs alternating between
 * v0_dev and v1_dev (BASELINE config 1); captured in one CUDA graph. */
int sk_composed_apply_repeat(const sk_stencil* s, const sk_grid_desc* g, const double* u_dev,
                             double* v0_dev, double* v1_dev, int repeats, void* stream);
int sk_composed_apply_host(const sk_stencil* s, const sk_grid_desc* g, const double* u_host,
                           double* v_host);

/* ---- fused explicit Cahn-Hilliard step ----------------------------------
 *   c <- c + dt * M * ( L f'(c) - kappa * B c ),  B = compose(L, L)
 * L = laplacian(dim, 2) (5/7-point), B its composition (13/25-point), as the
 * reference stepper builds them (cahn_hilliard.cpp:126-128). Periodic grids
 * only (cahn_hilliard.cpp:12-16). `lap` and `bilap` are the host-composed
 * stencils. Ping-pong between c_dev and scratch_dev; *result_is_scratch tells
 * which holds the final field. */
int sk_ch_explicit(const sk_stencil* lap, const sk_stencil* bilap, const sk_grid_desc* g,
                   const sk_ch_params* p, double dt, int64_t nsteps, double* c_dev,
                   double* scratch_dev, int* result_is_scratch, void* stream);
/* The same from host memory: c_host in, K steps, result back in c_host.
 * With a pinned (or sk_host_register'ed) 3D field of nz >= 4K + 8 planes the
 * upload, the steps and the download overlap (plane chunks; each step's
 * front advances as the planes it depends on arrive); the result is
 * bit-identical to the serial H2D -> steps -> D2H. */
int sk_ch_explicit_host(const sk_stencil* lap, const sk_stencil* bilap, const sk_grid_desc* g,
                        const sk_ch_params* p, double dt, int64_t nsteps, double* c_host);
/* One fused explicit step on a z-slab of a periodic 3D field (multi-GPU slab
 * decomposition): g describes the slab (n[2] = its interior
 * planes; x and y periodic); in_ghosted holds n[2] + 4 planes, two ghost
 * planes below and above the interior (the neighbours' planes, exchanged by
 * the caller); out receives the n[2] interior planes of c'. */
int sk_ch_explicit_slab(const sk_stencil* lap, const sk_stencil* bilap, const sk_grid_desc* g,
                        const sk_ch_params* p, double dt, const double* in_ghosted_dev, double* out_dev,
                        void* stream);
/* The same step with the halo exchange fused into its store epilogue: every
 * point of output planes 0, 1 is also stored at peer_lo (the two upper ghost
 * planes of the z-neighbour below, in ITS output buffer), every point of
 * planes n[2]-2, n[2]-1 at peer_hi (the two lower ghost planes of the
 * neighbour above): device pointers into this GPU's or a peer GPU's memory
 * (sk_ipc_open_handle; NVLink stores), either may be NULL. After the step
 * (stream-ordered) and a barrier with the neighbours, every rank's output
 * buffer is a complete ghosted input for the next step. Factored
 * formulation only; n[2] >= 4. */
int sk_ch_explicit_slab_peer(const sk_stencil* lap, const sk_stencil* bilap, const sk_grid_desc* g,
                             const sk_ch_params* p, double dt, const double* in_ghosted_dev, double* out_dev,
                             double* peer_lo_dev, double* peer_hi_dev, void* stream);
/* free_energy (cahn_hilliard.cpp:77-114): h^d sum f_chem + kappa/2 |central grad|^2 */
int sk_free_energy(const sk_grid_desc* g, const sk_ch_params* p, const double* c_dev,
                   double* energy_host, void* stream);

/* ---- IMEX Cahn-Hilliard stepper (cahn_hilliard.cpp:121-189) -------------
 * The reference's own CH path on the device: L = laplacian(d,2) and
 * B = compose(L,L) assembled on the GPU; per step chem = L f'(c), then
 * (I + dt M kappa B) c' = c + dt M chem (order 1) or the Crank-Nicolson /
 * Adams-Bashforth-2 system (order 2, bootstrapped by an order-1 step and
 * re-bootstrapped when dt changes), solved by sk_cg_solve from x0 = 0.
 * opts NULL: the stepper's default SolveOptions{rel_tol = 1e-12}. The stepper
 * keeps the AB2 history (prev_explicit_) and the cached implicit matrix
 * (ensure_implicit_matrix) between calls, like CahnHilliardStepper. */
typedef struct sk_ch_imex sk_ch_imex;
int sk_ch_imex_create(const sk_grid_desc* g, const sk_ch_params* p, const sk_solve_options* opts,
                      sk_ch_imex** out);
int sk_ch_imex_destroy(sk_ch_imex* s);
int sk_ch_imex_reset_history(sk_ch_imex* s);
/* nsteps IMEX steps of c_dev in place; last: report of the last CG solve,
 * cg_iterations: total CG iterations (both may be NULL). */
int sk_ch_imex_step(sk_ch_imex* s, double* c_dev, double dt, int order, int64_t nsteps,
                    sk_solve_report* last, int64_t* cg_iterations, void* stream);
/* which: 0 L, 1 B, 2 the current implicit matrix identity_plus_scaled(B, factor) */
int sk_ch_imex_matrix(const sk_ch_imex* s, int which, const sk_csr** out);
/* ch_init (cahn_hilliard.cpp:20-63) on the host, bit-identical (origin 0). */
int sk_ch_init_host(const sk_grid_desc* g, double c0, double eps_ic, double* c_host);

/* ---- spectral tools (linalg.cpp:74-106, 149-222) -------------------------
 * power_iteration: |Rayleigh quotient| of M from a seeded mt19937_64 start,
 * geometric-tail stopping rule; SK_ERR_NO_CONVERGENCE past max_iter.
 * periodic_spectrum: eigenvalues (affine_shift + affine_scale * h^s * symbol)
 * of every Fourier mode on an all-periodic grid (eigen_host: 2 doubles per
 * mode, x-fastest mode order, may be NULL), the spectral radius, the
 * continuous-torus symbol radius and max|ev| / min nonzero |ev|. */
int sk_power_iteration(const sk_csr* m, double tol, uint64_t seed, int64_t max_iter, double* out,
                       int64_t* iterations, void* stream);
int sk_periodic_spectrum(const sk_stencil* s, const sk_grid_desc* g, double affine_shift, double affine_scale,
                         double* eigen_host, double* spectral_radius, double* symbol_radius,
                         double* condition_estimate);

/* ---- CSR assembly (grid.cpp:62-158) and SpMV (kernels.cpp:8-17) --------- */
int sk_csr_assemble(const sk_stencil* s, const sk_grid_desc* g, int index_bits, sk_csr** out,
                    void* stream);
/* Re-assemble into an existing matrix of the same rows / nonzero count (no
 * allocation; e.g. new weights after an h change): SK_ERR_SHAPE_MISMATCH
 * otherwise. Cached solver plans of the matrix are invalidated. */
int sk_csr_assemble_into(const sk_stencil* s, const sk_grid_desc* g, sk_csr* m, void* stream);
int sk_csr_upload(int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr,
                  const int64_t* col_idx, const double* values, int index_bits, sk_csr** out);
int sk_csr_info(const sk_csr* m, int64_t* rows, int64_t* cols, int64_t* nnz, int* index_bits);
int sk_csr_download(const sk_csr* m, int64_t* row_ptr, int64_t* col_idx, double* values);
int sk_csr_destroy(sk_csr* m);
/* out = b * a (csr_matmul, linalg.cpp:253-283): per-row products summed per
 * column in the reference's order (bit-identical values), exact zeros
 * dropped, columns sorted. Device limit: 1024 products per row. */
int sk_csr_matmul(const sk_csr* b, const sk_csr* a, sk_csr** out, void* stream);
/* y = M x, per-row sequential accumulation in column order (bit-identical to
 * the reference's serial csr_matvec as built by its CMake Release flags). */
int sk_csr_matvec(const sk_csr* m, const double* x_dev, double* y_dev, void* stream);
int sk_csr_matvec_host(const sk_csr* m, const double* x_host, double* y_host);

/* ---- BLAS-1 (kernels.cpp:19-60); deterministic two-level reductions ----- */
int sk_dot(int64_t n, const double* a_dev, const double* b_dev, double* out_host, void* stream);
int sk_nrm2(int64_t n, const double* a_dev, double* out_host, void* stream);
int sk_sum(int64_t n, const double* a_dev, double* out_host, void* stream);
int sk_minmax(int64_t n, const double* a_dev, double* lo_host, double* hi_host, void* stream);
int sk_axpy(int64_t n, double a, const double* x_dev, double* y_dev, void* stream);  /* y += a x */
int sk_xpby(int64_t n, const double* x_dev, double b, double* y_dev, void* stream);  /* y = x + b y */

/* ---- conjugate gradients (linalg.cpp:15-72) ------------------------------
 * x0 = 0; accepts only when the TRUE residual ||b - M x|| <= rel_tol ||b||,
 * restarting from x on recurrence drift; SK_ERR_NO_CONVERGENCE when M is not
 * positive definite on the Krylov space or the budget runs out. x_dev receives
 * the last iterate even on failure; report may be NULL. */
int sk_cg_solve(const sk_csr* m, const double* b_dev, double* x_dev, const sk_solve_options* opts,
                sk_solve_report* report, void* stream);
int sk_cg_solve_host(const sk_csr* m, const double* b_host, double* x_host,
                     const sk_solve_options* opts, sk_solve_report* report);
/* Matrix-free CG (no reference symbol): the operator is the composed stencil
 * on the grid (any boundary kind), i.e. assemble(s, g) without the matrix;
 * same control flow and contract as sk_cg_solve. Results agree with the CSR
 * solve to the solver tolerance (products summed in orbit order). */
int sk_cg_solve_stencil(const sk_stencil* s, const sk_grid_desc* g, const double* b_dev, double* x_dev,
                        const sk_solve_options* opts, sk_solve_report* report, void* stream);

/* ---- exact-operator refinement (configs 2 / 5; no reference symbol) ------
 * The doubles of non-dyadic composed weights do not sum to zero (73-point:
 * -2.6e-15), a zeroth-order perturbation of size |sum| h^s that pollutes the
 * manufactured solution at fine grids. sk_stencil_create_exact
 * also takes coeff_lo[e] = coefficient_e - coeff[e] (the rounding error of
 * Rational::to_double, rational.hpp:32, as a double), so coeff + coeff_lo is
 * the exact rational to ~2^-106; every other entry point still uses coeff
 * (the reference's fp64 matrix). The grid scale is pow_int(h, h_power) as
 * the reference computes it (exact for the configs' dyadic h).
 * sk_residual_refined: r = b - A x with the
 * exact weights, evaluated in double-double (error-free products and
 * compensated sums), rounded to fp64. sk_cg_solve_stencil_refined: the
 * matrix-free CG (opts, stopping on the recurrence residual) followed by up
 * to max_refinements steps
 * x += CG(A_fl, r_refined) with inner tolerance inner_rel_tol (recurrence
 * criterion), stopping when ||d|| <= 1e-15 ||x||. */
typedef struct sk_refine_report {
  int64_t iterations;               /* CG iterations, all solves */
  int refinements;                  /* correction steps taken */
  double initial_true_rel_residual; /* fp64-operator true residual of the first CG solve */
  double refined_rel_residual;      /* ||b - A_exact x|| / ||b|| (double-double) at return */
  double last_correction_rel;       /* ||d|| / ||x|| of the last correction */
} sk_refine_report;
int sk_stencil_create_exact(int dim, int nent, const int32_t* offsets, const double* coeff,
                            const double* coeff_lo, int h_power, sk_stencil** out);
int sk_residual_refined(const sk_stencil* s, const sk_grid_desc* g, const double* b_dev,
                        const double* x_dev, double* r_dev, void* stream);
int sk_cg_solve_stencil_refined(const sk_stencil* s, const sk_grid_desc* g, const double* b_dev,
                                double* x_dev, const sk_solve_options* opts, double inner_rel_tol,
                                int max_refinements, sk_refine_report* report, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SK_CUDA_H */
