/* ORACLE TEST INFRASTRUCTURE — never linked into or called by the product.
 *
 * Plain-C restatement of the reference algorithms on the hot path, used by
 * tests/ (as the checker), __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg. Every function cites the reference file:line it follows
 * (paths relative to /root/reference/proj). Pinned against the compiled
 * reference (oracle/_ref/libstencilkit_ref.so) and the committed golden
 * fixtures in tests/golden/ by tests/test_oracle.py.
 */
#ifndef SK_ORACLE_H
#define SK_ORACLE_H

#include <stdint.h>

typedef struct sko_csr {
  int64_t rows, cols, nnz;
  int64_t* row_ptr;
  int64_t* col_idx;
  double* values;
} sko_csr;

/* bc: 0 periodic, 1 simply supported (odd reflection), 2 clamped (even reflection) */
int sko_assemble(int dim, int nent, const int* off, const double* coeff, int h_power, const int64_t* n, double h,
                 const int* bc, sko_csr* out);
int sko_assemble_row(int dim, int nent, const int* off, const double* coeff, int h_power, const int64_t* n, double h,
                     const int* bc, int64_t row, int64_t* cols, double* vals);
void sko_csr_free(sko_csr* m);
void sko_csr_matvec(const sko_csr* m, const double* x, double* y);
double sko_dot(int64_t n, const double* a, const double* b);
double sko_nrm2(int64_t n, const double* a);
double sko_sum(int64_t n, const double* a);
void sko_minmax(int64_t n, const double* a, double* lo, double* hi);
void sko_axpy(int64_t n, double a, const double* x, double* y);
void sko_xpby(int64_t n, const double* x, double b, double* y);
int sko_cg_solve(const sko_csr* m, const double* b, double* x, double rel_tol, int64_t max_iter, int deflate_mean,
                 int64_t* iterations, double* true_rel_residual);
void sko_apply_direct(int dim, int nent, const int* off, const double* coeff, int h_power, const int64_t* n, double h,
                      const int* bc, const double* u, double* v);
int sko_ch_explicit(int dim, int64_t n, double h, double mobility, double kappa, double rho_w, double c_alpha,
                    double c_beta, double dt, int64_t nsteps, double* c);
int sko_identity_plus_scaled(const sko_csr* m, double alpha, sko_csr* out);
int sko_ch_imex_seq(int dim, int64_t n, double h, double mobility, double kappa, double rho_w, double c_alpha,
                    double c_beta, double rel_tol, int nlegs, const double* dts, const int* orders,
                    const int64_t* steps, double* c);
int sko_ch_imex(int dim, int64_t n, double h, double mobility, double kappa, double rho_w, double c_alpha,
                double c_beta, double rel_tol, double dt, int order, int64_t nsteps, double* c);
int sko_csr_matmul(const sko_csr* b, const sko_csr* a, sko_csr* out);
int sko_power_iteration(const sko_csr* m, double tol, uint64_t seed, int64_t max_iter, double* out,
                        int64_t* iterations);
void sko_periodic_eigen(int dim, int nent, const int* off, const double* coeff, int h_power, const int64_t* n,
                        double h, double shift, double scale, double* eig, double* rho_out, double* cond_out);
void sko_ch_init(int dim, int64_t n, double h, double c0, double eps, double* out);
int sko_ch_explicit_dims(int dim, const int64_t* n, double h, double mobility, double kappa, double rho_w,
                         double c_alpha, double c_beta, double dt, int64_t nsteps, double* c);
double sko_free_energy(int dim, int64_t n, double h, double kappa, double rho_w, double c_alpha, double c_beta,
                       const double* c);
void sko_biharmonic_clamped(int dim, int64_t intervals, double* f, double* u_exact);
int sko_fit_loglog(int count, const double* h, const double* err, double* slope, double* coeff, double* resid);
void sko_uniform(uint64_t seed, int64_t count, double lo, double hi, double* out);
int sko_threads(void);

#endif
