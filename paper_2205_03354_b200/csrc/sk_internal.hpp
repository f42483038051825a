// Host-side internal types shared by the library translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <vector>

#include "sk_common.cuh"

// Device-ready stencil: the host composition result in canonical order
// (std::map<Offset, Rational> order, stencil.hpp:44-57), plus its
// classification onto one of the specialised symmetric kernels.
uint64_t sk_next_csr_uid();  // unique object ids (never reused) keying cached solver plans

struct sk_stencil {
  uint64_t uid = sk_next_csr_uid();
  int dim = 0;
  int nent = 0;
  int h_power = 0;
  std::vector<int> off;       // nent * 3, lexicographic entry order, unused axes 0
  std::vector<double> coeff;  // Rational::to_double of each entry
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};  // Stencil::support per axis
  int kclass = 0;             // 0 generic, 1 sym2d r<=2, 2 sym3d r<=2, 3 sym3d r<=4
  double orbit_coeff[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int* d_off = nullptr;       // device copy for the generic kernel / assembly
  double* d_coeff = nullptr;
  // exact-weight correction (sk_stencil_create_exact): coeff + coeff_lo is the
  // exact rational coefficient to ~2^-106 relative; used only by the refined
  // residual (sk_residual_refined). Empty: corrections are zero.
  std::vector<double> coeff_lo;
  double* d_coeff_lo = nullptr;
  // cached CUDA graph of sk_composed_apply_repeat: the captured kernels bake
  // in the buffers, the grid (extents, boundary kinds, h -> weights) and the
  // option epoch, all part of the key; rep_mu serialises concurrent callers
  struct RepKey {
    const void* ptr[3] = {nullptr, nullptr, nullptr};
    int repeats = 0, dim = 0;
    int64_t n[3] = {0, 0, 0};
    int bc[3] = {0, 0, 0};
    double h = 0;
    uint64_t epoch = 0;
    bool operator==(const RepKey& o) const {
      return ptr[0] == o.ptr[0] && ptr[1] == o.ptr[1] && ptr[2] == o.ptr[2] && repeats == o.repeats &&
             dim == o.dim && n[0] == o.n[0] && n[1] == o.n[1] && n[2] == o.n[2] && bc[0] == o.bc[0] &&
             bc[1] == o.bc[1] && bc[2] == o.bc[2] && h == o.h && epoch == o.epoch;
    }
  };
  std::mutex rep_mu;
  cudaGraphExec_t rep_exec = nullptr;
  RepKey rep_key;
  ~sk_stencil();
};

// Device-resident CSR (grid.hpp:39-46 layout; int32 columns opt-in).
struct sk_csr {
  uint64_t uid = sk_next_csr_uid();  // never reused: keys cached solver plans
  int64_t rows = 0, cols = 0, nnz = 0;
  int index_bits = 64;
  int64_t* row_ptr = nullptr;
  void* col = nullptr;
  double* val = nullptr;
  // SELL-32 copy used by SpMV / CG (built lazily): slices of 32 rows stored
  // column-major, so "thread = row, entry k" loads are coalesced while each
  // row is still summed sequentially in column order (bit-identical to CSR).
  int64_t* sell_ptr = nullptr;  // [slices + 1] first entry of each slice
  int32_t* sell_len = nullptr;  // [rows] row lengths
  double* sell_val = nullptr;
  void* sell_col = nullptr;     // int32 or int64 (index_bits)
  int64_t sell_entries = 0;
  ~sk_csr();
};

namespace sk {

int num_sms();

// Build the SELL-32 copy of a CSR (idempotent; not capturable: call before graph capture).
int csr_build_sell(sk_csr* m, cudaStream_t stream);

// Width checks of assemble (grid.cpp:66-75), shared by apply and assembly.
int check_width(const sk_stencil* s, const GridInfo& g);

// Launch one matrix-free application on `stream` (device pointers).
// input_stable: u is not written by the kernel launched just before, so the
// 2D kernel may load it before its programmatic-launch wait.
struct CgState;
constexpr int kApplyPqUnsupported = -1;
bool apply_pq_supported(const sk_stencil* s, const GridInfo& g);
int launch_apply_pq(const sk_stencil* s, const GridInfo& g, const double* p, double* q, CgState* st,
                    double* partials, cudaStream_t stream);
int launch_apply(const sk_stencil* s, const GridInfo& g, const double* u, double* v, cudaStream_t stream,
                 bool input_stable = false);
// the same apply from a ghost-padded field (radius-4 3D stencils; sk_cg.cu's
// PadLayout): kApplyPqUnsupported when not applicable
bool apply_padded_supported(const sk_stencil* s, const GridInfo& g);
// st != nullptr: q = A p fused with p.q -> alpha (kApplyPqUnsupported when the
// kernel for this stencil has no fused form)
int launch_apply_padded(const sk_stencil* s, const GridInfo& g, const double* u_origin, int64_t pitch,
                        int64_t plane, double* v, cudaStream_t stream, CgState* st = nullptr,
                        double* partials = nullptr);

// Fused matrix-free CG half-iteration on a 2D class-1 stencil (Mode::CgApply):
// q = A p' with p' = r + beta p formed on the load, alpha from p'.q.
// cg_apply_2d_ctas: CTA count (the partials it needs), 0 when the
// stencil/grid is not eligible.
struct CgState;
int cg_apply_2d_ctas(const sk_stencil* s, const GridInfo& g);
int launch_cg_apply_2d(const sk_stencil* s, const GridInfo& g, const double* p, const double* r, double* q,
                       CgState* st, double* partials, cudaStream_t stream);
struct Apply2DArgs;
// the operator part of the fused apply's arguments (weights, extents, boundary kinds, p, r, q)
void cg_apply_2d_args(const sk_stencil* s, const GridInfo& g, const double* p, const double* r, double* q,
                      Apply2DArgs* out);

// ---- conjugate gradients (sk_cg.cu) ----
// The operator q = A p: an assembled CSR (SELL SpMV, bit-identical to the
// reference's csr_matvec) or a matrix-free stencil on a periodic grid.
struct CgOperator {
  const sk_csr* m = nullptr;
  const sk_stencil* s = nullptr;
  GridInfo g{};
  int64_t n = 0;
};
// Workspace + captured iteration graph, reusable across solves.
struct CgPlan;
int cg_plan_create(const CgOperator& op, int check_every, cudaStream_t stream, CgPlan** out);
void cg_plan_destroy(CgPlan* p);
int cg_plan_solve(CgPlan* p, const double* b, double* x, const sk_solve_options* o, sk_solve_report* rep,
                  cudaStream_t stream);
int cg_solve(const sk_csr* m, const double* b, double* x, const sk_solve_options* o, sk_solve_report* rep,
             cudaStream_t stream);

// Internal per-thread non-blocking stream: graph capture when the caller
// passes the legacy stream, and the stream every *_host entry point runs on.
cudaStream_t capture_stream();
inline cudaStream_t host_stream() { return capture_stream(); }

// Stream-ordered scratch for *_host calls (pool allocator: no cudaMalloc
// synchronisation inside a timed end-to-end call).
struct AsyncBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  explicit AsyncBuf(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes ? bytes : 16, s); }
  double* d() const { return static_cast<double*>(p); }
  ~AsyncBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

// Copy host -> device, run `body` on the host stream, copy device -> host, sync.
template <class Body>
int host_roundtrip(const double* in_host, size_t in_count, double* out_host, size_t out_count, Body body) {
  cudaStream_t s = host_stream();
  AsyncBuf in(s), out(s);
  SK_CUDA_TRY(in.alloc(in_count * sizeof(double)));
  SK_CUDA_TRY(out.alloc(out_count * sizeof(double)));
  if (in_count) SK_CUDA_TRY(cudaMemcpyAsync(in.p, in_host, in_count * sizeof(double), cudaMemcpyHostToDevice, s));
  if (int st = body(in.d(), out.d(), s)) return st;
  if (out_count) SK_CUDA_TRY(cudaMemcpyAsync(out_host, out.p, out_count * sizeof(double), cudaMemcpyDeviceToHost, s));
  SK_CUDA_TRY(cudaStreamSynchronize(s));
  return SK_OK;
}

}  // namespace sk
