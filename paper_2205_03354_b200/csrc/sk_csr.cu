// Device CSR: GPU assembly from a composed stencil (grid.cpp:62-158) and the
// SpMV of kernels.cpp:8-17.
//
// Assembly design. Within a row the reference computes, per stencil entry, a
// wrapped or reflected column and a (possibly sign-flipped) value, sorts the
// (col, val) pairs, merges equal columns by summing in sorted order and drops
// exact zeros. That per-row result depends only on each axis index's
// BOUNDARY CLASS: the first -lo and last hi positions of an axis are their own
// classes, everything between is one "interior" class in which column =
// row-relative offset. So the host runs the reference's row algorithm ONCE per
// class tuple (<= 9^3 = 729 rows for the 73-point stencil, bit-identical
// arithmetic) to get a row template, and closed-form prefix sums over class
// multiplicities give row_ptr of any row without a scan. The device pass is a
// single streaming write of row_ptr / col_idx / values (16 B per nonzero):
// each warp owns 32 consecutive rows, lays their contiguous output span out
// lane-interleaved (coalesced stores), and finds each element's row by a
// 5-step binary search over the warp's 33 row pointers in shared memory.
#include <cuda_runtime.h>

#include <atomic>

#include <algorithm>
#include <cstring>
#include <utility>
#include <vector>

#include "sk_internal.hpp"
#include "sk_sell.cuh"

uint64_t sk_next_csr_uid() {
  static std::atomic<uint64_t> next{1};
  return next.fetch_add(1);
}

sk_csr::~sk_csr() {
  if (row_ptr) cudaFree(row_ptr);
  if (col) cudaFree(col);
  if (val) cudaFree(val);
  if (sell_ptr) cudaFree(sell_ptr);
  if (sell_len) cudaFree(sell_len);
  if (sell_val) cudaFree(sell_val);
  if (sell_col) cudaFree(sell_col);
}

namespace sk {

// ---- SELL-32 build (from the CSR, once per matrix) ---------------------------
__global__ void sell_len_kernel(int64_t rows, const int64_t* __restrict__ rp, int32_t* __restrict__ len,
                                int32_t* __restrict__ width) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int L = i < rows ? int(rp[i + 1] - rp[i]) : 0;
  if (i < rows) len[i] = L;
  const int w = __reduce_max_sync(0xffffffffu, unsigned(L));
  if ((i & 31) == 0) width[i >> 5] = w;
}

template <class IDX>
__global__ void sell_fill_kernel(int64_t rows, int64_t slices, const int64_t* __restrict__ rp,
                                 const IDX* __restrict__ col, const double* __restrict__ val,
                                 const int64_t* __restrict__ sp, IDX* __restrict__ scol, double* __restrict__ sval) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t s = i >> 5;
  if (s >= slices) return;
  const int lane = int(i & 31);
  const int L = i < rows ? int(rp[i + 1] - rp[i]) : 0;
  const int64_t b = i < rows ? rp[i] : 0;
  const int W = int((sp[s + 1] - sp[s]) >> 5);
  int64_t dst = sp[s] + lane;
  for (int k = 0; k < W; ++k, dst += 32) {
    sval[dst] = k < L ? val[b + k] : 0.0;
    scol[dst] = k < L ? col[b + k] : IDX(0);
  }
}

int csr_build_sell(sk_csr* m, cudaStream_t stream) {
  if (m->sell_val || m->rows == 0) return SK_OK;
  const int64_t slices = (m->rows + 31) / 32;
  int32_t* width = nullptr;
  SK_CUDA_TRY(cudaMalloc(&m->sell_len, sizeof(int32_t) * size_t(m->rows)));
  SK_CUDA_TRY(cudaMalloc(&width, sizeof(int32_t) * size_t(slices)));
  const unsigned grid = unsigned(slices * 32 / 256 + 1);
  sell_len_kernel<<<grid, 256, 0, stream>>>(m->rows, m->row_ptr, m->sell_len, width);
  SK_LAUNCH_CHECK("sell_len_kernel");
  std::vector<int32_t> w(static_cast<size_t>(slices));
  std::vector<int64_t> sp(static_cast<size_t>(slices) + 1, 0);
  cudaError_t e = cudaMemcpyAsync(w.data(), width, sizeof(int32_t) * size_t(slices), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  cudaFree(width);
  if (e != cudaSuccess) return cuda_fail(e, "sell widths");
  for (int64_t s = 0; s < slices; ++s) sp[size_t(s) + 1] = sp[size_t(s)] + 32 * int64_t(w[size_t(s)]);
  m->sell_entries = sp.back();
  const size_t ib = size_t(m->index_bits / 8);
  SK_CUDA_TRY(cudaMalloc(&m->sell_ptr, sizeof(int64_t) * sp.size()));
  SK_CUDA_TRY(cudaMalloc(&m->sell_val, sizeof(double) * size_t(std::max<int64_t>(m->sell_entries, 1))));
  SK_CUDA_TRY(cudaMalloc(&m->sell_col, ib * size_t(std::max<int64_t>(m->sell_entries, 1))));
  SK_CUDA_TRY(cudaMemcpyAsync(m->sell_ptr, sp.data(), sizeof(int64_t) * sp.size(), cudaMemcpyHostToDevice, stream));
  if (m->index_bits == 32)
    sell_fill_kernel<int32_t><<<grid, 256, 0, stream>>>(m->rows, slices, m->row_ptr,
                                                        static_cast<const int32_t*>(m->col), m->val, m->sell_ptr,
                                                        static_cast<int32_t*>(m->sell_col), m->sell_val);
  else
    sell_fill_kernel<int64_t><<<grid, 256, 0, stream>>>(m->rows, slices, m->row_ptr,
                                                        static_cast<const int64_t*>(m->col), m->val, m->sell_ptr,
                                                        static_cast<int64_t*>(m->sell_col), m->sell_val);
  SK_LAUNCH_CHECK("sell_fill_kernel");
  SK_CUDA_TRY(cudaStreamSynchronize(stream));
  return SK_OK;
}

template <class IDX>
__global__ void __launch_bounds__(256) sell_spmv_kernel(int64_t rows, const int64_t* __restrict__ sp,
                                                        const int32_t* __restrict__ len, const IDX* __restrict__ col,
                                                        const double* __restrict__ val, const double* __restrict__ x,
                                                        double* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  y[i] = sell_row_dot(i, sp, len, col, val, x);
}

// ---- SpMV ------------------------------------------------------------------
// One thread per row, entries in column order, separate multiply and add:
// y_i = ((v0*x0 + v1*x1) + ...), exactly the reference's Release-build
// rounding (kernels.cpp:13-15; test_kernels.cpp:26-35 pins the order).
template <class IDX>
__global__ void __launch_bounds__(256) spmv_kernel(int64_t rows, const int64_t* __restrict__ rp,
                                                   const IDX* __restrict__ col, const double* __restrict__ val,
                                                   const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int64_t b = __ldg(rp + i), e = __ldg(rp + i + 1);
  double acc = 0.0;
  for (int64_t k = b; k < e; ++k) acc = __dadd_rn(acc, __dmul_rn(__ldg(val + k), __ldg(x + __ldg(col + k))));
  y[i] = acc;
}

int csr_spmv(const sk_csr* m, const double* x, double* y, cudaStream_t stream) {
  if (m->rows == 0) return SK_OK;
  const unsigned grid = unsigned((m->rows + 255) / 256);
  if (int st = csr_build_sell(const_cast<sk_csr*>(m), stream)) return st;
  if (m->sell_val) {
    if (m->index_bits == 32)
      sell_spmv_kernel<int32_t><<<grid, 256, 0, stream>>>(m->rows, m->sell_ptr, m->sell_len,
                                                          static_cast<const int32_t*>(m->sell_col), m->sell_val, x, y);
    else
      sell_spmv_kernel<int64_t><<<grid, 256, 0, stream>>>(m->rows, m->sell_ptr, m->sell_len,
                                                          static_cast<const int64_t*>(m->sell_col), m->sell_val, x, y);
    SK_LAUNCH_CHECK("sell_spmv_kernel");
    return SK_OK;
  }
  if (m->index_bits == 32)
    spmv_kernel<int32_t><<<grid, 256, 0, stream>>>(m->rows, m->row_ptr, static_cast<const int32_t*>(m->col), m->val,
                                                   x, y);
  else
    spmv_kernel<int64_t><<<grid, 256, 0, stream>>>(m->rows, m->row_ptr, static_cast<const int64_t*>(m->col), m->val,
                                                   x, y);
  SK_LAUNCH_CHECK("spmv_kernel");
  return SK_OK;
}

// ---- assembly ----------------------------------------------------------------
namespace {

struct AxisClasses {
  int64_t un = 1;
  int rl = 0, rh = 0;
  bool singleton = true;  // every position its own class (short axes)
  int ncls = 1;
  std::vector<int64_t> start, size;
  std::vector<int> interior;
};

AxisClasses axis_classes(int64_t un, int lo, int hi, bool used) {
  AxisClasses c;
  c.un = un;
  if (!used) {
    c.ncls = 1;
    c.start = {0};
    c.size = {1};
    c.interior = {0};
    return c;
  }
  c.rl = std::max(0, -lo);
  c.rh = std::max(0, hi);
  if (un > int64_t(c.rl) + c.rh) {
    c.singleton = false;
    c.ncls = c.rl + 1 + c.rh;
    for (int k = 0; k < c.rl; ++k) {
      c.start.push_back(k);
      c.size.push_back(1);
      c.interior.push_back(0);
    }
    c.start.push_back(c.rl);
    c.size.push_back(un - c.rl - c.rh);
    c.interior.push_back(1);
    for (int k = 0; k < c.rh; ++k) {
      c.start.push_back(un - c.rh + k);
      c.size.push_back(1);
      c.interior.push_back(0);
    }
  } else {
    c.singleton = true;
    c.ncls = int(un);
    for (int64_t k = 0; k < un; ++k) {
      c.start.push_back(k);
      c.size.push_back(1);
      c.interior.push_back(0);
    }
  }
  return c;
}

// The reference row algorithm (grid.cpp:89-138) at one row, clamped =
// even reflection (value keeps its sign). Returns sorted, merged,
// zero-dropped (col, val).
std::vector<std::pair<int64_t, double>> reference_row(const sk_stencil* s, const GridInfo& g, const double* wval,
                                                      const int64_t* idx) {
  std::vector<std::pair<int64_t, double>> out;
  out.reserve(size_t(s->nent));
  for (int e = 0; e < s->nent; ++e) {
    double val = wval[e];
    int64_t col = 0, stride = 1;
    bool dropped = false;
    for (int a = 0; a < g.dim && !dropped; ++a) {
      const int64_t na = g.n[a];
      int64_t comp;
      if (g.bc[a] == SK_BC_PERIODIC) {
        comp = ((idx[a] + s->off[3 * e + a]) % na + na) % na;
      } else {
        int64_t gi = idx[a] + 1 + s->off[3 * e + a];
        if (gi < 0) {
          gi = -gi;
          if (g.bc[a] == SK_BC_SIMPLY_SUPPORTED) val = -val;
        } else if (gi > na - 1) {
          gi = 2 * (na - 1) - gi;
          if (g.bc[a] == SK_BC_SIMPLY_SUPPORTED) val = -val;
        }
        if (gi == 0 || gi == na - 1) {
          dropped = true;
          break;
        }
        comp = gi - 1;
      }
      col += stride * comp;
      stride *= g.un[a];
    }
    if (!dropped) out.emplace_back(col, val);
  }
  std::sort(out.begin(), out.end());
  size_t w = 0;
  for (size_t r = 0; r < out.size();) {
    const int64_t c = out[r].first;
    double v = 0;
    while (r < out.size() && out[r].first == c) v += out[r++].second;
    if (v != 0.0) out[w++] = {c, v};
  }
  out.resize(w);
  return out;
}

struct AsmTables {
  // per axis
  int64_t un[3];
  int rl[3], rh[3], singleton[3], ncls[3];
  // device buffers
  const int64_t* start;     // [3][16]
  const int* interior;      // [3][16]
  const int64_t* tnnz;      // [ntmpl]
  const int64_t* toff;      // [ntmpl] first slot
  const int64_t* tcol;      // [nslots] column of the slot relative to the row's base column
  const double* tval;       // [nslots]
  const int64_t* cum0;      // [ntmpl]
  const int64_t* t1;        // [nc1*nc2]
  const int64_t* cum1;      // [nc1*nc2]
  const int64_t* t2;        // [nc2]
  const int64_t* cum2;      // [nc2]
  int64_t rows;
};

__device__ __forceinline__ int axis_class(const AsmTables& t, int a, int64_t i) {
  if (t.singleton[a]) return int(i);
  if (i < t.rl[a]) return int(i);
  if (i >= t.un[a] - t.rh[a]) return t.rl[a] + 1 + int(i - (t.un[a] - t.rh[a]));
  return t.rl[a];
}

// One warp per 32 consecutive rows. Row phase (lane = row): the row's
// boundary-class template, its closed-form row pointer, and two per-row
// constants in shared memory: base = the column offset of the row's interior
// axes, sofs = template slot of the row's first entry minus its row pointer.
// Element phase (lane = entry, coalesced over the warp's contiguous entry
// range): find the row by a 5-step search over the 33 row pointers, then
// col = tcol[sofs + e] + base and val = tval[sofs + e] — two L1-resident
// table reads and two streaming stores per nonzero, no integer division.
template <class IDX>
__global__ void __launch_bounds__(256) assemble_kernel(const AsmTables t, int64_t* __restrict__ row_ptr,
                                                       IDX* __restrict__ col_idx, double* __restrict__ values) {
  __shared__ int64_t s_rp[8][33];
  __shared__ int64_t s_base[8][32];
  __shared__ int64_t s_sofs[8][32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t r0 = (int64_t(blockIdx.x) * 8 + warp) * 32;
  if (r0 >= t.rows) return;
  const int64_t r = r0 + lane;
  int64_t rp = 0, nnz = 0, base = 0, sofs = 0;
  if (r < t.rows) {
    const int64_t q = r / t.un[0];
    const int64_t i0 = r - q * t.un[0], i2 = q / t.un[1], i1 = q - i2 * t.un[1];
    const int c0 = axis_class(t, 0, i0), c1 = axis_class(t, 1, i1), c2 = axis_class(t, 2, i2);
    const int c12 = c2 * t.ncls[1] + c1;
    const int tid = c12 * t.ncls[0] + c0;
    nnz = __ldg(t.tnnz + tid);
    rp = __ldg(t.cum0 + tid) + (i0 - __ldg(t.start + 0 * 16 + c0)) * nnz + __ldg(t.cum1 + c12) +
         (i1 - __ldg(t.start + 1 * 16 + c1)) * __ldg(t.t1 + c12) + __ldg(t.cum2 + c2) +
         (i2 - __ldg(t.start + 2 * 16 + c2)) * __ldg(t.t2 + c2);
    base = (__ldg(t.interior + 0 * 16 + c0) ? i0 : 0) +
           t.un[0] * ((__ldg(t.interior + 1 * 16 + c1) ? i1 : 0) + t.un[1] * (__ldg(t.interior + 2 * 16 + c2) ? i2 : 0));
    sofs = __ldg(t.toff + tid) - rp;
    row_ptr[r] = rp;
    if (r == t.rows - 1) row_ptr[t.rows] = rp + nnz;
  }
  // rows past the end get an empty extent at the warp's end pointer
  const int last = t.rows - 1 - r0 < 31 ? int(t.rows - 1 - r0) : 31;
  const int64_t end = __shfl_sync(0xffffffffu, rp + nnz, last);
  s_rp[warp][lane] = r < t.rows ? rp : end;
  s_base[warp][lane] = base;
  s_sofs[warp][lane] = sofs;
  if (lane == 0) s_rp[warp][32] = end;
  __syncwarp();
  const int64_t begin = s_rp[warp][0];
  for (int64_t e = begin + lane; e < end; e += 32) {
    int lo = 0, hi = 32;  // find j: s_rp[j] <= e < s_rp[j+1]
#pragma unroll
    for (int step = 0; step < 5; ++step) {
      const int mid = (lo + hi) >> 1;
      if (s_rp[warp][mid] <= e) lo = mid; else hi = mid;
    }
    const int64_t slot = s_sofs[warp][lo] + e;
    __stcs(col_idx + e, IDX(__ldg(t.tcol + slot) + s_base[warp][lo]));
    __stcs(values + e, __ldg(t.tval + slot));
  }
}

// Host half of the assembly: the reference row algorithm once per boundary
// class tuple (reference_row), the slot tables and the closed-form row
// pointers, packed into one device blob.
struct AsmPlan {
  std::vector<unsigned char> blob;
  size_t o_start, o_int, o_tnnz, o_toff, o_tcol, o_tval, o_cum0, o_t1, o_cum1, o_t2, o_cum2;
  int64_t total = 0;
  AsmTables t{};
};

int asm_plan(const sk_stencil* s, const GridInfo& g, AsmPlan* P) {
  AxisClasses ac[3];
  for (int a = 0; a < 3; ++a) ac[a] = axis_classes(g.un[a], s->lo[a], s->hi[a], a < g.dim);
  for (int a = 0; a < 3; ++a)
    if (ac[a].ncls > 16) return fail(SK_ERR_INVALID_ARGUMENT, "stencil radius too large for GPU assembly (max 7 per side)");
  const int n0 = ac[0].ncls, n1 = ac[1].ncls, n2 = ac[2].ncls;
  const int ntmpl = n0 * n1 * n2;
  // scaled entry values: coeff.to_double() * pow_int(h, h_power) (grid.cpp:77-81)
  const double scale = pow_int(g.h, s->h_power);
  std::vector<double> wval(size_t(s->nent));
  for (int e = 0; e < s->nent; ++e) wval[size_t(e)] = s->coeff[size_t(e)] * scale;

  std::vector<int64_t> tnnz(static_cast<size_t>(ntmpl)), toff(static_cast<size_t>(ntmpl));
  std::vector<int64_t> tcol;
  std::vector<double> tval;
  for (int c2 = 0; c2 < n2; ++c2)
    for (int c1 = 0; c1 < n1; ++c1)
      for (int c0 = 0; c0 < n0; ++c0) {
        const int t = (c2 * n1 + c1) * n0 + c0;
        const int64_t rep[3] = {ac[0].start[size_t(c0)], ac[1].start[size_t(c1)], ac[2].start[size_t(c2)]};
        auto row = reference_row(s, g, wval.data(), rep);
        tnnz[size_t(t)] = int64_t(row.size());
        toff[size_t(t)] = int64_t(tval.size());
        const int cls[3] = {c0, c1, c2};
        for (const auto& [col, v] : row) {
          int64_t comp[3];
          int64_t rem = col;
          for (int a = 0; a < 3; ++a) {
            comp[a] = rem % g.un[a];
            rem /= g.un[a];
            if (ac[a].interior[size_t(cls[a])]) comp[a] -= rep[a];  // relative to the row on interior axes
          }
          tcol.push_back(comp[0] + g.un[0] * (comp[1] + g.un[1] * comp[2]));
          tval.push_back(v);
        }
      }
  // closed-form row pointers
  std::vector<int64_t> cum0(static_cast<size_t>(ntmpl)), t1(static_cast<size_t>(n1 * n2)),
      cum1(static_cast<size_t>(n1 * n2)), t2(static_cast<size_t>(n2)), cum2(static_cast<size_t>(n2));
  for (int c2 = 0; c2 < n2; ++c2)
    for (int c1 = 0; c1 < n1; ++c1) {
      int64_t acc = 0;
      for (int c0 = 0; c0 < n0; ++c0) {
        const int t = (c2 * n1 + c1) * n0 + c0;
        cum0[size_t(t)] = acc;
        acc += ac[0].size[size_t(c0)] * tnnz[size_t(t)];
      }
      t1[size_t(c2 * n1 + c1)] = acc;
    }
  int64_t total = 0;
  for (int c2 = 0; c2 < n2; ++c2) {
    int64_t acc = 0;
    for (int c1 = 0; c1 < n1; ++c1) {
      cum1[size_t(c2 * n1 + c1)] = acc;
      acc += ac[1].size[size_t(c1)] * t1[size_t(c2 * n1 + c1)];
    }
    t2[size_t(c2)] = acc;
    cum2[size_t(c2)] = total;
    total += ac[2].size[size_t(c2)] * acc;
  }
  std::vector<int64_t> start(48, 0);
  std::vector<int> interior(48, 0);
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < ac[a].ncls; ++c) {
      start[size_t(a * 16 + c)] = ac[a].start[size_t(c)];
      interior[size_t(a * 16 + c)] = ac[a].interior[size_t(c)];
    }
  const size_t nslots = std::max<size_t>(tval.size(), 1);
  auto& blob = P->blob;
  blob.clear();
  auto put = [&](const void* p, size_t bytes) {
    size_t off = (blob.size() + 15) & ~size_t(15);
    blob.resize(off + bytes);
    if (bytes) std::memcpy(blob.data() + off, p, bytes);
    return off;
  };
  tcol.resize(nslots, 0);
  tval.resize(nslots, 0.0);
  P->o_start = put(start.data(), start.size() * 8);
  P->o_int = put(interior.data(), interior.size() * 4);
  P->o_tnnz = put(tnnz.data(), tnnz.size() * 8);
  P->o_toff = put(toff.data(), toff.size() * 8);
  P->o_tcol = put(tcol.data(), tcol.size() * 8);
  P->o_tval = put(tval.data(), tval.size() * 8);
  P->o_cum0 = put(cum0.data(), cum0.size() * 8);
  P->o_t1 = put(t1.data(), t1.size() * 8);
  P->o_cum1 = put(cum1.data(), cum1.size() * 8);
  P->o_t2 = put(t2.data(), t2.size() * 8);
  P->o_cum2 = put(cum2.data(), cum2.size() * 8);
  P->total = total;
  AsmTables& t = P->t;
  for (int a = 0; a < 3; ++a) {
    t.un[a] = g.un[a];
    t.rl[a] = ac[a].rl;
    t.rh[a] = ac[a].rh;
    t.singleton[a] = ac[a].singleton ? 1 : 0;
    t.ncls[a] = ac[a].ncls;
  }
  t.rows = g.rows;
  return SK_OK;
}

// Device half: upload the blob, write row_ptr / col / val of m.
int asm_launch(AsmPlan& P, sk_csr* m, cudaStream_t stream) {
  if (m->rows == 0) {
    const int64_t zero = 0;
    SK_CUDA_TRY(cudaMemcpyAsync(m->row_ptr, &zero, sizeof(zero), cudaMemcpyHostToDevice, stream));
    SK_CUDA_TRY(cudaStreamSynchronize(stream));
    return SK_OK;
  }
  unsigned char* d_blob = nullptr;
  SK_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d_blob), P.blob.size(), stream));
  cudaError_t e = cudaMemcpyAsync(d_blob, P.blob.data(), P.blob.size(), cudaMemcpyHostToDevice, stream);
  AsmTables t = P.t;
  t.start = reinterpret_cast<const int64_t*>(d_blob + P.o_start);
  t.interior = reinterpret_cast<const int*>(d_blob + P.o_int);
  t.tnnz = reinterpret_cast<const int64_t*>(d_blob + P.o_tnnz);
  t.toff = reinterpret_cast<const int64_t*>(d_blob + P.o_toff);
  t.tcol = reinterpret_cast<const int64_t*>(d_blob + P.o_tcol);
  t.tval = reinterpret_cast<const double*>(d_blob + P.o_tval);
  t.cum0 = reinterpret_cast<const int64_t*>(d_blob + P.o_cum0);
  t.t1 = reinterpret_cast<const int64_t*>(d_blob + P.o_t1);
  t.cum1 = reinterpret_cast<const int64_t*>(d_blob + P.o_cum1);
  t.t2 = reinterpret_cast<const int64_t*>(d_blob + P.o_t2);
  t.cum2 = reinterpret_cast<const int64_t*>(d_blob + P.o_cum2);
  if (e == cudaSuccess) {
    const unsigned grid = unsigned((m->rows + 255) / 256);
    if (m->index_bits == 32)
      assemble_kernel<int32_t><<<grid, 256, 0, stream>>>(t, m->row_ptr, static_cast<int32_t*>(m->col), m->val);
    else
      assemble_kernel<int64_t><<<grid, 256, 0, stream>>>(t, m->row_ptr, static_cast<int64_t*>(m->col), m->val);
    g_launches++;
    e = cudaGetLastError();
  }
  cudaFreeAsync(d_blob, stream);
  if (e != cudaSuccess) return cuda_fail(e, "assemble_kernel");
  return SK_OK;
}

}  // namespace

// Free the SELL copy (rebuilt lazily by the next SpMV / CG plan).
static void csr_drop_sell(sk_csr* m) {
  if (!m->sell_val) return;
  cudaDeviceSynchronize();  // no SpMV in flight may still read it
  cudaFree(m->sell_ptr);
  cudaFree(m->sell_len);
  cudaFree(m->sell_val);
  cudaFree(m->sell_col);
  m->sell_ptr = nullptr;
  m->sell_len = nullptr;
  m->sell_val = nullptr;
  m->sell_col = nullptr;
  m->sell_entries = 0;
}

int csr_assemble(const sk_stencil* s, const GridInfo& g, int index_bits, sk_csr** out, cudaStream_t stream) {
  if (int st = check_width(s, g)) return st;
  if (index_bits != 32 && index_bits != 64) return fail(SK_ERR_INVALID_ARGUMENT, "index_bits must be 32 or 64");
  if (index_bits == 32 && g.rows > int64_t(INT32_MAX)) return fail(SK_ERR_INVALID_ARGUMENT, "grid too large for int32 columns");
  AsmPlan P;
  if (int st = asm_plan(s, g, &P)) return st;
  auto* m = new sk_csr;
  m->rows = m->cols = g.rows;
  m->nnz = P.total;
  m->index_bits = index_bits;
  cudaError_t e = cudaMalloc(&m->row_ptr, sizeof(int64_t) * size_t(g.rows + 1));
  if (e == cudaSuccess && P.total > 0) e = cudaMalloc(&m->col, size_t(P.total) * (index_bits / 8));
  if (e == cudaSuccess && P.total > 0) e = cudaMalloc(&m->val, sizeof(double) * size_t(P.total));
  if (e != cudaSuccess) {
    delete m;
    return cuda_fail(e, "csr_assemble allocation");
  }
  if (int st = asm_launch(P, m, stream)) {
    delete m;
    return st;
  }
  *out = m;
  return SK_OK;
}

// Re-assemble into an existing matrix of the same shape (no allocation): the
// pattern and values are rewritten; the SELL copy and every cached solver plan
// keyed by the matrix are invalidated (new uid).
int csr_assemble_into(const sk_stencil* s, const GridInfo& g, sk_csr* m, cudaStream_t stream) {
  if (int st = check_width(s, g)) return st;
  AsmPlan P;
  if (int st = asm_plan(s, g, &P)) return st;
  if (m->rows != g.rows || m->cols != g.rows || m->nnz != P.total)
    return fail(SK_ERR_SHAPE_MISMATCH, "matrix shape or nonzero count differs from the assembled operator");
  csr_drop_sell(m);
  m->uid = sk_next_csr_uid();
  return asm_launch(P, m, stream);
}

__global__ void narrow_cols(int64_t n, const int64_t* __restrict__ in, int32_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = int32_t(in[i]);
}
__global__ void widen_cols(int64_t n, const int32_t* __restrict__ in, int64_t* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

}  // namespace sk

using namespace sk;

extern "C" {

int sk_csr_assemble_into(const sk_stencil* s, const sk_grid_desc* gd, sk_csr* m, void* stream) {
  if (!s || !m) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil or matrix");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  return csr_assemble_into(s, g, m, as_stream(stream));
}

int sk_csr_assemble(const sk_stencil* s, const sk_grid_desc* gd, int index_bits, sk_csr** out, void* stream) {
  if (!s || !out) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil or output");
  *out = nullptr;
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  return csr_assemble(s, g, index_bits, out, as_stream(stream));
}

int sk_csr_upload(int64_t rows, int64_t cols, int64_t nnz, const int64_t* row_ptr, const int64_t* col_idx,
                  const double* values, int index_bits, sk_csr** out) {
  if (!out) return fail(SK_ERR_INVALID_ARGUMENT, "null output");
  *out = nullptr;
  if (rows < 0 || cols < 0 || nnz < 0 || !row_ptr || (nnz > 0 && (!col_idx || !values)))
    return fail(SK_ERR_INVALID_ARGUMENT, "bad CSR arrays");
  if (index_bits != 32 && index_bits != 64) return fail(SK_ERR_INVALID_ARGUMENT, "index_bits must be 32 or 64");
  if (row_ptr[0] != 0 || row_ptr[rows] != nnz) return fail(SK_ERR_SHAPE_MISMATCH, "row_ptr does not span nnz");
  if (index_bits == 32 && cols > int64_t(INT32_MAX)) return fail(SK_ERR_INVALID_ARGUMENT, "too many columns for int32");
  auto* m = new sk_csr;
  m->rows = rows;
  m->cols = cols;
  m->nnz = nnz;
  m->index_bits = index_bits;
  cudaError_t e = cudaMalloc(&m->row_ptr, sizeof(int64_t) * size_t(rows + 1));
  if (e == cudaSuccess) e = cudaMemcpy(m->row_ptr, row_ptr, sizeof(int64_t) * size_t(rows + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && nnz > 0) e = cudaMalloc(&m->val, sizeof(double) * size_t(nnz));
  if (e == cudaSuccess && nnz > 0) e = cudaMemcpy(m->val, values, sizeof(double) * size_t(nnz), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && nnz > 0) e = cudaMalloc(&m->col, size_t(nnz) * (index_bits / 8));
  if (e == cudaSuccess && nnz > 0) {
    if (index_bits == 64) {
      e = cudaMemcpy(m->col, col_idx, sizeof(int64_t) * size_t(nnz), cudaMemcpyHostToDevice);
    } else {
      int64_t* tmp = nullptr;
      e = cudaMalloc(&tmp, sizeof(int64_t) * size_t(nnz));
      if (e == cudaSuccess) e = cudaMemcpy(tmp, col_idx, sizeof(int64_t) * size_t(nnz), cudaMemcpyHostToDevice);
      if (e == cudaSuccess) {
        narrow_cols<<<1184, 256>>>(nnz, tmp, static_cast<int32_t*>(m->col));
        e = cudaDeviceSynchronize();
      }
      if (tmp) cudaFree(tmp);
    }
  }
  if (e != cudaSuccess) {
    delete m;
    return cuda_fail(e, "sk_csr_upload");
  }
  *out = m;
  return SK_OK;
}

int sk_csr_info(const sk_csr* m, int64_t* rows, int64_t* cols, int64_t* nnz, int* index_bits) {
  if (!m) return fail(SK_ERR_INVALID_ARGUMENT, "null matrix");
  if (rows) *rows = m->rows;
  if (cols) *cols = m->cols;
  if (nnz) *nnz = m->nnz;
  if (index_bits) *index_bits = m->index_bits;
  return SK_OK;
}

int sk_csr_download(const sk_csr* m, int64_t* row_ptr, int64_t* col_idx, double* values) {
  if (!m) return fail(SK_ERR_INVALID_ARGUMENT, "null matrix");
  if (row_ptr) SK_CUDA_TRY(cudaMemcpy(row_ptr, m->row_ptr, sizeof(int64_t) * size_t(m->rows + 1), cudaMemcpyDeviceToHost));
  if (m->nnz == 0) return SK_OK;
  if (values) SK_CUDA_TRY(cudaMemcpy(values, m->val, sizeof(double) * size_t(m->nnz), cudaMemcpyDeviceToHost));
  if (col_idx) {
    if (m->index_bits == 64) {
      SK_CUDA_TRY(cudaMemcpy(col_idx, m->col, sizeof(int64_t) * size_t(m->nnz), cudaMemcpyDeviceToHost));
    } else {
      int64_t* tmp = nullptr;
      SK_CUDA_TRY(cudaMalloc(&tmp, sizeof(int64_t) * size_t(m->nnz)));
      widen_cols<<<1184, 256>>>(m->nnz, static_cast<const int32_t*>(m->col), tmp);
      cudaError_t e = cudaMemcpy(col_idx, tmp, sizeof(int64_t) * size_t(m->nnz), cudaMemcpyDeviceToHost);
      cudaFree(tmp);
      if (e != cudaSuccess) return cuda_fail(e, "sk_csr_download");
    }
  }
  return SK_OK;
}

int sk_csr_destroy(sk_csr* m) {
  delete m;
  return SK_OK;
}

int sk_csr_matvec(const sk_csr* m, const double* x, double* y, void* stream) {
  if (!m) return fail(SK_ERR_INVALID_ARGUMENT, "null matrix");
  if (m->rows > 0 && (!x || !y)) return fail(SK_ERR_INVALID_ARGUMENT, "null vector");
  return csr_spmv(m, x, y, as_stream(stream));
}

int sk_csr_matvec_host(const sk_csr* m, const double* x_host, double* y_host) {
  if (!m) return fail(SK_ERR_INVALID_ARGUMENT, "null matrix");
  if (m->rows == 0) return SK_OK;
  return host_roundtrip(x_host, size_t(m->cols), y_host, size_t(m->rows),
                        [&](const double* x, double* y, cudaStream_t st) { return csr_spmv(m, x, y, st); });
}

}  // extern "C"
