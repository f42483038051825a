// Fused explicit Cahn-Hilliard stepping and the free-energy reduction.
//
// Reference pieces restated (no explicit stepper exists in the reference;
// SURVEY.md Appendix A): the stepper's matrices L = assemble(laplacian(d,2))
// and B = assemble(compose(L,L)) (cahn_hilliard.cpp:126-128) and its explicit
// chemistry term M L f'(c) (:146-152). One step is
//     c <- c + dt M (L f'(c) - kappa B c)
// computed in ONE pass per point (kernels in sk_stencil_kernels.cuh): the
// tile of c lands in shared memory, f'(c) is evaluated on the fly for the
// 5/7-point Laplacian, the 13/25-point composed B is summed by orbits, and
// the update is written to the ping-pong buffer. 16 B of HBM traffic per
// point per step (read c, write c').
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "sk_internal.hpp"
#include "sk_stencil_kernels.cuh"
#include "sk_stream3d.cuh"
#include "sk_chf3d.cuh"

namespace sk {

template <Mode M>
int launch_2d(const Apply2DArgs& a, cudaStream_t stream);
template <Mode M, class C, bool PQ = false>
int launch_3d(Args3D a, cudaStream_t stream);
using C3R2 = Cfg3CH;

namespace {

constexpr int kThreads = 256;

// ---- generic fallback pieces (any L/B the fast path does not cover) ------
__global__ void chem_kernel(int64_t n, const double* __restrict__ c, double* __restrict__ w, ChemParams p) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    w[i] = chem_prime(c[i], p);
}

// c' = c + dt M (a - kappa b)   (evaluation order of the restated step)
__global__ void ch_update_kernel(int64_t n, const double* __restrict__ c, const double* __restrict__ la,
                                 const double* __restrict__ lb, double dtm, double kappa, double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = __dadd_rn(c[i], __dmul_rn(dtm, __dsub_rn(la[i], __dmul_rn(kappa, lb[i]))));
}

// ---- free energy (cahn_hilliard.cpp:77-107), reference evaluation order --
__global__ void __launch_bounds__(kThreads)
    energy_kernel(const double* __restrict__ c, int dim, int64_t nx, int64_t ny, int64_t nz, double inv_2h,
                  double kappa, double rho_w, double c_alpha, double c_beta, double* partials, unsigned* counter,
                  double* out) {
  __shared__ double sh[32];
  const int64_t count = nx * ny * nz;
  const int64_t stride[3] = {1, nx, nx * ny};
  const int64_t nn[3] = {nx, ny, nz};
  double acc = 0.0;
  for (int64_t idx = int64_t(blockIdx.x) * kThreads + threadIdx.x; idx < count;
       idx += int64_t(gridDim.x) * kThreads) {
    const double ci = c[idx];
    const double a = __dsub_rn(ci, c_alpha), b = __dsub_rn(ci, c_beta);
    double cell = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(rho_w, a), a), b), b);  // f_chem, :65-68
    int64_t rem = idx;
    for (int ax = 0; ax < dim; ++ax) {
      const int64_t na = nn[ax];
      const int64_t ia = rem % na;
      rem /= na;
      const int64_t up = idx + stride[ax] * ((ia + 1 == na) ? 1 - na : 1);
      const int64_t dn = idx - stride[ax] * ((ia == 0) ? 1 - na : 1);
      const double grad = __dmul_rn(__dsub_rn(c[up], c[dn]), inv_2h);
      cell = __dadd_rn(cell, __dmul_rn(__dmul_rn(__dmul_rn(0.5, kappa), grad), grad));
    }
    acc += cell;
  }
  acc = block_sum<kThreads>(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  if (last_block(counter)) {
    const double t = reduce_partials<kThreads>(partials, gridDim.x, sh);
    if (threadIdx.x == 0) *out = t;
  }
}

bool is_lap_shape(const sk_stencil* s, int dim) {
  // 5/7-point: only the centre and axis-1 orbits
  const int want = dim == 2 ? 1 : 2;
  return s->kclass == want && s->orbit_coeff[2] == 0.0 && s->orbit_coeff[3] == 0.0;
}

bool is_bilap_shape(const sk_stencil* s, int dim) { return s->kclass == (dim == 2 ? 1 : 2); }

constexpr int kGraphSteps = 100;  // steps per full chunk graph (even: buffers return to start)

}  // namespace

// Field layouts of one 3D factored step (sk_chf3d.cuh LD / OUT): inside a
// captured chunk the field lives in ghost-padded buffers, so every step but
// the first loads one TMA box per plane without wrap logic.
enum ChfIo { kIoPlain = 0, kIoFirst = 1, kIoMid = 2, kIoLast = 3 };  // in/out: plain/plain, plain/pad, pad/pad, pad/plain

// whole tiles of the TMA kernel, even padded rows (16 B strides), int32 in-plane offsets.
// Measured (tools/kbench.py ch3d --n N, 100-step chunks, padded vs plain
// cp.async path): 256^3 57.2 vs 68.3 us, 384^3 184 vs 211 us, 512^3 444 vs
// 505 us. (Before the rotated-column schedule and 64x16 tiles the padded path
// lost from 384^3 up and was limited to ~21M points.)
static bool chf3d_padded_ok(const GridInfo& g) {
  using CT = CfgChf3T;
  // whole tiles of both the TMA kernel and the first step's cp.async kernel (CfgChf3: OUT 1)
  return g.dim == 3 && g.n[0] % CT::TX == 0 && g.n[1] % CT::TY == 0 && g.n[1] % CfgChf3::TY == 0 &&
         (g.n[0] + 2 * kPadL) * (g.n[1] + 2 * kPadT) < (int64_t(1) << 31);
}

static int make_tmap_padded(CUtensorMap* tm, const double* base, const GridInfo& g,
                            cuuint32_t box_x = cuuint32_t(ChfSmem<CfgChf3T, 1>::P),
                            cuuint32_t box_y = cuuint32_t(CfgChf3T::ROWS / kTmaSplit)) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t px = cuuint64_t(g.n[0] + 2 * kPadL), py = cuuint64_t(g.n[1] + 2 * kPadT);
  const cuuint64_t dims[3] = {px, py, cuuint64_t(g.n[2])};
  const cuuint64_t strides[2] = {px * 8, px * py * 8};
  const cuuint32_t box[3] = {box_x, box_y, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_64B,  // measured +1.6% at 256^3, +10% at 1024^3
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return SK_OK;
}

template <class C, int V, int LD, int OUT, bool FB>
static int launch_chf3d_as(const Args3D& a, const CUtensorMap& tm, int64_t grid, cudaStream_t stream) {
  using SM = ChfSmem<C, LD, FB>;
  auto kern = chf3d_kernel<C, V, LD, OUT, FB>;
  static const cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
  if (attr != cudaSuccess) return cuda_fail(attr, "chf3d smem attribute");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = SM::BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap launch with the previous step
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = option(SK_OPT_PDL) ? 1 : 0;
  SK_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a, tm));
  SK_LAUNCH_CHECK("chf3d_kernel");
  return SK_OK;
}

template <class C, int V, int LD, int OUT>
static int launch_chf3d(Args3D a, const CUtensorMap& tm, cudaStream_t stream) {
  // rotated, phase-aligned columns (seg_of); not for slabs (z_ghosted)
  a.zrot = a.z_ghosted ? 0 : 1;
  // balanced static schedule (measured faster than lockstep z-chunks at 256^3)
  const int64_t grid = persistent_grid<C>(a, num_sms(), /*lockstep=*/false);
  if (grid == 0) return fail(SK_ERR_INVALID_ARGUMENT, "grid too large for the 3D streaming kernels");
  // cp.async loads: the 16-byte or the 8-byte fallback instantiation (after
  // persistent_grid, which may clear bulk_ok); TMA loads need neither
  if constexpr (LD == 0) {
    if (!a.bulk_ok) return launch_chf3d_as<C, V, LD, OUT, true>(a, tm, grid, stream);
  }
  return launch_chf3d_as<C, V, LD, OUT, false>(a, tm, grid, stream);
}

// One fused step on the fast path (in -> out).
static int ch_step_fast(const sk_stencil* lap, const sk_stencil* bilap, const GridInfo& g, const sk_ch_params* p,
                        double dt, const double* in, double* out, cudaStream_t stream, bool bulk_ok_ptrs,
                        int io = kIoPlain, bool z_ghosted = false, int ghost = 2, double* peer_lo = nullptr,
                        double* peer_hi = nullptr) {
  const double dtm = dt * p->mobility;
  const double fac_b = -dtm * p->kappa;
  const double sb = pow_int(g.h, bilap->h_power), sl = pow_int(g.h, lap->h_power);
  OrbitW wb{};
  for (int i = 0; i < 8; ++i) wb.w[i] = (bilap->orbit_coeff[i] * sb) * fac_b;
  const double wl0 = (lap->orbit_coeff[0] * sl) * dtm, wl1 = (lap->orbit_coeff[1] * sl) * dtm;
  // f'(c) = 2 rho (c-a)(c-b)(2c-a-b) as a cubic (cahn_hilliard.cpp:70-73 expanded)
  const double ca = p->c_alpha, cb = p->c_beta, s = ca + cb, pr = ca * cb, r2 = 2.0 * p->rho_w;
  const Poly3 chem{2.0 * r2, -3.0 * r2 * s, r2 * (s * s + 2.0 * pr), -r2 * pr * s};
  if (g.dim == 2) {
    // both formulations run the composed 13-point kernel in 2D: with the
    // fields L2-resident a factored warp-row kernel (sk_chf3d.cuh's scheme
    // per tile) measured slower (14.8 vs 13.2 us at 2048^2)
    Apply2DArgs a{};
    a.u = in;
    a.v = out;
    a.nx = g.n[0];
    a.ny = g.n[1];
    a.w = wb;
    a.wl0 = wl0;
    a.wl1 = wl1;
    a.chem = chem;
    a.bulk_ok = bulk_ok_ptrs && (a.nx % 2 == 0) && a.nx >= 64 + 4 && a.ny >= 32 + 4;
    return launch_2d<Mode::CahnHilliard>(a, stream);
  }
  Args3D a{};
  a.u = in;
  a.v = out;
  a.nx = g.n[0];
  a.ny = g.n[1];
  a.nz = g.n[2];
  for (int i = 0; i < 8; ++i) a.w[i] = wb.w[i];
  a.wl0 = wl0;
  a.wl1 = wl1;
  a.chem = chem;
  a.bulk_ok = bulk_ok_ptrs && (a.nx % 2 == 0) && a.nx >= C3R2::TX + 2 * C3R2::R && a.ny >= C3R2::TY + 2 * C3R2::R;
  a.z_ghosted = z_ghosted ? 1 : 0;
  a.ghost = ghost;
  if (p->formulation == SK_CH_COMPOSED) return launch_3d<Mode::CahnHilliard, C3R2>(a, stream);
  // factored: mu = f' - kappa L c ; c' = c + dt M L mu
  a.kl0 = -p->kappa * (lap->orbit_coeff[0] * sl);
  a.kl1 = -p->kappa * (lap->orbit_coeff[1] * sl);
  using CF = CfgChf3;
  using CT = CfgChf3T;
  CUtensorMap tm{};
  if (io == kIoMid || io == kIoLast)
    if (int st = make_tmap_padded(&tm, in, g)) return st;
  if (peer_lo || peer_hi) {  // slab step with the halo stores fused in (OUT 2)
    a.peer_lo = peer_lo;
    a.peer_hi = peer_hi;
    return launch_chf3d<CF, 0, 0, 2>(a, tm, stream);
  }
  switch (io) {
    case kIoFirst: return launch_chf3d<CF, 0, 0, 1>(a, tm, stream);
    case kIoMid: return launch_chf3d<CT, 0, 1, 1>(a, tm, stream);
    case kIoLast: return launch_chf3d<CT, 0, 1, 0>(a, tm, stream);
    default: return launch_chf3d<CF, 0, 0, 0>(a, tm, stream);
  }
}

// ---- chunk graphs --------------------------------------------------------
// nsteps >= 2 run as chunks of at most kGraphSteps (+1 for the last) steps,
// each one cached CUDA graph. A plain chunk ping-pongs c <-> scratch; a
// padded chunk (3D factored, whole tiles) runs c -> pad -> ... -> pad -> out
// through two ghost-padded buffers, so every step but the first loads its
// tile planes with one TMA box and no wrap logic. Every chunk starts from c;
// all but the last end in c; the last ends where the ping-pong parity says
// (result_is_scratch = nsteps % 2).
//
// The padded buffers belong to the launch stream: chunks replayed on one
// stream are stream-ordered, so they may share a pair; chunks on different
// streams never do. Graphs are keyed by everything their kernels bake in.
struct ChKey {
  double v[16] = {};
  uint64_t lap_uid = 0, bilap_uid = 0, epoch = 0;
  const void* c = nullptr;
  const void* scratch = nullptr;
  cudaStream_t stream = nullptr;
  int64_t len = 0;
  int padded = 0, to_scratch = 0;
  bool operator==(const ChKey& o) const {
    for (int i = 0; i < 16; ++i)
      if (v[i] != o.v[i]) return false;
    return lap_uid == o.lap_uid && bilap_uid == o.bilap_uid && epoch == o.epoch && c == o.c &&
           scratch == o.scratch && stream == o.stream && len == o.len && padded == o.padded &&
           to_scratch == o.to_scratch;
  }
};

struct ChChunk {
  ChKey key;
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;  // kernels per replay
  uint64_t used = 0;
};

struct ChPads {
  cudaStream_t stream = nullptr;
  size_t elems = 0;
  double* pad[2] = {nullptr, nullptr};
  uint64_t used = 0;
};

struct ChCache {
  std::mutex mu;
  std::vector<ChChunk> chunks;
  std::vector<ChPads> pads;
  uint64_t tick = 0;
  static constexpr size_t kMaxChunks = 16, kMaxPads = 2;
  ~ChCache() {  // process exit: the context may already be gone; do not touch the device
    chunks.clear();
    pads.clear();
  }

  void drop_chunk(size_t i) {
    cudaGraphExecDestroy(chunks[i].exec);
    chunks.erase(chunks.begin() + long(i));
  }

  // padded pair of `stream` with `elems` doubles each (LRU, at most kMaxPads pairs)
  int get_pads(cudaStream_t stream, size_t elems, double** out) {
    for (auto& ps : pads)
      if (ps.stream == stream && ps.elems == elems) {
        ps.used = ++tick;
        out[0] = ps.pad[0];
        out[1] = ps.pad[1];
        return SK_OK;
      }
    for (size_t i = 0; i < pads.size();)  // a different size on this stream, or the LRU pair when full
      if (pads[i].stream == stream || (pads.size() >= kMaxPads && lru_pads() == i)) {
        release_pads(i);
        i = 0;
      } else {
        ++i;
      }
    ChPads ps;
    ps.stream = stream;
    ps.elems = elems;
    for (double*& b : ps.pad) {
      const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&b), elems * 8);
      if (e != cudaSuccess) {
        if (ps.pad[0]) cudaFree(ps.pad[0]);
        return cuda_fail(e, "ghost-padded CH buffers");
      }
    }
    ps.used = ++tick;
    out[0] = ps.pad[0];
    out[1] = ps.pad[1];
    pads.push_back(ps);
    return SK_OK;
  }

  size_t lru_pads() const {
    size_t j = 0;
    for (size_t i = 1; i < pads.size(); ++i)
      if (pads[i].used < pads[j].used) j = i;
    return j;
  }

  // free a padded pair and every graph that uses it (after the device drains)
  void release_pads(size_t i) {
    cudaDeviceSynchronize();
    const ChPads ps = pads[i];
    for (size_t k = 0; k < chunks.size();)
      if (chunks[k].key.padded && chunks[k].key.stream == ps.stream) drop_chunk(k);
      else ++k;
    cudaFree(ps.pad[0]);
    cudaFree(ps.pad[1]);
    pads.erase(pads.begin() + long(i));
  }
};

ChCache& ch_cache() {
  static ChCache* c = new ChCache;  // never destroyed: graphs may outlive static destruction order
  return *c;
}

// ---- host entry point: copies overlapped with the steps (z wavefront) -----
// A K-step call from host memory is PCIe-bound (a 256^3 field is 134 MB each
// way at ~54 GB/s against ~1.1 ms for 20 steps). Output plane z of step s
// depends only on input planes z-2s .. z+2s, so the field is uploaded in
// plane chunks on one stream while a second stream advances every step's
// front as far as the planes present allow and a third stream downloads the
// final step's planes as they complete: upload, stepping and download
// overlap.
//
// The periodic z axis is unrolled into a line of nz + T planes, T = 4K:
// positions [nz, nz + T) hold copies of planes [0, T) (device copies made as
// those planes land). On the line no step needs a wrap: step s produces
// positions [2s, P - 2s) once positions [0, P) are present, as slab launches
// on z ranges (in-buffer halos); the final step's positions [2K, nz + 2K) are
// the field, the last 2K of them planes 0 .. 2K-1. When the upload ends only
// the fronts' last C + T positions per step remain -- no ghost exchange, no
// per-step seam work. (The 2K^2 redundant plane-steps cost ~16% more
// stepping at K = 20, off the PCIe-bound critical path.)
//
// Ping-pong safety: step s writes buffer s % 2, which holds step s-2. Its
// front trails step s-1's by 2 positions at both ends, so every position it
// overwrites has already been consumed by step s-1; the tail copies of a
// chunk are made before the chunk's fronts run. Every plane is computed by
// the same kernel arithmetic as the serial path, so the result is
// bit-identical (tests/test_gpu_ch_host.py).
struct HostPipe {
  cudaStream_t up = nullptr, run = nullptr, down = nullptr;
  std::vector<cudaEvent_t> ev;
  double* buf = nullptr;
  size_t elems = 0;  // per buffer
  int init() {
    if (up) return SK_OK;
    SK_CUDA_TRY(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
    SK_CUDA_TRY(cudaStreamCreateWithFlags(&run, cudaStreamNonBlocking));
    SK_CUDA_TRY(cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking));
    return SK_OK;
  }
  int event(size_t i, cudaEvent_t* out) {
    while (ev.size() <= i) {
      cudaEvent_t e;
      SK_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
    *out = ev[i];
    return SK_OK;
  }
  int reserve(size_t n) {
    if (elems >= n) return SK_OK;
    if (buf) SK_CUDA_TRY(cudaFree(buf));
    buf = nullptr;
    elems = 0;
    SK_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&buf), 2 * n * sizeof(double)));
    elems = n;
    return SK_OK;
  }
};

static bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// eligible: 3D fast path, enough planes for the fronts to move (nz >= 4K + 8)
static bool ch_host_pipelined_ok(const sk_stencil* lap, const sk_stencil* bilap, const GridInfo& g, int64_t nsteps,
                                 const double* c_host) {
  return option(SK_OPT_CH_HOST_PIPELINE) && g.dim == 3 && nsteps >= 1 && is_lap_shape(lap, 3) &&
         is_bilap_shape(bilap, 3) && g.n[2] >= 4 * nsteps + 8 && host_pinned(c_host);
}

static int ch_host_pipelined_run(HostPipe& hp, const sk_stencil* lap, const sk_stencil* bilap, const GridInfo& g,
                                 const sk_ch_params* p, double dt, int64_t nsteps, double* c_host) {
  if (int st = hp.init()) return st;
  const int64_t nz = g.n[2], plane = g.n[0] * g.n[1], S = nsteps;
  const int64_t T = 4 * S, L = nz + T;  // the unrolled line (T <= nz - 8: ch_host_pipelined_ok)
  if (int st = hp.reserve(size_t(L * plane))) return st;
  double* X[2] = {hp.buf, hp.buf + hp.elems};
  const size_t pb = size_t(plane) * sizeof(double);
  // one range [z0, z1) of step s (1-based) on the line: X[(s-1)%2] -> X[s%2], halos in the buffer
  auto range = [&](int64_t s, int64_t z0, int64_t z1) -> int {
    if (z1 <= z0) return SK_OK;
    GridInfo gr = g;
    gr.n[2] = gr.un[2] = z1 - z0;
    gr.rows = plane * (z1 - z0);
    return ch_step_fast(lap, bilap, gr, p, dt, X[(s - 1) % 2] + z0 * plane, X[s % 2] + z0 * plane, hp.run, true,
                        kIoPlain, /*z_ghosted=*/true);
  };
  size_t nev = 0;
  auto handoff = [&](cudaStream_t from, cudaStream_t to) -> int {  // `to` waits for `from`'s work so far
    cudaEvent_t e;
    if (int st = hp.event(nev++, &e)) return st;
    SK_CUDA_TRY(cudaEventRecord(e, from));
    SK_CUDA_TRY(cudaStreamWaitEvent(to, e, 0));
    return SK_OK;
  };
  auto download = [&](int64_t a, int64_t b) -> int {  // final-step positions [a, b) -> planes (mod nz)
    for (int64_t lo = a; lo < b;) {
      const int64_t hi = lo < nz ? std::min(b, nz) : b, z = lo < nz ? lo : lo - nz;
      SK_CUDA_TRY(cudaMemcpyAsync(c_host + z * plane, X[S % 2] + lo * plane, size_t(hi - lo) * pb,
                                  cudaMemcpyDeviceToHost, hp.down));
      lo = hi;
    }
    return SK_OK;
  };
#ifdef SK_PIPE_TRACE  // tools-only timeline (tools/ab_build.py ... -DSK_PIPE_TRACE)
  std::vector<std::pair<std::string, cudaEvent_t>> tr;
  auto mark = [&](const std::string& what, cudaStream_t s) {
    cudaEvent_t e = nullptr;
    const cudaError_t c1 = cudaEventCreate(&e);
    const cudaError_t c2 = cudaEventRecord(e, s);
    if (c1 != cudaSuccess || c2 != cudaSuccess)
      fprintf(stderr, "[pipe] mark %s: %s / %s\n", what.c_str(), cudaGetErrorString(c1), cudaGetErrorString(c2));
    tr.push_back({what, e});
  };
#else
  auto mark = [](const auto&, cudaStream_t) {};
#endif
  // the calling thread's earlier work on the shared streams is ordered before this call
  if (int st = handoff(host_stream(), hp.up)) return st;
  mark("start", hp.up);
  // ~8 upload chunks (>= 8 planes each: fewer, larger launches for the fronts).
  // Measured at 256^3 x 20 (B200, PCIe Gen5): 4.3-4.4 ms against 6.15 ms for
  // the serial call. The stepping keeps pace with the upload until the last
  // chunk; then its cone (C + 4K positions per step) is stepped in two passes
  // so the lower half's final planes go down while the upper half is stepped
  // (4.5-4.8 ms in one pass). Splitting the last chunk finer (C/2, C/4, ...)
  // measured slower: each round is K launches.
  const int64_t C = std::max<int64_t>(8, (nz + 7) / 8);
  std::vector<int64_t> hi(size_t(S) + 1);
  for (int64_t s = 1; s <= S; ++s) hi[size_t(s)] = 2 * s;
  int64_t done = 2 * S;  // final-step positions downloaded: [2S, done)
  for (int64_t z0 = 0; z0 < nz; z0 += C) {
    const int64_t z1 = std::min(nz, z0 + C);
    SK_CUDA_TRY(cudaMemcpyAsync(X[0] + z0 * plane, c_host + z0 * plane, size_t(z1 - z0) * pb,
                                cudaMemcpyHostToDevice, hp.up));
    mark("up " + std::to_string(z1), hp.up);
    if (int st = handoff(hp.up, hp.run)) return st;
    if (z0 < T)  // this chunk's share of the tail copies, before any front overwrites buffer 0
      SK_CUDA_TRY(cudaMemcpyAsync(X[0] + (nz + z0) * plane, X[0] + z0 * plane, size_t(std::min(z1, T) - z0) * pb,
                                  cudaMemcpyDeviceToDevice, hp.run));
    const int64_t P = z1 == nz ? L : z1;  // positions present
    auto fronts = [&](int64_t cap) -> int {  // every front up to P - 2s, and for the final step below cap
      for (int64_t s = 1; s <= S; ++s) {
        const int64_t top = std::min(P - 2 * s, cap + 2 * (S - s));
        if (top > hi[size_t(s)]) {
          if (int st = range(s, hi[size_t(s)], top)) return st;
          hi[size_t(s)] = top;
        }
      }
      return SK_OK;
    };
    if (z1 == nz) {  // the last cone in two passes: the lower half's planes go down during the upper pass
      const int64_t mid = (hi[size_t(S)] + (P - 2 * S)) / 2;
      if (int st = fronts(mid)) return st;
      if (int st = handoff(hp.run, hp.down)) return st;
      if (int st = download(done, hi[size_t(S)])) return st;
      done = hi[size_t(S)];
    }
    if (int st = fronts(L)) return st;
    if (hi[size_t(S)] - done >= C / 2 || z1 == nz) {
      if (int st = handoff(hp.run, hp.down)) return st;
      if (int st = download(done, hi[size_t(S)])) return st;
      mark("down " + std::to_string(hi[size_t(S)]), hp.down);
      done = hi[size_t(S)];
    }
    mark("fronts " + std::to_string(z1), hp.run);
  }
  mark("down end", hp.down);
  SK_CUDA_TRY(cudaStreamSynchronize(hp.down));
  SK_CUDA_TRY(cudaStreamSynchronize(hp.run));
#ifdef SK_PIPE_TRACE
  for (auto& m : tr) {
    float ms = 0;
    const cudaError_t e = cudaEventElapsedTime(&ms, tr[0].second, m.second);
    fprintf(stderr, "[pipe] %-14s %8.3f ms %s\n", m.first.c_str(), ms, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  for (auto& m : tr) cudaEventDestroy(m.second);
#endif
  return SK_OK;
}

static int ch_host_pipelined(const sk_stencil* lap, const sk_stencil* bilap, const GridInfo& g, const sk_ch_params* p,
                             double dt, int64_t nsteps, double* c_host) {
  thread_local HostPipe hp;
  const int st = ch_host_pipelined_run(hp, lap, bilap, g, p, dt, nsteps, c_host);
  if (st != SK_OK) {  // drain: no copy may still touch the caller's field after an error return
    for (cudaStream_t s : {hp.up, hp.run, hp.down})
      if (s) cudaStreamSynchronize(s);
  }
  return st;
}

}  // namespace sk

using namespace sk;

extern "C" {

int sk_ch_explicit(const sk_stencil* lap, const sk_stencil* bilap, const sk_grid_desc* gd, const sk_ch_params* p,
                   double dt, int64_t nsteps, double* c, double* scratch, int* result_is_scratch, void* stream_p) {
  if (!lap || !bilap || !p) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil or params");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  for (int a = 0; a < g.dim; ++a)
    if (g.bc[a] != SK_BC_PERIODIC) return fail(SK_ERR_NON_PERIODIC, "Cahn-Hilliard runs on periodic grids");
  if (g.dim != 2 && g.dim != 3) return fail(SK_ERR_INVALID_ARGUMENT, "Cahn-Hilliard stepping is 2D or 3D");
  if (int st = check_width(lap, g)) return st;
  if (int st = check_width(bilap, g)) return st;
  if (!(dt > 0)) return fail(SK_ERR_INVALID_ARGUMENT, "dt must be positive");
  if (nsteps < 0) return fail(SK_ERR_INVALID_ARGUMENT, "nsteps must be >= 0");
  if (p->formulation != SK_CH_FACTORED && p->formulation != SK_CH_COMPOSED)
    return fail(SK_ERR_INVALID_ARGUMENT, "formulation must be SK_CH_FACTORED or SK_CH_COMPOSED");
  if (!c || !scratch || c == scratch) return fail(SK_ERR_INVALID_ARGUMENT, "bad field pointers");
  if (result_is_scratch) *result_is_scratch = int(nsteps % 2);
  if (nsteps == 0 || g.rows == 0) return SK_OK;
  cudaStream_t stream = as_stream(stream_p);
  const bool ptr_ok = ((reinterpret_cast<uintptr_t>(c) | reinterpret_cast<uintptr_t>(scratch)) & 15) == 0;
  const bool fast = is_lap_shape(lap, g.dim) && is_bilap_shape(bilap, g.dim);

  if (!fast) {  // generic: four passes per step
    const int64_t n = g.rows;
    double* tmp = nullptr;
    SK_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double) * size_t(3 * n), stream));
    double *w = tmp, *la = tmp + n, *lb = tmp + 2 * n;
    const ChemParams chem{p->rho_w, p->c_alpha, p->c_beta};
    const int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(kNumSMs) * 16));
    double* bufs[2] = {c, scratch};
    int st = SK_OK;
    for (int64_t k = 0; k < nsteps && st == SK_OK; ++k) {
      const double* in = bufs[k % 2];
      double* out = bufs[(k + 1) % 2];
      chem_kernel<<<grid, 256, 0, stream>>>(n, in, w, chem);
      g_launches++;
      st = launch_apply(lap, g, w, la, stream);
      if (st == SK_OK) st = launch_apply(bilap, g, in, lb, stream);
      if (st == SK_OK) {
        ch_update_kernel<<<grid, 256, 0, stream>>>(n, in, la, lb, dt * p->mobility, p->kappa, out);
        g_launches++;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) st = cuda_fail(e, "ch_update_kernel");
      }
    }
    cudaFreeAsync(tmp, stream);
    return st;
  }

  // fast path: one step launched directly; longer runs as cached chunk graphs
  if (nsteps == 1) return ch_step_fast(lap, bilap, g, p, dt, c, scratch, stream, ptr_ok);
  const bool padded = g.dim == 3 && p->formulation == SK_CH_FACTORED && ptr_ok && chf3d_padded_ok(g) &&
                      option(SK_OPT_CH_PADDED);
  ChKey base;
  const double v[16] = {dt, p->kappa, p->mobility, p->rho_w, p->c_alpha, p->c_beta, g.h,
                        double(g.n[0]), double(g.n[1]), double(g.n[2]), double(g.dim) + 10.0 * double(p->formulation),
                        lap->orbit_coeff[0], lap->orbit_coeff[1], bilap->orbit_coeff[0], bilap->orbit_coeff[1],
                        bilap->orbit_coeff[2] + 7.0 * bilap->orbit_coeff[3]};
  for (int i = 0; i < 16; ++i) base.v[i] = v[i];
  base.lap_uid = lap->uid;
  base.bilap_uid = bilap->uid;
  base.epoch = option_epoch();
  base.c = c;
  base.scratch = scratch;
  base.stream = stream;
  base.padded = padded ? 1 : 0;
  ChCache& cache = ch_cache();
  std::lock_guard<std::mutex> lock(cache.mu);
  for (int64_t done = 0; done < nsteps;) {
    const int64_t rem = nsteps - done;
    const int64_t len = rem <= kGraphSteps + 1 ? rem : kGraphSteps;  // never a 1-step chunk
    ChKey key = base;
    key.len = len;
    key.to_scratch = (done + len == nsteps) && (nsteps % 2) ? 1 : 0;  // padded chunks: where Last writes
    ChChunk* hit = nullptr;
    for (auto& ch : cache.chunks)
      if (ch.key == key) hit = &ch;
    if (!hit) {
      double* pad[2] = {nullptr, nullptr};
      if (padded) {
        const size_t elems = size_t(g.n[0] + 2 * kPadL) * size_t(g.n[1] + 2 * kPadT) * size_t(g.n[2]);
        if (int st = cache.get_pads(stream, elems, pad)) return st;
      }
      if (cache.chunks.size() >= ChCache::kMaxChunks) {  // evict the least recently used graph
        size_t j = 0;
        for (size_t i = 1; i < cache.chunks.size(); ++i)
          if (cache.chunks[i].used < cache.chunks[j].used) j = i;
        cache.drop_chunk(j);
      }
      cudaStream_t cap = stream ? stream : capture_stream();
      SK_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      int st = SK_OK;
      const int64_t l0 = g_launches.load();
      double* out_last = key.to_scratch ? scratch : c;
      for (int64_t k = 0; k < len && st == SK_OK; ++k) {
        if (!padded)  // plain ping-pong from c
          st = ch_step_fast(lap, bilap, g, p, dt, (k % 2) ? scratch : c, (k % 2) ? c : scratch, cap, ptr_ok);
        else if (k == 0)
          st = ch_step_fast(lap, bilap, g, p, dt, c, pad[0], cap, ptr_ok, kIoFirst);
        else if (k + 1 < len)
          st = ch_step_fast(lap, bilap, g, p, dt, pad[(k - 1) % 2], pad[k % 2], cap, ptr_ok, kIoMid);
        else
          st = ch_step_fast(lap, bilap, g, p, dt, pad[(k - 1) % 2], out_last, cap, ptr_ok, kIoLast);
      }
      const int64_t launches = g_launches.load() - l0;
      g_launches -= launches;  // capture does not execute; counted per replay below
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamEndCapture(cap, &graph);
      if (st != SK_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
      }
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      ChChunk ch;
      ch.key = key;
      ch.launches = launches;
      e = cudaGraphInstantiate(&ch.exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
      cache.chunks.push_back(ch);
      hit = &cache.chunks.back();
    }
    hit->used = ++cache.tick;
    SK_CUDA_TRY(cudaGraphLaunch(hit->exec, stream));
    g_launches += hit->launches;
    done += len;
  }
  return SK_OK;
}

int sk_ch_explicit_slab(const sk_stencil* lap, const sk_stencil* bilap, const sk_grid_desc* gd, const sk_ch_params* p,
                        double dt, const double* in_ghosted, double* out, void* stream_p) {
  if (!lap || !bilap || !p) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil or params");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  if (g.dim != 3) return fail(SK_ERR_INVALID_ARGUMENT, "slab stepping is 3D");
  for (int a = 0; a < 3; ++a)
    if (g.bc[a] != SK_BC_PERIODIC) return fail(SK_ERR_NON_PERIODIC, "Cahn-Hilliard runs on periodic grids");
  if (!is_lap_shape(lap, 3) || !is_bilap_shape(bilap, 3))
    return fail(SK_ERR_INVALID_ARGUMENT, "slab stepping needs the 7-point L and its 25-point composition");
  if (g.n[0] < 5 || g.n[1] < 5) return fail(SK_ERR_STENCIL_WIDER_THAN_GRID, "periodic axis narrower than stencil support");
  if (!(dt > 0)) return fail(SK_ERR_INVALID_ARGUMENT, "dt must be positive");
  if (p->formulation != SK_CH_FACTORED && p->formulation != SK_CH_COMPOSED)
    return fail(SK_ERR_INVALID_ARGUMENT, "formulation must be SK_CH_FACTORED or SK_CH_COMPOSED");
  if (!in_ghosted || !out) return fail(SK_ERR_INVALID_ARGUMENT, "bad field pointers");
  const int64_t plane = g.n[0] * g.n[1];
  const double* in = in_ghosted + 2 * plane;  // first interior plane
  const bool ptr_ok = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  return ch_step_fast(lap, bilap, g, p, dt, in, out, as_stream(stream_p), ptr_ok, kIoPlain, /*z_ghosted=*/true);
}

int sk_ch_explicit_slab_peer(const sk_stencil* lap, const sk_stencil* bilap, const sk_grid_desc* gd,
                             const sk_ch_params* p, double dt, const double* in_ghosted, double* out,
                             double* peer_lo, double* peer_hi, void* stream_p) {
  if (!lap || !bilap || !p) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil or params");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  if (g.dim != 3) return fail(SK_ERR_INVALID_ARGUMENT, "slab stepping is 3D");
  for (int a = 0; a < 3; ++a)
    if (g.bc[a] != SK_BC_PERIODIC) return fail(SK_ERR_NON_PERIODIC, "Cahn-Hilliard runs on periodic grids");
  if (!is_lap_shape(lap, 3) || !is_bilap_shape(bilap, 3))
    return fail(SK_ERR_INVALID_ARGUMENT, "slab stepping needs the 7-point L and its 25-point composition");
  if (g.n[0] < 5 || g.n[1] < 5) return fail(SK_ERR_STENCIL_WIDER_THAN_GRID, "periodic axis narrower than stencil support");
  if (g.n[2] < 4) return fail(SK_ERR_STENCIL_WIDER_THAN_GRID, "a slab with fused halo stores needs >= 4 planes");
  if (!(dt > 0)) return fail(SK_ERR_INVALID_ARGUMENT, "dt must be positive");
  if (p->formulation != SK_CH_FACTORED)
    return fail(SK_ERR_INVALID_ARGUMENT, "fused halo stores need the factored formulation (SK_CH_FACTORED)");
  if (!in_ghosted || !out) return fail(SK_ERR_INVALID_ARGUMENT, "bad field pointers");
  const int64_t plane = g.n[0] * g.n[1];
  const double* in = in_ghosted + 2 * plane;
  const bool ptr_ok = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out) |
                        reinterpret_cast<uintptr_t>(peer_lo) | reinterpret_cast<uintptr_t>(peer_hi)) & 15) == 0;
  if (!peer_lo && !peer_hi)
    return ch_step_fast(lap, bilap, g, p, dt, in, out, as_stream(stream_p), ptr_ok, kIoPlain, /*z_ghosted=*/true);
  return ch_step_fast(lap, bilap, g, p, dt, in, out, as_stream(stream_p), ptr_ok, kIoPlain, /*z_ghosted=*/true, 2,
                      peer_lo, peer_hi);
}

int sk_ch_explicit_host(const sk_stencil* lap, const sk_stencil* bilap, const sk_grid_desc* gd, const sk_ch_params* p,
                        double dt, int64_t nsteps, double* c_host) {
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  if (!c_host && g.rows > 0) return fail(SK_ERR_INVALID_ARGUMENT, "null host field");
  if (nsteps < 0) return fail(SK_ERR_INVALID_ARGUMENT, "nsteps must be >= 0");
  if (g.rows == 0) return SK_OK;
  if (nsteps > 0 && lap && bilap && p && dt > 0 && g.dim == 3) {
    bool periodic = true;
    for (int a = 0; a < 3; ++a) periodic = periodic && g.bc[a] == SK_BC_PERIODIC;
    if (periodic && check_width(lap, g) == SK_OK && check_width(bilap, g) == SK_OK &&
        (p->formulation == SK_CH_FACTORED || p->formulation == SK_CH_COMPOSED) &&
        ch_host_pipelined_ok(lap, bilap, g, nsteps, c_host))
      return ch_host_pipelined(lap, bilap, g, p, dt, nsteps, c_host);
  }
  // c_host -> c (device), steps ping-pong c <-> s, result -> c_host. The
  // device pair is per host thread and kept between calls, so repeated calls
  // replay the cached chunk graphs (keyed by the buffers) instead of
  // re-capturing them.
  struct Staging {
    double* buf = nullptr;
    size_t elems = 0;
  };
  thread_local Staging stage;
  cudaStream_t hs = host_stream();
  const size_t n = size_t(g.rows);
  if (stage.elems < n) {
    if (stage.buf) SK_CUDA_TRY(cudaFree(stage.buf));
    stage.buf = nullptr;
    stage.elems = 0;
    SK_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&stage.buf), 2 * n * sizeof(double)));
    stage.elems = n;
  }
  double* cd = stage.buf;
  double* sd = stage.buf + stage.elems;
  SK_CUDA_TRY(cudaMemcpyAsync(cd, c_host, n * sizeof(double), cudaMemcpyHostToDevice, hs));
  int in_scratch = 0;
  if (int e = sk_ch_explicit(lap, bilap, gd, p, dt, nsteps, cd, sd, &in_scratch, hs)) {
    cudaStreamSynchronize(hs);  // the upload may still read c_host
    return e;
  }
  SK_CUDA_TRY(cudaMemcpyAsync(c_host, in_scratch ? sd : cd, n * sizeof(double), cudaMemcpyDeviceToHost, hs));
  SK_CUDA_TRY(cudaStreamSynchronize(hs));
  return SK_OK;
}

int sk_free_energy(const sk_grid_desc* gd, const sk_ch_params* p, const double* c, double* energy, void* stream_p) {
  if (!p || !energy) return fail(SK_ERR_INVALID_ARGUMENT, "null params/output");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  for (int a = 0; a < g.dim; ++a)
    if (g.bc[a] != SK_BC_PERIODIC) return fail(SK_ERR_NON_PERIODIC, "Cahn-Hilliard runs on periodic grids");
  if (!c) return fail(SK_ERR_INVALID_ARGUMENT, "null field");
  cudaStream_t stream = as_stream(stream_p);
  int grid = int(std::min<int64_t>((g.rows + 1023) / 1024, int64_t(kNumSMs) * 8));
  if (grid < 1) grid = 1;
  double* ws = nullptr;
  SK_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ws), sizeof(double) * size_t(grid + 4) + 64, stream));
  double* out = ws + grid;
  unsigned* counter = reinterpret_cast<unsigned*>(out + 2);
  cudaMemsetAsync(counter, 0, sizeof(unsigned), stream);
  energy_kernel<<<grid, kThreads, 0, stream>>>(c, g.dim, g.n[0], g.n[1], g.n[2], 0.5 / g.h, p->kappa, p->rho_w,
                                               p->c_alpha, p->c_beta, ws, counter, out);
  g_launches++;
  cudaError_t e = cudaGetLastError();
  double total = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&total, out, sizeof(double), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  cudaFreeAsync(ws, stream);
  if (e != cudaSuccess) return cuda_fail(e, "energy_kernel");
  *energy = total * pow_int(g.h, g.dim);  // :106
  return SK_OK;
}

}  // extern "C"
