// Stencil handles, orbit classification and the matrix-free composed apply.
//
// Reference boundary: the reference has no matrix-free apply; its composed
// apply is assemble + csr_matvec (grid.cpp:166-172). sk_composed_apply
// computes the same v = S u without materialising the matrix.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "sk_internal.hpp"
#include "sk_stencil_kernels.cuh"
#include "sk_stream3d.cuh"
#include "sk_fac73.cuh"

sk_stencil::~sk_stencil() {
  if (rep_exec) cudaGraphExecDestroy(rep_exec);
  if (d_off) cudaFree(d_off);
  if (d_coeff) cudaFree(d_coeff);
  if (d_coeff_lo) cudaFree(d_coeff_lo);
}

namespace sk {

namespace {

using Key = std::array<int, 3>;

Key orbit_key(const int* o) {
  Key k{std::abs(o[0]), std::abs(o[1]), std::abs(o[2])};
  std::sort(k.begin(), k.end(), std::greater<int>());
  return k;
}

// number of distinct signed axis permutations of key living in `dim` axes
int orbit_size(const Key& key, int dim) {
  std::set<std::array<int, 3>> seen;
  std::array<int, 3> perm = {0, 1, 2};
  do {
    for (int sgn = 0; sgn < 8; ++sgn) {
      std::array<int, 3> v{};
      bool ok = true;
      for (int a = 0; a < 3; ++a) {
        int x = key[perm[a]];
        if (sgn & (1 << a)) x = -x;
        if (a >= dim && x != 0) ok = false;
        v[a] = x;
      }
      if (ok) seen.insert(v);
    }
  } while (std::next_permutation(perm.begin(), perm.end()));
  return static_cast<int>(seen.size());
}

const std::vector<Key>& class_orbits(int kclass) {
  static const std::vector<Key> c1 = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {2, 0, 0}};
  static const std::vector<Key> c3 = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {2, 0, 0},
                                      {2, 1, 0}, {2, 2, 0}, {3, 0, 0}, {4, 0, 0}};
  return kclass == 3 ? c3 : c1;  // classes 1 and 2 share the radius-2 orbit list
}

// Map the stencil onto a specialised symmetric kernel when every orbit is
// complete and carries a single coefficient; otherwise generic.
void classify(sk_stencil* s) {
  s->kclass = 0;
  if (s->dim < 2) return;
  std::map<Key, std::pair<double, int>> orbits;
  for (int e = 0; e < s->nent; ++e) {
    const Key k = orbit_key(&s->off[3 * e]);
    auto it = orbits.find(k);
    if (it == orbits.end()) {
      orbits[k] = {s->coeff[e], 1};
    } else {
      if (std::memcmp(&it->second.first, &s->coeff[e], sizeof(double)) != 0) return;  // not symmetric
      it->second.second++;
    }
  }
  for (const auto& [k, v] : orbits)
    if (v.second != orbit_size(k, s->dim)) return;  // incomplete orbit
  const std::vector<int> candidates = s->dim == 2 ? std::vector<int>{1} : std::vector<int>{2, 3};
  for (int kc : candidates) {
    const auto& list = class_orbits(kc);
    bool all_in = true;
    for (const auto& [k, v] : orbits)
      if (std::find(list.begin(), list.end(), k) == list.end()) all_in = false;
    if (!all_in) continue;
    s->kclass = kc;
    for (size_t i = 0; i < list.size(); ++i) {
      auto it = orbits.find(list[i]);
      s->orbit_coeff[i] = it == orbits.end() ? 0.0 : it->second.first;
    }
    return;
  }
}

template <class K>
int set_smem(K kernel, int bytes) {
  if (bytes > 48 * 1024) SK_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return SK_OK;
}

}  // namespace

cudaStream_t capture_stream() {
  thread_local cudaStream_t s = nullptr;
  if (!s) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  return s;
}

int check_width(const sk_stencil* s, const GridInfo& g) {
  if (s->dim != g.dim) return fail(SK_ERR_DIM_MISMATCH, "stencil/grid dimension mismatch");
  for (int a = 0; a < g.dim; ++a) {
    if (g.bc[a] == SK_BC_PERIODIC) {
      if (s->hi[a] - s->lo[a] > g.n[a] - 1)
        return fail(SK_ERR_STENCIL_WIDER_THAN_GRID, "periodic axis narrower than stencil support");
    } else if (std::max(std::abs(s->lo[a]), std::abs(s->hi[a])) > g.n[a] - 2) {
      return fail(SK_ERR_STENCIL_WIDER_THAN_GRID, "reflected ghost would leave the grid");
    }
  }
  return SK_OK;
}

// ---- kernel configurations ----------------------------------------------
#ifndef SK_T2_TY  // experiments: 2D tile height, points per thread
#define SK_T2_TY 32
#define SK_T2_PX 2
#define SK_T2_PY 4
#endif
using T2 = Tile2D<64, SK_T2_TY, SK_T2_PX, SK_T2_PY>;
using C3R2 = Cfg3R2;
using C3R4 = Cfg3R4;

int num_sms();
int num_sms() {
  static int n = [] {
    int dev = 0, v = kNumSMs;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <Mode M>
int launch_2d(const Apply2DArgs& a, cudaStream_t stream) {
  auto kern = stencil2d_kernel<M, 64, SK_T2_TY, SK_T2_PX, SK_T2_PY>;
  constexpr int smem = M == Mode::CgApply ? T2::SMEM_BYTES_CG : T2::SMEM_BYTES;
  static int once = set_smem(kern, smem);
  if (once != SK_OK) return once;
  dim3 grid(unsigned((a.nx + 63) / 64), unsigned((a.ny + SK_T2_TY - 1) / SK_T2_TY));
  // programmatic dependent launch: overlaps this grid's ramp-up (tile loads
  // and, for Apply, the whole computation) with the predecessor's tail
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(T2::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // (the fused CG apply follows K2 of the previous iteration: measured slower
  // with the programmatic edge)
  if (!option(SK_OPT_PDL) || M == Mode::CgApply) cfg.numAttrs = 0;
  SK_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a));
  SK_LAUNCH_CHECK("stencil2d_kernel");
  return SK_OK;
}

template <Mode M, class C, bool PQ = false>
int launch_3d(Args3D a, cudaStream_t stream);
template <Mode M, class C, bool PQ>
int launch_3d(Args3D a, cudaStream_t stream) {
  auto bulk = stream3d_kernel<M, C, false, PQ>;
  auto fallback = stream3d_kernel<M, C, true, PQ>;
  constexpr int bulk_smem = C::SMEM_BYTES - C::TABLE_BYTES;  // no boundary-map table
  static int once = set_smem(bulk, bulk_smem) != SK_OK ? SK_ERR_CUDA : set_smem(fallback, C::SMEM_BYTES);
  if (once != SK_OK) return once;
  // rotated columns (seg_of: balanced ranges, neighbour tiles in phase);
  // z-ghosted slabs: lockstep for the radius-2 apply (halo rows from L2),
  // balanced otherwise
  a.zrot = (a.z_ghosted && !a.in_pitch) ? 0 : 1;  // a padded field has its z halo: columns may rotate
  const int64_t grid = persistent_grid<C>(a, num_sms(), /*lockstep=*/!a.zrot && C::R == 2 && M == Mode::Apply);
  if (grid == 0) return fail(SK_ERR_INVALID_ARGUMENT, "grid too large for the 3D streaming kernels");
  if (a.bulk_ok)  // (after persistent_grid, which may clear it)
    bulk<<<unsigned(grid), C::THREADS, bulk_smem, stream>>>(a);
  else
    fallback<<<unsigned(grid), C::THREADS, C::SMEM_BYTES, stream>>>(a);
  SK_LAUNCH_CHECK("stream3d_kernel");
  return SK_OK;
}

template int launch_2d<Mode::CahnHilliard>(const Apply2DArgs&, cudaStream_t);

int cg_apply_2d_ctas(const sk_stencil* s, const GridInfo& g) {
  if (s->kclass != 1 || g.dim != 2) return 0;
  for (int a = 0; a < 2; ++a)
    if (g.un[a] < 5) return 0;  // streamable at radius 2
  return int(((g.un[0] + 63) / 64) * ((g.un[1] + SK_T2_TY - 1) / SK_T2_TY));
}

void cg_apply_2d_args(const sk_stencil* s, const GridInfo& g, const double* p, const double* r, double* q,
                      Apply2DArgs* out) {
  const double scale = pow_int(g.h, s->h_power);
  Apply2DArgs a{};
  for (int i = 0; i < 8; ++i) a.w.w[i] = s->orbit_coeff[i] * scale;
  a.u = p;
  a.v = q;
  a.nx = g.un[0];
  a.ny = g.un[1];
  a.bc[0] = g.bc[0];
  a.bc[1] = g.bc[1];
  a.r = r;
  *out = a;
}

int launch_cg_apply_2d(const sk_stencil* s, const GridInfo& g, const double* p, const double* r, double* q,
                       CgState* st, double* partials, cudaStream_t stream) {
  if (!cg_apply_2d_ctas(s, g)) return fail(SK_ERR_INVALID_ARGUMENT, "fused CG apply needs a 2D class-1 stencil");
  Apply2DArgs a{};
  cg_apply_2d_args(s, g, p, r, q, &a);
  a.st = st;
  a.partials = partials;
  return launch_2d<Mode::CgApply>(a, stream);
}
template int launch_3d<Mode::CahnHilliard, Cfg3CH>(Args3D, cudaStream_t);

int launch_generic(const sk_stencil* s, const GridInfo& g, const double* u, double* v, cudaStream_t stream) {
  GenericArgs a{};
  a.u = u;
  a.v = v;
  a.off = s->d_off;
  a.coeff = s->d_coeff;
  a.nent = s->nent;
  a.dim = g.dim;
  for (int d = 0; d < 3; ++d) {
    a.n[d] = g.n[d];
    a.un[d] = g.un[d];
    a.bc[d] = g.bc[d];
  }
  a.scale = pow_int(g.h, s->h_power);
  a.rows = g.rows;
  for (int d = 0; d < 3; ++d) {
    a.lo[d] = d < g.dim ? s->lo[d] : 0;
    a.hi[d] = d < g.dim ? s->hi[d] : 0;
  }
  if (g.rows == 0) return SK_OK;
  if (g.un[1] > 65535 || g.un[2] > 65535)
    return fail(SK_ERR_INVALID_ARGUMENT, "generic apply: more than 65535 unknowns along y or z");
  const int threads = 256;
  const size_t smem = size_t(s->nent) * 16;
  static int once = set_smem(stencil_generic_kernel, 227 * 1024);
  if (once != SK_OK) return once;
  if (smem > 227 * 1024) return fail(SK_ERR_INVALID_ARGUMENT, "generic apply: too many stencil entries");
  const dim3 grid(unsigned((g.un[0] + threads - 1) / threads), unsigned(g.un[1]), unsigned(g.un[2]));
  stencil_generic_kernel<<<grid, threads, smem, stream>>>(a);
  SK_LAUNCH_CHECK("stencil_generic_kernel");
  return SK_OK;
}

static bool all_periodic(const GridInfo& g) {
  for (int a = 0; a < g.dim; ++a)
    if (g.bc[a] != SK_BC_PERIODIC) return false;
  return true;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// The streaming kernels need every axis at least as wide as the stencil
// reach on both sides (periodic wrap / one reflection per side).
static bool streamable(const sk_stencil* s, const GridInfo& g, int radius) {
  for (int a = 0; a < g.dim; ++a)
    if (g.un[a] < 2 * radius + 1) return false;
  (void)s;
  return true;
}

// The uploaded stencil is compose(laplacian(3, 4), laplacian(3, 4)) (the
// 73-point composition of configs 5's operator, stencil.cpp:75-87): orbit
// coefficients 1607/24, -182/9, 32/9, 109/36, -2/9, 1/72, -2/9, 1/144 (as the
// reference's truncated doubles, within 2 ulp) and h^-4.
static bool is_l4l4(const sk_stencil* s) {
  if (s->kclass != 3 || s->dim != 3 || s->h_power != -4) return false;
  static const double want[8] = {1607.0 / 24, -182.0 / 9, 32.0 / 9, 109.0 / 36, -2.0 / 9, 1.0 / 72, -2.0 / 9, 1.0 / 144};
  for (int i = 0; i < 8; ++i)
    if (!(std::fabs(s->orbit_coeff[i] - want[i]) <= 4.5e-16 * std::fabs(want[i]))) return false;
  return true;
}

// Factored 73-point apply (sk_fac73.cuh): L4 weights (centre 3 * -30/12,
// axis +-1: 16/12, axis +-2: -1/12, generators.cpp:98) scaled by h^-2 per
// pass. 16-byte periodic path only (whole-tile halos, even nx); returns
// kApplyPqUnsupported when the grid needs the literal kernel instead.
template <bool PQ = false>
static int launch_fac73(Args3D a, double h_m2, cudaStream_t stream) {
  using C = CfgF2;
  using SM = F2Smem<C>;
  if (!a.bulk_ok || a.nx < C::TX + 2 * C::R || a.ny < C::TY + 2 * C::R) return kApplyPqUnsupported;
  const L4W lw{(3.0 * (-30.0 / 12.0)) * h_m2, (16.0 / 12.0) * h_m2, (-1.0 / 12.0) * h_m2};
  auto kern = fac73v2_kernel<C, PQ>;
  static int once = set_smem(kern, SM::BYTES);
  if (once != SK_OK) return once;
  a.zrot = 1;
  const int64_t grid = persistent_grid<C>(a, num_sms(), /*lockstep=*/false);
  if (grid == 0 || !a.bulk_ok) return kApplyPqUnsupported;
  kern<<<unsigned(grid), C::THREADS, SM::BYTES, stream>>>(a, lw);
  SK_LAUNCH_CHECK("fac73v2_kernel");
  return SK_OK;
}

int launch_apply(const sk_stencil* s, const GridInfo& g, const double* u, double* v, cudaStream_t stream,
                 bool input_stable) {
  const double scale = pow_int(g.h, s->h_power);
  OrbitW w{};
  for (int i = 0; i < 8; ++i) w.w[i] = s->orbit_coeff[i] * scale;  // == coeff.to_double()*pow_int (grid.cpp:80)
  const bool per = all_periodic(g);
  if (s->kclass == 1 && g.dim == 2 && streamable(s, g, 2)) {
    Apply2DArgs a{};
    a.u = u;
    a.v = v;
    a.nx = g.un[0];
    a.ny = g.un[1];
    a.w = w;
    a.bc[0] = g.bc[0];
    a.bc[1] = g.bc[1];
    a.input_stable = input_stable;
    a.bulk_ok = per && (a.nx % 2 == 0) && a.nx >= 64 + 4 && a.ny >= 32 + 4 && aligned16(u) && aligned16(v);
    return launch_2d<Mode::Apply>(a, stream);
  }
  if ((s->kclass == 2 || s->kclass == 3) && g.dim == 3 && streamable(s, g, s->kclass == 2 ? 2 : 4)) {
    Args3D a{};
    a.u = u;
    a.v = v;
    a.nx = g.un[0];
    a.ny = g.un[1];
    a.nz = g.un[2];
    for (int i = 0; i < 3; ++i) a.bc[i] = g.bc[i];
    for (int i = 0; i < 8; ++i) a.w[i] = w.w[i];
    if (s->kclass == 2) {
      a.bulk_ok = per && (a.nx % 2 == 0) && a.nx >= C3R2::TX + 2 * C3R2::R && a.ny >= C3R2::TY + 2 * C3R2::R &&
                  aligned16(u) && aligned16(v);
      return launch_3d<Mode::Apply, C3R2>(a, stream);
    }
    a.bulk_ok = per && (a.nx % 2 == 0) && a.nx >= C3R4::TX + 2 * C3R4::R && a.ny >= C3R4::TY + 2 * C3R4::R &&
                aligned16(u) && aligned16(v);
    if (per && is_l4l4(s)) {  // B = compose(L4, L4) on a periodic grid: two fused L4 passes possible
      if (option(SK_OPT_APPLY73_FACTORED)) {
        const int st = launch_fac73(a, pow_int(g.h, s->h_power / 2), stream);
        if (st != kApplyPqUnsupported) return st;
      }
    }
    if (a.bulk_ok && a.nx >= Cfg3R4P::TX + 2 * Cfg3R4P::R && a.ny >= Cfg3R4P::TY + 2 * Cfg3R4P::R)
      return launch_3d<Mode::Apply, Cfg3R4P>(a, stream);
    return launch_3d<Mode::Apply, C3R4>(a, stream);
  }
  return launch_generic(s, g, u, v, stream);
}

// Radius-4 apply from a ghost-padded field (matrix-free CG on non-periodic
// grids, sk_cg.cu): u_origin points at interior (0,0,0) of a layout with row
// pitch `pitch` and plane pitch `plane` whose halo (boundary zeros and the
// reflected / wrapped images, PadLayout) is filled, so the 16-byte loader
// runs without boundary maps. Same tile contents, hence the same bits, as
// the boundary-mapped loader. kApplyPqUnsupported: not applicable.
bool apply_padded_supported(const sk_stencil* s, const GridInfo& g) {
  return s->kclass == 3 && g.dim == 3 && streamable(s, g, 4) && g.un[0] >= Cfg3R4P::TX + 2 * Cfg3R4P::R &&
         g.un[1] >= Cfg3R4P::TY + 2 * Cfg3R4P::R;
}

int launch_apply_padded(const sk_stencil* s, const GridInfo& g, const double* u_origin, int64_t pitch,
                        int64_t plane, double* v, cudaStream_t stream, CgState* st, double* partials) {
  if (!apply_padded_supported(s, g)) return kApplyPqUnsupported;
  const bool pq = st != nullptr;
  const double scale = pow_int(g.h, s->h_power);
  Args3D a{};
  a.u = u_origin;
  a.v = v;
  a.nx = g.un[0];
  a.ny = g.un[1];
  a.nz = g.un[2];
  for (int i = 0; i < 3; ++i) a.bc[i] = g.bc[i];
  for (int i = 0; i < 8; ++i) a.w[i] = s->orbit_coeff[i] * scale;
  a.in_pitch = pitch;
  a.in_plane = plane;
  a.z_ghosted = 1;
  a.bulk_ok = (pitch % 2 == 0) && (plane % 2 == 0) && aligned16(u_origin) && aligned16(v) &&
              a.nx >= Cfg3R4P::TX + 2 * Cfg3R4P::R && a.ny >= Cfg3R4P::TY + 2 * Cfg3R4P::R &&
              plane * (a.nz + 8) < (int64_t(1) << 31);
  if (!a.bulk_ok) return kApplyPqUnsupported;
  // B = compose(L4, L4): the padded field holds every image the assembled
  // rows read (position-only reflections / wraps / zeros), so L4(L4 u_pad)
  // is the assembled operator exactly in rational arithmetic, as on a
  // periodic grid (rounding differs from the literal kernel)
  if (is_l4l4(s) && option(SK_OPT_APPLY73_FACTORED)) {
    a.cg = st;
    a.cg_partials = partials;
    const int r = pq ? launch_fac73<true>(a, pow_int(g.h, s->h_power / 2), stream)
                     : launch_fac73<false>(a, pow_int(g.h, s->h_power / 2), stream);
    if (r != kApplyPqUnsupported) return r;
  }
  if (pq) return kApplyPqUnsupported;  // the literal radius-4 kernel has no fused p.q (registers)
  return launch_3d<Mode::Apply, Cfg3R4P>(a, stream);
}

// Matrix-free CG: q = A p fused with p.q -> alpha (stream3d_kernel<..., PQ>)
// for the 3D streaming stencils; kApplyPqUnsupported: the caller runs the
// apply and a separate p.q pass. SK_OPT_CG_PQ = 0 disables it.
bool apply_pq_supported(const sk_stencil* s, const GridInfo& g) {
  // radius 2 only: the radius-4 kernel (234+ registers) slows down with the
  // epilogue (config 5 matrix-free: 0.457 -> 0.494 ms per iteration)
  return option(SK_OPT_CG_PQ) && g.dim == 3 && s->kclass == 2 && streamable(s, g, 2);
}

int launch_apply_pq(const sk_stencil* s, const GridInfo& g, const double* p, double* q, CgState* st,
                    double* partials, cudaStream_t stream) {
  if (!apply_pq_supported(s, g)) return kApplyPqUnsupported;
  const double scale = pow_int(g.h, s->h_power);
  const bool per = all_periodic(g);
  Args3D a{};
  a.u = p;
  a.v = q;
  a.nx = g.un[0];
  a.ny = g.un[1];
  a.nz = g.un[2];
  for (int i = 0; i < 3; ++i) a.bc[i] = g.bc[i];
  for (int i = 0; i < 8; ++i) a.w[i] = s->orbit_coeff[i] * scale;
  a.cg = st;
  a.cg_partials = partials;
  a.bulk_ok = per && (a.nx % 2 == 0) && a.nx >= C3R2::TX + 2 * C3R2::R && a.ny >= C3R2::TY + 2 * C3R2::R &&
              aligned16(p) && aligned16(q);
  return launch_3d<Mode::Apply, C3R2, true>(a, stream);
}

}  // namespace sk

using namespace sk;

extern "C" {

int sk_stencil_create(int dim, int nent, const int32_t* offsets, const double* coeff, int h_power,
                      sk_stencil** out) {
  if (!out) return fail(SK_ERR_INVALID_ARGUMENT, "null output handle");
  *out = nullptr;
  if (dim < 1 || dim > 3) return fail(SK_ERR_INVALID_ARGUMENT, "stencil dimension must be 1..3");
  if (nent < 0 || (nent > 0 && (!offsets || !coeff))) return fail(SK_ERR_INVALID_ARGUMENT, "bad entry arrays");
  // canonical form (stencil.cpp:15-28): lexicographic offsets, no zeros, never empty
  std::map<std::array<int, 3>, double> entries;
  for (int e = 0; e < nent; ++e) {
    std::array<int, 3> o{0, 0, 0};
    for (int a = 0; a < dim; ++a) o[a] = offsets[e * dim + a];
    if (entries.count(o)) return fail(SK_ERR_INVALID_ARGUMENT, "duplicate stencil offset");
    if (coeff[e] != 0.0) entries[o] = coeff[e];
  }
  if (entries.empty())
    return fail(SK_ERR_EMPTY_STENCIL, "all coefficients cancelled; empty stencil is not representable");
  auto* s = new sk_stencil;
  s->dim = dim;
  s->h_power = h_power;
  s->nent = static_cast<int>(entries.size());
  bool first = true;
  for (const auto& [o, c] : entries) {
    for (int a = 0; a < 3; ++a) {
      s->off.push_back(o[a]);
      if (first) {
        s->lo[a] = s->hi[a] = o[a];
      } else {
        s->lo[a] = std::min(s->lo[a], o[a]);
        s->hi[a] = std::max(s->hi[a], o[a]);
      }
    }
    s->coeff.push_back(c);
    first = false;
  }
  classify(s);
  cudaError_t e1 = cudaMalloc(&s->d_off, sizeof(int) * s->off.size());
  cudaError_t e2 = e1 == cudaSuccess ? cudaMalloc(&s->d_coeff, sizeof(double) * s->coeff.size()) : e1;
  if (e2 == cudaSuccess) e2 = cudaMemcpy(s->d_off, s->off.data(), sizeof(int) * s->off.size(), cudaMemcpyHostToDevice);
  if (e2 == cudaSuccess)
    e2 = cudaMemcpy(s->d_coeff, s->coeff.data(), sizeof(double) * s->coeff.size(), cudaMemcpyHostToDevice);
  if (e2 != cudaSuccess) {
    delete s;
    return cuda_fail(e2, "sk_stencil_create upload");
  }
  *out = s;
  return SK_OK;
}

int sk_stencil_destroy(sk_stencil* s) {
  delete s;
  return SK_OK;
}

int sk_stencil_kernel_class(const sk_stencil* s) { return s ? s->kclass : -1; }

int sk_composed_apply(const sk_stencil* s, const sk_grid_desc* gd, const double* u, double* v, void* stream) {
  if (!s) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  if (int st = check_width(s, g)) return st;
  if (g.rows > 0 && (!u || !v)) return fail(SK_ERR_INVALID_ARGUMENT, "null field pointer");
  if (u == v) return fail(SK_ERR_INVALID_ARGUMENT, "apply cannot run in place");
  return launch_apply(s, g, u, v, as_stream(stream));
}

int sk_composed_apply_repeat(const sk_stencil* s_c, const sk_grid_desc* gd, const double* u, double* v0,
                             double* v1, int repeats, void* stream_p) {
  auto* s = const_cast<sk_stencil*>(s_c);
  if (!s) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  if (int st = check_width(s, g)) return st;
  if (repeats < 0) return fail(SK_ERR_INVALID_ARGUMENT, "repeats must be >= 0");
  if (repeats == 0 || g.rows == 0) return SK_OK;
  if (!u || !v0 || !v1 || u == v0 || u == v1) return fail(SK_ERR_INVALID_ARGUMENT, "bad field pointers");
  cudaStream_t stream = as_stream(stream_p);
  sk_stencil::RepKey key;
  key.ptr[0] = u;
  key.ptr[1] = v0;
  key.ptr[2] = v1;
  key.repeats = repeats;
  key.dim = g.dim;
  for (int a = 0; a < 3; ++a) {
    key.n[a] = g.n[a];
    key.bc[a] = g.bc[a];
  }
  key.h = g.h;
  key.epoch = option_epoch();
  std::lock_guard<std::mutex> lock(s->rep_mu);
  if (!(s->rep_exec && s->rep_key == key)) {
    if (s->rep_exec) {
      cudaGraphExecDestroy(s->rep_exec);
      s->rep_exec = nullptr;
    }
    cudaStream_t cap = stream ? stream : capture_stream();
    SK_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    int st = SK_OK;
    const int64_t l0 = g_launches.load();
    for (int r = 0; r < repeats && st == SK_OK; ++r)
      st = launch_apply(s, g, u, (r % 2) ? v1 : v0, cap, /*input_stable=*/true);
    g_launches -= g_launches.load() - l0;  // capture does not execute; counted per replay below
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(cap, &graph);
    if (st != SK_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&s->rep_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    s->rep_key = key;
  }
  g_launches.fetch_add(repeats);  // the graph replays `repeats` kernels
  SK_CUDA_TRY(cudaGraphLaunch(s->rep_exec, stream));
  return SK_OK;
}

int sk_composed_apply_host(const sk_stencil* s, const sk_grid_desc* gd, const double* u_host, double* v_host) {
  if (!s) return fail(SK_ERR_INVALID_ARGUMENT, "null stencil");
  GridInfo g;
  if (int st = grid_info(gd, &g)) return st;
  if (int st = check_width(s, g)) return st;
  if (g.rows == 0) return SK_OK;
  if (!u_host || !v_host) return fail(SK_ERR_INVALID_ARGUMENT, "null host buffer");
  return host_roundtrip(u_host, size_t(g.rows), v_host, size_t(g.rows),
                        [&](const double* du, double* dv, cudaStream_t st) { return launch_apply(s, g, du, dv, st); });
}

}  // extern "C"
