// Library plumbing: error state, grid validation, memory/stream helpers.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <utility>

#include "sk_common.cuh"

namespace sk {

namespace {
thread_local std::string t_err;
}

std::atomic<int64_t> g_launches{0};

namespace {
// sk_set_option values (include/sk_cuda.h enum sk_option order); defaults
// are the measured-fastest paths
std::atomic<int> g_options[SK_OPT_COUNT] = {1, 1, 1, 1, -1, 1, 1, 1, 1, 1};
std::atomic<uint64_t> g_option_epoch{0};
}  // namespace

int option(int id) { return g_options[id].load(std::memory_order_relaxed); }
uint64_t option_epoch() { return g_option_epoch.load(std::memory_order_relaxed); }

void set_error(int status, const std::string& msg) {
  t_err = std::string(sk_status_name(status)) + ": " + msg;
}

int fail(int status, const std::string& msg) {
  set_error(status, msg);
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  int st = e == cudaErrorMemoryAllocation ? SK_ERR_OUT_OF_MEMORY
           : (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) ? SK_ERR_NO_DEVICE
                                                                           : SK_ERR_CUDA;
  set_error(st, std::string(what) + " -> " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  return st;
}

double pow_int(double base, int exp) {  // grid.cpp:10-15
  if (exp < 0) return 1.0 / pow_int(base, -exp);
  double r = 1.0;
  for (int k = 0; k < exp; ++k) r *= base;
  return r;
}

// GridSpec::validate (grid.cpp:17-25) + unknowns_per_axis / unknown_count (:27-35)
int grid_info(const sk_grid_desc* g, GridInfo* out) {
  if (!g) return fail(SK_ERR_INVALID_ARGUMENT, "null grid descriptor");
  if (g->dim < 1 || g->dim > 3) return fail(SK_ERR_INVALID_ARGUMENT, "grid dimension must be 1..3");
  GridInfo gi{};
  gi.dim = g->dim;
  gi.h = g->h;
  gi.rows = 1;
  for (int a = 0; a < 3; ++a) {
    if (a < g->dim) {
      if (g->n[a] < 3) return fail(SK_ERR_INVALID_ARGUMENT, "grid needs at least 3 points per axis");
      if (g->bc[a] < SK_BC_PERIODIC || g->bc[a] > SK_BC_CLAMPED)
        return fail(SK_ERR_INVALID_ARGUMENT, "unknown boundary kind");
      gi.n[a] = g->n[a];
      gi.bc[a] = g->bc[a];
      gi.un[a] = g->bc[a] == SK_BC_PERIODIC ? g->n[a] : g->n[a] - 2;
    } else {
      gi.n[a] = 1;
      gi.un[a] = 1;
      gi.bc[a] = SK_BC_PERIODIC;
    }
    gi.rows *= gi.un[a];
  }
  if (!(g->h > 0)) return fail(SK_ERR_INVALID_ARGUMENT, "grid spacing must be positive");
  *out = gi;
  return SK_OK;
}

}  // namespace sk

using namespace sk;

extern "C" {

const char* sk_last_error(void) { return t_err.c_str(); }

const char* sk_status_name(int s) {
  switch (s) {  // error.hpp:43-63 names
    case SK_OK: return "Ok";
    case SK_ERR_ZERO_SCALE: return "ZeroScale";
    case SK_ERR_DIM_MISMATCH: return "DimMismatch";
    case SK_ERR_POWER_MISMATCH: return "PowerMismatch";
    case SK_ERR_EMPTY_STENCIL: return "EmptyStencil";
    case SK_ERR_TRUNCATION_TOO_SMALL: return "TruncationTooSmall";
    case SK_ERR_NOT_NORMALIZED: return "NotNormalized";
    case SK_ERR_ACCURACY_EXCEEDS_TRUNCATION: return "AccuracyExceedsTruncation";
    case SK_ERR_MIXED_LEADING_ORDER: return "MixedLeadingOrder";
    case SK_ERR_SINGULAR_SYSTEM: return "SingularSystem";
    case SK_ERR_UNSUPPORTED_ACCURACY: return "UnsupportedAccuracy";
    case SK_ERR_STENCIL_WIDER_THAN_GRID: return "StencilWiderThanGrid";
    case SK_ERR_SHAPE_MISMATCH: return "ShapeMismatch";
    case SK_ERR_NO_CONVERGENCE: return "NoConvergence";
    case SK_ERR_NOT_DISSIPATIVE: return "NotDissipative";
    case SK_ERR_UNSTABLE_FOR_ALL_DT: return "UnstableForAllDt";
    case SK_ERR_NON_PERIODIC: return "NonPeriodic";
    case SK_ERR_ZERO_DENOMINATOR: return "ZeroDenominator";
    case SK_ERR_INVALID_ARGUMENT: return "InvalidArgument";
    case SK_ERR_CUDA: return "CudaError";
    case SK_ERR_OUT_OF_MEMORY: return "OutOfMemory";
    case SK_ERR_NO_DEVICE: return "NoDevice";
  }
  return "UnknownError";
}

int sk_version(void) { return 2; }

int sk_set_option(int opt, int value) {
  if (opt < 0 || opt >= SK_OPT_COUNT) return fail(SK_ERR_INVALID_ARGUMENT, "unknown option");
  const int lo = opt == SK_OPT_CG_COOP ? -1 : 0;
  if (value < lo || value > 1) return fail(SK_ERR_INVALID_ARGUMENT, "option value out of range");
  if (g_options[opt].exchange(value) != value) g_option_epoch.fetch_add(1);
  return SK_OK;
}

int sk_get_option(int opt, int* value) {
  if (opt < 0 || opt >= SK_OPT_COUNT) return fail(SK_ERR_INVALID_ARGUMENT, "unknown option");
  if (!value) return fail(SK_ERR_INVALID_ARGUMENT, "null output pointer");
  *value = g_options[opt].load();
  return SK_OK;
}

int64_t sk_launch_count(void) { return g_launches.load(); }

int sk_device_init(int device) {
  int count = 0;
  SK_CUDA_TRY(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return fail(SK_ERR_NO_DEVICE, "device ordinal out of range");
  SK_CUDA_TRY(cudaSetDevice(device));
  SK_CUDA_TRY(cudaFree(nullptr));
  // keep stream-ordered scratch in the pool between calls (no OS round trips)
  cudaMemPool_t pool;
  SK_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t keep = UINT64_MAX;
  SK_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  return SK_OK;
}

int sk_device_alloc(size_t bytes, void** out) {
  if (!out) return fail(SK_ERR_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  if (bytes == 0) return SK_OK;
  SK_CUDA_TRY(cudaMalloc(out, bytes));
  return SK_OK;
}

int sk_device_free(void* p) {
  if (p) SK_CUDA_TRY(cudaFree(p));
  return SK_OK;
}

int sk_ipc_get_handle(const void* base, unsigned char handle_out[64]) {
  if (!base || !handle_out) return fail(SK_ERR_INVALID_ARGUMENT, "null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  SK_CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(base)));
  std::memcpy(handle_out, &h, 64);
  return SK_OK;
}

int sk_ipc_open_handle(const unsigned char handle[64], void** base_out) {
  if (!handle || !base_out) return fail(SK_ERR_INVALID_ARGUMENT, "null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  *base_out = nullptr;
  SK_CUDA_TRY(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
  return SK_OK;
}

int sk_ipc_close_handle(void* base) {
  if (base) SK_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return SK_OK;
}

int sk_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return SK_OK;
  SK_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream)));
  return SK_OK;
}

int sk_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return SK_OK;
  SK_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
  SK_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  return SK_OK;
}

int sk_stream_sync(void* stream) {
  SK_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  return SK_OK;
}

int sk_stream_create(void** out) {
  if (!out) return fail(SK_ERR_INVALID_ARGUMENT, "null output pointer");
  cudaStream_t s = nullptr;
  SK_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = s;
  return SK_OK;
}

int sk_stream_destroy(void* stream) {
  if (stream) SK_CUDA_TRY(cudaStreamDestroy(as_stream(stream)));
  return SK_OK;
}

int sk_host_register(void* p, size_t bytes) {
  if (!p || bytes == 0) return fail(SK_ERR_INVALID_ARGUMENT, "bad host buffer");
  SK_CUDA_TRY(cudaHostRegister(p, bytes, cudaHostRegisterDefault));
  return SK_OK;
}

int sk_host_unregister(void* p) {
  SK_CUDA_TRY(cudaHostUnregister(p));
  return SK_OK;
}

int sk_event_create(void** ev) {
  if (!ev) return fail(SK_ERR_INVALID_ARGUMENT, "null event");
  cudaEvent_t e;
  SK_CUDA_TRY(cudaEventCreate(&e));
  *ev = e;
  return SK_OK;
}

int sk_event_destroy(void* ev) {
  if (ev) SK_CUDA_TRY(cudaEventDestroy(static_cast<cudaEvent_t>(ev)));
  return SK_OK;
}

int sk_event_record(void* ev, void* stream) {
  SK_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(ev), as_stream(stream)));
  return SK_OK;
}

int sk_event_elapsed_ms(void* a, void* b, float* ms) {
  SK_CUDA_TRY(cudaEventSynchronize(static_cast<cudaEvent_t>(b)));
  SK_CUDA_TRY(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)));
  return SK_OK;
}

int sk_l2_flush(void* stream) {
  static void* buf = nullptr;
  const size_t bytes = size_t(512) << 20;  // 512 MiB > 126 MB L2
  if (!buf) SK_CUDA_TRY(cudaMalloc(&buf, bytes));
  SK_CUDA_TRY(cudaMemsetAsync(buf, 0, bytes, as_stream(stream)));
  return SK_OK;
}

int sk_fill_uniform_host(uint64_t seed, int64_t count, double lo, double hi, double* out) {
  if (count < 0 || (count > 0 && !out)) return fail(SK_ERR_INVALID_ARGUMENT, "bad output buffer");
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(lo, hi);
  for (int64_t i = 0; i < count; ++i) out[i] = unit(rng);
  return SK_OK;
}

}  // extern "C"
