// Library-wide plumbing: thread-local error string, version, int scans.
#include <stdarg.h>

#include <cub/device/device_scan.cuh>

#include "ni_common.cuh"

namespace ni {

static thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};
thread_local FillReport g_fill_report{};
thread_local int g_fill_profile = 0;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

size_t scan_ws_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return bytes + 512;
}

__global__ void total_kernel(const int32_t* in, const int32_t* out, int64_t n, int32_t* total) {
  if (n > 0) total[0] = out[n - 1] + in[n - 1];
  else total[0] = 0;
}

int exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, int32_t* total_dev, void* ws,
                       cudaStream_t s) {
  size_t bytes = scan_ws_bytes(n) - 512;
  if (n > 0) NI_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws, bytes, in, out, (int)n, s));
  if (total_dev) {
    NI_COUNT_LAUNCH(), total_kernel<<<1, 1, 0, s>>>(in, out, n, total_dev);
    NI_LAUNCH_CHECK();
  }
  return NI_OK;
}

}  // namespace ni

extern "C" const char* ni_last_error(void) { return ni::g_last_error.c_str(); }

extern "C" const char* ni_version(void) { return "normint_b200 0.1.0 (sm_100a)"; }

extern "C" long long ni_launch_count(void) { return ni::g_launches.load(); }

extern "C" int ni_fill_last_report(double* cg_ms, long long* px_iters, int* max_iters, int* grid,
                                   int* ntiles, int* npartials) {
  const ni::FillReport& r = ni::g_fill_report;
  if (cg_ms) *cg_ms = r.cg_ms;
  if (px_iters) *px_iters = r.px_iters;
  if (max_iters) *max_iters = r.max_iters;
  if (grid) *grid = r.grid;
  if (ntiles) *ntiles = r.ntiles;
  if (npartials) *npartials = r.npartials;
  return NI_OK;
}

extern "C" int ni_fill_mg_last_report(int* levels, int* vcycles, int* n_per_level) {
  const ni::FillReport& r = ni::g_fill_report;
  if (levels) *levels = r.mg_levels;
  if (vcycles) *vcycles = r.mg_vcycles;
  if (n_per_level)
    for (int l = 0; l < 16; ++l) n_per_level[l] = r.mg_n[l];
  return NI_OK;
}

extern "C" int ni_set_fill_profiling(int on) {
  ni::g_fill_profile = on != 0;
  return NI_OK;
}

extern "C" int ni_fill_mg_last_profile(double* ms4, long long* px_vcycles) {
  const ni::FillReport& r = ni::g_fill_report;
  if (ms4)
    for (int k = 0; k < 4; ++k) ms4[k] = r.mg_ms[k];
  if (px_vcycles) *px_vcycles = r.mg_px_vcycles;
  return NI_OK;
}
