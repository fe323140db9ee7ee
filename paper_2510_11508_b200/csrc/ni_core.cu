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

// ---- read-back through the SMs (serving stream, pipeline.py's
// run_pipeline_stream): a device -> pinned-host copy done by a small kernel
// storing into mapped host memory instead of by a copy engine.  A copy-engine
// read-back of a whole batch (~0.5 GB, ~10 ms) holds the device->host queue,
// so every small control read of the next batch's pipeline (.cpu() of counts
// and flags) waits behind it; the kernel's posted PCIe writes leave that queue
// free.  Each thread moves 16-byte vectors, 4 in flight.
namespace ni {
__global__ void __launch_bounds__(512) d2h_mapped_kernel(const uint4* __restrict__ src,
                                                         uint4* __restrict__ dst, int64_t n16) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    const uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
                d = __ldcs(src + i + 3 * stride);
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = __ldcs(src + i);
}
__global__ void d2h_mapped_tail_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                       int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}
}  // namespace ni

// one implementation for both directions: `host` is the pinned (mapped) side
static int mapped_copy(const void* dev, void* host, size_t bytes, int ctas, ni_stream_t stream,
                       bool to_host, const char* who) {
  if (!dev || !host) {
    ni::set_error("invalid argument: null pointer");
    return NI_ERR_INVALID_ARG;
  }
  NI_CHECK_ARG(ctas > 0 && ctas <= 4096, "ctas must be in 1..4096");
  if (bytes == 0) return NI_OK;
  void* hptr = nullptr;
  // pinned host memory (cudaHostAlloc / cudaHostRegister) is mapped under UVA
  if (cudaHostGetDevicePointer(&hptr, host, 0) != cudaSuccess || !hptr) {
    cudaGetLastError();
    ni::set_error("%s: the host buffer is not pinned (mapped) host memory", who);
    return NI_ERR_INVALID_ARG;
  }
  NI_CHECK_ARG((reinterpret_cast<uintptr_t>(dev) & 15) == (reinterpret_cast<uintptr_t>(hptr) & 15),
               "source and destination must share their 16-byte alignment");
  cudaStream_t s = (cudaStream_t)stream;
  const auto* s8 = static_cast<const uint8_t*>(to_host ? dev : hptr);
  auto* d8 = static_cast<uint8_t*>(to_host ? hptr : const_cast<void*>(dev));
  const uintptr_t mis = reinterpret_cast<uintptr_t>(s8) & 15;
  size_t head = mis ? (16 - mis) : 0;
  if (head > bytes) head = bytes;
  if (head) {
    NI_COUNT_LAUNCH(), ni::d2h_mapped_tail_kernel<<<1, 16, 0, s>>>(s8, d8, int64_t(head));
    NI_LAUNCH_CHECK();
  }
  const int64_t n16 = int64_t((bytes - head) / 16);
  if (n16) {
    NI_COUNT_LAUNCH(), ni::d2h_mapped_kernel<<<ctas, 512, 0, s>>>(
        reinterpret_cast<const uint4*>(s8 + head), reinterpret_cast<uint4*>(d8 + head), n16);
    NI_LAUNCH_CHECK();
  }
  const size_t done = head + size_t(n16) * 16;
  if (done < bytes) {
    NI_COUNT_LAUNCH(), ni::d2h_mapped_tail_kernel<<<1, 16, 0, s>>>(s8 + done, d8 + done,
                                                                  int64_t(bytes - done));
    NI_LAUNCH_CHECK();
  }
  return NI_OK;
}

extern "C" int ni_copy_to_host(const void* src, void* host_dst, size_t bytes, int ctas,
                               ni_stream_t stream) {
  return mapped_copy(src, host_dst, bytes, ctas, stream, true, "ni_copy_to_host");
}

// The upload twin: a small kernel reads mapped pinned host memory and stores
// into device memory (serving stream: the next batch's normals + mask while the
// current batch computes).
extern "C" int ni_copy_from_host(void* dst, const void* host_src, size_t bytes, int ctas,
                                 ni_stream_t stream) {
  return mapped_copy(dst, const_cast<void*>(host_src), bytes, ctas, stream, false,
                     "ni_copy_from_host");
}
