// Memory-system probe for the fill sweep's access pattern (no CG math):
// every warp streams "items" of 32 rows x 32 float4 columns (+ a float and a
// byte plane) through a cp.async shared-memory ring and writes 30 float4 per
// row, like fill_cg_kernel.  Compares row-major strips (pitch P) against a
// tile-major layout (each item's rows contiguous) and a plain copy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NS = 8, WPB = 8, NT = 256;

__device__ __forceinline__ uint32_t s32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cpa(uint32_t d, const void* s, bool on) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.cg.shared.global [%0], [%1], 16;\n}\n"
               ::"r"(d), "l"(s), "r"(int(on)) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// mode 0: row-major, item (sx, sy) rows at (sy*30 + j) * P + sx*30 (+16 margin)
// mode 1: tile-major, item k rows at k*32*32 + j*32
__global__ void __launch_bounds__(NT, 2) probe(const float4* __restrict__ vin, float4* __restrict__ vout,
                                               const float* __restrict__ hw, int P, int nsx, int nitems,
                                               int mode, int* ticket, float* sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31;
  unsigned char* ring = sm + (threadIdx.x >> 5) * NS * 656;
  const uint32_t rs = s32(ring);
  float accum = 0.f;
  for (;;) {
    int k = 0;
    if (lane == 0) k = atomicAdd(ticket, 1);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= nitems) break;
    int64_t base, pitch;
    if (mode == 0) {
      const int sx = k % nsx, sy = k / nsx;
      base = int64_t(sy * 30) * P + sx * 30;
      pitch = P;
    } else {
      base = int64_t(k) * 32 * 32;
      pitch = 32;
    }
    const float4* src = vin + base + lane;
    const float* hsrc = hw + (base & ~int64_t(3)) + 4 * (lane < 9 ? lane : 0);
    for (int j = 0; j < NS - 2; ++j) {
      cpa(rs + (j & (NS - 1)) * 656 + 16 * lane, src + j * pitch, true);
      cpa(rs + (j & (NS - 1)) * 656 + 512 + 16 * lane, hsrc + j * pitch, lane < 9);
      commit();
    }
    for (int j = 0; j < 32; ++j) {
      const int jj = j + NS - 2;
      cpa(rs + (jj & (NS - 1)) * 656 + 16 * lane, src + jj * pitch, jj < 32);
      cpa(rs + (jj & (NS - 1)) * 656 + 512 + 16 * lane, hsrc + jj * pitch, jj < 32 && lane < 9);
      commit();
      waitg<NS - 2>();
      __syncwarp();
      const float4 v = *reinterpret_cast<const float4*>(ring + (j & (NS - 1)) * 656 + 16 * lane);
      const float h = *reinterpret_cast<const float*>(ring + (j & (NS - 1)) * 656 + 512 + 4 * lane);
      const float pl = __shfl_up_sync(0xffffffffu, v.z, 1);
      const float4 o = make_float4(v.x + h, v.y - pl, v.z * 1.0001f, v.w + 1.f);
      if (lane >= 1 && lane <= 30 && j >= 1 && j <= 30) vout[base + j * pitch + lane] = o;
      accum += o.x;
    }
    waitg<0>();
  }
  if (accum == 12345.f) *sink = accum;
}

__global__ void copyk(const float4* __restrict__ a, float4* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    b[i] = a[i];
}

int main() {
  const int W = 1024, H = 16 * 1060, P = 1104;
  const int nsx = (W + 29) / 30, nsy = (H - 2) / 30;
  const int nitems = nsx * nsy;
  const int64_t n_rm = int64_t(H + 40) * P, n_tm = int64_t(nitems) * 1024;
  const int64_t n = n_rm > n_tm ? n_rm : n_tm;
  float4 *a, *b;
  float* hw;
  int* tk;
  float* sink;
  cudaMalloc(&a, n * 16);
  cudaMalloc(&b, n * 16);
  cudaMalloc(&hw, n * 4);
  cudaMalloc(&tk, 4);
  cudaMalloc(&sink, 4);
  cudaMemset(a, 0, n * 16);
  cudaMemset(b, 0, n * 16);
  cudaMemset(hw, 0, n * 4);
  const size_t smem = size_t(WPB) * NS * 656;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(tk, 0, 4);
      cudaEventRecord(e0);
      if (mode < 2)
        probe<<<148 * 2, NT, smem>>>(a, b, hw, P, nsx, nitems, mode, tk, sink);
      else
        copyk<<<148 * 8, 256>>>(a, b, n_rm);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    // algorithmic bytes: probe: per item 32 rows x (512 + 144) read + 30 x 480 written
    const double bytes = mode < 2 ? double(nitems) * (32.0 * (512 + 144) + 30.0 * 480)
                                  : double(n_rm) * 32.0;
    printf("mode %d (%s): %.3f ms  %.1f GB/s  err=%s\n", mode,
           mode == 0 ? "row-major strips" : mode == 1 ? "tile-major" : "copy", best, bytes / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
