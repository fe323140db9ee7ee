// Standalone check of the TMA + mbarrier sequence used by ni_fill.cu.
// usage: tma_probe <variant>   (each variant in its own process)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

struct Args {
  CUtensorMap tm[2];
  float* out;
  int variant;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void probe(const __grid_constant__ Args a, int par, const CUtensorMap* gmap) {
  __shared__ __align__(128) float buf[8][32];
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x;
  const int v = a.variant;
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
  if (v != 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (v != 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (lane == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1024) : "memory");
    const CUtensorMap* m = (v == 4) ? gmap : &a.tm[par];
    int cx = -1, cy = -1;
    if (v == 3) cx = cy = 0;
    if (v == 6) { cx = 16; cy = 0; }
    if (v == 7) { cx = 0; cy = 16; }
    if (v == 8) { cx = -1; cy = 0; }
    if (v == 9) { cx = 0; cy = -1; }
    if (v == 10) { cx = 8; cy = 4; }
    if (v == 11) { cx = 0; cy = 40; }
    if (v == 12) { cx = 48; cy = 0; }
    if (v == 13) { cx = 30; cy = 0; }
    if (v == 14) { cx = 0; cy = 19; }
    if (v == 15) { cx = 39; cy = 0; }
    if (v == 16) { cx = 40; cy = 0; }
    if (v == 5) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(buf)), "l"(m), "r"(smem_u32(&bar)), "r"(cx), "r"(cy)
          : "memory");
    } else {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(buf)), "l"(m), "r"(smem_u32(&bar)), "r"(cx), "r"(cy)
          : "memory");
    }
  }
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(&bar)),
      "r"(0) : "memory");
  for (int r = 0; r < 8; ++r) a.out[r * 32 + lane] = buf[r][lane];
}

__global__ void probe2(const __grid_constant__ Args a, int cx, int cy, int bytes) {
  __shared__ __align__(128) float buf[8][64];
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x;
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (lane == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(buf)), "l"(&a.tm[0]), "r"(smem_u32(&bar)), "r"(cx), "r"(cy)
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(&bar)),
      "r"(0) : "memory");
  a.out[lane] = buf[0][lane];
}

int main(int argc, char** argv) {
  if (argc > 3) {
    const int cx = atoi(argv[1]), cy = atoi(argv[2]), bw = atoi(argv[3]);
    const int u8 = argc > 4 ? atoi(argv[4]) : 0;
    const int W = 100, H = 20, P = 112;
    float *d, *o;
    cudaMalloc(&d, H * P * 4);
    cudaMalloc(&o, 1024);
    cudaMemset(d, 0, H * P * 4);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled)fn;
    Args a;
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
    cuuint64_t str[1] = {(cuuint64_t)P * 4};
    cuuint32_t box[2] = {(cuuint32_t)bw, 8};
    cuuint32_t es[2] = {1, 1};
    if (u8) str[0] = P;
    CUresult r = enc(&a.tm[0], u8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    a.out = o;
    probe2<<<1, 32>>>(a, cx, cy, bw * 8 * (u8 ? 1 : 4));
    cudaError_t e = cudaDeviceSynchronize();
    printf("cx=%d cy=%d boxw=%d u8=%d encode=%d: %s\n", cx, cy, bw, u8, (int)r, cudaGetErrorString(e));
    return e != cudaSuccess;
  }
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  const int W = 40, H = 20, P = 48;
  std::vector<float> h(H * P);
  for (int y = 0; y < H; ++y) for (int x = 0; x < P; ++x) h[y * P + x] = y * 100 + x;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, 256 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled)fn;
  Args a;
  cuuint64_t dims[2] = {W, H};
  cuuint64_t str[1] = {P * 4};
  cuuint32_t box[2] = {32, 8};
  cuuint32_t es[2] = {1, 1};
  for (int i = 0; i < 2; ++i)
    enc(&a.tm[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, getenv("L2NONE") ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* gm;
  cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(gm, &a.tm[1], sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  a.out = o;
  a.variant = v;
  cudaMemset(o, 0xff, 1024);
  probe<<<1, 32>>>(a, 1, gm);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> got(256);
  cudaMemcpy(got.data(), o, 1024, cudaMemcpyDeviceToHost);
  printf("variant %d: %s  out[0]=%g out[1]=%g out[33]=%g out[40]=%g\n", v, cudaGetErrorString(e), got[0], got[1], got[33], got[40]);
  return e != cudaSuccess;
}
