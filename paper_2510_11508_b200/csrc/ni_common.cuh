// Shared helpers for the normint_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <string>

#include "../../include/normint_b200.h"

namespace ni {

// ---------------------------------------------------------------- errors

void set_error(const char* fmt, ...);

// Host-side count of this library's kernel launches (ni_launch_count()).
extern std::atomic<long long> g_launches;
#define NI_COUNT_LAUNCH() (::ni::g_launches.fetch_add(1, std::memory_order_relaxed))

// Diagnostics of the last ni_fill on this thread (ni_fill_last_report()).
struct FillReport {
  double cg_ms;        // device time of the persistent CG kernel (CUDA events)
  long long px_iters;  // sum over components of size * CG iterations
  int max_iters;       // largest per-component iteration count
  int grid;            // CTAs of the cooperative launch
  int ntiles;          // 32x32 tiles of the grid
  int npartials;       // (tile, component) partial slots
  int mg_levels;       // multigrid fill: coarse levels used
  int mg_vcycles;      // multigrid fill: V-cycles (PCG iterations + 1 of the longest unit)
  int mg_n[16];        // multigrid fill: unknowns per level (index 1..levels)
  // multigrid fill, filled only while profiling is on (ni_set_fill_profiling):
  // CUDA-event time summed over the V-cycles of pass A, the coarse levels,
  // pass B and the per-unit scalar step, and the active unit pixels summed
  // over V-cycles (the algorithmic work of the fine passes)
  double mg_ms[4];
  long long mg_px_vcycles;
};
extern thread_local int g_fill_profile;
extern thread_local FillReport g_fill_report;

#define NI_CUDA_TRY(expr)                                                              \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ::ni::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return NI_ERR_CUDA;                                                              \
    }                                                                                  \
  } while (0)

#define NI_LAUNCH_CHECK()                                                               \
  do {                                                                                  \
    cudaError_t _e = cudaGetLastError();                                                \
    if (_e != cudaSuccess) {                                                            \
      ::ni::set_error("%s:%d kernel launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return NI_ERR_CUDA;                                                               \
    }                                                                                   \
  } while (0)

// an environment knob read once per process (experiment switches; never per call)
#define NI_ENV_ONCE(name) ([] { static const char* v_ = getenv(name); return v_; }())

#define NI_CHECK_ARG(cond, msg)              \
  do {                                       \
    if (!(cond)) {                           \
      ::ni::set_error("invalid argument: %s", msg); \
      return NI_ERR_INVALID_ARG;             \
    }                                        \
  } while (0)

#define NI_TRY(expr)           \
  do {                         \
    int _s = (expr);           \
    if (_s != NI_OK) return _s; \
  } while (0)

// ------------------------------------------------------------ workspace

// Bump allocator over the caller's workspace; every carve is 256-B aligned.
struct Carver {
  char* base;
  size_t cap;
  size_t used = 0;
  Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <class T>
  T* take(size_t n) {
    size_t off = (used + 255) & ~size_t(255);
    used = off + n * sizeof(T);
    return reinterpret_cast<T*>(base ? base + off : nullptr);
  }
  bool ok() const { return used <= cap; }
};

// Size-only pass of a Carver (base = nullptr).
struct Sizer : Carver {
  Sizer() : Carver(nullptr, 0) {}
};

// ------------------------------------------------------------- the grid

struct Grid {
  int B, H, W, conn;
  int kf;        // forward edges per pixel (2 or 4)
  int64_t npix;  // B*H*W
};

inline Grid make_grid(int B, int H, int W, int conn) {
  Grid g;
  g.B = B;
  g.H = H;
  g.W = W;
  g.conn = conn;
  g.kf = conn == 8 ? 4 : 2;
  g.npix = int64_t(B) * H * W;
  return g;
}

// Forward offsets (graph.py:24-25), indexed by k.
__host__ __device__ __forceinline__ int fwd_du(int conn, int k) {
  return conn == 8 ? (k == 0 ? 1 : (k == 1 ? -1 : (k == 2 ? 0 : 1))) : (k == 0 ? 1 : 0);
}
__host__ __device__ __forceinline__ int fwd_dv(int conn, int k) {
  return conn == 8 ? (k == 0 ? 0 : 1) : (k == 0 ? 0 : 1);
}

// Does the forward neighbour (u+du, v+dv) of (u, v) lie in the same map?
// v is the row inside the map (0..H-1).
__device__ __forceinline__ bool fwd_inside(int u, int vloc, int du, int dv, int W, int H) {
  int uu = u + du;
  return uu >= 0 && uu < W && vloc + dv < H;
}

// -------------------------------------------------------------- numerics

// IEEE round-to-nearest products/sums, never contracted into FMA: these
// reproduce numpy's float64 results bit for bit.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum in a fixed order (deterministic).  `scratch` holds >= 32 doubles.
// Result valid in every thread.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = lane < nw ? scratch[lane] : 0.0;
  t = warp_sum(t);
  return t;
}

inline int div_up(int64_t a, int64_t b) { return int((a + b - 1) / b); }

constexpr int kSMs = 148;

// Exclusive scan of int32 values (n up to 2^31-1); workspace from scan_ws().
size_t scan_ws_bytes(int64_t n);
int exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, int32_t* total_dev, void* ws,
                       cudaStream_t s);

// Lock-free union-find over int32 parents: parent[x] <= x, roots hooked
// under the smaller id (so a flattened root is the smallest member).
__device__ __forceinline__ int uf_find(volatile int32_t* parent, int32_t x) {
  int32_t p = parent[x];
  while (p != x) {
    x = p;
    p = parent[x];
  }
  return x;
}

// Find with path halving: every visited node is re-pointed to its
// grandparent (an ancestor with a smaller id, so parent[x] <= x still holds
// and a concurrent hook is never lost: its union is retried from the old root).
__device__ __forceinline__ int uf_find_halve(volatile int32_t* parent, int32_t x) {
  int32_t p = parent[x];
  while (p != x) {
    const int32_t gp = parent[p];
    if (gp != p) parent[x] = gp;
    x = gp;
    p = parent[x];
  }
  return x;
}

// Union by hooking the larger root under the smaller one (atomicMin), retried
// until both endpoints share a root.  parent[x] <= x always holds.
__device__ __forceinline__ void uf_union(int32_t* parent, int32_t a, int32_t b) {
  volatile int32_t* vp = parent;
  while (true) {
    a = uf_find_halve(vp, a);
    b = uf_find_halve(vp, b);
    if (a == b) return;
    if (a < b) {
      int32_t t = a;
      a = b;
      b = t;
    }
    // a > b: try to hook root a under b
    int32_t old = atomicMin(parent + a, b);
    if (old == a) return;
    a = old;
  }
}

}  // namespace ni
