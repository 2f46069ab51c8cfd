// Shared device/host helpers for libgnnb200 (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gnn_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libgnnb200 targets sm_100a only"
#endif

namespace gnn {

constexpr unsigned kFull = 0xffffffffu;

// Last CUDA error seen by a GNN_ERR_CUDA return (per process; informative only).
void set_cuda_error(cudaError_t e);

#define GNN_CUDA_TRY(expr)                     \
  do {                                         \
    cudaError_t _e = (expr);                   \
    if (_e != cudaSuccess) {                   \
      ::gnn::set_cuda_error(_e);               \
      return GNN_ERR_CUDA;                     \
    }                                          \
  } while (0)

// Every kernel launch is followed by GNN_LAUNCH_CHECK(), which also bumps the
// process-wide launch counter (gnn_launch_counter()).
void note_launch();
#define GNN_LAUNCH_CHECK()                    \
  do {                                        \
    ::gnn::note_launch();                     \
    GNN_CUDA_TRY(cudaGetLastError());         \
  } while (0)

#define GNN_TRY(expr)        \
  do {                       \
    int _s = (expr);         \
    if (_s != GNN_OK) return _s; \
  } while (0)

inline cudaStream_t as_stream(gnn_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline size_t align_up(size_t a, size_t b) { return (a + b - 1) / b * b; }

// Bump allocator over a caller-provided workspace.
struct WsArena {
  char *base;
  size_t cap;
  size_t used = 0;
  WsArena(void *b, size_t c) : base(static_cast<char *>(b)), cap(c) {}
  template <class T>
  T *take(int64_t count) {
    size_t off = align_up(used, 256);
    size_t bytes = static_cast<size_t>(count > 0 ? count : 0) * sizeof(T);
    used = off + bytes;
    return reinterpret_cast<T *>(base + off);
  }
  bool ok() const { return used <= cap; }
};

// Size-only twin of WsArena for *_workspace() queries.
struct WsCounter {
  size_t used = 0;
  template <class T>
  void take(int64_t count) {
    used = align_up(used, 256) + static_cast<size_t>(count > 0 ? count : 0) * sizeof(T);
  }
};

int sm_count();

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Read-only, L1-allocating 128-bit gather (feature rows are reused across edges).
__device__ __forceinline__ float4 ldg_f4(const float *p) {
  return __ldg(reinterpret_cast<const float4 *>(p));
}
// Streaming loads for data touched once (index arrays).
__device__ __forceinline__ int ld_stream_i32(const int32_t *p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Packed fp32 pair arithmetic (sm_100 FADD2 / FFMA2): two lanes of a float4 per instruction.
__device__ __forceinline__ unsigned long long f2_bits(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ void f2_unbits(unsigned long long b, float &lo, float &hi) {
  lo = __uint_as_float((unsigned)(b & 0xffffffffull));
  hi = __uint_as_float((unsigned)(b >> 32));
}
__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  unsigned long long r0, r1;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r0) : "l"(f2_bits(a.x, a.y)), "l"(f2_bits(b.x, b.y)));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r1) : "l"(f2_bits(a.z, a.w)), "l"(f2_bits(b.z, b.w)));
  float4 o;
  f2_unbits(r0, o.x, o.y);
  f2_unbits(r1, o.z, o.w);
  return o;
}
// a + s * b
__device__ __forceinline__ float4 f4_fma(float s, float4 b, float4 a) {
  unsigned long long r0, r1, ss = f2_bits(s, s);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r0) : "l"(ss), "l"(f2_bits(b.x, b.y)), "l"(f2_bits(a.x, a.y)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r1) : "l"(ss), "l"(f2_bits(b.z, b.w)), "l"(f2_bits(a.z, a.w)));
  float4 o;
  f2_unbits(r0, o.x, o.y);
  f2_unbits(r1, o.z, o.w);
  return o;
}

// First index i in [lo,hi) with a[i] > x (upper bound), a nondecreasing.
template <class T>
__device__ __forceinline__ int64_t upper_bound_dev(const T *a, int64_t lo, int64_t hi, T x) {
  while (lo < hi) {
    int64_t mid = lo + ((hi - lo) >> 1);
    if (a[mid] <= x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
// First index i in [lo,hi) with a[i] >= x (lower bound).
template <class T>
__device__ __forceinline__ int64_t lower_bound_dev(const T *a, int64_t lo, int64_t hi, T x) {
  while (lo < hi) {
    int64_t mid = lo + ((hi - lo) >> 1);
    if (a[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// ---- device-wide primitives (scan.cu) ----
// Exclusive scan of int64 values: out[i] = sum_{j<i} in[i]; out[n] = total if out has n+1 slots
// (write_total). in and out may alias.
size_t scan_i64_workspace(int64_t n);
int exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, bool write_total, void *ws,
                       size_t ws_bytes, cudaStream_t st);
size_t scan_u32_workspace(int64_t n);
int exclusive_scan_u32(const uint32_t *in, uint32_t *out, int64_t n, void *ws, size_t ws_bytes,
                       cudaStream_t st);

}  // namespace gnn

// ---- mbarrier + 1-D bulk async copy (TMA engine, cp.async.bulk) ----------
namespace gnn {
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing on an mbarrier; bytes % 16 == 0, both addresses 16B aligned
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace gnn
