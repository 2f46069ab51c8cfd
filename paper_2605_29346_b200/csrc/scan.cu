// Device-wide exclusive scans (reduce-then-scan, three launches, deterministic).
// Used for CSR offsets (degree prefix sums, graph.py:110-112) and for the
// radix-sort digit-count tables.
#include "common.cuh"

namespace gnn {
namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(kFull, v, o);
    if ((int)lane_id() >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the block total in *total.
template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T *smem_warp, T *total) {
  const int w = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane_id() == 31) smem_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = (lane_id() < kScanThreads / 32) ? smem_warp[lane_id()] : T(0);
    T si = warp_incl_scan(s);
    if (lane_id() < kScanThreads / 32) smem_warp[lane_id()] = si - s;
    if (lane_id() == kScanThreads / 32 - 1) smem_warp[kScanThreads / 32] = si;
  }
  __syncthreads();
  T r = smem_warp[w] + inc - v;
  *total = smem_warp[kScanThreads / 32];
  __syncthreads();
  return r;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const T *__restrict__ in,
                                                                   int64_t n, T *block_sums) {
  __shared__ T sw[kScanThreads / 32 + 1];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + i;
    if (idx < n) s += in[idx];
  }
  T tot;
  block_excl_scan<T>(s, sw, &tot);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

// Single-block exclusive scan of the block sums, in place; writes grand total to *total.
template <class T>
__global__ void __launch_bounds__(kScanThreads) scan_spine_kernel(T *sums, int64_t nb, T *total) {
  __shared__ T sw[kScanThreads / 32 + 1];
  T carry = 0;
  for (int64_t c0 = 0; c0 < nb; c0 += kScanTile) {
    T v[kScanItems];
    T s = 0;
    int64_t base = c0 + (int64_t)threadIdx.x * kScanItems;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      v[i] = (base + i < nb) ? sums[base + i] : T(0);
      s += v[i];
    }
    T tot;
    T ex = block_excl_scan<T>(s, sw, &tot) + carry;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      if (base + i < nb) sums[base + i] = ex;
      ex += v[i];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(const T *in, T *out, int64_t n,
                                                                 const T *block_offs,
                                                                 const T *total, bool write_total) {
  __shared__ T sw[kScanThreads / 32 + 1];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? in[base + i] : T(0);
    s += v[i];
  }
  T tot;
  T ex = block_excl_scan<T>(s, sw, &tot) + block_offs[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = ex;
    ex += v[i];
  }
  if (write_total && blockIdx.x == 0 && threadIdx.x == 0) out[n] = *total;
}

// Small scans (<= kScanFusedTiles tiles, e.g. a replayed mini-batch's capacity
// arrays): the spine pass folds into the down-sweep — each block sums the tile
// totals before it (integers: exact, order-free), so a scan is two launches.
constexpr int64_t kScanFusedTiles = 512;
template <class T>
__global__ void __launch_bounds__(kScanThreads) scan_down_fused_kernel(const T *in, T *out, int64_t n,
                                                                       const T *block_sums,
                                                                       bool write_total) {
  __shared__ T sw[kScanThreads / 32 + 1];
  const int64_t nb = ceil_div(n, (int64_t)kScanTile);
  T pre = 0;
  for (int64_t i = threadIdx.x; i < (int64_t)blockIdx.x; i += kScanThreads) pre += block_sums[i];
  T ptot;
  block_excl_scan<T>(pre, sw, &ptot);  // block-wide sum of the preceding tiles' totals
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? in[base + i] : T(0);
    s += v[i];
  }
  T tot;
  T ex = block_excl_scan<T>(s, sw, &tot) + ptot;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = ex;
    ex += v[i];
  }
  if (write_total && blockIdx.x == nb - 1 && threadIdx.x == 0) out[n] = ptot + tot;
}

template <class T>
size_t scan_ws(int64_t n) {
  int64_t nb = ceil_div(n > 0 ? n : 1, kScanTile);
  WsCounter c;
  c.take<T>(nb);
  c.take<T>(1);
  return c.used;
}

template <class T>
int scan_impl(const T *in, T *out, int64_t n, bool write_total, void *ws, size_t ws_bytes,
              cudaStream_t st) {
  if (n <= 0) {
    if (write_total) GNN_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(T), st));
    return GNN_OK;
  }
  int64_t nb = ceil_div(n, kScanTile);
  WsArena a(ws, ws_bytes);
  T *sums = a.take<T>(nb);
  T *total = a.take<T>(1);
  if (!a.ok()) return GNN_ERR_WORKSPACE;
  if (nb == 1) {  // one tile: no preceding totals, one launch
    scan_down_fused_kernel<T><<<1, kScanThreads, 0, st>>>(in, out, n, sums, write_total);
    GNN_LAUNCH_CHECK();
    return GNN_OK;
  }
  scan_reduce_kernel<T><<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, sums);
  GNN_LAUNCH_CHECK();
  if (nb <= kScanFusedTiles) {
    scan_down_fused_kernel<T><<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, n, sums, write_total);
    GNN_LAUNCH_CHECK();
    return GNN_OK;
  }
  scan_spine_kernel<T><<<1, kScanThreads, 0, st>>>(sums, nb, total);
  GNN_LAUNCH_CHECK();
  scan_down_kernel<T><<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, n, sums, total, write_total);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

}  // namespace

size_t scan_i64_workspace(int64_t n) { return scan_ws<int64_t>(n); }
size_t scan_u32_workspace(int64_t n) { return scan_ws<uint32_t>(n); }

int exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, bool write_total, void *ws,
                       size_t ws_bytes, cudaStream_t st) {
  return scan_impl<int64_t>(in, out, n, write_total, ws, ws_bytes, st);
}
int exclusive_scan_u32(const uint32_t *in, uint32_t *out, int64_t n, void *ws, size_t ws_bytes,
                       cudaStream_t st) {
  return scan_impl<uint32_t>(in, out, n, false, ws, ws_bytes, st);
}

}  // namespace gnn
