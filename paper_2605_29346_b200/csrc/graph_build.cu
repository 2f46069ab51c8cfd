// Device graph builders: stable counting sort (LSD radix) of edge pairs into
// CSR, the transposed CSR (CSC) with edge ids, multigraph coalescing,
// make_csr validation, degrees, and the bit-exact PCG64 power-law generator.
//
// Reference semantics:
//   csr_from_edges      graph.py:106-114  (bincount -> cumsum -> argsort(kind="stable"))
//   make_csr            graph.py:91-103   (ValueError / RangeError)
//   build_subgraph_csr  sampler.py:242-256 (IndexError on source range)
//   generate/power-law  graph.py:254-262  (PCG64 stream, searchsorted side="right")
//
// Stability argument: every radix pass ranks the items of a tile in original
// order (warp-major rounds of 32 consecutive items, __match_any_sync peers,
// warp-private running counts), and tiles are laid out digit-major in the
// scanned count table, so each pass is a stable counting sort; LSD passes of
// stable sorts give the stable sort by the full key = argsort(kind="stable").
#include "common.cuh"

namespace gnn {
namespace {

constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsIpt = 16;
constexpr int kRsTile = kRsThreads * kRsIpt;  // 4096 items per tile
constexpr int kRsRounds = kRsIpt;            // rounds of 32 items per warp

enum SrcKind : int { SRC_I64 = 0, SRC_I32 = 1, SRC_IOTA = 2 };

struct SrcDesc {
  int kind;
  const void *p;
};

struct PassArgs {
  int64_t n;
  int64_t ntiles;
  int shift;
  SrcDesc key;
  int64_t key_limit;  // keys are clamped into [0, key_limit) for memory safety
  int nvals;
  SrcDesc val[2];
  int32_t *key_out;
  int32_t *val_out[2];
  uint32_t *counts;        // [R][ntiles]; raw counts (hist) / scanned bases (scatter)
  long long *minmax;       // [4] kmin,kmax,v0min,v0max, or null
};


template <int KIND>
__device__ __forceinline__ int64_t load_src(const void *p, int64_t i) {
  if constexpr (KIND == SRC_I64) return static_cast<const int64_t *>(p)[i];
  if constexpr (KIND == SRC_I32) return static_cast<const int32_t *>(p)[i];
  return i;
}

__device__ __forceinline__ int32_t clamp_key(int64_t k, int64_t limit) {
  k = k < 0 ? 0 : k;
  k = k >= limit ? limit - 1 : k;
  return static_cast<int32_t>(k);
}

__device__ __forceinline__ void block_minmax(long long lo, long long hi, long long *dst) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(kFull, lo, o));
    hi = max(hi, __shfl_xor_sync(kFull, hi, o));
  }
  if (lane_id() == 0) {
    atomicMin(dst, lo);
    atomicMax(dst + 1, hi);
  }
}

// CTA-wide min / max, then ONE pair of global atomics per CTA (per-warp
// atomics on the same two words serialise at the L2 slice).  All threads call.
template <int NW>
__device__ __forceinline__ void cta_minmax(long long lo, long long hi, long long *dst) {
  __shared__ long long red[2][NW];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(kFull, lo, o));
    hi = max(hi, __shfl_xor_sync(kFull, hi, o));
  }
  const int w = threadIdx.x >> 5;
  if (lane_id() == 0) {
    red[0][w] = lo;
    red[1][w] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < NW; ++i) {
      lo = min(lo, red[0][i]);
      hi = max(hi, red[1][i]);
    }
    if (lo != LLONG_MAX) atomicMin(dst, lo);
    if (hi != LLONG_MIN) atomicMax(dst + 1, hi);
  }
}

// Lanes of the warp holding the same BITS-bit digit as this lane (and valid):
// one ballot per digit bit (a short fixed sequence; MATCH.ANY measured slow).
template <int BITS>
__device__ __forceinline__ unsigned digit_peers(unsigned d, bool valid) {
  unsigned peers = __ballot_sync(kFull, valid);
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const bool bit = (d >> b) & 1u;
    const unsigned bb = __ballot_sync(kFull, bit);
    peers &= bit ? bb : ~bb;
  }
  return peers;
}

// Per-tile digit histogram (per-warp shared-memory counters; warp-aggregated
// adds via ballots or MATCH.ANY measured slower even with power-law keys).
template <int BITS, int KK>
__global__ void __launch_bounds__(kRsThreads) rs_hist_kernel(PassArgs a) {
  constexpr int R = 1 << BITS;
  extern __shared__ uint32_t smem_u32[];
  uint32_t *wh = smem_u32;  // [kRsWarps][R]
  const int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kRsWarps * R; i += kRsThreads) wh[i] = 0;
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * kRsTile + (int64_t)w * 32 * kRsRounds + lane_id();
  long long kmin = LLONG_MAX, kmax = LLONG_MIN;
  int64_t raw[kRsRounds];
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {  // all loads in flight first
    const int64_t i = base + (int64_t)r * 32;
    raw[r] = i < a.n ? load_src<KK>(a.key.p, i) : 0;
  }
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t i = base + (int64_t)r * 32;
    const bool valid = i < a.n;
    if (valid) {
      kmin = min(kmin, (long long)raw[r]);
      kmax = max(kmax, (long long)raw[r]);
    }
    if (valid) atomicAdd(&wh[w * R + ((clamp_key(raw[r], a.key_limit) >> a.shift) & (R - 1))], 1u);
  }
  if (a.minmax) cta_minmax<kRsWarps>(kmin, kmax, a.minmax);
  __syncthreads();
  for (int d = threadIdx.x; d < R; d += kRsThreads) {
    uint32_t s = 0;
#pragma unroll
    for (int ww = 0; ww < kRsWarps; ++ww) s += wh[ww * R + d];
    a.counts[(int64_t)d * a.ntiles + tile] = s;
  }
}

// Block-wide exclusive scan of v over the kScT threads (returns the prefix).
constexpr int kScT = 512;  // scatter CTA: 16 warps x 8 rounds of 32 = one 4096-item tile
constexpr int kScW = kScT / 32;
constexpr int kScRounds = kRsTile / kScT;
static_assert(kScRounds * kScT == kRsTile, "scatter and histogram tiles must match");

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *sw /*[kScW]*/) {
  const unsigned lane = lane_id();
  const int w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if ((int)lane >= o) x += y;
  }
  if (lane == 31) sw[w] = x;
  __syncthreads();
  uint32_t wsum = 0;
#pragma unroll
  for (int ww = 0; ww < kScW; ++ww) wsum += ww < w ? sw[ww] : 0u;
  __syncthreads();
  return wsum + x - v;
}

// Stable scatter of one tile: items are ranked in original order (warp-major
// rounds of 32 consecutive items, ballot-built digit peers, warp-private
// running counts), placed at their tile-local digit-sorted position in shared
// memory, and written out from there: consecutive threads then write
// consecutive addresses of one digit run (coalesced), instead of one
// scattered 4-byte store per item per array.  The
// tile's global loads (keys, values, its scanned digit bases) are all issued
// before the ranking, so a tile pays one memory latency (16 warps/CTA, 2
// CTAs/SM resident for digits <= 9 bits).
// Source kinds are compile-time (KK key, V0K value 0, V1K value 1 or -1).
template <int BITS, int KK, int V0K, int V1K>
__global__ void __launch_bounds__(kScT, BITS >= 10 ? 1 : 2) rs_scatter_kernel(PassArgs a) {
  constexpr int R = 1 << BITS;
  constexpr int DPT = R >= kScT ? R / kScT : 1;  // digits per thread in the scans
  extern __shared__ uint32_t smem_u32[];
  uint32_t *wc = smem_u32;                 // [kScW][R] running counts, then warp bases
  int64_t *gdelta = reinterpret_cast<int64_t *>(wc + kScW * R);  // [R] global - local
  int32_t *skey = reinterpret_cast<int32_t *>(gdelta + R);        // [kRsTile]
  int32_t *sv0 = skey + kRsTile;
  int32_t *sv1 = sv0 + kRsTile;
  __shared__ uint32_t sw[kScW];
  const int w = threadIdx.x >> 5;
  const unsigned lane = lane_id();
  for (int i = threadIdx.x; i < kScW * R; i += kScT) wc[i] = 0;
  const int64_t tile = blockIdx.x;
  const int64_t t0 = tile * kRsTile;
  const int tn = (int)min((int64_t)kRsTile, a.n - t0);
  const int64_t base = t0 + (int64_t)w * 32 * kScRounds + lane;

  // every global load of the tile in flight at once: keys, values, and this
  // tile's scanned digit bases (independent of the ranking)
  int32_t key[kScRounds], v0[kScRounds], v1[kScRounds];
  uint32_t rank[kScRounds];
  long long vmin = LLONG_MAX, vmax = LLONG_MIN;
#pragma unroll
  for (int r = 0; r < kScRounds; ++r) {
    const int64_t i = base + (int64_t)r * 32;
    const bool valid = i < a.n;
    key[r] = valid ? clamp_key(load_src<KK>(a.key.p, i), a.key_limit) : 0;
    const int64_t x0 = valid ? load_src<V0K>(a.val[0].p, i) : 0;
    if (valid) {
      vmin = min(vmin, (long long)x0);
      vmax = max(vmax, (long long)x0);
    }
    v0[r] = static_cast<int32_t>(x0);
    if constexpr (V1K >= 0) v1[r] = valid ? static_cast<int32_t>(load_src<V1K>(a.val[1].p, i)) : 0;
  }
  uint32_t gcnt[DPT];
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int d = threadIdx.x * DPT + j;
    gcnt[j] = d < R ? a.counts[(int64_t)d * a.ntiles + tile] : 0u;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kScRounds; ++r) {
    const bool valid = base + (int64_t)r * 32 < a.n;
    const unsigned d = (unsigned)(key[r] >> a.shift) & (R - 1);
#ifdef GNN_RS_MATCH
    const unsigned peers = __match_any_sync(kFull, valid ? d : (unsigned)R);
#else
    const unsigned peers = digit_peers<BITS>(d, valid);
#endif
    const unsigned lt = __popc(peers & lanemask_lt());
    const uint32_t cnt = valid ? wc[w * R + d] : 0u;
    rank[r] = cnt + lt;
    __syncwarp();
    if (valid && lt == 0) wc[w * R + d] = cnt + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // tile totals per digit -> tile-local digit starts (block scan over digits)
  uint32_t tot[DPT];
  uint32_t my = 0;
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int d = threadIdx.x * DPT + j;
    uint32_t t = 0;
    if (d < R) {
#pragma unroll
      for (int ww = 0; ww < kScW; ++ww) t += wc[ww * R + d];
    }
    tot[j] = t;
    my += t;
  }
  uint32_t run = block_excl_scan(my, sw);
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int d = threadIdx.x * DPT + j;
    if (d < R) {
      gdelta[d] = (int64_t)gcnt[j] - (int64_t)run;
      uint32_t wr = run;  // warp-local starts within the digit's tile run
#pragma unroll
      for (int ww = 0; ww < kScW; ++ww) {
        const uint32_t c = wc[ww * R + d];
        wc[ww * R + d] = wr;
        wr += c;
      }
    }
    run += tot[j];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kScRounds; ++r) {
    if (base + (int64_t)r * 32 < a.n) {
      const unsigned d = (unsigned)(key[r] >> a.shift) & (R - 1);
      const uint32_t lp = wc[w * R + d] + rank[r];
      skey[lp] = key[r];
      sv0[lp] = v0[r];
      if constexpr (V1K >= 0) sv1[lp] = v1[r];
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < tn; j += kScT) {
    const int32_t k = skey[j];
    const int64_t pos = gdelta[(unsigned)(k >> a.shift) & (R - 1)] + j;
    a.key_out[pos] = k;
    a.val_out[0][pos] = sv0[j];
    if constexpr (V1K >= 0) a.val_out[1][pos] = sv1[j];
  }
  if (a.minmax) cta_minmax<kScW>(vmin, vmax, a.minmax + 2);
}

template <int BITS, int KK, int V0K, int V1K>
int launch_pass_k(const PassArgs &a, cudaStream_t st, void *scan_ws, size_t scan_ws_bytes) {
  constexpr int R = 1 << BITS;
  const size_t smem_h = sizeof(uint32_t) * kRsWarps * R;
  const size_t smem_s = sizeof(uint32_t) * kScW * R + sizeof(int64_t) * R + sizeof(int32_t) * 3 * kRsTile;
  static bool attr_set = false;  // idempotent; benign race
  if (!attr_set) {
    GNN_CUDA_TRY(cudaFuncSetAttribute(rs_hist_kernel<BITS, KK>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_h));
    GNN_CUDA_TRY(cudaFuncSetAttribute(rs_scatter_kernel<BITS, KK, V0K, V1K>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s));
    attr_set = true;
  }
  rs_hist_kernel<BITS, KK><<<(unsigned)a.ntiles, kRsThreads, smem_h, st>>>(a);
  GNN_LAUNCH_CHECK();
  GNN_TRY(exclusive_scan_u32(a.counts, a.counts, (int64_t)R * a.ntiles, scan_ws, scan_ws_bytes, st));
  rs_scatter_kernel<BITS, KK, V0K, V1K><<<(unsigned)a.ntiles, kScT, smem_s, st>>>(a);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

// source-kind combinations the builders use: (i64 key, i64 val) csr_from_edges
// pass 0; (i32, i32) later passes / sort_pairs; (i32, i32, iota) the CSC pass 0
// (edge ids); (i32, i32, i32) its later passes
template <int BITS>
int launch_pass(const PassArgs &a, cudaStream_t st, void *scan_ws, size_t scan_ws_bytes) {
  const int kk = a.key.kind, v0 = a.val[0].kind, v1 = a.nvals > 1 ? a.val[1].kind : -1;
  if (kk == SRC_I64 && v0 == SRC_I64 && v1 < 0)
    return launch_pass_k<BITS, SRC_I64, SRC_I64, -1>(a, st, scan_ws, scan_ws_bytes);
  if (kk == SRC_I32 && v0 == SRC_I32 && v1 < 0)
    return launch_pass_k<BITS, SRC_I32, SRC_I32, -1>(a, st, scan_ws, scan_ws_bytes);
  if (kk == SRC_I32 && v0 == SRC_I32 && v1 == SRC_IOTA)
    return launch_pass_k<BITS, SRC_I32, SRC_I32, SRC_IOTA>(a, st, scan_ws, scan_ws_bytes);
  if (kk == SRC_I32 && v0 == SRC_I32 && v1 == SRC_I32)
    return launch_pass_k<BITS, SRC_I32, SRC_I32, SRC_I32>(a, st, scan_ws, scan_ws_bytes);
  return GNN_ERR_UNSUPPORTED;
}

int launch_pass_bits(int bits, const PassArgs &a, cudaStream_t st, void *sws, size_t sws_bytes) {
  switch (bits) {
    case 4: return launch_pass<4>(a, st, sws, sws_bytes);
    case 6: return launch_pass<6>(a, st, sws, sws_bytes);
    case 8: return launch_pass<8>(a, st, sws, sws_bytes);
    case 9: return launch_pass<9>(a, st, sws, sws_bytes);
    case 10: return launch_pass<10>(a, st, sws, sws_bytes);
    case 11: return launch_pass<11>(a, st, sws, sws_bytes);
    default: return GNN_ERR_UNSUPPORTED;
  }
}

int bit_width_u64(uint64_t x) { return x == 0 ? 0 : 64 - __builtin_clzll(x); }

struct RadixPlan {
  int nbits;
  int passes;
  int bits;  // per pass (instantiated width >= needed)
};

RadixPlan plan_radix(int64_t key_limit) {
  RadixPlan p;
  p.nbits = key_limit > 1 ? bit_width_u64((uint64_t)(key_limit - 1)) : 1;
  p.passes = (p.nbits + 10) / 11;
  int need = (p.nbits + p.passes - 1) / p.passes;
  static const int widths[] = {4, 6, 8, 9, 10, 11};
  p.bits = 11;
  for (int wdt : widths)
    if (wdt >= need) {
      p.bits = wdt;
      break;
    }
  return p;
}

// ------------------------------------------------------ stable sort driver
struct SortIO {
  int64_t n;
  int64_t key_limit;
  SrcDesc key;
  int nvals;
  SrcDesc val[2];
  int32_t *keys_sorted;  // final sorted keys [n]
  int32_t *vals_sorted[2];
};

void sort_ws_count(WsCounter &c, int64_t n, int64_t key_limit, int nvals) {
  RadixPlan p = plan_radix(key_limit);
  int64_t ntiles = ceil_div(n > 0 ? n : 1, kRsTile);
  int64_t cnt = ((int64_t)1 << p.bits) * ntiles;
  c.take<int32_t>(n);              // key ping
  c.take<int32_t>(n);              // key pong
  for (int v = 0; v < nvals; ++v) {
    c.take<int32_t>(n);
    c.take<int32_t>(n);
  }
  c.take<uint32_t>(cnt);
  c.take<long long>(4);
  c.used += scan_u32_workspace(cnt) + 256;
}

// Runs all passes; final outputs land in io.keys_sorted / io.vals_sorted.
// minmax (device [4]) receives key/val0 min/max of the pass-0 sources if non-null.
int stable_sort(const SortIO &io, long long *minmax, WsArena &ar, cudaStream_t st) {
  RadixPlan p = plan_radix(io.key_limit);
  const int64_t n = io.n;
  if (n == 0) return GNN_OK;
  int64_t ntiles = ceil_div(n, kRsTile);
  int64_t cnt = ((int64_t)1 << p.bits) * ntiles;
  int32_t *kb[2] = {ar.take<int32_t>(n), ar.take<int32_t>(n)};
  int32_t *vb[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  for (int v = 0; v < io.nvals; ++v) {
    vb[v][0] = ar.take<int32_t>(n);
    vb[v][1] = ar.take<int32_t>(n);
  }
  uint32_t *counts = ar.take<uint32_t>(cnt);
  size_t sws_bytes = scan_u32_workspace(cnt);
  void *sws = ar.take<char>((int64_t)sws_bytes);
  if (!ar.ok()) return GNN_ERR_WORKSPACE;

  SrcDesc kin = io.key;
  SrcDesc vin[2] = {io.val[0], io.val[1]};
  for (int pass = 0; pass < p.passes; ++pass) {
    const bool last = pass == p.passes - 1;
    PassArgs a{};
    a.n = n;
    a.ntiles = ntiles;
    a.shift = pass * p.bits;
    a.key = kin;
    a.key_limit = io.key_limit;
    a.nvals = io.nvals;
    a.val[0] = vin[0];
    a.val[1] = vin[1];
    a.key_out = last ? io.keys_sorted : kb[pass & 1];
    for (int v = 0; v < io.nvals; ++v) a.val_out[v] = last ? io.vals_sorted[v] : vb[v][pass & 1];
    a.counts = counts;
    a.minmax = (pass == 0) ? minmax : nullptr;
    GNN_TRY(launch_pass_bits(p.bits, a, st, sws, sws_bytes));
    kin = SrcDesc{SRC_I32, a.key_out};
    for (int v = 0; v < io.nvals; ++v) vin[v] = SrcDesc{SRC_I32, a.val_out[v]};
  }
  return GNN_OK;
}

// ------------------------------------------------ offsets from sorted keys
// offsets[k] = first position whose key is >= k (= bincount -> cumsum of
// graph.py:110-112 for sorted keys), streaming: position i with key boundary
// (key[i-1], key[i]] writes offsets[key[i-1]+1 .. key[i]] = i, so empty keys
// in the gap get the same start; the head (k <= key[0]) gets 0 and the tail
// (k > key[n-1]) n.  A thread fills at most kGapRun entries of a gap; entries
// of longer gaps stay at the -1 pre-fill and a second pass binary-searches
// them (so one huge gap never serialises on one thread).
constexpr int64_t kGapRun = 64;
__global__ void offsets_from_keys_kernel(const int32_t *__restrict__ keys, int64_t n, int64_t V,
                                         int64_t *offsets) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += stride) {
    const int64_t lo = i == 0 ? -1 : (int64_t)keys[i - 1];  // previous key (-1: before the head)
    const int64_t hi = i == n ? V : (int64_t)keys[i];       // this key (V: past the tail)
    const int64_t top = min(hi, lo + kGapRun);
    for (int64_t k = lo + 1; k <= top; ++k) offsets[k] = i;
  }
}
__global__ void offsets_fill_gaps_kernel(const int32_t *__restrict__ keys, int64_t n, int64_t V,
                                         int64_t *offsets) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= V; k += stride)
    if (offsets[k] < 0) offsets[k] = lower_bound_dev(keys, (int64_t)0, n, (int32_t)min(k, (int64_t)INT32_MAX));
}

unsigned grid_for(int64_t n, int threads) {
  int64_t b = ceil_div(n > 0 ? n : 1, threads);
  int64_t cap = (int64_t)sm_count() * 16;
  return (unsigned)(b < cap ? b : cap);
}

void offsets_ws_count(WsCounter &c, int64_t V) { (void)c, (void)V; }

// offsets[V+1] of sorted keys in [0, V)
int offsets_from_sorted(const int32_t *keys, int64_t n, int64_t V, int64_t *offsets, WsArena &ar,
                        cudaStream_t st) {
  (void)ar;
  if (n == 0) {
    GNN_CUDA_TRY(cudaMemsetAsync(offsets, 0, sizeof(int64_t) * (V + 1), st));
    return GNN_OK;
  }
  GNN_CUDA_TRY(cudaMemsetAsync(offsets, 0xff, sizeof(int64_t) * (V + 1), st));
  offsets_from_keys_kernel<<<grid_for(n + 1, 256), 256, 0, st>>>(keys, n, V, offsets);
  GNN_LAUNCH_CHECK();
  offsets_fill_gaps_kernel<<<grid_for(V + 1, 256), 256, 0, st>>>(keys, n, V, offsets);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

__global__ void init_minmax_kernel(long long *mm) {
  mm[0] = LLONG_MAX;
  mm[1] = LLONG_MIN;
  mm[2] = LLONG_MAX;
  mm[3] = LLONG_MIN;
}

// Shared by csr_from_edges and build_subgraph_csr.
size_t edges_ws(int64_t V, int64_t E) {
  WsCounter c;
  sort_ws_count(c, E, V > 0 ? V : 1, 1);
  c.take<int32_t>(E);  // sorted keys
  offsets_ws_count(c, V);
  c.take<long long>(4);
  return c.used + 1024;
}

// mode 0: csr_from_edges (src range -> SOURCE_RANGE, dst range -> RANGE)
// mode 1: build_subgraph_csr (src range -> INDEX, dst unchecked)
int build_from_edges(int mode, int64_t V, int64_t E, const int64_t *src, const int64_t *dst,
                     int64_t *offsets, int32_t *targets, void *ws, size_t ws_bytes,
                     cudaStream_t st) {
  if (V < 0 || E < 0 || (E > 0 && (!src || !dst || !targets)) || !offsets)
    return GNN_ERR_INVALID_ARGUMENT;
  if (E >= ((int64_t)1 << 32) || V > ((int64_t)1 << 31)) return GNN_ERR_UNSUPPORTED;
  if (ws_bytes < edges_ws(V, E)) return GNN_ERR_WORKSPACE;
  if (V == 0) {
    if (E > 0) return mode == 0 ? GNN_ERR_SOURCE_RANGE : GNN_ERR_INDEX;
    GNN_CUDA_TRY(cudaMemsetAsync(offsets, 0, sizeof(int64_t), st));
    return GNN_OK;
  }
  WsArena ar(ws, ws_bytes);
  long long *mm = ar.take<long long>(4);
  int32_t *skeys = ar.take<int32_t>(E);
  if (!ar.ok()) return GNN_ERR_WORKSPACE;
  init_minmax_kernel<<<1, 1, 0, st>>>(mm);
  GNN_LAUNCH_CHECK();
  SortIO io{};
  io.n = E;
  io.key_limit = V;
  io.key = SrcDesc{SRC_I64, src};
  io.nvals = 1;
  io.val[0] = SrcDesc{SRC_I64, dst};
  io.keys_sorted = skeys;
  io.vals_sorted[0] = targets;
  GNN_TRY(stable_sort(io, mm, ar, st));
  GNN_TRY(offsets_from_sorted(skeys, E, V, offsets, ar, st));
  long long h[4];
  GNN_CUDA_TRY(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, st));
  GNN_CUDA_TRY(cudaStreamSynchronize(st));
  if (E > 0) {
    if (h[0] < 0 || h[1] >= V) return mode == 0 ? GNN_ERR_SOURCE_RANGE : GNN_ERR_INDEX;
    if (mode == 0 && (h[2] < 0 || h[3] >= V)) return GNN_ERR_RANGE;
  }
  return GNN_OK;
}

// ---------------------------------------------------------- CSC (transpose)
// rows_of_edge[e] = r with offsets[r] <= e < offsets[r+1]; one tile of edges
// per block, offsets of the tile's row span staged in shared memory.
constexpr int kExpTile = 4096;
constexpr int kExpRun = 16;  // consecutive edges per thread: one search, then a forward walk
__global__ void __launch_bounds__(256) expand_rows_kernel(const int64_t *__restrict__ offsets,
                                                          int64_t num_rows, int64_t nnz,
                                                          int32_t *rows) {
  __shared__ int64_t soff[kExpTile + 2];
  __shared__ int64_t span[2];
  const int64_t e0 = (int64_t)blockIdx.x * kExpTile;
  const int64_t e1 = min(e0 + kExpTile, nnz);
  if (threadIdx.x == 0) {
    span[0] = upper_bound_dev(offsets, 0, num_rows + 1, e0) - 1;
    span[1] = upper_bound_dev(offsets, 0, num_rows + 1, e1 - 1) - 1;
  }
  __syncthreads();
  const int64_t r0 = span[0], r1 = span[1];
  const int64_t cnt = r1 - r0 + 2;  // offsets[r0 .. r1+1]
  const bool staged = cnt <= kExpTile + 2;
  if (staged)
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) soff[i] = offsets[r0 + i];
  __syncthreads();
  // thread t: edges e0 + t*kExpRun + [0, kExpRun), consecutive, row index walks forward
  const int64_t s0 = e0 + (int64_t)threadIdx.x * kExpRun;
  if (s0 >= e1) return;
  int64_t r = staged ? upper_bound_dev(soff, 0, cnt, s0) - 1 : upper_bound_dev(offsets, r0, r1 + 2, s0) - 1 - r0;
  int64_t rend = staged ? soff[r + 1] : offsets[r0 + r + 1];
  int32_t out[kExpRun];
#pragma unroll
  for (int k = 0; k < kExpRun; ++k) {
    const int64_t e = s0 + k;
    while (e >= rend && e < e1) {  // empty rows are skipped by the same walk
      ++r;
      rend = staged ? soff[r + 1] : offsets[r0 + r + 1];
    }
    out[k] = (int32_t)(r0 + r);
  }
  if (s0 + kExpRun <= e1 && ((reinterpret_cast<uintptr_t>(rows + s0) & 15u) == 0)) {
#pragma unroll
    for (int k = 0; k < kExpRun; k += 4)
      *reinterpret_cast<int4 *>(rows + s0 + k) = make_int4(out[k], out[k + 1], out[k + 2], out[k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < kExpRun; ++k)
      if (s0 + k < e1) rows[s0 + k] = out[k];
  }
}

size_t csc_ws(int64_t R, int64_t C, int64_t nnz) {
  WsCounter c;
  c.take<int32_t>(nnz);  // expanded rows
  c.take<int32_t>(nnz);  // sorted keys
  c.take<int32_t>(nnz);  // eid scratch when t_eid is null
  sort_ws_count(c, nnz, C > 0 ? C : 1, 2);
  offsets_ws_count(c, C);
  (void)R;
  return c.used + 1024;
}

int csc_impl(int64_t R, int64_t C, int64_t nnz, const int64_t *offsets, const int32_t *cols,
             int64_t *t_offsets, int32_t *t_rows, int32_t *t_eid, void *ws, size_t ws_bytes,
             cudaStream_t st) {
  if (R < 0 || C < 0 || nnz < 0 || !offsets || !t_offsets || (nnz > 0 && (!cols || !t_rows)))
    return GNN_ERR_INVALID_ARGUMENT;
  if (nnz >= ((int64_t)1 << 31) || C > ((int64_t)1 << 31)) return GNN_ERR_UNSUPPORTED;
  if (ws_bytes < csc_ws(R, C, nnz)) return GNN_ERR_WORKSPACE;
  if (C == 0) {
    if (nnz > 0) return GNN_ERR_RANGE;
    GNN_CUDA_TRY(cudaMemsetAsync(t_offsets, 0, sizeof(int64_t), st));
    return GNN_OK;
  }
  WsArena ar(ws, ws_bytes);
  int32_t *rows = ar.take<int32_t>(nnz);
  int32_t *skeys = ar.take<int32_t>(nnz);
  int32_t *eid_scratch = ar.take<int32_t>(nnz);
  if (!ar.ok()) return GNN_ERR_WORKSPACE;
  if (nnz > 0) {
    expand_rows_kernel<<<(unsigned)ceil_div(nnz, kExpTile), 256, 0, st>>>(offsets, R, nnz, rows);
    GNN_LAUNCH_CHECK();
    SortIO io{};
    io.n = nnz;
    io.key_limit = C;
    io.key = SrcDesc{SRC_I32, cols};
    io.nvals = 2;
    io.val[0] = SrcDesc{SRC_I32, rows};
    io.val[1] = SrcDesc{SRC_IOTA, nullptr};
    io.keys_sorted = skeys;
    io.vals_sorted[0] = t_rows;
    io.vals_sorted[1] = t_eid ? t_eid : eid_scratch;
    GNN_TRY(stable_sort(io, nullptr, ar, st));
  }
  return offsets_from_sorted(skeys, nnz, C, t_offsets, ar, st);
}

// ------------------------------------------------------------- coalescing
__global__ void mark_row_starts_kernel(const int64_t *__restrict__ offsets, int64_t R, int64_t nnz,
                                       int64_t *flag) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = offsets[r];
    if (o < nnz) flag[o] = 1;
  }
}
__global__ void mark_col_changes_kernel(const int32_t *__restrict__ cols, int64_t nnz,
                                        int64_t *flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == 0 || cols[i] != cols[i - 1]) flag[i] = 1;
  }
}
// u = exclusive scan of flags, with u[nnz] = total.  Run index of i = u[i+1]-1.
__global__ void coalesce_scatter_kernel(const int32_t *__restrict__ cols, int64_t nnz,
                                        const int64_t *__restrict__ u, int32_t *out_cols,
                                        int64_t *start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = u[i], b = u[i + 1];
    if (b != a) {
      out_cols[a] = cols[i];
      start[a] = i;
    }
    if (i == 0) start[u[nnz]] = nnz;
  }
}
__global__ void coalesce_mult_kernel(const int64_t *__restrict__ u, int64_t nnz,
                                     const int64_t *__restrict__ start, float *mult) {
  const int64_t total = u[nnz];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total;
       j += (int64_t)gridDim.x * blockDim.x)
    mult[j] = (float)(start[j + 1] - start[j]);
}
__global__ void coalesce_offsets_kernel(const int64_t *__restrict__ offsets, int64_t R,
                                        int64_t nnz, const int64_t *__restrict__ u,
                                        int64_t *out_offsets) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= R;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = offsets[r];
    out_offsets[r] = o < nnz ? u[o] : u[nnz];
  }
}

size_t coalesce_ws(int64_t R, int64_t nnz) {
  WsCounter c;
  c.take<int64_t>(nnz + 1);
  c.take<int64_t>(nnz + 1);
  c.used += scan_i64_workspace(nnz) + 256;
  (void)R;
  return c.used + 1024;
}

// ----------------------------------------------------------- validation
__global__ void validate_kernel(const int64_t *__restrict__ offsets, int64_t V, int64_t E,
                                const int32_t *__restrict__ targets, int *flags) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int f = 0;
  if (tid == 0 && (offsets[0] != 0 || offsets[V] != E)) f |= 1;
  for (int64_t v = tid; v < V; v += stride)
    if (offsets[v + 1] < offsets[v]) f |= 1;
  for (int64_t e = tid; e < E; e += stride) {
    int32_t t = targets[e];
    if (t < 0 || (int64_t)t >= V) f |= 2;
  }
  f = __reduce_or_sync(kFull, f);
  if (lane_id() == 0 && f) atomicOr(flags, f);
}

__global__ void degrees_kernel(const int64_t *__restrict__ offsets, int64_t V, int64_t *deg) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    deg[v] = offsets[v + 1] - offsets[v];
}

// ------------------------------------------------------- PCG64 generator
struct U128 {
  uint64_t hi, lo;
};
__device__ __forceinline__ U128 u128_mul(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
  return r;
}
__device__ __forceinline__ U128 u128_add(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
// numpy PCG64 = pcg_setseq_128_xsl_rr_64: state = state*M + inc; out = rotr(hi^lo, state>>122)
__device__ __constant__ U128 kPcgMult = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};

__device__ __forceinline__ U128 pcg_advance(U128 state, U128 inc, uint64_t delta) {
  U128 acc_mult = {0, 1}, acc_plus = {0, 0};
  U128 cur_mult = kPcgMult, cur_plus = inc;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult = u128_mul(acc_mult, cur_mult);
      acc_plus = u128_add(u128_mul(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = u128_mul(u128_add(cur_mult, U128{0, 1}), cur_plus);
    cur_mult = u128_mul(cur_mult, cur_mult);
    delta >>= 1;
  }
  return u128_add(u128_mul(acc_mult, state), acc_plus);
}
__device__ __forceinline__ uint64_t pcg_output(U128 s) {
  uint64_t v = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  return (v >> rot) | (v << ((64u - rot) & 63u));
}

constexpr int kGuideBits = 20;
constexpr int64_t kGuide = (int64_t)1 << kGuideBits;

__global__ void guide_kernel(const double *__restrict__ cdf, int64_t n, int32_t *guide) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= kGuide;
       b += (int64_t)gridDim.x * blockDim.x) {
    double x = (double)b / (double)kGuide;  // exact: power-of-two denominator
    guide[b] = (int32_t)upper_bound_dev(cdf, 0, n, x);
  }
}

constexpr int kGenChunk = 64;
// sampling draws: shorter chunks (a mini-batch hop is ~1e4-1e6 draws, each a
// chain of dependent gathers): more threads in flight per jump-ahead
constexpr int kDrawChunk = 8;
__global__ void __launch_bounds__(256) powerlaw_kernel(const double *__restrict__ cdf, int64_t n,
                                                       int64_t m, const int32_t *__restrict__ guide,
                                                       U128 state0, U128 inc, int64_t *src,
                                                       int64_t *dst) {
  const int64_t total = 2 * m;
  const int64_t nchunks = ceil_div(total, kGenChunk);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    int64_t p0 = c * kGenChunk;
    U128 s = pcg_advance(state0, inc, (uint64_t)p0);
    int64_t p1 = min(p0 + kGenChunk, total);
    for (int64_t p = p0; p < p1; ++p) {
      s = u128_add(u128_mul(s, kPcgMult), inc);
      double u = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
      int64_t b = (int64_t)(u * (double)kGuide);  // u in [b/G,(b+1)/G) exactly (power-of-two scale)
      int64_t idx = upper_bound_dev(cdf, (int64_t)guide[b], (int64_t)guide[b + 1], u);
      if (p < m)
        src[p] = idx;
      else
        dst[p - m] = idx;
    }
  }
}

// ------------------------------------------- row-block power-law build
// The per-rank build of the row-partitioned path: rank p never
// materialises the whole graph.  It regenerates the bit-exact edge stream of
// graph.py:256-261 chunk by chunk (edge i: src = draw i, dst = draw m+i) and
// keeps, in stream order, (src-lo, dst) for src in [lo,hi) (its CSR rows) and
// (dst-lo, src) for dst in [lo,hi) (its CSC rows).  Stable sorts of those
// pairs then give the block of the reference's CSR / transposed CSR exactly.
__global__ void __launch_bounds__(256) powerlaw_pairs_kernel(
    const double *__restrict__ cdf, int64_t m, const int32_t *__restrict__ guide, U128 state0,
    U128 inc, int64_t e0, int64_t e1, int32_t *src, int32_t *dst) {
  const int64_t nchunks = ceil_div(e1 - e0, kGenChunk);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < 2 * nchunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    const bool is_dst = c >= nchunks;
    const int64_t q0 = e0 + (is_dst ? c - nchunks : c) * kGenChunk;
    const int64_t q1 = min(q0 + kGenChunk, e1);
    U128 s = pcg_advance(state0, inc, (uint64_t)(is_dst ? m + q0 : q0));
    int32_t *out = is_dst ? dst : src;
    for (int64_t q = q0; q < q1; ++q) {
      s = u128_add(u128_mul(s, kPcgMult), inc);
      const double u = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
      const int64_t b = (int64_t)(u * (double)kGuide);
      out[q - e0] = (int32_t)upper_bound_dev(cdf, (int64_t)guide[b], (int64_t)guide[b + 1], u);
    }
  }
}

constexpr int kSelThreads = 256;
constexpr int kSelItems = 16;
constexpr int kSelTile = kSelThreads * kSelItems;

__device__ __forceinline__ int64_t sel_warp_incl(int64_t v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t n = __shfl_up_sync(kFull, v, o);
    if ((int)lane_id() >= o) v += n;
  }
  return v;
}

// exclusive block prefix of (a, b) per thread; totals in *ta / *tb
__device__ __forceinline__ void sel_block_scan(int64_t &a, int64_t &b, int64_t *ta, int64_t *tb) {
  __shared__ int64_t wa[kSelThreads / 32 + 1], wb[kSelThreads / 32 + 1];
  const int w = threadIdx.x >> 5;
  const int64_t ia = sel_warp_incl(a), ib = sel_warp_incl(b);
  if (lane_id() == 31) {
    wa[w] = ia;
    wb[w] = ib;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t ra = 0, rb = 0;
    for (int k = 0; k < kSelThreads / 32; ++k) {
      const int64_t xa = wa[k], xb = wb[k];
      wa[k] = ra;
      wb[k] = rb;
      ra += xa;
      rb += xb;
    }
    wa[kSelThreads / 32] = ra;
    wb[kSelThreads / 32] = rb;
  }
  __syncthreads();
  a = wa[w] + ia - a;
  b = wb[w] + ib - b;
  *ta = wa[kSelThreads / 32];
  *tb = wb[kSelThreads / 32];
}

// pass 1: kept counts per tile, [2][ntiles] (row 0: src in block, row 1: dst in block)
__global__ void __launch_bounds__(kSelThreads) block_select_count_kernel(
    int64_t n, const int32_t *__restrict__ src, const int32_t *__restrict__ dst, int64_t lo,
    int64_t hi, int64_t ntiles, int64_t *tilecnt) {
  const int64_t base = (int64_t)blockIdx.x * kSelTile + (int64_t)threadIdx.x * kSelItems;
  int64_t a = 0, b = 0;
#pragma unroll
  for (int j = 0; j < kSelItems; ++j) {
    const int64_t i = base + j;
    if (i < n) {
      const int64_t s = src[i], d = dst[i];
      a += (s >= lo && s < hi);
      b += (d >= lo && d < hi);
    }
  }
  int64_t ta, tb;
  sel_block_scan(a, b, &ta, &tb);
  if (threadIdx.x == 0) {
    tilecnt[blockIdx.x] = ta;
    tilecnt[ntiles + 1 + blockIdx.x] = tb;
  }
}

// pass 2: append the kept pairs in stream order after the running counts
__global__ void __launch_bounds__(kSelThreads) block_select_write_kernel(
    int64_t n, const int32_t *__restrict__ src, const int32_t *__restrict__ dst, int64_t lo,
    int64_t hi, int64_t ntiles, const int64_t *__restrict__ tilebase,
    const int64_t *__restrict__ count, int64_t cap, int32_t *r_key, int32_t *r_val, int32_t *c_key,
    int32_t *c_val) {
  const int64_t base = (int64_t)blockIdx.x * kSelTile + (int64_t)threadIdx.x * kSelItems;
  int32_t sv[kSelItems], dv[kSelItems];
  int64_t a = 0, b = 0;
#pragma unroll
  for (int j = 0; j < kSelItems; ++j) {
    const int64_t i = base + j;
    sv[j] = i < n ? src[i] : -1;
    dv[j] = i < n ? dst[i] : -1;
    a += (sv[j] >= lo && sv[j] < hi);
    b += (dv[j] >= lo && dv[j] < hi);
  }
  int64_t ta, tb;
  sel_block_scan(a, b, &ta, &tb);
  int64_t pa = count[0] + tilebase[blockIdx.x] + a;
  int64_t pb = count[1] + tilebase[ntiles + 1 + blockIdx.x] + b;
#pragma unroll
  for (int j = 0; j < kSelItems; ++j) {
    if (sv[j] >= lo && sv[j] < hi) {
      if (r_key && pa < cap) {  // past capacity: counted, not written (caller re-runs)
        r_key[pa] = (int32_t)(sv[j] - lo);
        r_val[pa] = dv[j];
      }
      ++pa;
    }
    if (dv[j] >= lo && dv[j] < hi) {
      if (c_key && pb < cap) {
        c_key[pb] = (int32_t)(dv[j] - lo);
        c_val[pb] = sv[j];
      }
      ++pb;
    }
  }
}

__global__ void block_count_add_kernel(int64_t *count, const int64_t *__restrict__ tilebase,
                                       int64_t ntiles) {
  if (threadIdx.x == 0) {
    count[0] += tilebase[ntiles];
    count[1] += tilebase[2 * ntiles + 1];
  }
}

}  // namespace
}  // namespace gnn

using namespace gnn;

extern "C" {

size_t gnn_powerlaw_block_workspace(int64_t n, int64_t chunk) {
  (void)n;
  WsCounter c;
  c.take<int32_t>(kGuide + 1);
  c.take<int32_t>(chunk);  // src chunk
  c.take<int32_t>(chunk);  // dst chunk
  const int64_t ntiles = ceil_div(chunk > 0 ? chunk : 1, kSelTile);
  c.take<int64_t>(2 * (ntiles + 1));  // tile counts -> bases (two scans)
  c.used += 2 * scan_i64_workspace(ntiles) + 256;
  return c.used + 1024;
}

int gnn_powerlaw_block(int64_t n, int64_t m, const double *cdf, uint64_t state_hi,
                       uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t lo, int64_t hi,
                       int64_t chunk, int64_t capacity, int32_t *r_key, int32_t *r_val,
                       int32_t *c_key, int32_t *c_val, int64_t *count, void *ws, size_t ws_bytes,
                       gnn_stream_t stream) {
  if (capacity < 0 || n < 1 || m < 0 || !cdf || lo < 0 || hi < lo || hi > n || chunk < kSelTile || !count ||
      (!r_key) != (!r_val) || (!c_key) != (!c_val))
    return GNN_ERR_INVALID_ARGUMENT;
  if (n >= ((int64_t)1 << 31)) return GNN_ERR_UNSUPPORTED;
  if (ws_bytes < gnn_powerlaw_block_workspace(n, chunk)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  WsArena ar(ws, ws_bytes);
  int32_t *guide = ar.take<int32_t>(kGuide + 1);
  int32_t *cs = ar.take<int32_t>(chunk);
  int32_t *cd = ar.take<int32_t>(chunk);
  const int64_t ntiles_max = ceil_div(chunk, kSelTile);
  int64_t *tiles = ar.take<int64_t>(2 * (ntiles_max + 1));
  const size_t sws_bytes = scan_i64_workspace(ntiles_max);
  void *sws0 = ar.take<char>((int64_t)sws_bytes);
  void *sws1 = ar.take<char>((int64_t)sws_bytes);
  if (!ar.ok()) return GNN_ERR_WORKSPACE;
  GNN_CUDA_TRY(cudaMemsetAsync(count, 0, 2 * sizeof(int64_t), st));
  if (m == 0) return GNN_OK;
  guide_kernel<<<grid_for(kGuide + 1, 256), 256, 0, st>>>(cdf, n, guide);
  GNN_LAUNCH_CHECK();
  const U128 s0{state_hi, state_lo}, inc{inc_hi, inc_lo};
  for (int64_t e0 = 0; e0 < m; e0 += chunk) {
    const int64_t e1 = e0 + chunk < m ? e0 + chunk : m;
    const int64_t len = e1 - e0, ntiles = ceil_div(len, kSelTile);
    powerlaw_pairs_kernel<<<grid_for(2 * ceil_div(len, kGenChunk), 256), 256, 0, st>>>(
        cdf, m, guide, s0, inc, e0, e1, cs, cd);
    GNN_LAUNCH_CHECK();
    block_select_count_kernel<<<(unsigned)ntiles, kSelThreads, 0, st>>>(len, cs, cd, lo, hi,
                                                                        ntiles, tiles);
    GNN_LAUNCH_CHECK();
    GNN_TRY(exclusive_scan_i64(tiles, tiles, ntiles, true, sws0, sws_bytes, st));
    GNN_TRY(exclusive_scan_i64(tiles + ntiles + 1, tiles + ntiles + 1, ntiles, true, sws1,
                               sws_bytes, st));
    block_select_write_kernel<<<(unsigned)ntiles, kSelThreads, 0, st>>>(
        len, cs, cd, lo, hi, ntiles, tiles, count, capacity, r_key, r_val, c_key, c_val);
    GNN_LAUNCH_CHECK();
    block_count_add_kernel<<<1, 32, 0, st>>>(count, tiles, ntiles);
    GNN_LAUNCH_CHECK();
  }
  return GNN_OK;
}

// Stable LSD radix sort of int32 (key, val) pairs by key in [0, key_limit)
// (the building block of the block CSR / CSC / coalesced orders).
size_t gnn_sort_pairs_workspace(int64_t n, int64_t key_limit) {
  WsCounter c;
  sort_ws_count(c, n, key_limit > 0 ? key_limit : 1, 1);
  return c.used + 1024;
}

int gnn_sort_pairs(int64_t n, int64_t key_limit, const int32_t *keys, const int32_t *vals,
                   int32_t *keys_out, int32_t *vals_out, void *ws, size_t ws_bytes,
                   gnn_stream_t stream) {
  if (n < 0 || key_limit < 1 || key_limit > ((int64_t)1 << 31) ||
      (n > 0 && (!keys || !vals || !keys_out || !vals_out)))
    return GNN_ERR_INVALID_ARGUMENT;
  if (n >= ((int64_t)1 << 32)) return GNN_ERR_UNSUPPORTED;
  if (ws_bytes < gnn_sort_pairs_workspace(n, key_limit)) return GNN_ERR_WORKSPACE;
  if (n == 0) return GNN_OK;
  WsArena ar(ws, ws_bytes);
  SortIO io{};
  io.n = n;
  io.key_limit = key_limit;
  io.key = SrcDesc{SRC_I32, keys};
  io.nvals = 1;
  io.val[0] = SrcDesc{SRC_I32, vals};
  io.keys_sorted = keys_out;
  io.vals_sorted[0] = vals_out;
  return stable_sort(io, nullptr, ar, as_stream(stream));
}

// offsets[R+1] of sorted int32 keys in [0, R) (run lengths -> exclusive scan)
size_t gnn_offsets_from_keys_workspace(int64_t R) {
  WsCounter c;
  offsets_ws_count(c, R);
  return c.used + 1024;
}

int gnn_offsets_from_keys(int64_t n, int64_t R, const int32_t *sorted_keys, int64_t *offsets,
                          void *ws, size_t ws_bytes, gnn_stream_t stream) {
  if (n < 0 || R < 0 || !offsets || (n > 0 && !sorted_keys)) return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_offsets_from_keys_workspace(R)) return GNN_ERR_WORKSPACE;
  WsArena ar(ws, ws_bytes);
  return offsets_from_sorted(sorted_keys, n, R, offsets, ar, as_stream(stream));
}

size_t gnn_csr_from_edges_workspace(int64_t V, int64_t E) { return edges_ws(V, E); }
int gnn_csr_from_edges(int64_t V, int64_t E, const int64_t *src, const int64_t *dst,
                       int64_t *offsets, int32_t *targets, void *ws, size_t ws_bytes,
                       gnn_stream_t stream) {
  return build_from_edges(0, V, E, src, dst, offsets, targets, ws, ws_bytes, as_stream(stream));
}

size_t gnn_subgraph_csr_workspace(int64_t n, int64_t E) { return edges_ws(n, E); }
int gnn_subgraph_csr(int64_t n, int64_t E, const int64_t *edge_src, const int64_t *edge_dst,
                     int64_t *offsets, int32_t *targets, void *ws, size_t ws_bytes,
                     gnn_stream_t stream) {
  return build_from_edges(1, n, E, edge_src, edge_dst, offsets, targets, ws, ws_bytes,
                          as_stream(stream));
}

size_t gnn_csr_validate_workspace(int64_t V, int64_t E) {
  (void)V;
  (void)E;
  return 256;
}
int gnn_csr_validate(int64_t V, int64_t E, const int64_t *offsets, const int32_t *targets,
                     void *ws, size_t ws_bytes, gnn_stream_t stream) {
  if (V < 0 || E < 0 || !offsets || (E > 0 && !targets) || !ws) return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < sizeof(int)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  int *flags = static_cast<int *>(ws);
  GNN_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(int), st));
  int64_t work = V > E ? V : E;
  validate_kernel<<<grid_for(work, 256), 256, 0, st>>>(offsets, V, E, targets, flags);
  GNN_LAUNCH_CHECK();
  int h = 0;
  GNN_CUDA_TRY(cudaMemcpyAsync(&h, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
  GNN_CUDA_TRY(cudaStreamSynchronize(st));
  if (h & 1) return GNN_ERR_CSR_INVARIANT;
  if (h & 2) return GNN_ERR_RANGE;
  return GNN_OK;
}

int gnn_degrees(int64_t V, const int64_t *offsets, int64_t *deg, gnn_stream_t stream) {
  if (V < 0 || (V > 0 && (!offsets || !deg))) return GNN_ERR_INVALID_ARGUMENT;
  if (V == 0) return GNN_OK;
  cudaStream_t st = as_stream(stream);
  degrees_kernel<<<grid_for(V, 256), 256, 0, st>>>(offsets, V, deg);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

size_t gnn_csc_from_csr_workspace(int64_t R, int64_t C, int64_t nnz) { return csc_ws(R, C, nnz); }
int gnn_csc_from_csr(int64_t R, int64_t C, int64_t nnz, const int64_t *offsets,
                     const int32_t *cols, int64_t *t_offsets, int32_t *t_rows, int32_t *t_eid,
                     void *ws, size_t ws_bytes, gnn_stream_t stream) {
  return csc_impl(R, C, nnz, offsets, cols, t_offsets, t_rows, t_eid, ws, ws_bytes,
                  as_stream(stream));
}

size_t gnn_csr_coalesce_workspace(int64_t R, int64_t nnz) { return coalesce_ws(R, nnz); }
int gnn_csr_coalesce(int64_t R, int64_t nnz, const int64_t *offsets, const int32_t *cols,
                     int64_t *out_offsets, int32_t *out_cols, float *out_mult, int64_t *out_nnz,
                     void *ws, size_t ws_bytes, gnn_stream_t stream) {
  if (R < 0 || nnz < 0 || !offsets || !out_offsets || !out_nnz ||
      (nnz > 0 && (!cols || !out_cols || !out_mult)))
    return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < coalesce_ws(R, nnz)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  WsArena ar(ws, ws_bytes);
  int64_t *u = ar.take<int64_t>(nnz + 1);
  int64_t *start = ar.take<int64_t>(nnz + 1);
  size_t sws_bytes = scan_i64_workspace(nnz);
  void *sws = ar.take<char>((int64_t)sws_bytes);
  if (!ar.ok()) return GNN_ERR_WORKSPACE;
  if (nnz > 0) {
    GNN_CUDA_TRY(cudaMemsetAsync(u, 0, sizeof(int64_t) * nnz, st));
    mark_row_starts_kernel<<<grid_for(R, 256), 256, 0, st>>>(offsets, R, nnz, u);
    GNN_LAUNCH_CHECK();
    mark_col_changes_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(cols, nnz, u);
    GNN_LAUNCH_CHECK();
  }
  GNN_TRY(exclusive_scan_i64(u, u, nnz, true, sws, sws_bytes, st));
  if (nnz > 0) {
    coalesce_scatter_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(cols, nnz, u, out_cols, start);
    GNN_LAUNCH_CHECK();
    coalesce_mult_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(u, nnz, start, out_mult);
    GNN_LAUNCH_CHECK();
  }
  coalesce_offsets_kernel<<<grid_for(R + 1, 256), 256, 0, st>>>(offsets, R, nnz, u, out_offsets);
  GNN_LAUNCH_CHECK();
  GNN_CUDA_TRY(cudaMemcpyAsync(out_nnz, u + nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GNN_CUDA_TRY(cudaStreamSynchronize(st));
  return GNN_OK;
}

__global__ void pack_weights_kernel(const int32_t *__restrict__ cols, const float *__restrict__ w,
                                    int64_t nnz, int col_bits, int32_t *out, int *flag) {
  const uint32_t cmax = 1u << col_bits;  // col_bits <= 31
  const float wmax = (float)(1ull << (32 - col_bits));
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = (uint32_t)cols[j];
    const float x = w[j];
    if (c >= cmax || !(x >= 0.f) || x >= wmax || x != truncf(x)) {
      atomicOr(flag, 1);
      continue;
    }
    out[j] = (int32_t)(c | ((uint32_t)x << col_bits));
  }
}

size_t gnn_csr_pack_weights_workspace(void) { return 256; }
int gnn_csr_pack_weights(int64_t nnz, const int32_t *cols, const float *weights, int32_t col_bits,
                         int32_t *out, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  if (nnz < 0 || col_bits < 1 || col_bits > 31 || (nnz > 0 && (!cols || !weights || !out)) || !ws)
    return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < sizeof(int)) return GNN_ERR_WORKSPACE;
  if (nnz == 0) return GNN_OK;
  cudaStream_t st = as_stream(stream);
  int *flag = static_cast<int *>(ws);
  GNN_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
  pack_weights_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(cols, weights, nnz, col_bits, out, flag);
  GNN_LAUNCH_CHECK();
  int h = 0;
  GNN_CUDA_TRY(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  GNN_CUDA_TRY(cudaStreamSynchronize(st));
  return h ? GNN_ERR_RANGE : GNN_OK;
}

size_t gnn_generate_powerlaw_workspace(int64_t n) {
  (void)n;
  return sizeof(int32_t) * (size_t)(kGuide + 1) + 256;
}
int gnn_generate_powerlaw(int64_t n, int64_t m, const double *cdf, uint64_t state_hi,
                          uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t *src,
                          int64_t *dst, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  if (n < 1 || m < 0 || !cdf || (m > 0 && (!src || !dst))) return GNN_ERR_INVALID_ARGUMENT;
  if (n >= ((int64_t)1 << 31)) return GNN_ERR_UNSUPPORTED;
  if (ws_bytes < gnn_generate_powerlaw_workspace(n)) return GNN_ERR_WORKSPACE;
  if (m == 0) return GNN_OK;
  cudaStream_t st = as_stream(stream);
  int32_t *guide = static_cast<int32_t *>(ws);
  guide_kernel<<<grid_for(kGuide + 1, 256), 256, 0, st>>>(cdf, n, guide);
  GNN_LAUNCH_CHECK();
  int64_t nchunks = ceil_div(2 * m, kGenChunk);
  powerlaw_kernel<<<grid_for(nchunks, 256), 256, 0, st>>>(cdf, n, m, guide, U128{state_hi, state_lo},
                                                          U128{inc_hi, inc_lo}, src, dst);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

}  // extern "C"

// --------------------------------- device-count concatenation (replayable)
// dst[off_in .. off_in + count) = src[0 .. count), *off_out = off_in + count,
// with count and off_in on device (*off_in = 0 when off_in is null): the
// sampled-subgraph assembly of a replayed mini-batch.
template <typename T>
__global__ void append_dev_kernel(T *dst, const T *__restrict__ src, const int64_t *count,
                                  int64_t cap, const int64_t *off_in, int64_t *off_out) {
  const int64_t n = min(*count, cap);
  const int64_t o = off_in ? *off_in : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[o + i] = src[i];
  if (off_out && blockIdx.x == 0 && threadIdx.x == 0) *off_out = o + n;
}
template <typename T>
__global__ void fill_tail_dev_kernel(T *dst, const int64_t *from, int64_t cap, T value) {
  for (int64_t i = *from + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = value;
}

// ------------------------------------------------ row-partition id remap
namespace gnn {
namespace {
__global__ void remap_ids_kernel(int64_t n, const int32_t *__restrict__ ids,
                                 const int64_t *__restrict__ bounds, int64_t P, int64_t stride,
                                 int32_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t id = ids[i];
    int64_t lo = 0, hi = P;  // largest q in [0,P) with bounds[q] <= id
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (bounds[mid] <= id)
        lo = mid;
      else
        hi = mid;
    }
    out[i] = (int32_t)(lo * stride + (id - bounds[lo]));
  }
}
}  // namespace
}  // namespace gnn

extern "C" int gnn_append_dev(void *dst, int64_t elem_bytes, const void *src, const int64_t *count,
                   int64_t cap, const int64_t *off_in, int64_t *off_out, gnn_stream_t stream) {
  if (!dst || !src || !count || cap < 0 || (elem_bytes != 4 && elem_bytes != 8))
    return GNN_ERR_INVALID_ARGUMENT;
  cudaStream_t st = as_stream(stream);
  const unsigned grid = grid_for(cap > 0 ? cap : 1, 256);
  if (elem_bytes == 4)
    append_dev_kernel<int32_t><<<grid, 256, 0, st>>>(static_cast<int32_t *>(dst),
                                                     static_cast<const int32_t *>(src), count, cap,
                                                     off_in, off_out);
  else
    append_dev_kernel<int64_t><<<grid, 256, 0, st>>>(static_cast<int64_t *>(dst),
                                                     static_cast<const int64_t *>(src), count, cap,
                                                     off_in, off_out);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_fill_tail_dev(void *dst, int64_t elem_bytes, const int64_t *from, int64_t cap,
                      int64_t value, gnn_stream_t stream) {
  if (!dst || !from || cap < 0 || (elem_bytes != 4 && elem_bytes != 8)) return GNN_ERR_INVALID_ARGUMENT;
  cudaStream_t st = as_stream(stream);
  const unsigned grid = grid_for(cap > 0 ? cap : 1, 256);
  if (elem_bytes == 4)
    fill_tail_dev_kernel<int32_t><<<grid, 256, 0, st>>>(static_cast<int32_t *>(dst), from, cap,
                                                        (int32_t)value);
  else
    fill_tail_dev_kernel<int64_t><<<grid, 256, 0, st>>>(static_cast<int64_t *>(dst), from, cap, value);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_remap_ids(int64_t n, const int32_t *ids, const int64_t *bounds, int64_t P,
                             int64_t block_stride, int32_t *out, gnn_stream_t stream) {
  using namespace gnn;
  if (n < 0 || P <= 0 || block_stride <= 0 || (n > 0 && (!ids || !bounds || !out)))
    return GNN_ERR_INVALID_ARGUMENT;
  if (P * block_stride >= ((int64_t)1 << 31)) return GNN_ERR_UNSUPPORTED;
  if (n == 0) return GNN_OK;
  cudaStream_t st = as_stream(stream);
  int64_t blocks = ceil_div(n, 256), cap = (int64_t)sm_count() * 16;
  remap_ids_kernel<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, st>>>(n, ids, bounds, P,
                                                                            block_stride, out);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

// ------------------------------------------- device sampled-block pipeline
// sample_hop (sampler.py:118-144) bit-exact with numpy's
// PCG64 stream (same jump-ahead as the generator above) and dedup_relabel
// (sampler.py:191-239) with first-occurrence local ids, deterministic
// (atomicMin of positions is order-independent).  Counts stay on device;
// the Python layer reads them once per hop to size the next hop.
namespace gnn {
namespace {

__global__ void sample_active_flags_kernel(const int64_t *__restrict__ offsets,
                                           const int64_t *__restrict__ frontier, int64_t F,
                                           int64_t *flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < F;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = frontier[i];
    flags[i] = offsets[v + 1] > offsets[v] ? 1 : 0;
  }
}
__global__ void sample_active_scatter_kernel(const int64_t *__restrict__ pos, int64_t F,
                                             int64_t fanout, int64_t *active, int64_t *count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < F;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (pos[i + 1] != pos[i]) active[pos[i]] = i;
    if (i == 0) *count = pos[F] * fanout;
  }
}
// One thread's chunk of kDrawChunk consecutive draws p (the reference's
// draw order: p = active-vertex rank * fanout + j): jump the PCG64 stream to
// p0, then run the chunk in phases — all uniforms, then all vertex lookups,
// then all degree reads, then all target reads — so each phase's loads are
// independent and in flight together instead of one dependent chain per draw.
__device__ __forceinline__ void draw_chunk(const int64_t *__restrict__ offsets,
                                           const int32_t *__restrict__ targets,
                                           const int64_t *__restrict__ frontier,
                                           const int64_t *__restrict__ active, int64_t fanout,
                                           U128 state0, U128 inc, int64_t p0, int64_t n,
                                           int64_t *src, int64_t *dst) {
  U128 s = pcg_advance(state0, inc, (uint64_t)p0);
  double u[kDrawChunk];
  int64_t v[kDrawChunk], base[kDrawChunk], deg[kDrawChunk];
#pragma unroll
  for (int k = 0; k < kDrawChunk; ++k) {
    s = u128_add(u128_mul(s, kPcgMult), inc);
    u[k] = (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
  }
#pragma unroll
  for (int k = 0; k < kDrawChunk; ++k) v[k] = p0 + k < n ? frontier[active[(p0 + k) / fanout]] : 0;
#pragma unroll
  for (int k = 0; k < kDrawChunk; ++k) {
    base[k] = p0 + k < n ? offsets[v[k]] : 0;
    deg[k] = p0 + k < n ? offsets[v[k] + 1] : 0;
  }
  int32_t t[kDrawChunk];
#pragma unroll
  for (int k = 0; k < kDrawChunk; ++k) {
    const int64_t pick = (int64_t)(u[k] * (double)(deg[k] - base[k]));  // numpy astype(int64)
    t[k] = p0 + k < n ? targets[base[k] + pick] : 0;
  }
#pragma unroll
  for (int k = 0; k < kDrawChunk; ++k)
    if (p0 + k < n) {
      src[p0 + k] = v[k];
      dst[p0 + k] = t[k];
    }
}

__global__ void __launch_bounds__(256) sample_draw_kernel(
    const int64_t *__restrict__ offsets, const int32_t *__restrict__ targets,
    const int64_t *__restrict__ frontier, const int64_t *__restrict__ active,
    const int64_t *__restrict__ count, int64_t cap, int64_t fanout, U128 state0, U128 inc,
    int64_t *src, int64_t *dst) {
  const int64_t n = *count;
  const int64_t nchunks = ceil_div(n, kDrawChunk);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    draw_chunk(offsets, targets, frontier, active, fanout, state0, inc, c * kDrawChunk, n, src,
               dst);
  }
}

__global__ void relabel_src_kernel(const int32_t *__restrict__ table, const int64_t *__restrict__ g,
                                   int64_t n, int32_t *out, int32_t *err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = table[g[i]];
    out[i] = l;
    if (l < 0) *err = 1;
  }
}
__global__ void fresh_first_kernel(const int32_t *__restrict__ table, const int64_t *__restrict__ g,
                                   int64_t n, int32_t *firstpos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (table[g[i]] < 0) atomicMin(firstpos + g[i], (int32_t)i);
}
__global__ void first_flags_kernel(const int32_t *__restrict__ table, const int32_t *__restrict__ firstpos,
                                   const int64_t *__restrict__ g, int64_t n, int64_t *flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (table[g[i]] < 0 && firstpos[g[i]] == (int32_t)i) ? 1 : 0;
}
__global__ void assign_new_kernel(const int64_t *__restrict__ rank, const int64_t *__restrict__ g,
                                  int64_t n, int64_t start, int32_t *table, int32_t *firstpos,
                                  int64_t *new_globals, int64_t *new_count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (rank[i + 1] != rank[i]) {
      const int64_t v = g[i];
      new_globals[rank[i]] = v;
      table[v] = (int32_t)(start + rank[i]);
      firstpos[v] = INT32_MAX;  // restore the scratch for the next hop
    }
    if (i == 0) *new_count = rank[n];
  }
}
__global__ void lookup_kernel(const int32_t *__restrict__ table, const int64_t *__restrict__ ids,
                              int64_t n, int32_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = table[ids[i]];
}
__global__ void assign_seq_kernel(int32_t *table, const int64_t *__restrict__ ids, int64_t n,
                                  int64_t start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    table[ids[i]] = (int32_t)(start + i);
}
unsigned grid_for(int64_t n) {
  int64_t b = ceil_div(n > 0 ? n : 1, 256), cap = (int64_t)sm_count() * 16;
  return (unsigned)(b < cap ? b : cap);
}

}  // namespace
}  // namespace gnn

extern "C" {

size_t gnn_sample_hop_workspace(int64_t F) {
  using namespace gnn;
  WsCounter c;
  c.take<int64_t>(F + 1);  // flags / positions
  c.take<int64_t>(F);      // active indices
  c.used += scan_i64_workspace(F) + 256;
  return c.used + 256;
}

int gnn_sample_hop(int64_t V, const int64_t *offsets, const int32_t *targets,
                   const int64_t *frontier, int64_t F, int64_t fanout, uint64_t state_hi,
                   uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t *src, int64_t *dst,
                   int64_t *count, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  using namespace gnn;
  if (V < 0 || F < 0 || fanout < 0 || !offsets || !count || (F > 0 && !frontier))
    return GNN_ERR_INVALID_ARGUMENT;
  if (F * fanout > 0 && (!src || !dst || !targets)) return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_sample_hop_workspace(F)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  if (F == 0 || fanout == 0) {
    GNN_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
    return GNN_OK;
  }
  WsArena ar(ws, ws_bytes);
  int64_t *pos = ar.take<int64_t>(F + 1);
  int64_t *active = ar.take<int64_t>(F);
  size_t sb = scan_i64_workspace(F);
  void *sws = ar.take<char>((int64_t)sb);
  if (!ar.ok()) return GNN_ERR_WORKSPACE;
  sample_active_flags_kernel<<<grid_for(F), 256, 0, st>>>(offsets, frontier, F, pos);
  GNN_LAUNCH_CHECK();
  GNN_TRY(exclusive_scan_i64(pos, pos, F, true, sws, sb, st));
  sample_active_scatter_kernel<<<grid_for(F), 256, 0, st>>>(pos, F, fanout, active, count);
  GNN_LAUNCH_CHECK();
  const U128 s0{state_hi, state_lo}, inc{inc_hi, inc_lo};
  sample_draw_kernel<<<grid_for(ceil_div(F * fanout, kDrawChunk)), 256, 0, st>>>(
      offsets, targets, frontier, active, count, F * fanout, fanout, s0, inc, src, dst);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

size_t gnn_dedup_relabel_workspace(int64_t n) {
  using namespace gnn;
  WsCounter c;
  c.take<int64_t>(n + 1);
  c.used += scan_i64_workspace(n) + 256;
  return c.used + 256;
}

int gnn_dedup_relabel(int64_t V, int32_t *table, int32_t *firstpos, const int64_t *src_g,
                      const int64_t *dst_g, int64_t n, int64_t start, int32_t *src_local,
                      int32_t *dst_local, int64_t *new_globals, int64_t *new_count,
                      int32_t *error_flag, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  using namespace gnn;
  if (V < 0 || n < 0 || start < 0 || !table || !firstpos || !new_count || !error_flag)
    return GNN_ERR_INVALID_ARGUMENT;
  if (n >= ((int64_t)1 << 31) || start + n >= ((int64_t)1 << 31)) return GNN_ERR_UNSUPPORTED;
  if (n > 0 && (!src_g || !dst_g || !src_local || !dst_local || !new_globals))
    return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_dedup_relabel_workspace(n)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  GNN_CUDA_TRY(cudaMemsetAsync(error_flag, 0, sizeof(int32_t), st));
  if (n == 0) {
    GNN_CUDA_TRY(cudaMemsetAsync(new_count, 0, sizeof(int64_t), st));
    return GNN_OK;
  }
  WsArena ar(ws, ws_bytes);
  int64_t *rank = ar.take<int64_t>(n + 1);
  size_t sb = scan_i64_workspace(n);
  void *sws = ar.take<char>((int64_t)sb);
  if (!ar.ok()) return GNN_ERR_WORKSPACE;
  const unsigned gr = grid_for(n);
  relabel_src_kernel<<<gr, 256, 0, st>>>(table, src_g, n, src_local, error_flag);
  GNN_LAUNCH_CHECK();
  fresh_first_kernel<<<gr, 256, 0, st>>>(table, dst_g, n, firstpos);
  GNN_LAUNCH_CHECK();
  first_flags_kernel<<<gr, 256, 0, st>>>(table, firstpos, dst_g, n, rank);
  GNN_LAUNCH_CHECK();
  GNN_TRY(exclusive_scan_i64(rank, rank, n, true, sws, sb, st));
  assign_new_kernel<<<gr, 256, 0, st>>>(rank, dst_g, n, start, table, firstpos, new_globals,
                                        new_count);
  GNN_LAUNCH_CHECK();
  lookup_kernel<<<gr, 256, 0, st>>>(table, dst_g, n, dst_local);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_table_lookup(const int32_t *table, const int64_t *ids, int64_t n, int32_t *out,
                     gnn_stream_t stream) {
  using namespace gnn;
  if (n < 0 || (n > 0 && (!table || !ids || !out))) return GNN_ERR_INVALID_ARGUMENT;
  if (n == 0) return GNN_OK;
  lookup_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(table, ids, n, out);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_table_assign(int32_t *table, const int64_t *ids, int64_t n, int64_t start,
                     gnn_stream_t stream) {
  using namespace gnn;
  if (n < 0 || start < 0 || (n > 0 && (!table || !ids))) return GNN_ERR_INVALID_ARGUMENT;
  if (n == 0) return GNN_OK;
  assign_seq_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(table, ids, n, start);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

}  // extern "C"

// ----------------- device-resident counts: capturable sampling (ZeroGNN DRMB)
// The same pipeline with every size on device: buffers are provisioned for a
// worst-case envelope (capacity), grids cover the capacity and threads past
// the live count exit early, and nothing synchronises
// the host, so a whole mini-batch is one CUDA graph replay.
namespace gnn {
namespace {

__global__ void sample_active_flags_dev_kernel(const int64_t *__restrict__ offsets,
                                               const int64_t *__restrict__ frontier,
                                               const int64_t *__restrict__ F_dev, int64_t cap,
                                               int64_t *flags) {
  const int64_t F = *F_dev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t f = 0;
    if (i < F) {
      const int64_t v = frontier[i];
      f = offsets[v + 1] > offsets[v] ? 1 : 0;
    }
    flags[i] = f;
  }
}
__global__ void relabel_src_dev_kernel(const int32_t *__restrict__ table,
                                       const int64_t *__restrict__ g, const int64_t *__restrict__ n_dev,
                                       int64_t cap, int32_t *out, int32_t *err) {
  const int64_t n = *n_dev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < min(n, cap);
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = table[g[i]];
    out[i] = l;
    if (l < 0) *err = 1;
  }
}
__global__ void fresh_first_dev_kernel(const int32_t *__restrict__ table,
                                       const int64_t *__restrict__ g, const int64_t *__restrict__ n_dev,
                                       int64_t cap, int32_t *firstpos) {
  const int64_t n = *n_dev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < min(n, cap);
       i += (int64_t)gridDim.x * blockDim.x)
    if (table[g[i]] < 0) atomicMin(firstpos + g[i], (int32_t)i);
}
__global__ void first_flags_dev_kernel(const int32_t *__restrict__ table,
                                       const int32_t *__restrict__ firstpos,
                                       const int64_t *__restrict__ g, const int64_t *__restrict__ n_dev,
                                       int64_t cap, int64_t *flags) {
  const int64_t n = *n_dev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i < n && table[g[i]] < 0 && firstpos[g[i]] == (int32_t)i) ? 1 : 0;
}
__global__ void assign_new_dev_kernel(const int64_t *__restrict__ rank, const int64_t *__restrict__ g,
                                      const int64_t *__restrict__ n_dev, int64_t cap,
                                      const int64_t *__restrict__ size_dev, int32_t *table,
                                      int32_t *firstpos, int64_t *new_globals, int64_t *new_count) {
  const int64_t n = min(*n_dev, cap), start = *size_dev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (rank[i + 1] != rank[i]) {
      const int64_t v = g[i];
      new_globals[rank[i]] = v;
      table[v] = (int32_t)(start + rank[i]);
      firstpos[v] = INT32_MAX;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *new_count = rank[cap];
}
__global__ void lookup_dev_kernel(const int32_t *__restrict__ table, const int64_t *__restrict__ ids,
                                  const int64_t *__restrict__ n_dev, int64_t cap, int32_t *out) {
  const int64_t n = min(*n_dev, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = table[ids[i]];
}
__global__ void size_add_kernel(int64_t *size_dev, const int64_t *__restrict__ add) {
  *size_dev += *add;
}
__global__ void sample_draw_dev_kernel(const int64_t *__restrict__ offsets,
                                       const int32_t *__restrict__ targets,
                                       const int64_t *__restrict__ frontier,
                                       const int64_t *__restrict__ active,
                                       const int64_t *__restrict__ count, int64_t fanout,
                                       const uint64_t *__restrict__ rng, int64_t *src, int64_t *dst) {
  const U128 state0{rng[0], rng[1]}, inc{rng[2], rng[3]};
  const int64_t n = *count;
  const int64_t nchunks = ceil_div(n, kDrawChunk);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    draw_chunk(offsets, targets, frontier, active, fanout, state0, inc, c * kDrawChunk, n, src,
               dst);
  }
}

}  // namespace
}  // namespace gnn

extern "C" {

size_t gnn_sample_hop_dev_workspace(int64_t F_cap) { return gnn_sample_hop_workspace(F_cap); }

int gnn_sample_hop_dev(int64_t V, const int64_t *offsets, const int32_t *targets,
                       const int64_t *frontier, const int64_t *F_dev, int64_t F_cap, int64_t fanout,
                       const uint64_t *rng_state, int64_t *src, int64_t *dst, int64_t *count,
                       void *ws, size_t ws_bytes, gnn_stream_t stream) {
  using namespace gnn;
  if (V < 0 || F_cap < 0 || fanout < 0 || !offsets || !F_dev || !count || !rng_state)
    return GNN_ERR_INVALID_ARGUMENT;
  if (F_cap * fanout > 0 && (!src || !dst || !targets || !frontier)) return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_sample_hop_dev_workspace(F_cap)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  if (F_cap == 0 || fanout == 0) {
    GNN_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
    return GNN_OK;
  }
  WsArena ar(ws, ws_bytes);
  int64_t *pos = ar.take<int64_t>(F_cap + 1);
  int64_t *active = ar.take<int64_t>(F_cap);
  size_t sb = scan_i64_workspace(F_cap);
  void *sws = ar.take<char>((int64_t)sb);
  if (!ar.ok()) return GNN_ERR_WORKSPACE;
  sample_active_flags_dev_kernel<<<grid_for(F_cap), 256, 0, st>>>(offsets, frontier, F_dev, F_cap,
                                                                   pos);
  GNN_LAUNCH_CHECK();
  GNN_TRY(exclusive_scan_i64(pos, pos, F_cap, true, sws, sb, st));
  sample_active_scatter_kernel<<<grid_for(F_cap), 256, 0, st>>>(pos, F_cap, fanout, active, count);
  GNN_LAUNCH_CHECK();
  sample_draw_dev_kernel<<<grid_for(ceil_div(F_cap * fanout, kDrawChunk)), 256, 0, st>>>(
      offsets, targets, frontier, active, count, fanout, rng_state, src, dst);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

size_t gnn_dedup_relabel_dev_workspace(int64_t n_cap) { return gnn_dedup_relabel_workspace(n_cap); }

int gnn_dedup_relabel_dev(int64_t V, int32_t *table, int32_t *firstpos, const int64_t *src_g,
                          const int64_t *dst_g, const int64_t *n_dev, int64_t n_cap,
                          int64_t *size_dev, int32_t *src_local, int32_t *dst_local,
                          int64_t *new_globals, int64_t *new_count, int32_t *error_flag, void *ws,
                          size_t ws_bytes, gnn_stream_t stream) {
  using namespace gnn;
  if (V < 0 || n_cap < 0 || !table || !firstpos || !n_dev || !size_dev || !new_count || !error_flag)
    return GNN_ERR_INVALID_ARGUMENT;
  if (n_cap >= ((int64_t)1 << 31)) return GNN_ERR_UNSUPPORTED;
  if (n_cap > 0 && (!src_g || !dst_g || !src_local || !dst_local || !new_globals))
    return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_dedup_relabel_dev_workspace(n_cap)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  if (n_cap == 0) {
    GNN_CUDA_TRY(cudaMemsetAsync(new_count, 0, sizeof(int64_t), st));
    return GNN_OK;
  }
  WsArena ar(ws, ws_bytes);
  int64_t *rank = ar.take<int64_t>(n_cap + 1);
  size_t sb = scan_i64_workspace(n_cap);
  void *sws = ar.take<char>((int64_t)sb);
  if (!ar.ok()) return GNN_ERR_WORKSPACE;
  const unsigned gr = grid_for(n_cap);
  relabel_src_dev_kernel<<<gr, 256, 0, st>>>(table, src_g, n_dev, n_cap, src_local, error_flag);
  GNN_LAUNCH_CHECK();
  fresh_first_dev_kernel<<<gr, 256, 0, st>>>(table, dst_g, n_dev, n_cap, firstpos);
  GNN_LAUNCH_CHECK();
  first_flags_dev_kernel<<<gr, 256, 0, st>>>(table, firstpos, dst_g, n_dev, n_cap, rank);
  GNN_LAUNCH_CHECK();
  GNN_TRY(exclusive_scan_i64(rank, rank, n_cap, true, sws, sb, st));
  assign_new_dev_kernel<<<gr, 256, 0, st>>>(rank, dst_g, n_dev, n_cap, size_dev, table, firstpos,
                                            new_globals, new_count);
  GNN_LAUNCH_CHECK();
  lookup_dev_kernel<<<gr, 256, 0, st>>>(table, dst_g, n_dev, n_cap, dst_local);
  GNN_LAUNCH_CHECK();
  size_add_kernel<<<1, 1, 0, st>>>(size_dev, new_count);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_table_lookup_dev(const int32_t *table, const int64_t *ids, const int64_t *n_dev,
                         int64_t n_cap, int32_t *out, gnn_stream_t stream) {
  using namespace gnn;
  if (n_cap < 0 || !n_dev || (n_cap > 0 && (!table || !ids || !out))) return GNN_ERR_INVALID_ARGUMENT;
  if (n_cap == 0) return GNN_OK;
  lookup_dev_kernel<<<grid_for(n_cap), 256, 0, as_stream(stream)>>>(table, ids, n_dev, n_cap, out);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

}  // extern "C"

namespace gnn {
namespace {
__global__ void fill_dev_kernel(int32_t *table, const int64_t *__restrict__ ids,
                                const int64_t *__restrict__ n_dev, int64_t cap, int32_t value) {
  const int64_t n = n_dev ? min(*n_dev, cap) : cap;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    table[ids[i]] = value;
}
}  // namespace
}  // namespace gnn

extern "C" int gnn_table_fill_dev(int32_t *table, const int64_t *ids, const int64_t *n_dev,
                                  int64_t n_cap, int32_t value, gnn_stream_t stream) {
  using namespace gnn;
  if (n_cap < 0 || (n_cap > 0 && (!table || !ids))) return GNN_ERR_INVALID_ARGUMENT;
  if (n_cap == 0) return GNN_OK;
  fill_dev_kernel<<<grid_for(n_cap), 256, 0, as_stream(stream)>>>(table, ids, n_dev, n_cap, value);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

// Feature gather of a sampled mini-batch (the reference pipeline's "gather"
// kernel class, execmodel.py:306-314): out[i, :] = X[ids[i], :].
namespace gnn {
namespace {
// n_dev (optional): the live row count on device; rows at or past it are not
// written (replayed mini-batches over a capacity-sized buffer)
__global__ void gather_rows_vec_kernel(const float4 *__restrict__ X, int64_t ldx4,
                                       const int64_t *__restrict__ ids, int64_t n, int64_t K4,
                                       float4 *out, int64_t ldo4, const int64_t *n_dev) {
  if (n_dev) n = min(n, *n_dev);
  const int64_t total = n * K4;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / K4, k = t % K4;
    out[i * ldo4 + k] = __ldg(X + ids[i] * ldx4 + k);
  }
}
__global__ void gather_rows_v2_kernel(const float2 *__restrict__ X, int64_t ldx2,
                                      const int64_t *__restrict__ ids, int64_t n, int64_t K2,
                                      float2 *out, int64_t ldo2, const int64_t *n_dev) {
  if (n_dev) n = min(n, *n_dev);
  const int64_t total = n * K2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / K2, k = t % K2;
    out[i * ldo2 + k] = __ldg(X + ids[i] * ldx2 + k);
  }
}
__global__ void gather_rows_kernel(const float *__restrict__ X, int64_t ldx,
                                   const int64_t *__restrict__ ids, int64_t n, int64_t K,
                                   float *out, int64_t ldo, const int64_t *n_dev) {
  if (n_dev) n = min(n, *n_dev);
  const int64_t total = n * K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / K, k = t % K;
    out[i * ldo + k] = __ldg(X + ids[i] * ldx + k);
  }
}
}  // namespace
}  // namespace gnn

namespace gnn {
namespace {
int gather_rows_impl(const float *X, int64_t ldx, const int64_t *ids, int64_t n, int64_t K,
                     float *out, int64_t ldo, const int64_t *n_dev, cudaStream_t st) {
  if (n < 0 || K < 0 || ldx < K || ldo < K || (n > 0 && K > 0 && (!X || !ids || !out)))
    return GNN_ERR_INVALID_ARGUMENT;
  if (n == 0 || K == 0) return GNN_OK;
  const bool v4 = K % 4 == 0 && ldx % 4 == 0 && ldo % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(X) & 15u) == 0 &&
                  (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  if (v4) {
    gather_rows_vec_kernel<<<grid_for(n * K / 4), 256, 0, st>>>(
        reinterpret_cast<const float4 *>(X), ldx / 4, ids, n, K / 4,
        reinterpret_cast<float4 *>(out), ldo / 4, n_dev);
  } else if (K % 2 == 0 && ldx % 2 == 0 && ldo % 2 == 0 &&
             (reinterpret_cast<uintptr_t>(X) & 7u) == 0 && (reinterpret_cast<uintptr_t>(out) & 7u) == 0) {
    // 8-byte vectors (e.g. Reddit's 602 features: rows of 2408 B)
    gather_rows_v2_kernel<<<grid_for(n * K / 2), 256, 0, st>>>(
        reinterpret_cast<const float2 *>(X), ldx / 2, ids, n, K / 2,
        reinterpret_cast<float2 *>(out), ldo / 2, n_dev);
  } else {
    gather_rows_kernel<<<grid_for(n * K), 256, 0, st>>>(X, ldx, ids, n, K, out, ldo, n_dev);
  }
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}
}  // namespace
}  // namespace gnn

extern "C" int gnn_gather_rows(const float *X, int64_t ldx, const int64_t *ids, int64_t n,
                               int64_t K, float *out, int64_t ldo, gnn_stream_t stream) {
  return gnn::gather_rows_impl(X, ldx, ids, n, K, out, ldo, nullptr, gnn::as_stream(stream));
}

extern "C" int gnn_gather_rows_dev(const float *X, int64_t ldx, const int64_t *ids,
                                   const int64_t *n_dev, int64_t n_cap, int64_t K, float *out,
                                   int64_t ldo, gnn_stream_t stream) {
  if (!n_dev) return GNN_ERR_INVALID_ARGUMENT;
  return gnn::gather_rows_impl(X, ldx, ids, n_cap, K, out, ldo, n_dev, gnn::as_stream(stream));
}
