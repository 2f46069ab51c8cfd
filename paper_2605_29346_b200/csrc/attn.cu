// SDDMM, edge-softmax and the GAT per-vertex helpers (GraphPy class-A
// kernels; GAT math of SURVEY.md Appendix A.6).
//
// Work decomposition: every edge kernel reuses the SpMM plan of the operand
// (gnn_spmm_plan_t): the nnz range is cut into chunks of P edges, one warp per
// chunk, chunk_row[w] = row of the chunk's first edge.  A warp walks the rows
// of its chunk in order, so the row side of every edge (X[row] for SDDMM,
// er[row] for GAT scores, the softmax row statistics) is loaded once per row
// piece and reused across its edges ("row-run reuse") —
// there is no materialised COO row array.
//
// Edge-softmax is a per-row reduction over edges; rows that span several
// chunks (the power-law mega rows) leave per-chunk partial statistics in
// workspace slots, a finalize kernel combines them in a fixed order, and an
// apply kernel normalises those rows' edges.  Rows inside one chunk are
// finished in the first kernel.  Every summation order is fixed: results are
// deterministic run to run, no atomics.
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace gnn {
namespace {

constexpr float kNegInf = -INFINITY;

unsigned grid_warps(int64_t nwarps, int threads) {
  return (unsigned)ceil_div(nwarps * 32, threads);
}
unsigned grid_1d_a(int64_t n, int threads) {
  int64_t b = ceil_div(n > 0 ? n : 1, threads);
  int64_t cap = (int64_t)sm_count() * 32;
  return (unsigned)(b < cap ? b : cap);
}
bool al16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Walks the rows of one chunk [e0,e1): row r with bounds [rs,re); offsets are
// fetched 32 row-ends per batched load and broadcast by shuffle.
struct RowWalk {
  const int64_t *off;
  int64_t R, r, rs, re, obuf;
  int bi;
  __device__ __forceinline__ RowWalk(const int64_t *o, int64_t nrows, int64_t r0) : off(o), R(nrows) {
    r = r0;
    rs = off[r];
    obuf = off[min(r + 1 + (int64_t)lane_id(), R)];
    bi = 0;
    re = shfl64(obuf, 0);
  }
  static __device__ __forceinline__ int64_t shfl64(int64_t v, int src) {
    int lo = __shfl_sync(kFull, (int)(v & 0xffffffff), src);
    int hi = __shfl_sync(kFull, (int)(v >> 32), src);
    return ((int64_t)hi << 32) | (uint32_t)lo;
  }
  // advance to the next row (whole warp)
  __device__ __forceinline__ void next() {
    ++r;
    rs = re;
    if (++bi == 32) {
      obuf = off[min(r + 1 + (int64_t)lane_id(), R)];
      bi = 0;
    }
    re = shfl64(obuf, bi);
  }
};

// ------------------------------------------------------------------ SDDMM
struct SddmmArgs {
  int64_t R, nnz, P, nwarps;
  const int64_t *offsets;
  const int32_t *cols;
  const int32_t *chunk_row;
  int H;
  int64_t F, K;
  const float *X;  // row side  [R, ldx]
  int64_t ldx;
  const float *Y;  // col side  [C, ldy]
  int64_t ldy;
  float *out;      // [nnz, H]
};

// Fast path: G lanes per edge, each lane owns float4 columns q = v*G + gl
// (v < VPL); LPH = F/4 lanes per head (power of two, <= G) reduce a head's dot
// by xor shuffles inside the group.  NG = 32/G edges per warp step, U steps
// unrolled so U gathers per lane are in flight.
// HM > 0 selects the general head mapping (any F % 4 == 0): each lane sums
// its vectors per head in registers and every head is reduced over the whole
// G-lane group; group lane 0 writes the edge's H outputs.
template <int G, int VPL, int HM>
__global__ void __launch_bounds__(256) sddmm_vec_kernel(SddmmArgs a, int LPH) {
  constexpr int NG = 32 / G;
  constexpr int U = VPL >= 2 ? 2 : 4;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= a.nwarps) return;
  const int lane = (int)lane_id();
  const int g = lane / G, gl = lane % G;
  const unsigned gmask = G == 32 ? kFull : (((1u << G) - 1u) << (g * G));
  const int64_t e0 = w * a.P, e1 = min(e0 + a.P, a.nnz);
  int64_t col[VPL];
  bool cv[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    col[v] = (int64_t)(v * G + gl) * 4;
    cv[v] = col[v] < a.K;
    if (!cv[v]) col[v] = 0;
  }
  int64_t r = a.chunk_row[w];
  int64_t re = a.offsets[r + 1];
  int64_t xr = -1;
  float4 xv[VPL];
  for (int64_t eb = e0 + g; eb < e1; eb += (int64_t)NG * U) {
    int32_t c[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = eb + (int64_t)u * NG;
      ok[u] = e < e1;
      c[u] = ok[u] ? __ldg(a.cols + e) : 0;
    }
    float4 yv[U][VPL];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        yv[u][v] = ok[u] ? ldg_f4(a.Y + (int64_t)c[u] * a.ldy + col[v]) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) break;  // group-uniform
      const int64_t e = eb + (int64_t)u * NG;
      while (e >= re) {
        ++r;
        re = a.offsets[r + 1];
      }
      if (r != xr) {
        xr = r;
#pragma unroll
        for (int v = 0; v < VPL; ++v) xv[v] = ldg_f4(a.X + r * a.ldx + col[v]);
      }
      if constexpr (HM == 0) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          float p = xv[v].x * yv[u][v].x;
          p = fmaf(xv[v].y, yv[u][v].y, p);
          p = fmaf(xv[v].z, yv[u][v].z, p);
          p = fmaf(xv[v].w, yv[u][v].w, p);
          for (int o = 1; o < LPH; o <<= 1) p += __shfl_xor_sync(gmask, p, o);
          if (cv[v] && (gl & (LPH - 1)) == 0) a.out[e * a.H + col[v] / a.F] = p;
        }
      } else {
        float ph[HM];
#pragma unroll
        for (int h = 0; h < HM; ++h) ph[h] = 0.f;
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          float p = xv[v].x * yv[u][v].x;
          p = fmaf(xv[v].y, yv[u][v].y, p);
          p = fmaf(xv[v].z, yv[u][v].z, p);
          p = fmaf(xv[v].w, yv[u][v].w, p);
          if (cv[v]) {
            const int hv = (int)(col[v] / a.F);
#pragma unroll
            for (int h = 0; h < HM; ++h) ph[h] += h == hv ? p : 0.f;
          }
        }
#pragma unroll
        for (int o = 1; o < G; o <<= 1)
#pragma unroll
          for (int h = 0; h < HM; ++h) ph[h] += __shfl_xor_sync(gmask, ph[h], o);
        if (gl == 0) {
          if (HM == 4 && a.H == 4 && (reinterpret_cast<uintptr_t>(a.out) & 15u) == 0) {
            *reinterpret_cast<float4 *>(a.out + e * 4) = make_float4(ph[0], ph[1], ph[2], ph[3]);
          } else {
#pragma unroll
            for (int h = 0; h < HM; ++h)
              if (h < a.H) a.out[e * a.H + h] = ph[h];
          }
        }
      }
    }
  }
}

// Generic path (any F, K): one lane per (edge), loop heads and features.
__global__ void __launch_bounds__(256) sddmm_scalar_kernel(SddmmArgs a) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= a.nwarps) return;
  const int lane = (int)lane_id();
  const int64_t e0 = w * a.P, e1 = min(e0 + a.P, a.nnz);
  int64_t r = a.chunk_row[w];
  int64_t re = a.offsets[r + 1];
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    while (e >= re) {
      ++r;
      re = a.offsets[r + 1];
    }
    const int64_t c = a.cols[e];
    const float *x = a.X + r * a.ldx;
    const float *y = a.Y + c * a.ldy;
    for (int h = 0; h < a.H; ++h) {
      float p = 0.f;
      for (int64_t f = h * a.F; f < (h + 1) * a.F; ++f) p = fmaf(__ldg(x + f), __ldg(y + f), p);
      a.out[e * a.H + h] = p;
    }
  }
}

// ------------------------------------------------------------ edge softmax
// Scores: either given (s[e*H+h]) or the GAT score computed on the fly,
// LeakyReLU(el[col*H+h] + er[row*H+h], slope).
struct SoftmaxArgs {
  int64_t R, nnz, P, nwarps;
  const int64_t *offsets;
  const int32_t *cols;
  const int32_t *chunk_row;
  const int32_t *chunk_split;
  const int32_t *split_rows;
  int64_t num_split;
  int H;
  const float *s;
  const float *el, *er;
  float slope;
  // forward
  float *alpha;
  // backward
  const float *alpha_in;
  const float *dalpha;
  float *ds;
  // workspace
  float *slots;  // [nwarps][2][2*H]
  float *stat;   // [num_split][2*H]
  // optional forward output: per-row (max, 1/sum) [R][2*H] — lets a backward
  // pass recompute alpha = exp(s - max) * (1/sum) bit-identically
  float *mstat;
  // segment sum: out[r,h] = sum over row r of vals[(eid ? eid[j] : j)*H + h]
  const int32_t *eid;
};

template <int HM>
struct Scores {
  float v[HM];
};

// Load the H scores of edge e (row r): GAT mode recomputes them from el/er.
template <int HM, bool GAT>
__device__ __forceinline__ void load_scores(const SoftmaxArgs &a, int64_t e, const float (&erow)[HM],
                                            float (&s)[HM]) {
  if constexpr (GAT) {
    const int64_t c = a.cols[e];
    if (HM == 4 && a.H == 4) {
      const float4 l = ldg_f4(a.el + c * 4);
      s[0] = l.x + erow[0];
      s[1] = l.y + erow[1];
      s[2] = l.z + erow[2];
      s[3] = l.w + erow[3];
    } else {
#pragma unroll
      for (int h = 0; h < HM; ++h) s[h] = h < a.H ? __ldg(a.el + c * a.H + h) + erow[h] : 0.f;
    }
#pragma unroll
    for (int h = 0; h < HM; ++h) s[h] = s[h] > 0.f ? s[h] : a.slope * s[h];
  } else {
    if (HM == 4 && a.H == 4) {
      const float4 l = *reinterpret_cast<const float4 *>(a.s + e * 4);
      s[0] = l.x;
      s[1] = l.y;
      s[2] = l.z;
      s[3] = l.w;
    } else {
#pragma unroll
      for (int h = 0; h < HM; ++h) s[h] = h < a.H ? a.s[e * a.H + h] : 0.f;
    }
  }
}

template <int HM, bool GAT>
__device__ __forceinline__ void load_erow(const SoftmaxArgs &a, int64_t r, float (&erow)[HM]) {
#pragma unroll
  for (int h = 0; h < HM; ++h) erow[h] = (GAT && h < a.H) ? __ldg(a.er + r * a.H + h) : 0.f;
}

__device__ __forceinline__ float rescale(float mo, float mn) {
  return mo == kNegInf ? 0.f : expf(mo - mn);
}
// (m,l) <- combine((m,l), (m2,l2)): online-softmax merge, fixed operand order.
__device__ __forceinline__ void ml_merge(float &m, float &l, float m2, float l2) {
  const float mn = fmaxf(m, m2);
  l = l * rescale(m, mn) + l2 * rescale(m2, mn);
  m = mn;
}

template <int HM>
__device__ __forceinline__ void warp_ml_reduce(float (&m)[HM], float (&l)[HM]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int h = 0; h < HM; ++h) {
      const float m2 = __shfl_xor_sync(kFull, m[h], o);
      const float l2 = __shfl_xor_sync(kFull, l[h], o);
      ml_merge(m[h], l[h], m2, l2);
    }
}

// All-reduce of 4 per-head values over the warp in 10 shuffles instead of
// 20: transpose-butterfly (after the bit-16 and bit-8 steps each lane holds
// one head, reduced over the lanes that differ in those bits), a 3-step tree
// over the remaining 8 lanes, then a broadcast of each head from lane 8h.
// Deterministic (fixed pairing); every lane ends with all four totals.
template <bool MAX>
__device__ __forceinline__ void warp_allreduce4(float (&t)[4]) {
  auto op = [](float x, float y) { return MAX ? fmaxf(x, y) : x + y; };
  const int lane = (int)lane_id();
  const bool u16 = (lane & 16) != 0, u8 = (lane & 8) != 0;
  float a0 = u16 ? t[2] : t[0], a1 = u16 ? t[3] : t[1];
  const float b0 = u16 ? t[0] : t[2], b1 = u16 ? t[1] : t[3];
  a0 = op(a0, __shfl_xor_sync(kFull, b0, 16));
  a1 = op(a1, __shfl_xor_sync(kFull, b1, 16));
  float k = u8 ? a1 : a0;
  k = op(k, __shfl_xor_sync(kFull, u8 ? a0 : a1, 8));
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) k = op(k, __shfl_xor_sync(kFull, k, o));
#pragma unroll
  for (int h = 0; h < 4; ++h) t[h] = __shfl_sync(kFull, k, 8 * h);
}

template <int HM>
__device__ __forceinline__ void warp_sum_reduce(float (&t)[HM]) {
  if constexpr (HM == 4) {
    warp_allreduce4<false>(t);
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int h = 0; h < HM; ++h) t[h] += __shfl_xor_sync(kFull, t[h], o);
  }
}

// Forward statistics + normalisation of one row piece [lo,hi) of row r:
// pass 1 row max, pass 2 sum of exp(s - max), pass 3 (whole rows) writes
// alpha — plain max / sum warp trees (an online (m,l) merge in the tree costs
// two exponentials per level per head).  Scores are recomputed per pass; the
// column ids and el rows are L1-resident after the first.
template <int HM>
__device__ __forceinline__ void warp_max_reduce(float (&t)[HM]) {
  if constexpr (HM == 4) {
    warp_allreduce4<true>(t);
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int h = 0; h < HM; ++h) t[h] = fmaxf(t[h], __shfl_xor_sync(kFull, t[h], o));
  }
}

// GAT, 4 heads, rows longer than a warp: two passes instead of three, each
// with 4 edges per lane in flight (column ids first, then the four el rows —
// the dependent id -> el chain is paid once per 4 edges).  Pass 1 keeps a
// per-lane online (max, sum): l <- s > m ? l e^(m-s) + 1 : l + e^(s-m), one
// exponential per edge and head, merged by a fixed xor tree; pass 2 (whole
// rows) writes alpha = e^(s-m) / l.
#ifndef GNN_SOFTMAX_ONLINE
#define GNN_SOFTMAX_ONLINE 1
#endif
constexpr int kSmU = 4;

__device__ __forceinline__ void gat4_scores(const SoftmaxArgs &a, int64_t e0, int64_t hi,
                                            const float (&erow)[4], float (&s)[kSmU][4]) {
  int32_t c[kSmU];
#pragma unroll
  for (int u = 0; u < kSmU; ++u) c[u] = e0 + 32 * u < hi ? a.cols[e0 + 32 * u] : -1;
#pragma unroll
  for (int u = 0; u < kSmU; ++u) {
    const float4 l = c[u] >= 0 ? ldg_f4(a.el + (int64_t)c[u] * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float t[4] = {l.x + erow[0], l.y + erow[1], l.z + erow[2], l.w + erow[3]};
#pragma unroll
    for (int h = 0; h < 4; ++h) s[u][h] = t[h] > 0.f ? t[h] : a.slope * t[h];
  }
}

__device__ __forceinline__ void gat4_write_alpha(const SoftmaxArgs &a, int64_t lo, int64_t hi,
                                                 const float (&erow)[4], const float (&m)[4],
                                                 const float (&inv)[4]) {
  const int lane = (int)lane_id();
  for (int64_t e0 = lo + lane; e0 < hi; e0 += 32 * kSmU) {
    float s[kSmU][4];
    gat4_scores(a, e0, hi, erow, s);
#pragma unroll
    for (int u = 0; u < kSmU; ++u)
      if (e0 + 32 * u < hi)
        *reinterpret_cast<float4 *>(a.alpha + (e0 + 32 * u) * 4) =
            make_float4(__expf(s[u][0] - m[0]) * inv[0], __expf(s[u][1] - m[1]) * inv[1],
                        __expf(s[u][2] - m[2]) * inv[2], __expf(s[u][3] - m[3]) * inv[3]);
  }
}

__device__ __forceinline__ void softmax_piece_gat4(const SoftmaxArgs &a, int64_t r, int64_t lo,
                                                   int64_t hi, bool whole, float *slot,
                                                   const float (&erow)[4]) {
  const int lane = (int)lane_id();
  float m[4], l[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    m[h] = kNegInf;
    l[h] = 0.f;
  }
  for (int64_t e0 = lo + lane; e0 < hi; e0 += 32 * kSmU) {
    float s[kSmU][4];
    gat4_scores(a, e0, hi, erow, s);
#pragma unroll
    for (int u = 0; u < kSmU; ++u)
      if (e0 + 32 * u < hi)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float d = s[u][h] - m[h];
          const float t = __expf(-fabsf(d));  // e^(m-s) when s > m (m = -inf: 0)
          const bool up = d > 0.f;
          l[h] = up ? fmaf(l[h], t, 1.f) : l[h] + t;
          m[h] = up ? s[u][h] : m[h];
        }
  }
  warp_ml_reduce<4>(m, l);
  if (!whole) {
    if (lane == 0)
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        slot[h] = m[h];
        slot[4 + h] = l[h];
      }
    return;
  }
  float inv[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) inv[h] = 1.f / l[h];
  if (a.mstat && lane == 0) {
    reinterpret_cast<float4 *>(a.mstat + r * 8)[0] = make_float4(m[0], m[1], m[2], m[3]);
    reinterpret_cast<float4 *>(a.mstat + r * 8)[1] = make_float4(inv[0], inv[1], inv[2], inv[3]);
  }
  gat4_write_alpha(a, lo, hi, erow, m, inv);
}

template <int HM, bool GAT>
__device__ __forceinline__ void softmax_piece(const SoftmaxArgs &a, int64_t r, int64_t lo, int64_t hi,
                                              bool whole, float *slot) {
  const int lane = (int)lane_id();
  float erow[HM];
  load_erow<HM, GAT>(a, r, erow);
  float m[HM], l[HM];
#pragma unroll
  for (int h = 0; h < HM; ++h) {
    m[h] = kNegInf;
    l[h] = 0.f;
  }
  if (whole && hi - lo <= 32) {
    // one edge per lane: the scores stay in registers for all three passes
    // (the general path below re-derives them per pass); same accumulation
    // order as the general path, so results are identical.  (Two edges per
    // lane for rows <= 64 measured slower: registers.)
    const int64_t e = lo + lane;
    const bool ok = e < hi;
    float sv[HM];
    if (ok) {
      load_scores<HM, GAT>(a, e, erow, sv);
    } else {
#pragma unroll
      for (int h = 0; h < HM; ++h) sv[h] = kNegInf;
    }
#pragma unroll
    for (int h = 0; h < HM; ++h) m[h] = sv[h];
    warp_max_reduce<HM>(m);
    float ex[HM];
#pragma unroll
    for (int h = 0; h < HM; ++h) {
      ex[h] = ok ? __expf(sv[h] - m[h]) : 0.f;
      l[h] = ex[h];
    }
    warp_sum_reduce<HM>(l);
    if (a.mstat && lane == 0)
#pragma unroll
      for (int h = 0; h < HM; ++h)
        if (h < a.H) {
          a.mstat[r * 2 * a.H + h] = m[h];
          a.mstat[r * 2 * a.H + a.H + h] = 1.f / l[h];
        }
    if (ok) {
      if (HM == 4 && a.H == 4) {
        *reinterpret_cast<float4 *>(a.alpha + e * 4) =
            make_float4(ex[0] * (1.f / l[0]), ex[1] * (1.f / l[1]), ex[2] * (1.f / l[2]),
                        ex[3] * (1.f / l[3]));
      } else {
#pragma unroll
        for (int h = 0; h < HM; ++h)
          if (h < a.H) a.alpha[e * a.H + h] = ex[h] * (1.f / l[h]);
      }
    }
    return;
  }
  if constexpr (GAT && HM == 4 && GNN_SOFTMAX_ONLINE) {
    if (a.H == 4) {
      softmax_piece_gat4(a, r, lo, hi, whole, slot, erow);
      return;
    }
  }
  for (int64_t e = lo + lane; e < hi; e += 32) {
    float s[HM];
    load_scores<HM, GAT>(a, e, erow, s);
#pragma unroll
    for (int h = 0; h < HM; ++h) m[h] = fmaxf(m[h], s[h]);
  }
  warp_max_reduce<HM>(m);
  for (int64_t e = lo + lane; e < hi; e += 32) {
    float s[HM];
    load_scores<HM, GAT>(a, e, erow, s);
#pragma unroll
    for (int h = 0; h < HM; ++h) l[h] += __expf(s[h] - m[h]);
  }
  warp_sum_reduce<HM>(l);
  if (!whole) {
    if (lane == 0)
#pragma unroll
      for (int h = 0; h < HM; ++h)
        if (h < a.H) {
          slot[h] = m[h];
          slot[a.H + h] = l[h];
        }
    return;
  }
  float inv[HM];
#pragma unroll
  for (int h = 0; h < HM; ++h) inv[h] = 1.f / l[h];
  if (a.mstat && lane == 0)
#pragma unroll
    for (int h = 0; h < HM; ++h)
      if (h < a.H) {
        a.mstat[r * 2 * a.H + h] = m[h];
        a.mstat[r * 2 * a.H + a.H + h] = inv[h];
      }
  for (int64_t e = lo + lane; e < hi; e += 32) {
    float s[HM];
    load_scores<HM, GAT>(a, e, erow, s);
    if (HM == 4 && a.H == 4) {
      *reinterpret_cast<float4 *>(a.alpha + e * 4) =
          make_float4(__expf(s[0] - m[0]) * inv[0], __expf(s[1] - m[1]) * inv[1],
                      __expf(s[2] - m[2]) * inv[2], __expf(s[3] - m[3]) * inv[3]);
    } else {
#pragma unroll
      for (int h = 0; h < HM; ++h)
        if (h < a.H) a.alpha[e * a.H + h] = __expf(s[h] - m[h]) * inv[h];
    }
  }
}

// Short whole rows, GAT, 4 heads: a run of consecutive rows holding at most
// 32 edges in total (all inside the warp's chunk) is one warp step, one edge
// per lane.  Row boundaries become a bit mask of segment heads; the row max
// and the row sum of exponentials are segmented inclusive scans over the
// lanes (fixed order), read back from each segment's last lane.  A row of
// ~10 edges then costs a third of a warp step instead of a whole one.
// Returns the number of rows consumed (>= 1: row r itself is whole and
// at most 32 long).
#ifndef GNN_SOFTMAX_BATCH
#define GNN_SOFTMAX_BATCH 1
#endif
__device__ __forceinline__ unsigned lanes_le(int l) { return l >= 31 ? ~0u : (2u << l) - 1u; }

template <bool MAX>
__device__ __forceinline__ void seg_scan4(float (&x)[4], int lane, int ss) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float t = __shfl_up_sync(kFull, x[h], d);
      if (lane - d >= ss) x[h] = MAX ? fmaxf(x[h], t) : x[h] + t;
    }
  }
}

__device__ __forceinline__ int softmax_batch_gat4(const SoftmaxArgs &a, int64_t r, int64_t bs,
                                                  int64_t e1) {
  const int lane = (int)lane_id();
  const bool in = r + lane < a.R;
  const int64_t o = a.offsets[in ? r + 1 + lane : a.R];  // row ends
  const bool valid = in && o - bs <= 32 && o <= e1;        // a prefix of the lanes
  const int nb = __popc(__ballot_sync(kFull, valid));
  const int64_t be = RowWalk::shfl64(o, nb - 1);
  const int n = (int)(be - bs);
  int64_t os = RowWalk::shfl64(o, lane > 0 ? lane - 1 : 0);  // row starts
  if (lane == 0) os = bs;
  const bool ne = lane < nb && o > os;
  const unsigned nem = __ballot_sync(kFull, ne);
  const unsigned heads = __reduce_or_sync(kFull, ne ? 1u << (int)(os - bs) : 0u);
  const unsigned below = heads & lanes_le(lane);
  const int ss = below ? 31 - __clz(below) : 0;          // this edge's segment start
  const unsigned above = heads & ~lanes_le(lane);
  const int se = above ? __ffs(above) - 1 : n;           // its end (exclusive)
  const int k = __popc(below) - 1;                       // segment index
  const bool act = lane < n;
  const int64_t row = r + (act ? __fns(nem, 0, k + 1) : 0);
  float s[4] = {kNegInf, kNegInf, kNegInf, kNegInf};
  const int64_t e = bs + lane;
  if (act) {
    const float4 er4 = ldg_f4(a.er + row * 4);
    const float4 l4 = ldg_f4(a.el + (int64_t)a.cols[e] * 4);
    const float t[4] = {l4.x + er4.x, l4.y + er4.y, l4.z + er4.z, l4.w + er4.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) s[h] = t[h] > 0.f ? t[h] : a.slope * t[h];
  }
  float m[4] = {s[0], s[1], s[2], s[3]};
  seg_scan4<true>(m, lane, ss);
  const int last = se - 1 >= 0 ? se - 1 : 0;
#pragma unroll
  for (int h = 0; h < 4; ++h) m[h] = __shfl_sync(kFull, m[h], last);
  float ex[4], l[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    ex[h] = act ? __expf(s[h] - m[h]) : 0.f;
    l[h] = ex[h];
  }
  seg_scan4<false>(l, lane, ss);
  float inv[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) inv[h] = 1.f / __shfl_sync(kFull, l[h], last);
  if (act) {
    *reinterpret_cast<float4 *>(a.alpha + e * 4) =
        make_float4(ex[0] * inv[0], ex[1] * inv[1], ex[2] * inv[2], ex[3] * inv[3]);
    if (a.mstat && lane == ss) {
      reinterpret_cast<float4 *>(a.mstat + row * 8)[0] = make_float4(m[0], m[1], m[2], m[3]);
      reinterpret_cast<float4 *>(a.mstat + row * 8)[1] = make_float4(inv[0], inv[1], inv[2], inv[3]);
    }
  }
  return nb;
}

// Backward of one row piece: S = sum alpha*dalpha; whole rows write
// ds = alpha (dalpha - S) (* LeakyReLU'(pre) in GAT mode).
template <int HM, bool GAT>
__device__ __forceinline__ void softmax_bwd_apply(const SoftmaxArgs &a, int64_t r, int64_t lo,
                                                  int64_t hi, const float (&S)[HM]) {
  const int lane = (int)lane_id();
  float erow[HM];
  load_erow<HM, GAT>(a, r, erow);
  for (int64_t e = lo + lane; e < hi; e += 32) {
    float pre[HM];
    if constexpr (GAT) {
      const int64_t c = a.cols[e];
#pragma unroll
      for (int h = 0; h < HM; ++h) pre[h] = h < a.H ? __ldg(a.el + c * a.H + h) + erow[h] : 0.f;
    }
#pragma unroll
    for (int h = 0; h < HM; ++h)
      if (h < a.H) {
        const float al = a.alpha_in[e * a.H + h];
        const float da = a.dalpha[e * a.H + h];
        float d = al * (da - S[h]);
        if constexpr (GAT) d = pre[h] > 0.f ? d : a.slope * d;
        a.ds[e * a.H + h] = d;
      }
  }
}

template <int HM, bool GAT>
__device__ __forceinline__ void softmax_bwd_piece(const SoftmaxArgs &a, int64_t r, int64_t lo,
                                                  int64_t hi, bool whole, float *slot) {
  const int lane = (int)lane_id();
  float S[HM];
#pragma unroll
  for (int h = 0; h < HM; ++h) S[h] = 0.f;
  if (whole && hi - lo <= 32 && HM == 4 && a.H == 4) {
    // one edge per lane: alpha / dalpha stay in registers for the apply
    const int64_t e = lo + lane;
    const bool ok = e < hi;
    const float4 al = ok ? *reinterpret_cast<const float4 *>(a.alpha_in + e * 4)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 da = ok ? *reinterpret_cast<const float4 *>(a.dalpha + e * 4)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    const float alv[4] = {al.x, al.y, al.z, al.w}, dav[4] = {da.x, da.y, da.z, da.w};
#pragma unroll
    for (int h = 0; h < HM; ++h) S[h] = fmaf(alv[h < 4 ? h : 0], dav[h < 4 ? h : 0], 0.f);
    warp_sum_reduce<HM>(S);
    if (ok) {
      float pre[4] = {1.f, 1.f, 1.f, 1.f};
      if constexpr (GAT) {
        const float4 l4 = ldg_f4(a.el + (int64_t)a.cols[e] * 4);
        const float er0 = __ldg(a.er + r * 4), er1 = __ldg(a.er + r * 4 + 1),
                    er2 = __ldg(a.er + r * 4 + 2), er3 = __ldg(a.er + r * 4 + 3);
        pre[0] = l4.x + er0;
        pre[1] = l4.y + er1;
        pre[2] = l4.z + er2;
        pre[3] = l4.w + er3;
      }
      float d[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        d[h] = alv[h] * (dav[h] - S[h < HM ? h : 0]);
        if constexpr (GAT) d[h] = pre[h] > 0.f ? d[h] : a.slope * d[h];
      }
      *reinterpret_cast<float4 *>(a.ds + e * 4) = make_float4(d[0], d[1], d[2], d[3]);
    }
    return;
  }
  for (int64_t e = lo + lane; e < hi; e += 32) {
#pragma unroll
    for (int h = 0; h < HM; ++h)
      if (h < a.H) S[h] = fmaf(a.alpha_in[e * a.H + h], a.dalpha[e * a.H + h], S[h]);
  }
  warp_sum_reduce<HM>(S);
  if (!whole) {
    if (lane == 0)
#pragma unroll
      for (int h = 0; h < HM; ++h)
        if (h < a.H) slot[h] = S[h];
    return;
  }
  softmax_bwd_apply<HM, GAT>(a, r, lo, hi, S);
}

// Kernel 1: one warp per chunk; whole rows finished, split-row pieces leave
// partials in slot[w][0] (carry-in piece) / slot[w][1] (trailing piece).
template <int HM, bool GAT, bool BWD>
__global__ void __launch_bounds__(256) softmax_rows_kernel(SoftmaxArgs a) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= a.nwarps) return;
  const int64_t e0 = w * a.P, e1 = min(e0 + a.P, a.nnz);
  RowWalk rw(a.offsets, a.R, a.chunk_row[w]);
  while (true) {
    const int64_t lo = max(rw.rs, e0), hi = min(rw.re, e1);
    if constexpr (GAT && !BWD && HM == 4 && GNN_SOFTMAX_BATCH) {
      if (a.H == 4 && rw.rs >= e0 && rw.re <= e1 && rw.re - rw.rs <= 32) {
        const int nb = softmax_batch_gat4(a, rw.r, rw.rs, e1);
        const int64_t r1 = rw.r + nb;
        const int64_t end = RowWalk::shfl64(a.offsets[min(r1, a.R)], 0);
        if (end >= e1 || r1 >= a.R) break;
        rw = RowWalk(a.offsets, a.R, r1);
        continue;
      }
    }
    if (hi > lo) {
      const bool carry = rw.rs < e0, trail = !carry && rw.re > e1;
      float *slot = a.slots + (w * 2 + (carry ? 0 : 1)) * 2 * a.H;
      if (BWD)
        softmax_bwd_piece<HM, GAT>(a, rw.r, lo, hi, !(carry || trail), slot);
      else
        softmax_piece<HM, GAT>(a, rw.r, lo, hi, !(carry || trail), slot);
    }
    if (rw.re >= e1 || rw.r + 1 >= a.R) break;
    rw.next();
  }
}

// Kernel 2: one warp per split row; partial j of row (chunks wa..wb) is
// slot[wa][1] for j = 0 and slot[wa+j][0] for j >= 1 (same convention as the
// SpMM).  Lane-strided merge in j order, then a fixed xor tree.
template <int HM, bool BWD>
__global__ void __launch_bounds__(256) softmax_split_finalize_kernel(SoftmaxArgs a) {
  const int64_t si = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (si >= a.num_split) return;
  const int lane = (int)lane_id();
  const int64_t r = a.split_rows[si];
  const int64_t rs = a.offsets[r], re = a.offsets[r + 1];
  const int64_t wa = rs / a.P, wb = (re - 1) / a.P;
  const int64_t np = wb - wa + 1;
  float m[HM], l[HM];
#pragma unroll
  for (int h = 0; h < HM; ++h) {
    m[h] = BWD ? 0.f : kNegInf;
    l[h] = 0.f;
  }
  for (int64_t j = lane; j < np; j += 32) {
    const float *slot = a.slots + ((wa + j) * 2 + (j == 0 ? 1 : 0)) * 2 * a.H;
#pragma unroll
    for (int h = 0; h < HM; ++h)
      if (h < a.H) {
        if (BWD)
          m[h] += slot[h];
        else
          ml_merge(m[h], l[h], slot[h], slot[a.H + h]);
      }
  }
  if (BWD)
    warp_sum_reduce<HM>(m);
  else
    warp_ml_reduce<HM>(m, l);
  if (lane == 0)
#pragma unroll
    for (int h = 0; h < HM; ++h)
      if (h < a.H) {
        a.stat[si * 2 * a.H + h] = m[h];
        a.stat[si * 2 * a.H + a.H + h] = l[h];
        if (!BWD && a.mstat) {
          a.mstat[r * 2 * a.H + h] = m[h];
          a.mstat[r * 2 * a.H + a.H + h] = 1.f / l[h];
        }
      }
}

// Kernel 3: one warp per chunk; normalises the chunk's split-row pieces.
template <int HM, bool GAT, bool BWD>
__global__ void __launch_bounds__(256) softmax_split_apply_kernel(SoftmaxArgs a) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= a.nwarps) return;
  const int64_t e0 = w * a.P, e1 = min(e0 + a.P, a.nnz);
  const int lane = (int)lane_id();
#pragma unroll 1
  for (int which = 0; which < 2; ++which) {
    const int32_t si = a.chunk_split[2 * w + which];
    if (si < 0) continue;
    const int64_t r = a.split_rows[si];
    const int64_t lo = max(a.offsets[r], e0), hi = min(a.offsets[r + 1], e1);
    float m[HM], l[HM];
#pragma unroll
    for (int h = 0; h < HM; ++h) {
      m[h] = h < a.H ? a.stat[si * 2 * a.H + h] : 0.f;
      l[h] = h < a.H ? a.stat[si * 2 * a.H + a.H + h] : 1.f;
    }
    if (BWD) {
      softmax_bwd_apply<HM, GAT>(a, r, lo, hi, m);
      continue;
    }
    float erow[HM];
    load_erow<HM, GAT>(a, r, erow);
    float inv[HM];
#pragma unroll
    for (int h = 0; h < HM; ++h) inv[h] = 1.f / l[h];
    if constexpr (GAT && HM == 4 && GNN_SOFTMAX_ONLINE) {
      if (a.H == 4) {
        gat4_write_alpha(a, lo, hi, erow, m, inv);
        continue;
      }
    }
    for (int64_t e = lo + lane; e < hi; e += 32) {
      float s[HM];
      load_scores<HM, GAT>(a, e, erow, s);
#pragma unroll
      for (int h = 0; h < HM; ++h)
        if (h < a.H) a.alpha[e * a.H + h] = __expf(s[h] - m[h]) * inv[h];
    }
  }
}

// ------------------------------------------------------------ segment sum
// Row sums of an edge tensor (GAT's der = rowsum(ds), del = colsum(ds) via
// the CSC + edge-ID).  Same chunk walk; whole rows write out[r], split-row
// pieces leave partials that the finalize kernel sums in fixed order.
template <int HM, bool EID>
__device__ __forceinline__ void segsum_piece(const SoftmaxArgs &a, int64_t r, int64_t lo, int64_t hi,
                                             bool whole, float *slot) {
  const int lane = (int)lane_id();
  float S[HM];
#pragma unroll
  for (int h = 0; h < HM; ++h) S[h] = 0.f;
  for (int64_t e = lo + lane; e < hi; e += 32) {
    const int64_t src = EID ? (int64_t)a.eid[e] : e;
    if (HM == 4 && a.H == 4) {
      const float4 v = *reinterpret_cast<const float4 *>(a.alpha_in + src * 4);
      S[0] += v.x;
      S[1] += v.y;
      S[2] += v.z;
      S[3] += v.w;
    } else {
#pragma unroll
      for (int h = 0; h < HM; ++h)
        if (h < a.H) S[h] += a.alpha_in[src * a.H + h];
    }
  }
  warp_sum_reduce<HM>(S);
  if (lane == 0)
#pragma unroll
    for (int h = 0; h < HM; ++h)
      if (h < a.H) (whole ? a.ds + r * a.H : slot)[h] = S[h];
}

// Runs of short whole rows (<= 32 edges together), 4 heads: one edge per
// lane, a segmented sum scan, the segment's last lane writes the row (rows
// without edges write 0).  Returns the rows consumed.
template <bool EID>
__device__ __forceinline__ int segsum_batch4(const SoftmaxArgs &a, int64_t r, int64_t bs, int64_t e1) {
  const int lane = (int)lane_id();
  const bool in = r + lane < a.R;
  const int64_t o = a.offsets[in ? r + 1 + lane : a.R];
  const bool valid = in && o - bs <= 32 && o <= e1;
  const int nb = __popc(__ballot_sync(kFull, valid));
  const int n = (int)(RowWalk::shfl64(o, nb - 1) - bs);
  int64_t os = RowWalk::shfl64(o, lane > 0 ? lane - 1 : 0);
  if (lane == 0) os = bs;
  const bool ne = lane < nb && o > os;
  const unsigned heads = __reduce_or_sync(kFull, ne ? 1u << (int)(os - bs) : 0u);
  const unsigned below = heads & lanes_le(lane);
  const int ss = below ? 31 - __clz(below) : 0;
  float x[4] = {0.f, 0.f, 0.f, 0.f};
  if (lane < n) {
    const int64_t e = bs + lane;
    const int64_t src = EID ? (int64_t)a.eid[e] : e;
    const float4 v = *reinterpret_cast<const float4 *>(a.alpha_in + src * 4);
    x[0] = v.x;
    x[1] = v.y;
    x[2] = v.z;
    x[3] = v.w;
  }
  seg_scan4<false>(x, lane, ss);
  // row j (< nb): its sum sits at the lane of its last edge, o_j - bs - 1
  float t[4];
  const int src_lane = ne ? (int)(o - bs) - 1 : 0;
#pragma unroll
  for (int h = 0; h < 4; ++h) t[h] = __shfl_sync(kFull, x[h], src_lane);
  if (lane < nb)
    *reinterpret_cast<float4 *>(a.ds + (r + lane) * 4) =
        ne ? make_float4(t[0], t[1], t[2], t[3]) : make_float4(0.f, 0.f, 0.f, 0.f);
  return nb;
}

template <int HM, bool EID>
__global__ void __launch_bounds__(256) segsum_rows_kernel(SoftmaxArgs a) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= a.nwarps) return;
  const int64_t e0 = w * a.P, e1 = min(e0 + a.P, a.nnz);
  RowWalk rw(a.offsets, a.R, a.chunk_row[w]);
  while (true) {
    const int64_t lo = max(rw.rs, e0), hi = min(rw.re, e1);
    if constexpr (HM == 4 && GNN_SOFTMAX_BATCH) {
      if (a.H == 4 && rw.rs >= e0 && rw.re <= e1 && rw.re - rw.rs <= 32) {
        const int64_t r1 = rw.r + segsum_batch4<EID>(a, rw.r, rw.rs, e1);
        const int64_t end = RowWalk::shfl64(a.offsets[min(r1, a.R)], 0);
        if (end >= e1 || r1 >= a.R) break;
        rw = RowWalk(a.offsets, a.R, r1);
        continue;
      }
    }
    if (hi > lo) {
      const bool carry = rw.rs < e0, trail = !carry && rw.re > e1;
      float *slot = a.slots + (w * 2 + (carry ? 0 : 1)) * 2 * a.H;
      segsum_piece<HM, EID>(a, rw.r, lo, hi, !(carry || trail), slot);
    }
    if (rw.re >= e1 || rw.r + 1 >= a.R) break;
    rw.next();
  }
}

template <int HM>
__global__ void __launch_bounds__(256) segsum_split_finalize_kernel(SoftmaxArgs a) {
  const int64_t si = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (si >= a.num_split) return;
  const int lane = (int)lane_id();
  const int64_t r = a.split_rows[si];
  const int64_t rs = a.offsets[r], re = a.offsets[r + 1];
  const int64_t wa = rs / a.P, wb = (re - 1) / a.P;
  const int64_t np = wb - wa + 1;
  float S[HM];
#pragma unroll
  for (int h = 0; h < HM; ++h) S[h] = 0.f;
  for (int64_t j = lane; j < np; j += 32) {
    const float *slot = a.slots + ((wa + j) * 2 + (j == 0 ? 1 : 0)) * 2 * a.H;
#pragma unroll
    for (int h = 0; h < HM; ++h)
      if (h < a.H) S[h] += slot[h];
  }
  warp_sum_reduce<HM>(S);
  if (lane == 0)
#pragma unroll
    for (int h = 0; h < HM; ++h)
      if (h < a.H) a.ds[r * a.H + h] = S[h];
}

template <int HM>
int launch_segsum(const SoftmaxArgs &a, bool eid, cudaStream_t st) {
  GNN_CUDA_TRY(cudaMemsetAsync(a.ds, 0, sizeof(float) * a.R * a.H, st));  // empty rows
  if (a.nwarps > 0) {
    if (eid)
      segsum_rows_kernel<HM, true><<<grid_warps(a.nwarps, 256), 256, 0, st>>>(a);
    else
      segsum_rows_kernel<HM, false><<<grid_warps(a.nwarps, 256), 256, 0, st>>>(a);
    GNN_LAUNCH_CHECK();
  }
  if (a.num_split > 0) {
    segsum_split_finalize_kernel<HM><<<grid_warps(a.num_split, 256), 256, 0, st>>>(a);
    GNN_LAUNCH_CHECK();
  }
  return GNN_OK;
}

template <int HM, bool GAT, bool BWD>
int launch_softmax(const SoftmaxArgs &a, cudaStream_t st) {
  if (a.nwarps > 0) {
    softmax_rows_kernel<HM, GAT, BWD><<<grid_warps(a.nwarps, 256), 256, 0, st>>>(a);
    GNN_LAUNCH_CHECK();
  }
  if (a.num_split > 0) {
    softmax_split_finalize_kernel<HM, BWD><<<grid_warps(a.num_split, 256), 256, 0, st>>>(a);
    GNN_LAUNCH_CHECK();
    softmax_split_apply_kernel<HM, GAT, BWD><<<grid_warps(a.nwarps, 256), 256, 0, st>>>(a);
    GNN_LAUNCH_CHECK();
  }
  return GNN_OK;
}

template <bool GAT, bool BWD>
int dispatch_softmax(const SoftmaxArgs &a, cudaStream_t st) {
  if (a.H == 1) return launch_softmax<1, GAT, BWD>(a, st);
  if (a.H <= 4) return launch_softmax<4, GAT, BWD>(a, st);
  if (a.H <= 8) return launch_softmax<8, GAT, BWD>(a, st);
  return launch_softmax<16, GAT, BWD>(a, st);
}

size_t softmax_ws_layout(const gnn_spmm_plan_t *plan, int64_t H, size_t *o_stat) {
  WsCounter c;
  c.take<float>(plan->num_warps * 2 * 2 * H);
  *o_stat = align_up(c.used, 256);
  c.take<float>(plan->num_split * 2 * H);
  return c.used + 256;
}

int softmax_common(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
                   const gnn_edge_scores_t *sc, void *ws, size_t ws_bytes, SoftmaxArgs &a) {
  if ((A && (A->col_bits || A->row_ids)) || !A || !plan || heads <= 0 || heads > 16 || !A->offsets || (A->nnz > 0 && !A->cols))
    return GNN_ERR_INVALID_ARGUMENT;
  if (plan->dev_counts || plan->edges_per_warp <= 0 || plan->num_warps != ceil_div(A->nnz, plan->edges_per_warp))
    return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_edge_softmax_workspace(plan, heads)) return GNN_ERR_WORKSPACE;
  a = SoftmaxArgs{};
  a.R = A->num_rows;
  a.nnz = A->nnz;
  a.P = plan->edges_per_warp;
  a.nwarps = plan->num_warps;
  a.offsets = A->offsets;
  a.cols = A->cols;
  a.chunk_row = plan->chunk_row;
  a.chunk_split = plan->chunk_split;
  a.split_rows = plan->split_rows;
  a.num_split = plan->num_split;
  a.H = (int)heads;
  if (sc) {
    a.s = sc->s;
    a.el = sc->el;
    a.er = sc->er;
    a.slope = sc->slope;
  }
  size_t o_stat;
  softmax_ws_layout(plan, heads, &o_stat);
  a.slots = static_cast<float *>(ws);
  a.stat = reinterpret_cast<float *>(static_cast<char *>(ws) + o_stat);
  return GNN_OK;
}

// -------------------------------------------------- GAT per-vertex helpers
// el[v,h] = <Wh[v,h,:], a_l[h,:]>, er likewise: one thread per (v,h).
__global__ void attn_proj_kernel(int64_t V, int H, int64_t F, const float *__restrict__ Wh,
                                 int64_t ldw, const float *__restrict__ al,
                                 const float *__restrict__ ar, float *el, float *er) {
  const int64_t total = V * H;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / H;
    const int h = (int)(t % H);
    const float *x = Wh + v * ldw + h * F;
    float sl = 0.f, sr = 0.f;
    for (int64_t f = 0; f < F; ++f) {
      const float xv = __ldg(x + f);
      sl = fmaf(xv, __ldg(al + h * F + f), sl);
      sr = fmaf(xv, __ldg(ar + h * F + f), sr);
    }
    el[t] = sl;
    er[t] = sr;
  }
}

// float4 form (F % 4 == 0, 16-byte rows): 4 lanes per (vertex, head), each
// summing every 4th float4 of the head's F features, then a 4-lane butterfly;
// a warp's loads cover 8 head rows contiguously (the thread-per-(v, h) form
// above issues one scattered 4-byte load per feature).
__global__ void attn_proj_vec_kernel(int64_t V, int H, int64_t F, const float *__restrict__ Wh,
                                     int64_t ldw, const float *__restrict__ al,
                                     const float *__restrict__ ar, float *el, float *er) {
  const int64_t total = V * H;
  const int gl = (int)(threadIdx.x & 3);
  const unsigned gmask = 0xfu << (threadIdx.x & 28);
  const int64_t F4 = F / 4;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2; t < total;
       t += ((int64_t)gridDim.x * blockDim.x) >> 2) {
    const int64_t v = t / H;
    const int h = (int)(t % H);
    const float4 *x = reinterpret_cast<const float4 *>(Wh + v * ldw + h * F);
    const float4 *a4 = reinterpret_cast<const float4 *>(al + h * F);
    const float4 *r4 = reinterpret_cast<const float4 *>(ar + h * F);
    float sl = 0.f, sr = 0.f;
    for (int64_t j = gl; j < F4; j += 4) {
      const float4 xv = ldg_f4(reinterpret_cast<const float *>(x + j));
      const float4 a = __ldg(a4 + j), b = __ldg(r4 + j);
      sl = fmaf(xv.x, a.x, fmaf(xv.y, a.y, fmaf(xv.z, a.z, fmaf(xv.w, a.w, sl))));
      sr = fmaf(xv.x, b.x, fmaf(xv.y, b.y, fmaf(xv.z, b.z, fmaf(xv.w, b.w, sr))));
    }
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) {
      sl += __shfl_xor_sync(gmask, sl, o, 4);
      sr += __shfl_xor_sync(gmask, sr, o, 4);
    }
    if (gl == 0) {
      el[t] = sl;
      er[t] = sr;
    }
  }
}

// One streaming pass over the vertices: thread = column k (< K <= 512, two
// passes of 256 for wider K), each CTA a contiguous vertex range, 4 rows in
// flight.  dWh[v,k] += del[v,h(k)] a_l[k] + der[v,h(k)] a_r[k] (in place) and
// the CTA's partial of da_l[k] = sum_v Wh[v,k] del[v,h(k)] (and da_r), summed
// over CTAs in fixed order by attn_proj_bwd_da_final_kernel.
constexpr int kProjBlocks = 1024;
__global__ void __launch_bounds__(256) attn_proj_bwd_kernel(
    int64_t V, int H, int64_t F, const float *__restrict__ Wh, int64_t ldw,
    const float *__restrict__ del, const float *__restrict__ der, const float *__restrict__ al,
    const float *__restrict__ ar, float *dWh, int64_t ldd, float *part) {
  const int64_t K = (int64_t)H * F;
  const int64_t per = ceil_div(V, gridDim.x);
  const int64_t v0 = blockIdx.x * per, v1 = min(v0 + per, V);
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const int64_t h = k / F;
    const float alk = __ldg(al + k), ark = __ldg(ar + k);
    float sl = 0.f, sr = 0.f;
    int64_t v = v0;
    for (; v + 3 < v1; v += 4) {
      float x[4], d[4], dl[4], dr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u] = __ldg(Wh + (v + u) * ldw + k);
        d[u] = dWh[(v + u) * ldd + k];
        dl[u] = __ldg(del + (v + u) * H + h);
        dr[u] = __ldg(der + (v + u) * H + h);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        sl = fmaf(x[u], dl[u], sl);
        sr = fmaf(x[u], dr[u], sr);
        dWh[(v + u) * ldd + k] = fmaf(dr[u], ark, fmaf(dl[u], alk, d[u]));
      }
    }
    for (; v < v1; ++v) {
      const float x = __ldg(Wh + v * ldw + k), dl = __ldg(del + v * H + h), dr = __ldg(der + v * H + h);
      sl = fmaf(x, dl, sl);
      sr = fmaf(x, dr, sr);
      dWh[v * ldd + k] = fmaf(dr, ark, fmaf(dl, alk, dWh[v * ldd + k]));
    }
    part[(int64_t)blockIdx.x * 2 * K + k] = sl;
    part[(int64_t)blockIdx.x * 2 * K + K + k] = sr;
  }
}
// float4 form (F % 4 == 0, 16-byte rows): row groups of K/4 lanes, each lane
// 4 consecutive columns of one head; 16-byte loads / stores of Wh and dWh keep
// more bytes in flight than the column-per-thread form above (which ran the
// products-shape layer-2 pass at ~2.5 TB/s).  Per-block partials of
// da = sum_v d{l,r}[v,h] * Wh[v,:] are reduced over the row groups in fixed
// order.
__global__ void __launch_bounds__(256) attn_proj_bwd_vec_kernel(
    int64_t V, int H, int64_t F, const float *__restrict__ Wh, int64_t ldw,
    const float *__restrict__ del, const float *__restrict__ der, const float *__restrict__ al,
    const float *__restrict__ ar, float *dWh, int64_t ldd, float *part) {
  __shared__ float4 red[2][256];
  const int64_t K = (int64_t)H * F;
  const int K4 = (int)(K / 4);
  const int groups = (int)blockDim.x / K4;  // row groups per block
  const int q = (int)threadIdx.x % K4, rg = (int)threadIdx.x / K4;
  const int64_t per = ceil_div(V, gridDim.x);
  const int64_t v0 = blockIdx.x * per, v1 = min(v0 + per, V);
  float4 sl = make_float4(0.f, 0.f, 0.f, 0.f), sr = sl;
  if (rg < groups) {
    const int64_t k = 4 * (int64_t)q;
    const int64_t h = k / F;
    const float4 alk = *reinterpret_cast<const float4 *>(al + k);
    const float4 ark = *reinterpret_cast<const float4 *>(ar + k);
#pragma unroll 2
    for (int64_t v = v0 + rg; v < v1; v += groups) {
      const float4 x = ldg_f4(Wh + v * ldw + k);
      float4 *dp = reinterpret_cast<float4 *>(dWh + v * ldd + k);
      const float4 d = *dp;
      const float dl = __ldg(del + v * H + h), dr = __ldg(der + v * H + h);
      sl = make_float4(fmaf(x.x, dl, sl.x), fmaf(x.y, dl, sl.y), fmaf(x.z, dl, sl.z), fmaf(x.w, dl, sl.w));
      sr = make_float4(fmaf(x.x, dr, sr.x), fmaf(x.y, dr, sr.y), fmaf(x.z, dr, sr.z), fmaf(x.w, dr, sr.w));
      *dp = make_float4(fmaf(dr, ark.x, fmaf(dl, alk.x, d.x)), fmaf(dr, ark.y, fmaf(dl, alk.y, d.y)),
                        fmaf(dr, ark.z, fmaf(dl, alk.z, d.z)), fmaf(dr, ark.w, fmaf(dl, alk.w, d.w)));
    }
  }
  red[0][threadIdx.x] = sl;
  red[1][threadIdx.x] = sr;
  __syncthreads();
  if (rg == 0) {
    float4 tl = make_float4(0.f, 0.f, 0.f, 0.f), tr = tl;
    for (int g = 0; g < groups; ++g) {
      const float4 a = red[0][g * K4 + q], b = red[1][g * K4 + q];
      tl = make_float4(tl.x + a.x, tl.y + a.y, tl.z + a.z, tl.w + a.w);
      tr = make_float4(tr.x + b.x, tr.y + b.y, tr.z + b.z, tr.w + b.w);
    }
    *reinterpret_cast<float4 *>(part + (int64_t)blockIdx.x * 2 * K + 4 * q) = tl;
    *reinterpret_cast<float4 *>(part + (int64_t)blockIdx.x * 2 * K + K + 4 * q) = tr;
  }
}
__global__ void attn_proj_bwd_da_final_kernel(int64_t K, int nb, const float *__restrict__ part,
                                              float *dal, float *dar) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 2 * K;
       k += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < nb; ++b) s += part[(int64_t)b * 2 * K + k];
    if (k < K)
      dal[k] = s;
    else
      dar[k - K] = s;
  }
}

// out[v,f] = (1/H) sum_h Y[v,h*F+f] (+ bias[f]);  backward: dY[v,h*F+f] = dout[v,f]/H
__global__ void head_mean_kernel(int64_t V, int H, int64_t F, const float *__restrict__ Y,
                                 int64_t ldy, const float *__restrict__ bias, float *out,
                                 int64_t ldo) {
  const int64_t total = V * F;
  const float inv = 1.f / (float)H;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / F, f = t % F;
    float s = 0.f;
    for (int h = 0; h < H; ++h) s += Y[v * ldy + h * F + f];
    s *= inv;
    if (bias) s += bias[f];
    out[v * ldo + f] = s;
  }
}
__global__ void head_mean_bwd_kernel(int64_t V, int H, int64_t F, const float *__restrict__ dout,
                                     int64_t ldo, float *dY, int64_t ldy) {
  const int64_t K = (int64_t)H * F;
  const int64_t total = V * K;
  const float inv = 1.f / (float)H;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / K, k = t % K;
    dY[v * ldy + k] = dout[v * ldo + k % F] * inv;
  }
}

// Reduce 4 per-lane head partials over a G-lane group (G >= 4) with a
// reduce-scatter butterfly: 2 + 1 shuffles leave each lane one head's
// partial, then log2(G) - 2 more finish it.  Returns the head sum; *head is
// the head this lane holds (complete on lanes with (gl & (G/4 - 1)) == 0).
template <int G>
__device__ __forceinline__ float reduce4_scatter(const float (&ph)[4], unsigned gmask, int gl,
                                                 int *head) {
  const bool b1 = (gl & (G / 2)) != 0, b2 = (gl & (G / 4)) != 0;
  const float sa = b1 ? ph[0] : ph[2], sb = b1 ? ph[1] : ph[3];
  const float k0 = (b1 ? ph[2] : ph[0]) + __shfl_xor_sync(gmask, sa, G / 2);
  const float k1 = (b1 ? ph[3] : ph[1]) + __shfl_xor_sync(gmask, sb, G / 2);
  float k = (b2 ? k1 : k0) + __shfl_xor_sync(gmask, b2 ? k0 : k1, G / 4);
#pragma unroll
  for (int o = G / 8; o > 0; o >>= 1) k += __shfl_xor_sync(gmask, k, o);
  *head = (b1 ? 2 : 0) + (b2 ? 1 : 0);
  return k;
}

// ----------------------------------------- fused GAT backward over the CSC
// One pass over the CSC (in-edges of every vertex u, with the edge-ID array)
// computes both products that need dY[v] of every edge (v -> u):
//   dWh[u,:]          = sum_j alpha[eid_j, head(:)] * dY[v_j, :]      (SpMMve^T)
//   dalpha[eid_j, h]  = < dY[v_j, head h], Wh[u, head h] >           (SDDMM)
// so dY is gathered once instead of twice.  Warp per plan chunk of the CSC,
// one row piece at a time; G lanes per edge x VPL float4 columns; NG = 32/G
// edges per step, U steps in flight.  Edge indices are loaded 32 at a time by
// the warp and broadcast by shuffle.  Split rows leave partials that
// gat_bwd_finalize sums in fixed order.
struct GatBwdArgs {
  int64_t R, nnz, P, nwarps;
  const int64_t *offsets;
  const int32_t *rows;  // CSC "cols": source vertices v
  const int32_t *eid;
  const int32_t *chunk_row;
  const int32_t *chunk_split;
  const int32_t *split_rows;
  int64_t num_split;
  const int32_t *empty_rows;
  int64_t num_empty;
  int H;
  int64_t F, K;
  const float *alpha;  // [E, H] CSR order
  const float *dY;
  int64_t ldy;
  const float *Wh;
  int64_t ldw;
  float *dWh;
  int64_t ldd;
  float *dalpha;       // [E, H] CSR order
  float *slots;        // [nwarps][2][K]
};

template <int G, int VPL, int HM, bool POW2>
__global__ void __launch_bounds__(256, (VPL == 1) ? 3 : 1) gat_bwd_csc_kernel(GatBwdArgs a, int LPH) {
  constexpr int NG = 32 / G;
  constexpr int U = VPL >= 3 ? 3 : 4;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= a.nwarps) return;
  const int lane = (int)lane_id();
  const int g = lane / G, gl = lane % G;
  const unsigned gmask = G == 32 ? kFull : (((1u << G) - 1u) << (g * G));
  const int64_t e0 = w * a.P, e1 = min(e0 + a.P, a.nnz);
  const bool h4 = HM == 4 && a.H == 4;
  int64_t col[VPL];
  int hd[VPL];
  bool cv[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    col[v] = (int64_t)(v * G + gl) * 4;
    cv[v] = col[v] < a.K;
    if (!cv[v]) col[v] = 0;
    hd[v] = (int)(col[v] / a.F);
  }
  RowWalk rw(a.offsets, a.R, a.chunk_row[w]);
  while (true) {
    const int64_t lo = max(rw.rs, e0), hi = min(rw.re, e1);
    if (hi > lo) {
      const int64_t u = rw.r;
      float4 self[VPL], acc[VPL];
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        self[v] = ldg_f4(a.Wh + u * a.ldw + col[v]);
        acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (int64_t b0 = lo; b0 < hi; b0 += 32) {
        const int nb = (int)min((int64_t)32, hi - b0);
        int32_t myc = 0, mye = 0;
        if (lane < nb) {
          myc = a.rows[b0 + lane];
          mye = a.eid[b0 + lane];
        }
        for (int k0 = 0; k0 < nb; k0 += NG * U) {
          int32_t c[U], ee[U];
          bool ok[U];
#pragma unroll
          for (int t = 0; t < U; ++t) {
            const int k = k0 + t * NG + g;
            ok[t] = k < nb;
            c[t] = __shfl_sync(kFull, myc, k & 31);
            ee[t] = __shfl_sync(kFull, mye, k & 31);
          }
          float4 x[U][VPL];
          float wg[U][VPL];
#pragma unroll
          for (int t = 0; t < U; ++t) {
#pragma unroll
            for (int v = 0; v < VPL; ++v)
              x[t][v] = ok[t] ? ldg_f4(a.dY + (int64_t)c[t] * a.ldy + col[v])
                              : make_float4(0.f, 0.f, 0.f, 0.f);
            // edge weights issued with the gathers (no second dependent latency)
            if (h4) {
              const float4 al = ok[t] ? ldg_f4(a.alpha + (int64_t)ee[t] * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int v = 0; v < VPL; ++v)
                wg[t][v] = hd[v] == 0 ? al.x : hd[v] == 1 ? al.y : hd[v] == 2 ? al.z : al.w;
            } else {
#pragma unroll
              for (int v = 0; v < VPL; ++v)
                wg[t][v] = ok[t] ? __ldg(a.alpha + (int64_t)ee[t] * a.H + hd[v]) : 0.f;
            }
          }
#pragma unroll
          for (int t = 0; t < U; ++t) {
            // SpMMve^T accumulation
#pragma unroll
            for (int v = 0; v < VPL; ++v) acc[v] = f4_fma(wg[t][v], x[t][v], acc[v]);
            // SDDMM: per-head dots with the row's own Wh
            if constexpr (POW2) {
#pragma unroll
              for (int v = 0; v < VPL; ++v) {
                float p = x[t][v].x * self[v].x;
                p = fmaf(x[t][v].y, self[v].y, p);
                p = fmaf(x[t][v].z, self[v].z, p);
                p = fmaf(x[t][v].w, self[v].w, p);
                for (int o = 1; o < LPH; o <<= 1) p += __shfl_xor_sync(gmask, p, o);
                if (ok[t] && cv[v] && (gl & (LPH - 1)) == 0)
                  a.dalpha[(int64_t)ee[t] * a.H + hd[v]] = p;
              }
            } else {
              float ph[HM];
#pragma unroll
              for (int h = 0; h < HM; ++h) ph[h] = 0.f;
#pragma unroll
              for (int v = 0; v < VPL; ++v) {
                float p = x[t][v].x * self[v].x;
                p = fmaf(x[t][v].y, self[v].y, p);
                p = fmaf(x[t][v].z, self[v].z, p);
                p = fmaf(x[t][v].w, self[v].w, p);
                if (cv[v])
#pragma unroll
                  for (int h = 0; h < HM; ++h) ph[h] += h == hd[v] ? p : 0.f;
              }
              bool done = false;
              if constexpr (HM == 4 && G >= 4) {
                if (a.H == 4) {
                  int hh;
                  const float sum = reduce4_scatter<G>(ph, gmask, gl, &hh);
                  if (ok[t] && (gl & (G / 4 - 1)) == 0) a.dalpha[(int64_t)ee[t] * 4 + hh] = sum;
                  done = true;
                }
              }
              if (!done) {
#pragma unroll
                for (int o = 1; o < G; o <<= 1)
#pragma unroll
                  for (int h = 0; h < HM; ++h) ph[h] += __shfl_xor_sync(gmask, ph[h], o);
                if (ok[t] && gl == 0)
#pragma unroll
                  for (int h = 0; h < HM; ++h)
                    if (h < a.H) a.dalpha[(int64_t)ee[t] * a.H + h] = ph[h];
              }
            }
          }
        }
      }
      // combine the NG groups (fixed xor tree), then store row / partial
#pragma unroll
      for (int o = G; o < 32; o <<= 1)
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          acc[v] = f4_add(acc[v], make_float4(__shfl_xor_sync(kFull, acc[v].x, o),
                                              __shfl_xor_sync(kFull, acc[v].y, o),
                                              __shfl_xor_sync(kFull, acc[v].z, o),
                                              __shfl_xor_sync(kFull, acc[v].w, o)));
      const bool carry = rw.rs < e0, trail = !carry && rw.re > e1;
      float *dst = (carry || trail) ? a.slots + (w * 2 + (carry ? 0 : 1)) * a.K : a.dWh + u * a.ldd;
      if (g == 0)
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          if (cv[v]) *reinterpret_cast<float4 *>(dst + col[v]) = acc[v];
    }
    if (rw.re >= e1 || rw.r + 1 >= a.R) break;
    rw.next();
  }
}

// Head-mean output layer: dY of the concatenated heads is dZ / H broadcast
// to every head, so the kernel gathers only dZ[v] (F floats, not H*F) and
// produces all heads from it:
//   dWh[u, h*F + f]  = scale * sum_j alpha[eid_j, h] * dZ[v_j, f]
//   dalpha[eid_j, h] = scale * < dZ[v_j, :], Wh[u, h*F : (h+1)*F] >
#ifndef GNN_GATM_MINB
#define GNN_GATM_MINB 3
#endif
template <int G, int VPL, int HM>
__global__ void __launch_bounds__(256, (VPL * HM <= 4) ? GNN_GATM_MINB : 1) gat_bwd_csc_mean_kernel(GatBwdArgs a, float scale) {
  constexpr int NG = 32 / G;
  constexpr int U = 4;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= a.nwarps) return;
  const int lane = (int)lane_id();
  const int g = lane / G, gl = lane % G;
  const unsigned gmask = G == 32 ? kFull : (((1u << G) - 1u) << (g * G));
  const int64_t e0 = w * a.P, e1 = min(e0 + a.P, a.nnz);
  const bool h4 = HM == 4 && a.H == 4;
  int64_t col[VPL];
  bool cv[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    col[v] = (int64_t)(v * G + gl) * 4;
    cv[v] = col[v] < a.F;
    if (!cv[v]) col[v] = 0;
  }
  RowWalk rw(a.offsets, a.R, a.chunk_row[w]);
  while (true) {
    const int64_t lo = max(rw.rs, e0), hi = min(rw.re, e1);
    if (hi > lo) {
      const int64_t u = rw.r;
      float4 self[HM][VPL], acc[HM][VPL];
#pragma unroll
      for (int h = 0; h < HM; ++h)
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          self[h][v] = (h < a.H && cv[v]) ? ldg_f4(a.Wh + u * a.ldw + h * a.F + col[v])
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
          acc[h][v] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      for (int64_t b0 = lo; b0 < hi; b0 += 32) {
        const int nb = (int)min((int64_t)32, hi - b0);
        int32_t myc = 0, mye = 0;
        if (lane < nb) {
          myc = a.rows[b0 + lane];
          mye = a.eid[b0 + lane];
        }
        for (int k0 = 0; k0 < nb; k0 += NG * U) {
          int32_t c[U], ee[U];
          bool ok[U];
#pragma unroll
          for (int t = 0; t < U; ++t) {
            const int k = k0 + t * NG + g;
            ok[t] = k < nb;
            c[t] = __shfl_sync(kFull, myc, k & 31);
            ee[t] = __shfl_sync(kFull, mye, k & 31);
          }
          float4 x[U][VPL];
          float wg[U][HM];
#pragma unroll
          for (int t = 0; t < U; ++t) {
#pragma unroll
            for (int v = 0; v < VPL; ++v)
              x[t][v] = (ok[t] && cv[v]) ? ldg_f4(a.dY + (int64_t)c[t] * a.ldy + col[v])
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
            if (h4) {
              const float4 al = ok[t] ? ldg_f4(a.alpha + (int64_t)ee[t] * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
              wg[t][0] = al.x;
              wg[t][1] = al.y;
              wg[t][2] = al.z;
              wg[t][3] = al.w;
            } else {
#pragma unroll
              for (int h = 0; h < HM; ++h)
                wg[t][h] = (ok[t] && h < a.H) ? __ldg(a.alpha + (int64_t)ee[t] * a.H + h) : 0.f;
            }
          }
#pragma unroll
          for (int t = 0; t < U; ++t) {
            float ph[HM];
#pragma unroll
            for (int h = 0; h < HM; ++h) {
              float p = 0.f;
#pragma unroll
              for (int v = 0; v < VPL; ++v) {
                acc[h][v] = f4_fma(wg[t][h], x[t][v], acc[h][v]);
                p = fmaf(x[t][v].x, self[h][v].x, p);
                p = fmaf(x[t][v].y, self[h][v].y, p);
                p = fmaf(x[t][v].z, self[h][v].z, p);
                p = fmaf(x[t][v].w, self[h][v].w, p);
              }
              ph[h] = p;
            }
            bool done = false;
            if constexpr (HM == 4 && G >= 4) {
              if (a.H == 4) {
                int hh;
                const float sum = reduce4_scatter<G>(ph, gmask, gl, &hh);
                if (ok[t] && (gl & (G / 4 - 1)) == 0) a.dalpha[(int64_t)ee[t] * 4 + hh] = sum * scale;
                done = true;
              }
            }
            if (!done) {
#pragma unroll
              for (int o = 1; o < G; o <<= 1)
#pragma unroll
                for (int h = 0; h < HM; ++h) ph[h] += __shfl_xor_sync(gmask, ph[h], o);
              if (ok[t] && gl == 0)
#pragma unroll
                for (int h = 0; h < HM; ++h)
                  if (h < a.H) a.dalpha[(int64_t)ee[t] * a.H + h] = ph[h] * scale;
            }
          }
        }
      }
#pragma unroll
      for (int o = G; o < 32; o <<= 1)
#pragma unroll
        for (int h = 0; h < HM; ++h)
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            acc[h][v] = f4_add(acc[h][v], make_float4(__shfl_xor_sync(kFull, acc[h][v].x, o),
                                                      __shfl_xor_sync(kFull, acc[h][v].y, o),
                                                      __shfl_xor_sync(kFull, acc[h][v].z, o),
                                                      __shfl_xor_sync(kFull, acc[h][v].w, o)));
      const bool carry = rw.rs < e0, trail = !carry && rw.re > e1;
      float *dst = (carry || trail) ? a.slots + (w * 2 + (carry ? 0 : 1)) * a.K : a.dWh + u * a.ldd;
      if (g == 0)
#pragma unroll
        for (int h = 0; h < HM; ++h)
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            if (h < a.H && cv[v]) {
              const float4 r = acc[h][v];
              *reinterpret_cast<float4 *>(dst + h * a.F + col[v]) =
                  make_float4(r.x * scale, r.y * scale, r.z * scale, r.w * scale);
            }
    }
    if (rw.re >= e1 || rw.r + 1 >= a.R) break;
    rw.next();
  }
}

// Split rows: sum the partials of row s (slot[wa][1], slot[wa+j][0]) in j order.
__global__ void gat_bwd_finalize_kernel(GatBwdArgs a) {
  const int64_t s = blockIdx.x;
  if (s >= a.num_split) return;
  const int64_t r = a.split_rows[s];
  const int64_t rs = a.offsets[r], re = a.offsets[r + 1];
  const int64_t wa = rs / a.P, wb = (re - 1) / a.P;
  for (int64_t c = threadIdx.x; c < a.K; c += blockDim.x) {
    float t = 0.f;
    for (int64_t j = 0; j <= wb - wa; ++j)
      t += a.slots[((wa + j) * 2 + (j == 0 ? 1 : 0)) * a.K + c];
    a.dWh[r * a.ldd + c] = t;
  }
}

__global__ void gat_bwd_empty_kernel(GatBwdArgs a) {
  const int64_t total = a.num_empty * a.K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    a.dWh[(int64_t)a.empty_rows[t / a.K] * a.ldd + t % a.K] = 0.f;
}

template <int G, int VPL>
void launch_gat_bwd(const GatBwdArgs &a, bool pow2, int LPH, unsigned grid, cudaStream_t st) {
  if (pow2)
    gat_bwd_csc_kernel<G, VPL, 1, true><<<grid, 256, 0, st>>>(a, LPH);
  else if (a.H <= 4)
    gat_bwd_csc_kernel<G, VPL, 4, false><<<grid, 256, 0, st>>>(a, LPH);
  else
    gat_bwd_csc_kernel<G, VPL, 8, false><<<grid, 256, 0, st>>>(a, LPH);
}


// ------------------------- GAT backward with alpha recomputed (4 heads)
// The forward softmax keeps per-row statistics (max m, 1/sum) next to er, so
// this backward never reads alpha [E,4] or writes dalpha: over the CSC, edge
// (v -> u) recomputes
//   alpha_h = exp(LeakyReLU(el[u,h] + er[v,h]) - m[v,h]) * inv[v,h]
// with the forward's exact operations (bit-identical), and the softmax
// backward folds in through one per-row scalar per head,
//   S[v,h] = sum_e alpha_e,h dalpha_e,h = < dY_h[v], Yagg_h[v] >
// (Yagg = the forward's pre-bias aggregate sum_e alpha_e Wh_h[u_e]; SpMMve is
// linear), so that
//   ds_e,h = alpha (dalpha - S[v,h]) * LeakyReLU'(pre)
// forms inside the same pass.  del[u] (column sums of ds) accumulates in
// registers; ds is written once, in CSC order (coalesced), for
// der[v] = row sums (gnn_segment_sum over the CSR through the CSR -> CSC
// position map).  Row statistics are packed per (v, h) as a float4
// {er, m, inv, S}: one 64-byte row gathered next to dY[v].

// S for a concatenated-heads layer (+bias, ReLU): dYm is the ReLU-masked
// upstream gradient; where the mask is 0 the product vanishes, elsewhere
// Y - b = Yagg exactly the aggregate the forward produced.  G lanes per row
// (G >= K/4), one float4 column each; F % 4 == 0 keeps a float4 in one head.
template <int G>
__global__ void __launch_bounds__(256) gat_rowstat_kernel(int64_t V, int64_t K,
                                                          const float *__restrict__ dYm, int64_t ldd,
                                                          const float *__restrict__ Y, int64_t ldy,
                                                          const float *__restrict__ bias,
                                                          const float *__restrict__ er,
                                                          const float *__restrict__ mstat,
                                                          float *__restrict__ P, int64_t ldp) {
  constexpr int NR = 32 / G;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (warp * NR >= V) return;
  const int lane = (int)lane_id();
  const int64_t v = warp * NR + lane / G;
  const int gl = lane % G;
  const unsigned gmask = G == 32 ? kFull : (((1u << G) - 1u) << ((lane / G) * G));
  const int64_t F = K / 4;
  const int64_t col = 4 * (int64_t)gl;
  float ph[4] = {0.f, 0.f, 0.f, 0.f};
  if (v < V && col < K) {
    const float4 x = ldg_f4(dYm + v * ldd + col);
    const float4 y = ldg_f4(Y + v * ldy + col);
    const float4 b = bias ? ldg_f4(bias + col) : make_float4(0.f, 0.f, 0.f, 0.f);
    float p = x.x * (y.x - b.x);
    p = fmaf(x.y, y.y - b.y, p);
    p = fmaf(x.z, y.z - b.z, p);
    p = fmaf(x.w, y.w - b.w, p);
    const int h = (int)(col / F);
#pragma unroll
    for (int hh = 0; hh < 4; ++hh) ph[hh] = hh == h ? p : 0.f;
  }
#pragma unroll
  for (int o = 1; o < G; o <<= 1)
#pragma unroll
    for (int hh = 0; hh < 4; ++hh) ph[hh] += __shfl_xor_sync(gmask, ph[hh], o);
  if (v < V && gl < 4) {
    const float S = gl == 0 ? ph[0] : gl == 1 ? ph[1] : gl == 2 ? ph[2] : ph[3];
    reinterpret_cast<float4 *>(P + v * ldp)[gl] =
        make_float4(__ldg(er + v * 4 + gl), __ldg(mstat + v * 8 + gl), __ldg(mstat + v * 8 + 4 + gl), S);
  }
}

// S for the head-mean output layer in the aggregate-then-transform order
// (gnn_spmm_shared_heads): the forward keeps Yc[v, 4i+h] = sum_e alpha_e,h
// X[u_e, i] and the head-h pre-mean logits are Yc_h W_h, so
//   S[v,h] = scale * < dZ[v], Yc_h[v] W_h > = scale * sum_i Yc[v,4i+h] (W_h dZ[v])_i.
// W [F1][4*Cp] staged in shared memory as float4 [F1][4][CP4]; thread per
// vertex, warp-uniform shared reads (broadcasts); grid-stride over vertices
// so every block stages W once.
template <int CP4>
__global__ void __launch_bounds__(128) gat_rowstat_mean_kernel(
    int64_t V, int64_t F1, int64_t Cp, const float *__restrict__ dZ, int64_t ldz,
    const float *__restrict__ Yc, int64_t ldc, const float *__restrict__ W, int64_t ldw, float scale,
    const float *__restrict__ er, const float *__restrict__ mstat, float *__restrict__ P, int64_t ldp) {
  extern __shared__ float4 Ws[];
  const int64_t nw = F1 * 4 * CP4;
  for (int64_t t = threadIdx.x; t < nw; t += blockDim.x) {
    const int64_t i = t / (4 * CP4), rem = t % (4 * CP4);
    const int64_t h = rem / CP4, c4 = rem % CP4;
    Ws[t] = 4 * c4 < Cp ? ldg_f4(W + i * ldw + h * Cp + 4 * c4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    float4 dz[CP4];
#pragma unroll
    for (int c = 0; c < CP4; ++c) dz[c] = ldg_f4(dZ + v * ldz + 4 * c);
    float S[4] = {0.f, 0.f, 0.f, 0.f};
    for (int64_t i = 0; i < F1; ++i) {
      const float4 yc = ldg_f4(Yc + v * ldc + 4 * i);
      const float ych[4] = {yc.x, yc.y, yc.z, yc.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float4 *w = Ws + (i * 4 + h) * CP4;
        float g0 = 0.f, g1 = 0.f;
#pragma unroll
        for (int c = 0; c < CP4; ++c) {
          const float4 wv = w[c];
          g0 = fmaf(wv.x, dz[c].x, g0);
          g1 = fmaf(wv.y, dz[c].y, g1);
          g0 = fmaf(wv.z, dz[c].z, g0);
          g1 = fmaf(wv.w, dz[c].w, g1);
        }
        S[h] = fmaf(ych[h], g0 + g1, S[h]);
      }
    }
#pragma unroll
    for (int h = 0; h < 4; ++h)
      reinterpret_cast<float4 *>(P + v * ldp)[h] =
          make_float4(__ldg(er + v * 4 + h), __ldg(mstat + v * 8 + h), __ldg(mstat + v * 8 + 4 + h),
                      scale * S[h]);
  }
}

struct GatRcArgs {
  int64_t R, nnz, P, nwarps;
  const int64_t *offsets;
  const int32_t *rows;  // CSC "cols": source vertices v
  const int32_t *chunk_row;
  const int32_t *split_rows;
  int64_t num_split;
  const int32_t *empty_rows;
  int64_t num_empty;
  int64_t F, K;          // per-head width; K = dWh row width (4F)
  const float *el;       // [V][4]
  float slope, scale;
  const float *dY;       // layer gradient rows [R floats | {er, m, inv, S} x 4] (R = K, or F for the mean form)
  int64_t ldy;
  const float *Wh;
  int64_t ldw;
  float *dWh;
  int64_t ldd;
  float *del;            // [R][4]
  float *ds;             // [nnz][4]: CSC order, or CSR order through ds_map
  const int32_t *ds_map; // optional CSC position -> CSR edge (the edge-ID array)
  float *slots;          // [nwarps][2][K + 4]
};


__device__ __forceinline__ float gat_alpha(float el, float4 st, float slope, float &pre) {
  pre = el + st.x;
  const float s = pre > 0.f ? pre : slope * pre;
  return __expf(s - st.y) * st.z;
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
// src_bytes = 0 writes zeros and reads nothing: predication without a branch
__device__ __forceinline__ void cp_async16_zfill(void *dst, const void *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The CSC pass is a gather of one row per edge (dY[v], 4F floats; head-mean
// form: dZ[v], F floats) plus the 64-byte statistics row of v, from arrays
// several times larger than L2: it needs many gathers in flight.  Each warp
// streams its chunk's edges through a private S-stage shared-memory ring, NB
// edges per stage, with cp.async (16-byte copies, L1 bypassed): S*NB edges
// in flight per warp at no register cost, S-1 stages ahead of the edge being
// reduced.  G lanes per edge, NG = 32/G edges per step; within a group lane
// gl owns head h = gl / (G/4) and CPL consecutive columns c0 of it.  Edges
// are taken in chunk order and a step never spans two CSC rows (a step at a
// row end runs with fewer groups), so every group accumulates the same row:
// at the row end the groups' dWh / del partials combine by xor shuffles.
// Every lane of head h recomputes alpha_h from the staged {er, m, inv, S}.
constexpr int kRcNB = 8;   // edges per stage
// stages per warp: as deep as two 8-warp blocks per SM allow (~110 KB each)
template <int Q>
constexpr int rc_stages() {
  return (110 * 1024) / (8 * kRcNB * Q * 16) < 4 ? 4 : (110 * 1024) / (8 * kRcNB * Q * 16);
}

template <int G, int CPL, bool MEAN>
struct RcShape {
  static constexpr int LPH = G / 4;              // lanes per head
  static constexpr int F = LPH * CPL;            // per-head width
  static constexpr int R = MEAN ? F : 4 * F;     // gathered floats per edge
  static constexpr int Q = (R + 16) / 4;         // float4 per edge slot (row + stats)
};

// fp32 pair helpers on 64-bit registers (sm_100 FFMA2): a += b * c lane-wise
__device__ __forceinline__ void ffma2(unsigned long long &a, unsigned long long b,
                                      unsigned long long c) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(b), "l"(c));
}
__device__ __forceinline__ unsigned long long pack2(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ float2 unpack2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}

template <int G, int CPL, bool MEAN, int MINB>
__global__ void __launch_bounds__(256, MINB) gat_bwd_rcp_kernel(GatRcArgs a) {
  using Sh = RcShape<G, CPL, MEAN>;
  constexpr int NG = 32 / G, LPH = Sh::LPH;
  constexpr int F = Sh::F, R = Sh::R, Q = Sh::Q, NB = kRcNB, S = rc_stages<Sh::Q>();
  constexpr int STAGE = NB * Q;                  // float4 per stage
  constexpr int CP2 = CPL / 2;                   // column pairs per lane
  static_assert(CPL % 2 == 0 && NB % NG == 0 && NB <= 32, "shape");
  constexpr int NCP = (STAGE + 31) / 32;         // 16-byte copies per lane per stage
  extern __shared__ float4 rc_smem[];
  const int nw = (int)(blockDim.x >> 5), wib = (int)(threadIdx.x >> 5);
  const uint32_t ring_s = smem_u32(rc_smem + (size_t)wib * S * STAGE);
  int32_t *mring = reinterpret_cast<int32_t *>(rc_smem + (size_t)nw * S * STAGE) + wib * S * NB;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= a.nwarps) return;
  const int lane = (int)lane_id();
  const int g = lane / G, gl = lane % G;
  const int h = gl / LPH, cl = gl % LPH, c0 = cl * CPL;
  const int64_t e0 = w * a.P;
  const int ne_all = (int)(min(e0 + a.P, a.nnz) - e0);   // edges of this chunk
  const int64_t e1 = e0 + ne_all;
  const int nst = (ne_all + NB - 1) / NB;
  // byte offsets of this lane's operands inside an edge slot
  const uint32_t xoff = 4u * (uint32_t)((MEAN ? 0 : h * F) + c0);
  const uint32_t soff = 4u * (uint32_t)(R + 4 * h);
  const char *dYb = reinterpret_cast<const char *>(a.dY);
  const int64_t ldyb = a.ldy * 4;

  // id batches of the issue side (32 edges): rows / CSR edge ids of cur, next
  const int32_t *rows = a.rows + e0;
  const int32_t *map = a.ds_map + e0;
  int32_t cur_v = lane < ne_all ? __ldg(rows + lane) : 0;
  int32_t cur_m = lane < ne_all ? __ldg(map + lane) : 0;
  int32_t nxt_v = 32 + lane < ne_all ? __ldg(rows + 32 + lane) : 0;
  int32_t nxt_m = 32 + lane < ne_all ? __ldg(map + 32 + lane) : 0;
  int cur_b = 0;

  // stage k: every lane copies NCP 16-byte pieces of the stage's rows (a row is the
  // gradient and the statistics of v, contiguous); zero-filled past the chunk end
  auto issue = [&](int k) {
    if (k < nst) {
      const int b = (k * NB) >> 5;
      if (b != cur_b) {  // k grows by one per call: advance one batch
        cur_v = nxt_v;
        cur_m = nxt_m;
        cur_b = b;
        const int e = (b + 1) * 32 + lane;
        nxt_v = e < ne_all ? __ldg(rows + e) : 0;
        nxt_m = e < ne_all ? __ldg(map + e) : 0;
      }
      const int off = (k * NB) & 31;
      const uint32_t dst = ring_s + (uint32_t)((k % S) * STAGE) * 16u;
#pragma unroll
      for (int i = 0; i < NCP; ++i) {
        const int f = i * 32 + lane;
        const int ei = f / Q, piece = f - ei * Q;
        const int32_t v = __shfl_sync(kFull, cur_v, (off + ei) & 31);
        if (STAGE % 32 == 0 || f < STAGE)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + 16u * f),
                       "l"(dYb + (int64_t)v * ldyb + 16 * piece), "r"(k * NB + ei < ne_all ? 16 : 0)
                       : "memory");
      }
      const int32_t m = __shfl_sync(kFull, cur_m, (off + (lane & (NB - 1))) & 31);
      if (lane < NB) mring[(k % S) * NB + lane] = m;
    }
    cp_async_commit();
  };

#pragma unroll
  for (int k = 0; k < S - 1; ++k) issue(k);

  RowWalk rw(a.offsets, a.R, a.chunk_row[w]);
  while (rw.re <= e0 && rw.r + 1 < a.R) rw.next();
  unsigned long long self[CP2], acc[CP2];
  float elu = 0.f, dl = 0.f;
  int re_rel = 0;  // end of the current row, relative to e0, clamped to the chunk
  auto row_begin = [&]() {
    const float *p = a.Wh + rw.r * a.ldw + h * F + c0;
#pragma unroll
    for (int j = 0; j < CP2; ++j) {
      const float2 t = __ldg(reinterpret_cast<const float2 *>(p) + j);
      self[j] = pack2(t.x, t.y);
      acc[j] = 0ull;
    }
    elu = __ldg(a.el + rw.r * 4 + h);
    dl = 0.f;
    re_rel = (int)(min(rw.re, e1) - e0);
  };
  auto row_end = [&]() {  // the warp's piece of row rw.r is complete
    float2 av[CP2];
#pragma unroll
    for (int j = 0; j < CP2; ++j) av[j] = unpack2(acc[j]);
#pragma unroll
    for (int o = G; o < 32; o <<= 1) {
#pragma unroll
      for (int j = 0; j < CP2; ++j) {
        av[j].x += __shfl_xor_sync(kFull, av[j].x, o);
        av[j].y += __shfl_xor_sync(kFull, av[j].y, o);
      }
      dl += __shfl_xor_sync(kFull, dl, o);
    }
    if (g != 0) return;
    const bool carry = rw.rs < e0, trail = !carry && rw.re > e1;
    float *drow = (carry || trail) ? a.slots + (w * 2 + (carry ? 0 : 1)) * (a.K + 4)
                                   : a.dWh + rw.r * a.ldd;
    const float sc = MEAN ? a.scale : 1.f;
#pragma unroll
    for (int j = 0; j < CP2; ++j)
      *reinterpret_cast<float2 *>(drow + h * F + c0 + 2 * j) = make_float2(av[j].x * sc, av[j].y * sc);
    if (cl == 0) ((carry || trail) ? drow + a.K : a.del + rw.r * 4)[h] = dl;
  };
  // one step: group g reduces the edge in slot `se`; act = false contributes nothing
  auto step = [&](uint32_t st0, int se, bool act, int32_t mapid) {
    const uint32_t slot = st0 + (uint32_t)(se * Q) * 16u;
    unsigned long long x[CP2];
#pragma unroll
    for (int j = 0; j + 1 < CP2; j += 2)
      asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x[j]), "=l"(x[j + 1])
                   : "r"(slot + xoff + 8u * j));
    if (CP2 % 2)
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(x[CP2 - 1]) : "r"(slot + xoff + 8u * (CP2 - 1)));
    float4 stv;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(stv.x), "=f"(stv.y), "=f"(stv.z), "=f"(stv.w) : "r"(slot + soff));
    float pre;
    float al = gat_alpha(elu, stv, a.slope, pre);
    al = act ? al : 0.f;
    const unsigned long long al2 = pack2(al, al);
    unsigned long long pa = 0ull, pb = 0ull;
#pragma unroll
    for (int j = 0; j < CP2; ++j) {
      ffma2(acc[j], al2, x[j]);
      ffma2((j & 1) ? pb : pa, x[j], self[j]);
    }
    const float2 va = unpack2(pa), vb = unpack2(pb);
    float p = (va.x + va.y) + (vb.x + vb.y);
#pragma unroll
    for (int o = 1; o < LPH; o <<= 1) p += __shfl_xor_sync(kFull, p, o);  // within the head
    if (MEAN) p *= a.scale;
    float d = al * (p - stv.w);
    d = pre > 0.f ? d : a.slope * d;
    dl += d;
    if (act && cl == 0) a.ds[(int64_t)mapid * 4 + h] = d;
  };
  row_begin();

  for (int k = 0; k < nst; ++k) {
    issue(k + S - 1);
    cp_async_wait<S - 1>();
    __syncwarp();
    const uint32_t st0 = ring_s + (uint32_t)((k % S) * STAGE) * 16u;
    const int32_t *mr = mring + (k % S) * NB;
    const int eb = k * NB;
    const int ne = min(NB, ne_all - eb);
    if (ne == NB && eb + NB <= re_rel) {
      // the whole stage lies in the current row: NB/NG full steps, no bookkeeping
#pragma unroll
      for (int u = 0; u < NB / NG; ++u) step(st0, u * NG + g, true, mr[u * NG + g]);
      if (eb + NB == re_rel && eb + NB < ne_all) {
        row_end();
        const int64_t en = e0 + eb + NB;
        do {
          rw.next();
        } while (rw.re <= en);
        row_begin();
      }
    } else {
      int ei = 0;
      while (ei < ne) {
        // n edges of the current row in this step (warp-uniform); group g takes edge
        // ei + g; an idle group (row end) reads the first edge's slot with alpha = 0
        const int n = min(min(NG, ne - ei), re_rel - (eb + ei));
        const bool act = g < n;
        step(st0, ei + (act ? g : 0), act, mr[ei + (act ? g : 0)]);
        ei += n;
        if (eb + ei == re_rel && eb + ei < ne_all) {  // row complete: flush, next non-empty row
          row_end();
          const int64_t en = e0 + eb + ei;
          do {
            rw.next();
          } while (rw.re <= en);
          row_begin();
        }
      }
    }
    __syncwarp();  // every lane is done with slot k % S before it is refilled
  }
  row_end();
}

// Split rows: partials of row s (slot[wa][1], slot[wa+j][0]) summed in j order.
__global__ void gat_rc_finalize_kernel(GatRcArgs a) {
  const int64_t s = blockIdx.x;
  if (s >= a.num_split) return;
  const int64_t r = a.split_rows[s];
  const int64_t rs = a.offsets[r], re = a.offsets[r + 1];
  const int64_t wa = rs / a.P, wb = (re - 1) / a.P;
  for (int64_t c = threadIdx.x; c < a.K + 4; c += blockDim.x) {
    float t = 0.f;
    for (int64_t j = 0; j <= wb - wa; ++j)
      t += a.slots[((wa + j) * 2 + (j == 0 ? 1 : 0)) * (a.K + 4) + c];
    if (c < a.K)
      a.dWh[r * a.ldd + c] = t;
    else
      a.del[r * 4 + (c - a.K)] = t;
  }
}

__global__ void gat_rc_empty_kernel(GatRcArgs a) {
  const int64_t W = a.K + 4;
  const int64_t total = a.num_empty * W;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = a.empty_rows[t / W], c = t % W;
    if (c < a.K)
      a.dWh[r * a.ldd + c] = 0.f;
    else
      a.del[r * 4 + (c - a.K)] = 0.f;
  }
}

__global__ void invert_permutation_kernel(int64_t n, const int32_t *__restrict__ perm,
                                          int32_t *__restrict__ inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    inv[perm[i]] = (int32_t)i;
}

int gat_rc_common(const gnn_csr_view_t *AT, const gnn_spmm_plan_t *plan, const float *el,
                  float slope, const float *dY, int64_t ldy, const float *Wh, int64_t ldw,
                  float *dWh, int64_t ldd, float *del, float *ds, void *ws, size_t ws_bytes,
                  int64_t F, int64_t K, int64_t R, GatRcArgs &a) {
  if (!AT || !plan || !AT->offsets || AT->col_bits || AT->row_ids || F <= 0 || F % 4 || K % 4)
    return GNN_ERR_INVALID_ARGUMENT;
  if (ldy % 4 || ldw % 4 || ldd % 4 || ldw < K || ldd < K || ldy < R + 16) return GNN_ERR_UNSUPPORTED;
  if (AT->num_rows > 0 && (!dWh || !Wh || !del || !el || !al16(Wh) || !al16(dWh)))
    return GNN_ERR_INVALID_ARGUMENT;
  if (AT->nnz > 0 && (!AT->cols || !AT->eid || !dY || !ds || !al16(dY)))
    return GNN_ERR_INVALID_ARGUMENT;
  if (plan->dev_counts || plan->edges_per_warp <= 0 || plan->num_warps != ceil_div(AT->nnz, plan->edges_per_warp))
    return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_gat_bwd_rc_workspace(plan, K)) return GNN_ERR_WORKSPACE;
  a = GatRcArgs{};
  a.R = AT->num_rows;
  a.nnz = AT->nnz;
  a.P = plan->edges_per_warp;
  a.nwarps = plan->num_warps;
  a.offsets = AT->offsets;
  a.rows = AT->cols;
  a.chunk_row = plan->chunk_row;
  a.split_rows = plan->split_rows;
  a.num_split = plan->num_split;
  a.empty_rows = plan->empty_rows;
  a.num_empty = plan->num_empty;
  a.F = F;
  a.K = K;
  a.el = el;
  a.slope = slope;
  a.scale = 1.f;
  a.dY = dY;
  a.ldy = ldy;
  a.Wh = Wh;
  a.ldw = ldw;
  a.dWh = dWh;
  a.ldd = ldd;
  a.del = del;
  a.ds = ds;
  a.ds_map = AT->eid;  // ds lands in CSR edge order (der = a plain CSR row sum)
  a.slots = static_cast<float *>(ws);
  return GNN_OK;
}

int gat_rc_tail(const GatRcArgs &a, cudaStream_t st) {
  if (a.num_split > 0) {
    gat_rc_finalize_kernel<<<(unsigned)a.num_split, 128, 0, st>>>(a);
    GNN_LAUNCH_CHECK();
  }
  if (a.num_empty > 0) {
    gat_rc_empty_kernel<<<grid_1d_a(a.num_empty * (a.K + 4), 256), 256, 0, st>>>(a);
    GNN_LAUNCH_CHECK();
  }
  return GNN_OK;
}

}  // namespace
}  // namespace gnn

using namespace gnn;

extern "C" {

int gnn_sddmm(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads, const float *X,
              int64_t ldx, const float *Y, int64_t ldy, int64_t K, float *out,
              gnn_stream_t stream) {
  if ((A && (A->col_bits || A->row_ids)) || !A || !plan || heads <= 0 || K <= 0 || K % heads != 0 || !A->offsets)
    return GNN_ERR_INVALID_ARGUMENT;
  if (A->nnz > 0 && (!A->cols || !X || !Y || !out || ldx < K || ldy < K))
    return GNN_ERR_INVALID_ARGUMENT;
  if (plan->dev_counts || plan->edges_per_warp <= 0 || plan->num_warps != ceil_div(A->nnz, plan->edges_per_warp))
    return GNN_ERR_INVALID_ARGUMENT;
  if (A->nnz == 0) return GNN_OK;
  cudaStream_t st = as_stream(stream);
  SddmmArgs a{};
  a.R = A->num_rows;
  a.nnz = A->nnz;
  a.P = plan->edges_per_warp;
  a.nwarps = plan->num_warps;
  a.offsets = A->offsets;
  a.cols = A->cols;
  a.chunk_row = plan->chunk_row;
  a.H = (int)heads;
  a.F = K / heads;
  a.K = K;
  a.X = X;
  a.ldx = ldx;
  a.Y = Y;
  a.ldy = ldy;
  a.out = out;
  const int64_t q = K / 4;  // float4 columns
  int G = 1;
  while (G < q && G < 32) G <<= 1;
  const int64_t lph = a.F / 4;
  const bool lph_pow2 = lph > 0 && (lph & (lph - 1)) == 0;
  const bool vec = K % 4 == 0 && a.F % 4 == 0 && ldx % 4 == 0 && ldy % 4 == 0 && al16(X) &&
                   al16(Y) && ceil_div(q, G) <= 4;
  const bool pow2 = lph_pow2 && lph <= G;
  const unsigned grid = grid_warps(a.nwarps, 256);
  const int VPL = (int)ceil_div(q, G);
  const int LPH = (int)lph;
  if (vec && pow2) {
    switch (G) {
      case 1: sddmm_vec_kernel<1, 1, 0><<<grid, 256, 0, st>>>(a, LPH); break;
      case 2: sddmm_vec_kernel<2, 1, 0><<<grid, 256, 0, st>>>(a, LPH); break;
      case 4: sddmm_vec_kernel<4, 1, 0><<<grid, 256, 0, st>>>(a, LPH); break;
      case 8: sddmm_vec_kernel<8, 1, 0><<<grid, 256, 0, st>>>(a, LPH); break;
      case 16: sddmm_vec_kernel<16, 1, 0><<<grid, 256, 0, st>>>(a, LPH); break;
      default:
        if (VPL == 1)
          sddmm_vec_kernel<32, 1, 0><<<grid, 256, 0, st>>>(a, LPH);
        else if (VPL == 2)
          sddmm_vec_kernel<32, 2, 0><<<grid, 256, 0, st>>>(a, LPH);
        else
          sddmm_vec_kernel<32, 4, 0><<<grid, 256, 0, st>>>(a, LPH);
    }
  } else if (vec && heads <= 8) {
    // general head mapping (e.g. GAT's 4 x 48 output heads); G >= 2 here
    const bool h4 = heads <= 4;
    switch (G) {
      case 2: h4 ? sddmm_vec_kernel<2, 1, 4><<<grid, 256, 0, st>>>(a, LPH)
                 : sddmm_vec_kernel<2, 1, 8><<<grid, 256, 0, st>>>(a, LPH); break;
      case 4: h4 ? sddmm_vec_kernel<4, 1, 4><<<grid, 256, 0, st>>>(a, LPH)
                 : sddmm_vec_kernel<4, 1, 8><<<grid, 256, 0, st>>>(a, LPH); break;
      case 8: h4 ? sddmm_vec_kernel<8, 1, 4><<<grid, 256, 0, st>>>(a, LPH)
                 : sddmm_vec_kernel<8, 1, 8><<<grid, 256, 0, st>>>(a, LPH); break;
      case 16: h4 ? sddmm_vec_kernel<16, 1, 4><<<grid, 256, 0, st>>>(a, LPH)
                  : sddmm_vec_kernel<16, 1, 8><<<grid, 256, 0, st>>>(a, LPH); break;
      default:
        if (VPL == 1)
          h4 ? sddmm_vec_kernel<32, 1, 4><<<grid, 256, 0, st>>>(a, LPH)
             : sddmm_vec_kernel<32, 1, 8><<<grid, 256, 0, st>>>(a, LPH);
        else if (VPL == 2)
          h4 ? sddmm_vec_kernel<32, 2, 4><<<grid, 256, 0, st>>>(a, LPH)
             : sddmm_vec_kernel<32, 2, 8><<<grid, 256, 0, st>>>(a, LPH);
        else
          h4 ? sddmm_vec_kernel<32, 4, 4><<<grid, 256, 0, st>>>(a, LPH)
             : sddmm_vec_kernel<32, 4, 8><<<grid, 256, 0, st>>>(a, LPH);
    }
  } else {
    sddmm_scalar_kernel<<<grid, 256, 0, st>>>(a);
  }
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

size_t gnn_edge_softmax_workspace(const gnn_spmm_plan_t *plan, int64_t heads) {
  if (!plan || heads <= 0) return 0;
  size_t o;
  return softmax_ws_layout(plan, heads, &o);
}

int gnn_edge_softmax_fwd(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
                         const gnn_edge_scores_t *sc, float *alpha, void *ws, size_t ws_bytes,
                         gnn_stream_t stream) {
  SoftmaxArgs a;
  GNN_TRY(softmax_common(A, plan, heads, sc, ws, ws_bytes, a));
  if (!sc) return GNN_ERR_INVALID_ARGUMENT;
  const bool gat = sc->s == nullptr;
  if (A->nnz > 0 && (!alpha || (gat && (!sc->el || !sc->er)))) return GNN_ERR_INVALID_ARGUMENT;
  if (A->nnz == 0) return GNN_OK;
  if (heads == 4 && (!al16(alpha) || (gat ? !al16(sc->el) : !al16(sc->s))))
    return GNN_ERR_INVALID_ARGUMENT;
  a.alpha = alpha;
  cudaStream_t st = as_stream(stream);
  return gat ? dispatch_softmax<true, false>(a, st) : dispatch_softmax<false, false>(a, st);
}

int gnn_edge_softmax_bwd(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
                         const float *alpha, const float *dalpha, const gnn_edge_scores_t *sc,
                         float *ds, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  SoftmaxArgs a;
  GNN_TRY(softmax_common(A, plan, heads, sc, ws, ws_bytes, a));
  const bool gat = sc && sc->el;
  if (A->nnz > 0 && (!alpha || !dalpha || !ds || (gat && !sc->er))) return GNN_ERR_INVALID_ARGUMENT;
  if (A->nnz == 0) return GNN_OK;
  a.alpha_in = alpha;
  a.dalpha = dalpha;
  a.ds = ds;
  cudaStream_t st = as_stream(stream);
  return gat ? dispatch_softmax<true, true>(a, st) : dispatch_softmax<false, true>(a, st);
}

int gnn_segment_sum(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
                    const float *vals, float *out, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  SoftmaxArgs a;
  GNN_TRY(softmax_common(A, plan, heads, nullptr, ws, ws_bytes, a));
  if (A->num_rows > 0 && !out) return GNN_ERR_INVALID_ARGUMENT;
  if (A->nnz > 0 && !vals) return GNN_ERR_INVALID_ARGUMENT;
  if (A->num_rows == 0) return GNN_OK;
  if (heads == 4 && !al16(vals)) return GNN_ERR_INVALID_ARGUMENT;
  a.alpha_in = vals;
  a.ds = out;
  a.eid = A->eid;
  cudaStream_t st = as_stream(stream);
  const bool e = A->eid != nullptr;
  if (heads == 1) return launch_segsum<1>(a, e, st);
  if (heads <= 4) return launch_segsum<4>(a, e, st);
  if (heads <= 8) return launch_segsum<8>(a, e, st);
  return launch_segsum<16>(a, e, st);
}

size_t gnn_gat_bwd_csc_workspace(const gnn_spmm_plan_t *plan, int64_t K) {
  if (!plan || K <= 0) return 0;
  return sizeof(float) * (size_t)(plan->num_warps * 2 * K) + 256;
}

int gnn_gat_bwd_csc(const gnn_csr_view_t *AT, const gnn_spmm_plan_t *plan, int64_t heads,
                    const float *alpha, const float *dY, int64_t ldy, const float *Wh, int64_t ldw,
                    int64_t K, float *dWh, int64_t ldd, float *dalpha, void *ws, size_t ws_bytes,
                    gnn_stream_t stream) {
  if ((AT && (AT->col_bits || AT->row_ids)) || !AT || !plan || heads <= 0 || heads > 8 || K <= 0 || K % heads != 0 || !AT->offsets)
    return GNN_ERR_INVALID_ARGUMENT;
  const int64_t F = K / heads;
  if (K % 4 || F % 4 || ldy % 4 || ldw % 4 || ldd % 4 || ldy < K || ldw < K || ldd < K)
    return GNN_ERR_UNSUPPORTED;
  if (AT->num_rows > 0 && (!dWh || !Wh || !al16(Wh) || !al16(dWh))) return GNN_ERR_INVALID_ARGUMENT;
  if (AT->nnz > 0 && (!AT->cols || !AT->eid || !alpha || !dY || !dalpha || !al16(dY)))
    return GNN_ERR_INVALID_ARGUMENT;
  if (heads == 4 && (!al16(alpha) || !al16(dalpha))) return GNN_ERR_INVALID_ARGUMENT;
  if (plan->dev_counts || plan->edges_per_warp <= 0 || plan->num_warps != ceil_div(AT->nnz, plan->edges_per_warp))
    return GNN_ERR_INVALID_ARGUMENT;
  const int64_t q = K / 4;
  if (q > 128) return GNN_ERR_UNSUPPORTED;
  if (ws_bytes < gnn_gat_bwd_csc_workspace(plan, K)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  GatBwdArgs a{};
  a.R = AT->num_rows;
  a.nnz = AT->nnz;
  a.P = plan->edges_per_warp;
  a.nwarps = plan->num_warps;
  a.offsets = AT->offsets;
  a.rows = AT->cols;
  a.eid = AT->eid;
  a.chunk_row = plan->chunk_row;
  a.chunk_split = plan->chunk_split;
  a.split_rows = plan->split_rows;
  a.num_split = plan->num_split;
  a.empty_rows = plan->empty_rows;
  a.num_empty = plan->num_empty;
  a.H = (int)heads;
  a.F = F;
  a.K = K;
  a.alpha = alpha;
  a.dY = dY;
  a.ldy = ldy;
  a.Wh = Wh;
  a.ldw = ldw;
  a.dWh = dWh;
  a.ldd = ldd;
  a.dalpha = dalpha;
  a.slots = static_cast<float *>(ws);
  // lane layout: exact fits first (e.g. 48 float4 columns -> 16 lanes x 3)
  int G, VPL;
  if (q <= 32) {
    G = 1;
    while (G < q) G <<= 1;
    VPL = 1;
  } else if (q % 16 == 0 && q / 16 <= 4 && q % 32 != 0) {
    G = 16;
    VPL = (int)(q / 16);
  } else {
    G = 32;
    VPL = (int)ceil_div(q, 32);
  }
  const int64_t lph = F / 4;
  const bool pow2 = (lph & (lph - 1)) == 0 && lph <= G && (G * 4) % F == 0;
  const int LPH = (int)lph;
  if (a.nwarps > 0) {
    const unsigned grid = grid_warps(a.nwarps, 256);
    if (VPL == 1) {
      switch (G) {
        case 1: launch_gat_bwd<1, 1>(a, pow2, LPH, grid, st); break;
        case 2: launch_gat_bwd<2, 1>(a, pow2, LPH, grid, st); break;
        case 4: launch_gat_bwd<4, 1>(a, pow2, LPH, grid, st); break;
        case 8: launch_gat_bwd<8, 1>(a, pow2, LPH, grid, st); break;
        case 16: launch_gat_bwd<16, 1>(a, pow2, LPH, grid, st); break;
        default: launch_gat_bwd<32, 1>(a, pow2, LPH, grid, st); break;
      }
    } else if (G == 16) {
      if (VPL == 3)
        launch_gat_bwd<16, 3>(a, pow2, LPH, grid, st);
      else
        launch_gat_bwd<16, 2>(a, pow2, LPH, grid, st);  // unreachable in practice (q%32 != 0)
    } else {
      if (VPL == 2)
        launch_gat_bwd<32, 2>(a, pow2, LPH, grid, st);
      else if (VPL == 3)
        launch_gat_bwd<32, 3>(a, pow2, LPH, grid, st);
      else
        launch_gat_bwd<32, 4>(a, pow2, LPH, grid, st);
    }
    GNN_LAUNCH_CHECK();
  }
  if (a.num_split > 0) {
    gat_bwd_finalize_kernel<<<(unsigned)a.num_split, 128, 0, st>>>(a);
    GNN_LAUNCH_CHECK();
  }
  if (a.num_empty > 0) {
    gat_bwd_empty_kernel<<<grid_1d_a(a.num_empty * K, 256), 256, 0, st>>>(a);
    GNN_LAUNCH_CHECK();
  }
  return GNN_OK;
}

int gnn_gat_bwd_csc_mean(const gnn_csr_view_t *AT, const gnn_spmm_plan_t *plan, int64_t heads,
                         const float *alpha, const float *dZ, int64_t ldz, float scale,
                         const float *Wh, int64_t ldw, int64_t F, float *dWh, int64_t ldd,
                         float *dalpha, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  if ((AT && (AT->col_bits || AT->row_ids)) || !AT || !plan || heads <= 0 || heads > 8 || F <= 0 || !AT->offsets)
    return GNN_ERR_INVALID_ARGUMENT;
  const int64_t K = heads * F;
  if (F % 4 || ldz % 4 || ldw % 4 || ldd % 4 || ldz < F || ldw < K || ldd < K || F > 128)
    return GNN_ERR_UNSUPPORTED;
  if (AT->num_rows > 0 && (!dWh || !Wh || !al16(Wh) || !al16(dWh))) return GNN_ERR_INVALID_ARGUMENT;
  if (AT->nnz > 0 && (!AT->cols || !AT->eid || !alpha || !dZ || !dalpha || !al16(dZ)))
    return GNN_ERR_INVALID_ARGUMENT;
  if (heads == 4 && (!al16(alpha) || !al16(dalpha))) return GNN_ERR_INVALID_ARGUMENT;
  if (plan->dev_counts || plan->edges_per_warp <= 0 || plan->num_warps != ceil_div(AT->nnz, plan->edges_per_warp))
    return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_gat_bwd_csc_workspace(plan, K)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  GatBwdArgs a{};
  a.R = AT->num_rows;
  a.nnz = AT->nnz;
  a.P = plan->edges_per_warp;
  a.nwarps = plan->num_warps;
  a.offsets = AT->offsets;
  a.rows = AT->cols;
  a.eid = AT->eid;
  a.chunk_row = plan->chunk_row;
  a.chunk_split = plan->chunk_split;
  a.split_rows = plan->split_rows;
  a.num_split = plan->num_split;
  a.empty_rows = plan->empty_rows;
  a.num_empty = plan->num_empty;
  a.H = (int)heads;
  a.F = F;
  a.K = K;
  a.alpha = alpha;
  a.dY = dZ;
  a.ldy = ldz;
  a.Wh = Wh;
  a.ldw = ldw;
  a.dWh = dWh;
  a.ldd = ldd;
  a.dalpha = dalpha;
  a.slots = static_cast<float *>(ws);
  const int64_t q = F / 4;
  if (a.nwarps > 0) {
    const unsigned grid = grid_warps(a.nwarps, 256);
    const bool h4 = heads <= 4;
#define GNN_GBM(G, VPL)                                                                 \
  (h4 ? gat_bwd_csc_mean_kernel<G, VPL, 4><<<grid, 256, 0, st>>>(a, scale)              \
      : gat_bwd_csc_mean_kernel<G, VPL, 8><<<grid, 256, 0, st>>>(a, scale))
    if (q <= 4)
      GNN_GBM(4, 1);
    else if (q <= 8)
      GNN_GBM(8, 1);
    else if (q <= 16)
      GNN_GBM(16, 1);
    else if (q <= 32)
      GNN_GBM(32, 1);
    else if (q <= 64)
      GNN_GBM(32, 2);
    else
      GNN_GBM(32, 4);
#undef GNN_GBM
    GNN_LAUNCH_CHECK();
  }
  if (a.num_split > 0) {
    gat_bwd_finalize_kernel<<<(unsigned)a.num_split, 128, 0, st>>>(a);
    GNN_LAUNCH_CHECK();
  }
  if (a.num_empty > 0) {
    gat_bwd_empty_kernel<<<grid_1d_a(a.num_empty * K, 256), 256, 0, st>>>(a);
    GNN_LAUNCH_CHECK();
  }
  return GNN_OK;
}

int gnn_gat_attn_proj(int64_t V, int64_t heads, int64_t F, const float *Wh, int64_t ldw,
                      const float *a_l, const float *a_r, float *el, float *er,
                      gnn_stream_t stream) {
  if (V < 0 || heads <= 0 || F <= 0 || ldw < heads * F) return GNN_ERR_INVALID_ARGUMENT;
  if (V == 0) return GNN_OK;
  if (!Wh || !a_l || !a_r || !el || !er) return GNN_ERR_INVALID_ARGUMENT;
  cudaStream_t st = as_stream(stream);
  if (F % 4 == 0 && ldw % 4 == 0 && al16(Wh) && al16(a_l) && al16(a_r)) {
    attn_proj_vec_kernel<<<grid_1d_a(V * heads * 4, 256), 256, 0, st>>>(V, (int)heads, F, Wh, ldw,
                                                                         a_l, a_r, el, er);
    GNN_LAUNCH_CHECK();
    return GNN_OK;
  }
  attn_proj_kernel<<<grid_1d_a(V * heads, 256), 256, 0, st>>>(V, (int)heads, F, Wh, ldw, a_l, a_r,
                                                              el, er);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

size_t gnn_gat_attn_proj_bwd_workspace(int64_t heads, int64_t F) {
  return (size_t)kProjBlocks * 2 * heads * F * sizeof(float) + 256;
}

int gnn_gat_attn_proj_bwd(int64_t V, int64_t heads, int64_t F, const float *Wh, int64_t ldw,
                          const float *a_l, const float *a_r, const float *del, const float *der,
                          float *dWh, int64_t ldd, float *da_l, float *da_r, void *ws,
                          size_t ws_bytes, gnn_stream_t stream) {
  if (V < 0 || heads <= 0 || F <= 0 || ldw < heads * F || ldd < heads * F)
    return GNN_ERR_INVALID_ARGUMENT;
  if (!a_l || !a_r || !da_l || !da_r) return GNN_ERR_INVALID_ARGUMENT;
  if (V > 0 && (!Wh || !del || !der || !dWh)) return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_gat_attn_proj_bwd_workspace(heads, F)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  const int64_t K = heads * F;
  float *part = static_cast<float *>(ws);
  const int nb = (int)(V < kProjBlocks ? (V > 0 ? V : 1) : kProjBlocks);
  const bool vec = F % 4 == 0 && K / 4 <= 256 && ldw % 4 == 0 && ldd % 4 == 0 && al16(Wh) &&
                   al16(dWh) && al16(a_l) && al16(a_r) && al16(part);
  if (V > 0 && vec) {
    attn_proj_bwd_vec_kernel<<<nb, 256, 0, st>>>(V, (int)heads, F, Wh, ldw, del, der, a_l, a_r,
                                                 dWh, ldd, part);
    GNN_LAUNCH_CHECK();
  } else if (V > 0) {
    const int threads = (int)(K >= 256 ? 256 : ceil_div(K, 32) * 32);
    attn_proj_bwd_kernel<<<nb, threads, 0, st>>>(V, (int)heads, F, Wh, ldw, del, der, a_l, a_r,
                                                 dWh, ldd, part);
    GNN_LAUNCH_CHECK();
  } else {
    GNN_CUDA_TRY(cudaMemsetAsync(part, 0, sizeof(float) * 2 * K, st));
  }
  attn_proj_bwd_da_final_kernel<<<(unsigned)ceil_div(2 * K, 256), 256, 0, st>>>(K, nb, part, da_l,
                                                                                da_r);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_head_mean(int64_t V, int64_t heads, int64_t F, const float *Y, int64_t ldy,
                  const float *bias, float *out, int64_t ldo, gnn_stream_t stream) {
  if (V < 0 || heads <= 0 || F <= 0 || ldy < heads * F || ldo < F) return GNN_ERR_INVALID_ARGUMENT;
  if (V == 0) return GNN_OK;
  if (!Y || !out) return GNN_ERR_INVALID_ARGUMENT;
  cudaStream_t st = as_stream(stream);
  head_mean_kernel<<<grid_1d_a(V * F, 256), 256, 0, st>>>(V, (int)heads, F, Y, ldy, bias, out, ldo);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_head_mean_bwd(int64_t V, int64_t heads, int64_t F, const float *dout, int64_t ldo,
                      float *dY, int64_t ldy, gnn_stream_t stream) {
  if (V < 0 || heads <= 0 || F <= 0 || ldy < heads * F || ldo < F) return GNN_ERR_INVALID_ARGUMENT;
  if (V == 0) return GNN_OK;
  if (!dY || !dout) return GNN_ERR_INVALID_ARGUMENT;
  cudaStream_t st = as_stream(stream);
  head_mean_bwd_kernel<<<grid_1d_a(V * heads * F, 256), 256, 0, st>>>(V, (int)heads, F, dout, ldo,
                                                                       dY, ldy);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_gat_softmax_fwd_stats(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
                              const gnn_edge_scores_t *sc, float *alpha, float *rowstat, void *ws,
                              size_t ws_bytes, gnn_stream_t stream) {
  SoftmaxArgs a;
  GNN_TRY(softmax_common(A, plan, heads, sc, ws, ws_bytes, a));
  if (!sc || sc->s || !sc->el || !sc->er || !rowstat) return GNN_ERR_INVALID_ARGUMENT;
  if (A->nnz > 0 && !alpha) return GNN_ERR_INVALID_ARGUMENT;
  if (A->nnz == 0) return GNN_OK;
  if (heads == 4 && (!al16(alpha) || !al16(sc->el))) return GNN_ERR_INVALID_ARGUMENT;
  a.alpha = alpha;
  a.mstat = rowstat;
  return dispatch_softmax<true, false>(a, as_stream(stream));
}

int gnn_gat_rowstat(int64_t V, int64_t K, const float *dYm, int64_t ldd, const float *Y,
                    int64_t ldy, const float *bias, const float *er, const float *rowstat,
                    float *stat, int64_t ldst, gnn_stream_t stream) {
  if (V < 0 || K <= 0 || K % 16 || K > 128 || ldd < K || ldy < K || ldd % 4 || ldy % 4)
    return GNN_ERR_INVALID_ARGUMENT;
  if (V == 0) return GNN_OK;
  if (!dYm || !Y || !er || !rowstat || !stat || !al16(dYm) || !al16(Y) || !al16(stat) ||
      (bias && !al16(bias)) || ldst < 16 || ldst % 4)
    return GNN_ERR_INVALID_ARGUMENT;
  cudaStream_t st = as_stream(stream);
  const int64_t q = K / 4;
  float *P = stat;
#define GNN_RS(G)                                                                          \
  gat_rowstat_kernel<G><<<(unsigned)ceil_div(ceil_div(V, 32 / G) * 32, 256), 256, 0, st>>>( \
      V, K, dYm, ldd, Y, ldy, bias, er, rowstat, P, ldst)
  if (q <= 4)
    GNN_RS(4);
  else if (q <= 8)
    GNN_RS(8);
  else if (q <= 16)
    GNN_RS(16);
  else
    GNN_RS(32);
#undef GNN_RS
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_gat_rowstat_mean(int64_t V, int64_t F1, int64_t Cp, const float *dZ, int64_t ldz,
                         const float *Yc, int64_t ldc, const float *W, int64_t ldw, float scale,
                         const float *er, const float *rowstat, float *stat, int64_t ldst,
                         gnn_stream_t stream) {
  if (V < 0 || F1 <= 0 || Cp <= 0 || Cp % 4 || Cp > 64 || ldz < Cp || ldc < 4 * F1 ||
      ldw < 4 * Cp || ldz % 4 || ldc % 4 || ldw % 4)
    return GNN_ERR_INVALID_ARGUMENT;
  if (V == 0) return GNN_OK;
  if (!dZ || !Yc || !W || !er || !rowstat || !stat || !al16(dZ) || !al16(Yc) || !al16(W) ||
      !al16(stat) || ldst < 16 || ldst % 4)
    return GNN_ERR_INVALID_ARGUMENT;
  cudaStream_t st = as_stream(stream);
  const int cp4 = (int)(Cp / 4);
  const size_t smem = sizeof(float4) * (size_t)(F1 * 4 * cp4);
  if (smem > 227 * 1024) return GNN_ERR_UNSUPPORTED;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(V, 128), (int64_t)sm_count() * 4);
  float *P = stat;
  int rc = GNN_OK;
  auto go = [&](auto kern) {
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
      rc = GNN_ERR_CUDA;
    if (rc == GNN_OK)
      kern<<<grid, 128, smem, st>>>(V, F1, Cp, dZ, ldz, Yc, ldc, W, ldw, scale, er, rowstat, P, ldst);
  };
  switch (cp4) {
    case 1: go(gat_rowstat_mean_kernel<1>); break;
    case 2: go(gat_rowstat_mean_kernel<2>); break;
    case 3: go(gat_rowstat_mean_kernel<3>); break;
    case 4: go(gat_rowstat_mean_kernel<4>); break;
    case 5: go(gat_rowstat_mean_kernel<5>); break;
    case 6: go(gat_rowstat_mean_kernel<6>); break;
    case 7: go(gat_rowstat_mean_kernel<7>); break;
    case 8: go(gat_rowstat_mean_kernel<8>); break;
    case 9: go(gat_rowstat_mean_kernel<9>); break;
    case 10: go(gat_rowstat_mean_kernel<10>); break;
    case 11: go(gat_rowstat_mean_kernel<11>); break;
    case 12: go(gat_rowstat_mean_kernel<12>); break;
    case 13: go(gat_rowstat_mean_kernel<13>); break;
    case 14: go(gat_rowstat_mean_kernel<14>); break;
    case 15: go(gat_rowstat_mean_kernel<15>); break;
    default: go(gat_rowstat_mean_kernel<16>); break;
  }
  if (rc != GNN_OK) return rc;
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

size_t gnn_gat_bwd_rc_workspace(const gnn_spmm_plan_t *plan, int64_t K) {
  if (!plan || K <= 0) return 0;
  return sizeof(float) * (size_t)(plan->num_warps * 2 * (K + 4)) + 256;
}

}  // extern "C"

namespace gnn {
namespace {
template <int G, int CPL, bool MEAN, int MINB>
int launch_gat_rcp(const GatRcArgs &a, cudaStream_t st) {
  using Sh = RcShape<G, CPL, MEAN>;
  constexpr int S = rc_stages<Sh::Q>();
  const size_t smem = 8 * (sizeof(float4) * S * kRcNB * Sh::Q + sizeof(int32_t) * S * kRcNB);
  auto kern = gat_bwd_rcp_kernel<G, CPL, MEAN, MINB>;
  if (smem > 48 * 1024)
    GNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (a.nwarps > 0) {
    kern<<<grid_warps(a.nwarps, 256), 256, smem, st>>>(a);
    GNN_LAUNCH_CHECK();
  }
  return gat_rc_tail(a, st);
}
}  // namespace
}  // namespace gnn

extern "C" {

int gnn_gat_bwd_rc(const gnn_csr_view_t *AT, const gnn_spmm_plan_t *plan, int64_t K,
                   const float *el, float slope, const float *dY, int64_t ldy, const float *Wh,
                   int64_t ldw, float *dWh, int64_t ldd, float *del, float *ds, void *ws,
                   size_t ws_bytes, gnn_stream_t stream) {
  GatRcArgs a;
  if (K <= 0 || K % 32 || K > 128) return GNN_ERR_UNSUPPORTED;
  GNN_TRY(gat_rc_common(AT, plan, el, slope, dY, ldy, Wh, ldw, dWh, ldd, del, ds, ws, ws_bytes,
                        K / 4, K, K, a));
  cudaStream_t st = as_stream(stream);
  // 16 lanes per edge (2 edges per step), 4 lanes per head, F/4 columns each
  switch (K / 32) {
    case 1: return launch_gat_rcp<16, 2, false, 2>(a, st);
    case 2: return launch_gat_rcp<16, 4, false, 2>(a, st);
    case 3: return launch_gat_rcp<16, 6, false, 2>(a, st);
    default: return launch_gat_rcp<16, 8, false, 2>(a, st);
  }
}

int gnn_gat_bwd_rc_mean(const gnn_csr_view_t *AT, const gnn_spmm_plan_t *plan, int64_t F,
                        float scale, const float *el, float slope, const float *dZ, int64_t ldz,
                        const float *Wh, int64_t ldw, float *dWh, int64_t ldd, float *del,
                        float *ds, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  GatRcArgs a;
  if (F <= 0 || F % 8 || F > 64) return GNN_ERR_UNSUPPORTED;
  GNN_TRY(gat_rc_common(AT, plan, el, slope, dZ, ldz, Wh, ldw, dWh, ldd, del, ds, ws, ws_bytes, F,
                        4 * F, F, a));
  a.scale = scale;
  cudaStream_t st = as_stream(stream);
  switch (F / 8) {
    case 1: return launch_gat_rcp<16, 2, true, 2>(a, st);
    case 2: return launch_gat_rcp<16, 4, true, 2>(a, st);
    case 3: return launch_gat_rcp<16, 6, true, 2>(a, st);
    case 4: return launch_gat_rcp<16, 8, true, 2>(a, st);
    case 5: return launch_gat_rcp<16, 10, true, 2>(a, st);
    case 6: return launch_gat_rcp<16, 12, true, 2>(a, st);
    case 7: return launch_gat_rcp<16, 14, true, 2>(a, st);
    default: return launch_gat_rcp<16, 16, true, 2>(a, st);
  }
}

int gnn_invert_permutation(int64_t n, const int32_t *perm, int32_t *inv, gnn_stream_t stream) {
  if (n < 0 || (n > 0 && (!perm || !inv))) return GNN_ERR_INVALID_ARGUMENT;
  if (n == 0) return GNN_OK;
  invert_permutation_kernel<<<grid_1d_a(n, 256), 256, 0, as_stream(stream)>>>(n, perm, inv);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

}  // extern "C"

namespace gnn {
int gemm_tc_rowdot(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *Bt,
                   int64_t ldb, const float *Y, int64_t ldy, float *S, int64_t ldS, int64_t hs,
                   void *ws, size_t ws_bytes, cudaStream_t st);
size_t gemm_tc_workspace(int64_t N, int64_t K);
namespace {
// stat[v] = {er, m, inv, scale * S} per head, S already in the w slots
__global__ void gat_rowstat_pack_kernel(int64_t V, float scale, const float *__restrict__ er,
                                        const float *__restrict__ mstat, float *__restrict__ P,
                                        int64_t ldp) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= V * 4) return;
  const int64_t v = t >> 2;
  const int h = (int)(t & 3);
  float4 *d = reinterpret_cast<float4 *>(P + v * ldp) + h;
  const float S = d->w;
  *d = make_float4(__ldg(er + v * 4 + h), __ldg(mstat + v * 8 + h), __ldg(mstat + v * 8 + 4 + h),
                   scale * S);
}
}  // namespace
}  // namespace gnn

extern "C" {

size_t gnn_gat_rowstat_mean_tc_workspace(int64_t F1, int64_t Cp) {
  if (F1 <= 0 || Cp <= 0) return 0;
  return gemm_tc_workspace(4 * F1 < 128 ? 4 * F1 : 128, Cp);
}

// gnn_gat_rowstat_mean on the tensor cores: G = dZ . W^T viewed [4*F1, Cp]
// (row 4i+h = W[i, h*Cp:(h+1)*Cp], so W must be dense: ldw == 4*Cp) in
// split-TF32, reduced against Yc in the GEMM epilogue — S[v,h] = sum_i
// Yc[v,4i+h] G[v,4i+h], the G tile never leaving the SM; then the row
// statistics are packed beside S.  UNSUPPORTED when the shapes do not fit
// the tensor-core path (the caller keeps gnn_gat_rowstat_mean).
int gnn_gat_rowstat_mean_tc(int64_t V, int64_t F1, int64_t Cp, const float *dZ, int64_t ldz,
                            const float *Yc, int64_t ldc, const float *W, int64_t ldw, float scale,
                            const float *er, const float *rowstat, float *stat, int64_t ldst,
                            void *ws, size_t ws_bytes, gnn_stream_t stream) {
  if (V < 0 || F1 <= 0 || Cp <= 0 || Cp % 4 || ldz < Cp || ldc < 4 * F1 || ldw < 4 * Cp)
    return GNN_ERR_INVALID_ARGUMENT;
  if (V == 0) return GNN_OK;
  if (!dZ || !Yc || !W || !er || !rowstat || !stat || !al16(stat) || ldst < 16 || ldst % 4)
    return GNN_ERR_INVALID_ARGUMENT;
  if (ldw != 4 * Cp) return GNN_ERR_UNSUPPORTED;
  if (ws_bytes < gnn_gat_rowstat_mean_tc_workspace(F1, Cp)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  GNN_TRY(gemm_tc_rowdot(V, 4 * F1, Cp, dZ, ldz, W, Cp, Yc, ldc, stat + 3, ldst, 4, ws, ws_bytes,
                         st));
  gat_rowstat_pack_kernel<<<(unsigned)ceil_div(V * 4, 256), 256, 0, st>>>(V, scale, er, rowstat,
                                                                          stat, ldst);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

}  // extern "C"
