// SpMMv / SpMMve (and their transposes via the CSC view) with a fused row
// epilogue (degree-norm, GIN self term, bias, ReLU, ReLU-backward mask,
// post-norm).  GraphPy semantics: PAPER.md:264-278 — no dummy |E| edge tensor
// for SpMMv, degree-norm fused in the same kernel, edge values of the
// transpose fetched through the edge-ID array (no eShuffle).
//
// Work decomposition (nnz-balanced, skew-proof):
//   * the nnz range is cut into chunks of P edges, one warp per chunk;
//   * a warp owns every non-empty row whose first edge lies in its chunk and
//     sums it over the chunk; rows that continue past the chunk end leave a
//     partial in slot[w][1]; the chunk's leading piece of a row that started
//     earlier leaves a partial in slot[w][0];
//   * within a warp, 32/G lane groups take consecutive edges of the row and
//     each lane gathers VW-wide vectors (float4 = 128-bit loads) of the
//     feature row; groups are combined with xor-shuffles;
//   * split rows (spanning >1 chunk; the power-law "mega rows") are finished
//     by one CTA per row that sums its partials in a fixed tree order, and
//     empty rows get epilogue(0) from a list — both lists come from the
//     per-graph plan, so a call never synchronises with the host.
// Summation order is fixed, so results are deterministic run to run.
#include <cuda.h>  // CUtensorMap (encode entry point fetched through the runtime)
#include <cstdlib>

#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace gnn {
namespace {

constexpr int kMaxParts = 8;  // one NVLink / NVSwitch box

struct SpmmArgs {
  int64_t R, nnz;
  const int64_t *dev_counts;  // device-count plan: [split, empty, groups, short] (else null)
  const int64_t *row_limit;   // rows >= *row_limit not computed (else null)
  const int64_t *offsets;
  const int32_t *cols;
  const float *vals;
  const int32_t *eid;
  const int64_t *deg_offsets;
  int heads;
  int64_t F;  // features per head
  const float *X;
  int64_t ldx;
  float *Y;
  int64_t ldy;
  int64_t K;
  gnn_epilogue_t epi;
  int64_t P;
  int64_t nwarps;
  const int32_t *chunk_row;    // [nwarps+1]
  const int32_t *chunk_split;  // [2*nwarps]: split index of carry-in / trailing row, or -1
  const int32_t *split_rows;
  const int32_t *split_group_base;  // [num_split+1]
  int *cnt1;                   // [num_groups] level-1 arrival counters (zeroed per call)
  int *cnt2;                   // [num_split]  level-2 arrival counters
  int64_t ncb;                 // column blocks (gridDim.y); counters are per column block
  float *l2;                   // [num_groups][K] level-2 partials
  float *slots;                // [nwarps][2][K]
  int stage;                 // StageMode
  const int32_t *row_ids;    // row-permuted operand: operand row i -> output row row_ids[i]
  int xdiv;                  // X column of output column c is c / xdiv (4: shared heads)
  float wscale;              // WM_SHARED4: scale on the edge weights
  int col_bits;              // packed weights (WM_PACKED): column id = cols[j] & col_mask,
  uint32_t col_mask;         //   edge weight = float(cols[j] >> col_bits)
  int bulk_ok;
  int warp_smem;             // bytes of shared memory per warp
  int64_t short_max;         // rows with 1 <= deg <= short_max: short-row kernel, skipped here
  // peer mode (row-partitioned multi-GPU): column id c lives in part c >> pshift
  // at row c & pmask of xt[part] — the owning rank's block, read in place over
  // NVLink through peer-mapped pointers instead of an all-gathered copy
  const float *xt[kMaxParts];
  uint32_t pshift, pmask;
};


template <int VW>
struct VecT;
template <>
struct VecT<4> {
  using T = float4;
  static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  static __device__ __forceinline__ T ld(const float *p) { return ldg_f4(p); }
  static __device__ __forceinline__ T ldc(const float *p) {
    return *reinterpret_cast<const float4 *>(p);
  }
  static __device__ __forceinline__ void st(float *p, T v) { *reinterpret_cast<float4 *>(p) = v; }
  static __device__ __forceinline__ T fma(float s, T b, T a) { return f4_fma(s, b, a); }
  static __device__ __forceinline__ T add(T a, T b) { return f4_add(a, b); }
  static __device__ __forceinline__ T shfl_xor(T v, int o) {
    return make_float4(__shfl_xor_sync(kFull, v.x, o), __shfl_xor_sync(kFull, v.y, o),
                       __shfl_xor_sync(kFull, v.z, o), __shfl_xor_sync(kFull, v.w, o));
  }
};
template <>
struct VecT<1> {
  using T = float;
  static __device__ __forceinline__ T zero() { return 0.f; }
  static __device__ __forceinline__ T ld(const float *p) { return __ldg(p); }
  static __device__ __forceinline__ T ldc(const float *p) { return *p; }
  static __device__ __forceinline__ void st(float *p, T v) { *p = v; }
  static __device__ __forceinline__ T fma(float s, T b, T a) { return fmaf(s, b, a); }
  static __device__ __forceinline__ T add(T a, T b) { return a + b; }
  static __device__ __forceinline__ T shfl_xor(T v, int o) { return __shfl_xor_sync(kFull, v, o); }
};

__device__ __forceinline__ int64_t out_row(const SpmmArgs &a, int64_t r) {
  return a.row_ids ? (int64_t)a.row_ids[r] : r;
}
__device__ __forceinline__ float inv_deg(const int64_t *off, int64_t r) {
  int64_t d = off[r + 1] - off[r];
  return d > 0 ? 1.0f / (float)d : 0.0f;
}

// Row epilogue for one scalar column.
__device__ __forceinline__ float epi_scalar(float y, int64_t r, int64_t c, const SpmmArgs &a,
                                            float norm_scale, float post_scale) {
  const gnn_epilogue_t &e = a.epi;
  if (e.flags & GNN_EPI_NORM) y *= norm_scale;
  if (e.flags & GNN_EPI_SELF) y = fmaf(e.self_scale, e.self_x[r * e.ld_self + c], y);
  if (e.flags & GNN_EPI_BIAS) y += e.bias[c];
  if (e.flags & GNN_EPI_RELU) y = fmaxf(y, 0.f);
  if (e.flags & GNN_EPI_MASK) y = e.mask[r * e.ld_mask + c] > 0.f ? y : 0.f;
  if (e.flags & GNN_EPI_POSTNORM) y *= post_scale;
  return y;
}

template <int VW>
__device__ __forceinline__ typename VecT<VW>::T epi_vec(typename VecT<VW>::T y, int64_t r,
                                                        int64_t c, const SpmmArgs &a, float ns,
                                                        float ps) {
  if constexpr (VW == 4) {
    const gnn_epilogue_t &e = a.epi;
    if (e.flags & GNN_EPI_NORM) y = make_float4(y.x * ns, y.y * ns, y.z * ns, y.w * ns);
    if (e.flags & GNN_EPI_SELF) y = f4_fma(e.self_scale, VecT<4>::ldc(e.self_x + r * e.ld_self + c), y);
    if (e.flags & GNN_EPI_BIAS) y = f4_add(y, VecT<4>::ldc(e.bias + c));
    if (e.flags & GNN_EPI_RELU)
      y = make_float4(fmaxf(y.x, 0.f), fmaxf(y.y, 0.f), fmaxf(y.z, 0.f), fmaxf(y.w, 0.f));
    if (e.flags & GNN_EPI_MASK) {
      float4 m = VecT<4>::ldc(e.mask + r * e.ld_mask + c);
      y = make_float4(m.x > 0.f ? y.x : 0.f, m.y > 0.f ? y.y : 0.f, m.z > 0.f ? y.z : 0.f,
                      m.w > 0.f ? y.w : 0.f);
    }
    if (e.flags & GNN_EPI_POSTNORM) y = make_float4(y.x * ps, y.y * ps, y.z * ps, y.w * ps);
    return y;
  } else {
    return epi_scalar(y, r, c, a, ns, ps);
  }
}

// -------------------------------------------------------------- main kernel
// Per warp: one chunk of P edges.  Lane 0 stages the chunk's column ids (and
// its edge values or edge ids) into shared memory with a 1-D bulk async copy
// (the TMA engine) while the warp reads its row bounds; the gather loop then
// only waits on the feature loads.  U edges per group are in flight per
// iteration (U*32/G per warp).
enum StageMode : int { STAGE_NONE = 0, STAGE_VALS = 1, STAGE_EID = 2, STAGE_VALS4 = 3 };
constexpr int kSub = 512;  // edges per ring sub-chunk of the nnz-split kernel
// Where an edge's weight comes from (compile-time, so the gather loop carries
// no per-edge mode test):
//   WM_NONE    implicit 1 (SpMMv)
//   WM_GLOBAL  vals[(e)*heads + head] read from global (multi-head SpMMve)
//   WM_SVALS   vals staged in the shared ring with the column ids (heads == 1)
//   WM_SEID    edge ids staged in the ring, vals[eid*heads + head] (SpMMve^T)
//   WM_PACKED  small integer weight in the high bits of the column id (the
//              coalesced multigraph operand: one 4-byte word per edge)
//   WM_SHARED4 four heads over ONE shared feature row: output column 4i+h =
//              sum_e vals[e*4+h] * X[col_e, i] (gnn_spmm_shared_heads); the
//              float4 of head weights per edge staged in the ring (STAGE_VALS4,
//              128-edge sub-chunks) so no register holds it during the gathers
//   WM_HEADS4  four heads, vals[e*4 + head] staged in the ring like WM_SHARED4's
//              (multi-head SpMMve over its own per-head columns)
enum WeightMode : int { WM_NONE = 0, WM_GLOBAL = 1, WM_SVALS = 2, WM_SEID = 3, WM_PACKED = 4,
                        WM_SHARED4 = 5, WM_HEADS4 = 6 };
template <int WM>
constexpr int stage_of() {
  return WM == WM_SVALS ? STAGE_VALS : WM == WM_SEID ? STAGE_EID : (WM == WM_SHARED4 || WM == WM_HEADS4) ? STAGE_VALS4 : STAGE_NONE;
}
// edges per ring sub-chunk
template <int WM>
constexpr int sub_of() {
  return (WM == WM_SHARED4 || WM == WM_HEADS4) ? 128 : kSub;
}

// Lane-invariant part of the gather: per-vector base pointers (column offset
// folded in; columns past K are clamped to column 0 and simply not stored).
// Column of a lane's slot v: slots interleave across the G lanes of a group
// (coalesced scalar / vector accesses), except the <G, 4, 4> shape — used only
// by the four-heads-over-one-row form (WM_SHARED4) — whose 4 slots are
// contiguous per lane, so its 4 X columns arrive in ONE 16-byte gather.
template <int G, int VPL, int VW>
__device__ __forceinline__ int slot_col(int v, int gl) {
  return (VPL == 4 && VW == 4) ? (gl * VPL + v) * VW : (v * G + gl) * VW;
}

template <int G, int VPL, int VW, bool PEER = false>
struct LaneCols {
  const char *xb[VPL];  // PEER: byte offset of the lane's column (no base)
  int head[VPL];
  __device__ __forceinline__ LaneCols(const SpmmArgs &a, int64_t cbase) {
    const int gl = (int)lane_id() % G;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      int64_t col = cbase + (int64_t)slot_col<G, VPL, VW>(v, gl);
      if (col >= a.K) col = 0;
      const int64_t xc = a.xdiv > 1 ? col / a.xdiv : col;
      xb[v] = PEER ? reinterpret_cast<const char *>(xc * 4)
                   : reinterpret_cast<const char *>(a.X + xc);
      head[v] = (int)(col / a.F);
    }
  }
};

template <int VW>
__device__ __forceinline__ typename VecT<VW>::T gather(const char *xb, int32_t c, uint32_t ldxb) {
  return VecT<VW>::ld(reinterpret_cast<const float *>(xb + (uint64_t)(uint32_t)c * ldxb));
}
// peer mode: part base from the kernel-parameter pointer table
template <int VW>
__device__ __forceinline__ typename VecT<VW>::T gather_peer(const SpmmArgs &a, const char *colb,
                                                            int32_t c, uint32_t ldxb) {
  const uint32_t cu = (uint32_t)c;
  const char *base = reinterpret_cast<const char *>(a.xt[cu >> a.pshift]);
  return VecT<VW>::ld(reinterpret_cast<const float *>(
      base + reinterpret_cast<uintptr_t>(colb) + (uint64_t)(cu & a.pmask) * ldxb));
}
template <int VW, bool PEER>
__device__ __forceinline__ typename VecT<VW>::T gather_x(const SpmmArgs &a, const char *xb,
                                                         int32_t c, uint32_t ldxb) {
  if constexpr (PEER)
    return gather_peer<VW>(a, xb, c, ldxb);
  else
    return gather<VW>(xb, c, ldxb);
}

// acc[v] += sum over this group's edges of w_e * X[c_e, cols of v] for the
// buffer-local edge range [is, ie); group g takes is+g, is+g+NG, ...  Full
// blocks of U edges per group run unpredicated; the remainder is one
// predicated block, so a piece costs a single gather latency.  The order is
// fixed by (G, U, piece bounds): deterministic.
template <int G, int VPL, int VW, int WM, bool PEER = false>
__device__ __forceinline__ void seg_accumulate(const SpmmArgs &a, const LaneCols<G, VPL, VW, PEER> &lc,
                                               const int32_t *scol, const void *sval,
                                               int64_t ebase, int is, int ie,
                                               typename VecT<VW>::T (&acc)[VPL]) {
  using V = VecT<VW>;
  constexpr bool HAS_VALS = WM != WM_NONE;
  constexpr int NG = 32 / G;
  constexpr int U = (VPL * VW >= 8) ? 4 : 8;
  const int g = (int)lane_id() / G;
  const uint32_t ldxb = (uint32_t)a.ldx * 4u;
  // packed: p -> (column, weight); otherwise the weight of ring entry i
  auto weight = [&](int i, int v, int32_t p) -> float {
    if constexpr (WM == WM_PACKED) return (float)((uint32_t)p >> a.col_bits);
    if constexpr (WM == WM_SVALS) return static_cast<const float *>(sval)[i];
    if constexpr (WM == WM_HEADS4) return static_cast<const float *>(sval)[i * 4 + lc.head[v]];
    const int64_t vi =
        WM == WM_SEID ? (int64_t) static_cast<const int32_t *>(sval)[i] : ebase + i;
    return __ldg(a.vals + vi * a.heads + lc.head[v]);
  };
  auto col = [&](int32_t p) -> int32_t {
    if constexpr (WM == WM_PACKED) return (int32_t)((uint32_t)p & a.col_mask);
    return p;
  };
  int i = is + g;
  if constexpr (WM == WM_SHARED4) {
    // every head of a lane's float4 reads the same X element: one scalar gather,
    // the 4 head weights as one float4
#ifndef GNN_SH4_U
#define GNN_SH4_U 4
#endif
    constexpr int US = GNN_SH4_U;  // edges in flight per group (weights staged: only the gathers hold registers)
    if constexpr (VPL == 4 && VW == 4) {
      // contiguous slots: one float4 gather of the lane's 4 X columns per edge,
      // 16 FMAs (4 columns x 4 heads) against the edge's float4 of head weights.
      // Full blocks of US edges per group run without per-edge predicates (the
      // predicated form spent a third of its instructions on zeroing and tests)
      for (; i + (US - 1) * NG < ie; i += NG * US) {
        float4 xv[US];
#pragma unroll
        for (int u = 0; u < US; ++u)
          xv[u] = ldg_f4(reinterpret_cast<const float *>(
              lc.xb[0] + (uint64_t)(uint32_t)scol[i + u * NG] * ldxb));
#pragma unroll
        for (int u = 0; u < US; ++u) {
          const float4 w4u = static_cast<const float4 *>(sval)[i + u * NG];
          const float xs4[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            acc[v].x = fmaf(w4u.x, xs4[v], acc[v].x);
            acc[v].y = fmaf(w4u.y, xs4[v], acc[v].y);
            acc[v].z = fmaf(w4u.z, xs4[v], acc[v].z);
            acc[v].w = fmaf(w4u.w, xs4[v], acc[v].w);
          }
        }
      }
      for (; i < ie; i += NG * US) {
        int32_t c[US];
        bool ok[US];
#pragma unroll
        for (int u = 0; u < US; ++u) {
          ok[u] = i + u * NG < ie;
          c[u] = ok[u] ? scol[i + u * NG] : 0;
        }
        float4 xv[US];
#pragma unroll
        for (int u = 0; u < US; ++u)
          xv[u] = ok[u] ? ldg_f4(reinterpret_cast<const float *>(lc.xb[0] + (uint64_t)(uint32_t)c[u] * ldxb))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < US; ++u) {
          // the edge's head weights from the staged ring (broadcast within the group)
          const float4 w4u = ok[u] ? static_cast<const float4 *>(sval)[i + u * NG]
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
          const float xs4[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            acc[v].x = fmaf(w4u.x, xs4[v], acc[v].x);
            acc[v].y = fmaf(w4u.y, xs4[v], acc[v].y);
            acc[v].z = fmaf(w4u.z, xs4[v], acc[v].z);
            acc[v].w = fmaf(w4u.w, xs4[v], acc[v].w);
          }
        }
      }
      return;
    }
    for (; i < ie; i += NG * US) {
      int32_t c[US];
      bool ok[US];
#pragma unroll
      for (int u = 0; u < US; ++u) {
        ok[u] = i + u * NG < ie;
        c[u] = ok[u] ? scol[i + u * NG] : 0;
      }
      float xs[US][VPL];
#pragma unroll
      for (int u = 0; u < US; ++u)
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          xs[u][v] = ok[u] ? __ldg(reinterpret_cast<const float *>(lc.xb[v] + (uint64_t)(uint32_t)c[u] * ldxb))
                           : 0.f;
      float4 w4[US];  // (the scale is applied once at the row's final store)
#pragma unroll
      for (int u = 0; u < US; ++u)
        w4[u] = ok[u] ? static_cast<const float4 *>(sval)[i + u * NG] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < US; ++u)
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          if constexpr (VW == 4) {
            acc[v].x = fmaf(w4[u].x, xs[u][v], acc[v].x);
            acc[v].y = fmaf(w4[u].y, xs[u][v], acc[v].y);
            acc[v].z = fmaf(w4[u].z, xs[u][v], acc[v].z);
            acc[v].w = fmaf(w4[u].w, xs[u][v], acc[v].w);
          }
        }
    }
    return;
  }
  for (; i + (U - 1) * NG < ie; i += NG * U) {
    int32_t p[U];
#pragma unroll
    for (int u = 0; u < U; ++u) p[u] = scol[i + u * NG];
    typename V::T x[U][VPL];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v < VPL; ++v) x[u][v] = gather_x<VW, PEER>(a, lc.xb[v], col(p[u]), ldxb);
    if constexpr (HAS_VALS) {
      float w[U][VPL];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < VPL; ++v) w[u][v] = weight(i + u * NG, v, p[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < VPL; ++v) acc[v] = V::fma(w[u][v], x[u][v], acc[v]);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < VPL; ++v) acc[v] = V::add(acc[v], x[u][v]);
    }
  }
  if (i < ie) {  // one predicated block: < U edges left for this group
    int32_t p[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ok[u] = i + u * NG < ie;
      p[u] = ok[u] ? scol[i + u * NG] : 0;
    }
    typename V::T x[U][VPL];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        x[u][v] = ok[u] ? gather_x<VW, PEER>(a, lc.xb[v], col(p[u]), ldxb) : V::zero();
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        if constexpr (HAS_VALS)
          acc[v] = V::fma(ok[u] ? weight(i + u * NG, v, p[u]) : 0.f, x[u][v], acc[v]);
        else
          acc[v] = V::add(acc[v], x[u][v]);
      }
  }
}

template <int G, int VPL, int VW>
__device__ __forceinline__ void group_reduce(typename VecT<VW>::T (&acc)[VPL]) {
  using V = VecT<VW>;
#pragma unroll
  for (int o = G; o < 32; o <<= 1)
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = V::add(acc[v], V::shfl_xor(acc[v], o));
}

template <int G, int VPL, int VW>
__device__ __forceinline__ void store_row(const SpmmArgs &a, float *dst, int64_t cbase,
                                          const typename VecT<VW>::T (&acc)[VPL], bool final_row,
                                          int64_t r) {
  using V = VecT<VW>;
  const int lane = (int)lane_id();
  const int g = lane / G, gl = lane % G;
  if (g != 0) return;
  float ns = 1.f, ps = 1.f;
  if (final_row) {
    if (a.epi.flags & GNN_EPI_NORM) ns = inv_deg(a.deg_offsets, r);
    if (a.epi.flags & GNN_EPI_POSTNORM) ps = inv_deg(a.epi.post_deg_offsets, r);
  }
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    int64_t col = cbase + (int64_t)slot_col<G, VPL, VW>(v, gl);
    if (col < a.K) {
      typename V::T y = acc[v];
      if (final_row) {
        if constexpr (VW == 4) {
          const float w = a.wscale;  // shared-heads scale, applied once per row
          y = make_float4(y.x * w, y.y * w, y.z * w, y.w * w);
        } else {
          y *= a.wscale;
        }
        y = epi_vec<VW>(y, r, col, a, ns, ps);
      }
      V::st(dst + col, y);
    }
  }
}

__device__ __forceinline__ int64_t shfl_i64(int64_t v, int src) {
  int lo = __shfl_sync(kFull, (int)(v & 0xffffffff), src);
  int hi = __shfl_sync(kFull, (int)(v >> 32), src);
  return ((int64_t)hi << 32) | (uint32_t)lo;
}

// ---------------------------------------------------------- split rows
// Partial j of split row s (spanning warps wa..wb, np = wb-wa+1): j==0 ->
// slot[wa][1], j>=1 -> slot[wa+j][0].  Partials are grouped by 64; the last
// warp to arrive at a group (fence + counter) sums the group in fixed order,
// and the last group to finish sums the group sums in fixed order and applies
// the epilogue.  Which warp arrives last varies, the summation order does not:
// results are deterministic.
constexpr int kGroupPartials = 64;

__device__ __forceinline__ const float *partial_ptr(const SpmmArgs &a, int64_t wa, int64_t j) {
  return a.slots + ((wa + j) * 2 + (j == 0 ? 1 : 0)) * a.K;
}

// Arrival: release-ordered atomic (MEMBAR.ALL.GPU + ATOMG, no L1 invalidate —
// a gpu-scope acquire/sc fence would flush the SM's L1 and with it the
// feature rows the other warps are reusing).  The last arriver reads the
// partials with strong relaxed loads served by L2, the point of coherence,
// issued under a control dependency on the atomic's result.
__device__ __forceinline__ int atom_add_release_gpu(int *p, int v) {
  int old;
  asm volatile("atom.release.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ float ld_relaxed_gpu(const float *p) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}

// Called by a whole warp right after it stored partial j of split row s for
// the column block [cbase, cbase+kb).
__device__ __forceinline__ void split_arrive(const SpmmArgs &a, int64_t s, int64_t j, int64_t cbase,
                                          int kb) {
  const int lane = (int)lane_id();
  const int64_t r = a.split_rows[s];
  const int64_t rs = a.offsets[r], re = a.offsets[r + 1];
  const int64_t orow = out_row(a, r);
  const int64_t wa = rs / a.P, wb = (re - 1) / a.P;
  const int64_t np = wb - wa + 1;
  const int64_t gi = j / kGroupPartials;
  const int64_t ng = ceil_div(np, kGroupPartials);
  const int64_t gbase = a.split_group_base[s];
  const int64_t rem = np - gi * kGroupPartials;
  const int m = (int)(rem < kGroupPartials ? rem : kGroupPartials);
  const int64_t cend = min(cbase + (int64_t)kb, a.K);
  __syncwarp();  // the partial's lanes happen-before lane 0's release
  int old = 0;
  if (lane == 0) old = atom_add_release_gpu(&a.cnt1[(gbase + gi) * a.ncb + blockIdx.y], 1);
  old = __shfl_sync(kFull, old, 0);
  if (old != m - 1) return;
  const float ns = (a.epi.flags & GNN_EPI_NORM) ? inv_deg(a.deg_offsets, orow) : 1.f;
  const float ps = (a.epi.flags & GNN_EPI_POSTNORM) ? inv_deg(a.epi.post_deg_offsets, orow) : 1.f;
  const int64_t j0 = gi * kGroupPartials;
  for (int64_t c = cbase + lane; c < cend; c += 32) {
    float t = 0.f;
#pragma unroll 8
    for (int k = 0; k < m; ++k) t += ld_relaxed_gpu(partial_ptr(a, wa, j0 + k) + c);
    if (ng == 1)
      a.Y[orow * a.ldy + c] = epi_scalar(t * a.wscale, orow, c, a, ns, ps);
    else
      a.l2[(gbase + gi) * a.K + c] = t;
  }
  if (ng == 1) return;
  __syncwarp();
  if (lane == 0) old = atom_add_release_gpu(&a.cnt2[s * a.ncb + blockIdx.y], 1);
  old = __shfl_sync(kFull, old, 0);
  if (old != (int)ng - 1) return;
  for (int64_t c = cbase + lane; c < cend; c += 32) {
    float t = 0.f;
#pragma unroll 8
    for (int64_t g2 = 0; g2 < ng; ++g2) t += ld_relaxed_gpu(a.l2 + (gbase + g2) * a.K + c);
    a.Y[orow * a.ldy + c] = epi_scalar(t * a.wscale, orow, c, a, ns, ps);
  }
}

// ------------------------------------------------------------- main kernel
// Persistent streaming: warp w owns the contiguous edge range [w*P, (w+1)*P)
// (P ~ nnz / resident warps) and streams it through a two-stage shared-memory
// ring of kSub-edge sub-chunks filled by 1-D bulk async copies (the TMA
// engine): column ids (+ edge values or edge ids).  Row accumulators carry
// across sub-chunk boundaries in registers; only rows crossing the warp's
// range boundaries produce partials (split rows, finished by split_arrive).

template <int G, int VPL, int VW, int WM, bool PEER = false>
#ifndef GNN_SPMM_MINB
#define GNN_SPMM_MINB 4  // resident CTAs per SM for column blocks <= 16 wide (64 regs); wider: 3
#endif
#ifndef GNN_SPMM_MINB_KB
#define GNN_SPMM_MINB_KB 32  // widest column block that runs at GNN_SPMM_MINB CTAs per SM
#endif
__global__ void __launch_bounds__(256, (G * VPL * VW <= GNN_SPMM_MINB_KB) ? GNN_SPMM_MINB : 3) spmm_main_kernel(SpmmArgs a) {
  using V = VecT<VW>;
  constexpr int KB = G * VPL * VW;
  extern __shared__ __align__(16) uint8_t spmm_smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = (int)lane_id();
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= a.nwarps) return;
  constexpr int stage = stage_of<WM>();
  constexpr int SUB = sub_of<WM>();
  constexpr int VW4 = stage == STAGE_VALS4 ? 4 : 1;              // ring words per edge value
  uint8_t *wbase = spmm_smem + (size_t)warp * a.warp_smem;
  uint64_t *bar = reinterpret_cast<uint64_t *>(wbase);           // [2]
  int32_t *scol = reinterpret_cast<int32_t *>(wbase + 16);       // [2][SUB]
  int32_t *sval = scol + 2 * SUB;                                // [2][SUB * VW4] (vals or eid bits)
  const int64_t cbase = (int64_t)blockIdx.y * KB;
  const int64_t e0 = w * a.P;
  const int64_t e1 = min(e0 + a.P, a.nnz);
  const int nsub = (int)ceil_div(e1 - e0, SUB);

  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int sc) {
    const int b = sc & 1;
    const int64_t s0 = e0 + (int64_t)sc * SUB;
    const int n = (int)min((int64_t)SUB, e1 - s0);
    const int nbulk = a.bulk_ok ? (n & ~3) : 0;
    int32_t *dc = scol + b * SUB;
    int32_t *dv = sval + b * SUB * VW4;
    for (int i = nbulk + lane; i < n; i += 32) {
      dc[i] = a.cols[s0 + i];
      if (stage == STAGE_VALS) dv[i] = __float_as_int(a.vals[s0 + i]);
      if (stage == STAGE_EID) dv[i] = a.eid[s0 + i];
      if (stage == STAGE_VALS4)
        reinterpret_cast<float4 *>(dv)[i] = ldg_f4(a.vals + (s0 + i) * 4);
    }
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)nbulk * 4u;
      mbar_arrive_expect_tx(bar + b, stage != STAGE_NONE ? (1u + VW4) * bytes : bytes);
      if (bytes) {
        bulk_g2s(dc, a.cols + s0, bytes, bar + b);
        if (stage == STAGE_VALS) bulk_g2s(dv, a.vals + s0, bytes, bar + b);
        if (stage == STAGE_EID) bulk_g2s(dv, a.eid + s0, bytes, bar + b);
        if (stage == STAGE_VALS4) bulk_g2s(dv, a.vals + s0 * 4, 4u * bytes, bar + b);
      }
    }
  };
  // a warp whose first row is past the live rows has nothing to do (checked
  // before any bulk copy is in flight)
  const int64_t r_first = a.chunk_row[w];
  const int64_t rlim = a.row_limit ? min(a.R, *a.row_limit) : a.R;
  if (r_first >= rlim) return;
  issue(0);

  // row bounds: 32 row ends per batched load
  int64_t r = r_first;
  int64_t rs = a.offsets[r];
  int64_t obuf = a.offsets[min(r + 1 + lane, a.R)];
  int bi = 0;
  int64_t re = shfl_i64(obuf, 0);
  const LaneCols<G, VPL, VW, PEER> lc(a, cbase);
  typename V::T acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = V::zero();
  bool done = false;

  int last_issued = 0, last_waited = -1;
  for (int sc = 0; sc < nsub && !done; ++sc) {
    const int b = sc & 1;
    const int64_t s0 = e0 + (int64_t)sc * SUB;
    const int64_t s1 = min(s0 + SUB, e1);
    if (sc + 1 < nsub) {
      issue(sc + 1);
      last_issued = sc + 1;
    }
    mbar_wait(bar + b, (uint32_t)((sc >> 1) & 1));
    last_waited = sc;
    __syncwarp();
    const int32_t *bc = scol + b * SUB;
    const int32_t *bv = sval + b * SUB * VW4;
    while (true) {
      const int64_t lo = max(rs, s0), hi = min(re, s1);
      const bool is_short = re - rs <= a.short_max;  // owned by the short-row kernel
      if (hi > lo && !is_short)
        seg_accumulate<G, VPL, VW, WM, PEER>(a, lc, bc, bv, s0, (int)(lo - s0),
                                             (int)(hi - s0), acc);
      if (re > s1) break;  // row continues in the next sub-chunk (or the next warp)
      if (re > rs && !is_short) {  // a row ends here
        group_reduce<G, VPL, VW>(acc);
        if (rs < e0) {     // carry-in piece of a row owned by an earlier warp
          store_row<G, VPL, VW>(a, a.slots + (w * 2 + 0) * a.K, cbase, acc, false, r);
          split_arrive(a, a.chunk_split[2 * w], w - rs / a.P, cbase, KB);
        } else {
          const int64_t orow = out_row(a, r);
          store_row<G, VPL, VW>(a, a.Y + orow * a.ldy, cbase, acc, true, orow);
        }
#pragma unroll
        for (int v = 0; v < VPL; ++v) acc[v] = V::zero();
      }
      ++r;
      rs = re;
      if (rs >= e1 || r >= rlim) {
        done = true;
        break;
      }
      if (++bi == 32) {
        obuf = a.offsets[min(r + 1 + lane, a.R)];
        bi = 0;
        // a whole window of empty rows (their epilogue is the plan's empty-row
        // pass): jump to the next non-empty row by binary search instead of
        // walking them one by one (a replayed mini-batch's capacity buffers
        // hold ~1e5 trailing empty rows)
        if (__all_sync(kFull, obuf == rs) && r + 32 < a.R) {
          int64_t lo = r + 32, hi = a.R;  // first row q >= lo with offsets[q + 1] > rs
          while (lo < hi) {
            const int64_t mid = lo + ((hi - lo) >> 1);
            if (a.offsets[mid + 1] > rs)
              hi = mid;
            else
              lo = mid + 1;
          }
          r = lo;
          if (r >= rlim) {
            done = true;
            break;
          }
          obuf = a.offsets[min(r + 1 + lane, a.R)];
        }
      }
      re = shfl_i64(obuf, bi);
    }
    __syncwarp();  // buffer b fully consumed before issue(sc + 2) refills it
  }
  // the loop can stop early (live-row limit): a prefetched sub-chunk's bulk copy
  // must land before the warp (and perhaps its CTA) exits
  if (last_issued > last_waited)
    mbar_wait(bar + (last_issued & 1), (uint32_t)((last_issued >> 1) & 1));
  if (!done && re > e1 && re - rs > a.short_max) {  // the range ends inside row r
    group_reduce<G, VPL, VW>(acc);
    if (rs < e0) {         // whole range inside one row: a carry-in piece
      store_row<G, VPL, VW>(a, a.slots + (w * 2 + 0) * a.K, cbase, acc, false, r);
      split_arrive(a, a.chunk_split[2 * w], w - rs / a.P, cbase, KB);
    } else {               // trailing piece of a row this warp owns
      store_row<G, VPL, VW>(a, a.slots + (w * 2 + 1) * a.K, cbase, acc, false, r);
      split_arrive(a, a.chunk_split[2 * w + 1], 0, cbase, KB);
    }
  }
}

// ------------------------------------------------------ TMA gather kernel
// Blackwell-native SpMM: the feature rows X[col_e, cbase:cbase+KB] of every
// edge are fetched by the TMA engine with cp.async.bulk.tensor.2d
// .tile::gather4 (4 indexed rows per instruction) into a per-warp 3-stage
// shared-memory ring, so no gather latency sits on a register dependency
// chain.  Each warp owns a contiguous edge range (persistent, 8 warps/SM,
// one CTA per SM); S = 8 KB/(4*KB) edges per stage; the S/4 issuing lanes
// prefetch their 4 column ids (and edge values) one stage ahead.  The
// consumers sum rows from shared memory with 128-bit LDS; row accumulators
// carry across stages; range-boundary rows go through split_arrive.  Every
// issued stage is consumed before the warp exits (a warp only finishes early
// inside its last stage), so no TMA write can outlive the CTA.
constexpr int kTmaStageBytes = 8192;
constexpr int kTmaStages = 3;

__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap *tm, int c0, int4 rows,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(tm), "r"(c0), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w), "r"(bar)
      : "memory");
}

template <int KB>
constexpr int tma_warp_bytes() {
  return (kTmaStages * kTmaStageBytes + kTmaStages * (kTmaStageBytes / (KB * 4)) * 4 + 64 + 1023) /
         1024 * 1024;
}

template <int KB, bool HAS_VALS>
__global__ void __launch_bounds__(256, 1) spmm_tma_kernel(const __grid_constant__ CUtensorMap tmX,
                                                          SpmmArgs a) {
  constexpr int G = KB >= 128 ? 32 : KB / 4;   // lanes per row
  constexpr int VPL = KB == 256 ? 2 : 1;       // float4 per lane
  constexpr int NG = 32 / G;
  constexpr int S = kTmaStageBytes / (KB * 4); // edges per stage
  constexpr int NI = S / 4;                    // issuing lanes (one gather4 each)
  constexpr int U = (S / NG) >= 8 ? 8 : (S / NG);
  using V = VecT<4>;
  extern __shared__ __align__(1024) uint8_t tma_smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = (int)lane_id();
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= a.nwarps) return;
  constexpr int kWarpBytes = tma_warp_bytes<KB>();  // 1 KB aligned: TMA smem destinations
  uint8_t *wb = tma_smem + (size_t)warp * kWarpBytes;
  float *sdata = reinterpret_cast<float *>(wb);                                // [3][S][KB]
  float *svals = reinterpret_cast<float *>(wb + kTmaStages * kTmaStageBytes);  // [3][S]
  uint64_t *bar =
      reinterpret_cast<uint64_t *>(wb + kTmaStages * kTmaStageBytes + kTmaStages * S * 4);
  const int64_t cbase = (int64_t)blockIdx.y * KB;
  const int64_t e0 = w * a.P;
  const int64_t e1 = min(e0 + a.P, a.nnz);
  const int nsub = (int)ceil_div(e1 - e0, S);

  if (lane == 0) {
    for (int i = 0; i < kTmaStages; ++i) mbar_init(bar + i, 1);
    fence_mbar_init();
  }
  __syncwarp();

  // lane l < NI owns edges [4l, 4l+4) of every stage
  auto load_idx = [&](int sc, int4 &rows, float4 &vv) {
    rows = make_int4(0, 0, 0, 0);
    vv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (sc >= nsub || lane >= NI) return;
    const int64_t e = e0 + (int64_t)sc * S + 4 * lane;
    if (e + 4 <= e1) {
      rows = __ldg(reinterpret_cast<const int4 *>(a.cols + e));
      if (HAS_VALS) vv = __ldg(reinterpret_cast<const float4 *>(a.vals + e));
    } else if (e < e1) {
      int t[4] = {0, 0, 0, 0};
      float f[4] = {0.f, 0.f, 0.f, 0.f};
      for (int k = 0; k < 4; ++k)
        if (e + k < e1) {
          t[k] = a.cols[e + k];
          if (HAS_VALS) f[k] = a.vals[e + k];
        }
      rows = make_int4(t[0], t[1], t[2], t[3]);
      vv = make_float4(f[0], f[1], f[2], f[3]);
    }
  };
  auto issue = [&](int sc, int4 rows, float4 vv) {
    if (sc >= nsub) return;
    const int st = sc % kTmaStages;
    const int n = (int)min((int64_t)S, e1 - (e0 + (int64_t)sc * S));
    const int ng4 = (n + 3) >> 2;
    if (lane == 0) mbar_arrive_expect_tx(bar + st, (uint32_t)(ng4 * 4 * KB * 4));
    __syncwarp();
    if (lane < ng4) {
      if (HAS_VALS) *reinterpret_cast<float4 *>(svals + st * S + 4 * lane) = vv;
      tma_gather4(smem_u32(sdata + (size_t)st * S * KB + 4 * lane * KB), &tmX, (int)cbase, rows,
                  smem_u32(bar + st));
    }
  };

  int4 ri;
  float4 vi;
  load_idx(0, ri, vi);
  issue(0, ri, vi);
  load_idx(1, ri, vi);
  issue(1, ri, vi);
  load_idx(2, ri, vi);

  int64_t r = a.chunk_row[w];
  int64_t rs = a.offsets[r];
  int64_t obuf = a.offsets[min(r + 1 + lane, a.R)];
  int bi = 0;
  int64_t re = shfl_i64(obuf, 0);
  const int g = lane / G, gl = lane % G;
  typename V::T acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = V::zero();
  bool done = false;

  for (int sc = 0; sc < nsub && !done; ++sc) {
    issue(sc + 2, ri, vi);  // stage (sc+2)%3 was consumed in iteration sc-1
    load_idx(sc + 3, ri, vi);
    const int st = sc % kTmaStages;
    const int64_t s0 = e0 + (int64_t)sc * S;
    const int64_t s1 = min(s0 + S, e1);
    mbar_wait(bar + st, (uint32_t)((sc / kTmaStages) & 1));
    const float *bd = sdata + (size_t)st * S * KB + gl * 4;
    const float *bv = svals + st * S;
    while (true) {
      const int lo = (int)(max(rs, s0) - s0), hi = (int)(min(re, s1) - s0);
      int i = lo + g;  // group g takes lo+g, lo+g+NG, ...
      for (; i + (U - 1) * NG < hi; i += NG * U) {
        float4 x[U][VPL];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            x[u][v] = *reinterpret_cast<const float4 *>(bd + (i + u * NG) * KB + v * 128);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            if constexpr (HAS_VALS)
              acc[v] = V::fma(bv[i + u * NG], x[u][v], acc[v]);
            else
              acc[v] = V::add(acc[v], x[u][v]);
          }
      }
      for (; i < hi; i += NG) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          float4 x = *reinterpret_cast<const float4 *>(bd + i * KB + v * 128);
          if constexpr (HAS_VALS)
            acc[v] = V::fma(bv[i], x, acc[v]);
          else
            acc[v] = V::add(acc[v], x);
        }
      }
      if (re > s1) break;
      if (re > rs) {
        group_reduce<G, VPL, 4>(acc);
        if (rs < e0) {
          store_row<G, VPL, 4>(a, a.slots + (w * 2 + 0) * a.K, cbase, acc, false, r);
          split_arrive(a, a.chunk_split[2 * w], w - rs / a.P, cbase, KB);
        } else {
          store_row<G, VPL, 4>(a, a.Y + r * a.ldy, cbase, acc, true, r);
        }
#pragma unroll
        for (int v = 0; v < VPL; ++v) acc[v] = V::zero();
      }
      ++r;
      rs = re;
      if (rs >= e1 || r >= a.R) {
        done = true;
        break;
      }
      if (++bi == 32) {
        obuf = a.offsets[min(r + 1 + lane, a.R)];
        bi = 0;
      }
      re = shfl_i64(obuf, bi);
    }
    __syncwarp();  // stage st consumed before issue() refills it
  }
  if (!done && re > e1) {
    group_reduce<G, VPL, 4>(acc);
    if (rs < e0) {
      store_row<G, VPL, 4>(a, a.slots + (w * 2 + 0) * a.K, cbase, acc, false, r);
      split_arrive(a, a.chunk_split[2 * w], w - rs / a.P, cbase, KB);
    } else {
      store_row<G, VPL, 4>(a, a.slots + (w * 2 + 1) * a.K, cbase, acc, false, r);
      split_arrive(a, a.chunk_split[2 * w + 1], 0, cbase, KB);
    }
  }
}

typedef CUresult (*TensorMapEncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                      const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                      const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

TensorMapEncodeFn get_encode_fn() {
  static TensorMapEncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<TensorMapEncodeFn>(p);
  }
  return fn;
}

// Row-gather tensor map over X[rows, K] (row stride ldx floats), box {KB, 1}.
bool make_gather_map(CUtensorMap *tm, const float *X, int64_t rows, int64_t K, int64_t ldx, int KB) {
  TensorMapEncodeFn enc = get_encode_fn();
  if (!enc || rows <= 0) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ldx * 4};
  cuuint32_t box[2] = {(cuuint32_t)KB, 1};
  cuuint32_t es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(X), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int KB>
int launch_tma(const SpmmArgs &a, bool has_vals, const CUtensorMap &tm, cudaStream_t st) {
  constexpr int S = kTmaStageBytes / (KB * 4);
  const size_t smem = (size_t)8 * tma_warp_bytes<KB>();
  (void)S;
  dim3 grid((unsigned)ceil_div(a.nwarps * 32, 256), (unsigned)ceil_div(a.K, KB));
  auto kern = has_vals ? spmm_tma_kernel<KB, true> : spmm_tma_kernel<KB, false>;
  GNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, 256, smem, st>>>(tm, a);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

// Short rows (1 <= deg <= short_max; the power-law tail): one lane group per
// row instead of a whole warp walking rows one by one — NG rows per warp in
// parallel, U edges of each in flight, fused epilogue per group.  The group's
// lanes load its column ids cooperatively (consecutive words, then a shuffle
// broadcast: one L1 request per G ids instead of G), in 32-bit row-relative
// arithmetic; the loop runs to the warp's longest row (the list is longest
// first, so neighbours are near-equal) so every shuffle is warp-converged.
// Summation order is fixed per row: deterministic.
template <int G, int VPL, int VW, int WM, bool PEER = false>
__global__ void __launch_bounds__(256, 4) spmm_short_rows_kernel(SpmmArgs a, const int32_t *__restrict__ rows,
                                                                 int64_t nrows) {
  using V = VecT<VW>;
  constexpr int NG = 32 / G;
  constexpr int U = (VPL * VW >= 8) ? 4 : 8;
  constexpr int KL = (U + G - 1) / G;  // ids each lane loads per block
  constexpr int KB = G * VPL * VW;
  const int lane = (int)lane_id();
  const int g = lane / G, gl = lane % G;
  const int gbase = lane & ~(G - 1);
  const int64_t cbase = (int64_t)blockIdx.y * KB;
  const int64_t i = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * NG + g;
  if (a.dev_counts) nrows = min(nrows, a.dev_counts[3]);
  bool valid = i < nrows;
  const int64_t r = valid ? rows[i] : 0;
  if (a.row_limit && r >= *a.row_limit) valid = false;
  const int64_t rs = valid ? a.offsets[r] : 0;
  const int n = valid ? (int)(a.offsets[r + 1] - rs) : 0;  // deg <= short_max
  int nmax = n;
#pragma unroll
  for (int o = 16; o >= G; o >>= 1) nmax = max(nmax, __shfl_xor_sync(kFull, nmax, o));
  const int32_t *cp = a.cols + rs;
  const LaneCols<G, VPL, VW, PEER> lc(a, cbase);
  const uint32_t ldxb = (uint32_t)a.ldx * 4u;
  const int cbits = a.col_bits;
  const uint32_t cmask = a.col_mask;
  typename V::T acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = V::zero();
  // one block of U edges per group; FULL (every group of the warp has U edges
  // left — the common case, rows being sorted longest first) runs without the
  // per-edge predicates, whose address / constant rematerialisation doubled
  // the instruction count of this (issue-bound at K >= 32) loop
  auto block = [&](int e, auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
    int32_t mine[KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) {
      const int j = gl + k * G;
      mine[k] = (j < U && (FULL || e + j < n)) ? __ldg(cp + e + j) : 0;
    }
    int32_t c[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ok[u] = FULL || e + u < n;
      c[u] = __shfl_sync(kFull, mine[u / G], gbase + u % G);
    }
    float pw[U];  // packed weights
    if constexpr (WM == WM_PACKED) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        pw[u] = (float)((uint32_t)c[u] >> cbits);
        c[u] = (int32_t)((uint32_t)c[u] & cmask);
      }
    }
    typename V::T x[U][VPL];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v < VPL; ++v) x[u][v] = ok[u] ? gather_x<VW, PEER>(a, lc.xb[v], c[u], ldxb) : V::zero();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (WM != WM_NONE) {
        float w[VPL];
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          if constexpr (WM == WM_PACKED) {
            w[v] = pw[u];  // 0 for the padding entries (c = 0)
          } else {
            const int64_t vi = ok[u] ? (WM == WM_SEID ? (int64_t)__ldg(a.eid + rs + e + u) : rs + e + u) : 0;
            w[v] = ok[u] ? __ldg(a.vals + vi * a.heads + lc.head[v]) : 0.f;
          }
        }
#pragma unroll
        for (int v = 0; v < VPL; ++v) acc[v] = V::fma(w[v], x[u][v], acc[v]);
      } else {
#pragma unroll
        for (int v = 0; v < VPL; ++v) acc[v] = V::add(acc[v], x[u][v]);
      }
    }
  };
  // (column blocks >= 32 wide only: at 16 the loop is L1-bound, not issue-bound,
  // and the extra vote cost ~1% on the papers100M shape)
  for (int e = 0; e < nmax; e += U) {
    if (KB >= 32 && __all_sync(kFull, e + U <= n))
      block(e, std::integral_constant<bool, true>());
    else
      block(e, std::integral_constant<bool, false>());
  }
  if (!valid) return;
  const int64_t orow = out_row(a, r);
  float ns = 1.f, ps = 1.f;
  if (a.epi.flags & GNN_EPI_NORM) ns = inv_deg(a.deg_offsets, orow);
  if (a.epi.flags & GNN_EPI_POSTNORM) ps = inv_deg(a.epi.post_deg_offsets, orow);
  float *dst = a.Y + orow * a.ldy;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int64_t col = cbase + (int64_t)(v * G + gl) * VW;
    if (col < a.K) V::st(dst + col, epi_vec<VW>(acc[v], orow, col, a, ns, ps));
  }
}

__global__ void spmm_empty_rows_kernel(SpmmArgs a, const int32_t *__restrict__ rows,
                                       int64_t nrows) {
  // device-count plans count only the empty rows below the live-row limit
  // (plan_counts_kernel), the list being ascending
  if (a.dev_counts) nrows = min(nrows, a.dev_counts[1]);
  const int64_t total = nrows * a.K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / a.K, c = t % a.K;
    int64_t r = out_row(a, rows[i]);
    float ps = (a.epi.flags & GNN_EPI_POSTNORM) ? inv_deg(a.epi.post_deg_offsets, r) : 1.f;
    a.Y[r * a.ldy + c] = epi_scalar(0.f, r, c, a, 0.f, ps);
  }
}

// ------------------------------------------------------------- planning
__global__ void plan_chunk_rows_kernel(const int64_t *__restrict__ off, int64_t R, int64_t nnz,
                                       int64_t P, int64_t nw, int32_t *chunk_row) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w <= nw;
       w += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = w * P;
    chunk_row[w] = (w == nw || e >= nnz) ? (int32_t)R
                                         : (int32_t)(upper_bound_dev(off, 0, R + 1, e) - 1);
  }
}
// Do the rows of degree > short_max form a prefix (a degree-sorted operand)?
// info[0] |= 1 on a long row after a non-long one; info[1] = long-row count.
__global__ void plan_long_prefix_kernel(const int64_t *__restrict__ off, int64_t R,
                                        int64_t short_max, unsigned long long *info) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const bool lg = off[r + 1] - off[r] > short_max;
    if (lg) atomicAdd(info + 1, 1ull);
    if (lg && r > 0 && off[r] - off[r - 1] <= short_max) atomicOr(info, 1ull);
  }
}
// Per-row plan flags, two counters per 64-bit word so one exclusive scan
// advances both (each count < 2^31, so the low field never carries):
//   fa = split-row flag | empty-row flag << 32
//   fb = groups of the split row | short-row flag << 32
__device__ __forceinline__ int64_t lo32(int64_t v) { return v & 0xffffffffll; }
__device__ __forceinline__ int64_t hi32(int64_t v) { return v >> 32; }
__global__ void plan_flags_kernel(const int64_t *__restrict__ off, int64_t R, int64_t P,
                                  int64_t short_max, int64_t main_nnz, int64_t *fa, int64_t *fb) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t rs = off[r], re = off[r + 1];
    const int64_t empty = re == rs ? 1 : 0;
    const int64_t shrt = (re > rs && re - rs <= short_max) ? 1 : 0;
    // split-row bookkeeping covers short rows too (inside the nnz-split range):
    // a call that does not use the short-row kernel (wide K) finishes them here
    const bool split = re > rs && re <= main_nnz && rs / P != (re - 1) / P;
    const int64_t groups = split ? ceil_div((re - 1) / P - rs / P + 1, kGroupPartials) : 0;
    fa[r] = (split ? 1 : 0) | (empty << 32);
    fb[r] = groups | (shrt << 32);
  }
}
__global__ void plan_scatter_kernel(const int64_t *__restrict__ off, int64_t R, int64_t P,
                                    const int64_t *__restrict__ fa, const int64_t *__restrict__ fb,
                                    int32_t *split_rows, int32_t *split_group_base,
                                    int32_t *chunk_split, int32_t *empty_rows, int32_t *short_rows) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a0 = fa[r], a1 = fa[r + 1], b0 = fb[r], b1 = fb[r + 1];
    if (lo32(a1) != lo32(a0)) {
      const int64_t si = lo32(a0);
      split_rows[si] = (int32_t)r;
      split_group_base[si] = (int32_t)lo32(b0);
      const int64_t wa = off[r] / P, wb = (off[r + 1] - 1) / P;
      chunk_split[2 * wa + 1] = (int32_t)si;  // trailing partial of the owner chunk
      for (int64_t w = wa + 1; w <= wb; ++w) chunk_split[2 * w] = (int32_t)si;  // carry-ins
    }
    if (hi32(a1) != hi32(a0)) empty_rows[hi32(a0)] = (int32_t)r;
    if (hi32(b1) != hi32(b0)) short_rows[hi32(b0)] = (int32_t)r;
    if (r == 0) split_group_base[lo32(fa[R])] = (int32_t)lo32(fb[R]);
  }
}
// [num_split, num_empty, num_groups, num_short] from the scanned totals; with
// a live-row limit, num_empty counts the (ascending) empty rows below it only —
// a replayed mini-batch's capacity rows past the limit need no epilogue
__global__ void plan_counts_kernel(const int64_t *fa, const int64_t *fb, int64_t R,
                                   const int64_t *row_limit, int64_t *counts) {
  counts[0] = lo32(fa[R]);
  counts[1] = hi32(fa[row_limit ? min(max(*row_limit, (int64_t)0), R) : R]);
  counts[2] = lo32(fb[R]);
  counts[3] = hi32(fb[R]);
}

// Degree order of the short-row list (longest first): the NG rows a warp of
// the group-per-row kernel runs side by side then have near-equal lengths,
// so no group idles behind a longer neighbour.  Counting sort on min(deg, R);
// the order among equal degrees is arbitrary (each row's result does not
// depend on where it is scheduled).
__global__ void short_hist_kernel(const int64_t *__restrict__ off, int64_t R,
                                  const int32_t *__restrict__ rows, int64_t n, int64_t *hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[i];
    const int64_t d = min(off[r + 1] - off[r], R);
    atomicAdd(reinterpret_cast<unsigned long long *>(hist + (R - d)), 1ull);
  }
}
__global__ void short_scatter_kernel(const int64_t *__restrict__ off, int64_t R,
                                     const int32_t *__restrict__ rows, int64_t n, int64_t *cursor,
                                     int32_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[i];
    const int64_t d = min(off[r + 1] - off[r], R);
    const int64_t pos =
        (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(cursor + (R - d)), 1ull);
    out[pos] = r;
  }
}

unsigned grid_1d(int64_t n, int threads) {
  int64_t b = ceil_div(n > 0 ? n : 1, threads);
  int64_t cap = (int64_t)sm_count() * 32;
  return (unsigned)(b < cap ? b : cap);
}

template <int G, int VPL, int VW, int WM, bool PEER>
struct MainKernel {
  static constexpr auto fn = spmm_main_kernel<G, VPL, VW, WM, PEER>;
};
template <int G, int VPL, int VW, int WM, bool PEER>
struct ShortKernel {
  static constexpr auto fn = spmm_short_rows_kernel<G, VPL, VW, WM, PEER>;
};
template <template <int, int, int, int, bool> class K, int G, int VPL, int VW, bool PEER>
auto pick_wm(int wm) {
  switch (wm) {
    case WM_GLOBAL: return K<G, VPL, VW, WM_GLOBAL, PEER>::fn;
    case WM_SVALS: return K<G, VPL, VW, WM_SVALS, PEER>::fn;
    case WM_SEID: return K<G, VPL, VW, WM_SEID, PEER>::fn;
    case WM_PACKED: return K<G, VPL, VW, WM_PACKED, PEER>::fn;
    case WM_SHARED4: return K<G, VPL, VW, WM_SHARED4, PEER>::fn;
    case WM_HEADS4: return K<G, VPL, VW, WM_HEADS4, PEER>::fn;
    default: return K<G, VPL, VW, WM_NONE, PEER>::fn;
  }
}

template <int G, int VPL, int VW, bool PEER = false>
int launch_main(const SpmmArgs &a, int wm, cudaStream_t st) {
  constexpr int KB = G * VPL * VW;
  dim3 grid((unsigned)ceil_div(a.nwarps * 32, 256), (unsigned)ceil_div(a.K, KB));
  const size_t smem = (size_t)a.warp_smem * 8;
  // Shared memory only holds the staged index chunks; give the rest of the
  // unified L1/shared array to L1 so hot feature rows stay cached.
  auto kern = pick_wm<MainKernel, G, VPL, VW, PEER>(wm);
  GNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  constexpr int minb = (KB <= GNN_SPMM_MINB_KB) ? GNN_SPMM_MINB : 3;  // resident CTAs (see the kernel)
  const int per_sm_kb = (int)((smem * minb + 1023) / 1024);
  const int carve = per_sm_kb * 100 / 228 + 1;
  GNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    carve > 100 ? 100 : carve));
  kern<<<grid, 256, smem, st>>>(a);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool env_is_zero(const char *name) {
  const char *v = getenv(name);
  return v && v[0] == '0' && v[1] == 0;
}

// Per-thread, per-device side stream + fork/join events for the concurrent
// short-row launch (GNN_SPMM_CONCURRENT=0 serialises it on the caller's stream).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream &side_stream() {
  static thread_local SideStream ss[64];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream &x = ss[dev & 63];
  if (!x.s) {
    cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
  }
  return x;
}
bool spmm_concurrent() {
  static const bool on = [] {
    const char *e = getenv("GNN_SPMM_CONCURRENT");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int G, int VPL, int VW, bool PEER = false>
int launch_short(const SpmmArgs &a, int wm, const gnn_spmm_plan_t *plan, cudaStream_t st) {
  constexpr int KB = G * VPL * VW;
  constexpr int NG = 32 / G;
  const int64_t warps = ceil_div(plan->num_short, NG);
  dim3 grid((unsigned)ceil_div(warps * 32, 256), (unsigned)ceil_div(a.K, KB));
  // the short kernel reads vals / eid straight from global: SVALS == GLOBAL there
  auto kern = pick_wm<ShortKernel, G, VPL, VW, PEER>((wm == WM_SVALS || wm == WM_HEADS4) ? WM_GLOBAL : wm);
  kern<<<grid, 256, 0, st>>>(a, plan->short_rows, plan->num_short);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

struct PlanLayout {
  int64_t nw;
  int64_t o_chunk, o_csplit, o_split, o_sgb, o_empty, o_short, total;
};
PlanLayout plan_layout(int64_t R, int64_t nnz, int64_t P) {
  PlanLayout L;
  L.nw = ceil_div(nnz, P);
  int64_t o = 0;
  L.o_chunk = o;
  o += L.nw + 1;
  L.o_csplit = o;
  o += 2 * L.nw;
  L.o_split = o;
  o += R;
  L.o_sgb = o;
  o += R + 1;
  L.o_empty = o;
  o += R;
  L.o_short = o;
  o += R;
  L.total = o;
  return L;
}

}  // namespace
}  // namespace gnn

using namespace gnn;

extern "C" {

size_t gnn_spmm_plan_buffer_ints(int64_t num_rows, int64_t nnz, int64_t edges_per_warp) {
  if (edges_per_warp <= 0) return 0;
  return (size_t)plan_layout(num_rows, nnz, edges_per_warp).total;
}

size_t gnn_spmm_plan_workspace(int64_t num_rows) {
  WsCounter c;
  for (int i = 0; i < 5; ++i) c.take<int64_t>(num_rows + 1);
  c.take<int32_t>(num_rows + 1);
  c.used += 5 * (scan_i64_workspace(num_rows) + 256);
  return c.used + 512;
}

int gnn_spmm_plan_build(const gnn_csr_view_t *A, int64_t P, int32_t *buf, gnn_spmm_plan_t *plan,
                        void *ws, size_t ws_bytes, gnn_stream_t stream) {
  return gnn_spmm_plan_build_ex(A, P, 0, buf, plan, ws, ws_bytes, stream);
}

int gnn_spmm_plan_build_ex(const gnn_csr_view_t *A, int64_t P, int64_t short_max, int32_t *buf,
                           gnn_spmm_plan_t *plan, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  if (!A || !plan || !buf || P <= 0 || P % 4 != 0 || A->num_rows < 0 ||
      !A->offsets || short_max < 0)
    return GNN_ERR_INVALID_ARGUMENT;
  if (A->num_rows >= ((int64_t)1 << 31) || ceil_div(A->nnz, P) >= ((int64_t)1 << 30))
    return GNN_ERR_UNSUPPORTED;
  if (ws_bytes < gnn_spmm_plan_workspace(A->num_rows)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  const int64_t R = A->num_rows;
  WsArena ar(ws, ws_bytes);
  int64_t *fa = ar.take<int64_t>(R + 1);
  int64_t *fb = ar.take<int64_t>(R + 1);
  size_t sb = scan_i64_workspace(R);
  void *s1 = ar.take<char>((int64_t)sb);
  void *s2 = ar.take<char>((int64_t)sb);
  int64_t *dh = ar.take<int64_t>(R + 1);   // short rows: degree histogram -> cursors
  int32_t *srt = ar.take<int32_t>(R + 1);  // short rows in degree order
  void *s5 = ar.take<char>((int64_t)sb);
  if (!ar.ok()) return GNN_ERR_WORKSPACE;
  // long rows a prefix (degree-sorted operand)?  then the nnz-split kernel
  // covers only their edges and never walks the short tail
  int64_t main_nnz = A->nnz;
  if (short_max > 0 && R > 0 && A->row_ids) {  // only a permuted (sorted) operand opts in
    unsigned long long *info = reinterpret_cast<unsigned long long *>(dh);
    GNN_CUDA_TRY(cudaMemsetAsync(info, 0, 2 * sizeof(unsigned long long), st));
    plan_long_prefix_kernel<<<grid_1d(R, 256), 256, 0, st>>>(A->offsets, R, short_max, info);
    GNN_LAUNCH_CHECK();
    unsigned long long hi[2] = {1, 0};
    GNN_CUDA_TRY(cudaMemcpyAsync(hi, info, sizeof(hi), cudaMemcpyDeviceToHost, st));
    GNN_CUDA_TRY(cudaStreamSynchronize(st));
    if (hi[0] == 0) {
      GNN_CUDA_TRY(cudaMemcpyAsync(&main_nnz, A->offsets + hi[1], sizeof(int64_t),
                                   cudaMemcpyDeviceToHost, st));
      GNN_CUDA_TRY(cudaStreamSynchronize(st));
    }
  }
  const PlanLayout L = plan_layout(R, main_nnz, P);
  plan_chunk_rows_kernel<<<grid_1d(L.nw + 1, 256), 256, 0, st>>>(A->offsets, R, main_nnz, P, L.nw,
                                                                 buf + L.o_chunk);
  GNN_LAUNCH_CHECK();
  if (L.nw > 0) GNN_CUDA_TRY(cudaMemsetAsync(buf + L.o_csplit, 0xff, sizeof(int32_t) * 2 * L.nw, st));
  if (R > 0) {
    plan_flags_kernel<<<grid_1d(R, 256), 256, 0, st>>>(A->offsets, R, P, short_max, main_nnz, fa,
                                                       fb);
    GNN_LAUNCH_CHECK();
  }
  GNN_TRY(exclusive_scan_i64(fa, fa, R, true, s1, sb, st));
  GNN_TRY(exclusive_scan_i64(fb, fb, R, true, s2, sb, st));
  if (R > 0) {
    plan_scatter_kernel<<<grid_1d(R, 256), 256, 0, st>>>(A->offsets, R, P, fa, fb, buf + L.o_split,
                                                         buf + L.o_sgb, buf + L.o_csplit,
                                                         buf + L.o_empty, buf + L.o_short);
    GNN_LAUNCH_CHECK();
  }
  int64_t tot[2] = {0, 0}, h[4];
  GNN_CUDA_TRY(cudaMemcpyAsync(&tot[0], fa + R, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GNN_CUDA_TRY(cudaMemcpyAsync(&tot[1], fb + R, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GNN_CUDA_TRY(cudaStreamSynchronize(st));
  h[0] = tot[0] & 0xffffffffll;
  h[1] = tot[0] >> 32;
  h[2] = tot[1] & 0xffffffffll;
  h[3] = tot[1] >> 32;
  if (h[3] > 1) {  // longest-first order of the short rows
    int32_t *sr = buf + L.o_short;
    GNN_CUDA_TRY(cudaMemsetAsync(dh, 0, sizeof(int64_t) * (R + 1), st));
    short_hist_kernel<<<grid_1d(h[3], 256), 256, 0, st>>>(A->offsets, R, sr, h[3], dh);
    GNN_LAUNCH_CHECK();
    GNN_TRY(exclusive_scan_i64(dh, dh, R, true, s5, sb, st));
    short_scatter_kernel<<<grid_1d(h[3], 256), 256, 0, st>>>(A->offsets, R, sr, h[3], dh, srt);
    GNN_LAUNCH_CHECK();
    GNN_CUDA_TRY(cudaMemcpyAsync(sr, srt, sizeof(int32_t) * h[3], cudaMemcpyDeviceToDevice, st));
  }
  plan->edges_per_warp = P;
  plan->num_warps = L.nw;
  plan->chunk_row = buf + L.o_chunk;
  plan->chunk_split = buf + L.o_csplit;
  plan->num_split = h[0];
  plan->split_rows = buf + L.o_split;
  plan->split_group_base = buf + L.o_sgb;
  plan->num_groups = h[2];
  plan->num_empty = h[1];
  plan->empty_rows = buf + L.o_empty;
  plan->short_max = short_max;
  plan->main_nnz = main_nnz;
  plan->num_short = h[3];
  plan->short_rows = buf + L.o_short;
  plan->dev_counts = nullptr;
  plan->row_limit = nullptr;
  return GNN_OK;
}


int gnn_spmm_plan_build_dev(const gnn_csr_view_t *A, int64_t P, int64_t short_max, int32_t *buf,
                            gnn_spmm_plan_t *plan, int64_t *counts, const int64_t *row_limit,
                            void *ws, size_t ws_bytes, gnn_stream_t stream) {
  if (!A || !plan || !buf || !counts || P <= 0 || P % 4 != 0 || A->num_rows < 0 || !A->offsets ||
      short_max < 0 || A->row_ids)
    return GNN_ERR_INVALID_ARGUMENT;
  if (A->num_rows >= ((int64_t)1 << 31) || ceil_div(A->nnz, P) >= ((int64_t)1 << 30))
    return GNN_ERR_UNSUPPORTED;
  if (ws_bytes < gnn_spmm_plan_workspace(A->num_rows)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  const int64_t R = A->num_rows;
  WsArena ar(ws, ws_bytes);
  int64_t *fa = ar.take<int64_t>(R + 1);
  int64_t *fb = ar.take<int64_t>(R + 1);
  size_t sb = scan_i64_workspace(R);
  void *s1 = ar.take<char>((int64_t)sb);
  void *s2 = ar.take<char>((int64_t)sb);
  if (!ar.ok()) return GNN_ERR_WORKSPACE;
  const int64_t nnz = A->nnz;
  const PlanLayout L = plan_layout(R, nnz, P);
  plan_chunk_rows_kernel<<<grid_1d(L.nw + 1, 256), 256, 0, st>>>(A->offsets, R, nnz, P, L.nw,
                                                                 buf + L.o_chunk);
  GNN_LAUNCH_CHECK();
  if (L.nw > 0) GNN_CUDA_TRY(cudaMemsetAsync(buf + L.o_csplit, 0xff, sizeof(int32_t) * 2 * L.nw, st));
  if (R > 0) {
    plan_flags_kernel<<<grid_1d(R, 256), 256, 0, st>>>(A->offsets, R, P, short_max, nnz, fa, fb);
    GNN_LAUNCH_CHECK();
  }
  GNN_TRY(exclusive_scan_i64(fa, fa, R, true, s1, sb, st));
  GNN_TRY(exclusive_scan_i64(fb, fb, R, true, s2, sb, st));
  if (R > 0) {
    plan_scatter_kernel<<<grid_1d(R, 256), 256, 0, st>>>(A->offsets, R, P, fa, fb, buf + L.o_split,
                                                         buf + L.o_sgb, buf + L.o_csplit,
                                                         buf + L.o_empty, buf + L.o_short);
    GNN_LAUNCH_CHECK();
  }
  plan_counts_kernel<<<1, 1, 0, st>>>(fa, fb, R, row_limit, counts);
  GNN_LAUNCH_CHECK();
  // capacities: a split row spans >= 2 chunks (<= nw of them); sum over split rows
  // of ceil(partials / 64) <= num_split + (nw + num_split) / 64
  const int64_t cap_split = L.nw < R ? L.nw : R;
  plan->edges_per_warp = P;
  plan->num_warps = L.nw;
  plan->chunk_row = buf + L.o_chunk;
  plan->chunk_split = buf + L.o_csplit;
  plan->num_split = cap_split;
  plan->split_rows = buf + L.o_split;
  plan->split_group_base = buf + L.o_sgb;
  plan->num_groups = cap_split + (L.nw + cap_split) / 64 + 1;
  plan->num_empty = R;
  plan->empty_rows = buf + L.o_empty;
  plan->short_max = short_max;
  plan->main_nnz = nnz;
  plan->num_short = short_max > 0 ? R : 0;
  plan->short_rows = buf + L.o_short;
  plan->dev_counts = counts;
  plan->row_limit = row_limit;
  return GNN_OK;
}

// Upper bound on gridDim.y of the main kernel (column blocks of >= 128 columns).
static int64_t spmm_column_blocks(int64_t K) { return ceil_div(K, 128); }

static size_t spmm_ws_layout(const gnn_spmm_plan_t *plan, int64_t K, size_t *o_slots, size_t *o_l2,
                             size_t *o_cnt) {
  WsCounter c;
  *o_slots = 0;
  c.take<float>(plan->num_warps * 2 * K);
  *o_l2 = align_up(c.used, 256);
  c.take<float>(plan->num_groups * K);
  *o_cnt = align_up(c.used, 256);
  c.take<int>((plan->num_groups + plan->num_split) * spmm_column_blocks(K));
  return c.used + 256;
}

size_t gnn_spmm_workspace(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t K) {
  if (!A || !plan || K <= 0) return 0;
  size_t a, b, c;
  return spmm_ws_layout(plan, K, &a, &b, &c);
}

static int spmm_impl(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
                     const float *X, int64_t ldx, float *Y, int64_t ldy, int64_t K,
                     const gnn_epilogue_t *epi, void *ws, size_t ws_bytes, gnn_stream_t stream,
                     const float *const *parts, int64_t nparts, int64_t part_log2,
                     float shared_scale = 0.f) {
  const bool peer = parts != nullptr;
  const bool shared = shared_scale != 0.f;  // four heads over one shared X row
  const int64_t xw = shared ? K / 4 : K;    // X columns read
  if (!A || !plan || !Y || K <= 0 || heads <= 0 || K % heads != 0 || ldy < K ||
      (A->nnz > 0 && (!X || ldx < xw || !A->cols)) || !A->offsets)
    return GNN_ERR_INVALID_ARGUMENT;
  if (shared && (heads != 4 || K % 4 != 0 || !A->vals || A->eid || A->col_bits || A->row_ids ||
                 peer || plan->main_nnz != A->nnz || !aligned16(A->vals)))
    return GNN_ERR_INVALID_ARGUMENT;
  if (A->eid && !A->vals) return GNN_ERR_INVALID_ARGUMENT;
  const bool packed = A->col_bits != 0;
  if (packed && (A->col_bits < 1 || A->col_bits > 31 || A->vals || heads != 1))
    return GNN_ERR_INVALID_ARGUMENT;
  if (packed && A->num_cols > ((int64_t)1 << A->col_bits)) return GNN_ERR_INVALID_ARGUMENT;
  if (heads > 1 && !A->vals) return GNN_ERR_INVALID_ARGUMENT;
  if (plan->edges_per_warp <= 0 || plan->edges_per_warp % 4 != 0 || plan->main_nnz < 0 ||
      plan->main_nnz > A->nnz || plan->num_warps != ceil_div(plan->main_nnz, plan->edges_per_warp))
    return GNN_ERR_INVALID_ARGUMENT;
  if (A->row_ids && (epi ? epi->flags & GNN_EPI_NORM : 0) && !A->deg_offsets)
    return GNN_ERR_INVALID_ARGUMENT;  // NORM of a permuted operand needs output-row degrees
  gnn_epilogue_t e{};
  if (epi) e = *epi;
  if (((e.flags & GNN_EPI_SELF) && (!e.self_x || e.ld_self < K)) ||
      ((e.flags & GNN_EPI_BIAS) && !e.bias) || ((e.flags & GNN_EPI_MASK) && (!e.mask || e.ld_mask < K)) ||
      ((e.flags & GNN_EPI_POSTNORM) && !e.post_deg_offsets))
    return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_spmm_workspace(A, plan, K)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);

  SpmmArgs a{};
  a.R = A->num_rows;
  a.nnz = plan->main_nnz;  // the nnz-split kernel's edge range
  a.dev_counts = plan->dev_counts;
  a.row_limit = plan->row_limit;
  a.row_ids = A->row_ids;
  a.offsets = A->offsets;
  a.cols = A->cols;
  a.vals = A->vals;
  a.eid = A->eid;
  a.deg_offsets = A->deg_offsets ? A->deg_offsets : A->offsets;
  a.heads = (int)heads;
  a.F = K / heads;
  a.X = X;
  a.ldx = ldx;
  a.Y = Y;
  a.ldy = ldy;
  a.K = K;
  a.epi = e;
  if (peer) {
    for (int64_t q = 0; q < nparts; ++q) a.xt[q] = parts[q];
    a.pshift = (uint32_t)part_log2;
    a.pmask = (uint32_t)((1ull << part_log2) - 1);
  }
  a.P = plan->edges_per_warp;
  a.nwarps = plan->num_warps;
  a.chunk_row = plan->chunk_row;
  a.chunk_split = plan->chunk_split;
  a.split_rows = plan->split_rows;
  a.split_group_base = plan->split_group_base;
  size_t o_slots, o_l2, o_cnt;
  spmm_ws_layout(plan, K, &o_slots, &o_l2, &o_cnt);
  char *wsb = static_cast<char *>(ws);
  a.slots = reinterpret_cast<float *>(wsb + o_slots);
  a.l2 = reinterpret_cast<float *>(wsb + o_l2);
  a.ncb = spmm_column_blocks(K);
  a.cnt1 = reinterpret_cast<int *>(wsb + o_cnt);
  a.cnt2 = a.cnt1 + plan->num_groups * a.ncb;
  if (plan->num_groups + plan->num_split > 0)
    GNN_CUDA_TRY(cudaMemsetAsync(
        a.cnt1, 0, sizeof(int) * (plan->num_groups + plan->num_split) * a.ncb, st));
  // four heads' weights staged in the ring (float4 per edge) instead of read per lane
  const bool heads4 = !shared && !packed && A->vals && !A->eid && heads == 4 && !peer &&
                      aligned16(A->vals) && !env_is_zero("GNN_SPMM_HEADS4_STAGE");
  a.stage = (shared || heads4) ? STAGE_VALS4
                   : !A->vals ? STAGE_NONE : (A->eid ? STAGE_EID : (heads == 1 ? STAGE_VALS : STAGE_NONE));
  const int wm = shared ? WM_SHARED4
                 : packed ? WM_PACKED
                          : !A->vals ? WM_NONE
                                     : (A->eid ? WM_SEID : (heads == 1 ? WM_SVALS : heads4 ? WM_HEADS4 : WM_GLOBAL));
  a.xdiv = shared ? 4 : 1;
  a.wscale = shared ? shared_scale : 1.f;
  a.col_bits = packed ? A->col_bits : 0;
  a.col_mask = packed ? (uint32_t)((1ull << A->col_bits) - 1) : 0xffffffffu;
  a.bulk_ok = aligned16(A->cols) &&
              ((a.stage != STAGE_VALS && a.stage != STAGE_VALS4) || aligned16(A->vals)) &&
              (a.stage != STAGE_EID || aligned16(A->eid));
  a.warp_smem = a.stage == STAGE_VALS4 ? (int)(16 + 2 * 128 * 4 + 2 * 128 * 16)
                                       : (int)(16 + 2 * kSub * 4 * (a.stage != STAGE_NONE ? 2 : 1));
  // short-row kernel only where it runs several rows per warp (32/G >= 2)
  {
    const bool v4 = K % 4 == 0 && ldx % 4 == 0 && ldy % 4 == 0 && aligned16(X) && aligned16(Y) &&
                    (a.F % 4 == 0);
    a.short_max = (v4 && K <= 64 && !shared) ? plan->short_max : 0;
  }
  // a plan whose nnz-split range stops before the short tail needs the short-row kernel
  if (plan->main_nnz < A->nnz && a.short_max == 0) return GNN_ERR_UNSUPPORTED;

  // The group-per-row tail and the nnz-split kernel write disjoint rows: run
  // them concurrently (side stream forked / joined with events — also inside
  // CUDA-graph capture), so the latency-bound nnz-split kernel and the
  // L1-bound short kernel share the SMs.
  auto launch_short_rows = [&](cudaStream_t ss) -> int {
    // same lane layout as the main kernel for this K (see launch_main dispatch)
    bool vec4 = K % 4 == 0 && ldx % 4 == 0 && ldy % 4 == 0 && aligned16(X) && aligned16(Y) &&
                (a.F % 4 == 0);
    if (vec4 && (e.flags & GNN_EPI_SELF)) vec4 = e.ld_self % 4 == 0 && aligned16(e.self_x);
    if (vec4 && (e.flags & GNN_EPI_MASK)) vec4 = e.ld_mask % 4 == 0 && aligned16(e.mask);
    if (vec4 && (e.flags & GNN_EPI_BIAS)) vec4 = aligned16(e.bias);
    if (peer) {
      if (K <= 16)
        GNN_TRY((launch_short<4, 1, 4, true>(a, wm, plan, ss)));
      else if (K <= 32)
        GNN_TRY((launch_short<8, 1, 4, true>(a, wm, plan, ss)));
      else
        GNN_TRY((launch_short<16, 1, 4, true>(a, wm, plan, ss)));
    } else if (vec4) {
      if (K <= 16)
        GNN_TRY((launch_short<4, 1, 4>(a, wm, plan, ss)));
      else if (K <= 32)
        GNN_TRY((launch_short<8, 1, 4>(a, wm, plan, ss)));
      else if (K <= 64)
        GNN_TRY((launch_short<16, 1, 4>(a, wm, plan, ss)));
      else if (K <= 128)
        GNN_TRY((launch_short<32, 1, 4>(a, wm, plan, ss)));
      else
        GNN_TRY((launch_short<32, 2, 4>(a, wm, plan, ss)));
    } else {
      if (K <= 32)
        GNN_TRY((launch_short<32, 1, 1>(a, wm, plan, ss)));
      else
        GNN_TRY((launch_short<32, 4, 1>(a, wm, plan, ss)));
    }
      return GNN_OK;
  };
  const bool run_short = plan->num_short > 0 && a.short_max > 0;
  const bool concurrent = run_short && a.nwarps > 0 && spmm_concurrent();
  SideStream *side = nullptr;
  if (run_short) {
    if (concurrent) {
      side = &side_stream();
      GNN_CUDA_TRY(cudaEventRecord(side->fork, st));
      GNN_CUDA_TRY(cudaStreamWaitEvent(side->s, side->fork, 0));
      {  // the side stream inherits the caller's L2 access-policy window (gnn_l2_window)
        cudaStreamAttrValue pv = {};
        if (cudaStreamGetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &pv) == cudaSuccess)
          cudaStreamSetAttribute(side->s, cudaStreamAttributeAccessPolicyWindow, &pv);
      }
      GNN_TRY(launch_short_rows(side->s));
      GNN_CUDA_TRY(cudaEventRecord(side->join, side->s));
    } else {
      GNN_TRY(launch_short_rows(st));
    }
  }
  if (a.nwarps > 0) {
    const bool hv = A->vals != nullptr;
    // float4 path needs 16B-aligned rows and heads that do not straddle a vector
    bool vec4 = K % 4 == 0 && ldx % 4 == 0 && ldy % 4 == 0 && aligned16(X) && aligned16(Y) &&
                (a.F % 4 == 0);
    if (vec4 && (e.flags & GNN_EPI_SELF)) vec4 = e.ld_self % 4 == 0 && aligned16(e.self_x);
    if (vec4 && (e.flags & GNN_EPI_MASK)) vec4 = e.ld_mask % 4 == 0 && aligned16(e.mask);
    if (vec4 && (e.flags & GNN_EPI_BIAS)) vec4 = aligned16(e.bias);
    if (shared && !vec4) return GNN_ERR_UNSUPPORTED;
    int s;
    const bool tma_ok = vec4 && !packed && !shared && !A->row_ids && plan->main_nnz == A->nnz && (a.stage == STAGE_NONE || a.stage == STAGE_VALS) && a.heads == 1 &&
                        a.P % 4 == 0 && aligned16(A->cols) && (!hv || aligned16(A->vals)) &&
                        plan->short_max == 0 && !peer && getenv("GNN_SPMM_TMA") != nullptr;
    CUtensorMap tm;
    const int kb = K <= 16 ? 16 : K <= 32 ? 32 : K <= 64 ? 64 : K <= 128 ? 128 : 256;
    if (tma_ok && make_gather_map(&tm, X, A->num_cols, K, ldx, kb)) {
      switch (kb) {
        case 16: s = launch_tma<16>(a, hv, tm, st); break;
        case 32: s = launch_tma<32>(a, hv, tm, st); break;
        case 64: s = launch_tma<64>(a, hv, tm, st); break;
        case 128: s = launch_tma<128>(a, hv, tm, st); break;
        default: s = launch_tma<256>(a, hv, tm, st); break;
      }
    } else if (peer) {
      if (!vec4 || K > 64) return GNN_ERR_UNSUPPORTED;
      if (K <= 16)
        s = launch_main<4, 1, 4, true>(a, wm, st);
      else if (K <= 32)
        s = launch_main<8, 1, 4, true>(a, wm, st);
      else
        s = launch_main<16, 1, 4, true>(a, wm, st);
    } else if (vec4) {
      if (K <= 16)
        s = launch_main<4, 1, 4>(a, wm, st);
      else if (K <= 32)
        s = launch_main<8, 1, 4>(a, wm, st);
      else if (K <= 64)
        s = launch_main<16, 1, 4>(a, wm, st);
      else if (K <= 128)
        s = launch_main<32, 1, 4>(a, wm, st);
      else if (shared)
        s = launch_main<16, 4, 4>(a, wm, st);  // 4 heads x 64 columns: float4 gathers
      else
        s = launch_main<32, 2, 4>(a, wm, st);  // 256 columns per block-column
    } else {
      if (K <= 32)
        s = launch_main<32, 1, 1>(a, wm, st);
      else
        s = launch_main<32, 4, 1>(a, wm, st);  // 128 columns per block-column
    }
    GNN_TRY(s);
  }
  if (side) GNN_CUDA_TRY(cudaStreamWaitEvent(st, side->join, 0));
  if (plan->num_empty > 0) {
    // grid-stride; a device-count plan's capacity (every row) is no reason for a
    // grid of every row
    const unsigned eg = plan->dev_counts ? (unsigned)std::min<int64_t>(grid_1d(plan->num_empty * K, 256),
                                                                       (int64_t)sm_count() * 4)
                                         : grid_1d(plan->num_empty * K, 256);
    spmm_empty_rows_kernel<<<eg, 256, 0, st>>>(a, plan->empty_rows, plan->num_empty);
    GNN_LAUNCH_CHECK();
  }
  return GNN_OK;
}

int gnn_spmm(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
             const float *X, int64_t ldx, float *Y, int64_t ldy, int64_t K,
             const gnn_epilogue_t *epi, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  return spmm_impl(A, plan, heads, X, ldx, Y, ldy, K, epi, ws, ws_bytes, stream, nullptr, 0, 0);
}

int gnn_spmm_shared_heads(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, const float *X,
                          int64_t ldx, int64_t F, float *Y, int64_t ldy, float scale,
                          const gnn_epilogue_t *epi, void *ws, size_t ws_bytes,
                          gnn_stream_t stream) {
  if (F <= 0 || scale == 0.f) return GNN_ERR_INVALID_ARGUMENT;
  return spmm_impl(A, plan, 4, X, ldx, Y, ldy, 4 * F, epi, ws, ws_bytes, stream, nullptr, 0, 0,
                   scale);
}

int gnn_spmm_peer(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, const float *const *parts,
                  int64_t nparts, int64_t part_rows_log2, int64_t ldx, float *Y, int64_t ldy,
                  int64_t K, const gnn_epilogue_t *epi, void *ws, size_t ws_bytes,
                  gnn_stream_t stream) {
  if (!parts || nparts <= 0 || nparts > kMaxParts || part_rows_log2 < 0 || part_rows_log2 > 30)
    return GNN_ERR_INVALID_ARGUMENT;
  if ((nparts << part_rows_log2) > ((int64_t)1 << 31)) return GNN_ERR_UNSUPPORTED;
  for (int64_t q = 0; q < nparts; ++q)
    if (!parts[q] || !aligned16(parts[q])) return GNN_ERR_INVALID_ARGUMENT;
  if (A && A->num_cols > (nparts << part_rows_log2)) return GNN_ERR_INVALID_ARGUMENT;
  return spmm_impl(A, plan, 1, parts[0], ldx, Y, ldy, K, epi, ws, ws_bytes, stream, parts, nparts,
                   part_rows_log2);
}

__global__ void degree_norm_kernel(int64_t R, const int64_t *__restrict__ off, float *X,
                                   int64_t ldx, int64_t K) {
  const int64_t total = R * K;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / K, c = t % K;
    X[r * ldx + c] *= inv_deg(off, r);
  }
}

int gnn_degree_norm_inplace(int64_t R, const int64_t *offsets, float *X, int64_t ldx, int64_t K,
                            gnn_stream_t stream) {
  if (R < 0 || K < 0 || ldx < K || (R > 0 && K > 0 && (!offsets || !X)))
    return GNN_ERR_INVALID_ARGUMENT;
  if (R == 0 || K == 0) return GNN_OK;
  cudaStream_t st = as_stream(stream);
  degree_norm_kernel<<<grid_1d(R * K, 256), 256, 0, st>>>(R, offsets, X, ldx, K);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

}  // extern "C"
