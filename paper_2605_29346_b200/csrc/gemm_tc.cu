// fp32-accurate dense transform C[M,N] = A[M,K] . B[K,N] (+bias)(relu) on the
// 5th-generation tensor cores (tcgen05, kind::tf32) with a split-TF32 scheme
//   A.B = A_hi.B_hi + A_hi.B_lo + A_lo.B_hi + A_lo.B_lo,  x_hi = x & 0xffffe000, x_lo = x - x_hi
// The tensor core truncates fp32 operands to TF32 (measured), so the raw A
// tile IS A_hi and only A_lo is materialised; B is tiny and pre-split into a
// [B_hi | B_lo] operand of width 2N, so each K-step is two MMAs
//   D[:, 0:2N] += A_raw . [B_hi|B_lo]^T  and  D += A_lo . [B_hi|B_lo]^T
// and the epilogue adds the two halves.  fp32 accumulation in tensor memory.  This is the only
// dense contraction on the path: X.W with X [V,K] fp32,
// W [K,N<=256] — HBM-bound (arithmetic intensity ~8 flop/B for N=16), so the
// design goal is to stream A at HBM speed.
//
// One persistent CTA per SM, 12 warps, warp-specialised:
//   warp 0      TMA producer: A tile [128 x 32] fp32 (SWIZZLE_128B) + B_hi/B_lo
//               tiles [N x 32] per k-block into a 5-stage smem ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, K=8)
//   warps 4-7   split warps: A -> A_hi (in place) + A_lo (second buffer)
//   warps 8-11  epilogue warpgroup: tcgen05.ld (32x32b) -> bias/relu -> global
// TMEM holds two accumulators so the epilogue of tile i overlaps tile i+1.
#include <algorithm>
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"

namespace gnn {
namespace {

constexpr int kTcM = 128;
constexpr int kTcBK = 32;  // fp32 elements per k-block = one 128-byte swizzle row
// smem ring depth: ~200 KB of stages whatever the B tile width
template <int NPAD>
constexpr int tc_stages() {
  return NPAD <= 16 ? 6 : (NPAD <= 32 ? 5 : (NPAD <= 64 ? 4 : 3));
}
constexpr int kTcThreads = 384;

struct TcArgs {
  int64_t M, N, K;
  int Npad;
  int nkb;
  int64_t mtiles;
  float *C;
  int64_t ldc;
  const float *bias;
  int relu;
  int vec_store;  // C rows 16-byte aligned: 128-bit epilogue stores
  const int64_t *rows_dev;  // live rows on device (tiles past them skipped), or null
  // row-dot epilogue (C not stored): S[row, c mod 4] (+)= sum_c C[row, c] * dotY[row, c]
  // over the block's N columns, S[row, h] at dotS[row * ldS + h * dot_hs]
  const float *dotY;
  int64_t lddot;
  float *dotS;
  int64_t ldS, dot_hs;
  int dot_acc;  // add to S (a later column block) instead of overwriting it
  // GAT concatenated-heads backward epilogue (EPI_GAT): with G = the product row,
  // C[r, c] = G[r, c] * (Y[r, c] > 0) (ReLU backward) and C[r, N + 4h .. 4h + 3] =
  // {er[r, h], m[r, h], inv[r, h], S[r, h]}, S[r, h] = sum over head h's F = N/4
  // columns of C[r, c] * (Y[r, c] - bias[c])  (the recompute backward's row stats)
  const float *gY, *gbias, *ger, *grs;
  int64_t ldgy;
  // GAT attention projections epilogue (EPI_PROJ): with C stored as usual, for
  // the 4 heads of width pF (a multiple of 16) el[r, h] (+)= sum_c C[r, c] al[c0g + c],
  // er likewise, over this column block [pn0, pn0 + N) of the full row (flat
  // [4 * pF] attention vectors); a head begun by an earlier block accumulates
  const float *pal, *par;
  float *pel, *per;
  int pF;
  int64_t pn0;
};

template <int NPAD>
constexpr size_t tc_smem_bytes() {
  return (size_t)tc_stages<NPAD>() * (2 * kTcM * kTcBK + 2 * NPAD * kTcBK) * 4 + 1024 + 1024;
}

constexpr int EPI_PLAIN = 0, EPI_DOT = 1, EPI_GAT = 2, EPI_PROJ = 3;
template <int NPAD, int EPI = EPI_PLAIN>
__global__ void __launch_bounds__(kTcThreads, 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                const __grid_constant__ CUtensorMap tmBhi,
                                                                const __grid_constant__ CUtensorMap tmBlo,
                                                                TcArgs p) {
  constexpr int kTcStages = tc_stages<NPAD>();
  extern __shared__ __align__(1024) uint8_t tc_raw[];
  // carve 1024-aligned regions
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~(uintptr_t)1023);
  constexpr size_t kA = (size_t)kTcM * kTcBK * 4;
  constexpr size_t kB = (size_t)NPAD * kTcBK * 4;
  float *sa = reinterpret_cast<float *>(base);
  float *salo = reinterpret_cast<float *>(base + kTcStages * kA);
  float *sbhi = reinterpret_cast<float *>(base + 2 * kTcStages * kA);  // [stage][hi rows|lo rows]
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + 2 * kTcStages * kA + 2 * kTcStages * kB);
  uint64_t *full = bars, *split = bars + kTcStages, *empty = bars + 2 * kTcStages;
  uint64_t *acc_full = bars + 3 * kTcStages, *acc_empty = acc_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = (int)lane_id();
  constexpr uint32_t kTxBytes = (uint32_t)(kA + 2 * kB);
  // every role walks the same tile sequence: live tiles only when rows_dev is set
  const int64_t mtiles = p.rows_dev ? min(p.mtiles, ceil_div(*p.rows_dev, (int64_t)kTcM)) : p.mtiles;
  constexpr int kAcc = 2 * NPAD;  // accumulator width: [hi half | lo half]
  constexpr int kTmemCols = (2 * kAcc) <= 32 ? 32 : (2 * kAcc) <= 64 ? 64 : (2 * kAcc) <= 128 ? 128 : (2 * kAcc) <= 256 ? 256 : 512;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(split + s, 4);  // one elected arrival per split warp
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + b, 1);
      mbar_init(acc_empty + b, 4);  // one per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // idesc: D f32, A/B tf32, K-major both, N = 2*NPAD, M=128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kAcc >> 3) << 17) |
                         ((uint32_t)(kTcM >> 4) << 24);

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < mtiles; t += gridDim.x) {
        const int m0 = (int)(t * kTcM);
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(empty + s, ph ^ 1);
          mbar_arrive_expect_tx(full + s, kTxBytes);
          tma_load_2d(smem_u32(sa + (size_t)s * kTcM * kTcBK), &tmA, kb * kTcBK, m0, smem_u32(full + s));
          tma_load_2d(smem_u32(sbhi + (size_t)s * 2 * NPAD * kTcBK), &tmBhi, kb * kTcBK, 0,
                      smem_u32(full + s));
          tma_load_2d(smem_u32(sbhi + (size_t)s * 2 * NPAD * kTcBK + NPAD * kTcBK), &tmBlo, kb * kTcBK,
                      0, smem_u32(full + s));
          if (++s == kTcStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int ab = 0;
      uint32_t aph = 0;
      for (int64_t t = blockIdx.x; t < mtiles; t += gridDim.x) {
        mbar_wait(acc_empty + ab, aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(ab * kAcc);
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(split + s, ph);
          tc_fence_after();
          const uint64_t ah = sw128_desc(smem_u32(sa + (size_t)s * kTcM * kTcBK));
          const uint64_t al = sw128_desc(smem_u32(salo + (size_t)s * kTcM * kTcBK));
          const uint64_t bc = sw128_desc(smem_u32(sbhi + (size_t)s * 2 * NPAD * kTcBK));  // [hi|lo] rows
#pragma unroll
          for (int k = 0; k < kTcBK / 8; ++k) {  // K=8 tf32 = 32 bytes per MMA: +2 in the >>4 address field
            const uint64_t o = (uint64_t)(k * 2);
            tc_mma_tf32(d, ah + o, bc + o, idesc, (kb | k) != 0);
            tc_mma_tf32(d, al + o, bc + o, idesc, 1);
          }
          tc_commit(empty + s);  // smem stage free once these MMAs retire
          if (kb == p.nkb - 1) tc_commit(acc_full + ab);
          if (++s == kTcStages) {
            s = 0;
            ph ^= 1;
          }
        }
        if (++ab == 2) {
          ab = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- split warps: A -> (A_hi in place, A_lo)
    const int tid = threadIdx.x - 128;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < mtiles; t += gridDim.x) {
      for (int kb = 0; kb < p.nkb; ++kb) {
        mbar_wait(full + s, ph);
        float4 *a4 = reinterpret_cast<float4 *>(sa + (size_t)s * kTcM * kTcBK);
        float4 *l4 = reinterpret_cast<float4 *>(salo + (size_t)s * kTcM * kTcBK);
#pragma unroll 4
        for (int i = tid; i < kTcM * kTcBK / 4; i += 128) {
          float4 x = a4[i];
          float4 h;
          h.x = __uint_as_float(__float_as_uint(x.x) & 0xffffe000u);
          h.y = __uint_as_float(__float_as_uint(x.y) & 0xffffe000u);
          h.z = __uint_as_float(__float_as_uint(x.z) & 0xffffe000u);
          h.w = __uint_as_float(__float_as_uint(x.w) & 0xffffe000u);
          l4[i] = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);  // raw A is A_hi to the MMA
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(split + s);
        if (++s == kTcStages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp >= 8) {
    // ---------------- epilogue warpgroup: TMEM lane quarter = warp % 4
    const int q = warp & 3;
    int ab = 0;
    uint32_t aph = 0;
    for (int64_t t = blockIdx.x; t < mtiles; t += gridDim.x) {
      mbar_wait(acc_full + ab, aph);
      tc_fence_after();
      const int64_t row = t * kTcM + q * 32 + lane;
      float *crow = p.C + row * p.ldc;
      float4 dacc = make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (EPI == EPI_DOT) {
        // row-dot epilogue: the row's Y slice is fetched 64 columns at a time
        // (16 loads in flight per thread) ahead of the TMEM reads it meets
        constexpr int kDR = NPAD < 64 ? NPAD : 64;
        for (int r0 = 0; r0 < NPAD; r0 += kDR) {
          float4 y4[kDR / 4];
#pragma unroll
          for (int j = 0; j < kDR / 4; ++j)
            y4[j] = row < p.M && r0 + 4 * j < p.N ? ldg_f4(p.dotY + row * p.lddot + r0 + 4 * j)
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int c1 = 0; c1 < kDR; c1 += 16) {
            uint32_t v[16], u[16];
            const uint32_t taddr =
                tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * kAcc + r0 + c1);
            tmem_ld16(taddr, v);
            tmem_ld16(taddr + NPAD, u);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 y = y4[c1 / 4 + j];
              dacc.x = fmaf(__uint_as_float(v[4 * j]) + __uint_as_float(u[4 * j]), y.x, dacc.x);
              dacc.y = fmaf(__uint_as_float(v[4 * j + 1]) + __uint_as_float(u[4 * j + 1]), y.y, dacc.y);
              dacc.z = fmaf(__uint_as_float(v[4 * j + 2]) + __uint_as_float(u[4 * j + 2]), y.z, dacc.z);
              dacc.w = fmaf(__uint_as_float(v[4 * j + 3]) + __uint_as_float(u[4 * j + 3]), y.w, dacc.w);
            }
          }
        }
      }
      if constexpr (EPI == EPI_GAT) {
        // ReLU backward + per-head row statistics; F = N / 4 columns per head, a
        // multiple of 16 (each 16-column chunk lies in one head)
        float S[4] = {0.f, 0.f, 0.f, 0.f};
        const int F = (int)(p.N >> 2);
        for (int c0 = 0; c0 < p.N; c0 += 16) {
          uint32_t v[16], u[16];
          const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * kAcc + c0);
          tmem_ld16(taddr, v);
          tmem_ld16(taddr + NPAD, u);
          float4 y4[4], b4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            y4[j] = row < p.M ? ldg_f4(p.gY + row * p.ldgy + c0 + 4 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
            b4[j] = ldg_f4(p.gbias + c0 + 4 * j);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float sh = 0.f;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float yv[4] = {y4[j].x, y4[j].y, y4[j].z, y4[j].w};
            const float bv[4] = {b4[j].x, b4[j].y, b4[j].z, b4[j].w};
            float mv[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float gv = __uint_as_float(v[4 * j + t]) + __uint_as_float(u[4 * j + t]);
              mv[t] = yv[t] > 0.f ? gv : 0.f;
              sh = fmaf(mv[t], yv[t] - bv[t], sh);
            }
            if (row < p.M)
              *reinterpret_cast<float4 *>(crow + c0 + 4 * j) = make_float4(mv[0], mv[1], mv[2], mv[3]);
          }
          const int h = c0 / F;
#pragma unroll
          for (int hh = 0; hh < 4; ++hh) S[hh] += hh == h ? sh : 0.f;
        }
        if (row < p.M) {
#pragma unroll
          for (int hh = 0; hh < 4; ++hh)
            *reinterpret_cast<float4 *>(crow + p.N + 4 * hh) =
                make_float4(__ldg(p.ger + row * 4 + hh), __ldg(p.grs + row * 8 + hh),
                            __ldg(p.grs + row * 8 + 4 + hh), S[hh]);
        }
      }
      float pl[4] = {0.f, 0.f, 0.f, 0.f}, pr[4] = {0.f, 0.f, 0.f, 0.f};
      for (int c0 = 0; c0 < NPAD && (EPI == EPI_PLAIN || EPI == EPI_PROJ); c0 += 16) {
        uint32_t v[16], u[16];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * kAcc + c0);
        tmem_ld16(taddr, v);
        tmem_ld16(taddr + NPAD, u);  // the B_lo half
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < p.M && p.vec_store && c0 + 16 <= p.N) {
          // full 16-column slice: 4 x 128-bit stores instead of 16 scalar ones
          float y[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            y[j] = __uint_as_float(v[j]) + __uint_as_float(u[j]);
            if (p.bias) y[j] += __ldg(p.bias + c0 + j);
            if (p.relu) y[j] = fmaxf(y[j], 0.f);
          }
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            *reinterpret_cast<float4 *>(crow + c0 + j) = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
          if constexpr (EPI == EPI_PROJ) {
            const int64_t cg = p.pn0 + c0;     // the chunk's first column of the full row
            const int h = (int)(cg / p.pF);    // one head per 16-column chunk
            float sl = 0.f, sr = 0.f;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              sl = fmaf(y[j], __ldg(p.pal + cg + j), sl);
              sr = fmaf(y[j], __ldg(p.par + cg + j), sr);
            }
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) {
              pl[hh] += hh == h ? sl : 0.f;
              pr[hh] += hh == h ? sr : 0.f;
            }
          }
        } else if (row < p.M) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int64_t c = c0 + j;
            if (c < p.N) {
              float y = __uint_as_float(v[j]) + __uint_as_float(u[j]);
              if (p.bias) y += p.bias[c];
              if (p.relu) y = fmaxf(y, 0.f);
              crow[c] = y;
            }
          }
        }
      }
      if (EPI == EPI_PROJ && row < p.M) {
        // heads this block touches: [pn0 / pF, (pn0 + N - 1) / pF]; one begun by an
        // earlier block (its first column < pn0) accumulates
        const int h0 = (int)(p.pn0 / p.pF), h1 = (int)((p.pn0 + p.N - 1) / p.pF);
#pragma unroll
        for (int hh = 0; hh < 4; ++hh)
          if (hh >= h0 && hh <= h1) {
            const bool acc = (int64_t)hh * p.pF < p.pn0;
            p.pel[row * 4 + hh] = acc ? p.pel[row * 4 + hh] + pl[hh] : pl[hh];
            p.per[row * 4 + hh] = acc ? p.per[row * 4 + hh] + pr[hh] : pr[hh];
          }
      }
      if (EPI == EPI_DOT && row < p.M) {
        float *sr = p.dotS + row * p.ldS;
        const float d[4] = {dacc.x, dacc.y, dacc.z, dacc.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) sr[h * p.dot_hs] = p.dot_acc ? sr[h * p.dot_hs] + d[h] : d[h];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + ab);
      if (++ab == 2) {
        ab = 0;
        aph ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols)
                 : "memory");
}

// ------------------------------------------------------------------------
// Weight-gradient shape C[M,N] = A^T B, A [K,M] (row stride lda), B [K,N]
// (ldb): the contraction runs over the K = |V| rows, so both operands are
// MN-major in shared memory.  MN-major tf32 operands have exactly one legal
// smem layout, SWIZZLE_128B_BASE32B (TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B):
// 128-byte MN rows (32 fp32), 4-row K groups (SBO = 512 B), MN atoms = the
// 32-column TMA boxes, 4 KB apart (LBO).  A is a 128-wide M tile (4 atoms,
// OOB columns zero-filled); B is an NB-wide N tile (NB/32 atoms) followed in
// shared memory by NB/32 atoms of B_lo written by the split warps, so
// [B_hi | B_lo] is ONE 2*NB-wide MN-major operand (same atom stride) and each
// 8-row K step is two MMAs (A_hi and A_lo against [B_hi|B_lo]).
// Work units = (m-tile, n-tile, k-split); each unit's [128 x NB] partial is
// written to global and the splits are summed in a fixed order.

// The tensor cores' fp32 accumulation rounds each MMA's sum toward zero, so a
// long chain of MMAs into one TMEM accumulator drifts when every product has
// the same sign (GIN's U1^T dY1 at 233K rows: 400 MMAs per split, 3.9e-5 of
// sum |terms| measured, 1e-5 required).  Each unit therefore accumulates
// kTnChunk k-blocks (16 MMA pairs) per TMEM pass and the epilogue warps add
// the chunk into fp32 registers (round-to-nearest), double-buffered so the
// next chunk's MMAs run under the read-out.
constexpr int kTnChunk = 2;

template <int NB>
constexpr int tn_stages() {
  return NB <= 32 ? 5 : (NB <= 64 ? 4 : 3);
}
template <int NB>
constexpr size_t tn_smem_bytes() {
  return (size_t)tn_stages<NB>() * (2 * kTcM * kTcBK + 2 * NB * kTcBK) * 4 + 2048;
}

struct TnArgs {
  int64_t M, N, K;
  int nkb_total;      // ceil(K / 32)
  int kb_per_split;
  int splits;
  int64_t mtiles, ntiles;
  float *partials;    // [splits][M][N]
  const int64_t *rows_dev;  // live contraction rows on device, or null
};

template <int NB>
__global__ void __launch_bounds__(kTcThreads, 1) gemm_tc_tn_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TnArgs p) {
  static_assert(NB == 32 || NB == 64 || NB == 128, "N tile = whole 32-column atoms, 2*NB <= 256");
  constexpr int kStages = tn_stages<NB>();
  constexpr int kAtomsB = NB / 32;
  extern __shared__ __align__(1024) uint8_t tn_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(tn_raw) + 1023) & ~(uintptr_t)1023);
  constexpr size_t kA = (size_t)kTcM * kTcBK * 4;   // 16 KB: 4 atoms of [32 rows x 128 B]
  constexpr size_t kB = (size_t)kTcBK * NB * 4;     // hi atoms; the lo atoms follow
  float *sa = reinterpret_cast<float *>(base);
  float *salo = reinterpret_cast<float *>(base + kStages * kA);
  float *sb = reinterpret_cast<float *>(base + 2 * kStages * kA);  // [stage][hi atoms | lo atoms]
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + 2 * kStages * kA + 2 * kStages * kB);
  uint64_t *full = bars, *split = bars + kStages, *empty = bars + 2 * kStages;
  uint64_t *acc_full = bars + 3 * kStages, *acc_empty = acc_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);
  const int warp = threadIdx.x >> 5;
  const int lane = (int)lane_id();
  constexpr uint32_t kTx = (uint32_t)(kA + kB);
  constexpr int kAcc = 2 * NB;                 // [hi | lo] accumulator columns
  constexpr int kTmemCols = 2 * kAcc < 32 ? 32 : 2 * kAcc;  // two accumulators
  const int64_t units = p.mtiles * p.ntiles * p.splits;
  // live contraction rows: k-blocks past them are skipped, and the rows of the
  // last live block past them are zeroed (a capacity buffer's tail is stale)
  const int64_t klive = p.rows_dev ? min(p.K, *p.rows_dev) : p.K;
  const int nkb_live = (int)ceil_div(klive, (int64_t)kTcBK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(split + s, 4);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + b, 1);
      mbar_init(acc_empty + b, 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // idesc: D f32, A/B tf32, A and B MN-major, N = 2*NB, M = 128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                         ((uint32_t)(kAcc >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);

  auto unit_of = [&](int64_t u, int &kb0, int &kb1, int &m0, int &n0, int64_t &sp) {
    const int64_t mt = u % p.mtiles;
    const int64_t nt = (u / p.mtiles) % p.ntiles;
    sp = u / (p.mtiles * p.ntiles);
    m0 = (int)(mt * kTcM);
    n0 = (int)(nt * NB);
    // the splits share the live k-blocks evenly (all of them without rows_dev)
    const int kbps = p.rows_dev ? (nkb_live + p.splits - 1) / p.splits : p.kb_per_split;
    kb1 = min(min(p.nkb_total, (int)sp * kbps + kbps), nkb_live);
    kb0 = min((int)sp * kbps, kb1);
  };

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int kb0, kb1, m0, n0;
        int64_t sp;
        unit_of(u, kb0, kb1, m0, n0, sp);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(empty + s, ph ^ 1);
          mbar_arrive_expect_tx(full + s, kTx);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            tma_load_2d(smem_u32(sa + (size_t)s * kTcM * kTcBK + j * 32 * kTcBK), &tmA, m0 + 32 * j,
                        kb * kTcBK, smem_u32(full + s));
#pragma unroll
          for (int j = 0; j < kAtomsB; ++j)
            tma_load_2d(smem_u32(sb + (size_t)s * 2 * NB * kTcBK + j * 32 * kTcBK), &tmB,
                        n0 + 32 * j, kb * kTcBK, smem_u32(full + s));
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int ab = 0;
      uint32_t aph = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int kb0, kb1, m0, n0;
        int64_t sp;
        unit_of(u, kb0, kb1, m0, n0, sp);
        uint32_t d = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
          const int kc = (kb - kb0) % kTnChunk;  // k-block within this accumulation chunk
          if (kc == 0) {
            mbar_wait(acc_empty + ab, aph ^ 1);
            tc_fence_after();
            d = tmem + (uint32_t)(ab * kAcc);
          }
          mbar_wait(split + s, ph);
          tc_fence_after();
          const uint32_t a_hi = smem_u32(sa + (size_t)s * kTcM * kTcBK);
          const uint32_t a_lo = smem_u32(salo + (size_t)s * kTcM * kTcBK);
          const uint32_t b_hl = smem_u32(sb + (size_t)s * 2 * NB * kTcBK);
#pragma unroll
          for (int k = 0; k < kTcBK / 8; ++k) {  // 8 K-rows per MMA = 1 KB of every atom
            const uint64_t ah = mn_desc(a_hi + k * 1024, 4096, 512, 1);
            const uint64_t al = mn_desc(a_lo + k * 1024, 4096, 512, 1);
            const uint64_t bc = mn_desc(b_hl + k * 1024, 4096, 512, 1);  // [hi atoms | lo atoms]
            tc_mma_tf32(d, ah, bc, idesc, (kc != 0 || k != 0) ? 1u : 0u);
            tc_mma_tf32(d, al, bc, idesc, 1);
          }
          tc_commit(empty + s);
          if (kc == kTnChunk - 1 || kb == kb1 - 1) {
            tc_commit(acc_full + ab);
            if (++ab == 2) {
              ab = 0;
              aph ^= 1;
            }
          }
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    const int tid = threadIdx.x - 128;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      int kb0, kb1, m0, n0;
      int64_t sp;
      unit_of(u, kb0, kb1, m0, n0, sp);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(full + s, ph);
        float4 *a4 = reinterpret_cast<float4 *>(sa + (size_t)s * kTcM * kTcBK);
        float4 *l4 = reinterpret_cast<float4 *>(salo + (size_t)s * kTcM * kTcBK);
        // rows of this block past the live count (kTcBK rows of 128 B per atom)
        const int live_rows = (int)min((int64_t)kTcBK, klive - (int64_t)kb * kTcBK);
#pragma unroll 4
        for (int i = tid; i < kTcM * kTcBK / 4; i += 128) {
          float4 x = a4[i];
          if (((i & 255) >> 3) >= live_rows) {  // row (i % 256) / 8 of atom i / 256
            x = make_float4(0.f, 0.f, 0.f, 0.f);
            a4[i] = x;
          }
          float4 h;
          h.x = __uint_as_float(__float_as_uint(x.x) & 0xffffe000u);
          h.y = __uint_as_float(__float_as_uint(x.y) & 0xffffe000u);
          h.z = __uint_as_float(__float_as_uint(x.z) & 0xffffe000u);
          h.w = __uint_as_float(__float_as_uint(x.w) & 0xffffe000u);
          l4[i] = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);  // raw A = A_hi
        }
        // B_lo atoms sit kB bytes after the hi atoms: same swizzle phase (4 KB multiple)
        const float4 *b4 = reinterpret_cast<const float4 *>(sb + (size_t)s * 2 * NB * kTcBK);
        float4 *bl4 = reinterpret_cast<float4 *>(sb + (size_t)s * 2 * NB * kTcBK + NB * kTcBK);
#pragma unroll 4
        for (int i = tid; i < NB * kTcBK / 4; i += 128) {
          const float4 x = b4[i];
          float4 lo;
          lo.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xffffe000u);
          lo.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xffffe000u);
          lo.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xffffe000u);
          lo.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xffffe000u);
          bl4[i] = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(split + s);
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp >= 8) {
    const int q = warp & 3;
    int ab = 0;
    uint32_t aph = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      int kb0, kb1, m0, n0;
      int64_t sp;
      unit_of(u, kb0, kb1, m0, n0, sp);
      const int64_t m = (int64_t)m0 + q * 32 + lane;
      float acc[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[j] = 0.f;
      const int nchunks = (kb1 - kb0 + kTnChunk - 1) / kTnChunk;
#pragma unroll 1
      for (int ch = 0; ch < nchunks; ++ch) {
        mbar_wait(acc_full + ab, aph);
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < NB; c0 += 16) {
          uint32_t v[16], w[16];
          const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * kAcc + c0);
          tmem_ld16(taddr, v);
          tmem_ld16(taddr + NB, w);  // B_lo half
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[c0 + j] += __uint_as_float(v[j]) + __uint_as_float(w[j]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + ab);
        if (++ab == 2) {
          ab = 0;
          aph ^= 1;
        }
      }
      if (m < p.M) {
        float *dst = p.partials + (sp * p.M + m) * p.N;
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (n0 + j < p.N) dst[n0 + j] = acc[j];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols)
                 : "memory");
}

// Split-K reduction: 8 lanes per output stride the splits (independent
// loads in flight instead of one dependent chain), fixed-order butterfly.
__global__ void tn_reduce_kernel(int64_t M, int64_t N, int splits, const float *__restrict__ partials,
                                 float *C, int64_t ldc) {
  const int64_t total = M * N;
  const int sub = (int)(threadIdx.x & 7);
  const unsigned mask8 = 0xffu << (threadIdx.x & 24);  // this output's 8 lanes
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3; t < total;
       t += ((int64_t)gridDim.x * blockDim.x) >> 3) {
    float s = 0.f;
    for (int z = sub; z < splits; z += 8) s += partials[(int64_t)z * total + t];
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) s += __shfl_xor_sync(mask8, s, o, 8);
    if (sub == 0) C[(t / N) * ldc + (t % N)] = s;
  }
}

// B [K,N] row-major (ldb) or B^T [N,K] (trans_b) -> Bt_hi / Bt_lo [Npad, Kpad] K-major, zero padded.
__global__ void split_b_kernel(const float *__restrict__ B, int64_t ldb, int trans_b, int64_t N,
                               int64_t K, int Npad, int64_t Kpad, float *bhi, float *blo) {
  const int64_t total = (int64_t)Npad * Kpad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / Kpad, k = i % Kpad;
    float x = 0.f;
    if (n < N && k < K) x = trans_b ? B[n * ldb + k] : B[k * ldb + n];
    const float h = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
    bhi[i] = h;
    blo[i] = x - h;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                             const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                             const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  }
  return fn;
}
bool map_2d_sw128(CUtensorMap *tm, const float *base, int64_t inner, int64_t outer, int64_t ld,
                  int box_outer) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)kTcBK, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool map_2d(CUtensorMap *tm, const float *base, int64_t inner, int64_t outer, int64_t ld,
            int box_inner, int box_outer, CUtensorMapSwizzle sw) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NPAD, int EPI = EPI_PLAIN>
int launch_tc(const CUtensorMap &ta, const CUtensorMap &tbh, const CUtensorMap &tbl,
              const TcArgs &p, cudaStream_t st) {
  const size_t smem = tc_smem_bytes<NPAD>();
  GNN_CUDA_TRY(cudaFuncSetAttribute(gemm_tc_kernel<NPAD, EPI>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t grid = p.mtiles < sm_count() ? p.mtiles : sm_count();
  gemm_tc_kernel<NPAD, EPI><<<(unsigned)grid, kTcThreads, smem, st>>>(ta, tbh, tbl, p);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

}  // namespace

// Tensor-core path applicability: A row-major with a 16-byte-multiple row
// stride (TMA), 16-byte aligned base, N <= 128.
bool gemm_tc_supported(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, int trans_a) {
  return !trans_a && M >= kTcM && N >= 1 && N <= 128 && K >= 1 && (lda * 4) % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(A) & 15u) == 0 && encode_fn() != nullptr &&
         getenv("GNN_GEMM_NO_TC") == nullptr;
}

static int tc_npad(int64_t N) { return N <= 16 ? 16 : N <= 32 ? 32 : N <= 64 ? 64 : 128; }

size_t gemm_tc_workspace(int64_t N, int64_t K) {
  const int64_t kpad = ceil_div(K, kTcBK) * kTcBK;
  return sizeof(float) * (size_t)(2 * tc_npad(N) * kpad) + 512;
}

int gemm_tc(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
            int64_t ldb, int trans_b, float *C, int64_t ldc, const float *bias, int relu, void *ws,
            size_t ws_bytes, cudaStream_t st, const int64_t *rows_dev) {
  const int npad = tc_npad(N);
  const int64_t kpad = ceil_div(K, kTcBK) * kTcBK;
  if (ws_bytes < gemm_tc_workspace(N, K)) return GNN_ERR_WORKSPACE;
  float *bhi = static_cast<float *>(ws);
  float *blo = bhi + (size_t)npad * kpad;
  split_b_kernel<<<(unsigned)ceil_div((int64_t)npad * kpad, 256), 256, 0, st>>>(
      B, ldb, trans_b, N, K, npad, kpad, bhi, blo);
  GNN_LAUNCH_CHECK();
  CUtensorMap ta, tbh, tbl;
  if (!map_2d_sw128(&ta, A, K, M, lda, kTcM) || !map_2d_sw128(&tbh, bhi, kpad, npad, kpad, npad) ||
      !map_2d_sw128(&tbl, blo, kpad, npad, kpad, npad))
    return GNN_ERR_UNSUPPORTED;
  TcArgs p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.Npad = npad;
  p.nkb = (int)(kpad / kTcBK);
  p.mtiles = ceil_div(M, kTcM);
  p.C = C;
  p.ldc = ldc;
  p.bias = bias;
  p.relu = relu;
  p.vec_store = (ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(C) & 15u) == 0);
  p.rows_dev = rows_dev;
  switch (npad) {
    case 16: return launch_tc<16>(ta, tbh, tbl, p, st);
    case 32: return launch_tc<32>(ta, tbh, tbl, p, st);
    case 64: return launch_tc<64>(ta, tbh, tbl, p, st);
    default: return launch_tc<128>(ta, tbh, tbl, p, st);
  }
}

// Row-dot form: S[m, h] = sum over columns c = h (mod 4) of (A Bt^T)[m, c] * Y[m, c],
// Bt [N, K] row-major (ldb), N % 4 == 0; the product never leaves the SM
// (128-column blocks, the later ones accumulating into S in block order).
int gemm_tc_rowdot(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *Bt,
                   int64_t ldb, const float *Y, int64_t ldy, float *S, int64_t ldS, int64_t hs,
                   void *ws, size_t ws_bytes, cudaStream_t st) {
  if (N % 4 || !gemm_tc_supported(M, 128, K, A, lda, 0) || (ldy % 4) ||
      (reinterpret_cast<uintptr_t>(Y) & 15u))
    return GNN_ERR_UNSUPPORTED;
  for (int64_t n0 = 0; n0 < N; n0 += 128) {
    const int64_t nb = N - n0 < 128 ? N - n0 : 128;
    const int npad = tc_npad(nb);
    const int64_t kpad = ceil_div(K, kTcBK) * kTcBK;
    if (ws_bytes < gemm_tc_workspace(nb, K)) return GNN_ERR_WORKSPACE;
    float *bhi = static_cast<float *>(ws);
    float *blo = bhi + (size_t)npad * kpad;
    split_b_kernel<<<(unsigned)ceil_div((int64_t)npad * kpad, 256), 256, 0, st>>>(
        Bt + n0 * ldb, ldb, 1, nb, K, npad, kpad, bhi, blo);
    GNN_LAUNCH_CHECK();
    CUtensorMap ta, tbh, tbl;
    if (!map_2d_sw128(&ta, A, K, M, lda, kTcM) || !map_2d_sw128(&tbh, bhi, kpad, npad, kpad, npad) ||
        !map_2d_sw128(&tbl, blo, kpad, npad, kpad, npad))
      return GNN_ERR_UNSUPPORTED;
    TcArgs p{};
    p.M = M;
    p.N = nb;
    p.K = K;
    p.Npad = npad;
    p.nkb = (int)(kpad / kTcBK);
    p.mtiles = ceil_div(M, kTcM);
    p.dotY = Y + n0;
    p.lddot = ldy;
    p.dotS = S;
    p.ldS = ldS;
    p.dot_hs = hs;
    p.dot_acc = n0 > 0;
    int rc;
    switch (npad) {
      case 16: rc = launch_tc<16, EPI_DOT>(ta, tbh, tbl, p, st); break;
      case 32: rc = launch_tc<32, EPI_DOT>(ta, tbh, tbl, p, st); break;
      case 64: rc = launch_tc<64, EPI_DOT>(ta, tbh, tbl, p, st); break;
      default: rc = launch_tc<128, EPI_DOT>(ta, tbh, tbl, p, st); break;
    }
    if (rc != GNN_OK) return rc;
  }
  return GNN_OK;
}

// GAT layer transform with the attention projections in the epilogue:
// C = A B (B [K, N] row-major, N = 4F, F % 16 == 0, 16-byte aligned C rows),
// el[r, h] = <C[r, hF:(h+1)F], al[h]>, er likewise (al / ar flat [4F]);
// 128-column blocks, heads straddling two blocks accumulate in block order.
int gemm_tc_gat_proj(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
                     int64_t ldb, float *C, int64_t ldc, int F, const float *al, const float *ar,
                     float *el, float *er, void *ws, size_t ws_bytes, cudaStream_t st) {
  if (N != 4 * (int64_t)F || F % 16 || ldc % 4 || (reinterpret_cast<uintptr_t>(C) & 15u) ||
      !gemm_tc_supported(M, 128, K, A, lda, 0))
    return GNN_ERR_UNSUPPORTED;
  for (int64_t n0 = 0; n0 < N; n0 += 128) {
    const int64_t nb = N - n0 < 128 ? N - n0 : 128;
    const int npad = tc_npad(nb);
    const int64_t kpad = ceil_div(K, kTcBK) * kTcBK;
    if (ws_bytes < gemm_tc_workspace(nb, K)) return GNN_ERR_WORKSPACE;
    float *bhi = static_cast<float *>(ws);
    float *blo = bhi + (size_t)npad * kpad;
    split_b_kernel<<<(unsigned)ceil_div((int64_t)npad * kpad, 256), 256, 0, st>>>(
        B + n0, ldb, 0, nb, K, npad, kpad, bhi, blo);
    GNN_LAUNCH_CHECK();
    CUtensorMap ta, tbh, tbl;
    if (!map_2d_sw128(&ta, A, K, M, lda, kTcM) || !map_2d_sw128(&tbh, bhi, kpad, npad, kpad, npad) ||
        !map_2d_sw128(&tbl, blo, kpad, npad, kpad, npad))
      return GNN_ERR_UNSUPPORTED;
    TcArgs p{};
    p.M = M;
    p.N = nb;
    p.K = K;
    p.Npad = npad;
    p.nkb = (int)(kpad / kTcBK);
    p.mtiles = ceil_div(M, kTcM);
    p.C = C + n0;
    p.ldc = ldc;
    p.vec_store = 1;
    p.pal = al;
    p.par = ar;
    p.pel = el;
    p.per = er;
    p.pF = F;
    p.pn0 = n0;
    int rc;
    switch (npad) {
      case 16: rc = launch_tc<16, EPI_PROJ>(ta, tbh, tbl, p, st); break;
      case 32: rc = launch_tc<32, EPI_PROJ>(ta, tbh, tbl, p, st); break;
      case 64: rc = launch_tc<64, EPI_PROJ>(ta, tbh, tbl, p, st); break;
      default: rc = launch_tc<128, EPI_PROJ>(ta, tbh, tbl, p, st); break;
    }
    if (rc != GNN_OK) return rc;
  }
  return GNN_OK;
}

// GAT concatenated-heads backward GEMM: dYm = relu'(Y) * (A Bt^T) with the
// per-head row statistics written after each row's N columns (EPI_GAT above).
// N = 4F, F % 16 == 0, N <= 128; C rows hold N + 16 floats.
int gemm_tc_gat_relu_stat(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                          const float *Bt, int64_t ldb, float *C, int64_t ldc, const float *Y,
                          int64_t ldy, const float *bias, const float *er, const float *rowstat,
                          void *ws, size_t ws_bytes, cudaStream_t st) {
  if (N % 64 || N > 128 || ldc < N + 16 || ldc % 4 || ldy % 4 || !gemm_tc_supported(M, N, K, A, lda, 0) ||
      (reinterpret_cast<uintptr_t>(C) & 15u) || (reinterpret_cast<uintptr_t>(Y) & 15u) ||
      (reinterpret_cast<uintptr_t>(bias) & 15u))
    return GNN_ERR_UNSUPPORTED;
  const int npad = tc_npad(N);
  const int64_t kpad = ceil_div(K, kTcBK) * kTcBK;
  if (ws_bytes < gemm_tc_workspace(N, K)) return GNN_ERR_WORKSPACE;
  float *bhi = static_cast<float *>(ws);
  float *blo = bhi + (size_t)npad * kpad;
  split_b_kernel<<<(unsigned)ceil_div((int64_t)npad * kpad, 256), 256, 0, st>>>(Bt, ldb, 1, N, K, npad,
                                                                              kpad, bhi, blo);
  GNN_LAUNCH_CHECK();
  CUtensorMap ta, tbh, tbl;
  if (!map_2d_sw128(&ta, A, K, M, lda, kTcM) || !map_2d_sw128(&tbh, bhi, kpad, npad, kpad, npad) ||
      !map_2d_sw128(&tbl, blo, kpad, npad, kpad, npad))
    return GNN_ERR_UNSUPPORTED;
  TcArgs p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.Npad = npad;
  p.nkb = (int)(kpad / kTcBK);
  p.mtiles = ceil_div(M, kTcM);
  p.C = C;
  p.ldc = ldc;
  p.gY = Y;
  p.ldgy = ldy;
  p.gbias = bias;
  p.ger = er;
  p.grs = rowstat;
  return npad == 64 ? launch_tc<64, EPI_GAT>(ta, tbh, tbl, p, st) : launch_tc<128, EPI_GAT>(ta, tbh, tbl, p, st);
}

// ---- A^T B (weight gradient) on tcgen05
bool gemm_tc_tn_supported(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                          const float *B, int64_t ldb) {
  return M >= 1 && N >= 1 && K >= 256 && (lda * 4) % 16 == 0 && (ldb * 4) % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(A) & 15u) == 0 && (reinterpret_cast<uintptr_t>(B) & 15u) == 0 &&
         encode_fn() != nullptr && getenv("GNN_GEMM_NO_TC") == nullptr;
}

static int tn_nb(int64_t N) { return N <= 32 ? 32 : N <= 64 ? 64 : 128; }

static void tn_plan(int64_t M, int64_t N, int64_t K, int64_t &mtiles, int64_t &ntiles, int &nkb,
                    int &kbps, int &splits) {
  mtiles = ceil_div(M, kTcM);
  ntiles = ceil_div(N, tn_nb(N));
  nkb = (int)ceil_div(K, kTcBK);
  // Units = (m-tile, n-tile, k-split) on a persistent grid of min(units, SMs)
  // CTAs: pick the split count that minimises the busiest CTA's k-blocks
  // (e.g. 602x16 over 233K rows: 60 splits -> 300 units on 148 SMs leaves 4
  // CTAs with 3 units = 1.48x the balanced time; 59 splits -> 295 units, at
  // most 2 per CTA).  Each unit also pays ~2 k-blocks of pipeline fill and
  // accumulator handoff; ties go to fewer splits (smaller partial buffer).
  const int64_t sms = sm_count();
  const int64_t tiles = mtiles * ntiles;
  int64_t best_sp = 1, best_cost = -1;
  const int64_t max_sp = std::min<int64_t>(nkb, 4 * sms);
  for (int64_t sp = 1; sp <= max_sp; ++sp) {
    const int64_t kb_each = ceil_div((int64_t)nkb, sp);
    const int64_t sp_real = ceil_div((int64_t)nkb, kb_each);
    const int64_t units = tiles * sp_real;
    const int64_t grid = units < sms ? units : sms;
    const int64_t cost = ceil_div(units, grid) * (kb_each + 2);  // +2: per-unit fill / handoff
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best_sp = sp;
    }
  }
  kbps = (int)ceil_div((int64_t)nkb, best_sp);
  splits = (int)ceil_div(nkb, kbps);
}

size_t gemm_tc_tn_workspace(int64_t M, int64_t N, int64_t K) {
  int64_t mtiles, ntiles;
  int nkb, kbps, splits;
  tn_plan(M, N, K, mtiles, ntiles, nkb, kbps, splits);
  return sizeof(float) * (size_t)(splits * M * N) + 512;
}

template <int NB>
static int launch_tn(const CUtensorMap &ta, const CUtensorMap &tb, const TnArgs &p,
                     cudaStream_t st) {
  constexpr size_t smem = tn_smem_bytes<NB>();
  GNN_CUDA_TRY(cudaFuncSetAttribute(gemm_tc_tn_kernel<NB>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t units = p.mtiles * p.ntiles * p.splits;
  const int64_t grid = units < sm_count() ? units : sm_count();
  gemm_tc_tn_kernel<NB><<<(unsigned)grid, kTcThreads, smem, st>>>(ta, tb, p);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gemm_tc_tn(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
               int64_t ldb, float *C, int64_t ldc, void *ws, size_t ws_bytes, cudaStream_t st,
               const int64_t *rows_dev) {
  TnArgs p{};
  int kbps, splits, nkb;
  int64_t mtiles, ntiles;
  tn_plan(M, N, K, mtiles, ntiles, nkb, kbps, splits);
  if (ws_bytes < gemm_tc_tn_workspace(M, N, K)) return GNN_ERR_WORKSPACE;
  p.M = M;
  p.N = N;
  p.K = K;
  p.nkb_total = nkb;
  p.kb_per_split = kbps;
  p.splits = splits;
  p.mtiles = mtiles;
  p.ntiles = ntiles;
  p.partials = static_cast<float *>(ws);
  p.rows_dev = rows_dev;
  CUtensorMap ta, tb;
  // A [K rows, M cols] and B [K rows, N cols]: boxes of 32 cols x 32 rows (OOB zero-filled)
  // MN-major tf32 operands: the only legal smem layout is SWIZZLE_128B_BASE32B
  if (!map_2d(&ta, A, M, K, lda, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
      !map_2d(&tb, B, N, K, ldb, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
    return GNN_ERR_UNSUPPORTED;
  switch (tn_nb(N)) {
    case 32: GNN_TRY(launch_tn<32>(ta, tb, p, st)); break;
    case 64: GNN_TRY(launch_tn<64>(ta, tb, p, st)); break;
    default: GNN_TRY(launch_tn<128>(ta, tb, p, st)); break;
  }
  tn_reduce_kernel<<<(unsigned)ceil_div(M * N * 8, 256), 256, 0, st>>>(M, N, splits, p.partials, C, ldc);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

}  // namespace gnn
