// Fused wide output layer on the tensor cores (tcgen05, kind::tf32, split-TF32):
// the papers100M-shape GCN head (hidden 16 -> 172 classes) in
// one persistent kernel, the [M, C] logits never leaving the SM:
//
//   Z = P W + b  ->  softmax-xent (loss, dz = (softmax - onehot) * scale)
//   dP = dz W^T * 1/deg(row)     dW = P^T dz     db = colsum(dz)
//
// Per 128-row tile (one CTA per SM, 10 warps):
//   warp 0      TMA producer: P tile [128 x 16] fp32 (SWIZZLE_64B), 2 stages
//   warp 1      TMEM allocator (512 columns) + single-thread MMA issuer
//   warps 2-9   epilogue: two warps per TMEM lane quarter (warp % 4), thread =
//               row, half of the classes each (88 columns)
// MMAs (M = 128, split-TF32: the tensor core truncates fp32 operands to TF32,
// so a raw operand is its own hi part and only lo parts are materialised;
// x.y ~ x_raw.y_hi + x_raw.y_lo + x_lo.y_hi):
//   M1  Z[128 x 176]          = P . W^T            (A smem SW64, B smem SW64)   TMEM [0,176)
//   M2  dP[128 x 16]          = dz . W             (A = dz in TMEM, B smem)     TMEM [352,368)
//       dW^T[classes 0-127]   = dz^T . [P|1]_(hi|lo) (A smem MN-major SW128_32B: dz rows as
//                                                    written, full 128-byte lines per MMA)  TMEM [368,416)
//   M3  dW^T[classes 128-255] = dz^T . [P|1]_(hi|lo)                            TMEM [416,464)
// (dW: B = [P_hi|1 ; P_lo|0] stacked along N, so each K step is two MMAs,
// A = dz^T raw then dz^T lo, and the epilogue adds the two 24-column halves)
// The epilogue reads Z once (registers), exchanges the row max / sum with its
// partner warp, writes dz (raw, lo) back into TMEM [0,352) for M2 and dz^T
// into shared memory for the weight gradient; the ones column of the B
// operand makes column 16 of dW^T the bias gradient.  dW accumulates per tile
// in TMEM (<= 48 MMAs per chain, see gemm_tc.cu kTnChunk on the tensor cores'
// rounding) and across tiles in fp32 registers; CTA partials are reduced in a
// fixed order by gcn_head_reduce_warp_kernel (dense.cu), so results are
// deterministic.  Semantics as gcn_head_wide_kernel (dense.cu), reference
// model: SURVEY Appendix A.4 output layer, PAPER.md:1736 (172 classes).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"

namespace gnn {
namespace {

constexpr int kHtThreads = 320;  // 10 warps: 204 registers per thread
constexpr int kHtRows = 128;
constexpr int kHtHalf = 88;               // classes per epilogue half
constexpr int kHtCP = 2 * kHtHalf;        // 176: padded classes (C <= 176)
constexpr int kHtDin = 16;                // P / W rows (din <= 16, zero padded)
constexpr int kHtNW = 24;                 // [P|1] width: din 16 + ones column + 7 zero columns
constexpr int kHtNB = 2 * kHtNW;          // dW^T MMA N: [P_hi|1 | P_lo|0], 48 rows of the B operand

// shared-memory carve (bytes; every region 1024-aligned)
constexpr int kOffWfHi = 0;                               // W^T [176][16] SW64: forward B
constexpr int kOffWfLo = kOffWfHi + kHtCP * 64;           // 11264
constexpr int kOffWdHi = kOffWfLo + kHtCP * 64;           // W [16][192] SW128: dP B (6 atoms of 2 KB)
constexpr int kOffWdLo = kOffWdHi + 6 * 2048;
constexpr int kOffP = kOffWdLo + 6 * 2048;                // P raw [2 stages][128][16] SW64
constexpr int kOffPlo = kOffP + 2 * 8192;                 // P lo [128][16] SW64
constexpr int kOffPt = kOffPlo + 8192;                    // [P_hi|1 ; P_lo|0]^T [48][128] SW128: 4 atoms of 6 KB
constexpr int kPtAtom = kHtNB * 128;
constexpr int kOffDzHi = kOffPt + 4 * kPtAtom;            // dz [128 rows][128 classes] MN-major SW128_32B
constexpr int kOffDzLo = kOffDzHi + 4 * 16384;
constexpr int kOffBar = kOffDzLo + 4 * 16384;
constexpr int kOffBias = kOffBar + 256;                   // b [176]
constexpr int kOffXchg = kOffBias + kHtCP * 4;            // partner-row exchange [3][2][128]
constexpr int kOffLred = kOffXchg + 3 * 2 * 128 * 4;      // loss partials [4] (double)
// No alignment slack: the kernel has no static shared memory, so the dynamic
// buffer starts at the CTA's (1024-aligned) shared window base — checked at
// run time (a misaligned base would trap, never silently corrupt).
constexpr int kHtSmem = kOffLred + 4 * 8;
static_assert(kOffWdHi % 1024 == 0 && kOffP % 1024 == 0 && kOffPt % 1024 == 0 &&
                  kOffDzHi % 1024 == 0 && kOffBar % 8 == 0,
              "1024-aligned operand regions");
static_assert(kHtSmem <= 227 * 1024, "fits one SM");

// dW^T blocks: [dz.P_hi | dz.P_lo] halves of 24 columns, summed by the epilogue
constexpr uint32_t kTmZ = 0, kTmZlo = 176, kTmDp = 352, kTmDw0 = 368, kTmDw1 = 416;

__device__ __forceinline__ float ex2_approx(float x) {  // MUFU.EX2 (as __expf uses)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// byte offset of (row r, fp32 column k) in a K-major SWIZZLE_64B tile (64-byte rows)
__device__ __forceinline__ uint32_t sw64_off(int r, int k) {
  return (uint32_t)(r * 64 + ((((k >> 2) ^ (r >> 1)) & 3) << 4) + (k & 3) * 4);
}
// byte offset of (row r, K index k) in a K-major SWIZZLE_128B operand made of
// 32-column atoms, each atom `atom_bytes` long (rows x 128 B)
__device__ __forceinline__ uint32_t sw128_off(int r, int k, int atom_bytes) {
  return (uint32_t)((k >> 5) * atom_bytes + r * 128 + (((((k & 31) >> 2) ^ r) & 7) << 4) + (k & 3) * 4);
}

// GNN_HT_PROF builds: per-CTA phase clocks of one epilogue thread per half
// (prof[cta][half][8] accumulated cycles), read by tools/prof_head.py
#ifdef GNN_HT_PROF
#define HT_T(k)                                                      \
  do {                                                               \
    const long long now_ = clock64();                                \
    if (lane == 0 && q == 0) ht_acc[k] += now_ - ht_last;            \
    ht_last = now_;                                                  \
  } while (0)
#else
#define HT_T(k) \
  do {          \
  } while (0)
#endif

struct HeadTcArgs {
  int64_t M;
  int din, C;
  const float *W, *b;
  const int64_t *labels, *deg_offsets;
  float scale;
  float *dP;
  int64_t lddp;
  int dp_vec;       // din == 16 and 16-byte dP rows: vector stores
  float *partials;  // [grid][din*C + C]
  double *lpart;    // [grid]
  int64_t ntiles;
  long long *prof;  // GNN_HT_PROF: [grid][2][8]
};

__global__ void __launch_bounds__(kHtThreads, 1) gcn_head_tc_kernel(const __grid_constant__ CUtensorMap tmP,
                                                                   HeadTcArgs a) {
  extern __shared__ __align__(1024) uint8_t ht_raw[];
  uint8_t *sm = ht_raw;  // the window base: 1024-aligned (no static shared memory precedes it)
  if (smem_u32(ht_raw) & 1023u) __trap();
  const uint32_t sb = smem_u32(sm);
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + kOffBar);
  uint64_t *p_full = bars, *p_empty = bars + 2;                     // [2] each
  uint64_t *p_ready = bars + 4, *z_full = bars + 5, *dz0_ready = bars + 6;
  uint64_t *dzt_free = bars + 7, *dz1_ready = bars + 8, *m3_done = bars + 9, *dp_full = bars + 10;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 11);
  double *lred = reinterpret_cast<double *>(sm + kOffLred);  // [quarter]

  const int warp = threadIdx.x >> 5, lane = (int)lane_id();
  const int din = a.din, C = a.C;

  // ---- one-time setup: barriers, TMEM, the constant operands
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(p_full + s, 1);
      mbar_init(p_empty + s, 1);
    }
    mbar_init(p_ready, 8);
    mbar_init(z_full, 1);
    mbar_init(dz0_ready, 8);
    mbar_init(dzt_free, 1);
    mbar_init(dz1_ready, 4);
    mbar_init(m3_done, 1);
    mbar_init(dp_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // W^T (forward B, SW64) and W (dP B, SW128), hi / lo, zero padded; [P|1]^T rows
  // 16..23 (ones row 16 in hi, zeros elsewhere) never change
  for (int i = threadIdx.x; i < kHtCP * kHtDin; i += kHtThreads) {
    const int n = i / kHtDin, k = i % kHtDin;  // class n, input feature k
    const float w = (n < C && k < din) ? a.W[(int64_t)k * C + n] : 0.f;
    const float h = tf32_hi(w);
    *reinterpret_cast<float *>(sm + kOffWfHi + sw64_off(n, k)) = h;
    *reinterpret_cast<float *>(sm + kOffWfLo + sw64_off(n, k)) = w - h;
  }
  for (int i = threadIdx.x; i < kHtDin * 192; i += kHtThreads) {
    const int n = i / 192, k = i % 192;  // input feature n, class k
    const float w = (k < C && n < din) ? a.W[(int64_t)n * C + k] : 0.f;
    const float h = tf32_hi(w);
    *reinterpret_cast<float *>(sm + kOffWdHi + sw128_off(n, k, 2048)) = h;
    *reinterpret_cast<float *>(sm + kOffWdLo + sw128_off(n, k, 2048)) = w - h;
  }
  float *sbias = reinterpret_cast<float *>(sm + kOffBias);
  // padded classes get bias -inf: logit -inf, exp 0, dz 0 with no per-class predicates
  for (int c = threadIdx.x; c < kHtCP; c += kHtThreads) sbias[c] = c < C ? a.b[c] : -INFINITY;
  for (int i = threadIdx.x; i < 8 * kHtRows; i += kHtThreads) {
    const int n = kHtDin + i / kHtRows, r = i % kHtRows;
    *reinterpret_cast<float *>(sm + kOffPt + sw128_off(n, r, kPtAtom)) = n == kHtDin ? 1.f : 0.f;
    *reinterpret_cast<float *>(sm + kOffPt + sw128_off(kHtNW + n, r, kPtAtom)) = 0.f;
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int it = 0;
      for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
        const int s = it & 1;
        mbar_wait(p_empty + s, ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(p_full + s, kHtRows * kHtDin * 4);
        tma_load_2d(sb + kOffP + s * 8192, &tmP, 0, (int)(t * kHtRows), smem_u32(p_full + s));
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t iZ = tf32_idesc_kk(kHtCP), iP = tf32_idesc_kk(16), iW = tf32_idesc_kk(kHtNB) | (1u << 15);  // A MN-major
      const uint64_t wf_hi = sw64_desc(sb + kOffWfHi), wf_lo = sw64_desc(sb + kOffWfLo);
      const uint64_t pl = sw64_desc(sb + kOffPlo);
      int it = 0;
      for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
        const int s = it & 1;
        const uint32_t ph = (uint32_t)(it & 1);
        // M1: Z = P W^T (P raw = hi to the tensor core)
        mbar_wait(p_ready, ph);
        tc_fence_after();
        const uint64_t pr = sw64_desc(sb + kOffP + s * 8192);
#pragma unroll
        for (int j = 0; j < 2; ++j) {  // K = 16 = two 8-wide steps (+32 B)
          const uint64_t o = (uint64_t)(2 * j);
          tc_mma_tf32(tmem + kTmZ, pr + o, wf_hi + o, iZ, j);
          tc_mma_tf32(tmem + kTmZ, pr + o, wf_lo + o, iZ, 1);
          tc_mma_tf32(tmem + kTmZ, pl + o, wf_hi + o, iZ, 1);
        }
        tc_commit(z_full);
        tc_commit(p_empty + s);
        // M2: dW^T for classes 0..127 first (frees the dz^T buffer for classes
        // 128..255 sooner), then dP = dz W (A = dz raw / lo in TMEM)
        mbar_wait(dz0_ready, ph);
        tc_fence_after();
        auto dw_block = [&](uint32_t dcol) {
#pragma unroll 2
          for (int j = 0; j < kHtRows / 8; ++j) {
            // A = dz^T, MN-major (classes contiguous): K-block of 32 rows = 4 class
            // atoms of 4 KB; 8 rows per MMA = +1 KB inside the K-block
            const uint32_t ao = (uint32_t)((j >> 2) * 16384 + (j & 3) * 1024);
            const uint64_t bo = (uint64_t)(((j >> 2) * kPtAtom + (j & 3) * 32) >> 4);
            const uint64_t ah = mn_desc(sb + kOffDzHi + ao, 4096, 512, 1);
            const uint64_t al = mn_desc(sb + kOffDzLo + ao, 4096, 512, 1);
            const uint64_t bp = sw128_desc(sb + kOffPt) + bo;  // [P_hi|1 ; P_lo|0]
            tc_mma_tf32(tmem + dcol, ah, bp, iW, j);  // dz_hi.P_hi | dz_hi.P_lo
            tc_mma_tf32(tmem + dcol, al, bp, iW, 1);  // + dz_lo.P_hi | dz_lo.P_lo
          }
        };
        dw_block(kTmDw0);
        tc_commit(dzt_free);
#pragma unroll 2
        for (int j = 0; j < kHtCP / 8; ++j) {
          const uint64_t bo = (uint64_t)(((j >> 2) * 2048 + (j & 3) * 32) >> 4);
          const uint64_t wh = sw128_desc(sb + kOffWdHi) + bo, wl = sw128_desc(sb + kOffWdLo) + bo;
          tc_mma_tf32_ts(tmem + kTmDp, tmem + kTmZ + 8 * j, wh, iP, j);
          tc_mma_tf32_ts(tmem + kTmDp, tmem + kTmZ + 8 * j, wl, iP, 1);
          tc_mma_tf32_ts(tmem + kTmDp, tmem + kTmZlo + 8 * j, wh, iP, 1);
        }
        tc_commit(dp_full);
        // M3: dW^T for classes 128..255 (rows >= C of the block are never read)
        mbar_wait(dz1_ready, ph);
        tc_fence_after();
        dw_block(kTmDw1);
        tc_commit(m3_done);
      }
    }
  } else {
    // ------------------------------------------------ epilogue
    const int q = warp & 3, hlf = (warp - 2) >> 2;
    const int rr = q * 32 + lane;                    // row within the tile = TMEM lane
    const int cbase = hlf * kHtHalf;                 // this thread's classes [cbase, cbase + 88)
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    float *xchg = reinterpret_cast<float *>(sm + kOffXchg);  // [3][2][128]: max, sum, label logit
    // dz (tile row rr, class m), MN-major SWIZZLE_128B_BASE32B (the dW A operand
    // dz^T read along classes): K-block rr >> 5 (16 KB) / class atom m >> 5
    // (4 KB) / row rr & 31 (128 B) / 32-byte granule ((m >> 3) & 3) ^ (rr & 3) /
    // word m & 7.  A thread writes its classes 4 at a time (16-byte stores).
    const uint32_t dzrow = (uint32_t)((rr >> 5) * 16384 + (rr & 31) * 128);
    const int rsw = rr & 3;
    auto dz_off = [&](int m) -> uint32_t {  // byte offset of class m (m % 4 == 0)
      return dzrow + (uint32_t)((m >> 5) * 4096 + ((((m >> 3) & 3) ^ rsw) << 5) + (m & 7) * 4);
    };
    uint8_t *dzh = sm + kOffDzHi, *dzl = sm + kOffDzLo;
    float accw[17];                                  // dW^T row (class) partial: din 0..15, db
#pragma unroll
    for (int k = 0; k < 17; ++k) accw[k] = 0.f;
    const int my_class = (hlf == 0 ? 0 : 128) + rr;  // the dW^T row this thread accumulates
    double lsum = 0.0;
#ifdef GNN_HT_PROF
    long long ht_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long ht_last = clock64();
#endif
    int it = 0;
    for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
      const int s = it & 1;
      const uint32_t ph = (uint32_t)(it & 1);
      const int64_t row = t * kHtRows + rr;
      const bool valid = row < a.M;
      // ---- E1: P lo (half 0) and [P|1]^T (half 1) from the landed P tile
      mbar_wait(p_full + s, (uint32_t)((it >> 1) & 1));
      HT_T(0);
      {
        const uint8_t *pt = sm + kOffP + s * 8192;
        float p[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 v = *reinterpret_cast<const float4 *>(pt + sw64_off(rr, 4 * c));
          p[4 * c] = v.x, p[4 * c + 1] = v.y, p[4 * c + 2] = v.z, p[4 * c + 3] = v.w;
        }
        if (hlf == 0) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            *reinterpret_cast<float4 *>(sm + kOffPlo + sw64_off(rr, 4 * c)) =
                make_float4(p[4 * c] - tf32_hi(p[4 * c]), p[4 * c + 1] - tf32_hi(p[4 * c + 1]),
                            p[4 * c + 2] - tf32_hi(p[4 * c + 2]), p[4 * c + 3] - tf32_hi(p[4 * c + 3]));
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const float h = tf32_hi(p[k]);
            *reinterpret_cast<float *>(sm + kOffPt + sw128_off(k, rr, kPtAtom)) = h;
            *reinterpret_cast<float *>(sm + kOffPt + sw128_off(kHtNW + k, rr, kPtAtom)) = p[k] - h;
          }
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
      const int64_t y = valid ? __ldg(a.labels + row) : -1;
      float rs = 1.f;
      if (valid && a.deg_offsets) {
        const int64_t dg = __ldg(a.deg_offsets + row + 1) - __ldg(a.deg_offsets + row);
        rs = dg > 0 ? 1.f / (float)dg : 0.f;
      }
      HT_T(1);
      // ---- E2: logits -> softmax -> dz
      mbar_wait(z_full, ph);
      HT_T(2);
      tc_fence_after();
      float z[kHtHalf];
#pragma unroll
      for (int c0 = 0; c0 < kHtHalf; c0 += 8) {
        uint32_t v[8];
        tmem_ld8(tq + kTmZ + cbase + c0, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) z[c0 + j] = __uint_as_float(v[j]);
      }
      tmem_wait_ld();
      float zy = 0.f;
      const int yl = (y >= cbase && y < cbase + kHtHalf) ? (int)(y - cbase) : -1;  // label column here
      const bool has_y = yl >= 0;
      // 8 independent partial maxima / sums: no 88-deep dependent chains
      float m8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) m8[k] = -INFINITY;
#pragma unroll
      for (int j = 0; j < kHtHalf; ++j) {
        z[j] += sbias[cbase + j];
        m8[j & 7] = fmaxf(m8[j & 7], z[j]);
        if (j == yl) zy = z[j];
      }
      float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                       fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      const int bar_id = 1 + q;  // the two warps (same warp % 4) holding the halves of these 32 rows
      xchg[(0 * 2 + hlf) * kHtRows + rr] = mx;
      asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
      mx = fmaxf(mx, xchg[(0 * 2 + (hlf ^ 1)) * kHtRows + rr]);
      float s8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      const float mxl = mx * 1.4426950408889634f;  // exp(z - mx) = 2^(z log2e - mx log2e)
#pragma unroll
      for (int j = 0; j < kHtHalf; ++j) {
        z[j] = ex2_approx(fmaf(z[j], 1.4426950408889634f, -mxl));
        s8[j & 7] += z[j];
      }
      float se = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
      xchg[(1 * 2 + hlf) * kHtRows + rr] = se;
      xchg[(2 * 2 + hlf) * kHtRows + rr] = has_y ? zy : 0.f;
      asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
      se += xchg[(1 * 2 + (hlf ^ 1)) * kHtRows + rr];
      if (hlf == 0 && valid) {
        const float zyt = has_y ? zy : xchg[(2 * 2 + 1) * kHtRows + rr];
        lsum += (y >= 0 && y < C) ? (double)(mx + logf(se) - zyt) : (double)NAN;
      }
      const float inv = 1.f / se, sc = valid ? a.scale : 0.f;  // rows past M: dz = 0
#pragma unroll
      for (int j = 0; j < kHtHalf; ++j) z[j] = (z[j] * inv - (j == yl ? 1.f : 0.f)) * sc;  // dz
      // dz raw -> TMEM [cbase, +88), dz lo -> TMEM [176 + cbase, +88)
#pragma unroll
      for (int c0 = 0; c0 < kHtHalf; c0 += 8) {
        float lo[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) lo[j] = z[c0 + j] - tf32_hi(z[c0 + j]);
        tmem_st8(tq + kTmZ + cbase + c0, z + c0);
        tmem_st8(tq + kTmZlo + cbase + c0, lo);
      }
      // dz^T of classes 0..127 -> shared memory (the dW A operand)
      const int nb0 = hlf == 0 ? kHtHalf : 128 - kHtHalf;  // 88 or 40 classes of block 0
#pragma unroll
      for (int j = 0; j < kHtHalf; j += 4) {
        if (j < nb0) {
          const uint32_t off = dz_off(cbase + j);
          const float4 h = make_float4(tf32_hi(z[j]), tf32_hi(z[j + 1]), tf32_hi(z[j + 2]), tf32_hi(z[j + 3]));
          *reinterpret_cast<float4 *>(dzh + off) = h;
          *reinterpret_cast<float4 *>(dzl + off) =
              make_float4(z[j] - h.x, z[j + 1] - h.y, z[j + 2] - h.z, z[j + 3] - h.w);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(dz0_ready);
      // block-0 rows of these 32 tile rows written: the partner (half 1) rewrites
      // classes 0..47 of the same rows with block 1 after dzt_free.  That order
      // already follows from dz0_ready -> MMA -> dzt_free; the named barrier makes
      // it explicit to every observer (compute-sanitizer racecheck included)
#ifndef HT_NO_NAMEDBAR
      if (hlf == 0) asm volatile("bar.arrive %0, 64;" ::"r"(5 + q) : "memory");
#endif
      HT_T(3);
      // ---- E3 / E4
      if (hlf == 1) {
        mbar_wait(dzt_free, ph);
#ifndef HT_NO_NAMEDBAR
        asm volatile("bar.sync %0, 64;" ::"r"(5 + q) : "memory");
#endif
        HT_T(4);
        // classes 128..175 of dz^T into the (now free) dW A operand, re-read from
        // TMEM (dz raw / lo stay there until M1 of the next tile, which needs this
        // warp's p_ready): nothing of E2 stays live in registers across the wait
#pragma unroll
        for (int c0 = 128 - kHtHalf; c0 < kHtHalf; c0 += 8) {
          uint32_t vr[8], vl[8];
          tmem_ld8(tq + kTmZ + cbase + c0, vr);
          tmem_ld8(tq + kTmZlo + cbase + c0, vl);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; j += 4) {  // class m = cbase + c0 + j - 128 of block 1
            const uint32_t off = dz_off(cbase + c0 + j - 128);
            *reinterpret_cast<float4 *>(dzh + off) =
                make_float4(tf32_hi(__uint_as_float(vr[j])), tf32_hi(__uint_as_float(vr[j + 1])),
                            tf32_hi(__uint_as_float(vr[j + 2])), tf32_hi(__uint_as_float(vr[j + 3])));
            *reinterpret_cast<float4 *>(dzl + off) =
                make_float4(__uint_as_float(vl[j]), __uint_as_float(vl[j + 1]), __uint_as_float(vl[j + 2]),
                            __uint_as_float(vl[j + 3]));
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(dz1_ready);
        HT_T(5);
        mbar_wait(m3_done, ph);
        HT_T(6);
        tc_fence_after();
      } else {
        mbar_wait(dp_full, ph);  // dW^T block 0 and dP
        HT_T(6);
        tc_fence_after();
      }
      {
        // half 0: dP row and dW^T rows of classes 0..127; half 1: classes 128..255
        uint32_t w16[16], w8[8], u16[16], u8[8];
        const uint32_t dwc = tq + (hlf == 0 ? kTmDw0 : kTmDw1);
        tmem_ld16(dwc, w16);
        tmem_ld8(dwc + 16, w8);
        tmem_ld16(dwc + kHtNW, u16);  // the P_lo half
        tmem_ld8(dwc + kHtNW + 16, u8);
        uint32_t dp[16];
        if (hlf == 0) tmem_ld16(tq + kTmDp, dp);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) accw[k] += __uint_as_float(w16[k]) + __uint_as_float(u16[k]);
        accw[16] += __uint_as_float(w8[0]) + __uint_as_float(u8[0]);
        if (hlf == 0 && valid) {
          float *dst = a.dP + row * a.lddp;
          if (a.dp_vec) {  // 16 columns, 16-byte rows: four 128-bit stores
#pragma unroll
            for (int k = 0; k < 16; k += 4)
              *reinterpret_cast<float4 *>(dst + k) =
                  make_float4(__uint_as_float(dp[k]) * rs, __uint_as_float(dp[k + 1]) * rs,
                              __uint_as_float(dp[k + 2]) * rs, __uint_as_float(dp[k + 3]) * rs);
          } else {
#pragma unroll
            for (int k = 0; k < 16; ++k)
              if (k < din) dst[k] = __uint_as_float(dp[k]) * rs;
          }
        }
      }
      tc_fence_before();
      HT_T(7);
    }
#ifdef GNN_HT_PROF
    if (lane == 0 && q == 0 && a.prof)
      for (int k = 0; k < 8; ++k) a.prof[((int64_t)blockIdx.x * 2 + hlf) * 8 + k] = ht_acc[k];
#endif
    // ---- CTA partials: dW^T row my_class -> partials[cta][k*C + class], db at [din*C + class]
    if (my_class < C) {
      float *out = a.partials + (int64_t)blockIdx.x * ((int64_t)din * C + C);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < din) out[(int64_t)k * C + my_class] = accw[k];
      out[(int64_t)din * C + my_class] = accw[16];
    }
    if (hlf == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(kFull, lsum, o);
      if (lane == 0) lred[q] = lsum;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) a.lpart[blockIdx.x] = (lred[0] + lred[1]) + (lred[2] + lred[3]);
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                             const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                             const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn head_encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void *ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  }
  return fn;
}

}  // namespace

// Tensor-core wide head; GNN_ERR_UNSUPPORTED when the shape / layout does not
// fit it (caller falls back to the SIMT wide kernel).  grid <= nb (the
// partials rows the workspace holds).
int gcn_head_tc(int64_t M, int64_t Din, int64_t C, const float *P, int64_t ldp, const float *W,
                const float *b, const int64_t *labels, const int64_t *deg_offsets, float scale,
                float *dP, int64_t lddp, float *partials, double *lpart, int64_t nb, cudaStream_t st) {
  const char *env = getenv("GNN_HEAD_TC");  // "0": SIMT wide kernel (A/B, tests)
  const bool off = env && env[0] == '0';
  if (off || Din < 1 || Din > kHtDin || C <= 64 || C > kHtCP || (ldp * 4) % 16 ||
      (reinterpret_cast<uintptr_t>(P) & 15u) || M >= ((int64_t)1 << 31) - kHtRows)
    return GNN_ERR_UNSUPPORTED;
  EncodeFn enc = head_encode_fn();
  if (!enc) return GNN_ERR_UNSUPPORTED;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)Din, (cuuint64_t)M};
  cuuint64_t strides[1] = {(cuuint64_t)ldp * 4};
  cuuint32_t box[2] = {(cuuint32_t)kHtDin, (cuuint32_t)kHtRows};
  cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(P), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return GNN_ERR_UNSUPPORTED;
  HeadTcArgs a{};
  a.M = M;
  a.din = (int)Din;
  a.C = (int)C;
  a.W = W;
  a.b = b;
  a.labels = labels;
  a.deg_offsets = deg_offsets;
  a.scale = scale;
  a.dP = dP;
  a.lddp = lddp;
  a.dp_vec = Din == 16 && lddp % 4 == 0 && (reinterpret_cast<uintptr_t>(dP) & 15u) == 0;
  a.partials = partials;
  a.lpart = lpart;
  a.ntiles = ceil_div(M, (int64_t)kHtRows);
#ifdef GNN_HT_PROF
  {
    static long long *prof = nullptr;
    if (!prof) cudaMalloc(&prof, sizeof(long long) * 2 * 8 * 1024);
    a.prof = prof;
    const char *dump = getenv("GNN_HT_PROF_DUMP");
    if (dump) {  // previous call's clocks -> file (debug builds only)
      static long long h[2 * 8 * 1024];
      cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost);
      if (FILE *f = fopen(dump, "w")) {
        for (int i = 0; i < 2 * 8 * 148; ++i) fprintf(f, "%lld%c", h[i], (i % 8 == 7) ? '\n' : ' ');
        fclose(f);
      }
    }
  }
#endif
  const int64_t grid = a.ntiles < nb ? a.ntiles : nb;
  GNN_CUDA_TRY(cudaFuncSetAttribute(gcn_head_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kHtSmem));
  gcn_head_tc_kernel<<<(unsigned)grid, kHtThreads, kHtSmem, st>>>(tm, a);
  GNN_LAUNCH_CHECK();
  // CTAs past the tile count (grid < nb) leave their partial rows untouched: zero them
  if (grid < nb) {
    GNN_CUDA_TRY(cudaMemsetAsync(partials + grid * (Din * C + C), 0,
                                 sizeof(float) * (size_t)((nb - grid) * (Din * C + C)), st));
    GNN_CUDA_TRY(cudaMemsetAsync(lpart + grid, 0, sizeof(double) * (size_t)(nb - grid), st));
  }
  return GNN_OK;
}

}  // namespace gnn
