// Dense pieces of the path: fp32 GEMM for the X.W transforms (SIMT fallback
// used where the tcgen05 kernel does not apply), split-K weight gradients, and
// deterministic column sums (bias gradients).
#include "common.cuh"

namespace gnn {
namespace {

constexpr int kGemmRows = 256;  // rows of C per CTA (one per thread)
constexpr int kGemmBK = 32;

// C[m, n0:n0+NT] for one row per thread; A tile staged through shared memory
// (coalesced either orientation), B tile broadcast from shared memory.
template <int NT>
__global__ void __launch_bounds__(kGemmRows) gemm_rowtile_kernel(
    int64_t M, int64_t N, int64_t Kd, const float *__restrict__ A, int64_t lda, int trans_a,
    const float *__restrict__ B, int64_t ldb, int trans_b, float *__restrict__ C, int64_t ldc,
    const float *__restrict__ bias, int relu, int64_t k_per_split, float *partials) {
  __shared__ float As[kGemmRows][kGemmBK + 1];
  __shared__ __align__(16) float Bs[kGemmBK][NT];
  const int tid = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.x * kGemmRows;
  const int64_t n0 = (int64_t)blockIdx.y * NT;
  const int64_t kbeg = (int64_t)blockIdx.z * k_per_split;
  const int64_t kend = min(Kd, kbeg + k_per_split);
  float acc[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j] = 0.f;

  for (int64_t k0 = kbeg; k0 < kend; k0 += kGemmBK) {
    // ---- A tile: rows m0..m0+255, k0..k0+31
    if (!trans_a) {
#pragma unroll 4
      for (int i = 0; i < kGemmBK; ++i) {
        int idx = i * kGemmRows + tid;
        int r = idx / kGemmBK, k = idx % kGemmBK;
        int64_t gm = m0 + r, gk = k0 + k;
        As[r][k] = (gm < M && gk < kend) ? A[gm * lda + gk] : 0.f;
      }
    } else {
#pragma unroll 4
      for (int i = 0; i < kGemmBK; ++i) {
        int64_t gm = m0 + tid, gk = k0 + i;
        As[tid][i] = (gm < M && gk < kend) ? A[gk * lda + gm] : 0.f;
      }
    }
    // ---- B tile: k0..k0+31, n0..n0+NT-1
    for (int idx = tid; idx < kGemmBK * NT; idx += kGemmRows) {
      int k = idx / NT, n = idx % NT;
      int64_t gk = k0 + k, gn = n0 + n;
      float v = 0.f;
      if (gk < kend && gn < N) v = trans_b ? B[gn * ldb + gk] : B[gk * ldb + gn];
      Bs[k][n] = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < kGemmBK; ++k) {
      float a = As[tid][k];
#pragma unroll
      for (int j = 0; j < NT; j += 4) {
        float4 b = *reinterpret_cast<const float4 *>(&Bs[k][j]);
        acc[j] = fmaf(a, b.x, acc[j]);
        acc[j + 1] = fmaf(a, b.y, acc[j + 1]);
        acc[j + 2] = fmaf(a, b.z, acc[j + 2]);
        acc[j + 3] = fmaf(a, b.w, acc[j + 3]);
      }
    }
    __syncthreads();
  }
  const int64_t m = m0 + tid;
  if (m >= M) return;
  if (partials) {
    float *p = partials + ((int64_t)blockIdx.z * M + m) * N;
#pragma unroll
    for (int j = 0; j < NT; ++j)
      if (n0 + j < N) p[n0 + j] = acc[j];
    return;
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    int64_t n = n0 + j;
    if (n < N) {
      float v = acc[j];
      if (bias) v += bias[n];
      if (relu) v = fmaxf(v, 0.f);
      C[m * ldc + n] = v;
    }
  }
}

__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int64_t splits,
                                     const float *__restrict__ partials, float *C, int64_t ldc,
                                     const float *__restrict__ bias, int relu) {
  const int64_t total = M * N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = t / N, n = t % N;
    float s = 0.f;
    for (int64_t z = 0; z < splits; ++z) s += partials[z * total + t];
    if (bias) s += bias[n];
    if (relu) s = fmaxf(s, 0.f);
    C[m * ldc + n] = s;
  }
}

struct GemmShape {
  int nt;
  int64_t mtiles, ntiles, splits, k_per_split;
};

GemmShape gemm_shape(int64_t M, int64_t N, int64_t Kd) {
  GemmShape g;
  g.nt = N <= 16 ? 16 : (N <= 32 ? 32 : 64);
  g.mtiles = ceil_div(M, kGemmRows);
  g.ntiles = ceil_div(N, g.nt);
  int64_t ctas = g.mtiles * g.ntiles;
  int64_t want = 2 * (int64_t)sm_count();
  g.splits = 1;
  if (ctas < want && Kd >= 4 * kGemmBK) {
    g.splits = ceil_div(want, ctas);
    int64_t max_splits = ceil_div(Kd, 4 * kGemmBK);
    if (g.splits > max_splits) g.splits = max_splits;
  }
  g.k_per_split = ceil_div(ceil_div(Kd, g.splits), kGemmBK) * kGemmBK;
  g.splits = ceil_div(Kd, g.k_per_split);
  if (g.splits < 1) g.splits = 1;
  return g;
}

// Rows per CTA of the column-sum style reductions: enough CTAs to fill every
// SM ~4 times (a fixed 2-4K-row block left a Reddit-size [V,64] pass on ~60-110
// CTAs), at most 4096 rows so the partial buffer stays small.
int64_t reduce_rows_per_block(int64_t M) {
  const int64_t target = 4 * (int64_t)sm_count();
  int64_t r = ceil_div(M > 0 ? M : 1, target);
  r = ceil_div(r, 64) * 64;
  return r < 64 ? 64 : (r > 4096 ? 4096 : r);
}

__global__ void colsum_partial_kernel(int64_t M, int64_t N, const float *__restrict__ X,
                                      int64_t ldx, float *partials, int64_t rpb) {
  // block b sums rows [b*rpb, ...) for every column; threads stride columns
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int64_t r1 = min(M, r0 + rpb);
  for (int64_t c = threadIdx.x; c < N; c += blockDim.x) {
    float s = 0.f;
    for (int64_t r = r0; r < r1; ++r) s += X[r * ldx + c];
    partials[(int64_t)blockIdx.x * N + c] = s;
  }
}
// narrow N: threads cover (row-slot, column) pairs, then a fixed-order smem reduction
template <int NCOL>
__global__ void __launch_bounds__(256) colsum_narrow_kernel(int64_t M, int64_t N,
                                                            const float *__restrict__ X,
                                                            int64_t ldx, float *partials,
                                                            int64_t rpb) {
  constexpr int SLOTS = 256 / NCOL;
  __shared__ float red[SLOTS][NCOL];
  const int c = threadIdx.x % NCOL, s = threadIdx.x / NCOL;
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int64_t r1 = min(M, r0 + rpb);
  float acc = 0.f;
  if (c < N)
#pragma unroll 4
    for (int64_t r = r0 + s; r < r1; r += SLOTS) acc += X[r * ldx + c];
  red[s][c] = acc;
  __syncthreads();
  if (s == 0 && c < N) {
    float t = 0.f;
    for (int k = 0; k < SLOTS; ++k) t += red[k][c];
    partials[(int64_t)blockIdx.x * N + c] = t;
  }
}
// warp per column, fixed-order butterfly (see sum_partials_kernel)
__global__ void colsum_final_kernel(int64_t nb, int64_t N, const float *__restrict__ partials,
                                    float *out) {
  const int lane = (int)(threadIdx.x & 31);
  for (int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; c < N;
       c += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    float s = 0.f;
    for (int64_t b = lane; b < nb; b += 32) s += partials[b * N + c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[c] = s;
  }
}

}  // namespace

// fused tensor-core wide output layer (head_tc.cu)
int gcn_head_tc(int64_t M, int64_t Din, int64_t C, const float *P, int64_t ldp, const float *W,
                const float *b, const int64_t *labels, const int64_t *deg_offsets, float scale,
                float *dP, int64_t lddp, float *partials, double *lpart, int64_t nb, cudaStream_t st);
// tcgen05 tensor-core path (gemm_tc.cu)
bool gemm_tc_supported(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, int trans_a);
size_t gemm_tc_workspace(int64_t N, int64_t K);
int gemm_tc_gat_proj(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
                     int64_t ldb, float *C, int64_t ldc, int F, const float *al, const float *ar,
                     float *el, float *er, void *ws, size_t ws_bytes, cudaStream_t st);
int gemm_tc_gat_relu_stat(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                          const float *Bt, int64_t ldb, float *C, int64_t ldc, const float *Y,
                          int64_t ldy, const float *bias, const float *er, const float *rowstat,
                          void *ws, size_t ws_bytes, cudaStream_t st);
int gemm_tc(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
            int64_t ldb, int trans_b, float *C, int64_t ldc, const float *bias, int relu, void *ws,
            size_t ws_bytes, cudaStream_t st, const int64_t *rows_dev = nullptr);

bool gemm_tc_tn_supported(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                          const float *B, int64_t ldb);
size_t gemm_tc_tn_workspace(int64_t M, int64_t N, int64_t K);
int gemm_tc_tn(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, const float *B,
               int64_t ldb, float *C, int64_t ldc, void *ws, size_t ws_bytes, cudaStream_t st,
               const int64_t *rows_dev = nullptr);

// SIMT fallback (transposed A, unaligned strides, small M).
int gemm_simt(int64_t M, int64_t N, int64_t Kd, const float *A, int64_t lda, int trans_a,
              const float *B, int64_t ldb, int trans_b, float *C, int64_t ldc, const float *bias,
              int relu, void *ws, size_t ws_bytes, cudaStream_t st) {
  GemmShape g = gemm_shape(M, N, Kd);
  float *partials = nullptr;
  if (g.splits > 1) {
    if (ws_bytes < sizeof(float) * (size_t)(g.splits * M * N)) return GNN_ERR_WORKSPACE;
    partials = static_cast<float *>(ws);
  }
  dim3 grid((unsigned)g.mtiles, (unsigned)g.ntiles, (unsigned)g.splits);
#define GNN_GEMM_LAUNCH(NT)                                                                    \
  gemm_rowtile_kernel<NT><<<grid, kGemmRows, 0, st>>>(M, N, Kd, A, lda, trans_a, B, ldb,       \
                                                      trans_b, C, ldc, bias, relu,             \
                                                      g.k_per_split, partials)
  if (g.nt == 16)
    GNN_GEMM_LAUNCH(16);
  else if (g.nt == 32)
    GNN_GEMM_LAUNCH(32);
  else
    GNN_GEMM_LAUNCH(64);
#undef GNN_GEMM_LAUNCH
  GNN_LAUNCH_CHECK();
  if (partials) {
    int64_t total = M * N;
    int64_t nblk = ceil_div(total, 256), cap = (int64_t)sm_count() * 8;
    unsigned blocks = (unsigned)(nblk < cap ? nblk : cap);
    splitk_reduce_kernel<<<blocks, 256, 0, st>>>(M, N, g.splits, partials, C, ldc, bias, relu);
    GNN_LAUNCH_CHECK();
  }
  return GNN_OK;
}

size_t gemm_simt_workspace(int64_t M, int64_t N, int64_t Kd) {
  GemmShape g = gemm_shape(M, N, Kd);
  return g.splits > 1 ? sizeof(float) * (size_t)(g.splits * M * N) + 256 : 256;
}

}  // namespace gnn

using namespace gnn;

extern "C" {

size_t gnn_colsum_workspace(int64_t M, int64_t N) {
  return sizeof(float) * (size_t)(ceil_div(M > 0 ? M : 1, reduce_rows_per_block(M)) * (N > 0 ? N : 1)) + 256;
}

int gnn_colsum(int64_t M, int64_t N, const float *X, int64_t ldx, float *out, void *ws,
               size_t ws_bytes, gnn_stream_t stream) {
  if (M < 0 || N < 0 || ldx < N || (N > 0 && !out) || (M > 0 && N > 0 && !X))
    return GNN_ERR_INVALID_ARGUMENT;
  if (N == 0) return GNN_OK;
  if (ws_bytes < gnn_colsum_workspace(M, N)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  if (M == 0) {
    GNN_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float) * N, st));
    return GNN_OK;
  }
  const int64_t rpb = reduce_rows_per_block(M);
  int64_t nb = ceil_div(M, rpb);
  float *partials = static_cast<float *>(ws);
  if (N <= 16)
    colsum_narrow_kernel<16><<<(unsigned)nb, 256, 0, st>>>(M, N, X, ldx, partials, rpb);
  else if (N <= 64)
    colsum_narrow_kernel<64><<<(unsigned)nb, 256, 0, st>>>(M, N, X, ldx, partials, rpb);
  else
    colsum_partial_kernel<<<(unsigned)nb, 256, 0, st>>>(M, N, X, ldx, partials, rpb);
  GNN_LAUNCH_CHECK();
  colsum_final_kernel<<<(unsigned)ceil_div(N * 32, (int64_t)256), 256, 0, st>>>(nb, N, partials, out);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

size_t gnn_gemm_workspace(int64_t M, int64_t N, int64_t Kd, int trans_a) {
  size_t a = gemm_simt_workspace(M, N, Kd);
  size_t b = trans_a ? gemm_tc_tn_workspace(M, N, Kd) : gemm_tc_workspace(N, Kd);
  return a > b ? a : b;
}

// rows_dev: live row count on device (the rows of C for the plain form, the
// contraction rows for A^T B); tensor-core paths only.
static int gemm_impl(int64_t M, int64_t N, int64_t Kd, const float *A, int64_t lda, int trans_a,
                     const float *B, int64_t ldb, int trans_b, float *C, int64_t ldc,
                     const float *bias, int relu, void *ws, size_t ws_bytes, cudaStream_t st,
                     const int64_t *rows_dev) {
  if (M < 0 || N < 0 || Kd < 0 || (M > 0 && N > 0 && (!C || ldc < N)) ||
      (M > 0 && Kd > 0 && (!A || (trans_a ? lda < M : lda < Kd))) ||
      (N > 0 && Kd > 0 && (!B || (trans_b ? ldb < Kd : ldb < N))))
    return GNN_ERR_INVALID_ARGUMENT;
  if (M == 0 || N == 0) return GNN_OK;
  if (gemm_tc_supported(M, N, Kd, A, lda, trans_a))
    return gemm_tc(M, N, Kd, A, lda, B, ldb, trans_b, C, ldc, bias, relu, ws, ws_bytes, st, rows_dev);
  if (N > 128 && gemm_tc_supported(M, 128, Kd, A, lda, trans_a)) {
    // wide outputs (e.g. GAT's heads x classes): 128-column slabs, A re-streamed per slab
    for (int64_t n0 = 0; n0 < N; n0 += 128) {
      const int64_t nb = N - n0 < 128 ? N - n0 : 128;
      GNN_TRY(gemm_tc(M, nb, Kd, A, lda, trans_b ? B + n0 * ldb : B + n0, ldb, trans_b, C + n0,
                      ldc, bias ? bias + n0 : nullptr, relu, ws, ws_bytes, st, rows_dev));
    }
    return GNN_OK;
  }
  if (trans_a && !trans_b && !bias && !relu && gemm_tc_tn_supported(M, N, Kd, A, lda, B, ldb))
    return gemm_tc_tn(M, N, Kd, A, lda, B, ldb, C, ldc, ws, ws_bytes, st, rows_dev);
  if (rows_dev) return GNN_ERR_UNSUPPORTED;
  return gemm_simt(M, N, Kd, A, lda, trans_a, B, ldb, trans_b, C, ldc, bias, relu, ws, ws_bytes,
                   st);
}

int gnn_gemm_gat_proj(int64_t M, int64_t N, int64_t Kd, const float *A, int64_t lda,
                      const float *B, int64_t ldb, float *C, int64_t ldc, int64_t F,
                      const float *a_l, const float *a_r, float *el, float *er, void *ws,
                      size_t ws_bytes, gnn_stream_t stream) {
  if (M < 0 || N <= 0 || Kd <= 0 || F <= 0 || !A || !B || !C || !a_l || !a_r || !el || !er ||
      ldb < N || ldc < N)
    return GNN_ERR_INVALID_ARGUMENT;
  if (M == 0) return GNN_OK;
  return gemm_tc_gat_proj(M, N, Kd, A, lda, B, ldb, C, ldc, (int)F, a_l, a_r, el, er, ws,
                          ws_bytes, as_stream(stream));
}

int gnn_gemm_gat_relu_stat(int64_t M, int64_t N, int64_t Kd, const float *A, int64_t lda,
                           const float *Bt, int64_t ldb, float *C, int64_t ldc, const float *Y,
                           int64_t ldy, const float *bias, const float *er, const float *rowstat,
                           void *ws, size_t ws_bytes, gnn_stream_t stream) {
  if (M < 0 || N <= 0 || Kd <= 0 || !A || !Bt || !C || !Y || !bias || !er || !rowstat ||
      ldb < Kd || ldy < N)
    return GNN_ERR_INVALID_ARGUMENT;
  if (M == 0) return GNN_OK;
  return gemm_tc_gat_relu_stat(M, N, Kd, A, lda, Bt, ldb, C, ldc, Y, ldy, bias, er, rowstat, ws,
                               ws_bytes, as_stream(stream));
}

int gnn_gemm(int64_t M, int64_t N, int64_t Kd, const float *A, int64_t lda, int trans_a,
             const float *B, int64_t ldb, int trans_b, float *C, int64_t ldc, const float *bias,
             int relu, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  return gemm_impl(M, N, Kd, A, lda, trans_a, B, ldb, trans_b, C, ldc, bias, relu, ws, ws_bytes,
                   as_stream(stream), nullptr);
}

int gnn_gemm_rows_dev(int64_t M, int64_t N, int64_t Kd, const float *A, int64_t lda, int trans_a,
                      const float *B, int64_t ldb, int trans_b, float *C, int64_t ldc,
                      const float *bias, int relu, const int64_t *rows_dev, void *ws,
                      size_t ws_bytes, gnn_stream_t stream) {
  if (!rows_dev) return GNN_ERR_INVALID_ARGUMENT;
  return gemm_impl(M, N, Kd, A, lda, trans_a, B, ldb, trans_b, C, ldc, bias, relu, ws, ws_bytes,
                   as_stream(stream), rows_dev);
}

}  // extern "C"

// ------------------------------------------------------------------------
// Fused row-wise helpers of the GNN layers' backward pass and loss.
namespace gnn {
namespace {


__device__ __forceinline__ float inv_deg_of(const int64_t *off, int64_t r) {
  int64_t d = off[r + 1] - off[r];
  return d > 0 ? 1.0f / (float)d : 0.0f;
}

// out = (mask>0 ? X : 0) * (1/deg(row) if deg_offsets); colsum partials of the
// masked, un-normalised values (the bias gradient).  Threads: (slot, column).
template <int NCOL>
__global__ void __launch_bounds__(256) mask_norm_colsum_kernel(
    int64_t M, int64_t N, const float *__restrict__ X, int64_t ldx, const float *__restrict__ mask,
    int64_t ldm, const int64_t *__restrict__ deg_offsets, float *out, int64_t ldo,
    float *partials, int64_t rpb, const int64_t *m_dev = nullptr) {
  if (m_dev) M = min(M, *m_dev);  // live rows (replayed mini-batch)
  constexpr int SLOTS = 256 / NCOL;
  __shared__ float red[SLOTS][NCOL];
  const int s = threadIdx.x / NCOL;
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int64_t r1 = min(M, r0 + rpb);
  for (int64_t c0 = 0; c0 < N; c0 += NCOL) {
    const int64_t c = c0 + threadIdx.x % NCOL;
    float acc = 0.f;
    if (c < N) {
#pragma unroll 4
      for (int64_t r = r0 + s; r < r1; r += SLOTS) {
        float v = X[r * ldx + c];
        if (mask && !(mask[r * ldm + c] > 0.f)) v = 0.f;
        acc += v;
        if (out) out[r * ldo + c] = deg_offsets ? v * inv_deg_of(deg_offsets, r) : v;
      }
    }
    red[s][threadIdx.x % NCOL] = acc;
    __syncthreads();
    if (s == 0 && c < N && partials) {
      float t = 0.f;
      for (int k = 0; k < SLOTS; ++k) t += red[k][threadIdx.x % NCOL];
      partials[(int64_t)blockIdx.x * N + c] = t;
    }
    __syncthreads();
  }
}

// float4 form (N % 4 == 0, 16-byte rows): a thread owns 4 columns of a row,
// so the row's 1/deg is computed once per 4 values instead of per value.
template <int C4P>
__global__ void __launch_bounds__(256) mask_norm_colsum_vec_kernel(
    int64_t M, int64_t N, const float *__restrict__ X, int64_t ldx, const float *__restrict__ mask,
    int64_t ldm, const int64_t *__restrict__ deg_offsets, float *out, int64_t ldo,
    float *partials, int64_t rpb, const int64_t *m_dev = nullptr) {
  if (m_dev) M = min(M, *m_dev);  // live rows (replayed mini-batch)
  constexpr int SLOTS = 256 / C4P;
  __shared__ float4 red[SLOTS][C4P];
  const int s = threadIdx.x / C4P, q = threadIdx.x % C4P;
  const int64_t n4 = N / 4;
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int64_t r1 = min(M, r0 + rpb);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (q < n4) {
#pragma unroll 4
    for (int64_t r = r0 + s; r < r1; r += SLOTS) {
      float4 v = *reinterpret_cast<const float4 *>(X + r * ldx + 4 * q);
      if (mask) {
        const float4 m = *reinterpret_cast<const float4 *>(mask + r * ldm + 4 * q);
        v = make_float4(m.x > 0.f ? v.x : 0.f, m.y > 0.f ? v.y : 0.f, m.z > 0.f ? v.z : 0.f,
                        m.w > 0.f ? v.w : 0.f);
      }
      acc = make_float4(acc.x + v.x, acc.y + v.y, acc.z + v.z, acc.w + v.w);
      if (out) {
        const float w = deg_offsets ? inv_deg_of(deg_offsets, r) : 1.f;
        *reinterpret_cast<float4 *>(out + r * ldo + 4 * q) = make_float4(v.x * w, v.y * w, v.z * w, v.w * w);
      }
    }
  }
  red[s][q] = acc;
  __syncthreads();
  if (s == 0 && q < n4 && partials) {
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < SLOTS; ++k) {
      const float4 a = red[k][q];
      t = make_float4(t.x + a.x, t.y + a.y, t.z + a.z, t.w + a.w);
    }
    *reinterpret_cast<float4 *>(partials + (int64_t)blockIdx.x * N + 4 * q) = t;
  }
}

// out[c] = sum_b partials[b*N + c]: one warp per column, lanes stride the
// partials, fixed-order butterfly (deterministic).  A thread-per-column loop
// over ~500 partials was a 46 us chain of dependent loads for N = 16.
__global__ void sum_partials_kernel(int64_t nb, int64_t N, const float *__restrict__ partials,
                                    float *out) {
  const int lane = (int)(threadIdx.x & 31);
  for (int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; c < N;
       c += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    float s = 0.f;
    for (int64_t b = lane; b < nb; b += 32) s += partials[b * N + c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[c] = s;
  }
}

// One warp per row: numerically stable log-softmax cross-entropy; writes
// dlogits = (softmax - onehot) * scale and a per-CTA partial of the loss.
// Warp per row; the row's logits are loaded once into registers (NPL per
// lane, C <= 32*NPL) and max, sum, loss and dZ are computed from them (one
// memory round trip per row instead of three).
template <int NPL>
__global__ void __launch_bounds__(256) softmax_xent_kernel(int64_t M, int64_t C,
                                                           const float *__restrict__ Z,
                                                           int64_t ldz,
                                                           const int64_t *__restrict__ labels,
                                                           float scale, float *dZ, int64_t ldd,
                                                           float *loss_partials) {
  __shared__ float wl[8];
  const int warp = threadIdx.x >> 5, lane = (int)lane_id();
  float lsum = 0.f;
  const int64_t rows_per_cta = 8 * 16;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  // the next row's logits and label are loaded before this row is reduced, so a
  // warp's 16 rows cost one memory round trip each only at the start
  const int64_t r_end = min(M, r0 + rows_per_cta);
  float vn[NPL];
  int64_t yn = 0;
  auto load_row = [&](int64_t r) {
    yn = r < r_end ? __ldg(labels + r) : 0;
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int64_t c = lane + 32 * j;
      vn[j] = (r < r_end && c < C) ? __ldg(Z + r * ldz + c) : -INFINITY;
    }
  };
  load_row(r0 + warp);
  for (int64_t r = r0 + warp; r < r_end; r += 8) {
    float v[NPL];
#pragma unroll
    for (int j = 0; j < NPL; ++j) v[j] = vn[j];
    const int64_t y = yn;
    load_row(r + 8);
    float mx = v[0];
#pragma unroll
    for (int j = 1; j < NPL; ++j) mx = fmaxf(mx, v[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
    float se = 0.f, zy = 0.f;
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
      const int64_t c = lane + 32 * j;
      if (c < C) se += expf(v[j] - mx);
      if (c == y) zy = v[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      se += __shfl_xor_sync(kFull, se, o);
      zy += __shfl_xor_sync(kFull, zy, o);
    }
    const float lse = mx + logf(se);
    // a label outside [0, C) poisons the loss (NaN) instead of reading past the row
    if (lane == 0) lsum += (y >= 0 && y < C) ? lse - zy : NAN;
    if (dZ) {
#pragma unroll
      for (int j = 0; j < NPL; ++j) {
        const int64_t c = lane + 32 * j;
        if (c < C) dZ[r * ldd + c] = (expf(v[j] - lse) - (c == y ? 1.f : 0.f)) * scale;
      }
    }
  }
  if (lane == 0) wl[warp] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += wl[k];
    loss_partials[blockIdx.x] = t;
  }
}

// wide C (> 256): three passes over global memory
__global__ void __launch_bounds__(256) softmax_xent_wide_kernel(int64_t M, int64_t C,
                                                                const float *__restrict__ Z,
                                                                int64_t ldz,
                                                                const int64_t *__restrict__ labels,
                                                                float scale, float *dZ, int64_t ldd,
                                                                float *loss_partials) {
  __shared__ float wl[8];
  const int warp = threadIdx.x >> 5, lane = (int)lane_id();
  float lsum = 0.f;
  const int64_t rows_per_cta = 8 * 16;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  for (int64_t r = r0 + warp; r < min(M, r0 + rows_per_cta); r += 8) {
    const float *z = Z + r * ldz;
    float mx = -INFINITY;
    for (int64_t c = lane; c < C; c += 32) mx = fmaxf(mx, z[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
    float se = 0.f;
    for (int64_t c = lane; c < C; c += 32) se += expf(z[c] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(kFull, se, o);
    const float lse = mx + logf(se);
    const int64_t y = labels[r];
    if (lane == 0) lsum += (y >= 0 && y < C) ? lse - z[y] : NAN;  // bad label -> NaN loss, no OOB read
    if (dZ) {
      for (int64_t c = lane; c < C; c += 32) {
        float p = expf(z[c] - lse);
        dZ[r * ldd + c] = (p - (c == y ? 1.f : 0.f)) * scale;
      }
    }
  }
  if (lane == 0) wl[warp] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += wl[k];
    loss_partials[blockIdx.x] = t;
  }
}

__global__ void loss_final_kernel(int64_t nb, const float *__restrict__ partials, float scale,
                                  float *loss) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < nb; i += 256) s += (double)partials[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = (float)(red[0] * (double)scale);
}

struct AdamParam {
  float *p;
  const float *g;
  float *m;
  float *v;
  int64_t n;
};

// Step count lives on device so a captured CUDA graph replays correctly.
__global__ void adam_kernel(const AdamParam *__restrict__ params, int nparams, float lr,
                            float beta1, float beta2, float eps, float weight_decay,
                            const int64_t *__restrict__ step) {
  const float t = (float)(*step + 1);
  const float bc1 = 1.f - powf(beta1, t), bc2 = 1.f - powf(beta2, t);
  for (int i = blockIdx.y; i < nparams; i += gridDim.y) {
    AdamParam P = params[i];
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P.n;
         j += (int64_t)gridDim.x * blockDim.x) {
      float g = P.g[j] + weight_decay * P.p[j];
      float m = beta1 * P.m[j] + (1.f - beta1) * g;
      float v = beta2 * P.v[j] + (1.f - beta2) * g * g;
      P.m[j] = m;
      P.v[j] = v;
      P.p[j] -= lr * (m / bc1) / (sqrtf(v / bc2) + eps);
    }
  }
}

__global__ void step_increment_kernel(int64_t *step) { *step += 1; }

}  // namespace
}  // namespace gnn

extern "C" {

size_t gnn_mask_norm_colsum_workspace(int64_t M, int64_t N) {
  return sizeof(float) * (size_t)(ceil_div(M > 0 ? M : 1, reduce_rows_per_block(M)) * (N > 0 ? N : 1)) + 256;
}

static int mask_norm_colsum_impl(int64_t M, int64_t N, const float *X, int64_t ldx, const float *mask,
                         int64_t ldm, const int64_t *deg_offsets, float *out, int64_t ldo,
                         float *colsum, void *ws, size_t ws_bytes, gnn_stream_t stream,
                                 const int64_t *m_dev) {
  if (M < 0 || N <= 0 || ldx < N || (mask && ldm < N) || (out && ldo < N) || (M > 0 && !X))
    return GNN_ERR_INVALID_ARGUMENT;
  if (colsum && ws_bytes < gnn_mask_norm_colsum_workspace(M, N)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  if (M == 0) {
    if (colsum) GNN_CUDA_TRY(cudaMemsetAsync(colsum, 0, sizeof(float) * N, st));
    return GNN_OK;
  }
  const int64_t rpb = reduce_rows_per_block(M);
  const int64_t nb = ceil_div(M, rpb);
  float *partials = colsum ? static_cast<float *>(ws) : nullptr;
  const auto al16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  const bool vec = N % 4 == 0 && N <= 64 && ldx % 4 == 0 && al16(X) &&
                   (!mask || (ldm % 4 == 0 && al16(mask))) && (!out || (ldo % 4 == 0 && al16(out))) &&
                   (!partials || al16(partials));
  if (vec) {
    if (N <= 16)
      mask_norm_colsum_vec_kernel<4><<<(unsigned)nb, 256, 0, st>>>(M, N, X, ldx, mask, ldm,
                                                                   deg_offsets, out, ldo, partials, rpb, m_dev);
    else if (N <= 32)
      mask_norm_colsum_vec_kernel<8><<<(unsigned)nb, 256, 0, st>>>(M, N, X, ldx, mask, ldm,
                                                                   deg_offsets, out, ldo, partials, rpb, m_dev);
    else
      mask_norm_colsum_vec_kernel<16><<<(unsigned)nb, 256, 0, st>>>(M, N, X, ldx, mask, ldm,
                                                                    deg_offsets, out, ldo, partials, rpb, m_dev);
  } else if (N <= 16)
    mask_norm_colsum_kernel<16><<<(unsigned)nb, 256, 0, st>>>(M, N, X, ldx, mask, ldm,
                                                             deg_offsets, out, ldo, partials, rpb, m_dev);
  else if (N <= 64)
    mask_norm_colsum_kernel<64><<<(unsigned)nb, 256, 0, st>>>(M, N, X, ldx, mask, ldm,
                                                             deg_offsets, out, ldo, partials, rpb, m_dev);
  else
    mask_norm_colsum_kernel<256><<<(unsigned)nb, 256, 0, st>>>(M, N, X, ldx, mask, ldm,
                                                              deg_offsets, out, ldo, partials, rpb, m_dev);
  GNN_LAUNCH_CHECK();
  if (colsum) {
    sum_partials_kernel<<<(unsigned)ceil_div(N * 32, (int64_t)256), 256, 0, st>>>(nb, N, partials,
                                                                                colsum);
    GNN_LAUNCH_CHECK();
  }
  return GNN_OK;
}

int gnn_mask_norm_colsum(int64_t M, int64_t N, const float *X, int64_t ldx, const float *mask,
                         int64_t ldm, const int64_t *deg_offsets, float *out, int64_t ldo,
                         float *colsum, void *ws, size_t ws_bytes, gnn_stream_t stream) {
  return mask_norm_colsum_impl(M, N, X, ldx, mask, ldm, deg_offsets, out, ldo, colsum, ws, ws_bytes,
                               stream, nullptr);
}

int gnn_mask_norm_colsum_dev(int64_t M, int64_t N, const float *X, int64_t ldx, const float *mask,
                             int64_t ldm, const int64_t *deg_offsets, float *out, int64_t ldo,
                             float *colsum, const int64_t *m_dev, void *ws, size_t ws_bytes,
                             gnn_stream_t stream) {
  if (!m_dev) return GNN_ERR_INVALID_ARGUMENT;
  return mask_norm_colsum_impl(M, N, X, ldx, mask, ldm, deg_offsets, out, ldo, colsum, ws, ws_bytes,
                               stream, m_dev);
}

size_t gnn_softmax_xent_workspace(int64_t M) {
  return sizeof(float) * (size_t)ceil_div(M > 0 ? M : 1, 128) + 256;
}

int gnn_softmax_xent(int64_t M, int64_t C, const float *Z, int64_t ldz, const int64_t *labels,
                     float grad_scale, float *dZ, int64_t ldd, float *loss, void *ws,
                     size_t ws_bytes, gnn_stream_t stream) {
  if (M <= 0 || C <= 0 || !Z || ldz < C || !labels || !loss || (dZ && ldd < C))
    return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_softmax_xent_workspace(M)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  const int64_t nb = ceil_div(M, 128);
  float *partials = static_cast<float *>(ws);
#define GNN_XENT(NPL)                                                                      \
  softmax_xent_kernel<NPL><<<(unsigned)nb, 256, 0, st>>>(M, C, Z, ldz, labels, grad_scale, dZ, \
                                                         ldd, partials)
  if (C <= 32)
    GNN_XENT(1);
  else if (C <= 64)
    GNN_XENT(2);
  else if (C <= 128)
    GNN_XENT(4);
  else if (C <= 256)
    GNN_XENT(8);
  else
    softmax_xent_wide_kernel<<<(unsigned)nb, 256, 0, st>>>(M, C, Z, ldz, labels, grad_scale, dZ,
                                                           ldd, partials);
#undef GNN_XENT
  GNN_LAUNCH_CHECK();
  loss_final_kernel<<<1, 256, 0, st>>>(nb, partials, 1.0f / (float)M, loss);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_adam_step(int nparams, const void *param_table, float lr, float beta1, float beta2,
                  float eps, float weight_decay, int64_t *step, gnn_stream_t stream) {
  if (nparams <= 0 || !param_table || !step) return GNN_ERR_INVALID_ARGUMENT;
  cudaStream_t st = as_stream(stream);
  dim3 grid(64u, (unsigned)(nparams < 65535 ? nparams : 65535));
  adam_kernel<<<grid, 256, 0, st>>>(static_cast<const AdamParam *>(param_table), nparams, lr,
                                    beta1, beta2, eps, weight_decay, step);
  GNN_LAUNCH_CHECK();
  step_increment_kernel<<<1, 1, 0, st>>>(step);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------
// Fused output layer (GCN/GIN trainers): one warp per row computes
//   z = P[r] W + b;  loss += lse(z) - z[y];  dz = (softmax(z) - onehot(y)) / M
//   dP[r] = (dz W^T) * rowscale(r)   (rowscale = 1/deg(r): the degree-norm of
//                                     the next backward SpMM's INPUT)
//   dW += P[r]^T dz;  db += dz       (register accumulators, fixed-order CTA reduction)
// Replaces gemm + xent + colsum + 2 gemms + norm (~9 launches) with 2.
namespace gnn {
namespace {

constexpr int kHeadWarps = 4;
constexpr int kHeadRowsPerWarp = 128;

// partials layout: float [nb][din*C + C] then double loss[nb] (8-byte aligned)
inline int64_t head_float_slots(int64_t nb, int64_t din, int64_t C) {
  return (nb * (din * C + C) + 1) / 2 * 2;
}

// Butterfly transpose-reduction: every lane holds v[0..NV) (NV = 16 or 32);
// afterwards lane l holds sum over all 32 lanes of v[l * NV / 32] in v[0]
// (NV=16: lanes 2k and 2k+1 hold value k; NV=32: lane k holds value k).
// NV/2 + NV/4 + ... + 1 (+1) shuffles instead of NV * 5.
template <int NV>
__device__ __forceinline__ float butterfly_reduce(float (&v)[NV]) {
  const int lane = (int)lane_id();
#pragma unroll
  for (int w = NV / 2, m = 16; w >= 1; w >>= 1, m >>= 1) {
    const bool upper = (lane & m) != 0;
#pragma unroll
    for (int j = 0; j < w; ++j) {
      const float send = upper ? v[j] : v[j + w];
      const float keep = upper ? v[j + w] : v[j];
      v[j] = keep + __shfl_xor_sync(kFull, send, m);
    }
  }
  // NV=32 consumed masks 16..1 (5 steps); NV=16 consumed 16..2: one more fold over bit 0
  if (NV == 16) v[0] += __shfl_xor_sync(kFull, v[0], 1);
  return v[0];
}

// One warp per row; lane l owns logit columns l and l+32.  Weights live in
// registers (W[k][l], W[k][l+32]); the row's P values are broadcast once and
// reused for the logits and the dW outer product; dP is one butterfly.
template <int DIN>
__global__ void __launch_bounds__(128) gcn_head_kernel(
    int64_t M, int din, int C, const float *__restrict__ P, int64_t ldp,
    const float *__restrict__ W, const float *__restrict__ b, const int64_t *__restrict__ labels,
    const int64_t *__restrict__ deg_offsets, float scale, float *dP, int64_t lddp,
    float *partials, double *lpart) {
  constexpr int NW = 4;  // warps per CTA
  constexpr int NV = DIN <= 16 ? 16 : 32;
  __shared__ float stage[NW][32];
  __shared__ double lred[NW];
  const int warp = threadIdx.x >> 5, lane = (int)lane_id();
  const bool v0 = lane < C, v1 = lane + 32 < C;
  float w0[DIN], w1[DIN];
#pragma unroll
  for (int k = 0; k < DIN; ++k) {
    w0[k] = (k < din && v0) ? W[k * C + lane] : 0.f;
    w1[k] = (k < din && v1) ? W[k * C + lane + 32] : 0.f;
  }
  const float bb0 = v0 ? b[lane] : 0.f, bb1 = v1 ? b[lane + 32] : 0.f;
  float aw0[DIN], aw1[DIN];
#pragma unroll
  for (int k = 0; k < DIN; ++k) aw0[k] = aw1[k] = 0.f;
  float ab0 = 0.f, ab1 = 0.f;
  double lsum = 0.0;
  const int64_t r0 = ((int64_t)blockIdx.x * NW + warp) * kHeadRowsPerWarp;
  const int64_t r1 = min(M, r0 + kHeadRowsPerWarp);
  for (int64_t r = r0; r < r1; ++r) {
    float pk[DIN];
#pragma unroll
    for (int k0 = 0; k0 < DIN; k0 += 32) {
      const float pv = (k0 + lane < din) ? __ldg(P + r * ldp + k0 + lane) : 0.f;
#pragma unroll
      for (int k = 0; k < 32 && k0 + k < DIN; ++k) pk[k0 + k] = __shfl_sync(kFull, pv, k);
    }
    float z0a = bb0, z0b = 0.f, z1a = bb1, z1b = 0.f;  // two chains each for ILP
#pragma unroll
    for (int k = 0; k < DIN; k += 2) {
      z0a = fmaf(pk[k], w0[k], z0a);
      z1a = fmaf(pk[k], w1[k], z1a);
      z0b = fmaf(pk[k + 1], w0[k + 1], z0b);
      z1b = fmaf(pk[k + 1], w1[k + 1], z1b);
    }
    const float z0 = z0a + z0b, z1 = z1a + z1b;
    float mx = fmaxf(v0 ? z0 : -INFINITY, v1 ? z1 : -INFINITY);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
    const float e0 = v0 ? __expf(z0 - mx) : 0.f, e1 = v1 ? __expf(z1 - mx) : 0.f;
    float se = e0 + e1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(kFull, se, o);
    const float inv = 1.f / se;
    const int y = (int)__ldg(labels + r);
    const float zy = __shfl_sync(kFull, y < 32 ? z0 : z1, y & 31);
    if (lane == 0) lsum += (y >= 0 && y < C) ? (double)(mx + logf(se) - zy) : (double)NAN;
    const float d0 = v0 ? (e0 * inv - (lane == y ? 1.f : 0.f)) * scale : 0.f;
    const float d1 = v1 ? (e1 * inv - (lane + 32 == y ? 1.f : 0.f)) * scale : 0.f;
    ab0 += d0;
    ab1 += d1;
#pragma unroll
    for (int k = 0; k < DIN; ++k) {
      aw0[k] = fmaf(pk[k], d0, aw0[k]);
      aw1[k] = fmaf(pk[k], d1, aw1[k]);
    }
    // dP[k] = sum_c dz_c W[k][c]: per-lane partials for every k, one butterfly per 32 k's
    float rs = 1.f;
    if (deg_offsets) {
      const int64_t dg = __ldg(deg_offsets + r + 1) - __ldg(deg_offsets + r);
      rs = dg > 0 ? 1.f / (float)dg : 0.f;
    }
#pragma unroll
    for (int k0 = 0; k0 < DIN; k0 += NV) {
      float part[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) part[j] = d0 * w0[k0 + j] + d1 * w1[k0 + j];
      const float dp = butterfly_reduce<NV>(part);
      const int k = k0 + (NV == 16 ? lane >> 1 : lane);
      if ((NV == 32 || (lane & 1) == 0) && k < din) dP[r * lddp + k] = dp * rs;
    }
  }
  // CTA reduction in fixed warp order: rows k<din of dW (two column halves), then db
  const int64_t NPF = (int64_t)din * C + C;
  float *out = partials + (int64_t)blockIdx.x * NPF;
#pragma unroll
  for (int k = 0; k <= DIN; ++k) {
    if (k < din || k == DIN) {
      const int kr = k < din ? k : din;  // partial row index (row din = db)
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        stage[warp][lane] = k < DIN ? (half ? aw1[k] : aw0[k]) : (half ? ab1 : ab0);
        __syncthreads();
        if (warp == 0) {
          float t = 0.f;
#pragma unroll
          for (int w2 = 0; w2 < NW; ++w2) t += stage[w2][lane];
          const int c = lane + 32 * half;
          if (c < C) out[(int64_t)kr * C + c] = t;
        }
        __syncthreads();
      }
    }
  }
  if (lane == 0) lred[warp] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w2 = 0; w2 < NW; ++w2) t += lred[w2];
    lpart[blockIdx.x] = t;
  }
}

__global__ void gcn_head_reduce_kernel(int64_t nb, int din, int C, const float *__restrict__ partials,
                                       const double *__restrict__ lpart, float *dW, float *db,
                                       float *loss, float loss_scale) {
  const int64_t NPF = (int64_t)din * C + C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= NPF;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < NPF) {
      float t = 0.f;
      for (int64_t b2 = 0; b2 < nb; ++b2) t += partials[b2 * NPF + i];
      if (i < (int64_t)din * C)
        dW[i] = t;
      else
        db[i - (int64_t)din * C] = t;
    } else {
      double t = 0.0;
      for (int64_t b2 = 0; b2 < nb; ++b2) t += lpart[b2];
      *loss = (float)(t * (double)loss_scale);
    }
  }
}

// Thread-per-row form (din <= 32): each thread owns one row end to end —
// logits (W, b broadcast from shared memory), softmax-CE, dz, dP = dz W^T *
// rowscale — with no cross-lane traffic; the CTA then forms its dW / db
// partials from the staged P and dz tiles in fixed row order.  The warp-per-
// row kernel above serialises ~150 dependent shuffle/FMA steps per row on
// 12 warps per SM; here 256 independent rows per CTA keep every lane busy.
constexpr int kHeadRowsPerCta = 256;

template <int DIN, int CM>
__global__ void __launch_bounds__(kHeadRowsPerCta, 2) gcn_head_rows_kernel(
    int64_t M, int din, int C, const float *__restrict__ P, int64_t ldp,
    const float *__restrict__ W, const float *__restrict__ b, const int64_t *__restrict__ labels,
    const int64_t *__restrict__ deg_offsets, float scale, float *dP, int64_t lddp,
    float *partials, double *lpart) {
  constexpr int T = kHeadRowsPerCta;
  constexpr int C4 = CM / 4;
  constexpr int LDD = CM + 4;            // dz tile row stride (16-byte rows)
  extern __shared__ __align__(16) float hsm[];
  float *Ws = hsm;                       // [DIN][CM] zero padded
  float *bs = Ws + DIN * CM;             // [CM]
  float *Ps = bs + CM;                   // [T][DIN + 1]
  float *Ds = Ps + T * (DIN + 1);        // [T][LDD]
  __shared__ double lred[T / 32];
  const int tid = threadIdx.x;
  for (int i = tid; i < DIN * CM; i += T) {
    const int k = i / CM, c = i % CM;
    Ws[i] = (k < din && c < C) ? W[k * C + c] : 0.f;
  }
  for (int c = tid; c < CM; c += T) bs[c] = c < C ? b[c] : 0.f;
  __syncthreads();
  const float4 *W4 = reinterpret_cast<const float4 *>(Ws);
  const int64_t r = (int64_t)blockIdx.x * T + tid;
  const bool valid = r < M;
  float p[DIN];
#pragma unroll
  for (int k = 0; k < DIN; ++k) p[k] = (valid && k < din) ? __ldg(P + r * ldp + k) : 0.f;
  float z[CM];
#pragma unroll
  for (int c = 0; c < CM; ++c) z[c] = bs[c];
#pragma unroll
  for (int k = 0; k < DIN; ++k)
#pragma unroll
    for (int q = 0; q < C4; ++q) {
      const float4 w = W4[k * C4 + q];  // broadcast: every lane reads the same word
      z[4 * q] = fmaf(p[k], w.x, z[4 * q]);
      z[4 * q + 1] = fmaf(p[k], w.y, z[4 * q + 1]);
      z[4 * q + 2] = fmaf(p[k], w.z, z[4 * q + 2]);
      z[4 * q + 3] = fmaf(p[k], w.w, z[4 * q + 3]);
    }
  const int y = valid ? (int)__ldg(labels + r) : -1;
  float mx = -INFINITY, zy = 0.f;
#pragma unroll
  for (int c = 0; c < CM; ++c) {
    if (c < C) mx = fmaxf(mx, z[c]);
    if (c == y) zy = z[c];
  }
  float se = 0.f;
#pragma unroll
  for (int c = 0; c < CM; ++c) {
    z[c] = c < C ? __expf(z[c] - mx) : 0.f;  // z now holds e_c
    se += z[c];
  }
  const float inv = 1.f / se;
  double lrow = 0.0;
#pragma unroll
  for (int c = 0; c < CM; ++c) z[c] = valid ? (z[c] * inv - (c == y ? 1.f : 0.f)) * scale : 0.f;
  float4 *D4 = reinterpret_cast<float4 *>(Ds + tid * LDD);
#pragma unroll
  for (int q = 0; q < C4; ++q) D4[q] = make_float4(z[4 * q], z[4 * q + 1], z[4 * q + 2], z[4 * q + 3]);
  if (valid) lrow = (y >= 0 && y < C) ? (double)(mx + logf(se) - zy) : (double)NAN;
  float rs = 1.f;
  if (valid && deg_offsets) {
    const int64_t dg = __ldg(deg_offsets + r + 1) - __ldg(deg_offsets + r);
    rs = dg > 0 ? 1.f / (float)dg : 0.f;
  }
#pragma unroll
  for (int k = 0; k < DIN; ++k) {
    Ps[tid * (DIN + 1) + k] = p[k];
    float t0 = 0.f, t1 = 0.f;
#pragma unroll
    for (int q = 0; q < C4; ++q) {
      const float4 w = W4[k * C4 + q];
      t0 = fmaf(z[4 * q], w.x, t0);
      t1 = fmaf(z[4 * q + 1], w.y, t1);
      t0 = fmaf(z[4 * q + 2], w.z, t0);
      t1 = fmaf(z[4 * q + 3], w.w, t1);
    }
    if (valid && k < din) dP[r * lddp + k] = (t0 + t1) * rs;
  }
  // loss: fixed-order block reduction (warp butterfly, then warps in order)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lrow += __shfl_xor_sync(kFull, lrow, o);
  if ((tid & 31) == 0) lred[tid >> 5] = lrow;
  __syncthreads();
  // dW[k][4q..4q+3] = sum_i P[i][k] dz[i][4q..]; db (item k == din) = sum_i dz[i][4q..]
  const int64_t NPF = (int64_t)din * C + C;
  float *out = partials + (int64_t)blockIdx.x * NPF;
  const int items = (din + 1) * C4;
  for (int it = tid; it < items; it += T) {
    const int k = it / C4, q = it % C4;
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k < din) {
      for (int i = 0; i < T; ++i) {
        const float pk = Ps[i * (DIN + 1) + k];
        const float4 d = reinterpret_cast<const float4 *>(Ds + i * LDD)[q];
        t.x = fmaf(pk, d.x, t.x);
        t.y = fmaf(pk, d.y, t.y);
        t.z = fmaf(pk, d.z, t.z);
        t.w = fmaf(pk, d.w, t.w);
      }
    } else {
      for (int i = 0; i < T; ++i) {
        const float4 d = reinterpret_cast<const float4 *>(Ds + i * LDD)[q];
        t.x += d.x;
        t.y += d.y;
        t.z += d.z;
        t.w += d.w;
      }
    }
    const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = 4 * q + j;
      if (c < C) out[(int64_t)k * C + c] = tv[j];
    }
  }
  if (tid == 0) {
    double t = 0.0;
    for (int w2 = 0; w2 < T / 32; ++w2) t += lred[w2];
    lpart[blockIdx.x] = t;
  }
}

template <int DIN, int CM>
size_t head_rows_smem() {
  return sizeof(float) * (size_t)(DIN * CM + CM + kHeadRowsPerCta * (DIN + 1) +
                                  kHeadRowsPerCta * (CM + 4));
}

// warp per output: lanes stride the CTA partials, fixed-order butterfly
__global__ void gcn_head_reduce_warp_kernel(int64_t nb, int din, int C,
                                            const float *__restrict__ partials,
                                            const double *__restrict__ lpart, float *dW, float *db,
                                            float *loss, float loss_scale) {
  const int64_t NPF = (int64_t)din * C + C;
  const int lane = (int)lane_id();
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i <= NPF;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if (i < NPF) {
      float t = 0.f;
      for (int64_t b2 = lane; b2 < nb; b2 += 32) t += partials[b2 * NPF + i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
      if (lane == 0) {
        if (i < (int64_t)din * C)
          dW[i] = t;
        else
          db[i - (int64_t)din * C] = t;
      }
    } else {
      double t = 0.0;
      for (int64_t b2 = lane; b2 < nb; b2 += 32) t += lpart[b2];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
      if (lane == 0) *loss = (float)(t * (double)loss_scale);
    }
  }
}

// Wide output layer (C > 64, e.g. the 172 classes of the papers100M shape):
// the [M, C] logits never exist in memory.  Thread per row, classes in
// chunks of 32: pass 1 forms each chunk's logits from the row's P (registers)
// and W (shared memory) and keeps an online max / sum; pass 2 recomputes the
// chunk, forms dz, accumulates dP = dz W^T, and stages dz in shared memory
// where each warp forms its 32 rows' share of dW = P^T dz (lane = class, DIN
// register accumulators), reduced across warps in fixed order into per-thread
// CTA accumulators.  Persistent grid: partials are [grid][din*C + C] and the
// fixed-order warp reduce of the narrow head finishes dW / db / loss.
constexpr int kWideT = 256;
constexpr int kWideWarps = kWideT / 32;

template <int DIN, int NCH>
size_t head_wide_smem() {
  constexpr int CP = NCH * 32;
  return sizeof(float) * (size_t)(DIN * CP + CP + kWideT * (DIN + 4) + kWideT * 33 +
                                  kWideWarps * (DIN + 1) * 32 + (DIN + 1) * CP);
}

template <int DIN, int NCH>
__global__ void __launch_bounds__(kWideT, 1) gcn_head_wide_kernel(
    int64_t M, int din, int C, const float *__restrict__ P, int64_t ldp,
    const float *__restrict__ W, const float *__restrict__ b, const int64_t *__restrict__ labels,
    const int64_t *__restrict__ deg_offsets, float scale, float *dP, int64_t lddp,
    float *partials, double *lpart) {
  constexpr int T = kWideT, CP = NCH * 32, LDP = DIN + 4, KR = DIN * 32 / T;
  extern __shared__ __align__(16) float hw[];
  float *Ws = hw;                    // [DIN][CP]
  float *bs = Ws + DIN * CP;         // [CP]
  float *Ps = bs + CP;               // [T][LDP]
  float *Ds = Ps + T * LDP;          // [T][33]
  float *St = Ds + T * 33;           // [warps][DIN+1][32]
  float *Acc = St + kWideWarps * (DIN + 1) * 32;  // [DIN+1][CP] CTA dW / db (row DIN) partials
  __shared__ double lred[kWideWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < DIN * CP; i += T) {
    const int k = i / CP, c = i % CP;
    Ws[i] = (k < din && c < C) ? W[(int64_t)k * C + c] : 0.f;
  }
  for (int c = tid; c < CP; c += T) bs[c] = c < C ? b[c] : 0.f;
  for (int i = tid; i < (DIN + 1) * CP; i += T) Acc[i] = 0.f;
  __syncthreads();
  double lsum = 0.0;
  const float4 *W4 = reinterpret_cast<const float4 *>(Ws);
  for (int64_t r0 = (int64_t)blockIdx.x * T; r0 < M; r0 += (int64_t)gridDim.x * T) {
    const int64_t r = r0 + tid;
    const bool valid = r < M;
    float p[DIN];
#pragma unroll
    for (int k = 0; k < DIN; ++k) p[k] = (valid && k < din) ? __ldg(P + r * ldp + k) : 0.f;
#pragma unroll
    for (int k = 0; k < DIN; k += 4)
      *reinterpret_cast<float4 *>(Ps + tid * LDP + k) = make_float4(p[k], p[k + 1], p[k + 2], p[k + 3]);
    const int64_t y = valid ? __ldg(labels + r) : -1;
    // ---- pass 1: online max / sum of exp over the class chunks
    float mx = -INFINITY, se = 0.f, zy = 0.f;
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
      float z[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) z[j] = bs[ch * 32 + j];
#pragma unroll
      for (int k = 0; k < DIN; ++k)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 w = W4[(k * CP + ch * 32) / 4 + q];
          z[4 * q] = fmaf(p[k], w.x, z[4 * q]);
          z[4 * q + 1] = fmaf(p[k], w.y, z[4 * q + 1]);
          z[4 * q + 2] = fmaf(p[k], w.z, z[4 * q + 2]);
          z[4 * q + 3] = fmaf(p[k], w.w, z[4 * q + 3]);
        }
      float cm = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int c = ch * 32 + j;
        if (c < C) cm = fmaxf(cm, z[j]);
        if (c == y) zy = z[j];
      }
      const float nm = fmaxf(mx, cm);
      float add = 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (ch * 32 + j < C) add += __expf(z[j] - nm);
      se = se * __expf(mx - nm) + add;
      mx = nm;
    }
    const float inv = 1.f / se;
    if (valid) lsum += (y >= 0 && y < C) ? (double)(mx + logf(se) - zy) : (double)NAN;
    float rs = 1.f;
    if (valid && deg_offsets) {
      const int64_t dg = __ldg(deg_offsets + r + 1) - __ldg(deg_offsets + r);
      rs = dg > 0 ? 1.f / (float)dg : 0.f;
    }
    float dp[DIN];
#pragma unroll
    for (int k = 0; k < DIN; ++k) dp[k] = 0.f;
    // ---- pass 2: dz per chunk, dP, and this chunk's dW / db partials
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
      float z[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) z[j] = bs[ch * 32 + j];
#pragma unroll
      for (int k = 0; k < DIN; ++k)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 w = W4[(k * CP + ch * 32) / 4 + q];
          z[4 * q] = fmaf(p[k], w.x, z[4 * q]);
          z[4 * q + 1] = fmaf(p[k], w.y, z[4 * q + 1]);
          z[4 * q + 2] = fmaf(p[k], w.z, z[4 * q + 2]);
          z[4 * q + 3] = fmaf(p[k], w.w, z[4 * q + 3]);
        }
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int c = ch * 32 + j;
        z[j] = (valid && c < C) ? (__expf(z[j] - mx) * inv - (c == y ? 1.f : 0.f)) * scale : 0.f;
        Ds[tid * 33 + j] = z[j];
      }
#pragma unroll
      for (int k = 0; k < DIN; ++k) {
        float t0 = 0.f, t1 = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 w = W4[(k * CP + ch * 32) / 4 + q];
          t0 = fmaf(z[4 * q], w.x, t0);
          t1 = fmaf(z[4 * q + 1], w.y, t1);
          t0 = fmaf(z[4 * q + 2], w.z, t0);
          t1 = fmaf(z[4 * q + 3], w.w, t1);
        }
        dp[k] += t0 + t1;
      }
      __syncthreads();
      // warp's 32 rows: lane = class column, DIN accumulators (+ db)
      float a[DIN];
#pragma unroll
      for (int k = 0; k < DIN; ++k) a[k] = 0.f;
      float ab = 0.f;
#pragma unroll 4
      for (int i = warp * 32; i < warp * 32 + 32; ++i) {
        const float d = Ds[i * 33 + lane];
        ab += d;
#pragma unroll
        for (int k = 0; k < DIN; k += 4) {
          const float4 pv = *reinterpret_cast<const float4 *>(Ps + i * LDP + k);
          a[k] = fmaf(pv.x, d, a[k]);
          a[k + 1] = fmaf(pv.y, d, a[k + 1]);
          a[k + 2] = fmaf(pv.z, d, a[k + 2]);
          a[k + 3] = fmaf(pv.w, d, a[k + 3]);
        }
      }
#pragma unroll
      for (int k = 0; k < DIN; ++k) St[(warp * (DIN + 1) + k) * 32 + lane] = a[k];
      St[(warp * (DIN + 1) + DIN) * 32 + lane] = ab;
      __syncthreads();
      // fixed-order cross-warp sum into the CTA accumulators (each (k, class)
      // item has one owning thread: deterministic, no atomics)
#pragma unroll
      for (int q = 0; q < KR; ++q) {
        const int k = warp + kWideWarps * q;
        float t = 0.f;
#pragma unroll
        for (int w2 = 0; w2 < kWideWarps; ++w2) t += St[(w2 * (DIN + 1) + k) * 32 + lane];
        Acc[k * CP + ch * 32 + lane] += t;
      }
      if (warp == 0) {
        float t = 0.f;
#pragma unroll
        for (int w2 = 0; w2 < kWideWarps; ++w2) t += St[(w2 * (DIN + 1) + DIN) * 32 + lane];
        Acc[DIN * CP + ch * 32 + lane] += t;
      }
      __syncthreads();
    }
    if (valid) {
#pragma unroll
      for (int k = 0; k < DIN; ++k)
        if (k < din) dP[r * lddp + k] = dp[k] * rs;
    }
  }
  const int64_t NPF = (int64_t)din * C + C;
  float *out = partials + (int64_t)blockIdx.x * NPF;
  for (int i = tid; i < (din + 1) * C; i += T) {
    const int k = i / C, c = i % C;
    out[i] = Acc[(k < din ? k : DIN) * CP + c];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(kFull, lsum, o);
  if (lane == 0) lred[warp] = lsum;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w2 = 0; w2 < kWideWarps; ++w2) t += lred[w2];
    lpart[blockIdx.x] = t;
  }
}

// Lane-per-class form of the wide head (Din <= 16): a warp owns a row at a
// time and lane l owns classes l, l+32, ..., l+32(NJ-1); W[k][class] (16 x NJ)
// and the warp's dW partials (16 x NJ) live in registers for the whole
// kernel, so per row the only traffic is the row of P (one 64-byte load),
// its label and its row of dP.  The thread-per-row form above reloads W from
// shared memory for every logit and is bound by those loads.
template <int NJ>
__global__ void __launch_bounds__(kWideT, 1) gcn_head_lanes_kernel(
    int64_t M, int din, int C, const float *__restrict__ P, int64_t ldp,
    const float *__restrict__ W, const float *__restrict__ b, const int64_t *__restrict__ labels,
    const int64_t *__restrict__ deg_offsets, float scale, float *dP, int64_t lddp,
    float *partials, double *lpart) {
  constexpr int CP = NJ * 32;
  extern __shared__ __align__(16) float hl[];  // [warps][17][CP] warp partials (dW rows, db)
  __shared__ double lred[kWideWarps];
  const int warp = threadIdx.x >> 5, lane = (int)lane_id();
  float w[16][NJ], acc[16][NJ], bb[NJ], accb[NJ];
  bool ok[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int c = lane + 32 * j;
    ok[j] = c < C;
    bb[j] = ok[j] ? b[c] : 0.f;
    accb[j] = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      w[k][j] = (ok[j] && k < din) ? W[(int64_t)k * C + c] : 0.f;
      acc[k][j] = 0.f;
    }
  }
  double lsum = 0.0;
  const int64_t nw = (int64_t)gridDim.x * kWideWarps;
  // software pipeline: the next row's P / label / degree are loaded while
  // this row computes (one HBM round trip per row would otherwise bound it)
  int64_t r = (int64_t)blockIdx.x * kWideWarps + warp;
  float pl_n = 0.f;
  int64_t y_n = 0, dg_n = 0;
  if (r < M) {
    pl_n = lane < din ? __ldg(P + r * ldp + lane) : 0.f;
    y_n = __ldg(labels + r);
    if (deg_offsets) dg_n = __ldg(deg_offsets + r + 1) - __ldg(deg_offsets + r);
  }
  for (; r < M; r += nw) {
    const float pl = pl_n;
    const int64_t y = y_n, dg = dg_n;
    const int64_t rn = r + nw;
    if (rn < M) {
      pl_n = lane < din ? __ldg(P + rn * ldp + lane) : 0.f;
      y_n = __ldg(labels + rn);
      if (deg_offsets) dg_n = __ldg(deg_offsets + rn + 1) - __ldg(deg_offsets + rn);
    }
    float p[16], z[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) z[j] = bb[j];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      p[k] = __shfl_sync(kFull, pl, k);
#pragma unroll
      for (int j = 0; j < NJ; ++j) z[j] = fmaf(p[k], w[k][j], z[j]);
    }
    float mx = -INFINITY, zsel = 0.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      if (ok[j]) mx = fmaxf(mx, z[j]);
      if (j == (int)(y >> 5)) zsel = z[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
    float se = 0.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      z[j] = ok[j] ? __expf(z[j] - mx) : 0.f;
      se += z[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(kFull, se, o);
    const float zy = __shfl_sync(kFull, zsel, (int)(y & 31));
    if (lane == 0) lsum += (y >= 0 && y < C) ? (double)(mx + logf(se) - zy) : (double)NAN;
    const float inv = 1.f / se;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = lane + 32 * j;
      z[j] = ok[j] ? (z[j] * inv - (c == y ? 1.f : 0.f)) * scale : 0.f;  // z = dz now
      accb[j] += z[j];
    }
    float part[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float t = 0.f;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        t = fmaf(z[j], w[k][j], t);
        acc[k][j] = fmaf(p[k], z[j], acc[k][j]);
      }
      part[k] = t;
    }
    const float dpv = butterfly_reduce<16>(part);  // lanes 2k, 2k+1: dP[k]
    const float rs = deg_offsets ? (dg > 0 ? 1.f / (float)dg : 0.f) : 1.f;
    const int k = lane >> 1;
    if ((lane & 1) == 0 && k < din) dP[r * lddp + k] = dpv * rs;
  }
  // CTA reduction in fixed warp order
  float *st = hl + (int64_t)warp * 17 * CP;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
#pragma unroll
    for (int k = 0; k < 16; ++k) st[k * CP + lane + 32 * j] = acc[k][j];
    st[16 * CP + lane + 32 * j] = accb[j];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(kFull, lsum, o);
  if (lane == 0) lred[warp] = lsum;
  __syncthreads();
  const int64_t NPF = (int64_t)din * C + C;
  float *out = partials + (int64_t)blockIdx.x * NPF;
  for (int i = threadIdx.x; i < (din + 1) * C; i += kWideT) {
    const int kk = i / C, c = i % C;
    const int row = kk < din ? kk : 16;
    float t = 0.f;
    for (int w2 = 0; w2 < kWideWarps; ++w2) t += hl[((int64_t)w2 * 17 + row) * CP + c];
    out[i] = t;
  }
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w2 = 0; w2 < kWideWarps; ++w2) t += lred[w2];
    lpart[blockIdx.x] = t;
  }
}

int64_t head_wide_grid(int64_t M) {
  const int64_t g = (int64_t)sm_count();
  const int64_t need = ceil_div(M > 0 ? M : 1, (int64_t)kWideT);
  return need < g ? need : g;
}

}  // namespace
}  // namespace gnn

extern "C" {

size_t gnn_gcn_head_workspace(int64_t M, int64_t Din, int64_t C) {
  const int64_t nb1 = ceil_div(M > 0 ? M : 1, (int64_t)kHeadWarps * kHeadRowsPerWarp);
  const int64_t nb2 = ceil_div(M > 0 ? M : 1, (int64_t)kHeadRowsPerCta);
  int64_t nb = nb1 > nb2 ? nb1 : nb2;
  if (C > 64) nb = head_wide_grid(M);  // persistent wide head
  return sizeof(float) * (size_t)head_float_slots(nb, Din, C) + sizeof(double) * (size_t)nb + 512;
}

int gnn_gcn_head_scaled(int64_t M, int64_t Din, int64_t C, const float *P, int64_t ldp,
                        const float *W, const float *b, const int64_t *labels,
                        const int64_t *deg_offsets, float grad_scale, float *dP, int64_t lddp,
                        float *dW, float *db, float *loss, void *ws, size_t ws_bytes,
                        gnn_stream_t stream) {
  if (M <= 0 || Din <= 0 || Din > 64 || C <= 0 || C > 256 || (C > 64 && Din > 32) || !P ||
      ldp < Din || !W || !b || !labels || !dP || lddp < Din || !dW || !db || !loss)
    return GNN_ERR_INVALID_ARGUMENT;
  if (ws_bytes < gnn_gcn_head_workspace(M, Din, C)) return GNN_ERR_WORKSPACE;
  cudaStream_t st = as_stream(stream);
  const float scale = grad_scale;
  float *partials = static_cast<float *>(ws);
  if (C > 64) {  // wide head: logits never materialised
    const int64_t nb = head_wide_grid(M);
    double *lpart = reinterpret_cast<double *>(partials + head_float_slots(nb, Din, C));
    // tensor-core form (head_tc.cu) where it applies, else the SIMT kernels below
    const int tc = gcn_head_tc(M, Din, C, P, ldp, W, b, labels, deg_offsets, scale, dP, lddp,
                               partials, lpart, nb, st);
    if (tc == GNN_OK) {
      const int64_t outs = Din * C + C + 1;
      gcn_head_reduce_warp_kernel<<<(unsigned)ceil_div(outs * 32, 256), 256, 0, st>>>(
          nb, (int)Din, (int)C, partials, lpart, dW, db, loss, grad_scale);
      GNN_LAUNCH_CHECK();
      return GNN_OK;
    }
    if (tc != GNN_ERR_UNSUPPORTED) return tc;
    const int nch = (int)ceil_div(C, (int64_t)32);
#define GNN_HEAD_WIDE(DN, NC)                                                                   \
  do {                                                                                          \
    const size_t sm = head_wide_smem<DN, NC>();                                                 \
    GNN_CUDA_TRY(cudaFuncSetAttribute(gcn_head_wide_kernel<DN, NC>,                             \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));   \
    gcn_head_wide_kernel<DN, NC><<<(unsigned)nb, kWideT, sm, st>>>(                             \
        M, (int)Din, (int)C, P, ldp, W, b, labels, deg_offsets, scale, dP, lddp, partials, lpart); \
  } while (0)
#define GNN_HEAD_WIDE_D(DN)                  \
  switch (nch) {                             \
    case 3: GNN_HEAD_WIDE(DN, 3); break;     \
    case 4: GNN_HEAD_WIDE(DN, 4); break;     \
    case 5: GNN_HEAD_WIDE(DN, 5); break;     \
    case 6: GNN_HEAD_WIDE(DN, 6); break;     \
    case 7: GNN_HEAD_WIDE(DN, 7); break;     \
    default: GNN_HEAD_WIDE(DN, 8); break;    \
  }
    // lane-per-class form: opt-in (GNN_HEAD_LANES=1); measured slower at the
    // papers100M shape (171 vs 148 ms: 8 warps/SM at 255 registers cannot hide
    // its shuffle-reduction chains), see DESIGN.md
    static const bool lanes_form = [] {
      const char *e = getenv("GNN_HEAD_LANES");
      return e && e[0] == '1';
    }();
    if (Din <= 16 && lanes_form) {
#define GNN_HEAD_LANES(NJ)                                                                      \
  do {                                                                                          \
    const size_t sm = sizeof(float) * (size_t)kWideWarps * 17 * (NJ * 32);                      \
    GNN_CUDA_TRY(cudaFuncSetAttribute(gcn_head_lanes_kernel<NJ>,                                \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));   \
    gcn_head_lanes_kernel<NJ><<<(unsigned)nb, kWideT, sm, st>>>(                                \
        M, (int)Din, (int)C, P, ldp, W, b, labels, deg_offsets, scale, dP, lddp, partials, lpart); \
  } while (0)
      switch (nch) {
        case 3: GNN_HEAD_LANES(3); break;
        case 4: GNN_HEAD_LANES(4); break;
        case 5: GNN_HEAD_LANES(5); break;
        case 6: GNN_HEAD_LANES(6); break;
        case 7: GNN_HEAD_LANES(7); break;
        default: GNN_HEAD_LANES(8); break;
      }
#undef GNN_HEAD_LANES
    } else if (Din <= 16) {
      GNN_HEAD_WIDE_D(16);
    } else {
      GNN_HEAD_WIDE_D(32);
    }
#undef GNN_HEAD_WIDE_D
#undef GNN_HEAD_WIDE
    GNN_LAUNCH_CHECK();
    const int64_t outs = Din * C + C + 1;
    gcn_head_reduce_warp_kernel<<<(unsigned)ceil_div(outs * 32, 256), 256, 0, st>>>(
        nb, (int)Din, (int)C, partials, lpart, dW, db, loss, grad_scale);
    GNN_LAUNCH_CHECK();
    return GNN_OK;
  }
  static const bool rows_form = [] {
    const char *e = getenv("GNN_HEAD_ROWS");
    return !(e && e[0] == '0');
  }();
  if (Din <= 32 && rows_form) {  // thread-per-row form
    const int64_t nb = ceil_div(M, (int64_t)kHeadRowsPerCta);
    double *lpart = reinterpret_cast<double *>(partials + head_float_slots(nb, Din, C));
#define GNN_HEAD_ROWS(DN, CMX)                                                                  \
  do {                                                                                          \
    const size_t sm = head_rows_smem<DN, CMX>();                                                \
    GNN_CUDA_TRY(cudaFuncSetAttribute(gcn_head_rows_kernel<DN, CMX>,                            \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));   \
    gcn_head_rows_kernel<DN, CMX><<<(unsigned)nb, kHeadRowsPerCta, sm, st>>>(                   \
        M, (int)Din, (int)C, P, ldp, W, b, labels, deg_offsets, scale, dP, lddp, partials, lpart); \
  } while (0)
    if (Din <= 16) {
      if (C <= 16) GNN_HEAD_ROWS(16, 16);
      else if (C <= 32) GNN_HEAD_ROWS(16, 32);
      else if (C <= 48) GNN_HEAD_ROWS(16, 48);
      else GNN_HEAD_ROWS(16, 64);
    } else {
      if (C <= 16) GNN_HEAD_ROWS(32, 16);
      else if (C <= 32) GNN_HEAD_ROWS(32, 32);
      else if (C <= 48) GNN_HEAD_ROWS(32, 48);
      else GNN_HEAD_ROWS(32, 64);
    }
#undef GNN_HEAD_ROWS
    GNN_LAUNCH_CHECK();
    const int64_t outs = Din * C + C + 1;
    gcn_head_reduce_warp_kernel<<<(unsigned)ceil_div(outs * 32, 256), 256, 0, st>>>(
        nb, (int)Din, (int)C, partials, lpart, dW, db, loss, grad_scale);
    GNN_LAUNCH_CHECK();
    return GNN_OK;
  }
  const int64_t nb = ceil_div(M, (int64_t)kHeadWarps * kHeadRowsPerWarp);
  double *lpart = reinterpret_cast<double *>(partials + head_float_slots(nb, Din, C));
#define GNN_HEAD(DN)                                                                            \
  gcn_head_kernel<DN><<<(unsigned)nb, 128, 0, st>>>(M, (int)Din, (int)C, P, ldp, W, b, labels, \
                                                    deg_offsets, scale, dP, lddp, partials, lpart)
  if (Din <= 16)
    GNN_HEAD(16);
  else if (Din <= 32)
    GNN_HEAD(32);
  else
    GNN_HEAD(64);
#undef GNN_HEAD
  GNN_LAUNCH_CHECK();
  gcn_head_reduce_kernel<<<(unsigned)ceil_div(Din * C + C + 1, 256), 256, 0, st>>>(
      nb, (int)Din, (int)C, partials, lpart, dW, db, loss, grad_scale);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_gcn_head(int64_t M, int64_t Din, int64_t C, const float *P, int64_t ldp, const float *W,
                 const float *b, const int64_t *labels, const int64_t *deg_offsets, float *dP,
                 int64_t lddp, float *dW, float *db, float *loss, void *ws, size_t ws_bytes,
                 gnn_stream_t stream) {
  if (M <= 0) return GNN_ERR_INVALID_ARGUMENT;
  return gnn_gcn_head_scaled(M, Din, C, P, ldp, W, b, labels, deg_offsets, 1.0f / (float)M, dP,
                             lddp, dW, db, loss, ws, ws_bytes, stream);
}

}  // extern "C"

// ------------------------------------------------- synthetic input synthesis
// Partition-independent synthetic features / labels for shapes too large to
// draw on the host (papers100M: X is 56.9 GB): element (r, k) of the global
// [V, K] matrix is a function of (seed, r*K + k) only, so every rank fills
// its row block [row0, row0+rows) with exactly the rows a single GPU would.
namespace gnn {
namespace {
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void fill_uniform_kernel(float *X, int64_t ldx, int64_t rows, int64_t cols,
                                    int64_t row0, uint64_t seed) {
  const uint64_t key = splitmix64(seed);
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, k = i - r * cols;
    const uint64_t h = splitmix64(key ^ (uint64_t)((row0 + r) * cols + k));
    // 24 random bits -> U[-1, 1) on a 2^-23 grid (exact in fp32)
    X[r * ldx + k] = (float)(int32_t)(h >> 40) * (1.0f / 8388608.0f) - 1.0f;
  }
}
__global__ void fill_labels_kernel(int64_t *y, int64_t n, int64_t row0, int64_t classes,
                                   uint64_t seed) {
  const uint64_t key = splitmix64(seed ^ 0xC1A55E5ull);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (int64_t)((splitmix64(key ^ (uint64_t)(row0 + i)) >> 11) % (uint64_t)classes);
}
}  // namespace
}  // namespace gnn

extern "C" {

int gnn_fill_uniform(float *X, int64_t ldx, int64_t rows, int64_t cols, int64_t row0,
                     uint64_t seed, gnn_stream_t stream) {
  using namespace gnn;
  if (rows < 0 || cols < 0 || ldx < cols || row0 < 0 || (rows * cols > 0 && !X))
    return GNN_ERR_INVALID_ARGUMENT;
  if (rows * cols == 0) return GNN_OK;
  const int64_t blocks = ceil_div(rows * cols, (int64_t)256), cap = (int64_t)sm_count() * 32;
  fill_uniform_kernel<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, as_stream(stream)>>>(
      X, ldx, rows, cols, row0, seed);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

int gnn_fill_labels(int64_t *y, int64_t n, int64_t row0, int64_t classes, uint64_t seed,
                    gnn_stream_t stream) {
  using namespace gnn;
  if (n < 0 || row0 < 0 || classes < 1 || (n > 0 && !y)) return GNN_ERR_INVALID_ARGUMENT;
  if (n == 0) return GNN_OK;
  const int64_t blocks = ceil_div(n, (int64_t)256), cap = (int64_t)sm_count() * 32;
  fill_labels_kernel<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, as_stream(stream)>>>(
      y, n, row0, classes, seed);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

}  // extern "C"
