// ABI housekeeping: version, error strings, device queries.
#include <atomic>

#include "common.cuh"

namespace gnn {

static std::atomic<int> g_last_cuda_error{0};
static std::atomic<long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_cuda_error(cudaError_t e) { g_last_cuda_error.store((int)e); }

int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
  if (dev < 64 && cache[dev] > 0) return cache[dev];
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    n = 148;
  if (dev < 64) cache[dev] = n;
  return n;
}

}  // namespace gnn

extern "C" {

int gnn_abi_version(void) { return 3; }

const char *gnn_strerror(int s) {
  switch (s) {
    case GNN_OK: return "ok";
    case GNN_ERR_INVALID_ARGUMENT: return "invalid argument";
    case GNN_ERR_CSR_INVARIANT: return "CSR invariant violated";
    case GNN_ERR_RANGE: return "target vertex id out of range";
    case GNN_ERR_INDEX: return "edge source local id out of range";
    case GNN_ERR_WORKSPACE: return "workspace too small";
    case GNN_ERR_CUDA: return "CUDA error";
    case GNN_ERR_UNSUPPORTED: return "unsupported shape";
    case GNN_ERR_SOURCE_RANGE: return "source vertex id out of range";
    default: return "unknown status";
  }
}

int gnn_last_cuda_error(void) { return gnn::g_last_cuda_error.load(); }

int gnn_device_sm_count(void) { return gnn::sm_count(); }

int64_t gnn_launch_counter(void) { return (int64_t)gnn::g_launches.load(); }

}  // extern "C"

// ------------------------------------------------------------ diagnostics
// L2 -> SM read-bandwidth probe: every CTA streams the whole (L2-resident)
// buffer `reps` times with 128-bit loads, starting at a CTA-dependent offset.
// Used by bench.py to state the on-chip roof next to the HBM roof.
namespace gnn {
namespace {
__global__ void __launch_bounds__(512) read_probe_kernel(const float4 *__restrict__ buf, int64_t n,
                                                         int reps, float *out) {
  // grid-stride passes over an L2-resident buffer, L1 bypassed (ld.global.cg),
  // 4 independent 128-bit loads in flight per thread
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int r = 0; r < reps; ++r) {
    int64_t i = t0;
    for (; i + 3 * stride < n; i += 4 * stride) {
      const float4 v0 = __ldcg(buf + i), v1 = __ldcg(buf + i + stride),
                   v2 = __ldcg(buf + i + 2 * stride), v3 = __ldcg(buf + i + 3 * stride);
      a0 += v0.x;
      a1 += v1.y;
      a2 += v2.z;
      a3 += v3.w;
    }
    for (; i < n; i += stride) a0 += __ldcg(buf + i).x;
  }
  if (a0 + a1 + a2 + a3 == 123456.789f) *out = a0;  // never true; keeps the loads
}
}  // namespace
}  // namespace gnn

extern "C" int gnn_read_probe(const float *buf, int64_t n_floats, int reps, float *out,
                              gnn_stream_t stream) {
  using namespace gnn;
  if (!buf || n_floats < 4 || reps <= 0 || !out) return GNN_ERR_INVALID_ARGUMENT;
  cudaStream_t st = as_stream(stream);
  read_probe_kernel<<<sm_count() * 4, 512, 0, st>>>(reinterpret_cast<const float4 *>(buf),
                                                   n_floats / 4, reps, out);
  GNN_LAUNCH_CHECK();
  return GNN_OK;
}

// Strided 2-D copy between host (pinned or pageable) and device or device
// and device, stream-ordered, no staging buffer: feature matrices go straight
// into a padded-row-stride device layout (no transient contiguous copy).
extern "C" int gnn_memcpy2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width,
                            size_t height, gnn_stream_t stream) {
  using namespace gnn;
  if ((height > 0 && width > 0) && (!dst || !src || dpitch < width || spitch < width))
    return GNN_ERR_INVALID_ARGUMENT;
  if (height == 0 || width == 0) return GNN_OK;
  GNN_CUDA_TRY(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault,
                                 as_stream(stream)));
  return GNN_OK;
}
