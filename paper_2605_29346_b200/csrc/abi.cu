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

int gnn_abi_version(void) { return 1; }

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
