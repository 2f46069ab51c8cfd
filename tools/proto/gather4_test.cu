// Probe: semantics of cp.async.bulk.tensor.2d ... tile::gather4 on sm_100a.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int r0, int r1, int r2, int r3, int nbytes, int col0) {
  __shared__ __align__(128) float buf[4 * 64];
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = -1.f;
  __syncthreads();
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  uint32_t d = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(nbytes) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 :: "r"(d), "l"(&tm), "r"(col0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" :: "r"(b) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int R = 1024, C = 48;
  std::vector<float> h(R * C);
  for (int r = 0; r < R; ++r) for (int c = 0; c < C; ++c) h[r * C + c] = r * 100.f + c;
  float *dX, *dout;
  cudaMalloc(&dX, h.size() * 4); cudaMalloc(&dout, 256 * 4);
  cudaMemcpy(dX, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  EncodeFn enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int boxes[][2] = {{16, 1}, {16, 4}, {32, 1}, {8, 1}};
  for (auto& bx : boxes) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t strides[1] = {(cuuint64_t)C * 4};
    cuuint32_t box[2] = {(cuuint32_t)bx[0], (cuuint32_t)bx[1]};
    cuuint32_t es[2] = {1, 1};
    CUresult rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dX, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box {%d,%d}: encode rc=%d\n", bx[0], bx[1], (int)rc);
    if (rc) continue;
    int nbytes = 4 * bx[0] * 4;  // 4 rows x box0 floats
    cudaMemset(dout, 0, 256 * 4);
    k<<<1, 128>>>(tm, dout, 5, 900, 17, 3, nbytes, 16);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  launch: %s\n", cudaGetErrorString(e));
    if (e) { cudaGetLastError(); continue; }
    std::vector<float> o(256);
    cudaMemcpy(o.data(), dout, 256 * 4, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 4 * bx[0] + 4 && i < 256; i += (bx[0] > 8 ? bx[0]/2 : 1)) printf("  o[%d]=%g", i, o[i]);
    printf("\n");
  }
  return 0;
}
