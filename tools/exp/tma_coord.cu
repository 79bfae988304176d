// Experiment: does cp.async.bulk.tensor (tile mode, fp64) accept an odd innermost start coordinate?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
using PFN = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                         const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                         CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap m, int cx, double* out) {
  __shared__ __align__(128) double buf[68 * 4];
  __shared__ __align__(8) uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar), d = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(68 * 4 * 8));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(d), "l"((uint64_t)&m), "r"(cx), "r"(0), "r"(b) : "memory");
    uint32_t done = 0;
    while (!done) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(done) : "r"(b));
    out[0] = buf[0]; out[1] = buf[1]; out[2] = buf[67];
  }
}
int main(int argc, char** argv) {
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN enc = (PFN)p;
  double* g; cudaMalloc(&g, 1024 * 16 * 8);
  double h[1024 * 16]; for (int i = 0; i < 1024 * 16; ++i) h[i] = i;
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  double* out; cudaMallocManaged(&out, 64);
  CUtensorMap m; cuuint64_t dims[2] = {1000, 16}, str[1] = {1024 * 8}; cuuint32_t box[2] = {68, 4}, es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int cx = argc > 1 ? atoi(argv[1]) : 0;
  k<<<1, 32>>>(m, cx, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("cx=%d -> %s  out=%g %g %g\n", cx, cudaGetErrorString(e), e ? -1.0 : out[0], e ? -1.0 : out[1], e ? -1.0 : out[2]);
  fflush(stdout);
  return 0;
}
