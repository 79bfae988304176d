// SHFL throughput / latency probe: W warps per SM, each running ILP independent
// 32-bit shfl.up chains for N iterations. Prints warp-shuffles per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(int* out, int n, long long* cyc) {
  int v[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = threadIdx.x * 7 + i;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) v[i] = __shfl_up_sync(0xffffffffu, v[i], 1) + 1;
  }
  long long t1 = clock64();
  int s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int ILP>
void run(int warps, int n) {
  int* out; long long* cyc;
  cudaMalloc(&out, 148 * warps * 32 * 4); cudaMalloc(&cyc, 148 * 8);
  k<ILP><<<148, warps * 32>>>(out, n, cyc);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double per_sm = (double)warps * ILP * n / c;
  printf("warps/SM=%2d ILP=%d: %.1f cycles per dependent shfl+add, %.3f warp-shfl per clock per SM\n", warps, ILP,
         (double)c / n, per_sm);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  run<1>(1, 100000); run<4>(1, 100000); run<8>(1, 100000);
  run<1>(4, 100000); run<4>(4, 100000); run<8>(4, 100000);
  run<8>(8, 100000); run<8>(16, 100000);
  return 0;
}
