// Does compute-sanitizer racecheck model mbarrier arrive/wait as synchronization?
// Warp 0 writes shared memory then arrives on an mbarrier; warp 1 waits on it and
// reads. Correct by the PTX memory model (arrive = release, try_wait = acquire).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(double* out) {
  __shared__ double buf[32];
  __shared__ __align__(8) uint64_t bar;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (w == 0) {
    buf[l] = l * 2.0;
    __syncwarp();
    if (l == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar)) : "memory");
  } else {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}"
                   : "=r"(done) : "r"(sa(&bar)) : "memory");
    out[l] = buf[31 - l];
  }
}
int main() {
  double* o;
  cudaMalloc(&o, 256);
  k<<<1, 64>>>(o);
  cudaDeviceSynchronize();
  double h[32];
  cudaMemcpy(h, o, 256, cudaMemcpyDeviceToHost);
  printf("mbar_race: out[0] = %g (expect 62)\n", h[0]);
  return 0;
}
