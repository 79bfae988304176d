// How long do __nanosleep(t) and mbarrier.try_wait(..., hint) really park a warp on sm_100a?
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(long long* out, int mode, unsigned t, int n) {
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
  __syncthreads();
  long long t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int i = 0; i < n; ++i) {
    if (mode == 0) {
      __nanosleep(t);
    } else {
      uint32_t done;
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0, %2;\nselp.u32 %0,1,0,p;\n}"
                   : "=r"(done) : "r"(sa(&bar)), "r"(t) : "memory");
      if (done) out[2] = 1;
    }
  }
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) { out[0] = clock64() - t0; out[1] = (long long)(g1 - g0); }
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[3];
  for (int mode = 0; mode < 2; ++mode)
    for (unsigned t : {100u, 1000u, 10000u, 100000u}) {
      cudaMemset(d, 0, 64);
      k<<<1, 32>>>(d, mode, t, 1000);
      cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
      printf("%s t=%u ns: %.1f ns per call (%.0f cycles)\n", mode ? "try_wait hint" : "nanosleep", t, h[1] / 1000.0,
             h[0] / 1000.0);
    }
  return 0;
}
