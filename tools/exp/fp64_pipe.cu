// Measures the sm_100a fp64 pipe: DADD latency (one dependent chain per
// thread) and throughput (16 independent chains per thread, all SMs busy),
// plus SHFL latency — the constants behind the temporal-blocking analysis
// (DESIGN.md §6.2, §12). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dadd_latency(double* out, long long* cycles, int n) {
  double x = out[threadIdx.x];
  const double y = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = __dadd_rn(x, y);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

__global__ void shfl_latency(double* out, long long* cycles, int n) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = __shfl_up_sync(0xffffffffu, x, 1);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

__global__ void dadd_throughput(double* out, int n) {
  double x[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) x[c] = out[threadIdx.x] + c;
  const double y = 1.0000001;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < 16; ++c) x[c] = __dadd_rn(x[c], y);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * 1 << 24);
  cudaMemset(out, 0, sizeof(double) * 1 << 24);
  cudaMalloc(&cyc, sizeof(long long));
  const int n = 4096;
  long long c = 0;
  dadd_latency<<<1, 32>>>(out, cyc, n);
  dadd_latency<<<1, 32>>>(out, cyc, n);
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double lat = (double)c / (16.0 * n);
  shfl_latency<<<1, 32>>>(out, cyc, n);
  shfl_latency<<<1, 32>>>(out, cyc, n);
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double slat = (double)c / (16.0 * n);
  const int blocks = sms * 8, threads = 256, nt = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dadd_throughput<<<blocks, threads>>>(out, 100);
  cudaEventRecord(e0);
  dadd_throughput<<<blocks, threads>>>(out, nt);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)blocks * threads * nt * 16;
  printf("{\"sms\": %d, \"clock_mhz_attr\": %d, \"dadd_latency_cycles\": %.2f, \"shfl_latency_cycles\": %.2f, "
         "\"dadd_tops\": %.3f, \"dadd_per_clk_per_sm_at_attr_clock\": %.1f}\n",
         sms, clk / 1000, lat, slat, ops / (ms * 1e-3) / 1e12, ops / (ms * 1e-3) / sms / (clk * 1e3));
  return 0;
}
