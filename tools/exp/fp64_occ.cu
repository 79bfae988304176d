// fp64 pipe throughput vs warps per SM and independent chains per thread, with
// the operand pattern of the Jacobi level update (two distinct register pairs
// per DADD, no constant operand): can 8 warps per SM (the 255-register
// T-blocked kernel) feed the pipe at all?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o fp64_occ fp64_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void chains(double* out, int n) {
  double x[K], z[K];
#pragma unroll
  for (int c = 0; c < K; ++c) {
    x[c] = out[threadIdx.x] + c;
    z[c] = out[threadIdx.x + 1] * c;
  }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      x[c] = __dadd_rn(x[c], z[c]);
      z[c] = __dadd_rn(z[c], x[(c + 1) % K]);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < K; ++c) s += x[c] + z[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K>
void run(int sms, int warps, double* out) {
  const int n = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chains<K><<<sms, 32 * warps>>>(out, 10);
  cudaEventRecord(e0);
  chains<K><<<sms, 32 * warps>>>(out, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warp_instr = (double)sms * warps * n * 2 * K;
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("{\"warps_per_sm\": %d, \"chains\": %d, \"ms\": %.3f, \"fp64_warp_instr_per_clk_per_sm\": %.3f}\n", warps, 2 * K,
         ms, warp_instr / sms / cycles);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * (1 << 22));
  cudaMemset(out, 0, sizeof(double) * (1 << 22));
  for (int w : {4, 8, 12, 16, 32}) {
    run<2>(sms, w, out);
    run<4>(sms, w, out);
    run<8>(sms, w, out);
  }
  return 0;
}
