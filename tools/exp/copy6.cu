// copy6.cu — the HBM ceiling of the PW advection's access pattern:
// three fp64 input streams read and three output streams written, same array
// sizes as configs[2] (514^3 padded planes) and configs[4] (1026^2 x 514).
// Kernels (each moves 48 B per interior point, the PW algorithmic bytes):
//   copy6_vec   grid-stride, 16-byte loads/stores, one point pair per thread
//   copy6_rows  like the PW kernel's write side: a thread owns x columns of R rows
//               and streams z; 8-byte stores, 8-byte loads (no reuse)
// Also a 1-read/1-write copy (the MEASURED_PEAKS "copy" pattern) for reference.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/exp/copy6 tools/exp/copy6.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void copy6_vec(const double2* __restrict__ u, const double2* __restrict__ v, const double2* __restrict__ w,
                          double2* __restrict__ a, double2* __restrict__ b, double2* __restrict__ c, long n2) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    const double2 x = __ldcs(u + i), y = __ldcs(v + i), z = __ldcs(w + i);
    __stcs(a + i, x);
    __stcs(b + i, y);
    __stcs(c + i, z);
  }
}

__global__ void copy2_vec(const double2* __restrict__ u, double2* __restrict__ a, long n2) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x)
    __stcs(a + i, __ldcs(u + i));
}

// z-streaming: CTA = 128 x 8 tile (threads 32 x 8, 4 columns... ) streams `pc` planes
__global__ void copy6_zstream(const double* __restrict__ u, const double* __restrict__ v, const double* __restrict__ w,
                              double* __restrict__ a, double* __restrict__ b, double* __restrict__ c, int nx, int ny,
                              int ldx, int nz, int pc) {
  const int x = 1 + blockIdx.x * 128 + threadIdx.x;  // blockDim.x = 128
  const int y = 1 + blockIdx.y * 8 + threadIdx.y;     // blockDim.y = 2, 4 rows each
  const long pe = (long)(ny + 2) * ldx;
  const int z0 = 1 + blockIdx.z * pc, z1 = min(nz, z0 + pc - 1);
  if (x > nx) return;
  for (int z = z0; z <= z1; ++z) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int yy = y + 2 * r;
      if (yy > ny) continue;
      const long o = z * pe + (long)yy * ldx + x;
      a[o] = __ldg(u + o);
      b[o] = __ldg(v + o);
      c[o] = __ldg(w + o);
    }
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 512, nzi = argc > 2 ? atoi(argv[2]) : n;
  const int nx = n, ny = n, nz = nzi, ldx = nx + 2;
  const long elems = (long)(nz + 2) * (ny + 2) * ldx;
  const double pts = (double)nx * ny * nz;
  double* f[6];
  for (int i = 0; i < 6; ++i) {
    CK(cudaMalloc(&f[i], elems * 8));
    CK(cudaMemset(f[i], 0, elems * 8));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](const char* name, double bytes, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    const int reps = 20;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("{\"kernel\": \"%s\", \"grid\": \"%dx%dx%d\", \"ms\": %.4f, \"GBps\": %.1f}\n", name, nx, ny, nz, ms,
           bytes / (ms * 1e-3) / 1e9);
  };
  const long n2 = elems / 2;
  for (int k = 1; k <= 8; k *= 2)
    timeit(k == 1 ? "copy6_vec_x1" : k == 2 ? "copy6_vec_x2" : k == 4 ? "copy6_vec_x4" : "copy6_vec_x8",
           48.0 * elems, [&] { copy6_vec<<<sms * k, 512>>>((double2*)f[0], (double2*)f[1], (double2*)f[2], (double2*)f[3], (double2*)f[4], (double2*)f[5], n2); });
  timeit("copy2_vec_x4", 16.0 * elems, [&] { copy2_vec<<<sms * 4, 512>>>((double2*)f[0], (double2*)f[3], n2); });
  for (int pc : {32, 64, 128})
    timeit(pc == 32 ? "copy6_zstream_pc32" : pc == 64 ? "copy6_zstream_pc64" : "copy6_zstream_pc128", 48.0 * pts, [&] {
      dim3 g((nx + 127) / 128, (ny + 7) / 8, (nz + pc - 1) / pc);
      copy6_zstream<<<g, dim3(128, 2)>>>(f[0], f[1], f[2], f[3], f[4], f[5], nx, ny, ldx, nz, pc);
    });
  return 0;
}
