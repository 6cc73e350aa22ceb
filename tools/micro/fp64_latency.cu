// Dependent-chain latency of FP64 ops on one warp (development microbench).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, double a, double b, long long *cyc) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    x = x + b; x = x + b; x = x + b; x = x + b;
  }
  long long t1 = clock64();
  double y = x;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    y = y * b; y = y * b; y = y * b; y = y * b;
  }
  long long t2 = clock64();
  double z = y;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    z = fma(z, b, a); z = fma(z, b, a); z = fma(z, b, a); z = fma(z, b, a);
  }
  long long t3 = clock64();
  float f = (float)z;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    f = f * 1.0001f + 0.5f; f = f * 1.0001f + 0.5f; f = f * 1.0001f + 0.5f; f = f * 1.0001f + 0.5f;
  }
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  out[threadIdx.x] = z + f;
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 256 * 8); cudaMallocManaged(&c, 64);
  k<<<1, 32>>>(o, 1.0, 1e-9, c); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, 1.0, 1e-9, c); cudaDeviceSynchronize();
  printf("per-op dependent latency (cycles): DADD %.2f DMUL %.2f DFMA %.2f FFMA %.2f\n", c[0] / 4096.0, c[1] / 4096.0,
         c[2] / 4096.0, c[3] / 4096.0);
  return 0;
}
