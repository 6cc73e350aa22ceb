// Max relative error of rsqrt.approx.ftz.f64 (MUFU.RSQ64H) against a correctly
// rounded reference, over random doubles in [2^-20, 2^40) (development).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rsqrt_err rsqrt_err.cu
#include <cstdio>
#include <cstdint>
#include <cmath>

__global__ void k(unsigned long long seed, long long n, double *maxrel) {
  double m = 0.0;
  unsigned long long s = seed ^ (blockIdx.x * 0x9E3779B97F4A7C15ull + threadIdx.x * 0xBF58476D1CE4E5B9ull);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const int ex = (int)(s % 60) - 20;
    const double mant = 1.0 + (double)(s >> 11) * 0x1p-53;
    const double x = ldexp(mant, ex);
    double y0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
    const double d = x * y0;           // filter distance
    const double r = sqrt(x);          // IEEE
    const double rel = fabs(d - r) / r;
    m = fmax(m, rel);
  }
  // block max
  __shared__ double sm[256];
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    unsigned long long *p = (unsigned long long *)maxrel;
    atomicMax(p, __double_as_longlong(sm[0]));
  }
}

int main() {
  double *d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  k<<<148 * 8, 256>>>(12345, 4000000000LL, d);
  double h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("max rel err of x*rsqrt.approx(x): %.6e = 2^%.3f\n", h, log2(h));
  return 0;
}
