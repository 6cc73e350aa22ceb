// Live peak measurement for the roofline denominators (MEASURED_PEAKS.json
// has no FP64/FP32 CUDA-core numbers): FP64 DADD issue rate (the relevant
// peak for -fmad=false code: one flop per FP64 instruction), FP64 DFMA and
// FP32 FFMA flop rates (2 flops per FMA).  Each thread runs 8 independent
// dependency chains so the pipes, not latency, bound the kernel.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "dmath.cuh"

namespace {

constexpr int kChains = 8;

__global__ void k_dadd(double *out, int iters, double c) {
  double x[kChains];
#pragma unroll
  for (int j = 0; j < kChains; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kChains; ++j) x[j] = x[j] + c;
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) s += x[j];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_dfma(double *out, int iters, double a, double c) {
  double x[kChains];
#pragma unroll
  for (int j = 0; j < kChains; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kChains; ++j) x[j] = fma(x[j], a, c);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) s += x[j];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_ffma(float *out, int iters, float a, float c) {
  float x[kChains];
#pragma unroll
  for (int j = 0; j < kChains; ++j) x[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kChains; ++j) x[j] = fmaf(x[j], a, c);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) s += x[j];
  if (s == 1234.5f) out[0] = s;
}

// Random gathers over an L1/L2-resident working set (the
// sampler's cell-word and corner loads): every thread runs 8 independent
// LCG address streams; E = 2, 4, 16 or 32 bytes per load (32 = two
// adjacent 16-byte loads, one 32-byte sector).
template <int E>
__global__ void k_gather(const uint4 *buf, uint32_t mask, int iters, uint32_t *out) {
  uint32_t st[kChains], acc = 0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) st[j] = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + j * 40503u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < kChains; ++j) {
      st[j] = st[j] * 1664525u + 1013904223u;
      const uint32_t idx = (st[j] >> 4) & mask;
      if (E == 2) {
        acc += __ldg(reinterpret_cast<const uint16_t *>(buf) + idx);
      } else if (E == 4) {
        acc += __ldg(reinterpret_cast<const uint32_t *>(buf) + idx);
      } else if (E == 16) {
        const uint4 v = __ldg(buf + idx);
        acc += v.x ^ v.w;
      } else {
        const uint4 v = __ldg(buf + 2 * idx), w = __ldg(buf + 2 * idx + 1);
        acc += v.x ^ w.w;
      }
      st[j] ^= acc & 1u;  // keep the loads live without serialising the chains
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <typename F>
double rate(F launch, double ops) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();  // warm-up
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return 3.0 * ops / (ms * 1e-3);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void k_sqrt_check(uint64_t n, uint64_t seed, unsigned long long *bad, unsigned long long *first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix64(seed ^ mix64(i));
    double x;
    switch (i % 3) {
      case 0:  // any finite non-negative double (subnormals included)
        x = __longlong_as_double((long long)(r & 0x7fefffffffffffffull));
        break;
      case 1: {  // s^2 +- k ulp: inputs whose sqrt sits next to a rounding midpoint
        const double s = 1.0 + (double)(r >> 11) * 0x1p-53;  // [1, 2)
        const int sh = (int)((r >> 3) & 255) - 128;
        const double sq = __dmul_rn(s, s) * exp2((double)(2 * sh));
        x = __longlong_as_double(__double_as_longlong(sq) + (long long)(r & 7) - 3);
        break;
      }
      default: {  // squared distances of the dock path
        x = 1e-4 + (double)(r >> 11) * 0x1p-53 * 1e4;
        break;
      }
    }
    if (!(x >= 0.0)) continue;
    const double a = vsd::dsqrt(x), b = sqrt(x);
    // dsqrt_dist2 (k_flatten's pair distances) on its domain: 0 or >= 2^-1000
    const double a2 = (x == 0.0 || x >= 0x1p-1000) ? vsd::dsqrt_dist2(x) : b;
    if (__double_as_longlong(a) != __double_as_longlong(b) || __double_as_longlong(a2) != __double_as_longlong(b)) {
      if (atomicAdd(bad, 1ull) == 0) *first = (unsigned long long)__double_as_longlong(x);
    }
  }
}

__global__ void k_div_check(uint64_t n, uint64_t seed, unsigned long long *bad, unsigned long long *first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix64(seed ^ mix64(i)), r2 = mix64(r);
    double a, b;
    switch (i % 3) {
      case 0: {  // random doubles in the fast-path range
        const long long ea = (long long)((r >> 52) % 800) - 400 + 1023, eb = (long long)((r2 >> 52) % 800) - 400 + 1023;
        a = __longlong_as_double((long long)((r & 0x800fffffffffffffull) | ((uint64_t)ea << 52)));
        b = __longlong_as_double((long long)((r2 & 0x800fffffffffffffull) | ((uint64_t)eb << 52)));
        break;
      }
      case 1: {  // a = q * b +- k ulp: quotients next to rounding midpoints
        const double q = 1.0 + (double)(r >> 11) * 0x1p-53;
        b = 1.0 + (double)(r2 >> 11) * 0x1p-53;
        const double qb = __dmul_rn(q, b);
        a = __longlong_as_double(__double_as_longlong(qb) + (long long)(r2 & 7) - 3);
        if (r & 1) a = -a;
        break;
      }
      default: {  // the dock path: unit-vector components / norms
        a = ((double)(r >> 11) * 0x1p-53 - 0.5) * 8.0;
        b = 1e-3 + (double)(r2 >> 11) * 0x1p-53 * 4.0;
        if ((r & 15) == 0) a = (r & 16) ? 0.0 : -0.0;
        break;
      }
    }
    if (!(vsd::drange_ok(a) && vsd::drange_ok(b)) || b == 0.0) continue;
    const double x = vsd::ddiv_r(a, b, vsd::drecip(b)), y = a / b;
    if (__double_as_longlong(x) != __double_as_longlong(y)) {
      if (atomicAdd(bad, 1ull) == 0) *first = (unsigned long long)__double_as_longlong(a);
    }
  }
}

}  // namespace

extern "C" int vs_selftest_div(int device, uint64_t n, uint64_t seed, uint64_t *mismatches, double *first_bad) {
  if (cudaSetDevice(device) != cudaSuccess) return 2;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  unsigned long long *buf = nullptr;
  if (cudaMalloc(&buf, 16) != cudaSuccess) return 3;
  cudaMemset(buf, 0, 16);
  k_div_check<<<sms * 8, 256>>>(n, seed, buf, buf + 1);
  unsigned long long h[2] = {0, 0};
  cudaMemcpy(h, buf, 16, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  if (mismatches) *mismatches = h[0];
  if (first_bad) {
    long long v = (long long)h[1];
    std::memcpy(first_bad, &v, sizeof v);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

extern "C" int vs_selftest_sqrt(int device, uint64_t n, uint64_t seed, uint64_t *mismatches, double *first_bad) {
  if (cudaSetDevice(device) != cudaSuccess) return 2;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  unsigned long long *buf = nullptr;
  if (cudaMalloc(&buf, 16) != cudaSuccess) return 3;
  cudaMemset(buf, 0, 16);
  k_sqrt_check<<<sms * 8, 256>>>(n, seed, buf, buf + 1);
  unsigned long long h[2] = {0, 0};
  cudaMemcpy(h, buf, 16, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  if (mismatches) *mismatches = h[0];
  if (first_bad) {
    long long v = (long long)h[1];
    std::memcpy(first_bad, &v, sizeof v);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

extern "C" int vs_measure_peaks(int device, double out[3]) {
  if (cudaSetDevice(device) != cudaSuccess) return 2;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  double *dbuf = nullptr;
  cudaMalloc(&dbuf, 64);
  const double lanes = static_cast<double>(blocks) * threads;
  out[0] = rate([&] { k_dadd<<<blocks, threads>>>(dbuf, iters, 1e-9); }, lanes * iters * kChains);
  out[1] = rate([&] { k_dfma<<<blocks, threads>>>(dbuf, iters, 0.999999, 1e-9); }, 2.0 * lanes * iters * kChains);
  out[2] = rate([&] { k_ffma<<<blocks, threads>>>(reinterpret_cast<float *>(dbuf), iters, 0.999999f, 1e-9f); },
                2.0 * lanes * iters * kChains);
  cudaFree(dbuf);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// Random-gather rate (loads per second) of E-byte loads over a ws_bytes
// working set (rounded down to a power of two elements).
extern "C" int vs_measure_gather(int device, int64_t ws_bytes, int32_t elem_bytes, double *loads_per_s) {
  if (cudaSetDevice(device) != cudaSuccess) return 2;
  if (!loads_per_s || (elem_bytes != 2 && elem_bytes != 4 && elem_bytes != 16 && elem_bytes != 32)) return 1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  uint64_t elems = 1;
  while (elems * 2 * elem_bytes <= (uint64_t)ws_bytes) elems *= 2;
  uint4 *buf = nullptr;
  if (cudaMalloc(&buf, elems * elem_bytes + 64) != cudaSuccess) return 3;
  cudaMemset(buf, 1, elems * elem_bytes + 64);
  uint32_t *out = nullptr;
  cudaMalloc(&out, 64);
  const int blocks = sms * 8, threads = 256, iters = 256;
  const uint32_t mask = (uint32_t)(elems - 1);
  const double loads = (double)blocks * threads * iters * kChains;
  double r = 0.0;
  switch (elem_bytes) {
    case 2: r = rate([&] { k_gather<2><<<blocks, threads>>>(buf, mask, iters, out); }, loads); break;
    case 4: r = rate([&] { k_gather<4><<<blocks, threads>>>(buf, mask, iters, out); }, loads); break;
    case 16: r = rate([&] { k_gather<16><<<blocks, threads>>>(buf, mask, iters, out); }, loads); break;
    default: r = rate([&] { k_gather<32><<<blocks, threads>>>(buf, mask, iters, out); }, loads); break;
  }
  *loads_per_s = r;
  cudaFree(buf);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

