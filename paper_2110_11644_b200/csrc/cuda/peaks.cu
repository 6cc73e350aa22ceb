// Live peak measurement for the roofline denominators (MEASURED_PEAKS.json
// has no FP64/FP32 CUDA-core numbers): FP64 DADD issue rate (the relevant
// peak for -fmad=false code: one flop per FP64 instruction), FP64 DFMA and
// FP32 FFMA flop rates (2 flops per FMA).  Each thread runs 8 independent
// dependency chains so the pipes, not latency, bound the kernel.
#include <cuda_runtime.h>

#include <cstdint>

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

}  // namespace

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
