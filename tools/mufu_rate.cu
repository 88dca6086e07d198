// Throughput of the far-field node's special-function candidates on one B200:
// MUFU.RSQ64H (rsqrt.approx.f64), FP32 MUFU.RSQ with the F2F conversions, and
// the integer-seed reciprocal square root, as operations per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kChains = 8, kIters = 4096;
__global__ void k_rsq64(double* out, double c) {
  double y[kChains];
  for (int k = 0; k < kChains; ++k) y[k] = 1.0 + threadIdx.x * 1e-3 + k;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int k = 0; k < kChains; ++k) {
      double r;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y[k]));
      y[k] = r + c;
    }
  double s = 0;
  for (int k = 0; k < kChains; ++k) s += y[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_rsq32cvt(double* out, double c) {
  double y[kChains];
  for (int k = 0; k < kChains; ++k) y[k] = 1.0 + threadIdx.x * 1e-3 + k;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int k = 0; k < kChains; ++k) y[k] = (double)rsqrtf((float)y[k]) + c;
  double s = 0;
  for (int k = 0; k < kChains; ++k) s += y[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dadd(double* out, double c) {
  double y[kChains];
  for (int k = 0; k < kChains; ++k) y[k] = 1.0 + threadIdx.x * 1e-3 + k;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int k = 0; k < kChains; ++k) y[k] = y[k] * 0.999 + c;
  double s = 0;
  for (int k = 0; k < kChains; ++k) s += y[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out; cudaMalloc(&out, 8 * 148 * 8 * 256);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*k)(double*, double), double ops_per_inner) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k<<<sms * 8, 256>>>(out, 1e-9);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)sms * 8 * 256 * kIters * kChains * ops_per_inner;
      if (rep) printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"per_s\": %.3e, \"per_clk_per_sm\": %.2f}\n", name, ms,
                      ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
  };
  run("rsqrt.approx.f64 (+DADD)", k_rsq64, 1.0);
  run("cvt.f32.f64 + rsqrtf + cvt.f64.f32 (+DADD)", k_rsq32cvt, 1.0);
  run("DFMA", k_dadd, 1.0);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
