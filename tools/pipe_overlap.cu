// Do the FP64 FMA pipe (DFMA) and the FP64 tensor path (DMMA) run concurrently
// on one SM?  Times a DFMA-only kernel, a DMMA-only kernel, both on two streams
// at once, and one kernel whose warps interleave the two.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_k(double* out, int iters, double s) {
  double a[8];
  for (int r = 0; r < 8; ++r) a[r] = threadIdx.x * 1e-3 + r;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = fma(a[q], s, 1e-9);
  double t = 0;
  for (int r = 0; r < 8; ++r) t += a[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void dmma_k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int r = 0; r < 8; ++r)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[r][0]), "+d"(c[r][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int r = 0; r < 8; ++r) s += c[r][0] + c[r][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void mixed_k(double* out, int iters, double sc) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2] = {};
  double f[8];
  for (int r = 0; r < 8; ++r) f[r] = threadIdx.x * 1e-3 + r;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[r][0]), "+d"(c[r][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int q = 0; q < 8; ++q) f[q] = fma(f[q], sc, 1e-9);
    }
  }
  double s = 0;
  for (int r = 0; r < 8; ++r) s += c[r][0] + c[r][1] + f[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 4, th = 256, itf = 4000, itm = 2000;
  auto tm = [&](auto f) { f(); cudaDeviceSynchronize(); cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); return ms; };
  float a = tm([&] { dfma_k<<<blocks, th>>>(out, itf, 0.999); });
  float b = tm([&] { dmma_k<<<blocks, th>>>(out, itm); });
  float c = tm([&] { cudaEventRecord(e0, 0); dfma_k<<<blocks, th, 0, s1>>>(out, itf, 0.999); dmma_k<<<blocks, th, 0, s2>>>(out + (1 << 20), itm); cudaDeviceSynchronize(); });
  float d = tm([&] { mixed_k<<<blocks, th>>>(out, itm, 0.999); });
  double dfma_fl = 2.0 * 64 * itf * blocks * th, dmma_fl = 512.0 * 8 * itm * blocks * (th / 32);
  double mixed_fl = 512.0 * 8 * itm * blocks * (th / 32) + 2.0 * 64 * itm * blocks * th;
  printf("dfma alone %.3f ms (%.1f TF)\ndmma alone %.3f ms (%.1f TF)\nboth streams %.3f ms (sum alone %.3f)\n", a, dfma_fl / a / 1e9, b,
         dmma_fl / b / 1e9, c, a + b);
  printf("mixed warps %.3f ms: %.1f TF combined (dmma part %.1f ms alone-equivalent)\n", d, mixed_fl / d / 1e9, b);
  return 0;
}
