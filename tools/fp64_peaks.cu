// Microbenchmark: FP64 DFMA pipe peak and DMMA (mma.sync f64 m8n8k4) peak on one B200.
// Used once to fill the FP64 roofline denominators (MEASURED_PEAKS.json has only bf16/HBM).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void dfma_loop(double* out, int iters, double s) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      a0 = fma(a0, s, 1e-9); a1 = fma(a1, s, 1e-9); a2 = fma(a2, s, 1e-9); a3 = fma(a3, s, 1e-9);
      a4 = fma(a4, s, 1e-9); a5 = fma(a5, s, 1e-9); a6 = fma(a6, s, 1e-9); a7 = fma(a7, s, 1e-9);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[r][0]), "+d"(c[r][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int r = 0; r < 8; ++r) s += c[r][0] + c[r][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ double rsq(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x * y, y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}
__global__ void rsqrt_loop(double* out, int iters) {
  double x = 1.0 + threadIdx.x, acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int i = 0; i < iters; ++i) {
    acc0 += rsq(x + acc0 * 1e-30); acc1 += rsq(x + 1.0 + acc1 * 1e-30);
    acc2 += rsq(x + 2.0 + acc2 * 1e-30); acc3 += rsq(x + 3.0 + acc3 * 1e-30);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
__global__ void rsqrt_acc(double* out, const double* in, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { double x = in[i]; out[i] = rsq(x) - 1.0 / sqrt(x); }
}
__global__ void log_loop(double* out, int iters) {
  double x = 1.5 + threadIdx.x, acc0 = 0, acc1 = 0;
  for (int i = 0; i < iters; ++i) { acc0 += log(x + acc0 * 1e-30); acc1 += log(x + 0.5 + acc1 * 1e-30); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, p.multiProcessorCount, clk);
  double* out; CK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256;
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    int it = 20000;
    dfma_loop<<<blocks, threads>>>(out, 100, 0.999);
    cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, it, 0.999); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 64 * it * (double)blocks * threads;
    printf("{\"kernel\": \"dfma\", \"tflops\": %.2f, \"ms\": %.2f}\n", fl / ms / 1e9, ms);
    it = 5000;
    dmma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0); dmma_loop<<<blocks, threads>>>(out, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    fl = 512.0 * 8 * it * (double)blocks * (threads / 32);
    printf("{\"kernel\": \"dmma_m8n8k4\", \"tflops\": %.2f, \"ms\": %.2f}\n", fl / ms / 1e9, ms);
    it = 20000;
    cudaEventRecord(e0); rsqrt_loop<<<blocks, threads>>>(out, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kernel\": \"rsqrt_custom\", \"grsqrt_per_s\": %.1f}\n", 4.0 * it * blocks * threads / ms / 1e6);
    it = 5000;
    cudaEventRecord(e0); log_loop<<<blocks, threads>>>(out, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kernel\": \"log_f64\", \"glog_per_s\": %.1f}\n", 2.0 * it * blocks * threads / ms / 1e6);
  }
  // rsqrt accuracy sweep
  int n = 1 << 22; double *in, *o2; CK(cudaMalloc(&in, n * 8)); CK(cudaMalloc(&o2, n * 8));
  double* h = new double[n];
  for (int i = 0; i < n; ++i) h[i] = 1e-12 * pow(1e26, (double)i / n) * (1.0 + 0.37 * (i % 7));
  cudaMemcpy(in, h, n * 8, cudaMemcpyHostToDevice);
  rsqrt_acc<<<(n + 255) / 256, 256>>>(o2, in, n); double* r = new double[n];
  cudaMemcpy(r, o2, n * 8, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < n; ++i) { double rel = fabs(r[i]) * sqrt(h[i]); if (rel > mx) mx = rel; }
  printf("{\"rsqrt_custom_max_rel_err\": %.3e}\n", mx);
  return 0;
}
