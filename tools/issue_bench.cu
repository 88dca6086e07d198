// Does an FP64 instruction (2 cycles of the half-rate FP64 pipe per warp instruction) also hold
// the scheduler's issue port for 2 cycles?  8 independent DFMA chains per thread with 0 / 1 / 2
// independent integer (IMAD) or FP32 (FFMA) instructions interleaved per DFMA, and the far-field
// node mix (4 FP64 + MUFU.RSQ64H, with and without one extra ALU instruction).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o issue_bench tools/issue_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIters = 2048;
template <int NI, int NF>
__global__ void k_mix(double* out, double c, int ic, float fc) {
  double y[8];
  int z[8];
  float f[8];
  for (int k = 0; k < 8; ++k) {
    y[k] = 1.0 + threadIdx.x * 1e-3 + k;
    z[k] = threadIdx.x + k;
    f[k] = threadIdx.x * 0.5f + k;
  }
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      y[k] = fma(y[k], 0.999, c);
#pragma unroll
      for (int j = 0; j < NI; ++j) z[(k + j) & 7] = z[(k + j) & 7] * ic + it;
#pragma unroll
      for (int j = 0; j < NF; ++j) f[(k + j) & 7] = fmaf(f[(k + j) & 7], fc, 1.0f);
    }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += y[k] + z[k] + f[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// far-field node: x = fma(r2, k, cw); y = rsq(x); acc = fma(y, fma(-(x y), y, 3), acc)
template <int EXTRA>
__global__ void k_node(double* out, double r2, int ic) {
  double cw[8], acc[8];
  int z = threadIdx.x;
  for (int k = 0; k < 8; ++k) {
    cw[k] = 1.0 + threadIdx.x * 1e-3 + k;
    acc[k] = 0.0;
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double x = fma(r2, 1.0 + k, cw[k]);
      double y;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
      acc[k] = fma(y, fma(-(x * y), y, 3.0), acc[k]);
#pragma unroll
      for (int j = 0; j < EXTRA; ++j) z = z * ic + it;
    }
    r2 += 1e-3;
  }
  double s = z;
  for (int k = 0; k < 8; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// the same node with the seed's low word taken from a register that stays zero (the MUFU writes
// the high word in place; no per-node zeroing instruction)
__device__ __forceinline__ double rsq_seed_z(double x, unsigned zlo) {
  double y, r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(zlo), "r"((unsigned)__double2hiint(y)));
  return r;
}
template <int EXTRA>
__global__ void k_node_z(double* out, double r2, int ic) {
  double cw[8], acc[8];
  int z = threadIdx.x;
  unsigned zlo;
  asm volatile("mov.u32 %0, 0;" : "=r"(zlo));
  for (int k = 0; k < 8; ++k) {
    cw[k] = 1.0 + threadIdx.x * 1e-3 + k;
    acc[k] = 0.0;
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double x = fma(r2, 1.0 + k, cw[k]);
      const double y = rsq_seed_z(x, zlo);
      acc[k] = fma(y, fma(-(x * y), y, 3.0), acc[k]);
#pragma unroll
      for (int j = 0; j < EXTRA; ++j) z = z * ic + it;
    }
    r2 += 1e-3;
  }
  double s = z;
  for (int k = 0; k < 8; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 8 * sms * 8 * 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, int warps_per_sm, auto... args) {
    const int blocks = sms * warps_per_sm / 4;  // 128-thread CTAs
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      kern<<<blocks, 128>>>(out, args...);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    // cycles per (DFMA | node) per scheduler: each scheduler runs warps_per_sm / 4 warps
    const double groups = (double)kIters * 8 * (warps_per_sm / 4.0);
    printf("{\"kernel\": \"%s\", \"warps_per_sm\": %d, \"ms\": %.3f, \"cycles_per_group_per_scheduler\": %.2f}\n", name,
           warps_per_sm, ms, ms * 1e-3 * clk * 1e3 / groups);
  };
  for (int w : {16, 32}) {
    run("DFMA", k_mix<0, 0>, w, 1e-9, 3, 0.5f);
    run("DFMA + 1 IMAD", k_mix<1, 0>, w, 1e-9, 3, 0.5f);
    run("DFMA + 2 IMAD", k_mix<2, 0>, w, 1e-9, 3, 0.5f);
    run("DFMA + 1 FFMA", k_mix<0, 1>, w, 1e-9, 3, 0.5f);
    run("DFMA + 1 IMAD + 1 FFMA", k_mix<1, 1>, w, 1e-9, 3, 0.5f);
    run("node (3 DFMA + DMUL + MUFU.RSQ64H)", k_node<0>, w, 0.5, 3);
    run("node, persistent zero low word", k_node_z<0>, w, 0.5, 3);
    run("node + 1 IMAD", k_node<1>, w, 0.5, 3);
    run("node + 2 IMAD", k_node<2>, w, 0.5, 3);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
