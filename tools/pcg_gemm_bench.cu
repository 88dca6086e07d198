// Row-block product of the sharded solve at the config-4 / 8-rank shape:
// Q^T (64 x m) = P_full^T (64 x n) * A_r^T, A_r column-major m x n; k_gemm_nt_sk
// tile widths and split counts.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   -I paper_2203_11733_b200/csrc tools/pcg_gemm_bench.cu -o tools/pcg_gemm_bench
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "gbem_gemm_sk.cuh"

using namespace gbem_sk;

template <int TN>
float run(double* C, const double* A, const double* B, int M, int m, long long n, long long mA, int S, int reps) {
  using Sh = SkShape<TN>;
  cudaFuncSetAttribute(k_gemm_nt_sk<TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM);
  long long kchunk = (n + S - 1) / S;
  kchunk = (kchunk + BK - 1) / BK * BK;
  dim3 grid(1, (m + TN - 1) / TN, S);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_gemm_nt_sk<TN><<<grid, Sh::THREADS, Sh::SMEM>>>(C, M, (long long)m * M, A, M, B, mA, M, m, n, kchunk, 1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r)
    k_gemm_nt_sk<TN><<<grid, Sh::THREADS, Sh::SMEM>>>(C, M, (long long)m * M, A, M, B, mA, M, m, n, kchunk, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return ms / reps;
}

float run_bulk(double* C, const double* A, const double* B, int M, int m, long long n, long long mA, int S, int reps) {
  cudaFuncSetAttribute(k_gemm_nt_sk_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SkBulk::SMEM);
  long long kchunk = (n + S - 1) / S;
  kchunk = (kchunk + BK - 1) / BK * BK;
  dim3 grid(1, (m + 63) / 64, S);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_gemm_nt_sk_bulk<<<grid, 128, SkBulk::SMEM>>>(C, M, (long long)m * M, A, M, B, mA, M, m, n, kchunk);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r)
    k_gemm_nt_sk_bulk<<<grid, 128, SkBulk::SMEM>>>(C, M, (long long)m * M, A, M, B, mA, M, m, n, kchunk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return ms / reps;
}

__global__ void fill_rand(double* p, long long n, unsigned seed) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) {
    unsigned x = (unsigned)i * 2654435761u + seed * 40503u;
    x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
    p[i] = (double)(x & 0xffff) / 65536.0 - 0.5;
  }
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 12032;
  const long long n = argc > 2 ? atoll(argv[2]) : 96200;
  const int M = 64;
  const long long mA = (m + 7) / 8 * 8;
  double *A, *B, *C;
  cudaMalloc(&A, sizeof(double) * n * M);
  cudaMalloc(&B, sizeof(double) * n * mA);
  cudaMalloc(&C, sizeof(double) * (size_t)m * M * 16);
  fill_rand<<<(unsigned)((n * M + 255) / 256), 256>>>(A, n * M, 3);
  fill_rand<<<(unsigned)((n * mA + 255) / 256), 256>>>(B, n * mA, 5);
  const double flops = 2.0 * M * m * (double)n;
  for (int S = 1; S <= 8; ++S) {
    float t64 = run<64>(C, A, B, M, m, n, mA, S, 5);
    float t128 = run<128>(C, A, B, M, m, n, mA, S, 5);
    float tb = run_bulk(C, A, B, M, m, n, mA, S, 5);
    printf("m=%d n=%lld S=%d  TN=64: %.3f ms %.2f TF   TN=128: %.3f ms %.2f TF   bulk: %.3f ms %.2f TF\n", m, n, S, t64,
           flops / t64 / 1e9, t128, flops / t128 / 1e9, tb, flops / tb / 1e9);
  }
  {  // bit-for-bit: bulk against the cp.async kernel, S = 3 (ragged last slice when n % 16 != 0)
    const int S = 3;
    double *C1, *C2;
    const size_t cn = (size_t)m * M * S;
    cudaMalloc(&C1, sizeof(double) * cn);
    cudaMalloc(&C2, sizeof(double) * cn);
    long long kchunk = (n + S - 1) / S;
    kchunk = (kchunk + BK - 1) / BK * BK;
    dim3 grid(1, (m + 63) / 64, S);
    k_gemm_nt_sk<64><<<grid, SkShape<64>::THREADS, SkShape<64>::SMEM>>>(C1, M, (long long)m * M, A, M, B, mA, M, m, n, kchunk, 1);
    k_gemm_nt_sk_bulk<<<grid, 128, SkBulk::SMEM>>>(C2, M, (long long)m * M, A, M, B, mA, M, m, n, kchunk);
    cudaDeviceSynchronize();
    double* h1 = (double*)malloc(sizeof(double) * cn);
    double* h2 = (double*)malloc(sizeof(double) * cn);
    cudaMemcpy(h1, C1, sizeof(double) * cn, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2, C2, sizeof(double) * cn, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t i = 0; i < cn; ++i) bad += h1[i] != h2[i];
    printf("bulk vs cp.async: %zu of %zu entries differ (%s)\n", bad, cn, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
