// gemm_bench.cu — microbenchmark of the DMMA trailing-update GEMM
// (paper_2203_11733_b200/csrc/gbem_dmma_gemm.cuh) against cuBLAS DGEMM/DSYRK.
//   ./gemm_bench [m=11264] [k=128]
// C (m x m, lower tiles) -= A (m x k) A^T, column-major.
#include <cublas_v2.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2203_11733_b200/csrc/gbem_dmma_gemm.cuh"

using namespace gbem_gemm;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                 \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

__global__ void fill(double* p, long long n, unsigned seed) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) {
    unsigned x = (unsigned)(i * 2654435761u) ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    p[i] = (x & 0xffffff) / 16777216.0 - 0.5;
  }
}

int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 11264;
  int k = argc > 2 ? atoi(argv[2]) : 128;
  long long ldc = m;
  double *C, *A, *C2;
  CK(cudaMalloc(&C, sizeof(double) * ldc * m));
  CK(cudaMalloc(&C2, sizeof(double) * ldc * m));
  CK(cudaMalloc(&A, sizeof(double) * (long long)m * k));
  fill<<<(unsigned)((ldc * m + 255) / 256), 256>>>(C, ldc * m, 1);
  fill<<<(unsigned)(((long long)m * k + 255) / 256), 256>>>(A, (long long)m * k, 2);
  CK(cudaMemcpy(C2, C, sizeof(double) * ldc * m, cudaMemcpyDeviceToDevice));
  CK(cudaFuncSetAttribute(k_gemm_nt<kSub, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Shape<64>::SMEM));
  int nt = (m + BM - 1) / BM;
  long long ntiles = lower_tiles_before<64>(nt);
  double flops = (double)m * (m + 1) / 2 * k * 2;  // lower triangle incl. diagonal, useful flops
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it)
      k_gemm_nt<kSub, 64><<<(unsigned)ntiles, GEMM_THREADS, Shape<64>::SMEM>>>(C, ldc, A, m, A, m, m, m, k, 1, 0);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kernel\": \"k_gemm_nt<kSub> lower\", \"m\": %d, \"k\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n", m, k,
           ms / 10, flops / (ms / 10 * 1e-3) / 1e12);
  }
  auto run_gen = [&](auto kern, int TBM, int TBN, int threads, size_t smem, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long ntr = (m + TBM - 1) / TBM;
    long long nb = (long long)(TBM / TBN) * ntr * (ntr + 1) / 2;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      for (int it = 0; it < 10; ++it) kern<<<(unsigned)nb, threads, smem>>>(C, ldc, A, m, m, k, 0, 0, nullptr, 0LL);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("{\"kernel\": \"%s\", \"m\": %d, \"k\": %d, \"ms\": %.4f, \"tflops\": %.2f, \"err\": \"%s\"}\n", name, m, k,
           ms / 10, flops / (ms / 10 * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
#define GEN(a, b, c, d, e, f) \
  run_gen(k_syrk_gen<a, b, c, d, e, f>, a, b, 32 * c * d, GenShape<a, b, c, d, e>::SMEM, "gen " #a "x" #b " w" #c "x" #d " st" #e " min" #f)
  GEN(64, 64, 2, 2, 2, 4);
#define BULK(a, b, c) \
  run_gen(k_syrk_bulk<a, b, c>, 64, 64, 128, BulkShape<a, b>::SMEM, "bulk bks" #a " st" #b " min" #c)
  if (getenv("GEMM_BENCH_BULK_ONLY")) {
    run_gen(k_syrk_bulk<16, 3, 4, true>, 64, 64, 128, BulkShape<16, 3>::SMEM, "bulk-split bks16 st3 min4");
    goto check;
  }
  if (k % 16 == 0 && m % 2 == 0) {
    BULK(8, 4, 4);
    BULK(8, 6, 4);
    BULK(16, 3, 4);
    run_gen(k_syrk_bulk<16, 3, 4, true>, 64, 64, 128, BulkShape<16, 3>::SMEM, "bulk-split bks16 st3 min4");
    run_gen(k_syrk_bulk<8, 4, 4, true>, 64, 64, 128, BulkShape<8, 4>::SMEM, "bulk-split bks8 st4 min4");
  }
  if (getenv("GEMM_BENCH_SHORT")) goto check;
  GEN(64, 64, 2, 2, 3, 3);
  GEN(128, 128, 4, 2, 2, 1);
  GEN(128, 128, 2, 4, 2, 1);
  GEN(96, 96, 3, 2, 2, 2);
  GEN(64, 64, 2, 2, 4, 3);
  GEN(64, 64, 2, 2, 3, 4);
  GEN(64, 64, 2, 2, 2, 5);
check:
  cublasHandle_t h;
  cublasCreate(&h);
  double alpha = -1.0, beta = 1.0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it)
      cublasDsyrk(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, m, k, &alpha, A, m, &beta, C2, ldc);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kernel\": \"cublasDsyrk lower\", \"m\": %d, \"k\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n", m, k,
           ms / 10, flops / (ms / 10 * 1e-3) / 1e12);
  }
  // correctness: one application each from the same start
  fill<<<(unsigned)((ldc * m + 255) / 256), 256>>>(C, ldc * m, 1);
  fill<<<(unsigned)((ldc * m + 255) / 256), 256>>>(C2, ldc * m, 1);
  k_syrk_gen<64, 64, 2, 2, 2, 4><<<(unsigned)((long long)((m + 63) / 64) * ((m + 63) / 64 + 1) / 2), 128,
                                   GenShape<64, 64, 2, 2, 2>::SMEM>>>(C, ldc, A, m, m, k, 0, 0);
  cublasDsyrk(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, m, k, &alpha, A, m, &beta, C2, ldc);
  CK(cudaDeviceSynchronize());
  std::vector<double> h1((size_t)ldc * m), h2((size_t)ldc * m);
  CK(cudaMemcpy(h1.data(), C, sizeof(double) * ldc * m, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2.data(), C2, sizeof(double) * ldc * m, cudaMemcpyDeviceToHost));
  double md = 0;
  for (int c = 0; c < m; ++c)
    for (int r = c; r < m; ++r) md = fmax(md, fabs(h1[(size_t)c * ldc + r] - h2[(size_t)c * ldc + r]));
  printf("{\"max_abs_diff_vs_cublas\": %.3e}\n", md);
  if (k % 16 == 0 && m % 2 == 0) {
    fill<<<(unsigned)((ldc * m + 255) / 256), 256>>>(C2, ldc * m, 1);
    k_syrk_bulk<16, 3, 4, true><<<(unsigned)((long long)((m + 63) / 64) * ((m + 63) / 64 + 1) / 2), 128, BulkShape<16, 3>::SMEM>>>(
        C2, ldc, A, m, m, k, 0, 0);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h2.data(), C2, sizeof(double) * ldc * m, cudaMemcpyDeviceToHost));
    md = 0;
    for (int c = 0; c < m; ++c)
      for (int r = c; r < m; ++r) md = fmax(md, fabs(h1[(size_t)c * ldc + r] - h2[(size_t)c * ldc + r]));
    printf("{\"max_abs_diff_bulk_vs_gen\": %.3e}\n", md);
  }
  return 0;
}
