// Bit-for-bit check of k_syrk_bulk against k_syrk_gen over shapes (ragged tiles, odd rows), repeated.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../paper_2203_11733_b200/csrc/gbem_dmma_gemm.cuh"
using namespace gbem_gemm;
__global__ void fill(double* p, long long n, unsigned seed) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) {
    unsigned x = (unsigned)i * 2654435761u + seed * 40503u;
    x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
    p[i] = (double)(x & 0xffff) / 65536.0 - 0.5;
  }
}
template <class KB>
int run(KB kb, size_t smem_b, int m, int k, int lda, int reps, const char* name) {
  double *A, *C1, *C2;
  cudaMalloc(&A, sizeof(double) * (size_t)lda * k + 64);
  cudaMalloc(&C1, sizeof(double) * (size_t)lda * m);
  cudaMalloc(&C2, sizeof(double) * (size_t)lda * m);
  fill<<<(unsigned)(((long long)lda * k + 255) / 256), 256>>>(A, (long long)lda * k, 7);
  const int nt = (m + 63) / 64;
  const unsigned tiles = (unsigned)((long long)nt * (nt + 1) / 2);
  cudaFuncSetAttribute(k_syrk_gen<64, 64, 2, 2, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GenShape<64, 64, 2, 2, 2>::SMEM);
  cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b);
  fill<<<(unsigned)(((long long)lda * m + 255) / 256), 256>>>(C1, (long long)lda * m, 1);
  k_syrk_gen<64, 64, 2, 2, 2, 4><<<tiles, 128, GenShape<64, 64, 2, 2, 2>::SMEM>>>(C1, lda, A, lda, m, k, 0, 0, nullptr, 0LL);
  std::vector<double> h1((size_t)lda * m), h2((size_t)lda * m);
  cudaMemcpy(h1.data(), C1, sizeof(double) * h1.size(), cudaMemcpyDeviceToHost);
  int bad_total = 0;
  for (int rep = 0; rep < reps; ++rep) {
    fill<<<(unsigned)(((long long)lda * m + 255) / 256), 256>>>(C2, (long long)lda * m, 1);
    kb<<<tiles, 128, smem_b>>>(C2, lda, A, lda, m, k, 0, 0, nullptr, 0LL);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s m=%d k=%d: %s\n", name, m, k, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h2.data(), C2, sizeof(double) * h2.size(), cudaMemcpyDeviceToHost);
    long long bad = 0; int fr = -1, fc = -1;
    for (int c = 0; c < m; ++c)
      for (int r = c; r < m; ++r)
        if (h1[(size_t)c * lda + r] != h2[(size_t)c * lda + r]) { if (!bad) { fr = r; fc = c; } ++bad; }
    if (bad) printf("%s m=%d k=%d lda=%d rep %d: %lld mismatches, first (r=%d, c=%d) tile (%d,%d)\n", name, m, k, lda, rep, bad, fr, fc, fr / 64, fc / 64);
    bad_total += bad != 0;
  }
  printf("%s m=%d k=%d lda=%d: %d of %d runs differ\n", name, m, k, lda, bad_total, reps);
  cudaFree(A); cudaFree(C1); cudaFree(C2);
  return bad_total;
}
int main(int argc, char** argv) {
  int fails = 0;
  const bool quick = argc > 1 && argv[1][0] == 'q';  // the -m gpu test: the shapes below 13k rows
  const int shapes[][3] = {{33000, 640, 33000}, {26000, 1536, 26000}, {4001, 256, 4008}, {1000, 128, 1000}, {777, 384, 784}, {12345, 512, 12352}, {64, 128, 64}, {130, 1024, 136}};
  for (auto& s : shapes) {
    if (quick && s[0] > 13000) continue;
    fails += run(k_syrk_bulk<16, 3, 4, true>, BulkShape<16, 3>::SMEM, s[0], s[1], s[2], 3, "split16x3");
    fails += run(k_syrk_bulk<16, 3, 4, false>, BulkShape<16, 3>::SMEM, s[0], s[1], s[2], 2, "rot16x3");
  }
  printf("FAILS %d\n", fails);
  return fails != 0;
}
