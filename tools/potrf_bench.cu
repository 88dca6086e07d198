// Phase timing of the diagonal-block factor kernel (clock64 hooks compiled in
// with GBEM_POTRF_TIMING); one 128 x 128 SPD block.
#define GBEM_POTRF_TIMING 1
#include "../paper_2203_11733_b200/csrc/gbem_solver.cu"
#include <cstdio>
#include <vector>
int main() {
  const int n = 128;
  std::vector<double> h(n * n);
  for (int c = 0; c < n; ++c)
    for (int r = 0; r < n; ++r) h[c * n + r] = (r == c ? n : 0.0) + 1.0 / (1.0 + r + c);
  double *A, *Li; int* info;
  cudaMalloc(&A, 8 * n * n); cudaMalloc(&Li, 8 * n * n); cudaMalloc(&info, 4);
  cudaFuncSetAttribute(k_potrf_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPotrfSmem);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(A, h.data(), 8 * n * n, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_potrf_diag<<<1, kPotrfThreads, kPotrfSmem>>>(A, n, n, 0, Li, info);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long clk[128]; cudaMemcpyFromSymbol(clk, g_potrf_clk, sizeof(clk));
    printf("kernel %.1f us (%s); phase cycles from start:", ms * 1000, cudaGetErrorString(cudaGetLastError()));
    int ids[] = {23, 1, 2, 3, 4, 5, 6, 7, 8, 9, 13, 14, 15, 10, 11, 12, 20, 21, 22};
    for (int k : ids) printf(" [%d]=%lld", k, clk[k] - clk[0]);
    printf("\n");
  }
  return 0;
}
