// Per-phase cycle counts of the cooperative forward/backward solve
// (GBEM_SOLVE_TIMING hooks), CTA 0 and a middle CTA, forward sweep.
// The factor content does not affect timing: A is filled with small values and
// the diagonal-block inverses are identities.
#define GBEM_SOLVE_TIMING 1
#include "../paper_2203_11733_b200/csrc/gbem_solver.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 11340;
  const int R = argc > 2 ? atoi(argv[2]) : 6;
  const long long lda = ((n + 7) / 8) * 8;
  const int nblk = (n + NB - 1) / NB;
  double *A, *Li, *B, *X, *S;
  cudaMalloc(&A, 8 * lda * n); cudaMalloc(&Li, 8LL * nblk * NB * NB);
  cudaMalloc(&B, 8LL * n * R); cudaMalloc(&X, 8LL * n * R); cudaMalloc(&S, 8LL * n * R);
  cudaMemset(A, 0, 8 * lda * n);
  std::vector<double> h(NB * NB, 0.0);
  for (int i = 0; i < NB; ++i) h[i * NB + i] = 1.0;
  for (int b = 0; b < nblk; ++b) cudaMemcpy(Li + (size_t)b * NB * NB, h.data(), 8 * NB * NB, cudaMemcpyHostToDevice);
  cudaMemset(B, 0, 8LL * n * R);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  auto fn = (void*)k_solve_coop<8>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSolveSmem);
  for (int rep = 0; rep < 3; ++rep) {
    long long z[16] = {};
    cudaMemcpyToSymbol(g_solve_clk, z, sizeof(z));
    int nn = n, RR = R, dd = 0;
    const double* cA = A; const double* cL = Li; const double* cB = B;
    void* args[] = {(void*)&cA, (void*)&lda, (void*)&cL, (void*)&nn, (void*)&RR, (void*)&cB, (void*)&X, (void*)&S, (void*)&dd};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel(fn, dim3(nsm), dim3(kSolveThreads), args, kSolveSmem, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c[16]; cudaMemcpyFromSymbol(c, g_solve_clk, sizeof(c));
    printf("n=%d R=%d %.3f ms (%s)\n", n, R, ms, cudaGetErrorString(cudaGetLastError()));
    const char* names[] = {"ws load", "Ls wait", "diag", "update", "prefetch issue", "grid sync"};
    for (int w = 0; w < 2; ++w) {
      printf("  CTA %s:", w ? "mid" : "0");
      for (int k = 0; k < 6; ++k) printf(" %s %.2f us/step |", names[k], c[w * 8 + k] / 1.965e3 / nblk);
      printf("\n");
    }
  }
  return 0;
}
