// cost of cooperative-groups grid.sync() on B200 (148 CTAs x 256 threads)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, double* out) {
  cg::grid_group g = cg::this_grid();
  double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) { x = x * 0.999 + 1e-3; g.sync(); }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = x;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  int iters = 1000; void* args[] = {&iters, &o};
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks : {148, 296, 592}) {
    cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("blocks %d: %.3f us per grid.sync (%s)\n", blocks, ms * 1000 / iters, cudaGetErrorString(cudaGetLastError()));
  }
}
