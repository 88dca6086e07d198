// Probe: SM partitioning with green contexts (driver API) + runtime-API kernel
// launches on their streams; records which SMs each partition's CTAs ran on.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>
#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)
#define RT(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)
__global__ void k_smid(int* out, long long spin) {
  unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  long long t0 = clock64(); while (clock64() - t0 < spin) {}
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}
int main() {
  RT(cudaSetDevice(0));
  RT(cudaFree(0));
  CUdevice dev; CU(cuDeviceGet(&dev, 0));
  CUdevResource res; CU(cuDeviceGetDevResource(dev, &res, CU_DEV_RESOURCE_TYPE_SM));
  printf("SMs: %u\n", res.sm.smCount);
  for (unsigned flags = 0; flags < 2; ++flags)
    for (unsigned want : {1u, 2u, 4u, 8u}) {  // what a request for `want` SMs really reserves
      CUdevResource p2, r2; unsigned n2 = 1;
      CUresult rc = cuDevSmResourceSplitByCount(&p2, &n2, &res, &r2, flags, want);
      printf("split flags=%u minCount=%u -> rc=%d side %u SMs, rest %u SMs\n", flags, want, (int)rc, p2.sm.smCount, r2.sm.smCount);
    }
  CUdevResource part, rest; unsigned ng = 1;
  CU(cuDevSmResourceSplitByCount(&part, &ng, &res, &rest, 0, 8));
  printf("groups %u: side %u SMs, rest %u SMs\n", ng, part.sm.smCount, rest.sm.smCount);
  CUdevResourceDesc d1, d2; CU(cuDevResourceGenerateDesc(&d1, &part, 1)); CU(cuDevResourceGenerateDesc(&d2, &rest, 1));
  CUgreenCtx g1, g2; CU(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM)); CU(cuGreenCtxCreate(&g2, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s1, s2; CU(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0)); CU(cuGreenCtxStreamCreate(&s2, g2, CU_STREAM_NON_BLOCKING, 0));
  int* d; RT(cudaMalloc(&d, 4 * 4096));  // primary-context allocation used from both partitions
  k_smid<<<64, 128, 0, (cudaStream_t)s1>>>(d, 100000);
  RT(cudaGetLastError());
  k_smid<<<1024, 128, 0, (cudaStream_t)s2>>>(d + 1024, 100000);
  RT(cudaGetLastError());
  RT(cudaDeviceSynchronize());
  std::vector<int> h(4096); RT(cudaMemcpy(h.data(), d, 4 * 4096, cudaMemcpyDeviceToHost));
  std::set<int> a(h.begin(), h.begin() + 64), b(h.begin() + 1024, h.begin() + 2048);
  int overlap = 0; for (int x : a) overlap += b.count(x);
  printf("side partition used %zu SMs, main used %zu SMs, overlap %d\n", a.size(), b.size(), overlap);
  // event across partitions
  cudaEvent_t ev; RT(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  k_smid<<<8, 128, 0, (cudaStream_t)s1>>>(d, 1000); RT(cudaEventRecord(ev, (cudaStream_t)s1));
  RT(cudaStreamWaitEvent((cudaStream_t)s2, ev, 0)); k_smid<<<8, 128, 0, (cudaStream_t)s2>>>(d, 1000);
  RT(cudaDeviceSynchronize());
  printf("cross-partition event ok\n");
  return 0;
}
