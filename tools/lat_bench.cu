// Dependent-chain latencies on the B200 SM: DFMA, LDS.64, SHFL (64-bit), MUFU.RSQ64H.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters, double x0) {
  __shared__ double s[1024];
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { s[i] = 1.0 + i * 1e-9; idx[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  double a = x0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, 1.0000001, 1e-12);
  long long t1 = clock64();
  int p = threadIdx.x & 1023;
  for (int i = 0; i < iters; ++i) p = idx[p];
  long long t2 = clock64();
  double v = a;
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31) + 1e-9;
  long long t3 = clock64();
  double r = a;
  for (int i = 0; i < iters; ++i) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r)); r = y + 1.0; }
  long long t4 = clock64();
  double m = a;
  for (int i = 0; i < iters; ++i) m = m * 1.0000001;
  long long t5 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = a + p + v + r + m;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024 * 148); cudaMalloc(&c, 64);
  const int it = 4096;
  for (int th : {32, 512}) {
    k<<<1, th>>>(o, c, it, 1.0);
    long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("threads %d: dfma %.1f  lds(dep) %.1f  shfl64+dadd %.1f  rsq64h+dadd %.1f  dmul %.1f cyc/op (%s)\n", th,
           h[0] / (double)it, h[1] / (double)it, h[2] / (double)it, h[3] / (double)it, h[4] / (double)it,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
