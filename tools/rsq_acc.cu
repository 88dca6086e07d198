// accuracy of rsqrt.approx.ftz.f64 (MUFU.RSQ64H) and of one 2nd-order Newton step
#include <cstdio>
#include <cmath>
__global__ void k(const double* x, double* o1, double* o2, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x[i]));
  double e = fma(-x[i] * y, y, 1.0);
  double y2 = fma(y * e, 0.5, y);
  o1[i] = y; o2[i] = y2;
}
int main() {
  int n = 1 << 22; double *x, *a, *b;
  cudaMallocManaged(&x, 8 * n); cudaMallocManaged(&a, 8 * n); cudaMallocManaged(&b, 8 * n);
  for (int i = 0; i < n; ++i) x[i] = 1e-10 * pow(1e22, (double)i / n) * (1.0 + 0.013 * (i % 97));
  k<<<(n + 255) / 256, 256>>>(x, a, b, n); cudaDeviceSynchronize();
  double m1 = 0, m2 = 0, s2 = 0;
  for (int i = 0; i < n; ++i) {
    long double t = 1.0L / sqrtl((long double)x[i]);
    double e1 = (double)fabsl((a[i] - t) / t), e2 = (double)((b[i] - t) / t);
    if (e1 > m1) m1 = e1; if (fabs(e2) > m2) m2 = fabs(e2); s2 += e2;
  }
  printf("MUFU.RSQ64H max rel err %.3e ; after one 2nd-order step max %.3e mean %.3e\n", m1, m2, s2 / n);
}
