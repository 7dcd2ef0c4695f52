// Accuracy of the MUFU.RCP64H seed (rcp.approx.ftz.f64) and of one / two
// Newton corrections of a quotient, over d in [1, 2) (sampled densely).
#include <cstdio>
#include <cstdint>
__device__ double rcp_seed(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
__device__ unsigned long long to_key(double e) { return (unsigned long long)__double_as_longlong(fabs(e)); }
__global__ void k(unsigned long long *mx, long n) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  double e0 = 0, e1 = 0, eb = 0;
  for (; i < n; i += (long)gridDim.x * blockDim.x) {
    const double d = 1.0 + (double)i / (double)n + 1e-17 * (double)(i & 7);
    const double r0 = rcp_seed(d);
    e0 = fmax(e0, fabs(fma(-d, r0, 1.0)));
    const double nn = 0.7 + 0.2 * (double)(i & 1023) / 1024.0;
    const double y0 = nn * r0;
    const double y1 = fma(r0, fma(-d, y0, nn), y0);
    const double ex = nn / d;
    e1 = fmax(e1, fabs(y1 - ex) / ex);
    eb = fmax(eb, (ex - y1) / ex);  // signed: positive = low
  }
  atomicMax(mx + 0, to_key(e0));
  atomicMax(mx + 1, to_key(e1));
  atomicMax(mx + 2, to_key(eb));
}
int main() {
  unsigned long long *m, h[3];
  cudaMalloc(&m, 24);
  cudaMemset(m, 0, 24);
  k<<<1184, 256>>>(m, 1L << 32);
  cudaMemcpy(h, m, 24, cudaMemcpyDeviceToHost);
  double v[3];
  for (int j = 0; j < 3; j++) v[j] = *(double *)&h[j];
  printf("seed |1 - d r0| max %.3e (2^%.2f)\none-correction quotient rel err max %.3e; low-biased max %.3e\n", v[0],
         __builtin_log2(v[0]), v[1], v[2]);
  return 0;
}
