#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ long long clk() { long long v; asm volatile("mov.u64 %0, %%clock64;" : "=l"(v)); return v; }
__device__ __forceinline__ void rotation(double alpha, double beta, double gamma, double* c, double* s) {
  const double zeta = (beta - alpha) / (2.0 * gamma);
  double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
  *c = rsqrt(fma(t, t, 1.0)); *s = *c * t;
}
__device__ __forceinline__ void rotation2(double alpha, double beta, double gamma, double* c, double* s) {
  const double d = beta - alpha, g2 = 2.0 * gamma;
  double t = copysign(g2, d) / (fabs(d) + sqrt(fma(d, d, g2 * g2)));
  *c = rsqrt(fma(t, t, 1.0)); *s = *c * t;
}
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double sh[1024];
  double a = 1.0 + threadIdx.x * 1e-3, b = 2.0, g = 0.3, c, s;
  long long t0 = clk();
  for (int i = 0; i < iters; ++i) { rotation(a, b, g, &c, &s); a = c + 1.0; g = s * 0.5 + 0.1; }
  long long t1 = clk();
  for (int i = 0; i < iters; ++i) { rotation2(a, b, g, &c, &s); a = c + 1.0; g = s * 0.5 + 0.1; }
  long long t2 = clk();
  for (int i = 0; i < iters; ++i) { __syncthreads(); }
  long long t3 = clk();
  double v = a;
  for (int i = 0; i < iters; ++i) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  long long t4 = clk();
  for (int i = 0; i < iters; ++i) { v = fma(v, 1.0000001, 1e-9); }
  long long t5 = clk();
  sh[threadIdx.x] = v;
  for (int i = 0; i < iters; ++i) { v = sh[(threadIdx.x + (int)v) & 1023] + 1.0; }
  long long t6 = clk();
  for (int i = 0; i < iters; ++i) { v = 1.0 / (v + 1.0); }
  long long t7 = clk();
  for (int i = 0; i < iters; ++i) { v = sqrt(v + 1.0); }
  long long t8 = clk();
  out[threadIdx.x] = c + s + v;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / iters; cyc[1] = (t2 - t1) / iters; cyc[2] = (t3 - t2) / iters; cyc[3] = (t4 - t3) / iters;
    cyc[4] = (t5 - t4) / iters; cyc[5] = (t6 - t5) / iters; cyc[6] = (t7 - t6) / iters; cyc[7] = (t8 - t7) / iters;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMallocManaged(&c, 64);
  for (int th : {32, 512}) {
    k<<<1, th>>>(o, c, 1000); cudaDeviceSynchronize();
    k<<<1, th>>>(o, c, 1000); cudaDeviceSynchronize();
    printf("threads %d: rotation %lld  rotation2 %lld  syncthreads %lld  shfl-reduce(5) %lld  dfma %lld  lds %lld  ddiv %lld  dsqrt %lld clk\n",
           th, c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]);
  }
}
