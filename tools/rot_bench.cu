#include "../paper_2106_13402_b200/csrc/jacobi.cu"
using namespace utv::jac;
// fp64 variants of the rotation angle for comparison
__device__ __forceinline__ bool rot_sqrt_rsqrt(double alpha, double beta, double gamma, double tol2, double* c, double* s) {
  const double ab = alpha * beta;
  const bool rot = gamma * gamma > tol2 * ab;
  if (gamma == 0.0 || !rot) return false;
  const double d = beta - alpha, g = 2.0 * gamma;
  const double h = sqrt(fma(d, d, g * g));
  const double u = h + fabs(d);
  const double q = rsqrt(2.0 * h * u);
  *c = u * q;
  *s = (d < 0.0 ? -g : g) * q;
  return true;
}
__device__ __forceinline__ bool rot_zeta(double alpha, double beta, double gamma, double tol2, double* c, double* s) {
  const double ab = alpha * beta;
  const bool rot = gamma * gamma > tol2 * ab;
  if (gamma == 0.0 || !rot) return false;
  const double zeta = (beta - alpha) / (2.0 * gamma);
  const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
  *c = rsqrt(fma(t, t, 1.0));
  *s = *c * t;
  return true;
}
__device__ __forceinline__ long long clk() { long long v; asm volatile("mov.u64 %0, %%clock64;" : "=l"(v)); return v; }
__global__ void k(long long* out, double* o, int iters) {
  __shared__ double G[32 * 33];
  for (int i = threadIdx.x; i < 32 * 33; i += blockDim.x) G[i] = 1.0 + 0.01 * i;
  __syncthreads();
  double a = 1.0 + threadIdx.x * 1e-3, b = 2.0, g = 0.3, c = 0, s = 0;
  long long t0 = clk();
  for (int i = 0; i < iters; ++i) { rotation(a, b, g, 1e-40, &c, &s); a = c + 1.0; g = s * 0.5 + 0.1; }
  long long t1 = clk();
  double dx = 1.0, dy = 2.0, cK = 0.9, sK = 0.1; bool rK = true;
  unsigned w = 1 | (17 << 5) | ((3 | (0 << 4) | (9 << 5)) << 10) | ((5 | (1 << 4) | (20 << 5)) << 20);
  for (int i = 0; i < iters; ++i) { rotate_next(w, G, 1e-40, &cK, &sK, &rK, &dx, &dy); w ^= (unsigned)(cK > 2.0); }
  long long t2 = clk();
  double v = 1.0;
  for (int i = 0; i < iters; ++i) { v = __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31) + 1.0; }
  long long t3 = clk();
  for (int i = 0; i < iters; ++i) { v = G[((int)v) & 511] + 1.0; }
  long long t4 = clk();
  for (int i = 0; i < iters; ++i) { rot_sqrt_rsqrt(a, b, g, 1e-40, &c, &s); a = c + 1.0; g = s * 0.5 + 0.1; }
  long long t5 = clk();
  for (int i = 0; i < iters; ++i) { rot_zeta(a, b, g, 1e-40, &c, &s); a = c + 1.0; g = s * 0.5 + 0.1; }
  long long t6 = clk();
  o[threadIdx.x] = c + s + dx + dy + cK + v;
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = (t3 - t2) / iters; out[3] = (t4 - t3) / iters; out[4] = (t5 - t4) / iters; out[5] = (t6 - t5) / iters; }
}
int main() {
  long long* c; double* o; cudaMallocManaged(&c, 64); cudaMalloc(&o, 8 * 1024);
  k<<<1, 32>>>(c, o, 1000); cudaDeviceSynchronize(); k<<<1, 32>>>(c, o, 1000); cudaDeviceSynchronize();
  printf("rotation %lld  rotate_next %lld  shfl.f64 %lld  lds.f64 %lld  sqrt+rsqrt %lld  zeta %lld clk (%s)\n", c[0], c[1], c[2], c[3], c[4], c[5], cudaGetErrorString(cudaGetLastError()));
}
