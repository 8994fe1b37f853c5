// Microbenchmark: cost of one grid-wide barrier (cooperative launch) for
// several barrier implementations and grid sizes.  nvcc -arch=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void bar_fence_sc(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
  }
  __syncthreads();
}
__device__ __forceinline__ void bar_release(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
  }
  __syncthreads();
}
template <int KIND>
__global__ void k(unsigned* ctr, int iters, double* sink) {
  double x = threadIdx.x;
  for (int i = 1; i <= iters; ++i) {
    if (KIND == 0) bar_fence_sc(ctr, i * gridDim.x);
    else bar_release(ctr, i * gridDim.x);
    x += 1.0;
  }
  if (x < 0) *sink = x;
}
int main() {
  unsigned* ctr; double* sink;
  cudaMalloc(&ctr, 4); cudaMalloc(&sink, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int kind = 0; kind < 2; ++kind)
    for (int G : {8, 32, 64, 128, 148}) {
      int iters = 2000;
      void* args[] = {&ctr, &iters, &sink};
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(ctr, 0, 4);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel(kind == 0 ? (void*)k<0> : (void*)k<1>, dim3(G), dim3(256), args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("kind=%d G=%3d: %.3f us per barrier\n", kind, G, ms * 1e3 / iters);
      }
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
