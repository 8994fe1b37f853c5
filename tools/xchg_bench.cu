// Microbenchmark: per-column cross-CTA exchange cost of the panel QR.
//   K0: counter barrier only
//   K1: record write + counter barrier + fixed-order read of G records (current panel)
//   K2: flag-in-data ("LL") records: each double stored as two {32-bit half, flag} pairs
//       in one 16-byte store; readers poll the records themselves (no counter)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xchg_bench xchg_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NB = 32;
constexpr int PM = 19;  // ceil(148 / 8)

__device__ __forceinline__ void arrive_wait(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
  }
  __syncthreads();
}

template <int KIND>
__global__ void k(unsigned* ctr, double* part, uint4* ll, int iters, double* sink) {
  __shared__ double red[8 * NB];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, g = blockIdx.x, G = gridDim.x;
  double x = 1.0 + t * 1e-3 + g;
  for (int it = 1; it <= iters; ++it) {
    const int par = it & 1;
    if (KIND == 0) {
      arrive_wait(ctr, it * G);
      x += 1.0;
    } else if (KIND == 1) {
      if (t < 2 * NB) part[((size_t)par * G + g) * 2 * NB + t] = x;
      arrive_wait(ctr, it * G);
      double v[PM];
#pragma unroll
      for (int q = 0; q < PM; ++q) {
        const int r = warp + 8 * q;
        v[q] = r < G ? __ldcg(&part[((size_t)par * G + r) * 2 * NB + lane]) : 0.0;
      }
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < PM; ++q) s += v[q];
      red[warp * NB + lane] = s;
      __syncthreads();
      double tot = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) tot += red[w * NB + lane];
      x += tot * 1e-30;
      __syncthreads();
    } else {
      // writer: warp 0 stores this CTA's record (32 doubles) with flag = it
      if (warp == 0) {
        const unsigned long long b = __double_as_longlong(x);
        uint4 w = make_uint4((unsigned)b, (unsigned)it, (unsigned)(b >> 32), (unsigned)it);
        uint4* dst = ll + ((size_t)par * G + g) * NB + lane;
        asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w) : "memory");
      }
      double v[PM];
      unsigned pending = 0;
#pragma unroll
      for (int q = 0; q < PM; ++q) {
        v[q] = 0.0;
        if (warp + 8 * q < G) pending |= 1u << q;
      }
      while (pending) {
#pragma unroll
        for (int q = 0; q < PM; ++q) {
          if (pending & (1u << q)) {
            const uint4* src = ll + ((size_t)par * G + warp + 8 * q) * NB + lane;
            uint4 r;
            asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(src) : "memory");
            if (r.y == (unsigned)it && r.w == (unsigned)it) {
              v[q] = __longlong_as_double(((unsigned long long)r.z << 32) | r.x);
              pending &= ~(1u << q);
            }
          }
        }
        pending = __reduce_or_sync(0xffffffffu, pending);  // keep the warp converged
      }
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < PM; ++q) s += v[q];
      red[warp * NB + lane] = s;
      __syncthreads();
      double tot = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) tot += red[w * NB + lane];
      x += tot * 1e-30;
      __syncthreads();
    }
  }
  if (x < 0) *sink = x;
}

int main() {
  unsigned* ctr; double* part; uint4* ll; double* sink;
  cudaMalloc(&ctr, 4); cudaMalloc(&part, 2 * 148 * 64 * 8); cudaMalloc(&ll, 2 * 148 * 32 * 16); cudaMalloc(&sink, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  void* fns[3] = {(void*)k<0>, (void*)k<1>, (void*)k<2>};
  for (int kind = 0; kind < 3; ++kind)
    for (int G : {32, 64, 148}) {
      int iters = 4000;
      void* args[] = {&ctr, &part, &ll, &iters, &sink};
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(ctr, 0, 4);
        cudaMemset(ll, 0, 2 * 148 * 32 * 16);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel(fns[kind], dim3(G), dim3(256), args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("kind=%d G=%3d: %.3f us per exchange\n", kind, G, ms * 1e3 / iters);
      }
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
