// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) and DFMA.
// Measures the denominators the roofline uses for FP64 work (MEASURED_PEAKS.json has none).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; i++) { acc[i][0] = 0; acc[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fma(acc[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"results\": [\n", nsm, clk);
  const int iters = 20000;
  bool first = true;
  for (int warps : {4, 8, 16, 32}) {
    for (int rep = 0; rep < 2; ++rep) {
      dim3 grid(nsm * 2), block(32 * warps / 2);
      dmma_loop<8><<<grid, block>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<8><<<grid, block>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * grid.x * (block.x / 32);
      if (rep) { printf("%s {\"kind\": \"dmma_m8n8k4\", \"warps_per_sm\": %d, \"tflops\": %.3f}\n", first ? "" : ",", warps, flops / ms / 1e9); first = false; }
    }
  }
  for (int warps : {4, 8, 16, 32}) {
    for (int rep = 0; rep < 2; ++rep) {
      dim3 grid(nsm * 2), block(32 * warps / 2);
      dfma_loop<8><<<grid, block>>>(out, 100);
      cudaEventRecord(e0);
      dfma_loop<8><<<grid, block>>>(out, iters * 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * (double)iters * 4 * grid.x * block.x;
      if (rep) printf(", {\"kind\": \"dfma\", \"warps_per_sm\": %d, \"tflops\": %.3f}\n", warps, flops / ms / 1e9);
    }
  }
  printf("]}\n");
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { fprintf(stderr, "cuda error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
