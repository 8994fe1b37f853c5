// Dense TF32 tcgen05 peak for B200 (sm_100a): the roofline denominator of the
// 3xTF32 GEMM (K10, csrc/gemm_tf32.cu).  MEASURED_PEAKS.json holds only bf16.
//
// One CTA per SM; operands resident in shared memory (K-major, 128B swizzle,
// the same descriptors K10 uses), accumulator in TMEM; one elected thread
// issues `iters` x 4 tcgen05.mma.cta_group::1.kind::tf32 (M=128, N, K=8) back
// to back and commits to an mbarrier.  No global traffic: a pure tensor-pipe
// rate.  FLOPs = 2*128*N*8 per MMA.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tf32_peak tools/tf32_peak.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t kmajor_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N>
__host__ __device__ constexpr uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int N>
__global__ void __launch_bounds__(128) tf32_peak_kernel(int iters, int* sink) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint32_t tmem_base_s;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* f = (float*)base;
  for (int i = threadIdx.x; i < (128 + N) * 32; i += blockDim.x) f[i] = 1e-3f * (float)(i % 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"((uint32_t)(N < 32 ? 32 : N)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(base), b = a + 128 * 128;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t acc = (it | ks) != 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(kmajor_sw128_desc(a + ks * 32)), "l"(kmajor_sw128_desc(b + ks * 32)),
            "r"(idesc_tf32<N>()), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(smem_u32(&bar)), "r"(0u)
          : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"((uint32_t)(N < 32 ? 32 : N)));
  }
  if (threadIdx.x == 0 && iters < 0) sink[blockIdx.x] = (int)tmem;
}

template <int N>
static double run(int nsm, int iters) {
  const int smem = (128 + N) * 128 + 1024;
  cudaFuncSetAttribute(tf32_peak_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int* sink;
  cudaMalloc(&sink, 4096 * sizeof(int));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tf32_peak_kernel<N><<<nsm, 128, smem>>>(100, sink);
  cudaEventRecord(e0);
  tf32_peak_kernel<N><<<nsm, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(sink);
  const double flops = 2.0 * 128 * N * 8 * 4.0 * iters * nsm;
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 40000;
  double t128[3], t256[3];
  for (int r = 0; r < 3; ++r) {
    t128[r] = run<128>(nsm, iters);
    t256[r] = run<256>(nsm, iters);
  }
  double b128 = 0, b256 = 0;
  for (int r = 0; r < 3; ++r) {
    b128 = t128[r] > b128 ? t128[r] : b128;
    b256 = t256[r] > b256 ? t256[r] : b256;
  }
  printf("{\"sms\": %d, \"clock_khz\": %d, \"kind\": \"tcgen05.mma.cta_group::1.kind::tf32 M=128 K=8\", "
         "\"tflops_n128\": %.1f, \"tflops_n256\": %.1f}\n",
         nsm, clk, b128, b256);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    fprintf(stderr, "cuda error %s\n", cudaGetErrorString(err));
    return 1;
  }
  return 0;
}
