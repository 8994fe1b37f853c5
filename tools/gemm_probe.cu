// Per-phase cycles of the DMMA GEMM's consumer warps 0/1 of CTA 0 (clock64,
// -DGEMM_PROBE build): tile-start wait, main loop (of which full-barrier
// waits), epilogue.  Usage: tools/gemm_probe.sh [K ...]
#define GEMM_PROBE
#include "../paper_2106_13402_b200/csrc/gemm.cu"

__global__ void fill(double* p, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    p[i] = (double)((i * 2654435761u) % 1000) / 1000.0 - 0.5;
}

int main(int argc, char** argv) {
  using namespace utv;
  const int M = 16384, N = 16384;
  double *A, *B, *C, *ws;
  const int Kmax = 2048;
  cudaMalloc(&A, 8L * M * Kmax); cudaMalloc(&B, 8L * N * Kmax); cudaMalloc(&C, 8L * M * N);
  const size_t wsn = 64L << 20;
  cudaMalloc(&ws, 8 * wsn);
  fill<<<1184, 256>>>(A, (long)M * Kmax); fill<<<1184, 256>>>(B, (long)N * Kmax); fill<<<1184, 256>>>(C, (long)M * N);
  for (int ai = 1; ai < argc; ++ai) {
    const int K = atoi(argv[ai]);
    for (double beta : {0.0, 1.0}) {
      for (int rep = 0; rep < 2; ++rep) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(gemm::g_gprobe, z, sizeof(z));
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        int rc = dgemm(false, true, M, N, K, -1.0, A, M, B, N, beta, C, M, ws, wsn, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long pr[16];
        cudaMemcpyFromSymbol(pr, gemm::g_gprobe, sizeof(pr));
        if (rep == 0) continue;
        printf("NT K=%d beta=%.0f rc=%d: %.3f ms %.2f TF/s (%s)\n", K, beta, rc, ms, 2.0 * M * N * K / ms / 1e9,
               cudaGetErrorString(cudaGetLastError()));
        for (int w = 0; w < 2; ++w) {
          const double t = (double)pr[w * 8 + 4];
          printf("  warp %d: %.0f tiles; per tile: start-wait %.0f, main loop %.0f (full waits %.0f), epilogue %.0f cycles\n",
                 w, t, pr[w * 8 + 0] / t, pr[w * 8 + 1] / t, pr[w * 8 + 2] / t, pr[w * 8 + 3] / t);
        }
      }
    }
  }
}
