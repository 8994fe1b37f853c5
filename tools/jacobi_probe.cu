// Per-phase timing of the Jacobi rounds kernel (CTA 0, %globaltimer probes).
// Build + run: tools/jacobi_probe.sh <n> ...  (links the library objects
// except jacobi.o).  Input: a dense n x n pseudo-random matrix.
#define JAC_PROBE
#include "../paper_2106_13402_b200/csrc/jacobi.cu"

__global__ void fill(double* p, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
    p[i] = (double)(h & 0xFFFFFF) / 8388608.0 - 1.0;
  }
}

int main(int argc, char** argv) {
  using namespace utv;
  const int n = argc > 1 ? atoi(argv[1]) : 256;
  double *A, *U, *V, *sig, *ws;
  int* status;
  const size_t wsn = gesvj_ws_doubles(n);
  cudaMalloc(&A, 8L * n * n); cudaMalloc(&U, 8L * n * n); cudaMalloc(&V, 8L * n * n);
  cudaMalloc(&sig, 8L * n); cudaMalloc(&ws, 8 * wsn); cudaMalloc(&status, 4);
  fill<<<296, 256>>>(A, (long)n * n);
  const char* names[7] = {"load A,V slices", "partial Gram", "cluster sync + DSMEM reduce",
                          "sub-rounds", "apply J", "store A,V slices", "grid barrier"};
  for (int rep = 0; rep < 3; ++rep) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(jac::g_probe, z, sizeof(z));
    cudaMemcpyToSymbol(jac::g_probe2, z, sizeof(z));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    int rc = gesvj(Mat{A, n, n, n}, sig, Mat{U, n, n, n}, Mat{V, n, n, n}, ws, wsn, status, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long pr[8];
    cudaMemcpyFromSymbol(pr, jac::g_probe, sizeof(pr));
    int sw = 0;
    cudaMemcpy(&sw, status, 4, cudaMemcpyDeviceToHost);
    if (rep < 2) continue;
    printf("n=%d rc=%d sweeps=%d: %.3f ms  (%s)\n", n, rc, sw, ms, cudaGetErrorString(cudaGetLastError()));
    unsigned long long tot = 0;
    for (int k = 0; k < 7; ++k) tot += pr[k];
    unsigned long long p2[8];
    cudaMemcpyFromSymbol(p2, jac::g_probe2, sizeof(p2));
    printf("  sub-round (%llu): worker work %.0f + wait %.0f clk; rotation warp work %.0f + wait %.0f clk\n", p2[2],
           (double)p2[0] / p2[2], (double)p2[1] / p2[2], (double)p2[3] / p2[5], (double)p2[4] / p2[5]);
    printf("  SM clock over the rounds kernel: %.0f MHz\n", 1e3 * pr[7] / tot);
    for (int k = 0; k < 7; ++k)
      printf("  %-34s %8.1f us  %5.1f%%\n", names[k], pr[k] / 1e3, 100.0 * pr[k] / tot);
  }
}
