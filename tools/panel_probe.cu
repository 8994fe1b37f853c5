// Per-phase timing of the fused panel QR kernel (CTA 0, %globaltimer probes).
// Build: see tools/gpu_probe.sh.  Usage: panel_probe <rows> [max_ctas]
#define PANEL_PROBE
#include "../paper_2106_13402_b200/csrc/panel.cu"

__global__ void fill(double* p, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
    p[i] = (double)(h & 0xFFFFFF) / 8388608.0 - 1.0;
  }
}

int main(int argc, char** argv) {
  using namespace utv;
  const int rows = argc > 1 ? atoi(argv[1]) : 2048, cols = 256;
  const int ctas = argc > 2 ? atoi(argv[2]) : 0;
  double *P0, *P, *Y, *T, *fro2, *ws;
  cudaMalloc(&P0, 8L * rows * cols); cudaMalloc(&P, 8L * rows * cols); cudaMalloc(&Y, 8L * rows * cols);
  cudaMalloc(&T, 8L * cols * cols); cudaMalloc(&fro2, 8); cudaMalloc(&ws, 8 * panel_ws_doubles());
  fill<<<296, 256>>>(P0, (long)rows * cols);
  double f = (double)rows * cols / 3.0;
  cudaMemcpy(fro2, &f, 8, cudaMemcpyHostToDevice);
  const char* names[14] = {"leaf load", "col: local dots+record", "col: barrier", "col: record sum",
                           "leaf: ts/tail", "leaf: R/Y write", "A: Y^T X partials", "A->C barrier",
                           "C: cross-CTA reduce", "C->D barrier", "(unused)", "col: reflector+rank-1",
                           "T off-diagonal build", "D: trailing update"};
  for (int rep = 0; rep < 3; ++rep) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(pqr::g_probe, z, sizeof(z));
    cudaMemcpy(P, P0, 8L * rows * cols, cudaMemcpyDeviceToDevice);
    cudaMemset(T, 0, 8L * cols * cols);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    int rc = panel_qr(Mat{P, rows, rows, cols}, Mat{Y, rows, rows, cols}, Mat{T, cols, cols, cols}, fro2, ws, 0, ctas);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long pr[16];
    cudaMemcpyFromSymbol(pr, pqr::g_probe, sizeof(pr));
    if (rep < 2) continue;
    printf("rows=%d ctas=%d rc=%d: %.3f ms  (%s)\n", rows, ctas, rc, ms, cudaGetErrorString(cudaGetLastError()));
    unsigned long long tot = 0;
    for (int k = 0; k < 14; ++k) tot += pr[k];
    for (int k = 0; k < 14; ++k)
      if (pr[k]) printf("  %-24s %8.1f us  %5.1f%%\n", names[k], pr[k] / 1e3, 100.0 * pr[k] / tot);
  }
}
