// Device-side generators and parity metrics: the
// reference builds its test matrices on the CPU (matgen.py:17-98 — 51 s at
// n = 2000 through the Python Householder QR) and sweeps error curves with
// numpy (bench.py:63-72).  At n = 16384 both are infeasible on the host.
//
//  * gen_bie_kernel / gen_kahan_kernel: the two deterministic matrices of
//    matgen.py:58-91, elementwise.
//  * trailing_fro: e_k = ||T[k:, k:]||_F for k = 1..n-1 (bench.py:63-72) in
//    O(mn) through e_k^2 = e_{k+1}^2 + sum_{j>=k} T_kj^2 + sum_{i>k} T_ik^2:
//    one column pass, one row pass, one fixed-order suffix scan (bitwise
//    reproducible, no atomics).
#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace met {
constexpr double PI = 3.14159265358979323846;

// a_ij = -(1/(2 pi)) log(2 |sin(pi (i-j)/n)|) (2 pi / n), a_ii = log(n)/n
__global__ void gen_bie_kernel(double* A, long lda, int n) {
  const long total = (long)n * n;
  const double w = 2.0 * PI / n;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total; t += (long)gridDim.x * blockDim.x) {
    const int i = (int)(t % n), j = (int)(t / n);
    double v;
    if (i == j) {
      v = log((double)n) / n;
    } else {
      const double dist = 2.0 * fabs(sin(PI * (double)(i - j) / n));
      v = -(1.0 / (2.0 * PI)) * log(dist) * w;
    }
    A[i + (long)j * lda] = v;
  }
}

// Kahan: diag(s^i) (I - c * strict_upper)
__global__ void gen_kahan_kernel(double* A, long lda, int n, double s, double c) {
  const long total = (long)n * n;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total; t += (long)gridDim.x * blockDim.x) {
    const int i = (int)(t % n), j = (int)(t / n);
    const double u = (i == j) ? 1.0 : (j > i ? -c : 0.0);
    A[i + (long)j * lda] = pow(s, (double)i) * u;
  }
}

// col[j] = sum_{i > j} T_ij^2 (one block per column, fixed-order tree)
__global__ void colsq_kernel(const double* __restrict__ T, long ldt, int m, int n, double* col) {
  __shared__ double sh[32];
  const int j = blockIdx.x;
  double acc = 0.0;
  for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) {
    const double x = T[i + (long)j * ldt];
    acc = fma(x, x, acc);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) col[j] = v;
  }
}

// row[i] = sum_{j >= i} T_ij^2 (one thread per row; coalesced along i)
__global__ void rowsq_kernel(const double* __restrict__ T, long ldt, int m, int n, double* row) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || i >= n) return;
  double acc = 0.0;
  for (int j = i; j < n; ++j) {
    const double x = T[i + (long)j * ldt];
    acc = fma(x, x, acc);
  }
  row[i] = acc;
}

// e[k-1] = sqrt(sum_{k' >= k} (row[k'] + col[k'])), k = 1..n-1 (single thread, fixed order)
__global__ void suffix_kernel(const double* row, const double* col, int m, int n, double* e) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double s = 0.0;
  for (int k = n - 1; k >= 1; --k) {
    if (k < m) s += row[k] + col[k];
    e[k - 1] = sqrt(s > 0.0 ? s : 0.0);
  }
}

inline int grid(long total) {
  const long g = (total + 255) / 256;
  const long cap = 8L * num_sms();
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}
}  // namespace met

int gen_bie(double* A, long lda, int n, cudaStream_t st) {
  ProfScope ps(PROF_OPS, 0.0, 8.0 * n * (double)n, st);
  met::gen_bie_kernel<<<met::grid((long)n * n), 256, 0, st>>>(A, lda, n);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int gen_kahan(double* A, long lda, int n, double theta, cudaStream_t st) {
  ProfScope ps(PROF_OPS, 0.0, 8.0 * n * (double)n, st);
  met::gen_kahan_kernel<<<met::grid((long)n * n), 256, 0, st>>>(A, lda, n, sin(theta), cos(theta));
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

size_t trailing_fro_ws_doubles(int m, int n) { return 2 * (size_t)round_up(m > n ? m : n, 4) + 64; }

int trailing_fro(const double* T, long ldt, int m, int n, double* e, double* ws, cudaStream_t st) {
  if (n < 2) return UTV_OK;
  const long mx = m > n ? m : n;
  double* col = ws;
  double* row = ws + round_up(mx, 4);
  ProfScope ps(PROF_OPS, 4.0 * m * (double)n, 8.0 * 2.0 * m * n, st, 3);
  met::colsq_kernel<<<n, 256, 0, st>>>(T, ldt, m, n, col);
  UTV_CUDA(cudaGetLastError());
  met::rowsq_kernel<<<ceil_div(m < n ? m : n, 128), 128, 0, st>>>(T, ldt, m, n, row);
  UTV_CUDA(cudaGetLastError());
  met::suffix_kernel<<<1, 32, 0, st>>>(row, col, m, n, e);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

}  // namespace utv
