// K7: small fused ops on column-major blocks (HBM-bound, vectorised grid-stride).
//  * sumsq: deterministic Frobenius reductions (ErrorTracker, randutv.py:52-62;
//    qr.py:86 threshold; record_trailing randutv.py:160-161).
//  * structured writes: identity (randutv.py:115-116), zero blocks
//    (randutv.py:149), diag(sigma) (randutv.py:154,169-171), block copies.
#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace ops {
constexpr int RED_BLOCKS = 296;  // 2 x 148 SMs; fixed so the reduction order is fixed
constexpr int RED_THREADS = 512;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < (int)(blockDim.x >> 5)) ? sh[l] : 0.0;
    v = warp_sum(v);
  }
  __syncthreads();
  return v;
}

// Partial sums of squares: block b handles columns b, b+G, ... (one warp row
// sweep per column, coalesced along the contiguous dimension).
__global__ void sumsq_partial(const double* __restrict__ A, long lda, int rows, int cols,
                              double* __restrict__ part) {
  __shared__ double sh[32];
  double acc = 0.0;
  const long total = (long)rows * cols;
  if (rows >= 256) {
    for (int c = blockIdx.x; c < cols; c += gridDim.x) {
      const double* col = A + (long)c * lda;
      for (int r = threadIdx.x; r < rows; r += blockDim.x) {
        const double x = col[r];
        acc = fma(x, x, acc);
      }
    }
  } else {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
         i += (long)gridDim.x * blockDim.x) {
      const double x = A[(i % rows) + (i / rows) * lda];
      acc = fma(x, x, acc);
    }
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void sumsq_partial_f32(const float* __restrict__ A, long lda, int rows, int cols,
                                  double* __restrict__ part) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int c = blockIdx.x; c < cols; c += gridDim.x) {
    const float* col = A + (long)c * lda;
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
      const double x = col[r];
      acc = fma(x, x, acc);
    }
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void sum_partials(const double* __restrict__ part, int n, double* out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) *out = acc;
}

__global__ void fill_kernel(double* A, long lda, int rows, int cols, double diag_val,
                            double off_val) {
  const long total = (long)rows * cols;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i % rows), c = (int)(i / rows);
    A[r + (long)c * lda] = (r == c) ? diag_val : off_val;
  }
}

__global__ void diag_kernel(double* A, long lda, int rows, int cols, const double* d) {
  const long total = (long)rows * cols;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i % rows), c = (int)(i / rows);
    A[r + (long)c * lda] = (r == c) ? d[r] : 0.0;
  }
}

__global__ void copy_kernel(const double* __restrict__ S, long lds, double* __restrict__ D,
                            long ldd, int rows, int cols) {
  const long total = (long)rows * cols;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i % rows), c = (int)(i / rows);
    D[r + (long)c * ldd] = S[r + (long)c * lds];
  }
}

// LAPACK dlaset semantics: uplo 0 = whole, 1 = strictly upper + diag,
// 2 = strictly lower + diag; off-diagonal entries <- alpha, diagonal <- beta.
// uplo 3 / 4: strictly upper / lower part only (diagonal untouched).
template <typename F>
__global__ void laset_kernel(F* A, long lda, int rows, int cols, int uplo, F alpha, F beta) {
  const long total = (long)rows * cols;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i % rows), c = (int)(i / rows);
    if (r == c) { if (uplo < 3) A[r + (long)c * lda] = beta; }
    else if (uplo == 3 ? r < c : (uplo == 4 ? r > c : false)) A[r + (long)c * lda] = alpha;
    else if (uplo == 0 || (uplo == 1 && r < c) || (uplo == 2 && r > c)) A[r + (long)c * lda] = alpha;
  }
}

// *flag <- 1 if any entry of the block is NaN or +-Inf (flag zeroed by the
// caller); the finite half of check_matrix (matrix.py:36-49) on the device.
__global__ void nonfinite_kernel(const double* A, long lda, int rows, int cols, int* flag) {
  const long total = (long)rows * cols;
  int bad = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i % rows), c = (int)(i / rows);
    bad |= !isfinite(A[r + (long)c * lda]);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// A <- alpha * diag(d) A (rows, side 0) or alpha * A diag(d) (cols, side 1).
__global__ void dscale_kernel(double* A, long lda, int rows, int cols, const double* d, int side,
                              double alpha) {
  const long total = (long)rows * cols;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i % rows), c = (int)(i / rows);
    A[r + (long)c * lda] *= alpha * d[side == 0 ? r : c];
  }
}

template <class S, class D>
__global__ void cvt_kernel(const S* __restrict__ src, long lds, D* __restrict__ dst, long ldd,
                           int rows, int cols) {
  const long total = (long)rows * cols;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i % rows), c = (int)(i / rows);
    dst[r + (long)c * ldd] = (D)src[r + (long)c * lds];
  }
}

__global__ void sumsq_partial_f32(const float* __restrict__ A, long lda, int rows, int cols,
                                  double* __restrict__ part);

// A (fp32) <- A * 2^-e with 2^e ~ sqrt(*ss): exact rescaling (no rounding),
// keeps the unstabilised fp32 sampler inside the normal range.
__global__ void pow2_scale_kernel(float* A, long lda, int rows, int cols, const double* ss) {
  const double v = *ss;
  if (!(v > 0.0) || !isfinite(v)) return;
  int e;
  frexp(sqrt(v), &e);
  const float f = ldexpf(1.0f, -e);
  const long total = (long)rows * cols;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i % rows), c = (int)(i / rows);
    A[r + (long)c * lda] *= f;
  }
}

__global__ void diag_f32_kernel(float* A, long lda, int rows, int cols, const double* d) {
  const long total = (long)rows * cols;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int r = (int)(i % rows), c = (int)(i / rows);
    A[r + (long)c * lda] = (r == c) ? (float)d[r] : 0.0f;
  }
}

// B (n x m) = A^T (A m x n), 32 x 32 tiles through padded shared memory.
__global__ void transpose_kernel(const double* __restrict__ A, long lda, double* __restrict__ B,
                                 long ldb, int m, int n) {
  __shared__ double tile[32][33];
  const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = r0 + threadIdx.x, c = c0 + j;
    if (r < m && c < n) tile[j][threadIdx.x] = A[r + (long)c * lda];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = c0 + threadIdx.x, c = r0 + j;  // B row = A col
    if (r < n && c < m) B[r + (long)c * ldb] = tile[threadIdx.x][j];
  }
}

inline int grid_for(long total) {
  const long g = (total + 255) / 256;
  const long cap = 8L * num_sms();
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}
}  // namespace ops

size_t sumsq_scratch_doubles() { return ops::RED_BLOCKS; }

int sumsq(const double* A, long lda, int rows, int cols, double* out, double* scratch,
          cudaStream_t st) {
  if (rows <= 0 || cols <= 0) {
    UTV_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
    return UTV_OK;
  }
  ProfScope ps(PROF_OPS, 2.0 * rows * cols, 8.0 * rows * cols, st, 2);
  ops::sumsq_partial<<<ops::RED_BLOCKS, ops::RED_THREADS, 0, st>>>(A, lda, rows, cols, scratch);
  UTV_CUDA(cudaGetLastError());
  ops::sum_partials<<<1, 512, 0, st>>>(scratch, ops::RED_BLOCKS, out);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int set_identity(double* A, long lda, int rows, int cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return UTV_OK;
  ProfScope ps(PROF_OPS, 0.0, 8.0 * rows * cols, st);
  ops::fill_kernel<<<ops::grid_for((long)rows * cols), 256, 0, st>>>(A, lda, rows, cols, 1.0, 0.0);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int set_zero(double* A, long lda, int rows, int cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return UTV_OK;
  if (lda == rows) {
    UTV_CUDA(cudaMemsetAsync(A, 0, sizeof(double) * rows * (size_t)cols, st));
    return UTV_OK;
  }
  UTV_CUDA(cudaMemset2DAsync(A, lda * sizeof(double), 0, rows * sizeof(double), cols, st));
  return UTV_OK;
}

int copy_mat(const double* src, long lds, double* dst, long ldd, int rows, int cols,
             cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return UTV_OK;
  UTV_CUDA(cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, lds * sizeof(double),
                             rows * sizeof(double), cols, cudaMemcpyDeviceToDevice, st));
  return UTV_OK;
}

int laset(int uplo, int rows, int cols, double alpha, double beta, double* A, long lda,
          cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return UTV_OK;
  ProfScope ps(PROF_OPS, 0.0, 8.0 * rows * cols, st);
  ops::laset_kernel<<<ops::grid_for((long)rows * cols), 256, 0, st>>>(A, lda, rows, cols, uplo,
                                                                      alpha, beta);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int laset_f32(int uplo, int rows, int cols, float alpha, float beta, float* A, long lda,
              cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return UTV_OK;
  ProfScope ps(PROF_OPS, 0.0, 4.0 * rows * cols, st);
  ops::laset_kernel<<<ops::grid_for((long)rows * cols), 256, 0, st>>>(A, lda, rows, cols, uplo,
                                                                      alpha, beta);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int nonfinite(const double* A, long lda, int rows, int cols, int* flag, cudaStream_t st) {
  UTV_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  if (rows <= 0 || cols <= 0) return UTV_OK;
  ProfScope ps(PROF_OPS, 0.0, 8.0 * rows * cols, st);
  const long cap = 8L * num_sms();
  const long g = std::min<long>(cap, ((long)rows * cols + 255) / 256);
  ops::nonfinite_kernel<<<(int)std::max<long>(g, 1), 256, 0, st>>>(A, lda, rows, cols, flag);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int diag_scale(int side, int rows, int cols, const double* d, double alpha, double* A, long lda,
               cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return UTV_OK;
  ProfScope ps(PROF_OPS, (double)rows * cols, 16.0 * rows * cols, st);
  ops::dscale_kernel<<<ops::grid_for((long)rows * cols), 256, 0, st>>>(A, lda, rows, cols, d, side,
                                                                       alpha);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int set_diag(double* A, long lda, int nr, int nc, const double* d, cudaStream_t st) {
  if (nr <= 0 || nc <= 0) return UTV_OK;
  ProfScope ps(PROF_OPS, 0.0, 8.0 * nr * nc, st);
  ops::diag_kernel<<<ops::grid_for((long)nr * nc), 256, 0, st>>>(A, lda, nr, nc, d);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int sumsq_f32(const float* A, long lda, int rows, int cols, double* out, double* scratch,
              cudaStream_t st) {
  if (rows <= 0 || cols <= 0) {
    UTV_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
    return UTV_OK;
  }
  ProfScope ps(PROF_OPS, 2.0 * rows * cols, 4.0 * rows * cols, st, 2);
  ops::sumsq_partial_f32<<<ops::RED_BLOCKS, ops::RED_THREADS, 0, st>>>(A, lda, rows, cols, scratch);
  UTV_CUDA(cudaGetLastError());
  ops::sum_partials<<<1, 512, 0, st>>>(scratch, ops::RED_BLOCKS, out);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int cvt_f32_to_f64(const float* src, long lds, double* dst, long ldd, int rows, int cols,
                   cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return UTV_OK;
  ProfScope ps(PROF_OPS, 0.0, 12.0 * rows * cols, st);
  ops::cvt_kernel<float, double><<<ops::grid_for((long)rows * cols), 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int cvt_f64_to_f32(const double* src, long lds, float* dst, long ldd, int rows, int cols,
                   cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return UTV_OK;
  ProfScope ps(PROF_OPS, 0.0, 12.0 * rows * cols, st);
  ops::cvt_kernel<double, float><<<ops::grid_for((long)rows * cols), 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int pow2_normalize_f32(float* A, long lda, int rows, int cols, double* ss, double* scratch,
                       cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return UTV_OK;
  UTV_CHECK(sumsq_f32(A, lda, rows, cols, ss, scratch, st));
  ProfScope ps(PROF_OPS, (double)rows * cols, 8.0 * rows * cols, st);
  ops::pow2_scale_kernel<<<ops::grid_for((long)rows * cols), 256, 0, st>>>(A, lda, rows, cols, ss);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int set_diag_f32(float* A, long lda, int nr, int nc, const double* d, cudaStream_t st) {
  if (nr <= 0 || nc <= 0) return UTV_OK;
  ProfScope ps(PROF_OPS, 0.0, 4.0 * nr * nc, st);
  ops::diag_f32_kernel<<<ops::grid_for((long)nr * nc), 256, 0, st>>>(A, lda, nr, nc, d);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

int transpose(const double* A, long lda, double* B, long ldb, int m, int n, cudaStream_t st) {
  if (m <= 0 || n <= 0) return UTV_OK;
  ProfScope ps(PROF_OPS, 0.0, 16.0 * m * n, st);
  dim3 grid(ceil_div(m, 32), ceil_div(n, 32)), block(32, 8);
  ops::transpose_kernel<<<grid, block, 0, st>>>(A, lda, B, ldb, m, n);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

}  // namespace utv
