// Householder reconstruction kernels for the TSQR path of row-sharded
// powerURV: the tall QR of A-hat is computed as a TSQR
// tree whose explicit thin Q is turned back into the reference's compact-WY
// factor (Y, Twy) of hqr_full (qr.py:71-100):
//
//   Q - S = L U'   (LU without pivoting, s_j = -sign(pivot_j), sign(0) = +1)
//   Y = L,  Twy = -U' S L1^{-T},  R = S R_tsqr.
//
// With |s_j - pivot| >= 1 every tau_j = |pivot_j| + 1 lies in [1, 2], which
// is exactly the dlarfg branch hqr_full takes (beta = -sign(alpha)||x||), so
// the reconstruction reproduces hqr_full's Y, Twy and R up to roundoff for
// full-rank input (the skip rule, tau = 0, only arises for exactly
// dependent columns).
//
// Kernels (column blocks of NB = 32):
//  * lu_diag_kernel: the NB x NB diagonal block, in place, one CTA (with the
//    sign choice).
//  * lu_panel_kernel: rows-parallel; each thread solves l (1 x NB) U11 = x
//    for its rows by forward substitution — no inter-CTA communication.
//  * lu_u12_kernel: U12 = L11^{-1} A12 for the NB top rows (column-parallel).
//  * the trailing update A22 -= L21 U12 is a DMMA GEMM (K = NB).
#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace lu {
constexpr int NB = 32;
constexpr int THREADS = 256;

// M = op(A) upper triangular: element M[k][j] (k <= j).
__device__ __forceinline__ double mval(const double* A, long lda, bool trans, int k, int j) {
  return trans ? A[j + (long)k * lda] : A[k + (long)j * lda];
}

// In-place factorisation of the jb x jb diagonal block at (j0, j0) of P
// (one CTA): (D - S) = L11 U11 with s_k = -sign(pivot_k), signs -> s[j0..].
__global__ void __launch_bounds__(THREADS) lu_diag_kernel(double* P, long ldp, int j0, int jb,
                                                           double* s) {
  __shared__ double U[NB][NB + 1];
  const int t = threadIdx.x;
  for (int idx = t; idx < jb * jb; idx += THREADS) {
    const int r = idx % jb, c = idx / jb;
    U[r][c] = P[(j0 + r) + (long)(j0 + c) * ldp];
  }
  __syncthreads();
  for (int k = 0; k < jb; ++k) {
    const double pk = U[k][k];
    const double sk = pk >= 0.0 ? -1.0 : 1.0;  // sign(0) = +1
    const double d = pk - sk;
    __syncthreads();
    if (t == 0) {
      U[k][k] = d;
      s[j0 + k] = sk;
    }
    if (t > k && t < jb) U[t][k] = U[t][k] / d;
    __syncthreads();
    const int w = jb - k - 1;
    for (int idx = t; idx < w * w; idx += THREADS) {
      const int r = k + 1 + idx % w, c = k + 1 + idx / w;
      U[r][c] = fma(-U[r][k], U[k][c], U[r][c]);
    }
    __syncthreads();
  }
  for (int idx = t; idx < jb * jb; idx += THREADS) {
    const int r = idx % jb, c = idx / jb;
    P[(j0 + r) + (long)(j0 + c) * ldp] = U[r][c];
  }
}

// Rows [rbeg, rows) of the column block [j0, j0+jb) of P:
//   x <- x * M_jj^{-1},  M_jj = op(A)[j0.., j0..] upper (unit diagonal if `unit`).
// Row-parallel forward substitution, no inter-CTA communication.
struct PanelArgs {
  double* P;
  long ldp;
  long rbeg, rows;
  int j0, jb;
  const double* A;
  long lda;
  int trans, unit;
};

__global__ void __launch_bounds__(THREADS) lu_panel_kernel(PanelArgs a) {
  __shared__ double U[NB][NB + 1];
  __shared__ double dinv[NB];
  const int t = threadIdx.x;
  const int jb = a.jb;
  for (int idx = t; idx < jb * jb; idx += THREADS) {
    const int r = idx % jb, c = idx / jb;
    U[r][c] = (r <= c) ? (r == c && a.unit ? 1.0 : mval(a.A, a.lda, a.trans, a.j0 + r, a.j0 + c)) : 0.0;
  }
  __syncthreads();
  if (t < jb) dinv[t] = 1.0 / U[t][t];
  __syncthreads();
  for (long i = a.rbeg + blockIdx.x * (long)THREADS + t; i < a.rows; i += (long)gridDim.x * THREADS) {
    double x[NB];
    double* row = a.P + i + (long)a.j0 * a.ldp;
#pragma unroll
    for (int c = 0; c < NB; ++c) x[c] = (c < jb) ? row[(long)c * a.ldp] : 0.0;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c < jb) {
        double v = x[c];
#pragma unroll
        for (int k = 0; k < c; ++k) v = fma(-x[k], U[k][c], v);
        x[c] = a.unit ? v : v * dinv[c];
      }
    }
#pragma unroll
    for (int c = 0; c < NB; ++c)
      if (c < jb) row[(long)c * a.ldp] = x[c];
  }
}

// U12 = L11^{-1} A12: top rows [j0, j0+jb) of columns [c0, ncols) of P.
__global__ void __launch_bounds__(THREADS) lu_u12_kernel(double* P, long ldp, int j0, int jb,
                                                          int c0, int ncols) {
  __shared__ double L[NB][NB + 1];
  const int t = threadIdx.x;
  for (int idx = t; idx < jb * jb; idx += THREADS) {
    const int r = idx % jb, c = idx / jb;
    L[r][c] = P[(j0 + r) + (long)(j0 + c) * ldp];
  }
  __syncthreads();
  for (int c = c0 + blockIdx.x * THREADS + t; c < ncols; c += gridDim.x * THREADS) {
    double* col = P + j0 + (long)c * ldp;
    double x[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) x[r] = (r < jb) ? col[r] : 0.0;
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      if (r < jb) {
        double v = x[r];
#pragma unroll
        for (int k = 0; k < r; ++k) v = fma(-L[r][k], x[k], v);
        x[r] = v;  // unit lower
      }
    }
#pragma unroll
    for (int r = 0; r < NB; ++r)
      if (r < jb) col[r] = x[r];
  }
}
}  // namespace lu

static int row_grid(long rows) {
  long g = (rows + lu::THREADS - 1) / lu::THREADS;
  const long cap = 4L * num_sms();
  if (g > cap) g = cap;
  return g < 1 ? 1 : (int)g;
}

size_t lu_ws_doubles() { return SPLITK_WS; }

// B[:, j1:c1) -= B[:, j0:j1) M[j0:j1, j1:c1),  M = op(A) upper.
static int trsm_update(bool trans, const double* A, long lda, Mat B, int j0, int j1, int c1,
                       double* ws, size_t ws_doubles, cudaStream_t st) {
  const int m = B.rows;
  if (!trans)
    return dgemm(false, false, m, c1 - j1, j1 - j0, -1.0, B.at(0, j0), B.ld,
                 A + j0 + (long)j1 * lda, lda, 1.0, B.at(0, j1), B.ld, ws, ws_doubles, st);
  // M[j0.., j1..] = A[j1.., j0..]^T
  return dgemm(false, true, m, c1 - j1, j1 - j0, -1.0, B.at(0, j0), B.ld,
               A + j1 + (long)j0 * lda, lda, 1.0, B.at(0, j1), B.ld, ws, ws_doubles, st);
}

// Outer block width of the two-level LU / trsm: the NB-wide kernels and
// K = NB updates stay inside one NB2-wide column panel (HBM-bound but narrow),
// the wide trailing updates are K = NB2 DMMA GEMMs (tensor-bound).
constexpr int NB2 = 256;

// In-place LU without pivoting of (P - diag(s)) for the columns [c0, c1) of a
// rows x n panel, rows [c0, rows), updating only columns < c1 (NB blocks).
static int getrf_signed_cols(Mat P, int c0, int c1, double* s, double* ws, size_t ws_doubles,
                             cudaStream_t st) {
  const int rows = P.rows;
  for (int j0 = c0; j0 < c1; j0 += lu::NB) {
    const int jb = c1 - j0 < lu::NB ? c1 - j0 : lu::NB;
    {
      ProfScope ps(PROF_OPS, 2.0 / 3.0 * jb * jb * jb, 16.0 * jb * jb, st);
      lu::lu_diag_kernel<<<1, lu::THREADS, 0, st>>>(P.p, P.ld, j0, jb, s);
      UTV_CUDA(cudaGetLastError());
    }
    if (j0 + jb < rows) {
      lu::PanelArgs a;
      a.P = P.p; a.ldp = P.ld; a.rbeg = j0 + jb; a.rows = rows; a.j0 = j0; a.jb = jb;
      a.A = P.p; a.lda = P.ld; a.trans = 0; a.unit = 0;
      ProfScope ps(PROF_OPS, (double)(rows - j0 - jb) * jb * jb, 16.0 * (rows - j0 - jb) * jb, st);
      lu::lu_panel_kernel<<<row_grid(rows - j0 - jb), lu::THREADS, 0, st>>>(a);
      UTV_CUDA(cudaGetLastError());
    }
    if (j0 + jb < c1) {
      {
        ProfScope ps(PROF_OPS, (double)jb * jb * (c1 - j0 - jb), 16.0 * jb * (c1 - j0 - jb), st);
        lu::lu_u12_kernel<<<ceil_div(c1 - j0 - jb, lu::THREADS), lu::THREADS, 0, st>>>(
            P.p, P.ld, j0, jb, j0 + jb, c1);
        UTV_CUDA(cudaGetLastError());
      }
      // A22 -= L21 U12 inside the panel
      UTV_CHECK(dgemm(false, false, rows - j0 - jb, c1 - j0 - jb, jb, -1.0, P.at(j0 + jb, j0), P.ld,
                      P.at(j0, j0 + jb), P.ld, 1.0, P.at(j0 + jb, j0 + jb), P.ld, ws, ws_doubles, st));
    }
  }
  return UTV_OK;
}

// In-place LU without pivoting of (P - diag(s)) for a rows x n panel (rows >= n):
// L (unit lower trapezoidal) below the diagonal, U' on/above, s[0..n) = signs.
// Right-looking over NB2-wide panels: panel LU (NB blocks), U12 = L11^{-1} A12
// by NB-block forward substitution, A22 -= L21 U12 as one K = NB2 GEMM.
int getrf_signed(Mat P, double* s, double* ws, size_t ws_doubles, cudaStream_t st) {
  const int rows = P.rows, n = P.cols;
  if (rows < n) return -1;
  for (int J0 = 0; J0 < n; J0 += NB2) {
    const int J1 = n - J0 < NB2 ? n : J0 + NB2;
    UTV_CHECK(getrf_signed_cols(P, J0, J1, s, ws, ws_doubles, st));
    if (J1 >= n) break;
    for (int j0 = J0; j0 < J1; j0 += lu::NB) {
      const int jb = J1 - j0 < lu::NB ? J1 - j0 : lu::NB;
      {
        ProfScope ps(PROF_OPS, (double)jb * jb * (n - J1), 16.0 * jb * (n - J1), st);
        lu::lu_u12_kernel<<<ceil_div(n - J1, lu::THREADS), lu::THREADS, 0, st>>>(P.p, P.ld, j0, jb,
                                                                                  J1, n);
        UTV_CUDA(cudaGetLastError());
      }
      if (j0 + jb < J1)
        UTV_CHECK(dgemm(false, false, J1 - j0 - jb, n - J1, jb, -1.0, P.at(j0 + jb, j0), P.ld,
                        P.at(j0, J1), P.ld, 1.0, P.at(j0 + jb, J1), P.ld, ws, ws_doubles, st));
    }
    UTV_CHECK(dgemm(false, false, rows - J1, n - J1, J1 - J0, -1.0, P.at(J1, J0), P.ld,
                    P.at(J0, J1), P.ld, 1.0, P.at(J1, J1), P.ld, ws, ws_doubles, st));
  }
  return UTV_OK;
}

// B[:, c0:c1) <- B[:, c0:c1) M[c0:c1, c0:c1]^{-1} (NB blocks, updates inside the panel).
static int trsm_cols(bool trans, bool unit, const double* A, long lda, Mat B, int c0, int c1,
                     double* ws, size_t ws_doubles, cudaStream_t st) {
  const int m = B.rows;
  for (int j0 = c0; j0 < c1; j0 += lu::NB) {
    const int jb = c1 - j0 < lu::NB ? c1 - j0 : lu::NB;
    lu::PanelArgs a;
    a.P = B.p; a.ldp = B.ld; a.rbeg = 0; a.rows = m; a.j0 = j0; a.jb = jb;
    a.A = A; a.lda = lda; a.trans = trans ? 1 : 0; a.unit = unit ? 1 : 0;
    {
      ProfScope ps(PROF_OPS, (double)m * jb * jb, 16.0 * m * jb, st);
      lu::lu_panel_kernel<<<row_grid(m), lu::THREADS, 0, st>>>(a);
      UTV_CUDA(cudaGetLastError());
    }
    if (j0 + jb < c1) UTV_CHECK(trsm_update(trans, A, lda, B, j0, j0 + jb, c1, ws, ws_doubles, st));
  }
  return UTV_OK;
}

// B (m x n) <- B * M^{-1}, M = op(A) upper triangular n x n:
// uplo 'U' + trans 'N' (M = A) or uplo 'L' + trans 'T' (M = A^T); unit diagonal optional.
// Two levels like getrf_signed: NB2-wide panels solved in NB blocks, then
// B[:, J1:] -= X_J M[J0:J1, J1:] as one K = NB2 GEMM.
int trsm_right_upper(bool trans, bool unit, int n, const double* A, long lda, Mat B, double* ws,
                     size_t ws_doubles, cudaStream_t st) {
  const int m = B.rows;
  if (B.cols != n) return -1;
  if (m <= 0 || n <= 0) return UTV_OK;
  for (int J0 = 0; J0 < n; J0 += NB2) {
    const int J1 = n - J0 < NB2 ? n : J0 + NB2;
    UTV_CHECK(trsm_cols(trans, unit, A, lda, B, J0, J1, ws, ws_doubles, st));
    if (J1 < n) UTV_CHECK(trsm_update(trans, A, lda, B, J0, J1, n, ws, ws_doubles, st));
  }
  return UTV_OK;
}

}  // namespace utv
