// Column-pivoted Householder QR (HQRCP) — the paper's comparator,
// utvkit qr.py:152-204.
//
// The reference is the Businger-Golub right-looking algorithm: per column,
// greedy largest-norm pivot with a 1e-12 tie window resolving to the leftmost
// column, reflector (qr.py:43-60 convention and skip rule), rank-1 update of
// the whole trailing block, squared-norm downdate with an exact recompute when
// the estimate falls below eps of its reference value.  Every pivot depends on
// the previous column's update, so the algorithm is a sequence of min(m,n)
// dependent steps, each streaming the trailing block once: HBM-bound.
//
// B200 design: ONE persistent cooperative kernel, one grid barrier per column.
//  * Columns stay at their physical position; each CTA owns the physical
//    columns c = g, g+G, ...  The permutation lives replicated in every CTA's
//    shared memory (all CTAs perform the same swaps), so no column is moved.
//  * After the barrier every CTA redundantly (and bit-identically: fixed-order
//    reductions) picks the pivot from the double-buffered norm array and
//    builds the reflector from the pivot column in L2; no second barrier.
//  * The update of an owned column is column-local: load rows j..m-1 into
//    registers (coalesced, RPT per thread), dot with v (smem), block reduce,
//    update in registers, store, downdate its norm (recompute from the
//    registers when the reference would).  One HBM read + write of the
//    trailing block per step — the Level-2 bound of the reference algorithm.
//  * R is written in pivoted order into a separate output buffer by the
//    column's owner, so the pivot column other CTAs are reading is never
//    overwritten inside a step.
// Twy is formed afterwards: 256-wide diagonal blocks from Y^T Y (DMMA GEMM)
// and the forward recursion (qr.py:63-68), then merged by build_t.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "utv_internal.h"

namespace utv {
namespace pqp {

constexpr int THREADS = 256;
constexpr int NW = THREADS / 32;
constexpr int MAXDIM = 16384;  // v (m doubles) + perm (n ints) + flags fit one CTA's smem
// Beyond MAXDIM rows or columns the same kernel runs with the per-CTA
// reflector, permutation and flags in global memory (L2) and the column
// update in two strided passes instead of registers (BIG); the per-thread
// summation order is the same, so results are bitwise identical.
constexpr double EPS = 2.220446049250313e-16;  // matrix.py:13
constexpr double TIE = 1e-12;                   // qr.py:148 _PIVOT_TIE_RTOL

struct Args {
  double* A;    // physical working copy, m x n (destroyed)
  long lda;
  double* R;    // output, pivoted column order, m x n
  long ldr;
  double* Y;    // output, m x r, zero-initialised
  long ldy;
  double* tau;  // r
  int* perm;    // n
  double* nrm;  // [2][n] squared norms (physical index); nrm[0..n) initialised
  double* ref;  // [n]
  const double* fro2;
  int m, n, r;
  unsigned* ctr;
  double* vbig;          // BIG: [G][m] reflector copies
  int* pbig;             // BIG: [G][n] permutation copies
  unsigned char* dbig;   // BIG: [G][n] pivoted flags
};

__host__ __device__ inline size_t smem_bytes(int m, int n) {
  return (size_t)m * 8 + 16 * NW * 8 + (size_t)n * 4 + (size_t)n + 64;
}

// Fixed-order block reductions (identical result in every CTA for identical
// inputs).  `buf` alternates between two [NW] slots so one barrier suffices.
__device__ __forceinline__ double block_sum(double x, double* buf) {
  x = warp_sum(x);
  if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = x;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) s += buf[w];
  return s;
}
template <int K>
__device__ __forceinline__ void block_sum_k(double (&x)[K], double* buf) {
#pragma unroll
  for (int b = 0; b < K; ++b) {
    x[b] = warp_sum(x[b]);
    if ((threadIdx.x & 31) == 0) buf[b * NW + (threadIdx.x >> 5)] = x[b];
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < K; ++b) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += buf[b * NW + w];
    x[b] = s;
  }
}
__device__ __forceinline__ double block_max(double x, double* buf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = x;
  __syncthreads();
  double s = buf[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) s = fmax(s, buf[w]);
  return s;
}
__device__ __forceinline__ int block_min_int(int x, int* buf) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = min(x, __shfl_xor_sync(0xffffffffu, x, o));
  if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = x;
  __syncthreads();
  int s = buf[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) s = min(s, buf[w]);
  return s;
}

template <int RPT, bool BIG>
__global__ void __launch_bounds__(THREADS, 1) qrcp_kernel(Args a) {
  extern __shared__ double sm[];
  const int t = threadIdx.x, g = blockIdx.x, G = gridDim.x;
  double* v = BIG ? a.vbig + (size_t)g * a.m : sm;        // [m] reflector of the current column
  double* red = BIG ? sm : v + a.m;                        // [4][4*NW] reduction slots
  int* perm_s = BIG ? a.pbig + (size_t)g * a.n : (int*)(red + 16 * NW);  // [n] logical -> physical
  unsigned char* done_s = BIG ? a.dbig + (size_t)g * a.n : (unsigned char*)(perm_s + a.n);  // [n] pivoted

  const int m = a.m, n = a.n;
  const double thresh = EPS * sqrt(*a.fro2);  // qr.py:162 (eps * ||A||_F)
  for (int k = t; k < n; k += THREADS) {
    perm_s[k] = k;
    done_s[k] = 0;
  }
  __syncthreads();
  int rb = 0;  // alternating reduction slot
  auto rbuf = [&]() {
    rb = (rb + 1) & 3;
    return red + rb * 4 * NW;
  };
  unsigned nbar = 0;

  for (int j = 0; j < a.r; ++j) {
    const double* ncur = a.nrm + (size_t)(j & 1) * n;
    double* nnxt = a.nrm + (size_t)((j + 1) & 1) * n;

    // ---- pivot (qr.py:171-180): leftmost logical column within the tie window ----
    double lmax = 0.0;
    for (int k = j + t; k < n; k += THREADS) lmax = fmax(lmax, __ldcg(ncur + perm_s[k]));
    const double top = block_max(lmax, rbuf());
    int piv = j;
    if (top > 0.0) {
      const double lim = top * (1.0 - TIE);
      int lk = INT_MAX;
      for (int k = j + t; k < n; k += THREADS)
        if (__ldcg(ncur + perm_s[k]) >= lim) {
          lk = k;
          break;
        }
      piv = block_min_int(lk, (int*)rbuf());
    }
    if (t == 0) {
      const int pj = perm_s[piv];
      perm_s[piv] = perm_s[j];
      perm_s[j] = pj;
      done_s[pj] = 1;
    }
    __syncthreads();
    const int p = perm_s[j];

    // ---- reflector of A[j:, p] (qr.py:43-60), redundantly in every CTA ----
    const int nr = m - j;
    const double* colp = a.A + (long)p * a.lda + j;
    double sig = 0.0;
    for (int i = t; i < nr; i += THREADS) {
      const double x = __ldcg(colp + i);
      v[i] = x;
      if (i > 0) sig = fma(x, x, sig);
    }
    const double sigma = block_sum(sig, rbuf());  // also publishes v[]
    const double alpha = __ldcg(colp);  // not v[0]: thread 0 overwrites it below
    const double xnorm = sqrt(alpha * alpha + sigma);
    const bool skip = (xnorm <= thresh) || (sigma == 0.0);
    double tau = 0.0, beta = alpha;
    if (!skip) {
      const double sgn = alpha >= 0.0 ? 1.0 : -1.0;
      const double v1 = alpha + sgn * xnorm;
      tau = 2.0 / (1.0 + sigma / (v1 * v1));
      beta = -sgn * xnorm;
      for (int i = t; i < nr; i += THREADS) v[i] = i == 0 ? 1.0 : v[i] / v1;
      __syncthreads();
    }

    // ---- outputs of column j (the pivot's owner) ----
    if (p % G == g) {
      double* yj = a.Y + (long)j * a.ldy;
      double* rj = a.R + (long)j * a.ldr;
      const double* ap = a.A + (long)p * a.lda;
      for (int i = t; i < m; i += THREADS) {
        if (i >= j) yj[i] = skip ? (i == j ? 1.0 : 0.0) : v[i - j];
        rj[i] = i < j ? ap[i] : (i == j ? beta : 0.0);
      }
      if (t == 0) a.tau[j] = tau;
    }

    // ---- update + downdate of the owned trailing columns (qr.py:190-204) ----
    for (int c = g; c < n; c += G) {
      if (done_s[c]) continue;
      double* col = a.A + (long)c * a.lda + j;
      double x[RPT];
      // every thread derives the new row-j entry itself (v[0] = 1, so it is
      // fma(-1, w, A[j,c]) exactly as thread 0 stores it): no extra barrier
      double rj = col[0];
      if (BIG) {
        if (!skip) {
          double d = 0.0;
          for (int i = t; i < nr; i += THREADS) d = fma(v[i], col[i], d);
          const double w = tau * block_sum(d, rbuf());
          for (int i = t; i < nr; i += THREADS) col[i] = fma(-v[i], w, col[i]);
          rj = fma(-1.0, w, rj);
        }
        double nn = fmax(__ldcg(ncur + c) - rj * rj, 0.0);
        if (nn <= EPS * a.ref[c]) {
          double s = 0.0;
          for (int i = t; i < nr; i += THREADS)
            if (i >= 1) s = fma(col[i], col[i], s);
          nn = block_sum(s, rbuf());
          if (t == 0) a.ref[c] = nn;
        }
        if (t == 0) nnxt[c] = nn;
        continue;
      }
      if (!skip) {
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int i = t + k * THREADS;
          x[k] = i < nr ? col[i] : 0.0;
        }
        double d = 0.0;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int i = t + k * THREADS;
          if (i < nr) d = fma(v[i], x[k], d);
        }
        const double w = tau * block_sum(d, rbuf());
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int i = t + k * THREADS;
          if (i < nr) {
            x[k] = fma(-v[i], w, x[k]);
            col[i] = x[k];
          }
        }
        rj = fma(-1.0, w, rj);
      }
      double nn = fmax(__ldcg(ncur + c) - rj * rj, 0.0);
      if (nn <= EPS * a.ref[c]) {  // exact recompute (qr.py:200-204)
        double s = 0.0;
        if (!skip) {
#pragma unroll
          for (int k = 0; k < RPT; ++k) {
            const int i = t + k * THREADS;
            if (i >= 1 && i < nr) s = fma(x[k], x[k], s);
          }
        } else {
          for (int i = t; i < nr; i += THREADS)
            if (i >= 1) s = fma(col[i], col[i], s);
        }
        nn = block_sum(s, rbuf());
        if (t == 0) a.ref[c] = nn;
      }
      if (t == 0) nnxt[c] = nn;
    }

    ++nbar;
    if (G > 1) grid_barrier(a.ctr, nbar * (unsigned)G);
    else __syncthreads();
  }
  if (g == 0)
    for (int k = t; k < n; k += THREADS) a.perm[k] = perm_s[k];
}

// Squared column norms (qr.py:165): nrm[c] = ref[c] = sum_i A[i,c]^2.
__global__ void colnorm_kernel(const double* __restrict__ A, long lda, int m, double* nrm,
                               double* ref) {
  __shared__ double buf[NW];
  const int c = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += THREADS) {
    const double x = A[i + (long)c * lda];
    s = fma(x, x, s);
  }
  s = block_sum(s, buf);
  if (threadIdx.x == 0) {
    nrm[c] = s;
    ref[c] = s;
  }
}

// Columns r..n-1 of R (wide case) were never pivoted: gather them in
// permuted order.
__global__ void gather_tail_kernel(const double* __restrict__ A, long lda, double* R, long ldr,
                                   const int* __restrict__ perm, int m, int r) {
  const int k = r + blockIdx.x;
  const double* src = A + (long)perm[k] * lda;
  for (int i = threadIdx.x; i < m; i += blockDim.x) R[i + (long)k * ldr] = src[i];
}

// Diagonal block of Twy from the Gram matrix S = Yb^T Yb and tau by the
// forward recursion of qr.py:63-68:  T[r,i] = -tau_i sum_{q=r}^{i-1} T[r,q] S[q,i].
// Row r only depends on row r, so each thread owns one row.
__global__ void larft_kernel(const double* __restrict__ S, long lds, const double* __restrict__ tau,
                             double* T, long ldt, int r) {
  const int j0 = blockIdx.x * QR_PANEL;
  const int jb = min(QR_PANEL, r - j0);
  const int row = threadIdx.x;
  if (row >= jb) return;
  const double* Sb = S + (size_t)blockIdx.x * QR_PANEL * lds;  // [jb][lds] column-major block
  double* Tb = T + j0 + (long)j0 * ldt;
  Tb[row + (long)row * ldt] = tau[j0 + row];
  for (int i = row + 1; i < jb; ++i) {
    double s = 0.0;
    for (int q = row; q < i; ++q) s = fma(Tb[row + (long)q * ldt], Sb[q + (long)i * lds], s);
    Tb[row + (long)i * ldt] = -tau[j0 + i] * s;
  }
}

}  // namespace pqp

int qrcp_max_dim() { return INT_MAX; }

static bool qrcp_big(int m, int n) {
  static const bool forced = getenv("UTV_QRCP_BIG") != nullptr;  // test knob
  return forced || m > pqp::MAXDIM || n > pqp::MAXDIM;
}

static size_t qrcp_big_doubles(int m, int n) {
  // one reflector / permutation / flag copy per CTA (at most one CTA per SM)
  return (size_t)num_sms() * ((size_t)m + (size_t)(n + 1) / 2 + (size_t)(n + 7) / 8 + 64);
}

size_t qrcp_ws_doubles(int m, int n) {
  const int r = m < n ? m : n;
  const int nblk = (r + QR_PANEL - 1) / QR_PANEL;
  return 3 * (size_t)n + r + 64 + sumsq_scratch_doubles() + (size_t)nblk * QR_PANEL * QR_PANEL +
         2 * (size_t)round_up(r, 4) * QR_PANEL + SPLITK_WS + 2048 +
         (qrcp_big(m, n) ? qrcp_big_doubles(m, n) : 0);
}

static int g_qrcp_attr[4] = {0, 0, 0, 0};

int qrcp(int m, int n, double* A, long lda, double* R, long ldr, double* Y, long ldy, double* T,
         long ldt, int* perm, double* ws, size_t ws_doubles, cudaStream_t st) {
  using namespace pqp;
  if (m < 1) return -1;
  if (n < 1) return -2;
  if (ws_doubles < qrcp_ws_doubles(m, n)) return UTV_ERR_WORKSPACE;
  const int r = m < n ? m : n;
  Arena ar{(char*)ws, ws_doubles * sizeof(double), 0};
  double* nrm = ar.take(2 * (size_t)n);
  double* ref = ar.take(n);
  double* fro2 = ar.take(8);
  unsigned* ctr = (unsigned*)ar.take(8);
  double* tau = ar.take(r);
  double* red = ar.take(sumsq_scratch_doubles());
  const int nblk = (r + QR_PANEL - 1) / QR_PANEL;
  double* S = ar.take((size_t)nblk * QR_PANEL * QR_PANEL);
  const size_t bt_n = 2 * (size_t)round_up(r, 4) * QR_PANEL + SPLITK_WS + 512;
  double* bt = ar.take(bt_n);
  if (!bt) return UTV_ERR_WORKSPACE;
  const bool big = qrcp_big(m, n);
  double* vbig = nullptr;
  int* pbig = nullptr;
  unsigned char* dbig = nullptr;
  if (big) {
    const size_t ns = num_sms();
    vbig = ar.take(ns * (size_t)m);
    pbig = (int*)ar.take(ns * (size_t)((n + 1) / 2));
    dbig = (unsigned char*)ar.take(ns * (size_t)((n + 7) / 8));
    if (!dbig) return UTV_ERR_WORKSPACE;
  }

  UTV_CHECK(sumsq(A, lda, m, n, fro2, red, st));
  UTV_CHECK(set_zero(Y, ldy, m, r, st));
  UTV_CHECK(set_zero(T, ldt, r, r, st));
  {
    ProfScope ps(PROF_OPS, 2.0 * m * n, 8.0 * m * n, st);
    colnorm_kernel<<<n, THREADS, 0, st>>>(A, lda, m, nrm, ref);
    UTV_CUDA(cudaGetLastError());
  }
  Args a;
  a.A = A; a.lda = lda; a.R = R; a.ldr = ldr; a.Y = Y; a.ldy = ldy;
  a.tau = tau; a.perm = perm; a.nrm = nrm; a.ref = ref; a.fro2 = fro2;
  a.m = m; a.n = n; a.r = r; a.ctr = ctr;
  a.vbig = vbig; a.pbig = pbig; a.dbig = dbig;
  const size_t smem = big ? 16 * NW * sizeof(double) : smem_bytes(m, n);
  void* fn;
  int ti;
  if (big) { fn = (void*)qrcp_kernel<1, true>; ti = 3; }
  else if (m <= 4 * THREADS) { fn = (void*)qrcp_kernel<4, false>; ti = 0; }
  else if (m <= 16 * THREADS) { fn = (void*)qrcp_kernel<16, false>; ti = 1; }
  else { fn = (void*)qrcp_kernel<64, false>; ti = 2; }
  if (!g_qrcp_attr[ti]) {
    UTV_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  big ? (int)smem : (int)smem_bytes(MAXDIM, MAXDIM)));
    g_qrcp_attr[ti] = 1;
  }
  // every co-resident CTA streams its own column: more CTAs per SM hide the
  // per-column load -> reduce -> store latency chain (small m: 2 per SM)
  int occ = 1;
  UTV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, THREADS, smem));
  if (occ < 1) return UTV_ERR_CUDA;
  if (getenv("UTV_QRCP_OCC1") || big) occ = 1;  // BIG: one workspace copy per SM
  int G = (n + 3) / 4;
  if (G > occ * num_sms()) G = occ * num_sms();
  if (G < 1) G = 1;
  {
    // algorithmic: sum_j 4 (m-j)(n-j) flops; one read + write of the trailing block per step
    double fl = 0.0, by = 0.0;
    for (int j = 0; j < r; ++j) {
      fl += 4.0 * (double)(m - j) * (n - j);
      by += 16.0 * (double)(m - j) * (n - j - 1);
    }
    ProfScope ps(PROF_QRCP, fl, by, st);
    UTV_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned), st));
    void* args[] = {&a};
    UTV_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(THREADS), args, smem, st));
  }
  if (n > r) {
    gather_tail_kernel<<<n - r, THREADS, 0, st>>>(A, lda, R, ldr, perm, m, r);
    UTV_CUDA(cudaGetLastError());
  }
  // Twy: diagonal blocks (Gram + forward recursion), then the block merges
  const long lds = QR_PANEL;
  for (int b = 0; b < nblk; ++b) {
    const int j0 = b * QR_PANEL, jb = (r - j0 < QR_PANEL) ? r - j0 : QR_PANEL;
    UTV_CHECK(dgemm(true, false, jb, jb, m - j0, 1.0, Y + j0 + (long)j0 * ldy, ldy,
                    Y + j0 + (long)j0 * ldy, ldy, 0.0, S + (size_t)b * QR_PANEL * lds, lds,
                    bt, SPLITK_WS, st));
  }
  {
    ProfScope ps(PROF_OPS, (double)r * QR_PANEL * QR_PANEL / 3.0, 16.0 * r * QR_PANEL, st);
    larft_kernel<<<nblk, QR_PANEL, 0, st>>>(S, lds, tau, T, ldt, r);
    UTV_CUDA(cudaGetLastError());
  }
  UTV_CHECK(build_t(Mat{Y, ldy, m, r}, Mat{T, ldt, r, r}, bt, bt_n, st));
  return UTV_OK;
}

}  // namespace utv
