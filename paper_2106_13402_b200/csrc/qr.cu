// K3 panel QR (geqr2 + larft), K4 blocked QR (geqrf + full compact-WY
// triangle), K2 compact-WY apply (larfb) and K5 orgqr.
//
// Reference semantics (utvkit qr.py):
//  * reflector: beta = -sign(alpha)||x||, sign(0)=+1, v0 = 1,
//    tau = 2/(1+sigma/v1^2)                                 (qr.py:43-60)
//  * skip rule: ||x|| <= eps*||A||_F (whole input) or sigma == 0 =>
//    tau = 0, Y[j,j] = 1, R below diagonal zeroed          (qr.py:53-54,86-93)
//  * forward compact-WY triangle                            (qr.py:63-68)
//  * apply_q left/right, trans                              (qr.py:103-121)
//  * materialize_q                                          (qr.py:124-131)
//
// B200 design:
//  * leaf_qr_kernel factors a rows x 32 leaf with one cooperative grid of
//    up to 148 CTAs, each holding a row slab in shared memory.  Per column a
//    single fixed-order grid reduction delivers ||x||^2, x^T P (all columns)
//    and the row j broadcast, from which the reflector, the rank-1 update
//    and the WY column follow without a second pass.
//  * 32-wide leaves are combined right-looking inside a <= 256-wide panel
//    (K=32 updates stay L2-resident), panels are combined right-looking with
//    K=256 DMMA GEMM updates; triangles merge as T12 = -T1 (Y1^T Y2) T2.
#include <cooperative_groups.h>

#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace qr {
constexpr int NB = 32;       // leaf width
constexpr int LT = 256;      // leaf threads
constexpr int RC_MIN = 64;   // min rows per CTA (row j of every column lives in CTA 0)
constexpr int RC_MAX = 640;  // max rows per CTA (smem)
constexpr int GMAX = 128;
constexpr int PANEL = QR_PANEL;  // outer panel width
constexpr double EPS = 2.220446049250313e-16;

struct LeafArgs {
  double* P;
  long ldp;
  double* Y;
  long ldy;
  double* T;
  long ldt;
  int rows, jb, rc;
  const double* fro2;
  double* part;   // [2][G][NB]
  double* rowj;   // [2][NB]
  unsigned* ctr;  // zeroed before launch
};

__host__ __device__ inline size_t leaf_smem_doubles(int rc) {
  return (size_t)(rc + 1) * NB + NB * (NB + 1) + 8 * NB + 5 * NB + 8;
}

__global__ void __launch_bounds__(LT) leaf_qr_kernel(LeafArgs a) {
  extern __shared__ double sm[];
  const int ld = a.rc + 1;  // odd pitch: column-strided access is conflict free
  double* tile = sm;
  double* Ts = tile + (size_t)ld * NB;
  double* red = Ts + NB * (NB + 1);
  double* S = red + 8 * NB;
  double* R = S + NB;
  double* W = R + NB;
  double* Z = W + NB;
  const int g = blockIdx.x, G = gridDim.x;
  const int r0 = g * a.rc;
  const int nr = max(0, min(a.rc, a.rows - r0));
  const int jb = a.jb;
  const double thr = EPS * sqrt(*a.fro2);

  for (int idx = threadIdx.x; idx < nr * jb; idx += LT) {
    const int i = idx % nr, c = idx / nr;
    tile[i + c * ld] = a.P[(r0 + i) + (long)c * a.ldp];
  }
  if (g == 0)
    for (int idx = threadIdx.x; idx < NB * (NB + 1); idx += LT) Ts[idx] = 0.0;
  __syncthreads();

  for (int j = 0; j < jb; ++j) {
    const int i_lo = max(0, j + 1 - r0);  // first local row with global index > j
    {  // local partials S_c = sum_{i>j} x_i P[i,c]
      const int c = threadIdx.x & 31, grp = threadIdx.x >> 5;
      double acc = 0.0;
      if (c < jb)
        for (int i = i_lo + grp; i < nr; i += 8) acc = fma(tile[i + j * ld], tile[i + c * ld], acc);
      red[grp * NB + c] = acc;
    }
    __syncthreads();
    if (threadIdx.x < NB) {
      const int c = threadIdx.x;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += red[q * NB + c];
      a.part[((j & 1) * G + g) * NB + c] = s;
      if (g == 0) a.rowj[(j & 1) * NB + c] = (c < jb) ? tile[j + c * ld] : 0.0;
    }
    if (G > 1) grid_barrier(a.ctr, (unsigned)G * (unsigned)(j + 1));
    else __syncthreads();
    if (threadIdx.x < NB) {
      const int c = threadIdx.x;
      double s = 0.0;
      for (int q = 0; q < G; ++q) s += __ldcg(&a.part[((j & 1) * G + q) * NB + c]);
      S[c] = s;
      R[c] = __ldcg(&a.rowj[(j & 1) * NB + c]);
    }
    __syncthreads();

    const double sigma = S[j], alpha = R[j];
    const double xnorm = sqrt(alpha * alpha + sigma);
    const bool skip = (xnorm <= thr) || (sigma == 0.0);
    if (!skip) {
      const double sgn = alpha >= 0.0 ? 1.0 : -1.0;
      const double v1 = alpha + sgn * xnorm;
      const double tau = 2.0 / (1.0 + sigma / (v1 * v1));
      if (threadIdx.x < NB) {
        const int c = threadIdx.x;
        W[c] = (c > j && c < jb) ? tau * (R[c] + S[c] / v1) : 0.0;
        Z[c] = (c < j) ? R[c] + S[c] / v1 : 0.0;
      }
      __syncthreads();
      for (int i = i_lo + threadIdx.x; i < nr; i += LT) {
        const double vi = tile[i + j * ld] / v1;
        for (int c = j + 1; c < jb; ++c) tile[i + c * ld] = fma(-vi, W[c], tile[i + c * ld]);
        tile[i + j * ld] = vi;
      }
      if (g == 0) {
        if (threadIdx.x < NB) {
          const int c = threadIdx.x;
          if (c > j && c < jb) tile[j + c * ld] -= W[c];
          if (c == j) tile[j + j * ld] = -sgn * xnorm;
        }
        if (threadIdx.x < j) {
          const int r = threadIdx.x;
          double s = 0.0;
          for (int l = r; l < j; ++l) s = fma(Ts[r + l * (NB + 1)], Z[l], s);
          Ts[r + j * (NB + 1)] = -tau * s;
        }
        if (threadIdx.x == 0) Ts[j + j * (NB + 1)] = tau;
      }
    } else {
      for (int i = i_lo + threadIdx.x; i < nr; i += LT) tile[i + j * ld] = 0.0;
    }
    __syncthreads();
  }

  for (int idx = threadIdx.x; idx < nr * jb; idx += LT) {
    const int i = idx % nr, c = idx / nr;
    const int gi = r0 + i;
    const double v = tile[i + c * ld];
    a.P[gi + (long)c * a.ldp] = (gi <= c) ? v : 0.0;
    a.Y[gi + (long)c * a.ldy] = (gi < c) ? 0.0 : (gi == c ? 1.0 : v);
  }
  if (g == 0)
    for (int idx = threadIdx.x; idx < jb * jb; idx += LT) {
      const int r = idx % jb, c = idx / jb;
      a.T[r + (long)c * a.ldt] = Ts[r + c * (NB + 1)];
    }
}

inline void leaf_geometry(int rows, int* rc, int* G) {
  int r = (rows + GMAX - 1) / GMAX;
  r = (r + 31) / 32 * 32;
  if (r < RC_MIN) r = RC_MIN;
  *rc = r;
  *G = (rows + r - 1) / r;
}

constexpr size_t LEAF_WS = 2 * GMAX * NB + 2 * NB + 64;
}  // namespace qr

static bool g_leaf_attr = false;

static int leaf_qr(Mat P, Mat Y, Mat T, const double* fro2, double* lws, cudaStream_t st) {
  int rc, G;
  qr::leaf_geometry(P.rows, &rc, &G);
  if (rc > qr::RC_MAX) {
    fprintf(stderr, "libutvb200: panel with %d rows exceeds the leaf QR limit (%d)\n", P.rows,
            qr::RC_MAX * qr::GMAX);
    return -1;
  }
  qr::LeafArgs a;
  a.P = P.p; a.ldp = P.ld;
  a.Y = Y.p; a.ldy = Y.ld;
  a.T = T.p; a.ldt = T.ld;
  a.rows = P.rows; a.jb = P.cols; a.rc = rc;
  a.fro2 = fro2;
  a.part = lws;
  a.rowj = lws + 2 * qr::GMAX * qr::NB;
  a.ctr = (unsigned*)(lws + 2 * qr::GMAX * qr::NB + 2 * qr::NB);
  const size_t smem = qr::leaf_smem_doubles(rc) * sizeof(double);
  if (!g_leaf_attr) {
    UTV_CUDA(cudaFuncSetAttribute(qr::leaf_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(qr::leaf_smem_doubles(qr::RC_MAX) * sizeof(double))));
    g_leaf_attr = true;
  }
  // algorithmic: 4*rows*jb^2 flops (geqr2 + larft), panel read + R/Y write
  ProfScope ps(PROF_PANEL, 4.0 * P.rows * (double)P.cols * P.cols, 8.0 * 3.0 * P.rows * P.cols, st);
  if (G > 1) {
    UTV_CUDA(cudaMemsetAsync(a.ctr, 0, sizeof(unsigned), st));
    void* args[] = {&a};
    UTV_CUDA(cudaLaunchCooperativeKernel((void*)qr::leaf_qr_kernel, dim3(G), dim3(qr::LT), args,
                                         smem, st));
  } else {
    qr::leaf_qr_kernel<<<1, qr::LT, smem, st>>>(a);
    UTV_CUDA(cudaGetLastError());
  }
  return UTV_OK;
}

// ---------------------------------------------------------------------------
// K2: B <- Q^(T) B (side L) or B Q^(T) (side R), Q = I - Y T Y^T.
// ---------------------------------------------------------------------------
size_t larfb_ws_doubles(int brows, int bcols, int w) {
  const long other = brows > bcols ? brows : bcols;
  return 2 * (size_t)w * other + 512 + SPLITK_WS;
}

int larfb(char side, bool trans, Mat Y, Mat T, Mat B, double* ws, size_t ws_doubles,
          cudaStream_t st) {
  const int k = Y.rows, w = Y.cols;
  if (B.rows <= 0 || B.cols <= 0 || w <= 0) return UTV_OK;
  Arena ar{(char*)ws, ws_doubles * sizeof(double), 0};
  if (side == 'L') {
    const int nb = B.cols;
    const long ldw = round_up(w, 4);
    double* W1 = ar.take((size_t)ldw * nb);
    double* W2 = ar.take((size_t)ldw * nb);
    double* gws = ar.take(SPLITK_WS);
    if (!gws) return UTV_ERR_WORKSPACE;
    UTV_CHECK(dgemm(true, false, w, nb, k, 1.0, Y.p, Y.ld, B.p, B.ld, 0.0, W1, ldw, gws, SPLITK_WS, st));
    // op(T) = T^T when applying Q^T from the left (trans), else T.
    UTV_CHECK(dgemm(trans, false, w, nb, w, 1.0, T.p, T.ld, W1, ldw, 0.0, W2, ldw, gws, SPLITK_WS, st));
    UTV_CHECK(dgemm(false, false, k, nb, w, -1.0, Y.p, Y.ld, W2, ldw, 1.0, B.p, B.ld, gws, SPLITK_WS, st));
  } else {
    const int mb = B.rows;
    const long ldw = round_up(mb, 4);
    double* W1 = ar.take((size_t)ldw * w);
    double* W2 = ar.take((size_t)ldw * w);
    double* gws = ar.take(SPLITK_WS);
    if (!gws) return UTV_ERR_WORKSPACE;
    UTV_CHECK(dgemm(false, false, mb, w, k, 1.0, B.p, B.ld, Y.p, Y.ld, 0.0, W1, ldw, gws, SPLITK_WS, st));
    UTV_CHECK(dgemm(false, trans, mb, w, w, 1.0, W1, ldw, T.p, T.ld, 0.0, W2, ldw, gws, SPLITK_WS, st));
    UTV_CHECK(dgemm(false, true, mb, k, w, -1.0, W2, ldw, Y.p, Y.ld, 1.0, B.p, B.ld, gws, SPLITK_WS, st));
  }
  return UTV_OK;
}

int orgqr(Mat Y, Mat T, Mat Q, double* ws, size_t ws_doubles, cudaStream_t st) {
  const int m = Y.rows, w = Y.cols, nc = Q.cols;
  Arena ar{(char*)ws, ws_doubles * sizeof(double), 0};
  const long ldw = round_up(w, 4);
  double* W = ar.take((size_t)ldw * nc);
  double* gws = ar.take(SPLITK_WS);
  if (!gws) return UTV_ERR_WORKSPACE;
  // W = T * Y[:nc, :]^T  (w x nc)
  UTV_CHECK(dgemm(false, true, w, nc, w, 1.0, T.p, T.ld, Y.p, Y.ld, 0.0, W, ldw, gws, SPLITK_WS, st));
  UTV_CHECK(set_identity(Q.p, Q.ld, m, nc, st));
  UTV_CHECK(dgemm(false, false, m, nc, w, -1.0, Y.p, Y.ld, W, ldw, 1.0, Q.p, Q.ld, gws, SPLITK_WS, st));
  return UTV_OK;
}

// ---------------------------------------------------------------------------
// K3/K4: blocked Householder QR.
// ---------------------------------------------------------------------------
size_t geqrf_ws_doubles(int rows, int cols, bool /*want_t*/) {
  // outer level (256-wide panels) + one nested 32-wide level, each with its
  // leaf scratch, merge temporaries and larfb workspace (+ arena rounding).
  const size_t outer = qr::LEAF_WS + 2 * (size_t)round_up(cols, 4) * qr::PANEL +
                       larfb_ws_doubles(rows, cols, qr::PANEL);
  const size_t inner = qr::LEAF_WS + 2 * (size_t)qr::PANEL * qr::NB +
                       larfb_ws_doubles(rows, qr::PANEL, qr::NB);
  return 4096 + sumsq_scratch_doubles() + outer + inner;
}

// T[:j0, j0:j0+jb] = -T[:j0,:j0] (Y[j0:, :j0]^T Y[j0:, j0:j0+jb]) T[j0.., j0..]
static int merge_t(Mat Y, Mat T, int j0, int jb, double* S1, double* S2, double* gws,
                   cudaStream_t st) {
  if (j0 == 0) return UTV_OK;
  const int rows = Y.rows - j0;
  const long lds = round_up(j0, 4);
  UTV_CHECK(dgemm(true, false, j0, jb, rows, 1.0, Y.at(j0, 0), Y.ld, Y.at(j0, j0), Y.ld, 0.0, S1,
                  lds, gws, SPLITK_WS, st));
  UTV_CHECK(dgemm(false, false, j0, jb, j0, 1.0, T.p, T.ld, S1, lds, 0.0, S2, lds, gws, SPLITK_WS, st));
  UTV_CHECK(dgemm(false, false, j0, jb, jb, -1.0, S2, lds, T.at(j0, j0), T.ld, 0.0, T.at(0, j0),
                  T.ld, gws, SPLITK_WS, st));
  return UTV_OK;
}

// Right-looking blocked QR of P with block width `blk`; leaves are 32 wide.
static int geqrf_level(Mat P, Mat Y, Mat T, bool want_t, int blk, const double* fro2,
                       Arena& ar, cudaStream_t st) {
  const int rows = P.rows, cols = P.cols;
  size_t mark = ar.used;
  double* lws = ar.take(qr::LEAF_WS);
  double* S1 = ar.take((size_t)round_up(cols, 4) * blk);
  double* S2 = ar.take((size_t)round_up(cols, 4) * blk);
  const size_t lfb_n = larfb_ws_doubles(rows, cols, blk);
  double* lfb = ar.take(lfb_n);
  if (!lfb) return UTV_ERR_WORKSPACE;
  double* gws = lfb + (lfb_n - SPLITK_WS);
  for (int j0 = 0; j0 < cols; j0 += blk) {
    const int jb = cols - j0 < blk ? cols - j0 : blk;
    Mat Pp = P.sub(j0, j0, rows - j0, jb);
    Mat Yp = Y.sub(j0, j0, rows - j0, jb);
    Mat Tp = T.sub(j0, j0, jb, jb);
    if (j0 > 0) UTV_CHECK(set_zero(Y.at(0, j0), Y.ld, j0, jb, st));
    if (blk == qr::NB) {
      UTV_CHECK(leaf_qr(Pp, Yp, Tp, fro2, lws, st));
    } else {
      UTV_CHECK(geqrf_level(Pp, Yp, Tp, true, qr::NB, fro2, ar, st));
    }
    if (j0 + jb < cols)
      UTV_CHECK(larfb('L', true, Yp, Tp, P.sub(j0, j0 + jb, rows - j0, cols - j0 - jb), lfb, lfb_n, st));
    if (want_t) UTV_CHECK(merge_t(Y, T, j0, jb, S1, S2, gws, st));
  }
  ar.used = mark;
  return UTV_OK;
}

int larfb_panels(char side, bool trans, Mat Y, Mat T, Mat B, double* ws, size_t ws_doubles,
                 cudaStream_t st) {
  const int k = Y.rows, w = Y.cols;
  const int np = (w + qr::PANEL - 1) / qr::PANEL;
  // forward order for B Q and Q^T B, reverse for B Q^T and Q B
  const bool fwd = (side == 'R') != trans;
  for (int jj = 0; jj < np; ++jj) {
    const int j = fwd ? jj : np - 1 - jj;
    const int j0 = j * qr::PANEL, jb = (w - j0 < qr::PANEL) ? w - j0 : qr::PANEL;
    Mat Yj = Y.sub(j0, j0, k - j0, jb), Tj = T.sub(j0, j0, jb, jb);
    if (side == 'R')
      UTV_CHECK(larfb('R', trans, Yj, Tj, B.sub(0, j0, B.rows, k - j0), ws, ws_doubles, st));
    else
      UTV_CHECK(larfb('L', trans, Yj, Tj, B.sub(j0, 0, k - j0, B.cols), ws, ws_doubles, st));
  }
  return UTV_OK;
}

int orgqr_panels(Mat Y, Mat T, Mat Q, double* ws, size_t ws_doubles, cudaStream_t st) {
  const int m = Y.rows, w = Y.cols, nc = Q.cols;
  UTV_CHECK(set_identity(Q.p, Q.ld, m, nc, st));
  const int np = (w + qr::PANEL - 1) / qr::PANEL;
  for (int j = np - 1; j >= 0; --j) {
    const int j0 = j * qr::PANEL, jb = (w - j0 < qr::PANEL) ? w - j0 : qr::PANEL;
    if (j0 >= nc) continue;  // Q_j leaves the leading columns of I untouched
    UTV_CHECK(larfb('L', false, Y.sub(j0, j0, m - j0, jb), T.sub(j0, j0, jb, jb),
                    Q.sub(j0, j0, m - j0, nc - j0), ws, ws_doubles, st));
  }
  return UTV_OK;
}

size_t build_t_ws_doubles(int rows, int cols) {
  return 2 * (size_t)round_up(cols, 4) * qr::PANEL + SPLITK_WS + 1024;
}

int build_t(Mat Y, Mat T, double* ws, size_t ws_doubles, cudaStream_t st) {
  const int cols = Y.cols;
  Arena ar{(char*)ws, ws_doubles * sizeof(double), 0};
  double* S1 = ar.take((size_t)round_up(cols, 4) * qr::PANEL);
  double* S2 = ar.take((size_t)round_up(cols, 4) * qr::PANEL);
  double* gws = ar.take(SPLITK_WS);
  if (!gws) return UTV_ERR_WORKSPACE;
  for (int j0 = qr::PANEL; j0 < cols; j0 += qr::PANEL) {
    const int jb = cols - j0 < qr::PANEL ? cols - j0 : qr::PANEL;
    UTV_CHECK(merge_t(Y, T, j0, jb, S1, S2, gws, st));
  }
  return UTV_OK;
}

int geqrf(Mat P, Mat Y, Mat Tw, bool want_t, double* ws, size_t ws_doubles, cudaStream_t st) {
  if (P.rows < P.cols) return -1;
  Arena ar{(char*)ws, ws_doubles * sizeof(double), 0};
  double* fro2 = ar.take(8);
  double* red = ar.take(sumsq_scratch_doubles());
  if (!red) return UTV_ERR_WORKSPACE;
  UTV_CHECK(sumsq(P.p, P.ld, P.rows, P.cols, fro2, red, st));
  UTV_CHECK(set_zero(Tw.p, Tw.ld, P.cols, P.cols, st));
  const int blk = P.cols > qr::PANEL ? qr::PANEL : qr::NB;
  // want_t == false still delivers complete QR_PANEL-wide diagonal blocks of
  // T (what larfb_panels / orgqr_panels / build_t consume): a single-panel
  // QR therefore always merges its 32-wide leaf triangles.
  return geqrf_level(P, Y, Tw, want_t || blk == qr::NB, blk, fro2, ar, st);
}

}  // namespace utv
