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
//  * every <= 256-wide panel is ONE cooperative launch (panel.cu: geqr2,
//    intra-panel updates and larft fused, slab-resident leaves);
//  * panels are combined right-looking with K=256 DMMA GEMM updates;
//    triangles merge as T12 = -T1 (Y1^T Y2) T2.
#include <cstdlib>

#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace qr {
constexpr int PANEL = QR_PANEL;  // outer panel width
}  // namespace qr

// ---------------------------------------------------------------------------
// K2: B <- Q^(T) B (side L) or B Q^(T) (side R), Q = I - Y T Y^T.
// ---------------------------------------------------------------------------
size_t larfb_ws_doubles(int brows, int bcols, int w) {
  // two W buffers of round_up(w, 4) x other (side L) or round_up(rows, 4) x w
  // (side R) doubles: both leading dimensions are padded to 4
  const long other = brows > bcols ? brows : bcols;
  return 2 * (size_t)round_up(w, 4) * round_up(other, 4) + 512 + SPLITK_WS;
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
// side stream scratch of one group factorisation: the intra-group larfb
// (B = rows x QR_PANEL, w = QR_PANEL) and the local T merge temporaries
static size_t side_ws_doubles(int rows) {
  return larfb_ws_doubles(rows, qr::PANEL, qr::PANEL) + 2 * (size_t)qr::PANEL * qr::PANEL + 1024;
}

size_t geqrf_ws_doubles(int rows, int cols, bool /*want_t*/) {
  // taller than the fused panel kernel accepts: TSQR + reconstruction (tsqr.cu)
  if (rows > panel_rows_max())
    return 4096 + tsqr_ws_doubles(rows, cols, 1, panel_rows_max()) +
           (size_t)round_up(cols, 4) * cols + reconstruct_ws_doubles(cols);
  // fused panel QR scratch + merge temporaries + trailing larfb workspace +
  // the look-ahead side stream's private larfb / merge scratch
  return 4096 + sumsq_scratch_doubles() + panel_ws_doubles() +
         2 * (size_t)round_up(cols, 4) * QR_GROUP + larfb_ws_doubles(rows, cols, QR_GROUP) +
         side_ws_doubles(rows);
}

// T[:j0, j0:j0+jb] = -T[:j0,:j0] (Y[j0:, :j0]^T Y[j0:, j0:j0+jb]) T[j0.., j0..]
static int merge_t(Mat Y, Mat T, int j0, int jb, double* S1, double* S2, double* gws,
                   cudaStream_t st) {
  if (j0 == 0) return UTV_OK;
  const int rows = Y.rows - j0;
  const long lds = round_up(j0, 4);
  UTV_CHECK(dgemm(true, false, j0, jb, rows, 1.0, Y.at(j0, 0), Y.ld, Y.at(j0, j0), Y.ld, 0.0, S1,
                  lds, gws, SPLITK_WS, st));
  UTV_CHECK(dgemm_ex(false, false, j0, jb, j0, 1.0, T.p, T.ld, S1, lds, 0.0, S2, lds, gws, SPLITK_WS,
                     st, true));  // T11 upper triangular
  UTV_CHECK(dgemm(false, false, j0, jb, jb, -1.0, S2, lds, T.at(j0, j0), T.ld, 0.0, T.at(0, j0),
                  T.ld, gws, SPLITK_WS, st));
  return UTV_OK;
}

// Update granularity of the blocked QR (QR_PANEL or QR_GROUP columns per
// trailing update; tuning knob UTV_QR_GROUP) and of the panel-blocked
// applies (UTV_APPLY_GROUP).  Both default to QR_PANEL: the K = 512 update
// GEMMs run 7% faster (32 vs 30 TF/s, tools/gemm_ab.py), but the wider
// look-ahead group (two panels + their inner update on 48 SMs) and the
// 512-wide middle products cost more than that in powerURV
// (profiles/r02_ab_groups.txt: 2.997 s at 256/256 vs 3.118 s at 512/512).
static int env_group(const char* name) {
  const char* e = getenv(name);
  const int v = e ? atoi(e) : qr::PANEL;
  return v == QR_GROUP ? QR_GROUP : qr::PANEL;
}
static int qr_group() {
  static const int g = env_group("UTV_QR_GROUP");
  return g;
}
static int apply_group() {
  static const int g = env_group("UTV_APPLY_GROUP");
  return g;
}

// Factor the columns [g0, g0 + gw) (they already hold every earlier
// group's update): QR_PANEL-wide fused panels, each first updated by the
// group's earlier panels (K = QR_PANEL); whenever a panel completes a
// QR_GROUP-aligned pair, the pair's T is merged locally
// (T12 = -T1 (Y1^T Y2) T2), so T's QR_GROUP-wide diagonal blocks are always
// complete whatever the update granularity.  Runs on stream s with a CTA
// budget.
static int factor_group(Mat P, Mat Y, Mat T, int g0, int gw, const double* fro2, double* pws,
                        double* sws, cudaStream_t s, int ctas) {
  const int rows = P.rows;
  const size_t lfb_n = larfb_ws_doubles(rows, qr::PANEL, qr::PANEL);
  double* S1 = sws + lfb_n;
  double* S2 = S1 + (size_t)qr::PANEL * qr::PANEL;
  double* gws = sws + (lfb_n - SPLITK_WS);
  gemm_set_max_ctas(ctas);
  int rc = UTV_OK;
  for (int p0 = g0; p0 < g0 + gw && rc == UTV_OK; p0 += qr::PANEL) {
    const int pw = min(qr::PANEL, g0 + gw - p0);
    if (p0 > 0) rc = set_zero(Y.at(0, p0), Y.ld, p0, pw, s);
    if (rc == UTV_OK && p0 > g0)
      rc = larfb('L', true, Y.sub(g0, g0, rows - g0, p0 - g0), T.sub(g0, g0, p0 - g0, p0 - g0),
                 P.sub(g0, p0, rows - g0, pw), sws, lfb_n, s);
    if (rc == UTV_OK)
      rc = panel_qr(P.sub(p0, p0, rows - p0, pw), Y.sub(p0, p0, rows - p0, pw), T.sub(p0, p0, pw, pw),
                    fro2, pws, s, ctas);
    const int q0 = p0 - qr::PANEL;  // the pair [q0, p0 + pw) is QR_GROUP-aligned
    if (rc == UTV_OK && p0 % QR_GROUP == qr::PANEL && (qr_group() == QR_GROUP || apply_group() == QR_GROUP))
      rc = merge_t(Y.sub(q0, q0, rows - q0, qr::PANEL + pw), T.sub(q0, q0, qr::PANEL + pw, qr::PANEL + pw),
                   qr::PANEL, pw, S1, S2, gws, s);
  }
  gemm_set_max_ctas(0);
  return rc;
}

// Right-looking blocked QR over QR_GROUP-wide groups of QR_PANEL-wide fused
// panels, K = QR_GROUP DMMA trailing updates, optional T merges.
// Look-ahead: the trailing update of group j is split into the next group's
// columns (narrow) and the rest (wide); group j+1 is factored on a
// high-priority side stream (on <= 48 SMs) while the wide update runs on the
// others, taking the latency-bound panels off the critical path.
// grp_ev (optional, one per QR_PANEL columns): recorded on st as soon as the
// columns of that panel are final in P (R) and Y — their panel is factored
// and every earlier group's update has reached them — so the caller can
// consume R / Y column blocks (copy them out, merge T) while the QR runs.
static int geqrf_blocked(Mat P, Mat Y, Mat T, bool want_t, const double* fro2, Arena& ar,
                         cudaStream_t st, const cudaEvent_t* grp_ev, ProgressFn cb, void* cb_ctx,
                         int cb_kind) {
  const int rows = P.rows, cols = P.cols, grp = qr_group();
  double* pws = ar.take(panel_ws_doubles());
  double* S1 = ar.take((size_t)round_up(cols, 4) * grp);
  double* S2 = ar.take((size_t)round_up(cols, 4) * grp);
  double* sws = ar.take(side_ws_doubles(rows));
  const size_t lfb_n = larfb_ws_doubles(rows, cols, grp);
  double* lfb = ar.take(lfb_n);
  if (!lfb) return UTV_ERR_WORKSPACE;
  double* gws = lfb + (lfb_n - SPLITK_WS);
  cudaStream_t sa = nullptr;
  cudaEvent_t ev_narrow = nullptr, ev_panel = nullptr;
  const bool lookahead = cols > grp;
  if (lookahead) {
    UTV_CHECK(aux_stream_for(st, 1, &sa));
    UTV_CHECK(aux_event_for(st, 4, &ev_narrow));
    UTV_CHECK(aux_event_for(st, 5, &ev_panel));
  }
  static const int LA_CTAS = [] {
    const char* e = getenv("UTV_LA_CTAS");  // tuning knob (default 64, profiles/r02_la_sweep.txt)
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : 64;
  }();
  static const int LA_ADAPT = [] {
    const char* e = getenv("UTV_LA_ADAPT");  // tuning knob: wide width below which the group gets all SMs
    return e ? atoi(e) : 0;
  }();
  bool factored = false;  // group g0 already factored (look-ahead) on sa
  for (int g0 = 0; g0 < cols; g0 += grp) {
    const int gw = cols - g0 < grp ? cols - g0 : grp;
    Mat Yg = Y.sub(g0, g0, rows - g0, gw);
    Mat Tg = T.sub(g0, g0, gw, gw);
    if (factored) {
      UTV_CUDA(cudaStreamWaitEvent(st, ev_panel, 0));
    } else {
      UTV_CHECK(factor_group(P, Y, T, g0, gw, fro2, pws, sws, st, 0));
    }
    factored = false;
    if (grp_ev)
      for (int p0 = g0; p0 < g0 + gw; p0 += qr::PANEL) {
        UTV_CUDA(cudaEventRecord(grp_ev[p0 / qr::PANEL], st));
        if (cb) cb(cb_ctx, cb_kind, p0 / qr::PANEL);
      }
    const int g1 = g0 + gw;
    if (g1 < cols) {
      const int gw1 = cols - g1 < grp ? cols - g1 : grp;
      UTV_CHECK(larfb('L', true, Yg, Tg, P.sub(g0, g1, rows - g0, gw1), lfb, lfb_n, st));
      if (g1 + gw1 < cols) {
        // group j+1 on the side stream, the wide update on the main stream
        UTV_CUDA(cudaEventRecord(ev_narrow, st));
        UTV_CUDA(cudaStreamWaitEvent(sa, ev_narrow, 0));
        UTV_CHECK(factor_group(P, Y, T, g1, gw1, fro2, pws, sws, sa,
                               (cols - g1 - gw1) < LA_ADAPT ? 0 : LA_CTAS));
        UTV_CUDA(cudaEventRecord(ev_panel, sa));
        factored = true;
        UTV_CHECK(larfb('L', true, Yg, Tg, P.sub(g0, g1 + gw1, rows - g0, cols - g1 - gw1), lfb,
                        lfb_n, st));
      }
    }
    if (want_t) UTV_CHECK(merge_t(Y, T, g0, gw, S1, S2, gws, st));
  }
  return UTV_OK;
}

int larfb_panels(char side, bool trans, Mat Y, Mat T, Mat B, double* ws, size_t ws_doubles,
                 cudaStream_t st) {
  const int k = Y.rows, w = Y.cols;
  const int np = (w + apply_group() - 1) / apply_group();
  // forward order for B Q and Q^T B, reverse for B Q^T and Q B
  const bool fwd = (side == 'R') != trans;
  for (int jj = 0; jj < np; ++jj) {
    const int j = fwd ? jj : np - 1 - jj;
    const int j0 = j * apply_group(), jb = (w - j0 < apply_group()) ? w - j0 : apply_group();
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
  const int np = (w + apply_group() - 1) / apply_group();
  for (int j = np - 1; j >= 0; --j) {
    const int j0 = j * apply_group(), jb = (w - j0 < apply_group()) ? w - j0 : apply_group();
    if (j0 >= nc) continue;  // Q_j leaves the leading columns of I untouched
    UTV_CHECK(larfb('L', false, Y.sub(j0, j0, m - j0, jb), T.sub(j0, j0, jb, jb),
                    Q.sub(j0, j0, m - j0, nc - j0), ws, ws_doubles, st));
  }
  return UTV_OK;
}

int merge_t_block(Mat Y, Mat T, int j0, int jb, double* ws, size_t ws_doubles, cudaStream_t st) {
  const int cols = Y.cols;
  Arena ar{(char*)ws, ws_doubles * sizeof(double), 0};
  double* S1 = ar.take((size_t)round_up(cols, 4) * qr::PANEL);
  double* S2 = ar.take((size_t)round_up(cols, 4) * qr::PANEL);
  double* gws = ar.take(SPLITK_WS);
  if (!gws) return UTV_ERR_WORKSPACE;
  return merge_t(Y, T, j0, jb, S1, S2, gws, st);
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

// Panels taller than the fused kernel's row limit (148 slabs of <= 512 rows):
// TSQR over row chunks on this GPU, then the Householder reconstruction
// (tsqr.cu) so that Y, the dense forward Tw and R = S R_tsqr are hqr_full's
// (qr.py:71-100) up to roundoff for full-rank input.  The skip rule
// (tau = 0 for an exactly dependent column) is not reproduced on this path.
static int geqrf_tall(Mat P, Mat Y, Mat Tw, double* ws, size_t ws_doubles, cudaStream_t st) {
  static Comm* self = [] {
    Comm* c[1];
    new_local_group(1, c);
    return c[0];
  }();
  const int m = P.rows, n = P.cols;
  const int cap = panel_rows_max();
  const size_t ts_n = tsqr_ws_doubles(m, n, 1, cap);
  Arena ar{(char*)ws, ws_doubles * sizeof(double), 0};
  double* ts = ar.take(ts_n);
  const long ldn = round_up(n, 4);
  double* Rn = ar.take((size_t)ldn * n);
  double* rc = ar.take(reconstruct_ws_doubles(n));
  if (!rc) return UTV_ERR_WORKSPACE;
  UTV_CHECK(tsqr(self, P, Y, Mat{Rn, ldn, n, n}, cap, ts, ts_n, st));  // Q -> Y, P destroyed
  UTV_CHECK(householder_reconstruct(self, Y, Tw, Mat{Rn, ldn, n, n}, rc,
                                    reconstruct_ws_doubles(n), st));
  UTV_CHECK(set_zero(P.p, P.ld, m, n, st));
  return copy_mat(Rn, ldn, P.p, P.ld, n, n, st);
}

int geqrf(Mat P, Mat Y, Mat Tw, bool want_t, double* ws, size_t ws_doubles, cudaStream_t st) {
  return geqrf_ev(P, Y, Tw, want_t, ws, ws_doubles, st, nullptr);
}

int geqrf_ev(Mat P, Mat Y, Mat Tw, bool want_t, double* ws, size_t ws_doubles, cudaStream_t st,
             const cudaEvent_t* grp_ev, ProgressFn cb, void* cb_ctx, int cb_kind) {
  if (P.rows < P.cols) return -1;
  if (P.rows > panel_rows_max()) {
    UTV_CHECK(geqrf_tall(P, Y, Tw, ws, ws_doubles, st));
    if (grp_ev)  // TSQR: every column is final at the end
      for (int p0 = 0; p0 < P.cols; p0 += qr::PANEL) {
        UTV_CUDA(cudaEventRecord(grp_ev[p0 / qr::PANEL], st));
        if (cb) cb(cb_ctx, cb_kind, p0 / qr::PANEL);
      }
    return UTV_OK;
  }
  Arena ar{(char*)ws, ws_doubles * sizeof(double), 0};
  double* fro2 = ar.take(8);
  double* red = ar.take(sumsq_scratch_doubles());
  if (!red) return UTV_ERR_WORKSPACE;
  UTV_CHECK(sumsq(P.p, P.ld, P.rows, P.cols, fro2, red, st));
  UTV_CHECK(set_zero(Tw.p, Tw.ld, P.cols, P.cols, st));
  // want_t == false still delivers complete QR_GROUP-wide diagonal blocks of
  // T (what larfb_panels / orgqr_panels / build_t consume).
  return geqrf_blocked(P, Y, Tw, want_t, fro2, ar, st, grp_ev, cb, cb_ctx, cb_kind);
}

}  // namespace utv
