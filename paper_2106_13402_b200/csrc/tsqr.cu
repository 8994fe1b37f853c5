// TSQR + Householder reconstruction, and the row-sharded powerURV driver
// (BASELINE config C4: powerURV q=1 on 524288 x 4096 fp64, rows sharded over
// 1/2/4/8 B200).  The reference algorithm is
// power_urv_from_sample (powerurv.py:41-72), single process; here one
// process per GPU (SPMD), rank i owning the row block A_i (m_i x n, m_i >= n)
// and a replicated G.  Per power round (powerurv.py:63-68):
//
//   Yhat_i = A_i V                    local DMMA GEMM
//   Vhat   = thin Q of Yhat           TSQR: local chunked Householder QRs,
//                                     ALLGATHER of the n x n R factors, a
//                                     redundant QR of the stacked R's (same
//                                     bits on every rank), the explicit Q
//                                     rebuilt down the tree
//   Y      = sum_i A_i^T Vhat_i       local GEMM + ALLREDUCE
//   Vq     = hqr_full(Y)              redundant on every rank (n x n)
//
// Final step (powerurv.py:70-71): Ahat_i = A_i Q(Vq) (Q(Vq) explicit, one
// m_i x n x n product), TSQR of Ahat, then the Householder reconstruction
// (LAPACK dorhr_col; lu.cu): rank 0 factors ONLY the top n x n block,
// Q_0[:n] - S = L11 U', BROADCASTs L11\U' and S, and every rank forms its
// rows of Y = Q U'^{-1} with a triangular solve (rank 0's top rows are L11);
// Twy = -U' S L11^{-T} and R = S R_tsqr are formed redundantly.  With
// tau_j = |pivot_j| + 1 in [1, 2] this is the dlarfg branch hqr_full takes,
// so (Uq, R) equal hqr_full(Ahat)'s up to roundoff.  Vhat's column space is
// all the next hqr_full(Y) needs (Householder vectors are invariant under
// column-sign flips), so the inner thin QRs skip reconstruction.
//
// The same TSQR + reconstruction serves the single-GPU geqrf for panels
// taller than the fused panel kernel's row limit (qr.cu, P = 1).
#include <algorithm>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "utv_internal.h"

namespace utv {

int tsqr_default_cap() { return panel_rows_max(); }

// m rows -> chunks of <= cap rows, each >= n rows (balanced); empty on failure
static std::vector<std::pair<int, int>> row_chunks(int m, int n, int cap) {
  std::vector<std::pair<int, int>> out;
  if (m <= cap) {
    out.emplace_back(0, m);
    return out;
  }
  const int k = (m + cap - 1) / cap;
  const int base = m / k;
  if (base < n) return out;
  int r = 0;
  for (int i = 0; i < k; ++i) {
    const int nr = base + (i < m % k ? 1 : 0);
    out.emplace_back(r, nr);
    r += nr;
  }
  return out;
}

struct TsqrWs {
  int nch;
  long ldm, ldn, ldst, ldg;
  double *Yl, *Tl, *stk, *Ys, *Ts, *F, *snd, *rcv, *gst, *Yg, *Tg, *Ei, *W1, *W2, *qr, *gws;
  size_t qr_n;
};

static size_t plan_tsqr(int m, int n, int P, int cap, TsqrWs* w, double* base) {
  size_t used = 0;
  auto take = [&](size_t nd) -> double* {
    double* p = base ? (double*)((char*)base + used) : nullptr;
    used += round_up((long)(nd * sizeof(double)), 256);
    return p;
  };
  TsqrWs v{};
  v.nch = std::max(1, (int)row_chunks(m, n, cap).size());
  v.ldm = round_up(m, 4);
  v.ldn = round_up(n, 4);
  v.ldst = round_up((long)v.nch * n, 4);
  v.ldg = round_up((long)P * n, 4);
  const size_t nn = (size_t)v.ldn * n;
  v.Yl = take((size_t)v.ldm * n);
  v.Tl = take(nn * v.nch);
  if (v.nch > 1) {
    v.stk = take((size_t)v.ldst * n);
    v.Ys = take((size_t)v.ldst * n);
    v.Ts = take(nn);
    v.F = take((size_t)v.ldst * n);
  }
  if (P > 1) {
    v.snd = take(nn);
    v.rcv = take(nn * P);
    v.gst = take((size_t)v.ldg * n);
    v.Yg = take((size_t)v.ldg * n);
    v.Tg = take(nn);
  }
  v.Ei = take(nn);
  v.W1 = take(nn);
  v.W2 = take(nn);
  const int qr_rows = std::max({std::min(m, cap), v.nch > 1 ? v.nch * n : 0, P > 1 ? P * n : 0});
  v.qr_n = geqrf_ws_doubles(qr_rows, n, true);
  v.qr = take(v.qr_n);
  v.gws = take(SPLITK_WS);
  if (w) *w = v;
  return used / sizeof(double) + 64;
}

size_t tsqr_ws_doubles(int m, int n, int nranks, int cap) {
  return plan_tsqr(m, n, nranks, cap, nullptr, nullptr);
}

// out = Q [top; 0] for Q = I - Y T Y^T (Y: k x n unit lower, T: the dense n x n
// forward triangle, top: n x n).  The zero block below top is never touched:
// W = T (Y1^T top) (a TRMM-shaped product, half the flops), then
// out = [top; 0] - Y W is one k x n x n product.
static int q_times_top(Mat Y, Mat T, Mat top, Mat out, double* W1, double* W2, long ldw,
                       double* gws, cudaStream_t st) {
  const int k = Y.rows, n = Y.cols;
  UTV_CHECK(dgemm(true, false, n, n, n, 1.0, Y.p, Y.ld, top.p, top.ld, 0.0, W1, ldw, gws,
                  SPLITK_WS, st));
  UTV_CHECK(dgemm_ex(false, false, n, n, n, 1.0, T.p, T.ld, W1, ldw, 0.0, W2, ldw, gws, SPLITK_WS,
                     st, true));
  UTV_CHECK(copy_mat(top.p, top.ld, out.p, out.ld, n, n, st));
  UTV_CHECK(dgemm(false, false, n, n, n, -1.0, Y.p, Y.ld, W2, ldw, 1.0, out.p, out.ld, gws,
                  SPLITK_WS, st));
  if (k > n)
    UTV_CHECK(dgemm(false, false, k - n, n, n, -1.0, Y.p + n, Y.ld, W2, ldw, 0.0, out.p + n, out.ld,
                    gws, SPLITK_WS, st));
  return UTV_OK;
}

int tsqr(Comm* comm, Mat X, Mat Q, Mat R, int cap, double* ws, size_t ws_doubles, cudaStream_t st) {
  const int m = X.rows, n = X.cols, P = comm->size;
  if (m < n) return -2;
  const auto chunks = row_chunks(m, n, cap);
  if (chunks.empty()) {
    fprintf(stderr, "libutvb200: cannot split %d rows into chunks of %d..%d rows\n", m, n, cap);
    return -2;
  }
  if (ws_doubles < plan_tsqr(m, n, P, cap, nullptr, nullptr)) return UTV_ERR_WORKSPACE;
  TsqrWs w;
  plan_tsqr(m, n, P, cap, &w, ws);
  const long ldn = w.ldn;
  const size_t nn = (size_t)ldn * n;
  const int nch = (int)chunks.size();
  // ---- leaves: local Householder QRs of the row chunks (X chunk <- R_c) ----
  for (int c = 0; c < nch; ++c) {
    const int r0 = chunks[c].first, nr = chunks[c].second;
    UTV_CHECK(geqrf(X.sub(r0, 0, nr, n), Mat{w.Yl + r0, w.ldm, nr, n}, Mat{w.Tl + c * nn, ldn, n, n},
                    true, w.qr, w.qr_n, st));
  }
  Mat rloc = X.sub(0, 0, n, n);
  if (nch > 1) {
    for (int c = 0; c < nch; ++c)
      UTV_CHECK(copy_mat(X.at(chunks[c].first, 0), X.ld, w.stk + (long)c * n, w.ldst, n, n, st));
    UTV_CHECK(geqrf(Mat{w.stk, w.ldst, nch * n, n}, Mat{w.Ys, w.ldst, nch * n, n},
                    Mat{w.Ts, ldn, n, n}, true, w.qr, w.qr_n, st));
    rloc = Mat{w.stk, w.ldst, n, n};
  }
  // ---- across ranks: allgather the R's, redundant QR of the stack ----
  Mat Ei{w.Ei, ldn, n, n};
  if (P > 1) {
    UTV_CHECK(copy_mat(rloc.p, rloc.ld, w.snd, ldn, n, n, st));
    UTV_CHECK(comm->allgather(w.snd, w.rcv, nn, st));
    for (int p = 0; p < P; ++p)
      UTV_CHECK(copy_mat(w.rcv + p * nn, ldn, w.gst + (long)p * n, w.ldg, n, n, st));
    UTV_CHECK(geqrf(Mat{w.gst, w.ldg, P * n, n}, Mat{w.Yg, w.ldg, P * n, n}, Mat{w.Tg, ldn, n, n},
                    true, w.qr, w.qr_n, st));
    UTV_CHECK(copy_mat(w.gst, w.ldg, R.p, R.ld, n, n, st));
    // E_i = rows [rank n, rank n + n) of Q_g [I; 0] = I_i - Yg_i (Tg Yg1^T)
    UTV_CHECK(dgemm_ex(false, true, n, n, n, 1.0, w.Tg, ldn, w.Yg, w.ldg, 0.0, w.W1, ldn, w.gws,
                       SPLITK_WS, st, true));
    if (comm->rank == 0) UTV_CHECK(set_identity(w.Ei, ldn, n, n, st));
    UTV_CHECK(dgemm(false, false, n, n, n, -1.0, w.Yg + (long)comm->rank * n, w.ldg, w.W1, ldn,
                    comm->rank == 0 ? 1.0 : 0.0, w.Ei, ldn, w.gws, SPLITK_WS, st));
  } else {
    UTV_CHECK(copy_mat(rloc.p, rloc.ld, R.p, R.ld, n, n, st));
    UTV_CHECK(set_identity(w.Ei, ldn, n, n, st));
  }
  // ---- back down the local tree ----
  if (nch > 1) {
    UTV_CHECK(q_times_top(Mat{w.Ys, w.ldst, nch * n, n}, Mat{w.Ts, ldn, n, n}, Ei,
                          Mat{w.F, w.ldst, nch * n, n}, w.W1, w.W2, ldn, w.gws, st));
  }
  for (int c = 0; c < nch; ++c) {
    const int r0 = chunks[c].first, nr = chunks[c].second;
    Mat top = nch > 1 ? Mat{w.F + (long)c * n, w.ldst, n, n} : Ei;
    UTV_CHECK(q_times_top(Mat{w.Yl + r0, w.ldm, nr, n}, Mat{w.Tl + c * nn, ldn, n, n}, top,
                          Q.sub(r0, 0, nr, n), w.W1, w.W2, ldn, w.gws, st));
  }
  return UTV_OK;
}

size_t reconstruct_ws_doubles(int n) {
  return round_up(n, 4) * (size_t)(n + 1) + lu_ws_doubles() + 1024;
}

int householder_reconstruct(Comm* comm, Mat Q, Mat Tw, Mat R, double* ws, size_t ws_doubles,
                            cudaStream_t st) {
  const int m = Q.rows, n = Q.cols;
  if (ws_doubles < reconstruct_ws_doubles(n)) return UTV_ERR_WORKSPACE;
  const long ldn = round_up(n, 4);
  double* buf = ws;                       // [L11\U' | s]: ldn x (n + 1)
  double* s = buf + ldn * n;
  double* luw = buf + round_up(ldn * (n + 1), 32);
  Mat top{buf, ldn, n, n};
  if (comm->rank == 0) {
    if (m < n) return -2;
    UTV_CHECK(copy_mat(Q.p, Q.ld, buf, ldn, n, n, st));
    UTV_CHECK(getrf_signed(top, s, luw, lu_ws_doubles(), st));  // Q0[:n] - S = L11 U'
  }
  UTV_CHECK(comm->broadcast(buf, (size_t)ldn * (n + 1), 0, st));
  // Y_i = Q_i U'^{-1}; on rank 0 the top n rows are L11 (unit lower)
  if (comm->rank == 0) {
    UTV_CHECK(copy_mat(buf, ldn, Q.p, Q.ld, n, n, st));
    UTV_CHECK(laset(1, n, n, 0.0, 1.0, Q.p, Q.ld, st));
    if (m > n) UTV_CHECK(trsm_right_upper(false, false, n, buf, ldn, Q.sub(n, 0, m - n, n), luw,
                                          lu_ws_doubles(), st));
  } else {
    UTV_CHECK(trsm_right_upper(false, false, n, buf, ldn, Q, luw, lu_ws_doubles(), st));
  }
  // Twy = -U' S L11^{-T} (redundant on every rank)
  UTV_CHECK(copy_mat(buf, ldn, Tw.p, Tw.ld, n, n, st));
  UTV_CHECK(laset(4, n, n, 0.0, 0.0, Tw.p, Tw.ld, st));  // keep U' (upper incl. diagonal)
  UTV_CHECK(diag_scale(1, n, n, s, -1.0, Tw.p, Tw.ld, st));
  UTV_CHECK(trsm_right_upper(true, true, n, buf, ldn, Tw, luw, lu_ws_doubles(), st));
  // R = S R_tsqr
  UTV_CHECK(diag_scale(0, n, n, s, 1.0, R.p, R.ld, st));
  return UTV_OK;
}

// ---------------------------------------------------------------------------
// row-sharded powerURV driver
// ---------------------------------------------------------------------------
struct ShWs {
  double *Yh, *V, *Yn, *Rt, *ts, *rc, *qr, *og;
  size_t ts_n, rc_n, qr_n, og_n;
  long ldm, ldn;
};

static size_t plan_sharded(int m, int n, int P, int cap, ShWs* w, double* base) {
  size_t used = 0;
  auto take = [&](size_t nd) -> double* {
    double* p = base ? (double*)((char*)base + used) : nullptr;
    used += round_up((long)(nd * sizeof(double)), 256);
    return p;
  };
  ShWs v{};
  v.ldm = round_up(m, 4);
  v.ldn = round_up(n, 4);
  const size_t nn = (size_t)v.ldn * n;
  v.ts_n = tsqr_ws_doubles(m, n, P, cap);
  v.rc_n = reconstruct_ws_doubles(n);
  v.qr_n = geqrf_ws_doubles(n, n, true);
  v.og_n = nn + SPLITK_WS + 1024;
  v.Yh = take((size_t)v.ldm * n);
  v.V = take(nn);
  v.Yn = take(nn);
  v.Rt = take(nn);
  v.ts = take(v.ts_n);
  v.rc = take(v.rc_n);
  v.qr = take(v.qr_n);
  v.og = take(v.og_n);
  if (w) *w = v;
  return used / sizeof(double) + 64;
}

size_t powerurv_sharded_ws_doubles(int m, int n, int nranks, int cap) {
  return plan_sharded(m, n, nranks, cap <= 0 ? panel_rows_max() : std::min(cap, panel_rows_max()),
                      nullptr, nullptr);
}

// Every rank must call with the same n, q and replicated G; m (this rank's
// rows) >= n.  Ranks agree on the arguments through one tiny allreduce
// before any work (a rank with a bad argument would otherwise leave the
// others blocked in a collective); that is the only host synchronisation.
int powerurv_sharded(Comm* comm, int m, int n, int q, Mat A, Mat G, Mat Uy, Mat Ut, Mat R, Mat Vy,
                     Mat Vt, int cap, double* ws, size_t ws_doubles, cudaStream_t st) {
  cap = cap <= 0 ? panel_rows_max() : std::min(cap, panel_rows_max());
  int local = 0;
  if (n < 1) local = -3;
  else if (m < n) local = -2;
  else if (q < 0) local = -4;
  else if (row_chunks(m, n, cap).empty()) local = -2;
  else if (ws_doubles < plan_sharded(m, n, comm->size, cap, nullptr, nullptr)) local = UTV_ERR_WORKSPACE;
  if (comm->size > 1) {
    double h[4] = {local != 0 ? 1.0 : 0.0, (double)n, (double)q, 1.0}, *d = nullptr;
    UTV_CUDA(cudaMallocAsync((void**)&d, sizeof(h), st));
    UTV_CUDA(cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, st));
    const int rc = comm->allreduce_sum(d, 4, st);
    UTV_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    UTV_CUDA(cudaFreeAsync(d, st));
    UTV_CUDA(cudaStreamSynchronize(st));
    UTV_CHECK(rc);
    if (local) return local;
    const double P = comm->size;
    if (h[0] != 0.0 || h[1] != P * n || h[2] != P * q || h[3] != P) return UTV_ERR_COMM;
  } else if (local) {
    return local;
  }
  ShWs w;
  plan_sharded(m, n, comm->size, cap, &w, ws);
  const long ldn = w.ldn;
  Mat Yh{w.Yh, w.ldm, m, n}, Rt{w.Rt, ldn, n, n}, Yn{w.Yn, ldn, n, n};
  double* gws = w.og + ldn * n;  // the orgqr scratch doubles as GEMM split-K scratch
  if (q == 0) {
    UTV_CHECK(copy_mat(G.p, G.ld, w.Yn, ldn, n, n, st));  // Vq = hqr_full(G) (powerurv.py:58-59)
    UTV_CHECK(geqrf(Yn, Vy, Vt, true, w.qr, w.qr_n, st));
  } else {
    for (int it = 0; it < q; ++it) {  // powerurv.py:63-68
      const double* vp = G.p;
      long ldv = G.ld;
      if (it > 0) {
        UTV_CHECK(orgqr(Vy, Vt, Mat{w.V, ldn, n, n}, w.og, w.og_n, st));
        vp = w.V;
        ldv = ldn;
      }
      UTV_CHECK(dgemm(false, false, m, n, n, 1.0, A.p, A.ld, vp, ldv, 0.0, w.Yh, w.ldm, gws,
                      SPLITK_WS, st));                                        // :64
      UTV_CHECK(tsqr(comm, Yh, Uy, Rt, cap, w.ts, w.ts_n, st));               // :65 (Q into Uy)
      UTV_CHECK(dgemm(true, false, n, n, m, 1.0, A.p, A.ld, Uy.p, Uy.ld, 0.0, w.Yn, ldn, gws,
                      SPLITK_WS, st));                                        // :66 partial
      UTV_CHECK(comm->allreduce_sum(w.Yn, (size_t)ldn * n, st));
      UTV_CHECK(geqrf(Yn, Vy, Vt, true, w.qr, w.qr_n, st));                  // :67
    }
  }
  // :70 A Q(Vq) with Q(Vq) explicit (2n^3) and one m x n x n product
  UTV_CHECK(orgqr(Vy, Vt, Mat{w.V, ldn, n, n}, w.og, w.og_n, st));
  UTV_CHECK(dgemm(false, false, m, n, n, 1.0, A.p, A.ld, w.V, ldn, 0.0, w.Yh, w.ldm, gws, SPLITK_WS,
                  st));
  UTV_CHECK(tsqr(comm, Yh, Uy, Rt, cap, w.ts, w.ts_n, st));                   // :71
  UTV_CHECK(householder_reconstruct(comm, Uy, Ut, Rt, w.rc, w.rc_n, st));
  UTV_CHECK(copy_mat(w.Rt, ldn, R.p, R.ld, n, n, st));
  return UTV_OK;
}

}  // namespace utv
