// Device driver for powerURV (Algorithm 1 of arXiv 2106.13402; reference
// powerurv.py:41-72), one stream, no host synchronisation.
//
//   q == 0: Vq = hqr_full(G)
//   else  : V = G; q x { Yhat = A V; Vhat = thinQ(Yhat); Y = A^T Vhat;
//                        Vq = hqr_full(Y); V = Q(Vq) (skipped after the last
//                        round: the reference's last materialisation is dead,
//                        powerurv.py:68-70) }
//   Ahat = A Q(Vq) via compact WY (powerurv.py:70); (Uq, R) = hqr_full(Ahat).
//
// Only the two returned factors (Uq, Vq) need the dense n x n compact-WY
// triangle of the reference's QFactor; every intermediate QR keeps its
// panel-blocked form (diagonal 256 x 256 blocks of T) and is applied panel
// by panel (larfb_panels).  Vhat and the intermediate V are never
// materialised (see the loop): the executed FLOPs are 4n^3/3 per materialise
// below SURVEY §8d's count (which bench.py keeps as the metric's numerator).
#include "common.cuh"
#include <cstdio>
#include <cstdlib>

#include "utv_internal.h"

namespace utv {

struct PurvWs {
  double *Yh, *Yq, *Tq, *Vh, *Vc, *Yn, *gws, *qr, *lfb, *bt;
  long ldm, ldn;
  size_t qr_n, lfb_n, bt_n;
};

static size_t plan_purv(int m, int n, PurvWs* w, double* base) {
  size_t used = 0;
  auto take = [&](size_t nd) -> double* {
    double* p = base ? (double*)((char*)base + used) : nullptr;
    used += round_up((long)(nd * sizeof(double)), 256);
    return p;
  };
  PurvWs v;
  v.ldm = round_up(m, 4);
  v.ldn = round_up(n, 4);
  v.qr_n = geqrf_ws_doubles(m, n, true);
  v.lfb_n = larfb_ws_doubles(m, n, QR_GROUP);
  v.bt_n = build_t_ws_doubles(m, n);
  v.Yh = take(v.ldm * n);
  v.Yq = take(v.ldm * n);
  v.Tq = take(v.ldn * n);
  v.Vh = take(v.ldm * n);
  v.Vc = take(v.ldn * n);
  v.Yn = take(v.ldn * n);
  v.gws = take(SPLITK_WS);
  v.qr = take(v.qr_n);
  v.lfb = take(v.lfb_n);
  v.bt = take(v.bt_n);
  if (w) *w = v;
  return used / sizeof(double) + 64;
}

size_t powerurv_ws_doubles(int m, int n) { return plan_purv(m, n, nullptr, nullptr); }

// Library-owned per-panel progress events for the final QR when the caller
// passes none (drivers enqueue under the driver lock, so one pool suffices).
static const cudaEvent_t* progress_events(int n) {
  constexpr int MAXG = 256;
  static cudaEvent_t pool[MAXG];
  static int made = 0;
  if (n > MAXG) return nullptr;
  while (made < n) {
    if (cudaEventCreateWithFlags(&pool[made], cudaEventDisableTiming) != cudaSuccess) return nullptr;
    ++made;
  }
  return pool;
}

// vq_ready (optional): recorded once Vq (Y and the dense T) is final, so the
// caller can start copying it out while A Q(Vq) and the final QR run.
// r_ready (optional): recorded once R and Uq.Y are final (before Uq's dense
// triangle is built), so the caller can start copying them out.
// yhat0 (optional, q >= 1): the caller already formed Yhat = A G (e.g. as
// K-chunked products while G was still being drawn on the host); G is then
// not read.
// r_cols / t_cols (optional, ceil(n / QR_PANEL) events each): r_cols[j] is
// recorded once columns [j*256, (j+1)*256) of R and Uq.Y are final (during
// the final QR), t_cols[j] once the same columns of Uq's dense triangle are
// (merged on the low-priority stream while the final QR still runs).
int powerurv(int m, int n, int q, Mat A, Mat G, Mat Uy, Mat Ut, Mat R, Mat Vy, Mat Vt, double* ws,
             size_t ws_doubles, cudaStream_t st, cudaEvent_t vq_ready, const double* yhat0,
             long ldy0, cudaEvent_t r_ready, const cudaEvent_t* r_cols, const cudaEvent_t* t_cols,
             ProgressFn cb, void* cb_ctx) {
  if (m < n) return -1;
  if (q < 0) return -3;
  if (ws_doubles < plan_purv(m, n, nullptr, nullptr)) return UTV_ERR_WORKSPACE;
  PurvWs w;
  plan_purv(m, n, &w, ws);
  // UTV_PHASES=1: per-phase device times on stderr (diagnostics only)
  static const bool phases = getenv("UTV_PHASES") != nullptr;
  cudaEvent_t pev[32];
  const char* pname[32];
  int np = 0;
  auto mark = [&](const char* name) {
    if (!phases || np >= 32) return;
    cudaEventCreate(&pev[np]);
    cudaEventRecord(pev[np], st);
    pname[np++] = name;
  };
  mark("start");
  static const int BT_SIDE = [] {
    const char* e = getenv("UTV_PURV_BT_SIDE");  // tuning knob; 0 = in stream order
    return e ? atoi(e) : 64;
  }();
  cudaStream_t sb = nullptr;
  cudaEvent_t ev_bt0 = nullptr, ev_bt1 = nullptr;
  bool bt_side = false;
  if (q == 0) {
    // Vq = hqr_full(G) (powerurv.py:58-59); G is read-only -> work on a copy
    UTV_CHECK(copy_mat(G.p, G.ld, w.Yn, w.ldn, n, n, st));
    UTV_CHECK(geqrf(Mat{w.Yn, w.ldn, n, n}, Vy, Vt, true, w.qr, w.qr_n, st));
    if (vq_ready) UTV_CUDA(cudaEventRecord(vq_ready, st));
    if (vq_ready && cb) cb(cb_ctx, 0, 0);
  } else {
    // Neither Vhat nor the next round's V is ever formed: with Q the
    // Householder QR of Yhat, Y = A^T Vhat = ((Q^T A)[:n, :])^T, and
    // A V = A Q(Vq) — compact-WY applications to a copy of A cost
    // 4mn^2 - 2n^3 and 2mn^2 flops against 4mn^2 - 2n^3/3 and 2mn^2 + 4n^3/3
    // for materialise-then-multiply (same products, different association).
    for (int it = 0; it < q; ++it) {
      const bool last = (it + 1 == q);
      // Yhat = A V (powerurv.py:64); round 0: V = G
      if (it == 0 && yhat0) {
        UTV_CHECK(copy_mat(yhat0, ldy0, w.Yh, w.ldm, m, n, st));
      } else if (it == 0) {
        UTV_CHECK(dgemm(false, false, m, n, n, 1.0, A.p, A.ld, G.p, G.ld, 0.0, w.Yh, w.ldm, w.gws,
                        SPLITK_WS, st));
      } else {
        UTV_CHECK(copy_mat(A.p, A.ld, w.Yh, w.ldm, m, n, st));
        UTV_CHECK(larfb_panels('R', false, Vy, Vt, Mat{w.Yh, w.ldm, m, n}, w.lfb, w.lfb_n, st));
      }
      mark("A*V");
      // [Q, ~] = hqr_full(Yhat) (powerurv.py:65, thin Q = Q[:, :n])
      Mat Yq{w.Yq, w.ldm, m, n}, Tq{w.Tq, w.ldn, n, n};
      UTV_CHECK(geqrf(Mat{w.Yh, w.ldm, m, n}, Yq, Tq, false, w.qr, w.qr_n, st));
      mark("geqrf(Yhat)");
      // Y = A^T Vhat (powerurv.py:66) = transpose of the first n rows of Q^T A
      UTV_CHECK(copy_mat(A.p, A.ld, w.Vh, w.ldm, m, n, st));
      UTV_CHECK(larfb_panels('L', true, Yq, Tq, Mat{w.Vh, w.ldm, m, n}, w.lfb, w.lfb_n, st));
      UTV_CHECK(transpose(w.Vh, w.ldm, w.Yn, w.ldn, n, n, st));
      mark("A^T*Vhat");
      // Vq = hqr_full(Y) (powerurv.py:67); dense T only for the returned factor
      UTV_CHECK(geqrf(Mat{w.Yn, w.ldn, n, n}, Vy, Vt, false, w.qr, w.qr_n, st));
      mark("geqrf(Y)");
      (void)last;
    }
    // Vq's dense triangle is only returned: its off-diagonal blocks are built
    // on a low-priority side stream (CTA budget) while A Q(Vq) — which reads
    // only the diagonal blocks — and the final QR run; it fills the SMs the
    // QR's latency-bound panels leave idle.
    if (BT_SIDE > 0) {
      UTV_CHECK(aux_stream_low(&sb));
      UTV_CHECK(aux_event(6, &ev_bt0));
      UTV_CHECK(aux_event(7, &ev_bt1));
      UTV_CUDA(cudaEventRecord(ev_bt0, st));
      UTV_CUDA(cudaStreamWaitEvent(sb, ev_bt0, 0));
      gemm_set_max_ctas(BT_SIDE);
      const int rc = build_t(Vy, Vt, w.bt, w.bt_n, sb);
      gemm_set_max_ctas(0);
      UTV_CHECK(rc);
      UTV_CUDA(cudaEventRecord(ev_bt1, sb));
      if (vq_ready) UTV_CUDA(cudaEventRecord(vq_ready, sb));
      if (vq_ready && cb) cb(cb_ctx, 0, 0);
      bt_side = true;
    } else {
      UTV_CHECK(build_t(Vy, Vt, w.bt, w.bt_n, st));
      if (vq_ready) UTV_CUDA(cudaEventRecord(vq_ready, st));
      if (vq_ready && cb) cb(cb_ctx, 0, 0);
    }
    mark("build_t(V)");
  }
  // Ahat = A Q(Vq) (powerurv.py:70), formed in R's storage, panel by panel
  UTV_CHECK(copy_mat(A.p, A.ld, R.p, R.ld, m, n, st));
  UTV_CHECK(larfb_panels('R', false, Vy, Vt, R, w.lfb, w.lfb_n, st));
  mark("A*Q(V)");
  // (Uq, R) = hqr_full(Ahat) (powerurv.py:71).  Uq's dense triangle: each
  // off-diagonal column block T[:j0, j0:j0+256] needs only Y's columns
  // < j0 + 256, so the merges run on the low-priority side stream as the
  // final QR's panels complete (per-panel events) instead of after it, and
  // column blocks of R, Uq.Y and Uq.Twy become final (copyable) progressively.
  // Progressive merges on the side stream measured slower (they compete
  // with the final QR's critical path: powerURV 2.94 -> 3.01 s at n=16384),
  // so by default the triangle is built after the QR (tuning knob
  // UTV_PURV_PROG_T=1 enables them); the per-panel r_cols events still let
  // R and Uq.Y stream out during the QR.
  static const bool prog_t = [] {
    const char* e = getenv("UTV_PURV_PROG_T");
    return e ? atoi(e) != 0 : false;
  }();
  const int ngrp = (n + QR_PANEL - 1) / QR_PANEL;
  const cudaEvent_t* evr = r_cols;
  if (prog_t && bt_side && !evr) evr = progress_events(ngrp);
  if (prog_t && bt_side && evr) {
    UTV_CHECK(geqrf_ev(R, Uy, Ut, false, w.qr, w.qr_n, st, evr, r_cols ? cb : nullptr, cb_ctx, 1));
    mark("geqrf(Ahat)");
    if (r_ready) UTV_CUDA(cudaEventRecord(r_ready, st));
    gemm_set_max_ctas(BT_SIDE);
    int rc = UTV_OK;
    for (int g = 0; g < ngrp && rc == UTV_OK; ++g) {
      const int j0 = g * QR_PANEL, jb = min(QR_PANEL, n - j0);
      if (cudaStreamWaitEvent(sb, evr[g], 0) != cudaSuccess) rc = UTV_ERR_CUDA;
      if (rc == UTV_OK && j0 > 0) rc = merge_t_block(Uy, Ut, j0, jb, w.bt, w.bt_n, sb);
      if (rc == UTV_OK && t_cols && cudaEventRecord(t_cols[g], sb) != cudaSuccess) rc = UTV_ERR_CUDA;
      if (rc == UTV_OK && t_cols && cb) cb(cb_ctx, 2, g);
    }
    gemm_set_max_ctas(0);
    UTV_CHECK(rc);
    UTV_CUDA(cudaEventRecord(ev_bt1, sb));
    UTV_CUDA(cudaStreamWaitEvent(st, ev_bt1, 0));  // the call completes on st
    mark("build_t(U) side");
  } else {
    UTV_CHECK(geqrf_ev(R, Uy, Ut, false, w.qr, w.qr_n, st, r_cols, cb, cb_ctx, 1));
    mark("geqrf(Ahat)");
    if (r_ready) UTV_CUDA(cudaEventRecord(r_ready, st));  // R and Uq.Y are final; Uq.Twy follows
    if (bt_side) UTV_CUDA(cudaStreamWaitEvent(st, ev_bt1, 0));  // w.bt reused below
    if (t_cols) {
      // build_t's merges one column block at a time (the same kernels, in
      // the same order), each block's event recorded as soon as it is final:
      // the cheap early blocks leave the GPU while the later merges run
      for (int g = 0; g < ngrp; ++g) {
        const int j0 = g * QR_PANEL, jb = min(QR_PANEL, n - j0);
        if (j0 > 0) UTV_CHECK(merge_t_block(Uy, Ut, j0, jb, w.bt, w.bt_n, st));
        UTV_CUDA(cudaEventRecord(t_cols[g], st));
        if (cb) cb(cb_ctx, 2, g);
      }
    } else {
      UTV_CHECK(build_t(Uy, Ut, w.bt, w.bt_n, st));
    }
    mark("build_t(U)");
  }
  if (phases) {
    cudaEventSynchronize(pev[np - 1]);
    for (int i = 1; i < np; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, pev[i - 1], pev[i]);
      fprintf(stderr, "[powerurv phase] %-14s %9.3f ms\n", pname[i], ms);
    }
    for (int i = 0; i < np; ++i) cudaEventDestroy(pev[i]);
  }
  return UTV_OK;
}

}  // namespace utv
