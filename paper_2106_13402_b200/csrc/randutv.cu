// Device driver for blocked randUTV, basic variant (Algorithm 3 of
// arXiv 2106.13402; reference randutv.py:110-193 with boosted=False).
//
// The whole step loop runs on one CUDA stream without host synchronisation:
// sampling GEMMs (K1), panel QRs (K3), compact-WY updates (K2), the b x b
// Jacobi SVD (K6) and the small rotations (K1).  The Gaussian blocks are the
// exact draws of the reference RNG (randutv.py:189, C order), staged on the
// device by the caller: block i is a b x k_i column-major matrix (the C-order
// k_i x b draw), i.e. G_i^T, at column offset sum_{i'<i} k_i' of G.
#include "common.cuh"
#include "utv_internal.h"

namespace utv {

struct RutvWs {
  double *Y, *Z, *Yv, *Tv, *Yu, *Tu, *sig, *Us, *Vs, *tmp, *red, *gws, *qr, *lfb, *svd;
  long ldy, ldz, ldb, ldtmp;
  size_t qr_n, lfb_n, svd_n;
};

static size_t plan_rutv(int m, int n, int b, RutvWs* w, double* base, size_t avail) {
  Arena ar{(char*)base, avail * sizeof(double), 0};
  const long ldy = round_up(n, 4), ldz = round_up(m, 4), ldb = round_up(b, 4);
  const long mx = m > n ? m : n;
  const long ldtmp = round_up(mx, 4);
  RutvWs v;
  v.ldy = ldy; v.ldz = ldz; v.ldb = ldb; v.ldtmp = ldtmp;
  v.qr_n = geqrf_ws_doubles(m, b, true);
  v.lfb_n = larfb_ws_doubles(m, m, b);
  v.svd_n = gesvj_ws_doubles(b);
  // NOTE: with base == nullptr the arena only measures.
  auto take = [&](size_t nd) -> double* {
    size_t bytes = round_up((long)(nd * sizeof(double)), 256);
    double* p = base ? (double*)(ar.base + ar.used) : nullptr;
    ar.used += bytes;
    return p;
  };
  v.Y = take(ldy * b);
  v.Z = take(ldz * b);
  v.Yv = take(ldy * b);
  v.Tv = take(ldb * b);
  v.Yu = take(ldz * b);
  v.Tu = take(ldb * b);
  v.sig = take(ldb);
  v.Us = take(ldb * b);
  v.Vs = take(ldb * b);
  v.tmp = take(ldtmp * b + (size_t)ldb * mx);
  v.red = take(sumsq_scratch_doubles());
  v.gws = take(SPLITK_WS);
  v.qr = take(v.qr_n);
  v.lfb = take(v.lfb_n);
  v.svd = take(v.svd_n);
  if (w) *w = v;
  return ar.used / sizeof(double) + 64;
}

size_t randutv_ws_doubles(int m, int n, int b) { return plan_rutv(m, n, b, nullptr, nullptr, 0); }

// dst (r x c) <- op(src) * S   or   S^T * src, through tmp, written back in place.
static int rotate_right(Mat X, const double* S, long lds, int b, const RutvWs& w, cudaStream_t st) {
  // X (r x b) <- X * S
  if (X.rows <= 0) return UTV_OK;
  UTV_CHECK(dgemm(false, false, X.rows, b, b, 1.0, X.p, X.ld, S, lds, 0.0, w.tmp, w.ldtmp, w.gws,
                  SPLITK_WS, st));
  return copy_mat(w.tmp, w.ldtmp, X.p, X.ld, X.rows, b, st);
}

static int rotate_left_t(Mat X, const double* S, long lds, int b, const RutvWs& w, cudaStream_t st) {
  // X (b x c) <- S^T * X
  if (X.cols <= 0) return UTV_OK;
  UTV_CHECK(dgemm(true, false, b, X.cols, b, 1.0, S, lds, X.p, X.ld, 0.0, w.tmp, w.ldb, w.gws,
                  SPLITK_WS, st));
  return copy_mat(w.tmp, w.ldb, X.p, X.ld, b, X.cols, st);
}

int randutv_basic(int m, int n, int b, int q, Mat T, Mat U, Mat V, const double* G, long ldg,
                  double* errsq, double* trail2, int* svd_status, double* ws, size_t ws_doubles,
                  cudaStream_t st) {
  if (m < n) return -1;
  if (b < 1) return -3;
  if (q < 0) return -4;
  RutvWs w;
  const size_t need = plan_rutv(m, n, b, nullptr, nullptr, 0);
  if (ws_doubles < need) return UTV_ERR_WORKSPACE;
  plan_rutv(m, n, b, &w, ws, ws_doubles);

  const int nsteps = (n + b - 1) / b;
  long gcol = 0;
  for (int i = 0; i < nsteps; ++i) {
    const int lo = i * b, mid = lo + b;
    const int k = m - lo, kc = n - lo;
    if (kc > b) {
      Mat Bk = T.sub(lo, lo, k, kc);
      // ---- sampling (randutv.py:185-193): Y = B^T G; q x Y = B^T (B Y) ----
      UTV_CHECK(dgemm(true, true, kc, b, k, 1.0, Bk.p, Bk.ld, G + gcol * ldg, ldg, 0.0, w.Y, w.ldy,
                      w.gws, SPLITK_WS, st));
      gcol += k;
      for (int r = 0; r < q; ++r) {
        UTV_CHECK(dgemm(false, false, k, b, kc, 1.0, Bk.p, Bk.ld, w.Y, w.ldy, 0.0, w.Z, w.ldz,
                        w.gws, SPLITK_WS, st));
        UTV_CHECK(dgemm(true, false, kc, b, k, 1.0, Bk.p, Bk.ld, w.Z, w.ldz, 0.0, w.Y, w.ldy,
                        w.gws, SPLITK_WS, st));
      }
      // ---- right transform: [Vq, ~] = hqr_full(Y) (randutv.py:141) ----
      Mat Ym{w.Y, w.ldy, kc, b}, Yv{w.Yv, w.ldy, kc, b}, Tv{w.Tv, w.ldb, b, b};
      UTV_CHECK(geqrf(Ym, Yv, Tv, true, w.qr, w.qr_n, st));
      UTV_CHECK(larfb('R', false, Yv, Tv, T.sub(0, lo, m, kc), w.lfb, w.lfb_n, st));
      UTV_CHECK(larfb('R', false, Yv, Tv, V.sub(0, lo, n, kc), w.lfb, w.lfb_n, st));
      // ---- left transform: [Uq, R] = hqr_full(T[lo:, lo:mid]) (randutv.py:146) ----
      Mat Yu{w.Yu, w.ldz, k, b}, Tu{w.Tu, w.ldb, b, b};
      UTV_CHECK(geqrf(T.sub(lo, lo, k, b), Yu, Tu, true, w.qr, w.qr_n, st));
      UTV_CHECK(larfb('R', false, Yu, Tu, U.sub(0, lo, m, k), w.lfb, w.lfb_n, st));
      UTV_CHECK(larfb('L', true, Yu, Tu, T.sub(lo, mid, k, kc - b), w.lfb, w.lfb_n, st));
      // T[mid:, lo:mid] is already exactly zero (geqrf writes R with zeros below).
      // ---- b x b SVD and rotations (randutv.py:151-156) ----
      Mat Us{w.Us, w.ldb, b, b}, Vs{w.Vs, w.ldb, b, b};
      UTV_CHECK(gesvj(T.sub(lo, lo, b, b), w.sig, Us, Vs, w.svd, w.svd_n, svd_status + i, st));
      UTV_CHECK(rotate_right(U.sub(0, lo, m, b), w.Us, w.ldb, b, w, st));
      UTV_CHECK(rotate_right(V.sub(0, lo, n, b), w.Vs, w.ldb, b, w, st));
      UTV_CHECK(set_diag(T.at(lo, lo), T.ld, b, b, w.sig, st));
      UTV_CHECK(rotate_left_t(T.sub(lo, mid, b, kc - b), w.Us, w.ldb, b, w, st));
      UTV_CHECK(rotate_right(T.sub(0, lo, lo, b), w.Vs, w.ldb, b, w, st));
      // ---- error tracking (randutv.py:159-161) ----
      UTV_CHECK(sumsq(T.at(lo, lo), T.ld, b, kc, errsq + i, w.red, st));
      if (trail2) UTV_CHECK(sumsq(T.at(mid, mid), T.ld, m - mid, kc - b, trail2 + i, w.red, st));
    } else {
      // ---- final narrow block: dense SVD (randutv.py:164-177) ----
      Mat Us{w.Us, w.ldb, kc, kc}, Vs{w.Vs, w.ldb, kc, kc};
      if (k > kc) {
        // tall block: QR first, then the kc x kc SVD of R; the full U of the
        // block is Q * blockdiag(U_small, I).
        Mat Yu{w.Yu, w.ldz, k, kc}, Tu{w.Tu, w.ldb, kc, kc};
        UTV_CHECK(geqrf(T.sub(lo, lo, k, kc), Yu, Tu, true, w.qr, w.qr_n, st));
        UTV_CHECK(larfb('R', false, Yu, Tu, U.sub(0, lo, m, k), w.lfb, w.lfb_n, st));
      }
      UTV_CHECK(gesvj(T.sub(lo, lo, kc, kc), w.sig, Us, Vs, w.svd, w.svd_n, svd_status + i, st));
      UTV_CHECK(rotate_right(U.sub(0, lo, m, kc), w.Us, w.ldb, kc, w, st));
      UTV_CHECK(rotate_right(V.sub(0, lo, n, kc), w.Vs, w.ldb, kc, w, st));
      UTV_CHECK(set_diag(T.at(lo, lo), T.ld, k, kc, w.sig, st));
      UTV_CHECK(rotate_right(T.sub(0, lo, lo, kc), w.Vs, w.ldb, kc, w, st));
      UTV_CHECK(sumsq(T.at(lo, lo), T.ld, k, kc, errsq + i, w.red, st));
      if (trail2) UTV_CUDA(cudaMemsetAsync(trail2 + i, 0, sizeof(double), st));
    }
  }
  return UTV_OK;
}

}  // namespace utv
