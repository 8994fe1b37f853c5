// Device driver for blocked randUTV (arXiv 2106.13402): the basic variant
// (Algorithm 3; reference randutv.py:110-193 with boosted=False) and the
// boosted / partial variants (Algorithm 2; randutv.py:130-139, 196-264).
//
// Each step runs on one CUDA stream without host synchronisation: sampling
// GEMMs (K1), panel QRs (K3), compact-WY updates (K2), the b x b Jacobi SVD
// (K6) and the small rotations (K1).  The Gaussian blocks are the exact
// draws of the reference RNG (C order), staged on the device by the caller:
// a C-order k x w draw is a w x k column-major matrix, i.e. G^T.
//
// randutv_basic() loops over all steps in one call; randutv_step() runs one
// step (the host loop of the boosted/partial variants, which may stop early
// on the tracked error, randutv.py:123-124).  The boosted sampler's carried
// columns (w_next, randutv.py:135-138) live in the caller's workspace
// between steps.
#include <mutex>

#include "common.cuh"
#include <cstdlib>

#include "utv_internal.h"

namespace utv {

struct RutvWs {
  double *Y, *Z, *X, *Bs, *W, *Yv, *Tv, *Yu, *Tu, *Yy, *Ty, *Cs, *sig, *Us, *Vs, *tmp, *red, *gws,
      *qr, *lfb, *svd, *wn;
  double *Yv2, *Tv2, *lfb2;  // basic pipelined loop: second-parity Q_v, side-stream larfb scratch
  long ldn, ldm, ldb, ldtmp;
  size_t qr_n, lfb_n, svd_n;
  int* meta;  // [0] = carried columns in wn (boosted)
};

// p < 0: basic variant (no boosted buffers); p >= 0: boosted with p oversampling.
static size_t plan_rutv(int m, int n, int b, int p_in, RutvWs* w, double* base) {
  const bool bst = p_in >= 0;
  const int p = bst ? p_in : 0;
  size_t used = 0;
  auto take = [&](size_t nd) -> double* {
    double* ptr = base ? (double*)((char*)base + used) : nullptr;
    used += round_up((long)(nd * sizeof(double)), 256);
    return ptr;
  };
  const int wd = b + p;  // widest sample
  const long ldn = round_up(n, 4), ldm = round_up(m, 4), ldb = round_up(wd, 4);
  const long mx = m > n ? m : n;
  RutvWs v;
  v.ldn = ldn; v.ldm = ldm; v.ldb = ldb;
  v.ldtmp = round_up(mx, 4);
  v.qr_n = geqrf_ws_doubles((int)mx, wd, true);
  v.lfb_n = larfb_ws_doubles(m, m, wd);
  v.svd_n = gesvj_ws_doubles(wd);
  v.Y = take(ldn * wd);
  v.Z = take(ldm * wd);
  v.X = bst ? take(ldm * wd) : nullptr;
  v.Bs = bst ? take(ldm * wd) : nullptr;
  v.W = bst ? take(ldn * wd) : nullptr;
  v.Yy = bst ? take(ldm * wd) : nullptr;
  v.Ty = bst ? take(ldb * wd) : nullptr;
  v.Cs = bst ? take(ldm * wd) : nullptr;
  v.wn = bst ? take(ldm * wd) : nullptr;
  v.Yv = take(ldn * wd);
  v.Tv = take(ldb * wd);
  v.Yu = take(ldm * wd);
  v.Tu = take(ldb * wd);
  v.sig = take(ldb);
  v.Us = take(ldb * wd);
  v.Vs = take(ldb * wd);
  v.tmp = take(v.ldtmp * wd + (size_t)ldb * mx);
  v.red = take(sumsq_scratch_doubles());
  v.gws = take(SPLITK_WS);
  v.qr = take(v.qr_n);
  v.lfb = take(v.lfb_n);
  v.svd = take(v.svd_n);
  v.meta = (int*)take(8);
  v.Yv2 = bst ? nullptr : take(ldn * wd);
  v.Tv2 = bst ? nullptr : take(ldb * wd);
  v.lfb2 = bst ? nullptr : take(v.lfb_n);
  if (w) *w = v;
  return used / sizeof(double) + 64;
}

size_t randutv_ws_doubles(int m, int n, int b) { return plan_rutv(m, n, b, -1, nullptr, nullptr); }
size_t randutv_ws_doubles_p(int m, int n, int b, int p) { return plan_rutv(m, n, b, p, nullptr, nullptr); }

// X (r x c) <- X * S  (through tmp)
static int rotate_right(Mat X, const double* S, long lds, int c, const RutvWs& w, cudaStream_t st) {
  if (X.rows <= 0) return UTV_OK;
  UTV_CHECK(dgemm(false, false, X.rows, c, c, 1.0, X.p, X.ld, S, lds, 0.0, w.tmp, w.ldtmp, w.gws,
                  SPLITK_WS, st));
  return copy_mat(w.tmp, w.ldtmp, X.p, X.ld, X.rows, c, st);
}

// X (c x cols) <- S^T * X
static int rotate_left_t(Mat X, const double* S, long lds, int c, const RutvWs& w, cudaStream_t st) {
  if (X.cols <= 0) return UTV_OK;
  UTV_CHECK(dgemm(true, false, c, X.cols, c, 1.0, S, lds, X.p, X.ld, 0.0, w.tmp, w.ldb, w.gws,
                  SPLITK_WS, st));
  return copy_mat(w.tmp, w.ldb, X.p, X.ld, c, X.cols, st);
}

// Basic sampler (randutv.py:185-193): Y (kc x b) = B^T G, q x Y = B^T (B Y).
static int sample_basic(Mat Bk, int b, int q, const double* G, long ldg, const RutvWs& w,
                        cudaStream_t st) {
  const int k = Bk.rows, kc = Bk.cols;
  UTV_CHECK(dgemm(true, true, kc, b, k, 1.0, Bk.p, Bk.ld, G, ldg, 0.0, w.Y, w.ldn, w.gws, SPLITK_WS, st));
  for (int r = 0; r < q; ++r) {
    UTV_CHECK(dgemm(false, false, k, b, kc, 1.0, Bk.p, Bk.ld, w.Y, w.ldn, 0.0, w.Z, w.ldm, w.gws,
                    SPLITK_WS, st));
    UTV_CHECK(dgemm(true, false, kc, b, k, 1.0, Bk.p, Bk.ld, w.Z, w.ldm, 0.0, w.Y, w.ldn, w.gws,
                    SPLITK_WS, st));
  }
  return UTV_OK;
}

// Boosted sampler (randutv.py:196-225) + basis selection by
// svd_tall_thin_left (svd.py:61-82) and the carried columns (:135-138).
// On exit Yv/Tv hold hqr_full(W[:, :b]) and wn/meta[0] the next carried block.
static int boosted_right_basis(int i, Mat Bk, int b, int p, int q, const double* G, long ldg,
                               int pc, int ncols, const RutvWs& w, cudaStream_t st) {
  const int k = Bk.rows, kc = Bk.cols;
  int wcols;
  if (i == 0) {
    // step 1: all b + p columns powered (G is (b+p) x m)
    wcols = b + p;
    UTV_CHECK(dgemm(true, true, kc, wcols, k, 1.0, Bk.p, Bk.ld, G, ldg, 0.0, w.Y, w.ldn, w.gws, SPLITK_WS, st));
    for (int r = 0; r < q; ++r) {
      UTV_CHECK(dgemm(false, false, k, wcols, kc, 1.0, Bk.p, Bk.ld, w.Y, w.ldn, 0.0, w.Z, w.ldm, w.gws, SPLITK_WS, st));
      UTV_CHECK(dgemm(true, false, kc, wcols, k, 1.0, Bk.p, Bk.ld, w.Z, w.ldm, 0.0, w.Y, w.ldn, w.gws, SPLITK_WS, st));
    }
  } else {
    // fresh b columns, q-1 full rounds, then x = B y
    UTV_CHECK(dgemm(true, true, kc, b, k, 1.0, Bk.p, Bk.ld, G, ldg, 0.0, w.Y, w.ldn, w.gws, SPLITK_WS, st));
    for (int r = 0; r < q - 1; ++r) {
      UTV_CHECK(dgemm(false, false, k, b, kc, 1.0, Bk.p, Bk.ld, w.Y, w.ldn, 0.0, w.Z, w.ldm, w.gws, SPLITK_WS, st));
      UTV_CHECK(dgemm(true, false, kc, b, k, 1.0, Bk.p, Bk.ld, w.Z, w.ldm, 0.0, w.Y, w.ldn, w.gws, SPLITK_WS, st));
    }
    UTV_CHECK(dgemm(false, false, k, b, kc, 1.0, Bk.p, Bk.ld, w.Y, w.ldn, 0.0, w.X, w.ldm, w.gws, SPLITK_WS, st));
    // project off the carried subspace: x -= w (w^T x), w = [w_next; 0] (k x pc)
    if (pc > 0) {
      UTV_CHECK(dgemm(true, false, pc, b, k, 1.0, w.wn, w.ldm, w.X, w.ldm, 0.0, w.Z, w.ldb, w.gws, SPLITK_WS, st));
      UTV_CHECK(dgemm(false, false, k, b, pc, -1.0, w.wn, w.ldm, w.Z, w.ldb, 1.0, w.X, w.ldm, w.gws, SPLITK_WS, st));
    }
    // basis = [thin Q of x | w]  (hqr_full(x) -> materialize_q(qx, b))
    UTV_CHECK(geqrf(Mat{w.X, w.ldm, k, b}, Mat{w.Yy, w.ldm, k, b}, Mat{w.Ty, w.ldb, b, b}, true,
                    w.qr, w.qr_n, st));
    UTV_CHECK(orgqr(Mat{w.Yy, w.ldm, k, b}, Mat{w.Ty, w.ldb, b, b}, Mat{w.Bs, w.ldm, k, b}, w.lfb,
                    w.lfb_n, st));
    if (pc > 0) UTV_CHECK(copy_mat(w.wn, w.ldm, w.Bs + (long)b * w.ldm, w.ldm, k, pc, st));
    wcols = b + pc;
    UTV_CHECK(dgemm(true, false, kc, wcols, k, 1.0, Bk.p, Bk.ld, w.Bs, w.ldm, 0.0, w.Y, w.ldn, w.gws, SPLITK_WS, st));
  }
  // svd_tall_thin_left(y): [Qy, R] = hqr_full(y); W = Qy blockdiag(Uhat, I)
  // (only the first b + p columns are used, randutv.py:133-136)
  const int wl = b + p;
  UTV_CHECK(geqrf(Mat{w.Y, w.ldn, kc, wcols}, Mat{w.Yy, w.ldm, kc, wcols}, Mat{w.Ty, w.ldb, wcols, wcols},
                  true, w.qr, w.qr_n, st));
  UTV_CHECK(gesvj(Mat{w.Y, w.ldn, wcols, wcols}, w.sig, Mat{w.Us, w.ldb, wcols, wcols},
                  Mat{w.Vs, w.ldb, wcols, wcols}, w.svd, w.svd_n, w.meta + 2, st));
  const int wlc = wl < kc ? wl : kc;
  UTV_CHECK(set_zero(w.Cs, w.ldm, kc, wlc, st));
  UTV_CHECK(copy_mat(w.Us, w.ldb, w.Cs, w.ldm, wcols, wcols < wlc ? wcols : wlc, st));
  if (wlc > wcols) UTV_CHECK(set_identity(w.Cs + wcols + (long)wcols * w.ldm, w.ldm, kc - wcols, wlc - wcols, st));
  UTV_CHECK(larfb_panels('L', false, Mat{w.Yy, w.ldm, kc, wcols}, Mat{w.Ty, w.ldb, wcols, wcols},
                         Mat{w.Cs, w.ldm, kc, wlc}, w.lfb, w.lfb_n, st));
  // vq = hqr_full(W[:, :b]) (randutv.py:134)
  UTV_CHECK(copy_mat(w.Cs, w.ldm, w.W, w.ldn, kc, b, st));
  Mat Yv{w.Yv, w.ldn, kc, b}, Tv{w.Tv, w.ldb, b, b};
  UTV_CHECK(geqrf(Mat{w.W, w.ldn, kc, b}, Yv, Tv, true, w.qr, w.qr_n, st));
  return UTV_OK;
}

// ---- phases of a regular step (lo = i b, k = m - lo, kc = n - lo) ----
// front_b: right transform (randutv.py:143-144) and the T-panel QR (:146).
static int front_b(int lo, Mat T, Mat U, Mat V, Mat Yv, Mat Tv, int k, int kc, int b,
                   const RutvWs& w, cudaStream_t st) {
  const int m = T.rows, n = V.rows;
  UTV_CHECK(larfb('R', false, Yv, Tv, T.sub(0, lo, m, kc), w.lfb, w.lfb_n, st));
  UTV_CHECK(larfb('R', false, Yv, Tv, V.sub(0, lo, n, kc), w.lfb, w.lfb_n, st));
  Mat Yu{w.Yu, w.ldm, k, b}, Tu{w.Tu, w.ldb, b, b};
  return geqrf(T.sub(lo, lo, k, b), Yu, Tu, true, w.qr, w.qr_n, st);
}
// front_c: left transform (randutv.py:147-149); T[mid:, lo:mid] is already
// exactly zero (geqrf writes R with zeros below).
static int front_c(int lo, Mat T, Mat U, int k, int kc, int b, const RutvWs& w, cudaStream_t st) {
  const int m = T.rows, mid = lo + b;
  Mat Yu{w.Yu, w.ldm, k, b}, Tu{w.Tu, w.ldb, b, b};
  UTV_CHECK(larfb('R', false, Yu, Tu, U.sub(0, lo, m, k), w.lfb, w.lfb_n, st));
  return larfb('L', true, Yu, Tu, T.sub(lo, mid, k, kc - b), w.lfb, w.lfb_n, st);
}
// step_svd: b x b SVD of R = T[lo:mid, lo:mid] (randutv.py:151).
static int step_svd(int lo, Mat T, int b, int* status, const RutvWs& w, cudaStream_t st) {
  return gesvj(T.sub(lo, lo, b, b), w.sig, Mat{w.Us, w.ldb, b, b}, Mat{w.Vs, w.ldb, b, b}, w.svd,
               w.svd_n, status, st);
}
// step_back: rotations, diag(sigma), error tracking (randutv.py:152-161).
static int step_back(int i, int lo, Mat T, Mat U, Mat V, int m, int n, int kc, int b, double* errsq,
                     double* trail2, const RutvWs& w, cudaStream_t st) {
  const int mid = lo + b;
  UTV_CHECK(rotate_right(U.sub(0, lo, m, b), w.Us, w.ldb, b, w, st));
  UTV_CHECK(rotate_right(V.sub(0, lo, n, b), w.Vs, w.ldb, b, w, st));
  UTV_CHECK(set_diag(T.at(lo, lo), T.ld, b, b, w.sig, st));
  UTV_CHECK(rotate_left_t(T.sub(lo, mid, b, kc - b), w.Us, w.ldb, b, w, st));
  UTV_CHECK(rotate_right(T.sub(0, lo, lo, b), w.Vs, w.ldb, b, w, st));
  UTV_CHECK(sumsq(T.at(lo, lo), T.ld, b, kc, errsq + i, w.red, st));
  if (trail2) UTV_CHECK(sumsq(T.at(mid, mid), T.ld, m - mid, kc - b, trail2 + i, w.red, st));
  return UTV_OK;
}

// One step i (0-based) of randUTV.  G: this step's Gaussian block (transposed
// C-order draw).  p = 0 and boosted = false is the basic variant.  *is_final
// is set when the step was the final dense-SVD step; *carried (host) is the
// boosted sampler's carried column count, updated for the next step.
int randutv_step(int i, int m, int n, int b, int p, int q, bool boosted, Mat T, Mat U, Mat V,
                 const double* G, long ldg, double* errsq, double* trail2, int* svd_status,
                 double* ws, size_t ws_doubles, int* carried, int* is_final, cudaStream_t st) {
  *is_final = 0;
  RutvWs w;
  if (ws_doubles < plan_rutv(m, n, b, boosted ? p : -1, nullptr, nullptr)) return UTV_ERR_WORKSPACE;
  plan_rutv(m, n, b, boosted ? p : -1, &w, ws);
  const int lo = i * b, mid = lo + b;
  const int k = m - lo, kc = n - lo;
  if (kc > b + (boosted ? p : 0)) {
    Mat Bk = T.sub(lo, lo, k, kc);
    Mat Yv{w.Yv, w.ldn, kc, b}, Tv{w.Tv, w.ldb, b, b};
    if (boosted) {
      UTV_CHECK(boosted_right_basis(i, Bk, b, p, q, G, ldg, *carried, kc, w, st));
      // carried block for the next step (randutv.py:135-138)
      if (p > 0 && (kc - b) > b + p) {
        // (Q_v^T W[:, b:b+p])[b:, :] -> wn (rows kc-b = next step's kc; padded later)
        UTV_CHECK(larfb('L', true, Yv, Tv, Mat{w.Cs + (long)b * w.ldm, w.ldm, kc, p}, w.lfb,
                        w.lfb_n, st));
        UTV_CHECK(set_zero(w.wn, w.ldm, m - mid, p, st));
        UTV_CHECK(copy_mat(w.Cs + b + (long)b * w.ldm, w.ldm, w.wn, w.ldm, kc - b, p, st));
        *carried = p;
      } else {
        *carried = 0;
      }
    } else {
      // ---- sampling (randutv.py:185-193) + [Vq, ~] = hqr_full(Y) (:141) ----
      UTV_CHECK(sample_basic(Bk, b, q, G, ldg, w, st));
      UTV_CHECK(geqrf(Mat{w.Y, w.ldn, kc, b}, Yv, Tv, true, w.qr, w.qr_n, st));
    }
    UTV_CHECK(front_b(lo, T, U, V, Yv, Tv, k, kc, b, w, st));
    UTV_CHECK(front_c(lo, T, U, k, kc, b, w, st));
    UTV_CHECK(step_svd(lo, T, b, svd_status + i, w, st));
    UTV_CHECK(step_back(i, lo, T, U, V, m, n, kc, b, errsq, trail2, w, st));
    return UTV_OK;
  }
  *is_final = 1;
  // ---- final narrow block: dense SVD (randutv.py:164-177) ----
  Mat Us{w.Us, w.ldb, kc, kc}, Vs{w.Vs, w.ldb, kc, kc};
  if (k > kc) {
    // tall block: QR first, then the kc x kc SVD of R; the full U of the
    // block is Q * blockdiag(U_small, I).
    Mat Yu{w.Yu, w.ldm, k, kc}, Tu{w.Tu, w.ldb, kc, kc};
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
  return UTV_OK;
}

// Side stream for the latency-bound b x b Jacobi SVD (created once, high
// priority so its few CTAs are dispatched ahead of the GEMM tiles).
static int side_stream(cudaStream_t* s1, cudaEvent_t* ev, cudaStream_t* s2 = nullptr) {
  static cudaStream_t g_s1 = nullptr, g_s2 = nullptr;
  static cudaEvent_t g_ev[5];
  static std::once_flag once;
  static int err = 0;
  std::call_once(once, [] {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&g_s1, cudaStreamNonBlocking, hi) != cudaSuccess) err = 1;
    if (cudaStreamCreateWithPriority(&g_s2, cudaStreamNonBlocking, lo) != cudaSuccess) err = 1;
    for (int e = 0; e < 5; ++e)
      if (cudaEventCreateWithFlags(&g_ev[e], cudaEventDisableTiming) != cudaSuccess) err = 1;
  });
  if (err) return UTV_ERR_CUDA;
  *s1 = g_s1;
  if (s2) *s2 = g_s2;
  for (int e = 0; e < (s2 ? 5 : 2); ++e) ev[e] = g_ev[e];
  return UTV_OK;
}

// Whole basic loop, software-pipelined over two streams: the Jacobi SVD of
// step i runs on the side stream while the main stream proceeds with the
// left transform of step i and the sampling + Y-panel QR of step i+1; the
// rotations of step i follow on the main stream just before step i+1's
// right transform (the first operation that touches rows lo:mid of T
// again).  Data dependencies are unchanged, so results are bitwise the same
// as the one-stream step sequence.
int randutv_basic_range(int i0, int i1, int m, int n, int b, int q, Mat T, Mat U, Mat V,
                        const double* G, long ldg, double* errsq, double* trail2, int* svd_status,
                        double* ws, size_t ws_doubles, cudaStream_t st, int carry);

int randutv_basic(int m, int n, int b, int q, Mat T, Mat U, Mat V, const double* G, long ldg,
                  double* errsq, double* trail2, int* svd_status, double* ws, size_t ws_doubles,
                  cudaStream_t st) {
  return randutv_basic_range(0, (n + b - 1) / b, m, n, b, q, T, U, V, G, ldg, errsq, trail2,
                             svd_status, ws, ws_doubles, st, 0);
}

// Steps [i0, i1) of the basic loop (G = the block of step i0 at column 0).
// Lets the host draw the next steps' Gaussian blocks while these run.
// carry bit 0: the previous range left step i0-1's SVD in flight (its
// rotations are applied here, where the one-call loop would); bit 1: leave
// step i1-1's SVD in flight for the next range.  Without the carry, every
// range boundary drains the SVD pipeline (~3-5 ms per boundary).
int randutv_basic_range(int i0, int i1, int m, int n, int b, int q, Mat T, Mat U, Mat V,
                        const double* G, long ldg, double* errsq, double* trail2, int* svd_status,
                        double* ws, size_t ws_doubles, cudaStream_t st, int carry) {
  if (m < n) return -1;
  if (b < 1) return -3;
  if (q < 0) return -4;
  if (ws_doubles < plan_rutv(m, n, b, -1, nullptr, nullptr)) return UTV_ERR_WORKSPACE;
  RutvWs w;
  plan_rutv(m, n, b, -1, &w, ws);
  // Streams: st = critical path (sampling, T transforms, panel QRs, rotations);
  // s1 (high priority) = the b x b Jacobi SVD of step i; s2 = the U and V
  // right transforms, which only the next rotations read: they fill the SMs
  // the latency-bound panel QRs leave idle (panels get PBUD CTAs, s2 GEMMs
  // at most SIDE CTAs, the Jacobi the rest).
  // ev: [0] R ready (st), [1] SVD done (s1), [2] T right done (st),
  //     [3] Q_u ready (st), [4] U/V transforms of the pending step done (s2).
  static const int SIDE = [] {
    const char* e = getenv("UTV_RU_SIDE");  // tuning knob; 0 = transforms on st
    return e ? atoi(e) : 88;
  }();
  static const int PBUD = [] {
    const char* e = getenv("UTV_RU_PANEL");
    return e ? atoi(e) : 48;
  }();
  cudaStream_t s1, s2;
  cudaEvent_t ev[5];
  UTV_CHECK(side_stream(&s1, ev, &s2));
  const int nsteps = (n + b - 1) / b < i1 ? (n + b - 1) / b : i1;
  long gcol = 0;
  int pending = ((carry & 1) && i0 > 0) ? i0 - 1 : -1;  // step whose SVD (and side transforms) are in flight
  auto finish_pending = [&]() -> int {
    if (pending < 0) return UTV_OK;
    UTV_CUDA(cudaStreamWaitEvent(st, ev[1], 0));
    if (SIDE > 0) UTV_CUDA(cudaStreamWaitEvent(st, ev[4], 0));
    UTV_CHECK(step_back(pending, pending * b, T, U, V, m, n, n - pending * b, b, errsq, trail2, w, st));
    pending = -1;
    return UTV_OK;
  };
  for (int i = i0; i < nsteps; ++i) {
    const int lo = i * b;
    const int k = m - lo, kc = n - lo;
    if (kc <= b) {
      UTV_CHECK(finish_pending());
      int carried = 0, fin = 0;
      UTV_CHECK(randutv_step(i, m, n, b, 0, q, false, T, U, V, nullptr, ldg, errsq, trail2,
                             svd_status, ws, ws_doubles, &carried, &fin, st));
      break;
    }
    Mat Bk = T.sub(lo, lo, k, kc);
    const bool alt = SIDE > 0 && (i & 1);  // Q_v double buffer (s2 may still read the other)
    Mat Yv{alt ? w.Yv2 : w.Yv, w.ldn, kc, b}, Tv{alt ? w.Tv2 : w.Tv, w.ldb, b, b};
    // sampling (randutv.py:185-193) + [Vq, ~] = hqr_full(Y) (:141)
    UTV_CHECK(sample_basic(Bk, b, q, G + gcol * ldg, ldg, w, st));
    UTV_CHECK(geqrf(Mat{w.Y, w.ldn, kc, b}, Yv, Tv, true, w.qr, w.qr_n, st));
    gcol += k;
    UTV_CHECK(finish_pending());
    Mat Yu{w.Yu, w.ldm, k, b}, Tu{w.Tu, w.ldb, b, b};
    if (SIDE <= 0) {
      UTV_CHECK(front_b(lo, T, U, V, Yv, Tv, k, kc, b, w, st));
    } else {
      // T right on st (randutv.py:143); V right on s2 (:144); QR of the T panel (:145)
      UTV_CHECK(larfb('R', false, Yv, Tv, T.sub(0, lo, m, kc), w.lfb, w.lfb_n, st));
      UTV_CUDA(cudaEventRecord(ev[2], st));
      UTV_CUDA(cudaStreamWaitEvent(s2, ev[2], 0));
      gemm_set_max_ctas(SIDE);
      const int rc = larfb('R', false, Yv, Tv, V.sub(0, lo, n, kc), w.lfb2, w.lfb_n, s2);
      gemm_set_max_ctas(0);
      UTV_CHECK(rc);
      panel_set_max_ctas(PBUD);
      const int rq = geqrf(T.sub(lo, lo, k, b), Yu, Tu, true, w.qr, w.qr_n, st);
      panel_set_max_ctas(0);
      UTV_CHECK(rq);
    }
    UTV_CUDA(cudaEventRecord(ev[0], st));
    UTV_CUDA(cudaStreamWaitEvent(s1, ev[0], 0));
    UTV_CHECK(step_svd(lo, T, b, svd_status + i, w, s1));
    UTV_CUDA(cudaEventRecord(ev[1], s1));
    pending = i;
    if (SIDE <= 0) {
      UTV_CHECK(front_c(lo, T, U, k, kc, b, w, st));
    } else {
      // U right on s2 (randutv.py:147), T left on st (:148)
      UTV_CUDA(cudaEventRecord(ev[3], st));
      UTV_CUDA(cudaStreamWaitEvent(s2, ev[3], 0));
      gemm_set_max_ctas(SIDE);
      const int rc = larfb('R', false, Yu, Tu, U.sub(0, lo, m, k), w.lfb2, w.lfb_n, s2);
      gemm_set_max_ctas(0);
      UTV_CHECK(rc);
      UTV_CUDA(cudaEventRecord(ev[4], s2));
      UTV_CHECK(larfb('L', true, Yu, Tu, T.sub(lo, lo + b, k, kc - b), w.lfb, w.lfb_n, st));
    }
  }
  if (!(carry & 2) || pending < 0 || pending + 1 >= (n + b - 1) / b) UTV_CHECK(finish_pending());
  return UTV_OK;
}

}  // namespace utv
