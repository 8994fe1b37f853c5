// fp32 variant of blocked randUTV (basic), BASELINE config C5
// (randUTV b=512 q=2 fp32/TF32 on 32768^2, rank 2000).  Same step loop as
// randutv.cu (reference randutv.py:110-193), with T, U, V and every GEMM in
// FP32 on the tcgen05 tensor cores (3xTF32 split, K10):
//
//  * sampling Y = B^T G, q x Y = B^T (B Y) (randutv.py:189-192), unstabilised
//    like the reference; after every half-application Y is rescaled by a
//    power of two (exact, subspace unchanged) so rank-deficient trailing
//    blocks (||T22|| ~ eps32 ||A||, Y ~ ||T22||^(2q+1)) stay in fp32's
//    normal range (SURVEY §7 hard part 6);
//  * the latency-bound panel QRs (K3) and the b x b Jacobi SVD (K6) run in
//    fp64 on converted copies of the fp32 panels — they are not FLOP-bound,
//    and fp64 there only tightens the result; Y, T_wy, R, U_s, V_s and sigma
//    are rounded back to fp32;
//  * the compact-WY updates and the small-SVD rotations are 3xTF32 GEMMs.
// Requirements: m, n, b multiples of 4 and leading dimensions multiples of 4
// (TMA: 16-byte strides and sub-matrix origins).
#include <mutex>

#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace {
struct F32Mat {
  float* p;
  long ld;
  int rows, cols;
  float* at(long r, long c) const { return p + r + c * ld; }
  F32Mat sub(int r, int c, int nr, int nc) const { return F32Mat{p + r + (long)c * ld, ld, nr, nc}; }
};

int copy32(const float* src, long lds, float* dst, long ldd, int rows, int cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return UTV_OK;
  UTV_CUDA(cudaMemcpy2DAsync(dst, ldd * sizeof(float), src, lds * sizeof(float), rows * sizeof(float),
                             cols, cudaMemcpyDeviceToDevice, st));
  return UTV_OK;
}

struct Ws32 {
  // fp32
  float *Y, *Z, *Yv, *Tv, *Yu, *Tu, *Us, *Vs, *W1, *W2, *tmp;
  long ldn, ldm, ldb, ldx;
  // fp64
  double *P64, *Y64, *T64, *Us64, *Vs64, *Rs, *sig, *red, *ss, *qr, *svd;
  long ld64;
  size_t qr_n, svd_n;
};

size_t plan32(int m, int n, int b, Ws32* w, char* base) {
  size_t used = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + used : nullptr;
    used += round_up((long)bytes, 256);
    return p;
  };
  Ws32 v;
  const long mx = m > n ? m : n;
  v.ldn = round_up(n, 4);
  v.ldm = round_up(m, 4);
  v.ldb = round_up(b, 4);
  v.ldx = round_up(mx, 4);
  v.ld64 = round_up(mx, 4);
  v.qr_n = geqrf_ws_doubles((int)mx, b, true);
  v.svd_n = gesvj_ws_doubles(b);
  v.Y = (float*)take(4 * v.ldn * b);
  v.Z = (float*)take(4 * v.ldm * b);
  v.Yv = (float*)take(4 * v.ldn * b);
  v.Tv = (float*)take(4 * v.ldb * b);
  v.Yu = (float*)take(4 * v.ldm * b);
  v.Tu = (float*)take(4 * v.ldb * b);
  v.Us = (float*)take(4 * v.ldb * b);
  v.Vs = (float*)take(4 * v.ldb * b);
  v.W1 = (float*)take(4 * v.ldx * b);
  v.W2 = (float*)take(4 * v.ldx * b);
  v.tmp = (float*)take(4 * v.ldx * b);
  v.P64 = (double*)take(8 * v.ld64 * b);
  v.Y64 = (double*)take(8 * v.ld64 * b);
  v.T64 = (double*)take(8 * v.ldb * b);
  v.Us64 = (double*)take(8 * v.ldb * b);
  v.Vs64 = (double*)take(8 * v.ldb * b);
  v.Rs = (double*)take(8 * v.ldb * b);
  v.sig = (double*)take(8 * v.ldb);
  v.red = (double*)take(8 * sumsq_scratch_doubles());
  v.ss = (double*)take(8 * 16);
  v.qr = (double*)take(8 * v.qr_n);
  v.svd = (double*)take(8 * v.svd_n);
  if (w) *w = v;
  return used + 4096;
}

// B <- Q^(T) B (side L) or B Q (side R) with Q = I - Y T Y^T (fp32, 3 GEMMs).
int larfb32(char side, bool trans, F32Mat Y, F32Mat T, F32Mat B, const Ws32& w, cudaStream_t st) {
  const int k = Y.rows, wd = Y.cols;
  if (B.rows <= 0 || B.cols <= 0 || wd <= 0) return UTV_OK;
  if (side == 'L') {
    const int nb = B.cols;
    UTV_CHECK(sgemm_tf32x3(true, false, wd, nb, k, 1.0f, Y.p, Y.ld, B.p, B.ld, 0.0f, w.W1, w.ldb, st));
    UTV_CHECK(sgemm_tf32x3(trans, false, wd, nb, wd, 1.0f, T.p, T.ld, w.W1, w.ldb, 0.0f, w.W2, w.ldb, st));
    UTV_CHECK(sgemm_tf32x3(false, false, k, nb, wd, -1.0f, Y.p, Y.ld, w.W2, w.ldb, 1.0f, B.p, B.ld, st));
  } else {
    const int mb = B.rows;
    UTV_CHECK(sgemm_tf32x3(false, false, mb, wd, k, 1.0f, B.p, B.ld, Y.p, Y.ld, 0.0f, w.W1, w.ldx, st));
    UTV_CHECK(sgemm_tf32x3(false, trans, mb, wd, wd, 1.0f, w.W1, w.ldx, T.p, T.ld, 0.0f, w.W2, w.ldx, st));
    UTV_CHECK(sgemm_tf32x3(false, true, mb, k, wd, -1.0f, w.W2, w.ldx, Y.p, Y.ld, 1.0f, B.p, B.ld, st));
  }
  return UTV_OK;
}

// fp64 Householder QR of an fp32 panel: P (rows x c) -> R written back (zeros
// below the diagonal), Y and T returned in fp32.
int panel_qr32(F32Mat P, float* Y32, long ldy, float* T32, long ldt, const Ws32& w, cudaStream_t st) {
  const int rows = P.rows, c = P.cols;
  UTV_CHECK(cvt_f32_to_f64(P.p, P.ld, w.P64, w.ld64, rows, c, st));
  UTV_CHECK(geqrf(Mat{w.P64, w.ld64, rows, c}, Mat{w.Y64, w.ld64, rows, c}, Mat{w.T64, w.ldb, c, c},
                  true, w.qr, w.qr_n, st));
  UTV_CHECK(cvt_f64_to_f32(w.P64, w.ld64, P.p, P.ld, rows, c, st));
  UTV_CHECK(cvt_f64_to_f32(w.Y64, w.ld64, Y32, ldy, rows, c, st));
  UTV_CHECK(cvt_f64_to_f32(w.T64, w.ldb, T32, ldt, c, c, st));
  return UTV_OK;
}

int rot_right32(F32Mat X, const float* S, long lds, int c, const Ws32& w, cudaStream_t st) {
  if (X.rows <= 0) return UTV_OK;
  UTV_CHECK(sgemm_tf32x3(false, false, X.rows, c, c, 1.0f, X.p, X.ld, S, lds, 0.0f, w.tmp, w.ldx, st));
  return copy32(w.tmp, w.ldx, X.p, X.ld, X.rows, c, st);
}

int rot_left_t32(F32Mat X, const float* S, long lds, int c, const Ws32& w, cudaStream_t st) {
  if (X.cols <= 0) return UTV_OK;
  UTV_CHECK(sgemm_tf32x3(true, false, c, X.cols, c, 1.0f, S, lds, X.p, X.ld, 0.0f, w.tmp, w.ldb, st));
  return copy32(w.tmp, w.ldb, X.p, X.ld, c, X.cols, st);
}
}  // namespace

size_t randutv32_ws_bytes(int m, int n, int b) { return plan32(m, n, b, nullptr, nullptr); }

int randutv_basic_f32(int m, int n, int b, int q, float* Tp, long ldt, float* Up, long ldu,
                      float* Vp, long ldv, const float* G, long ldg, double* errsq, double* trail2,
                      int* svd_status, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (m < n) return -1;
  if (b < 1 || (b & 3)) return -3;
  if (q < 0) return -4;
  if ((m & 3) || (n & 3)) return -1;
  if ((ldt & 3) || (ldu & 3) || (ldv & 3) || (ldg & 3)) return UTV_ERR_ALIGN;
  if (ws_bytes < plan32(m, n, b, nullptr, nullptr)) return UTV_ERR_WORKSPACE;
  Ws32 w;
  plan32(m, n, b, &w, (char*)ws);
  F32Mat T{Tp, ldt, m, n}, U{Up, ldu, m, m}, V{Vp, ldv, n, n};

  // Software-pipelined like the fp64 loop (randutv.cu): the fp64 Jacobi SVD
  // of step i runs on a high-priority side stream (on a private copy of R)
  // while the main stream runs step i's left transform and step i+1's
  // sampling + Y-panel QR; step i's rotations follow on the main stream.
  cudaStream_t s1 = nullptr;
  cudaEvent_t ev[2];
  {
    static cudaStream_t g_s1 = nullptr;
    static cudaEvent_t g_ev[2];
    static std::once_flag once;
    static int err = 0;
    std::call_once(once, [] {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      if (cudaStreamCreateWithPriority(&g_s1, cudaStreamNonBlocking, hi) != cudaSuccess) err = 1;
      for (int e = 0; e < 2; ++e)
        if (cudaEventCreateWithFlags(&g_ev[e], cudaEventDisableTiming) != cudaSuccess) err = 1;
    });
    if (err) return UTV_ERR_CUDA;
    s1 = g_s1;
    ev[0] = g_ev[0];
    ev[1] = g_ev[1];
  }
  auto back = [&](int j) -> int {  // rotations, diag(sigma), error tracking of step j
    const int lo = j * b, mid = lo + b, kc = n - lo;
    UTV_CHECK(cvt_f64_to_f32(w.Us64, w.ldb, w.Us, w.ldb, b, b, st));
    UTV_CHECK(cvt_f64_to_f32(w.Vs64, w.ldb, w.Vs, w.ldb, b, b, st));
    UTV_CHECK(rot_right32(U.sub(0, lo, m, b), w.Us, w.ldb, b, w, st));
    UTV_CHECK(rot_right32(V.sub(0, lo, n, b), w.Vs, w.ldb, b, w, st));
    UTV_CHECK(set_diag_f32(T.at(lo, lo), T.ld, b, b, w.sig, st));
    UTV_CHECK(rot_left_t32(T.sub(lo, mid, b, kc - b), w.Us, w.ldb, b, w, st));
    UTV_CHECK(rot_right32(T.sub(0, lo, lo, b), w.Vs, w.ldb, b, w, st));
    UTV_CHECK(sumsq_f32(T.at(lo, lo), T.ld, b, kc, errsq + j, w.red, st));
    if (trail2) UTV_CHECK(sumsq_f32(T.at(mid, mid), T.ld, m - mid, kc - b, trail2 + j, w.red, st));
    return UTV_OK;
  };
  const int nsteps = (n + b - 1) / b;
  long gcol = 0;
  int pending = -1;
  for (int i = 0; i < nsteps; ++i) {
    const int lo = i * b, mid = lo + b;
    const int k = m - lo, kc = n - lo;
    if (kc > b) {
      F32Mat Bk = T.sub(lo, lo, k, kc);
      const float* Gi = G + gcol * ldg;  // b x k: G_i^T
      gcol += k;
      // ---- sampling (randutv.py:185-193), power-of-two rescaled ----
      UTV_CHECK(sgemm_tf32x3(true, true, kc, b, k, 1.0f, Bk.p, Bk.ld, Gi, ldg, 0.0f, w.Y, w.ldn, st));
      UTV_CHECK(pow2_normalize_f32(w.Y, w.ldn, kc, b, w.ss, w.red, st));
      for (int r = 0; r < q; ++r) {
        UTV_CHECK(sgemm_tf32x3(false, false, k, b, kc, 1.0f, Bk.p, Bk.ld, w.Y, w.ldn, 0.0f, w.Z, w.ldm, st));
        UTV_CHECK(pow2_normalize_f32(w.Z, w.ldm, k, b, w.ss, w.red, st));
        UTV_CHECK(sgemm_tf32x3(true, false, kc, b, k, 1.0f, Bk.p, Bk.ld, w.Z, w.ldm, 0.0f, w.Y, w.ldn, st));
        UTV_CHECK(pow2_normalize_f32(w.Y, w.ldn, kc, b, w.ss, w.red, st));
      }
      UTV_CHECK(panel_qr32(F32Mat{w.Y, w.ldn, kc, b}, w.Yv, w.ldn, w.Tv, w.ldb, w, st));
      if (pending >= 0) {
        UTV_CUDA(cudaStreamWaitEvent(st, ev[1], 0));
        UTV_CHECK(back(pending));
        pending = -1;
      }
      // ---- right transform (randutv.py:141-144) ----
      F32Mat Yv{w.Yv, w.ldn, kc, b}, Tv{w.Tv, w.ldb, b, b};
      UTV_CHECK(larfb32('R', false, Yv, Tv, T.sub(0, lo, m, kc), w, st));
      UTV_CHECK(larfb32('R', false, Yv, Tv, V.sub(0, lo, n, kc), w, st));
      // ---- left transform (randutv.py:146-149); R (fp64) kept for the SVD ----
      UTV_CHECK(panel_qr32(T.sub(lo, lo, k, b), w.Yu, w.ldm, w.Tu, w.ldb, w, st));
      UTV_CHECK(copy_mat(w.P64, w.ld64, w.Rs, w.ldb, b, b, st));
      UTV_CUDA(cudaEventRecord(ev[0], st));
      UTV_CUDA(cudaStreamWaitEvent(s1, ev[0], 0));
      UTV_CHECK(gesvj(Mat{w.Rs, w.ldb, b, b}, w.sig, Mat{w.Us64, w.ldb, b, b},
                      Mat{w.Vs64, w.ldb, b, b}, w.svd, w.svd_n, svd_status + i, s1));
      UTV_CUDA(cudaEventRecord(ev[1], s1));
      pending = i;
      F32Mat Yu{w.Yu, w.ldm, k, b}, Tu{w.Tu, w.ldb, b, b};
      UTV_CHECK(larfb32('R', false, Yu, Tu, U.sub(0, lo, m, k), w, st));
      UTV_CHECK(larfb32('L', true, Yu, Tu, T.sub(lo, mid, k, kc - b), w, st));
    } else {
      if (pending >= 0) {
        UTV_CUDA(cudaStreamWaitEvent(st, ev[1], 0));
        UTV_CHECK(back(pending));
        pending = -1;
      }
      // ---- final narrow block (randutv.py:164-177) ----
      if (k > kc) {
        UTV_CHECK(panel_qr32(T.sub(lo, lo, k, kc), w.Yu, w.ldm, w.Tu, w.ldb, w, st));
        UTV_CHECK(larfb32('R', false, F32Mat{w.Yu, w.ldm, k, kc}, F32Mat{w.Tu, w.ldb, kc, kc},
                          U.sub(0, lo, m, k), w, st));
      } else {
        UTV_CHECK(cvt_f32_to_f64(T.at(lo, lo), T.ld, w.P64, w.ld64, kc, kc, st));
      }
      UTV_CHECK(gesvj(Mat{w.P64, w.ld64, kc, kc}, w.sig, Mat{w.Us64, w.ldb, kc, kc},
                      Mat{w.Vs64, w.ldb, kc, kc}, w.svd, w.svd_n, svd_status + i, st));
      UTV_CHECK(cvt_f64_to_f32(w.Us64, w.ldb, w.Us, w.ldb, kc, kc, st));
      UTV_CHECK(cvt_f64_to_f32(w.Vs64, w.ldb, w.Vs, w.ldb, kc, kc, st));
      UTV_CHECK(rot_right32(U.sub(0, lo, m, kc), w.Us, w.ldb, kc, w, st));
      UTV_CHECK(rot_right32(V.sub(0, lo, n, kc), w.Vs, w.ldb, kc, w, st));
      UTV_CHECK(set_diag_f32(T.at(lo, lo), T.ld, k, kc, w.sig, st));
      UTV_CHECK(rot_right32(T.sub(0, lo, lo, kc), w.Vs, w.ldb, kc, w, st));
      UTV_CHECK(sumsq_f32(T.at(lo, lo), T.ld, k, kc, errsq + i, w.red, st));
      if (trail2) UTV_CUDA(cudaMemsetAsync(trail2 + i, 0, sizeof(double), st));
      break;
    }
  }
  if (pending >= 0) {
    UTV_CUDA(cudaStreamWaitEvent(st, ev[1], 0));
    UTV_CHECK(back(pending));
  }
  return UTV_OK;
}

}  // namespace utv
