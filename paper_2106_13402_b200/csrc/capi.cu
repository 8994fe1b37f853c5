// extern "C" entry points of libutvb200 (declared in include/utv_b200.h).
// No C++ exception crosses this boundary; every function returns a status.
#include "../../include/utv_b200.h"
#include "common.cuh"
#include "utv_internal.h"

namespace utv {
size_t randutv_ws_doubles(int m, int n, int b);
int randutv_basic(int m, int n, int b, int q, Mat T, Mat U, Mat V, const double* G, long ldg,
                  double* errsq, double* trail2, int* svd_status, double* ws, size_t ws_doubles,
                  cudaStream_t st);
size_t randutv_ws_doubles_p(int m, int n, int b, int p);
int randutv_basic_range(int i0, int i1, int m, int n, int b, int q, Mat T, Mat U, Mat V,
                        const double* G, long ldg, double* errsq, double* trail2, int* svd_status,
                        double* ws, size_t ws_doubles, cudaStream_t st, int carry);
int randutv_step(int i, int m, int n, int b, int p, int q, bool boosted, Mat T, Mat U, Mat V,
                 const double* G, long ldg, double* errsq, double* trail2, int* svd_status,
                 double* ws, size_t ws_doubles, int* carried, int* is_final, cudaStream_t st);
size_t randutv32_ws_bytes(int m, int n, int b);
int randutv_basic_f32(int m, int n, int b, int q, float* Tp, long ldt, float* Up, long ldu,
                      float* Vp, long ldv, const float* G, long ldg, double* errsq, double* trail2,
                      int* svd_status, void* ws, size_t ws_bytes, cudaStream_t st);
size_t powerurv_ws_doubles(int m, int n);
size_t powerurv_sharded_ws_doubles(int m, int n, int nranks, int cap);
int powerurv_sharded(Comm* comm, int m, int n, int q, Mat A, Mat G, Mat Uy, Mat Ut, Mat R, Mat Vy,
                     Mat Vt, int cap, double* ws, size_t ws_doubles, cudaStream_t st);
int powerurv(int m, int n, int q, Mat A, Mat G, Mat Uy, Mat Ut, Mat R, Mat Vy, Mat Vt, double* ws,
             size_t ws_doubles, cudaStream_t st, cudaEvent_t vq_ready, const double* yhat0 = nullptr,
             long ldy0 = 0, cudaEvent_t r_ready = nullptr, const cudaEvent_t* r_cols = nullptr,
             const cudaEvent_t* t_cols = nullptr, ProgressFn cb = nullptr, void* cb_ctx = nullptr);
}  // namespace utv

using namespace utv;

static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }
static inline size_t B(size_t doubles) { return doubles * sizeof(double) + 4096; }
static inline bool ld_ok(long ld, int rows) { return ld >= (rows > 1 ? rows : 1) && (ld & 1) == 0; }

// Drivers on the shared side streams/events: bound-device check, then the
// enqueue runs under the process-wide driver lock (streams.cu).
#define UTV_DRIVER_GUARD()                                 \
  UTV_CHECK(check_device());                               \
  std::lock_guard<std::mutex> driver_lock_(driver_mutex())

extern "C" {

int utv_version(void) { return 100; }

int utv_device_sms(void) {
  int n = 0, dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

size_t utv_dgemm_bufsize(int, int, int) { return B(SPLITK_WS); }

int utv_dgemm(char transa, char transb, int m, int n, int k, double alpha, const double* A,
              long lda, const double* Bm, long ldb, double beta, double* C, long ldc, void* work,
              size_t lwork, void* stream) {
  const bool ta = (transa == 'T' || transa == 't'), tb = (transb == 'T' || transb == 't');
  if (!ta && transa != 'N' && transa != 'n') return -1;
  if (!tb && transb != 'N' && transb != 'n') return -2;
  if (m < 0) return -3;
  if (n < 0) return -4;
  if (k < 0) return -5;
  if (k > 0 && !ld_ok(lda, ta ? k : m)) return -8;
  if (k > 0 && !ld_ok(ldb, tb ? n : k)) return -10;
  if (!ld_ok(ldc, m)) return -13;
  return dgemm(ta, tb, m, n, k, alpha, A, lda, Bm, ldb, beta, C, ldc, (double*)work,
               work ? lwork / sizeof(double) : 0, S(stream));
}

size_t utv_dsumsq_bufsize(void) { return B(sumsq_scratch_doubles()); }

int utv_dsumsq(int m, int n, const double* A, long lda, double* out, void* work, size_t lwork,
               void* stream) {
  if (m < 0) return -1;
  if (n < 0) return -2;
  if (lwork < sumsq_scratch_doubles() * sizeof(double)) return UTV_ERR_WORKSPACE;
  return sumsq(A, lda, m, n, out, (double*)work, S(stream));
}

size_t utv_dgeqrf_bufsize(int m, int n) { return B(geqrf_ws_doubles(m, n, true)); }

int utv_dgeqrf(int m, int n, double* A, long lda, double* Y, long ldy, double* T, long ldt,
               void* work, size_t lwork, void* stream) {
  if (m < 1) return -1;
  if (n < 1 || n > m) return -2;
  if (!ld_ok(lda, m)) return -4;
  if (!ld_ok(ldy, m)) return -6;
  if (!ld_ok(ldt, n)) return -8;
  return geqrf(Mat{A, lda, m, n}, Mat{Y, ldy, m, n}, Mat{T, ldt, n, n}, true, (double*)work,
               lwork / sizeof(double), S(stream));
}

size_t utv_dlarfb_bufsize(int m, int n, int w) { return B(larfb_ws_doubles(m, n, w)); }

int utv_dlarfb(char side, char trans, int m, int n, int k, int w, const double* Y, long ldy,
               const double* T, long ldt, double* Bm, long ldb, void* work, size_t lwork,
               void* stream) {
  const bool left = (side == 'L' || side == 'l');
  if (!left && side != 'R' && side != 'r') return -1;
  const bool tr = (trans == 'T' || trans == 't');
  if (!tr && trans != 'N' && trans != 'n') return -2;
  if (m < 0) return -3;
  if (n < 0) return -4;
  if (k < 1 || (left ? m != k : n != k)) return -5;
  if (w < 1 || w > k) return -6;
  if (!ld_ok(ldy, k)) return -8;
  if (!ld_ok(ldt, w)) return -10;
  if (!ld_ok(ldb, m)) return -12;
  // wide factors: apply panel by panel (only the QR_PANEL diagonal blocks of
  // T are read; identical result, no w x w x rows middle product)
  if (w > QR_PANEL)
    return larfb_panels(left ? 'L' : 'R', tr, Mat{(double*)Y, ldy, k, w}, Mat{(double*)T, ldt, w, w},
                        Mat{Bm, ldb, m, n}, (double*)work, lwork / sizeof(double), S(stream));
  return larfb(left ? 'L' : 'R', tr, Mat{(double*)Y, ldy, k, w}, Mat{(double*)T, ldt, w, w},
               Mat{Bm, ldb, m, n}, (double*)work, lwork / sizeof(double), S(stream));
}

int utv_dgeqrf_rows_max(void) { return panel_rows_max(); }

size_t utv_dgeqp3_bufsize(int m, int n) { return B(qrcp_ws_doubles(m, n)); }
int utv_dgeqp3_max_dim(void) { return qrcp_max_dim(); }

int utv_dgeqp3_f64(int m, int n, double* A, long lda, double* R, long ldr, double* Y, long ldy,
                   double* T, long ldt, int* perm, void* work, size_t lwork, void* stream) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  const int r = m < n ? m : n;
  if (!ld_ok(lda, m)) return -4;
  if (!ld_ok(ldr, m)) return -6;
  if (!ld_ok(ldy, m)) return -8;
  if (!ld_ok(ldt, r)) return -10;
  if (perm == nullptr) return -11;
  return qrcp(m, n, A, lda, R, ldr, Y, ldy, T, ldt, perm, (double*)work, lwork / sizeof(double),
              S(stream));
}

int utv_randutv_basic_steps_f64(int i0, int i1, int m, int n, int b, int q, double* T, long ldt,
                                double* U, long ldu, double* V, long ldv, const double* G, long ldg,
                                double* errsq, double* trail2, int* svd_status, void* work,
                                size_t lwork, void* stream) {
  if (i0 < 0 || i1 < i0) return -1;
  if (m < n || n < 1) return -3;
  if (b < 1 || b > 1024) return -5;
  if (q < 0) return -6;
  if (!ld_ok(ldt, m)) return -8;
  if (!ld_ok(ldu, m)) return -10;
  if (!ld_ok(ldv, n)) return -12;
  UTV_DRIVER_GUARD();
  return randutv_basic_range(i0, i1, m, n, b, q, Mat{T, ldt, m, n}, Mat{U, ldu, m, m},
                             Mat{V, ldv, n, n}, G, ldg, errsq, trail2, svd_status, (double*)work,
                             lwork / sizeof(double), S(stream), 0);
}

int utv_randutv_basic_steps_carry_f64(int i0, int i1, int carry, int m, int n, int b, int q,
                                      double* T, long ldt, double* U, long ldu, double* V, long ldv,
                                      const double* G, long ldg, double* errsq, double* trail2,
                                      int* svd_status, void* work, size_t lwork, void* stream) {
  if (i0 < 0 || i1 < i0) return -1;
  if (carry < 0 || carry > 3) return -3;
  if (m < n || n < 1) return -4;
  if (b < 1 || b > 1024) return -6;
  if (q < 0) return -7;
  if (!ld_ok(ldt, m)) return -9;
  if (!ld_ok(ldu, m)) return -11;
  if (!ld_ok(ldv, n)) return -13;
  UTV_DRIVER_GUARD();
  return randutv_basic_range(i0, i1, m, n, b, q, Mat{T, ldt, m, n}, Mat{U, ldu, m, m},
                             Mat{V, ldv, n, n}, G, ldg, errsq, trail2, svd_status, (double*)work,
                             lwork / sizeof(double), S(stream), carry);
}

size_t utv_randutv_step_bufsize(int m, int n, int b, int p, int) { return B(randutv_ws_doubles_p(m, n, b, p)); }

int utv_randutv_step_f64(int i, int m, int n, int b, int p, int q, int boosted, double* T, long ldt,
                         double* U, long ldu, double* V, long ldv, const double* G, long ldg,
                         double* errsq, double* trail2, int* svd_status, int* carried,
                         int* is_final, void* work, size_t lwork, void* stream) {
  if (i < 0 || (long)i * b >= n) return -1;
  if (m < n || n < 1) return -2;
  if (b < 1 || b + p > 1024) return -4;
  if (p < 0) return -5;
  if (q < 0 || (boosted && q < 1)) return -6;
  if (!ld_ok(ldt, m)) return -9;
  if (!ld_ok(ldu, m)) return -11;
  if (!ld_ok(ldv, n)) return -13;
  if (!carried || !is_final) return -19;
  UTV_DRIVER_GUARD();
  return randutv_step(i, m, n, b, boosted ? p : 0, q, boosted != 0, Mat{T, ldt, m, n},
                      Mat{U, ldu, m, m}, Mat{V, ldv, n, n}, G, ldg, errsq, trail2, svd_status,
                      (double*)work, lwork / sizeof(double), carried, is_final, S(stream));
}

size_t utv_randutv_basic_f32_bufsize(int m, int n, int b, int) { return randutv32_ws_bytes(m, n, b); }

int utv_randutv_basic_f32(int m, int n, int b, int q, float* T, long ldt, float* U, long ldu,
                          float* V, long ldv, const float* G, long ldg, double* errsq,
                          double* trail2, int* svd_status, void* work, size_t lwork, void* stream) {
  if (m < 1 || n < 1) return -1;
  if (b < 1 || b > 1024) return -3;
  if (q < 0) return -4;
  if (ldt < m) return -6;
  if (ldu < m) return -8;
  if (ldv < n) return -10;
  UTV_DRIVER_GUARD();
  return randutv_basic_f32(m, n, b, q, T, ldt, U, ldu, V, ldv, G, ldg, errsq, trail2, svd_status,
                           work, lwork, S(stream));
}

int utv_sgemm_tf32x3(char transa, char transb, int m, int n, int k, float alpha, const float* A,
                     long lda, const float* Bm, long ldb, float beta, float* C, long ldc,
                     void* stream) {
  const bool ta = (transa == 'T' || transa == 't'), tb = (transb == 'T' || transb == 't');
  if (!ta && transa != 'N' && transa != 'n') return -1;
  if (!tb && transb != 'N' && transb != 'n') return -2;
  if (m < 0) return -3;
  if (n < 0) return -4;
  if (k < 0) return -5;
  if (k > 0 && (lda < (ta ? k : m) || (lda & 3))) return -8;
  if (k > 0 && (ldb < (tb ? n : k) || (ldb & 3))) return -10;
  if (ldc < (m > 1 ? m : 1)) return -13;
  return sgemm_tf32x3(ta, tb, m, n, k, alpha, A, lda, Bm, ldb, beta, C, ldc, S(stream));
}

int utv_dlacpy(int m, int n, const double* A, long lda, double* Bm, long ldb, void* stream) {
  if (m < 0) return -1;
  if (n < 0) return -2;
  if (lda < m) return -4;
  if (ldb < m) return -6;
  return copy_mat(A, lda, Bm, ldb, m, n, S(stream));
}

int utv_dlaset(char uplo, int m, int n, double alpha, double beta, double* A, long lda,
               void* stream) {
  int u;
  if (uplo == 'U' || uplo == 'u') u = 1;
  else if (uplo == 'L' || uplo == 'l') u = 2;
  else if (uplo == 'A' || uplo == 'a') u = 0;
  else return -1;
  if (m < 0) return -2;
  if (n < 0) return -3;
  if (lda < m) return -7;
  return laset(u, m, n, alpha, beta, A, lda, S(stream));
}

int utv_slaset(char uplo, int m, int n, float alpha, float beta, float* A, long lda,
               void* stream) {
  int u;
  if (uplo == 'U' || uplo == 'u') u = 1;
  else if (uplo == 'L' || uplo == 'l') u = 2;
  else if (uplo == 'A' || uplo == 'a') u = 0;
  else return -1;
  if (m < 0) return -2;
  if (n < 0) return -3;
  if (lda < m) return -7;
  return laset_f32(u, m, n, alpha, beta, A, lda, S(stream));
}

int utv_zero(void* p, size_t bytes, void* stream) {
  if (bytes && !p) return -1;
  if (bytes) UTV_CUDA(cudaMemsetAsync(p, 0, bytes, S(stream)));
  return UTV_OK;
}

int utv_dnonfinite(int m, int n, const double* A, long lda, int* flag, void* stream) {
  if (m < 0) return -1;
  if (n < 0) return -2;
  if (lda < m) return -4;
  if (!flag) return -5;
  return nonfinite(A, lda, m, n, flag, S(stream));
}

int utv_dtranspose(int m, int n, const double* A, long lda, double* Bm, long ldb, void* stream) {
  if (m < 0) return -1;
  if (n < 0) return -2;
  if (lda < m) return -4;
  if (ldb < n) return -6;
  return transpose(A, lda, Bm, ldb, m, n, S(stream));
}

int utv_dgen_bie(int n, double* A, long lda, void* stream) {
  if (n < 1) return -1;
  if (lda < n) return -3;
  return gen_bie(A, lda, n, S(stream));
}

int utv_dgen_kahan(int n, double theta, double* A, long lda, void* stream) {
  if (n < 1) return -1;
  if (lda < n) return -4;
  return gen_kahan(A, lda, n, theta, S(stream));
}

size_t utv_dtrailing_fro_bufsize(int m, int n) { return B(trailing_fro_ws_doubles(m, n)); }

int utv_dtrailing_fro(int m, int n, const double* T, long ldt, double* e, void* work, size_t lwork,
                      void* stream) {
  if (m < 1) return -1;
  if (n < 1) return -2;
  if (ldt < m) return -4;
  if (lwork < trailing_fro_ws_doubles(m, n) * sizeof(double)) return UTV_ERR_WORKSPACE;
  return trailing_fro(T, ldt, m, n, e, (double*)work, S(stream));
}

int utv_dtri_zero(char uplo, int m, int n, double* A, long lda, void* stream) {
  int u;
  if (uplo == 'U' || uplo == 'u') u = 3;
  else if (uplo == 'L' || uplo == 'l') u = 4;
  else return -1;
  if (m < 0) return -2;
  if (n < 0) return -3;
  if (lda < m) return -5;
  return laset(u, m, n, 0.0, 0.0, A, lda, S(stream));
}

int utv_ddiag_scale(char side, int m, int n, const double* d, double alpha, double* A, long lda,
                    void* stream) {
  const bool left = (side == 'L' || side == 'l');
  if (!left && side != 'R' && side != 'r') return -1;
  if (m < 0) return -2;
  if (n < 0) return -3;
  if (lda < m) return -7;
  return diag_scale(left ? 0 : 1, m, n, d, alpha, A, lda, S(stream));
}

size_t utv_dgetrf_signed_bufsize(int, int) { return B(lu_ws_doubles()); }

int utv_dgetrf_signed(int m, int n, double* A, long lda, double* s, void* work, size_t lwork,
                      void* stream) {
  if (m < 1) return -1;
  if (n < 1 || n > m) return -2;
  if (!ld_ok(lda, m)) return -4;
  if (lwork < lu_ws_doubles() * sizeof(double)) return UTV_ERR_WORKSPACE;
  return getrf_signed(Mat{A, lda, m, n}, s, (double*)work, lwork / sizeof(double), S(stream));
}

size_t utv_dtrsm_bufsize(int, int) { return B(lu_ws_doubles()); }

int utv_dtrsm_right(char uplo, char trans, char diag, int m, int n, const double* A, long lda,
                    double* Bm, long ldb, void* work, size_t lwork, void* stream) {
  const bool up = (uplo == 'U' || uplo == 'u');
  if (!up && uplo != 'L' && uplo != 'l') return -1;
  const bool tr = (trans == 'T' || trans == 't');
  if (!tr && trans != 'N' && trans != 'n') return -2;
  const bool unit = (diag == 'U' || diag == 'u');
  if (!unit && diag != 'N' && diag != 'n') return -3;
  if (up == tr) return -2;  // only op(A) upper: (U, N) or (L, T)
  if (m < 0) return -4;
  if (n < 0) return -5;
  if (!ld_ok(lda, n)) return -7;
  if (!ld_ok(ldb, m)) return -9;
  if (lwork < lu_ws_doubles() * sizeof(double)) return UTV_ERR_WORKSPACE;
  return trsm_right_upper(tr, unit, n, A, lda, Mat{Bm, ldb, m, n}, (double*)work,
                          lwork / sizeof(double), S(stream));
}

size_t utv_dorgqr_bufsize(int m, int ncols, int w) {
  return B((size_t)round_up(w, 4) * ncols + SPLITK_WS + 1024);
}

int utv_dorgqr(int m, int ncols, int w, const double* Y, long ldy, const double* T, long ldt,
               double* Q, long ldq, void* work, size_t lwork, void* stream) {
  if (m < 1) return -1;
  if (ncols < 1 || ncols > m) return -2;
  if (w < 1 || w > m) return -3;
  if (!ld_ok(ldy, m)) return -5;
  if (!ld_ok(ldt, w)) return -7;
  if (!ld_ok(ldq, m)) return -9;
  return orgqr(Mat{(double*)Y, ldy, m, w}, Mat{(double*)T, ldt, w, w}, Mat{Q, ldq, m, ncols},
               (double*)work, lwork / sizeof(double), S(stream));
}

size_t utv_dgesvj_bufsize(int n) { return B(gesvj_ws_doubles(n)); }

int utv_dgesvj(int n, const double* A, long lda, double* sigma, double* U, long ldu, double* V,
               long ldv, int* status, void* work, size_t lwork, void* stream) {
  if (n < 1 || n > 1024) return -1;
  if (lda < n) return -3;
  if (ldu < n) return -6;
  if (ldv < n) return -8;
  return gesvj(Mat{(double*)A, lda, n, n}, sigma, Mat{U, ldu, n, n}, Mat{V, ldv, n, n},
               (double*)work, lwork / sizeof(double), status, S(stream));
}

int utv_dgesvj_ex(int n, const double* A, long lda, double* sigma, double* U, long ldu, double* V,
                  long ldv, int* status, int transpose, void* work, size_t lwork, void* stream) {
  if (n < 1 || n > 1024) return -1;
  if (lda < n) return -3;
  if (ldu < n) return -6;
  if (ldv < n) return -8;
  if (transpose < -1 || transpose > 1) return -10;
  return gesvj_ex(Mat{(double*)A, lda, n, n}, sigma, Mat{U, ldu, n, n}, Mat{V, ldv, n, n},
                  (double*)work, lwork / sizeof(double), status, S(stream), transpose);
}

size_t utv_randutv_basic_bufsize(int m, int n, int b, int) { return B(randutv_ws_doubles(m, n, b)); }

int utv_randutv_basic_f64(int m, int n, int b, int q, double* T, long ldt, double* U, long ldu,
                          double* V, long ldv, const double* G, long ldg, double* errsq,
                          double* trail2, int* svd_status, void* work, size_t lwork,
                          void* stream) {
  if (m < 1) return -1;
  if (n < 1 || n > m) return -2;
  if (b < 1 || b > 1024) return -3;
  if (q < 0) return -4;
  if (!ld_ok(ldt, m)) return -6;
  if (!ld_ok(ldu, m)) return -8;
  if (!ld_ok(ldv, n)) return -10;
  if (n > b && !ld_ok(ldg, b)) return -12;
  UTV_DRIVER_GUARD();
  return randutv_basic(m, n, b, q, Mat{T, ldt, m, n}, Mat{U, ldu, m, m}, Mat{V, ldv, n, n}, G, ldg,
                       errsq, trail2, svd_status, (double*)work, lwork / sizeof(double),
                       S(stream));
}

size_t utv_powerurv_bufsize(int m, int n, int) { return B(powerurv_ws_doubles(m, n)); }

int utv_powerurv_f64(int m, int n, int q, const double* A, long lda, const double* G, long ldg,
                     double* Uy, long lduy, double* Ut, long ldut, double* R, long ldr,
                     double* Vy, long ldvy, double* Vt, long ldvt, void* work, size_t lwork,
                     void* stream) {
  return utv_powerurv_f64_ev(m, n, q, A, lda, G, ldg, Uy, lduy, Ut, ldut, R, ldr, Vy, ldvy, Vt, ldvt,
                             work, lwork, stream, nullptr, nullptr);
}

int utv_powerurv_f64_ev(int m, int n, int q, const double* A, long lda, const double* G, long ldg,
                        double* Uy, long lduy, double* Ut, long ldut, double* R, long ldr,
                        double* Vy, long ldvy, double* Vt, long ldvt, void* work, size_t lwork,
                        void* stream, void* vq_ready, void* r_ready) {
  if (m < 1) return -1;
  if (n < 1 || n > m) return -2;
  if (q < 0) return -3;
  if (!ld_ok(lda, m)) return -5;
  if (!ld_ok(ldg, n)) return -7;
  if (!ld_ok(lduy, m)) return -9;
  if (!ld_ok(ldut, n)) return -11;
  if (!ld_ok(ldr, m)) return -13;
  if (!ld_ok(ldvy, n)) return -15;
  if (!ld_ok(ldvt, n)) return -17;
  UTV_DRIVER_GUARD();
  return powerurv(m, n, q, Mat{(double*)A, lda, m, n}, Mat{(double*)G, ldg, n, n},
                  Mat{Uy, lduy, m, n}, Mat{Ut, ldut, n, n}, Mat{R, ldr, m, n}, Mat{Vy, ldvy, n, n},
                  Mat{Vt, ldvt, n, n}, (double*)work, lwork / sizeof(double), S(stream),
                  (cudaEvent_t)vq_ready, nullptr, 0, (cudaEvent_t)r_ready);
}

int utv_powerurv_f64_yhat(int m, int n, int q, const double* A, long lda, const double* Yhat0,
                          long ldy0, double* Uy, long lduy, double* Ut, long ldut, double* R,
                          long ldr, double* Vy, long ldvy, double* Vt, long ldvt, void* work,
                          size_t lwork, void* stream, void* vq_ready, void* r_ready) {
  if (m < 1) return -1;
  if (n < 1 || n > m) return -2;
  if (q < 1) return -3;
  if (!ld_ok(lda, m)) return -5;
  if (Yhat0 == nullptr) return -6;
  if (!ld_ok(ldy0, m)) return -7;
  if (!ld_ok(lduy, m)) return -9;
  if (!ld_ok(ldut, n)) return -11;
  if (!ld_ok(ldr, m)) return -13;
  if (!ld_ok(ldvy, n)) return -15;
  if (!ld_ok(ldvt, n)) return -17;
  UTV_DRIVER_GUARD();
  return powerurv(m, n, q, Mat{(double*)A, lda, m, n}, Mat{nullptr, n, n, n},
                  Mat{Uy, lduy, m, n}, Mat{Ut, ldut, n, n}, Mat{R, ldr, m, n}, Mat{Vy, ldvy, n, n},
                  Mat{Vt, ldvt, n, n}, (double*)work, lwork / sizeof(double), S(stream),
                  (cudaEvent_t)vq_ready, Yhat0, ldy0, (cudaEvent_t)r_ready);
}

int utv_powerurv_f64_cols(int m, int n, int q, const double* A, long lda, const double* G, long ldg,
                          const double* Yhat0, long ldy0, double* Uy, long lduy, double* Ut,
                          long ldut, double* R, long ldr, double* Vy, long ldvy, double* Vt,
                          long ldvt, void* work, size_t lwork, void* stream, void* vq_ready,
                          int ncols_ev, void* const* r_cols, void* const* t_cols,
                          void* progress_cb, void* progress_ctx) {
  if (m < 1) return -1;
  if (n < 1 || n > m) return -2;
  if (q < 0 || (Yhat0 && q < 1)) return -3;
  if (!ld_ok(lda, m)) return -5;
  if (!Yhat0 && (!G || !ld_ok(ldg, n))) return -7;
  if (Yhat0 && !ld_ok(ldy0, m)) return -9;
  if (!ld_ok(lduy, m)) return -11;
  if (!ld_ok(ldut, n)) return -13;
  if (!ld_ok(ldr, m)) return -15;
  if (!ld_ok(ldvy, n)) return -17;
  if (!ld_ok(ldvt, n)) return -19;
  const int ngrp = (n + QR_PANEL - 1) / QR_PANEL;
  if ((r_cols || t_cols) && ncols_ev != ngrp) return -24;
  UTV_DRIVER_GUARD();
  return powerurv(m, n, q, Mat{(double*)A, lda, m, n}, Mat{(double*)G, ldg, n, n},
                  Mat{Uy, lduy, m, n}, Mat{Ut, ldut, n, n}, Mat{R, ldr, m, n}, Mat{Vy, ldvy, n, n},
                  Mat{Vt, ldvt, n, n}, (double*)work, lwork / sizeof(double), S(stream),
                  (cudaEvent_t)vq_ready, Yhat0, ldy0, nullptr, (const cudaEvent_t*)r_cols,
                  (const cudaEvent_t*)t_cols, (ProgressFn)progress_cb, progress_ctx);
}

size_t utv_powerurv_sharded_bufsize(int m_local, int n, int nranks, int chunk_rows) {
  return B(powerurv_sharded_ws_doubles(m_local, n, nranks < 1 ? 1 : nranks, chunk_rows));
}

int utv_powerurv_sharded_f64(utv_comm_t comm, int m_local, int n, int q, const double* A, long lda,
                             const double* G, long ldg, double* Uy, long lduy, double* Ut,
                             long ldut, double* R, long ldr, double* Vy, long ldvy, double* Vt,
                             long ldvt, int chunk_rows, void* work, size_t lwork, void* stream) {
  if (!comm) return -1;
  // argument errors are reported after the ranks agree (see powerurv_sharded)
  int bad = 0;
  if (!ld_ok(lda, m_local)) bad = -6;
  else if (!ld_ok(ldg, n)) bad = -8;
  else if (!ld_ok(lduy, m_local)) bad = -10;
  else if (!ld_ok(ldut, n)) bad = -12;
  else if (!ld_ok(ldr, n)) bad = -14;
  else if (!ld_ok(ldvy, n)) bad = -16;
  else if (!ld_ok(ldvt, n)) bad = -18;
  if (bad) m_local = -1;  // forces the agreed failure path
  UTV_CHECK(check_device());
  const int rc = powerurv_sharded((Comm*)comm, m_local, n, q, Mat{(double*)A, lda, m_local, n},
                                  Mat{(double*)G, ldg, n, n}, Mat{Uy, lduy, m_local, n},
                                  Mat{Ut, ldut, n, n}, Mat{R, ldr, n, n}, Mat{Vy, ldvy, n, n},
                                  Mat{Vt, ldvt, n, n}, chunk_rows, (double*)work,
                                  lwork / sizeof(double), S(stream));
  return bad ? bad : rc;
}

}  // extern "C"
