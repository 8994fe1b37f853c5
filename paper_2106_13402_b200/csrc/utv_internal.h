// Internal (C++) interfaces shared by the libutvb200 translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "common.cuh"

namespace utv {

int num_sms();

// ---- auxiliary streams / events (streams.cu) ----
// stream 0: randUTV side-stream SVD; stream 1: blocked-QR look-ahead panels.
// events 0-1: randUTV fp64, 2-3: randUTV fp32, 4-5: QR look-ahead.
int aux_stream(int idx, cudaStream_t* s);
int aux_event(int idx, cudaEvent_t* e);
// the same, private to the caller's stream `key` (a set per distinct key)
int aux_stream_for(cudaStream_t key, int idx, cudaStream_t* s);
int aux_event_for(cudaStream_t key, int idx, cudaEvent_t* e);
// lowest-priority non-blocking stream (deferred work: powerURV's dense Vq triangle).
// events 6-7: powerURV side build_t.
int aux_stream_low(cudaStream_t* s);

// ---- process model (streams.cu) ----
int check_device();          // UTV_ERR_DEVICE if the current device is not the bound one
}  // namespace utv
#include <mutex>
namespace utv {
std::mutex& driver_mutex();  // serialises the side-stream drivers' enqueue

// ---- launch accounting / profiling (prof.cu) ----
enum ProfCat {
  PROF_GEMM = 0,      // DMMA GEMM kernel (flops = 2MNK)
  PROF_SPLITK = 1,    // split-K reduction
  PROF_PANEL = 2,     // panel QR leaf kernel
  PROF_JACOBI = 3,    // Jacobi rounds kernel
  PROF_JFINISH = 4,   // Jacobi finish kernel
  PROF_OPS = 5,       // reductions / structured writes / copies
  PROF_GEMM_TF32 = 6, // 3xTF32 tcgen05 GEMM (flops = 2MNK useful)
  PROF_QRCP = 7,      // column-pivoted QR kernel (HBM-bound, bytes = trailing read + write)
  PROF_NCAT = 8
};
struct ProfScope {
  ProfScope(int cat, double flops, double bytes, cudaStream_t st, int launches = 1);
  ~ProfScope();
  int cat_;
  double flops_, bytes_;
  cudaStream_t st_;
  void* a_;
};

// Split-K scratch reserved by every multi-GEMM routine (1024 tiles of 128x128, 128 MiB).
constexpr size_t SPLITK_WS = 1024ull * 128 * 128;

// ---- K1 GEMM (gemm.cu) ----
int choose_splits(int tiles, int K);
// CTA budget for the next dgemm launches on this host thread (0 = all SMs).
void gemm_set_max_ctas(int n);
// Per-stream [ticket, done] counter pair of the dynamic tile schedulers
// (self-resetting; kernels on one stream run in order, so they can share it).
int* gemm_sched_slot(cudaStream_t st);
size_t dgemm_ws_doubles(int M, int N, int K);
int dgemm(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, long lda,
          const double* B, long ldb, double beta, double* C, long ldc, double* ws,
          size_t ws_doubles, cudaStream_t st);
// tri_a: A (not transposed, M == K) is upper triangular — the k-blocks below
// each tile's first row are skipped (TRMM-shaped product at half the flops).
int dgemm_ex(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, long lda,
             const double* B, long ldb, double beta, double* C, long ldc, double* ws,
             size_t ws_doubles, cudaStream_t st, bool tri_a);

// ---- K10 3xTF32 GEMM (gemm_tf32.cu): fp32 operands, ld % 4 == 0, 16B-aligned A/B ----
int sgemm_tf32x3(bool ta, bool tb, int M, int N, int K, float alpha, const float* A, long lda,
                 const float* B, long ldb, float beta, float* C, long ldc, cudaStream_t st);

// ---- small device ops (ops.cu) ----
// out[0] = sum of squares of the rows x cols block (deterministic two-pass).
int sumsq(const double* A, long lda, int rows, int cols, double* out, double* scratch,
          cudaStream_t st);
size_t sumsq_scratch_doubles();
int set_identity(double* A, long lda, int rows, int cols, cudaStream_t st);
int set_zero(double* A, long lda, int rows, int cols, cudaStream_t st);
int copy_mat(const double* src, long lds, double* dst, long ldd, int rows, int cols,
             cudaStream_t st);
// LAPACK dlaset: uplo 0 all / 1 upper / 2 lower off-diagonal <- alpha, diagonal <- beta.
int laset(int uplo, int rows, int cols, double alpha, double beta, double* A, long lda,
          cudaStream_t st);
int laset_f32(int uplo, int rows, int cols, float alpha, float beta, float* A, long lda,
              cudaStream_t st);
// *flag (device int) <- 1 if any entry is NaN/Inf, else 0.
int nonfinite(const double* A, long lda, int rows, int cols, int* flag, cudaStream_t st);
// A <- alpha diag(d) A (side 0) or alpha A diag(d) (side 1).
int diag_scale(int side, int rows, int cols, const double* d, double alpha, double* A, long lda,
               cudaStream_t st);
// device generators / metrics (metrics.cu)
int gen_bie(double* A, long lda, int n, cudaStream_t st);
int gen_kahan(double* A, long lda, int n, double theta, cudaStream_t st);
size_t trailing_fro_ws_doubles(int m, int n);
int trailing_fro(const double* T, long ldt, int m, int n, double* e, double* ws, cudaStream_t st);
// B (n x m) = A^T (A m x n)
int transpose(const double* A, long lda, double* B, long ldb, int m, int n, cudaStream_t st);
// fp32 helpers of the C5 path (ops.cu)
int sumsq_f32(const float* A, long lda, int rows, int cols, double* out, double* scratch,
              cudaStream_t st);
int cvt_f32_to_f64(const float* src, long lds, double* dst, long ldd, int rows, int cols,
                   cudaStream_t st);
int cvt_f64_to_f32(const double* src, long lds, float* dst, long ldd, int rows, int cols,
                   cudaStream_t st);
int pow2_normalize_f32(float* A, long lda, int rows, int cols, double* ss, double* scratch,
                       cudaStream_t st);
int set_diag_f32(float* A, long lda, int nr, int nc, const double* d, cudaStream_t st);
// diag block: A[:nr, :nc] = 0 except A[i,i] = d[i] (i < min(nr, nc)).
int set_diag(double* A, long lda, int nr, int nc, const double* d, cudaStream_t st);

// ---- K3 panel QR + K4 blocked QR (qr.cu) ----
// Householder QR of the rows x cols panel P (rows >= cols), in place:
// P <- R (zeros below the diagonal); Y (rows x cols, unit lower, zeros above)
// and the forward compact-WY triangle Tw (cols x cols) are written out.
// thr_src: device scalar holding ||input||_F^2 (threshold = eps*sqrt(.)).
size_t geqrf_ws_doubles(int rows, int cols, bool want_t);
// Fused single-launch panel QR (panel.cu), cols <= QR_PANEL, rows <= panel_rows_max():
// P <- R, Y, T (full cols x cols forward triangle; T must be zero below the diagonal).
size_t panel_ws_doubles();
int panel_rows_max();
// CTA budget for the next full-width panel_qr launches on this host thread (0 = all SMs).
void panel_set_max_ctas(int n);
int panel_qr(Mat P, Mat Y, Mat T, const double* fro2, double* ws, cudaStream_t st,
             int max_ctas = 0);
int geqrf(Mat P, Mat Y, Mat Tw, bool want_t, double* ws, size_t ws_doubles, cudaStream_t st);
// The same, recording grp_ev[j] on st once columns [j*QR_PANEL, (j+1)*QR_PANEL)
// of R (in P) and Y are final (grp_ev: ceil(cols / QR_PANEL) events).
// Host progress callback of the streaming drivers: called right after the
// cudaEventRecord of a progress event has been ENQUEUED (kind, index), so a
// caller whose host thread is held by the launch queue can still hand copy
// jobs to another thread in time.
typedef void (*ProgressFn)(void* ctx, int kind, int index);
int geqrf_ev(Mat P, Mat Y, Mat Tw, bool want_t, double* ws, size_t ws_doubles, cudaStream_t st,
             const cudaEvent_t* grp_ev, ProgressFn cb = nullptr, void* cb_ctx = nullptr,
             int cb_kind = 0);

// ---- K2 compact-WY apply (qr.cu) ----
// side 'L': B <- Q^(T) B ; side 'R': B <- B Q^(T);  Q = I - Y T Y^T, Y is k x w.
size_t larfb_ws_doubles(int brows, int bcols, int w);
int larfb(char side, bool trans, Mat Y, Mat T, Mat B, double* ws, size_t ws_doubles,
          cudaStream_t st);
// Q[:, :ncols] = I - Y (T Y[:ncols,:]^T)
int orgqr(Mat Y, Mat T, Mat Q, double* ws, size_t ws_doubles, cudaStream_t st);

// Panel-blocked variants: Q = Q_1 Q_2 ... Q_p with Q_j = I - Y_j T_j Y_j^T,
// T_j the QR_GROUP-wide diagonal blocks of T (off-diagonal blocks unused).
// Cost 2*rows*w*k-ish instead of the dense-T 3-GEMM form (no w x w x rows
// middle product, no full T needed).
constexpr int QR_PANEL = 256;
// Optional wider compact-WY block for the blocked QR's trailing updates and
// the panel-blocked applies (UTV_QR_GROUP / UTV_APPLY_GROUP = 512): two
// QR_PANEL panels whose T is merged locally.  Measured slower end to end,
// so both default to QR_PANEL (qr.cu).
constexpr int QR_GROUP = 512;
int larfb_panels(char side, bool trans, Mat Y, Mat T, Mat B, double* ws, size_t ws_doubles,
                 cudaStream_t st);
int orgqr_panels(Mat Y, Mat T, Mat Q, double* ws, size_t ws_doubles, cudaStream_t st);
// Fill the off-diagonal QR_PANEL blocks of T from Y and the diagonal blocks
// (T12 = -T11 (Y1^T Y2) T22), turning a panel-blocked T into the dense
// forward compact-WY triangle of the whole product (qr.py:63-68 semantics).
size_t build_t_ws_doubles(int rows, int cols);
int build_t(Mat Y, Mat T, double* ws, size_t ws_doubles, cudaStream_t st);
// One off-diagonal column block of build_t: T[:j0, j0:j0+jb] (ws: build_t_ws_doubles).
int merge_t_block(Mat Y, Mat T, int j0, int jb, double* ws, size_t ws_doubles, cudaStream_t st);

// ---- column-pivoted QR comparator (qrcp.cu), qr.py:152-204 ----
int qrcp_max_dim();
size_t qrcp_ws_doubles(int m, int n);
int qrcp(int m, int n, double* A, long lda, double* R, long ldr, double* Y, long ldy, double* T,
         long ldt, int* perm, double* ws, size_t ws_doubles, cudaStream_t st);

// ---- Householder reconstruction for TSQR (lu.cu) ----
// In-place LU without pivoting of (P - diag(s)), rows >= cols, s_j = -sign(pivot_j).
int getrf_signed(Mat P, double* s, double* ws, size_t ws_doubles, cudaStream_t st);
// B <- B * op(A)^{-1}, op(A) upper triangular (A upper + !trans, or A lower + trans).
int trsm_right_upper(bool trans, bool unit, int n, const double* A, long lda, Mat B, double* ws,
                     size_t ws_doubles, cudaStream_t st);
size_t lu_ws_doubles();

// ---- K6 Jacobi SVD (jacobi.cu) ----
// A (n x n, read only): sigma (desc, device), U (n x n), V (n x n) with the
// reference sign rule (svd.py:53-57).  *status_dev (device int) receives the
// number of sweeps used, or -1 if the sweep cap was hit (no host sync here).
size_t gesvj_ws_doubles(int n);
int gesvj(Mat A, double* sigma, Mat U, Mat V, double* ws, size_t ws_doubles, int* status_dev,
          cudaStream_t st);
// transpose: -1 default (rounds on A^T), 0 on A, 1 on A^T
int gesvj_ex(Mat A, double* sigma, Mat U, Mat V, double* ws, size_t ws_doubles, int* status_dev,
             cudaStream_t st, int transpose);

// ---- communicators (comm.cu): collectives on FP64 device buffers, caller's stream ----
struct Comm {
  int rank = 0, size = 1;
  virtual ~Comm() {}
  virtual int allreduce_sum(double* buf, size_t count, cudaStream_t st) = 0;
  // recv = [send of rank 0 | send of rank 1 | ...], count doubles each
  virtual int allgather(const double* send, double* recv, size_t count, cudaStream_t st) = 0;
  virtual int broadcast(double* buf, size_t count, int root, cudaStream_t st) = 0;
};
// P in-process ranks (threads); out[0..P-1] are owned by the caller (delete each).
Comm* new_local_group(int nranks, Comm** out);

// ---- TSQR + Householder reconstruction (tsqr.cu) ----
// Thin QR of the row-sharded X (this rank: X.rows x n, X.rows >= n; X is
// destroyed) into the explicit Q (this rank's rows) and the replicated R
// (n x n, zeros below the diagonal).  Local row chunks of <= cap rows.
size_t tsqr_ws_doubles(int m, int n, int nranks, int cap);
int tsqr(Comm* comm, Mat X, Mat Q, Mat R, int cap, double* ws, size_t ws_doubles, cudaStream_t st);
// Householder form (hqr_full semantics, qr.py:71-100) of a sharded explicit
// thin Q: Q <- Y (this rank's rows), Tw <- the dense forward triangle,
// R <- S R (replicated).  Rank 0 must own >= n rows.
size_t reconstruct_ws_doubles(int n);
int householder_reconstruct(Comm* comm, Mat Q, Mat Tw, Mat R, double* ws, size_t ws_doubles,
                            cudaStream_t st);
// Row-chunk cap of the single-launch panel QR (panel.cu) in use by geqrf.
int tsqr_default_cap();

}  // namespace utv
