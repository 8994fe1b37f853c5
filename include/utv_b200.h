/*
 * libutvb200 — C ABI of the B200-native powerURV / randUTV hot path.
 *
 * The reference (utvkit, arXiv 2106.13402) has no FFI layer: its boundary is
 * the Python API re-exported by utvkit/__init__.py.  Each entry point below
 * replaces one reference function on that path (file:line cited); the
 * Python package paper_2106_13402_b200 binds them with ctypes and keeps the
 * reference's signatures, result types and exceptions.
 *
 * Conventions
 *  - All matrices are column-major FP64 device pointers with an explicit
 *    leading dimension.  Leading dimensions must be EVEN (TMA stride rule);
 *    pointers must be 8-byte aligned.
 *  - `work` is a caller-allocated device workspace of `lwork` bytes; query
 *    the size with the matching *_bufsize function.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  No entry
 *    point synchronises the host; results are ready when the stream is.
 *  - Return value: 0 ok; -i = argument i is invalid (LAPACK `info` style);
 *    -1000 CUDA error; -1001 workspace too small; -1002 alignment;
 *    -1003 wrong device (see the process model); -1004 communicator error;
 *    > 0 numerical failure reported through a device status word.
 *  - Deterministic: identical inputs give bitwise identical outputs.
 *  - Process model: one device per process.  The library binds to the
 *    first device it is used on (side streams, events, tile-scheduler slots
 *    and split-K turn counters live there); the drivers and the sharded
 *    entry return -1003 when called with another current device.  Calls
 *    from several host threads are safe on distinct caller streams; the
 *    side-stream drivers (utv_randutv_basic_f64 / _steps_f64 / _step_f64 /
 *    _f32, utv_powerurv_f64*) enqueue under a process-wide lock, and the
 *    step ranges of ONE factorisation (utv_randutv_basic_steps_f64,
 *    utv_randutv_step_f64) must not interleave with another randUTV call.
 *    (The Python package serialises its public calls.)
 */
#ifndef UTV_B200_H
#define UTV_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Library/ABI version (major*100 + minor). */
int utv_version(void);

/* Number of SMs of the current device (0 if no device). */
int utv_device_sms(void);

/* C = alpha*op(A)*op(B) + beta*C ; op = 'N' | 'T'.
 * Replaces numpy `@` on the hot path (randutv.py:190-192, qr.py:116,120,131,
 * powerurv.py:64,66, randutv.py:152-156).  FP64 DMMA tensor cores, TMA. */
size_t utv_dgemm_bufsize(int m, int n, int k);
int utv_dgemm(char transa, char transb, int m, int n, int k, double alpha, const double* A,
              long lda, const double* B, long ldb, double beta, double* C, long ldc, void* work,
              size_t lwork, void* stream);

/* FP32 C = alpha*op(A)*op(B) + beta*C on the tcgen05 tensor cores with the
 * 3xTF32 split (hi*hi + hi*lo + lo*hi, hi = rna_tf32(x)): FP32-level accuracy
 * for the fp32 randUTV variant (BASELINE C5).  lda/ldb multiples of 4, A/B
 * 16-byte aligned (TMA). */
int utv_sgemm_tf32x3(char transa, char transb, int m, int n, int k, float alpha, const float* A,
                     long lda, const float* B, long ldb, float beta, float* C, long ldc,
                     void* stream);

/* Sum of squares of an m x n block -> *out (device scalar).
 * Replaces frobenius_norm (matrix.py:79-81) and ErrorTracker.update's panel
 * mass (randutv.py:52-62). */
size_t utv_dsumsq_bufsize(void);
int utv_dsumsq(int m, int n, const double* A, long lda, double* out, void* work, size_t lwork,
               void* stream);

/* Householder QR, m >= n: A <- R (zeros below the diagonal), Y (m x n unit
 * lower trapezoidal, zeros above), T (n x n upper, forward compact WY).
 * Replaces hqr_full (qr.py:71-100) incl. _reflector (qr.py:43-60) and
 * _append_twy_column (qr.py:63-68); skip rule and sign convention kept. */
size_t utv_dgeqrf_bufsize(int m, int n);
int utv_dgeqrf(int m, int n, double* A, long lda, double* Y, long ldy, double* T, long ldt,
               void* work, size_t lwork, void* stream);

/* Apply Q = I - Y T Y^T (k x k, w reflectors) to the m x n block B:
 * side 'L': B <- Q B or Q^T B (trans 'N'/'T'), requires m == k;
 * side 'R': B <- B Q or B Q^T, requires n == k.
 * Replaces apply_q (qr.py:103-121). */
size_t utv_dlarfb_bufsize(int m, int n, int w);
int utv_dlarfb(char side, char trans, int m, int n, int k, int w, const double* Y, long ldy,
               const double* T, long ldt, double* B, long ldb, void* work, size_t lwork,
               void* stream);

/* Largest row count utv_dgeqrf accepts (148 CTAs x 512-row slabs); taller
 * inputs are split into row chunks by the caller (TSQR). */
int utv_dgeqrf_rows_max(void);

/* Column-pivoted Householder QR (HQRCP), replaces hqrcp (qr.py:152-204):
 * A[:, perm] = Q R with Q = I - Y T Y^T (Y m x r unit lower trapezoidal, T
 * r x r upper, r = min(m, n)), R m x n in pivoted column order, perm[k] the
 * original index of column k (0-based, the reference's `perm`).  Greedy
 * largest-norm pivoting with the reference's 1e-12 tie window (leftmost),
 * skip rule and norm downdate/recompute.  A is overwritten (working storage).
 * Any m, n: beyond 16384 rows or columns the kernel keeps its per-CTA
 * reflector and permutation in the workspace (utv_dgeqp3_max_dim() now
 * returns INT_MAX; kept for callers that probed the old limit). */
size_t utv_dgeqp3_bufsize(int m, int n);
int utv_dgeqp3_max_dim(void);
int utv_dgeqp3_f64(int m, int n, double* A, long lda, double* R, long ldr, double* Y, long ldy,
                   double* T, long ldt, int* perm, void* work, size_t lwork, void* stream);

/* Device generators (matgen.py:58-91: gen_bie, gen_kahan) and the Frobenius
 * error curve e_k = ||T[k:, k:]||_F, k = 1..n-1 (bench.py:63-72) -> e (device,
 * n-1 doubles), O(mn), fixed-order (bitwise reproducible). */
int utv_dgen_bie(int n, double* A, long lda, void* stream);
int utv_dgen_kahan(int n, double theta, double* A, long lda, void* stream);
size_t utv_dtrailing_fro_bufsize(int m, int n);
int utv_dtrailing_fro(int m, int n, const double* T, long ldt, double* e, void* work, size_t lwork,
                      void* stream);

/* Block utilities for the TSQR tree (LAPACK dlacpy / dlaset semantics):
 * B <- A;  A <- alpha off the diagonal of the uplo ('U', 'L', 'A') part, beta
 * on the diagonal;  A <- alpha diag(d) A (side 'L') or alpha A diag(d) ('R'). */
int utv_dlacpy(int m, int n, const double* A, long lda, double* B, long ldb, void* stream);
int utv_dlaset(char uplo, int m, int n, double alpha, double beta, double* A, long lda,
               void* stream);
int utv_ddiag_scale(char side, int m, int n, const double* d, double alpha, double* A, long lda,
                    void* stream);
/* bytes of device memory <- 0 on the stream (status / mass vectors). */
int utv_zero(void* p, size_t bytes, void* stream);
/* FP32 dlaset (identity / zero initialisation of the fp32 randUTV's U, V). */
int utv_slaset(char uplo, int m, int n, float alpha, float beta, float* A, long lda, void* stream);
/* *flag (device int) <- 1 if any entry of the m x n block is NaN or +-Inf,
 * else 0: the finite test of check_matrix (matrix.py:36-49) on an uploaded
 * copy, so the public API raises ValueError before any RNG draw. */
int utv_dnonfinite(int m, int n, const double* A, long lda, int* flag, void* stream);
/* B (n x m) = A^T (A is m x n).  Used to take a C-order host draw (the
 * reference's gaussian() before its np.asfortranarray copy, matrix.py:52-60)
 * to column-major on the device instead of transposing 2 GiB on the host. */
int utv_dtranspose(int m, int n, const double* A, long lda, double* B, long ldb, void* stream);
/* Zero the strictly upper ('U') or strictly lower ('L') part of A (diagonal kept). */
int utv_dtri_zero(char uplo, int m, int n, double* A, long lda, void* stream);

/* Householder reconstruction for TSQR (row-sharded powerURV):
 * in-place LU without pivoting of (A - diag(s)), m >= n, with
 * s_j = -sign(pivot_j) (sign(0) = +1) chosen on the fly; L (unit lower) below
 * the diagonal, U' on and above it, s (device, n) out.  For an orthonormal Q
 * this gives hqr_full's Y = L and Twy = -U' S L1^{-T} (qr.py:71-100; LAPACK
 * dorhr_col). */
size_t utv_dgetrf_signed_bufsize(int m, int n);
int utv_dgetrf_signed(int m, int n, double* A, long lda, double* s, void* work, size_t lwork,
                      void* stream);

/* B (m x n) <- B * op(A)^{-1} with op(A) upper triangular n x n:
 * (uplo 'U', trans 'N') or (uplo 'L', trans 'T'); diag 'U' = unit. */
size_t utv_dtrsm_bufsize(int m, int n);
int utv_dtrsm_right(char uplo, char trans, char diag, int m, int n, const double* A, long lda,
                    double* B, long ldb, void* work, size_t lwork, void* stream);

/* Q[:, :ncols] = I - Y (T Y[:ncols, :]^T), Y is m x w.
 * Replaces materialize_q (qr.py:124-131) / hqr_thin's Q (qr.py:134-138). */
size_t utv_dorgqr_bufsize(int m, int ncols, int w);
int utv_dorgqr(int m, int ncols, int w, const double* Y, long ldy, const double* T, long ldt,
               double* Q, long ldq, void* work, size_t lwork, void* stream);

/* SVD of an n x n block by one-sided Jacobi: sigma descending, full U, V,
 * reference sign rule.  *status (device int) = sweeps used, -1 = no
 * convergence.  Replaces svd_dense(a, "full") (svd.py:37-58). n <= 1024. */
size_t utv_dgesvj_bufsize(int n);
int utv_dgesvj(int n, const double* A, long lda, double* sigma, double* U, long ldu, double* V,
               long ldv, int* status, void* work, size_t lwork, void* stream);
/* The same with the rounds' orientation chosen explicitly: transpose = 1
 * runs the rotations on A^T (the default of utv_dgesvj: fewer rotations on
 * randUTV's graded triangles), 0 on A (columns of A itself: the convergence
 * test then measures A's own column orthogonality — what the blocked
 * Jacobi of svd_dense beyond n = 1024 needs), -1 the default. */
int utv_dgesvj_ex(int n, const double* A, long lda, double* sigma, double* U, long ldu, double* V,
                  long ldv, int* status, int transpose, void* work, size_t lwork, void* stream);

/* Blocked randUTV, basic variant (randutv_basic, randutv.py:228-235 ->
 * _randutv 110-182, _sample_basic 185-193).
 *  T (m x n): on entry A, on exit T.   U (m x m), V (n x n): on entry I.
 *  G: the reference's Gaussian draws; block i (k_i = m - i*b rows) is the
 *     C-order k_i x b draw, i.e. a b x k_i column-major matrix with leading
 *     dimension ldg (>= b, even), stored at column offset sum_{i'<i} k_i'.
 *  errsq[i]  (device, ceil(n/b)): ||T[lo:mid, lo:]||_F^2 after step i.
 *  trail2[i] (device or NULL):    ||T[mid:, mid:]||_F^2 after step i.
 *  svd_status[i] (device int): Jacobi sweeps of step i (-1 = no convergence). */
size_t utv_randutv_basic_bufsize(int m, int n, int b, int q);
int utv_randutv_basic_f64(int m, int n, int b, int q, double* T, long ldt, double* U, long ldu,
                          double* V, long ldv, const double* G, long ldg, double* errsq,
                          double* trail2, int* svd_status, void* work, size_t lwork,
                          void* stream);

/* Steps [i0, i1) of utv_randutv_basic_f64 (same workspace; G = the block of
 * step i0 at column 0).  Lets the host draw later steps' Gaussian blocks
 * while earlier steps run; consecutive ranges give the same bits as one call. */
int utv_randutv_basic_steps_f64(int i0, int i1, int m, int n, int b, int q, double* T, long ldt,
                                double* U, long ldu, double* V, long ldv, const double* G, long ldg,
                                double* errsq, double* trail2, int* svd_status, void* work,
                                size_t lwork, void* stream);
/* The same with the SVD pipeline carried across range boundaries: carry
 * bit 0 = the previous range (steps [.., i0)) was called with bit 1 and left
 * step i0-1's b x b SVD in flight; bit 1 = leave step i1-1's SVD in flight
 * (its rotations of U, V and T columns [(i1-1) b, i1 b) are then applied by
 * the next range, so only columns < (i1-1) b are final on return).  Same
 * bits as one utv_randutv_basic_f64 call.  Replaces the per-step loop of
 * _randutv (randutv.py:110-182) split into host-fed groups. */
int utv_randutv_basic_steps_carry_f64(int i0, int i1, int carry, int m, int n, int b, int q,
                                      double* T, long ldt, double* U, long ldu, double* V, long ldv,
                                      const double* G, long ldg, double* errsq, double* trail2,
                                      int* svd_status, void* work, size_t lwork, void* stream);

/* One step i (0-based) of blocked randUTV — the host loop of the boosted
 * (Algorithm 2) and partial variants (randutv_boosted / randutv_partial,
 * randutv.py:130-139, 196-264), which may stop early on the tracked error.
 * boosted = 0: basic sampler (G = this step's b x k_i block).  boosted = 1:
 * oversampled sampler with recycling; G = (b+p) x m at i = 0, b x k_i after.
 * *carried (host, in/out): carried columns of the recycled block (0 at i=0).
 * *is_final (host, out): 1 when the step was the final dense SVD. */
size_t utv_randutv_step_bufsize(int m, int n, int b, int p, int q);
int utv_randutv_step_f64(int i, int m, int n, int b, int p, int q, int boosted, double* T, long ldt,
                         double* U, long ldu, double* V, long ldv, const double* G, long ldg,
                         double* errsq, double* trail2, int* svd_status, int* carried,
                         int* is_final, void* work, size_t lwork, void* stream);

/* fp32 variant of randutv_basic (BASELINE C5): T, U, V, G fp32; every GEMM
 * 3xTF32 on tcgen05; panel QRs and the b x b Jacobi SVD in fp64 on converted
 * panels.  m, n, b and all leading dimensions multiples of 4. */
size_t utv_randutv_basic_f32_bufsize(int m, int n, int b, int q);
int utv_randutv_basic_f32(int m, int n, int b, int q, float* T, long ldt, float* U, long ldu,
                          float* V, long ldv, const float* G, long ldg, double* errsq,
                          double* trail2, int* svd_status, void* work, size_t lwork,
                          void* stream);

/* powerURV (power_urv_from_sample, powerurv.py:41-72; power_urv :75-79;
 * rurv :82-84 with q = 0).  A (m x n, read only), G (n x n, read only).
 * Outputs Uq = (Uy m x n, Ut n x n), R (m x n), Vq = (Vy n x n, Vt n x n). */
size_t utv_powerurv_bufsize(int m, int n, int q);
int utv_powerurv_f64(int m, int n, int q, const double* A, long lda, const double* G, long ldg,
                     double* Uy, long lduy, double* Ut, long ldut, double* R, long ldr,
                     double* Vy, long ldvy, double* Vt, long ldvt, void* work, size_t lwork,
                     void* stream);
/* Same, plus two cudaEvent_t (each may be null): vq_ready is recorded once
 * Vq.Y and Vq.Twy are final, before A Q(Vq) and the final QR; r_ready once
 * R and Uq.Y are final, before Uq's dense triangle is built — so the caller
 * can copy results out while the factorisation finishes. */
int utv_powerurv_f64_ev(int m, int n, int q, const double* A, long lda, const double* G, long ldg,
                        double* Uy, long lduy, double* Ut, long ldut, double* R, long ldr,
                        double* Vy, long ldvy, double* Vt, long ldvt, void* work, size_t lwork,
                        void* stream, void* vq_ready, void* r_ready);
/* power_urv (powerurv.py:75-79 -> power_urv_from_sample :41-72, its first
 * product :64 supplied): q >= 1 and Yhat = A G given by the caller
 * (m x n, device, read only) instead of G: the public power_urv
 * forms it as K-chunked products while G is still being drawn on the host
 * (row block by row block of the reference's C-order draw), so the host
 * RNG overlaps the device. */
int utv_powerurv_f64_yhat(int m, int n, int q, const double* A, long lda, const double* Yhat0,
                          long ldy0, double* Uy, long lduy, double* Ut, long ldut, double* R,
                          long ldr, double* Vy, long ldvy, double* Vt, long ldvt, void* work,
                          size_t lwork, void* stream, void* vq_ready, void* r_ready);

/* powerURV with progressive results: G (or, for q >= 1, Yhat0 = A G instead
 * of G — pass the other as NULL) and ncols_ev = ceil(n / 256) events per
 * array (each array may be NULL).  r_cols[j] is recorded once columns
 * [256 j, 256 j + 256) of R and Uq.Y are final — during the final QR,
 * panel by panel — and t_cols[j] once the same columns of Uq.Twy are: the
 * dense triangle's column blocks are merged on a low-priority side stream
 * as the panels complete (powerurv.py:70-71 + qr.py:63-68), so a caller can
 * copy every output out while the factorisation still runs.  vq_ready as
 * in utv_powerurv_f64_ev.  progress_cb (optional, void cb(void* ctx, int
 * kind, int index)) is called on the calling host thread right after each
 * progress event's record has been ENQUEUED (kind 0: vq_ready, 1: r_cols[index],
 * 2: t_cols[index]): the launch queue holds the calling thread for most of
 * the device run, so copy jobs must be handed to another thread from there. */
int utv_powerurv_f64_cols(int m, int n, int q, const double* A, long lda, const double* G, long ldg,
                          const double* Yhat0, long ldy0, double* Uy, long lduy, double* Ut,
                          long ldut, double* R, long ldr, double* Vy, long ldvy, double* Vt,
                          long ldvt, void* work, size_t lwork, void* stream, void* vq_ready,
                          int ncols_ev, void* const* r_cols, void* const* t_cols,
                          void* progress_cb, void* progress_ctx);

/* ---- Row-sharded powerURV over several GPUs (BASELINE C4) ----
 * The reference has no multi-GPU path (powerurv.py:41-72 is one process);
 * this is its SPMD form: one process (or, for emulation, one host thread)
 * per rank, rank i owning the row block A_i (m_i x n, m_i >= n) and the
 * same n x n G.  Collectives run on the caller's stream through a
 * utv_comm_t: NCCL (libnccl is dlopen'ed, the process's loaded copy
 * preferred; UTV_NCCL_LIB overrides) or an in-process local group of P
 * ranks (threads; device-to-device copies + a host barrier; rank-order
 * sums).  Per power round: local GEMM, TSQR (allgather of n x n R's),
 * local GEMM + allreduce of the n x n Y, redundant hqr_full(Y); final TSQR
 * + Householder reconstruction (rank 0 factors the top n x n block and
 * broadcasts it; every rank solves for its own rows).
 *
 * utv_comm_nccl_unique_id: 128-byte ncclUniqueId (rank 0; ship it to the
 *   other ranks out of band, e.g. torch.distributed.broadcast_object_list).
 * utv_comm_init_nccl: collective over all ranks; binds the current device.
 * utv_comm_from_nccl: borrow an existing ncclComm_t (not destroyed).
 * utv_comm_init_local: nranks handles of one in-process group (comms[r] is
 *   rank r; drive each from its own host thread and stream).
 * Returns -1004 (UTV_ERR_COMM) when NCCL is unavailable or a collective fails. */
typedef struct utv_comm_s utv_comm_s;
typedef utv_comm_s* utv_comm_t;
int utv_comm_nccl_available(void);
int utv_comm_nccl_unique_id(void* id128);
int utv_comm_init_nccl(const void* id128, int nranks, int rank, utv_comm_t* comm);
int utv_comm_from_nccl(void* nccl_comm, utv_comm_t* comm);
int utv_comm_init_local(int nranks, utv_comm_t* comms);
int utv_comm_rank(const utv_comm_s* comm);
int utv_comm_size(const utv_comm_s* comm);
int utv_comm_destroy(utv_comm_t comm);
/* The three collectives of the sharded path, exposed for tests: in-place
 * sum; recv = rank-ordered concatenation of count doubles each; in place. */
int utv_comm_allreduce_sum_f64(utv_comm_t comm, double* buf, size_t count, void* stream);
int utv_comm_allgather_f64(utv_comm_t comm, const double* send, double* recv, size_t count,
                           void* stream);
int utv_comm_broadcast_f64(utv_comm_t comm, double* buf, size_t count, int root, void* stream);

/* Row-sharded power_urv_from_sample (powerurv.py:41-72), SPMD: every rank
 * calls with its m_local rows of A, the same n, q and G.  Outputs: this
 * rank's rows of Uq.Y (Uy, m_local x n) and the replicated Uq.Twy (Ut),
 * R (n x n; rows n.. of the reference's m x n R are zero), Vq.Y (Vy) and
 * Vq.Twy (Vt), all n x n.  chunk_rows (<= 0: the panel-QR limit,
 * utv_dgeqrf_rows_max) caps the local TSQR leaves.  The ranks first agree
 * on (n, q, argument validity) with one 4-double allreduce and a stream
 * synchronisation; a rank with an invalid argument returns its own code,
 * the others -1004.  The Householder reconstruction does not reproduce
 * hqr_full's skip rule (tau = 0) for exactly dependent columns. */
size_t utv_powerurv_sharded_bufsize(int m_local, int n, int nranks, int chunk_rows);
int utv_powerurv_sharded_f64(utv_comm_t comm, int m_local, int n, int q, const double* A, long lda,
                             const double* G, long ldg, double* Uy, long lduy, double* Ut,
                             long ldut, double* R, long ldr, double* Vy, long ldvy, double* Vt,
                             long ldvt, int chunk_rows, void* work, size_t lwork, void* stream);

/* Instrumentation (no reference counterpart).
 * utv_launch_count: number of libutvb200 kernel launches since load.
 * utv_profile_begin/end: bracket launches with CUDA events; end() syncs the
 * device and fills per-category totals (categories: 0 DMMA GEMM, 1 split-K
 * reduce, 2 panel-QR leaf, 3 Jacobi rounds, 4 Jacobi finish, 5 small ops,
 * 6 3xTF32 GEMM, 7 column-pivoted QR); returns the number of categories.
 * utv_profile_busy: per-category union of the launch intervals across all
 * streams (ms) of the last utv_profile_end — concurrent launches counted once. */
long long utv_launch_count(void);
void utv_profile_begin(void);
int utv_profile_end(double* ms, double* flops, double* bytes, long long* count);
int utv_profile_busy(double* busy_ms);

#ifdef __cplusplus
}
#endif
#endif /* UTV_B200_H */
