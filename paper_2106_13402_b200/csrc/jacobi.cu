// K6: one-sided (Hestenes) Jacobi SVD of the small b x b block.
//
// Replaces svd_dense(r_panel[:b,:], "full") (randutv.py:151 -> svd.py:37-58,
// LAPACK gesdd in the reference) and the final narrow-block SVD
// (randutv.py:166).  Output contract of the reference:
//   * sigma descending, >= 0
//   * full U, V orthogonal
//   * sign rule: each pair flipped so that the first largest-|.| entry of the
//     V column is positive (svd.py:53-57)
//   * exactly zero block -> U = V = I (gesdd behaviour)
//
// B200 design: block one-sided Jacobi.  Columns are split into 2G blocks of
// W=16; a cooperative grid of G CTAs processes the G block pairs of one
// round-robin round concurrently (each pair resident in shared memory, one
// warp per column pair, warp-shuffle dot products), then grid-syncs.  A and
// the accumulated V live in an L2-resident workspace between rounds.  A
// second kernel forms sigma, sorts, normalises U = A V / sigma, completes
// null columns of U by CGS2 against the standard basis, and applies the sign
// rule.
#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace jac {
constexpr int MAX_SWEEPS = 40;
constexpr double EPS = 2.220446049250313e-16;

struct Args {
  double* A;   // n x npad, ld
  double* V;   // n x npad, ld
  long ld;
  int n, nblk;  // nblk = 2G blocks of W columns
  double tol;
  int* rot;     // [MAX_SWEEPS] rotation counters (zeroed)
  int* status;  // sweeps used / -1
  unsigned* ctr;
};

__device__ inline void round_pair(int N, int r, int k, int* p, int* q) {
  // circle method on N players: player N-1 fixed
  if (k == 0) {
    *p = N - 1;
    *q = r;
  } else {
    *p = (r + k) % (N - 1);
    *q = (r - k + (N - 1)) % (N - 1);
  }
}

// Rotate columns x, y (length n, smem) so that they become orthogonal.
// Returns true when a rotation was applied.  Executed by one full warp; the
// three dot products share one interleaved shuffle tree.
__device__ __forceinline__ bool rotate_pair(double* __restrict__ ax, double* __restrict__ ay,
                                            double* __restrict__ vx, double* __restrict__ vy,
                                            int n, double tol2) {
  const int lane = threadIdx.x & 31;
  double alpha = 0.0, beta = 0.0, gamma = 0.0;
  for (int i = lane; i < n; i += 32) {
    const double x = ax[i], y = ay[i];
    alpha = fma(x, x, alpha);
    beta = fma(y, y, beta);
    gamma = fma(x, y, gamma);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    alpha += __shfl_xor_sync(0xffffffffu, alpha, o);
    beta += __shfl_xor_sync(0xffffffffu, beta, o);
    gamma += __shfl_xor_sync(0xffffffffu, gamma, o);
  }
  // |gamma| > tol * sqrt(alpha * beta), evaluated without square roots when
  // the product is safely representable.
  const double ab = alpha * beta;
  bool rot;
  if (ab > 1e-280 && ab < 1e280) rot = gamma * gamma > tol2 * ab;
  else rot = fabs(gamma) > sqrt(tol2) * sqrt(alpha) * sqrt(beta);
  if (gamma == 0.0 || !rot) return false;
  const double zeta = (beta - alpha) / (2.0 * gamma);
  double t;
  if (fabs(zeta) > 1e150)
    t = 0.5 / zeta;
  else
    t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
  const double c = rsqrt(fma(t, t, 1.0));
  const double s = c * t;
  for (int i = lane; i < n; i += 32) {
    const double x = ax[i], y = ay[i];
    ax[i] = fma(c, x, -s * y);
    ay[i] = fma(s, x, c * y);
    const double u = vx[i], w = vy[i];
    vx[i] = fma(c, u, -s * w);
    vy[i] = fma(s, u, c * w);
  }
  return true;
}

// Persistent cooperative kernel: G CTAs, 2G blocks of W columns.  Every round
// each CTA owns one block pair (circle-method tournament over blocks) and
// rotates only the W^2 cross pairs (W sub-rounds of W disjoint pairs, one
// warp per pair); the intra-block pairs are swept once per sweep in round 0.
// Sequential sub-rounds per sweep: (W-1) + (2G-1) W  ~ n.
template <int W>
__global__ void __launch_bounds__(32 * W, 1) jacobi_rounds_kernel(Args a) {
  extern __shared__ double sm[];
  const int n = a.n;
  const int ldS = n;
  double* As = sm;                        // 2W columns
  double* Vs = sm + (size_t)2 * W * ldS;  // 2W columns
  __shared__ int s_rot;
  const int G = gridDim.x, g = blockIdx.x;
  const int N = a.nblk;
  const int warp = threadIdx.x >> 5;
  const double tol2 = a.tol * a.tol;
  unsigned bar = 0;
  int sweep = 0;
  for (; sweep < MAX_SWEEPS; ++sweep) {
    for (int r = 0; r < N - 1; ++r) {
      int bp, bq;
      round_pair(N, r, g, &bp, &bq);
      // load the two blocks (16-byte vector loads; n is padded to even)
      const int n2 = n >> 1;
      for (int idx = threadIdx.x; idx < 2 * W * n2; idx += 32 * W) {
        const int c = idx / n2, i = (idx - c * n2) * 2;
        const int gc = (c < W ? bp * W + c : bq * W + (c - W));
        const double2 va = __ldcg((const double2*)&a.A[i + (long)gc * a.ld]);
        const double2 vv = __ldcg((const double2*)&a.V[i + (long)gc * a.ld]);
        *(double2*)&As[c * ldS + i] = va;
        *(double2*)&Vs[c * ldS + i] = vv;
      }
      if (threadIdx.x == 0) s_rot = 0;
      __syncthreads();
      int nrot = 0;
      if (r == 0) {
        // intra-block pairs of both resident blocks: round robin on W columns
        for (int sr = 0; sr < W - 1; ++sr) {
          const int blk = warp / (W / 2), k = warp % (W / 2);
          int x, y;
          round_pair(W, sr, k, &x, &y);
          x += blk * W;
          y += blk * W;
          nrot += rotate_pair(As + x * ldS, As + y * ldS, Vs + x * ldS, Vs + y * ldS, n, tol2);
          __syncthreads();
        }
      }
      // cross pairs (i, W + (i + s) mod W)
      for (int s = 0; s < W; ++s) {
        const int x = warp, y = W + ((warp + s) % W);
        nrot += rotate_pair(As + x * ldS, As + y * ldS, Vs + x * ldS, Vs + y * ldS, n, tol2);
        __syncthreads();
      }
      if ((threadIdx.x & 31) == 0 && nrot) atomicAdd(&s_rot, nrot);
      __syncthreads();
      if (threadIdx.x == 0 && s_rot) atomicAdd(&a.rot[sweep], s_rot);
      for (int idx = threadIdx.x; idx < 2 * W * n2; idx += 32 * W) {
        const int c = idx / n2, i = (idx - c * n2) * 2;
        const int gc = (c < W ? bp * W + c : bq * W + (c - W));
        *(double2*)&a.A[i + (long)gc * a.ld] = *(const double2*)&As[c * ldS + i];
        *(double2*)&a.V[i + (long)gc * a.ld] = *(const double2*)&Vs[c * ldS + i];
      }
      ++bar;
      if (G > 1) grid_barrier(a.ctr, bar * G);
      else __syncthreads();
    }
    if (__ldcg(&a.rot[sweep]) == 0) break;
  }
  if (g == 0 && threadIdx.x == 0) *a.status = (sweep < MAX_SWEEPS) ? sweep + 1 : -1;
}

__device__ inline double block_reduce_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
  return t;
}

// Single CTA: sigma, sort (stable, descending), U = A/sigma, null-column
// completion (CGS2 against e_i), sign rule.  n <= 1024.
__global__ void __launch_bounds__(1024) jacobi_finish_kernel(const double* __restrict__ A,
                                                            const double* __restrict__ V,
                                                            long ld, int n, double* sigma,
                                                            double* U, long ldu, double* Vo,
                                                            long ldv, double* scratch,
                                                            int sign_on_u) {
  extern __shared__ double sm[];
  double* sig = sm;            // n
  int* perm = (int*)(sig + n);  // n
  double* uvec = (double*)(perm + n + (n & 1));  // n
  double* coef = uvec + n;     // n
  __shared__ double red[32];
  __shared__ int s_nzero;
  const int t = threadIdx.x;
  // column norms (one warp per column)
  const int warp = t >> 5, lane = t & 31, nw = blockDim.x >> 5;
  for (int c = warp; c < n; c += nw) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) {
      const double x = A[i + (long)c * ld];
      s = fma(x, x, s);
    }
    s = warp_sum(s);
    if (lane == 0) sig[c] = sqrt(s);
  }
  __syncthreads();
  // stable descending rank
  for (int c = t; c < n; c += blockDim.x) {
    const double v = sig[c];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
      const double w = sig[i];
      rank += (w > v) || (w == v && i < c);
    }
    perm[rank] = c;
  }
  if (t == 0) s_nzero = 0;
  __syncthreads();
  // permuted outputs; U = A / sigma for nonzero columns
  for (int k = t; k < n; k += blockDim.x) {
    sigma[k] = sig[perm[k]];
    if (sig[perm[k]] == 0.0) atomicAdd(&s_nzero, 1);
  }
  for (int idx = t; idx < n * n; idx += blockDim.x) {
    const int k = idx / n, i = idx - k * n;
    const int c = perm[k];
    const double s = sig[c];
    Vo[i + (long)k * ldv] = V[i + (long)c * ld];
    U[i + (long)k * ldu] = (s > 0.0) ? A[i + (long)c * ld] / s : 0.0;
  }
  __syncthreads();
  // complete null columns of U: CGS2 of e_cand against all filled columns
  const int nz = s_nzero;
  int cand = 0;
  for (int k = n - nz; k < n; ++k) {
    while (true) {
      for (int i = t; i < n; i += blockDim.x) uvec[i] = (i == cand) ? 1.0 : 0.0;
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int l = t; l < k; l += blockDim.x) {  // coef_l = U[:, l]^T u
          double s = 0.0;
          for (int i = 0; i < n; ++i) s = fma(U[i + (long)l * ldu], uvec[i], s);
          coef[l] = s;
        }
        __syncthreads();
        for (int i = t; i < n; i += blockDim.x) {
          double s = uvec[i];
          for (int l = 0; l < k; ++l) s = fma(-U[i + (long)l * ldu], coef[l], s);
          uvec[i] = s;
        }
        __syncthreads();
      }
      double nrm2 = 0.0;
      for (int i = t; i < n; i += blockDim.x) nrm2 = fma(uvec[i], uvec[i], nrm2);
      nrm2 = block_reduce_sum(nrm2, red);
      ++cand;
      if (nrm2 > 0.25 || cand >= n) {
        const double inv = 1.0 / sqrt(nrm2);
        for (int i = t; i < n; i += blockDim.x) U[i + (long)k * ldu] = uvec[i] * inv;
        __syncthreads();
        break;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  // sign rule: first argmax |V[:, k]| must be positive (V of the caller's
  // matrix: the U output here when the rounds ran on its transpose)
  const double* Sg = sign_on_u ? U : Vo;
  const long lds = sign_on_u ? ldu : ldv;
  for (int k = warp; k < n; k += nw) {
    double best = -1.0;
    int bi = n;
    for (int i = lane; i < n; i += 32) {
      const double v = fabs(Sg[i + (long)k * lds]);
      if (v > best) { best = v; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const bool flip = Sg[bi + (long)k * lds] < 0.0;
    __syncwarp();
    if (flip)
      for (int i = lane; i < n; i += 32) {
        Vo[i + (long)k * ldv] = -Vo[i + (long)k * ldv];
        U[i + (long)k * ldu] = -U[i + (long)k * ldu];
      }
  }
}
}  // namespace jac

// Column-block width: the resident block pair (A and V, 2W columns each) must
// fit the 200 KB smem budget: 4 W n 8 bytes.
static inline int jac_width(int n) {
  const int ne = n + (n & 1);
  static const int forced = [] {  // tuning knob: UTV_JAC_W = 4 / 8 / 16
    const char* e = getenv("UTV_JAC_W");
    return e ? atoi(e) : 0;
  }();
  if ((forced == 4 || forced == 8 || forced == 16) && (size_t)4 * forced * ne * 8 <= 200 * 1024)
    return forced;
  if ((size_t)4 * 16 * ne * 8 <= 200 * 1024) return 16;
  if ((size_t)4 * 8 * ne * 8 <= 200 * 1024) return 8;
  return 4;
}

static inline int jac_blocks(int n, int W) {
  int nb = (n + W - 1) / W;
  if (nb & 1) nb++;
  if (nb < 2) nb = 2;
  return nb;
}

size_t gesvj_ws_doubles(int n) {
  const long ld = round_up(n, 4);
  const int W = jac_width(n);
  const long npad = (long)jac_blocks(n, W) * W;
  return 2 * ld * npad + 2048 + (size_t)jac::MAX_SWEEPS + 64 + 4 * 32;
}

static bool g_jac_attr = false;

int gesvj(Mat A, double* sigma, Mat U, Mat V, double* ws, size_t ws_doubles, int* status_dev,
          cudaStream_t st) {
  return gesvj_ex(A, sigma, U, V, ws, ws_doubles, status_dev, st, -1);
}

// orient: -1 = the default (UTV_JAC_TRANSPOSE, on), 0 = rounds on A, 1 = on A^T.
int gesvj_ex(Mat A, double* sigma, Mat U, Mat V, double* ws, size_t ws_doubles, int* status_dev,
             cudaStream_t st, int orient) {
  const int n = A.rows;
  if (n <= 0) return UTV_OK;
  if (n > 1024) return -1;
  const long ld = round_up(n, 4);
  const int W = jac_width(n);
  const int nblk = jac_blocks(n, W);
  const long npad = (long)nblk * W;
  Arena ar{(char*)ws, ws_doubles * sizeof(double), 0};
  double* Aw = ar.take(ld * npad);
  double* Vw = ar.take(ld * npad);
  double* ctl = ar.take(jac::MAX_SWEEPS + 64);
  double* scratch = ar.take(1024);
  if (!scratch) return UTV_ERR_WORKSPACE;
  // rows are padded to an even count (16-byte vector moves); padding is zero
  const int ne = n + (n & 1);
  // The rounds run on A^T (UTV_JAC_TRANSPOSE, default on): for the graded
  // upper-triangular blocks randUTV hands in, the columns of R^T start much
  // closer to orthogonal, so far fewer rotations fire (256^2 Gaussian-decay
  // block 6.2 -> 2.8 ms, tools/jacobi_transpose_probe.py).  A^T = W S X^T
  // gives A = X S W^T: the outputs swap (U <- normalised columns, with the
  // null-column completion, goes to V; W goes to U) and the sign rule reads V.
  static const bool tr_default = [] {
    const char* e = getenv("UTV_JAC_TRANSPOSE");
    return e ? atoi(e) != 0 : true;
  }();
  const bool tr = orient < 0 ? tr_default : orient != 0;
  UTV_CHECK(set_zero(Aw, ld, (int)ld, (int)npad, st));
  if (tr) UTV_CHECK(transpose(A.p, A.ld, Aw, ld, n, n, st));
  else UTV_CHECK(copy_mat(A.p, A.ld, Aw, ld, n, n, st));
  UTV_CHECK(set_zero(Vw, ld, (int)ld, (int)npad, st));
  UTV_CHECK(set_identity(Vw, ld, n, n, st));
  UTV_CUDA(cudaMemsetAsync(ctl, 0, (jac::MAX_SWEEPS + 64) * sizeof(double), st));
  jac::Args a;
  a.A = Aw; a.V = Vw; a.ld = ld;
  a.n = ne; a.nblk = nblk;
  a.tol = 4.0 * sqrt((double)n) * jac::EPS;
  a.rot = (int*)ctl;
  a.ctr = (unsigned*)(ctl + jac::MAX_SWEEPS);
  a.status = status_dev;
  const int G = nblk / 2;
  const size_t smem = (size_t)4 * W * ne * sizeof(double);
  if (!g_jac_attr) {
    for (auto f : {jac::jacobi_rounds_kernel<16>, jac::jacobi_rounds_kernel<8>, jac::jacobi_rounds_kernel<4>})
      UTV_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    UTV_CUDA(cudaFuncSetAttribute(jac::jacobi_finish_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    g_jac_attr = true;
  }
  if (smem > 200 * 1024) return -1;
  {
  ProfScope ps(PROF_JACOBI, 0.0, 0.0, st);
  void* kfn = W == 16 ? (void*)jac::jacobi_rounds_kernel<16>
              : (W == 8 ? (void*)jac::jacobi_rounds_kernel<8> : (void*)jac::jacobi_rounds_kernel<4>);
  void* args[] = {&a};
  if (G > 1) {
    UTV_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(32 * W), args, smem, st));
  } else {
    UTV_CUDA(cudaLaunchKernel(kfn, dim3(1), dim3(32 * W), args, smem, st));
  }
  }
  const size_t smem2 = (size_t)4 * (n + 2) * sizeof(double);
  ProfScope ps2(PROF_JFINISH, 0.0, 0.0, st);
  if (tr)
    jac::jacobi_finish_kernel<<<1, 1024, smem2, st>>>(Aw, Vw, ld, n, sigma, V.p, V.ld, U.p, U.ld,
                                                      scratch, 1);
  else
    jac::jacobi_finish_kernel<<<1, 1024, smem2, st>>>(Aw, Vw, ld, n, sigma, U.p, U.ld, V.p, V.ld,
                                                      scratch, 0);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

}  // namespace utv
