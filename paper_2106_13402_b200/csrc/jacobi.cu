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
// B200 design: block one-sided Jacobi in Gram form.  Columns are split into
// 2P blocks of 16; every round of the circle-method tournament a thread-block
// cluster of C CTAs owns one block pair, CTA r holding a slice of R = ne / C
// rows of the pair's 32 columns of A and V in shared memory.  The cluster
// forms the pair's 32 x 32 Gram matrix (DMMA partials summed over DSMEM),
// runs the rotation sub-rounds on it (a pipelined rotation warp computes the
// next sub-round's rotations while 16 warps apply the current one to G and
// to the accumulated rotation J; no dot products), and applies J to its A and
// V rows (DMMA); A and V live in an L2-resident workspace between rounds
// (grid barrier).  The rounds were smem-bandwidth bound when every rotation
// re-read and rewrote both columns (tools/jacobi_probe.cu: 1.76 us per
// sub-round at n = 256, now ~0.55 us).  A second kernel
// forms sigma, sorts, normalises U = A V / sigma, completes null columns of U
// by CGS2 against the standard basis, and applies the sign rule.
#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace jac {
// Diagnostics: build with -DJAC_PROBE (tools/jacobi_probe.cu) to accumulate
// CTA 0's per-phase %globaltimer durations into g_probe.
#ifdef JAC_PROBE
__device__ unsigned long long g_probe[8];
__device__ unsigned long long g_probe2[8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
#define JPROBE(k)                                  \
  if (blockIdx.x == 0 && threadIdx.x == 0) {       \
    const unsigned long long now_ = gtime();       \
    g_probe[k] += now_ - probe_last;               \
    probe_last = now_;                             \
  }
#else
#define JPROBE(k)
#endif
constexpr int MAX_SWEEPS = 40;
constexpr double EPS = 2.220446049250313e-16;

constexpr int JW = 16;       // column block width
constexpr int JC = 2 * JW;   // resident block pair = one warp's lanes
constexpr int GP = JC + 1;   // odd pitch of the smem row-major tiles

struct Args {
  double* A;   // ne x npad, ld (rows >= n zero)
  double* V;   // ne x npad, ld
  long ld;
  int ne, nblk;  // padded rows (a multiple of 2 * cluster size); 2P blocks of JW columns
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

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ double ld_dsmem(const double* p, unsigned rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
  return v;
}

// Rotation of columns (x, y) that annihilates gamma = a_x^T a_y, from the
// Gram entries (alpha = |a_x|^2, beta = |a_y|^2): a_x' = c a_x - s a_y,
// a_y' = s a_x + c a_y, t = s / c the smaller root of t^2 + 2 zeta t - 1 = 0,
// zeta = (beta - alpha) / (2 gamma).  Returns false when
// |gamma| <= tol sqrt(alpha beta) (the convergence test).  With
// d = beta - alpha, g = 2 gamma, h = sqrt(d^2 + g^2):
//   c = (h + |d|) / sqrt(2 h (h + |d|)),  s = sign(d) g / sqrt(2 h (h + |d|))
// (c^2 + s^2 = 1, no cancellation) — one sqrt and one rsqrt on the
// dependent chain: 294 cycles against 513 for the zeta form with its two
// divisions (tools/rot_bench.cu); the rotation is the critical path of
// every sub-round.  (d, g) are rescaled exactly by a power of two when out
// of the safe range.
__device__ __forceinline__ bool rotation(double alpha, double beta, double gamma, double tol2,
                                         double* c, double* s) {
  const double ab = alpha * beta;
  bool rot;
  if (ab > 1e-280 && ab < 1e280) rot = gamma * gamma > tol2 * ab;
  else rot = fabs(gamma) > sqrt(tol2) * sqrt(alpha) * sqrt(beta);
  if (gamma == 0.0 || !rot) return false;
  double d = beta - alpha, g = 2.0 * gamma;
  const double m = fmax(fabs(d), fabs(g));
  if (m > 1e150 || m < 1e-150) {
    const int e = (int)((__double_as_longlong(m) >> 52) & 0x7ff);  // biased exponent, m normal
    const double sc = __longlong_as_double((long long)(2046 - e) << 52);  // 2^(1023 - e), exact
    d *= sc;
    g *= sc;
  }
  const double h = sqrt(fma(d, d, g * g));
  const double u = h + fabs(d);
  const double q = rsqrt(2.0 * h * u);
  *c = u * q;
  *s = (d < 0.0 ? -g : g) * q;
  return true;
}

// Pair p (0..JW-1) of a sub-round.  Intra (round 0 of a sweep): circle method
// inside each of the two blocks, JW/2 pairs each.  Cross step s: (p, JW + (p + s) mod JW).
__device__ __forceinline__ void pair_of(bool cross, int step, int p, int* x, int* y) {
  if (cross) {
    *x = p;
    *y = JW + ((p + step) % JW);
  } else {
    const int blk = p / (JW / 2), k = p % (JW / 2);
    round_pair(JW, step, k, x, y);
    *x += blk * JW;
    *y += blk * JW;
  }
}

// Sub-round schedule: NSUB = (JW - 1) intra + JW cross sub-rounds.  Per
// sub-round u and index i (0..JC-1): pair id (bits 0-3), role y (bit 4),
// partner index (bits 5-9); the pair list (x, y) per u.
constexpr int NSUB = 2 * JW - 1;

struct Sched {
  unsigned short idx[NSUB][JC];
  unsigned char px[NSUB][JW], py[NSUB][JW];
};

__device__ __forceinline__ void build_sched(Sched* sc) {
  for (int t = threadIdx.x; t < NSUB * JW; t += blockDim.x) {
    const int u = t / JW, p = t % JW;
    int x, y;
    pair_of(u >= JW - 1, u >= JW - 1 ? u - (JW - 1) : u, p, &x, &y);
    sc->px[u][p] = (unsigned char)x;
    sc->py[u][p] = (unsigned char)y;
    sc->idx[u][x] = (unsigned short)(p | (y << 5));
    sc->idx[u][y] = (unsigned short)(p | 16 | (x << 5));
  }
}

// The 2 x 2 block update of Gn = Q^T G Q: rows (i, partner i2) x columns
// (xq, yq) of G -> row i of the block of Gn.  rp / rq: rotations of the
// row / column pairs (identity if not rotated), yi: i is the y of its pair,
// zero: the block is the annihilated pair's own (that entry is set to 0).
__device__ __forceinline__ void gram_rot2(double a0, double a1, double b0, double b1, double2 rp,
                                          double2 rq, int yi, bool zero, double* g0, double* g1) {
  // row i of R_p^T M (R = [c s; -s c]): x-row c m_x - s m_y, y-row s m_x + c m_y
  double n0, n1;
  if (yi) {
    n0 = fma(rp.y, b0, rp.x * a0);
    n1 = fma(rp.y, b1, rp.x * a1);
  } else {
    n0 = fma(rp.x, a0, -rp.y * b0);
    n1 = fma(rp.x, a1, -rp.y * b1);
  }
  *g0 = fma(n0, rq.x, -n1 * rq.y);
  *g1 = fma(n0, rq.y, n1 * rq.x);
  if (zero) {
    if (yi) *g0 = 0.0;
    else *g1 = 0.0;
  }
}

// Look-ahead table: for sub-round u >= 1 and pair p, the pair (x, y) of u
// and, for x and y, their pair / role / partner in sub-round u - 1
// (5 + 5 + 2 x 10 bits), so the rotation warp forms the three Gram entries
// of every pair of u from G_{u-1} without dependent index loads.
__device__ __forceinline__ void build_lookahead(const Sched* sc, unsigned* la) {
  for (int t = threadIdx.x; t < NSUB * JW; t += blockDim.x) {
    const int u = t / JW, pp = t % JW;
    if (u == 0) continue;
    const unsigned x = sc->px[u][pp], y = sc->py[u][pp];
    const unsigned ix = sc->idx[u - 1][x] & 0x3ff, iy = sc->idx[u - 1][y] & 0x3ff;
    la[t] = x | (y << 5) | (ix << 10) | (iy << 20);
  }
}

// Diagonal of the rotated 2 x 2 pair block [[al, ga], [ga, be]] (the
// update threads' arithmetic for those entries, G symmetric).
__device__ __forceinline__ void pair_diag(double al, double be, double ga, double2 r, bool rot, double* dx,
                                          double* dy) {
  if (!rot) {
    *dx = al;
    *dy = be;
    return;
  }
  double g0, g1, h0, h1;
  gram_rot2(al, ga, ga, be, r, r, 0, true, &g0, &g1);
  gram_rot2(ga, be, al, ga, r, r, 1, true, &h0, &h1);
  *dx = g0;
  *dy = h1;
}

// Rotation warp, lane p: rotation of pair p of sub-round u + 1 from
// G_u = Q_u^T G_{u-1} Q_u.  The diagonal entries come from the lanes that
// rotated them in sub-round u (their registers dX, dY; shuffles), so only
// the off-diagonal gamma is formed from G_{u-1} (4 loads).  Updates
// (cK, sK, rK, dX, dY) to sub-round u + 1.
__device__ __forceinline__ void rotate_next(unsigned w, const double* __restrict__ G, double tol2,
                                            double* cK, double* sK, bool* rK, double* dX, double* dY) {
  const int x = w & 31, y = (w >> 5) & 31;
  const int px = (w >> 10) & 15, rx = (w >> 14) & 1, x2 = (w >> 15) & 31;
  const int py = (w >> 20) & 15, ry = (w >> 24) & 1, y2 = (w >> 25) & 31;
  const int cy0 = ry ? y2 : y, cy1 = ry ? y : y2;
  const double m0 = G[x * GP + cy0], m1 = G[x * GP + cy1], m2 = G[x2 * GP + cy0], m3 = G[x2 * GP + cy1];
  const unsigned full = 0xffffffffu;
  const double ax = __shfl_sync(full, *dX, px), ay = __shfl_sync(full, *dY, px);
  const double bx = __shfl_sync(full, *dX, py), by = __shfl_sync(full, *dY, py);
  const double2 rpx = make_double2(__shfl_sync(full, *cK, px), __shfl_sync(full, *sK, px));
  const double2 rpy = make_double2(__shfl_sync(full, *cK, py), __shfl_sync(full, *sK, py));
  const double al = rx ? ay : ax, be = ry ? by : bx;
  double g0, g1;
  gram_rot2(m0, m1, m2, m3, rpx, rpy, rx, false, &g0, &g1);
  const double ga = ry ? g1 : g0;
  double c = 1.0, sn = 0.0;
  const bool rot = rotation(al, be, ga, tol2, &c, &sn);
  *cK = c;
  *sK = sn;
  *rK = rot;
  pair_diag(al, be, ga, make_double2(c, sn), rot, dX, dY);
}

// Block one-sided Jacobi, Gram formulation.  2P blocks of JW columns; every
// round of the circle-method tournament pairs them up; pair p is owned by one
// thread-block cluster of C CTAs, CTA r holding rows [r R, (r+1) R) of the
// pair's 2 JW columns of A and V in shared memory (R = ne / C).  Per round:
//   1. partial Gram G_r = A_r^T A_r (JC x JC) of the slice;
//   2. G = sum_r G_r read over DSMEM in rank order (every CTA of the cluster
//      forms the same G bitwise);
//   3. the JW - 1 intra-block sub-rounds (round 0 of a sweep) and JW cross
//      sub-rounds run on G (JC x JC), accumulating the rotations into J;
//   4. A_r <- A_r J, V_r <- V_r J; store; grid barrier.
// The rotations, their order and the convergence test are those of the
// classic column-pair sweep; only the column updates are batched per round
// (one small GEMM instead of ~JW rotations of every column), and the rows are
// split over C SMs.
//
// Sub-rounds are software-pipelined over one block barrier each: warps
// 0..JW-1 apply sub-round k (Gn = Q_k^T G Q_k, J <- J Q_k) while the extra
// rotation warp JW forms, from the same G and Q_k, the three Gram entries of
// every pair of sub-round k+1 and computes Q_{k+1}.
constexpr int JTHREADS = 32 * (JW + 1);

__global__ void __launch_bounds__(JTHREADS, 1) jacobi_rounds_kernel(Args a) {
  extern __shared__ double sm[];
  unsigned C, r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(C));
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  const int p = blockIdx.x / C;
  const int R = a.ne / C;
  const long row0 = (long)r * R;
  double* As = sm;                  // R x JC row-major, pitch GP
  double* Vs = As + (size_t)R * GP;
  double* Gp = Vs + (size_t)R * GP;  // JC x JC partial (dense, pitch JC)
  double* G = Gp + JC * JC;          // JC x GP, two buffers
  double* J = G + 2 * JC * GP;       // JC x GP
  __shared__ unsigned s_mask[2];
  __shared__ double2 CS[2][JW];
  __shared__ Sched sc;
  __shared__ unsigned la[NSUB * JW];
  build_sched(&sc);
  __syncthreads();
  build_lookahead(&sc, la);
  const int N = a.nblk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool rwarp = warp == JW;  // the rotation warp
  const double tol2 = a.tol * a.tol;
  unsigned bar = 0;
  int sweep = 0;
#ifdef JAC_PROBE
  unsigned long long probe_last = gtime();
  const long long clk0 = clock64();
  long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  for (; sweep < MAX_SWEEPS; ++sweep) {
    for (int rr = 0; rr < N - 1; ++rr) {
      int bp, bq;
      round_pair(N, rr, p, &bp, &bq);
      // 1. load the slice (16-byte global loads along the columns)
      const int R2 = R >> 1;
      for (int idx = threadIdx.x; idx < JC * R2; idx += JTHREADS) {
        const int col = idx / R2, i = (idx - col * R2) * 2;
        const int gc = col < JW ? bp * JW + col : bq * JW + (col - JW);
        const long off = row0 + i + (long)gc * a.ld;
        const double2 va = __ldcg((const double2*)&a.A[off]);
        const double2 vv = __ldcg((const double2*)&a.V[off]);
        As[i * GP + col] = va.x;
        As[(i + 1) * GP + col] = va.y;
        Vs[i * GP + col] = vv.x;
        Vs[(i + 1) * GP + col] = vv.y;
      }
      for (int idx = threadIdx.x; idx < JC * JC; idx += JTHREADS) {
        const int i = idx / JC, j = idx - i * JC;
        J[i * GP + j] = (i == j) ? 1.0 : 0.0;
      }
      __syncthreads();
      JPROBE(0);
      // 2. partial Gram A_r^T A_r on the FP64 tensor cores (DMMA 8x8x4):
      //    warp w owns the 8x8 output tile (w / 4, w % 4), K = R slice rows
      if (!rwarp) {
        const int g = lane >> 2, tq = lane & 3;
        const int i0 = 8 * (warp >> 2), j0 = 8 * (warp & 3);
        // four independent accumulator chains over the k-steps (R is a
        // multiple of 8: k0 and k0 + 4 of every 8-row tile), summed at the end
        double c[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        int k0 = 0;
        for (; k0 + 16 <= R; k0 += 16) {
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int kk = k0 + 4 * h + tq;
            dmma884(c[h][0], c[h][1], As[kk * GP + i0 + g], As[kk * GP + j0 + g]);  // (A^T)[i][k] A[k][j]
          }
        }
        for (; k0 < R; k0 += 4) {
          const int kk = k0 + tq;
          dmma884(c[0][0], c[0][1], As[kk * GP + i0 + g], As[kk * GP + j0 + g]);
        }
        Gp[(i0 + g) * JC + j0 + 2 * tq] = (c[0][0] + c[1][0]) + (c[2][0] + c[3][0]);
        Gp[(i0 + g) * JC + j0 + 2 * tq + 1] = (c[0][1] + c[1][1]) + (c[2][1] + c[3][1]);
      }
      JPROBE(1);
      if (C > 1) cluster_sync_all();
      else __syncthreads();
      for (int idx = threadIdx.x; idx < JC * JC; idx += JTHREADS) {
        double part[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < (int)C) part[q] = (q == (int)r) ? Gp[idx] : ld_dsmem(&Gp[idx], q);
        double g = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < (int)C) g += part[q];
        G[(idx / JC) * GP + (idx % JC)] = g;
      }
      __syncthreads();
      JPROBE(2);
      // 3. sub-rounds on G (ping-pong buffers), pipelined
      const int u0 = rr == 0 ? 0 : JW - 1;  // first schedule index of this round
      const int K = NSUB - u0;
      double cK = 1.0, sK = 0.0, dX = 0.0, dY = 0.0;  // rotation warp state (own pair)
      bool rK = false;
      if (rwarp) {  // rotations of the first sub-round, from G directly
        const int pl = lane & (JW - 1);
        const int x = sc.px[u0][pl], y = sc.py[u0][pl];
        const double al = G[x * GP + x], be = G[y * GP + y], ga = G[x * GP + y];
        rK = rotation(al, be, ga, tol2, &cK, &sK);
        pair_diag(al, be, ga, make_double2(cK, sK), rK, &dX, &dY);
        const unsigned mask = __ballot_sync(0xffffffffu, rK) & ((1u << JW) - 1);
        if (lane < JW) CS[0][lane] = make_double2(cK, sK);
        if (lane == 0) s_mask[0] = mask;
      }
      __syncthreads();
      int nrot = 0;
      const double* gc = G;
      double* gn = G + JC * GP;
      for (int k = 0; k < K; ++k) {
#ifdef JAC_PROBE
        const long long c0 = clock64();
#endif
        const int u = u0 + k;
        const double2* cs = CS[k & 1];
        const unsigned mask = s_mask[k & 1];
        nrot += __popc(mask);
        if (threadIdx.x < JW * JW) {
          // 2 x 2 block (row pair pb, column pair q) of Gn: both rows
          const int pb = threadIdx.x / JW, q = threadIdx.x % JW;
          const int xp = sc.px[u][pb], yp = sc.py[u][pb], xq = sc.px[u][q], yq = sc.py[u][q];
          const double m00 = gc[xp * GP + xq], m01 = gc[xp * GP + yq];
          const double m10 = gc[yp * GP + xq], m11 = gc[yp * GP + yq];
          const double2 rp = cs[pb], rq = cs[q];
          const bool z = pb == q && ((mask >> q) & 1);
          double g0, g1, h0, h1;
          gram_rot2(m00, m01, m10, m11, rp, rq, 0, z, &g0, &g1);
          gram_rot2(m10, m11, m00, m01, rp, rq, 1, z, &h0, &h1);
          gn[xp * GP + xq] = g0;
          gn[xp * GP + yq] = g1;
          gn[yp * GP + xq] = h0;
          gn[yp * GP + yq] = h1;
        } else if (!rwarp) {
          // J <- J Q: rows k and k + JW of column pair q
          const int tt = threadIdx.x - JW * JW, q = tt % JW, k0 = tt / JW;
          if ((mask >> q) & 1) {
            const int xq = sc.px[u][q], yq = sc.py[u][q];
            const double2 rq = cs[q];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int kk = k0 + h * JW;
              const double jx = J[kk * GP + xq], jy = J[kk * GP + yq];
              J[kk * GP + xq] = fma(rq.x, jx, -rq.y * jy);
              J[kk * GP + yq] = fma(rq.y, jx, rq.x * jy);
            }
          }
        } else if (k + 1 < K) {
          rotate_next(la[(u + 1) * JW + (lane & (JW - 1))], gc, tol2, &cK, &sK, &rK, &dX, &dY);
          const unsigned m2 = __ballot_sync(0xffffffffu, rK) & ((1u << JW) - 1);
          if (lane < JW) CS[(k + 1) & 1][lane] = make_double2(cK, sK);
          if (lane == 0) s_mask[(k + 1) & 1] = m2;
        }
#ifdef JAC_PROBE
        const long long c1 = clock64();
#endif
        __syncthreads();
#ifdef JAC_PROBE
        {
          const int o = threadIdx.x == 0 ? 0 : 3;
          pacc[o] += c1 - c0;
          pacc[o + 1] += clock64() - c1;
          pacc[o + 2] += 1;
        }
#endif
        const double* t = gc;
        gc = gn;
        gn = const_cast<double*>(t);
      }
      JPROBE(3);
      // 4. A_r <- A_r J, V_r <- V_r J (warp w rows w, w + JW, ...), store
      if (nrot) {
        // DMMA 8x8x4: job = (8-row tile, matrix A or V); each warp computes
        // its tile's 8 x 32 block of M_r J and writes it back over its own rows
        if (!rwarp) {
          const int g = lane >> 2, tq = lane & 3;
          const int jobs = 2 * (R / 8);
          for (int job = warp; job < jobs; job += JW) {
            double* M = (job & 1) ? Vs : As;
            const int r0 = 8 * (job >> 1);
            double acc[4][2];
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = 0.0;
#pragma unroll
            for (int l0 = 0; l0 < JC; l0 += 4) {
              const double av = M[(r0 + g) * GP + l0 + tq];
#pragma unroll
              for (int c = 0; c < 4; ++c) dmma884(acc[c][0], acc[c][1], av, J[(l0 + tq) * GP + 8 * c + g]);
            }
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              M[(r0 + g) * GP + 8 * c + 2 * tq] = acc[c][0];
              M[(r0 + g) * GP + 8 * c + 2 * tq + 1] = acc[c][1];
            }
          }
        }
        __syncthreads();
        JPROBE(4);
        for (int idx = threadIdx.x; idx < JC * R2; idx += JTHREADS) {
          const int col = idx / R2, i = (idx - col * R2) * 2;
          const int gc2 = col < JW ? bp * JW + col : bq * JW + (col - JW);
          const long off = row0 + i + (long)gc2 * a.ld;
          *(double2*)&a.A[off] = make_double2(As[i * GP + col], As[(i + 1) * GP + col]);
          *(double2*)&a.V[off] = make_double2(Vs[i * GP + col], Vs[(i + 1) * GP + col]);
        }
        if (r == 0 && threadIdx.x == 0) atomicAdd(&a.rot[sweep], nrot);
      }
      JPROBE(5);
      ++bar;
      grid_barrier(a.ctr, bar * gridDim.x);
      JPROBE(6);
    }
    if (__ldcg(&a.rot[sweep]) == 0) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.status = (sweep < MAX_SWEEPS) ? sweep + 1 : -1;
#ifdef JAC_PROBE
  if (blockIdx.x == 0 && threadIdx.x == 0) g_probe[7] += clock64() - clk0;
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int o = 0; o < 3; ++o) g_probe2[o] += pacc[o];
  if (blockIdx.x == 0 && threadIdx.x == 32 * JW)
    for (int o = 3; o < 8; ++o) g_probe2[o] += pacc[o];
#endif
  if (C > 1) cluster_sync_all();  // no CTA leaves while its Gp may still be read
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

// Cluster size C (CTAs per block pair, each holding ne / C rows of the pair
// in shared memory).  Rows per CTA stay <= 256 (smem), CTAs <= 148 (the
// cooperative grid must be co-resident).  Tuning knob UTV_JAC_CLUSTER.
static inline int jac_blocks(int n) {
  int nb = (n + jac::JW - 1) / jac::JW;
  if (nb & 1) nb++;
  if (nb < 2) nb = 2;
  return nb;
}

static inline int jac_cluster(int n) {
  static const int forced = [] {
    const char* e = getenv("UTV_JAC_CLUSTER");
    return e ? atoi(e) : 0;
  }();
  const int pairs = jac_blocks(n) / 2;
  int c = forced == 1 || forced == 2 || forced == 4 || forced == 8 ? forced : (n >= 128 ? 4 : (n >= 32 ? 2 : 1));
  while (c > 1 && pairs * c > 148) c >>= 1;
  while (c < 8 && (round_up(n, 8 * c) / c) > 256) c <<= 1;
  return c;
}

static inline long jac_ld(int n) { return round_up(n, 64); }  // >= round_up(n, 8 C), C <= 8

size_t gesvj_ws_doubles(int n) {
  const long ld = jac_ld(n);
  const long npad = (long)jac_blocks(n) * jac::JW;
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
  const long ld = jac_ld(n);
  const int nblk = jac_blocks(n);
  const long npad = (long)nblk * jac::JW;
  const int C = jac_cluster(n);
  Arena ar{(char*)ws, ws_doubles * sizeof(double), 0};
  double* Aw = ar.take(ld * npad);
  double* Vw = ar.take(ld * npad);
  double* ctl = ar.take(jac::MAX_SWEEPS + 64);
  double* scratch = ar.take(1024);
  if (!scratch) return UTV_ERR_WORKSPACE;
  // rows are padded to a multiple of 8C (equal slices of whole 8-row DMMA
  // tiles); padding is zero
  const int ne = (int)round_up(n, 8 * C);
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
  a.ne = ne; a.nblk = nblk;
  a.tol = 4.0 * sqrt((double)n) * jac::EPS;
  a.rot = (int*)ctl;
  a.ctr = (unsigned*)(ctl + jac::MAX_SWEEPS);
  a.status = status_dev;
  if (!g_jac_attr) {
    UTV_CUDA(cudaFuncSetAttribute(jac::jacobi_rounds_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    UTV_CUDA(cudaFuncSetAttribute(jac::jacobi_finish_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    g_jac_attr = true;
  }
  {
    ProfScope ps(PROF_JACOBI, 0.0, 0.0, st);
    // a cooperative cluster grid the device cannot hold co-resident (fewer
    // SMs, MIG) falls back to smaller clusters: same rotations, same bits
    // up to the Gram partial-sum grouping
    for (int c = C;; c >>= 1) {
      const int nec = (int)round_up(n, 8 * c);  // 8-row tiles per slice (DMMA)
      const int R = nec / c;
      const size_t smem =
          ((size_t)2 * R * jac::GP + jac::JC * jac::JC + 3 * jac::JC * jac::GP) * sizeof(double);
      if (smem > 200 * 1024) return -1;
      a.ne = nec;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((nblk / 2) * c);
      cfg.blockDim = dim3(jac::JTHREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative;
      at[1].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      const cudaError_t e = cudaLaunchKernelEx(&cfg, jac::jacobi_rounds_kernel, a);
      if (e == cudaSuccess) break;
      if (c == 1 || (e != cudaErrorCooperativeLaunchTooLarge)) {
        fprintf(stderr, "libutvb200: jacobi_rounds_kernel launch failed: %s\n", cudaGetErrorString(e));
        return UTV_ERR_CUDA;
      }
      (void)cudaGetLastError();  // clear the launch error, retry with half the cluster
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
