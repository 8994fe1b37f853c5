// K3 (fused): Householder QR of a rows x cols panel, cols <= 256, in ONE
// cooperative launch — geqr2 + the intra-panel trailing updates + larft.
//
// Replaces hqr_full's column loop (qr.py:87-99: _reflector qr.py:43-60,
// rank-1 update :94-95, _append_twy_column :63-68) for one panel of the
// blocked QR.  Reference conventions are kept exactly: beta =
// -sign(alpha)||x|| with sign(0)=+1, v0 = 1, tau = 2/(1+sigma/v1^2), skip
// (tau = 0, identity reflector, zeros below the diagonal) when ||x|| <=
// eps*||A||_F of the whole hqr_full input or sigma == 0, forward compact-WY
// triangle.
//
// B200 design (latency-bound; the panel, <= 32 MiB, lives in L2):
//  * G <= 148 CTAs (one per SM), each owning a row slab of rc <= 512 rows.
//    The panel is processed in 32-column leaves; the current leaf's slab is
//    resident in shared memory.
//  * Per column: one fixed-order grid reduction (every CTA writes its 32
//    partial dots, one grid barrier, every CTA reads all partials with 256
//    threads in parallel) yields ||x||^2, x^T P[:, leaf] and row J, from
//    which the reflector, the rank-1 update and the leaf's WY column follow.
//    The 32x32 leaf triangle is built redundantly by every CTA (no extra
//    communication).
//  * Per leaf: the partial products Y_leaf^T [Y_prev | P_trail] of every
//    slab are reduced across CTAs (2 grid barriers); P_trail -= Y_leaf
//    (T_leaf^T W) is applied slab-locally; Y_prev^T Y_leaf is kept for T.
//  * After the last leaf, the off-diagonal blocks of T follow from
//    T12 = -T11 (Y1^T Y2) T22 row by row (one warp per row, no barriers).
//  All reductions are in a fixed order: results are bitwise reproducible.
#include "common.cuh"
#include <cstdlib>

#include "utv_internal.h"

namespace utv {

namespace pqr {
// Diagnostics: build with -DPANEL_PROBE (tools/panel_probe.cu) to accumulate
// CTA 0's per-phase %globaltimer durations into g_probe.
#ifdef PANEL_PROBE
#ifndef PANEL_PROBE_CTA
#define PANEL_PROBE_CTA 0
#endif
__device__ unsigned long long g_probe[16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
#define PROBE(k)                                   \
  if (blockIdx.x == PANEL_PROBE_CTA && threadIdx.x == 0) { \
    const unsigned long long now_ = gtime();       \
    g_probe[k] += now_ - probe_last;               \
    probe_last = now_;                             \
  }
#else
#define PROBE(k)
#endif
constexpr int NB = 32;
constexpr int THREADS = 256;
constexpr int RC_MIN = 64;
constexpr int RC_MAX = 512;
constexpr int GMAX = 148;
constexpr int PW = QR_PANEL;     // max panel width
constexpr int XR = 64;           // staged rows per sub-chunk (phase A)
constexpr int XC = 128;          // staged X columns per chunk
constexpr int XRP = XR + 1;      // odd pitch of the staged [col][row] chunk
constexpr int PMAX = (GMAX + 3) / 4;  // partial records summed per thread
constexpr double EPS = 2.220446049250313e-16;

struct Args {
  double* P;
  long ldp;
  double* Y;
  long ldy;
  double* T;
  long ldt;
  int rows, cols, rc;
  const double* fro2;
  double* part;   // [2][G][2*NB]
  double* wpart;  // [G][NB][PW]
  double* wsum;   // [NB][PW]
  double* S;      // [PW][PW] Gram blocks Y[:, :j0]^T Y[:, leaf], ld PW
  unsigned* ctr;  // zeroed before launch
};

__host__ __device__ inline size_t smem_doubles(int rc) {
  return (size_t)(rc + 1) * NB + NB * (NB + 1) + 8 * NB + 4 * NB + (size_t)XC * XRP + 8 * PW + rc + 16;
}

// TALL: slabs of >= THREADS rows per CTA (rc >= 256: the C4 TSQR leaves),
// which take the batched trailing-update path in phase D; a separate
// instantiation so the short-slab kernel's code is unchanged.
template <bool TALL>
__global__ void __launch_bounds__(THREADS, 1) panel_qr_kernel(Args a) {
  extern __shared__ double sm[];
  const int ld = a.rc + 1;  // odd pitch: column-strided access is conflict free
  double* tile = sm;
  double* Ts = tile + (size_t)ld * NB;  // [NB][NB+1], Ts[r + c*(NB+1)]
  double* red = Ts + NB * (NB + 1);     // [8][NB] / [4][2*NB]
  double* Sv = red + 8 * NB;
  double* Rv = Sv + NB;
  double* Wv = Rv + NB;
  double* Zv = Wv + NB;
  double* Xs = Zv + NB;                 // [XC][XRP] staged chunk / [XC][NB] W' chunk
  double* rowbuf = Xs + (size_t)XC * XRP;  // [8 warps][PW]
  double* vrow = rowbuf + 8 * PW;          // [rc] reflector entries of the current column

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = blockIdx.x, G = gridDim.x;
  const int r0 = g * a.rc;
  const int nr = max(0, min(a.rc, a.rows - r0));
  const int cols = a.cols;
  const double thr = EPS * sqrt(*a.fro2);
  const int nleaf = (cols + NB - 1) / NB;
  unsigned nbar = 0;
#ifdef PANEL_PROBE
  unsigned long long probe_last = gtime();
#endif
  int step = 0;  // global column-step counter (partials double buffer)
  auto gsync = [&]() {
    ++nbar;
    if (G > 1) grid_barrier(a.ctr, nbar * (unsigned)G);
    else __syncthreads();
  };
  // Split barrier: arrive, do independent work, then wait.
  auto garrive = [&]() {
    ++nbar;
    __syncthreads();
    if (G > 1 && t == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.ctr) : "memory");
  };
  auto gwait = [&]() {
    if (G > 1 && t == 0) {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.ctr) : "memory");
      } while (v < nbar * (unsigned)G);
    }
    __syncthreads();
  };
  // Leaf-triangle column pj (qr.py:63-68), computed redundantly in every CTA
  // while the next column's grid barrier is in flight:
  // Ts[r][pj] = -tau * sum_{q=r}^{pj-1} Ts[r][q] Z[q], 4 rows per warp.
  int pend = -1;
  double ptau = 0.0;
  auto ts_column = [&]() {
    if (pend < 0) return;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = warp * 4 + k;
      double s = (lane >= r && lane < pend) ? Ts[r + lane * (NB + 1)] * Zv[lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0 && r < pend) Ts[r + pend * (NB + 1)] = -ptau * s;
    }
    if (t == 0) Ts[pend + pend * (NB + 1)] = ptau;
    pend = -1;
  };

  for (int l = 0; l < nleaf; ++l) {
    const int j0 = l * NB;
    const int jb = min(NB, cols - j0);
    // ---- load the leaf slab (all slab rows) ----
    for (int idx = t; idx < nr * jb; idx += THREADS) {
      const int i = idx % nr, c = idx / nr;
      tile[i + c * ld] = a.P[(r0 + i) + (long)(j0 + c) * a.ldp];
    }
    for (int idx = t; idx < NB * (NB + 1); idx += THREADS) Ts[idx] = 0.0;
    __syncthreads();
    PROBE(0);

    // ---- column steps ----
    for (int jj = 0; jj < jb; ++jj, ++step) {
      const int J = j0 + jj;
      const int i_lo = max(0, J + 1 - r0);
      const bool owner = (J >= r0) && (J < r0 + nr);
      const int par = step & 1;
      {  // local partials S_c = sum_{i>J} x_i P[i,c]
        const int c = lane, grp = warp;
        double acc = 0.0;
        if (c < jb)
          for (int i = i_lo + grp; i < nr; i += 8) acc = fma(tile[i + jj * ld], tile[i + c * ld], acc);
        red[grp * NB + c] = acc;
      }
      __syncthreads();
      // partial record of this CTA: [0, NB) dots, [NB, 2NB) row J (owner only,
      // zeros elsewhere, so the cross-CTA sum delivers row J exactly)
      if (t < 2 * NB) {
        double s = 0.0;
        if (t < NB) {
#pragma unroll
          for (int q = 0; q < 8; ++q) s += red[q * NB + t];
        } else if (owner && t - NB < jb) {
          s = tile[(J - r0) + (t - NB) * ld];
        }
        a.part[((size_t)par * G + g) * 2 * NB + t] = s;
      }
      PROBE(1);
      garrive();
      ts_column();  // previous column's triangle entries, hidden behind the barrier
      gwait();
      PROBE(2);
      // every CTA: sum the G dot records (threads 0..127: 4 interleaved groups,
      // all loads in flight, fixed order); row J is read from its owner's
      // record alone (the other records hold zeros there, so this is the
      // same value the full sum gave) — half the L2 traffic of the exchange
      if (t < 4 * NB) {
        const int e = t & (NB - 1), q0 = t / NB;
        double v[PMAX];
#pragma unroll
        for (int k = 0; k < PMAX; ++k) {
          const int q = q0 + 4 * k;
          v[k] = (q < G) ? __ldcg(&a.part[((size_t)par * G + q) * 2 * NB + e]) : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < PMAX; ++k) s += v[k];
        red[q0 * 2 * NB + e] = s;
      } else if (t < 5 * NB) {
        const int e = t - 4 * NB;
        const int gJ = J / a.rc;  // the CTA whose slab holds row J
        Rv[e] = (gJ < G) ? __ldcg(&a.part[((size_t)par * G + gJ) * 2 * NB + NB + e]) : 0.0;
      }
      __syncthreads();
      if (t < NB) Sv[t] = (red[t] + red[2 * NB + t]) + (red[4 * NB + t] + red[6 * NB + t]);
      __syncthreads();

      PROBE(3);
      const double sigma = Sv[jj], alpha = Rv[jj];
      const double xnorm = sqrt(alpha * alpha + sigma);
      const bool skip = (xnorm <= thr) || (sigma == 0.0);
      if (!skip) {
        const double sgn = alpha >= 0.0 ? 1.0 : -1.0;
        const double v1 = alpha + sgn * xnorm;
        const double tau = 2.0 / (1.0 + sigma / (v1 * v1));
        if (t < NB) {
          Wv[t] = (t > jj && t < jb) ? tau * (Rv[t] + Sv[t] / v1) : 0.0;
          Zv[t] = (t < jj) ? Rv[t] + Sv[t] / v1 : 0.0;
        }
        __syncthreads();
        // v_i = x_i / v1 once per row (reference rounding: true division)
        for (int i = i_lo + t; i < nr; i += THREADS) vrow[i] = tile[i + jj * ld] / v1;
        __syncthreads();
        // rank-1 update of the leaf columns right of jj: 64 row lanes x 4 column groups
        {
          const int tr = t & 63, tc = t >> 6;
          for (int c = jj + 1 + tc; c < jb; c += 4) {
            const double w = Wv[c];
            double* col = tile + c * ld;
            for (int i = i_lo + tr; i < nr; i += 64) col[i] = fma(-vrow[i], w, col[i]);
          }
        }
        if (owner && t < NB && t > jj && t < jb) tile[(J - r0) + t * ld] -= Wv[t];
        pend = jj;
        ptau = tau;
        __syncthreads();
        for (int i = i_lo + t; i < nr; i += THREADS) tile[i + jj * ld] = vrow[i];
        if (owner && t == 0) tile[(J - r0) + jj * ld] = -sgn * xnorm;
      } else {
        for (int i = i_lo + t; i < nr; i += THREADS) tile[i + jj * ld] = 0.0;
      }
      __syncthreads();
      PROBE(11);
    }
    ts_column();  // last column of the leaf
    __syncthreads();
    PROBE(4);

    // ---- write R / Y of the leaf; turn the tile into Y form ----
    for (int idx = t; idx < nr * jb; idx += THREADS) {
      const int i = idx % nr, c = idx / nr;
      const int gi = r0 + i, C = j0 + c;
      const double v = tile[i + c * ld];
      a.P[gi + (long)C * a.ldp] = (gi <= C) ? v : 0.0;
      const double yv = (gi < C) ? 0.0 : (gi == C ? 1.0 : v);
      a.Y[gi + (long)C * a.ldy] = yv;
      tile[i + c * ld] = yv;
    }
    if (g == 0)
      for (int idx = t; idx < jb * jb; idx += THREADS) {
        const int r = idx % jb, c = idx / jb;
        a.T[(j0 + r) + (long)(j0 + c) * a.ldt] = Ts[r + c * (NB + 1)];
      }
    __syncthreads();

    const int nX = cols - jb;  // X = [Y[:, :j0] | P[:, j0+jb:cols]]
    if (nX <= 0) continue;     // single-leaf panel: nothing else to do
    const int i0 = max(0, j0 - r0);  // first slab row with Y_leaf possibly != 0

    PROBE(5);
    // ---- phase A: partials of Y_leaf^T X over this slab ----
    for (int cb = 0; cb < nX; cb += XC) {
      const int ncb = min(XC, nX - cb);
      double acc[4][4];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int d = 0; d < 4; ++d) acc[x][d] = 0.0;
      const int jq = warp * 4;
      for (int rb = i0; rb < nr; rb += XR) {
        const int nrb = min(XR, nr - rb);
        for (int idx = t; idx < ncb * nrb; idx += THREADS) {
          const int i = idx % nrb, x = idx / nrb;
          const int xg = cb + x;
          const long gi = r0 + rb + i;
          Xs[x * XRP + i] = (xg < j0) ? a.Y[gi + (long)xg * a.ldy]
                                      : a.P[gi + (long)(xg + jb) * a.ldp];
        }
        __syncthreads();
        for (int i = 0; i < nrb; ++i) {
          double y[4], xv[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) y[x] = (jq + x < jb) ? tile[(rb + i) + (jq + x) * ld] : 0.0;
#pragma unroll
          for (int d = 0; d < 4; ++d) xv[d] = Xs[(lane + 32 * d) * XRP + i];
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int d = 0; d < 4; ++d) acc[x][d] = fma(y[x], xv[d], acc[x][d]);
        }
        __syncthreads();
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          const int c = lane + 32 * d;
          if (jq + x < jb && c < ncb) a.wpart[((size_t)g * NB + jq + x) * PW + cb + c] = acc[x][d];
        }
    }
    PROBE(6);
    gsync();
    PROBE(7);

    // ---- phase C: reduce the partials across CTAs (8 lanes per entry) ----
    {
      const int E = jb * nX;
      const int sub = t & 7;
      for (int e0 = g * (THREADS / 8); e0 < E; e0 += G * (THREADS / 8)) {
        const int e = e0 + (t >> 3);
        double s = 0.0;
        if (e < E) {
          const int x = e % nX, r = e / nX;
#pragma unroll 4
          for (int q = sub; q < G; q += 8) s += __ldcg(&a.wpart[((size_t)q * NB + r) * PW + x]);
        }
        // fixed-order combine of the 8 sub-sums
        s += __shfl_down_sync(0xffffffffu, s, 4, 8);
        s += __shfl_down_sync(0xffffffffu, s, 2, 8);
        s += __shfl_down_sync(0xffffffffu, s, 1, 8);
        if (sub == 0 && e < E) {
          const int x = e % nX, r = e / nX;
          if (x < j0) a.S[x + (size_t)(j0 + r) * PW] = s;  // (Y_prev^T Y_leaf)[x, r]
          else a.wsum[(size_t)r * PW + (x - j0)] = s;      // W[r, trailing col]
        }
      }
    }
    PROBE(8);
    gsync();
    PROBE(9);

    // ---- phase D: P_trail -= Y_leaf (T_leaf^T W), slab-local ----
    const int nT = cols - j0 - jb;
    for (int cb = 0; cb < nT; cb += XC) {
      const int ncb = min(XC, nT - cb);
      double* Wc = Xs;                  // [c][NB] reduced W chunk
      double* Wp = Xs + XC * NB;        // [c][NB] T_leaf^T W chunk
      for (int idx = t; idx < ncb * NB; idx += THREADS) {
        const int c = idx % ncb, r = idx / ncb;  // coalesced along c
        Wc[c * NB + r] = __ldcg(&a.wsum[(size_t)r * PW + cb + c]);
      }
      __syncthreads();
      for (int idx = t; idx < ncb * NB; idx += THREADS) {
        const int r = idx & (NB - 1), c = idx >> 5;
        double s = 0.0;
        for (int q = 0; q <= r; ++q)  // (T^T)[r][q] = Ts[q][r], T upper triangular
          s = fma(Ts[q + r * (NB + 1)], Wc[c * NB + q], s);
        Wp[c * NB + r] = (r < jb) ? s : 0.0;
      }
      __syncthreads();
      // rows x column groups so every thread has work even for short slabs
      const int nrow = nr - i0;
      const int cg = nrow >= THREADS ? 1 : (nrow >= THREADS / 2 ? 2 : (nrow >= THREADS / 4 ? 4 : 8));
      const int rl = THREADS / cg;
      const int tr = t % rl, tcg = t / rl;
      if (TALL && cg == 1) {
        // tall slabs (>= 256 rows per CTA, the C4 TSQR leaves): a thread walks
        // all trailing columns of its rows, so the P read-modify-writes of DB
        // columns are issued together (one L2/HBM round trip per element
        // otherwise; 74,898-row panel 3.93 -> 3.68 ms).  Same arithmetic, same bits.
        constexpr int DB = 8;
        for (int i = i0 + tr; i < nr; i += rl) {
          double y[NB];
#pragma unroll
          for (int r = 0; r < NB; ++r) y[r] = tile[i + r * ld];  // zero beyond jb
          double* prow = a.P + (r0 + i) + (long)(j0 + jb + cb) * a.ldp;
          for (int c0 = 0; c0 < ncb; c0 += DB) {
            double pv[DB];
#pragma unroll
            for (int u = 0; u < DB; ++u) pv[u] = (c0 + u < ncb) ? __ldcg(prow + (long)(c0 + u) * a.ldp) : 0.0;
#pragma unroll
            for (int u = 0; u < DB; ++u) {
              const int c = c0 + u;
              if (c >= ncb) break;
              const double2* w2 = (const double2*)(Wp + c * NB);
              double s = 0.0;
#pragma unroll
              for (int r = 0; r < NB / 2; ++r) {
                const double2 w = w2[r];
                s = fma(y[2 * r], w.x, s);
                s = fma(y[2 * r + 1], w.y, s);
              }
              prow[(long)c * a.ldp] = pv[u] - s;
            }
          }
        }
      } else {
        for (int i = i0 + tr; i < nr; i += rl) {
          double y[NB];
#pragma unroll
          for (int r = 0; r < NB; ++r) y[r] = tile[i + r * ld];  // zero beyond jb
          double* prow = a.P + (r0 + i);
          for (int c = tcg; c < ncb; c += cg) {
            const double2* w2 = (const double2*)(Wp + c * NB);
            double s = 0.0;
#pragma unroll
            for (int r = 0; r < NB / 2; ++r) {
              const double2 w = w2[r];
              s = fma(y[2 * r], w.x, s);
              s = fma(y[2 * r + 1], w.y, s);
            }
            double* pp = prow + (long)(j0 + jb + cb + c) * a.ldp;
            *pp -= s;
          }
        }
      }
      __syncthreads();
    }
    PROBE(13);
  }

  PROBE(10);
  // ---- T off-diagonal blocks: T12 = -T11 (Y1^T Y2) T22, one warp per row ----
  // Leaf by leaf: every CTA stages S[:j0L, leaf L] and T_LL in smem, then its
  // warps finish entries T[r, leaf L] of their rows (a row's earlier entries
  // are its own earlier results, re-read from T).
  if (nleaf > 1) {
    double* rb = rowbuf + warp * PW;
    for (int L = 1; L < nleaf; ++L) {
      const int j0L = L * NB, jbL = min(NB, cols - j0L);
      double* Ss = Xs;                  // [q][NB], q < j0L
      double* TL = Xs + (PW - NB) * NB; // [m][NB]
      if (g * 8 < j0L) {                // CTAs that own rows of this leaf
        for (int idx = t; idx < j0L * NB; idx += THREADS) {
          const int q = idx % j0L, c = idx / j0L;
          Ss[q * NB + c] = (c < jbL) ? __ldcg(&a.S[q + (size_t)(j0L + c) * PW]) : 0.0;
        }
        for (int idx = t; idx < NB * NB; idx += THREADS) {
          const int m = idx & (NB - 1), c = idx >> 5;
          TL[m * NB + c] = (m < jbL && c < jbL) ? __ldcg(&a.T[(j0L + m) + (long)(j0L + c) * a.ldt]) : 0.0;
        }
      }
      __syncthreads();
      for (int r = g * 8 + warp; r < j0L; r += G * 8) {
        const int c0 = (r / NB) * NB;
        for (int c = c0 + lane; c < j0L; c += 32) rb[c] = __ldcg(&a.T[r + (long)c * a.ldt]);
        __syncwarp();
        double u = 0.0;
        for (int q = c0; q < j0L; ++q) u = fma(rb[q], Ss[q * NB + lane], u);
        double v = 0.0;
#pragma unroll 8
        for (int m = 0; m < NB; ++m) v = fma(__shfl_sync(0xffffffffu, u, m), TL[m * NB + lane], v);
        if (lane < jbL) a.T[r + (long)(j0L + lane) * a.ldt] = -v;
        __syncwarp();
      }
      __syncthreads();
    }
  }
  PROBE(12);
}

inline void geometry(int rows, int* rc, int* G, int max_ctas) {
  const int gm = (max_ctas > 0 && max_ctas < GMAX) ? max_ctas : GMAX;
  int r = (rows + gm - 1) / gm;
  r = (r + 31) / 32 * 32;
  if (r < RC_MIN) r = RC_MIN;
  *rc = r;
  *G = (rows + r - 1) / r;
}
}  // namespace pqr

size_t panel_ws_doubles() {
  using namespace pqr;
  return 4 * (size_t)GMAX * NB + (size_t)GMAX * NB * PW + (size_t)NB * PW +
         (size_t)PW * PW + 64 + 6 * 32;
}

int panel_rows_max() { return pqr::RC_MAX * pqr::GMAX; }

static bool g_panel_attr = false;
static thread_local int g_panel_budget = 0;
void panel_set_max_ctas(int n) { g_panel_budget = n; }

int panel_qr(Mat P, Mat Y, Mat T, const double* fro2, double* ws, cudaStream_t st, int max_ctas) {
  if (P.cols > pqr::PW || P.cols < 1 || P.rows < P.cols) return -1;
  static const int env_ctas = [] {
    const char* e = getenv("UTV_PANEL_CTAS");  // diagnostics: CTA budget of full-width panels
    return e ? atoi(e) : 0;
  }();
  if (max_ctas == 0) max_ctas = g_panel_budget;
  if (max_ctas == 0 && env_ctas > 0) max_ctas = env_ctas;
  int rc, G;
  pqr::geometry(P.rows, &rc, &G, max_ctas);
  if (rc > pqr::RC_MAX) pqr::geometry(P.rows, &rc, &G, 0);  // too tall for the budget: all SMs
  if (rc > pqr::RC_MAX) {
    fprintf(stderr, "libutvb200: panel with %d rows exceeds the panel QR limit (%d)\n", P.rows,
            panel_rows_max());
    return -1;
  }
  if (G > num_sms()) return -1;
  pqr::Args a;
  a.P = P.p; a.ldp = P.ld;
  a.Y = Y.p; a.ldy = Y.ld;
  a.T = T.p; a.ldt = T.ld;
  a.rows = P.rows; a.cols = P.cols; a.rc = rc;
  a.fro2 = fro2;
  Arena ar{(char*)ws, panel_ws_doubles() * sizeof(double), 0};
  a.part = ar.take(4 * (size_t)pqr::GMAX * pqr::NB);
  a.wpart = ar.take((size_t)pqr::GMAX * pqr::NB * pqr::PW);
  a.wsum = ar.take((size_t)pqr::NB * pqr::PW);
  a.S = ar.take((size_t)pqr::PW * pqr::PW);
  a.ctr = (unsigned*)ar.take(8);
  if (!a.ctr) return UTV_ERR_WORKSPACE;
  const size_t smem = pqr::smem_doubles(rc) * sizeof(double);
  if (!g_panel_attr) {
    for (auto f : {pqr::panel_qr_kernel<false>, pqr::panel_qr_kernel<true>})
      UTV_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(pqr::smem_doubles(pqr::RC_MAX) * sizeof(double))));
    g_panel_attr = true;
  }
  void* kfn = rc >= pqr::THREADS ? (void*)pqr::panel_qr_kernel<true> : (void*)pqr::panel_qr_kernel<false>;
  // algorithmic: 2*rows*cols^2 - 2/3 cols^3 (geqr2) + larft; panel read + R/Y write
  const double c = P.cols;
  ProfScope ps(PROF_PANEL, 2.0 * P.rows * c * c - 2.0 / 3.0 * c * c * c + P.rows * c * c,
               8.0 * 3.0 * P.rows * c, st);
  if (G > 1) {
    UTV_CUDA(cudaMemsetAsync(a.ctr, 0, sizeof(unsigned), st));
    void* args[] = {&a};
    UTV_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(pqr::THREADS), args, smem, st));
  } else {
    void* args[] = {&a};
    UTV_CUDA(cudaLaunchKernel(kfn, dim3(1), dim3(pqr::THREADS), args, smem, st));
  }
  return UTV_OK;
}

}  // namespace utv
