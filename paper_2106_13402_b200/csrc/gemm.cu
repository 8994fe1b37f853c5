// K1: FP64 GEMM on the B200 DMMA tensor pipe, operands staged by TMA.
//
//   C = alpha * op(A) * op(B) + beta * C      (column-major, op in {N, T})
//
// Replaces every numpy `@` on the hot path: sampling (randutv.py:190-192),
// the three GEMMs of apply_q (qr.py:116,120), materialize_q (qr.py:131),
// A*V / A^T*Vhat in powerURV (powerurv.py:64,66) and the small-SVD rotations
// (randutv.py:152-156,167-172).
//
// Design (sm_100a):
//  * CTA tile 128x128x16, 8 DMMA warps (2x4, warp tile 64x32, ~255 regs),
//    persistent: min(tiles, 148) CTAs walk the tile list.  Thread 0 also
//    drives TMA through a full/empty mbarrier ring of 128B-swizzled smem
//    tiles, running STAGES-1 k-blocks ahead across tile boundaries so the
//    next tile's operands land while the current epilogue runs.
//  * beta != 0: the C tile is TMA-prefetched into a 128 KB smem buffer
//    during the main loop (3-stage ring); beta == 0: 6-stage ring.  The
//    epilogue stores from the accumulator fragments directly (every warp
//    store fills whole 32 B sectors), so no DRAM round trip is exposed.
//  * mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4). tcgen05 has no f64 kind.
//  * Fragment rows/cols are mapped onto the 128B-swizzled tiles with a
//    permutation that makes every 64-bit fragment load bank-conflict free
//    (see DESIGN.md "GEMM smem layout").
//  * TMA zero-fills out-of-bounds boxes, so ragged M/N/K need no predication
//    on the load side; sub-matrix pointers that are not 16B aligned are
//    handled by shifting the tensor-map origin one element up.
//  * Split-K over a deterministic workspace + fixed-order reduction when the
//    MxN tile count cannot fill 148 SMs.
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace gemm {
constexpr int BM = 128, BN = 128, BK = 16;
constexpr int NCW = 8;                   // consumer warps
constexpr int THREADS = NCW * 32;        // thread 0 also issues TMA
constexpr int A_ST = BM * BK;            // doubles per stage
constexpr int B_ST = BN * BK;
constexpr uint32_t STAGE_BYTES = (A_ST + B_ST) * 8;
constexpr uint32_t C_BYTES = BM * BN * 8;
// Ring depth: 6 stages when the tile needs no C input; 3 stages + a 128 KB
// smem C tile (TMA-prefetched during the main loop) when beta != 0.
template <bool HASC>
struct Cfg {
  static constexpr int STAGES = HASC ? 3 : 6;
  static constexpr size_t SMEM =
      (size_t)STAGES * STAGE_BYTES + (HASC ? C_BYTES : 0) + 1024 + (2 * STAGES + 2) * 8 + 64;
};

struct Args {
  int M, N, K;
  int a_sh, b_sh;    // M/N-origin shift of A_N / B_T tiles (0 or 1), see DESIGN.md
  int k_sh;          // K-origin shift: logical k = k' - k_sh
  int c_sh;          // row shift of the C tensor map (HASC only)
  int a3d, b3d;      // N-major operand mapped as a 3-D {16, K, blocks} tensor (1 TMA per stage)
  int k_split;       // k' elements per split (multiple of BK)
  int tm, tn, tiles; // tile grid (tiles = tm * tn * splits)
  double alpha, beta;
  double* C;
  long ldc;
  double* ws;  // split-K partials [split][N][M] (ld = M)
  int* sched;  // dynamic tile scheduler [ticket, done] (self-resetting), or null = static
  int tri_a;   // A (N-major, M == K, unshifted) is upper triangular: skip k-blocks below the tile
  // fused split-K: split z of an output tile adds its partial to the running
  // sum of splits < z (tile-major ws, 128x128 per tile) after a per-tile
  // semaphore says z's turn; the last split applies alpha/beta to C.  Same
  // summation order as the separate reduce kernel -> the same bits.
  int* flags;  // per-tile turn counters (self-resetting), null = separate reduce kernel
  int wstore;  // HASC: per-warp TMA stores of the C tile (tmCw, 16 x 32 boxes)
};

#ifdef GEMM_PROBE
// tools/gemm_probe.cu: per-phase clock64 cycles of warps 0 and 1 of CTA 0
// [w][0] tile-start wait (first stage), [1] main loop, [2] of which
// full-barrier waits, [3] epilogue, [4] tiles
__device__ unsigned long long g_gprobe[2][8];
#endif
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Physical double offset inside a 128B-swizzled tile whose 128-byte line is
// `line` and whose logical element within that line is `idx` (0..15).
__device__ __forceinline__ int swz(int line, int idx) {
  return line * 16 + ((((idx >> 1) ^ line) & 7) << 1) + (idx & 1);
}

// A_N tile [mblk][k][16m]; A_T tile [m][16k]; B_N [n][16k]; B_T [nblk][k][16n].
template <bool TA>
__device__ __forceinline__ int a_off_of(int k, int m) {
  if (TA) return swz(m, k);
  return swz(((m >> 4) << 4) + k, m & 15);
}
template <bool TB>
__device__ __forceinline__ int b_off_of(int k, int n) {
  if (!TB) return swz(n, k);
  return swz(((n >> 4) << 4) + k, n & 15);
}

// Logical row (0..127) of fragment row r in warp m-tile t.
template <bool TA>
__device__ __forceinline__ int frag_row(int wm, int t, int r) {
  if (TA) return wm * 64 + t * 8 + (r & 3) * 2 + (r >> 2);
  int mblk = wm * 4 + (t >> 1);
  return mblk * 16 + (t & 1) * 4 + (r & 1) + ((r >> 1) & 1) * 8 + (r >> 2) * 2;
}
template <bool TB>
__device__ __forceinline__ int frag_col(int wn, int u, int c) {
  if (!TB) return wn * 32 + u * 8 + (c & 3) * 2 + (c >> 2);
  int nblk = wn * 2 + (u >> 1);
  return nblk * 16 + (u & 1) * 4 + (c & 1) + ((c >> 1) & 1) * 8 + (c >> 2) * 2;
}

struct TileCoord {
  int mc, nc, z;
};
__device__ __forceinline__ TileCoord tile_of(const Args& p, int t) {
  const int per = p.tm * p.tn;
  TileCoord c;
  c.z = t / per;
  const int r = t - c.z * per;
  c.nc = (r / p.tm) * BN;
  c.mc = (r % p.tm) * BM;
  return c;
}

// Persistent DMMA GEMM.  Each CTA walks tiles blockIdx.x, +gridDim.x, ...
// Thread 0 is the TMA producer; its cursor runs STAGES-1 k-blocks ahead of
// the consumers across tile boundaries, so the next tile's operands stream
// in while the current tile's epilogue runs.  The epilogue stores straight
// from the accumulator fragments (32B-sector-complete, fire and forget);
// when beta != 0 the C tile was TMA-prefetched into smem during the main
// loop, so no DRAM round trip is exposed.
template <bool TA, bool TB, bool HASC>
__global__ void __launch_bounds__(THREADS, 1)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC,
                     const __grid_constant__ CUtensorMap tmCw, const Args p) {
  constexpr int STAGES = Cfg<HASC>::STAGES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment (128B swizzle atoms) by offsetting the shared pointer
  // itself: a round trip through uintptr_t would turn every operand load
  // into a generic 64-bit LD instead of LDS.
  double* smem = (double*)(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  double* sA = smem;
  double* sB = smem + STAGES * A_ST;
  double* sC = sB + STAGES * B_ST;                       // HASC only (1024B aligned)
  uint64_t* bars = (uint64_t*)(sC + (HASC ? BM * BN : 0));
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = smem_u32(bars + STAGES);
  const uint32_t cfull = smem_u32(bars + 2 * STAGES);
  // every warp done with the smem C tile (its TMA stores have read it): the
  // next tile's C may be prefetched over it (per-warp epilogue, p.wstore)
  const uint32_t cempty = smem_u32(bars + 2 * STAGES + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ktot = p.K + p.k_sh;
  // k' range of a tile: its split, clipped below at the tile's first row
  // when A is upper triangular (A[i, k] = 0 for k < i)
  auto kbeg_of = [&](const TileCoord& c) {
    const int kb = c.z * p.k_split;
    return p.tri_a ? max(kb, (c.mc / BK) * BK) : kb;
  };
  auto nk_of = [&](const TileCoord& c) {
    const int kb = kbeg_of(c);
    const int ke = min(ktot, c.z * p.k_split + p.k_split);
    return (ke - kb + BK - 1) / BK;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, NCW);
    }
    mbar_init(cfull, 1);
    mbar_init(cempty, NCW);
    fence_barrier_init();
  }
  __syncthreads();

  // ---- tile scheduling ----
  // Dynamic: thread 0 takes tickets from a global counter (the last CTA to
  // run dry resets it for the next launch on the stream), so CTAs that start
  // late — their SM held by a concurrent kernel on another stream — simply
  // find the work done.  Tile ids travel to the consumers through a smem ring
  // published before the first TMA (or sentinel arrive) of each tile.
  __shared__ int tq[8];
  int pseq = 0;  // tiles started by the producer
  // triangular A: a (tile, split) unit entirely left of the tile's first
  // row has no work and is skipped (the reduce kernel skips it too)
  auto empty_unit = [&](int t) {
    if (!p.tri_a) return false;
    const TileCoord c = tile_of(p, t);
    return (c.mc / BK) * BK >= min(ktot, (c.z + 1) * p.k_split);
  };
  int nt_pre = -1;  // prefetched scheduler ticket (thread 0)
  auto next_tile = [&](int prev) -> int {
    if (!p.sched) {
      int t = prev < 0 ? (int)blockIdx.x : prev + (int)gridDim.x;
      while (t < p.tiles && empty_unit(t)) t += (int)gridDim.x;
      return t < p.tiles ? t : -1;
    }
    // the ticket taken when this CTA started producing its current tile
    // (nt_pre) hides the atomic's round trip from the TMA producer
    int t = nt_pre >= 0 ? nt_pre : atomicAdd(p.sched, 1);
    nt_pre = -1;
    while (true) {
      if (t >= p.tiles) break;
      if (!empty_unit(t)) return t;
      t = atomicAdd(p.sched, 1);
    }
    if (atomicAdd(p.sched + 1, 1) == (int)gridDim.x - 1) {
      atomicExch(p.sched, 0);
      atomicExch(p.sched + 1, 0);
    }
    return -1;
  };
  // ---- producer state (thread 0 only) ----
  int ptile = -1, pit = 0, pnk = 0, pkb = 0;
  long pg = 0;  // global produced k-block count
  TileCoord pc{};
  bool pdone = false;
  if (threadIdx.x == 0) {
    ptile = next_tile(-1);
    if (ptile >= 0) {
      pc = tile_of(p, ptile);
      pnk = nk_of(pc);
      pkb = kbeg_of(pc);
    }
  }
  auto produce_one = [&]() {
    if (pdone) return;
    if (ptile < 0) {
      // sentinel: publish -1 and complete the slot's phase without data
      const int s = (int)(pg % STAGES);
      if (pg >= STAGES) mbar_wait(empty0 + 8 * s, (uint32_t)(((pg / STAGES) & 1) ^ 1));
      tq[pseq & 7] = -1;
      ++pseq;
      mbar_arrive(full0 + 8 * s);
      ++pg;
      pdone = true;
      return;
    }
    const int s = (int)(pg % STAGES);
    if (pg >= STAGES) mbar_wait(empty0 + 8 * s, (uint32_t)(((pg / STAGES) & 1) ^ 1));
    const uint32_t fb = full0 + 8 * s;
    if (pit == 0) {
      tq[(pseq++) & 7] = ptile;
      if (p.sched && pnk > 1) nt_pre = atomicAdd(p.sched, 1);  // consumed at this tile's last k-block
    }
    mbar_arrive_expect_tx(fb, STAGE_BYTES);
    const int k = pkb + pit * BK;  // k' (even)
    const uint32_t dA = smem_u32(sA + s * A_ST), dB = smem_u32(sB + s * B_ST);
    if (TA) {
      tma_load_2d(dA, &tmA, fb, k, pc.mc);
    } else if (p.a3d) {
      tma_load_3d(dA, &tmA, fb, 0, k - p.k_sh, pc.mc >> 4);
    } else {
#pragma unroll
      for (int i = 0; i < BM / 16; ++i) tma_load_2d(dA + i * 2048, &tmA, fb, pc.mc + 16 * i, k - p.k_sh);
    }
    if (!TB) {
      tma_load_2d(dB, &tmB, fb, k, pc.nc);
    } else if (p.b3d) {
      tma_load_3d(dB, &tmB, fb, 0, k - p.k_sh, pc.nc >> 4);
    } else {
#pragma unroll
      for (int i = 0; i < BN / 16; ++i) tma_load_2d(dB + i * 2048, &tmB, fb, pc.nc + 16 * i, k - p.k_sh);
    }
    ++pg;
    if (++pit == pnk) {
      pit = 0;
      ptile = next_tile(ptile);
      if (ptile >= 0) {
        pc = tile_of(p, ptile);
        pnk = nk_of(pc);
        pkb = kbeg_of(pc);
      }
    }
  };
  auto load_c = [&](int t) {
    const TileCoord c = tile_of(p, t);
    const int m0 = c.mc - (TA ? 0 : p.a_sh), n0 = c.nc - (TB ? p.b_sh : 0);
    mbar_arrive_expect_tx(cfull, C_BYTES);
#pragma unroll
    for (int i = 0; i < BM / 16; ++i)
      tma_load_2d(smem_u32(sC + i * 16 * BN), &tmC, cfull, m0 + p.c_sh + 16 * i, n0);
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (HASC && p.beta != 0.0 && ptile >= 0) load_c(ptile);
    for (int i = 0; i < STAGES - 1; ++i) produce_one();
  }

  const int wm = warp & 1, wn = warp >> 1;
  const int fr = lane >> 2, fk = lane & 3;
  int arow[8], bcol[4];
#pragma unroll
  for (int t = 0; t < 8; ++t) arow[t] = frag_row<TA>(wm, t, fr);
#pragma unroll
  for (int u = 0; u < 4; ++u) bcol[u] = frag_col<TB>(wn, u, fr);

  long g = 0;   // global consumed k-block count
#ifdef GEMM_PROBE
  long long gp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const bool gprobe = blockIdx.x == 0 && lane == 0 && warp < 2;
  long long gt0 = clock64();
#endif
  for (int local = 0;; ++local) {
    // the first stage of the tile publishes its id (or the -1 sentinel)
    if (threadIdx.x == 0 && pg < g + STAGES) produce_one();
    __syncwarp();
    mbar_wait(full0 + 8 * (int)(g % STAGES), (uint32_t)((g / STAGES) & 1));
    const int tile = tq[local & 7];
#ifdef GEMM_PROBE
    long long gt1 = clock64();
    gp[0] += gt1 - gt0;
#endif
    if (tile < 0) break;
    const TileCoord tc = tile_of(p, tile);
    const int nk = nk_of(tc);
    double acc[8][4][2];
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;

    const bool zero_k0 = (p.k_sh != 0) && (tc.z == 0);
    for (int it = 0; it < nk; ++it, ++g) {
      if (threadIdx.x == 0 && it > 0 && pg < g + STAGES) produce_one();
      __syncwarp();
      const int s = (int)(g % STAGES);
#ifdef GEMM_PROBE
      const long long gw0 = clock64();
#endif
      mbar_wait(full0 + 8 * s, (uint32_t)((g / STAGES) & 1));
#ifdef GEMM_PROBE
      gp[2] += clock64() - gw0;
#endif
      const double* a = sA + s * A_ST;
      const double* b = sB + s * B_ST;
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        const int k = kk * 4 + fk;
        double af[8], bf[4];
#pragma unroll
        for (int t = 0; t < 8; ++t) af[t] = a[a_off_of<TA>(k, arow[t])];
        // k' = 0 is the logical row k = -1 when the K origin is shifted: when
        // both operands carry real data there (TN), zero it in registers.
        if (zero_k0 && it == 0 && kk == 0 && fk == 0) {
#pragma unroll
          for (int t = 0; t < 8; ++t) af[t] = 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) bf[u] = b[b_off_of<TB>(k, bcol[u])];
#pragma unroll
        for (int t = 0; t < 8; ++t)
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma884(acc[t][u][0], acc[t][u][1], af[t], bf[u]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * s);
    }

    // ---------------- epilogue ----------------
#ifdef GEMM_PROBE
    {
      const long long gt2 = clock64();
      gp[1] += gt2 - gt1;
      gt1 = gt2;
      gp[4] += 1;
    }
#endif
    const int m0 = tc.mc - (TA ? 0 : p.a_sh), n0 = tc.nc - (TB ? p.b_sh : 0);
    if (!HASC && p.flags) {
      // fused split-K (no C tile prefetch: splits > 1 never has HASC)
      const int per = p.tm * p.tn;
      const int r = tile - tc.z * per;
      const int zf = p.tri_a ? ((tc.mc / BK) * BK) / p.k_split : 0;   // first non-empty split
      const int zl = p.tiles / per - 1;
      const bool first = tc.z == zf, last = tc.z == zl;
      double* wt = p.ws + (size_t)r * (BM * BN);
      if (!first) {
        if (threadIdx.x == 0) {
          while (ld_acquire(p.flags + r) != tc.z - zf) __nanosleep(64);
        }
        __syncthreads();
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int ml = frag_row<TA>(wm, t, fr);
        const int m = m0 + ml;
        const bool mok = (m >= 0 && m < p.M);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int nl = frag_col<TB>(wn, u, 2 * fk + j);
            double* wp = wt + ml + nl * BM;
            double v = acc[t][u][j];
            if (!first) v = __ldcg(wp) + v;                 // splits summed in split order
            if (!last) {
              __stcg(wp, v);
            } else {
              const int n = n0 + nl;
              if (mok && n >= 0 && n < p.N) {
                double* c = p.C + m + (long)n * p.ldc;
                *c = (p.beta == 0.0) ? p.alpha * v : fma(p.beta, *c, p.alpha * v);
              }
            }
          }
      }
      __syncthreads();  // every thread's partial stores issued
      if (threadIdx.x == 0) {
        __threadfence();
        if (last) p.flags[r] = 0;                          // reset for the next launch
        else st_release(p.flags + r, tc.z - zf + 1);
      }
      continue;
    }
    if (HASC && p.beta != 0.0) mbar_wait(cfull, (uint32_t)(local & 1));
    double* w = p.ws ? p.ws + (size_t)tc.z * p.N * p.M : nullptr;
    // beta != 0 with an unshifted C map: alpha*acc + beta*C is written back
    // over the prefetched C tile in smem and leaves by one TMA store, so the
    // warps start the next tile without draining 128 KB of stores first.
    // (tile origins at a -1 row/column shift keep the direct stores)
    // A TMA store writes whole 16-byte granules: with an odd row count the
    // granule holding row M-1 also covers row M, outside the matrix, so the
    // tile containing the last row of an odd-M matrix keeps the direct stores.
    const bool tstore = HASC && p.c_sh == 0 && !w && m0 >= 0 && n0 >= 0 &&
                        ((p.M & 1) == 0 || m0 + BM <= p.M);
    // Fast paths (the common case): the smem C tile, or a direct store of an
    // interior tile.  Per fragment row t the eight sC values are gathered
    // before any is written back (stores cannot alias the later loads, so
    // the LDS issue back to back instead of one LDS -> DFMA -> STS round
    // trip per element), and interior stores go through eight precomputed
    // column pointers with compile-time row offsets (no bounds or address
    // arithmetic per element).  tools/gemm_probe.cu: the epilogue took
    // ~7000 of ~80000 cycles per K = 256 tile.
    const bool interior = !w && m0 >= 0 && n0 >= 0 && m0 + BM <= p.M && n0 + BN <= p.N;
    if (HASC && tstore) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int ml = frag_row<TA>(wm, t, fr);
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // four values at a time (register pressure)
          double* cs[4];
          double cv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            cs[k] = &sC[swz((ml >> 4) * BN + frag_col<TB>(wn, 2 * h + (k >> 1), 2 * fk + (k & 1)), ml & 15)];
          if (p.beta != 0.0) {
#pragma unroll
            for (int k = 0; k < 4; ++k) cv[k] = *cs[k];
#pragma unroll
            for (int k = 0; k < 4; ++k) *cs[k] = fma(p.beta, cv[k], p.alpha * acc[t][2 * h + (k >> 1)][k & 1]);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) *cs[k] = p.alpha * acc[t][2 * h + (k >> 1)][k & 1];
          }
        }
      }
    } else if (!HASC && interior) {
      double* cp[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        cp[k] = p.C + m0 + (long)(n0 + frag_col<TB>(wn, k >> 1, 2 * fk + (k & 1))) * p.ldc;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int ml = frag_row<TA>(wm, t, fr);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double v = p.alpha * acc[t][k >> 1][k & 1];
          cp[k][ml] = (p.beta == 0.0) ? v : fma(p.beta, cp[k][ml], v);
        }
      }
    } else {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int ml = frag_row<TA>(wm, t, fr);
      const int m = m0 + ml;
      const bool mok = (m >= 0 && m < p.M);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int nl = frag_col<TB>(wn, u, 2 * fk + j);
          const int n = n0 + nl;
          double v = p.alpha * acc[t][u][j];
          if (HASC) {
            double* cs = &sC[swz((ml >> 4) * BN + nl, ml & 15)];
            if (p.beta != 0.0) v = fma(p.beta, *cs, v);
          }
          if (mok && n >= 0 && n < p.N) {
            if (w) w[m + (size_t)n * p.M] = acc[t][u][j];
            else p.C[m + (long)n * p.ldc] = v;
          }
        }
    }
    }
    if (HASC && p.wstore) {
      // per-warp epilogue: each warp stores its own 64 x 32 sub-tile with
      // four 16 x 32 TMA boxes as soon as IT has written them — no CTA
      // barrier, so the other warps are already into the next tile's main
      // loop; thread 0 prefetches the next C tile once all eight warps'
      // stores have read sC (cempty).
      if (tstore) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rg = wm * 4 + i;  // 16-row group of this warp
            tma_store_2d(&tmCw, smem_u32(sC + rg * 16 * BN + wn * 32 * 16), m0 + 16 * rg, n0 + 32 * wn);
          }
          bulk_commit();
          bulk_wait_read0();
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(cempty);
      if (threadIdx.x == 0) {
        mbar_wait(cempty, (uint32_t)(local & 1));
        const int nxt = tq[(local + 1) & 7];
        if (nxt >= 0 && p.beta != 0.0) load_c(nxt);
      }
    } else if (HASC) {
      if (tstore) fence_proxy_async_smem();  // generic smem writes -> async proxy
      __syncthreads();  // every warp is done with sC
      if (threadIdx.x == 0) {
        if (tstore) {
#pragma unroll
          for (int i = 0; i < BM / 16; ++i) tma_store_2d(&tmC, smem_u32(sC + i * 16 * BN), m0 + 16 * i, n0);
          bulk_commit();
          bulk_wait_read0();  // sC may be refilled once the store has read it
        }
        const int nxt = tq[(local + 1) & 7];  // published: the producer runs >= 1 k-block ahead
        if (nxt >= 0 && p.beta != 0.0) load_c(nxt);
      }
    }
#ifdef GEMM_PROBE
    gt0 = clock64();
    gp[3] += gt0 - gt1;
#endif
  }
#ifdef GEMM_PROBE
  if (gprobe)
    for (int i = 0; i < 8; ++i) g_gprobe[warp][i] += gp[i];
#endif
  if (HASC && (threadIdx.x == 0 || (p.wstore && lane == 0))) bulk_wait0();
}

// C = alpha * sum_s ws[s] + beta * C, summed in split order (deterministic).
// tri_ksplit > 0 (triangular A): splits that lie entirely left of a row
// tile's first k were never computed and are skipped.
__global__ void splitk_reduce_kernel(const double* __restrict__ ws, int splits, int M, int N,
                                     double alpha, double beta, double* C, long ldc,
                                     int tri_ksplit) {
  // 2-D walk (column n, row pair m, m+1): no 64-bit index division per
  // element, 16-byte partial loads (the workspace has ld = M, M even here
  // or the pair degrades to one row), all splits' loads in flight together.
  const size_t total = (size_t)M * N;
  const int pairs = (M + 1) >> 1;
  const bool vec = (M & 1) == 0;
  for (int n = blockIdx.y; n < N; n += gridDim.y) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < pairs; p += gridDim.x * blockDim.x) {
      const int m = 2 * p;
      const int z0 = tri_ksplit > 0 ? ((m / BM) * BM / BK * BK) / tri_ksplit : 0;  // m, m+1: same tile
      const size_t i = (size_t)n * M + m;
      double s0 = 0.0, s1 = 0.0;
      if (vec) {
#pragma unroll 4
        for (int z = z0; z < splits; ++z) {
          const double2 w = __ldcs((const double2*)(ws + (size_t)z * total + i));
          s0 += w.x;
          s1 += w.y;
        }
      } else {
        for (int z = z0; z < splits; ++z) {
          s0 += __ldcs(ws + (size_t)z * total + i);
          if (m + 1 < M) s1 += __ldcs(ws + (size_t)z * total + i + 1);
        }
      }
      double* c = C + m + (long)n * ldc;
      c[0] = (beta == 0.0) ? alpha * s0 : fma(beta, c[0], alpha * s0);
      if (m + 1 < M) c[1] = (beta == 0.0) ? alpha * s1 : fma(beta, c[1], alpha * s1);
    }
  }
}

__global__ void scale_kernel(int M, int N, double beta, double* C, long ldc) {
  const size_t total = (size_t)M * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int m = (int)(i % M), n = (int)(i / M);
    double* c = C + m + (long)n * ldc;
    *c = (beta == 0.0) ? 0.0 : beta * *c;
  }
}

}  // namespace gemm

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
typedef CUresult (*PFN_memRange)(CUdeviceptr*, size_t*, CUdeviceptr);
static PFN_memRange g_range = nullptr;
static std::once_flag g_encode_once;
static int g_num_sms = 0;

static int get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    void* fr = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_range = (PFN_memRange)fr;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    for (auto f : {gemm::dgemm_tma_kernel<false, false, false>, gemm::dgemm_tma_kernel<false, true, false>,
                   gemm::dgemm_tma_kernel<true, false, false>, gemm::dgemm_tma_kernel<true, true, false>})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm::Cfg<false>::SMEM);
    for (auto f : {gemm::dgemm_tma_kernel<false, false, true>, gemm::dgemm_tma_kernel<false, true, true>,
                   gemm::dgemm_tma_kernel<true, false, true>, gemm::dgemm_tma_kernel<true, true, true>})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm::Cfg<true>::SMEM);
  });
  return g_encode ? UTV_OK : UTV_ERR_CUDA;
}

int num_sms() {
  get_encode();
  return g_num_sms > 0 ? g_num_sms : 148;
}

// ---- dynamic tile scheduler slots: one [ticket, done] pair per stream ----
static std::mutex g_sched_mu;
static int* g_sched = nullptr;
static cudaStream_t g_sched_streams[64];
static int g_sched_n = 0;

int* gemm_sched_slot(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_sched_mu);
  if (!g_sched) {
    if (cudaMalloc((void**)&g_sched, 2 * 64 * sizeof(int)) != cudaSuccess) return nullptr;
    if (cudaMemset(g_sched, 0, 2 * 64 * sizeof(int)) != cudaSuccess) return nullptr;
  }
  for (int i = 0; i < g_sched_n; ++i)
    if (g_sched_streams[i] == st) return g_sched + 2 * i;
  if (g_sched_n == 64) return nullptr;  // fall back to static scheduling
  g_sched_streams[g_sched_n] = st;
  return g_sched + 2 * (g_sched_n++);
}

// ---- fused split-K turn counters: FLAG_TILES per stream slot ----
constexpr int FLAG_TILES = 4096;
static int* g_flags = nullptr;

static int* gemm_flag_slot(cudaStream_t st) {
  int* sched = gemm_sched_slot(st);  // same slot index as the tile scheduler
  if (!sched) return nullptr;
  std::lock_guard<std::mutex> lk(g_sched_mu);
  if (!g_flags) {
    if (cudaMalloc((void**)&g_flags, sizeof(int) * 64 * FLAG_TILES) != cudaSuccess) return nullptr;
    if (cudaMemset(g_flags, 0, sizeof(int) * 64 * FLAG_TILES) != cudaSuccess) return nullptr;
  }
  return g_flags + (size_t)((sched - g_sched) / 2) * FLAG_TILES;
}

// CTA budget of the next GEMM launches on this host thread (0 = all SMs):
// drivers lower it while a latency-bound kernel runs on a side stream.
static thread_local int g_max_ctas = 0;
void gemm_set_max_ctas(int n) { g_max_ctas = n; }

// Tensor map over a column-major (rows x cols) matrix with leading dim ld.
// TMA needs a 16B-aligned origin and 16B-aligned box starts in dim0, so an
// 8B-aligned (odd-row) sub-matrix is mapped from one element above; *shift
// returns that offset (0/1).  Box starts stay even; the kernel shifts its
// logical tile origin instead (M/N dims) or runs the K loop over k' = k +
// shift with the other operand reading k' - shift (TMA zero-fills the
// out-of-range k = -1 slot, so the extra row contributes exactly 0).
static int make_map(CUtensorMap* map, const double* p, long rows, long cols, long ld,
                    uint32_t box0, uint32_t box1, int* shift) {
  if ((ld & 1) || ((uintptr_t)p & 7)) return UTV_ERR_ALIGN;
  int sh = ((uintptr_t)p & 15) ? 1 : 0;
  const double* base = p - sh;
  cuuint64_t dims[2] = {(cuuint64_t)(rows + sh), (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box,
                        es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "libutvb200: cuTensorMapEncodeTiled failed (%d) rows=%ld cols=%ld ld=%ld\n",
            (int)r, rows, cols, ld);
    return UTV_ERR_CUDA;
  }
  *shift = sh;
  return UTV_OK;
}

// 3-D view {16 rows, cols, ceil((rows+sh)/16) row blocks} of an N-major
// operand, so one TMA box {16, 16, 8} moves a whole 128 x 16 tile.  Rows past
// `rows` in the last block are READ (not zero-filled); they only feed output
// rows/columns that are never stored, so the map is used only when that
// over-read stays inside the pointer's allocation (cuMemGetAddressRange).
// Returns false (caller keeps the 2-D map) otherwise.
static bool make_map3d(CUtensorMap* map, const double* p, long rows, long cols, long ld, int sh) {
  if (!g_range || cols <= 0) return false;
  const double* base = p - sh;
  const long nblk = (rows + sh + 15) / 16;
  CUdeviceptr abase = 0;
  size_t asize = 0;
  if (g_range(&abase, &asize, (CUdeviceptr)p) != CUDA_SUCCESS) return false;
  const uint64_t last = (uint64_t)(base + (cols - 1) * ld + 16 * nblk);  // one past the over-read
  if ((uint64_t)base < abase || last > abase + asize) return false;
  if (nblk > (1l << 31) || ld * 8 >= (1l << 40)) return false;
  cuuint64_t dims[3] = {16, (cuuint64_t)cols, (cuuint64_t)nblk};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 8), 128};
  cuuint32_t box[3] = {16, 16, (cuuint32_t)(gemm::BM / 16)};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)base, dims, strides, box,
                        es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

size_t dgemm_ws_doubles(int M, int N, int K) {
  // Upper bound of split-K workspace chosen by dgemm() below.
  int tiles = ceil_div(M, gemm::BM) * ceil_div(N, gemm::BN);
  int splits = choose_splits(tiles, K);
  return splits > 1 ? (size_t)splits * M * N : 0;
}

int choose_splits(int tiles, int K) {
  const int sms = num_sms();
  const int kblocks = ceil_div(K, gemm::BK);
  const double eff1 = (double)tiles / (ceil_div(tiles, sms) * sms);
  if (tiles >= sms) {
    // Many tiles: split only a long-K GEMM whose last wave is badly filled
    // (e.g. the 16384 x 256 sampling GEMMs: 256 tiles = 1.73 waves).
    if (eff1 >= 0.9 || kblocks < 64) return 1;
    int best = 1;
    double best_eff = eff1;
    for (int s = 2; s <= 8 && kblocks / s >= 32; ++s) {
      const int units = tiles * s;
      const double eff = (double)units / (ceil_div(units, sms) * sms);
      if (eff > best_eff + 0.03) {
        best = s;
        best_eff = eff;
      }
    }
    return best;
  }
  if (kblocks < 8) return 1;
  // Few tiles: pick the split count (each split keeps >= 8 k-blocks)
  // maximising wave efficiency; ties go to fewer splits.
  int best = 1;
  double best_eff = eff1;
  for (int s = 2; s <= 64 && kblocks / s >= 8; ++s) {
    const int units = tiles * s;
    const double eff = (double)units / (ceil_div(units, sms) * sms);
    if (eff > best_eff + 0.02) {
      best = s;
      best_eff = eff;
    }
    if (units >= 2 * sms && eff > 0.9) break;
  }
  return best;
}

int dgemm(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, long lda,
          const double* B, long ldb, double beta, double* C, long ldc, double* ws,
          size_t ws_doubles, cudaStream_t st) {
  return dgemm_ex(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_doubles, st, false);
}

int dgemm_ex(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, long lda,
             const double* B, long ldb, double beta, double* C, long ldc, double* ws,
             size_t ws_doubles, cudaStream_t st, bool tri_a) {
  if (M <= 0 || N <= 0) return UTV_OK;
  UTV_CHECK(get_encode());
  if (K <= 0 || alpha == 0.0) {
    if (beta == 1.0) return UTV_OK;
    ProfScope ps(PROF_OPS, 0.0, 16.0 * M * N, st);
    gemm::scale_kernel<<<min(4 * num_sms(), ceil_div((long)M * N, 256)), 256, 0, st>>>(M, N, beta, C, ldc);
    UTV_CUDA(cudaGetLastError());
    return UTV_OK;
  }
  // TN with K-origins of different parity: re-stage the smaller operand with
  // the other's parity (rare: only odd block sizes / odd user offsets).
  const double* Ause = A;
  long ldause = lda;
  const double* Buse = B;
  long ldbuse = ldb;
  double* tmp = nullptr;
  if (ta && !tb && (((uintptr_t)A & 15) != 0) != (((uintptr_t)B & 15) != 0)) {
    const bool copyA = (long)K * M <= (long)K * N;
    const int sh = copyA ? (((uintptr_t)B & 15) ? 1 : 0) : (((uintptr_t)A & 15) ? 1 : 0);
    const long cols = copyA ? M : N;
    const long ldt = round_up(K + 1, 2);
    UTV_CUDA(cudaMallocAsync((void**)&tmp, sizeof(double) * (ldt * cols + 2), st));
    double* dst = tmp + sh;
    UTV_CHECK(copy_mat(copyA ? A : B, copyA ? lda : ldb, dst, ldt, K, (int)cols, st));
    if (copyA) { Ause = dst; ldause = ldt; } else { Buse = dst; ldbuse = ldt; }
  }
  CUtensorMap mA, mB;
  int shA = 0, shB = 0;
  if (ta) UTV_CHECK(make_map(&mA, Ause, K, M, ldause, 16, gemm::BM, &shA));
  else UTV_CHECK(make_map(&mA, Ause, M, K, ldause, 16, 16, &shA));
  if (tb) UTV_CHECK(make_map(&mB, Buse, N, K, ldbuse, 16, 16, &shB));
  else UTV_CHECK(make_map(&mB, Buse, K, N, ldbuse, 16, gemm::BN, &shB));
  const int a_sh = ta ? 0 : shA, b_sh = tb ? shB : 0;
  int a3d = 0, b3d = 0;
  if (!ta) {
    CUtensorMap m3;
    if (make_map3d(&m3, Ause, M, K, ldause, shA)) { mA = m3; a3d = 1; }
  }
  if (tb) {
    CUtensorMap m3;
    if (make_map3d(&m3, Buse, N, K, ldbuse, shB)) { mB = m3; b3d = 1; }
  }
  const int k_sh = ta ? shA : (!tb ? shB : 0);

  const int tm = ceil_div(M + a_sh, gemm::BM), tn = ceil_div(N + b_sh, gemm::BN);
  const int Kp = K + k_sh;
  // triangular A only in the plain layout (no origin shifts, one split)
  const bool tri = tri_a && !ta && a_sh == 0 && k_sh == 0 && M == K;
  // (split-K units left of a row tile's first k are skipped, see empty_unit)
  int splits = choose_splits(tm * tn, Kp);
  if (ws == nullptr) splits = 1;
  while (splits > 1 && (size_t)splits * M * N > ws_doubles) --splits;
  int kper = (int)round_up(ceil_div(Kp, splits), gemm::BK);
  splits = ceil_div(Kp, kper);

  // beta != 0 without split-K: the C tile is TMA-prefetched; its map must
  // share the A tile's row parity (always true for even offsets).
  // beta == 0 may also take the smem-staged epilogue (accumulators -> smem ->
  // one TMA store, no C prefetch): the warps start the next tile after the
  // ~0.5 us smem write instead of ~2 us of direct global stores, at the
  // price of the 3-stage ring.  Tuning knob UTV_GEMM_TSTORE0 (0 = off).
  static const bool tstore0 = [] {
    const char* e = getenv("UTV_GEMM_TSTORE0");
    return e ? atoi(e) != 0 : false;
  }();
  bool hasc = (beta != 0.0 || tstore0) && splits == 1;
  CUtensorMap mC = mA;
  int c_sh = 0;
  if (hasc) {
    UTV_CHECK(make_map(&mC, C, M, N, ldc, 16, gemm::BN, &c_sh));
    if (c_sh != a_sh) hasc = false;
  }
  // per-warp C stores (16 x 32 boxes of the same swizzled smem tile)
  static const bool wstore = [] {
    const char* e = getenv("UTV_GEMM_WSTORE");  // tuning knob (0 = one CTA-wide TMA store)
    return e ? atoi(e) != 0 : true;
  }();
  CUtensorMap mCw = mC;
  if (hasc && wstore) {
    int c_sh2 = 0;
    UTV_CHECK(make_map(&mCw, C, M, N, ldc, 16, 32, &c_sh2));
  }
  // beta != 0 with a C map of the wrong parity (odd offsets only): route
  // through the split-K workspace path (one split) + the reduce kernel.
  double* ctmp = nullptr;
  if (beta != 0.0 && splits == 1 && !hasc) {
    if (ws == nullptr || ws_doubles < (size_t)M * N) {
      UTV_CUDA(cudaMallocAsync((void**)&ctmp, sizeof(double) * (size_t)M * N, st));
      ws = ctmp;
    }
  }
  const bool use_ws = splits > 1 || (beta != 0.0 && !hasc);

  gemm::Args a;
  a.M = M; a.N = N; a.K = K;
  a.a_sh = a_sh; a.b_sh = b_sh; a.k_sh = k_sh; a.c_sh = c_sh;
  a.a3d = a3d; a.b3d = b3d;
  a.k_split = kper;
  a.tm = tm; a.tn = tn; a.tiles = tm * tn * splits;
  a.alpha = alpha; a.beta = beta;
  a.C = C; a.ldc = ldc;
  a.ws = use_ws ? ws : nullptr;
  a.sched = gemm_sched_slot(st);
  a.tri_a = tri ? 1 : 0;
  // Fused split-K when the dynamic scheduler is on (tickets in split-major
  // order: a split only ever waits for a lower ticket, already held by a
  // running CTA -> no deadlock), the per-tile sums fit the workspace
  // tile-major, and the serial chain of S epilogues stays short.
  static const int fuse_max = [] {
    // tuning knob, default 0 = the separate reduce kernel: the serial chain
    // of S epilogues measured slower than one reduce launch (TN 256x16384x16384:
    // 33.5 -> 32.3 TF/s; headline step +35 ms in randUTV, profiles/r02_ab_groups.txt)
    const char* e = getenv("UTV_SPLITK_FUSE_MAX");
    return e ? atoi(e) : 0;
  }();
  a.wstore = (hasc && wstore) ? 1 : 0;
  a.flags = nullptr;
  if (splits > 1 && splits <= fuse_max && a.sched && tm * tn <= FLAG_TILES &&
      (size_t)tm * tn * gemm::BM * gemm::BN <= ws_doubles)
    a.flags = gemm_flag_slot(st);
  const bool fused = a.flags != nullptr;
  double fl = 2.0 * M * N * K;
  if (tri) {
    fl = 0.0;
    for (int t = 0; t < tm; ++t) {
      const int mc = t * gemm::BM, rows = min(gemm::BM, M - mc);
      fl += 2.0 * N * rows * (K - (mc / gemm::BK) * gemm::BK);
    }
  }
  int cap = num_sms();
  if (g_max_ctas > 0 && g_max_ctas < cap) cap = g_max_ctas;
  static const int env_cap = [] {  // debug knob: grid cap of every GEMM (0 = off)
    const char* e = getenv("UTV_GEMM_CTAS");
    return e ? atoi(e) : 0;
  }();
  if (env_cap > 0 && env_cap < cap) cap = env_cap;
  const int grid = a.tiles < cap ? a.tiles : cap;
  {
  ProfScope ps(PROF_GEMM, fl, 8.0 * ((double)M * K + (double)K * N + (beta != 0.0 ? 2.0 : 1.0) * M * N), st);
  if (hasc) {
    const size_t sm = gemm::Cfg<true>::SMEM;
    if (!ta && !tb) gemm::dgemm_tma_kernel<false, false, true><<<grid, gemm::THREADS, sm, st>>>(mA, mB, mC, mCw, a);
    else if (!ta && tb) gemm::dgemm_tma_kernel<false, true, true><<<grid, gemm::THREADS, sm, st>>>(mA, mB, mC, mCw, a);
    else if (ta && !tb) gemm::dgemm_tma_kernel<true, false, true><<<grid, gemm::THREADS, sm, st>>>(mA, mB, mC, mCw, a);
    else gemm::dgemm_tma_kernel<true, true, true><<<grid, gemm::THREADS, sm, st>>>(mA, mB, mC, mCw, a);
  } else {
    const size_t sm = gemm::Cfg<false>::SMEM;
    if (!ta && !tb) gemm::dgemm_tma_kernel<false, false, false><<<grid, gemm::THREADS, sm, st>>>(mA, mB, mC, mCw, a);
    else if (!ta && tb) gemm::dgemm_tma_kernel<false, true, false><<<grid, gemm::THREADS, sm, st>>>(mA, mB, mC, mCw, a);
    else if (ta && !tb) gemm::dgemm_tma_kernel<true, false, false><<<grid, gemm::THREADS, sm, st>>>(mA, mB, mC, mCw, a);
    else gemm::dgemm_tma_kernel<true, true, false><<<grid, gemm::THREADS, sm, st>>>(mA, mB, mC, mCw, a);
  }
  UTV_CUDA(cudaGetLastError());
  }
  if (use_ws && !fused) {
    const long total = (long)M * N;
    ProfScope ps(PROF_SPLITK, 0.0, 8.0 * (splits + (beta != 0.0 ? 2 : 1)) * total, st);
    const int gx = ceil_div(ceil_div(M, 2), 256);
    const int gy = (int)std::min<long>(N, std::max<long>(1, 8L * num_sms() / gx));
    gemm::splitk_reduce_kernel<<<dim3(gx, gy), 256, 0, st>>>(ws, splits, M, N, alpha, beta, C, ldc,
                                                            tri ? kper : 0);
    UTV_CUDA(cudaGetLastError());
  }
  if (ctmp) UTV_CUDA(cudaFreeAsync(ctmp, st));
  if (tmp) UTV_CUDA(cudaFreeAsync(tmp, st));
  return UTV_OK;
}

}  // namespace utv
