// K10: FP32 GEMM on the 5th-generation tensor cores, 3xTF32 split.
//
//   C = alpha * op(A) * op(B) + beta * C      (fp32, column-major, op in {N, T})
//
// The fp32 variant of randUTV (BASELINE C5) needs
// FP32-accurate products: plain TF32 sampling wrecks rank revelation
// (SURVEY §7 hard part 6).  Every operand element is split x = hi + lo with
// hi = rna_tf32(x) and lo = x - hi (exact in fp32); the tensor cores
// accumulate hi*hi + hi*lo + lo*hi in FP32 (TMEM).  With hi rounded to
// nearest, |lo| <= 2^-11 |x| and the (truncated) tf32 lo loses at most
// 2^-22 |x|: the product error is fp32-level.
//
// Design (sm_100a, warp-specialised, persistent):
//   warp 0      TMA producer: raw fp32 tiles A (128 x 32) and B (128 x 32)
//               into a RAW_STAGES ring (mbarrier full/empty, expect_tx);
//               K-major A tiles arrive 128B-swizzled
//   warp 1      TMEM allocator + MMA issuer (one elected lane):
//               12 x tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=128, K=8)
//               per 32-deep k-block, A from TMEM, B from shared memory,
//               tcgen05.commit -> mbarriers
//   warps 4-11  converters: A rows -> hi / lo straight into TMEM
//               (tcgen05.st, each warp in its lane quarter, 16 k columns);
//               B (K- or MN-major) -> hi / lo tiles in the canonical K-major
//               128B-swizzled UMMA layout in shared memory;
//               tcgen05.fence + fence.proxy.async before arrival
//   warps 12-27 epilogue: tcgen05.ld 32x32b from a double-buffered TMEM
//               accumulator (2 x 128 columns).  The tensor-core FP32
//               accumulator does not round to nearest, so K is split into
//               512-deep chunks folded with round-to-nearest adds into a
//               running sum in TMEM — long-K products stay fp32-accurate;
//               alpha/beta, coalesced stores; overlaps the next tile's MMAs.
// TMEM (512 columns): [0, 256) accumulators, [256, 384) running sum,
// [384, 512) A hi|lo for the two conversion stages.  Moving A's split out of
// shared memory halved the converters' smem stores, which had saturated
// the L1/smem pipe (l1tex 81% -> 57%).  16 converter warps (8 epilogue)
// measured slower (C5 sampling GEMM 186 -> 173 TF/s useful).
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "utv_internal.h"

namespace utv {

namespace tf32 {
constexpr int BM = 128, BN = 128, BK = 32;
constexpr int RAW_STAGES = 4, CONV_STAGES = 2, ACC_STAGES = 2;
constexpr int THREADS = 896;                  // 28 warps
constexpr int CONV_WARP0 = 4, NCONV = 8;      // converter warps 4..11
constexpr int EPI_WARP0 = 12;                 // epilogue warps 12..27 (4 per TMEM lane quarter)
constexpr int EPI_COLS = 32;                  // accumulator columns per epilogue thread
constexpr int CHUNK_KB = 16;                  // k-blocks (512 k) per TMEM accumulation chunk
constexpr uint32_t TILE_BYTES = BM * BK * 4;  // 16 KB (A or B, raw or hi or lo)
constexpr uint32_t RAW_BYTES = 2 * TILE_BYTES;
constexpr uint32_t CONV_BYTES = 2 * TILE_BYTES;  // hiB loB (A's hi/lo live in TMEM)
constexpr size_t SMEM = (size_t)RAW_STAGES * RAW_BYTES + (size_t)CONV_STAGES * CONV_BYTES + 1024 + 512;
constexpr uint32_t SUM_COL = ACC_STAGES * BN;   // running chunk sum (128 columns) after the buffers
constexpr uint32_t A_COL = SUM_COL + BN;         // A operand hi|lo per conversion stage (2 x 64 columns)
constexpr uint32_t TMEM_COLS = 512;              // 2 x 128 accumulator + 128 running sum + 128 A

struct Args {
  int M, N, K;
  int tm, tn, tiles;
  float alpha, beta;
  float* C;
  long ldc;
  int* sched;  // dynamic tile scheduler [ticket, done] (self-resetting) or null
};

// K-major, 128B-swizzled UMMA shared-memory descriptor (SM100, version 1):
// rows of 128 B, 8-row atoms 1024 B apart (SBO), LBO unused (1).
__device__ __forceinline__ uint64_t kmajor_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // version (Blackwell)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M=128, N=128.
__host__ __device__ constexpr uint32_t idesc_tf32() {
  return (1u << 4)                    // c_format F32
         | (2u << 7)                  // a_format TF32
         | (2u << 10)                 // b_format TF32
         | ((uint32_t)(BN >> 3) << 17)
         | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc_tf32()), "r"(accum));
}

// A from TMEM (M = 128 lanes x 8 tf32 columns), B from shared memory.
__device__ __forceinline__ void umma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc_tf32()), "r"(accum));
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(THREADS, 1)
    sgemm_tf32x3_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const Args p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* raw = smem;                                   // [RAW_STAGES][A | B]
  unsigned char* conv = raw + RAW_STAGES * RAW_BYTES;          // [CONV_STAGES][hiA loA hiB loB]
  uint64_t* bars = (uint64_t*)(conv + CONV_STAGES * CONV_BYTES);
  const uint32_t raw_full = smem_u32(bars), raw_empty = raw_full + 8 * RAW_STAGES;
  const uint32_t conv_full = raw_empty + 8 * RAW_STAGES, conv_empty = conv_full + 8 * CONV_STAGES;
  const uint32_t acc_full = conv_empty + 8 * CONV_STAGES, acc_empty = acc_full + 8 * ACC_STAGES;
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * (RAW_STAGES + CONV_STAGES + ACC_STAGES));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (p.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RAW_STAGES; ++s) {
      mbar_init(raw_full + 8 * s, 1);
      mbar_init(raw_empty + 8 * s, NCONV);
    }
    for (int s = 0; s < CONV_STAGES; ++s) {
      mbar_init(conv_full + 8 * s, NCONV);
      mbar_init(conv_empty + 8 * s, 1);
    }
    for (int s = 0; s < ACC_STAGES; ++s) {
      mbar_init(acc_full + 8 * s, 2);  // tcgen05.commit + the MMA lane's release arrive
      mbar_init(acc_empty + 8 * s, 16);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem_base = *tmem_slot;

  // Tile ids (dynamic tickets, -1 = no more work) travel producer ->
  // converters -> MMA -> epilogue through tq[], published before the first
  // barrier arrival of each tile; the sentinel flows down the same barriers.
  volatile int* tq = (volatile int*)(tmem_slot + 2);  // [16]
  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      long g = 0;
      int prev = -1;
      for (int local = 0;; ++local) {
        int tile;
        if (!p.sched) {
          tile = prev < 0 ? (int)blockIdx.x : prev + (int)gridDim.x;
          if (tile >= p.tiles) tile = -1;
        } else {
          tile = atomicAdd(p.sched, 1);
          if (tile >= p.tiles) {
            tile = -1;
            if (atomicAdd(p.sched + 1, 1) == (int)gridDim.x - 1) {
              atomicExch(p.sched, 0);
              atomicExch(p.sched + 1, 0);
            }
          }
        }
        prev = tile;
        const int s0 = (int)(g % RAW_STAGES);
        if (g >= RAW_STAGES) mbar_wait(raw_empty + 8 * s0, (uint32_t)(((g / RAW_STAGES) & 1) ^ 1));
        tq[local & 15] = tile;
        if (tile < 0) {
          mbar_arrive(raw_full + 8 * s0);  // sentinel: completes the phase with no data
          break;
        }
        const int mc = (tile % p.tm) * BM, nc = (tile / p.tm) * BN;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = (int)(g % RAW_STAGES);
          if (kb > 0 && g >= RAW_STAGES) mbar_wait(raw_empty + 8 * s, (uint32_t)(((g / RAW_STAGES) & 1) ^ 1));
          const uint32_t fb = raw_full + 8 * s;
          mbar_arrive_expect_tx(fb, RAW_BYTES);
          const uint32_t dA = smem_u32(raw + s * RAW_BYTES), dB = dA + TILE_BYTES;
          const int k = kb * BK;
          // A: TA -> K-major box {32 k, 128 m}; else MN-major box {128 m, 32 k}
          if (TA) tma_load_2d(dA, &tmA, fb, k, mc);
          else tma_load_2d(dA, &tmA, fb, mc, k);
          // B: !TB -> K-major box {32 k, 128 n}; else MN-major box {128 n, 32 k}
          if (!TB) tma_load_2d(dB, &tmB, fb, k, nc);
          else tma_load_2d(dB, &tmB, fb, nc, k);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    // The tensor-core FP32 accumulator does not round to nearest, so long K
    // sums drift; every CHUNK_KB k-blocks the accumulator goes to the
    // epilogue, which adds the chunks in registers (RN).  Chunks alternate
    // between the two TMEM buffers.
    long g = 0;
    long ch = 0;  // global chunk counter (TMEM buffer = ch % ACC_STAGES)
    for (int local = 0;; ++local) {
      const int c0 = (int)(g % CONV_STAGES);
      mbar_wait(conv_full + 8 * c0, (uint32_t)((g / CONV_STAGES) & 1));
      const int tile = tq[local & 15];
      if (tile < 0) {
        const int as = (int)(ch % ACC_STAGES);
        if (ch >= ACC_STAGES) mbar_wait(acc_empty + 8 * as, (uint32_t)(((ch / ACC_STAGES) & 1) ^ 1));
        if (lane == 0) {  // sentinel to the epilogue (2 arrivals complete the phase)
          mbar_arrive(acc_full + 8 * as);
          mbar_arrive(acc_full + 8 * as);
        }
        break;
      }
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int as = (int)(ch % ACC_STAGES);
        const bool chunk_start = (kb % CHUNK_KB) == 0;
        const bool chunk_end = (kb % CHUNK_KB) == CHUNK_KB - 1 || kb == nk - 1;
        if (chunk_start && ch >= ACC_STAGES)
          mbar_wait(acc_empty + 8 * as, (uint32_t)(((ch / ACC_STAGES) & 1) ^ 1));
        const int c = (int)(g % CONV_STAGES);
        if (kb > 0) mbar_wait(conv_full + 8 * c, (uint32_t)((g / CONV_STAGES) & 1));
        fence_after_sync();
        if (lane == 0) {
          const uint32_t tmem_d = tmem_base + as * BN;
          const uint32_t base = smem_u32(conv + c * CONV_BYTES);
          const uint32_t hiB = base, loB = base + TILE_BYTES;
          const uint32_t hiA = tmem_base + A_COL + c * 2 * BK, loA = hiA + BK;  // TMEM columns
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint32_t off = ks * 32;  // 8 tf32 = 32 bytes along K (B in smem)
            const uint32_t acc0 = (!chunk_start || ks > 0) ? 1u : 0u;
            umma_tf32_ts(tmem_d, loA + ks * 8, kmajor_sw128_desc(hiB + off), acc0);
            umma_tf32_ts(tmem_d, hiA + ks * 8, kmajor_sw128_desc(loB + off), 1u);
            umma_tf32_ts(tmem_d, hiA + ks * 8, kmajor_sw128_desc(hiB + off), 1u);
          }
          umma_commit(conv_empty + 8 * c);
          if (chunk_end) {
            umma_commit(acc_full + 8 * as);
            mbar_arrive(acc_full + 8 * as);  // release: publishes the tile id to the epilogue
          }
        }
        __syncwarp();
        if (chunk_end) ++ch;
      }
    }
  } else if (warp >= CONV_WARP0 && warp < CONV_WARP0 + NCONV) {
    // ================= converters: raw -> hi/lo, K-major SW128 =================
    const int ct = threadIdx.x - CONV_WARP0 * 32;  // 0..255
    long g = 0;
    for (int local = 0;; ++local) {
      {
        const int s0 = (int)(g % RAW_STAGES);
        mbar_wait(raw_full + 8 * s0, (uint32_t)((g / RAW_STAGES) & 1));
      }
      const int tile = tq[local & 15];
      if (tile < 0) {
        // sentinel to the MMA warp: complete the next conversion slot's phase
        const int c = (int)(g % CONV_STAGES);
        if (g >= CONV_STAGES) mbar_wait(conv_empty + 8 * c, (uint32_t)(((g / CONV_STAGES) & 1) ^ 1));
        __syncwarp();
        if (lane == 0) mbar_arrive(conv_full + 8 * c);
        break;
      }
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = (int)(g % RAW_STAGES), c = (int)(g % CONV_STAGES);
        if (kb > 0) mbar_wait(raw_full + 8 * s, (uint32_t)((g / RAW_STAGES) & 1));
        if (g >= CONV_STAGES) mbar_wait(conv_empty + 8 * c, (uint32_t)(((g / CONV_STAGES) & 1) ^ 1));
        const float* rA = (const float*)(raw + s * RAW_BYTES);
        const float* rB = rA + BM * BK;
        float* cb = (float*)(conv + c * CONV_BYTES);
        // ---- A: row m = 32 (warp & 3) + lane, k half kh, straight to TMEM
        //      (tcgen05.st: a warp reaches only its lane quarter) ----
        {
          const int cw = warp - CONV_WARP0, kh = cw >> 2, m = 32 * (warp & 3) + lane;
          float hv[16], lv[16];
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            const int k = kh * 16 + j;
            float4 x;
            if (TA) {  // K-major raw tile, 128B-swizzled by the TMA
              x = *(const float4*)(rA + m * BK + (((k >> 2) ^ (m & 7)) << 2));
            } else {   // MN-major raw tile: consecutive lanes read consecutive rows
              x.x = rA[(k + 0) * BM + m];
              x.y = rA[(k + 1) * BM + m];
              x.z = rA[(k + 2) * BM + m];
              x.w = rA[(k + 3) * BM + m];
            }
            hv[j + 0] = rna_tf32(x.x); lv[j + 0] = x.x - hv[j + 0];
            hv[j + 1] = rna_tf32(x.y); lv[j + 1] = x.y - hv[j + 1];
            hv[j + 2] = rna_tf32(x.z); lv[j + 2] = x.z - hv[j + 2];
            hv[j + 3] = rna_tf32(x.w); lv[j + 3] = x.w - hv[j + 3];
          }
          const uint32_t ta = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + A_COL + c * 2 * BK + kh * 16;
          tmem_st16(ta, hv);
          tmem_st16(ta + BK, lv);
        }
        // ---- B: 128 rows x 8 quads = 1024 quads, 4 per thread, K-major SW128 smem ----
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int idx = it * 256 + ct;
          const bool kmaj = !TB;
          // K-major raw rows are 128 B: 8 consecutive threads read one row
          // (conflict-free float4); MN-major raw: consecutive threads take
          // consecutive rows (conflict-free scalar columns)
          const int r = kmaj ? ((idx >> 3) & 127) : (idx & 127);  // row (n)
          const int qd = kmaj ? (idx & 7) : ((idx >> 7) & 7);       // k quad
          float4 x;
          if (kmaj) {
            x = *(const float4*)(rB + r * BK + qd * 4);
          } else {
            x.x = rB[(qd * 4 + 0) * BM + r];
            x.y = rB[(qd * 4 + 1) * BM + r];
            x.z = rB[(qd * 4 + 2) * BM + r];
            x.w = rB[(qd * 4 + 3) * BM + r];
          }
          float4 h, l;
          h.x = rna_tf32(x.x); l.x = x.x - h.x;
          h.y = rna_tf32(x.y); l.y = x.y - h.y;
          h.z = rna_tf32(x.z); l.z = x.z - h.z;
          h.w = rna_tf32(x.w); l.w = x.w - h.w;
          const int off = r * 32 + ((qd ^ (r & 7)) << 2);  // floats, 128B-swizzled
          float* hi = cb;
          float* lo = hi + BM * BK;
          *(float4*)(hi + off) = h;
          *(float4*)(lo + off) = l;
        }
        fence_before_sync();  // tcgen05.st (A) -> the MMA thread, via the mbarrier
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(conv_full + 8 * c);
          mbar_arrive(raw_empty + 8 * s);
        }
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ================= epilogue =================
    // 16 warps: lane quarter q = warp & 3 (TMEM lanes 32q..32q+31), column
    // slice h = (warp - EPI_WARP0) >> 2 (EPI_COLS columns).  Chunk
    // accumulators are summed with round-to-nearest adds into a running sum
    // kept in TMEM (columns SUM_COL..), 16 columns at a time — no thread
    // holds a whole row slice in registers (the 896-thread block leaves 72
    // registers per thread) — and each accumulator buffer is released as
    // soon as it has been folded in; the tile then goes from the running sum
    // to C.
    const int q = warp & 3, h = (warp - EPI_WARP0) >> 2;
    const int nchunk = (nk + CHUNK_KB - 1) / CHUNK_KB;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t saddr = tmem_base + lane_off + SUM_COL + h * EPI_COLS;
    long ch = 0;
    for (int local = 0;; ++local) {
      int tile = 0;
      for (int cc = 0; cc < nchunk; ++cc, ++ch) {
        const int as = (int)(ch % ACC_STAGES);
        mbar_wait(acc_full + 8 * as, (uint32_t)((ch / ACC_STAGES) & 1));
        if (cc == 0) {
          tile = tq[local & 15];
          if (tile < 0) break;
        }
        fence_after_sync();
        const uint32_t taddr = tmem_base + lane_off + as * BN + h * EPI_COLS;
#pragma unroll
        for (int c0 = 0; c0 < EPI_COLS; c0 += 16) {
          float v[16];
          tmem_ld16(taddr + c0, v);
          if (cc > 0) {
            float sum[16];
            tmem_ld16(saddr + c0, sum);
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = sum[j] + v[j];
          }
          tmem_st16(saddr + c0, v);
        }
        fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + 8 * as);
      }
      if (tile < 0) break;
      const int mc = (tile % p.tm) * BM, nc = (tile / p.tm) * BN + h * EPI_COLS;
      const int m = mc + q * 32 + lane;
#pragma unroll
      for (int c0 = 0; c0 < EPI_COLS; c0 += 16) {
        float v[16];
        tmem_ld16(saddr + c0, v);  // warp-collective: outside the row guard
        if (m < p.M) {
#pragma unroll
          for (int j0 = 0; j0 < 16; j0 += 8) {
            float cv[8];
            if (p.beta != 0.0f) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int n = nc + c0 + j0 + j;
                cv[j] = (n < p.N) ? p.C[m + (long)n * p.ldc] : 0.0f;
              }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int n = nc + c0 + j0 + j;
              if (n < p.N) {
                const float r = p.alpha * v[j0 + j];
                p.C[m + (long)n * p.ldc] = (p.beta == 0.0f) ? r : fmaf(p.beta, cv[j], r);
              }
            }
          }
        }
      }
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(TMEM_COLS)
                 : "memory");
  }
}
}  // namespace tf32

static PFN_cuTensorMapEncodeTiled_v12000 g_enc32 = nullptr;
static std::once_flag g_enc32_once;

static int get_enc32() {
  std::call_once(g_enc32_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_enc32 = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    for (auto f : {tf32::sgemm_tf32x3_kernel<false, false>, tf32::sgemm_tf32x3_kernel<false, true>,
                   tf32::sgemm_tf32x3_kernel<true, false>, tf32::sgemm_tf32x3_kernel<true, true>})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tf32::SMEM);
  });
  return g_enc32 ? UTV_OK : UTV_ERR_CUDA;
}

// Plain (non-swizzled) fp32 map over a column-major rows x cols matrix.
static int make_map32(CUtensorMap* map, const float* p, long rows, long cols, long ld, uint32_t box0,
                      uint32_t box1, bool sw128 = false) {
  if ((ld & 3) || ((uintptr_t)p & 15)) return UTV_ERR_ALIGN;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_enc32(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)p, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE,
                       sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "libutvb200: fp32 tensor map failed (%d) rows=%ld cols=%ld ld=%ld\n", (int)r,
            rows, cols, ld);
    return UTV_ERR_CUDA;
  }
  return UTV_OK;
}

__global__ void sscale_kernel(int M, int N, float beta, float* C, long ldc) {
  const size_t total = (size_t)M * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int m = (int)(i % M), n = (int)(i / M);
    float* c = C + m + (long)n * ldc;
    *c = (beta == 0.0f) ? 0.0f : beta * *c;
  }
}

int sgemm_tf32x3(bool ta, bool tb, int M, int N, int K, float alpha, const float* A, long lda,
                 const float* B, long ldb, float beta, float* C, long ldc, cudaStream_t st) {
  if (M <= 0 || N <= 0) return UTV_OK;
  UTV_CHECK(get_enc32());
  if (K <= 0 || alpha == 0.0f) {
    if (beta == 1.0f) return UTV_OK;
    ProfScope ps(PROF_OPS, 0.0, 8.0 * M * N, st);
    sscale_kernel<<<4 * num_sms(), 256, 0, st>>>(M, N, beta, C, ldc);
    UTV_CUDA(cudaGetLastError());
    return UTV_OK;
  }
  if (((uintptr_t)C & 3) || ldc < M) return UTV_ERR_ALIGN;
  CUtensorMap mA, mB;
  // A (op(A) is M x K): TA -> stored K x M (K contiguous); else M x K (M contiguous)
  if (ta) UTV_CHECK(make_map32(&mA, A, K, M, lda, tf32::BK, tf32::BM, true));  // rows read per lane
  else UTV_CHECK(make_map32(&mA, A, M, K, lda, tf32::BM, tf32::BK));
  // B (op(B) is K x N): !TB -> stored K x N (K contiguous); else N x K (N contiguous)
  if (!tb) UTV_CHECK(make_map32(&mB, B, K, N, ldb, tf32::BK, tf32::BN));
  else UTV_CHECK(make_map32(&mB, B, N, K, ldb, tf32::BN, tf32::BK));
  tf32::Args a;
  a.M = M; a.N = N; a.K = K;
  a.tm = ceil_div(M, tf32::BM);
  a.tn = ceil_div(N, tf32::BN);
  a.tiles = a.tm * a.tn;
  a.alpha = alpha; a.beta = beta;
  a.C = C; a.ldc = ldc;
  a.sched = gemm_sched_slot(st);
  const int grid = a.tiles < num_sms() ? a.tiles : num_sms();
  ProfScope ps(PROF_GEMM_TF32, 2.0 * M * N * K,
               4.0 * ((double)M * K + (double)K * N + (beta != 0.0f ? 2.0 : 1.0) * M * N), st);
  if (!ta && !tb) tf32::sgemm_tf32x3_kernel<false, false><<<grid, tf32::THREADS, tf32::SMEM, st>>>(mA, mB, a);
  else if (!ta && tb) tf32::sgemm_tf32x3_kernel<false, true><<<grid, tf32::THREADS, tf32::SMEM, st>>>(mA, mB, a);
  else if (ta && !tb) tf32::sgemm_tf32x3_kernel<true, false><<<grid, tf32::THREADS, tf32::SMEM, st>>>(mA, mB, a);
  else tf32::sgemm_tf32x3_kernel<true, true><<<grid, tf32::THREADS, tf32::SMEM, st>>>(mA, mB, a);
  UTV_CUDA(cudaGetLastError());
  return UTV_OK;
}

}  // namespace utv
