// Row-parallel dense layers of the policy on the 5th-generation tensor cores:
//   C[M, N] = epilogue([A1 | A2][M, K] @ W[K, N] + bias)
// tcgen05.mma kind::tf32 (M=128, N=BN, K=8) with a 3xTF32 split
//   A W ~= A_hi W_hi + A_hi W_lo + A_lo W_hi,  x_hi = tf32_rn(x), x_lo = tf32_rn(x - x_hi)
// so products carry ~fp32 accuracy (single-pass tf32 measured 4e-4 on logits, outside
// the 1e-4 bar).  Accumulator in TMEM; the epilogue warps own one row
// each and apply bias + relu/sigmoid, or residual + LayerNorm (+ optional per-forward
// row scale for the trunk's modulation), replacing the reference's affine / relu /
// sigmoid / add / layer_norm chains (tensor.py:133-180, 330-351, 378).
//
// Persistent CTA per SM, 9 warps:
//   warp 8 (one thread): TMA of the fp32 A chunk (128 rows x 32 cols, 128-B swizzle,
//           OOB rows/cols zero-filled), cp.async.bulk of the prepacked W_hi/W_lo chunk,
//           and the MMA issue;
//   warps 0-3: split the landed A chunk in shared memory: hi = tf32_rn(x) in place,
//           lo = tf32_rn(x - hi) into the twin buffer (same swizzled layout);
//   warps 4-7: epilogue, one accumulator row per thread.
// NS-stage smem ring + double-buffered TMEM accumulator, all handshakes on mbarriers,
// so TMA, split, MMA and the previous tile's epilogue all overlap.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "engine.cuh"

namespace go {
namespace tg {

constexpr int BM = 128, BK = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// one lane of a converged warp (the MMA issuer)
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}"
               : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void umma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_ss_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// no-swizzle K-major canonical layout (the prepacked B tiles)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// 128-B swizzled K-major layout (TMA-written A tiles): rows of 128 B, 8-row groups
// 1024 B apart; the K step inside the swizzle atom advances the start address.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ float tf32rn(float x) {
  uint32_t y;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(y) : "f"(x));
  return __uint_as_float(y);
}
#define TG_LD16(taddr, r)                                                                    \
  asm volatile(                                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%" \
      "15}, [%16];"                                                                          \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),  \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),           \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                                                \
      : "r"(taddr))
#define TG_ST16(taddr, r)                                                                    \
  asm volatile(                                                                              \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%" \
      "14,%15,%16};" ::"r"(taddr),                                                           \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),      \
      "r"(r[15]))

struct Args {
  int K1, K2;                                // A1 columns (multiple of 32 if A2), A2 columns
  const float* Bpk;                          // [nblk][nch][2][BN*32]
  const float* bias;
  float* C;
  int64_t ldc;
  int64_t M;
  int N;
  int nch;
  const float* resid;                        // LN mode: C = LN(resid + acc + bias)
  int64_t ldr;
  const float* ln_g;
  const float* ln_b;
  const float* rowscale;                     // optional: C2 = C * rowscale[row_fwd[r]]
  const int32_t* row_fwd;
  float* C2;
  int64_t ldc2;
  int vec;                                   // C, C2 rows 16-B aligned: float4 stores
  int32_t* ovf;                              // fp16 path: set if some |A| leaves fp16 range
  const int32_t* gate;                       // tf32 re-run: run only if *gate != 0
};

// fp16 path: W is prepacked as W * 2^W16_SHIFT so W_lo stays a normal fp16; the
// epilogue scales the accumulator back by 2^-W16_SHIFT (exact).
constexpr int W16_SHIFT = 8;
constexpr float A16_LIMIT = 32768.f;  // |A| above this re-runs the GEMM in tf32

// MH = number of 128-row M halves per tile (2: each W chunk in shared memory feeds two
// accumulators, halving the weight bytes pulled from L2 per output row).
// H: fp16 operands (kind::f16, K=16 per MMA).  The A slot then holds the raw fp32 TMA
// chunk, which the split warps overwrite with its fp16 hi (first 8 KB) and lo halves.
// WRCH > 0: the whole packed W (<= WRCH 32-k chunks, one N block) is loaded into shared
// memory once per CTA and stays resident; the ring then carries only A chunks, so more
// A bytes are in flight (these GEMMs are HBM-bound) and W is not re-read from L2 per tile.
template <int BN, int MH, bool H = false, int WRCH = 0>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;  // 16 KB: one fp32 (or tf32 hi / lo) tile
  static constexpr int A_SLOT = H ? A_BYTES : 2 * A_BYTES;
  static constexpr int B_BYTES = BN * BK * (H ? 2 : 4);  // one of W_hi / W_lo
  static constexpr int W_RES = WRCH * 2 * B_BYTES;        // resident W (hi + lo chunks)
  static constexpr int STAGE = MH * A_SLOT + (WRCH ? 0 : 2 * B_BYTES);  // multiple of 1024
  // epilogue staging (4 warps x [32][36]) + bias[256] + ln gamma/beta[128]
  static constexpr int EPI_BYTES = 4 * 32 * 36 * 4 + 512 * 4;
  static constexpr int ALIGN_PAD = 1024;  // the swizzled A tiles need 1024-B alignment
  // 227 KB opt-in limit minus staging, barriers and alignment; >= 2 stages or the refill
  // schedule (stage of chunk g-1 refilled after chunk g is issued) cannot progress
  static constexpr int BUDGET = 232448 - EPI_BYTES - 1536 - ALIGN_PAD - W_RES;
  static constexpr int NSMAX = WRCH ? 12 : H ? 6 : 4;
  static constexpr int NS = (BUDGET / STAGE) < NSMAX ? (BUDGET / STAGE) : NSMAX;
  static_assert(NS >= 2, "tc_gemm needs at least two smem stages");
  static_assert(STAGE % 1024 == 0, "stage must keep 1024-B alignment");
  static constexpr uint32_t TCOLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr uint32_t ACOLS = MH * TCOLS;   // one accumulator set (all halves)
  static constexpr uint32_t TALLOC = 2 * ACOLS;   // double-buffered
  static_assert(TALLOC <= 512, "accumulators exceed TMEM");
  static constexpr size_t SMEM = (size_t)NS * STAGE + W_RES + EPI_BYTES + 1536 + ALIGN_PAD;
};

constexpr int G_THREADS = 320;  // warps 0-3 split A, 4-7 epilogue, 8 MMA issue, 9 loads

template <int ACT>
__device__ __forceinline__ float activate(float x) {
  if (ACT == 1) return x > 0.f ? x : 0.f;
  if (ACT == 2) return __frcp_rn(1.f + __expf(-x));
  return x;
}

// Persistent, warp-specialised tile loop: CTA b processes tiles b, b + grid, ...
// (tile t -> m tile t / nblk, n block t % nblk).  The smem ring and the two TMEM
// accumulators carry their phases across tiles, so the loads and MMAs of tile i+1
// overlap the epilogue of tile i.
template <int BN, int MH, bool LN, int ACT, bool H, int WRCH = 0>
__global__ void __launch_bounds__(G_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA1,
                   const __grid_constant__ CUtensorMap tmA2, Args a, int nblk, int ntiles) {
  static_assert(!H || MH == 1, "fp16 path uses one accumulator per tile");
  using CF = Cfg<BN, MH, H, WRCH>;
  static_assert(WRCH == 0 || (H && MH == 1), "resident W: fp16 path only");
  if (a.gate && *a.gate == 0) return;  // tf32 re-run not needed
  constexpr int TM = BM * MH;  // rows per tile
  constexpr int NS = CF::NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* stage_base =
      smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // 1024-B aligned
  uint8_t* w_res = stage_base + (size_t)NS * CF::STAGE;  // WRCH chunks (hi, lo) if resident
  float* epi = reinterpret_cast<float*>(w_res + CF::W_RES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(w_res + CF::W_RES + CF::EPI_BYTES);
  uint64_t* full = bars;                // [NS] tx bytes: A (TMA) + B (bulk)
  uint64_t* a_full = bars + NS;         // [NS] 128 arrivals: A split into hi/lo
  uint64_t* done = bars + 2 * NS;       // [NS] MMA commit: stage free
  uint64_t* acc_full = bars + 3 * NS;   // [2] MMA commit: accumulator ready
  uint64_t* acc_empty = bars + 3 * NS + 2;  // [2] 128 arrivals: accumulator drained
  uint64_t* w_full = bars + 3 * NS + 4;     // [1] resident W landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * NS + 5);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto A_hi = [&](int s, int h) {
    return reinterpret_cast<float*>(stage_base + (size_t)s * CF::STAGE + (size_t)h * CF::A_SLOT);
  };
  auto A_lo = [&](int s, int h) { return A_hi(s, h) + BM * BK; };  // tf32 path only
  auto B_hi = [&](int s) {
    return reinterpret_cast<uint8_t*>(stage_base + (size_t)s * CF::STAGE + (size_t)MH * CF::A_SLOT);
  };
  auto B_lo = [&](int s) { return B_hi(s) + CF::B_BYTES; };
  const int nch = a.nch;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (warp == 8) {
    if (lane == 0) {
      for (int s = 0; s < NS; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&a_full[s], 128);
        mbar_init(&done[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&acc_full[b], 1);
        mbar_init(&acc_empty[b], 128);
      }
      mbar_init(w_full, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA1)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA2)) : "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(CF::TALLOC));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_slot;

  const int total = my_tiles * nch;
  if (warp == 9) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      auto load = [&](int g) {
        const int s = g % NS;
        const int t = blockIdx.x + (g / nch) * gridDim.x;
        const int c = g % nch;
        const int m0 = (t / nblk) * TM;
        const int k0 = c * BK;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(a.Bpk) +
                             ((size_t)(t % nblk) * nch + c) * 2 * CF::B_BYTES;
        mbar_expect_tx(&full[s], MH * CF::A_BYTES + (WRCH ? 0 : 2 * CF::B_BYTES));
        for (int h = 0; h < MH; ++h) {
          if (k0 < a.K1) tma_2d(A_hi(s, h), &tmA1, k0, m0 + h * BM, &full[s]);
          else tma_2d(A_hi(s, h), &tmA2, k0 - a.K1, m0 + h * BM, &full[s]);
        }
        if constexpr (WRCH == 0) {
          bulk_g2s(B_hi(s), src, CF::B_BYTES, &full[s]);
          bulk_g2s(B_lo(s), src + CF::B_BYTES, CF::B_BYTES, &full[s]);
        }
      };
      if constexpr (WRCH > 0) {  // the whole W (one N block): nch x (hi, lo) chunks
        if (my_tiles > 0) {
          mbar_expect_tx(w_full, nch * 2 * CF::B_BYTES);
          for (int c = 0; c < nch; ++c)
            bulk_g2s(w_res + (size_t)c * 2 * CF::B_BYTES,
                     reinterpret_cast<const uint8_t*>(a.Bpk) + (size_t)c * 2 * CF::B_BYTES,
                     2 * CF::B_BYTES, w_full);
        }
      }
      for (int g = 0; g < total; ++g) {
        if (g >= NS) mbar_wait(&done[g % NS], ((g / NS) - 1) & 1);  // stage consumed
        load(g);
      }
    }
    __syncwarp();
  } else if (warp == 8) {
    // ------------------------------------------------ MMA issue (converged, one elected lane)
    constexpr uint32_t ID = H ? idesc_f16(BM, BN) : idesc_tf32(BM, BN);
    if constexpr (WRCH > 0) {
      if (my_tiles > 0) mbar_wait(w_full, 0);
    }
    int g = 0;
    for (int tl = 0; tl < my_tiles; ++tl) {
      const int ab = tl & 1;
      if (tl >= 2) mbar_wait(&acc_empty[ab], ((tl >> 1) - 1) & 1);
      fence_after();
      const uint32_t tacc = tbase + ab * CF::ACOLS;
      for (int c = 0; c < nch; ++c, ++g) {
        const int s = g % NS;
        const uint32_t ph = (g / NS) & 1;
        mbar_wait(&full[s], ph);
        mbar_wait(&a_full[s], ph);
        fence_after();
        if (elect_one()) {
          const uint32_t bh =
              WRCH ? smem_u32(w_res + (size_t)c * 2 * CF::B_BYTES) : smem_u32(B_hi(s));
          const uint32_t bl = bh + CF::B_BYTES;
          if constexpr (H) {
            // fp16 hi at +0, lo at +8 KB; 8-half K chunks 2 KB apart (A) / BN*16 B (B)
            const uint64_t da = sdesc(smem_u32(A_hi(s, 0)), 2048, 128);
            const uint64_t dbh0 = sdesc(bh, BN * 16, 128), dbl0 = sdesc(bl, BN * 16, 128);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              // K steps add (bytes >> 4) to the descriptors' start-address field
              const uint64_t dah = da + kk * 256, dal = da + 512 + kk * 256;
              const uint64_t dbh = dbh0 + kk * 2 * BN, dbl = dbl0 + kk * 2 * BN;
              umma_ss_f16(tacc, dah, dbh, ID, (c > 0 || kk > 0));
              umma_ss_f16(tacc, dah, dbl, ID, 1);
              umma_ss_f16(tacc, dal, dbh, ID, 1);
            }
          } else {
#pragma unroll
            for (int k = 0; k < BK / 8; ++k) {
              const uint64_t dbh = sdesc(bh + k * 32 * BN, 16 * BN, 128);
              const uint64_t dbl = sdesc(bl + k * 32 * BN, 16 * BN, 128);
#pragma unroll
              for (int h = 0; h < MH; ++h) {
                const uint64_t dah = sdesc_sw128(smem_u32(A_hi(s, h)) + k * 32);
                const uint64_t dal = sdesc_sw128(smem_u32(A_lo(s, h)) + k * 32);
                const uint32_t th = tacc + h * CF::TCOLS;
                umma_ss(th, dah, dbh, ID, (c > 0 || k > 0));
                umma_ss(th, dah, dbl, ID, 1);
                umma_ss(th, dal, dbh, ID, 1);
              }
            }
          }
          umma_commit(&done[s]);
          if (c == nch - 1) umma_commit(&acc_full[ab]);
        }
        __syncwarp();
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------ A split: hi in place, lo in the twin
    // (elementwise, so the lo tile inherits the TMA's swizzled layout)
    const int lt = threadIdx.x;  // 0..127
    for (int g = 0; g < total; ++g) {
      const int s = g % NS;
      mbar_wait(&full[s], (g / NS) & 1);
      if constexpr (H) {
        // thread = one A row: read its 128-B swizzled fp32 row, then (after all rows are
        // in registers) write fp16 hi / lo in the no-swizzle K-major canonical layout
        const float4* rp = reinterpret_cast<const float4*>(A_hi(s, 0)) + lt * 8;
        float4 x[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = rp[c ^ (lt & 7)];
        bool big = false;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          big |= !(fabsf(x[c].x) <= A16_LIMIT) || !(fabsf(x[c].y) <= A16_LIMIT) ||
                 !(fabsf(x[c].z) <= A16_LIMIT) || !(fabsf(x[c].w) <= A16_LIMIT);
        if (big) atomicOr(a.ovf, 1);
        asm volatile("bar.sync 2, 128;" ::: "memory");  // raw reads done before overwrite
        __half* a16 = reinterpret_cast<__half*>(A_hi(s, 0));
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          const float v[8] = {x[2 * kc].x,     x[2 * kc].y,     x[2 * kc].z,     x[2 * kc].w,
                              x[2 * kc + 1].x, x[2 * kc + 1].y, x[2 * kc + 1].z, x[2 * kc + 1].w};
          __align__(16) __half hi[8], lo[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            hi[e] = __float2half_rn(v[e]);
            lo[e] = __float2half_rn(v[e] - __half2float(hi[e]));
          }
          const int off = kc * (BM * 8) + lt * 8;  // (r>>3)*64 + (r&7)*8 == r*8
          *reinterpret_cast<uint4*>(a16 + off) = *reinterpret_cast<const uint4*>(hi);
          *reinterpret_cast<uint4*>(a16 + 4096 + off) = *reinterpret_cast<const uint4*>(lo);
        }
      } else {
#pragma unroll
        for (int hh = 0; hh < MH; ++hh) {
          float4* hp = reinterpret_cast<float4*>(A_hi(s, hh));
          float4* lp = reinterpret_cast<float4*>(A_lo(s, hh));
          float4 x[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = hp[i * 128 + lt];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 h = make_float4(tf32rn(x[i].x), tf32rn(x[i].y), tf32rn(x[i].z), tf32rn(x[i].w));
            const float4 l = make_float4(tf32rn(x[i].x - h.x), tf32rn(x[i].y - h.y),
                                         tf32rn(x[i].z - h.z), tf32rn(x[i].w - h.w));
            hp[i * 128 + lt] = h;
            lp[i * 128 + lt] = l;
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&a_full[s]);
    }
  } else {
    // ------------------------------------------------ epilogue: thread = accumulator row
    // Each thread holds one accumulator row (tcgen05.ld 32x32b); 32x32 blocks are
    // transposed through a padded smem tile (row stride 36 floats: conflict-free
    // STS.128 / LDS.128) so every global load/store is a float4 and each warp
    // instruction touches 4 full 128-B lines.
    constexpr float ASCALE = H ? 1.f / (1 << W16_SHIFT) : 1.f;  // undo the W prescale
    const int ew = warp - 4;                 // TMEM lane quarter
    const int et = threadIdx.x - 128;        // 0..127
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    float* stg = epi + ew * 32 * 36;
    float* s_bias = epi + 4 * 32 * 36;       // [256]
    float* s_g = s_bias + 256;               // [128]
    float* s_b = s_g + 128;                  // [128]
    const int rq = lane >> 3, c4 = lane & 7;
    auto epi_bar = [] { asm volatile("bar.sync 1, 128;" ::: "memory"); };
    auto ld4 = [](const float* p) { return *reinterpret_cast<const float4*>(p); };
    for (int tl = 0; tl < my_tiles; ++tl) {
      const int t = blockIdx.x + tl * gridDim.x;
      const int64_t m0 = (int64_t)(t / nblk) * TM;
      const int n0 = (t % nblk) * BN;
      const int ab = tl & 1;
      epi_bar();  // previous tile's parameter reads are done
      for (int i = et; i < BN; i += 128) {
        s_bias[i] = (a.bias && n0 + i < a.N) ? a.bias[n0 + i] : 0.f;
        if (LN) {
          s_g[i] = a.ln_g[i];
          s_b[i] = a.ln_b[i];
        }
      }
      epi_bar();
      mbar_wait(&acc_full[ab], (tl >> 1) & 1);
      fence_after();
#pragma unroll 1
      for (int mh = 0; mh < MH; ++mh) {
      const int64_t rbase = m0 + mh * BM + ew * 32;
      const uint32_t tacc = tbase + ab * CF::ACOLS + mh * CF::TCOLS + lane_off;
      const int64_t row = rbase + lane;
      const bool rv = row < a.M;
      // y[32] of this thread's row (columns c0..c0+31 of the block) -> C, coalesced
      auto store32 = [&](float* C, int64_t ldc, int c0, const float* y) {
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(stg + lane * 36 + 4 * q) =
              make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i * 4 + rq;
          const int cl = c0 + c4 * 4;  // column within the block
          const int64_t gr = rbase + r;
          const int n = n0 + cl;
          if (gr < a.M && cl < BN && n < a.N) {
            const float4 v = ld4(stg + r * 36 + c4 * 4);
            float* dst = C + gr * ldc + n;
            if (a.vec && n + 4 <= a.N) {
              *reinterpret_cast<float4*>(dst) = v;
            } else {
              const float vv[4] = {v.x, v.y, v.z, v.w};
              for (int e = 0; e < 4 && n + e < a.N; ++e) dst[e] = vv[e];
            }
          }
        }
      };
      if (LN) {
        // pass 1: x = acc + bias + resid, kept in TMEM; running sum
        float s = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t u[32];
          TG_LD16(tacc + c0, u);
          TG_LD16(tacc + c0 + 16, (u + 16));
          float rr[32];
          if (a.resid) {
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int r = i * 4 + rq;
              const int64_t gr = rbase + r;
              const float4 v = gr < a.M ? __ldg(reinterpret_cast<const float4*>(
                                              a.resid + gr * a.ldr + c0 + c4 * 4))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
              *reinterpret_cast<float4*>(stg + r * 36 + c4 * 4) = v;
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 v = ld4(stg + lane * 36 + 4 * q);
              rr[4 * q] = v.x; rr[4 * q + 1] = v.y; rr[4 * q + 2] = v.z; rr[4 * q + 3] = v.w;
            }
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 b4 = ld4(s_bias + c0 + 4 * q);
            const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = 4 * q + e;
              float x = __uint_as_float(u[j]) * ASCALE + bb[e];
              if (a.resid) x += rr[j];
              s += x;
              u[j] = __float_as_uint(x);
            }
          }
          TG_ST16(tacc + c0, u);
          TG_ST16(tacc + c0 + 16, (u + 16));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        const float mu = s / BN;
        float q = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t u[32];
          TG_LD16(tacc + c0, u);
          TG_LD16(tacc + c0 + 16, (u + 16));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float d = __uint_as_float(u[j]) - mu;
            q += d * d;
          }
        }
        const float inv = 1.f / sqrtf(q / BN + 1e-5f);
        const float* rs = (a.rowscale && rv) ? a.rowscale + (int64_t)a.row_fwd[row] * BN : nullptr;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t u[32];
          TG_LD16(tacc + c0, u);
          TG_LD16(tacc + c0 + 16, (u + 16));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float y[32];
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const float4 g4 = ld4(s_g + c0 + 4 * q4), b4 = ld4(s_b + c0 + 4 * q4);
            const float gg[4] = {g4.x, g4.y, g4.z, g4.w}, bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = 4 * q4 + e;
              y[j] = gg[e] * ((__uint_as_float(u[j]) - mu) * inv) + bb[e];
            }
          }
          if (a.C) store32(a.C, a.ldc, c0, y);
          if (a.rowscale) {
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4) {
              const float4 r4 = rs ? __ldg(reinterpret_cast<const float4*>(rs + c0) + q4)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
              y[4 * q4] *= r4.x; y[4 * q4 + 1] *= r4.y; y[4 * q4 + 2] *= r4.z; y[4 * q4 + 3] *= r4.w;
            }
            store32(a.C2, a.ldc2, c0, y);
          }
        }
      } else {
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t u[32];
          TG_LD16(tacc + c0, u);
          if (c0 + 16 < BN) TG_LD16(tacc + c0 + 16, (u + 16));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float y[32];
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const float4 b4 = ld4(s_bias + c0 + 4 * q4);  // s_bias has 256 entries: in range
            const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = 4 * q4 + e;
              y[j] = activate<ACT>(__uint_as_float(u[j]) * ASCALE + bb[e]);
            }
          }
          if (a.C) store32(a.C, a.ldc, c0, y);
          if (a.rowscale) {  // C2 = C * rowscale[forward of the row] (trunk modulation)
            const float* rs = rv ? a.rowscale + (int64_t)a.row_fwd[row] * a.N + n0 + c0 : nullptr;
#pragma unroll
            for (int j = 0; j < 32; ++j) y[j] *= (rs && n0 + c0 + j < a.N) ? __ldg(rs + j) : 0.f;
            store32(a.C2, a.ldc2, c0, y);
          }
        }
      }
      }  // M halves
      fence_before();
      mbar_arrive(&acc_empty[ab]);
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 8) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                 "r"(CF::TALLOC));
  }
}

#include "tc_ffn.cuh"

// Pack W[K, N] (row-major, ldw) into [nblk][nch][hi|lo][BN*32] UMMA K-major canonical
// B tiles: element (n, k) of a block at (k/4)*(BN/8*32) + (n/8)*32 + (n%8)*4 + k%4.
// Up to three column blocks (W0 | W1 | W2) concatenate into one weight (merged QKV).
__global__ void pack_b_kernel(const float* __restrict__ W0, const float* __restrict__ W1,
                              const float* __restrict__ W2, int Nsub, int64_t ldw, int K, int N,
                              int BN, int nch, int nblk, float* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)nblk * nch * BN * BK;
  if (i >= total) return;
  int64_t per_blk = (int64_t)nch * BN * BK;
  int b = (int)(i / per_blk);
  int64_t rem = i % per_blk;
  int c = (int)(rem / (BN * BK));
  int e = (int)(rem % (BN * BK));
  int n_l = e / BK, k_l = e % BK;
  int n = b * BN + n_l, k = c * BK + k_l;
  float w = 0.f;
  if (n < N && k < K) {
    const int part = n / Nsub, nn = n % Nsub;
    const float* W = part == 0 ? W0 : (part == 1 ? W1 : W2);
    w = W[(int64_t)k * ldw + nn];
  }
  float h = tf32rn(w), l = tf32rn(w - h);
  int off = (k_l >> 2) * (BN / 8 * 32) + (n_l >> 3) * 32 + (n_l & 7) * 4 + (k_l & 3);
  float* dst = out + ((int64_t)b * nch + c) * 2 * BN * BK;
  dst[off] = h;
  dst[BN * BK + off] = l;
}

// fp16 twin of pack_b_kernel: W * 2^W16_SHIFT split into fp16 hi / lo, element (n, k)
// of a block at (k/8)*(BN*8) + (n/8)*64 + (n%8)*8 + k%8 (no-swizzle K-major, 8 halfs/16 B).
__global__ void pack_b16_kernel(const float* __restrict__ W0, const float* __restrict__ W1,
                                const float* __restrict__ W2, int Nsub, int64_t ldw, int K,
                                int N, int BN, int nch, int nblk, __half* __restrict__ out,
                                int32_t* __restrict__ ovf) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)nblk * nch * BN * BK;
  if (i >= total) return;
  int64_t per_blk = (int64_t)nch * BN * BK;
  int b = (int)(i / per_blk);
  int64_t rem = i % per_blk;
  int c = (int)(rem / (BN * BK));
  int e = (int)(rem % (BN * BK));
  int n_l = e / BK, k_l = e % BK;
  int n = b * BN + n_l, k = c * BK + k_l;
  float w = 0.f;
  if (n < N && k < K) {
    const int part = n / Nsub, nn = n % Nsub;
    const float* W = part == 0 ? W0 : (part == 1 ? W1 : W2);
    w = W[(int64_t)k * ldw + nn] * (float)(1 << W16_SHIFT);
    // a weight beyond the fp16 range routes this GEMM to its tf32 re-run
    if (ovf && !(fabsf(w) <= 65504.f)) atomicOr(ovf, 1);
  }
  const __half h = __float2half_rn(w);
  const __half l = __float2half_rn(w - __half2float(h));
  int off = (k_l >> 3) * (BN * 8) + (n_l >> 3) * 64 + (n_l & 7) * 8 + (k_l & 7);
  __half* dst = out + ((int64_t)b * nch + c) * 2 * BN * BK;
  dst[off] = h;
  dst[BN * BK + off] = l;
}

}  // namespace tg

int tc_gemm_bn(int N) {
  if (N <= 16) return 16;
  if (N <= 32) return 32;
  if (N <= 48) return 48;
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  if (N <= 144) return 144;
  return 256;
}

size_t tc_gemm_packed_floats(int K, int N) {
  int BN = tc_gemm_bn(N);
  int nblk = (int)cdiv(N, BN);
  int nch = (int)cdiv(K, tg::BK);
  return (size_t)nblk * nch * 2 * BN * tg::BK;
}

// fp16 twin (W scaled by 2^W16_SHIFT): same element count, 2 bytes each.
void tc_gemm_pack16(const float* W0, const float* W1, const float* W2, int Nsub, int64_t ldw,
                    int K, int N, void* out, cudaStream_t st, int32_t* ovf) {
  int BN = tc_gemm_bn(N);
  int nblk = (int)cdiv(N, BN);
  int nch = (int)cdiv(K, tg::BK);
  int64_t total = (int64_t)nblk * nch * BN * tg::BK;
  tg::pack_b16_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(
      W0, W1 ? W1 : W0, W2 ? W2 : W0, Nsub, ldw, K, N, BN, nch, nblk, static_cast<__half*>(out),
      ovf);
  LAUNCH_CHECK();
}

// fp16 pack with an explicit block width (the fused FFN wants 128-column blocks).
void tc_gemm_pack16_bn(const float* W, int64_t ldw, int K, int N, int BN, void* out,
                       cudaStream_t st, int32_t* ovf) {
  int nblk = (int)cdiv(N, BN);
  int nch = (int)cdiv(K, tg::BK);
  int64_t total = (int64_t)nblk * nch * BN * tg::BK;
  tg::pack_b16_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(
      W, W, W, N, ldw, K, N, BN, nch, nblk, static_cast<__half*>(out), ovf);
  LAUNCH_CHECK();
}

// Pack W = [W0 | W1 | W2] (each [K, Nsub] row-major with ldw; N = parts * Nsub).
void tc_gemm_pack(const float* W0, const float* W1, const float* W2, int Nsub, int64_t ldw, int K,
                  int N, float* out, cudaStream_t st) {
  int BN = tc_gemm_bn(N);
  int nblk = (int)cdiv(N, BN);
  int nch = (int)cdiv(K, tg::BK);
  int64_t total = (int64_t)nblk * nch * BN * tg::BK;
  tg::pack_b_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(W0, W1 ? W1 : W0, W2 ? W2 : W0,
                                                                Nsub, ldw, K, N, BN, nch, nblk,
                                                                out);
  LAUNCH_CHECK();
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p)
      GO_THROW(GO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D fp32 map over A[rows, cols] (row stride ld floats): boxes of 128 rows x 32 cols,
// 128-B swizzle, out-of-range rows/cols read as zero.
CUtensorMap a_map(const float* A, int64_t rows, int cols, int64_t ld) {
  GO_CHECK((uintptr_t)A % 16 == 0 && ld % 4 == 0, "A rows must be 16-B aligned");
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)tg::BK, (cuuint32_t)tg::BM};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(A), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) GO_THROW(GO_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return m;
}

template <int BN, int MH, bool LN, int ACT, bool H, int WRCH = 0>
void launch(const CUtensorMap& m1, const CUtensorMap& m2, const tg::Args& a, int nblk,
            cudaStream_t st) {
  using CF = tg::Cfg<BN, MH, H, WRCH>;
  static bool attr = false;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(tg::tc_gemm_kernel<BN, MH, LN, ACT, H, WRCH>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM));
    attr = true;
  }
  const int ntiles = (int)cdiv(a.M, tg::BM * MH) * nblk;
  const int grid = std::min(ntiles, num_sms());
  tg::tc_gemm_kernel<BN, MH, LN, ACT, H, WRCH><<<grid, tg::G_THREADS, CF::SMEM, st>>>(
      m1, m2, a, nblk, ntiles);
  LAUNCH_CHECK();
}

// GO_GEMM_F16=0 keeps the tf32 operands
static bool use_f16() {
  const char* e = getenv("GO_GEMM_F16");
  return !(e && e[0] == '0');
}

// fp16-operand GEMM, then the tf32 GEMM gated on the fp16 pass's range flag (a no-op
// launch unless some |A| left the fp16 range); or the tf32 GEMM alone.
template <int BN, bool LN, int ACT>
void launch_all(const float* A1, int64_t lda1, const float* A2, int64_t lda2, tg::Args a,
                const TcW& W, int nblk, cudaStream_t st) {
  GO_CHECK(a.M < ((int64_t)1 << 31), "too many rows for one GEMM launch");
  const CUtensorMap m1 = a_map(A1, a.M, a.K1, lda1);
  const CUtensorMap m2 = A2 ? a_map(A2, a.M, a.K2, lda2) : m1;
  if (W.gate) {  // tf32 re-run of a fused kernel's layer, gated on its range flag
    a.gate = W.gate;
    a.Bpk = W.w32;
    launch<BN, 1, LN, ACT, false>(m1, m2, a, nblk, st);
    return;
  }
  const bool f16 = W.w16 && W.ovf && use_f16();
  if (f16) {
    tg::Args a16 = a;
    a16.Bpk = static_cast<const float*>(W.w16);
    a16.ovf = W.ovf;
    a16.gate = nullptr;
    // resident W when the whole packed W is one N block of <= 4 chunks (K <= 128): the
    // ring keeps >= 8 A stages (larger K would leave fewer A bytes in flight)
    if (nblk == 1 && a.nch <= 4 && tg::Cfg<BN, 1, true, 4>::NS >= 6)
      launch<BN, 1, LN, ACT, true, 4>(m1, m2, a16, nblk, st);
    else
      launch<BN, 1, LN, ACT, true>(m1, m2, a16, nblk, st);
    a.gate = W.ovf;
  }
  a.Bpk = W.w32;
  launch<BN, 1, LN, ACT, false>(m1, m2, a, nblk, st);
}

template <int BN>
void launch_act(int act, const float* A1, int64_t lda1, const float* A2, int64_t lda2,
                const tg::Args& a, const TcW& W, int nblk, cudaStream_t st) {
  switch (act) {
    case 1: launch_all<BN, false, 1>(A1, lda1, A2, lda2, a, W, nblk, st); break;
    case 2: launch_all<BN, false, 2>(A1, lda1, A2, lda2, a, W, nblk, st); break;
    default: launch_all<BN, false, 0>(A1, lda1, A2, lda2, a, W, nblk, st); break;
  }
}

}  // namespace

// C = act([A1|A2] @ W + bias) with W prepacked by tc_gemm_pack(K1+K2, N).
void tc_gemm(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
             const TcW& Wpk, const float* bias, float* C, int64_t ldc, int64_t M, int N,
             int act, cudaStream_t st) {
  if (M <= 0) return;
  GO_CHECK(A2 == nullptr || K1 % tg::BK == 0, "concat split must be a multiple of 32");
  tg::Args a{};
  a.K1 = K1; a.K2 = A2 ? K2 : 0;
  a.bias = bias; a.C = C; a.ldc = ldc; a.M = M; a.N = N;
  a.nch = (int)cdiv(K1 + a.K2, tg::BK);
  a.vec = ((uintptr_t)C % 16 == 0) && ldc % 4 == 0;
  int BN = tc_gemm_bn(N);
  int nblk = (int)cdiv(N, BN);
  switch (BN) {
    case 16: launch_act<16>(act, A1, lda1, A2, lda2, a, Wpk, nblk, st); break;
    case 32: launch_act<32>(act, A1, lda1, A2, lda2, a, Wpk, nblk, st); break;
    case 48: launch_act<48>(act, A1, lda1, A2, lda2, a, Wpk, nblk, st); break;
    case 64: launch_act<64>(act, A1, lda1, A2, lda2, a, Wpk, nblk, st); break;
    case 128: launch_act<128>(act, A1, lda1, A2, lda2, a, Wpk, nblk, st); break;
    case 144: launch_act<144>(act, A1, lda1, A2, lda2, a, Wpk, nblk, st); break;
    default: launch_act<256>(act, A1, lda1, A2, lda2, a, Wpk, nblk, st); break;
  }
}

// C2 = act([A1|A2] @ W + bias) * rowscale[row_fwd[r]] (per-forward row vector of N),
// optionally also C unscaled (C may be null).
void tc_gemm_scaled(const float* A1, int64_t lda1, int K1, const TcW& Wpk, const float* bias,
                    float* C, int64_t ldc, const float* rowscale, const int32_t* row_fwd,
                    float* C2, int64_t ldc2, int64_t M, int N, int act, cudaStream_t st) {
  if (M <= 0) return;
  GO_CHECK(rowscale && row_fwd && C2, "tc_gemm_scaled needs rowscale, row_fwd and C2");
  tg::Args a{};
  a.K1 = K1; a.K2 = 0;
  a.bias = bias; a.C = C; a.ldc = ldc; a.M = M; a.N = N;
  a.nch = (int)cdiv(K1, tg::BK);
  a.rowscale = rowscale; a.row_fwd = row_fwd; a.C2 = C2; a.ldc2 = ldc2;
  a.vec = (C == nullptr || ((uintptr_t)C % 16 == 0 && ldc % 4 == 0)) &&
          ((uintptr_t)C2 % 16 == 0 && ldc2 % 4 == 0);
  int BN = tc_gemm_bn(N);
  int nblk = (int)cdiv(N, BN);
  switch (BN) {
    case 16: launch_act<16>(act, A1, lda1, nullptr, 0, a, Wpk, nblk, st); break;
    case 32: launch_act<32>(act, A1, lda1, nullptr, 0, a, Wpk, nblk, st); break;
    case 48: launch_act<48>(act, A1, lda1, nullptr, 0, a, Wpk, nblk, st); break;
    case 64: launch_act<64>(act, A1, lda1, nullptr, 0, a, Wpk, nblk, st); break;
    case 128: launch_act<128>(act, A1, lda1, nullptr, 0, a, Wpk, nblk, st); break;
    case 144: launch_act<144>(act, A1, lda1, nullptr, 0, a, Wpk, nblk, st); break;
    default: launch_act<256>(act, A1, lda1, nullptr, 0, a, Wpk, nblk, st); break;
  }
}

// Fused trunk feed-forward block (tc_ffn.cuh).  W1_16: [128, 512] packed by
// tc_gemm_pack16_bn(.., BN = 128); W2_16: [512, 128] packed by tc_gemm_pack16.
void tc_ffn(const float* X, int64_t ldx, const void* W1_16, const void* W2_16, const float* b1,
            const float* b2, const float* g, const float* beta, float* C, int64_t ldc,
            const float* rowscale, const int32_t* row_fwd, float* C2, int64_t ldc2, int64_t M,
            int32_t* ovf, cudaStream_t st, bool layernorm) {
  if (M <= 0) return;
  GO_CHECK(ovf, "tc_ffn needs a range flag");
  GO_CHECK(layernorm || (C && !rowscale), "tc_ffn without LayerNorm writes C only");
  GO_CHECK((C == nullptr || ((uintptr_t)C % 16 == 0 && ldc % 4 == 0)) &&
               (C2 == nullptr || ((uintptr_t)C2 % 16 == 0 && ldc2 % 4 == 0)) && ldx % 4 == 0 &&
               (uintptr_t)X % 16 == 0,
           "tc_ffn rows must be 16-B aligned");
  GO_CHECK(rowscale == nullptr || (row_fwd && C2), "tc_ffn rowscale needs row_fwd and C2");
  static bool attr = false;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(tg::ffn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)tg::FF_SMEM));
    attr = true;
  }
  tg::FfnArgs a{};
  a.X = X; a.ldx = ldx;
  a.W1 = static_cast<const uint8_t*>(W1_16);
  a.W2 = static_cast<const uint8_t*>(W2_16);
  a.b1 = b1; a.b2 = b2; a.ln_g = g; a.ln_b = beta;
  a.C = C; a.ldc = ldc; a.rowscale = rowscale; a.row_fwd = row_fwd; a.C2 = C2; a.ldc2 = ldc2;
  a.M = M; a.ovf = ovf; a.ln = layernorm ? 1 : 0;
  const CUtensorMap mx = a_map(X, M, 128, ldx);
  const int ntiles = (int)cdiv(M, tg::BM);
  const int grid = std::min(ntiles, num_sms());
  tg::ffn_kernel<<<grid, tg::FF_THREADS, tg::FF_SMEM, st>>>(mx, a, ntiles);
  LAUNCH_CHECK();
}

// C = LN(resid + [A1|A2] @ W + bias) * g + b  (N == 128); optional C2 = C * rowscale[f].
void tc_gemm_ln(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
                const TcW& Wpk, const float* bias, const float* resid, int64_t ldr,
                const float* g, const float* beta, float* C, int64_t ldc, const float* rowscale,
                const int32_t* row_fwd, float* C2, int64_t ldc2, int64_t M, int N,
                cudaStream_t st) {
  if (M <= 0) return;
  GO_CHECK(N == 128, "fused LayerNorm epilogue needs N == 128");
  GO_CHECK(A2 == nullptr || K1 % tg::BK == 0, "concat split must be a multiple of 32");
  tg::Args a{};
  a.K1 = K1; a.K2 = A2 ? K2 : 0;
  a.bias = bias; a.C = C; a.ldc = ldc; a.M = M; a.N = N;
  a.nch = (int)cdiv(K1 + a.K2, tg::BK);
  a.resid = resid; a.ldr = ldr; a.ln_g = g; a.ln_b = beta;
  a.rowscale = rowscale; a.row_fwd = row_fwd; a.C2 = C2; a.ldc2 = ldc2;
  GO_CHECK(resid == nullptr || ((uintptr_t)resid % 16 == 0 && ldr % 4 == 0),
           "LayerNorm residual rows must be 16-B aligned");
  a.vec = (C == nullptr || ((uintptr_t)C % 16 == 0 && ldc % 4 == 0)) &&
          (C2 == nullptr || ((uintptr_t)C2 % 16 == 0 && ldc2 % 4 == 0));
  launch_all<128, true, 0>(A1, lda1, A2, lda2, a, Wpk, 1, st);
}

}  // namespace go
