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
// CTA: 128 rows x BN columns, 5 warps.  Warps 0-3 load the A tile (fp32 rows,
// float4), split it into hi/lo and store both in the UMMA K-major canonical layout;
// they are also the epilogue.  Warp 4 (one thread) streams the prepacked W_hi/W_lo
// chunks with cp.async.bulk and issues the MMAs.  Multi-stage smem ring, mbarriers.
#include <algorithm>
#include <cstring>

#include "engine.cuh"

namespace go {
namespace tg {

constexpr int BM = 128, BK = 32;
constexpr int THREADS = 160;

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
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
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

struct Args {
  const float* A1;
  int64_t lda1;
  int K1;
  const float* A2;
  int64_t lda2;
  int K2;
  const float* Bpk;  // [nblk][nch][2][BN*32]
  const float* bias;
  float* C;
  int64_t ldc;
  int64_t M;
  int N;
  int nch;
  int act;                                   // 0 none, 1 relu, 2 sigmoid
  const float* resid;                        // LN mode: C = LN(resid + acc + bias)
  int64_t ldr;
  const float* ln_g;
  const float* ln_b;
  const float* rowscale;                     // optional: C2 = C * rowscale[row_fwd[r]]
  const int32_t* row_fwd;
  float* C2;
  int64_t ldc2;
};

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;  // 16 KB per hi/lo tile
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int EPI_BYTES = 4 * 32 * 33 * 4;  // epilogue staging, 4 warps
  // 227 KB opt-in limit minus staging and barriers; >= 2 stages or the B refill schedule
  // (stage of chunk g-1 refilled after chunk g is issued) cannot make progress
  static constexpr int BUDGET = 232448 - EPI_BYTES - 1536;
  static constexpr int NS = (BUDGET / STAGE) < 4 ? (BUDGET / STAGE) : 4;
  static_assert(NS >= 2, "tc_gemm needs at least two smem stages");
  static constexpr uint32_t TCOLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr uint32_t TALLOC = 2 * TCOLS;  // double-buffered accumulator
  static constexpr size_t SMEM = (size_t)NS * STAGE + EPI_BYTES + 1536;
};

constexpr int G_THREADS = 288;  // warps 0-3 load A, 4-7 epilogue, 8 = B producer + MMA issuer

#define TG_ST16(taddr, r)                                                                    \
  asm volatile(                                                                              \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%" \
      "14,%15,%16};" ::"r"(taddr),                                                           \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),      \
      "r"(r[15]))

// Persistent, warp-specialised tile loop: CTA b processes tiles b, b + grid, ...
// (tile t -> m tile t / nblk, n block t % nblk).  The smem ring and the two TMEM
// accumulators carry their phases across tiles, so the loads and MMAs of tile i+1
// overlap the epilogue of tile i.
template <int BN, bool LN>
__global__ void __launch_bounds__(G_THREADS, 1) tc_gemm_kernel(Args a, int nblk, int ntiles) {
  using CF = Cfg<BN>;
  constexpr int NS = CF::NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* stage_base = smem_raw;
  float* epi = reinterpret_cast<float*>(smem_raw + (size_t)NS * CF::STAGE);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (size_t)NS * CF::STAGE + CF::EPI_BYTES);
  uint64_t* a_full = bars;              // [NS] 128 arrivals
  uint64_t* b_full = bars + NS;         // [NS] tx bytes
  uint64_t* done = bars + 2 * NS;       // [NS] MMA commit: stage free
  uint64_t* acc_full = bars + 3 * NS;   // [2] MMA commit: accumulator ready
  uint64_t* acc_empty = bars + 3 * NS + 2;  // [2] 128 arrivals: accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * NS + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto A_hi = [&](int s) { return reinterpret_cast<float*>(stage_base + (size_t)s * CF::STAGE); };
  auto A_lo = [&](int s) { return A_hi(s) + BM * BK; };
  auto B_hi = [&](int s) { return A_hi(s) + 2 * BM * BK; };
  auto B_lo = [&](int s) { return B_hi(s) + BN * BK; };
  const int nch = a.nch;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (warp == 8) {
    if (lane == 0) {
      for (int s = 0; s < NS; ++s) {
        mbar_init(&a_full[s], 128);
        mbar_init(&b_full[s], 1);
        mbar_init(&done[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&acc_full[b], 1);
        mbar_init(&acc_empty[b], 128);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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

  if (warp == 8) {
    // ------------------------------------------------ B producer + MMA issuer
    if (lane == 0) {
      constexpr uint32_t ID = idesc_tf32(BM, BN);
      const int total = my_tiles * nch;
      auto load_b = [&](int g) {
        const int s = g % NS;
        const int t = blockIdx.x + (g / nch) * gridDim.x;
        const int c = g % nch;
        const float* src = a.Bpk + ((size_t)(t % nblk) * nch + c) * 2 * BN * BK;
        mbar_expect_tx(&b_full[s], 2 * CF::B_BYTES);
        bulk_g2s(B_hi(s), src, CF::B_BYTES, &b_full[s]);
        bulk_g2s(B_lo(s), src + BN * BK, CF::B_BYTES, &b_full[s]);
      };
      for (int g = 0; g < NS && g < total; ++g) load_b(g);
      int g = 0;
      for (int tl = 0; tl < my_tiles; ++tl) {
        const int ab = tl & 1;
        if (tl >= 2) mbar_wait(&acc_empty[ab], ((tl >> 1) - 1) & 1);
        fence_after();
        const uint32_t tacc = tbase + ab * CF::TCOLS;
        for (int c = 0; c < nch; ++c, ++g) {
          const int s = g % NS;
          const uint32_t ph = (g / NS) & 1;
          mbar_wait(&a_full[s], ph);
          mbar_wait(&b_full[s], ph);
          fence_after();
          const uint32_t ah = smem_u32(A_hi(s)), al = smem_u32(A_lo(s));
          const uint32_t bh = smem_u32(B_hi(s)), bl = smem_u32(B_lo(s));
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const uint64_t dah = sdesc(ah + k * 4096, 2048, 128);
            const uint64_t dal = sdesc(al + k * 4096, 2048, 128);
            const uint64_t dbh = sdesc(bh + k * 32 * BN, 16 * BN, 128);
            const uint64_t dbl = sdesc(bl + k * 32 * BN, 16 * BN, 128);
            umma_ss(tacc, dah, dbh, ID, (c > 0 || k > 0));
            umma_ss(tacc, dah, dbl, ID, 1);
            umma_ss(tacc, dal, dbh, ID, 1);
          }
          umma_commit(&done[s]);
          if (g >= 1 && (g - 1) + NS < total) {
            mbar_wait(&done[(g - 1) % NS], ((g - 1) / NS) & 1);
            load_b(g - 1 + NS);
          }
        }
        umma_commit(&acc_full[ab]);
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ------------------------------------------------ A loaders: coalesced rows, hi/lo split
    const int lt = threadIdx.x;  // 0..127
    const int kc = lt & 7;
    int g = 0;
    for (int tl = 0; tl < my_tiles; ++tl) {
      const int t = blockIdx.x + tl * gridDim.x;
      const int64_t m0 = (int64_t)(t / nblk) * BM;
      for (int c = 0; c < nch; ++c, ++g) {
        const int s = g % NS;
        if (g >= NS) mbar_wait(&done[s], ((g / NS) - 1) & 1);
        float* ah = A_hi(s);
        float* al = A_lo(s);
        const int k0 = c * BK;
        const bool first = k0 < a.K1;
        const float* base = first ? a.A1 : a.A2;
        const int64_t lda = first ? a.lda1 : a.lda2;
        const int kend = first ? a.K1 : a.K2;
        const int kl = (first ? k0 : k0 - a.K1) + kc * 4;
        float4 x[BM / 16];
#pragma unroll
        for (int i = 0; i < BM / 16; ++i) {  // issue all loads first (8 in flight)
          const int64_t row = m0 + i * 16 + (lt >> 3);
          x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row < a.M) {
            const float* src = base + row * lda;
            if (kl + 4 <= kend) {
              x[i] = *reinterpret_cast<const float4*>(src + kl);
            } else if (kl < kend) {
              float tt[4] = {0.f, 0.f, 0.f, 0.f};
              for (int e = 0; e < 4 && kl + e < kend; ++e) tt[e] = src[kl + e];
              x[i] = make_float4(tt[0], tt[1], tt[2], tt[3]);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < BM / 16; ++i) {
          const int rr = i * 16 + (lt >> 3);
          float4 h = make_float4(tf32rn(x[i].x), tf32rn(x[i].y), tf32rn(x[i].z), tf32rn(x[i].w));
          float4 l = make_float4(tf32rn(x[i].x - h.x), tf32rn(x[i].y - h.y),
                                 tf32rn(x[i].z - h.z), tf32rn(x[i].w - h.w));
          const int off = kc * 512 + (rr >> 3) * 32 + (rr & 7) * 4;
          *reinterpret_cast<float4*>(ah + off) = h;
          *reinterpret_cast<float4*>(al + off) = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&a_full[s]);
      }
    }
  } else {
    // ------------------------------------------------ epilogue: thread = accumulator row
    const int ew = warp - 4;                 // TMEM lane quarter
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    float* stg = epi + ew * 32 * 33;         // [32 rows][33] staging for coalesced stores
    for (int tl = 0; tl < my_tiles; ++tl) {
      const int t = blockIdx.x + tl * gridDim.x;
      const int64_t m0 = (int64_t)(t / nblk) * BM;
      const int n0 = (t % nblk) * BN;
      const int ab = tl & 1;
      mbar_wait(&acc_full[ab], (tl >> 1) & 1);
      fence_after();
      const uint32_t tacc = tbase + ab * CF::TCOLS + lane_off;
      const int64_t row = m0 + ew * 32 + lane;
      const bool rv = row < a.M;
      // write a 32x32 block (rows of this warp, 32 columns from c0) to C coalesced
      auto flush = [&](float* C, int64_t ldc, int c0) {
        __syncwarp();
        for (int i = 0; i < 32; ++i) {
          const int64_t rr = m0 + ew * 32 + i;
          const int n = n0 + c0 + lane;
          if (rr < a.M && n < a.N && c0 + lane < BN) C[rr * ldc + n] = stg[i * 33 + lane];
        }
        __syncwarp();
      };
      if (LN) {
        float mu = 0.f, inv = 0.f;
        // pass 1: x = acc + bias + resid, kept in TMEM; running sum
        float s = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t u[16];
          TG_LD16(tacc + c0, u);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float x = __uint_as_float(u[j]) + (a.bias ? a.bias[c0 + j] : 0.f);
            if (a.resid && rv) x += a.resid[row * a.ldr + c0 + j];
            s += x;
            u[j] = __float_as_uint(x);
          }
          TG_ST16(tacc + c0, u);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        mu = s / BN;
        float q = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t u[16];
          TG_LD16(tacc + c0, u);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float d = __uint_as_float(u[j]) - mu;
            q += d * d;
          }
        }
        inv = 1.f / sqrtf(q / BN + 1e-5f);
        const float* rs = (a.rowscale && rv) ? a.rowscale + (int64_t)a.row_fwd[row] * BN : nullptr;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t u[32];
          TG_LD16(tacc + c0, u);
          TG_LD16(tacc + c0 + 16, (u + 16));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float y[32];
#pragma unroll
          for (int j = 0; j < 32; ++j)
            y[j] = a.ln_g[c0 + j] * ((__uint_as_float(u[j]) - mu) * inv) + a.ln_b[c0 + j];
          if (a.C) {
#pragma unroll
            for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = y[j];
            flush(a.C, a.ldc, c0);
          }
          if (a.rowscale) {
#pragma unroll
            for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = rs ? y[j] * rs[c0 + j] : 0.f;
            flush(a.C2, a.ldc2, c0);
          }
        }
      } else {
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t u[32];
          TG_LD16(tacc + c0, u);
          if (c0 + 16 < BN) TG_LD16(tacc + c0 + 16, (u + 16));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = n0 + c0 + j;
            float x = (c0 + j < BN) ? __uint_as_float(u[j]) : 0.f;
            if (a.bias && n < a.N) x += a.bias[n];
            if (a.act == 1) x = x > 0.f ? x : 0.f;
            else if (a.act == 2) x = 1.f / (1.f + expf(-x));
            stg[lane * 33 + j] = x;
          }
          flush(a.C, a.ldc, c0);
        }
      }
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

template <int BN, bool LN>
static void launch(const tg::Args& a, int nblk, cudaStream_t st) {
  using CF = tg::Cfg<BN>;
  static bool attr = false;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(tg::tc_gemm_kernel<BN, LN>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM));
    attr = true;
  }
  const int ntiles = (int)cdiv(a.M, tg::BM) * nblk;
  const int grid = std::min(ntiles, num_sms());
  tg::tc_gemm_kernel<BN, LN><<<grid, tg::G_THREADS, CF::SMEM, st>>>(a, nblk, ntiles);
  LAUNCH_CHECK();
}

// C = act([A1|A2] @ W + bias) with W prepacked by tc_gemm_pack(K1+K2, N).
void tc_gemm(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
             const float* Wpk, const float* bias, float* C, int64_t ldc, int64_t M, int N,
             int act, cudaStream_t st) {
  if (M <= 0) return;
  GO_CHECK(A2 == nullptr || K1 % tg::BK == 0, "concat split must be a multiple of 32");
  GO_CHECK(lda1 % 4 == 0 && (A2 == nullptr || lda2 % 4 == 0), "A rows must be 16-B aligned");
  tg::Args a{};
  a.A1 = A1; a.lda1 = lda1; a.K1 = K1; a.A2 = A2; a.lda2 = lda2; a.K2 = A2 ? K2 : 0;
  a.Bpk = Wpk; a.bias = bias; a.C = C; a.ldc = ldc; a.M = M; a.N = N;
  a.nch = (int)cdiv(K1 + a.K2, tg::BK);
  a.act = act;
  int BN = tc_gemm_bn(N);
  int nblk = (int)cdiv(N, BN);
  switch (BN) {
    case 16: launch<16, false>(a, nblk, st); break;
    case 32: launch<32, false>(a, nblk, st); break;
    case 48: launch<48, false>(a, nblk, st); break;
    case 64: launch<64, false>(a, nblk, st); break;
    case 128: launch<128, false>(a, nblk, st); break;
    case 144: launch<144, false>(a, nblk, st); break;
    default: launch<256, false>(a, nblk, st); break;
  }
}

// C = LN(resid + [A1|A2] @ W + bias) * g + b  (N == 128); optional C2 = C * rowscale[f].
void tc_gemm_ln(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
                const float* Wpk, const float* bias, const float* resid, int64_t ldr,
                const float* g, const float* beta, float* C, int64_t ldc, const float* rowscale,
                const int32_t* row_fwd, float* C2, int64_t ldc2, int64_t M, int N,
                cudaStream_t st) {
  if (M <= 0) return;
  GO_CHECK(N == 128, "fused LayerNorm epilogue needs N == 128");
  GO_CHECK(A2 == nullptr || K1 % tg::BK == 0, "concat split must be a multiple of 32");
  tg::Args a{};
  a.A1 = A1; a.lda1 = lda1; a.K1 = K1; a.A2 = A2; a.lda2 = lda2; a.K2 = A2 ? K2 : 0;
  a.Bpk = Wpk; a.bias = bias; a.C = C; a.ldc = ldc; a.M = M; a.N = N;
  a.nch = (int)cdiv(K1 + a.K2, tg::BK);
  a.resid = resid; a.ldr = ldr; a.ln_g = g; a.ln_b = beta;
  a.rowscale = rowscale; a.row_fwd = row_fwd; a.C2 = C2; a.ldc2 = ldc2;
  launch<128, true>(a, 1, st);
}

}  // namespace go
