// Full N x N task-head attention (policy.py:210, multi_head_attention(h, h)) on the
// 5th-generation tensor cores: tcgen05.mma kind::tf32, accumulators in TMEM,
// K/V tiles streamed by cp.async.bulk into shared memory, online softmax in the
// exp2 domain by 8 softmax warps (one thread per query row).
//
// CTA = one head x 256 queries of one forward (two 128-row M tiles), 10 warps:
//   warps 0-3  softmax for query tile 0 (TMEM lanes 0-127, warp w -> lanes 32w..)
//   warps 4-7  softmax for query tile 1
//   warp  8    producer: bulk copies of K_j / V_j (4 KB each) into an 8-stage ring
//   warp  9    MMA issuer (one elected thread):
//                S_j = Q K_j^T   (M=128, N=64, K=16 as 2 x K8, A/B from smem)
//                O_j = P_j V_j   (M=128, N=16, K=64 as 8 x K8, A=P from TMEM)
// Per key tile of 64, each query tile uses S[b] (64 TMEM cols) and O[b] (16 cols),
// b = j & 1, so S_{j+1} is computed while the softmax works on S_j.  O_j is
// produced per tile (not accumulated across tiles) and folded into registers by the
// softmax threads with their own rescale, so the running-max correction never has
// to touch TMEM.  P is truncated to tf32 before use and the row sum l is taken over
// the same truncated values, so the normalisation is exactly consistent.
//
// Numerics: Q/K/V are rounded to tf32 (round-to-nearest) by the repack kernel;
// softmax statistics and accumulation are fp32.  Error vs the float64 reference:
// logits ~1e-5 normwise (tests/test_gpu_parity.py enforces 1e-4).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "engine.cuh"

namespace go {
namespace tc {

constexpr int KT = 64;             // keys per tile
constexpr int QT = 128;            // queries per M tile
constexpr int NQT = 3;             // M tiles per CTA (12 softmax warps)
constexpr int NS = 8;              // K/V pipeline stages
constexpr int TILE_BYTES = KT * 16 * 4;  // 4 KB: 64 rows x 16 fp32
constexpr int PRODUCER_WARP = NQT * 4;
constexpr int MMA_WARP = NQT * 4 + 1;
constexpr int NUM_THREADS = (NQT * 4 + 2) * 32;
constexpr uint32_t O_COL = NQT * 128;  // O buffers after the S buffers
constexpr uint32_t TMEM_COLS = 512;

struct Work {
  int32_t f;       // forward
  int32_t q0;      // first local query row of this CTA
  int32_t n;       // rows of the forward
  int32_t tiles;   // key tiles of the forward
  int64_t row0;    // batch row of local row 0
  int64_t tile0;   // first key tile of the forward in the blocked K/V arrays
};

// ---------------------------------------------------------------- PTX helpers
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
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
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
// D[tmem] (+)= A[smem] * B[smem]
__device__ __forceinline__ void umma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

#define TC_LD32(taddr, r)                                                                    \
  asm volatile(                                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%" \
      "15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"          \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),  \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),           \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),        \
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),        \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),        \
        "=r"(r[31])                                                                          \
      : "r"(taddr))
#define TC_ST32(taddr, r)                                                                    \
  asm volatile(                                                                              \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%" \
      "14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(   \
          taddr),                                                                            \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),      \
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),    \
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),    \
      "r"(r[29]), "r"(r[30]), "r"(r[31]))
#define TC_ST16(taddr, r)                                                                    \
  asm volatile(                                                                              \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%" \
      "14,%15,%16};" ::"r"(taddr),                                                           \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),      \
      "r"(r[15]))
#define TC_LD16(taddr, r)                                                                    \
  asm volatile(                                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%" \
      "15}, [%16];"                                                                          \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),  \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),           \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                                                \
      : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Shared-memory matrix descriptor, no swizzle ("interleave"), K-major canonical
// layout: core matrices of 8 rows x 16 B stored contiguously; SBO = byte stride
// between 8-row groups, LBO = byte stride between the two 16-B K chunks.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                 // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
// Instruction descriptor: kind::tf32, D f32, A/B tf32 K-major, shape M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

struct Smem {
  float q[NQT][QT * 16];               // A tiles, K-major canonical (16 KB)
  float kv[NS][2][KT * 16];            // [stage][K|V] 4 KB each (64 KB)
  uint64_t kv_full[NS], kv_empty[NS];
  uint64_t s_full[NQT][2], p_full[NQT][2], o_full[NQT][2], o_free[NQT][2];
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(NUM_THREADS, 1)
    attn_tc_kernel(const float* __restrict__ qh, const float* __restrict__ kb,
                   const float* __restrict__ vb, int64_t R, int64_t Ttot,
                   const Work* __restrict__ works, float* __restrict__ out, int64_t ldo,
                   int d_head, const int32_t* __restrict__ flag) {
  if (flag && !(*flag & 1)) return;  // no bound above BOUND_LIMIT: another kernel ran
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Work w = works[blockIdx.x];
  const int head = blockIdx.y;
  const int T = w.tiles;
  const float* kbase = kb + ((int64_t)head * Ttot + w.tile0) * (KT * 16);
  const float* vbase = vb + ((int64_t)head * Ttot + w.tile0) * (KT * 16);

  // ---- setup: barriers, TMEM, Q tiles
  if (warp == PRODUCER_WARP && lane == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    for (int t = 0; t < NQT; ++t)
      for (int b = 0; b < 2; ++b) {
        mbar_init(&sm.s_full[t][b], 1);
        mbar_init(&sm.p_full[t][b], 128);
        mbar_init(&sm.o_full[t][b], 1);
        mbar_init(&sm.o_free[t][b], 128);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // Q: row-major [R][16] per head -> K-major canonical [c][g][8][4]
  for (int i = threadIdx.x; i < NQT * QT * 4; i += NUM_THREADS) {
    int qt = i / (QT * 4), rem = i % (QT * 4);
    int r = rem >> 2, c = rem & 3;
    int lr = w.q0 + qt * QT + r;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lr < w.n)
      v = *reinterpret_cast<const float4*>(qh + ((int64_t)head * R + w.row0 + lr) * 16 + c * 4);
    *reinterpret_cast<float4*>(&sm.q[qt][c * (QT * 4) + (r >> 3) * 32 + (r & 7) * 4]) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp == PRODUCER_WARP) {
    // ---------------- producer
    if (lane == 0) {
      for (int j = 0; j < T; ++j) {
        int s = j % NS;
        if (j >= NS) mbar_wait(&sm.kv_empty[s], ((j / NS) - 1) & 1);
        mbar_expect_tx(&sm.kv_full[s], 2 * TILE_BYTES);
        bulk_g2s(sm.kv[s][0], kbase + (int64_t)j * (KT * 16), TILE_BYTES, &sm.kv_full[s]);
        bulk_g2s(sm.kv[s][1], vbase + (int64_t)j * (KT * 16), TILE_BYTES, &sm.kv_full[s]);
      }
    }
    __syncwarp();
  } else if (warp == MMA_WARP) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t ID_S = idesc_tf32(QT, KT);
      constexpr uint32_t ID_O = idesc_tf32(QT, 16);
      uint32_t qaddr[NQT];
      for (int t = 0; t < NQT; ++t) qaddr[t] = smem_u32(sm.q[t]);
      auto issue_pv = [&](int j) {
        int s = j % NS, b = j & 1;
        uint32_t vaddr = smem_u32(sm.kv[s][1]);
        for (int t = 0; t < NQT; ++t) {
          mbar_wait(&sm.p_full[t][b], (j >> 1) & 1);
          if (j >= 2) mbar_wait(&sm.o_free[t][b], ((j >> 1) - 1) & 1);
          fence_after();
          uint32_t d = tbase + O_COL + t * 32 + b * 16;
          uint32_t a = tbase + t * 128 + b * 64;
#pragma unroll
          for (int k = 0; k < KT / 8; ++k)  // V^T tile: K chunks of 4 keys at 256 B
            umma_ts(d, a + k * 8, sdesc(vaddr + k * 512, 256, 128), ID_O, k > 0);
          umma_commit(&sm.o_full[t][b]);
        }
        umma_commit(&sm.kv_empty[s]);
      };
      for (int j = 0; j < T; ++j) {
        int s = j % NS, b = j & 1;
        mbar_wait(&sm.kv_full[s], (j / NS) & 1);
        fence_after();
        uint32_t kaddr = smem_u32(sm.kv[s][0]);
        for (int t = 0; t < NQT; ++t) {
          uint32_t d = tbase + t * 128 + b * 64;
#pragma unroll
          for (int k = 0; k < 2; ++k)  // dims 8k..8k+7: chunks 2k, 2k+1
            umma_ss(d, sdesc(qaddr[t] + k * 4096, 2048, 128), sdesc(kaddr + k * 2048, 1024, 128),
                    ID_S, k > 0);
          umma_commit(&sm.s_full[t][b]);
        }
        if (j >= 1) issue_pv(j - 1);
      }
      if (T >= 1) issue_pv(T - 1);
    }
    __syncwarp();
  } else {
    // ---------------- softmax: one thread per query row
    const int t = warp >> 2;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const int lr = w.q0 + t * QT + row;
    float m = -INFINITY, l = 0.f;
    float oacc[16];
#pragma unroll
    for (int d = 0; d < 16; ++d) oacc[d] = 0.f;
    float mt[2] = {0.f, 0.f};
    auto fold = [&](int j) {
      int b = j & 1;
      mbar_wait(&sm.o_full[t][b], (j >> 1) & 1);
      fence_after();
      uint32_t r[16];
      TC_LD16(tbase + lane_off + O_COL + t * 32 + b * 16, r);
      tmem_wait_ld();
      fence_before();
      mbar_arrive(&sm.o_free[t][b]);
      float sc = ex2(mt[b] - m);
#pragma unroll
      for (int d = 0; d < 16; ++d) oacc[d] = fmaf(sc, __uint_as_float(r[d]), oacc[d]);
    };
    for (int j = 0; j < T; ++j) {
      int b = j & 1;
      mbar_wait(&sm.s_full[t][b], (j >> 1) & 1);
      fence_after();
      uint32_t sr[64];
      const uint32_t sa = tbase + lane_off + t * 128 + b * 64;
      TC_LD32(sa, sr);
      TC_LD32(sa + 32, (sr + 32));
      tmem_wait_ld();
      const int kvalid = w.n - j * KT;  // keys of this tile inside the forward
      if (kvalid < KT) {
#pragma unroll
        for (int i = 0; i < KT; ++i)
          if (i >= kvalid) sr[i] = __float_as_uint(-INFINITY);
      }
      // row max with 8 independent chains (dependent FMNMX chains were the stall)
      float mx[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx[i] = __uint_as_float(sr[i]);
#pragma unroll
      for (int i = 8; i < KT; ++i) mx[i & 7] = fmaxf(mx[i & 7], __uint_as_float(sr[i]));
      const float tm = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                             fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      float mn = fmaxf(m, tm);
      if (mn > m) {
        float corr = ex2(m - mn);
        l *= corr;
#pragma unroll
        for (int d = 0; d < 16; ++d) oacc[d] *= corr;
        m = mn;
      }
      float ls[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) ls[i] = 0.f;
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        uint32_t pb = __float_as_uint(ex2(__uint_as_float(sr[i]) - m)) & 0xFFFFE000u;
        ls[i & 7] += __uint_as_float(pb);
        sr[i] = pb;
      }
      l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
      TC_ST32(sa, sr);
      TC_ST32(sa + 32, (sr + 32));
      tmem_wait_st();
      fence_before();
      mbar_arrive(&sm.p_full[t][b]);
      mt[b] = m;
      if (j >= 1) fold(j - 1);
    }
    if (T >= 1) fold(T - 1);
    if (lr < w.n) {
      float inv = 1.f / l;
      float* o = out + (w.row0 + lr) * ldo + head * d_head;
      for (int d = 0; d < d_head; ++d) o[d] = oacc[d] * inv;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                 "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------------------------
// Repack the QKV projections [R, n_head*d_head] into the tensor-core layouts:
//   qh [H][R][16]     row-major, scaled by log2(e)/sqrt(d_head), tf32-rounded
//   kb [H][Ttot][..]  per 64-key tile, K-major canonical:  (c, g, r, e) at c*256 + g*32 + r*4 + e
//   vb [H][Ttot][..]  per 64-key tile, V^T K-major:        (kc, dg, rd, e) at kc*64 + dg*32 + rd*4 + e
// Rows past a forward's end (inside its last tile) are zero.
__device__ __forceinline__ float tf32r(float x) {
  uint32_t y;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(y) : "f"(x));
  return __uint_as_float(y);
}

__global__ void repack_kernel(const float* __restrict__ q, const float* __restrict__ k,
                              const float* __restrict__ v, int64_t ld, int n_head, int d_head,
                              const int64_t* __restrict__ tile_fwd_row0,
                              const int32_t* __restrict__ tile_n, int64_t Ttot, int64_t R,
                              float qscale, float* __restrict__ qh, float* __restrict__ kb,
                              float* __restrict__ vb, const int32_t* __restrict__ flag) {
  if (flag && !(*flag & 1)) return;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (head, tile, row)
  int64_t total = (int64_t)n_head * Ttot * KT;
  if (idx >= total) return;
  int head = (int)(idx / (Ttot * KT));
  int64_t rem = idx % (Ttot * KT);
  int64_t tile = rem / KT;
  int rk = (int)(rem % KT);
  int local = (int)tile_n[3 * tile + 1] * KT + rk;  // row within the forward
  bool valid = local < tile_n[3 * tile];
  int64_t grow = tile_fwd_row0[tile] + local;
  float* kt = kb + ((int64_t)head * Ttot + tile) * (KT * 16);
  float* vt = vb + ((int64_t)head * Ttot + tile) * (KT * 16);
  for (int d = 0; d < 16; ++d) {
    float kv = 0.f, vv = 0.f, qv = 0.f;
    if (valid && d < d_head) {
      int64_t o = grow * ld + head * d_head + d;
      kv = tf32r(k[o]);
      vv = tf32r(v[o]);
      qv = tf32r(q[o] * qscale);
    }
    kt[(d >> 2) * 256 + (rk >> 3) * 32 + (rk & 7) * 4 + (d & 3)] = kv;
    vt[(rk >> 2) * 64 + (d >> 3) * 32 + (d & 7) * 4 + (rk & 3)] = vv;
    if (valid) qh[((int64_t)head * R + grow) * 16 + d] = qv;
  }
}


// ------------------------------------------------------------------------------------
// Fixed-offset variant (d_head <= 15).  Column 15 of the padded head dimension is
// spare, so it carries the softmax bookkeeping through the tensor core:
//   Q[:,15] = -b_i  with b_i >= max_j s_ij (Cauchy-Schwarz: |q_i| * max_j |k_j|)
//   K[:,15] = 1     =>  the S MMA returns s_ij - b_i <= 0 directly
//   V[:,15] = 1     =>  the PV MMA returns l_i = sum_j p_ij in O[:,15], computed from
//                       exactly the tf32 P the numerator used.
// No running max, no rescale, no row sum and no per-tile O traffic: the softmax warps
// only do tcgen05.ld S -> ex2 -> tcgen05.st P, and O accumulates across all key tiles
// in TMEM.  Padding keys have all-zero K and V rows, so they contribute nothing.  Used
// when every b_i <= BOUND_LIMIT (exp2 then never underflows for scores within 2 b_i
// of the bound); otherwise the online-softmax kernel above takes the launch.
constexpr float BOUND_LIMIT = 60.f;

// The fixed kernel runs two CTAs per SM (TMEM 2 x 256 columns) so the softmax warps
// of two independent CTAs interleave on each SM sub-partition and keep the MUFU pipe
// busy through each other's tcgen05.ld/st and barrier latencies.  Each 64-key K/V
// tile is consumed as two 32-key halves (S sub-tiles of 32 TMEM columns, double
// buffered per query tile): 3 x 2 x 32 S columns + 3 x 16 O columns = 240 <= 256.
// O accumulates in TMEM over DRAIN_U sub-tiles only; at each group boundary the MMA
// thread commits o_ready, the softmax thread adds the group's O into a float sum in
// shared memory (tc_attention16.cu explains why: the tensor core's accumulate drifts
// over thousands of additions), and the next group restarts the accumulator.
constexpr int HK = 32;                      // keys per softmax sub-tile
constexpr int NSF = 6;                      // K/V ring stages per CTA
constexpr int DRAIN_U = 16;                 // 32-key sub-tiles per accumulation group
constexpr uint32_t O_COL_F = NQT * 2 * HK;  // O accumulators after the S buffers
constexpr uint32_t TMEM_COLS_F = 256;

struct SmemF {
  float q[NQT][QT * 16];
  float kv[NSF][2][KT * 16];
  float osum[NQT][16][QT];  // drained O groups, [tile][column][row]
  uint64_t kv_full[NSF], kv_empty[NSF];
  uint64_t s_full[NQT][2], p_full[NQT][2], o_ready[NQT], o_done[NQT];
  uint32_t tmem_base;
};

// Launch flag bits (attention_full_tc): 1 = the online kernel takes the launch,
// 2 = the tf32 kernel takes the launch, 4 = the tf32 kernel takes the work items the
// fp16 kernel marked in wflag.  primary: the tf32 kernel is the first choice (no fp16
// pass before it).
__device__ __forceinline__ bool tf32_launch(int32_t flag, bool primary) {
  return !(flag & 1) && (primary || (flag & 6));
}
__device__ __forceinline__ bool tf32_work(int32_t flag, bool primary, const int32_t* wflag,
                                          int64_t item) {
  if (!tf32_launch(flag, primary)) return false;
  return primary || (flag & 2) || wflag[item];
}

// Pipelined softmax loop: 16-column chunks, the next chunk's tcgen05.ld in flight while
// this chunk's ex2s issue.
__global__ void __launch_bounds__(NUM_THREADS, 2)
    attn_tc_fixed_kernel(const float* __restrict__ qh, const float* __restrict__ kb,
                         const float* __restrict__ vb, int64_t R, int64_t Ttot,
                         const Work* __restrict__ works, float* __restrict__ out, int64_t ldo,
                         int d_head, const int32_t* __restrict__ flag,
                         const int32_t* __restrict__ wflag, bool primary) {
  if (!tf32_work(*flag, primary, wflag, (int64_t)blockIdx.y * gridDim.x + blockIdx.x)) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SmemF& sm = *reinterpret_cast<SmemF*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Work w = works[blockIdx.x];
  const int head = blockIdx.y;
  const int T = w.tiles;
  const int U = 2 * T;  // 32-key sub-tiles
  const float* kbase = kb + ((int64_t)head * Ttot + w.tile0) * (KT * 16);
  const float* vbase = vb + ((int64_t)head * Ttot + w.tile0) * (KT * 16);
  if (warp == PRODUCER_WARP && lane == 0) {
    for (int s = 0; s < NSF; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
    }
    for (int t = 0; t < NQT; ++t) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(&sm.s_full[t][b], 1);
        mbar_init(&sm.p_full[t][b], 128);
      }
      mbar_init(&sm.o_ready[t], 1);
      mbar_init(&sm.o_done[t], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(TMEM_COLS_F));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < NQT * QT * 4; i += NUM_THREADS) {
    int qt = i / (QT * 4), rem = i % (QT * 4);
    int r = rem >> 2, c = rem & 3;
    int lr = w.q0 + qt * QT + r;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lr < w.n)
      v = *reinterpret_cast<const float4*>(qh + ((int64_t)head * R + w.row0 + lr) * 16 + c * 4);
    *reinterpret_cast<float4*>(&sm.q[qt][c * (QT * 4) + (r >> 3) * 32 + (r & 7) * 4]) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp == PRODUCER_WARP) {
    if (lane == 0) {
      for (int j = 0; j < T; ++j) {
        int s = j % NSF;
        if (j >= NSF) mbar_wait(&sm.kv_empty[s], ((j / NSF) - 1) & 1);
        mbar_expect_tx(&sm.kv_full[s], 2 * TILE_BYTES);
        bulk_g2s(sm.kv[s][0], kbase + (int64_t)j * (KT * 16), TILE_BYTES, &sm.kv_full[s]);
        bulk_g2s(sm.kv[s][1], vbase + (int64_t)j * (KT * 16), TILE_BYTES, &sm.kv_full[s]);
      }
    }
    __syncwarp();
  } else if (warp == MMA_WARP) {
    if (lane == 0) {
      constexpr uint32_t ID_S = idesc_tf32(QT, HK);
      constexpr uint32_t ID_O = idesc_tf32(QT, 16);
      uint32_t qaddr[NQT];
      for (int t = 0; t < NQT; ++t) qaddr[t] = smem_u32(sm.q[t]);
      // Per query tile t the issue order is  ... PV(u, t), S(u + 2, t) ...  as soon as
      // P(u, t) is in TMEM, so each query tile's softmax warps always have the next S
      // ready and never wait for the other query tiles.  S(u + 2, t) reuses the TMEM
      // buffer of P(u, t), which the in-order tensor pipe has consumed by then.
      auto wait_kv = [&](int u) {
        if ((u & 1) == 0) {
          const int j = u >> 1;
          mbar_wait(&sm.kv_full[j % NSF], (j / NSF) & 1);
          fence_after();
        }
      };
      auto issue_s = [&](int u, int t) {
        const int j = u >> 1, h = u & 1, s = j % NSF, b = u & 1;
        const uint32_t kaddr = smem_u32(sm.kv[s][0]) + h * (HK * 4 * 4);
        const uint32_t d = tbase + t * 2 * HK + b * HK;
#pragma unroll
        for (int k = 0; k < 2; ++k)
          umma_ss(d, sdesc(qaddr[t] + k * 4096, 2048, 128), sdesc(kaddr + k * 2048, 1024, 128),
                  ID_S, k > 0);
        umma_commit(&sm.s_full[t][b]);
      };
      for (int u = 0; u < 2 && u < U; ++u) {
        wait_kv(u);
        for (int t = 0; t < NQT; ++t) issue_s(u, t);
      }
      for (int u = 0; u < U; ++u) {
        const int j = u >> 1, h = u & 1, s = j % NSF, b = u & 1;
        const bool more = u + 2 < U;
        if (more) wait_kv(u + 2);
        const uint32_t vaddr = smem_u32(sm.kv[s][1]) + h * (HK * 16 * 4);
        for (int t = 0; t < NQT; ++t) {
          mbar_wait(&sm.p_full[t][b], (u >> 1) & 1);
          fence_after();
          const uint32_t d = tbase + O_COL_F + t * 16;
          const uint32_t a = tbase + t * 2 * HK + b * HK;
#pragma unroll
          for (int k = 0; k < HK / 8; ++k)  // a new accumulation group restarts O
            umma_ts(d, a + k * 8, sdesc(vaddr + k * 512, 256, 128), ID_O,
                    (u % DRAIN_U != 0 || k > 0));
          if ((u + 1) % DRAIN_U == 0 && u + 1 < U) umma_commit(&sm.o_ready[t]);
          if (more) issue_s(u + 2, t);
        }
        if (h == 1) umma_commit(&sm.kv_empty[s]);  // both halves' PV issued
      }
      for (int t = 0; t < NQT; ++t) umma_commit(&sm.o_done[t]);
    }
    __syncwarp();
  } else {
    // chunk c = 2u + h: columns [16h, 16h + 16) of sub-tile u.  The tcgen05.ld of chunk
    // c + 1 is issued before chunk c's ex2s, so the MUFU queue never waits on a TMEM
    // load; P(u) is released after its second chunk's tcgen05.st lands.
    const int t = warp >> 2;
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t base = tbase + lane_off + t * 2 * HK;
    const uint32_t obase = tbase + lane_off + O_COL_F + t * 16;
    float* osum = &sm.osum[t][0][row];
#pragma unroll
    for (int d = 0; d < 16; ++d) osum[d * QT] = 0.f;
    auto caddr = [&](int c) { return base + ((c >> 1) & 1) * HK + (c & 1) * 16; };
    uint32_t ra[16], rb[16];
    if (U > 0) {
      mbar_wait(&sm.s_full[t][0], 0);
      fence_after();
      TC_LD16(caddr(0), ra);
      tmem_wait_ld();
    }
    for (int u = 0; u < U; ++u) {
      const int c = 2 * u;
      TC_LD16(caddr(c + 1), rb);
#pragma unroll
      for (int i = 0; i < 16; ++i) ra[i] = __float_as_uint(ex2(__uint_as_float(ra[i])));
      TC_ST16(caddr(c), ra);
      tmem_wait_ld();
      const bool more = u + 1 < U;
      if (more) {
        mbar_wait(&sm.s_full[t][(u + 1) & 1], ((u + 1) >> 1) & 1);
        fence_after();
        TC_LD16(caddr(c + 2), ra);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) rb[i] = __float_as_uint(ex2(__uint_as_float(rb[i])));
      TC_ST16(caddr(c + 1), rb);
      tmem_wait_st();
      if (u > 0 && u % DRAIN_U == 0) {  // O = sub-tiles [u - DRAIN_U, u); PV(u) waits on us
        mbar_wait(&sm.o_ready[t], ((u / DRAIN_U) - 1) & 1);
        fence_after();
        TC_LD16(obase, rb);
        tmem_wait_ld();
#pragma unroll
        for (int d = 0; d < 16; ++d) osum[d * QT] += __uint_as_float(rb[d]);
      }
      fence_before();
      mbar_arrive(&sm.p_full[t][u & 1]);
      if (more) tmem_wait_ld();
    }
    mbar_wait(&sm.o_done[t], 0);
    fence_after();
    if (U > 0) {
      uint32_t r[16];
      TC_LD16(obase, r);
      tmem_wait_ld();
#pragma unroll
      for (int d = 0; d < 16; ++d) osum[d * QT] += __uint_as_float(r[d]);
    }
    const int lr = w.q0 + t * QT + row;
    if (lr < w.n) {
      float inv = 1.f / osum[15 * QT];
      float* o = out + (w.row0 + lr) * ldo + head * d_head;
      for (int d = 0; d < d_head; ++d) o[d] = osum[d * QT] * inv;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                 "r"(TMEM_COLS_F));
  }
}

// K/V for the fixed variant: column 15 = 1 on valid rows; max |k| per (forward, head).
__global__ void repack_kv_fixed_kernel(const float* __restrict__ k, const float* __restrict__ v,
                                       int64_t ld, int n_head, int d_head,
                                       const int64_t* __restrict__ tile_fwd_row0,
                                       const int32_t* __restrict__ tile_n, int64_t Ttot,
                                       float* __restrict__ kb, float* __restrict__ vb,
                                       unsigned* __restrict__ kmax,
                                       const int32_t* __restrict__ flag, bool primary) {
  if (!tf32_launch(*flag, primary)) return;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)n_head * Ttot * KT;
  if (idx >= total) return;
  int head = (int)(idx / (Ttot * KT));
  int64_t rem = idx % (Ttot * KT);
  int64_t tile = rem / KT;
  int rk = (int)(rem % KT);
  int local = (int)tile_n[3 * tile + 1] * KT + rk;
  bool valid = local < tile_n[3 * tile];
  int fwd = tile_n[3 * tile + 2];
  int64_t grow = tile_fwd_row0[tile] + local;
  float* kt = kb + ((int64_t)head * Ttot + tile) * (KT * 16);
  float* vt = vb + ((int64_t)head * Ttot + tile) * (KT * 16);
  float nk = 0.f;
  for (int d = 0; d < 16; ++d) {
    float kv = 0.f, vv = 0.f;
    if (valid) {
      if (d < d_head) {
        int64_t o = grow * ld + head * d_head + d;
        kv = tf32r(k[o]);
        vv = tf32r(v[o]);
        nk = fmaf(kv, kv, nk);
      } else if (d == 15) {
        kv = 1.f;
        vv = 1.f;
      }
    }
    kt[(d >> 2) * 256 + (rk >> 3) * 32 + (rk & 7) * 4 + (d & 3)] = kv;
    vt[(rk >> 2) * 64 + (d >> 3) * 32 + (d & 7) * 4 + (rk & 3)] = vv;
  }
  if (valid) atomicMax(&kmax[fwd * n_head + head], __float_as_uint(sqrtf(nk)));
}

// Q for the fixed variant: scaled by log2(e)/sqrt(d_head), tf32-rounded, column 15 =
// -b_i with b_i = |q_i| * max|k| * (1 + 2^-8) + 2^-8 (>= every score, after rounding).
__global__ void repack_q_fixed_kernel(const float* __restrict__ q, int64_t ld, int n_head,
                                      int d_head, int64_t R, const int32_t* __restrict__ row_fwd,
                                      const unsigned* __restrict__ kmax, float qscale,
                                      float* __restrict__ qh, int32_t* __restrict__ flag,
                                      bool primary) {
  if (!tf32_launch(*flag, primary)) return;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= R * n_head) return;
  int64_t r = idx / n_head;
  int head = (int)(idx % n_head);
  float qv[16];
  float nq = 0.f;
  for (int d = 0; d < 16; ++d) {
    float x = d < d_head ? tf32r(q[r * ld + head * d_head + d] * qscale) : 0.f;
    qv[d] = x;
    nq = fmaf(x, x, nq);
  }
  float km = __uint_as_float(kmax[row_fwd[r] * n_head + head]);
  float bnd = sqrtf(nq) * km * (1.f + 1.f / 256.f) + 1.f / 256.f;
  if (!(bnd <= BOUND_LIMIT)) atomicOr(flag, 1);
  qv[15] = -bnd;
  float* o = qh + ((int64_t)head * R + r) * 16;
  for (int d = 0; d < 16; ++d) o[d] = qv[d];
}
}  // namespace tc

bool tc_attention_supported(int d_head) { return d_head <= 16; }

void tc_build_tables(const std::vector<int64_t>& row_off, std::vector<TcWork>& works,
                     std::vector<int64_t>& tile_row0, std::vector<int32_t>& tile_n) {
  int F = (int)row_off.size() - 1;
  int64_t tb = 0;
  for (int f = 0; f < F; ++f) {
    int64_t n = row_off[f + 1] - row_off[f];
    int32_t T = (int32_t)cdiv(n, tc::KT);
    for (int64_t q0 = 0; q0 < n; q0 += tc::NQT * tc::QT)
      works.push_back(TcWork{f, (int32_t)q0, (int32_t)n, T, row_off[f], tb});
    for (int32_t t = 0; t < T; ++t) {
      tile_row0.push_back(row_off[f]);
      tile_n.push_back((int32_t)n);
      tile_n.push_back(t);
      tile_n.push_back(f);
    }
    tb += T;
  }
}

int64_t tc_attention_scratch_ints(int F, int n_head, int64_t num_works) {
  return 1 + (int64_t)F * n_head + (int64_t)n_head * num_works;
}

void attention_full_tc(const float* q, const float* k, const float* v, int64_t ld, int n_head,
                       int d_head, int64_t R, int64_t Ttot, const TcWork* works_dev,
                       int64_t num_works, const int64_t* tile_row0_dev,
                       const int32_t* tile_n_dev, float* qh, float* kb, float* vb, float* out,
                       int64_t ldo, const int32_t* row_fwd, int F, int32_t* scratch,
                       cudaStream_t st) {
  if (num_works <= 0) return;
  if (d_head > 16) GO_THROW(GO_ERR_UNSUPPORTED, "tensor-core attention needs d_head <= 16");
  static bool attr = false;
  const size_t smem = sizeof(tc::Smem) + 1024;
  const size_t smemf = sizeof(tc::SmemF) + 1024;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(tc::attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    CUDA_CHECK(cudaFuncSetAttribute(tc::attn_tc_fixed_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemf));
    attr = true;
  }
  // A/B switch (tests and timing only): GO_ATTN=tf32 makes the tf32 fixed-offset kernel
  // the first choice, GO_ATTN=online forces the online-softmax kernel
  const char* force = getenv("GO_ATTN");
  const bool use16 = d_head <= 15 && !(force && (!strcmp(force, "tf32") || !strcmp(force, "online")));
  float qscale = (float)(1.4426950408889634 / std::sqrt((double)d_head));
  int64_t total = (int64_t)n_head * Ttot * tc::KT;
  dim3 grid((unsigned)num_works, (unsigned)n_head);
  bool fixed_ok = d_head <= 15 && !(force && !strcmp(force, "online"));
  if (fixed_ok) {
    // scratch: [0] launch flag, [1, 1 + F*H) max |k| per (forward, head),
    // then per (head, work item) fallback marks of the fp16 kernel
    int32_t* flag = scratch;
    unsigned* kmax = reinterpret_cast<unsigned*>(scratch + 1);
    int32_t* wflag = scratch + 1 + (int64_t)F * n_head;
    CUDA_CHECK(cudaMemsetAsync(
        scratch, 0, (size_t)tc_attention_scratch_ints(F, n_head, num_works) * 4, st));
    if (use16)
      attention_f16_tc(q, k, v, ld, n_head, d_head, R, Ttot, works_dev, num_works, tile_row0_dev,
                       tile_n_dev, qh, kb, vb, out, ldo, row_fwd, kmax, flag, wflag, qscale, st);
    const bool primary = !use16;
    tc::repack_kv_fixed_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(
        k, v, ld, n_head, d_head, tile_row0_dev, tile_n_dev, Ttot, kb, vb, kmax, flag, primary);
    LAUNCH_CHECK();
    tc::repack_q_fixed_kernel<<<(unsigned)cdiv(R * n_head, 256), 256, 0, st>>>(
        q, ld, n_head, d_head, R, row_fwd, kmax, qscale, qh, flag, primary);
    LAUNCH_CHECK();
    tc::attn_tc_fixed_kernel<<<grid, tc::NUM_THREADS, smemf, st>>>(
        qh, kb, vb, R, Ttot, reinterpret_cast<const tc::Work*>(works_dev), out, ldo, d_head, flag,
        wflag, primary);
    LAUNCH_CHECK();
    // fallback for bounds > BOUND_LIMIT: the online kernel re-packs and runs only if flagged
    tc::repack_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(
        q, k, v, ld, n_head, d_head, tile_row0_dev, tile_n_dev, Ttot, R, qscale, qh, kb, vb, flag);
    LAUNCH_CHECK();
    tc::attn_tc_kernel<<<grid, tc::NUM_THREADS, smem, st>>>(
        qh, kb, vb, R, Ttot, reinterpret_cast<const tc::Work*>(works_dev), out, ldo, d_head, flag);
    LAUNCH_CHECK();
    return;
  }
  tc::repack_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(
      q, k, v, ld, n_head, d_head, tile_row0_dev, tile_n_dev, Ttot, R, qscale, qh, kb, vb, nullptr);
  LAUNCH_CHECK();
  tc::attn_tc_kernel<<<grid, tc::NUM_THREADS, smem, st>>>(
      qh, kb, vb, R, Ttot, reinterpret_cast<const tc::Work*>(works_dev), out, ldo, d_head, nullptr);
  LAUNCH_CHECK();
}

}  // namespace go
