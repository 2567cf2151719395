// Task-head N x N attention, fp16 tensor-core kernel (policy.py:210 multi_head_attention
// over all rows), the default path of every forward's heads.
//
// Per (head, 384 queries) CTA, two CTAs per SM (TMEM 2 x 256 columns), 16 warps:
//   warps 0-11  softmax: one thread per query row (3 tiles x 128 TMEM lanes)
//   warp 12     producer: cp.async.bulk of 64-key K and V^T fp16 tiles into an 8-stage ring
//   warps 13-15 one MMA-issuing thread per query tile:
//     S = Q K^T      kind::f16, M=128, N=64, K=16: one MMA per 64-key tile
//     O += P V       kind::f16, M=128, N=16, A = P packed fp16x2 in TMEM: 4 MMAs
//
// Fixed-offset softmax.  Q[:,15] = 15 - b_i (b_i >= |q_i| max|k|, a Cauchy-Schwarz bound)
// against K[:,15] = 1 makes the MMA return S' = s - b_i + 15 <= 15, so P' = 2^S' <= 2^15
// never overflows fp16, and while b_i <= F16_LIMIT = 14 every S' >= -13 gives a normal
// fp16 P'.  V[:,15] = 1 makes O[:,15] the row sum of exactly the P' the numerator used,
// so the 2^(15 - b_i) scale cancels in O / O[:,15]: no running max, no rescale.
// Half of the exponentials run as an fp16x2 polynomial on the FMA pipe (ptx::
// exp2_poly_f16x2_lp), half on MUFU.EX2 (16/clk/SM): together 1.24x the MUFU rate.
//
// Accumulation.  The tensor core's fp32 accumulate does not round the low bits of
// small addends to nearest; summed over the 1,250 key tiles of an 80k-node graph (where
// the random-init rows are nearly parallel and every addend has the same sign pattern)
// that drift reached 1.4e-4 of the logits.  So O accumulates in TMEM over only DRAIN = 16
// key tiles; at each group boundary the softmax thread, which owns its row, reads the
// 16 O columns and adds them into a float sum in shared memory (IEEE round-to-nearest,
// ~80 additions at 80k keys, two columns per packed FADD2), and the MMA thread restarts
// the accumulator.  Measured at cfg4 (scripts/parity_variants.py): logits 1.41e-4 ->
// 5.6e-6 normwise from float64 (DRAIN = 8: 4.8e-6 for twice the drain instructions;
// 32: 7.6e-6).  The drain needs no extra barrier: S(j) is
// issued after PV(j-1) by the same thread and tcgen05 MMAs complete in order, so when
// s_full(j) fires O holds exactly tiles [.., j-1], and PV(j) (accumulate = 0) waits for
// p_full(j), which this thread signals only after the drain.
//
// Fallback per work item.  A row whose bound exceeds F16_LIMIT gets NaN in Q[:,15]
// (repack_q16_kernel); the CTA owning it sees the NaN while staging Q, marks its
// (work, head) in wflag, sets bit 4 of the launch flag and exits, and the tf32 kernel
// (tc_attention.cu) recomputes only the marked work items.  Bounds above BOUND_LIMIT
// (bit 1) and operands outside the fp16 range (bit 2) still move the whole launch.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cuda_fp16.h>

#include "engine.cuh"
#include "tcgen05.cuh"

namespace go {
namespace t16 {

using namespace ptx;

constexpr int KT = 64;   // keys per K/V tile (tile tables shared with the tf32 path)
constexpr int QT = 128;  // queries per M tile
constexpr int NQT = 3;   // M tiles per CTA
constexpr int NS = 8;    // K/V ring stages
constexpr int DRAIN = 16;  // key tiles per TMEM accumulation group
constexpr int NP = 4;    // of every 8 exponential pairs, NP on the FMA-pipe polynomial
constexpr int TILE_BYTES = KT * 16 * 2;
constexpr int PRODUCER_WARP = NQT * 4;
constexpr int MMA_WARP0 = NQT * 4 + 1;
constexpr int NUM_THREADS = (NQT * 5 + 1) * 32;
constexpr uint32_t S_COLS = KT;            // S columns per query tile (P packed into half)
constexpr uint32_t O_COL = NQT * S_COLS;   // O accumulators after the S buffers
constexpr uint32_t TMEM_COLS = 256;
static_assert(O_COL + NQT * 16 <= TMEM_COLS, "TMEM budget");
constexpr float F16_LIMIT = 14.f;
constexpr float BOUND_LIMIT = 60.f;
constexpr float RANGE_LIMIT = 60000.f;

struct Smem {
  uint16_t q[NQT][QT * 16];
  uint16_t kv[NS][2][KT * 16];
  float4 osum[NQT][4][QT];   // sum of the drained O groups, [tile][column/4][row]
  uint64_t kv_full[NS], kv_empty[NS];
  uint64_t s_full[NQT], p_full[NQT], o_done[NQT];
  uint32_t tmem_base;
  int32_t fallback;
};

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
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
// {a.x + b.x, a.y + b.y} in one packed fp32 add (FADD2), IEEE round-to-nearest
__device__ __forceinline__ float2 add_f32x2(float2 a, float2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
  return *reinterpret_cast<const float2*>(&r);
}
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// 16 S columns -> 8 packed fp16x2 P columns; pairs at odd positions first on the
// polynomial so MUFU and FMA work interleave
__device__ __forceinline__ void softmax16(const uint32_t* r, uint32_t* pk) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool poly = (i & 1) ? ((i >> 1) < NP) : ((4 + (i >> 1)) < NP);
    const float x0 = __uint_as_float(r[2 * i]), x1 = __uint_as_float(r[2 * i + 1]);
    pk[i] = poly ? exp2_poly_f16x2_lp(x0, x1) : pack_f16x2(ex2f(x0), ex2f(x1));
  }
}

__global__ void __launch_bounds__(NUM_THREADS, 2)
    attn_f16_kernel(const uint16_t* __restrict__ qh, const uint16_t* __restrict__ kb,
                    const uint16_t* __restrict__ vb, int64_t R, int64_t Ttot,
                    const TcWork* __restrict__ works, float* __restrict__ out, int64_t ldo,
                    int d_head, int32_t* __restrict__ flag, int32_t* __restrict__ wflag) {
  if (*flag & 3) return;  // the whole launch goes to the tf32 or the online kernel
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TcWork w = works[blockIdx.x];
  const int head = blockIdx.y;
  const int T = w.tiles;
  const uint16_t* kbase = kb + ((int64_t)head * Ttot + w.tile0) * (KT * 16);
  const uint16_t* vbase = vb + ((int64_t)head * Ttot + w.tile0) * (KT * 16);
  if (threadIdx.x == 0) sm.fallback = 0;
  __syncthreads();
  // Q: per query tile, K-major canonical (two 8-half K chunks of 8-row core matrices);
  // the chunk holding column 15 carries the NaN fallback marker
  bool marked = false;
  for (int i = threadIdx.x; i < NQT * QT * 2; i += NUM_THREADS) {
    const int qt = i / (QT * 2), rem = i % (QT * 2);
    const int r = rem >> 1, c = rem & 1;
    const int lr = w.q0 + qt * QT + r;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (lr < w.n) {
      v = *reinterpret_cast<const uint4*>(qh + ((int64_t)head * R + w.row0 + lr) * 16 + c * 8);
      marked |= c == 1 && ((v.w >> 16) & 0x7FFFu) > 0x7C00u;  // column 15 is NaN
    }
    *reinterpret_cast<uint4*>(&sm.q[qt][c * (QT * 8) + (r >> 3) * 64 + (r & 7) * 8]) = v;
  }
  if (marked) sm.fallback = 1;
  __syncthreads();
  if (sm.fallback) {
    if (threadIdx.x == 0) {
      wflag[(int64_t)head * gridDim.x + blockIdx.x] = 1;
      atomicOr(flag, 4);
    }
    return;
  }
  if (warp == PRODUCER_WARP && lane == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], NQT);
    }
    for (int t = 0; t < NQT; ++t) {
      mbar_init(&sm.s_full[t], 1);
      mbar_init(&sm.p_full[t], 128);
      mbar_init(&sm.o_done[t], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp == PRODUCER_WARP) {
    if (lane == 0) {
      for (int j = 0; j < T; ++j) {
        const int s = j % NS;
        if (j >= NS) mbar_wait_sleep(&sm.kv_empty[s], ((j / NS) - 1) & 1);
        mbar_expect_tx(&sm.kv_full[s], 2 * TILE_BYTES);
        bulk_g2s(sm.kv[s][0], kbase + (int64_t)j * (KT * 16), TILE_BYTES, &sm.kv_full[s]);
        bulk_g2s(sm.kv[s][1], vbase + (int64_t)j * (KT * 16), TILE_BYTES, &sm.kv_full[s]);
      }
    }
    __syncwarp();
  } else if (warp >= MMA_WARP0) {
    if (lane == 0) {
      const int t = warp - MMA_WARP0;
      constexpr uint32_t ID_S = idesc_f16(QT, KT);
      constexpr uint32_t ID_O = idesc_f16(QT, 16);
      const uint64_t qd = sdesc(smem_u32(sm.q[t]), QT * 16, 128);
      const uint32_t sd = tbase + t * S_COLS;
      const uint32_t od = tbase + O_COL + t * 16;
      auto issue_s = [&](int j) {
        const int s = j % NS;
        mbar_wait_sleep(&sm.kv_full[s], (j / NS) & 1);
        fence_after();
        umma_ss_f16(sd, qd, sdesc(smem_u32(sm.kv[s][0]), KT * 16, 128), ID_S, 0);
        umma_commit(&sm.s_full[t]);
      };
      if (T > 0) issue_s(0);
      for (int j = 0; j < T; ++j) {
        const int s = j % NS;
        const uint32_t vaddr = smem_u32(sm.kv[s][1]);
        mbar_wait_sleep(&sm.p_full[t], j & 1);
        fence_after();
#pragma unroll
        for (int kk = 0; kk < KT / 16; ++kk)  // a new accumulation group restarts O
          umma_ts_f16(od, sd + kk * 8, sdesc(vaddr + kk * 512, 256, 128), ID_O,
                      (j % DRAIN != 0 || kk > 0));
        if (j + 1 < T) issue_s(j + 1);  // in order after the PV that reads P
        umma_commit(&sm.kv_empty[s]);
      }
      umma_commit(&sm.o_done[t]);
    }
    __syncwarp();
  } else {
    // softmax: thread = query row.  64 S columns in 4 chunks of 16, the next chunk's
    // tcgen05.ld in flight while this chunk's exponentials issue; chunk c's P (8 packed
    // columns) lands on columns [8c, 8c + 8), all inside chunks already consumed.
    const int t = warp >> 2;
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t base = tbase + lane_off + t * S_COLS;
    const uint32_t obase = tbase + lane_off + O_COL + t * 16;
    float4* osum = &sm.osum[t][0][row];
#pragma unroll
    for (int c = 0; c < 4; ++c) osum[c * QT] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto drain = [&]() {  // O of the group just finished -> float sum in smem
      uint32_t r[16];
      PTX_LD16(obase, r);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float4 a = osum[c * QT];
        const float2 lo = add_f32x2(make_float2(a.x, a.y),
                                    make_float2(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1])));
        const float2 hi = add_f32x2(make_float2(a.z, a.w),
                                    make_float2(__uint_as_float(r[4 * c + 2]), __uint_as_float(r[4 * c + 3])));
        osum[c * QT] = make_float4(lo.x, lo.y, hi.x, hi.y);
      }
    };
    uint32_t ra[16], rb[16], pk[8];
    auto tile = [&](int j, bool drain_first) {
      mbar_wait_sleep(&sm.s_full[t], j & 1);
      fence_after();
      if (drain_first) drain();  // O = tiles [j - DRAIN, j), stable once s_full(j) fired
      PTX_LD16_AT(base, 0, ra);
      tmem_wait_ld();
      PTX_LD16_AT(base, 16, rb);
      softmax16(ra, pk);
      PTX_ST8_AT(base, 0, pk);
      tmem_wait_ld();
      PTX_LD16_AT(base, 32, ra);
      softmax16(rb, pk);
      PTX_ST8_AT(base, 8, pk);
      tmem_wait_ld();
      PTX_LD16_AT(base, 48, rb);
      softmax16(ra, pk);
      PTX_ST8_AT(base, 16, pk);
      tmem_wait_ld();
      softmax16(rb, pk);
      PTX_ST8_AT(base, 24, pk);
      tmem_wait_st();
      fence_before();
      mbar_arrive(&sm.p_full[t]);
    };
    for (int g0 = 0; g0 < T; g0 += DRAIN) {  // groups of DRAIN key tiles
      const int g1 = min(g0 + DRAIN, T);
      for (int j = g0; j < g1; ++j) tile(j, j == g0 && g0 > 0);
    }
    mbar_wait_sleep(&sm.o_done[t], 0);
    fence_after();
    if (T > 0) drain();
    const int lr = w.q0 + t * QT + row;
    if (lr < w.n) {
      float v[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 a = osum[c * QT];
        v[4 * c] = a.x;
        v[4 * c + 1] = a.y;
        v[4 * c + 2] = a.z;
        v[4 * c + 3] = a.w;
      }
      const float inv = 1.f / v[15];
      float* o = out + (w.row0 + lr) * ldo + head * d_head;
      for (int d = 0; d < d_head; ++d) o[d] = v[d] * inv;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == MMA_WARP0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                 "r"(TMEM_COLS));
  }
}

// K and V^T tiles in fp16: K[:,15] = V[:,15] = 1 on valid keys, zero rows past the end;
// max |k| (of the rounded values) per (forward, head); flags |k|, |v| out of fp16 range.
// One CTA per 64-key tile for every head: warps read whole K|V row slices (lanes along
// the columns: coalesced), the tile is assembled in shared memory and written back as
// 16-B vectors in both UMMA layouts, and one atomic per head carries the tile's max |k|
// (grid.y covers the heads four at a time).
// (Round 1's thread-per-(8 keys, 8 dims) mapping read 32-B pieces of 128 rows per warp
// instruction: ~1 TB/s.)
constexpr int RP_THREADS = 128;
constexpr int RP_MAXH = 4;
__global__ void __launch_bounds__(RP_THREADS)
    repack_kv16_kernel(const float* __restrict__ k, const float* __restrict__ v, int64_t ld,
                       int n_head, int d_head, const int64_t* __restrict__ tile_fwd_row0,
                       const int32_t* __restrict__ tile_n, int64_t Ttot,
                       __half* __restrict__ kb, __half* __restrict__ vb,
                       unsigned* __restrict__ kmax, int32_t* __restrict__ flag) {
  __shared__ __align__(16) __half Ks[RP_MAXH][KT][16];
  __shared__ __align__(16) __half Vs[RP_MAXH][KT][16];
  __shared__ unsigned hmax[RP_MAXH];
  const int64_t tile = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = tile_n[3 * tile], fwd = tile_n[3 * tile + 2];
  const int lt0 = tile_n[3 * tile + 1] * KT;  // first row of the tile within its forward
  const int64_t grow0 = tile_fwd_row0[tile] + lt0;
  const int h0 = blockIdx.y * RP_MAXH;                 // heads [h0, h0 + hc) in this CTA
  const int hc = min(RP_MAXH, n_head - h0);
  const int W = hc * d_head;
  if (tid < RP_MAXH) hmax[tid] = 0u;
  bool big = false;
  // ---- rows: warp per key, lane per column c of [K (W columns) | V (W columns)]
  {
    int cd[4], ch[4];
    bool cv[4], cisv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // 2W <= 128 columns
      const int c = lane + 32 * j;
      cv[j] = c < 2 * W;
      cisv[j] = c >= W;
      const int cc = cisv[j] ? c - W : c;
      ch[j] = cc / d_head;
      cd[j] = cc - ch[j] * d_head;
    }
    // all of this warp's loads first (16 rows x 4 columns per lane in flight), then the
    // fp16 conversion and the shared-memory stores
    constexpr int RPW = KT / (RP_THREADS / 32);  // rows per warp
    float xs[RPW][4];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int key = warp + r * (RP_THREADS / 32);
      const bool valid = lt0 + key < n;
      const int64_t ro = (grow0 + key) * ld;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float x = 0.f;
        if (valid && cv[j]) {
          const int64_t o = ro + (int64_t)(h0 + ch[j]) * d_head + cd[j];
          x = cisv[j] ? v[o] : k[o];
        }
        xs[r][j] = x;
      }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int key = warp + r * (RP_THREADS / 32);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!cv[j]) continue;
        big |= !(fabsf(xs[r][j]) <= RANGE_LIMIT);
        (cisv[j] ? Vs : Ks)[ch[j]][key][cd[j]] = __float2half_rn(xs[r][j]);
      }
    }
  }
  // ---- padding dims: d_head..14 zero, 15 = 1 on valid keys (offset / row-sum column)
  for (int i = tid; i < hc * KT; i += RP_THREADS) {
    const int h = i / KT, key = i - h * KT;
    for (int d = d_head; d < 16; ++d) {
      const __half x = __float2half_rn((d == 15 && lt0 + key < n) ? 1.f : 0.f);
      Ks[h][key][d] = x;
      Vs[h][key][d] = x;
    }
  }
  __syncthreads();
  // ---- K row form: element (key, d) at (d>>3)*(KT*8) + key*8 + (d&7); max |k| per head
  for (int i = tid; i < hc * KT * 2; i += RP_THREADS) {
    const int dh = i & 1, hk = i >> 1, h = hk / KT, key = hk - h * KT;
    const uint4 w = *reinterpret_cast<const uint4*>(&Ks[h][key][8 * dh]);
    __half* kt = kb + ((int64_t)(h0 + h) * Ttot + tile) * (KT * 16);
    *reinterpret_cast<uint4*>(kt + dh * (KT * 8) + key * 8) = w;
    if (dh == 0 && lt0 + key < n) {
      // |k|^2 as the two 8-dim halves summed separately, then added (the round-1 order)
      float n0 = 0.f, n1 = 0.f;
      for (int d = 0; d < d_head && d < 8; ++d) {
        const float kk = __half2float(Ks[h][key][d]);
        n0 = fmaf(kk, kk, n0);
      }
      for (int d = 8; d < d_head; ++d) {
        const float kk = __half2float(Ks[h][key][d]);
        n1 = fmaf(kk, kk, n1);
      }
      atomicMax(&hmax[h], __float_as_uint(sqrtf(n0 + n1)));
    }
  }
  // ---- V^T: element (key, d) at (key>>3)*128 + (d>>3)*64 + (d&7)*8 + (key&7)
  for (int i = tid; i < hc * (KT / 8) * 16; i += RP_THREADS) {
    const int d = i & 15, hg = i >> 4, h = hg / (KT / 8), g = hg - h * (KT / 8);
    __align__(16) __half col[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) col[e] = Vs[h][8 * g + e][d];
    __half* vt = vb + ((int64_t)(h0 + h) * Ttot + tile) * (KT * 16);
    *reinterpret_cast<uint4*>(vt + g * 128 + (d >> 3) * 64 + (d & 7) * 8) =
        *reinterpret_cast<const uint4*>(col);
  }
  __syncthreads();
  if (tid < hc && lt0 < n) atomicMax(&kmax[fwd * n_head + h0 + tid], hmax[tid]);
  if (big) atomicOr(flag, 2);
}

// Q in fp16, scaled by log2(e)/sqrt(d_head); column 15 = 15 - b_i, or NaN when b_i >
// F16_LIMIT (the fp16 kernel hands that row's work item to the tf32 kernel).  Flag bits:
// 1 = some bound > BOUND_LIMIT (online kernel for the launch), 2 = |q| outside the fp16
// range (tf32 kernel for the launch).
__global__ void repack_q16_kernel(const float* __restrict__ q, int64_t ld, int n_head, int d_head,
                                  int64_t R, const int32_t* __restrict__ row_fwd,
                                  const unsigned* __restrict__ kmax, float qscale,
                                  __half* __restrict__ qh, int32_t* __restrict__ flag) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= R * n_head) return;
  const int64_t r = idx / n_head;
  const int head = (int)(idx % n_head);
  __align__(16) __half qv[16];
  float nq = 0.f;
  bool big = false;
  for (int d = 0; d < 16; ++d) {
    float x = 0.f;
    if (d < d_head) {
      x = q[r * ld + head * d_head + d] * qscale;
      big |= !(fabsf(x) <= RANGE_LIMIT);
    }
    qv[d] = __float2half_rn(x);
    x = __half2float(qv[d]);
    nq = fmaf(x, x, nq);
  }
  const float km = __uint_as_float(kmax[row_fwd[r] * n_head + head]);
  const float bnd = sqrtf(nq) * km * (1.f + 1.f / 256.f) + 1.f / 256.f;
  if (!(bnd <= BOUND_LIMIT)) atomicOr(flag, 1);
  else if (big) atomicOr(flag, 2);
  qv[15] = bnd > F16_LIMIT ? __ushort_as_half((unsigned short)0x7E00u) : __float2half_rn(15.f - bnd);
  uint4* o = reinterpret_cast<uint4*>(qh + ((int64_t)head * R + r) * 16);
  o[0] = reinterpret_cast<const uint4*>(qv)[0];
  o[1] = reinterpret_cast<const uint4*>(qv)[1];
}

}  // namespace t16

void attention_f16_tc(const float* q, const float* k, const float* v, int64_t ld, int n_head,
                      int d_head, int64_t R, int64_t Ttot, const TcWork* works_dev,
                      int64_t num_works, const int64_t* tile_row0_dev, const int32_t* tile_n_dev,
                      void* qh, void* kb, void* vb, float* out, int64_t ldo,
                      const int32_t* row_fwd, unsigned* kmax, int32_t* flag, int32_t* wflag,
                      float qscale, cudaStream_t st) {
  static bool attr = false;
  const size_t smem = sizeof(t16::Smem) + 1024;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(t16::attn_f16_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  GO_CHECK(d_head <= 15, "repack_kv16 needs d_head <= 15");
  const dim3 rgrid((unsigned)Ttot, (unsigned)cdiv(n_head, t16::RP_MAXH));
  t16::repack_kv16_kernel<<<rgrid, t16::RP_THREADS, 0, st>>>(
      k, v, ld, n_head, d_head, tile_row0_dev, tile_n_dev, Ttot, static_cast<__half*>(kb),
      static_cast<__half*>(vb), kmax, flag);
  LAUNCH_CHECK();
  t16::repack_q16_kernel<<<(unsigned)cdiv(R * n_head, 256), 256, 0, st>>>(
      q, ld, n_head, d_head, R, row_fwd, kmax, qscale, static_cast<__half*>(qh), flag);
  LAUNCH_CHECK();
  dim3 grid((unsigned)num_works, (unsigned)n_head);
  t16::attn_f16_kernel<<<grid, t16::NUM_THREADS, smem, st>>>(
      static_cast<const uint16_t*>(qh), static_cast<const uint16_t*>(kb),
      static_cast<const uint16_t*>(vb), R, Ttot, works_dev, out, ldo, d_head, flag, wflag);
  LAUNCH_CHECK();
}

}  // namespace go
