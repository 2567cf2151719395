// The PPO tape's task-head attention on the 5th-generation tensor cores (policy.py:196-203,
// multi_head_attention(h, h) over all N rows, and its reverse; tensor.py:382-388).
//
// The training step needs fp32-class attention (Adam's first steps are ~lr*sign(g), so the
// gradient noise of single-fp16 products moved 5% of the reference's coordinates; see
// attn_bwd_mma.cu), so every fp16 operand is a 2-term split x = hi + lo and each product
// takes three kind::f16 MMAs (hi.hi + hi.lo + lo.hi, ~2^-21 relative).  Operands are
// packed once per call into 64-row tiles per (head, forward) in the two UMMA K-major
// canonical layouts the products need (tape_pack_kernel):
//   row form   (64 rows x 16 dims, dims contiguous)   B operand of S = Q K^T, G = dO V^T
//   transposed (16 dims x 64 rows, rows contiguous)   B operand of O += P V
// Forward (tape_fwd_kernel): the inference kernel's fixed-offset structure
// (tc_attention16.cu) with split S, MUFU exponentials (no polynomial), P split into hi and lo
// TMEM regions, split PV, the accumulator drained every 16 key tiles, and the log2-sum-exp
// lse = log2(row sum) + b - 15 the backward recomputes P from.  Rows whose bound exceeds
// F16_LIMIT flag the call; the caller then runs the mma.sync forward instead.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cuda_fp16.h>

#include "engine.cuh"
#include "tcgen05.cuh"
#include "train.cuh"

namespace go {
namespace tt {

using namespace ptx;

constexpr int KT = 64;     // rows per packed tile (keys per step)
constexpr int QT = 128;    // queries per M tile
constexpr int NQT = 3;     // M tiles per CTA
constexpr int NS = 6;      // K/V ring stages
constexpr int DRAIN = 16;  // key tiles per TMEM accumulation group
constexpr int TILE_HALVES = KT * 16;
constexpr int TILE_BYTES = TILE_HALVES * 2;
constexpr int PRODUCER_WARP = NQT * 4;
constexpr int MMA_WARP0 = NQT * 4 + 1;
constexpr int NUM_THREADS = (NQT * 5 + 1) * 32;
constexpr uint32_t TCOLS_PER_TILE = 144;  // S 64 | P_hi 32 | P_lo 32 | O 16
constexpr uint32_t TMEM_COLS = 512;
constexpr float F16_LIMIT = 14.f;
constexpr float RANGE = 60000.f;

// ---------------------------------------------------------------------------------------
// packing: per (head, 64-row tile) row form and / or transposed form, hi and lo halves.
// col15: 0 -> zero, 1 -> one on valid rows (K's offset column, V's row-sum column),
// 2 -> c15[row * n_head + head] (Q's 15 - bound).  kmax (optional): max row norm of the
// scaled values per (forward, head).  Thread = (head, tile, 8-row group, 8-dim half).
__global__ void tape_pack_kernel(const float* __restrict__ x, int64_t ld, int n_head, int d_head,
                                 float scale, const int64_t* __restrict__ tile_row0,
                                 const int32_t* __restrict__ tile_n, int64_t Ttot, int col15,
                                 const float* __restrict__ c15, __half* __restrict__ row_hi,
                                 __half* __restrict__ row_lo, __half* __restrict__ t_hi,
                                 __half* __restrict__ t_lo, unsigned* __restrict__ kmax,
                                 int32_t* __restrict__ flag) {
  constexpr int G = KT / 8;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)n_head * Ttot * G * 2;
  const bool live = idx < total;
  const int64_t id = live ? idx : total - 1;
  const int dh = (int)(id & 1);
  const int64_t gi = id >> 1;
  const int head = (int)(gi / (Ttot * G));
  const int64_t rem = gi % (Ttot * G);
  const int64_t tile = rem / G;
  const int g = (int)(rem % G);
  const int n = tile_n[3 * tile], fwd = tile_n[3 * tile + 2];
  const int local0 = tile_n[3 * tile + 1] * KT + g * 8;
  const int64_t grow0 = tile_row0[tile] + local0;
  const int64_t toff = ((int64_t)head * Ttot + tile) * TILE_HALVES;
  __align__(16) __half th[8][8], tl[8][8];  // transposed: [d - 8 dh][row]
  float nmax = 0.f;
  bool big = false;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const bool valid = local0 + e < n;
    __align__(16) __half rh[8], rl[8];
    float nr = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int d = dh * 8 + i;
      float v = 0.f;
      if (valid) {
        if (d < d_head) {
          v = x[(grow0 + e) * ld + head * d_head + d] * scale;
          big |= !(fabsf(v) <= RANGE);
          nr = fmaf(v, v, nr);
        } else if (d == 15) {
          v = col15 == 1 ? 1.f : col15 == 2 ? c15[(grow0 + e) * n_head + head] : 0.f;
        }
      }
      const __half h = __float2half_rn(v);
      const __half l = __float2half_rn(v - __half2float(h));
      rh[i] = h;
      rl[i] = l;
      th[i][e] = h;
      tl[i][e] = l;
    }
    nr += __shfl_xor_sync(0xffffffffu, nr, 1);
    nmax = fmaxf(nmax, nr);
    if (live && row_hi) {
      const int64_t o = toff + dh * (KT * 8) + g * 64 + e * 8;
      *reinterpret_cast<uint4*>(row_hi + o) = *reinterpret_cast<const uint4*>(rh);
      *reinterpret_cast<uint4*>(row_lo + o) = *reinterpret_cast<const uint4*>(rl);
    }
  }
  if (!live) return;
  if (t_hi) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t o = toff + g * 128 + dh * 64 + i * 8;
      *reinterpret_cast<uint4*>(t_hi + o) = *reinterpret_cast<const uint4*>(th[i]);
      *reinterpret_cast<uint4*>(t_lo + o) = *reinterpret_cast<const uint4*>(tl[i]);
    }
  }
  if (kmax && dh == 0 && local0 < n)
    atomicMax(&kmax[fwd * n_head + head], __float_as_uint(sqrtf(nmax)));
  if (big) atomicOr(flag, 1);
}

// per (row, head): b = |q| max|k| (1 + 2^-8) + 2^-8 >= every scaled score, and the Q offset
// column value 15 - b; flags bounds beyond the fp16 limit
__global__ void tape_bound_kernel(const float* __restrict__ q, int64_t ld, int n_head, int d_head,
                                  float qscale, int64_t R, const int32_t* __restrict__ row_fwd,
                                  const unsigned* __restrict__ kmax, float* __restrict__ bound,
                                  float* __restrict__ c15, int32_t* __restrict__ flag) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= R * n_head) return;
  const int64_t r = idx / n_head;
  const int head = (int)(idx % n_head);
  float nq = 0.f;
  for (int d = 0; d < d_head; ++d) {
    const float v = q[r * ld + head * d_head + d] * qscale;
    nq = fmaf(v, v, nq);
  }
  const float km = __uint_as_float(kmax[row_fwd[r] * n_head + head]);
  const float b = sqrtf(nq) * km * (1.f + 1.f / 256.f) + 1.f / 256.f;
  if (!(b <= F16_LIMIT)) atomicOr(flag, 2);
  bound[idx] = b;
  c15[idx] = 15.f - b;
}

// ---------------------------------------------------------------------------------------
// forward with log2-sum-exp
struct FwdSmem {
  uint16_t q[NQT][2][QT * 16];     // [tile][hi, lo] A operand, M = 128 K-major canonical
  uint16_t kv[NS][4][TILE_HALVES];  // K_hi, K_lo (row form), V^T_hi, V^T_lo (transposed)
  float4 osum[NQT][4][QT];
  uint64_t kv_full[NS], kv_empty[NS];
  uint64_t s_full[NQT], p_full[NQT], o_done[NQT];
  uint32_t tmem_base;
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
__device__ __forceinline__ float2 add_f32x2(float2 a, float2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
  return *reinterpret_cast<const float2*>(&r);
}
// packed fp32 pair arithmetic (FADD2 / FMUL2: one issue slot for two lanes' worth)
__device__ __forceinline__ float2 sub_f32x2(float2 a, float2 b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
  return *reinterpret_cast<const float2*>(&r);
}
__device__ __forceinline__ float2 mul_f32x2(float2 a, float2 b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
  return *reinterpret_cast<const float2*>(&r);
}
// a pair of fp32 values -> fp16x2 hi and lo words (x = hi + lo), the residual in FADD2
__device__ __forceinline__ void split2(float2 x, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x.x, x.y);
  const float2 r = sub_f32x2(x, __half22float2(h));
  const __half2 l = __floats2half2_rn(r.x, r.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
// 16 fp32 values -> 8 packed fp16x2 hi words and 8 lo words (x = hi + lo)
__device__ __forceinline__ void split16(const float* v, uint32_t* hi, uint32_t* lo) {
#pragma unroll
  for (int i = 0; i < 8; ++i) split2(make_float2(v[2 * i], v[2 * i + 1]), hi[i], lo[i]);
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    tape_fwd_kernel(const __half* __restrict__ q_hi, const __half* __restrict__ q_lo,
                    const __half* __restrict__ k_hi, const __half* __restrict__ k_lo,
                    const __half* __restrict__ vt_hi, const __half* __restrict__ vt_lo,
                    int64_t Ttot, const TcWork* __restrict__ works,
                    const float* __restrict__ bound, int n_head, float* __restrict__ out,
                    int64_t ldo, int d_head, float* __restrict__ lse,
                    const int32_t* __restrict__ flag) {
  if (*flag) return;  // the caller runs the mma.sync forward
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TcWork w = works[blockIdx.x];
  const int head = blockIdx.y;
  const int T = w.tiles;
  const int64_t hbase = ((int64_t)head * Ttot + w.tile0) * TILE_HALVES;
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
  // Q: query tile qt = packed tiles 2 i, 2 i + 1 of this forward; row-form d-chunk dh of
  // packed tile u lands at dh * (QT * 8) + u * (KT * 8) halves (M = 128 K-major layout)
  for (int i = threadIdx.x; i < NQT * 2 * 2 * 2 * (KT * 8 / 8); i += NUM_THREADS) {
    // i -> (qt, part hi/lo, u, dh, 16-byte word within the 1 KB block)
    const int wd = i % (KT * 8 / 8);
    const int dh = (i / 64) & 1, u = (i / 128) & 1, part = (i / 256) & 1, qt = i / 512;
    const int tl = (w.q0 + qt * QT) / KT + u;  // local tile of the forward
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (tl < T) {
      const __half* src = (part ? q_lo : q_hi) + hbase + (int64_t)tl * TILE_HALVES +
                          dh * (KT * 8) + wd * 8;
      v = *reinterpret_cast<const uint4*>(src);
    }
    *reinterpret_cast<uint4*>(&sm.q[qt][part][dh * (QT * 8) + u * (KT * 8) + wd * 8]) = v;
  }
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp == PRODUCER_WARP) {
    if (lane == 0) {
      const __half* srcs[4] = {k_hi, k_lo, vt_hi, vt_lo};
      for (int j = 0; j < T; ++j) {
        const int s = j % NS;
        if (j >= NS) mbar_wait_sleep(&sm.kv_empty[s], ((j / NS) - 1) & 1);
        mbar_expect_tx(&sm.kv_full[s], 4 * TILE_BYTES);
#pragma unroll
        for (int a = 0; a < 4; ++a)
          bulk_g2s(sm.kv[s][a], srcs[a] + hbase + (int64_t)j * TILE_HALVES, TILE_BYTES,
                   &sm.kv_full[s]);
      }
    }
    __syncwarp();
  } else if (warp >= MMA_WARP0) {
    if (lane == 0) {
      const int t = warp - MMA_WARP0;
      constexpr uint32_t ID_S = idesc_f16(QT, KT);
      constexpr uint32_t ID_O = idesc_f16(QT, 16);
      const uint64_t qh = sdesc(smem_u32(sm.q[t][0]), QT * 16, 128);
      const uint64_t ql = sdesc(smem_u32(sm.q[t][1]), QT * 16, 128);
      const uint32_t sc = tbase + t * TCOLS_PER_TILE;
      const uint32_t ph = sc + 64, pl = sc + 96, oc = sc + 128;
      auto issue_s = [&](int j) {
        const int s = j % NS;
        mbar_wait_sleep(&sm.kv_full[s], (j / NS) & 1);
        fence_after();
        const uint64_t kh = sdesc(smem_u32(sm.kv[s][0]), KT * 16, 128);
        const uint64_t kl = sdesc(smem_u32(sm.kv[s][1]), KT * 16, 128);
        umma_ss_f16(sc, qh, kh, ID_S, 0);
        umma_ss_f16(sc, qh, kl, ID_S, 1);
        umma_ss_f16(sc, ql, kh, ID_S, 1);
        umma_commit(&sm.s_full[t]);
      };
      if (T > 0) issue_s(0);
      for (int j = 0; j < T; ++j) {
        const int s = j % NS;
        const uint32_t vh = smem_u32(sm.kv[s][2]), vl = smem_u32(sm.kv[s][3]);
        mbar_wait_sleep(&sm.p_full[t], j & 1);
        fence_after();
#pragma unroll
        for (int kk = 0; kk < KT / 16; ++kk) {
          const uint64_t bh = sdesc(vh + kk * 512, 256, 128), bl = sdesc(vl + kk * 512, 256, 128);
          umma_ts_f16(oc, ph + kk * 8, bh, ID_O, (j % DRAIN != 0 || kk > 0));
          umma_ts_f16(oc, ph + kk * 8, bl, ID_O, 1);
          umma_ts_f16(oc, pl + kk * 8, bh, ID_O, 1);
        }
        if (j + 1 < T) issue_s(j + 1);  // in order after the PV that reads P
        umma_commit(&sm.kv_empty[s]);
      }
      umma_commit(&sm.o_done[t]);
    }
    __syncwarp();
  } else {
    const int t = warp >> 2;
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t sbase = tbase + lane_off + t * TCOLS_PER_TILE;
    const uint32_t pbase_h = sbase + 64, pbase_l = sbase + 96, obase = sbase + 128;
    float4* osum = &sm.osum[t][0][row];
#pragma unroll
    for (int c = 0; c < 4; ++c) osum[c * QT] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto drain = [&]() {
      uint32_t r[16];
      PTX_LD16(obase, r);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 a = osum[c * QT];
        const float2 lo = add_f32x2(make_float2(a.x, a.y), make_float2(__uint_as_float(r[4 * c]),
                                                                      __uint_as_float(r[4 * c + 1])));
        const float2 hi = add_f32x2(make_float2(a.z, a.w), make_float2(__uint_as_float(r[4 * c + 2]),
                                                                      __uint_as_float(r[4 * c + 3])));
        osum[c * QT] = make_float4(lo.x, lo.y, hi.x, hi.y);
      }
    };
    for (int j = 0; j < T; ++j) {
      mbar_wait_sleep(&sm.s_full[t], j & 1);
      fence_after();
      if (j > 0 && j % DRAIN == 0) drain();  // O = tiles [j - DRAIN, j), stable here
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[16], hi[8], lo[8];
        float p[16];
        PTX_LD16(sbase + 16 * c, r);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) p[i] = ex2f(__uint_as_float(r[i]));  // S' <= 15
        split16(p, hi, lo);
        PTX_ST8(pbase_h + 8 * c, hi);
        PTX_ST8(pbase_l + 8 * c, lo);
      }
      tmem_wait_st();
      fence_before();
      mbar_arrive(&sm.p_full[t]);
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
      const int64_t gr = w.row0 + lr;
      const float inv = 1.f / v[15];
      float* o = out + gr * ldo + head * d_head;
      for (int d = 0; d < d_head; ++d) o[d] = v[d] * inv;
      // v[15] = sum 2^(s - b + 15): log2 sum 2^s = log2 v[15] + b - 15
      lse[gr * n_head + head] = log2f(v[15]) + bound[gr * n_head + head] - 15.f;
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


// ---------------------------------------------------------------------------------------
// backward.  FA2 recomputation from the forward's log2-sum-exp:
//   P = 2^(s - lse) with s = q.k log2(e)/sqrt(d); D_q = dO_q . O_q;
//   dS = P (dO.v - D); dv = sum_q P dO_q; dk = (1/log2 e) sum_q dS q_s; dq = scale sum_k dS k
// dO enters scaled by gs (a power of two bringing max|dO| into [0.5, 1)), P by 2^15 and dS
// by dsc (a power of two bringing its bound 2 max|dO_q| max|v_k| to 2^14) before the fp16
// splits, so small values keep fp16-normal hi / lo terms (attn_bwd_mma.cu, same scales).
constexpr int BNS = 4;  // backward ring stages
constexpr float PSCALE = 32768.f;

struct BwdScales {
  unsigned bits[3];  // max|dO|, max |v| row norm, max |dO gs| row norm (float bit patterns)
};
__device__ __forceinline__ float grad_scale_t(const unsigned* b) {
  const float m = __uint_as_float(b[0]);
  if (!(m > 0.f) || !(m <= 3.0e38f)) return 1.f;
  return exp2f(-ceilf(log2f(m)));
}
__device__ __forceinline__ float ds_scale_t(const unsigned* b) {
  const float x = 2.f * __uint_as_float(b[1]) * __uint_as_float(b[2]);
  if (!(x > 0.f) || !(x <= 3.0e38f)) return 1.f;
  return exp2f(fminf(14.f - ceilf(log2f(x)), 60.f));
}

// max|dO| over the head columns
__global__ void absmax_t_kernel(const float* __restrict__ x, int64_t ld, int64_t M, int W,
                                unsigned* __restrict__ out) {
  float m = 0.f;
  const int64_t n = M * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / W;
    const float a = fabsf(x[r * ld + (i - r * W)]);
    m = a > m || a != a ? a : m;
  }
  for (int o = 16; o; o >>= 1) {
    const float t = __shfl_xor_sync(0xffffffffu, m, o);
    m = t > m || t != t ? t : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// per (head, row): lse and D*gs head-major (the backward kernels read them by query row),
// max |v| and max |dO gs| row norms
__global__ void bwd_rows_kernel(const float* __restrict__ v, const float* __restrict__ dO,
                                int64_t ld, const float* __restrict__ lse,
                                const float* __restrict__ D, int n_head, int d_head, int64_t R,
                                unsigned* __restrict__ bits, float* __restrict__ lse_h,
                                float* __restrict__ d_h) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= R * n_head) return;
  const int64_t r = idx / n_head;
  const int h = (int)(idx % n_head);
  const float gs = grad_scale_t(bits);
  float nv = 0.f, nd = 0.f;
  for (int d = 0; d < d_head; ++d) {
    const float a = v[r * ld + h * d_head + d], b = dO[r * ld + h * d_head + d] * gs;
    nv = fmaf(a, a, nv);
    nd = fmaf(b, b, nd);
  }
  atomicMax(bits + 1, __float_as_uint(sqrtf(nv)));
  atomicMax(bits + 2, __float_as_uint(sqrtf(nd)));
  lse_h[(int64_t)h * R + r] = lse[idx];
  d_h[(int64_t)h * R + r] = D[idx] * gs;
}

// dO scaled by gs (the pack kernel takes a scale argument; gs is only known on the device)
__global__ void scale_rows_kernel(const float* __restrict__ x, int64_t ld, int64_t R, int W,
                                  const unsigned* __restrict__ bits, float* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= R * W) return;
  const int64_t r = i / W;
  y[i] = x[r * ld + (i - r * W)] * grad_scale_t(bits);
}

// lse and D * gs per (head, 64-row tile): the dk / dv kernel's producer copies a chunk's
// 64 + 64 values with its operand tiles (512 B, aligned)
__global__ void tile_lsd_kernel(const float* __restrict__ lse, const float* __restrict__ D,
                                int n_head, const int64_t* __restrict__ tile_row0,
                                const int32_t* __restrict__ tile_n, int64_t Ttot,
                                const unsigned* __restrict__ bits, float* __restrict__ lsd) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n_head * Ttot * KT) return;
  const int j = (int)(idx % KT);
  const int64_t ht = idx / KT;
  const int head = (int)(ht / Ttot);
  const int64_t t = ht % Ttot;
  const int n = tile_n[3 * t], local = tile_n[3 * t + 1] * KT + j;
  const int64_t row = tile_row0[t] + local;
  const bool ok = local < n;
  float* o = lsd + ht * 2 * KT;
  // lse - 15: 2^(s - lse + 15) = 2^15 P comes straight from the MUFU; padded queries get
  // +inf so their P is exactly 0 without a per-element mask
  o[j] = ok ? lse[row * n_head + head] - 15.f : __int_as_float(0x7f800000);
  o[KT + j] = ok ? D[row * n_head + head] * grad_scale_t(bits) : 0.f;
}

// dk, dv: key-major.  CTA = one head x 128 keys (two packed tiles) of one forward, 1 CTA per
// SM.  TMEM: S^T and G^T double-buffered (2 x (64 + 64)) | P^T hi, lo | dS^T hi, lo
// (32 each) | dv 16 | dk 16.  Warps 0-15: four per TMEM lane quarter, each owning 16 of a
// chunk's 64 query columns; warp 16: producer (bulk copies of the 64-query chunk: Q and dO
// row form, Q^T and dO^T, the chunk's lse / D); warp 17: MMA issue.  Per chunk c:
// S^T = K Q^T and G^T = V dO^T into buffer c & 1 (3 split MMAs each, issued two chunks
// ahead), the softmax warps write P^T = 2^15 2^(s - lse) and dS^T = dsc P (g - D) as hi /
// lo fp16 into TMEM once the previous chunk's products have read them (pv_done), then
// dv += P^T dO and dk += dS^T Q (12 MMAs each).  dv / dk are drained every DRAIN chunks into
// fp32 sums in shared memory.
constexpr int KV_SOFT = 16;
constexpr int KV_PRODUCER = KV_SOFT;
constexpr int KV_MMA = KV_SOFT + 1;
constexpr int KV_THREADS = (KV_SOFT + 2) * 32;
constexpr uint32_t C_SG = 0;  // buffer b: S^T at 128 b, G^T at 128 b + 64
constexpr uint32_t C_PH = 256, C_PL = 288, C_DH = 320, C_DL = 352, C_DV = 384, C_DK = 400;

struct KvSmem {
  uint16_t k[2][QT * 16];  // A operands (M = 128 keys): K hi / lo
  uint16_t v[2][QT * 16];  // V hi / lo
  uint16_t ch[BNS][8][TILE_HALVES];  // Q hi, lo, dO hi, lo (row form); Q^T hi, lo, dO^T hi, lo
  float lsd[BNS][2 * KT];            // the chunk's lse, D * gs
  float4 acc[2][4][QT];  // [dv, dk][column / 4][key] drained sums
  uint64_t full[BNS], empty[BNS];
  uint64_t s_full[2], p_full, pv_done, done;
  uint32_t tmem_base;
};

__device__ __forceinline__ void load_a128(uint16_t* dst, const __half* tiles, int T, int tl0,
                                          int tid, int nthreads) {
  // two consecutive row-form tiles -> M = 128 K-major layout
  for (int i = tid; i < 2 * 2 * 64; i += nthreads) {
    const int wd = i % 64, dh = (i / 64) & 1, u = i / 128;
    const int tl = tl0 + u;
    uint4 val = make_uint4(0u, 0u, 0u, 0u);
    if (tl < T)
      val = *reinterpret_cast<const uint4*>(tiles + (int64_t)tl * TILE_HALVES + dh * (KT * 8) +
                                            wd * 8);
    *reinterpret_cast<uint4*>(dst + dh * (QT * 8) + u * (KT * 8) + wd * 8) = val;
  }
}

__global__ void __launch_bounds__(KV_THREADS, 1)
    tape_dkv_kernel(const __half* __restrict__ kr_hi, const __half* __restrict__ kr_lo,
                    const __half* __restrict__ vr_hi, const __half* __restrict__ vr_lo,
                    const __half* __restrict__ qr_hi, const __half* __restrict__ qr_lo,
                    const __half* __restrict__ qt_hi, const __half* __restrict__ qt_lo,
                    const __half* __restrict__ or_hi, const __half* __restrict__ or_lo,
                    const __half* __restrict__ ot_hi, const __half* __restrict__ ot_lo,
                    int64_t Ttot, const TcWork* __restrict__ works,
                    const float* __restrict__ lsd_t, const unsigned* __restrict__ bits,
                    int d_head, float* __restrict__ dk, float* __restrict__ dv, int64_t ld,
                    float kscale, const int32_t* __restrict__ flag) {
  if (*flag) return;  // an operand left the fp16 range: the gated mma.sync path runs
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  KvSmem& sm = *reinterpret_cast<KvSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TcWork w = works[blockIdx.x];
  const int head = blockIdx.y;
  const int T = w.tiles;
  const int64_t hb = ((int64_t)head * Ttot + w.tile0) * TILE_HALVES;
  const float* lsd_h = lsd_t + ((int64_t)head * Ttot + w.tile0) * 2 * KT;
  const int nchunks = T;  // 64-query chunks of the forward
  if (warp == KV_PRODUCER && lane == 0) {
    for (int s = 0; s < BNS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.s_full[0], 1);
    mbar_init(&sm.s_full[1], 1);
    mbar_init(&sm.p_full, KV_SOFT * 32);
    mbar_init(&sm.pv_done, 1);
    mbar_init(&sm.done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == KV_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const int tl0 = w.q0 / KT;  // the key tile pair of this CTA
  load_a128(sm.k[0], kr_hi + hb, T, tl0, threadIdx.x, KV_THREADS);
  load_a128(sm.k[1], kr_lo + hb, T, tl0, threadIdx.x, KV_THREADS);
  load_a128(sm.v[0], vr_hi + hb, T, tl0, threadIdx.x, KV_THREADS);
  load_a128(sm.v[1], vr_lo + hb, T, tl0, threadIdx.x, KV_THREADS);
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp == KV_PRODUCER) {
    if (lane == 0) {
      const __half* srcs[8] = {qr_hi, qr_lo, or_hi, or_lo, qt_hi, qt_lo, ot_hi, ot_lo};
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % BNS;
        if (c >= BNS) mbar_wait_sleep(&sm.empty[s], ((c / BNS) - 1) & 1);
        mbar_expect_tx(&sm.full[s], 8 * TILE_BYTES + 2 * KT * 4);
#pragma unroll
        for (int a = 0; a < 8; ++a)
          bulk_g2s(sm.ch[s][a], srcs[a] + hb + (int64_t)c * TILE_HALVES, TILE_BYTES,
                   &sm.full[s]);
        bulk_g2s(sm.lsd[s], lsd_h + (int64_t)c * 2 * KT, 2 * KT * 4, &sm.full[s]);
      }
    }
    __syncwarp();
  } else if (warp == KV_MMA) {
    if (lane == 0) {
      constexpr uint32_t ID_S = idesc_f16(QT, KT);
      constexpr uint32_t ID_O = idesc_f16(QT, 16);
      const uint64_t kh = sdesc(smem_u32(sm.k[0]), QT * 16, 128);
      const uint64_t kl = sdesc(smem_u32(sm.k[1]), QT * 16, 128);
      const uint64_t vh = sdesc(smem_u32(sm.v[0]), QT * 16, 128);
      const uint64_t vl = sdesc(smem_u32(sm.v[1]), QT * 16, 128);
      auto issue_sg = [&](int c) {
        const int s = c % BNS;
        mbar_wait_sleep(&sm.full[s], (c / BNS) & 1);
        fence_after();
        const uint64_t qh = sdesc(smem_u32(sm.ch[s][0]), KT * 16, 128);
        const uint64_t ql = sdesc(smem_u32(sm.ch[s][1]), KT * 16, 128);
        const uint64_t oh = sdesc(smem_u32(sm.ch[s][2]), KT * 16, 128);
        const uint64_t ol = sdesc(smem_u32(sm.ch[s][3]), KT * 16, 128);
        const uint32_t sc = tbase + C_SG + (c & 1) * 128, gc = sc + 64;
        umma_ss_f16(sc, kh, qh, ID_S, 0);
        umma_ss_f16(sc, kh, ql, ID_S, 1);
        umma_ss_f16(sc, kl, qh, ID_S, 1);
        umma_ss_f16(gc, vh, oh, ID_S, 0);
        umma_ss_f16(gc, vh, ol, ID_S, 1);
        umma_ss_f16(gc, vl, oh, ID_S, 1);
        umma_commit(&sm.s_full[c & 1]);
      };
      for (int c = 0; c < 2 && c < nchunks; ++c) issue_sg(c);
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % BNS;
        mbar_wait_sleep(&sm.p_full, c & 1);
        fence_after();
        const uint32_t qth = smem_u32(sm.ch[s][4]), qtl = smem_u32(sm.ch[s][5]);
        const uint32_t oth = smem_u32(sm.ch[s][6]), otl = smem_u32(sm.ch[s][7]);
        const bool first = (c % DRAIN) == 0;
#pragma unroll
        for (int kk = 0; kk < KT / 16; ++kk) {
          const uint64_t b_oh = sdesc(oth + kk * 512, 256, 128), b_ol = sdesc(otl + kk * 512, 256, 128);
          const uint64_t b_qh = sdesc(qth + kk * 512, 256, 128), b_ql = sdesc(qtl + kk * 512, 256, 128);
          const uint32_t acc0 = !(first && kk == 0);
          umma_ts_f16(tbase + C_DV, tbase + C_PH + kk * 8, b_oh, ID_O, acc0);
          umma_ts_f16(tbase + C_DV, tbase + C_PH + kk * 8, b_ol, ID_O, 1);
          umma_ts_f16(tbase + C_DV, tbase + C_PL + kk * 8, b_oh, ID_O, 1);
          umma_ts_f16(tbase + C_DK, tbase + C_DH + kk * 8, b_qh, ID_O, acc0);
          umma_ts_f16(tbase + C_DK, tbase + C_DH + kk * 8, b_ql, ID_O, 1);
          umma_ts_f16(tbase + C_DK, tbase + C_DL + kk * 8, b_qh, ID_O, 1);
        }
        umma_commit(&sm.pv_done);   // P^T / dS^T free, dv / dk through chunk c
        umma_commit(&sm.empty[s]);
        if (c + 2 < nchunks) issue_sg(c + 2);  // into the S^T / G^T buffer chunk c vacated
      }
      umma_commit(&sm.done);
    }
    __syncwarp();
  } else {
    // softmax: thread = key row; the four warps of a lane quarter take 16 query columns each
    const int quarter = warp & 3, part = warp >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lo = (uint32_t)(quarter * 32) << 16;
    const float gsc = grad_scale_t(bits);
    const float dsc = ds_scale_t(bits);
    const int col = part * 16;  // query columns [col, col + 16) of every chunk
    // warps of parts 0 / 1 drain dv / dk (parts 2, 3 only compute)
    float4* acc = &sm.acc[part & 1][0][row];
    if (part < 2) {
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) acc[c4 * QT] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    auto drain = [&]() {
      uint32_t r[16];
      PTX_LD16(tbase + lo + (part ? C_DK : C_DV), r);
      tmem_wait_ld();
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const float4 a = acc[c4 * QT];
        const float2 x = add_f32x2(make_float2(a.x, a.y), make_float2(__uint_as_float(r[4 * c4]),
                                                                     __uint_as_float(r[4 * c4 + 1])));
        const float2 y = add_f32x2(make_float2(a.z, a.w), make_float2(__uint_as_float(r[4 * c4 + 2]),
                                                                     __uint_as_float(r[4 * c4 + 3])));
        acc[c4 * QT] = make_float4(x.x, x.y, y.x, y.y);
      }
    };
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % BNS;
      mbar_wait_sleep(&sm.s_full[c & 1], (c >> 1) & 1);
      fence_after();
      uint32_t rs[16], rg[16], ph[8], pl[8], dh8[8], dl8[8];
      const uint32_t sc = tbase + lo + C_SG + (c & 1) * 128;
      PTX_LD16(sc + col, rs);
      PTX_LD16(sc + 64 + col, rg);
      const float2* ls = reinterpret_cast<const float2*>(sm.lsd[s] + col);
      const float2* dd = reinterpret_cast<const float2*>(sm.lsd[s] + KT + col);
      const float2 cds = make_float2(dsc / PSCALE, dsc / PSCALE);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 x = sub_f32x2(make_float2(__uint_as_float(rs[2 * i]), __uint_as_float(rs[2 * i + 1])),
                                   ls[i]);
        const float2 p2 = make_float2(ex2f(x.x), ex2f(x.y));  // 2^15 P
        const float2 g = sub_f32x2(make_float2(__uint_as_float(rg[2 * i]), __uint_as_float(rg[2 * i + 1])),
                                   dd[i]);
        split2(p2, ph[i], pl[i]);
        split2(mul_f32x2(mul_f32x2(p2, g), cds), dh8[i], dl8[i]);
      }
      if (c > 0) {  // the previous chunk's products have read P^T / dS^T
        mbar_wait_sleep(&sm.pv_done, (c - 1) & 1);
        fence_after();
        if (part < 2 && c % DRAIN == 0) drain();  // dv / dk of chunks [c - DRAIN, c)
      }
      // packed columns: query pair (2m, 2m+1) of the chunk -> column m of the region
      PTX_ST8(tbase + lo + C_PH + col / 2, ph);
      PTX_ST8(tbase + lo + C_PL + col / 2, pl);
      PTX_ST8(tbase + lo + C_DH + col / 2, dh8);
      PTX_ST8(tbase + lo + C_DL + col / 2, dl8);
      tmem_wait_st();
      fence_before();
      mbar_arrive(&sm.p_full);
    }
    mbar_wait_sleep(&sm.done, 0);
    fence_after();
    if (part < 2) {
      if (nchunks > 0) drain();
      const int kr = w.q0 + row;  // local key row
      if (kr < w.n) {
        const float scl = part ? kscale / (gsc * dsc) : 1.f / (gsc * PSCALE);
        float* o = (part ? dk : dv) + (w.row0 + kr) * ld + head * d_head;
        float vv[16];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const float4 a = acc[c4 * QT];
          vv[4 * c4] = a.x;
          vv[4 * c4 + 1] = a.y;
          vv[4 * c4 + 2] = a.z;
          vv[4 * c4 + 3] = a.w;
        }
        for (int d = 0; d < d_head; ++d) o[d] = vv[d] * scl;
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == KV_MMA) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                 "r"(TMEM_COLS));
  }
}


// dq: query-major.  CTA = one head x 2 query tiles (256 queries) of one forward, 1 CTA per
// SM; per query tile 4 softmax warps (thread = query row), one MMA warp; one producer warp.
// TMEM per tile: S 64 | G 64 | dS hi, lo 32 + 32 | dq 16.  Per 64-key chunk: S = Q K^T and
// G = dO V^T (3 split MMAs each), dS = dsc 2^(s - lse) (g - D) as hi / lo fp16 into TMEM,
// dq += dS K (12 MMAs, B = K^T tiles), drained every DRAIN chunks.
constexpr int DQ_NT = 2;
constexpr int DQ_PRODUCER = DQ_NT * 4;
constexpr int DQ_MMA0 = DQ_NT * 4 + 1;
constexpr int DQ_THREADS = (DQ_NT * 5 + 1) * 32;
constexpr int DQ_NS = 6;
constexpr uint32_t DQ_COLS = 208;  // S 0 | G 64 | dS hi 128 | dS lo 160 | dq 192

struct DqSmem {
  uint16_t a[DQ_NT][4][QT * 16];  // [tile][Q hi, Q lo, dO hi, dO lo] A operands (M = 128)
  uint16_t kv[DQ_NS][6][TILE_HALVES];  // K hi, lo, V hi, lo (row form), K^T hi, lo
  float4 acc[DQ_NT][4][QT];
  uint64_t full[DQ_NS], empty[DQ_NS];
  uint64_t s_full[DQ_NT], p_full[DQ_NT], done[DQ_NT];
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(DQ_THREADS, 1)
    tape_dq_kernel(const __half* __restrict__ qr_hi, const __half* __restrict__ qr_lo,
                   const __half* __restrict__ or_hi, const __half* __restrict__ or_lo,
                   const __half* __restrict__ kr_hi, const __half* __restrict__ kr_lo,
                   const __half* __restrict__ vr_hi, const __half* __restrict__ vr_lo,
                   const __half* __restrict__ kt_hi, const __half* __restrict__ kt_lo,
                   int64_t Ttot, const TcWork* __restrict__ works, int64_t R,
                   const float* __restrict__ lse_h, const float* __restrict__ d_h,
                   const unsigned* __restrict__ bits, int d_head, float* __restrict__ dq,
                   int64_t ld, float scale, const int32_t* __restrict__ flag) {
  if (*flag) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  DqSmem& sm = *reinterpret_cast<DqSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TcWork w = works[blockIdx.x];
  const int head = blockIdx.y;
  const int T = w.tiles;
  const int64_t hb = ((int64_t)head * Ttot + w.tile0) * TILE_HALVES;
  if (warp == DQ_PRODUCER && lane == 0) {
    for (int s = 0; s < DQ_NS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], DQ_NT);
    }
    for (int t = 0; t < DQ_NT; ++t) {
      mbar_init(&sm.s_full[t], 1);
      mbar_init(&sm.p_full[t], 128);
      mbar_init(&sm.done[t], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == DQ_MMA0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const __half* asrc[4] = {qr_hi, qr_lo, or_hi, or_lo};
  for (int t = 0; t < DQ_NT; ++t)
    for (int a = 0; a < 4; ++a)
      load_a128(sm.a[t][a], asrc[a] + hb, T, (w.q0 + t * QT) / KT, threadIdx.x, DQ_THREADS);
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp == DQ_PRODUCER) {
    if (lane == 0) {
      const __half* srcs[6] = {kr_hi, kr_lo, vr_hi, vr_lo, kt_hi, kt_lo};
      for (int j = 0; j < T; ++j) {
        const int s = j % DQ_NS;
        if (j >= DQ_NS) mbar_wait_sleep(&sm.empty[s], ((j / DQ_NS) - 1) & 1);
        mbar_expect_tx(&sm.full[s], 6 * TILE_BYTES);
#pragma unroll
        for (int a = 0; a < 6; ++a)
          bulk_g2s(sm.kv[s][a], srcs[a] + hb + (int64_t)j * TILE_HALVES, TILE_BYTES,
                   &sm.full[s]);
      }
    }
    __syncwarp();
  } else if (warp >= DQ_MMA0) {
    if (lane == 0) {
      const int t = warp - DQ_MMA0;
      constexpr uint32_t ID_S = idesc_f16(QT, KT);
      constexpr uint32_t ID_O = idesc_f16(QT, 16);
      const uint64_t qh = sdesc(smem_u32(sm.a[t][0]), QT * 16, 128);
      const uint64_t ql = sdesc(smem_u32(sm.a[t][1]), QT * 16, 128);
      const uint64_t oh = sdesc(smem_u32(sm.a[t][2]), QT * 16, 128);
      const uint64_t ol = sdesc(smem_u32(sm.a[t][3]), QT * 16, 128);
      const uint32_t cb = tbase + t * DQ_COLS;
      auto issue_sg = [&](int j) {
        const int s = j % DQ_NS;
        mbar_wait_sleep(&sm.full[s], (j / DQ_NS) & 1);
        fence_after();
        const uint64_t kh = sdesc(smem_u32(sm.kv[s][0]), KT * 16, 128);
        const uint64_t kl = sdesc(smem_u32(sm.kv[s][1]), KT * 16, 128);
        const uint64_t vh = sdesc(smem_u32(sm.kv[s][2]), KT * 16, 128);
        const uint64_t vl = sdesc(smem_u32(sm.kv[s][3]), KT * 16, 128);
        umma_ss_f16(cb, qh, kh, ID_S, 0);
        umma_ss_f16(cb, qh, kl, ID_S, 1);
        umma_ss_f16(cb, ql, kh, ID_S, 1);
        umma_ss_f16(cb + 64, oh, vh, ID_S, 0);
        umma_ss_f16(cb + 64, oh, vl, ID_S, 1);
        umma_ss_f16(cb + 64, ol, vh, ID_S, 1);
        umma_commit(&sm.s_full[t]);
      };
      if (T > 0) issue_sg(0);
      for (int j = 0; j < T; ++j) {
        const int s = j % DQ_NS;
        const uint32_t kth = smem_u32(sm.kv[s][4]), ktl = smem_u32(sm.kv[s][5]);
        mbar_wait_sleep(&sm.p_full[t], j & 1);
        fence_after();
        const bool first = (j % DRAIN) == 0;
#pragma unroll
        for (int kk = 0; kk < KT / 16; ++kk) {
          const uint64_t bh = sdesc(kth + kk * 512, 256, 128), bl = sdesc(ktl + kk * 512, 256, 128);
          umma_ts_f16(cb + 192, cb + 128 + kk * 8, bh, ID_O, !(first && kk == 0));
          umma_ts_f16(cb + 192, cb + 128 + kk * 8, bl, ID_O, 1);
          umma_ts_f16(cb + 192, cb + 160 + kk * 8, bh, ID_O, 1);
        }
        if (j + 1 < T) issue_sg(j + 1);  // after the products that read dS
        umma_commit(&sm.empty[s]);
      }
      umma_commit(&sm.done[t]);
    }
    __syncwarp();
  } else {
    const int t = warp >> 2;
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lo = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t cb = tbase + lo + t * DQ_COLS;
    const float gsc = grad_scale_t(bits), dsc = ds_scale_t(bits);
    const int lr = w.q0 + t * QT + row;
    const bool valid = lr < w.n;
    const float l = valid ? lse_h[(int64_t)head * R + w.row0 + lr] : 0.f;
    const float D = valid ? d_h[(int64_t)head * R + w.row0 + lr] : 0.f;
    const float2 l2 = make_float2(l, l), D2 = make_float2(D, D), dsc2 = make_float2(dsc, dsc);
    float4* acc = &sm.acc[t][0][row];
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4) acc[c4 * QT] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto drain = [&]() {
      uint32_t r[16];
      PTX_LD16(cb + 192, r);
      tmem_wait_ld();
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const float4 a = acc[c4 * QT];
        const float2 x = add_f32x2(make_float2(a.x, a.y), make_float2(__uint_as_float(r[4 * c4]),
                                                                     __uint_as_float(r[4 * c4 + 1])));
        const float2 y = add_f32x2(make_float2(a.z, a.w), make_float2(__uint_as_float(r[4 * c4 + 2]),
                                                                     __uint_as_float(r[4 * c4 + 3])));
        acc[c4 * QT] = make_float4(x.x, x.y, y.x, y.y);
      }
    };
    for (int j = 0; j < T; ++j) {
      mbar_wait_sleep(&sm.s_full[t], j & 1);
      fence_after();
      if (j > 0 && j % DRAIN == 0) drain();  // dq of chunks [j - DRAIN, j) complete
      const int k0 = j * KT;
      const bool full = valid && k0 + KT <= w.n;  // no padded key in this chunk
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t rs[16], rg[16], dh8[8], dl8[8];
        PTX_LD16(cb + 16 * c, rs);
        PTX_LD16(cb + 64 + 16 * c, rg);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 x = sub_f32x2(make_float2(__uint_as_float(rs[2 * i]), __uint_as_float(rs[2 * i + 1])), l2);
          float2 p2 = make_float2(ex2f(x.x), ex2f(x.y));
          if (!full) {
            const int kk = k0 + 16 * c + 2 * i;
            p2.x = valid && kk < w.n ? p2.x : 0.f;
            p2.y = valid && kk + 1 < w.n ? p2.y : 0.f;
          }
          const float2 g = sub_f32x2(make_float2(__uint_as_float(rg[2 * i]), __uint_as_float(rg[2 * i + 1])), D2);
          split2(mul_f32x2(mul_f32x2(p2, g), dsc2), dh8[i], dl8[i]);
        }
        PTX_ST8(cb + 128 + 8 * c, dh8);
        PTX_ST8(cb + 160 + 8 * c, dl8);
      }
      tmem_wait_st();
      fence_before();
      mbar_arrive(&sm.p_full[t]);
    }
    mbar_wait_sleep(&sm.done[t], 0);
    fence_after();
    if (T > 0) drain();
    if (valid) {
      const float scl = scale / (gsc * dsc);
      float* o = dq + (w.row0 + lr) * ld + head * d_head;
      float vv[16];
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const float4 a = acc[c4 * QT];
        vv[4 * c4] = a.x;
        vv[4 * c4 + 1] = a.y;
        vv[4 * c4 + 2] = a.z;
        vv[4 * c4 + 3] = a.w;
      }
      for (int d = 0; d < d_head; ++d) o[d] = vv[d] * scl;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == DQ_MMA0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                 "r"(TMEM_COLS));
  }
}

}  // namespace tt

size_t tape_attention_tc_scratch(int64_t R, int F, int n_head) {
  // 64-row tiles: at most R / 64 + F of them; up to 12 packed tile arrays (backward: K, V, Q,
  // dO row form and Q^T, dO^T, hi and lo), per-(row, head) bounds / offsets or lse / D,
  // the scaled dO rows, kmax, flags
  const int64_t Ttot = R / tt::KT + F + 1;
  return (size_t)12 * n_head * Ttot * tt::TILE_BYTES + (size_t)R * n_head * 8 +
         (size_t)n_head * Ttot * 2 * tt::KT * 4 + 256 + (size_t)R * n_head * 16 * 4 +
         (size_t)F * n_head * 4 + 8192;
}

// The tape forward of the full N x N head attention on tcgen05.  Returns the device flag:
// non-zero when some score bound exceeds the fp16 limit or an operand left the fp16 range
// (the forward kernel then writes nothing and the caller's gated mma.sync forward runs).
const int32_t* tape_attention_fwd_tc(const float* q, const float* k, const float* v, int64_t ld,
                           int n_head, int d_head, int64_t R, int F, const TcWork* works_dev,
                           int64_t num_works, const int64_t* tile_row0_dev,
                           const int32_t* tile_n_dev, int64_t Ttot, const int32_t* row_fwd,
                           float* out, int64_t ldo, float* lse, void* scratch,
                           cudaStream_t st) {
  GO_CHECK(d_head >= 1 && d_head <= 15, "tape_attention_fwd_tc needs d_head <= 15");
  static bool attr = false;
  const size_t smem = sizeof(tt::FwdSmem) + 1024;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(tt::tape_fwd_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int64_t tile_elems = (int64_t)n_head * Ttot * tt::TILE_HALVES;
  __half* base = reinterpret_cast<__half*>(scratch);
  __half *qh = base, *ql = qh + tile_elems, *kh = ql + tile_elems, *kl = kh + tile_elems;
  __half *vh = kl + tile_elems, *vl = vh + tile_elems;
  float* bound = reinterpret_cast<float*>(vl + tile_elems);
  float* c15 = bound + R * n_head;
  unsigned* kmax = reinterpret_cast<unsigned*>(c15 + R * n_head);
  int32_t* flag = reinterpret_cast<int32_t*>(kmax + (int64_t)F * n_head);
  CUDA_CHECK(cudaMemsetAsync(kmax, 0, ((size_t)F * n_head + 1) * 4, st));
  const float qscale = (float)(1.4426950408889634 / std::sqrt((double)d_head));
  const int64_t threads = (int64_t)n_head * Ttot * (tt::KT / 8) * 2;
  const unsigned blocks = (unsigned)cdiv(threads, 256);
  tt::tape_pack_kernel<<<blocks, 256, 0, st>>>(k, ld, n_head, d_head, 1.f, tile_row0_dev,
                                                tile_n_dev, Ttot, 1, nullptr, kh, kl, nullptr,
                                                nullptr, kmax, flag);
  LAUNCH_CHECK();
  tt::tape_pack_kernel<<<blocks, 256, 0, st>>>(v, ld, n_head, d_head, 1.f, tile_row0_dev,
                                                tile_n_dev, Ttot, 1, nullptr, nullptr, nullptr,
                                                vh, vl, nullptr, flag);
  LAUNCH_CHECK();
  tt::tape_bound_kernel<<<(unsigned)cdiv(R * n_head, 256), 256, 0, st>>>(
      q, ld, n_head, d_head, qscale, R, row_fwd, kmax, bound, c15, flag);
  LAUNCH_CHECK();
  tt::tape_pack_kernel<<<blocks, 256, 0, st>>>(q, ld, n_head, d_head, qscale, tile_row0_dev,
                                                tile_n_dev, Ttot, 2, c15, qh, ql, nullptr,
                                                nullptr, nullptr, flag);
  LAUNCH_CHECK();

  dim3 grid((unsigned)num_works, (unsigned)n_head);
  if (num_works > 0) {
    tt::tape_fwd_kernel<<<grid, tt::NUM_THREADS, smem, st>>>(qh, ql, kh, kl, vh, vl, Ttot,
                                                            works_dev, bound, n_head, out, ldo,
                                                            d_head, lse, flag);
    LAUNCH_CHECK();
  }
  return flag;
}


// dk, dv of the full N x N head attention on tcgen05 (tape_dkv_kernel).  kv_works: one
// entry per (forward, 128 keys) (TcWork with q0 = first local key).  Computes D = dO.O into
// Dbuf first.  Returns false when an operand left the fp16 range (nothing written then).
const int32_t* tape_attention_bwd_tc(const float* q, const float* k, const float* v, const float* O,
                           const float* dO, int64_t ld, int n_head, int d_head, int64_t R,
                           int F, const float* lse, const TcWork* kv_works_dev,
                           int64_t num_kv_works, const TcWork* q_works_dev,
                           int64_t num_q_works, const int64_t* tile_row0_dev,
                           const int32_t* tile_n_dev, int64_t Ttot, float* Dbuf, float* dq,
                           float* dk, float* dv, void* scratch, cudaStream_t st) {
  GO_CHECK(d_head >= 1 && d_head <= 16, "tape_attention_bwd_tc needs d_head <= 16");
  static bool attr = false;
  const size_t smem = sizeof(tt::KvSmem) + 1024;
  const size_t smem_q = sizeof(tt::DqSmem) + 1024;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(tt::tape_dkv_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_CHECK(cudaFuncSetAttribute(tt::tape_dq_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_q));
    attr = true;
  }
  const int64_t W = (int64_t)n_head * d_head;
  const int64_t te = (int64_t)n_head * Ttot * tt::TILE_HALVES;
  __half* t = reinterpret_cast<__half*>(scratch);
  __half *krh = t, *krl = t + te, *vrh = t + 2 * te, *vrl = t + 3 * te;
  __half *qrh = t + 4 * te, *qrl = t + 5 * te, *qth = t + 6 * te, *qtl = t + 7 * te;
  __half *orh = t + 8 * te, *orl = t + 9 * te, *oth = t + 10 * te, *otl = t + 11 * te;
  float* lsd = reinterpret_cast<float*>(t + 12 * te);  // [H][Ttot][2][64], bulk-copied
  float* lse_h = lsd + (int64_t)n_head * Ttot * 2 * tt::KT;
  float* d_h = lse_h + R * n_head;
  float* dOs = d_h + R * n_head;
  unsigned* bits = reinterpret_cast<unsigned*>(dOs + R * W);
  int32_t* flag = reinterpret_cast<int32_t*>(bits + 4);
  CUDA_CHECK(cudaMemsetAsync(bits, 0, 8 * 4, st));
  attention_backward_D(dO, O, ld, n_head, d_head, R, Dbuf, st);
  tt::absmax_t_kernel<<<(unsigned)std::min<int64_t>(cdiv(R * W, 256), 148 * 8), 256, 0, st>>>(
      dO, ld, R, (int)W, bits);
  LAUNCH_CHECK();
  tt::bwd_rows_kernel<<<(unsigned)cdiv(R * n_head, 256), 256, 0, st>>>(
      v, dO, ld, lse, Dbuf, n_head, d_head, R, bits, lse_h, d_h);
  LAUNCH_CHECK();
  tt::scale_rows_kernel<<<(unsigned)cdiv(R * W, 256), 256, 0, st>>>(dO, ld, R, (int)W, bits, dOs);
  LAUNCH_CHECK();
  tt::tile_lsd_kernel<<<(unsigned)cdiv((int64_t)n_head * Ttot * tt::KT, 256), 256, 0, st>>>(
      lse, Dbuf, n_head, tile_row0_dev, tile_n_dev, Ttot, bits, lsd);
  LAUNCH_CHECK();
  const float qscale = (float)(1.4426950408889634 / std::sqrt((double)d_head));
  const int64_t threads = (int64_t)n_head * Ttot * (tt::KT / 8) * 2;
  const unsigned blocks = (unsigned)cdiv(threads, 256);
  auto pack = [&](const float* x, int64_t ldx, float sc, __half* rh, __half* rl, __half* th,
                  __half* tl) {
    tt::tape_pack_kernel<<<blocks, 256, 0, st>>>(x, ldx, n_head, d_head, sc, tile_row0_dev,
                                                  tile_n_dev, Ttot, 0, nullptr, rh, rl, th, tl,
                                                  nullptr, flag);
    LAUNCH_CHECK();
  };
  pack(k, ld, 1.f, krh, krl, nullptr, nullptr);
  pack(v, ld, 1.f, vrh, vrl, nullptr, nullptr);
  pack(q, ld, qscale, qrh, qrl, qth, qtl);
  pack(dOs, W, 1.f, orh, orl, oth, otl);

  dim3 grid((unsigned)num_kv_works, (unsigned)n_head);
  if (num_kv_works > 0) {
    tt::tape_dkv_kernel<<<grid, tt::KV_THREADS, smem, st>>>(
        krh, krl, vrh, vrl, qrh, qrl, qth, qtl, orh, orl, oth, otl, Ttot, kv_works_dev, lsd,
        bits, d_head, dk, dv, ld, (float)(1.0 / 1.4426950408889634), flag);
    LAUNCH_CHECK();
  }
  // dq: K^T tiles into the Q^T slots (stream-ordered after the dk / dv kernel read them)
  pack(k, ld, 1.f, nullptr, nullptr, qth, qtl);
  dim3 gq((unsigned)num_q_works, (unsigned)n_head);
  if (num_q_works > 0) {
    tt::tape_dq_kernel<<<gq, tt::DQ_THREADS, smem_q, st>>>(
        qrh, qrl, orh, orl, krh, krl, vrh, vrl, qth, qtl, Ttot, q_works_dev, R, lse_h, d_h,
        bits, d_head, dq, ld, (float)(1.0 / std::sqrt((double)d_head)), flag);
    LAUNCH_CHECK();
  }
  return flag;
}

}  // namespace go
