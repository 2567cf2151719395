// Segmented (block-banded) trunk attention on warp-level tensor-core MMAs
// (policy.py:157-177: the queries of segment s attend to the keys of segments s-1 and s
// of the same forward; multi_head_attention / scaled_dot_attention, tensor.py:382-388).
//
// The trunk's attention is tiny per query (<= 2S = 128 keys, d_head = 15), so it is
// bound by moving Q/K/V once and by the per-key instruction count, not by tensor math.
// The SIMT kernel (attention.cu) spends 32 FFMA + 8 LDS per (query, key); here a warp
// handles 16 queries with mma.sync.m16n8k16 (fp16 operands, fp32 accumulation):
//   S  = Q K^T   8 MMAs per 64-key chunk (n-tiles of 8 keys, K = 16 = padded d_head)
//   O += P V     8 MMAs per 64-key chunk (4 k-steps of 16 keys x 2 n-tiles of 8 dims)
// with the S accumulator fragments reused directly as the A fragments of P (the
// m16n8k16 C layout equals the A layout), exact online softmax (running max) per row.
// CTA = one 64-query tile of the banded tile list x one head, 4 warps; key chunks of 64
// staged in shared memory as fp16 (K row-major, V transposed), rows padded so the
// fragment loads are bank-conflict free.
//
// Precision: Q (pre-scaled by log2(e)/sqrt(d)), K, V and P rounded to fp16 (10-bit
// mantissa, the same as the head attention's operands); operands beyond the fp16 range
// set *flag and the caller re-runs the SIMT kernel gated on it.
#include <cmath>
#include <cuda_fp16.h>

#include "engine.cuh"

namespace go {
namespace tm {

constexpr int QT = 64;      // queries per CTA
constexpr int KC = 64;      // keys per chunk
constexpr int KS = 24;      // Ks row stride (halves): 48 B, conflict-free fragment loads
constexpr float RANGE = 60000.f;
constexpr float PSCALE = 32768.f;  // SPLIT: P (<= 1) is packed as 2^15 P

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// B fragments of both 8-dim n-tiles of a 16-row k-step from a row-major [row][dim] smem
// block: ldmatrix.x4.trans (lanes 0-7 / 8-15 / 16-23 / 24-31 address rows 0-7 / 8-15 of
// dims 0-7, then of dims 8-15); b[0..1] n-tile 0, b[2..3] n-tile 1
__device__ __forceinline__ void ldsm_bT(const __half* blk, int stride, int lane, uint32_t* b) {
  const __half* p = blk + ((lane & 7) + ((lane >> 3) & 1) * 8) * stride + (lane >> 4) * 8;
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// SPLIT (the PPO tape's forward): every fp16 operand is a 2-term split x = hi + lo and
// each product takes three MMAs (hi.hi + hi.lo + lo.hi), ~2^-21 relative -- the update's
// Adam step needs fp32-class logits and log-sum-exps (see attn_bwd_mma.cu).
template <bool SPLIT>
__global__ void __launch_bounds__(128) trunk_mma_kernel(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    int64_t ld, int d_head, const AttnTile* __restrict__ tiles, float* __restrict__ out,
    int64_t ldo, float qscale, int32_t* __restrict__ flag, float* __restrict__ lse, int n_head) {
  constexpr int KS2 = SPLIT ? 40 : KS;  // halves per key row (hi 0..15, lo 16..31)
  __shared__ __align__(16) __half Ks[KC * KS2];
  __shared__ __align__(16) __half Vs[KC * KS2];  // row-major [key][d] (lo at +16)
  const AttnTile tl = tiles[blockIdx.x];
  const int head = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t col0 = (int64_t)head * d_head;
  bool big = false;

  // A fragments of this warp's 16 queries (rows g and g + 8, dims 2tq.. and 2tq+8..)
  uint32_t qa[4], ql[4];
  {
    const int64_t r0 = tl.q0 + warp * 16 + g, r1 = r0 + 8;
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t r = (i & 1) ? r1 : r0;  // order: (r0,d0) (r1,d0) (r0,d8) (r1,d8) pairs
      const int d = 2 * tq + ((i >> 2) ? 8 : 0) + ((i >> 1) & 1);
      float val = 0.f;
      if (r < tl.q1 && d < d_head) val = q[r * ld + col0 + d] * qscale;
      big |= !(fabsf(val) <= RANGE);
      x[i] = val;
    }
    // x[0]=(r0,2tq) x[1]=(r1,2tq) x[2]=(r0,2tq+1) x[3]=(r1,2tq+1) x[4..7] same at +8
    const int pi[4][2] = {{0, 2}, {1, 3}, {4, 6}, {5, 7}};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      qa[j] = pack2(x[pi[j][0]], x[pi[j][1]]);
      if (SPLIT) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&qa[j]));
        ql[j] = pack2(x[pi[j][0]] - f.x, x[pi[j][1]] - f.y);
      }
    }
  }
  float o[2][4];
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[n][e] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int64_t kc = tl.k0; kc < tl.k1; kc += KC) {
    const int64_t rem = tl.k1 - kc;
    const int nk = rem < KC ? (int)rem : KC;
    __syncthreads();
    {
      // stage: thread = (key, 8-dim half); K and V row-major [key][d] (V's B fragments
      // come out transposed through ldmatrix.trans)
      const int key = tid >> 1, d0 = (tid & 1) * 8;
      __align__(16) __half kr[8], kl[8], vr[8], vl[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int d = d0 + i;
        float kv = 0.f, vv = 0.f;
        if (key < nk && d < d_head) {
          kv = k[(kc + key) * ld + col0 + d];
          vv = v[(kc + key) * ld + col0 + d];
          big |= !(fabsf(kv) <= RANGE) || !(fabsf(vv) <= RANGE);
        } else if (SPLIT && key < nk && d == d_head) {
          vv = 1.f;  // ones column: the MMA accumulates the row sum next to O
        }
        kr[i] = __float2half_rn(kv);
        vr[i] = __float2half_rn(vv);
        if (SPLIT) {
          kl[i] = __float2half_rn(kv - __half2float(kr[i]));
          vl[i] = __float2half_rn(vv - __half2float(vr[i]));
        }
      }
      *reinterpret_cast<uint4*>(&Ks[key * KS2 + d0]) = *reinterpret_cast<const uint4*>(kr);
      *reinterpret_cast<uint4*>(&Vs[key * KS2 + d0]) = *reinterpret_cast<const uint4*>(vr);
      if (SPLIT) {
        *reinterpret_cast<uint4*>(&Ks[key * KS2 + 16 + d0]) = *reinterpret_cast<const uint4*>(kl);
        *reinterpret_cast<uint4*>(&Vs[key * KS2 + 16 + d0]) = *reinterpret_cast<const uint4*>(vl);
      }
    }
    __syncthreads();
    // S = Q K^T: 8 n-tiles of 8 keys
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
      const __half* kp = &Ks[(8 * n + g) * KS2 + 2 * tq];
      const uint32_t b0 = *reinterpret_cast<const uint32_t*>(kp);
      const uint32_t b1 = *reinterpret_cast<const uint32_t*>(kp + 8);
      if (SPLIT) {
        mma16816(s[n], ql, b0, b1);
        mma16816(s[n], qa, *reinterpret_cast<const uint32_t*>(kp + 16),
                 *reinterpret_cast<const uint32_t*>(kp + 24));
      }
      mma16816(s[n], qa, b0, b1);
    }
    // online softmax over the chunk (rows g: s[.][0..1], g + 8: s[.][2..3])
    float c0 = -INFINITY, c1 = -INFINITY;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int key = 8 * n + 2 * tq;
      if (key >= nk) s[n][0] = s[n][2] = -INFINITY;
      if (key + 1 >= nk) s[n][1] = s[n][3] = -INFINITY;
      c0 = fmaxf(c0, fmaxf(s[n][0], s[n][1]));
      c1 = fmaxf(c1, fmaxf(s[n][2], s[n][3]));
    }
    c0 = fmaxf(c0, __shfl_xor_sync(0xffffffffu, c0, 1));
    c0 = fmaxf(c0, __shfl_xor_sync(0xffffffffu, c0, 2));
    c1 = fmaxf(c1, __shfl_xor_sync(0xffffffffu, c1, 1));
    c1 = fmaxf(c1, __shfl_xor_sync(0xffffffffu, c1, 2));
    const float n0 = fmaxf(m0, c0), n1 = fmaxf(m1, c1);
    const float f0 = ex2(m0 - n0), f1 = ex2(m1 - n1);  // 0 on the first chunk
    m0 = n0;
    m1 = n1;
    l0 *= f0;
    l1 *= f1;
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      o[n][0] *= f0;
      o[n][1] *= f0;
      o[n][2] *= f1;
      o[n][3] *= f1;
    }
    uint32_t pa[8][2], pl[8][2];  // P as fp16 pairs: [n-tile][row g | row g+8]
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float p0 = ex2(s[n][0] - m0), p1 = ex2(s[n][1] - m0);
      float p2 = ex2(s[n][2] - m1), p3 = ex2(s[n][3] - m1);
      l0 += p0 + p1;
      l1 += p2 + p3;
      if (SPLIT) {  // 2^15 P: small P stay fp16-normal (hi) and the lo term keeps its bits
        p0 *= PSCALE;
        p1 *= PSCALE;
        p2 *= PSCALE;
        p3 *= PSCALE;
      }
      pa[n][0] = pack2(p0, p1);
      pa[n][1] = pack2(p2, p3);
      if (SPLIT) {
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&pa[n][0]));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&pa[n][1]));
        pl[n][0] = pack2(p0 - a.x, p1 - a.y);
        pl[n][1] = pack2(p2 - b.x, p3 - b.y);
      }
    }
    // O += P V: k-steps of 16 keys (n-tiles 2kk, 2kk+1), n-tiles of 8 dims.  SPLIT: the
    // chunk's PV goes to a fresh accumulator added to O with IEEE FADDs (the MMA's own
    // fp32 accumulation drops the low bits of small addends with a consistent sign)
    float oc[2][4] = {};
    float(*od)[4] = SPLIT ? oc : o;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t a[4] = {pa[2 * kk][0], pa[2 * kk][1], pa[2 * kk + 1][0], pa[2 * kk + 1][1]};
      const uint32_t al[4] = {pl[2 * kk][0], pl[2 * kk][1], pl[2 * kk + 1][0], pl[2 * kk + 1][1]};
      uint32_t bh[4], bl[4] = {0u, 0u, 0u, 0u};
      ldsm_bT(Vs + 16 * kk * KS2, KS2, lane, bh);
      if (SPLIT) ldsm_bT(Vs + 16 * kk * KS2 + 16, KS2, lane, bl);
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        if (SPLIT) {
          mma16816(od[n], al, bh[2 * n], bh[2 * n + 1]);
          mma16816(od[n], a, bl[2 * n], bl[2 * n + 1]);
        }
        mma16816(od[n], a, bh[2 * n], bh[2 * n + 1]);
      }
    }
    if (SPLIT) {
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[n][e] += oc[n][e];
    }
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  if (SPLIT && d_head < 16) {
    // row sums from the ones column (dim d_head), accumulated exactly like O (per-chunk
    // MMA sums added with FADDs) so numerator and denominator share their rounding
    const int holder = (lane & ~3) | ((d_head >> 1) & 3);
    const int n = d_head >> 3, e = d_head & 1;
    const float s0 = __shfl_sync(0xffffffffu, o[n][e], holder);
    const float s1 = __shfl_sync(0xffffffffu, o[n][2 + e], holder);
    l0 = s0 / PSCALE;
    l1 = s1 / PSCALE;
  }
  const float i0 = (SPLIT ? 1.f / PSCALE : 1.f) / l0, i1 = (SPLIT ? 1.f / PSCALE : 1.f) / l1;
  const int64_t r0 = tl.q0 + warp * 16 + g, r1 = r0 + 8;
  if (lse && tq == 0) {  // log2-sum-exp of the scaled scores (the training tape's P recompute)
    if (r0 < tl.q1) lse[r0 * n_head + head] = m0 + log2f(l0);
    if (r1 < tl.q1) lse[r1 * n_head + head] = m1 + log2f(l1);
  }
#pragma unroll
  for (int n = 0; n < 2; ++n) {
    const int d = 8 * n + 2 * tq;
    if (r0 < tl.q1) {
      if (d < d_head) out[r0 * ldo + col0 + d] = o[n][0] * i0;
      if (d + 1 < d_head) out[r0 * ldo + col0 + d + 1] = o[n][1] * i0;
    }
    if (r1 < tl.q1) {
      if (d < d_head) out[r1 * ldo + col0 + d] = o[n][2] * i1;
      if (d + 1 < d_head) out[r1 * ldo + col0 + d + 1] = o[n][3] * i1;
    }
  }
  if (big) atomicOr(flag, 1);
}

}  // namespace tm

bool trunk_mma_supported(int d_head) { return d_head >= 1 && d_head <= 16; }

void trunk_attention_mma(const float* q, const float* k, const float* v, int64_t ld, int n_head,
                         int d_head, const AttnTile* tiles_dev, int64_t num_tiles, float* out,
                         int64_t ldo, int32_t* flag, cudaStream_t st, float* lse, bool split) {
  if (num_tiles <= 0) return;
  GO_CHECK(d_head <= 16, "trunk_attention_mma needs d_head <= 16");
  CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(int32_t), st));
  const float qscale = (float)(1.4426950408889634 / std::sqrt((double)d_head));
  dim3 grid((unsigned)num_tiles, (unsigned)n_head);
  if (split)
    tm::trunk_mma_kernel<true><<<grid, 128, 0, st>>>(q, k, v, ld, d_head, tiles_dev, out, ldo,
                                                     qscale, flag, lse, n_head);
  else
    tm::trunk_mma_kernel<false><<<grid, 128, 0, st>>>(q, k, v, ld, d_head, tiles_dev, out, ldo,
                                                      qscale, flag, lse, n_head);
  LAUNCH_CHECK();
}

}  // namespace go
