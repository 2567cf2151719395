// Multi-head softmax attention over key ranges (SIMT fp32, online softmax).
// One kernel serves both attentions of the policy:
//   trunk  (policy.py:157-177): segment s's queries attend to rows of segments
//          s-1 and s  -> tiles with k0 = max(seg_lo - S, f0), k1 = seg_hi
//   heads  (policy.py:210):     all N x N pairs -> k0 = f0, k1 = f1
// scaled_dot_attention = softmax(q k^T / sqrt(d_k)) v (tensor.py:382-388).
#include "engine.cuh"

namespace go {

constexpr int ATT_Q = 64;   // queries per CTA (one per thread)
constexpr int ATT_KC = 64;  // keys per shared-memory chunk

template <int DH>
__global__ void __launch_bounds__(ATT_Q) attn_kernel(const float* __restrict__ q,
                                                     const float* __restrict__ k,
                                                     const float* __restrict__ v, int64_t ld,
                                                     int d_head, const AttnTile* __restrict__ tiles,
                                                     float* __restrict__ out, int64_t ldo,
                                                     float scale_log2,
                                                     float* __restrict__ lse, int n_head,
                                                     const int32_t* __restrict__ gate,
                                                     const float* __restrict__ kalt,
                                                     const float* __restrict__ valt) {
  if (gate && *gate == 0) return;
  __shared__ __align__(16) float Ks[ATT_KC][DH];
  __shared__ __align__(16) float Vs[ATT_KC][DH];
  const AttnTile tl = tiles[blockIdx.x];
  const int head = blockIdx.y;
  const int64_t col0 = (int64_t)head * d_head;
  const int64_t row = tl.q0 + threadIdx.x;
  const bool active = row < tl.q1;
  float qr[DH], acc[DH];
#pragma unroll
  for (int d = 0; d < DH; ++d) {
    qr[d] = (active && d < d_head) ? q[row * ld + col0 + d] * scale_log2 : 0.f;
    acc[d] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int64_t kc = tl.k0; kc < tl.k1; kc += ATT_KC) {
    const int64_t rem_k = tl.k1 - kc;
    const int nk = rem_k < ATT_KC ? (int)rem_k : ATT_KC;
    for (int idx = threadIdx.x; idx < ATT_KC * DH; idx += ATT_Q) {
      int j = idx / DH, d = idx % DH;
      bool ok = j < nk && d < d_head;
      // kalt / valt: the keys before the tile's first query (the previous segment of
      // a banded trunk tile) come from the cache-hook buffers (policy.py:170-172)
      const bool pre = kalt && kc + j < tl.q0;
      Ks[j][d] = ok ? (pre ? kalt : k)[(kc + j) * ld + col0 + d] : 0.f;
      Vs[j][d] = ok ? (pre ? valt : v)[(kc + j) * ld + col0 + d] : 0.f;
    }
    __syncthreads();
    float s[ATT_KC];
    float cmax = -INFINITY;
#pragma unroll
    for (int j = 0; j < ATT_KC; ++j) {
      float t = 0.f;
#pragma unroll
      for (int d = 0; d < DH; ++d) t = fmaf(qr[d], Ks[j][d], t);
      s[j] = (j < nk) ? t : -INFINITY;
      cmax = fmaxf(cmax, s[j]);
    }
    float mnew = fmaxf(m, cmax);
    float corr = exp2f(m - mnew);
    l *= corr;
#pragma unroll
    for (int d = 0; d < DH; ++d) acc[d] *= corr;
    m = mnew;
#pragma unroll
    for (int j = 0; j < ATT_KC; ++j) {
      float p = exp2f(s[j] - m);
      l += p;
#pragma unroll
      for (int d = 0; d < DH; ++d) acc[d] = fmaf(p, Vs[j][d], acc[d]);
    }
    __syncthreads();
  }
  if (active) {
    float inv = 1.f / l;
    for (int d = 0; d < d_head; ++d) out[row * ldo + col0 + d] = acc[d] * inv;
    // log2-domain log-sum-exp of the scaled scores, for the backward pass
    if (lse) lse[row * n_head + head] = m + log2f(l);
  }
}

void attention(const float* q, const float* k, const float* v, int64_t ld, int n_head,
               int d_head, const AttnTile* tiles_dev, int64_t num_tiles, float* out,
               int64_t ldo, cudaStream_t st, float* lse, const int32_t* gate,
               const float* kalt, const float* valt) {
  if (num_tiles <= 0) return;
  float scale_log2 = (float)(1.4426950408889634 / sqrt((double)d_head));
  dim3 grid((unsigned)num_tiles, (unsigned)n_head);
#define GO_ATT(DHV)                                                                          \
  attn_kernel<DHV><<<grid, ATT_Q, 0, st>>>(q, k, v, ld, d_head, tiles_dev, out, ldo,           \
                                           scale_log2, lse, n_head, gate, kalt, valt)
  if (d_head <= 4) GO_ATT(4);
  else if (d_head <= 8) GO_ATT(8);
  else if (d_head <= 16) GO_ATT(16);
  else if (d_head <= 32) GO_ATT(32);
  else if (d_head <= 64) GO_ATT(64);
  else GO_THROW(GO_ERR_UNSUPPORTED, "d_head %d > 64", d_head);
#undef GO_ATT
  LAUNCH_CHECK();
}

}  // namespace go
