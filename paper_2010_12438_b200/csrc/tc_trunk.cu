// Segmented (block-banded) trunk attention on the 5th-generation tensor cores
// (policy.py:157-177: the queries of segment s attend to the keys of segments s-1 and
// s of the same forward; multi_head_attention / scaled_dot_attention, tensor.py:382-388).
//
// One CTA = one head x 128 consecutive query rows of one forward (an M=128 tile that
// spans 128/S segments) and the union of their key windows (<= 240 keys; 192 for the
// default S = 64), 5 warps:
//   all warps  stage Q (scaled by log2(e)/sqrt(d_head)), K and V^T in shared memory in
//              the UMMA K-major canonical layout, tf32-rounded; V[:,15] = 1 so the PV
//              MMA also returns each row's softmax denominator;
//   warp 4     S = Q K^T (kind::tf32, M=128, N=keys, K=16) into TMEM, then, once P is
//              back in TMEM, O = P V (M=128, N=16, K=keys, A = P from TMEM);
//   warps 0-3  one query row per thread: exact row max over the row's own window
//              (keys outside it are masked to P = 0), P = 2^(s - max) written over S.
// Output: O[:, d] / O[:, 15] for d < d_head, row-major like the SIMT attention.
#include <algorithm>
#include <cmath>

#include "engine.cuh"
#include "tcgen05.cuh"

namespace go {
namespace tt {

using namespace ptx;

constexpr int QT = 128;
constexpr int KPAD = 256;  // key capacity of the staging buffers
constexpr int NKMAX = TRUNK_TC_MAX_KEYS;
constexpr uint32_t O_COL = NKMAX;  // O after the S columns
constexpr uint32_t TMEM_COLS = 256;
constexpr int THREADS = 160;

struct Smem {
  float q[QT * 16];
  float k[KPAD * 16];
  float vt[KPAD * 16];
  uint64_t bar_s, bar_p, bar_o;
  uint32_t tmem;
};

__global__ void __launch_bounds__(THREADS) trunk_attn_tc_kernel(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    int64_t ld, int d_head, int S, float qscale, const TrunkTile* __restrict__ tiles,
    float* __restrict__ out, int64_t ldo) {
  __shared__ __align__(1024) Smem sm;
  const TrunkTile T = tiles[blockIdx.x];
  const int head = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NKP = (T.nk + 15) & ~15;
  const int64_t col = (int64_t)head * d_head;
  if (warp == 4) {
    if (lane == 0) {
      mbar_init(&sm.bar_s, 1);
      mbar_init(&sm.bar_p, 128);
      mbar_init(&sm.bar_o, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < QT * 16; i += THREADS) {
    const int r = i >> 4, d = i & 15;
    const float x = (r < T.nq && d < d_head) ? tf32_rn(q[(T.q0 + r) * ld + col + d] * qscale) : 0.f;
    sm.q[(d >> 2) * (QT * 4) + (r >> 3) * 32 + (r & 7) * 4 + (d & 3)] = x;
  }
  for (int i = tid; i < NKP * 16; i += THREADS) {
    const int r = i >> 4, d = i & 15;
    const bool ok = r < T.nk;
    float kv = 0.f, vv = 0.f;
    if (ok && d < d_head) {
      kv = tf32_rn(k[(T.k0 + r) * ld + col + d]);
      vv = tf32_rn(v[(T.k0 + r) * ld + col + d]);
    } else if (ok && d == 15) {
      vv = 1.f;
    }
    sm.k[(d >> 2) * (KPAD * 4) + (r >> 3) * 32 + (r & 7) * 4 + (d & 3)] = kv;
    sm.vt[(r >> 2) * 64 + (d >> 3) * 32 + (d & 7) * 4 + (r & 3)] = vv;
  }
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = sm.tmem;

  if (warp == 4) {
    if (lane == 0) {
      const uint32_t qa = smem_u32(sm.q), ka = smem_u32(sm.k), va = smem_u32(sm.vt);
      const uint32_t id_s = idesc_tf32(QT, NKP);
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
        umma_ss(tbase, sdesc(qa + kk * 4096, 2048, 128),
                sdesc(ka + kk * (2 * KPAD * 16), KPAD * 16, 128), id_s, kk > 0);
      umma_commit(&sm.bar_s);
      mbar_wait(&sm.bar_p, 0);
      fence_after();
      constexpr uint32_t id_o = idesc_tf32(QT, 16);
      for (int kk = 0; kk < NKP / 8; ++kk)
        umma_ts(tbase + O_COL, tbase + kk * 8, sdesc(va + kk * 512, 256, 128), id_o, kk > 0);
      umma_commit(&sm.bar_o);
    }
    __syncwarp();
  } else {
    const int r = tid;  // query row of the tile (TMEM lane)
    const bool active = r < T.nq;
    const int64_t row = T.q0 + r;
    int c0 = 0, c1 = 0;  // this row's key window, relative to k0
    if (active) {
      const int64_t s = (row - T.f0) / S;
      const int64_t kl = T.f0 + (s > 0 ? (s - 1) * S : 0);
      const int64_t kh = T.f0 + (s + 1) * S < T.f1 ? T.f0 + (s + 1) * S : T.f1;
      c0 = (int)(kl - T.k0);
      c1 = (int)(kh - T.k0);
    }
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    mbar_wait(&sm.bar_s, 0);
    fence_after();
    float m = -INFINITY;
    for (int cb = 0; cb < NKP; cb += 16) {
      uint32_t u[16];
      PTX_LD16(tbase + lane_off + cb, u);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (cb + j >= c0 && cb + j < c1) m = fmaxf(m, __uint_as_float(u[j]));
    }
    for (int cb = 0; cb < NKP; cb += 16) {
      uint32_t u[16];
      PTX_LD16(tbase + lane_off + cb, u);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const bool in = cb + j >= c0 && cb + j < c1;
        u[j] = __float_as_uint(in ? ex2f(__uint_as_float(u[j]) - m) : 0.f);
      }
      PTX_ST16(tbase + lane_off + cb, u);
    }
    tmem_wait_st();
    fence_before();
    mbar_arrive(&sm.bar_p);
    mbar_wait(&sm.bar_o, 0);
    fence_after();
    uint32_t o[16];
    PTX_LD16(tbase + lane_off + O_COL, o);
    tmem_wait_ld();
    if (active) {
      const float inv = 1.f / __uint_as_float(o[15]);
      float* dst = out + row * ldo + col;
      for (int d = 0; d < d_head; ++d) dst[d] = __uint_as_float(o[d]) * inv;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 4)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                 "r"(TMEM_COLS));
}

}  // namespace tt

bool trunk_tc_build_tiles(const std::vector<int64_t>& row_off, int64_t S,
                          std::vector<TrunkTile>& out) {
  bool ok = S >= 1;
  for (size_t f = 0; ok && f + 1 < row_off.size(); ++f) {
    const int64_t f0 = row_off[f], f1 = row_off[f + 1];
    for (int64_t q0 = f0; q0 < f1; q0 += tt::QT) {
      const int64_t nq = std::min<int64_t>(tt::QT, f1 - q0);
      const int64_t sf = (q0 - f0) / S, sl = (q0 + nq - 1 - f0) / S;
      const int64_t k0 = f0 + (sf > 0 ? (sf - 1) * S : 0);
      const int64_t k1 = std::min(f1, f0 + (sl + 1) * S);
      if (k1 - k0 > tt::NKMAX) ok = false;
      out.push_back(TrunkTile{q0, k0, f0, f1, (int32_t)nq, (int32_t)(k1 - k0)});
    }
  }
  if (!ok) out.clear();
  return ok;
}

void trunk_attention_tc(const float* q, const float* k, const float* v, int64_t ld, int n_head,
                        int d_head, int S, const TrunkTile* tiles_dev, int64_t num_tiles,
                        float* out, int64_t ldo, cudaStream_t st) {
  if (num_tiles <= 0) return;
  GO_CHECK(d_head <= 15, "tensor-core trunk attention needs d_head <= 15");
  const float qscale = (float)(1.4426950408889634 / std::sqrt((double)d_head));
  // 64 KB of (unused) dynamic shared memory caps residency at the two CTAs per SM
  // whose 256-column TMEM allocations fit, so no resident CTA spins in tcgen05.alloc
  constexpr int PAD = 64 * 1024;
  static bool attr = false;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(tt::trunk_attn_tc_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, PAD));
    attr = true;
  }
  dim3 grid((unsigned)num_tiles, (unsigned)n_head);
  tt::trunk_attn_tc_kernel<<<grid, tt::THREADS, PAD, st>>>(q, k, v, ld, d_head, S, qscale,
                                                           tiles_dev, out, ldo);
  LAUNCH_CHECK();
}

}  // namespace go
