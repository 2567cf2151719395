// Segmented (block-banded) trunk attention on the 5th-generation tensor cores
// (policy.py:157-177: the queries of segment s attend to the keys of segments s-1 and
// s of the same forward; multi_head_attention / scaled_dot_attention, tensor.py:382-388).
//
// One CTA = 128 consecutive query rows of one forward (an M=128 tile spanning 128/S
// segments), all heads, and the union of the rows' key windows (<= 192 keys; 192 for
// the default S = 64), 5 warps:
//   all warps  stage Q (scaled by log2(e)/sqrt(d_head)), K and V^T of every head in
//              shared memory as fp16 in the UMMA K-major canonical layout, reading each
//              QKV row once; V[:,15] = 1 so the PV MMA also returns the row sums;
//   warp 4     per head: S = Q K^T (kind::f16, M=128, N=keys, K=16) into TMEM, then,
//              once P is back in TMEM, O_h = P V (M=128, N=16, K=keys, A = P from TMEM);
//   warps 0-3  one query row per thread: exact max over the row's own window (keys
//              outside it get P = 0), P = 2^(s - max) packed fp16x2 over S.
// fp16 carries tf32's 10 mantissa bits; P <= 1 with an exact row max, so only terms
// below 2^-14 of the largest lose relative precision.  Operands outside the fp16 range
// set a flag and the SIMT kernel re-runs the launch (gated on that flag).
#include <algorithm>
#include <cmath>
#include <cuda_fp16.h>

#include "engine.cuh"
#include "tcgen05.cuh"

namespace go {
namespace tt {

using namespace ptx;

constexpr int QT = 128;
constexpr int KMAX = TRUNK_TC_MAX_KEYS;  // 192
constexpr int HMAX = 3;
constexpr uint32_t O_COL = KMAX;         // O_h at O_COL + 16 h
constexpr uint32_t TMEM_COLS = 256;
constexpr int THREADS = 160;
constexpr float RANGE_LIMIT = 60000.f;

struct Smem {
  __half q[HMAX][QT * 16];
  __half k[HMAX][KMAX * 16];
  __half vt[HMAX][KMAX * 16];
  uint64_t bar_s, bar_p, bar_o;
  uint32_t tmem;
};

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__global__ void __launch_bounds__(THREADS) trunk_attn_tc_kernel(
    const float* __restrict__ qkv, int64_t ld, int n_head, int d_head, int S, float qscale,
    const TrunkTile* __restrict__ tiles, float* __restrict__ out, int64_t ldo,
    int32_t* __restrict__ flag) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const TrunkTile T = tiles[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NKP = (T.nk + 15) & ~15;
  const int W = n_head * d_head;
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
  // ---- staging: a warp per row, a lane per column (head / dim fixed per lane, so no
  // division in the loops), 4 rows in flight per warp; padding columns d_head..15 are
  // written by the lanes past the row width
  bool big = false;
  {
    constexpr int NW = THREADS / 32;
    const int RW = n_head * 16;  // padded row width (all heads)
    // Q: lanes cover the padded width in passes of 32
    for (int cb = 0; cb < RW; cb += 32) {
      const int cp = cb + lane;  // padded column: head cp / 16, dim cp % 16
      const int h = cp >> 4, d = cp & 15;
      const bool real = cp < RW && d < d_head;
      const int c = h * d_head + d;
#pragma unroll 4
      for (int r = warp; r < QT; r += NW) {
        float x = 0.f;
        if (real && r < T.nq) {
          x = qkv[(T.q0 + r) * ld + c] * qscale;
          big |= !(fabsf(x) <= RANGE_LIMIT);
        }
        if (cp < RW)
          sm.q[h][(d >> 3) * (QT * 8) + (r >> 3) * 64 + (r & 7) * 8 + (d & 7)] = __float2half_rn(x);
      }
    }
    for (int cb = 0; cb < RW; cb += 32) {
      const int cp = cb + lane;
      const int h = cp >> 4, d = cp & 15;
      const bool real = cp < RW && d < d_head;
      const int c = h * d_head + d;
#pragma unroll 4
      for (int r = warp; r < NKP; r += NW) {
        float kx = 0.f, vx = 0.f;
        if (r < T.nk) {
          if (real) {
            kx = qkv[(T.k0 + r) * ld + W + c];
            vx = qkv[(T.k0 + r) * ld + 2 * W + c];
            big |= !(fabsf(kx) <= RANGE_LIMIT) || !(fabsf(vx) <= RANGE_LIMIT);
          } else if (d == 15) {
            vx = 1.f;  // V[:,15] = 1: the PV MMA returns the row sum in O[:,15]
          }
        }
        if (cp < RW) {
          sm.k[h][(d >> 3) * (KMAX * 8) + (r >> 3) * 64 + (r & 7) * 8 + (d & 7)] = __float2half_rn(kx);
          sm.vt[h][(r >> 3) * 128 + (d >> 3) * 64 + (d & 7) * 8 + (r & 7)] = __float2half_rn(vx);
        }
      }
    }
  }
  if (big) atomicOr(flag, 1);
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = sm.tmem;

  if (warp == 4) {
    if (lane == 0) {
      const uint32_t id_s = idesc_f16(QT, NKP);
      constexpr uint32_t id_o = idesc_f16(QT, 16);
      for (int h = 0; h < n_head; ++h) {
        // S_h overwrites P_{h-1}: the in-order tensor pipe has consumed it by then
        umma_ss_f16(tbase, sdesc(smem_u32(sm.q[h]), QT * 16, 128),
                    sdesc(smem_u32(sm.k[h]), KMAX * 16, 128), id_s, 0);
        umma_commit(&sm.bar_s);
        mbar_wait(&sm.bar_p, h & 1);
        fence_after();
        const uint32_t va = smem_u32(sm.vt[h]);
        for (int kk = 0; kk < NKP / 16; ++kk)
          umma_ts_f16(tbase + O_COL + 16 * h, tbase + kk * 8, sdesc(va + kk * 512, 256, 128),
                      id_o, kk > 0);
      }
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
    for (int h = 0; h < n_head; ++h) {
      mbar_wait(&sm.bar_s, h & 1);
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
      // P for columns [cb, cb + 16) -> packed columns [cb/2, cb/2 + 8): already read
      for (int cb = 0; cb < NKP; cb += 16) {
        uint32_t u[16], pk[8];
        PTX_LD16(tbase + lane_off + cb, u);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = cb + 2 * j;
          const float p0 = (c >= c0 && c < c1) ? ex2f(__uint_as_float(u[2 * j]) - m) : 0.f;
          const float p1 = (c + 1 >= c0 && c + 1 < c1) ? ex2f(__uint_as_float(u[2 * j + 1]) - m) : 0.f;
          pk[j] = pack_f16x2(p0, p1);
        }
        PTX_ST8(tbase + lane_off + cb / 2, pk);
      }
      tmem_wait_st();
      fence_before();
      mbar_arrive(&sm.bar_p);
    }
    mbar_wait(&sm.bar_o, 0);
    fence_after();
    for (int h = 0; h < n_head; ++h) {
      uint32_t o[16];
      PTX_LD16(tbase + lane_off + O_COL + 16 * h, o);
      tmem_wait_ld();
      if (active) {
        const float inv = 1.f / __uint_as_float(o[15]);
        float* dst = out + row * ldo + (int64_t)h * d_head;
        for (int d = 0; d < d_head; ++d) dst[d] = __uint_as_float(o[d]) * inv;
      }
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
      if (k1 - k0 > tt::KMAX) ok = false;
      out.push_back(TrunkTile{q0, k0, f0, f1, (int32_t)nq, (int32_t)(k1 - k0)});
    }
  }
  if (!ok) out.clear();
  return ok;
}

bool trunk_tc_supported(int n_head, int d_head) {
  return n_head <= tt::HMAX && d_head <= 15;
}

void trunk_attention_tc(const float* qkv, int64_t ld, int n_head, int d_head, int S,
                        const TrunkTile* tiles_dev, int64_t num_tiles, float* out, int64_t ldo,
                        int32_t* flag, cudaStream_t st) {
  if (num_tiles <= 0) return;
  GO_CHECK(trunk_tc_supported(n_head, d_head), "tensor-core trunk attention: unsupported heads");
  const float qscale = (float)(1.4426950408889634 / std::sqrt((double)d_head));
  // dynamic shared memory padded so at most two CTAs share an SM: their two 256-column
  // TMEM allocations fill it, and no resident CTA spins in tcgen05.alloc
  constexpr int SMEM = 100 * 1024;
  static_assert(sizeof(tt::Smem) <= SMEM, "trunk attention smem");
  static bool attr = false;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(tt::trunk_attn_tc_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    attr = true;
  }
  tt::trunk_attn_tc_kernel<<<(unsigned)num_tiles, tt::THREADS, SMEM, st>>>(
      qkv, ld, n_head, d_head, S, qscale, tiles_dev, out, ldo, flag);
  LAUNCH_CHECK();
}

}  // namespace go
