// Weight gradients of the PPO tape on the 5th-generation tensor cores:
//   dW[K1+K2, N] += [A1 | A2]^T dY,   db[N] += sum_rows dY
// (tensor.py:158-165 affine backward, the gradient of every dense layer of the policy).
//
// The reduction runs over the rows of a minibatch (up to 20 x 80,001 at cfg5), so the GEMM is
// split along the rows: CTA (chunk, n-tile, m-tile) accumulates a 128-feature x NT-column tile
// of its row chunk in TMEM and writes it to a partial buffer; a second kernel sums the
// chunks in a fixed order into dW (deterministic, no atomics).
//
// Per CTA, 5 warps: warps 0-3 stage 32-row steps into a 2-stage shared-memory ring -- each
// thread owns one feature (A) and one column (dY), loads 4 rows per pass (coalesced across
// the warp, any leading dimension: the attention output has ld = 45), splits every value
// into tf32 hi + lo and stores them as one 16-byte K-major core-matrix row -- and warp 4
// issues the MMAs: tcgen05 kind::tf32, M = 128 features, N = NT columns, K = 8 rows per
// instruction, three products per K step (A_hi dY_hi + A_hi dY_lo + A_lo dY_hi: fp32-class
// results, no range limits).  The accumulator is double-buffered in TMEM and drained every
// GROUP steps (1,024 rows) into an IEEE fp32 sum in shared memory by the staging warps, so
// the tensor core's accumulate never sums more than 384 MMAs (its fp32 accumulate does not
// round to nearest; see tc_attention16.cu).
#include <algorithm>
#include <cstring>

#include "engine.cuh"
#include "tcgen05.cuh"
#include "train.cuh"

namespace go {
namespace wg {

using namespace ptx;

constexpr int MT = 128;     // features per CTA (MMA M)
constexpr int KS = 32;      // rows per pipeline step
constexpr int NSTAGE = 2;   // shared-memory ring depth
constexpr int GROUP = 32;   // steps per TMEM accumulation group
constexpr int STAGE_THREADS = 128;
constexpr int THREADS = STAGE_THREADS + 32;

template <int NT>
struct Smem {
  // K-major canonical (no swizzle): element (row m, k) at
  // (k >> 2) * (ROWS * 4) + (m >> 3) * 32 + (m & 7) * 4 + (k & 3) floats
  float a[NSTAGE][2][KS * MT];
  float d[NSTAGE][2][KS * NT];
  float acc[NT][MT];  // drained groups, [column][feature]
  uint64_t full[NSTAGE], empty[NSTAGE], acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};

template <int NT>
constexpr uint32_t tmem_cols() {
  return 2 * NT <= 32 ? 32 : 2 * NT <= 64 ? 64 : 2 * NT <= 128 ? 128 : 256;
}

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = tf32_rn(x);
  lo = tf32_rn(x - hi);
}

template <int NT>
__global__ void __launch_bounds__(THREADS) wgrad_tc_kernel(
    const float* __restrict__ A1, int64_t lda1, int K1, const float* __restrict__ A2,
    int64_t lda2, int K2, const float* __restrict__ dY, int64_t ldd, int64_t M, int N,
    int64_t rows_per_chunk, float* __restrict__ part, float* __restrict__ part_b) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<NT>& sm = *reinterpret_cast<Smem<NT>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int Kin = K1 + K2;
  const int64_t c = blockIdx.x;
  const int n0 = blockIdx.y * NT, m0 = blockIdx.z * MT;
  const int64_t r_begin = c * rows_per_chunk;
  const int64_t r_end = min(M, r_begin + rows_per_chunk);
  const int steps = (int)((r_end - r_begin + KS - 1) / KS);
  const int groups = (steps + GROUP - 1) / GROUP;
  constexpr uint32_t TCOLS = tmem_cols<NT>();
  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&sm.full[s], STAGE_THREADS);
      mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.acc_full[b], 1);
      mbar_init(&sm.acc_empty[b], STAGE_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < NT * MT; i += THREADS) (&sm.acc[0][0])[i] = 0.f;
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp == 4) {
    if ((tid & 31) == 0) {
      constexpr uint32_t ID = idesc_tf32(MT, NT);
      for (int j = 0; j < steps; ++j) {
        const int s = j % NSTAGE, g = j / GROUP, buf = g & 1;
        if (j % GROUP == 0 && g >= 2) mbar_wait(&sm.acc_empty[buf], ((g >> 1) - 1) & 1);
        mbar_wait(&sm.full[s], (j / NSTAGE) & 1);
        fence_after();
        const uint32_t d = tbase + buf * NT;
        const uint32_t ah = smem_u32(sm.a[s][0]), al = smem_u32(sm.a[s][1]);
        const uint32_t dh = smem_u32(sm.d[s][0]), dl = smem_u32(sm.d[s][1]);
#pragma unroll
        for (int kk = 0; kk < KS / 8; ++kk) {
          const uint32_t ao = kk * 2 * (MT * 16), bo = kk * 2 * (NT * 16);
          const uint64_t a_hi = sdesc(ah + ao, MT * 16, 128), a_lo = sdesc(al + ao, MT * 16, 128);
          const uint64_t b_hi = sdesc(dh + bo, NT * 16, 128), b_lo = sdesc(dl + bo, NT * 16, 128);
          umma_ss(d, a_hi, b_hi, ID, (j % GROUP != 0 || kk > 0));
          umma_ss(d, a_hi, b_lo, ID, 1);
          umma_ss(d, a_lo, b_hi, ID, 1);
        }
        umma_commit(&sm.empty[s]);
        if ((j + 1) % GROUP == 0 || j + 1 == steps) umma_commit(&sm.acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // staging: thread = feature m (A) and column n (dY, tid < NT)
    const int m = tid, n = tid;
    const int k = m0 + m, col = n0 + n;
    const float* pa = nullptr;
    int64_t lda = 0;
    if (k < K1) {
      pa = A1 + k;
      lda = lda1;
    } else if (k < Kin) {
      pa = A2 + (k - K1);
      lda = lda2;
    }
    const float* pd = (n < NT && col < N) ? dY + col : nullptr;
    float colsum = 0.f;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    auto drain = [&](int g) {
      const int buf = g & 1;
      mbar_wait(&sm.acc_full[buf], (g >> 1) & 1);
      fence_after();
#pragma unroll 1
      for (int c16 = 0; c16 < NT; c16 += 16) {
        uint32_t r[16];
        PTX_LD16(tbase + lane_off + buf * NT + c16, r);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 16; ++q) sm.acc[c16 + q][m] += __uint_as_float(r[q]);
      }
      fence_before();
      mbar_arrive(&sm.acc_empty[buf]);
    };
    for (int j = 0; j < steps; ++j) {
      const int s = j % NSTAGE;
      if (j >= NSTAGE) mbar_wait(&sm.empty[s], ((j / NSTAGE) - 1) & 1);
      if (j % GROUP == 0 && j > 0) drain(j / GROUP - 1);
      const int64_t r0 = r_begin + (int64_t)j * KS;
      float va[KS], vd[KS];
#pragma unroll
      for (int i = 0; i < KS; ++i) {
        const int64_t r = r0 + i;
        const bool ok = r < r_end;
        va[i] = (pa && ok) ? __ldg(pa + r * lda) : 0.f;
        vd[i] = (pd && ok) ? __ldg(pd + r * ldd) : 0.f;
      }
      float* ahi = sm.a[s][0];
      float* alo = sm.a[s][1];
      const int ao = (m >> 3) * 32 + (m & 7) * 4;
#pragma unroll
      for (int q = 0; q < KS / 4; ++q) {
        float4 h, l;
        split_tf32(va[4 * q], h.x, l.x);
        split_tf32(va[4 * q + 1], h.y, l.y);
        split_tf32(va[4 * q + 2], h.z, l.z);
        split_tf32(va[4 * q + 3], h.w, l.w);
        *reinterpret_cast<float4*>(ahi + q * (MT * 4) + ao) = h;
        *reinterpret_cast<float4*>(alo + q * (MT * 4) + ao) = l;
      }
      if (n < NT) {
        float* dhi = sm.d[s][0];
        float* dlo = sm.d[s][1];
        const int bo = (n >> 3) * 32 + (n & 7) * 4;
#pragma unroll
        for (int q = 0; q < KS / 4; ++q) {
          float4 h, l;
          split_tf32(vd[4 * q], h.x, l.x);
          split_tf32(vd[4 * q + 1], h.y, l.y);
          split_tf32(vd[4 * q + 2], h.z, l.z);
          split_tf32(vd[4 * q + 3], h.w, l.w);
          *reinterpret_cast<float4*>(dhi + q * (NT * 4) + bo) = h;
          *reinterpret_cast<float4*>(dlo + q * (NT * 4) + bo) = l;
        }
        if (part_b)
#pragma unroll
          for (int i = 0; i < KS; ++i) colsum += vd[i];
      }
      fence_async_smem();
      mbar_arrive(&sm.full[s]);
    }
    if (groups > 0) drain(groups - 1);
    // partial tile -> part[c][col][k] (coalesced over the features)
    if (k < Kin)
      for (int q = 0; q < NT; ++q)
        if (n0 + q < N) part[(c * N + n0 + q) * (int64_t)Kin + k] = sm.acc[q][m];
    if (part_b && blockIdx.z == 0 && pd) part_b[c * N + col] = colsum;
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 4) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                 "r"(TCOLS));
  }
}

// dW[k][n] += sum_c part[c][n][k], db[n] += sum_c part_b[c][n], chunks in order
__global__ void wgrad_reduce_kernel(const float* __restrict__ part,
                                    const float* __restrict__ part_b, int64_t chunks, int Kin,
                                    int N, float* __restrict__ dW, int64_t ldw,
                                    float* __restrict__ db) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)N * Kin;
  if (idx < total) {
    const int n = (int)(idx / Kin), k = (int)(idx % Kin);
    float s = 0.f;
    for (int64_t c = 0; c < chunks; ++c) s += part[c * total + idx];
    dW[(int64_t)k * ldw + n] += s;
  }
  if (db && idx < N) {
    float s = 0.f;
    for (int64_t c = 0; c < chunks; ++c) s += part_b[c * N + idx];
    db[idx] += s;
  }
}

template <int NT>
void launch(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
            const float* dY, int64_t ldd, int64_t M, int N, float* dW, float* db,
            cudaStream_t st) {
  static bool attr = false;
  const size_t smem = sizeof(Smem<NT>) + 1024;
  if (!attr) {
    CUDA_CHECK(cudaFuncSetAttribute(wgrad_tc_kernel<NT>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int Kin = K1 + K2;
  const int mt = (int)cdiv(Kin, MT), nt = (int)cdiv(N, NT);
  // enough CTAs to fill the SMs twice, rows per chunk a multiple of the step
  const int64_t want = std::max<int64_t>(1, (2 * num_sms()) / (mt * nt));
  int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(want, cdiv(M, 4 * KS)));
  const int64_t rpc = round_up(cdiv(M, chunks), KS);
  chunks = cdiv(M, rpc);
  float* part = nullptr;
  const size_t pbytes = (size_t)chunks * N * Kin * sizeof(float);
  const size_t bbytes = db ? (size_t)chunks * N * sizeof(float) : 0;
  CUDA_CHECK(cudaMallocAsync(&part, pbytes + bbytes + 16, st));
  float* part_b = db ? part + (size_t)chunks * N * Kin : nullptr;
  dim3 grid((unsigned)chunks, (unsigned)nt, (unsigned)mt);
  wgrad_tc_kernel<NT><<<grid, THREADS, smem, st>>>(A1, lda1, K1, A2, lda2, K2, dY, ldd, M, N,
                                                   rpc, part, part_b);
  LAUNCH_CHECK();
  const int64_t total = std::max<int64_t>((int64_t)N * Kin, N);
  wgrad_reduce_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(part, part_b, chunks, Kin, N,
                                                                  dW, N, db);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaFreeAsync(part, st));
}

}  // namespace wg

void wgrad_tc(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
              const float* dY, int64_t ldd, int64_t M, int N, float* dW, float* db,
              cudaStream_t st) {
  if (M <= 0 || N <= 0 || (K1 + K2) <= 0) return;
  if (N <= 16) wg::launch<16>(A1, lda1, K1, A2, lda2, K2, dY, ldd, M, N, dW, db, st);
  else if (N <= 48) wg::launch<48>(A1, lda1, K1, A2, lda2, K2, dY, ldd, M, N, dW, db, st);
  else wg::launch<128>(A1, lda1, K1, A2, lda2, K2, dY, ldd, M, N, dW, db, st);
}

}  // namespace go
