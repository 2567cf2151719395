// Attention backward on warp-level tensor-core MMAs (the PPO tape's reverse of
// multi_head_attention / scaled_dot_attention, tensor.py:382-388, for both the
// block-banded trunk, policy.py:157-177, and the full N x N task-head attention,
// policy.py:196-203).  FA2-style recomputation from the saved log2-sum-exp:
//   P = exp2(s2 - lse2), s2 = q.k * log2(e)/sqrt(d)
//   D_i = dO_i . O_i ; dS = P (dO.v - D) ; dq = scale sum_j dS k_j ;
//   dk = scale sum_i dS q_i ; dv = sum_i P dO_i
// Two kernels, both mma.sync.m16n8k16 (fp16 operands, fp32 accumulation), d_head <= 16:
//   dq  : query-major, CTA = 64 queries x head; per 64-key chunk S = Q K^T and
//         G = dO V^T (8 + 8 MMAs per warp), dS in registers, dq += dS K (8 MMAs);
//   dkv : key-major, CTA = 64 keys x head; per 64-query chunk S^T = K Q^T and
//         G^T = V dO^T, dv += P^T dO and dk += dS^T Q (the C fragments of S^T / G^T are
//         reused directly as the A fragments of P^T / dS^T; the B fragments of dO / Q /
//         K come from the row-major staged chunk through ldmatrix.trans).
// Chunks are staged with double-buffered cp.async; a forward kernel (fwd_kernel, with
// the log2-sum-exp) shares the packed operands.
// Operands are pre-packed once per call into fp16 rows ([H][M][32]: hi and lo halves of
// a 2-term split, three MMAs per product, so the gradients stay fp32-class): Q pre-scaled by log2(e)/sqrt(d), dO by a power of two
// that brings max|dO| into [0.5, 1) (gradients are far below fp16's normal range
// otherwise; undone exactly on output).  P and dS are split the same way in registers,
// scaled by powers of two (2^15 for P <= 1, 2^(14 - ceil log2 bound) for dS) so small
// values keep fp16-normal hi and lo terms instead of the subnormals' fixed 2^-24 step,
// which summed over 80k keys is otherwise the dominant error.
// Anything outside the fp16 range (or a non-finite dS) sets *flag and the caller re-runs
// the fp32 SIMT kernels gated on it.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cuda_fp16.h>

#include "train.cuh"

namespace go {
namespace ab {

constexpr int TS = 64;      // rows per tile / chunk
constexpr float RANGE = 60000.f;
constexpr float PSCALE = 32768.f;  // P (<= 1) enters the MMAs as 2^15 P (fp16-normal)

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
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t ld32(const __half* p) {
  return *reinterpret_cast<const uint32_t*>(p);
}

// max |dO| over the head columns (non-negative floats order like their bit patterns)
__global__ void absmax_kernel(const float* __restrict__ x, int64_t ld, int64_t M, int W,
                              unsigned* __restrict__ out, const int32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;  // gated: only when the tcgen05 tape flagged the call
  float m = 0.f;
  const int64_t n = M * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / W;
    const float a = fabsf(x[r * ld + (i - r * W)]);
    m = a > m || a != a ? a : m;  // keep NaN visible
  }
  for (int o = 16; o; o >>= 1) {
    const float t = __shfl_xor_sync(0xffffffffu, m, o);
    m = t > m || t != t ? t : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

__device__ __forceinline__ float grad_scale(const unsigned* bits) {
  const float m = __uint_as_float(*bits);
  if (!(m > 0.f) || !(m <= 3.0e38f)) return 1.f;
  return exp2f(-ceilf(log2f(m)));  // power of two: max|dO| * gs in [0.5, 1]
}

// fp16 rows per head: Q*qscale, K, V, dO*gs -> [H][M][RW]; with SPLIT each value is
// stored as hi = fp16(x) in halves 0..15 and lo = fp16(x - hi) in halves 16..31, so
// three MMAs (hi.hi + hi.lo + lo.hi) give products to ~2^-21 relative (fp32-class:
// Adam turns gradient noise on near-zero coordinates into full +-lr steps, so the
// update needs the fp32-level gradient the SIMT kernels give).
template <bool SPLIT>
__global__ void pack_kernel(const float* __restrict__ q, const float* __restrict__ k,
                            const float* __restrict__ v, const float* __restrict__ dO, int64_t ld,
                            int64_t M, int n_head, int d_head, float qscale,
                            const unsigned* __restrict__ gbits, __half* __restrict__ Qh,
                            __half* __restrict__ Kh, __half* __restrict__ Vh,
                            __half* __restrict__ Oh, int32_t* __restrict__ flag,
                            const int32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;
  constexpr int RW = SPLIT ? 32 : 16;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (head, row)
  if (i >= M * n_head) return;
  const int h = (int)(i / M);
  const int64_t r = i - (int64_t)h * M;
  const float gs = grad_scale(gbits);
  const int64_t src = r * ld + (int64_t)h * d_head;
  bool big = false;
  float nrm[4] = {0.f, 0.f, 0.f, 0.f};
  const float* srcs[4] = {q, k, v, dO};
  const float mul[4] = {qscale, 1.f, 1.f, gs};
  __half* dsts[4] = {Qh, Kh, Vh, Oh};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (srcs[t] == nullptr) continue;  // forward: no dO
    __align__(16) __half row[RW];
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      // V carries a ones column at d_head: the forward's MMAs accumulate the softmax row
      // sum next to O (dO's column d_head is 0, so the backward products ignore it)
      float x = d < d_head ? srcs[t][src + d] * mul[t] : (t == 2 && d == d_head ? 1.f : 0.f);
      big |= !(fabsf(x) <= RANGE);
      nrm[t] = fmaf(x, x, nrm[t]);
      row[d] = __float2half_rn(x);
      if (SPLIT) row[16 + d] = __float2half_rn(x - __half2float(row[d]));
    }
    uint4* o = reinterpret_cast<uint4*>(dsts[t] + i * RW);
#pragma unroll
    for (int j = 0; j < RW / 8; ++j) o[j] = reinterpret_cast<const uint4*>(row)[j];
  }
  // max row norms of V and of the scaled dO: |dO_q.(v_k - o_q)| <= 2 |dO_q| max|v| bounds dS
  atomicMax(const_cast<unsigned*>(gbits) + 1, __float_as_uint(sqrtf(nrm[2])));
  atomicMax(const_cast<unsigned*>(gbits) + 2, __float_as_uint(sqrtf(nrm[3])));
  if (big) atomicOr(flag, 1);
}

// power-of-two scale bringing the dS bound to 2^14 (fp16-normal hi/lo terms for small dS)
__device__ __forceinline__ float ds_scale(const unsigned* gbits) {
  const float b = 2.f * __uint_as_float(gbits[1]) * __uint_as_float(gbits[2]);
  if (!(b > 0.f) || !(b <= 3.0e38f)) return 1.f;
  return exp2f(fminf(14.f - ceilf(log2f(b)), 60.f));
}

template <bool SPLIT>
struct Frag {  // A fragment (16 rows x 16 dims), hi and (SPLIT) lo parts
  uint32_t h[4], l[4];
};

// A fragment of a packed row block: rows r0 = base+g, r1 = base+g+8
template <bool SPLIT>
__device__ __forceinline__ void load_afrag(const __half* __restrict__ X, int64_t r0, int64_t r1,
                                           int64_t lim, int tq, Frag<SPLIT>& a) {
  constexpr int RW = SPLIT ? 32 : 16;
#pragma unroll
  for (int p = 0; p < (SPLIT ? 2 : 1); ++p) {
    uint32_t* d = p ? a.l : a.h;
    const int c = p * 16 + 2 * tq;
    d[0] = r0 < lim ? ld32(X + r0 * RW + c) : 0u;
    d[1] = r1 < lim ? ld32(X + r1 * RW + c) : 0u;
    d[2] = r0 < lim ? ld32(X + r0 * RW + c + 8) : 0u;
    d[3] = r1 < lim ? ld32(X + r1 * RW + c + 8) : 0u;
  }
}

// C += A B with B's (k = 16, n = 8) fragment at b (hi) / bl (lo)
template <bool SPLIT>
__device__ __forceinline__ void mma3(float* c, const Frag<SPLIT>& a, uint32_t b0, uint32_t b1,
                                     uint32_t l0, uint32_t l1) {
  if (SPLIT) {
    mma16816(c, a.l, b0, b1);
    mma16816(c, a.h, l0, l1);
  }
  mma16816(c, a.h, b0, b1);
}

// split a pair of fp32 values into fp16x2 hi and lo
template <bool SPLIT>
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  hi = pack2(x0, x1);
  if (SPLIT) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&hi));
    lo = pack2(x0 - f.x, x1 - f.y);
  }
}

template <bool SPLIT>
constexpr int row_stride() { return SPLIT ? 40 : 24; }  // halves; conflict-free fragments

// asynchronous staging (cp.async, zero-filled rows past n) into one of two buffers, so
// the next chunk's rows load while this chunk computes
template <bool SPLIT>
__device__ __forceinline__ void stage_cp(const __half* __restrict__ X,
                                         const __half* __restrict__ Y, int64_t c, int n,
                                         __half* Xs, __half* Ys, int tid) {
  constexpr int RW = SPLIT ? 32 : 16, RS2 = row_stride<SPLIT>();
  const int row = tid >> 1, half = (tid & 1) * 8;
  const bool ok = row < n;
  const int64_t r = ok ? c + row : 0;
#pragma unroll
  for (int p = 0; p < (SPLIT ? 2 : 1); ++p) {
    const uint32_t xs = static_cast<uint32_t>(__cvta_generic_to_shared(Xs + row * RS2 + p * 16 + half));
    const uint32_t ys = static_cast<uint32_t>(__cvta_generic_to_shared(Ys + row * RS2 + p * 16 + half));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(xs),
                 "l"(X + r * RW + p * 16 + half), "r"(ok ? 16 : 0));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ys),
                 "l"(Y + r * RW + p * 16 + half), "r"(ok ? 16 : 0));
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// B fragments (k = 16 rows of a row-major [row][dim] smem block, n = 8 dims) for both
// n-tiles of a k-step straight from the row-major block: ldmatrix.x4.trans, lanes 0-7 /
// 8-15 / 16-23 / 24-31 address rows 0-7 / 8-15 (dims 0-7), rows 0-7 / 8-15 (dims 8-15);
// b[0], b[1] = n-tile 0's (b0, b1), b[2], b[3] = n-tile 1's.  Replaces a transposed copy.
__device__ __forceinline__ void ldsm_bT(const __half* blk, int stride, int lane, uint32_t* b) {
  const __half* p = blk + ((lane & 7) + ((lane >> 3) & 1) * 8) * stride + (lane >> 4) * 8;
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}

template <bool SPLIT>
__global__ void __launch_bounds__(128) dq_kernel(
    const __half* __restrict__ Qh, const __half* __restrict__ Kh, const __half* __restrict__ Vh,
    const __half* __restrict__ Oh, int64_t M, const float* __restrict__ lse,
    const float* __restrict__ Dv, int n_head, int d_head, const AttnTile* __restrict__ tiles,
    float* __restrict__ dq, int64_t ld, float scale, const unsigned* __restrict__ gbits,
    int32_t* __restrict__ flag, const int32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;
  constexpr int RW = SPLIT ? 32 : 16, RS2 = row_stride<SPLIT>();
  __shared__ __align__(16) __half Ks2[2][TS * RS2];
  __shared__ __align__(16) __half Vs2[2][TS * RS2];
  const AttnTile tl = tiles[blockIdx.x];
  const int h = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
  const __half* Q = Qh + (int64_t)h * M * RW;
  const __half* K = Kh + (int64_t)h * M * RW;
  const __half* V = Vh + (int64_t)h * M * RW;
  const __half* O = Oh + (int64_t)h * M * RW;
  const float gs = grad_scale(gbits);
  const int64_t r0 = tl.q0 + warp * 16 + g, r1 = r0 + 8;
  Frag<SPLIT> qa, oa;
  load_afrag<SPLIT>(Q, r0, r1, tl.q1, tq, qa);
  load_afrag<SPLIT>(O, r0, r1, tl.q1, tq, oa);
  const float l0 = r0 < tl.q1 ? lse[r0 * n_head + h] : 0.f;
  const float l1 = r1 < tl.q1 ? lse[r1 * n_head + h] : 0.f;
  const float D0 = r0 < tl.q1 ? Dv[r0 * n_head + h] * gs : 0.f;
  const float D1 = r1 < tl.q1 ? Dv[r1 * n_head + h] * gs : 0.f;
  const float dsc = SPLIT ? ds_scale(gbits) : 1.f;
  float acc[2][4] = {};
  bool bad = false;
  if (tl.k0 < tl.k1)
    stage_cp<SPLIT>(K, V, tl.k0, (tl.k1 - tl.k0) < TS ? (int)(tl.k1 - tl.k0) : TS, Ks2[0],
                    Vs2[0], tid);
  int buf = 0;
  for (int64_t kc = tl.k0; kc < tl.k1; kc += TS, buf ^= 1) {
    const int nk = (tl.k1 - kc) < TS ? (int)(tl.k1 - kc) : TS;
    const int64_t kn = kc + TS;
    if (kn < tl.k1) {
      stage_cp<SPLIT>(K, V, kn, (tl.k1 - kn) < TS ? (int)(tl.k1 - kn) : TS, Ks2[buf ^ 1],
                      Vs2[buf ^ 1], tid);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const __half* Ks = Ks2[buf];
    const __half* Vs = Vs2[buf];
    // streamed per 16-key k-step: S and G for its two n-tiles, dS as the A fragment, then
    // the dq MMAs; per-chunk MMA sums are added to acc with IEEE FADDs (two-level
    // accumulation: the MMA's fp32 accumulate drops the low bits of small addends with a
    // consistent sign)
    float cacc[2][4] = {};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      Frag<SPLIT> pa;
#pragma unroll
      for (int hn = 0; hn < 2; ++hn) {
        const int n = 2 * kk + hn;
        float s[4] = {0.f, 0.f, 0.f, 0.f}, gg[4] = {0.f, 0.f, 0.f, 0.f};
        const __half* kp = &Ks[(8 * n + g) * RS2 + 2 * tq];
        const __half* vp = &Vs[(8 * n + g) * RS2 + 2 * tq];
        mma3<SPLIT>(s, qa, ld32(kp), ld32(kp + 8), SPLIT ? ld32(kp + 16) : 0u,
                    SPLIT ? ld32(kp + 24) : 0u);
        mma3<SPLIT>(gg, oa, ld32(vp), ld32(vp + 8), SPLIT ? ld32(vp + 16) : 0u,
                    SPLIT ? ld32(vp + 24) : 0u);
        const int key = 8 * n + 2 * tq;
        float ds[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool ok = key + (e & 1) < nk;
          const float p = ok ? ex2(s[e] - (e < 2 ? l0 : l1)) : 0.f;
          ds[e] = p * (gg[e] - (e < 2 ? D0 : D1)) * dsc;
          bad |= !(fabsf(ds[e]) <= RANGE);
        }
        // n-tile 2kk + hn is half hn of the k-step: A regs {0,1} or {2,3}
        const int j = hn * 2;
        split2<SPLIT>(ds[0], ds[1], pa.h[j], pa.l[j]);
        split2<SPLIT>(ds[2], ds[3], pa.h[j + 1], pa.l[j + 1]);
      }
      uint32_t bh[4], bl[4] = {0u, 0u, 0u, 0u};
      ldsm_bT(Ks + 16 * kk * RS2, RS2, lane, bh);
      if (SPLIT) ldsm_bT(Ks + 16 * kk * RS2 + 16, RS2, lane, bl);
#pragma unroll
      for (int n = 0; n < 2; ++n)
        mma3<SPLIT>(cacc[n], pa, bh[2 * n], bh[2 * n + 1], bl[2 * n], bl[2 * n + 1]);
    }
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[n][e] += cacc[n][e];
    __syncthreads();  // required: the next iteration's cp.async (into buf ^ 1 of that
                      // iteration, i.e. this `buf`) refills the buffer just read
  }
  const float c = scale / (gs * dsc);
  const int64_t col0 = (int64_t)h * d_head;
#pragma unroll
  for (int n = 0; n < 2; ++n) {
    const int d = 8 * n + 2 * tq;
    if (r0 < tl.q1) {
      if (d < d_head) dq[r0 * ld + col0 + d] = acc[n][0] * c;
      if (d + 1 < d_head) dq[r0 * ld + col0 + d + 1] = acc[n][1] * c;
    }
    if (r1 < tl.q1) {
      if (d < d_head) dq[r1 * ld + col0 + d] = acc[n][2] * c;
      if (d + 1 < d_head) dq[r1 * ld + col0 + d + 1] = acc[n][3] * c;
    }
  }
  if (bad) atomicOr(flag, 1);
}

template <bool SPLIT>
__global__ void __launch_bounds__(128, 4) dkv_kernel(
    const __half* __restrict__ Qh, const __half* __restrict__ Kh, const __half* __restrict__ Vh,
    const __half* __restrict__ Oh, int64_t M, const float* __restrict__ lse,
    const float* __restrict__ Dv, int n_head, int d_head, const KvTile* __restrict__ tiles,
    float* __restrict__ dk_a, float* __restrict__ dv_a, float* __restrict__ dk_b,
    float* __restrict__ dv_b, int64_t ld, float kscale, const unsigned* __restrict__ gbits,
    int32_t* __restrict__ flag, const int32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;
  constexpr int RW = SPLIT ? 32 : 16, RS2 = row_stride<SPLIT>();
  __shared__ __align__(16) __half Qs2[2][TS * RS2];
  __shared__ __align__(16) __half Os2[2][TS * RS2];
  __shared__ __align__(8) float Ls2[2][TS], Dd2[2][TS];
  const KvTile tl = tiles[blockIdx.x];
  const int h = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
  const __half* Q = Qh + (int64_t)h * M * RW;
  const __half* K = Kh + (int64_t)h * M * RW;
  const __half* V = Vh + (int64_t)h * M * RW;
  const __half* O = Oh + (int64_t)h * M * RW;
  const float gs = grad_scale(gbits);
  const int64_t r0 = tl.k0 + warp * 16 + g, r1 = r0 + 8;  // this thread's key rows
  Frag<SPLIT> ka, va;
  load_afrag<SPLIT>(K, r0, r1, tl.k1, tq, ka);
  load_afrag<SPLIT>(V, r0, r1, tl.k1, tq, va);
  bool bad = false;
  const int64_t col0 = (int64_t)h * d_head;
  const float dsc = SPLIT ? ds_scale(gbits) : 1.f;
  const float psc = SPLIT ? PSCALE : 1.f;
  for (int part = 0; part < 2; ++part) {
    const int64_t qa0 = part ? tl.qb0 : tl.qa0, qe = part ? tl.qb1 : tl.qa1;
    float* dko = part ? dk_b : dk_a;
    float* dvo = part ? dv_b : dv_a;
    if (!dko) continue;
    float dk[2][4] = {}, dv[2][4] = {};
    __syncthreads();  // the previous part's last chunk is done with both buffers
    if (qa0 < qe)
      stage_cp<SPLIT>(Q, O, qa0, (qe - qa0) < TS ? (int)(qe - qa0) : TS, Qs2[0], Os2[0], tid);
    int buf = 0;
    for (int64_t qc = qa0; qc < qe; qc += TS, buf ^= 1) {
      const int nq = (qe - qc) < TS ? (int)(qe - qc) : TS;
      const int64_t qn = qc + TS;
      if (qn < qe) {
        stage_cp<SPLIT>(Q, O, qn, (qe - qn) < TS ? (int)(qe - qn) : TS, Qs2[buf ^ 1],
                        Os2[buf ^ 1], tid);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      float* Ls = Ls2[buf];
      float* Dd = Dd2[buf];
      if (tid < TS) Ls[tid] = tid < nq ? lse[(qc + tid) * n_head + h] : 0.f;
      else Dd[tid - TS] = tid - TS < nq ? Dv[(qc + tid - TS) * n_head + h] * gs : 0.f;
      __syncthreads();
      const __half* Qs = Qs2[buf];
      const __half* Os = Os2[buf];
      Frag<SPLIT> pp[4], pd[4];
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        float s[4] = {0.f, 0.f, 0.f, 0.f}, gg[4] = {0.f, 0.f, 0.f, 0.f};
        const __half* qp = &Qs[(8 * n + g) * RS2 + 2 * tq];
        const __half* op = &Os[(8 * n + g) * RS2 + 2 * tq];
        mma3<SPLIT>(s, ka, ld32(qp), ld32(qp + 8), SPLIT ? ld32(qp + 16) : 0u,
                  SPLIT ? ld32(qp + 24) : 0u);   // S^T
        mma3<SPLIT>(gg, va, ld32(op), ld32(op + 8), SPLIT ? ld32(op + 16) : 0u,
                  SPLIT ? ld32(op + 24) : 0u);  // (dO.v)^T
        const int qi = 8 * n + 2 * tq;
        const float2 lq = *reinterpret_cast<const float2*>(&Ls[qi]);
        const float2 dq2 = *reinterpret_cast<const float2*>(&Dd[qi]);
        float p[4], ds[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool ok = qi + (e & 1) < nq;
          p[e] = ok ? ex2(s[e] - ((e & 1) ? lq.y : lq.x)) : 0.f;
          ds[e] = p[e] * (gg[e] - ((e & 1) ? dq2.y : dq2.x)) * dsc;
          p[e] *= psc;
          bad |= !(fabsf(ds[e]) <= RANGE);
        }
        const int j = (n & 1) * 2;
        split2<SPLIT>(p[0], p[1], pp[n >> 1].h[j], pp[n >> 1].l[j]);
        split2<SPLIT>(p[2], p[3], pp[n >> 1].h[j + 1], pp[n >> 1].l[j + 1]);
        split2<SPLIT>(ds[0], ds[1], pd[n >> 1].h[j], pd[n >> 1].l[j]);
        split2<SPLIT>(ds[2], ds[3], pd[n >> 1].h[j + 1], pd[n >> 1].l[j + 1]);
      }
      float cdv[2][4] = {}, cdk[2][4] = {};  // per-chunk sums (two-level accumulation)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t oh[4], ol[4] = {0u, 0u, 0u, 0u}, qh[4], ql[4] = {0u, 0u, 0u, 0u};
        ldsm_bT(Os + 16 * kk * RS2, RS2, lane, oh);
        ldsm_bT(Qs + 16 * kk * RS2, RS2, lane, qh);
        if (SPLIT) {
          ldsm_bT(Os + 16 * kk * RS2 + 16, RS2, lane, ol);
          ldsm_bT(Qs + 16 * kk * RS2 + 16, RS2, lane, ql);
        }
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          mma3<SPLIT>(cdv[n], pp[kk], oh[2 * n], oh[2 * n + 1], ol[2 * n], ol[2 * n + 1]);
          mma3<SPLIT>(cdk[n], pd[kk], qh[2 * n], qh[2 * n + 1], ql[2 * n], ql[2 * n + 1]);
        }
      }
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          dv[n][e] += cdv[n][e];
          dk[n][e] += cdk[n][e];
        }
      __syncthreads();  // required: the next iteration's cp.async (into buf ^ 1 of that
                      // iteration, i.e. this `buf`) refills the buffer just read
    }
    const float cv = 1.f / (gs * psc), ck = kscale / (gs * dsc);
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      const int d = 8 * n + 2 * tq;
      if (r0 < tl.k1) {
        if (d < d_head) {
          dko[r0 * ld + col0 + d] = dk[n][0] * ck;
          dvo[r0 * ld + col0 + d] = dv[n][0] * cv;
        }
        if (d + 1 < d_head) {
          dko[r0 * ld + col0 + d + 1] = dk[n][1] * ck;
          dvo[r0 * ld + col0 + d + 1] = dv[n][1] * cv;
        }
      }
      if (r1 < tl.k1) {
        if (d < d_head) {
          dko[r1 * ld + col0 + d] = dk[n][2] * ck;
          dvo[r1 * ld + col0 + d] = dv[n][2] * cv;
        }
        if (d + 1 < d_head) {
          dko[r1 * ld + col0 + d + 1] = dk[n][3] * ck;
          dvo[r1 * ld + col0 + d + 1] = dv[n][3] * cv;
        }
      }
    }
  }
  if (bad) atomicOr(flag, 1);
}

// forward with log2-sum-exp on the packed operands (the PPO tape's forward of both the
// banded trunk and the N x N head attention): S = Q K^T (3 split MMAs per 8-key n-tile),
// exact online max, P = exp2(S - m) scaled by 2^15 and split, O += P V from the row-major
// V block through ldmatrix.trans, per-chunk sums added with FADDs, row sums from V's ones
// column.  d_head <= 15 (the ones column needs a free slot).
template <bool SPLIT>
__global__ void __launch_bounds__(128) fwd_kernel(
    const __half* __restrict__ Qh, const __half* __restrict__ Kh, const __half* __restrict__ Vh,
    int64_t M, int n_head, int d_head, const AttnTile* __restrict__ tiles,
    float* __restrict__ out, int64_t ldo, float* __restrict__ lse,
    const int32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;
  constexpr int RW = SPLIT ? 32 : 16, RS2 = row_stride<SPLIT>();
  __shared__ __align__(16) __half Ks2[2][TS * RS2];
  __shared__ __align__(16) __half Vs2[2][TS * RS2];
  const AttnTile tl = tiles[blockIdx.x];
  const int h = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
  const __half* Q = Qh + (int64_t)h * M * RW;
  const __half* K = Kh + (int64_t)h * M * RW;
  const __half* V = Vh + (int64_t)h * M * RW;
  const int64_t r0 = tl.q0 + warp * 16 + g, r1 = r0 + 8;
  Frag<SPLIT> qa;
  load_afrag<SPLIT>(Q, r0, r1, tl.q1, tq, qa);
  float o[2][4] = {};
  float m0 = -INFINITY, m1 = -INFINITY;
  const float psc = SPLIT ? PSCALE : 1.f;
  if (tl.k0 < tl.k1)
    stage_cp<SPLIT>(K, V, tl.k0, (tl.k1 - tl.k0) < TS ? (int)(tl.k1 - tl.k0) : TS, Ks2[0],
                    Vs2[0], tid);
  int buf = 0;
  for (int64_t kc = tl.k0; kc < tl.k1; kc += TS, buf ^= 1) {
    const int nk = (tl.k1 - kc) < TS ? (int)(tl.k1 - kc) : TS;
    const int64_t kn = kc + TS;
    if (kn < tl.k1) {
      stage_cp<SPLIT>(K, V, kn, (tl.k1 - kn) < TS ? (int)(tl.k1 - kn) : TS, Ks2[buf ^ 1],
                      Vs2[buf ^ 1], tid);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const __half* Ks = Ks2[buf];
    const __half* Vs = Vs2[buf];
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
      const __half* kp = &Ks[(8 * n + g) * RS2 + 2 * tq];
      mma3<SPLIT>(s[n], qa, ld32(kp), ld32(kp + 8), SPLIT ? ld32(kp + 16) : 0u,
                  SPLIT ? ld32(kp + 24) : 0u);
    }
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
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      o[n][0] *= f0;
      o[n][1] *= f0;
      o[n][2] *= f1;
      o[n][3] *= f1;
    }
    Frag<SPLIT> pa[4];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const float p0 = ex2(s[n][0] - m0) * psc, p1 = ex2(s[n][1] - m0) * psc;
      const float p2 = ex2(s[n][2] - m1) * psc, p3 = ex2(s[n][3] - m1) * psc;
      const int j = (n & 1) * 2;
      split2<SPLIT>(p0, p1, pa[n >> 1].h[j], pa[n >> 1].l[j]);
      split2<SPLIT>(p2, p3, pa[n >> 1].h[j + 1], pa[n >> 1].l[j + 1]);
    }
    float oc[2][4] = {};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t bh[4], bl[4] = {0u, 0u, 0u, 0u};
      ldsm_bT(Vs + 16 * kk * RS2, RS2, lane, bh);
      if (SPLIT) ldsm_bT(Vs + 16 * kk * RS2 + 16, RS2, lane, bl);
#pragma unroll
      for (int n = 0; n < 2; ++n)
        mma3<SPLIT>(oc[n], pa[kk], bh[2 * n], bh[2 * n + 1], bl[2 * n], bl[2 * n + 1]);
    }
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[n][e] += oc[n][e];
    __syncthreads();  // required: the next iteration's cp.async (into buf ^ 1 of that
                      // iteration, i.e. this `buf`) refills the buffer just read
  }
  // row sums (x 2^15) from the ones column d_head, held by lane quad member (d_head/2)&3
  const int holder = (lane & ~3) | ((d_head >> 1) & 3);
  const int cn = d_head >> 3, ce = d_head & 1;
  const float l0 = __shfl_sync(0xffffffffu, o[cn][ce], holder);
  const float l1 = __shfl_sync(0xffffffffu, o[cn][2 + ce], holder);
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  if (lse && tq == 0) {
    if (r0 < tl.q1) lse[r0 * n_head + h] = m0 + log2f(l0 / psc);
    if (r1 < tl.q1) lse[r1 * n_head + h] = m1 + log2f(l1 / psc);
  }
  const int64_t col0 = (int64_t)h * d_head;
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
}

}  // namespace ab

size_t attention_backward_mma_scratch(int64_t M, int n_head) {
  return (size_t)4 * M * n_head * 32 * sizeof(__half) + 256 * 5;
}

template <bool SPLIT>
static void launch_bwd(const float* q, const float* k, const float* v, const float* dO,
                       int64_t ld, const float* lse, int n_head, int d_head,
                       const AttnTile* qtiles, int64_t nq, const KvTile* ktiles, int64_t nk,
                       const float* Dbuf, int64_t M, float* dq, float* dk_a, float* dv_a,
                       float* dk_b, float* dv_b, char* base, int32_t* flag, cudaStream_t st, const int32_t* gate) {
  constexpr int RW = SPLIT ? 32 : 16;
  const size_t rows = (size_t)M * n_head * RW;
  __half* Qh = reinterpret_cast<__half*>(base);
  __half* Kh = Qh + rows;
  __half* Vh = Kh + rows;
  __half* Oh = Vh + rows;
  unsigned* gbits = reinterpret_cast<unsigned*>(Oh + rows);
  const double sc = 1.0 / std::sqrt((double)d_head);
  const float scale = (float)sc, qscale = (float)(1.4426950408889634 * sc);
  CUDA_CHECK(cudaMemsetAsync(gbits, 0, 3 * sizeof(unsigned), st));
  const int64_t W = (int64_t)n_head * d_head;
  ab::absmax_kernel<<<(unsigned)std::min<int64_t>(cdiv(M * W, 256), 148 * 8), 256, 0, st>>>(
      dO, ld, M, (int)W, gbits, gate);
  LAUNCH_CHECK();
  ab::pack_kernel<SPLIT><<<(unsigned)cdiv(M * n_head, 128), 128, 0, st>>>(
      q, k, v, dO, ld, M, n_head, d_head, qscale, gbits, Qh, Kh, Vh, Oh, flag, gate);
  LAUNCH_CHECK();
  if (nq > 0) {
    ab::dq_kernel<SPLIT><<<dim3((unsigned)nq, (unsigned)n_head), 128, 0, st>>>(
        Qh, Kh, Vh, Oh, M, lse, Dbuf, n_head, d_head, qtiles, dq, ld, scale, gbits, flag, gate);
    LAUNCH_CHECK();
  }
  if (nk > 0) {
    // dk = scale * sum dS q and the packed q carries log2(e) * scale: multiply by 1/log2(e)
    ab::dkv_kernel<SPLIT><<<dim3((unsigned)nk, (unsigned)n_head), 128, 0, st>>>(
        Qh, Kh, Vh, Oh, M, lse, Dbuf, n_head, d_head, ktiles, dk_a, dv_a, dk_b, dv_b, ld,
        (float)(1.0 / 1.4426950408889634), gbits, flag, gate);
    LAUNCH_CHECK();
  }
}

void attention_forward_mma(const float* q, const float* k, const float* v, int64_t ld,
                                int n_head, int d_head, const AttnTile* tiles, int64_t nt,
                                int64_t M, float* out, int64_t ldo, float* lse, void* scratch,
                                int32_t* flag, cudaStream_t st, const int32_t* gate) {
  if (nt <= 0 || M <= 0) return;
  GO_CHECK(d_head >= 1 && d_head <= 15, "attention_forward_mma needs d_head <= 15");
  const size_t rows = (size_t)M * n_head * 32;
  __half* Qh = reinterpret_cast<__half*>(scratch);
  __half* Kh = Qh + rows;
  __half* Vh = Kh + rows;
  unsigned* gbits = reinterpret_cast<unsigned*>(Vh + 2 * rows);
  const float qscale = (float)(1.4426950408889634 / std::sqrt((double)d_head));
  CUDA_CHECK(cudaMemsetAsync(gbits, 0, 3 * sizeof(unsigned), st));
  CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(int32_t), st));
  ab::pack_kernel<true><<<(unsigned)cdiv(M * n_head, 128), 128, 0, st>>>(
      q, k, v, nullptr, ld, M, n_head, d_head, qscale, gbits, Qh, Kh, Vh, nullptr, flag, gate);
  LAUNCH_CHECK();
  ab::fwd_kernel<true><<<dim3((unsigned)nt, (unsigned)n_head), 128, 0, st>>>(
      Qh, Kh, Vh, M, n_head, d_head, tiles, out, ldo, lse, gate);
  LAUNCH_CHECK();
}

void attention_backward_mma(const float* q, const float* k, const float* v, const float* O,
                            const float* dO, int64_t ld, const float* lse, int n_head,
                            int d_head, const AttnTile* qtiles, int64_t nq, const KvTile* ktiles,
                            int64_t nk, float* Dbuf, int64_t M, float* dq, float* dk_a,
                            float* dv_a, float* dk_b, float* dv_b, void* scratch,
                            int32_t* flag, cudaStream_t st, const int32_t* gate) {
  if (M <= 0) return;
  GO_CHECK(d_head >= 1 && d_head <= 16, "attention_backward_mma needs d_head <= 16");
  CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(int32_t), st));
  attention_backward_D(dO, O, ld, n_head, d_head, M, Dbuf, st);
  char* base = reinterpret_cast<char*>(scratch);
  // split-fp16 operands (three MMAs per product); the single-pass instantiation measured
  // ~1e-3 relative gradient error in round 1 and is not launched
  launch_bwd<true>(q, k, v, dO, ld, lse, n_head, d_head, qtiles, nq, ktiles, nk, Dbuf, M, dq,
                   dk_a, dv_a, dk_b, dv_b, base, flag, st, gate);
  // fp32 SIMT re-run, a no-op unless the fp16 range check fired
  attention_backward_simt(q, k, v, dO, ld, lse, n_head, d_head, qtiles, nq, ktiles, nk, Dbuf, dq,
                          dk_a, dv_a, dk_b, dv_b, flag, st);
}

}  // namespace go
