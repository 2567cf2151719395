// Dense row-parallel kernels: fp32 GEMM with fused bias/activation, residual +
// LayerNorm, modulation, means.  These replace the reference's affine / relu /
// sigmoid / concat / layer_norm / mean_rows primitives (tensor.py:148-180,
// 266-351, 378) on the policy path.
#include "engine.cuh"

namespace go {

// ---------------------------------------------------------------------------------
// C[M,N] = act([A1 | A2] @ W + bias).  A1 is [M,K1] (lda1), A2 is [M,K2] (lda2): the
// reference's concat-then-affine (embedding.py:94-95, policy.py:207-208) without
// materialising the concat.  W is [K1+K2, N] row-major (ldw).  act: 0 none, 1 relu,
// 2 sigmoid.  64x64 tile, 256 threads, 4x4 register micro-tile, fp32 FMA.
constexpr int GBM = 64, GBN = 64, GBK = 16;

__global__ void __launch_bounds__(256) gemm_kernel(const float* __restrict__ A1, int64_t lda1,
                                                   int K1, const float* __restrict__ A2,
                                                   int64_t lda2, int K2,
                                                   const float* __restrict__ W, int64_t ldw,
                                                   const float* __restrict__ bias,
                                                   float* __restrict__ C, int64_t ldc,
                                                   int64_t M, int N, int act) {
  __shared__ float As[GBK][GBM + 4];
  __shared__ float Ws[GBK][GBN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * GBM;
  const int n0 = blockIdx.y * GBN;
  const int K = K1 + K2;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += GBK) {
    // A tile: 64 rows x 16 k -> 1024 elements, 4 per thread
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int idx = tid + r * 256;
      int mm = idx >> 4, kk = idx & 15;
      int64_t m = m0 + mm;
      int k = k0 + kk;
      float v = 0.f;
      if (m < M && k < K) v = (k < K1) ? A1[m * lda1 + k] : A2[m * lda2 + (k - K1)];
      As[kk][mm] = v;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int idx = tid + r * 256;
      int kk = idx >> 6, nn = idx & 63;
      int k = k0 + kk, n = n0 + nn;
      Ws[kk][nn] = (k < K && n < N) ? W[(int64_t)k * ldw + n] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j] + (bias ? bias[n] : 0.f);
      if (act == 1) v = v > 0.f ? v : 0.f;
      else if (act == 2) v = 1.f / (1.f + expf(-v));
      C[m * ldc + n] = v;
    }
  }
}

void gemm(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
          const float* W, int64_t ldw, const float* bias, float* C, int64_t ldc, int64_t M,
          int N, int act, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  dim3 grid((unsigned)cdiv(M, GBM), (unsigned)cdiv(N, GBN));
  gemm_kernel<<<grid, 256, 0, st>>>(A1, lda1, K1, A2, lda2, K2, W, ldw, bias, C, ldc, M, N,
                                    act);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// out = LayerNorm(a + b) * g + beta over the last axis (tensor.py:330-351, eps 1e-5);
// b may be null.  One warp per row.
__global__ void add_ln_kernel(const float* __restrict__ a, int64_t lda,
                              const float* __restrict__ b, int64_t ldb,
                              const float* __restrict__ g, const float* __restrict__ beta,
                              float* __restrict__ out, int64_t ldo, int64_t M, int D) {
  int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (row >= M) return;
  constexpr int MAXV = 32;  // D <= 1024
  float v[MAXV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    int c = lane + 32 * i;
    float x = 0.f;
    if (c < D) {
      x = a[row * lda + c];
      if (b) x += b[row * ldb + c];
    }
    v[i] = x;
    s += x;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  float mu = s / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    int c = lane + 32 * i;
    if (c < D) {
      float d = v[i] - mu;
      q += d * d;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  float inv = 1.f / sqrtf(q / D + 1e-5f);
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    int c = lane + 32 * i;
    if (c < D) out[row * ldo + c] = g[c] * ((v[i] - mu) * inv) + beta[c];
  }
}

void add_layernorm(const float* a, int64_t lda, const float* b, int64_t ldb, const float* g,
                   const float* beta, float* out, int64_t ldo, int64_t M, int D,
                   cudaStream_t st) {
  if (M <= 0) return;
  if (D > 1024) GO_THROW(GO_ERR_UNSUPPORTED, "layer_norm width %d > 1024", D);
  add_ln_kernel<<<(unsigned)cdiv(M, 8), 256, 0, st>>>(a, lda, b, ldb, g, beta, out, ldo, M, D);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
__global__ void mul_rowvec_kernel(const float* __restrict__ x, int64_t ldx,
                                  const float* __restrict__ vec, int64_t ldv,
                                  const int32_t* __restrict__ row_fwd, float* __restrict__ out,
                                  int64_t ldo, int64_t M, int D) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * D) return;
  int64_t r = i / D;
  int c = (int)(i - r * D);
  out[r * ldo + c] = x[r * ldx + c] * vec[(int64_t)row_fwd[r] * ldv + c];
}

void mul_rowvec(const float* x, int64_t ldx, const float* vec, int64_t ldv,
                const int32_t* row_fwd, float* out, int64_t ldo, int64_t M, int D,
                cudaStream_t st) {
  if (M <= 0) return;
  mul_rowvec_kernel<<<(unsigned)cdiv(M * D, 256), 256, 0, st>>>(x, ldx, vec, ldv, row_fwd, out,
                                                                ldo, M, D);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// row -> forward index (row_off is [F+1], sorted)
__global__ void row_fwd_kernel(const int64_t* __restrict__ row_off, int F, int64_t R,
                               int32_t* __restrict__ row_fwd) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  int lo = 0, hi = F - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (row_off[mid] <= r) lo = mid;
    else hi = mid - 1;
  }
  row_fwd[r] = lo;
}

void row_fwd_fill(const int64_t* row_off_dev, int F, int64_t R, int32_t* row_fwd,
                  cudaStream_t st) {
  if (R <= 0) return;
  row_fwd_kernel<<<(unsigned)cdiv(R, 256), 256, 0, st>>>(row_off_dev, F, R, row_fwd);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// Per-forward column means (tensor.py:266 mean_rows), deterministic two-pass:
// chunk partial sums, then an ordered reduction per forward.

__global__ void mean_partial_kernel(const float* __restrict__ x, int64_t ldx,
                                    const int64_t* __restrict__ chunk_row0,
                                    const int64_t* __restrict__ chunk_row1, int D,
                                    float* __restrict__ part, int32_t* __restrict__ flag) {
  // 4 row groups x (blockDim / 4) columns; 4 independent accumulators per thread (the
  // serial 256-row chain of one accumulator was latency-bound); fixed combine order
  __shared__ float red[4][128];
  const int64_t c = blockIdx.x;
  const int64_t r0 = chunk_row0[c], r1 = chunk_row1[c];
  const int ncol = blockDim.x >> 2;
  const int grp = threadIdx.x / ncol, lc = threadIdx.x % ncol;
  bool bad = false;
  for (int col0 = 0; col0 < D; col0 += ncol) {
    const int col = col0 + lc;
    float s[4] = {0.f, 0.f, 0.f, 0.f};
    if (col < D) {
      int64_t r = r0 + grp;
      for (; r + 12 < r1; r += 16) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float v = x[(r + 4 * u) * ldx + col];
          bad |= !isfinite(v);
          s[u] += v;
        }
      }
      for (int u = 0; r < r1; r += 4, ++u) {
        const float v = x[r * ldx + col];
        bad |= !isfinite(v);
        s[u & 3] += v;
      }
    }
    red[grp][lc] = (s[0] + s[1]) + (s[2] + s[3]);
    __syncthreads();
    if (grp == 0 && col < D) part[c * D + col] = (red[0][lc] + red[1][lc]) + (red[2][lc] + red[3][lc]);
    __syncthreads();
  }
  // fused non-finite check of the rows being averaged (embedding.py:96-97)
  if (flag && bad) atomicOr(flag, 1);
}

__global__ void mean_final_kernel(const float* __restrict__ part,
                                  const int64_t* __restrict__ fchunk0,
                                  const int64_t* __restrict__ fchunk1,
                                  const int64_t* __restrict__ row_off, int D,
                                  float* __restrict__ out, int64_t ldo) {
  int f = blockIdx.x;
  int64_t n = row_off[f + 1] - row_off[f];
  for (int col = threadIdx.x; col < D; col += blockDim.x) {
    double s = 0.0;
    for (int64_t c = fchunk0[f]; c < fchunk1[f]; ++c) s += part[c * D + col];
    out[(int64_t)f * ldo + col] = n > 0 ? (float)(s / (double)n) : 0.f;
  }
}

void mean_rows(const float* x, int64_t ldx, const int64_t* row_off_dev, int F,
               const int64_t* chunk_tab, int64_t nc, int D, float* out, int64_t ldo,
               float* part, cudaStream_t st, int32_t* finite_flag) {
  // chunk_tab (device): [nc] chunk row0, [nc] chunk row1, [F] first chunk, [F] end chunk
  if (nc > 0)
    mean_partial_kernel<<<(unsigned)nc, 512, 0, st>>>(x, ldx, chunk_tab, chunk_tab + nc, D,
                                                      part, finite_flag);
  mean_final_kernel<<<F, 128, 0, st>>>(part, chunk_tab + 2 * nc, chunk_tab + 2 * nc + F,
                                       row_off_dev, D, out, ldo);
  if (nc > 0) g_launch_count++;
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
__global__ void check_finite_kernel(const float* __restrict__ x, int64_t ld, int64_t M, int D,
                                    int32_t* flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * D) return;
  int64_t r = i / D;
  int c = (int)(i - r * D);
  if (!isfinite(x[r * ld + c])) atomicOr(flag, 1);
}

void check_finite(const float* x, int64_t ld, int64_t M, int D, int32_t* flag,
                  cudaStream_t st) {
  if (M <= 0) return;
  check_finite_kernel<<<(unsigned)cdiv(M * D, 256), 256, 0, st>>>(x, ld, M, D, flag);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// Modulation vector per forward (policy.py:122-132).  The block runs on a length-1
// sequence, so softmax over its single key is exactly 1 and attention = V-projection.
// One CTA per forward; vectors in shared memory.
__device__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

__global__ void modulate_kernel(const float* __restrict__ ge, int64_t ldg, int gs_dim,
                                const float* __restrict__ in_w, const float* __restrict__ in_b,
                                BlockW w, int dm, int wd, int di, float* __restrict__ mod) {
  extern __shared__ float sm[];
  float* g = sm;           // dm
  float* v = g + dm;       // wd
  float* h = v + wd;       // dm
  float* f = h + dm;       // di
  float* t = f + di;       // dm
  float* red = t + dm;     // 32
  int fwd = blockIdx.x;
  const float* x = ge + (int64_t)fwd * ldg;
  for (int c = threadIdx.x; c < dm; c += blockDim.x) {
    float s = in_b[c];
    for (int k = 0; k < gs_dim; ++k) s = fmaf(x[k], in_w[(int64_t)k * dm + c], s);
    g[c] = s;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < wd; c += blockDim.x) {
    float s = w.v_b[c];
    for (int k = 0; k < dm; ++k) s = fmaf(g[k], w.v_w[(int64_t)k * wd + c], s);
    v[c] = s;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < dm; c += blockDim.x) {
    float s = w.o_b[c];
    for (int k = 0; k < wd; ++k) s = fmaf(v[k], w.o_w[(int64_t)k * dm + c], s);
    t[c] = g[c] + s;
  }
  __syncthreads();
  auto ln = [&](float* src, const float* gg, const float* bb, float* dst) {
    float s = 0.f;
    for (int c = threadIdx.x; c < dm; c += blockDim.x) s += src[c];
    float mu = block_sum(s, red) / dm;
    float q = 0.f;
    for (int c = threadIdx.x; c < dm; c += blockDim.x) q += (src[c] - mu) * (src[c] - mu);
    float inv = 1.f / sqrtf(block_sum(q, red) / dm + 1e-5f);
    __syncthreads();
    for (int c = threadIdx.x; c < dm; c += blockDim.x) dst[c] = gg[c] * ((src[c] - mu) * inv) + bb[c];
    __syncthreads();
  };
  ln(t, w.ln1_g, w.ln1_b, h);
  for (int c = threadIdx.x; c < di; c += blockDim.x) {
    float s = w.b1[c];
    for (int k = 0; k < dm; ++k) s = fmaf(h[k], w.w1[(int64_t)k * di + c], s);
    f[c] = s > 0.f ? s : 0.f;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < dm; c += blockDim.x) {
    float s = w.b2[c];
    for (int k = 0; k < di; ++k) s = fmaf(f[k], w.w2[(int64_t)k * dm + c], s);
    t[c] = h[c] + s;
  }
  __syncthreads();
  ln(t, w.ln2_g, w.ln2_b, g);
  for (int c = threadIdx.x; c < dm; c += blockDim.x)
    mod[(int64_t)fwd * dm + c] = 2.f / (1.f + expf(-g[c]));
}

void modulate(const float* graph_embed, int64_t ldg, int F, int gs_dim, const float* in_w,
              const float* in_b, const BlockW& w, int d_model, int wd, int d_inner,
              float* mod_out, cudaStream_t st) {
  if (F <= 0) return;
  size_t sm = (size_t)(3 * d_model + wd + d_inner + d_model + 32) * sizeof(float);
  modulate_kernel<<<F, 256, sm, st>>>(graph_embed, ldg, gs_dim, in_w, in_b, w, d_model, wd,
                                      d_inner, mod_out);
  LAUNCH_CHECK();
}

__global__ void value_kernel(const float* __restrict__ mean, int D, const float* __restrict__ w,
                             const float* __restrict__ b, float* __restrict__ out) {
  int f = blockIdx.x;
  float s = 0.f;
  for (int c = threadIdx.x; c < D; c += 32) s = fmaf(mean[(int64_t)f * D + c], w[c], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) out[f] = s + b[0];
}

void value_head(const float* mean, int F, int D, const float* w, const float* b, float* out,
                cudaStream_t st) {
  if (F <= 0) return;
  value_kernel<<<F, 32, 0, st>>>(mean, D, w, b, out);
  LAUNCH_CHECK();
}

}  // namespace go
