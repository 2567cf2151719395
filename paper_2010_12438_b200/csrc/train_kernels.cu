// Backward kernels of the PPO update (training.py:146-233 through the reference
// tape's closures, tensor.py:87-388).  SIMT fp32; weight gradients accumulate with
// atomics into a float32 gradient blob laid out like the parameter blob.
#include "engine.cuh"
#include "train.cuh"

namespace go {

// ---------------------------------------------------------------------------------
// C[M,N] (+)= A[M,K] @ B,  B = W[K,N] (ldw) or, with TW, B(k,n) = W[n*ldw + k] (W^T).
template <bool TW, bool ACC>
__global__ void __launch_bounds__(256) gemm2_kernel(const float* __restrict__ A, int64_t lda,
                                                    const float* __restrict__ W, int64_t ldw,
                                                    float* __restrict__ C, int64_t ldc,
                                                    int64_t M, int N, int K) {
  __shared__ float As[16][68];
  __shared__ float Bs[16][68];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * 64;
  const int n0 = blockIdx.y * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int idx = tid + r * 256;
      int mm = idx >> 4, kk = idx & 15;
      int64_t m = m0 + mm;
      int k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? A[m * lda + k] : 0.f;
      int kk2 = idx >> 6, nn = idx & 63;
      int kb = k0 + kk2, n = n0 + nn;
      float b = 0.f;
      if (kb < K && n < N) b = TW ? W[(int64_t)n * ldw + kb] : W[(int64_t)kb * ldw + n];
      Bs[kk2][nn] = b;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
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
      if (ACC) C[m * ldc + n] += acc[i][j];
      else C[m * ldc + n] = acc[i][j];
    }
  }
}

void dgemm_nt(const float* dY, int64_t ldd, const float* W, int64_t ldw, float* dX, int64_t ldx,
              int64_t M, int Kin, int Nout, bool accumulate, cudaStream_t st) {
  // dX[M, Kin] (+)= dY[M, Nout] @ W[Kin, Nout]^T
  if (M <= 0 || Kin <= 0) return;
  dim3 grid((unsigned)cdiv(M, 64), (unsigned)cdiv(Kin, 64));
  if (accumulate)
    gemm2_kernel<true, true><<<grid, 256, 0, st>>>(dY, ldd, W, ldw, dX, ldx, M, Kin, Nout);
  else
    gemm2_kernel<true, false><<<grid, 256, 0, st>>>(dY, ldd, W, ldw, dX, ldx, M, Kin, Nout);
  LAUNCH_CHECK();
}

// out[c][r] = W[r * ldw + c] for a rows x cols weight (the tcgen05 dX GEMM's B = W^T)
__global__ void transpose_kernel(const float* __restrict__ W, int64_t ldw, int rows, int cols,
                                 float* __restrict__ out) {
  __shared__ float t[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    t[i][threadIdx.x] = (r < rows && c < cols) ? W[(int64_t)r * ldw + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows) out[(int64_t)c * rows + r] = t[threadIdx.x][i];
  }
}

void transpose(const float* W, int64_t ldw, int rows, int cols, float* out, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  transpose_kernel<<<dim3((unsigned)cdiv(cols, 32), (unsigned)cdiv(rows, 32)), dim3(32, 8), 0,
                     st>>>(W, ldw, rows, cols, out);
  LAUNCH_CHECK();
}

// dW[K1+K2, N] += [A1 | A2]^T @ dY ; db[N] += sum_r dY.  Grid: (K tiles, N tiles, row chunks).
__global__ void __launch_bounds__(256) wgrad_kernel(const float* __restrict__ A1, int64_t lda1,
                                                    int K1, const float* __restrict__ A2,
                                                    int64_t lda2, int K2,
                                                    const float* __restrict__ dY, int64_t ldd,
                                                    int64_t M, int N, float* __restrict__ dW,
                                                    int64_t ldw, float* __restrict__ db,
                                                    int64_t rows_per_chunk) {
  __shared__ float As[16][68];  // [row][k]
  __shared__ float Ds[16][68];  // [row][n]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int k0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  const int K = K1 + K2;
  const int64_t r_begin = (int64_t)blockIdx.z * rows_per_chunk;
  const int64_t r_end = min(M, r_begin + rows_per_chunk);
  float acc[4][4] = {};
  float bacc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t r0 = r_begin; r0 < r_end; r0 += 16) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int idx = tid + q * 256;
      int rr = idx >> 6, cc = idx & 63;
      int64_t r = r0 + rr;
      int k = k0 + cc, n = n0 + cc;
      float a = 0.f, d = 0.f;
      if (r < r_end) {
        if (k < K) a = k < K1 ? A1[r * lda1 + k] : A2[r * lda2 + (k - K1)];
        if (n < N) d = dY[r * ldd + n];
      }
      As[rr][cc] = a;
      Ds[rr][cc] = d;
    }
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
      float a[4], d[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[rr][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) d[j] = Ds[rr][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], d[j], acc[i][j]);
      if (db && ty == 0 && blockIdx.x == 0)
#pragma unroll
        for (int j = 0; j < 4; ++j) bacc[j] += d[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int k = k0 + ty * 4 + i;
    if (k >= K) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n < N) atomicAdd(&dW[(int64_t)k * ldw + n], acc[i][j]);
    }
  }
  if (db && ty == 0 && blockIdx.x == 0)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n < N) atomicAdd(&db[n], bacc[j]);
    }
}

void wgrad(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
           const float* dY, int64_t ldd, int64_t M, int N, float* dW, float* db,
           cudaStream_t st) {
  // tcgen05 split-tf32 GEMM (tc_wgrad.cu); GO_TRAIN_GEMM=simt keeps the fp32 SIMT kernel
  static const bool simt = [] {
    const char* e = getenv("GO_TRAIN_GEMM");
    return e && !strcmp(e, "simt");
  }();
  if (!simt) {
    wgrad_tc(A1, lda1, K1, A2, lda2, K2, dY, ldd, M, N, dW, db, st);
    return;
  }
  if (M <= 0 || N <= 0 || (K1 + K2) <= 0) return;
  int64_t chunks = std::min<int64_t>(cdiv(M, 256), 4 * num_sms());
  int64_t rpc = round_up(cdiv(M, chunks), 16);
  chunks = cdiv(M, rpc);
  dim3 grid((unsigned)cdiv(K1 + K2, 64), (unsigned)cdiv(N, 64), (unsigned)chunks);
  wgrad_kernel<<<grid, 256, 0, st>>>(A1, lda1, K1, A2, lda2, K2, dY, ldd, M, N, dW, N, db, rpc);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// LayerNorm backward (tensor.py:344-351): out = g * xhat + b with xhat = (u - mu) * inv.
// dx (+)= inv * (dxh - mean(dxh) - xhat * mean(dxh * xhat)), dxh = dout * g;
// dg += sum_r dout * xhat ; db += sum_r dout.  8 warps/block, 8 rows per warp.
__global__ void ln_bwd_kernel(const float* __restrict__ u, int64_t ldu,
                              const float* __restrict__ g, const float* __restrict__ dout,
                              int64_t ldd, float* __restrict__ dx, int64_t ldx, int accumulate,
                              int64_t M, int D, float* __restrict__ dg, float* __restrict__ db) {
  extern __shared__ float sred[];  // [2][D]
  for (int c = threadIdx.x; c < 2 * D; c += blockDim.x) sred[c] = 0.f;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int MAXV = 32;
  for (int rr = 0; rr < 8; ++rr) {
    int64_t row = ((int64_t)blockIdx.x * 8 + warp) * 8 + rr;
    if (row >= M) break;
    float v[MAXV], dv[MAXV];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      int c = lane + 32 * i;
      v[i] = c < D ? u[row * ldu + c] : 0.f;
      s += v[i];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    float mu = s / D;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      int c = lane + 32 * i;
      if (c < D) q += (v[i] - mu) * (v[i] - mu);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    float inv = 1.f / sqrtf(q / D + 1e-5f);
    float a = 0.f, bsum = 0.f;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      int c = lane + 32 * i;
      float xh = (v[i] - mu) * inv;
      float d = c < D ? dout[row * ldd + c] : 0.f;
      if (c < D) {
        atomicAdd(&sred[c], d * xh);
        atomicAdd(&sred[D + c], d);
      }
      float dxh = c < D ? d * g[c] : 0.f;
      dv[i] = dxh;
      v[i] = xh;
      a += dxh;
      bsum += dxh * xh;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
    }
    a /= D;
    bsum /= D;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      int c = lane + 32 * i;
      if (c < D) {
        float r = inv * (dv[i] - a - v[i] * bsum);
        if (accumulate) dx[row * ldx + c] += r;
        else dx[row * ldx + c] = r;
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    atomicAdd(&dg[c], sred[c]);
    atomicAdd(&db[c], sred[D + c]);
  }
}

void ln_backward(const float* u, int64_t ldu, const float* g, const float* dout, int64_t ldd,
                 float* dx, int64_t ldx, bool accumulate, int64_t M, int D, float* dg, float* db,
                 cudaStream_t st) {
  if (M <= 0) return;
  if (D > 1024) GO_THROW(GO_ERR_UNSUPPORTED, "layer_norm width %d > 1024", D);
  ln_bwd_kernel<<<(unsigned)cdiv(M, 64), 256, 2 * D * sizeof(float), st>>>(
      u, ldu, g, dout, ldd, dx, ldx, accumulate ? 1 : 0, M, D, dg, db);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// elementwise helpers
__global__ void act_bwd_kernel(float* __restrict__ d, int64_t ldd, const float* __restrict__ y,
                               int64_t ldy, int64_t M, int D, int act) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * D) return;
  int64_t r = i / D;
  int c = (int)(i - r * D);
  float yv = y[r * ldy + c];
  float& dv = d[r * ldd + c];
  if (act == 1) dv = yv > 0.f ? dv : 0.f;       // relu (mask on the output)
  else dv = dv * yv * (1.f - yv);                // sigmoid
}

void act_backward(float* d, int64_t ldd, const float* y, int64_t ldy, int64_t M, int D, int act,
                  cudaStream_t st) {
  if (M <= 0) return;
  act_bwd_kernel<<<(unsigned)cdiv(M * D, 256), 256, 0, st>>>(d, ldd, y, ldy, M, D, act);
  LAUNCH_CHECK();
}

__global__ void add_kernel(float* __restrict__ a, int64_t lda, const float* __restrict__ b,
                           int64_t ldb, int64_t M, int D) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * D) return;
  int64_t r = i / D;
  int c = (int)(i - r * D);
  a[r * lda + c] += b[r * ldb + c];
}

void add_into(float* a, int64_t lda, const float* b, int64_t ldb, int64_t M, int D,
              cudaStream_t st) {
  if (M <= 0) return;
  add_kernel<<<(unsigned)cdiv(M * D, 256), 256, 0, st>>>(a, lda, b, ldb, M, D);
  LAUNCH_CHECK();
}

// segment_max backward (tensor.py:254-260): scatter-add to the argmax rows.
__global__ void segmax_bwd_kernel(const float* __restrict__ dpool, int64_t ldp,
                                  const int32_t* __restrict__ arg, int64_t M, int D,
                                  float* __restrict__ dt, int64_t ldt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * D) return;
  int64_t r = i / D;
  int c = (int)(i - r * D);
  int32_t a = arg[r * D + c];
  if (a >= 0) atomicAdd(&dt[(int64_t)a * ldt + c], dpool[r * ldp + c]);
}

void segmax_backward(const float* dpool, int64_t ldp, const int32_t* arg, int64_t M, int D,
                     float* dt, int64_t ldt, cudaStream_t st) {
  if (M <= 0) return;
  segmax_bwd_kernel<<<(unsigned)cdiv(M * D, 256), 256, 0, st>>>(dpool, ldp, arg, M, D, dt, ldt);
  LAUNCH_CHECK();
}

// xm = x * mod[f]:  dx = dxm * mod ; dmod[f] += sum_r dxm * x
__global__ void rowvec_bwd_kernel(const float* __restrict__ dxm, int64_t ldd,
                                  const float* __restrict__ x, int64_t ldx,
                                  const float* __restrict__ mod, const int32_t* __restrict__ row_fwd,
                                  float* __restrict__ dx, int64_t ldo, float* __restrict__ dmod,
                                  int64_t M, int D) {
  // block: 256 threads over columns (D <= 256 per pass), rows chunk of 64
  int64_t r0 = (int64_t)blockIdx.x * 64;
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    float acc = 0.f;
    int cur = -1;
    for (int64_t r = r0; r < min(M, r0 + 64); ++r) {
      int f = row_fwd[r];
      if (f != cur) {
        if (cur >= 0) atomicAdd(&dmod[(int64_t)cur * D + c], acc);
        acc = 0.f;
        cur = f;
      }
      float d = dxm[r * ldd + c];
      acc += d * x[r * ldx + c];
      dx[r * ldo + c] = d * mod[(int64_t)f * D + c];
    }
    if (cur >= 0) atomicAdd(&dmod[(int64_t)cur * D + c], acc);
  }
}

void rowvec_backward(const float* dxm, int64_t ldd, const float* x, int64_t ldx, const float* mod,
                     const int32_t* row_fwd, float* dx, int64_t ldo, float* dmod, int64_t M, int D,
                     cudaStream_t st) {
  if (M <= 0) return;
  rowvec_bwd_kernel<<<(unsigned)cdiv(M, 64), 256, 0, st>>>(dxm, ldd, x, ldx, mod, row_fwd, dx, ldo,
                                                          dmod, M, D);
  LAUNCH_CHECK();
}

// dh[r] += dG[f] / n_f  (mean_rows backward)
__global__ void mean_bwd_kernel(float* __restrict__ dh, int64_t ldh, const float* __restrict__ dG,
                                const int64_t* __restrict__ row_off,
                                const int32_t* __restrict__ row_fwd, int64_t M, int D) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * D) return;
  int64_t r = i / D;
  int c = (int)(i - r * D);
  int f = row_fwd[r];
  float n = (float)(row_off[f + 1] - row_off[f]);
  dh[r * ldh + c] += dG[(int64_t)f * D + c] / n;
}

void mean_backward(float* dh, int64_t ldh, const float* dG, const int64_t* row_off,
                   const int32_t* row_fwd, int64_t M, int D, cudaStream_t st) {
  if (M <= 0) return;
  mean_bwd_kernel<<<(unsigned)cdiv(M * D, 256), 256, 0, st>>>(dh, ldh, dG, row_off, row_fwd, M, D);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// Attention backward (FA2 recomputation with the saved log2-sum-exp):
//   P = exp2(s2 - lse2), s2 = (q.k) * scale * log2e
//   D_i = dO_i . O_i ; dS = P (dO.v - D) ; dq = scale sum_j dS k_j ; dk = scale sum_i dS q_i
//   dv = sum_i P dO_i.
__global__ void attn_bwd_D_kernel(const float* __restrict__ dO, const float* __restrict__ O,
                                  int64_t ld, int n_head, int d_head, int64_t M,
                                  float* __restrict__ Dout) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * n_head) return;
  int64_t r = i / n_head;
  int h = (int)(i - r * n_head);
  float s = 0.f;
  for (int d = 0; d < d_head; ++d) s += dO[r * ld + h * d_head + d] * O[r * ld + h * d_head + d];
  Dout[i] = s;
}

template <int DH>
__global__ void __launch_bounds__(64) attn_bwd_dq_kernel(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ dO, int64_t ld, const float* __restrict__ lse,
    const float* __restrict__ Dv, int n_head, int d_head, const AttnTile* __restrict__ tiles,
    float* __restrict__ dq, float scale, float scale_log2, const int32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ __align__(16) float Ks[64][DH];
  __shared__ __align__(16) float Vs[64][DH];
  const AttnTile tl = tiles[blockIdx.x];
  const int h = blockIdx.y;
  const int64_t c0 = (int64_t)h * d_head;
  const int64_t row = tl.q0 + threadIdx.x;
  const bool active = row < tl.q1;
  float qr[DH], dor[DH], acc[DH];
  float l2 = 0.f, Di = 0.f;
#pragma unroll
  for (int d = 0; d < DH; ++d) {
    bool ok = active && d < d_head;
    qr[d] = ok ? q[row * ld + c0 + d] * scale_log2 : 0.f;
    dor[d] = ok ? dO[row * ld + c0 + d] : 0.f;
    acc[d] = 0.f;
  }
  if (active) {
    l2 = lse[row * n_head + h];
    Di = Dv[row * n_head + h];
  }
  for (int64_t kc = tl.k0; kc < tl.k1; kc += 64) {
    int nk = (tl.k1 - kc) < 64 ? (int)(tl.k1 - kc) : 64;
    for (int idx = threadIdx.x; idx < 64 * DH; idx += 64) {
      int j = idx / DH, d = idx % DH;
      bool ok = j < nk && d < d_head;
      Ks[j][d] = ok ? k[(kc + j) * ld + c0 + d] : 0.f;
      Vs[j][d] = ok ? v[(kc + j) * ld + c0 + d] : 0.f;
    }
    __syncthreads();
    for (int j = 0; j < nk; ++j) {
      float s = 0.f, dp = 0.f;
#pragma unroll
      for (int d = 0; d < DH; ++d) {
        s = fmaf(qr[d], Ks[j][d], s);
        dp = fmaf(dor[d], Vs[j][d], dp);
      }
      float p = exp2f(s - l2);
      float ds = p * (dp - Di);
#pragma unroll
      for (int d = 0; d < DH; ++d) acc[d] = fmaf(ds, Ks[j][d], acc[d]);
    }
    __syncthreads();
  }
  if (active)
    for (int d = 0; d < d_head; ++d) dq[row * ld + c0 + d] = acc[d] * scale;
}

template <int DH>
__global__ void __launch_bounds__(64) attn_bwd_dkv_kernel(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ dO, int64_t ld, const float* __restrict__ lse,
    const float* __restrict__ Dv, int n_head, int d_head, const KvTile* __restrict__ tiles,
    float* __restrict__ dk_a, float* __restrict__ dv_a, float* __restrict__ dk_b,
    float* __restrict__ dv_b, float scale, float scale_log2, const int32_t* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ __align__(16) float Qs[64][DH];
  __shared__ __align__(16) float Ds_[64][DH];
  __shared__ float Ls[64], Dd[64];
  const KvTile tl = tiles[blockIdx.x];
  const int h = blockIdx.y;
  const int64_t c0 = (int64_t)h * d_head;
  const int64_t key = tl.k0 + threadIdx.x;
  const bool active = key < tl.k1;
  float kr[DH], vr[DH];
#pragma unroll
  for (int d = 0; d < DH; ++d) {
    bool ok = active && d < d_head;
    kr[d] = ok ? k[key * ld + c0 + d] : 0.f;
    vr[d] = ok ? v[key * ld + c0 + d] : 0.f;
  }
  for (int part = 0; part < 2; ++part) {
    const int64_t qa = part ? tl.qb0 : tl.qa0, qe = part ? tl.qb1 : tl.qa1;
    float dk[DH], dv[DH];
#pragma unroll
    for (int d = 0; d < DH; ++d) dk[d] = dv[d] = 0.f;
    for (int64_t qc = qa; qc < qe; qc += 64) {
      int nq = (qe - qc) < 64 ? (int)(qe - qc) : 64;
      for (int idx = threadIdx.x; idx < 64 * DH; idx += 64) {
        int i = idx / DH, d = idx % DH;
        bool ok = i < nq && d < d_head;
        Qs[i][d] = ok ? q[(qc + i) * ld + c0 + d] * scale_log2 : 0.f;
        Ds_[i][d] = ok ? dO[(qc + i) * ld + c0 + d] : 0.f;
      }
      if (threadIdx.x < nq) {
        Ls[threadIdx.x] = lse[(qc + threadIdx.x) * n_head + h];
        Dd[threadIdx.x] = Dv[(qc + threadIdx.x) * n_head + h];
      }
      __syncthreads();
      for (int i = 0; i < nq; ++i) {
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int d = 0; d < DH; ++d) {
          s = fmaf(Qs[i][d], kr[d], s);
          dp = fmaf(Ds_[i][d], vr[d], dp);
        }
        float p = exp2f(s - Ls[i]);
        float ds = p * (dp - Dd[i]);
#pragma unroll
        for (int d = 0; d < DH; ++d) {
          dv[d] = fmaf(p, Ds_[i][d], dv[d]);
          dk[d] = fmaf(ds, Qs[i][d], dk[d]);  // Qs carries scale*log2e; fixed below
        }
      }
      __syncthreads();
    }
    float* dko = part ? dk_b : dk_a;
    float* dvo = part ? dv_b : dv_a;
    if (active && dko) {
      // dk = scale * sum ds q  ;  Qs held q * scale * log2e  ->  divide by log2e
      for (int d = 0; d < d_head; ++d) {
        dko[key * ld + c0 + d] = dk[d] * (scale / scale_log2);
        dvo[key * ld + c0 + d] = dv[d];
      }
    }
  }
}

void attention_backward_D(const float* dO, const float* O, int64_t ld, int n_head, int d_head,
                          int64_t M, float* Dbuf, cudaStream_t st) {
  if (M <= 0) return;
  attn_bwd_D_kernel<<<(unsigned)cdiv(M * n_head, 256), 256, 0, st>>>(dO, O, ld, n_head, d_head, M,
                                                                     Dbuf);
  LAUNCH_CHECK();
}

void attention_backward_simt(const float* q, const float* k, const float* v, const float* dO,
                             int64_t ld, const float* lse, int n_head, int d_head,
                             const AttnTile* qtiles, int64_t nq, const KvTile* ktiles, int64_t nk,
                             const float* Dbuf, float* dq, float* dk_a, float* dv_a, float* dk_b,
                             float* dv_b, const int32_t* gate, cudaStream_t st) {
  float scale = (float)(1.0 / std::sqrt((double)d_head));
  float scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d_head));
  dim3 gq((unsigned)nq, (unsigned)n_head), gk((unsigned)nk, (unsigned)n_head);
#define GO_BWD(DHV)                                                                             \
  do {                                                                                          \
    if (nq > 0) {                                                                               \
      attn_bwd_dq_kernel<DHV><<<gq, 64, 0, st>>>(q, k, v, dO, ld, lse, Dbuf, n_head, d_head,     \
                                                 qtiles, dq, scale, scale_log2, gate);          \
      LAUNCH_CHECK();                                                                           \
    }                                                                                           \
    if (nk > 0) {                                                                               \
      attn_bwd_dkv_kernel<DHV><<<gk, 64, 0, st>>>(q, k, v, dO, ld, lse, Dbuf, n_head, d_head,    \
                                                  ktiles, dk_a, dv_a, dk_b, dv_b, scale,        \
                                                  scale_log2, gate);                            \
      LAUNCH_CHECK();                                                                           \
    }                                                                                           \
  } while (0)
  if (d_head <= 4) GO_BWD(4);
  else if (d_head <= 8) GO_BWD(8);
  else if (d_head <= 16) GO_BWD(16);
  else if (d_head <= 32) GO_BWD(32);
  else if (d_head <= 64) GO_BWD(64);
  else GO_THROW(GO_ERR_UNSUPPORTED, "d_head %d > 64", d_head);
#undef GO_BWD
}

void attention_backward(const float* q, const float* k, const float* v, const float* O,
                        const float* dO, int64_t ld, const float* lse, int n_head, int d_head,
                        const AttnTile* qtiles, int64_t nq, const KvTile* ktiles, int64_t nk,
                        float* Dbuf, int64_t M, float* dq, float* dk_a, float* dv_a, float* dk_b,
                        float* dv_b, cudaStream_t st) {
  if (M <= 0) return;
  attention_backward_D(dO, O, ld, n_head, d_head, M, Dbuf, st);
  attention_backward_simt(q, k, v, dO, ld, lse, n_head, d_head, qtiles, nq, ktiles, nk, Dbuf, dq,
                          dk_a, dv_a, dk_b, dv_b, nullptr, st);
}

// ---------------------------------------------------------------------------------
// PPO per-row loss and dL/dlogits (training.py:159-185), float64 arithmetic.
__global__ void ppo_loss_kernel(const float* __restrict__ logits, int a, int64_t R,
                                const int32_t* __restrict__ actions,
                                const int32_t* __restrict__ row_node,
                                const double* __restrict__ old_logp,
                                const int32_t* __restrict__ row_fwd,
                                const int64_t* __restrict__ row_off,
                                const double* __restrict__ fparams,  // [F][4]: adv, temp, reward, -
                                double eps, double c_ent, int T, int C, int t_index,
                                float* __restrict__ dlogits, double* __restrict__ stats) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  int f = row_fwd[r];
  double n = (double)(row_off[f + 1] - row_off[f]);
  double A = fparams[4 * f], temp = fparams[4 * f + 1];
  double z[32], p[32];
  double mx = -INFINITY;
  for (int j = 0; j < a; ++j) {
    z[j] = (double)logits[r * a + j] / temp;
    mx = fmax(mx, z[j]);
  }
  double s = 0.0;
  for (int j = 0; j < a; ++j) s += exp(z[j] - mx);
  double lse = mx + log(s);
  int act = actions[row_off[f] + row_node[r]];
  for (int j = 0; j < a; ++j) {
    z[j] -= lse;  // logp
    p[j] = exp(z[j]);
  }
  double ratio = exp(z[act] - old_logp[r]);
  double lo = 1.0 - eps, hi = 1.0 + eps;
  double cl = fmin(fmax(ratio, lo), hi);
  double a1 = ratio * A, a2 = cl * A;
  bool take_a = a1 <= a2;
  double surr = take_a ? a1 : a2;
  bool inside = ratio >= lo && ratio <= hi;
  double dsurr_dr = take_a ? A : (inside ? A : 0.0);
  double ent = 0.0;
  for (int j = 0; j < a; ++j) ent -= p[j] * z[j];
  const double ksurr = -1.0 / (T * n * C), kent = -c_ent / (T * n * C);
  double g[32], gs = 0.0;
  for (int j = 0; j < a; ++j) {
    g[j] = kent * (-p[j] * (z[j] + 1.0));
    if (j == act) g[j] += ksurr * dsurr_dr * ratio;
    gs += g[j];
  }
  for (int j = 0; j < a; ++j) dlogits[r * a + j] = (float)((g[j] - p[j] * gs) / temp);
  double* st = stats + ((int64_t)f * 3 + t_index) * 4;
  atomicAdd(&st[0], surr);
  atomicAdd(&st[1], ent);
  atomicAdd(&st[2], ratio);
  atomicAdd(&st[3], fabs(ratio - 1.0) > eps ? 1.0 : 0.0);
}

void ppo_loss(const float* logits, int a, int64_t R, const int32_t* actions,
              const int32_t* row_node, const double* old_logp, const int32_t* row_fwd,
              const int64_t* row_off, const double* fparams, double eps, double c_ent, int T,
              int C, int t_index, float* dlogits, double* stats, cudaStream_t st) {
  if (R <= 0) return;
  if (a > 32) GO_THROW(GO_ERR_UNSUPPORTED, "action space %d > 32", a);
  ppo_loss_kernel<<<(unsigned)cdiv(R, 128), 128, 0, st>>>(logits, a, R, actions, row_node,
                                                          old_logp, row_fwd, row_off, fparams, eps,
                                                          c_ent, T, C, t_index, dlogits, stats);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// value = mean(rep) . value_w + value_b ; dvalue_f = c_v * 2 (value_f - reward_f) / C.
// drep[r] += dvalue_f * value_w / n_f ; dvalue_w += sum_f dvalue_f * mean_f ; dvalue_b.
__global__ void value_bwd_kernel(const float* __restrict__ value, const float* __restrict__ mean,
                                 const double* __restrict__ rewards, int F, int D, double c_v,
                                 int C, const float* __restrict__ vw, float* __restrict__ dvalue,
                                 float* __restrict__ dvw, float* __restrict__ dvb,
                                 double* __restrict__ vstats) {
  for (int f = 0; f < F; ++f) {
    double err = (double)value[f] - rewards[f];
    float dv = (float)(c_v * 2.0 * err / C);
    if (threadIdx.x == 0) {
      dvalue[f] = dv;
      atomicAdd(dvb, dv);
      vstats[f] = err * err;
    }
    for (int c = threadIdx.x; c < D; c += blockDim.x) atomicAdd(&dvw[c], dv * mean[(int64_t)f * D + c]);
  }
}

__global__ void value_rep_bwd_kernel(float* __restrict__ drep, int64_t ld,
                                     const float* __restrict__ dvalue,
                                     const float* __restrict__ vw,
                                     const int64_t* __restrict__ row_off,
                                     const int32_t* __restrict__ row_fwd, int64_t M, int D) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * D) return;
  int64_t r = i / D;
  int c = (int)(i - r * D);
  int f = row_fwd[r];
  drep[r * ld + c] += dvalue[f] * vw[c] / (float)(row_off[f + 1] - row_off[f]);
}

void value_backward(const float* value, const float* mean, const double* rewards, int F, int D,
                    double c_v, int C, const float* vw, float* dvalue, float* dvw, float* dvb,
                    double* vstats, float* drep, int64_t ldr, const int64_t* row_off,
                    const int32_t* row_fwd, int64_t M, cudaStream_t st) {
  value_bwd_kernel<<<1, 128, 0, st>>>(value, mean, rewards, F, D, c_v, C, vw, dvalue, dvw, dvb,
                                      vstats);
  LAUNCH_CHECK();
  if (M > 0) {
    value_rep_bwd_kernel<<<(unsigned)cdiv(M * D, 256), 256, 0, st>>>(drep, ldr, dvalue, vw, row_off,
                                                                     row_fwd, M, D);
    LAUNCH_CHECK();
  }
}

// ---------------------------------------------------------------------------------
// embed/in_w gradient for in-kernel features (graph.py:268-313): the feature row is
// sparse, so dW[c] += feat[r][c] * dh0[r] touches 5 + T weight rows per node.
__global__ void inproj_wgrad_kernel(const GraphView* __restrict__ views,
                                    const int64_t* __restrict__ row_off,
                                    const int32_t* __restrict__ row_fwd, int64_t R,
                                    const int32_t* __restrict__ prev, int T, int tc0, int tc1,
                                    int tc2, const float* __restrict__ dh, int64_t ldh, int D,
                                    int F, float* __restrict__ dW, float* __restrict__ db) {
  extern __shared__ float sw[];  // [(F + 1) * D]: rows of dW, last row = db
  for (int i = threadIdx.x; i < (F + 1) * D; i += blockDim.x) sw[i] = 0.f;
  __syncthreads();
  int64_t r0 = (int64_t)blockIdx.x * 128;
  for (int64_t r = r0; r < min(R, r0 + 128); ++r) {
    int f = row_fwd[r];
    const GraphView& G = views[f];
    int64_t lr = r - row_off[f];
    const float* s4 = G.static4 + lr * 4;
    int op = G.op_row[lr];
    int acts[3] = {0, 0, 0};
    int tcs[3] = {tc0, tc1, tc2};
    if (prev) {
      int node = G.order[lr];
      for (int t = 0; t < T; ++t) acts[t] = prev[(int64_t)t * R + row_off[f] + node];
    }
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
      float g = dh[r * ldh + c];
      sw[op * D + c] += g;
      sw[12 * D + c] += s4[0] * g;
      sw[13 * D + c] += s4[1] * g;
      sw[14 * D + c] += s4[2] * g;
      sw[15 * D + c] += s4[3] * g;
      if (prev)
        for (int t = 0; t < T; ++t) sw[(tcs[t] + acts[t]) * D + c] += g;
      sw[F * D + c] += g;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < F * D; i += blockDim.x)
    if (sw[i] != 0.f) atomicAdd(&dW[i], sw[i]);
  for (int c = threadIdx.x; c < D; c += blockDim.x) atomicAdd(&db[c], sw[F * D + c]);
}

void inproj_wgrad(const GraphView* views, const int64_t* row_off, const int32_t* row_fwd,
                  int64_t R, const int32_t* prev, int T, const int32_t* tcol, const float* dh,
                  int64_t ldh, int D, int Fdim, float* dW, float* db, cudaStream_t st) {
  if (R <= 0) return;
  size_t smem = (size_t)(Fdim + 1) * D * sizeof(float);
  if (smem > 48 * 1024) GO_THROW(GO_ERR_UNSUPPORTED, "feature width too large");
  inproj_wgrad_kernel<<<(unsigned)cdiv(R, 128), 128, smem, st>>>(
      views, row_off, row_fwd, R, prev, T, tcol[0], tcol[1], tcol[2], dh, ldh, D, Fdim, dW, db);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// Modulation block backward, one CTA per forward.  Recomputes the length-1 block
// (policy.py:122-132) in shared memory, then back-propagates dmod to dG (graph
// embedding) and to the block's and policy/in_w's parameters.
__device__ float bsum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  __syncthreads();
  return s;
}

__global__ void modulate_bwd_kernel(const float* __restrict__ ge, int gs,
                                    const float* __restrict__ in_w, const float* __restrict__ in_b,
                                    BlockW w, int dm, int wd, int di,
                                    const float* __restrict__ dmod, float* __restrict__ dge,
                                    BlockG gr, float* __restrict__ d_in_w, float* __restrict__ d_in_b) {
  extern __shared__ float sm[];
  float* g = sm;            // dm  block input
  float* v = g + dm;        // wd  V projection
  float* u1 = v + wd;       // dm  g + o
  float* h1 = u1 + dm;      // dm  LN1 out
  float* f1 = h1 + dm;      // di  relu(h1 W1 + b1)
  float* u2 = f1 + di;      // dm  h1 + f2
  float* y = u2 + dm;       // dm  LN2 out
  float* dy = y + dm;       // dm
  float* du = dy + dm;      // dm (scratch)
  float* dh = du + dm;      // dm
  float* df = dh + dm;      // di
  float* dv = df + di;      // wd
  float* dg = dv + wd;      // dm
  float* red = dg + dm;     // 32
  const int fw = blockIdx.x;
  const float* x = ge + (int64_t)fw * gs;
  // ---- forward recompute
  for (int c = threadIdx.x; c < dm; c += blockDim.x) {
    float s = in_b[c];
    for (int k = 0; k < gs; ++k) s = fmaf(x[k], in_w[(int64_t)k * dm + c], s);
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
    u1[c] = g[c] + s;
  }
  __syncthreads();
  auto stats = [&](const float* src, float& mu, float& inv) {
    float s = 0.f;
    for (int c = threadIdx.x; c < dm; c += blockDim.x) s += src[c];
    mu = bsum(s, red) / dm;
    float q = 0.f;
    for (int c = threadIdx.x; c < dm; c += blockDim.x) q += (src[c] - mu) * (src[c] - mu);
    inv = 1.f / sqrtf(bsum(q, red) / dm + 1e-5f);
  };
  float mu1, inv1, mu2, inv2;
  stats(u1, mu1, inv1);
  for (int c = threadIdx.x; c < dm; c += blockDim.x)
    h1[c] = w.ln1_g[c] * ((u1[c] - mu1) * inv1) + w.ln1_b[c];
  __syncthreads();
  for (int c = threadIdx.x; c < di; c += blockDim.x) {
    float s = w.b1[c];
    for (int k = 0; k < dm; ++k) s = fmaf(h1[k], w.w1[(int64_t)k * di + c], s);
    f1[c] = s > 0.f ? s : 0.f;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < dm; c += blockDim.x) {
    float s = w.b2[c];
    for (int k = 0; k < di; ++k) s = fmaf(f1[k], w.w2[(int64_t)k * dm + c], s);
    u2[c] = h1[c] + s;
  }
  __syncthreads();
  stats(u2, mu2, inv2);
  for (int c = threadIdx.x; c < dm; c += blockDim.x)
    y[c] = w.ln2_g[c] * ((u2[c] - mu2) * inv2) + w.ln2_b[c];
  __syncthreads();
  // ---- backward: mod = 2 sigmoid(y)
  for (int c = threadIdx.x; c < dm; c += blockDim.x) {
    float sgm = 1.f / (1.f + expf(-y[c]));
    dy[c] = dmod[(int64_t)fw * dm + c] * 2.f * sgm * (1.f - sgm);
  }
  __syncthreads();
  auto ln_bwd = [&](const float* src, float mu, float inv, const float* gain, float* dgain,
                    float* dbias, const float* dout, float* dx) {
    float a = 0.f, b = 0.f;
    for (int c = threadIdx.x; c < dm; c += blockDim.x) {
      float xh = (src[c] - mu) * inv;
      float dxh = dout[c] * gain[c];
      a += dxh;
      b += dxh * xh;
      atomicAdd(&dgain[c], dout[c] * xh);
      atomicAdd(&dbias[c], dout[c]);
    }
    a = bsum(a, red) / dm;
    b = bsum(b, red) / dm;
    for (int c = threadIdx.x; c < dm; c += blockDim.x) {
      float xh = (src[c] - mu) * inv;
      dx[c] = inv * (dout[c] * gain[c] - a - xh * b);
    }
    __syncthreads();
  };
  ln_bwd(u2, mu2, inv2, w.ln2_g, gr.ln2_g, gr.ln2_b, dy, du);  // du = d u2
  // u2 = h1 + f1 W2 + b2
  for (int c = threadIdx.x; c < di; c += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < dm; ++k) s = fmaf(du[k], w.w2[(int64_t)c * dm + k], s);
    df[c] = f1[c] > 0.f ? s : 0.f;
    for (int k = 0; k < dm; ++k) atomicAdd(&gr.w2[(int64_t)c * dm + k], f1[c] * du[k]);
  }
  for (int c = threadIdx.x; c < dm; c += blockDim.x) atomicAdd(&gr.b2[c], du[c]);
  __syncthreads();
  for (int c = threadIdx.x; c < dm; c += blockDim.x) {
    float s = du[c];
    for (int k = 0; k < di; ++k) s = fmaf(df[k], w.w1[(int64_t)c * di + k], s);
    dh[c] = s;
    for (int k = 0; k < di; ++k) atomicAdd(&gr.w1[(int64_t)c * di + k], h1[c] * df[k]);
  }
  for (int c = threadIdx.x; c < di; c += blockDim.x) atomicAdd(&gr.b1[c], df[c]);
  __syncthreads();
  ln_bwd(u1, mu1, inv1, w.ln1_g, gr.ln1_g, gr.ln1_b, dh, du);  // du = d u1
  // u1 = g + v Wo + bo ; v = g Wv + bv
  for (int c = threadIdx.x; c < wd; c += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < dm; ++k) s = fmaf(du[k], w.o_w[(int64_t)c * dm + k], s);
    dv[c] = s;
    for (int k = 0; k < dm; ++k) atomicAdd(&gr.o_w[(int64_t)c * dm + k], v[c] * du[k]);
  }
  for (int c = threadIdx.x; c < dm; c += blockDim.x) atomicAdd(&gr.o_b[c], du[c]);
  __syncthreads();
  for (int c = threadIdx.x; c < dm; c += blockDim.x) {
    float s = du[c];
    for (int k = 0; k < wd; ++k) s = fmaf(dv[k], w.v_w[(int64_t)c * wd + k], s);
    dg[c] = s;
    for (int k = 0; k < wd; ++k) atomicAdd(&gr.v_w[(int64_t)c * wd + k], g[c] * dv[k]);
  }
  for (int c = threadIdx.x; c < wd; c += blockDim.x) atomicAdd(&gr.v_b[c], dv[c]);
  __syncthreads();
  // g = x in_w + in_b
  for (int k = threadIdx.x; k < gs; k += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < dm; ++c) {
      s = fmaf(dg[c], in_w[(int64_t)k * dm + c], s);
      atomicAdd(&d_in_w[(int64_t)k * dm + c], x[k] * dg[c]);
    }
    dge[(int64_t)fw * gs + k] = s;
  }
  for (int c = threadIdx.x; c < dm; c += blockDim.x) atomicAdd(&d_in_b[c], dg[c]);
}

void modulate_backward(const float* ge, int F, int gs, const float* in_w, const float* in_b,
                       const BlockW& w, int dm, int wd, int di, const float* dmod, float* dge,
                       const BlockG& gr, float* d_in_w, float* d_in_b, cudaStream_t st) {
  if (F <= 0) return;
  size_t smem = (size_t)(10 * dm + 2 * wd + 2 * di + 32) * sizeof(float);
  modulate_bwd_kernel<<<F, 256, smem, st>>>(ge, gs, in_w, in_b, w, dm, wd, di, dmod, dge, gr,
                                            d_in_w, d_in_b);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// Fused Adam over the whole blob (tensor.py:428-441): every parameter steps, g = 0
// where no gradient flowed.  bc1 = 1 - beta1^t, bc2 = 1 - beta2^t (host float64).
__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                            float* __restrict__ m, float* __restrict__ v, int64_t n, float lr,
                            float b1, float b2, float eps, float bc1, float bc2) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float gi = g[i];
  float mi = b1 * m[i] + (1.f - b1) * gi;
  float vi = b2 * v[i] + (1.f - b2) * gi * gi;
  m[i] = mi;
  v[i] = vi;
  p[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
}

void adam(float* p, const float* g, float* m, float* v, int64_t n, double lr, double b1,
          double b2, double eps, int64_t step, cudaStream_t st) {
  if (n <= 0) return;
  double bc1 = 1.0 - std::pow(b1, (double)step), bc2 = 1.0 - std::pow(b2, (double)step);
  adam_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(p, g, m, v, n, (float)lr, (float)b1,
                                                     (float)b2, (float)eps, (float)bc1,
                                                     (float)bc2);
  LAUNCH_CHECK();
}

// Float64-master Adam, the reference's arithmetic (tensor.py:428-441) operation for
// operation: m = b1*m + (1-b1)*g; v = b2*v + (1-b2)*g*g; p -= lr*(m/bc1)/(sqrt(v/bc2)+eps)
// with explicit _rn intrinsics so no FMA contraction changes a rounding.  The master
// parameters and moments stay float64 on the device across the whole update; the
// kernels read the float32 copy written here.
__global__ void adam64_kernel(double* __restrict__ p, float* __restrict__ p32,
                              const float* __restrict__ g, double* __restrict__ m,
                              double* __restrict__ v, int64_t n, double lr, double b1,
                              double b2, double eps, double bc1, double bc2) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double gi = (double)g[i];
  double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dadd_rn(1.0, -b1), gi));
  double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(__dadd_rn(1.0, -b2), gi), gi));
  m[i] = mi;
  v[i] = vi;
  double mhat = __ddiv_rn(mi, bc1);
  double vhat = __ddiv_rn(vi, bc2);
  double step = __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps));
  double pi = __dadd_rn(p[i], -step);
  p[i] = pi;
  p32[i] = (float)pi;
}

void adam64(double* p, float* p32, const float* g, double* m, double* v, int64_t n, double lr,
            double b1, double b2, double eps, int64_t step, cudaStream_t st) {
  if (n <= 0) return;
  double bc1 = 1.0 - std::pow(b1, (double)step), bc2 = 1.0 - std::pow(b2, (double)step);
  adam64_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(p, p32, g, m, v, n, lr, b1, b2, eps,
                                                       bc1, bc2);
  LAUNCH_CHECK();
}

}  // namespace go
