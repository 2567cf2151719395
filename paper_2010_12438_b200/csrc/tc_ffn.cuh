// Fused feed-forward block of the trunk (policy.py:170-177; transformer_block's
// out = LN(h + FF(h)), FF(h) = relu(h W1 + b1) W2 + b2, d_model = 128, d_inner = 512):
//   C = LN(X + relu(X W1 + b1) W2 + b2) * g + b,   C2 = C * rowscale[forward]
// (or, for a task head, C = relu(X W1 + b1) W2 + b2 without residual / LN, policy.py:212-214)
// in ONE persistent kernel, so the 512-wide intermediate never leaves the SM (it was
// 40% of the dense layers' HBM traffic as an fp32 [R, 512] round trip).  Included by
// tc_gemm.cu (shares its helpers and launch plumbing).
//
// Per 128-row tile, in 128-column chunks c = 0..3 of the intermediate H:
//   G1(c): D1[c&1] = X W1[:, 128c:128c+128]        (TMEM, double-buffered)
//   E1(c): H_c = relu(D1 + b1) split to fp16 hi/lo  (smem, the A operand of G2)
//   G2(c): D2 += H_c W2[128c:128c+128, :]            (TMEM)
// issued as G1(0) G1(1) G2(0) G1(2) G2(1) G1(3) G2(2) G2(3), so E1(c) overlaps G1(c+1)
// and G2(c-1).  Both GEMMs are 3-pass fp16 (hi*hi + hi*lo + lo*hi, kind::f16) like
// tc_gemm, in the same order with the same splits, so the output is bit-identical to
// the two unfused GEMMs; weights are prepacked (x 2^8) in 128-column blocks of 32-k
// chunks.  X or H beyond the fp16 range sets *ovf and the caller re-runs the unfused
// tf32 layers (gated on the flag).
//
// 9 warps: 0-3 split X (thread = row) then drain D1 into H; 4-7 the LayerNorm epilogue
// (thread = row); 8 loads (TMA for X, bulk copies for the weight chunks) and issues the
// MMAs.  TMEM: D1 x 2 (256 columns) + D2 (128).  SMEM: X hi/lo 64 KB + H hi/lo 64 KB +
// a 4-stage ring of 16 KB weight chunks + epilogue staging.
//
// Measured (ncu, 2 cfg4 forwards): 402 us against 476 us for the two unfused GEMMs.  The
// kernel is bound by streaming 512 KB of W1/W2 hi/lo chunks per 128-row tile from L2
// through the 4-stage ring (tensor pipe ~28% busy); a variant with double-buffered H
// halves and D2 was slower (536 us: its in-order MMA issue blocked behind the LayerNorm
// warps).  Sharing each weight chunk between two row tiles (M = 256) is the next step.

struct FfnArgs {
  const float* X;  // input and residual (global, fp32)
  int64_t ldx;
  const uint8_t* W1;  // [4 n-blocks][4 k-chunks][hi|lo][128 x 32] fp16
  const uint8_t* W2;  // [1][16 k-chunks][hi|lo][128 x 32] fp16
  const float* b1;    // [512]
  const float* b2;    // [128]
  const float* ln_g;
  const float* ln_b;
  float* C;  // optional
  int64_t ldc;
  const float* rowscale;  // optional ([F, 128]); with C2
  const int32_t* row_fwd;
  float* C2;
  int64_t ldc2;
  int64_t M;
  int32_t* ovf;
  int ln;  // 1: C = LN(X + FF(X)) (trunk block); 0: C = FF(X) (task head, policy.py:212-214)
};

constexpr int FF_CHUNK = 16384;  // one 32-k chunk: fp32 TMA box, or fp16 hi (8 KB) + lo
constexpr int FF_NSW = 4;        // weight ring stages
constexpr int FF_EPI = 4 * 32 * 36 * 4 + 512 * 4;
constexpr size_t FF_SMEM = 1024 + 8 * FF_CHUNK + FF_NSW * FF_CHUNK + FF_EPI + 1024;

__global__ void __launch_bounds__(G_THREADS, 1)
    ffn_kernel(const __grid_constant__ CUtensorMap tmX, FfnArgs a, int ntiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* Xs = base;                    // 4 chunks
  uint8_t* Hs = base + 4 * FF_CHUNK;     // 4 chunks
  uint8_t* Ws = base + 8 * FF_CHUNK;     // FF_NSW stages
  float* epi = reinterpret_cast<float*>(Ws + FF_NSW * FF_CHUNK);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(epi) + FF_EPI);
  uint64_t* x_full = bars + 0;
  uint64_t* x_ready = bars + 1;
  uint64_t* x_empty = bars + 2;
  uint64_t* h_full = bars + 3;
  uint64_t* h_empty = bars + 4;
  uint64_t* d2_full = bars + 5;
  uint64_t* d2_empty = bars + 6;
  uint64_t* d1_full = bars + 7;    // [2]
  uint64_t* d1_empty = bars + 9;   // [2]
  uint64_t* w_full = bars + 11;    // [FF_NSW]
  uint64_t* w_done = bars + 11 + FF_NSW;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11 + 2 * FF_NSW);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr float ASCALE = 1.f / (1 << W16_SHIFT);

  if (warp == 8) {
    if (lane == 0) {
      mbar_init(x_full, 1);
      mbar_init(x_ready, 128);
      mbar_init(x_empty, 1);
      mbar_init(h_full, 128);
      mbar_init(h_empty, 1);
      mbar_init(d2_full, 1);
      mbar_init(d2_empty, 128);
      for (int b = 0; b < 2; ++b) {
        mbar_init(&d1_full[b], 1);
        mbar_init(&d1_empty[b], 128);
      }
      for (int s = 0; s < FF_NSW; ++s) {
        mbar_init(&w_full[s], 1);
        mbar_init(&w_done[s], 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t D1 = tbase, D2 = tbase + 256;  // D1[b] at +128 b

  if (warp == 8) {
    if (lane == 0) {
      constexpr uint32_t ID = idesc_f16(BM, 128);
      // job order per tile: G1 0, G1 1, G2 0, G1 2, G2 1, G1 3, G2 2, G2 3 (4 weight
      // chunks each: G1(c) -> W1 block c, k-chunks 0..3; G2(c) -> W2 k-chunks 4c..4c+3)
      // (bit-packed tables: a dynamically indexed local array would live in local memory,
      // where a single active lane pulls a whole line per word)
      auto job_g1 = [](int j) { return ((0x2Bu >> j) & 1u) != 0; };       // G1 at j = 0,1,3,5
      auto job_c = [](int j) { return (int)((0x32312010u >> (4 * j)) & 0xFu); };
      const int total = my_tiles * 32;  // weight chunks
      auto load_w = [&](int g) {
        const int s = g % FF_NSW;
        const int i = g % 32, j = i >> 2, kc = i & 3;
        const uint8_t* src = job_g1(j) ? a.W1 + (size_t)(job_c(j) * 4 + kc) * 2 * 8192
                                       : a.W2 + (size_t)(job_c(j) * 4 + kc) * 2 * 8192;
        mbar_expect_tx(&w_full[s], FF_CHUNK);
        bulk_g2s(Ws + (size_t)s * FF_CHUNK, src, FF_CHUNK, &w_full[s]);
      };
      auto load_x = [&](int tl) {
        const int m0 = (blockIdx.x + tl * gridDim.x) * BM;
        mbar_expect_tx(x_full, 4 * FF_CHUNK);
        for (int kc = 0; kc < 4; ++kc) tma_2d(Xs + kc * FF_CHUNK, &tmX, kc * BK, m0, x_full);
      };
      if (my_tiles > 0) load_x(0);
      for (int g = 0; g < FF_NSW && g < total; ++g) load_w(g);
      int g = 0;
      for (int tl = 0; tl < my_tiles; ++tl) {
        for (int j = 0; j < 8; ++j) {
          const int c = job_c(j);
          const bool g1 = job_g1(j);
          const int u = tl * 4 + c;  // use index of D1[c & 1] and of the H buffer
          uint32_t dacc;
          const uint8_t* abase;
          if (g1) {
            if (c == 0) mbar_wait(x_ready, tl & 1);
            if (u >= 2) mbar_wait(&d1_empty[c & 1], ((u >> 1) - 1) & 1);
            dacc = D1 + (c & 1) * 128;
            abase = Xs;
          } else {
            mbar_wait(h_full, u & 1);
            if (c == 0 && tl >= 1) mbar_wait(d2_empty, (tl - 1) & 1);
            dacc = D2;
            abase = Hs;
          }
          fence_after();
          for (int kc = 0; kc < 4; ++kc, ++g) {
            const int s = g % FF_NSW;
            mbar_wait(&w_full[s], (g / FF_NSW) & 1);
            fence_after();
            const uint32_t a16 = smem_u32(abase + kc * FF_CHUNK);
            const uint32_t bh = smem_u32(Ws + (size_t)s * FF_CHUNK), bl = bh + 8192;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t dah = sdesc(a16 + kk * 4096, 2048, 128);
              const uint64_t dal = sdesc(a16 + 8192 + kk * 4096, 2048, 128);
              const uint64_t dbh = sdesc(bh + kk * 2 * 128 * 16, 128 * 16, 128);
              const uint64_t dbl = sdesc(bl + kk * 2 * 128 * 16, 128 * 16, 128);
              const uint32_t acc0 = g1 ? (kc > 0 || kk > 0) : (c > 0 || kc > 0 || kk > 0);
              umma_ss_f16(dacc, dah, dbh, ID, acc0);
              umma_ss_f16(dacc, dah, dbl, ID, 1);
              umma_ss_f16(dacc, dal, dbh, ID, 1);
            }
            umma_commit(&w_done[s]);
            if (g >= 1 && (g - 1) + FF_NSW < total) {
              mbar_wait(&w_done[(g - 1) % FF_NSW], ((g - 1) / FF_NSW) & 1);
              load_w(g - 1 + FF_NSW);
            }
          }
          if (g1) {
            umma_commit(&d1_full[c & 1]);
            if (c == 3) umma_commit(x_empty);
          } else {
            umma_commit(h_empty);
            if (c == 3) umma_commit(d2_full);
          }
          if (j == 6 && tl + 1 < my_tiles) {  // X of the next tile, once G1(3) is done
            mbar_wait(x_empty, tl & 1);
            load_x(tl + 1);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ------------------------------------------- X split, then D1 -> H (thread = row)
    const int lt = threadIdx.x;  // row 0..127
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    for (int tl = 0; tl < my_tiles; ++tl) {
      mbar_wait(x_full, tl & 1);
      bool big = false;
#pragma unroll 1
      for (int kc = 0; kc < 4; ++kc) {
        uint8_t* ch = Xs + kc * FF_CHUNK;
        const float4* rp = reinterpret_cast<const float4*>(ch) + lt * 8;
        float4 x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = rp[q ^ (lt & 7)];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          big |= !(fabsf(x[q].x) <= A16_LIMIT) || !(fabsf(x[q].y) <= A16_LIMIT) ||
                 !(fabsf(x[q].z) <= A16_LIMIT) || !(fabsf(x[q].w) <= A16_LIMIT);
        asm volatile("bar.sync 2, 128;" ::: "memory");  // raw reads done before overwrite
        __half* a16 = reinterpret_cast<__half*>(ch);
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
          const float v[8] = {x[2 * k8].x,     x[2 * k8].y,     x[2 * k8].z,     x[2 * k8].w,
                              x[2 * k8 + 1].x, x[2 * k8 + 1].y, x[2 * k8 + 1].z, x[2 * k8 + 1].w};
          __align__(16) __half hi[8], lo[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            hi[e] = __float2half_rn(v[e]);
            lo[e] = __float2half_rn(v[e] - __half2float(hi[e]));
          }
          const int off = k8 * (BM * 8) + lt * 8;
          *reinterpret_cast<uint4*>(a16 + off) = *reinterpret_cast<const uint4*>(hi);
          *reinterpret_cast<uint4*>(a16 + 4096 + off) = *reinterpret_cast<const uint4*>(lo);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(x_ready);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int u = tl * 4 + c;
        mbar_wait(&d1_full[c & 1], (u >> 1) & 1);
        fence_after();
        const uint32_t tacc = D1 + (c & 1) * 128 + lane_off;
        if (u >= 1) mbar_wait(h_empty, (u - 1) & 1);  // G2(c-1) has read H
#pragma unroll 1
        for (int c0 = 0; c0 < 128; c0 += 32) {
          uint32_t r[32];
          TG_LD16(tacc + c0, r);
          TG_LD16(tacc + c0 + 16, (r + 16));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const float4* b4 = reinterpret_cast<const float4*>(a.b1 + c * 128 + c0);
          __half* h16 = reinterpret_cast<__half*>(Hs + (c0 >> 5) * FF_CHUNK);
#pragma unroll
          for (int k8 = 0; k8 < 4; ++k8) {
            const float4 bb0 = __ldg(b4 + 2 * k8), bb1 = __ldg(b4 + 2 * k8 + 1);
            const float bb[8] = {bb0.x, bb0.y, bb0.z, bb0.w, bb1.x, bb1.y, bb1.z, bb1.w};
            __align__(16) __half hi[8], lo[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              float v = __uint_as_float(r[8 * k8 + e]) * ASCALE + bb[e];
              v = v > 0.f ? v : 0.f;
              big |= !(v <= A16_LIMIT);
              hi[e] = __float2half_rn(v);
              lo[e] = __float2half_rn(v - __half2float(hi[e]));
            }
            const int off = k8 * (BM * 8) + lt * 8;
            *reinterpret_cast<uint4*>(h16 + off) = *reinterpret_cast<const uint4*>(hi);
            *reinterpret_cast<uint4*>(h16 + 4096 + off) = *reinterpret_cast<const uint4*>(lo);
          }
        }
        fence_before();
        mbar_arrive(&d1_empty[c & 1]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(h_full);
      }
      if (big) atomicOr(a.ovf, 1);
    }
  } else {
    // ------------------------------------------- LayerNorm epilogue (thread = row)
    const int ew = warp - 4;
    const int et = threadIdx.x - 128;
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    float* stg = epi + ew * 32 * 36;
    float* s_b2 = epi + 4 * 32 * 36;  // [128]
    float* s_g = s_b2 + 128;
    float* s_b = s_g + 128;
    s_b2[et] = a.b2[et];
    s_g[et] = a.ln ? a.ln_g[et] : 1.f;
    s_b[et] = a.ln ? a.ln_b[et] : 0.f;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const int rq = lane >> 3, c4 = lane & 7;
    auto ld4 = [](const float* p) { return *reinterpret_cast<const float4*>(p); };
    for (int tl = 0; tl < my_tiles; ++tl) {
      const int64_t rbase = (int64_t)(blockIdx.x + tl * gridDim.x) * BM + ew * 32;
      const int64_t row = rbase + lane;
      const bool rv = row < a.M;
      auto store32 = [&](float* C, int64_t ldc, int c0, const float* y) {
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(stg + lane * 36 + 4 * q) =
              make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i * 4 + rq;
          const int64_t gr = rbase + r;
          if (gr < a.M)
            *reinterpret_cast<float4*>(C + gr * ldc + c0 + c4 * 4) = ld4(stg + r * 36 + c4 * 4);
        }
      };
      mbar_wait(d2_full, tl & 1);
      fence_after();
      const uint32_t tacc = D2 + lane_off;
      if (!a.ln) {  // plain C = acc + b2
#pragma unroll 1
        for (int c0 = 0; c0 < 128; c0 += 32) {
          uint32_t u[32];
          TG_LD16(tacc + c0, u);
          TG_LD16(tacc + c0 + 16, (u + 16));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float y[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) y[j] = __uint_as_float(u[j]) * ASCALE + s_b2[c0 + j];
          store32(a.C, a.ldc, c0, y);
        }
        fence_before();
        mbar_arrive(d2_empty);
        continue;
      }
      // pass 1: x = acc + b2 + X (residual), kept in TMEM; running sum
      float s = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t u[32];
        TG_LD16(tacc + c0, u);
        TG_LD16(tacc + c0 + 16, (u + 16));
        float rr[32];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i * 4 + rq;
          const int64_t gr = rbase + r;
          const float4 v = gr < a.M ? __ldg(reinterpret_cast<const float4*>(
                                          a.X + gr * a.ldx + c0 + c4 * 4))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<float4*>(stg + r * 36 + c4 * 4) = v;
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = ld4(stg + lane * 36 + 4 * q);
          rr[4 * q] = v.x; rr[4 * q + 1] = v.y; rr[4 * q + 2] = v.z; rr[4 * q + 3] = v.w;
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float x = __uint_as_float(u[j]) * ASCALE + s_b2[c0 + j] + rr[j];
          s += x;
          u[j] = __float_as_uint(x);
        }
        TG_ST16(tacc + c0, u);
        TG_ST16(tacc + c0 + 16, (u + 16));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      const float mu = s / 128.f;
      float q = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t u[32];
        TG_LD16(tacc + c0, u);
        TG_LD16(tacc + c0 + 16, (u + 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float d = __uint_as_float(u[j]) - mu;
          q += d * d;
        }
      }
      const float inv = 1.f / sqrtf(q / 128.f + 1e-5f);
      const float* rs = (a.rowscale && rv) ? a.rowscale + (int64_t)a.row_fwd[row] * 128 : nullptr;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t u[32];
        TG_LD16(tacc + c0, u);
        TG_LD16(tacc + c0 + 16, (u + 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float y[32];
#pragma unroll
        for (int j = 0; j < 32; ++j)
          y[j] = s_g[c0 + j] * ((__uint_as_float(u[j]) - mu) * inv) + s_b[c0 + j];
        if (a.C) store32(a.C, a.ldc, c0, y);
        if (a.rowscale) {
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const float4 r4 = rs ? __ldg(reinterpret_cast<const float4*>(rs + c0) + q4)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
            y[4 * q4] *= r4.x; y[4 * q4 + 1] *= r4.y; y[4 * q4 + 2] *= r4.z; y[4 * q4 + 3] *= r4.w;
          }
          store32(a.C2, a.ldc2, c0, y);
        }
      }
      fence_before();
      mbar_arrive(d2_empty);
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 8) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}
