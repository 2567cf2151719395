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
// 9 warps: 0-3 drain D1 into H (thread = row); 4-7 split X into fp16 hi/lo, then run the
// LayerNorm epilogue of the previous tile (thread = row); 8 loads (TMA for X, bulk copies
// for the weight chunks) and issues the MMAs.  TMEM: D1 x 2 (256 columns) + D2 x 2 (256).
// SMEM: X hi/lo 64 KB + H hi/lo 64 KB (four 32-column k-slots, each with its own
// full / empty barrier) + a 4-stage ring of 16 KB weight chunks + epilogue staging.
//
// Round 2 (ncu source counters on the round-1 kernel: the weight ring never stalled the MMA
// thread; it spun on the single H buffer and the single D2): H is handed over per 32-column
// k-slot, so G2(c) starts on the first slot the D1 warps finish and E1(c+1) refills a slot
// as soon as G2(c) has read it; D2 is double-buffered, so the LayerNorm of tile t runs
// under tile t+1's MMAs; the X split moved to the epilogue warps (idle while the MMAs run);
// the D1 drain uses fp32x2 / fp16x2 arithmetic with the bias in shared memory; the MMA
// warp issues converged (one elected lane) and a separate producer warp refills the
// weight ring, so the issuing thread never waits for a stage to drain.  ncu launch list
// (8 cfg4 forwards, 640,008 rows per launch): 775 -> 469 us per launch; tensor pipe
// 29% -> 55% active.  The kernel is now bound by shared-memory bandwidth: the three
// SS-operand MMA passes read 1.5 MB per 128-row tile and the TMA / split / drain /
// epilogue traffic adds 1.3 MB (l1tex shared wavefronts 48% + tensor-core 55%).

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
constexpr int FF_EPI = 4 * 32 * 36 * 4 + 512 * 4 + 512 * 4;  // staging, b2/g/b, b1
constexpr size_t FF_SMEM = 1024 + 8 * FF_CHUNK + FF_NSW * FF_CHUNK + FF_EPI + 1024;

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
        "l"(*reinterpret_cast<uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}

constexpr int FF_THREADS = 320;  // + warp 9: the load producer

__global__ void __launch_bounds__(FF_THREADS, 1)
    ffn_kernel(const __grid_constant__ CUtensorMap tmX, FfnArgs a, int ntiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* Xs = base;                    // 4 chunks
  uint8_t* Hs = base + 4 * FF_CHUNK;     // 4 k-slots
  uint8_t* Ws = base + 8 * FF_CHUNK;     // FF_NSW stages
  float* epi = reinterpret_cast<float*>(Ws + FF_NSW * FF_CHUNK);
  float* s_b2 = epi + 4 * 32 * 36;  // [128]
  float* s_g = s_b2 + 128;
  float* s_b = s_g + 128;
  float* s_b1 = s_b + 256;          // [512]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(epi) + FF_EPI);
  uint64_t* x_full = bars + 0;
  uint64_t* x_ready = bars + 1;
  uint64_t* x_empty = bars + 2;
  uint64_t* h_full = bars + 3;     // [4] per k-slot
  uint64_t* h_empty = bars + 7;    // [4]
  uint64_t* d2_full = bars + 11;   // [2]
  uint64_t* d2_empty = bars + 13;  // [2]
  uint64_t* d1_full = bars + 15;   // [2]
  uint64_t* d1_empty = bars + 17;  // [2]
  uint64_t* w_full = bars + 19;    // [FF_NSW]
  uint64_t* w_done = bars + 19 + FF_NSW;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 19 + 2 * FF_NSW);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr float ASCALE = 1.f / (1 << W16_SHIFT);

  if (warp == 8) {
    if (lane == 0) {
      mbar_init(x_full, 1);
      mbar_init(x_ready, 128);
      mbar_init(x_empty, 1);
      for (int k = 0; k < 4; ++k) {
        mbar_init(&h_full[k], 128);
        mbar_init(&h_empty[k], 1);
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&d2_full[b], 1);
        mbar_init(&d2_empty[b], 128);
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
  } else if (warp < 4) {
    for (int i = threadIdx.x; i < 512; i += 128) s_b1[i] = a.b1[i];
  } else if (warp < 8) {
    const int et = threadIdx.x - 128;
    s_b2[et] = a.b2[et];
    s_g[et] = a.ln ? a.ln_g[et] : 1.f;
    s_b[et] = a.ln ? a.ln_b[et] : 0.f;
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t D1 = tbase, D2 = tbase + 256;  // D1[b] at +128 b, D2[b] at +128 b

  // job order per tile: G1 0, G1 1, G2 0, G1 2, G2 1, G1 3, G2 2, G2 3 (4 weight chunks
  // each: G1(c) -> W1 block c, k-chunks 0..3; G2(c) -> W2 k-chunks 4c..4c+3).  (Issuing
  // G1(3) before G2(1), to release the X tile earlier, measured 2.5% slower.)
  // (bit-packed tables: a dynamically indexed local array would live in local memory)
  auto job_g1 = [](int j) { return ((0x2Bu >> j) & 1u) != 0; };  // G1 at j = 0,1,3,5
  auto job_c = [](int j) { return (int)((0x32312010u >> (4 * j)) & 0xFu); };
  const int total = my_tiles * 32;  // weight chunks
  if (warp == 9) {
    // ------------------------------------------- producer: X tiles and weight chunks
    if (lane == 0) {
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
      for (int g = 0; g < total; ++g) {
        const int tl = g >> 5;
        // X of the next tile once G1(3) (chunks 20..23) has read this one (chunk 27's
        // weight slot waits for chunk 23 anyway)
        if ((g & 31) == 27 && tl + 1 < my_tiles) {
          mbar_wait(x_empty, tl & 1);
          load_x(tl + 1);
        }
        if (g >= FF_NSW) mbar_wait(&w_done[g % FF_NSW], ((g / FF_NSW) - 1) & 1);
        load_w(g);
      }
    }
    __syncwarp();
  } else if (warp == 8) {
    // ------------------------------------------- MMA issue (warp converged, one elected lane)
    constexpr uint32_t ID = idesc_f16(BM, 128);
    // descriptors of the chunk bases; K steps add (bytes >> 4) to the start-address field
    const uint64_t dX = sdesc(smem_u32(Xs), 2048, 128), dH = sdesc(smem_u32(Hs), 2048, 128);
    const uint64_t dW = sdesc(smem_u32(Ws), 128 * 16, 128);
    int g = 0;
    for (int tl = 0; tl < my_tiles; ++tl) {
      for (int j = 0; j < 8; ++j) {
        const int c = job_c(j);
        const bool g1 = job_g1(j);
        const int u = tl * 4 + c;  // use index of D1[c & 1] and of the H slots
        uint32_t dacc;
        if (g1) {
          if (c == 0) mbar_wait(x_ready, tl & 1);
          if (u >= 2) mbar_wait(&d1_empty[c & 1], ((u >> 1) - 1) & 1);
          dacc = D1 + (c & 1) * 128;
        } else {
          if (c == 0 && tl >= 2) mbar_wait(&d2_empty[tl & 1], ((tl >> 1) - 1) & 1);
          dacc = D2 + (tl & 1) * 128;
        }
        const uint64_t dA0 = g1 ? dX : dH;
        for (int kc = 0; kc < 4; ++kc, ++g) {
          const int s = g % FF_NSW;
          if (!g1) mbar_wait(&h_full[kc], u & 1);
          mbar_wait(&w_full[s], (g / FF_NSW) & 1);
          fence_after();
          if (elect_one()) {
            const uint64_t da = dA0 + (uint64_t)(kc * (FF_CHUNK >> 4));
            const uint64_t db = dW + (uint64_t)(s * (FF_CHUNK >> 4));
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t dah = da + kk * 256, dal = da + 512 + kk * 256;
              const uint64_t dbh = db + kk * 256, dbl = db + 512 + kk * 256;
              const uint32_t acc0 = g1 ? (kc > 0 || kk > 0) : (c > 0 || kc > 0 || kk > 0);
              umma_ss_f16(dacc, dah, dbh, ID, acc0);
              umma_ss_f16(dacc, dah, dbl, ID, 1);
              umma_ss_f16(dacc, dal, dbh, ID, 1);
            }
            umma_commit(&w_done[s]);
            if (!g1) umma_commit(&h_empty[kc]);
            if (kc == 3) {
              if (g1) {
                umma_commit(&d1_full[c & 1]);
                if (c == 3) umma_commit(x_empty);
              } else if (c == 3) {
                umma_commit(&d2_full[tl & 1]);
              }
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------- D1 -> relu(D1 + b1) -> H hi/lo (thread = row)
    const int lt = threadIdx.x;  // row 0..127
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const float2 ascale2 = make_float2(ASCALE, ASCALE);
    __half2 hmax = __float2half2_rn(0.f);
    for (int tl = 0; tl < my_tiles; ++tl) {
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int u = tl * 4 + c;
        mbar_wait(&d1_full[c & 1], (u >> 1) & 1);
        fence_after();
        const uint32_t tacc = D1 + (c & 1) * 128 + lane_off;
#pragma unroll 1
        for (int kc = 0; kc < 4; ++kc) {
          uint32_t r[32];
          TG_LD16(tacc + kc * 32, r);
          TG_LD16(tacc + kc * 32 + 16, (r + 16));
          if (u >= 1) mbar_wait(&h_empty[kc], (u - 1) & 1);  // G2(c-1) has read slot kc
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const float2* b2p = reinterpret_cast<const float2*>(s_b1 + c * 128 + kc * 32);
          uint32_t* h16 = reinterpret_cast<uint32_t*>(Hs + kc * FF_CHUNK);
#pragma unroll
          for (int k8 = 0; k8 < 4; ++k8) {
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int jj = 8 * k8 + 2 * e;
              float2 v = ffma2(make_float2(__uint_as_float(r[jj]), __uint_as_float(r[jj + 1])),
                               ascale2, b2p[jj >> 1]);
              v.x = v.x > 0.f ? v.x : 0.f;
              v.y = v.y > 0.f ? v.y : 0.f;
              const __half2 h = __floats2half2_rn(v.x, v.y);
              hmax = __hmax2(hmax, h);
              const __half2 l = __float22half2_rn(fsub2(v, __half22float2(h)));
              hi[e] = *reinterpret_cast<const uint32_t*>(&h);
              lo[e] = *reinterpret_cast<const uint32_t*>(&l);
            }
            const int off = (k8 * (BM * 8) + lt * 8) >> 1;  // in 32-bit words
            *reinterpret_cast<uint4*>(h16 + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            *reinterpret_cast<uint4*>(h16 + 2048 + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&h_full[kc]);
        }
        fence_before();
        mbar_arrive(&d1_empty[c & 1]);
      }
    }
    // range check on the fp16-rounded values (running __hmax2): flags every relu(v) above
    // 2^15 and, conservatively, values that round onto it
    const float2 hm = __half22float2(hmax);
    if (!(hm.x < A16_LIMIT) || !(hm.y < A16_LIMIT)) atomicOr(a.ovf, 1);
  } else {
    // ------------------------- X split (thread = row), then LayerNorm of the previous tile
    const int ew = warp - 4;
    const int et = threadIdx.x - 128;  // row 0..127
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    float* stg = epi + ew * 32 * 36;
    const int rq = lane >> 3, c4 = lane & 7;
    auto ld4 = [](const float* p) { return *reinterpret_cast<const float4*>(p); };
    bool big = false;
    auto split_x = [&](int tl) {
      mbar_wait(x_full, tl & 1);
#pragma unroll 1
      for (int kc = 0; kc < 4; ++kc) {
        uint8_t* ch = Xs + kc * FF_CHUNK;
        const float4* rp = reinterpret_cast<const float4*>(ch) + et * 8;
        float4 x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = rp[q ^ (et & 7)];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          big |= !(fabsf(x[q].x) <= A16_LIMIT) || !(fabsf(x[q].y) <= A16_LIMIT) ||
                 !(fabsf(x[q].z) <= A16_LIMIT) || !(fabsf(x[q].w) <= A16_LIMIT);
        asm volatile("bar.sync 2, 128;" ::: "memory");  // raw reads done before overwrite
        uint32_t* a16 = reinterpret_cast<uint32_t*>(ch);
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
          const float2 v[4] = {make_float2(x[2 * k8].x, x[2 * k8].y),
                               make_float2(x[2 * k8].z, x[2 * k8].w),
                               make_float2(x[2 * k8 + 1].x, x[2 * k8 + 1].y),
                               make_float2(x[2 * k8 + 1].z, x[2 * k8 + 1].w)};
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const __half2 h = __float22half2_rn(v[e]);
            const __half2 l = __float22half2_rn(fsub2(v[e], __half22float2(h)));
            hi[e] = *reinterpret_cast<const uint32_t*>(&h);
            lo[e] = *reinterpret_cast<const uint32_t*>(&l);
          }
          const int off = (k8 * (BM * 8) + et * 8) >> 1;
          *reinterpret_cast<uint4*>(a16 + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<uint4*>(a16 + 2048 + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(x_ready);
    };
    auto epilogue = [&](int tl) {
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
      mbar_wait(&d2_full[tl & 1], (tl >> 1) & 1);
      fence_after();
      const uint32_t tacc = D2 + (tl & 1) * 128 + lane_off;
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
        mbar_arrive(&d2_empty[tl & 1]);
        return;
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
      mbar_arrive(&d2_empty[tl & 1]);
    };
    for (int tl = 0; tl <= my_tiles; ++tl) {
      if (tl < my_tiles) split_x(tl);
      if (tl >= 1) epilogue(tl - 1);
    }
    if (big) atomicOr(a.ovf, 1);
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 8) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}
