// Softmax-exponential throughput probe for the task-head attention (tc_attention16.cu):
// 16 fp32 scores -> 8 packed fp16x2 probabilities per thread per iteration, with NP of
// the 8 pairs computed by the FMA-pipe polynomial (exp2_poly_f16x2 in tcgen05.cuh)
// and the rest by MUFU.EX2.  Also measures tcgen05.mma kind::f16 issue cost with one
// (dependent) or four (independent) accumulators.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2010_12438_b200/csrc \
//        -o scripts/exp_probe scripts/exp_probe.cu
#include <cstdint>
#include <cstdio>

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tcgen05.cuh"

using namespace go::ptx;

constexpr int ITERS = 2048;

template <int NP>
__global__ void __launch_bounds__(384, 2) softmax_probe(uint32_t* out, float shift) {
  __shared__ float xs[384 * 16];
  for (int i = 0; i < 16; ++i) xs[threadIdx.x * 16 + i] = -0.37f * i - shift * threadIdx.x * 1e-3f + 3.f;
  __syncthreads();
  uint32_t acc = 0;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(&xs[threadIdx.x * 16]);
  for (int it = 0; it < ITERS; ++it) {
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; i += 4)
      asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(x[i]), "=f"(x[i + 1]), "=f"(x[i + 2]), "=f"(x[i + 3])
                   : "r"(base + i * 4) : "memory");
    uint32_t pk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < NP)
        pk[i] = exp2_poly_f16x2(x[2 * i], x[2 * i + 1]);
      else
        pk[i] = pack_f16x2_rn(ex2_approx(x[2 * i]), ex2_approx(x[2 * i + 1]));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= pk[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// accuracy of the polynomial against exact exp2 over [-14, 15] (fp16 output)
__global__ void poly_accuracy(float* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const float x0 = -14.f + 29.f * (2 * i) / (2.f * 65536.f);
  const float x1 = -14.f + 29.f * (2 * i + 1) / (2.f * 65536.f);
  const uint32_t p = exp2_poly_f16x2(x0, x1);
  const float y0 = __half2float(__ushort_as_half((unsigned short)(p & 0xffff)));
  const float y1 = __half2float(__ushort_as_half((unsigned short)(p >> 16)));
  const double e0 = fabs(y0 / exp2((double)x0) - 1.0), e1 = fabs(y1 / exp2((double)x1) - 1.0);
  err[2 * i] = (float)e0;
  err[2 * i + 1] = (float)e1;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// kind::f16 MMA issue cost, M=128; NACC accumulators round-robin (1 = dependent chain)
template <int N, bool TS, int NACC, int M = 128>
__global__ void mma_probe(long long* out, int iters) {
  __shared__ __align__(1024) uint16_t a[128 * 16];
  __shared__ __align__(1024) uint16_t b[256 * 16];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  for (int i = threadIdx.x; i < 128 * 16; i += blockDim.x) a[i] = 0;
  for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) b[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = tm;
  if (threadIdx.x == 0) {
    const uint64_t da = sdesc(su32(a), 128 * 16, 128), db = sdesc(su32(b), N * 16, 128);
    constexpr uint32_t id = idesc_f16(M, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = t + 256 + (i % NACC) * (N <= 64 ? 64 : N);
      if (TS)
        umma_ts_f16(d, t, db, id, 1);
      else
        umma_ss_f16(d, da, db, id, 1);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int N, bool TS, int NACC, int M = 128>
void run_mma(long long* d, int sms) {
  const int iters = 4096;
  mma_probe<N, TS, NACC, M><<<sms, 128>>>(d, iters);
  mma_probe<N, TS, NACC, M><<<sms, 128>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("{\"probe\": \"mma\", \"kind\": \"f16\", \"M\": %d, \"N\": %d, \"K\": 16, \"a_from\": \"%s\", "
         "\"accumulators\": %d, \"cycles_per_mma\": %.2f}\n",
         M, N, TS ? "tmem" : "smem", NACC, avg / iters);
}

template <int NP>
void run_softmax(uint32_t* buf, int sms, double clk_hz) {
  const int blocks = sms * 2, threads = 384;
  softmax_probe<NP><<<blocks, threads>>>(buf, 1.f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) softmax_probe<NP><<<blocks, threads>>>(buf, 1.f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  const double elems = 5.0 * blocks * threads * ITERS * 16.0;
  const double rate = elems / (ms * 1e-3);
  printf("{\"probe\": \"softmax\", \"poly_pairs_of_8\": %d, \"gexp_s\": %.1f, \"per_clk_per_sm_at_attr_clock\": %.2f}\n",
         NP, rate / 1e9, rate / (sms * clk_hz));
}

int main() {
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  uint32_t* buf;
  cudaMalloc(&buf, 64 << 20);
  float* err;
  cudaMalloc(&err, 2 * 65536 * 4);
  poly_accuracy<<<256, 256>>>(err);
  static float herr[2 * 65536];
  cudaMemcpy(herr, err, sizeof(herr), cudaMemcpyDeviceToHost);
  double mx = 0, mean = 0;
  for (int i = 0; i < 2 * 65536; ++i) {
    mx = herr[i] > mx ? herr[i] : mx;
    mean += herr[i];
  }
  printf("{\"probe\": \"poly_accuracy\", \"max_rel_err\": %.3e, \"mean_rel_err\": %.3e}\n", mx,
         mean / (2 * 65536));
  const double clk = clk_khz * 1e3;
  run_softmax<0>(buf, sms, clk);
  run_softmax<2>(buf, sms, clk);
  run_softmax<3>(buf, sms, clk);
  run_softmax<4>(buf, sms, clk);
  run_softmax<5>(buf, sms, clk);
  run_softmax<6>(buf, sms, clk);
  run_softmax<8>(buf, sms, clk);
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  run_mma<16, true, 1>(d, sms);
  run_mma<16, true, 4>(d, sms);
  run_mma<32, false, 1>(d, sms);
  run_mma<32, false, 4>(d, sms);
  run_mma<64, false, 1>(d, sms);
  run_mma<64, false, 4>(d, sms);
  run_mma<128, false, 1>(d, sms);
  run_mma<128, false, 2>(d, sms);
  run_mma<16, false, 4, 64>(d, sms);
  run_mma<128, false, 2, 64>(d, sms);
  run_mma<256, false, 1, 64>(d, sms);
  run_mma<256, false, 1>(d, sms);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
