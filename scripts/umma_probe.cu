// Issue-rate probe for tcgen05.mma kind::tf32 at the small shapes the attention
// kernels use: cycles per MMA for M=128, K=8 and N in {16, 32, 64, 128, 256}, with A
// from shared memory (ss) or from TMEM (ts).  One CTA per SM, one issuing thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/umma_probe scripts/umma_probe.cu
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// KIND 0: kind::tf32 (K=8); KIND 1: kind::f16 with fp16 inputs (K=16)
template <int N, bool TS, int KIND = 0>
__global__ void probe(long long* out, int iters) {
  __shared__ __align__(1024) float a[128 * 8];
  __shared__ __align__(1024) float b[256 * 8];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) a[i] = 0.f;
  for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) b[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tm;
  if (threadIdx.x == 0) {
    const uint64_t da = sdesc(su32(a), 128 * 16, 128), db = sdesc(su32(b), N * 16, 128);
    const uint32_t id = KIND == 0 ? idesc(128, N)
                                  : ((1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (KIND == 1 && TS)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(t + 256),
                     "r"(t), "l"(db), "r"(id) : "memory");
      else if (KIND == 1)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(t + 256),
                     "l"(da), "l"(db), "r"(id) : "memory");
      else if (TS)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(t + 256),
                     "r"(t), "l"(db), "r"(id) : "memory");
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(t + 256),
                     "l"(da), "l"(db), "r"(id) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W%=;\n}\n" ::"r"(su32(&bar)) : "memory");
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int N, bool TS, int KIND = 0>
void run(long long* d, int sms) {
  const int iters = 4096;
  probe<N, TS, KIND><<<sms, 128>>>(d, iters);
  probe<N, TS, KIND><<<sms, 128>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const int K = KIND == 0 ? 8 : 16;
  printf("{\"kind\": \"%s\", \"M\": 128, \"N\": %d, \"K\": %d, \"a_from\": \"%s\", "
         "\"cycles_per_mma\": %.2f, \"flops_per_clk_per_sm\": %.1f}\n",
         KIND == 0 ? "tf32" : "f16", N, K, TS ? "tmem" : "smem", avg / iters,
         2.0 * 128 * N * K * iters / avg);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  run<16, false>(d, sms);
  run<32, false>(d, sms);
  run<64, false>(d, sms);
  run<128, false>(d, sms);
  run<256, false>(d, sms);
  run<16, true>(d, sms);
  run<32, true>(d, sms);
  run<64, true>(d, sms);
  run<128, true>(d, sms);
  run<16, false, 1>(d, sms);
  run<32, false, 1>(d, sms);
  run<64, false, 1>(d, sms);
  run<128, false, 1>(d, sms);
  run<16, true, 1>(d, sms);
  run<32, true, 1>(d, sms);
  run<64, true, 1>(d, sms);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
