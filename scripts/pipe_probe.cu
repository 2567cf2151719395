// Which pipe does cvt.rn.f16x2.f32 (F2FP) issue on?  Throughput of F2FP alone, MUFU.EX2
// alone, and interleaved (if both share the XU pipe the mix runs at the sum of the costs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/pipe_probe scripts/pipe_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
constexpr int IT = 4096;
__global__ void f2fp_k(uint32_t* o, float s) {
  float a[8]; uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) a[i] = s + threadIdx.x * 1e-3f + i;
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      uint32_t r;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i + 1]));
      acc += r;
      a[i] = __uint_as_float(__float_as_uint(a[i]) ^ (r & 1));
    }
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void ex2_k(uint32_t* o, float s) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -(s + threadIdx.x * 1e-3f + i * 0.1f);
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i]));
      a[i] = -y;
    }
  }
  float t = 0; for (int i = 0; i < 8; ++i) t += a[i];
  o[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(t);
}
// 8 ex2 + 4 cvt per iteration (the MUFU-path mix of the attention softmax)
__global__ void mix_k(uint32_t* o, float s) {
  float a[8]; uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) a[i] = -(s + threadIdx.x * 1e-3f + i * 0.1f);
  for (int it = 0; it < IT; ++it) {
    float y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y[i]) : "f"(a[i]));
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      uint32_t r;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(y[i]), "f"(y[i + 1]));
      acc += r;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = -y[i];
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <class K>
double tk(K k, uint32_t* b, int blocks) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<blocks, 512>>>(b, 0.5f);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<blocks, 512>>>(b, 0.5f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 5;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* b; cudaMalloc(&b, 64 << 20);
  const int blocks = sms * 4;
  const double thr = (double)blocks * 512 * IT;
  double t1 = tk(f2fp_k, b, blocks), t2 = tk(ex2_k, b, blocks), t3 = tk(mix_k, b, blocks);
  printf("{\"f2fp_per_s\": %.3e, \"ex2_per_s\": %.3e, \"mix_ex2_per_s\": %.3e, "
         "\"mix_f2fp_per_s\": %.3e}\n", thr * 4 / (t1 * 1e-3), thr * 8 / (t2 * 1e-3),
         thr * 8 / (t3 * 1e-3), thr * 4 / (t3 * 1e-3));
  return 0;
}
