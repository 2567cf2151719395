// Measures MUFU.EX2 throughput (ex2.approx.ftz.f32) and FP32 FMA throughput on the
// local GPU, so the task-head attention roofline has a measured exp2 denominator.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mufu_peak scripts/mufu_peak.cu
// Prints one JSON line: {"ex2_per_clk_per_sm": ..., "ex2_gops": ..., "fma_tflops": ...}
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int ILP = 8;

__global__ void ex2_kernel(float* out, float seed) {
  float v[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = -(seed + threadIdx.x * 1e-3f + i * 1e-2f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
      v[i] = -y;  // keeps the argument in (-1, 0]: ex2 of it stays in (0.5, 1]
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void fma_kernel(float* out, float seed) {
  float v[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = seed + threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) v[i] = fmaf(v[i], 0.999f, 1e-3f);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ex2 with a packed fp32 -> f16x2 conversion of each result pair: if the conversion
// shares the MUFU pipe the rate drops below ex2_kernel's
__global__ void ex2_cvt_kernel(float* out, float seed) {
  float v[ILP];
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = -(seed + threadIdx.x * 1e-3f + i * 1e-2f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; i += 2) {
      float y0, y1;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(v[i]));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y1) : "f"(v[i + 1]));
      uint32_t h;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(y1), "f"(y0));
      acc ^= h;
      v[i] = -y0;
      v[i + 1] = -y1;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)(acc & 1);
}

template <typename K>
static double time_kernel(K kern, int blocks, int threads, float* buf) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, threads>>>(buf, 0.5f);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(buf, 0.5f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5.0;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  float* buf;
  cudaMalloc(&buf, 16 << 20);
  const int threads = 512, blocks = p.multiProcessorCount * 4;
  const double ops = (double)blocks * threads * ITERS * ILP;
  double ms_e = time_kernel(ex2_kernel, blocks, threads, buf);
  double ms_f = time_kernel(fma_kernel, blocks, threads, buf);
  double ms_c = time_kernel(ex2_cvt_kernel, blocks, threads, buf);
  double ex2_s = ops / (ms_e * 1e-3);
  double fma_s = ops / (ms_f * 1e-3);
  fprintf(stderr, "ex2+cvt.f16x2 per pair: ex2 rate %.1f Gop/s (vs %.1f without)\n",
          ops / (ms_c * 1e-3) / 1e9, ex2_s / 1e9);
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"ex2_gops\": %.1f, \"ex2_per_clk_per_sm_at_attr_clock\": %.2f, "
         "\"fma_tflops\": %.2f, \"fma_per_clk_per_sm_at_attr_clock\": %.1f}\n",
         p.multiProcessorCount, clk_khz / 1e3, ex2_s / 1e9,
         ex2_s / (p.multiProcessorCount * clk_khz * 1e3), 2.0 * fma_s / 1e12,
         fma_s / (p.multiProcessorCount * clk_khz * 1e3));
  return 0;
}
