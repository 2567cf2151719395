// Throughput and accuracy of the packed-fp16 MUFU exponential (ex2.approx.f16x2) against
// the fp32 one, for the task-head softmax (VERDICT r1 "next" #5): if the MUFU returns two
// fp16 exponentials per issue, P = 2^S' can come from MUFU alone (S' is packed to fp16 for
// the polynomial half already).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ex2h_probe scripts/ex2h_probe.cu
// Prints one JSON line.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int ILP = 8;

__global__ void ex2_f32_kernel(float* out, float seed) {
  float v[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = -(seed + threadIdx.x * 1e-3f + i * 1e-2f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
      v[i] = -y;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ILP independent f16x2 chains: each ex2.approx.f16x2 produces two exponentials
__global__ void ex2_f16x2_kernel(float* out, float seed) {
  uint32_t v[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    __half2 h = __floats2half2_rn(-(seed + threadIdx.x * 1e-3f + i * 1e-2f), -(seed + i * 2e-2f));
    v[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      uint32_t y;
      asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(v[i]));
      v[i] = y ^ 0x80008000u;  // negate both halves: arguments stay in (-1, 0]
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    __half2 h = *reinterpret_cast<__half2*>(&v[i]);
    s += __low2float(h) + __high2float(h);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// the softmax's pattern: two fp32 scores -> cvt.rn.f16x2.f32 -> ex2.approx.f16x2
__global__ void cvt_ex2_f16x2_kernel(float* out, float seed) {
  float v[2 * ILP];
#pragma unroll
  for (int i = 0; i < 2 * ILP; ++i) v[i] = -(seed + threadIdx.x * 1e-3f + i * 1e-2f);
  uint32_t acc = 0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      uint32_t h, y;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(v[2 * i + 1]), "f"(v[2 * i]));
      asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(h));
      acc += y;
      v[2 * i] += 1e-7f;
      v[2 * i + 1] -= 1e-7f;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(acc & 0xFF) + v[0];
}

// accuracy over the fixed-offset softmax's range [-14, 15.5]
__global__ void accuracy_kernel(float* maxrel) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = 1 << 20;
  if (i >= n) return;
  const float x = -14.f + 29.5f * (float)i / (float)n;
  __half hx = __float2half_rn(x);  // the kernel rounds S' to fp16 first
  __half2 h2 = __halves2half2(hx, hx);
  uint32_t y;
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(*reinterpret_cast<uint32_t*>(&h2)));
  const float got = __low2float(*reinterpret_cast<__half2*>(&y));
  const double want = exp2((double)x);
  const float rel = (float)(fabs(got - want) / want);
  atomicMax(reinterpret_cast<int*>(maxrel), __float_as_int(rel));
  // the same error on the fp16-rounded argument (what the polynomial half also sees)
  const double want_h = exp2((double)__half2float(hx));
  const float rel_h = (float)(fabs(got - want_h) / want_h);
  atomicMax(reinterpret_cast<int*>(maxrel) + 1, __float_as_int(rel_h));
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
  float* buf;
  cudaMalloc(&buf, 16 << 20);
  const int threads = 512, blocks = p.multiProcessorCount * 4;
  const double instr = (double)blocks * threads * ITERS * ILP;
  const double t32 = time_kernel(ex2_f32_kernel, blocks, threads, buf);
  const double t16 = time_kernel(ex2_f16x2_kernel, blocks, threads, buf);
  const double tcv = time_kernel(cvt_ex2_f16x2_kernel, blocks, threads, buf);
  float* mr;
  cudaMalloc(&mr, 8);
  cudaMemset(mr, 0, 8);
  accuracy_kernel<<<(1 << 20) / 256, 256>>>(mr);
  float rel[2];
  cudaMemcpy(rel, mr, 8, cudaMemcpyDeviceToHost);
  printf("{\"ex2_f32_gexp_s\": %.1f, \"ex2_f16x2_gexp_s\": %.1f, \"cvt_ex2_f16x2_gexp_s\": %.1f, "
         "\"f16x2_max_rel_err\": %.3g, \"f16x2_max_rel_err_vs_rounded_arg\": %.3g}\n",
         instr / (t32 * 1e-3) / 1e9, 2 * instr / (t16 * 1e-3) / 1e9,
         2 * instr / (tcv * 1e-3) / 1e9, rel[0], rel[1]);
  return 0;
}
