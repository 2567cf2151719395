// Layout probe: tcgen05.mma kind::f16 with an fp16 accumulator (idesc D format = F16).
// A (128 x 16) and B (64 x 16) hold small integers; prints how the 128 x 64 result is
// laid out across TMEM columns (packed two per 32-bit column, or one per column).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2010_12438_b200/csrc -o scripts/f16acc_probe scripts/f16acc_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "tcgen05.cuh"
using namespace go::ptx;

__global__ void probe(uint32_t* out) {
  __shared__ __align__(1024) __half a[128 * 16];
  __shared__ __align__(1024) __half b[64 * 16];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  // canonical K-major: element (row, k) at (k>>3)*(ROWS*8) + (row>>3)*64 + (row&7)*8 + (k&7)
  for (int i = threadIdx.x; i < 128 * 16; i += blockDim.x) {
    int row = i / 16, k = i % 16;
    a[(k >> 3) * (128 * 8) + (row >> 3) * 64 + (row & 7) * 8 + (k & 7)] = __float2half(k == 0 ? (float)row : 0.f);
  }
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) {
    int n = i / 16, k = i % 16;
    b[(k >> 3) * (64 * 8) + (n >> 3) * 64 + (n & 7) * 8 + (k & 7)] = __float2half(k == 0 ? (float)(n + 1) * 0.25f : 0.f);
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tm)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem(); fence_before(); __syncthreads(); fence_after();
  const uint32_t t = tm;
  if (threadIdx.x == 0) {
    // D format F16: bits [4,6) = 0
    const uint32_t id = ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    umma_ss_f16(t, sdesc(smem_u32(a), 128 * 16, 128), sdesc(smem_u32(b), 64 * 16, 128), id, 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after();
  uint32_t r[16];
  const int warp = threadIdx.x >> 5;
  for (int c = 0; c < 64; c += 16) {
    PTX_LD16(t + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) out[threadIdx.x * 64 + c + i] = r[i];
  }
  fence_before(); __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(t));
}

int main() {
  uint32_t* d; cudaMalloc(&d, 128 * 64 * 4);
  cudaMemset(d, 0, 128 * 64 * 4);
  probe<<<1, 128>>>(d);
  static uint32_t h[128 * 64];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int row : {0, 1, 5, 33, 127}) {
    printf("row %d:", row);
    for (int c = 0; c < 40; ++c) {
      uint32_t v = h[row * 64 + c];
      __half lo = __ushort_as_half((unsigned short)(v & 0xffff)), hi = __ushort_as_half((unsigned short)(v >> 16));
      printf(" [%g|%g]", __half2float(lo), __half2float(hi));
    }
    printf("\n");
  }
  printf("expected row r col n = r * (n+1)/4\n");
  return 0;
}
