// Micro-benchmark: random float2 gathers and float2/float4 reductions into a table of S bytes.
// Tells the effective L2 capacity for random row access and the red throughput on this B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_random l2_random.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void k_gather(const float2* __restrict__ t, uint32_t mask, uint64_t n, float2* out, uint32_t seed) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t r = hash32((uint32_t)i * 8u + k + seed) & mask;
    const float2 v = __ldg(t + r);
    acc.x += v.x; acc.y += v.y;
  }
  out[i] = acc;
}

__global__ void k_red2(float2* __restrict__ t, uint32_t mask, uint64_t n, uint32_t seed) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t r = hash32((uint32_t)i * 8u + k + seed) & mask;
    atomicAdd(t + r, make_float2(1.f, 2.f));
  }
}

// 4 float4 reds per thread (the same 8 rows as pairs r, r^1)
__global__ void k_red4(float2* __restrict__ t, uint32_t mask, uint64_t n, uint32_t seed) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t r = hash32((uint32_t)i * 8u + k + seed) & mask & ~1u;
    atomicAdd(reinterpret_cast<float4*>(t + r), make_float4(1.f, 2.f, 3.f, 4.f));
  }
}

int main() {
  const uint64_t n = 16u << 20;  // threads (x 8 accesses)
  float2 *t, *out;
  cudaMalloc(&t, 512ull << 20);
  cudaMalloc(&out, n * 8);
  cudaMemset(t, 0, 512ull << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  printf("table_MB  gather_ms  gather_Gacc/s  red2_ms  red2_Gop/s  red4_ms  red4_Gop/s(x2 rows)\n");
  for (uint32_t mb : {8u, 16u, 32u, 48u, 64u, 80u, 96u, 112u, 128u, 192u, 256u, 512u}) {
    const uint32_t rows = (uint32_t)((uint64_t)mb << 20) / 8u;
    uint32_t mask = 1; while (mask < rows) mask <<= 1; mask = mask - 1;
    if (mask + 1 > rows) mask = (mask >> 1);  // power of two <= rows
    const uint64_t bytes = (uint64_t)(mask + 1) * 8;
    float ms[3];
    for (int which = 0; which < 3; ++which) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (which == 0) k_gather<<<(n + 255) / 256, 256>>>(t, mask, n, out, rep);
        if (which == 1) k_red2<<<(n + 255) / 256, 256>>>(t, mask, n, rep);
        if (which == 2) k_red4<<<(n + 255) / 256, 256>>>(t, mask, n, rep);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms[which], a, b);
      }
    }
    printf("%8.0f  %9.3f  %13.1f  %7.3f  %10.1f  %7.3f  %10.1f\n", bytes / 1048576.0, ms[0], n * 8 / ms[0] / 1e6,
           ms[1], n * 8 / ms[1] / 1e6, ms[2], n * 4 / ms[2] / 1e6);
  }
  cudaError_t e = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
