// Micro-benchmark: random float2 / float4 gather rate vs table size (exact sizes, modulo
// indexing), to pick encode pass-slice sizes.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int V>
__global__ void k_gather(const float4* __restrict__ t, uint32_t rows, uint64_t n, float* out, uint32_t seed) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t r = hash32((uint32_t)i * 8u + k + seed) % rows;  // float4 row
    if (V == 2) {
      const float2 v = __ldg(reinterpret_cast<const float2*>(t) + 2 * r + (k & 1));
      acc += v.x + v.y;
    } else {
      const float4 v = __ldg(t + r);
      acc += v.x + v.y + v.z + v.w;
    }
  }
  out[i] = acc;
}

int main() {
  const uint64_t n = 16u << 20;
  float4* t;
  float* out;
  cudaMalloc(&t, 512ull << 20);
  cudaMalloc(&out, n * 4);
  cudaMemset(t, 0, 512ull << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("table_MB  f2_Gacc/s  f4_Gacc/s\n");
  for (uint32_t mb : {8u, 16u, 24u, 32u, 40u, 48u, 56u, 64u, 72u, 80u, 88u, 96u, 104u, 112u, 120u, 128u, 160u, 256u}) {
    const uint32_t rows = (uint32_t)(((uint64_t)mb << 20) / 16u);
    float r2 = 0, r4 = 0;
    for (int v = 0; v < 2; ++v) {
      for (int w = 0; w < 2; ++w) {  // warm
        if (v == 0) k_gather<2><<<n / 256, 256>>>(t, rows, n, out, w);
        else k_gather<4><<<n / 256, 256>>>(t, rows, n, out, w);
      }
      cudaEventRecord(a);
      for (int rep = 0; rep < 5; ++rep) {
        if (v == 0) k_gather<2><<<n / 256, 256>>>(t, rows, n, out, 17 + rep);
        else k_gather<4><<<n / 256, 256>>>(t, rows, n, out, 17 + rep);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double rate = 5.0 * n * 8 / (ms * 1e-3) / 1e9;
      (v == 0 ? r2 : r4) = (float)rate;
    }
    printf("%8u  %9.1f  %9.1f\n", mb, r2, r4);
  }
  return 0;
}
