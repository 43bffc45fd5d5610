// Micro-benchmark: tcgen05.mma round-trip latency (issue -> commit -> mbarrier wait) for
// chains of dependent MMAs (same accumulator) and independent ones (distinct accumulators).
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "../../paper_2405_04416_b200/csrc/tc.cuh"
using namespace dg;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a_tmem), "l"(b),
      "r"(idesc), "r"(acc));
}

__global__ void k_lat(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) { tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  uint32_t phase = 0;
  const uint64_t a = tc::smem_desc(tc::smem_u32(sm), 2048, 128);
  const uint64_t b = tc::smem_desc(tc::smem_u32(sm + 32768), 1024, 128);
  const int Ns[3] = {8, 64, 128};
  int o = 0;
  for (int ni = 0; ni < 3; ++ni) {
    const uint32_t id = tc::idesc_bf16(128, Ns[ni], 0, 0);
    const uint32_t id64mn = tc::idesc_bf16(64, Ns[ni], 1, 1), id64k = tc::idesc_bf16(64, Ns[ni], 0, 0);
    const uint64_t amn = tc::smem_desc(tc::smem_u32(sm), 128, 2048), bmn = tc::smem_desc(tc::smem_u32(sm + 32768), 128, 2048);
    for (int mode = 0; mode < 5; ++mode) {       // 0: chain, 1: indep, 2: A in TMEM, 3: M=64 MN-major SS, 4: M=64 K-major SS
      for (int cnt = 1; cnt <= 32; cnt *= 2) {
        unsigned long long best = ~0ull;
        for (int rep = 0; rep < 5; ++rep) {
          __syncthreads();
          const unsigned long long t0 = clock64();
          if (warp == 0) {
            if (tc::elect_one()) {
              for (int i = 0; i < cnt; ++i) {
                if (mode == 2) mma_ts(tmem, tmem + 256, b, id, i > 0 ? 1u : 0u);
                else if (mode == 3) tc::mma_bf16(tmem, amn, bmn, id64mn, i > 0 ? 1u : 0u);
                else if (mode == 4) tc::mma_bf16(tmem, a, b, id64k, i > 0 ? 1u : 0u);
                else tc::mma_bf16(tmem + (mode ? (uint32_t)((i % 4) * 64) : 0u), a, b, id, i > 0 ? 1u : 0u);
              }
              tc::commit(&mbar);
            }
            __syncwarp();
          }
          tc::mbar_wait(&mbar, phase);
          phase ^= 1u;
          tc::fence_after();
          const unsigned long long t1 = clock64();
          if (t1 - t0 < best) best = t1 - t0;
        }
        if (threadIdx.x == 0) out[o] = best;
        ++o;
      }
    }
  }
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 128 * 8); cudaMemset(d, 0, 128 * 8);
  cudaFuncSetAttribute(k_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  k_lat<<<1, 128, 80 * 1024>>>(d);
  unsigned long long h[128] = {};
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  const int Ns[3] = {8, 64, 128};
  int o = 0;
  for (int ni = 0; ni < 3; ++ni)
    for (int mode = 0; mode < 5; ++mode) {
      const char* nm[5] = {"chain", "indep", "ts-ch", "m64mn", "m64k "};
      printf("N=%3d %s:", Ns[ni], nm[mode]);
      for (int cnt = 1; cnt <= 32; cnt *= 2) printf("  %2d:%5llu", cnt, h[o++]);
      printf("\n");
    }
  return 0;
}
