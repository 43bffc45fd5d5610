// Self-test: thread/register -> (TMEM lane, column) maps of the 16-lane tcgen05.ld/st shapes
// (.16x64b, .16x128b, .16x256b, .x1) at lane offsets 0 and 16 of a warp's sub-partition —
// the fragment layouts a two-half-tile (M = 64, lane halves) MLP backward would need.
// Writes value lane * 1000 + column with 32x32b stores, loads with each shape, prints the map.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "../../paper_2405_04416_b200/csrc/tc.cuh"
using namespace dg;

__device__ __forceinline__ void st8(uint32_t a, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

__global__ void k(uint32_t* out, int lane_off) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc(&slot, 32);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t t = slot + ((uint32_t)(warp * 32) << 16);
  uint32_t r[8];
  for (int c = 0; c < 8; ++c) r[c] = (uint32_t)((warp * 32 + lane) * 1000 + c);
  st8(t, r);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  const uint32_t a = t + ((uint32_t)lane_off << 16);
  uint32_t v[4] = {0, 0, 0, 0};
  // 16x64b.x1: 1 register; 16x128b.x1: 2; 16x256b.x1: 4
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(v[0]) : "r"(a));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  out[(0 * 4 + warp) * 32 * 4 + lane * 4 + 0] = v[0];
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(a));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  out[(1 * 4 + warp) * 32 * 4 + lane * 4 + 0] = v[0];
  out[(1 * 4 + warp) * 32 * 4 + lane * 4 + 1] = v[1];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(a));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 4; ++j) out[(2 * 4 + warp) * 32 * 4 + lane * 4 + j] = v[j];
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(slot, 32);
}

int main() {
  uint32_t* d;
  const int n = 3 * 4 * 32 * 4;
  cudaMalloc(&d, n * 4);
  static uint32_t h[3 * 4 * 32 * 4];
  const char* names[3] = {"16x64b.x1", "16x128b.x1", "16x256b.x1"};
  const int regs[3] = {1, 2, 4};
  for (int off : {0, 16}) {
    cudaMemset(d, 0xff, n * 4);
    k<<<1, 128>>>(d, off);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, n * 4, cudaMemcpyDeviceToHost);
    printf("lane offset %d: %s\n", off, cudaGetErrorString(e));
    for (int s = 0; s < 3; ++s) {
      printf("  %s (warp 1, value = lane*1000 + col):\n", names[s]);
      for (int lane = 0; lane < 32; ++lane) {
        printf("    t%02d:", lane);
        for (int j = 0; j < regs[s]; ++j) {
          const uint32_t v = h[(s * 4 + 1) * 32 * 4 + lane * 4 + j];
          printf(" r%d=(L%u,c%u)", j, v / 1000 - 32, v % 1000);
        }
        printf("\n");
      }
    }
  }
  return 0;
}
