// kernels_tc.cu — tcgen05 self-test: proves the operand-layout conventions of tc.cuh on the
// device (K-major forward GEMM, MN-major-B input-gradient GEMM, MN-major-A/B weight-gradient
// GEMM accumulated over K = 128 samples), each as a 3-term split-bf16 product with fp32
// accumulation in TMEM.  Exposed as dg_selftest_tcgen05 for the GPU tests.
#include <cuda_bf16.h>

#include "kernels.h"
#include "tc.cuh"

namespace dg {

namespace {

// A[128x64], B[64x64], X[128x32] fp32 in global; outputs Y0 = A B^T, Y1 = A B, Y2 = A^T X.
__global__ void __launch_bounds__(128, 1) k_tc_selftest(const float* __restrict__ A,
                                                        const float* __restrict__ B,
                                                        const float* __restrict__ X,
                                                        float* __restrict__ Y0,
                                                        float* __restrict__ Y1,
                                                        float* __restrict__ Y2) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t(*sA)[128 * 64 * 2] = reinterpret_cast<uint8_t(*)[128 * 64 * 2]>(smem);
  uint8_t(*sB)[64 * 64 * 2] = reinterpret_cast<uint8_t(*)[64 * 64 * 2]>(smem + 2 * 128 * 64 * 2);
  uint8_t(*sX)[128 * 32 * 2] =
      reinterpret_cast<uint8_t(*)[128 * 32 * 2]>(smem + 2 * 128 * 64 * 2 + 2 * 64 * 64 * 2);
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 64; e += 128) {
    const int r = e / 64, c = e % 64;
    uint16_t h, l;
    tc::split_bf16(A[e], h, l);
    const uint32_t off = tc::core_offset(r, c, 128);
    *reinterpret_cast<uint16_t*>(sA[0] + off) = h;
    *reinterpret_cast<uint16_t*>(sA[1] + off) = l;
  }
  for (int e = tid; e < 64 * 64; e += 128) {
    const int r = e / 64, c = e % 64;
    uint16_t h, l;
    tc::split_bf16(B[e], h, l);
    const uint32_t off = tc::core_offset(r, c, 64);
    *reinterpret_cast<uint16_t*>(sB[0] + off) = h;
    *reinterpret_cast<uint16_t*>(sB[1] + off) = l;
  }
  for (int e = tid; e < 128 * 32; e += 128) {
    const int r = e / 32, c = e % 32;
    uint16_t h, l;
    tc::split_bf16(X[e], h, l);
    const uint32_t off = tc::core_offset(r, c, 128);
    *reinterpret_cast<uint16_t*>(sX[0] + off) = h;
    *reinterpret_cast<uint16_t*>(sX[1] + off) = l;
  }
  if (warp == 0) tc::tmem_alloc(&tslot, 256);
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tslot;
  if (tid == 0) {
    const uint32_t a0 = tc::smem_u32(sA[0]), a1 = tc::smem_u32(sA[1]);
    const uint32_t b0 = tc::smem_u32(sB[0]), b1 = tc::smem_u32(sB[1]);
    const uint32_t x0 = tc::smem_u32(sX[0]), x1 = tc::smem_u32(sX[1]);
    // Y0 = A B^T : A K-major (SBO 128, LBO 2048), B K-major [N=64 x K=64] (SBO 128, LBO 1024)
    {
      const uint32_t id = tc::idesc_bf16(128, 64, 0, 0);
      for (int k = 0; k < 4; ++k) {
        const uint32_t ao = k * 2 * 2048, bo = k * 2 * 1024;
        tc::mma_bf16(tbase + 0, tc::smem_desc(a0 + ao, 2048, 128), tc::smem_desc(b0 + bo, 1024, 128), id, k > 0);
        tc::mma_bf16(tbase + 0, tc::smem_desc(a0 + ao, 2048, 128), tc::smem_desc(b1 + bo, 1024, 128), id, 1);
        tc::mma_bf16(tbase + 0, tc::smem_desc(a1 + ao, 2048, 128), tc::smem_desc(b0 + bo, 1024, 128), id, 1);
      }
    }
    // Y1 = A B : B stored [K=64 rows x N=64 cols] read MN-major (SBO 1024, LBO 128)
    {
      const uint32_t id = tc::idesc_bf16(128, 64, 0, 1);
      for (int k = 0; k < 4; ++k) {
        const uint32_t ao = k * 2 * 2048, bo = k * 2 * 128;
        tc::mma_bf16(tbase + 64, tc::smem_desc(a0 + ao, 2048, 128), tc::smem_desc(b0 + bo, 128, 1024), id, k > 0);
        tc::mma_bf16(tbase + 64, tc::smem_desc(a0 + ao, 2048, 128), tc::smem_desc(b1 + bo, 128, 1024), id, 1);
        tc::mma_bf16(tbase + 64, tc::smem_desc(a1 + ao, 2048, 128), tc::smem_desc(b0 + bo, 128, 1024), id, 1);
      }
    }
    // Y2 = A^T X : M = 64 (A cols), N = 32, K = 128 samples; both MN-major (SBO 2048, LBO 128)
    {
      const uint32_t id = tc::idesc_bf16(64, 32, 1, 1);
      for (int k = 0; k < 8; ++k) {
        const uint32_t o = k * 2 * 128;
        tc::mma_bf16(tbase + 128, tc::smem_desc(a0 + o, 128, 2048), tc::smem_desc(x0 + o, 128, 2048), id, k > 0);
        tc::mma_bf16(tbase + 128, tc::smem_desc(a0 + o, 128, 2048), tc::smem_desc(x1 + o, 128, 2048), id, 1);
        tc::mma_bf16(tbase + 128, tc::smem_desc(a1 + o, 128, 2048), tc::smem_desc(x0 + o, 128, 2048), id, 1);
      }
    }
    tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  for (int c0 = 0; c0 < 64; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tbase + lane_base + c0, v);
    tc::tmem_wait_ld();
    for (int i = 0; i < 16; ++i) Y0[tid * 64 + c0 + i] = v[i];
    tc::tmem_ld16(tbase + lane_base + 64 + c0, v);
    tc::tmem_wait_ld();
    for (int i = 0; i < 16; ++i) Y1[tid * 64 + c0 + i] = v[i];
  }
  for (int c0 = 0; c0 < 32; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tbase + lane_base + 128 + c0, v);
    tc::tmem_wait_ld();
    const int lane = tid & 31;
    if (lane < 16) {  // M = 64: row m lives in lane (m % 16) + 32 (m / 16)
      const int m = warp * 16 + lane;
      for (int i = 0; i < 16; ++i) Y2[m * 32 + c0 + i] = v[i];
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tbase, 256);
}

}  // namespace

int tc_selftest(const float* A, const float* B, const float* X, float* Y0, float* Y1, float* Y2,
                cudaStream_t s) {
  const int bytes = 2 * 128 * 64 * 2 + 2 * 64 * 64 * 2 + 2 * 128 * 32 * 2;
  cudaFuncSetAttribute(k_tc_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  k_tc_selftest<<<1, 128, bytes, s>>>(A, B, X, Y0, Y1, Y2);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace dg
