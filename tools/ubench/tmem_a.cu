// Self-test: tcgen05.mma kind::f16 with the A operand in TMEM (M=128, K=16 per MMA).
// Establishes the TMEM A layout: lane = row m, 32-bit column j packs (k = 2j, 2j + 1) as
// (low, high) bf16 halves; checks D = A . B^T against a CPU reference for N = 16 and 64,
// and the hi/lo split product for a K=64 chain.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>
#include <cuda_bf16.h>
#include "../../paper_2405_04416_b200/csrc/tc.cuh"
using namespace dg;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a_tmem), "l"(b),
      "r"(idesc), "r"(acc));
}

// A: 128 x K (bf16, row-major), B: N x K (bf16 row-major) -> D 128 x N fp32
template <int N, int K>
__global__ void k_test(const uint16_t* A, const uint16_t* B, float* D, int swap) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B tile K-major canonical: byte(r, c) = ((c/8)*(N/8) + r/8)*128 + (r%8)*16 + (c%8)*2
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, c = e % K;
    *reinterpret_cast<uint16_t*>(sm + tc::core_offset(r, c, N)) = B[e];
  }
  if (warp == 0) tc::tmem_alloc(&slot, 256);
  if (tid == 0) { tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  const uint32_t a_col = 128;  // A at columns [128, 128 + K/2)
  // thread = row (warp w -> lanes 32w..)
  const int row = warp * 32 + lane;
  for (int c8 = 0; c8 < K / 16; ++c8) {
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) {
      const uint32_t lo = A[row * K + c8 * 16 + 2 * j], hi = A[row * K + c8 * 16 + 2 * j + 1];
      r[j] = swap ? ((lo << 16) | hi) : (lo | (hi << 16));
    }
    tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + a_col + c8 * 8, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) {
    if (tc::elect_one()) {
      const uint32_t id = tc::idesc_bf16(128, N, 0, 0);
      const uint32_t b_lbo = (N / 8) * 128;
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sm), b_lbo, 128);
      for (int k = 0; k < K / 16; ++k)
        mma_ts(tmem, tmem + a_col + k * 8, bd + ((k * 2 * b_lbo) >> 4), id, k > 0);
      tc::commit(&mbar);
    }
    __syncwarp();
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  for (int c = 0; c < N; c += 8) {
    float v[8];
    tc::tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    tc::tmem_wait_ld();
    for (int j = 0; j < 8; ++j) D[row * N + c + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 256);
}

template <int N, int K>
void run(int swap) {
  std::mt19937 rng(7);
  std::uniform_int_distribution<int> U(-8, 8);
  std::vector<uint16_t> A(128 * K), B(N * K);
  std::vector<float> Af(128 * K), Bf(N * K);
  for (size_t i = 0; i < A.size(); ++i) { Af[i] = U(rng) / 4.0f; __nv_bfloat16 b = __float2bfloat16(Af[i]); A[i] = *reinterpret_cast<uint16_t*>(&b); }
  for (size_t i = 0; i < B.size(); ++i) { Bf[i] = U(rng) / 4.0f; __nv_bfloat16 b = __float2bfloat16(Bf[i]); B[i] = *reinterpret_cast<uint16_t*>(&b); }
  uint16_t *dA, *dB; float* dD;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_test<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_test<N, K><<<1, 128, 64 * 1024>>>(dA, dB, dD, swap);
  std::vector<float> D(128 * N);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += double(Af[m * K + k]) * Bf[n * K + k];
      maxerr = std::max(maxerr, std::fabs(ref - D[m * N + n]));
    }
  printf("N=%d K=%d swap=%d: max|err| = %g  (%s)\n", N, K, swap, maxerr, cudaGetErrorString(e));
}

int main() {
  run<16, 16>(0); run<16, 16>(1);
  run<64, 16>(0); run<64, 64>(0); run<16, 64>(0);
  return 0;
}
