// Self-test: tcgen05.mma M=64 (cta_group::1) with the D (and TMEM A) address at lane offset
// 0 or 16.  Prints where the 64 result rows land in the 128 TMEM lanes, for A from shared
// memory (ss) and A from TMEM (ts, A stored in the same lane pattern as D).
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

constexpr int N = 16, K = 16;
// A: 64 x K, B: N x K (bf16 row-major).  out: 128 lanes x N columns read back.
__global__ void k_test(const uint16_t* A, const uint16_t* B, float* out, int lane_off, int ts) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* sa = sm;          // A K-major canonical [64 x K]
  uint8_t* sb = sm + 8192;   // B K-major canonical [N x K]
  for (int e = tid; e < 64 * K; e += blockDim.x) {
    const int r = e / K, c = e % K;
    *reinterpret_cast<uint16_t*>(sa + tc::core_offset(r, c, 64)) = A[e];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, c = e % K;
    *reinterpret_cast<uint16_t*>(sb + tc::core_offset(r, c, N)) = B[e];
  }
  if (warp == 0) tc::tmem_alloc(&slot, 256);
  if (tid == 0) { tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  // zero D region for all lanes
  {
    uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int c = 0; c < 64; c += 8) tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + c, z);
  }
  const uint32_t a_col = 128;
  if (ts) {  // A row i at lane (i % 16) + 32 (i / 16) + lane_off
    const int li = lane - lane_off;
    uint32_t r[8];
    const bool mine = li >= 0 && li < 16;
    const int row = mine ? warp * 16 + li : 0;
    for (int j = 0; j < 8; ++j) {
      const uint32_t lo = A[row * K + 2 * j], hi = A[row * K + 2 * j + 1];
      r[j] = mine ? (lo | (hi << 16)) : 0u;
    }
    tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + a_col, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) {
    if (tc::elect_one()) {
      const uint32_t id = tc::idesc_bf16(64, N, 0, 0);
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sb), (N / 8) * 128, 128);
      const uint32_t d = tmem + ((uint32_t)lane_off << 16);
      if (ts) {
        tc::mma_bf16_ts(d, tmem + ((uint32_t)lane_off << 16) + a_col, bd, id, 0);
      } else {
        const uint64_t ad = tc::smem_desc(tc::smem_u32(sa), (64 / 8) * 128, 128);
        tc::mma_bf16(d, ad, bd, id, 0);
      }
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
    for (int j = 0; j < 8; ++j) out[(warp * 32 + lane) * N + c + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 256);
}

int main() {
  std::mt19937 rng(7);
  std::uniform_int_distribution<int> U(-8, 8);
  std::vector<uint16_t> A(64 * K), B(N * K);
  std::vector<float> Af(64 * K), Bf(N * K);
  for (size_t i = 0; i < A.size(); ++i) { Af[i] = U(rng) / 4.0f; __nv_bfloat16 b = __float2bfloat16(Af[i]); A[i] = *reinterpret_cast<uint16_t*>(&b); }
  for (size_t i = 0; i < B.size(); ++i) { Bf[i] = U(rng) / 4.0f; __nv_bfloat16 b = __float2bfloat16(Bf[i]); B[i] = *reinterpret_cast<uint16_t*>(&b); }
  std::vector<double> ref(64 * N);
  for (int m = 0; m < 64; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += double(Af[m * K + k]) * Bf[n * K + k];
      ref[m * N + n] = s;
    }
  uint16_t *dA, *dB; float* dO;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dO, 128 * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  for (int ts = 0; ts < 2; ++ts)
    for (int off : {0, 16}) {
      cudaMemset(dO, 0, 128 * N * 4);
      k_test<<<1, 128, 32 * 1024>>>(dA, dB, dO, off, ts);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> O(128 * N);
      cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
      // for each result row m, find the lane holding it
      int ok = 0;
      std::vector<int> where(64, -1);
      for (int m = 0; m < 64; ++m)
        for (int l = 0; l < 128; ++l) {
          bool match = true;
          for (int n = 0; n < N; ++n) match &= std::fabs(O[l * N + n] - ref[m * N + n]) < 1e-3;
          if (match) { where[m] = l; ++ok; break; }
        }
      int nonzero = 0;
      for (int l = 0; l < 128; ++l) { bool nz = false; for (int n = 0; n < N; ++n) nz |= O[l * N + n] != 0.f; nonzero += nz; }
      printf("%s lane_off=%2d: %s  rows found %d/64, nonzero lanes %d; row->lane:", ts ? "ts" : "ss", off,
             cudaGetErrorString(e), ok, nonzero);
      for (int m = 0; m < 64; m += 7) printf(" %d->%d", m, where[m]);
      printf("\n");
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
