// kernels_mlp_tc.cu — stage 4 on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// The fused density + colour MLP (field.cpp:230-327, mlp.cpp:55-138) for a tile of 128
// samples of one field.  Every layer is a tcgen05.mma GEMM with operands staged in shared
// memory (canonical no-swizzle core-matrix layout, tc.cuh) and the fp32 accumulator in TMEM;
// one elected thread issues the MMAs, tcgen05.commit arrives on an mbarrier, and the warps
// run the epilogue (tcgen05.ld -> bias/activation/clip -> split -> next operand in smem).
//
// Precision: each operand x is split into bf16 hi + bf16 lo (x = hi + lo + O(2^-17 |x|)) and
// every product is hi*hi + hi*lo + lo*hi accumulated in fp32 (3 MMAs per K step) — the
// error-compensated ("split-bf16") scheme SURVEY §2.3 requires, since plain TF32/bf16 misses
// the 1e-4 bar.
//
// Forward (k_mlp_fwd_tc):  X[128x32] -> H1 = relu(X Wd0^T + b) [64] -> raw = H1 Wd1^T + b [16]
//   -> Cin = [clip(raw1..15) | SH16(dir) | app] [48] -> C1 = act(Cin Wc0^T + b) [64]
//   -> C2 = act(C1 Wc1^T + b) [64] -> rgb = sigmoid(clip(C2 Wc2^T + b)) [3], sigma = exp(clip(raw0)).
#include <cuda_bf16.h>

#include "dg_common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace dg {

namespace {

constexpr int TM = 128;   // samples per tile (MMA M)
constexpr int NTH = 256;  // 8 warps: warp w reads TMEM lane quadrant w % 4, column half w / 4

// Weight operand tiles (B, K-major): rows = out (padded), cols = in (padded).
struct TcWeights {
  uint8_t d0[2][64 * 32 * 2];
  uint8_t d1[2][16 * 64 * 2];
  uint8_t c0[2][64 * 48 * 2];
  uint8_t c1[2][64 * 64 * 2];
  uint8_t c2[2][16 * 64 * 2];
  float bd0[64], bd1[16], bc0[64], bc1[64], bc2[16];
};

struct FwdTcSmem {
  TcWeights w;
  uint8_t a[2][TM * 64 * 2];  // activation operand (A, K-major), hi / lo
  float sig_raw[TM];
  uint64_t mbar;
  uint32_t tslot;
};

__device__ __forceinline__ void put_split(uint8_t* hi, uint8_t* lo, uint32_t off, float v) {
  uint16_t h, l;
  tc::split_bf16(v, h, l);
  *reinterpret_cast<uint16_t*>(hi + off) = h;
  *reinterpret_cast<uint16_t*>(lo + off) = l;
}

// Stage one layer's W[out][in] (fp32, global) as split-bf16 K-major tiles [Np x Kp].
__device__ void stage_layer(const float* __restrict__ W, int out, int in, int Np, int Kp,
                            uint8_t* hi, uint8_t* lo) {
  for (int e = threadIdx.x; e < Np * Kp; e += NTH) {
    const int o = e / Kp, i = e % Kp;
    const float v = (o < out && i < in) ? W[o * in + i] : 0.f;
    put_split(hi, lo, tc::core_offset(o, i, Np), v);
  }
}

__device__ void stage_weights_tc(const FieldDesc& fd, const float* __restrict__ params, TcWeights& w) {
  const float* base = params + fd.base;
  const int enc = (int)fd.L * 2, cin = 31 + (int)fd.app_dim;
  stage_layer(base + fd.dw0, 64, enc, 64, 32, w.d0[0], w.d0[1]);
  stage_layer(base + fd.dw1, 16, 64, 16, 64, w.d1[0], w.d1[1]);
  stage_layer(base + fd.cw0, 64, cin, 64, 48, w.c0[0], w.c0[1]);
  stage_layer(base + fd.cw1, 64, 64, 64, 64, w.c1[0], w.c1[1]);
  stage_layer(base + fd.cw2, 3, 64, 16, 64, w.c2[0], w.c2[1]);
  for (int e = threadIdx.x; e < 64; e += NTH) {
    w.bd0[e] = base[fd.db0 + e];
    w.bc0[e] = base[fd.cb0 + e];
    w.bc1[e] = base[fd.cb1 + e];
  }
  for (int e = threadIdx.x; e < 16; e += NTH) {
    w.bd1[e] = base[fd.db1 + e];
    w.bc2[e] = e < 3 ? base[fd.cb2 + e] : 0.f;
  }
}

// D[tm][N] (+)= A[tm x K] . B[N x K]^T, split-bf16 (3 MMAs per 16-wide K step).
// A tile rows = TM (K-major, SBO 128, LBO TM/8*128); B tile rows = N (SBO 128, LBO N/8*128).
__device__ __forceinline__ void gemm_kmajor(uint32_t d_tmem, const uint8_t (*a)[TM * 64 * 2],
                                            const uint8_t* b_hi, const uint8_t* b_lo, int N, int K,
                                            bool accumulate) {
  const uint32_t id = tc::idesc_bf16(TM, N, 0, 0);
  const uint32_t a0 = tc::smem_u32(a[0]), a1 = tc::smem_u32(a[1]);
  const uint32_t b0 = tc::smem_u32(b_hi), b1 = tc::smem_u32(b_lo);
  const uint32_t a_lbo = (TM / 8) * 128, b_lbo = (N / 8) * 128;
  for (int k = 0; k < K / 16; ++k) {
    const uint32_t ao = k * 2 * a_lbo, bo = k * 2 * b_lbo;
    const uint64_t ah = tc::smem_desc(a0 + ao, a_lbo, 128), al = tc::smem_desc(a1 + ao, a_lbo, 128);
    const uint64_t bh = tc::smem_desc(b0 + bo, b_lbo, 128), bl = tc::smem_desc(b1 + bo, b_lbo, 128);
    tc::mma_bf16(d_tmem, ah, bh, id, (accumulate || k > 0) ? 1u : 0u);
    tc::mma_bf16(d_tmem, ah, bl, id, 1u);
    tc::mma_bf16(d_tmem, al, bh, id, 1u);
  }
}


// D[TM x N] = A[TM x K] . B[N x K]^T for an A tile given as hi/lo base pointers.
__device__ __forceinline__ void gemm_kmajor_t(uint32_t d_tmem, const uint8_t* a_hi, const uint8_t* a_lo,
                                              const uint8_t* b_hi, const uint8_t* b_lo, int N, int K) {
  const uint32_t id = tc::idesc_bf16(TM, N, 0, 0);
  const uint32_t a0 = tc::smem_u32(a_hi), a1 = tc::smem_u32(a_lo);
  const uint32_t b0 = tc::smem_u32(b_hi), b1 = tc::smem_u32(b_lo);
  const uint32_t a_lbo = (TM / 8) * 128, b_lbo = (N / 8) * 128;
  for (int k = 0; k < K / 16; ++k) {
    const uint32_t ao = k * 2 * a_lbo, bo = k * 2 * b_lbo;
    const uint64_t ah = tc::smem_desc(a0 + ao, a_lbo, 128), al = tc::smem_desc(a1 + ao, a_lbo, 128);
    const uint64_t bh = tc::smem_desc(b0 + bo, b_lbo, 128), bl = tc::smem_desc(b1 + bo, b_lbo, 128);
    tc::mma_bf16(d_tmem, ah, bh, id, k > 0 ? 1u : 0u);
    tc::mma_bf16(d_tmem, ah, bl, id, 1u);
    tc::mma_bf16(d_tmem, al, bh, id, 1u);
  }
}

// Write 8 consecutive columns [c0, c0+8) of row r of the activation operand.
__device__ __forceinline__ void put_chunk(uint8_t (*a)[TM * 64 * 2], int r, int c0, const float* v) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint16_t h0, l0, h1, l1;
    tc::split_bf16(v[2 * j], h0, l0);
    tc::split_bf16(v[2 * j + 1], h1, l1);
    h[j] = (uint32_t)h0 | ((uint32_t)h1 << 16);
    l[j] = (uint32_t)l0 | ((uint32_t)l1 << 16);
  }
  const uint32_t off = tc::core_offset(r, c0, TM);
  *reinterpret_cast<uint4*>(a[0] + off) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(a[1] + off) = make_uint4(l[0], l[1], l[2], l[3]);
}

__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + expf(-x)); }
__device__ __forceinline__ float clip15(float v) { return v > 15.f ? 15.f : (v < -15.f ? -15.f : v); }

__device__ __forceinline__ void sh16(float x, float y, float z, float* o) {  // sh.hpp:14-35
  const float xy = x * y, xz = x * z, yz = y * z, x2 = x * x, y2 = y * y, z2 = z * z;
  o[0] = 0.28209479177387814f;
  o[1] = -0.48860251190291987f * y;
  o[2] = 0.48860251190291987f * z;
  o[3] = -0.48860251190291987f * x;
  o[4] = 1.0925484305920792f * xy;
  o[5] = -1.0925484305920792f * yz;
  o[6] = 0.31539156525252005f * (3.0f * z2 - 1.0f);
  o[7] = -1.0925484305920792f * xz;
  o[8] = 0.5462742152960396f * (x2 - y2);
  o[9] = -0.5900435899266435f * y * (3.0f * x2 - y2);
  o[10] = 2.890611442640554f * xy * z;
  o[11] = -0.4570457994644658f * y * (5.0f * z2 - 1.0f);
  o[12] = 0.3731763325901154f * z * (5.0f * z2 - 3.0f);
  o[13] = -0.4570457994644658f * x * (5.0f * z2 - 1.0f);
  o[14] = 1.445305721320277f * z * (x2 - y2);
  o[15] = -0.5900435899266435f * x * (x2 - 3.0f * y2);
}

__device__ __forceinline__ int tile_field(const MlpLaunch& m, uint32_t tile) {
  int f = 0;
  while (f + 1 < (int)m.n_fields && tile >= m.tile_off[f + 1]) ++f;
  return f;
}

// Sync point between an epilogue (generic smem writes / TMEM reads) and the next MMA issue.
__device__ __forceinline__ void to_mma() {
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
}

// Load 32 consecutive TMEM columns [c0, c0+32) of this thread's lane into v.
__device__ __forceinline__ void ld32(uint32_t taddr, float* v) {
  float a[16], b[16];
  tc::tmem_ld16(taddr, a);
  tc::tmem_ld16(taddr + 16, b);
  tc::tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = a[i];
    v[16 + i] = b[i];
  }
}

__global__ void __launch_bounds__(NTH, 2) k_mlp_fwd_tc(MlpLaunch m) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  FwdTcSmem& sm = *reinterpret_cast<FwdTcSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, half = warp >> 2;
  const int row = quad * 32 + lane;  // TMEM lane == sample row of the tile
  if (warp == 0) tc::tmem_alloc(&sm.tslot, 64);
  if (tid == 0) {
    tc::mbar_init(&sm.mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = sm.tslot;
  const uint32_t my_lanes = tmem + ((uint32_t)(quad * 32) << 16);
  uint32_t phase = 0;
  int loaded = -1;
  auto mma_done = [&]() {
    if (tid == 0) tc::commit(&sm.mbar);
    tc::mbar_wait(&sm.mbar, phase);
    phase ^= 1u;
    tc::fence_after();
  };
  for (uint32_t tile = blockIdx.x; tile < m.n_tiles; tile += gridDim.x) {
    const int f = tile_field(m, tile);
    const FieldDesc& fd = m.fields[f];
    const uint64_t s0 = m.field_off[f] + (uint64_t)(tile - m.tile_off[f]) * TM;
    const uint64_t rem = m.field_off[f + 1] - s0;
    const int count = rem < (uint64_t)TM ? (int)rem : TM;
    if (f != loaded) {
      __syncthreads();
      stage_weights_tc(fd, m.params, sm.w);
      loaded = f;
    }
    const int act_c = fd.coarse ? 2 : 1;
    const bool valid = row < count;
    const uint64_t gs = s0 + row;
    // ---- X tile: thread (row, half) writes levels [8 half, 8 half + 8) = 2 chunks ----
    {
      float v[16];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int l = half * 8 + j;
        float2 x = make_float2(0.f, 0.f);
        if (valid && l < (int)m.levels)
          x = reinterpret_cast<const float2*>(m.X)[(uint64_t)l * m.x_stride + gs];
        v[2 * j] = x.x;
        v[2 * j + 1] = x.y;
      }
      put_chunk(sm.a, row, half * 16, v);
      put_chunk(sm.a, row, half * 16 + 8, v + 8);
    }
    to_mma();
    // ---- L1: H1 = relu(X Wd0^T + b) ----
    if (tid == 0) gemm_kmajor(tmem, sm.a, sm.w.d0[0], sm.w.d0[1], 64, 32, false);
    mma_done();
    {
      float v[32];
      ld32(my_lanes + half * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i] + sm.w.bd0[half * 32 + i], 0.f);
#pragma unroll
      for (int c = 0; c < 4; ++c) put_chunk(sm.a, row, half * 32 + 8 * c, v + 8 * c);
    }
    to_mma();
    // ---- L2: raw16 = H1 Wd1^T + b ; Cin = [clip(raw1..15) | SH16 | app | 0] ----
    if (tid == 0) gemm_kmajor(tmem, sm.a, sm.w.d1[0], sm.w.d1[1], 16, 64, false);
    mma_done();
    {
      float raw[16];
      tc::tmem_ld16(my_lanes, raw);
      tc::tmem_wait_ld();
      float cin[48];
#pragma unroll
      for (int i = 0; i < 16; ++i) raw[i] = clip15(raw[i] + sm.w.bd1[i]);
#pragma unroll
      for (int i = 0; i < 15; ++i) cin[i] = raw[1 + i];
      float sh[16];
      const float* app = nullptr;
      if (valid) {
        const RayRec& r = m.rec[m.s_item[gs]];
        sh16((float)r.d[0], (float)r.d[1], (float)r.d[2], sh);
        app = m.app_per_sample ? m.app_override + gs * fd.app_dim
                               : (m.app_override ? m.app_override : m.app_table + (uint64_t)r.img * fd.app_dim);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) sh[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) cin[15 + i] = sh[i];
      for (int i = 0; i < 17; ++i) cin[31 + i] = (app && i < (int)fd.app_dim) ? app[i] : 0.f;
      if (half == 0) {
        sm.sig_raw[row] = raw[0];
        put_chunk(sm.a, row, 0, cin);
        put_chunk(sm.a, row, 8, cin + 8);
        put_chunk(sm.a, row, 16, cin + 16);
      } else {
        put_chunk(sm.a, row, 24, cin + 24);
        put_chunk(sm.a, row, 32, cin + 32);
        put_chunk(sm.a, row, 40, cin + 40);
      }
    }
    to_mma();
    // ---- L3: C1 = act(Cin Wc0^T + b) ----
    if (tid == 0) gemm_kmajor(tmem, sm.a, sm.w.c0[0], sm.w.c0[1], 64, 48, false);
    mma_done();
    {
      float v[32];
      ld32(my_lanes + half * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float z = v[i] + sm.w.bc0[half * 32 + i];
        v[i] = act_c == 2 ? sigm(z) : fmaxf(z, 0.f);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) put_chunk(sm.a, row, half * 32 + 8 * c, v + 8 * c);
    }
    to_mma();
    // ---- L4: C2 = act(C1 Wc1^T + b) ----
    if (tid == 0) gemm_kmajor(tmem, sm.a, sm.w.c1[0], sm.w.c1[1], 64, 64, false);
    mma_done();
    {
      float v[32];
      ld32(my_lanes + half * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float z = v[i] + sm.w.bc1[half * 32 + i];
        v[i] = act_c == 2 ? sigm(z) : fmaxf(z, 0.f);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) put_chunk(sm.a, row, half * 32 + 8 * c, v + 8 * c);
    }
    to_mma();
    // ---- L5: rgb = sigmoid(clip(C2 Wc2^T + b)) ----
    if (tid == 0) gemm_kmajor(tmem, sm.a, sm.w.c2[0], sm.w.c2[1], 16, 64, false);
    mma_done();
    {
      float v[16];
      tc::tmem_ld16(my_lanes, v);
      tc::tmem_wait_ld();
      if (half == 0 && valid)
        m.out[gs] = make_float4(expf(sm.sig_raw[row]), sigm(clip15(v[0] + sm.w.bc2[0])),
                                sigm(clip15(v[1] + sm.w.bc2[1])), sigm(clip15(v[2] + sm.w.bc2[2])));
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 64);
}


// ============================================================================ backward
// Per tile of 128 samples: recompute the forward (keeping every layer input in smem), then
//   B1  G5  = d raw_rgb (clip/sigmoid adjoint)            dWc2 += G5^T C2 ; dC2 = G5 Wc2
//   B2  G4  = dC2 * act'(C2)                              dWc1 += G4^T C1 ; dC1 = G4 Wc1
//   B3  G3  = dC1 * act'(C1)                              dWc0 += G3^T Cin; dCin = G3 Wc0[:, :16]
//   B4  G2  = [sigma path, clip-masked dCin[0..14]]       dWd1 += G2^T H1 ; dH1 = G2 Wd1
//   B5  G1  = dH1 * relu'(H1)                             dWd0 += G1^T X  ; dX = G1 Wd0
//   B6  dX -> global (level-major), for the hash-grid backward.
// The weight gradients dW = G^T A are M=64 tcgen05 GEMMs over K = 128 samples that read the
// G and A tiles through MN-major descriptors (no transposed copies) and accumulate in TMEM for
// every tile a CTA processes; each activation tile carries an extra ones column so the same
// GEMM yields the bias gradient.  TMEM is flushed with one atomicAdd per weight per CTA.
constexpr int XW = 40, HW = 72, CW = 56;  // tile widths incl. the ones chunk

struct BwdTcSmem {
  TcWeights w;
  uint8_t g5[2][TM * 16 * 2];  // followed by >= 12 KB of valid smem (M=64 MN-major reads 64 cols)
  uint8_t x[2][TM * XW * 2];
  uint8_t h1[2][TM * HW * 2];
  uint8_t cin[2][TM * CW * 2];
  uint8_t c1[2][TM * HW * 2];
  uint8_t c2[2][TM * HW * 2];
  float sig_raw[TM];
  float gsig[TM];
  uint32_t dmask[TM];
  uint64_t mbar;
  uint32_t tslot;
};

// TMEM columns: [0,64) transient accumulator; dW accumulators (M = 64 rows = out features).
constexpr uint32_t TD_C2 = 128, TD_C1 = 200, TD_C0 = 272, TD_D1 = 328, TD_D0 = 400;

// Write 8 consecutive columns of row r into a tile with TM rows (any width).
__device__ __forceinline__ void put8(uint8_t* hi, uint8_t* lo, int r, int c0, const float* v) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint16_t h0, l0, h1, l1;
    tc::split_bf16(v[2 * j], h0, l0);
    tc::split_bf16(v[2 * j + 1], h1, l1);
    h[j] = (uint32_t)h0 | ((uint32_t)h1 << 16);
    l[j] = (uint32_t)l0 | ((uint32_t)l1 << 16);
  }
  const uint32_t off = tc::core_offset(r, c0, TM);
  *reinterpret_cast<uint4*>(hi + off) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(lo + off) = make_uint4(l[0], l[1], l[2], l[3]);
}

// Read back 8 consecutive columns of row r (hi + lo).
__device__ __forceinline__ void get8(const uint8_t* hi, const uint8_t* lo, int r, int c0, float* v) {
  const uint32_t off = tc::core_offset(r, c0, TM);
  const uint4 h = *reinterpret_cast<const uint4*>(hi + off);
  const uint4 l = *reinterpret_cast<const uint4*>(lo + off);
  const uint32_t hh[4] = {h.x, h.y, h.z, h.w}, ll[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v[2 * j] = __uint_as_float(hh[j] << 16) + __uint_as_float(ll[j] << 16);
    v[2 * j + 1] = __uint_as_float(hh[j] & 0xffff0000u) + __uint_as_float(ll[j] & 0xffff0000u);
  }
}

// D (M=64 x N) (+)= G^T A over K = TM samples; G tile (TM x >=64 cols span), A tile (TM x N);
// both read MN-major (SBO = TM/8*128, LBO = 128).
__device__ __forceinline__ void gemm_wgrad(uint32_t d_tmem, const uint8_t* g_hi, const uint8_t* g_lo,
                                           const uint8_t* a_hi, const uint8_t* a_lo, int N,
                                           bool accumulate) {
  const uint32_t id = tc::idesc_bf16(64, N, 1, 1);
  const uint32_t g0 = tc::smem_u32(g_hi), g1 = tc::smem_u32(g_lo);
  const uint32_t a0 = tc::smem_u32(a_hi), a1 = tc::smem_u32(a_lo);
  constexpr uint32_t SBO = (TM / 8) * 128;
  for (int k = 0; k < TM / 16; ++k) {
    const uint32_t o = k * 256;
    const uint64_t gh = tc::smem_desc(g0 + o, 128, SBO), gl = tc::smem_desc(g1 + o, 128, SBO);
    const uint64_t ah = tc::smem_desc(a0 + o, 128, SBO), al = tc::smem_desc(a1 + o, 128, SBO);
    tc::mma_bf16(d_tmem, gh, ah, id, (accumulate || k > 0) ? 1u : 0u);
    tc::mma_bf16(d_tmem, gh, al, id, 1u);
    tc::mma_bf16(d_tmem, gl, ah, id, 1u);
  }
}

// D (TM x N) = G W : G tile K-major [TM x K=out], W tile stored [Wrows=out x cols=in]
// read MN-major (SBO = Wrows/8*128, LBO = 128); N = number of leading input columns.
__device__ __forceinline__ void gemm_igrad(uint32_t d_tmem, const uint8_t* g_hi, const uint8_t* g_lo,
                                           const uint8_t* w_hi, const uint8_t* w_lo, int Wrows, int N,
                                           int K) {
  const uint32_t id = tc::idesc_bf16(TM, N, 0, 1);
  const uint32_t g0 = tc::smem_u32(g_hi), g1 = tc::smem_u32(g_lo);
  const uint32_t w0 = tc::smem_u32(w_hi), w1 = tc::smem_u32(w_lo);
  constexpr uint32_t G_LBO = (TM / 8) * 128;
  const uint32_t W_SBO = (uint32_t)(Wrows / 8) * 128;
  for (int k = 0; k < K / 16; ++k) {
    const uint32_t go = k * 2 * G_LBO, wo = k * 256;
    const uint64_t gh = tc::smem_desc(g0 + go, G_LBO, 128), gl = tc::smem_desc(g1 + go, G_LBO, 128);
    const uint64_t wh = tc::smem_desc(w0 + wo, 128, W_SBO), wl = tc::smem_desc(w1 + wo, 128, W_SBO);
    tc::mma_bf16(d_tmem, gh, wh, id, k > 0 ? 1u : 0u);
    tc::mma_bf16(d_tmem, gh, wl, id, 1u);
    tc::mma_bf16(d_tmem, gl, wh, id, 1u);
  }
}

// One dW accumulator (M=64 layout: row o in TMEM lane (o % 16) + 32 (o / 16)) -> atomics.
// Columns [0, in) are dW, column `ones` (the ones chunk) is the bias gradient.
__device__ void flush_dw(uint32_t tmem, uint32_t col0, int N, int out, int in, int ones, float* gW,
                         float* gb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, half = warp >> 2;
  const int o = quad * 16 + lane;
  for (int g = half; g < N / 8; g += 2) {
    float v[8];
    tc::tmem_ld8(tmem + ((uint32_t)(quad * 32) << 16) + col0 + 8 * g, v);
    tc::tmem_wait_ld();
    if (lane < 16 && o < out) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = 8 * g + j;
        if (v[j] == 0.f) continue;
        if (i < in) atomicAdd(gW + o * in + i, v[j]);
        else if (i == ones) atomicAdd(gb + o, v[j]);
      }
    }
  }
}

__device__ void flush_all(uint32_t tmem, const FieldDesc& fd, float* __restrict__ grads) {
  float* base = grads + fd.base;
  const int enc = (int)fd.L * 2, cin = 31 + (int)fd.app_dim;
  flush_dw(tmem, TD_C2, HW, 3, 64, 64, base + fd.cw2, base + fd.cb2);
  flush_dw(tmem, TD_C1, HW, 64, 64, 64, base + fd.cw1, base + fd.cb1);
  flush_dw(tmem, TD_C0, CW, 64, cin, 48, base + fd.cw0, base + fd.cb0);
  flush_dw(tmem, TD_D1, HW, 16, 64, 64, base + fd.dw1, base + fd.db1);
  flush_dw(tmem, TD_D0, XW, 64, enc, 32, base + fd.dw0, base + fd.db0);
}

__device__ __forceinline__ void ones_chunk(uint8_t* hi, uint8_t* lo, int c0) {
  float v[8] = {1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int r = threadIdx.x; r < TM; r += NTH) put8(hi, lo, r, c0, v);
}

__global__ void __launch_bounds__(NTH, 1) k_mlp_bwd_tc(MlpLaunch m) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  BwdTcSmem& sm = *reinterpret_cast<BwdTcSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, half = warp >> 2;
  const int row = quad * 32 + lane;
  if (warp == 0) tc::tmem_alloc(&sm.tslot, 512);
  if (tid == 0) {
    tc::mbar_init(&sm.mbar, 1);
    tc::fence_mbar_init();
  }
  // ones columns (bias gradients through the dW GEMMs); never overwritten below
  ones_chunk(sm.x[0], sm.x[1], 32);
  ones_chunk(sm.h1[0], sm.h1[1], 64);
  ones_chunk(sm.cin[0], sm.cin[1], 48);
  ones_chunk(sm.c1[0], sm.c1[1], 64);
  ones_chunk(sm.c2[0], sm.c2[1], 64);
  for (int e = tid; e < TM * 16 * 2 / 4; e += NTH) {  // G5 columns 3..15 stay zero
    reinterpret_cast<uint32_t*>(sm.g5[0])[e] = 0u;
    reinterpret_cast<uint32_t*>(sm.g5[1])[e] = 0u;
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = sm.tslot;
  const uint32_t my_lanes = tmem + ((uint32_t)(quad * 32) << 16);
  uint32_t phase = 0;
  auto mma_done = [&]() {
    if (tid == 0) tc::commit(&sm.mbar);
    tc::mbar_wait(&sm.mbar, phase);
    phase ^= 1u;
    tc::fence_after();
  };
  const uint32_t per = (m.n_tiles + gridDim.x - 1) / gridDim.x;
  const uint32_t t_begin = blockIdx.x * per;
  const uint32_t t_end = min(m.n_tiles, t_begin + per);
  int loaded = -1;
  bool fresh = true;  // next dW GEMMs start a new accumulation
  for (uint32_t tile = t_begin; tile < t_end; ++tile) {
    const int f = tile_field(m, tile);
    const FieldDesc& fd = m.fields[f];
    const uint64_t s0 = m.field_off[f] + (uint64_t)(tile - m.tile_off[f]) * TM;
    const uint64_t rem = m.field_off[f + 1] - s0;
    const int count = rem < (uint64_t)TM ? (int)rem : TM;
    if (f != loaded) {
      if (loaded >= 0) flush_all(tmem, m.fields[loaded], m.grads);
      tc::fence_before();
      __syncthreads();
      tc::fence_after();
      stage_weights_tc(fd, m.params, sm.w);
      loaded = f;
      fresh = true;
    }
    const int act_c = fd.coarse ? 2 : 1;
    const bool valid = row < count;
    const uint64_t gs = s0 + row;
    // ---------------- forward recompute ----------------
    {
      float v[16];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int l = half * 8 + j;
        float2 xx = make_float2(0.f, 0.f);
        if (valid && l < (int)m.levels)
          xx = reinterpret_cast<const float2*>(m.X)[(uint64_t)l * m.x_stride + gs];
        v[2 * j] = xx.x;
        v[2 * j + 1] = xx.y;
      }
      put8(sm.x[0], sm.x[1], row, half * 16, v);
      put8(sm.x[0], sm.x[1], row, half * 16 + 8, v + 8);
    }
    to_mma();
    if (tid == 0) gemm_kmajor_t(tmem, sm.x[0], sm.x[1], sm.w.d0[0], sm.w.d0[1], 64, 32);
    mma_done();
    {
      float v[32];
      ld32(my_lanes + half * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i] + sm.w.bd0[half * 32 + i], 0.f);
#pragma unroll
      for (int c = 0; c < 4; ++c) put8(sm.h1[0], sm.h1[1], row, half * 32 + 8 * c, v + 8 * c);
    }
    to_mma();
    if (tid == 0) gemm_kmajor_t(tmem, sm.h1[0], sm.h1[1], sm.w.d1[0], sm.w.d1[1], 16, 64);
    mma_done();
    {
      float raw[16];
      tc::tmem_ld16(my_lanes, raw);
      tc::tmem_wait_ld();
      float cin[48];
      uint32_t mask = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float z = raw[i] + sm.w.bd1[i];
        mask |= (z > 15.f || z < -15.f ? 1u : 0u) << i;
        raw[i] = clip15(z);
      }
#pragma unroll
      for (int i = 0; i < 15; ++i) cin[i] = raw[1 + i];
      float sh[16];
      const float* app = nullptr;
      if (valid) {
        const RayRec& r = m.rec[m.s_item[gs]];
        sh16((float)r.d[0], (float)r.d[1], (float)r.d[2], sh);
        app = m.app_per_sample ? m.app_override + gs * fd.app_dim
                               : (m.app_override ? m.app_override : m.app_table + (uint64_t)r.img * fd.app_dim);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) sh[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) cin[15 + i] = sh[i];
      for (int i = 0; i < 17; ++i) cin[31 + i] = (app && i < (int)fd.app_dim) ? app[i] : 0.f;
      if (half == 0) {
        sm.sig_raw[row] = raw[0];
        sm.dmask[row] = mask;
        put8(sm.cin[0], sm.cin[1], row, 0, cin);
        put8(sm.cin[0], sm.cin[1], row, 8, cin + 8);
        put8(sm.cin[0], sm.cin[1], row, 16, cin + 16);
      } else {
        put8(sm.cin[0], sm.cin[1], row, 24, cin + 24);
        put8(sm.cin[0], sm.cin[1], row, 32, cin + 32);
        put8(sm.cin[0], sm.cin[1], row, 40, cin + 40);
      }
    }
    to_mma();
    if (tid == 0) gemm_kmajor_t(tmem, sm.cin[0], sm.cin[1], sm.w.c0[0], sm.w.c0[1], 64, 48);
    mma_done();
    {
      float v[32];
      ld32(my_lanes + half * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float z = v[i] + sm.w.bc0[half * 32 + i];
        v[i] = act_c == 2 ? sigm(z) : fmaxf(z, 0.f);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) put8(sm.c1[0], sm.c1[1], row, half * 32 + 8 * c, v + 8 * c);
    }
    to_mma();
    if (tid == 0) gemm_kmajor_t(tmem, sm.c1[0], sm.c1[1], sm.w.c1[0], sm.w.c1[1], 64, 64);
    mma_done();
    {
      float v[32];
      ld32(my_lanes + half * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float z = v[i] + sm.w.bc1[half * 32 + i];
        v[i] = act_c == 2 ? sigm(z) : fmaxf(z, 0.f);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) put8(sm.c2[0], sm.c2[1], row, half * 32 + 8 * c, v + 8 * c);
    }
    to_mma();
    if (tid == 0) gemm_kmajor_t(tmem, sm.c2[0], sm.c2[1], sm.w.c2[0], sm.w.c2[1], 16, 64);
    mma_done();
    // ---------------- B1: colour head adjoint (field.cpp:298-306) ----------------
    {
      float v[16];
      tc::tmem_ld16(my_lanes, v);
      tc::tmem_wait_ld();
      if (half == 0) {
        const float4 up = valid ? m.grad_in[gs] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float ug[3] = {up.y, up.z, up.w};
        float g[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const float z = v[k] + sm.w.bc2[k];
          const bool clipped = z > 15.f || z < -15.f;
          const float sg = sigm(clip15(z));
          g[k] = clipped ? 0.f : ug[k] * sg * (1.f - sg);
        }
        put8(sm.g5[0], sm.g5[1], row, 0, g);
        // sigma path of the density raw gradient (field.cpp:313)
        sm.gsig[row] = (sm.dmask[row] & 1u) ? 0.f : up.x * expf(sm.sig_raw[row]);
      }
    }
    to_mma();
    if (tid == 0) {
      gemm_wgrad(tmem + TD_C2, sm.g5[0], sm.g5[1], sm.c2[0], sm.c2[1], HW, !fresh);
      gemm_igrad(tmem, sm.g5[0], sm.g5[1], sm.w.c2[0], sm.w.c2[1], 16, 64, 16);
    }
    mma_done();
    // ---------------- B2: G4 = dC2 * act'(C2) -> c2 tile ----------------
    {
      float v[32], a[32];
      ld32(my_lanes + half * 32, v);
#pragma unroll
      for (int c = 0; c < 4; ++c) get8(sm.c2[0], sm.c2[1], row, half * 32 + 8 * c, a + 8 * c);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= act_c == 2 ? a[i] * (1.f - a[i]) : (a[i] > 0.f ? 1.f : 0.f);
#pragma unroll
      for (int c = 0; c < 4; ++c) put8(sm.c2[0], sm.c2[1], row, half * 32 + 8 * c, v + 8 * c);
    }
    to_mma();
    if (tid == 0) {
      gemm_wgrad(tmem + TD_C1, sm.c2[0], sm.c2[1], sm.c1[0], sm.c1[1], HW, !fresh);
      gemm_igrad(tmem, sm.c2[0], sm.c2[1], sm.w.c1[0], sm.w.c1[1], 64, 64, 64);
    }
    mma_done();
    // ---------------- B3: G3 = dC1 * act'(C1) -> c1 tile ----------------
    {
      float v[32], a[32];
      ld32(my_lanes + half * 32, v);
#pragma unroll
      for (int c = 0; c < 4; ++c) get8(sm.c1[0], sm.c1[1], row, half * 32 + 8 * c, a + 8 * c);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= act_c == 2 ? a[i] * (1.f - a[i]) : (a[i] > 0.f ? 1.f : 0.f);
#pragma unroll
      for (int c = 0; c < 4; ++c) put8(sm.c1[0], sm.c1[1], row, half * 32 + 8 * c, v + 8 * c);
    }
    to_mma();
    if (tid == 0) {
      gemm_wgrad(tmem + TD_C0, sm.c1[0], sm.c1[1], sm.cin[0], sm.cin[1], CW, !fresh);
      gemm_igrad(tmem, sm.c1[0], sm.c1[1], sm.w.c0[0], sm.w.c0[1], 64, 16, 64);
    }
    mma_done();
    // ---------------- B4: G2 = density raw gradient -> cin tile cols 0..15 ----------------
    {
      float v[16];
      tc::tmem_ld16(my_lanes, v);
      tc::tmem_wait_ld();
      if (half == 0) {
        const uint32_t mask = sm.dmask[row];
        float g[16];
        g[0] = sm.gsig[row];
#pragma unroll
        for (int k = 1; k < 16; ++k) g[k] = ((mask >> k) & 1u) ? 0.f : v[k - 1];
        put8(sm.cin[0], sm.cin[1], row, 0, g);
        put8(sm.cin[0], sm.cin[1], row, 8, g + 8);
      }
    }
    to_mma();
    if (tid == 0) {
      gemm_wgrad(tmem + TD_D1, sm.cin[0], sm.cin[1], sm.h1[0], sm.h1[1], HW, !fresh);
      gemm_igrad(tmem, sm.cin[0], sm.cin[1], sm.w.d1[0], sm.w.d1[1], 16, 64, 16);
    }
    mma_done();
    // ---------------- B5: G1 = dH1 * relu'(H1) -> h1 tile ----------------
    {
      float v[32], a[32];
      ld32(my_lanes + half * 32, v);
#pragma unroll
      for (int c = 0; c < 4; ++c) get8(sm.h1[0], sm.h1[1], row, half * 32 + 8 * c, a + 8 * c);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= a[i] > 0.f ? 1.f : 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) put8(sm.h1[0], sm.h1[1], row, half * 32 + 8 * c, v + 8 * c);
    }
    to_mma();
    if (tid == 0) {
      gemm_wgrad(tmem + TD_D0, sm.h1[0], sm.h1[1], sm.x[0], sm.x[1], XW, !fresh);
      gemm_igrad(tmem, sm.h1[0], sm.h1[1], sm.w.d0[0], sm.w.d0[1], 64, 32, 64);
    }
    mma_done();
    fresh = false;
    // ---------------- B6: dX -> global, level-major ----------------
    {
      float v[16];
      tc::tmem_ld16(my_lanes + half * 16, v);
      tc::tmem_wait_ld();
      if (valid) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int l = half * 8 + j;
          if (l < (int)m.levels)
            reinterpret_cast<float2*>(m.dX)[(uint64_t)l * m.x_stride + gs] = make_float2(v[2 * j], v[2 * j + 1]);
        }
      }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
  if (loaded >= 0) flush_all(tmem, m.fields[loaded], m.grads);
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 512);
}

}  // namespace

void launch_mlp_fwd_tc(const MlpLaunch& m, int num_sms, cudaStream_t s) {
  if (!m.n_tiles) return;
  static bool attr = false;
  const int smem = (int)sizeof(FwdTcSmem) + 1024;
  if (!attr) {
    cudaFuncSetAttribute(k_mlp_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const uint32_t want = (uint32_t)num_sms * 2;
  const unsigned grid = m.n_tiles < want ? m.n_tiles : want;
  k_mlp_fwd_tc<<<grid, NTH, smem, s>>>(m);
}

void launch_mlp_bwd_tc(const MlpLaunch& m, int num_sms, cudaStream_t s) {
  if (!m.n_tiles) return;
  static bool attr = false;
  const int smem = (int)sizeof(BwdTcSmem) + 1024;
  if (!attr) {
    cudaFuncSetAttribute(k_mlp_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const unsigned grid = m.n_tiles < (uint32_t)num_sms ? m.n_tiles : (uint32_t)num_sms;
  k_mlp_bwd_tc<<<grid, NTH, smem, s>>>(m);
}

}  // namespace dg
