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

#include <algorithm>

#include "dg_common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace dg {

namespace {

constexpr int TM = 128;   // samples per tile (MMA M)
#ifndef MLP_FWD_MINB
#define MLP_FWD_MINB 2
#endif
constexpr int NTF = 256;  // forward: 8 warps, MLP_FWD_MINB CTAs/SM (their MMAs and epilogues interleave)
constexpr int NTB = 512;  // backward: 16 warps, 1 CTA/SM (212 KB of operand tiles)
// Warp w reads TMEM lane quadrant w % 4 (tcgen05.ld rule) and owns column part w / 4.

// Weight operand tiles (B, K-major): rows = out (padded), cols = in (padded).
struct TcWeights {
  uint8_t d0[2][64 * 32 * 2];
  uint8_t d1[2][16 * 64 * 2];
  uint8_t c0[2][64 * 48 * 2];
  uint8_t c1[2][64 * 64 * 2];
  uint8_t c2[2][16 * 64 * 2];
  float bd0[64], bd1[16], bc0[64], bc1[64], bc2[16];
};

// Two fp32 -> packed bf16x2 hi and lo (x = hi + lo + O(2^-17 |x|)); same values as
// tc::split_bf16, two lanes per cvt.
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(a - hf.x, b - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// TMEM A-operand region (tcgen05.mma A from TMEM, tools/ubench/tmem_a.cu): the next GEMM's
// activation / gradient tile, hi halves at columns [A_HI, A_HI + K/2), lo at + A_LO_OFF.
// Reading A from TMEM instead of shared memory removes the 4 KB/MMA smem A-read that bounds
// a small-N tcgen05.mma at ~39 cycles (11 cycles from TMEM at N = 16; tools/ubench/mma_latency.cu).
constexpr uint32_t A_HI = 64, A_LO_OFF = 32;

// Destination of an operand tile row: the smem copy (K-major core-matrix layout, hi / lo;
// null when the tile is consumed only from TMEM) and this thread's lane of the TMEM A region.
struct Sink {
  uint8_t* hi;
  uint8_t* lo;
  uint32_t ta;  // lane base | A_HI
};

// Write 8 consecutive columns [c0, c0+8) of row r (split once, stored to both copies).
// Warp-uniform (tcgen05.st is .sync.aligned).
__device__ __forceinline__ void put8(const Sink& k, int r, int c0, const float* v) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) split2(v[2 * j], v[2 * j + 1], h[j], l[j]);
  if (k.hi) {
    const uint32_t off = tc::core_offset(r, c0, TM);
    *reinterpret_cast<uint4*>(k.hi + off) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(k.lo + off) = make_uint4(l[0], l[1], l[2], l[3]);
  }
  tc::tmem_st4(k.ta + (uint32_t)(c0 >> 1), h);
  tc::tmem_st4(k.ta + A_LO_OFF + (uint32_t)(c0 >> 1), l);
}

// smem-only variant (ones columns, weight-gradient operands that never feed a TMEM-A GEMM).
__device__ __forceinline__ void put8s(uint8_t* hi, uint8_t* lo, int r, int c0, const float* v) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) split2(v[2 * j], v[2 * j + 1], h[j], l[j]);
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

// Stage one layer's W[out][in] (fp32, global) as split-bf16 K-major tiles [Np x Kp].
__device__ void stage_layer(const float* __restrict__ W, int out, int in, int Np, int Kp,
                            uint8_t* hi, uint8_t* lo) {
  for (int e = threadIdx.x; e < Np * Kp / 2; e += blockDim.x) {
    const int o = (2 * e) / Kp, i = (2 * e) % Kp;
    const float a = (o < out && i < in) ? W[o * in + i] : 0.f;
    const float b = (o < out && i + 1 < in) ? W[o * in + i + 1] : 0.f;
    uint32_t h, l;
    split2(a, b, h, l);
    const uint32_t off = tc::core_offset(o, i, Np);
    *reinterpret_cast<uint32_t*>(hi + off) = h;
    *reinterpret_cast<uint32_t*>(lo + off) = l;
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
  for (int e = threadIdx.x; e < 64; e += blockDim.x) {
    w.bd0[e] = base[fd.db0 + e];
    w.bc0[e] = base[fd.cb0 + e];
    w.bc1[e] = base[fd.cb1 + e];
  }
  for (int e = threadIdx.x; e < 16; e += blockDim.x) {
    w.bd1[e] = base[fd.db1 + e];
    w.bc2[e] = e < 3 ? base[fd.cb2 + e] : 0.f;
  }
}

// D[TM x N] = A[TM x K] . B[N x K]^T, split-bf16 (3 MMAs per 16-wide K step), A in the TMEM
// A region (hi at column a, lo at a + A_LO_OFF; 8 columns per K step), B in smem (K-major,
// rows = N: SBO 128, LBO N/8*128).  Descriptors are built once; a K step only advances the
// 14-bit start-address field (smem offsets < 256 KB never carry out of it).
template <int N, int K>
__device__ __forceinline__ void gemm_ts(uint32_t d_tmem, uint32_t a, const uint8_t* b_hi, const uint8_t* b_lo) {
  constexpr uint32_t id = tc::idesc_bf16(TM, N, 0, 0);
  constexpr uint32_t b_lbo = (N / 8) * 128;
  const uint64_t bh = tc::smem_desc(tc::smem_u32(b_hi), b_lbo, 128);
  const uint64_t bl = tc::smem_desc(tc::smem_u32(b_lo), b_lbo, 128);
#pragma unroll
  for (int k = 0; k < K / 16; ++k) {
    const uint32_t bo = (k * 2 * b_lbo) >> 4;
    tc::mma_bf16_ts(d_tmem, a + 8 * k, bh + bo, id, k > 0 ? 1u : 0u);
    tc::mma_bf16_ts(d_tmem, a + 8 * k, bl + bo, id, 1u);
    tc::mma_bf16_ts(d_tmem, a + A_LO_OFF + 8 * k, bh + bo, id, 1u);
  }
}

// sigmoid with the SFU exp and reciprocal (relative error ~1e-7 for |x| <= 15-ish inputs).
#ifdef DG_TC_PRECISE_SIGM
__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + expf(-x)); }
#else
__device__ __forceinline__ float sigm(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
#endif
__device__ __forceinline__ float clip15(float v) { return v > 15.f ? 15.f : (v < -15.f ? -15.f : v); }

// SH16 components 1..15 (sh.hpp:14-35); component 0 is the constant 0.28209479177387814.
__device__ __forceinline__ void sh15(float x, float y, float z, float* o) {
  const float xy = x * y, xz = x * z, yz = y * z, x2 = x * x, y2 = y * y, z2 = z * z;
  o[0] = -0.48860251190291987f * y;
  o[1] = 0.48860251190291987f * z;
  o[2] = -0.48860251190291987f * x;
  o[3] = 1.0925484305920792f * xy;
  o[4] = -1.0925484305920792f * yz;
  o[5] = 0.31539156525252005f * (3.0f * z2 - 1.0f);
  o[6] = -1.0925484305920792f * xz;
  o[7] = 0.5462742152960396f * (x2 - y2);
  o[8] = -0.5900435899266435f * y * (3.0f * x2 - y2);
  o[9] = 2.890611442640554f * xy * z;
  o[10] = -0.4570457994644658f * y * (5.0f * z2 - 1.0f);
  o[11] = 0.3731763325901154f * z * (5.0f * z2 - 3.0f);
  o[12] = -0.4570457994644658f * x * (5.0f * z2 - 1.0f);
  o[13] = 1.445305721320277f * z * (x2 - y2);
  o[14] = -0.5900435899266435f * x * (x2 - 3.0f * y2);
}
constexpr float kSH0 = 0.28209479177387814f;

// Colour-MLP hidden activation of 16 pre-activations z = v + b (field.cpp:196-199: sigmoid in
// the coarse field, ReLU in the fine one).  The branch is uniform, so a ReLU tile never pays
// for the two SFU ops of the sigmoid.
__device__ __forceinline__ void act16(float* v, const float* b, int act) {
  if (act == 2) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = sigm(v[i] + (b ? b[i] : 0.f));
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i] + (b ? b[i] : 0.f), 0.f);
  }
}

struct TileGeo {
  int f;
  uint32_t s0;  // first sample (sample counts fit 32 bits, the ray ids do)
  int count;
  uint32_t t_end, s_end;  // the field's tile / sample end: the next tile of the same field
                          // is derived without touching the offset tables
  uint32_t t_beg, s_beg;  // the field's first tile / sample
};
__device__ __forceinline__ TileGeo tile_geo(const MlpLaunch& m, uint32_t tile) {
  int f = 0;
  while (f + 1 < (int)m.n_fields && tile >= __ldg(m.tile_off + f + 1)) ++f;
  TileGeo g;
  g.f = f;
  g.s0 = __ldg(m.field_off + f) + (tile - __ldg(m.tile_off + f)) * (uint32_t)TM;
  g.t_end = __ldg(m.tile_off + f + 1);
  g.s_end = __ldg(m.field_off + f + 1);
  g.t_beg = __ldg(m.tile_off + f);
  g.s_beg = __ldg(m.field_off + f);
  const uint32_t rem = g.s_end - g.s0;
  g.count = rem < (uint32_t)TM ? (int)rem : TM;
  return g;
}
// any later tile (the forward strides its tiles over the grid)
__device__ __forceinline__ TileGeo tile_geo_at(const MlpLaunch& m, const TileGeo& c, uint32_t tile) {
  if (tile >= c.t_end) return tile_geo(m, tile);
  TileGeo g = c;
  g.s0 = c.s_beg + (tile - c.t_beg) * (uint32_t)TM;
  const uint32_t rem = c.s_end - g.s0;
  g.count = rem < (uint32_t)TM ? (int)rem : TM;
  return g;
}
// the tile after `c` (consecutive tiles of one CTA)
__device__ __forceinline__ TileGeo tile_geo_next(const MlpLaunch& m, const TileGeo& c, uint32_t tile) {
  if (tile >= c.t_end) return tile_geo(m, tile);
  TileGeo g = c;
  g.s0 = c.s0 + (uint32_t)TM;
  const uint32_t rem = c.s_end - g.s0;
  g.count = rem < (uint32_t)TM ? (int)rem : TM;
  return g;
}

// Per-thread register prefetch of one tile's global inputs, issued during the previous tile
// so the tile's epilogues never wait on HBM/L2:  X (this part's levels), the upstream
// gradient (part 0), and the dependent chain  item -> RayRec (dir, image) -> appearance row.
// Column parts of the Cin tile: part 0 = clip(raw1..15) + SH0, part SHP = SH1..15 + app0,
// part APP = app1..16.
template <int NP>
struct Pref {
  static constexpr int XL = 16 / NP;  // levels per part
  static constexpr int SHP = 1, APP = NP == 4 ? 2 : 1;
  float x[2 * XL];
  float4 g;
  uint32_t item;
  uint32_t img;
  double dir[3];
  float app[17];
  uint64_t gs;
  bool valid;

  __device__ __forceinline__ void start(const MlpLaunch& m, bool v, uint64_t gsample, int part,
                                        bool want_g) {
    valid = v;
    gs = gsample;
#pragma unroll
    for (int j = 0; j < XL; ++j) {
      const int l = part * XL + j;
      float2 xx = make_float2(0.f, 0.f);
      if (v && l < (int)m.levels)
        xx = __ldcs(reinterpret_cast<const float2*>(m.X) + (uint64_t)l * m.x_stride + gs);
      x[2 * j] = xx.x;
      x[2 * j + 1] = xx.y;
    }
    if (part == SHP || part == APP) item = v ? __ldg(m.s_item + gs) : 0u;
    if (want_g && part == 0)
      g = v ? __ldcs(m.grad_in + gs) : make_float4(0.f, 0.f, 0.f, 0.f);
  }

  __device__ __forceinline__ void grad(const MlpLaunch& m, int part) {
    if (part == 0)
      g = valid ? __ldcs(m.grad_in + gs) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __device__ __forceinline__ void rec(const MlpLaunch& m, int part) {
    if ((part == SHP || part == APP) && valid) {
      const RayRec& r = m.rec[item];
      if (part == SHP) {
        dir[0] = r.d[0];
        dir[1] = r.d[1];
        dir[2] = r.d[2];
      }
      img = r.img;
    }
  }
  __device__ __forceinline__ void appearance(const MlpLaunch& m, const FieldDesc& fd, int part) {
    if (part != SHP && part != APP) return;
    const int dim = (int)fd.app_dim;
    const float* src = nullptr;
    if (valid)
      src = m.app_per_sample ? m.app_override + gs * fd.app_dim
                             : (m.app_override ? m.app_override : m.app_table + (uint64_t)img * fd.app_dim);
#pragma unroll
    for (int i = 0; i < 17; ++i) {
      const bool mine = (part == SHP && i == 0) || (part == APP && i >= 1);
      app[i] = (mine && src && i < dim) ? __ldg(src + i) : 0.f;
    }
  }
  // Write this part's columns of Cin (raw16 = clipped density output, part 0 only).
  __device__ __forceinline__ void put_cin(const Sink& k, int row, int part, const float* raw) {
    if (part == 0) {
      float c[16];
#pragma unroll
      for (int i = 0; i < 15; ++i) c[i] = raw[1 + i];
      c[15] = valid ? kSH0 : 0.f;
      put8(k, row, 0, c);
      put8(k, row, 8, c + 8);
    }
    if (part == SHP) {
      float c[16];
      if (valid) {
        sh15((float)dir[0], (float)dir[1], (float)dir[2], c);
      } else {
#pragma unroll
        for (int i = 0; i < 15; ++i) c[i] = 0.f;
      }
      c[15] = app[0];
      put8(k, row, 16, c);
      put8(k, row, 24, c + 8);
    }
    if (part == APP) {
      put8(k, row, 32, app + 1);
      put8(k, row, 40, app + 9);
    }
  }
  __device__ __forceinline__ void put_x(const Sink& k, int row, int part) {
#pragma unroll
    for (int c = 0; c < XL / 4; ++c) put8(k, row, part * 2 * XL + 8 * c, x + 8 * c);
  }
};

// Sync point between an epilogue (generic smem writes, TMEM loads / stores) and the next MMA.
__device__ __forceinline__ void to_mma() {
  tc::tmem_wait_st();
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
}

// Load 16 consecutive TMEM columns of this thread's lane.
__device__ __forceinline__ void ld16(uint32_t taddr, float (&v)[16]) {
  tc::tmem_ld16(taddr, v);
  tc::tmem_wait_ld();
}

// The MMAs of a stage and their commit come from one elected lane of warp 0.
#define ISSUE(...)                      \
  do {                                  \
    if (warp == 0) {                    \
      if (tc::elect_one()) {            \
        __VA_ARGS__;                    \
        tc::commit(&sm.mbar);           \
      }                                 \
      __syncwarp();                     \
    }                                   \
  } while (0)

// The same from warp `w`.
#define ISSUE_W(w, ...)                 \
  do {                                  \
    if (warp == (w)) {                  \
      if (tc::elect_one()) {            \
        __VA_ARGS__;                    \
        tc::commit(&sm.mbar);           \
      }                                 \
      __syncwarp();                     \
    }                                   \
  } while (0)

// Critical MMAs, their commit (the next epilogue waits for it), then background MMAs whose
// completion a later commit covers (commit tracks every earlier tcgen05 op of the thread).
template <class Crit, class Back>
__device__ __forceinline__ void issue2(int warp, uint64_t* mbar, Crit crit, Back back) {
  if (warp == 0) {
    if (tc::elect_one()) {
      crit();
      tc::commit(mbar);
      back();
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------- forward
// The forward runs in split-tf32 (x = hi + lo + O(2^-22 |x|), hi.hi + hi.lo + lo.hi exact in
// the fp32 accumulator): its pre-activations decide the ReLU / clip masks the backward uses
// (MlpLaunch::masks), and a mask must agree with the fp64 reference's for every unit that is
// not within fp32 noise of its kink.  Split-bf16 (2^-17) flipped ~1.5e-4 of the samples'
// masks in a trained state (tools/diag/diag_mlp_prec.py), each flip switching a whole unit's
// gradient contribution on or off.

// tf32 weight tiles (B, K-major, 32-bit core matrices): rows = out (padded), cols = in.
struct TcWeights32 {
  uint32_t d0[2][64 * 32];
  uint32_t d1[2][16 * 64];
  uint32_t c0[2][64 * 48];
  uint32_t c1[2][64 * 64];
  uint32_t c2[2][16 * 64];
  float bd0[64], bd1[16], bc0[64], bc1[64], bc2[16];
};

__device__ void stage_layer32(const float* __restrict__ W, int out, int in, int Np, int Kp, uint32_t* hi,
                              uint32_t* lo) {
  for (int e = threadIdx.x; e < Np * Kp; e += blockDim.x) {
    const int o = e / Kp, i = e % Kp;
    const float a = (o < out && i < in) ? W[o * in + i] : 0.f;
    uint32_t h, l;
    tc::split_tf32(a, h, l);
    const uint32_t off = tc::core_offset32(o, i, Np) >> 2;
    hi[off] = h;
    lo[off] = l;
  }
}

__device__ void stage_weights_tf32(const FieldDesc& fd, const float* __restrict__ params, TcWeights32& w) {
  const float* base = params + fd.base;
  const int enc = (int)fd.L * 2, cin = 31 + (int)fd.app_dim;
  stage_layer32(base + fd.dw0, 64, enc, 64, 32, w.d0[0], w.d0[1]);
  stage_layer32(base + fd.dw1, 16, 64, 16, 64, w.d1[0], w.d1[1]);
  stage_layer32(base + fd.cw0, 64, cin, 64, 48, w.c0[0], w.c0[1]);
  stage_layer32(base + fd.cw1, 64, 64, 64, 64, w.c1[0], w.c1[1]);
  stage_layer32(base + fd.cw2, 3, 64, 16, 64, w.c2[0], w.c2[1]);
  for (int e = threadIdx.x; e < 64; e += blockDim.x) {
    w.bd0[e] = base[fd.db0 + e];
    w.bc0[e] = base[fd.cb0 + e];
    w.bc1[e] = base[fd.cb1 + e];
  }
  for (int e = threadIdx.x; e < 16; e += blockDim.x) {
    w.bd1[e] = base[fd.db1 + e];
    w.bc2[e] = e < 3 ? base[fd.cb2 + e] : 0.f;
  }
}

// TMEM A region of the forward: hi at [A32_HI, A32_HI + K), lo at + A32_LO_OFF (one column per k).
constexpr uint32_t A32_HI = 64, A32_LO_OFF = 64;

// 8 consecutive columns [c0, c0 + 8) of this thread's row into the tf32 A region.
__device__ __forceinline__ void put8_32(uint32_t ta, int c0, const float* v) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    uint32_t h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) tc::split_tf32(v[4 * q + j], h[j], l[j]);
    tc::tmem_st4(ta + (uint32_t)(c0 + 4 * q), h);
    tc::tmem_st4(ta + A32_LO_OFF + (uint32_t)(c0 + 4 * q), l);
  }
}

// D[TM x N] = A[TM x K] . B[N x K]^T in split-tf32 (3 MMAs per 8-wide K step); A in the TMEM
// A region, B in smem (K-major 32-bit core matrices: SBO 128, LBO N/8*128).
template <int N, int K>
__device__ __forceinline__ void gemm_ts32(uint32_t d_tmem, uint32_t a, const uint32_t* b_hi, const uint32_t* b_lo) {
  constexpr uint32_t id = tc::idesc_tf32(TM, N, 0, 0);
  constexpr uint32_t b_lbo = (N / 8) * 128;
  const uint64_t bh = tc::smem_desc(tc::smem_u32(b_hi), b_lbo, 128);
  const uint64_t bl = tc::smem_desc(tc::smem_u32(b_lo), b_lbo, 128);
#pragma unroll
  for (int k = 0; k < K / 8; ++k) {
    const uint32_t bo = (k * 2 * b_lbo) >> 4;
    tc::mma_tf32_ts(d_tmem, a + 8 * k, bh + bo, id, k > 0 ? 1u : 0u);
    tc::mma_tf32_ts(d_tmem, a + 8 * k, bl + bo, id, 1u);
    tc::mma_tf32_ts(d_tmem, a + A32_LO_OFF + 8 * k, bh + bo, id, 1u);
  }
}

// bits i of the ReLU mask (z > 0) of 16 pre-activations
__device__ __forceinline__ uint32_t relu_bits16(const float* z) {
  uint32_t b = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) b |= (z[i] > 0.f ? 1u : 0u) << i;
  return b;
}

constexpr int kCinS = 36;  // row stride (floats) of the staged Cin columns: conflict-free float4s
struct FwdTcSmem {
  TcWeights32 w;
  float cin_s[TM * kCinS];
  float sig_raw[TM];
  uint64_t mbar;
  uint32_t tslot;
};

// Forward: 2 column parts (warps 0-3 / 4-7) x 4 lane quadrants; each thread owns one sample row
// and 32 of the 64 hidden columns.  Activations never touch shared memory: each epilogue
// writes the next layer's split operand straight into the TMEM A region.  TMEM: [0, 64) the
// accumulator, [64, 192) the A operand (hi, lo).  Tiles are strided over the grid.  With
// m.masks set, each pre-activation's sign (and the two clip flags) go to HBM for the backward:
// mask word w of sample s at masks[w * x_stride + s]: w = 0..3, one per 16-column part p of
// the backward: h1 bits of columns 16p..16p+15 | c1 bits << 16; w = 4, 5: c2 columns 0-31,
// 32-63; w = 6: raw clip bits 0-15 | colour clip bits 16-18.
__global__ void __launch_bounds__(NTF, MLP_FWD_MINB) k_mlp_fwd_tc(MlpLaunch m) {
  constexpr int NP = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  FwdTcSmem& sm = *reinterpret_cast<FwdTcSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, part = warp >> 2;
  const int row = quad * 32 + lane;  // TMEM lane == sample row of the tile
  const int fiw = (int)m.issue_warp_fwd;  // the MMA-issuing warp
  if (warp == 0) tc::tmem_alloc(&sm.tslot, 256);
  if (tid == 0) {
    tc::mbar_init(&sm.mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = sm.tslot;
  const uint32_t my_lanes = tmem + ((uint32_t)(quad * 32) << 16);
  const uint32_t ta = my_lanes + A32_HI;
  const uint32_t a_op = tmem + A32_HI;
  uint32_t* const masks = m.masks;
  uint32_t phase = 0;
  auto mma_done = [&]() {
    tc::mbar_wait(&sm.mbar, phase);
    phase ^= 1u;
    tc::fence_after();
  };
  uint32_t tile = blockIdx.x;
  if (tile < m.n_tiles) {
    TileGeo cur = tile_geo(m, tile);
    Pref<NP> pf;
    pf.start(m, row < cur.count, cur.s0 + row, part, false);
    pf.rec(m, part);
    stage_weights_tf32(m.fields[cur.f], m.params, sm.w);
    int loaded = cur.f;
    int act_c = m.fields[cur.f].coarse ? 2 : 1;  // colour activation of the loaded field
    auto put_x = [&]() {
#pragma unroll
      for (int c = 0; c < 2; ++c) put8_32(ta, part * 16 + 8 * c, pf.x + 8 * c);
    };
    put_x();
    for (;;) {
      const bool valid = row < cur.count;
      const uint64_t gs = cur.s0 + row;
      const uint32_t next = tile + gridDim.x;
      const bool has_next = next < m.n_tiles;
      const TileGeo nx = has_next ? tile_geo_at(m, cur, next) : cur;
      const bool store_mask = masks != nullptr && valid;
      to_mma();
      // ---- L1: H1 = relu(X Wd0^T + b) ----
      ISSUE_W(fiw, gemm_ts32<64, 32>(tmem, a_op, sm.w.d0[0], sm.w.d0[1]));
      if (part == 1) {  // Cin columns 16-47 (SH1..15, appearance) of this tile's row -> smem
        float* cs = sm.cin_s + row * kCinS;
        float c[16];
        if (valid) {
          sh15((float)pf.dir[0], (float)pf.dir[1], (float)pf.dir[2], c);
        } else {
#pragma unroll
          for (int i = 0; i < 15; ++i) c[i] = 0.f;
        }
        // appearance row (L2-resident table; read here, used at L2's epilogue)
        const int dim = (int)m.fields[cur.f].app_dim;
        const float* src = nullptr;
        if (valid)
          src = m.app_per_sample ? m.app_override + gs * (uint32_t)dim
                                 : (m.app_override ? m.app_override : m.app_table + (uint64_t)pf.img * dim);
        float a[17];
#pragma unroll
        for (int i = 0; i < 17; ++i) a[i] = (src && i < dim) ? __ldg(src + i) : 0.f;
        c[15] = a[0];
#pragma unroll
        for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(cs + i) = make_float4(c[i], c[i + 1], c[i + 2], c[i + 3]);
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(cs + 16 + i) = make_float4(a[1 + i], a[2 + i], a[3 + i], a[4 + i]);
      }
      pf.start(m, has_next && row < nx.count, nx.s0 + row, part, false);  // next tile: X, item
      mma_done();
      {
        uint32_t bits = 0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          float v[16];
          ld16(my_lanes + part * 32 + 16 * q, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += sm.w.bd0[part * 32 + 16 * q + i];
          bits |= relu_bits16(v) << (16 * q);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
          put8_32(ta, part * 32 + 16 * q, v);
          put8_32(ta, part * 32 + 16 * q + 8, v + 8);
        }
        if (store_mask) {  // low halves of words 2 part, 2 part + 1 (the backward's 16-column parts)
          uint16_t* mh = reinterpret_cast<uint16_t*>(masks + (uint64_t)(2 * part) * m.x_stride + gs);
          __stcs(mh, (uint16_t)(bits & 0xffffu));
          __stcs(mh + 2 * m.x_stride, (uint16_t)(bits >> 16));
        }
      }
      to_mma();
      // ---- L2: raw16 = H1 Wd1^T + b ; Cin = [clip(raw1..15) | SH16 | app | 0] ----
      ISSUE_W(fiw, gemm_ts32<16, 64>(tmem, a_op, sm.w.d1[0], sm.w.d1[1]));
      mma_done();
      uint32_t clip_bits = 0;
      {
        float raw[16];
        if (part == 0) {
          ld16(my_lanes, raw);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float z = raw[i] + sm.w.bd1[i];
            clip_bits |= (z > 15.f || z < -15.f ? 1u : 0u) << i;
            raw[i] = clip15(z);
          }
          sm.sig_raw[row] = raw[0];
        }
        float c[16];
        if (part == 0) {
#pragma unroll
          for (int i = 0; i < 15; ++i) c[i] = raw[1 + i];
          c[15] = valid ? kSH0 : 0.f;
          put8_32(ta, 0, c);
          put8_32(ta, 8, c + 8);
        } else {  // part 1: the SH / appearance columns staged at the tile start
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float* cs = sm.cin_s + row * kCinS + 16 * h;
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              const float4 q = *reinterpret_cast<const float4*>(cs + i);
              c[i] = q.x;
              c[i + 1] = q.y;
              c[i + 2] = q.z;
              c[i + 3] = q.w;
            }
            put8_32(ta, 16 + 16 * h, c);
            put8_32(ta, 24 + 16 * h, c + 8);
          }
        }
      }
      pf.rec(m, part);  // next tile's RayRec (item arrived during L1/L2)
      to_mma();
      // ---- L3: C1 = act(Cin Wc0^T + b) ----
      ISSUE_W(fiw, gemm_ts32<64, 48>(tmem, a_op, sm.w.c0[0], sm.w.c0[1]));
      mma_done();
      {
        uint32_t bits = 0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          float v[16];
          ld16(my_lanes + part * 32 + 16 * q, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += sm.w.bc0[part * 32 + 16 * q + i];
          bits |= relu_bits16(v) << (16 * q);
          act16(v, nullptr, act_c);
          put8_32(ta, part * 32 + 16 * q, v);
          put8_32(ta, part * 32 + 16 * q + 8, v + 8);
        }
        if (store_mask) {  // high halves of words 2 part, 2 part + 1
          uint16_t* mh = reinterpret_cast<uint16_t*>(masks + (uint64_t)(2 * part) * m.x_stride + gs) + 1;
          __stcs(mh, (uint16_t)(bits & 0xffffu));
          __stcs(mh + 2 * m.x_stride, (uint16_t)(bits >> 16));
        }
      }
      to_mma();
      // ---- L4: C2 = act(C1 Wc1^T + b) ----
      ISSUE_W(fiw, gemm_ts32<64, 64>(tmem, a_op, sm.w.c1[0], sm.w.c1[1]));
      mma_done();
      {
        uint32_t bits = 0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          float v[16];
          ld16(my_lanes + part * 32 + 16 * q, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += sm.w.bc1[part * 32 + 16 * q + i];
          bits |= relu_bits16(v) << (16 * q);
          act16(v, nullptr, act_c);
          put8_32(ta, part * 32 + 16 * q, v);
          put8_32(ta, part * 32 + 16 * q + 8, v + 8);
        }
        if (store_mask) __stcs(masks + (uint64_t)(4 + part) * m.x_stride + gs, bits);
      }
      to_mma();
      // ---- L5: rgb = sigmoid(clip(C2 Wc2^T + b)) ----
      ISSUE_W(fiw, gemm_ts32<16, 64>(tmem, a_op, sm.w.c2[0], sm.w.c2[1]));
      mma_done();
      if (part == 0) {
        float v[16];
        ld16(my_lanes, v);
        float z[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          z[k] = v[k] + sm.w.bc2[k];
          clip_bits |= (z[k] > 15.f || z[k] < -15.f ? 1u : 0u) << (16 + k);
        }
        if (valid) {
          const float4 o = make_float4(expf(sm.sig_raw[row]), sigm(clip15(z[0])), sigm(clip15(z[1])),
                                       sigm(clip15(z[2])));
          __stcs(m.out + (m.perm ? __ldg(m.perm + gs) : gs), o);
          if (m.perm && m.out_tile) __stcs(m.out_tile + gs, o);
        }
        if (store_mask) __stcs(masks + 6ull * m.x_stride + gs, clip_bits);
      }
      if (!has_next) break;
      if (nx.f != loaded) {
        __syncthreads();  // every thread is done with the old biases
        stage_weights_tf32(m.fields[nx.f], m.params, sm.w);
        loaded = nx.f;
        act_c = m.fields[nx.f].coarse ? 2 : 1;
      }
      put_x();  // the A region is free: every MMA has completed
      tile = next;
      cur = nx;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 256);
}

// Evaluation forward (dg_render / evaluate_rays): split-bf16 (3 MMAs per 16-wide K step, 2^-17
// operand error, inside the render's 1e-4 bar) — there is no backward, so no ReLU decision
// needs the training forward's split-tf32 precision, and bf16 operands pack two per TMEM column
// (half the epilogue stores, full-rate MMAs).  TMEM: [0, 64) the accumulator, [64, 128) A.
struct EvalTcSmem {
  TcWeights w;
  float sig_raw[TM];
  uint64_t mbar;
  uint32_t tslot;
};

// 2 column parts (warps 0-3 / 4-7) x 4 lane quadrants; each thread owns one sample row and 32 of
// the 64 hidden columns; tiles strided over the grid (as k_mlp_fwd_tc).
#ifndef MLP_EVAL_MINB
#define MLP_EVAL_MINB 4  // CTAs per SM (128 TMEM columns and ~47 KB of smem each): 2 -> 4 +2.4 % render
#endif
__global__ void __launch_bounds__(NTF, MLP_EVAL_MINB) k_mlp_eval_tc(MlpLaunch m) {
  constexpr int NP = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  EvalTcSmem& sm = *reinterpret_cast<EvalTcSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, part = warp >> 2;
  const int row = quad * 32 + lane;  // TMEM lane == sample row of the tile
  if (warp == 0) tc::tmem_alloc(&sm.tslot, 128);
  if (tid == 0) {
    tc::mbar_init(&sm.mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = sm.tslot;
  const uint32_t my_lanes = tmem + ((uint32_t)(quad * 32) << 16);
  const Sink act{nullptr, nullptr, my_lanes + A_HI};
  const uint32_t a_op = tmem + A_HI;
  uint32_t phase = 0;
  auto mma_done = [&]() {
    tc::mbar_wait(&sm.mbar, phase);
    phase ^= 1u;
    tc::fence_after();
  };
  uint32_t tile = blockIdx.x;
  if (tile < m.n_tiles) {
    TileGeo cur = tile_geo(m, tile);
    Pref<NP> pf;
    pf.start(m, row < cur.count, cur.s0 + row, part, false);
    pf.rec(m, part);
    pf.appearance(m, m.fields[cur.f], part);
    stage_weights_tc(m.fields[cur.f], m.params, sm.w);
    int loaded = cur.f;
    int act_c = m.fields[cur.f].coarse ? 2 : 1;  // colour activation of the loaded field
    pf.put_x(act, row, part);
    for (;;) {
      const bool valid = row < cur.count;
      const uint64_t gs = cur.s0 + row;
      const uint32_t next = tile + gridDim.x;
      const bool has_next = next < m.n_tiles;
      const TileGeo nx = has_next ? tile_geo_at(m, cur, next) : cur;
      to_mma();
      // ---- L1: H1 = relu(X Wd0^T + b) ----
      ISSUE(gemm_ts<64, 32>(tmem, a_op, sm.w.d0[0], sm.w.d0[1]));
      float cin_app[17];
#pragma unroll
      for (int i = 0; i < 17; ++i) cin_app[i] = pf.app[i];
      const double d0 = pf.dir[0], d1 = pf.dir[1], d2 = pf.dir[2];
      pf.start(m, has_next && row < nx.count, nx.s0 + row, part, false);  // next tile: X, item
      mma_done();
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float v[16];
        ld16(my_lanes + part * 32 + 16 * q, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i] + sm.w.bd0[part * 32 + 16 * q + i], 0.f);
        put8(act, row, part * 32 + 16 * q, v);
        put8(act, row, part * 32 + 16 * q + 8, v + 8);
      }
      to_mma();
      // ---- L2: raw16 = H1 Wd1^T + b ; Cin = [clip(raw1..15) | SH16 | app | 0] ----
      ISSUE(gemm_ts<16, 64>(tmem, a_op, sm.w.d1[0], sm.w.d1[1]));
      mma_done();
      {
        float raw[16];
        if (part == 0) {
          ld16(my_lanes, raw);
#pragma unroll
          for (int i = 0; i < 16; ++i) raw[i] = clip15(raw[i] + sm.w.bd1[i]);
          sm.sig_raw[row] = raw[0];
        }
        // this tile's dir / app were prefetched into the (now next-tile) registers: restore
        Pref<NP> cp;
        cp.valid = valid;
        cp.dir[0] = d0;
        cp.dir[1] = d1;
        cp.dir[2] = d2;
#pragma unroll
        for (int i = 0; i < 17; ++i) cp.app[i] = cin_app[i];
        cp.put_cin(act, row, part, raw);
      }
      pf.rec(m, part);  // next tile's RayRec (item arrived during L1/L2)
      to_mma();
      // ---- L3: C1 = act(Cin Wc0^T + b) ----
      ISSUE(gemm_ts<64, 48>(tmem, a_op, sm.w.c0[0], sm.w.c0[1]));
      mma_done();
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float v[16];
        ld16(my_lanes + part * 32 + 16 * q, v);
        act16(v, sm.w.bc0 + part * 32 + 16 * q, act_c);
        put8(act, row, part * 32 + 16 * q, v);
        put8(act, row, part * 32 + 16 * q + 8, v + 8);
      }
      to_mma();
      // ---- L4: C2 = act(C1 Wc1^T + b) ----
      ISSUE(gemm_ts<64, 64>(tmem, a_op, sm.w.c1[0], sm.w.c1[1]));
      mma_done();
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float v[16];
        ld16(my_lanes + part * 32 + 16 * q, v);
        act16(v, sm.w.bc1 + part * 32 + 16 * q, act_c);
        put8(act, row, part * 32 + 16 * q, v);
        put8(act, row, part * 32 + 16 * q + 8, v + 8);
      }
      pf.appearance(m, m.fields[nx.f], part);  // next tile's appearance rows
      to_mma();
      // ---- L5: rgb = sigmoid(clip(C2 Wc2^T + b)) ----
      ISSUE(gemm_ts<16, 64>(tmem, a_op, sm.w.c2[0], sm.w.c2[1]));
      mma_done();
      if (part == 0) {
        float v[16];
        ld16(my_lanes, v);
        if (valid)
          __stcs(m.out + (m.perm ? __ldg(m.perm + gs) : gs),
                 make_float4(expf(sm.sig_raw[row]), sigm(clip15(v[0] + sm.w.bc2[0])),
                             sigm(clip15(v[1] + sm.w.bc2[1])), sigm(clip15(v[2] + sm.w.bc2[2]))));
      }
      if (!has_next) break;
      if (nx.f != loaded) {
        __syncthreads();  // every thread is done with the old biases
        stage_weights_tc(m.fields[nx.f], m.params, sm.w);
        loaded = nx.f;
        act_c = m.fields[nx.f].coarse ? 2 : 1;
      }
      pf.put_x(act, row, part);  // the A region is free: every MMA has completed
      tile = next;
      cur = nx;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 128);
}


// ============================================================================ backward
// Per tile of 128 samples: recompute the forward's hidden layers (keeping every layer input in
// smem; the output layer is not recomputed: the colour-head adjoint and the sigma path take
// the forward's stored sigma / rgb, MlpLaunch::out_tile, with its clip flags), then
//   B1  G5  = d raw_rgb (clip/sigmoid adjoint)            dWc2 += G5^T C2 ; dC2 = G5 Wc2
//   B2  G4  = dC2 * act'(C2)                              dWc1 += G4^T C1 ; dC1 = G4 Wc1
//   B3  G3  = dC1 * act'(C1)                              dWc0 += G3^T Cin; dCin = G3 Wc0[:, :16]
//   B4  G2  = [sigma path, clip-masked dCin[0..14]]       dWd1 += G2^T H1 ; dH1 = G2 Wd1
//   B5  G1  = dH1 * relu'(H1)                             dWd0 += G1^T X  ; dX = G1 Wd0
//   B6  dX -> global (level-major), for the hash-grid backward.
// Input-gradient GEMMs (dC2, ...) take G from the TMEM A region.  The weight gradients
// dW = G^T A are M=64 tcgen05 GEMMs over K = 128 samples reading the G and activation tiles
// in smem through MN-major descriptors (no transposed copies); bias gradients are G^T . 1
// against a constant ones tile.  Both accumulate in TMEM over every tile a CTA processes and
// are flushed with one atomicAdd per weight per CTA.
// Weight-gradient GEMMs are off the critical path: a stage issues its input-gradient GEMM,
// commits (the next epilogue waits only for that), then issues the weight-gradient GEMMs.  The
// G tiles rotate through buffers no in-flight weight-gradient GEMM reads:
//   G5 -> g5, G4 -> s, G3 -> c2, G2 -> s, G1 -> c2,  and the next tile's x reaches smem only at
//   its first epilogue (the previous tile's dWd0 GEMM reads x).
// 16 warps: 4 lane quadrants x 4 column parts, so every epilogue is 16 columns per thread.
constexpr int XW = 32, HW = 64, CW = 48;  // activation tile widths

// Bias gradients ride in the weight-gradient GEMMs: the hi activation tiles of x / cin sit
// right before, and those of h1 / c1 right after, a 2 KB chunk whose column 0 is 1 (bf16
// exact, so its lo part is 0 and the hi.lo product skips it): B = [A | 1] (append) or
// [1 | A] (prepend) gives dW and db in one N+8-wide MMA.  The output layer's 3 bias
// gradients are warp-reduced in the B1 epilogue instead.
struct BwdTcSmem {
  TcWeights w;
  uint8_t g5[2][TM * 16 * 2];  // G5 hi / lo (the N = 16 operand of dWc2^T)
  uint8_t x_hi[TM * XW * 2];
  uint8_t ones_a[TM * 8 * 2];  // [x | 1] and [1 | h1]
  uint8_t h1_hi[TM * HW * 2];
  uint8_t cin_hi[TM * CW * 2];
  uint8_t ones_b[TM * 8 * 2];  // [cin | 1] and [1 | c1]
  uint8_t c1_hi[TM * HW * 2];
  uint8_t x_lo[TM * XW * 2];
  uint8_t h1_lo[TM * HW * 2];
  uint8_t cin_lo[TM * CW * 2];
  uint8_t c1_lo[TM * HW * 2];
  uint8_t c2[2][TM * HW * 2];
  uint8_t s[2][TM * 64 * 2];   // G4 / G2
  float bias_c2[4];            // output-layer bias gradient, summed over the CTA's tiles
  float sig_raw[TM];
  float gsig[TM];
  uint32_t dmask[TM];
  uint64_t mbar;
  uint64_t mbar_b;  // k_mlp_bwd_tc_relu: completion of the input-gradient chain's GEMMs
  uint32_t tslot;
};

static_assert(sizeof(BwdTcSmem) <= 232448, "backward tile set exceeds 227 KB of shared memory");

// TMEM columns: [0,64) accumulator, [64,128) A operand; dW accumulators (M = 64 rows = out
// features, row o at lane (o % 16) + 32 (o / 16)) with the bias column folded in: appended
// after dW (C0: [cin | 1], D0: [x | 1]) or prepended (C1: [1 | c1], D1: [1 | h1]).
// The dW block fills columns [256, 512): the paired ReLU backward (k_mlp_bwd_tc_relu) keeps a
// second accumulator and A region at [128, 256).
constexpr uint32_t TD_C2 = 256;                    // dWc2^T: 16 of 64 (bias: epilogue)
constexpr uint32_t TB_C1 = 272, TD_C1 = 280;       // 8 + 64
constexpr uint32_t TD_C0 = 344, TB_C0 = 392;       // 48 + 8
constexpr uint32_t TB_D1 = 400, TD_D1 = 408;       // 8 + 64
constexpr uint32_t TD_D0 = 472, TB_D0 = 504;       // 32 + 8
constexpr uint32_t kNoBias = 0xffffffffu;

// D (M=64 x N) (+)= G^T A over K = TM samples; G tile (TM x >=64 cols span), A tile (TM x N);
// both read MN-major (SBO = TM/8*128, LBO = 128).
template <int N>
__device__ __forceinline__ void gemm_wgrad(uint32_t d_tmem, const uint8_t* g_hi, const uint8_t* g_lo,
                                           const uint8_t* a_hi, const uint8_t* a_lo, bool accumulate) {
  constexpr uint32_t id = tc::idesc_bf16(64, N, 1, 1);
  constexpr uint32_t SBO = (TM / 8) * 128;
  const uint64_t gh = tc::smem_desc(tc::smem_u32(g_hi), 128, SBO);
  const uint64_t gl = tc::smem_desc(tc::smem_u32(g_lo), 128, SBO);
  const uint64_t ah = tc::smem_desc(tc::smem_u32(a_hi), 128, SBO);
  const uint64_t al = tc::smem_desc(tc::smem_u32(a_lo), 128, SBO);
  const uint32_t acc0 = accumulate ? 1u : 0u;
#pragma unroll
  for (int k = 0; k < TM / 16; ++k) {
    const uint32_t o = (k * 256) >> 4;
    tc::mma_bf16(d_tmem, gh + o, ah + o, id, k > 0 ? 1u : acc0);
    tc::mma_bf16(d_tmem, gh + o, al + o, id, 1u);
    tc::mma_bf16(d_tmem, gl + o, ah + o, id, 1u);
  }
}

// dW and db in one accumulation: B = the hi tile extended by the ones chunk (N + 8 columns,
// b_ext = the first chunk: the ones chunk when prepended, the tile when appended) for the
// hi.hi and lo.hi products; the hi.lo product uses the lo tile alone (N columns, at d_lo =
// d + 8 when prepended), the ones' lo part being 0.
template <int N, bool kPrepend>
__device__ __forceinline__ void gemm_wgrad_bias(uint32_t d_tmem, const uint8_t* g_hi, const uint8_t* g_lo,
                                                const uint8_t* b_ext, const uint8_t* a_lo, bool accumulate) {
  constexpr uint32_t id_ext = tc::idesc_bf16(64, N + 8, 1, 1);
  constexpr uint32_t id = tc::idesc_bf16(64, N, 1, 1);
  constexpr uint32_t SBO = (TM / 8) * 128;
  const uint64_t gh = tc::smem_desc(tc::smem_u32(g_hi), 128, SBO);
  const uint64_t gl = tc::smem_desc(tc::smem_u32(g_lo), 128, SBO);
  const uint64_t be = tc::smem_desc(tc::smem_u32(b_ext), 128, SBO);
  const uint64_t al = tc::smem_desc(tc::smem_u32(a_lo), 128, SBO);
  const uint32_t acc0 = accumulate ? 1u : 0u;
  const uint32_t d_lo = kPrepend ? d_tmem + 8 : d_tmem;
#pragma unroll
  for (int k = 0; k < TM / 16; ++k) {
    const uint32_t o = (k * 256) >> 4;
    tc::mma_bf16(d_tmem, gh + o, be + o, id_ext, k > 0 ? 1u : acc0);
    tc::mma_bf16(d_lo, gh + o, al + o, id, 1u);
    tc::mma_bf16(d_tmem, gl + o, be + o, id_ext, 1u);
  }
}

// D (TM x N) = G W : G in the TMEM A region [TM x K=out], W tile stored [Wrows=out x cols=in]
// in smem read MN-major (SBO = Wrows/8*128, LBO = 128); N = number of leading input columns.
template <int Wrows, int N, int K>
__device__ __forceinline__ void gemm_igrad(uint32_t d_tmem, uint32_t a, const uint8_t* w_hi,
                                           const uint8_t* w_lo) {
  constexpr uint32_t id = tc::idesc_bf16(TM, N, 0, 1);
  constexpr uint32_t W_SBO = (uint32_t)(Wrows / 8) * 128;
  const uint64_t wh = tc::smem_desc(tc::smem_u32(w_hi), 128, W_SBO);
  const uint64_t wl = tc::smem_desc(tc::smem_u32(w_lo), 128, W_SBO);
#pragma unroll
  for (int k = 0; k < K / 16; ++k) {
    const uint32_t wo = (k * 256) >> 4;
    tc::mma_bf16_ts(d_tmem, a + 8 * k, wh + wo, id, k > 0 ? 1u : 0u);
    tc::mma_bf16_ts(d_tmem, a + 8 * k, wl + wo, id, 1u);
    tc::mma_bf16_ts(d_tmem, a + A_LO_OFF + 8 * k, wh + wo, id, 1u);
  }
}

// One dW accumulator (M=64 layout: row o in TMEM lane (o % 16) + 32 (o / 16)) -> atomics:
// columns [0, in) of col0 are dW, column 0 of bcol is the bias gradient.
__device__ void flush_dw(uint32_t tmem, uint32_t col0, int N, int out, int in, uint32_t bcol, float* gW,
                         float* gb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, part = warp >> 2, parts = (int)(blockDim.x >> 7);
  const int o = quad * 16 + lane;
  const uint32_t lanes = tmem + ((uint32_t)(quad * 32) << 16);
  for (int g = part; g <= N / 8; g += parts) {
    if (g == N / 8 && bcol == kNoBias) break;
    float v[8];
    tc::tmem_ld8(lanes + (g < N / 8 ? col0 + 8 * g : bcol), v);
    tc::tmem_wait_ld();
    if (lane < 16 && o < out) {
      if (g == N / 8) {
        if (v[0] != 0.f) atomicAdd(gb + o, v[0]);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = 8 * g + j;
          if (i < in && v[j] != 0.f) atomicAdd(gW + o * in + i, v[j]);
        }
      }
    }
  }
}

__device__ void flush_all(uint32_t tmem, const FieldDesc& fd, float* __restrict__ grads, float* bias_c2) {
  float* base = grads + fd.base;
  const int enc = (int)fd.L * 2, cin = 31 + (int)fd.app_dim;
  if (threadIdx.x < 3) {  // the epilogue-reduced output-layer bias
    if (bias_c2[threadIdx.x] != 0.f) atomicAdd(base + fd.cb2 + threadIdx.x, bias_c2[threadIdx.x]);
    bias_c2[threadIdx.x] = 0.f;
  }
  {  // dWc2^T: row i (C2 feature) in lane (i % 16) + 32 (i / 16), column o (output, < 3)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, quad = warp & 3;
    if ((warp >> 2) == 0) {
      float v[8];
      tc::tmem_ld8(tmem + ((uint32_t)(quad * 32) << 16) + TD_C2, v);
      tc::tmem_wait_ld();
      const int i = quad * 16 + lane;
      if (lane < 16) {
        float* gW = base + fd.cw2;
#pragma unroll
        for (int o = 0; o < 3; ++o)
          if (v[o] != 0.f) atomicAdd(gW + o * 64 + i, v[o]);
      }
    }
  }
  flush_dw(tmem, TD_C1, HW, 64, 64, TB_C1, base + fd.cw1, base + fd.cb1);
  flush_dw(tmem, TD_C0, CW, 64, cin, TB_C0, base + fd.cw0, base + fd.cb0);
  flush_dw(tmem, TD_D1, HW, 16, 64, TB_D1, base + fd.dw1, base + fd.db1);
  flush_dw(tmem, TD_D0, XW, 64, enc, TB_D0, base + fd.dw0, base + fd.db0);
}

// G = act'(a) * dv for 16 columns of row r; a is read back from the activation tile (hi, lo),
// G goes to `out` (its smem tile for the weight gradient + the TMEM A region).
// ReLU layers use the forward's mask bits (the sign of the split-tf32 pre-activation); the
// sigmoid derivative comes from the activation value.
__device__ __forceinline__ void grad_act16(const uint8_t* a_hi, const uint8_t* a_lo, const Sink& out,
                                           int r, int c0, float* v, int act, uint32_t bits) {
  if (act == 2) {
    float a[16];
    get8(a_hi, a_lo, r, c0, a);
    get8(a_hi, a_lo, r, c0 + 8, a + 8);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] *= a[i] * (1.f - a[i]);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = ((bits >> i) & 1u) ? v[i] : 0.f;
  }
  put8(out, r, c0, v);
  put8(out, r, c0 + 8, v + 8);
}

__global__ void __launch_bounds__(NTB, 1) k_mlp_bwd_tc(MlpLaunch m, uint32_t t_lo, uint32_t t_hi) {
  constexpr int NP = 4;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  BwdTcSmem& sm = *reinterpret_cast<BwdTcSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, part = warp >> 2;
  const int row = quad * 32 + lane;
  const int c16 = part * 16;  // this thread's 16 columns of a 64-wide layer
  if (warp == 0) tc::tmem_alloc(&sm.tslot, 512);
  if (tid == 0) {
    tc::mbar_init(&sm.mbar, 1);
    tc::fence_mbar_init();
  }
  // ones tile (bias-gradient B operand, MN-major [K = 128 samples x N = 8]): column 0 = 1
  for (int r = tid; r < TM; r += NTB) {
    *reinterpret_cast<uint4*>(sm.ones_a + tc::core_offset(r, 0, TM)) = make_uint4(0x3f80u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(sm.ones_b + tc::core_offset(r, 0, TM)) = make_uint4(0x3f80u, 0u, 0u, 0u);
  }
  if (tid < 4) sm.bias_c2[tid] = 0.f;
  for (int i = tid; i < (int)(sizeof(sm.g5) / 16); i += NTB)  // G5 columns 3-15 stay 0
    reinterpret_cast<uint4*>(sm.g5)[i] = make_uint4(0u, 0u, 0u, 0u);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = sm.tslot;
  const uint32_t my_lanes = tmem + ((uint32_t)(quad * 32) << 16);
  const uint32_t a_op = tmem + A_HI, ta = my_lanes + A_HI;
  // operand tiles: smem copy (weight-gradient GEMMs) + TMEM A region (the next GEMM)
  const Sink sxt{nullptr, nullptr, ta}, sh1{sm.h1_hi, sm.h1_lo, ta}, scin{sm.cin_hi, sm.cin_lo, ta};
  const Sink sc1{sm.c1_hi, sm.c1_lo, ta}, sc2{sm.c2[0], sm.c2[1], ta}, sg5{sm.g5[0], sm.g5[1], ta};
  const Sink ss{sm.s[0], sm.s[1], ta};
  float xk[8];  // this tile's X chunk: TMEM A at once, the smem copy at the first epilogue
  uint32_t phase = 0;
#ifdef DG_TRACE_MLP
  // phase clocks of CTA 0 (threads 0 and 480): per stage [barrier entry, barrier exit, MMA done]
  int tr_tile = 0, tr_pt = 0;
  auto trace = [&]() {
    if (blockIdx.x == 0 && (tid == 0 || tid == 480) && tr_tile < 64 && tr_pt < 32)
      m.trace[(tr_tile * 2 + (tid ? 1 : 0)) * 32 + tr_pt] = clock64();
    ++tr_pt;
  };
#else
  auto trace = []() {};
#endif
  auto mma_done = [&]() {
    tc::mbar_wait(&sm.mbar, phase);
    phase ^= 1u;
    tc::fence_after();
    trace();
  };
  auto sync_mma = [&]() {
    trace();
    to_mma();
    trace();
  };
  // balanced contiguous tile range per CTA of [t_lo, t_hi)
  const uint32_t t_begin = t_lo + (uint32_t)(((uint64_t)blockIdx.x * (t_hi - t_lo)) / gridDim.x);
  const uint32_t t_end = t_lo + (uint32_t)(((uint64_t)(blockIdx.x + 1) * (t_hi - t_lo)) / gridDim.x);
  int loaded = -1;
  if (t_begin < t_end) {
    uint32_t tile = t_begin;
    TileGeo cur = tile_geo(m, tile);
    Pref<NP> pf;
    pf.start(m, row < cur.count, cur.s0 + row, part, true);
    pf.rec(m, part);
    pf.appearance(m, m.fields[cur.f], part);
    stage_weights_tc(m.fields[cur.f], m.params, sm.w);
    loaded = cur.f;
    bool fresh = true;  // next dW GEMMs start a new accumulation
    int act_c = m.fields[cur.f].coarse ? 2 : 1;  // colour activation of the loaded field
    pf.put_x(sxt, row, part);
#pragma unroll
    for (int i = 0; i < 8; ++i) xk[i] = pf.x[i];
    for (;;) {
      const bool valid = row < cur.count;
      const uint64_t gs = cur.s0 + row;
      const uint32_t next = tile + 1;
      const bool has_next = next < t_end;
      const TileGeo nx = has_next ? tile_geo_next(m, cur, next) : cur;
      // this tile's prefetched dir / app / upstream gradient move out of the prefetch registers
      float cur_app[17];
#pragma unroll
      for (int i = 0; i < 17; ++i) cur_app[i] = pf.app[i];
      const double d0 = pf.dir[0], d1 = pf.dir[1], d2 = pf.dir[2];
      const float4 up = pf.g;
      // the forward's masks of this tile: first needed at B1, five epilogues from now, so the
      // loads are issued here rather than held in prefetch registers through the previous tile
      // (this part's 16 columns: h1 bits 0-15 | c1 bits 16-31, the c2 word; part 0: clip word)
      uint32_t mk_relu = 0u, mk_c2 = 0u, mk_clip = 0u;
      float4 o_fwd = make_float4(0.f, 0.f, 0.f, 0.f);  // the forward's (sigma, rgb), part 0
      if (valid) {
        mk_relu = __ldcs(m.masks + (uint64_t)part * m.x_stride + gs);
        mk_c2 = __ldcs(m.masks + (uint64_t)(4 + (part >> 1)) * m.x_stride + gs);
        if (part == 0) {
          mk_clip = __ldcs(m.masks + 6ull * m.x_stride + gs);
          o_fwd = __ldcs(m.out_tile + gs);
        }
      }
      sync_mma();
      // ---------------- forward recompute (A operands from TMEM) ----------------
      ISSUE(gemm_ts<64, 32>(tmem, a_op, sm.w.d0[0], sm.w.d0[1]));
      pf.start(m, has_next && row < nx.count, nx.s0 + row, part, false);  // next: X, item
      mma_done();
      {
        put8s(sm.x_hi, sm.x_lo, row, part * 8, xk);  // the previous tile's dWd0 GEMM is done
        float v[16];
        ld16(my_lanes + c16, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i] + sm.w.bd0[c16 + i], 0.f);
        put8(sh1, row, c16, v);
        put8(sh1, row, c16 + 8, v + 8);
      }
      sync_mma();
      ISSUE(gemm_ts<16, 64>(tmem, a_op, sm.w.d1[0], sm.w.d1[1]));
      mma_done();
      {
        float raw[16];
        if (part == 0) {
          ld16(my_lanes, raw);
#pragma unroll
          for (int i = 0; i < 16; ++i) raw[i] = clip15(raw[i] + sm.w.bd1[i]);
          sm.sig_raw[row] = raw[0];
        }
        Pref<NP> cp;
        cp.valid = valid;
        cp.dir[0] = d0;
        cp.dir[1] = d1;
        cp.dir[2] = d2;
#pragma unroll
        for (int i = 0; i < 17; ++i) cp.app[i] = cur_app[i];
        cp.put_cin(scin, row, part, raw);
      }
      sync_mma();
      ISSUE(gemm_ts<64, 48>(tmem, a_op, sm.w.c0[0], sm.w.c0[1]));
      mma_done();
      {
        float v[16];
        ld16(my_lanes + c16, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float z = v[i] + sm.w.bc0[c16 + i];
          v[i] = act_c == 2 ? sigm(z) : fmaxf(z, 0.f);
        }
        put8(sc1, row, c16, v);
        put8(sc1, row, c16 + 8, v + 8);
      }
      pf.rec(m, part);  // next tile's RayRec
      sync_mma();
      ISSUE(gemm_ts<64, 64>(tmem, a_op, sm.w.c1[0], sm.w.c1[1]));
      mma_done();
      {
        float v[16];
        ld16(my_lanes + c16, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float z = v[i] + sm.w.bc1[c16 + i];
          v[i] = act_c == 2 ? sigm(z) : fmaxf(z, 0.f);
        }
        // C2 feeds only dWc2 here (its smem tile): the output layer is not recomputed
        put8s(sm.c2[0], sm.c2[1], row, c16, v);
        put8s(sm.c2[0], sm.c2[1], row, c16 + 8, v + 8);
      }
      mk_c2 = (mk_c2 >> (((uint32_t)part & 1u) * 16u)) & 0xffffu;
      // ---------------- B1: colour head adjoint (field.cpp:298-306) ----------------
      // from the forward's outputs (sigma = exp(clip(raw0)), rgb = sigmoid(clip(z))) and its
      // clip flags, so the output-layer GEMM is not recomputed
      if (part == 0) {
        sm.dmask[row] = mk_clip & 0xffffu;  // the forward's clip flags
        const float ug[3] = {up.y, up.z, up.w};
        const float sgs[3] = {o_fwd.y, o_fwd.z, o_fwd.w};
        float g[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) g[k] = 0.f;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const bool clipped = (mk_clip >> (16 + k)) & 1u;
          g[k] = clipped ? 0.f : ug[k] * sgs[k] * (1.f - sgs[k]);
        }
        // columns 8-15 of G5 are always 0: zeroed once in shared memory; in the TMEM A region
        // they keep the previous operand's finite values, which meet zero-padded Wc2 rows
        put8(sg5, row, 0, g);
        // sigma path of the density raw gradient (field.cpp:313): up.sigma * exp(raw0)
        sm.gsig[row] = (sm.dmask[row] & 1u) ? 0.f : up.x * o_fwd.x;
      }
      pf.grad(m, part);  // next tile's upstream gradient
      sync_mma();
      issue2(warp, &sm.mbar, [&] { gemm_igrad<16, 64, 16>(tmem, a_op, sm.w.c2[0], sm.w.c2[1]); },
             // dWc2 transposed: D[64 C2 features x 16] = C2^T G5 (the c2 tile as the M = 64 operand,
             // G5 as a 16-column B): a quarter of the B bytes of G5^T C2 at N = 64
             [&] { gemm_wgrad<16>(tmem + TD_C2, sm.c2[0], sm.c2[1], sm.g5[0], sm.g5[1], !fresh); });
      mma_done();
      // ---------------- B2: G4 = dC2 * act'(C2) -> s ----------------
      {
        float v[16];
        ld16(my_lanes + c16, v);
        grad_act16(sm.c2[0], sm.c2[1], ss, row, c16, v, act_c, mk_c2);
      }
      sync_mma();
      issue2(warp, &sm.mbar, [&] { gemm_igrad<64, 64, 64>(tmem, a_op, sm.w.c1[0], sm.w.c1[1]); },
             [&] { gemm_wgrad_bias<HW, true>(tmem + TB_C1, sm.s[0], sm.s[1], sm.ones_b, sm.c1_lo, !fresh); });
      mma_done();
      // ---------------- B3: G3 = dC1 * act'(C1) -> c2 ----------------
      {
        float v[16];
        ld16(my_lanes + c16, v);
        grad_act16(sm.c1_hi, sm.c1_lo, sc2, row, c16, v, act_c, mk_relu >> 16);
      }
      pf.appearance(m, m.fields[nx.f], part);  // next tile's appearance rows
      sync_mma();
      issue2(warp, &sm.mbar, [&] { gemm_igrad<64, 16, 64>(tmem, a_op, sm.w.c0[0], sm.w.c0[1]); },
             [&] { gemm_wgrad_bias<CW, false>(tmem + TD_C0, sm.c2[0], sm.c2[1], sm.cin_hi, sm.cin_lo, !fresh); });
      mma_done();
      // ---------------- B4: G2 = density raw gradient -> s cols 0..15 ----------------
      if (part == 0) {
        float v[16];
        ld16(my_lanes, v);
        const uint32_t mask = sm.dmask[row];
        float g[16];
        g[0] = sm.gsig[row];
#pragma unroll
        for (int k = 1; k < 16; ++k) g[k] = ((mask >> k) & 1u) ? 0.f : v[k - 1];
        put8(ss, row, 0, g);
        put8(ss, row, 8, g + 8);
      } else if (part == 1) {
        // output-layer bias gradient db = G5^T . 1 (off the critical path: part 1 is idle in
        // this 16-column epilogue; G5 stays in smem until the next tile's B1)
        float g5[8];
        get8(sm.g5[0], sm.g5[1], row, 0, g5);
        float b0 = g5[0], b1 = g5[1], b2 = g5[2];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          b0 += __shfl_xor_sync(0xffffffffu, b0, o);
          b1 += __shfl_xor_sync(0xffffffffu, b1, o);
          b2 += __shfl_xor_sync(0xffffffffu, b2, o);
        }
        if (lane == 0) {
          atomicAdd(&sm.bias_c2[0], b0);
          atomicAdd(&sm.bias_c2[1], b1);
          atomicAdd(&sm.bias_c2[2], b2);
        }
      }
      sync_mma();
      issue2(warp, &sm.mbar, [&] { gemm_igrad<16, 64, 16>(tmem, a_op, sm.w.d1[0], sm.w.d1[1]); },
             [&] { gemm_wgrad_bias<HW, true>(tmem + TB_D1, sm.s[0], sm.s[1], sm.ones_a, sm.h1_lo, !fresh); });
      mma_done();
      // ---------------- B5: G1 = dH1 * relu'(H1) -> c2 ----------------
      {
        float v[16];
        ld16(my_lanes + c16, v);
        grad_act16(sm.h1_hi, sm.h1_lo, sc2, row, c16, v, 1, mk_relu & 0xffffu);
      }
      sync_mma();
      issue2(warp, &sm.mbar, [&] { gemm_igrad<64, 32, 64>(tmem, a_op, sm.w.d0[0], sm.w.d0[1]); },
             [&] { gemm_wgrad_bias<XW, false>(tmem + TD_D0, sm.c2[0], sm.c2[1], sm.x_hi, sm.x_lo, !fresh); });
      mma_done();
      fresh = false;
      // ---------------- B6: dX -> global, level-major; next tile's X into the x tile ----------------
      {
        float v[8];
        tc::tmem_ld8(my_lanes + part * 8, v);
        tc::tmem_wait_ld();
        if (valid) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int l = part * 4 + j;
            if (l < (int)m.levels)
              __stcs(reinterpret_cast<float2*>(m.dX) + (uint64_t)l * m.x_stride + gs,
                     make_float2(v[2 * j], v[2 * j + 1]));
          }
        }
      }
#ifdef DG_TRACE_MLP
      ++tr_tile;
      tr_pt = 0;
#endif
      if (!has_next || nx.f != loaded) {  // the weight-gradient GEMMs must land before a flush
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        issue2(warp, &sm.mbar, [] {}, [] {});
        mma_done();
      }
      if (!has_next) break;
      if (nx.f != loaded) {
        flush_all(tmem, m.fields[loaded], m.grads, sm.bias_c2);
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        stage_weights_tc(m.fields[nx.f], m.params, sm.w);
        loaded = nx.f;
        act_c = m.fields[nx.f].coarse ? 2 : 1;
        fresh = true;
      }
      pf.put_x(sxt, row, part);  // A region is free (the dX GEMM completed); smem x at F1
#pragma unroll
      for (int i = 0; i < 8; ++i) xk[i] = pf.x[i];
      tile = next;
      cur = nx;
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (loaded >= 0) flush_all(tmem, m.fields[loaded], m.grads, sm.bias_c2);
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 512);
}

// ------------------------------------------------------------ backward, ReLU fields
// In a ReLU field (the fine field, field.cpp:196-199) every activation derivative of the
// backward comes from the forward's stored masks, so the input-gradient chain
// G5 -> dC2 -> G4 -> dC1 -> G3 -> dCin -> G2 -> dH1 -> G1 -> dX never waits for the forward
// recompute, which feeds only the weight gradients.  The two chains run as paired stages, each
// with its own TMEM accumulator and A region, so a tile has 5 MMA waits instead of 9:
//   S1  F1 = X Wd0^T      (-> H1 = relu)            | dC2 = G5 Wc2      (-> G4 = dC2 * c2 mask)
//       + the previous tile's dWd0
//   S2  F2 = H1 Wd1^T     (-> raw -> Cin)           | dC1 = G4 Wc1      (-> G3 = dC1 * c1 mask)
//   S3  F3 = Cin Wc0^T    (-> C1)                   | dCin = G3 Wc0     (-> G2)      + dWc0
//   S4  F4 = C1 Wc1^T     (-> C2)                   | dH1 = G2 Wd1      (-> G1)      + dWc1
//   S5                                              | dX = G1 Wd0                    + dWc2, dWd1
// Every weight-gradient GEMM is issued behind a stage's critical GEMMs and runs under the
// next epilogue.  G5 comes from the forward's stored outputs and clip flags (as in
// k_mlp_bwd_tc).  Operand tiles are placed so that no in-flight GEMM's operand is
// overwritten: two 64-column buffers (s, c2) swap roles every tile — A holds G4 then G1
// (copied out of the TMEM A region at S5's epilogue), B holds G3 then C2 — X reaches its smem
// tile at S2's epilogue (after the previous tile's dWd0), and G2 the cin tile at S4's
// epilogue (copied out of the TMEM A region, after dWc0 has read Cin).
// Same arithmetic as k_mlp_bwd_tc (split-bf16 operands, fp32 TMEM accumulation, dW / db over
// all of a CTA's tiles); only the issue order of the GEMMs differs.
constexpr uint32_t TF_ACC = 0, TF_A = 64, TB_ACC = 128, TB_A = 192;

// 16 columns [c0, c0 + 16) of this thread's row of a TMEM A region (packed bf16 pairs, hi at ta,
// lo at ta + A_LO_OFF) -> the smem operand tile (hi / lo), bit for bit.
__device__ __forceinline__ void a_to_smem16(uint32_t ta, int r, int c0, uint8_t* hi, uint8_t* lo) {
  float h[8], l[8];
  tc::tmem_ld8(ta + (uint32_t)(c0 >> 1), h);
  tc::tmem_ld8(ta + A_LO_OFF + (uint32_t)(c0 >> 1), l);
  tc::tmem_wait_ld();
  const uint32_t o0 = tc::core_offset(r, c0, TM), o1 = tc::core_offset(r, c0 + 8, TM);
  *reinterpret_cast<uint4*>(hi + o0) =
      make_uint4(__float_as_uint(h[0]), __float_as_uint(h[1]), __float_as_uint(h[2]), __float_as_uint(h[3]));
  *reinterpret_cast<uint4*>(hi + o1) =
      make_uint4(__float_as_uint(h[4]), __float_as_uint(h[5]), __float_as_uint(h[6]), __float_as_uint(h[7]));
  *reinterpret_cast<uint4*>(lo + o0) =
      make_uint4(__float_as_uint(l[0]), __float_as_uint(l[1]), __float_as_uint(l[2]), __float_as_uint(l[3]));
  *reinterpret_cast<uint4*>(lo + o1) =
      make_uint4(__float_as_uint(l[4]), __float_as_uint(l[5]), __float_as_uint(l[6]), __float_as_uint(l[7]));
}

// v[i] kept where bit i of `bits` is set (ReLU derivative from the forward's mask)
__device__ __forceinline__ void mask16(float* v, uint32_t bits) {
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = ((bits >> i) & 1u) ? v[i] : 0.f;
}

__global__ void __launch_bounds__(NTB, 1) k_mlp_bwd_tc_relu(MlpLaunch m, uint32_t t_lo, uint32_t t_hi) {
  constexpr int NP = 4;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  BwdTcSmem& sm = *reinterpret_cast<BwdTcSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, part = warp >> 2;
  const int row = quad * 32 + lane;
  const int c16 = part * 16;  // this thread's 16 columns of a 64-wide layer
  // MMAs are issued from warp m.issue_warp (default 8: part 2, the lightest epilogues)
  const int iw = warp == (int)m.issue_warp ? 0 : 1;
  if (warp == 0) tc::tmem_alloc(&sm.tslot, 512);
  if (tid == 0) {
    tc::mbar_init(&sm.mbar, 1);
    tc::mbar_init(&sm.mbar_b, 1);
    tc::fence_mbar_init();
  }
  for (int r = tid; r < TM; r += NTB) {
    *reinterpret_cast<uint4*>(sm.ones_a + tc::core_offset(r, 0, TM)) = make_uint4(0x3f80u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(sm.ones_b + tc::core_offset(r, 0, TM)) = make_uint4(0x3f80u, 0u, 0u, 0u);
  }
  if (tid < 4) sm.bias_c2[tid] = 0.f;
  for (int i = tid; i < (int)(sizeof(sm.g5) / 16); i += NTB)  // G5 columns 3-15 stay 0
    reinterpret_cast<uint4*>(sm.g5)[i] = make_uint4(0u, 0u, 0u, 0u);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = sm.tslot;
  const uint32_t my_lanes = tmem + ((uint32_t)(quad * 32) << 16);
  const uint32_t aF = tmem + TF_A, aB = tmem + TB_A;            // A operands of the two chains
  const uint32_t taF = my_lanes + TF_A, taB = my_lanes + TB_A;  // this thread's lane of them
  const Sink fT{nullptr, nullptr, taF}, fH1{sm.h1_hi, sm.h1_lo, taF}, fCin{sm.cin_hi, sm.cin_lo, taF};
  const Sink fC1{sm.c1_hi, sm.c1_lo, taF};
  const Sink bT{nullptr, nullptr, taB};
  if (part == 0) {  // G5's K columns 8-15 meet zero Wc2 rows: the region must start finite
    const uint32_t z[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int c = 0; c < 32; c += 4) {
      tc::tmem_st4(taB + (uint32_t)c, z);
      tc::tmem_st4(taB + A_LO_OFF + (uint32_t)c, z);
    }
  }
  // Each stage commits its forward-recompute GEMM and its input-gradient GEMM to separate
  // mbarriers (sm.mbar, sm.mbar_b): the recompute's epilogue starts while the input-gradient
  // GEMM still runs.  A commit covers every earlier tcgen05 op of the issuing thread.
  uint32_t phase = 0, phase_b = 0;
  auto done_f = [&]() {
    tc::mbar_wait(&sm.mbar, phase);
    phase ^= 1u;
    tc::fence_after();
  };
  auto done_b = [&]() {
    tc::mbar_wait(&sm.mbar_b, phase_b);
    phase_b ^= 1u;
    tc::fence_after();
  };
  // stage issue from warp 12: recompute GEMM, commit, input-gradient GEMM, commit, background
  auto issue3 = [&](auto fwd, auto bwd, auto back) {
    if (iw == 0) {
      if (tc::elect_one()) {
        fwd();
        tc::commit(&sm.mbar);
        bwd();
        tc::commit(&sm.mbar_b);
        back();
      }
      __syncwarp();
    }
  };
  // the same with the input-gradient GEMM first (where it is the shorter of the two, so its
  // epilogue starts while the recompute GEMM runs)
  auto issue3b = [&](auto fwd, auto bwd, auto back) {
    if (iw == 0) {
      if (tc::elect_one()) {
        bwd();
        tc::commit(&sm.mbar_b);
        fwd();
        tc::commit(&sm.mbar);
        back();
      }
      __syncwarp();
    }
  };
  auto issue_b = [&](auto bwd, auto back) {
    if (iw == 0) {
      if (tc::elect_one()) {
        bwd();
        tc::commit(&sm.mbar_b);
        back();
      }
      __syncwarp();
    }
  };
  // the forward's masks / outputs of a tile row (see k_mlp_fwd_tc for the word layout)
  auto load_fwd = [&](const TileGeo& g, bool ok, uint32_t& relu, uint32_t& c2, uint32_t& clip, float4& o) {
    relu = c2 = clip = 0u;
    o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ok && row < g.count) {
      const uint64_t s = (uint64_t)g.s0 + row;
      relu = __ldcs(m.masks + (uint64_t)part * m.x_stride + s);
      c2 = __ldcs(m.masks + (uint64_t)(4 + (part >> 1)) * m.x_stride + s);
      if (part == 0) {
        clip = __ldcs(m.masks + 6ull * m.x_stride + s);
        o = __ldcs(m.out_tile + s);
      }
    }
  };
  const uint32_t t_begin = t_lo + (uint32_t)(((uint64_t)blockIdx.x * (t_hi - t_lo)) / gridDim.x);
  const uint32_t t_end = t_lo + (uint32_t)(((uint64_t)(blockIdx.x + 1) * (t_hi - t_lo)) / gridDim.x);
  int loaded = -1;
  if (t_begin < t_end) {
    uint32_t tile = t_begin;
    TileGeo cur = tile_geo(m, tile);
    Pref<NP> pf;
    pf.start(m, row < cur.count, cur.s0 + row, part, true);
    pf.rec(m, part);
    pf.appearance(m, m.fields[cur.f], part);
    uint32_t mk_relu, mk_c2, mk_clip;
    float4 o_fwd;
    load_fwd(cur, true, mk_relu, mk_c2, mk_clip, o_fwd);
    if (m.fields[cur.f].coarse) __trap();  // sigmoid fields take k_mlp_bwd_tc
    stage_weights_tc(m.fields[cur.f], m.params, sm.w);
    loaded = cur.f;
    bool fresh = true;        // next dW GEMMs start a new accumulation
    bool pend = false;        // the previous tile's dWd0 is still to be issued
    bool pend_fresh = false;  // ... and starts its accumulation
    int par = 0;              // tile parity: which of s / c2 is buffer A (G4, G1) and B (G3, C2)
    // the previous tile's dWd0 (G1 in its buffer A = this tile's B)
    auto issue_pending = [&](int p_prev) {
      if (!pend) return;
      auto g1 = p_prev ? sm.c2 : sm.s;
      gemm_wgrad_bias<XW, false>(tmem + TD_D0, g1[0], g1[1], sm.x_hi, sm.x_lo, !pend_fresh);
    };
    for (;;) {
      auto bufA = par ? sm.c2 : sm.s;
      auto bufB = par ? sm.s : sm.c2;
      const Sink bA{bufA[0], bufA[1], taB}, bB{bufB[0], bufB[1], taB};
      const bool valid = row < cur.count;
      const uint64_t gs = cur.s0 + row;
      const uint32_t next = tile + 1;
      const bool has_next = next < t_end;
      const TileGeo nx = has_next ? tile_geo_next(m, cur, next) : cur;
      float cur_app[17];
#pragma unroll
      for (int i = 0; i < 17; ++i) cur_app[i] = pf.app[i];
      const double d0 = pf.dir[0], d1 = pf.dir[1], d2 = pf.dir[2];
      const float4 up = pf.g;
      // ---------------- prologue: X -> A_F; G5 (colour-head adjoint, field.cpp:298-306) -> A_B
      pf.put_x(fT, row, part);
      float xk[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) xk[i] = pf.x[i];
      float g5v[3] = {0.f, 0.f, 0.f};
      if (part == 0) {
        const uint32_t dm = mk_clip & 0xffffu;  // the forward's clip flags
        sm.dmask[row] = dm;
        const float ug[3] = {up.y, up.z, up.w};
        const float sgs[3] = {o_fwd.y, o_fwd.z, o_fwd.w};
        float g[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) g[k] = 0.f;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const bool clipped = (mk_clip >> (16 + k)) & 1u;
          g[k] = clipped ? 0.f : ug[k] * sgs[k] * (1.f - sgs[k]);
          g5v[k] = g[k];
        }
        put8(bT, row, 0, g);
        // sigma path of the density raw gradient (field.cpp:313): up.sigma * exp(raw0)
        sm.gsig[row] = (dm & 1u) ? 0.f : up.x * o_fwd.x;
      }
      to_mma();
      // ---------------- S1: F1 | dC2, + the previous tile's dWd0 ----------------
      issue3b([&] { gemm_ts<64, 32>(tmem + TF_ACC, aF, sm.w.d0[0], sm.w.d0[1]); },
              [&] { gemm_igrad<16, 64, 16>(tmem + TB_ACC, aB, sm.w.c2[0], sm.w.c2[1]); },
              [&] { issue_pending(par ^ 1); });
      pend = false;
      pf.start(m, has_next && row < nx.count, nx.s0 + row, part, false);  // next: X, item
      done_b();
      {
        if (part == 0) {  // G5 for dWc2 (the previous tile's dWc2 is done)
          float g[8] = {g5v[0], g5v[1], g5v[2], 0.f, 0.f, 0.f, 0.f, 0.f};
          put8s(sm.g5[0], sm.g5[1], row, 0, g);
        }
        float v[16];
        ld16(my_lanes + TB_ACC + (uint32_t)c16, v);
        mask16(v, (mk_c2 >> (((uint32_t)part & 1u) * 16u)) & 0xffffu);
        put8(bA, row, c16, v);  // G4 (buffer A held the previous tile's C2: dWc2 is done)
        put8(bA, row, c16 + 8, v + 8);
        done_f();
        ld16(my_lanes + TF_ACC + (uint32_t)c16, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i] + sm.w.bd0[c16 + i], 0.f);
        put8(fH1, row, c16, v);  // the previous tile's dWd1 is done
        put8(fH1, row, c16 + 8, v + 8);
      }
      to_mma();
      // ---------------- S2: F2 | dC1 ----------------
      issue3([&] { gemm_ts<16, 64>(tmem + TF_ACC, aF, sm.w.d1[0], sm.w.d1[1]); },
             [&] { gemm_igrad<64, 64, 64>(tmem + TB_ACC, aB, sm.w.c1[0], sm.w.c1[1]); }, [] {});
      pf.rec(m, part);  // next tile's RayRec
      done_f();
      // the previous tile's dWd0 is done: X to its smem tile.  Cin column parts: part 3 the
      // density outputs (cols 0-15), parts 1 / 2 SH / appearance (16-47), part 0 none (it
      // builds G5 and copies G2 in other epilogues)
      const int cpart = part == 3 ? 0 : (part == 0 ? 3 : part);
      put8s(sm.x_hi, sm.x_lo, row, part * 8, xk);
      {
        float raw[16];
        if (cpart == 0) {
          ld16(my_lanes + TF_ACC, raw);
#pragma unroll
          for (int i = 0; i < 16; ++i) raw[i] = clip15(raw[i] + sm.w.bd1[i]);
          sm.sig_raw[row] = raw[0];
        }
        Pref<NP> cp;
        cp.valid = valid;
        cp.dir[0] = d0;
        cp.dir[1] = d1;
        cp.dir[2] = d2;
#pragma unroll
        for (int i = 0; i < 17; ++i) cp.app[i] = cur_app[i];
        cp.put_cin(fCin, row, cpart, raw);
      }
      done_b();
      {
        float v[16];
        ld16(my_lanes + TB_ACC + (uint32_t)c16, v);
        mask16(v, mk_relu >> 16);  // c1 bits of this part's columns
        put8(bB, row, c16, v);  // G3 (buffer B held the previous tile's G1: dWd0 is done)
        put8(bB, row, c16 + 8, v + 8);
      }
      to_mma();
      // ---------------- S3: F3 | dCin, + dWc0 ----------------
      issue3b([&] { gemm_ts<64, 48>(tmem + TF_ACC, aF, sm.w.c0[0], sm.w.c0[1]); },
              [&] { gemm_igrad<64, 16, 64>(tmem + TB_ACC, aB, sm.w.c0[0], sm.w.c0[1]); },
              [&] { gemm_wgrad_bias<CW, false>(tmem + TD_C0, bufB[0], bufB[1], sm.cin_hi, sm.cin_lo, !fresh); });
      pf.appearance(m, m.fields[nx.f], part);  // next tile's appearance rows
      done_b();
      if (part == 3) {  // G2 = [sigma path, clip-masked dCin[0..14]] -> A_B (smem copy at S4)
        float v[16];
        ld16(my_lanes + TB_ACC, v);
        const uint32_t mask = sm.dmask[row];
        float g[16];
        g[0] = sm.gsig[row];
#pragma unroll
        for (int k = 1; k < 16; ++k) g[k] = ((mask >> k) & 1u) ? 0.f : v[k - 1];
        put8(bT, row, 0, g);
        put8(bT, row, 8, g + 8);
      } else if (part == 1) {  // output-layer bias gradient db = G5^T . 1
        float g5[8];
        get8(sm.g5[0], sm.g5[1], row, 0, g5);
        float b0 = g5[0], b1 = g5[1], b2 = g5[2];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          b0 += __shfl_xor_sync(0xffffffffu, b0, o);
          b1 += __shfl_xor_sync(0xffffffffu, b1, o);
          b2 += __shfl_xor_sync(0xffffffffu, b2, o);
        }
        if (lane == 0) {
          atomicAdd(&sm.bias_c2[0], b0);
          atomicAdd(&sm.bias_c2[1], b1);
          atomicAdd(&sm.bias_c2[2], b2);
        }
      }
      done_f();
      {
        float v[16];
        ld16(my_lanes + TF_ACC + (uint32_t)c16, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i] + sm.w.bc0[c16 + i], 0.f);
        put8(fC1, row, c16, v);
        put8(fC1, row, c16 + 8, v + 8);
      }
      to_mma();
      // ---------------- S4: F4 | dH1, + dWc1 ----------------
      issue3b([&] { gemm_ts<64, 64>(tmem + TF_ACC, aF, sm.w.c1[0], sm.w.c1[1]); },
              [&] { gemm_igrad<16, 64, 16>(tmem + TB_ACC, aB, sm.w.d1[0], sm.w.d1[1]); },
             [&] { gemm_wgrad_bias<HW, true>(tmem + TB_C1, bufA[0], bufA[1], sm.ones_b, sm.c1_lo, !fresh); });
      pf.grad(m, part);  // next tile's upstream gradient
      uint32_t n_relu, n_c2, n_clip;
      float4 n_o;
      load_fwd(nx, has_next, n_relu, n_c2, n_clip, n_o);
      done_b();
      // G2 -> cin tile for dWd1 (dWc0 has read cin), before G1 overwrites its A_B columns
      if (part == 0) a_to_smem16(taB, row, 0, sm.cin_hi, sm.cin_lo);
      {
        float v[16];
        ld16(my_lanes + TB_ACC + (uint32_t)c16, v);
        mask16(v, mk_relu & 0xffffu);  // h1 bits
        put8(bT, row, c16, v);
        put8(bT, row, c16 + 8, v + 8);
        done_f();
        ld16(my_lanes + TF_ACC + (uint32_t)c16, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i] + sm.w.bc1[c16 + i], 0.f);
        // C2 feeds only dWc2 (its smem tile in buffer B: dWc0 has read G3 from it)
        put8s(bufB[0], bufB[1], row, c16, v);
        put8s(bufB[0], bufB[1], row, c16 + 8, v + 8);
      }
      to_mma();
      // ---------------- S5: dX, + dWc2, dWd1 ----------------
      issue_b([&] { gemm_igrad<64, 32, 64>(tmem + TB_ACC, aB, sm.w.d0[0], sm.w.d0[1]); },
              [&] {
                // dWc2 transposed: D[64 C2 features x 16] = C2^T G5
                gemm_wgrad<16>(tmem + TD_C2, bufB[0], bufB[1], sm.g5[0], sm.g5[1], !fresh);
                // G2's 16 columns from the cin tile (the M = 64 operand's rows 16-63 are unused)
                gemm_wgrad_bias<HW, true>(tmem + TB_D1, sm.cin_hi, sm.cin_lo, sm.ones_a, sm.h1_lo, !fresh);
              });
      done_b();
      {  // dX -> global, level-major
        float v[8];
        tc::tmem_ld8(my_lanes + TB_ACC + (uint32_t)(part * 8), v);
        tc::tmem_wait_ld();
        if (valid) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int l = part * 4 + j;
            if (l < (int)m.levels)
              __stcs(reinterpret_cast<float2*>(m.dX) + (uint64_t)l * m.x_stride + gs,
                     make_float2(v[2 * j], v[2 * j + 1]));
          }
        }
      }
      a_to_smem16(taB, row, c16, bufA[0], bufA[1]);  // G1 -> buffer A (dWc1 has read G4)
      pend = true;  // dWd0 goes behind the next tile's first critical GEMMs
      pend_fresh = fresh;
      fresh = false;
      par ^= 1;
      if (!has_next || nx.f != loaded) {  // every weight-gradient GEMM must land before a flush
        to_mma();
        issue_b([&] { issue_pending(par ^ 1); }, [] {});  // the commit covers all
        pend = false;
        done_b();
      }
      if (!has_next) break;
      if (nx.f != loaded) {
        flush_all(tmem, m.fields[loaded], m.grads, sm.bias_c2);
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        if (m.fields[nx.f].coarse) __trap();
        stage_weights_tc(m.fields[nx.f], m.params, sm.w);
        loaded = nx.f;
        fresh = true;
      }
      mk_relu = n_relu;
      mk_c2 = n_c2;
      mk_clip = n_clip;
      o_fwd = n_o;
      tile = next;
      cur = nx;
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (loaded >= 0) flush_all(tmem, m.fields[loaded], m.grads, sm.bias_c2);
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
  const uint32_t want = (uint32_t)num_sms * MLP_FWD_MINB;
  const unsigned grid = m.n_tiles < want ? m.n_tiles : want;
  k_mlp_fwd_tc<<<grid, NTF, smem, s>>>(m);
}

void launch_mlp_eval_tc(const MlpLaunch& m, int num_sms, cudaStream_t s) {
  if (!m.n_tiles) return;
  static bool attr = false;
  const int smem = (int)sizeof(EvalTcSmem) + 1024;
  if (!attr) {
    cudaFuncSetAttribute(k_mlp_eval_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const uint32_t want = (uint32_t)num_sms * MLP_EVAL_MINB;
  const unsigned grid = m.n_tiles < want ? m.n_tiles : want;
  k_mlp_eval_tc<<<grid, NTF, smem, s>>>(m);
}

void launch_mlp_bwd_tc(const MlpLaunch& m0, int num_sms, cudaStream_t s) {
  if (!m0.n_tiles) return;
  MlpLaunch m = m0;
  if (!m.out_tile) m.out_tile = m.out;  // the forward's outputs by tile row
  static bool attr = false;
  const int smem = (int)sizeof(BwdTcSmem);  // no-swizzle operands need 16-byte alignment only
  if (!attr) {
    cudaFuncSetAttribute(k_mlp_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_mlp_bwd_tc_relu, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  // the leading ReLU-field tiles take the paired kernel (the context's DG_MLP_BWD_SERIAL=1
  // leaves relu_tiles at 0: every tile the serial kernel)
  const uint32_t split = std::min(m.relu_tiles, m.n_tiles);
  auto grid_of = [&](uint32_t n) { return (unsigned)std::min<uint32_t>(n, (uint32_t)num_sms); };
  if (split) k_mlp_bwd_tc_relu<<<grid_of(split), NTB, smem, s>>>(m, 0u, split);
  if (split < m.n_tiles) k_mlp_bwd_tc<<<grid_of(m.n_tiles - split), NTB, smem, s>>>(m, split, m.n_tiles);
}

}  // namespace dg
