// kernels_mlp.cu — stage 4: the fused density + colour MLP, forward and backward.
//
//   forward   query_density + query_color (field.cpp:230-288; mlp.cpp:55-82; sh.hpp:14-35):
//             encode[32] -> 64 ReLU -> 16 (clip 15, sigma = exp(raw0)) ;
//             [raw1..15 | SH16(dir) | appearance] -> 64 act -> 64 act -> 3 (clip, sigmoid)
//   backward  field_backward (field.cpp:290-327; mlp.cpp:84-138): recomputes the forward of a
//             sample tile from the cached encoding, back-propagates, accumulates every weight
//             and bias gradient in registers across the CTA's tiles (one flush of atomics per
//             CTA and field) and writes d(encoding) for the hash-grid backward.
//
// Layout: a tile is TILE samples of ONE field (partition x cascade).  Activations live in
// shared memory feature-major ([feature][sample], row stride TILE + 4); each layer is a
// register-blocked FFMA GEMM (micro-tile MM outputs x MS samples per thread).  Weights are
// staged once per field in both orientations.  fp32 throughout (plain TF32 misses
// the 1e-4 bar).
#include "dg_common.cuh"
#include "kernels.h"

namespace dg {

namespace {

constexpr int NT = 256;

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// Shared weights in "k-major" form for y[m] = sum_k W(k, m) x[k]:
//   forward uses W^T ([in][out]), the input-gradient GEMMs use W ([out][in]).
struct WeightsT {  // forward (transposed), padded
  float d0[kEnc * kHidden];      // [32][64]
  float d1[kHidden * kDensOut];  // [64][16]
  float c0[kColorIn * kHidden];  // [48][64]
  float c1[kHidden * kHidden];   // [64][64]
  float c2[kHidden * 4];         // [64][4]
  float bd0[kHidden], bd1[kDensOut], bc0[kHidden], bc1[kHidden], bc2[4];
};
struct WeightsN {  // backward (natural [out][in]), padded
  float d0[kHidden * kEnc];      // [64][32]
  float d1[kDensOut * kHidden];  // [16][64]
  float c0[kHidden * kColorIn];  // [64][48]
  float c1[kHidden * kHidden];   // [64][64]
  float c2[4 * kHidden];         // [4][64]
};

__device__ __forceinline__ float relu(float x) { return x > 0.f ? x : 0.f; }
__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + expf(-x)); }

// Stage one field's weights into shared memory (zero padding in the unused rows/cols).
__device__ void load_weights(const FieldDesc& fd, const float* __restrict__ params, WeightsT& wt,
                             WeightsN* wn) {
  const float* base = params + fd.base;
  const int enc = (int)fd.L * 2;
  const int cin = 31 + (int)fd.app_dim;
  for (int e = threadIdx.x; e < kEnc * kHidden; e += NT) {
    const int i = e / kHidden, o = e % kHidden;  // wt.d0[i][o]
    const float v = i < enc ? base[fd.dw0 + o * enc + i] : 0.f;
    wt.d0[e] = v;
    if (wn) wn->d0[o * kEnc + i] = v;
  }
  for (int e = threadIdx.x; e < kHidden * kDensOut; e += NT) {
    const int i = e / kDensOut, o = e % kDensOut;
    const float v = base[fd.dw1 + o * kHidden + i];
    wt.d1[e] = v;
    if (wn) wn->d1[o * kHidden + i] = v;
  }
  for (int e = threadIdx.x; e < kColorIn * kHidden; e += NT) {
    const int i = e / kHidden, o = e % kHidden;
    const float v = i < cin ? base[fd.cw0 + o * cin + i] : 0.f;
    wt.c0[e] = v;
    if (wn) wn->c0[o * kColorIn + i] = v;
  }
  for (int e = threadIdx.x; e < kHidden * kHidden; e += NT) {
    const int i = e / kHidden, o = e % kHidden;
    const float v = base[fd.cw1 + o * kHidden + i];
    wt.c1[e] = v;
    if (wn) wn->c1[o * kHidden + i] = v;
  }
  for (int e = threadIdx.x; e < kHidden * 4; e += NT) {
    const int i = e / 4, o = e % 4;
    const float v = o < 3 ? base[fd.cw2 + o * kHidden + i] : 0.f;
    wt.c2[e] = v;
    if (wn) wn->c2[o * kHidden + i] = v;
  }
  for (int e = threadIdx.x; e < kHidden; e += NT) {
    wt.bd0[e] = base[fd.db0 + e];
    wt.bc0[e] = base[fd.cb0 + e];
    wt.bc1[e] = base[fd.cb1 + e];
  }
  for (int e = threadIdx.x; e < kDensOut; e += NT) wt.bd1[e] = base[fd.db1 + e];
  for (int e = threadIdx.x; e < 4; e += NT) wt.bc2[e] = e < 3 ? base[fd.cb2 + e] : 0.f;
}

enum Act { ACT_NONE = 0, ACT_RELU = 1, ACT_SIGMOID = 2 };

// y[m][s] = act(bias[m] + sum_k W[k*ldw + m] * x[k][s]) for m < M, s < TILE.
template <int TILE, int M, int K, int MM, int MS>
__device__ __forceinline__ void gemm_layer(const float* __restrict__ W, int ldw,
                                           const float* __restrict__ bias,
                                           const float* __restrict__ x, float* __restrict__ y,
                                           int act) {
  constexpr int LD = TILE + 4;
  constexpr int NG = M / MM;
  constexpr int NS = TILE / MS;
  static_assert(NG * NS <= NT, "micro-tiling exceeds the CTA");
  const int tid = threadIdx.x;
  if (tid >= NG * NS) return;
  const int mg = tid % NG, sg = tid / NG;
  float acc[MM][MS];
#pragma unroll
  for (int j = 0; j < MM; ++j) {
    const float b = bias ? bias[mg * MM + j] : 0.f;
#pragma unroll
    for (int s = 0; s < MS; ++s) acc[j][s] = b;
  }
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    float w[MM], v[MS];
    if constexpr (MM % 4 == 0) {
#pragma unroll
      for (int j = 0; j < MM; j += 4) {
        const float4 t = *reinterpret_cast<const float4*>(W + k * ldw + mg * MM + j);
        w[j] = t.x; w[j + 1] = t.y; w[j + 2] = t.z; w[j + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < MM; ++j) w[j] = W[k * ldw + mg * MM + j];
    }
    if constexpr (MS % 4 == 0) {
#pragma unroll
      for (int s = 0; s < MS; s += 4) {
        const float4 t = *reinterpret_cast<const float4*>(x + k * LD + sg * MS + s);
        v[s] = t.x; v[s + 1] = t.y; v[s + 2] = t.z; v[s + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int s = 0; s < MS; ++s) v[s] = x[k * LD + sg * MS + s];
    }
#pragma unroll
    for (int j = 0; j < MM; ++j)
#pragma unroll
      for (int s = 0; s < MS; ++s) acc[j][s] = fmaf(w[j], v[s], acc[j][s]);
  }
#pragma unroll
  for (int j = 0; j < MM; ++j)
#pragma unroll
    for (int s = 0; s < MS; ++s) {
      float a = acc[j][s];
      if (act == ACT_RELU) a = relu(a);
      else if (act == ACT_SIGMOID) a = sigm(a);
      y[(mg * MM + j) * LD + sg * MS + s] = a;
    }
}

// Input gradient with the activation derivative taken from the stored post-activation:
// g_out[m][s] = (sum_k W[k*ldw+m] g_in[k][s]) * act'(post[m][s]); in place over post allowed.
template <int TILE, int M, int K, int MM, int MS>
__device__ __forceinline__ void gemm_back(const float* __restrict__ W, int ldw,
                                          const float* __restrict__ g_in, float* post_then_grad,
                                          int act) {
  constexpr int LD = TILE + 4;
  constexpr int NG = M / MM;
  constexpr int NS = TILE / MS;
  static_assert(NG * NS <= NT, "micro-tiling exceeds the CTA");
  const int tid = threadIdx.x;
  if (tid >= NG * NS) return;
  const int mg = tid % NG, sg = tid / NG;
  float acc[MM][MS];
#pragma unroll
  for (int j = 0; j < MM; ++j)
#pragma unroll
    for (int s = 0; s < MS; ++s) acc[j][s] = 0.f;
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    float w[MM], v[MS];
#pragma unroll
    for (int j = 0; j < MM; ++j) w[j] = W[k * ldw + mg * MM + j];
#pragma unroll
    for (int s = 0; s < MS; ++s) v[s] = g_in[k * LD + sg * MS + s];
#pragma unroll
    for (int j = 0; j < MM; ++j)
#pragma unroll
      for (int s = 0; s < MS; ++s) acc[j][s] = fmaf(w[j], v[s], acc[j][s]);
  }
#pragma unroll
  for (int j = 0; j < MM; ++j)
#pragma unroll
    for (int s = 0; s < MS; ++s) {
      float* p = post_then_grad + (mg * MM + j) * LD + sg * MS + s;
      float d = 1.f;
      if (act == ACT_RELU) d = *p > 0.f ? 1.f : 0.f;
      else if (act == ACT_SIGMOID) d = *p * (1.f - *p);
      *p = acc[j][s] * d;
    }
}

// Weight-gradient accumulation: acc[j][i] += sum_s g[(og*MO+j)][s] * a[(ig*MI+i)][s].
template <int TILE, int OUT, int IN, int MO, int MI>
__device__ __forceinline__ void wgrad(const float* __restrict__ g, const float* __restrict__ a,
                                      float (&acc)[MO][MI]) {
  constexpr int LD = TILE + 4;
  constexpr int NI = IN / MI;
  constexpr int NO = OUT / MO;
  static_assert(NI * NO <= NT, "wgrad tiling exceeds the CTA");
  const int tid = threadIdx.x;
  if (tid >= NI * NO) return;
  const int ig = tid % NI, og = tid / NI;
#pragma unroll 2
  for (int s = 0; s < TILE; s += 4) {
    float4 gv[MO], av[MI];
#pragma unroll
    for (int j = 0; j < MO; ++j) gv[j] = *reinterpret_cast<const float4*>(g + (og * MO + j) * LD + s);
#pragma unroll
    for (int i = 0; i < MI; ++i) av[i] = *reinterpret_cast<const float4*>(a + (ig * MI + i) * LD + s);
#pragma unroll
    for (int j = 0; j < MO; ++j)
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        acc[j][i] = fmaf(gv[j].x, av[i].x, acc[j][i]);
        acc[j][i] = fmaf(gv[j].y, av[i].y, acc[j][i]);
        acc[j][i] = fmaf(gv[j].z, av[i].z, acc[j][i]);
        acc[j][i] = fmaf(gv[j].w, av[i].w, acc[j][i]);
      }
  }
}

template <int TILE, int OUT, int IN, int MO, int MI>
__device__ __forceinline__ void wgrad_flush(float (&acc)[MO][MI], float* __restrict__ dst, int ld,
                                            int rows, int cols) {
  constexpr int NI = IN / MI;
  constexpr int NO = OUT / MO;
  const int tid = threadIdx.x;
  if (tid >= NI * NO) return;
  const int ig = tid % NI, og = tid / NI;
#pragma unroll
  for (int j = 0; j < MO; ++j)
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int o = og * MO + j, c = ig * MI + i;
      if (o < rows && c < cols && acc[j][i] != 0.f) atomicAdd(dst + o * ld + c, acc[j][i]);
      acc[j][i] = 0.f;
    }
}

// SH basis (sh.hpp:14-35) in fp32.
__device__ __forceinline__ void sh16(float x, float y, float z, float* o) {
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

__device__ __forceinline__ int field_of_tile(const MlpLaunch& m, uint32_t tile) {
  int f = 0;
  while (f + 1 < (int)m.n_fields && tile >= m.tile_off[f + 1]) ++f;
  return f;
}

__device__ __forceinline__ float clip15(float v, bool& clipped) {
  clipped = v > 15.f || v < -15.f;
  return v > 15.f ? 15.f : (v < -15.f ? -15.f : v);
}

// Load a tile's encodings (level-major float2 rows in global) into x[32][LD]; zero-pad.
template <int TILE>
__device__ __forceinline__ void load_x(const MlpLaunch& m, uint64_t s0, int count,
                                       float* __restrict__ x) {
  constexpr int LD = TILE + 4;
  for (int e = threadIdx.x; e < TILE * 16; e += NT) {
    const int l = e / TILE, s = e % TILE;
    float2 v = make_float2(0.f, 0.f);
    if (s < count && l < (int)m.levels)
      v = reinterpret_cast<const float2*>(m.X)[(uint64_t)l * m.x_stride + s0 + s];
    x[(2 * l) * LD + s] = v.x;
    x[(2 * l + 1) * LD + s] = v.y;
  }
}

// Colour-input rows [0..14] = clipped raw[1..15] (shifted in place), [15..30] SH, [31..] app,
// padded with zeros to 48.  Returns the clipped raw0 per sample in sig_raw and clip masks.
template <int TILE>
__device__ __forceinline__ void build_color_input(const MlpLaunch& m, const FieldDesc& fd,
                                                  uint64_t s0, int count, float* __restrict__ buf,
                                                  float* __restrict__ sig_raw,
                                                  uint32_t* __restrict__ dmask) {
  constexpr int LD = TILE + 4;
  for (int s = threadIdx.x; s < TILE; s += NT) {
    bool c0;
    sig_raw[s] = clip15(buf[s], c0);
    uint32_t mask = c0 ? 1u : 0u;
    for (int r = 0; r < 15; ++r) {
      bool c;
      buf[r * LD + s] = clip15(buf[(r + 1) * LD + s], c);
      mask |= (c ? 1u : 0u) << (r + 1);
    }
    dmask[s] = mask;
    float sh[16];
    const float* app = nullptr;
    if (s < count) {
      const uint64_t gs = s0 + s;
      const RayRec& r = m.rec[m.s_item[gs]];
      sh16((float)r.d[0], (float)r.d[1], (float)r.d[2], sh);
      app = m.app_per_sample ? m.app_override + gs * fd.app_dim
                             : (m.app_override ? m.app_override : m.app_table + (uint64_t)r.img * fd.app_dim);
    } else {
      for (int k = 0; k < 16; ++k) sh[k] = 0.f;
    }
    for (int k = 0; k < 16; ++k) buf[(15 + k) * LD + s] = sh[k];
    for (int k = 0; k < kColorIn - 31; ++k)
      buf[(31 + k) * LD + s] = (app && k < (int)fd.app_dim) ? app[k] : 0.f;
  }
}

// ------------------------------------------------------------------ forward
constexpr int FT = 128;  // samples per forward tile
constexpr int FLD = FT + 4;

struct FwdSmem {
  WeightsT w;
  float a[kHidden * FLD];
  float b[kHidden * FLD];
  float sig_raw[FT];
  uint32_t dmask[FT];
};

__global__ void __launch_bounds__(NT, 2) k_mlp_fwd(MlpLaunch m) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(smem_raw);
  int loaded = -1;
  for (uint32_t tile = blockIdx.x; tile < m.n_tiles; tile += gridDim.x) {
    const int f = field_of_tile(m, tile);
    const FieldDesc& fd = m.fields[f];
    const uint64_t s0 = m.field_off[f] + (uint64_t)(tile - m.tile_off[f]) * FT;
    const int count = (int)umin64(FT, m.field_off[f + 1] - s0);
    if (f != loaded) {
      __syncthreads();
      load_weights(fd, m.params, sm.w, nullptr);
      loaded = f;
    }
    load_x<FT>(m, s0, count, sm.a);
    __syncthreads();
    gemm_layer<FT, kHidden, kEnc, 4, 8>(sm.w.d0, kHidden, sm.w.bd0, sm.a, sm.b, ACT_RELU);
    __syncthreads();
    gemm_layer<FT, kDensOut, kHidden, 4, 2>(sm.w.d1, kDensOut, sm.w.bd1, sm.b, sm.a, ACT_NONE);
    __syncthreads();
    build_color_input<FT>(m, fd, s0, count, sm.a, sm.sig_raw, sm.dmask);
    __syncthreads();
    const int cact = fd.coarse ? ACT_SIGMOID : ACT_RELU;
    gemm_layer<FT, kHidden, kColorIn, 4, 8>(sm.w.c0, kHidden, sm.w.bc0, sm.a, sm.b, cact);
    __syncthreads();
    gemm_layer<FT, kHidden, kHidden, 4, 8>(sm.w.c1, kHidden, sm.w.bc1, sm.b, sm.a, cact);
    __syncthreads();
    gemm_layer<FT, 4, kHidden, 4, 1>(sm.w.c2, 4, sm.w.bc2, sm.a, sm.b, ACT_NONE);
    __syncthreads();
    for (int s = threadIdx.x; s < count; s += NT) {
      bool c;
      const float r = sigm(clip15(sm.b[0 * FLD + s], c));
      const float g = sigm(clip15(sm.b[1 * FLD + s], c));
      const float b = sigm(clip15(sm.b[2 * FLD + s], c));
      m.out[m.perm ? m.perm[s0 + s] : s0 + s] = make_float4(expf(sm.sig_raw[s]), r, g, b);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ backward
constexpr int BT = 64;  // samples per backward tile
constexpr int BLD = BT + 4;

struct BwdSmem {
  WeightsT w;
  WeightsN wn;
  float x[kEnc * BLD];        // encoding -> (reused as dX staging)
  float h1[kHidden * BLD];    // density hidden post-act -> its gradient
  float cin[kColorIn * BLD];  // colour input -> rows 0..15 reused for the 16 density-raw grads
  float c1[kHidden * BLD];    // colour hidden 1 post-act -> gradient
  float c2[kHidden * BLD];    // colour hidden 2 post-act -> gradient
  float g3[4 * BLD];          // colour raw grads / colour raw
  float sig_raw[BT];
  uint32_t dmask[BT];
};

struct GradRegs {
  float c2[1][1];  // [4][64]
  float c1[4][4];  // [64][64]
  float c0[4][3];  // [64][48]
  float d1[1][4];  // [16][64]
  float d0[4][2];  // [64][32]
  float bias;      // tid < 212
};

__device__ __forceinline__ void zero_regs(GradRegs& g) {
  g.c2[0][0] = 0.f;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) g.c1[j][i] = 0.f;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 3; ++i) g.c0[j][i] = 0.f;
  for (int i = 0; i < 4; ++i) g.d1[0][i] = 0.f;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 2; ++i) g.d0[j][i] = 0.f;
  g.bias = 0.f;
}

__device__ void flush_grads(GradRegs& g, const FieldDesc& fd, float* __restrict__ grads) {
  float* base = grads + fd.base;
  const int enc = (int)fd.L * 2;
  const int cin = 31 + (int)fd.app_dim;
  wgrad_flush<BT, 4, kHidden, 1, 1>(g.c2, base + fd.cw2, kHidden, 3, kHidden);
  wgrad_flush<BT, kHidden, kHidden, 4, 4>(g.c1, base + fd.cw1, kHidden, kHidden, kHidden);
  wgrad_flush<BT, kHidden, kColorIn, 4, 3>(g.c0, base + fd.cw0, cin, kHidden, cin);
  wgrad_flush<BT, kDensOut, kHidden, 1, 4>(g.d1, base + fd.dw1, kHidden, kDensOut, kHidden);
  wgrad_flush<BT, kHidden, kEnc, 4, 2>(g.d0, base + fd.dw0, enc, kHidden, enc);
  const int tid = threadIdx.x;
  if (g.bias != 0.f) {
    if (tid < 64) atomicAdd(base + fd.cb0 + tid, g.bias);
    else if (tid < 128) atomicAdd(base + fd.cb1 + (tid - 64), g.bias);
    else if (tid < 131) atomicAdd(base + fd.cb2 + (tid - 128), g.bias);
    else if (tid < 195) atomicAdd(base + fd.db0 + (tid - 131), g.bias);
    else if (tid < 211) atomicAdd(base + fd.db1 + (tid - 195), g.bias);
  }
  g.bias = 0.f;
}

__device__ __forceinline__ float row_sum(const float* r, int count) {
  float a = 0.f;
  for (int s = 0; s < count; ++s) a += r[s];
  return a;
}

__global__ void __launch_bounds__(NT, 1) k_mlp_bwd(MlpLaunch m) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
  GradRegs gr;
  zero_regs(gr);
  // contiguous tile range per CTA so field changes (flushes) are rare
  const uint32_t per = (m.n_tiles + gridDim.x - 1) / gridDim.x;
  const uint32_t t_begin = blockIdx.x * per;
  const uint32_t t_end = min(m.n_tiles, t_begin + per);
  int loaded = -1;
  const int tid = threadIdx.x;
  for (uint32_t tile = t_begin; tile < t_end; ++tile) {
    const int f = field_of_tile(m, tile);
    const FieldDesc& fd = m.fields[f];
    const uint64_t s0 = m.field_off[f] + (uint64_t)(tile - m.tile_off[f]) * BT;
    const int count = (int)umin64(BT, m.field_off[f + 1] - s0);
    if (f != loaded) {
      if (loaded >= 0) flush_grads(gr, m.fields[loaded], m.grads);
      __syncthreads();
      load_weights(fd, m.params, sm.w, &sm.wn);
      loaded = f;
    }
    const int cact = fd.coarse ? ACT_SIGMOID : ACT_RELU;
    // ---- forward recompute ----
    load_x<BT>(m, s0, count, sm.x);
    __syncthreads();
    gemm_layer<BT, kHidden, kEnc, 4, 4>(sm.w.d0, kHidden, sm.w.bd0, sm.x, sm.h1, ACT_RELU);
    __syncthreads();
    gemm_layer<BT, kDensOut, kHidden, 4, 1>(sm.w.d1, kDensOut, sm.w.bd1, sm.h1, sm.cin, ACT_NONE);
    __syncthreads();
    build_color_input<BT>(m, fd, s0, count, sm.cin, sm.sig_raw, sm.dmask);
    __syncthreads();
    gemm_layer<BT, kHidden, kColorIn, 4, 4>(sm.w.c0, kHidden, sm.w.bc0, sm.cin, sm.c1, cact);
    __syncthreads();
    gemm_layer<BT, kHidden, kHidden, 4, 4>(sm.w.c1, kHidden, sm.w.bc1, sm.c1, sm.c2, cact);
    __syncthreads();
    gemm_layer<BT, 4, kHidden, 4, 1>(sm.w.c2, 4, sm.w.bc2, sm.c2, sm.g3, ACT_NONE);
    __syncthreads();
    // ---- colour head: d raw = clipped ? 0 : drgb * s (1 - s) (field.cpp:298-306) ----
    for (int s = tid; s < BT; s += NT) {
      float4 up = s < count ? m.grad_in[s0 + s] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float ug[3] = {up.y, up.z, up.w};
      for (int k = 0; k < 3; ++k) {
        bool c;
        const float sg = sigm(clip15(sm.g3[k * BLD + s], c));
        sm.g3[k * BLD + s] = c ? 0.f : ug[k] * sg * (1.f - sg);
      }
      sm.g3[3 * BLD + s] = 0.f;
      // density raw0 gradient: clipped ? 0 : dsigma * sigma (field.cpp:313)
      sm.sig_raw[s] = (sm.dmask[s] & 1u) ? 0.f : up.x * expf(sm.sig_raw[s]);
    }
    __syncthreads();
    // layer c2 (64 -> 3)
    wgrad<BT, 4, kHidden, 1, 1>(sm.g3, sm.c2, gr.c2);
    if (tid >= 128 && tid < 131) gr.bias += row_sum(sm.g3 + (tid - 128) * BLD, BT);
    __syncthreads();
    gemm_back<BT, kHidden, 4, 4, 4>(sm.wn.c2, kHidden, sm.g3, sm.c2, cact);
    __syncthreads();
    // layer c1 (64 -> 64)
    wgrad<BT, kHidden, kHidden, 4, 4>(sm.c2, sm.c1, gr.c1);
    if (tid >= 64 && tid < 128) gr.bias += row_sum(sm.c2 + (tid - 64) * BLD, BT);
    __syncthreads();
    gemm_back<BT, kHidden, kHidden, 4, 4>(sm.wn.c1, kHidden, sm.c2, sm.c1, cact);
    __syncthreads();
    // layer c0 (48 -> 64)
    wgrad<BT, kHidden, kColorIn, 4, 3>(sm.c1, sm.cin, gr.c0);
    if (tid < 64) gr.bias += row_sum(sm.c1 + tid * BLD, BT);
    __syncthreads();
    // colour-input grads for the 15 density features -> cin rows 1..15 hold the density-raw
    // gradient; row 0 gets the sigma path (field.cpp:311-315)
    gemm_back<BT, 16, kHidden, 4, 1>(sm.wn.c0, kColorIn, sm.c1, sm.cin, ACT_NONE);
    __syncthreads();
    for (int s = tid; s < BT; s += NT) {
      const uint32_t mask = sm.dmask[s];
      for (int r = 15; r >= 1; --r)
        sm.cin[r * BLD + s] = ((mask >> r) & 1u) ? 0.f : sm.cin[(r - 1) * BLD + s];
      sm.cin[s] = sm.sig_raw[s];
    }
    __syncthreads();
    // layer d1 (64 -> 16)
    wgrad<BT, kDensOut, kHidden, 1, 4>(sm.cin, sm.h1, gr.d1);
    if (tid >= 195 && tid < 211) gr.bias += row_sum(sm.cin + (tid - 195) * BLD, BT);
    __syncthreads();
    gemm_back<BT, kHidden, kDensOut, 4, 4>(sm.wn.d1, kHidden, sm.cin, sm.h1, ACT_RELU);
    __syncthreads();
    // layer d0 (32 -> 64)
    wgrad<BT, kHidden, kEnc, 4, 2>(sm.h1, sm.x, gr.d0);
    if (tid >= 131 && tid < 195) gr.bias += row_sum(sm.h1 + (tid - 131) * BLD, BT);
    __syncthreads();
    gemm_back<BT, kEnc, kHidden, 4, 2>(sm.wn.d0, kEnc, sm.h1, sm.x, ACT_NONE);
    __syncthreads();
    for (int e = tid; e < BT * 16; e += NT) {
      const int l = e / BT, s = e % BT;
      if (s < count && l < (int)m.levels)
        reinterpret_cast<float2*>(m.dX)[(uint64_t)l * m.x_stride + s0 + s] =
            make_float2(sm.x[(2 * l) * BLD + s], sm.x[(2 * l + 1) * BLD + s]);
    }
    __syncthreads();
  }
  if (loaded >= 0) flush_grads(gr, m.fields[loaded], m.grads);
}

}  // namespace

void launch_mlp_fwd(const MlpLaunch& m, cudaStream_t s) {
  if (!m.n_tiles) return;
  static bool attr = false;
  const int smem = (int)sizeof(FwdSmem);
  if (!attr) {
    cudaFuncSetAttribute(k_mlp_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(m.n_tiles < (uint32_t)sms * 2 ? m.n_tiles : (uint32_t)sms * 2);
  k_mlp_fwd<<<grid, NT, smem, s>>>(m);
}

void launch_mlp_bwd(const MlpLaunch& m, int num_sms, cudaStream_t s) {
  if (!m.n_tiles) return;
  static bool attr = false;
  const int smem = (int)sizeof(BwdSmem);
  if (!attr) {
    cudaFuncSetAttribute(k_mlp_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const unsigned grid = (unsigned)(m.n_tiles < (uint32_t)num_sms ? m.n_tiles : (uint32_t)num_sms);
  k_mlp_bwd<<<grid, NT, smem, s>>>(m);
}

}  // namespace dg
