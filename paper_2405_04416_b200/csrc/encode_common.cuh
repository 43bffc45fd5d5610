// encode_common.cuh — lattice corners of one hash-grid level and the paired-row gather,
// shared by the encode kernels (kernels_encode.cu) and the occupancy query (kernels_occ.cu).
// HashGrid::encode's per-level inner loop (grid.cpp:107-130).
#pragma once

#include "geometry.cuh"

namespace dg {

struct Corners {
  uint32_t row[8];
  float w[8];
};

// Lattice corners of one level for normalised point p; zero-weight corners get row = NONE
// and are skipped by the callers exactly as the reference skips them (grid.cpp:119-120).
// Lattice indices, fractions and corner weights are fp64 (bit-exact rows; the weight rounds
// once to fp32, features accumulate in fp32); the row arithmetic is hoisted per axis.
__device__ __forceinline__ void level_corners(const LevelDesc& lv, const double p[3], Corners& c) {
  const AxisW ax = lattice_axis(p[0], lv.n[0]);
  const AxisW ay = lattice_axis(p[1], lv.n[1]);
  const AxisW az = lattice_axis(p[2], lv.n[2]);
  const double fx[2] = {dsub(1.0, ax.frac), ax.frac};
  const double fy[2] = {dsub(1.0, ay.frac), ay.frac};
  const double fz[2] = {dsub(1.0, az.frac), az.frac};
  // row = x ^ (y * P1) ^ (z * P2) (hashed) or x + nx (y + ny z) (one-to-one), per axis parts
  uint32_t rx[2], ry[2], rz[2];
  if (lv.hashed) {
    rx[0] = ax.i0;
    rx[1] = ax.i1;
    ry[0] = ay.i0 * 2654435761u;
    ry[1] = ay.i1 * 2654435761u;
    rz[0] = az.i0 * 805459861u;
    rz[1] = az.i1 * 805459861u;
  } else {
    rx[0] = ax.i0;
    rx[1] = ax.i1;
    ry[0] = lv.n[0] * ay.i0;
    ry[1] = lv.n[0] * ay.i1;
    rz[0] = lv.n[0] * lv.n[1] * az.i0;
    rz[1] = lv.n[0] * lv.n[1] * az.i1;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int cx = k & 1, cy = (k >> 1) & 1, cz = (k >> 2) & 1;
    const double w = dmul(dmul(fx[cx], fy[cy]), fz[cz]);
    c.w[k] = (float)w;
    const uint32_t row = lv.hashed ? ((rx[cx] ^ ry[cy] ^ rz[cz]) & lv.mask) : (rx[cx] + ry[cy] + rz[cz]);
    c.row[k] = w == 0.0 ? 0xffffffffu : row;
  }
}

// Per-axis lattice indices and fractions of one level (fp64, bit-exact).
struct LatticeAxes {
  AxisW a[3];
};

__device__ __forceinline__ LatticeAxes lattice_axes(const LevelDesc& lv, const double p[3]) {
  LatticeAxes la;
  la.a[0] = lattice_axis(p[0], lv.n[0]);
  la.a[1] = lattice_axis(p[1], lv.n[1]);
  la.a[2] = lattice_axis(p[2], lv.n[2]);
  return la;
}

// The eight fp32 corner weights of one level from its lattice axes: the fp64 factors rounded
// once, multiplied in fp32 (<= 2 ulp from the rounded fp64 product; a weight only scales the
// upstream gradient, it never feeds a nonlinearity); a corner whose fp64 factor is 0 gets
// weight 0 and is skipped by the callers (grid.cpp:119-120; the fp64 product cannot underflow).
__device__ __forceinline__ void corner_weights_w32(const LatticeAxes& la, float w[8], bool zero[8]) {
  const double fx[2] = {dsub(1.0, la.a[0].frac), la.a[0].frac};
  const double fy[2] = {dsub(1.0, la.a[1].frac), la.a[1].frac};
  const double fz[2] = {dsub(1.0, la.a[2].frac), la.a[2].frac};
  const float gx[2] = {(float)fx[0], (float)fx[1]}, gy[2] = {(float)fy[0], (float)fy[1]};
  const float gz[2] = {(float)fz[0], (float)fz[1]};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int cx = k & 1, cy = (k >> 1) & 1, cz = (k >> 2) & 1;
    w[k] = __fmul_rn(__fmul_rn(gx[cx], gy[cy]), gz[cz]);
    zero[k] = fx[cx] == 0.0 || fy[cy] == 0.0 || fz[cz] == 0.0;
  }
}

// Table row of lattice vertex (ix, iy, iz) of a level (grid.cpp:75-84).
__device__ __forceinline__ uint32_t vertex_row(const LevelDesc& lv, uint32_t ix, uint32_t iy, uint32_t iz) {
  return lv.hashed ? ((ix ^ (iy * 2654435761u) ^ (iz * 805459861u)) & lv.mask)
                   : (ix + lv.n[0] * iy + lv.n[0] * lv.n[1] * iz);
}

// The backward's corners: the same fp64 indices and fractions as level_corners, fp32 weights
// (corner_weights_w32).
__device__ __forceinline__ void corners_w32(const LevelDesc& lv, const LatticeAxes& la, Corners& c) {
  bool zero[8];
  corner_weights_w32(la, c.w, zero);
  const AxisW& ax = la.a[0];
  const AxisW& ay = la.a[1];
  const AxisW& az = la.a[2];
  uint32_t rx[2], ry[2], rz[2];
  if (lv.hashed) {
    rx[0] = ax.i0;
    rx[1] = ax.i1;
    ry[0] = ay.i0 * 2654435761u;
    ry[1] = ay.i1 * 2654435761u;
    rz[0] = az.i0 * 805459861u;
    rz[1] = az.i1 * 805459861u;
  } else {
    rx[0] = ax.i0;
    rx[1] = ax.i1;
    ry[0] = lv.n[0] * ay.i0;
    ry[1] = lv.n[0] * ay.i1;
    rz[0] = lv.n[0] * lv.n[1] * az.i0;
    rz[1] = lv.n[0] * lv.n[1] * az.i1;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int cx = k & 1, cy = (k >> 1) & 1, cz = (k >> 2) & 1;
    const uint32_t row = lv.hashed ? ((rx[cx] ^ ry[cy] ^ rz[cz]) & lv.mask) : (rx[cx] + ry[cy] + rz[cz]);
    c.row[k] = zero[k] ? 0xffffffffu : row;
  }
}

// The training forward's gather of one level (k_encode_fwd) from its lattice axes: fp32 corner
// weights (corner_weights_w32: <= 2 ulp from the reference's rounded fp64 products, i.e.
// ~1e-7 of a feature), the two x-neighbour corners of each (y, z) pair fetched as one aligned
// float4 when their rows share it.  A zero-weight corner contributes 0 * v (the reference skips
// it: identical for finite tables).  SLICED: only rows in [lo, hi) are fetched.
template <bool SLICED>
__device__ __forceinline__ float2 gather_level_w32(const LevelDesc& lv, const LatticeAxes& la,
                                                   const float2* __restrict__ table, uint32_t lo, uint32_t hi) {
  float w[8];
  bool zero[8];
  corner_weights_w32(la, w, zero);
  const uint32_t x0 = la.a[0].i0, x1 = la.a[0].i1;
  uint32_t base[4];
  if (lv.hashed) {
    const uint32_t y0 = la.a[1].i0 * 2654435761u, y1 = la.a[1].i1 * 2654435761u;
    const uint32_t z0 = la.a[2].i0 * 805459861u, z1 = la.a[2].i1 * 805459861u;
    base[0] = y0 ^ z0;
    base[1] = y1 ^ z0;
    base[2] = y0 ^ z1;
    base[3] = y1 ^ z1;
  } else {
    const uint32_t nx = lv.n[0], nxy = lv.n[0] * lv.n[1];
    const uint32_t y0 = nx * la.a[1].i0, y1 = nx * la.a[1].i1, z0 = nxy * la.a[2].i0, z1 = nxy * la.a[2].i1;
    base[0] = y0 + z0;
    base[1] = y1 + z0;
    base[2] = y0 + z1;
    base[3] = y1 + z1;
  }
  const float4* t4 = reinterpret_cast<const float4*>(table);
  float4 q[4];
  float2 b[4];
  uint32_t r0s[4];
  bool pr[4], in0[4], in1[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t r0 = lv.hashed ? ((x0 ^ base[j]) & lv.mask) : x0 + base[j];
    const uint32_t r1 = lv.hashed ? ((x1 ^ base[j]) & lv.mask) : x1 + base[j];
    r0s[j] = r0;
    pr[j] = (r0 ^ r1) == 1u;
    in0[j] = !SLICED || (r0 >= lo && r0 < hi);
    in1[j] = !SLICED || (r1 >= lo && r1 < hi);
    q[j] = in0[j] || (pr[j] && in1[j]) ? __ldg(t4 + (r0 >> 1)) : make_float4(0.f, 0.f, 0.f, 0.f);
    b[j] = !pr[j] && in1[j] ? __ldg(table + r1) : make_float2(0.f, 0.f);
  }
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool odd = r0s[j] & 1u;
    float2 v0 = odd ? make_float2(q[j].z, q[j].w) : make_float2(q[j].x, q[j].y);
    float2 v1 = pr[j] ? (odd ? make_float2(q[j].x, q[j].y) : make_float2(q[j].z, q[j].w)) : b[j];
    const float w0 = (zero[2 * j] || !in0[j]) ? 0.f : w[2 * j];
    const float w1 = (zero[2 * j + 1] || !in1[j]) ? 0.f : w[2 * j + 1];
    acc.x = fmaf(w0, v0.x, acc.x);
    acc.y = fmaf(w0, v0.y, acc.y);
    acc.x = fmaf(w1, v1.x, acc.x);
    acc.y = fmaf(w1, v1.y, acc.y);
  }
  return acc;
}

// One-to-one levels through their paired copy (kernels_pairs.cu: pairs[r] = rows r, r + 1):
// corner pair (x0, x0 + 1) of (y, z) combo j is pairs[x0 + base_j], always one aligned 16-byte
// access.  r0[j] = that pair row (kNoRow when outside the pass's slice [lo, hi)); w[k] = the
// corner weights (0 for a zero-weight corner, as the reference skips it; a clamped x1 == x0
// has weight 0).
constexpr uint32_t kNoRow = 0xffffffffu;
template <bool SLICED>
__device__ __forceinline__ void paired_corners(const LevelDesc& lv, const LatticeAxes& la, uint32_t lo, uint32_t hi,
                                               uint32_t r0[4], float w[8]) {
  bool zero[8];
  corner_weights_w32(la, w, zero);
#pragma unroll
  for (int k = 0; k < 8; ++k) w[k] = zero[k] ? 0.f : w[k];
  const uint32_t nx = lv.n[0], nxy = lv.n[0] * lv.n[1];
  const uint32_t y0 = nx * la.a[1].i0, y1 = nx * la.a[1].i1, z0 = nxy * la.a[2].i0, z1 = nxy * la.a[2].i1;
  const uint32_t base[4] = {y0 + z0, y1 + z0, y0 + z1, y1 + z1};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t r = la.a[0].i0 + base[j];
    r0[j] = (!SLICED || (r >= lo && r < hi)) ? r : kNoRow;
  }
}

template <bool SLICED>
__device__ __forceinline__ float2 gather_level_paired(const LevelDesc& lv, const LatticeAxes& la,
                                                      const float4* __restrict__ pairs, uint32_t lo, uint32_t hi) {
  uint32_t r0[4];
  float w[8];
  paired_corners<SLICED>(lv, la, lo, hi, r0, w);
  float4 q[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) q[j] = r0[j] != kNoRow ? __ldg(pairs + r0[j]) : make_float4(0.f, 0.f, 0.f, 0.f);
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    acc.x = fmaf(w[2 * j], q[j].x, acc.x);
    acc.y = fmaf(w[2 * j], q[j].y, acc.y);
    acc.x = fmaf(w[2 * j + 1], q[j].z, acc.x);
    acc.y = fmaf(w[2 * j + 1], q[j].w, acc.y);
  }
  return acc;
}

// Row pairing: the two x-neighbour corners (cx = 0, 1) of each (cy, cz) land in rows
// i ^ h and (i + 1) ^ h (hashed) or r and r + 1 (one-to-one); when those differ only in bit 0
// (half the time) they are one 16-byte aligned float4 (every level table is 16-byte aligned),
// fetched or reduced with one vector access instead of two.
__device__ __forceinline__ bool is_pair(uint32_t r0, uint32_t r1) {
  return r0 != 0xffffffffu && r1 != 0xffffffffu && (r0 ^ r1) == 1u;
}

__device__ __forceinline__ float2 gather_level_pairs(const float2* __restrict__ table, const Corners& c) {
  const float4* t4 = reinterpret_cast<const float4*>(table);
  float4 q[4];
  float2 b[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t r0 = c.row[2 * j], r1 = c.row[2 * j + 1];
    if (is_pair(r0, r1)) {
      q[j] = __ldg(t4 + (r0 >> 1));
      b[j] = make_float2(0.f, 0.f);
    } else {
      const float2 a = r0 != 0xffffffffu ? __ldg(table + r0) : make_float2(0.f, 0.f);
      q[j] = make_float4(a.x, a.y, 0.f, 0.f);
      b[j] = r1 != 0xffffffffu ? __ldg(table + r1) : make_float2(0.f, 0.f);
    }
  }
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t r0 = c.row[2 * j], r1 = c.row[2 * j + 1];
    float2 v0, v1;
    if (is_pair(r0, r1)) {
      const bool odd = r0 & 1u;
      v0 = odd ? make_float2(q[j].z, q[j].w) : make_float2(q[j].x, q[j].y);
      v1 = odd ? make_float2(q[j].x, q[j].y) : make_float2(q[j].z, q[j].w);
    } else {
      v0 = make_float2(q[j].x, q[j].y);
      v1 = b[j];
    }
    acc.x = fmaf(c.w[2 * j], v0.x, acc.x);
    acc.y = fmaf(c.w[2 * j], v0.y, acc.y);
    acc.x = fmaf(c.w[2 * j + 1], v1.x, acc.x);
    acc.y = fmaf(c.w[2 * j + 1], v1.y, acc.y);
  }
  return acc;
}

}  // namespace dg
