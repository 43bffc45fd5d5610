// kernels_encode.cu — stage 3: multi-resolution hash-grid encode forward and backward.
//
//   k_encode_fwd   HashGrid::encode (grid.cpp:107-130) on the march samples; one thread per
//                  (level, sample), a warp = 32 consecutive samples (mostly one ray) of one
//                  level, each lane with its 8 corner gathers in flight at once (float2
//                  rows, F = 2).  Position, lattice indices and corner weights are fp64 and
//                  bit-exact (geometry.cuh); features accumulate in fp32.
//   k_encode_bwd   HashGrid::encode_backward (grid.cpp:132-157): the same corners receive
//                  w * upstream through vector float2 atomics (red.global.add.v2.f32).
//
// Features and their gradients are level-major: X[l][s] (float2), l < L, s < n_total.
//
// Algorithmic traffic: 8 corners x L levels x 8 B = 1024 B/sample gathered
// forward; the backward read-modify-writes the same 1024 B.
#include "geometry.cuh"
#include "kernels.h"

namespace dg {

namespace {

struct Corners {
  uint32_t row[8];
  float w[8];
};

// Lattice corners of one level for normalised point p; zero-weight corners get w = 0 and
// are skipped by the callers exactly as the reference skips them (grid.cpp:119-120).
__device__ __forceinline__ void level_corners(const LevelDesc& lv, const double p[3], Corners& c) {
  const AxisW ax = lattice_axis(p[0], lv.n[0]);
  const AxisW ay = lattice_axis(p[1], lv.n[1]);
  const AxisW az = lattice_axis(p[2], lv.n[2]);
  const double fx[2] = {dsub(1.0, ax.frac), ax.frac};
  const double fy[2] = {dsub(1.0, ay.frac), ay.frac};
  const double fz[2] = {dsub(1.0, az.frac), az.frac};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int cx = k & 1, cy = (k >> 1) & 1, cz = (k >> 2) & 1;
    const double w = dmul(dmul(fx[cx], fy[cy]), fz[cz]);
    c.w[k] = (float)w;
    c.row[k] = w == 0.0 ? 0xffffffffu
                        : table_row(lv, cx ? ax.i1 : ax.i0, cy ? ay.i1 : ay.i0, cz ? az.i1 : az.i0);
  }
}

__device__ __forceinline__ float2 gather_level(const float2* __restrict__ table, const Corners& c) {
  float2 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    v[k] = c.row[k] != 0xffffffffu ? __ldg(table + c.row[k]) : make_float2(0.f, 0.f);
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    acc.x = fmaf(c.w[k], v[k].x, acc.x);
    acc.y = fmaf(c.w[k], v[k].y, acc.y);
  }
  return acc;
}

__device__ __forceinline__ void scatter_level(float2* __restrict__ table, const Corners& c, float2 up) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (c.row[k] == 0xffffffffu) continue;
    atomicAdd(table + c.row[k], make_float2(c.w[k] * up.x, c.w[k] * up.y));
  }
}

// Level-major launch: grid (sample chunks, levels).  CTAs are dispatched roughly in blockIdx
// order, so the device works through one level's table at a time: a dense level (<= 2^24
// rows) or one hashed 2^24-row table (128 MiB) is the live working set, which keeps the L2
// hit rate high instead of streaming every level's random rows from HBM at once.  Features
// are stored level-major too (X[l][s] float2), so every store is coalesced.
__global__ void __launch_bounds__(256) k_encode_fwd(FieldLaunch f, float* __restrict__ X) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t l = blockIdx.y;
  if (s >= f.n_total) return;
  const uint32_t casc = s >= f.fine_total ? 1u : 0u;
  const uint32_t item = f.s_item[s];
  const FieldDesc& fd = f.fields[casc * f.n_local + f.item_part[item]];
  const RayRec& r = f.rec[item];
  double p[3];
  normalized_point(fd.box_lo, fd.box_hi, r.o, r.d, f.s_t[s], p);
  Corners c;
  level_corners(fd.lv[l], p, c);
  const float2 acc = gather_level(reinterpret_cast<const float2*>(f.params + fd.base + fd.lv[l].offset), c);
  reinterpret_cast<float2*>(X)[(uint64_t)l * f.n_total + s] = acc;
}

__global__ void __launch_bounds__(256) k_encode_bwd(FieldLaunch f, const float* __restrict__ dX) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t l = blockIdx.y;
  if (s >= f.n_total) return;
  const float2 up = reinterpret_cast<const float2*>(dX)[(uint64_t)l * f.n_total + s];
  if (up.x == 0.f && up.y == 0.f) return;
  const uint32_t casc = s >= f.fine_total ? 1u : 0u;
  const uint32_t item = f.s_item[s];
  const FieldDesc& fd = f.fields[casc * f.n_local + f.item_part[item]];
  const RayRec& r = f.rec[item];
  double p[3];
  normalized_point(fd.box_lo, fd.box_hi, r.o, r.d, f.s_t[s], p);
  Corners c;
  level_corners(fd.lv[l], p, c);
  scatter_level(reinterpret_cast<float2*>(f.grads + fd.base + fd.lv[l].offset), c, up);
}

__global__ void k_encode_points(const FieldDesc* __restrict__ field, const float* __restrict__ params,
                                const double* __restrict__ pts, uint64_t n, float* __restrict__ X,
                                uint32_t* __restrict__ rows) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t l = blockIdx.y;
  if (s >= n) return;
  const FieldDesc& fd = *field;
  const double p[3] = {pts[3 * s], pts[3 * s + 1], pts[3 * s + 2]};
  Corners c;
  level_corners(fd.lv[l], p, c);
  if (rows)
    for (int k = 0; k < 8; ++k) rows[(s * fd.L + l) * 8 + k] = c.row[k];
  reinterpret_cast<float2*>(X)[(uint64_t)l * n + s] =
      gather_level(reinterpret_cast<const float2*>(params + fd.base + fd.lv[l].offset), c);
}

__global__ void k_encode_points_bwd(const FieldDesc* __restrict__ field, float* __restrict__ grads,
                                    const double* __restrict__ pts, const float* __restrict__ dX,
                                    uint64_t n) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t l = blockIdx.y;
  if (s >= n) return;
  const FieldDesc& fd = *field;
  const float2 up = reinterpret_cast<const float2*>(dX)[(uint64_t)l * n + s];
  if (up.x == 0.f && up.y == 0.f) return;
  const double p[3] = {pts[3 * s], pts[3 * s + 1], pts[3 * s + 2]};
  Corners c;
  level_corners(fd.lv[l], p, c);
  scatter_level(reinterpret_cast<float2*>(grads + fd.base + fd.lv[l].offset), c, up);
}

inline dim3 grid_lv(uint64_t n, uint32_t L) { return dim3((unsigned)((n + 255) / 256), L); }

}  // namespace

void launch_encode_fwd(const FieldLaunch& f, float* X, cudaStream_t s) {
  if (!f.n_total) return;
  k_encode_fwd<<<grid_lv(f.n_total, f.levels), 256, 0, s>>>(f, X);
}

void launch_encode_bwd(const FieldLaunch& f, const float* dX, cudaStream_t s) {
  if (!f.n_total) return;
  k_encode_bwd<<<grid_lv(f.n_total, f.levels), 256, 0, s>>>(f, dX);
}

void launch_encode_points(const FieldDesc* field, const float* params, const double* pts,
                          uint64_t n, uint32_t levels, float* X, uint32_t* rows, cudaStream_t s) {
  if (!n) return;
  k_encode_points<<<grid_lv(n, levels), 256, 0, s>>>(field, params, pts, n, X, rows);
}

void launch_encode_points_bwd(const FieldDesc* field, float* grads, const double* pts,
                              const float* dX, uint64_t n, uint32_t levels, cudaStream_t s) {
  if (!n) return;
  k_encode_points_bwd<<<grid_lv(n, levels), 256, 0, s>>>(field, grads, pts, dX, n);
}

}  // namespace dg
