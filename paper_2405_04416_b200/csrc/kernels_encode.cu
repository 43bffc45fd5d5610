// kernels_encode.cu — stage 3: multi-resolution hash-grid encode forward and backward.
//
//   k_encode_fwd   HashGrid::encode (grid.cpp:107-130) on the march samples; one thread per
//                  (sample, level), 16 lanes per sample, so a warp covers 2 samples x 16
//                  levels and each lane has its 8 corner gathers in flight at once (float2
//                  rows, F = 2).  Position, lattice indices and corner weights are fp64 and
//                  bit-exact (geometry.cuh); features accumulate in fp32.
//   k_encode_bwd   HashGrid::encode_backward (grid.cpp:132-157): the same corners receive
//                  w * upstream through vector float2 atomics (red.global.add.v2.f32).
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

__global__ void __launch_bounds__(256) k_encode_fwd(FieldLaunch f, float* __restrict__ X) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t s = tid >> 4;
  const uint32_t l = (uint32_t)(tid & 15);
  if (s >= f.n_total) return;
  const uint32_t casc = s >= f.fine_total ? 1u : 0u;
  const uint32_t item = f.s_item[s];
  const FieldDesc& fd = f.fields[casc * f.n_local + f.item_part[item]];
  float2 acc = make_float2(0.f, 0.f);
  if (l < fd.L) {
    const RayRec& r = f.rec[item];
    double p[3];
    normalized_point(fd.box_lo, fd.box_hi, r.o, r.d, f.s_t[s], p);
    Corners c;
    level_corners(fd.lv[l], p, c);
    acc = gather_level(reinterpret_cast<const float2*>(f.params + fd.base + fd.lv[l].offset), c);
  }
  reinterpret_cast<float2*>(X)[s * 16 + l] = acc;
}

__global__ void __launch_bounds__(256) k_encode_bwd(FieldLaunch f, const float* __restrict__ dX) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t s = tid >> 4;
  const uint32_t l = (uint32_t)(tid & 15);
  if (s >= f.n_total) return;
  const uint32_t casc = s >= f.fine_total ? 1u : 0u;
  const uint32_t item = f.s_item[s];
  const FieldDesc& fd = f.fields[casc * f.n_local + f.item_part[item]];
  if (l >= fd.L) return;
  const float2 up = reinterpret_cast<const float2*>(dX)[s * 16 + l];
  if (up.x == 0.f && up.y == 0.f) return;
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
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t s = tid >> 4;
  const uint32_t l = (uint32_t)(tid & 15);
  if (s >= n) return;
  const FieldDesc& fd = *field;
  float2 acc = make_float2(0.f, 0.f);
  if (l < fd.L) {
    const double p[3] = {pts[3 * s], pts[3 * s + 1], pts[3 * s + 2]};
    Corners c;
    level_corners(fd.lv[l], p, c);
    if (rows)
      for (int k = 0; k < 8; ++k) rows[(s * fd.L + l) * 8 + k] = c.row[k];
    acc = gather_level(reinterpret_cast<const float2*>(params + fd.base + fd.lv[l].offset), c);
  }
  reinterpret_cast<float2*>(X)[s * 16 + l] = acc;
}

__global__ void k_encode_points_bwd(const FieldDesc* __restrict__ field, float* __restrict__ grads,
                                    const double* __restrict__ pts, const float* __restrict__ dX,
                                    uint64_t n) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t s = tid >> 4;
  const uint32_t l = (uint32_t)(tid & 15);
  if (s >= n) return;
  const FieldDesc& fd = *field;
  if (l >= fd.L) return;
  const float2 up = reinterpret_cast<const float2*>(dX)[s * 16 + l];
  if (up.x == 0.f && up.y == 0.f) return;
  const double p[3] = {pts[3 * s], pts[3 * s + 1], pts[3 * s + 2]};
  Corners c;
  level_corners(fd.lv[l], p, c);
  scatter_level(reinterpret_cast<float2*>(grads + fd.base + fd.lv[l].offset), c, up);
}

inline unsigned grid16(uint64_t n) { return (unsigned)((n * 16 + 255) / 256); }

}  // namespace

void launch_encode_fwd(const FieldLaunch& f, float* X, cudaStream_t s) {
  if (!f.n_total) return;
  k_encode_fwd<<<grid16(f.n_total), 256, 0, s>>>(f, X);
}

void launch_encode_bwd(const FieldLaunch& f, const float* dX, cudaStream_t s) {
  if (!f.n_total) return;
  k_encode_bwd<<<grid16(f.n_total), 256, 0, s>>>(f, dX);
}

void launch_encode_points(const FieldDesc* field, const float* params, const double* pts,
                          uint64_t n, float* X, uint32_t* rows, cudaStream_t s) {
  if (!n) return;
  k_encode_points<<<grid16(n), 256, 0, s>>>(field, params, pts, n, X, rows);
}

void launch_encode_points_bwd(const FieldDesc* field, float* grads, const double* pts,
                              const float* dX, uint64_t n, cudaStream_t s) {
  if (!n) return;
  k_encode_points_bwd<<<grid16(n), 256, 0, s>>>(field, grads, pts, dX, n);
}

}  // namespace dg
