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

// Streaming accesses (sample arrays, features) bypass L2 residency so the hash tables keep it.
__device__ __forceinline__ float2 ld_stream(const float2* p) {
  float2 v;
  asm volatile("ld.global.cs.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream(float2* p, float2 v) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y));
}

// Warp-aggregated scatter of one level: lanes hold consecutive samples (mostly one ray, in t
// order), so at coarse levels neighbouring lanes share cells and hence identical corner rows.
// For each corner slot, runs of equal (field, row) in lane order are summed with a segmented
// shuffle scan and the run's last lane issues a single float2 red.
__device__ __forceinline__ void scatter_level_agg(float2* __restrict__ table, const Corners& c,
                                                  float2 up, uint32_t field, bool valid) {
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t row = valid ? c.row[k] : 0xffffffffu;
    const uint32_t prev_row = __shfl_up_sync(0xffffffffu, row, 1);
    const uint32_t prev_fld = __shfl_up_sync(0xffffffffu, field, 1);
    const bool head = lane == 0 || prev_row != row || prev_fld != field;
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    const unsigned run = 31u - __clz(heads & (0xffffffffu >> (31u - lane)));  // run start lane
    float vx = c.w[k] * up.x, vy = c.w[k] * up.y;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float tx = __shfl_up_sync(0xffffffffu, vx, off);
      const float ty = __shfl_up_sync(0xffffffffu, vy, off);
      if (lane >= (unsigned)off && lane - off >= run) {
        vx += tx;
        vy += ty;
      }
    }
    const bool tail = lane == 31 || ((heads >> (lane + 1)) & 1u);
    if (tail && row != 0xffffffffu && (vx != 0.f || vy != 0.f))
      atomicAdd(table + row, make_float2(vx, vy));
  }
}

// Level-group launch: grid (sample chunks, level groups).  Group 0 holds the leading dense
// (one-to-one) levels, whose tables fit in L2 together; every hashed level (2^T rows) is its
// own group.  CTAs are dispatched roughly in blockIdx order, so the device works through one
// group's tables at a time and they stay L2-resident instead of streaming all 16 levels'
// random rows from HBM at once.  Features are level-major (X[l][s] float2): coalesced.
__global__ void __launch_bounds__(256) k_encode_fwd(FieldLaunch f, float* __restrict__ X) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= f.n_total) return;
  const uint32_t l0 = blockIdx.y == 0 ? 0u : f.dense_levels + blockIdx.y - 1;
  const uint32_t l1 = blockIdx.y == 0 ? f.dense_levels : l0 + 1;
  const uint32_t casc = s >= f.fine_total ? 1u : 0u;
  const uint32_t item = __ldcs(f.s_item + s);
  const FieldDesc& fd = f.fields[casc * f.n_local + f.item_part[item]];
  const RayRec& r = f.rec[item];
  double p[3];
  normalized_point(fd.box_lo, fd.box_hi, r.o, r.d, __ldcs(f.s_t + s), p);
  for (uint32_t l = l0; l < l1; ++l) {
    Corners c;
    level_corners(fd.lv[l], p, c);
    const float2 acc = gather_level(reinterpret_cast<const float2*>(f.params + fd.base + fd.lv[l].offset), c);
    st_stream(reinterpret_cast<float2*>(X) + (uint64_t)l * f.n_total + s, acc);
  }
}

__global__ void __launch_bounds__(256) k_encode_bwd(FieldLaunch f, const float* __restrict__ dX) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = s < f.n_total;
  const uint32_t l0 = blockIdx.y == 0 ? 0u : f.dense_levels + blockIdx.y - 1;
  const uint32_t l1 = blockIdx.y == 0 ? f.dense_levels : l0 + 1;
  uint32_t fidx = 0;
  double p[3] = {0.0, 0.0, 0.0};
  const FieldDesc* fdp = f.fields;
  if (valid) {
    const uint32_t casc = s >= f.fine_total ? 1u : 0u;
    const uint32_t item = __ldcs(f.s_item + s);
    fidx = casc * f.n_local + f.item_part[item];
    fdp = f.fields + fidx;
    const RayRec& r = f.rec[item];
    normalized_point(fdp->box_lo, fdp->box_hi, r.o, r.d, __ldcs(f.s_t + s), p);
  }
  const FieldDesc& fd = *fdp;
  for (uint32_t l = l0; l < l1; ++l) {
    float2 up = make_float2(0.f, 0.f);
    Corners c;
    if (valid) {
      up = ld_stream(reinterpret_cast<const float2*>(dX) + (uint64_t)l * f.n_total + s);
      level_corners(fd.lv[l], p, c);
    }
    float2* table = reinterpret_cast<float2*>(f.grads + fd.base + fd.lv[l].offset);
    if (l < f.agg_levels) {  // coarse levels: consecutive samples share corners
      scatter_level_agg(table, c, up, fidx, valid && (up.x != 0.f || up.y != 0.f));
    } else if (valid && (up.x != 0.f || up.y != 0.f)) {
      scatter_level(table, c, up);
    }
  }
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

inline dim3 grid_groups(const FieldLaunch& f) {
  return dim3((unsigned)((f.n_total + 255) / 256), 1u + (f.levels - f.dense_levels));
}

}  // namespace

void launch_encode_fwd(const FieldLaunch& f, float* X, cudaStream_t s) {
  if (!f.n_total) return;
  k_encode_fwd<<<grid_groups(f), 256, 0, s>>>(f, X);
}

void launch_encode_bwd(const FieldLaunch& f, const float* dX, cudaStream_t s) {
  if (!f.n_total) return;
  k_encode_bwd<<<grid_groups(f), 256, 0, s>>>(f, dX);
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
