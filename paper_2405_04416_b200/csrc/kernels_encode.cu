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
#include <algorithm>
#include <cstdlib>

#include "encode_common.cuh"
#include "geometry.cuh"
#include "kernels.h"

namespace dg {

namespace {

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

__device__ __forceinline__ void scatter_level_pairs(float2* __restrict__ table, const Corners& c, float2 up) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t r0 = c.row[2 * j], r1 = c.row[2 * j + 1];
    const float2 g0 = make_float2(c.w[2 * j] * up.x, c.w[2 * j] * up.y);
    const float2 g1 = make_float2(c.w[2 * j + 1] * up.x, c.w[2 * j + 1] * up.y);
    if (is_pair(r0, r1)) {
      const float4 v = (r0 & 1u) ? make_float4(g1.x, g1.y, g0.x, g0.y) : make_float4(g0.x, g0.y, g1.x, g1.y);
      atomicAdd(reinterpret_cast<float4*>(table) + (r0 >> 1), v);
    } else {
      if (r0 != 0xffffffffu) atomicAdd(table + r0, g0);
      if (r1 != 0xffffffffu) atomicAdd(table + r1, g1);
    }
  }
}

// lattice_axis's upper index for lower index i0 (grid.cpp:22-41: clamped to n - 1)
__device__ __forceinline__ uint32_t la_i1_of(uint32_t i0, uint32_t n) { return i0 + 1 < n - 1 ? i0 + 1 : n - 1; }

// Keep only the corners whose row lies in this pass's slice of the level table (bounds from the
// host: EncPass::lo / hi, slot = the sample's field in an all-fields pass, else 0).
__device__ __forceinline__ void clip_to_slice(const EncPass& ps, uint32_t slot, Corners& c) {
  if (ps.S == 1) return;
  const uint32_t lo = slot ? ps.lo[1] : ps.lo[0], hi = slot ? ps.hi[1] : ps.hi[0];  // no dynamic index
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (c.row[k] < lo || c.row[k] >= hi) c.row[k] = 0xffffffffu;
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
// shuffle scan and the run's last lane issues a single float2 red.  The scan runs only
// ceil(log2(longest run)) steps (warp-uniform, from the run-head ballot).
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
    // run length seen from its head lane: distance to the next head (or the warp end)
    const unsigned later = lane < 31 ? heads & (0xfffffffeu << lane) : 0u;
    const unsigned len = head ? (later ? (unsigned)(__ffs(later) - 1) : 32u) - lane : 0u;
    const unsigned longest = __reduce_max_sync(0xffffffffu, len);
    float vx = c.w[k] * up.x, vy = c.w[k] * up.y;
    for (unsigned off = 1; off < longest; off <<= 1) {
      const float tx = __shfl_up_sync(0xffffffffu, vx, off);
      const float ty = __shfl_up_sync(0xffffffffu, vy, off);
      if (lane >= off && lane - off >= run) {
        vx += tx;
        vy += ty;
      }
    }
    const bool tail = lane == 31 || ((heads >> (lane + 1)) & 1u);
    if (tail && row != 0xffffffffu && (vx != 0.f || vy != 0.f))
      atomicAdd(table + row, make_float2(vx, vy));
  }
}

// Field of sample s (samples are field-major; field_off lives in the kernel parameters).
__device__ __forceinline__ uint32_t sample_field(const FieldLaunch& f, uint64_t s) {
  uint32_t lo = 0, hi = f.n_fields;  // field_off[lo] <= s < field_off[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (s >= f.field_off[mid]) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Normalised position of sample s: from the per-sample cache (PC) or re-derived from
// (item, t) exactly as the march fill does (grid.cpp:109 normalisation).
template <bool PC>
__device__ __forceinline__ void load_point(const FieldLaunch& f, uint64_t s, const FieldDesc& fd,
                                           double p[3]) {
  if (PC) {
    p[0] = __ldcs(f.s_p + s);
    p[1] = __ldcs(f.s_p + f.n_total + s);
    p[2] = __ldcs(f.s_p + 2 * (uint64_t)f.n_total + s);
  } else {
    const RayRec& r = f.rec[__ldcs(f.s_item + s)];
    normalized_point(fd.box_lo, fd.box_hi, r.o, r.d, __ldcs(f.s_t + s), p);
  }
}

// grid (sample chunks, passes).  CTAs are dispatched roughly in blockIdx order, so the device
// works through one pass (a few small tables, or one slice of a large one) at a time and
// that working set stays L2-resident.  Features are level-major (X[l][s] float2): coalesced.
// Slice k > 0 of a level runs in a later launch and adds into X.  The sample's normalised
// position (fp64, bit-exact) comes from the march, so a pass is: 3 streaming loads, the
// lattice math, 8 gathers.
// ALL: every pass of the launch covers every local field's samples (one partition per GPU);
// otherwise each pass covers one field's samples (several partitions per GPU).
template <bool PC, bool ALL>
__global__ void __launch_bounds__(256) k_encode_fwd(FieldLaunch f, float* __restrict__ X) {
  const EncPass ps = f.pass[blockIdx.y];
  const uint64_t s = (ALL ? 0ull : (uint64_t)f.field_off[ps.f]) + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= (ALL ? (uint64_t)f.n_total : (uint64_t)f.field_off[ps.f + 1])) return;
  const uint32_t fidx = ALL ? sample_field(f, s) : ps.f;
  const FieldDesc& fd = f.fields[fidx];
  double p[3];
  load_point<PC>(f, s, fd, p);
  for (uint32_t l = ps.l0; l < ps.l1; ++l) {
    Corners c;
    level_corners(fd.lv[l], p, c);
    clip_to_slice(ps, ALL ? fidx : 0u, c);
    float2 acc = gather_level_pairs(reinterpret_cast<const float2*>(f.params + fd.base + fd.lv[l].offset), c);
    float2* xp = reinterpret_cast<float2*>(X) + (uint64_t)l * f.n_total + s;
    if (ps.k > 0) {
      const float2 o = ld_stream(xp);
      acc.x += o.x;
      acc.y += o.y;
    }
    st_stream(xp, acc);
  }
}

#ifndef ENC_BWD_MINB
#define ENC_BWD_MINB 5  // 5 CTAs per SM (48 registers, 16 B of spills): ~1 % faster than 4
#endif
template <bool PC, bool ALL>
__global__ void __launch_bounds__(256, ENC_BWD_MINB) k_encode_bwd(FieldLaunch f, const float* __restrict__ dX) {
  const EncPass ps = f.pass[blockIdx.y];
  const uint32_t bx = f.cta_mul ? (uint32_t)(((uint64_t)blockIdx.x * f.cta_mul) % gridDim.x) : blockIdx.x;
  const uint64_t s = (ALL ? 0ull : (uint64_t)f.field_off[ps.f]) + (uint64_t)bx * blockDim.x + threadIdx.x;
  const bool valid = s < (ALL ? (uint64_t)f.n_total : (uint64_t)f.field_off[ps.f + 1]);
  const uint32_t fidx = ALL ? (valid ? sample_field(f, s) : 0u) : ps.f;
  double p[3] = {0.0, 0.0, 0.0};
  const FieldDesc& fd = f.fields[fidx];
  if (valid) load_point<PC>(f, s, fd, p);
  for (uint32_t l = ps.l0; l < ps.l1; ++l) {
    float2 up = make_float2(0.f, 0.f);
    Corners c;
    if (valid) {
      up = ld_stream(reinterpret_cast<const float2*>(dX) + (uint64_t)l * f.n_total + s);
      level_corners_w32(fd.lv[l], p, c);
      clip_to_slice(ps, ALL ? fidx : 0u, c);
    }
    float2* table = reinterpret_cast<float2*>(f.grads + fd.base + fd.lv[l].offset);
    if (l < f.agg_levels) {  // coarse levels: consecutive samples share corners
      scatter_level_agg(table, c, up, fidx, valid && (up.x != 0.f || up.y != 0.f));
    } else if (valid && (up.x != 0.f || up.y != 0.f)) {
      scatter_level_pairs(table, c, up);
    }
  }
}

// Backward over spatially ordered samples (kernels_order.cu): a warp's 32 consecutive samples
// are a compact blob of the field, so at the coarse levels all of its active lanes usually sit
// in one lattice cell and share its 8 corners.  Such a warp sums its 8 x 2 corner
// contributions across the lanes (a transposing butterfly: 16 shuffles, after which lane L
// holds the sum of value (L >> 1) & 15) and issues 8 float2 reds instead of 256; other warps
// scatter per lane (corner pairs merged, as k_encode_bwd).  CTAs visit their sample chunks in
// a strided order (f.cta_mul) so that concurrently running CTAs work on distant blobs and
// their reds do not contend for the same rows.
#ifndef ENC_ORD_MINB
#define ENC_ORD_MINB 4
#endif
template <bool ALL>
__global__ void __launch_bounds__(256, ENC_ORD_MINB) k_encode_bwd_ord(FieldLaunch f, const float* __restrict__ dX) {
  const EncPass ps = f.pass[blockIdx.y];
  const uint32_t bx = f.cta_mul ? (uint32_t)(((uint64_t)blockIdx.x * f.cta_mul) % gridDim.x) : blockIdx.x;
  const uint64_t base = ALL ? 0ull : (uint64_t)f.field_off[ps.f];
  const uint64_t end = ALL ? (uint64_t)f.n_total : (uint64_t)f.field_off[ps.f + 1];
  const uint64_t s = base + (uint64_t)bx * blockDim.x + threadIdx.x;
  const bool valid = s < end;
  const uint32_t fidx = ALL ? (valid ? sample_field(f, s) : 0u) : ps.f;
  const FieldDesc& fd = f.fields[fidx];
  double p[3] = {0.0, 0.0, 0.0};
  if (valid) load_point<true>(f, s, fd, p);
  const unsigned lane = threadIdx.x & 31;
  // a warp whose samples span two fields never takes the shared-cell path
  const uint32_t f_lo = __shfl_sync(0xffffffffu, fidx, 0), f_hi = __reduce_max_sync(0xffffffffu, valid ? fidx : 0u);
  const bool one_field = f_lo == f_hi;
  for (uint32_t l = ps.l0; l < ps.l1; ++l) {
    const LevelDesc& lv = fd.lv[l];
    float2 up = make_float2(0.f, 0.f);
    if (valid) up = ld_stream(reinterpret_cast<const float2*>(dX) + (uint64_t)l * f.n_total + s);
    const bool act = valid && (up.x != 0.f || up.y != 0.f);
    const unsigned amask = __ballot_sync(0xffffffffu, act);
    if (!amask) continue;
    float2* table = reinterpret_cast<float2*>(f.grads + fd.base + lv.offset);
    LatticeAxes la;
    if (act) la = lattice_axes(lv, p);
    const int lead = __ffs(amask) - 1;
    uint32_t cell[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) cell[a] = __shfl_sync(0xffffffffu, act ? la.a[a].i0 : 0u, lead);
    const bool same = !act || (la.a[0].i0 == cell[0] && la.a[1].i0 == cell[1] && la.a[2].i0 == cell[2]);
    if (one_field && __all_sync(0xffffffffu, same)) {
      float v[16];
      {
        float w[8];
        bool zero[8];
        if (act) corner_weights_w32(la, w, zero);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float wk = (act && !zero[k]) ? w[k] : 0.f;
          v[2 * k] = wk * up.x;
          v[2 * k + 1] = wk * up.y;
        }
      }
#pragma unroll
      for (int step = 0; step < 4; ++step) {
        const int o = 16 >> step, half = 8 >> step;
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i < half) {
            const float send = upper ? v[i] : v[half + i];
            const float keep = upper ? v[half + i] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
      }
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
      // lane 4k holds corner k's x sum, lane 4k + 2 its y sum
      const float vy = __shfl_down_sync(0xffffffffu, v[0], 2);
      if ((lane & 3) == 0 && (v[0] != 0.f || vy != 0.f)) {
        const uint32_t k = lane >> 2;
        const uint32_t x = (k & 1) ? la_i1_of(cell[0], lv.n[0]) : cell[0];
        const uint32_t y = ((k >> 1) & 1) ? la_i1_of(cell[1], lv.n[1]) : cell[1];
        const uint32_t z = ((k >> 2) & 1) ? la_i1_of(cell[2], lv.n[2]) : cell[2];
        const uint32_t row = vertex_row(lv, x, y, z);
        const uint32_t slot = ALL ? fidx : 0u;
        const bool in = ps.S == 1 || (row >= (slot ? ps.lo[1] : ps.lo[0]) && row < (slot ? ps.hi[1] : ps.hi[0]));
        if (in) atomicAdd(table + row, make_float2(v[0], vy));
      }
    } else {
      Corners c;
      if (act) {
        corners_w32(lv, la, c);
        clip_to_slice(ps, ALL ? fidx : 0u, c);
      }
      if (l < f.agg_levels) scatter_level_agg(table, c, up, fidx, act);  // warp-uniform branch
      else if (act) scatter_level_pairs(table, c, up);
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

}  // namespace

namespace {
// CTAs along x for a chunk of passes: the largest field among them
unsigned pass_blocks(const FieldLaunch& f, const EncPass* p, uint32_t n) {
  uint64_t m = 0;
  for (uint32_t i = 0; i < n; ++i)
    m = std::max<uint64_t>(m, p[i].f == kAllFields ? (uint64_t)f.n_total : f.field_off[p[i].f + 1] - f.field_off[p[i].f]);
  return (unsigned)((m + 255) / 256);
}
}  // namespace

int launch_encode_fwd(const FieldLaunch& f, const std::vector<EncPass>& passes, float* X, cudaStream_t s) {
  if (!f.n_total || passes.empty()) return 0;
  static const bool split = std::getenv("DG_ENC_SPLIT_LAUNCH") != nullptr;  // per-pass timing
  int launches = 0;
  for (uint32_t k = 0;; ++k) {  // slice k of every pass group, in pass order (k > 0 adds into X)
    std::vector<EncPass> pk;
    for (const EncPass& p : passes)
      if (p.k == k) pk.push_back(p);
    if (pk.empty()) break;
    const uint32_t chunk = split ? 1u : (uint32_t)kMaxEncPass;
    for (uint32_t i = 0; i < pk.size(); i += chunk) {
      FieldLaunch h = f;
      h.n_pass = std::min<uint32_t>(chunk, (uint32_t)pk.size() - i);
      for (uint32_t j = 0; j < h.n_pass; ++j) h.pass[j] = pk[i + j];
      const dim3 grid(pass_blocks(h, h.pass, h.n_pass), h.n_pass);
      const bool all = h.pass[0].f == kAllFields;  // a pass list is all-fields or per-field
      if (f.s_p) {
        if (all) k_encode_fwd<true, true><<<grid, 256, 0, s>>>(h, X);
        else k_encode_fwd<true, false><<<grid, 256, 0, s>>>(h, X);
      } else {
        if (all) k_encode_fwd<false, true><<<grid, 256, 0, s>>>(h, X);
        else k_encode_fwd<false, false><<<grid, 256, 0, s>>>(h, X);
      }
      ++launches;
    }
  }
  return launches;
}

int launch_encode_bwd(const FieldLaunch& f, const std::vector<EncPass>& passes, const float* dX, cudaStream_t s) {
  if (!f.n_total || passes.empty()) return 0;
  static const bool split = std::getenv("DG_ENC_SPLIT_LAUNCH") != nullptr;  // per-pass timing
  const uint32_t chunk = split ? 1u : (uint32_t)kMaxEncPass;
  int launches = 0;
  for (uint32_t i = 0; i < passes.size(); i += chunk) {  // reds commute: any grouping
    FieldLaunch h = f;
    h.n_pass = std::min<uint32_t>(chunk, (uint32_t)passes.size() - i);
    for (uint32_t j = 0; j < h.n_pass; ++j) h.pass[j] = passes[i + j];
    const dim3 grid(pass_blocks(h, h.pass, h.n_pass), h.n_pass);
    const bool all = h.pass[0].f == kAllFields;
    if (f.s_p && f.box_bwd) {
      if (all) k_encode_bwd_ord<true><<<grid, 256, 0, s>>>(h, dX);
      else k_encode_bwd_ord<false><<<grid, 256, 0, s>>>(h, dX);
    } else if (f.s_p) {
      if (all) k_encode_bwd<true, true><<<grid, 256, 0, s>>>(h, dX);
      else k_encode_bwd<true, false><<<grid, 256, 0, s>>>(h, dX);
    } else {
      if (all) k_encode_bwd<false, true><<<grid, 256, 0, s>>>(h, dX);
      else k_encode_bwd<false, false><<<grid, 256, 0, s>>>(h, dX);
    }
    ++launches;
  }
  return launches;
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
