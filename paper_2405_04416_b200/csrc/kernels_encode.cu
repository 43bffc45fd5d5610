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

// Warp-aggregated scatter of one level (the coarse levels, where neighbouring lanes share a
// lattice cell: consecutive samples of a ray, or of a spatially ordered chunk run).  Lanes are
// split into runs of equal (field, cell) in lane order; lanes of a run share all 8 corner rows,
// so one segmented shuffle scan per corner value (its depth ceil(log2(longest run)), found
// once per level) leaves each run's sums in its last lane, which issues the run's reds
// (corner pairs merged).  Inactive lanes (zero upstream) form runs of their own and issue none.
// PAIRED: a paired one-to-one level (kernels_pairs.cu): c.row[2j] is combo j's pair row (kNoRow
// outside the slice), and the run tail issues one float4 red per combo into the paired
// gradient copy.
template <bool PAIRED = false>
__device__ __forceinline__ void scatter_level_agg(void* __restrict__ dst, const Corners& c, const AxisW* ax,
                                                  float2 up, uint32_t field, bool act) {
  const unsigned lane = threadIdx.x & 31;
  const uint32_t key = act ? (ax[0].i0 | (ax[1].i0 << 11) | (ax[2].i0 << 22)) ^ (field << 31) : 0xffffffffu;
  const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
  const bool head = lane == 0 || prev != key || !act;
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  const unsigned run = 31u - __clz(heads & (0xffffffffu >> (31u - lane)));  // run start lane
  const unsigned later = lane < 31 ? heads & (0xfffffffeu << lane) : 0u;
  const unsigned len = head ? (later ? (unsigned)(__ffs(later) - 1) : 32u) - lane : 0u;
  const unsigned longest = __reduce_max_sync(0xffffffffu, len);
  float2 g[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) g[k] = make_float2(c.w[k] * up.x, c.w[k] * up.y);
  for (unsigned off = 1; off < longest; off <<= 1) {
    const bool take = lane >= off && lane - off >= run;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float tx = __shfl_up_sync(0xffffffffu, g[k].x, off);
      const float ty = __shfl_up_sync(0xffffffffu, g[k].y, off);
      if (take) {
        g[k].x += tx;
        g[k].y += ty;
      }
    }
  }
  const bool tail = lane == 31 || ((heads >> (lane + 1)) & 1u);
  if (!(tail && act)) return;
  if (PAIRED) {
    float4* pg = static_cast<float4*>(dst);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 g0 = g[2 * j], g1 = g[2 * j + 1];
      if (c.row[2 * j] != kNoRow && (g0.x != 0.f || g0.y != 0.f || g1.x != 0.f || g1.y != 0.f))
        atomicAdd(pg + c.row[2 * j], make_float4(g0.x, g0.y, g1.x, g1.y));
    }
    return;
  }
  float2* table = static_cast<float2*>(dst);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t r0 = c.row[2 * j], r1 = c.row[2 * j + 1];
    const float2 g0 = g[2 * j], g1 = g[2 * j + 1];
    if (is_pair(r0, r1)) {
      const float4 v = (r0 & 1u) ? make_float4(g1.x, g1.y, g0.x, g0.y) : make_float4(g0.x, g0.y, g1.x, g1.y);
      atomicAdd(reinterpret_cast<float4*>(table) + (r0 >> 1), v);
    } else {
      if (r0 != 0xffffffffu) atomicAdd(table + r0, g0);
      if (r1 != 0xffffffffu) atomicAdd(table + r1, g1);
    }
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
// (no minimum-blocks bound: `__launch_bounds__(256, 1)` lets ptxas take 72 registers, +0.4 ms)
#ifdef ENC_FWD_MINB
#define ENC_FWD_BOUNDS __launch_bounds__(256, ENC_FWD_MINB)
#else
#define ENC_FWD_BOUNDS __launch_bounds__(256)
#endif
template <bool PC, bool ALL>
__global__ void ENC_FWD_BOUNDS k_encode_fwd(FieldLaunch f, float* __restrict__ X) {
  const EncPass ps = f.pass[blockIdx.y];
  const uint64_t s = (ALL ? 0ull : (uint64_t)f.field_off[ps.f]) + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= (ALL ? (uint64_t)f.n_total : (uint64_t)f.field_off[ps.f + 1])) return;
  const uint32_t fidx = ALL ? sample_field(f, s) : ps.f;
  const FieldDesc& fd = f.fields[fidx];
  double p[3];
  load_point<PC>(f, s, fd, p);
  const uint32_t slo = (ALL && fidx) ? ps.lo[1] : ps.lo[0], shi = (ALL && fidx) ? ps.hi[1] : ps.hi[0];
  for (uint32_t l = ps.l0; l < ps.l1; ++l) {
    const LevelDesc lv = fd.lv[l];
    const LatticeAxes la = lattice_axes(lv, p);
    float2 acc;
    if (lv.poff != kNoPair && f.pairs) {  // one-to-one level through its paired copy (uniform)
      acc = ps.S > 1 ? gather_level_paired<true>(lv, la, f.pairs + lv.poff, slo, shi)
                     : gather_level_paired<false>(lv, la, f.pairs + lv.poff, 0u, 0u);
    } else {
      const float2* table = reinterpret_cast<const float2*>(f.params + fd.base + lv.offset);
      acc = ps.S > 1 ? gather_level_w32<true>(lv, la, table, slo, shi)
                     : gather_level_w32<false>(lv, la, table, 0u, 0u);
    }
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
#define ENC_BWD_MINB 4  // 4 CTAs per SM (64 registers; the per-cell run scan holds 16 sums)
#endif
// PAIRED: the launch's passes contain paired one-to-one levels (kernels_pairs.cu); the hashed
// level passes run the variant without that code path (register allocation).
template <bool PC, bool ALL, bool PAIRED>
__global__ void __launch_bounds__(256, ENC_BWD_MINB) k_encode_bwd(FieldLaunch f, const float* __restrict__ dX) {
  const EncPass ps = f.pass[blockIdx.y];
  const uint32_t bx = f.cta_mul ? (uint32_t)(((uint64_t)blockIdx.x * f.cta_mul) % gridDim.x) : blockIdx.x;
  const uint64_t s = (ALL ? 0ull : (uint64_t)f.field_off[ps.f]) + (uint64_t)bx * blockDim.x + threadIdx.x;
  const bool valid = s < (ALL ? (uint64_t)f.n_total : (uint64_t)f.field_off[ps.f + 1]);
  const uint32_t fidx = ALL ? (valid ? sample_field(f, s) : 0u) : ps.f;
  double p[3] = {0.0, 0.0, 0.0};
  const FieldDesc& fd = f.fields[fidx];
  if (valid) load_point<PC>(f, s, fd, p);
  const uint32_t slot = (ALL && fidx) ? 1u : 0u;
  for (uint32_t l = ps.l0; l < ps.l1; ++l) {
    float2 up = make_float2(0.f, 0.f);
    Corners c;
    LatticeAxes la;
    const bool paired = PAIRED && fd.lv[l].poff != kNoPair;  // uniform per (field, level)
    if (valid) {
      up = ld_stream(reinterpret_cast<const float2*>(dX) + (uint64_t)l * f.n_total + s);
      la = lattice_axes(fd.lv[l], p);
      if (paired) {
        uint32_t r0[4];
        if (ps.S > 1) paired_corners<true>(fd.lv[l], la, slot ? ps.lo[1] : ps.lo[0], slot ? ps.hi[1] : ps.hi[0], r0, c.w);
        else paired_corners<false>(fd.lv[l], la, 0u, 0u, r0, c.w);
#pragma unroll
        for (int j = 0; j < 4; ++j) c.row[2 * j] = r0[j];
      } else {
        corners_w32(fd.lv[l], la, c);
        clip_to_slice(ps, slot, c);
      }
    }
    const bool act = valid && (up.x != 0.f || up.y != 0.f);
    if (paired) {
      float4* pg = f.pgrads + fd.lv[l].poff;
      if (l < f.agg_levels) {
        scatter_level_agg<true>(pg, c, la.a, up, fidx, act);
      } else if (act) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float w0 = c.w[2 * j], w1 = c.w[2 * j + 1];
          if (c.row[2 * j] != kNoRow && (w0 != 0.f || w1 != 0.f))
            atomicAdd(pg + c.row[2 * j], make_float4(w0 * up.x, w0 * up.y, w1 * up.x, w1 * up.y));
        }
      }
      continue;
    }
    float2* table = reinterpret_cast<float2*>(f.grads + fd.base + fd.lv[l].offset);
    if (l < f.agg_levels) {  // coarse levels: neighbouring lanes share cells (warp-uniform branch)
      scatter_level_agg(table, c, la.a, up, fidx, act);
    } else if (act) {
      scatter_level_pairs(table, c, up);
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
  for (int paired = 1; paired >= 0; --paired) {  // passes with paired levels first (reds commute)
    std::vector<EncPass> pk;
    for (const EncPass& p : passes)
      if ((f.pgrads != nullptr && p.paired != 0) == (paired != 0)) pk.push_back(p);
    for (uint32_t i = 0; i < pk.size(); i += chunk) {
      FieldLaunch h = f;
      h.n_pass = std::min<uint32_t>(chunk, (uint32_t)pk.size() - i);
      for (uint32_t j = 0; j < h.n_pass; ++j) h.pass[j] = pk[i + j];
      const dim3 grid(pass_blocks(h, h.pass, h.n_pass), h.n_pass);
      const bool all = h.pass[0].f == kAllFields;
      if (f.s_p && paired) {
        if (all) k_encode_bwd<true, true, true><<<grid, 256, 0, s>>>(h, dX);
        else k_encode_bwd<true, false, true><<<grid, 256, 0, s>>>(h, dX);
      } else if (f.s_p) {
        if (all) k_encode_bwd<true, true, false><<<grid, 256, 0, s>>>(h, dX);
        else k_encode_bwd<true, false, false><<<grid, 256, 0, s>>>(h, dX);
      } else {
        if (all) k_encode_bwd<false, true, false><<<grid, 256, 0, s>>>(h, dX);
        else k_encode_bwd<false, false, false><<<grid, 256, 0, s>>>(h, dX);
      }
      ++launches;
    }
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
