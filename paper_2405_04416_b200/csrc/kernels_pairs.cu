// kernels_pairs.cu — paired copies of the one-to-one (dense) level tables.
//
// A lattice corner pair (x0, x0 + 1) of a one-to-one level sits in rows r and r + 1
// (grid.cpp:75-84: row = x + nx (y + ny z)), one aligned float4 only when r is even.  The
// encode kernels read and scatter such a pair through a paired copy instead: pairs[r] =
// (row r, row r + 1) as one float4, so every (y, z) corner pair is exactly one 16-byte gather
// forward and one `red.global.add.v4.f32` backward (4 per sample and level instead of ~6).
//   k_pairs_expand   pairs[r] = (T[r], T[r + 1])            before the forward (after Adam)
//   k_pairs_fold     grad T[r] += G[r].xy + G[r - 1].zw     after the backward, before Adam
// The canonical tables (Adam, checkpoints, the occupancy query, the stage API) are untouched.
#include "kernels.h"

namespace dg {

namespace {

// segment of global pair index i (segments are contiguous in pair0 order)
__device__ __forceinline__ uint32_t pair_seg(const PairSeg* __restrict__ segs, uint32_t nseg, uint64_t i) {
  uint32_t lo = 0, hi = nseg;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (i >= segs[mid].pair0) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void k_pairs_expand(const PairSeg* __restrict__ segs, uint32_t nseg, uint64_t total,
                               const float* __restrict__ params, float4* __restrict__ pairs) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const PairSeg sg = segs[pair_seg(segs, nseg, i)];
  const uint64_t r = i - sg.pair0;
  const float2* t = reinterpret_cast<const float2*>(params + sg.table);
  const float2 a = t[r];
  const float2 b = r + 1 < sg.rows ? t[r + 1] : make_float2(0.f, 0.f);
  __stcg(pairs + i, make_float4(a.x, a.y, b.x, b.y));
}

__global__ void k_pairs_fold(const PairSeg* __restrict__ segs, uint32_t nseg, uint64_t total,
                             const float4* __restrict__ pgrads, float* __restrict__ grads) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const PairSeg sg = segs[pair_seg(segs, nseg, i)];
  const uint64_t r = i - sg.pair0;
  const float4 g = __ldcs(pgrads + i);
  float2 acc = make_float2(g.x, g.y);
  if (r > 0) {
    const float4 p = __ldcs(pgrads + i - 1);
    acc.x += p.z;
    acc.y += p.w;
  }
  if (acc.x != 0.f || acc.y != 0.f) {
    float2* t = reinterpret_cast<float2*>(grads + sg.table) + r;
    float2 v = *t;
    v.x += acc.x;
    v.y += acc.y;
    *t = v;
  }
}

}  // namespace

void launch_pairs_expand(const PairSeg* segs, uint32_t nseg, uint64_t total, const float* params, float4* pairs,
                         cudaStream_t s) {
  if (total) k_pairs_expand<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(segs, nseg, total, params, pairs);
}

void launch_pairs_fold(const PairSeg* segs, uint32_t nseg, uint64_t total, float4* pgrads, float* grads,
                       cudaStream_t s) {
  if (!total) return;
  k_pairs_fold<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(segs, nseg, total, pgrads, grads);
  cudaMemsetAsync(pgrads, 0, total * sizeof(float4), s);  // zero for the next backward
}

}  // namespace dg
