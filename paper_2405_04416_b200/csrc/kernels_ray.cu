// kernels_ray.cu — per-ray / per-item kernels of stages 1, 2 and 5.
//
//   k_segment_home    plan_batch (worker.cpp:141-165) + segment_ray (partition.cpp:254-296)
//   k_pack_dispatch   exchange-1 send layout (RayDispatch, wire.cpp:29-46)
//   k_item_setup      Worker::handle_training_batch phase-1 head (worker.cpp:268-284)
//                     + cascade_march sample count (worker.cpp:79-110)
//   k_march_fill      cascade_march sample emission into field-major sample arrays
//   k_composite       local_render (render.cpp:46-78) per (ray, partition) item
//   k_pack_partials   exchange-2 send layout (PartialScatter, worker.cpp:314-334)
//   k_merge_backward  backward_ray (worker.cpp:403-522): merge_forward, losses, merge_backward,
//                     distortion, local_render_backward (render.cpp:101-179, train.cpp:8-75)
//   k_home_merge      dispatch_eval driver merge (worker.cpp:801-826)
#include <cub/cub.cuh>

#include "geometry.cuh"
#include "kernels.h"

namespace dg {

namespace {

__device__ __forceinline__ void load_geo(Geo& sg, const Geo* g) {
  const uint32_t* src = reinterpret_cast<const uint32_t*>(g);
  uint32_t* dst = reinterpret_cast<uint32_t*>(&sg);
  for (int i = threadIdx.x; i < (int)(sizeof(Geo) / 4); i += blockDim.x) dst[i] = src[i];
  __syncthreads();
}

__global__ void k_segment_home(const Geo* __restrict__ geo, const double* __restrict__ o,
                               const double* __restrict__ d, uint64_t n,
                               const uint8_t* __restrict__ slot_of_part, uint8_t* __restrict__ nseg,
                               uint8_t* __restrict__ sched, uint32_t* __restrict__ flags,
                               unsigned long long* __restrict__ dropped) {
  __shared__ Geo sg;
  load_geo(sg, geo);
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool miss = false;
  if (i < n) {
    double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]};
    double dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
    uint8_t reg[kMaxSeg];
    double te[kMaxSeg], tx[kMaxSeg];
    const int ns = segment_ray(sg, oo, dd, reg, te, tx);
    nseg[i] = (uint8_t)ns;
    uint8_t* sc = sched + i * kMaxSeg;
    for (int s = 0; s < kMaxSeg; ++s) sc[s] = s < ns ? reg[s] : 0xff;
    for (int s = 0; s < ns; ++s) flags[(uint64_t)slot_of_part[reg[s]] * n + i] = 1u;
    miss = ns == 0;
  }
  const unsigned m = __ballot_sync(0xffffffffu, miss);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(dropped, (unsigned long long)__popc(m));
}

__global__ void k_pack_dispatch(uint64_t n, const uint8_t* __restrict__ nseg,
                                const uint8_t* __restrict__ sched,
                                const uint8_t* __restrict__ slot_of_part,
                                const uint32_t* __restrict__ pos, const double* __restrict__ o,
                                const double* __restrict__ d, const float* __restrict__ gt,
                                const uint32_t* __restrict__ img, uint64_t first_ray_id,
                                RayRec* __restrict__ out, PeerDst peer) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int ns = nseg[i];
  if (ns == 0) return;
  RayRec r;
  for (int a = 0; a < 3; ++a) {
    r.o[a] = o[3 * i + a];
    r.d[a] = d[3 * i + a];
    r.gt[a] = gt ? gt[3 * i + a] : 0.0f;
  }
  r.img = img ? img[i] : 0u;
  r.ray_id = (uint32_t)(first_ray_id + i);
  r.pad = 0;
  for (int s = 0; s < ns; ++s) {
    const uint32_t p = sched[i * kMaxSeg + s];
    const uint64_t slot = slot_of_part[p];
    if (peer.base) {  // straight into the owner's item array (peer store over NVLink)
      RayRec* dst = static_cast<RayRec*>(peer.base[p % peer.world]);
      dst[peer.off[p] + pos[slot * n + i] - pos[slot * n]] = r;
    } else {
      out[pos[slot * n + i]] = r;
    }
  }
  if (peer.base) __threadfence_system();
}

__device__ __forceinline__ uint32_t part_of_item(const uint32_t* off, uint32_t n_local, uint32_t i) {
  uint32_t p = 0;
  while (p + 1 < n_local && i >= off[p + 1]) ++p;
  return p;
}

__device__ __forceinline__ double round_f32(double v) { return (double)(float)v; }

__global__ void k_item_setup(const Geo* __restrict__ geo, const PartDesc* __restrict__ parts,
                             const uint8_t* __restrict__ occ,
                             const uint32_t* __restrict__ part_item_off, uint32_t n_local,
                             uint32_t n_items, ItemArrays it, uint32_t P, double step,
                             uint64_t seed, uint64_t batch_id, int jitter, int wire_f32,
                             uint32_t n_images, uint32_t* __restrict__ error) {
  __shared__ Geo sg;
  load_geo(sg, geo);
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const uint32_t lp = part_of_item(part_item_off, n_local, i);
  const PartDesc& pd = parts[lp];
  RayRec r = it.rec[i];
  uint8_t reg[kMaxSeg];
  double te[kMaxSeg], tx[kMaxSeg];
  const int ns = segment_ray(sg, r.o, r.d, reg, te, tx);
  int mo = -1;
  for (int s = 0; s < ns; ++s)
    if (reg[s] == pd.global_id) mo = s;
  if (mo < 0) {  // "dispatched ray does not intersect this region" (worker.cpp:274-276)
    atomicOr(error, 2u);
    it.nseg[i] = 0;
    it.order[i] = 0;
    it.part[i] = (uint8_t)lp;
    it.cnt[i] = it.cnt[n_items + i] = it.ncb[i] = 0u;
    for (uint32_t q = 0; q < P; ++q) it.contains[(uint64_t)q * n_items + i] = 0u;
    return;
  }
  if (r.img >= n_images) atomicOr(error, 1u);  // AppearanceTable::row (field.cpp:125-130)
  if (wire_f32) {  // WireWriter::real rounding of the RayDispatch payload (wire.hpp:55-62)
    for (int a = 0; a < 3; ++a) {
      r.o[a] = round_f32(r.o[a]);
      r.d[a] = round_f32(r.d[a]);
    }
    for (int s = 0; s < ns; ++s) {
      te[s] = round_f32(te[s]);
      tx[s] = round_f32(tx[s]);
    }
    it.rec[i] = r;
  }
  const double t0 = te[mo], t1 = tx[mo];
  it.te[i] = t0;
  it.tx[i] = t1;
  it.t0[i] = ns > 0 ? te[0] : 0.0;
  it.t1[i] = ns > 0 ? tx[ns - 1] : 0.0;
  it.nseg[i] = (uint8_t)ns;
  it.order[i] = (uint8_t)mo;
  it.part[i] = (uint8_t)lp;
  uint8_t* sc = it.sched + (uint64_t)i * kMaxSeg;
  for (int s = 0; s < kMaxSeg; ++s) sc[s] = s < ns ? reg[s] : 0xff;
  for (uint32_t q = 0; q < P; ++q) it.contains[(uint64_t)q * n_items + i] = 0u;
  for (int s = 0; s < ns; ++s)
    if (reg[s] != pd.global_id) it.contains[(uint64_t)reg[s] * n_items + i] = 1u;
  // sample counts of cascade_march
  const double offset = jitter ? dmul(step, counter_uniform(seed, (uint64_t)r.ray_id, batch_id))
                               : dmul(0.5, step);
  uint32_t nf = 0, nc = 0, ncb = 0, nr = 0;
  double fa, fb;
  auto count = [&](double a, double b, int casc) {  // O(1) per occupied run
    const uint32_t k = ladder_count(a, b, t0, t1, offset, step);
    if (casc == 0) {
      nf += k;
    } else {
      nc += k;
      if (nf == 0) ncb += k;
    }
    if (k && nr < (uint32_t)kMaxRuns) {  // the fill kernel replays the runs instead of walking
      it.runs[(uint64_t)i * kMaxRuns + nr] = make_double2(a, b);
      it.run_casc[(uint64_t)i * kMaxRuns + nr] = (uint8_t)casc;
    }
    if (k) ++nr;
  };
  const bool has_fine = cascade_runs(pd, occ, r.o, r.d, t0, t1, fa, fb, count);
  if (!has_fine) ncb = nc;
  it.nrun[i] = nr <= (uint32_t)kMaxRuns ? (uint8_t)nr : kRunsOverflow;
  it.cnt[i] = nf;
  it.cnt[n_items + i] = nc;
  it.ncb[i] = ncb;
}

// One warp per item, replaying the occupied runs recorded by the item setup.  A lane per run
// computes the run's ladder range (first index k0, count n) and warp scans turn the counts
// into output slots (fine and coarse samples keep march order in their own arrays); then the
// item's samples are emitted 32 at a time, each lane locating its run by binary search over
// the run prefix, so long runs (a mostly occupied grid) and many short runs (a fragmented
// one after occupancy updates) both keep every lane busy and the writes coalesce.  Items with
// more than kMaxRuns runs are left to k_march_fill_walk.
__device__ __forceinline__ uint32_t warp_excl_scan_u(uint32_t v) {
  const unsigned lane = threadIdx.x & 31;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  return x - v;
}

constexpr int kFillWarps = 4;

__global__ void __launch_bounds__(32 * kFillWarps) k_march_fill(const PartDesc* __restrict__ parts,
                                                               const uint8_t* __restrict__ occ,
                                                               uint32_t n_items, ItemArrays it,
                                                               SampleArrays sm, double step, uint64_t seed,
                                                               uint64_t batch_id, int jitter, uint32_t n_fine) {
  __shared__ uint32_t s_excl[kFillWarps][kMaxRuns];  // exclusive prefix of the run counts
  __shared__ uint32_t s_out[kFillWarps][kMaxRuns];   // output slot of the run's first sample
  __shared__ long long s_k0[kFillWarps][kMaxRuns];
  __shared__ double s_hi[kFillWarps][kMaxRuns];
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t i = (uint32_t)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const uint32_t lane = threadIdx.x & 31;
  if (i >= n_items) return;  // warp-uniform
  const uint8_t nr = it.nrun[i];
  if (nr == kRunsOverflow) return;  // k_march_fill_walk
  const RayRec& r = it.rec[i];
  const double te = it.te[i], tx = it.tx[i];
  const double offset = jitter ? dmul(step, counter_uniform(seed, (uint64_t)r.ray_id, batch_id))
                               : dmul(0.5, step);
  const double base = dadd(te, offset), half = dmul(0.5, step);
  const uint32_t pf = it.off[i], pc = it.off[n_items + i];
  uint32_t tot = 0, tot_f = 0, tot_c = 0;
  for (uint32_t r0 = 0; r0 < nr; r0 += 32) {
    const uint32_t k = r0 + lane;
    Ladder L{0, 0u, 0.0};
    uint32_t casc = 0;
    if (k < nr) {
      const double2 rr = it.runs[(uint64_t)i * kMaxRuns + k];
      casc = it.run_casc[(uint64_t)i * kMaxRuns + k];
      L = ladder_range(rr.x, rr.y, te, tx, offset, step);
    }
    const uint32_t nf = casc == 0 ? L.n : 0u, nc = casc == 0 ? 0u : L.n;
    const uint32_t ex = warp_excl_scan_u(L.n), exf = warp_excl_scan_u(nf), exc = warp_excl_scan_u(nc);
    if (k < nr) {
      s_excl[w][k] = tot + ex;
      s_out[w][k] = casc == 0 ? pf + tot_f + exf : pc + tot_c + exc;
      s_k0[w][k] = L.k0;
      s_hi[w][k] = L.hi;
    }
    tot += __shfl_sync(0xffffffffu, ex + L.n, 31);
    tot_f += __shfl_sync(0xffffffffu, exf + nf, 31);
    tot_c += __shfl_sync(0xffffffffu, exc + nc, 31);
  }
  __syncwarp();
  for (uint32_t q = lane; q < tot; q += 32) {
    // the run holding q: the last run whose exclusive prefix is <= q (recorded runs are non-empty)
    uint32_t lo = 0, hi = nr;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_excl[w][mid] <= q) lo = mid;
      else hi = mid;
    }
    const uint32_t j = q - s_excl[w][lo];
    const double t = dadd(base, dmul((double)(s_k0[w][lo] + j), step));
    const uint32_t o = s_out[w][lo] + j;
    sm.t[o] = t;
    sm.delta[o] = smin(step, dsub(s_hi[w][lo], dsub(t, half)));
    sm.item[o] = i;
    if (sm.p) {  // the per-sample position cache (normalised once, here, from the same t)
      const PartDesc& pd = parts[it.part[i]];
      const bool coarse = o >= n_fine;
      double pp[3];
      normalized_point(coarse ? pd.coarse_lo : pd.fine_lo, coarse ? pd.coarse_hi : pd.fine_hi, r.o, r.d, t, pp);
      sm.p[o] = pp[0];
      sm.p[sm.pn + o] = pp[1];
      sm.p[2 * sm.pn + o] = pp[2];
    }
  }
}

// Items whose runs overflowed kMaxRuns: one thread per item walks the grid again and emits
// in order (cascade_march, worker.cpp:79-110).
__global__ void k_march_fill_walk(const PartDesc* __restrict__ parts, const uint8_t* __restrict__ occ,
                                  uint32_t n_items, ItemArrays it, SampleArrays sm, double step,
                                  uint64_t seed, uint64_t batch_id, int jitter) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_items || it.nrun[i] != kRunsOverflow) return;
  const PartDesc& pd = parts[it.part[i]];
  const RayRec& r = it.rec[i];
  const double offset = jitter ? dmul(step, counter_uniform(seed, (uint64_t)r.ray_id, batch_id))
                               : dmul(0.5, step);
  uint32_t pf = it.off[i], pc = it.off[n_items + i];
  double fa, fb;
  auto emit = [&](double t, double delta, int casc) {
    const uint32_t s = casc == 0 ? pf++ : pc++;
    sm.t[s] = t;
    sm.delta[s] = delta;
    sm.item[s] = i;
    if (sm.p) {
      double pp[3];
      normalized_point(casc ? pd.coarse_lo : pd.fine_lo, casc ? pd.coarse_hi : pd.fine_hi, r.o, r.d, t, pp);
      sm.p[s] = pp[0];
      sm.p[sm.pn + s] = pp[1];
      sm.p[2 * sm.pn + s] = pp[2];
    }
  };
  cascade_march(pd, occ, r.o, r.d, it.te[i], it.tx[i], step, offset, fa, fb, emit);
}

// Visit an item's samples in t order: coarse-before, fine, coarse-after.
template <class F>
__device__ __forceinline__ void for_item_samples(const ItemArrays& it, uint32_t n_items, uint32_t i,
                                                 F&& f) {
  const uint32_t fo = it.off[i], nf = it.cnt[i];
  const uint32_t co = it.off[n_items + i], nc = it.cnt[n_items + i], ncb = it.ncb[i];
  for (uint32_t k = 0; k < ncb; ++k) f(co + k);
  for (uint32_t k = 0; k < nf; ++k) f(fo + k);
  for (uint32_t k = ncb; k < nc; ++k) f(co + k);
}

template <class F>
__device__ __forceinline__ void for_item_samples_rev(const ItemArrays& it, uint32_t n_items,
                                                     uint32_t i, F&& f) {
  const uint32_t fo = it.off[i], nf = it.cnt[i];
  const uint32_t co = it.off[n_items + i], nc = it.cnt[n_items + i], ncb = it.ncb[i];
  for (uint32_t k = nc; k-- > ncb;) f(co + k);
  for (uint32_t k = nf; k-- > 0;) f(fo + k);
  for (uint32_t k = ncb; k-- > 0;) f(co + k);
}

__global__ void k_composite(uint32_t n_items, ItemArrays it, SampleArrays sm, int with_depth) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  float T = 1.0f, tau = 0.0f, r = 0.0f, g = 0.0f, b = 0.0f, dep = 0.0f;
  // distortion aggregates for the cross-segment correction (local_distortion_inputs,
  // worker.cpp:62-75, and loss_distortion, train.cpp:38-57): s, ds on the ray's [t0, t1]
  const bool xd = it.xdist != nullptr;
  const double ray_t0 = xd ? it.t0[i] : 0.0;
  const float inv_span = xd ? (float)(1.0 / (it.t1[i] - ray_t0)) : 0.0f;
  float Wp = 0.0f, Mp = 0.0f, pair = 0.0f, interval = 0.0f;
  for_item_samples(it, n_items, i, [&](uint32_t s) {
    const float4 o = sm.out[s];
    const float x = o.x * (float)sm.delta[s];
    const float alpha = -expm1f(-x);
    const float w = T * alpha;
    r = fmaf(o.y, w, r);
    g = fmaf(o.z, w, g);
    b = fmaf(o.w, w, b);
    if (with_depth) dep = fmaf(w, (float)sm.t[s], dep);
    if (xd) {
      const float ss = (float)(sm.t[s] - ray_t0) * inv_span;
      const float ds = (float)sm.delta[s] * inv_span;
      pair += 2.0f * w * (ss * Wp - Mp);
      interval += w * w * ds;
      Wp += w;
      Mp += w * ss;
    }
    T *= expf(-x);
    tau += x;
  });
  it.partial[i] = make_float4(r, g, b, tau);
  it.depth[i] = dep;
  if (xd) it.xdist[i] = make_float4(Wp, Mp, pair + interval / 3.0f, 0.0f);
}

__device__ __forceinline__ uint32_t ordinal(const ItemArrays& it, uint32_t n_items,
                                            const uint32_t* part_item_off, uint32_t lp, uint32_t q,
                                            uint32_t i) {
  const uint64_t row = (uint64_t)q * n_items;
  return it.cscan[row + i] - it.cscan[row + part_item_off[lp]];
}

__global__ void k_pack_partials(uint32_t n_items, ItemArrays it, const uint32_t* __restrict__ part_item_off,
                                const uint8_t* __restrict__ global_of_local,
                                const uint64_t* __restrict__ stream_off, uint32_t P,
                                PartialRec* __restrict__ send, float4* __restrict__ send_x,
                                PeerDst peer, PeerDst peer_x) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const uint32_t lp = it.part[i];
  const uint32_t gid = global_of_local[lp];
  const int ns = it.nseg[i];
  if (ns <= 1) return;
  const float4 pr = it.partial[i];
  PartialRec rec;
  rec.rgb[0] = pr.x;
  rec.rgb[1] = pr.y;
  rec.rgb[2] = pr.z;
  rec.tau = pr.w;
  rec.depth = it.depth[i];
  rec.ray_id = it.rec[i].ray_id;
  const uint8_t* sc = it.sched + (uint64_t)i * kMaxSeg;
  const bool cross = send_x || peer_x.base;
  const float4 x = cross ? it.xdist[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = 0; s < ns; ++s) {
    const uint32_t q = sc[s];
    if (q == gid) continue;
    // stream (gid -> q) starts at stream_off: in the local send buffer, or (peer mode) in the
    // receive buffer of q's owner, written there directly
    const uint64_t at = stream_off[gid * P + q] + ordinal(it, n_items, part_item_off, lp, q, i);
    if (peer.base) {
      static_cast<PartialRec*>(peer.base[q % peer.world])[at] = rec;
      if (peer_x.base) static_cast<float4*>(peer_x.base[q % peer.world])[at] = x;
    } else {
      send[at] = rec;
      if (send_x) send_x[at] = x;
    }
  }
  if (peer.base) __threadfence_system();
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// exclusive prefix sum over lanes (lane 0 gets 0)
__device__ __forceinline__ float warp_excl_scan(float v) {
  const unsigned lane = threadIdx.x & 31;
  float x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  return x - v;
}
// exclusive suffix sum over lanes (lane 31 gets 0)
__device__ __forceinline__ float warp_excl_rscan(float v) {
  const unsigned lane = threadIdx.x & 31;
  float x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_down_sync(0xffffffffu, x, o);
    if (lane + o < 32) x += y;
  }
  return x - v;
}


__global__ void k_merge_backward(uint32_t n_items, ItemArrays it,
                                 const uint32_t* __restrict__ part_item_off,
                                 const PartDesc* __restrict__ parts,
                                 const uint64_t* __restrict__ stream_off, uint32_t P,
                                 const PartialRec* __restrict__ recv, const float4* __restrict__ recv_x,
                                 SampleArrays sm, double lambda_t, double lambda_d, double t_clamp,
                                 int wire_f32, LossAccum* __restrict__ loss) {
  // one warp per item: the per-item merge is computed by every lane (broadcast loads), the
  // per-sample passes run 32 samples at a time with warp scans
  const uint32_t i = (uint32_t)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const uint32_t lane = threadIdx.x & 31;
  double l_rgb = 0.0, l_t = 0.0, l_d = 0.0;
  uint32_t lp = 0;
  if (i < n_items) {
    lp = it.part[i];
    const uint32_t gid = parts[lp].global_id;
    const int ns = it.nseg[i];
    const int mo = it.order[i];
    const RayRec& rr = it.rec[i];
    const uint8_t* sc = it.sched + (uint64_t)i * kMaxSeg;
    double pc[kMaxSeg][3], pT[kMaxSeg], tau_tot = 0.0;
    double xW[kMaxSeg], xM[kMaxSeg], xD[kMaxSeg];  // cross-correction aggregates per segment
    const bool cross = it.xdist != nullptr;
    bool bad = false;
    for (int s = 0; s < ns; ++s) {
      float4 v, xv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (s == mo) {
        v = it.partial[i];
        if (cross) xv = it.xdist[i];
      } else {
        const uint32_t q = sc[s];
        const uint64_t at = stream_off[q * P + gid] + ordinal(it, n_items, part_item_off, lp, q, i);
        const PartialRec rec = recv[at];
        if (rec.ray_id != rr.ray_id) bad = true;
        v = make_float4(rec.rgb[0], rec.rgb[1], rec.rgb[2], rec.tau);
        if (cross) xv = recv_x[at];
      }
      xW[s] = xv.x;
      xM[s] = xv.y;
      xD[s] = xv.z;
      pc[s][0] = v.x;
      pc[s][1] = v.y;
      pc[s][2] = v.z;
      // wire_f32: the reference merges float-rounded T (quantize_partial, wire.cpp:207-217)
      pT[s] = wire_f32 ? (double)(float)exp(-(double)v.w) : exp(-(double)v.w);
      tau_tot += v.w;
    }
    if (bad) atomicOr(&loss->error, 2u);  // "missing partial" (worker.cpp:371-376)
    // merge_forward (render.cpp:101-116)
    double C[3] = {0.0, 0.0, 0.0}, prefix = 1.0;
    double pre[kMaxSeg + 1];
    for (int s = 0; s < ns; ++s) {
      pre[s] = prefix;
      for (int a = 0; a < 3; ++a) C[a] += pc[s][a] * prefix;
      prefix *= pT[s];
    }
    pre[ns] = prefix;
    const double T = prefix;
    const double gt[3] = {rr.gt[0], rr.gt[1], rr.gt[2]};
    // 1 - min(T, 1 - eps) (train.cpp:20-33); 1 - T from the optical depth when T -> 1
    const double one_minus_T = wire_f32 ? 1.0 - T : -expm1(-tau_tot);
    const double omc = (1.0 - t_clamp < T) ? 1.0 - (1.0 - t_clamp) : one_minus_T;
    if (sc[0] == gid) {  // first owner reports (worker.cpp:409-416)
      for (int a = 0; a < 3; ++a) l_rgb += (C[a] - gt[a]) * (C[a] - gt[a]);
      l_t = -log(omc);
    }
    double up_c[3];
    for (int a = 0; a < 3; ++a) up_c[a] = (C[a] - gt[a]) * 2.0;
    const double up_t = lambda_t * (1.0 / omc);
    // merge_backward for my segment (render.cpp:118-143)
    double suffix = 1.0;
    for (int s = ns - 1; s > mo; --s) suffix *= pT[s];
    double g_c[3];
    for (int a = 0; a < 3; ++a) g_c[a] = up_c[a] * pre[mo];
    double running = 1.0, color_term = 0.0;
    for (int k = mo + 1; k < ns; ++k) {
      color_term += running * (up_c[0] * pc[k][0] + up_c[1] * pc[k][1] + up_c[2] * pc[k][2]);
      running *= pT[k];
    }
    double g_t = up_t * pre[mo] * suffix + pre[mo] * color_term;
    // cross-segment distortion (worker.cpp:453-511): ray-level loss at the first owner, the
    // cross terms of my samples' weight gradient, and d L / d T_mine through later prefixes
    double lw = 0.0, lm = 0.0, ew = 0.0, em = 0.0, l_full = 0.0;
    if (cross) {
      if (sc[0] == gid) {
        for (int m = 0; m < ns; ++m) l_full += pre[m] * pre[m] * xD[m];
        for (int a = 0; a < ns; ++a)
          for (int m = a + 1; m < ns; ++m) l_full += 2.0 * pre[a] * pre[m] * (xW[a] * xM[m] - xM[a] * xW[m]);
      }
      if (lambda_d > 0.0) {
        for (int m = 0; m < ns; ++m) {
          if (m > mo) {
            lw += pre[m] * xW[m];
            lm += pre[m] * xM[m];
          } else if (m < mo) {
            ew += pre[m] * xW[m];
            em += pre[m] * xM[m];
          }
        }
        double t_grad = 0.0;
        for (int m = mo + 1; m < ns; ++m) {
          double dl = 2.0 * pre[m] * xD[m];
          for (int a = 0; a < m; ++a) dl += 2.0 * pre[a] * (xW[a] * xM[m] - xM[a] * xW[m]);
          for (int m2 = m + 1; m2 < ns; ++m2) dl += 2.0 * pre[m2] * (xW[m] * xM[m2] - xM[m] * xW[m2]);
          double prod_excl = 1.0;
          for (int j = 0; j < m; ++j)
            if (j != mo) prod_excl *= pT[j];
          t_grad += dl * prod_excl;
        }
        g_t += lambda_d * t_grad;
      }
    }
    // local forward recompute: prefix per sample, distortion totals (worker.cpp:435-451)
    const double ray_t0 = it.t0[i];
    const float inv_span = (float)(1.0 / (it.t1[i] - ray_t0));
    const uint32_t fo = it.off[i], nf = it.cnt[i];
    const uint32_t co = it.off[n_items + i], nc = it.cnt[n_items + i], ncb = it.ncb[i];
    const uint32_t n = nf + nc;
    auto sample_at = [&](uint32_t j) {  // t order: coarse-before, fine, coarse-after
      return j < ncb ? co + j : (j < ncb + nf ? fo + (j - ncb) : co + j - nf);
    };
    float cx = 0.0f, cW = 0.0f, cM = 0.0f, pair = 0.0f, interval = 0.0f;
    for (uint32_t jb = 0; jb < n; jb += 32) {
      const uint32_t j = jb + lane;
      const bool v = j < n;
      const uint32_t s = v ? sample_at(j) : 0u;
      const float x = v ? sm.out[s].x * (float)sm.delta[s] : 0.0f;
      const float ex_x = warp_excl_scan(x);
      const float Tl = expf(-(cx + ex_x));
      const float alpha = -expm1f(-x);
      const float w = v ? Tl * alpha : 0.0f;
      const float ss = v ? (float)((sm.t[s] - ray_t0)) * inv_span : 0.0f;
      const float ds = v ? (float)sm.delta[s] * inv_span : 0.0f;
      const float Wp = cW + warp_excl_scan(w), Mp = cM + warp_excl_scan(w * ss);
      pair += 2.0f * w * (ss * Wp - Mp);
      interval += w * w * ds;
      if (v) sm.grad[s] = make_float4(Tl, 0.f, 0.f, 0.f);  // stash prefix for the reverse sweep
      cx += warp_sum_f(x);
      cW += warp_sum_f(w);
      cM += warp_sum_f(w * ss);
    }
    const float Wt = cW, Mt = cM;
    pair = warp_sum_f(pair);
    interval = warp_sum_f(interval);
    if (cross) l_d = l_full;  // only the first owner reports, the whole ray
    else if (n > 0) l_d = (double)(pair + interval / 3.0f);
    const float xp = (float)pre[mo], xlw = (float)lw, xlm = (float)lm, xew = (float)ew, xem = (float)em;
    // reverse sweep: local_render_backward with the distortion weight channel (render.cpp:145-179);
    // suffix sums by reverse warp scans, the tail colour recurrence c <- alpha u + om c as an
    // affine-map suffix scan
    const float ucx = (float)g_c[0], ucy = (float)g_c[1], ucz = (float)g_c[2];
    const float ut = (float)g_t;
    const float ld = (float)lambda_d;
    float cWs = 0.0f, cMs = 0.0f, cxs = 0.0f, ctc = 0.0f;
    if (n > 0) {
      for (int64_t jb = (int64_t)((n - 1) / 32) * 32; jb >= 0; jb -= 32) {
        const uint32_t j = (uint32_t)jb + lane;
        const bool v = j < n;
        const uint32_t s = v ? sample_at(j) : 0u;
        const float4 o = v ? sm.out[s] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float delta = v ? (float)sm.delta[s] : 0.0f;
        const float x = o.x * delta;
        const float alpha = -expm1f(-x);
        const float om = v ? expf(-x) : 1.0f;
        const float pf = v ? sm.grad[s].x : 0.0f;
        const float w = pf * alpha;
        const float ss = v ? (float)((sm.t[s] - ray_t0)) * inv_span : 0.0f;
        const float ds = delta * inv_span;
        const float Ws = cWs + warp_excl_rscan(w), Ms = cMs + warp_excl_rscan(w * ss);
        const float tail_t = expf(-(cxs + warp_excl_rscan(x)));
        float wup = 0.0f;
        if (ld > 0.0f) {
          const float Wl = Wt - Ws - w, Ml = Mt - Ms - w * ss;
          const float gd = 2.0f * (ss * Wl - Ml) + 2.0f * (Ms - ss * Ws) + (2.0f / 3.0f) * w * ds;
          wup = cross ? ld * (xp * xp * gd + 2.0f * xp * (xlm - ss * xlw + ss * xew - xem)) : ld * gd;
        }
        const float u = ucx * o.y + ucy * o.z + ucz * o.w + wup;
        // suffix composition of c -> a c + b (a = om, b = alpha u) over the later lanes
        float A = om, B = v ? alpha * u : 0.0f;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const float A2 = __shfl_down_sync(0xffffffffu, A, off), B2 = __shfl_down_sync(0xffffffffu, B, off);
          if (lane + off < 32) {
            B = A * B2 + B;
            A = A * A2;
          }
        }
        float An = __shfl_down_sync(0xffffffffu, A, 1), Bn = __shfl_down_sync(0xffffffffu, B, 1);
        if (lane == 31) {
          An = 1.0f;
          Bn = 0.0f;
        }
        const float tail_c = An * ctc + Bn;
        const float alpha_grad = pf * (u - tail_c) - ut * pf * tail_t;
        const float dsig = alpha_grad * delta * om;
        const float cw = pf * alpha;
        if (v) {
          const float4 g = make_float4(dsig, ucx * cw, ucy * cw, ucz * cw);
          if (sm.inv) sm.grad_ord[sm.inv[s]] = g;  // the MLP backward reads it in sample order
          else sm.grad[s] = g;
        }
        ctc = __shfl_sync(0xffffffffu, A, 0) * ctc + __shfl_sync(0xffffffffu, B, 0);
        cWs += warp_sum_f(w);
        cMs += warp_sum_f(w * ss);
        cxs += warp_sum_f(x);
      }
    }
  }
  // per-partition loss sums: lane 0 of each item's warp; items of a block share a partition
  // almost always, so one atomic per block and partition
  __shared__ double red[3][4];
  __shared__ uint32_t red_lp[4];
  const uint32_t wib = threadIdx.x >> 5;  // 4 warps (items) per block
  if (lane == 0) {
    red[0][wib] = i < n_items ? l_rgb : 0.0;
    red[1][wib] = i < n_items ? l_t : 0.0;
    red[2][wib] = i < n_items ? l_d : 0.0;
    red_lp[wib] = i < n_items ? lp : 0xffffffffu;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int a = 0; a < 4; ++a) {
      if (red_lp[a] == 0xffffffffu) continue;
      double x0 = red[0][a], x1 = red[1][a], x2 = red[2][a];
      for (int b = a + 1; b < 4; ++b)
        if (red_lp[b] == red_lp[a]) {
          x0 += red[0][b];
          x1 += red[1][b];
          x2 += red[2][b];
          red_lp[b] = 0xffffffffu;
        }
      atomicAdd(&loss->rgb[red_lp[a]], x0);
      atomicAdd(&loss->trans[red_lp[a]], x1);
      atomicAdd(&loss->dist[red_lp[a]], x2);
    }
  }
}

__global__ void k_pair_counts(uint32_t n_items, uint32_t n_local, uint32_t P,
                              const uint32_t* __restrict__ part_item_off,
                              const uint32_t* __restrict__ cscan, uint32_t* __restrict__ out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_local * P) return;
  const uint32_t lp = t / P, q = t % P;
  const uint64_t row = (uint64_t)q * n_items;
  out[t] = cscan[row + part_item_off[lp + 1]] - cscan[row + part_item_off[lp]];
}

// dispatch_eval's driver merge in schedule order (worker.cpp:801-826): optional early
// termination once the running transmittance drops below the threshold (the crossing entry
// is kept, worker.cpp:815-818) and the region-attribution colour of evaluate_image
// (worker.cpp:864-878) over the merged entries.
__global__ void k_home_merge(uint64_t n, const uint8_t* __restrict__ nseg,
                             const uint8_t* __restrict__ sched, const uint8_t* __restrict__ slot_of_part,
                             const uint32_t* __restrict__ pos, const float4* __restrict__ partial,
                             const float* __restrict__ depth, const PartialRec* __restrict__ reply,
                             float* __restrict__ rgb, float* __restrict__ trans,
                             float* __restrict__ depth_out, int early_term, double term_thr,
                             float* __restrict__ attribution) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int ns = nseg[i];
  double C[3] = {0.0, 0.0, 0.0}, prefix = 1.0, dep = 0.0, at[3] = {0.0, 0.0, 0.0};
  for (int s = 0; s < ns; ++s) {
    const uint32_t p = sched[i * kMaxSeg + s];
    const uint32_t idx = pos[(uint64_t)slot_of_part[p] * n + i];
    float4 v;
    float dp;
    if (reply) {
      const PartialRec r = reply[idx];
      v = make_float4(r.rgb[0], r.rgb[1], r.rgb[2], r.tau);
      dp = r.depth;
    } else {
      v = partial[idx];
      dp = depth[idx];
    }
    C[0] += v.x * prefix;
    C[1] += v.y * prefix;
    C[2] += v.z * prefix;
    dep += dp * prefix;
    const double Ts = exp(-(double)v.w);
    if (attribution) {
      const double w = prefix * (1.0 - Ts), hue = (double)p * 0.61803398875;
      at[0] += (0.5 + 0.5 * cos(6.2831853 * hue)) * w;
      at[1] += (0.5 + 0.5 * cos(6.2831853 * (hue + 1.0 / 3.0))) * w;
      at[2] += (0.5 + 0.5 * cos(6.2831853 * (hue + 2.0 / 3.0))) * w;
    }
    prefix *= Ts;
    if (early_term && prefix < term_thr) break;
  }
  rgb[3 * i] = (float)C[0];
  rgb[3 * i + 1] = (float)C[1];
  rgb[3 * i + 2] = (float)C[2];
  trans[i] = (float)prefix;
  depth_out[i] = (float)dep;
  if (attribution) {
    attribution[3 * i] = (float)at[0];
    attribution[3 * i + 1] = (float)at[1];
    attribution[3 * i + 2] = (float)at[2];
  }
}

// evaluate_image ray generation (worker.cpp:841-853): pixel (x, y) of one camera, row-major.
__global__ void k_camera_rays(const double* __restrict__ pose, uint32_t width, uint64_t n,
                              double* __restrict__ o, double* __restrict__ d) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t x = (uint32_t)(i % width), y = (uint32_t)(i / width);
  // pose: R[9], t[3], fx, fy, cx, cy
  double R[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = pose[k];
  double dd[3];
  pixel_ray_dir(R, pose[12], pose[13], pose[14], pose[15], dadd((double)x, 0.5), dadd((double)y, 0.5), dd);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    o[3 * i + a] = pose[9 + a];
    d[3 * i + a] = dd[a];
  }
}

__global__ void k_segment_full(const Geo* __restrict__ geo, const double* __restrict__ o,
                               const double* __restrict__ d, uint64_t n, uint8_t* __restrict__ nseg,
                               uint8_t* __restrict__ sched, double* __restrict__ te,
                               double* __restrict__ tx) {
  __shared__ Geo sg;
  load_geo(sg, geo);
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]};
  double dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
  uint8_t reg[kMaxSeg];
  double a[kMaxSeg], b[kMaxSeg];
  const int ns = segment_ray(sg, oo, dd, reg, a, b);
  nseg[i] = (uint8_t)ns;
  for (int s = 0; s < kMaxSeg; ++s) {
    sched[i * kMaxSeg + s] = s < ns ? reg[s] : 0xff;
    te[i * kMaxSeg + s] = s < ns ? a[s] : 0.0;
    tx[i * kMaxSeg + s] = s < ns ? b[s] : 0.0;
  }
}

__global__ void k_u8_to_u16(const uint8_t* in, uint16_t* out, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] == 0xff ? 0 : in[i];
}

__global__ void k_march_points(const PartDesc* __restrict__ part, const uint8_t* __restrict__ occ,
                               const double* __restrict__ o, const double* __restrict__ d,
                               const double* __restrict__ t0, const double* __restrict__ t1,
                               const uint64_t* __restrict__ ray_id, uint64_t n, double step,
                               uint64_t seed, uint64_t batch_id, int jitter,
                               uint32_t* __restrict__ counts, const uint64_t* __restrict__ offsets,
                               double* __restrict__ t, double* __restrict__ delta,
                               uint8_t* __restrict__ cascade) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]};
  const double dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
  const double offset = jitter ? dmul(step, counter_uniform(seed, ray_id[i], batch_id)) : dmul(0.5, step);
  double fa, fb;
  uint32_t k = 0;
  const uint64_t base = offsets ? offsets[i] : 0;
  auto emit = [&](double tt, double dl, int casc) {
    if (t) {
      t[base + k] = tt;
      delta[base + k] = dl;
      cascade[base + k] = (uint8_t)casc;
    }
    ++k;
  };
  cascade_march(*part, occ, oo, dd, t0[i], t1[i], step, offset, fa, fb, emit);
  if (!t) counts[i] = k;
}

__global__ void k_items_to_records(uint32_t n, const float4* __restrict__ partial,
                                   const float* __restrict__ depth, const RayRec* __restrict__ rec,
                                   PartialRec* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 v = partial[i];
  PartialRec r;
  r.rgb[0] = v.x;
  r.rgb[1] = v.y;
  r.rgb[2] = v.z;
  r.tau = v.w;
  r.depth = depth[i];
  r.ray_id = rec[i].ray_id;
  out[i] = r;
}

inline unsigned blocks(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void launch_segment_home(const Geo* geo, const double* o, const double* d, uint64_t n,
                         const uint8_t* slot_of_part, uint8_t* nseg, uint8_t* sched,
                         uint32_t* flags, unsigned long long* dropped, cudaStream_t s) {
  if (!n) return;
  k_segment_home<<<blocks(n, 128), 128, 0, s>>>(geo, o, d, n, slot_of_part, nseg, sched, flags,
                                                 dropped);
}

void launch_pack_dispatch(uint64_t n, uint32_t, const uint8_t* nseg, const uint8_t* sched,
                          const uint8_t* slot_of_part, const uint32_t* pos, const double* o,
                          const double* d, const float* gt, const uint32_t* img,
                          uint64_t first_ray_id, RayRec* out, PeerDst peer, cudaStream_t s) {
  if (!n) return;
  k_pack_dispatch<<<blocks(n, 256), 256, 0, s>>>(n, nseg, sched, slot_of_part, pos, o, d, gt, img,
                                                 first_ray_id, out, peer);
}

void launch_item_setup(const Geo* geo, const PartDesc* parts, const uint8_t* occ,
                       const uint32_t* part_item_off, uint32_t n_local, uint32_t n_items,
                       ItemArrays it, uint32_t P, double step, uint64_t seed, uint64_t batch_id,
                       int jitter, int wire_f32, uint32_t n_images, uint32_t* error,
                       cudaStream_t s) {
  if (!n_items) return;
  k_item_setup<<<blocks(n_items, 128), 128, 0, s>>>(geo, parts, occ, part_item_off, n_local,
                                                    n_items, it, P, step, seed, batch_id, jitter,
                                                    wire_f32, n_images, error);
}

void launch_march_fill(const PartDesc* parts, const uint8_t* occ, uint32_t n_items,
                       ItemArrays it, SampleArrays sm, uint32_t n_fine, double step, uint64_t seed,
                       uint64_t batch_id, int jitter, cudaStream_t s) {
  if (!n_items) return;
  k_march_fill<<<blocks((uint64_t)n_items * 32, 32 * kFillWarps), 32 * kFillWarps, 0, s>>>(
      parts, occ, n_items, it, sm, step, seed, batch_id, jitter, n_fine);
  k_march_fill_walk<<<blocks(n_items, 128), 128, 0, s>>>(parts, occ, n_items, it, sm, step, seed, batch_id,
                                                         jitter);
}

void launch_composite(uint32_t n_items, ItemArrays it, SampleArrays sm, uint32_t,
                      int with_depth, cudaStream_t s) {
  if (!n_items) return;
  k_composite<<<blocks(n_items, 128), 128, 0, s>>>(n_items, it, sm, with_depth);
}

void launch_pack_partials(uint32_t n_items, ItemArrays it, const uint32_t* part_item_off,
                          const uint8_t* global_of_local, const uint64_t* stream_off, uint32_t P,
                          PartialRec* send, float4* send_x, PeerDst peer, PeerDst peer_x,
                          cudaStream_t s) {
  if (!n_items) return;
  k_pack_partials<<<blocks(n_items, 256), 256, 0, s>>>(n_items, it, part_item_off, global_of_local,
                                                       stream_off, P, send, send_x, peer, peer_x);
}

void launch_merge_backward(uint32_t n_items, ItemArrays it, const uint32_t* part_item_off,
                           const PartDesc* parts, const uint64_t* stream_off, uint32_t P,
                           const PartialRec* recv, const float4* recv_x, SampleArrays sm, uint32_t,
                           double lambda_t, double lambda_d, double t_clamp, int wire_f32,
                           LossAccum* loss, cudaStream_t s) {
  if (!n_items) return;
  k_merge_backward<<<blocks((uint64_t)n_items * 32, 128), 128, 0, s>>>(n_items, it, part_item_off, parts,
                                                        stream_off, P, recv, recv_x, sm, lambda_t,
                                                        lambda_d, t_clamp, wire_f32, loss);
}

void launch_pair_counts(uint32_t n_items, uint32_t n_local, uint32_t P, const uint32_t* part_item_off,
                        const uint32_t*, const uint32_t* cscan, uint32_t* out, cudaStream_t s) {
  k_pair_counts<<<blocks((uint64_t)n_local * P, 128), 128, 0, s>>>(n_items, n_local, P,
                                                                   part_item_off, cscan, out);
}

void launch_home_merge(uint64_t n, uint32_t, const uint8_t* nseg, const uint8_t* sched,
                       const uint8_t* slot_of_part, const uint32_t* pos, const float4* partial,
                       const float* depth, const PartialRec* reply, int, float* rgb, float* trans,
                       float* depth_out, int early_term, double term_thr, float* attribution,
                       cudaStream_t s) {
  if (!n) return;
  k_home_merge<<<blocks(n, 256), 256, 0, s>>>(n, nseg, sched, slot_of_part, pos, partial, depth,
                                              reply, rgb, trans, depth_out, early_term, term_thr,
                                              attribution);
}

void launch_camera_rays(const double* pose, uint32_t width, uint64_t n, double* o, double* d,
                        cudaStream_t s) {
  if (!n) return;
  k_camera_rays<<<blocks(n, 128), 128, 0, s>>>(pose, width, n, o, d);
}

void launch_segment_full(const Geo* geo, const double* o, const double* d, uint64_t n, uint8_t* nseg,
                         uint8_t* sched, double* te, double* tx, cudaStream_t s) {
  if (!n) return;
  k_segment_full<<<blocks(n, 128), 128, 0, s>>>(geo, o, d, n, nseg, sched, te, tx);
}

void launch_u8_to_u16(const uint8_t* in, uint16_t* out, uint64_t n, cudaStream_t s) {
  if (!n) return;
  k_u8_to_u16<<<blocks(n, 256), 256, 0, s>>>(in, out, n);
}

void launch_march_points(const PartDesc* part, const uint8_t* occ, const double* o, const double* d,
                         const double* t0, const double* t1, const uint64_t* ray_id, uint64_t n,
                         double step, uint64_t seed, uint64_t batch_id, int jitter, uint32_t* counts,
                         const uint64_t* offsets, double* t, double* delta, uint8_t* cascade,
                         cudaStream_t s) {
  if (!n) return;
  k_march_points<<<blocks(n, 128), 128, 0, s>>>(part, occ, o, d, t0, t1, ray_id, n, step, seed,
                                                batch_id, jitter, counts, offsets, t, delta, cascade);
}

void launch_items_to_records(uint32_t n, const float4* partial, const float* depth, const RayRec* rec,
                             PartialRec* out, cudaStream_t s) {
  if (!n) return;
  k_items_to_records<<<blocks(n, 256), 256, 0, s>>>(n, partial, depth, rec, out);
}

}  // namespace dg
