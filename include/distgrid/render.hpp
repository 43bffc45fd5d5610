// distgrid/render.hpp — the segmented renderer of the reference API (render.hpp:13-117):
// march_segment, local_render (+ accumulate_distortion_stats), merge_forward / merge_backward
// and local_render_backward with the reference's types and exceptions.  Each call runs the
// device kernels of kernels_render_api.cu / kernels_stage_api.cu (fp64 arithmetic in the
// reference's order, fp64 in and out: the *_f64 C-ABI entry points); the batched overloads
// at the end do a whole batch of segments / rays per launch.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "distgrid/detail/device.hpp"
#include "distgrid/geometry.hpp"
#include "distgrid/grid.hpp"
#include "distgrid/vecmath.hpp"

namespace distgrid {

struct RaySegment {
  uint64_t ray_id = 0;
  uint32_t region_id = 0;
  uint32_t order_index = 0;  // position of the segment along its ray
  double t_enter = 0.0;
  double t_exit = 0.0;
};

// What one region contributes to one ray (exchanged in training: color + transmittance).
struct PartialRender {
  uint64_t ray_id = 0;
  uint32_t region_id = 0;
  Vec3 color;
  double transmittance = 1.0;
  double depth_sum = 0.0;         // sum of w_k t_k (evaluation)
  double weight_sum = 0.0;        // distortion aggregates (accumulate_distortion_stats)
  double weight_moment = 0.0;
  double distortion_local = 0.0;
};

struct MergedRender {
  uint64_t ray_id = 0;
  Vec3 color;
  double transmittance = 1.0;
  double depth = 0.0;
};

struct MarchSample {
  double t = 0.0;      // midpoint
  double delta = 0.0;  // covered length
};

struct MarchConfig {
  double step = 0.0;
  bool jitter = false;      // training: offset = step * counter_uniform(seed, ray, step index)
  uint64_t jitter_seed = 0;
  uint64_t jitter_step = 0;
};

struct ShadedSample {
  double sigma = 0.0;
  Vec3 color;
};

struct LocalRenderCache {
  std::vector<double> alpha;
  std::vector<double> prefix;  // transmittance in front of each sample, within the segment
};

struct MergeGrad {
  Vec3 color_grad;
  double transmittance_grad = 0.0;
};

namespace rdetail {
static_assert(sizeof(Vec3) == 24 && sizeof(MarchSample) == 16 && sizeof(ShadedSample) == 32,
              "packed layouts");
inline const double* dp(const void* p) { return static_cast<const double*>(p); }

// Split AoS samples / shading into the SoA arrays the kernels take.
struct SampleSoa {
  std::vector<double> t, delta, sigma, rgb;
  SampleSoa(std::span<const MarchSample> s, std::span<const ShadedSample> sh) {
    const size_t n = s.size();
    t.resize(n);
    delta.resize(n);
    sigma.resize(n);
    rgb.resize(3 * n);
    for (size_t k = 0; k < n; ++k) {
      t[k] = s[k].t;
      delta[k] = s[k].delta;
      sigma[k] = sh[k].sigma;
      rgb[3 * k] = sh[k].color.x;
      rgb[3 * k + 1] = sh[k].color.y;
      rgb[3 * k + 2] = sh[k].color.z;
    }
  }
};
}  // namespace rdetail

// ---- march_segment (render.cpp:10-37) --------------------------------------------------
// Batched: segment g spans [t_enter, t_exit) of segments[g] with occupied[g] as its intervals.
inline std::vector<std::vector<MarchSample>> march_segments(std::span<const RaySegment> segments,
                                                            std::span<const std::vector<RayInterval>> occupied,
                                                            const MarchConfig& config) {
  if (segments.size() != occupied.size()) throw std::invalid_argument("march: size mismatch");
  if (!(config.step > 0.0)) throw std::invalid_argument("march: step must be positive");
  const size_t n = segments.size();
  std::vector<double> te(n), tx(n), iv;
  std::vector<uint64_t> iv_off(n + 1, 0), rid(n), off(n + 1, 0);
  for (size_t g = 0; g < n; ++g) {
    te[g] = segments[g].t_enter;
    tx[g] = segments[g].t_exit;
    rid[g] = segments[g].ray_id;
    for (const RayInterval& r : occupied[g]) {
      iv.push_back(r.t_near);
      iv.push_back(r.t_far);
    }
    iv_off[g + 1] = iv.size() / 2;
  }
  std::vector<uint32_t> cnt(n);
  dg_ctx* c = detail::stage_ctx();
  const int32_t jit = config.jitter ? 1 : 0;
  detail::check(dg_march_segment(c, te.data(), tx.data(), iv_off.data(), iv.data(), rid.data(), n, config.step,
                                 jit, config.jitter_seed, config.jitter_step, cnt.data(), nullptr, nullptr,
                                 nullptr, DG_MEM_HOST));
  for (size_t g = 0; g < n; ++g) off[g + 1] = off[g] + cnt[g];
  std::vector<double> t(off[n]), dl(off[n]);
  if (off[n])
    detail::check(dg_march_segment(c, te.data(), tx.data(), iv_off.data(), iv.data(), rid.data(), n,
                                   config.step, jit, config.jitter_seed, config.jitter_step, nullptr, off.data(),
                                   t.data(), dl.data(), DG_MEM_HOST));
  std::vector<std::vector<MarchSample>> out(n);
  for (size_t g = 0; g < n; ++g)
    for (uint64_t k = off[g]; k < off[g + 1]; ++k) out[g].push_back({t[k], dl[k]});
  return out;
}

inline std::vector<MarchSample> march_segment(double t_enter, double t_exit, std::span<const RayInterval> occupied,
                                              const MarchConfig& config, uint64_t ray_id) {
  RaySegment s;
  s.ray_id = ray_id;
  s.t_enter = t_enter;
  s.t_exit = t_exit;
  const std::vector<RayInterval> iv(occupied.begin(), occupied.end());
  return march_segments(std::span<const RaySegment>(&s, 1), std::span<const std::vector<RayInterval>>(&iv, 1),
                        config)[0];
}

// Convenience overload walking one occupancy grid (render.cpp:39-44): occupancy_skip, then the
// ladder, both on the device.
inline std::vector<MarchSample> march_segment(const Ray& ray, const RaySegment& segment, const OccupancyGrid& occ,
                                              const MarchConfig& config) {
  const std::vector<RayInterval> iv = occupancy_skip(ray, segment.t_enter, segment.t_exit, occ);
  return march_segment(segment.t_enter, segment.t_exit, iv, config, segment.ray_id);
}

// ---- local_render (render.cpp:46-78) + accumulate_distortion_stats (80-99) ---------------
inline PartialRender local_render(uint64_t ray_id, uint32_t region_id, std::span<const MarchSample> samples,
                                  std::span<const ShadedSample> shaded, LocalRenderCache* cache = nullptr) {
  if (samples.size() != shaded.size()) throw std::invalid_argument("render: sample/shading size mismatch");
  const size_t n = samples.size();
  const rdetail::SampleSoa soa(samples, shaded);
  const uint64_t off[2] = {0, n};
  double rgb[3], T, depth;
  std::vector<double> cc(cache ? 2 * n : 0);
  detail::check(dg_local_render_f64(detail::stage_ctx(), soa.t.data(), soa.delta.data(), soa.sigma.data(),
                                    soa.rgb.data(), off, 1, nullptr, nullptr, rgb, &T, &depth, nullptr,
                                    cache ? cc.data() : nullptr, DG_MEM_HOST));
  if (cache) {
    cache->alpha.resize(n);
    cache->prefix.resize(n);
    for (size_t k = 0; k < n; ++k) {
      cache->alpha[k] = cc[2 * k];
      cache->prefix[k] = cc[2 * k + 1];
    }
  }
  PartialRender p;
  p.ray_id = ray_id;
  p.region_id = region_id;
  p.color = Vec3(rgb[0], rgb[1], rgb[2]);
  p.transmittance = T;
  p.depth_sum = depth;
  return p;
}

inline void accumulate_distortion_stats(PartialRender& partial, std::span<const MarchSample> samples,
                                        const LocalRenderCache& cache, double ray_t0, double ray_t1) {
  const size_t n = samples.size();
  if (cache.alpha.size() != n || cache.prefix.size() != n)
    throw std::invalid_argument("render: distortion stats require the forward cache");
  std::vector<double> t(n), dl(n), cc(2 * n);
  for (size_t k = 0; k < n; ++k) {
    t[k] = samples[k].t;
    dl[k] = samples[k].delta;
    cc[2 * k] = cache.alpha[k];
    cc[2 * k + 1] = cache.prefix[k];
  }
  const uint64_t off[2] = {0, n};
  double out[3] = {partial.weight_sum, partial.weight_moment, partial.distortion_local};
  detail::check(dg_distortion_stats_f64(detail::stage_ctx(), t.data(), dl.data(), cc.data(), off, 1, &ray_t0,
                                        &ray_t1, out, DG_MEM_HOST));
  partial.weight_sum = out[0];
  partial.weight_moment = out[1];
  partial.distortion_local = out[2];
}

// ---- merge_forward / merge_backward (render.cpp:101-143) ----------------------------------
// Batched: ray r merges partials[ray_off[r] .. ray_off[r + 1]) in schedule order.
inline std::vector<MergedRender> merge_forward(std::span<const PartialRender> partials,
                                               std::span<const uint64_t> ray_off) {
  if (ray_off.empty()) throw std::invalid_argument("merge: offsets need n + 1 entries");
  const size_t nr = ray_off.size() - 1, ns = partials.size();
  std::vector<double> rgb(3 * ns), T(ns), dep(ns), orgb(3 * nr), oT(nr), od(nr);
  for (size_t i = 0; i < ns; ++i) {
    for (int a = 0; a < 3; ++a) rgb[3 * i + a] = partials[i].color[a];
    T[i] = partials[i].transmittance;
    dep[i] = partials[i].depth_sum;
  }
  detail::check(dg_merge_forward_f64(detail::stage_ctx(), rgb.data(), T.data(), dep.data(), ray_off.data(), nr,
                                     orgb.data(), oT.data(), od.data(), DG_MEM_HOST));
  std::vector<MergedRender> out(nr);
  for (size_t r = 0; r < nr; ++r) {
    out[r].ray_id = ray_off[r] < ns ? partials[ray_off[r]].ray_id : 0;
    out[r].color = Vec3(orgb[3 * r], orgb[3 * r + 1], orgb[3 * r + 2]);
    out[r].transmittance = oT[r];
    out[r].depth = od[r];
  }
  return out;
}

inline MergedRender merge_forward(std::span<const PartialRender> partials) {
  if (partials.empty()) throw std::invalid_argument("merge: no partials");
  const uint64_t off[2] = {0, partials.size()};
  return merge_forward(partials, std::span<const uint64_t>(off, 2))[0];
}

inline std::vector<MergeGrad> merge_backward(const Vec3& color_upstream, double transmittance_upstream,
                                             std::span<const PartialRender> partials) {
  const size_t n = partials.size();
  std::vector<MergeGrad> out(n);
  if (n == 0) return out;
  std::vector<double> rgb(3 * n), T(n), grgb(3 * n), gT(n);
  for (size_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) rgb[3 * i + a] = partials[i].color[a];
    T[i] = partials[i].transmittance;
  }
  const uint64_t off[2] = {0, n};
  const double up[3] = {color_upstream.x, color_upstream.y, color_upstream.z};
  detail::check(dg_merge_backward_f64(detail::stage_ctx(), rgb.data(), T.data(), off, 1, up, &transmittance_upstream,
                                      grgb.data(), gT.data(), DG_MEM_HOST));
  for (size_t i = 0; i < n; ++i) {
    out[i].color_grad = Vec3(grgb[3 * i], grgb[3 * i + 1], grgb[3 * i + 2]);
    out[i].transmittance_grad = gT[i];
  }
  return out;
}

// ---- local_render_backward (render.cpp:145-179) -------------------------------------------
// The device sweep re-derives (alpha, prefix) from sigma and delta with the forward's own
// arithmetic, which reproduces the cache bit for bit; the cache argument is validated as the
// reference does.
inline void local_render_backward(std::span<const MarchSample> samples, std::span<const ShadedSample> shaded,
                                  const LocalRenderCache& cache, const Vec3& color_upstream,
                                  double transmittance_upstream, std::span<const double> weight_upstream,
                                  std::span<double> sigma_grads, std::span<Vec3> color_grads) {
  const size_t n = samples.size();
  if (cache.alpha.size() != n || cache.prefix.size() != n)
    throw std::invalid_argument("render: backward requires the forward cache");
  if (sigma_grads.size() != n || color_grads.size() != n || shaded.size() != n)
    throw std::invalid_argument("render: gradient output size mismatch");
  if (!weight_upstream.empty() && weight_upstream.size() != n)
    throw std::invalid_argument("render: weight upstream size mismatch");
  const rdetail::SampleSoa soa(samples, shaded);
  const uint64_t off[2] = {0, n};
  const double up[3] = {color_upstream.x, color_upstream.y, color_upstream.z};
  detail::check(dg_local_render_backward_f64(
      detail::stage_ctx(), soa.t.data(), soa.delta.data(), soa.sigma.data(), soa.rgb.data(), off, 1, up,
      &transmittance_upstream, weight_upstream.empty() ? nullptr : weight_upstream.data(), sigma_grads.data(),
      reinterpret_cast<double*>(color_grads.data()), DG_MEM_HOST));
}

}  // namespace distgrid
