// distgrid_b200/distgrid.hpp — C++ facade with the reference's names over the C ABI.
//
// A drop-in for the per-ray path of the reference library (proj/include/distgrid/*.hpp):
//   RunConfig (config.hpp:13-78), Vec3/Aabb (vecmath.hpp), Ray (geometry.hpp:12-19),
//   SupervisedRay (dataset.hpp:79-83), RaySegment (render.hpp:15-21), StepStats
//   (worker.hpp:153-162), MergedRender (render.hpp:38-43), split_regions / segment_ray
//   (partition.hpp:83-91), and DistributedRun::{training_step, evaluate_rays, start, stop}
//   (worker.hpp:182-226).  Errors are rethrown as the reference's exception classes.
// Header-only; link with libdg_b200.so.  Numbers are computed on the GPU (sm_100a) — there
// is no CPU path behind these calls.
#pragma once

#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "distgrid_b200.h"

namespace distgrid {

struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};

struct Aabb {
  Vec3 lo, hi;
};

struct Ray {
  Vec3 origin;
  Vec3 dir;  // unit length
  uint64_t pixel_id = 0;
  uint32_t image_id = 0;
};

struct SupervisedRay {
  Ray ray;
  Vec3 color_gt;
  uint32_t image_id = 0;
};

struct RaySegment {
  uint64_t ray_id = 0;
  uint32_t region_id = 0;
  uint32_t order_index = 0;
  double t_enter = 0.0;
  double t_exit = 0.0;
};

struct MergedRender {
  uint64_t ray_id = 0;
  Vec3 color;
  double transmittance = 1.0;
  double depth = 0.0;
};

// CameraPose (partition.hpp:15-30): camera-to-world rotation (row-major), pinhole intrinsics.
struct CameraPose {
  uint32_t image_id = 0;
  double rotation[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  Vec3 translation;
  double fx = 0.0, fy = 0.0, cx = 0.0, cy = 0.0;
  uint32_t width = 0, height = 0;
};

// EvalImage (worker.hpp:164-171).
struct EvalImage {
  uint32_t width = 0, height = 0;
  std::vector<Vec3> color;
  std::vector<double> transmittance;
  std::vector<double> depth;
  std::vector<Vec3> attribution;
};

struct StepStats {
  uint64_t step = 0;
  double loss_rgb = 0.0;
  double loss_transmittance = 0.0;
  double loss_distortion = 0.0;
  double lr = 0.0;
  uint64_t rays = 0;
  uint64_t dropped_rays = 0;
  uint64_t bytes_sent = 0;
};

// The reference's exception mapping.
inline void check(int rc) {
  if (rc == DG_OK) return;
  const std::string msg = dg_last_error();
  switch (rc) {
    case DG_EINVAL: throw std::invalid_argument(msg);
    case DG_ERANGE: throw std::out_of_range(msg);
    case DG_EPROTO: throw std::runtime_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// RunConfig: defaults of config.hpp:13-78 (dg_default_config), plus the two boxes of the
// manifest (split_regions inputs).
struct RunConfig : dg_run_config {
  RunConfig() { dg_default_config(this); }
};

struct PartitionManifest {
  uint32_t kx = 1, ky = 1;
  Aabb inner, outer;
  double ground_altitude = 0.0;
  std::vector<double> x_planes, y_planes;
  uint32_t region_count() const { return kx * ky; }
};

// partition.cpp:206-252 — the planes are computed exactly as the reference (host setup).
inline PartitionManifest split_regions(const Aabb& inner, const Aabb& outer, uint32_t kx,
                                       uint32_t ky, double ground_altitude) {
  if (kx < 1 || ky < 1) throw std::invalid_argument("split_regions: kx, ky must be >= 1");
  PartitionManifest m;
  m.kx = kx;
  m.ky = ky;
  m.inner = inner;
  m.outer = outer;
  m.ground_altitude = ground_altitude;
  for (uint32_t i = 0; i <= kx; ++i)
    m.x_planes.push_back(i == 0 ? inner.lo.x : i == kx ? inner.hi.x
                                              : inner.lo.x + (inner.hi.x - inner.lo.x) * double(i) / double(kx));
  for (uint32_t i = 0; i <= ky; ++i)
    m.y_planes.push_back(i == 0 ? inner.lo.y : i == ky ? inner.hi.y
                                              : inner.lo.y + (inner.hi.y - inner.lo.y) * double(i) / double(ky));
  return m;
}

inline void apply_manifest(RunConfig& c, const PartitionManifest& m) {
  c.kx = m.kx;
  c.ky = m.ky;
  const double il[3] = {m.inner.lo.x, m.inner.lo.y, m.inner.lo.z};
  const double ih[3] = {m.inner.hi.x, m.inner.hi.y, m.inner.hi.z};
  const double ol[3] = {m.outer.lo.x, m.outer.lo.y, m.outer.lo.z};
  const double oh[3] = {m.outer.hi.x, m.outer.hi.y, m.outer.hi.z};
  for (int a = 0; a < 3; ++a) {
    c.inner_lo[a] = il[a];
    c.inner_hi[a] = ih[a];
    c.outer_lo[a] = ol[a];
    c.outer_hi[a] = oh[a];
  }
  c.ground_altitude = m.ground_altitude;
}

// DistributedRun: every partition of the manifest on this process's GPU(s).  With
// world > 1 (one process per GPU, torchrun-style) construct with rank/world and call
// init_nccl() with a shared unique id; each rank then passes its contiguous shard.
class DistributedRun {
 public:
  DistributedRun(const RunConfig& config, const PartitionManifest& manifest,
                 std::span<const uint32_t> image_ids = {}, std::span<const float> appearance = {},
                 int device = -1, int rank = 0, int world = 1)
      : config_(config) {
    apply_manifest(config_, manifest);
    check(dg_ctx_create(&config_, device, rank, world, &ctx_));
    uint32_t total = 0, local = 0;
    check(dg_partition_count(ctx_, &total, &local));
    for (uint32_t p = 0; p < total; ++p) {
      int r = 0;
      check(dg_partition_rank(ctx_, p, &r));
      if (r == rank) check(dg_init_params_reference(ctx_, p));  // worker.cpp:186-190
    }
    if (!image_ids.empty())
      check(dg_set_appearance(ctx_, image_ids.data(), appearance.data(), uint32_t(image_ids.size())));
  }
  ~DistributedRun() { dg_ctx_destroy(ctx_); }
  DistributedRun(const DistributedRun&) = delete;
  DistributedRun& operator=(const DistributedRun&) = delete;

  void init_nccl(const uint8_t id[DG_NCCL_UNIQUE_ID_BYTES]) { check(dg_comm_init_nccl(ctx_, id)); }

  // Lock-step semantics need no worker threads: start/stop keep the reference's API shape.
  void start() {
    if (running_) throw std::logic_error("run already started");
    running_ = true;
  }
  void stop() { running_ = false; }
  bool running() const { return running_; }

  StepStats training_step(std::span<const SupervisedRay> batch, uint64_t step,
                          uint64_t first_ray_id = 0) {
    const size_t n = batch.size();
    o_.resize(3 * n);
    d_.resize(3 * n);
    gt_.resize(3 * n);
    img_.resize(n);
    for (size_t i = 0; i < n; ++i) {
      const SupervisedRay& r = batch[i];
      o_[3 * i] = r.ray.origin.x;
      o_[3 * i + 1] = r.ray.origin.y;
      o_[3 * i + 2] = r.ray.origin.z;
      d_[3 * i] = r.ray.dir.x;
      d_[3 * i + 1] = r.ray.dir.y;
      d_[3 * i + 2] = r.ray.dir.z;
      gt_[3 * i] = float(r.color_gt.x);
      gt_[3 * i + 1] = float(r.color_gt.y);
      gt_[3 * i + 2] = float(r.color_gt.z);
      img_[i] = r.image_id;
    }
    dg_ray_batch b{o_.data(), d_.data(), gt_.data(), img_.data(), n, first_ray_id, DG_MEM_HOST, 0};
    dg_step_stats st{};
    check(dg_train_step(ctx_, &b, step, &st));
    StepStats out;
    out.step = st.step;
    out.loss_rgb = st.loss_rgb;
    out.loss_transmittance = st.loss_transmittance;
    out.loss_distortion = st.loss_distortion;
    out.lr = st.lr;
    out.rays = st.rays;
    out.dropped_rays = st.dropped_rays;
    out.bytes_sent = st.bytes_sent;
    return out;
  }

  std::vector<MergedRender> evaluate_rays(std::span<const Ray> rays,
                                          std::span<const double> appearance_vec) {
    const size_t n = rays.size();
    o_.resize(3 * n);
    d_.resize(3 * n);
    for (size_t i = 0; i < n; ++i) {
      o_[3 * i] = rays[i].origin.x;
      o_[3 * i + 1] = rays[i].origin.y;
      o_[3 * i + 2] = rays[i].origin.z;
      d_[3 * i] = rays[i].dir.x;
      d_[3 * i + 1] = rays[i].dir.y;
      d_[3 * i + 2] = rays[i].dir.z;
    }
    std::vector<float> app(appearance_vec.begin(), appearance_vec.end());
    std::vector<float> rgb(3 * n), T(n), depth(n);
    dg_ray_batch b{o_.data(), d_.data(), nullptr, nullptr, n, 0, DG_MEM_HOST, 0};
    dg_merged m{rgb.data(), T.data(), depth.data(), nullptr, DG_MEM_HOST, 0};
    check(dg_render(ctx_, &b, app.data(), &m));
    std::vector<MergedRender> out(n);
    for (size_t i = 0; i < n; ++i) {
      out[i].ray_id = i;
      out[i].color = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
      out[i].transmittance = T[i];
      out[i].depth = depth[i];
    }
    return out;
  }

  // DistributedRun::evaluate_image (worker.cpp:836-880): one ray per pixel centre, merged
  // colour / transmittance / depth and the per-region attribution.
  EvalImage evaluate_image(const CameraPose& pose, std::span<const double> appearance_vec) {
    dg_camera cam{};
    cam.image_id = pose.image_id;
    cam.width = pose.width;
    cam.height = pose.height;
    for (int k = 0; k < 9; ++k) cam.rotation[k] = pose.rotation[k];
    cam.translation[0] = pose.translation.x;
    cam.translation[1] = pose.translation.y;
    cam.translation[2] = pose.translation.z;
    cam.fx = pose.fx;
    cam.fy = pose.fy;
    cam.cx = pose.cx;
    cam.cy = pose.cy;
    const size_t n = size_t(pose.width) * pose.height;
    std::vector<float> app(appearance_vec.begin(), appearance_vec.end());
    std::vector<float> rgb(3 * n), T(n), depth(n), attr(3 * n);
    dg_merged m{rgb.data(), T.data(), depth.data(), attr.data(), DG_MEM_HOST, 0};
    check(dg_render_image(ctx_, &cam, app.empty() ? nullptr : app.data(), &m));
    EvalImage out;
    out.width = pose.width;
    out.height = pose.height;
    out.color.resize(n);
    out.transmittance.resize(n);
    out.depth.resize(n);
    out.attribution.resize(n);
    for (size_t i = 0; i < n; ++i) {
      out.color[i] = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
      out.transmittance[i] = T[i];
      out.depth[i] = depth[i];
      out.attribution[i] = {attr[3 * i], attr[3 * i + 1], attr[3 * i + 2]};
    }
    return out;
  }

  // segment_ray over a batch (partition.cpp:254-296), on the device.
  std::vector<std::vector<RaySegment>> segment_rays(std::span<const Ray> rays) {
    const size_t n = rays.size();
    std::vector<double> o(3 * n), d(3 * n), te(n * DG_MAX_SEGMENTS), tx(n * DG_MAX_SEGMENTS);
    std::vector<uint8_t> ns(n);
    std::vector<uint16_t> reg(n * DG_MAX_SEGMENTS);
    for (size_t i = 0; i < n; ++i) {
      o[3 * i] = rays[i].origin.x;
      o[3 * i + 1] = rays[i].origin.y;
      o[3 * i + 2] = rays[i].origin.z;
      d[3 * i] = rays[i].dir.x;
      d[3 * i + 1] = rays[i].dir.y;
      d[3 * i + 2] = rays[i].dir.z;
    }
    check(dg_segment_rays(ctx_, o.data(), d.data(), n, ns.data(), reg.data(), te.data(), tx.data(),
                          DG_MEM_HOST));
    std::vector<std::vector<RaySegment>> out(n);
    for (size_t i = 0; i < n; ++i)
      for (uint32_t s = 0; s < ns[i]; ++s)
        out[i].push_back({rays[i].pixel_id, reg[i * DG_MAX_SEGMENTS + s], s,
                          te[i * DG_MAX_SEGMENTS + s], tx[i * DG_MAX_SEGMENTS + s]});
    return out;
  }

  // Flat state of one region (FieldParams::parameter_arrays order, fine then coarse).
  std::vector<float> parameters(uint32_t region) {
    uint64_t n = 0;
    check(dg_param_count(ctx_, region, &n));
    std::vector<float> p(n);
    check(dg_get_params(ctx_, region, p.data()));
    return p;
  }
  void set_parameters(uint32_t region, std::span<const float> p) {
    check(dg_set_params(ctx_, region, p.data()));
  }

  dg_ctx* handle() { return ctx_; }

 private:
  RunConfig config_;
  dg_ctx* ctx_ = nullptr;
  bool running_ = false;
  std::vector<double> o_, d_;
  std::vector<float> gt_;
  std::vector<uint32_t> img_;
};

}  // namespace distgrid
