// distgrid/worker.hpp — DistributedRun, Worker views, StepStats and EvalImage of the reference
// API (worker.hpp:60-240), over the device training / evaluation path (dg_train_step,
// dg_render, dg_render_image).  The constructor takes the reference's (RunConfig,
// PartitionManifest, AppearanceTable) and initialises every region exactly as the reference's
// Worker constructor does (worker.cpp:176-200: mt19937_64 streams, all cells occupied).
// One process drives every partition on its GPU; with world > 1 (one process per GPU) pass
// rank / world and call init_nccl (or use the C ABI's peer-memory backend) and each rank trains
// on its contiguous shard of the batch.  worker(i) is a view of region i's state (parameters,
// Adam moments, occupancy, step), read from the device on access; the lock-step device path has
// no worker threads, so start()/stop() only keep the reference's state machine.
// Not here: train_loop / evaluate_split_psnr (they read a Dataset) and the wire Transport.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <vector>

#include "distgrid/config.hpp"
#include "distgrid/detail/device.hpp"
#include "distgrid/field.hpp"
#include "distgrid/partition.hpp"
#include "distgrid/render.hpp"
#include "distgrid/train.hpp"

namespace distgrid {

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

struct EvalImage {
  uint32_t width = 0, height = 0;
  std::vector<Vec3> color;
  std::vector<double> transmittance;
  std::vector<double> depth;
  std::vector<Vec3> attribution;
};

// worker.cpp:902-925: per-region grid configs and the march step of a run
inline GridConfig make_fine_grid_config(const RunConfig& c, const Aabb& fine_box) {
  GridConfig g;
  g.levels = c.grid_levels;
  g.table_length = 1u << c.fine_table_log2;
  g.features_per_level = c.grid_features;
  g.base_resolution = c.base_resolution;
  g.max_resolution = c.max_resolution;
  g.aspect = fine_box.extent();
  return g;
}
inline GridConfig make_coarse_grid_config(const RunConfig& c, const Aabb& coarse_box) {
  GridConfig g = make_fine_grid_config(c, coarse_box);
  g.table_length = 1u << c.coarse_table_log2;
  return g;
}
inline double march_step_for(const RunConfig& c, const Aabb& outer_box) {
  return max_component(outer_box.extent()) / c.march_step_divisor;
}

class DistributedRun;

// Region i of a run: reads its state from the device (value snapshots).
class Worker {
 public:
  uint32_t region_id() const { return region_; }
  const RegionBox& region() const;
  uint64_t step() const {
    uint64_t s = 0;
    detail::check(dg_get_step(ctx_, &s));
    return s;
  }
  // parameters in FieldParams::parameter_arrays order, fine field then coarse (fp32 on device)
  std::vector<float> parameters() const {
    uint64_t n = 0;
    detail::check(dg_param_count(ctx_, region_, &n));
    std::vector<float> p(n);
    detail::check(dg_get_params(ctx_, region_, p.data()));
    return p;
  }
  void set_parameters(std::span<const float> p) {
    uint64_t n = 0;
    detail::check(dg_param_count(ctx_, region_, &n));
    if (p.size() != n) throw std::invalid_argument("worker: parameter vector size");
    detail::check(dg_set_params(ctx_, region_, p.data()));
  }
  // Adam moments (same layout) and step count
  void adam_state(std::vector<float>& m, std::vector<float>& v, uint64_t& t) const {
    uint64_t n = 0;
    detail::check(dg_param_count(ctx_, region_, &n));
    m.resize(n);
    v.resize(n);
    detail::check(dg_get_adam(ctx_, region_, m.data(), v.data(), &t));
  }
  FieldParams fine_field() const { return field(0); }
  FieldParams coarse_field() const { return field(1); }
  OccupancyGrid occ_fine() const { return occupancy(0); }
  OccupancyGrid occ_coarse() const { return occupancy(1); }

 private:
  friend class DistributedRun;
  Worker(dg_ctx* c, uint32_t region, const DistributedRun* run) : ctx_(c), region_(region), run_(run) {}
  FieldParams field(uint32_t cascade) const;
  OccupancyGrid occupancy(uint32_t cascade) const;

  dg_ctx* ctx_;
  uint32_t region_;
  const DistributedRun* run_;
};

class DistributedRun {
 public:
  DistributedRun(const RunConfig& config, const PartitionManifest& manifest, const AppearanceTable& appearance)
      : DistributedRun(config, manifest, appearance, -1, 0, 1) {}
  // one process per GPU: partition p on rank p % world
  DistributedRun(const RunConfig& config, const PartitionManifest& manifest, const AppearanceTable& appearance,
                 int device, int rank, int world)
      : config_(config), manifest_(manifest), rank_(rank), world_(world) {
    config_.validate();
    if (manifest_.kx != config_.partitions_x || manifest_.ky != config_.partitions_y)
      throw std::invalid_argument("run: manifest tiling differs from the config's partitions");
    manifest_.validate();
    double il[3], ih[3], ol[3], oh[3];
    pdetail::boxes(manifest_, il, ih, ol, oh);
    const dg_run_config c = to_dg_config(config_, il, ih, ol, oh, manifest_.ground_altitude);
    dg_ctx* raw = nullptr;
    detail::check(dg_ctx_create(&c, device, rank, world, &raw));
    ctx_.reset(raw);
    for (uint32_t p = 0; p < manifest_.region_count(); ++p) {
      int r = 0;
      detail::check(dg_partition_rank(raw, p, &r));
      if (r == rank) detail::check(dg_init_params_reference(raw, p));  // worker.cpp:186-190
    }
    if (appearance.dim != config_.appearance_dim && !appearance.image_ids.empty())
      throw std::invalid_argument("run: appearance table width differs from appearance_dim");
    if (!appearance.image_ids.empty()) {
      const std::vector<float> rows(appearance.rows.begin(), appearance.rows.end());
      detail::check(dg_set_appearance(raw, appearance.image_ids.data(), rows.data(),
                                      uint32_t(appearance.image_ids.size())));
    }
    for (uint32_t p = 0; p < manifest_.region_count(); ++p)
      workers_.push_back(std::unique_ptr<Worker>(new Worker(raw, p, this)));
  }
  ~DistributedRun() = default;
  DistributedRun(const DistributedRun&) = delete;
  DistributedRun& operator=(const DistributedRun&) = delete;

  void init_nccl(const uint8_t id[DG_NCCL_UNIQUE_ID_BYTES]) { detail::check(dg_comm_init_nccl(ctx_.get(), id)); }

  uint32_t worker_count() const { return uint32_t(workers_.size()); }
  // region's view (its state lives on rank region % world)
  Worker& worker(uint32_t region) { return *workers_.at(region); }
  const PartitionManifest& manifest() const { return manifest_; }

  void start() {
    if (running_) throw std::logic_error("run: already started");
    running_ = true;
  }
  void stop() { running_ = false; }
  bool running() const { return running_; }

  // Lock-step training iteration over this rank's shard (ray ids first_ray_id + i).
  StepStats training_step(std::span<const SupervisedRay> batch, uint64_t step, uint64_t first_ray_id = 0) {
    const size_t n = batch.size();
    o_.resize(3 * n);
    d_.resize(3 * n);
    gt_.resize(3 * n);
    img_.resize(n);
    for (size_t i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) {
        o_[3 * i + a] = batch[i].ray.origin[a];
        d_[3 * i + a] = batch[i].ray.dir[a];
        gt_[3 * i + a] = float(batch[i].color_gt[a]);
      }
      img_[i] = batch[i].image_id;
    }
    const dg_ray_batch b{o_.data(), d_.data(), gt_.data(), img_.data(), n, first_ray_id, DG_MEM_HOST, 0};
    dg_step_stats st{};
    detail::check(dg_train_step(ctx_.get(), &b, step, &st));
    bytes_sent_ += st.bytes_sent;
    scatter_bytes_ += st.partial_bytes_sent;
    scatter_entries_ += st.partial_records_sent;
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

  std::vector<MergedRender> evaluate_rays(std::span<const Ray> rays, std::span<const double> appearance_vec,
                                          uint64_t first_ray_id = 0) {
    const size_t n = rays.size();
    o_.resize(3 * n);
    d_.resize(3 * n);
    for (size_t i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) {
        o_[3 * i + a] = rays[i].origin[a];
        d_[3 * i + a] = rays[i].dir[a];
      }
    const std::vector<float> app(appearance_vec.begin(), appearance_vec.end());
    std::vector<float> rgb(3 * n), T(n), depth(n);
    const dg_ray_batch b{o_.data(), d_.data(), nullptr, nullptr, n, first_ray_id, DG_MEM_HOST, 0};
    dg_merged m{rgb.data(), T.data(), depth.data(), nullptr, DG_MEM_HOST, 0};
    detail::check(dg_render(ctx_.get(), &b, app.empty() ? nullptr : app.data(), &m));
    std::vector<MergedRender> out(n);
    for (size_t i = 0; i < n; ++i) {
      out[i].ray_id = first_ray_id + i;
      out[i].color = Vec3(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
      out[i].transmittance = T[i];
      out[i].depth = depth[i];
    }
    return out;
  }

  // One ray per pixel centre, merged colour / transmittance / depth and region attribution.
  EvalImage evaluate_image(const CameraPose& pose, std::span<const double> appearance_vec) {
    pose.validate();
    dg_camera cam{};
    cam.image_id = pose.image_id;
    cam.width = pose.width;
    cam.height = pose.height;
    for (int k = 0; k < 9; ++k) cam.rotation[k] = pose.rotation.m[k];
    for (int a = 0; a < 3; ++a) cam.translation[a] = pose.translation[a];
    cam.fx = pose.fx;
    cam.fy = pose.fy;
    cam.cx = pose.cx;
    cam.cy = pose.cy;
    const size_t n = size_t(pose.width) * pose.height;
    const std::vector<float> app(appearance_vec.begin(), appearance_vec.end());
    std::vector<float> rgb(3 * n), T(n), depth(n), attr(3 * n);
    dg_merged m{rgb.data(), T.data(), depth.data(), attr.data(), DG_MEM_HOST, 0};
    detail::check(dg_render_image(ctx_.get(), &cam, app.empty() ? nullptr : app.data(), &m));
    EvalImage out;
    out.width = pose.width;
    out.height = pose.height;
    for (size_t i = 0; i < n; ++i) {
      out.color.emplace_back(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
      out.transmittance.push_back(T[i]);
      out.depth.push_back(depth[i]);
      out.attribution.emplace_back(attr[3 * i], attr[3 * i + 1], attr[3 * i + 2]);
    }
    return out;
  }

  // Traffic this rank sent to other ranks, summed over the training steps so far (with one rank
  // every exchange is local and the counts stay 0): both exchanges, then exchange 2 alone —
  // its records are 24 bytes (rgb, -ln T, depth, ray id; + 16 with cross-segment distortion).
  uint64_t worker_bytes_sent() const { return bytes_sent_; }
  uint64_t scatter_payload_bytes() const { return scatter_bytes_; }
  uint64_t scatter_entries() const { return scatter_entries_; }

  dg_ctx* handle() const { return ctx_.get(); }

 private:
  friend class Worker;
  RunConfig config_;
  PartitionManifest manifest_;
  int rank_ = 0, world_ = 1;
  detail::CtxPtr ctx_;
  std::vector<std::unique_ptr<Worker>> workers_;
  bool running_ = false;
  uint64_t bytes_sent_ = 0, scatter_bytes_ = 0, scatter_entries_ = 0;
  std::vector<double> o_, d_;
  std::vector<float> gt_;
  std::vector<uint32_t> img_;
};

inline const RegionBox& Worker::region() const { return run_->manifest_.regions.at(region_); }

inline FieldParams Worker::field(uint32_t cascade) const {
  const RegionBox& rb = region();
  const RunConfig& c = run_->config_;
  FieldParams f;
  f.level = cascade ? CascadeLevel::Coarse : CascadeLevel::Fine;
  f.appearance_dim = c.appearance_dim;
  const GridConfig g = cascade ? make_coarse_grid_config(c, rb.coarse) : make_fine_grid_config(c, rb.fine);
  Rng unused(0);
  GridConfig g0 = g;  // shapes only: tables are filled from the device below
  f.grid = HashGrid(g0, unused);
  const uint32_t dw[] = {f.grid.feature_width(), kHiddenWidth, 1 + kDensityFeatureWidth};
  f.density_mlp = Mlp(dw, Activation::ReLU, unused);
  const uint32_t cw[] = {kDensityFeatureWidth + kShWidth + c.appearance_dim, kHiddenWidth, kHiddenWidth, 3};
  f.color_mlp = Mlp(cw, cascade ? Activation::Sigmoid : Activation::ReLU, unused);
  const std::vector<float> p = parameters();
  std::vector<dg_array_desc> arrays(64);
  uint32_t na = 0;
  detail::check(dg_param_layout(ctx_, region_, arrays.data(), uint32_t(arrays.size()), &na));
  arrays.resize(na);
  std::vector<std::span<double>> dst = f.parameter_arrays();
  size_t k = 0;
  for (const dg_array_desc& a : arrays) {
    if (a.cascade != cascade) continue;
    if (k >= dst.size() || dst[k].size() != a.size) throw std::runtime_error("worker: parameter layout mismatch");
    for (uint64_t i = 0; i < a.size; ++i) dst[k][i] = double(p[a.offset + i]);
    ++k;
  }
  return f;
}

inline OccupancyGrid Worker::occupancy(uint32_t cascade) const {
  const RegionBox& rb = region();
  const RunConfig& c = run_->config_;
  OccupancyGrid g(cascade ? rb.coarse : rb.fine, c.occ_resolution, c.occ_decay,
                  c.occ_threshold_early * c.occ_threshold_scale);
  const uint64_t n = g.cell_count();
  std::vector<float> den(n);
  std::vector<uint8_t> bits(n);
  double thr = 0.0;
  detail::check(dg_get_occupancy_density(ctx_, region_, cascade, den.data(), &thr));
  detail::check(dg_get_occupancy(ctx_, region_, cascade, bits.data()));
  g.assign(std::vector<double>(den.begin(), den.end()), std::move(bits), thr);
  return g;
}

}  // namespace distgrid
