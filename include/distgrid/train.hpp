// distgrid/train.hpp — losses, learning-rate schedule and Adam of the reference API
// (train.hpp:14-83): loss_rgb / loss_transmittance / loss_distortion and their gradients run
// the per-ray / per-segment device kernels (k_ray_losses, k_distortion; fp64), AdamState::step
// runs k_adam_f64 over each caller array (train.cpp:91-115, same operation order).  Batch
// sums are added on the host in batch order, as the reference sums them.
// RayCache keeps its entries on the device (dg_ray_cache_*: the reference's two mt19937_64
// streams on the host, pixel rays built and gathered on the GPU).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <vector>

#include "distgrid/dataset.hpp"
#include "distgrid/detail/device.hpp"
#include "distgrid/rng.hpp"
#include "distgrid/vecmath.hpp"

namespace distgrid {

struct LossConfig {
  double lambda_transmittance = 1e-3;
  double lambda_distortion = 1e-3;
  double transmittance_clamp = 1e-6;
};

namespace tdetail {
// per-ray (loss_rgb, loss_T, d_rgb, d_T) of n rays on the device
struct RayLosses {
  std::vector<double> l_rgb, l_T, d_rgb, d_T;
  RayLosses(const double* rgb, const double* gt, const double* T, size_t n, double eps, bool want_rgb,
            bool want_T) {
    l_rgb.resize(n);
    l_T.resize(n);
    if (want_rgb) d_rgb.resize(3 * n);
    if (want_T) d_T.resize(n);
    detail::check(dg_ray_losses_f64(detail::stage_ctx(), rgb, gt, T, n, eps, l_rgb.data(), l_T.data(),
                                    want_rgb ? d_rgb.data() : nullptr, want_T ? d_T.data() : nullptr,
                                    DG_MEM_HOST));
  }
};
inline const double* flat(std::span<const Vec3> v) { return reinterpret_cast<const double*>(v.data()); }
}  // namespace tdetail

// sum over the batch of |C - C_gt|^2
inline double loss_rgb(std::span<const Vec3> rendered, std::span<const Vec3> ground_truth) {
  if (rendered.size() != ground_truth.size()) throw std::invalid_argument("loss: batch size mismatch");
  const size_t n = rendered.size();
  if (n == 0) return 0.0;
  const std::vector<double> T(n, 0.0);
  const tdetail::RayLosses l(tdetail::flat(rendered), tdetail::flat(ground_truth), T.data(), n, 1e-6, false, false);
  double total = 0.0;
  for (double v : l.l_rgb) total += v;
  return total;
}

inline Vec3 loss_rgb_grad(const Vec3& rendered, const Vec3& ground_truth) {
  const double T = 0.0;
  const tdetail::RayLosses l(&rendered.x, &ground_truth.x, &T, 1, 1e-6, true, false);
  return Vec3(l.d_rgb[0], l.d_rgb[1], l.d_rgb[2]);
}

inline double loss_transmittance(std::span<const double> transmittance, double eps = 1e-6) {
  const size_t n = transmittance.size();
  if (n == 0) return 0.0;
  const std::vector<double> zero(3 * n, 0.0);
  const tdetail::RayLosses l(zero.data(), zero.data(), transmittance.data(), n, eps, false, false);
  double total = 0.0;
  for (double v : l.l_T) total += v;
  return total;
}

inline double loss_transmittance_single(double transmittance, double eps = 1e-6) {
  return loss_transmittance(std::span<const double>(&transmittance, 1), eps);
}

inline double loss_transmittance_grad(double transmittance, double eps = 1e-6) {
  const double zero[3] = {0.0, 0.0, 0.0};
  const tdetail::RayLosses l(zero, zero, &transmittance, 1, eps, false, true);
  return l.d_T[0];
}

// Batched distortion over segments: segment g owns [seg_off[g], seg_off[g + 1]).
inline void loss_distortion(std::span<const double> weights, std::span<const double> midpoints,
                            std::span<const double> interval_lengths, std::span<const uint64_t> seg_off,
                            std::span<double> loss, std::span<double> grads) {
  if (seg_off.empty() || loss.size() + 1 != seg_off.size())
    throw std::invalid_argument("loss: distortion offsets need n + 1 entries");
  if (!grads.empty() && grads.size() != weights.size())
    throw std::invalid_argument("loss: distortion grad size mismatch");
  detail::check(dg_distortion_loss(detail::stage_ctx(), weights.data(), midpoints.data(), interval_lengths.data(),
                                   seg_off.data(), loss.size(), loss.data(), grads.empty() ? nullptr : grads.data(),
                                   DG_MEM_HOST));
}

inline double loss_distortion(std::span<const double> weights, std::span<const double> midpoints,
                              std::span<const double> interval_lengths) {
  const size_t n = weights.size();
  if (midpoints.size() != n || interval_lengths.size() != n)
    throw std::invalid_argument("loss: distortion input size mismatch");
  const uint64_t off[2] = {0, n};
  double l = 0.0;
  loss_distortion(weights, midpoints, interval_lengths, std::span<const uint64_t>(off, 2),
                  std::span<double>(&l, 1), {});
  return l;
}

inline void loss_distortion_grad(std::span<const double> weights, std::span<const double> midpoints,
                                 std::span<const double> interval_lengths, std::span<double> grads) {
  const size_t n = weights.size();
  if (grads.size() != n) throw std::invalid_argument("loss: distortion grad size mismatch");
  if (midpoints.size() != n || interval_lengths.size() != n)
    throw std::invalid_argument("loss: distortion input size mismatch");
  const uint64_t off[2] = {0, n};
  double l = 0.0;
  loss_distortion(weights, midpoints, interval_lengths, std::span<const uint64_t>(off, 2),
                  std::span<double>(&l, 1), grads);
}

// Cosine decay lr_start -> lr_end over total_steps (train.cpp:77-80; dg_lr_at).
struct LrSchedule {
  double lr_start = 0.05;
  double lr_end = 0.005;
  uint64_t total_steps = 1;

  double at(uint64_t step) const {
    dg_run_config c;
    dg_default_config(&c);
    c.lr_start = lr_start;
    c.lr_end = lr_end;
    c.total_steps = total_steps;
    return dg_lr_at(&c, step);
  }
};

struct AdamConfig {
  double beta1 = 0.9;
  double beta2 = 0.99;
  double eps = 1e-15;
};

// Per-array first / second moments; step() advances the shared step count, then updates every
// array on the device with the bias corrections of the new count.
class AdamState {
 public:
  AdamState() = default;
  explicit AdamState(std::span<const size_t> array_sizes) {
    for (size_t n : array_sizes) {
      m_.emplace_back(n, 0.0);
      v_.emplace_back(n, 0.0);
    }
  }

  void step(std::span<const std::span<double>> params, std::span<const std::span<const double>> grads, double lr,
            const AdamConfig& config = {}) {
    if (params.size() != m_.size() || grads.size() != m_.size())
      throw std::invalid_argument("adam: array count mismatch");
    for (size_t a = 0; a < params.size(); ++a)
      if (params[a].size() != m_[a].size() || grads[a].size() != m_[a].size())
        throw std::invalid_argument("adam: parameter shape mismatch");
    ++t_;
    for (size_t a = 0; a < params.size(); ++a)
      detail::check(dg_adam_update_f64(detail::stage_ctx(), params[a].data(), grads[a].data(), m_[a].data(),
                                       v_[a].data(), params[a].size(), t_, lr, config.beta1, config.beta2,
                                       config.eps, DG_MEM_HOST));
  }

  uint64_t step_count() const { return t_; }
  void set_step_count(uint64_t t) { t_ = t; }
  std::vector<std::vector<double>>& first_moments() { return m_; }
  std::vector<std::vector<double>>& second_moments() { return v_; }
  const std::vector<std::vector<double>>& first_moments() const { return m_; }
  const std::vector<std::vector<double>>& second_moments() const { return v_; }

 private:
  std::vector<std::vector<double>> m_, v_;
  uint64_t t_ = 0;
};

// In-memory reservoir of supervised rays refreshed from a Dataset (train.cpp:117-159).  The
// entries live on the device; refresh / draw / snapshot are serialised by a mutex, so a draw
// never sees a half-written entry.  The device cache is built from the dataset passed to the
// first refresh (and rebuilt if a different dataset object is passed later).
class RayCache {
 public:
  RayCache(size_t capacity, uint64_t seed) : capacity_(capacity), seed_(seed) {
    if (capacity == 0) throw std::invalid_argument("ray cache: capacity must be positive");
  }
  RayCache(const RayCache&) = delete;
  RayCache& operator=(const RayCache&) = delete;
  ~RayCache() {
    if (cache_) dg_ray_cache_destroy(cache_);
  }

  size_t size() const {
    std::lock_guard<std::mutex> lock(mu_);
    if (!cache_) return 0;
    uint64_t s = 0, cap = 0;
    detail::check(dg_ray_cache_size(cache_, &s, &cap));
    return size_t(s);
  }
  size_t capacity() const { return capacity_; }

  void refresh(const Dataset& dataset, size_t count) {
    std::lock_guard<std::mutex> lock(mu_);
    bind(dataset);
    detail::check(dg_ray_cache_refresh(cache_, count));
  }

  std::vector<SupervisedRay> draw_batch(size_t batch_size) {
    std::lock_guard<std::mutex> lock(mu_);
    if (!cache_) throw std::runtime_error("ray cache: empty");
    std::vector<double> o(3 * batch_size), d(3 * batch_size);
    std::vector<float> gt(3 * batch_size);
    std::vector<uint32_t> img(batch_size);
    std::vector<uint64_t> pix(batch_size);
    detail::check(dg_ray_cache_draw_host(cache_, batch_size, o.data(), d.data(), gt.data(), img.data(), pix.data()));
    return rays(o, d, gt, img, pix, batch_size);
  }

  std::vector<SupervisedRay> snapshot() const {
    std::lock_guard<std::mutex> lock(mu_);
    if (!cache_) return {};
    uint64_t n = 0, cap = 0;
    detail::check(dg_ray_cache_size(cache_, &n, &cap));
    std::vector<double> o(3 * n), d(3 * n);
    std::vector<float> gt(3 * n);
    std::vector<uint32_t> img(n);
    std::vector<uint64_t> pix(n);
    detail::check(dg_ray_cache_snapshot(cache_, o.data(), d.data(), gt.data(), img.data(), pix.data()));
    return rays(o, d, gt, img, pix, n);
  }

  dg_ray_cache* handle() const { return cache_; }

 private:
  static std::vector<SupervisedRay> rays(const std::vector<double>& o, const std::vector<double>& d,
                                         const std::vector<float>& gt, const std::vector<uint32_t>& img,
                                         const std::vector<uint64_t>& pix, size_t n) {
    std::vector<SupervisedRay> out(n);
    for (size_t i = 0; i < n; ++i) {
      SupervisedRay& r = out[i];
      r.ray.origin = Vec3(o[3 * i], o[3 * i + 1], o[3 * i + 2]);
      r.ray.dir = Vec3(d[3 * i], d[3 * i + 1], d[3 * i + 2]);
      r.ray.pixel_id = pix[i];
      r.ray.image_id = img[i];
      r.color_gt = Vec3(gt[3 * i], gt[3 * i + 1], gt[3 * i + 2]);
      r.image_id = img[i];
    }
    return out;
  }

  void bind(const Dataset& ds) {
    if (cache_ && bound_ == &ds) return;
    bool any_train = false;
    for (uint8_t t : ds.is_train) any_train |= t != 0;
    if (!any_train) throw std::invalid_argument("ray cache: dataset has no train images");
    std::vector<dg_camera> cams(ds.size());
    std::vector<const uint8_t*> imgs(ds.size());
    for (size_t i = 0; i < ds.size(); ++i) {
      const CameraPose& p = ds.poses[i];
      dg_camera& c = cams[i];
      c.image_id = p.image_id;
      c.width = ds.images[i].width;
      c.height = ds.images[i].height;
      c.is_train = ds.is_train[i];
      for (int k = 0; k < 9; ++k) c.rotation[k] = p.rotation.m[k];
      for (int a = 0; a < 3; ++a) c.translation[a] = p.translation[a];
      c.fx = p.fx;
      c.fy = p.fy;
      c.cx = p.cx;
      c.cy = p.cy;
      imgs[i] = ds.images[i].rgb.data();
    }
    if (cache_) dg_ray_cache_destroy(cache_);
    cache_ = nullptr;
    detail::check(dg_ray_cache_create(-1, cams.data(), imgs.data(), uint32_t(ds.size()), capacity_, seed_, &cache_));
    bound_ = &ds;
  }

  size_t capacity_;
  uint64_t seed_;
  const Dataset* bound_ = nullptr;
  dg_ray_cache* cache_ = nullptr;
  mutable std::mutex mu_;
};

}  // namespace distgrid
