// distgrid/field.hpp — one radiance sub-field of the reference API (field.hpp:10-99):
// AppearanceTable, FieldParams (hash grid + density MLP + colour MLP), FieldGrads and
// query_density / query_color / field_backward.  The parameters are host arrays with the
// reference's value semantics and initialisation; every evaluation runs on the field's device
// context (fp32 parameters): query_density -> k_encode_points + k_field_density, query_color ->
// k_field_color, field_backward -> the training path's encode / MLP backward kernels
// (dg_field_backward), with gradients added into the caller's FieldGrads.  query_field /
// field_backward over spans are the batched device overloads.
// Not here: build_appearance_table (Gram-matrix PCA over dataset images, outside the per-ray
// path; a table is passed in as rows).
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "distgrid/detail/field_ctx.hpp"
#include "distgrid/grid.hpp"
#include "distgrid/mlp.hpp"
#include "distgrid/vecmath.hpp"

namespace distgrid {

inline constexpr uint32_t kDensityFeatureWidth = 15;
inline constexpr uint32_t kHiddenWidth = 64;
inline constexpr uint32_t kShWidth = 16;
inline constexpr double kOutputClip = 15.0;

enum class CascadeLevel : uint8_t { Fine = 0, Coarse = 1 };

struct AppearanceTable {
  uint32_t dim = 0;
  std::vector<uint32_t> image_ids;
  std::vector<double> rows;  // image-major

  std::span<const double> row(uint32_t image_id) const {
    for (size_t i = 0; i < image_ids.size(); ++i)
      if (image_ids[i] == image_id) return std::span<const double>(rows.data() + i * dim, dim);
    throw std::out_of_range("appearance: unknown image id");
  }
  std::vector<double> mean_row() const {
    std::vector<double> m(dim, 0.0);
    if (image_ids.empty()) return m;
    for (size_t i = 0; i < image_ids.size(); ++i)
      for (uint32_t k = 0; k < dim; ++k) m[k] += rows[i * dim + k];
    for (double& v : m) v /= double(image_ids.size());
    return m;
  }
};

struct FieldParams {
  CascadeLevel level = CascadeLevel::Fine;
  HashGrid grid;
  Mlp density_mlp;
  Mlp color_mlp;
  uint32_t appearance_dim = 16;

  FieldParams() = default;
  // grid, then density [2L, 64, 16] (ReLU), then colour [15 + 16 + d_app, 64, 64, 3] (ReLU fine,
  // Sigmoid coarse), all from the one stream (field.cpp:189-201)
  FieldParams(CascadeLevel lvl, const GridConfig& grid_config, uint32_t app_dim, Rng& rng)
      : level(lvl), grid(grid_config, rng), appearance_dim(app_dim) {
    const uint32_t dw[] = {grid.feature_width(), kHiddenWidth, 1 + kDensityFeatureWidth};
    density_mlp = Mlp(dw, Activation::ReLU, rng);
    const uint32_t cw[] = {kDensityFeatureWidth + kShWidth + app_dim, kHiddenWidth, kHiddenWidth, 3};
    color_mlp = Mlp(cw, lvl == CascadeLevel::Coarse ? Activation::Sigmoid : Activation::ReLU, rng);
  }

  std::vector<std::span<double>> parameter_arrays() {
    std::vector<std::span<double>> a = grid.parameter_arrays();
    for (auto& s : density_mlp.parameter_arrays()) a.push_back(s);
    for (auto& s : color_mlp.parameter_arrays()) a.push_back(s);
    return a;
  }

  // the field's context with the current parameters in its cascade slot
  dg_ctx* device() const {
    const GridConfig& g = grid.config();
    if (g.features_per_level != 2)
      throw std::invalid_argument("field: the device path requires features_per_level == 2");
    if (!dev_.p) {
      const double ext[3] = {g.aspect.x, g.aspect.y, g.aspect.z};
      dev_.p = std::make_unique<detail::FieldCtx>(ext, g.levels, g.base_resolution, g.max_resolution,
                                                  detail::log2_exact(g.table_length), appearance_dim);
    }
    std::vector<std::span<const double>> a;
    for (const HashGridLevel& lv : grid.levels()) a.emplace_back(lv.table);
    for (const Mlp* m : {&density_mlp, &color_mlp})
      for (const DenseLayer& l : m->layers()) {
        a.emplace_back(l.weights);
        a.emplace_back(l.bias);
      }
    dev_.p->upload(slot(), a);
    return dev_.p->get();
  }
  uint32_t slot() const { return level == CascadeLevel::Coarse ? 1u : 0u; }
  detail::FieldCtx& device_state() const { return *dev_.p; }

 private:
  mutable detail::DeviceSlot<detail::FieldCtx> dev_;
};

struct FieldGrads {
  HashGridGrads grid;
  std::vector<DenseLayerGrads> density_mlp;
  std::vector<DenseLayerGrads> color_mlp;

  void zero() {
    grid.zero();
    for (auto* v : {&density_mlp, &color_mlp})
      for (DenseLayerGrads& g : *v) {
        std::fill(g.weights.begin(), g.weights.end(), 0.0);
        std::fill(g.bias.begin(), g.bias.end(), 0.0);
      }
  }
  // sinks in FieldParams::parameter_arrays order
  std::vector<std::span<double>> arrays() {
    std::vector<std::span<double>> a;
    for (auto& g : grid.level_grads) a.emplace_back(g);
    for (auto* v : {&density_mlp, &color_mlp})
      for (DenseLayerGrads& g : *v) {
        a.emplace_back(g.weights);
        a.emplace_back(g.bias);
      }
    return a;
  }
};

inline FieldGrads make_field_grads(const FieldParams& p) {
  return FieldGrads{p.grid.make_grads(), p.density_mlp.make_grads(), p.color_mlp.make_grads()};
}

// What field_backward needs of one evaluated sample: its inputs (the device backward
// recomputes the forward activations from them) and the forward outputs.
struct FieldSampleCache {
  Vec3 point;      // normalised
  Vec3 direction;  // unit
  std::vector<double> appearance;
  std::vector<double> density_feature;
  double sigma = 0.0;
  Vec3 color;
};

struct DensityResult {
  double sigma = 0.0;
  std::array<double, kDensityFeatureWidth> feature{};
};

// ---- batched device overloads ----
// sigma and the 15 density features of n normalised points
inline void query_density(std::span<const Vec3> points, const FieldParams& params, std::span<double> sigma,
                          std::span<double> features) {
  const size_t n = points.size();
  if (sigma.size() != n || features.size() != n * kDensityFeatureWidth)
    throw std::invalid_argument("field: query_density output size");
  for (const Vec3& p : points)
    if (p.x < 0.0 || p.x > 1.0 || p.y < 0.0 || p.y > 1.0 || p.z < 0.0 || p.z > 1.0)
      throw std::invalid_argument("grid: encode point outside the unit box");
  if (!n) return;
  std::vector<float> s(n), f(n * kDensityFeatureWidth);
  detail::check(dg_field_density(params.device(), 0, params.slot(), reinterpret_cast<const double*>(points.data()),
                                 n, s.data(), f.data()));
  std::copy(s.begin(), s.end(), sigma.begin());
  std::copy(f.begin(), f.end(), features.begin());
}

// rgb of n samples from their density features, unit directions and appearance rows
inline void query_color(std::span<const double> features, std::span<const Vec3> directions,
                        std::span<const double> appearance, const FieldParams& params, std::span<Vec3> rgb) {
  const size_t n = directions.size();
  if (features.size() != n * kDensityFeatureWidth || appearance.size() != n * params.appearance_dim ||
      rgb.size() != n)
    throw std::invalid_argument("field: query_color input size");
  if (!n) return;
  const std::vector<float> f(features.begin(), features.end()), a(appearance.begin(), appearance.end());
  std::vector<float> d(3 * n), out(3 * n);
  for (size_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) d[3 * i + k] = float(directions[i][k]);
  detail::check(dg_field_color(params.device(), 0, params.slot(), f.data(), d.data(), a.data(), n, out.data()));
  for (size_t i = 0; i < n; ++i) rgb[i] = Vec3(out[3 * i], out[3 * i + 1], out[3 * i + 2]);
}

// field_backward over n samples (dL/dsigma, dL/drgb each); grads += the parameter gradients
inline void field_backward(const FieldParams& params, std::span<const Vec3> points, std::span<const Vec3> directions,
                           std::span<const double> appearance, std::span<const double> sigma_grad,
                           std::span<const Vec3> color_grad, FieldGrads& grads) {
  const size_t n = points.size();
  if (directions.size() != n || sigma_grad.size() != n || color_grad.size() != n ||
      appearance.size() != n * params.appearance_dim)
    throw std::invalid_argument("field: backward input size");
  if (!n) return;
  std::vector<float> d(3 * n), a(appearance.begin(), appearance.end()), sg(sigma_grad.begin(), sigma_grad.end()),
      cg(3 * n);
  for (size_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      d[3 * i + k] = float(directions[i][k]);
      cg[3 * i + k] = float(color_grad[i][k]);
    }
  dg_ctx* c = params.device();
  detail::check(dg_zero_grads(c));
  detail::check(dg_field_backward(c, 0, params.slot(), reinterpret_cast<const double*>(points.data()), d.data(),
                                  a.data(), sg.data(), cg.data(), n, DG_MEM_HOST));
  params.device_state().add_grads(params.slot(), grads.arrays());
}

// ---- the reference's per-sample calls ----
inline DensityResult query_density(const Vec3& point, const FieldParams& params, FieldSampleCache* cache = nullptr) {
  DensityResult r;
  query_density(std::span<const Vec3>(&point, 1), params, std::span<double>(&r.sigma, 1), r.feature);
  if (cache) {
    cache->point = point;
    cache->sigma = r.sigma;
    cache->density_feature.assign(r.feature.begin(), r.feature.end());
  }
  return r;
}

inline Vec3 query_color(std::span<const double> density_feature, const Vec3& direction,
                        std::span<const double> appearance, const FieldParams& params,
                        FieldSampleCache* cache = nullptr) {
  if (density_feature.size() != kDensityFeatureWidth) throw std::invalid_argument("field: feature width");
  if (appearance.size() != params.appearance_dim) throw std::invalid_argument("field: appearance width");
  Vec3 rgb;
  query_color(density_feature, std::span<const Vec3>(&direction, 1), appearance, params, std::span<Vec3>(&rgb, 1));
  if (cache) {
    cache->direction = direction;
    cache->appearance.assign(appearance.begin(), appearance.end());
    cache->color = rgb;
  }
  return rgb;
}

// `sigma` is the forward's density (the device recomputes it from the cached point)
inline void field_backward(const FieldParams& params, const FieldSampleCache& cache, double sigma, double sigma_grad,
                           const Vec3& color_grad, FieldGrads& grads) {
  (void)sigma;
  field_backward(params, std::span<const Vec3>(&cache.point, 1), std::span<const Vec3>(&cache.direction, 1),
                 cache.appearance, std::span<const double>(&sigma_grad, 1), std::span<const Vec3>(&color_grad, 1),
                 grads);
}

}  // namespace distgrid
