// distgrid/grid.hpp — the multi-resolution hash grid of the reference API (grid.hpp:14-147):
// GridConfig, grid_shape, MappingMode, HashGridLevel, table_index, HashGridGrads, HashGrid and
// the OccupancyGrid value type.  Configuration, shapes and the integer index are host
// functions (they define the layout); HashGrid::encode / encode_backward run the device kernels
// (k_encode_points / k_encode_points_bwd: bit-exact fp64 corner indices and weights, fp32
// tables, fp32 accumulation, red.global scatters) on the grid's own context, and have batched
// overloads for whole point sets.  The host tables are the reference's double arrays; the device
// copy is fp32 (tables are fp32 on the training path).
// occupancy_skip runs the device DDA (k_occupancy_skip, the march's walk over a row-major
// bitfield).  OccupancyGrid::decay_and_update takes the caller's host density callback, so it is
// host bookkeeping around that callback here; the training path's update runs on the device
// inside dg_train_step.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <span>
#include <stdexcept>
#include <vector>

#include "distgrid/detail/field_ctx.hpp"
#include "distgrid/geometry.hpp"
#include "distgrid/rng.hpp"
#include "distgrid/vecmath.hpp"

namespace distgrid {

struct GridConfig {
  uint32_t levels = 8;
  uint32_t table_length = 1u << 15;  // power of two
  uint32_t features_per_level = 2;
  uint32_t base_resolution = 16;
  uint32_t max_resolution = 512;
  Vec3 aspect{1.0, 1.0, 1.0};

  void validate() const {
    if (levels < 1) throw std::invalid_argument("grid: levels must be >= 1");
    if (table_length == 0 || (table_length & (table_length - 1)))
      throw std::invalid_argument("grid: table_length must be a power of two");
    if (features_per_level < 1) throw std::invalid_argument("grid: features_per_level must be >= 1");
    if (base_resolution > max_resolution) throw std::invalid_argument("grid: base_resolution must be <= max_resolution");
    if (!(aspect.x > 0.0 && aspect.y > 0.0 && aspect.z > 0.0))
      throw std::invalid_argument("grid: aspect components must be positive");
  }

  // geometric progression base -> max over the levels (llround of base * growth^level)
  uint32_t level_resolution(uint32_t level) const {
    if (level >= levels) throw std::out_of_range("grid: level index out of range");
    if (levels == 1) return base_resolution;
    const double growth = std::exp((std::log(double(max_resolution)) - std::log(double(base_resolution))) /
                                   double(levels - 1));
    return uint32_t(std::llround(double(base_resolution) * std::pow(growth, double(level))));
  }
};

enum class MappingMode : uint8_t { OneToOne = 0, Hashed = 1 };

struct LevelShape {
  uint32_t nx = 0, ny = 0, nz = 0;
  uint64_t voxel_count() const { return uint64_t(nx) * ny * nz; }
};

inline LevelShape grid_shape(const GridConfig& config, uint32_t level) {
  const double n = double(config.level_resolution(level));
  const double s = max_component(config.aspect);
  return LevelShape{uint32_t(std::ceil(config.aspect.x / s * n)), uint32_t(std::ceil(config.aspect.y / s * n)),
                    uint32_t(std::ceil(config.aspect.z / s * n))};
}

struct HashGridLevel {
  LevelShape shape;
  MappingMode mapping_mode = MappingMode::OneToOne;
  uint32_t features = 2;
  std::vector<double> table;  // rows() x features

  uint32_t rows() const { return uint32_t(table.size() / features); }
};

// Row of lattice vertex (ix, iy, iz): row-major when one-to-one, else the XOR spatial hash with
// primes (1, 2654435761, 805459861) in wrapping u32 arithmetic, masked to the table length.
inline uint32_t table_index(uint32_t ix, uint32_t iy, uint32_t iz, const HashGridLevel& level) {
  if (ix >= level.shape.nx || iy >= level.shape.ny || iz >= level.shape.nz)
    throw std::out_of_range("grid: voxel coordinate out of range");
  if (level.mapping_mode == MappingMode::OneToOne) return ix + level.shape.nx * (iy + level.shape.ny * iz);
  return (ix ^ (iy * 2654435761u) ^ (iz * 805459861u)) & (level.rows() - 1);
}

struct HashGridGrads {
  std::vector<std::vector<double>> level_grads;
  void zero() {
    for (auto& g : level_grads) std::fill(g.begin(), g.end(), 0.0);
  }
};

class HashGrid {
 public:
  HashGrid() = default;
  // tables U[-1e-4, 1e-4] from rng, level by level, row-major (grid.cpp:90-105)
  HashGrid(const GridConfig& config, Rng& rng) : config_(config) {
    config_.validate();
    levels_.resize(config_.levels);
    for (uint32_t l = 0; l < config_.levels; ++l) {
      HashGridLevel& lv = levels_[l];
      lv.shape = grid_shape(config_, l);
      lv.features = config_.features_per_level;
      const bool one_to_one = lv.shape.voxel_count() <= config_.table_length;
      lv.mapping_mode = one_to_one ? MappingMode::OneToOne : MappingMode::Hashed;
      lv.table.resize((one_to_one ? lv.shape.voxel_count() : config_.table_length) * lv.features);
      for (double& v : lv.table) v = rng.uniform(-1e-4, 1e-4);
    }
  }

  const GridConfig& config() const { return config_; }
  // mutable access: the device copy is refreshed before every later device call
  std::vector<HashGridLevel>& levels() {
    exposed_ = true;
    return levels_;
  }
  const std::vector<HashGridLevel>& levels() const { return levels_; }
  uint32_t feature_width() const { return config_.levels * config_.features_per_level; }

  // ---- batched device overloads ----
  // features of n normalised points: out[i * feature_width() + k]
  std::vector<double> encode(std::span<const Vec3> points) const {
    check_points(points);
    const size_t n = points.size(), w = feature_width();
    std::vector<float> f(n * w);
    if (n) detail::check(dg_encode(device(), 0, 0, flat(points), n, f.data(), nullptr, DG_MEM_HOST));
    return std::vector<double>(f.begin(), f.end());
  }
  // grads += sum_i encode_backward(points[i], upstream[i * width ...])
  void encode_backward(std::span<const Vec3> points, std::span<const double> upstream, HashGridGrads& grads) const {
    check_points(points);
    const size_t n = points.size(), w = feature_width();
    if (upstream.size() != n * w) throw std::invalid_argument("grid: encode_backward upstream size");
    if (grads.level_grads.size() != levels_.size()) throw std::invalid_argument("grid: grads shape");
    if (!n) return;
    const std::vector<float> up(upstream.begin(), upstream.end());
    dg_ctx* c = device();
    detail::check(dg_zero_grads(c));
    detail::check(dg_encode_backward(c, 0, 0, flat(points), up.data(), n, DG_MEM_HOST));
    std::vector<std::span<double>> sinks;
    for (auto& g : grads.level_grads) sinks.emplace_back(g);
    dev_.p->add_grads(0, sinks);
  }

  // ---- the reference's per-point calls ----
  void encode(const Vec3& point, std::span<double> out) const {
    if (out.size() != feature_width()) throw std::invalid_argument("grid: encode output size");
    const std::vector<double> f = encode(std::span<const Vec3>(&point, 1));
    std::copy(f.begin(), f.end(), out.begin());
  }
  void encode_backward(const Vec3& point, std::span<const double> upstream, HashGridGrads& grads) const {
    if (upstream.size() != feature_width()) throw std::invalid_argument("grid: encode_backward upstream size");
    encode_backward(std::span<const Vec3>(&point, 1), upstream, grads);
  }

  HashGridGrads make_grads() const {
    HashGridGrads g;
    for (const HashGridLevel& lv : levels_) g.level_grads.emplace_back(lv.table.size(), 0.0);
    return g;
  }

  std::vector<std::span<double>> parameter_arrays() {
    exposed_ = true;
    std::vector<std::span<double>> a;
    for (HashGridLevel& lv : levels_) a.emplace_back(lv.table);
    return a;
  }

  // the grid's context with this object's current tables (HashGrid alone: fine slot 0)
  dg_ctx* device() const {
    if (config_.features_per_level != 2)
      throw std::invalid_argument("grid: the device path requires features_per_level == 2");
    if (!dev_.p) {
      const double ext[3] = {config_.aspect.x, config_.aspect.y, config_.aspect.z};
      dev_.p = std::make_unique<detail::FieldCtx>(ext, config_.levels, config_.base_resolution,
                                                  config_.max_resolution, detail::log2_exact(config_.table_length), 16);
      stale_ = true;
    }
    if (stale_ || exposed_) {
      std::vector<std::span<const double>> a;
      for (const HashGridLevel& lv : levels_) a.emplace_back(lv.table);
      dev_.p->upload(0, a);
      stale_ = false;
    }
    return dev_.p->get();
  }

 private:
  static const double* flat(std::span<const Vec3> p) { return reinterpret_cast<const double*>(p.data()); }
  static void check_points(std::span<const Vec3> points) {
    for (const Vec3& p : points)
      if (p.x < 0.0 || p.x > 1.0 || p.y < 0.0 || p.y > 1.0 || p.z < 0.0 || p.z > 1.0)
        throw std::invalid_argument("grid: encode point outside the unit box");
  }

  GridConfig config_;
  std::vector<HashGridLevel> levels_;
  mutable detail::DeviceSlot<detail::FieldCtx> dev_;
  mutable bool stale_ = true;
  bool exposed_ = false;
};

// Occupancy of one region cascade (grid.hpp:96-140): the bitfield and densities, as a value
// (Worker snapshots fill it from the device; the device update runs inside dg_train_step).
class OccupancyGrid {
 public:
  OccupancyGrid() = default;
  OccupancyGrid(const Aabb& box, uint32_t longest_axis_resolution, double decay = 0.99, double threshold = 0.6)
      : box_(box), decay_(decay), threshold_(threshold) {
    GridConfig g;
    g.levels = 1;
    g.base_resolution = g.max_resolution = longest_axis_resolution;
    g.aspect = box.extent();
    shape_ = grid_shape(g, 0);
    density_.assign(cell_count(), 0.0);
    bitfield_.assign(cell_count(), 0);
  }

  const Aabb& box() const { return box_; }
  LevelShape shape() const { return shape_; }
  double threshold() const { return threshold_; }
  void set_threshold(double t) {
    threshold_ = t;
    recompute_bitfield();
  }
  double decay() const { return decay_; }
  uint64_t cell_count() const { return shape_.voxel_count(); }
  std::vector<double>& density() { return density_; }
  const std::vector<double>& density() const { return density_; }
  const std::vector<uint8_t>& bitfield() const { return bitfield_; }
  bool cell_occupied(uint64_t idx) const { return bitfield_[idx] != 0; }
  uint64_t cell_index(uint32_t ix, uint32_t iy, uint32_t iz) const {
    return ix + uint64_t(shape_.nx) * (iy + uint64_t(shape_.ny) * iz);
  }
  Aabb cell_box(uint32_t ix, uint32_t iy, uint32_t iz) const {
    const Vec3 cell = box_.extent() / Vec3(double(shape_.nx), double(shape_.ny), double(shape_.nz));
    const Vec3 lo = box_.lo + cell * Vec3(double(ix), double(iy), double(iz));
    return Aabb(lo, lo + cell);
  }
  // every cell at the threshold and occupied (the untrained state, worker.cpp:199-200)
  void fill_occupied() {
    std::fill(density_.begin(), density_.end(), threshold_);
    std::fill(bitfield_.begin(), bitfield_.end(), uint8_t(1));
  }
  void recompute_bitfield() {
    for (size_t i = 0; i < density_.size(); ++i) bitfield_[i] = density_[i] >= threshold_ ? 1 : 0;
  }
  // density[i] <- max(density[i] * decay, density_at(jittered point of cell i)) over every cell
  // (warm-up) or 1/4 uniform + 1/4 occupied cells, then the bitfield (grid.cpp:201-229)
  void decay_and_update(const std::function<double(const Vec3&)>& density_at, uint64_t step, bool warm_up,
                        Rng& rng) {
    (void)step;
    const uint64_t total = cell_count();
    auto visit = [&](uint64_t idx) {
      const uint32_t ix = uint32_t(idx % shape_.nx), iy = uint32_t((idx / shape_.nx) % shape_.ny),
                     iz = uint32_t(idx / (uint64_t(shape_.nx) * shape_.ny));
      const Aabb c = cell_box(ix, iy, iz);
      const double px = rng.uniform(c.lo.x, c.hi.x);
      const double py = rng.uniform(c.lo.y, c.hi.y);
      const double pz = rng.uniform(c.lo.z, c.hi.z);
      density_[idx] = std::max(density_[idx] * decay_, density_at(Vec3(px, py, pz)));
    };
    if (warm_up) {
      for (uint64_t i = 0; i < total; ++i) visit(i);
    } else {
      std::vector<uint64_t> occ;
      for (uint64_t i = 0; i < total; ++i)
        if (bitfield_[i]) occ.push_back(i);
      const uint64_t k = std::max<uint64_t>(total / 4, 1);
      for (uint64_t i = 0; i < k; ++i) visit(rng.uniform_index(total));
      if (!occ.empty())
        for (uint64_t i = 0; i < k; ++i) visit(occ[rng.uniform_index(occ.size())]);
    }
    recompute_bitfield();
  }
  // device snapshot (Worker views)
  void assign(std::vector<double> density, std::vector<uint8_t> bits, double threshold) {
    density_ = std::move(density);
    bitfield_ = std::move(bits);
    threshold_ = threshold;
  }

 private:
  Aabb box_;
  LevelShape shape_;
  std::vector<double> density_;
  std::vector<uint8_t> bitfield_;
  double decay_ = 0.99;
  double threshold_ = 0.6;
};

// Batched occupancy_skip: the occupied runs of [t0[i], t1[i]] along rays[i], in increasing t
// (runs of consecutive occupied cells merged; the caller keeps [t0, t1] inside the box).
inline std::vector<std::vector<RayInterval>> occupancy_skip(std::span<const Ray> rays, std::span<const double> t0,
                                                            std::span<const double> t1, const OccupancyGrid& occ) {
  const size_t n = rays.size();
  if (t0.size() != n || t1.size() != n) throw std::invalid_argument("occupancy_skip: size mismatch");
  std::vector<double> o(3 * n), d(3 * n);
  for (size_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      o[3 * i + a] = rays[i].origin[a];
      d[3 * i + a] = rays[i].dir[a];
    }
  const LevelShape sh = occ.shape();
  const uint32_t shape[3] = {sh.nx, sh.ny, sh.nz};
  const double lo[3] = {occ.box().lo.x, occ.box().lo.y, occ.box().lo.z};
  const double hi[3] = {occ.box().hi.x, occ.box().hi.y, occ.box().hi.z};
  std::vector<uint32_t> cnt(n);
  dg_ctx* c = detail::stage_ctx();
  detail::check(dg_occupancy_skip(c, occ.bitfield().data(), shape, lo, hi, o.data(), d.data(), t0.data(), t1.data(),
                                  n, cnt.data(), nullptr, nullptr, DG_MEM_HOST));
  std::vector<uint64_t> off(n + 1, 0);
  for (size_t i = 0; i < n; ++i) off[i + 1] = off[i] + cnt[i];
  std::vector<double> iv(2 * off[n]);
  if (off[n])
    detail::check(dg_occupancy_skip(c, occ.bitfield().data(), shape, lo, hi, o.data(), d.data(), t0.data(),
                                    t1.data(), n, nullptr, off.data(), iv.data(), DG_MEM_HOST));
  std::vector<std::vector<RayInterval>> out(n);
  for (size_t i = 0; i < n; ++i)
    for (uint64_t k = off[i]; k < off[i + 1]; ++k) out[i].push_back(RayInterval{iv[2 * k], iv[2 * k + 1]});
  return out;
}

inline std::vector<RayInterval> occupancy_skip(const Ray& ray, double t0, double t1, const OccupancyGrid& occ) {
  return occupancy_skip(std::span<const Ray>(&ray, 1), std::span<const double>(&t0, 1),
                        std::span<const double>(&t1, 1), occ)[0];
}

}  // namespace distgrid
