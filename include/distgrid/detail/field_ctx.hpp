// distgrid/detail/field_ctx.hpp — the device side of one facade field object (HashGrid,
// FieldParams): a one-region context whose fine and coarse sub-fields both have the object's
// grid shape (box = [0, aspect]), so a fine field lives in cascade slot 0 and a coarse one (with
// its sigmoid colour network) in slot 1.  The object's host arrays (the reference's value
// semantics) are uploaded as fp32 before device work; gradients come back from the context's
// sink and are added into the caller's host sink (+=, as the reference accumulates).
#pragma once

#include <cmath>
#include <memory>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "distgrid/detail/device.hpp"

namespace distgrid {
namespace detail {

class FieldCtx {
 public:
  // extent: the grid's aspect (box [0, extent]); table_log2 for both sub-fields
  FieldCtx(const double extent[3], uint32_t levels, uint32_t base_res, uint32_t max_res, uint32_t table_log2,
           uint32_t appearance_dim) {
    dg_run_config c;
    dg_default_config(&c);
    for (int a = 0; a < 3; ++a) {
      c.inner_lo[a] = c.outer_lo[a] = 0.0;
      c.inner_hi[a] = c.outer_hi[a] = extent[a];
    }
    c.kx = c.ky = 1;
    c.grid_levels = levels;
    c.base_resolution = base_res;
    c.max_resolution = max_res;
    c.fine_table_log2 = c.coarse_table_log2 = table_log2;
    c.appearance_dim = appearance_dim;
    c.occ_resolution = 8;
    c.occupancy_updates = 0;
    dg_ctx* raw = nullptr;
    check(dg_ctx_create(&c, -1, 0, 1, &raw));
    ctx_.reset(raw);
    uint64_t n = 0;
    check(dg_param_count(raw, 0, &n));
    flat_.assign(n, 0.f);
    uint32_t na = 0;
    arrays_.resize(64);
    check(dg_param_layout(raw, 0, arrays_.data(), uint32_t(arrays_.size()), &na));
    arrays_.resize(na);
  }

  dg_ctx* get() const { return ctx_.get(); }

  // The slot's arrays in FieldParams::parameter_arrays order (levels, density W b W b, colour
  // W b W b W b); a field with fewer arrays (a bare HashGrid) passes only its levels.
  void upload(uint32_t slot, const std::vector<std::span<const double>>& arrays) {
    size_t k = 0;
    for (const dg_array_desc& a : arrays_) {
      if (a.cascade != slot) continue;
      if (k >= arrays.size()) break;
      if (arrays[k].size() != a.size) throw std::invalid_argument("field: parameter array size mismatch");
      for (uint64_t i = 0; i < a.size; ++i) flat_[a.offset + i] = float(arrays[k][i]);
      ++k;
    }
    check(dg_set_params(ctx_.get(), 0, flat_.data()));
  }

  // Adds the slot's device gradients into `sinks` (same order as upload) and zeroes the sink
  // on the device.
  void add_grads(uint32_t slot, const std::vector<std::span<double>>& sinks) {
    std::vector<float> g(flat_.size());
    check(dg_get_grads(ctx_.get(), 0, g.data()));
    check(dg_zero_grads(ctx_.get()));
    size_t k = 0;
    for (const dg_array_desc& a : arrays_) {
      if (a.cascade != slot) continue;
      if (k >= sinks.size()) break;
      for (uint64_t i = 0; i < a.size; ++i) sinks[k][i] += double(g[a.offset + i]);
      ++k;
    }
  }

 private:
  CtxPtr ctx_;
  std::vector<float> flat_;
  std::vector<dg_array_desc> arrays_;
};

// Holder that is empty again after a copy: a copied field object builds its own context.
template <class T>
struct DeviceSlot {
  std::unique_ptr<T> p;
  DeviceSlot() = default;
  DeviceSlot(const DeviceSlot&) {}
  DeviceSlot& operator=(const DeviceSlot&) {
    p.reset();
    return *this;
  }
  DeviceSlot(DeviceSlot&&) = default;
  DeviceSlot& operator=(DeviceSlot&&) = default;
};

inline uint32_t log2_exact(uint32_t v) {
  uint32_t l = 0;
  while ((1u << l) < v) ++l;
  if ((1u << l) != v) throw std::invalid_argument("grid: table_length must be a power of two");
  return l;
}

}  // namespace detail
}  // namespace distgrid
