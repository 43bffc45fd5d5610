// distgrid/geometry.hpp — Ray, RayInterval and the slab test of the reference API
// (geometry.hpp:12-35), over the device kernel k_ray_aabb (geometry.cpp:7-28 restated with
// correctly rounded fp64 intrinsics, bit-exact).  The batched overload is the one to use in
// bulk: one launch for n rays.
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <vector>

#include "distgrid/detail/device.hpp"
#include "distgrid/vecmath.hpp"

namespace distgrid {

struct Ray {
  Vec3 origin;
  Vec3 dir;  // unit length
  uint64_t pixel_id = 0;
  uint32_t image_id = 0;

  Vec3 at(double t) const { return origin + dir * t; }
};

struct RayInterval {
  double t_near = 0.0;
  double t_far = 0.0;
};

// Batched slab test: out[i] is the clipped (t >= 0) overlap of ray i with `box`, or empty.
inline std::vector<std::optional<RayInterval>> ray_aabb_intersect(std::span<const Vec3> origins,
                                                                  std::span<const Vec3> dirs,
                                                                  const Aabb& box) {
  if (origins.size() != dirs.size()) throw std::invalid_argument("ray_aabb_intersect: size mismatch");
  const size_t n = origins.size();
  static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 is three packed doubles");
  std::vector<uint8_t> hit(n);
  std::vector<double> tn(n), tf(n);
  const double lo[3] = {box.lo.x, box.lo.y, box.lo.z}, hi[3] = {box.hi.x, box.hi.y, box.hi.z};
  detail::check(dg_ray_aabb(detail::stage_ctx(), reinterpret_cast<const double*>(origins.data()),
                            reinterpret_cast<const double*>(dirs.data()), n, lo, hi, hit.data(), tn.data(),
                            tf.data(), DG_MEM_HOST));
  std::vector<std::optional<RayInterval>> out(n);
  for (size_t i = 0; i < n; ++i)
    if (hit[i]) out[i] = RayInterval{tn[i], tf[i]};
  return out;
}

inline std::optional<RayInterval> ray_aabb_intersect(const Vec3& origin, const Vec3& dir, const Aabb& box) {
  return ray_aabb_intersect(std::span<const Vec3>(&origin, 1), std::span<const Vec3>(&dir, 1), box)[0];
}

inline std::optional<RayInterval> ray_aabb_intersect(const Ray& ray, const Aabb& box) {
  return ray_aabb_intersect(ray.origin, ray.dir, box);
}

}  // namespace distgrid
