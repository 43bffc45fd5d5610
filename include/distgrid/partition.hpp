// distgrid/partition.hpp — the spatial partition of the reference API (partition.hpp:11-91):
// CameraPose, RegionBox, PartitionManifest (region_at, validate), split_regions and
// segment_ray.  The manifest is host-side setup, built exactly as partition.cpp:206-252 builds
// it (planes computed once, shared bitwise).  segment_ray runs the device kernel
// (k_segment_home's segment_ray, bit-exact fp64) on a context configured with the manifest;
// segment_rays does a whole batch in one launch.
// Not here: project_fov_footprint / compute_boxes and the manifest JSON I/O (scene setup from
// camera poses, outside the per-ray path).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <span>
#include <stdexcept>
#include <tuple>
#include <vector>

#include "distgrid/detail/device.hpp"
#include "distgrid/geometry.hpp"
#include "distgrid/render.hpp"
#include "distgrid/vecmath.hpp"

namespace distgrid {

struct CameraPose {
  uint32_t image_id = 0;
  Mat3 rotation;     // camera-to-world
  Vec3 translation;  // camera centre
  double fx = 0.0, fy = 0.0;
  double cx = 0.0, cy = 0.0;
  uint32_t width = 0, height = 0;

  // R R^T = I within 1e-6, det R = +1, positive focal lengths, non-empty image
  void validate() const {
    const Mat3 rt = rotation.transposed();
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double v = 0.0;
        for (int k = 0; k < 3; ++k) v += rotation(r, k) * rt(k, c);
        if (std::abs(v - (r == c ? 1.0 : 0.0)) > 1e-6) throw std::invalid_argument("pose: rotation is not orthonormal");
      }
    if (std::abs(rotation.det() - 1.0) > 1e-6) throw std::invalid_argument("pose: rotation determinant is not +1");
    if (fx <= 0.0 || fy <= 0.0 || width == 0 || height == 0) throw std::invalid_argument("pose: invalid intrinsics");
  }
  Vec3 pixel_ray_dir(double x, double y) const {
    return normalize(rotation * Vec3((x - cx) / fx, (y - cy) / fy, 1.0));
  }
};

struct RegionBox {
  uint32_t region_id = 0;
  Aabb fine;    // the region's reconstructed core
  Aabb coarse;  // extended to the outer bounds on scene-edge sides
  std::vector<uint32_t> neighbor_ids;
};

struct PartitionManifest {
  uint32_t kx = 1, ky = 1;
  Aabb inner, outer;
  double ground_altitude = 0.0;
  std::vector<RegionBox> regions;
  std::vector<double> x_planes, y_planes;  // kx + 1 / ky + 1 values, inner bounds included

  uint32_t region_count() const { return kx * ky; }

  // cell containing (x, y): upper_bound over the interior planes, clamped to the edge cells
  uint32_t region_at(double x, double y) const {
    auto cell = [](const std::vector<double>& pl, double v) {
      return uint32_t(std::upper_bound(pl.begin() + 1, pl.end() - 1, v) - pl.begin() - 1);
    };
    return cell(y_planes, y) * kx + cell(x_planes, x);
  }

  // partition.cpp:47-85: the tiling is closely paved (shared boundaries bitwise equal).
  void validate() const {
    auto fail = [](const char* m) { throw std::runtime_error(std::string("manifest: ") + m); };
    if (regions.size() != size_t(kx) * ky) fail("region count");
    if (x_planes.size() != kx + 1 || y_planes.size() != ky + 1) fail("plane count");
    if (x_planes.front() != inner.lo.x || x_planes.back() != inner.hi.x || y_planes.front() != inner.lo.y ||
        y_planes.back() != inner.hi.y)
      fail("planes do not span the inner box");
    for (size_t i = 0; i + 1 < x_planes.size(); ++i)
      if (!(x_planes[i] < x_planes[i + 1])) fail("x planes not increasing");
    for (size_t i = 0; i + 1 < y_planes.size(); ++i)
      if (!(y_planes[i] < y_planes[i + 1])) fail("y planes not increasing");
    double fine_volume = 0.0;
    for (uint32_t iy = 0; iy < ky; ++iy)
      for (uint32_t ix = 0; ix < kx; ++ix) {
        const RegionBox& r = regions[size_t(iy) * kx + ix];
        if (r.region_id != iy * kx + ix) fail("region id order");
        if (r.fine.lo.x != x_planes[ix] || r.fine.hi.x != x_planes[ix + 1] || r.fine.lo.y != y_planes[iy] ||
            r.fine.hi.y != y_planes[iy + 1])
          fail("fine box not aligned to planes (overlap or gap)");
        if (r.fine.lo.z != inner.lo.z || r.fine.hi.z != inner.hi.z) fail("altitude range not shared");
        if (!r.coarse.contains(r.fine)) fail("fine not inside coarse");
        const Vec3 clo(ix == 0 ? outer.lo.x : x_planes[ix], iy == 0 ? outer.lo.y : y_planes[iy], outer.lo.z);
        const Vec3 chi(ix == kx - 1 ? outer.hi.x : x_planes[ix + 1], iy == ky - 1 ? outer.hi.y : y_planes[iy + 1],
                       outer.hi.z);
        if (r.coarse.lo.x != clo.x || r.coarse.hi.x != chi.x || r.coarse.lo.y != clo.y || r.coarse.hi.y != chi.y)
          fail("coarse box not aligned to planes (overlap or gap)");
        if (r.coarse.lo.z != outer.lo.z || r.coarse.hi.z != outer.hi.z) fail("coarse altitude range");
        fine_volume += r.fine.volume();
      }
    if (std::abs(fine_volume - inner.volume()) > 1e-9 * std::max(1.0, inner.volume()))
      fail("fine boxes do not tile the inner box");
  }
};

inline PartitionManifest split_regions(const Aabb& inner, const Aabb& outer, uint32_t kx, uint32_t ky,
                                       double ground_altitude) {
  if (kx < 1 || ky < 1) throw std::invalid_argument("split_regions: kx, ky must be >= 1");
  PartitionManifest m;
  m.kx = kx;
  m.ky = ky;
  m.inner = inner;
  m.outer = outer;
  m.ground_altitude = ground_altitude;
  auto planes = [](double lo, double hi, uint32_t k) {
    std::vector<double> p(k + 1);
    for (uint32_t i = 0; i <= k; ++i)
      p[i] = i == 0 ? lo : i == k ? hi : lo + (hi - lo) * double(i) / double(k);
    return p;
  };
  m.x_planes = planes(inner.lo.x, inner.hi.x, kx);
  m.y_planes = planes(inner.lo.y, inner.hi.y, ky);
  for (uint32_t id = 0; id < kx * ky; ++id) {
    const uint32_t ix = id % kx, iy = id / kx;
    RegionBox r;
    r.region_id = id;
    r.fine = Aabb(Vec3(m.x_planes[ix], m.y_planes[iy], inner.lo.z),
                  Vec3(m.x_planes[ix + 1], m.y_planes[iy + 1], inner.hi.z));
    r.coarse = Aabb(Vec3(ix == 0 ? outer.lo.x : m.x_planes[ix], iy == 0 ? outer.lo.y : m.y_planes[iy], outer.lo.z),
                    Vec3(ix + 1 == kx ? outer.hi.x : m.x_planes[ix + 1],
                         iy + 1 == ky ? outer.hi.y : m.y_planes[iy + 1], outer.hi.z));
    for (int dy = -1; dy <= 1; ++dy)  // 8-neighbourhood in row-major order
      for (int dx = -1; dx <= 1; ++dx) {
        const int nx = int(ix) + dx, ny = int(iy) + dy;
        if ((dx || dy) && nx >= 0 && ny >= 0 && nx < int(kx) && ny < int(ky))
          r.neighbor_ids.push_back(uint32_t(ny) * kx + uint32_t(nx));
      }
    m.regions.push_back(std::move(r));
  }
  m.validate();
  return m;
}

namespace pdetail {
inline void boxes(const PartitionManifest& m, double il[3], double ih[3], double ol[3], double oh[3]) {
  for (int a = 0; a < 3; ++a) {
    il[a] = m.inner.lo[a];
    ih[a] = m.inner.hi[a];
    ol[a] = m.outer.lo[a];
    oh[a] = m.outer.hi[a];
  }
}

// A small device context carrying the manifest's geometry (its planes are recomputed from
// the boxes with the same expression, so they equal the manifest's bitwise; a manifest with
// other planes is rejected).  Cached per thread for the last manifest seen.
inline dg_ctx* manifest_ctx(const PartitionManifest& m) {
  using Key = std::tuple<std::vector<double>, std::vector<double>, std::vector<double>, double>;
  thread_local Key key;
  thread_local detail::CtxPtr ctx;
  double il[3], ih[3], ol[3], oh[3];
  boxes(m, il, ih, ol, oh);
  Key k{m.x_planes, m.y_planes, {il[0], il[1], il[2], ih[0], ih[1], ih[2], ol[0], ol[1], ol[2], oh[0], oh[1], oh[2]},
        m.ground_altitude};
  if (ctx && k == key) return ctx.get();
  const PartitionManifest ref = split_regions(m.inner, m.outer, m.kx, m.ky, m.ground_altitude);
  if (ref.x_planes != m.x_planes || ref.y_planes != m.y_planes)
    throw std::invalid_argument("segment_ray: the device path needs split_regions' equal-width planes");
  dg_run_config c;
  dg_default_config(&c);
  for (int a = 0; a < 3; ++a) {
    c.inner_lo[a] = il[a];
    c.inner_hi[a] = ih[a];
    c.outer_lo[a] = ol[a];
    c.outer_hi[a] = oh[a];
  }
  c.ground_altitude = m.ground_altitude;
  c.kx = m.kx;
  c.ky = m.ky;
  c.grid_levels = 1;  // geometry only: the smallest grids the context accepts
  c.base_resolution = c.max_resolution = 2;
  c.fine_table_log2 = c.coarse_table_log2 = 4;
  c.occ_resolution = 8;
  c.occupancy_updates = 0;
  dg_ctx* raw = nullptr;
  detail::check(dg_ctx_create(&c, -1, 0, 1, &raw));
  ctx.reset(raw);
  key = std::move(k);
  return raw;
}
}  // namespace pdetail

// Batched segment_ray: out[i] lists ray i's segments ordered by t_enter (ray_id = pixel_id).
inline std::vector<std::vector<RaySegment>> segment_rays(std::span<const Ray> rays, const PartitionManifest& m) {
  const size_t n = rays.size();
  std::vector<double> o(3 * n), d(3 * n), te(n * DG_MAX_SEGMENTS), tx(n * DG_MAX_SEGMENTS);
  std::vector<uint8_t> ns(n);
  std::vector<uint16_t> reg(n * DG_MAX_SEGMENTS);
  for (size_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      o[3 * i + a] = rays[i].origin[a];
      d[3 * i + a] = rays[i].dir[a];
    }
  detail::check(dg_segment_rays(pdetail::manifest_ctx(m), o.data(), d.data(), n, ns.data(), reg.data(), te.data(),
                                tx.data(), DG_MEM_HOST));
  std::vector<std::vector<RaySegment>> out(n);
  for (size_t i = 0; i < n; ++i)
    for (uint32_t s = 0; s < ns[i]; ++s) {
      const size_t k = i * DG_MAX_SEGMENTS + s;
      out[i].push_back(RaySegment{rays[i].pixel_id, reg[k], s, te[k], tx[k]});
    }
  return out;
}

inline std::vector<RaySegment> segment_ray(const Ray& ray, const PartitionManifest& manifest) {
  return segment_rays(std::span<const Ray>(&ray, 1), manifest)[0];
}

}  // namespace distgrid
