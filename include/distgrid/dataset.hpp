// distgrid/dataset.hpp — the dataset value types the batch feed reads (dataset.hpp:10-86):
// Image, TransmittanceMap, Dataset, SupervisedRay.  The pixel rays themselves are built on the
// device by the ray cache (train.hpp RayCache -> dg_ray_cache_*, make_pixel_ray's arithmetic).
// Not here: PPM / pose / transmittance-map file I/O and the synthetic dataset generator
// (scene rendering with the quadrature oracle) — dataset production, outside the per-ray path.
#pragma once

#include <cstdint>
#include <vector>

#include "distgrid/geometry.hpp"
#include "distgrid/partition.hpp"
#include "distgrid/vecmath.hpp"

namespace distgrid {

struct Image {
  uint32_t width = 0, height = 0;
  std::vector<uint8_t> rgb;  // interleaved, row-major, top-left origin

  double pixel_channel(uint32_t x, uint32_t y, int c) const {
    return double(rgb[(size_t(y) * width + x) * 3 + c]) / 255.0;
  }
};

struct TransmittanceMap {
  uint32_t width = 0, height = 0;
  std::vector<float> values;
};

struct Dataset {
  std::vector<Image> images;
  std::vector<TransmittanceMap> transmittance;  // optional
  std::vector<CameraPose> poses;                // aligned with images
  std::vector<uint8_t> is_train;                // 1 train, 0 validation

  size_t size() const { return images.size(); }
  std::vector<uint32_t> split_ids(bool train) const {
    std::vector<uint32_t> ids;
    for (size_t i = 0; i < poses.size(); ++i)
      if ((is_train[i] != 0) == train) ids.push_back(poses[i].image_id);
    return ids;
  }
};

struct SupervisedRay {
  Ray ray;
  Vec3 color_gt;
  uint32_t image_id = 0;
};

}  // namespace distgrid
