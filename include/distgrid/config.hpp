// distgrid/config.hpp — RunConfig with the reference's field names and defaults
// (config.hpp:13-78), and its mapping onto the C ABI's dg_run_config (the manifest supplies
// the boxes and the tiling).  Host-only.  Not here: the JSON I/O and the FNV-1a hash of the
// canonical serialization (config I/O is outside the per-ray path; checkpoint calls take the
// caller's hash verbatim).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "distgrid/train.hpp"
#include "distgrid_b200.h"

namespace distgrid {

struct RunConfig {
  std::string dataset_dir;
  std::string out_dir = "out";
  uint32_t partitions_x = 1;
  uint32_t partitions_y = 1;
  std::string transport = "local";  // the device path exchanges over NCCL / peer memory instead
  uint16_t tcp_base_port = 29700;
  uint64_t seed = 1;
  bool wire_f32 = false;

  uint32_t fine_table_log2 = 15;
  uint32_t coarse_table_log2 = 12;
  uint32_t grid_levels = 8;
  uint32_t grid_features = 2;
  uint32_t base_resolution = 16;
  uint32_t max_resolution = 512;
  uint32_t appearance_dim = 16;

  double march_step_divisor = 1024.0;  // step = longest outer axis / divisor

  uint32_t occ_resolution = 128;
  double occ_decay = 0.99;
  uint64_t occ_warmup_steps = 4096;
  uint64_t occ_update_interval = 16;
  double occ_threshold_early = 0.6;
  double occ_threshold_late = 60.0;
  uint64_t occ_threshold_switch_step = 10000;
  double occ_threshold_scale = 1.0;

  uint64_t total_steps = 20000;
  uint32_t batch_size = 4096;
  uint64_t cache_capacity = 1ull << 20;
  uint64_t cache_refresh_interval = 64;
  uint64_t cache_refresh_count = 16384;
  LossConfig loss;
  double lr_start = 0.05;
  double lr_end = 0.005;
  bool distortion_cross_correction = false;

  double altitude_margin = 0.25;

  bool eval_early_termination = false;
  double eval_termination_threshold = 1e-4;

  uint64_t log_interval = 100;
  uint64_t checkpoint_interval = 0;

  // config.cpp:23-36; the device path adds its own limits (grid_features == 2, <= 16 levels,
  // <= 64 partitions) when the context is created.
  void validate() const {
    if (partitions_x < 1 || partitions_y < 1) throw std::invalid_argument("config: partitions must be >= 1");
    if (transport != "local" && transport != "tcp")
      throw std::invalid_argument("config: transport must be 'local' or 'tcp'");
    if (batch_size == 0 || total_steps == 0)
      throw std::invalid_argument("config: batch_size and total_steps must be positive");
    if (march_step_divisor <= 0.0) throw std::invalid_argument("config: march_step_divisor must be positive");
    if (!(loss.transmittance_clamp > 0.0 && loss.transmittance_clamp < 1.0))
      throw std::invalid_argument("config: transmittance clamp must be in (0,1)");
    if (loss.lambda_transmittance < 0.0 || loss.lambda_distortion < 0.0)
      throw std::invalid_argument("config: loss weights must be non-negative");
  }
};

// RunConfig + the manifest's boxes -> the ABI struct (dg_default_config fills the Adam
// constants of Worker::Setup, worker.hpp:79-80).
inline dg_run_config to_dg_config(const RunConfig& r, const double inner_lo[3], const double inner_hi[3],
                                  const double outer_lo[3], const double outer_hi[3], double ground_altitude) {
  dg_run_config c;
  dg_default_config(&c);
  for (int a = 0; a < 3; ++a) {
    c.inner_lo[a] = inner_lo[a];
    c.inner_hi[a] = inner_hi[a];
    c.outer_lo[a] = outer_lo[a];
    c.outer_hi[a] = outer_hi[a];
  }
  c.ground_altitude = ground_altitude;
  c.kx = r.partitions_x;
  c.ky = r.partitions_y;
  c.grid_levels = r.grid_levels;
  c.grid_features = r.grid_features;
  c.base_resolution = r.base_resolution;
  c.max_resolution = r.max_resolution;
  c.fine_table_log2 = r.fine_table_log2;
  c.coarse_table_log2 = r.coarse_table_log2;
  c.appearance_dim = r.appearance_dim;
  c.march_step_divisor = r.march_step_divisor;
  c.occ_resolution = r.occ_resolution;
  c.occ_decay = r.occ_decay;
  c.occ_warmup_steps = r.occ_warmup_steps;
  c.occ_update_interval = r.occ_update_interval;
  c.occ_threshold_early = r.occ_threshold_early;
  c.occ_threshold_late = r.occ_threshold_late;
  c.occ_threshold_switch_step = r.occ_threshold_switch_step;
  c.occ_threshold_scale = r.occ_threshold_scale;
  c.seed = r.seed;
  c.total_steps = r.total_steps;
  c.lr_start = r.lr_start;
  c.lr_end = r.lr_end;
  c.lambda_transmittance = r.loss.lambda_transmittance;
  c.lambda_distortion = r.loss.lambda_distortion;
  c.transmittance_clamp = r.loss.transmittance_clamp;
  c.wire_f32 = r.wire_f32 ? 1u : 0u;
  c.distortion_cross_correction = r.distortion_cross_correction ? 1u : 0u;
  c.occupancy_updates = 1;
  c.eval_early_termination = r.eval_early_termination ? 1u : 0u;
  c.eval_termination_threshold = r.eval_termination_threshold;
  return c;
}

}  // namespace distgrid
