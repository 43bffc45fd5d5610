// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libdistgrid_ref.so).
// It lets the Python tests, the golden-fixture generator and bench.py's reference arm
// call the reference's own code path:
//   DistributedRun::training_step / evaluate_rays   (proj/src/worker.cpp:730-834)
//   segment_ray, cascade_march, HashGrid::encode, query_density/query_color,
//   field_backward, AdamState::step                  (the stage functions of SURVEY §8a)
// Nothing here is shipped or measured as the product; the product is libdg_b200.so.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "distgrid/checkpoint.hpp"
#include "distgrid/config.hpp"
#include "distgrid/dataset.hpp"
#include "distgrid/field.hpp"
#include "distgrid/partition.hpp"
#include "distgrid/render.hpp"
#include "distgrid/train.hpp"
#include "distgrid/worker.hpp"
#include "distgrid_b200.h"

using namespace distgrid;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}

RunConfig to_run_config(const dg_run_config& c) {
  RunConfig r;
  r.partitions_x = c.kx;
  r.partitions_y = c.ky;
  r.transport = "local";
  r.seed = c.seed;
  r.wire_f32 = c.wire_f32 != 0;
  r.fine_table_log2 = c.fine_table_log2;
  r.coarse_table_log2 = c.coarse_table_log2;
  r.grid_levels = c.grid_levels;
  r.grid_features = c.grid_features;
  r.base_resolution = c.base_resolution;
  r.max_resolution = c.max_resolution;
  r.appearance_dim = c.appearance_dim;
  r.march_step_divisor = c.march_step_divisor;
  r.occ_resolution = c.occ_resolution;
  r.occ_decay = c.occ_decay;
  r.occ_warmup_steps = c.occ_warmup_steps;
  r.occ_update_interval = c.occ_update_interval;
  r.occ_threshold_early = c.occ_threshold_early;
  r.occ_threshold_late = c.occ_threshold_late;
  r.occ_threshold_switch_step = c.occ_threshold_switch_step;
  r.occ_threshold_scale = c.occ_threshold_scale;
  r.total_steps = c.total_steps;
  r.loss.lambda_transmittance = c.lambda_transmittance;
  r.loss.lambda_distortion = c.lambda_distortion;
  r.loss.transmittance_clamp = c.transmittance_clamp;
  r.lr_start = c.lr_start;
  r.lr_end = c.lr_end;
  r.distortion_cross_correction = c.distortion_cross_correction != 0;
  r.eval_early_termination = c.eval_early_termination != 0;
  r.eval_termination_threshold = c.eval_termination_threshold;
  return r;
}

Aabb box_of(const double lo[3], const double hi[3]) {
  return Aabb{Vec3{lo[0], lo[1], lo[2]}, Vec3{hi[0], hi[1], hi[2]}};
}

PartitionManifest manifest_of(const dg_run_config& c) {
  return split_regions(box_of(c.inner_lo, c.inner_hi), box_of(c.outer_lo, c.outer_hi), c.kx, c.ky,
                       c.ground_altitude);
}

struct Harness {
  RunConfig config;
  PartitionManifest manifest;
  AppearanceTable appearance;
  std::unique_ptr<DistributedRun> run;
  // Per-region stand-alone fields for stage calls (copies of the worker fields).
  std::vector<FieldGrads> stage_grads_fine, stage_grads_coarse;
};

std::vector<std::span<double>> all_arrays(Worker& w) {
  std::vector<std::span<double>> a;
  for (auto& s : w.fine_field().parameter_arrays()) a.push_back(s);
  for (auto& s : w.coarse_field().parameter_arrays()) a.push_back(s);
  return a;
}

std::vector<std::span<double>> grad_arrays(FieldGrads& g) {
  std::vector<std::span<double>> a;
  for (auto& l : g.grid.level_grads) a.emplace_back(l);
  for (auto& layer : g.density_mlp) {
    a.emplace_back(layer.weights);
    a.emplace_back(layer.bias);
  }
  for (auto& layer : g.color_mlp) {
    a.emplace_back(layer.weights);
    a.emplace_back(layer.bias);
  }
  return a;
}

}  // namespace

extern "C" {

const char* refh_last_error() { return g_err.c_str(); }

void* refh_create(const dg_run_config* cfg, uint32_t n_images, const double* app_rows) {
  try {
    auto h = std::make_unique<Harness>();
    h->config = to_run_config(*cfg);
    h->manifest = manifest_of(*cfg);
    h->appearance.dim = cfg->appearance_dim;
    for (uint32_t i = 0; i < n_images; ++i) h->appearance.image_ids.push_back(i);
    h->appearance.rows.assign(app_rows, app_rows + size_t(n_images) * cfg->appearance_dim);
    h->run = std::make_unique<DistributedRun>(h->config, h->manifest, h->appearance);
    for (uint32_t r = 0; r < h->run->worker_count(); ++r) {
      h->stage_grads_fine.push_back(make_field_grads(h->run->worker(r).fine_field()));
      h->stage_grads_coarse.push_back(make_field_grads(h->run->worker(r).coarse_field()));
    }
    return h.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void refh_destroy(void* p) { delete static_cast<Harness*>(p); }

uint64_t refh_param_count(void* p, uint32_t region) {
  auto* h = static_cast<Harness*>(p);
  uint64_t n = 0;
  for (auto& a : all_arrays(h->run->worker(region))) n += a.size();
  return n;
}

int refh_get_params(void* p, uint32_t region, double* out) {
  auto* h = static_cast<Harness*>(p);
  for (auto& a : all_arrays(h->run->worker(region))) {
    std::memcpy(out, a.data(), a.size() * sizeof(double));
    out += a.size();
  }
  return 0;
}

int refh_set_params(void* p, uint32_t region, const double* in) {
  auto* h = static_cast<Harness*>(p);
  for (auto& a : all_arrays(h->run->worker(region))) {
    std::memcpy(a.data(), in, a.size() * sizeof(double));
    in += a.size();
  }
  return 0;
}

// Adam moments are private to Worker; the checkpoint round trip is the reference's own
// accessor (worker.cpp:602-626).
int refh_get_adam(void* p, uint32_t region, double* m, double* v, uint64_t* step_count,
                  uint64_t* worker_step) {
  auto* h = static_cast<Harness*>(p);
  const WorkerCheckpoint ck = h->run->worker(region).make_checkpoint(0);
  for (const auto& a : ck.adam.first_moments()) {
    std::memcpy(m, a.data(), a.size() * sizeof(double));
    m += a.size();
  }
  for (const auto& a : ck.adam.second_moments()) {
    std::memcpy(v, a.data(), a.size() * sizeof(double));
    v += a.size();
  }
  *step_count = ck.adam.step_count();
  *worker_step = ck.step;
  return 0;
}

int refh_set_adam(void* p, uint32_t region, const double* m, const double* v, uint64_t step_count,
                  uint64_t worker_step) {
  auto* h = static_cast<Harness*>(p);
  try {
    Worker& w = h->run->worker(region);
    WorkerCheckpoint ck = w.make_checkpoint(0);
    for (auto& a : ck.adam.first_moments()) {
      std::memcpy(a.data(), m, a.size() * sizeof(double));
      m += a.size();
    }
    for (auto& a : ck.adam.second_moments()) {
      std::memcpy(a.data(), v, a.size() * sizeof(double));
      v += a.size();
    }
    ck.adam.set_step_count(step_count);
    ck.step = worker_step;
    w.load_state(ck);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// bits: one u8 per cell; density := threshold where set, 0 elsewhere.
int refh_set_occupancy(void* p, uint32_t region, uint32_t cascade, const uint8_t* bits) {
  auto* h = static_cast<Harness*>(p);
  Worker& w = h->run->worker(region);
  OccupancyGrid& occ = cascade == 0 ? w.occ_fine() : w.occ_coarse();
  for (uint64_t i = 0; i < occ.cell_count(); ++i)
    occ.density()[i] = bits[i] ? occ.threshold() : 0.0;
  occ.recompute_bitfield();
  return 0;
}

int refh_get_occupancy(void* p, uint32_t region, uint32_t cascade, uint8_t* bits, double* density) {
  auto* h = static_cast<Harness*>(p);
  Worker& w = h->run->worker(region);
  const OccupancyGrid& occ = cascade == 0 ? w.occ_fine() : w.occ_coarse();
  for (uint64_t i = 0; i < occ.cell_count(); ++i) {
    bits[i] = occ.bitfield()[i];
    if (density) density[i] = occ.density()[i];
  }
  return 0;
}

// DistributedRun::training_step on the given batch. stats: loss_rgb, loss_t, loss_dist, lr,
// rays, dropped.
int refh_train_step(void* p, const double* origin, const double* dir, const double* color_gt,
                    const uint32_t* image_id, uint64_t n, uint64_t step, double* stats) {
  auto* h = static_cast<Harness*>(p);
  try {
    std::vector<SupervisedRay> batch(n);
    for (uint64_t i = 0; i < n; ++i) {
      batch[i].ray.origin = {origin[3 * i], origin[3 * i + 1], origin[3 * i + 2]};
      batch[i].ray.dir = {dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]};
      batch[i].ray.pixel_id = i;
      batch[i].image_id = image_id ? image_id[i] : 0;
      batch[i].ray.image_id = batch[i].image_id;
      batch[i].color_gt = {color_gt[3 * i], color_gt[3 * i + 1], color_gt[3 * i + 2]};
    }
    h->run->start();
    StepStats s;
    try {
      s = h->run->training_step(batch, step);
    } catch (...) {
      h->run->stop();
      throw;
    }
    h->run->stop();
    stats[0] = s.loss_rgb;
    stats[1] = s.loss_transmittance;
    stats[2] = s.loss_distortion;
    stats[3] = s.lr;
    stats[4] = double(s.rays);
    stats[5] = double(s.dropped_rays);
    stats[6] = double(s.bytes_sent);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int refh_eval_rays(void* p, const double* origin, const double* dir, uint64_t n,
                   const double* appearance, double* rgb, double* transmittance, double* depth) {
  auto* h = static_cast<Harness*>(p);
  try {
    std::vector<Ray> rays(n);
    for (uint64_t i = 0; i < n; ++i) {
      rays[i].origin = {origin[3 * i], origin[3 * i + 1], origin[3 * i + 2]};
      rays[i].dir = {dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]};
      rays[i].pixel_id = i;
    }
    std::vector<double> app(appearance, appearance + h->config.appearance_dim);
    h->run->start();
    std::vector<MergedRender> out;
    try {
      out = h->run->evaluate_rays(rays, app);
    } catch (...) {
      h->run->stop();
      throw;
    }
    h->run->stop();
    for (uint64_t i = 0; i < n; ++i) {
      for (int k = 0; k < 3; ++k) rgb[3 * i + k] = out[i].color[k];
      transmittance[i] = out[i].transmittance;
      depth[i] = out[i].depth;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// DistributedRun::evaluate_image (worker.cpp:836-880): colour, T, depth, attribution per pixel.
int refh_eval_image(void* p, const dg_camera* cam, const double* appearance, double* rgb,
                    double* transmittance, double* depth, double* attribution) {
  auto* h = static_cast<Harness*>(p);
  try {
    CameraPose pose;
    pose.image_id = cam->image_id;
    for (int j = 0; j < 9; ++j) pose.rotation.m[j] = cam->rotation[j];
    pose.translation = Vec3{cam->translation[0], cam->translation[1], cam->translation[2]};
    pose.fx = cam->fx;
    pose.fy = cam->fy;
    pose.cx = cam->cx;
    pose.cy = cam->cy;
    pose.width = cam->width;
    pose.height = cam->height;
    std::vector<double> app(appearance, appearance + h->config.appearance_dim);
    h->run->start();
    EvalImage img;
    try {
      img = h->run->evaluate_image(pose, app);
    } catch (...) {
      h->run->stop();
      throw;
    }
    h->run->stop();
    const uint64_t n = uint64_t(cam->width) * cam->height;
    for (uint64_t i = 0; i < n; ++i) {
      for (int k = 0; k < 3; ++k) {
        rgb[3 * i + k] = img.color[i][k];
        attribution[3 * i + k] = img.attribution[i][k];
      }
      transmittance[i] = img.transmittance[i];
      depth[i] = img.depth[i];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- stage functions ----

int refh_segment_rays(const dg_run_config* cfg, const double* origin, const double* dir,
                      uint64_t n, uint8_t* nseg, uint16_t* region, double* t_enter,
                      double* t_exit) {
  try {
    const PartitionManifest m = manifest_of(*cfg);
    for (uint64_t i = 0; i < n; ++i) {
      Ray ray{{origin[3 * i], origin[3 * i + 1], origin[3 * i + 2]},
              {dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]}, i, 0};
      const auto segs = segment_ray(ray, m);
      nseg[i] = uint8_t(segs.size());
      for (size_t s = 0; s < segs.size(); ++s) {
        region[i * DG_MAX_SEGMENTS + s] = uint16_t(segs[s].region_id);
        t_enter[i * DG_MAX_SEGMENTS + s] = segs[s].t_enter;
        t_exit[i * DG_MAX_SEGMENTS + s] = segs[s].t_exit;
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// cascade_march for n (ray, [t0,t1]) pairs in `region`; samples written consecutively.
int refh_cascade_march(void* p, uint32_t region_id, const double* origin, const double* dir,
                       const double* t0, const double* t1, const uint64_t* ray_id, uint64_t n,
                       int jitter, uint64_t batch_id, uint32_t* counts, double* t, double* delta,
                       uint8_t* cascade, uint64_t capacity) {
  auto* h = static_cast<Harness*>(p);
  try {
    Worker& w = h->run->worker(region_id);
    MarchConfig march;
    march.step = march_step_for(h->config, h->manifest.outer);
    march.jitter = jitter != 0;
    march.jitter_seed = h->config.seed;
    march.jitter_step = batch_id;
    uint64_t off = 0;
    for (uint64_t i = 0; i < n; ++i) {
      Ray ray{{origin[3 * i], origin[3 * i + 1], origin[3 * i + 2]},
              {dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]}, ray_id[i], 0};
      const auto samples = cascade_march(ray, w.region(), w.occ_fine(), w.occ_coarse(), t0[i], t1[i],
                                         march, ray_id[i]);
      counts[i] = uint32_t(samples.size());
      for (const auto& s : samples) {
        if (off >= capacity) throw std::out_of_range("harness: sample capacity");
        t[off] = s.sample.t;
        delta[off] = s.sample.delta;
        cascade[off] = s.cascade;
        ++off;
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// HashGrid::encode; rows: n x L x 8 (UINT32_MAX for w == 0 corners), via table_index.
int refh_encode(void* p, uint32_t region_id, uint32_t cascade, const double* points, uint64_t n,
                double* out, uint32_t* rows) {
  auto* h = static_cast<Harness*>(p);
  try {
    Worker& w = h->run->worker(region_id);
    const HashGrid& grid = cascade == 0 ? w.fine_field().grid : w.coarse_field().grid;
    const uint32_t width = grid.feature_width();
    const uint32_t L = grid.config().levels;
    for (uint64_t i = 0; i < n; ++i) {
      const Vec3 pt{points[3 * i], points[3 * i + 1], points[3 * i + 2]};
      grid.encode(pt, std::span<double>(out + i * width, width));
      if (rows) {
        for (uint32_t l = 0; l < L; ++l) {
          const HashGridLevel& level = grid.levels()[l];
          const uint32_t ext[3] = {level.shape.nx, level.shape.ny, level.shape.nz};
          uint32_t i0[3], i1[3];
          double frac[3];
          for (int a = 0; a < 3; ++a) {
            if (ext[a] == 1) {
              i0[a] = i1[a] = 0;
              frac[a] = 0.0;
              continue;
            }
            const double pos = pt[a] * double(ext[a] - 1);
            uint32_t lo = uint32_t(std::floor(pos));
            if (lo > ext[a] - 1) lo = ext[a] - 1;
            i0[a] = lo;
            i1[a] = std::min(lo + 1, ext[a] - 1);
            frac[a] = pos - double(lo);
          }
          for (int c = 0; c < 8; ++c) {
            const int cx = c & 1, cy = (c >> 1) & 1, cz = (c >> 2) & 1;
            const double wgt = (cx ? frac[0] : 1.0 - frac[0]) * (cy ? frac[1] : 1.0 - frac[1]) *
                               (cz ? frac[2] : 1.0 - frac[2]);
            rows[(i * L + l) * 8 + c] =
                wgt == 0.0 ? 0xffffffffu
                           : table_index(cx ? i1[0] : i0[0], cy ? i1[1] : i0[1], cz ? i1[2] : i0[2],
                                         level);
          }
        }
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int refh_field_forward(void* p, uint32_t region_id, uint32_t cascade, const double* points,
                       const double* dirs, const double* appearance, uint64_t n, double* sigma,
                       double* rgb) {
  auto* h = static_cast<Harness*>(p);
  try {
    Worker& w = h->run->worker(region_id);
    const FieldParams& f = cascade == 0 ? w.fine_field() : w.coarse_field();
    const uint32_t d = h->config.appearance_dim;
    for (uint64_t i = 0; i < n; ++i) {
      const Vec3 pt{points[3 * i], points[3 * i + 1], points[3 * i + 2]};
      const Vec3 dir{dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]};
      const DensityResult r = query_density(pt, f);
      const Vec3 c = query_color(r.feature, dir, std::span<const double>(appearance + i * d, d), f);
      sigma[i] = r.sigma;
      for (int k = 0; k < 3; ++k) rgb[3 * i + k] = c[k];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// field_backward accumulated into the harness's own grad sink for (region, cascade).
int refh_field_backward(void* p, uint32_t region_id, uint32_t cascade, const double* points,
                        const double* dirs, const double* appearance, const double* sigma_grad,
                        const double* rgb_grad, uint64_t n) {
  auto* h = static_cast<Harness*>(p);
  try {
    Worker& w = h->run->worker(region_id);
    const FieldParams& f = cascade == 0 ? w.fine_field() : w.coarse_field();
    FieldGrads& g = cascade == 0 ? h->stage_grads_fine[region_id] : h->stage_grads_coarse[region_id];
    const uint32_t d = h->config.appearance_dim;
    for (uint64_t i = 0; i < n; ++i) {
      const Vec3 pt{points[3 * i], points[3 * i + 1], points[3 * i + 2]};
      const Vec3 dir{dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]};
      FieldSampleCache cache;
      const DensityResult r = query_density(pt, f, &cache);
      query_color(r.feature, dir, std::span<const double>(appearance + i * d, d), f, &cache);
      field_backward(f, cache, r.sigma, sigma_grad[i],
                     Vec3{rgb_grad[3 * i], rgb_grad[3 * i + 1], rgb_grad[3 * i + 2]}, g);
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Flat (fine then coarse) stage-gradient sink of a region; zero it with zero != 0.
int refh_stage_grads(void* p, uint32_t region_id, double* out, int zero) {
  auto* h = static_cast<Harness*>(p);
  for (FieldGrads* g : {&h->stage_grads_fine[region_id], &h->stage_grads_coarse[region_id]}) {
    for (auto& a : grad_arrays(*g)) {
      if (out) {
        std::memcpy(out, a.data(), a.size() * sizeof(double));
        out += a.size();
      }
    }
    if (zero) g->zero();
  }
  return 0;
}

double refh_march_step(void* p) {
  auto* h = static_cast<Harness*>(p);
  return march_step_for(h->config, h->manifest.outer);
}

// Reference default config (config.hpp), expressed as a dg_run_config.
void refh_default_config(dg_run_config* c) {
  const RunConfig r;
  std::memset(c, 0, sizeof(*c));
  for (int a = 0; a < 3; ++a) {
    c->inner_lo[a] = c->outer_lo[a] = 0.0;
    c->inner_hi[a] = c->outer_hi[a] = 1.0;
  }
  c->kx = r.partitions_x;
  c->ky = r.partitions_y;
  c->grid_levels = r.grid_levels;
  c->grid_features = r.grid_features;
  c->base_resolution = r.base_resolution;
  c->max_resolution = r.max_resolution;
  c->fine_table_log2 = r.fine_table_log2;
  c->coarse_table_log2 = r.coarse_table_log2;
  c->appearance_dim = r.appearance_dim;
  c->march_step_divisor = r.march_step_divisor;
  c->occ_resolution = r.occ_resolution;
  c->occ_decay = r.occ_decay;
  c->occ_warmup_steps = r.occ_warmup_steps;
  c->occ_update_interval = r.occ_update_interval;
  c->occ_threshold_early = r.occ_threshold_early;
  c->occ_threshold_late = r.occ_threshold_late;
  c->occ_threshold_switch_step = r.occ_threshold_switch_step;
  c->occ_threshold_scale = r.occ_threshold_scale;
  c->seed = r.seed;
  c->total_steps = r.total_steps;
  c->lr_start = r.lr_start;
  c->lr_end = r.lr_end;
  c->lambda_transmittance = r.loss.lambda_transmittance;
  c->lambda_distortion = r.loss.lambda_distortion;
  c->transmittance_clamp = r.loss.transmittance_clamp;
  const AdamConfig ad;
  c->adam_beta1 = ad.beta1;
  c->adam_beta2 = ad.beta2;
  c->adam_eps = ad.eps;
  c->wire_f32 = r.wire_f32;
  c->distortion_cross_correction = r.distortion_cross_correction;
  c->occupancy_updates = 1;
  c->eval_early_termination = r.eval_early_termination;
  c->eval_termination_threshold = r.eval_termination_threshold;
}

// ---- CPU baseline: T replicas of the reference DistributedRun, one per host thread ----
// Each replica trains on its own slice of the rays (the reference has no intra-worker
// parallelism, worker.cpp:268-312); returns wall seconds for `steps` lock-step iterations.
double refh_time_replicas(void* const* runs, uint32_t n_runs, const double* origin,
                          const double* dir, const double* color_gt, uint64_t rays_per_run,
                          uint64_t steps, uint64_t first_step) {
  std::vector<std::thread> threads;
  std::vector<std::exception_ptr> errs(n_runs);
  const auto t0 = std::chrono::steady_clock::now();
  for (uint32_t r = 0; r < n_runs; ++r) {
    threads.emplace_back([&, r] {
      try {
        auto* h = static_cast<Harness*>(runs[r]);
        std::vector<SupervisedRay> batch(rays_per_run);
        for (uint64_t i = 0; i < rays_per_run; ++i) {
          const uint64_t j = r * rays_per_run + i;
          batch[i].ray.origin = {origin[3 * j], origin[3 * j + 1], origin[3 * j + 2]};
          batch[i].ray.dir = {dir[3 * j], dir[3 * j + 1], dir[3 * j + 2]};
          batch[i].ray.pixel_id = i;
          batch[i].color_gt = {color_gt[3 * j], color_gt[3 * j + 1], color_gt[3 * j + 2]};
        }
        h->run->start();
        for (uint64_t s = 0; s < steps; ++s) h->run->training_step(batch, first_step + s);
        h->run->stop();
      } catch (...) {
        errs[r] = std::current_exception();
      }
    });
  }
  for (auto& t : threads) t.join();
  const auto t1 = std::chrono::steady_clock::now();
  for (auto& e : errs)
    if (e) {
      try {
        std::rethrow_exception(e);
      } catch (const std::exception& ex) {
        fail(ex);
        return -1.0;
      }
    }
  return std::chrono::duration<double>(t1 - t0).count();
}

// ---- CPU baseline (ii): the reference's stage functions on a host thread pool ----
// Throughputs of region 0's own functions: out[0] segment_ray + cascade_march (rays/s),
// out[1] HashGrid::encode (samples/s), out[2] query_density + query_color (samples/s),
// out[3] forward-with-cache + field_backward incl. encode_backward into per-thread FieldGrads
// sinks (samples/s, bwd_threads threads: each sink is a full copy of the tables' shape),
// out[4] AdamState::step over the fine field's arrays, chunked across threads (params/s).
// Reads of grids and fields are thread-safe (const); nothing is written but the sinks.
int refh_stage_bench(void* p, const double* origin, const double* dir, uint64_t n_rays,
                     const double* points, const double* dirs, uint64_t n_pts, int threads,
                     int bwd_threads, double* out) {
  auto* h = static_cast<Harness*>(p);
  try {
    Worker& w = h->run->worker(0);
    const FieldParams& f = w.fine_field();
    const uint32_t dapp = h->config.appearance_dim;
    const std::vector<double> app(dapp, 0.1);
    auto pool = [](int nt, uint64_t n, auto&& body) {
      std::vector<std::thread> ts;
      std::vector<std::exception_ptr> errs(nt);
      const auto t0 = std::chrono::steady_clock::now();
      for (int k = 0; k < nt; ++k)
        ts.emplace_back([&, k] {
          try {
            body(k, n * k / nt, n * (k + 1) / nt);
          } catch (...) {
            errs[k] = std::current_exception();
          }
        });
      for (auto& t : ts) t.join();
      for (auto& e : errs)
        if (e) std::rethrow_exception(e);
      return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    MarchConfig march;
    march.step = march_step_for(h->config, h->manifest.outer);
    march.jitter = true;
    march.jitter_seed = h->config.seed;
    march.jitter_step = 1;
    double sec = pool(threads, n_rays, [&](int, uint64_t lo, uint64_t hi) {
      uint64_t sink = 0;
      for (uint64_t i = lo; i < hi; ++i) {
        Ray ray{{origin[3 * i], origin[3 * i + 1], origin[3 * i + 2]},
                {dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]}, i, 0};
        for (const RaySegment& sg : segment_ray(ray, h->manifest))
          if (sg.region_id == 0)
            sink += cascade_march(ray, w.region(), w.occ_fine(), w.occ_coarse(), sg.t_enter, sg.t_exit, march, i).size();
      }
      if (sink == 0xffffffffffffffffull) throw std::runtime_error("unreachable");
    });
    out[0] = double(n_rays) / sec;
    const uint32_t width = f.grid.feature_width();
    sec = pool(threads, n_pts, [&](int, uint64_t lo, uint64_t hi) {
      std::vector<double> x(width);
      for (uint64_t i = lo; i < hi; ++i)
        f.grid.encode(Vec3{points[3 * i], points[3 * i + 1], points[3 * i + 2]}, x);
    });
    out[1] = double(n_pts) / sec;
    sec = pool(threads, n_pts, [&](int, uint64_t lo, uint64_t hi) {
      for (uint64_t i = lo; i < hi; ++i) {
        const DensityResult r = query_density(Vec3{points[3 * i], points[3 * i + 1], points[3 * i + 2]}, f);
        query_color(r.feature, Vec3{dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]}, app, f);
      }
    });
    out[2] = double(n_pts) / sec;
    std::vector<FieldGrads> sinks;
    for (int k = 0; k < bwd_threads; ++k) sinks.push_back(make_field_grads(f));
    sec = pool(bwd_threads, n_pts, [&](int k, uint64_t lo, uint64_t hi) {
      for (uint64_t i = lo; i < hi; ++i) {
        FieldSampleCache cache;
        const DensityResult r =
            query_density(Vec3{points[3 * i], points[3 * i + 1], points[3 * i + 2]}, f, &cache);
        query_color(r.feature, Vec3{dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]}, app, f, &cache);
        field_backward(f, cache, r.sigma, 0.01, Vec3{0.01, -0.02, 0.03}, sinks[k]);
      }
    });
    out[3] = double(n_pts) / sec;
    sinks.clear();
    // Adam over every fine array, each array cut into `threads` chunks with its own state
    std::vector<std::span<double>> arrays;
    for (auto& a : w.fine_field().parameter_arrays()) arrays.push_back(a);
    uint64_t n_par = 0;
    for (auto& a : arrays) n_par += a.size();
    std::vector<std::vector<double>> params(arrays.size()), grads(arrays.size());
    for (size_t a = 0; a < arrays.size(); ++a) {
      params[a].assign(arrays[a].begin(), arrays[a].end());
      grads[a].assign(arrays[a].size(), 1e-3);
    }
    std::vector<AdamState> states(threads);
    std::vector<std::vector<std::span<double>>> tp(threads);
    std::vector<std::vector<std::span<const double>>> tg(threads);
    for (int k = 0; k < threads; ++k) {
      std::vector<size_t> sizes;
      for (size_t a = 0; a < arrays.size(); ++a) {
        const size_t n = params[a].size(), lo = n * k / threads, hi = n * (k + 1) / threads;
        tp[k].emplace_back(params[a].data() + lo, hi - lo);
        tg[k].emplace_back(grads[a].data() + lo, hi - lo);
        sizes.push_back(hi - lo);
      }
      states[k] = AdamState(sizes);
    }
    sec = pool(threads, uint64_t(threads), [&](int k, uint64_t, uint64_t) { states[k].step(tp[k], tg[k], 0.01); });
    out[4] = double(n_par) / sec;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- .dgcw checkpoints (checkpoint.cpp:241-283) through the Worker's own state calls ----
int refh_save_checkpoint(void* p, uint32_t region, uint64_t config_hash, const char* path) {
  try {
    auto* h = static_cast<Harness*>(p);
    save_worker_checkpoint(path, h->run->worker(region).make_checkpoint(config_hash));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int refh_load_checkpoint(void* p, uint32_t region, const char* path, uint64_t* config_hash) {
  try {
    auto* h = static_cast<Harness*>(p);
    const WorkerCheckpoint ck = load_worker_checkpoint(path);
    h->run->worker(region).load_state(ck);
    if (config_hash) *config_hash = ck.config_hash;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- RayCache / make_pixel_ray (train.cpp:117-159, dataset.cpp:312-324) ----
struct RefRayCache {
  Dataset dataset;
  std::unique_ptr<RayCache> cache;
};

void* refh_ray_cache_create(const dg_camera* cams, const uint8_t* const* images, uint32_t n_images,
                            uint64_t capacity, uint64_t seed) {
  try {
    auto r = std::make_unique<RefRayCache>();
    for (uint32_t i = 0; i < n_images; ++i) {
      const dg_camera& k = cams[i];
      CameraPose pose;
      pose.image_id = k.image_id;
      for (int j = 0; j < 9; ++j) pose.rotation.m[j] = k.rotation[j];
      pose.translation = Vec3{k.translation[0], k.translation[1], k.translation[2]};
      pose.fx = k.fx;
      pose.fy = k.fy;
      pose.cx = k.cx;
      pose.cy = k.cy;
      pose.width = k.width;
      pose.height = k.height;
      Image img;
      img.width = k.width;
      img.height = k.height;
      img.rgb.assign(images[i], images[i] + size_t(k.width) * k.height * 3);
      r->dataset.poses.push_back(pose);
      r->dataset.images.push_back(std::move(img));
      r->dataset.is_train.push_back(k.is_train ? 1 : 0);
    }
    r->cache = std::make_unique<RayCache>(capacity, seed);
    return r.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void refh_ray_cache_destroy(void* p) { delete static_cast<RefRayCache*>(p); }

int refh_ray_cache_refresh(void* p, uint64_t count) {
  try {
    auto* r = static_cast<RefRayCache*>(p);
    r->cache->refresh(r->dataset, count);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

static void put_ray(const SupervisedRay& s, uint64_t i, double* origin, double* dir, double* color,
                    uint32_t* image_id, uint64_t* pixel_id) {
  const double o[3] = {s.ray.origin.x, s.ray.origin.y, s.ray.origin.z};
  const double d[3] = {s.ray.dir.x, s.ray.dir.y, s.ray.dir.z};
  const double c[3] = {s.color_gt.x, s.color_gt.y, s.color_gt.z};
  for (int a = 0; a < 3; ++a) {
    origin[3 * i + a] = o[a];
    dir[3 * i + a] = d[a];
    color[3 * i + a] = c[a];
  }
  image_id[i] = s.image_id;
  pixel_id[i] = s.ray.pixel_id;
}

uint64_t refh_ray_cache_snapshot(void* p, double* origin, double* dir, double* color, uint32_t* image_id,
                                 uint64_t* pixel_id) {
  auto* r = static_cast<RefRayCache*>(p);
  const std::vector<SupervisedRay> e = r->cache->snapshot();
  if (origin)
    for (uint64_t i = 0; i < e.size(); ++i) put_ray(e[i], i, origin, dir, color, image_id, pixel_id);
  return e.size();
}

int refh_ray_cache_draw(void* p, uint64_t n, double* origin, double* dir, double* color, uint32_t* image_id,
                        uint64_t* pixel_id) {
  try {
    auto* r = static_cast<RefRayCache*>(p);
    const std::vector<SupervisedRay> b = r->cache->draw_batch(n);
    for (uint64_t i = 0; i < b.size(); ++i) put_ray(b[i], i, origin, dir, color, image_id, pixel_id);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
