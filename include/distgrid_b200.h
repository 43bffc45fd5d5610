/*
 * distgrid_b200.h — the C ABI of the B200-native DistGrid per-ray train/render path.
 *
 * This is the drop-in boundary for the hot path of the reference C++ library
 * (/root/reference/proj, namespace distgrid).  The reference has no FFI; its public
 * boundary is the C++ API in proj/include/distgrid/<module>.hpp.  Each entry point below names
 * the reference interface it replaces (file:line, paths relative to proj/).  The C++
 * facade in include/distgrid_b200/distgrid.hpp re-exposes these under the reference
 * names; Python tests/bench bind them with ctypes (paper_2405_04416_b200/dg.py).
 *
 * Conventions (mirroring the reference):
 *  - every call returns an int status (dg_status); dg_last_error() gives a thread-local
 *    message.  DG_EINVAL <-> std::invalid_argument, DG_ERANGE <-> std::out_of_range,
 *    DG_EPROTO <-> std::runtime_error (protocol / missing partial), DG_ETIMEOUT <->
 *    TransportTimeout, DG_ECUDA / DG_ENCCL for device / collective failures.
 *  - one context per GPU; a context owns every partition p with part_rank[p] == rank.
 *    A context is used from one host thread at a time (mirrors Worker ownership,
 *    worker.hpp:60-63).
 *  - gradients accumulate (+=) into context-owned sinks that dg_adam_step zeroes,
 *    exactly as FieldGrads / AdamState in the reference (worker.cpp:524-547).
 *  - buffers flagged DG_MEM_HOST are staged through the context; DG_MEM_DEVICE pointers
 *    are used in place on the context's stream.
 *
 * No torch types cross this boundary: plain pointers, sizes and PODs only.
 */
#ifndef DISTGRID_B200_H
#define DISTGRID_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DG_ABI_VERSION 2
#define DG_MAX_SEGMENTS 16   /* kx + ky - 1 <= 16  (partition.cpp:254-296) */
#define DG_MAX_PARTITIONS 64 /* kx * ky <= 64 */
#define DG_MAX_LEVELS 16     /* grid_levels; F must be 2 on the device path */

typedef enum dg_status {
  DG_OK = 0,
  DG_EINVAL = 1,
  DG_ERANGE = 2,
  DG_EPROTO = 3,
  DG_ETIMEOUT = 4,
  DG_ECUDA = 5,
  DG_ENCCL = 6,
  DG_ENOMEM = 7
} dg_status;

typedef enum dg_mem { DG_MEM_HOST = 0, DG_MEM_DEVICE = 1 } dg_mem;

/*
 * Run configuration: the RunConfig fields that define the path (config.hpp:13-78)
 * plus the two boxes handed to split_regions (partition.hpp:83-88).
 */
typedef struct dg_run_config {
  /* partition: split_regions(inner, outer, kx, ky, ground_altitude) */
  double inner_lo[3], inner_hi[3];
  double outer_lo[3], outer_hi[3];
  double ground_altitude;
  uint32_t kx, ky;
  /* hash grids (config.hpp:24-30) */
  uint32_t grid_levels;
  uint32_t grid_features;
  uint32_t base_resolution;
  uint32_t max_resolution;
  uint32_t fine_table_log2;
  uint32_t coarse_table_log2;
  uint32_t appearance_dim;
  /* ray marching (config.hpp:33): step = longest outer axis / divisor */
  double march_step_divisor;
  /* occupancy (config.hpp:36-43) */
  uint32_t occ_resolution;
  double occ_decay;
  uint64_t occ_warmup_steps;
  uint64_t occ_update_interval;
  double occ_threshold_early;
  double occ_threshold_late;
  uint64_t occ_threshold_switch_step;
  double occ_threshold_scale;
  /* training (config.hpp:46-58, train.hpp:14-18, 50-54) */
  uint64_t seed;
  uint64_t total_steps;
  double lr_start, lr_end;
  double lambda_transmittance;
  double lambda_distortion;
  double transmittance_clamp;
  double adam_beta1, adam_beta2, adam_eps;
  uint32_t wire_f32;                    /* config.hpp:21 (partials are f32 on this path) */
  uint32_t distortion_cross_correction; /* config.hpp:56 (worker.cpp:289-299, 453-511) */
  uint32_t occupancy_updates;           /* 1: run Worker::update_occupancy cadence */
  uint32_t eval_early_termination;      /* config.hpp:60 (dispatch_eval, worker.cpp:815-818) */
  double eval_termination_threshold;    /* config.hpp:61 */
} dg_run_config;

/* RunConfig defaults (config.hpp:13-78) with inner = outer = [0,1]^3. */
void dg_default_config(dg_run_config* cfg);

/* A batch of supervised rays (dataset.hpp:79-83: SupervisedRay), structure of arrays.
 * Ray ids are batch indices (worker.cpp:153): ray i of this shard has global id
 * first_ray_id + i, which keys the per-ray jitter (worker.cpp:258-262). */
typedef struct dg_ray_batch {
  const double* origin;     /* n x 3 */
  const double* dir;        /* n x 3, unit */
  const float* color_gt;    /* n x 3 (train only; may be NULL for render) */
  const uint32_t* image_id; /* n (may be NULL: image 0) */
  uint64_t n;
  uint64_t first_ray_id;
  int32_t mem;              /* dg_mem of all four arrays */
  int32_t reserved;
} dg_ray_batch;

/* worker.hpp:153-162 StepStats (losses are sums over rays, unweighted by lambda). */
typedef struct dg_step_stats {
  uint64_t step;
  double loss_rgb;
  double loss_transmittance;
  double loss_distortion;
  double lr;
  uint64_t rays;
  uint64_t dropped_rays;
  uint64_t bytes_sent;   /* exchange bytes (both exchanges), this rank */
  uint64_t samples;      /* march samples shaded on this rank */
  uint64_t items;        /* (ray, partition) segments owned by this rank */
  uint64_t h2d_bytes;    /* host->device bytes this call moved (batch staging + tables) */
  uint64_t d2h_bytes;    /* device->host bytes this call moved (counts, losses) */
  /* exchange 2 alone (PartialScatter, wire.cpp:72-90): bytes and records this rank sent to
   * other ranks (DistributedRun::scatter_payload_bytes / scatter_entries) */
  uint64_t partial_bytes_sent;
  uint64_t partial_records_sent;
} dg_step_stats;

/* render.hpp:38-43 MergedRender, structure of arrays. */
typedef struct dg_merged {
  float* rgb;           /* n x 3 */
  float* transmittance; /* n */
  float* depth;         /* n */
  float* attribution;   /* n x 3 or NULL: region-attribution colour (evaluate_image, worker.cpp:864-878) */
  int32_t mem;
  int32_t reserved;
} dg_merged;

/* One parameter array of a partition's flat state, in the order of
 * FieldParams::parameter_arrays (field.cpp:203-208) for fine then coarse, which is the
 * order AdamState sees in Worker::apply_updates (worker.cpp:524-547). */
typedef struct dg_array_desc {
  uint64_t offset; /* in floats, into the partition's flat parameter vector */
  uint64_t size;
  uint32_t cascade; /* 0 fine, 1 coarse */
  uint32_t kind;    /* 0 grid level, 1 density W, 2 density b, 3 color W, 4 color b */
  uint32_t index;   /* level or layer index */
  uint32_t reserved;
} dg_array_desc;

typedef struct dg_ctx dg_ctx;

const char* dg_last_error(void);
int dg_abi_version(void);

/* ---- context (replaces Worker construction, worker.cpp:178-206; DistributedRun ctor
 * worker.cpp:630-690).  Partition p lives on rank p % world.  device < 0: use the
 * current device.  Parameters start zeroed: call dg_init_params_reference or
 * dg_set_params.  Occupancy starts fill_occupied (worker.cpp:199-200). ---- */
int dg_ctx_create(const dg_run_config* cfg, int device, int rank, int world, dg_ctx** out);
int dg_ctx_destroy(dg_ctx* ctx);
int dg_partition_count(const dg_ctx* ctx, uint32_t* n_total, uint32_t* n_local);
int dg_partition_rank(const dg_ctx* ctx, uint32_t partition, int* rank);
int dg_march_step(const dg_ctx* ctx, double* step); /* worker.cpp:923-925 */
/* region boxes after split_regions (partition.cpp:206-252) */
int dg_region_boxes(const dg_ctx* ctx, uint32_t partition, double fine_lo[3], double fine_hi[3],
                    double coarse_lo[3], double coarse_hi[3]);
/* level shapes (grid.cpp:65-73), mapping modes and rows (grid.cpp:90-105) */
int dg_grid_levels(const dg_ctx* ctx, uint32_t partition, uint32_t cascade, uint32_t* shapes /*L x 3*/,
                   uint32_t* modes /*L*/, uint64_t* rows /*L*/);

/* ---- state: injection for parity, extraction for checkpoints ---- */
int dg_param_count(const dg_ctx* ctx, uint32_t partition, uint64_t* n_floats);
int dg_param_layout(const dg_ctx* ctx, uint32_t partition, dg_array_desc* arrays,
                    uint32_t capacity, uint32_t* n_arrays);
int dg_set_params(dg_ctx* ctx, uint32_t partition, const float* host_params);
int dg_get_params(dg_ctx* ctx, uint32_t partition, float* host_params);
int dg_get_grads(dg_ctx* ctx, uint32_t partition, float* host_grads);
int dg_zero_grads(dg_ctx* ctx);
int dg_set_adam(dg_ctx* ctx, uint32_t partition, const float* m, const float* v, uint64_t step_count);
int dg_get_adam(dg_ctx* ctx, uint32_t partition, float* m, float* v, uint64_t* step_count);
/* Worker::step_ (worker.hpp:144): the lr schedule index of the next step. */
int dg_set_step(dg_ctx* ctx, uint64_t step);
int dg_get_step(const dg_ctx* ctx, uint64_t* step);
/* In-memory snapshot of the whole training state on the device (parameters, Adam moments
 * and t, occupancy bitfields / densities / thresholds / sampling stream, step counter):
 * restore = 0 takes it, restore = 1 puts it back (gradients zeroed), so a window of steps
 * can be replayed from identical state. */
int dg_state_snapshot(dg_ctx* ctx, int restore);
/* Reference-exact initialisation (worker.cpp:186-190, grid.cpp:90-105, mlp.cpp:38-53):
 * mt19937_64 streams seeded with counter_hash(seed, 0xf1e1d|0xc0a45e, region), rounded
 * to fp32.  Host-side, once per partition (not on the per-step path). */
int dg_init_params_reference(dg_ctx* ctx, uint32_t partition);
/* Fast device-side random init for throughput runs: tables U[-1e-4,1e-4], Xavier MLPs,
 * counter-hash stream (not the reference's mt19937 stream). */
int dg_init_params_fast(dg_ctx* ctx, uint32_t partition, uint64_t seed);
/* Occupancy bitfields (grid.hpp:99-141), one u8 per cell, row-major ix-fastest. */
int dg_occupancy_shape(const dg_ctx* ctx, uint32_t partition, uint32_t cascade, uint32_t shape[3]);
int dg_set_occupancy(dg_ctx* ctx, uint32_t partition, uint32_t cascade, const uint8_t* bits);
int dg_get_occupancy(dg_ctx* ctx, uint32_t partition, uint32_t cascade, uint8_t* bits);
/* OccupancyGrid density (fp32 here, f64 in the reference) and current threshold; set
 * recomputes the bitfield as density >= threshold (grid.hpp:99-141). */
int dg_get_occupancy_density(dg_ctx* ctx, uint32_t partition, uint32_t cascade, float* density,
                             double* threshold);
int dg_set_occupancy_density(dg_ctx* ctx, uint32_t partition, uint32_t cascade, const float* density,
                             double threshold);
int dg_get_config(const dg_ctx* ctx, dg_run_config* out);

/* ---- checkpoint interop: the reference's per-worker .dgcw file
 * (checkpoint.cpp:241-283, v1): both cascade fields as f32 tables / MLPs behind shape headers,
 * both occupancy grids (f32 density, f32 threshold), Adam moments as f64.  config_hash is the
 * caller's RunConfig::hash() (config.cpp:163-166), written verbatim and returned on load;
 * region_id = partition.  A GPU-trained partition can be loaded by the reference
 * (Worker::load_state) and vice versa. */
int dg_save_checkpoint(dg_ctx* ctx, uint32_t partition, uint64_t config_hash, const char* path);
int dg_load_checkpoint(dg_ctx* ctx, uint32_t partition, const char* path, uint64_t* config_hash);
/* Appearance rows (field.hpp:21-29 AppearanceTable); image ids must be < 2^20. */
int dg_set_appearance(dg_ctx* ctx, const uint32_t* image_ids, const float* rows, uint32_t n_images);

/* ---- composed path ---- */
/* DistributedRun::training_step (worker.cpp:730-755) + Worker::handle_training_batch
 * (worker.cpp:251-401) for this rank's partitions.  With world > 1 every rank passes its
 * home shard (contiguous global ray ids) and the exchanges run over the communicator. */
int dg_train_step(dg_ctx* ctx, const dg_ray_batch* batch, uint64_t step, dg_step_stats* stats);
/* DistributedRun::evaluate_rays (worker.cpp:757-834): jitter off, partials merged at the
 * home rank in schedule order, depth carried.  appearance: appearance_dim floats (host). */
int dg_render(dg_ctx* ctx, const dg_ray_batch* batch, const float* appearance, dg_merged* out);
/* DistributedRun::evaluate_image (worker.cpp:836-880): every pixel of one camera (dg_camera,
 * declared with the ray cache below), rays built on the device; out holds width*height
 * entries row-major, attribution (region palette weighted by absorbed transmittance) if set. */
struct dg_camera;
int dg_render_image(dg_ctx* ctx, const struct dg_camera* camera, const float* appearance, dg_merged* out);

/* ---- communicator (replaces transport.hpp:30-98) ---- */
#define DG_NCCL_UNIQUE_ID_BYTES 128
int dg_comm_unique_id(uint8_t id[DG_NCCL_UNIQUE_ID_BYTES]);
int dg_comm_init_nccl(dg_ctx* ctx, const uint8_t id[DG_NCCL_UNIQUE_ID_BYTES]);
/* Host-staged exchange: the context copies send blocks to host and calls back
 * (used for multi-process tests over gloo; never the production path). */
typedef int (*dg_alltoallv_fn)(void* user, const void* send, const uint64_t* send_bytes,
                                void* recv, const uint64_t* recv_bytes);
int dg_comm_init_host(dg_ctx* ctx, dg_alltoallv_fn fn, void* user);
/* Peer-memory backend (one node): every rank's receive buffers are CUDA-IPC mapped into the
 * others, and the dispatch / partial pack kernels store each record directly into its owner's
 * buffer in the owner's final layout.  fn is a host all-gather (recv = world x bytes, rank
 * order) that carries the per-step count matrices, the IPC handles and the barriers; the
 * caller implements it over its launcher's channel (MPI, torch.distributed, sockets). */
typedef int (*dg_allgather_fn)(void* user, const void* send, uint64_t bytes, void* recv);
int dg_comm_init_peer(dg_ctx* ctx, dg_allgather_fn fn, void* user);
/* How long a step waits for its peers before failing (Worker::Setup::recv_timeout,
 * worker.hpp:82; default 120000 ms).  On expiry the step returns DG_ETIMEOUT ("missing
 * PartialScatter", worker.cpp:340-347) and an NCCL communicator is aborted (ncclCommAbort);
 * an asynchronous NCCL failure returns DG_ENCCL.  An aborted context must be recreated. */
int dg_set_comm_timeout(dg_ctx* ctx, uint64_t timeout_ms);

/* ---- ray cache / pixel-ray batch feed ----
 * RayCache (train.cpp:117-159) over a dataset uploaded once: images (u8 RGB, row-major) and
 * camera poses (partition.hpp:15-28).  refresh() samples `count` (train image, pixel) pairs
 * from the reference's refresh stream and builds the rays on the device with make_pixel_ray
 * (dataset.cpp:312-324); draw() picks entries with the reference's draw stream and gathers
 * them into a device-resident dg_ray_batch (owned by the cache, valid until the next draw)
 * that dg_train_step consumes directly. */
typedef struct dg_camera {
  uint32_t image_id, width, height, is_train;
  double rotation[9]; /* camera-to-world, row-major */
  double translation[3];
  double fx, fy, cx, cy;
} dg_camera;
typedef struct dg_ray_cache dg_ray_cache;
int dg_ray_cache_create(int device, const dg_camera* cams, const uint8_t* const* images, uint32_t n_images,
                        uint64_t capacity, uint64_t seed, dg_ray_cache** out);
void dg_ray_cache_destroy(dg_ray_cache* cache);
int dg_ray_cache_size(const dg_ray_cache* cache, uint64_t* size, uint64_t* capacity);
int dg_ray_cache_refresh(dg_ray_cache* cache, uint64_t count);
int dg_ray_cache_draw(dg_ray_cache* cache, uint64_t n, dg_ray_batch* out);
int dg_ray_cache_snapshot(dg_ray_cache* cache, double* origin, double* dir, float* color_gt,
                          uint32_t* image_id, uint64_t* pixel_id);
/* dg_ray_cache_draw into host arrays (n x 3 origin / dir / colour, n image ids, n pixel ids). */
int dg_ray_cache_draw_host(dg_ray_cache* cache, uint64_t n, double* origin, double* dir, float* color_gt,
                           uint32_t* image_id, uint64_t* pixel_id);

/* ---- exchange planning (host only, no context or device needed) ----
 * The layouts both per-step exchanges use (exchange_plan.h), exported so multi-process tests
 * can check the protocol on CPU.  Partition p lives on rank p % world.
 * dg_plan_dispatch: send_cnt[P] records this rank sends to each partition, cnt_recv[W*P] the
 * count vectors of every rank -> send/recv bytes per rank (72-byte records), item_off[nl+1]
 * of the local partitions, and the W*nl block permutation recv [src][lp] -> items [lp][src].
 * dg_plan_partials: pair_cnt[nl*P] (items of local lq whose schedule contains p) -> P*P
 * stream offsets (records) and send/recv bytes per rank (24-byte records). */
int dg_plan_dispatch(int rank, int world, uint32_t P, const uint64_t* send_cnt, const uint64_t* cnt_recv,
                     uint64_t* send_bytes, uint64_t* recv_bytes, uint32_t* item_off, uint64_t* block_src,
                     uint64_t* block_dst);
int dg_plan_partials(int rank, int world, uint32_t P, const uint32_t* pair_cnt, uint64_t* send_off,
                     uint64_t* recv_off, uint64_t* send_bytes, uint64_t* recv_bytes);

/* ---- stage entry points (per-stage parity + the facade's batched overloads) ---- */
/* segment_ray over a batch (partition.cpp:254-296, geometry.cpp:7-28): nseg per ray,
 * region/t_enter/t_exit in n x DG_MAX_SEGMENTS slots.  Bit-exact fp64. */
int dg_segment_rays(dg_ctx* ctx, const double* origin, const double* dir, uint64_t n,
                    uint8_t* nseg, uint16_t* region, double* t_enter, double* t_exit, int32_t mem);
/* cascade_march (worker.cpp:79-110) for n (ray, segment) pairs owned by `partition`.
 * Pass t/delta/cascade == NULL to get counts only; otherwise offsets (exclusive scan of
 * counts) place each ray's samples.  Bit-exact fp64. */
int dg_cascade_march(dg_ctx* ctx, uint32_t partition, const double* origin, const double* dir,
                     const double* t0, const double* t1, const uint64_t* ray_id, uint64_t n,
                     int32_t jitter, uint64_t batch_id, uint32_t* counts, const uint64_t* offsets,
                     double* t, double* delta, uint8_t* cascade, int32_t mem);
/* HashGrid::encode over n normalised points (grid.cpp:107-130).  rows (optional):
 * n x L x 8 table rows (UINT32_MAX for skipped zero-weight corners), bit-exact. */
int dg_encode(dg_ctx* ctx, uint32_t partition, uint32_t cascade, const double* points, uint64_t n,
              float* features, uint32_t* rows, int32_t mem);
/* HashGrid::encode_backward (grid.cpp:132-157): accumulates into the grad sink. */
int dg_encode_backward(dg_ctx* ctx, uint32_t partition, uint32_t cascade, const double* points,
                       const float* upstream, uint64_t n, int32_t mem);
/* query_density + query_color (field.cpp:230-288) on normalised points. */
int dg_field_forward(dg_ctx* ctx, uint32_t partition, uint32_t cascade, const double* points,
                     const float* dirs, const float* appearance, uint64_t n, float* sigma,
                     float* rgb, int32_t mem);
/* query_density (field.cpp:230-254) alone: sigma = exp(clip(raw0)) and the 15 clipped density
 * features per point (host buffers). */
int dg_field_density(dg_ctx* ctx, uint32_t partition, uint32_t cascade, const double* points, uint64_t n,
                     float* sigma, float* features);
/* query_color (field.cpp:256-288) alone from caller-given density features (n x 15), unit
 * directions and appearance rows (n x appearance_dim) -> rgb (host buffers). */
int dg_field_color(dg_ctx* ctx, uint32_t partition, uint32_t cascade, const float* features, const float* dirs,
                   const float* appearance, uint64_t n, float* rgb);
/* field_backward (field.cpp:290-327): accumulates into the grad sink. */
int dg_field_backward(dg_ctx* ctx, uint32_t partition, uint32_t cascade, const double* points,
                      const float* dirs, const float* appearance, const float* sigma_grad,
                      const float* rgb_grad, uint64_t n, int32_t mem);
/* Worker::apply_updates (worker.cpp:524-547): dense Adam over every local parameter with
 * lr = LrSchedule::at(step_) (train.cpp:77-80, 91-115), then zero the grads. */
int dg_adam_step(dg_ctx* ctx, double lr);
double dg_lr_at(const dg_run_config* cfg, uint64_t step);

/* ---- compositing stages (batched overloads of render.hpp / train.hpp, fp64 inside) ----
 * Segment g owns samples [seg_off[g], seg_off[g+1]) (seg_off: n_seg + 1 entries from 0, in
 * march order); ray r owns segments [ray_off[r], ray_off[r+1]) in schedule order.  rgb is
 * 3 floats per sample / segment / ray.  All arrays on the host or all on the device (mem). */
/* local_render (render.cpp:46-78): per segment rgb, transmittance and depth_sum (optional);
 * with out_distortion (3 per segment: weight_sum, weight_moment, distortion_local) also
 * accumulate_distortion_stats (render.cpp:80-99) over the ray span [ray_t0, ray_t1]. */
int dg_local_render(dg_ctx* ctx, const double* t, const double* delta, const float* sigma,
                    const float* rgb, const uint64_t* seg_off, uint64_t n_seg, const double* ray_t0,
                    const double* ray_t1, float* out_rgb, float* out_transmittance,
                    float* out_depth_sum, double* out_distortion, int32_t mem);
/* local_render_backward (render.cpp:145-179): per-sample sigma / rgb gradients from the
 * segment upstream (d_rgb, d_transmittance) and an optional per-sample weight upstream. */
int dg_local_render_backward(dg_ctx* ctx, const double* t, const double* delta, const float* sigma,
                             const float* rgb, const uint64_t* seg_off, uint64_t n_seg,
                             const float* d_rgb, const float* d_transmittance,
                             const float* weight_upstream, float* sigma_grad, float* rgb_grad,
                             int32_t mem);
/* merge_forward (render.cpp:101-116); DG_EINVAL for a ray with no partials. */
int dg_merge_forward(dg_ctx* ctx, const float* seg_rgb, const float* seg_transmittance,
                     const float* seg_depth_sum, const uint64_t* ray_off, uint64_t n_rays,
                     float* rgb, float* transmittance, float* depth, int32_t mem);
/* merge_backward (render.cpp:118-143): per-segment dL/dC_i, dL/dT_i. */
int dg_merge_backward(dg_ctx* ctx, const float* seg_rgb, const float* seg_transmittance,
                      const uint64_t* ray_off, uint64_t n_rays, const float* d_rgb,
                      const float* d_transmittance, float* seg_d_rgb, float* seg_d_transmittance,
                      int32_t mem);
/* loss_rgb / loss_rgb_grad, loss_transmittance_single / loss_transmittance_grad
 * (train.cpp:8-36) per ray; any output may be NULL. */
int dg_ray_losses(dg_ctx* ctx, const float* rgb, const float* color_gt, const float* transmittance,
                  uint64_t n, double eps, double* loss_rgb, double* loss_transmittance, float* d_rgb,
                  float* d_transmittance, int32_t mem);
/* loss_distortion + loss_distortion_grad (train.cpp:38-75) per segment. */
int dg_distortion_loss(dg_ctx* ctx, const double* weights, const double* midpoints,
                       const double* interval_lengths, const uint64_t* seg_off, uint64_t n_seg,
                       double* loss, double* grads, int32_t mem);

/* ---- fp64 twins of the compositing stages (the C++ facade's reference-precision path,
 * include/distgrid/render.hpp, train.hpp): the same kernels with double inputs / outputs.
 * dg_local_render_f64 can also return the LocalRenderCache (alpha, prefix per sample). */
int dg_local_render_f64(dg_ctx* ctx, const double* t, const double* delta, const double* sigma,
                        const double* rgb, const uint64_t* seg_off, uint64_t n_seg, const double* ray_t0,
                        const double* ray_t1, double* out_rgb, double* out_transmittance,
                        double* out_depth_sum, double* out_distortion, double* out_cache, int32_t mem);
int dg_local_render_backward_f64(dg_ctx* ctx, const double* t, const double* delta, const double* sigma,
                                 const double* rgb, const uint64_t* seg_off, uint64_t n_seg,
                                 const double* d_rgb, const double* d_transmittance,
                                 const double* weight_upstream, double* sigma_grad, double* rgb_grad,
                                 int32_t mem);
int dg_merge_forward_f64(dg_ctx* ctx, const double* seg_rgb, const double* seg_transmittance,
                         const double* seg_depth_sum, const uint64_t* ray_off, uint64_t n_rays, double* rgb,
                         double* transmittance, double* depth, int32_t mem);
int dg_merge_backward_f64(dg_ctx* ctx, const double* seg_rgb, const double* seg_transmittance,
                          const uint64_t* ray_off, uint64_t n_rays, const double* d_rgb,
                          const double* d_transmittance, double* seg_d_rgb, double* seg_d_transmittance,
                          int32_t mem);
int dg_ray_losses_f64(dg_ctx* ctx, const double* rgb, const double* color_gt, const double* transmittance,
                      uint64_t n, double eps, double* loss_rgb, double* loss_transmittance, double* d_rgb,
                      double* d_transmittance, int32_t mem);
/* accumulate_distortion_stats (render.cpp:80-99) from a LocalRenderCache (alpha, prefix per
 * sample, as dg_local_render_f64 returns it): out[3 * g] = weight_sum, weight_moment,
 * distortion_local of segment g over its ray span; segments with an empty span are left as
 * they are (out is read and written). */
int dg_distortion_stats_f64(dg_ctx* ctx, const double* t, const double* delta, const double* cache,
                            const uint64_t* seg_off, uint64_t n_seg, const double* ray_t0, const double* ray_t1,
                            double* out, int32_t mem);
/* ray_aabb_intersect (geometry.cpp:7-28) of n rays against one box: hit, t_near, t_far. */
int dg_ray_aabb(dg_ctx* ctx, const double* origin, const double* dir, uint64_t n, const double box_lo[3],
                const double box_hi[3], uint8_t* hit, double* t_near, double* t_far, int32_t mem);
/* march_segment (render.cpp:10-37) over caller-given occupied intervals: segment g spans
 * [t_enter[g], t_exit[g]) with intervals [interval_off[g], interval_off[g+1]) of `intervals`
 * (t_near, t_far pairs).  Two phases as dg_cascade_march: counts only (t == NULL), then the
 * samples at offsets[g].  jitter: offset = step * counter_uniform(jitter_seed, ray_id[g],
 * jitter_step), else step / 2.  DG_EINVAL unless step > 0. */
int dg_march_segment(dg_ctx* ctx, const double* t_enter, const double* t_exit, const uint64_t* interval_off,
                     const double* intervals, const uint64_t* ray_id, uint64_t n, double step, int32_t jitter,
                     uint64_t jitter_seed, uint64_t jitter_step, uint32_t* counts, const uint64_t* offsets,
                     double* t, double* delta, int32_t mem);
/* occupancy_skip (grid.cpp:235-304): the occupied runs of [t0, t1] along each ray through a
 * caller's bitfield (shape[0] x shape[1] x shape[2] cells, ix fastest, over [box_lo, box_hi]).
 * Two phases as dg_march_segment: counts, then (t_near, t_far) pairs at offsets. */
int dg_occupancy_skip(dg_ctx* ctx, const uint8_t* bits, const uint32_t shape[3], const double box_lo[3],
                      const double box_hi[3], const double* origin, const double* dir, const double* t0,
                      const double* t1, uint64_t n, uint32_t* counts, const uint64_t* offsets, double* intervals,
                      int32_t mem);
/* AdamState::step (train.cpp:91-115) on one caller-owned fp64 array: m, v updated in place,
 * t = the step count after this step (bias corrections 1 - beta^t). */
int dg_adam_update_f64(dg_ctx* ctx, double* params, const double* grads, double* m, double* v, uint64_t n,
                       uint64_t t, double lr, double beta1, double beta2, double eps, int32_t mem);

/* ---- introspection of the last dg_train_step / dg_render on this rank ---- */
typedef struct dg_item_view {
  uint64_t n_items;       /* (ray, partition) segments of this partition */
  uint64_t n_fine;        /* fine samples */
  uint64_t n_coarse;      /* coarse samples */
} dg_item_view;
int dg_last_items(dg_ctx* ctx, uint32_t partition, dg_item_view* view);
/* per item: global ray id, my schedule order, t_enter/t_exit, sample count */
int dg_last_item_data(dg_ctx* ctx, uint32_t partition, uint64_t* ray_id, uint8_t* order,
                      double* t_enter, double* t_exit, uint32_t* n_samples);
/* per item samples in t order (concatenated in item order): t, delta, cascade */
int dg_last_samples(dg_ctx* ctx, uint32_t partition, double* t, double* delta, uint8_t* cascade);
/* per sample of the last training step, in dg_last_samples order (each output optional):
 * normalised field position [n][3] (worker.cpp:46), encoded features [n][2L], field output
 * [n][4] (sigma, rgb), compositing upstream [n][4] (dsigma, drgb), features gradient [n][2L],
 * the forward's ReLU / clip mask words [n][7] (tcgen05 path) */
int dg_last_sample_data(dg_ctx* ctx, uint32_t partition, double* pos, float* features,
                        float* field_out, float* upstream, float* d_features, uint32_t* masks);
/* per item own partial (rgb, T) as computed by the composite kernel */
int dg_last_partials(dg_ctx* ctx, uint32_t partition, float* rgb, float* transmittance);
/* launches of this library's kernels since the context was created */
int dg_kernel_launches(const dg_ctx* ctx, uint64_t* n);
/* per-stage device time of the last step (ms), measured with events on the ctx stream */
typedef struct dg_stage_times {
  float segment, march, encode_fwd, mlp_fwd, composite, exchange, merge_bwd, mlp_bwd, encode_bwd,
      adam, total;
  /* exchange 1 alone (dispatch records to the owners; inside `segment`), and the bytes this
   * rank sent to other ranks in exchange 1 / exchange 2 (MB) */
  float dispatch_exchange, dispatch_mb, partial_mb;
  float reserved[2];
} dg_stage_times;
int dg_enable_stage_timing(dg_ctx* ctx, int enable);
int dg_last_stage_times(dg_ctx* ctx, dg_stage_times* t);
/* Waits (host) for every call's work, including the last training step's Adam update, which
 * runs on a side stream so that the next step's segmentation / march overlaps it.  Every API
 * call that reads or writes parameters, gradients or moments orders itself after that update;
 * dg_fence does only that ordering (no host wait): work the caller queues afterwards on the
 * context's stream (dg_set_stream) sees the updated parameters. */
int dg_synchronize(dg_ctx* ctx);
int dg_fence(dg_ctx* ctx);
/* Diagnostics: runs the tcgen05 operand-layout self-test on the current device.
 * Host fp32 inputs A[128x64], B[64x64], X[128x32]; outputs Y0 = A B^T, Y1 = A B (128x64) and
 * Y2 = A^T X (64x32), each a split-bf16 (3-term) tcgen05.mma product accumulated in TMEM. */
int dg_selftest_tcgen05(const float* A, const float* B, const float* X, float* Y0, float* Y1,
                        float* Y2);
/* the context's CUDA stream (cudaStream_t) so callers can record events on it */
int dg_get_stream(dg_ctx* ctx, void** stream);
/* run every later call of this context on the caller's cudaStream_t (NULL: back to the
 * context's own stream); waits for the work already queued on the current stream */
int dg_set_stream(dg_ctx* ctx, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DISTGRID_B200_H */
