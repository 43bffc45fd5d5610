// kernels.h — launch wrappers for the sm_100a kernels (one translation unit each).
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "dg_common.cuh"

namespace dg {

// Per-item state after setup (structure of arrays, capacity NI).
constexpr int kMaxRuns = 64;
constexpr uint8_t kRunsOverflow = 0xff;

struct ItemArrays {
  RayRec* rec;        // dispatch record (origin/dir rounded in place when wire_f32)
  double* te;         // my segment t_enter / t_exit
  double* tx;
  double* t0;         // schedule.front().t_enter / schedule.back().t_exit
  double* t1;
  uint8_t* nseg;
  uint8_t* order;     // my index in the schedule
  uint8_t* part;      // local partition index
  uint8_t* sched;     // NI x 16 global partition ids
  uint32_t* cnt;      // [2][NI]: fine, coarse sample counts (scanned in place -> offsets)
  uint32_t* off;      // [2][NI] exclusive offsets (fine region, coarse region)
  uint32_t* ncb;      // coarse samples before the fine box
  double2* runs;      // [NI][kMaxRuns] occupied runs of the cascade march (lo, hi), from item setup
  uint8_t* run_casc;  // [NI][kMaxRuns] cascade of each run
  uint8_t* nrun;      // runs recorded per item; kRunsOverflow: more than kMaxRuns (walk again)
  uint32_t* contains; // [P][NI] 1 when partition q is in the schedule and q != mine
  uint32_t* cscan;    // exclusive scan of contains
  float4* partial;    // rgb, optical depth tau (T = exp(-tau)) of my segment
  float* depth;       // depth_sum of my segment
  float4* xdist;      // distortion_cross_correction only (else null): weight_sum,
                      // weight_moment, distortion_local of my segment (worker.cpp:289-299)
};

struct SampleArrays {
  double* t;
  double* delta;
  uint32_t* item;
  double* p;       // normalised field position (grid.cpp:109 / worker.cpp:215), SoA [3][pn]
  uint64_t pn;     // samples (stride of p)
  float* X;        // n x 32 encoded features
  float4* out;     // sigma, r, g, b
  float4* grad;    // dsigma, dr, dg, db
  float* dX;       // n x 32
  const uint32_t* inv;  // sample order (kernels_order.cu): march sample -> sorted slot; null: none
  float4* grad_ord;     // with inv: the merge backward's upstream, stored at the sorted slot
};

struct LossAccum {
  double rgb[kMaxPart];
  double trans[kMaxPart];
  double dist[kMaxPart];
  uint32_t error;     // bit 0: unknown image id, bit 1: partial protocol mismatch
  uint32_t pad;
};

// Peer-memory destinations of a pack kernel (PeerComm): base[r] is rank r's receive buffer
// mapped into this process (CUDA IPC; the own rank's is local), off[p] a per-partition record
// offset.  base == nullptr: pack into the local send buffer instead.
struct PeerDst {
  void* const* base;
  const uint64_t* off;
  uint32_t world;
};

// ---- ray-side kernels (kernels_ray.cu) ----
void launch_segment_home(const Geo* geo, const double* o, const double* d, uint64_t n,
                         const uint8_t* slot_of_part, uint8_t* nseg, uint8_t* sched,
                         uint32_t* flags, unsigned long long* dropped, cudaStream_t s);
void launch_pack_dispatch(uint64_t n, uint32_t P, const uint8_t* nseg, const uint8_t* sched,
                          const uint8_t* slot_of_part, const uint32_t* pos, const double* o,
                          const double* d, const float* gt, const uint32_t* img,
                          uint64_t first_ray_id, RayRec* out, PeerDst peer, cudaStream_t s);
void launch_item_setup(const Geo* geo, const PartDesc* parts, const uint8_t* occ,
                       const uint32_t* part_item_off, uint32_t n_local, uint32_t n_items,
                       ItemArrays it, uint32_t P, double step, uint64_t seed, uint64_t batch_id,
                       int jitter, int wire_f32, uint32_t n_images, uint32_t* error,
                       cudaStream_t s);
void launch_march_fill(const PartDesc* parts, const uint8_t* occ, uint32_t n_items,
                       ItemArrays it, SampleArrays sm, uint32_t fine_total, double step,
                       uint64_t seed, uint64_t batch_id, int jitter, cudaStream_t s);
void launch_composite(uint32_t n_items, ItemArrays it, SampleArrays sm, uint32_t fine_total,
                      int with_depth, cudaStream_t s);
void launch_pack_partials(uint32_t n_items, ItemArrays it, const uint32_t* part_item_off,
                          const uint8_t* local_of_global, const uint64_t* stream_off,
                          uint32_t P, PartialRec* send, float4* send_x, PeerDst peer, PeerDst peer_x,
                          cudaStream_t s);
void launch_merge_backward(uint32_t n_items, ItemArrays it, const uint32_t* part_item_off,
                           const PartDesc* parts, const uint64_t* stream_off, uint32_t P,
                           const PartialRec* recv, const float4* recv_x, SampleArrays sm,
                           uint32_t fine_total, double lambda_t, double lambda_d, double t_clamp,
                           int wire_f32, LossAccum* loss, cudaStream_t s);
void launch_pair_counts(uint32_t n_items, uint32_t n_local, uint32_t P, const uint32_t* part_item_off,
                        const uint32_t* contains, const uint32_t* cscan, uint32_t* out,
                        cudaStream_t s);
// eval: home merge in schedule order from item partials (world == 1) or reply records
void launch_home_merge(uint64_t n, uint32_t P, const uint8_t* nseg, const uint8_t* sched,
                       const uint8_t* slot_of_part, const uint32_t* pos, const float4* partial,
                       const float* depth, const PartialRec* reply, int wire_f32, float* rgb, float* trans,
                       float* depth_out, int early_term, double term_thr, float* attribution,
                       cudaStream_t s);
void launch_camera_rays(const double* pose, uint32_t width, uint64_t n, double* o, double* d,
                        cudaStream_t s);

// stage-entry helpers
void launch_segment_full(const Geo* geo, const double* o, const double* d, uint64_t n, uint8_t* nseg,
                         uint8_t* sched, double* te, double* tx, cudaStream_t s);
void launch_u8_to_u16(const uint8_t* in, uint16_t* out, uint64_t n, cudaStream_t s);
void launch_march_points(const PartDesc* part, const uint8_t* occ, const double* o, const double* d,
                         const double* t0, const double* t1, const uint64_t* ray_id, uint64_t n,
                         double step, uint64_t seed, uint64_t batch_id, int jitter, uint32_t* counts,
                         const uint64_t* offsets, double* t, double* delta, uint8_t* cascade,
                         cudaStream_t s);
void launch_items_to_records(uint32_t n, const float4* partial, const float* depth, const RayRec* rec,
                             PartialRec* out, cudaStream_t s);

// ---- field kernels ----
// One encode pass: levels [l0, l1) restricted to row slice k of S of each level's table, so
// the tables a pass touches stay L2-resident (random rows of a 128 MB table miss L2; a
// 64 MB slice does not).  Slice bounds are even, so a float4 row pair never straddles two.
// One encode pass: levels [l0, l1) of field f, row slice k of S (a slice's table rows fit the
// pass's L2 budget); the pass covers only field f's samples.
struct EncPass {
  uint8_t l0, l1, k, S;
  uint8_t f, paired, pad1, pad2;  // paired: a level of the pass has a paired copy (kernels_pairs.cu)
  // S > 1 (a single level l0): table rows [lo, hi) of slice k, per field (f == kAllFields:
  // fields 0 and 1 of the single local partition; otherwise slot 0 is field f)
  uint32_t lo[2], hi[2];
};
constexpr int kMaxEncPass = 256;  // per launch; longer pass lists are launched in chunks
constexpr uint8_t kAllFields = 0xff;  // EncPass.f: every local field's samples in one pass

// Paired copy of one one-to-one level table (kernels_pairs.cu): pairs[pair0 + i] = rows i and
// i + 1 of the table at params[table], as one float4 (row `rows` reads as 0).
struct PairSeg {
  uint64_t pair0;   // float4 index in the pair buffers
  uint64_t table;   // float offset of the table in the parameter / gradient buffers
  uint64_t rows;
};
void launch_pairs_expand(const PairSeg* segs, uint32_t nseg, uint64_t total, const float* params, float4* pairs,
                         cudaStream_t s);
void launch_pairs_fold(const PairSeg* segs, uint32_t nseg, uint64_t total, float4* pgrads, float* grads,
                       cudaStream_t s);

struct FieldLaunch {
  const FieldDesc* fields;     // [2][n_local] (cascade-major)
  const PartDesc* parts;
  const ItemArrays* it_dummy;  // unused
  const RayRec* rec;           // items
  const uint8_t* item_part;
  const double* s_t;
  const uint32_t* s_item;
  uint32_t fine_total;
  uint32_t n_total;
  uint32_t n_local;
  uint32_t levels;
  uint32_t agg_levels;     // levels whose backward scatter is warp-aggregated
  uint32_t cta_mul;        // backward: CTA x visits sample chunk (x * cta_mul) % gridDim.x (0: x)
  const float4* pairs;     // paired one-to-one level tables (LevelDesc::poff), forward
  float4* pgrads;          // their gradients, backward (folded into grads by launch_pairs_fold)
  const float* params;
  float* grads;
  uint32_t n_pass;         // passes of this launch (grid.y)
  EncPass pass[kMaxEncPass];
  const double* s_p;       // per-sample normalised position, SoA [3][n_total] (k_march_fill)
  uint32_t n_fields;       // 2 n_local; samples are field-major
  uint32_t field_off[2 * kMaxPart + 1];
};
// Forward: one launch per slice index (slice k > 0 adds into X written by slice 0); returns
// the number of launches.  Backward: one launch over every pass (reds commute).
size_t order_sort_tmp_bytes(uint32_t n);
int launch_order_field(const double* p, const uint32_t* item, uint64_t stride, uint64_t off, uint32_t n,
                       uint32_t C, uint32_t bits, uint32_t* perm, uint32_t* inv, double* p_out,
                       uint32_t* item_out, uint32_t* scratch, void* tmp, size_t tmp_bytes, cudaStream_t s);
int launch_encode_fwd(const FieldLaunch& f, const std::vector<EncPass>& passes, float* X, cudaStream_t s);
int launch_encode_bwd(const FieldLaunch& f, const std::vector<EncPass>& passes, const float* dX, cudaStream_t s);
// stand-alone points variant (stage entry points): all points belong to one field
void launch_encode_points(const FieldDesc* field, const float* params, const double* pts,
                          uint64_t n, uint32_t levels, float* X, uint32_t* rows, cudaStream_t s);
void launch_encode_points_bwd(const FieldDesc* field, float* grads, const double* pts,
                              const float* dX, uint64_t n, uint32_t levels, cudaStream_t s);

// MLP: tiles never straddle fields.  field_off: n_fields+1 sample offsets.
struct MlpLaunch {
  const FieldDesc* fields;
  uint32_t n_fields;
  const uint32_t* field_off;   // device, n_fields + 1
  const uint32_t* tile_off;    // device, n_fields + 1 (prefix of tiles)
  uint32_t n_tiles;
  uint32_t relu_tiles;         // bwd (tc): the leading tiles of ReLU (fine) fields, which take the
                               // paired kernel k_mlp_bwd_tc_relu; 0: every tile the serial one
  uint32_t issue_warp;         // k_mlp_bwd_tc_relu: the warp whose elected lane issues the MMAs
  uint32_t issue_warp_fwd;     // k_mlp_fwd_tc: the same (0-7)
  const float* X;              // level-major [levels][x_stride] float2
  uint64_t x_stride;           // samples per level row of X / dX
  uint32_t levels;
  const float* dirs_f;         // optional per-sample dirs (stage entry) else from items
  const RayRec* rec;
  const uint32_t* s_item;      // item of each sample (in sample order when perm is set)
  const uint32_t* perm;        // sample order: tile row -> march sample (index of out); null: identity
  const float* app_table;      // [n_images][app_dim]
  const float* app_override;   // eval: one vector for all samples (or per-sample when app_per_sample)
  int app_per_sample;
  const float* params;
  float* grads;
  float4* out;                 // fwd: sigma, rgb
  float4* out_tile;            // train: the forward's (sigma, rgb) by tile row as well (written by
                               // the forward when perm is set, else = out), read by the backward
  const float4* grad_in;       // bwd: dsigma, drgb
  float* dX;                   // bwd, level-major like X
  uint32_t* masks;             // tc path: [7][x_stride] ReLU / clip masks, written by the forward,
                               // read by the backward (kernels_mlp_tc.cu); null: not stored
  unsigned long long* trace;   // DG_TRACE_MLP builds only (tools/trace_mlp.cu): phase clocks
};
void launch_mlp_fwd(const MlpLaunch& m, cudaStream_t s);
void launch_mlp_bwd(const MlpLaunch& m, int num_sms, cudaStream_t s);
// tcgen05 (split-bf16) variants (kernels_mlp_tc.cu); tiles of 128 samples
void launch_mlp_fwd_tc(const MlpLaunch& m, int num_sms, cudaStream_t s);
void launch_mlp_bwd_tc(const MlpLaunch& m, int num_sms, cudaStream_t s);  // tile_off at 128
// evaluation forward (no masks, no backward): split-bf16
void launch_mlp_eval_tc(const MlpLaunch& m, int num_sms, cudaStream_t s);

// ---- compositing stage entry points (kernels_render_api.cu), fp64 like the reference ----
// fp64 arithmetic in the reference's order; R = float (the C ABI's fp32 stage I/O) or double
// (the *_f64 entry points behind the C++ facade, include/distgrid/*.hpp)
template <class R>
void launch_local_render(const double* t, const double* delta, const R* sigma, const R* rgb,
                         const uint64_t* seg_off, uint64_t n_seg, const double* ray_t0,
                         const double* ray_t1, R* out_rgb, R* out_T, R* out_depth,
                         double* out_dist, double* cache, cudaStream_t s);
template <class R>
void launch_local_render_bwd(const double* delta, const R* rgb, const uint64_t* seg_off, uint64_t n_seg,
                             const double* cache, const R* d_rgb, const R* d_T, const R* w_up,
                             R* sigma_grad, R* rgb_grad, cudaStream_t s);
template <class R>
void launch_merge_fwd(const R* srgb, const R* sT, const R* sdepth, const uint64_t* ray_off,
                      uint64_t n_rays, R* rgb, R* T, R* depth, cudaStream_t s);
template <class R>
void launch_merge_bwd(const R* srgb, const R* sT, const uint64_t* ray_off, uint64_t n_rays,
                      const R* d_rgb, const R* d_T, R* sd_rgb, R* sd_T, cudaStream_t s);
template <class R>
void launch_ray_losses(const R* rgb, const R* gt, const R* T, uint64_t n, double eps,
                       double* l_rgb, double* l_T, R* d_rgb, R* d_T, cudaStream_t s);
void launch_distortion_stats(const double* t, const double* delta, const double* cache, const uint64_t* seg_off,
                             uint64_t n_seg, const double* ray_t0, const double* ray_t1, double* out,
                             cudaStream_t s);
void launch_distortion(const double* w, const double* s_, const double* ds, const uint64_t* seg_off,
                       uint64_t n_seg, double* loss, double* grad, cudaStream_t s);

// ---- per-function stage entry points of the facade (kernels_stage_api.cu) ----
void launch_ray_aabb(const double* o, const double* d, uint64_t n, const double lo[3], const double hi[3],
                     uint8_t* hit, double* tn, double* tf, cudaStream_t s);
void launch_march_segment(const double* te, const double* tx, const uint64_t* iv_off, const double* iv,
                          const uint64_t* ray_id, uint64_t n, double step, int jitter, uint64_t seed,
                          uint64_t batch, uint32_t* counts, const uint64_t* out_off, double* t, double* delta,
                          cudaStream_t s);
void launch_field_density(const FieldDesc* field, const float* params, const float* X, uint64_t n, float* sigma,
                          float* feat, cudaStream_t s);
void launch_field_color(const FieldDesc* field, const float* params, const float* feat, const float* dirs,
                        const float* app, uint64_t n, float* rgb, cudaStream_t s);
void launch_occupancy_skip(const uint8_t* bits, const uint32_t shape[3], const double lo[3], const double hi[3],
                           const double* o, const double* d, const double* t0, const double* t1, uint64_t n,
                           uint32_t* counts, const uint64_t* out_off, double* iv, cudaStream_t s);
void launch_adam_f64(double* p, const double* g, double* m, double* v, uint64_t n, double lr, double b1,
                     double b2, double eps, double bias1, double bias2, cudaStream_t s);

// ---- optimizer / init (kernels_adam.cu) ----
void launch_adam(float* p, float* g, float* m, float* v, uint64_t n, float lr, float b1, float b2,
                 float eps, float inv_bias1, float inv_bias2, cudaStream_t s,
                 const uint32_t* abort_flag = nullptr, uint32_t abort_mask = 0, bool spread = false);
void launch_fill_uniform(float* p, uint64_t n, float lo, float hi, uint64_t seed, cudaStream_t s);

// ---- occupancy update (kernels_occ.cu) ----
int launch_occ_query(const FieldDesc* field, const float* params, const double* pw, uint64_t n,
                     float* sigma, cudaStream_t s);
void launch_occ_apply(float* density, const uint32_t* cells, const float* sigma, uint64_t n,
                      float decay, cudaStream_t s);
void launch_occ_bits(const float* density, uint8_t* bits, const uint32_t shape[3], float threshold,
                     cudaStream_t s);

// ---- tcgen05 self-test (kernels_tc.cu) ----
int tc_selftest(const float* A, const float* B, const float* X, float* Y0, float* Y1, float* Y2,
                cudaStream_t s);

}  // namespace dg
