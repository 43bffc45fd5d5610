#include <numeric>
// runtime.cu — the C ABI (include/distgrid_b200.h): context, state, and the composed
// per-step pipeline that replaces DistributedRun::training_step / evaluate_rays
// (worker.cpp:730-834) and Worker::handle_training_batch (worker.cpp:251-401).
//
// Per step, on each rank (one GPU), for the partitions it owns:
//   K1  segment home rays, count per destination partition, scan, pack dispatch records
//   X1  exchange 1 (rays -> owners): all-to-all-v, then a block transpose into items
//   K2  item setup (owner recomputes the schedule bit-exactly) + sample count, scan, fill
//   K3  hash-grid encode (fwd)            K4  fused MLP (fwd)
//   K5a composite -> own partial          X2  exchange 2 (partials -> every other owner)
//   K5b merge + losses + merge/composite backward per item
//   K4b MLP backward (weight grads, d encoding)   K3b hash-grid backward (atomics)
//   K6  dense Adam + grad zeroing (every rank, every step, even with no rays)
// Single-rank runs skip the all-to-all copies: the exchange buffers alias.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <future>
#include <thread>
#include <tuple>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "comm.h"
#include "exchange_plan.h"
#include "geometry.cuh"
#include "kernels.h"

using namespace dg;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return set_err(DG_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                     __FILE__, __LINE__);                                                 \
  } while (0)

#define TRY(call)                 \
  do {                            \
    int rc_ = (call);             \
    if (rc_ != DG_OK) return rc_; \
  } while (0)

}  // namespace

namespace dg {
// Error reporting for the other host translation units (ray_cache.cu): sets dg_last_error.
int set_error(int code, const char* msg) { return set_err(code, "%s", msg); }
}  // namespace dg

namespace {

// ---------------------------------------------------------------- host layout math
uint32_t level_resolution(uint32_t levels, uint32_t base, uint32_t maxr, uint32_t level) {
  if (levels == 1) return base;  // grid.cpp:56-63
  const double growth = std::exp((std::log(double(maxr)) - std::log(double(base))) / double(levels - 1));
  return uint32_t(std::llround(double(base) * std::pow(growth, double(level))));
}

void grid_shape(const double aspect[3], uint32_t nres, uint32_t out[3]) {  // grid.cpp:65-73
  const double n = double(nres);
  const double s = smax(aspect[0], smax(aspect[1], aspect[2]));
  for (int a = 0; a < 3; ++a) out[a] = uint32_t(std::ceil(aspect[a] / s * n));
}

// A device buffer that only grows.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  int ensure(size_t want) {
    if (want <= bytes) return DG_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t n = std::max<size_t>(want + want / 4, 256);
    if (cudaMalloc(&p, n) != cudaSuccess) {
      cudaGetLastError();
      return set_err(DG_ENOMEM, "cudaMalloc(%zu) failed", n);
    }
    bytes = n;
    return DG_OK;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace

struct dg_ctx {
  dg_run_config cfg{};
  int device = 0, rank = 0, world = 1;
  uint32_t P = 1;
  std::vector<uint32_t> local;          // global ids of local partitions (ascending)
  std::vector<int> part_rank;           // rank of each global partition
  std::vector<uint8_t> slot_of_part;    // rank-major slot of each partition
  std::vector<uint32_t> part_of_slot;
  std::vector<uint8_t> local_of_global; // 0xff when remote
  Geo geo{};
  std::vector<PartDesc> parts;
  std::vector<FieldDesc> fields;        // [2][n_local] cascade-major
  std::vector<uint64_t> part_param_off; // per local partition (floats, device layout)
  std::vector<uint64_t> part_param_cnt; // flat (reference-order) count
  std::vector<uint64_t> field_dev_off;  // [2][n_local] device offset of each field
  std::vector<uint64_t> field_size;     // [2][n_local] flat (reference-order) floats
  // flat <-> device mapping of one field: every level table starts 16-byte aligned on the
  // device (paired-row float4 gathers / reds), so the device layout has small gaps
  struct Seg {
    uint64_t dev, flat, count;  // relative to the field's device base / flat start
  };
  std::vector<std::vector<Seg>> field_segs;  // [2][n_local]
  // paired copies of the one-to-one level tables (kernels_pairs.cu)
  bool enc_paired = true;          // DG_ENC_PAIRED=0 disables
  uint64_t pair_rows = 0;
  std::vector<PairSeg> pair_segs;  // one per (field, one-to-one level)
  DBuf pairs, pgrads, pair_segs_d;
  std::vector<std::vector<dg_array_desc>> layouts;
  uint64_t enc_budget_fwd = 192ull << 20;  // encode pass budgets (DG_ENC_FWD_MB / DG_ENC_BWD_MB)
  uint64_t enc_budget_bwd = 96ull << 20;
  uint64_t enc_group_fwd = 0, enc_group_bwd = 0;  // level-grouping budgets (0: = slice budget)
  uint64_t enc_hgroup_fwd = 64ull << 20;   // forward grouping budget of passes with a hashed level
                                           // (DG_ENC_FWD_HGROUP_MB; 0: the grouping budget)
  uint64_t enc_hgroup_bwd = 32ull << 20;   // the backward's (DG_ENC_BWD_HGROUP_MB)
  bool enc_pcache = true;                  // per-sample position cache (DG_ENC_PCACHE)
  int sample_order = 1;                    // spatial sample order: 1 when a field's tables > 64 MB,
                                           // 0 never, 2 always (DG_SAMPLE_ORDER)
  uint32_t order_bits = 8;                 // Morton cells per axis = 2^order_bits (DG_ORDER_BITS)
  uint32_t order_chunk = 8;                // samples per sorted chunk (DG_ORDER_CHUNK)
  uint32_t bwd_cta_mul = 7919;             // encode backward CTA visiting stride (DG_ENC_BWD_STRIDE)
  bool mlp_bwd_paired = true;              // ReLU fields take k_mlp_bwd_tc_relu (DG_MLP_BWD_SERIAL=1: off)
  uint32_t mlp_issue_warp = 8;             // k_mlp_bwd_tc_relu's MMA-issuing warp (DG_MLP_ISSUE_WARP)
  uint32_t mlp_issue_warp_fwd = 0;         // k_mlp_fwd_tc's (DG_MLP_FWD_ISSUE_WARP)
  bool ordered = false;                    // the last front half ordered its samples
  DBuf s_perm, s_inv, s_p_alt, s_item_ord, s_grad_ord, s_out_ord, ord_scratch, ord_tmp;
  double enc_agg_samples_per_cell = 1.5;   // warp-aggregate levels with >= this many samples/cell (DG_ENC_AGG)
  uint64_t n_params = 0;
  uint64_t occ_bytes = 0;                 // bricked bitfields (all local partitions, both cascades)
  uint64_t occ_den_n = 0;                 // linear densities (floats)
  std::vector<double> occ_thr;            // [n_local][2] current thresholds
  std::vector<std::mt19937_64> occ_rng;   // Worker::occ_rng_ per local partition (worker.cpp:186)
  uint64_t occ_updates = 0;
  // warm-up updates draw 3 uniforms per cell in a fixed order, independent of the state, so
  // the next update's jitter points are generated on a host thread while the GPU trains
  double* occ_host = nullptr;             // pinned, all (partition, cascade) warm-up points
  uint64_t occ_host_n = 0;                // doubles
  std::future<void> occ_prefetch;
  bool occ_prefetched = false;
  // occ_rng before the pending prefetch drew from it: restored when the step is moved
  // (dg_set_step / checkpoint load) so the stream holds exactly the draws of the updates that
  // actually ran, as the reference's occ_rng_ does (load_state leaves it alone, worker.cpp:615-626)
  std::vector<std::mt19937_64> occ_rng_before;
  // ... and go up to the device on a copy stream as soon as they are drawn, so the 24 B/cell
  // transfer overlaps the training steps before the update instead of stalling it
  cudaStream_t stream_copy = nullptr;
  // The training step's Adam runs on its own stream, so the next step's front half (which
  // touches no parameter) overlaps it; every later use of the parameters / gradients / moments
  // (the next step's encode, any API call) first orders the context stream after ev_adam.
  cudaStream_t stream_adam = nullptr;
  cudaEvent_t ev_grads = nullptr, ev_adam = nullptr;
  bool adam_pending = false;
  bool adam_spread = true;  // DG_ADAM_SPREAD=0: the resident grid-stride Adam grid
  DBuf adam_flag;  // the step's error word as k_adam reads it
  // Pinned staging arena for the step's small host <-> device transfers.  A pageable source
  // makes cudaMemcpyAsync wait for the stream to drain and a pageable destination makes it
  // synchronous, so every plan upload / count readback would otherwise cost a full pipeline
  // bubble.  Bump-allocated per API call (pin_reset) after the stream is idle.
  uint8_t* pin = nullptr;
  size_t pin_cap = 0, pin_used = 0;
  cudaEvent_t ev_occ_up = nullptr, ev_occ_used = nullptr;
  bool occ_uploaded = false;
  double step = 0.0;
  uint64_t adam_t = 0;
  uint64_t worker_step = 0;
  uint32_t n_images = 0, app_rows = 0;
  cudaStream_t stream = nullptr;      // the stream every call runs on (dg_set_stream)
  cudaStream_t own_stream = nullptr;  // the context's own stream
  int num_sms = 148;
  int mlp_impl = 1;  // 1: tcgen05 split-bf16 forward (default), 0: FFMA fp32 (DG_MLP=ffma)
  std::unique_ptr<Comm> comm;
  uint64_t comm_timeout_ms = 120000;  // Worker::Setup::recv_timeout (worker.hpp:82)
  uint64_t launches = 0;
  bool timing = false;
  cudaEvent_t ev[12] = {};
  dg_stage_times times{};

  // in-memory snapshot of the training state (dg_state_snapshot)
  struct Snapshot {
    DBuf params, m, v, occ, occ_den;
    std::vector<double> occ_thr;
    std::vector<std::mt19937_64> occ_rng;
    uint64_t adam_t = 0, worker_step = 0;
    bool valid = false;
  } snap;
  // persistent device state
  DBuf out_attr, cam_o, cam_d, cam_pose, it_xdist, send_x, recv_x, it_runs, it_runc, it_nrun;
  bool cross_active = false;  // training step with distortion_cross_correction
  RayRec* items_rec = nullptr;  // this step's item records: rec, or the peer backend's item buffer
  DBuf peer_off;                // per-partition record offsets of the peer-memory dispatch
  DBuf d_geo, d_parts, d_fields, params, grads, adam_m, adam_v, occ, occ_den, app, slot_of_part_d,
      local_of_global_d, global_of_local_d;
  // per-step scratch
  DBuf h_o, h_d, h_gt, h_img, h_nseg, h_sched, h_flags, h_pos, cub_tmp, small, dropped, loss,
      error, rec, it_te, it_tx, it_t0, it_t1, it_nseg, it_order, it_part, it_sched, it_cnt,
      it_off, it_ncb, it_contains, it_cscan, it_partial, it_depth, part_item_off_d, s_t, s_delta, s_p,
      s_item, s_X, s_out, s_grad, s_dX, s_mask, field_off_d, tile_off_f, tile_off_b, stream_send_d,
      stream_recv_d, send_buf, recv_buf, x_send, x_recv, out_rgb, out_T, out_depth, eval_app,
      perm_tab, occ_pts, occ_cells, occ_sigma, occ_pts_warm;
  // last step (introspection)
  std::vector<uint32_t> part_item_off;   // n_local + 1
  std::vector<uint32_t> field_off;       // 2 n_local + 1
  uint32_t n_items = 0, n_fine = 0, n_coarse = 0;
  bool have_last = false;
  uint64_t h2d = 0, d2h = 0;  // bytes moved by the current call
};

namespace {

int ctx_setup(dg_ctx* c) {
  const dg_run_config& cfg = c->cfg;
  if (cfg.kx < 1 || cfg.ky < 1) return set_err(DG_EINVAL, "split_regions: kx, ky must be >= 1");
  if (cfg.kx * cfg.ky > DG_MAX_PARTITIONS) return set_err(DG_EINVAL, "too many partitions (max 64)");
  if (cfg.kx + cfg.ky - 1 > DG_MAX_SEGMENTS) return set_err(DG_EINVAL, "kx + ky - 1 must be <= 16");
  if (cfg.grid_features != 2) return set_err(DG_EINVAL, "device path requires grid_features == 2");
  if (cfg.grid_levels < 1 || cfg.grid_levels > DG_MAX_LEVELS)
    return set_err(DG_EINVAL, "grid_levels must be in [1, 16]");
  if (cfg.appearance_dim > 17) return set_err(DG_EINVAL, "appearance_dim must be <= 17");
  if (cfg.fine_table_log2 > 30 || cfg.coarse_table_log2 > 30)
    return set_err(DG_EINVAL, "table_log2 must be <= 30");
  if (cfg.base_resolution > cfg.max_resolution)
    return set_err(DG_EINVAL, "grid: base_resolution must be <= max_resolution");
  if (!(cfg.march_step_divisor > 0.0)) return set_err(DG_EINVAL, "march_step_divisor must be positive");
  if (!(cfg.transmittance_clamp > 0.0 && cfg.transmittance_clamp < 1.0))
    return set_err(DG_EINVAL, "config: transmittance clamp must be in (0,1)");
  c->P = cfg.kx * cfg.ky;
  // split_regions (partition.cpp:206-252): planes computed once, shared bitwise
  Geo& g = c->geo;
  std::memset(&g, 0, sizeof g);
  for (int a = 0; a < 3; ++a) {
    g.outer_lo[a] = cfg.outer_lo[a];
    g.outer_hi[a] = cfg.outer_hi[a];
  }
  for (uint32_t i = 0; i <= cfg.kx; ++i)
    g.xp[i] = i == 0 ? cfg.inner_lo[0]
              : i == cfg.kx ? cfg.inner_hi[0]
                            : cfg.inner_lo[0] + (cfg.inner_hi[0] - cfg.inner_lo[0]) * double(i) / double(cfg.kx);
  for (uint32_t i = 0; i <= cfg.ky; ++i)
    g.yp[i] = i == 0 ? cfg.inner_lo[1]
              : i == cfg.ky ? cfg.inner_hi[1]
                            : cfg.inner_lo[1] + (cfg.inner_hi[1] - cfg.inner_lo[1]) * double(i) / double(cfg.ky);
  g.kx = cfg.kx;
  g.ky = cfg.ky;
  g.P = c->P;
  for (int a = 0; a < 3; ++a)
    if (!(cfg.inner_lo[a] <= cfg.inner_hi[a]) || !(cfg.outer_lo[a] <= cfg.inner_lo[a]) ||
        !(cfg.inner_hi[a] <= cfg.outer_hi[a]))
      return set_err(DG_EINVAL, "manifest: fine not inside coarse");
  // march step (worker.cpp:923-925)
  const double ext[3] = {cfg.outer_hi[0] - cfg.outer_lo[0], cfg.outer_hi[1] - cfg.outer_lo[1],
                         cfg.outer_hi[2] - cfg.outer_lo[2]};
  c->step = smax(ext[0], smax(ext[1], ext[2])) / cfg.march_step_divisor;
  // placement: partition p on rank p % world; rank-major slot order
  c->part_rank.resize(c->P);
  c->local_of_global.assign(c->P, 0xff);
  for (uint32_t p = 0; p < c->P; ++p) {
    c->part_rank[p] = int(p % uint32_t(c->world));
    if (c->part_rank[p] == c->rank) {
      c->local_of_global[p] = uint8_t(c->local.size());
      c->local.push_back(p);
    }
  }
  c->slot_of_part.assign(c->P, 0);
  for (int r = 0; r < c->world; ++r)
    for (uint32_t p = 0; p < c->P; ++p)
      if (c->part_rank[p] == r) {
        c->slot_of_part[p] = uint8_t(c->part_of_slot.size());
        c->part_of_slot.push_back(p);
      }
  // per local partition: boxes, occupancy shapes, field layouts
  const uint32_t nl = uint32_t(c->local.size());
  c->parts.resize(nl);
  c->fields.resize(2 * nl);
  c->layouts.resize(nl);
  c->field_dev_off.assign(2 * nl, 0);
  c->field_size.assign(2 * nl, 0);
  c->field_segs.assign(2 * nl, {});
  if (const char* e = std::getenv("DG_ENC_PAIRED")) c->enc_paired = std::strcmp(e, "0") != 0;
  c->pair_rows = 0;
  c->pair_segs.clear();
  uint64_t poff = 0, ooff = 0, doff = 0;
  for (uint32_t lp = 0; lp < nl; ++lp) {
    const uint32_t gid = c->local[lp];
    const uint32_t ix = gid % cfg.kx, iy = gid / cfg.kx;
    PartDesc& pd = c->parts[lp];
    std::memset(&pd, 0, sizeof pd);
    pd.global_id = gid;
    pd.fine_lo[0] = g.xp[ix];
    pd.fine_lo[1] = g.yp[iy];
    pd.fine_lo[2] = cfg.inner_lo[2];
    pd.fine_hi[0] = g.xp[ix + 1];
    pd.fine_hi[1] = g.yp[iy + 1];
    pd.fine_hi[2] = cfg.inner_hi[2];
    pd.coarse_lo[0] = ix == 0 ? cfg.outer_lo[0] : g.xp[ix];
    pd.coarse_lo[1] = iy == 0 ? cfg.outer_lo[1] : g.yp[iy];
    pd.coarse_lo[2] = cfg.outer_lo[2];
    pd.coarse_hi[0] = ix == cfg.kx - 1 ? cfg.outer_hi[0] : g.xp[ix + 1];
    pd.coarse_hi[1] = iy == cfg.ky - 1 ? cfg.outer_hi[1] : g.yp[iy + 1];
    pd.coarse_hi[2] = cfg.outer_hi[2];
    c->part_param_off.push_back(poff);
    uint64_t flat = 0;  // reference-order offset within the partition
    for (int casc = 0; casc < 2; ++casc) {
      const double* lo = casc == 0 ? pd.fine_lo : pd.coarse_lo;
      const double* hi = casc == 0 ? pd.fine_hi : pd.coarse_hi;
      const double aspect[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
      // occupancy grid (grid.cpp:161-172)
      grid_shape(aspect, cfg.occ_resolution, pd.occ_n[casc]);
      const uint32_t bdim[3] = {kOccBX, kOccBY, kOccBZ};
      uint64_t bricks = 1;
      for (int a = 0; a < 3; ++a) {
        pd.occ_nb[casc][a] = (pd.occ_n[casc][a] + bdim[a] - 1) / bdim[a];
        bricks *= pd.occ_nb[casc][a];
      }
      pd.occ_off[casc] = ooff;  // bricked bitfield
      ooff += bricks * (kOccBX * kOccBY * kOccBZ);
      pd.den_off[casc] = doff;  // linear density
      doff += uint64_t(pd.occ_n[casc][0]) * pd.occ_n[casc][1] * pd.occ_n[casc][2];
      // hash grid (grid.cpp:90-105) + MLPs (field.cpp:189-201)
      FieldDesc& fd = c->fields[casc * nl + lp];
      std::memset(&fd, 0, sizeof fd);
      for (int a = 0; a < 3; ++a) {
        fd.box_lo[a] = lo[a];
        fd.box_hi[a] = hi[a];
      }
      fd.L = cfg.grid_levels;
      fd.coarse = uint32_t(casc);
      fd.app_dim = cfg.appearance_dim;
      fd.part = lp;
      fd.base = poff;
      const uint32_t T = 1u << (casc == 0 ? cfg.fine_table_log2 : cfg.coarse_table_log2);
      std::vector<dg_ctx::Seg>& segs = c->field_segs[casc * nl + lp];
      uint64_t o = 0, of = 0;  // device / flat offsets within the field
      auto seg = [&](uint64_t count) {
        if (!segs.empty() && segs.back().dev + segs.back().count == o &&
            segs.back().flat + segs.back().count == of)
          segs.back().count += count;
        else
          segs.push_back({o, of, count});
      };
      for (uint32_t l = 0; l < cfg.grid_levels; ++l) {
        LevelDesc& lv = fd.lv[l];
        const uint32_t n = level_resolution(cfg.grid_levels, cfg.base_resolution, cfg.max_resolution, l);
        grid_shape(aspect, n, lv.n);
        const uint64_t vox = uint64_t(lv.n[0]) * lv.n[1] * lv.n[2];
        lv.hashed = vox <= T ? 0u : 1u;
        const uint64_t rows = lv.hashed ? T : vox;
        lv.mask = lv.hashed ? T - 1 : 0u;
        lv.rows = uint32_t(rows);
        o = (o + 3) & ~uint64_t(3);  // 16-byte aligned table: row pairs (2m, 2m+1) are float4s
        lv.offset = o;
        lv.poff = kNoPair;
        // one-to-one level: x-neighbour pairs as one float4, when the paired copy (16 B per row)
        // still fits L2 next to the rest of its pass (the backward's float4 reds RMW it)
        if (!lv.hashed && c->enc_paired && rows * 16 <= (64ull << 20)) {
          lv.poff = c->pair_rows;
          c->pair_segs.push_back({c->pair_rows, poff + o, rows});
          c->pair_rows += rows;
        }
        c->layouts[lp].push_back({flat + of, rows * 2, uint32_t(casc), 0u, l, 0u});
        seg(rows * 2);
        o += rows * 2;
        of += rows * 2;
      }
      const uint32_t enc = cfg.grid_levels * 2, cin = 31 + cfg.appearance_dim;
      auto add = [&](uint64_t& field_off, uint64_t size, uint32_t kind, uint32_t idx) {
        field_off = o;
        c->layouts[lp].push_back({flat + of, size, uint32_t(casc), kind, idx, 0u});
        seg(size);
        o += size;
        of += size;
      };
      add(fd.dw0, 64ull * enc, 1, 0);
      add(fd.db0, 64, 2, 0);
      add(fd.dw1, 16ull * 64, 1, 1);
      add(fd.db1, 16, 2, 1);
      add(fd.cw0, 64ull * cin, 3, 0);
      add(fd.cb0, 64, 4, 0);
      add(fd.cw1, 64ull * 64, 3, 1);
      add(fd.cb1, 64, 4, 1);
      add(fd.cw2, 3ull * 64, 3, 2);
      add(fd.cb2, 3, 4, 2);
      fd.size = o;
      c->field_dev_off[casc * nl + lp] = poff;
      c->field_size[casc * nl + lp] = of;
      flat += of;
      poff += o;
      poff = (poff + 3) & ~uint64_t(3);  // 16-byte alignment of every field (float2/float4 access)
    }
    c->part_param_cnt.push_back(flat);
  }
  c->n_params = poff;
  c->occ_bytes = std::max<uint64_t>(ooff, 16);
  c->occ_den_n = std::max<uint64_t>(doff, 16);
  return DG_OK;
}

int upload(DBuf& b, const void* src, size_t bytes, cudaStream_t s) {
  TRY(b.ensure(bytes ? bytes : 16));
  if (bytes) CU(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, s));
  return DG_OK;
}

void* pin_alloc(dg_ctx* c, size_t bytes) {
  const size_t at = (c->pin_used + 15) & ~size_t(15);
  if (!c->pin || at + bytes > c->pin_cap) return nullptr;
  c->pin_used = at + bytes;
  return c->pin + at;
}

// Wait for the step's stream.  With a multi-rank backend the wait polls the backend for
// asynchronous failures and gives up after its timeout (Worker::Setup::recv_timeout,
// worker.hpp:82): a dead or stalled peer turns into DG_ETIMEOUT / DG_ENCCL (the reference
// throws "missing PartialScatter", worker.cpp:340-347) instead of a hang; the backend is then
// aborted so the device work blocked on the peer returns.
int step_sync(dg_ctx* c) {
  if (!c->comm || c->world == 1) {
    CU(cudaStreamSynchronize(c->stream));
    return DG_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  const auto deadline = t0 + c->comm->timeout();
  for (uint32_t spin = 0;; ++spin) {
    const cudaError_t e = cudaStreamQuery(c->stream);
    if (e == cudaSuccess) return DG_OK;
    if (e != cudaErrorNotReady) return set_err(DG_ECUDA, "CUDA error: %s", cudaGetErrorString(e));
    std::string err;
    const int rc = c->comm->poll(err);
    if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
    if (std::chrono::steady_clock::now() > deadline) {
      c->comm->abort();
      return set_err(DG_ETIMEOUT, "worker: missing PartialScatter (no progress from peers within %lld ms)",
                     (long long)c->comm->timeout().count());
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

int pin_reset(dg_ctx* c) {
  TRY(step_sync(c));  // nothing in flight reads the arena any more
  c->pin_used = 0;
  return DG_OK;
}

// Small step-time upload through the pinned arena (falls back to a plain copy when full).
int upload_small(dg_ctx* c, DBuf& b, const void* src, size_t bytes) {
  void* h = bytes ? pin_alloc(c, bytes) : nullptr;
  if (!h) return upload(b, src, bytes, c->stream);
  std::memcpy(h, src, bytes);
  TRY(b.ensure(bytes));
  CU(cudaMemcpyAsync(b.p, h, bytes, cudaMemcpyHostToDevice, c->stream));
  return DG_OK;
}

// Pinned landing slot for a small readback (nullptr when the arena is full: callers then
// read into their own memory).
template <class T>
T* pin_slot(dg_ctx* c, size_t count) {
  return static_cast<T*>(pin_alloc(c, count * sizeof(T)));
}

void occ_start_prefetch(dg_ctx* c);

int ctx_alloc(dg_ctx* c) {
  cudaStream_t s = c->stream;
  TRY(upload(c->d_geo, &c->geo, sizeof(Geo), s));
  TRY(upload(c->d_parts, c->parts.data(), sizeof(PartDesc) * c->parts.size(), s));
  TRY(upload(c->d_fields, c->fields.data(), sizeof(FieldDesc) * c->fields.size(), s));
  TRY(upload(c->slot_of_part_d, c->slot_of_part.data(), c->slot_of_part.size(), s));
  std::vector<uint8_t> gol(c->local.begin(), c->local.end());
  TRY(upload(c->global_of_local_d, gol.data(), gol.size(), s));
  TRY(upload(c->local_of_global_d, c->local_of_global.data(), c->local_of_global.size(), s));
  const size_t pb = std::max<uint64_t>(c->n_params, 4) * sizeof(float);
  for (DBuf* b : {&c->params, &c->grads, &c->adam_m, &c->adam_v}) {
    TRY(b->ensure(pb));
    CU(cudaMemsetAsync(b->p, 0, pb, s));
  }
  if (c->pair_rows) {
    TRY(c->pairs.ensure(c->pair_rows * 16 + 16));
    TRY(c->pgrads.ensure(c->pair_rows * 16 + 16));
    CU(cudaMemsetAsync(c->pgrads.p, 0, c->pair_rows * 16, s));
    TRY(upload(c->pair_segs_d, c->pair_segs.data(), c->pair_segs.size() * sizeof(PairSeg), s));
  }
  TRY(c->occ.ensure(c->occ_bytes));
  CU(cudaMemsetAsync(c->occ.p, 1, c->occ_bytes, s));  // fill_occupied (worker.cpp:199-200)
  // occupancy densities start at the initial threshold (grid.cpp:188-191)
  const double thr0 = c->cfg.occ_threshold_early * c->cfg.occ_threshold_scale;
  c->occ_thr.assign(2 * c->local.size(), thr0);
  TRY(c->occ_den.ensure(c->occ_den_n * sizeof(float)));
  {
    std::vector<float> den(c->occ_den_n, float(thr0));
    CU(cudaMemcpyAsync(c->occ_den.p, den.data(), den.size() * sizeof(float), cudaMemcpyHostToDevice, s));
    CU(cudaStreamSynchronize(s));
  }
  for (uint32_t gid : c->local) c->occ_rng.emplace_back(splitmix64(counter_hash(c->cfg.seed, 0x0cc0, gid, 0)));
  if (c->cfg.occupancy_updates) {  // buffers for the largest (warm-up) update, allocated once
    uint64_t max_cells = 0, all_cells = 0;
    for (const PartDesc& pd : c->parts)
      for (int casc = 0; casc < 2; ++casc) {
        const uint64_t n = uint64_t(pd.occ_n[casc][0]) * pd.occ_n[casc][1] * pd.occ_n[casc][2];
        max_cells = std::max(max_cells, n);
        all_cells += n;
      }
    TRY(c->occ_pts.ensure(max_cells * 3 * sizeof(double) + 16));
    TRY(c->occ_sigma.ensure(max_cells * sizeof(float) + 16));
    c->occ_host_n = all_cells * 3;
    CU(cudaHostAlloc(reinterpret_cast<void**>(&c->occ_host), c->occ_host_n * sizeof(double) + 16,
                     cudaHostAllocDefault));
    TRY(c->occ_pts_warm.ensure(c->occ_host_n * sizeof(double) + 16));
    occ_start_prefetch(c);
  }
  // default appearance: one zero row for image 0
  c->app_rows = 1;
  c->n_images = 1;
  TRY(c->app.ensure(64 * sizeof(float)));
  CU(cudaMemsetAsync(c->app.p, 0, 64 * sizeof(float), s));
  TRY(c->dropped.ensure(sizeof(unsigned long long)));
  TRY(c->loss.ensure(sizeof(LossAccum)));
  TRY(c->error.ensure(sizeof(uint32_t)));
  CU(cudaStreamSynchronize(s));
  return DG_OK;
}

template <class T>
int exclusive_scan(dg_ctx* c, const T* in, T* out, uint64_t n) {
  size_t tmp = 0;
  CU(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, c->stream));
  TRY(c->cub_tmp.ensure(tmp + 16));
  CU(cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tmp, in, out, n, c->stream));
  return DG_OK;
}

void mark(dg_ctx* c, int i) {
  if (c->timing) cudaEventRecord(c->ev[i], c->stream);
}

ItemArrays item_arrays(dg_ctx* c) {
  ItemArrays it;
  it.rec = c->items_rec;
  it.te = c->it_te.as<double>();
  it.tx = c->it_tx.as<double>();
  it.t0 = c->it_t0.as<double>();
  it.t1 = c->it_t1.as<double>();
  it.nseg = c->it_nseg.as<uint8_t>();
  it.order = c->it_order.as<uint8_t>();
  it.part = c->it_part.as<uint8_t>();
  it.sched = c->it_sched.as<uint8_t>();
  it.cnt = c->it_cnt.as<uint32_t>();
  it.off = c->it_off.as<uint32_t>();
  it.ncb = c->it_ncb.as<uint32_t>();
  it.runs = c->it_runs.as<double2>();
  it.run_casc = c->it_runc.as<uint8_t>();
  it.nrun = c->it_nrun.as<uint8_t>();
  it.contains = c->it_contains.as<uint32_t>();
  it.cscan = c->it_cscan.as<uint32_t>();
  it.partial = c->it_partial.as<float4>();
  it.depth = c->it_depth.as<float>();
  it.xdist = c->cross_active ? c->it_xdist.as<float4>() : nullptr;
  return it;
}

SampleArrays sample_arrays(dg_ctx* c) {
  SampleArrays sm;
  sm.t = c->s_t.as<double>();
  sm.delta = c->s_delta.as<double>();
  sm.item = c->s_item.as<uint32_t>();
  sm.p = c->enc_pcache ? c->s_p.as<double>() : nullptr;
  sm.pn = uint64_t(c->n_fine) + c->n_coarse;
  sm.X = c->s_X.as<float>();
  sm.out = c->s_out.as<float4>();
  sm.grad = c->s_grad.as<float4>();
  sm.dX = c->s_dX.as<float>();
  sm.inv = c->ordered ? c->s_inv.as<uint32_t>() : nullptr;
  sm.grad_ord = c->ordered ? c->s_grad_ord.as<float4>() : nullptr;
  return sm;
}

// Stage the batch into device buffers (host -> device when mem == HOST).
int stage_batch(dg_ctx* c, const dg_ray_batch* b, const double*& o, const double*& d,
                const float*& gt, const uint32_t*& img) {
  const uint64_t n = b->n;
  if (b->mem == DG_MEM_DEVICE) {
    o = b->origin;
    d = b->dir;
    gt = b->color_gt;
    img = b->image_id;
    return DG_OK;
  }
  cudaStream_t s = c->stream;
  c->h2d += n * 48 + (b->color_gt ? n * 12 : 0) + (b->image_id ? n * 4 : 0);
  TRY(c->h_o.ensure(n * 24 + 16));
  TRY(c->h_d.ensure(n * 24 + 16));
  if (n) CU(cudaMemcpyAsync(c->h_o.p, b->origin, n * 24, cudaMemcpyHostToDevice, s));
  if (n) CU(cudaMemcpyAsync(c->h_d.p, b->dir, n * 24, cudaMemcpyHostToDevice, s));
  o = c->h_o.as<double>();
  d = c->h_d.as<double>();
  gt = nullptr;
  img = nullptr;
  if (b->color_gt) {
    TRY(c->h_gt.ensure(n * 12 + 16));
    if (n) CU(cudaMemcpyAsync(c->h_gt.p, b->color_gt, n * 12, cudaMemcpyHostToDevice, s));
    gt = c->h_gt.as<float>();
  }
  if (b->image_id) {
    TRY(c->h_img.ensure(n * 4 + 16));
    if (n) CU(cudaMemcpyAsync(c->h_img.p, b->image_id, n * 4, cudaMemcpyHostToDevice, s));
    img = c->h_img.as<uint32_t>();
  }
  return DG_OK;
}

// Block transpose between [a][b] and [b][a] layouts of fixed-size records (8-byte words).
__global__ void k_block_permute(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                uint32_t words, const uint64_t* __restrict__ tab, uint32_t nblk,
                                uint64_t total) {
  // tab: [nblk] src start, [nblk] dst start, [nblk] count (records)
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= total) return;
  uint32_t b = 0;
  while (b + 1 < nblk && r >= tab[b + 1]) ++b;
  const uint64_t k = r - tab[b];
  const uint64_t so = tab[b] + k, dof = tab[nblk + b] + k;
  for (uint32_t w = 0; w < words; ++w) dst[dof * words + w] = src[so * words + w];
}

// Runs the K1/X1/K2 front half shared by train and render.  On return the items and
// sample arrays are filled (march done) and c->part_item_off / c->field_off describe them.
// Spatial sample order (kernels_order.cu): after the march, each field's samples are radix-
// sorted by the Morton code of their normalised position (2^order_bits cells per axis).  The
// encode passes, the MLP tiles, X / dX and the ReLU masks then run in that order; positions and
// item ids are gathered into it once (s_p / s_item_ord), and the MLP reads its upstream and
// writes its outputs through s_perm (sorted slot -> march sample), so the march / compositing /
// merge arrays keep the march (ray, t) order.  Samples of one lattice cell now share a CTA: the
// forward's corner rows hit L1 / L2 instead of HBM, and the backward scatters from spatially
// compact CTAs (visited in a strided CTA order so concurrently running CTAs do not contend for
// the same rows).
int order_samples(dg_ctx* c, uint64_t NS, cudaStream_t s) {
  c->ordered = false;
  if (!c->sample_order || !c->enc_pcache || !NS) return DG_OK;
  // Only when a field's level tables outgrow what random accesses keep L2-resident (~75 MB on
  // this B200, tools/ubench/l2_curve.cu; the encode passes group levels up to 192 / 96 MB): with
  // small tables (C1: 4 MB per level, ~40 MB per field) every gather hits L2 in march order
  // already and the sort would be pure overhead; C2 (32 MB per level, ~0.3 GB per field) gains
  // 4.56 -> 5.31 M training and 12.3 -> 17.2 M render rays/s.  DG_SAMPLE_ORDER=2 forces it.
  if (c->sample_order == 1) {
    uint64_t big = 0;
    for (const FieldDesc& fd : c->fields) {
      uint64_t field_bytes = 0;
      for (uint32_t l = 0; l < fd.L; ++l) field_bytes += uint64_t(fd.lv[l].rows) * 8;
      big = std::max(big, field_bytes);
    }
    if (big < (64ull << 20)) return DG_OK;
  }
  const uint32_t C = c->order_chunk;
  TRY(c->s_perm.ensure(NS * 4 + 16));
  TRY(c->s_inv.ensure(NS * 4 + 16));
  TRY(c->s_p_alt.ensure(NS * 24 + 16));
  TRY(c->s_item_ord.ensure(NS * 4 + 16));
  TRY(c->s_grad_ord.ensure(NS * 16 + 16));
  TRY(c->ord_scratch.ensure((NS / C + 1) * 16 + 16));
  const size_t tb = order_sort_tmp_bytes(uint32_t(NS / C + 1));
  TRY(c->ord_tmp.ensure(tb + 16));
  for (size_t f = 0; f + 1 < c->field_off.size(); ++f) {
    const uint32_t o = c->field_off[f], n = c->field_off[f + 1] - o;
    const int k = launch_order_field(c->s_p.as<double>(), c->s_item.as<uint32_t>(), NS, o, n, C, c->order_bits,
                                     c->s_perm.as<uint32_t>(), c->s_inv.as<uint32_t>(), c->s_p_alt.as<double>(),
                                     c->s_item_ord.as<uint32_t>(), c->ord_scratch.as<uint32_t>(), c->ord_tmp.p, tb, s);
    if (k < 0) return set_err(DG_ECUDA, "sample order: radix sort failed");
    c->launches += k;
  }
  std::swap(c->s_p.p, c->s_p_alt.p);  // s_p now holds the positions in sample order
  std::swap(c->s_p.bytes, c->s_p_alt.bytes);
  c->ordered = true;
  return DG_OK;
}

int front_half(dg_ctx* c, const dg_ray_batch* b, int train, uint64_t batch_id, uint64_t* dropped_out,
               uint64_t* bytes_sent) {
  c->ordered = false;
  cudaStream_t s = c->stream;
  const uint64_t n = b->n;
  const uint32_t P = c->P, nl = uint32_t(c->local.size());
  const double* o;
  const double* d;
  const float* gt;
  const uint32_t* img;
  TRY(stage_batch(c, b, o, d, gt, img));
  mark(c, 0);
  // ---- K1: segment home rays ----
  const uint64_t nf = uint64_t(P) * n + 1;
  TRY(c->h_nseg.ensure(n + 16));
  TRY(c->h_sched.ensure(n * kMaxSeg + 16));
  TRY(c->h_flags.ensure(nf * 4));
  TRY(c->h_pos.ensure(nf * 4));
  CU(cudaMemsetAsync(c->h_flags.p, 0, nf * 4, s));
  CU(cudaMemsetAsync(c->dropped.p, 0, 8, s));
  CU(cudaMemsetAsync(c->error.p, 0, 4, s));
  launch_segment_home(c->d_geo.as<Geo>(), o, d, n, c->slot_of_part_d.as<uint8_t>(),
                      c->h_nseg.as<uint8_t>(), c->h_sched.as<uint8_t>(), c->h_flags.as<uint32_t>(),
                      c->dropped.as<unsigned long long>(), s);
  ++c->launches;
  TRY(exclusive_scan(c, c->h_flags.as<uint32_t>(), c->h_pos.as<uint32_t>(), nf));
  // per-slot dispatch counts: pos[slot * n] for slot = 0..P
  TRY(c->small.ensure(4096 * 4));
  std::vector<uint32_t> slot_start(P + 1);
  uint32_t* ss_pin = pin_slot<uint32_t>(c, P + 1);
  unsigned long long* dr_pin = pin_slot<unsigned long long>(c, 1);
  unsigned long long dropped = 0;
  CU(cudaMemcpy2DAsync(ss_pin ? ss_pin : slot_start.data(), 4, c->h_pos.as<uint32_t>(), n ? n * 4 : 4, 4,
                       P + 1, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(dr_pin ? dr_pin : &dropped, c->dropped.p, 8, cudaMemcpyDeviceToHost, s));
  TRY(step_sync(c));
  if (ss_pin) std::memcpy(slot_start.data(), ss_pin, (P + 1) * 4);
  if (dr_pin) dropped = *dr_pin;
  c->d2h += (P + 1) * 4 + 8;
  if (n == 0)
    for (auto& v : slot_start) v = 0;
  *dropped_out = dropped;
  std::vector<uint64_t> send_cnt(P);  // records to each partition (by global id)
  for (uint32_t p = 0; p < P; ++p)
    send_cnt[p] = slot_start[c->slot_of_part[p] + 1] - slot_start[c->slot_of_part[p]];
  const uint64_t total_send = slot_start[P];
  // ---- X1: dispatch ----
  std::vector<uint32_t> pio(nl + 1, 0);
  uint64_t n_items = 0;
  if (c->world == 1) {
    mark(c, 11);
    for (uint32_t lp = 0; lp < nl; ++lp) pio[lp + 1] = pio[lp] + uint32_t(send_cnt[c->local[lp]]);
    n_items = total_send;
    TRY(c->rec.ensure(n_items * sizeof(RayRec) + 16));
    launch_pack_dispatch(n, P, c->h_nseg.as<uint8_t>(), c->h_sched.as<uint8_t>(),
                         c->slot_of_part_d.as<uint8_t>(), c->h_pos.as<uint32_t>(), o, d, gt, img,
                         b->first_ray_id, c->rec.as<RayRec>(), PeerDst{nullptr, nullptr, 1}, s);
    ++c->launches;
    c->items_rec = c->rec.as<RayRec>();
  } else if (PeerComm* pc = c->comm->peer()) {
    // Exchange 1 over peer memory: the full count matrix (every rank's per-partition counts)
    // gives every owner's item layout [local partition][src rank][ray]; the pack kernel then
    // stores each record at its final place in the owner's item array, so neither the
    // all-to-all copy nor the receive-side block permute exists.
    const int W = c->world;
    std::string err;
    std::vector<uint64_t> all(uint64_t(W) * P);  // all[src * P + p]
    int rc = pc->allgather(send_cnt.data(), uint64_t(P) * 8, all.data(), err);
    if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
    std::vector<uint64_t> part_base(P, 0), items_of(W, 0);
    for (int r = 0; r < W; ++r) {
      uint64_t off = 0;
      for (uint32_t p : local_partitions(r, W, P))
        for (int src = 0; src < W; ++src) {
          if (src == c->rank) part_base[p] = off;
          off += all[uint64_t(src) * P + p];
        }
      items_of[r] = off;
    }
    for (uint32_t lp = 0; lp < nl; ++lp) {
      uint64_t t = 0;
      for (int src = 0; src < W; ++src) t += all[uint64_t(src) * P + c->local[lp]];
      pio[lp + 1] = pio[lp] + uint32_t(t);
    }
    n_items = items_of[c->rank];
    rc = pc->reserve(PeerComm::kItems, *std::max_element(items_of.begin(), items_of.end()) * sizeof(RayRec) + 16,
                     err);
    if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
    TRY(upload_small(c, c->peer_off, part_base.data(), part_base.size() * 8));
    {  // the block table of the staged path: the render's reply exchange walks it back
      DispatchPlan plan;
      plan_dispatch(c->rank, W, P, send_cnt.data(), all.data(), sizeof(RayRec), plan);
      std::vector<uint64_t> tab(plan.block_src);
      tab.insert(tab.end(), plan.block_dst.begin(), plan.block_dst.end());
      TRY(upload_small(c, c->perm_tab, tab.data(), tab.size() * 8));
    }
    mark(c, 11);
    launch_pack_dispatch(n, P, c->h_nseg.as<uint8_t>(), c->h_sched.as<uint8_t>(),
                         c->slot_of_part_d.as<uint8_t>(), c->h_pos.as<uint32_t>(), o, d, gt, img,
                         b->first_ray_id, nullptr,
                         PeerDst{pc->peers_dev(PeerComm::kItems), c->peer_off.as<uint64_t>(), uint32_t(W)}, s);
    ++c->launches;
    for (uint32_t p = 0; p < P; ++p)
      if (int(p % uint32_t(W)) != c->rank) *bytes_sent += send_cnt[p] * sizeof(RayRec);
    rc = pc->barrier(s, err);  // every rank's records are in place
    if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
    c->h2d += P * 8;
    c->items_rec = static_cast<RayRec*>(pc->local(PeerComm::kItems));
  } else {
    const int W = c->world;
    TRY(c->x_send.ensure(total_send * sizeof(RayRec) + 16));
    launch_pack_dispatch(n, P, c->h_nseg.as<uint8_t>(), c->h_sched.as<uint8_t>(),
                         c->slot_of_part_d.as<uint8_t>(), c->h_pos.as<uint32_t>(), o, d, gt, img,
                         b->first_ray_id, c->x_send.as<RayRec>(), PeerDst{nullptr, nullptr, 1}, s);
    ++c->launches;
    // counts exchange: every rank sends its full per-partition count vector to every peer
    std::vector<uint64_t> cnt_send(uint64_t(W) * P), cnt_recv(uint64_t(W) * P);
    for (int r = 0; r < W; ++r)
      for (uint32_t p = 0; p < P; ++p) cnt_send[uint64_t(r) * P + p] = send_cnt[p];
    TRY(c->send_buf.ensure(cnt_send.size() * 8));
    TRY(c->recv_buf.ensure(cnt_recv.size() * 8));
    TRY(upload_small(c, c->send_buf, cnt_send.data(), cnt_send.size() * 8));
    std::vector<uint64_t> sb(W, uint64_t(P) * 8), rb(W, uint64_t(P) * 8);
    std::string err;
    int rc = c->comm->alltoallv(c->send_buf.p, sb, c->recv_buf.p, rb, s, err);
    if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
    uint64_t* cr_pin = pin_slot<uint64_t>(c, cnt_recv.size());
    CU(cudaMemcpyAsync(cr_pin ? cr_pin : cnt_recv.data(), c->recv_buf.p, cnt_recv.size() * 8,
                       cudaMemcpyDeviceToHost, s));
    TRY(step_sync(c));
    if (cr_pin) std::memcpy(cnt_recv.data(), cr_pin, cnt_recv.size() * 8);
    c->h2d += cnt_send.size() * 8;
    c->d2h += cnt_recv.size() * 8;
    // cnt_recv[src][p]: records src sends to partition p -> layouts (exchange_plan.cpp)
    DispatchPlan plan;
    plan_dispatch(c->rank, W, P, send_cnt.data(), cnt_recv.data(), sizeof(RayRec), plan);
    n_items = plan.n_items;
    TRY(c->x_recv.ensure(n_items * sizeof(RayRec) + 16));
    mark(c, 11);
    rc = c->comm->alltoallv(c->x_send.p, plan.send_bytes, c->x_recv.p, plan.recv_bytes, s, err);
    if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
    for (int r = 0; r < W; ++r)
      if (r != c->rank) *bytes_sent += plan.send_bytes[r];
    pio = plan.item_off;
    const uint32_t nblk = nl * uint32_t(W);
    std::vector<uint64_t> tab(plan.block_src);
    tab.insert(tab.end(), plan.block_dst.begin(), plan.block_dst.end());
    TRY(upload_small(c, c->perm_tab, tab.data(), tab.size() * 8));
    TRY(c->rec.ensure(n_items * sizeof(RayRec) + 16));
    if (n_items) {
      k_block_permute<<<unsigned((n_items + 255) / 256), 256, 0, s>>>(
          c->x_recv.as<uint64_t>(), c->rec.as<uint64_t>(), sizeof(RayRec) / 8,
          c->perm_tab.as<uint64_t>(), nblk, n_items);
      ++c->launches;
    }
    c->items_rec = c->rec.as<RayRec>();
  }
  mark(c, 1);
  // ---- K2: item setup + counts ----
  const uint32_t NI = uint32_t(n_items);
  c->n_items = NI;
  c->part_item_off = pio;
  TRY(upload_small(c, c->part_item_off_d, pio.data(), pio.size() * 4));
  c->h2d += pio.size() * 4;
  TRY(c->it_te.ensure(uint64_t(NI) * 8 + 16));
  TRY(c->it_tx.ensure(uint64_t(NI) * 8 + 16));
  TRY(c->it_t0.ensure(uint64_t(NI) * 8 + 16));
  TRY(c->it_t1.ensure(uint64_t(NI) * 8 + 16));
  TRY(c->it_nseg.ensure(NI + 16));
  TRY(c->it_order.ensure(NI + 16));
  TRY(c->it_part.ensure(NI + 16));
  TRY(c->it_sched.ensure(uint64_t(NI) * kMaxSeg + 16));
  TRY(c->it_cnt.ensure((2ull * NI + 1) * 4));
  TRY(c->it_off.ensure((2ull * NI + 1) * 4));
  TRY(c->it_ncb.ensure(uint64_t(NI) * 4 + 16));
  TRY(c->it_runs.ensure(uint64_t(NI) * kMaxRuns * sizeof(double2) + 16));
  TRY(c->it_runc.ensure(uint64_t(NI) * kMaxRuns + 16));
  TRY(c->it_nrun.ensure(uint64_t(NI) + 16));
  TRY(c->it_contains.ensure((uint64_t(P) * NI + 1) * 4));
  TRY(c->it_cscan.ensure((uint64_t(P) * NI + 1) * 4));
  TRY(c->it_partial.ensure(uint64_t(NI) * 16 + 16));
  TRY(c->it_depth.ensure(uint64_t(NI) * 4 + 16));
  if (c->cfg.distortion_cross_correction) TRY(c->it_xdist.ensure(uint64_t(NI) * 16 + 16));
  CU(cudaMemsetAsync(c->it_cnt.as<uint32_t>() + 2ull * NI, 0, 4, s));
  CU(cudaMemsetAsync(c->it_contains.as<uint32_t>() + uint64_t(P) * NI, 0, 4, s));
  ItemArrays it = item_arrays(c);
  launch_item_setup(c->d_geo.as<Geo>(), c->d_parts.as<PartDesc>(), c->occ.as<uint8_t>(),
                    c->part_item_off_d.as<uint32_t>(), nl, NI, it, P, c->step, c->cfg.seed,
                    batch_id, train, int(c->cfg.wire_f32), c->app_rows, c->error.as<uint32_t>(), s);
  ++c->launches;
  TRY(exclusive_scan(c, c->it_cnt.as<uint32_t>(), c->it_off.as<uint32_t>(), 2ull * NI + 1));
  if (train && P > 1)
    TRY(exclusive_scan(c, c->it_contains.as<uint32_t>(), c->it_cscan.as<uint32_t>(),
                       uint64_t(P) * NI + 1));
  // field sample ranges: off[pio[lp]] (fine) and off[NI + pio[lp]] (coarse), lp = 0..nl
  std::vector<uint32_t> fo(2 * (nl + 1));
  uint32_t* fo_pin = pin_slot<uint32_t>(c, fo.size() + 1);  // + the error flag
  uint32_t* fo_dst = fo_pin ? fo_pin : fo.data();
  uint32_t err_flag = 0;
  for (uint32_t k = 0; k <= nl; ++k) {
    CU(cudaMemcpyAsync(&fo_dst[k], c->it_off.as<uint32_t>() + pio[k], 4, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(&fo_dst[nl + 1 + k], c->it_off.as<uint32_t>() + NI + pio[k], 4,
                       cudaMemcpyDeviceToHost, s));
  }
  CU(cudaMemcpyAsync(fo_pin ? &fo_pin[fo.size()] : &err_flag, c->error.p, 4, cudaMemcpyDeviceToHost, s));
  TRY(step_sync(c));
  if (fo_pin) {
    std::memcpy(fo.data(), fo_pin, fo.size() * 4);
    err_flag = fo_pin[fo.size()];
  }
  c->d2h += fo.size() * 4 + 4;
  if (err_flag & 1u) return set_err(DG_ERANGE, "appearance: unknown image id");
  if (err_flag & 2u) return set_err(DG_EPROTO, "worker: dispatched ray does not intersect this region");
  // fields: [fine lp 0..nl-1][coarse lp 0..nl-1]
  c->field_off.assign(2 * nl + 1, 0);
  for (uint32_t lp = 0; lp < nl; ++lp) c->field_off[lp] = fo[lp];
  for (uint32_t lp = 0; lp < nl; ++lp) c->field_off[nl + lp] = fo[nl + 1 + lp];
  c->field_off[2 * nl] = fo[2 * nl + 1];
  c->n_fine = fo[nl];
  c->n_coarse = fo[2 * nl + 1] - fo[nl];
  const uint64_t NS = uint64_t(c->n_fine) + c->n_coarse;
  TRY(c->s_t.ensure(NS * 8 + 16));
  TRY(c->s_delta.ensure(NS * 8 + 16));
  TRY(c->s_item.ensure(NS * 4 + 16));
  if (c->enc_pcache) TRY(c->s_p.ensure(NS * 24 + 16));
  TRY(c->s_X.ensure(NS * kEnc * 4 + 16));
  TRY(c->s_out.ensure(NS * 16 + 16));
  TRY(c->s_grad.ensure(NS * 16 + 16));
  TRY(c->s_dX.ensure(NS * kEnc * 4 + 16));
  if (train && c->mlp_impl) TRY(c->s_mask.ensure(NS * 7 * 4 + 16));
  SampleArrays sm = sample_arrays(c);
  launch_march_fill(c->d_parts.as<PartDesc>(), c->occ.as<uint8_t>(), NI, it, sm, c->n_fine,
                    c->step, c->cfg.seed, batch_id, train, s);
  c->launches += 2;  // march fill (runs, with the position cache) + overflow walk
  TRY(order_samples(c, NS, s));
  // tile tables
  std::vector<uint32_t> tf(2 * nl + 1, 0), tb(2 * nl + 1, 0);
  for (uint32_t f = 0; f < 2 * nl; ++f) {
    const uint32_t cnt = c->field_off[f + 1] - c->field_off[f];
    tf[f + 1] = tf[f] + (cnt + 127) / 128;
    tb[f + 1] = tb[f] + (cnt + 63) / 64;
  }
  TRY(upload_small(c, c->field_off_d, c->field_off.data(), c->field_off.size() * 4));
  TRY(upload_small(c, c->tile_off_f, tf.data(), tf.size() * 4));
  TRY(upload_small(c, c->tile_off_b, tb.data(), tb.size() * 4));
  c->h2d += (c->field_off.size() + tf.size() + tb.size()) * 4;
  mark(c, 2);
  c->have_last = true;
  return DG_OK;
}

// The paired copies of the one-to-one level tables (kernels_pairs.cu), from the current
// parameters (after the last Adam step or dg_set_params).
int pairs_expand(dg_ctx* c, cudaStream_t s) {
  if (!c->pair_rows) return DG_OK;
  launch_pairs_expand(c->pair_segs_d.as<PairSeg>(), uint32_t(c->pair_segs.size()), c->pair_rows,
                      c->params.as<float>(), c->pairs.as<float4>(), s);
  ++c->launches;
  return DG_OK;
}

FieldLaunch field_launch(dg_ctx* c, uint64_t budget, std::vector<EncPass>& passes, uint64_t group,
                         uint64_t hgroup) {
  if (!group) group = budget;
  FieldLaunch f{};
  f.fields = c->d_fields.as<FieldDesc>();
  f.parts = c->d_parts.as<PartDesc>();
  f.rec = c->items_rec;
  f.item_part = c->it_part.as<uint8_t>();
  f.s_t = c->s_t.as<double>();
  f.s_item = c->s_item.as<uint32_t>();
  f.fine_total = c->n_fine;
  f.n_total = c->n_fine + c->n_coarse;
  f.n_local = uint32_t(c->local.size());
  f.levels = c->cfg.grid_levels;
  // Passes, per field (a partition's fine or coarse sub-field) that has samples: runs of
  // consecutive levels whose tables fit the slice budget go together; a larger level is cut
  // into S row slices of <= budget each.  Each pass covers only its field's samples, so with
  // several partitions on a GPU the L2 working set is still one table slice.  Measured on
  // B200 (tools/ubench/l2_random.cu): random float2 gathers / reds run 2.2x / 3.5x faster on
  // a 64 MB table than on a 128 MB one.
  // With a single partition per GPU (the fine + coarse fields of one region) one pass covers
  // both fields' samples (kAllFields), as measured fastest there.
  passes.clear();
  const uint32_t nf = uint32_t(c->field_off.size() - 1);
  const bool merged = c->local.size() == 1;
  for (uint32_t fi = 0; fi < (merged ? 1u : nf); ++fi) {
    if (!merged && c->field_off[fi + 1] == c->field_off[fi]) continue;  // no samples in this field
    auto level_bytes = [&](uint32_t l) {
      if (!merged) return uint64_t(c->fields[fi].lv[l].rows) * 8;
      uint64_t b = 0;
      for (const FieldDesc& fd : c->fields) b += uint64_t(fd.lv[l].rows) * 8;
      return b;
    };
    // a pass holding a hashed level groups up to hgroup bytes (if set): a hashed level's
    // gathers are random over its whole table, so several of them in one pass thrash L2 (C2:
    // 32 MB levels, six to a 192 MB pass), while the one-to-one levels' gathers follow the
    // sample order and group well up to the budget (C4: levels 0-8, 118 MB, in one pass)
    // (hashed tables of a few MB, e.g. the coarse field's, stay L2-resident and do not count)
    auto big_hashed = [](const LevelDesc& lv) { return lv.hashed && uint64_t(lv.rows) * 8 >= (8ull << 20); };
    auto level_hashed = [&](uint32_t l) {
      if (!merged) return big_hashed(c->fields[fi].lv[l]);
      for (const FieldDesc& fd : c->fields)
        if (big_hashed(fd.lv[l])) return true;
      return false;
    };
    for (uint32_t l = 0; l < f.levels;) {
      uint32_t l1 = l + 1;
      uint64_t bytes = level_bytes(l);
      const uint64_t gb = std::min(group, budget);  // a sliced pass is always a single level
      bool any_hashed = level_hashed(l);
      while (l1 < f.levels) {
        const bool h = any_hashed || level_hashed(l1);
        const uint64_t lim = h && hgroup ? std::min(gb, hgroup) : gb;
        if (bytes + level_bytes(l1) > lim) break;
        any_hashed = h;
        bytes += level_bytes(l1++);
      }
      const uint32_t S = std::min<uint64_t>(64, std::max<uint64_t>(1, (bytes + budget - 1) / budget));
      for (uint32_t k = 0; k < S; ++k) {
        EncPass ps{uint8_t(l), uint8_t(l1), uint8_t(k), uint8_t(S), merged ? kAllFields : uint8_t(fi), 0, 0, 0,
                   {0u, 0u}, {0xffffffffu, 0xffffffffu}};
        for (uint32_t ll = l; ll < l1; ++ll)  // the pass holds paired one-to-one levels
          for (uint32_t fj = 0; fj < nf; ++fj)
            if ((merged || fj == fi) && c->fields[fj].lv[ll].poff != kNoPair) ps.paired = 1;
        for (uint32_t slot = 0; slot < 2 && S > 1; ++slot) {  // slice bounds, even rows
          const uint32_t fld = merged ? slot : fi;
          if (fld >= c->fields.size()) break;
          const uint64_t rows = c->fields[fld].lv[l].rows;
          ps.lo[slot] = uint32_t((rows * k / S) & ~1ull);
          ps.hi[slot] = k + 1 == S ? 0xffffffffu : uint32_t((rows * (k + 1) / S) & ~1ull);
        }
        passes.push_back(ps);
      }
      l = l1;
    }
  }
  f.n_pass = 0;
  // warp aggregation where ~1.5+ consecutive samples share a cell: cell = extent / n vs. step
  const FieldDesc& f0 = c->fields[0];
  uint32_t agg = 0;
  const double ext = std::max(f0.box_hi[0] - f0.box_lo[0],
                              std::max(f0.box_hi[1] - f0.box_lo[1], f0.box_hi[2] - f0.box_lo[2]));
  const double maxn_agg = ext / (c->enc_agg_samples_per_cell * c->step);
  for (uint32_t l = 0; l < f0.L; ++l)
    if (double(std::max(f0.lv[l].n[0], std::max(f0.lv[l].n[1], f0.lv[l].n[2]))) <= maxn_agg) agg = l + 1;
  f.agg_levels = agg;
  f.params = c->params.as<float>();
  f.grads = c->grads.as<float>();
  f.pairs = c->pair_rows ? c->pairs.as<float4>() : nullptr;
  f.pgrads = c->pair_rows ? c->pgrads.as<float4>() : nullptr;
  f.s_p = c->enc_pcache ? c->s_p.as<double>() : nullptr;
  f.n_fields = uint32_t(c->field_off.size() - 1);
  for (size_t i = 0; i < c->field_off.size(); ++i) f.field_off[i] = c->field_off[i];
  return f;
}

MlpLaunch mlp_launch(dg_ctx* c, bool bwd) {
  MlpLaunch m{};
  m.fields = c->d_fields.as<FieldDesc>();
  m.n_fields = uint32_t(2 * c->local.size());
  m.field_off = c->field_off_d.as<uint32_t>();
  std::vector<uint32_t> dummy;
  const uint32_t nl = uint32_t(c->local.size());
  uint32_t tiles = 0;
  for (uint32_t f = 0; f < 2 * nl; ++f) {
    const uint32_t cnt = c->field_off[f + 1] - c->field_off[f];
    tiles += bwd ? (cnt + 63) / 64 : (cnt + 127) / 128;
    if (f + 1 == nl && !bwd && c->mlp_bwd_paired) m.relu_tiles = tiles;  // fields 0..nl-1: fine (ReLU)
  }
  m.issue_warp = c->mlp_issue_warp;
  m.issue_warp_fwd = c->mlp_issue_warp_fwd;
  m.tile_off = bwd ? c->tile_off_b.as<uint32_t>() : c->tile_off_f.as<uint32_t>();
  m.n_tiles = tiles;
  m.X = c->s_X.as<float>();
  m.x_stride = uint64_t(c->n_fine) + c->n_coarse;
  m.levels = c->cfg.grid_levels;
  m.rec = c->items_rec;
  m.s_item = c->ordered ? c->s_item_ord.as<uint32_t>() : c->s_item.as<uint32_t>();
  m.perm = c->ordered ? c->s_perm.as<uint32_t>() : nullptr;
  m.app_table = c->app.as<float>();
  m.params = c->params.as<float>();
  m.grads = c->grads.as<float>();
  m.out = c->s_out.as<float4>();
  m.grad_in = c->ordered ? c->s_grad_ord.as<float4>() : c->s_grad.as<float4>();
  m.dX = c->s_dX.as<float>();
  m.masks = c->s_mask.as<uint32_t>();  // set by the training step's forward, read by its backward
  return m;
}

// Exchange-2 stream tables.  Stream (q -> p) carries the partials of q's items whose
// schedule contains p, in ray order; pair_cnt[lq][p] is known locally and is symmetric.
int exchange_partials(dg_ctx* c, const std::vector<uint32_t>& pair_cnt, uint64_t* bytes_sent,
                      const PartialRec** recv_out, const float4** recv_x_out) {
  cudaStream_t s = c->stream;
  const uint32_t P = c->P, nl = uint32_t(c->local.size());
  const int W = c->world;
  const bool cross = c->cross_active;
  if (PeerComm* pc = W > 1 ? c->comm->peer() : nullptr) {
    // Exchange 2 over peer memory: with every rank's pair counts, every receiver's stream
    // layout is known, so the pack kernel stores each partial (and its cross-distortion
    // aggregates) straight into the receiving owner's buffer.
    const uint32_t nl_max = (P + uint32_t(W) - 1) / uint32_t(W);
    std::vector<uint32_t> mine(uint64_t(nl_max) * P, 0), all(uint64_t(W) * nl_max * P);
    std::copy(pair_cnt.begin(), pair_cnt.end(), mine.begin());
    std::string err;
    int rc = pc->allgather(mine.data(), mine.size() * 4, all.data(), err);
    if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
    std::vector<PartialPlan> plans(W);
    uint64_t need = 0;
    for (int r = 0; r < W; ++r) {
      plan_partials(r, W, P, all.data() + uint64_t(r) * nl_max * P, sizeof(PartialRec), plans[r]);
      need = std::max(need, plans[r].recv_total);
    }
    rc = pc->reserve(PeerComm::kPartials, need * sizeof(PartialRec) + 16, err);
    if (rc == DG_OK && cross) rc = pc->reserve(PeerComm::kCross, need * sizeof(float4) + 16, err);
    if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
    std::vector<uint64_t> dst(uint64_t(P) * P, 0);  // stream (q -> p): offset in p's owner's buffer
    for (uint32_t q : c->local)
      for (uint32_t p = 0; p < P; ++p)
        if (p != q) dst[uint64_t(q) * P + p] = plans[p % uint32_t(W)].recv_off[uint64_t(q) * P + p];
    TRY(upload_small(c, c->stream_send_d, dst.data(), dst.size() * 8));
    TRY(upload_small(c, c->stream_recv_d, plans[c->rank].recv_off.data(), plans[c->rank].recv_off.size() * 8));
    c->h2d += (dst.size() + plans[c->rank].recv_off.size()) * 8;
    const PeerDst pd{pc->peers_dev(PeerComm::kPartials), nullptr, uint32_t(W)};
    const PeerDst px{cross ? pc->peers_dev(PeerComm::kCross) : nullptr, nullptr, uint32_t(W)};
    launch_pack_partials(c->n_items, item_arrays(c), c->part_item_off_d.as<uint32_t>(),
                         c->global_of_local_d.as<uint8_t>(), c->stream_send_d.as<uint64_t>(), P, nullptr,
                         nullptr, pd, px, s);
    ++c->launches;
    for (uint32_t lq = 0; lq < nl; ++lq)  // records to other ranks (both streams)
      for (uint32_t p = 0; p < P; ++p)
        if (int(p % uint32_t(W)) != c->rank && p != c->local[lq])
          *bytes_sent += uint64_t(pair_cnt[uint64_t(lq) * P + p]) * (sizeof(PartialRec) + (cross ? sizeof(float4) : 0));
    rc = pc->barrier(s, err);
    if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
    *recv_out = static_cast<const PartialRec*>(pc->local(PeerComm::kPartials));
    *recv_x_out = cross ? static_cast<const float4*>(pc->local(PeerComm::kCross)) : nullptr;
    return DG_OK;
  }
  PartialPlan plan;
  plan_partials(c->rank, W, P, pair_cnt.data(), sizeof(PartialRec), plan);
  const std::vector<uint64_t>& send_off = plan.send_off;
  const std::vector<uint64_t>& recv_off = plan.recv_off;
  const std::vector<uint64_t>& sbytes = plan.send_bytes;
  const std::vector<uint64_t>& rbytes = plan.recv_bytes;
  const uint64_t so = plan.send_total, ro = plan.recv_total;
  TRY(upload_small(c, c->stream_send_d, send_off.data(), send_off.size() * 8));
  TRY(upload_small(c, c->stream_recv_d, recv_off.data(), recv_off.size() * 8));
  c->h2d += (send_off.size() + recv_off.size()) * 8;
  TRY(c->send_buf.ensure(so * sizeof(PartialRec) + 16));
  // cross-segment distortion: the three aggregates travel in a parallel stream (16 B/record)
  if (cross) TRY(c->send_x.ensure(so * sizeof(float4) + 16));
  launch_pack_partials(c->n_items, item_arrays(c), c->part_item_off_d.as<uint32_t>(),
                       c->global_of_local_d.as<uint8_t>(), c->stream_send_d.as<uint64_t>(), P,
                       c->send_buf.as<PartialRec>(), cross ? c->send_x.as<float4>() : nullptr,
                       PeerDst{nullptr, nullptr, 1}, PeerDst{nullptr, nullptr, 1}, s);
  ++c->launches;
  *recv_x_out = cross ? c->send_x.as<float4>() : nullptr;
  if (W == 1) {
    *recv_out = c->send_buf.as<PartialRec>();  // single rank: the streams alias
    return DG_OK;
  }
  TRY(c->recv_buf.ensure(ro * sizeof(PartialRec) + 16));
  std::string err;
  int rc = c->comm->alltoallv(c->send_buf.p, sbytes, c->recv_buf.p, rbytes, s, err);
  if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
  for (int r = 0; r < W; ++r)
    if (r != c->rank) *bytes_sent += sbytes[r];
  *recv_out = c->recv_buf.as<PartialRec>();
  if (cross) {
    std::vector<uint64_t> xs(W), xr(W);
    for (int r = 0; r < W; ++r) {
      xs[r] = sbytes[r] / sizeof(PartialRec) * sizeof(float4);
      xr[r] = rbytes[r] / sizeof(PartialRec) * sizeof(float4);
    }
    TRY(c->recv_x.ensure(ro * sizeof(float4) + 16));
    rc = c->comm->alltoallv(c->send_x.p, xs, c->recv_x.p, xr, s, err);
    if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
    for (int r = 0; r < W; ++r)
      if (r != c->rank) *bytes_sent += xs[r];
    *recv_x_out = c->recv_x.as<float4>();
  }
  return DG_OK;
}

template <class T>
int d2h(std::vector<T>& v, const void* src, uint64_t n, cudaStream_t s) {
  v.resize(n);
  if (n) CU(cudaMemcpyAsync(v.data(), src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  return DG_OK;
}


// The jitter point of one sampled cell (grid.cpp:206-214): cell_box + 3 Rng::uniform draws.
inline void occ_point(std::mt19937_64& rng, const double lo[3], const double cell[3],
                      const uint32_t sh[3], uint64_t idx, double* out) {
  const uint64_t ii[3] = {idx % sh[0], (idx / sh[0]) % sh[1], idx / (uint64_t(sh[0]) * sh[1])};
  for (int a = 0; a < 3; ++a) {
    const double clo = lo[a] + cell[a] * double(ii[a]);
    const double chi = clo + cell[a];
    out[a] = clo + (chi - clo) * (double(rng() >> 11) * 0x1.0p-53);
  }
}

inline void occ_geometry(const PartDesc& pd, int casc, const double*& lo, double cell[3], uint64_t& total) {
  const uint32_t* sh = pd.occ_n[casc];
  total = uint64_t(sh[0]) * sh[1] * sh[2];
  lo = casc == 0 ? pd.fine_lo : pd.coarse_lo;
  const double* hi = casc == 0 ? pd.fine_hi : pd.coarse_hi;
  for (int a = 0; a < 3; ++a) cell[a] = (hi[a] - lo[a]) / double(sh[a]);
}

// Fill the pinned buffer with one warm-up update's points for every local partition, in the
// reference's order (per partition: fine grid cells 0..n-1, then coarse; 3 draws per cell).
void occ_generate_warm(dg_ctx* c) {
  uint64_t k = 0;
  for (uint32_t lp = 0; lp < c->local.size(); ++lp)
    for (int casc = 0; casc < 2; ++casc) {
      const double* lo;
      double cell[3];
      uint64_t total;
      occ_geometry(c->parts[lp], casc, lo, cell, total);
      for (uint64_t i = 0; i < total; ++i, k += 3)
        occ_point(c->occ_rng[lp], lo, cell, c->parts[lp].occ_n[casc], i, c->occ_host + k);
    }
}

bool next_update_is_warm(const dg_ctx* c, uint64_t after_step) {
  const uint64_t iv = c->cfg.occ_update_interval;
  if (!c->cfg.occupancy_updates || iv == 0) return false;
  const uint64_t next = (after_step / iv + 1) * iv;
  return next <= c->cfg.occ_warmup_steps;
}

void occ_start_prefetch(dg_ctx* c) {
  if (!c->occ_host || !next_update_is_warm(c, c->worker_step)) return;
  c->occ_rng_before = c->occ_rng;
  c->occ_prefetch = std::async(std::launch::async, [c] { occ_generate_warm(c); });
  c->occ_prefetched = true;
  c->occ_uploaded = false;
}

// Drawn warm-up points -> device on the copy stream (non-blocking unless `block`).  The copy
// waits for the previous update's queries to be done with the device buffer.
int occ_try_upload(dg_ctx* c, bool block) {
  if (c->occ_uploaded || !c->occ_prefetched || !c->occ_prefetch.valid()) return DG_OK;
  if (!block && c->occ_prefetch.wait_for(std::chrono::seconds(0)) != std::future_status::ready)
    return DG_OK;
  c->occ_prefetch.wait();
  CU(cudaStreamWaitEvent(c->stream_copy, c->ev_occ_used, 0));
  CU(cudaMemcpyAsync(c->occ_pts_warm.p, c->occ_host, c->occ_host_n * sizeof(double),
                     cudaMemcpyHostToDevice, c->stream_copy));
  CU(cudaEventRecord(c->ev_occ_up, c->stream_copy));
  c->h2d += c->occ_host_n * sizeof(double);
  c->occ_uploaded = true;
  return DG_OK;
}

// Worker::update_occupancy (worker.cpp:549-562) + OccupancyGrid::decay_and_update
// (grid.cpp:201-229).  The jitter points are the reference's mt19937_64 draws in its order
// (fine grid, then coarse grid, same stream); sigma is evaluated on the device.
int order_after_adam(dg_ctx* c);

int occupancy_update(dg_ctx* c) {
  const dg_run_config& cfg = c->cfg;
  const uint64_t step = c->worker_step;
  if (!cfg.occupancy_updates || step == 0 || cfg.occ_update_interval == 0 ||
      step % cfg.occ_update_interval != 0)
    return DG_OK;
  cudaStream_t s = c->stream;
  TRY(order_after_adam(c));  // the density query reads the updated parameters
  const double threshold =
      (step < cfg.occ_threshold_switch_step ? cfg.occ_threshold_early : cfg.occ_threshold_late) *
      cfg.occ_threshold_scale;
  const bool warm_up = step <= cfg.occ_warmup_steps;
  const uint32_t nl = uint32_t(c->local.size());
  if (warm_up) {
    if (!c->occ_prefetched) {  // nothing drawn ahead (e.g. state just injected): draw now
      c->occ_rng_before = c->occ_rng;
      c->occ_prefetch = std::async(std::launch::deferred, [c] { occ_generate_warm(c); });
      c->occ_prefetched = true;
      c->occ_uploaded = false;
    }
    TRY(occ_try_upload(c, true));
    CU(cudaStreamWaitEvent(s, c->ev_occ_up, 0));
  }
  uint64_t k = 0;  // offset into the prefetched warm-up points
  for (uint32_t lp = 0; lp < nl; ++lp) {
    const PartDesc& pd = c->parts[lp];
    for (int casc = 0; casc < 2; ++casc) {  // set_threshold: recompute the bitfield
      c->occ_thr[lp * 2 + casc] = threshold;
      launch_occ_bits(c->occ_den.as<float>() + pd.den_off[casc], c->occ.as<uint8_t>() + pd.occ_off[casc],
                      pd.occ_n[casc], float(threshold), s);
      ++c->launches;
    }
    for (int casc = 0; casc < 2; ++casc) {
      const double* lo;
      double cell[3];
      uint64_t total;
      occ_geometry(pd, casc, lo, cell, total);
      const FieldDesc* fd = c->d_fields.as<FieldDesc>() + casc * nl + lp;
      float* den = c->occ_den.as<float>() + pd.den_off[casc];
      if (warm_up) {  // every cell once, in order: cell index == point index
        c->launches += launch_occ_query(fd, c->params.as<float>(), c->occ_pts_warm.as<double>() + k, total,
                                        c->occ_sigma.as<float>(), s);
        k += 3 * total;
        launch_occ_apply(den, nullptr, c->occ_sigma.as<float>(), total, float(cfg.occ_decay), s);
      } else {
        std::mt19937_64& rng = c->occ_rng[lp];
        // occupied cells = the bitfield just recomputed (density >= threshold, k_occ_bits)
        std::vector<float> hd(total);
        CU(cudaMemcpyAsync(hd.data(), den, total * sizeof(float), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        std::vector<uint64_t> occupied;
        for (uint64_t i = 0; i < total; ++i)
          if (hd[i] >= float(threshold)) occupied.push_back(i);
        const uint64_t n_uniform = std::max<uint64_t>(total / 4, 1);
        std::vector<uint32_t> cells;
        std::vector<double> pts;
        auto sample = [&](uint64_t idx) {
          cells.push_back(uint32_t(idx));
          pts.resize(pts.size() + 3);
          occ_point(rng, lo, cell, pd.occ_n[casc], idx, pts.data() + pts.size() - 3);
        };
        for (uint64_t i = 0; i < n_uniform; ++i) sample(rng() % total);
        if (!occupied.empty())
          for (uint64_t i = 0; i < n_uniform; ++i) sample(occupied[rng() % occupied.size()]);
        const uint64_t n = cells.size();
        CU(cudaMemcpyAsync(c->occ_pts.p, pts.data(), pts.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        c->launches += launch_occ_query(fd, c->params.as<float>(), c->occ_pts.as<double>(), n,
                                        c->occ_sigma.as<float>(), s);
        // cells may repeat: apply sequentially in draw order on the host
        std::vector<float> sig(n);
        CU(cudaMemcpyAsync(sig.data(), c->occ_sigma.p, n * sizeof(float), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        for (uint64_t q = 0; q < n; ++q) hd[cells[q]] = std::max(hd[cells[q]] * float(cfg.occ_decay), sig[q]);
        CU(cudaMemcpyAsync(den, hd.data(), total * sizeof(float), cudaMemcpyHostToDevice, s));
        CU(cudaStreamSynchronize(s));
        c->h2d += pts.size() * sizeof(double) + total * sizeof(float);
      }
      launch_occ_bits(den, c->occ.as<uint8_t>() + pd.occ_off[casc], pd.occ_n[casc], float(threshold), s);
      c->launches += warm_up ? 2 : 1;  // (apply +) bits
    }
  }
  ++c->occ_updates;
  if (warm_up) {
    CU(cudaEventRecord(c->ev_occ_used, s));
    CU(cudaEventSynchronize(c->ev_occ_up));  // the pinned buffer is reused by the next prefetch
    c->occ_prefetched = c->occ_uploaded = false;
    occ_start_prefetch(c);
  }
  return DG_OK;
}

// The context stream after the last step's asynchronous Adam update (no host wait).
int order_after_adam(dg_ctx* c) {
  if (!c->adam_pending) return DG_OK;
  CU(cudaStreamWaitEvent(c->stream, c->ev_adam, 0));
  c->adam_pending = false;
  return DG_OK;
}

// Every API entry but dg_train_step's front half: argument check + ordering after the last
// step's Adam (parameters, gradients and moments are final for the caller).
int check_ctx(const dg_ctx* cc) {
  if (!cc) return set_err(DG_EINVAL, "null context");
  return order_after_adam(const_cast<dg_ctx*>(cc));
}

int check_part(const dg_ctx* c, uint32_t partition, uint32_t* lp) {
  TRY(check_ctx(c));
  if (partition >= c->P) return set_err(DG_ERANGE, "partition %u out of range", partition);
  if (c->local_of_global[partition] == 0xff)
    return set_err(DG_EINVAL, "partition %u is not owned by rank %d", partition, c->rank);
  *lp = c->local_of_global[partition];
  return DG_OK;
}

}  // namespace

// =============================================================================== C ABI
extern "C" {

const char* dg_last_error(void) { return g_err.c_str(); }
int dg_abi_version(void) { return DG_ABI_VERSION; }

void dg_default_config(dg_run_config* c) {
  std::memset(c, 0, sizeof *c);
  for (int a = 0; a < 3; ++a) {
    c->inner_lo[a] = c->outer_lo[a] = 0.0;
    c->inner_hi[a] = c->outer_hi[a] = 1.0;
  }
  c->kx = c->ky = 1;
  c->grid_levels = 8;
  c->grid_features = 2;
  c->base_resolution = 16;
  c->max_resolution = 512;
  c->fine_table_log2 = 15;
  c->coarse_table_log2 = 12;
  c->appearance_dim = 16;
  c->march_step_divisor = 1024.0;
  c->occ_resolution = 128;
  c->occ_decay = 0.99;
  c->occ_warmup_steps = 4096;
  c->occ_update_interval = 16;
  c->occ_threshold_early = 0.6;
  c->occ_threshold_late = 60.0;
  c->occ_threshold_switch_step = 10000;
  c->occ_threshold_scale = 1.0;
  c->seed = 1;
  c->total_steps = 20000;
  c->lr_start = 0.05;
  c->lr_end = 0.005;
  c->lambda_transmittance = 1e-3;
  c->lambda_distortion = 1e-3;
  c->transmittance_clamp = 1e-6;
  c->adam_beta1 = 0.9;
  c->adam_beta2 = 0.99;
  c->adam_eps = 1e-15;
  c->occupancy_updates = 1;
  c->eval_early_termination = 0;          // config.hpp:60-61
  c->eval_termination_threshold = 1e-4;
}

double dg_lr_at(const dg_run_config* cfg, uint64_t step) {  // train.cpp:77-80
  const double progress = cfg->total_steps == 0 ? 1.0 : double(step) / double(cfg->total_steps);
  return cfg->lr_end + 0.5 * (cfg->lr_start - cfg->lr_end) * (1.0 + std::cos(M_PI * progress));
}

int dg_ctx_create(const dg_run_config* cfg, int device, int rank, int world, dg_ctx** out) {
  if (!cfg || !out) return set_err(DG_EINVAL, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return set_err(DG_EINVAL, "bad rank/world");
  auto c = std::make_unique<dg_ctx>();
  c->cfg = *cfg;
  c->rank = rank;
  c->world = world;
  if (device < 0) CU(cudaGetDevice(&device));
  c->device = device;
  CU(cudaSetDevice(device));
  CU(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  TRY(ctx_setup(c.get()));
  if (const char* e = std::getenv("DG_MLP")) c->mlp_impl = std::strcmp(e, "ffma") == 0 ? 0 : 1;
  if (const char* e = std::getenv("DG_ENC_FWD_MB"))
    c->enc_budget_fwd = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10)) << 20;
  if (const char* e = std::getenv("DG_ENC_PCACHE")) c->enc_pcache = std::strcmp(e, "0") != 0;
  if (const char* e = std::getenv("DG_SAMPLE_ORDER")) c->sample_order = std::atoi(e);
  if (const char* e = std::getenv("DG_ORDER_CHUNK")) c->order_chunk = std::min(64u, std::max(1u, uint32_t(std::atoi(e))));
  if (const char* e = std::getenv("DG_ORDER_BITS")) c->order_bits = std::min(10u, std::max(1u, uint32_t(std::atoi(e))));
  if (const char* e = std::getenv("DG_ENC_BWD_STRIDE")) c->bwd_cta_mul = uint32_t(std::strtoul(e, nullptr, 10));
  if (const char* e = std::getenv("DG_MLP_BWD_SERIAL")) c->mlp_bwd_paired = std::strcmp(e, "0") == 0;
  if (const char* e = std::getenv("DG_MLP_ISSUE_WARP")) c->mlp_issue_warp = uint32_t(std::strtoul(e, nullptr, 10)) % 16u;
  if (const char* e = std::getenv("DG_MLP_FWD_ISSUE_WARP")) c->mlp_issue_warp_fwd = uint32_t(std::strtoul(e, nullptr, 10)) % 8u;
  if (const char* e = std::getenv("DG_ENC_AGG")) c->enc_agg_samples_per_cell = std::max(0.01, std::atof(e));
  if (const char* e = std::getenv("DG_ENC_BWD_MB"))
    c->enc_budget_bwd = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10)) << 20;
  if (const char* e = std::getenv("DG_ENC_FWD_GROUP_MB")) c->enc_group_fwd = std::strtoull(e, nullptr, 10) << 20;
  if (const char* e = std::getenv("DG_ENC_FWD_HGROUP_MB")) c->enc_hgroup_fwd = std::strtoull(e, nullptr, 10) << 20;
  if (const char* e = std::getenv("DG_ENC_BWD_HGROUP_MB")) c->enc_hgroup_bwd = std::strtoull(e, nullptr, 10) << 20;
  if (const char* e = std::getenv("DG_ENC_BWD_GROUP_MB")) c->enc_group_bwd = std::strtoull(e, nullptr, 10) << 20;
  // the step stream at the highest priority, the side-stream Adam at the lowest: the next
  // step's front half takes SMs ahead of the update's remaining CTAs
  int prio_lo = 0, prio_hi = 0;
  CU(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CU(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi));
  c->own_stream = c->stream;
  CU(cudaStreamCreateWithFlags(&c->stream_copy, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithPriority(&c->stream_adam, cudaStreamNonBlocking, prio_lo));
  if (const char* e = std::getenv("DG_ADAM_SPREAD")) c->adam_spread = std::strcmp(e, "0") != 0;
  CU(cudaEventCreateWithFlags(&c->ev_grads, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&c->ev_adam, cudaEventDisableTiming));
  c->pin_cap = 1 << 20;
  CU(cudaHostAlloc(reinterpret_cast<void**>(&c->pin), c->pin_cap, cudaHostAllocDefault));
  CU(cudaEventCreateWithFlags(&c->ev_occ_up, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&c->ev_occ_used, cudaEventDisableTiming));
  for (auto& e : c->ev) CU(cudaEventCreate(&e));
  TRY(ctx_alloc(c.get()));
  *out = c.release();
  return DG_OK;
}

int dg_ctx_destroy(dg_ctx* c) {
  if (!c) return DG_OK;
  cudaSetDevice(c->device);
  if (c->occ_prefetch.valid()) c->occ_prefetch.wait();
  if (c->occ_host) cudaFreeHost(c->occ_host);
  if (c->pin) cudaFreeHost(c->pin);
  cudaStreamSynchronize(c->stream);
  if (c->stream_copy) cudaStreamSynchronize(c->stream_copy);
  if (c->stream_adam) cudaStreamSynchronize(c->stream_adam);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->ev_occ_up) cudaEventDestroy(c->ev_occ_up);
  if (c->ev_occ_used) cudaEventDestroy(c->ev_occ_used);
  if (c->ev_grads) cudaEventDestroy(c->ev_grads);
  if (c->ev_adam) cudaEventDestroy(c->ev_adam);
  cudaStream_t s = c->own_stream, sc = c->stream_copy, sa = c->stream_adam;
  delete c;
  if (s) cudaStreamDestroy(s);
  if (sc) cudaStreamDestroy(sc);
  if (sa) cudaStreamDestroy(sa);
  return DG_OK;
}

int dg_partition_count(const dg_ctx* c, uint32_t* n_total, uint32_t* n_local) {
  TRY(check_ctx(c));
  if (n_total) *n_total = c->P;
  if (n_local) *n_local = uint32_t(c->local.size());
  return DG_OK;
}

int dg_partition_rank(const dg_ctx* c, uint32_t p, int* rank) {
  TRY(check_ctx(c));
  if (p >= c->P) return set_err(DG_ERANGE, "partition out of range");
  *rank = c->part_rank[p];
  return DG_OK;
}

int dg_march_step(const dg_ctx* c, double* step) {
  TRY(check_ctx(c));
  *step = c->step;
  return DG_OK;
}

int dg_region_boxes(const dg_ctx* c, uint32_t p, double fl[3], double fh[3], double cl[3], double ch[3]) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  const PartDesc& pd = c->parts[lp];
  for (int a = 0; a < 3; ++a) {
    fl[a] = pd.fine_lo[a];
    fh[a] = pd.fine_hi[a];
    cl[a] = pd.coarse_lo[a];
    ch[a] = pd.coarse_hi[a];
  }
  return DG_OK;
}

int dg_grid_levels(const dg_ctx* c, uint32_t p, uint32_t cascade, uint32_t* shapes, uint32_t* modes,
                   uint64_t* rows) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (cascade > 1) return set_err(DG_EINVAL, "cascade must be 0 or 1");
  const FieldDesc& fd = c->fields[cascade * c->local.size() + lp];
  for (uint32_t l = 0; l < fd.L; ++l) {
    for (int a = 0; a < 3; ++a) shapes[3 * l + a] = fd.lv[l].n[a];
    if (modes) modes[l] = fd.lv[l].hashed;
    if (rows) rows[l] = fd.lv[l].hashed ? uint64_t(fd.lv[l].mask) + 1
                                        : uint64_t(fd.lv[l].n[0]) * fd.lv[l].n[1] * fd.lv[l].n[2];
  }
  return DG_OK;
}

int dg_param_count(const dg_ctx* c, uint32_t p, uint64_t* n) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  *n = c->part_param_cnt[lp];
  return DG_OK;
}

int dg_param_layout(const dg_ctx* c, uint32_t p, dg_array_desc* arrays, uint32_t capacity, uint32_t* n) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  const auto& L = c->layouts[lp];
  *n = uint32_t(L.size());
  for (uint32_t i = 0; i < L.size() && i < capacity; ++i) arrays[i] = L[i];
  return DG_OK;
}

// Flat (reference-order, fine then coarse) <-> device layout (each field 16-byte aligned).
static int copy_part(dg_ctx* c, uint32_t p, DBuf& buf, float* host, const float* in) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  const size_t nl = c->local.size();
  uint64_t flat = 0;
  for (int casc = 0; casc < 2; ++casc) {
    float* dev = buf.as<float>() + c->field_dev_off[casc * nl + lp];
    for (const dg_ctx::Seg& g : c->field_segs[casc * nl + lp]) {
      const size_t bytes = g.count * sizeof(float);
      if (in) CU(cudaMemcpyAsync(dev + g.dev, in + flat + g.flat, bytes, cudaMemcpyHostToDevice, c->stream));
      else CU(cudaMemcpyAsync(host + flat + g.flat, dev + g.dev, bytes, cudaMemcpyDeviceToHost, c->stream));
    }
    flat += c->field_size[casc * nl + lp];
  }
  CU(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

int dg_set_params(dg_ctx* c, uint32_t p, const float* in) { return copy_part(c, p, c->params, nullptr, in); }
int dg_get_params(dg_ctx* c, uint32_t p, float* out) { return copy_part(c, p, c->params, out, nullptr); }
int dg_get_grads(dg_ctx* c, uint32_t p, float* out) { return copy_part(c, p, c->grads, out, nullptr); }

int dg_zero_grads(dg_ctx* c) {
  TRY(check_ctx(c));
  CU(cudaMemsetAsync(c->grads.p, 0, c->n_params * sizeof(float), c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

int dg_set_adam(dg_ctx* c, uint32_t p, const float* m, const float* v, uint64_t t) {
  TRY(copy_part(c, p, c->adam_m, nullptr, m));
  TRY(copy_part(c, p, c->adam_v, nullptr, v));
  c->adam_t = t;
  return DG_OK;
}

int dg_get_adam(dg_ctx* c, uint32_t p, float* m, float* v, uint64_t* t) {
  TRY(copy_part(c, p, c->adam_m, m, nullptr));
  TRY(copy_part(c, p, c->adam_v, v, nullptr));
  if (t) *t = c->adam_t;
  return DG_OK;
}

int dg_set_step(dg_ctx* c, uint64_t step) {
  TRY(check_ctx(c));
  if (c->occ_prefetched) {
    // undo the draws of a prefetch made for the old step: wait for the drawing thread and the
    // upload that reads its pinned buffer, then rewind the stream to before it
    if (c->occ_prefetch.valid()) c->occ_prefetch.wait();
    if (c->occ_uploaded) CU(cudaEventSynchronize(c->ev_occ_up));
    c->occ_rng = c->occ_rng_before;
    c->occ_prefetched = c->occ_uploaded = false;
  }
  c->worker_step = step;
  occ_start_prefetch(c);
  return DG_OK;
}

int dg_get_step(const dg_ctx* c, uint64_t* step) {
  TRY(check_ctx(c));
  *step = c->worker_step;
  return DG_OK;
}

// Device-side copy of everything a training step mutates (parameters, Adam moments and t,
// occupancy bitfields / densities / thresholds / sampling stream, the step counter), so a
// window of steps can be replayed from the same state (e.g. bench.py's end-to-end pass).
int dg_state_snapshot(dg_ctx* c, int restore) {
  TRY(check_ctx(c));
  CU(cudaSetDevice(c->device));
  dg_ctx::Snapshot& sn = c->snap;
  const size_t pb = std::max<uint64_t>(c->n_params, 4) * sizeof(float);
  const size_t ob = c->occ_bytes, db = c->occ_den_n * sizeof(float);
  struct Pair {
    DBuf* live;
    DBuf* copy;
    size_t bytes;
  } pairs[] = {{&c->params, &sn.params, pb}, {&c->adam_m, &sn.m, pb}, {&c->adam_v, &sn.v, pb},
               {&c->occ, &sn.occ, ob}, {&c->occ_den, &sn.occ_den, db}};
  TRY(step_sync(c));
  if (c->occ_prefetch.valid()) c->occ_prefetch.wait();
  if (c->occ_uploaded) CU(cudaEventSynchronize(c->ev_occ_up));
  if (!restore) {
    for (Pair& p : pairs) {
      TRY(p.copy->ensure(p.bytes));
      CU(cudaMemcpyAsync(p.copy->p, p.live->p, p.bytes, cudaMemcpyDeviceToDevice, c->stream));
    }
    sn.occ_thr = c->occ_thr;
    sn.occ_rng = c->occ_prefetched ? c->occ_rng_before : c->occ_rng;
    sn.adam_t = c->adam_t;
    sn.worker_step = c->worker_step;
    sn.valid = true;
  } else {
    if (!sn.valid) return set_err(DG_EINVAL, "no snapshot taken");
    for (Pair& p : pairs)
      CU(cudaMemcpyAsync(p.live->p, p.copy->p, p.bytes, cudaMemcpyDeviceToDevice, c->stream));
    CU(cudaMemsetAsync(c->grads.p, 0, pb, c->stream));
    c->occ_thr = sn.occ_thr;
    c->occ_rng = sn.occ_rng;
    c->adam_t = sn.adam_t;
    c->worker_step = sn.worker_step;
    c->occ_prefetched = c->occ_uploaded = false;
    occ_start_prefetch(c);
  }
  CU(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

// worker.cpp:186-190: Rng(counter_hash(seed, 0xf1e1d|0xc0a45e, region)); grid levels in order
// (uniform[-1e-4,1e-4]), then each MLP layer's weights (Xavier bound), biases zero.
int dg_init_params_reference(dg_ctx* c, uint32_t p) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  std::vector<float> host(c->part_param_cnt[lp], 0.0f);
  for (int casc = 0; casc < 2; ++casc) {
    const uint64_t salt = casc == 0 ? 0xf1e1dull : 0xc0a45eull;
    std::mt19937_64 eng(splitmix64(counter_hash(c->cfg.seed, salt, p, 0)));
    auto uni = [&](double lo, double hi) {
      return lo + (hi - lo) * (double(eng() >> 11) * 0x1.0p-53);
    };
    const FieldDesc& fd = c->fields[casc * c->local.size() + lp];
    // flat offsets of this field's arrays (dg_array_desc: kind 0 = level table, 1/3 = weights)
    auto flat_of = [&](uint32_t kind, uint32_t idx) -> uint64_t {
      for (const dg_array_desc& a : c->layouts[lp])
        if (a.cascade == uint32_t(casc) && a.kind == kind && a.index == idx) return a.offset;
      return 0;
    };
    for (uint32_t l = 0; l < fd.L; ++l) {
      const uint64_t off = flat_of(0, l), rows = fd.lv[l].rows;
      for (uint64_t k = 0; k < rows * 2; ++k) host[off + k] = float(uni(-1e-4, 1e-4));
    }
    const uint32_t enc = fd.L * 2, cin = 31 + fd.app_dim;
    struct L3 {
      uint64_t off;
      uint32_t in, out;
    } layers[] = {{flat_of(1, 0), enc, 64}, {flat_of(1, 1), 64, 16}, {flat_of(3, 0), cin, 64},
                  {flat_of(3, 1), 64, 64}, {flat_of(3, 2), 64, 3}};
    for (const L3& L : layers) {
      const double bound = std::sqrt(6.0 / double(L.in + L.out));
      for (uint64_t k = 0; k < uint64_t(L.in) * L.out; ++k) host[L.off + k] = float(uni(-bound, bound));
    }
  }
  return dg_set_params(c, p, host.data());
}

int dg_init_params_fast(dg_ctx* c, uint32_t p, uint64_t seed) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  float* base = c->params.as<float>();
  for (int casc = 0; casc < 2; ++casc) {
    const FieldDesc& fd = c->fields[casc * c->local.size() + lp];
    const uint64_t grid_floats = fd.dw0;
    launch_fill_uniform(base + fd.base, grid_floats, -1e-4f, 1e-4f, counter_hash(seed, p, casc, 1), c->stream);
    const uint32_t enc = fd.L * 2, cin = 31 + fd.app_dim;
    struct L3 {
      uint64_t w, b;
      uint32_t in, out;
    } layers[] = {{fd.dw0, fd.db0, enc, 64}, {fd.dw1, fd.db1, 64, 16}, {fd.cw0, fd.cb0, cin, 64},
                  {fd.cw1, fd.cb1, 64, 64}, {fd.cw2, fd.cb2, 64, 3}};
    int li = 0;
    for (const L3& L : layers) {
      const float bound = float(std::sqrt(6.0 / double(L.in + L.out)));
      launch_fill_uniform(base + fd.base + L.w, uint64_t(L.in) * L.out, -bound, bound,
                          counter_hash(seed, p, casc, 100 + li++), c->stream);
      CU(cudaMemsetAsync(base + fd.base + L.b, 0, L.out * sizeof(float), c->stream));
    }
  }
  c->launches += 12;
  CU(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

int dg_occupancy_shape(const dg_ctx* c, uint32_t p, uint32_t cascade, uint32_t shape[3]) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (cascade > 1) return set_err(DG_EINVAL, "cascade must be 0 or 1");
  for (int a = 0; a < 3; ++a) shape[a] = c->parts[lp].occ_n[cascade][a];
  return DG_OK;
}

static int occ_copy(dg_ctx* c, uint32_t p, uint32_t cascade, uint8_t* out, const uint8_t* in) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (cascade > 1) return set_err(DG_EINVAL, "cascade must be 0 or 1");
  const PartDesc& pd = c->parts[lp];
  const uint32_t* sh = pd.occ_n[cascade];
  const uint32_t* nb = pd.occ_nb[cascade];
  const uint64_t bytes = uint64_t(nb[0]) * nb[1] * nb[2] * (kOccBX * kOccBY * kOccBZ);
  uint8_t* dev = c->occ.as<uint8_t>() + pd.occ_off[cascade];
  std::vector<uint8_t> br(bytes, 1);  // bricked image (padding cells stay occupied, never walked)
  if (in) {
    for (uint32_t z = 0; z < sh[2]; ++z)
      for (uint32_t y = 0; y < sh[1]; ++y)
        for (uint32_t x = 0; x < sh[0]; ++x) br[occ_addr(nb, x, y, z)] = in[(uint64_t(z) * sh[1] + y) * sh[0] + x];
    CU(cudaMemcpyAsync(dev, br.data(), bytes, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  } else {
    CU(cudaMemcpyAsync(br.data(), dev, bytes, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    for (uint32_t z = 0; z < sh[2]; ++z)
      for (uint32_t y = 0; y < sh[1]; ++y)
        for (uint32_t x = 0; x < sh[0]; ++x) out[(uint64_t(z) * sh[1] + y) * sh[0] + x] = br[occ_addr(nb, x, y, z)];
  }
  return DG_OK;
}

int dg_set_occupancy(dg_ctx* c, uint32_t p, uint32_t cascade, const uint8_t* bits) {
  TRY(occ_copy(c, p, cascade, nullptr, bits));
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  // density := threshold where occupied, 0 elsewhere (as OccupancyGrid::recompute_bitfield sees it)
  const PartDesc& pd = c->parts[lp];
  const uint64_t n = uint64_t(pd.occ_n[cascade][0]) * pd.occ_n[cascade][1] * pd.occ_n[cascade][2];
  const float thr = float(c->occ_thr[lp * 2 + cascade]);
  std::vector<float> den(n);
  for (uint64_t i = 0; i < n; ++i) den[i] = bits[i] ? thr : 0.0f;
  CU(cudaMemcpyAsync(c->occ_den.as<float>() + pd.den_off[cascade], den.data(), n * sizeof(float),
                     cudaMemcpyHostToDevice, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return DG_OK;
}
int dg_get_occupancy(dg_ctx* c, uint32_t p, uint32_t cascade, uint8_t* bits) {
  return occ_copy(c, p, cascade, bits, nullptr);
}

// OccupancyGrid density + threshold (grid.hpp:99-141); the set variant recomputes the
// bitfield (recompute_bitfield: density >= threshold) on the device.
int dg_get_occupancy_density(dg_ctx* c, uint32_t p, uint32_t cascade, float* density, double* threshold) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (cascade > 1) return set_err(DG_EINVAL, "cascade must be 0 or 1");
  CU(cudaSetDevice(c->device));
  const PartDesc& pd = c->parts[lp];
  const uint64_t n = uint64_t(pd.occ_n[cascade][0]) * pd.occ_n[cascade][1] * pd.occ_n[cascade][2];
  if (density)
    CU(cudaMemcpyAsync(density, c->occ_den.as<float>() + pd.den_off[cascade], n * sizeof(float),
                       cudaMemcpyDeviceToHost, c->stream));
  if (threshold) *threshold = c->occ_thr[lp * 2 + cascade];
  CU(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

int dg_set_occupancy_density(dg_ctx* c, uint32_t p, uint32_t cascade, const float* density, double threshold) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (cascade > 1 || !density) return set_err(DG_EINVAL, "cascade must be 0 or 1, density non-null");
  CU(cudaSetDevice(c->device));
  const PartDesc& pd = c->parts[lp];
  const uint64_t n = uint64_t(pd.occ_n[cascade][0]) * pd.occ_n[cascade][1] * pd.occ_n[cascade][2];
  CU(cudaMemcpyAsync(c->occ_den.as<float>() + pd.den_off[cascade], density, n * sizeof(float),
                     cudaMemcpyHostToDevice, c->stream));
  c->occ_thr[lp * 2 + cascade] = threshold;
  launch_occ_bits(c->occ_den.as<float>() + pd.den_off[cascade], c->occ.as<uint8_t>() + pd.occ_off[cascade],
                  pd.occ_n[cascade], float(threshold), c->stream);
  ++c->launches;
  CU(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

int dg_get_config(const dg_ctx* c, dg_run_config* out) {
  TRY(check_ctx(c));
  if (!out) return set_err(DG_EINVAL, "null config");
  *out = c->cfg;
  return DG_OK;
}

int dg_set_appearance(dg_ctx* c, const uint32_t* ids, const float* rows, uint32_t n) {
  TRY(check_ctx(c));
  uint32_t max_id = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (ids[i] >= (1u << 20)) return set_err(DG_ERANGE, "appearance: image id >= 2^20");
    max_id = std::max(max_id, ids[i]);
  }
  const uint32_t d = c->cfg.appearance_dim;
  const uint32_t nrows = n ? max_id + 1 : 1;
  std::vector<float> table(uint64_t(nrows) * d + 16, 0.0f);
  for (uint32_t i = 0; i < n; ++i)
    std::memcpy(&table[uint64_t(ids[i]) * d], rows + uint64_t(i) * d, d * sizeof(float));
  TRY(upload(c->app, table.data(), table.size() * sizeof(float), c->stream));
  CU(cudaStreamSynchronize(c->stream));
  c->app_rows = n ? nrows : 0;  // ids with no row are rejected in the step (DG_ERANGE)
  c->n_images = n;
  return DG_OK;
}

int dg_train_step(dg_ctx* c, const dg_ray_batch* b, uint64_t step, dg_step_stats* stats) {
  if (!c) return set_err(DG_EINVAL, "null context");  // no Adam ordering yet: the front half
                                                      // overlaps the previous step's update
  if (!b) return set_err(DG_EINVAL, "null batch");
  if (b->n && (!b->origin || !b->dir || !b->color_gt)) return set_err(DG_EINVAL, "batch: missing arrays");
  if (b->n >= (1ull << 32) || b->first_ray_id + b->n > (1ull << 32))
    return set_err(DG_EINVAL, "batch: ray ids must fit in 32 bits");
  if (c->world > 1 && !c->comm) return set_err(DG_EINVAL, "world > 1 needs dg_comm_init_*");
  CU(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const uint32_t P = c->P, nl = uint32_t(c->local.size());
  uint64_t dropped = 0, bytes = 0;
  c->h2d = c->d2h = 0;
  TRY(pin_reset(c));
  c->cross_active = c->cfg.distortion_cross_correction != 0;
  TRY(occ_try_upload(c, false));
  TRY(front_half(c, b, 1, step, &dropped, &bytes));
  const uint64_t bytes_x1 = bytes;
  const uint32_t NI = c->n_items;
  ItemArrays it = item_arrays(c);
  SampleArrays sm = sample_arrays(c);
  // pair counts for exchange 2 (P > 1)
  std::vector<uint32_t> pair_cnt(uint64_t(nl) * P, 0);
  uint32_t* pair_pin = nullptr;
  if (P > 1 && NI) {
    TRY(c->small.ensure(uint64_t(nl) * P * 4 + 16));
    launch_pair_counts(NI, nl, P, c->part_item_off_d.as<uint32_t>(), nullptr,
                       c->it_cscan.as<uint32_t>(), c->small.as<uint32_t>(), s);
    ++c->launches;
    pair_pin = pin_slot<uint32_t>(c, pair_cnt.size());
    CU(cudaMemcpyAsync(pair_pin ? pair_pin : pair_cnt.data(), c->small.p, pair_cnt.size() * 4,
                       cudaMemcpyDeviceToHost, s));
    c->d2h += pair_cnt.size() * 4;
  }
  CU(cudaMemsetAsync(c->loss.p, 0, sizeof(LossAccum), s));
  // K3 / K4 forward (from here on the parameters are read: after the previous step's Adam)
  {
    TRY(order_after_adam(c));
    TRY(pairs_expand(c, s));
    std::vector<EncPass> passes;
    const FieldLaunch fl = field_launch(c, c->enc_budget_fwd, passes, c->enc_group_fwd, c->enc_hgroup_fwd);
    c->launches += launch_encode_fwd(fl, passes, sm.X, s) - 1;
  }
  mark(c, 3);
  MlpLaunch mf = mlp_launch(c, false);
  if (c->mlp_impl) {
    // the backward reads the forward's outputs by tile row (colour-head adjoint, sigma path)
    if (c->ordered) TRY(c->s_out_ord.ensure((uint64_t(c->n_fine) + c->n_coarse) * 16 + 16));
    mf.out_tile = c->ordered ? c->s_out_ord.as<float4>() : mf.out;
    launch_mlp_fwd_tc(mf, c->num_sms, s);
  }
  else launch_mlp_fwd(mf, s);
  mark(c, 4);
  launch_composite(NI, it, sm, c->n_fine, 0, s);
  mark(c, 5);
  c->launches += 3;
  // X2: partial exchange (alias on a single rank)
  if (P > 1) {
    TRY(step_sync(c));  // pair counts on the host
    if (pair_pin) std::memcpy(pair_cnt.data(), pair_pin, pair_cnt.size() * 4);
  }
  const PartialRec* recv = c->send_buf.as<PartialRec>();
  const float4* recv_x = nullptr;
  if (P > 1) {
    TRY(exchange_partials(c, pair_cnt, &bytes, &recv, &recv_x));
  } else {
    TRY(c->stream_recv_d.ensure(16));
  }
  mark(c, 6);
  // K5b merge / losses / composite backward
  launch_merge_backward(NI, it, c->part_item_off_d.as<uint32_t>(), c->d_parts.as<PartDesc>(),
                        P > 1 ? c->stream_recv_d.as<uint64_t>() : nullptr, P, recv, recv_x, sm,
                        c->n_fine, c->cfg.lambda_transmittance, c->cfg.lambda_distortion,
                        c->cfg.transmittance_clamp, int(c->cfg.wire_f32), c->loss.as<LossAccum>(), s);
  mark(c, 7);
  // K4b / K3b backward
  if (c->mlp_impl) {
    MlpLaunch mb = mlp_launch(c, false);  // 128-sample tiles
    mb.out_tile = c->ordered ? c->s_out_ord.as<float4>() : mb.out;
    launch_mlp_bwd_tc(mb, c->num_sms, s);
  } else {
    launch_mlp_bwd(mlp_launch(c, true), c->num_sms, s);
  }
  mark(c, 8);
  {
    std::vector<EncPass> passes;
    FieldLaunch fl = field_launch(c, c->enc_budget_bwd, passes, c->enc_group_bwd, c->enc_hgroup_bwd);
    if (c->ordered && c->bwd_cta_mul) {  // a CTA stride coprime with the CTA count along x
      uint64_t nb = 0;
      for (const EncPass& p : passes)
        nb = std::max<uint64_t>(nb, p.f == kAllFields ? fl.n_total : fl.field_off[p.f + 1] - fl.field_off[p.f]);
      nb = (nb + 255) / 256;
      uint64_t m = c->bwd_cta_mul % std::max<uint64_t>(nb, 1);
      if (m == 0) m = 1;
      while (nb > 1 && std::gcd(m, nb) != 1) ++m;
      fl.cta_mul = uint32_t(m);
    }
    c->launches += launch_encode_bwd(fl, passes, sm.dX, s) - 1;
    if (c->pair_rows) {  // the paired one-to-one levels' gradients into the tables
      launch_pairs_fold(c->pair_segs_d.as<PairSeg>(), uint32_t(c->pair_segs.size()), c->pair_rows,
                        c->pgrads.as<float4>(), c->grads.as<float>(), s);
      ++c->launches;
    }
  }
  mark(c, 9);
  c->launches += 3;
  // K6 Adam over every local parameter, lr at the pre-increment step (worker.cpp:544)
  const double lr = dg_lr_at(&c->cfg, c->worker_step);
  const double bias1 = 1.0 - std::pow(c->cfg.adam_beta1, double(c->adam_t + 1));
  const double bias2 = 1.0 - std::pow(c->cfg.adam_beta2, double(c->adam_t + 1));
  // k_adam skips the update (and discards the gradients) when the merge flagged a missing
  // partial, so an aborted step leaves params, moments, t and the step counter untouched
  // (the reference throws before apply_updates, worker.cpp:371-380)
  // on the Adam stream: the call returns once the losses are read, and the next step's front
  // half (no parameter access) runs under the update
  // Adam reads its own copy of the error word: the next step clears the loss accumulator
  // while this update may still be queued
  TRY(c->adam_flag.ensure(16));
  CU(cudaMemcpyAsync(c->adam_flag.p, &c->loss.as<LossAccum>()->error, sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                     s));
  CU(cudaEventRecord(c->ev_grads, s));
  CU(cudaStreamWaitEvent(c->stream_adam, c->ev_grads, 0));
  launch_adam(c->params.as<float>(), c->grads.as<float>(), c->adam_m.as<float>(), c->adam_v.as<float>(),
              c->n_params, float(lr), float(c->cfg.adam_beta1), float(c->cfg.adam_beta2),
              float(c->cfg.adam_eps), float(1.0 / bias1), float(1.0 / bias2), c->stream_adam,
              c->adam_flag.as<uint32_t>(), 2u, c->adam_spread);
  ++c->launches;
  if (c->timing) cudaEventRecord(c->ev[10], c->stream_adam);
  CU(cudaEventRecord(c->ev_adam, c->stream_adam));
  c->adam_pending = true;
  LossAccum la;
  LossAccum* la_pin = pin_slot<LossAccum>(c, 1);
  CU(cudaMemcpyAsync(la_pin ? la_pin : &la, c->loss.p, sizeof la, cudaMemcpyDeviceToHost, s));
  TRY(step_sync(c));
  if (la_pin) la = *la_pin;
  c->d2h += sizeof la;
  if (la.error & 2u) return set_err(DG_EPROTO, "worker: missing partial in batch %llu", (unsigned long long)step);
  c->adam_t += 1;
  c->worker_step = step + 1;
  TRY(occupancy_update(c));
  if (c->timing) {
    CU(cudaStreamSynchronize(c->stream_adam));  // stage timing (diagnostic) waits for Adam
    float* t = &c->times.segment;
    for (int k = 0; k < 10; ++k) cudaEventElapsedTime(&t[k], c->ev[k], c->ev[k + 1]);
    cudaEventElapsedTime(&c->times.total, c->ev[0], c->ev[10]);
    cudaEventElapsedTime(&c->times.dispatch_exchange, c->ev[11], c->ev[1]);
    c->times.dispatch_mb = float(double(bytes_x1) * 1e-6);
    c->times.partial_mb = float(double(bytes - bytes_x1) * 1e-6);
  }
  if (stats) {
    std::memset(stats, 0, sizeof *stats);
    stats->step = step;
    for (uint32_t lp = 0; lp < nl; ++lp) {  // ControlSync per worker (wire.cpp:117-128)
      const bool f32 = c->cfg.wire_f32 != 0;
      stats->loss_rgb += f32 ? double(float(la.rgb[lp])) : la.rgb[lp];
      stats->loss_transmittance += f32 ? double(float(la.trans[lp])) : la.trans[lp];
      stats->loss_distortion += f32 ? double(float(la.dist[lp])) : la.dist[lp];
    }
    stats->lr = dg_lr_at(&c->cfg, step);
    stats->rays = b->n - dropped;
    stats->dropped_rays = dropped;
    stats->bytes_sent = bytes;
    stats->samples = uint64_t(c->n_fine) + c->n_coarse;
    stats->items = NI;
    stats->h2d_bytes = c->h2d;
    stats->d2h_bytes = c->d2h;
    stats->partial_bytes_sent = bytes - bytes_x1;
    stats->partial_records_sent =
        (bytes - bytes_x1) / (sizeof(PartialRec) + (c->cross_active ? sizeof(float4) : 0));
  }
  return DG_OK;
}

int dg_render(dg_ctx* c, const dg_ray_batch* b, const float* appearance, dg_merged* out) {
  TRY(check_ctx(c));
  if (!b || !out) return set_err(DG_EINVAL, "null argument");
  if (b->n && (!b->origin || !b->dir)) return set_err(DG_EINVAL, "batch: missing arrays");
  if (c->world > 1 && !c->comm) return set_err(DG_EINVAL, "world > 1 needs dg_comm_init_*");
  CU(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  uint64_t dropped = 0, bytes = 0;
  c->cross_active = false;  // evaluation carries no distortion aggregates
  dg_ray_batch bb = *b;
  bb.color_gt = nullptr;
  bb.image_id = nullptr;
  // eval appearance vector through the wire (EvalRequest reals, wire.cpp:170-176)
  std::vector<float> app(c->cfg.appearance_dim + 1, 0.0f);
  for (uint32_t k = 0; k < c->cfg.appearance_dim; ++k) app[k] = appearance ? appearance[k] : 0.0f;
  TRY(pin_reset(c));
  TRY(upload_small(c, c->eval_app, app.data(), app.size() * sizeof(float)));
  const uint32_t saved_rows = c->app_rows;
  c->app_rows = std::max<uint32_t>(c->app_rows, 1);
  const int rc = front_half(c, &bb, 0, 0, &dropped, &bytes);
  c->app_rows = saved_rows;
  TRY(rc);
  const uint32_t NI = c->n_items;
  ItemArrays it = item_arrays(c);
  SampleArrays sm = sample_arrays(c);
  {
    TRY(pairs_expand(c, s));
    std::vector<EncPass> passes;
    const FieldLaunch fl = field_launch(c, c->enc_budget_fwd, passes, c->enc_group_fwd, c->enc_hgroup_fwd);
    c->launches += launch_encode_fwd(fl, passes, sm.X, s) - 1;
  }
  MlpLaunch mf = mlp_launch(c, false);
  mf.masks = nullptr;  // evaluation has no backward
  mf.app_override = c->eval_app.as<float>();
  if (c->mlp_impl) launch_mlp_eval_tc(mf, c->num_sms, s);  // split-bf16: no ReLU decision kept
  else launch_mlp_fwd(mf, s);
  launch_composite(NI, it, sm, c->n_fine, 1, s);
  c->launches += 3;
  const uint64_t n = b->n;
  float* rgb = out->rgb;
  float* tr = out->transmittance;
  float* dep = out->depth;
  float* attr = out->attribution;
  if (out->mem != DG_MEM_DEVICE) {
    TRY(c->out_rgb.ensure(n * 12 + 16));
    TRY(c->out_T.ensure(n * 4 + 16));
    TRY(c->out_depth.ensure(n * 4 + 16));
    rgb = c->out_rgb.as<float>();
    tr = c->out_T.as<float>();
    dep = c->out_depth.as<float>();
    if (attr) {
      TRY(c->out_attr.ensure(n * 12 + 16));
      attr = c->out_attr.as<float>();
    }
  }
  const PartialRec* reply = nullptr;
  if (c->world > 1) {
    // reply: items [lp][src] -> send [src][lp] (the home rank's dispatch layout)
    const int W = c->world;
    const uint32_t nl = uint32_t(c->local.size());
    // per (lp, src) counts from part_item_off and the gather table of front_half
    std::vector<uint64_t> tab(2 * uint64_t(nl) * W);
    // re-derive counts from the perm table (src_start, dst_start) uploaded in front_half
    std::vector<uint64_t> perm(2 * uint64_t(nl) * W);
    CU(cudaMemcpyAsync(perm.data(), c->perm_tab.p, perm.size() * 8, cudaMemcpyDeviceToHost, s));
    TRY(step_sync(c));
    const uint32_t nblk = nl * uint32_t(W);
    std::vector<uint64_t> cnt(nblk);
    for (uint32_t k = 0; k < nblk; ++k)
      cnt[k] = (k + 1 < nblk ? perm[k + 1] : NI) - perm[k];
    // blocks in [src][lp] order: src_start = perm[k], dst(items) start = perm[nblk + k]
    std::vector<PartialRec> dummy;
    TRY(c->send_buf.ensure(uint64_t(NI) * sizeof(PartialRec) + 16));
    // pack partial records in item order first
    {
      std::vector<uint64_t> t2(2 * nblk);
      for (uint32_t k = 0; k < nblk; ++k) {
        t2[k] = perm[nblk + k];  // source (items) start for block k
        t2[nblk + k] = perm[k];  // destination (reply send) start
      }
      // k_block_permute walks blocks by source start, which must be ascending: items are
      // [lp][src] so sort the blocks by item start.
      std::vector<uint32_t> order(nblk);
      for (uint32_t k = 0; k < nblk; ++k) order[k] = k;
      std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b2) { return t2[a] < t2[b2]; });
      std::vector<uint64_t> t3(2 * nblk);
      for (uint32_t k = 0; k < nblk; ++k) {
        t3[k] = t2[order[k]];
        t3[nblk + k] = t2[nblk + order[k]];
      }
      TRY(upload(c->perm_tab, t3.data(), t3.size() * 8, s));
    }
    // item partials -> PartialRec (in item order) in recv_buf, then permute into send_buf
    TRY(c->recv_buf.ensure(uint64_t(NI) * sizeof(PartialRec) + 16));
    {
      launch_items_to_records(NI, it.partial, it.depth, it.rec, c->recv_buf.as<PartialRec>(), s);
    }
    if (NI) {
      k_block_permute<<<unsigned((NI + 255) / 256), 256, 0, s>>>(
          c->recv_buf.as<uint64_t>(), c->send_buf.as<uint64_t>(), sizeof(PartialRec) / 8,
          c->perm_tab.as<uint64_t>(), nblk, NI);
      c->launches += 2;
    }
    std::vector<uint64_t> sbytes(W, 0), rbytes(W, 0);
    for (int r = 0; r < W; ++r)
      for (uint32_t lp = 0; lp < nl; ++lp) sbytes[r] += cnt[uint64_t(r) * nl + lp] * sizeof(PartialRec);
    // home side: what I dispatched to each rank comes back
    std::vector<uint32_t> slot_start(c->P + 1);
    CU(cudaMemcpy2DAsync(slot_start.data(), 4, c->h_pos.as<uint32_t>(), n ? n * 4 : 4, 4, c->P + 1,
                         cudaMemcpyDeviceToHost, s));
    TRY(step_sync(c));
    for (uint32_t p = 0; p < c->P; ++p)
      rbytes[c->part_rank[p]] +=
          uint64_t(slot_start[c->slot_of_part[p] + 1] - slot_start[c->slot_of_part[p]]) * sizeof(PartialRec);
    uint64_t rtot = 0;
    for (auto v : rbytes) rtot += v;
    TRY(c->x_recv.ensure(rtot + 16));
    std::string err;
    const int rc2 = c->comm->alltoallv(c->send_buf.p, sbytes, c->x_recv.p, rbytes, s, err);
    if (rc2 != DG_OK) return set_err(rc2, "%s", err.c_str());
    reply = c->x_recv.as<PartialRec>();
  }
  launch_home_merge(n, c->P, c->h_nseg.as<uint8_t>(), c->h_sched.as<uint8_t>(),
                    c->slot_of_part_d.as<uint8_t>(), c->h_pos.as<uint32_t>(), it.partial, it.depth,
                    reply, int(c->cfg.wire_f32), rgb, tr, dep, int(c->cfg.eval_early_termination),
                    c->cfg.eval_termination_threshold, attr, s);
  ++c->launches;
  if (out->mem != DG_MEM_DEVICE && n) {
    CU(cudaMemcpyAsync(out->rgb, rgb, n * 12, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(out->transmittance, tr, n * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(out->depth, dep, n * 4, cudaMemcpyDeviceToHost, s));
    if (attr) CU(cudaMemcpyAsync(out->attribution, attr, n * 12, cudaMemcpyDeviceToHost, s));
  }
  TRY(step_sync(c));
  return DG_OK;
}

// DistributedRun::evaluate_image (worker.cpp:836-880): one ray per pixel (row-major, pixel
// centres, CameraPose::pixel_ray_dir) generated on the device, rendered through dg_render;
// out arrays hold width * height entries (attribution optional).  Ray ids are pixel indices.
int dg_render_image(dg_ctx* c, const dg_camera* cam, const float* appearance, dg_merged* out) {
  TRY(check_ctx(c));
  if (!cam || !out || cam->width == 0 || cam->height == 0) return set_err(DG_EINVAL, "render_image: bad camera");
  CU(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const uint64_t n = uint64_t(cam->width) * cam->height;
  double pose[16];
  for (int k = 0; k < 9; ++k) pose[k] = cam->rotation[k];
  for (int k = 0; k < 3; ++k) pose[9 + k] = cam->translation[k];
  pose[12] = cam->fx;
  pose[13] = cam->fy;
  pose[14] = cam->cx;
  pose[15] = cam->cy;
  TRY(upload(c->cam_pose, pose, sizeof pose, s));
  TRY(c->cam_o.ensure(n * 24 + 16));
  TRY(c->cam_d.ensure(n * 24 + 16));
  launch_camera_rays(c->cam_pose.as<double>(), cam->width, n, c->cam_o.as<double>(), c->cam_d.as<double>(), s);
  ++c->launches;
  std::vector<uint32_t> img(1, cam->image_id);
  dg_ray_batch b{c->cam_o.as<double>(), c->cam_d.as<double>(), nullptr, nullptr, n, 0, DG_MEM_DEVICE, 0};
  return dg_render(c, &b, appearance, out);
}

int dg_comm_unique_id(uint8_t id[DG_NCCL_UNIQUE_ID_BYTES]) {
  std::string err;
  const int rc = nccl_unique_id(id, err);
  if (rc != DG_OK) return set_err(rc, "%s", err.c_str());
  return DG_OK;
}

int dg_comm_init_nccl(dg_ctx* c, const uint8_t id[DG_NCCL_UNIQUE_ID_BYTES]) {
  TRY(check_ctx(c));
  std::string err;
  Comm* comm = make_nccl_comm(id, c->rank, c->world, c->device, err,
                              std::chrono::milliseconds(c->comm_timeout_ms));
  if (!comm) return set_err(DG_ENCCL, "%s", err.c_str());
  c->comm.reset(comm);
  return DG_OK;
}

int dg_set_comm_timeout(dg_ctx* c, uint64_t timeout_ms) {
  TRY(check_ctx(c));
  if (timeout_ms == 0) return set_err(DG_EINVAL, "timeout must be positive");
  c->comm_timeout_ms = timeout_ms;
  if (c->comm) c->comm->set_timeout(std::chrono::milliseconds(timeout_ms));
  return DG_OK;
}

int dg_comm_init_host(dg_ctx* c, dg_alltoallv_fn fn, void* user) {
  TRY(check_ctx(c));
  if (!fn) return set_err(DG_EINVAL, "null callback");
  c->comm.reset(make_host_comm(fn, user, c->rank, c->world));
  c->comm->set_timeout(std::chrono::milliseconds(c->comm_timeout_ms));
  return DG_OK;
}

int dg_comm_init_peer(dg_ctx* c, dg_allgather_fn fn, void* user) {
  TRY(check_ctx(c));
  if (!fn) return set_err(DG_EINVAL, "null callback");
  CU(cudaSetDevice(c->device));
  c->comm.reset(new PeerComm(fn, user, c->rank, c->world));
  c->comm->set_timeout(std::chrono::milliseconds(c->comm_timeout_ms));
  return DG_OK;
}

// ---------------------------------------------------------------- stage entry points
int dg_segment_rays(dg_ctx* c, const double* origin, const double* dir, uint64_t n, uint8_t* nseg,
                    uint16_t* region, double* t_enter, double* t_exit, int32_t mem) {
  TRY(check_ctx(c));
  cudaStream_t s = c->stream;
  DBuf o, d, ns, sc, te, tx;
  const double* od = origin;
  const double* dd = dir;
  if (mem != DG_MEM_DEVICE) {
    TRY(upload(o, origin, n * 24, s));
    TRY(upload(d, dir, n * 24, s));
    od = o.as<double>();
    dd = d.as<double>();
  }
  TRY(ns.ensure(n + 16));
  TRY(sc.ensure(n * kMaxSeg + 16));
  TRY(te.ensure(n * kMaxSeg * 8 + 16));
  TRY(tx.ensure(n * kMaxSeg * 8 + 16));
  launch_segment_full(c->d_geo.as<Geo>(), od, dd, n, ns.as<uint8_t>(), sc.as<uint8_t>(),
                      te.as<double>(), tx.as<double>(), s);
  ++c->launches;
  std::vector<uint8_t> hs(n * kMaxSeg);
  if (mem != DG_MEM_DEVICE) {
    CU(cudaMemcpyAsync(nseg, ns.p, n, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(hs.data(), sc.p, n * kMaxSeg, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(t_enter, te.p, n * kMaxSeg * 8, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(t_exit, tx.p, n * kMaxSeg * 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    for (uint64_t i = 0; i < n * kMaxSeg; ++i) region[i] = hs[i] == 0xff ? 0 : hs[i];
  } else {
    CU(cudaMemcpyAsync(nseg, ns.p, n, cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(t_enter, te.p, n * kMaxSeg * 8, cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(t_exit, tx.p, n * kMaxSeg * 8, cudaMemcpyDeviceToDevice, s));
    launch_u8_to_u16(sc.as<uint8_t>(), region, n * kMaxSeg, s);
    CU(cudaStreamSynchronize(s));
  }
  return DG_OK;
}

int dg_cascade_march(dg_ctx* c, uint32_t p, const double* origin, const double* dir, const double* t0,
                     const double* t1, const uint64_t* ray_id, uint64_t n, int32_t jitter,
                     uint64_t batch_id, uint32_t* counts, const uint64_t* offsets, double* t,
                     double* delta, uint8_t* cascade, int32_t mem) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (mem == DG_MEM_DEVICE) return set_err(DG_EINVAL, "dg_cascade_march: host buffers only");
  cudaStream_t s = c->stream;
  DBuf o, d, a, b, rid, cnt, off, tt, dl, cs;
  TRY(upload(o, origin, n * 24, s));
  TRY(upload(d, dir, n * 24, s));
  TRY(upload(a, t0, n * 8, s));
  TRY(upload(b, t1, n * 8, s));
  TRY(upload(rid, ray_id, n * 8, s));
  TRY(cnt.ensure(n * 4 + 16));
  uint64_t total = 0;
  if (t) {
    if (!offsets || !counts) return set_err(DG_EINVAL, "fill mode needs counts and offsets");
    for (uint64_t i = 0; i < n; ++i) total = std::max(total, offsets[i] + counts[i]);
    TRY(upload(off, offsets, n * 8, s));
    TRY(tt.ensure(total * 8 + 16));
    TRY(dl.ensure(total * 8 + 16));
    TRY(cs.ensure(total + 16));
  }
  launch_march_points(c->d_parts.as<PartDesc>() + lp, c->occ.as<uint8_t>(), o.as<double>(), d.as<double>(),
                      a.as<double>(), b.as<double>(), rid.as<uint64_t>(), n, c->step, c->cfg.seed,
                      batch_id, jitter, cnt.as<uint32_t>(), t ? off.as<uint64_t>() : nullptr,
                      t ? tt.as<double>() : nullptr, t ? dl.as<double>() : nullptr,
                      t ? cs.as<uint8_t>() : nullptr, s);
  ++c->launches;
  if (!t) {
    CU(cudaMemcpyAsync(counts, cnt.p, n * 4, cudaMemcpyDeviceToHost, s));
  } else {
    CU(cudaMemcpyAsync(t, tt.p, total * 8, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(delta, dl.p, total * 8, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(cascade, cs.p, total, cudaMemcpyDeviceToHost, s));
  }
  CU(cudaStreamSynchronize(s));
  return DG_OK;
}

int dg_encode(dg_ctx* c, uint32_t p, uint32_t cascade, const double* points, uint64_t n,
              float* features, uint32_t* rows, int32_t mem) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (cascade > 1) return set_err(DG_EINVAL, "cascade must be 0 or 1");
  cudaStream_t s = c->stream;
  const FieldDesc* fd = c->d_fields.as<FieldDesc>() + cascade * c->local.size() + lp;
  const uint32_t L = c->cfg.grid_levels;
  DBuf pts, X, R;
  const double* pd = points;
  if (mem != DG_MEM_DEVICE) {
    TRY(upload(pts, points, n * 24, s));
    pd = pts.as<double>();
  }
  TRY(X.ensure(n * kEnc * 4 + 16));
  if (rows) TRY(R.ensure(n * L * 8 * 4 + 16));
  launch_encode_points(fd, c->params.as<float>(), pd, n, L, X.as<float>(), rows ? R.as<uint32_t>() : nullptr, s);
  ++c->launches;
  // features: n x (L*2) compacted from the padded n x 32 rows
  std::vector<float> hx(n * kEnc);
  CU(cudaMemcpyAsync(hx.data(), X.p, n * kEnc * 4, cudaMemcpyDeviceToHost, s));
  if (rows) {
    if (mem == DG_MEM_DEVICE) CU(cudaMemcpyAsync(rows, R.p, n * L * 8 * 4, cudaMemcpyDeviceToDevice, s));
    else CU(cudaMemcpyAsync(rows, R.p, n * L * 8 * 4, cudaMemcpyDeviceToHost, s));
  }
  CU(cudaStreamSynchronize(s));
  std::vector<float> packed(n * L * 2);  // level-major [L][n] float2 -> [n][L*2]
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t l = 0; l < L; ++l) {
      packed[i * L * 2 + 2 * l] = hx[(l * n + i) * 2];
      packed[i * L * 2 + 2 * l + 1] = hx[(l * n + i) * 2 + 1];
    }
  if (mem == DG_MEM_DEVICE) CU(cudaMemcpy(features, packed.data(), packed.size() * 4, cudaMemcpyHostToDevice));
  else std::memcpy(features, packed.data(), packed.size() * 4);
  return DG_OK;
}

int dg_encode_backward(dg_ctx* c, uint32_t p, uint32_t cascade, const double* points,
                       const float* upstream, uint64_t n, int32_t mem) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (cascade > 1) return set_err(DG_EINVAL, "cascade must be 0 or 1");
  if (mem == DG_MEM_DEVICE) return set_err(DG_EINVAL, "dg_encode_backward: host buffers only");
  cudaStream_t s = c->stream;
  const uint32_t L = c->cfg.grid_levels;
  std::vector<float> up(n * kEnc, 0.0f);  // [n][L*2] -> level-major [L][n] float2
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t l = 0; l < L; ++l) {
      up[(l * n + i) * 2] = upstream[i * L * 2 + 2 * l];
      up[(l * n + i) * 2 + 1] = upstream[i * L * 2 + 2 * l + 1];
    }
  DBuf pts, dX;
  TRY(upload(pts, points, n * 24, s));
  TRY(upload(dX, up.data(), up.size() * 4, s));
  launch_encode_points_bwd(c->d_fields.as<FieldDesc>() + cascade * c->local.size() + lp, c->grads.as<float>(),
                           pts.as<double>(), dX.as<float>(), n, L, s);
  ++c->launches;
  CU(cudaStreamSynchronize(s));
  return DG_OK;
}

// Field stage entries: build one-sample "items" so the production MLP kernels run unchanged.
static int field_stage(dg_ctx* c, uint32_t p, uint32_t cascade, const double* points, const float* dirs,
                       const float* app, uint64_t n, const float* sig_grad, const float* rgb_grad,
                       float* sigma, float* rgb) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (cascade > 1) return set_err(DG_EINVAL, "cascade must be 0 or 1");
  cudaStream_t s = c->stream;
  const uint32_t nl = uint32_t(c->local.size());
  const uint32_t f = cascade * nl + lp;
  const FieldDesc* fd = c->d_fields.as<FieldDesc>() + f;
  DBuf pts, X, recs, items, appb, out, gin, dX, foff, toff;
  TRY(upload(pts, points, n * 24, s));
  TRY(X.ensure(n * kEnc * 4 + 16));
  launch_encode_points(fd, c->params.as<float>(), pts.as<double>(), n, c->cfg.grid_levels, X.as<float>(), nullptr, s);
  std::vector<RayRec> rr(n);
  std::vector<uint32_t> ids(n);
  for (uint64_t i = 0; i < n; ++i) {
    std::memset(&rr[i], 0, sizeof(RayRec));
    for (int a = 0; a < 3; ++a) rr[i].d[a] = dirs[3 * i + a];
    ids[i] = uint32_t(i);
  }
  TRY(upload(recs, rr.data(), n * sizeof(RayRec), s));
  TRY(upload(items, ids.data(), n * 4, s));
  TRY(upload(appb, app, n * c->cfg.appearance_dim * 4, s));
  // fields 0..2nl-1 with only field f non-empty
  std::vector<uint32_t> fo(2 * nl + 1, 0), tf(2 * nl + 1, 0), tb(2 * nl + 1, 0);
  for (uint32_t k = f + 1; k <= 2 * nl; ++k) {
    fo[k] = uint32_t(n);
    tf[k] = uint32_t((n + 127) / 128);
    tb[k] = uint32_t((n + 63) / 64);
  }
  TRY(upload(foff, fo.data(), fo.size() * 4, s));
  MlpLaunch m{};
  m.fields = c->d_fields.as<FieldDesc>();
  m.n_fields = 2 * nl;
  m.field_off = foff.as<uint32_t>();
  m.X = X.as<float>();
  m.x_stride = n;
  m.levels = c->cfg.grid_levels;
  m.rec = recs.as<RayRec>();
  m.s_item = items.as<uint32_t>();
  m.app_override = appb.as<float>();
  m.app_per_sample = 1;
  m.params = c->params.as<float>();
  m.grads = c->grads.as<float>();
  TRY(out.ensure(n * 16 + 16));
  m.out = out.as<float4>();
  m.out_tile = m.out;  // no sample permutation here: tile rows are the caller's points
  DBuf masks;
  if (!sig_grad) {
    TRY(upload(toff, tf.data(), tf.size() * 4, s));
    m.tile_off = toff.as<uint32_t>();
    m.n_tiles = tf[2 * nl];
    if (c->mlp_impl) launch_mlp_fwd_tc(m, c->num_sms, s);
    else launch_mlp_fwd(m, s);
    std::vector<float4> h(n);
    CU(cudaMemcpyAsync(h.data(), out.p, n * 16, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    for (uint64_t i = 0; i < n; ++i) {
      sigma[i] = h[i].x;
      rgb[3 * i] = h[i].y;
      rgb[3 * i + 1] = h[i].z;
      rgb[3 * i + 2] = h[i].w;
    }
    c->launches += 2;
    return DG_OK;
  }
  std::vector<float4> g(n);
  for (uint64_t i = 0; i < n; ++i)
    g[i] = make_float4(sig_grad[i], rgb_grad[3 * i], rgb_grad[3 * i + 1], rgb_grad[3 * i + 2]);
  TRY(upload(gin, g.data(), n * 16, s));
  TRY(dX.ensure(n * kEnc * 4 + 16));
  if (c->mlp_impl) {  // the tcgen05 backward takes its ReLU / clip masks from the forward
    TRY(masks.ensure(n * 7 * 4 + 16));
    m.masks = masks.as<uint32_t>();
    TRY(upload(toff, tf.data(), tf.size() * 4, s));
    m.tile_off = toff.as<uint32_t>();
    m.n_tiles = tf[2 * nl];
    launch_mlp_fwd_tc(m, c->num_sms, s);
    ++c->launches;
  }
  const std::vector<uint32_t>& tt = c->mlp_impl ? tf : tb;
  TRY(upload(toff, tt.data(), tt.size() * 4, s));
  m.tile_off = toff.as<uint32_t>();
  m.n_tiles = tt[2 * nl];
  m.grad_in = gin.as<float4>();
  m.dX = dX.as<float>();
  m.relu_tiles = cascade == 0 && c->mlp_bwd_paired ? m.n_tiles : 0u;  // the fine field: ReLU units
  m.issue_warp = c->mlp_issue_warp;
  m.issue_warp_fwd = c->mlp_issue_warp_fwd;
  if (c->mlp_impl) launch_mlp_bwd_tc(m, c->num_sms, s);
  else launch_mlp_bwd(m, c->num_sms, s);
  launch_encode_points_bwd(fd, c->grads.as<float>(), pts.as<double>(), dX.as<float>(), n, c->cfg.grid_levels, s);
  c->launches += 3;
  CU(cudaStreamSynchronize(s));
  return DG_OK;
}

int dg_field_forward(dg_ctx* c, uint32_t p, uint32_t cascade, const double* points, const float* dirs,
                     const float* app, uint64_t n, float* sigma, float* rgb, int32_t mem) {
  if (mem == DG_MEM_DEVICE) return set_err(DG_EINVAL, "dg_field_forward: host buffers only");
  return field_stage(c, p, cascade, points, dirs, app, n, nullptr, nullptr, sigma, rgb);
}

int dg_field_density(dg_ctx* c, uint32_t p, uint32_t cascade, const double* points, uint64_t n, float* sigma,
                     float* features) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (cascade > 1) return set_err(DG_EINVAL, "cascade must be 0 or 1");
  if (n && (!points || !sigma || !features)) return set_err(DG_EINVAL, "null argument");
  if (!n) return DG_OK;
  cudaStream_t s = c->stream;
  const FieldDesc* fd = c->d_fields.as<FieldDesc>() + cascade * c->local.size() + lp;
  DBuf pts, X, sg, ft;
  TRY(upload(pts, points, n * 24, s));
  TRY(X.ensure(n * kEnc * 4 + 16));
  TRY(sg.ensure(n * 4 + 16));
  TRY(ft.ensure(n * 60 + 16));
  launch_encode_points(fd, c->params.as<float>(), pts.as<double>(), n, c->cfg.grid_levels, X.as<float>(), nullptr, s);
  launch_field_density(fd, c->params.as<float>(), X.as<float>(), n, sg.as<float>(), ft.as<float>(), s);
  c->launches += 2;
  CU(cudaMemcpyAsync(sigma, sg.p, n * 4, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(features, ft.p, n * 60, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return DG_OK;
}

int dg_field_color(dg_ctx* c, uint32_t p, uint32_t cascade, const float* features, const float* dirs,
                   const float* app, uint64_t n, float* rgb) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (cascade > 1) return set_err(DG_EINVAL, "cascade must be 0 or 1");
  if (n && (!features || !dirs || !rgb || (c->cfg.appearance_dim && !app))) return set_err(DG_EINVAL, "null argument");
  if (!n) return DG_OK;
  cudaStream_t s = c->stream;
  const FieldDesc* fd = c->d_fields.as<FieldDesc>() + cascade * c->local.size() + lp;
  DBuf ft, dr, ap, out;
  TRY(upload(ft, features, n * 60, s));
  TRY(upload(dr, dirs, n * 12, s));
  TRY(upload(ap, app, n * c->cfg.appearance_dim * 4, s));
  TRY(out.ensure(n * 12 + 16));
  launch_field_color(fd, c->params.as<float>(), ft.as<float>(), dr.as<float>(), ap.as<float>(), n, out.as<float>(), s);
  ++c->launches;
  CU(cudaMemcpyAsync(rgb, out.p, n * 12, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return DG_OK;
}

int dg_field_backward(dg_ctx* c, uint32_t p, uint32_t cascade, const double* points, const float* dirs,
                      const float* app, const float* sigma_grad, const float* rgb_grad, uint64_t n,
                      int32_t mem) {
  if (mem == DG_MEM_DEVICE) return set_err(DG_EINVAL, "dg_field_backward: host buffers only");
  if (!sigma_grad || !rgb_grad) return set_err(DG_EINVAL, "null gradients");
  return field_stage(c, p, cascade, points, dirs, app, n, sigma_grad, rgb_grad, nullptr, nullptr);
}

// ---------------------------------------------------------- compositing stage entry points
}  // extern "C"

namespace {

// Inputs / outputs of a stage call: device pointers pass through, host arrays are staged.
struct StageIo {
  dg_ctx* c;
  int32_t mem;
  std::vector<std::unique_ptr<DBuf>> tmp;
  std::vector<std::tuple<void*, const DBuf*, size_t>> back;  // host dst, device src, bytes
  template <class T>
  int in(const T* p, uint64_t n, const T** out) {
    if (!p || mem == DG_MEM_DEVICE || n == 0) {
      *out = p;
      return DG_OK;
    }
    tmp.emplace_back(new DBuf);
    TRY(upload(*tmp.back(), p, n * sizeof(T), c->stream));
    *out = tmp.back()->as<T>();
    return DG_OK;
  }
  template <class T>
  int out(T* p, uint64_t n, T** dev) {
    if (!p || mem == DG_MEM_DEVICE || n == 0) {
      *dev = p;
      return DG_OK;
    }
    tmp.emplace_back(new DBuf);
    TRY(tmp.back()->ensure(n * sizeof(T)));
    back.emplace_back(p, tmp.back().get(), n * sizeof(T));
    *dev = tmp.back()->as<T>();
    return DG_OK;
  }
  int finish() {
    for (auto& [h, d, bytes] : back) CU(cudaMemcpyAsync(h, d->p, bytes, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return DG_OK;
  }
};

// Segment offsets (n + 1 entries, non-decreasing, from 0) on the host, for validation and
// for the sample totals.
int host_offsets(dg_ctx* c, const uint64_t* off, uint64_t n, int32_t mem, std::vector<uint64_t>& h) {
  if (!off) return set_err(DG_EINVAL, "null offsets");
  h.resize(n + 1);
  if (mem == DG_MEM_DEVICE) CU(cudaMemcpy(h.data(), off, (n + 1) * 8, cudaMemcpyDeviceToHost));
  else std::memcpy(h.data(), off, (n + 1) * 8);
  if (h[0] != 0) return set_err(DG_EINVAL, "offsets must start at 0");
  for (uint64_t i = 0; i < n; ++i)
    if (h[i + 1] < h[i]) return set_err(DG_EINVAL, "offsets must be non-decreasing");
  return DG_OK;
}

template <class R>
int local_render_impl(dg_ctx* c, const double* t, const double* delta, const R* sigma, const R* rgb,
                    const uint64_t* seg_off, uint64_t n_seg, const double* ray_t0, const double* ray_t1,
                    R* out_rgb, R* out_T, R* out_depth_sum, double* out_distortion,
                    int32_t mem, double* out_cache = nullptr) {
  TRY(check_ctx(c));
  if (!out_rgb || !out_T) return set_err(DG_EINVAL, "null outputs");
  std::vector<uint64_t> off;
  TRY(host_offsets(c, seg_off, n_seg, mem, off));
  const uint64_t ns = off[n_seg];
  if (ns && (!t || !delta || !sigma || !rgb)) return set_err(DG_EINVAL, "null sample arrays");
  if (out_distortion && (!ray_t0 || !ray_t1)) return set_err(DG_EINVAL, "distortion stats need the ray span");
  StageIo io{c, mem, {}, {}};
  const double *dt, *dd, *t0 = nullptr, *t1 = nullptr;
  const R *dsig, *drgb;
  const uint64_t* doff;
  TRY(io.in(t, ns, &dt));
  TRY(io.in(delta, ns, &dd));
  TRY(io.in(sigma, ns, &dsig));
  TRY(io.in(rgb, 3 * ns, &drgb));
  TRY(io.in(seg_off, n_seg + 1, &doff));
  TRY(io.in(ray_t0, n_seg, &t0));
  TRY(io.in(ray_t1, n_seg, &t1));
  R *orgb, *oT, *odep;
  double* odist;
  TRY(io.out(out_rgb, 3 * n_seg, &orgb));
  TRY(io.out(out_T, n_seg, &oT));
  TRY(io.out(out_depth_sum, n_seg, &odep));
  TRY(io.out(out_distortion, 3 * n_seg, &odist));
  double* ocache;
  TRY(io.out(out_cache, 2 * ns, &ocache));
  launch_local_render(dt, dd, dsig, drgb, doff, n_seg, out_distortion ? t0 : nullptr,
                      out_distortion ? t1 : nullptr, orgb, oT, odep, odist, ocache, c->stream);
  ++c->launches;
  return io.finish();
}

template <class R>
int local_render_backward_impl(dg_ctx* c, const double* t, const double* delta, const R* sigma,
                             const R* rgb, const uint64_t* seg_off, uint64_t n_seg, const R* d_rgb,
                             const R* d_transmittance, const R* weight_upstream, R* sigma_grad,
                             R* rgb_grad, int32_t mem) {
  TRY(check_ctx(c));
  if (!d_rgb || !d_transmittance) return set_err(DG_EINVAL, "null upstream");
  std::vector<uint64_t> off;
  TRY(host_offsets(c, seg_off, n_seg, mem, off));
  const uint64_t ns = off[n_seg];
  if (ns && (!t || !delta || !sigma || !rgb || !sigma_grad || !rgb_grad))
    return set_err(DG_EINVAL, "null sample arrays");
  StageIo io{c, mem, {}, {}};
  const double *dt, *dd;
  const R *dsig, *drgb, *ug, *ut, *uw;
  const uint64_t* doff;
  TRY(io.in(t, ns, &dt));
  TRY(io.in(delta, ns, &dd));
  TRY(io.in(sigma, ns, &dsig));
  TRY(io.in(rgb, 3 * ns, &drgb));
  TRY(io.in(seg_off, n_seg + 1, &doff));
  TRY(io.in(d_rgb, 3 * n_seg, &ug));
  TRY(io.in(d_transmittance, n_seg, &ut));
  TRY(io.in(weight_upstream, ns, &uw));
  R *sg, *cg;
  TRY(io.out(sigma_grad, ns, &sg));
  TRY(io.out(rgb_grad, 3 * ns, &cg));
  // the forward sweep's (alpha, prefix) cache (LocalRenderCache), then the reverse sweep
  DBuf cache, scratch;
  TRY(cache.ensure(ns * 16 + 16));
  TRY(scratch.ensure(n_seg * 4 * sizeof(R) + 16));
  R* srgb = scratch.as<R>();
  launch_local_render<R>(dt, dd, dsig, drgb, doff, n_seg, nullptr, nullptr, srgb, srgb + 3 * n_seg,
                         static_cast<R*>(nullptr), nullptr, cache.as<double>(), c->stream);
  launch_local_render_bwd(dd, drgb, doff, n_seg, cache.as<double>(), ug, ut, uw, sg, cg, c->stream);
  c->launches += 2;
  return io.finish();
}

template <class R>
int merge_forward_impl(dg_ctx* c, const R* seg_rgb, const R* seg_transmittance,
                     const R* seg_depth_sum, const uint64_t* ray_off, uint64_t n_rays, R* rgb,
                     R* transmittance, R* depth, int32_t mem) {
  TRY(check_ctx(c));
  if (!rgb || !transmittance) return set_err(DG_EINVAL, "null outputs");
  std::vector<uint64_t> off;
  TRY(host_offsets(c, ray_off, n_rays, mem, off));
  for (uint64_t r = 0; r < n_rays; ++r)
    if (off[r + 1] == off[r]) return set_err(DG_EINVAL, "merge: no partials");  // render.cpp:102
  const uint64_t ns = off[n_rays];
  StageIo io{c, mem, {}, {}};
  const R *sr, *sT, *sd;
  const uint64_t* doff;
  TRY(io.in(seg_rgb, 3 * ns, &sr));
  TRY(io.in(seg_transmittance, ns, &sT));
  TRY(io.in(seg_depth_sum, ns, &sd));
  TRY(io.in(ray_off, n_rays + 1, &doff));
  R *orgb, *oT, *od;
  TRY(io.out(rgb, 3 * n_rays, &orgb));
  TRY(io.out(transmittance, n_rays, &oT));
  TRY(io.out(depth, n_rays, &od));
  launch_merge_fwd(sr, sT, sd, doff, n_rays, orgb, oT, od, c->stream);
  ++c->launches;
  return io.finish();
}

template <class R>
int merge_backward_impl(dg_ctx* c, const R* seg_rgb, const R* seg_transmittance, const uint64_t* ray_off,
                      uint64_t n_rays, const R* d_rgb, const R* d_transmittance, R* seg_d_rgb,
                      R* seg_d_transmittance, int32_t mem) {
  TRY(check_ctx(c));
  if (!d_rgb || !d_transmittance || !seg_d_rgb || !seg_d_transmittance) return set_err(DG_EINVAL, "null argument");
  std::vector<uint64_t> off;
  TRY(host_offsets(c, ray_off, n_rays, mem, off));
  for (uint64_t r = 0; r < n_rays; ++r)
    if (off[r + 1] - off[r] > uint64_t(kMaxSeg)) return set_err(DG_EINVAL, "merge: more than %d partials", kMaxSeg);
  const uint64_t ns = off[n_rays];
  StageIo io{c, mem, {}, {}};
  const R *sr, *sT, *ug, *ut;
  const uint64_t* doff;
  TRY(io.in(seg_rgb, 3 * ns, &sr));
  TRY(io.in(seg_transmittance, ns, &sT));
  TRY(io.in(ray_off, n_rays + 1, &doff));
  TRY(io.in(d_rgb, 3 * n_rays, &ug));
  TRY(io.in(d_transmittance, n_rays, &ut));
  R *og, *ot;
  TRY(io.out(seg_d_rgb, 3 * ns, &og));
  TRY(io.out(seg_d_transmittance, ns, &ot));
  launch_merge_bwd(sr, sT, doff, n_rays, ug, ut, og, ot, c->stream);
  ++c->launches;
  return io.finish();
}

template <class R>
int ray_losses_impl(dg_ctx* c, const R* rgb, const R* color_gt, const R* transmittance, uint64_t n,
                  double eps, double* loss_rgb, double* loss_transmittance, R* d_rgb, R* d_transmittance,
                  int32_t mem) {
  TRY(check_ctx(c));
  if (n && (!rgb || !color_gt || !transmittance)) return set_err(DG_EINVAL, "null inputs");
  StageIo io{c, mem, {}, {}};
  const R *r, *g, *T;
  TRY(io.in(rgb, 3 * n, &r));
  TRY(io.in(color_gt, 3 * n, &g));
  TRY(io.in(transmittance, n, &T));
  double *lr, *lt;
  R *dr, *dt;
  TRY(io.out(loss_rgb, n, &lr));
  TRY(io.out(loss_transmittance, n, &lt));
  TRY(io.out(d_rgb, 3 * n, &dr));
  TRY(io.out(d_transmittance, n, &dt));
  launch_ray_losses(r, g, T, n, eps, lr, lt, dr, dt, c->stream);
  ++c->launches;
  return io.finish();
}

}  // namespace

extern "C" {

int dg_local_render(dg_ctx* c, const double* t, const double* delta, const float* sigma, const float* rgb,
                    const uint64_t* seg_off, uint64_t n_seg, const double* ray_t0, const double* ray_t1,
                    float* out_rgb, float* out_T, float* out_depth_sum, double* out_distortion,
                    int32_t mem) {
  return local_render_impl<float>(c, t, delta, sigma, rgb, seg_off, n_seg, ray_t0, ray_t1, out_rgb, out_T, out_depth_sum, out_distortion, mem);
}

int dg_local_render_f64(dg_ctx* c, const double* t, const double* delta, const double* sigma, const double* rgb,
                    const uint64_t* seg_off, uint64_t n_seg, const double* ray_t0, const double* ray_t1,
                    double* out_rgb, double* out_T, double* out_depth_sum, double* out_distortion,
                    double* out_cache, int32_t mem) {
  return local_render_impl<double>(c, t, delta, sigma, rgb, seg_off, n_seg, ray_t0, ray_t1, out_rgb, out_T,
                                   out_depth_sum, out_distortion, mem, out_cache);
}

int dg_local_render_backward(dg_ctx* c, const double* t, const double* delta, const float* sigma,
                             const float* rgb, const uint64_t* seg_off, uint64_t n_seg, const float* d_rgb,
                             const float* d_transmittance, const float* weight_upstream, float* sigma_grad,
                             float* rgb_grad, int32_t mem) {
  return local_render_backward_impl<float>(c, t, delta, sigma, rgb, seg_off, n_seg, d_rgb, d_transmittance, weight_upstream, sigma_grad, rgb_grad, mem);
}

int dg_local_render_backward_f64(dg_ctx* c, const double* t, const double* delta, const double* sigma,
                             const double* rgb, const uint64_t* seg_off, uint64_t n_seg, const double* d_rgb,
                             const double* d_transmittance, const double* weight_upstream, double* sigma_grad,
                             double* rgb_grad, int32_t mem) {
  return local_render_backward_impl<double>(c, t, delta, sigma, rgb, seg_off, n_seg, d_rgb, d_transmittance, weight_upstream, sigma_grad, rgb_grad, mem);
}

int dg_merge_forward(dg_ctx* c, const float* seg_rgb, const float* seg_transmittance,
                     const float* seg_depth_sum, const uint64_t* ray_off, uint64_t n_rays, float* rgb,
                     float* transmittance, float* depth, int32_t mem) {
  return merge_forward_impl<float>(c, seg_rgb, seg_transmittance, seg_depth_sum, ray_off, n_rays, rgb, transmittance, depth, mem);
}

int dg_merge_forward_f64(dg_ctx* c, const double* seg_rgb, const double* seg_transmittance,
                     const double* seg_depth_sum, const uint64_t* ray_off, uint64_t n_rays, double* rgb,
                     double* transmittance, double* depth, int32_t mem) {
  return merge_forward_impl<double>(c, seg_rgb, seg_transmittance, seg_depth_sum, ray_off, n_rays, rgb, transmittance, depth, mem);
}

int dg_merge_backward(dg_ctx* c, const float* seg_rgb, const float* seg_transmittance, const uint64_t* ray_off,
                      uint64_t n_rays, const float* d_rgb, const float* d_transmittance, float* seg_d_rgb,
                      float* seg_d_transmittance, int32_t mem) {
  return merge_backward_impl<float>(c, seg_rgb, seg_transmittance, ray_off, n_rays, d_rgb, d_transmittance, seg_d_rgb, seg_d_transmittance, mem);
}

int dg_merge_backward_f64(dg_ctx* c, const double* seg_rgb, const double* seg_transmittance, const uint64_t* ray_off,
                      uint64_t n_rays, const double* d_rgb, const double* d_transmittance, double* seg_d_rgb,
                      double* seg_d_transmittance, int32_t mem) {
  return merge_backward_impl<double>(c, seg_rgb, seg_transmittance, ray_off, n_rays, d_rgb, d_transmittance, seg_d_rgb, seg_d_transmittance, mem);
}

int dg_ray_losses(dg_ctx* c, const float* rgb, const float* color_gt, const float* transmittance, uint64_t n,
                  double eps, double* loss_rgb, double* loss_transmittance, float* d_rgb, float* d_transmittance,
                  int32_t mem) {
  return ray_losses_impl<float>(c, rgb, color_gt, transmittance, n, eps, loss_rgb, loss_transmittance, d_rgb, d_transmittance, mem);
}

int dg_ray_losses_f64(dg_ctx* c, const double* rgb, const double* color_gt, const double* transmittance, uint64_t n,
                  double eps, double* loss_rgb, double* loss_transmittance, double* d_rgb, double* d_transmittance,
                  int32_t mem) {
  return ray_losses_impl<double>(c, rgb, color_gt, transmittance, n, eps, loss_rgb, loss_transmittance, d_rgb, d_transmittance, mem);
}

int dg_distortion_loss(dg_ctx* c, const double* weights, const double* midpoints, const double* interval_lengths,
                       const uint64_t* seg_off, uint64_t n_seg, double* loss, double* grads, int32_t mem) {
  TRY(check_ctx(c));
  std::vector<uint64_t> off;
  TRY(host_offsets(c, seg_off, n_seg, mem, off));
  const uint64_t ns = off[n_seg];
  if (ns && (!weights || !midpoints || !interval_lengths)) return set_err(DG_EINVAL, "null inputs");
  StageIo io{c, mem, {}, {}};
  const double *w, *m, *ds;
  const uint64_t* doff;
  TRY(io.in(weights, ns, &w));
  TRY(io.in(midpoints, ns, &m));
  TRY(io.in(interval_lengths, ns, &ds));
  TRY(io.in(seg_off, n_seg + 1, &doff));
  double *ol, *og;
  TRY(io.out(loss, n_seg, &ol));
  TRY(io.out(grads, ns, &og));
  launch_distortion(w, m, ds, doff, n_seg, ol, og, c->stream);
  ++c->launches;
  return io.finish();
}

int dg_distortion_stats_f64(dg_ctx* c, const double* t, const double* delta, const double* cache,
                            const uint64_t* seg_off, uint64_t n_seg, const double* ray_t0, const double* ray_t1,
                            double* out, int32_t mem) {
  TRY(check_ctx(c));
  std::vector<uint64_t> off;
  TRY(host_offsets(c, seg_off, n_seg, mem, off));
  const uint64_t ns = off[n_seg];
  if (!out || (n_seg && (!ray_t0 || !ray_t1)) || (ns && (!t || !delta || !cache)))
    return set_err(DG_EINVAL, "null argument");
  StageIo io{c, mem, {}, {}};
  const double *dt, *dd, *dc, *t0, *t1;
  const uint64_t* doff;
  TRY(io.in(t, ns, &dt));
  TRY(io.in(delta, ns, &dd));
  TRY(io.in(cache, 2 * ns, &dc));
  TRY(io.in(seg_off, n_seg + 1, &doff));
  TRY(io.in(ray_t0, n_seg, &t0));
  TRY(io.in(ray_t1, n_seg, &t1));
  double* o;
  TRY(io.in(static_cast<const double*>(out), 3 * n_seg, const_cast<const double**>(&o)));
  if (mem != DG_MEM_DEVICE && n_seg) io.back.emplace_back(out, io.tmp.back().get(), 3 * n_seg * 8);
  launch_distortion_stats(dt, dd, dc, doff, n_seg, t0, t1, o, c->stream);
  ++c->launches;
  return io.finish();
}

int dg_ray_aabb(dg_ctx* c, const double* origin, const double* dir, uint64_t n, const double box_lo[3],
                const double box_hi[3], uint8_t* hit, double* t_near, double* t_far, int32_t mem) {
  TRY(check_ctx(c));
  if (!box_lo || !box_hi || (n && (!origin || !dir || !hit || !t_near || !t_far)))
    return set_err(DG_EINVAL, "null argument");
  StageIo io{c, mem, {}, {}};
  const double *o, *d;
  TRY(io.in(origin, 3 * n, &o));
  TRY(io.in(dir, 3 * n, &d));
  uint8_t* h;
  double *tn, *tf;
  TRY(io.out(hit, n, &h));
  TRY(io.out(t_near, n, &tn));
  TRY(io.out(t_far, n, &tf));
  launch_ray_aabb(o, d, n, box_lo, box_hi, h, tn, tf, c->stream);
  ++c->launches;
  return io.finish();
}

int dg_march_segment(dg_ctx* c, const double* t_enter, const double* t_exit, const uint64_t* interval_off,
                     const double* intervals, const uint64_t* ray_id, uint64_t n, double step, int32_t jitter,
                     uint64_t jitter_seed, uint64_t jitter_step, uint32_t* counts, const uint64_t* offsets,
                     double* t, double* delta, int32_t mem) {
  TRY(check_ctx(c));
  if (!(step > 0.0)) return set_err(DG_EINVAL, "march: step must be positive");  // render.cpp:13
  if (!counts && !t) return set_err(DG_EINVAL, "march: need counts or outputs");
  if (t && (!offsets || !delta)) return set_err(DG_EINVAL, "march: outputs need offsets and delta");
  std::vector<uint64_t> ivo;
  TRY(host_offsets(c, interval_off, n, mem, ivo));
  const uint64_t niv = ivo[n];
  if (niv && !intervals) return set_err(DG_EINVAL, "null intervals");
  if (n && (!t_enter || !t_exit)) return set_err(DG_EINVAL, "null segment bounds");
  StageIo io{c, mem, {}, {}};
  const double *te, *tx, *iv;
  const uint64_t *ivd, *rid, *od = nullptr;
  TRY(io.in(t_enter, n, &te));
  TRY(io.in(t_exit, n, &tx));
  TRY(io.in(interval_off, n + 1, &ivd));
  TRY(io.in(intervals, 2 * niv, &iv));
  TRY(io.in(ray_id, n, &rid));
  uint32_t* cnt;
  TRY(io.out(counts, n, &cnt));
  double *ot = nullptr, *odl = nullptr;
  if (t) {
    std::vector<uint64_t> oo;
    TRY(host_offsets(c, offsets, n, mem, oo));
    TRY(io.in(offsets, n + 1, &od));
    TRY(io.out(t, oo[n], &ot));
    TRY(io.out(delta, oo[n], &odl));
  }
  launch_march_segment(te, tx, ivd, iv, rid, n, step, jitter, jitter_seed, jitter_step, cnt, od, ot, odl,
                       c->stream);
  ++c->launches;
  return io.finish();
}

int dg_occupancy_skip(dg_ctx* c, const uint8_t* bits, const uint32_t shape[3], const double box_lo[3],
                      const double box_hi[3], const double* origin, const double* dir, const double* t0,
                      const double* t1, uint64_t n, uint32_t* counts, const uint64_t* offsets, double* intervals,
                      int32_t mem) {
  TRY(check_ctx(c));
  if (!bits || !shape || !box_lo || !box_hi) return set_err(DG_EINVAL, "null argument");
  if (!counts && !intervals) return set_err(DG_EINVAL, "occupancy_skip: need counts or outputs");
  if (intervals && !offsets) return set_err(DG_EINVAL, "occupancy_skip: outputs need offsets");
  if (n && (!origin || !dir || !t0 || !t1)) return set_err(DG_EINVAL, "null queries");
  const uint64_t cells = uint64_t(shape[0]) * shape[1] * shape[2];
  StageIo io{c, mem, {}, {}};
  const uint8_t* b;
  const double *o, *d, *a, *z;
  const uint64_t* od = nullptr;
  TRY(io.in(bits, cells, &b));
  TRY(io.in(origin, 3 * n, &o));
  TRY(io.in(dir, 3 * n, &d));
  TRY(io.in(t0, n, &a));
  TRY(io.in(t1, n, &z));
  uint32_t* cnt;
  TRY(io.out(counts, n, &cnt));
  double* iv = nullptr;
  if (intervals) {
    std::vector<uint64_t> oo;
    TRY(host_offsets(c, offsets, n, mem, oo));
    TRY(io.in(offsets, n + 1, &od));
    TRY(io.out(intervals, 2 * oo[n], &iv));
  }
  launch_occupancy_skip(b, shape, box_lo, box_hi, o, d, a, z, n, cnt, od, iv, c->stream);
  ++c->launches;
  return io.finish();
}

int dg_adam_update_f64(dg_ctx* c, double* params, const double* grads, double* m, double* v, uint64_t n,
                       uint64_t t, double lr, double beta1, double beta2, double eps, int32_t mem) {
  TRY(check_ctx(c));
  if (n && (!params || !grads || !m || !v)) return set_err(DG_EINVAL, "null argument");
  if (t == 0) return set_err(DG_EINVAL, "adam: t counts the steps taken, including this one (>= 1)");
  StageIo io{c, mem, {}, {}};
  const double* g;
  double *p, *dm, *dv;
  TRY(io.in(grads, n, &g));
  // in/out arrays: upload, update in place, read back
  const double *pi, *mi, *vi;
  TRY(io.in(static_cast<const double*>(params), n, &pi));
  TRY(io.in(static_cast<const double*>(m), n, &mi));
  TRY(io.in(static_cast<const double*>(v), n, &vi));
  p = const_cast<double*>(pi);
  dm = const_cast<double*>(mi);
  dv = const_cast<double*>(vi);
  if (mem != DG_MEM_DEVICE && n) {
    io.back.emplace_back(params, io.tmp[1].get(), n * 8);
    io.back.emplace_back(m, io.tmp[2].get(), n * 8);
    io.back.emplace_back(v, io.tmp[3].get(), n * 8);
  }
  const double bias1 = 1.0 - std::pow(beta1, double(t));
  const double bias2 = 1.0 - std::pow(beta2, double(t));
  launch_adam_f64(p, g, dm, dv, n, lr, beta1, beta2, eps, bias1, bias2, c->stream);
  ++c->launches;
  return io.finish();
}

int dg_adam_step(dg_ctx* c, double lr) {
  TRY(check_ctx(c));
  c->adam_t += 1;
  const double bias1 = 1.0 - std::pow(c->cfg.adam_beta1, double(c->adam_t));
  const double bias2 = 1.0 - std::pow(c->cfg.adam_beta2, double(c->adam_t));
  launch_adam(c->params.as<float>(), c->grads.as<float>(), c->adam_m.as<float>(), c->adam_v.as<float>(),
              c->n_params, float(lr), float(c->cfg.adam_beta1), float(c->cfg.adam_beta2),
              float(c->cfg.adam_eps), float(1.0 / bias1), float(1.0 / bias2), c->stream);
  ++c->launches;
  CU(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

// ---------------------------------------------------------------- introspection
int dg_last_items(dg_ctx* c, uint32_t p, dg_item_view* v) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (!c->have_last) return set_err(DG_EINVAL, "no step has run");
  const uint32_t nl = uint32_t(c->local.size());
  v->n_items = c->part_item_off[lp + 1] - c->part_item_off[lp];
  v->n_fine = c->field_off[lp + 1] - c->field_off[lp];
  v->n_coarse = c->field_off[nl + lp + 1] - c->field_off[nl + lp];
  return DG_OK;
}

int dg_last_item_data(dg_ctx* c, uint32_t p, uint64_t* ray_id, uint8_t* order, double* te, double* tx,
                      uint32_t* n_samples) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (!c->have_last) return set_err(DG_EINVAL, "no step has run");
  cudaStream_t s = c->stream;
  const uint32_t a = c->part_item_off[lp], n = c->part_item_off[lp + 1] - a, NI = c->n_items;
  std::vector<RayRec> rec;
  std::vector<uint8_t> ord;
  std::vector<double> vte, vtx;
  std::vector<uint32_t> cnt;
  TRY(d2h(rec, c->items_rec + a, n, s));
  TRY(d2h(ord, c->it_order.as<uint8_t>() + a, n, s));
  TRY(d2h(vte, c->it_te.as<double>() + a, n, s));
  TRY(d2h(vtx, c->it_tx.as<double>() + a, n, s));
  TRY(d2h(cnt, c->it_cnt.p, 2ull * NI, s));
  CU(cudaStreamSynchronize(s));
  for (uint32_t i = 0; i < n; ++i) {
    if (ray_id) ray_id[i] = rec[i].ray_id;
    if (order) order[i] = ord[i];
    if (te) te[i] = vte[i];
    if (tx) tx[i] = vtx[i];
    if (n_samples) n_samples[i] = cnt[a + i] + cnt[NI + a + i];
  }
  return DG_OK;
}

int dg_last_samples(dg_ctx* c, uint32_t p, double* t, double* delta, uint8_t* cascade) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (!c->have_last) return set_err(DG_EINVAL, "no step has run");
  cudaStream_t s = c->stream;
  const uint32_t NI = c->n_items;
  const uint64_t NS = uint64_t(c->n_fine) + c->n_coarse;
  std::vector<uint32_t> cnt, off, ncb;
  std::vector<double> st, sd;
  TRY(d2h(cnt, c->it_cnt.p, 2ull * NI, s));
  TRY(d2h(off, c->it_off.p, 2ull * NI, s));
  TRY(d2h(ncb, c->it_ncb.p, NI, s));
  TRY(d2h(st, c->s_t.p, NS, s));
  TRY(d2h(sd, c->s_delta.p, NS, s));
  CU(cudaStreamSynchronize(s));
  uint64_t k = 0;
  auto put = [&](uint32_t idx, uint8_t casc) {
    t[k] = st[idx];
    delta[k] = sd[idx];
    if (cascade) cascade[k] = casc;
    ++k;
  };
  for (uint32_t i = c->part_item_off[lp]; i < c->part_item_off[lp + 1]; ++i) {
    for (uint32_t j = 0; j < ncb[i]; ++j) put(off[NI + i] + j, 1);
    for (uint32_t j = 0; j < cnt[i]; ++j) put(off[i] + j, 0);
    for (uint32_t j = ncb[i]; j < cnt[NI + i]; ++j) put(off[NI + i] + j, 1);
  }
  return DG_OK;
}

// Per-sample state of the last training step, in dg_last_samples order: the normalised field
// position the march wrote and the encode read (worker.cpp:46), the encoded features
// (k_encode_fwd), the field outputs (k_mlp_fwd*: sigma, rgb), the upstream gradient of the
// merge / compositing backward (k_merge_backward: dsigma, drgb) and the encoding's upstream
// (k_mlp_bwd*: dL/dfeatures) and the forward's ReLU / clip mask words (tcgen05 path, the layout
// of kernels_mlp_tc.cu's k_mlp_fwd_tc).  Every output is optional.
int dg_last_sample_data(dg_ctx* c, uint32_t p, double* pos, float* features, float* field_out,
                        float* upstream, float* d_features, uint32_t* masks) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (!c->have_last) return set_err(DG_EINVAL, "no step has run");
  if (pos && !c->enc_pcache) return set_err(DG_EINVAL, "position cache disabled (DG_ENC_PCACHE=0)");
  cudaStream_t s = c->stream;
  const uint32_t NI = c->n_items, L = c->cfg.grid_levels;
  const uint64_t NS = uint64_t(c->n_fine) + c->n_coarse;
  std::vector<uint32_t> cnt, off, ncb;
  std::vector<double> hp;
  std::vector<float> hx, ho, hg, hdx;
  TRY(d2h(cnt, c->it_cnt.p, 2ull * NI, s));
  TRY(d2h(off, c->it_off.p, 2ull * NI, s));
  TRY(d2h(ncb, c->it_ncb.p, NI, s));
  if (pos) TRY(d2h(hp, c->s_p.p, 3 * NS, s));
  if (features) TRY(d2h(hx, c->s_X.p, 2ull * L * NS, s));
  if (field_out) TRY(d2h(ho, c->s_out.p, 4 * NS, s));
  if (upstream) TRY(d2h(hg, c->ordered ? c->s_grad_ord.p : c->s_grad.p, 4 * NS, s));
  if (d_features) TRY(d2h(hdx, c->s_dX.p, 2ull * L * NS, s));
  std::vector<uint32_t> hm;
  if (masks) {
    if (!c->mlp_impl) return set_err(DG_EINVAL, "masks exist on the tcgen05 path only");
    TRY(d2h(hm, c->s_mask.p, 7 * NS, s));
  }
  // positions, features, their gradients and the masks are in sample order when the step
  // ordered its samples (s_perm: sorted slot -> march sample); map them back
  std::vector<uint32_t> perm, inv;
  if (c->ordered) {
    TRY(d2h(perm, c->s_perm.p, NS, s));
  }
  CU(cudaStreamSynchronize(s));
  if (c->ordered) {
    inv.assign(NS, 0);
    for (uint64_t j = 0; j < NS; ++j) inv[perm[j]] = uint32_t(j);
  }
  uint64_t k = 0;
  auto put = [&](uint64_t idx) {
    const uint64_t o = c->ordered ? inv[idx] : idx;
    for (int a = 0; a < 3 && pos; ++a) pos[3 * k + a] = hp[a * NS + o];
    for (uint32_t l = 0; l < L; ++l)
      for (int f = 0; f < 2; ++f) {
        if (features) features[(k * L + l) * 2 + f] = hx[(l * NS + o) * 2 + f];
        if (d_features) d_features[(k * L + l) * 2 + f] = hdx[(l * NS + o) * 2 + f];
      }
    for (int a = 0; a < 4; ++a) {
      if (field_out) field_out[4 * k + a] = ho[4 * idx + a];
      if (upstream) upstream[4 * k + a] = hg[4 * o + a];
    }
    for (int w = 0; w < 7 && masks; ++w) masks[7 * k + w] = hm[w * NS + o];
    ++k;
  };
  for (uint32_t i = c->part_item_off[lp]; i < c->part_item_off[lp + 1]; ++i) {
    for (uint32_t j = 0; j < ncb[i]; ++j) put(off[NI + i] + j);
    for (uint32_t j = 0; j < cnt[i]; ++j) put(off[i] + j);
    for (uint32_t j = ncb[i]; j < cnt[NI + i]; ++j) put(off[NI + i] + j);
  }
  return DG_OK;
}

int dg_last_partials(dg_ctx* c, uint32_t p, float* rgb, float* transmittance) {
  uint32_t lp;
  TRY(check_part(c, p, &lp));
  if (!c->have_last) return set_err(DG_EINVAL, "no step has run");
  const uint32_t a = c->part_item_off[lp], n = c->part_item_off[lp + 1] - a;
  std::vector<float4> v;
  TRY(d2h(v, c->it_partial.as<float4>() + a, n, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (uint32_t i = 0; i < n; ++i) {
    rgb[3 * i] = v[i].x;
    rgb[3 * i + 1] = v[i].y;
    rgb[3 * i + 2] = v[i].z;
    transmittance[i] = std::exp(-v[i].w);
  }
  return DG_OK;
}

int dg_kernel_launches(const dg_ctx* c, uint64_t* n) {
  TRY(check_ctx(c));
  *n = c->launches;
  return DG_OK;
}

int dg_enable_stage_timing(dg_ctx* c, int enable) {
  TRY(check_ctx(c));
  c->timing = enable != 0;
  return DG_OK;
}

int dg_last_stage_times(dg_ctx* c, dg_stage_times* t) {
  TRY(check_ctx(c));
  *t = c->times;
  return DG_OK;
}

int dg_selftest_tcgen05(const float* A, const float* B, const float* X, float* Y0, float* Y1,
                        float* Y2) {
  DBuf a, b, x, y0, y1, y2;
  cudaStream_t s = nullptr;
  TRY(upload(a, A, 128 * 64 * 4, s));
  TRY(upload(b, B, 64 * 64 * 4, s));
  TRY(upload(x, X, 128 * 32 * 4, s));
  TRY(y0.ensure(128 * 64 * 4));
  TRY(y1.ensure(128 * 64 * 4));
  TRY(y2.ensure(64 * 32 * 4));
  if (tc_selftest(a.as<float>(), b.as<float>(), x.as<float>(), y0.as<float>(), y1.as<float>(),
                  y2.as<float>(), s) != 0)
    return set_err(DG_ECUDA, "tcgen05 self-test launch failed");
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(Y0, y0.p, 128 * 64 * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(Y1, y1.p, 128 * 64 * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(Y2, y2.p, 64 * 32 * 4, cudaMemcpyDeviceToHost));
  return DG_OK;
}

int dg_get_stream(dg_ctx* c, void** stream) {
  TRY(check_ctx(c));
  *stream = (void*)c->stream;
  return DG_OK;
}

int dg_set_stream(dg_ctx* c, void* stream) {
  TRY(check_ctx(c));
  CU(cudaSetDevice(c->device));
  CU(cudaStreamSynchronize(c->stream));  // work queued on the previous stream is done
  c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
  return DG_OK;
}

int dg_synchronize(dg_ctx* c) {
  TRY(check_ctx(c));  // orders the stream after the last step's Adam
  CU(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

int dg_fence(dg_ctx* c) { return check_ctx(c); }

}  // extern "C"
