// checkpoint.cpp — §8f row 3: .dgcw checkpoint interop with the reference.
//
// Byte layout of save_worker_checkpoint / load_worker_checkpoint (checkpoint.cpp:241-283,
// version 1, little endian):
//   "DGCW" u32 version  u64 config_hash  u64 step  u32 region_id
//   field(fine) field(coarse)   field = u8 cascade, u32 appearance_dim, grid, mlp(density), mlp(colour)
//     grid = u32 levels, u32 table_length, u32 features, u32 base_res, u32 max_res, f64 aspect[3],
//            per level: u32 index, u32 nx, ny, nz, u8 mapping, u32 features, f32_array table
//     mlp  = u8 activation, u32 n_layers, per layer: u32 out, u32 in, f32_array W, f32_array b
//   occupancy(fine) occupancy(coarse) = f64 box lo[3] hi[3], u32 shape[3], f64 decay,
//                                       f32_array density, f32 threshold
//   u64 adam step_count, u32 n_arrays, n_arrays x f64_array m, n_arrays x f64_array v
// f32_array / f64_array = u64 count + values.  Host code over the public C ABI getters.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "distgrid_b200.h"

namespace dg {
int set_error(int code, const char* msg);
}

namespace {

constexpr uint32_t kVersion = 1;

struct Writer {
  FILE* f = nullptr;
  bool ok = true;
  void raw(const void* p, size_t n) {
    if (n && fwrite(p, 1, n, f) != n) ok = false;
  }
  void u8(uint8_t v) { raw(&v, 1); }
  void u32(uint32_t v) { raw(&v, 4); }
  void u64(uint64_t v) { raw(&v, 8); }
  void f64(double v) { raw(&v, 8); }
  void f32_array(const float* v, uint64_t n) {
    u64(n);
    raw(v, n * 4);
  }
  void f64_array_from_f32(const float* v, uint64_t n) {
    u64(n);
    std::vector<double> d(v, v + n);
    raw(d.data(), n * 8);
  }
};

struct Reader {
  FILE* f = nullptr;
  bool ok = true;
  void raw(void* p, size_t n) {
    if (n && fread(p, 1, n, f) != n) ok = false;
  }
  uint8_t u8() {
    uint8_t v = 0;
    raw(&v, 1);
    return v;
  }
  uint32_t u32() {
    uint32_t v = 0;
    raw(&v, 4);
    return v;
  }
  uint64_t u64() {
    uint64_t v = 0;
    raw(&v, 8);
    return v;
  }
  double f64() {
    double v = 0;
    raw(&v, 8);
    return v;
  }
  // f32_array into dst (expected count n); false on a count mismatch
  bool f32_array(float* dst, uint64_t n) {
    const uint64_t m = u64();
    if (!ok || m != n) return false;
    raw(dst, n * 4);
    return ok;
  }
  bool f64_array_to_f32(float* dst, uint64_t n) {
    const uint64_t m = u64();
    if (!ok || m != n) return false;
    std::vector<double> d(n);
    raw(d.data(), n * 8);
    for (uint64_t i = 0; i < n; ++i) dst[i] = float(d[i]);
    return ok;
  }
};

struct PartitionView {  // what the file needs about one partition, from the C ABI
  dg_run_config cfg{};
  double box[2][2][3]{};  // [cascade][lo/hi][axis]
  std::vector<uint32_t> shapes[2], modes[2];
  std::vector<dg_array_desc> arrays;
  uint64_t n_params = 0;
  uint32_t occ_shape[2][3]{};
};

int view(dg_ctx* c, uint32_t p, PartitionView& v) {
  int rc = dg_get_config(c, &v.cfg);
  if (rc) return rc;
  rc = dg_region_boxes(c, p, v.box[0][0], v.box[0][1], v.box[1][0], v.box[1][1]);
  if (rc) return rc;
  const uint32_t L = v.cfg.grid_levels;
  for (uint32_t cas = 0; cas < 2; ++cas) {
    v.shapes[cas].resize(3 * L);
    v.modes[cas].resize(L);
    if ((rc = dg_grid_levels(c, p, cas, v.shapes[cas].data(), v.modes[cas].data(), nullptr))) return rc;
    if ((rc = dg_occupancy_shape(c, p, cas, v.occ_shape[cas]))) return rc;
  }
  if ((rc = dg_param_count(c, p, &v.n_params))) return rc;
  uint32_t n = 0;
  v.arrays.resize(2 * (L + 10));
  if ((rc = dg_param_layout(c, p, v.arrays.data(), uint32_t(v.arrays.size()), &n))) return rc;
  v.arrays.resize(n);
  return DG_OK;
}

// The arrays of one cascade in FieldParams::parameter_arrays order: L tables, then density
// W0 b0 W1 b1, colour W0 b0 W1 b1 W2 b2 (field.cpp:203-208).
std::vector<const dg_array_desc*> cascade_arrays(const PartitionView& v, uint32_t cas) {
  std::vector<const dg_array_desc*> out;
  for (const dg_array_desc& a : v.arrays)
    if (a.cascade == cas) out.push_back(&a);
  return out;
}

struct MlpShape {
  uint32_t act;
  std::vector<std::pair<uint32_t, uint32_t>> layers;  // (out, in)
};

void mlp_shapes(const PartitionView& v, uint32_t cas, MlpShape& dens, MlpShape& col) {
  const uint32_t enc = v.cfg.grid_levels * v.cfg.grid_features, cin = 15 + 16 + v.cfg.appearance_dim;
  dens.act = 1;  // ReLU (field.cpp:189-201)
  dens.layers = {{64, enc}, {16, 64}};
  col.act = cas == 0 ? 1 : 2;  // ReLU fine, Sigmoid coarse
  col.layers = {{64, cin}, {64, 64}, {3, 64}};
}

}  // namespace

extern "C" int dg_save_checkpoint(dg_ctx* c, uint32_t p, uint64_t config_hash, const char* path) {
  PartitionView v;
  int rc = view(c, p, v);
  if (rc) return rc;
  std::vector<float> params(v.n_params), m(v.n_params), s(v.n_params);
  uint64_t adam_steps = 0, step = 0;
  if ((rc = dg_get_params(c, p, params.data())) || (rc = dg_get_adam(c, p, m.data(), s.data(), &adam_steps)) ||
      (rc = dg_get_step(c, &step)))
    return rc;
  Writer w;
  w.f = fopen(path, "wb");
  if (!w.f) return dg::set_error(DG_EINVAL, (std::string("checkpoint: cannot open for writing: ") + path).c_str());
  w.raw("DGCW", 4);
  w.u32(kVersion);
  w.u64(config_hash);
  w.u64(step);
  w.u32(p);
  const uint32_t L = v.cfg.grid_levels;
  for (uint32_t cas = 0; cas < 2; ++cas) {
    const auto arr = cascade_arrays(v, cas);
    w.u8(uint8_t(cas));
    w.u32(v.cfg.appearance_dim);
    w.u32(L);
    w.u32(1u << (cas == 0 ? v.cfg.fine_table_log2 : v.cfg.coarse_table_log2));
    w.u32(v.cfg.grid_features);
    w.u32(v.cfg.base_resolution);
    w.u32(v.cfg.max_resolution);
    for (int a = 0; a < 3; ++a) w.f64(v.box[cas][1][a] - v.box[cas][0][a]);  // Aabb::extent
    for (uint32_t l = 0; l < L; ++l) {
      w.u32(l);
      for (int a = 0; a < 3; ++a) w.u32(v.shapes[cas][3 * l + a]);
      w.u8(uint8_t(v.modes[cas][l]));
      w.u32(v.cfg.grid_features);
      w.f32_array(params.data() + arr[l]->offset, arr[l]->size);
    }
    MlpShape dens, col;
    mlp_shapes(v, cas, dens, col);
    uint32_t k = L;
    for (const MlpShape* mlp : {&dens, &col}) {
      w.u8(uint8_t(mlp->act));
      w.u32(uint32_t(mlp->layers.size()));
      for (const auto& [out, in] : mlp->layers) {
        w.u32(out);
        w.u32(in);
        w.f32_array(params.data() + arr[k]->offset, arr[k]->size);
        w.f32_array(params.data() + arr[k + 1]->offset, arr[k + 1]->size);
        k += 2;
      }
    }
  }
  for (uint32_t cas = 0; cas < 2; ++cas) {
    for (int h = 0; h < 2; ++h)
      for (int a = 0; a < 3; ++a) w.f64(v.box[cas][h][a]);
    const uint32_t* sh = v.occ_shape[cas];
    for (int a = 0; a < 3; ++a) w.u32(sh[a]);
    w.f64(v.cfg.occ_decay);
    std::vector<float> den(uint64_t(sh[0]) * sh[1] * sh[2]);
    double thr = 0.0;
    if ((rc = dg_get_occupancy_density(c, p, cas, den.data(), &thr))) {
      fclose(w.f);
      return rc;
    }
    w.f32_array(den.data(), den.size());
    const float t32 = float(thr);
    w.raw(&t32, 4);
  }
  w.u64(adam_steps);
  w.u32(uint32_t(v.arrays.size()));
  for (const float* src : {m.data(), s.data()})
    for (const dg_array_desc& a : v.arrays) w.f64_array_from_f32(src + a.offset, a.size);
  const bool ok = w.ok && fclose(w.f) == 0;
  if (!ok) return dg::set_error(DG_EINVAL, "checkpoint: write failed");
  return DG_OK;
}

extern "C" int dg_load_checkpoint(dg_ctx* c, uint32_t p, const char* path, uint64_t* config_hash) {
  PartitionView v;
  int rc = view(c, p, v);
  if (rc) return rc;
  Reader r;
  r.f = fopen(path, "rb");
  if (!r.f) return dg::set_error(DG_EINVAL, (std::string("checkpoint: cannot open: ") + path).c_str());
  auto bad = [&](const char* why) {
    fclose(r.f);
    return dg::set_error(DG_EINVAL, (std::string("checkpoint: ") + why).c_str());
  };
  char magic[4];
  r.raw(magic, 4);
  if (!r.ok || std::memcmp(magic, "DGCW", 4) != 0) return bad("bad magic");
  if (r.u32() != kVersion) return bad("unsupported version");
  const uint64_t hash = r.u64();
  const uint64_t step = r.u64();
  if (r.u32() != p) return bad("region mismatch");  // Worker::load_state (worker.cpp:616-617)
  std::vector<float> params(v.n_params, 0.0f), m(v.n_params), s(v.n_params);
  const uint32_t L = v.cfg.grid_levels;
  for (uint32_t cas = 0; cas < 2; ++cas) {
    const auto arr = cascade_arrays(v, cas);
    if (r.u8() != cas || r.u32() != v.cfg.appearance_dim) return bad("field header mismatch");
    const uint32_t T = 1u << (cas == 0 ? v.cfg.fine_table_log2 : v.cfg.coarse_table_log2);
    if (r.u32() != L || r.u32() != T || r.u32() != v.cfg.grid_features || r.u32() != v.cfg.base_resolution ||
        r.u32() != v.cfg.max_resolution)
      return bad("grid config mismatch");
    for (int a = 0; a < 3; ++a) r.f64();  // aspect: only its ratios matter; shapes are checked
    for (uint32_t l = 0; l < L; ++l) {
      if (r.u32() != l) return bad("level index out of order");
      for (int a = 0; a < 3; ++a)
        if (r.u32() != v.shapes[cas][3 * l + a]) return bad("level shape does not match its config");
      if (r.u8() != v.modes[cas][l] || r.u32() != v.cfg.grid_features) return bad("level mode mismatch");
      if (!r.f32_array(params.data() + arr[l]->offset, arr[l]->size)) return bad("table size mismatch");
    }
    MlpShape dens, col;
    mlp_shapes(v, cas, dens, col);
    uint32_t k = L;
    for (const MlpShape* mlp : {&dens, &col}) {
      if (r.u8() != mlp->act || r.u32() != mlp->layers.size()) return bad("mlp header mismatch");
      for (const auto& [out, in] : mlp->layers) {
        if (r.u32() != out || r.u32() != in) return bad("layer shape mismatch");
        if (!r.f32_array(params.data() + arr[k]->offset, arr[k]->size) ||
            !r.f32_array(params.data() + arr[k + 1]->offset, arr[k + 1]->size))
          return bad("layer shape mismatch");
        k += 2;
      }
    }
  }
  std::vector<float> den[2];
  double thr[2];
  for (uint32_t cas = 0; cas < 2; ++cas) {
    for (int h = 0; h < 6; ++h) r.f64();
    const uint32_t* sh = v.occ_shape[cas];
    for (int a = 0; a < 3; ++a)
      if (r.u32() != sh[a]) return bad("occupancy shape mismatch");
    r.f64();  // decay: from the run config
    den[cas].resize(uint64_t(sh[0]) * sh[1] * sh[2]);
    if (!r.f32_array(den[cas].data(), den[cas].size())) return bad("occupancy density size mismatch");
    float t32;
    r.raw(&t32, 4);
    thr[cas] = double(t32);
  }
  const uint64_t adam_steps = r.u64();
  if (r.u32() != v.arrays.size()) return bad("adam array count mismatch");
  for (float* dst : {m.data(), s.data()})
    for (const dg_array_desc& a : v.arrays)
      if (!r.f64_array_to_f32(dst + a.offset, a.size)) return bad("adam array size mismatch");
  if (!r.ok) return bad("truncated file");
  fclose(r.f);
  if ((rc = dg_set_params(c, p, params.data())) || (rc = dg_set_adam(c, p, m.data(), s.data(), adam_steps)) ||
      (rc = dg_set_step(c, step)))
    return rc;
  for (uint32_t cas = 0; cas < 2; ++cas)
    if ((rc = dg_set_occupancy_density(c, p, cas, den[cas].data(), thr[cas]))) return rc;
  if (config_hash) *config_hash = hash;
  return DG_OK;
}
