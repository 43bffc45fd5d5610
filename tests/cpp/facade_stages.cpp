// The facade's stage-level API (include/distgrid/*.hpp) used as the reference's per-function API
// is used: HashGrid / FieldParams built from an Rng, query_density / query_color /
// field_backward per sample and batched, losses, LrSchedule, AdamState, segment_ray.  Writes
// every input and output as raw doubles to argv[1]; tests/test_gpu_facade.py checks them against
// the oracle (fp64) at the bars of the parity suite.
#include <cstdio>
#include <vector>

#include "distgrid_b200/distgrid.hpp"

using namespace distgrid;

namespace {
std::vector<double> out;
void put(double v) { out.push_back(v); }
void put(std::span<const double> v) { out.insert(out.end(), v.begin(), v.end()); }
void put(const Vec3& v) {
  put(v.x);
  put(v.y);
  put(v.z);
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const int N = 64;
  Rng rng(2024);
  GridConfig gc;
  gc.levels = 8;
  gc.table_length = 1u << 12;
  gc.base_resolution = 16;
  gc.max_resolution = 128;
  Rng init(7);
  FieldParams fp(CascadeLevel::Fine, gc, 16, init);
  // a trained-like table range, so the features are not all ~1e-4
  for (std::span<double> a : fp.grid.parameter_arrays())
    for (double& v : a) v = rng.uniform(-0.5, 0.5);

  std::vector<Vec3> pts(N), dirs(N);
  std::vector<double> app(size_t(N) * 16);
  for (int i = 0; i < N; ++i) {
    pts[i] = Vec3(rng.uniform(), rng.uniform(), rng.uniform());
    dirs[i] = normalize(Vec3(rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, 1)));
  }
  for (double& a : app) a = rng.uniform(-1, 1);
  for (const Vec3& p : pts) put(p);
  for (const Vec3& d : dirs) put(d);
  put(app);
  for (std::span<double> a : fp.parameter_arrays()) put(a);

  // HashGrid::encode, batched
  put(fp.grid.encode(pts));
  // per-sample query_density / query_color (the reference's call sequence)
  std::vector<FieldSampleCache> caches(N);
  std::vector<double> sigma(N);
  for (int i = 0; i < N; ++i) {
    const DensityResult d = query_density(pts[i], fp, &caches[i]);
    sigma[i] = d.sigma;
    put(d.sigma);
    put(std::span<const double>(d.feature));
    const Vec3 rgb = query_color(d.feature, dirs[i], std::span<const double>(app).subspan(size_t(i) * 16, 16), fp,
                                 &caches[i]);
    put(rgb);
  }
  // field_backward: half per sample through the caches, half batched
  std::vector<double> sg(N);
  std::vector<Vec3> cg(N);
  for (int i = 0; i < N; ++i) {
    sg[i] = rng.uniform(-1, 1);
    cg[i] = Vec3(rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, 1));
  }
  put(sg);
  for (const Vec3& c : cg) put(c);
  FieldGrads grads = make_field_grads(fp);
  for (int i = 0; i < N / 2; ++i) field_backward(fp, caches[i], sigma[i], sg[i], cg[i], grads);
  const size_t h = N / 2;
  field_backward(fp, std::span<const Vec3>(pts).subspan(h), std::span<const Vec3>(dirs).subspan(h),
                 std::span<const double>(app).subspan(h * 16), std::span<const double>(sg).subspan(h),
                 std::span<const Vec3>(cg).subspan(h), grads);
  for (std::span<double> a : grads.arrays()) put(a);

  // losses (train.cpp:8-75)
  std::vector<Vec3> ra(8), rb(8);
  for (int i = 0; i < 8; ++i) {
    ra[i] = Vec3(rng.uniform(), rng.uniform(), rng.uniform());
    rb[i] = Vec3(rng.uniform(), rng.uniform(), rng.uniform());
    put(ra[i]);
    put(rb[i]);
  }
  put(loss_rgb(ra, rb));
  put(loss_rgb_grad(ra[0], rb[0]));
  std::vector<double> T{0.0, 0.3, 0.999999999, 1.0};
  put(T);
  put(loss_transmittance(T));
  for (double t : T) put(loss_transmittance_grad(t));
  std::vector<double> w(10), s(10), ds(10), dg(10);
  double acc = 0.0;
  for (int k = 0; k < 10; ++k) {
    w[k] = rng.uniform(0.0, 0.2);
    acc += rng.uniform(0.01, 0.1);
    s[k] = acc;
    ds[k] = rng.uniform(0.01, 0.05);
  }
  put(w);
  put(s);
  put(ds);
  put(loss_distortion(w, s, ds));
  loss_distortion_grad(w, s, ds, dg);
  put(dg);
  // LrSchedule and two Adam steps on one array (train.cpp:77-115)
  LrSchedule lr{0.05, 0.005, 1000};
  for (uint64_t st : {0ull, 1ull, 500ull, 999ull, 1000ull}) put(lr.at(st));
  const size_t sizes[1] = {5};
  AdamState adam(sizes);
  std::vector<double> p{0.1, -0.2, 0.3, 0.0, 1.0}, g1{0.5, -1.0, 0.0, 2.0, 1e-3}, g2{-0.5, 0.25, 1.0, 0.0, 1e-3};
  put(p);
  put(g1);
  put(g2);
  for (const std::vector<double>* g : {&g1, &g2}) {
    const std::span<double> ps[1] = {p};
    const std::span<const double> gs[1] = {*g};
    adam.step(ps, gs, 0.01);
  }
  put(p);
  put(adam.first_moments()[0]);
  put(adam.second_moments()[0]);
  put(double(adam.step_count()));
  // segment_ray on a 2 x 2 manifest (partition.cpp:254-296)
  const Aabb inner(Vec3(0.3, 0.25, 0.0), Vec3(1.6, 1.8, 0.8)), outer(Vec3(0, 0, 0), Vec3(2, 2, 1));
  const PartitionManifest m = split_regions(inner, outer, 2, 2, 0.0);
  for (int i = 0; i < 32; ++i) {
    Ray r;
    r.origin = Vec3(rng.uniform(-0.5, 2.5), rng.uniform(-0.5, 2.5), 1.2);
    r.dir = normalize(Vec3(rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, -0.2)));
    r.pixel_id = uint64_t(i);
    const std::vector<RaySegment> segs = segment_ray(r, m);
    put(r.origin);
    put(r.dir);
    put(double(segs.size()));
    for (int k = 0; k < 4; ++k) {
      const bool v = k < int(segs.size());
      put(v ? double(segs[k].region_id) : -1.0);
      put(v ? segs[k].t_enter : 0.0);
      put(v ? segs[k].t_exit : 0.0);
    }
  }
  std::FILE* f = std::fopen(argv[1], "wb");
  std::fwrite(out.data(), sizeof(double), out.size(), f);
  std::fclose(f);
  std::printf("facade_stages wrote %zu doubles\n", out.size());
  return 0;
}
