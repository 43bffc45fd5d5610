// Phase-clock trace of k_mlp_bwd_tc on synthetic data (diagnostic; not part of the library).
// Build: make -C tools/trace   Run (GPU): tools/trace/trace_mlp
// Prints, per backward stage, the mean cycles of: epilogue (MMA done -> barrier entry),
// barrier (entry -> exit, incl. MMA issue by thread 0) and MMA wait (exit -> MMA done).
#define DG_TRACE_MLP 1
#include "../../paper_2405_04416_b200/csrc/kernels_mlp_tc.cu"

#include <cstdio>
#include <random>
#include <vector>

using namespace dg;

int main() {
  const int L = 16, app = 16, cin = 31 + app;
  const uint32_t tiles_per_cta = 32, ctas = 148;
  const uint64_t n = uint64_t(tiles_per_cta) * ctas * 128;
  FieldDesc fd{};
  fd.L = L;
  fd.coarse = 0;
  fd.app_dim = app;
  fd.base = 0;
  uint64_t o = 0;
  auto add = [&](uint64_t& f, uint64_t sz) { f = o; o += sz; };
  add(fd.dw0, 64 * 32); add(fd.db0, 64); add(fd.dw1, 16 * 64); add(fd.db1, 16);
  add(fd.cw0, 64 * cin); add(fd.cb0, 64); add(fd.cw1, 64 * 64); add(fd.cb1, 64);
  add(fd.cw2, 3 * 64); add(fd.cb2, 3);
  fd.size = o;
  std::mt19937 rng(1);
  std::uniform_real_distribution<float> U(-0.3f, 0.3f);
  std::vector<float> params(o);
  for (auto& v : params) v = U(rng);
  std::vector<float> X(n * 32);
  for (auto& v : X) v = U(rng);
  std::vector<float4> gin(n);
  for (auto& v : gin) v = make_float4(U(rng), U(rng), U(rng), U(rng));
  const uint32_t n_items = 4096;
  std::vector<RayRec> rec(n_items);
  for (auto& r : rec) {
    r = RayRec{};
    r.d[0] = 0.6; r.d[1] = 0.0; r.d[2] = -0.8;
    r.img = 0;
  }
  std::vector<uint32_t> item(n);
  for (uint64_t i = 0; i < n; ++i) item[i] = uint32_t((i / 120) % n_items);
  std::vector<float> appt(app);
  for (auto& v : appt) v = U(rng);
  uint32_t foff[2] = {0, uint32_t(n)}, toff[2] = {0, uint32_t(n / 128)};
  auto up = [](const void* h, size_t b) { void* d; cudaMalloc(&d, b); cudaMemcpy(d, h, b, cudaMemcpyHostToDevice); return d; };
  MlpLaunch m{};
  m.fields = (const FieldDesc*)up(&fd, sizeof fd);
  m.n_fields = 1;
  m.field_off = (const uint32_t*)up(foff, 8);
  m.tile_off = (const uint32_t*)up(toff, 8);
  m.n_tiles = uint32_t(n / 128);
  m.X = (const float*)up(X.data(), X.size() * 4);
  m.x_stride = n;
  m.levels = L;
  m.rec = (const RayRec*)up(rec.data(), rec.size() * sizeof(RayRec));
  m.s_item = (const uint32_t*)up(item.data(), n * 4);
  m.app_table = (const float*)up(appt.data(), app * 4);
  m.params = (const float*)up(params.data(), o * 4);
  void* g; cudaMalloc(&g, o * 4); cudaMemset(g, 0, o * 4);
  m.grads = (float*)g;
  m.grad_in = (const float4*)up(gin.data(), n * 16);
  void* dx; cudaMalloc(&dx, n * 32 * 4);
  m.dX = (float*)dx;
  // the forward's ReLU / clip masks (every ReLU unit on, nothing clipped) and outputs
  std::vector<uint32_t> masks(n * 7, 0xffffffffu);
  for (uint64_t i = 0; i < n; ++i) masks[6 * n + i] = 0u;
  m.masks = (uint32_t*)up(masks.data(), masks.size() * 4);
  std::vector<float4> outs(n);
  std::uniform_real_distribution<float> U01(0.05f, 0.95f);
  for (auto& v : outs) v = make_float4(U01(rng), U01(rng), U01(rng), U01(rng));
  m.out = (float4*)up(outs.data(), n * 16);
  m.out_tile = m.out;
  void* tr; cudaMalloc(&tr, 64 * 2 * 32 * 8); cudaMemset(tr, 0, 64 * 2 * 32 * 8);
  m.trace = (unsigned long long*)tr;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    launch_mlp_bwd_tc(m, ctas, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("k_mlp_bwd_tc %llu samples: %.3f ms (%.2f us/tile/CTA)  err=%s\n", (unsigned long long)n, ms,
           ms * 1000.0 / tiles_per_cta, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<unsigned long long> t(64 * 2 * 32);
  cudaMemcpy(t.data(), tr, t.size() * 8, cudaMemcpyDeviceToHost);
  // points per tile: [sync_in, sync_out, mma_done] x 9 stages (the output layer is not
  // recomputed: B1's colour-head adjoint runs in the F4 epilogue)
  constexpr int NST = 9;
  const char* names[NST] = {"F1 x.Wd0", "F2 h1.Wd1", "F3 cin.Wc0", "F4 c1.Wc1",
                            "B1 g5", "B2 G4", "B3 G3", "B4 G2", "B5 G1"};
  for (int who = 0; who < 2; ++who) {
    printf("thread %d: stage  epi_before  barrier+issue  mma_wait   (cycles, mean over tiles 2..30)\n", who ? 480 : 0);
    double tot = 0;
    for (int st = 0; st < NST; ++st) {
      double e = 0, bi = 0, w = 0;
      int cnt = 0;
      for (int tile = 2; tile < 31; ++tile) {
        const unsigned long long* p = &t[(tile * 2 + who) * 32];
        const unsigned long long prev_done = st == 0 ? t[((tile - 1) * 2 + who) * 32 + 3 * NST - 1] : p[3 * st - 1];
        e += double(p[3 * st] - prev_done);
        bi += double(p[3 * st + 1] - p[3 * st]);
        w += double(p[3 * st + 2] - p[3 * st + 1]);
        ++cnt;
      }
      printf("  %-11s %10.0f %14.0f %9.0f\n", names[st], e / cnt, bi / cnt, w / cnt);
      tot += (e + bi + w) / cnt;
    }
    printf("  total per tile %.0f cycles\n", tot);
  }
  return 0;
}
