// Drives the C++ facade exactly as a reference user drives distgrid::DistributedRun
// (tools/distgrid.cpp cmd_train / cmd_eval): reads rays from argv[1], writes results to argv[2].
#include <cstdio>
#include <fstream>
#include <vector>

#include "distgrid_b200/distgrid.hpp"

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  std::ifstream in(argv[1], std::ios::binary);
  uint64_t n = 0;
  in.read(reinterpret_cast<char*>(&n), 8);
  std::vector<double> buf(n * 9);
  in.read(reinterpret_cast<char*>(buf.data()), n * 9 * 8);
  std::vector<distgrid::SupervisedRay> batch(n);
  std::vector<distgrid::Ray> rays(n);
  for (uint64_t i = 0; i < n; ++i) {
    const double* r = &buf[9 * i];
    batch[i].ray = {{r[0], r[1], r[2]}, {r[3], r[4], r[5]}, i, 0};
    batch[i].color_gt = {r[6], r[7], r[8]};
    rays[i] = batch[i].ray;
  }
  distgrid::RunConfig cfg;
  cfg.grid_levels = 8;
  cfg.max_resolution = 128;
  cfg.fine_table_log2 = 12;
  cfg.march_step_divisor = 64;
  cfg.total_steps = 1000;
  cfg.partitions_x = 2;
  cfg.partitions_y = 1;
  const distgrid::Aabb box{{0, 0, 0}, {2, 1, 1}};
  const auto manifest = distgrid::split_regions(box, box, 2, 1, 0.0);
  distgrid::AppearanceTable table;  // the reference constructor (worker.hpp:177-178)
  table.dim = 16;
  table.image_ids = {0};
  table.rows.assign(16, 0.25);
  std::vector<float> app(16, 0.25f);
  distgrid::DistributedRun run(cfg, manifest, table);
  run.start();
  std::FILE* out = std::fopen(argv[2], "w");
  for (uint64_t step = 0; step < 2; ++step) {
    const auto st = run.training_step(batch, step);
    std::fprintf(out, "step %llu %.17g %.17g %.17g %llu\n", (unsigned long long)step, st.loss_rgb,
                 st.loss_transmittance, st.loss_distortion, (unsigned long long)st.rays);
  }
  std::vector<double> appd(app.begin(), app.end());
  const auto merged = run.evaluate_rays(rays, appd);
  for (uint64_t i = 0; i < n; ++i)
    std::fprintf(out, "ray %.9g %.9g %.9g %.9g %.9g\n", merged[i].color.x, merged[i].color.y,
                 merged[i].color.z, merged[i].transmittance, merged[i].depth);
  distgrid::CameraPose pose;  // looking down -z from above the scene
  pose.rotation(1, 1) = -1;
  pose.rotation(2, 2) = -1;
  pose.translation = {1.0, 0.5, 3.0};
  pose.fx = pose.fy = 20.0;
  pose.cx = 8.0;
  pose.cy = 6.0;
  pose.width = 16;
  pose.height = 12;
  const auto image = run.evaluate_image(pose, appd);
  double csum = 0.0, asum = 0.0;
  for (size_t i = 0; i < image.color.size(); ++i) {
    csum += image.color[i].x + image.color[i].y + image.color[i].z;
    asum += image.attribution[i].x + image.attribution[i].y + image.attribution[i].z;
  }
  std::fprintf(out, "image %u %u %.9g %.9g\n", image.width, image.height, csum, asum);
  const auto segs = distgrid::segment_rays(rays, manifest);
  uint64_t total = 0;
  for (const auto& s : segs) total += s.size();
  std::fprintf(out, "segments %llu\n", (unsigned long long)total);
  // worker views and the traffic counters of the reference's DistributedRun
  std::fprintf(out, "workers %u step %llu %llu bytes %llu %llu %llu\n", run.worker_count(),
               (unsigned long long)run.worker(0).step(), (unsigned long long)run.worker(1).step(),
               (unsigned long long)run.worker_bytes_sent(), (unsigned long long)run.scatter_payload_bytes(),
               (unsigned long long)run.scatter_entries());
  const distgrid::FieldParams fine = run.worker(1).fine_field();
  std::fprintf(out, "fine_field levels %zu density_in %u color_in %u region %u\n", fine.grid.levels().size(),
               fine.density_mlp.input_width(), fine.color_mlp.input_width(), run.worker(1).region().region_id);
  run.stop();
  try {
    run.stop();
    run.start();
    run.start();
  } catch (const std::logic_error&) {
    std::fprintf(out, "logic_error ok\n");
  }
  std::fclose(out);
  return 0;
}
