// geometry.cuh — stages 1-2 as device functions, bit-exact fp64.
//
//   ray_aabb        geometry.cpp:7-28
//   segment_ray     partition.cpp:254-296 (+ region_at 35-45)
//   occupancy walk  grid.cpp:235-304 (streamed: each closed run is handed to the ladder)
//   ladder          render.cpp:10-37
//   cascade_march   worker.cpp:79-110
//   position        worker.cpp:46
#pragma once

#include "dg_common.cuh"

namespace dg {

__device__ __forceinline__ bool ray_aabb(const double o[3], const double d[3], const double lo[3],
                                         const double hi[3], double& tn_out, double& tf_out) {
  double t_near = 0.0;
  double t_far = __longlong_as_double(0x7ff0000000000000ll);  // +inf
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double oo = o[a], dd = d[a];
    if (dd == 0.0) {
      if (oo < lo[a] || oo > hi[a]) return false;
      continue;
    }
    double t0 = ddiv(dsub(lo[a], oo), dd);
    double t1 = ddiv(dsub(hi[a], oo), dd);
    if (t0 > t1) {
      const double tmp = t0;
      t0 = t1;
      t1 = tmp;
    }
    t_near = smax(t_near, t0);
    t_far = smin(t_far, t1);
    if (t_near > t_far) return false;
  }
  tn_out = t_near;
  tf_out = t_far;
  return true;
}

__device__ __forceinline__ uint32_t locate_plane(const double* planes, uint32_t n_planes, double v) {
  uint32_t i = 1;  // upper_bound over planes[1 .. n-1)
  while (i < n_planes - 1 && !(v < planes[i])) ++i;
  return i - 1;
}

// Returns the number of segments; region/te/tx get nseg entries.
__device__ __forceinline__ int segment_ray(const Geo& g, const double o[3], const double d[3],
                                           uint8_t* region, double* te, double* tx) {
  double tn, tf;
  if (!ray_aabb(o, d, g.outer_lo, g.outer_hi, tn, tf) || !(tf > tn)) return 0;
  double cuts[kMaxSeg + 2];
  int nc = 0;
  cuts[nc++] = tn;
  cuts[nc++] = tf;
  for (int axis = 0; axis < 2; ++axis) {
    const double* planes = axis == 0 ? g.xp : g.yp;
    const uint32_t np = (axis == 0 ? g.kx : g.ky) + 1;
    const double dd = d[axis];
    if (dd == 0.0) continue;
    for (uint32_t i = 1; i + 1 < np; ++i) {
      const double t = ddiv(dsub(planes[i], o[axis]), dd);
      if (t > tn && t < tf) cuts[nc++] = t;
    }
  }
  for (int i = 1; i < nc; ++i) {  // std::sort of a NaN-free multiset
    const double v = cuts[i];
    int j = i - 1;
    while (j >= 0 && cuts[j] > v) {
      cuts[j + 1] = cuts[j];
      --j;
    }
    cuts[j + 1] = v;
  }
  int ns = 0;
  for (int i = 0; i + 1 < nc; ++i) {
    if (!(cuts[i + 1] > cuts[i])) continue;
    const double t_mid = dmul(0.5, dadd(cuts[i], cuts[i + 1]));
    const double px = dadd(o[0], dmul(d[0], t_mid));
    const double py = dadd(o[1], dmul(d[1], t_mid));
    const uint32_t reg = locate_plane(g.yp, g.ky + 1, py) * g.kx + locate_plane(g.xp, g.kx + 1, px);
    if (ns > 0 && region[ns - 1] == reg) {
      tx[ns - 1] = cuts[i + 1];
    } else {
      region[ns] = (uint8_t)reg;
      te[ns] = cuts[i];
      tx[ns] = cuts[i + 1];
      ++ns;
    }
  }
  return ns;
}

// Ladder over one occupied interval (render.cpp:21-35); emits (t, delta).
template <class Emit>
__device__ __forceinline__ void ladder(double iv_lo, double iv_hi, double t_enter, double t_exit,
                                       double offset, double step, Emit& emit) {
  const double lo = smax(iv_lo, t_enter);
  const double hi = smin(iv_hi, t_exit);
  if (!(hi > lo)) return;
  long long k = (long long)ceil(ddiv(dsub(dsub(lo, t_enter), offset), step));
  if (k < 0) k = 0;
  const double base = dadd(t_enter, offset);
  const double half = dmul(0.5, step);
  for (;; ++k) {
    const double t = dadd(base, dmul((double)k, step));
    if (t >= hi) break;
    const double slab_start = dsub(t, half);
    emit(t, smin(step, dsub(hi, slab_start)));
  }
}

// Amanatides-Woo walk over one occupancy grid (grid.cpp:235-304); every closed run of
// occupied cells is passed to on_run(start, end) in increasing t.
template <class Occupied, class OnRun>
__device__ __forceinline__ void occupancy_walk_fn(const double o[3], const double d[3], double t0,
                                                  double t1, const double lo[3], const double hi[3],
                                                  const uint32_t n[3], const Occupied& occupied_at,
                                                  OnRun& on_run) {
  if (!(t1 > t0)) return;
  double cell[3], entry[3], t_next[3], t_delta[3];
  int idx[3], stp[3];
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    cell[a] = ddiv(dsub(hi[a], lo[a]), (double)n[a]);
    entry[a] = dadd(o[a], dmul(d[a], t0));
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double local = ddiv(dsub(entry[a], lo[a]), cell[a]);
    int i = (int)floor(local);
    i = (i < 0) ? 0 : ((int)n[a] - 1 < i ? (int)n[a] - 1 : i);
    idx[a] = i;
    const double dd = d[a];
    if (dd > 0.0) {
      stp[a] = 1;
      t_delta[a] = ddiv(cell[a], dd);
      const double boundary = dadd(lo[a], dmul(cell[a], (double)(i + 1)));
      t_next[a] = dadd(t0, ddiv(dsub(boundary, entry[a]), dd));
    } else if (dd < 0.0) {
      stp[a] = -1;
      t_delta[a] = ddiv(-cell[a], dd);
      const double boundary = dadd(lo[a], dmul(cell[a], (double)i));
      t_next[a] = dadd(t0, ddiv(dsub(boundary, entry[a]), dd));
    } else {
      stp[a] = 0;
      t_delta[a] = inf;
      t_next[a] = inf;
    }
  }
  double t_cur = t0;
  bool run_open = false;
  double run_start = 0.0;
  while (t_cur < t1) {
    int ea = 0;
    if (t_next[1] < t_next[ea]) ea = 1;
    if (t_next[2] < t_next[ea]) ea = 2;
    const double t_exit = smin(t_next[ea], t1);
    const bool occupied = occupied_at((uint32_t)idx[0], (uint32_t)idx[1], (uint32_t)idx[2]);
    if (occupied && !run_open) {
      run_open = true;
      run_start = t_cur;
    } else if (!occupied && run_open) {
      run_open = false;
      on_run(run_start, t_cur);
    }
    if (t_exit >= t1) {
      t_cur = t1;
      break;
    }
    t_cur = t_exit;
    idx[ea] += stp[ea];
    if (idx[ea] < 0 || idx[ea] >= (int)n[ea]) break;
    t_next[ea] = dadd(t_next[ea], t_delta[ea]);
  }
  if (run_open) on_run(run_start, t_cur);
}

// The walk over the device's bricked bitfield (4x4x8-cell bricks, occ_addr).
template <class OnRun>
__device__ __forceinline__ void occupancy_walk(const double o[3], const double d[3], double t0,
                                               double t1, const double lo[3], const double hi[3],
                                               const uint32_t n[3], const uint32_t nb[3],
                                               const uint8_t* bits, OnRun& on_run) {
  const auto bricked = [&](uint32_t ix, uint32_t iy, uint32_t iz) {
    return __ldg(bits + occ_addr(nb, ix, iy, iz)) != 0;
  };
  occupancy_walk_fn(o, d, t0, t1, lo, hi, n, bricked, on_run);
}

// Closed-form sample range of ladder() on one run: first index k0 and count n of the t_k =
// base + k step in [lo, hi).  t_k is non-decreasing in k under round-to-nearest, so the
// estimate is corrected by evaluating t_k exactly as the ladder does at the boundary
// (bit-exact count).
struct Ladder {
  long long k0;
  uint32_t n;
  double hi;
};

__device__ __forceinline__ Ladder ladder_range(double iv_lo, double iv_hi, double t_enter, double t_exit,
                                               double offset, double step) {
  const double lo = smax(iv_lo, t_enter);
  const double hi = smin(iv_hi, t_exit);
  if (!(hi > lo)) return Ladder{0, 0u, hi};
  long long k0 = (long long)ceil(ddiv(dsub(dsub(lo, t_enter), offset), step));
  if (k0 < 0) k0 = 0;
  const double base = dadd(t_enter, offset);
  long long k1 = (long long)ceil(ddiv(dsub(hi, base), step));
  if (k1 < k0) k1 = k0;
  while (k1 > k0 && dadd(base, dmul((double)(k1 - 1), step)) >= hi) --k1;
  while (dadd(base, dmul((double)k1, step)) < hi) ++k1;
  return Ladder{k0, (uint32_t)(k1 - k0), hi};
}

__device__ __forceinline__ uint32_t ladder_count(double iv_lo, double iv_hi, double t_enter, double t_exit,
                                                 double offset, double step) {
  return ladder_range(iv_lo, iv_hi, t_enter, t_exit, offset, step).n;
}

// cascade_march's occupancy walks (worker.cpp:79-110) as runs: on_run(lo, hi, cascade) for
// every occupied run in increasing t; the fine-box walk's runs are cascade 0, the coarse
// walks' runs cascade 1 (the ladder's per-sample tag t in [fine_a, fine_b) is constant on a
// run).  Returns has_fine.
template <class OnRun>
__device__ __forceinline__ bool cascade_runs(const PartDesc& pd, const uint8_t* occ, const double o[3],
                                             const double d[3], double t0, double t1, double& fine_a,
                                             double& fine_b, OnRun& on_run) {
  fine_a = t1;
  fine_b = t1;
  bool has_fine = false;
  double tn, tf;
  if (ray_aabb(o, d, pd.fine_lo, pd.fine_hi, tn, tf)) {
    fine_a = sclamp(tn, t0, t1);
    fine_b = sclamp(tf, t0, t1);
    has_fine = fine_b > fine_a;
  }
  const double fa = fine_a, fb = fine_b;
  auto coarse = [&](double a, double b) { on_run(a, b, 1); };
  auto fine = [&](double a, double b) { on_run(a, b, 0); };
  const uint8_t* occ_f = occ + pd.occ_off[0];
  const uint8_t* occ_c = occ + pd.occ_off[1];
  if (has_fine) {
    if (fa > t0)
      occupancy_walk(o, d, t0, fa, pd.coarse_lo, pd.coarse_hi, pd.occ_n[1], pd.occ_nb[1], occ_c, coarse);
    occupancy_walk(o, d, fa, fb, pd.fine_lo, pd.fine_hi, pd.occ_n[0], pd.occ_nb[0], occ_f, fine);
    if (fb < t1)
      occupancy_walk(o, d, fb, t1, pd.coarse_lo, pd.coarse_hi, pd.occ_n[1], pd.occ_nb[1], occ_c, coarse);
  } else {
    occupancy_walk(o, d, t0, t1, pd.coarse_lo, pd.coarse_hi, pd.occ_n[1], pd.occ_nb[1], occ_c, coarse);
  }
  return has_fine;
}

// cascade_march (worker.cpp:79-110).  emit(t, delta, cascade) in increasing t.
// Returns has_fine and fills fine_a/fine_b (the cascade split) for the caller.
template <class Emit>
__device__ __forceinline__ bool cascade_march(const PartDesc& pd, const uint8_t* occ, const double o[3],
                                              const double d[3], double t0, double t1, double step,
                                              double offset, double& fine_a, double& fine_b,
                                              Emit& emit) {
  fine_a = t1;
  fine_b = t1;
  bool has_fine = false;
  double tn, tf;
  if (ray_aabb(o, d, pd.fine_lo, pd.fine_hi, tn, tf)) {
    fine_a = sclamp(tn, t0, t1);
    fine_b = sclamp(tf, t0, t1);
    has_fine = fine_b > fine_a;
  }
  const double fa = fine_a, fb = fine_b;
  auto tagged = [&](double t, double delta) {
    emit(t, delta, (has_fine && t >= fa && t < fb) ? 0 : 1);
  };
  auto run = [&](double a, double b) { ladder(a, b, t0, t1, offset, step, tagged); };
  const uint8_t* occ_f = occ + pd.occ_off[0];
  const uint8_t* occ_c = occ + pd.occ_off[1];
  if (has_fine) {
    if (fa > t0)
      occupancy_walk(o, d, t0, fa, pd.coarse_lo, pd.coarse_hi, pd.occ_n[1], pd.occ_nb[1], occ_c, run);
    occupancy_walk(o, d, fa, fb, pd.fine_lo, pd.fine_hi, pd.occ_n[0], pd.occ_nb[0], occ_f, run);
    if (fb < t1)
      occupancy_walk(o, d, fb, t1, pd.coarse_lo, pd.coarse_hi, pd.occ_n[1], pd.occ_nb[1], occ_c, run);
  } else {
    occupancy_walk(o, d, t0, t1, pd.coarse_lo, pd.coarse_hi, pd.occ_n[1], pd.occ_nb[1], occ_c, run);
  }
  return has_fine;
}

// worker.cpp:46: p = clamp(box.to_unit(o + d*t), 0, 1)
__device__ __forceinline__ void normalized_point(const double lo[3], const double hi[3],
                                                 const double o[3], const double d[3], double t,
                                                 double p[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double at = dadd(o[a], dmul(d[a], t));
    p[a] = sclamp(ddiv(dsub(at, lo[a]), dsub(hi[a], lo[a])), 0.0, 1.0);
  }
}

// grid.cpp:22-41 for one axis + the corner weight factor.
struct AxisW {
  uint32_t i0, i1;
  double frac;
};
__device__ __forceinline__ AxisW lattice_axis(double p, uint32_t n) {
  AxisW w;
  if (n == 1) {
    w.i0 = w.i1 = 0;
    w.frac = 0.0;
    return w;
  }
  const double pos = dmul(p, (double)(n - 1));
  uint32_t i0 = (uint32_t)floor(pos);
  if (i0 > n - 1) i0 = n - 1;
  w.i0 = i0;
  w.i1 = (i0 + 1 < n - 1) ? i0 + 1 : n - 1;
  w.frac = dsub(pos, (double)i0);
  return w;
}

// grid.cpp:75-84
__device__ __forceinline__ uint32_t table_row(const LevelDesc& lv, uint32_t ix, uint32_t iy, uint32_t iz) {
  if (!lv.hashed) return ix + lv.n[0] * (iy + lv.n[1] * iz);
  return (ix ^ (iy * 2654435761u) ^ (iz * 805459861u)) & lv.mask;
}

// CameraPose::pixel_ray_dir (partition.cpp:30-33): normalize(R * ((x - cx)/fx, (y - cy)/fy, 1)),
// Mat3 * Vec3 row by row left to right, normalize = v / sqrt(dot(v, v)); fp64, bit-exact.
__device__ __forceinline__ void pixel_ray_dir(const double R[9], double fx, double fy, double cx, double cy,
                                              double x, double y, double out[3]) {
  const double cam[3] = {ddiv(dsub(x, cx), fx), ddiv(dsub(y, cy), fy), 1.0};
  double v[3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
    v[r] = dadd(dadd(dmul(R[3 * r], cam[0]), dmul(R[3 * r + 1], cam[1])), dmul(R[3 * r + 2], cam[2]));
  const double len = __dsqrt_rn(dadd(dadd(dmul(v[0], v[0]), dmul(v[1], v[1])), dmul(v[2], v[2])));
#pragma unroll
  for (int a = 0; a < 3; ++a) out[a] = ddiv(v[a], len);
}

}  // namespace dg
