/*
 * dg_oracle.c — TEST INFRASTRUCTURE ONLY (see dg_oracle.h).
 *
 * Plain-C restatement of the reference DistGrid per-ray path in IEEE fp64.  Built with
 * -ffp-contract=off; every expression keeps the reference's evaluation order so that the
 * restatement is bit-identical to the reference build (checked in
 * tests/test_oracle_vs_reference.py).  File:line citations are relative to
 * /root/reference/proj.
 */
#include "dg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static char g_err[256];
const char* or_last_error(void) { return g_err; }
static int or_fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}

/* std::max / std::min / std::clamp semantics (first argument wins ties). */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double sclamp(double v, double lo, double hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}
static inline int iclamp(int v, int lo, int hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }

/* Test-only: when set, every gradient contribution t is also accumulated as |t| into the
 * parallel array g_abs (same offsets as the grads base g_gbase).  Used to state the gradient
 * tolerance relative to sum |contributions| (the standard bound for reordered fp sums). */
static double* g_abs = NULL;
/* Test-only sample log (or_run_sample_log): the encoding's upstream gradient of the current
 * field_backward call lands here when set. */
static double* g_enc_grad_out = NULL;
static const double* g_gbase = NULL;
#define OR_ABS(ptr, val)                                     \
  do {                                                       \
    if (g_abs) g_abs[(ptr) - g_gbase] += fabs(val);          \
  } while (0)

/* ------------------------------------------------------------------ rng.hpp:8-62 */
uint64_t or_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

uint64_t or_counter_hash(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t h = or_splitmix64(seed ^ 0x6a09e667f3bcc909ull);
  h = or_splitmix64(h ^ a);
  h = or_splitmix64(h ^ b);
  h = or_splitmix64(h ^ c);
  return h;
}

double or_counter_uniform(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return (double)(or_counter_hash(seed, a, b, c) >> 11) * 0x1.0p-53;
}

/* std::mt19937_64 (the published MT19937-64 algorithm). */
void or_mt64_seed(or_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = 312;
}

uint64_t or_mt64_next(or_mt64* g) {
  static const uint64_t mag01[2] = {0ull, 0xB5026F5AA96619E9ull};
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  if (g->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ull)];
    }
    for (; i < 311; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ull)];
    }
    x = (g->mt[311] & UM) | (g->mt[0] & LM);
    g->mt[311] = g->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ull)];
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= (x >> 43);
  return x;
}

void or_rng_init(or_mt64* g, uint64_t seed) { or_mt64_seed(g, or_splitmix64(seed)); }
double or_rng_uniform(or_mt64* g) { return (double)(or_mt64_next(g) >> 11) * 0x1.0p-53; }
double or_rng_uniform_range(or_mt64* g, double lo, double hi) {
  return lo + (hi - lo) * or_rng_uniform(g);
}

/* ------------------------------------------------------- grid.cpp:56-73 (shapes) */
uint32_t or_level_resolution(uint32_t levels, uint32_t base, uint32_t maxr, uint32_t level) {
  if (levels == 1) return base;
  const double growth = exp((log((double)maxr) - log((double)base)) / (double)(levels - 1));
  return (uint32_t)llround((double)base * pow(growth, (double)level));
}

or_shape or_grid_shape(const double aspect[3], uint32_t nres) {
  const double n = (double)nres;
  const double s = smax(aspect[0], smax(aspect[1], aspect[2])); /* max_component */
  or_shape sh;
  sh.nx = (uint32_t)ceil(aspect[0] / s * n);
  sh.ny = (uint32_t)ceil(aspect[1] / s * n);
  sh.nz = (uint32_t)ceil(aspect[2] / s * n);
  return sh;
}

/* grid.cpp:90-105 — level shapes, mapping mode, rows; flat offsets in doubles. */
static void grid_layout(or_grid* g, const dg_run_config* cfg, uint32_t table_log2,
                        const or_box* box) {
  const double aspect[3] = {box->hi[0] - box->lo[0], box->hi[1] - box->lo[1],
                            box->hi[2] - box->lo[2]};
  g->L = cfg->grid_levels;
  g->F = cfg->grid_features;
  g->T = 1u << table_log2;
  uint64_t off = 0;
  for (uint32_t l = 0; l < g->L; ++l) {
    const uint32_t n = or_level_resolution(cfg->grid_levels, cfg->base_resolution,
                                           cfg->max_resolution, l);
    g->shape[l] = or_grid_shape(aspect, n);
    const uint64_t voxels = (uint64_t)g->shape[l].nx * g->shape[l].ny * g->shape[l].nz;
    g->hashed[l] = voxels <= g->T ? 0u : 1u;
    g->rows[l] = g->hashed[l] ? g->T : voxels;
    g->offset[l] = off;
    off += g->rows[l] * g->F;
  }
  g->size = off;
}

/* field.cpp:189-201 — FieldParams widths, flat order of parameter_arrays. */
static void field_layout(or_field_layout* f, const dg_run_config* cfg, uint32_t table_log2,
                         const or_box* box, uint32_t coarse) {
  grid_layout(&f->grid, cfg, table_log2, box);
  f->coarse = coarse;
  f->enc_width = f->grid.L * f->grid.F;
  f->color_in = 15 + 16 + cfg->appearance_dim;
  uint64_t o = f->grid.size;
  f->dw0 = o; o += 64ull * f->enc_width;
  f->db0 = o; o += 64;
  f->dw1 = o; o += 16ull * 64;
  f->db1 = o; o += 16;
  f->cw0 = o; o += 64ull * f->color_in;
  f->cb0 = o; o += 64;
  f->cw1 = o; o += 64ull * 64;
  f->cb1 = o; o += 64;
  f->cw2 = o; o += 3ull * 64;
  f->cb2 = o; o += 3;
  f->size = o;
}

/* partition.cpp:206-252 split_regions (+ worker.cpp:901-925 grid configs, march step). */
int or_model_init(or_model* m, const dg_run_config* cfg) {
  memset(m, 0, sizeof *m);
  m->cfg = *cfg;
  const uint32_t kx = cfg->kx, ky = cfg->ky;
  if (kx < 1 || ky < 1) return or_fail("split_regions: kx, ky must be >= 1");
  if (kx * ky > DG_MAX_PARTITIONS || kx + ky - 1 > DG_MAX_SEGMENTS)
    return or_fail("oracle: too many partitions");
  if (cfg->grid_levels > OR_MAX_LEVELS) return or_fail("oracle: too many levels");
  m->P = kx * ky;
  for (int a = 0; a < 3; ++a) {
    m->inner.lo[a] = cfg->inner_lo[a];
    m->inner.hi[a] = cfg->inner_hi[a];
    m->outer.lo[a] = cfg->outer_lo[a];
    m->outer.hi[a] = cfg->outer_hi[a];
  }
  for (uint32_t i = 0; i <= kx; ++i)
    m->x_planes[i] = i == 0    ? m->inner.lo[0]
                     : i == kx ? m->inner.hi[0]
                               : m->inner.lo[0] + (m->inner.hi[0] - m->inner.lo[0]) * (double)i /
                                                      (double)kx;
  for (uint32_t i = 0; i <= ky; ++i)
    m->y_planes[i] = i == 0    ? m->inner.lo[1]
                     : i == ky ? m->inner.hi[1]
                               : m->inner.lo[1] + (m->inner.hi[1] - m->inner.lo[1]) * (double)i /
                                                      (double)ky;
  for (uint32_t iy = 0; iy < ky; ++iy) {
    for (uint32_t ix = 0; ix < kx; ++ix) {
      const uint32_t r = iy * kx + ix;
      or_box* f = &m->fine[r];
      or_box* c = &m->coarse[r];
      f->lo[0] = m->x_planes[ix];
      f->lo[1] = m->y_planes[iy];
      f->lo[2] = m->inner.lo[2];
      f->hi[0] = m->x_planes[ix + 1];
      f->hi[1] = m->y_planes[iy + 1];
      f->hi[2] = m->inner.hi[2];
      c->lo[0] = ix == 0 ? m->outer.lo[0] : m->x_planes[ix];
      c->lo[1] = iy == 0 ? m->outer.lo[1] : m->y_planes[iy];
      c->lo[2] = m->outer.lo[2];
      c->hi[0] = ix == kx - 1 ? m->outer.hi[0] : m->x_planes[ix + 1];
      c->hi[1] = iy == ky - 1 ? m->outer.hi[1] : m->y_planes[iy + 1];
      c->hi[2] = m->outer.hi[2];
      field_layout(&m->field[r][0], cfg, cfg->fine_table_log2, f, 0);
      field_layout(&m->field[r][1], cfg, cfg->coarse_table_log2, c, 1);
      m->nparams[r] = m->field[r][0].size + m->field[r][1].size;
      for (int k = 0; k < 2; ++k) {
        const or_box* b = k == 0 ? f : c;
        const double aspect[3] = {b->hi[0] - b->lo[0], b->hi[1] - b->lo[1], b->hi[2] - b->lo[2]};
        m->occ_shape[r][k] = or_grid_shape(aspect, cfg->occ_resolution);
      }
    }
  }
  const double ext[3] = {m->outer.hi[0] - m->outer.lo[0], m->outer.hi[1] - m->outer.lo[1],
                         m->outer.hi[2] - m->outer.lo[2]};
  m->step = smax(ext[0], smax(ext[1], ext[2])) / cfg->march_step_divisor;
  return 0;
}

/* ------------------------------------------------------- geometry.cpp:7-28 */
int or_ray_aabb(const double o[3], const double d[3], const or_box* box, double* t_near_out,
                double* t_far_out) {
  double t_near = 0.0;
  double t_far = INFINITY;
  for (int axis = 0; axis < 3; ++axis) {
    const double oo = o[axis], dd = d[axis];
    const double lo = box->lo[axis], hi = box->hi[axis];
    if (dd == 0.0) {
      if (oo < lo || oo > hi) return 0;
      continue;
    }
    double t0 = (lo - oo) / dd;
    double t1 = (hi - oo) / dd;
    if (t0 > t1) {
      const double tmp = t0;
      t0 = t1;
      t1 = tmp;
    }
    t_near = smax(t_near, t0);
    t_far = smin(t_far, t1);
    if (t_near > t_far) return 0;
  }
  *t_near_out = t_near;
  *t_far_out = t_far;
  return 1;
}

/* ------------------------------------------------------- partition.cpp:35-45 */
static uint32_t locate_plane(const double* planes, uint32_t n_planes, double v) {
  /* upper_bound over planes[1 .. n-1) */
  uint32_t i = 1;
  while (i < n_planes - 1 && !(v < planes[i])) ++i;
  return i - 1;
}

uint32_t or_region_at(const or_model* m, double x, double y) {
  const uint32_t ix = locate_plane(m->x_planes, m->cfg.kx + 1, x);
  const uint32_t iy = locate_plane(m->y_planes, m->cfg.ky + 1, y);
  return iy * m->cfg.kx + ix;
}

/* ------------------------------------------------------- partition.cpp:254-296 */
int or_segment_ray(const or_model* m, const double o[3], const double d[3], uint32_t* region,
                   double* t_enter, double* t_exit) {
  double tn, tf;
  if (!or_ray_aabb(o, d, &m->outer, &tn, &tf) || !(tf > tn)) return 0;
  double cuts[2 + 2 * DG_MAX_PARTITIONS];
  int nc = 0;
  cuts[nc++] = tn;
  cuts[nc++] = tf;
  for (int axis = 0; axis < 2; ++axis) {
    const double* planes = axis == 0 ? m->x_planes : m->y_planes;
    const uint32_t np = (axis == 0 ? m->cfg.kx : m->cfg.ky) + 1;
    const double dd = d[axis];
    if (dd == 0.0) continue;
    for (uint32_t i = 1; i + 1 < np; ++i) {
      const double t = (planes[i] - o[axis]) / dd;
      if (t > tn && t < tf) cuts[nc++] = t;
    }
  }
  for (int i = 1; i < nc; ++i) { /* std::sort: any correct sort of a NaN-free multiset */
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
    const double t_mid = 0.5 * (cuts[i] + cuts[i + 1]);
    const double px = o[0] + d[0] * t_mid;
    const double py = o[1] + d[1] * t_mid;
    const uint32_t reg = or_region_at(m, px, py);
    if (ns > 0 && region[ns - 1] == reg) {
      t_exit[ns - 1] = cuts[i + 1];
    } else {
      region[ns] = reg;
      t_enter[ns] = cuts[i];
      t_exit[ns] = cuts[i + 1];
      ++ns;
    }
  }
  return ns;
}

/* ------------------------------------------------------- grid.cpp:235-304 */
int or_occupancy_skip(const double o[3], const double d[3], double t0, double t1,
                      const or_box* box, or_shape shape, const uint8_t* bits, double* iv,
                      int cap) {
  int n = 0;
  if (!(t1 > t0)) return 0;
  const uint32_t ext[3] = {shape.nx, shape.ny, shape.nz};
  double cell[3];
  for (int a = 0; a < 3; ++a) cell[a] = (box->hi[a] - box->lo[a]) / (double)ext[a];
  int idx[3], step[3];
  double t_next[3], t_delta[3], entry[3];
  for (int a = 0; a < 3; ++a) entry[a] = o[a] + d[a] * t0;
  for (int a = 0; a < 3; ++a) {
    const double local = (entry[a] - box->lo[a]) / cell[a];
    idx[a] = iclamp((int)floor(local), 0, (int)ext[a] - 1);
    const double dd = d[a];
    if (dd > 0.0) {
      step[a] = 1;
      t_delta[a] = cell[a] / dd;
      const double boundary = box->lo[a] + cell[a] * (double)(idx[a] + 1);
      t_next[a] = t0 + (boundary - entry[a]) / dd;
    } else if (dd < 0.0) {
      step[a] = -1;
      t_delta[a] = -cell[a] / dd;
      const double boundary = box->lo[a] + cell[a] * (double)idx[a];
      t_next[a] = t0 + (boundary - entry[a]) / dd;
    } else {
      step[a] = 0;
      t_delta[a] = INFINITY;
      t_next[a] = INFINITY;
    }
  }
  double t_cur = t0;
  int run_open = 0;
  double run_start = 0.0;
  while (t_cur < t1) {
    int ea = 0;
    if (t_next[1] < t_next[ea]) ea = 1;
    if (t_next[2] < t_next[ea]) ea = 2;
    const double t_exit = smin(t_next[ea], t1);
    const uint64_t cidx =
        (uint64_t)idx[0] + (uint64_t)ext[0] * ((uint64_t)idx[1] + (uint64_t)ext[1] * (uint64_t)idx[2]);
    const int occupied = bits[cidx] != 0;
    if (occupied && !run_open) {
      run_open = 1;
      run_start = t_cur;
    } else if (!occupied && run_open) {
      run_open = 0;
      if (n < cap) {
        iv[2 * n] = run_start;
        iv[2 * n + 1] = t_cur;
      }
      ++n;
    }
    if (t_exit >= t1) {
      t_cur = t1;
      break;
    }
    t_cur = t_exit;
    idx[ea] += step[ea];
    if (idx[ea] < 0 || idx[ea] >= (int)ext[ea]) break;
    t_next[ea] += t_delta[ea];
  }
  if (run_open) {
    if (n < cap) {
      iv[2 * n] = run_start;
      iv[2 * n + 1] = t_cur;
    }
    ++n;
  }
  return n;
}

/* ------------------------------------------------------- render.cpp:10-37 */
int or_march_segment(double t_enter, double t_exit, const double* iv, int n_iv, double step,
                     int jitter, uint64_t seed, uint64_t ray_id, uint64_t batch_id, double* t,
                     double* delta, int cap) {
  int n = 0;
  if (!(t_exit > t_enter)) return 0;
  const double offset =
      jitter ? step * or_counter_uniform(seed, ray_id, batch_id, 0) : 0.5 * step;
  for (int i = 0; i < n_iv; ++i) {
    const double lo = smax(iv[2 * i], t_enter);
    const double hi = smin(iv[2 * i + 1], t_exit);
    if (!(hi > lo)) continue;
    int64_t k = (int64_t)ceil((lo - t_enter - offset) / step);
    if (k < 0) k = 0;
    for (;; ++k) {
      const double tt = t_enter + offset + (double)k * step;
      if (tt >= hi) break;
      const double slab_start = tt - 0.5 * step;
      if (n < cap) {
        t[n] = tt;
        delta[n] = smin(step, hi - slab_start);
      }
      ++n;
    }
  }
  return n;
}

/* ------------------------------------------------------- worker.cpp:79-110 */
#define OR_MAX_IV 4096
int or_cascade_march(const or_model* m, uint32_t region, const uint8_t* occ_fine,
                     const uint8_t* occ_coarse, const double o[3], const double d[3], double t0,
                     double t1, int jitter, uint64_t ray_id, uint64_t batch_id, double* t,
                     double* delta, uint8_t* cascade, int cap) {
  static double iv[2 * OR_MAX_IV];
  int n_iv = 0;
  double fine_a = t1, fine_b = t1;
  int has_fine = 0;
  double tn, tf;
  if (or_ray_aabb(o, d, &m->fine[region], &tn, &tf)) {
    fine_a = sclamp(tn, t0, t1);
    fine_b = sclamp(tf, t0, t1);
    has_fine = fine_b > fine_a;
  }
  const or_box* fb = &m->fine[region];
  const or_box* cb = &m->coarse[region];
  const or_shape fs = m->occ_shape[region][0], cs = m->occ_shape[region][1];
#define OR_APPEND(a, b, box, sh, bits)                                                     \
  do {                                                                                     \
    const int k_ = or_occupancy_skip(o, d, (a), (b), (box), (sh), (bits), iv + 2 * n_iv,   \
                                     OR_MAX_IV - n_iv);                                    \
    if (n_iv + k_ > OR_MAX_IV) return or_fail("oracle: interval capacity");                \
    n_iv += k_;                                                                            \
  } while (0)
  if (has_fine) {
    if (fine_a > t0) OR_APPEND(t0, fine_a, cb, cs, occ_coarse);
    OR_APPEND(fine_a, fine_b, fb, fs, occ_fine);
    if (fine_b < t1) OR_APPEND(fine_b, t1, cb, cs, occ_coarse);
  } else {
    OR_APPEND(t0, t1, cb, cs, occ_coarse);
  }
#undef OR_APPEND
  const int n = or_march_segment(t0, t1, iv, n_iv, m->step, jitter, m->cfg.seed, ray_id, batch_id,
                                 t, delta, cap);
  if (n > cap) return or_fail("oracle: sample capacity");
  for (int k = 0; k < n; ++k)
    cascade[k] = (has_fine && t[k] >= fine_a && t[k] < fine_b) ? 0 : 1;
  return n;
}

/* worker.cpp:46 — p = clamp(box.to_unit(ray.at(t)), 0, 1); vecmath.hpp:68-70,86,108 */
void or_normalized_point(const or_box* box, const double o[3], const double d[3], double t,
                         double p[3]) {
  for (int a = 0; a < 3; ++a) {
    const double at = o[a] + d[a] * t;
    const double u = (at - box->lo[a]) / (box->hi[a] - box->lo[a]);
    p[a] = sclamp(u, 0.0, 1.0);
  }
}

/* ------------------------------------------------------- grid.cpp:22-41, 75-84 */
typedef struct {
  uint32_t i0[3], i1[3];
  double frac[3];
} corner_weights;

static corner_weights lattice_weights(const double p[3], or_shape sh) {
  const uint32_t ext[3] = {sh.nx, sh.ny, sh.nz};
  corner_weights cw;
  for (int a = 0; a < 3; ++a) {
    const uint32_t n = ext[a];
    if (n == 1) {
      cw.i0[a] = 0;
      cw.i1[a] = 0;
      cw.frac[a] = 0.0;
      continue;
    }
    const double pos = p[a] * (double)(n - 1);
    uint32_t i0 = (uint32_t)floor(pos);
    if (i0 > n - 1) i0 = n - 1;
    cw.i0[a] = i0;
    cw.i1[a] = (i0 + 1 < n - 1) ? i0 + 1 : n - 1;
    cw.frac[a] = pos - (double)i0;
  }
  return cw;
}

uint32_t or_table_index(const or_grid* g, uint32_t level, uint32_t ix, uint32_t iy, uint32_t iz) {
  const or_shape s = g->shape[level];
  if (!g->hashed[level]) return ix + s.nx * (iy + s.ny * iz);
  const uint32_t h = ix ^ (iy * 2654435761u) ^ (iz * 805459861u);
  return h & (uint32_t)(g->rows[level] - 1);
}

static inline double corner_w(const corner_weights* cw, int corner) {
  const int cx = corner & 1, cy = (corner >> 1) & 1, cz = (corner >> 2) & 1;
  return (cx ? cw->frac[0] : 1.0 - cw->frac[0]) * (cy ? cw->frac[1] : 1.0 - cw->frac[1]) *
         (cz ? cw->frac[2] : 1.0 - cw->frac[2]);
}

static inline uint32_t corner_row(const or_grid* g, uint32_t l, const corner_weights* cw,
                                  int corner) {
  const int cx = corner & 1, cy = (corner >> 1) & 1, cz = (corner >> 2) & 1;
  return or_table_index(g, l, cx ? cw->i1[0] : cw->i0[0], cy ? cw->i1[1] : cw->i0[1],
                        cz ? cw->i1[2] : cw->i0[2]);
}

/* grid.cpp:107-130 */
void or_encode(const or_grid* g, const double* table, const double p[3], double* out,
               uint32_t* rows) {
  const uint32_t F = g->F;
  for (uint32_t l = 0; l < g->L; ++l) {
    const corner_weights cw = lattice_weights(p, g->shape[l]);
    double* dst = out + (size_t)l * F;
    for (uint32_t k = 0; k < F; ++k) dst[k] = 0.0;
    for (int c = 0; c < 8; ++c) {
      const double w = corner_w(&cw, c);
      if (w == 0.0) {
        if (rows) rows[l * 8 + c] = 0xffffffffu;
        continue;
      }
      const uint32_t row = corner_row(g, l, &cw, c);
      if (rows) rows[l * 8 + c] = row;
      if (!table) continue; /* rows only (full-size index checks without the tables) */
      const double* src = table + g->offset[l] + (size_t)row * F;
      for (uint32_t k = 0; k < F; ++k) dst[k] += w * src[k];
    }
  }
}

/* grid.cpp:132-157 */
void or_encode_backward(const or_grid* g, double* grads, const double p[3], const double* up) {
  const uint32_t F = g->F;
  for (uint32_t l = 0; l < g->L; ++l) {
    const corner_weights cw = lattice_weights(p, g->shape[l]);
    const double* u = up + (size_t)l * F;
    for (int c = 0; c < 8; ++c) {
      const double w = corner_w(&cw, c);
      if (w == 0.0) continue;
      const uint32_t row = corner_row(g, l, &cw, c);
      double* dst = grads + g->offset[l] + (size_t)row * F;
      for (uint32_t k = 0; k < F; ++k) {
        dst[k] += w * u[k];
        OR_ABS(dst + k, w * u[k]);
      }
    }
  }
}

/* ------------------------------------------------------- sh.hpp:14-35 */
void or_sh_encode(const double dd[3], double out[16]) {
  const double x = dd[0], y = dd[1], z = dd[2];
  const double xy = x * y, xz = x * z, yz = y * z;
  const double x2 = x * x, y2 = y * y, z2 = z * z;
  out[0] = 0.28209479177387814;
  out[1] = -0.48860251190291987 * y;
  out[2] = 0.48860251190291987 * z;
  out[3] = -0.48860251190291987 * x;
  out[4] = 1.0925484305920792 * xy;
  out[5] = -1.0925484305920792 * yz;
  out[6] = 0.31539156525252005 * (3.0 * z2 - 1.0);
  out[7] = -1.0925484305920792 * xz;
  out[8] = 0.5462742152960396 * (x2 - y2);
  out[9] = -0.5900435899266435 * y * (3.0 * x2 - y2);
  out[10] = 2.890611442640554 * xy * z;
  out[11] = -0.4570457994644658 * y * (5.0 * z2 - 1.0);
  out[12] = 0.3731763325901154 * z * (5.0 * z2 - 3.0);
  out[13] = -0.4570457994644658 * x * (5.0 * z2 - 1.0);
  out[14] = 1.445305721320277 * z * (x2 - y2);
  out[15] = -0.5900435899266435 * x * (x2 - 3.0 * y2);
}

/* ------------------------------------------------------- mlp.cpp:10-36, 55-82 */
static inline double act(double z, int sigmoid) {
  return sigmoid ? 1.0 / (1.0 + exp(-z)) : (z > 0.0 ? z : 0.0);
}
static inline double act_grad(double z, int sigmoid) {
  if (sigmoid) {
    const double s = 1.0 / (1.0 + exp(-z));
    return s * (1.0 - s);
  }
  return z > 0.0 ? 1.0 : 0.0;
}

/* Test-only ReLU decision override (or_run_mask_override): a unit whose pre-activation lies
 * within fp32 noise of 0 may round to either side; with c->ovr set, the ReLU layers (h1, and
 * c1 / c2 of the fine field) take their on/off decision from c->mask instead of the sign of z. */
static inline int relu_on(const or_field_cache* c, int layer, int r, double z) {
  return c->ovr ? (int)((c->mask[layer] >> r) & 1u) : z > 0.0;
}
static inline double act_m(const or_field_cache* c, int layer, int r, double z, int sigmoid) {
  if (sigmoid || !c->ovr) return act(z, sigmoid);
  return relu_on(c, layer, r, z) ? z : 0.0;
}
static inline double act_grad_m(const or_field_cache* c, int layer, int r, double z, int sigmoid) {
  if (sigmoid || !c->ovr) return act_grad(z, sigmoid);
  return relu_on(c, layer, r, z) ? 1.0 : 0.0;
}

/* One dense layer: y = b + W x, bias-first sequential dot (mlp.cpp:64-71). */
static void dense(const double* W, const double* b, const double* x, uint32_t in, uint32_t out,
                  double* y) {
  for (uint32_t r = 0; r < out; ++r) {
    const double* wrow = W + (size_t)r * in;
    double acc = b[r];
    for (uint32_t c = 0; c < in; ++c) acc += wrow[c] * x[c];
    y[r] = acc;
  }
}

static inline double clip_output(double v, uint8_t* clipped) { /* field.cpp:14-25 */
  if (v > 15.0) {
    *clipped = 1;
    return 15.0;
  }
  if (v < -15.0) {
    *clipped = 1;
    return -15.0;
  }
  *clipped = 0;
  return v;
}

/* query_density + query_color (field.cpp:230-288) with the caches field_backward needs. */
void or_field_forward(const or_field_layout* f, const double* params, const double p[3],
                      const double dir[3], const double* app, or_field_cache* c) {
  memcpy(c->point, p, sizeof c->point);
  or_encode(&f->grid, params, p, c->enc, NULL);
  /* density MLP: [enc -> 64 ReLU -> 16] */
  dense(params + f->dw0, params + f->db0, c->enc, f->enc_width, 64, c->h1);
  double a1[64];
  for (int r = 0; r < 64; ++r) a1[r] = act_m(c, 0, r, c->h1[r], 0);
  double raw[16];
  dense(params + f->dw1, params + f->db1, a1, 64, 16, raw);
  for (int k = 0; k < 16; ++k) c->draw[k] = clip_output(raw[k], &c->dclip[k]);
  c->sigma = exp(c->draw[0]);
  /* colour input [feature 15 | sh 16 | appearance] */
  for (int k = 0; k < 15; ++k) c->cin[k] = c->draw[1 + k];
  or_sh_encode(dir, c->cin + 15);
  const uint32_t dapp = f->color_in - 31;
  for (uint32_t k = 0; k < dapp; ++k) c->cin[31 + k] = app[k];
  const int sig = f->coarse != 0;
  dense(params + f->cw0, params + f->cb0, c->cin, f->color_in, 64, c->c1);
  double a2[64], a3[64];
  for (int r = 0; r < 64; ++r) a2[r] = act_m(c, 1, r, c->c1[r], sig);
  dense(params + f->cw1, params + f->cb1, a2, 64, 64, c->c2);
  for (int r = 0; r < 64; ++r) a3[r] = act_m(c, 2, r, c->c2[r], sig);
  double craw[3];
  dense(params + f->cw2, params + f->cb2, a3, 64, 3, craw);
  for (int k = 0; k < 3; ++k) {
    c->craw[k] = clip_output(craw[k], &c->cclip[k]);
    c->rgb[k] = 1.0 / (1.0 + exp(-c->craw[k]));
  }
}

/* Mlp::backward for one layer (mlp.cpp:84-138): accumulate W/b grads, optional input grad. */
static void dense_backward(const double* W, double* gW, double* gb, const double* in,
                           const double* delta, uint32_t n_in, uint32_t n_out, double* in_grad) {
  for (uint32_t r = 0; r < n_out; ++r) {
    const double dv = delta[r];
    if (dv == 0.0) continue;
    double* wg = gW + (size_t)r * n_in;
    for (uint32_t c = 0; c < n_in; ++c) {
      wg[c] += dv * in[c];
      OR_ABS(wg + c, dv * in[c]);
    }
    gb[r] += dv;
    OR_ABS(gb + r, dv);
  }
  if (in_grad) {
    for (uint32_t c = 0; c < n_in; ++c) in_grad[c] = 0.0;
    for (uint32_t r = 0; r < n_out; ++r) {
      const double dv = delta[r];
      if (dv == 0.0) continue;
      const double* wrow = W + (size_t)r * n_in;
      for (uint32_t c = 0; c < n_in; ++c) in_grad[c] += dv * wrow[c];
    }
  }
}

/* field.cpp:290-327 */
void or_field_backward(const or_field_layout* f, const double* params, double* grads,
                       const or_field_cache* c, double sigma_grad, const double color_grad[3]) {
  double cin_grad[15 + 16 + 64];
  memset(cin_grad, 0, sizeof cin_grad);
  const int sig = f->coarse != 0;
  if (color_grad[0] != 0.0 || color_grad[1] != 0.0 || color_grad[2] != 0.0) {
    double draw3[3];
    for (int k = 0; k < 3; ++k) {
      const double s = 1.0 / (1.0 + exp(-c->craw[k]));
      draw3[k] = c->cclip[k] ? 0.0 : color_grad[k] * s * (1.0 - s);
    }
    /* colour MLP backward: layers 2, 1, 0 */
    double a2[64], a3[64], d3[64], d2[64];
    for (int r = 0; r < 64; ++r) {
      a2[r] = act_m(c, 1, r, c->c1[r], sig);
      a3[r] = act_m(c, 2, r, c->c2[r], sig);
    }
    dense_backward(params + f->cw2, grads + f->cw2, grads + f->cb2, a3, draw3, 64, 3, d3);
    for (int r = 0; r < 64; ++r) d3[r] *= act_grad_m(c, 2, r, c->c2[r], sig);
    dense_backward(params + f->cw1, grads + f->cw1, grads + f->cb1, a2, d3, 64, 64, d2);
    for (int r = 0; r < 64; ++r) d2[r] *= act_grad_m(c, 1, r, c->c1[r], sig);
    dense_backward(params + f->cw0, grads + f->cw0, grads + f->cb0, c->cin, d2, f->color_in, 64,
                   cin_grad);
  }
  double draw[16];
  draw[0] = c->dclip[0] ? 0.0 : sigma_grad * c->sigma;
  for (int k = 0; k < 15; ++k) draw[1 + k] = c->dclip[1 + k] ? 0.0 : cin_grad[k];
  int any = 0;
  for (int k = 0; k < 16; ++k)
    if (draw[k] != 0.0) {
      any = 1;
      break;
    }
  if (!any) return;
  double a1[64], d1[64];
  for (int r = 0; r < 64; ++r) a1[r] = act_m(c, 0, r, c->h1[r], 0);
  dense_backward(params + f->dw1, grads + f->dw1, grads + f->db1, a1, draw, 64, 16, d1);
  for (int r = 0; r < 64; ++r) d1[r] *= act_grad_m(c, 0, r, c->h1[r], 0);
  double enc_grad[2 * OR_MAX_LEVELS * 4];
  dense_backward(params + f->dw0, grads + f->dw0, grads + f->db0, c->enc, d1, f->enc_width, 64,
                 enc_grad);
  if (g_enc_grad_out) memcpy(g_enc_grad_out, enc_grad, sizeof(double) * f->enc_width);
  or_encode_backward(&f->grid, grads, c->point, enc_grad);
}

/* ------------------------------------------------------- render.cpp:46-78 */
void or_local_render(const double* t, const double* delta, const double* sigma,
                     const double* rgb, int n, double out_rgb[3], double* out_T,
                     double* out_depth, double* alpha_c, double* prefix_c) {
  double prefix = 1.0;
  double col[3] = {0.0, 0.0, 0.0};
  double depth_sum = 0.0;
  for (int k = 0; k < n; ++k) {
    const double alpha = 1.0 - exp(-sigma[k] * delta[k]);
    if (alpha_c) alpha_c[k] = alpha;
    if (prefix_c) prefix_c[k] = prefix;
    const double w = prefix * alpha;
    for (int a = 0; a < 3; ++a) col[a] += rgb[3 * k + a] * w;
    depth_sum += w * t[k];
    prefix *= 1.0 - alpha;
  }
  for (int a = 0; a < 3; ++a) out_rgb[a] = col[a];
  *out_T = prefix;
  if (out_depth) *out_depth = depth_sum;
}

/* render.cpp:101-116 */
void or_merge_forward(const double* rgb, const double* T, const double* depth, int n,
                      double out_rgb[3], double* out_T, double* out_depth) {
  double prefix = 1.0, dep = 0.0;
  double col[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) col[a] += rgb[3 * i + a] * prefix;
    dep += (depth ? depth[i] : 0.0) * prefix;
    prefix *= T[i];
  }
  for (int a = 0; a < 3; ++a) out_rgb[a] = col[a];
  *out_T = prefix;
  if (out_depth) *out_depth = dep;
}

static inline double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

/* render.cpp:118-143 */
void or_merge_backward(const double up_c[3], double up_t, const double* rgb, const double* T,
                       int n, double* grad_c, double* grad_t) {
  double prefix[DG_MAX_SEGMENTS + 1], suffix[DG_MAX_SEGMENTS + 1];
  for (int i = 0; i <= n; ++i) prefix[i] = suffix[i] = 1.0;
  for (int i = 0; i < n; ++i) prefix[i + 1] = prefix[i] * T[i];
  for (int i = n - 1; i >= 0; --i) suffix[i] = T[i] * suffix[i + 1];
  for (int i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) grad_c[3 * i + a] = up_c[a] * prefix[i];
    const double t_grad = up_t * prefix[i] * suffix[i + 1];
    double running = 1.0, color_term = 0.0;
    for (int k = i + 1; k < n; ++k) {
      color_term += running * dot3(up_c, rgb + 3 * k);
      running *= T[k];
    }
    grad_t[i] = t_grad + prefix[i] * color_term;
  }
}

/* train.cpp:20-32 */
double or_loss_transmittance(double T, double eps) { return -log(1.0 - smin(T, 1.0 - eps)); }
double or_loss_transmittance_grad(double T, double eps) { return 1.0 / (1.0 - smin(T, 1.0 - eps)); }

/* train.cpp:38-54 */
double or_loss_distortion(const double* w, const double* s, const double* ds, int n) {
  double w_prefix = 0.0, m_prefix = 0.0, pair = 0.0, interval = 0.0;
  for (int k = 0; k < n; ++k) {
    pair += 2.0 * w[k] * (s[k] * w_prefix - m_prefix);
    interval += w[k] * w[k] * ds[k];
    w_prefix += w[k];
    m_prefix += w[k] * s[k];
  }
  return pair + interval / 3.0;
}

/* train.cpp:56-75 */
void or_loss_distortion_grad(const double* w, const double* s, const double* ds, int n,
                             double* g) {
  double w_total = 0.0, m_total = 0.0;
  for (int k = 0; k < n; ++k) {
    w_total += w[k];
    m_total += w[k] * s[k];
  }
  double w_prefix = 0.0, m_prefix = 0.0;
  for (int k = 0; k < n; ++k) {
    const double w_suffix = w_total - w_prefix - w[k];
    const double m_suffix = m_total - m_prefix - w[k] * s[k];
    g[k] = 2.0 * (s[k] * w_prefix - m_prefix) + 2.0 * (m_suffix - s[k] * w_suffix) +
           (2.0 / 3.0) * w[k] * ds[k];
    w_prefix += w[k];
    m_prefix += w[k] * s[k];
  }
}

/* render.cpp:145-179 */
void or_local_render_backward(const double* delta, const double* rgb, const double* alpha,
                              const double* prefix, int n, const double up_c[3], double up_t,
                              const double* weight_up, double* sigma_grad, double* color_grad) {
  double tail_color = 0.0, tail_trans = 1.0;
  for (int k = n - 1; k >= 0; --k) {
    const double a = alpha[k], pf = prefix[k];
    const double u = dot3(up_c, rgb + 3 * k) + (weight_up ? weight_up[k] : 0.0);
    const double alpha_grad = pf * (u - tail_color) - up_t * pf * tail_trans;
    sigma_grad[k] = alpha_grad * delta[k] * (1.0 - a);
    for (int c = 0; c < 3; ++c) color_grad[3 * k + c] = up_c[c] * (pf * a);
    tail_color = a * u + (1.0 - a) * tail_color;
    tail_trans *= 1.0 - a;
  }
}

/* train.cpp:77-80 */
double or_lr_at(const dg_run_config* cfg, uint64_t step) {
  const double progress = cfg->total_steps == 0 ? 1.0 : (double)step / (double)cfg->total_steps;
  return cfg->lr_end + 0.5 * (cfg->lr_start - cfg->lr_end) * (1.0 + cos(M_PI * progress));
}

/* train.cpp:91-115 (t is the post-increment step count) */
void or_adam_step(double* p, double* g, double* m, double* v, uint64_t n, double lr, double b1,
                  double b2, double eps, uint64_t t) {
  const double bias1 = 1.0 - pow(b1, (double)t);
  const double bias2 = 1.0 - pow(b2, (double)t);
  for (uint64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    const double m_hat = m[i] / bias1;
    const double v_hat = v[i] / bias2;
    p[i] -= lr * m_hat / (sqrt(v_hat) + eps);
  }
}

/* =================================================================== composed run */
struct or_run {
  or_model m;
  double* params[DG_MAX_PARTITIONS];
  double* grads[DG_MAX_PARTITIONS];
  double* last_grads[DG_MAX_PARTITIONS];
  double* abs_grads[DG_MAX_PARTITIONS];
  double* am[DG_MAX_PARTITIONS];
  double* av[DG_MAX_PARTITIONS];
  uint64_t at[DG_MAX_PARTITIONS];
  uint64_t wstep[DG_MAX_PARTITIONS];
  uint8_t* occ_bits[DG_MAX_PARTITIONS][2];
  double* occ_den[DG_MAX_PARTITIONS][2];
  double occ_thr[DG_MAX_PARTITIONS][2];
  or_mt64 occ_rng[DG_MAX_PARTITIONS];
  uint32_t n_images;
  double* app;
  /* test-only per-sample log of one region's training samples (or_run_sample_log) */
  int32_t slog_region;
  double* slog;
  uint64_t slog_cap, slog_n;
  /* test-only ReLU decisions per training sample of a region (or_run_mask_override) */
  const uint32_t* movr[DG_MAX_PARTITIONS];
  uint64_t movr_n[DG_MAX_PARTITIONS];
  uint64_t ovr_units; /* over the last train step: decisions against the sign of z, largest |z| */
  double ovr_max_z;
};

int or_run_mask_override(or_run* r, uint32_t region, const uint32_t* words, uint64_t n) {
  if (region >= DG_MAX_PARTITIONS) return or_fail("mask override: region out of range");
  r->movr[region] = words;
  r->movr_n[region] = words ? n : 0;
  return 0;
}

static const uint32_t* mask_ovr(const or_run* r, uint32_t g, uint64_t k) {
  return r->movr[g] && k < r->movr_n[g] ? r->movr[g] + 6 * k : NULL;
}

void or_run_override_stats(const or_run* r, uint64_t* units, double* max_abs_z) {
  *units = r->ovr_units;
  *max_abs_z = r->ovr_max_z;
}

/* Count the units of one overridden sample whose decision goes against the sign of z (the
 * ReLU layers: h1 always, c1 / c2 in the fine field). */
static void ovr_account(or_run* r, const or_field_cache* c, int coarse) {
  if (!c->ovr) return;
  const double* pre[3] = {c->h1, c->c1, c->c2};
  for (int q = 0; q < (coarse ? 1 : 3); ++q)
    for (int u = 0; u < 64; ++u)
      if (((c->mask[q] >> u) & 1u) != (pre[q][u] > 0.0 ? 1u : 0u)) {
        r->ovr_units += 1;
        r->ovr_max_z = fmax(r->ovr_max_z, fabs(pre[q][u]));
      }
}

int or_run_sample_log(or_run* r, int32_t region, double* buf, uint64_t capacity) {
  r->slog_region = region;
  r->slog = buf;
  r->slog_cap = capacity;
  r->slog_n = 0;
  return 0;
}
uint64_t or_run_sample_log_count(const or_run* r) { return r->slog_n; }

const or_model* or_run_model(const or_run* r) { return &r->m; }
double* or_run_params(or_run* r, uint32_t g) { return r->params[g]; }
double* or_run_grads(or_run* r, uint32_t g) { return r->last_grads[g]; }
double* or_run_abs_grads(or_run* r, uint32_t g) { return r->abs_grads[g]; }
double* or_run_adam_m(or_run* r, uint32_t g) { return r->am[g]; }
double* or_run_adam_v(or_run* r, uint32_t g) { return r->av[g]; }
uint64_t* or_run_adam_t(or_run* r, uint32_t g) { return &r->at[g]; }
uint64_t* or_run_worker_step(or_run* r, uint32_t g) { return &r->wstep[g]; }
uint8_t* or_run_occ_bits(or_run* r, uint32_t g, uint32_t c) { return r->occ_bits[g][c]; }
double* or_run_occ_density(or_run* r, uint32_t g, uint32_t c) { return r->occ_den[g][c]; }
double* or_run_occ_threshold(or_run* r, uint32_t g, uint32_t c) { return &r->occ_thr[g][c]; }

static uint64_t occ_cells(const or_run* r, uint32_t g, uint32_t c) {
  const or_shape s = r->m.occ_shape[g][c];
  return (uint64_t)s.nx * s.ny * s.nz;
}

void or_run_set_occupancy(or_run* r, uint32_t g, uint32_t c, const uint8_t* bits) {
  const uint64_t n = occ_cells(r, g, c);
  for (uint64_t i = 0; i < n; ++i) {
    r->occ_den[g][c][i] = bits[i] ? r->occ_thr[g][c] : 0.0;
    r->occ_bits[g][c][i] = r->occ_den[g][c][i] >= r->occ_thr[g][c] ? 1 : 0;
  }
}

or_run* or_run_create(const dg_run_config* cfg, uint32_t n_images, const double* app_rows) {
  or_run* r = (or_run*)calloc(1, sizeof(or_run));
  if (!r) return NULL;
  if (or_model_init(&r->m, cfg) != 0) {
    free(r);
    return NULL;
  }
  for (uint32_t g = 0; g < r->m.P; ++g) {
    const uint64_t n = r->m.nparams[g];
    r->params[g] = (double*)calloc(n, sizeof(double));
    r->grads[g] = (double*)calloc(n, sizeof(double));
    r->last_grads[g] = (double*)calloc(n, sizeof(double));
    r->abs_grads[g] = (double*)calloc(n, sizeof(double));
    r->am[g] = (double*)calloc(n, sizeof(double));
    r->av[g] = (double*)calloc(n, sizeof(double));
    for (int c = 0; c < 2; ++c) {
      const uint64_t cells = occ_cells(r, g, (uint32_t)c);
      r->occ_bits[g][c] = (uint8_t*)malloc(cells);
      r->occ_den[g][c] = (double*)malloc(cells * sizeof(double));
      /* worker.cpp:194-200: threshold early*scale, fill_occupied */
      r->occ_thr[g][c] = cfg->occ_threshold_early * cfg->occ_threshold_scale;
      for (uint64_t i = 0; i < cells; ++i) {
        r->occ_den[g][c][i] = r->occ_thr[g][c];
        r->occ_bits[g][c][i] = 1;
      }
    }
    or_rng_init(&r->occ_rng[g], or_counter_hash(cfg->seed, 0x0cc0, g, 0));
  }
  r->n_images = n_images;
  r->app = (double*)malloc(sizeof(double) * (size_t)(n_images ? n_images : 1) * cfg->appearance_dim);
  if (n_images) memcpy(r->app, app_rows, sizeof(double) * (size_t)n_images * cfg->appearance_dim);
  return r;
}

void or_run_destroy(or_run* r) {
  if (!r) return;
  for (uint32_t g = 0; g < r->m.P; ++g) {
    free(r->params[g]);
    free(r->grads[g]);
    free(r->last_grads[g]);
    free(r->abs_grads[g]);
    free(r->am[g]);
    free(r->av[g]);
    for (int c = 0; c < 2; ++c) {
      free(r->occ_bits[g][c]);
      free(r->occ_den[g][c]);
    }
  }
  free(r->app);
  free(r);
}

static inline double fround(double v, int f32) { return f32 ? (double)(float)v : v; }

/* Per-ray dispatch record as a worker sees it after the wire (wire.cpp:29-68). */
typedef struct {
  uint64_t ray_id;
  double o[3], d[3], gt[3];
  uint32_t image;
  int nseg;
  uint32_t region[DG_MAX_SEGMENTS];
  double te[DG_MAX_SEGMENTS], tx[DG_MAX_SEGMENTS];
} or_dray;

/* grid.cpp:201-229 decay_and_update + worker.cpp:549-562 update_occupancy */
static void occupancy_update(or_run* r, uint32_t g) {
  const dg_run_config* cfg = &r->m.cfg;
  const uint64_t step = r->wstep[g];
  if (!cfg->occupancy_updates) return;
  if (step == 0 || step % cfg->occ_update_interval != 0) return;
  const double threshold = (step < cfg->occ_threshold_switch_step ? cfg->occ_threshold_early
                                                                    : cfg->occ_threshold_late) *
                           cfg->occ_threshold_scale;
  const int warm_up = step <= cfg->occ_warmup_steps;
  or_mt64* rng = &r->occ_rng[g];
  for (int c = 0; c < 2; ++c) { /* set_threshold: recompute the bitfield */
    r->occ_thr[g][c] = threshold;
    const uint64_t n = occ_cells(r, g, (uint32_t)c);
    for (uint64_t i = 0; i < n; ++i) r->occ_bits[g][c][i] = r->occ_den[g][c][i] >= threshold;
  }
  for (int c = 0; c < 2; ++c) {
    const or_box* box = c == 0 ? &r->m.fine[g] : &r->m.coarse[g];
    const or_shape sh = r->m.occ_shape[g][c];
    const or_field_layout* f = &r->m.field[g][c];
    const double* params = r->params[g] + (c == 0 ? 0 : r->m.field[g][0].size);
    const uint64_t total = occ_cells(r, g, (uint32_t)c);
    double* den = r->occ_den[g][c];
    uint8_t* bits = r->occ_bits[g][c];
    const double cell[3] = {(box->hi[0] - box->lo[0]) / (double)sh.nx,
                            (box->hi[1] - box->lo[1]) / (double)sh.ny,
                            (box->hi[2] - box->lo[2]) / (double)sh.nz};
#define OR_SAMPLE_CELL(IDX)                                                                \
  do {                                                                                     \
    const uint64_t idx_ = (IDX);                                                           \
    const uint32_t ix_ = (uint32_t)(idx_ % sh.nx);                                         \
    const uint32_t iy_ = (uint32_t)((idx_ / sh.nx) % sh.ny);                               \
    const uint32_t iz_ = (uint32_t)(idx_ / ((uint64_t)sh.nx * sh.ny));                     \
    double lo_[3], hi_[3], pw_[3], pu_[3];                                                 \
    const uint32_t ii_[3] = {ix_, iy_, iz_};                                               \
    for (int a_ = 0; a_ < 3; ++a_) {                                                       \
      lo_[a_] = box->lo[a_] + cell[a_] * (double)ii_[a_];                                  \
      hi_[a_] = lo_[a_] + cell[a_];                                                        \
    }                                                                                      \
    for (int a_ = 0; a_ < 3; ++a_) pw_[a_] = or_rng_uniform_range(rng, lo_[a_], hi_[a_]);  \
    for (int a_ = 0; a_ < 3; ++a_)                                                         \
      pu_[a_] = sclamp((pw_[a_] - box->lo[a_]) / (box->hi[a_] - box->lo[a_]), 0.0, 1.0);   \
    or_field_cache fc_ = {0};                                                                 \
    const double zero3_[3] = {0.0, 0.0, 1.0};                                              \
    or_field_forward(f, params, pu_, zero3_, r->app, &fc_);                                \
    den[idx_] = smax(den[idx_] * cfg->occ_decay, fc_.sigma);                               \
  } while (0)
    if (warm_up) {
      for (uint64_t i = 0; i < total; ++i) OR_SAMPLE_CELL(i);
    } else {
      uint64_t* occupied = (uint64_t*)malloc(sizeof(uint64_t) * (total ? total : 1));
      uint64_t n_occ = 0;
      for (uint64_t i = 0; i < total; ++i)
        if (bits[i]) occupied[n_occ++] = i;
      const uint64_t n_uniform = total / 4 > 1 ? total / 4 : 1;
      for (uint64_t i = 0; i < n_uniform; ++i) {
        const uint64_t pick = or_mt64_next(rng) % total;
        OR_SAMPLE_CELL(pick);
      }
      if (n_occ)
        for (uint64_t i = 0; i < n_uniform; ++i) {
          const uint64_t pick = occupied[or_mt64_next(rng) % n_occ];
          OR_SAMPLE_CELL(pick);
        }
      free(occupied);
    }
#undef OR_SAMPLE_CELL
    for (uint64_t i = 0; i < total; ++i) bits[i] = den[i] >= threshold ? 1 : 0;
  }
}

/* shade one sample (worker.cpp:35-52) */
static void shade(or_run* r, uint32_t g, int cascade, const or_dray* dr, double t,
                  const double* app, or_field_cache* fc, const uint32_t* ovr) {
  const or_box* box = cascade == 0 ? &r->m.fine[g] : &r->m.coarse[g];
  double p[3];
  or_normalized_point(box, dr->o, dr->d, t, p);
  fc->ovr = ovr != NULL;
  for (int q = 0; q < 3 && ovr; ++q) fc->mask[q] = (uint64_t)ovr[2 * q] | ((uint64_t)ovr[2 * q + 1] << 32);
  const double* params = r->params[g] + (cascade == 0 ? 0 : r->m.field[g][0].size);
  or_field_forward(&r->m.field[g][cascade], params, p, dr->d, app, fc);
}

#define OR_SCAP 65536

/* DistributedRun::training_step (worker.cpp:730-755) with every Worker's
 * handle_training_batch (worker.cpp:251-401) and backward_ray (403-522). */
int or_run_train_step(or_run* r, const double* origin, const double* dir, const double* color_gt,
                      const uint32_t* image_id, uint64_t n, uint64_t step, double* stats) {
  const or_model* m = &r->m;
  const dg_run_config* cfg = &m->cfg;
  const int f32 = cfg->wire_f32 != 0;
  if (cfg->distortion_cross_correction) return or_fail("oracle: cross correction unsupported");
  or_dray* rays = (or_dray*)calloc(n ? n : 1, sizeof(or_dray));
  uint64_t dropped = 0;
  r->ovr_units = 0;
  r->ovr_max_z = 0.0;
  /* plan_batch (worker.cpp:141-165) + wire rounding (wire.cpp:29-46) */
  for (uint64_t i = 0; i < n; ++i) {
    or_dray* d = &rays[i];
    const double* o = origin + 3 * i;
    const double* dd = dir + 3 * i;
    d->nseg = or_segment_ray(m, o, dd, d->region, d->te, d->tx);
    if (d->nseg == 0) {
      ++dropped;
      continue;
    }
    d->ray_id = i;
    for (int a = 0; a < 3; ++a) {
      d->o[a] = fround(o[a], f32);
      d->d[a] = fround(dd[a], f32);
      d->gt[a] = fround(color_gt[3 * i + a], f32);
    }
    d->image = image_id ? image_id[i] : 0;
    for (int s = 0; s < d->nseg; ++s) {
      d->te[s] = fround(d->te[s], f32);
      d->tx[s] = fround(d->tx[s], f32);
    }
  }
  /* own partial per (ray, segment order), quantized (wire.cpp:207-217) */
  double* prgb = (double*)calloc((n ? n : 1) * DG_MAX_SEGMENTS * 3, sizeof(double));
  double* pT = (double*)calloc((n ? n : 1) * DG_MAX_SEGMENTS, sizeof(double));
  static double st[OR_SCAP], sd[OR_SCAP], ssig[OR_SCAP], srgb[3 * OR_SCAP];
  static double salpha[OR_SCAP], sprefix[OR_SCAP], sw[OR_SCAP], ss[OR_SCAP], sds[OR_SCAP],
      swup[OR_SCAP], sgs[OR_SCAP], sgc[3 * OR_SCAP];
  static uint8_t sc[OR_SCAP];
  static or_field_cache fcache[2048];
  int rc = 0;
  double loss_rgb[DG_MAX_PARTITIONS], loss_t[DG_MAX_PARTITIONS], loss_d[DG_MAX_PARTITIONS];
  /* Phase 1 for every worker (independent across workers). */
  for (uint32_t g = 0; g < m->P && rc == 0; ++g) {
    uint64_t ks = 0; /* the region's sample ordinal (mask override index) */
    for (uint64_t i = 0; i < n; ++i) {
      const or_dray* d = &rays[i];
      int mo = -1;
      for (int s = 0; s < d->nseg; ++s)
        if (d->region[s] == g) mo = s;
      if (mo < 0) continue;
      if (d->image >= r->n_images) {
        rc = or_fail("appearance: unknown image id");
        break;
      }
      const double* app = r->app + (size_t)d->image * cfg->appearance_dim;
      const int ns = or_cascade_march(m, g, r->occ_bits[g][0], r->occ_bits[g][1], d->o, d->d,
                                      d->te[mo], d->tx[mo], 1, d->ray_id, step, st, sd, sc, OR_SCAP);
      if (ns < 0) {
        rc = -1;
        break;
      }
      for (int k = 0; k < ns; ++k) {
        or_field_cache fc;
        shade(r, g, sc[k], d, st[k], app, &fc, mask_ovr(r, g, ks++));
        ssig[k] = fc.sigma;
        for (int a = 0; a < 3; ++a) srgb[3 * k + a] = fc.rgb[a];
      }
      double c[3], T;
      or_local_render(st, sd, ssig, srgb, ns, c, &T, NULL, NULL, NULL);
      for (int a = 0; a < 3; ++a) prgb[(i * DG_MAX_SEGMENTS + mo) * 3 + a] = fround(c[a], f32);
      pT[i * DG_MAX_SEGMENTS + mo] = fround(T, f32);
    }
  }
  /* Phase 3 per worker: merge, losses, backward (worker.cpp:362-385, 403-522). */
  for (uint32_t g = 0; g < m->P && rc == 0; ++g) {
    loss_rgb[g] = loss_t[g] = loss_d[g] = 0.0;
    memset(r->abs_grads[g], 0, sizeof(double) * m->nparams[g]);
    g_abs = r->abs_grads[g];
    g_gbase = r->grads[g];
    uint64_t ks = 0;
    for (uint64_t i = 0; i < n; ++i) {
      const or_dray* d = &rays[i];
      int mo = -1;
      for (int s = 0; s < d->nseg; ++s)
        if (d->region[s] == g) mo = s;
      if (mo < 0) continue;
      const int nsg = d->nseg;
      const double* prgb_i = prgb + i * DG_MAX_SEGMENTS * 3;
      const double* pT_i = pT + i * DG_MAX_SEGMENTS;
      double C[3], T;
      or_merge_forward(prgb_i, pT_i, NULL, nsg, C, &T, NULL);
      if (d->region[0] == g) {
        const double diff[3] = {C[0] - d->gt[0], C[1] - d->gt[1], C[2] - d->gt[2]};
        loss_rgb[g] += dot3(diff, diff);
        loss_t[g] += or_loss_transmittance(T, cfg->transmittance_clamp);
      }
      const double up_c[3] = {(C[0] - d->gt[0]) * 2.0, (C[1] - d->gt[1]) * 2.0,
                              (C[2] - d->gt[2]) * 2.0};
      const double up_t =
          cfg->lambda_transmittance * or_loss_transmittance_grad(T, cfg->transmittance_clamp);
      double gc[DG_MAX_SEGMENTS * 3], gt_[DG_MAX_SEGMENTS];
      or_merge_backward(up_c, up_t, prgb_i, pT_i, nsg, gc, gt_);
      /* recompute the local forward with caches */
      const double* app = r->app + (size_t)d->image * cfg->appearance_dim;
      const int ns = or_cascade_march(m, g, r->occ_bits[g][0], r->occ_bits[g][1], d->o, d->d,
                                      d->te[mo], d->tx[mo], 1, d->ray_id, step, st, sd, sc, OR_SCAP);
      if (ns > 2048) {
        rc = or_fail("oracle: too many samples per segment");
        break;
      }
      for (int k = 0; k < ns; ++k) {
        shade(r, g, sc[k], d, st[k], app, &fcache[k], mask_ovr(r, g, ks++));
        ovr_account(r, &fcache[k], r->m.field[g][sc[k]].coarse);
        ssig[k] = fcache[k].sigma;
        for (int a = 0; a < 3; ++a) srgb[3 * k + a] = fcache[k].rgb[a];
      }
      double cl[3], Tl;
      or_local_render(st, sd, ssig, srgb, ns, cl, &Tl, NULL, salpha, sprefix);
      /* local_distortion_inputs (worker.cpp:62-75) */
      const double ray_t0 = d->te[0], ray_t1 = d->tx[nsg - 1];
      const double inv_span = 1.0 / (ray_t1 - ray_t0);
      for (int k = 0; k < ns; ++k) {
        sw[k] = sprefix[k] * salpha[k];
        ss[k] = (st[k] - ray_t0) * inv_span;
        sds[k] = sd[k] * inv_span;
        swup[k] = 0.0;
      }
      if (ns > 0) {
        loss_d[g] += or_loss_distortion(sw, ss, sds, ns);
        if (cfg->lambda_distortion > 0.0) {
          or_loss_distortion_grad(sw, ss, sds, ns, swup);
          for (int k = 0; k < ns; ++k) swup[k] *= cfg->lambda_distortion;
        }
      }
      or_local_render_backward(sd, srgb, salpha, sprefix, ns, gc + 3 * mo, gt_[mo], swup, sgs, sgc);
      for (int k = 0; k < ns; ++k) {
        const int casc = sc[k];
        const or_field_layout* f = &m->field[g][casc];
        const uint64_t off = casc == 0 ? 0 : m->field[g][0].size;
        double* rec = NULL;
        if (r->slog && (int32_t)g == r->slog_region && r->slog_n < r->slog_cap) {
          /* pos 3 | features 32 | sigma, rgb | dsigma, drgb | d features 32  (OR_SLOG_REC) */
          rec = r->slog + r->slog_n * OR_SLOG_REC;
          memset(rec, 0, sizeof(double) * OR_SLOG_REC);
          memcpy(rec, fcache[k].point, sizeof(double) * 3);
          memcpy(rec + 3, fcache[k].enc, sizeof(double) * f->enc_width);
          rec[35] = fcache[k].sigma;
          memcpy(rec + 36, fcache[k].rgb, sizeof(double) * 3);
          rec[39] = sgs[k];
          memcpy(rec + 40, sgc + 3 * k, sizeof(double) * 3);
          const double* pre[3] = {fcache[k].h1, fcache[k].c1, fcache[k].c2};
          for (int q = 0; q < 3; ++q) {
            uint32_t w0 = 0, w1 = 0;
            double mn = INFINITY;
            for (int u = 0; u < 64; ++u) {
              if (pre[q][u] > 0.0) {
                if (u < 32) w0 |= 1u << u;
                else w1 |= 1u << (u - 32);
              }
              mn = fmin(mn, fabs(pre[q][u]));
            }
            rec[75 + 2 * q] = (double)w0;
            rec[76 + 2 * q] = (double)w1;
            rec[81 + q] = mn;
          }
          g_enc_grad_out = rec + 43;
          ++r->slog_n;
        }
        or_field_backward(f, r->params[g] + off, r->grads[g] + off, &fcache[k], sgs[k], sgc + 3 * k);
        g_enc_grad_out = NULL;
      }
    }
    g_abs = NULL;
    g_gbase = NULL;
    if (rc) break;
    /* apply_updates (worker.cpp:524-547): Adam with lr at the pre-increment step_ */
    const double lr = or_lr_at(cfg, r->wstep[g]);
    r->at[g] += 1;
    memcpy(r->last_grads[g], r->grads[g], sizeof(double) * m->nparams[g]);
    or_adam_step(r->params[g], r->grads[g], r->am[g], r->av[g], m->nparams[g], lr,
                 cfg->adam_beta1, cfg->adam_beta2, cfg->adam_eps, r->at[g]);
    memset(r->grads[g], 0, sizeof(double) * m->nparams[g]);
    r->wstep[g] = step + 1;
    occupancy_update(r, g);
  }
  if (rc == 0) {
    stats[0] = stats[1] = stats[2] = 0.0;
    for (uint32_t g = 0; g < m->P; ++g) { /* ControlSync through the wire (wire.cpp:117-128) */
      stats[0] += fround(loss_rgb[g], f32);
      stats[1] += fround(loss_t[g], f32);
      stats[2] += fround(loss_d[g], f32);
    }
    stats[3] = or_lr_at(cfg, step);
    stats[4] = (double)(n - dropped);
    stats[5] = (double)dropped;
  }
  free(rays);
  free(prgb);
  free(pT);
  return rc;
}

/* DistributedRun::dispatch_eval + Worker::handle_eval_request (worker.cpp:564-600,757-829),
 * with the driver's early termination (worker.cpp:815-818) and, when attribution != NULL, the
 * region-attribution colour of evaluate_image (worker.cpp:864-878) over the merged partials. */
int or_run_eval_rays_ex(or_run* r, const double* origin, const double* dir, uint64_t n,
                        const double* appearance, double* rgb, double* T, double* depth,
                        double* attribution);
int or_run_eval_rays(or_run* r, const double* origin, const double* dir, uint64_t n,
                     const double* appearance, double* rgb, double* T, double* depth) {
  return or_run_eval_rays_ex(r, origin, dir, n, appearance, rgb, T, depth, NULL);
}

int or_run_eval_rays_ex(or_run* r, const double* origin, const double* dir, uint64_t n,
                        const double* appearance, double* rgb, double* T, double* depth,
                        double* attribution) {
  const or_model* m = &r->m;
  const dg_run_config* cfg = &m->cfg;
  const int f32 = cfg->wire_f32 != 0;
  double app[64];
  for (uint32_t k = 0; k < cfg->appearance_dim && k < 64; ++k) app[k] = fround(appearance[k], f32);
  static double st[OR_SCAP], sd[OR_SCAP], ssig[OR_SCAP], srgb[3 * OR_SCAP];
  static uint8_t sc[OR_SCAP];
  for (uint64_t i = 0; i < n; ++i) {
    or_dray d;
    memset(&d, 0, sizeof d);
    d.nseg = or_segment_ray(m, origin + 3 * i, dir + 3 * i, d.region, d.te, d.tx);
    rgb[3 * i] = rgb[3 * i + 1] = rgb[3 * i + 2] = 0.0;
    T[i] = 1.0;
    depth[i] = 0.0;
    if (attribution) attribution[3 * i] = attribution[3 * i + 1] = attribution[3 * i + 2] = 0.0;
    if (d.nseg == 0) continue;
    d.ray_id = i;
    for (int a = 0; a < 3; ++a) {
      d.o[a] = fround(origin[3 * i + a], f32);
      d.d[a] = fround(dir[3 * i + a], f32);
    }
    double prgb[DG_MAX_SEGMENTS * 3], pT[DG_MAX_SEGMENTS], pdep[DG_MAX_SEGMENTS];
    for (int s = 0; s < d.nseg; ++s) {
      const uint32_t g = d.region[s];
      const double te = fround(d.te[s], f32), tx = fround(d.tx[s], f32);
      const int ns = or_cascade_march(m, g, r->occ_bits[g][0], r->occ_bits[g][1], d.o, d.d, te, tx,
                                      0, i, 0, st, sd, sc, OR_SCAP);
      if (ns < 0) return -1;
      for (int k = 0; k < ns; ++k) {
        or_field_cache fc;
        shade(r, g, sc[k], &d, st[k], app, &fc, NULL);
        ssig[k] = fc.sigma;
        for (int a = 0; a < 3; ++a) srgb[3 * k + a] = fc.rgb[a];
      }
      double c[3], tt, dep;
      or_local_render(st, sd, ssig, srgb, ns, c, &tt, &dep, NULL, NULL);
      for (int a = 0; a < 3; ++a) prgb[3 * s + a] = fround(c[a], f32);
      pT[s] = fround(tt, f32);
      pdep[s] = fround(dep, f32);
    }
    int used = d.nseg;
    if (cfg->eval_early_termination) { /* worker.cpp:815-818: keep the entry that crosses */
      double prefix = 1.0;
      for (int s = 0; s < d.nseg; ++s) {
        prefix *= pT[s];
        if (prefix < cfg->eval_termination_threshold) {
          used = s + 1;
          break;
        }
      }
    }
    double C[3], TT, D;
    or_merge_forward(prgb, pT, pdep, used, C, &TT, &D);
    for (int a = 0; a < 3; ++a) rgb[3 * i + a] = C[a];
    T[i] = TT;
    depth[i] = D;
    if (attribution) { /* worker.cpp:864-878 */
      double prefix = 1.0, at[3] = {0.0, 0.0, 0.0};
      for (int s = 0; s < used; ++s) {
        const double weight = prefix * (1.0 - pT[s]);
        const double hue = (double)d.region[s] * 0.61803398875;
        const double pal[3] = {0.5 + 0.5 * cos(6.2831853 * hue), 0.5 + 0.5 * cos(6.2831853 * (hue + 1.0 / 3.0)),
                               0.5 + 0.5 * cos(6.2831853 * (hue + 2.0 / 3.0))};
        for (int a = 0; a < 3; ++a) at[a] += pal[a] * weight;
        prefix *= pT[s];
      }
      for (int a = 0; a < 3; ++a) attribution[3 * i + a] = at[a];
    }
  }
  return 0;
}

/* ---- stage wrappers for the per-stage parity tests (flat partition arrays) ---- */
uint64_t or_model_size(void) { return sizeof(or_model); }

int or_stage_cascade_march(const or_model* m, uint32_t region, const uint8_t* occ_fine,
                           const uint8_t* occ_coarse, const double* o, const double* d,
                           const double* t0, const double* t1, const uint64_t* ray_id, uint64_t n,
                           int jitter, uint64_t batch_id, uint32_t* counts, double* t,
                           double* delta, uint8_t* cascade, uint64_t cap) {
  uint64_t off = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const int k = or_cascade_march(m, region, occ_fine, occ_coarse, o + 3 * i, d + 3 * i, t0[i],
                                   t1[i], jitter, ray_id[i], batch_id, t + off, delta + off,
                                   cascade + off, (int)(cap - off));
    if (k < 0) return -1;
    counts[i] = (uint32_t)k;
    off += (uint64_t)k;
  }
  return 0;
}

void or_stage_encode(const or_model* m, uint32_t region, uint32_t cascade, const double* params,
                     const double* pts, uint64_t n, double* out, uint32_t* rows) {
  const or_field_layout* f = &m->field[region][cascade];
  const double* base = params ? params + (cascade == 0 ? 0 : m->field[region][0].size) : NULL;
  for (uint64_t i = 0; i < n; ++i)
    or_encode(&f->grid, base, pts + 3 * i, out + i * f->enc_width,
              rows ? rows + i * f->grid.L * 8 : NULL);
}

void or_stage_field_forward(const or_model* m, uint32_t region, uint32_t cascade,
                            const double* params, const double* pts, const double* dirs,
                            const double* app, uint64_t n, double* sigma, double* rgb) {
  const or_field_layout* f = &m->field[region][cascade];
  const double* base = params + (cascade == 0 ? 0 : m->field[region][0].size);
  or_field_cache c = {0};
  for (uint64_t i = 0; i < n; ++i) {
    or_field_forward(f, base, pts + 3 * i, dirs + 3 * i, app + i * m->cfg.appearance_dim, &c);
    sigma[i] = c.sigma;
    for (int k = 0; k < 3; ++k) rgb[3 * i + k] = c.rgb[k];
  }
}

void or_stage_field_backward(const or_model* m, uint32_t region, uint32_t cascade,
                             const double* params, double* grads, const double* pts,
                             const double* dirs, const double* app, const double* dsigma,
                             const double* drgb, uint64_t n) {
  const or_field_layout* f = &m->field[region][cascade];
  const uint64_t off = cascade == 0 ? 0 : m->field[region][0].size;
  or_field_cache c = {0};
  for (uint64_t i = 0; i < n; ++i) {
    or_field_forward(f, params + off, pts + 3 * i, dirs + 3 * i, app + i * m->cfg.appearance_dim, &c);
    or_field_backward(f, params + off, grads + off, &c, dsigma[i], drgb + 3 * i);
  }
}


/* ======================================================================== ray cache */
/* partition.cpp:30-33: normalize(rotation * ((x - cx) / fx, (y - cy) / fy, 1)); Mat3 * Vec3
 * row by row left to right (vecmath.hpp), normalize = v / sqrt(dot(v, v)). */
void or_make_pixel_ray(const or_camera* cam, const uint8_t* rgb, uint32_t x, uint32_t y, double origin[3],
                       double dir[3], double color[3], uint32_t* image_id, uint64_t* pixel_id) {
  const double px = (double)x + 0.5, py = (double)y + 0.5; /* dataset.cpp:317 */
  const double c[3] = {(px - cam->cx) / cam->fx, (py - cam->cy) / cam->fy, 1.0};
  double v[3];
  for (int r = 0; r < 3; ++r)
    v[r] = cam->rotation[3 * r] * c[0] + cam->rotation[3 * r + 1] * c[1] + cam->rotation[3 * r + 2] * c[2];
  const double len = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  for (int a = 0; a < 3; ++a) {
    origin[a] = cam->translation[a];
    dir[a] = v[a] / len;
    /* Image::pixel_channel, dataset.hpp:19-21 */
    color[a] = (double)rgb[((size_t)y * cam->width + x) * 3 + a] / 255.0;
  }
  *image_id = cam->image_id;
  *pixel_id = ((uint64_t)cam->image_id << 32) | ((uint64_t)y * cam->width + x);
}

struct or_ray_cache {
  uint64_t capacity, size, cursor;
  or_mt64 refresh_rng, draw_rng;
  uint32_t n_images, n_train;
  const or_camera* cams;
  const uint8_t* const* images;
  uint32_t* train;
  double *origin, *dir, *color;
  uint32_t* image_id;
  uint64_t* pixel_id;
};

/* train.cpp:117-121: Rng(splitmix64(seed ^ tag)) per stream (Rng seeds its engine with
 * splitmix64 of its argument again, rng.hpp:34). */
or_ray_cache* or_ray_cache_create(const or_camera* cams, const uint8_t* const* images, uint32_t n_images,
                                  uint64_t capacity, uint64_t seed) {
  if (capacity == 0 || n_images == 0) return NULL;
  or_ray_cache* c = (or_ray_cache*)calloc(1, sizeof(or_ray_cache));
  c->capacity = capacity;
  or_rng_init(&c->refresh_rng, or_splitmix64(seed ^ 0x5261794361636865ull));
  or_rng_init(&c->draw_rng, or_splitmix64(seed ^ 0x4261746368447277ull));
  c->n_images = n_images;
  c->cams = cams;
  c->images = images;
  c->train = (uint32_t*)malloc(sizeof(uint32_t) * n_images);
  for (uint32_t i = 0; i < n_images; ++i)
    if (cams[i].is_train) c->train[c->n_train++] = i;
  c->origin = (double*)malloc(sizeof(double) * 3 * capacity);
  c->dir = (double*)malloc(sizeof(double) * 3 * capacity);
  c->color = (double*)malloc(sizeof(double) * 3 * capacity);
  c->image_id = (uint32_t*)malloc(sizeof(uint32_t) * capacity);
  c->pixel_id = (uint64_t*)malloc(sizeof(uint64_t) * capacity);
  return c;
}

void or_ray_cache_destroy(or_ray_cache* c) {
  if (!c) return;
  free(c->train);
  free(c->origin);
  free(c->dir);
  free(c->color);
  free(c->image_id);
  free(c->pixel_id);
  free(c);
}

uint64_t or_ray_cache_size(const or_ray_cache* c) { return c->size; }

/* train.cpp:123-143 */
int or_ray_cache_refresh(or_ray_cache* c, uint64_t count) {
  if (c->n_train == 0) return DG_EINVAL;
  for (uint64_t i = 0; i < count; ++i) {
    const uint32_t img = c->train[or_mt64_next(&c->refresh_rng) % c->n_train];
    const or_camera* cam = &c->cams[img];
    const uint32_t x = (uint32_t)(or_mt64_next(&c->refresh_rng) % cam->width);
    const uint32_t y = (uint32_t)(or_mt64_next(&c->refresh_rng) % cam->height);
    uint64_t slot;
    if (c->size < c->capacity) {
      slot = c->size++;
    } else {
      slot = c->cursor;
      c->cursor = (c->cursor + 1) % c->capacity;
    }
    or_make_pixel_ray(cam, c->images[img], x, y, c->origin + 3 * slot, c->dir + 3 * slot,
                      c->color + 3 * slot, c->image_id + slot, c->pixel_id + slot);
  }
  return DG_OK;
}

/* train.cpp:150-157 */
int or_ray_cache_draw(or_ray_cache* c, uint64_t n, double* origin, double* dir, double* color,
                      uint32_t* image_id, uint64_t* pixel_id) {
  if (c->size == 0) return DG_EPROTO;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t e = or_mt64_next(&c->draw_rng) % c->size;
    for (int a = 0; a < 3; ++a) {
      if (origin) origin[3 * i + a] = c->origin[3 * e + a];
      if (dir) dir[3 * i + a] = c->dir[3 * e + a];
      if (color) color[3 * i + a] = c->color[3 * e + a];
    }
    if (image_id) image_id[i] = c->image_id[e];
    if (pixel_id) pixel_id[i] = c->pixel_id[e];
  }
  return DG_OK;
}

void or_ray_cache_snapshot(const or_ray_cache* c, double* origin, double* dir, double* color,
                           uint32_t* image_id, uint64_t* pixel_id) {
  memcpy(origin, c->origin, sizeof(double) * 3 * c->size);
  memcpy(dir, c->dir, sizeof(double) * 3 * c->size);
  memcpy(color, c->color, sizeof(double) * 3 * c->size);
  memcpy(image_id, c->image_id, sizeof(uint32_t) * c->size);
  memcpy(pixel_id, c->pixel_id, sizeof(uint64_t) * c->size);
}
