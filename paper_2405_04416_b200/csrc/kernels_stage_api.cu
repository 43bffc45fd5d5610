// kernels_stage_api.cu — per-function entry points behind the C++ facade (include/distgrid/):
// the reference's free functions whose inputs are explicit (not a context's partition state),
// batched, fp64 in the reference's evaluation order (no contraction: dadd/dmul/ddiv):
//   ray_aabb_intersect   geometry.cpp:7-28   one thread per ray, one box per call
//   march_segment        render.cpp:10-37    one thread per segment over caller intervals
//   occupancy_skip       grid.cpp:235-304    one thread per query over a caller bitfield
//   AdamState::step      train.cpp:91-115    fp64 moments over caller arrays
#include "geometry.cuh"
#include "kernels.h"

namespace dg {

namespace {

__global__ void k_ray_aabb(const double* __restrict__ o, const double* __restrict__ d, uint64_t n,
                           double lo0, double lo1, double lo2, double hi0, double hi1, double hi2,
                           uint8_t* __restrict__ hit, double* __restrict__ tn, double* __restrict__ tf) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]};
  const double dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
  const double lo[3] = {lo0, lo1, lo2}, hi[3] = {hi0, hi1, hi2};
  double a = 0.0, b = 0.0;
  const bool h = ray_aabb(oo, dd, lo, hi, a, b);
  hit[i] = h ? 1 : 0;
  tn[i] = h ? a : 0.0;
  tf[i] = h ? b : 0.0;
}

// Counts (t == nullptr) or samples at out_off[g] of segment g: the ladder over each of its
// occupied intervals in the caller's order (intervals are not merged, as in the reference).
__global__ void k_march_segment(const double* __restrict__ te, const double* __restrict__ tx,
                                const uint64_t* __restrict__ iv_off, const double* __restrict__ iv,
                                const uint64_t* __restrict__ ray_id, uint64_t n, double step, int jitter,
                                uint64_t seed, uint64_t batch, uint32_t* __restrict__ counts,
                                const uint64_t* __restrict__ out_off, double* __restrict__ t,
                                double* __restrict__ delta) {
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  const double t_enter = te[g], t_exit = tx[g];
  uint32_t cnt = 0;
  if (t_exit > t_enter) {
    const double offset = jitter ? dmul(step, counter_uniform(seed, ray_id ? ray_id[g] : 0, batch))
                                 : dmul(0.5, step);
    uint64_t at = t ? out_off[g] : 0;
    struct Emit {
      double* t;
      double* delta;
      uint64_t* at;
      uint32_t* cnt;
      __device__ void operator()(double tt, double dd) {
        if (t) {
          t[*at] = tt;
          delta[*at] = dd;
          ++*at;
        }
        ++*cnt;
      }
    } emit{t, delta, &at, &cnt};
    for (uint64_t k = iv_off[g]; k < iv_off[g + 1]; ++k)
      ladder(iv[2 * k], iv[2 * k + 1], t_enter, t_exit, offset, step, emit);
  }
  if (counts) counts[g] = cnt;
}

// occupancy_skip (grid.cpp:235-304) over a caller's row-major bitfield (ix fastest): counts
// (iv == nullptr) or the occupied runs of query q at out_off[q], as (t_near, t_far) pairs.
__global__ void k_occupancy_skip(const uint8_t* __restrict__ bits, uint32_t nx, uint32_t ny, uint32_t nz,
                                 double lo0, double lo1, double lo2, double hi0, double hi1, double hi2,
                                 const double* __restrict__ o, const double* __restrict__ d,
                                 const double* __restrict__ t0, const double* __restrict__ t1, uint64_t n,
                                 uint32_t* __restrict__ counts, const uint64_t* __restrict__ out_off,
                                 double* __restrict__ iv) {
  const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const double oo[3] = {o[3 * q], o[3 * q + 1], o[3 * q + 2]};
  const double dd[3] = {d[3 * q], d[3 * q + 1], d[3 * q + 2]};
  const double lo[3] = {lo0, lo1, lo2}, hi[3] = {hi0, hi1, hi2};
  const uint32_t sh[3] = {nx, ny, nz};
  const auto linear = [&](uint32_t ix, uint32_t iy, uint32_t iz) {
    return bits[ix + (uint64_t)nx * (iy + (uint64_t)ny * iz)] != 0;
  };
  uint32_t cnt = 0;
  uint64_t at = iv ? out_off[q] : 0;
  auto on_run = [&](double a, double b) {
    if (iv) {
      iv[2 * at] = a;
      iv[2 * at + 1] = b;
      ++at;
    }
    ++cnt;
  };
  occupancy_walk_fn(oo, dd, t0[q], t1[q], lo, hi, sh, linear, on_run);
  if (counts) counts[q] = cnt;
}

__global__ void k_adam_f64(double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m,
                           double* __restrict__ v, uint64_t n, double lr, double b1, double b2, double eps,
                           double bias1, double bias2) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double gi = g[i];
    const double mi = dadd(dmul(b1, m[i]), dmul(dsub(1.0, b1), gi));
    const double vi = dadd(dmul(b2, v[i]), dmul(dmul(dsub(1.0, b2), gi), gi));
    m[i] = mi;
    v[i] = vi;
    const double m_hat = ddiv(mi, bias1);
    const double v_hat = ddiv(vi, bias2);
    p[i] = dsub(p[i], ddiv(dmul(lr, m_hat), dadd(__dsqrt_rn(v_hat), eps)));
  }
}

// ---- query_density / query_color as separate stages (field.cpp:230-288) ------------------
// The training path fuses the two MLPs per tile; the reference API hands the 15 density
// features from one call to the next, so the facade gets them as two small FFMA kernels (one
// thread per sample, fp32, bias-first sequential dots as mlp.cpp:64-71).
__device__ __forceinline__ float clip15f(float v) { return v > 15.f ? 15.f : (v < -15.f ? -15.f : v); }
__device__ __forceinline__ float sigmoidf(float v) { return 1.f / (1.f + expf(-v)); }

__global__ void k_field_density(const FieldDesc* __restrict__ field, const float* __restrict__ params,
                                const float* __restrict__ X, uint64_t n, float* __restrict__ sigma,
                                float* __restrict__ feat) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const FieldDesc& fd = *field;
  const float* P = params + fd.base;
  const int enc = 2 * (int)fd.L;
  float x[2 * kMaxLevels];
  for (int l = 0; l < (int)fd.L; ++l) {
    const float2 v = reinterpret_cast<const float2*>(X)[(uint64_t)l * n + s];
    x[2 * l] = v.x;
    x[2 * l + 1] = v.y;
  }
  float h[64];
  for (int j = 0; j < 64; ++j) {
    float a = P[fd.db0 + j];
    for (int i = 0; i < enc; ++i) a += P[fd.dw0 + (uint64_t)j * enc + i] * x[i];
    h[j] = a > 0.f ? a : 0.f;
  }
  for (int k = 0; k < 16; ++k) {
    float a = P[fd.db1 + k];
    for (int j = 0; j < 64; ++j) a += P[fd.dw1 + (uint64_t)k * 64 + j] * h[j];
    a = clip15f(a);
    if (k == 0)
      sigma[s] = expf(a);
    else
      feat[s * 15 + (k - 1)] = a;
  }
}

__device__ void sh_basis16(float x, float y, float z, float* o) {  // sh.hpp:14-35, degree <= 3
  const float x2 = x * x, y2 = y * y, z2 = z * z;
  o[0] = 0.28209479177387814f;
  o[1] = -0.48860251190291987f * y;
  o[2] = 0.48860251190291987f * z;
  o[3] = -0.48860251190291987f * x;
  o[4] = 1.0925484305920792f * x * y;
  o[5] = -1.0925484305920792f * y * z;
  o[6] = 0.31539156525252005f * (3.0f * z2 - 1.0f);
  o[7] = -1.0925484305920792f * x * z;
  o[8] = 0.5462742152960396f * (x2 - y2);
  o[9] = -0.5900435899266435f * y * (3.0f * x2 - y2);
  o[10] = 2.890611442640554f * x * y * z;
  o[11] = -0.4570457994644658f * y * (5.0f * z2 - 1.0f);
  o[12] = 0.3731763325901154f * z * (5.0f * z2 - 3.0f);
  o[13] = -0.4570457994644658f * x * (5.0f * z2 - 1.0f);
  o[14] = 1.445305721320277f * z * (x2 - y2);
  o[15] = -0.5900435899266435f * x * (x2 - 3.0f * y2);
}

__global__ void k_field_color(const FieldDesc* __restrict__ field, const float* __restrict__ params,
                              const float* __restrict__ feat, const float* __restrict__ dirs,
                              const float* __restrict__ app, uint64_t n, float* __restrict__ rgb) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const FieldDesc& fd = *field;
  const float* P = params + fd.base;
  const int dim = (int)fd.app_dim, cin = 31 + dim;
  float in[48];
  for (int k = 0; k < 15; ++k) in[k] = feat[s * 15 + k];
  sh_basis16(dirs[3 * s], dirs[3 * s + 1], dirs[3 * s + 2], in + 15);
  for (int k = 0; k < dim; ++k) in[31 + k] = app[s * dim + k];
  float h1[64], h2[64];
  for (int j = 0; j < 64; ++j) {
    float a = P[fd.cb0 + j];
    for (int i = 0; i < cin; ++i) a += P[fd.cw0 + (uint64_t)j * cin + i] * in[i];
    h1[j] = fd.coarse ? sigmoidf(a) : (a > 0.f ? a : 0.f);
  }
  for (int j = 0; j < 64; ++j) {
    float a = P[fd.cb1 + j];
    for (int i = 0; i < 64; ++i) a += P[fd.cw1 + (uint64_t)j * 64 + i] * h1[i];
    h2[j] = fd.coarse ? sigmoidf(a) : (a > 0.f ? a : 0.f);
  }
  for (int c = 0; c < 3; ++c) {
    float a = P[fd.cb2 + c];
    for (int j = 0; j < 64; ++j) a += P[fd.cw2 + (uint64_t)c * 64 + j] * h2[j];
    rgb[3 * s + c] = sigmoidf(clip15f(a));
  }
}

inline unsigned nblk(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void launch_ray_aabb(const double* o, const double* d, uint64_t n, const double lo[3], const double hi[3],
                     uint8_t* hit, double* tn, double* tf, cudaStream_t s) {
  if (n)
    k_ray_aabb<<<nblk(n, 128), 128, 0, s>>>(o, d, n, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], hit, tn, tf);
}

void launch_march_segment(const double* te, const double* tx, const uint64_t* iv_off, const double* iv,
                          const uint64_t* ray_id, uint64_t n, double step, int jitter, uint64_t seed,
                          uint64_t batch, uint32_t* counts, const uint64_t* out_off, double* t, double* delta,
                          cudaStream_t s) {
  if (n)
    k_march_segment<<<nblk(n, 128), 128, 0, s>>>(te, tx, iv_off, iv, ray_id, n, step, jitter, seed, batch,
                                                  counts, out_off, t, delta);
}

void launch_field_density(const FieldDesc* field, const float* params, const float* X, uint64_t n, float* sigma,
                          float* feat, cudaStream_t s) {
  if (n) k_field_density<<<nblk(n, 64), 64, 0, s>>>(field, params, X, n, sigma, feat);
}

void launch_field_color(const FieldDesc* field, const float* params, const float* feat, const float* dirs,
                        const float* app, uint64_t n, float* rgb, cudaStream_t s) {
  if (n) k_field_color<<<nblk(n, 64), 64, 0, s>>>(field, params, feat, dirs, app, n, rgb);
}

void launch_occupancy_skip(const uint8_t* bits, const uint32_t shape[3], const double lo[3], const double hi[3],
                           const double* o, const double* d, const double* t0, const double* t1, uint64_t n,
                           uint32_t* counts, const uint64_t* out_off, double* iv, cudaStream_t s) {
  if (n)
    k_occupancy_skip<<<nblk(n, 128), 128, 0, s>>>(bits, shape[0], shape[1], shape[2], lo[0], lo[1], lo[2], hi[0],
                                                   hi[1], hi[2], o, d, t0, t1, n, counts, out_off, iv);
}

void launch_adam_f64(double* p, const double* g, double* m, double* v, uint64_t n, double lr, double b1,
                     double b2, double eps, double bias1, double bias2, cudaStream_t s) {
  if (n) {
    const uint64_t want = (n + 255) / 256;
    k_adam_f64<<<(unsigned)(want < 4096 ? want : 4096), 256, 0, s>>>(p, g, m, v, n, lr, b1, b2, eps, bias1, bias2);
  }
}

}  // namespace dg
