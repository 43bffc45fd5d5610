// kernels_render_api.cu — the compositing stage entry points of the C ABI:
// batched device overloads of local_render / accumulate_distortion_stats (render.cpp:46-99),
// merge_forward / merge_backward (render.cpp:101-143), local_render_backward
// (render.cpp:145-179) and the losses (train.cpp:8-75).  The training step itself runs the
// fused warp-per-item kernels in kernels_ray.cu; these serve callers that drive the stages one
// by one (the reference's per-function API), so they keep the reference's fp64 arithmetic and
// sweep order exactly: one thread per segment (or ray), inputs widened to fp64.
#include "kernels.h"

namespace dg {

namespace {

template <class R>
__global__ void k_local_render(const double* __restrict__ t, const double* __restrict__ delta,
                               const R* __restrict__ sigma, const R* __restrict__ rgb,
                               const uint64_t* __restrict__ seg_off, uint64_t n_seg,
                               const double* __restrict__ ray_t0, const double* __restrict__ ray_t1,
                               R* __restrict__ out_rgb, R* __restrict__ out_T,
                               R* __restrict__ out_depth, double* __restrict__ out_dist,
                               double* __restrict__ cache) {
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_seg) return;
  const uint64_t a = seg_off[g], b = seg_off[g + 1];
  double prefix = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, depth = 0.0;
  // accumulate_distortion_stats (render.cpp:80-99) when the ray span is given
  const bool dist = ray_t0 && ray_t1 && out_dist;
  const double span = dist ? dsub(ray_t1[g], ray_t0[g]) : 0.0;
  const bool dist_on = dist && span > 0.0;
  const double inv_span = dist_on ? ddiv(1.0, span) : 0.0;
  double w_sum = 0.0, m_sum = 0.0, pair = 0.0, interval = 0.0;
  for (uint64_t k = a; k < b; ++k) {
    const double alpha = dsub(1.0, exp(-dmul((double)sigma[k], delta[k])));
    if (cache) {
      cache[2 * k] = alpha;
      cache[2 * k + 1] = prefix;
    }
    const double w = dmul(prefix, alpha);
    c0 = dadd(c0, dmul((double)rgb[3 * k], w));
    c1 = dadd(c1, dmul((double)rgb[3 * k + 1], w));
    c2 = dadd(c2, dmul((double)rgb[3 * k + 2], w));
    depth = dadd(depth, dmul(w, t[k]));
    if (dist_on) {
      const double s = dmul(dsub(t[k], ray_t0[g]), inv_span);
      pair = dadd(pair, dmul(dmul(2.0, w), dsub(dmul(s, w_sum), m_sum)));
      interval = dadd(interval, dmul(dmul(dmul(w, w), delta[k]), inv_span));
      w_sum = dadd(w_sum, w);
      m_sum = dadd(m_sum, dmul(w, s));
    }
    prefix = dmul(prefix, dsub(1.0, alpha));
  }
  out_rgb[3 * g] = (R)c0;
  out_rgb[3 * g + 1] = (R)c1;
  out_rgb[3 * g + 2] = (R)c2;
  out_T[g] = (R)prefix;
  if (out_depth) out_depth[g] = (R)depth;
  if (dist) {
    out_dist[3 * g] = w_sum;
    out_dist[3 * g + 1] = m_sum;
    out_dist[3 * g + 2] = dadd(pair, ddiv(interval, 3.0));
  }
}

// local_render_backward: reverse sweep with tail_color / tail_trans (no division), on the
// (alpha, prefix) cache written by the forward sweep.
template <class R>
__global__ void k_local_render_bwd(const double* __restrict__ delta, const R* __restrict__ rgb,
                                   const uint64_t* __restrict__ seg_off, uint64_t n_seg,
                                   const double* __restrict__ cache, const R* __restrict__ d_rgb,
                                   const R* __restrict__ d_T, const R* __restrict__ w_up,
                                   R* __restrict__ sigma_grad, R* __restrict__ rgb_grad) {
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_seg) return;
  const uint64_t a = seg_off[g], b = seg_off[g + 1];
  const double u0 = d_rgb[3 * g], u1 = d_rgb[3 * g + 1], u2 = d_rgb[3 * g + 2], ut = d_T[g];
  double tail_color = 0.0, tail_trans = 1.0;
  for (uint64_t k = b; k-- > a;) {
    const double alpha = cache[2 * k], prefix = cache[2 * k + 1];
    double u = dadd(dadd(dmul(u0, (double)rgb[3 * k]), dmul(u1, (double)rgb[3 * k + 1])),
                    dmul(u2, (double)rgb[3 * k + 2]));
    if (w_up) u = dadd(u, (double)w_up[k]);
    const double alpha_grad = dsub(dmul(prefix, dsub(u, tail_color)), dmul(dmul(ut, prefix), tail_trans));
    sigma_grad[k] = (R)dmul(dmul(alpha_grad, delta[k]), dsub(1.0, alpha));
    const double pw = dmul(prefix, alpha);
    rgb_grad[3 * k] = (R)dmul(u0, pw);
    rgb_grad[3 * k + 1] = (R)dmul(u1, pw);
    rgb_grad[3 * k + 2] = (R)dmul(u2, pw);
    tail_color = dadd(dmul(alpha, u), dmul(dsub(1.0, alpha), tail_color));
    tail_trans = dmul(tail_trans, dsub(1.0, alpha));
  }
}

template <class R>
__global__ void k_merge_fwd(const R* __restrict__ srgb, const R* __restrict__ sT,
                            const R* __restrict__ sdepth, const uint64_t* __restrict__ ray_off,
                            uint64_t n_rays, R* __restrict__ rgb, R* __restrict__ T,
                            R* __restrict__ depth) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  double prefix = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, d = 0.0;
  for (uint64_t i = ray_off[r]; i < ray_off[r + 1]; ++i) {
    c0 = dadd(c0, dmul((double)srgb[3 * i], prefix));
    c1 = dadd(c1, dmul((double)srgb[3 * i + 1], prefix));
    c2 = dadd(c2, dmul((double)srgb[3 * i + 2], prefix));
    if (sdepth) d = dadd(d, dmul((double)sdepth[i], prefix));
    prefix = dmul(prefix, (double)sT[i]);
  }
  rgb[3 * r] = (R)c0;
  rgb[3 * r + 1] = (R)c1;
  rgb[3 * r + 2] = (R)c2;
  T[r] = (R)prefix;
  if (depth) depth[r] = (R)d;
}

// merge_backward: prefix / suffix products (no division by a possibly-zero T_i) and the
// occlusion term sum_{k>i} (prod_{i<j<k} T_j) dC . C_k, in the reference's loop order.
template <class R>
__global__ void k_merge_bwd(const R* __restrict__ srgb, const R* __restrict__ sT,
                            const uint64_t* __restrict__ ray_off, uint64_t n_rays,
                            const R* __restrict__ d_rgb, const R* __restrict__ d_T,
                            R* __restrict__ sd_rgb, R* __restrict__ sd_T) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  const uint64_t a = ray_off[r], n = ray_off[r + 1] - a;
  if (n > (uint64_t)kMaxSeg) return;  // validated on the host
  double pre[kMaxSeg + 1], suf[kMaxSeg + 1];
  pre[0] = 1.0;
  for (uint64_t i = 0; i < n; ++i) pre[i + 1] = dmul(pre[i], (double)sT[a + i]);
  suf[n] = 1.0;
  for (uint64_t i = n; i-- > 0;) suf[i] = dmul((double)sT[a + i], suf[i + 1]);
  const double u0 = d_rgb[3 * r], u1 = d_rgb[3 * r + 1], u2 = d_rgb[3 * r + 2], ut = d_T[r];
  for (uint64_t i = 0; i < n; ++i) {
    sd_rgb[3 * (a + i)] = (R)dmul(u0, pre[i]);
    sd_rgb[3 * (a + i) + 1] = (R)dmul(u1, pre[i]);
    sd_rgb[3 * (a + i) + 2] = (R)dmul(u2, pre[i]);
    const double t_grad = dmul(dmul(ut, pre[i]), suf[i + 1]);
    double running = 1.0, color_term = 0.0;
    for (uint64_t k = i + 1; k < n; ++k) {
      const double dc = dadd(dadd(dmul(u0, (double)srgb[3 * (a + k)]), dmul(u1, (double)srgb[3 * (a + k) + 1])),
                             dmul(u2, (double)srgb[3 * (a + k) + 2]));
      color_term = dadd(color_term, dmul(running, dc));
      running = dmul(running, (double)sT[a + k]);
    }
    sd_T[a + i] = (R)dadd(t_grad, dmul(pre[i], color_term));
  }
}

// loss_rgb / loss_rgb_grad and loss_transmittance(_single) / loss_transmittance_grad per ray.
template <class R>
__global__ void k_ray_losses(const R* __restrict__ rgb, const R* __restrict__ gt,
                             const R* __restrict__ T, uint64_t n, double eps,
                             double* __restrict__ l_rgb, double* __restrict__ l_T,
                             R* __restrict__ d_rgb, R* __restrict__ d_T) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double sq = 0.0;
  for (int a = 0; a < 3; ++a) {
    const double d = dsub((double)rgb[3 * r + a], (double)gt[3 * r + a]);
    sq = dadd(sq, dmul(d, d));
    if (d_rgb) d_rgb[3 * r + a] = (R)dmul(d, 2.0);
  }
  if (l_rgb) l_rgb[r] = sq;
  const double tc = smin((double)T[r], dsub(1.0, eps));
  if (l_T) l_T[r] = -log(dsub(1.0, tc));
  if (d_T) d_T[r] = (R)ddiv(1.0, dsub(1.0, tc));
}

// loss_distortion + loss_distortion_grad over each segment's (w, s, ds) (train.cpp:38-75).
__global__ void k_distortion(const double* __restrict__ w, const double* __restrict__ s,
                             const double* __restrict__ ds, const uint64_t* __restrict__ seg_off,
                             uint64_t n_seg, double* __restrict__ loss, double* __restrict__ grad) {
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_seg) return;
  const uint64_t a = seg_off[g], b = seg_off[g + 1];
  double wp = 0.0, mp = 0.0, pair = 0.0, interval = 0.0;
  for (uint64_t k = a; k < b; ++k) {
    pair = dadd(pair, dmul(dmul(2.0, w[k]), dsub(dmul(s[k], wp), mp)));
    interval = dadd(interval, dmul(dmul(w[k], w[k]), ds[k]));
    wp = dadd(wp, w[k]);
    mp = dadd(mp, dmul(w[k], s[k]));
  }
  if (loss) loss[g] = dadd(pair, ddiv(interval, 3.0));
  if (!grad) return;
  const double wt = wp, mt = mp;
  wp = 0.0;
  mp = 0.0;
  for (uint64_t k = a; k < b; ++k) {
    const double ws = dsub(dsub(wt, wp), w[k]);
    const double ms = dsub(dsub(mt, mp), dmul(w[k], s[k]));
    grad[k] = dadd(dadd(dmul(2.0, dsub(dmul(s[k], wp), mp)), dmul(2.0, dsub(ms, dmul(s[k], ws)))),
                   dmul(dmul(ddiv(2.0, 3.0), w[k]), ds[k]));
    wp = dadd(wp, w[k]);
    mp = dadd(mp, dmul(w[k], s[k]));
  }
}

// accumulate_distortion_stats (render.cpp:80-99) from a LocalRenderCache (alpha, prefix per
// sample): weight sum, weight moment and the local distortion over the ray span [t0, t1].
__global__ void k_distortion_stats(const double* __restrict__ t, const double* __restrict__ delta,
                                   const double* __restrict__ cache, const uint64_t* __restrict__ seg_off,
                                   uint64_t n_seg, const double* __restrict__ ray_t0,
                                   const double* __restrict__ ray_t1, double* __restrict__ out) {
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_seg) return;
  const double span = dsub(ray_t1[g], ray_t0[g]);
  if (!(span > 0.0)) return;  // the partial is left untouched
  const double inv_span = ddiv(1.0, span);
  double w_sum = 0.0, m_sum = 0.0, pair = 0.0, interval = 0.0;
  for (uint64_t k = seg_off[g]; k < seg_off[g + 1]; ++k) {
    const double w = dmul(cache[2 * k + 1], cache[2 * k]);
    const double s = dmul(dsub(t[k], ray_t0[g]), inv_span);
    pair = dadd(pair, dmul(dmul(2.0, w), dsub(dmul(s, w_sum), m_sum)));
    interval = dadd(interval, dmul(dmul(dmul(w, w), delta[k]), inv_span));
    w_sum = dadd(w_sum, w);
    m_sum = dadd(m_sum, dmul(w, s));
  }
  out[3 * g] = w_sum;
  out[3 * g + 1] = m_sum;
  out[3 * g + 2] = dadd(pair, ddiv(interval, 3.0));
}

inline unsigned nblk(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

template <class R>
void launch_local_render(const double* t, const double* delta, const R* sigma, const R* rgb,
                         const uint64_t* seg_off, uint64_t n_seg, const double* ray_t0,
                         const double* ray_t1, R* out_rgb, R* out_T, R* out_depth,
                         double* out_dist, double* cache, cudaStream_t s) {
  if (n_seg)
    k_local_render<R><<<nblk(n_seg, 128), 128, 0, s>>>(t, delta, sigma, rgb, seg_off, n_seg, ray_t0, ray_t1,
                                                        out_rgb, out_T, out_depth, out_dist, cache);
}
template <class R>
void launch_local_render_bwd(const double* delta, const R* rgb, const uint64_t* seg_off, uint64_t n_seg,
                             const double* cache, const R* d_rgb, const R* d_T, const R* w_up,
                             R* sigma_grad, R* rgb_grad, cudaStream_t s) {
  if (n_seg)
    k_local_render_bwd<R><<<nblk(n_seg, 128), 128, 0, s>>>(delta, rgb, seg_off, n_seg, cache, d_rgb, d_T, w_up,
                                                            sigma_grad, rgb_grad);
}
template <class R>
void launch_merge_fwd(const R* srgb, const R* sT, const R* sdepth, const uint64_t* ray_off,
                      uint64_t n_rays, R* rgb, R* T, R* depth, cudaStream_t s) {
  if (n_rays) k_merge_fwd<R><<<nblk(n_rays, 128), 128, 0, s>>>(srgb, sT, sdepth, ray_off, n_rays, rgb, T, depth);
}
template <class R>
void launch_merge_bwd(const R* srgb, const R* sT, const uint64_t* ray_off, uint64_t n_rays,
                      const R* d_rgb, const R* d_T, R* sd_rgb, R* sd_T, cudaStream_t s) {
  if (n_rays)
    k_merge_bwd<R><<<nblk(n_rays, 128), 128, 0, s>>>(srgb, sT, ray_off, n_rays, d_rgb, d_T, sd_rgb, sd_T);
}
template <class R>
void launch_ray_losses(const R* rgb, const R* gt, const R* T, uint64_t n, double eps,
                       double* l_rgb, double* l_T, R* d_rgb, R* d_T, cudaStream_t s) {
  if (n) k_ray_losses<R><<<nblk(n, 128), 128, 0, s>>>(rgb, gt, T, n, eps, l_rgb, l_T, d_rgb, d_T);
}
#define DG_RENDER_API_INST(R)                                                                              \
  template void launch_local_render<R>(const double*, const double*, const R*, const R*, const uint64_t*,   \
                                       uint64_t, const double*, const double*, R*, R*, R*, double*, double*, \
                                       cudaStream_t);                                                        \
  template void launch_local_render_bwd<R>(const double*, const R*, const uint64_t*, uint64_t, const double*, \
                                           const R*, const R*, const R*, R*, R*, cudaStream_t);              \
  template void launch_merge_fwd<R>(const R*, const R*, const R*, const uint64_t*, uint64_t, R*, R*, R*,     \
                                    cudaStream_t);                                                           \
  template void launch_merge_bwd<R>(const R*, const R*, const uint64_t*, uint64_t, const R*, const R*, R*, R*, \
                                    cudaStream_t);                                                           \
  template void launch_ray_losses<R>(const R*, const R*, const R*, uint64_t, double, double*, double*, R*, R*, \
                                     cudaStream_t);
DG_RENDER_API_INST(float)
DG_RENDER_API_INST(double)
#undef DG_RENDER_API_INST
void launch_distortion_stats(const double* t, const double* delta, const double* cache, const uint64_t* seg_off,
                             uint64_t n_seg, const double* ray_t0, const double* ray_t1, double* out,
                             cudaStream_t s) {
  if (n_seg) k_distortion_stats<<<nblk(n_seg, 128), 128, 0, s>>>(t, delta, cache, seg_off, n_seg, ray_t0, ray_t1, out);
}
void launch_distortion(const double* w, const double* s_, const double* ds, const uint64_t* seg_off,
                       uint64_t n_seg, double* loss, double* grad, cudaStream_t s) {
  if (n_seg) k_distortion<<<nblk(n_seg, 128), 128, 0, s>>>(w, s_, ds, seg_off, n_seg, loss, grad);
}

}  // namespace dg
