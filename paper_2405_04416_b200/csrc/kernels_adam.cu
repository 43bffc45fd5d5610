// kernels_adam.cu — stage 6: dense Adam over every local parameter, fused with the
// gradient zeroing (AdamState::step train.cpp:91-115 + FieldGrads::zero field.cpp:210-220,
// as Worker::apply_updates does them back to back, worker.cpp:524-547).
//
// HBM-bound: 16 B read (p, g, m, v) + 16 B written (p, m, v, g = 0) per parameter.
#include "kernels.h"

namespace dg {

namespace {

__device__ __forceinline__ void adam1(float& p, float& g, float& m, float& v, float lr, float b1,
                                      float b2, float eps, float inv_bias1, float inv_bias2) {
  m = b1 * m + (1.f - b1) * g;
  v = b2 * v + (1.f - b2) * g * g;
  const float m_hat = m * inv_bias1;
  const float v_hat = v * inv_bias2;
  p -= lr * m_hat / (sqrtf(v_hat) + eps);
  g = 0.f;
}

__global__ void __launch_bounds__(256) k_adam(float4* __restrict__ p, float4* __restrict__ g,
                                              float4* __restrict__ m, float4* __restrict__ v,
                                              uint64_t n4, float lr, float b1, float b2, float eps,
                                              float inv_bias1, float inv_bias2,
                                              const uint32_t* __restrict__ abort_flag, uint32_t abort_mask) {
  // An aborted step (e.g. a missing partial, worker.cpp:371-376) must leave p, m, v untouched,
  // as the reference throws before apply_updates; its gradients are discarded.
  if (abort_flag && (*abort_flag & abort_mask)) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (uint64_t)gridDim.x * blockDim.x)
      g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    float4 pp = p[i], gg = g[i], mm = m[i], vv = v[i];
    adam1(pp.x, gg.x, mm.x, vv.x, lr, b1, b2, eps, inv_bias1, inv_bias2);
    adam1(pp.y, gg.y, mm.y, vv.y, lr, b1, b2, eps, inv_bias1, inv_bias2);
    adam1(pp.z, gg.z, mm.z, vv.z, lr, b1, b2, eps, inv_bias1, inv_bias2);
    adam1(pp.w, gg.w, mm.w, vv.w, lr, b1, b2, eps, inv_bias1, inv_bias2);
    p[i] = pp;
    g[i] = gg;
    m[i] = mm;
    v[i] = vv;
  }
}

__global__ void k_adam_tail(float* p, float* g, float* m, float* v, uint64_t start, uint64_t n,
                            float lr, float b1, float b2, float eps, float inv_bias1,
                            float inv_bias2, const uint32_t* abort_flag, uint32_t abort_mask) {
  const uint64_t i = start + threadIdx.x;
  if (i >= n) return;
  if (abort_flag && (*abort_flag & abort_mask))
    g[i] = 0.f;
  else
    adam1(p[i], g[i], m[i], v[i], lr, b1, b2, eps, inv_bias1, inv_bias2);
}

__global__ void k_fill_uniform(float* __restrict__ p, uint64_t n, float lo, float hi, uint64_t seed) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = counter_hash(seed, i, 0x5eed, 0);
    const float u = (float)((double)(h >> 11) * 0x1.0p-53);
    p[i] = lo + (hi - lo) * u;
  }
}

}  // namespace

// spread: one float4 per thread (many short CTAs) instead of a resident grid-stride grid, so
// that kernels of a higher-priority stream (the next training step's front half) get SMs as
// CTAs retire while this update runs on its side stream.
void launch_adam(float* p, float* g, float* m, float* v, uint64_t n, float lr, float b1, float b2,
                 float eps, float inv_bias1, float inv_bias2, cudaStream_t s, const uint32_t* abort_flag,
                 uint32_t abort_mask, bool spread) {
  const uint64_t n4 = n / 4;
  if (n4) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (n4 + 255) / 256;
    const unsigned grid = (unsigned)(spread || want < (uint64_t)sms * 8 ? want : (uint64_t)sms * 8);
    k_adam<<<grid, 256, 0, s>>>(reinterpret_cast<float4*>(p), reinterpret_cast<float4*>(g),
                                reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), n4, lr,
                                b1, b2, eps, inv_bias1, inv_bias2, abort_flag, abort_mask);
  }
  if (n % 4)
    k_adam_tail<<<1, 4, 0, s>>>(p, g, m, v, n4 * 4, n, lr, b1, b2, eps, inv_bias1, inv_bias2, abort_flag,
                                abort_mask);
}

void launch_fill_uniform(float* p, uint64_t n, float lo, float hi, uint64_t seed, cudaStream_t s) {
  if (!n) return;
  k_fill_uniform<<<1184, 256, 0, s>>>(p, n, lo, hi, seed);
}

}  // namespace dg
