// kernels_occ.cu — occupancy-grid update.
//
//   OccupancyGrid::decay_and_update (grid.cpp:201-229) + Worker::update_occupancy
//   (worker.cpp:549-562):  density[i] <- max(density[i] * decay, sigma(jittered point of i))
//   for the sampled cells, then bitfield = density >= threshold.  The jittered points come
//   from the reference's own mt19937_64 stream (generated on the host, in the reference's
//   draw order) so the sampled set is identical; sigma = query_density(p).sigma is evaluated
//   here: fp64 bit-exact lattice indices, fp32 gathers, density MLP [enc -> 64 ReLU -> raw0].
#include "encode_common.cuh"
#include "geometry.cuh"
#include "kernels.h"

namespace dg {

namespace {

// sigma = query_density(p).sigma at the jittered points: the training encode's corners and
// paired-row gathers (same rows, weights and accumulation order), then the density MLP
// [enc -> 64 ReLU -> raw0] with the weights broadcast from shared memory.  One thread per
// cell; a level-pass split (encode kernel + MLP kernel) measured slower.
__global__ void __launch_bounds__(128) k_occ_query(const FieldDesc* __restrict__ field,
                                                   const float* __restrict__ params,
                                                   const double* __restrict__ pw, uint64_t n,
                                                   float* __restrict__ sigma) {
  __shared__ __align__(16) float w0[kHidden * kEnc];  // [o][i]
  __shared__ float b0[kHidden];
  __shared__ float w1[kHidden];         // row 0 of the second layer
  __shared__ float b1;
  const FieldDesc& fd = *field;
  const float* base = params + fd.base;
  const int enc = (int)fd.L * 2;
  for (int e = threadIdx.x; e < kHidden * kEnc; e += blockDim.x) {
    const int o = e / kEnc, i = e % kEnc;
    w0[e] = i < enc ? base[fd.dw0 + o * enc + i] : 0.f;
  }
  for (int e = threadIdx.x; e < kHidden; e += blockDim.x) {
    b0[e] = base[fd.db0 + e];
    w1[e] = base[fd.dw1 + e];
  }
  if (threadIdx.x == 0) b1 = base[fd.db1];
  __syncthreads();
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  // worker.cpp:215: p = clamp(box.to_unit(world point), 0, 1)
  double p[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
    p[a] = sclamp(ddiv(dsub(pw[3 * s + a], fd.box_lo[a]), dsub(fd.box_hi[a], fd.box_lo[a])), 0.0, 1.0);
  float x[kEnc];
#pragma unroll
  for (int i = 0; i < kEnc; ++i) x[i] = 0.f;
  for (uint32_t l = 0; l < fd.L; ++l) {
    Corners c;
    level_corners(fd.lv[l], p, c);
    const float2 v = gather_level_pairs(reinterpret_cast<const float2*>(base + fd.lv[l].offset), c);
    x[2 * l] = v.x;
    x[2 * l + 1] = v.y;
  }
  float raw = b1;
  const float4* w04 = reinterpret_cast<const float4*>(w0);
  for (int o = 0; o < kHidden; ++o) {
    float h = b0[o];
#pragma unroll
    for (int q = 0; q < kEnc / 4; ++q) {  // broadcast 16-byte shared loads
      const float4 w = w04[o * (kEnc / 4) + q];
      h = fmaf(w.x, x[4 * q], h);
      h = fmaf(w.y, x[4 * q + 1], h);
      h = fmaf(w.z, x[4 * q + 2], h);
      h = fmaf(w.w, x[4 * q + 3], h);
    }
    raw = fmaf(w1[o], h > 0.f ? h : 0.f, raw);
  }
  raw = raw > 15.f ? 15.f : (raw < -15.f ? -15.f : raw);
  sigma[s] = expf(raw);
}

// Warm-up sweep: every cell exactly once, so the update is a pure element-wise max.
__global__ void k_occ_apply(float* __restrict__ density, const uint32_t* __restrict__ cells,
                            const float* __restrict__ sigma, uint64_t n, float decay) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint64_t c = cells ? cells[s] : s;
  density[c] = fmaxf(density[c] * decay, sigma[s]);
}

// recompute_bitfield: density (linear, x fastest) >= threshold, into the bricked bitfield.
__global__ void k_occ_bits(const float* __restrict__ density, uint8_t* __restrict__ bits, uint32_t nx,
                           uint32_t ny, uint32_t nz, float threshold) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t n = (uint64_t)nx * ny * nz;
  if (s >= n) return;
  const uint32_t x = (uint32_t)(s % nx), y = (uint32_t)((s / nx) % ny), z = (uint32_t)(s / ((uint64_t)nx * ny));
  const uint32_t nb[3] = {(nx + kOccBX - 1) / kOccBX, (ny + kOccBY - 1) / kOccBY, (nz + kOccBZ - 1) / kOccBZ};
  bits[occ_addr(nb, x, y, z)] = density[s] >= threshold ? 1 : 0;
}

inline unsigned nb(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

int launch_occ_query(const FieldDesc* field, const float* params, const double* pw, uint64_t n,
                     float* sigma, cudaStream_t s) {
  if (!n) return 0;
  k_occ_query<<<nb(n, 128), 128, 0, s>>>(field, params, pw, n, sigma);
  return 1;
}
void launch_occ_apply(float* density, const uint32_t* cells, const float* sigma, uint64_t n,
                      float decay, cudaStream_t s) {
  if (n) k_occ_apply<<<nb(n, 256), 256, 0, s>>>(density, cells, sigma, n, decay);
}
void launch_occ_bits(const float* density, uint8_t* bits, const uint32_t shape[3], float threshold,
                     cudaStream_t s) {
  const uint64_t n = (uint64_t)shape[0] * shape[1] * shape[2];
  if (n) k_occ_bits<<<nb(n, 256), 256, 0, s>>>(density, bits, shape[0], shape[1], shape[2], threshold);
}

}  // namespace dg
