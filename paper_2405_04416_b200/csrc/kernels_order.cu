// kernels_order.cu — spatial sample order for the encode passes (SURVEY §8 north_star:
// "coalesced by sorting samples per level and block").
//
// The march emits each field's samples ray by ray in t order.  They are cut into chunks of C
// consecutive samples (a short stretch of one ray, C x step long); each chunk's key is the
// Morton code of its middle sample's normalised position quantised to 2^bits cells per axis,
// and the chunks are radix-sorted by key within their field (the field's last partial chunk
// stays at its end).  Consecutive threads of an encode pass then touch neighbouring lattice
// cells, so their corner rows hit L1 / L2 instead of HBM.  Sorting chunks instead of samples
// keeps the sort C times smaller and makes every gather / scatter through the permutation a
// run of C consecutive samples (C = 8: one 64-byte DRAM granule of an fp64 array).
#include <cub/device/device_radix_sort.cuh>

#include "kernels.h"

namespace dg {

namespace {

__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 10 bits -> every third bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// key of chunk q of a field: the Morton code of its middle sample's position
__global__ void k_order_keys(const double* __restrict__ p, uint64_t stride, uint64_t off, uint32_t chunks,
                             uint32_t C, uint32_t bits, uint32_t* __restrict__ key, uint32_t* __restrict__ id) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= chunks) return;
  const uint64_t s = off + (uint64_t)q * C + C / 2;
  const double scale = double(1u << bits);
  uint32_t c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double v = p[a * stride + s] * scale;
    c[a] = v <= 0.0 ? 0u : (v >= scale ? (1u << bits) - 1u : (uint32_t)v);
  }
  key[q] = spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2);
  id[q] = q;
}

// Sorted slot j of a field (j < n) -> its march sample s = off + chunk[j / C] * C + j % C (the
// tail past the full chunks keeps its place); perm[off + j] = s, the positions and item ids
// gathered into slot order, inv[s] = off + j.
__global__ void k_order_gather(const double* __restrict__ p, const uint32_t* __restrict__ item, uint64_t stride,
                               uint64_t off, uint32_t n, uint32_t C, uint32_t chunks,
                               const uint32_t* __restrict__ chunk, uint32_t* __restrict__ perm,
                               double* __restrict__ p_out, uint32_t* __restrict__ item_out,
                               uint32_t* __restrict__ inv) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t q = j / C;
  const uint64_t s = off + (q < chunks ? (uint64_t)__ldg(chunk + q) * C + (j - q * C) : (uint64_t)j);
  const uint64_t t = off + j;
  const double x = p[s], y = p[stride + s], z = p[2 * stride + s];
  const uint32_t it = item[s];
  __stcs(p_out + t, x);
  __stcs(p_out + stride + t, y);
  __stcs(p_out + 2 * stride + t, z);
  __stcs(item_out + t, it);
  __stcs(perm + t, (uint32_t)s);
  inv[s] = (uint32_t)t;
}

}  // namespace

size_t order_sort_tmp_bytes(uint32_t n) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, n, 0, 30);
  return tmp;
}

// Orders the samples [off, off + n) of one field (see the file comment).  scratch: 4 * ceil(n / C)
// u32 (keys in / out, ids in / out); tmp: order_sort_tmp_bytes(n).  Returns the launch count or
// -1 when the sort fails.
int launch_order_field(const double* p, const uint32_t* item, uint64_t stride, uint64_t off, uint32_t n,
                       uint32_t C, uint32_t bits, uint32_t* perm, uint32_t* inv, double* p_out,
                       uint32_t* item_out, uint32_t* scratch, void* tmp, size_t tmp_bytes, cudaStream_t s) {
  if (!n) return 0;
  const uint32_t chunks = n / C;
  uint32_t* k_in = scratch;
  uint32_t* k_out = scratch + chunks;
  uint32_t* i_in = scratch + 2 * (size_t)chunks;
  uint32_t* i_out = scratch + 3 * (size_t)chunks;
  int launches = 1;
  if (chunks) {
    k_order_keys<<<(chunks + 255) / 256, 256, 0, s>>>(p, stride, off, chunks, C, bits, k_in, i_in);
    size_t t = tmp_bytes;
    if (cub::DeviceRadixSort::SortPairs(tmp, t, k_in, k_out, i_in, i_out, chunks, 0, 3 * bits, s) != cudaSuccess)
      return -1;
    launches += 2;
  }
  k_order_gather<<<(n + 255) / 256, 256, 0, s>>>(p, item, stride, off, n, C, chunks, i_out, perm, p_out,
                                                 item_out, inv);
  return launches;
}

}  // namespace dg
