// ray_cache.cu — §8f row 2: the ray cache / pixel-ray batch feed on the GPU.
//
//   RayCache (train.cpp:117-159) + make_pixel_ray (dataset.cpp:312-324) +
//   CameraPose::pixel_ray_dir (partition.cpp:30-33).
//
// The images (u8 RGB) and camera poses live on the device; the cache entries are a
// device-resident ring of SupervisedRays (SoA).  The reference's two mt19937_64 streams
// (refresh: image, x, y per ray; draw: one index per ray) are sequential by definition and
// stay on the host — 3 + 1 engine calls per ray — so the sampled pixels and drawn entries are
// the reference's exactly; the GPU builds the rays (fp64, bit-exact direction) and gathers
// drawn batches straight into the device RayBatch that dg_train_step consumes (no host copy
// of ray data on the training path).
#include <cstdio>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "geometry.cuh"

namespace dg {
int set_error(int code, const char* msg);

namespace {

struct DevPose {  // CameraPose (partition.hpp:15-28) + its image
  double R[9];
  double t[3];
  double fx, fy, cx, cy;
  uint32_t image_id, width, height, pad;
  uint64_t pixel_off;  // byte offset of the image's RGB in the pixel buffer
};

// dataset.cpp:312-324 + partition.cpp:30-33, fp64 without contraction (bit-exact).
__global__ void k_make_pixel_rays(const DevPose* __restrict__ poses, const uint8_t* __restrict__ pixels,
                                  const uint32_t* __restrict__ req, uint64_t n, double* __restrict__ origin,
                                  double* __restrict__ dir, float* __restrict__ gt,
                                  uint32_t* __restrict__ image, uint64_t* __restrict__ pixel_id) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t img = req[4 * i], x = req[4 * i + 1], y = req[4 * i + 2], slot = req[4 * i + 3];
  const DevPose& p = poses[img];
  double dd[3];
  pixel_ray_dir(p.R, p.fx, p.fy, p.cx, p.cy, dadd((double)x, 0.5), dadd((double)y, 0.5), dd);  // dataset.cpp:317
  const uint8_t* px = pixels + p.pixel_off + ((uint64_t)y * p.width + x) * 3;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    origin[3 * (uint64_t)slot + a] = p.t[a];
    dir[3 * (uint64_t)slot + a] = dd[a];
    gt[3 * (uint64_t)slot + a] = (float)ddiv((double)px[a], 255.0);  // Image::pixel_channel
  }
  image[slot] = p.image_id;
  pixel_id[slot] = ((uint64_t)p.image_id << 32) | ((uint64_t)y * p.width + x);
}

// draw_batch: batch[i] = entries[idx[i]]
__global__ void k_gather_rays(const uint32_t* __restrict__ idx, uint64_t n, const double* __restrict__ o,
                              const double* __restrict__ d, const float* __restrict__ gt,
                              const uint32_t* __restrict__ img, const uint64_t* __restrict__ pix,
                              double* __restrict__ bo, double* __restrict__ bd, float* __restrict__ bgt,
                              uint32_t* __restrict__ bimg, uint64_t* __restrict__ bpix) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t e = idx[i];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    bo[3 * i + a] = o[3 * e + a];
    bd[3 * i + a] = d[3 * e + a];
    bgt[3 * i + a] = gt[3 * e + a];
  }
  bimg[i] = img[e];
  bpix[i] = pix[e];
}

uint64_t splitmix(uint64_t x) {  // rng.hpp:8-15
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  ~Buf() {
    if (p) cudaFree(p);
  }
  bool ensure(size_t want) {
    if (want <= bytes) return true;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (cudaMalloc(&p, want ? want : 16) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    bytes = want ? want : 16;
    return true;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace
}  // namespace dg

using dg::set_error;

struct dg_ray_cache {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t capacity = 0, size = 0, cursor = 0;
  std::mt19937_64 refresh_rng, draw_rng;  // train.cpp:117-121
  std::vector<uint32_t> train_indices;
  std::vector<uint32_t> width, height;
  dg::Buf poses, pixels;
  dg::Buf e_origin, e_dir, e_gt, e_img, e_pix;  // entries (capacity)
  dg::Buf req, idx;                             // staging
  dg::Buf b_origin, b_dir, b_gt, b_img, b_pix;  // drawn batch
  std::vector<uint32_t> h_req, h_idx;
  uint64_t batch_cap = 0;
};

#define RC_CU(call)                                                                  \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      std::string m_ = std::string(#call) + " failed: " + cudaGetErrorString(e_);    \
      return set_error(DG_ECUDA, m_.c_str());                                        \
    }                                                                                \
  } while (0)

extern "C" {

int dg_ray_cache_create(int device, const dg_camera* cams, const uint8_t* const* images, uint32_t n_images,
                        uint64_t capacity, uint64_t seed, dg_ray_cache** out) {
  if (!out || !cams || !images || n_images == 0) return set_error(DG_EINVAL, "ray cache: no images");
  if (capacity == 0) return set_error(DG_EINVAL, "ray cache: capacity must be positive");
  if (capacity >= (1ull << 32)) return set_error(DG_EINVAL, "ray cache: capacity must be < 2^32");
  auto* c = new dg_ray_cache();
  std::unique_ptr<dg_ray_cache> guard(c);
  if (device < 0) RC_CU(cudaGetDevice(&device));
  c->device = device;
  RC_CU(cudaSetDevice(device));
  RC_CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->capacity = capacity;
  c->refresh_rng.seed(dg::splitmix(dg::splitmix(seed ^ 0x5261794361636865ull)));  // Rng(x) seeds with splitmix64(x)
  c->draw_rng.seed(dg::splitmix(dg::splitmix(seed ^ 0x4261746368447277ull)));
  std::vector<dg::DevPose> hp(n_images);
  uint64_t off = 0;
  for (uint32_t i = 0; i < n_images; ++i) {
    const dg_camera& k = cams[i];
    if (k.width == 0 || k.height == 0 || !images[i]) return set_error(DG_EINVAL, "ray cache: empty image");
    dg::DevPose& p = hp[i];
    for (int j = 0; j < 9; ++j) p.R[j] = k.rotation[j];
    for (int j = 0; j < 3; ++j) p.t[j] = k.translation[j];
    p.fx = k.fx;
    p.fy = k.fy;
    p.cx = k.cx;
    p.cy = k.cy;
    p.image_id = k.image_id;
    p.width = k.width;
    p.height = k.height;
    p.pad = 0;
    p.pixel_off = off;
    off += uint64_t(k.width) * k.height * 3;
    c->width.push_back(k.width);
    c->height.push_back(k.height);
    if (k.is_train) c->train_indices.push_back(i);
  }
  if (!c->poses.ensure(hp.size() * sizeof(dg::DevPose)) || !c->pixels.ensure(off) ||
      !c->e_origin.ensure(capacity * 24) || !c->e_dir.ensure(capacity * 24) || !c->e_gt.ensure(capacity * 12) ||
      !c->e_img.ensure(capacity * 4) || !c->e_pix.ensure(capacity * 8))
    return set_error(DG_ENOMEM, "ray cache: device allocation failed");
  RC_CU(cudaMemcpyAsync(c->poses.p, hp.data(), hp.size() * sizeof(dg::DevPose), cudaMemcpyHostToDevice, c->stream));
  for (uint32_t i = 0; i < n_images; ++i)
    RC_CU(cudaMemcpyAsync(c->pixels.as<uint8_t>() + hp[i].pixel_off, images[i],
                          uint64_t(hp[i].width) * hp[i].height * 3, cudaMemcpyHostToDevice, c->stream));
  RC_CU(cudaStreamSynchronize(c->stream));
  *out = guard.release();
  return DG_OK;
}

void dg_ray_cache_destroy(dg_ray_cache* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaStream_t s = c->stream;
  delete c;
  if (s) cudaStreamDestroy(s);
}

int dg_ray_cache_size(const dg_ray_cache* c, uint64_t* size, uint64_t* capacity) {
  if (!c) return set_error(DG_EINVAL, "ray cache: null");
  if (size) *size = c->size;
  if (capacity) *capacity = c->capacity;
  return DG_OK;
}

// RayCache::refresh (train.cpp:123-143): `count` rays sampled uniformly over (train image,
// pixel); appended until full, then overwriting the oldest entries in ring order.
int dg_ray_cache_refresh(dg_ray_cache* c, uint64_t count) {
  if (!c) return set_error(DG_EINVAL, "ray cache: null");
  if (c->train_indices.empty()) return set_error(DG_EINVAL, "ray cache: dataset has no train images");
  RC_CU(cudaSetDevice(c->device));
  // host: the reference's draw sequence and slot assignment; only each slot's last write
  // survives (a refresh larger than the capacity wraps the ring)
  std::vector<int64_t> last(c->capacity, -1);
  c->h_req.resize(4 * count);
  for (uint64_t i = 0; i < count; ++i) {
    const uint32_t img = c->train_indices[c->refresh_rng() % c->train_indices.size()];
    const uint32_t x = uint32_t(c->refresh_rng() % c->width[img]);
    const uint32_t y = uint32_t(c->refresh_rng() % c->height[img]);
    uint64_t slot;
    if (c->size < c->capacity) {
      slot = c->size++;
    } else {
      slot = c->cursor;
      c->cursor = (c->cursor + 1) % c->capacity;
    }
    c->h_req[4 * i] = img;
    c->h_req[4 * i + 1] = x;
    c->h_req[4 * i + 2] = y;
    c->h_req[4 * i + 3] = uint32_t(slot);
    last[slot] = int64_t(i);
  }
  uint64_t m = 0;  // compact to the surviving writes
  for (uint64_t i = 0; i < count; ++i)
    if (last[c->h_req[4 * i + 3]] == int64_t(i)) {
      for (int k = 0; k < 4; ++k) c->h_req[4 * m + k] = c->h_req[4 * i + k];
      ++m;
    }
  if (m == 0) return DG_OK;
  if (!c->req.ensure(m * 16)) return set_error(DG_ENOMEM, "ray cache: staging allocation failed");
  RC_CU(cudaMemcpyAsync(c->req.p, c->h_req.data(), m * 16, cudaMemcpyHostToDevice, c->stream));
  dg::k_make_pixel_rays<<<unsigned((m + 127) / 128), 128, 0, c->stream>>>(
      c->poses.as<dg::DevPose>(), c->pixels.as<uint8_t>(), c->req.as<uint32_t>(), m, c->e_origin.as<double>(),
      c->e_dir.as<double>(), c->e_gt.as<float>(), c->e_img.as<uint32_t>(), c->e_pix.as<uint64_t>());
  RC_CU(cudaGetLastError());
  RC_CU(cudaStreamSynchronize(c->stream));  // h_req is reused
  return DG_OK;
}

// RayCache::draw_batch (train.cpp:150-157): uniform draw with replacement into a device
// RayBatch owned by the cache (valid until the next draw); first_ray_id = 0 as the batch
// index is the ray id (worker.cpp:153).
int dg_ray_cache_draw(dg_ray_cache* c, uint64_t n, dg_ray_batch* out) {
  if (!c || !out) return set_error(DG_EINVAL, "ray cache: null");
  if (c->size == 0) return set_error(DG_EPROTO, "ray cache: empty");
  RC_CU(cudaSetDevice(c->device));
  c->h_idx.resize(n);
  for (uint64_t i = 0; i < n; ++i) c->h_idx[i] = uint32_t(c->draw_rng() % c->size);
  if (n > c->batch_cap) {
    if (!c->b_origin.ensure(n * 24) || !c->b_dir.ensure(n * 24) || !c->b_gt.ensure(n * 12) ||
        !c->b_img.ensure(n * 4) || !c->b_pix.ensure(n * 8) || !c->idx.ensure(n * 4))
      return set_error(DG_ENOMEM, "ray cache: batch allocation failed");
    c->batch_cap = n;
  }
  if (n) {
    RC_CU(cudaMemcpyAsync(c->idx.p, c->h_idx.data(), n * 4, cudaMemcpyHostToDevice, c->stream));
    dg::k_gather_rays<<<unsigned((n + 255) / 256), 256, 0, c->stream>>>(
        c->idx.as<uint32_t>(), n, c->e_origin.as<double>(), c->e_dir.as<double>(), c->e_gt.as<float>(),
        c->e_img.as<uint32_t>(), c->e_pix.as<uint64_t>(), c->b_origin.as<double>(), c->b_dir.as<double>(),
        c->b_gt.as<float>(), c->b_img.as<uint32_t>(), c->b_pix.as<uint64_t>());
    RC_CU(cudaGetLastError());
  }
  RC_CU(cudaStreamSynchronize(c->stream));
  out->origin = c->b_origin.as<double>();
  out->dir = c->b_dir.as<double>();
  out->color_gt = c->b_gt.as<float>();
  out->image_id = c->b_img.as<uint32_t>();
  out->n = n;
  out->first_ray_id = 0;
  out->mem = DG_MEM_DEVICE;
  out->reserved = 0;
  return DG_OK;
}

// RayCache::draw_batch (train.cpp:150-158) into host arrays (the facade's RayCache).
int dg_ray_cache_draw_host(dg_ray_cache* c, uint64_t n, double* origin, double* dir, float* color_gt,
                           uint32_t* image_id, uint64_t* pixel_id) {
  dg_ray_batch b;
  const int rc = dg_ray_cache_draw(c, n, &b);
  if (rc != DG_OK || n == 0) return rc;
  if (origin) RC_CU(cudaMemcpyAsync(origin, c->b_origin.p, n * 24, cudaMemcpyDeviceToHost, c->stream));
  if (dir) RC_CU(cudaMemcpyAsync(dir, c->b_dir.p, n * 24, cudaMemcpyDeviceToHost, c->stream));
  if (color_gt) RC_CU(cudaMemcpyAsync(color_gt, c->b_gt.p, n * 12, cudaMemcpyDeviceToHost, c->stream));
  if (image_id) RC_CU(cudaMemcpyAsync(image_id, c->b_img.p, n * 4, cudaMemcpyDeviceToHost, c->stream));
  if (pixel_id) RC_CU(cudaMemcpyAsync(pixel_id, c->b_pix.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
  RC_CU(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

// RayCache::snapshot (train.cpp:145-148): host copy of the entries in storage order.
int dg_ray_cache_snapshot(dg_ray_cache* c, double* origin, double* dir, float* color_gt, uint32_t* image_id,
                          uint64_t* pixel_id) {
  if (!c) return set_error(DG_EINVAL, "ray cache: null");
  RC_CU(cudaSetDevice(c->device));
  const uint64_t n = c->size;
  if (origin) RC_CU(cudaMemcpyAsync(origin, c->e_origin.p, n * 24, cudaMemcpyDeviceToHost, c->stream));
  if (dir) RC_CU(cudaMemcpyAsync(dir, c->e_dir.p, n * 24, cudaMemcpyDeviceToHost, c->stream));
  if (color_gt) RC_CU(cudaMemcpyAsync(color_gt, c->e_gt.p, n * 12, cudaMemcpyDeviceToHost, c->stream));
  if (image_id) RC_CU(cudaMemcpyAsync(image_id, c->e_img.p, n * 4, cudaMemcpyDeviceToHost, c->stream));
  if (pixel_id) RC_CU(cudaMemcpyAsync(pixel_id, c->e_pix.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
  RC_CU(cudaStreamSynchronize(c->stream));
  return DG_OK;
}

}  // extern "C"
