// dg_common.cuh — shared device types and the bit-exact fp64 helpers.
//
// Stages 1-3 (segmentation, march, lattice indices) must match the reference CPU
// oracle bit for bit.  The reference is built without FMA
// contraction, so every fp64 operation on those paths goes through the _rn intrinsics,
// which nvcc never fuses, and std::max/min/clamp tie semantics are spelled out.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "distgrid_b200.h"

namespace dg {

constexpr int kMaxSeg = DG_MAX_SEGMENTS;
constexpr int kMaxPart = DG_MAX_PARTITIONS;
constexpr int kMaxLevels = DG_MAX_LEVELS;
constexpr int kEnc = 32;       // encoded width on device: L*F padded to 32 (F == 2)
constexpr int kHidden = 64;    // field.hpp:15
constexpr int kColorIn = 48;   // 15 + 16 + d_app(<=16) padded to 48
constexpr int kDensOut = 16;   // 1 + 15

// ---- bit-exact fp64 (no contraction) ----
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
// std::max(a,b) returns a unless a < b; std::min(a,b) returns a unless b < a.
__host__ __device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__host__ __device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__host__ __device__ __forceinline__ double sclamp(double v, double lo, double hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}

// ---- rng.hpp:8-29 ----
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t counter_hash(uint64_t seed, uint64_t a, uint64_t b,
                                                          uint64_t c) {
  uint64_t h = splitmix64(seed ^ 0x6a09e667f3bcc909ull);
  h = splitmix64(h ^ a);
  h = splitmix64(h ^ b);
  h = splitmix64(h ^ c);
  return h;
}
__device__ __forceinline__ double counter_uniform(uint64_t seed, uint64_t a, uint64_t b) {
  return dmul((double)(counter_hash(seed, a, b, 0) >> 11), 0x1.0p-53);
}

// ---- descriptors (device-resident, built on the host at context creation) ----
struct LevelDesc {
  uint32_t n[3];     // lattice shape (grid.cpp:65-73)
  uint32_t hashed;   // MappingMode::Hashed (grid.cpp:97-99)
  uint32_t mask;     // rows - 1 when hashed
  uint32_t rows;     // table rows (2^T when hashed, n0 n1 n2 when one-to-one)
  uint64_t offset;   // floats from the field base to this level's table (rows x 2)
  uint64_t poff;     // paired copy (one-to-one levels): float4 index of row 0 in the context's
                     // pair buffers (pairs[r] = rows r, r + 1 of the table; kNoPair: none)
};
constexpr uint64_t kNoPair = ~0ull;

struct FieldDesc {   // one (partition, cascade) sub-field: FieldParams + its box
  double box_lo[3], box_hi[3];
  uint32_t L;        // levels
  uint32_t coarse;   // sigmoid hidden units in the colour MLP (field.cpp:196-199)
  uint32_t app_dim;
  uint32_t part;     // local partition index
  LevelDesc lv[kMaxLevels];
  uint64_t base;     // float offset of this field in the context's parameter buffer
  uint64_t dw0, db0, dw1, db1, cw0, cb0, cw1, cb1, cw2, cb2;  // relative to base
  uint64_t size;
};

struct PartDesc {    // one local partition (region)
  double fine_lo[3], fine_hi[3];
  double coarse_lo[3], coarse_hi[3];
  uint32_t occ_n[2][3];
  uint32_t occ_nb[2][3];  // bricks per axis of the bitfield (occ_addr)
  uint64_t occ_off[2];    // byte offsets of the bricked bitfields in the occupancy buffer
  uint64_t den_off[2];    // float offsets of the (linear) densities
  uint32_t global_id;
  uint32_t pad;
};

struct Geo {         // PartitionManifest planes + outer box (partition.cpp:206-252)
  double outer_lo[3], outer_hi[3];
  double xp[kMaxPart + 1], yp[kMaxPart + 1];
  uint32_t kx, ky, P, pad;
};

// Occupancy bitfield layout: 4 x 4 x 8 cell bricks of 128 bytes (one L1 line), bricks in
// x-fastest order.  A ray's DDA walk (grid.cpp:235-304) touches a new line every 4-8 cells
// instead of every cell a linear z-stride layout would cost.
constexpr uint32_t kOccBX = 4, kOccBY = 4, kOccBZ = 8;
__host__ __device__ __forceinline__ uint64_t occ_addr(const uint32_t nb[3], uint32_t x, uint32_t y,
                                                       uint32_t z) {
  const uint64_t brick = ((uint64_t)(z / kOccBZ) * nb[1] + y / kOccBY) * nb[0] + x / kOccBX;
  return brick * (kOccBX * kOccBY * kOccBZ) + ((z % kOccBZ) * kOccBY + y % kOccBY) * kOccBX + x % kOccBX;
}

// Dispatch record (exchange 1): DispatchRay minus the schedule, which the owner
// recomputes bit-exactly from (origin, dir).
struct __align__(8) RayRec {
  double o[3];
  double d[3];
  float gt[3];
  uint32_t img;
  uint32_t ray_id;
  uint32_t pad;
};
static_assert(sizeof(RayRec) == 72, "RayRec layout");

// Partial record (exchange 2 / eval reply): PartialEntry payload (wire.hpp:143-155).
// The segment transmittance travels as its optical depth tau (T = exp(-tau)): the same
// information as T, but 1 - T = -expm1(-tau) stays accurate when T -> 1, where the
// transmittance loss gradient lambda / (1 - T) (train.cpp:30-33) is largest.
struct __align__(8) PartialRec {
  float rgb[3];
  float tau;
  float depth;
  uint32_t ray_id;
};
static_assert(sizeof(PartialRec) == 24, "PartialRec layout");

}  // namespace dg
