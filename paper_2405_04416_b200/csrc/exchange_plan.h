// exchange_plan.h — host-side layout planning of the two per-step exchanges.
//
// Pure host code (no device work), shared by the runtime and exported through the C ABI
// (dg_plan_dispatch / dg_plan_partials) so multi-process CPU tests can check the protocol.
//
// Placement: partition p lives on rank p % world (the runtime's rule, worker.cpp:630-690 keeps
// one Worker per region; here several regions may share a rank).
//
// Exchange 1 (rays -> owners, RayDispatch, wire.cpp:29-46): a rank's send buffer is laid out
// [dest rank][partition on dest][ray]; the receiver gets [src rank][local partition][ray] and
// block-permutes it into items [local partition][src rank][ray], which is global ray order
// because home shards are contiguous in rank order.
//
// Exchange 2 (partials among owners, PartialScatter, worker.cpp:314-360): stream (q -> p)
// carries q's partials for the rays whose schedule contains p, in ray order; its length is
// pair_cnt(q, p) = #rays through both q and p, symmetric, so both ends size it locally.
#pragma once

#include <cstdint>
#include <vector>

namespace dg {

struct DispatchPlan {
  std::vector<uint64_t> send_bytes, recv_bytes;  // per rank
  std::vector<uint32_t> item_off;                // n_local + 1: items of each local partition
  std::vector<uint64_t> block_src, block_dst;    // W * n_local blocks: recv [src][lp] -> items
  uint64_t n_items = 0;
};

// send_cnt[p]: records this rank sends to partition p (global id); cnt_recv[src * P + p]:
// records rank src sends to partition p (the count vectors every rank broadcasts).
void plan_dispatch(int rank, int world, uint32_t P, const uint64_t* send_cnt, const uint64_t* cnt_recv,
                   uint64_t rec_bytes, DispatchPlan& out);

struct PartialPlan {
  std::vector<uint64_t> send_off, recv_off;      // P x P record offsets of stream (q -> p)
  std::vector<uint64_t> send_bytes, recv_bytes;  // per rank
  uint64_t send_total = 0, recv_total = 0;       // records
};

// pair_cnt[lq * P + p]: items of local partition lq whose ray schedule contains p.
void plan_partials(int rank, int world, uint32_t P, const uint32_t* pair_cnt, uint64_t rec_bytes,
                   PartialPlan& out);

// local partitions of a rank, ascending
std::vector<uint32_t> local_partitions(int rank, int world, uint32_t P);

}  // namespace dg
