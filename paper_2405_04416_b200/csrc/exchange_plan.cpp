// exchange_plan.cpp — see exchange_plan.h.
#include "exchange_plan.h"

#include "distgrid_b200.h"

namespace dg {

std::vector<uint32_t> local_partitions(int rank, int world, uint32_t P) {
  std::vector<uint32_t> l;
  for (uint32_t p = 0; p < P; ++p)
    if (int(p % uint32_t(world)) == rank) l.push_back(p);
  return l;
}

void plan_dispatch(int rank, int world, uint32_t P, const uint64_t* send_cnt, const uint64_t* cnt_recv,
                   uint64_t rec_bytes, DispatchPlan& out) {
  const std::vector<uint32_t> local = local_partitions(rank, world, P);
  const uint32_t nl = uint32_t(local.size());
  const int W = world;
  out.send_bytes.assign(W, 0);
  out.recv_bytes.assign(W, 0);
  for (uint32_t p = 0; p < P; ++p) out.send_bytes[p % uint32_t(W)] += send_cnt[p] * rec_bytes;
  for (int r = 0; r < W; ++r)
    for (uint32_t lp = 0; lp < nl; ++lp) out.recv_bytes[r] += cnt_recv[uint64_t(r) * P + local[lp]] * rec_bytes;
  out.item_off.assign(nl + 1, 0);
  for (uint32_t lp = 0; lp < nl; ++lp) {
    uint64_t t = 0;
    for (int r = 0; r < W; ++r) t += cnt_recv[uint64_t(r) * P + local[lp]];
    out.item_off[lp + 1] = out.item_off[lp] + uint32_t(t);
  }
  out.n_items = out.item_off[nl];
  const uint32_t nblk = nl * uint32_t(W);
  out.block_src.assign(nblk, 0);
  out.block_dst.assign(nblk, 0);
  uint64_t acc = 0;
  std::vector<uint64_t> run(nl, 0);
  for (int r = 0; r < W; ++r)  // received blocks in [src][lp] order
    for (uint32_t lp = 0; lp < nl; ++lp) {
      const uint64_t c = cnt_recv[uint64_t(r) * P + local[lp]];
      out.block_src[uint64_t(r) * nl + lp] = acc;
      out.block_dst[uint64_t(r) * nl + lp] = out.item_off[lp] + run[lp];
      acc += c;
      run[lp] += c;
    }
}

void plan_partials(int rank, int world, uint32_t P, const uint32_t* pair_cnt, uint64_t rec_bytes,
                   PartialPlan& out) {
  const std::vector<uint32_t> local = local_partitions(rank, world, P);
  const uint32_t nl = uint32_t(local.size());
  const int W = world;
  std::vector<int> local_of(P, -1);
  for (uint32_t lp = 0; lp < nl; ++lp) local_of[local[lp]] = int(lp);
  auto cnt = [&](uint32_t q, uint32_t p) -> uint64_t {  // records in stream q -> p (symmetric)
    if (local_of[q] >= 0) return pair_cnt[uint64_t(local_of[q]) * P + p];
    return pair_cnt[uint64_t(local_of[p]) * P + q];
  };
  out.send_off.assign(uint64_t(P) * P, 0);
  out.recv_off.assign(uint64_t(P) * P, 0);
  out.send_bytes.assign(W, 0);
  out.recv_bytes.assign(W, 0);
  uint64_t so = 0, ro = 0;
  for (int r = 0; r < W; ++r) {  // send layout: [dest r][q local][p on r]
    const uint64_t start = so;
    for (uint32_t lq = 0; lq < nl; ++lq)
      for (uint32_t p = 0; p < P; ++p)
        if (int(p % uint32_t(W)) == r && p != local[lq]) {
          out.send_off[uint64_t(local[lq]) * P + p] = so;
          so += cnt(local[lq], p);
        }
    out.send_bytes[r] = (so - start) * rec_bytes;
  }
  for (int r = 0; r < W; ++r) {  // recv layout: [src r][q on r][p local]
    const uint64_t start = ro;
    for (uint32_t q = 0; q < P; ++q)
      if (int(q % uint32_t(W)) == r)
        for (uint32_t lp = 0; lp < nl; ++lp)
          if (q != local[lp]) {
            out.recv_off[uint64_t(q) * P + local[lp]] = ro;
            ro += cnt(q, local[lp]);
          }
    out.recv_bytes[r] = (ro - start) * rec_bytes;
  }
  out.send_total = so;
  out.recv_total = ro;
}

}  // namespace dg

// ---- C ABI (host only; distgrid_b200.h) ----
using namespace dg;

extern "C" int dg_plan_dispatch(int rank, int world, uint32_t P, const uint64_t* send_cnt,
                                const uint64_t* cnt_recv, uint64_t* send_bytes, uint64_t* recv_bytes,
                                uint32_t* item_off, uint64_t* block_src, uint64_t* block_dst) {
  if (world < 1 || rank < 0 || rank >= world || P < 1 || P > DG_MAX_PARTITIONS || !send_cnt || !cnt_recv)
    return DG_EINVAL;
  DispatchPlan pl;
  plan_dispatch(rank, world, P, send_cnt, cnt_recv, 72, pl);
  for (int r = 0; r < world; ++r) {
    if (send_bytes) send_bytes[r] = pl.send_bytes[r];
    if (recv_bytes) recv_bytes[r] = pl.recv_bytes[r];
  }
  for (size_t i = 0; i < pl.item_off.size(); ++i)
    if (item_off) item_off[i] = pl.item_off[i];
  for (size_t i = 0; i < pl.block_src.size(); ++i) {
    if (block_src) block_src[i] = pl.block_src[i];
    if (block_dst) block_dst[i] = pl.block_dst[i];
  }
  return DG_OK;
}

extern "C" int dg_plan_partials(int rank, int world, uint32_t P, const uint32_t* pair_cnt, uint64_t* send_off,
                                uint64_t* recv_off, uint64_t* send_bytes, uint64_t* recv_bytes) {
  if (world < 1 || rank < 0 || rank >= world || P < 1 || P > DG_MAX_PARTITIONS || !pair_cnt) return DG_EINVAL;
  PartialPlan pl;
  plan_partials(rank, world, P, pair_cnt, 24, pl);
  for (uint64_t i = 0; i < uint64_t(P) * P; ++i) {
    if (send_off) send_off[i] = pl.send_off[i];
    if (recv_off) recv_off[i] = pl.recv_off[i];
  }
  for (int r = 0; r < world; ++r) {
    if (send_bytes) send_bytes[r] = pl.send_bytes[r];
    if (recv_bytes) recv_bytes[r] = pl.recv_bytes[r];
  }
  return DG_OK;
}
