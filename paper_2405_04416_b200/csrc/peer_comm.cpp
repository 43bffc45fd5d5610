// peer_comm.cpp — the peer-memory exchange backend (see comm.h, PeerComm).
//
// Buffers: one cudaMalloc per kind (items, partials, cross aggregates, generic stage), with a
// capacity that is uniform across ranks and grows collectively (every rank derives the same
// need from the same all-gathered counts).  Growth: every rank unmaps its peers' old buffers,
// a barrier, free + allocate its own, all-gather the new IPC handles, map the peers' buffers.
#include <chrono>
#include <cstring>

#include "comm.h"

namespace dg {

namespace {

bool cu_ok(cudaError_t e, const char* what, std::string& err) {
  if (e == cudaSuccess) return true;
  err = std::string("peer comm: ") + what + ": " + cudaGetErrorString(e);
  cudaGetLastError();
  return false;
}

}  // namespace

PeerComm::PeerComm(dg_allgather_fn fn, void* user, int rank, int world)
    : fn_(fn), user_(user), rank_(rank), world_(world) {}

void PeerComm::unmap(Buf& b) {
  for (int r = 0; r < world_; ++r)
    if (r != rank_ && r < int(b.peer.size()) && b.peer[r]) cudaIpcCloseMemHandle(b.peer[r]);
  b.peer.assign(world_, nullptr);
}

PeerComm::~PeerComm() {
  for (Buf& b : buf_) {
    unmap(b);
    if (b.local) cudaFree(b.local);
    if (b.dev) cudaFree(b.dev);
  }
  for (int r = 0; r < int(ctrl_peer_.size()); ++r)
    if (r != rank_ && ctrl_peer_[r]) cudaIpcCloseMemHandle(ctrl_peer_[r]);
  if (ctrl_) cudaFree(ctrl_);
  if (ctrl_s_) cudaStreamDestroy(ctrl_s_);
  if (ctrl_pin_) cudaFreeHost(ctrl_pin_);
}

int PeerComm::host_allgather(const void* send, uint64_t bytes, void* recv, std::string& err) {
  if (fn_(user_, send, bytes, recv) != 0) {
    err = "peer comm: all-gather callback failed";
    return DG_ETIMEOUT;
  }
  return DG_OK;
}

// The control buffer and its peers' mappings (the one exchange that needs the host callback).
int PeerComm::control_init(std::string& err) {
  const uint64_t bytes = uint64_t(world_) * (8 + 2 * kSlot);
  if (!cu_ok(cudaMalloc(&ctrl_, bytes), "cudaMalloc (control)", err)) return DG_ENOMEM;
  if (!cu_ok(cudaMemset(ctrl_, 0, bytes), "cudaMemset (control)", err)) return DG_ECUDA;
  if (!cu_ok(cudaStreamCreateWithFlags(&ctrl_s_, cudaStreamNonBlocking), "cudaStreamCreate", err)) return DG_ECUDA;
  if (!cu_ok(cudaHostAlloc(reinterpret_cast<void**>(&ctrl_pin_), 8 * (1 + world_) + kSlot * world_,
                           cudaHostAllocDefault),
             "cudaHostAlloc (control)", err))
    return DG_ENOMEM;
  cudaIpcMemHandle_t h;
  if (!cu_ok(cudaIpcGetMemHandle(&h, ctrl_), "cudaIpcGetMemHandle (control)", err)) return DG_ECUDA;
  std::vector<cudaIpcMemHandle_t> all(world_);
  int rc = host_allgather(&h, sizeof h, all.data(), err);
  if (rc != DG_OK) return rc;
  ctrl_peer_.assign(world_, nullptr);
  for (int r = 0; r < world_; ++r) {
    if (r == rank_) {
      ctrl_peer_[r] = ctrl_;
      continue;
    }
    if (!cu_ok(cudaIpcOpenMemHandle(&ctrl_peer_[r], all[r], cudaIpcMemLazyEnablePeerAccess),
               "cudaIpcOpenMemHandle (control)", err))
      return DG_ECUDA;
  }
  // every rank has mapped every control buffer before anyone writes into one
  const uint8_t token = 1;
  std::vector<uint8_t> t(world_);
  rc = host_allgather(&token, 1, t.data(), err);
  if (rc != DG_OK) return rc;
  ctrl_ok_ = true;
  return DG_OK;
}

int PeerComm::allgather(const void* send, uint64_t bytes, void* recv, std::string& err) {
  if (!ctrl_ok_) {
    if (bytes > kSlot || fn_ == nullptr) return host_allgather(send, bytes, recv, err);
    const int rc = control_init(err);
    if (rc != DG_OK) return rc;
  }
  if (bytes > kSlot) return host_allgather(send, bytes, recv, err);
  const uint64_t epoch = ++epoch_;
  uint64_t* src_epoch = ctrl_pin_;
  uint64_t* flags = ctrl_pin_ + 1;
  uint8_t* stage = reinterpret_cast<uint8_t*>(ctrl_pin_ + 1 + world_);
  *src_epoch = epoch;
  std::memcpy(stage, send, bytes);
  // payload into slot [epoch parity][rank] of every control buffer, then the epoch into flag
  // [rank]; one stream, so each flag lands after its payload.  Two slot sets: a rank that has
  // finished epoch e can write e + 1 while a slower peer still reads e, but it cannot start
  // e + 2 before every peer has raised its flag to e + 1, i.e. finished reading e.
  const uint64_t slots = 8 * uint64_t(world_) + kSlot * uint64_t(world_) * (epoch & 1);
  for (int q = 0; q < world_; ++q) {
    uint8_t* base = static_cast<uint8_t*>(ctrl_peer_[q]);
    if (!cu_ok(cudaMemcpyAsync(base + slots + kSlot * rank_, stage, bytes, cudaMemcpyDefault, ctrl_s_),
               "control payload copy", err))
      return DG_ECUDA;
  }
  for (int q = 0; q < world_; ++q) {
    uint8_t* base = static_cast<uint8_t*>(ctrl_peer_[q]);
    if (!cu_ok(cudaMemcpyAsync(base + 8 * rank_, src_epoch, 8, cudaMemcpyDefault, ctrl_s_),
               "control flag copy", err))
      return DG_ECUDA;
  }
  if (!cu_ok(cudaStreamSynchronize(ctrl_s_), "control stream sync", err)) return DG_ECUDA;
  // poll this rank's flags until every peer's epoch has arrived
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    if (!cu_ok(cudaMemcpyAsync(flags, ctrl_, 8 * world_, cudaMemcpyDeviceToHost, ctrl_s_), "control poll", err) ||
        !cu_ok(cudaStreamSynchronize(ctrl_s_), "control poll sync", err))
      return DG_ECUDA;
    bool all = true;
    for (int r = 0; r < world_; ++r) all = all && flags[r] >= epoch;
    if (all) break;
    if (std::chrono::steady_clock::now() - t0 > timeout()) {
      err = "peer comm: missing PartialScatter (a peer did not reach the exchange in time)";
      return DG_ETIMEOUT;
    }
  }
  // the slots: every rank wrote its payload before its flag
  for (int r = 0; r < world_; ++r)
    if (!cu_ok(cudaMemcpyAsync(stage + bytes * r, static_cast<uint8_t*>(ctrl_) + slots + kSlot * r, bytes,
                               cudaMemcpyDeviceToHost, ctrl_s_),
               "control read", err))
      return DG_ECUDA;
  if (!cu_ok(cudaStreamSynchronize(ctrl_s_), "control read sync", err)) return DG_ECUDA;
  std::memcpy(recv, stage, bytes * world_);
  return DG_OK;
}

int PeerComm::barrier(cudaStream_t s, std::string& err) {
  if (!cu_ok(cudaStreamSynchronize(s), "stream sync", err)) return DG_ECUDA;
  const uint8_t token = 1;
  std::vector<uint8_t> all(world_);
  return allgather(&token, 1, all.data(), err);
}

int PeerComm::reserve(int k, uint64_t need, std::string& err) {
  Buf& b = buf_[k];
  if (need <= b.cap && b.local) return DG_OK;
  const uint64_t cap = need + need / 4 + 4096;
  unmap(b);
  int rc = barrier(nullptr, err);  // nobody maps the old buffers any more
  if (rc != DG_OK) return rc;
  if (b.local) cudaFree(b.local);
  b.local = nullptr;
  b.cap = 0;
  if (!cu_ok(cudaMalloc(&b.local, cap), "cudaMalloc", err)) return DG_ENOMEM;
  b.cap = cap;
  cudaIpcMemHandle_t h;
  if (!cu_ok(cudaIpcGetMemHandle(&h, b.local), "cudaIpcGetMemHandle", err)) return DG_ECUDA;
  std::vector<cudaIpcMemHandle_t> all(world_);
  rc = allgather(&h, sizeof h, all.data(), err);
  if (rc != DG_OK) return rc;
  b.peer.assign(world_, nullptr);
  for (int r = 0; r < world_; ++r) {
    if (r == rank_) {
      b.peer[r] = b.local;
      continue;
    }
    if (!cu_ok(cudaIpcOpenMemHandle(&b.peer[r], all[r], cudaIpcMemLazyEnablePeerAccess),
               "cudaIpcOpenMemHandle", err))
      return DG_ECUDA;
  }
  if (!b.dev && !cu_ok(cudaMalloc(reinterpret_cast<void**>(&b.dev), sizeof(void*) * world_), "cudaMalloc",
                       err))
    return DG_ENOMEM;
  if (!cu_ok(cudaMemcpy(b.dev, b.peer.data(), sizeof(void*) * world_, cudaMemcpyHostToDevice), "cudaMemcpy",
             err))
    return DG_ECUDA;
  return DG_OK;
}

// All-to-all-v through the stage buffers: rank r's stage holds [src][block] in rank order
// (= the recv layout), each sender copies its block into every receiver's stage over the
// peer mapping, a barrier, then each rank copies its stage into recv.
int PeerComm::alltoallv(const void* send, const std::vector<uint64_t>& sb, void* recv,
                        const std::vector<uint64_t>& rb, cudaStream_t s, std::string& err) {
  const int W = world_;
  std::vector<uint64_t> all(uint64_t(W) * W);  // all[src * W + dst]
  int rc = allgather(sb.data(), sizeof(uint64_t) * W, all.data(), err);
  if (rc != DG_OK) return rc;
  uint64_t need = 0;
  for (int dst = 0; dst < W; ++dst) {
    uint64_t t = 0;
    for (int src = 0; src < W; ++src) t += all[uint64_t(src) * W + dst];
    need = std::max(need, t);
  }
  rc = reserve(kStage, need, err);
  if (rc != DG_OK) return rc;
  uint64_t soff = 0;
  for (int dst = 0; dst < W; ++dst) {
    uint64_t at = 0;  // my block's place in dst's stage
    for (int src = 0; src < rank_; ++src) at += all[uint64_t(src) * W + dst];
    if (sb[dst] &&
        !cu_ok(cudaMemcpyAsync(static_cast<char*>(buf_[kStage].peer[dst]) + at,
                               static_cast<const char*>(send) + soff, sb[dst], cudaMemcpyDeviceToDevice, s),
               "peer copy", err))
      return DG_ECUDA;
    soff += sb[dst];
  }
  rc = barrier(s, err);
  if (rc != DG_OK) return rc;
  uint64_t rt = 0;
  for (int src = 0; src < W; ++src) rt += rb[src];
  if (rt && !cu_ok(cudaMemcpyAsync(recv, buf_[kStage].local, rt, cudaMemcpyDeviceToDevice, s), "stage copy", err))
    return DG_ECUDA;
  // the stage is reused by the next call: done with it before anyone writes it again
  return cu_ok(cudaStreamSynchronize(s), "stream sync", err) ? DG_OK : DG_ECUDA;
}

}  // namespace dg
