// comm.h — the exchange backend behind dg_comm_init_* (replaces the reference Transport,
// transport.hpp:30-98).  One all-to-all-v primitive over device buffers whose per-peer blocks
// are contiguous in rank order.  Production: NCCL grouped send/recv over NVLink/NVSwitch
// (libnccl resolved at run time, so the library also loads where NCCL is absent).  Tests:
// a host-staged backend that hands the blocks to a caller-provided callback (gloo).
#pragma once

#include <chrono>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "distgrid_b200.h"

namespace dg {

class PeerComm;

class Comm {
 public:
  virtual ~Comm() = default;
  // the peer-memory backend, whose receive buffers the pack kernels write directly
  virtual PeerComm* peer() { return nullptr; }
  // send/recv: device buffers; bytes per peer (rank order).  Returns DG_OK or an error code;
  // err receives a message.
  virtual int alltoallv(const void* send, const std::vector<uint64_t>& send_bytes, void* recv,
                        const std::vector<uint64_t>& recv_bytes, cudaStream_t s,
                        std::string& err) = 0;
  virtual const char* name() const = 0;
  // Asynchronous failure of the backend (a dead or failed peer): DG_OK or an error code.
  virtual int poll(std::string& err) { return DG_OK; }
  // Give up on every in-flight exchange (the device work waiting on peers returns).
  virtual void abort() {}
  // How long a step may wait for its peers (Worker::Setup::recv_timeout, worker.hpp:82).
  virtual void set_timeout(std::chrono::milliseconds t) { timeout_ = t; }
  virtual std::chrono::milliseconds timeout() const { return timeout_; }

 protected:
  std::chrono::milliseconds timeout_{120000};
};

// Exchanges over peer memory (one node, NVLink / NVSwitch): every rank's receive buffers are
// CUDA-IPC mapped into every other rank, so the two pack kernels store each record straight
// into its owner's buffer, in the owner's final layout — no staging buffer, no collective copy
// kernel, no receive-side permute.  The per-step count matrices and the barriers travel over a
// control buffer in device memory, CUDA-IPC mapped like the data buffers: a rank copies its
// payload into slot [rank] of every peer's control buffer and then an epoch word into flag
// [rank] (one copy stream, so the flag lands after the payload), and polls its own flags until
// every peer's epoch has arrived (bounded by the step timeout).  The host all-gather callback
// only bootstraps the control buffer's IPC handles.  No kernel ever waits on a peer: a barrier
// is a stream sync + an all-gather, after which every rank's pack kernel has completed.
class PeerComm final : public Comm {
 public:
  enum { kItems = 0, kPartials = 1, kCross = 2, kStage = 3, kBufs = 4 };
  PeerComm(dg_allgather_fn fn, void* user, int rank, int world);
  ~PeerComm() override;
  // generic all-to-all-v (staged through kStage) for the exchanges without a fused pack
  int alltoallv(const void* send, const std::vector<uint64_t>& send_bytes, void* recv,
                const std::vector<uint64_t>& recv_bytes, cudaStream_t s, std::string& err) override;
  const char* name() const override { return "peer"; }
  PeerComm* peer() override { return this; }
  // all-gather of `bytes` per rank (rank order) over the control buffer; the host callback
  // before the control buffer exists
  int allgather(const void* send, uint64_t bytes, void* recv, std::string& err);
  int barrier(cudaStream_t s, std::string& err);
  uint64_t control_exchanges() const { return epoch_; }
  // collective: every rank's buffer k holds >= need bytes afterwards (need identical on all ranks)
  int reserve(int k, uint64_t need, std::string& err);
  void* local(int k) const { return buf_[k].local; }
  void* const* peers_dev(int k) const { return buf_[k].dev; }
  int rank() const { return rank_; }
  int world() const { return world_; }

 private:
  struct Buf {
    void* local = nullptr;
    uint64_t cap = 0;
    std::vector<void*> peer;  // mapped bases (own rank: local)
    void** dev = nullptr;     // the same pointers on the device
  };
  void unmap(Buf& b);
  int host_allgather(const void* send, uint64_t bytes, void* recv, std::string& err);
  int control_init(std::string& err);
  static constexpr uint64_t kSlot = 16384;  // bytes per rank and exchange (count matrices, handles)
  dg_allgather_fn fn_;
  void* user_;
  int rank_, world_;
  Buf buf_[kBufs];
  // control buffer: [world] epoch flags (u64), then [2 (epoch parity)][world] slots of kSlot bytes
  void* ctrl_ = nullptr;
  std::vector<void*> ctrl_peer_;
  cudaStream_t ctrl_s_ = nullptr;
  uint64_t* ctrl_pin_ = nullptr;  // pinned: [0] epoch source, [1..world] flag readback, staging after
  uint64_t epoch_ = 0;
  bool ctrl_ok_ = false;
};

Comm* make_nccl_comm(const uint8_t id[DG_NCCL_UNIQUE_ID_BYTES], int rank, int world, int device,
                     std::string& err, std::chrono::milliseconds timeout);
Comm* make_host_comm(dg_alltoallv_fn fn, void* user, int rank, int world);
int nccl_unique_id(uint8_t id[DG_NCCL_UNIQUE_ID_BYTES], std::string& err);

}  // namespace dg
