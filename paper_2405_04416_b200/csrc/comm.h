// comm.h — the exchange backend behind dg_comm_init_* (replaces the reference Transport,
// transport.hpp:30-98).  One all-to-all-v primitive over device buffers whose per-peer blocks
// are contiguous in rank order.  Production: NCCL grouped send/recv over NVLink/NVSwitch
// (libnccl resolved at run time, so the library also loads where NCCL is absent).  Tests:
// a host-staged backend that hands the blocks to a caller-provided callback (gloo).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "distgrid_b200.h"

namespace dg {

class Comm {
 public:
  virtual ~Comm() = default;
  // send/recv: device buffers; bytes per peer (rank order).  Returns DG_OK or an error code;
  // err receives a message.
  virtual int alltoallv(const void* send, const std::vector<uint64_t>& send_bytes, void* recv,
                        const std::vector<uint64_t>& recv_bytes, cudaStream_t s,
                        std::string& err) = 0;
  virtual const char* name() const = 0;
};

Comm* make_nccl_comm(const uint8_t id[DG_NCCL_UNIQUE_ID_BYTES], int rank, int world, int device,
                     std::string& err);
Comm* make_host_comm(dg_alltoallv_fn fn, void* user, int rank, int world);
int nccl_unique_id(uint8_t id[DG_NCCL_UNIQUE_ID_BYTES], std::string& err);

}  // namespace dg
