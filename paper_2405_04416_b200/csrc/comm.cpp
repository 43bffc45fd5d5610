// comm.cpp — NCCL (dlopen'd) and host-staged all-to-all-v backends.
#include "comm.h"

#include <dlfcn.h>

#include <cstring>
#include <mutex>

namespace dg {

namespace {

// Minimal NCCL ABI (nccl.h, 2.2x): opaque comm, 128-byte unique id.
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclSuccess = 0 };
enum { ncclInt8 = 0, ncclUint8 = 1 };

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl(std::string& err) {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // Prefer an NCCL already loaded into the process (e.g. torch's), else the system one.
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!api.h) api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
#define DG_SYM(field, sym) api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.h, sym))
    DG_SYM(GetUniqueId, "ncclGetUniqueId");
    DG_SYM(CommInitRank, "ncclCommInitRank");
    DG_SYM(CommDestroy, "ncclCommDestroy");
    DG_SYM(Send, "ncclSend");
    DG_SYM(Recv, "ncclRecv");
    DG_SYM(GroupStart, "ncclGroupStart");
    DG_SYM(GroupEnd, "ncclGroupEnd");
    DG_SYM(GetErrorString, "ncclGetErrorString");
#undef DG_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.Send && api.Recv && api.GroupStart &&
             api.GroupEnd;
  });
  if (!api.ok) err = "NCCL not available (libnccl.so.2 could not be loaded)";
  return api;
}

class NcclComm final : public Comm {
 public:
  NcclComm(ncclComm_t c, int rank, int world) : comm_(c), rank_(rank), world_(world) {}
  ~NcclComm() override {
    std::string e;
    NcclApi& api = nccl(e);
    if (api.ok && api.CommDestroy) api.CommDestroy(comm_);
  }
  int alltoallv(const void* send, const std::vector<uint64_t>& sb, void* recv,
                const std::vector<uint64_t>& rb, cudaStream_t s, std::string& err) override {
    NcclApi& api = nccl(err);
    if (!api.ok) return DG_ENCCL;
    uint64_t so = 0, ro = 0;
    std::vector<uint64_t> soff(world_), roff(world_);
    for (int r = 0; r < world_; ++r) {
      soff[r] = so;
      roff[r] = ro;
      so += sb[r];
      ro += rb[r];
    }
    // self block: a device copy, the rest grouped send/recv (all-to-all-v over NVSwitch)
    if (sb[rank_] != rb[rank_]) {
      err = "alltoallv: self block size mismatch";
      return DG_EPROTO;
    }
    if (sb[rank_]) {
      if (cudaMemcpyAsync(static_cast<char*>(recv) + roff[rank_],
                          static_cast<const char*>(send) + soff[rank_], sb[rank_],
                          cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
        err = "alltoallv: self copy failed";
        return DG_ECUDA;
      }
    }
    ncclResult_t rc = api.GroupStart();
    for (int r = 0; r < world_ && rc == ncclSuccess; ++r) {
      if (r == rank_) continue;
      if (sb[r]) rc = api.Send(static_cast<const char*>(send) + soff[r], sb[r], ncclUint8, r, comm_, s);
      if (rc == ncclSuccess && rb[r])
        rc = api.Recv(static_cast<char*>(recv) + roff[r], rb[r], ncclUint8, r, comm_, s);
    }
    const ncclResult_t rc2 = api.GroupEnd();
    if (rc != ncclSuccess || rc2 != ncclSuccess) {
      err = std::string("NCCL all-to-all failed: ") +
            (api.GetErrorString ? api.GetErrorString(rc != ncclSuccess ? rc : rc2) : "?");
      return DG_ENCCL;
    }
    return DG_OK;
  }
  const char* name() const override { return "nccl"; }

 private:
  ncclComm_t comm_;
  int rank_, world_;
};

class HostComm final : public Comm {
 public:
  HostComm(dg_alltoallv_fn fn, void* user, int rank, int world)
      : fn_(fn), user_(user), rank_(rank), world_(world) {}
  int alltoallv(const void* send, const std::vector<uint64_t>& sb, void* recv,
                const std::vector<uint64_t>& rb, cudaStream_t s, std::string& err) override {
    uint64_t st = 0, rt = 0;
    for (int r = 0; r < world_; ++r) {
      st += sb[r];
      rt += rb[r];
    }
    std::vector<uint8_t> hs(st ? st : 1), hr(rt ? rt : 1);
    if (st && cudaMemcpyAsync(hs.data(), send, st, cudaMemcpyDeviceToHost, s) != cudaSuccess) {
      err = "host comm: D2H failed";
      return DG_ECUDA;
    }
    cudaStreamSynchronize(s);
    const int rc = fn_(user_, hs.data(), sb.data(), hr.data(), rb.data());
    if (rc != 0) {
      err = "host comm: exchange callback failed";
      return DG_ETIMEOUT;
    }
    if (rt && cudaMemcpyAsync(recv, hr.data(), rt, cudaMemcpyHostToDevice, s) != cudaSuccess) {
      err = "host comm: H2D failed";
      return DG_ECUDA;
    }
    cudaStreamSynchronize(s);
    return DG_OK;
  }
  const char* name() const override { return "host"; }

 private:
  dg_alltoallv_fn fn_;
  void* user_;
  int rank_, world_;
};

}  // namespace

int nccl_unique_id(uint8_t id[DG_NCCL_UNIQUE_ID_BYTES], std::string& err) {
  NcclApi& api = nccl(err);
  if (!api.ok) return DG_ENCCL;
  ncclUniqueId uid;
  if (api.GetUniqueId(&uid) != ncclSuccess) {
    err = "ncclGetUniqueId failed";
    return DG_ENCCL;
  }
  std::memcpy(id, uid.internal, DG_NCCL_UNIQUE_ID_BYTES);
  return DG_OK;
}

Comm* make_nccl_comm(const uint8_t id[DG_NCCL_UNIQUE_ID_BYTES], int rank, int world, int device,
                     std::string& err) {
  NcclApi& api = nccl(err);
  if (!api.ok) return nullptr;
  cudaSetDevice(device);
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, DG_NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  const ncclResult_t rc = api.CommInitRank(&c, world, uid, rank);
  if (rc != ncclSuccess) {
    err = std::string("ncclCommInitRank failed: ") + (api.GetErrorString ? api.GetErrorString(rc) : "?");
    return nullptr;
  }
  return new NcclComm(c, rank, world);
}

Comm* make_host_comm(dg_alltoallv_fn fn, void* user, int rank, int world) {
  return new HostComm(fn, user, rank, world);
}

}  // namespace dg
