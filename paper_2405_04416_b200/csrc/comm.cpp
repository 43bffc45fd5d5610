// comm.cpp — NCCL (dlopen'd) and host-staged all-to-all-v backends.
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <mutex>
#include <thread>

namespace dg {

namespace {

// The NCCL API is resolved at run time (dlopen), so the library also loads where NCCL is
// absent; the types come from the system nccl.h (ncclConfig_t carries its own size / version,
// so a newer runtime accepts it).
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  // non-blocking communicators: init, group launches and errors are polled against a deadline
  bool nonblocking() const { return CommInitRankConfig && CommGetAsyncError && CommAbort; }
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
    DG_SYM(CommInitRankConfig, "ncclCommInitRankConfig");
    DG_SYM(CommDestroy, "ncclCommDestroy");
    DG_SYM(CommAbort, "ncclCommAbort");
    DG_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
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

std::string nccl_msg(NcclApi& api, const char* what, ncclResult_t rc) {
  return std::string(what) + ": " + (api.GetErrorString ? api.GetErrorString(rc) : "?");
}

using Clock = std::chrono::steady_clock;

// Poll a non-blocking communicator until it leaves ncclInProgress (or the deadline passes).
ncclResult_t nccl_settle(NcclApi& api, ncclComm_t comm, Clock::time_point deadline, bool* timed_out) {
  ncclResult_t st = ncclInProgress;
  *timed_out = false;
  while (true) {
    if (api.CommGetAsyncError(comm, &st) != ncclSuccess) return ncclInternalError;
    if (st != ncclInProgress) return st;
    if (Clock::now() > deadline) {
      *timed_out = true;
      return ncclInProgress;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

class NcclComm final : public Comm {
 public:
  NcclComm(ncclComm_t c, int rank, int world, bool nb) : comm_(c), rank_(rank), world_(world), nb_(nb) {}
  ~NcclComm() override {
    std::string e;
    NcclApi& api = nccl(e);
    if (!api.ok || !comm_) return;
    if (aborted_ || !api.CommDestroy) return;
    api.CommDestroy(comm_);
  }
  int alltoallv(const void* send, const std::vector<uint64_t>& sb, void* recv,
                const std::vector<uint64_t>& rb, cudaStream_t s, std::string& err) override {
    NcclApi& api = nccl(err);
    if (!api.ok) return DG_ENCCL;
    if (aborted_) {
      err = "NCCL communicator was aborted after an earlier exchange failure";
      return DG_ENCCL;
    }
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
    for (int r = 0; r < world_ && (rc == ncclSuccess || rc == ncclInProgress); ++r) {
      if (r == rank_) continue;
      if (sb[r]) rc = api.Send(static_cast<const char*>(send) + soff[r], sb[r], ncclUint8, r, comm_, s);
      if ((rc == ncclSuccess || rc == ncclInProgress) && rb[r])
        rc = api.Recv(static_cast<char*>(recv) + roff[r], rb[r], ncclUint8, r, comm_, s);
    }
    ncclResult_t rc2 = api.GroupEnd();
    if (nb_ && rc2 == ncclInProgress) {  // the group is being set up (connections to peers)
      bool to = false;
      rc2 = nccl_settle(api, comm_, Clock::now() + timeout_, &to);
      if (to) {
        abort();
        err = "NCCL all-to-all: timed out connecting to peers (missing PartialScatter)";
        return DG_ETIMEOUT;
      }
    }
    if ((rc != ncclSuccess && rc != ncclInProgress) || rc2 != ncclSuccess) {
      err = nccl_msg(api, "NCCL all-to-all failed", rc != ncclSuccess && rc != ncclInProgress ? rc : rc2);
      return DG_ENCCL;
    }
    return DG_OK;
  }
  int poll(std::string& err) override {
    if (aborted_) {
      err = "NCCL communicator aborted";
      return DG_ENCCL;
    }
    NcclApi& api = nccl(err);
    if (!api.CommGetAsyncError) return DG_OK;
    ncclResult_t st = ncclSuccess;
    if (api.CommGetAsyncError(comm_, &st) != ncclSuccess || (st != ncclSuccess && st != ncclInProgress)) {
      err = nccl_msg(api, "NCCL asynchronous error", st);
      abort();
      return DG_ENCCL;
    }
    return DG_OK;
  }
  void abort() override {
    std::string e;
    NcclApi& api = nccl(e);
    if (!aborted_ && api.CommAbort) api.CommAbort(comm_);  // NCCL kernels in flight return
    aborted_ = true;
  }
  const char* name() const override { return "nccl"; }

 private:
  ncclComm_t comm_;
  int rank_, world_;
  bool nb_;
  bool aborted_ = false;
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
                     std::string& err, std::chrono::milliseconds timeout) {
  NcclApi& api = nccl(err);
  if (!api.ok) return nullptr;
  cudaSetDevice(device);
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, DG_NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  const bool nb = api.nonblocking();
  ncclResult_t rc;
  if (nb) {
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    rc = api.CommInitRankConfig(&c, world, uid, rank, &cfg);
    if (rc == ncclInProgress) {
      bool to = false;
      rc = nccl_settle(api, c, Clock::now() + timeout, &to);
      if (to) {
        api.CommAbort(c);
        err = "ncclCommInitRankConfig: timed out waiting for peers";
        return nullptr;
      }
    }
  } else {
    rc = api.CommInitRank(&c, world, uid, rank);
  }
  if (rc != ncclSuccess) {
    err = nccl_msg(api, "ncclCommInitRank failed", rc);
    if (c && api.CommAbort) api.CommAbort(c);
    return nullptr;
  }
  NcclComm* comm = new NcclComm(c, rank, world, nb);
  comm->set_timeout(timeout);
  return comm;
}

Comm* make_host_comm(dg_alltoallv_fn fn, void* user, int rank, int world) {
  return new HostComm(fn, user, rank, world);
}

}  // namespace dg
