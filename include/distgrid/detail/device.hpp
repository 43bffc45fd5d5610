// distgrid/detail/device.hpp — glue between the facade headers and the C ABI
// (include/distgrid_b200.h, libdg_b200.so): status codes become the reference's exception
// classes, and stateless stage functions run on one lazily created per-thread
// context.  Every computation behind the facade runs on the GPU; there is no host fallback.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>

#include "distgrid_b200.h"

namespace distgrid {
namespace detail {

// DG_EINVAL -> invalid_argument (e.g. render.cpp:49-50, grid.cpp:111), DG_ERANGE ->
// out_of_range (grid.cpp:57,76-77), everything else (protocol, missing partials, I/O, CUDA,
// NCCL, timeouts) -> runtime_error.
inline void check(int rc) {
  if (rc == DG_OK) return;
  const std::string msg = dg_last_error();
  if (rc == DG_EINVAL) throw std::invalid_argument(msg);
  if (rc == DG_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

struct CtxDeleter {
  void operator()(dg_ctx* c) const {
    if (c) dg_ctx_destroy(c);
  }
};
using CtxPtr = std::unique_ptr<dg_ctx, CtxDeleter>;

// A minimal context (one region, one tiny grid level, no occupancy updates) whose stream and
// scratch carry the stateless stage calls (compositing, merges, losses, march, slab test,
// Adam over caller arrays).  One per host thread: a context is single-threaded.
inline dg_ctx* stage_ctx() {
  thread_local CtxPtr ctx = [] {
    dg_run_config cfg;
    dg_default_config(&cfg);
    cfg.grid_levels = 1;
    cfg.base_resolution = 2;
    cfg.max_resolution = 2;
    cfg.fine_table_log2 = 4;
    cfg.coarse_table_log2 = 4;
    cfg.occ_resolution = 8;
    cfg.occupancy_updates = 0;
    dg_ctx* c = nullptr;
    check(dg_ctx_create(&cfg, -1, 0, 1, &c));
    return CtxPtr(c);
  }();
  return ctx.get();
}

}  // namespace detail
}  // namespace distgrid
