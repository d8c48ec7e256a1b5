// b200_session.hpp -- glue between the reference's stateless C++ API and the
// device contexts of libdpdb (include/dpdb.h).  Internal to the drop-in.
//
// The reference's hot-path functions take host containers (ParticleStore,
// CellGrid, NeighborTable, inc/core.hpp:29-47, inc/cell_grid.hpp:21-70,
// inc/neighbor_table.hpp:18-40) and a WorkerPool.  The drop-in keeps one
// device context per calling thread, rebuilt when the box, the pair/run
// parameters or the capacity change, uploads the containers each call and
// downloads the results: the host containers stay the source of truth, as
// the reference's callers expect.  The WorkerPool argument is accepted and
// ignored (the device is the worker team).  libdpdb has no CPU fallback:
// without an sm_100 device every call throws dpd::Error.
#pragma once
#include <cstdint>
#include <string>

#include "dpd/core.hpp"
#include "dpd/error.hpp"
#include "dpdb.h"

namespace dpd::b200 {

// The reference's four categories (inc/error.hpp:8-13); libdpdb's device
// error (5) has no counterpart and surfaces as io (an environment failure).
[[noreturn]] void raise(int rc, const std::string& what);
void check(int rc, const dpdb_ctx* ctx, const char* where);

dpdb_box to_box(const SimBox& box);
dpdb_params to_params(const PairParams& p);

struct ContextKey {
    dpdb_box box{};
    dpdb_params params{};
    dpdb_run run{};
    std::size_t capacity = 0;
};

// The calling thread's context for this key (created or re-created on demand).
dpdb_ctx* context(const ContextKey& key);

// Default pair parameters of a given cutoff (the builder and the reorder use
// only r_c + skin and the grid; the pair coefficients do not matter there).
PairParams cutoff_params(double r_c);
dpdb_run run_config(double skin, std::uint32_t max_neighbors, std::uint32_t seed, int sub_bits);

// Upload the store's particles (x, v, tag, species, molecule) in their order.
void upload(dpdb_ctx* ctx, const ParticleStore& store);

}  // namespace dpd::b200
