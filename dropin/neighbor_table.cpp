// neighbor_table.cpp (B200 drop-in) -- the reference's missing
// src/neighbor_table.cpp slot (CMakeLists.txt:21): the declarations of
// inc/neighbor_table.hpp:42-59 over libdpdb.
//
//   build_neighbor_table  -> dpdb_build_neighbors: the ordered, atomics-free
//                            range builder (k_build_range) in the reference's
//                            split layout (core ascending from the front, skin
//                            from the back), 32x32 tile-transposed (tiled = true;
//                            readers go through the accessors either way)
//   join_core_skin        -> dpdb_table_layout(op 0) (k_join)
//   tile_transpose        -> dpdb_table_layout(op 1) (k_tile_transpose)
//   dump_neighbor_csv     -> host text dump of the table (debug output)
//
// The fine stencil argument is not needed: the builder walks the coarse
// stencil's cells as index ranges (octant-trimmed) and never materialises the
// fine stencil; the rows are the same (ascending index = fine-stencil order).
#include <cmath>
#include <ostream>
#include <string>
#include <vector>

#include "b200_session.hpp"
#include "dpd/neighbor_table.hpp"

namespace dpd {

NeighborTable build_neighbor_table(const ParticleStore& store, const CellGrid& grid, const FineStencil&,
                                   const SimBox& box, double r_c, double skin, std::uint32_t max_neighbors,
                                   WorkerPool&) {
    const std::size_t n = store.n;
    for (int k = 0; k < 3; ++k)
        if (grid.ghost_lo[k] || grid.ghost_hi[k])
            fail(ErrorCategory::config,
                 "B200 drop-in: grids with ghost layers run through the brick API (dpdb_create_domain)");
    b200::ContextKey key;
    key.box = b200::to_box(box);
    key.params = b200::to_params(b200::cutoff_params(r_c));
    key.run = b200::run_config(skin, max_neighbors, 1, grid.sub_bits);
    key.capacity = std::max<std::size_t>(n, 1);
    dpdb_ctx* ctx = b200::context(key);
    dpdb_grid_info info{};
    b200::check(dpdb_grid(ctx, &info), ctx, "grid");
    for (int k = 0; k < 3; ++k)
        if (info.ncell[k] != grid.ncell[k])
            fail(ErrorCategory::config, "build_neighbor_table: grid must be CellGrid::make(box, r_c + skin)");
    NeighborTable t;
    t.n_rows = (std::uint32_t)n;
    t.max_neighbors = max_neighbors;
    t.n_rows_pad = (std::uint32_t)((n + 31) & ~std::size_t(31));
    t.core_count.assign(n, 0);
    t.skin_count.assign(n, 0);
    t.entries.assign((std::size_t)t.n_rows_pad * max_neighbors, 0u);
    if (!n) return t;
    b200::upload(ctx, store);
    // the rows refer to the store's order: it must already be the grid order
    std::vector<std::uint32_t> perm(n);
    b200::check(dpdb_reorder(ctx, perm.data()), ctx, "build_neighbor_table");
    for (std::size_t i = 0; i < n; ++i)
        if (perm[i] != i)
            fail(ErrorCategory::config, "build_neighbor_table: particles not in cell order (reorder_particles first)");
    b200::check(dpdb_build_neighbors(ctx), ctx, "build_neighbor_table");
    int32_t tiled = 0, joined = 0;
    b200::check(dpdb_get_neighbors(ctx, t.entries.data(), t.core_count.data(), t.skin_count.data(), &tiled,
                                   &joined),
                ctx, "build_neighbor_table");
    t.tiled = tiled != 0;
    t.joined = joined != 0;
    return t;
}

void join_core_skin(NeighborTable& table, WorkerPool&) {
    if (table.joined) return;
    b200::check(dpdb_table_layout(0, 0, table.n_rows, table.max_neighbors, table.entries.data(),
                                  table.core_count.data(), table.skin_count.data(), table.tiled, 0),
                nullptr, "join_core_skin");
    table.joined = true;
}

void tile_transpose(NeighborTable& table, WorkerPool&) {
    b200::check(dpdb_table_layout(0, 1, table.n_rows, table.max_neighbors, table.entries.data(), nullptr,
                                  nullptr, table.tiled, table.joined),
                nullptr, "tile_transpose");
    table.tiled = !table.tiled;
}

void dump_neighbor_csv(const NeighborTable& table, const ParticleStore& store, const SimBox& box,
                       const std::array<bool, 3>& wrap, std::ostream& os) {
    os << "i_tag,j_tag,distance,partition\n";
    for (std::uint32_t i = 0; i < table.n_rows; ++i) {
        auto row = [&](std::uint32_t j, const char* part) {
            double d2 = 0.0;
            for (int k = 0; k < 3; ++k) {
                double d = store.coord[k][i] - store.coord[k][j];
                const double L = box.length(k);
                if (wrap[k]) d -= L * std::nearbyint(d / L);
                d2 += d * d;
            }
            os << store.tag[i] << ',' << store.tag[j] << ',' << std::sqrt(d2) << ',' << part << '\n';
        };
        for (std::uint32_t k = 0; k < table.core_count[i]; ++k) row(table.core_at(i, k), "core");
        for (std::uint32_t k = 0; k < table.skin_count[i]; ++k) row(table.skin_at(i, k), "skin");
    }
}

}  // namespace dpd
