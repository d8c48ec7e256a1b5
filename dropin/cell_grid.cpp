// cell_grid.cpp (B200 drop-in) -- replaces the reference's src/cell_grid.cpp:
// every declaration of inc/cell_grid.hpp, with the reorder on the device.
//
//   CellGrid::make (both)      inc/cell_grid.hpp:39-43  -> dpdb_grid_plan (host,
//                              the same grid every libdpdb context builds)
//   reorder_particles          inc/cell_grid.hpp:78-79  -> dpdb_reorder: sort keys,
//                              stable radix sort, gather and cell list on the
//                              device; the sorter argument is unused
//   local_cell_ranks           inc/cell_grid.hpp:82-83  -> dpdb_sort_keys (device)
//   build_cell_list            inc/cell_grid.hpp:74     -> host boundary scan over
//                              the caller's ranks (the device fuses the same
//                              scan into its permute kernel)
//   local_cell_of / ghost_cell_of / sub_code / key_bits -> the grid arithmetic
//                              of the device key kernel, per particle
//
// Single-domain grids only for the device paths (no ghost layers): a brick of
// a decomposition runs through libdpdb's brick API (dpdb_create_domain).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>
#include <vector>

#include "b200_session.hpp"
#include "dpd/cell_grid.hpp"
#include "dpd/morton.hpp"

namespace dpd {
namespace {

CellGrid grid_from_plan(const SimBox& box, const double* lo, const double* hi, const int32_t* dims,
                        const int32_t* coords, double cell_target, int sub_bits) {
    const dpdb_box b = b200::to_box(box);
    dpdb_grid_info info{};
    int32_t glo[3], ghi[3];
    b200::check(dpdb_grid_plan(&b, lo, hi, dims, coords, cell_target, sub_bits, &info, glo, ghi, nullptr),
                nullptr, "CellGrid::make");
    CellGrid g;
    for (int k = 0; k < 3; ++k) {
        g.ncell[k] = info.ncell[k];
        g.ncell_ext[k] = info.ncell_ext[k];
        g.ghost_lo[k] = glo[k];
        g.ghost_hi[k] = ghi[k];
        g.wrapmode[k] = info.wrapmode[k] != 0;
        g.cell_size[k] = info.cell_size[k];
        g.inv_cell[k] = info.inv_cell[k];
        g.slab_lo[k] = lo ? lo[k] : box.lo[k];
        g.slab_hi[k] = hi ? hi[k] : box.hi[k];
        g.origin[k] = info.origin[k];
    }
    g.sub_bits = sub_bits;
    g.bits_per_axis = info.bits_per_axis;
    g.n_local_cells = info.n_local_cells;
    g.n_total_cells = info.n_total_cells;
    g.rank_of_cell.assign(info.n_total_cells, 0u);
    b200::check(dpdb_grid_plan(&b, lo, hi, dims, coords, cell_target, sub_bits, &info, nullptr, nullptr,
                               g.rank_of_cell.data()),
                nullptr, "CellGrid::make");
    g.cell_of_rank.assign(info.n_total_cells, 0u);
    for (std::uint32_t c = 0; c < info.n_total_cells; ++c) g.cell_of_rank[g.rank_of_cell[c]] = c;
    return g;
}

// A cell target that reproduces grid's lattice in libdpdb's planner
// (ncell_k = floor(len_k / target)): just above the largest
// len_k / (ncell_k + 1), which lies below every len_k / ncell_k.
double target_of(const CellGrid& g) {
    double t = 0.0;
    for (int k = 0; k < 3; ++k)
        t = std::max(t, (g.slab_hi[k] - g.slab_lo[k]) / (g.ncell[k] + 1));
    return std::nextafter(t, 1e300);
}

// The device context holding `grid`'s lattice (single domain: the slab is the box).
dpdb_ctx* grid_context(const CellGrid& g, std::size_t n) {
    for (int k = 0; k < 3; ++k)
        if (g.ghost_lo[k] || g.ghost_hi[k])
            fail(ErrorCategory::config,
                 "B200 drop-in: grids with ghost layers run through the brick API (dpdb_create_domain)");
    SimBox box;
    for (int k = 0; k < 3; ++k) {
        box.lo[k] = g.slab_lo[k];
        box.hi[k] = g.slab_hi[k];
        box.periodic[k] = g.wrapmode[k];
        box.wall[k] = false;
    }
    b200::ContextKey key;
    key.box = b200::to_box(box);
    key.params = b200::to_params(b200::cutoff_params(target_of(g)));
    key.run = b200::run_config(0.0, 32, 1, g.sub_bits);
    key.capacity = std::max<std::size_t>(n, 1);
    dpdb_ctx* ctx = b200::context(key);
    dpdb_grid_info info{};
    b200::check(dpdb_grid(ctx, &info), ctx, "grid");
    for (int k = 0; k < 3; ++k)
        if (info.ncell[k] != g.ncell[k])
            fail(ErrorCategory::config, "B200 drop-in: grid lattice not reproducible on the device");
    return ctx;
}

int cell_index(double x, double lo, double inv, int n) {
    const int c = (int)std::floor((x - lo) * inv);
    return std::min(std::max(c, 0), n - 1);
}

}  // namespace

CellGrid CellGrid::make(const SimBox& box, double cell_target, int sub_bits) {
    return grid_from_plan(box, nullptr, nullptr, nullptr, nullptr, cell_target, sub_bits);
}

CellGrid CellGrid::make(const SimBox& box, const Vec3& slab_lo, const Vec3& slab_hi, const IVec3& dims,
                        const IVec3& my_coords, double cell_target, int sub_bits) {
    const double lo[3] = {slab_lo.x, slab_lo.y, slab_lo.z}, hi[3] = {slab_hi.x, slab_hi.y, slab_hi.z};
    const int32_t d[3] = {dims[0], dims[1], dims[2]}, c[3] = {my_coords[0], my_coords[1], my_coords[2]};
    return grid_from_plan(box, lo, hi, d, c, cell_target, sub_bits);
}

IVec3 CellGrid::local_cell_of(const Vec3& x) const {
    IVec3 c{};
    for (int k = 0; k < 3; ++k) {
        if (!(x[k] >= slab_lo[k] && x[k] < slab_hi[k]))
            fail(ErrorCategory::protocol,
                 "particle outside its domain slab (missed migration), axis " + std::to_string(k));
        c[k] = ghost_lo[k] + cell_index(x[k], slab_lo[k], inv_cell[k], ncell[k]);
    }
    return c;
}

IVec3 CellGrid::ghost_cell_of(const Vec3& x) const {
    IVec3 c{};
    for (int k = 0; k < 3; ++k) c[k] = cell_index(x[k], origin[k], inv_cell[k], ncell_ext[k]);
    return c;
}

std::uint32_t CellGrid::sub_code(const Vec3& x, const IVec3& cell) const {
    const int nsub = 1 << sub_bits;
    std::uint32_t s[3];
    for (int k = 0; k < 3; ++k) {
        const double corner = origin[k] + cell[k] * cell_size[k];
        s[k] = (std::uint32_t)std::min(std::max((int)std::floor((x[k] - corner) * inv_cell[k] * nsub), 0),
                                       nsub - 1);
    }
    return morton_encode(s[0], s[1], s[2], sub_bits);
}

int CellGrid::key_bits() const {
    int b = 0;
    while ((1ull << b) < n_total_cells) ++b;
    const int bits = b + 3 * sub_bits;
    if (bits > 32) fail(ErrorCategory::config, "cell grid: sort key exceeds 32 bits");
    return (bits + 3) & ~3;
}

void build_cell_list(CellGrid& grid, std::span<const std::uint32_t> ranks) {
    const std::uint32_t nc = grid.n_total_cells;
    grid.cell_start.assign((std::size_t)nc + 1, (std::uint32_t)ranks.size());
    std::uint32_t next = 0;  // first rank whose start is not set yet
    for (std::size_t i = 0; i < ranks.size(); ++i) {
        const std::uint32_t r = ranks[i];
        if (r >= nc) fail(ErrorCategory::config, "build_cell_list: cell rank out of range");
        if (r + 1 < next) fail(ErrorCategory::config, "build_cell_list: ranks are not sorted");
        for (; next <= r; ++next) grid.cell_start[next] = (std::uint32_t)i;
    }
}

std::vector<std::uint32_t> reorder_particles(ParticleStore& store, const CellGrid& grid, RadixSorter&,
                                             WorkerPool&) {
    const std::size_t n = store.n;
    std::vector<std::uint32_t> perm(n);
    if (!n) return perm;
    dpdb_ctx* ctx = grid_context(grid, n);
    b200::upload(ctx, store);
    const bool has_f = store.force[0].size() >= n;
    if (has_f)
        b200::check(dpdb_upload_forces(ctx, store.force[0].data(), store.force[1].data(), store.force[2].data()),
                    ctx, "upload_forces");
    b200::check(dpdb_reorder(ctx, perm.data()), ctx, "reorder_particles");
    const bool has_sp = store.species.size() >= n;
    std::vector<std::uint32_t> sig(n);
    b200::check(dpdb_download(ctx, store.coord[0].data(), store.coord[1].data(), store.coord[2].data(),
                              store.veloc[0].data(), store.veloc[1].data(), store.veloc[2].data(),
                              has_f ? store.force[0].data() : nullptr, has_f ? store.force[1].data() : nullptr,
                              has_f ? store.force[2].data() : nullptr, store.tag.data(),
                              has_sp ? store.species.data() : nullptr, nullptr),
                ctx, "download");
    // arrays the device does not carry back travel with the permutation
    auto carry = [&](std::vector<std::uint32_t>& a) {
        if (a.size() < n) return;
        std::vector<std::uint32_t> b(a.size());
        for (std::size_t i = 0; i < n; ++i) b[perm[i]] = a[i];
        a.swap(b);
    };
    carry(store.molecule);
    carry(store.signature);
    return perm;
}

std::vector<std::uint32_t> local_cell_ranks(const ParticleStore& store, const CellGrid& grid, WorkerPool&) {
    const std::size_t n = store.n;
    std::vector<std::uint32_t> keys(n);
    if (!n) return keys;
    dpdb_ctx* ctx = grid_context(grid, n);
    b200::upload(ctx, store);
    b200::check(dpdb_sort_keys(ctx, keys.data()), ctx, "local_cell_ranks");
    for (auto& k : keys) k >>= 3 * grid.sub_bits;
    return keys;
}

}  // namespace dpd
