// ref_slots.cpp -- TEST INFRASTRUCTURE.  The reference-side implementation of
// the slots the reference does not ship (src/neighbor_table.cpp,
// src/forces.cpp, src/integrate.cpp; CMakeLists.txt:21-23), on the
// reference's own types, delegating to the C restatement in dpd_oracle.c.
// Linked with the reference's five shipped sources into the REF build of the
// drop-in caller (tests/cpp/ref_caller.cpp) so the same unchanged caller runs
// once on the reference path and once on the B200 drop-in (dropin/), and
// tests/test_gpu_dropin.py compares the two.  Never part of the product.
#include <vector>

#include "dpd/forces.hpp"
#include "dpd/integrate.hpp"
#include "dpd/neighbor_table.hpp"
#include "dpd/stencil.hpp"

extern "C" {
#include "dpd_oracle.h"
}

namespace dpd {
namespace {
orc_box obox(const SimBox& b) {
    orc_box o{};
    for (int k = 0; k < 3; ++k) {
        o.lo[k] = b.lo[k];
        o.hi[k] = b.hi[k];
        o.periodic[k] = b.periodic[k];
        o.wall[k] = b.wall[k];
    }
    return o;
}
void ocheck(int rc) {
    if (rc) throw Error(static_cast<ErrorCategory>(rc), orc_last_error());
}
}  // namespace

NeighborTable build_neighbor_table(const ParticleStore& store, const CellGrid& grid, const FineStencil&,
                                   const SimBox& box, double r_c, double skin, std::uint32_t maxn,
                                   WorkerPool& pool) {
    orc_grid g{};
    for (int k = 0; k < 3; ++k) {
        g.ncell[k] = grid.ncell[k];
        g.ncell_ext[k] = grid.ncell_ext[k];
        g.ghost_lo[k] = grid.ghost_lo[k];
        g.ghost_hi[k] = grid.ghost_hi[k];
        g.wrapmode[k] = grid.wrapmode[k];
        g.cell_size[k] = grid.cell_size[k];
        g.inv_cell[k] = grid.inv_cell[k];
        g.slab_lo[k] = grid.slab_lo[k];
        g.slab_hi[k] = grid.slab_hi[k];
        g.origin[k] = grid.origin[k];
    }
    g.sub_bits = grid.sub_bits;
    g.bits_per_axis = grid.bits_per_axis;
    g.n_local_cells = grid.n_local_cells;
    g.n_total_cells = grid.n_total_cells;
    const CoarseStencil cs = build_coarse_stencil(grid, box);
    const orc_box b = obox(box);
    NeighborTable t;
    t.n_rows = (std::uint32_t)store.n;
    t.max_neighbors = maxn;
    t.n_rows_pad = (t.n_rows + 31u) & ~31u;
    t.entries.assign((std::size_t)std::max(t.n_rows_pad, 32u) * maxn, 0u);
    t.core_count.assign(std::max<std::size_t>(store.n, 1), 0);
    t.skin_count.assign(std::max<std::size_t>(store.n, 1), 0);
    ocheck(orc_build_neighbor_table(&g, &b, grid.cell_start.data(), cs.offsets.data(), cs.cells.data(), store.n,
                                    store.n, store.coord[0].data(), store.coord[1].data(), store.coord[2].data(),
                                    store.tag.data(), r_c, skin, maxn, t.entries.data(), t.core_count.data(),
                                    t.skin_count.data(), (int)pool.size()));
    t.core_count.resize(store.n);
    t.skin_count.resize(store.n);
    t.entries.resize((std::size_t)t.n_rows_pad * maxn);
    return t;
}

void join_core_skin(NeighborTable& t, WorkerPool&) {
    if (t.joined) return;
    orc_join_core_skin(t.n_rows, t.max_neighbors, t.tiled, t.entries.data(), t.core_count.data(),
                       t.skin_count.data());
    t.joined = true;
}

void tile_transpose(NeighborTable& t, WorkerPool&) {
    orc_tile_transpose(t.n_rows_pad, t.max_neighbors, t.entries.data());
    t.tiled = !t.tiled;
}

void compute_forces(ParticleStore& s, const NeighborTable& t, const PairParams& p, const BondTopology& bonds,
                    const PairRandomState& state, const SimBox& box) {
    const std::size_t n = s.n;
    orc_params op{};
    ocheck(orc_params_make((int32_t)p.n_species, p.a.data(), p.gamma.data(), p.kbt, p.s, p.r_c, p.dt, &op));
    const orc_box b = obox(box);
    std::vector<std::uint32_t> sig(n);
    orc_signatures(n, s.tag.data(), s.veloc[0].data(), s.veloc[1].data(), s.veloc[2].data(), sig.data());
    for (int k = 0; k < 3; ++k) s.force[k].assign(n, 0.0);
    const bool sp = s.species.size() >= n && p.n_species > 1;
    ocheck(orc_compute_forces(&op, &b, n, s.coord[0].data(), s.coord[1].data(), s.coord[2].data(),
                              s.veloc[0].data(), s.veloc[1].data(), s.veloc[2].data(), s.tag.data(),
                              sp ? s.species.data() : nullptr, sig.data(), state.step_mix, t.max_neighbors,
                              t.tiled, t.joined, t.entries.data(), t.core_count.data(), t.skin_count.data(),
                              s.force[0].data(), s.force[1].data(), s.force[2].data(), 4));
    if (bonds.bonds.empty()) return;
    std::uint32_t mt = 0;
    for (std::size_t i = 0; i < n; ++i) mt = std::max(mt, s.tag[i]);
    std::vector<std::uint32_t> iot((std::size_t)mt + 1, 0xFFFFFFFFu);
    for (std::size_t i = 0; i < n; ++i) iot[s.tag[i]] = (std::uint32_t)i;
    std::vector<orc_bond> ob;
    for (const Bond& bd : bonds.bonds) ob.push_back({bd.tag_i, bd.tag_j, bd.k, bd.r0});
    ocheck(orc_bond_forces(&b, ob.size(), ob.data(), iot.size(), iot.data(), s.coord[0].data(), s.coord[1].data(),
                           s.coord[2].data(), s.force[0].data(), s.force[1].data(), s.force[2].data()));
}

void verlet_step(ParticleStore& s, const PairParams& p, StepPhase phase, const SimBox& box, WallMode) {
    const orc_box b = obox(box);
    if (phase == StepPhase::Phase1)
        ocheck(orc_verlet_phase1(&b, p.dt, s.n, s.coord[0].data(), s.coord[1].data(), s.coord[2].data(),
                                 s.veloc[0].data(), s.veloc[1].data(), s.veloc[2].data(), s.force[0].data(),
                                 s.force[1].data(), s.force[2].data(), s.tag.data()));
    else
        orc_verlet_phase2(p.dt, s.n, s.veloc[0].data(), s.veloc[1].data(), s.veloc[2].data(), s.force[0].data(),
                          s.force[1].data(), s.force[2].data());
}

}  // namespace dpd
