// forces.cpp (B200 drop-in) -- the reference's missing src/forces.cpp slot
// (CMakeLists.txt:22): compute_forces of SPEC.md:434-451 over libdpdb.
//
// The caller's table is imported as is (dpdb_set_neighbors) and evaluated by
// the device pair kernel (k_force: per-step |r| <= r_c re-check, C + D + R
// with the signature/TEA pair random numbers and fp32 Box-Muller, 2^-18
// fixed-point accumulation -- order-free, so the row order is immaterial and
// Newton's third law holds exactly); harmonic bonds are added per particle
// (k_bonds).  Forces come back as the device's fp32 values in fp64 storage:
// within 1e-5 of the fp64 reference per particle (tests/test_gpu_dropin.py).
#include <algorithm>
#include <vector>

#include "b200_session.hpp"
#include "dpd/forces.hpp"

namespace dpd {

void compute_forces(ParticleStore& store, const NeighborTable& table, const PairParams& params,
                    const BondTopology& bonds, const PairRandomState& state, const SimBox& box) {
    const std::size_t n = store.n;
    if (table.n_rows != n) fail(ErrorCategory::config, "compute_forces: table rows differ from the store");
    for (int k = 0; k < 3; ++k) store.force[k].assign(n, 0.0);
    if (!n) return;
    b200::ContextKey key;
    key.box = b200::to_box(box);
    key.params = b200::to_params(params);
    key.run = b200::run_config(0.0, table.max_neighbors, state.global_seed, 2);
    key.capacity = n;
    dpdb_ctx* ctx = b200::context(key);
    b200::upload(ctx, store);
    const std::size_t nb = bonds.bonds.size();
    std::vector<std::uint32_t> ti(nb), tj(nb);
    std::vector<double> kk(nb), r0(nb);
    for (std::size_t b = 0; b < nb; ++b) {
        ti[b] = bonds.bonds[b].tag_i;
        tj[b] = bonds.bonds[b].tag_j;
        kk[b] = bonds.bonds[b].k;
        r0[b] = bonds.bonds[b].r0;
    }
    b200::check(dpdb_set_bonds(ctx, nb, ti.data(), tj.data(), kk.data(), r0.data()), ctx, "compute_forces");
    b200::check(dpdb_set_neighbors(ctx, table.entries.data(), table.core_count.data(), table.skin_count.data(),
                                   table.tiled, table.joined),
                ctx, "compute_forces");
    b200::check(dpdb_compute_forces(ctx, state.step), ctx, "compute_forces");
    b200::check(dpdb_download(ctx, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, store.force[0].data(),
                              store.force[1].data(), store.force[2].data(), nullptr, nullptr, nullptr),
                ctx, "compute_forces");
}

}  // namespace dpd
