// integrate.cpp (B200 drop-in) -- the reference's missing src/integrate.cpp
// slot (CMakeLists.txt:23): verlet_step of SPEC.md:488-514 over libdpdb
// (k_integrate: fp64 state, each half kick its own rounding, periodic wrap /
// bounce-forward walls in the same pass).  The device holds forces in fp32:
// a store whose forces are fp32 values (compute_forces's output) steps
// bit-identically to the fp64 reference formula.
#include "b200_session.hpp"
#include "dpd/integrate.hpp"

namespace dpd {

void verlet_step(ParticleStore& store, const PairParams& params, StepPhase phase, const SimBox& box,
                 WallMode wall_mode) {
    const std::size_t n = store.n;
    if (!n) return;
    if (store.force[0].size() < n) fail(ErrorCategory::config, "verlet_step: forces not computed");
    b200::ContextKey key;
    key.box = b200::to_box(box);
    key.params = b200::to_params(params);
    key.run = b200::run_config(0.0, 32, 1, 2);
    key.run.wall_mode = wall_mode == WallMode::bounce_back ? 1 : 0;
    key.capacity = n;
    dpdb_ctx* ctx = b200::context(key);
    b200::upload(ctx, store);
    b200::check(dpdb_upload_forces(ctx, store.force[0].data(), store.force[1].data(), store.force[2].data()),
                ctx, "verlet_step");
    const bool p1 = phase == StepPhase::Phase1;
    b200::check(p1 ? dpdb_verlet_phase1(ctx) : dpdb_verlet_phase2(ctx), ctx, "verlet_step");
    b200::check(dpdb_download(ctx, p1 ? store.coord[0].data() : nullptr, p1 ? store.coord[1].data() : nullptr,
                              p1 ? store.coord[2].data() : nullptr, store.veloc[0].data(), store.veloc[1].data(),
                              store.veloc[2].data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr),
                ctx, "verlet_step");
}

}  // namespace dpd
