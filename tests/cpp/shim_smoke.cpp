// Uses the C++ drop-in shim exactly like code written against the reference
// headers would (reorder_particles -> build_neighbor_table -> compute_forces
// -> verlet_step), then the device-resident loop.  Built by tests/test_abi.py
// (link check, CPU) and run by tests/test_gpu_shim.py (B200).
#include <cstdio>
#include <random>

#include "dpd_b200.hpp"

using namespace dpd::b200;

int main() {
    SimBox box;
    box.hi = {8.0, 8.0, 8.0};
    const auto params = PairParams::make(1, {25.0}, {4.5}, 1.0, 1.0, 1.0, 0.01);
    RunConfig run;
    ParticleStore st;
    const std::size_t n = 1536;
    st.resize(n);
    std::mt19937_64 g(7);
    std::uniform_real_distribution<double> u(0.0, 8.0);
    std::normal_distribution<double> nv(0.0, 1.0);
    for (std::size_t i = 0; i < n; ++i) {
        for (int k = 0; k < 3; ++k) {
            st.coord[k][i] = u(g);
            st.veloc[k][i] = nv(g);
        }
        st.tag[i] = (std::uint32_t)(i + 1);
    }
    try {
        Device dev(box, params, run, n);
        const auto perm = reorder_particles(st, dev);
        NeighborTable t = build_neighbor_table(st, dev, run.max_neighbors);
        std::size_t pairs = 0;
        for (std::uint32_t i = 0; i < t.n_rows; ++i) pairs += t.core_count[i];
        join_core_skin(t, dev);
        compute_forces(st, dev, 0);
        double net[3] = {0, 0, 0};
        for (std::size_t i = 0; i < n; ++i)
            for (int k = 0; k < 3; ++k) net[k] += st.force[k][i];
        verlet_step(st, dev, StepPhase::Phase1);
        dev.upload(st);
        dev.setup();
        dev.step(20);
        const dpdb_thermo th = dev.thermo();
        std::printf("shim ok n=%zu perm0=%u core_pairs=%zu joined=%d net_force=(%.2e,%.2e,%.2e) kbt=%.4f "
                    "fastlog(2^31)=%.17g\n",
                    n, perm[0], pairs, (int)t.joined, net[0], net[1], net[2], th.kbt,
                    fastlog(2147483648u));
        return (th.kbt > 0 && t.joined) ? 0 : 1;
    } catch (const Error& e) {
        std::printf("shim error [%d]: %s\n", e.exit_code(), e.what());
        return e.exit_code();
    }
}
