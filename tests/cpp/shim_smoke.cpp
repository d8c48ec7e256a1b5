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
        std::size_t pairs = 0, entries = 0;
        for (std::uint32_t i = 0; i < t.n_rows; ++i) {
            pairs += t.core_count[i];
            entries += t.core_count[i] + t.skin_count[i];
        }
        {  // dump_neighbor_csv (inc/neighbor_table.hpp:57-59): header + one line per entry
            std::FILE* f = std::tmpfile();
            dump_neighbor_csv(t, st, box, {true, true, true}, f);
            std::rewind(f);
            std::size_t lines = 0;
            for (int c; (c = std::fgetc(f)) != EOF;) lines += c == '\n';
            std::fclose(f);
            if (lines != entries + 1) {
                std::printf("dump_neighbor_csv: %zu lines for %zu entries\n", lines, entries);
                return 3;
            }
        }
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
        // per-step thermo lines, observables, device init (the reference's run() path)
        const auto lines = dev.step_thermo(10);
        dev.profile_reset(8, 2, 0);
        dev.profile_sample();
        std::vector<double> sv(8);
        std::vector<std::uint64_t> cnt(8);
        const std::int64_t ns = dev.profile(sv, cnt);
        std::uint64_t tot = 0;
        for (auto c : cnt) tot += c;
        const auto hist = dev.rdf_counts(13, 1.3);
        Device dev2(box, params, run, n);
        dev2.init_random(n, 1.0, 7);
        dev2.setup();
        dev2.step(5);
        if (lines.size() != 10 || lines.back().step != dev.current_step() || ns != 1 || tot != n ||
            hist[10] == 0 || dev2.current_step() != 5) {
            std::printf("shim observables wrong\n");
            return 2;
        }
        write_thermo_csv(stdout, {lines.back()}, 0.01);
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
