// dpd_b200.hpp -- C++ drop-in shim over libdpdb.so (include/dpdb.h).
//
// Re-exposes the reference's C++ hot-path API (same names, argument meaning
// and error behaviour) on top of the B200 engine, so code written against
// /root/reference/proj/include/dpd/*.hpp switches by changing the include
// and passing a dpd::b200::Device where the reference passed a WorkerPool:
//
//   reference (namespace dpd)                         this shim (namespace dpd::b200)
//   ---------------------------------------------------------------------------------
//   Error / ErrorCategory      inc/error.hpp:8-28      Error / ErrorCategory (same codes)
//   SimBox                     inc/core.hpp:15-25      SimBox
//   ParticleStore              inc/core.hpp:29-47      ParticleStore
//   PairParams::make           inc/core.hpp:51-68      PairParams::make
//   RunConfig                  inc/core.hpp:83-109     RunConfig (hot-path fields)
//   BondTopology               inc/core.hpp:70-81      BondTopology
//   RadixSorter::sort          inc/radix_sort.hpp:19   radix_sort(keys, vals, bits, dev)
//   reorder_particles          inc/cell_grid.hpp:78    reorder_particles(store, dev)
//   build_cell_list            inc/cell_grid.hpp:74    cell_start(dev)  (built by reorder)
//   build_coarse_stencil       inc/stencil.hpp:24      coarse_stencil(dev)
//   expand_fine_stencil        inc/stencil.hpp:39      fine_stencil(dev)
//   build_neighbor_table       inc/neighbor_table.hpp:45  build_neighbor_table(store, dev)
//   join_core_skin             inc/neighbor_table.hpp:51  join_core_skin(table, dev)
//   tile_transpose             inc/neighbor_table.hpp:55  tile_transpose(table, dev)
//   compute_forces             SPEC.md:434             compute_forces(store, dev, step)
//   verlet_step                SPEC.md:488             verlet_step(store, dev, phase)
//   compute_temperature        inc/core.hpp:116        compute_temperature(dev)
//   tea_hash / make_signature / pair_uniforms / gaussian / fastlog /
//   fastcos2pi / fastpow       inc/rng.hpp, inc/fastmath.hpp   same names (device-evaluated)
//
// Header-only; link with -ldpdb (paper_1311_0402_b200/libdpdb.so).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dpdb.h"

namespace dpd::b200 {

enum class ErrorCategory { config = 1, physics = 2, protocol = 3, io = 4, device = 5 };

class Error : public std::runtime_error {
public:
    Error(ErrorCategory cat, const std::string& what) : std::runtime_error(what), category_(cat) {}
    ErrorCategory category() const { return category_; }
    int exit_code() const { return static_cast<int>(category_); }

private:
    ErrorCategory category_;
};

inline void check(int rc, const dpdb_ctx* ctx = nullptr) {
    if (rc) throw Error(static_cast<ErrorCategory>(rc), dpdb_last_error(ctx));
}

struct Vec3 {
    double x = 0, y = 0, z = 0;
};

struct SimBox {
    Vec3 lo{0, 0, 0};
    Vec3 hi{1, 1, 1};
    std::array<bool, 3> periodic{true, true, true};
    std::array<bool, 3> wall{false, false, false};
    double length(int k) const { return (&hi.x)[k] - (&lo.x)[k]; }
    dpdb_box c() const {
        dpdb_box b{};
        for (int k = 0; k < 3; ++k) {
            b.lo[k] = (&lo.x)[k];
            b.hi[k] = (&hi.x)[k];
            b.periodic[k] = periodic[k];
            b.wall[k] = wall[k];
        }
        return b;
    }
};

struct ParticleStore {
    std::size_t n = 0;
    std::array<std::vector<double>, 3> coord, veloc, force;
    std::vector<std::uint32_t> tag;
    std::vector<std::uint8_t> species;
    std::vector<std::uint32_t> signature;
    std::vector<std::uint32_t> molecule;
    void resize(std::size_t m) {
        n = m;
        for (int k = 0; k < 3; ++k) {
            coord[k].resize(m);
            veloc[k].resize(m);
            force[k].resize(m);
        }
        tag.resize(m);
        species.resize(m);
        signature.resize(m);
        molecule.resize(m);
    }
};

struct PairParams {
    std::size_t n_species = 1;
    std::vector<double> a, gamma, sigma;
    double s = 1.0, r_c = 1.0, kbt = 1.0, dt = 0.01;
    static PairParams make(std::size_t n_species, std::vector<double> a, std::vector<double> gamma,
                           double kbt, double s, double r_c, double dt) {
        if (r_c <= 0) throw Error(ErrorCategory::config, "pair params: r_c must be positive");
        if (s <= 0) throw Error(ErrorCategory::config, "pair params: weight exponent s must be positive");
        if (a.size() != n_species * n_species || gamma.size() != n_species * n_species)
            throw Error(ErrorCategory::config, "pair params: matrix size mismatch");
        PairParams p;
        p.n_species = n_species;
        p.sigma.resize(gamma.size());
        for (std::size_t q = 0; q < gamma.size(); ++q) p.sigma[q] = std::sqrt(2.0 * gamma[q] * kbt);
        p.a = std::move(a);
        p.gamma = std::move(gamma);
        p.kbt = kbt;
        p.s = s;
        p.r_c = r_c;
        p.dt = dt;
        return p;
    }
    dpdb_params c() const {
        dpdb_params p{};
        p.n_species = (int32_t)n_species;
        for (std::size_t q = 0; q < a.size() && q < 16; ++q) {
            p.a[q] = a[q];
            p.gamma[q] = gamma[q];
        }
        p.kbt = kbt;
        p.s = s;
        p.r_c = r_c;
        p.dt = dt;
        return p;
    }
};

struct Bond {
    std::uint32_t tag_i, tag_j;
    double k, r0;
    std::uint8_t style = 0;  // 0 harmonic, 1 FENE with R0 = r0 (unpinned)
};
struct Angle {  // harmonic angle around the middle tag_b (unpinned)
    std::uint32_t tag_a, tag_b, tag_c;
    double k, theta0;
};
struct BondTopology {
    std::vector<Bond> bonds;
    std::vector<Angle> angles;
};

struct RunConfig {
    int rebuild_every = 10;
    double skin = 0.3;
    double body_force = 0.0;
    int drive_axis = 2;
    int partition_axis = 0;
    std::uint32_t seed = 1;
    std::uint32_t max_neighbors = 128;
    int sub_bits = 2;
    int wall_mode = 0;  // 0 specular bounce-forward, 1 bounce-back
    dpdb_run c() const {
        dpdb_run r{};
        r.rebuild_every = rebuild_every;
        r.skin = skin;
        r.body_force = body_force;
        r.drive_axis = drive_axis;
        r.partition_axis = partition_axis;
        r.seed = seed;
        r.max_neighbors = max_neighbors;
        r.sub_bits = sub_bits;
        r.wall_mode = wall_mode;
        return r;
    }
};

// NeighborTable, inc/neighbor_table.hpp:18-40 (host copy; same accessors)
struct NeighborTable {
    std::uint32_t n_rows = 0, max_neighbors = 0, n_rows_pad = 0;
    bool tiled = false, joined = false;
    std::vector<std::uint32_t> entries;
    std::vector<std::uint16_t> core_count, skin_count;
    std::size_t raw_index(std::uint32_t i, std::uint32_t k) const {
        if (!tiled) return std::size_t(i) * max_neighbors + k;
        return std::size_t((i & ~31u) + (k & 31u)) * max_neighbors + (k & ~31u) + (i & 31u);
    }
    std::uint32_t entry(std::uint32_t i, std::uint32_t k) const { return entries[raw_index(i, k)]; }
    std::uint32_t core_at(std::uint32_t i, std::uint32_t k) const { return entry(i, k); }
    std::uint32_t skin_at(std::uint32_t i, std::uint32_t k) const {
        return joined ? entry(i, core_count[i] + k) : entry(i, max_neighbors - 1 - k);
    }
};

// The device side of one domain (replaces the reference's WorkerPool&
// argument): owns the dpdb context, the resident SoA state and the table.
class Device {
public:
    Device(const SimBox& box, const PairParams& p, const RunConfig& run, std::size_t capacity,
           int device = 0) {
        const dpdb_box b = box.c();
        const dpdb_params pp = p.c();
        const dpdb_run r = run.c();
        check(dpdb_create(device, &b, &pp, &r, capacity, &ctx_));
    }
    ~Device() { dpdb_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    dpdb_ctx* get() const { return ctx_; }
    void ck(int rc) const { check(rc, ctx_); }

    void upload(const ParticleStore& s) {
        ck(dpdb_upload(ctx_, s.n, s.coord[0].data(), s.coord[1].data(), s.coord[2].data(),
                       s.veloc[0].data(), s.veloc[1].data(), s.veloc[2].data(), s.tag.data(),
                       s.species.empty() ? nullptr : s.species.data(),
                       s.molecule.empty() ? nullptr : s.molecule.data()));
    }
    void download(ParticleStore& s) {
        std::size_t n = 0;
        ck(dpdb_size(ctx_, &n));
        s.resize(n);
        ck(dpdb_download(ctx_, s.coord[0].data(), s.coord[1].data(), s.coord[2].data(),
                         s.veloc[0].data(), s.veloc[1].data(), s.veloc[2].data(),
                         s.force[0].data(), s.force[1].data(), s.force[2].data(), s.tag.data(),
                         s.species.data(), s.signature.data()));
    }
    dpdb_grid_info grid() const {
        dpdb_grid_info g{};
        ck(dpdb_grid(ctx_, &g));
        return g;
    }
    void setup() { ck(dpdb_setup(ctx_)); }
    void step(std::int64_t nsteps) { ck(dpdb_step(ctx_, nsteps)); }
    // nsteps steps with every step's thermo line (dpdb_step_thermo)
    std::vector<dpdb_thermo> step_thermo(std::int64_t nsteps) {
        std::vector<dpdb_thermo> out((size_t)nsteps);
        ck(dpdb_step_thermo(ctx_, nsteps, out.data()));
        return out;
    }
    dpdb_thermo thermo() {
        dpdb_thermo t{};
        ck(dpdb_thermo_get(ctx_, &t));
        return t;
    }
    // init_random on the device; chains ahead of the solvent
    void init_random(std::size_t n, double kbt, std::uint32_t seed, std::uint32_t n_chains = 0,
                     const std::vector<std::uint8_t>& chain_species = {}, std::uint8_t solvent = 0,
                     double r0 = 0.38, double bond_k = 80.0) {
        ck(dpdb_init_random(ctx_, n, kbt, seed, n_chains, (std::uint32_t)chain_species.size(),
                            chain_species.empty() ? nullptr : chain_species.data(), solvent, r0,
                            bond_k));
    }
    // restart entry: setup at `step`, keeping uploaded forces
    void setup_at(std::int64_t step, bool keep_forces) { ck(dpdb_setup_at(ctx_, step, keep_forces)); }
    void upload_forces(const ParticleStore& s) {
        ck(dpdb_upload_forces(ctx_, s.force[0].data(), s.force[1].data(), s.force[2].data()));
    }
    // bonded topology (inc/core.hpp:70-81; FENE and angles beyond the reference)
    void set_topology(const BondTopology& t) {
        std::vector<std::uint32_t> bi, bj, aa, ab, ac;
        std::vector<double> bk, br, ak, at;
        std::vector<std::uint8_t> bs;
        for (const auto& b : t.bonds) {
            bi.push_back(b.tag_i);
            bj.push_back(b.tag_j);
            bk.push_back(b.k);
            br.push_back(b.r0);
            bs.push_back(b.style);
        }
        for (const auto& q : t.angles) {
            aa.push_back(q.tag_a);
            ab.push_back(q.tag_b);
            ac.push_back(q.tag_c);
            ak.push_back(q.k);
            at.push_back(q.theta0);
        }
        ck(dpdb_set_bonds_styled(ctx_, bi.size(), bi.data(), bj.data(), bk.data(), br.data(), bs.data()));
        ck(dpdb_set_angles(ctx_, aa.size(), aa.data(), ab.data(), ac.data(), ak.data(), at.data()));
    }
    // velocity_profile accumulation
    void profile_reset(std::uint32_t bins, int bin_axis, int vel_axis) {
        ck(dpdb_profile_reset(ctx_, bins, bin_axis, vel_axis));
    }
    void profile_sample() { ck(dpdb_profile_sample(ctx_)); }
    // per-bin (sum of velocities, count) and the sample count
    std::int64_t profile(std::vector<double>& sum_v, std::vector<std::uint64_t>& count) {
        std::int64_t ns = 0;
        ck(dpdb_profile_get(ctx_, sum_v.data(), count.data(), &ns));
        return ns;
    }
    // pair-distance histogram of the current table (every pair once)
    std::vector<std::uint64_t> rdf_counts(std::uint32_t bins, double rmax) {
        std::vector<std::uint64_t> h(bins);
        ck(dpdb_rdf(ctx_, bins, rmax, h.data()));
        return h;
    }
    std::int64_t current_step() const { return dpdb_current_step(ctx_); }

private:
    dpdb_ctx* ctx_ = nullptr;
};

// ------------------------------------------------ reference entry points
// reorder_particles (inc/cell_grid.hpp:78-79): permutes the store, returns old -> new
inline std::vector<std::uint32_t> reorder_particles(ParticleStore& store, Device& dev) {
    dev.upload(store);
    std::vector<std::uint32_t> perm(store.n);
    dev.ck(dpdb_reorder(dev.get(), perm.data()));
    dev.download(store);
    return perm;
}

// cell_start of the last reorder (build_cell_list, inc/cell_grid.hpp:74)
inline std::vector<std::uint32_t> cell_start(Device& dev) {
    std::vector<std::uint32_t> cs(dev.grid().n_total_cells + 1);
    dev.ck(dpdb_cell_start(dev.get(), cs.data()));
    return cs;
}

inline std::pair<std::vector<std::uint32_t>, std::vector<std::uint32_t>> coarse_stencil(Device& dev) {
    std::vector<std::uint32_t> off(dev.grid().n_local_cells + 1);
    dev.ck(dpdb_coarse_stencil(dev.get(), off.data(), nullptr));
    std::vector<std::uint32_t> cells(off.back());
    dev.ck(dpdb_coarse_stencil(dev.get(), off.data(), cells.data()));
    return {off, cells};
}

inline std::pair<std::vector<std::uint32_t>, std::vector<std::uint32_t>> fine_stencil(Device& dev) {
    std::vector<std::uint32_t> off(dev.grid().n_local_cells + 1);
    dev.ck(dpdb_fine_stencil(dev.get(), off.data(), nullptr));
    std::vector<std::uint32_t> idx(off.back());
    dev.ck(dpdb_fine_stencil(dev.get(), off.data(), idx.data()));
    return {off, idx};
}

// build_neighbor_table (inc/neighbor_table.hpp:45-47) on a store that
// reorder_particles already sorted: re-deriving the cell list of a sorted
// store is the identity permutation (the sort is stable).
inline NeighborTable build_neighbor_table(const ParticleStore& store, Device& dev,
                                          std::uint32_t max_neighbors) {
    dev.upload(store);
    dev.ck(dpdb_reorder(dev.get(), nullptr));
    dev.ck(dpdb_build_neighbors(dev.get()));
    NeighborTable t;
    std::size_t n = 0;
    dev.ck(dpdb_size(dev.get(), &n));
    t.n_rows = (std::uint32_t)n;
    t.max_neighbors = max_neighbors;
    t.n_rows_pad = (std::uint32_t)((n + 31) & ~std::size_t(31));
    t.entries.assign(std::size_t(t.n_rows_pad) * max_neighbors, 0);
    t.core_count.resize(n);
    t.skin_count.resize(n);
    int32_t tiled = 0, joined = 0;
    dev.ck(dpdb_get_neighbors(dev.get(), t.entries.data(), t.core_count.data(), t.skin_count.data(),
                              &tiled, &joined));
    t.tiled = tiled;
    t.joined = joined;
    return t;
}

// join_core_skin / tile_transpose (inc/neighbor_table.hpp:51,55) on the device table
inline void join_core_skin(NeighborTable& t, Device& dev) {
    dev.ck(dpdb_join_core_skin(dev.get()));
    int32_t tiled = 0, joined = 0;
    dev.ck(dpdb_get_neighbors(dev.get(), t.entries.data(), t.core_count.data(), t.skin_count.data(),
                              &tiled, &joined));
    t.tiled = tiled;
    t.joined = joined;
}
inline void tile_transpose(NeighborTable& t, Device& dev) {
    dev.ck(dpdb_tile_transpose(dev.get()));
    int32_t tiled = 0, joined = 0;
    dev.ck(dpdb_get_neighbors(dev.get(), t.entries.data(), t.core_count.data(), t.skin_count.data(),
                              &tiled, &joined));
    t.tiled = tiled;
    t.joined = joined;
}

// compute_forces + bonds + body force for PairRandomState::at(seed, step)
inline void compute_forces(ParticleStore& store, Device& dev, std::uint32_t step) {
    dev.ck(dpdb_compute_forces(dev.get(), step));
    dev.download(store);
}

enum class StepPhase { Phase1, Phase2 };
// verlet_step on the device-resident state
inline void verlet_step(ParticleStore& store, Device& dev, StepPhase phase) {
    dev.ck(phase == StepPhase::Phase1 ? dpdb_verlet_phase1(dev.get()) : dpdb_verlet_phase2(dev.get()));
    dev.download(store);
}

inline double compute_temperature(Device& dev) { return dev.thermo().kbt; }

// RadixSorter::sort contract (inc/radix_sort.hpp:11-27) on device 0
inline void radix_sort(std::vector<std::uint32_t>& keys, std::vector<std::uint32_t>& vals,
                       int bit_length, int device = 0) {
    if (keys.size() != vals.size())
        throw Error(ErrorCategory::config, "radix sort: keys/values length mismatch");
    check(dpdb_radix_sort(device, keys.data(), vals.data(), keys.size(), bit_length));
}

// ---------------------------------------- RNG / fastmath (device-evaluated)
struct TeaPair {
    std::uint32_t v0, v1;
};
inline TeaPair tea_hash(int rounds, std::uint32_t v0, std::uint32_t v1, int device = 0) {
    std::uint32_t out[2];
    check(dpdb_eval(device, DPDB_OP_TEA_HASH, 1, &v0, &v1, (std::uint32_t)rounds, out));
    return {out[0], out[1]};
}
inline std::uint32_t make_signature(std::uint32_t tag, const Vec3& v, int device = 0) {
    std::uint32_t out;
    const double vv[3] = {v.x, v.y, v.z};
    check(dpdb_eval(device, DPDB_OP_SIGNATURE, 1, &tag, vv, 0, &out));
    return out;
}
struct PairRandomState {
    std::uint32_t global_seed = 1, step = 0, step_mix = 0;
    static PairRandomState at(std::uint32_t seed, std::uint32_t step, int device = 0) {
        std::uint32_t mix;
        check(dpdb_eval(device, DPDB_OP_STEP_MIX, 1, &seed, &step, 0, &mix));
        return {seed, step, mix};
    }
};
inline TeaPair pair_uniforms(std::uint32_t sig_i, std::uint32_t sig_j, std::uint32_t tag_i,
                             std::uint32_t tag_j, const PairRandomState& st, int device = 0) {
    const std::uint32_t s[2] = {sig_i, sig_j}, t[2] = {tag_i, tag_j};
    std::uint32_t out[2];
    check(dpdb_eval(device, DPDB_OP_PAIR_UNIFORMS, 1, s, t, st.step_mix, out));
    return {out[0], out[1]};
}
inline double gaussian(std::uint32_t ua, std::uint32_t ub, int device = 0) {
    double out;
    check(dpdb_eval(device, DPDB_OP_GAUSSIAN64, 1, &ua, &ub, 0, &out));
    return out;
}
inline double fastlog(std::uint32_t v, int device = 0) {
    double out;
    check(dpdb_eval(device, DPDB_OP_FASTLOG, 1, &v, nullptr, 0, &out));
    return out;
}
inline double fastcos2pi(std::uint32_t v, int device = 0) {
    double out;
    check(dpdb_eval(device, DPDB_OP_FASTCOS2PI, 1, &v, nullptr, 0, &out));
    return out;
}
inline double fastpow(double a, double b, int device = 0) {
    double out;
    check(dpdb_eval(device, DPDB_OP_FASTPOW, 1, &a, &b, 0, &out));
    return out;
}

// ------------------------------------------------ observables and outputs
// (same definitions as paper_1311_0402_b200/observables.py, io.py)

// estimate_viscosity: least squares u(z) = (g rho / (2 mu)) z (d - z)
inline double estimate_viscosity(const std::vector<double>& z, const std::vector<double>& u, double g,
                                 double rho, double d) {
    double pu = 0, pp = 0;
    for (std::size_t k = 0; k < z.size(); ++k) {
        if (!(u[k] == u[k])) continue;  // empty bin (nan)
        const double phi = z[k] * (d - z[k]);
        pu += phi * u[k];
        pp += phi * phi;
    }
    return g * rho / (2.0 * (pu / pp));
}

// analytic_transient_profile (Eq. 9), n_terms terms of the series
inline double analytic_transient_profile(double z, double t, double F, double d, double nu,
                                         long n_terms = 200000) {
    const double pi = 3.14159265358979323846;
    double u = F * d * d / (8.0 * nu) * (1.0 - (2.0 * z / d) * (2.0 * z / d));
    for (long n = 0; n < n_terms; ++n) {
        const double k = 2.0 * n + 1.0;
        const double term = 4.0 * F * d * d / (nu * pi * pi * pi * k * k * k) * std::cos(k * pi * z / d) *
                            std::exp(-k * k * pi * pi * nu * t / (d * d));
        u -= (n % 2 ? -1.0 : 1.0) * term;
    }
    return u;
}

// XYZ frame: count line, comment line, "name x y z" per particle
inline void write_xyz(std::FILE* f, const ParticleStore& s, const char* comment = "",
                      const char* names = "SABC") {
    std::fprintf(f, "%zu\n%s\n", s.n, comment);
    for (std::size_t i = 0; i < s.n; ++i)
        std::fprintf(f, "%c %.10g %.10g %.10g\n", names[s.species.empty() ? 0 : s.species[i]],
                     s.coord[0][i], s.coord[1][i], s.coord[2][i]);
}

// thermo CSV: step, time, kbt, px, py, pz, n
inline void write_thermo_csv(std::FILE* f, const std::vector<dpdb_thermo>& rec, double dt) {
    std::fprintf(f, "step,time,kbt,px,py,pz,n\n");
    for (const auto& r : rec)
        std::fprintf(f, "%lld,%.10g,%.17g,%.17g,%.17g,%.17g,%llu\n", (long long)r.step, r.step * dt, r.kbt,
                     r.momentum[0], r.momentum[1], r.momentum[2], (unsigned long long)r.n);
}

// minimum_image (src/core.cpp:129-139): half-open on periodic axes
inline Vec3 minimum_image(Vec3 dr, const SimBox& box) {
    for (int k = 0; k < 3; ++k) {
        if (!box.periodic[k]) continue;
        const double L = box.length(k);
        double& d = (&dr.x)[k];
        if (d >= 0.5 * L)
            d -= L;
        else if (d < -0.5 * L)
            d += L;
    }
    return dr;
}

// dump_neighbor_csv (inc/neighbor_table.hpp:57-59): one line per table entry,
// i_tag, j_tag, distance (fp64 minimum image on the `wrap` axes), partition
// (core / skin); the store must be the one the table was built from
inline void dump_neighbor_csv(const NeighborTable& t, const ParticleStore& s, const SimBox& box,
                              const std::array<bool, 3>& wrap, std::FILE* f) {
    std::fprintf(f, "i_tag,j_tag,distance,partition\n");
    SimBox wb = box;
    wb.periodic = wrap;
    for (std::uint32_t i = 0; i < t.n_rows; ++i) {
        for (int part = 0; part < 2; ++part) {
            const std::uint32_t cnt = part ? t.skin_count[i] : t.core_count[i];
            for (std::uint32_t k = 0; k < cnt; ++k) {
                const std::uint32_t j = part ? t.skin_at(i, k) : t.core_at(i, k);
                Vec3 d{s.coord[0][i] - s.coord[0][j], s.coord[1][i] - s.coord[1][j],
                       s.coord[2][i] - s.coord[2][j]};
                d = minimum_image(d, wb);
                std::fprintf(f, "%u,%u,%.17g,%s\n", s.tag[i], s.tag[j],
                             std::sqrt(d.x * d.x + d.y * d.y + d.z * d.z), part ? "skin" : "core");
            }
        }
    }
}

}  // namespace dpd::b200
