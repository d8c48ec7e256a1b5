// b200_session.cpp -- per-thread device contexts for the drop-in (see the header).
#include "b200_session.hpp"

#include <cstring>
#include <memory>
#include <vector>

namespace dpd::b200 {

[[noreturn]] void raise(int rc, const std::string& what) {
    ErrorCategory cat = ErrorCategory::io;
    if (rc == DPDB_ECONFIG) cat = ErrorCategory::config;
    else if (rc == DPDB_EPHYSICS) cat = ErrorCategory::physics;
    else if (rc == DPDB_EPROTOCOL) cat = ErrorCategory::protocol;
    throw Error(cat, rc == DPDB_EDEVICE ? "device: " + what : what);
}

void check(int rc, const dpdb_ctx* ctx, const char* where) {
    if (rc) raise(rc, std::string(where) + ": " + dpdb_last_error(ctx));
}

dpdb_box to_box(const SimBox& box) {
    dpdb_box b{};
    for (int k = 0; k < 3; ++k) {
        b.lo[k] = box.lo[k];
        b.hi[k] = box.hi[k];
        b.periodic[k] = box.periodic[k];
        b.wall[k] = box.wall[k];
    }
    return b;
}

dpdb_params to_params(const PairParams& p) {
    dpdb_params q{};
    q.n_species = (int32_t)p.n_species;
    for (std::size_t i = 0; i < p.n_species * p.n_species && i < 16; ++i) {
        q.a[i] = p.a[i];
        q.gamma[i] = p.gamma[i];
    }
    q.kbt = p.kbt;
    q.s = p.s;
    q.r_c = p.r_c;
    q.dt = p.dt;
    return q;
}

PairParams cutoff_params(double r_c) {
    PairParams p;
    p.n_species = 1;
    p.a = {25.0};
    p.gamma = {4.5};
    p.sigma = {3.0};
    p.r_c = r_c;
    return p;
}

dpdb_run run_config(double skin, std::uint32_t max_neighbors, std::uint32_t seed, int sub_bits) {
    dpdb_run r{};
    r.rebuild_every = 10;
    r.skin = skin;
    r.drive_axis = 2;
    r.seed = seed;
    r.max_neighbors = max_neighbors;
    r.sub_bits = sub_bits;
    return r;
}

namespace {
struct Slot {
    ContextKey key;
    dpdb_ctx* ctx = nullptr;
    ~Slot() {
        if (ctx) dpdb_destroy(ctx);
    }
};
thread_local Slot g_slot;

bool same(const ContextKey& a, const ContextKey& b) {
    return std::memcmp(&a.box, &b.box, sizeof a.box) == 0 &&
           std::memcmp(&a.params, &b.params, sizeof a.params) == 0 &&
           std::memcmp(&a.run, &b.run, sizeof a.run) == 0;
}
}  // namespace

dpdb_ctx* context(const ContextKey& key) {
    if (g_slot.ctx && same(g_slot.key, key) && g_slot.key.capacity >= key.capacity) return g_slot.ctx;
    if (g_slot.ctx) {
        dpdb_destroy(g_slot.ctx);
        g_slot.ctx = nullptr;
    }
    dpdb_ctx* c = nullptr;
    check(dpdb_create(0, &key.box, &key.params, &key.run, key.capacity ? key.capacity : 1, &c), nullptr,
          "dpdb_create");
    g_slot.key = key;
    g_slot.ctx = c;
    return c;
}

void upload(dpdb_ctx* ctx, const ParticleStore& s) {
    const std::size_t n = s.n;
    const bool sp = s.species.size() >= n && n, mol = s.molecule.size() >= n && n;
    check(dpdb_upload(ctx, n, s.coord[0].data(), s.coord[1].data(), s.coord[2].data(), s.veloc[0].data(),
                      s.veloc[1].data(), s.veloc[2].data(), s.tag.data(), sp ? s.species.data() : nullptr,
                      mol ? s.molecule.data() : nullptr),
          ctx, "upload");
}

}  // namespace dpd::b200
