// ref_shim.cpp -- extern "C" wrappers around the reference's OWN shipped
// code (headers under /root/reference/proj/include, sources under
// /root/reference/proj/src), compiled in place by oracle/Makefile into
// oracle/_ref/libdpdref.so.  TEST INFRASTRUCTURE ONLY: it exists to pin the
// C restatement in oracle/dpd_oracle.c and to generate tests/golden/.
// No reference source is copied into this repository.
#include <chrono>
#include <cstdint>
#include <memory>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "dpd/cell_grid.hpp"
#include "dpd/core.hpp"
#include "dpd/error.hpp"
#include "dpd/fastmath.hpp"
#include "dpd/morton.hpp"
#include "dpd/parallel.hpp"
#include "dpd/radix_sort.hpp"
#include "dpd/rng.hpp"
#include "dpd/stencil.hpp"

namespace {
thread_local std::string g_err;
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const dpd::Error& e) {
        g_err = e.what();
        return e.exit_code();
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}
dpd::SimBox make_box(const double lo[3], const double hi[3], const int32_t periodic[3]) {
    dpd::SimBox b;
    b.lo = {lo[0], lo[1], lo[2]};
    b.hi = {hi[0], hi[1], hi[2]};
    for (int k = 0; k < 3; ++k) {
        b.periodic[k] = periodic[k] != 0;
        b.wall[k] = false;
    }
    return b;
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_tea_hash(int rounds, uint32_t v0, uint32_t v1, uint32_t out[2]) {
    const auto p = dpd::tea_hash(rounds, v0, v1);
    out[0] = p.v0;
    out[1] = p.v1;
}
uint32_t ref_bit_reverse(uint32_t x) { return dpd::bit_reverse(x); }
uint32_t ref_make_signature(uint32_t tag, double vx, double vy, double vz) {
    return dpd::make_signature(tag, dpd::Vec3{vx, vy, vz});
}
uint32_t ref_step_mix(uint32_t seed, uint32_t step) {
    return dpd::PairRandomState::at(seed, step).step_mix;
}
void ref_pair_uniforms(uint32_t si, uint32_t sj, uint32_t ti, uint32_t tj, uint32_t seed,
                       uint32_t step, uint32_t out[2]) {
    const auto p = dpd::pair_uniforms(si, sj, ti, tj, dpd::PairRandomState::at(seed, step));
    out[0] = p.v0;
    out[1] = p.v1;
}
double ref_gaussian(uint32_t a, uint32_t b) { return dpd::gaussian(a, b); }
double ref_fastlog(uint32_t v) { return dpd::fastlog(v); }
double ref_fastcos2pi(uint32_t v) { return dpd::fastcos2pi(v); }
double ref_fastpow(double a, double b) { return dpd::fastpow(a, b); }
double ref_power2(int n) { return dpd::power2(n); }
double ref_exp2_frac(double x) { return dpd::exp2_frac(x); }
double ref_log2_frac(double x) { return dpd::log2_frac(x); }

int ref_morton_encode(uint32_t ix, uint32_t iy, uint32_t iz, int bits, uint32_t* code) {
    return guarded([&] { *code = dpd::morton_encode(ix, iy, iz, bits); });
}

int ref_radix_sort(uint32_t* keys, uint32_t* vals, size_t n, int bits, unsigned workers) {
    return guarded([&] {
        dpd::WorkerPool pool(workers);
        dpd::radix_sort(std::span<uint32_t>(keys, n), std::span<uint32_t>(vals, n), bits, pool);
    });
}

// Single-domain grid geometry.  out_i: ncell[3], ncell_ext[3], wrapmode[3],
// bits_per_axis, n_local_cells, n_total_cells, key_bits.  out_d: cell_size[3],
// inv_cell[3], origin[3].
int ref_grid_info(const double lo[3], const double hi[3], const int32_t periodic[3],
                  double cell_target, int sub_bits, int64_t out_i[13], double out_d[9]) {
    return guarded([&] {
        const auto box = make_box(lo, hi, periodic);
        const auto g = dpd::CellGrid::make(box, cell_target, sub_bits);
        for (int k = 0; k < 3; ++k) {
            out_i[k] = g.ncell[k];
            out_i[3 + k] = g.ncell_ext[k];
            out_i[6 + k] = g.wrapmode[k];
            out_d[k] = g.cell_size[k];
            out_d[3 + k] = g.inv_cell[k];
            out_d[6 + k] = g.origin[k];
        }
        out_i[9] = g.bits_per_axis;
        out_i[10] = g.n_local_cells;
        out_i[11] = g.n_total_cells;
        out_i[12] = g.key_bits();
    });
}

// rank_of_cell[n_total_cells]
int ref_grid_ranks(const double lo[3], const double hi[3], const int32_t periodic[3],
                   double cell_target, int sub_bits, uint32_t* rank_of_cell) {
    return guarded([&] {
        const auto g = dpd::CellGrid::make(make_box(lo, hi, periodic), cell_target, sub_bits);
        std::memcpy(rank_of_cell, g.rank_of_cell.data(), g.rank_of_cell.size() * 4);
    });
}

// Full reorder + cell list + stencils on one domain (src/cell_grid.cpp:166,
// 157, 136; src/stencil.cpp:7, 43).  x,y,z,tag are permuted in place.
// perm[n]; cell_start[n_total+1]; coff[n_local+1]; ccells[27*n_local];
// foff[n_local+1]; fidx may be NULL (then only foff is filled).
int ref_reorder_cells(const double lo[3], const double hi[3], const int32_t periodic[3],
                      double cell_target, int sub_bits, unsigned workers, size_t n, double* x,
                      double* y, double* z, uint32_t* tag, uint32_t* perm, uint32_t* cell_start,
                      uint32_t* coff, uint32_t* ccells, uint32_t* foff, uint32_t* fidx,
                      size_t fidx_cap) {
    return guarded([&] {
        const auto box = make_box(lo, hi, periodic);
        auto g = dpd::CellGrid::make(box, cell_target, sub_bits);
        dpd::ParticleStore st;
        st.resize(n);
        for (size_t i = 0; i < n; ++i) {
            st.coord[0][i] = x[i];
            st.coord[1][i] = y[i];
            st.coord[2][i] = z[i];
            st.tag[i] = tag[i];
        }
        dpd::WorkerPool pool(workers);
        dpd::RadixSorter sorter;
        const auto p = dpd::reorder_particles(st, g, sorter, pool);
        for (size_t i = 0; i < n; ++i) {
            x[i] = st.coord[0][i];
            y[i] = st.coord[1][i];
            z[i] = st.coord[2][i];
            tag[i] = st.tag[i];
            perm[i] = p[i];
        }
        const auto ranks = dpd::local_cell_ranks(st, g, pool);
        dpd::build_cell_list(g, ranks);
        std::memcpy(cell_start, g.cell_start.data(), g.cell_start.size() * 4);
        const auto cs = dpd::build_coarse_stencil(g, box);
        std::memcpy(coff, cs.offsets.data(), cs.offsets.size() * 4);
        std::memcpy(ccells, cs.cells.data(), cs.cells.size() * 4);
        const auto fs = dpd::expand_fine_stencil(cs, g, pool);
        std::memcpy(foff, fs.offsets.data(), fs.offsets.size() * 4);
        if (fidx) {
            if (fs.indices.size() > fidx_cap)
                dpd::fail(dpd::ErrorCategory::config, "fine stencil larger than buffer");
            std::memcpy(fidx, fs.indices.data(), fs.indices.size() * 4);
        }
    });
}

// build_cell_list on explicit ranks (error behaviour on unsorted input)
int ref_build_cell_list(uint32_t n_total_cells, const uint32_t* ranks, size_t n,
                        uint32_t* cell_start) {
    return guarded([&] {
        dpd::CellGrid g;
        g.n_total_cells = n_total_cells;
        dpd::build_cell_list(g, std::span<const uint32_t>(ranks, n));
        std::memcpy(cell_start, g.cell_start.data(), g.cell_start.size() * 4);
    });
}

double ref_temperature(size_t n, const double* vx, const double* vy, const double* vz) {
    dpd::ParticleStore st;
    st.resize(n);
    for (size_t i = 0; i < n; ++i) {
        st.veloc[0][i] = vx[i];
        st.veloc[1][i] = vy[i];
        st.veloc[2][i] = vz[i];
    }
    double t = -1;
    guarded([&] { t = dpd::compute_temperature(st); });
    return t;
}

void ref_minimum_image(const double dr[3], const double lo[3], const double hi[3],
                       const int32_t periodic[3], double out[3]) {
    const auto r = dpd::minimum_image(dpd::Vec3{dr[0], dr[1], dr[2]}, make_box(lo, hi, periodic));
    out[0] = r.x;
    out[1] = r.y;
    out[2] = r.z;
}

int ref_params_sigma(int n_species, const double* a, const double* gamma, double kbt, double s,
                     double r_c, double dt, double* sigma) {
    return guarded([&] {
        const auto p = dpd::PairParams::make(
            n_species, std::vector<double>(a, a + n_species * n_species),
            std::vector<double>(gamma, gamma + n_species * n_species), kbt, s, r_c, dt);
        std::memcpy(sigma, p.sigma.data(), p.sigma.size() * 8);
    });
}

// ---- CPU baseline: the reference's own reorder step inside the oracle's
// whole-step driver (orc_sim_set_reorder_hook).  One persistent grid,
// WorkerPool and RadixSorter per run, as the reference's runner would hold.
struct RefSimCtx {
    dpd::SimBox box;
    dpd::CellGrid grid;
    std::unique_ptr<dpd::WorkerPool> pool;
    dpd::RadixSorter sorter;
    dpd::ParticleStore st;
};

void* ref_sim_ctx_create(const double lo[3], const double hi[3], const int32_t periodic[3],
                         double cell_target, int sub_bits, unsigned workers) {
    auto* c = new RefSimCtx();
    if (guarded([&] {
            c->box = make_box(lo, hi, periodic);
            c->grid = dpd::CellGrid::make(c->box, cell_target, sub_bits);
            c->pool = std::make_unique<dpd::WorkerPool>(workers);
        })) {
        delete c;
        return nullptr;
    }
    return c;
}

void ref_sim_ctx_destroy(void* c) { delete static_cast<RefSimCtx*>(c); }

// reorder_particles (src/cell_grid.cpp:166-198, RadixSorter src/radix_sort.cpp:16-74)
// + local_cell_ranks + build_cell_list on the driver's arrays; *seconds covers
// those three reference calls only (not the copies into / out of the store)
int ref_sim_reorder(void* vc, size_t n, double* x[3], double* v[3], uint32_t* tag, uint8_t* species,
                    uint32_t* cell_start, double* seconds) {
    auto* c = static_cast<RefSimCtx*>(vc);
    return guarded([&] {
        auto& st = c->st;
        if (st.n != n) st.resize(n);
        for (int k = 0; k < 3; ++k) {
            std::memcpy(st.coord[k].data(), x[k], n * 8);
            std::memcpy(st.veloc[k].data(), v[k], n * 8);
        }
        std::memcpy(st.tag.data(), tag, n * 4);
        std::memcpy(st.species.data(), species, n);
        const auto t0 = std::chrono::steady_clock::now();
        dpd::reorder_particles(st, c->grid, c->sorter, *c->pool);
        const auto ranks = dpd::local_cell_ranks(st, c->grid, *c->pool);
        dpd::build_cell_list(c->grid, ranks);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (int k = 0; k < 3; ++k) {
            std::memcpy(x[k], st.coord[k].data(), n * 8);
            std::memcpy(v[k], st.veloc[k].data(), n * 8);
        }
        std::memcpy(tag, st.tag.data(), n * 4);
        std::memcpy(species, st.species.data(), n);
        std::memcpy(cell_start, c->grid.cell_start.data(), c->grid.cell_start.size() * 4);
    });
}

} // extern "C"
