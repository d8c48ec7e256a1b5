// ref_caller.cpp -- an unchanged caller of the reference's hot-path C++ API.
//
// Written only against the reference's headers (/root/reference/proj/include:
// dpd/cell_grid.hpp, stencil.hpp, neighbor_table.hpp, radix_sort.hpp, rng.hpp,
// core.hpp, parallel.hpp) plus the two slot headers the reference's build
// names but does not ship (dpd/forces.hpp, dpd/integrate.hpp, dropin/include).
// The same source is linked twice (dropin/Makefile):
//   REF  -- the reference's five shipped sources + oracle/ref_slots.cpp
//   B200 -- the drop-in (dropin/*.cpp over libdpdb.so) + the reference's
//           core.cpp / parallel.cpp / stencil.cpp
// and tests/test_gpu_dropin.py compares the two outputs.
//
//   ref_caller L OUT   (box L^3 at rho 3, seed 1)
// OUT: a sequence of records  u32 name_len, name, u32 dtype (0 u32, 1 f64,
// 2 u16), u64 count, data.  Errors: "ERROR <category> <message>" on stderr
// and the category as exit code (the reference CLI's convention, inc/error.hpp).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "dpd/cell_grid.hpp"
#include "dpd/forces.hpp"
#include "dpd/integrate.hpp"
#include "dpd/neighbor_table.hpp"
#include "dpd/parallel.hpp"
#include "dpd/radix_sort.hpp"
#include "dpd/rng.hpp"
#include "dpd/stencil.hpp"

namespace {
FILE* g_out = nullptr;

template <class T>
void put(const char* name, const T* data, std::size_t n, std::uint32_t dtype) {
    const std::uint32_t len = (std::uint32_t)std::strlen(name);
    const std::uint64_t cnt = n;
    std::fwrite(&len, 4, 1, g_out);
    std::fwrite(name, 1, len, g_out);
    std::fwrite(&dtype, 4, 1, g_out);
    std::fwrite(&cnt, 8, 1, g_out);
    if (n) std::fwrite(data, sizeof(T), n, g_out);
    std::fflush(g_out);
}
void put(const char* name, const std::vector<std::uint32_t>& v) { put(name, v.data(), v.size(), 0); }
void put(const char* name, const std::vector<double>& v) { put(name, v.data(), v.size(), 1); }
void put(const char* name, const std::vector<std::uint16_t>& v) { put(name, v.data(), v.size(), 2); }

// rows through the accessors (inc/neighbor_table.hpp:33-39): counts + CSR
void put_rows(const char* tag, const dpd::NeighborTable& t) {
    std::vector<std::uint16_t> nc(t.n_rows), ns(t.n_rows);
    std::vector<std::uint32_t> flat;
    for (std::uint32_t i = 0; i < t.n_rows; ++i) {
        nc[i] = t.core_count[i];
        ns[i] = t.skin_count[i];
        for (std::uint32_t k = 0; k < nc[i]; ++k) flat.push_back(t.core_at(i, k));
        for (std::uint32_t k = 0; k < ns[i]; ++k) flat.push_back(t.skin_at(i, k));
    }
    put((std::string(tag) + ".core").c_str(), nc);
    put((std::string(tag) + ".skin").c_str(), ns);
    put((std::string(tag) + ".rows").c_str(), flat);
}
}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: ref_caller L OUT\n");
        return 1;
    }
    const double L = std::atof(argv[1]);
    g_out = std::fopen(argv[2], "wb");
    if (!g_out) return 4;
    try {
        using namespace dpd;
        SimBox box;
        box.lo = {0.0, 0.0, 0.0};
        box.hi = {L, L, L};
        const std::size_t n = (std::size_t)std::llround(3.0 * L * L * L);
        ParticleStore s;
        s.resize(n);
        TeaStream ts(1u);
        for (std::size_t i = 0; i < n; ++i) {
            for (int k = 0; k < 3; ++k) s.coord[k][i] = ts.next_u01() * L;
            for (int k = 0; k < 3; ++k) s.veloc[k][i] = ts.next_gaussian();
            s.tag[i] = (std::uint32_t)(i + 1);
        }
        WorkerPool pool(4);

        CellGrid grid = CellGrid::make(box, 1.3);
        const std::uint32_t geo[] = {(std::uint32_t)grid.ncell[0], (std::uint32_t)grid.ncell[1],
                                     (std::uint32_t)grid.ncell[2], grid.n_local_cells, grid.n_total_cells,
                                     (std::uint32_t)grid.bits_per_axis, (std::uint32_t)grid.key_bits()};
        put("grid.geometry", geo, 7, 0);
        put("grid.rank_of_cell", grid.rank_of_cell);
        put("grid.cell_of_rank", grid.cell_of_rank);
        const double geod[] = {grid.cell_size[0], grid.inv_cell[0], grid.origin[0], grid.slab_hi[2]};
        put("grid.cellsize", geod, 4, 1);

        RadixSorter sorter;
        const std::vector<std::uint32_t> perm = reorder_particles(s, grid, sorter, pool);
        put("reorder.perm", perm);
        put("reorder.tag", s.tag);
        put("reorder.x", s.coord[0]);
        const std::vector<std::uint32_t> ranks = local_cell_ranks(s, grid, pool);
        put("cell.ranks", ranks);
        build_cell_list(grid, ranks);
        put("cell.start", grid.cell_start);
        const CoarseStencil cs = build_coarse_stencil(grid, box);
        const FineStencil fs = expand_fine_stencil(cs, grid, pool);
        for (std::size_t i = 0; i < n; ++i) s.signature[i] = make_signature(s.tag[i], s.velocity(i));
        put("signature", s.signature);

        NeighborTable t = build_neighbor_table(s, grid, fs, box, 1.0, 0.3, 128, pool);
        put_rows("table", t);
        join_core_skin(t, pool);
        tile_transpose(t, pool);
        put_rows("table.joined", t);

        const PairParams p = PairParams::make(1, {25.0}, {4.5}, 1.0, 1.0, 1.0, 0.01);
        BondTopology bonds;
        for (std::uint32_t b = 1; b + 1 <= (std::uint32_t)n && b < 4000; b += 40) bonds.bonds.push_back({b, b + 1, 80.0, 0.38});
        compute_forces(s, t, p, bonds, PairRandomState::at(1u, 7u), box);
        put("force.x", s.force[0]);
        put("force.y", s.force[1]);
        put("force.z", s.force[2]);

        // the integrator on the same fp32-valued forces in both builds (the
        // device holds forces in fp32): a fixed field from the tags
        for (int k = 0; k < 3; ++k)
            for (std::size_t i = 0; i < n; ++i) {
                const std::uint32_t h = (s.tag[i] * 2654435761u + 40503u * (std::uint32_t)k) >> 8;
                s.force[k][i] = (double)(float)((double)(h & 0xFFFFu) / 65536.0 * 40.0 - 20.0);
            }
        verlet_step(s, p, StepPhase::Phase1, box);
        put("verlet1.x", s.coord[0]);
        put("verlet1.vz", s.veloc[2]);
        verlet_step(s, p, StepPhase::Phase2, box);
        put("verlet2.vy", s.veloc[1]);

        std::vector<std::uint32_t> keys(n), vals(n);
        TeaStream kr(9u);
        for (std::size_t i = 0; i < n; ++i) keys[i] = kr.next_u32() & 0x00FFFFFFu;
        std::iota(vals.begin(), vals.end(), 0u);
        sorter.sort(keys, vals, 24, pool);
        put("radix.keys", keys);
        put("radix.vals", vals);
    } catch (const dpd::Error& e) {
        std::fprintf(stderr, "ERROR %d %s\n", e.exit_code(), e.what());
        std::fclose(g_out);
        return e.exit_code();
    }
    std::fclose(g_out);
    return 0;
}
