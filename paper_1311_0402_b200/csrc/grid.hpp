// grid.hpp -- host-side binning geometry of the B200 engine.
//
// Built once per context (the reference builds it once per run): the cell
// lattice, Morton ranks and the coarse stencil are pure functions of the
// box, so they live on the host and are uploaded as small tables.  The
// per-rebuild work (keys, sort, permute, cell list, neighbor build) is on
// the device.
//
//   CellGrid::make / assign_ranks   src/cell_grid.cpp:16-95
//   CellGrid::key_bits              src/cell_grid.cpp:130-134
//   build_coarse_stencil            src/stencil.cpp:7-41
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "dpdb.h"

namespace dpdb {

inline int ceil_log2(uint32_t v) { return v <= 1 ? 0 : 32 - __builtin_clz(v - 1); }

inline uint32_t morton3(uint32_t x, uint32_t y, uint32_t z, int bits) {
    uint32_t c = 0;
    for (int b = 0; b < bits; ++b) {
        c |= ((x >> b) & 1u) << (3 * b);
        if (3 * b + 1 < 32) c |= ((y >> b) & 1u) << (3 * b + 1);
        if (3 * b + 2 < 32) c |= ((z >> b) & 1u) << (3 * b + 2);
    }
    return c;
}

struct HostGrid {
    int ncell[3]{1, 1, 1}, ncell_ext[3]{1, 1, 1}, ghost_lo[3]{}, ghost_hi[3]{};
    bool wrap[3]{};
    double cell_size[3]{}, inv_cell[3]{}, slab_lo[3]{}, slab_hi[3]{}, origin[3]{};
    int sub_bits = 2, bits_per_axis = 1;
    uint32_t n_local_cells = 0, n_total_cells = 0;
    std::vector<uint32_t> rank_of_cell, cell_of_rank;

    size_t ext_index(const int c[3]) const {
        return ((size_t)c[2] * ncell_ext[1] + c[1]) * ncell_ext[0] + c[0];
    }
    void ext_coords(size_t idx, int c[3]) const {
        c[0] = (int)(idx % ncell_ext[0]);
        idx /= ncell_ext[0];
        c[1] = (int)(idx % ncell_ext[1]);
        c[2] = (int)(idx / ncell_ext[1]);
    }
    bool is_local(const int c[3]) const {
        for (int k = 0; k < 3; ++k)
            if (c[k] < ghost_lo[k] || c[k] >= ghost_lo[k] + ncell[k]) return false;
        return true;
    }
    int key_bits() const { return (ceil_log2(n_total_cells) + 3 * sub_bits + 3) & ~3; }
    int raw_key_bits() const { return ceil_log2(n_total_cells) + 3 * sub_bits; }

    // returns 0 or an error category, message in err
    int make(const dpdb_box& box, const double slo[3], const double shi[3], const int dims[3],
             const int coords[3], double target, int sb, std::string& err) {
        if (!(target > 0)) {
            err = "cell grid: cell target must be positive";
            return DPDB_ECONFIG;
        }
        sub_bits = sb;
        for (int k = 0; k < 3; ++k) {
            slab_lo[k] = slo[k];
            slab_hi[k] = shi[k];
            const double len = shi[k] - slo[k];
            if (len < target) {
                err = "cell grid: slab thinner than cutoff+skin on axis " + std::to_string(k);
                return DPDB_ECONFIG;
            }
            ncell[k] = std::max(1, (int)std::floor(len / target));
            cell_size[k] = len / ncell[k];
            inv_cell[k] = ncell[k] / len;
            wrap[k] = dims[k] == 1 && box.periodic[k];
            const bool lower = dims[k] > 1 && (coords[k] > 0 || box.periodic[k]);
            const bool upper = dims[k] > 1 && (coords[k] < dims[k] - 1 || box.periodic[k]);
            ghost_lo[k] = lower;
            ghost_hi[k] = upper;
            ncell_ext[k] = ncell[k] + lower + upper;
            origin[k] = slo[k] - ghost_lo[k] * cell_size[k];
        }
        const size_t total = (size_t)ncell_ext[0] * ncell_ext[1] * ncell_ext[2];
        n_total_cells = (uint32_t)total;
        n_local_cells = (uint32_t)ncell[0] * ncell[1] * ncell[2];
        bits_per_axis = 1;
        for (int k = 0; k < 3; ++k) bits_per_axis = std::max(bits_per_axis, ceil_log2(ncell_ext[k]));
        if (3 * bits_per_axis > 32) {
            err = "cell grid: too many cells per axis";
            return DPDB_ECONFIG;
        }
        if (raw_key_bits() > 32) {
            err = "cell grid: sort key exceeds 32 bits";
            return DPDB_ECONFIG;
        }
        // locals by local-lattice Morton code, then ghosts by ext-lattice code
        std::vector<std::pair<uint32_t, uint32_t>> loc, gh;
        loc.reserve(n_local_cells);
        gh.reserve(total - n_local_cells);
        for (size_t idx = 0; idx < total; ++idx) {
            int c[3];
            ext_coords(idx, c);
            if (is_local(c))
                loc.emplace_back(morton3(c[0] - ghost_lo[0], c[1] - ghost_lo[1], c[2] - ghost_lo[2],
                                         bits_per_axis),
                                 (uint32_t)idx);
            else
                gh.emplace_back(morton3(c[0], c[1], c[2], bits_per_axis), (uint32_t)idx);
        }
        std::sort(loc.begin(), loc.end());
        std::sort(gh.begin(), gh.end());
        rank_of_cell.assign(total, 0);
        cell_of_rank.assign(total, 0);
        uint32_t r = 0;
        for (auto& p : loc) {
            rank_of_cell[p.second] = r;
            cell_of_rank[r++] = p.second;
        }
        for (auto& p : gh) {
            rank_of_cell[p.second] = r;
            cell_of_rank[r++] = p.second;
        }
        return DPDB_OK;
    }

    // <= 27 neighbor ranks per local cell, ascending and unique; stride-32
    // rows for the device plus counts.  Also the per-cell min-image flags:
    //   bits 0-2: the neighbor builder must apply the fp32 minimum image on
    //             axis k (cell touches the periodic seam, or ncell_k < 5 so an
    //             interior cell could see |dx| >= L/2)
    //   bits 3-5: the force kernel must (3 cell layers from the seam, or
    //             ncell_k < 8, covering drift between rebuilds)
    //
    // codes (optional, k_build_range's cell culling): per stencil slot the
    // offset (ox+1) | (oy+1) << 2 | (oz+1) << 4 of that cell from the centre
    // cell, or 0xFF (never cull) when the slot stands for several offsets (deduplicated
    // small grids) or a wrapped axis has < 5 cells (the nearest image need not
    // be the geometric neighbor); cell_lo: each local cell's lower corner in
    // the pos4 frame (x - slab centre), fp32.
    void coarse_stencil(std::vector<uint32_t>& rows, std::vector<uint8_t>& counts,
                        std::vector<uint8_t>& flags, std::vector<uint8_t>* codes = nullptr,
                        std::vector<float>* cell_lo = nullptr) const {
        rows.assign((size_t)n_local_cells * 32, 0);
        counts.assign(n_local_cells, 0);
        flags.assign(n_local_cells, 0);
        bool cull = true;
        for (int k = 0; k < 3; ++k)
            if (wrap[k] && ncell[k] < 5) cull = false;
        if (codes) codes->assign((size_t)n_local_cells * 32, 0xFF);
        if (cell_lo) cell_lo->assign((size_t)n_local_cells * 4, 0.f);
        for (uint32_t r = 0; r < n_local_cells; ++r) {
            int c[3];
            ext_coords(cell_of_rank[r], c);
            if (cell_lo)
                for (int k = 0; k < 3; ++k)
                    (*cell_lo)[(size_t)r * 4 + k] =
                        (float)(origin[k] + c[k] * cell_size[k] - 0.5 * (slab_lo[k] + slab_hi[k]));
            uint32_t list[27];
            std::pair<uint32_t, int> coded[27];
            int m = 0;
            for (int dz = -1; dz <= 1; ++dz)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int off[3] = {dx, dy, dz};
                        int nc[3];
                        bool ok = true;
                        for (int k = 0; k < 3 && ok; ++k) {
                            int v = c[k] + off[k];
                            if (wrap[k])
                                v = (v + ncell[k]) % ncell[k];
                            else if (v < 0 || v >= ncell_ext[k])
                                ok = false;
                            nc[k] = v;
                        }
                        if (ok) {
                            coded[m] = {rank_of_cell[ext_index(nc)], (dx + 1) | (dy + 1) << 2 | (dz + 1) << 4};
                            list[m] = coded[m].first;
                            ++m;
                        }
                    }
            std::sort(list, list + m);
            const int u = (int)(std::unique(list, list + m) - list);
            std::copy(list, list + u, rows.begin() + (size_t)r * 32);
            counts[r] = (uint8_t)u;
            if (codes && cull && u == m) {
                std::sort(coded, coded + m);
                for (int q = 0; q < m; ++q) (*codes)[(size_t)r * 32 + q] = (uint8_t)coded[q].second;
            }
            uint8_t f = 0;
            for (int k = 0; k < 3; ++k) {
                if (!wrap[k]) continue;
                const int lc = c[k] - ghost_lo[k];
                if (ncell[k] < 5 || lc == 0 || lc == ncell[k] - 1) f |= (uint8_t)(1u << k);
                if (ncell[k] < 8 || lc <= 2 || lc >= ncell[k] - 3) f |= (uint8_t)(8u << k);
            }
            flags[r] = f;
        }
    }
};

}  // namespace dpdb
