// domain.cuh -- brick decomposition kernels (paper Alg. 6).
// Included by kernels.cuh (namespace dpdb).
//
// One context owns one brick (slab).  Locals live at [0, n), ghosts at
// [n, n + ng) of the same SoA arrays.  Directions d in [0, 26) enumerate the
// neighbor offsets (dx, dy, dz) in z-major order with the centre removed;
// opposite(d) = 25 - d.
#pragma once

__host__ __device__ __forceinline__ void dir_offset(int d26, int off[3]) {
    const int d = d26 < 13 ? d26 : d26 + 1;
    off[0] = d % 3 - 1;
    off[1] = (d / 3) % 3 - 1;
    off[2] = d / 9 - 1;
}
__host__ __device__ __forceinline__ int dir_index(int dx, int dy, int dz) {
    const int d = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
    return d < 13 ? d : d - 1;
}

struct BorderArgs {
    const double* x[3];
    double lo[3], hi[3];   // slab bounds
    double cut;            // r_c + skin
    uint32_t valid_dirs;   // bit d: a neighbor exists in direction d
    uint32_t n;
};

// 26-bit mask of send directions of a local particle (border_determination,
// S:563-571): within `cut` of the faces/edges/corner of direction d
__device__ __forceinline__ uint32_t border_mask(const BorderArgs& a, uint32_t i) {
    int lo_side[3], hi_side[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double x = a.x[k][i];
        lo_side[k] = x < a.lo[k] + a.cut;
        hi_side[k] = x >= a.hi[k] - a.cut;
    }
    uint32_t m = 0;
    for (int d = 0; d < 26; ++d) {
        int off[3];
        dir_offset(d, off);
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 3; ++k)
            ok = ok && (off[k] == 0 || (off[k] < 0 ? lo_side[k] : hi_side[k]));
        if (ok) m |= 1u << d;
    }
    return m & a.valid_dirs;
}

// Generic multi-list stream compaction by 26 flags per element (Alg. 6:
// flag -> per-block counts -> scan -> scatter), ascending element order inside
// every list, deterministic.  mask_of(i) supplies the flags.
constexpr int MD_THREADS = 256;

__global__ void __launch_bounds__(MD_THREADS) k_dir_count(const uint32_t* __restrict__ masks,
                                                          uint32_t n, uint32_t nblocks,
                                                          uint32_t* __restrict__ counts) {
    __shared__ uint32_t wc[MD_THREADS / 32][26];
    const uint32_t i = blockIdx.x * MD_THREADS + threadIdx.x;
    const uint32_t m = i < n ? masks[i] : 0u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int d = 0; d < 26; ++d) {
        const uint32_t b = __ballot_sync(0xFFFFFFFFu, (m >> d) & 1u);
        if (lane == 0) wc[warp][d] = __popc(b);
    }
    __syncthreads();
    if (threadIdx.x < 26) {
        uint32_t s = 0;
        for (int w = 0; w < MD_THREADS / 32; ++w) s += wc[w][threadIdx.x];
        counts[threadIdx.x * nblocks + blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(MD_THREADS) k_dir_scatter(const uint32_t* __restrict__ masks,
                                                            uint32_t n, uint32_t nblocks,
                                                            const uint32_t* __restrict__ offs,
                                                            uint32_t* __restrict__ lists) {
    __shared__ uint32_t wc[MD_THREADS / 32][26];
    const uint32_t i = blockIdx.x * MD_THREADS + threadIdx.x;
    const uint32_t m = i < n ? masks[i] : 0u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    uint32_t rank[26];
    for (int d = 0; d < 26; ++d) {
        const uint32_t b = __ballot_sync(0xFFFFFFFFu, (m >> d) & 1u);
        rank[d] = __popc(b & lt);
        if (lane == 0) wc[warp][d] = __popc(b);
    }
    __syncthreads();
    for (int d = 0; d < 26; ++d) {
        if (!((m >> d) & 1u)) continue;
        uint32_t base = offs[d * nblocks + blockIdx.x];
        for (int w = 0; w < warp; ++w) base += wc[w][d];
        lists[base + rank[d]] = i;
    }
}

__global__ void k_border_masks(BorderArgs a, uint32_t* masks) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < a.n) masks[i] = border_mask(a, i);
}

// Migration flags: a local that left the slab goes to the
// neighbor brick holding it; more than one brick away is a protocol error.
struct MigrateArgs {
    const double* x[3];
    const uint32_t* tag;
    double box_lo[3], slab_len[3], slab_lo[3], slab_hi[3];
    int dims[3], coords[3];
    uint32_t valid_dirs;
    uint32_t n;
    DevErr* err;
};

__global__ void k_migrate_masks(MigrateArgs a, uint32_t* masks) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    int off[3];
    bool out = false, bad = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double x = a.x[k][i];
        off[k] = 0;
        if (x >= a.slab_lo[k] && x < a.slab_hi[k]) continue;
        out = true;
        int dest = (int)floor((x - a.box_lo[k]) / a.slab_len[k]);
        dest = min(max(dest, 0), a.dims[k] - 1);
        const int delta = ((dest - a.coords[k]) % a.dims[k] + a.dims[k]) % a.dims[k];
        if (delta == 1)
            off[k] = 1;
        else if (delta == a.dims[k] - 1)
            off[k] = -1;
        else
            bad = true;
        if (a.dims[k] == 2) off[k] = x < a.slab_lo[k] ? -1 : 1;
    }
    uint32_t m = 0;
    if (out && !bad) {
        const int d = dir_index(off[0], off[1], off[2]);
        if ((a.valid_dirs >> d) & 1u)
            m = 1u << d;
        else
            bad = true;
    }
    if (bad) raise_err(a.err, DPDB_EPROTOCOL, EW_MIGRATION, a.tag[i], 0);
    masks[i] = m;
}

// ghost / migrant wire record (GhostPacket payload, device side)
struct GhostRec {
    double x[3];
    double v[3];
    uint32_t tag;
    uint32_t sp_mol;  // species (8 bits) | molecule << 8 (molecule < 2^24)
};
struct GhostUpd {
    double x[3];
    double v[3];
};

struct PackArgs {
    const double* x[3];
    const double* v[3];
    const uint32_t* tag;
    const uint8_t* sp;
    const uint32_t* mol;
    const uint32_t* lists;     // concatenated per-direction index lists
    const uint32_t* dir_off;   // [27] list offsets
    double shift[26][3];       // periodic image shift per direction
    uint32_t total;
};

__device__ __forceinline__ int find_dir(const uint32_t* off, uint32_t s) {
    int d = 0;
    while (d < 25 && off[d + 1] <= s) ++d;
    return d;
}

template <bool FULL>
__global__ void k_pack(PackArgs a, void* out) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= a.total) return;
    const int d = find_dir(a.dir_off, s);
    const uint32_t i = a.lists[s];
    if (FULL) {
        GhostRec r;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            r.x[k] = __dadd_rn(a.x[k][i], a.shift[d][k]);
            r.v[k] = a.v[k][i];
        }
        r.tag = a.tag[i];
        r.sp_mol = (uint32_t)a.sp[i] | ((a.mol ? a.mol[i] : 0u) << 8);
        static_cast<GhostRec*>(out)[s] = r;
    } else {
        GhostUpd r;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            r.x[k] = __dadd_rn(a.x[k][i], a.shift[d][k]);
            r.v[k] = a.v[k][i];
        }
        static_cast<GhostUpd*>(out)[s] = r;
    }
}

struct UnpackArgs {
    double* x[3];
    double* v[3];
    uint32_t* tag;
    uint8_t* sp;
    uint32_t* mol;
    uint32_t* keys;      // ghost keys (FULL)
    uint32_t* vals;
    const uint32_t* slot_of;  // update: receive index -> ghost slot
    float4* pos4;
    int4* posq;
    float4* vel4;
    PosQ pq;
    DevGrid grid;
    uint32_t base;       // first slot (n for ghosts, n_keep for migrants)
    uint32_t count;
    int multi;
    int ghost;           // ghost keys (clamped ghost_cell_of) vs local keys
    DevErr* err;
};

// ext-lattice cell of a ghost (CellGrid::ghost_cell_of, src/cell_grid.cpp:110-117)
__device__ __forceinline__ uint32_t ghost_key_of(const DevGrid& g, const double p[3]) {
    int c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int ci = __double2int_rd(__dmul_rn(__dsub_rn(p[k], g.origin[k]), g.inv_cell[k]));
        c[k] = min(max(ci, 0), g.ncell_ext[k] - 1);
    }
    const uint32_t rank =
        g.rank_of_cell[((size_t)c[2] * g.ncell_ext[1] + c[1]) * g.ncell_ext[0] + c[0]];
    const int nsub = 1 << g.sub_bits;
    uint32_t s[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double cell_lo = __dadd_rn(g.origin[k], __dmul_rn((double)c[k], g.cell_size[k]));
        const int si = __double2int_rd(
            __dmul_rn(__dmul_rn(__dsub_rn(p[k], cell_lo), g.inv_cell[k]), (double)nsub));
        s[k] = (uint32_t)min(max(si, 0), nsub - 1);
    }
    uint32_t sub = 0;
    for (int b = 0; b < g.sub_bits; ++b)
        sub |= (((s[0] >> b) & 1u) << (3 * b)) | (((s[1] >> b) & 1u) << (3 * b + 1)) |
               (((s[2] >> b) & 1u) << (3 * b + 2));
    return (rank << (3 * g.sub_bits)) | sub;
}

// Ghost update as one put (Alg. 6's "border determination + put"):
// the sender reads each send-list particle's fp64 state and writes it, with
// the periodic image shift of its direction, straight into the receiving
// brick's ghost slot -- x, v and the receiver-frame fp32 streams (pos4, posq,
// vel4 + signature), the same arithmetic as k_pack + k_unpack<false> -- with
// plain stores through the receiver's pointers (device memory of another
// brick on this GPU, or of a peer GPU over NVLink with peer access on).  No
// record buffer, no copy, no unpack launch.
struct PutDir {  // the receiver in one direction of the sender
    double* x[3];
    double* v[3];
    const uint32_t* tag;
    const uint8_t* sp;
    const uint32_t* slot_of;  // receiver's receive index -> ghost slot (fixed at the rebuild)
    float4* pos4;
    int4* posq;
    float4* vel4;
    PosQ pq;
    double centre[3];
    double shift[3];  // sender-side periodic image shift of this direction
    uint32_t rbase;   // receiver's receive index of this direction's first record
    int multi;
};

struct PutArgs {
    const double* x[3];
    const double* v[3];
    const uint32_t* lists;  // sender's concatenated send lists
    uint32_t off[27];       // list offsets per direction
    uint32_t total;
    PutDir dir[26];
};

__global__ void __launch_bounds__(256) k_put(const __grid_constant__ PutArgs a) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= a.total) return;
    const int d = find_dir(a.off, s);
    const PutDir& P = a.dir[d];
    const uint32_t i = a.lists[s];
    const uint32_t g = P.slot_of[P.rbase + (s - a.off[d])];
    double x[3], v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        x[k] = __dadd_rn(a.x[k][i], P.shift[k]);
        v[k] = a.v[k][i];
        P.x[k][g] = x[k];
        P.v[k][g] = v[k];
    }
    const uint32_t tag = P.tag[g];
    const uint32_t tw = P.multi ? (tag | ((uint32_t)P.sp[g] << 28)) : tag;
    const uint32_t sig = make_signature(tag, v[0], v[1], v[2]);
    P.pos4[g] = make_float4((float)(x[0] - P.centre[0]), (float)(x[1] - P.centre[1]),
                            (float)(x[2] - P.centre[2]), __uint_as_float(tw));
    P.posq[g] = posq_of(P.pq, x[0], x[1], x[2], tw);
    P.vel4[g] = make_float4((float)v[0], (float)v[1], (float)v[2], __uint_as_float(sig));
}

template <bool FULL>
__global__ void k_unpack(UnpackArgs a, const void* in) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= a.count) return;
    if (FULL) {
        const GhostRec rec = static_cast<const GhostRec*>(in)[r];
        const uint32_t g = a.base + r;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            a.x[k][g] = rec.x[k];
            a.v[k][g] = rec.v[k];
        }
        a.tag[g] = rec.tag;
        a.sp[g] = (uint8_t)(rec.sp_mol & 0xFFu);
        if (a.mol) a.mol[g] = rec.sp_mol >> 8;
        uint32_t key = 0;
        if (a.ghost) {
            key = ghost_key_of(a.grid, rec.x);
        } else if (!sort_key_of(a.grid, rec.x[0], rec.x[1], rec.x[2], key)) {
            key = 0xFFFFFFFFu;  // misrouted migrant: dropped, and the step fails
            raise_err(a.err, DPDB_EPROTOCOL, EW_MIGRATION, rec.tag, 0);
        }
        a.keys[g] = key;
        a.vals[g] = g;
    } else {
        const GhostUpd rec = static_cast<const GhostUpd*>(in)[r];
        const uint32_t g = a.slot_of[r];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            a.x[k][g] = rec.x[k];
            a.v[k][g] = rec.v[k];
        }
        const uint32_t tag = a.tag[g];
        const uint32_t tw = a.multi ? (tag | ((uint32_t)a.sp[g] << 28)) : tag;
        const uint32_t sig = make_signature(tag, rec.v[0], rec.v[1], rec.v[2]);
        a.pos4[g] = make_float4((float)(rec.x[0] - a.grid.centre[0]),
                                (float)(rec.x[1] - a.grid.centre[1]),
                                (float)(rec.x[2] - a.grid.centre[2]), __uint_as_float(tw));
        a.posq[g] = posq_of(a.pq, rec.x[0], rec.x[1], rec.x[2], tw);
        a.vel4[g] = make_float4((float)rec.v[0], (float)rec.v[1], (float)rec.v[2],
                                __uint_as_float(sig));
    }
}
