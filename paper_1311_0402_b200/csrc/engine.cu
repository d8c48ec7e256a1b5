// engine.cu -- host side of the B200 DPD engine: device context, Alg. 1 step
// driver and the C ABI declared in include/dpdb.h.
//
// Host code is C++; every per-particle operation is a hand-written sm_100a
// kernel (kernels.cuh).  There is no CPU fallback: without a compute
// capability 10.x device every entry point fails with DPDB_EDEVICE.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <array>
#include <vector>

#include "dpdb.h"
#include "grid.hpp"
#include "kernels.cuh"

using dpdb::DevErr;
using dpdb::HostGrid;

namespace {
thread_local std::string g_thread_err;
// dpdb_create_domain passes the brick through these (same thread, same call)
thread_local const int32_t* g_pending_dims = nullptr;
thread_local const int32_t* g_pending_coords = nullptr;

constexpr int BUILD_WARPS = 4;
constexpr int BUILD_TILES = 2;
constexpr int RED_BLOCKS = 296;

enum Stage { ST_INTEGRATE = 0, ST_SORT = 1, ST_BUILD = 2, ST_FORCE = 3, ST_OTHER = 4, ST_N = 5 };
}  // namespace

struct dpdb_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    // bricks: the ghost update runs on halo_stream while the interior force
    // blocks run on stream (ev_pack: send records packed; ev_halo: ghosts in)
    cudaStream_t halo_stream = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
    uint8_t* blk_ghost{};  // per force block: 1 if any row has a ghost partner (set by the builder)
    // velocity_profile accumulators: 2 * nbins u64 (fixed-point sums, counts)
    unsigned long long* prof_acc{};
    uint32_t prof_nbins = 0;
    int prof_bin_axis = 2, prof_vel_axis = 0;
    int64_t prof_samples = 0;
    dpdb_box box{};
    dpdb_params params{};
    dpdb_run run{};
    HostGrid grid;
    double sigma[16]{};
    size_t cap = 0, n = 0, n_pad = 0;
    uint32_t maxn = 128;
    // device state
    double *x[3]{}, *v[3]{}, *x2[3]{}, *v2[3]{};
    float *f[3]{}, *f2[3]{};
    uint32_t *tag{}, *tag2{}, *mol{}, *mol2{};
    uint8_t *sp{}, *sp2{};
    float4 *pos4{}, *vel4{}, *vel4n{};  // n: next-step streams of the fused force pass
    int4 *posq{}, *posqn{};  // pair-force frame (PosQ) + the fused pass's next-step buffer
    uint32_t *keys{}, *keys2{}, *vals{}, *vals2{}, *hist{};
    uint32_t* rs_work{};  // onesweep sort: tile status words, digit histograms, tile counters
    uint32_t *cell_start{}, *ostart{}, *rank_of_cell{}, *stencil{};
    uint8_t *stencil_n{}, *cell_flags{}, *stencil_code{};
    float4* cell_lo{};
    uint32_t *entries{}, *counts{}, *fwalk{};
    uint32_t* plist{};  // walk layouts: per-tile flat pair lists of the force kernel (k_tile_compact)
    uint2* rowmeta{};
    // table layout: 0 reference (split/joined), 1 ballot walk (k_build), 2 lane
    // walk (k_build_lane), 3 range walk (k_build_range: front entries only)
    int walk = 0;
    // builder: 2 = k_build_range (default), 1 = k_build_lane (DPDB_BUILDER=lane),
    // 0 = the ballot k_build (DPDB_BUILDER=ballot)
    int builder = 2;
    DevErr* err{};
    // error polling inside long dpdb_step calls: at each rebuild the device
    // error word is copied (async) to pinned memory; the next rebuild reads the
    // copy if it has landed and stops the loop early on an error
    DevErr* err_host{};
    cudaEvent_t err_ev = nullptr;
    bool err_pending = false;
    double *red{}, *red_out{};
    uint32_t* tmp_u32{};
    // bonds (CSR by tag; index_of_tag refreshed at every permute)
    uint32_t *bond_off{}, *bond_partner{}, *index_of_tag{};
    float *bond_k{}, *bond_r0{};
    uint8_t* bond_style{};
    // angles (CSR by tag: each angle at its three members with their role)
    uint32_t* ang_off{};
    uint4* ang_rec{};
    float *ang_k{}, *ang_t0{};
    size_t n_bonds = 0;  // bonded terms present: bonds + angles
    bool styled = false;  // FENE bonds or angles present (bond styles / angle CSR uploaded)
    uint32_t max_tag = 0;
    // host copies of the topology (both CSRs are rebuilt when either changes)
    std::vector<uint32_t> h_bi, h_bj, h_aa, h_ab, h_ac;
    std::vector<double> h_bk, h_br, h_ak, h_at;
    std::vector<uint8_t> h_bs;
    // flags
    bool has_mol = false, have_sorted = false, have_table = false, tiled = true, joined = false;
    bool multi = false;  // n_species > 1: species packed into pos4.w bits 28-31
    bool no_fuse = false;  // DPDB_FUSE=0: keep the Verlet pass a separate kernel (A/B)
    // range builder: flat pair lists grouped by partner line; DPDB_BUCKET=0
    // keeps the row order (A/B)
    bool bucket_lists = true;
    uint32_t num_sms = 148;   // multiprocessors of the device
    // per-step thermo (dpdb_step_thermo): block partials of the phase-2 pass
    // and the records, written by the device straight into mapped pinned memory
    double* thermo_part{};
    // dpdb_step_thermo: the one-CTA record fold runs on th_stream, off the
    // step's critical path; the producers alternate between two partial
    // buffers (thermo_part <-> thermo_part2) so step s+1 never waits for it
    double* thermo_part2{};
    cudaStream_t th_stream = nullptr;
    cudaEvent_t th_prod[2]{}, th_cons[2]{};
    int th_idx = 0;
    double *thermo_host{}, *thermo_host_dev{};
    size_t thermo_cap = 0;  // records
    int64_t step = 0;
    std::string last_error;
    // stage timing
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<int> ev_stage;
    size_t ev_used = 0;
    int64_t launches[ST_N]{};
    // brick decomposition (domain_host.inc); single domain: dims = 1
    int dims[3]{1, 1, 1}, coords[3]{};
    uint32_t md_valid = 0;     // bit d: a neighbor brick exists in direction d
    double md_shift[26][3]{};  // periodic image shift of ghosts sent in direction d
    size_t ng = 0;             // ghosts at [n, n + ng)
    uint32_t *md_masks{}, *md_mig{}, *md_mlist{}, *md_glist{}, *md_slot{}, *md_doff{}, *md_dbase{};
    size_t md_list_cap = 0;
    uint32_t md_moff[27]{}, md_goff[27]{};
    uint32_t md_n_out = 0, md_n_all = 0;
    bool md_in_rebuild = false, md_pending_p2 = false;
    bool md_integrated = false;  // the next step's Verlet pass already ran in the force epilogue
    // brick per-step thermo: record base (device-visible) and the step of record 0
    double* md_rec = nullptr;
    int64_t md_rec_step0 = 0, md_rec_n = 0;
    std::array<int32_t, 26> md_gcnt{};  // ghosts this brick sends per direction
    std::array<int32_t, 26> md_rcnt{};  // ghosts it receives per direction
    void *md_sbuf{}, *md_rbuf{};         // packed records out / in (device)
    size_t md_scap = 0, md_rcap = 0;
    // NCCL transport (one brick per process)
    void* nccl_comm = nullptr;
    int nccl_rank = -1, nccl_size = 0;
    bool nccl_mock = false;  // attached to the in-process NCCL stand-in (tests)
    int md_peer[26]{};
    int32_t *md_dcnt{}, *md_hcnt{};      // device / pinned count exchange
    double *md_dsum{}, *md_hsum{};       // device / pinned thermo exchange
};

namespace {

int md_dirs(const dpdb_ctx* ctx, int d, int nb[3]);  // domain_host.inc
void md_release(dpdb_ctx* ctx);                      // domain_host.inc

int fail(dpdb_ctx* ctx, int code, const std::string& msg) {
    if (ctx)
        ctx->last_error = msg;
    else
        g_thread_err = msg;
    return code;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(ctx, DPDB_EDEVICE, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define CKL()                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = cudaGetLastError();                                                  \
        if (e_ != cudaSuccess)                                                                \
            return fail(ctx, DPDB_EDEVICE, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
    } while (0)

#define TRY(...)                    \
    do {                            \
        int rc_ = (__VA_ARGS__);    \
        if (rc_) return rc_;        \
    } while (0)

inline unsigned blocks_for(size_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

template <class T>
int dalloc(dpdb_ctx* ctx, T*& p, size_t count) {
    CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    return 0;
}

int check_device(dpdb_ctx* ctx) {
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->th_stream) CK(cudaStreamSynchronize(ctx->th_stream));
    DevErr e{};
    CK(cudaMemcpy(&e, ctx->err, sizeof e, cudaMemcpyDeviceToHost));
    if (!e.code) return 0;
    CK(cudaMemset(ctx->err, 0, sizeof(DevErr)));
    std::string msg;
    switch (e.what) {
        case dpdb::EW_NONFINITE:
            msg = "blow-up: non-finite or escaped particle, tag " + std::to_string(e.tag);
            break;
        case dpdb::EW_MIGRATION:
            msg = "particle outside its domain slab (missed migration), tag " + std::to_string(e.tag);
            break;
        case dpdb::EW_OVERFLOW:
            msg = "neighbor table: row overflow (max_neighbors=" + std::to_string(ctx->maxn) +
                  ", needed " + std::to_string(e.tag2) + ") for particle tag " + std::to_string(e.tag);
            break;
        case dpdb::EW_COINCIDENT:
            msg = "coincident particles, tags " + std::to_string(e.tag) + " and " + std::to_string(e.tag2);
            break;
        case dpdb::EW_BOND:
            msg = "bond " + std::to_string(e.tag) + "-" + std::to_string(e.tag2) + ": missing endpoint";
            break;
        case dpdb::EW_FENE:
            msg = "FENE bond " + std::to_string(e.tag) + "-" + std::to_string(e.tag2) +
                  ": stretched to or beyond its maximum extension R0";
            break;
        default:
            msg = "device error";
    }
    return fail(ctx, e.code, msg);
}

// Per-step record fold off the critical path: the record kernel runs on
// th_stream once the producer (force epilogue or k_integrate) has written its
// block partials; the next producer writes the other partial buffer, after the
// fold that last read it.
template <class Launch>
int thermo_fold(dpdb_ctx* ctx, Launch launch) {
    const int k = ctx->th_idx;
    CK(cudaEventRecord(ctx->th_prod[k], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->th_stream, ctx->th_prod[k], 0));
    launch(ctx->th_stream, ctx->thermo_part);
    CKL();
    CK(cudaEventRecord(ctx->th_cons[k], ctx->th_stream));
    ctx->launches[ST_OTHER]++;
    std::swap(ctx->thermo_part, ctx->thermo_part2);
    ctx->th_idx = k ^ 1;
    CK(cudaStreamWaitEvent(ctx->stream, ctx->th_cons[k ^ 1], 0));
    return 0;
}


void mark(dpdb_ctx* ctx, int stage) {
    if (!ctx->timing) return;
    if (ctx->ev_used == ctx->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->ev_pool.push_back(e);
        ctx->ev_stage.push_back(0);
    }
    cudaEventRecord(ctx->ev_pool[ctx->ev_used], ctx->stream);
    ctx->ev_stage[ctx->ev_used] = stage;
    ++ctx->ev_used;
}

dpdb::DevGrid dev_grid(const dpdb_ctx* ctx) {
    dpdb::DevGrid g{};
    const HostGrid& h = ctx->grid;
    for (int k = 0; k < 3; ++k) {
        g.slab_lo[k] = h.slab_lo[k];
        g.slab_hi[k] = h.slab_hi[k];
        g.inv_cell[k] = h.inv_cell[k];
        g.origin[k] = h.origin[k];
        g.cell_size[k] = h.cell_size[k];
        g.centre[k] = (h.slab_lo[k] + h.slab_hi[k]) / 2;
        g.ncell[k] = h.ncell[k];
        g.ncell_ext[k] = h.ncell_ext[k];
        g.ghost_lo[k] = h.ghost_lo[k];
    }
    g.sub_bits = h.sub_bits;
    g.rank_of_cell = ctx->rank_of_cell;
    return g;
}

dpdb::BoundaryArgs boundary(const dpdb_ctx* ctx) {
    dpdb::BoundaryArgs b{};
    for (int k = 0; k < 3; ++k) {
        b.lo[k] = ctx->box.lo[k];
        b.hi[k] = ctx->box.hi[k];
        b.L[k] = ctx->box.hi[k] - ctx->box.lo[k];
        b.periodic[k] = ctx->box.periodic[k];
        b.wall[k] = ctx->box.wall[k];
    }
    b.bounce_back = ctx->run.wall_mode == 1;
    return b;
}

// The pair-force frame (dpdb::PosQ, kernels.cuh): wrap axes map the slab
// [lo, lo + L) onto the whole int32 circle; other axes use the largest power
// of two that keeps |x - centre| <= L/2 + ghost layers + a margin in range.
// qs: length per quantum (fp32), what the force kernels multiply by.
dpdb::PosQ posq_frame(const dpdb_ctx* ctx, float qs[3]) {
    dpdb::PosQ q{};
    const HostGrid& g = ctx->grid;
    for (int k = 0; k < 3; ++k) {
        const double len = g.slab_hi[k] - g.slab_lo[k];
        q.wrap[k] = g.wrap[k] ? 1 : 0;
        if (q.wrap[k]) {
            q.org[k] = g.slab_lo[k];
            q.s[k] = 4294967296.0 / len;
            if (qs) qs[k] = (float)(len / 4294967296.0);
        } else {
            const double half = 0.5 * len + 2.0 * (ctx->params.r_c + ctx->run.skin) + 16.0;
            const int e = (int)std::floor(std::log2(2147483647.0 / half));
            q.org[k] = 0.5 * (g.slab_lo[k] + g.slab_hi[k]);
            q.s[k] = std::ldexp(1.0, e);
            if (qs) qs[k] = std::ldexp(1.0f, -e);
        }
    }
    return q;
}

// fp32 wrap lengths of the single-domain slab (wrapmode axes)
void wrap_lengths(const dpdb_ctx* ctx, float L[3], float H[3]) {
    for (int k = 0; k < 3; ++k) {
        const double len = ctx->grid.slab_hi[k] - ctx->grid.slab_lo[k];
        L[k] = (float)len;
        H[k] = (float)(0.5 * len);
    }
}

// defer_wrap (brick runs, non-rebuild steps): no periodic wrap on axes split
// across bricks -- a local that crosses the seam keeps its unwrapped
// coordinate (consistent with its neighbors and with the shifted ghost
// copies) until the next rebuild wraps and migrates it
dpdb::IntegrateArgs integrate_args(dpdb_ctx* ctx, bool defer_wrap) {
    dpdb::IntegrateArgs a{};
    for (int k = 0; k < 3; ++k) {
        a.x[k] = ctx->x[k];
        a.v[k] = ctx->v[k];
        a.f[k] = ctx->f[k];
    }
    a.tag = ctx->tag;
    a.sp = ctx->multi ? ctx->sp : nullptr;
    a.pos4 = ctx->pos4;
    a.posq = ctx->posq;
    a.vel4 = ctx->vel4;
    a.pq = posq_frame(ctx, nullptr);
    a.keys = ctx->keys;
    a.vals = ctx->vals;
    a.err = ctx->err;
    a.bnd = boundary(ctx);
    if (defer_wrap)
        for (int k = 0; k < 3; ++k)
            if (ctx->dims[k] > 1) a.bnd.periodic[k] = 0;  // walls still reflect
    a.grid = dev_grid(ctx);
    a.dt = ctx->params.dt;
    a.h = 0.5 * ctx->params.dt;
    a.n = (uint32_t)ctx->n;
    return a;
}

template <bool P2, bool P1, bool KEYS, bool STREAMS>
int launch_integrate(dpdb_ctx* ctx, bool defer_wrap = false, bool thermo = false) {
    if (!ctx->n) return 0;
    dpdb::IntegrateArgs a = integrate_args(ctx, defer_wrap);
    if (P2 && thermo) a.thermo_part = ctx->thermo_part;
    dpdb::k_integrate<P2, P1, KEYS, STREAMS><<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(a);
    CKL();
    ctx->launches[ST_INTEGRATE]++;
    return 0;
}

constexpr size_t THERMO_RING = 4096;  // records preallocated per context

// onesweep LSD radix sort (kernels.cuh): one histogram pass for every digit,
// then one binning kernel per 8-bit digit with decoupled look-back
int radix_sort_on(dpdb_ctx* ctx, cudaStream_t st, uint32_t*& k, uint32_t*& v, uint32_t*& k2,
                  uint32_t*& v2, uint32_t* work, size_t n, int bits) {
    if (n == 0 || bits == 0) return 0;
    const uint32_t tiles = (uint32_t)((n + dpdb::OS_TILE - 1) / dpdb::OS_TILE);
    const int passes = (bits + 7) / 8;
    CK(cudaMemsetAsync(work, 0, dpdb::onesweep_work_words(n) * 4, st));
    uint32_t* ghist = work + (size_t)4 * tiles * 256;
    uint32_t* counters = ghist + 4 * 256;
    dpdb::k_onesweep_hist<<<std::min<uint32_t>(tiles, 4 * 148), 256, 0, st>>>(k, (uint32_t)n, passes, ghist);
    for (int p = 0; p < passes; ++p) {
        const int width = std::min(8, bits - 8 * p);
        dpdb::k_onesweep<<<tiles, dpdb::OS_THREADS, 0, st>>>(k, v, k2, v2, (uint32_t)n, 8 * p, (1u << width) - 1u,
                                                             ghist + 256 * p, work + (size_t)p * tiles * 256,
                                                             counters + p);
        std::swap(k, k2);
        std::swap(v, v2);
    }
    CKL();
    if (ctx) ctx->launches[ST_SORT] += 1 + passes;
    return 0;
}

int do_sort(dpdb_ctx* ctx) {
    return radix_sort_on(ctx, ctx->stream, ctx->keys, ctx->vals, ctx->keys2, ctx->vals2, ctx->rs_work,
                         ctx->n, ctx->grid.key_bits());
}

// index_of_tag refresh for bonds
__global__ void k_index_of_tag(const uint32_t* tag, uint32_t n, uint32_t* iot, uint32_t max_tag) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n && tag[t] <= max_tag) iot[tag[t]] = t;
}

int refresh_bond_index(dpdb_ctx* ctx) {
    if (!ctx->n_bonds || !ctx->n) return 0;
    CK(cudaMemsetAsync(ctx->index_of_tag, 0xFF, ((size_t)ctx->max_tag + 1) * 4, ctx->stream));
    k_index_of_tag<<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(ctx->tag, (uint32_t)ctx->n,
                                                                    ctx->index_of_tag, ctx->max_tag);
    CKL();
    ctx->launches[ST_OTHER]++;
    return 0;
}

int do_permute(dpdb_ctx* ctx, bool forces) {
    if (!ctx->n) {
        CK(cudaMemsetAsync(ctx->cell_start, 0, ((size_t)ctx->grid.n_total_cells + 1) * 4, ctx->stream));
        if (ctx->ostart)
            CK(cudaMemsetAsync(ctx->ostart, 0, ((size_t)ctx->grid.n_total_cells * 8 + 1) * 4, ctx->stream));
        ctx->have_sorted = true;
        return 0;
    }
    dpdb::PermuteArgs a{};
    for (int k = 0; k < 3; ++k) {
        a.xin[k] = ctx->x[k];
        a.vin[k] = ctx->v[k];
        a.xout[k] = ctx->x2[k];
        a.vout[k] = ctx->v2[k];
        a.fin[k] = ctx->f[k];
        a.fout[k] = ctx->f2[k];
        a.centre[k] = (ctx->grid.slab_lo[k] + ctx->grid.slab_hi[k]) / 2;
    }
    a.tag_in = ctx->tag;
    a.tag_out = ctx->tag2;
    a.sp_in = ctx->sp;
    a.sp_out = ctx->sp2;
    a.mol_in = ctx->mol;
    a.mol_out = ctx->mol2;
    a.order = ctx->vals;
    a.keys = ctx->keys;
    a.cell_start = ctx->cell_start;
    a.ostart = ctx->ostart;
    a.pos4 = ctx->pos4;
    a.posq = ctx->posq;
    a.vel4 = ctx->vel4;
    a.pq = posq_frame(ctx, nullptr);
    a.n = (uint32_t)ctx->n;
    a.n_total_cells = ctx->grid.n_total_cells;
    a.key_shift = 3 * ctx->grid.sub_bits;
    a.multi = ctx->multi;
    const unsigned nb = blocks_for(ctx->n, 256);
    if (forces && ctx->has_mol)
        dpdb::k_permute<true, true><<<nb, 256, 0, ctx->stream>>>(a);
    else if (forces)
        dpdb::k_permute<true, false><<<nb, 256, 0, ctx->stream>>>(a);
    else if (ctx->has_mol)
        dpdb::k_permute<false, true><<<nb, 256, 0, ctx->stream>>>(a);
    else
        dpdb::k_permute<false, false><<<nb, 256, 0, ctx->stream>>>(a);
    CKL();
    ctx->launches[ST_SORT]++;
    for (int k = 0; k < 3; ++k) {
        std::swap(ctx->x[k], ctx->x2[k]);
        std::swap(ctx->v[k], ctx->v2[k]);
        if (forces) std::swap(ctx->f[k], ctx->f2[k]);
    }
    std::swap(ctx->tag, ctx->tag2);
    std::swap(ctx->sp, ctx->sp2);
    if (ctx->has_mol) std::swap(ctx->mol, ctx->mol2);
    ctx->have_sorted = true;
    ctx->have_table = false;
    return refresh_bond_index(ctx);
}

size_t build_smem(const dpdb_ctx* ctx) {
    constexpr int P = 32 * BUILD_TILES;
    return BUILD_WARPS * 32 * sizeof(float4) + P * 4 + ((size_t)ctx->maxn + 1) * (P + 1) * 4 +
           BUILD_WARPS * 32 * 4;  // + per-thread trash words
}

int launch_build(dpdb_ctx* ctx, bool joined_out);

// The force kernel's per-tile flat pair lists from a walk layout's front entries
int do_compact(dpdb_ctx* ctx) {
    const unsigned tiles = (unsigned)((ctx->n + 31) / 32);
    dpdb::k_tile_compact<<<(tiles + dpdb::TC_WARPS - 1) / dpdb::TC_WARPS, dpdb::TC_WARPS * 32, 0, ctx->stream>>>(
        ctx->entries, ctx->fwalk, (uint32_t)ctx->n, ctx->maxn, ctx->plist);
    CKL();
    ctx->launches[ST_BUILD]++;
    return 0;
}

// joined_out: write rows already joined (core asc, skin asc) -- the step
// pipeline's layout; the per-stage API builds the reference's split layout.
int do_build(dpdb_ctx* ctx, bool joined_out) {
    TRY(launch_build(ctx, joined_out));
    // the range builder appends the flat lists itself; the lane / ballot walk
    // layouts are compacted from their tile-transposed rows
    if (ctx->walk && ctx->walk != 3 && ctx->n) TRY(do_compact(ctx));
    return 0;
}

int launch_build(dpdb_ctx* ctx, bool joined_out) {
    if (!ctx->have_sorted) return fail(ctx, DPDB_ECONFIG, "build_neighbor_table: particles not reordered");
    ctx->tiled = true;
    ctx->joined = joined_out;
    ctx->walk = joined_out ? (ctx->builder == 2 ? 3 : ctx->builder == 1 ? 2 : 1) : 0;
    ctx->have_table = true;
    if (!ctx->n) return 0;
    dpdb::BuildArgs a{};
    a.pos4 = ctx->pos4;
    a.keys = ctx->keys;
    a.cell_start = ctx->cell_start;
    a.ostart = ctx->ostart;
    a.stencil = ctx->stencil;
    a.stencil_n = ctx->stencil_n;
    a.cell_flags = ctx->cell_flags;
    a.entries = ctx->entries;
    a.counts = ctx->counts;
    a.fwalk = ctx->fwalk;
    a.rowmeta = ctx->rowmeta;
    a.plist = ctx->plist;
    a.force_block = dpdb::FORCE_BLOCK;
    a.bucket = ctx->bucket_lists ? 1 : 0;
    a.err = ctx->err;
    a.n_local = (uint32_t)ctx->n;
    a.maxn = ctx->maxn;
    a.n_local_cells = ctx->grid.n_local_cells;
    a.key_shift = 3 * ctx->grid.sub_bits;
    const double rc = ctx->params.r_c, rs = ctx->params.r_c + ctx->run.skin;
    a.cut_c = (float)(rc * rc);
    a.cut_s = (float)(rs * rs);
    wrap_lengths(ctx, a.L, a.H);
    if (ctx->builder == 2) {
        a.blk_ghost = ctx->blk_ghost;
        a.stencil_code = ctx->stencil_code;
        a.cell_lo = ctx->cell_lo;
        for (int k = 0; k < 3; ++k) a.csz[k] = (float)ctx->grid.cell_size[k];
        const double rm = rs + 1e-3;  // margin over the fp32 frame's rounding
        a.cut_cull = (float)(rm * rm);
        const unsigned nb = (unsigned)((ctx->n + dpdb::RB_BLOCK - 1) / dpdb::RB_BLOCK);
        // ghost rows exist only in a brick (ghost cell layers); otherwise the
        // per-candidate ghost-partner test is compiled out
        const bool gh = ctx->grid.n_total_cells > ctx->grid.n_local_cells;
        if (joined_out && gh)
            dpdb::k_build_range<true, true><<<nb, dpdb::RB_THREADS, dpdb::RB_SMEM, ctx->stream>>>(a);
        else if (joined_out)
            dpdb::k_build_range<true, false><<<nb, dpdb::RB_THREADS, dpdb::RB_SMEM, ctx->stream>>>(a);
        else if (gh)
            dpdb::k_build_range<false, true><<<nb, dpdb::RB_THREADS, dpdb::RB_SMEM, ctx->stream>>>(a);
        else
            dpdb::k_build_range<false, false><<<nb, dpdb::RB_THREADS, dpdb::RB_SMEM, ctx->stream>>>(a);
        CKL();
        ctx->launches[ST_BUILD]++;
        return 0;
    }
    // other builders do not flag ghost-partner blocks: mark every block
    // boundary so an interior/boundary split computes everything after the halo
    CK(cudaMemsetAsync(ctx->blk_ghost, 1, ctx->n / dpdb::FORCE_BLOCK + 1, ctx->stream));
    if (ctx->builder == 1) {
        if (joined_out)
            dpdb::k_build_lane<true><<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(a);
        else
            dpdb::k_build_lane<false><<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(a);
        CKL();
        ctx->launches[ST_BUILD]++;
        return 0;
    }
    constexpr int P = 32 * BUILD_TILES;
    const size_t smem = build_smem(ctx);
    if (joined_out)
        dpdb::k_build<BUILD_WARPS, BUILD_TILES, true>
            <<<blocks_for(ctx->n, P), BUILD_WARPS * 32, smem, ctx->stream>>>(a);
    else
        dpdb::k_build<BUILD_WARPS, BUILD_TILES, false>
            <<<blocks_for(ctx->n, P), BUILD_WARPS * 32, smem, ctx->stream>>>(a);
    CKL();
    ctx->launches[ST_BUILD]++;
    return 0;
}

int do_streams(dpdb_ctx* ctx, uint32_t* sig_out) {
    if (!ctx->n) return 0;
    const HostGrid& g = ctx->grid;
    dpdb::k_streams<<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(
        ctx->x[0], ctx->x[1], ctx->x[2], ctx->v[0], ctx->v[1], ctx->v[2], ctx->tag,
        ctx->multi ? ctx->sp : nullptr, ctx->pos4, ctx->posq, ctx->vel4, sig_out,
        (g.slab_lo[0] + g.slab_hi[0]) / 2, (g.slab_lo[1] + g.slab_hi[1]) / 2, (g.slab_lo[2] + g.slab_hi[2]) / 2,
        posq_frame(ctx, nullptr), (uint32_t)ctx->n);
    CKL();
    ctx->launches[ST_OTHER]++;
    return 0;
}

template <bool MULTI, bool TILED, bool JOINED, bool WALK = false>
void force_launch(dpdb_ctx* ctx, const dpdb::ForceArgs& a, bool body) {
    const unsigned nb = blocks_for(ctx->n, dpdb::FORCE_BLOCK);
    constexpr int T = dpdb::FORCE_WARPS * 32;
    if (body)
        dpdb::k_force<MULTI, TILED, JOINED, true, WALK><<<nb, T, 0, ctx->stream>>>(a);
    else
        dpdb::k_force<MULTI, TILED, JOINED, false, WALK><<<nb, T, 0, ctx->stream>>>(a);
}

template <bool MULTI, bool BODY>
void force_walk_launch(dpdb_ctx* ctx, const dpdb::ForceArgs& a, int fuse) {
    const unsigned nb = blocks_for(ctx->n, dpdb::FORCE_BLOCK);
    constexpr int T = dpdb::FORCE_WARPS * 32;
    if (fuse == dpdb::FUSE_STREAMS)  // fused variants: maxn == 128 only (can_fuse)
        dpdb::k_force_walk<MULTI, BODY, 128, dpdb::FUSE_STREAMS><<<nb, T, 0, ctx->stream>>>(a);
    else if (fuse == dpdb::FUSE_KEYS)
        dpdb::k_force_walk<MULTI, BODY, 128, dpdb::FUSE_KEYS><<<nb, T, 0, ctx->stream>>>(a);
    else if (ctx->maxn == 128)
        dpdb::k_force_walk<MULTI, BODY, 128, dpdb::FUSE_NONE><<<nb, T, 0, ctx->stream>>>(a);
    else
        dpdb::k_force_walk<MULTI, BODY, 0, dpdb::FUSE_NONE><<<nb, T, 0, ctx->stream>>>(a);
}

template <bool MULTI>
void force_dispatch_layout(dpdb_ctx* ctx, const dpdb::ForceArgs& a, bool body, int fuse) {
    if (ctx->walk) {
        if (body) force_walk_launch<MULTI, true>(ctx, a, fuse);
        else force_walk_launch<MULTI, false>(ctx, a, fuse);
    }
    else if (ctx->tiled && !ctx->joined) force_launch<MULTI, true, false>(ctx, a, body);
    else if (ctx->tiled) force_launch<MULTI, true, true>(ctx, a, body);
    else if (!ctx->joined) force_launch<MULTI, false, false>(ctx, a, body);
    else force_launch<MULTI, false, true>(ctx, a, body);
}

// Whether the step loop may run the next Verlet pass inside the force kernel:
// single domain, walk layout with 128-slot rows (the walk kernel adds the
// bonded terms -- harmonic / FENE bonds and harmonic angles -- in its
// epilogue, so bonded systems fuse too).
bool can_fuse(const dpdb_ctx* ctx) {
    return ctx->walk && ctx->maxn == 128 && !ctx->md_valid &&
           ctx->dims[0] * ctx->dims[1] * ctx->dims[2] == 1 && !ctx->no_fuse;
}

// fuse (step loop only, can_fuse): FUSE_STREAMS / FUSE_KEYS run phase 2 of
// this step + phase 1 of the next in the force kernel's epilogue; the forces
// themselves are then not stored.
dpdb::BondArgs bond_args(dpdb_ctx* ctx) {
    dpdb::BondArgs b{};
    b.boff = ctx->bond_off;
    b.bpartner = ctx->bond_partner;
    b.bk = ctx->bond_k;
    b.br0 = ctx->bond_r0;
    b.bstyle = ctx->bond_style;
    b.aoff = ctx->ang_off;
    b.arec = ctx->ang_rec;
    b.ak = ctx->ang_k;
    b.at0 = ctx->ang_t0;
    b.index_of_tag = ctx->index_of_tag;
    b.posq = ctx->posq;
    for (int k = 0; k < 3; ++k) b.f[k] = ctx->f[k];
    posq_frame(ctx, b.qs);
    b.err = ctx->err;
    b.n = (uint32_t)ctx->n;
    b.max_tag = ctx->max_tag;
    b.tag_mask = ctx->multi ? 0x0FFFFFFFu : 0xFFFFFFFFu;
    return b;
}

// part (bricks, walk layout): -1 every block; 0 the interior blocks (no ghost
// partner: they can run while the ghost update is in flight); 1 the rest
int do_forces(dpdb_ctx* ctx, uint32_t step, int fuse = dpdb::FUSE_NONE, bool thermo = false,
              int part = -1, bool defer_wrap = false) {
    if (!ctx->have_table) return fail(ctx, DPDB_ECONFIG, "compute_forces: neighbor table not built");
    if (!ctx->n) return 0;
    const dpdb_params& p = ctx->params;
    dpdb::ForceArgs a{};
    a.posq = ctx->posq;
    a.vel4 = ctx->vel4;
    a.entries = ctx->entries;
    a.counts = ctx->counts;
    a.fwalk = ctx->fwalk;
    a.plist = ctx->plist;
    a.xpart = ctx->x[ctx->run.partition_axis];
    for (int k = 0; k < 3; ++k) a.f[k] = ctx->f[k];
    a.err = ctx->err;
    a.n = (uint32_t)ctx->n;
    a.maxn = ctx->maxn;
    a.step_mix = dpdb::step_mix_of(ctx->run.seed, step);
    a.rc2 = (float)(p.r_c * p.r_c);
    a.inv_rc = (float)(1.0 / p.r_c);
    a.a = (float)p.a[0];
    a.gamma = (float)p.gamma[0];
    a.sigma_dt = (float)(ctx->sigma[0] / std::sqrt(p.dt));
    posq_frame(ctx, a.qs);
    for (int k = 0; k < 3; ++k) {
        a.xd[k] = ctx->x[k];
        const double len = ctx->grid.slab_hi[k] - ctx->grid.slab_lo[k];
        a.Lw[k] = ctx->grid.wrap[k] ? len : 0.0;
        a.iLw[k] = ctx->grid.wrap[k] ? 1.0 / len : 0.0;
    }
    const bool body = ctx->run.body_force != 0.0;
    a.body_g = (float)ctx->run.body_force;
    a.drive_axis = ctx->run.drive_axis;
    const int pa = ctx->run.partition_axis;
    a.body_mid64 = 0.5 * (ctx->box.lo[pa] + ctx->box.hi[pa]);
    a.s_exp = (float)p.s;
    a.smode = p.s == 1.0 ? 1 : p.s == 2.0 ? 2 : p.s == 3.0 ? 3 : 0;  // S:428, integer s bypass
    a.ns = (uint32_t)p.n_species;
    for (int q = 0; q < p.n_species * p.n_species; ++q) {
        a.ta[q] = (float)p.a[q];
        a.tg[q] = (float)p.gamma[q];
        a.ts[q] = (float)(ctx->sigma[q] / std::sqrt(p.dt));
    }
    // bonded terms ride in the walk kernel's epilogue; the reference-layout kernel needs k_bonds
    const bool bonds_after = ctx->n_bonds && !ctx->walk;
    if (ctx->n_bonds && !bonds_after) {
        a.has_bonds = 1;
        a.bd = bond_args(ctx);
    }
    if (part >= 0) {
        a.blk_sel = ctx->blk_ghost;
        a.sel_val = (uint32_t)part;
    }
    if (fuse != dpdb::FUSE_NONE) {
        a.ia = integrate_args(ctx, defer_wrap);
        // x(n+1) goes to the second buffer: close pairs of other blocks read x(n)
        // through a.xd while this launch runs (the caller swaps x / x2 after it)
        for (int k = 0; k < 3; ++k) a.ia.x[k] = ctx->x2[k];
        if (thermo) a.ia.thermo_part = ctx->thermo_part;
        a.posqn = ctx->posqn;
        a.vel4n = ctx->vel4n;
    }
    if (ctx->multi || a.smode != 1 || a.has_bonds)  // bonds: in the GENERAL epilogue
        force_dispatch_layout<true>(ctx, a, body, fuse);
    else
        force_dispatch_layout<false>(ctx, a, body, fuse);
    CKL();
    ctx->launches[ST_FORCE]++;
    if (bonds_after && part != 0) {  // split force pass: once, after the boundary part
        dpdb::BondArgs b = bond_args(ctx);
        dpdb::k_bonds<<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(b);
        CKL();
        ctx->launches[ST_FORCE]++;
    }
    return 0;
}

int do_reorder_all(dpdb_ctx* ctx, bool forces) {
    TRY(launch_integrate<false, false, true, false>(ctx));
    TRY(do_sort(ctx));
    return do_permute(ctx, forces);
}

int require_ctx(const dpdb_ctx* ctx) {
    if (!ctx) return fail(nullptr, DPDB_ECONFIG, "null context");
    return 0;
}

// Runs body() between two events on the context stream; stage_ms[0..5]
// from the mark() events body records (the time since the previous mark goes
// to the stage the mark names), stage_launches from the launch counters.
template <class F>
int timed_run(dpdb_ctx* ctx, F&& body, double* ms, double* stage_ms, int64_t* stage_launches) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int s = 0; s < ST_N; ++s) ctx->launches[s] = 0;
    ctx->timing = stage_ms != nullptr;
    ctx->ev_used = 0;
    CK(cudaEventRecord(e0, ctx->stream));
    const int rc = body();
    cudaEventRecord(e1, ctx->stream);
    ctx->timing = false;
    if (rc) return rc;
    TRY(check_device(ctx));
    float total = 0;
    CK(cudaEventElapsedTime(&total, e0, e1));
    if (ms) *ms = total;
    if (stage_ms) {
        for (int s = 0; s <= ST_N; ++s) stage_ms[s] = 0;
        cudaEvent_t prev = e0;
        for (size_t q = 0; q < ctx->ev_used; ++q) {
            float d = 0;
            cudaEventElapsedTime(&d, prev, ctx->ev_pool[q]);
            stage_ms[ctx->ev_stage[q]] += d;
            prev = ctx->ev_pool[q];
        }
        stage_ms[ST_N] = total;
    }
    if (stage_launches) {
        int64_t tot = 0;
        for (int s = 0; s < ST_N; ++s) {
            stage_launches[s] = ctx->launches[s];
            tot += ctx->launches[s];
        }
        stage_launches[ST_N] = tot;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return 0;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

const char* dpdb_version(void) { return "dpdb 0.1 (sm_100a)"; }

const char* dpdb_last_error(const dpdb_ctx* ctx) {
    return ctx ? ctx->last_error.c_str() : g_thread_err.c_str();
}

int dpdb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return -1;
    int ok = 0;
    for (int d = 0; d < n; ++d) {
        cudaDeviceProp p;
        if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++ok;
    }
    return ok;
}

int dpdb_create(int device, const dpdb_box* box, const dpdb_params* params, const dpdb_run* run,
                size_t capacity, dpdb_ctx** out) {
    dpdb_ctx* ctx = nullptr;
    if (!out || !box || !params || !run) return fail(nullptr, DPDB_ECONFIG, "null argument");
    *out = nullptr;
    // validation mirrors SimBox::validate, PairParams::make, RunConfig::validate
    for (int k = 0; k < 3; ++k) {
        if (!(box->hi[k] > box->lo[k]))
            return fail(nullptr, DPDB_ECONFIG, "box: hi must exceed lo on axis " + std::to_string(k));
        if (box->periodic[k] && box->wall[k])
            return fail(nullptr, DPDB_ECONFIG, "box: axis cannot be periodic and walled");
    }
    if (!(params->r_c > 0)) return fail(nullptr, DPDB_ECONFIG, "pair params: r_c must be positive");
    if (!(params->s > 0)) return fail(nullptr, DPDB_ECONFIG, "pair params: weight exponent s must be positive");
    if (params->n_species < 1 || params->n_species > 4)
        return fail(nullptr, DPDB_ECONFIG, "pair params: 1..4 species supported");
    const int ns = params->n_species;
    for (int i = 0; i < ns; ++i)
        for (int j = 0; j < i; ++j)
            if (params->a[i * ns + j] != params->a[j * ns + i] ||
                params->gamma[i * ns + j] != params->gamma[j * ns + i])
                return fail(nullptr, DPDB_ECONFIG, "pair params: matrices must be symmetric");
    if (run->rebuild_every < 1) return fail(nullptr, DPDB_ECONFIG, "run: rebuild interval must be >= 1");
    if (!(run->skin >= 0)) return fail(nullptr, DPDB_ECONFIG, "run: skin distance must be >= 0");
    if (capacity > (size_t(1) << 26))
        return fail(nullptr, DPDB_ECONFIG, "capacity: at most 2^26 particles per device context");
    if (run->max_neighbors == 0 || run->max_neighbors % 32 || run->max_neighbors > 4096)
        return fail(nullptr, DPDB_ECONFIG, "run: max_neighbors must be a multiple of 32 in [32, 4096]");
    if (run->wall_mode != 0 && run->wall_mode != 1)
        return fail(nullptr, DPDB_ECONFIG, "run: wall_mode must be 0 (specular) or 1 (bounce-back)");
    if (run->drive_axis < 0 || run->drive_axis > 2 || run->partition_axis < 0 || run->partition_axis > 2)
        return fail(nullptr, DPDB_ECONFIG, "run: axes must be 0, 1 or 2");
    ctx = new dpdb_ctx();
    ctx->device = device;
    ctx->box = *box;
    ctx->params = *params;
    ctx->run = *run;
    ctx->maxn = run->max_neighbors;
    if (const char* b = std::getenv("DPDB_BUILDER"))
        ctx->builder = !std::strcmp(b, "ballot") ? 0 : !std::strcmp(b, "lane") ? 1 : 2;
    ctx->multi = params->n_species > 1;
    if (const char* f = std::getenv("DPDB_FUSE")) ctx->no_fuse = std::strcmp(f, "0") == 0;
    if (const char* f = std::getenv("DPDB_BUCKET")) ctx->bucket_lists = std::strcmp(f, "0") != 0;
    {
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
            ctx->num_sms = (uint32_t)sms;
    }
    for (int q = 0; q < ns * ns; ++q) ctx->sigma[q] = std::sqrt(2.0 * params->gamma[q] * params->kbt);
    std::string err;
    // brick geometry (decompose): uniform half-open slabs
    double slo[3], shi[3];
    for (int k = 0; k < 3; ++k) {
        ctx->dims[k] = g_pending_dims ? g_pending_dims[k] : 1;
        ctx->coords[k] = g_pending_coords ? g_pending_coords[k] : 0;
        const double len = (box->hi[k] - box->lo[k]) / ctx->dims[k];
        slo[k] = box->lo[k] + ctx->coords[k] * len;
        shi[k] = ctx->coords[k] == ctx->dims[k] - 1 ? box->hi[k] : box->lo[k] + (ctx->coords[k] + 1) * len;
    }
    int rc = ctx->grid.make(*box, slo, shi, ctx->dims, ctx->coords, params->r_c + run->skin,
                            run->sub_bits, err);
    for (int d = 0; d < 26; ++d) {
        int nb[3], off[3];
        if (!md_dirs(ctx, d, nb)) continue;
        ctx->md_valid |= 1u << d;
        dpdb::dir_offset(d, off);
        for (int k = 0; k < 3; ++k) {
            const int c = ctx->coords[k] + off[k];
            const double L = box->hi[k] - box->lo[k];
            ctx->md_shift[d][k] = c >= ctx->dims[k] ? -L : (c < 0 ? L : 0.0);
        }
    }
    if (rc) {
        fail(nullptr, rc, err);
        delete ctx;
        return rc;
    }
    {
        int ndev = 0;
        cudaDeviceProp prop;
        const char* why = nullptr;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
            why = "no CUDA device (the engine has no CPU fallback)";
        else if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10)
            why = "device is not compute capability 10.x (sm_100a build)";
        if (why) {
            fail(nullptr, DPDB_EDEVICE, std::string(why) + ", device " + std::to_string(device));
            delete ctx;
            return DPDB_EDEVICE;
        }
    }
    auto bail = [&](int code) {
        g_thread_err = ctx->last_error;
        dpdb_destroy(ctx);
        return code;
    };
    if (cudaSetDevice(device) != cudaSuccess) return bail(fail(ctx, DPDB_EDEVICE, "cudaSetDevice"));
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->halo_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_pack, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->th_stream, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(ctx, DPDB_EDEVICE, "cudaStreamCreate"));
    for (int k = 0; k < 2; ++k)
        if (cudaEventCreateWithFlags(&ctx->th_prod[k], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->th_cons[k], cudaEventDisableTiming) != cudaSuccess)
            return bail(fail(ctx, DPDB_EDEVICE, "cudaEventCreate"));
    ctx->cap = std::max<size_t>(capacity, 1);
    ctx->n_pad = (ctx->cap + 31) & ~(size_t)31;
    const size_t c = ctx->n_pad;
    const HostGrid& g = ctx->grid;
    for (int k = 0; k < 3; ++k) {
        if ((rc = dalloc(ctx, ctx->x[k], c)) || (rc = dalloc(ctx, ctx->v[k], c)) ||
            (rc = dalloc(ctx, ctx->x2[k], c)) || (rc = dalloc(ctx, ctx->v2[k], c)) ||
            (rc = dalloc(ctx, ctx->f[k], c)) || (rc = dalloc(ctx, ctx->f2[k], c)))
            return bail(rc);
    }
    const uint32_t tiles = (uint32_t)((c + dpdb::RS_TILE - 1) / dpdb::RS_TILE);
    if ((rc = dalloc(ctx, ctx->tag, c)) || (rc = dalloc(ctx, ctx->tag2, c)) ||
        (rc = dalloc(ctx, ctx->sp, c)) || (rc = dalloc(ctx, ctx->sp2, c)) ||
        (rc = dalloc(ctx, ctx->mol, c)) || (rc = dalloc(ctx, ctx->mol2, c)) ||
        (rc = dalloc(ctx, ctx->pos4, c)) || (rc = dalloc(ctx, ctx->vel4, c)) ||
        (rc = dalloc(ctx, ctx->posq, c)) || (rc = dalloc(ctx, ctx->posqn, c)) ||
        (rc = dalloc(ctx, ctx->vel4n, c)) ||
        (rc = dalloc(ctx, ctx->keys, c)) || (rc = dalloc(ctx, ctx->keys2, c)) ||
        (rc = dalloc(ctx, ctx->vals, c)) || (rc = dalloc(ctx, ctx->vals2, c)) ||
        (rc = dalloc(ctx, ctx->rs_work, dpdb::onesweep_work_words(c))) ||
        (rc = dalloc(ctx, ctx->hist, std::max<size_t>((size_t)256 * tiles + 256,
                                                      26 * (c / dpdb::MD_THREADS + 1) + 64))) ||
        (rc = dalloc(ctx, ctx->cell_start, (size_t)g.n_total_cells + 1)) ||
        (g.sub_bits >= 1 && (rc = dalloc(ctx, ctx->ostart, (size_t)g.n_total_cells * 8 + 1))) ||
        (rc = dalloc(ctx, ctx->rank_of_cell, (size_t)g.n_total_cells)) ||
        (rc = dalloc(ctx, ctx->stencil, (size_t)g.n_local_cells * 32)) ||
        (rc = dalloc(ctx, ctx->stencil_n, (size_t)g.n_local_cells)) ||
        (rc = dalloc(ctx, ctx->cell_flags, (size_t)g.n_local_cells)) ||
        (rc = dalloc(ctx, ctx->stencil_code, (size_t)g.n_local_cells * 32)) ||
        (rc = dalloc(ctx, ctx->cell_lo, (size_t)g.n_local_cells)) ||
        (rc = dalloc(ctx, ctx->entries, c * ctx->maxn)) || (rc = dalloc(ctx, ctx->counts, c)) ||
        (rc = dalloc(ctx, ctx->plist, c * ctx->maxn + 512)) ||
        (rc = dalloc(ctx, ctx->fwalk, c)) || (rc = dalloc(ctx, ctx->rowmeta, c)) ||
        (rc = dalloc(ctx, ctx->md_masks, c)) || (rc = dalloc(ctx, ctx->md_mig, c)) ||
        (rc = dalloc(ctx, ctx->md_slot, c)) || (rc = dalloc(ctx, ctx->md_doff, 64)) ||
        (rc = dalloc(ctx, ctx->md_dbase, 32)) ||
        (rc = dalloc(ctx, ctx->md_mlist, ctx->md_valid ? 8 * c : 1)) ||
        (rc = dalloc(ctx, ctx->md_glist, ctx->md_valid ? 8 * c : 1)) ||
        (rc = dalloc(ctx, ctx->err, 1)) || (rc = dalloc(ctx, ctx->red, (size_t)RED_BLOCKS * 4)) ||
        (rc = dalloc(ctx, ctx->red_out, 16)) || (rc = dalloc(ctx, ctx->tmp_u32, c)) ||
        (rc = dalloc(ctx, ctx->thermo_part, 4 * (c / 256 + 1))) ||
        (rc = dalloc(ctx, ctx->thermo_part2, 4 * (c / 256 + 1))) ||
        (rc = dalloc(ctx, ctx->blk_ghost, c / dpdb::FORCE_BLOCK + 1)))
        return bail(rc);
    ctx->md_list_cap = ctx->md_valid ? 8 * c : 1;  // a corner particle sits in 7 lists
    if (cudaHostAlloc(reinterpret_cast<void**>(&ctx->err_host), sizeof(DevErr), cudaHostAllocDefault) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->err_ev, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(ctx, DPDB_EDEVICE, "error-poll buffer"));
    std::memset(ctx->err_host, 0, sizeof(DevErr));
    if (cudaMemset(ctx->err, 0, sizeof(DevErr)) != cudaSuccess ||
        cudaMemset(ctx->counts, 0, c * 4) != cudaSuccess ||
        // k_force_walk reads rows past their end (masked): every word must be
        // a valid particle index from the start
        cudaMemset(ctx->entries, 0, c * ctx->maxn * 4) != cudaSuccess ||
        // and so does its phase A on the flat pair lists (prefetch past a tile's list end)
        cudaMemset(ctx->plist, 0, (c * ctx->maxn + 512) * 4) != cudaSuccess ||
        cudaMemset(ctx->sp, 0, c) != cudaSuccess || cudaMemset(ctx->sp2, 0, c) != cudaSuccess ||
        cudaMemset(ctx->f[0], 0, c * 4) != cudaSuccess || cudaMemset(ctx->f[1], 0, c * 4) != cudaSuccess ||
        cudaMemset(ctx->f[2], 0, c * 4) != cudaSuccess)
        return bail(fail(ctx, DPDB_EDEVICE, "cudaMemset"));
    std::vector<uint32_t> rows;
    std::vector<uint8_t> cnt, flags, codes;
    std::vector<float> clo;
    g.coarse_stencil(rows, cnt, flags, &codes, &clo);
    if (cudaMemcpy(ctx->stencil_code, codes.data(), codes.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(ctx->cell_lo, clo.data(), clo.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(ctx->rank_of_cell, g.rank_of_cell.data(), g.rank_of_cell.size() * 4,
                   cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(ctx->stencil, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(ctx->stencil_n, cnt.data(), cnt.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(ctx->cell_flags, flags.data(), flags.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return bail(fail(ctx, DPDB_EDEVICE, "upload of grid tables failed"));
    const size_t smem = build_smem(ctx);
    if (cudaFuncSetAttribute(dpdb::k_build<BUILD_WARPS, BUILD_TILES, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaFuncSetAttribute(dpdb::k_build<BUILD_WARPS, BUILD_TILES, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return bail(fail(ctx, DPDB_ECONFIG, "max_neighbors too large for the builder's shared memory"));
    if (cudaFuncSetAttribute(dpdb::k_build_range<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dpdb::RB_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(dpdb::k_build_range<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dpdb::RB_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(dpdb::k_build_range<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dpdb::RB_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(dpdb::k_build_range<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dpdb::RB_SMEM) != cudaSuccess)
        return bail(fail(ctx, DPDB_EDEVICE, "range builder shared memory"));
    // per-step thermo records (dpdb_step_thermo): a mapped pinned ring sized
    // for typical calls, so no host allocation lands in a step call (larger
    // calls grow it once)
    if (cudaHostAlloc(reinterpret_cast<void**>(&ctx->thermo_host), THERMO_RING * 5 * sizeof(double),
                      cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->thermo_host_dev), ctx->thermo_host, 0) !=
            cudaSuccess)
        return bail(fail(ctx, DPDB_EDEVICE, "thermo record buffer"));
    ctx->thermo_cap = THERMO_RING;
    *out = ctx;
    return 0;
}

int dpdb_destroy(dpdb_ctx* ctx) {
    if (!ctx) return 0;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    md_release(ctx);
    void* ptrs[] = {ctx->tag, ctx->tag2, ctx->mol, ctx->mol2, ctx->sp, ctx->sp2, ctx->pos4,
                    ctx->vel4, ctx->posq, ctx->posqn, ctx->vel4n, ctx->keys, ctx->keys2, ctx->vals, ctx->vals2, ctx->hist, ctx->rs_work,
                    ctx->cell_start, ctx->ostart, ctx->rank_of_cell, ctx->stencil, ctx->stencil_n,
                    ctx->cell_flags, ctx->stencil_code, ctx->cell_lo, ctx->entries, ctx->counts, ctx->fwalk, ctx->plist, ctx->rowmeta,
                    ctx->err, ctx->red, ctx->red_out, ctx->thermo_part, ctx->thermo_part2, ctx->blk_ghost, ctx->prof_acc,
                    ctx->tmp_u32, ctx->bond_off, ctx->bond_partner, ctx->index_of_tag,
                    ctx->bond_k, ctx->bond_r0, ctx->bond_style, ctx->ang_off, ctx->ang_rec, ctx->ang_k,
                    ctx->ang_t0, ctx->md_masks, ctx->md_mig, ctx->md_slot,
                    ctx->md_doff, ctx->md_dbase, ctx->md_mlist, ctx->md_glist};
    for (size_t q = 0; q < sizeof(ptrs) / sizeof(ptrs[0]); ++q)  // each buffer once
        if (ptrs[q] && std::find(ptrs, ptrs + q, ptrs[q]) == ptrs + q) cudaFree(ptrs[q]);
    if (ctx->thermo_host) cudaFreeHost(ctx->thermo_host);
    if (ctx->err_host) cudaFreeHost(ctx->err_host);
    if (ctx->err_ev) cudaEventDestroy(ctx->err_ev);
    for (int k = 0; k < 3; ++k) {
        void* q[] = {ctx->x[k], ctx->v[k], ctx->x2[k], ctx->v2[k], ctx->f[k], ctx->f2[k]};
        for (void* p : q)
            if (p) cudaFree(p);
    }
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->halo_stream) cudaStreamDestroy(ctx->halo_stream);
    if (ctx->ev_pack) cudaEventDestroy(ctx->ev_pack);
    if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
    if (ctx->th_stream) {
        cudaStreamSynchronize(ctx->th_stream);
        cudaStreamDestroy(ctx->th_stream);
    }
    for (int k = 0; k < 2; ++k) {
        if (ctx->th_prod[k]) cudaEventDestroy(ctx->th_prod[k]);
        if (ctx->th_cons[k]) cudaEventDestroy(ctx->th_cons[k]);
    }
    delete ctx;
    return 0;
}

int dpdb_grid(const dpdb_ctx* ctx, dpdb_grid_info* o) {
    TRY(require_ctx(ctx));
    const HostGrid& g = ctx->grid;
    for (int k = 0; k < 3; ++k) {
        o->ncell[k] = g.ncell[k];
        o->ncell_ext[k] = g.ncell_ext[k];
        o->wrapmode[k] = g.wrap[k];
        o->cell_size[k] = g.cell_size[k];
        o->inv_cell[k] = g.inv_cell[k];
        o->origin[k] = g.origin[k];
    }
    o->bits_per_axis = g.bits_per_axis;
    o->key_bits = g.key_bits();
    o->n_local_cells = g.n_local_cells;
    o->n_total_cells = g.n_total_cells;
    return 0;
}

int dpdb_grid_ranks(const dpdb_ctx* ctx, uint32_t* rank_of_cell) {
    TRY(require_ctx(ctx));
    std::memcpy(rank_of_cell, ctx->grid.rank_of_cell.data(), ctx->grid.rank_of_cell.size() * 4);
    return 0;
}

void* dpdb_stream(dpdb_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int dpdb_grid_plan(const dpdb_box* box, const double slab_lo[3], const double slab_hi[3],
                   const int32_t dims[3], const int32_t coords[3], double cell_target,
                   int32_t sub_bits, dpdb_grid_info* o, int32_t ghost_lo[3], int32_t ghost_hi[3],
                   uint32_t* rank_of_cell) {
    if (!box || !o) return fail(nullptr, DPDB_ECONFIG, "grid_plan: null argument");
    if (sub_bits < 0 || sub_bits > 4) return fail(nullptr, DPDB_ECONFIG, "grid_plan: sub_bits must be 0..4");
    const int one[3] = {1, 1, 1}, zero[3] = {0, 0, 0};
    int d3[3], c3[3];
    double lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
        d3[k] = dims ? dims[k] : one[k];
        c3[k] = coords ? coords[k] : zero[k];
        lo[k] = slab_lo ? slab_lo[k] : box->lo[k];
        hi[k] = slab_hi ? slab_hi[k] : box->hi[k];
        if (d3[k] < 1 || c3[k] < 0 || c3[k] >= d3[k])
            return fail(nullptr, DPDB_ECONFIG, "grid_plan: coords outside the decomposition");
    }
    HostGrid g;
    std::string err;
    const int rc = g.make(*box, lo, hi, d3, c3, cell_target, sub_bits, err);
    if (rc) return fail(nullptr, rc, err);
    for (int k = 0; k < 3; ++k) {
        o->ncell[k] = g.ncell[k];
        o->ncell_ext[k] = g.ncell_ext[k];
        o->wrapmode[k] = g.wrap[k];
        o->cell_size[k] = g.cell_size[k];
        o->inv_cell[k] = g.inv_cell[k];
        o->origin[k] = g.origin[k];
        if (ghost_lo) ghost_lo[k] = g.ghost_lo[k];
        if (ghost_hi) ghost_hi[k] = g.ghost_hi[k];
    }
    o->bits_per_axis = g.bits_per_axis;
    o->key_bits = g.key_bits();
    o->n_local_cells = g.n_local_cells;
    o->n_total_cells = g.n_total_cells;
    if (rank_of_cell) std::memcpy(rank_of_cell, g.rank_of_cell.data(), g.rank_of_cell.size() * 4);
    return 0;
}

int dpdb_upload(dpdb_ctx* ctx, size_t n, const double* x, const double* y, const double* z,
                const double* vx, const double* vy, const double* vz, const uint32_t* tag,
                const uint8_t* species, const uint32_t* molecule) {
    TRY(require_ctx(ctx));
    if (n > ctx->cap) return fail(ctx, DPDB_ECONFIG, "upload: n exceeds context capacity");
    if (n && (!x || !y || !z || !vx || !vy || !vz || !tag))
        return fail(ctx, DPDB_ECONFIG, "upload: null array");
    if (ctx->multi) {  // species share the tag word on the device (bits 28-31)
        for (size_t i = 0; i < n; ++i) {
            if (tag[i] >= (1u << 28))
                return fail(ctx, DPDB_ECONFIG, "upload: tags must be < 2^28 with several species");
            if (species && species[i] >= (uint32_t)ctx->params.n_species)
                return fail(ctx, DPDB_ECONFIG, "upload: species index out of range");
        }
    }
    CK(cudaSetDevice(ctx->device));
    const double* xs[3] = {x, y, z};
    const double* vs[3] = {vx, vy, vz};
    for (int k = 0; k < 3; ++k) {
        CK(cudaMemcpyAsync(ctx->x[k], xs[k], n * 8, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->v[k], vs[k], n * 8, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemsetAsync(ctx->f[k], 0, ctx->n_pad * 4, ctx->stream));
    }
    CK(cudaMemcpyAsync(ctx->tag, tag, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    if (species)
        CK(cudaMemcpyAsync(ctx->sp, species, n, cudaMemcpyHostToDevice, ctx->stream));
    else
        CK(cudaMemsetAsync(ctx->sp, 0, ctx->n_pad, ctx->stream));
    ctx->has_mol = molecule != nullptr;
    if (molecule) CK(cudaMemcpyAsync(ctx->mol, molecule, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    ctx->n = n;
    ctx->have_sorted = ctx->have_table = false;
    ctx->step = 0;
    TRY(refresh_bond_index(ctx));
    CK(cudaStreamSynchronize(ctx->stream));
    return 0;
}

int dpdb_init_random(dpdb_ctx* ctx, size_t n, double kbt, uint32_t seed, uint32_t n_chains,
                     uint32_t chain_len, const uint8_t* chain_species, uint8_t solvent_species,
                     double r0, double bond_k) {
    TRY(require_ctx(ctx));
    // init_random validation
    if (n == 0) return fail(ctx, DPDB_ECONFIG, "init_random: empty system (round(rho V) = 0)");
    if (n > ctx->cap) return fail(ctx, DPDB_ECONFIG, "init_random: n exceeds context capacity");
    if (n > 0x0FFFFFFFu / 6) return fail(ctx, DPDB_ECONFIG, "init_random: too many particles for the draw counter");
    if (!(kbt >= 0)) return fail(ctx, DPDB_ECONFIG, "init_random: kbt must be >= 0");
    if (n_chains && (chain_len < 2 || chain_len > 32 || !chain_species))
        return fail(ctx, DPDB_ECONFIG, "init_random: chains of 2..32 beads with a species per bead");
    if ((size_t)n_chains * chain_len > n) return fail(ctx, DPDB_ECONFIG, "init_random: chains exceed n");
    for (int k = 0; k < 3; ++k)
        if (n_chains && r0 * (chain_len - 1) >= ctx->box.hi[k] - ctx->box.lo[k] && !ctx->box.periodic[k])
            return fail(ctx, DPDB_ECONFIG, "init_random: chain longer than the box");
    const uint32_t ns = (uint32_t)ctx->params.n_species;
    if (solvent_species >= ns) return fail(ctx, DPDB_ECONFIG, "init_random: species index out of range");
    for (uint32_t b = 0; n_chains && b < chain_len; ++b)
        if (chain_species[b] >= ns) return fail(ctx, DPDB_ECONFIG, "init_random: species index out of range");
    CK(cudaSetDevice(ctx->device));
    dpdb::InitArgs a{};
    for (int k = 0; k < 3; ++k) {
        a.x[k] = ctx->x[k];
        a.v[k] = ctx->v[k];
        a.lo[k] = ctx->box.lo[k];
        a.hi[k] = ctx->box.hi[k];
        a.periodic[k] = ctx->box.periodic[k];
        CK(cudaMemsetAsync(ctx->f[k], 0, ctx->n_pad * 4, ctx->stream));
    }
    a.tag = ctx->tag;
    a.sp = ctx->sp;
    a.mol = n_chains ? ctx->mol : nullptr;
    a.sk = std::sqrt(kbt);
    a.seed = seed;
    a.n = (uint32_t)n;
    a.n_chains = n_chains;
    a.chain_len = n_chains ? chain_len : 1;
    for (uint32_t b = 0; n_chains && b < chain_len; ++b) a.chain_sp[b] = chain_species[b];
    a.solvent_sp = solvent_species;
    a.r0 = r0;
    CK(cudaMemsetAsync(ctx->sp, 0, ctx->n_pad, ctx->stream));
    dpdb::k_init_particles<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(a);
    CKL();
    if (n_chains) {
        dpdb::k_init_chains<<<(n_chains + 127) / 128, 128, 0, ctx->stream>>>(a);
        CKL();
    }
    dpdb::k_init_mean<<<1, 32, 0, ctx->stream>>>(a, ctx->red_out);
    dpdb::k_init_subtract<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(a, ctx->red_out);
    CKL();
    ctx->n = n;
    ctx->has_mol = n_chains > 0;
    ctx->have_sorted = ctx->have_table = false;
    ctx->step = 0;
    if (n_chains) {  // bonds along each chain (BondTopology)
        std::vector<uint32_t> ti, tj;
        std::vector<double> kk, rr;
        for (uint32_t c = 0; c < n_chains; ++c)
            for (uint32_t b = 0; b + 1 < chain_len; ++b) {
                const uint32_t t = c * chain_len + b + 1;  // tag = index + 1
                ti.push_back(t);
                tj.push_back(t + 1);
                kk.push_back(bond_k);
                rr.push_back(r0);
            }
        TRY(dpdb_set_bonds(ctx, ti.size(), ti.data(), tj.data(), kk.data(), rr.data()));
    } else {
        TRY(refresh_bond_index(ctx));
    }
    return check_device(ctx);
}

int dpdb_upload_forces(dpdb_ctx* ctx, const double* fx, const double* fy, const double* fz) {
    TRY(require_ctx(ctx));
    const double* fs[3] = {fx, fy, fz};
    std::vector<float> tmp(ctx->n);
    for (int k = 0; k < 3; ++k) {
        for (size_t i = 0; i < ctx->n; ++i) tmp[i] = (float)fs[k][i];
        CK(cudaMemcpy(ctx->f[k], tmp.data(), ctx->n * 4, cudaMemcpyHostToDevice));
    }
    return 0;
}

int dpdb_download(dpdb_ctx* ctx, double* x, double* y, double* z, double* vx, double* vy,
                  double* vz, double* fx, double* fy, double* fz, uint32_t* tag, uint8_t* species,
                  uint32_t* signature) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    const size_t n = ctx->n;
    double* xs[3] = {x, y, z};
    double* vs[3] = {vx, vy, vz};
    double* fs[3] = {fx, fy, fz};
    for (int k = 0; k < 3; ++k) {
        if (xs[k]) CK(cudaMemcpyAsync(xs[k], ctx->x[k], n * 8, cudaMemcpyDeviceToHost, ctx->stream));
        if (vs[k]) CK(cudaMemcpyAsync(vs[k], ctx->v[k], n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (tag) CK(cudaMemcpyAsync(tag, ctx->tag, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (species) CK(cudaMemcpyAsync(species, ctx->sp, n, cudaMemcpyDeviceToHost, ctx->stream));
    if (signature) {
        TRY(do_streams(ctx, ctx->tmp_u32));
        CK(cudaMemcpyAsync(signature, ctx->tmp_u32, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (fx || fy || fz) {
        std::vector<float> tmp(n);
        for (int k = 0; k < 3; ++k) {
            if (!fs[k]) continue;
            CK(cudaMemcpyAsync(tmp.data(), ctx->f[k], n * 4, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            for (size_t i = 0; i < n; ++i) fs[k][i] = tmp[i];
        }
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return 0;
}

int dpdb_size(const dpdb_ctx* ctx, size_t* n) {
    TRY(require_ctx(ctx));
    *n = ctx->n;
    return 0;
}

namespace {
// rebuild both bonded CSRs (bonds at both endpoints, angles at their three
// members) over tags 0..max_tag of either list, upload, refresh index_of_tag
int upload_bonded(dpdb_ctx* ctx) {
    void* old[] = {ctx->bond_off, ctx->bond_partner, ctx->index_of_tag, ctx->bond_k, ctx->bond_r0,
                   ctx->bond_style, ctx->ang_off, ctx->ang_rec, ctx->ang_k, ctx->ang_t0};
    for (void* p : old)
        if (p) cudaFree(p);
    ctx->bond_off = ctx->bond_partner = ctx->index_of_tag = ctx->ang_off = nullptr;
    ctx->bond_k = ctx->bond_r0 = ctx->ang_k = ctx->ang_t0 = nullptr;
    ctx->bond_style = nullptr;
    ctx->ang_rec = nullptr;
    const size_t nb = ctx->h_bi.size(), na = ctx->h_aa.size();
    ctx->n_bonds = nb + na;
    ctx->styled = na > 0;
    for (size_t q = 0; q < nb && !ctx->styled; ++q) ctx->styled = ctx->h_bs[q] != 0;
    if (!ctx->n_bonds) return 0;
    uint32_t max_tag = 0;
    for (size_t q = 0; q < nb; ++q) max_tag = std::max({max_tag, ctx->h_bi[q], ctx->h_bj[q]});
    for (size_t q = 0; q < na; ++q) max_tag = std::max({max_tag, ctx->h_aa[q], ctx->h_ab[q], ctx->h_ac[q]});
    ctx->max_tag = max_tag;
    // bonds: CSR by tag, each bond listed at both endpoints (full-list convention)
    std::vector<uint32_t> off((size_t)max_tag + 2, 0), partner(2 * nb);
    std::vector<float> kk(2 * nb), rr(2 * nb);
    std::vector<uint8_t> st(2 * nb);
    for (size_t q = 0; q < nb; ++q) {
        off[ctx->h_bi[q] + 1]++;
        off[ctx->h_bj[q] + 1]++;
    }
    for (size_t t = 1; t < off.size(); ++t) off[t] += off[t - 1];
    std::vector<uint32_t> fill(off.begin(), off.end() - 1);
    for (size_t q = 0; q < nb; ++q) {
        const uint32_t ends[2][2] = {{ctx->h_bi[q], ctx->h_bj[q]}, {ctx->h_bj[q], ctx->h_bi[q]}};
        for (auto& e : ends) {
            const uint32_t p = fill[e[0]]++;
            partner[p] = e[1];
            kk[p] = (float)ctx->h_bk[q];
            rr[p] = (float)ctx->h_br[q];
            st[p] = ctx->h_bs[q];
        }
    }
    // angles: CSR by tag, (other, other, role) at each member
    std::vector<uint32_t> aoff((size_t)max_tag + 2, 0);
    std::vector<uint4> arec(3 * na);
    std::vector<float> ak(3 * na), at(3 * na);
    for (size_t q = 0; q < na; ++q) {
        aoff[ctx->h_aa[q] + 1]++;
        aoff[ctx->h_ab[q] + 1]++;
        aoff[ctx->h_ac[q] + 1]++;
    }
    for (size_t t = 1; t < aoff.size(); ++t) aoff[t] += aoff[t - 1];
    std::vector<uint32_t> afill(aoff.begin(), aoff.end() - 1);
    for (size_t q = 0; q < na; ++q) {
        const uint32_t A = ctx->h_aa[q], B = ctx->h_ab[q], C = ctx->h_ac[q];
        const uint4 recs[3] = {make_uint4(B, C, 0u, 0u), make_uint4(A, C, 1u, 0u), make_uint4(B, A, 2u, 0u)};
        const uint32_t who[3] = {A, B, C};
        for (int r = 0; r < 3; ++r) {
            const uint32_t p = afill[who[r]]++;
            arec[p] = recs[r];
            ak[p] = (float)ctx->h_ak[q];
            at[p] = (float)ctx->h_at[q];
        }
    }
    int rc;
    if ((rc = dalloc(ctx, ctx->bond_off, off.size())) || (rc = dalloc(ctx, ctx->bond_partner, std::max<size_t>(2 * nb, 1))) ||
        (rc = dalloc(ctx, ctx->bond_k, std::max<size_t>(2 * nb, 1))) ||
        (rc = dalloc(ctx, ctx->bond_r0, std::max<size_t>(2 * nb, 1))) ||
        (rc = dalloc(ctx, ctx->bond_style, std::max<size_t>(2 * nb, 1))) ||
        (rc = dalloc(ctx, ctx->index_of_tag, (size_t)max_tag + 1)))
        return rc;
    CK(cudaMemcpy(ctx->bond_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
    if (nb) {
        CK(cudaMemcpy(ctx->bond_partner, partner.data(), partner.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->bond_k, kk.data(), kk.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->bond_r0, rr.data(), rr.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->bond_style, st.data(), st.size(), cudaMemcpyHostToDevice));
    }
    if (na) {
        if ((rc = dalloc(ctx, ctx->ang_off, aoff.size())) || (rc = dalloc(ctx, ctx->ang_rec, 3 * na)) ||
            (rc = dalloc(ctx, ctx->ang_k, 3 * na)) || (rc = dalloc(ctx, ctx->ang_t0, 3 * na)))
            return rc;
        CK(cudaMemcpy(ctx->ang_off, aoff.data(), aoff.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->ang_rec, arec.data(), arec.size() * sizeof(uint4), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->ang_k, ak.data(), ak.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->ang_t0, at.data(), at.size() * 4, cudaMemcpyHostToDevice));
    }
    TRY(refresh_bond_index(ctx));
    CK(cudaStreamSynchronize(ctx->stream));
    return 0;
}
}  // namespace

int dpdb_set_bonds(dpdb_ctx* ctx, size_t nb, const uint32_t* ti, const uint32_t* tj, const double* k,
                   const double* r0) {
    return dpdb_set_bonds_styled(ctx, nb, ti, tj, k, r0, nullptr);
}

int dpdb_set_bonds_styled(dpdb_ctx* ctx, size_t nb, const uint32_t* ti, const uint32_t* tj,
                          const double* k, const double* r0, const uint8_t* style) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    // BondTopology::validate, src/core.cpp:104-114
    std::vector<std::pair<uint32_t, uint32_t>> seen;
    seen.reserve(nb);
    for (size_t b = 0; b < nb; ++b) {
        if (ti[b] == tj[b])
            return fail(ctx, DPDB_ECONFIG, "bond topology: self bond on tag " + std::to_string(ti[b]));
        if (style && style[b] > 1) return fail(ctx, DPDB_ECONFIG, "bond topology: style must be 0 (harmonic) or 1 (FENE)");
        if (style && style[b] == 1 && !(r0[b] > 0))
            return fail(ctx, DPDB_ECONFIG, "bond topology: FENE needs a positive maximum extension R0");
        seen.emplace_back(std::min(ti[b], tj[b]), std::max(ti[b], tj[b]));
    }
    std::sort(seen.begin(), seen.end());
    for (size_t b = 1; b < seen.size(); ++b)
        if (seen[b] == seen[b - 1])
            return fail(ctx, DPDB_ECONFIG, "bond topology: duplicate bond " +
                                               std::to_string(seen[b].first) + "-" +
                                               std::to_string(seen[b].second));
    ctx->h_bi.assign(ti, ti + nb);
    ctx->h_bj.assign(tj, tj + nb);
    ctx->h_bk.assign(k, k + nb);
    ctx->h_br.assign(r0, r0 + nb);
    ctx->h_bs.assign(nb, 0);
    if (style) ctx->h_bs.assign(style, style + nb);
    return upload_bonded(ctx);
}

int dpdb_set_angles(dpdb_ctx* ctx, size_t na, const uint32_t* ta, const uint32_t* tb,
                    const uint32_t* tc, const double* k, const double* theta0) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    for (size_t q = 0; q < na; ++q)
        if (ta[q] == tb[q] || tb[q] == tc[q] || ta[q] == tc[q])
            return fail(ctx, DPDB_ECONFIG, "angle topology: three distinct tags needed at angle " +
                                               std::to_string(q));
    ctx->h_aa.assign(ta, ta + na);
    ctx->h_ab.assign(tb, tb + na);
    ctx->h_ac.assign(tc, tc + na);
    ctx->h_ak.assign(k, k + na);
    ctx->h_at.assign(theta0, theta0 + na);
    return upload_bonded(ctx);
}

int dpdb_sort_keys(dpdb_ctx* ctx, uint32_t* keys) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    TRY(launch_integrate<false, false, true, false>(ctx));
    TRY(check_device(ctx));
    CK(cudaMemcpy(keys, ctx->keys, ctx->n * 4, cudaMemcpyDeviceToHost));
    return 0;
}

int dpdb_reorder(dpdb_ctx* ctx, uint32_t* perm) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    TRY(do_reorder_all(ctx, true));
    TRY(check_device(ctx));
    if (perm && ctx->n) {
        std::vector<uint32_t> order(ctx->n);
        CK(cudaMemcpy(order.data(), ctx->vals, ctx->n * 4, cudaMemcpyDeviceToHost));
        for (size_t t = 0; t < ctx->n; ++t) perm[order[t]] = (uint32_t)t;
    }
    return 0;
}

int dpdb_cell_start(dpdb_ctx* ctx, uint32_t* cs) {
    TRY(require_ctx(ctx));
    if (!ctx->have_sorted) return fail(ctx, DPDB_ECONFIG, "cell list: particles not reordered");
    CK(cudaMemcpy(cs, ctx->cell_start, ((size_t)ctx->grid.n_total_cells + 1) * 4, cudaMemcpyDeviceToHost));
    return 0;
}

int dpdb_coarse_stencil(dpdb_ctx* ctx, uint32_t* offsets, uint32_t* cells) {
    TRY(require_ctx(ctx));
    std::vector<uint32_t> rows;
    std::vector<uint8_t> cnt, flags;
    ctx->grid.coarse_stencil(rows, cnt, flags);
    offsets[0] = 0;
    for (uint32_t r = 0; r < ctx->grid.n_local_cells; ++r) {
        if (cells) std::memcpy(cells + offsets[r], rows.data() + (size_t)r * 32, cnt[r] * 4);
        offsets[r + 1] = offsets[r] + cnt[r];
    }
    return 0;
}

int dpdb_fine_stencil(dpdb_ctx* ctx, uint32_t* foff, uint32_t* fidx) {
    TRY(require_ctx(ctx));
    if (!ctx->have_sorted) return fail(ctx, DPDB_ECONFIG, "fine stencil: particles not reordered");
    const HostGrid& g = ctx->grid;
    std::vector<uint32_t> cs((size_t)g.n_total_cells + 1), coff(g.n_local_cells + 1);
    CK(cudaMemcpy(cs.data(), ctx->cell_start, cs.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> rows;
    std::vector<uint8_t> cnt, flags;
    g.coarse_stencil(rows, cnt, flags);
    foff[0] = 0;
    for (uint32_t r = 0; r < g.n_local_cells; ++r) {
        uint32_t w = foff[r];
        for (uint32_t a = 0; a < cnt[r]; ++a) {
            const uint32_t c = rows[(size_t)r * 32 + a];
            if (fidx)
                for (uint32_t j = cs[c]; j < cs[c + 1]; ++j) fidx[w++] = j;
            else
                w += cs[c + 1] - cs[c];
        }
        foff[r + 1] = w;
    }
    return 0;
}

int dpdb_build_neighbors(dpdb_ctx* ctx) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    TRY(do_streams(ctx, nullptr));
    TRY(do_build(ctx, false));
    return check_device(ctx);
}

namespace {
// Restore the reference's joined rows (core ascending, skin ascending) from a
// force-walk layout:
//  1 (k_build): rowmeta (c1, c2, s1, s2), walk order = core[0,c1) core[c2,nc)
//    skin[0,s1) skin[s2,ns) core[c1,c2) skin[s1,s2);
//  2 (k_build_lane): n_front = fwalk & 0x1FFF entries ascending from the front,
//    the rest reversed from the back; bit 31 marks skin entries.
// Front entries (j | skin << 31, ascending) of every row from the range
// builder's per-tile flat lists: tile t's list holds sum_r fwalk[32t + r]
// items j | r << 26 | skin << 31, each row's items in ascending order.
int walk3_front(dpdb_ctx* ctx, const std::vector<uint32_t>& fw, std::vector<std::vector<uint32_t>>& front) {
    const size_t n = ctx->n, maxn = ctx->maxn;
    std::vector<uint32_t> pl(((n + 31) & ~size_t(31)) * maxn);
    CK(cudaMemcpy(pl.data(), ctx->plist, pl.size() * 4, cudaMemcpyDeviceToHost));
    front.assign(n, {});
    for (size_t t0 = 0; t0 < n; t0 += 32) {
        size_t cnt = 0;
        for (size_t i = t0; i < std::min(n, t0 + 32); ++i) cnt += std::min<size_t>(fw[i] & 0x1FFFu, maxn);
        for (size_t k = 0; k < cnt; ++k) {
            const uint32_t e = pl[t0 * maxn + k];
            const size_t i = t0 + ((e >> 26) & 31u);
            if (i < n) front[i].push_back((e & 0x03FFFFFFu) | (e & 0x80000000u));
        }
    }
    return 0;
}

// Full-row counts (core | skin << 13 | flags << 26, as k_build_range writes
// for the reference layout) of a layout-3 table: front entries + their
// in-block transposes.
int walk3_counts(dpdb_ctx* ctx, std::vector<uint32_t>& fw, std::vector<std::vector<uint32_t>>& front,
                 std::vector<std::vector<uint32_t>>& extra, std::vector<uint32_t>& cnt) {
    const size_t n = ctx->n;
    fw.resize(n);
    cnt.resize(n);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(fw.data(), ctx->fwalk, n * 4, cudaMemcpyDeviceToHost));
    TRY(walk3_front(ctx, fw, front));
    extra.assign(n, {});
    for (size_t i = 0; i < n; ++i)
        for (uint32_t e : front[i]) {
            const size_t j = e & 0x7FFFFFFFu;
            if (j > i && j < n && j / dpdb::FORCE_BLOCK == i / dpdb::FORCE_BLOCK)
                extra[j].push_back((uint32_t)i | (e & 0x80000000u));
        }
    for (size_t i = 0; i < n; ++i) {
        uint32_t nc = 0, ns = 0;
        for (uint32_t e : front[i]) (e >> 31 ? ns : nc)++;
        for (uint32_t e : extra[i]) (e >> 31 ? ns : nc)++;
        cnt[i] = std::min(nc, 8191u) | (std::min(ns, 8191u) << 13) | (fw[i] & 0xFC000000u);
    }
    return 0;
}

int unwalk(dpdb_ctx* ctx) {
    if (!ctx->walk) return 0;
    const int layout = ctx->walk;
    const size_t n = ctx->n, rows = (n + 31) & ~(size_t)31, maxn = ctx->maxn;
    ctx->walk = 0;
    if (!rows) return 0;
    std::vector<uint32_t> raw(rows * maxn), cnt(n), fw(n), out(rows * maxn, 0u);
    std::vector<uint2> meta(n);
    CK(cudaStreamSynchronize(ctx->stream));
    if (layout != 3) {
        CK(cudaMemcpy(raw.data(), ctx->entries, raw.size() * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(cnt.data(), ctx->counts, n * 4, cudaMemcpyDeviceToHost));
    }
    if (layout == 1) CK(cudaMemcpy(meta.data(), ctx->rowmeta, n * sizeof(uint2), cudaMemcpyDeviceToHost));
    if (layout >= 2) CK(cudaMemcpy(fw.data(), ctx->fwalk, n * 4, cudaMemcpyDeviceToHost));
    // layout 3: the front entries live in the tiles' flat lists (k_build_range);
    // the in-block j < i entries of row i are the transposes of front entries
    // (j -> i, j > i, same force block); the full rows' counts follow
    std::vector<std::vector<uint32_t>> front(layout == 3 ? n : 0), extra(layout == 3 ? n : 0);
    if (layout == 3) {
        TRY(walk3_counts(ctx, fw, front, extra, cnt));
        CK(cudaMemcpy(ctx->counts, cnt.data(), n * 4, cudaMemcpyHostToDevice));
    }
    auto idx = [&](size_t i, size_t k) { return ((i & ~size_t(31)) + (k & 31)) * maxn + (k & ~size_t(31)) + (i & 31); };
    std::vector<uint32_t> row(maxn), core, skin;
    for (size_t i = 0; i < n; ++i) {
        const uint32_t nc = cnt[i] & 0x1FFFu, ns = (cnt[i] >> 13) & 0x1FFFu;
        uint32_t w = 0;
        if (layout == 1) {
            const uint32_t c1 = meta[i].x & 0xFFFFu, c2 = meta[i].x >> 16;
            const uint32_t s1 = meta[i].y & 0xFFFFu, s2 = meta[i].y >> 16;
            const uint32_t A = c1, B = A + (nc - c2), C = B + s1, D = C + (ns - s2), E = D + (c2 - c1);
            for (uint32_t k = 0; k < A; ++k) row[w++] = raw[idx(i, k)];
            for (uint32_t k = D; k < E; ++k) row[w++] = raw[idx(i, k)];
            for (uint32_t k = A; k < B; ++k) row[w++] = raw[idx(i, k)];
            for (uint32_t k = B; k < C; ++k) row[w++] = raw[idx(i, k)];
            for (uint32_t k = E; k < nc + ns; ++k) row[w++] = raw[idx(i, k)];
            for (uint32_t k = C; k < D; ++k) row[w++] = raw[idx(i, k)];
        } else {
            const uint32_t tot = std::min<uint32_t>(nc + ns, (uint32_t)maxn);
            const uint32_t nf = std::min<uint32_t>(fw[i] & 0x1FFFu, tot), nb = tot - nf;
            core.clear();
            skin.clear();
            auto put = [&](uint32_t e) { (e >> 31 ? skin : core).push_back(e & 0x7FFFFFFFu); };
            if (layout == 3)
                for (uint32_t e : front[i]) put(e);
            else
                for (uint32_t k = 0; k < nf; ++k) put(raw[idx(i, k)]);
            if (layout == 2)
                for (uint32_t q = 0; q < nb; ++q) put(raw[idx(i, maxn - 1 - q)]);
            else
                for (uint32_t e : extra[i]) put(e);
            std::sort(core.begin(), core.end());
            std::sort(skin.begin(), skin.end());
            for (uint32_t e : core) row[w++] = e;
            for (uint32_t e : skin) row[w++] = e;
        }
        for (uint32_t k = 0; k < w; ++k) out[idx(i, k)] = row[k];
    }
    CK(cudaMemcpy(ctx->entries, out.data(), out.size() * 4, cudaMemcpyHostToDevice));
    return 0;
}
}  // namespace

int dpdb_join_core_skin(dpdb_ctx* ctx) {
    TRY(require_ctx(ctx));
    if (!ctx->have_table) return fail(ctx, DPDB_ECONFIG, "join_core_skin: no table");
    TRY(unwalk(ctx));
    if (ctx->joined) return 0;
    if (ctx->n) {
        dpdb::k_join<<<blocks_for(ctx->n, 256), 256, 0, ctx->stream>>>(ctx->entries, ctx->counts,
                                                                      (uint32_t)ctx->n, ctx->maxn,
                                                                      ctx->tiled);
        CKL();
    }
    ctx->joined = true;
    return check_device(ctx);
}

int dpdb_tile_transpose(dpdb_ctx* ctx) {
    TRY(require_ctx(ctx));
    if (!ctx->have_table) return fail(ctx, DPDB_ECONFIG, "tile_transpose: no table");
    TRY(unwalk(ctx));
    const uint32_t rows = (uint32_t)((ctx->n + 31) & ~(size_t)31);
    if (rows) {
        dim3 grid(ctx->maxn / 32, rows / 32), blk(32, 8);
        dpdb::k_tile_transpose<<<grid, blk, 0, ctx->stream>>>(ctx->entries, rows, ctx->maxn);
        CKL();
    }
    ctx->tiled = !ctx->tiled;
    return check_device(ctx);
}

int dpdb_get_neighbors(dpdb_ctx* ctx, uint32_t* entries, uint16_t* core, uint16_t* skin,
                       int32_t* tiled, int32_t* joined) {
    TRY(require_ctx(ctx));
    if (!ctx->have_table) return fail(ctx, DPDB_ECONFIG, "get_neighbors: no table");
    TRY(unwalk(ctx));
    const size_t n = ctx->n, rows = (n + 31) & ~(size_t)31, maxn = ctx->maxn;
    std::vector<uint32_t> cnt(n);
    CK(cudaMemcpy(cnt.data(), ctx->counts, n * 4, cudaMemcpyDeviceToHost));
    if (entries && rows) {
        std::vector<uint32_t> raw(rows * maxn);
        CK(cudaMemcpy(raw.data(), ctx->entries, raw.size() * 4, cudaMemcpyDeviceToHost));
        std::memset(entries, 0, rows * maxn * 4);
        auto idx = [&](uint32_t i, uint32_t k) -> size_t {
            return ctx->tiled ? (size_t)((i & ~31u) + (k & 31u)) * maxn + (k & ~31u) + (i & 31u)
                              : (size_t)i * maxn + k;
        };
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t nc = cnt[i] & 0x1FFFu, ns = (cnt[i] >> 13) & 0x1FFFu;
            for (uint32_t k = 0; k < nc; ++k) entries[idx(i, k)] = raw[idx(i, k)];
            for (uint32_t s = 0; s < ns; ++s) {
                const uint32_t k = ctx->joined ? nc + s : (uint32_t)(maxn - 1 - s);
                entries[idx(i, k)] = raw[idx(i, k)];
            }
        }
    }
    for (size_t i = 0; i < n; ++i) {
        if (core) core[i] = (uint16_t)(cnt[i] & 0x1FFFu);
        if (skin) skin[i] = (uint16_t)((cnt[i] >> 13) & 0x1FFFu);
    }
    if (tiled) *tiled = ctx->tiled;
    if (joined) *joined = ctx->joined;
    return 0;
}

int dpdb_set_neighbors(dpdb_ctx* ctx, const uint32_t* entries, const uint16_t* core,
                       const uint16_t* skin, int32_t tiled, int32_t joined) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    const size_t n = ctx->n, rows = (n + 31) & ~(size_t)31, maxn = ctx->maxn;
    if (n && (!entries || !core || !skin)) return fail(ctx, DPDB_ECONFIG, "set_neighbors: null array");
    std::vector<uint32_t> cnt(n);
    for (size_t i = 0; i < n; ++i) {
        if ((uint32_t)core[i] + skin[i] > maxn)
            return fail(ctx, DPDB_ECONFIG, "set_neighbors: row longer than max_neighbors");
        cnt[i] = core[i] | ((uint32_t)skin[i] << 13);
    }
    // the force kernels apply the minimum image through the posq frame: no per-row flags needed
    CK(cudaStreamSynchronize(ctx->stream));
    if (n) {
        CK(cudaMemcpy(ctx->entries, entries, rows * maxn * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->counts, cnt.data(), n * 4, cudaMemcpyHostToDevice));
    }
    ctx->tiled = tiled != 0;
    ctx->joined = joined != 0;
    ctx->walk = 0;
    ctx->have_table = true;
    return 0;
}

int dpdb_table_layout(int device, int op, size_t n_rows, uint32_t maxn, uint32_t* entries,
                      const uint16_t* core, const uint16_t* skin, int32_t tiled, int32_t joined) {
    dpdb_ctx* ctx = nullptr;  // CK/CKL report through the thread's error slot
    if (op != 0 && op != 1) return fail(nullptr, DPDB_ECONFIG, "table_layout: op must be 0 (join) or 1 (transpose)");
    if (maxn == 0 || maxn % 32) return fail(nullptr, DPDB_ECONFIG, "table_layout: max_neighbors must be a multiple of 32");
    if (!n_rows) return 0;
    if (!entries || (op == 0 && (!core || !skin))) return fail(nullptr, DPDB_ECONFIG, "table_layout: null array");
    if (op == 0 && joined) return 0;
    const int nd = dpdb_device_count();
    if (nd <= 0 || device < 0 || device >= nd)
        return fail(nullptr, DPDB_EDEVICE, "no compute capability 10.x device (the engine has no CPU fallback)");
    CK(cudaSetDevice(device));
    const size_t rows = (n_rows + 31) & ~(size_t)31;
    uint32_t *d_e = nullptr, *d_c = nullptr;
    CK(cudaMalloc(&d_e, rows * maxn * 4));
    int rc = 0;
    if (op == 0) {
        std::vector<uint32_t> cnt(n_rows);
        for (size_t i = 0; i < n_rows; ++i) cnt[i] = core[i] | ((uint32_t)skin[i] << 13);
        if (cudaMalloc(&d_c, n_rows * 4) != cudaSuccess ||
            cudaMemcpy(d_c, cnt.data(), n_rows * 4, cudaMemcpyHostToDevice) != cudaSuccess)
            rc = fail(nullptr, DPDB_EDEVICE, "table_layout: device allocation");
    }
    if (!rc && cudaMemcpy(d_e, entries, rows * maxn * 4, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = fail(nullptr, DPDB_EDEVICE, "table_layout: copy in");
    if (!rc) {
        if (op == 0)
            dpdb::k_join<<<blocks_for(n_rows, 256), 256>>>(d_e, d_c, (uint32_t)n_rows, maxn, tiled != 0);
        else
            dpdb::k_tile_transpose<<<dim3(maxn / 32, (unsigned)(rows / 32)), dim3(32, 8)>>>(d_e, (uint32_t)rows, maxn);
        if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
            cudaMemcpy(entries, d_e, rows * maxn * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
            rc = fail(nullptr, DPDB_EDEVICE, "table_layout: kernel");
    }
    cudaFree(d_e);
    if (d_c) cudaFree(d_c);
    (void)ctx;
    return rc;
}

int dpdb_signatures(dpdb_ctx* ctx, uint32_t* sig) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    TRY(do_streams(ctx, ctx->tmp_u32));
    CK(cudaMemcpyAsync(sig, ctx->tmp_u32, ctx->n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    return check_device(ctx);
}

int dpdb_compute_forces(dpdb_ctx* ctx, uint32_t step) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    TRY(do_streams(ctx, nullptr));
    TRY(do_forces(ctx, step));
    return check_device(ctx);
}

int dpdb_verlet_phase1(dpdb_ctx* ctx) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    TRY((launch_integrate<false, true, false, false>(ctx)));
    return check_device(ctx);
}

int dpdb_verlet_phase2(dpdb_ctx* ctx) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    TRY((launch_integrate<true, false, false, false>(ctx)));
    return check_device(ctx);
}

int dpdb_setup(dpdb_ctx* ctx) { return dpdb_setup_at(ctx, 0, 0); }

int dpdb_setup_at(dpdb_ctx* ctx, int64_t step, int32_t keep_forces) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    if (step < 0) return fail(ctx, DPDB_ECONFIG, "setup: step must be >= 0");
    ctx->step = step;
    TRY(do_reorder_all(ctx, keep_forces != 0));  // uploaded forces travel with the reorder
    TRY(do_build(ctx, true));
    if (!keep_forces) TRY(do_forces(ctx, (uint32_t)step));
    return check_device(ctx);
}

namespace {
// Alg. 1 loop.  When can_fuse, the Verlet pass between two force
// evaluations (phase 2 of step n + phase 1 of step n+1, plus the next step's
// fp32 streams or sort keys) runs in the epilogue of step n's force kernel,
// on the forces the block just reduced -- same arithmetic, one HBM pass fewer.
// rec (dpdb_step_thermo): device-visible record array, 5 doubles per step;
// the pass that applies phase 2 of step n also reduces its thermo partials
// and k_thermo_final writes record n -- no host synchronisation per step.
int thermo_record(dpdb_ctx* ctx, uint32_t nblocks, double* rec) {
    return thermo_fold(ctx, [&](cudaStream_t st, const double* part) {
        dpdb::k_thermo_final<<<1, 256, 0, st>>>(part, nblocks, (uint32_t)ctx->n, ctx->step, rec);
    });
}
// Look at the error word: true when the copy enqueued at the previous
// rebuild shows an error (the call then stops early; check_device reports
// it).  Enqueues the next copy.  A row overflow or a blow-up is thus caught
// within two rebuild periods of happening instead of at the end of a long
// dpdb_step call.  Single-domain loop only: brick ranks would have to agree
// to stop together (their collectives), so they check at the end of a call.
bool poll_error(dpdb_ctx* ctx) {
    if (!ctx->err_host) return false;
    // wait for the previous rebuild's copy: the host then runs at most one
    // rebuild period ahead of the device (that period's launches keep the
    // device fed meanwhile), so a small system cannot queue thousands of
    // steps past an error
    if (ctx->err_pending && cudaEventSynchronize(ctx->err_ev) == cudaSuccess) {
        ctx->err_pending = false;
        if (ctx->err_host->code) return true;
    }
    if (!ctx->err_pending &&
        cudaMemcpyAsync(ctx->err_host, ctx->err, sizeof(DevErr), cudaMemcpyDeviceToHost, ctx->stream) ==
            cudaSuccess &&
        cudaEventRecord(ctx->err_ev, ctx->stream) == cudaSuccess)
        ctx->err_pending = true;
    return false;
}

int run_steps(dpdb_ctx* ctx, int64_t nsteps, double* rec = nullptr) {
    if (!ctx->have_table) return fail(ctx, DPDB_ECONFIG, "step: call dpdb_setup first");
    const bool th = rec != nullptr;
    const uint32_t nb_int = (uint32_t)((ctx->n + 255) / 256);
    const uint32_t nb_force = (uint32_t)((ctx->n + dpdb::FORCE_BLOCK - 1) / dpdb::FORCE_BLOCK);
    bool integrated = false;  // this step's Verlet pass already ran in the last force kernel
    for (int64_t s = 0; s < nsteps; ++s) {
        ctx->step += 1;
        const bool rebuild = ctx->step % ctx->run.rebuild_every == 0;
        mark(ctx, ST_OTHER);
        // the integrate kernel here applies phase 2 of the previous step (s > 0)
        const bool th_prev = th && s > 0 && !integrated;
        if (rebuild) {
            if (!integrated) {
                if (s > 0) TRY((launch_integrate<true, true, true, false>(ctx, false, th_prev)));
                else TRY((launch_integrate<false, true, true, false>(ctx)));
                mark(ctx, ST_INTEGRATE);
            }
        } else if (!integrated) {
            if (s > 0) TRY((launch_integrate<true, true, false, true>(ctx, false, th_prev)));
            else TRY((launch_integrate<false, true, false, true>(ctx)));
            mark(ctx, ST_INTEGRATE);
        }
        if (th_prev) {
            ctx->step -= 1;  // the record belongs to the previous step
            TRY(thermo_record(ctx, nb_int, rec + 5 * (s - 1)));
            ctx->step += 1;
        }
        if (rebuild) {
            if (poll_error(ctx)) break;  // a kernel already reported an error: stop stepping
            TRY(do_sort(ctx));
            TRY(do_permute(ctx, false));
            mark(ctx, ST_SORT);
            TRY(do_build(ctx, true));
            mark(ctx, ST_BUILD);
        }
        const bool fuse = s + 1 < nsteps && can_fuse(ctx);
        const bool next_rebuild = (ctx->step + 1) % ctx->run.rebuild_every == 0;
        TRY(do_forces(ctx, (uint32_t)ctx->step,
                      fuse ? (next_rebuild ? dpdb::FUSE_KEYS : dpdb::FUSE_STREAMS) : dpdb::FUSE_NONE, th));
        if (fuse)
            for (int k = 0; k < 3; ++k) std::swap(ctx->x[k], ctx->x2[k]);
        if (fuse && !next_rebuild) {  // pos4 is not written: the builder reads it after a permute
            std::swap(ctx->posq, ctx->posqn);
            std::swap(ctx->vel4, ctx->vel4n);
        }
        integrated = fuse;
        mark(ctx, ST_FORCE);
        if (fuse && th) TRY(thermo_record(ctx, nb_force, rec + 5 * s));
    }
    if (nsteps > 0) {
        TRY((launch_integrate<true, false, false, false>(ctx, false, th)));
        mark(ctx, ST_INTEGRATE);
        if (th) TRY(thermo_record(ctx, nb_int, rec + 5 * (nsteps - 1)));
    }
    return 0;
}

}  // namespace

int dpdb_step(dpdb_ctx* ctx, int64_t nsteps) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    TRY(run_steps(ctx, nsteps));
    return check_device(ctx);
}

int dpdb_step_thermo(dpdb_ctx* ctx, int64_t nsteps, dpdb_thermo* out) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    if (nsteps < 0) return fail(ctx, DPDB_ECONFIG, "step_thermo: nsteps must be >= 0");
    if (!nsteps) return 0;
    if (!ctx->n) return fail(ctx, DPDB_EPHYSICS, "temperature of an empty system");
    if ((size_t)nsteps > ctx->thermo_cap) {
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->thermo_host) CK(cudaFreeHost(ctx->thermo_host));
        ctx->thermo_host = nullptr;
        ctx->thermo_cap = 0;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->thermo_host), (size_t)nsteps * 5 * sizeof(double),
                         cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->thermo_host_dev), ctx->thermo_host, 0));
        ctx->thermo_cap = (size_t)nsteps;
    }
    TRY(run_steps(ctx, nsteps, ctx->thermo_host_dev));
    TRY(check_device(ctx));
    for (int64_t s = 0; s < nsteps; ++s) {
        const double* r = ctx->thermo_host + 5 * s;
        out[s].step = (int64_t)r[0];
        out[s].n = ctx->n;
        out[s].kbt = r[1];
        for (int k = 0; k < 3; ++k) out[s].momentum[k] = r[2 + k];
    }
    return 0;
}

int dpdb_step_timed(dpdb_ctx* ctx, int64_t nsteps, double* ms, double* stage_ms,
                    int64_t* stage_launches) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    return timed_run(ctx, [&] { return run_steps(ctx, nsteps); }, ms, stage_ms, stage_launches);
}

int64_t dpdb_current_step(const dpdb_ctx* ctx) { return ctx ? ctx->step : -1; }

int dpdb_table_stats(dpdb_ctx* ctx, double* mean_row, double* mean_core, uint32_t* max_row) {
    TRY(require_ctx(ctx));
    if (!ctx->have_table) return fail(ctx, DPDB_ECONFIG, "table_stats: no table");
    std::vector<uint32_t> cnt(ctx->n);
    if (ctx->walk == 3) {  // the range builder's walk layout carries no full-row counts
        std::vector<uint32_t> fw;
        std::vector<std::vector<uint32_t>> front, extra;
        TRY(walk3_counts(ctx, fw, front, extra, cnt));
    } else {
        CK(cudaMemcpy(cnt.data(), ctx->counts, ctx->n * 4, cudaMemcpyDeviceToHost));
    }
    double s = 0, sc = 0;
    uint32_t mx = 0;
    for (uint32_t c : cnt) {
        const uint32_t nc = c & 0x1FFFu, ns = (c >> 13) & 0x1FFFu;
        s += nc + ns;
        sc += nc;
        mx = std::max(mx, nc + ns);
    }
    const double inv = ctx->n ? 1.0 / (double)ctx->n : 0.0;
    if (mean_row) *mean_row = s * inv;
    if (mean_core) *mean_core = sc * inv;
    if (max_row) *max_row = mx;
    return 0;
}

// ------------------------------------------------ validation observables
int dpdb_profile_reset(dpdb_ctx* ctx, uint32_t nbins, int32_t bin_axis, int32_t vel_axis) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    if (nbins < 1 || nbins > (uint32_t)dpdb::PROF_MAX_BINS)
        return fail(ctx, DPDB_ECONFIG, "velocity_profile: 1..1024 bins");
    if (bin_axis < 0 || bin_axis > 2 || vel_axis < 0 || vel_axis > 2)
        return fail(ctx, DPDB_ECONFIG, "velocity_profile: axes must be 0, 1 or 2");
    if (nbins > ctx->prof_nbins) {
        if (ctx->prof_acc) CK(cudaFree(ctx->prof_acc));
        ctx->prof_acc = nullptr;
        ctx->prof_nbins = 0;
        CK(cudaMalloc(&ctx->prof_acc, 2 * (size_t)nbins * sizeof(unsigned long long)));
    }
    ctx->prof_nbins = nbins;
    ctx->prof_bin_axis = bin_axis;
    ctx->prof_vel_axis = vel_axis;
    ctx->prof_samples = 0;
    CK(cudaMemsetAsync(ctx->prof_acc, 0, 2 * (size_t)nbins * sizeof(unsigned long long), ctx->stream));
    return 0;
}

int dpdb_profile_sample(dpdb_ctx* ctx) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    if (!ctx->prof_nbins) return fail(ctx, DPDB_ECONFIG, "velocity_profile: call dpdb_profile_reset first");
    const int ba = ctx->prof_bin_axis;
    const double lo = ctx->box.lo[ba], w = (ctx->box.hi[ba] - ctx->box.lo[ba]) / ctx->prof_nbins;
    if (ctx->n) {
        const unsigned nb = std::min<unsigned>(blocks_for(ctx->n, 256), 4 * 148);
        dpdb::k_profile<<<nb, 256, 0, ctx->stream>>>(ctx->x[ba], ctx->v[ctx->prof_vel_axis],
                                                     (uint32_t)ctx->n, lo, 1.0 / w, ctx->prof_nbins,
                                                     ctx->prof_acc);
        CKL();
        ctx->launches[ST_OTHER]++;
    }
    ctx->prof_samples += 1;
    return check_device(ctx);
}

int dpdb_profile_get(dpdb_ctx* ctx, double* sum_v, uint64_t* count, int64_t* nsamples) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    const uint32_t nb = ctx->prof_nbins;
    if (!nb) return fail(ctx, DPDB_ECONFIG, "velocity_profile: call dpdb_profile_reset first");
    std::vector<unsigned long long> h(2 * (size_t)nb);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(h.data(), ctx->prof_acc, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    for (uint32_t b = 0; b < nb; ++b) {
        if (sum_v) sum_v[b] = (double)(long long)h[b] / dpdb::PROF_SCALE;
        if (count) count[b] = h[nb + b];
    }
    if (nsamples) *nsamples = ctx->prof_samples;
    return 0;
}

int dpdb_rdf(dpdb_ctx* ctx, uint32_t nbins, double rmax, uint64_t* hist) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    if (!ctx->have_table) return fail(ctx, DPDB_ECONFIG, "rdf: neighbor table not built");
    if (nbins < 1 || nbins > 8192) return fail(ctx, DPDB_ECONFIG, "rdf: 1..8192 bins");
    if (!(rmax > 0) || rmax > ctx->params.r_c + ctx->run.skin + 1e-12)
        return fail(ctx, DPDB_ECONFIG, "rdf: 0 < rmax <= r_c + skin (the table's reach)");
    TRY(unwalk(ctx));  // walk layouts: back to reference rows
    TRY(do_streams(ctx, nullptr));  // pos4 of the current state (the fused loop writes posq only)
    unsigned long long* d = reinterpret_cast<unsigned long long*>(ctx->tmp_u32);
    if ((size_t)nbins * 2 > ctx->n_pad) return fail(ctx, DPDB_ECONFIG, "rdf: more bins than scratch");
    CK(cudaMemsetAsync(d, 0, nbins * sizeof(unsigned long long), ctx->stream));
    if (ctx->n) {
        dpdb::RdfArgs a{};
        a.pos4 = ctx->pos4;
        a.entries = ctx->entries;
        a.counts = ctx->counts;
        a.fwalk = ctx->fwalk;
        a.n = (uint32_t)ctx->n;
        a.maxn = ctx->maxn;
        a.nbins = nbins;
        a.layout = ctx->walk == 3 ? 3 : 0;
        a.tiled = ctx->tiled;
        a.joined = ctx->joined;
        for (int k = 0; k < 3; ++k) a.wrap[k] = ctx->grid.wrap[k];
        wrap_lengths(ctx, a.L, a.H);
        a.bins_per_r = (float)(nbins / rmax);
        dpdb::k_rdf<<<blocks_for(ctx->n, 256), 256, nbins * 4, ctx->stream>>>(a, d);
        CKL();
        ctx->launches[ST_OTHER]++;
    }
    std::vector<unsigned long long> h(nbins);
    CK(cudaMemcpyAsync(h.data(), d, nbins * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (uint32_t b = 0; b < nbins; ++b) hist[b] = h[b];
    return check_device(ctx);
}

int dpdb_thermo_get(dpdb_ctx* ctx, dpdb_thermo* out) {
    TRY(require_ctx(ctx));
    CK(cudaSetDevice(ctx->device));
    out->step = ctx->step;
    out->n = ctx->n;
    if (!ctx->n) return fail(ctx, DPDB_EPHYSICS, "temperature of an empty system");
    dpdb::k_sum3<<<RED_BLOCKS, 256, 0, ctx->stream>>>(ctx->v[0], ctx->v[1], ctx->v[2], nullptr,
                                                      (uint32_t)ctx->n, ctx->red);
    dpdb::k_sum_partials<<<1, 256, 0, ctx->stream>>>(ctx->red, RED_BLOCKS, ctx->red_out);
    dpdb::k_mean_from_sum<<<1, 32, 0, ctx->stream>>>(ctx->red_out, 1.0 / (double)ctx->n);
    // second pass around the device-resident mean; one read-back for both
    dpdb::k_sum3<<<RED_BLOCKS, 256, 0, ctx->stream>>>(ctx->v[0], ctx->v[1], ctx->v[2],
                                                      ctx->red_out + 4, (uint32_t)ctx->n, ctx->red);
    dpdb::k_sum_partials<<<1, 256, 0, ctx->stream>>>(ctx->red, RED_BLOCKS, ctx->red_out + 8);
    double r[16];
    CK(cudaMemcpyAsync(r, ctx->red_out, sizeof r, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < 3; ++k) out->momentum[k] = r[k];
    out->kbt = r[8 + 3] / (3.0 * (double)ctx->n);
    return 0;
}

int dpdb_eval(int device, int op, size_t n, const void* in0, const void* in1, uint32_t param,
              void* out) {
    dpdb_ctx* ctx = nullptr;
    size_t s0 = 4, s1 = 4, so = 4;
    switch (op) {
        case DPDB_OP_TEA_HASH: so = 8; break;
        case DPDB_OP_SIGNATURE: s1 = 24; break;
        case DPDB_OP_PAIR_UNIFORMS: s0 = 8; s1 = 8; so = 8; break;
        case DPDB_OP_GAUSSIAN64: so = 8; break;
        case DPDB_OP_GAUSSIAN32: break;
        case DPDB_OP_GAUSSIAN_HOT: break;
        case DPDB_OP_FASTLOG: s1 = 0; so = 8; break;
        case DPDB_OP_FASTCOS2PI: s1 = 0; so = 8; break;
        case DPDB_OP_FASTPOW: s0 = 8; s1 = 8; so = 8; break;
        case DPDB_OP_MORTON: s0 = 12; s1 = 0; break;
        case DPDB_OP_FASTLOG32: s1 = 0; break;
        case DPDB_OP_STEP_MIX: break;
        default: return fail(nullptr, DPDB_ECONFIG, "eval: unknown op");
    }
    if (!n) return 0;
    CK(cudaSetDevice(device));
    void *d0 = nullptr, *d1 = nullptr, *dout = nullptr;
    CK(cudaMalloc(&d0, n * s0));
    if (s1) CK(cudaMalloc(&d1, n * s1));
    CK(cudaMalloc(&dout, n * so));
    CK(cudaMemcpy(d0, in0, n * s0, cudaMemcpyHostToDevice));
    if (s1) CK(cudaMemcpy(d1, in1, n * s1, cudaMemcpyHostToDevice));
    dpdb::k_eval<<<blocks_for(n, 256), 256>>>(op, (uint32_t)n, d0, d1, param, dout);
    CKL();
    CK(cudaMemcpy(out, dout, n * so, cudaMemcpyDeviceToHost));
    cudaFree(d0);
    if (d1) cudaFree(d1);
    cudaFree(dout);
    return 0;
}

int dpdb_radix_sort(int device, uint32_t* keys, uint32_t* vals, size_t n, int bit_length) {
    dpdb_ctx* ctx = nullptr;
    if (bit_length < 0 || bit_length > 32 || bit_length % 4 != 0)
        return fail(nullptr, DPDB_ECONFIG, "radix sort: bit length must be a multiple of 4, <= 32");
    if (n == 0 || bit_length == 0) return 0;
    CK(cudaSetDevice(device));
    uint32_t *k = nullptr, *v = nullptr, *k2 = nullptr, *v2 = nullptr, *h = nullptr;
    CK(cudaMalloc(&k, n * 4));
    CK(cudaMalloc(&v, n * 4));
    CK(cudaMalloc(&k2, n * 4));
    CK(cudaMalloc(&v2, n * 4));
    CK(cudaMalloc(&h, dpdb::onesweep_work_words(n) * 4));
    CK(cudaMemcpy(k, keys, n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(v, vals, n * 4, cudaMemcpyHostToDevice));
    int rc = radix_sort_on(nullptr, 0, k, v, k2, v2, h, n, bit_length);
    if (!rc) {
        CK(cudaMemcpy(keys, k, n * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(vals, v, n * 4, cudaMemcpyDeviceToHost));
    }
    cudaFree(k);
    cudaFree(v);
    cudaFree(k2);
    cudaFree(v2);
    cudaFree(h);
    return rc;
}

}  // extern "C"

#include "domain_host.inc"
static_assert(dpdb::RB_BLOCK == dpdb::FORCE_BLOCK, "range builder CTA must own one force block");
