// kernels.cuh -- sm_100a kernels of the B200 DPD engine.
//
// Data layout in HBM (one domain, n particles, n_pad = n rounded up to 32):
//   x[3], v[3]          fp64 SoA master state (ParticleStore, inc/core.hpp:29-47)
//   f[3]                fp32 SoA forces (accumulated in fp32)
//   tag u32, species u8, molecule u32
//   pos4 float4         (x - slab_centre as fp32 | tag bits)   P:234 precision model
//                       (the builder's frozen distance frame)
//   posq int4           (x in int32 fixed point | tag bits): the pair-force frame
//   vel4 float4         (v as fp32 | signature bits)
//   keys/vals u32       radix sort ping-pong; sorted keys double as cell ranks
//   cell_start u32      [n_total_cells + 1]
//   stencil u32         [n_local_cells][32] coarse stencil ranks (<=27 used)
//   entries u32         [n_pad][maxn] neighbor table, 32x32 tile-transposed,
//                       core from the front, skin reversed from the back
//                       (inc/neighbor_table.hpp:12-31)
//   counts u32          core | skin << 13 | force-wrap-flags << 26
#pragma once
#include <cuda_runtime.h>

// warps per pair-force CTA; the force block (and the range builder's CTA
// block) is 32 * TPW particles per warp (A/B: 8 warps x 2 tiles -> 512, 16 x 2 -> 1024)
#ifndef DPDB_FORCE_WARPS
#define DPDB_FORCE_WARPS 8
#endif
// 32-row tiles each warp of a force CTA takes (block = 32 * TPW * WARPS particles)
#ifndef DPDB_FORCE_TPW
#define DPDB_FORCE_TPW 2
#endif

#include <cstdint>
#include <type_traits>

#include "dpd_math.cuh"

namespace dpdb {

struct DevErr {
    int code;       // first error category seen (atomicCAS from 0)
    uint32_t tag;   // offending particle tag
    uint32_t tag2;  // second tag (pair errors)
    int what;       // kernel-specific detail code
};

enum ErrWhat : int {
    EW_NONFINITE = 1,
    EW_ESCAPED = 2,
    EW_MIGRATION = 3,
    EW_OVERFLOW = 4,
    EW_COINCIDENT = 5,
    EW_BOND = 6,
    EW_FENE = 7,
};

__device__ __forceinline__ void raise_err(DevErr* e, int code, int what, uint32_t t1, uint32_t t2) {
    if (atomicCAS(&e->code, 0, code) == 0) {
        e->what = what;
        e->tag = t1;
        e->tag2 = t2;
    }
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ------------------------------------------------------------ geometry
struct DevGrid {
    double slab_lo[3], slab_hi[3], inv_cell[3], origin[3], cell_size[3], centre[3];
    int ncell[3], ncell_ext[3], ghost_lo[3];
    int sub_bits;
    const uint32_t* rank_of_cell;
};

// src/cell_grid.cpp:97-128 + inc/cell_grid.hpp:66-68, bit-exact (no fma)
__device__ __forceinline__ bool sort_key_of(const DevGrid& g, double x, double y, double z,
                                            uint32_t& key) {
    const double p[3] = {x, y, z};
    int c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (!(p[k] >= g.slab_lo[k] && p[k] < g.slab_hi[k])) return false;
        int ci = __double2int_rd(__dmul_rn(__dsub_rn(p[k], g.slab_lo[k]), g.inv_cell[k]));
        ci = min(max(ci, 0), g.ncell[k] - 1);
        c[k] = ci + g.ghost_lo[k];
    }
    const uint32_t rank =
        g.rank_of_cell[((size_t)c[2] * g.ncell_ext[1] + c[1]) * g.ncell_ext[0] + c[0]];
    const int nsub = 1 << g.sub_bits;
    uint32_t s[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double cell_lo = __dadd_rn(g.origin[k], __dmul_rn((double)c[k], g.cell_size[k]));
        int si = __double2int_rd(
            __dmul_rn(__dmul_rn(__dsub_rn(p[k], cell_lo), g.inv_cell[k]), (double)nsub));
        s[k] = (uint32_t)min(max(si, 0), nsub - 1);
    }
    uint32_t sub = 0;
    for (int b = 0; b < g.sub_bits; ++b)
        sub |= (((s[0] >> b) & 1u) << (3 * b)) | (((s[1] >> b) & 1u) << (3 * b + 1)) |
               (((s[2] >> b) & 1u) << (3 * b + 2));
    key = (rank << (3 * g.sub_bits)) | sub;
    return true;
}

// ------------------------------------------------- pair-force frame
// Fixed-point position frame of the pair-force kernels (posq).  The builder's
// fp32 slab-centre frame (pos4, frozen by inc/neighbor_table.hpp:43-44 for
// bit-exact rows) rounds x - centre to 24 bits: 3.8e-6 at |x - c| ~ 60 (C3),
// 7.6e-6 at ~90 (C5), which for a close pair (r ~ 1e-3) turns into a 1e-2
// error of the pair direction.  posq keeps 32 bits per axis instead:
//   wrap axes (single-domain periodic): q = (x - lo) * 2^32 / L taken mod
//     2^32, so the int32 difference of two particles IS the minimum image
//     (src/core.cpp:129-139) at L / 2^32 resolution (2.6e-8 at C3);
//   other axes: q = (x - centre) * 2^e, the largest power of two that keeps
//     the slab, its ghost layers and a margin inside int32.
// The force kernels form dx = (float)(q_i - q_j) * qs: exact integer
// difference, one rounding.
struct PosQ {
    double org[3];  // lo (wrap axes) or slab centre
    double s[3];    // quanta per length unit
    int wrap[3];
};

__device__ __forceinline__ int quant_axis(double x, double org, double s, int wrap) {
    const long long q = __double2ll_rn(__dmul_rn(__dsub_rn(x, org), s));
    if (wrap) return (int)(unsigned)(unsigned long long)q;  // mod 2^32
    return (int)min(max(q, -2147483647LL), 2147483647LL);
}

__device__ __forceinline__ int4 posq_of(const PosQ& p, double x0, double x1, double x2, uint32_t tw) {
    return make_int4(quant_axis(x0, p.org[0], p.s[0], p.wrap[0]), quant_axis(x1, p.org[1], p.s[1], p.wrap[1]),
                     quant_axis(x2, p.org[2], p.s[2], p.wrap[2]), (int)tw);
}

// --------------------------------------------------------- integrator
struct BoundaryArgs {
    double lo[3], hi[3], L[3];
    int periodic[3], wall[3];
    int bounce_back;  // walls reverse the whole velocity (else the normal component)
};

// periodic wrap right after the position update, walls
// mirror the position and reverse the normal velocity (specular; the
// bounce-back switch reverses the other components in integrate_particle);
// returns false if the particle is still outside (escaped)
__device__ __forceinline__ bool apply_boundary(const BoundaryArgs& b, int k, double& x, double& v,
                                               bool& hit_wall) {
    if (b.periodic[k]) {
        if (x < b.lo[k]) {
            x = __dadd_rn(x, b.L[k]);
            if (x >= b.hi[k]) x = b.lo[k];
        } else if (x >= b.hi[k]) {
            x = __dsub_rn(x, b.L[k]);
            if (x < b.lo[k]) x = b.lo[k];
        }
        return x >= b.lo[k] && x < b.hi[k];
    }
    if (b.wall[k]) {
        if (x >= b.hi[k]) {
            x = __dsub_rn(__dmul_rn(2.0, b.hi[k]), x);
            v = -v;
            hit_wall = true;
            if (x >= b.hi[k]) x = nextafter(b.hi[k], b.lo[k]);
        } else if (x < b.lo[k]) {
            x = __dsub_rn(__dmul_rn(2.0, b.lo[k]), x);
            v = -v;
            hit_wall = true;
            if (x >= b.hi[k]) x = nextafter(b.hi[k], b.lo[k]);
        }
        return x >= b.lo[k] && x < b.hi[k];
    }
    return true;
}

struct IntegrateArgs {
    double* x[3];
    double* v[3];
    const float* f[3];
    const uint32_t* tag;
    const uint8_t* sp;  // species (multi-species runs only, else nullptr)
    float4* pos4;
    int4* posq;
    float4* vel4;
    PosQ pq;
    uint32_t* keys;
    uint32_t* vals;
    DevErr* err;
    BoundaryArgs bnd;
    DevGrid grid;
    double dt, h;
    uint32_t n;
    double* thermo_part;  // PHASE2 passes: per-block (sum v_x, v_y, v_z, |v|^2) of the full-step v, or null
};

// Fixed-order block sum of four fp64 values (one per thread) for the per-step
// thermo: shuffle tree inside each warp, then warp 0 adds the warp sums in
// warp order.  Deterministic for a given block shape.  All threads call it.
template <int THREADS>
__device__ __forceinline__ void block_sum4(double (&v)[4], double* out) {
    __shared__ double ws[THREADS / 32][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xFFFFFFFFu, v[q], o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0)
#pragma unroll
        for (int q = 0; q < 4; ++q) ws[w][q] = v[q];
    __syncthreads();
    if (threadIdx.x < 4) {
        double acc = 0.0;
        for (int k = 0; k < THREADS / 32; ++k) acc += ws[k][threadIdx.x];
        out[threadIdx.x] = acc;
    }
}

// Fused Verlet: [phase 2 of the previous step] + phase 1 of this step +
// boundary + either the sort keys (rebuild step; the permute kernel then
// writes the fp32 streams) or the fp32 force streams with signatures.
// Each half kick is its own rounding so the fp64 trajectory equals the
// reference's phase2-then-phase1 sequence bit for bit.
// One particle; f is the particle's force (k_integrate reads it from memory,
// the fused pair-force kernel hands over its freshly reduced sum).  STREAMS
// writes posq + vel4 (the pair kernel's inputs) and pos4 when non-null (the
// fused epilogue skips it: only the builder reads pos4, after a permute).
template <bool PHASE2, bool PHASE1, bool KEYS, bool STREAMS>
__device__ __forceinline__ void integrate_particle(const IntegrateArgs& a, uint32_t i, const float f[3],
                                                   const double xin[3], const double vin[3],
                                                   uint32_t tag, uint32_t spc, float4* pos4,
                                                   int4* posq, float4* vel4, double vfull[3]) {
    double xs[3], vs[3];
    bool ok = true;
    uint32_t walls = 0;  // axes whose wall reflected this particle
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double v = vin[k];
        if (PHASE2 || PHASE1) {
            const double fk = (double)f[k];
            if (PHASE2) v = __dadd_rn(v, __dmul_rn(a.h, fk));
            vfull[k] = v;  // the full-step velocity (after phase 2), for the thermo
            if (PHASE1) v = __dadd_rn(v, __dmul_rn(a.h, fk));
        }
        double x = xin[k];
        if (PHASE1) {
            x = __dadd_rn(x, __dmul_rn(a.dt, v));
            bool hit = false;
            if (!(isfinite(x) && isfinite(v)))
                ok = false;
            else if (!apply_boundary(a.bnd, k, x, v, hit))
                ok = false;
            walls |= (uint32_t)hit << k;
            a.x[k][i] = x;
        }
        xs[k] = x;
        vs[k] = v;
    }
    if (PHASE1 && walls && a.bnd.bounce_back)  // bounce-back: the tangential components too
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (!(walls >> k & 1u)) vs[k] = -vs[k];
    if (PHASE2 || PHASE1)
#pragma unroll
        for (int k = 0; k < 3; ++k) a.v[k][i] = vs[k];
    if (!ok) raise_err(a.err, DPDB_EPHYSICS, EW_NONFINITE, tag, 0);
    if (KEYS) {
        uint32_t key = 0xFFFFFFFFu;
        if (!sort_key_of(a.grid, xs[0], xs[1], xs[2], key))
            raise_err(a.err, DPDB_EPROTOCOL, EW_MIGRATION, tag, 0);
        a.keys[i] = key;
        a.vals[i] = i;
    }
    if (STREAMS) {
        const uint32_t sig = make_signature(tag, vs[0], vs[1], vs[2]);
        const uint32_t tw = a.sp ? (tag | (spc << 28)) : tag;  // species in bits 28+
        if (pos4)
            pos4[i] = make_float4((float)(xs[0] - a.grid.centre[0]), (float)(xs[1] - a.grid.centre[1]),
                                  (float)(xs[2] - a.grid.centre[2]), __uint_as_float(tw));
        posq[i] = posq_of(a.pq, xs[0], xs[1], xs[2], tw);
        vel4[i] = make_float4((float)vs[0], (float)vs[1], (float)vs[2], __uint_as_float(sig));
    }
}

template <bool PHASE2, bool PHASE1, bool KEYS, bool STREAMS>
__global__ void __launch_bounds__(256) k_integrate(IntegrateArgs a) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    double vf[3] = {0.0, 0.0, 0.0};
    if (i < a.n) {
        float f[3] = {0.f, 0.f, 0.f};
        double x[3], v[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (PHASE2 || PHASE1) f[k] = a.f[k][i];
            x[k] = a.x[k][i];
            v[k] = a.v[k][i];
        }
        const uint32_t tag = (STREAMS || PHASE1) ? a.tag[i] : 0u;  // signature / error report
        const uint32_t spc = (STREAMS && a.sp) ? a.sp[i] : 0u;
        integrate_particle<PHASE2, PHASE1, KEYS, STREAMS>(a, i, f, x, v, tag, spc, a.pos4, a.posq, a.vel4,
                                                          vf);
    }
    if (PHASE2 && a.thermo_part) {  // uniform per launch
        double s4[4] = {vf[0], vf[1], vf[2], vf[0] * vf[0] + vf[1] * vf[1] + vf[2] * vf[2]};
        block_sum4<256>(s4, a.thermo_part + 4 * blockIdx.x);
    }
}

// Thread t folds partials t, t + 256, ... in that order; the loads of eight
// consecutive ones are issued before their adds (a plain loop serialises one
// memory latency per partial: ~10 us for 8192 partials).
__device__ __forceinline__ void fold_partials4(const double* part, uint32_t nparts, double (&v)[4]) {
    const double2* p2 = reinterpret_cast<const double2*>(part);
    for (uint32_t b0 = threadIdx.x; b0 < nparts; b0 += 256u * 8u) {
        double2 lo[8], hi[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t b = b0 + 256u * k;
            lo[k] = b < nparts ? p2[2 * b] : make_double2(0.0, 0.0);
            hi[k] = b < nparts ? p2[2 * b + 1] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            v[0] += lo[k].x;
            v[1] += lo[k].y;
            v[2] += hi[k].x;
            v[3] += hi[k].y;
        }
    }
}

// Brick runs: the raw per-brick sums {step, sum v_x, sum v_y, sum v_z,
// sum |v|^2} of one step (combined across bricks in brick order by the host)
__global__ void __launch_bounds__(256) k_thermo_sums(const double* part, uint32_t nblocks, int64_t step,
                                                     double* rec) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    fold_partials4(part, nblocks, v);
    __shared__ double tot[4];
    block_sum4<256>(v, tot);
    __syncthreads();
    if (threadIdx.x == 0) {
        rec[0] = (double)step;
#pragma unroll
        for (int q = 0; q < 4; ++q) rec[1 + q] = tot[q];
    }
}

// Per-step thermo record from the block partials of the pass that applied
// phase 2 (fixed order): rec = {step, kT, P_x, P_y, P_z} with
// kT = (sum |v|^2 - |sum v|^2 / n) / (3 n), the COM-subtracted temperature of
// compute_temperature (src/core.cpp:141-149) in one pass.
__global__ void __launch_bounds__(256) k_thermo_final(const double* part, uint32_t nblocks, uint32_t n,
                                                      int64_t step, double* rec) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    fold_partials4(part, nblocks, v);
    __shared__ double tot[4];
    block_sum4<256>(v, tot);
    __syncthreads();
    if (threadIdx.x == 0) {
        const double p2 = tot[0] * tot[0] + tot[1] * tot[1] + tot[2] * tot[2];
        rec[0] = (double)step;
        rec[1] = (tot[3] - p2 / (double)n) / (3.0 * (double)n);
        rec[2] = tot[0];
        rec[3] = tot[1];
        rec[4] = tot[2];
    }
}

// ------------------------------------------------------- radix sort
// Stable LSD radix sort (the RadixSorter::sort contract, inc/radix_sort.hpp:11-27;
// paper Alg. 2) with 8-bit digits; in-tile ranks from warp
// match/ballot -- stable by construction (tile order, then round, then warp,
// then lane).  k_scan_digits / block_excl_scan_1024 also serve the brick
// migration lists.
constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;

// block-wide exclusive scan helper (1024 threads)
__device__ __forceinline__ uint32_t block_excl_scan_1024(uint32_t v, uint32_t* warp_sums,
                                                         uint32_t& total) {
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31) warp_sums[w] = incl;
    __syncthreads();
    if (w == 0) {
        const uint32_t ws = warp_sums[lane];
        uint32_t wi = ws;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= (uint32_t)o) wi += y;
        }
        warp_sums[lane] = wi - ws;
        if (lane == 31) warp_sums[32] = wi;
    }
    __syncthreads();
    const uint32_t r = warp_sums[w] + incl - v;
    total = warp_sums[32];
    __syncthreads();
    return r;
}

// Per-digit exclusive scan over the tiles (digit-major histogram row d), one
// block per digit; totals[d] = count of digit d.
__global__ void __launch_bounds__(1024) k_scan_digits(uint32_t* __restrict__ hist,
                                                      uint32_t num_tiles,
                                                      uint32_t* __restrict__ totals) {
    __shared__ uint32_t ws[33];
    uint32_t* row = hist + (size_t)blockIdx.x * num_tiles;
    uint32_t run = 0;
    for (uint32_t b = 0; b < num_tiles; b += 1024) {
        const uint32_t t = b + threadIdx.x;
        const uint32_t v = t < num_tiles ? row[t] : 0u;
        uint32_t tot;
        const uint32_t ex = block_excl_scan_1024(v, ws, tot);
        if (t < num_tiles) row[t] = run + ex;
        run += tot;
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = run;
}

// ---- onesweep LSD radix sort (single-pass digit binning with decoupled
// look-back): one histogram kernel for every digit position, then one kernel
// per 8-bit digit.  Each CTA takes the next 4096-key tile in launch order (a
// tile counter, so every tile it waits on belongs to a CTA already resident),
// ranks its keys stably, publishes its per-digit counts, looks back over the
// earlier tiles' published counts / inclusive prefixes for its global offsets
// (no global scan pass, no host round trip), stages the tile digit-sorted in
// shared memory and writes it out in contiguous runs.  Stable order: tile,
// then round, then warp, then lane -- the input index order.
constexpr int OS_THREADS = RS_THREADS;
constexpr int OS_ITEMS = RS_ITEMS;
constexpr int OS_TILE = RS_TILE;
constexpr uint32_t OS_AGG = 1u << 30, OS_INC = 2u << 30, OS_VAL = (1u << 30) - 1u;

// words of sort workspace for n keys: [4][tiles][256] status, [4][256] histograms, [4] tile counters
inline size_t onesweep_work_words(size_t n) {
    const size_t tiles = (n + OS_TILE - 1) / OS_TILE;
    return 4 * tiles * 256 + 4 * 256 + 32;
}

// Every thread takes 16 consecutive keys (four 16-byte loads) and adds runs
// of equal digits at once: the input is the previous order, nearly sorted, so
// the high digits change rarely along a run and most shared adds disappear.
__global__ void __launch_bounds__(256) k_onesweep_hist(const uint32_t* __restrict__ keys, uint32_t n, int passes,
                                                       uint32_t* __restrict__ ghist) {
    __shared__ uint32_t h[4][256];
    for (int p = 0; p < 4; ++p) h[p][threadIdx.x] = 0;
    __syncthreads();
    const uint32_t stride = gridDim.x * blockDim.x * 16u;
    for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) * 16u; b < n; b += stride) {
        uint32_t k[16];
        if (b + 16 <= n) {  // the key arrays are cudaMalloc-aligned
            const uint4* q = reinterpret_cast<const uint4*>(keys + b);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint4 w = __ldg(q + c);
                k[4 * c] = w.x;
                k[4 * c + 1] = w.y;
                k[4 * c + 2] = w.z;
                k[4 * c + 3] = w.w;
            }
        } else {
#pragma unroll
            for (int c = 0; c < 16; ++c) k[c] = b + c < n ? __ldg(keys + b + c) : 0u;
        }
        const uint32_t m = min(16u, n - b);
        for (int p = 0; p < passes; ++p) {
            uint32_t cur = (k[0] >> (8 * p)) & 0xFFu, run = 0;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const uint32_t d = (k[c] >> (8 * p)) & 0xFFu;
                if ((uint32_t)c < m && d != cur) {
                    atomicAdd(&h[p][cur], run);
                    cur = d;
                    run = 0;
                }
                run += (uint32_t)c < m;
            }
            atomicAdd(&h[p][cur], run);
        }
    }
    __syncthreads();
    for (int p = 0; p < passes; ++p)
        if (h[p][threadIdx.x]) atomicAdd(&ghist[p * 256 + threadIdx.x], h[p][threadIdx.x]);
}

// exclusive scan of 256 values, one per thread of a 256-thread block
__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t v, uint32_t* ws /*[8]*/) {
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31) ws[w] = incl;
    __syncthreads();
    uint32_t off = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) off += q < (int)w ? ws[q] : 0u;
    __syncthreads();
    return off + incl - v;
}

#ifndef DPDB_RS_BATCH
#define DPDB_RS_BATCH 2
#endif
__global__ void __launch_bounds__(OS_THREADS) k_onesweep(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, uint32_t n, int shift, uint32_t mask, const uint32_t* __restrict__ ghist,
    uint32_t* status, uint32_t* tile_counter) {
    constexpr int RB = DPDB_RS_BATCH;
    static_assert(OS_ITEMS % RB == 0, "batches must tile the rounds");
    __shared__ uint32_t s_tile, s_ws[8];
    __shared__ uint32_t s_run[256], s_base[256], s_lstart[256];
    __shared__ union {
        struct {
            uint32_t cnt[RB][8][256], pref[RB][8][256];
        } rk;
        struct {
            uint32_t k[OS_TILE], v[OS_TILE];
        } st;
    } u;
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) s_tile = atomicAdd(tile_counter, 1u);
    s_run[t] = 0;
#pragma unroll
    for (int rr = 0; rr < RB; ++rr)
#pragma unroll
        for (int w = 0; w < 8; ++w) u.rk.cnt[rr][w][t] = 0;
    const uint32_t gstart = block_excl_scan_256(ghist[t], s_ws);  // barriers inside
    const uint32_t tile = s_tile;
    const uint32_t t0 = tile * OS_TILE;
    uint32_t key[OS_ITEMS], val[OS_ITEMS], lr[OS_ITEMS];
#pragma unroll
    for (int r = 0; r < OS_ITEMS; ++r) {  // all loads in flight first
        const uint32_t idx = t0 + r * OS_THREADS + t;
        key[r] = idx < n ? __ldg(kin + idx) : 0u;
        val[r] = idx < n ? __ldg(vin + idx) : 0u;
    }
    const uint32_t lt = lanemask_lt();
    // local stable ranks: per (round, warp) a match_any count per digit, then a
    // per-digit running prefix over (round, warp) order
#pragma unroll
    for (int r0 = 0; r0 < OS_ITEMS; r0 += RB) {
        uint32_t d[RB], rank[RB];
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
            const int r = r0 + rr;
            const bool valid = t0 + r * OS_THREADS + t < n;
            d[rr] = valid ? (key[r] >> shift) & mask : 256u + lane;
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d[rr]);
            rank[rr] = __popc(peers & lt);
            if (valid && (__ffs(peers) - 1) == (int)lane) u.rk.cnt[rr][warp][d[rr]] = __popc(peers);
        }
        __syncthreads();
        {
            uint32_t run = s_run[t];
#pragma unroll
            for (int rr = 0; rr < RB; ++rr)
#pragma unroll
                for (int w = 0; w < 8; ++w) {
                    const uint32_t c = u.rk.cnt[rr][w][t];
                    u.rk.pref[rr][w][t] = run;
                    u.rk.cnt[rr][w][t] = 0;
                    run += c;
                }
            s_run[t] = run;
        }
        __syncthreads();
#pragma unroll
        for (int rr = 0; rr < RB; ++rr)
            lr[r0 + rr] = d[rr] < 256u ? u.rk.pref[rr][warp][d[rr]] + rank[rr] : 0u;
    }
    // decoupled look-back, thread t = digit t
    const uint32_t cnt = s_run[t];
    uint32_t* my = status + (size_t)tile * 256 + t;
    uint32_t prefix = 0;
    if (tile == 0) {
        __stcg(my, OS_INC | cnt);
    } else {
        __stcg(my, OS_AGG | cnt);
        // windows of 8 predecessors per round trip: their status loads are
        // independent, so a chain of published aggregates resolves 8 tiles
        // per memory latency; a window stops at the first unpublished tile
        // (retried) or at an inclusive prefix (done)
        int p = (int)tile - 1;
        bool done = false;
        while (!done) {
            uint32_t w[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                w[q] = p - q >= 0 ? *(const volatile uint32_t*)(status + (size_t)(p - q) * 256 + t) : OS_INC;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (done) break;
                if ((w[q] & (OS_AGG | OS_INC)) == 0u) break;  // not published yet: retry from here
                prefix += w[q] & OS_VAL;
                --p;
                done = (w[q] & OS_INC) != 0u;
            }
        }
        __stcg(my, OS_INC | (prefix + cnt));
    }
    s_base[t] = gstart + prefix;
    s_lstart[t] = block_excl_scan_256(cnt, s_ws);  // barriers inside (also fences the rank scratch)
    __syncthreads();
    // stage the tile digit-sorted, then write contiguous runs
#pragma unroll
    for (int r = 0; r < OS_ITEMS; ++r) {
        if (t0 + r * OS_THREADS + t < n) {
            const uint32_t pos = s_lstart[(key[r] >> shift) & mask] + lr[r];
            u.st.k[pos] = key[r];
            u.st.v[pos] = val[r];
        }
    }
    __syncthreads();
    const uint32_t tn = min((uint32_t)OS_TILE, n - t0);
    for (uint32_t i = t; i < tn; i += OS_THREADS) {
        const uint32_t k = u.st.k[i], d = (k >> shift) & mask;
        const uint32_t dst = s_base[d] + (i - s_lstart[d]);
        kout[dst] = k;
        vout[dst] = u.st.v[i];
    }
}

// ------------------------------------------------ permute + cell list
struct PermuteArgs {
    const double* xin[3];
    const double* vin[3];
    double* xout[3];
    double* vout[3];
    const float* fin[3];
    float* fout[3];
    const uint32_t* tag_in;
    uint32_t* tag_out;
    const uint8_t* sp_in;
    uint8_t* sp_out;
    const uint32_t* mol_in;
    uint32_t* mol_out;
    const uint32_t* order;       // sorted vals: order[to] = from
    const uint32_t* keys;        // sorted keys
    uint32_t* cell_start;        // [n_total_cells + 1]
    uint32_t* ostart;            // [8 n_total_cells + 1] octant starts (nullable, sub_bits >= 1)
    float4* pos4;
    int4* posq;
    float4* vel4;
    PosQ pq;
    double centre[3];
    uint32_t n, n_total_cells;
    int key_shift;               // 3 * sub_bits
    int multi;                   // pack species into pos4.w bits 28-31
};

// reorder_particles' gather (src/cell_grid.cpp:180-195) fused with the
// cell-boundary detection of build_cell_list (src/cell_grid.cpp:136-155) and
// the fp32 stream + signature pack for the force/neighbor kernels.
template <bool FORCES, bool MOL>
__global__ void __launch_bounds__(256) k_permute(PermuteArgs a) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.n) return;
    const uint32_t from = a.order[t];
    double xs[3], vs[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        xs[k] = a.xin[k][from];
        vs[k] = a.vin[k][from];
        a.xout[k][t] = xs[k];
        a.vout[k][t] = vs[k];
        if (FORCES) a.fout[k][t] = a.fin[k][from];
    }
    const uint32_t tag = a.tag_in[from];
    a.tag_out[t] = tag;
    const uint8_t spc = a.sp_in[from];
    a.sp_out[t] = spc;
    if (MOL) a.mol_out[t] = a.mol_in[from];
    const uint32_t sig = make_signature(tag, vs[0], vs[1], vs[2]);
    const uint32_t tw = a.multi ? (tag | ((uint32_t)spc << 28)) : tag;  // species in bits 28+
    a.pos4[t] = make_float4((float)(xs[0] - a.centre[0]), (float)(xs[1] - a.centre[1]),
                            (float)(xs[2] - a.centre[2]), __uint_as_float(tw));
    a.posq[t] = posq_of(a.pq, xs[0], xs[1], xs[2], tw);
    a.vel4[t] = make_float4((float)vs[0], (float)vs[1], (float)vs[2], __uint_as_float(sig));
    // cell_start[c] = first t with rank >= c
    const uint32_t rmax = a.n_total_cells - 1u;  // clamp: a bad key already raised an error
    const uint32_t r = min(a.keys[t] >> a.key_shift, rmax);
    const uint32_t c0 = t == 0 ? 0u : min(a.keys[t - 1] >> a.key_shift, rmax) + 1u;
    for (uint32_t c = c0; c <= r; ++c) a.cell_start[c] = t;
    if (t == a.n - 1)
        for (uint32_t c = r + 1; c <= a.n_total_cells; ++c) a.cell_start[c] = a.n;
    if (a.ostart) {
        // the same boundary detection one level down: octant = top 3 bits of
        // the sub-cell Morton code, so a cell's particles come octant by octant
        const int os = a.key_shift - 3;
        const uint32_t omax = 8u * a.n_total_cells - 1u;
        const uint32_t ro = min(a.keys[t] >> os, omax);
        const uint32_t o0 = t == 0 ? 0u : min(a.keys[t - 1] >> os, omax) + 1u;
        for (uint32_t c = o0; c <= ro; ++c) a.ostart[c] = t;
        if (t == a.n - 1)
            for (uint32_t c = ro + 1; c <= omax + 1u; ++c) a.ostart[c] = a.n;
    }
}

// fp32 streams + signatures from the current fp64 state (no reorder)
__global__ void __launch_bounds__(256) k_streams(const double* __restrict__ x0,
                                                 const double* __restrict__ x1,
                                                 const double* __restrict__ x2,
                                                 const double* __restrict__ v0,
                                                 const double* __restrict__ v1,
                                                 const double* __restrict__ v2,
                                                 const uint32_t* __restrict__ tag,
                                                 const uint8_t* __restrict__ sp, float4* pos4,
                                                 int4* posq, float4* vel4, uint32_t* sig_out,
                                                 double c0, double c1, double c2, PosQ pq,
                                                 uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double vx = v0[i], vy = v1[i], vz = v2[i];
    const uint32_t t = tag[i];
    const uint32_t sig = make_signature(t, vx, vy, vz);
    const uint32_t tw = sp ? (t | ((uint32_t)sp[i] << 28)) : t;
    pos4[i] = make_float4((float)(x0[i] - c0), (float)(x1[i] - c1), (float)(x2[i] - c2),
                          __uint_as_float(tw));
    posq[i] = posq_of(pq, x0[i], x1[i], x2[i], tw);
    vel4[i] = make_float4((float)vx, (float)vy, (float)vz, __uint_as_float(sig));
    if (sig_out) sig_out[i] = sig;
}

// ------------------------------------------------- neighbor builder
struct BuildArgs {
    const float4* pos4;
    const uint32_t* keys;        // sorted keys (rank = key >> key_shift)
    const uint32_t* cell_start;
    const uint32_t* ostart;      // k_build_range: octant starts [8 n_total_cells + 1] or null
    const uint32_t* stencil;     // [n_local_cells][32]
    const uint8_t* stencil_n;
    const uint8_t* cell_flags;
    uint32_t* entries;
    uint32_t* counts;
    uint32_t* fwalk;    // walk layout: n_eval | force-wrap-flags << 26
    uint2* rowmeta;     // walk layout: (c1 | c2 << 16, s1 | s2 << 16)
    uint32_t* plist;    // k_build_range walk layout: per-tile flat pair lists (j | r << 26 | skin << 31)
    DevErr* err;
    uint32_t n_local, maxn, n_local_cells;
    uint32_t force_block;  // power of two
    int key_shift;
    float cut_c, cut_s;
    float L[3], H[3];
    // k_build_range only: per-slot stencil offset codes and the cell boxes
    const uint8_t* stencil_code;  // [n_local_cells][32]: (ox+1) | (oy+1) << 2 | (oz+1) << 4, 0xFF = never cull
    const float4* cell_lo;        // [n_local_cells]: lower corner in the pos4 frame
    uint8_t* blk_ghost;           // per force block: any row with a ghost partner (j >= n_local)
    float csz[3];                 // cell side per axis (fp32)
    float cut_cull;               // (r_c + skin + margin)^2
    int bucket;                   // k_build_range walk layout: flat lists grouped by partner line
};

// fp32 minimum image, src/core.cpp:129-139 semantics with L, L/2 in fp32
__device__ __forceinline__ float min_image_f(float d, float L, float H) {
    if (d >= H)
        d = __fsub_rn(d, L);
    else if (d < -H)
        d = __fadd_rn(d, L);
    return d;
}

// Inner loop of the builder for one chunk of 32 candidates (one per lane)
// against the nb particles of the current batch: fp32 distance exactly as the
// oracle (no contraction), two ballots, insertion at count + popc(ballot &
// lanemask_lt).  Branch-free: every lane stores once per i, misses and
// overflow go to a trash row (row maxn) of the staging buffer.
template <bool WRAP, int STRIDE>
__device__ __forceinline__ uint32_t build_batch_impl(const float4* slots, uint32_t nb, float4 pj,
                                                     uint32_t j, bool valid, uint32_t ba,
                                                     uint32_t mycnt, uint32_t fl,
                                                     const BuildArgs& a, uint32_t* bufc,
                                                     uint32_t* trash, uint32_t lt, int lane) {
    const uint32_t maxn = a.maxn;
    for (uint32_t ii = 0; ii < nb; ++ii) {
        const float4 pi = slots[ii];
        float dx = __fsub_rn(pi.x, pj.x);
        float dy = __fsub_rn(pi.y, pj.y);
        float dz = __fsub_rn(pi.z, pj.z);
        if (WRAP) {
            if (fl & 1u) dx = min_image_f(dx, a.L[0], a.H[0]);
            if (fl & 2u) dy = min_image_f(dy, a.L[1], a.H[1]);
            if (fl & 4u) dz = min_image_f(dz, a.L[2], a.H[2]);
        }
        const float d2 =
            __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
        const bool cand = valid && j != ba + ii;
        const bool hc = cand && d2 <= a.cut_c;
        const bool hs = cand && !hc && d2 <= a.cut_s;
        const uint32_t mc = __ballot_sync(0xFFFFFFFFu, hc);
        const uint32_t ms = __ballot_sync(0xFFFFFFFFu, hs);
        const uint32_t c = __shfl_sync(0xFFFFFFFFu, mycnt, ii);
        const uint32_t kc = (c & 0xFFFFu) + __popc(mc & lt);
        const uint32_t ks = maxn - 1u - ((c >> 16) + __popc(ms & lt));  // wraps on overflow
        uint32_t kp = hc ? kc : (hs ? ks : maxn);
        kp = min(kp, maxn);
        // misses and overflow: each lane its own trash word (no two lanes of
        // the CTA store to one address)
        *(kp < maxn ? bufc + kp * STRIDE + ii : trash) = j;
        const uint32_t nw = c + __popc(mc) + ((uint32_t)__popc(ms) << 16);
        mycnt = ((uint32_t)lane == ii) ? nw : mycnt;
    }
    return mycnt;
}

// Atomics-free ordered builder (Alg. 3).  One CTA owns P = 32*TILES
// consecutive particles (TILES 32-row tiles of the table); its warps take the
// cells overlapping that range round-robin.  For each cell: the fine stencil is
// never materialized -- each lane locates its candidate k through a shuffle
// binary search over the <=27 stencil-cell prefix sums (P:170's fine stencil
// implicitly), so 32 candidates from several cells share one chunk.  For every
// i of the cell: ballot(core hit) / ballot(skin hit); the insertion point is
// the row count + popc(ballot & lanemask_lt) -- deterministic, ordered, no
// atomics.  Rows are staged in shared memory and written out already
// tile-transposed, so the paper's separate join/transpose passes vanish.
template <int WARPS, int TILES, bool JOINED_OUT>
__global__ void __launch_bounds__(WARPS * 32) k_build(BuildArgs a) {
    constexpr int P = 32 * TILES;
    constexpr int STRIDE = P + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float4* slots = reinterpret_cast<float4*>(smem_raw);
    uint32_t* cnt_s = reinterpret_cast<uint32_t*>(slots + WARPS * 32);
    uint32_t* buf = cnt_s + P;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* trash = buf + (size_t)(a.maxn + 1) * STRIDE + threadIdx.x;  // one word per thread
    const uint32_t i0 = blockIdx.x * P;
    if (i0 >= a.n_local) return;
    const uint32_t iend = min(i0 + (uint32_t)P, a.n_local);
    for (int t = threadIdx.x; t < P; t += WARPS * 32) cnt_s[t] = 0;
    __syncthreads();
    const uint32_t lt = lanemask_lt();
    const uint32_t rl = a.n_local_cells - 1u;  // clamp: a bad key already raised an error
    const uint32_t r0 = min(a.keys[i0] >> a.key_shift, rl);
    const uint32_t r1 = min(a.keys[iend - 1] >> a.key_shift, rl);
    const uint32_t maxn = a.maxn;
    for (uint32_t r = r0 + warp; r <= r1; r += WARPS) {
        const uint32_t ca = max(a.cell_start[r], i0), cb = min(a.cell_start[r + 1], iend);
        if (ca >= cb) continue;
        const uint32_t ns = a.stencil_n[r];
        uint32_t sstart = 0, scount = 0;
        if ((uint32_t)lane < ns) {
            const uint32_t sc = a.stencil[(size_t)r * 32 + lane];
            sstart = a.cell_start[sc];
            scount = a.cell_start[sc + 1] - sstart;
        }
        uint32_t incl = scount;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t excl = incl - scount;
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        const uint32_t fl = a.cell_flags[r] & 7u;
        for (uint32_t ba = ca; ba < cb; ba += 32) {
            const uint32_t nb = min(32u, cb - ba);
            if ((uint32_t)lane < nb) slots[warp * 32 + lane] = a.pos4[ba + lane];
            uint32_t mycnt = 0;  // lane l: core | skin << 16 of particle ba + l
            __syncwarp();
            for (uint32_t base = 0; base < total; base += 32) {
                const uint32_t k = base + lane;
                const bool valid = k < total;
                int s = 0;
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1) {
                    const uint32_t v = __shfl_sync(0xFFFFFFFFu, incl, s + st - 1);
                    if (v <= k) s += st;
                }
                const uint32_t j = __shfl_sync(0xFFFFFFFFu, sstart, s) + k -
                                   __shfl_sync(0xFFFFFFFFu, excl, s);
                float4 pj = make_float4(0.f, 0.f, 0.f, 0.f);
                if (valid) pj = __ldg(a.pos4 + j);
                const uint32_t colb = ba - i0;
                if (fl)
                    mycnt = build_batch_impl<true, STRIDE>(slots + warp * 32, nb, pj, j, valid, ba,
                                                           mycnt, fl, a, buf + colb, trash, lt, lane);
                else
                    mycnt = build_batch_impl<false, STRIDE>(slots + warp * 32, nb, pj, j, valid, ba,
                                                            mycnt, 0u, a, buf + colb, trash, lt, lane);
            }
            if ((uint32_t)lane < nb) cnt_s[ba - i0 + lane] = mycnt;
            __syncwarp();
        }
    }
    __syncthreads();
    // write-out, one 32-row tile per warp: tile-transposed raw_index layout
    for (int tt = warp; tt < TILES; tt += WARPS) {
        const uint32_t ti0 = i0 + 32u * tt;
        if (ti0 >= iend) break;
        const uint32_t col = 32u * tt + lane;
        const uint32_t i = ti0 + lane;
        const bool row = i < iend;
        const uint32_t c = row ? cnt_s[col] : 0u;
        const uint32_t nc = c & 0xFFFFu, nsk = c >> 16;
        if (row && nc + nsk > maxn)
            raise_err(a.err, DPDB_EPHYSICS, EW_OVERFLOW, __float_as_uint(a.pos4[i].w), nc + nsk);
        const uint32_t maxc = __reduce_max_sync(0xFFFFFFFFu, min(nc, maxn));
        const uint32_t maxs = __reduce_max_sync(0xFFFFFFFFu, min(nsk, maxn));
        uint32_t* tb = a.entries + (size_t)ti0 * maxn + lane;
        uint32_t n_eval = 0;
        if (JOINED_OUT) {
            // Walk order for the force kernel (join_core_skin folded in):
            // the entries the force kernel evaluates first -- j outside this
            // particle's force block, or j > i -- core then skin, each ascending;
            // then the in-block j < i entries (that pair is taken by j).  With
            // rowmeta the exact ascending rows are recovered for export.
            const uint32_t ncc = min(nc, maxn), nss = min(nsk, maxn - ncc);
            const uint32_t fb0 = i & ~(a.force_block - 1u);
            auto lower = [&](uint32_t v, bool skin, uint32_t cnt) {  // #entries < v
                uint32_t lo = 0, hi = cnt;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    const uint32_t r = skin ? maxn - 1u - mid : mid;
                    if (buf[r * STRIDE + col] < v)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                return lo;
            };
            const uint32_t c1 = lower(fb0, false, ncc), c2 = lower(i, false, ncc);
            const uint32_t s1 = lower(fb0, true, nss), s2 = lower(i, true, nss);
            const uint32_t A = c1, B = A + (ncc - c2), Cq = B + s1, D = Cq + (nss - s2);
            const uint32_t E = D + (c2 - c1);
            n_eval = D;
            const uint32_t nt = ncc + nss;
            const uint32_t maxt = __reduce_max_sync(0xFFFFFFFFu, nt);
            for (uint32_t k = 0; k < maxt; ++k) {
                uint32_t src;
                if (k < A)
                    src = k;
                else if (k < B)
                    src = c2 + (k - A);
                else if (k < Cq)
                    src = maxn - 1u - (k - B);
                else if (k < D)
                    src = maxn - 1u - (s2 + (k - Cq));
                else if (k < E)
                    src = c1 + (k - D);
                else
                    src = maxn - 1u - (s1 + (k - E));
                tb[(k & 31u) * maxn + (k & ~31u)] = k < nt ? buf[src * STRIDE + col] : 0u;
            }
            if (row) a.rowmeta[i] = make_uint2(c1 | (c2 << 16), s1 | (s2 << 16));
        } else {
            for (uint32_t k = 0; k < maxc; ++k)
                tb[(k & 31u) * maxn + (k & ~31u)] = k < nc ? buf[k * STRIDE + col] : 0u;
            for (uint32_t s = 0; s < maxs; ++s) {
                const uint32_t k = maxn - 1 - s;
                tb[(k & 31u) * maxn + (k & ~31u)] = s < nsk ? buf[k * STRIDE + col] : 0u;
            }
        }
        if (row) {
            const uint32_t ff = (a.cell_flags[min(a.keys[i] >> a.key_shift, rl)] >> 3) & 7u;
            a.counts[i] = min(nc, 8191u) | (min(nsk, 8191u) << 13) | (ff << 26);
            if (JOINED_OUT) a.fwalk[i] = n_eval | (ff << 26);
        }
    }
}

// Lane-per-row ordered builder (same rows as k_build, bit for bit).  Lane l
// of a warp owns row i = 32w + l and walks its own 27 stencil cells in
// ascending rank order and each cell's particles in ascending index order, so
// its row comes out strictly ascending with no atomics, no sort and no
// cross-lane staging; the next stencil cell's range is prefetched one cell
// ahead.  Consecutive rows share most stencil cells (Morton order), so the
// candidate loads of a warp mostly hit the same L1 lines.  Entries are stored
// straight into the 32x32 tile-transposed layout (raw_index):
//   !WALK: the reference split layout, core from the front, skin reversed
//          from the back (inc/neighbor_table.hpp:18-40);
//    WALK: the force walk -- the entries the force kernel evaluates (j outside
//          i's force block, or j > i) ascending from the front, skin entries
//          tagged with bit 31; the in-block j < i entries (that pair is taken
//          by j) from the back.  fwalk = n_front | force flags << 26.
template <bool WALK>
__global__ void __launch_bounds__(256) k_build_lane(BuildArgs a) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool row = i < a.n_local;
    if (__all_sync(0xFFFFFFFFu, !row)) return;
    const uint32_t maxn = a.maxn;
    const uint32_t rl = a.n_local_cells - 1u;  // clamp: a bad key already raised an error
    uint32_t r = 0, ns = 0, fl = 0;
    float4 pi = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row) {
        r = min(a.keys[i] >> a.key_shift, rl);
        ns = a.stencil_n[r];
        fl = a.cell_flags[r];
        pi = a.pos4[i];
    }
    const uint32_t wfl = fl & 7u;
    const bool anywrap = __any_sync(0xFFFFFFFFu, wfl != 0u);
    const uint32_t* srow = a.stencil + (size_t)r * 32;
    const uint32_t fb0 = i & ~(a.force_block - 1u);
    uint32_t s = 0, j = 0, jend = 0, nx_s = 0, nx_e = 0;
    if (ns > 0) {
        const uint32_t sc = srow[0];
        j = a.cell_start[sc];
        jend = a.cell_start[sc + 1];
    }
    if (ns > 1) {
        const uint32_t sc = srow[1];
        nx_s = a.cell_start[sc];
        nx_e = a.cell_start[sc + 1];
    }
    uint32_t* rowp = a.entries + (size_t)(i & ~31u) * maxn + (i & 31u);
    uint32_t kf = 0, kb = 0, nc = 0, nsk = 0;
    bool active = ns > 0;
    while (true) {
        while (active && j >= jend) {  // next non-empty stencil cell
            if (++s >= ns) {
                active = false;
                break;
            }
            j = nx_s;
            jend = nx_e;
            if (s + 1 < ns) {
                const uint32_t sc = srow[s + 1];
                nx_s = a.cell_start[sc];
                nx_e = a.cell_start[sc + 1];
            }
        }
        if (!__any_sync(0xFFFFFFFFu, active)) break;
        if (active) {
            const float4 pj = __ldg(a.pos4 + j);
            float dx = __fsub_rn(pi.x, pj.x);
            float dy = __fsub_rn(pi.y, pj.y);
            float dz = __fsub_rn(pi.z, pj.z);
            if (anywrap) {
                if (wfl & 1u) dx = min_image_f(dx, a.L[0], a.H[0]);
                if (wfl & 2u) dy = min_image_f(dy, a.L[1], a.H[1]);
                if (wfl & 4u) dz = min_image_f(dz, a.L[2], a.H[2]);
            }
            const float d2 =
                __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
            const bool hit = d2 <= a.cut_s && j != i;
            if (hit) {
                const bool core = d2 <= a.cut_c;
                const bool front = WALK ? (j < fb0 || j > i) : core;
                const uint32_t k = front ? kf : maxn - 1u - kb;
                if (kf + kb < maxn)
                    rowp[(k & 31u) * maxn + (k & ~31u)] = (WALK && !core) ? (j | 0x80000000u) : j;
                kf += front;
                kb += !front;
                nc += core;
                nsk += !core;
            }
            ++j;
        }
    }
    if (row) {
        if (nc + nsk > maxn)
            raise_err(a.err, DPDB_EPHYSICS, EW_OVERFLOW, __float_as_uint(pi.w), nc + nsk);
        const uint32_t ff = (fl >> 3) & 7u;
        a.counts[i] = min(nc, 8191u) | (min(nsk, 8191u) << 13) | (ff << 26);
        if (WALK) a.fwalk[i] = min(kf, maxn) | (ff << 26);
    }
}

// Range-list ordered builder (same rows as k_build_lane, bit for bit); the
// step pipeline's default.  One CTA of RB_THREADS lanes owns one force block
// of RB_BLOCK rows and takes it in RB_BLOCK / RB_THREADS passes (lane = row).
// Per row, two phases:
//
//  1. Ranges.  The lane walks its <= 27 stencil cells in ascending rank
//     order, drops the cells whose box lies farther than r_c + skin from its
//     own position (conservative point-to-box distance with a 1e-3 margin, so
//     no cell holding a hit is ever dropped; off when a wrapped axis has < 5
//     cells), cuts out the index range it must not test -- itself, and in the
//     walk layout the in-block j < i (that pair belongs to row j) -- and
//     stores the surviving contiguous index ranges in shared memory
//     (slot-major, bank-conflict free).  The ranges stay ascending, so the
//     row stays ordered.
//  2. Walk.  The lane tests its candidates range after range with one
//     position load, the oracle's fp32 distance and one compare each.  A
//     cursor runs two candidates ahead of the test (two position loads in
//     flight per lane); moving to the next range is two shared loads, so
//     lanes never diverge on cell switches.  Hits are stored straight into
//     the 32x32 tile-transposed layout (raw_index).  No atomics and no sort
//     for the rows.
//
// !WALK: the reference split layout (core from the front, skin reversed from
//        the back), counts = core | skin << 13 | flags << 26.
// GH: the context has ghost rows (a brick); only then is each hit tested for a
//     ghost partner (the block's blk_ghost flag).
//  WALK: only the entries the force kernel evaluates (j outside the block or
//        j > i) -- the row's "front" entries -- are kept: the walk stores them
//        in the row's tile-transposed scratch row, then the warp writes the
//        tile's flat pair list (the force kernel's input) as items
//        j | row << 26 | skin << 31 grouped by the partner's cache line (a
//        counting sort on bits 3-6 of j; each row's items stay ascending
//        within a group); fwalk = n_front | flags.  The in-block j < i
//        entries are not stored -- they are exactly the transposes of the
//        block's front entries (unwalk restores them).  No atomics: the full
//        row length n_front + n_back is bounded by n_front + the length of the
//        cut-out index ranges; only a row whose bound exceeds max_neighbors
//        walks its cut-out ranges (cut_hits) to count n_back exactly for the
//        overflow check.
// predicated select (keeps the compiler from branching on small selects)
__device__ __forceinline__ float fsel(bool p, float a, float b) {
    float r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.f32 %0, %1, %2, q;\n\t}"
        : "=f"(r)
        : "f"(a), "f"(b), "r"((uint32_t)p));
    return r;
}

constexpr int RB_BLOCK = 32 * DPDB_FORCE_TPW * DPDB_FORCE_WARPS;  // == FORCE_BLOCK (force.cuh)
#ifndef DPDB_RB_THREADS
#define DPDB_RB_THREADS 256
#endif
constexpr int RB_THREADS = DPDB_RB_THREADS;  // lanes per CTA (RB_BLOCK / RB_THREADS passes)
constexpr int RB_SLOTS = 29;     // 27 stencil cells + one split by the cut-out + a trash slot
constexpr size_t RB_SMEM = (size_t)RB_SLOTS * RB_THREADS * 6;
constexpr uint32_t RB_NONE = 0xFFFFFFFFu;
#ifndef DPDB_RB_AHEAD
#define DPDB_RB_AHEAD 2
#endif
constexpr int RB_AHEAD = DPDB_RB_AHEAD;
// flat-list bucket of a partner: bits [BUCKET_SHIFT, BUCKET_SHIFT + 4) of j
// (A/B: a multiplicative hash of the line j >> 3 instead was 0.7% slower)
#ifndef DPDB_BUCKET_SHIFT
#define DPDB_BUCKET_SHIFT 3
#endif
constexpr int BUCKET_SHIFT = DPDB_BUCKET_SHIFT;  // walk lookahead (A/B: 2 vs 4 position loads in flight per lane)

// Rows whose front count + cut-out length could exceed max_neighbors: the
// exact number of in-block j < i within r_c + skin (the row's back entries),
// the builder's own fp32 test over every stencil cell's [max(start, b0), i).
__device__ __noinline__ uint32_t cut_hits(const float4* __restrict__ pos4, const uint32_t* __restrict__ stencil,
                                          uint32_t ns, const uint32_t* __restrict__ cell_start, uint32_t i,
                                          uint32_t b0, float4 pi, uint32_t wfl, float3 L, float3 H, float cut_s) {
    uint32_t n = 0;
    for (uint32_t s = 0; s < ns; ++s) {
        const uint32_t c = stencil[s];
        const uint32_t st = max(cell_start[c], b0), en = min(cell_start[c + 1], i);
        for (uint32_t j = st; j < en; ++j) {
            const float4 pj = pos4[j];
            float dx = __fsub_rn(pi.x, pj.x), dy = __fsub_rn(pi.y, pj.y), dz = __fsub_rn(pi.z, pj.z);
            if (wfl & 1u) dx = min_image_f(dx, L.x, H.x);
            if (wfl & 2u) dy = min_image_f(dy, L.y, H.y);
            if (wfl & 4u) dz = min_image_f(dz, L.z, H.z);
            const float d2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
            n += d2 <= cut_s;
        }
    }
    return n;
}

#ifndef DPDB_RB_MINB
#define DPDB_RB_MINB (1024 / DPDB_RB_THREADS)
#endif
template <bool WALK, bool GH>
__global__ void __launch_bounds__(RB_THREADS, DPDB_RB_MINB) k_build_range(BuildArgs a) {
    extern __shared__ uint32_t rb_smem[];  // RB_SMEM bytes (dynamic: > 48 KB)
    uint32_t(*rs)[RB_THREADS] = reinterpret_cast<uint32_t(*)[RB_THREADS]>(rb_smem);
    uint16_t(*rl)[RB_THREADS] =
        reinterpret_cast<uint16_t(*)[RB_THREADS]>(rb_smem + RB_SLOTS * RB_THREADS);
    const uint32_t t = threadIdx.x;
    const uint32_t b0 = blockIdx.x * RB_BLOCK;
    const uint32_t bn = min((uint32_t)RB_BLOCK, a.n_local - b0);
    const uint32_t bend = b0 + bn;
    const uint32_t maxn = a.maxn;
    __shared__ uint32_t ghost_seen;
    if (t == 0) ghost_seen = 0u;
    __syncthreads();
    uint32_t cnt[RB_BLOCK / RB_THREADS];  // nc | nsk << 16 per pass
    uint32_t kfs[RB_BLOCK / RB_THREADS];

#pragma unroll 1
    for (int pass = 0; pass < RB_BLOCK / RB_THREADS; ++pass) {
        const uint32_t i = b0 + pass * RB_THREADS + t;
        const bool row = i < bend;
        uint32_t r = 0, ns = 0, fl = 0;
        float4 pi = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row) {
            r = min(a.keys[i] >> a.key_shift, a.n_local_cells - 1u);
            ns = a.stencil_n[r];
            fl = a.cell_flags[r];
            pi = a.pos4[i];
        }
        // ---- phase 1: ranges.  Per axis, the squared distance from pi to the
        // lower / upper half of the cells at offset -1, 0, +1 (slab [lo, hi]:
        // max(0, lo - l, l - hi)); an octant of a stencil cell is in reach iff
        // the three axis terms sum to <= cut_cull.  The kept range of a cell is
        // trimmed to [first kept octant, last kept octant]: particles are
        // sorted octant by octant inside a cell, so this stays one range.
        float hd[3][6];
        {
            const float4 lo = row ? a.cell_lo[r] : make_float4(0.f, 0.f, 0.f, 0.f);
            const float l[3] = {pi.x - lo.x, pi.y - lo.y, pi.z - lo.z};
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float h = 0.5f * a.csz[k];
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    const float s0 = (float)(q - 2) * h, s1 = s0 + h;  // slab [-a + q a/2, ...]
                    const float d = fmaxf(fmaxf(s0 - l[k], l[k] - s1), 0.f);
                    hd[k][q] = d * d;
                }
            }
        }
        const uint32_t cut_lo = WALK ? b0 : i;  // excluded index range [cut_lo, i]
        const uint32_t* otab = a.ostart ? a.ostart : a.cell_start;
        const int osh = a.ostart ? 3 : 0;
        uint32_t nr = 0, cutl = 0;
        const uint32_t* srow = a.stencil + (size_t)r * 32;
        const uint8_t* crow = a.stencil_code + (size_t)r * 32;
        bool big = false;
#pragma unroll 1
        for (uint32_t s0 = 0; s0 < ns; s0 += 4) {
            uint32_t st[4], en[4], lo_i[4], hi_i[4];
            bool kp[4];
            // four stencil slots per 16-byte load (rows are padded to 32)
            const uint4 sc4 = *reinterpret_cast<const uint4*>(srow + s0);
            const uint32_t cd4 = *reinterpret_cast<const uint32_t*>(crow + s0);
            const uint32_t sc[4] = {sc4.x, sc4.y, sc4.z, sc4.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const bool v = s0 + q < ns;
                const uint32_t c = (cd4 >> (8 * q)) & 0xFFu;
                uint32_t m = 0xFFu;
                if (c != 0xFFu) {
                    float d0[3], d1[3];  // lower / upper half of the cell at this offset, per axis
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const uint32_t o = (c >> (2 * k)) & 3u;
                        d0[k] = fsel(o == 2u, hd[k][4], fsel(o == 0u, hd[k][0], hd[k][2]));
                        d1[k] = fsel(o == 2u, hd[k][5], fsel(o == 0u, hd[k][1], hd[k][3]));
                    }
                    const float yz[4] = {d0[1] + d0[2], d1[1] + d0[2], d0[1] + d1[2], d1[1] + d1[2]};
                    m = 0u;
#pragma unroll
                    for (int h = 0; h < 8; ++h)
                        m |= (uint32_t)(((h & 1) ? d1[0] : d0[0]) + yz[h >> 1] <= a.cut_cull) << h;
                }
                if (!a.ostart) m = m ? 1u : 0u;  // cell granularity only
                kp[q] = v && m != 0u;
                lo_i[q] = (sc[q] << osh) + (m ? __ffs(m) - 1 : 0);
                hi_i[q] = (sc[q] << osh) + (m ? 32 - __clz(m) : 1);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                st[q] = otab[lo_i[q]];
                en[q] = otab[hi_i[q]];
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                // branch-free: both pieces are always written, nr advances only
                // over the kept non-empty ones (slot RB_SLOTS - 1 absorbs the rest)
                const bool keep = kp[q];
                const uint32_t e1 = min(en[q], cut_lo), s2 = max(st[q], i + 1u);
                if (WALK) {  // cut-out [max(st, b0), min(en, i)): the row's possible back entries
                    const uint32_t c0 = max(st[q], cut_lo), c1 = min(en[q], i);
                    cutl += keep && c1 > c0 ? c1 - c0 : 0u;
                }
                const uint32_t l1 = e1 > st[q] ? e1 - st[q] : 0u;
                const uint32_t l2 = en[q] > s2 ? en[q] - s2 : 0u;
                big |= keep && max(l1, l2) > 0xFFFFu;
                rs[nr][t] = st[q];
                rl[nr][t] = (uint16_t)min(l1, 0xFFFFu);
                nr += keep && l1;
                rs[nr][t] = s2;
                rl[nr][t] = (uint16_t)min(l2, 0xFFFFu);
                nr += keep && l2;
            }
        }
        if (big) raise_err(a.err, DPDB_EPHYSICS, EW_OVERFLOW, __float_as_uint(pi.w), 0xFFFFu);
        // ---- phase 2: walk the ranges, cursor two candidates ahead.  Written
        // branch-light: lanes past their last candidate keep testing their own
        // position (masked by v), and the range switch is a predicated pair of
        // shared loads.
        const uint32_t wfl = fl & 7u;
        const bool anywrap = __any_sync(0xFFFFFFFFu, wfl != 0u);
        uint32_t cs = 0, cj = 0, ce = 0;  // cursor: range, next index, range end
        if (nr) {
            cj = rs[0][t];
            ce = cj + rl[0][t];
        }
        // The next candidate, or i itself once the lane's ranges are exhausted
        // (the ranges never hold i: the sentinel needs no separate flag, which
        // the compiler would carry as a byte or a 0/1 word across the loop).
        // Ranges are non-empty, so a switch always yields a candidate.
        auto adv = [&]() -> uint32_t {
            if (cj >= ce && cs + 1 < nr) {
                ++cs;
                cj = rs[cs][t];
                ce = cj + rl[cs][t];
            }
            const bool v = cj < ce;
            const uint32_t j = v ? cj : i;
            cj += v;
            return j;
        };
        // RB_AHEAD candidates in flight per lane (cursor RB_AHEAD ahead of the test)
        uint32_t jq[RB_AHEAD];
        float4 pq[RB_AHEAD];
#pragma unroll
        for (int q = 0; q < RB_AHEAD; ++q) jq[q] = adv();
#pragma unroll
        for (int q = 0; q < RB_AHEAD; ++q) pq[q] = __ldg(a.pos4 + jq[q]);
        uint32_t* rowp = a.entries + (size_t)(i & ~31u) * maxn + (i & 31u);
        uint32_t kf = 0, kb = 0, nc = 0, nsk = 0;
        const float cut_s = a.cut_s, cut_c = a.cut_c;
        // branch-free min image (min_image_f semantics): axes without wrap get
        // H = +inf, so neither correction fires
        const float inf = __int_as_float(0x7F800000);
        const float Lx = a.L[0], Ly = a.L[1], Lz = a.L[2];
        const float Hx = (wfl & 1u) ? a.H[0] : inf, Hy = (wfl & 2u) ? a.H[1] : inf,
                    Hz = (wfl & 4u) ? a.H[2] : inf;
        auto mimg = [](float d, float L, float H) {
            const float lo = __fsub_rn(d, L), hi = __fadd_rn(d, L);
            return d >= H ? lo : (d < -H ? hi : d);
        };
        // the walk is instantiated twice: warps with no wrapped row (the bulk)
        // issue no minimum-image instructions at all
        auto walk = [&](auto wrapc) {
            constexpr bool WRAPW = decltype(wrapc)::value;
            auto test = [&](uint32_t j, float4 pj) {
                float dx = __fsub_rn(pi.x, pj.x);
                float dy = __fsub_rn(pi.y, pj.y);
                float dz = __fsub_rn(pi.z, pj.z);
                if (WRAPW) {
                    dx = mimg(dx, Lx, Hx);
                    dy = mimg(dy, Ly, Hy);
                    dz = mimg(dz, Lz, Hz);
                }
                const float d2 =
                    __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
                const bool hit = j != i && d2 <= cut_s;
                const bool core = d2 <= cut_c;
                if (GH && hit && j >= a.n_local) ghost_seen = 1u;  // same value from every writer
                if (WALK) {
                    // predicated store into the tile-transposed scratch rows (no
                    // branch); the slot of entry kf from kf itself (raw_index)
                    const uint32_t* wp = rowp + ((kf & 31u) * maxn + (kf & ~31u));
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.global.u32 [%0], %1;\n\t}"
                                 ::"l"(wp), "r"(core ? j : (j | 0x80000000u)),
                                 "r"((uint32_t)(hit && kf < maxn)));
                    kf += hit;
                } else {
                    const uint32_t k = core ? kf : maxn - 1u - kb;
                    if (hit && kf + kb < maxn) rowp[(k & 31u) * maxn + (k & ~31u)] = j;
                    kf += hit && core;
                    kb += hit && !core;
                }
                nc += hit && core;
                nsk += hit && !core;
            };
            while (__any_sync(0xFFFFFFFFu, jq[0] != i)) {
#pragma unroll
                for (int q = 0; q < RB_AHEAD; ++q) {
                    test(jq[q], pq[q]);
                    jq[q] = adv();
                    pq[q] = __ldg(a.pos4 + jq[q]);
                }
            }
        };
        if (anywrap)
            walk(std::true_type{});
        else
            walk(std::false_type{});
        cnt[pass] = min(nc, 0xFFFFu) | (min(nsk, 0xFFFFu) << 16);  // saturate: >= 65535 overflows maxn anyway
        kfs[pass] = kf;
        if (WALK && a.bucket) {
            // The tile's flat pair list for the force kernel, grouped by the
            // partner's cache line: the 32 rows of a tile are neighbours and
            // share most candidates (C3: ~577 items, ~160 distinct partners in
            // ~47 lines of 8 particles), so with the items of a line side by
            // side a 32-lane gather of the force kernel touches a few lines
            // instead of ~20 (row order) and its pair batches hold distinct
            // owner rows.  A counting sort on 4 bits of the line (j >> 3): each
            // lane (row) counts its own items in its column of a [bucket][lane]
            // u16 histogram (this warp's share of rl), a scan turns the counts
            // into offsets in (bucket, row) order, the items are placed in this
            // warp's share of rs (both free after the walk) and written out
            // coalesced.  No atomics, deterministic; order = bucket, row,
            // ascending j.  Tiles longer than the staging keep the row order.
            const uint32_t lane = t & 31u, wbase = t & ~31u;
            const uint32_t kfc = min(kf, maxn);
            uint32_t tot = kfc;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) tot += __shfl_xor_sync(0xFFFFFFFFu, tot, d);
            constexpr uint32_t STG = RB_SLOTS * 32;  // staging words per warp
            uint32_t* tl = a.plist + (size_t)(i & ~31u) * maxn;
            const uint32_t rowbits = lane << 26;
            auto bucket_of = [](uint32_t e) { return (e >> BUCKET_SHIFT) & 15u; };
            auto hist = [&](uint32_t h) -> uint16_t& { return rl[h >> 5][wbase + (h & 31u)]; };  // h = b*32 + lane
            __syncwarp();
            if (tot <= STG) {
#pragma unroll
                for (uint32_t b = 0; b < 16; ++b) hist(b * 32u + lane) = 0;
                for (uint32_t m = 0; m < kfc; ++m) {
                    uint16_t& h = hist(bucket_of(rowp[(m & 31u) * maxn + (m & ~31u)]) * 32u + lane);
                    h = (uint16_t)(h + 1u);
                }
                __syncwarp();
                // exclusive offsets in (bucket, lane) order: lanes 2b, 2b+1
                // scan the two halves of bucket b's 32 counters
                {
                    const uint32_t b = lane >> 1, l0 = (lane & 1u) * 16u;
                    uint32_t c[16], run = 0;
#pragma unroll
                    for (uint32_t l = 0; l < 16; ++l) {
                        c[l] = hist(b * 32u + l0 + l);
                        run += c[l];
                    }
                    uint32_t incl = run;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                        if (lane >= (uint32_t)d) incl += y;
                    }
                    uint32_t o = incl - run;
                    __syncwarp();
#pragma unroll
                    for (uint32_t l = 0; l < 16; ++l) {
                        hist(b * 32u + l0 + l) = (uint16_t)o;
                        o += c[l];
                    }
                }
                __syncwarp();
                for (uint32_t m = 0; m < kfc; ++m) {
                    const uint32_t e = rowp[(m & 31u) * maxn + (m & ~31u)];
                    uint16_t& h = hist(bucket_of(e) * 32u + lane);
                    const uint32_t q = h;
                    rs[q >> 5][wbase + (q & 31u)] = (e & 0x83FFFFFFu) | rowbits;
                    h = (uint16_t)(q + 1u);
                }
                __syncwarp();
                for (uint32_t q = lane; q < tot; q += 32) tl[q] = rs[q >> 5][wbase + (q & 31u)];
                __syncwarp();
            } else {  // row order, straight from the rows
                uint32_t off = kfc;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, off, d);
                    if (lane >= (uint32_t)d) off += y;
                }
                off -= kfc;
                for (uint32_t m = 0; m < kfc; ++m)
                    tl[off + m] = (rowp[(m & 31u) * maxn + (m & ~31u)] & 0x83FFFFFFu) | rowbits;
            }
        } else if (WALK) {
            // The tile's flat pair list for the force kernel: the warp's rows
            // back-to-back in row order (exclusive warp scan of the row
            // lengths), each item j | row << 26 | skin << 31.  The rows just
            // written are read back coalesced (L1/L2 hits) and staged in this
            // warp's columns of the range-list shared memory (free after the
            // walk) so the list is written coalesced.
            const uint32_t lane = t & 31u, wbase = t & ~31u;
            const uint32_t kfc = min(kf, maxn);
            uint32_t off = kfc;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, off, d);
                if (lane >= (uint32_t)d) off += y;
            }
            const uint32_t tot = __shfl_sync(0xFFFFFFFFu, off, 31);
            off -= kfc;
            const uint32_t maxkf = __reduce_max_sync(0xFFFFFFFFu, kfc);
            const uint32_t rowbits = lane << 26;
            uint32_t* tl = a.plist + (size_t)(i & ~31u) * maxn;
            constexpr uint32_t STG = RB_SLOTS * 32;  // staging words per warp
            __syncwarp();
            for (uint32_t c0 = 0; c0 < tot; c0 += STG) {
                for (uint32_t m = 0; m < maxkf; ++m) {
                    const uint32_t e = rowp[(m & 31u) * maxn + (m & ~31u)];
                    const uint32_t q = off + m - c0;  // wraps (large) below the round
                    if (m < kfc && q < STG) rs[q >> 5][wbase + (q & 31u)] = (e & 0x83FFFFFFu) | rowbits;
                }
                __syncwarp();
                const uint32_t len = min(tot - c0, STG);
                for (uint32_t q = lane; q < len; q += 32) tl[c0 + q] = rs[q >> 5][wbase + (q & 31u)];
                __syncwarp();
            }
        }
        if (WALK && row && kf + cutl > maxn) {  // the bound cannot rule out an overflow: count exactly
            const uint32_t nb = cut_hits(a.pos4, a.stencil + (size_t)r * 32, ns, a.cell_start, i, b0, pi, wfl,
                                         make_float3(a.L[0], a.L[1], a.L[2]),
                                         make_float3(a.H[0], a.H[1], a.H[2]), a.cut_s);
            if (kf + nb > maxn) raise_err(a.err, DPDB_EPHYSICS, EW_OVERFLOW, __float_as_uint(pi.w), kf + nb);
        }
    }
    __syncthreads();
    if (t == 0 && a.blk_ghost) a.blk_ghost[blockIdx.x] = ghost_seen ? 1 : 0;
#pragma unroll
    for (int pass = 0; pass < RB_BLOCK / RB_THREADS; ++pass) {
        const uint32_t i = b0 + pass * RB_THREADS + t;
        if (i >= bend) break;
        const uint32_t nc = cnt[pass] & 0xFFFFu, nsk = cnt[pass] >> 16;
        const uint32_t r = min(a.keys[i] >> a.key_shift, a.n_local_cells - 1u);
        const uint32_t ff = (a.cell_flags[r] >> 3) & 7u;
        if (WALK) {  // counts of the full rows are formed on export (unwalk)
            a.fwalk[i] = min(kfs[pass], maxn) | (ff << 26);
            continue;
        }
        if (nc + nsk > maxn)
            raise_err(a.err, DPDB_EPHYSICS, EW_OVERFLOW, __float_as_uint(a.pos4[i].w), nc + nsk);
        a.counts[i] = min(nc, 8191u) | (min(nsk, 8191u) << 13) | (ff << 26);
    }
}

// layout transforms of the table
__device__ __forceinline__ size_t raw_index(bool tiled, uint32_t maxn, uint32_t i, uint32_t k) {
    return tiled ? (size_t)((i & ~31u) + (k & 31u)) * maxn + (k & ~31u) + (i & 31u)
                 : (size_t)i * maxn + k;
}

__global__ void k_join(uint32_t* entries, const uint32_t* counts, uint32_t n, uint32_t maxn,
                       bool tiled) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c = counts[i], nc = c & 0x1FFFu, ns = (c >> 13) & 0x1FFFu;
    // skin entries sit at maxn-1-s; the joined slot nc+s < maxn-1-s until they meet
    for (uint32_t s = 0; s < ns; ++s) {
        const uint32_t from = maxn - 1 - s, to = nc + s;
        if (to >= from) break;
        // swap keeps the not-yet-moved tail intact
        const size_t pf = raw_index(tiled, maxn, i, from), pt = raw_index(tiled, maxn, i, to);
        const uint32_t tmp = entries[pt];
        entries[pt] = entries[pf];
        entries[pf] = tmp;
    }
}

// in-place 32x32 tile transpose; one CTA (32x8 threads) per tile
__global__ void k_tile_transpose(uint32_t* entries, uint32_t n_rows_pad, uint32_t maxn) {
    __shared__ uint32_t t[32][33];
    const uint32_t tr = blockIdx.y * 32, tc = blockIdx.x * 32;
    for (int y = threadIdx.y; y < 32; y += 8)
        t[y][threadIdx.x] = entries[(size_t)(tr + y) * maxn + tc + threadIdx.x];
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += 8)
        entries[(size_t)(tr + y) * maxn + tc + threadIdx.x] = t[threadIdx.x][y];
}

// Harmonic bonds: F = -K (r - r0) e on each endpoint.  Bonds are
// stored as a static CSR over TAGS (each bond at both endpoints), resolved
// to current indices through index_of_tag (refreshed at every reorder), and
// evaluated per particle -- deterministic, no atomics, like the full pair list.
struct BondArgs {
    const uint32_t* boff;       // [max_tag + 2]
    const uint32_t* bpartner;   // partner tag
    const float* bk;
    const float* br0;
    const uint8_t* bstyle;      // 0 harmonic, 1 FENE (unpinned)
    const uint32_t* aoff;       // angles: [max_tag + 2] CSR over tags, or null
    const uint4* arec;          // (tag of the first other, tag of the second other, role, 0)
    const float* ak;
    const float* at0;
    const uint32_t* index_of_tag;
    const int4* posq;   // the pair-force frame (minimum image on wrap axes by int32 wrap)
    float* f[3];
    DevErr* err;
    float qs[3];        // length per posq quantum
    uint32_t n, max_tag;
    uint32_t tag_mask;  // 0x0FFFFFFF when species ride in pos4.w
};

__device__ __forceinline__ void bonded_delta(const BondArgs& a, const int4& p, const int4& q,
                                             float d[3]) {
    d[0] = (float)(p.x - q.x) * a.qs[0];
    d[1] = (float)(p.y - q.y) * a.qs[1];
    d[2] = (float)(p.z - q.z) * a.qs[2];
}

// Bonded force on particle i: every bond of i in CSR order -- harmonic
// F = -K (r - r0) e or FENE F = -K r / (1 - (r / R0)^2) e (R0 in the
// r0 slot; r >= R0 is a physics error) -- then every angle i belongs to, a
// harmonic angle U = K (theta - theta0)^2 / 2 around the middle bead b of
// (a, b, c): F_a = K (theta - theta0) / sin(theta) (r2 / (|r1||r2|) - cos(theta)
// r1 / |r1|^2) with r1 = x_a - x_b, r2 = x_c - x_b, F_c likewise, F_b = -(F_a + F_c).
// FENE and angles have no reference implementation (SURVEY hard part 7:
// restated from the standard formulas, unpinned).  false if i has no bonded
// term.  Shared by k_bonds and the pair kernel epilogue (no atomics: each
// particle sums its own terms).
// STYLED: bond styles (FENE) and angle terms too (k_bonds).  The pair
// kernel's fused epilogue carries harmonic bonds alone (STYLED = false), so
// its register allocation does not pay for the rest; contexts with FENE bonds
// or angles run k_bonds after the pair kernel, unfused.
template <bool STYLED>
__device__ __forceinline__ bool bond_force(const BondArgs& a, uint32_t i, float& fx, float& fy,
                                           float& fz) {
    const int4 pi = a.posq[i];
    const uint32_t tag = (uint32_t)pi.w & a.tag_mask;
    if (tag > a.max_tag) return false;
    const uint32_t b0 = a.boff[tag], b1 = a.boff[tag + 1];
    const uint32_t e0 = STYLED && a.aoff ? a.aoff[tag] : 0u, e1 = STYLED && a.aoff ? a.aoff[tag + 1] : 0u;
    if (b0 == b1 && e0 == e1) return false;
    fx = fy = fz = 0.f;
    uint32_t fene_bad = 0;  // partner tag of an overstretched FENE bond (raised once)
    for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t pt = a.bpartner[b];
        const uint32_t j = a.index_of_tag[pt];
        if (j >= a.n) {
            raise_err(a.err, DPDB_EPHYSICS, EW_BOND, tag, pt);
            continue;
        }
        float d[3];
        bonded_delta(a, pi, a.posq[j], d);
        const float r = sqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        const float k = a.bk[b], r0 = a.br0[b];
        const bool fene = STYLED && a.bstyle && a.bstyle[b] == 1;
        const float x = r / r0;
        const bool stretched = fene && !(x < 1.f);
        fene_bad = stretched ? pt | 0x80000000u : fene_bad;
        const float cc = fene ? (stretched ? 0.f : -k / (1.f - x * x))
                              : (r > 0.f ? -k * (r - r0) / r : 0.f);
        fx += cc * d[0];
        fy += cc * d[1];
        fz += cc * d[2];
    }
    if (STYLED && fene_bad) raise_err(a.err, DPDB_EPHYSICS, EW_FENE, tag, fene_bad & 0x7FFFFFFFu);
    for (uint32_t e = e0; STYLED && e < e1; ++e) {
        const uint4 rec = a.arec[e];
        const uint32_t j1 = a.index_of_tag[rec.x], j2 = a.index_of_tag[rec.y];
        if (j1 >= a.n || j2 >= a.n) {
            raise_err(a.err, DPDB_EPHYSICS, EW_BOND, tag, j1 >= a.n ? rec.x : rec.y);
            continue;
        }
        // roles: 0 -> i is end a (others: b, c); 1 -> i is the middle b (a, c);
        // 2 -> i is end c (b, a)
        const int4 q1 = a.posq[j1], q2 = a.posq[j2];
        const int4 pa = rec.z == 1 ? q1 : pi;
        const int4 pb = rec.z == 1 ? pi : q1;
        const int4 pc = q2;  // role 0: c; role 1: c; role 2: a (symmetric in a <-> c)
        float r1[3], r2[3];
        bonded_delta(a, pa, pb, r1);
        bonded_delta(a, pc, pb, r2);
        const float l1 = sqrtf(r1[0] * r1[0] + r1[1] * r1[1] + r1[2] * r1[2]);
        const float l2 = sqrtf(r2[0] * r2[0] + r2[1] * r2[1] + r2[2] * r2[2]);
        if (!(l1 > 0.f && l2 > 0.f)) continue;
        float c = (r1[0] * r2[0] + r1[1] * r2[1] + r1[2] * r2[2]) / (l1 * l2);
        c = fminf(fmaxf(c, -1.f), 1.f);
        const float th = acosf(c);
        const float sn = fmaxf(sqrtf(fmaxf(1.f - c * c, 0.f)), 1e-6f);
        const float g = a.ak[e] * (th - a.at0[e]) / sn;
        float fa[3], fc[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            fa[k] = g * (r2[k] / (l1 * l2) - c * r1[k] / (l1 * l1));
            fc[k] = g * (r1[k] / (l1 * l2) - c * r2[k] / (l2 * l2));
        }
        if (rec.z == 1) {  // middle bead
            fx -= fa[0] + fc[0];
            fy -= fa[1] + fc[1];
            fz -= fa[2] + fc[2];
        } else {  // an end (roles 0 and 2 are mirror images: pa is this particle)
            fx += fa[0];
            fy += fa[1];
            fz += fa[2];
        }
    }
    return true;
}

__global__ void k_bonds(BondArgs a) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    float fx, fy, fz;
    if (!bond_force<true>(a, i, fx, fy, fz)) return;
    a.f[0][i] += fx;
    a.f[1][i] += fy;
    a.f[2][i] += fz;
}

#include "force.cuh"
#include "domain.cuh"

// --------------------------------------------------- observables
// deterministic two-level reductions (fixed tree, fixed partial order)
__global__ void __launch_bounds__(256) k_sum3(const double* __restrict__ a0,
                                              const double* __restrict__ a1,
                                              const double* __restrict__ a2, const double* mean,
                                              uint32_t n, double* partial) {
    __shared__ double s[4][256];
    double acc[4] = {0, 0, 0, 0};
    const double m0 = mean ? mean[0] : 0.0, m1 = mean ? mean[1] : 0.0, m2 = mean ? mean[2] : 0.0;
    for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
        const double x = a0[i], y = a1[i], z = a2[i];
        acc[0] += x;
        acc[1] += y;
        acc[2] += z;
        const double dx = x - m0, dy = y - m1, dz = z - m2;
        acc[3] += dx * dx + dy * dy + dz * dz;
    }
    for (int q = 0; q < 4; ++q) s[q][threadIdx.x] = acc[q];
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < (unsigned)o)
            for (int q = 0; q < 4; ++q) s[q][threadIdx.x] += s[q][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x < 4) partial[blockIdx.x * 4 + threadIdx.x] = s[threadIdx.x][0];
}

// fixed-order sum of the block partials: thread t adds blocks t, t + 256, ...
// then block_sum4 (deterministic for a given nblocks); launch with 256 threads
__global__ void __launch_bounds__(256) k_sum_partials(const double* partial, int nblocks, double* out) {
    double acc[4] = {0, 0, 0, 0};
    fold_partials4(partial, (uint32_t)nblocks, acc);
    block_sum4<256>(acc, out);
}

__global__ void k_mean_from_sum(double* sum, double inv_n) {
    if (threadIdx.x < 3) sum[4 + threadIdx.x] = sum[threadIdx.x] * inv_n;
}

// ------------------------------------------------------ init_random
// init_random (restated, the reference's init.cpp is not
// shipped) as counter-based draws, so every particle is independent: draw c of
// stream `seed` is tea_hash(16, seed, c).  Particle i: position component k from
// draw 6i + k (uniform in [lo, hi)), velocity component k = sqrt(kT) *
// gaussian(draw 6i + 3 + k) -- bit-exact with the oracle's init_fluid.  Chains
// come first (chain c = particles [c L, c L + L)): bead 0 is placed like a
// solvent particle, bead b > 0 at bead b-1 + r0 * u with the unit vector u
// from draws 6i (cos theta = 2 u - 1) and 6i + 1 (phi = 2 pi u), wrapped
// periodically -- the SPEC's random walk with step r0.
struct InitArgs {
    double* x[3];
    double* v[3];
    uint32_t* tag;
    uint8_t* sp;
    uint32_t* mol;
    double lo[3], hi[3];
    int periodic[3];
    double sk;  // sqrt(kT)
    uint32_t seed, n, n_chains, chain_len;
    uint8_t chain_sp[32];
    uint8_t solvent_sp;
    double r0;
};

__device__ __forceinline__ uint2 tea16_draw(uint32_t seed, uint32_t c) {
    uint32_t a = seed, b = c;
    tea_rounds(16, a, b);
    return make_uint2(a, b);
}

__global__ void __launch_bounds__(256) k_init_particles(InitArgs a) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    const uint32_t nb = a.n_chains * a.chain_len;
    const bool bead = i < nb;
    const uint32_t b = bead ? i % a.chain_len : 0u;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (b == 0) {
            const uint2 h = tea16_draw(a.seed, 6u * i + (uint32_t)k);
            const double L = __dsub_rn(a.hi[k], a.lo[k]);
            double p = __dadd_rn(a.lo[k], __dmul_rn(L, (double)h.x * 0x1p-32));
            if (p >= a.hi[k]) p = a.lo[k];
            a.x[k][i] = p;
        }
        const uint2 g = tea16_draw(a.seed, 6u * i + 3u + (uint32_t)k);
        a.v[k][i] = __dmul_rn(a.sk, gaussian64(g.x, g.y));
    }
    a.tag[i] = i + 1u;
    a.sp[i] = bead ? a.chain_sp[b] : a.solvent_sp;
    if (a.mol) a.mol[i] = bead ? i / a.chain_len + 1u : 0u;
}

// one thread per chain: the random walk of beads 1..L-1
__global__ void __launch_bounds__(128) k_init_chains(InitArgs a) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= a.n_chains) return;
    uint32_t i = c * a.chain_len;
    double p[3] = {a.x[0][i], a.x[1][i], a.x[2][i]};
    for (uint32_t b = 1; b < a.chain_len; ++b) {
        ++i;
        const uint2 h0 = tea16_draw(a.seed, 6u * i), h1 = tea16_draw(a.seed, 6u * i + 1u);
        const double ct = __dsub_rn(__dmul_rn(2.0, (double)h0.x * 0x1p-32), 1.0);
        const double st = sqrt(fmax(__dsub_rn(1.0, __dmul_rn(ct, ct)), 0.0));
        const double ph = __dmul_rn(6.283185307179586, (double)h1.x * 0x1p-32);
        const double u[3] = {__dmul_rn(st, cos(ph)), __dmul_rn(st, sin(ph)), ct};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double q = __dadd_rn(p[k], __dmul_rn(a.r0, u[k]));
            const double L = __dsub_rn(a.hi[k], a.lo[k]);
            if (a.periodic[k]) {
                if (q < a.lo[k]) q = __dadd_rn(q, L);
                else if (q >= a.hi[k]) q = __dsub_rn(q, L);
                if (q >= a.hi[k] || q < a.lo[k]) q = a.lo[k];
            } else {  // closed axis: reflect back inside
                if (q < a.lo[k]) q = __dsub_rn(__dmul_rn(2.0, a.lo[k]), q);
                if (q >= a.hi[k]) q = nextafter(a.hi[k], a.lo[k]);
            }
            p[k] = q;
            a.x[k][i] = q;
        }
    }
}

// zero net momentum: the mean of each component summed in index order
// by one thread (the oracle's sequential sum, bit for bit), then subtracted
__global__ void k_init_mean(InitArgs a, double* mean) {
    const int k = threadIdx.x;
    if (k >= 3) return;
    double m = 0.0;
    for (uint32_t i = 0; i < a.n; ++i) m = __dadd_rn(m, a.v[k][i]);
    mean[k] = m / (double)a.n;
}
__global__ void __launch_bounds__(256) k_init_subtract(InitArgs a, const double* mean) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
#pragma unroll
    for (int k = 0; k < 3; ++k) a.v[k][i] = __dsub_rn(a.v[k][i], mean[k]);
}

// ------------------------------------------------ validation observables
// velocity_profile: per-bin sums of the drive-axis velocity and
// particle counts along the profile axis.  Velocities are accumulated as
// 2^-24 fixed point in int64 (shared, then global): integer sums commute, so
// the profile is bitwise reproducible whatever the launch order.
constexpr double PROF_SCALE = 16777216.0;  // 2^24
constexpr int PROF_MAX_BINS = 1024;

__global__ void __launch_bounds__(256) k_profile(const double* __restrict__ xb,
                                                 const double* __restrict__ vd, uint32_t n, double lo,
                                                 double inv_w, uint32_t nbins,
                                                 unsigned long long* acc) {
    __shared__ unsigned long long s_sum[PROF_MAX_BINS];
    __shared__ unsigned int s_cnt[PROF_MAX_BINS];
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) {
        s_sum[b] = 0ull;
        s_cnt[b] = 0u;
    }
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double f = floor((xb[i] - lo) * inv_w);
        const uint32_t b = f < 0.0 ? 0u : (f >= (double)nbins ? nbins - 1u : (uint32_t)f);
        const long long q = __double2ll_rn(vd[i] * PROF_SCALE);
        atomicAdd(&s_sum[b], (unsigned long long)q);  // two's complement: signed sums wrap correctly
        atomicAdd(&s_cnt[b], 1u);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) {
        if (s_cnt[b]) {
            atomicAdd(&acc[b], s_sum[b]);
            atomicAdd(&acc[nbins + b], (unsigned long long)s_cnt[b]);
        }
    }
}

// Pair-distance histogram of the current neighbor table (radial distribution
// numerator): every pair once (the entry with j > i), fp32 distance on the
// pos4 frame with the fp32 minimum image of the builder, bin = floor(r *
// nbins / rmax) in fp32 (r = IEEE sqrt).  layout 0: reference rows (split or
// joined, tiled or not); layout 3: range-walk front entries (bit 31 = skin).
struct RdfArgs {
    const float4* pos4;
    const uint32_t* entries;
    const uint32_t* counts;
    const uint32_t* fwalk;
    uint32_t n, maxn, nbins;
    int layout, tiled, joined;
    int wrap[3];
    float L[3], H[3];
    float bins_per_r;
};

__global__ void __launch_bounds__(256) k_rdf(RdfArgs a, unsigned long long* hist) {
    extern __shared__ unsigned int s_h[];
    for (uint32_t b = threadIdx.x; b < a.nbins; b += blockDim.x) s_h[b] = 0u;
    __syncthreads();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < a.n) {
        const float4 pi = a.pos4[i];
        uint32_t nf, nc = 0;
        if (a.layout == 3) {
            nf = min(a.fwalk[i] & 0x1FFFu, a.maxn);
        } else {
            nc = a.counts[i] & 0x1FFFu;
            nf = min(nc + ((a.counts[i] >> 13) & 0x1FFFu), a.maxn);
        }
        for (uint32_t m = 0; m < nf; ++m) {
            uint32_t k = m;
            if (a.layout == 0 && !a.joined && m >= nc) k = a.maxn - 1u - (m - nc);  // skin from the back
            const size_t off = a.tiled ? (size_t)((i & ~31u) + (k & 31u)) * a.maxn + (k & ~31u) + (i & 31u)
                                       : (size_t)i * a.maxn + k;
            const uint32_t j = a.entries[off] & 0x7FFFFFFFu;
            if (j <= i) continue;
            const float4 pj = a.pos4[j];
            float d[3] = {__fsub_rn(pi.x, pj.x), __fsub_rn(pi.y, pj.y), __fsub_rn(pi.z, pj.z)};
#pragma unroll
            for (int q = 0; q < 3; ++q)
                if (a.wrap[q]) d[q] = min_image_f(d[q], a.L[q], a.H[q]);
            const float r2 = __fadd_rn(__fadd_rn(__fmul_rn(d[0], d[0]), __fmul_rn(d[1], d[1])),
                                       __fmul_rn(d[2], d[2]));
            const float r = __fsqrt_rn(r2);
            const float fb = __fmul_rn(r, a.bins_per_r);
            if (fb < (float)a.nbins) atomicAdd(&s_h[(uint32_t)fb], 1u);
        }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < a.nbins; b += blockDim.x)
        if (s_h[b]) atomicAdd(&hist[b], (unsigned long long)s_h[b]);
}

// ------------------------------------------------ parity primitives
__global__ void k_eval(int op, uint32_t n, const void* in0, const void* in1, uint32_t param,
                       void* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t* u0 = static_cast<const uint32_t*>(in0);
    const uint32_t* u1 = static_cast<const uint32_t*>(in1);
    switch (op) {
        case DPDB_OP_TEA_HASH: {
            uint32_t a = u0[i], b = u1[i];
            tea_rounds((int)param, a, b);
            static_cast<uint32_t*>(out)[2 * i] = a;
            static_cast<uint32_t*>(out)[2 * i + 1] = b;
        } break;
        case DPDB_OP_SIGNATURE: {
            const double* v = static_cast<const double*>(in1);
            static_cast<uint32_t*>(out)[i] = make_signature(u0[i], v[3 * i], v[3 * i + 1], v[3 * i + 2]);
        } break;
        case DPDB_OP_PAIR_UNIFORMS: {
            const uint32_t si = u0[2 * i], sj = u0[2 * i + 1];
            const uint32_t ti = u1[2 * i], tj = u1[2 * i + 1];
            uint32_t a = ti < tj ? si : sj, b = (ti < tj ? sj : si) ^ param;
            tea4(a, b);
            static_cast<uint32_t*>(out)[2 * i] = a;
            static_cast<uint32_t*>(out)[2 * i + 1] = b;
        } break;
        case DPDB_OP_GAUSSIAN64:
            static_cast<double*>(out)[i] = gaussian64(u0[i], u1[i]);
            break;
        case DPDB_OP_GAUSSIAN32:
            static_cast<float*>(out)[i] = gaussian32(u0[i], u1[i]);
            break;
        case DPDB_OP_FASTLOG:
            static_cast<double*>(out)[i] = fastlog64(u0[i]);
            break;
        case DPDB_OP_FASTCOS2PI:
            static_cast<double*>(out)[i] = fastcos2pi64(u0[i]);
            break;
        case DPDB_OP_FASTPOW: {
            const double* d0 = static_cast<const double*>(in0);
            const double* d1 = static_cast<const double*>(in1);
            static_cast<double*>(out)[i] = fastpow64(d0[i], d1[i]);
        } break;
        case DPDB_OP_MORTON: {
            const uint32_t x = u0[3 * i], y = u0[3 * i + 1], z = u0[3 * i + 2];
            uint32_t c = 0;
            for (uint32_t b = 0; b < param; ++b)
                c |= (((x >> b) & 1u) << (3 * b)) | (((y >> b) & 1u) << (3 * b + 1)) |
                     (((z >> b) & 1u) << (3 * b + 2));
            static_cast<uint32_t*>(out)[i] = c;
        } break;
        case DPDB_OP_FASTLOG32:
            static_cast<float*>(out)[i] = fastlog32(u0[i]);
            break;
        case DPDB_OP_GAUSSIAN_HOT:
            static_cast<float*>(out)[i] = gaussian_pair(u0[i], u1[i]);
            break;
        case DPDB_OP_STEP_MIX:
            static_cast<uint32_t*>(out)[i] = step_mix_of(u0[i], u1[i]);
            break;
        default:
            break;
    }
}

}  // namespace dpdb
