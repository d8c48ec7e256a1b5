// force.cuh -- DPD pair-force kernel (conservative + dissipative + random)
// for sm_100a.  Included by kernels.cuh (namespace dpdb).
//
//   compute_forces / dpd_pair_force   SPEC.md:425-442 (impl. not shipped)
//   random term, RNG                  P:234-309, inc/rng.hpp:77-91
#pragma once
#include <type_traits>

struct ForceArgs {
    const int4* posq;   // fixed-point positions | tag word (PosQ, kernels.cuh)
    const float4* vel4;
    const uint32_t* entries;
    const uint32_t* counts;
    const uint32_t* fwalk;  // walk layout only: n_eval | flags << 26
    const uint32_t* plist;  // walk layout: per-tile flat pair list (k_tile_compact)
    const double* xpart;  // fp64 coordinate on the partition axis (body force)
    float* f[3];
    DevErr* err;
    uint32_t n, maxn;
    uint32_t step_mix;
    float rc2, inv_rc;
    float a, gamma, sigma_dt;  // single species: a, gamma, sigma / sqrt(dt)
    float qs[3];        // length per posq quantum, per axis
    // close pairs (r < CLOSE_R): the pair vector again from the fp64 master
    // coordinates (a posq quantum of 4e-8 is still 4e-5 of a 1e-3 separation)
    const double* xd[3];
    double Lw[3], iLw[3];  // wrap lengths (0: no wrap on that axis) and inverses
    float body_g;
    int drive_axis;
    double body_mid64;
    float s_exp;
    int smode;                     // 1, 2, 3: integer weight exponent; 0: fastpow path
    uint32_t ns;                   // species count (MULTI)
    float ta[16], tg[16], ts[16];  // a_ij, gamma_ij, sigma_ij / sqrt(dt)
    // k_force_walk<.., FUSE>: the next Verlet pass (phase 2 of this step +
    // phase 1 of the next) runs in the epilogue on the block's fresh forces;
    // streams go to posqn / vel4n (the other buffer: neighbors still read this
    // step's), keys to ia.keys / ia.vals when the next step rebuilds.
    IntegrateArgs ia;
    int4* posqn;
    float4* vel4n;
    // bricks: run only the blocks with blk_sel[block] == sel_val (interior /
    // boundary split around the ghost update); null = every block
    const uint8_t* blk_sel;
    uint32_t sel_val;
    // k_force_walk<GENERAL>: the bonded terms (harmonic / FENE bonds, harmonic
    // angles) added in the epilogue (else k_bonds runs after the pair kernel)
    int has_bonds;
    BondArgs bd;
};

enum ForceFuse : int { FUSE_NONE = 0, FUSE_STREAMS = 1, FUSE_KEYS = 2 };

// approximate fp32 transcendentals with flush-to-zero (the pair path only;
// the bit-exact builder/integrator paths never use these)
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sin_ftz(float x) {
    float y;
    asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float lg2_ftz(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Box-Muller on the TEA-4 words in fp32 (inc/rng.hpp:88-91: xi = sqrt(-2 ln u_a)
// cos(2 pi u_b), u = word * 2^-32, u_a = 0 -> 1).
//   -2 ln u: u < 1 - 2^-8: MUFU lg2 of u (exact float of the word times
//     2^-32), absolute error ~1e-7 where |ln u| >= 3.9e-3, so rad = sqrt(-2 ln u)
//     is off by <= 1.3e-6; u >= 1 - 2^-8: the series -ln(1 - t) = t + t^2/2 +
//     t^3/3 with t = (2^32 - word) 2^-32 exact (< 2^24 quanta), truncation
//     < t^4/4 -- no cancellation as u -> 1.
//   cos(2 pi u_b) = -/+ sin(pi y), y = (u_b mod 2^31 - 2^30) 2^-31 in
//     [-1/2, 1/2) (the reference's sign-from-top-bit reduction, inc/fastmath.hpp:54-57).
// |xi - xi_ref| < 4e-6 over the whole word range (test_gpu_rng).
__device__ __forceinline__ float gaussian_hot(uint32_t ua, uint32_t ub) {
    ua = max(ua, 1u);
    float m2;  // -2 ln u
    if (__builtin_expect(ua >= 0xFF000000u, 0)) {  // 1 word in 256: the series, a (rarely divergent) branch
        const float t = __uint2float_rn(0u - ua) * 0x1p-32f;               // 1 - u (exact near 1)
        m2 = 2.0f * (t * fmaf(t, fmaf(t, 0.333333333f, 0.5f), 1.0f));     // -ln u near 1
    } else {
        m2 = lg2_ftz(__uint2float_rn(ua) * 0x1p-32f) * -1.386294361f;    // log2 u, u < 1
    }
    const float rad = m2 * rsqrt_ftz(m2);
    const float y = (float)(int)((ub & 0x7FFFFFFFu) - 0x40000000u) * 1.4629180792671596e-9f;  // pi 2^-31
    const float s = sin_ftz(y);
    return (ub >> 31) ? rad * s : -(rad * s);
}

__device__ __forceinline__ float gaussian_pair(uint32_t ua, uint32_t ub) { return gaussian_hot(ua, ub); }

// Pair vector in the posq frame: exact int32 difference (the minimum image on
// wrap axes), one rounding to fp32.
__device__ __forceinline__ void posq_delta(const ForceArgs& a, const int4& p, const int4& q, float& dx,
                                           float& dy, float& dz) {
    dx = (float)(p.x - q.x) * a.qs[0];
    dy = (float)(p.y - q.y) * a.qs[1];
    dz = (float)(p.z - q.z) * a.qs[2];
}

// r^2 below which the pair vector is re-formed from the fp64 master state
// (r < 0.05: the posq quantum, <= 4.2e-8 up to L = 180, is then < 1.2e-6 of r;
// about 1 pair in 8000 takes this branch)
constexpr float CLOSE_R2 = 0.0025f;

// The fp64 pair vector of the oracle (S:434-442 with src/core.cpp:129-139's
// minimum image on wrap axes), rounded once to fp32; rare, so divergent.
__device__ __forceinline__ float close_delta(const ForceArgs& a, uint32_t i, uint32_t j, float& dx, float& dy,
                                             float& dz) {
    double d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        d[k] = __dsub_rn(a.xd[k][i], a.xd[k][j]);
        if (a.Lw[k] > 0.0) d[k] = __dsub_rn(d[k], __dmul_rn(a.Lw[k], rint(__dmul_rn(d[k], a.iLw[k]))));
    }
    dx = (float)d[0];
    dy = (float)d[1];
    dz = (float)d[2];
    return fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}

__device__ __forceinline__ float weight_pow_f(float w, float s, int mode) {
    if (mode == 1) return w;
    if (mode == 2) return w * w;
    if (mode == 3) return w * w * w;
    return w > 0.f ? exp2f(s * __log2f(w)) : 0.f;
}

constexpr int FORCE_WARPS = DPDB_FORCE_WARPS;  // warps per CTA (kernels.cuh)
constexpr int FORCE_TPW = DPDB_FORCE_TPW;       // 32-row tiles per warp (kernels.cuh)
constexpr int FORCE_TILES = FORCE_TPW * FORCE_WARPS;  // 32-row tiles per CTA block
constexpr int FORCE_BLOCK = 32 * FORCE_TILES;   // B particles per block (== RB_BLOCK)
constexpr int FQ = 64;  // per-warp pair queue (slots)
// Forces are accumulated as 2^-18 fixed-point int32 (|F| < 8192 per particle,
// resolution 3.8e-6): integer sums commute, so the result does not depend on
// the order in which lanes or warps deliver their shares.
constexpr float FIX_SCALE = 262144.0f;
constexpr float FIX_INV = 1.0f / 262144.0f;

// The C + D + R force of one pair as fixed-point shares
// q = rint(F * 2^18) of F_ij = mag * r_ij.  Every product and sum is pinned
// (explicit fmaf / __fmul_rn: the compiler may not pick a contraction), so
// all pair kernels -- k_force and k_force_walk, fused or not -- give identical
// bits for the same pair.
template <bool GENERAL>
__device__ __forceinline__ void pair_shares(float dx, float dy, float dz, float r2, const float4& vo,
                                            const float4& vj, float xi, float ca, float cg, float cs,
                                            float inv_rc, float s_exp, int smode, int& qx, int& qy,
                                            int& qz) {
    const float rinv = rsqrt_ftz(r2);
    const float w = fmaxf(fmaf(__fmul_rn(-r2, rinv), inv_rc, 1.f), 0.f);
    const float wr = GENERAL ? weight_pow_f(w, s_exp, smode) : w;
    const float dvx = __fsub_rn(vo.x, vj.x), dvy = __fsub_rn(vo.y, vj.y), dvz = __fsub_rn(vo.z, vj.z);
    const float ev = __fmul_rn(fmaf(dz, dvz, fmaf(dy, dvy, __fmul_rn(dx, dvx))), rinv);
    const float fr = __fmul_rn(__fmul_rn(cs, wr), xi);                       // random
    const float fd = fmaf(-__fmul_rn(cg, __fmul_rn(wr, wr)), ev, fr);        // - dissipative
    const float mag = __fmul_rn(fmaf(ca, w, fd), __fmul_rn(rinv, FIX_SCALE));  // + conservative
    qx = __float2int_rn(__fmul_rn(mag, dx));
    qy = __float2int_rn(__fmul_rn(mag, dy));
    qz = __float2int_rn(__fmul_rn(mag, dz));
}

// Offset of row position m of lane `lane` in its 32-row tile (raw_index,
// inc/neighbor_table.hpp:27-31), relative to entries + i0*maxn + lane.
template <bool TILED, bool JOINED>
__device__ __forceinline__ uint32_t row_offset(uint32_t lane, uint32_t m, uint32_t nc,
                                               uint32_t maxn) {
    const uint32_t k = (JOINED || m < nc) ? m : maxn - 1u - (m - nc);
    return TILED ? (k & 31u) * maxn + (k & ~31u) : lane * (maxn - 1u) + k;
}

// Pair force: warp-level pair compaction + a
// block-local half list + order-free fixed-point accumulation.
//
// A CTA owns a block of FORCE_BLOCK consecutive particles (a compact Morton
// region) and a shared int32 force accumulator for them.  Each warp walks one
// 32-row tile of the table at a time (lane = i & 31).  Phase A, per row
// position m: every lane re-checks its candidate (the per-step |r| <= r_c
// test) and in-range pairs are appended to a per-warp shared-memory queue at
// popc(ballot & lanemask_lt), so the expensive part never runs with idle
// lanes.  A pair whose partner j lies in the same block is taken only by its
// lower index (the pair RNG is symmetric in (i, j), inc/rng.hpp:74-83, so
// F_ji = -F_ij); pairs that cross the block boundary are evaluated from both
// sides, so no global atomics are needed.  Phase B, whenever 32 pairs are
// queued: one pair per lane -- TEA-4 uniforms from the tag-ordered
// signatures, fp32 Box-Muller, C + D + R -- rounded once to fixed point q and
// added as +q to i and -q to j in the block accumulator.  Deterministic run
// to run, and Newton's third law holds exactly.  Row entries and candidate
// positions are software-pipelined (entries 3 ahead, positions 1 ahead).
//
// WALK: the table is in the builder's walk layout (k_build_lane<true>): each
// row lists first the entries this particle evaluates (n_eval = fwalk & 0x1FFF,
// skin entries tagged with bit 31), so the in-block j < i entries are never
// loaded.
//
// GENERAL: any weight exponent s and n_species > 1 (posq.w = tag |
// species << 28, C/D/R coefficients from the ns x ns tables of PairParams,
// inc/core.hpp:51-68).  !GENERAL is the single-species s = 1 fast path.
template <bool GENERAL, bool TILED, bool JOINED, bool BODY, bool WALK>
__global__ void __launch_bounds__(FORCE_WARPS * 32) k_force(ForceArgs a) {
    __shared__ float4 q_d[FORCE_WARPS][FQ];   // (dx, dy, dz, tag_j) in the posq frame
    __shared__ uint32_t q_j[FORCE_WARPS][FQ]; // j | in_block << 26 | owner lane << 27
    __shared__ float4 own_v[FORCE_WARPS][32];
    __shared__ uint32_t own_t[FORCE_WARPS][32];
    __shared__ int acc[FORCE_BLOCK * 3];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t b0 = blockIdx.x * FORCE_BLOCK;
    const uint32_t bn = min((uint32_t)FORCE_BLOCK, a.n - b0);  // particles in this block
    for (int t = threadIdx.x; t < FORCE_BLOCK * 3; t += FORCE_WARPS * 32) acc[t] = 0;
    __syncthreads();
    const uint32_t lt = lanemask_lt();
    const uint32_t maxn = a.maxn;
    bool coincident = false;
    uint32_t bad_tag = 0;

    // static round-robin over the block's tiles (a dynamic hand-out through a
    // shared counter measured 7% slower: it costs registers in the hot loop)
    for (uint32_t tile = warp; tile < FORCE_TILES; tile += FORCE_WARPS) {
        const uint32_t il0 = 32u * tile;
        if (il0 >= bn) break;
        const uint32_t il = il0 + lane;  // my index in the block
        const uint32_t i = b0 + il;
        const bool live = il < bn;
        int4 pi = make_int4(0, 0, 0, 0);
        float4 vi = make_float4(0.f, 0.f, 0.f, 0.f);
        uint32_t c = 0;
        if (live) {
            pi = a.posq[i];
            vi = a.vel4[i];
            c = WALK ? a.fwalk[i] : a.counts[i];
        }
        own_v[warp][lane] = vi;
        const uint32_t nc = WALK ? 0u : c & 0x1FFFu;
        const uint32_t tot = WALK ? (c & 0x1FFFu) : nc + ((c >> 13) & 0x1FFFu);
        const uint32_t maxtot = __reduce_max_sync(0xFFFFFFFFu, tot);
        const uint32_t tag_me = (uint32_t)pi.w;
        own_t[warp][lane] = tag_me;
        uint32_t qhead = 0, qtail = 0;
        __syncwarp();

        auto process = [&](uint32_t h, uint32_t cnt) {
            __syncwarp();
            const uint32_t s = (h + lane) & (FQ - 1);
            if ((uint32_t)lane < cnt) {
                const float4 d4 = q_d[warp][s];
                const uint32_t jj = q_j[warp][s];
                const uint32_t o = jj >> 27, j = jj & 0x03FFFFFFu;
                const float4 vo = own_v[warp][o];
                float dx = d4.x, dy = d4.y, dz = d4.z;
                float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                if (r2 < CLOSE_R2) r2 = close_delta(a, b0 + il0 + o, j, dx, dy, dz);
                if (r2 == 0.f) {
                    coincident = true;
                    bad_tag = own_t[warp][o];
                }
                uint32_t tag_i = own_t[warp][o], tag_j = __float_as_uint(d4.w);
                float ca = a.a, cg = a.gamma, cs = a.sigma_dt;
                if (GENERAL && a.ns > 1) {  // species ride in the top 4 bits of the tag word
                    const uint32_t q = (tag_i >> 28) * a.ns + (tag_j >> 28);
                    ca = a.ta[q];
                    cg = a.tg[q];
                    cs = a.ts[q];
                    tag_i &= 0x0FFFFFFFu;
                    tag_j &= 0x0FFFFFFFu;
                }
                const uint32_t sig_i = __float_as_uint(vo.w);
                const float4 vj = __ldg(a.vel4 + j);
                const uint32_t sig_j = __float_as_uint(vj.w);
                const bool ifirst = tag_i < tag_j;
                uint32_t u0 = ifirst ? sig_i : sig_j;
                uint32_t u1 = (ifirst ? sig_j : sig_i) ^ a.step_mix;
                tea4(u0, u1);
                const float xi = gaussian_pair(u0, u1);
                int qx, qy, qz;
                pair_shares<GENERAL>(dx, dy, dz, r2, vo, vj, xi, ca, cg, cs, a.inv_rc, a.s_exp, a.smode,
                                     qx, qy, qz);
                int* ai = acc + 3 * (il0 + o);
                atomicAdd(ai + 0, qx);
                atomicAdd(ai + 1, qy);
                atomicAdd(ai + 2, qz);
                if (jj & (1u << 26)) {  // partner in this block takes -q
                    int* aj = acc + 3 * (j - b0);
                    atomicAdd(aj + 0, -qx);
                    atomicAdd(aj + 1, -qy);
                    atomicAdd(aj + 2, -qz);
                }
            }
            __syncwarp();
        };

        // software pipeline: entries e0..e2 (positions m, m+1, m+2), position p0 (m)
        const uint32_t* erow = a.entries + (size_t)(b0 + il0) * maxn + lane;
        uint32_t e0 = 0, e1 = 0, e2 = 0;
        constexpr bool JN = JOINED || WALK;
        constexpr uint32_t EMASK = WALK ? 0x7FFFFFFFu : 0xFFFFFFFFu;  // walk: bit 31 = skin
        if (0 < tot) e0 = __ldg(erow + row_offset<TILED, JN>(lane, 0, nc, maxn)) & EMASK;
        if (1 < tot) e1 = __ldg(erow + row_offset<TILED, JN>(lane, 1, nc, maxn)) & EMASK;
        if (2 < tot) e2 = __ldg(erow + row_offset<TILED, JN>(lane, 2, nc, maxn)) & EMASK;
        int4 p0 = make_int4(0, 0, 0, 0);
        if (0 < tot) p0 = __ldg(a.posq + e0);
        for (uint32_t m = 0; m < maxtot; ++m) {
            const uint32_t j = e0;
            const int4 pj = p0;
            const uint32_t jl = j - b0;
            const bool inblk = jl < bn;
            const bool act = m < tot && (WALK || !(inblk && jl < il));  // lower index takes it
            e0 = e1;
            e1 = e2;
            if (m + 3 < tot) e2 = __ldg(erow + row_offset<TILED, JN>(lane, m + 3, nc, maxn)) & EMASK;
            if (m + 1 < tot) p0 = __ldg(a.posq + e0);
            float dx, dy, dz;
            posq_delta(a, pi, pj, dx, dy, dz);
            const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            const bool hit = act && r2 <= a.rc2;
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, hit);
            if (hit) {
                const uint32_t s = (qtail + __popc(bal & lt)) & (FQ - 1);
                q_d[warp][s] = make_float4(dx, dy, dz, __int_as_float(pj.w));
                q_j[warp][s] = j | ((uint32_t)inblk << 26) | ((uint32_t)lane << 27);
            }
            qtail += __popc(bal);
            if (qtail - qhead >= 32u) {
                process(qhead, 32u);
                qhead += 32u;
            }
        }
        if (qtail > qhead) process(qhead, qtail - qhead);
        __syncwarp();
    }
    if (coincident) raise_err(a.err, DPDB_EPHYSICS, EW_COINCIDENT, bad_tag, 0u);
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < bn; t += FORCE_WARPS * 32) {
        const uint32_t i = b0 + t;
        float fx = (float)acc[3 * t + 0] * FIX_INV;
        float fy = (float)acc[3 * t + 1] * FIX_INV;
        float fz = (float)acc[3 * t + 2] * FIX_INV;
        if (BODY) {
            const float g = a.xpart[i] < a.body_mid64 ? a.body_g : -a.body_g;
            if (a.drive_axis == 0)
                fx += g;
            else if (a.drive_axis == 1)
                fy += g;
            else
                fz += g;
        }
        a.f[0][i] = fx;
        a.f[1][i] = fy;
        a.f[2][i] = fz;
    }
}

// Per-tile flat pair list for k_force_walk (built once per neighbor build).
// A walk-layout tile stores each of its 32 rows' front entries (the pairs the
// row evaluates) in the 32x32 tile-transposed layout, so a lane-per-row
// filter runs max(row length) steps with lanes idle past their row's end
// (~45% of the filter's issue slots at C3).  This rewrites tile t's entries
// as one flat list at plist + 32 t maxn: row r's entries (ascending) at the
// exclusive prefix of the earlier rows' lengths, each packed as
// j | r << 26 | skin << 31 -- the pair queue's own format, so the filter
// takes 32 items per step with every lane busy.  One warp per tile; entries
// are read coalesced (one 128-byte line per row position) and staged in
// shared memory so the list is written coalesced too.  Deterministic: no
// atomics, the order is the rows' order.
constexpr int TC_WARPS = 8;
constexpr int TC_STAGE = 1024;  // entries per staging round (a tile holds ~530 at C3)

__global__ void __launch_bounds__(TC_WARPS * 32) k_tile_compact(const uint32_t* __restrict__ entries,
                                                                const uint32_t* __restrict__ fwalk,
                                                                uint32_t n, uint32_t maxn,
                                                                uint32_t* __restrict__ plist) {
    __shared__ uint32_t stage[TC_WARPS][TC_STAGE];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t i0 = (blockIdx.x * TC_WARPS + warp) * 32u;
    if (i0 >= n) return;
    const uint32_t i = i0 + lane;
    const uint32_t tot = i < n ? min(fwalk[i] & 0x1FFFu, maxn) : 0u;
    uint32_t off = tot;  // inclusive scan of the row lengths
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, off, d);
        if (lane >= d) off += y;
    }
    const uint32_t cnt = __shfl_sync(0xFFFFFFFFu, off, 31);
    off -= tot;
    const uint32_t maxtot = __reduce_max_sync(0xFFFFFFFFu, tot);
    const uint32_t* ep = entries + (size_t)i0 * maxn + lane;
    uint32_t* out = plist + (size_t)i0 * maxn;
    const uint32_t rb = (uint32_t)lane << 26;
    for (uint32_t c0 = 0; c0 < cnt; c0 += TC_STAGE) {
        for (uint32_t m = 0; m < maxtot; ++m) {
            const uint32_t e = ep[(m & 31u) * maxn + (m & ~31u)];
            const uint32_t q = off + m - c0;  // wraps (large) below the round
            if (m < tot && q < (uint32_t)TC_STAGE) stage[warp][q] = (e & 0x83FFFFFFu) | rb;
        }
        __syncwarp();
        const uint32_t len = min(cnt - c0, (uint32_t)TC_STAGE);
        for (uint32_t q = lane; q < len; q += 32) out[c0 + q] = stage[warp][q];
        __syncwarp();
    }
}

// Force kernel for the step pipeline's walk layout (the range builder's
// line-grouped flat lists; k_build_lane<true> / k_build<.., true> through
// k_tile_compact): same physics, pair set and fixed-point accumulation as
// k_force, restructured so the per-candidate filter (phase A) is as cheap as
// the hardware allows -- ~18 front candidates are filtered per particle but
// only ~8 pairs evaluated.
//
// Phase A (one flat-list item per lane, 32 items per step, every lane busy):
// the list word and the partner's posq, fp32 distance, |r| <= r_c, a ballot,
// and one 4-byte shared store of the item (j | row << 26 | skin << 31) into
// the warp's pair queue.  Everything else the pair needs (d, tags, in-block
// test) is recomputed in phase B, which runs with all 32 lanes busy.  A group
// is 4 steps: its 4 partner gathers are issued back to back and the next
// group's list words prefetched, so each warp keeps up to 8 loads in flight.
// With the range builder's line-grouped lists the 32 gathers of a step touch a
// few cache lines and a queued batch holds several owner rows.  The queue
// (160 slots) is drained once per group, in whole batches of 32.
//
// Each warp takes tiles (w, FORCE_TILES - 1 - w) of the block: in-block pairs are taken by
// the lower index, so early tiles carry more pairs; pairing them with late
// tiles evens out the work before the block's final barrier.
#ifndef FW_MINB
// resident CTAs per SM the register allocation must allow: 40 warps / SM
// (48 registers, 8 bytes of spill; A/B at 8 warps per CTA with the flat pair
// list: 4 CTAs 0.5079 ms, 5 CTAs 0.4996 ms, 6 CTAs (40 registers) 0.5426 ms)
#define FW_MINB (40 / DPDB_FORCE_WARPS)
#endif
#ifndef DPDB_FW_PREFETCH
#define DPDB_FW_PREFETCH 0
#endif
constexpr bool FW_PREFETCH = DPDB_FW_PREFETCH;  // A/B switch: L1 prefetch of vel4[j] in phase A
// Interleaved drain (A/B knob): the queue is drained FW_IL batches at a time,
// lane l of batch b taking entry l * FW_IL + b.  With row-ordered flat lists a
// plain batch of 32 consecutive pairs has ~8 lanes per owner row and its
// i-side shared atomics serialise on one address (IL 2 was 1% faster there);
// the builder's line-grouped lists already mix the rows of a batch, and IL 1
// is faster (0.442 vs 0.448 ms).
#ifndef DPDB_FW_IL
#define DPDB_FW_IL 1
#endif
constexpr int FW_IL = DPDB_FW_IL;
#ifndef DPDB_FW_G
#define DPDB_FW_G 4
#endif
constexpr int FW_G = DPDB_FW_G;  // phase-A steps (of 32 items) per group: gathers in flight per lane
constexpr int FW_Q = 32 * FW_IL + 32 * FW_G;  // < 32 FW_IL leftovers + FW_G x 32 hits per group

template <bool GENERAL, bool BODY, int MAXN, int FUSE>
__global__ void __launch_bounds__(FORCE_WARPS * 32, GENERAL ? 32 / FORCE_WARPS : FW_MINB)
    k_force_walk(ForceArgs a) {  // GENERAL (species tables, bonded epilogue): 64 registers
    static_assert(FORCE_TPW % 2 == 0, "tiles are dealt in snake order, two per round");
    __shared__ uint32_t q_j[FORCE_WARPS][FW_Q];  // plist items: j | owner row << 26 | skin << 31
    __shared__ int4 own_p[FORCE_WARPS][32];
    __shared__ float4 own_v[FORCE_WARPS][32];
    __shared__ int acc[FORCE_BLOCK * 3];
    // GENERAL: the species-pair coefficients (a, gamma, sigma/sqrt(dt)) in
    // shared memory -- indexed from the kernel parameters, lanes with different
    // species pairs would serialise on the constant cache
    __shared__ float4 coef[GENERAL ? 16 : 1];
    const uint32_t blk = blockIdx.x;
    if (a.blk_sel && a.blk_sel[blk] != a.sel_val) return;  // whole CTA
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t b0 = blk * FORCE_BLOCK;
    const uint32_t bn = min((uint32_t)FORCE_BLOCK, a.n - b0);
    for (int t = threadIdx.x; t < FORCE_BLOCK * 3; t += FORCE_WARPS * 32) acc[t] = 0;
    if (GENERAL && threadIdx.x < 16) coef[threadIdx.x] = make_float4(a.ta[threadIdx.x], a.tg[threadIdx.x], a.ts[threadIdx.x], 0.f);
    __syncthreads();
    const uint32_t lt = lanemask_lt();
    const uint32_t maxn = MAXN ? (uint32_t)MAXN : a.maxn;

#pragma unroll 1
    for (int pass = 0; pass < FORCE_TPW; ++pass) {
        // snake order: warp w takes tiles w, 2W-1-w, 2W+w, 4W-1-w, ...
        const uint32_t tile = (uint32_t)(pass * FORCE_WARPS + ((pass & 1) ? FORCE_WARPS - 1 - warp : warp));
        const uint32_t il0 = 32u * tile;
        if (il0 >= bn) continue;
        const uint32_t il = il0 + lane;
        const bool live = il < bn;
        int4 pi = make_int4(0, 0, 0, 0);
        float4 vi = make_float4(0.f, 0.f, 0.f, 0.f);
        uint32_t c = 0;
        if (live) {
            pi = a.posq[b0 + il];
            vi = a.vel4[b0 + il];
            c = a.fwalk[b0 + il];
        }
        const uint32_t tot = min(c & 0x1FFFu, maxn);
        own_p[warp][lane] = pi;
        own_v[warp][lane] = vi;
        __syncwarp();
        uint32_t qtail = 0;

        auto process = [&](uint32_t e, bool valid) {  // queue entry e on this lane
            if (valid) {
                const uint32_t jw = q_j[warp][e];
                const uint32_t o = (jw >> 26) & 31u, j = jw & 0x03FFFFFFu;
                const int4 po = own_p[warp][o];
                const float4 vo = own_v[warp][o];
                const int4 pj = __ldg(a.posq + j);
                const float4 vj = __ldg(a.vel4 + j);
                float dx, dy, dz;
                posq_delta(a, po, pj, dx, dy, dz);
                float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                if (r2 < CLOSE_R2) {  // rare: the fp64 pair vector (and the coincidence check)
                    r2 = close_delta(a, b0 + il0 + o, j, dx, dy, dz);
                    if (r2 == 0.f)  // raised on the spot: no flag held live through the loop
                        raise_err(a.err, DPDB_EPHYSICS, EW_COINCIDENT,
                                  (uint32_t)po.w & (GENERAL && a.ns > 1 ? 0x0FFFFFFFu : 0xFFFFFFFFu), 0u);
                }
                uint32_t tag_i = (uint32_t)po.w, tag_j = (uint32_t)pj.w;
                float ca = a.a, cg = a.gamma, cs = a.sigma_dt;
                if (GENERAL && a.ns > 1) {  // species ride in the top 4 bits of the tag word
                    const float4 cf = coef[(tag_i >> 28) * a.ns + (tag_j >> 28)];
                    ca = cf.x;
                    cg = cf.y;
                    cs = cf.z;
                    tag_i &= 0x0FFFFFFFu;
                    tag_j &= 0x0FFFFFFFu;
                }
                const uint32_t sig_i = __float_as_uint(vo.w), sig_j = __float_as_uint(vj.w);
                const bool ifirst = tag_i < tag_j;
                uint32_t u0 = ifirst ? sig_i : sig_j;
                uint32_t u1 = (ifirst ? sig_j : sig_i) ^ a.step_mix;
                tea4(u0, u1);
                const float xi = gaussian_pair(u0, u1);
                int qx, qy, qz;
                pair_shares<GENERAL>(dx, dy, dz, r2, vo, vj, xi, ca, cg, cs, a.inv_rc, a.s_exp, a.smode,
                                     qx, qy, qz);
                int* ai = acc + 3 * (il0 + o);
                atomicAdd(ai + 0, qx);
                atomicAdd(ai + 1, qy);
                atomicAdd(ai + 2, qz);
                const uint32_t jl = j - b0;
                if (jl < bn) {  // partner in this block (then j > i): it takes -q
                    int* aj = acc + 3 * jl;
                    atomicAdd(aj + 0, -qx);
                    atomicAdd(aj + 1, -qy);
                    atomicAdd(aj + 2, -qz);
                }
            }
        };

        // Phase A over the tile's flat pair list (k_tile_compact): 32 items per
        // step, every lane busy; a group is 4 steps: the 4 partner positions
        // are gathered back to back, the next group's list words prefetched.
        // Items past the list end load the block's first particle instead (one
        // shared line) and are masked by the bound.
        const uint32_t cnt = __reduce_add_sync(0xFFFFFFFFu, tot);
        const uint32_t* pl = a.plist + (size_t)(b0 + il0) * maxn + lane;
        const char* pb = reinterpret_cast<const char*>(a.posq);
        const char* vb = reinterpret_cast<const char*>(a.vel4);
        uint32_t* qw = q_j[warp];
        const float rc2 = a.rc2;
        auto group = [&](uint32_t c0, const uint32_t (&cur)[FW_G], uint32_t (&nxt)[FW_G]) {
            int4 p[FW_G];
#pragma unroll
            for (int k = 0; k < FW_G; ++k) {
                const uint32_t jk = c0 + 32u * k + lane < cnt ? (cur[k] & 0x03FFFFFFu) : b0;
                p[k] = __ldg(reinterpret_cast<const int4*>(pb + ((size_t)jk << 4)));
            }
#pragma unroll
            for (int k = 0; k < FW_G; ++k) nxt[k] = __ldg(pl + c0 + 32u * FW_G + 32u * k);  // coalesced
#pragma unroll
            for (int k = 0; k < FW_G; ++k) {
                const int4 po = own_p[warp][(cur[k] >> 26) & 31u];
                float dx, dy, dz;
                posq_delta(a, po, p[k], dx, dy, dz);
                const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                const bool hit = c0 + 32u * k + lane < cnt && r2 <= rc2;
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, hit);
                if (hit) qw[qtail + __popc(bal & lt)] = cur[k];
                if (FW_PREFETCH && hit)  // phase B's vel4[j] gather then hits L1
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(vb + ((size_t)(cur[k] & 0x03FFFFFFu) << 4)));
                qtail += __popc(bal);
            }
            // drain FW_IL interleaved batches, then move the (< 32 FW_IL)
            // leftovers to the front
            if (qtail >= 32u * FW_IL) {
                __syncwarp();
                uint32_t h = 0;
                do {
#pragma unroll
                    for (int b = 0; b < FW_IL; ++b) process(h + (uint32_t)lane * FW_IL + b, true);
                    h += 32u * FW_IL;
                } while (qtail - h >= 32u * FW_IL);
                __syncwarp();
                const uint32_t left = qtail - h;
                uint32_t mv[FW_IL];
#pragma unroll
                for (int b = 0; b < FW_IL; ++b) {
                    const uint32_t e = (uint32_t)lane + 32u * b;
                    mv[b] = e < left ? qw[h + e] : 0u;
                }
                __syncwarp();
#pragma unroll
                for (int b = 0; b < FW_IL; ++b) {
                    const uint32_t e = (uint32_t)lane + 32u * b;
                    if (e < left) qw[e] = mv[b];
                }
                __syncwarp();
                qtail = left;
            }
        };
        uint32_t ea[FW_G], eb[FW_G];
#pragma unroll
        for (int k = 0; k < FW_G; ++k) ea[k] = __ldg(pl + 32u * k);
#pragma unroll 1
        for (uint32_t c0 = 0; c0 < cnt; c0 += 64u * FW_G) {
            group(c0, ea, eb);
            if (c0 + 32u * FW_G >= cnt) break;
            group(c0 + 32u * FW_G, eb, ea);
        }
        __syncwarp();
        if (qtail > 0) {  // the rest, interleaved the same way
            const uint32_t nb = (qtail + 31u) >> 5;
            for (uint32_t b = 0; b < nb; ++b) {
                const uint32_t e = (uint32_t)lane * nb + b;
                process(e, e < qtail);
            }
        }
        __syncwarp();
    }
    // FUSE: fetch the block's fp64 x, v and tags for the Verlet epilogue before
    // the barrier, so the loads overlap the wait for the block's last warps
    constexpr int PER_T = FORCE_BLOCK / (FORCE_WARPS * 32);
    double ex[FUSE ? PER_T : 1][6];
    uint32_t etag[FUSE ? PER_T : 1], esp[FUSE ? PER_T : 1];
    // bond forces (independent of the pair sums): evaluated before the barrier
    // too, their dependent tag -> index -> position loads hide behind it
    // (GENERAL instantiations only: the host dispatches bonded systems there)
    float bf[PER_T][3];
    bool bset[PER_T];
#pragma unroll
    for (int q = 0; q < PER_T; ++q) {
        const uint32_t t = threadIdx.x + q * FORCE_WARPS * 32;
        bset[q] = GENERAL && a.has_bonds && t < bn &&
                  bond_force<true>(a.bd, b0 + t, bf[q][0], bf[q][1], bf[q][2]);
    }
    if (FUSE != FUSE_NONE) {
#pragma unroll
        for (int q = 0; q < PER_T; ++q) {
            const uint32_t t = threadIdx.x + q * FORCE_WARPS * 32;
            if (t < bn) {
                const uint32_t i = b0 + t;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    ex[q][k] = a.xd[k][i];  // the epilogue writes x(n+1) to the other buffer (ia.x):
                    ex[q][3 + k] = a.ia.v[k][i];  // other blocks' close pairs still read x(n)
                }
                etag[q] = a.ia.tag[i];
                esp[q] = a.ia.sp ? a.ia.sp[i] : 0u;
            }
        }
    }
    __syncthreads();
    double th[4] = {0.0, 0.0, 0.0, 0.0};  // FUSE: this thread's thermo partial
#pragma unroll
    for (int q = 0; q < PER_T; ++q) {
        const uint32_t t = threadIdx.x + q * FORCE_WARPS * 32;
        if (t >= bn) break;
        const uint32_t i = b0 + t;
        float fx = (float)acc[3 * t + 0] * FIX_INV;
        float fy = (float)acc[3 * t + 1] * FIX_INV;
        float fz = (float)acc[3 * t + 2] * FIX_INV;
        if (BODY) {
            const float g = a.xpart[i] < a.body_mid64 ? a.body_g : -a.body_g;
            if (a.drive_axis == 0)
                fx += g;
            else if (a.drive_axis == 1)
                fy += g;
            else
                fz += g;
        }
        if (GENERAL && bset[q]) {  // same fp32 adds as k_bonds after the pair kernel
            fx += bf[q][0];
            fy += bf[q][1];
            fz += bf[q][2];
        }
        if (FUSE == FUSE_NONE) {
            a.f[0][i] = fx;
            a.f[1][i] = fy;
            a.f[2][i] = fz;
        } else {
            const float f[3] = {fx, fy, fz};
            const int qq = FUSE ? q : 0;
            const double x[3] = {ex[qq][0], ex[qq][1], ex[qq][2]};
            const double v[3] = {ex[qq][3], ex[qq][4], ex[qq][5]};
            double vf[3];
            integrate_particle<true, true, FUSE == FUSE_KEYS, FUSE == FUSE_STREAMS>(
                a.ia, i, f, x, v, etag[qq], esp[qq], nullptr, a.posqn, a.vel4n, vf);
            th[0] += vf[0];
            th[1] += vf[1];
            th[2] += vf[2];
            th[3] += vf[0] * vf[0] + vf[1] * vf[1] + vf[2] * vf[2];
        }
    }
    if (FUSE != FUSE_NONE && a.ia.thermo_part)  // uniform per launch
        block_sum4<FORCE_WARPS * 32>(th, a.ia.thermo_part + 4 * blk);
}
