/*
 * dpd_oracle.c -- CPU restatement of the reference DPD hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see dpd_oracle.h).  Compiled with
 * -O2 -ffp-contract=off -fopenmp.  Never linked into the product library.
 */
#include "dpd_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static _Thread_local char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int set_err(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

static inline uint64_t dbits(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
}
static inline double bitsd(uint64_t u) {
    double d;
    memcpy(&d, &u, 8);
    return d;
}

/* ======================================================================
 * fastmath -- restates inc/fastmath.hpp:26-151 (frozen minimax tables of
 * inc/fastmath.hpp:35-57 are data and must be bit-identical).
 * ==================================================================== */
#define FM_SQRT2 1.4142135623730951
static const double fm_ln2_hi = 0x1.62e42fef00000p-1;
static const double fm_ln2_lo = 0x1.473de6af278edp-34;
static const double fm_2_over_ln2 = 0x1.71547652b82fep+1;
static const double fm_2_over_ln2_res = 0x1.777d0ffda0d24p-55;

static const double fm_lnq[6] = {
    0x1.555555555397ap-1, 0x1.999999a28e942p-2, 0x1.2492417a9975ap-2,
    0x1.c72276984c243p-3, 0x1.732c520e537b1p-3, 0x1.587592fb5a518p-3,
};
static const double fm_log2q[7] = {
    0x1.ec709dc3a0455p-1, 0x1.2776c50ee73bep-1, 0x1.a61762d1f5b51p-2, 0x1.484afcfb984e8p-2,
    0x1.0ca11d4fbc32dp-2, 0x1.c479f5cc9ee5ep-3, 0x1.b52725f185dd3p-3,
};
static const double fm_exp2r[11] = {
    0x1.62e42fefa39f5p-1,  0x1.ebfbdff82c04bp-3,  0x1.c6b08d7065838p-5, 0x1.3b2ab6f73416fp-7,
    0x1.5d87ff4d2262ap-10, 0x1.4308fa1dd16ddp-13, 0x1.ffcfc6a9b62c8p-17, 0x1.628f3583fa66bp-20,
    0x1.b85f42cc9ad9ap-24, 0x1.c2c47913b09f9p-28, 0x1.58566e8b85bdfp-31,
};
static const double fm_sinp[6] = {
    0x1.921fb5441e49dp+1,  -0x1.4abbce4f1a2d1p+2, 0x1.466bbfc24f863p+1,
    -0x1.32d11201b18c4p-1, 0x1.500ff7f212ce7p-4,  -0x1.cc345a6170d5cp-8,
};

/* inc/fastmath.hpp:59-64: Horner with explicit fma, highest degree first */
static double poly_eval(const double* c, int n, double x) {
    double acc = c[n - 1];
    for (int k = n - 2; k >= 0; --k) acc = fma(acc, x, c[k]);
    return acc;
}

/* inc/fastmath.hpp:71-86: log2 of x in [1,2) as hi+lo */
static void log2_frac_pair(double x, double* hi, double* lo) {
    const int big = x >= FM_SQRT2;
    const double xr = big ? 0.5 * x : x;
    const double z = (xr - 1.0) / (xr + 1.0);
    const double w = z * z;
    const double tail = w * poly_eval(fm_log2q, 7, w);
    const double s_hi = fm_2_over_ln2 + tail;
    const double s_lo = ((fm_2_over_ln2 - s_hi) + tail) + fm_2_over_ln2_res;
    const double p_hi = z * s_hi;
    const double p_lo = fma(z, s_hi, -p_hi) + z * s_lo;
    const double k = big ? 1.0 : 0.0;
    const double r_hi = k + p_hi;
    *lo = ((k - r_hi) + p_hi) + p_lo;
    *hi = r_hi;
}

/* inc/fastmath.hpp:92-94 */
double orc_power2(int n) { return bitsd((uint64_t)(1023 + n) << 52); }
/* inc/fastmath.hpp:97-99 */
double orc_exp2_frac(double x) { return fma(x, poly_eval(fm_exp2r, 11, x), 1.0); }
/* inc/fastmath.hpp:102-105 */
double orc_log2_frac(double x) {
    double h, l;
    log2_frac_pair(x, &h, &l);
    return h + l;
}

/* inc/fastmath.hpp:108-118 */
double orc_fastlog(uint32_t v) {
    const int e = 31 - __builtin_clz(v);
    const double m = (double)v * orc_power2(-e);
    const int big = m >= FM_SQRT2;
    const double x = big ? 0.5 * m : m;
    const double di = (double)(e + big - 32);
    const double z = (x - 1.0) / (x + 1.0);
    const double w = z * z;
    const double lnx = fma(z * w, poly_eval(fm_lnq, 6, w), 2.0 * z);
    return fma(di, fm_ln2_hi, fma(di, fm_ln2_lo, lnx));
}

/* inc/fastmath.hpp:122-130 */
double orc_fastcos2pi(uint32_t v) {
    const uint32_t top = v >> 31;
    const double u = (double)(v & 0x7FFFFFFFu) * 0x1p-31;
    const double y = u - 0.5;
    const double s = y * poly_eval(fm_sinp, 6, y * y);
    return bitsd(dbits(s) ^ ((uint64_t)(top ^ 1u) << 63));
}

/* inc/fastmath.hpp:135-151 */
double orc_fastpow(double a, double b) {
    const uint64_t ab = dbits(a);
    const int ie = (int)(ab >> 52) - 1023;
    const double m = bitsd((ab & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull);
    double lhi, llo;
    log2_frac_pair(m, &lhi, &llo);
    const double di = (double)ie;
    const double y = b * (di + lhi);
    double ii = floor(y);
    if (ii > 1024.0) ii = 1024.0;
    if (ii < -1022.0) ii = -1022.0;
    double frac = fma(b, lhi, fma(b, di, -ii));
    frac = fma(b, llo, frac);
    return orc_power2((int)ii) * orc_exp2_frac(frac);
}

/* ======================================================================
 * rng -- restates inc/rng.hpp:16-107
 * ==================================================================== */
static const uint32_t tea_delta = 0x9E3779B9u;
static const uint32_t tea_k0 = 0xA341316Cu, tea_k1 = 0xC8013EA4u, tea_k2 = 0xAD90777Du,
                      tea_k3 = 0x7E95761Eu;

/* inc/rng.hpp:25-33 */
void orc_tea_hash(int rounds, uint32_t v0, uint32_t v1, uint32_t out[2]) {
    uint32_t acc = 0;
    for (int r = 0; r < rounds; ++r) {
        acc += tea_delta;
        v0 += ((v1 << 4) + tea_k0) ^ ((v1 >> 5) + tea_k1) ^ (v1 + acc);
        v1 += ((v0 << 4) + tea_k2) ^ ((v0 >> 5) + tea_k3) ^ (v0 + acc);
    }
    out[0] = v0;
    out[1] = v1;
}

/* inc/rng.hpp:35-40 (bit reversal; any correct reversal is equivalent) */
uint32_t orc_bit_reverse(uint32_t x) {
    uint32_t r = 0;
    for (int b = 0; b < 32; ++b) r |= ((x >> b) & 1u) << (31 - b);
    return r;
}

/* inc/rng.hpp:43-45: leading 11 fraction bits of a double */
uint32_t orc_mantissa11(double v) { return (uint32_t)(dbits(v) >> 41) & 0x7FFu; }

/* inc/rng.hpp:49-62 */
uint32_t orc_make_signature(uint32_t tag, double vx, double vy, double vz) {
    const uint32_t m[3] = {orc_mantissa11(vx), orc_mantissa11(vy), orc_mantissa11(vz)};
    uint32_t word = 0;
    for (int bit = 0; bit < 32; ++bit) /* bit 3k+a <- bit k of component a */
        word |= ((m[bit % 3] >> (bit / 3)) & 1u) << bit;
    uint32_t h[2];
    orc_tea_hash(16, orc_bit_reverse(tag), word, h);
    return h[0] ^ h[1];
}

/* inc/rng.hpp:70-72 */
uint32_t orc_step_mix(uint32_t seed, uint32_t step) {
    uint32_t h[2];
    orc_tea_hash(4, seed, step, h);
    return h[1];
}

/* inc/rng.hpp:77-83 */
void orc_pair_uniforms(uint32_t sig_i, uint32_t sig_j, uint32_t tag_i, uint32_t tag_j,
                       uint32_t step_mix, uint32_t out[2]) {
    const int i_first = tag_i < tag_j;
    orc_tea_hash(4, i_first ? sig_i : sig_j, (i_first ? sig_j : sig_i) ^ step_mix, out);
}

/* inc/rng.hpp:88-91 */
double orc_gaussian(uint32_t ua, uint32_t ub) {
    if (ua == 0) ua = 1;
    return sqrt(-2.0 * orc_fastlog(ua)) * orc_fastcos2pi(ub);
}

void orc_signatures(size_t n, const uint32_t* tag, const double* vx, const double* vy,
                    const double* vz, uint32_t* sig) {
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; ++i) sig[i] = orc_make_signature(tag[i], vx[i], vy[i], vz[i]);
}

/* ======================================================================
 * morton -- restates inc/morton.hpp:32-40 (x least significant)
 * ==================================================================== */
static uint32_t interleave3(uint32_t ix, uint32_t iy, uint32_t iz, int bits) {
    uint32_t code = 0;
    for (int b = 0; b < bits && 3 * b < 32; ++b) {
        code |= ((ix >> b) & 1u) << (3 * b);
        if (3 * b + 1 < 32) code |= ((iy >> b) & 1u) << (3 * b + 1);
        if (3 * b + 2 < 32) code |= ((iz >> b) & 1u) << (3 * b + 2);
    }
    return code;
}

int orc_morton_encode(uint32_t ix, uint32_t iy, uint32_t iz, int bits, uint32_t* code) {
    if (bits < 0 || 3 * bits > 32)
        return set_err(ORC_ECONFIG, "morton: 3*bits_per_axis must be <= 32");
    const uint32_t lim = bits >= 32 ? 0xFFFFFFFFu : (1u << bits) - 1u;
    if (ix > lim || iy > lim || iz > lim)
        return set_err(ORC_ECONFIG, "morton: lattice coordinate out of range");
    *code = interleave3(ix, iy, iz, bits);
    return ORC_OK;
}

/* ======================================================================
 * radix sort -- restates the contract of inc/radix_sort.hpp:11-27 and the
 * 4-bit LSD passes of src/radix_sort.cpp:35-68 (chunked histogram,
 * digit-major scan, stable scatter).  Output is independent of nthreads.
 * ==================================================================== */
int orc_radix_sort(uint32_t* keys, uint32_t* vals, size_t n, int bit_length, int nthreads) {
    if (bit_length < 0 || bit_length > 32 || bit_length % 4)
        return set_err(ORC_ECONFIG, "radix sort: bit length must be a multiple of 4, <= 32");
    if (n == 0 || bit_length == 0) return ORC_OK;
    if (nthreads < 1) nthreads = 1;
    if ((size_t)nthreads > n) nthreads = (int)n;
    uint32_t* kb = (uint32_t*)malloc(n * 4);
    uint32_t* vb = (uint32_t*)malloc(n * 4);
    size_t* cnt = (size_t*)calloc((size_t)nthreads * 16, sizeof(size_t));
    uint32_t *ks = keys, *vs = vals, *kd = kb, *vd = vb;
    for (int shift = 0; shift < bit_length; shift += 4) {
#pragma omp parallel num_threads(nthreads)
        {
#ifdef _OPENMP
            const int t = omp_get_thread_num();
            const int nt = omp_get_num_threads();
#else
            const int t = 0, nt = 1;
#endif
            const size_t b = n * (size_t)t / (size_t)nt;
            const size_t e = n * (size_t)(t + 1) / (size_t)nt;
            size_t local[16] = {0};
            for (size_t i = b; i < e; ++i) local[(ks[i] >> shift) & 15u]++;
            for (int d = 0; d < 16; ++d) cnt[(size_t)t * 16 + d] = local[d];
#pragma omp barrier
#pragma omp single
            {
                size_t run = 0;
                for (int d = 0; d < 16; ++d)
                    for (int c = 0; c < nt; ++c) {
                        const size_t x = cnt[(size_t)c * 16 + d];
                        cnt[(size_t)c * 16 + d] = run;
                        run += x;
                    }
            }
            size_t pos[16];
            for (int d = 0; d < 16; ++d) pos[d] = cnt[(size_t)t * 16 + d];
            for (size_t i = b; i < e; ++i) {
                const size_t p = pos[(ks[i] >> shift) & 15u]++;
                kd[p] = ks[i];
                vd[p] = vs[i];
            }
        }
        uint32_t* tk = ks; ks = kd; kd = tk;
        uint32_t* tv = vs; vs = vd; vd = tv;
    }
    if (ks != keys) {
        memcpy(keys, ks, n * 4);
        memcpy(vals, vs, n * 4);
    }
    free(kb);
    free(vb);
    free(cnt);
    return ORC_OK;
}

/* ======================================================================
 * cell grid -- restates src/cell_grid.cpp:16-134, inc/cell_grid.hpp:21-70
 * ==================================================================== */
static int ceil_log2u(uint32_t v) { return v <= 1 ? 0 : 32 - __builtin_clz(v - 1); }

typedef struct {
    uint32_t code, idx;
} code_idx;

static int cmp_code(const void* a, const void* b) {
    const code_idx* x = (const code_idx*)a;
    const code_idx* y = (const code_idx*)b;
    if (x->code != y->code) return x->code < y->code ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static void ext_coords(const orc_grid* g, size_t idx, int32_t c[3]) {
    c[0] = (int32_t)(idx % (size_t)g->ncell_ext[0]);
    idx /= (size_t)g->ncell_ext[0];
    c[1] = (int32_t)(idx % (size_t)g->ncell_ext[1]);
    c[2] = (int32_t)(idx / (size_t)g->ncell_ext[1]);
}
static size_t ext_index(const orc_grid* g, const int32_t c[3]) {
    return ((size_t)c[2] * (size_t)g->ncell_ext[1] + (size_t)c[1]) * (size_t)g->ncell_ext[0] +
           (size_t)c[0];
}
static int is_local(const orc_grid* g, const int32_t c[3]) {
    for (int k = 0; k < 3; ++k)
        if (c[k] < g->ghost_lo[k] || c[k] >= g->ghost_lo[k] + g->ncell[k]) return 0;
    return 1;
}

/* src/cell_grid.cpp:16-59 (assign_ranks): locals by local-lattice Morton,
 * then ghosts by ext-lattice Morton */
static int rank_cells(orc_grid* g) {
    const size_t total = (size_t)g->ncell_ext[0] * g->ncell_ext[1] * g->ncell_ext[2];
    g->n_total_cells = (uint32_t)total;
    g->n_local_cells = (uint32_t)g->ncell[0] * g->ncell[1] * g->ncell[2];
    int bits = 1;
    for (int k = 0; k < 3; ++k) {
        const int b = ceil_log2u((uint32_t)g->ncell_ext[k]);
        if (b > bits) bits = b;
    }
    g->bits_per_axis = bits;
    if (3 * bits > 32) return set_err(ORC_ECONFIG, "cell grid: too many cells per axis");
    code_idx* loc = (code_idx*)malloc(sizeof(code_idx) * (g->n_local_cells + 1));
    code_idx* gh = (code_idx*)malloc(sizeof(code_idx) * (total - g->n_local_cells + 1));
    size_t nl = 0, ng = 0;
    for (size_t idx = 0; idx < total; ++idx) {
        int32_t c[3];
        ext_coords(g, idx, c);
        if (is_local(g, c)) {
            loc[nl].code = interleave3((uint32_t)(c[0] - g->ghost_lo[0]),
                                       (uint32_t)(c[1] - g->ghost_lo[1]),
                                       (uint32_t)(c[2] - g->ghost_lo[2]), bits);
            loc[nl++].idx = (uint32_t)idx;
        } else {
            gh[ng].code = interleave3((uint32_t)c[0], (uint32_t)c[1], (uint32_t)c[2], bits);
            gh[ng++].idx = (uint32_t)idx;
        }
    }
    qsort(loc, nl, sizeof(code_idx), cmp_code);
    qsort(gh, ng, sizeof(code_idx), cmp_code);
    g->rank_of_cell = (uint32_t*)calloc(total, 4);
    g->cell_of_rank = (uint32_t*)calloc(total, 4);
    uint32_t r = 0;
    for (size_t a = 0; a < nl; ++a, ++r) {
        g->rank_of_cell[loc[a].idx] = r;
        g->cell_of_rank[r] = loc[a].idx;
    }
    for (size_t a = 0; a < ng; ++a, ++r) {
        g->rank_of_cell[gh[a].idx] = r;
        g->cell_of_rank[r] = gh[a].idx;
    }
    free(loc);
    free(gh);
    return ORC_OK;
}

/* src/cell_grid.cpp:67-95 */
int orc_grid_make(const orc_box* box, const double slab_lo[3], const double slab_hi[3],
                  const int32_t dims[3], const int32_t coords[3], double cell_target,
                  int32_t sub_bits, orc_grid* g) {
    memset(g, 0, sizeof *g);
    if (cell_target <= 0) return set_err(ORC_ECONFIG, "cell grid: cell target must be positive");
    g->sub_bits = sub_bits;
    for (int k = 0; k < 3; ++k) {
        g->slab_lo[k] = slab_lo[k];
        g->slab_hi[k] = slab_hi[k];
        const double len = slab_hi[k] - slab_lo[k];
        if (len < cell_target)
            return set_err(ORC_ECONFIG, "cell grid: slab thinner than cutoff+skin on axis %d", k);
        int nc = (int)floor(len / cell_target);
        if (nc < 1) nc = 1;
        g->ncell[k] = nc;
        g->cell_size[k] = len / nc;
        g->inv_cell[k] = nc / len;
        g->wrapmode[k] = dims[k] == 1 && box->periodic[k];
        const int lower = dims[k] > 1 && (coords[k] > 0 || box->periodic[k]);
        const int upper = dims[k] > 1 && (coords[k] < dims[k] - 1 || box->periodic[k]);
        g->ghost_lo[k] = lower;
        g->ghost_hi[k] = upper;
        g->ncell_ext[k] = nc + lower + upper;
        g->origin[k] = slab_lo[k] - g->ghost_lo[k] * g->cell_size[k];
    }
    return rank_cells(g);
}

void orc_grid_free(orc_grid* g) {
    free(g->rank_of_cell);
    free(g->cell_of_rank);
    g->rank_of_cell = g->cell_of_rank = NULL;
}

/* src/cell_grid.cpp:130-134 */
int orc_grid_key_bits(const orc_grid* g) {
    const int bits = ceil_log2u(g->n_total_cells) + 3 * g->sub_bits;
    if (bits > 32) return -set_err(ORC_ECONFIG, "cell grid: sort key exceeds 32 bits");
    return (bits + 3) & ~3;
}

/* src/cell_grid.cpp:97-108 */
int orc_local_cell_of(const orc_grid* g, const double x[3], int32_t c[3]) {
    for (int k = 0; k < 3; ++k) {
        if (!(x[k] >= g->slab_lo[k] && x[k] < g->slab_hi[k]))
            return set_err(ORC_EPROTOCOL,
                           "particle outside its domain slab (missed migration), axis %d", k);
        int ci = (int)floor((x[k] - g->slab_lo[k]) * g->inv_cell[k]);
        if (ci < 0) ci = 0;
        if (ci > g->ncell[k] - 1) ci = g->ncell[k] - 1;
        c[k] = ci + g->ghost_lo[k];
    }
    return ORC_OK;
}

/* src/cell_grid.cpp:119-128 */
uint32_t orc_sub_code(const orc_grid* g, const double x[3], const int32_t c[3]) {
    const int nsub = 1 << g->sub_bits;
    uint32_t s[3];
    for (int k = 0; k < 3; ++k) {
        const double cell_lo = g->origin[k] + c[k] * g->cell_size[k];
        int si = (int)floor((x[k] - cell_lo) * g->inv_cell[k] * nsub);
        if (si < 0) si = 0;
        if (si > nsub - 1) si = nsub - 1;
        s[k] = (uint32_t)si;
    }
    return interleave3(s[0], s[1], s[2], g->sub_bits);
}

/* src/cell_grid.cpp:168-175 (key generation of reorder_particles) */
int orc_sort_keys(const orc_grid* g, size_t n, const double* x, const double* y,
                  const double* z, uint32_t* keys) {
    int err = ORC_OK;
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; ++i) {
        const double p[3] = {x[i], y[i], z[i]};
        int32_t c[3];
        if (orc_local_cell_of(g, p, c) != ORC_OK) {
#pragma omp atomic write
            err = ORC_EPROTOCOL;
            keys[i] = 0;
            continue;
        }
        const uint32_t rank = g->rank_of_cell[ext_index(g, c)];
        keys[i] = (rank << (3 * g->sub_bits)) | orc_sub_code(g, p, c);
    }
    if (err) return set_err(err, "particle outside its domain slab (missed migration)");
    return ORC_OK;
}

/* src/cell_grid.cpp:166-198: keys -> stable radix sort -> order/perm */
int orc_reorder_order(const orc_grid* g, size_t n, const double* x, const double* y,
                      const double* z, uint32_t* order, uint32_t* perm, int nthreads) {
    uint32_t* keys = (uint32_t*)malloc((n + 1) * 4);
    int rc = orc_sort_keys(g, n, x, y, z, keys);
    if (rc == ORC_OK) {
        for (size_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
        const int kb = orc_grid_key_bits(g);
        rc = kb < 0 ? -kb : orc_radix_sort(keys, order, n, kb, nthreads);
    }
    if (rc == ORC_OK && perm)
        for (size_t to = 0; to < n; ++to) perm[order[to]] = (uint32_t)to;
    free(keys);
    return rc;
}

/* src/cell_grid.cpp:157-164 */
int orc_local_cell_ranks(const orc_grid* g, size_t n, const double* x, const double* y,
                         const double* z, uint32_t* ranks) {
    for (size_t i = 0; i < n; ++i) {
        const double p[3] = {x[i], y[i], z[i]};
        int32_t c[3];
        const int rc = orc_local_cell_of(g, p, c);
        if (rc) return rc;
        ranks[i] = g->rank_of_cell[ext_index(g, c)];
    }
    return ORC_OK;
}

/* src/cell_grid.cpp:136-155: cell_start[r] = first index with rank >= r */
int orc_build_cell_list(uint32_t n_total_cells, const uint32_t* ranks, size_t n,
                        uint32_t* cell_start) {
    uint32_t next = 0; /* first cell whose start is not yet written */
    for (size_t i = 0; i < n; ++i) {
        if (i > 0 && ranks[i] < ranks[i - 1])
            return set_err(ORC_EPROTOCOL, "cell list: particle array not sorted by cell rank");
        while (next <= ranks[i] && next < n_total_cells) cell_start[next++] = (uint32_t)i;
    }
    while (next <= n_total_cells) cell_start[next++] = (uint32_t)n;
    return ORC_OK;
}

/* src/stencil.cpp:7-41: <=27 wrapped neighbor ranks, ascending, unique */
static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y);
}

int orc_coarse_stencil(const orc_grid* g, uint32_t* offsets, uint32_t* cells) {
    offsets[0] = 0;
    for (uint32_t r = 0; r < g->n_local_cells; ++r) {
        int32_t c[3];
        ext_coords(g, g->cell_of_rank[r], c);
        uint32_t list[27];
        int m = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int off[3] = {dx, dy, dz};
                    int32_t nc[3];
                    int ok = 1;
                    for (int k = 0; k < 3 && ok; ++k) {
                        int v = c[k] + off[k];
                        if (g->wrapmode[k])
                            v = (v + g->ncell[k]) % g->ncell[k];
                        else if (v < 0 || v >= g->ncell_ext[k])
                            ok = 0;
                        nc[k] = v;
                    }
                    if (ok) list[m++] = g->rank_of_cell[ext_index(g, nc)];
                }
        qsort(list, (size_t)m, 4, cmp_u32);
        int u = 0;
        for (int a = 0; a < m; ++a)
            if (u == 0 || list[a] != list[u - 1]) list[u++] = list[a];
        memcpy(cells + offsets[r], list, (size_t)u * 4);
        offsets[r + 1] = offsets[r] + (uint32_t)u;
    }
    return ORC_OK;
}

/* src/stencil.cpp:43-62.  fidx may be NULL to query sizes only. */
int orc_fine_stencil(uint32_t n_local_cells, const uint32_t* coff, const uint32_t* ccells,
                     const uint32_t* cell_start, uint32_t* foff, uint32_t* fidx) {
    foff[0] = 0;
    for (uint32_t r = 0; r < n_local_cells; ++r) {
        uint32_t cnt = 0;
        for (uint32_t a = coff[r]; a < coff[r + 1]; ++a)
            cnt += cell_start[ccells[a] + 1] - cell_start[ccells[a]];
        foff[r + 1] = foff[r] + cnt;
    }
    if (!fidx) return ORC_OK;
#pragma omp parallel for schedule(static)
    for (uint32_t r = 0; r < n_local_cells; ++r) {
        uint32_t w = foff[r];
        for (uint32_t a = coff[r]; a < coff[r + 1]; ++a)
            for (uint32_t j = cell_start[ccells[a]]; j < cell_start[ccells[a] + 1]; ++j)
                fidx[w++] = j;
    }
    return ORC_OK;
}

/* ======================================================================
 * neighbor table -- restatement of the missing src/neighbor_table.cpp from
 * its contract inc/neighbor_table.hpp:12-59, S:209-235 and Alg. 3.
 * PARITY UNPINNED (no reference implementation shipped).  Frozen choices:
 *   - fp32 coordinates: (float)(x - slab_centre), slab_centre = (lo+hi)/2
 *   - r_ij = xf_i - xf_j per axis in fp32; on wrapmode axes the fp32
 *     minimum image of src/core.cpp:129-139 (>= +L/2 -> -L, < -L/2 -> +L)
 *     with L and L/2 rounded to fp32
 *   - d2 = (dx*dx + dy*dy) + dz*dz, every op rounded to fp32 (no fma)
 *   - core: d2 <= (float)(r_c*r_c); skin: (float)(r_c^2) < d2 <= (float)((r_c+skin)^2)
 *   - j == i skipped explicitly; candidates in fine-stencil order
 *   - overflow (core+skin > maxn): physics error naming the tag
 * ==================================================================== */
size_t orc_raw_index(int tiled, uint32_t maxn, uint32_t i, uint32_t k) {
    if (!tiled) return (size_t)i * maxn + k;
    return (size_t)((i & ~31u) + (k & 31u)) * maxn + (k & ~31u) + (i & 31u);
}

int orc_build_neighbor_table(const orc_grid* g, const orc_box* box, const uint32_t* cell_start,
                             const uint32_t* coff, const uint32_t* ccells, size_t n_local,
                             size_t n_all, const double* x, const double* y, const double* z,
                             const uint32_t* tag, double r_c, double skin, uint32_t maxn,
                             uint32_t* entries, uint16_t* core, uint16_t* skinc, int nthreads) {
    (void)box;
    if (maxn == 0 || maxn % 32)
        return set_err(ORC_ECONFIG, "neighbor table: max_neighbors must be a positive multiple of 32");
    double ctr[3];
    float wrapL[3], wrapH[3];
    for (int k = 0; k < 3; ++k) {
        ctr[k] = (g->slab_lo[k] + g->slab_hi[k]) / 2;
        wrapL[k] = (float)(g->slab_hi[k] - g->slab_lo[k]);
        wrapH[k] = (float)(0.5 * (g->slab_hi[k] - g->slab_lo[k]));
    }
    const float cut_c = (float)(r_c * r_c);
    const float cut_s = (float)((r_c + skin) * (r_c + skin));
    float* xf = (float*)malloc(sizeof(float) * 3 * (n_all + 1));
    for (size_t j = 0; j < n_all; ++j) {
        xf[3 * j + 0] = (float)(x[j] - ctr[0]);
        xf[3 * j + 1] = (float)(y[j] - ctr[1]);
        xf[3 * j + 2] = (float)(z[j] - ctr[2]);
    }
    int err = ORC_OK;
    uint32_t err_tag = 0;
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
    for (uint32_t r = 0; r < g->n_local_cells; ++r) {
        for (uint32_t i = cell_start[r]; i < cell_start[r + 1] && i < n_local; ++i) {
            uint32_t nc = 0, ns = 0;
            for (uint32_t a = coff[r]; a < coff[r + 1]; ++a) {
                const uint32_t cc = ccells[a];
                for (uint32_t j = cell_start[cc]; j < cell_start[cc + 1]; ++j) {
                    if (j == i) continue;
                    float d[3];
                    for (int k = 0; k < 3; ++k) {
                        float t = xf[3 * i + k] - xf[3 * j + k];
                        if (g->wrapmode[k]) {
                            if (t >= wrapH[k])
                                t = t - wrapL[k];
                            else if (t < -wrapH[k])
                                t = t + wrapL[k];
                        }
                        d[k] = t;
                    }
                    const float xx = d[0] * d[0];
                    const float yy = d[1] * d[1];
                    const float zz = d[2] * d[2];
                    const float d2 = (xx + yy) + zz;
                    if (d2 <= cut_c) {
                        if (nc + ns < maxn) entries[(size_t)i * maxn + nc] = j;
                        ++nc;
                    } else if (d2 <= cut_s) {
                        if (nc + ns < maxn) entries[(size_t)i * maxn + (maxn - 1 - ns)] = j;
                        ++ns;
                    }
                }
            }
            if (nc + ns > maxn) {
#pragma omp critical
                {
                    if (!err) {
                        err = ORC_EPHYSICS;
                        err_tag = tag ? tag[i] : i;
                    }
                }
                nc = ns = 0;
            }
            core[i] = (uint16_t)nc;
            skinc[i] = (uint16_t)ns;
        }
    }
    free(xf);
    if (err)
        return set_err(err, "neighbor table: row overflow (max_neighbors=%u) for particle tag %u",
                       maxn, err_tag);
    return ORC_OK;
}

/* test helper (not a reference function): the core_at / skin_at accessors of
 * inc/neighbor_table.hpp:33-39 applied to two tables in any layouts */
static inline uint32_t tbl_skin_at(int tiled, int joined, uint32_t maxn, const uint32_t* e,
                                   uint32_t nc, uint32_t i, uint32_t k) {
    return e[orc_raw_index(tiled, maxn, i, joined ? nc + k : maxn - 1 - k)];
}

int64_t orc_table_diff(uint32_t n_rows, uint32_t maxn, int tiled_a, int joined_a,
                       const uint32_t* ent_a, const uint16_t* core_a, const uint16_t* skin_a,
                       int tiled_b, int joined_b, const uint32_t* ent_b, const uint16_t* core_b,
                       const uint16_t* skin_b, int nthreads) {
    int64_t first = INT64_MAX;
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static, 4096) num_threads(nthreads) reduction(min : first)
    for (int64_t ii = 0; ii < (int64_t)n_rows; ++ii) {
        const uint32_t i = (uint32_t)ii;
        int bad = core_a[i] != core_b[i] || skin_a[i] != skin_b[i];
        for (uint32_t k = 0; !bad && k < core_a[i]; ++k)
            bad = ent_a[orc_raw_index(tiled_a, maxn, i, k)] != ent_b[orc_raw_index(tiled_b, maxn, i, k)];
        for (uint32_t k = 0; !bad && k < skin_a[i]; ++k)
            bad = tbl_skin_at(tiled_a, joined_a, maxn, ent_a, core_a[i], i, k) !=
                  tbl_skin_at(tiled_b, joined_b, maxn, ent_b, core_b[i], i, k);
        if (bad && ii < first) first = ii;
    }
    return first == INT64_MAX ? -1 : first;
}

/* core asc then skin asc, counts kept (core_count, skin_count) */
void orc_join_core_skin(uint32_t n_rows, uint32_t maxn, int tiled, uint32_t* entries,
                        uint16_t* core, uint16_t* skinc) {
    (void)core;
    uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * maxn);
    for (uint32_t i = 0; i < n_rows; ++i) {
        const uint32_t nc = core[i], ns = skinc[i];
        for (uint32_t k = 0; k < ns; ++k) tmp[k] = entries[orc_raw_index(tiled, maxn, i, maxn - 1 - k)];
        for (uint32_t k = 0; k < ns; ++k) entries[orc_raw_index(tiled, maxn, i, nc + k)] = tmp[k];
    }
    free(tmp);
}

/* in-place transpose of each 32x32 tile (involution) */
void orc_tile_transpose(uint32_t n_rows_pad, uint32_t maxn, uint32_t* entries) {
    for (uint32_t tr = 0; tr < n_rows_pad; tr += 32)
        for (uint32_t tc = 0; tc < maxn; tc += 32)
            for (uint32_t a = 0; a < 32; ++a)
                for (uint32_t b = a + 1; b < 32; ++b) {
                    const size_t p = (size_t)(tr + a) * maxn + tc + b;
                    const size_t q = (size_t)(tr + b) * maxn + tc + a;
                    const uint32_t t = entries[p];
                    entries[p] = entries[q];
                    entries[q] = t;
                }
}

/* ======================================================================
 * forces -- restatement of the missing src/forces.cpp from S:405-475 and
 * P:59-88.  fp64 throughout.  PARITY UNPINNED.
 * ==================================================================== */
/* src/core.cpp:77-102 */
int orc_params_make(int32_t n_species, const double* a, const double* gamma, double kbt,
                    double s, double r_c, double dt, orc_params* p) {
    memset(p, 0, sizeof *p);
    if (r_c <= 0) return set_err(ORC_ECONFIG, "pair params: r_c must be positive");
    if (s <= 0) return set_err(ORC_ECONFIG, "pair params: weight exponent s must be positive");
    if (n_species < 1 || n_species > 4)
        return set_err(ORC_ECONFIG, "pair params: 1..4 species supported");
    for (int i = 0; i < n_species; ++i)
        for (int j = 0; j < i; ++j)
            if (a[i * n_species + j] != a[j * n_species + i] ||
                gamma[i * n_species + j] != gamma[j * n_species + i])
                return set_err(ORC_ECONFIG, "pair params: matrices must be symmetric");
    p->n_species = n_species;
    for (int q = 0; q < n_species * n_species; ++q) {
        p->a[q] = a[q];
        p->gamma[q] = gamma[q];
        p->sigma[q] = sqrt(2.0 * gamma[q] * kbt);
    }
    p->s = s;
    p->r_c = r_c;
    p->kbt = kbt;
    p->dt = dt;
    return ORC_OK;
}

static inline double weight_pow(double w, double s) {
    if (s == 1.0) return w;
    if (s == 2.0) return w * w;
    if (s == 3.0) return w * w * w;
    return orc_fastpow(w, s);
}

/* force on i from j; dr = x_i - x_j, dv = v_i - v_j, |dr| <= r_c */
int orc_pair_force(const orc_params* p, uint8_t si, uint8_t sj, const double dr[3],
                   const double dv[3], double xi, double f[3]) {
    const double r2 = dr[0] * dr[0] + dr[1] * dr[1] + dr[2] * dr[2];
    const double r = sqrt(r2);
    f[0] = f[1] = f[2] = 0.0;
    if (r == 0.0) return set_err(ORC_EPHYSICS, "coincident particles");
    if (r > p->r_c) return ORC_OK;
    const int q = si * p->n_species + sj;
    const double w = 1.0 - r / p->r_c;
    const double wr = weight_pow(w, p->s);
    const double inv_r = 1.0 / r;
    const double e[3] = {dr[0] * inv_r, dr[1] * inv_r, dr[2] * inv_r};
    const double ev = e[0] * dv[0] + e[1] * dv[1] + e[2] * dv[2];
    const double mag = p->a[q] * w - p->gamma[q] * (wr * wr) * ev +
                       p->sigma[q] * wr * xi / sqrt(p->dt);
    for (int k = 0; k < 3; ++k) f[k] = mag * e[k];
    return ORC_OK;
}

/* per-i full row, per-step |r|<=r_c re-check, row order */
int orc_compute_forces(const orc_params* p, const orc_box* box, size_t n_local,
                       const double* x, const double* y, const double* z, const double* vx,
                       const double* vy, const double* vz, const uint32_t* tag,
                       const uint8_t* species, const uint32_t* sig, uint32_t step_mix,
                       uint32_t maxn, int tiled, int joined, const uint32_t* entries,
                       const uint16_t* core, const uint16_t* skinc, double* fx, double* fy,
                       double* fz, int nthreads) {
    double L[3];
    for (int k = 0; k < 3; ++k) L[k] = box->hi[k] - box->lo[k];
    const double rc2 = p->r_c * p->r_c;
    int err = ORC_OK;
    uint32_t et0 = 0, et1 = 0;
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (size_t i = 0; i < n_local; ++i) {
        double acc[3] = {0, 0, 0};
        const uint32_t nc = core[i], ns = skinc[i];
        for (uint32_t m = 0; m < nc + ns; ++m) {
            uint32_t k;
            if (m < nc)
                k = m;
            else
                k = joined ? m : maxn - 1 - (m - nc);
            const uint32_t j = entries[orc_raw_index(tiled, maxn, (uint32_t)i, k)];
            double dr[3] = {x[i] - x[j], y[i] - y[j], z[i] - z[j]};
            for (int a = 0; a < 3; ++a) { /* src/core.cpp:129-139 */
                if (!box->periodic[a]) continue;
                if (dr[a] >= 0.5 * L[a])
                    dr[a] -= L[a];
                else if (dr[a] < -0.5 * L[a])
                    dr[a] += L[a];
            }
            const double r2 = dr[0] * dr[0] + dr[1] * dr[1] + dr[2] * dr[2];
            if (r2 > rc2) continue;
            if (r2 == 0.0) {
#pragma omp critical
                if (!err) {
                    err = ORC_EPHYSICS;
                    et0 = tag[i];
                    et1 = tag[j];
                }
                continue;
            }
            uint32_t u[2];
            orc_pair_uniforms(sig[i], sig[j], tag[i], tag[j], step_mix, u);
            const double xi = orc_gaussian(u[0], u[1]);
            const double dv[3] = {vx[i] - vx[j], vy[i] - vy[j], vz[i] - vz[j]};
            double f[3];
            orc_pair_force(p, species ? species[i] : 0, species ? species[j] : 0, dr, dv, xi, f);
            acc[0] += f[0];
            acc[1] += f[1];
            acc[2] += f[2];
        }
        fx[i] = acc[0];
        fy[i] = acc[1];
        fz[i] = acc[2];
    }
    if (err) return set_err(err, "coincident particles, tags %u and %u", et0, et1);
    return ORC_OK;
}

/* F = K (r - r0) along the bond, attractive when r > r0 */
int orc_bond_forces(const orc_box* box, size_t nb, const orc_bond* bonds, size_t n_tags,
                    const uint32_t* index_of_tag, const double* x, const double* y,
                    const double* z, double* fx, double* fy, double* fz) {
    for (size_t b = 0; b < nb; ++b) {
        const uint32_t ti = bonds[b].tag_i, tj = bonds[b].tag_j;
        if (ti >= n_tags || tj >= n_tags || index_of_tag[ti] == UINT32_MAX ||
            index_of_tag[tj] == UINT32_MAX)
            return set_err(ORC_EPHYSICS, "bond %u-%u: missing endpoint", ti, tj);
        const uint32_t i = index_of_tag[ti], j = index_of_tag[tj];
        double dr[3] = {x[i] - x[j], y[i] - y[j], z[i] - z[j]};
        for (int a = 0; a < 3; ++a) {
            if (!box->periodic[a]) continue;
            const double L = box->hi[a] - box->lo[a];
            if (dr[a] >= 0.5 * L)
                dr[a] -= L;
            else if (dr[a] < -0.5 * L)
                dr[a] += L;
        }
        const double r = sqrt(dr[0] * dr[0] + dr[1] * dr[1] + dr[2] * dr[2]);
        if (r == 0.0) return set_err(ORC_EPHYSICS, "bond %u-%u: zero length", ti, tj);
        const double c = -bonds[b].k * (r - bonds[b].r0) / r;
        fx[i] += c * dr[0];
        fy[i] += c * dr[1];
        fz[i] += c * dr[2];
        fx[j] -= c * dr[0];
        fy[j] -= c * dr[1];
        fz[j] -= c * dr[2];
    }
    return ORC_OK;
}

/* +g on the drive axis below the box midpoint of the partition
 * axis, -g at or above it (double Poiseuille) */
void orc_body_force(double midpoint, size_t n, const double* pos_p, double g, double* f_drive) {
    if (g == 0.0) return;
    for (size_t i = 0; i < n; ++i) f_drive[i] += pos_p[i] < midpoint ? g : -g;
}

/* ======================================================================
 * integrate -- restatement of the missing src/integrate.cpp.
 * h = 0.5*dt; v = v + h*f; x = x + dt*v; periodic wrap right after the
 * position update; specular walls.  PARITY UNPINNED.
 * ==================================================================== */
static inline int wrap_axis(double* xp, double* vp, double lo, double hi, int periodic, int wall) {
    double x = *xp;
    if (periodic) {
        const double L = hi - lo;
        if (x < lo) {
            x = x + L;
            if (x >= hi) x = lo;
        } else if (x >= hi) {
            x = x - L;
            if (x < lo) x = lo;
        }
        *xp = x;
        return x >= lo && x < hi;
    }
    if (wall) {
        if (x >= hi) {
            x = 2.0 * hi - x;
            *vp = -*vp;
            if (x >= hi) x = nextafter(hi, lo);
        } else if (x < lo) {
            x = 2.0 * lo - x;
            *vp = -*vp;
            if (x >= hi) x = nextafter(hi, lo);
        }
        *xp = x;
        return x >= lo && x < hi;
    }
    return 1;
}

int orc_verlet_phase1(const orc_box* box, double dt, size_t n, double* x, double* y, double* z,
                      double* vx, double* vy, double* vz, const double* fx, const double* fy,
                      const double* fz, const uint32_t* tag) {
    const double h = 0.5 * dt;
    int err = 0;
    uint32_t etag = 0;
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; ++i) {
        double* xs[3] = {&x[i], &y[i], &z[i]};
        double* vs[3] = {&vx[i], &vy[i], &vz[i]};
        const double fs[3] = {fx[i], fy[i], fz[i]};
        int ok = 1;
        for (int k = 0; k < 3; ++k) {
            *vs[k] = *vs[k] + h * fs[k];
            *xs[k] = *xs[k] + dt * *vs[k];
            if (!isfinite(*xs[k]) || !isfinite(*vs[k])) ok = 0;
            else if (!wrap_axis(xs[k], vs[k], box->lo[k], box->hi[k], box->periodic[k], box->wall[k]))
                ok = 0;
        }
        if (!ok) {
#pragma omp critical
            if (!err) {
                err = ORC_EPHYSICS;
                etag = tag ? tag[i] : (uint32_t)i;
            }
        }
    }
    if (err) return set_err(err, "blow-up: non-finite or escaped particle, tag %u", etag);
    return ORC_OK;
}

void orc_verlet_phase2(double dt, size_t n, double* vx, double* vy, double* vz,
                       const double* fx, const double* fy, const double* fz) {
    const double h = 0.5 * dt;
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; ++i) {
        vx[i] = vx[i] + h * fx[i];
        vy[i] = vy[i] + h * fy[i];
        vz[i] = vz[i] + h * fz[i];
    }
}

/* src/core.cpp:141-149 */
int orc_compute_temperature(size_t n, const double* vx, const double* vy, const double* vz,
                            double* kbt) {
    if (n == 0) return set_err(ORC_EPHYSICS, "temperature of an empty system");
    double m[3] = {0, 0, 0};
    for (size_t i = 0; i < n; ++i) {
        m[0] += vx[i];
        m[1] += vy[i];
        m[2] += vz[i];
    }
    for (int k = 0; k < 3; ++k) m[k] *= 1.0 / (double)n;
    double s = 0;
    for (size_t i = 0; i < n; ++i) {
        const double a = vx[i] - m[0], b = vy[i] - m[1], c = vz[i] - m[2];
        s += a * a + b * b + c * c;
    }
    *kbt = s / (3.0 * (double)n);
    return ORC_OK;
}

/* ======================================================================
 * init -- S:44-52 (the reference init.cpp is missing).  Counter-based
 * TeaStream draws (inc/rng.hpp:95-107): particle i uses counters 6i..6i+5
 * for x,y,z,vx,vy,vz; velocities sqrt(kbt)*gaussian, COM removed.
 * ==================================================================== */
int orc_init_fluid(const orc_box* box, size_t n, double kbt, uint32_t seed, double* x,
                   double* y, double* z, double* vx, double* vy, double* vz, uint32_t* tag) {
    if (n == 0) return set_err(ORC_ECONFIG, "init: empty system");
    const double sk = sqrt(kbt);
    double* xs[3] = {x, y, z};
    double* vs[3] = {vx, vy, vz};
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; ++i) {
        for (int k = 0; k < 3; ++k) {
            uint32_t h[2];
            orc_tea_hash(16, seed, (uint32_t)(6 * i + k), h);
            const double L = box->hi[k] - box->lo[k];
            double p = box->lo[k] + L * ((double)h[0] * 0x1p-32);
            if (p >= box->hi[k]) p = box->lo[k];
            xs[k][i] = p;
            orc_tea_hash(16, seed, (uint32_t)(6 * i + 3 + k), h);
            vs[k][i] = sk * orc_gaussian(h[0], h[1]);
        }
        tag[i] = (uint32_t)(i + 1);
    }
    for (int k = 0; k < 3; ++k) {
        double m = 0;
        for (size_t i = 0; i < n; ++i) m += vs[k][i];
        m /= (double)n;
        for (size_t i = 0; i < n; ++i) vs[k][i] -= m;
    }
    return ORC_OK;
}

/* ======================================================================
 * whole-step CPU driver: Alg. 1 on one domain.
 * Step numbering frozen: setup forces use step 0; loop step n (1-based)
 * runs phase1, rebuild if n % R == 0, signatures from the post-phase-1
 * velocity, forces with step_mix(seed, n), body force, phase2.
 * ==================================================================== */
struct orc_sim {
    /* CPU-baseline instrumentation: wall seconds per stage (integrate, reorder,
     * build, forces) and an optional reorder hook (the reference's own shipped
     * reorder_particles + cell list, oracle/ref_shim.cpp) */
    double t_stage[4];
    orc_reorder_hook hook;
    void* hook_ctx;
    orc_box box;
    orc_params p;
    orc_grid g;
    double skin;
    int rebuild_every, drive_axis, partition_axis, nthreads;
    uint32_t maxn, seed;
    double body_force;
    size_t n, n_pad;
    int64_t step;
    double *x[3], *v[3], *f[3];
    uint32_t *tag, *sig, *order, *cell_start, *coff, *ccells, *entries;
    uint8_t* species;
    uint16_t *core, *skinc;
    void* scratch;
};

static int sim_reorder_own(orc_sim* s);
static int sim_reorder(orc_sim* s) {
    const size_t n = s->n;
    if (s->hook) {
        double inner = 0.0;
        const int rc = s->hook(s->hook_ctx, n, s->x, s->v, s->tag, s->species, s->cell_start, &inner);
        s->t_stage[1] += inner;
        return rc;
    }
    const double t0 = omp_get_wtime();
    const int rc0 = sim_reorder_own(s);
    s->t_stage[1] += omp_get_wtime() - t0;
    return rc0;
}

static int sim_reorder_own(orc_sim* s) {
    const size_t n = s->n;
    int rc = orc_reorder_order(&s->g, n, s->x[0], s->x[1], s->x[2], s->order, NULL, s->nthreads);
    if (rc) return rc;
    double* tmp = (double*)s->scratch;
    for (int k = 0; k < 3; ++k) {
        double* arrs[2] = {s->x[k], s->v[k]};
        for (int a = 0; a < 2; ++a) {
#pragma omp parallel for schedule(static) num_threads(s->nthreads)
            for (size_t t = 0; t < n; ++t) tmp[t] = arrs[a][s->order[t]];
            memcpy(arrs[a], tmp, n * 8);
        }
    }
    uint32_t* t32 = (uint32_t*)tmp;
    for (size_t t = 0; t < n; ++t) t32[t] = s->tag[s->order[t]];
    memcpy(s->tag, t32, n * 4);
    uint8_t* t8 = (uint8_t*)tmp;
    for (size_t t = 0; t < n; ++t) t8[t] = s->species[s->order[t]];
    memcpy(s->species, t8, n);
    /* cell list */
    uint32_t* ranks = (uint32_t*)tmp;
    rc = orc_local_cell_ranks(&s->g, n, s->x[0], s->x[1], s->x[2], ranks);
    if (rc) return rc;
    return orc_build_cell_list(s->g.n_total_cells, ranks, n, s->cell_start);
}

static int sim_forces(orc_sim* s) {
    orc_signatures(s->n, s->tag, s->v[0], s->v[1], s->v[2], s->sig);
    const uint32_t mix = orc_step_mix(s->seed, (uint32_t)s->step);
    int rc = orc_compute_forces(&s->p, &s->box, s->n, s->x[0], s->x[1], s->x[2], s->v[0],
                                s->v[1], s->v[2], s->tag, s->species, s->sig, mix, s->maxn, 0, 0,
                                s->entries, s->core, s->skinc, s->f[0], s->f[1], s->f[2],
                                s->nthreads);
    if (rc) return rc;
    if (s->body_force != 0.0) {
        const double mid = 0.5 * (s->box.lo[s->partition_axis] + s->box.hi[s->partition_axis]);
        double* pp = s->x[s->partition_axis];
        double* fd = s->f[s->drive_axis];
        orc_body_force(mid, s->n, pp, s->body_force, fd);
    }
    return ORC_OK;
}

static int sim_build(orc_sim* s) {
    return orc_build_neighbor_table(&s->g, &s->box, s->cell_start, s->coff, s->ccells, s->n, s->n,
                                    s->x[0], s->x[1], s->x[2], s->tag, s->p.r_c, s->skin, s->maxn,
                                    s->entries, s->core, s->skinc, s->nthreads);
}

orc_sim* orc_sim_create(const orc_box* box, const orc_params* p, double skin, int rebuild_every,
                        uint32_t maxn, uint32_t seed, double body_force, int drive_axis,
                        int partition_axis, size_t n, const double* x, const double* y,
                        const double* z, const double* vx, const double* vy, const double* vz,
                        const uint32_t* tag, const uint8_t* species, int nthreads) {
    orc_sim* s = (orc_sim*)calloc(1, sizeof(orc_sim));
    s->box = *box;
    s->p = *p;
    s->skin = skin;
    s->rebuild_every = rebuild_every;
    s->maxn = maxn;
    s->seed = seed;
    s->body_force = body_force;
    s->drive_axis = drive_axis;
    s->partition_axis = partition_axis;
    s->nthreads = nthreads < 1 ? 1 : nthreads;
    s->n = n;
    s->n_pad = (n + 31) & ~(size_t)31;
    const int32_t dims[3] = {1, 1, 1}, crd[3] = {0, 0, 0};
    if (orc_grid_make(box, box->lo, box->hi, dims, crd, p->r_c + skin, 2, &s->g)) {
        free(s);
        return NULL;
    }
    const double* src_x[3] = {x, y, z};
    const double* src_v[3] = {vx, vy, vz};
    for (int k = 0; k < 3; ++k) {
        s->x[k] = (double*)malloc(n * 8 + 8);
        s->v[k] = (double*)malloc(n * 8 + 8);
        s->f[k] = (double*)calloc(n + 1, 8);
        memcpy(s->x[k], src_x[k], n * 8);
        memcpy(s->v[k], src_v[k], n * 8);
    }
    s->tag = (uint32_t*)malloc(n * 4 + 4);
    memcpy(s->tag, tag, n * 4);
    s->species = (uint8_t*)calloc(n + 1, 1);
    if (species) memcpy(s->species, species, n);
    s->sig = (uint32_t*)malloc(n * 4 + 4);
    s->order = (uint32_t*)malloc(n * 4 + 4);
    s->cell_start = (uint32_t*)malloc(((size_t)s->g.n_total_cells + 1) * 4);
    s->coff = (uint32_t*)malloc(((size_t)s->g.n_local_cells + 1) * 4);
    s->ccells = (uint32_t*)malloc((size_t)s->g.n_local_cells * 27 * 4);
    orc_coarse_stencil(&s->g, s->coff, s->ccells);
    s->entries = (uint32_t*)malloc(s->n_pad * maxn * 4 + 4);
    s->core = (uint16_t*)calloc(s->n_pad + 1, 2);
    s->skinc = (uint16_t*)calloc(s->n_pad + 1, 2);
    s->scratch = malloc(n * 8 + 8);
    s->step = 0;
    if (sim_reorder(s) || sim_build(s) || sim_forces(s)) {
        orc_sim_destroy(s);
        return NULL;
    }
    return s;
}

void orc_sim_destroy(orc_sim* s) {
    if (!s) return;
    for (int k = 0; k < 3; ++k) {
        free(s->x[k]);
        free(s->v[k]);
        free(s->f[k]);
    }
    free(s->tag);
    free(s->species);
    free(s->sig);
    free(s->order);
    free(s->cell_start);
    free(s->coff);
    free(s->ccells);
    free(s->entries);
    free(s->core);
    free(s->skinc);
    free(s->scratch);
    orc_grid_free(&s->g);
    free(s);
}

int orc_sim_run(orc_sim* s, int64_t nsteps) {
    for (int64_t t = 0; t < nsteps; ++t) {
        double t0 = omp_get_wtime();
        int rc = orc_verlet_phase1(&s->box, s->p.dt, s->n, s->x[0], s->x[1], s->x[2], s->v[0],
                                   s->v[1], s->v[2], s->f[0], s->f[1], s->f[2], s->tag);
        s->t_stage[0] += omp_get_wtime() - t0;
        if (rc) return rc;
        s->step += 1;
        if (s->step % s->rebuild_every == 0) {
            rc = sim_reorder(s);
            if (rc) return rc;
            t0 = omp_get_wtime();
            rc = sim_build(s);
            s->t_stage[2] += omp_get_wtime() - t0;
            if (rc) return rc;
        }
        t0 = omp_get_wtime();
        rc = sim_forces(s);
        s->t_stage[3] += omp_get_wtime() - t0;
        if (rc) return rc;
        t0 = omp_get_wtime();
        orc_verlet_phase2(s->p.dt, s->n, s->v[0], s->v[1], s->v[2], s->f[0], s->f[1], s->f[2]);
        s->t_stage[0] += omp_get_wtime() - t0;
    }
    return ORC_OK;
}

int orc_sim_set_reorder_hook(orc_sim* s, orc_reorder_hook hook, void* ctx) {
    s->hook = hook;
    s->hook_ctx = ctx;
    return ORC_OK;
}

void orc_sim_stage_seconds(orc_sim* s, double out[4], int reset) {
    for (int k = 0; k < 4; ++k) {
        out[k] = s->t_stage[k];
        if (reset) s->t_stage[k] = 0.0;
    }
}

int64_t orc_sim_step_index(const orc_sim* s) { return s->step; }
size_t orc_sim_n(const orc_sim* s) { return s->n; }

void orc_sim_get(const orc_sim* s, double* x, double* y, double* z, double* vx, double* vy,
                 double* vz, double* fx, double* fy, double* fz, uint32_t* tag) {
    double* outs[9] = {x, y, z, vx, vy, vz, fx, fy, fz};
    const double* ins[9] = {s->x[0], s->x[1], s->x[2], s->v[0], s->v[1],
                            s->v[2], s->f[0], s->f[1], s->f[2]};
    for (int a = 0; a < 9; ++a)
        if (outs[a]) memcpy(outs[a], ins[a], s->n * 8);
    if (tag) memcpy(tag, s->tag, s->n * 4);
}

double orc_sim_temperature(const orc_sim* s) {
    double t = 0;
    orc_compute_temperature(s->n, s->v[0], s->v[1], s->v[2], &t);
    return t;
}
