/*
 * dpd_oracle.h -- CPU restatement of the reference DPD hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 engine (paper_1311_0402_b200/libdpdb.so).  Only tests/, the smoke()
 * entry in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * leg may load it.  The product path never calls into it.
 *
 * Every function cites the reference file:line it restates:
 *   inc/ = /root/reference/proj/include/dpd/   src/ = /root/reference/proj/src/
 *   S:   = /root/reference/SPEC.md              P:   = /root/reference/PAPER.md
 *
 * Parity pinning:
 *   - fastmath / rng / morton / radix / cell grid / reorder / cell list /
 *     stencils are checked bit-for-bit against the reference's own shipped
 *     code (oracle/_ref, built from /root/reference by oracle/Makefile) and
 *     against the golden fixtures in tests/golden/ generated from it.
 *   - neighbor builder, forces, bonds, integrator: the reference .cpp files
 *     are absent (CMakeLists.txt:21-23 lists them, they are not shipped), so
 *     these are "parity unpinned" restatements of inc/neighbor_table.hpp and
 *     SPEC.md; they are pinned by the SPEC examples and O(N^2) brute force.
 *
 * Floating-point contract: compiled with -ffp-contract=off so that every
 * a*b+c is two roundings, exactly like the CUDA kernels which use
 * __dmul_rn/__dadd_rn/__fmul_rn/__fadd_rn on the bit-exact paths.
 */
#ifndef DPD_ORACLE_H
#define DPD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error categories, inc/error.hpp:8-13 */
enum { ORC_OK = 0, ORC_ECONFIG = 1, ORC_EPHYSICS = 2, ORC_EPROTOCOL = 3, ORC_EIO = 4 };
const char* orc_last_error(void);

/* ---------------------------------------------------------------- fastmath */
double orc_power2(int n);
double orc_exp2_frac(double x);
double orc_log2_frac(double x);
double orc_fastlog(uint32_t v);
double orc_fastcos2pi(uint32_t v);
double orc_fastpow(double a, double b);

/* --------------------------------------------------------------------- rng */
void orc_tea_hash(int rounds, uint32_t v0, uint32_t v1, uint32_t out[2]);
uint32_t orc_bit_reverse(uint32_t x);
uint32_t orc_mantissa11(double v);
uint32_t orc_make_signature(uint32_t tag, double vx, double vy, double vz);
uint32_t orc_step_mix(uint32_t seed, uint32_t step);
void orc_pair_uniforms(uint32_t sig_i, uint32_t sig_j, uint32_t tag_i, uint32_t tag_j,
                       uint32_t step_mix, uint32_t out[2]);
double orc_gaussian(uint32_t ua, uint32_t ub);
/* batch helpers for tests */
void orc_signatures(size_t n, const uint32_t* tag, const double* vx, const double* vy,
                    const double* vz, uint32_t* sig);

/* ------------------------------------------------------------------ morton */
int orc_morton_encode(uint32_t ix, uint32_t iy, uint32_t iz, int bits, uint32_t* code);

/* ------------------------------------------------------------------- radix */
int orc_radix_sort(uint32_t* keys, uint32_t* vals, size_t n, int bit_length, int nthreads);

/* -------------------------------------------------------------------- grid */
typedef struct {
    double lo[3], hi[3];
    int32_t periodic[3], wall[3];
} orc_box;

typedef struct {
    int32_t ncell[3], ncell_ext[3], ghost_lo[3], ghost_hi[3], wrapmode[3];
    double cell_size[3], inv_cell[3], slab_lo[3], slab_hi[3], origin[3];
    int32_t sub_bits, bits_per_axis;
    uint32_t n_local_cells, n_total_cells;
    uint32_t* rank_of_cell; /* ext lattice index -> rank */
    uint32_t* cell_of_rank; /* rank -> ext lattice index */
} orc_grid;

int orc_grid_make(const orc_box* box, const double slab_lo[3], const double slab_hi[3],
                  const int32_t dims[3], const int32_t coords[3], double cell_target,
                  int32_t sub_bits, orc_grid* g);
void orc_grid_free(orc_grid* g);
int orc_grid_key_bits(const orc_grid* g);
/* ext-lattice cell of a local particle; error (protocol) outside the slab */
int orc_local_cell_of(const orc_grid* g, const double x[3], int32_t c[3]);
uint32_t orc_sub_code(const orc_grid* g, const double x[3], const int32_t c[3]);

/* sort keys of n local particles (rank << 3*sub_bits | sub_code) */
int orc_sort_keys(const orc_grid* g, size_t n, const double* x, const double* y,
                  const double* z, uint32_t* keys);
/* stable order of the keys: order[to] = from; perm[from] = to */
int orc_reorder_order(const orc_grid* g, size_t n, const double* x, const double* y,
                      const double* z, uint32_t* order, uint32_t* perm, int nthreads);
/* cell ranks of already-sorted particles + boundary-detection cell list */
int orc_local_cell_ranks(const orc_grid* g, size_t n, const double* x, const double* y,
                         const double* z, uint32_t* ranks);
int orc_build_cell_list(uint32_t n_total_cells, const uint32_t* ranks, size_t n,
                        uint32_t* cell_start /* n_total_cells+1 */);

/* coarse stencil: offsets[n_local_cells+1], cells[<=27*n_local_cells] */
int orc_coarse_stencil(const orc_grid* g, uint32_t* offsets, uint32_t* cells);
/* fine stencil sizes then fill */
int orc_fine_stencil(uint32_t n_local_cells, const uint32_t* coff, const uint32_t* ccells,
                     const uint32_t* cell_start, uint32_t* foff, uint32_t* fidx);

/* ---------------------------------------------------------- neighbor table */
/* entries: n_rows_pad*maxn, row-major (tiled=0).  Rows for particles
 * [0, n_local); candidates j in [0, n_all) (locals then ghosts). */
int orc_build_neighbor_table(const orc_grid* g, const orc_box* box, const uint32_t* cell_start,
                             const uint32_t* coff, const uint32_t* ccells, size_t n_local,
                             size_t n_all, const double* x, const double* y, const double* z,
                             const uint32_t* tag, double r_c, double skin, uint32_t maxn,
                             uint32_t* entries, uint16_t* core, uint16_t* skinc, int nthreads);
void orc_join_core_skin(uint32_t n_rows, uint32_t maxn, int tiled, uint32_t* entries,
                        uint16_t* core, uint16_t* skinc);
void orc_tile_transpose(uint32_t n_rows_pad, uint32_t maxn, uint32_t* entries);
size_t orc_raw_index(int tiled, uint32_t maxn, uint32_t i, uint32_t k);
/* test helper: compare table A (any layout) with table B (any layout) row by
 * row through the inc/neighbor_table.hpp:33-39 accessors; returns the first
 * differing row (counts or any core/skin entry), or -1 when identical */
int64_t orc_table_diff(uint32_t n_rows, uint32_t maxn, int tiled_a, int joined_a,
                       const uint32_t* ent_a, const uint16_t* core_a, const uint16_t* skin_a,
                       int tiled_b, int joined_b, const uint32_t* ent_b, const uint16_t* core_b,
                       const uint16_t* skin_b, int nthreads);

/* ------------------------------------------------------------------ forces */
typedef struct {
    int32_t n_species;
    double a[16], gamma[16], sigma[16]; /* n_species^2 <= 16 */
    double s, r_c, kbt, dt;
} orc_params;

int orc_params_make(int32_t n_species, const double* a, const double* gamma, double kbt,
                    double s, double r_c, double dt, orc_params* p);

/* full-row force evaluation.  joined: row layout flag. */
int orc_compute_forces(const orc_params* p, const orc_box* box, size_t n_local,
                       const double* x, const double* y, const double* z, const double* vx,
                       const double* vy, const double* vz, const uint32_t* tag,
                       const uint8_t* species, const uint32_t* sig, uint32_t step_mix,
                       uint32_t maxn, int tiled, int joined, const uint32_t* entries,
                       const uint16_t* core, const uint16_t* skinc, double* fx, double* fy,
                       double* fz, int nthreads);
/* single pair, for examples: force on i */
int orc_pair_force(const orc_params* p, uint8_t si, uint8_t sj, const double dr[3],
                   const double dv[3], double xi, double f[3]);

typedef struct {
    uint32_t tag_i, tag_j;
    double k, r0;
} orc_bond;
/* harmonic bonds; index_of_tag: tag -> local index or UINT32_MAX */
int orc_bond_forces(const orc_box* box, size_t nb, const orc_bond* bonds, size_t n_tags,
                    const uint32_t* index_of_tag, const double* x, const double* y,
                    const double* z, double* fx, double* fy, double* fz);
void orc_body_force(double midpoint, size_t n, const double* pos_p, double g, double* f_drive);

/* -------------------------------------------------------------- integrate */
int orc_verlet_phase1(const orc_box* box, double dt, size_t n, double* x, double* y, double* z,
                      double* vx, double* vy, double* vz, const double* fx, const double* fy,
                      const double* fz, const uint32_t* tag);
void orc_verlet_phase2(double dt, size_t n, double* vx, double* vy, double* vz,
                       const double* fx, const double* fy, const double* fz);
int orc_compute_temperature(size_t n, const double* vx, const double* vy, const double* vz,
                            double* kbt);

/* ------------------------------------------------------------ init */
int orc_init_fluid(const orc_box* box, size_t n, double kbt, uint32_t seed, double* x,
                   double* y, double* z, double* vx, double* vy, double* vz, uint32_t* tag);

/* ---------------------------------------------------- whole-step CPU driver */
typedef struct orc_sim orc_sim;
orc_sim* orc_sim_create(const orc_box* box, const orc_params* p, double skin, int rebuild_every,
                        uint32_t maxn, uint32_t seed, double body_force, int drive_axis,
                        int partition_axis, size_t n, const double* x, const double* y,
                        const double* z, const double* vx, const double* vy, const double* vz,
                        const uint32_t* tag, const uint8_t* species, int nthreads);
void orc_sim_destroy(orc_sim* s);
/* reorder step replacement for the CPU baseline (the reference's own shipped
 * reorder_particles, oracle/ref_shim.cpp ref_sim_reorder): permute x, v, tag,
 * species in place, fill cell_start, report the seconds spent in *seconds */
typedef int (*orc_reorder_hook)(void* ctx, size_t n, double* x[3], double* v[3], uint32_t* tag,
                                uint8_t* species, uint32_t* cell_start, double* seconds);
int orc_sim_set_reorder_hook(orc_sim* s, orc_reorder_hook hook, void* ctx);
/* wall seconds per stage since the last reset: integrate, reorder, build, forces */
void orc_sim_stage_seconds(orc_sim* s, double out[4], int reset);
int orc_sim_run(orc_sim* s, int64_t nsteps);
int64_t orc_sim_step_index(const orc_sim* s);
size_t orc_sim_n(const orc_sim* s);
void orc_sim_get(const orc_sim* s, double* x, double* y, double* z, double* vx, double* vy,
                 double* vz, double* fx, double* fy, double* fz, uint32_t* tag);
double orc_sim_temperature(const orc_sim* s);

#ifdef __cplusplus
}
#endif
#endif
