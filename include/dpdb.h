/*
 * dpdb.h -- C ABI of the B200-native DPD engine (libdpdb.so).
 *
 * This is the drop-in boundary for the reference's per-step hot path.  The
 * reference is a C++20 library whose hot-path entry points are:
 *
 *   CellGrid::make                    inc/cell_grid.hpp:39-43
 *   reorder_particles                 inc/cell_grid.hpp:78-79  (src/cell_grid.cpp:166-198)
 *   local_cell_ranks/build_cell_list  inc/cell_grid.hpp:74,82  (src/cell_grid.cpp:136-164)
 *   RadixSorter::sort / radix_sort    inc/radix_sort.hpp:15-27 (src/radix_sort.cpp:16-74)
 *   build_coarse_stencil              inc/stencil.hpp:24       (src/stencil.cpp:7-41)
 *   expand_fine_stencil               inc/stencil.hpp:39-40    (src/stencil.cpp:43-62)
 *   build_neighbor_table              inc/neighbor_table.hpp:45-47 (impl. not shipped)
 *   join_core_skin / tile_transpose   inc/neighbor_table.hpp:51,55
 *   make_signature / pair_uniforms /
 *   gaussian / fastlog / fastcos2pi /
 *   fastpow / tea_hash                inc/rng.hpp:25-91, inc/fastmath.hpp:92-151
 *   compute_forces / bond_forces      SPEC.md:434-451 (impl. not shipped)
 *   verlet_step / apply_body_force    SPEC.md:488-505 (impl. not shipped)
 *   compute_temperature               inc/core.hpp:116 (src/core.cpp:141-149)
 *
 * The reference's own declarations (same signatures and types, compiled
 * against its unmodified headers) are implemented over this ABI in dropin/:
 * src/cell_grid.cpp and src/radix_sort.cpp are replaced, the missing
 * src/neighbor_table.cpp, src/forces.cpp and src/integrate.cpp slots are
 * filled.
 *
 * Conventions (mirroring the reference's):
 *   - return 0 on success, otherwise the reference ErrorCategory value
 *     (inc/error.hpp:8-13): 1 config, 2 physics, 3 protocol, 4 io; plus
 *     5 = CUDA/device error.  dpdb_last_error() gives the message.
 *   - host arrays are caller-owned and only touched during the call; every
 *     call is synchronous at the boundary and runs on the context's stream.
 *   - a context is not thread-safe (the reference's WorkerPool runs one job
 *     at a time, src/parallel.cpp:63-83).
 *   - there is no CPU fallback: creating a context without an sm_100 device
 *     fails with code 5.
 */
#ifndef DPDB_H
#define DPDB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPDB_OK 0
#define DPDB_ECONFIG 1
#define DPDB_EPHYSICS 2
#define DPDB_EPROTOCOL 3
#define DPDB_EIO 4
#define DPDB_EDEVICE 5

/* SimBox, inc/core.hpp:15-25 */
typedef struct {
    double lo[3], hi[3];
    int32_t periodic[3];
    int32_t wall[3];
} dpdb_box;

/* PairParams, inc/core.hpp:51-68 (sigma derived: sigma^2 = 2 gamma kbt) */
typedef struct {
    int32_t n_species;          /* 1..4 */
    double a[16], gamma[16];    /* n_species x n_species, row-major, symmetric */
    double kbt, s, r_c, dt;
} dpdb_params;

/* RunConfig subset, inc/core.hpp:83-109 */
typedef struct {
    int32_t rebuild_every;      /* default 10 */
    double skin;                /* default 0.3 */
    double body_force;          /* double-Poiseuille g, 0 = off */
    int32_t drive_axis;         /* default 2 */
    int32_t partition_axis;     /* default 0 */
    uint32_t seed;              /* default 1 */
    uint32_t max_neighbors;     /* default 128, multiple of 32, <= 4096 */
    int32_t sub_bits;           /* default 2 (inc/cell_grid.hpp:30) */
    int32_t wall_mode;          /* walls: 0 specular "bounce-forward" (default),
                                   1 bounce-back (every velocity component reversed) */
} dpdb_run;

/* thermo line */
typedef struct {
    int64_t step;
    uint64_t n;
    double kbt;                 /* compute_temperature, COM-subtracted */
    double momentum[3];
} dpdb_thermo;

/* CellGrid geometry, inc/cell_grid.hpp:21-70 */
typedef struct {
    int32_t ncell[3], ncell_ext[3], wrapmode[3];
    int32_t bits_per_axis, key_bits;
    uint32_t n_local_cells, n_total_cells;
    double cell_size[3], inv_cell[3], origin[3];
} dpdb_grid_info;

typedef struct dpdb_ctx dpdb_ctx;

const char* dpdb_version(void);
/* last error of ctx (or of the calling thread when ctx is NULL) */
const char* dpdb_last_error(const dpdb_ctx* ctx);
/* number of CUDA devices with compute capability 10.x, or -1 on error */
int dpdb_device_count(void);

/* ---------------------------------------------------------------- context */
int dpdb_create(int device, const dpdb_box* box, const dpdb_params* params, const dpdb_run* run,
                size_t capacity, dpdb_ctx** out);
int dpdb_destroy(dpdb_ctx* ctx);
int dpdb_grid(const dpdb_ctx* ctx, dpdb_grid_info* out);
/* rank_of_cell[n_total_cells] (ext lattice index -> rank) */
int dpdb_grid_ranks(const dpdb_ctx* ctx, uint32_t* rank_of_cell);
/* CUDA stream of the context (cudaStream_t) for interop */
void* dpdb_stream(dpdb_ctx* ctx);
/* CellGrid::make (inc/cell_grid.hpp:39-43, src/cell_grid.cpp:16-95) on the
 * host, no device involved: the cell geometry of the slab [slab_lo, slab_hi)
 * of a dims decomposition at coords (slab_lo/slab_hi/dims/coords all NULL:
 * the single-domain grid over the box), cells >= cell_target per axis,
 * 2^sub_bits sub-cells per axis.  ghost_lo/ghost_hi (may be NULL) receive the
 * ghost layers; rank_of_cell may be NULL (size: out->n_total_cells).  The
 * same grid every context on that box builds. */
int dpdb_grid_plan(const dpdb_box* box, const double slab_lo[3], const double slab_hi[3],
                   const int32_t dims[3], const int32_t coords[3], double cell_target,
                   int32_t sub_bits, dpdb_grid_info* out, int32_t ghost_lo[3], int32_t ghost_hi[3],
                   uint32_t* rank_of_cell);

/* ------------------------------------------------------- state transfer */
/* ParticleStore SoA, inc/core.hpp:29-47.  species/molecule may be NULL. */
int dpdb_upload(dpdb_ctx* ctx, size_t n, const double* x, const double* y, const double* z,
                const double* vx, const double* vy, const double* vz, const uint32_t* tag,
                const uint8_t* species, const uint32_t* molecule);
int dpdb_upload_forces(dpdb_ctx* ctx, const double* fx, const double* fy, const double* fz);
/* any pointer may be NULL */
int dpdb_download(dpdb_ctx* ctx, double* x, double* y, double* z, double* vx, double* vy,
                  double* vz, double* fx, double* fy, double* fz, uint32_t* tag,
                  uint8_t* species, uint32_t* signature);
int dpdb_size(const dpdb_ctx* ctx, size_t* n);
/* Harmonic bonds (BondTopology, inc/core.hpp:70-81): K (r - r0) along the bond */
/* init_random on the device: n particles uniform in the box,
 * Maxwell-Boltzmann velocities at kbt with zero net momentum, counter-based
 * draws tea_hash(16, seed, c) (bit-exact with the oracle's init_fluid when
 * n_chains = 0).  The first n_chains * chain_len particles form chains (random
 * walks with step r0, species chain_species[b] per bead, molecule = chain + 1,
 * harmonic bonds of stiffness bond_k and rest length r0 between neighbours);
 * the rest are solvent of species solvent_species.  Tags 1..n. */
int dpdb_init_random(dpdb_ctx* ctx, size_t n, double kbt, uint32_t seed, uint32_t n_chains,
                     uint32_t chain_len, const uint8_t* chain_species, uint8_t solvent_species,
                     double r0, double bond_k);
int dpdb_set_bonds(dpdb_ctx* ctx, size_t nb, const uint32_t* tag_i, const uint32_t* tag_j,
                   const double* k, const double* r0);
/* bonds with a style per bond: 0 harmonic, 1 FENE
 * F = -K r / (1 - (r/R0)^2), R0 given in r0 (no reference implementation:
 * the standard formula, unpinned; r >= R0 is a physics error) */
int dpdb_set_bonds_styled(dpdb_ctx* ctx, size_t nb, const uint32_t* ti, const uint32_t* tj,
                          const double* k, const double* r0, const uint8_t* style);
/* harmonic angles U = K (theta - theta0)^2 / 2 around the middle tag tb of
 * (ta, tb, tc), theta0 in radians (unpinned: no reference implementation);
 * evaluated per particle with the bonds (no atomics) */
int dpdb_set_angles(dpdb_ctx* ctx, size_t na, const uint32_t* ta, const uint32_t* tb,
                    const uint32_t* tc, const double* k, const double* theta0);

/* ------------------------------------------- per-stage entry points */
/* sort keys of the current (unsorted) state, src/cell_grid.cpp:168-175 */
int dpdb_sort_keys(dpdb_ctx* ctx, uint32_t* keys);
/* reorder_particles: keys -> stable radix sort -> permute -> cell list.
 * perm (old -> new, may be NULL) as returned by the reference. */
int dpdb_reorder(dpdb_ctx* ctx, uint32_t* perm);
int dpdb_cell_start(dpdb_ctx* ctx, uint32_t* cell_start /* n_total_cells + 1 */);
/* coarse stencil in the reference CSR form: offsets[n_local_cells+1], cells[] */
int dpdb_coarse_stencil(dpdb_ctx* ctx, uint32_t* offsets, uint32_t* cells);
/* fine stencil (expand_fine_stencil): offsets[n_local_cells+1]; indices may be
 * NULL to query the size (offsets[n_local_cells]) */
int dpdb_fine_stencil(dpdb_ctx* ctx, uint32_t* offsets, uint32_t* indices);
/* build_neighbor_table over the current (reordered) state */
int dpdb_build_neighbors(dpdb_ctx* ctx);
/* layout transforms of the device table */
int dpdb_join_core_skin(dpdb_ctx* ctx);
int dpdb_tile_transpose(dpdb_ctx* ctx);
/* export: entries[n_rows_pad * max_neighbors] in the table's CURRENT layout,
 * unused slots zeroed; core/skin counts u16 per row.  tiled and joined report
 * the layout flags (NeighborTable::tiled/joined, inc/neighbor_table.hpp:22-23). */
int dpdb_get_neighbors(dpdb_ctx* ctx, uint32_t* entries, uint16_t* core, uint16_t* skin,
                       int32_t* tiled, int32_t* joined);
/* import a neighbor table (NeighborTable, inc/neighbor_table.hpp:18-40) for
 * the current particle order: entries[n_rows_pad * max_neighbors] in the
 * given layout (tiled / joined flags), core/skin counts per row.  The next
 * dpdb_compute_forces evaluates exactly these rows (the reference's
 * compute_forces(store, table, ...) contract). */
int dpdb_set_neighbors(dpdb_ctx* ctx, const uint32_t* entries, const uint16_t* core,
                       const uint16_t* skin, int32_t tiled, int32_t joined);
/* join_core_skin (op 0) / tile_transpose (op 1) of a caller-owned table
 * (inc/neighbor_table.hpp:49-55) on the device, in place:
 * entries[round_up(n_rows, 32) * max_neighbors] in the layout given by
 * tiled / joined, counts per row.  No context needed. */
int dpdb_table_layout(int device, int op, size_t n_rows, uint32_t max_neighbors, uint32_t* entries,
                      const uint16_t* core, const uint16_t* skin, int32_t tiled, int32_t joined);
/* per-particle signatures from the current fp64 velocities */
int dpdb_signatures(dpdb_ctx* ctx, uint32_t* sig);
/* compute_forces + bond_forces + apply_body_force with step_mix(seed, step) */
int dpdb_compute_forces(dpdb_ctx* ctx, uint32_t step);
int dpdb_verlet_phase1(dpdb_ctx* ctx);
int dpdb_verlet_phase2(dpdb_ctx* ctx);

/* ------------------------------------------------- device-resident path */
/* Alg. 1 setup: reorder, cell list, build, signatures, forces(step 0) */
int dpdb_setup(dpdb_ctx* ctx);
/* restart: setup as at step `step` -- reorder, neighbor build and,
 * unless keep_forces, forces with step_mix(seed, step).  A restart uploads the
 * saved forces (dpdb_upload_forces) and keeps them: f(n) was evaluated with the
 * half-step velocity, so it is state, not recomputable from v(n).  A state saved
 * after dpdb_step at a rebuild step (step % rebuild_every == 0) then continues
 * bitwise like the uninterrupted run. */
int dpdb_setup_at(dpdb_ctx* ctx, int64_t step, int32_t keep_forces);
/* nsteps of Alg. 1's main loop; rebuild every rebuild_every */
int dpdb_step(dpdb_ctx* ctx, int64_t nsteps);
int dpdb_thermo_get(dpdb_ctx* ctx, dpdb_thermo* out);

/* Validation observables.
 * velocity_profile: nbins slabs of the box along bin_axis; each sample adds
 * every particle's vel_axis velocity (2^-24 fixed point, bitwise reproducible)
 * and a count to its slab.  get returns per-slab velocity sums and counts
 * accumulated over nsamples samples (mean = sum / count; the double-Poiseuille
 * fold and the viscosity fit are host-side, paper_1311_0402_b200.observables). */
int dpdb_profile_reset(dpdb_ctx* ctx, uint32_t nbins, int32_t bin_axis, int32_t vel_axis);
int dpdb_profile_sample(dpdb_ctx* ctx);
int dpdb_profile_get(dpdb_ctx* ctx, double* sum_v, uint64_t* count, int64_t* nsamples);
/* histogram of pair distances r < rmax <= r_c + skin over the current neighbor
 * table, every pair once, fp32 distance of the builder (RDF numerator) */
int dpdb_rdf(dpdb_ctx* ctx, uint32_t nbins, double rmax, uint64_t* hist);
/* Runs nsteps like dpdb_step and records the thermo line of every step
 * (out[0..nsteps-1]): the pass that applies a step's phase-2 kick also reduces
 * its kinetic partials on the device and writes the record into mapped pinned
 * host memory, so there is no host synchronisation per step.  kbt is the
 * COM-subtracted temperature of compute_temperature (src/core.cpp:141-149) in
 * one pass: (sum |v|^2 - |sum v|^2 / n) / (3 n); momentum = sum v. */
int dpdb_step_thermo(dpdb_ctx* ctx, int64_t nsteps, dpdb_thermo* out);
/* Runs nsteps like dpdb_step and returns the device time (CUDA events on the
 * context stream, ms).  stage_ms[0..5] (may be NULL): integrate, sort+permute,
 * build, force, other, total; stage_launches[0..5] likewise (kernel launches). */
int dpdb_step_timed(dpdb_ctx* ctx, int64_t nsteps, double* ms, double* stage_ms,
                    int64_t* stage_launches);
int64_t dpdb_current_step(const dpdb_ctx* ctx);
/* mean / max row length (core + skin) of the current table; mean_core too */
int dpdb_table_stats(dpdb_ctx* ctx, double* mean_row, double* mean_core, uint32_t* max_row);

/* --------------------------------------- device primitives (parity) */
enum {
    DPDB_OP_TEA_HASH = 1,      /* in0,in1 u32; param = rounds; out u32[2n] */
    DPDB_OP_SIGNATURE = 2,     /* in0 u32 tag; in1 f64[3n] v (xyz interleaved); out u32 */
    DPDB_OP_PAIR_UNIFORMS = 3, /* in0 u32[2n] sig, in1 u32[2n] tag; param = step_mix; out u32[2n] */
    DPDB_OP_GAUSSIAN64 = 4,    /* in0,in1 u32; out f64 */
    DPDB_OP_GAUSSIAN32 = 5,    /* in0,in1 u32; out f32 (hot-path variant) */
    DPDB_OP_FASTLOG = 6,       /* in0 u32; out f64 */
    DPDB_OP_FASTCOS2PI = 7,    /* in0 u32; out f64 */
    DPDB_OP_FASTPOW = 8,       /* in0,in1 f64; out f64 */
    DPDB_OP_MORTON = 9,        /* in0 u32[3n]; param = bits; out u32 */
    DPDB_OP_FASTLOG32 = 10,    /* in0 u32; out f32 */
    DPDB_OP_STEP_MIX = 11,     /* in0 u32 seed, in1 u32 step; out u32 */
    DPDB_OP_GAUSSIAN_HOT = 12  /* in0,in1 u32; out f32 (the force kernels' Box-Muller) */
};
int dpdb_eval(int device, int op, size_t n, const void* in0, const void* in1, uint32_t param,
              void* out);
/* stable LSD radix sort on the device (RadixSorter::sort contract): host
 * arrays in/out, bit_length multiple of 4 and <= 32 */
int dpdb_radix_sort(int device, uint32_t* keys, uint32_t* vals, size_t n, int bit_length);

/* ------------------------------------------- brick decomposition (§8e)
 * decompose / border_determination / exchange_ghosts / migrate_strays and
 * the GhostPacket wire records of the spec (paper Alg. 6,
 * P:316-331).  One context owns one brick: uniform half-open slabs of the
 * global box, locals at [0, n), ghosts at [n, n + ng).  Directions
 * d = 0..25 enumerate the neighbor offsets (dx, dy, dz) in z-major order
 * with the centre removed; the opposite of d is 25 - d.  Every exchange
 * buffer is DEVICE memory holding records in direction order; the transport
 * (in-process peer copies below, or NCCL between processes) delivers to
 * brick b, for each d, what the brick at b + d packed for direction 25 - d. */
#define DPDB_MD_MIGRANTS 0     /* full record: x, v (f64), tag, species | molecule << 8 */
#define DPDB_MD_GHOST_FULL 1   /* same record, x shifted by the periodic image */
#define DPDB_MD_GHOST_UPDATE 2 /* x (shifted), v only; receiver order fixed at rebuild */

/* decompose: the brick at `coords` of a dims[0]xdims[1]xdims[2] grid */
int dpdb_create_domain(int device, const dpdb_box* box, const dpdb_params* params,
                       const dpdb_run* run, const int32_t dims[3], const int32_t coords[3],
                       size_t capacity, dpdb_ctx** out);
int dpdb_domain_info(const dpdb_ctx* ctx, double slab_lo[3], double slab_hi[3], int32_t dims[3],
                     int32_t coords[3]);
/* coordinates of the neighbor brick in direction d; DPDB_ECONFIG if none */
int dpdb_md_neighbor(const dpdb_ctx* ctx, int dir, int32_t nb_coords[3]);
int dpdb_md_record_bytes(int what);
/* Per-brick protocol.  Setup: begin_setup, accept_migrants(NULL, NULL, gc),
 * exchange GHOST_FULL (gc), accept_ghosts, forces.  Rebuild step:
 * begin_rebuild(mc), exchange MIGRANTS (mc), accept_migrants(.., gc),
 * exchange GHOST_FULL (gc), accept_ghosts, forces.  Other steps: begin_step,
 * exchange GHOST_UPDATE (the counts of the last rebuild), accept_update,
 * forces.  finish applies the pending half-kick (end of the last step). */
int dpdb_md_begin_setup(dpdb_ctx* ctx);
int dpdb_md_begin_rebuild(dpdb_ctx* ctx, int32_t migrant_counts[26]);
int dpdb_md_pack(dpdb_ctx* ctx, int what, void* dev_out);
int dpdb_md_accept_migrants(dpdb_ctx* ctx, const void* dev_in, const int32_t counts[26],
                            int32_t ghost_counts[26]);
int dpdb_md_accept_ghosts(dpdb_ctx* ctx, const void* dev_in, const int32_t counts[26]);
int dpdb_md_begin_step(dpdb_ctx* ctx);
int dpdb_md_accept_update(dpdb_ctx* ctx, const void* dev_in, const int32_t counts[26]);
int dpdb_md_forces(dpdb_ctx* ctx);
int dpdb_md_finish(dpdb_ctx* ctx);
/* sum of v, v^2 over the locals (for a cross-brick temperature) */
int dpdb_md_sums(dpdb_ctx* ctx, double out[4]);
int dpdb_md_ghost_count(const dpdb_ctx* ctx, size_t* ng);
/* force blocks of the current table and how many of them are interior (no
 * ghost partner: their forces run while the ghost update is in flight) */
int dpdb_md_block_split(dpdb_ctx* ctx, size_t* n_blocks, size_t* n_interior);
/* the ghosts [n, n + ng) as this brick holds them (x shifted to its image) */
int dpdb_md_download_ghosts(dpdb_ctx* ctx, double* x, double* y, double* z, double* vx,
                            double* vy, double* vz, uint32_t* tag);
/* In-process transport: all bricks of a decomposition in one process (one
 * or several GPUs; cudaMemcpyPeerAsync over NVLink between GPUs). */
int dpdb_group_setup(dpdb_ctx* const* ctxs, int n_bricks);
int dpdb_group_step(dpdb_ctx* const* ctxs, int n_bricks, int64_t nsteps);
/* dpdb_group_step with every step's thermo line (combined over the bricks in
 * brick order; the per-brick sums are reduced on the devices by the pass that
 * applies each step's phase 2 and land in mapped pinned memory) */
int dpdb_group_step_thermo(dpdb_ctx* const* ctxs, int n_bricks, int64_t nsteps, dpdb_thermo* out);

/* NCCL transport: one brick per process (rank = coords[0] + dims[0] *
 * (coords[1] + dims[1] * coords[2])).  Rank 0 makes the id, the caller
 * broadcasts it (e.g. over torch.distributed), every rank attaches.  The step
 * then runs entirely on the brick's stream: pack -> grouped ncclSend/Recv per
 * neighbor direction -> unpack -> forces, no host sync between rebuilds
 * (a rebuild all-gathers 26 counts per rank).  NCCL is loaded at run time. */
#define DPDB_NCCL_ID_BYTES 128
int dpdb_nccl_unique_id(uint8_t id[DPDB_NCCL_ID_BYTES]);
int dpdb_nccl_attach(dpdb_ctx* ctx, const uint8_t id[DPDB_NCCL_ID_BYTES], int nranks, int rank);
/* TEST transport: attach the nranks bricks of ONE process (one host thread
 * per brick afterwards, each calling dpdb_dist_*) to an in-process stand-in
 * of NCCL's grouped Send / Recv and AllGather (device copies, NCCL's
 * per-peer ordering and completion semantics), so the NCCL driver's
 * multi-rank call sequence runs on a single GPU. */
int dpdb_nccl_mock_attach(dpdb_ctx* const* ctxs, int nranks);
int dpdb_dist_setup(dpdb_ctx* ctx);
int dpdb_dist_step(dpdb_ctx* ctx, int64_t nsteps);
/* dpdb_dist_step recording this brick's per-step sums: sums[5 s + 0..4] =
 * {step, sum v_x, sum v_y, sum v_z, sum |v|^2} over its locals (the caller adds
 * the ranks' records in rank order: kT = (S2 - |P|^2 / N) / (3 N)) */
int dpdb_dist_step_thermo(dpdb_ctx* ctx, int64_t nsteps, double* sums);
/* as dpdb_step_timed: device time (ms, CUDA events on the brick's stream),
 * stage_ms[0..5] = integrate, (unused), rebuild (migration + full halo + sort
 * + build), force, other (halo update), total; stage_launches likewise */
int dpdb_dist_step_timed(dpdb_ctx* ctx, int64_t nsteps, double* ms, double* stage_ms,
                         int64_t* stage_launches);
/* global thermo line: per-brick partial sums all-gathered, added in rank order */
int dpdb_dist_thermo(dpdb_ctx* ctx, dpdb_thermo* out);

#ifdef __cplusplus
}
#endif
#endif
