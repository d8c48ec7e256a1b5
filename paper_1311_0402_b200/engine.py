"""Host-side mirror of the reference's C++ simulation API over libdpdb.so.

Names, argument meaning and error behaviour follow the reference headers so
the parity tests read like the reference's own (missing) tests:

    SimBox, ParticleStore, PairParams, RunConfig   inc/core.hpp:15-109
    NeighborTable (raw_index/core_at/skin_at)      inc/neighbor_table.hpp:18-40
    radix_sort                                     inc/radix_sort.hpp:15-17
    tea_hash/make_signature/pair_uniforms/gaussian inc/rng.hpp:25-91
    fastlog/fastcos2pi/fastpow                     inc/fastmath.hpp:108-151
    Engine.reorder_particles/build_cell_list/...   inc/cell_grid.hpp:72-83 etc.

Every call runs the hand-written sm_100a kernels; errors raise DPDError
carrying the reference ErrorCategory code.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import OP, Box, DPDError, GridInfo, Params, Run, Thermo, check, lib, ptr


# ------------------------------------------------------------------ types
@dataclass
class SimBox:
    """inc/core.hpp:15-25."""
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)
    periodic: tuple = (True, True, True)
    wall: tuple = (False, False, False)

    def length(self, k):
        return self.hi[k] - self.lo[k]

    def volume(self):
        return self.length(0) * self.length(1) * self.length(2)

    def _c(self):
        b = Box()
        for k in range(3):
            b.lo[k], b.hi[k] = self.lo[k], self.hi[k]
            b.periodic[k], b.wall[k] = int(self.periodic[k]), int(self.wall[k])
        return b


@dataclass
class PairParams:
    """inc/core.hpp:51-68; sigma derived so sigma^2 = 2 gamma kbt (src/core.cpp:77-102)."""
    n_species: int = 1
    a: np.ndarray = field(default_factory=lambda: np.array([25.0]))
    gamma: np.ndarray = field(default_factory=lambda: np.array([4.5]))
    s: float = 1.0
    r_c: float = 1.0
    kbt: float = 1.0
    dt: float = 0.01

    @staticmethod
    def make(n_species, a, gamma, kbt, s, r_c, dt):
        a = np.broadcast_to(np.asarray(a, np.float64), (n_species * n_species,)).copy()
        g = np.broadcast_to(np.asarray(gamma, np.float64), (n_species * n_species,)).copy()
        if r_c <= 0:
            raise DPDError(1, "pair params: r_c must be positive")
        if s <= 0:
            raise DPDError(1, "pair params: weight exponent s must be positive")
        A, G = a.reshape(n_species, n_species), g.reshape(n_species, n_species)
        if not (np.array_equal(A, A.T) and np.array_equal(G, G.T)):
            raise DPDError(1, "pair params: matrices must be symmetric")
        return PairParams(n_species, a, g, s, r_c, kbt, dt)

    @property
    def sigma(self):
        return np.sqrt(2.0 * self.gamma * self.kbt)

    def _c(self):
        p = Params()
        p.n_species = self.n_species
        for q in range(self.n_species ** 2):
            p.a[q], p.gamma[q] = float(self.a[q]), float(self.gamma[q])
        p.kbt, p.s, p.r_c, p.dt = self.kbt, self.s, self.r_c, self.dt
        return p


@dataclass
class RunConfig:
    """inc/core.hpp:83-109 (hot-path subset)."""
    rebuild_every: int = 10
    skin: float = 0.3
    body_force: float = 0.0
    drive_axis: int = 2
    partition_axis: int = 0
    seed: int = 1
    max_neighbors: int = 128
    sub_bits: int = 2
    wall_mode: int = 0  # 0 specular (default), 1 bounce-back (S:525 design switch)

    def _c(self):
        r = Run()
        r.rebuild_every, r.skin, r.body_force = self.rebuild_every, self.skin, self.body_force
        r.drive_axis, r.partition_axis, r.seed = self.drive_axis, self.partition_axis, self.seed
        r.max_neighbors, r.sub_bits = self.max_neighbors, self.sub_bits
        r.wall_mode = self.wall_mode
        return r


@dataclass
class ParticleStore:
    """SoA particle storage, inc/core.hpp:29-47."""
    coord: list
    veloc: list
    tag: np.ndarray
    species: np.ndarray | None = None
    molecule: np.ndarray | None = None
    force: list | None = None
    signature: np.ndarray | None = None

    @property
    def n(self):
        return len(self.tag)

    @staticmethod
    def from_arrays(x, y, z, vx, vy, vz, tag, species=None, molecule=None):
        f = lambda a: np.ascontiguousarray(a, np.float64)
        return ParticleStore([f(x), f(y), f(z)], [f(vx), f(vy), f(vz)],
                             np.ascontiguousarray(tag, np.uint32),
                             None if species is None else np.ascontiguousarray(species, np.uint8),
                             None if molecule is None else np.ascontiguousarray(molecule, np.uint32))


@dataclass
class NeighborTable:
    """inc/neighbor_table.hpp:18-40 (host copy of the device table)."""
    n_rows: int
    max_neighbors: int
    n_rows_pad: int
    tiled: bool
    joined: bool
    entries: np.ndarray
    core_count: np.ndarray
    skin_count: np.ndarray

    def raw_index(self, i, k):
        m = self.max_neighbors
        if not self.tiled:
            return i * m + k
        return ((i & ~31) + (k & 31)) * m + (k & ~31) + (i & 31)

    def entry(self, i, k):
        return int(self.entries[self.raw_index(i, k)])

    def core_at(self, i, k):
        return self.entry(i, k)

    def skin_at(self, i, k):
        if self.joined:
            return self.entry(i, int(self.core_count[i]) + k)
        return self.entry(i, self.max_neighbors - 1 - k)

    def core_row(self, i):
        k = np.arange(int(self.core_count[i]))
        return self.entries[self.raw_index(i, k)]

    def skin_row(self, i):
        """skin entries ascending"""
        s = np.arange(int(self.skin_count[i]))
        k = (int(self.core_count[i]) + s) if self.joined else (self.max_neighbors - 1 - s)
        return self.entries[self.raw_index(i, k)]

    def rows(self):
        """Logical rows as (core ascending, skin ascending) arrays (vectorised)."""
        m = self.max_neighbors
        E = self.entries.reshape(self.n_rows_pad, m)
        if self.tiled:  # undo the 32x32 tile transpose
            E = E.reshape(self.n_rows_pad // 32, 32, m // 32, 32).transpose(0, 3, 2, 1)
            E = E.reshape(self.n_rows_pad, m)
        return E


# ---------------------------------------------------------------- engine
class Engine:
    """One device context: the B200 side of a domain (ParticleStore + grid +
    neighbor table + forces) driven through the C ABI."""

    def __init__(self, box: SimBox, params: PairParams, run: RunConfig | None = None,
                 capacity: int = 1, device: int = 0, dims=None, coords=None):
        self.box, self.params, self.run = box, params, run or RunConfig()
        self.device = device
        L = lib()
        h = C.c_void_p()
        self._cb, self._cp, self._cr = box._c(), params._c(), self.run._c()
        if dims is None:
            check(L.dpdb_create(device, C.byref(self._cb), C.byref(self._cp), C.byref(self._cr),
                                int(capacity), C.byref(h)))
        else:  # one brick of a decomposition
            d = np.ascontiguousarray(dims, np.int32)
            c = np.ascontiguousarray(coords, np.int32)
            check(L.dpdb_create_domain(device, C.byref(self._cb), C.byref(self._cp),
                                       C.byref(self._cr), ptr(d), ptr(c), int(capacity),
                                       C.byref(h)))
        self.dims = tuple(int(v) for v in (dims if dims is not None else (1, 1, 1)))
        self.coords = tuple(int(v) for v in (coords if coords is not None else (0, 0, 0)))
        self.h = h.value
        gi = GridInfo()
        check(L.dpdb_grid(self.h, C.byref(gi)), self.h)
        self.grid = gi
        self.n_local_cells = gi.n_local_cells
        self.n_total_cells = gi.n_total_cells
        self.capacity = int(capacity)

    def close(self):
        if getattr(self, "h", None):
            lib().dpdb_destroy(self.h)
            self.h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc):
        check(rc, self.h)

    # ---------------------------------------------------------- state
    @property
    def n(self):
        n = C.c_size_t()
        self._check(lib().dpdb_size(self.h, C.byref(n)))
        return n.value

    def upload(self, store: ParticleStore):
        self._keep = store
        self._check(lib().dpdb_upload(self.h, store.n, *[ptr(a) for a in store.coord],
                                      *[ptr(a) for a in store.veloc], ptr(store.tag),
                                      ptr(store.species), ptr(store.molecule)))

    def init_random(self, n: int, kbt: float = 1.0, seed: int = 1, n_chains: int = 0,
                    chain_species=(), solvent_species: int = 0, r0: float = 0.38,
                    bond_k: float = 80.0):
        """init_random on the device: uniform positions,
        Maxwell-Boltzmann velocities with zero net momentum, optional chains
        (random walks with step r0, harmonic bonds k, r0) ahead of the solvent."""
        cs = np.ascontiguousarray(np.asarray(chain_species, np.uint8))
        self._keep = None
        self._check(lib().dpdb_init_random(self.h, int(n), float(kbt), int(seed), int(n_chains),
                                           int(len(cs)), ptr(cs) if len(cs) else None,
                                           int(solvent_species), float(r0), float(bond_k)))

    def upload_forces(self, fx, fy, fz):
        f = [np.ascontiguousarray(a, np.float64) for a in (fx, fy, fz)]
        self._check(lib().dpdb_upload_forces(self.h, *[ptr(a) for a in f]))

    def download(self) -> ParticleStore:
        n = self.n
        a = [np.zeros(n) for _ in range(9)]
        tag = np.zeros(n, np.uint32)
        sp = np.zeros(n, np.uint8)
        sig = np.zeros(n, np.uint32)
        self._check(lib().dpdb_download(self.h, *[ptr(x) for x in a], ptr(tag), ptr(sp), ptr(sig)))
        return ParticleStore(a[0:3], a[3:6], tag, sp, None, a[6:9], sig)

    def download_state(self, coord, veloc):
        """Positions and velocities into caller-owned float64 arrays (e.g.
        pinned buffers: no staging copy); the other fields are skipped."""
        arrs = list(coord) + list(veloc)
        for a in arrs:
            if a.dtype != np.float64 or not a.flags.c_contiguous or len(a) < self.n:
                raise ValueError("download_state: contiguous float64 arrays of length >= n")
        self._check(lib().dpdb_download(self.h, *[ptr(x) for x in arrs], None, None, None,
                                        None, None, None))

    BOND_HARMONIC, BOND_FENE = 0, 1

    def set_bonds(self, tag_i, tag_j, k, r0, style=None):
        """Bond topology (inc/core.hpp:70-79).  style per bond: 0 harmonic
        (default), 1 FENE with R0 in r0 (unpinned)."""
        ti, tj = (np.ascontiguousarray(t, np.uint32) for t in (tag_i, tag_j))
        kk, rr = (np.ascontiguousarray(np.broadcast_to(np.asarray(v, np.float64), ti.shape))
                  for v in (k, r0))
        if style is None:
            self._check(lib().dpdb_set_bonds(self.h, len(ti), ptr(ti), ptr(tj), ptr(kk), ptr(rr)))
        else:
            st = np.ascontiguousarray(np.broadcast_to(np.asarray(style, np.uint8), ti.shape))
            self._check(lib().dpdb_set_bonds_styled(self.h, len(ti), ptr(ti), ptr(tj), ptr(kk), ptr(rr),
                                                    ptr(st)))

    def set_angles(self, tag_a, tag_b, tag_c, k, theta0):
        """Harmonic angles U = K (theta - theta0)^2 / 2 around the middle tag_b
        (unpinned: no reference implementation)."""
        ta, tb, tc = (np.ascontiguousarray(t, np.uint32) for t in (tag_a, tag_b, tag_c))
        kk, t0 = (np.ascontiguousarray(np.broadcast_to(np.asarray(v, np.float64), ta.shape))
                  for v in (k, theta0))
        self._check(lib().dpdb_set_angles(self.h, len(ta), ptr(ta), ptr(tb), ptr(tc), ptr(kk), ptr(t0)))

    # -------------------------------------------------- stage entry points
    def sort_keys(self):
        out = np.zeros(self.n, np.uint32)
        self._check(lib().dpdb_sort_keys(self.h, ptr(out)))
        return out

    def reorder_particles(self):
        """src/cell_grid.cpp:166-198 + cell list; returns perm old -> new."""
        perm = np.zeros(self.n, np.uint32)
        self._check(lib().dpdb_reorder(self.h, ptr(perm)))
        return perm

    def cell_start(self):
        out = np.zeros(self.n_total_cells + 1, np.uint32)
        self._check(lib().dpdb_cell_start(self.h, ptr(out)))
        return out

    def rank_of_cell(self):
        out = np.zeros(self.n_total_cells, np.uint32)
        self._check(lib().dpdb_grid_ranks(self.h, ptr(out)))
        return out

    def coarse_stencil(self):
        off = np.zeros(self.n_local_cells + 1, np.uint32)
        self._check(lib().dpdb_coarse_stencil(self.h, ptr(off), None))
        cells = np.zeros(max(int(off[-1]), 1), np.uint32)
        self._check(lib().dpdb_coarse_stencil(self.h, ptr(off), ptr(cells)))
        return off, cells[: off[-1]]

    def fine_stencil(self):
        off = np.zeros(self.n_local_cells + 1, np.uint32)
        self._check(lib().dpdb_fine_stencil(self.h, ptr(off), None))
        idx = np.zeros(max(int(off[-1]), 1), np.uint32)
        self._check(lib().dpdb_fine_stencil(self.h, ptr(off), ptr(idx)))
        return off, idx[: off[-1]]

    def build_neighbor_table(self):
        self._check(lib().dpdb_build_neighbors(self.h))

    def join_core_skin(self):
        self._check(lib().dpdb_join_core_skin(self.h))

    def tile_transpose(self):
        self._check(lib().dpdb_tile_transpose(self.h))

    def neighbor_table(self) -> NeighborTable:
        n = self.n
        pad = (n + 31) // 32 * 32
        m = self.run.max_neighbors
        ent = np.zeros(max(pad, 32) * m, np.uint32)
        core = np.zeros(max(n, 1), np.uint16)
        skin = np.zeros(max(n, 1), np.uint16)
        tl, jn = C.c_int32(), C.c_int32()
        self._check(lib().dpdb_get_neighbors(self.h, ptr(ent), ptr(core), ptr(skin),
                                             C.addressof(tl), C.addressof(jn)))
        return NeighborTable(n, m, pad, bool(tl.value), bool(jn.value), ent[: pad * m], core[:n],
                             skin[:n])

    def signatures(self):
        out = np.zeros(self.n, np.uint32)
        self._check(lib().dpdb_signatures(self.h, ptr(out)))
        return out

    def compute_forces(self, step: int):
        self._check(lib().dpdb_compute_forces(self.h, int(step)))
        s = self.download()
        return s.force

    def verlet_phase1(self):
        self._check(lib().dpdb_verlet_phase1(self.h))

    def verlet_phase2(self):
        self._check(lib().dpdb_verlet_phase2(self.h))

    # --------------------------------------------------- device-resident run
    def setup(self):
        self._check(lib().dpdb_setup(self.h))

    def setup_at(self, step: int, keep_forces: bool = False):
        """Restart entry: setup with the step counter at `step`;
        keep_forces keeps forces uploaded with upload_forces (restart state)."""
        self._check(lib().dpdb_setup_at(self.h, int(step), int(bool(keep_forces))))

    def step(self, nsteps: int = 1):
        self._check(lib().dpdb_step(self.h, int(nsteps)))

    def step_thermo(self, nsteps: int):
        """dpdb_step_thermo: run nsteps and return every step's thermo line as
        arrays (step, kbt, momentum[n, 3]); the records are reduced on the
        device and land in pinned host memory without a per-step sync."""
        recs = (Thermo * max(int(nsteps), 1))()
        self._check(lib().dpdb_step_thermo(self.h, int(nsteps), recs))
        k = int(nsteps)
        return dict(step=np.array([recs[i].step for i in range(k)], np.int64),
                    kbt=np.array([recs[i].kbt for i in range(k)]),
                    momentum=np.array([tuple(recs[i].momentum) for i in range(k)]).reshape(k, 3))

    # ------------------------------------------- validation observables
    def profile_reset(self, nbins: int = 50, bin_axis: int = 2, vel_axis: int = 0):
        """velocity_profile: start accumulating slab averages."""
        self._check(lib().dpdb_profile_reset(self.h, int(nbins), int(bin_axis), int(vel_axis)))
        self._prof_nbins = int(nbins)

    def profile_sample(self):
        self._check(lib().dpdb_profile_sample(self.h))

    def profile(self):
        """(sum of velocities, counts, samples) per slab since profile_reset."""
        nb = self._prof_nbins
        sv, cnt, ns = np.zeros(nb), np.zeros(nb, np.uint64), C.c_int64()
        self._check(lib().dpdb_profile_get(self.h, ptr(sv), ptr(cnt), C.byref(ns)))
        return sv, cnt, ns.value

    def rdf_counts(self, nbins: int, rmax: float):
        """Pair-distance histogram (every pair once) of the current table."""
        h = np.zeros(int(nbins), np.uint64)
        self._check(lib().dpdb_rdf(self.h, int(nbins), float(rmax), ptr(h)))
        return h

    def step_timed(self, nsteps: int, stages: bool = False):
        ms = C.c_double()
        st = np.zeros(6) if stages else None
        ln = np.zeros(6, np.int64)
        self._check(lib().dpdb_step_timed(self.h, int(nsteps), C.byref(ms), ptr(st), ptr(ln)))
        return ms.value, st, ln

    def table_stats(self):
        m, mc, mx = C.c_double(), C.c_double(), C.c_uint32()
        self._check(lib().dpdb_table_stats(self.h, C.byref(m), C.byref(mc), C.byref(mx)))
        return dict(mean_row=m.value, mean_core=mc.value, max_row=mx.value)

    @property
    def current_step(self):
        return lib().dpdb_current_step(self.h)

    def thermo(self):
        t = Thermo()
        self._check(lib().dpdb_thermo_get(self.h, C.byref(t)))
        return dict(step=t.step, n=t.n, kbt=t.kbt, momentum=tuple(t.momentum))


# ----------------------------------------------------- device primitives
def _eval(op, n, in0, in1, param, out, device=0):
    check(lib().dpdb_eval(device, OP[op], n, ptr(in0), ptr(in1), int(param), ptr(out)))
    return out


def tea_hash(rounds, v0, v1, device=0):
    v0, v1 = (np.ascontiguousarray(np.atleast_1d(v), np.uint32) for v in (v0, v1))
    out = np.zeros(2 * len(v0), np.uint32)
    return _eval("TEA_HASH", len(v0), v0, v1, rounds, out, device).reshape(-1, 2)


def make_signature(tag, velocity, device=0):
    tag = np.ascontiguousarray(np.atleast_1d(tag), np.uint32)
    v = np.ascontiguousarray(np.asarray(velocity, np.float64).reshape(-1, 3))
    return _eval("SIGNATURE", len(tag), tag, v, 0, np.zeros(len(tag), np.uint32), device)


def step_mix(seed, step, device=0):
    s, t = (np.ascontiguousarray(np.atleast_1d(v), np.uint32) for v in (seed, step))
    s, t = np.broadcast_arrays(s, t)
    s, t = np.ascontiguousarray(s), np.ascontiguousarray(t)
    return _eval("STEP_MIX", len(s), s, t, 0, np.zeros(len(s), np.uint32), device)


def pair_uniforms(sig_i, sig_j, tag_i, tag_j, mix, device=0):
    sig = np.ascontiguousarray(np.stack([np.atleast_1d(sig_i), np.atleast_1d(sig_j)], 1), np.uint32)
    tag = np.ascontiguousarray(np.stack([np.atleast_1d(tag_i), np.atleast_1d(tag_j)], 1), np.uint32)
    out = np.zeros(2 * len(sig), np.uint32)
    return _eval("PAIR_UNIFORMS", len(sig), sig, tag, mix, out, device).reshape(-1, 2)


def gaussian(ua, ub, device=0, fp32=False, hot=False):
    """xi from two TEA words: fp64 bit-exact (inc/rng.hpp:88-91), or fp32
    (fp32=True: gaussian32; hot=True: the force kernels' ftz-intrinsic form)."""
    ua, ub = (np.ascontiguousarray(np.atleast_1d(v), np.uint32) for v in (ua, ub))
    if hot:
        return _eval("GAUSSIAN_HOT", len(ua), ua, ub, 0, np.zeros(len(ua), np.float32), device)
    if fp32:
        return _eval("GAUSSIAN32", len(ua), ua, ub, 0, np.zeros(len(ua), np.float32), device)
    return _eval("GAUSSIAN64", len(ua), ua, ub, 0, np.zeros(len(ua)), device)


def fastlog(v, device=0, fp32=False):
    v = np.ascontiguousarray(np.atleast_1d(v), np.uint32)
    if fp32:
        return _eval("FASTLOG32", len(v), v, None, 0, np.zeros(len(v), np.float32), device)
    return _eval("FASTLOG", len(v), v, None, 0, np.zeros(len(v)), device)


def fastcos2pi(v, device=0):
    v = np.ascontiguousarray(np.atleast_1d(v), np.uint32)
    return _eval("FASTCOS2PI", len(v), v, None, 0, np.zeros(len(v)), device)


def fastpow(a, b, device=0):
    a, b = (np.ascontiguousarray(np.atleast_1d(v), np.float64) for v in (a, b))
    return _eval("FASTPOW", len(a), a, b, 0, np.zeros(len(a)), device)


def morton_encode(ix, iy, iz, bits_per_axis, device=0):
    if bits_per_axis < 0 or 3 * bits_per_axis > 32:
        raise DPDError(1, "morton: 3*bits_per_axis must be <= 32")
    c = np.ascontiguousarray(np.stack([np.atleast_1d(ix), np.atleast_1d(iy), np.atleast_1d(iz)], 1),
                             np.uint32)
    lim = (1 << bits_per_axis) - 1
    if (c > lim).any():
        raise DPDError(1, "morton: lattice coordinate out of range")
    return _eval("MORTON", len(c), c, None, bits_per_axis, np.zeros(len(c), np.uint32), device)


def radix_sort(keys, values, bit_length, device=0):
    """RadixSorter::sort contract (inc/radix_sort.hpp:11-27), on the device, in place."""
    if keys.dtype != np.uint32 or values.dtype != np.uint32:
        raise TypeError("radix_sort: uint32 keys/values")
    if len(keys) != len(values):
        raise DPDError(1, "radix sort: keys/values length mismatch")
    check(lib().dpdb_radix_sort(device, ptr(keys), ptr(values), len(keys), int(bit_length)))
    return keys, values


def device_count():
    return lib().dpdb_device_count()
