"""ctypes bindings for the CPU oracle (TEST INFRASTRUCTURE ONLY).

``liboracle.so`` is our C restatement of the reference hot path
(oracle/dpd_oracle.c).  ``_ref/libdpdref.so`` is the reference's own
shipped C++ compiled in place from /root/reference (oracle/Makefile); it is
optional -- absent on machines that never saw /root/reference.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg import this module.  The product package
paper_1311_0402_b200 never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libdpdref.so")

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class Box(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("periodic", C.c_int32 * 3), ("wall", C.c_int32 * 3)]


class Grid(C.Structure):
    _fields_ = [("ncell", C.c_int32 * 3), ("ncell_ext", C.c_int32 * 3),
                ("ghost_lo", C.c_int32 * 3), ("ghost_hi", C.c_int32 * 3),
                ("wrapmode", C.c_int32 * 3),
                ("cell_size", C.c_double * 3), ("inv_cell", C.c_double * 3),
                ("slab_lo", C.c_double * 3), ("slab_hi", C.c_double * 3),
                ("origin", C.c_double * 3),
                ("sub_bits", C.c_int32), ("bits_per_axis", C.c_int32),
                ("n_local_cells", C.c_uint32), ("n_total_cells", C.c_uint32),
                ("rank_of_cell", C.POINTER(C.c_uint32)),
                ("cell_of_rank", C.POINTER(C.c_uint32))]


class Params(C.Structure):
    _fields_ = [("n_species", C.c_int32), ("a", C.c_double * 16),
                ("gamma", C.c_double * 16), ("sigma", C.c_double * 16),
                ("s", C.c_double), ("r_c", C.c_double), ("kbt", C.c_double),
                ("dt", C.c_double)]


class Bond(C.Structure):
    _fields_ = [("tag_i", C.c_uint32), ("tag_j", C.c_uint32), ("k", C.c_double),
                ("r0", C.c_double)]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build():
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def use_native_build(workdir):
    """CPU-baseline build recipe: compile the oracle
    with -O3 -march=native -ffp-contract=off -fopenmp for THIS host into
    workdir and make it the library of this process.  Returns the path, or
    None (then the portable prebuilt liboracle.so stays in use)."""
    global _lib
    if _lib is not None:
        return None
    out = os.path.join(workdir, "liboracle_native.so")
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    try:
        subprocess.run([cc, "-O3", "-march=native", "-fPIC", "-std=c11", "-ffp-contract=off",
                        "-fopenmp", "-shared", "-o", out, os.path.join(HERE, "dpd_oracle.c"), "-lm"],
                       check=True, capture_output=True, timeout=120)
    except (OSError, subprocess.SubprocessError):
        return None
    L = C.CDLL(out)
    _declare(L)
    _lib = L
    return out


def ref():
    """The reference's own compiled code, or None when it was never built."""
    global _ref
    if _ref is None and os.path.exists(REF_PATH):
        R = C.CDLL(REF_PATH)
        _declare_ref(R)
        _ref = R
    return _ref


def _declare(L):
    d, u, i, sz = C.c_double, C.c_uint32, C.c_int, C.c_size_t
    sig = {
        "orc_last_error": (C.c_char_p, []),
        "orc_power2": (d, [i]), "orc_exp2_frac": (d, [d]), "orc_log2_frac": (d, [d]),
        "orc_fastlog": (d, [u]), "orc_fastcos2pi": (d, [u]), "orc_fastpow": (d, [d, d]),
        "orc_tea_hash": (None, [i, u, u, u32p]),
        "orc_bit_reverse": (u, [u]), "orc_mantissa11": (u, [d]),
        "orc_make_signature": (u, [u, d, d, d]), "orc_step_mix": (u, [u, u]),
        "orc_pair_uniforms": (None, [u, u, u, u, u, u32p]),
        "orc_gaussian": (d, [u, u]),
        "orc_signatures": (None, [sz, u32p, f64p, f64p, f64p, u32p]),
        "orc_morton_encode": (i, [u, u, u, i, C.POINTER(u)]),
        "orc_radix_sort": (i, [u32p, u32p, sz, i, i]),
        "orc_grid_make": (i, [C.POINTER(Box), f64p, f64p, C.POINTER(C.c_int32 * 3),
                              C.POINTER(C.c_int32 * 3), d, C.c_int32, C.POINTER(Grid)]),
        "orc_grid_free": (None, [C.POINTER(Grid)]),
        "orc_grid_key_bits": (i, [C.POINTER(Grid)]),
        "orc_sort_keys": (i, [C.POINTER(Grid), sz, f64p, f64p, f64p, u32p]),
        "orc_reorder_order": (i, [C.POINTER(Grid), sz, f64p, f64p, f64p, u32p, u32p, i]),
        "orc_local_cell_ranks": (i, [C.POINTER(Grid), sz, f64p, f64p, f64p, u32p]),
        "orc_build_cell_list": (i, [u, u32p, sz, u32p]),
        "orc_coarse_stencil": (i, [C.POINTER(Grid), u32p, u32p]),
        "orc_fine_stencil": (i, [u, u32p, u32p, u32p, u32p, C.c_void_p]),
        "orc_build_neighbor_table": (i, [C.POINTER(Grid), C.POINTER(Box), u32p, u32p, u32p,
                                         sz, sz, f64p, f64p, f64p, u32p, d, d, u,
                                         u32p, u16p, u16p, i]),
        "orc_join_core_skin": (None, [u, u, i, u32p, u16p, u16p]),
        "orc_table_diff": (C.c_int64, [u, u, i, i, u32p, u16p, u16p, i, i, u32p, u16p, u16p, i]),
        "orc_tile_transpose": (None, [u, u, u32p]),
        "orc_params_make": (i, [C.c_int32, f64p, f64p, d, d, d, d, C.POINTER(Params)]),
        "orc_compute_forces": (i, [C.POINTER(Params), C.POINTER(Box), sz,
                                   f64p, f64p, f64p, f64p, f64p, f64p, u32p, C.c_void_p,
                                   u32p, u, u, i, i, u32p, u16p, u16p, f64p, f64p, f64p, i]),
        "orc_pair_force": (i, [C.POINTER(Params), C.c_uint8, C.c_uint8, f64p, f64p, d, f64p]),
        "orc_body_force": (None, [d, sz, f64p, d, f64p]),
        "orc_bond_forces": (i, [C.POINTER(Box), sz, C.POINTER(Bond), sz, u32p, f64p, f64p, f64p,
                                f64p, f64p, f64p]),
        "orc_raw_index": (sz, [i, u, u, u]),
        "orc_verlet_phase1": (i, [C.POINTER(Box), d, sz, f64p, f64p, f64p, f64p, f64p, f64p,
                                  f64p, f64p, f64p, C.c_void_p]),
        "orc_verlet_phase2": (None, [d, sz, f64p, f64p, f64p, f64p, f64p, f64p]),
        "orc_compute_temperature": (i, [sz, f64p, f64p, f64p, C.POINTER(d)]),
        "orc_init_fluid": (i, [C.POINTER(Box), sz, d, u, f64p, f64p, f64p, f64p, f64p, f64p,
                               u32p]),
        "orc_sim_create": (C.c_void_p, [C.POINTER(Box), C.POINTER(Params), d, i, u, u, d, i, i,
                                        sz, f64p, f64p, f64p, f64p, f64p, f64p, u32p,
                                        C.c_void_p, i]),
        "orc_sim_destroy": (None, [C.c_void_p]),
        "orc_sim_run": (i, [C.c_void_p, C.c_int64]),
        "orc_sim_step_index": (C.c_int64, [C.c_void_p]),
        "orc_sim_n": (sz, [C.c_void_p]),
        "orc_sim_get": (None, [C.c_void_p] + [C.c_void_p] * 10),
        "orc_sim_temperature": (d, [C.c_void_p]),
        "orc_sim_set_reorder_hook": (i, [C.c_void_p, C.c_void_p, C.c_void_p]),
        "orc_sim_stage_seconds": (None, [C.c_void_p, np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS"), i]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _declare_ref(R):
    d, u, i, sz = C.c_double, C.c_uint32, C.c_int, C.c_size_t
    i32x3 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
    sig = {
        "ref_last_error": (C.c_char_p, []),
        "ref_tea_hash": (None, [i, u, u, u32p]),
        "ref_bit_reverse": (u, [u]),
        "ref_make_signature": (u, [u, d, d, d]),
        "ref_step_mix": (u, [u, u]),
        "ref_pair_uniforms": (None, [u, u, u, u, u, u, u32p]),
        "ref_gaussian": (d, [u, u]), "ref_fastlog": (d, [u]), "ref_fastcos2pi": (d, [u]),
        "ref_fastpow": (d, [d, d]), "ref_power2": (d, [i]), "ref_exp2_frac": (d, [d]),
        "ref_log2_frac": (d, [d]),
        "ref_morton_encode": (i, [u, u, u, i, C.POINTER(u)]),
        "ref_radix_sort": (i, [u32p, u32p, sz, i, C.c_uint]),
        "ref_grid_info": (i, [f64p, f64p, i32x3, d, i,
                              np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS"), f64p]),
        "ref_grid_ranks": (i, [f64p, f64p, i32x3, d, i, u32p]),
        "ref_reorder_cells": (i, [f64p, f64p, i32x3, d, i, C.c_uint, sz, f64p, f64p, f64p, u32p,
                                  u32p, u32p, u32p, u32p, u32p, C.c_void_p, sz]),
        "ref_build_cell_list": (i, [u, u32p, sz, u32p]),
        "ref_temperature": (d, [sz, f64p, f64p, f64p]),
        "ref_minimum_image": (None, [f64p, f64p, f64p, i32x3, f64p]),
        "ref_params_sigma": (i, [i, f64p, f64p, d, d, d, d, f64p]),
        "ref_sim_ctx_create": (C.c_void_p, [f64p, f64p, i32x3, d, i, C.c_uint]),
        "ref_sim_ctx_destroy": (None, [C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(R, name)
        f.restype = res
        f.argtypes = args


def check(rc, L=None):
    if rc:
        L = L or lib()
        raise OracleError(rc, L.orc_last_error().decode())


# ---------------------------------------------------------------- helpers
def make_box(lo, hi, periodic=(1, 1, 1), wall=(0, 0, 0)):
    b = Box()
    for k in range(3):
        b.lo[k] = lo[k]
        b.hi[k] = hi[k]
        b.periodic[k] = int(periodic[k])
        b.wall[k] = int(wall[k])
    return b


class OGrid:
    """Single-domain (or slab) cell grid owned by the oracle."""

    def __init__(self, box, cell_target, sub_bits=2, slab_lo=None, slab_hi=None,
                 dims=(1, 1, 1), coords=(0, 0, 0)):
        L = lib()
        self.box = box
        self.g = Grid()
        lo = np.array(slab_lo if slab_lo is not None else list(box.lo), dtype=np.float64)
        hi = np.array(slab_hi if slab_hi is not None else list(box.hi), dtype=np.float64)
        d3 = (C.c_int32 * 3)(*dims)
        c3 = (C.c_int32 * 3)(*coords)
        check(L.orc_grid_make(C.byref(box), lo, hi, C.byref(d3), C.byref(c3), cell_target,
                              sub_bits, C.byref(self.g)))
        self.nlc = self.g.n_local_cells
        self.ntc = self.g.n_total_cells

    def __del__(self):
        try:
            lib().orc_grid_free(C.byref(self.g))
        except Exception:
            pass

    def key_bits(self):
        return lib().orc_grid_key_bits(C.byref(self.g))

    def rank_of_cell(self):
        return np.ctypeslib.as_array(self.g.rank_of_cell, shape=(self.ntc,)).copy()

    def keys(self, x, y, z):
        out = np.zeros(len(x), np.uint32)
        check(lib().orc_sort_keys(C.byref(self.g), len(x), x, y, z, out))
        return out

    def order(self, x, y, z, nthreads=1):
        n = len(x)
        order = np.zeros(n, np.uint32)
        perm = np.zeros(n, np.uint32)
        check(lib().orc_reorder_order(C.byref(self.g), n, x, y, z, order, perm, nthreads))
        return order, perm

    def cell_start(self, x, y, z):
        n = len(x)
        ranks = np.zeros(n, np.uint32)
        check(lib().orc_local_cell_ranks(C.byref(self.g), n, x, y, z, ranks))
        cs = np.zeros(self.ntc + 1, np.uint32)
        check(lib().orc_build_cell_list(self.ntc, ranks, n, cs))
        return cs

    def coarse(self):
        off = np.zeros(self.nlc + 1, np.uint32)
        cells = np.zeros(self.nlc * 27 + 1, np.uint32)
        check(lib().orc_coarse_stencil(C.byref(self.g), off, cells))
        return off, cells[: off[-1]].copy()

    def fine(self, coff, ccells, cs):
        foff = np.zeros(self.nlc + 1, np.uint32)
        lib().orc_fine_stencil(self.nlc, coff, np.ascontiguousarray(ccells, np.uint32), cs, foff,
                               None)
        fidx = np.zeros(int(foff[-1]) + 1, np.uint32)
        lib().orc_fine_stencil(self.nlc, coff, np.ascontiguousarray(ccells, np.uint32), cs, foff,
                               fidx.ctypes.data)
        return foff, fidx[: foff[-1]].copy()

    def neighbor_table(self, x, y, z, tag, r_c, skin, maxn=128, cs=None, coarse=None,
                       n_local=None, nthreads=1):
        n_all = len(x)
        n_local = n_all if n_local is None else n_local
        if cs is None:
            cs = self.cell_start(x, y, z)
        coff, ccells = coarse if coarse is not None else self.coarse()
        n_pad = (n_local + 31) // 32 * 32
        entries = np.zeros(max(n_pad, 32) * maxn, np.uint32)
        core = np.zeros(max(n_pad, 1), np.uint16)
        skinc = np.zeros(max(n_pad, 1), np.uint16)
        check(lib().orc_build_neighbor_table(C.byref(self.g), C.byref(self.box), cs, coff,
                                             np.ascontiguousarray(ccells, np.uint32), n_local,
                                             n_all, x, y, z, tag, r_c, skin, maxn, entries, core,
                                             skinc, nthreads))
        return entries.reshape(-1, maxn), core, skinc


def table_diff(maxn, a, b, nthreads=8):
    """First row where two tables differ (counts or entries through the
    core_at / skin_at accessors), -1 when identical.  a, b: (tiled, joined,
    entries, core, skin)."""
    n = len(a[3])
    assert len(b[3]) >= n
    return int(lib().orc_table_diff(n, maxn, int(a[0]), int(a[1]),
                                    np.ascontiguousarray(a[2]).reshape(-1), a[3], a[4],
                                    int(b[0]), int(b[1]), np.ascontiguousarray(b[2]).reshape(-1),
                                    np.ascontiguousarray(b[3][:n]), np.ascontiguousarray(b[4][:n]),
                                    nthreads))


def make_params(a=25.0, gamma=4.5, kbt=1.0, s=1.0, r_c=1.0, dt=0.01, n_species=1):
    a = np.broadcast_to(np.asarray(a, np.float64), (n_species * n_species,)).copy()
    g = np.broadcast_to(np.asarray(gamma, np.float64), (n_species * n_species,)).copy()
    p = Params()
    check(lib().orc_params_make(n_species, a, g, kbt, s, r_c, dt, C.byref(p)))
    return p


def init_fluid(box, n, kbt=1.0, seed=1):
    x, y, z, vx, vy, vz = (np.zeros(n) for _ in range(6))
    tag = np.zeros(n, np.uint32)
    check(lib().orc_init_fluid(C.byref(box), n, kbt, seed, x, y, z, vx, vy, vz, tag))
    return x, y, z, vx, vy, vz, tag


def signatures(tag, vx, vy, vz):
    out = np.zeros(len(tag), np.uint32)
    lib().orc_signatures(len(tag), tag, vx, vy, vz, out)
    return out


def compute_forces(params, box, x, y, z, vx, vy, vz, tag, sig, step_mix, entries, core, skinc,
                   maxn, tiled=False, joined=False, species=None, nthreads=1):
    n = len(core) if len(core) < len(x) else len(x)
    n = min(n, len(x))
    fx, fy, fz = np.zeros(n), np.zeros(n), np.zeros(n)
    sp = None if species is None else species.ctypes.data
    check(lib().orc_compute_forces(C.byref(params), C.byref(box), n, x, y, z, vx, vy, vz, tag,
                                   sp, sig, step_mix, maxn, int(tiled), int(joined),
                                   np.ascontiguousarray(entries).reshape(-1), core, skinc,
                                   fx, fy, fz, nthreads))
    return fx, fy, fz


class Sim:
    """Whole-step CPU driver (Alg. 1) -- the CPU baseline and trajectory oracle."""

    def __init__(self, box, params, state, skin=0.3, rebuild_every=10, maxn=128, seed=1,
                 body_force=0.0, drive_axis=2, partition_axis=0, species=None, nthreads=1):
        x, y, z, vx, vy, vz, tag = state
        L = lib()
        sp = None if species is None else np.ascontiguousarray(species, np.uint8).ctypes.data
        self._keep = (box, params)
        self.h = L.orc_sim_create(C.byref(box), C.byref(params), skin, rebuild_every, maxn, seed,
                                  body_force, drive_axis, partition_axis, len(x), x, y, z, vx, vy,
                                  vz, tag, sp, nthreads)
        if not self.h:
            raise OracleError(-1, L.orc_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_sim_destroy(self.h)
            self.h = None
        if getattr(self, "_refctx", None):
            ref().ref_sim_ctx_destroy(self._refctx)
            self._refctx = None

    def run(self, nsteps):
        check(lib().orc_sim_run(self.h, nsteps))

    @property
    def step(self):
        return lib().orc_sim_step_index(self.h)

    def state(self):
        n = lib().orc_sim_n(self.h)
        arrs = [np.zeros(n) for _ in range(9)]
        tag = np.zeros(n, np.uint32)
        lib().orc_sim_get(self.h, *[a.ctypes.data for a in arrs], tag.ctypes.data)
        return dict(x=arrs[0], y=arrs[1], z=arrs[2], vx=arrs[3], vy=arrs[4], vz=arrs[5],
                    fx=arrs[6], fy=arrs[7], fz=arrs[8], tag=tag)

    def temperature(self):
        return lib().orc_sim_temperature(self.h)

    def use_reference_reorder(self, box, cell_target=1.3, workers=1):
        """Run the reorder step with the reference's own shipped
        reorder_particles + RadixSorter + cell list (oracle/_ref); False when
        the reference build is absent."""
        R = ref()
        if R is None:
            return False
        lo = np.array(list(box.lo), np.float64)
        hi = np.array(list(box.hi), np.float64)
        per = np.array(list(box.periodic), np.int32)
        self._refctx = R.ref_sim_ctx_create(lo, hi, per, cell_target, 2, workers)
        if not self._refctx:
            return False
        fn = C.cast(R.ref_sim_reorder, C.c_void_p)
        check(lib().orc_sim_set_reorder_hook(self.h, fn, self._refctx))
        return True

    def stage_seconds(self, reset=True):
        """(integrate, reorder, build, forces) wall seconds since the last reset"""
        out = np.zeros(4)
        lib().orc_sim_stage_seconds(self.h, out, int(reset))
        return out
