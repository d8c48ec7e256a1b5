"""ctypes binding of libdpdb.so (include/dpdb.h).

Fails loudly when the CUDA library is missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdpdb.so")


class DPDError(RuntimeError):
    """Error with the reference's ErrorCategory code (inc/error.hpp:8-13)."""

    CATEGORY = {1: "config", 2: "physics", 3: "protocol", 4: "io", 5: "device"}

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{self.CATEGORY.get(code, code)}] {msg}")
        self.code = code
        self.category = self.CATEGORY.get(code, str(code))


class Box(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("periodic", C.c_int32 * 3), ("wall", C.c_int32 * 3)]


class Params(C.Structure):
    _fields_ = [("n_species", C.c_int32), ("a", C.c_double * 16), ("gamma", C.c_double * 16),
                ("kbt", C.c_double), ("s", C.c_double), ("r_c", C.c_double), ("dt", C.c_double)]


class Run(C.Structure):
    _fields_ = [("rebuild_every", C.c_int32), ("skin", C.c_double), ("body_force", C.c_double),
                ("drive_axis", C.c_int32), ("partition_axis", C.c_int32), ("seed", C.c_uint32),
                ("max_neighbors", C.c_uint32), ("sub_bits", C.c_int32), ("wall_mode", C.c_int32)]


class Thermo(C.Structure):
    _fields_ = [("step", C.c_int64), ("n", C.c_uint64), ("kbt", C.c_double),
                ("momentum", C.c_double * 3)]


class GridInfo(C.Structure):
    _fields_ = [("ncell", C.c_int32 * 3), ("ncell_ext", C.c_int32 * 3), ("wrapmode", C.c_int32 * 3),
                ("bits_per_axis", C.c_int32), ("key_bits", C.c_int32),
                ("n_local_cells", C.c_uint32), ("n_total_cells", C.c_uint32),
                ("cell_size", C.c_double * 3), ("inv_cell", C.c_double * 3),
                ("origin", C.c_double * 3)]


OP = dict(TEA_HASH=1, SIGNATURE=2, PAIR_UNIFORMS=3, GAUSSIAN64=4, GAUSSIAN32=5, FASTLOG=6,
          FASTCOS2PI=7, FASTPOW=8, MORTON=9, FASTLOG32=10, STEP_MIX=11, GAUSSIAN_HOT=12)

# every symbol include/dpdb.h declares (checked by tests/test_abi.py)
SYMBOLS = {
    "dpdb_version": (C.c_char_p, []),
    "dpdb_last_error": (C.c_char_p, [C.c_void_p]),
    "dpdb_device_count": (C.c_int, []),
    "dpdb_create": (C.c_int, [C.c_int, C.POINTER(Box), C.POINTER(Params), C.POINTER(Run),
                              C.c_size_t, C.POINTER(C.c_void_p)]),
    "dpdb_destroy": (C.c_int, [C.c_void_p]),
    "dpdb_grid": (C.c_int, [C.c_void_p, C.POINTER(GridInfo)]),
    "dpdb_grid_ranks": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dpdb_grid_plan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                 C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "dpdb_set_neighbors": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]),
    "dpdb_table_layout": (C.c_int, [C.c_int, C.c_int, C.c_size_t, C.c_uint32, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_int32, C.c_int32]),
    "dpdb_stream": (C.c_void_p, [C.c_void_p]),
    "dpdb_upload": (C.c_int, [C.c_void_p, C.c_size_t] + [C.c_void_p] * 9),
    "dpdb_upload_forces": (C.c_int, [C.c_void_p] + [C.c_void_p] * 3),
    "dpdb_download": (C.c_int, [C.c_void_p] + [C.c_void_p] * 12),
    "dpdb_size": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    "dpdb_set_bonds": (C.c_int, [C.c_void_p, C.c_size_t] + [C.c_void_p] * 4),
    "dpdb_set_bonds_styled": (C.c_int, [C.c_void_p, C.c_size_t] + [C.c_void_p] * 5),
    "dpdb_set_angles": (C.c_int, [C.c_void_p, C.c_size_t] + [C.c_void_p] * 5),
    "dpdb_sort_keys": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dpdb_reorder": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dpdb_cell_start": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dpdb_coarse_stencil": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "dpdb_fine_stencil": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "dpdb_build_neighbors": (C.c_int, [C.c_void_p]),
    "dpdb_join_core_skin": (C.c_int, [C.c_void_p]),
    "dpdb_tile_transpose": (C.c_int, [C.c_void_p]),
    "dpdb_get_neighbors": (C.c_int, [C.c_void_p] + [C.c_void_p] * 5),
    "dpdb_signatures": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dpdb_compute_forces": (C.c_int, [C.c_void_p, C.c_uint32]),
    "dpdb_verlet_phase1": (C.c_int, [C.c_void_p]),
    "dpdb_verlet_phase2": (C.c_int, [C.c_void_p]),
    "dpdb_setup": (C.c_int, [C.c_void_p]),
    "dpdb_step": (C.c_int, [C.c_void_p, C.c_int64]),
    "dpdb_setup_at": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32]),
    "dpdb_thermo_get": (C.c_int, [C.c_void_p, C.POINTER(Thermo)]),
    "dpdb_step_thermo": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(Thermo)]),
    "dpdb_init_random": (C.c_int, [C.c_void_p, C.c_size_t, C.c_double, C.c_uint32, C.c_uint32,
                                    C.c_uint32, C.c_void_p, C.c_uint8, C.c_double, C.c_double]),
    "dpdb_profile_reset": (C.c_int, [C.c_void_p, C.c_uint32, C.c_int32, C.c_int32]),
    "dpdb_profile_sample": (C.c_int, [C.c_void_p]),
    "dpdb_profile_get": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]),
    "dpdb_rdf": (C.c_int, [C.c_void_p, C.c_uint32, C.c_double, C.c_void_p]),
    "dpdb_step_timed": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_double), C.c_void_p,
                                  C.c_void_p]),
    "dpdb_current_step": (C.c_int64, [C.c_void_p]),
    "dpdb_table_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.POINTER(C.c_uint32)]),
    "dpdb_eval": (C.c_int, [C.c_int, C.c_int, C.c_size_t, C.c_void_p, C.c_void_p, C.c_uint32,
                            C.c_void_p]),
    "dpdb_radix_sort": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]),
    # brick decomposition
    "dpdb_create_domain": (C.c_int, [C.c_int, C.POINTER(Box), C.POINTER(Params), C.POINTER(Run),
                                     C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "dpdb_domain_info": (C.c_int, [C.c_void_p] + [C.c_void_p] * 4),
    "dpdb_md_neighbor": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "dpdb_md_record_bytes": (C.c_int, [C.c_int]),
    "dpdb_md_begin_setup": (C.c_int, [C.c_void_p]),
    "dpdb_md_begin_rebuild": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dpdb_md_pack": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "dpdb_md_accept_migrants": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "dpdb_md_accept_ghosts": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "dpdb_md_begin_step": (C.c_int, [C.c_void_p]),
    "dpdb_md_accept_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "dpdb_md_forces": (C.c_int, [C.c_void_p]),
    "dpdb_md_finish": (C.c_int, [C.c_void_p]),
    "dpdb_md_sums": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dpdb_md_ghost_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    "dpdb_md_block_split": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "dpdb_md_download_ghosts": (C.c_int, [C.c_void_p] + [C.c_void_p] * 7),
    "dpdb_group_setup": (C.c_int, [C.c_void_p, C.c_int]),
    "dpdb_group_step": (C.c_int, [C.c_void_p, C.c_int, C.c_int64]),
    "dpdb_group_step_thermo": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.POINTER(Thermo)]),
    "dpdb_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "dpdb_nccl_attach": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "dpdb_nccl_mock_attach": (C.c_int, [C.c_void_p, C.c_int]),
    "dpdb_dist_setup": (C.c_int, [C.c_void_p]),
    "dpdb_dist_step": (C.c_int, [C.c_void_p, C.c_int64]),
    "dpdb_dist_step_thermo": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
    "dpdb_dist_step_timed": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_double), C.c_void_p,
                                       C.c_void_p]),
    "dpdb_dist_thermo": (C.c_int, [C.c_void_p, C.POINTER(Thermo)]),
}

NCCL_ID_BYTES = 128

MD_MIGRANTS, MD_GHOST_FULL, MD_GHOST_UPDATE = 0, 1, 2

_lib = None


def lib():
    """Load libdpdb.so; raises (never falls back) when it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} missing: build it with `make -C paper_1311_0402_b200/csrc` "
                "(the engine has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SYMBOLS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ptr(a):
    return None if a is None else a.ctypes.data


def check(rc, ctx=None):
    if rc:
        raise DPDError(rc, lib().dpdb_last_error(ctx).decode())
