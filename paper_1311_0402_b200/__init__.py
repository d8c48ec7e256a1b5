"""B200-native DPD engine (Tang & Karniadakis, arXiv:1311.0402 capabilities).

The product is libdpdb.so: C++ host code + hand-written sm_100a kernels behind
the C ABI in include/dpdb.h.  This package is the Python mirror of the
reference's C++ API over that ABI (engine.py) plus its build helper.
"""
from __future__ import annotations

import os
import subprocess

from ._lib import DPDError, LIB_PATH, lib  # noqa: F401
from .engine import (  # noqa: F401
    Engine, NeighborTable, PairParams, ParticleStore, RunConfig, SimBox, device_count,
    fastcos2pi, fastlog, fastpow, gaussian, make_signature, morton_encode, pair_uniforms,
    radix_sort, step_mix, tea_hash,
)
from .domain import BrickGroup, DistBrick, HaloExchange, NcclBrick  # noqa: F401

HERE = os.path.dirname(os.path.abspath(__file__))


def build(verbose: bool = False) -> str:
    """Compile libdpdb.so for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-C", os.path.join(HERE, "csrc")] + ([] if verbose else ["-s"]),
                   check=True)
    return LIB_PATH
