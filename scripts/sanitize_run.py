"""Small end-to-end exercise of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): single-domain fused loop with rebuilds
(range builder + flat pair lists + fused Verlet epilogue + thermo), the
stage-by-stage ABI (reference layout: k_force, joins/transposes), the lane and
ballot builders, bonded amphiphile chains (FENE + angles in the epilogue),
walls + body force, observables (profile, rdf), a 2x2x1 brick group with the
overlapped halo update, the radix sort and the parity primitives."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_1311_0402_b200 as dpd  # noqa: E402
from paper_1311_0402_b200 import domain as D  # noqa: E402
import dpdsys as _sys  # noqa: E402


def fluid_run():
    box, obox, st = _sys.fluid((9, 8, 7), 3.0, seed=5)
    e = _sys.engine(box, st, run=dpd.RunConfig(rebuild_every=4))
    e.setup()
    e.step_thermo(9)
    e.rdf_counts(26, 1.3)
    e.profile_reset(8, 2, 0)
    e.step(3)
    e.profile_sample()
    e.neighbor_table()
    e.close()


def stage_api():
    box, obox, st = _sys.fluid((8, 8, 8), 3.0, seed=6)
    e = _sys.engine(box, st)
    e.reorder_particles()
    e.build_neighbor_table()
    e.compute_forces(1)
    e.join_core_skin()
    e.tile_transpose()
    e.compute_forces(2)
    e.verlet_phase1()
    e.verlet_phase2()
    e.close()


def builders():
    for b in ("lane", "ballot"):
        os.environ["DPDB_BUILDER"] = b
        box, obox, st = _sys.fluid((8, 7, 9), 3.0, seed=7)
        e = _sys.engine(box, st, run=dpd.RunConfig(rebuild_every=3))
        e.setup()
        e.step(4)
        e.close()
    os.environ.pop("DPDB_BUILDER")


def bonded_walls():
    L = (9.0, 8.0, 8.0)
    p = dpd.PairParams.make(3, [15, 15, 120, 15, 15, 120, 120, 120, 15], 4.5, 1.0, 1.0, 1.0, 0.01)
    box = dpd.SimBox((0.0, 0.0, 0.0), L, (True, True, False), (False, False, True))
    n, nc = 1700, 20
    e = dpd.Engine(box, p, dpd.RunConfig(body_force=0.05, drive_axis=0, partition_axis=2), capacity=n)
    e.init_random(n, 1.0, 3, nc, [2, 2, 2, 1, 1, 2, 2, 2], 0, 0.38, 80.0)
    first = np.arange(nc) * 8 + 1
    ti = (first[:, None] + np.arange(7)[None, :]).ravel()
    e.set_bonds(ti, ti + 1, 40.0, 2.0, style=1)
    ta = (first[:, None] + np.arange(6)[None, :]).ravel()
    e.set_angles(ta, ta + 1, ta + 2, 4.0, np.pi)
    e.setup()
    e.step(12)
    e.close()


def bricks():
    box, obox, st = _sys.fluid((12, 12, 8), 3.0, seed=8)
    g = D.BrickGroup(box, dpd.PairParams(), dpd.RunConfig(rebuild_every=3), (2, 2, 1), capacity=len(st[0]))
    g.upload(dpd.ParticleStore.from_arrays(*st))
    g.setup()
    g.step(7)
    g.download()
    g.close()


def primitives():
    k = np.random.default_rng(0).integers(0, 2**20, 5000).astype(np.uint32)
    dpd.radix_sort(k, np.arange(5000, dtype=np.uint32), 20)
    a = np.arange(1, 4000, dtype=np.uint32)
    dpd.gaussian(a, a[::-1].copy(), hot=True)


if __name__ == "__main__":
    for f in (fluid_run, stage_api, builders, bonded_walls, bricks, primitives):
        f()
        print("ok", f.__name__, flush=True)
