"""The drop-in boundary on the GPU: the same unchanged caller
(tests/cpp/ref_caller.cpp, reference headers only) built once on the
reference path (its five shipped sources + the oracle restatement of the
missing slots, oracle/_ref/ref_caller) and once on the B200 drop-in
(dropin/*.cpp over libdpdb.so, dropin/_build/b200_caller); both prebuilt by
__graft_entry__.build() where /root/reference exists.  Identical inputs and
seeds; the outputs must agree:
  * CellGrid::make, reorder_particles (perm, order), local_cell_ranks,
    build_cell_list, signatures, RadixSorter::sort: bit-exact;
  * build_neighbor_table rows (core/skin counts and entries through the
    accessors), before and after join_core_skin + tile_transpose: bit-exact;
  * compute_forces (pairs + harmonic bonds): rel-L2 <= 1e-5 and every
    particle within 1e-5 of rms|F| (fp32 device forces vs the fp64 oracle);
  * verlet_step on fp32-valued forces: bit-exact."""
import os

import numpy as np
import pytest

import dropin_io as D

pytestmark = pytest.mark.gpu

EXACT = ["grid.geometry", "grid.rank_of_cell", "grid.cell_of_rank", "grid.cellsize", "reorder.perm",
         "reorder.tag", "reorder.x", "cell.ranks", "cell.start", "signature", "table.core", "table.skin",
         "table.rows", "table.joined.core", "table.joined.skin", "table.joined.rows", "radix.keys",
         "radix.vals"]


@pytest.mark.parametrize("L", [12, 21])
def test_drop_in_matches_reference_path(tmp_path, L):
    if not (os.access(D.REF_BIN, os.X_OK) and os.access(D.B200_BIN, os.X_OK)):
        pytest.skip("callers not built (build() builds them where /root/reference exists)")
    rc, err, ref = D.run(D.REF_BIN, L, str(tmp_path / "ref.bin"))
    assert rc == 0, err
    rc, err, b2 = D.run(D.B200_BIN, L, str(tmp_path / "b200.bin"))
    assert rc == 0, err
    for k in EXACT:
        assert np.array_equal(ref[k], b2[k]), k
    F = np.stack([ref["force." + a] for a in "xyz"], 1)
    G = np.stack([b2["force." + a] for a in "xyz"], 1)
    rms = np.sqrt((F ** 2).sum(1).mean())
    l2 = np.linalg.norm(G - F) / np.linalg.norm(F)
    mx = np.sqrt(((G - F) ** 2).sum(1)).max() / rms
    print(f"L={L}: forces rel L2 {l2:.2e}, max/rms {mx:.2e}")
    assert l2 <= 1e-5 and mx <= 1e-5
    for k in ("verlet1.x", "verlet1.vz", "verlet2.vy"):  # identical fp32 force fields
        assert np.array_equal(ref[k], b2[k]), k
