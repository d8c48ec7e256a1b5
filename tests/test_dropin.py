"""The drop-in boundary on CPU (no GPU): an unchanged caller written against
the reference's own headers (/root/reference/proj/include) compiles and links
against the B200 drop-in (dropin/ + libdpdb.so) and against the reference's
own shipped sources (oracle/_ref/ref_caller).  Without a device the drop-in
path fails loudly at its first device call (no CPU fallback) after the
host-side CellGrid::make, which must equal the reference's."""
import os
import subprocess

import numpy as np
import pytest

import dropin_io as D

REF_TREE = "/root/reference/proj"


def _build():
    if not os.path.isdir(os.path.join(REF_TREE, "src")):
        pytest.skip("reference tree absent (the GPU box runs the prebuilt callers)")
    subprocess.run(["make", "-s", "-C", os.path.join(D.ROOT, "paper_1311_0402_b200", "csrc")], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(D.ROOT, "dropin")], check=True)


def test_caller_builds_against_reference_headers(tmp_path):
    _build()
    assert os.access(D.B200_BIN, os.X_OK) and os.access(D.REF_BIN, os.X_OK)
    # the drop-in binary resolves libdpdb.so from the repo, not the oracle
    ldd = subprocess.run(["ldd", D.B200_BIN], capture_output=True, text=True).stdout
    assert "libdpdb.so" in ldd and "liboracle" not in ldd


def test_reference_path_runs_and_drop_in_fails_loudly_without_gpu(tmp_path):
    _build()
    import paper_1311_0402_b200 as dpd

    if dpd.device_count() > 0:
        pytest.skip("a device is present: tests/test_gpu_dropin.py covers this")
    rc, err, ref = D.run(D.REF_BIN, 10, str(tmp_path / "ref.bin"))
    assert rc == 0, err
    rc, err, b2 = D.run(D.B200_BIN, 10, str(tmp_path / "b200.bin"))
    assert rc == 4 and "device" in err and "no CPU fallback" in err, (rc, err)
    # CellGrid::make is host-side in both: identical grids
    for k in ("grid.geometry", "grid.rank_of_cell", "grid.cell_of_rank", "grid.cellsize"):
        assert np.array_equal(ref[k], b2[k]), k
    assert "reorder.perm" in ref and "reorder.perm" not in b2
