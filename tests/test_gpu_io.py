"""write_outputs: restart round trip bitwise on one domain,
XYZ / thermo / profile formats."""
import numpy as np
import pytest

import paper_1311_0402_b200 as dpd
from paper_1311_0402_b200 import io as dio
import dpdsys as _sys

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fuse", ["1", "0"])
def test_restart_round_trip_bitwise(tmp_path, monkeypatch, fuse):
    """save at step k (a rebuild step), reload, run to k + 100 -> bitwise
    equal to the uninterrupted run."""
    monkeypatch.setenv("DPDB_FUSE", fuse)
    box, obox, st = _sys.fluid((10, 9, 8), 3.0, seed=13)
    a = _sys.engine(box, st)
    a.setup()
    a.step(20)
    path = tmp_path / "state.rst"
    dio.save_restart(path, a)
    a.step(100)
    b = dpd.Engine(box, dpd.PairParams(), dpd.RunConfig(), capacity=len(st[0]))
    assert dio.load_restart(path, b) == 20
    b.step(100)
    sa, sb = a.download(), b.download()
    oa, ob = np.argsort(sa.tag), np.argsort(sb.tag)
    for u, w in zip(sa.coord + sa.veloc + sa.force, sb.coord + sb.veloc + sb.force):
        assert np.array_equal(u[oa], w[ob])
    assert b.current_step == 120


def test_restart_rejects_bad_files(tmp_path):
    p = tmp_path / "bad.rst"
    p.write_bytes(b"not a restart file at all, too short?" * 3)
    with pytest.raises(ValueError):
        dio.read_restart(p)


def test_text_outputs(tmp_path):
    box, obox, st = _sys.fluid((6, 6, 6), 3.0, seed=2)
    e = _sys.engine(box, st)
    e.setup()
    rec = e.step_thermo(5)
    s = e.download()
    dio.write_xyz(tmp_path / "f.xyz", s, comment="step 5")
    lines = (tmp_path / "f.xyz").read_text().splitlines()
    assert int(lines[0]) == len(s.tag) and lines[1] == "step 5" and len(lines) == len(s.tag) + 2
    assert lines[2].split()[0] == "S" and np.isclose(float(lines[2].split()[1]), s.coord[0][0])
    dio.write_thermo_csv(tmp_path / "t.csv", rec, 0.01, len(s.tag))
    t = np.genfromtxt(tmp_path / "t.csv", delimiter=",", names=True)
    assert np.array_equal(t["step"], rec["step"]) and np.array_equal(t["kbt"], rec["kbt"])  # exact
    one = dpd.ParticleStore.from_arrays([1.0], [2.0], [3.0], [0.0], [0.0], [0.0], [1])
    dio.write_xyz(tmp_path / "one.xyz", one)
    assert len((tmp_path / "one.xyz").read_text().splitlines()) == 3
