"""The command line: run writes thermo / profile / XYZ / restart,
bricks via --domains, bench, ulp-sweep; errors exit with the category."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CFG = """[box]
hi = 10 8 12
[fluid]
density = 3.0
kbt = 1.0
seed = 4
[pair]
gamma = 4.5
a = 25
[run]
dt = 0.01
steps = 120
body_force = 0.05
drive_axis = 0
partition_axis = 2
[profile]
bins = 12
axis = 2
every = 20
start = 40
"""


def cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1311_0402_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=300)


def test_run_writes_outputs(tmp_path):
    cfg = tmp_path / "s.cfg"
    cfg.write_text(CFG)
    r = cli("run", str(cfg), "--out", str(tmp_path / "o"))
    assert r.returncode == 0, r.stdout + r.stderr
    t = np.genfromtxt(tmp_path / "o" / "thermo.csv", delimiter=",", names=True)
    # kT includes the driven mean flow (only the COM is subtracted): starts at 1, grows
    assert list(t["step"]) == list(range(0, 121)) and abs(t["kbt"][0] - 1) < 0.1
    assert np.all(np.isfinite(t["kbt"])) and t["kbt"][-1] > t["kbt"][0]
    p = np.genfromtxt(tmp_path / "o" / "profile.csv", delimiter=",", names=True)
    assert len(p) == 12 and np.all(p["count"] > 0)
    lines = (tmp_path / "o" / "final.xyz").read_text().splitlines()
    assert int(lines[0]) == 2880 and lines[1] == "step 120"
    from paper_1311_0402_b200 import io as dio
    store, step, seed, hdr = dio.read_restart(tmp_path / "o" / "restart.bin")
    assert step == 120 and seed == 4 and len(store.tag) == 2880
    r = cli("run", str(cfg), "--out", str(tmp_path / "b"), "--domains", "2x1x1")
    assert r.returncode == 0, r.stdout + r.stderr
    tb = np.genfromtxt(tmp_path / "b" / "thermo.csv", delimiter=",", names=True)
    assert list(tb["step"]) == list(range(0, 121))


def test_bench_ulp_and_errors(tmp_path):
    r = cli("bench", os.path.join(ROOT, "configs", "c3_fluid.cfg"), "--steps", "20")
    assert r.returncode == 0 and "M particle-steps/s" in r.stdout, r.stdout + r.stderr
    r = cli("ulp-sweep", "gaussian_hot", "--samples", "2000")
    assert r.returncode == 0 and r.stdout.startswith("input,output,reference,ulp_error")
    assert len(r.stdout.splitlines()) == 2001 and "ulp histogram" in r.stderr
    bad = tmp_path / "bad.cfg"
    bad.write_text("[box]\nhi = 1 1 1\n")
    r = cli("run", str(bad))
    assert r.returncode == 1 and "missing required keys" in r.stderr
