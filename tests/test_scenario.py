"""Scenario files: the shipped paper parameter sets parse to
the SPEC's example values; missing / unknown keys and constraint violations are
named.  CPU only."""
import os

import numpy as np
import pytest

from paper_1311_0402_b200 import DPDError
from paper_1311_0402_b200.scenario import parse_config, parse_text

CFG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs")


def test_poiseuille_steady_cfg():
    """sigma = 4.5, rho = 6.0, kT = 0.5, dt = 0.001, g = 0.055, box 12x8x8, a = 0."""
    s = parse_config(os.path.join(CFG, "poiseuille_steady.cfg"))
    assert s.box.hi == (12.0, 8.0, 8.0) and s.n == 4608  # S:48 "total of 4608 particles"
    assert s.kbt == 0.5 and s.params.dt == 0.001 and s.run.body_force == 0.055
    assert np.allclose(s.params.sigma, 4.5) and np.all(s.params.a == 0)
    assert s.profile == dict(bins=32, axis=2, every=100, start=60000)


def test_self_assembly_cfg():
    """rho 5, sigma 3, gamma 4.5, kT 1, dt 0.01, BBBAABBB, r0 0.38, K 80,
    a(A,A)=a(A,S)=a(S,S)=a(B,B)=15, a(A,B)=a(B,S)=120."""
    s = parse_config(os.path.join(CFG, "self_assembly.cfg"))
    assert s.species == ["S", "A", "B"] and s.n == round(5.0 * 27 ** 3)
    a = s.params.a.reshape(3, 3)
    S, A, B = 0, 1, 2
    assert a[A, A] == a[A, S] == a[S, S] == a[B, B] == 15 and a[A, B] == a[B, A] == a[B, S] == 120
    assert np.allclose(s.params.gamma, 4.5) and np.allclose(s.params.sigma, 3.0)
    assert s.chains == dict(fraction=0.1, sequence="BBBAABBB", r0=0.38, k=80.0, solvent="S",
                            bond="harmonic", fene_r0=1.5, angle_k=0.0, angle_theta0=180.0)
    assert s.n_chains == round(0.1 * s.n) // 8


def test_other_shipped_cfgs_parse():
    for f in sorted(os.listdir(CFG)):
        if f.endswith(".cfg"):
            parse_config(os.path.join(CFG, f))
    assert parse_config(os.path.join(CFG, "c3_fluid.cfg")).n == 4194304


def test_empty_file_lists_every_missing_key():
    """empty file -> error listing every missing required key."""
    with pytest.raises(DPDError) as ex:
        parse_text("")
    for k in ("box.hi", "fluid.kbt", "pair.a", "run.dt", "run.steps", "fluid.density",
              "pair.sigma"):
        assert k in str(ex.value)


@pytest.mark.parametrize("text,needle", [
    ("[box]\nhi = 1 1 1\nbogus = 3\n", "unknown key box.bogus"),
    ("[nope]\n", "unknown section"),
    ("[box]\nhi = 1 1\n[fluid]\ndensity=3\nkbt=1\n[pair]\na=25\ngamma=4.5\n[run]\ndt=0.01\nsteps=1\n",
     "box.hi needs 3"),
    ("[box]\nhi = 4 4 4\n[fluid]\ndensity=3\nkbt=1\n[pair]\na=25\ngamma=4.5\nsigma=5\n[run]\ndt=0.01\nsteps=1\n",
     "sigma^2 = 2 gamma kbt"),
    ("[box]\nhi = 0.1 0.1 0.1\n[fluid]\ndensity=0.1\nkbt=1\n[pair]\na=25\ngamma=4.5\n[run]\ndt=0.01\nsteps=1\n",
     "empty system"),
])
def test_violations_are_named(text, needle):
    with pytest.raises(DPDError) as ex:
        parse_text(text)
    assert needle in str(ex.value)
