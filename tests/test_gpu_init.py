"""init_random on the device: bit-exact with
the oracle's init_fluid for a fluid, chains as random walks with step r0 and
bonds along them, zero net momentum, reproducible per seed."""
import numpy as np
import pytest

import oracle as O
import paper_1311_0402_b200 as dpd

pytestmark = pytest.mark.gpu


def test_init_fluid_bitexact_vs_oracle():
    L = (12.0, 8.0, 8.0)
    n = 4608  # box 12x8x8 at rho 6
    obox = O.make_box((0, 0, 0), L)
    st = O.init_fluid(obox, n, 0.5, 7)
    e = dpd.Engine(dpd.SimBox((0.0, 0.0, 0.0), L), dpd.PairParams(), dpd.RunConfig(), capacity=n)
    e.init_random(n, 0.5, 7)
    s = e.download()
    for k in range(3):
        assert np.array_equal(s.coord[k], st[k])
        assert np.array_equal(s.veloc[k], st[3 + k])
    assert np.array_equal(s.tag, st[6])


def test_init_chains_geometry_and_bonds():
    L = (10.0, 10.0, 10.0)
    p = dpd.PairParams.make(3, [15, 15, 15, 15, 15, 120, 15, 120, 15], 4.5, 1.0, 1.0, 1.0, 0.01)
    n, nc, seq = 5000, 60, [2, 2, 2, 1, 1, 2, 2, 2]
    e = dpd.Engine(dpd.SimBox((0.0, 0.0, 0.0), L), p, dpd.RunConfig(), capacity=n)
    e.init_random(n, 1.0, 3, nc, seq, 0, 0.38, 80.0)
    s = e.download()
    assert np.array_equal(s.tag, np.arange(1, n + 1))
    assert np.array_equal(s.species[: nc * 8], np.tile(seq, nc)) and np.all(s.species[nc * 8:] == 0)
    X = np.stack(s.coord, 1)
    assert np.all((X >= 0) & (X < 10.0))
    d = X[1: nc * 8] - X[: nc * 8 - 1]
    d -= 10.0 * np.round(d / 10.0)
    r = np.linalg.norm(d, axis=1)
    within = np.arange(1, nc * 8) % 8 != 0  # consecutive beads of one chain
    assert np.allclose(r[within], 0.38, rtol=0, atol=1e-12)
    V = np.stack(s.veloc, 1)
    assert np.abs(V.sum(0)).max() < 1e-9  # zero net momentum
    # bonds are live: the setup forces include K (r - r0) = 0 at the rest length
    e.setup()
    e.step(5)
    # same seed -> bitwise the same state
    e2 = dpd.Engine(dpd.SimBox((0.0, 0.0, 0.0), L), p, dpd.RunConfig(), capacity=n)
    e2.init_random(n, 1.0, 3, nc, seq, 0, 0.38, 80.0)
    s2 = e2.download()
    for k in range(3):
        assert np.array_equal(s.coord[k], s2.coord[k]) and np.array_equal(s.veloc[k], s2.veloc[k])


def test_init_errors():
    e = dpd.Engine(dpd.SimBox((0.0, 0.0, 0.0), (4.0, 4.0, 4.0)), dpd.PairParams(), dpd.RunConfig(),
                   capacity=100)
    with pytest.raises(dpd.DPDError) as ex:
        e.init_random(0, 1.0, 1)
    assert "empty system" in str(ex.value)
    with pytest.raises(dpd.DPDError):
        e.init_random(200, 1.0, 1)  # beyond capacity
    with pytest.raises(dpd.DPDError):
        e.init_random(100, 1.0, 1, 5, [1] * 8, 0)  # species 1 with one species


def test_self_assembly_aggregates():
    """SPEC invariant (paper section 4.5), desk scale: 98,415 particles,
    10% BBBAABBB amphiphiles in solvent with the paper's repulsion matrix; the
    hydrophobic B beads aggregate -- the largest B cluster (union-find at
    contact distance r_c) holds > 50 chains within the SPEC's 2e5 steps
    (here after 5e4) and is several times the random initial one."""
    import os
    from paper_1311_0402_b200.scenario import largest_cluster, parse_config
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = parse_config(os.path.join(root, "configs", "self_assembly.cfg"))
    e = s.engine()
    e.setup()
    nb = s.n_chains * 8

    def biggest():
        st = e.download()
        mol = np.where(st.tag <= nb, (st.tag - 1) // 8 + 1, 0)
        return largest_cluster(st.coord, st.species, mol, s.box, [s.species.index("B")])

    c0 = biggest()
    e.step(50000)
    c1 = biggest()
    assert c1[1] > 50 and c1[1] >= 3 * c0[1], (c0, c1)
    assert abs(e.thermo()["kbt"] - 1.0) < 0.03


def test_fene_angle_chains_run_stably(tmp_path):
    """A scenario with FENE chains and harmonic angles (beyond the reference)
    runs: bonds stay inside R0, temperature stays at kT."""
    from paper_1311_0402_b200.scenario import parse_text
    s = parse_text("""[box]
hi = 12 12 12
[fluid]
density = 3
kbt = 1
seed = 2
species = S A B
[pair]
gamma = 4.5
a = 25
a.A.B = 50
[run]
dt = 0.01
steps = 2000
[chains]
fraction = 0.2
sequence = BBBAABBB
r0 = 0.5
k = 20
bond = fene
fene_r0 = 1.5
angle_k = 3
angle_theta0 = 180
""")
    e = s.engine()
    e.setup()
    rec = e.step_thermo(2000)
    assert abs(rec["kbt"][1000:].mean() - 1.0) < 0.05
    st = e.download()
    o = np.argsort(st.tag)
    X = np.stack(st.coord, 1)[o]
    nb = s.n_chains * 8
    d = X[1:nb] - X[:nb - 1]
    d -= 12.0 * np.round(d / 12.0)
    r = np.linalg.norm(d, axis=1)[np.arange(1, nb) % 8 != 0]
    assert r.max() < 1.5 and r.mean() < 1.2
