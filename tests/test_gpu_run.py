"""Integrator parity (bit-exact fp64 Verlet) and whole-step runs of
Alg. 1 against the oracle's CPU driver (statistical agreement)."""
import numpy as np
import pytest

import oracle as O
import paper_1311_0402_b200 as dpd
import dpdsys as _sys

pytestmark = pytest.mark.gpu


def f32_forces(n, seed):
    return [(np.random.default_rng(seed + k).normal(size=n) * 20).astype(np.float32).astype(np.float64)
            for k in range(3)]


@pytest.mark.parametrize("per,wall", [((1, 1, 1), (0, 0, 0)), ((0, 1, 1), (1, 0, 0))])
def test_verlet_bitexact(per, wall):
    box, obox, st = _sys.fluid((8, 8, 8), 3.0, per, seed=3, wall=wall)
    n = len(st[0])
    st = [a.copy() for a in st]
    # push a few particles across the boundaries
    st[0][:20] = 8.0 - 1e-4
    st[3][:20] = 3.0
    st[0][20:40] = 1e-4
    st[3][20:40] = -3.0
    F = f32_forces(n, 1)
    e = _sys.engine(box, st)
    e.upload_forces(*F)
    e.verlet_phase1()
    e.verlet_phase2()
    s = e.download()
    x, y, z, vx, vy, vz = [a.copy() for a in st[:6]]
    O.check(O.lib().orc_verlet_phase1(obox, 0.01, n, x, y, z, vx, vy, vz, *F, None))
    O.lib().orc_verlet_phase2(0.01, n, vx, vy, vz, *F)
    for got, ref in zip(s.coord + s.veloc, [x, y, z, vx, vy, vz]):
        assert np.array_equal(got, ref)
    assert (s.coord[0] >= 0).all() and (s.coord[0] < 8).all()


def test_blowup_is_physics_error():
    box, obox, st = _sys.fluid((8, 8, 8), 3.0, seed=3)
    st = [a.copy() for a in st]
    st[3][7] = np.inf
    e = _sys.engine(box, st)
    with pytest.raises(dpd.DPDError) as ex:
        e.verlet_phase1()
    assert ex.value.code == 2


@pytest.mark.parametrize("s_exp", [1.0, 0.5])
def test_fused_step_equals_stagewise_api(s_exp):
    """dpdb_step's fused kernels (phase2+phase1+streams, reorder, build, force)
    reproduce the stage-by-stage ABI sequence of Alg. 1 bit for bit (s = 0.5:
    the general weight-exponent path of the walk kernel)."""
    box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=21)
    p = dpd.PairParams.make(1, 25.0, 4.5, 1.0, s_exp, 1.0, 0.01)
    a = _sys.engine(box, st, params=p)
    a.setup()
    b = _sys.engine(box, st, params=p)
    b.reorder_particles()
    b.build_neighbor_table()
    b.compute_forces(0)
    for step in range(1, 26):
        a.step(1)
        b.verlet_phase1()
        if step % 10 == 0:
            b.reorder_particles()
            b.build_neighbor_table()
        b.compute_forces(step)
        b.verlet_phase2()
    sa, sb = a.download(), b.download()
    assert np.array_equal(sa.tag, sb.tag)
    for u, w in zip(sa.coord + sa.veloc + sa.force, sb.coord + sb.veloc + sb.force):
        assert np.array_equal(u, w)
    c = _sys.engine(box, st, params=p)  # one call of 25 steps == 25 calls of one step
    c.setup()
    c.step(25)
    sc = c.download()
    for u, w in zip(sa.coord + sa.veloc, sc.coord + sc.veloc):
        assert np.array_equal(u, w)


@pytest.mark.parametrize("case", ["poiseuille_walls", "two_species"])
def test_fused_force_integrate_equals_separate_pass(monkeypatch, case):
    """The step loop runs the Verlet pass inside the force kernel's epilogue
    (DPDB_FUSE default); DPDB_FUSE=0 keeps it a separate kernel.  Both give
    the same trajectory bit for bit, across rebuilds (the fused pass then
    writes the sort keys), with body force + walls and with two species."""
    if case == "poiseuille_walls":
        box, obox, st = _sys.fluid((10, 8, 12), 3.0, (1, 1, 0), seed=23, wall=(0, 0, 1))
        params, run = dpd.PairParams(), dpd.RunConfig(rebuild_every=4, body_force=0.05, drive_axis=0,
                                                      partition_axis=2)
    else:
        box, obox, st = _sys.fluid((11, 11, 11), 3.0, seed=29)
        st = list(st)
        sp = (np.arange(len(st[0])) % 2).astype(np.uint8)
        params, run = dpd.PairParams.make(2, [25, 40, 40, 25], 4.5, 1.0, 1.0, 1.0, 0.01), dpd.RunConfig(rebuild_every=5)
    out = []
    for fuse in ("1", "0"):
        monkeypatch.setenv("DPDB_FUSE", fuse)
        e = dpd.Engine(box, params, run, capacity=len(st[0]))
        ps = dpd.ParticleStore.from_arrays(*st)
        if case == "two_species":
            ps.species = sp
        e.upload(ps)
        e.setup()
        e.step(13)
        out.append(e.download())
    for u, w in zip(out[0].coord + out[0].veloc + out[0].force, out[1].coord + out[1].veloc + out[1].force):
        assert np.array_equal(u, w)


@pytest.mark.parametrize("case", ["fluid_1m", "two_species"])
def test_line_grouped_lists_equal_row_ordered(monkeypatch, case):
    """The range builder groups each tile's flat pair list by partner cache
    line (DPDB_BUCKET default); DPDB_BUCKET=0 keeps row order.  Same pair set,
    order-free fixed-point sums: identical trajectories, forces and thermo
    records bit for bit, across rebuilds."""
    if case == "fluid_1m":
        n = 2**20
        L = (n / 3.0) ** (1.0 / 3.0)
        box, obox, st = _sys.fluid((L, L, L), 3.0, seed=7)
        params, run = dpd.PairParams(), dpd.RunConfig()
    else:
        box, obox, st = _sys.fluid((11, 11, 11), 3.0, seed=29)
        params = dpd.PairParams.make(2, [25, 40, 40, 25], 4.5, 1.0, 1.0, 1.0, 0.01)
        run = dpd.RunConfig(rebuild_every=5)
    out = []
    for b in ("1", "0"):
        monkeypatch.setenv("DPDB_BUCKET", b)
        e = dpd.Engine(box, params, run, capacity=len(st[0]))
        ps = dpd.ParticleStore.from_arrays(*st)
        if case == "two_species":
            ps.species = (np.arange(len(st[0])) % 2).astype(np.uint8)
        e.upload(ps)
        e.setup()
        rec = e.step_thermo(23)
        out.append((e.download(), rec))
        e.close()
    (a, ra), (b, rb) = out
    for u, w in zip(a.coord + a.veloc + a.force, b.coord + b.veloc + b.force):
        assert np.array_equal(u, w)
    for k in ra:
        assert np.array_equal(ra[k], rb[k])


@pytest.mark.parametrize("extra", [False, True])
def test_bonded_pipeline_equals_stagewise_api(extra):
    """With bonds the step loop adds the bond forces in the pair kernel's
    epilogue (and still fuses the Verlet pass); the stage-by-stage ABI adds
    them with the separate k_bonds pass.  Same trajectory bit for bit (three
    species, 8-bead chains; extra: FENE bonds + harmonic angles)."""
    L = (10.0, 10.0, 10.0)
    p = dpd.PairParams.make(3, [15, 15, 120, 15, 15, 120, 120, 120, 15], 4.5, 1.0, 1.0, 1.0, 0.01)
    box = dpd.SimBox((0.0, 0.0, 0.0), L)
    n, nc, seq = 5000, 60, [2, 2, 2, 1, 1, 2, 2, 2]

    def fresh():
        e = dpd.Engine(box, p, dpd.RunConfig(), capacity=n)
        e.init_random(n, 1.0, 9, nc, seq, 0, 0.38, 80.0)
        if extra:
            first = np.arange(nc) * 8 + 1
            ti = (first[:, None] + np.arange(7)[None, :]).ravel()
            e.set_bonds(ti, ti + 1, 40.0, 2.0, style=1)
            ta = (first[:, None] + np.arange(6)[None, :]).ravel()
            e.set_angles(ta, ta + 1, ta + 2, 4.0, np.pi)
        return e

    a = fresh()
    a.setup()
    a.step(23)
    b = fresh()
    b.reorder_particles()
    b.build_neighbor_table()
    b.compute_forces(0)
    for step in range(1, 24):
        b.verlet_phase1()
        if step % 10 == 0:
            b.reorder_particles()
            b.build_neighbor_table()
        b.compute_forces(step)
        b.verlet_phase2()
    sa, sb = a.download(), b.download()
    oa, ob = np.argsort(sa.tag), np.argsort(sb.tag)
    for u, w in zip(sa.coord + sa.veloc + sa.force, sb.coord + sb.veloc + sb.force):
        assert np.array_equal(u[oa], w[ob])


def test_first_step_vs_oracle_driver():
    """Setup + one step against the oracle's Alg. 1 driver.  After one step
    the fp64 positions agree to fp32-force rounding; beyond that trajectories
    are compared statistically only (a velocity differing in its 11 leading
    mantissa bits changes a signature, P:241-266 / SURVEY hard part 4)."""
    box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=21)
    e = _sys.engine(box, st)
    e.setup()
    e.step(1)
    s = e.download()
    sim = O.Sim(obox, _sys.oparams(dpd.PairParams()), st, nthreads=8)
    sim.run(1)
    r = sim.state()
    og, orr = np.argsort(s.tag), np.argsort(r["tag"])
    for k, key in enumerate("xyz"):
        d = s.coord[k][og] - r[key][orr]
        d -= 12.0 * np.round(d / 12.0)
        assert np.abs(d).max() < 1e-7


def test_long_run_statistics_vs_oracle():
    box, obox, st = _sys.fluid((10, 10, 10), 3.0, seed=22)
    e = _sys.engine(box, st)
    e.setup()
    sim = O.Sim(obox, _sys.oparams(dpd.PairParams()), st, nthreads=8)
    e.step(300)
    sim.run(300)
    tg, to = [], []
    for _ in range(20):
        e.step(10)
        sim.run(10)
        tg.append(e.thermo()["kbt"])
        to.append(sim.temperature())
    assert abs(np.mean(tg) - 1.0) < 0.03 and abs(np.mean(to) - 1.0) < 0.03
    assert abs(np.mean(tg) - np.mean(to)) < 0.03


def test_thermostat_c1():
    """C1: 98,304 particles, rho=3: k_B T within 2% of target."""
    box, obox, st = _sys.fluid((32, 32, 32), 3.0, seed=1)
    e = _sys.engine(box, st)
    e.setup()
    e.step(300)
    T = []
    for _ in range(20):
        e.step(25)
        th = e.thermo()
        T.append(th["kbt"])
        assert max(abs(m) for m in th["momentum"]) < 1e-6 * len(st[0])
    assert abs(np.mean(T) - 1.0) < 0.02


def test_c3_properties_4m():
    """C3 size (4,194,304 particles): size-independent properties of the table
    and forces after a rebuild -- symmetric ascending rows, zero net force."""
    L = (2**22 / 3.0) ** (1 / 3)
    box, obox, st = _sys.fluid((L, L, L), 3.0, seed=3)
    n = len(st[0])
    e = _sys.engine(box, st)
    e.setup()
    e.step(300)
    t = e.neighbor_table()
    sel = np.random.default_rng(0).integers(0, n, 2000)
    for i in sel:
        c = t.core_row(i).astype(np.int64)
        assert np.all(np.diff(c) > 0) and np.all(np.diff(t.skin_row(i).astype(np.int64)) > 0)
        for j in c[:3]:
            assert i in t.core_row(j) or i in t.skin_row(j)
    mean_row = (t.core_count.astype(np.float64) + t.skin_count).mean()
    assert 25.0 < mean_row < 28.3  # ideal gas: rho 4pi/3 1.3^3 = 27.6; a=25 depletes g(r<1)
    F = np.stack(e.download().force, 1)
    rms = np.sqrt((F ** 2).sum(1).mean())
    assert np.abs(F.sum(0)).max() < 1e-5 * rms * np.sqrt(n)
    assert abs(e.thermo()["kbt"] - 1.0) < 0.05


@pytest.mark.parametrize("fuse", ["1", "0"])
def test_step_thermo_records(monkeypatch, fuse):
    """dpdb_step_thermo: every step's thermo line is reduced on the device by
    the pass that applies that step's phase-2 kick (fused force epilogue or the
    separate Verlet pass); the records match dpdb_thermo_get after each single
    step, and the trajectory is the one dpdb_step gives."""
    monkeypatch.setenv("DPDB_FUSE", fuse)
    box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=31)
    a = _sys.engine(box, st, run=dpd.RunConfig(rebuild_every=4))
    b = _sys.engine(box, st, run=dpd.RunConfig(rebuild_every=4))
    a.setup()
    b.setup()
    ref = []
    for _ in range(11):
        a.step(1)
        ref.append(a.thermo())
    rec = b.step_thermo(11)
    assert list(rec["step"]) == [t["step"] for t in ref]
    n = len(st[0])
    for k, t in enumerate(ref):
        assert abs(rec["kbt"][k] - t["kbt"]) <= 1e-12 * t["kbt"]
        assert np.allclose(rec["momentum"][k], t["momentum"], rtol=0, atol=1e-9 * n)
    sa, sb = a.download(), b.download()
    for u, w in zip(sa.coord + sa.veloc + sa.force, sb.coord + sb.veloc + sb.force):
        assert np.array_equal(u, w)
    rec2 = b.step_thermo(3)  # a second call continues the step count
    assert list(rec2["step"]) == [12, 13, 14]


def test_step_thermo_long_call_and_interleaving():
    """A call longer than the preallocated record ring (4096) grows it; the
    side-stream record folds alternate between two partial buffers, so
    records stay exact across interleaved dpdb_step / dpdb_thermo calls."""
    box, obox, st = _sys.fluid((6, 6, 6), 3.0, seed=33)
    a = _sys.engine(box, st, run=dpd.RunConfig(rebuild_every=5))
    b = _sys.engine(box, st, run=dpd.RunConfig(rebuild_every=5))
    a.setup()
    b.setup()
    rec = b.step_thermo(4101)
    assert len(rec["step"]) == 4101 and rec["step"][0] == 1 and rec["step"][-1] == 4101
    assert np.all(np.isfinite(rec["kbt"])) and abs(rec["kbt"][-100:].mean() - 1.0) < 0.1
    a.step(4100)
    a.step(1)
    t = a.thermo()
    assert t["step"] == 4101 and abs(rec["kbt"][-1] - t["kbt"]) <= 1e-12 * t["kbt"]
    def one(e):
        e.step(1)
        return e.thermo()

    for k in range(3):  # interleaved: step_thermo, step, thermo, step_thermo
        r1 = b.step_thermo(2)
        b.step(1)
        t1 = b.thermo()
        r2 = b.step_thermo(1)
        ref = [one(a) for _ in range(4)]
        got = [(r1["step"][0], r1["kbt"][0]), (r1["step"][1], r1["kbt"][1]),
               (t1["step"], t1["kbt"]), (r2["step"][0], r2["kbt"][0])]
        for (s_, kt), t in zip(got, ref):
            assert s_ == t["step"] and abs(kt - t["kbt"]) <= 1e-12 * t["kbt"], (k, s_)


@pytest.mark.parametrize("mode", [0, 1])
def test_closed_box_walls(mode):
    """walls on every axis, ideal gas with a = gamma = sigma = 0:
    no particle ever outside the box and kinetic energy conserved exactly
    (reflections only flip velocity signs), for the specular bounce-forward
    (default) and the bounce-back switch; bounce-back reverses the whole
    velocity of a particle that hits a wall."""
    L = (6.0, 5.0, 4.0)
    box, obox, st = _sys.fluid(L, 3.0, (0, 0, 0), seed=19, wall=(1, 1, 1))
    st = list(st)
    for k in range(3):
        st[3 + k] = st[3 + k] * 20.0  # fast particles: many wall hits per step
    p = dpd.PairParams.make(1, 0.0, 0.0, 0.0, 1.0, 1.0, 0.01)
    e = _sys.engine(box, st, params=p, run=dpd.RunConfig(wall_mode=mode))
    e.setup()
    ke0 = sum(float(np.dot(v, v)) for v in e.download().veloc)
    for _ in range(20):
        e.step(5)
        s = e.download()
        X = np.stack(s.coord, 1)
        assert np.all(X >= 0) and np.all(X < np.array(L))
    assert sum(float(np.dot(v, v)) for v in s.veloc) == pytest.approx(ke0, rel=1e-12)
    # one particle crossing hi by eps
    one = dpd.Engine(dpd.SimBox((0.0, 0.0, 0.0), L, (False,) * 3, (True,) * 3), p,
                     dpd.RunConfig(wall_mode=mode), capacity=1)
    one.upload(dpd.ParticleStore.from_arrays([5.99], [2.0], [2.0], [2.0], [0.5], [-0.25], [1]))
    one.setup()
    one.step(1)
    s = one.download()
    assert s.coord[0][0] == pytest.approx(6.0 - 0.01, abs=1e-12)
    v = [s.veloc[k][0] for k in range(3)]
    assert v == ([-2.0, 0.5, -0.25] if mode == 0 else [-2.0, -0.5, 0.25])


def test_error_stops_a_long_step_call_early():
    """A blow-up inside a long dpdb_step call is reported as a physics error
    naming the particle, and the call stops a few rebuild periods after it
    (the error word is copied and polled without a host sync at every
    rebuild; the host runs ahead of the device by its launch queue) instead
    of running all the remaining steps on garbage."""
    box, obox, st = _sys.fluid((8, 8, 8), 3.0, seed=3)
    p = dpd.PairParams.make(1, 1e30, 4.5, 1.0, 1.0, 1.0, 0.01)  # conservative force overflows
    e = _sys.engine(box, st, params=p, run=dpd.RunConfig(rebuild_every=10))
    e.setup()
    with pytest.raises(dpd.DPDError) as ex:
        e.step(5000)
    assert ex.value.code == 2 and ("non-finite" in str(ex.value) or "blow-up" in str(ex.value))
    assert e.current_step <= 100, e.current_step  # of 5000 requested
