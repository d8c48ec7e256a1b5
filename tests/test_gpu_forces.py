"""Device pair/bond/body forces vs the oracle.

Tolerances (north_star: "per-step forces match within 1e-5 relative in fp32"),
both against the SPEC oracle (fp64 coordinates, fp64 math):
        ||F_gpu - F_ref||_2 / ||F_ref||_2 <= 1e-5
        max_i |F_gpu,i - F_ref,i| / rms|F_ref| <= 1e-5   (every particle)
The device pair vector comes from the int32 fixed-point frame (posq) or, for
r < 0.05, from the fp64 state; the pair math is fp32 with the MUFU-based
Box-Muller (|xi - xi_ref| < 4e-6) and 2^-18 fixed-point accumulation.
"""
import numpy as np
import pytest

import oracle as O
import paper_1311_0402_b200 as dpd
import dpdsys as _sys

pytestmark = pytest.mark.gpu

REL_L2 = 1e-5
REL_MAX = 1e-5  # per particle, relative to rms |F|


def device_forces(box, st, step, params=None, run=None):
    e = _sys.engine(box, st, params=params, run=run)
    e.reorder_particles()
    e.build_neighbor_table()
    f = e.compute_forces(step)
    s = e.download()
    return e, np.stack(f, 1), s


def oracle_forces(e, s, obox, params, step, seed=1, paper=False):
    t = e.neighbor_table()
    sig = O.signatures(s.tag, *s.veloc)
    assert np.array_equal(sig, s.signature)  # device signatures are bit-exact
    x = [np.ascontiguousarray(a) for a in s.coord]
    v = [np.ascontiguousarray(a) for a in s.veloc]
    box = obox
    if paper:
        ctr = [(obox.lo[k] + obox.hi[k]) / 2 for k in range(3)]
        x = [(x[k] - ctr[k]).astype(np.float32).astype(np.float64) for k in range(3)]
        v = [a.astype(np.float32).astype(np.float64) for a in v]
        box = O.make_box([obox.lo[k] - ctr[k] for k in range(3)],
                         [obox.hi[k] - ctr[k] for k in range(3)],
                         tuple(obox.periodic))
    mix = O.lib().orc_step_mix(seed, step)
    sp = np.ascontiguousarray(s.species, np.uint8) if params.n_species > 1 else None
    f = O.compute_forces(_sys.oparams(params), box, *x, *v, s.tag, sig, mix, t.entries,
                         t.core_count, t.skin_count, t.max_neighbors, tiled=t.tiled,
                         joined=t.joined, species=sp, nthreads=8)
    return np.stack(f, 1)


def test_forces_multispecies_vesicle_matrix():
    """Three species with the paper's repulsion matrix:
    a(A,A)=a(A,S)=a(S,S)=a(B,B)=15, a(A,B)=a(B,S)=120, gamma 4.5 (sigma 3)."""
    box, obox, st = _sys.fluid((10, 10, 10), 5.0, seed=31)
    n = len(st[0])
    species = np.random.default_rng(1).integers(0, 3, n).astype(np.uint8)  # A=0 B=1 S=2
    a = np.array([[15, 120, 15], [120, 15, 120], [15, 120, 15]], np.float64).reshape(-1)
    p = dpd.PairParams.make(3, a, 4.5, 1.0, 1.0, 1.0, 0.01)
    e = dpd.Engine(box, p, dpd.RunConfig(), capacity=n)
    e.upload(dpd.ParticleStore.from_arrays(*st, species=species))
    e.reorder_particles()
    e.build_neighbor_table()
    Fg = np.stack(e.compute_forces(4), 1)
    s = e.download()
    F = oracle_forces(e, s, obox, p, 4)
    assert np.linalg.norm(Fg - F) / np.linalg.norm(F) <= REL_L2
    assert np.abs(Fg.sum(0)).max() <= 1e-3
    e.setup()
    e.step(50)
    assert np.isfinite(e.thermo()["kbt"])


@pytest.mark.parametrize("L,per,step", [((32, 32, 32), (1, 1, 1), 0),
                                        ((32, 32, 32), (1, 1, 1), 123),
                                        ((10.0, 7.3, 5.1), (1, 0, 1), 5),
                                        ((6.0, 6.0, 6.0), (0, 0, 0), 9)])
def test_forces_vs_oracle(L, per, step):
    box, obox, st = _sys.fluid(L, 3.0, per, seed=11)
    p = dpd.PairParams()
    e, Fg, s = device_forces(box, st, step, p)
    Fspec = oracle_forces(e, s, obox, p, step)
    rms = np.sqrt((Fspec ** 2).sum(1).mean())
    l2 = np.linalg.norm(Fg - Fspec) / np.linalg.norm(Fspec)
    mx = np.sqrt(((Fg - Fspec) ** 2).sum(1)).max() / rms
    print(f"rel L2 vs spec {l2:.2e}; max_i |dF_i|/rms {mx:.2e}")
    assert l2 <= REL_L2
    assert mx <= REL_MAX
    # momentum conservation of the full-list kernel (pair symmetry of xi)
    assert np.abs(Fg.sum(0)).max() <= 1e-5 * rms * np.sqrt(len(Fg))


@pytest.mark.parametrize("s_exp", [2.0, 0.5])
def test_forces_weight_exponent(s_exp):
    box, obox, st = _sys.fluid((8, 8, 8), 3.0, seed=4)
    p = dpd.PairParams(s=s_exp)
    e, Fg, s = device_forces(box, st, 3, p)
    Fspec = oracle_forces(e, s, obox, p, 3)
    assert np.linalg.norm(Fg - Fspec) / np.linalg.norm(Fspec) <= REL_L2


def test_body_force_double_poiseuille():
    box, obox, st = _sys.fluid((8, 8, 8), 3.0, seed=5)
    p = dpd.PairParams(a=np.array([0.0]))
    run = dpd.RunConfig(body_force=0.055, drive_axis=2, partition_axis=0)
    e, Fg, s = device_forces(box, st, 1, p, run)
    F0 = oracle_forces(e, s, obox, p, 1)
    g = np.where(s.coord[0] < 4.0, 0.055, -0.055)
    assert np.linalg.norm(Fg[:, 2] - (F0[:, 2] + g)) / np.linalg.norm(F0) <= REL_L2
    assert np.allclose(Fg[:, :2], F0[:, :2], atol=1e-4)


def test_bonds_harmonic():
    box, obox, st = _sys.fluid((8, 8, 8), 3.0, seed=6)
    n = len(st[0])
    ti = np.arange(1, n, 8, dtype=np.uint32)
    tj = ti + 1
    p = dpd.PairParams()
    e = _sys.engine(box, st)
    e.set_bonds(ti, tj, 80.0, 0.38)
    e.reorder_particles()
    e.build_neighbor_table()
    Fg = np.stack(e.compute_forces(2), 1)
    s = e.download()
    F = oracle_forces(e, s, obox, p, 2)
    iot = np.full(n + 1, np.iinfo(np.uint32).max, np.uint32)
    iot[s.tag] = np.arange(n, dtype=np.uint32)
    bonds = (O.Bond * len(ti))(*[O.Bond(int(a), int(b), 80.0, 0.38) for a, b in zip(ti, tj)])
    fx, fy, fz = (np.ascontiguousarray(F[:, k]) for k in range(3))
    O.check(O.lib().orc_bond_forces(obox, len(ti), bonds, n + 1, iot, *[np.ascontiguousarray(a) for a in s.coord],
                                    fx, fy, fz))
    Fo = np.stack([fx, fy, fz], 1)
    assert np.linalg.norm(Fg - Fo) / np.linalg.norm(Fo) <= REL_L2
    # missing endpoint -> physics error
    e.set_bonds([1], [n + 5], 80.0, 0.38)
    with pytest.raises(dpd.DPDError) as ex:
        e.compute_forces(2)
    assert ex.value.code == 2


def test_isolated_and_pair():
    box = dpd.SimBox((0, 0, 0), (6.0, 6.0, 6.0), (True,) * 3)
    e = dpd.Engine(box, dpd.PairParams(), dpd.RunConfig(), capacity=3)
    z = np.array([1.0, 1.5, 4.0])
    e.upload(dpd.ParticleStore.from_arrays(z, [1.0, 1.0, 4.0], [1.0, 1.0, 4.0], [0.3, -0.2, 1.0],
                                           [0.0, 0.1, 0.0], [0.0, 0.0, 0.0], [1, 2, 3]))
    e.reorder_particles()
    e.build_neighbor_table()
    f = np.stack(e.compute_forces(0), 1)
    s = e.download()
    iso = np.nonzero(s.tag == 3)[0][0]
    assert np.all(f[iso] == 0)
    a, b = np.nonzero(s.tag == 1)[0][0], np.nonzero(s.tag == 2)[0][0]
    assert np.array_equal(f[a], -f[b])  # S:441, bitwise


def test_coincident_particles_error():
    box = dpd.SimBox((0, 0, 0), (6.0, 6.0, 6.0), (True,) * 3)
    e = dpd.Engine(box, dpd.PairParams(), dpd.RunConfig(), capacity=2)
    one = np.ones(2)
    e.upload(dpd.ParticleStore.from_arrays(one, one, one, one * 0, one * 0, one * 0, [1, 2]))
    e.reorder_particles()
    e.build_neighbor_table()
    with pytest.raises(dpd.DPDError) as ex:
        e.compute_forces(0)
    assert ex.value.code == 2


def _bonded_reference(X, L, bonds, angles):
    """fp64 forces of FENE / harmonic bonds and harmonic angles from the
    standard formulas (tags 1..n are indices + 1): -grad U."""
    F = np.zeros_like(X)

    def mi(d):
        return d - L * np.round(d / L)

    for (i, j, K, r0, style) in bonds:
        d = mi(X[i] - X[j])
        r = np.linalg.norm(d)
        c = -K / (1 - (r / r0) ** 2) if style == 1 else -K * (r - r0) / r
        F[i] += c * d
        F[j] -= c * d
    for (a, b, c_, K, t0) in angles:
        r1, r2 = mi(X[a] - X[b]), mi(X[c_] - X[b])
        l1, l2 = np.linalg.norm(r1), np.linalg.norm(r2)
        cs = np.dot(r1, r2) / (l1 * l2)
        th = np.arccos(np.clip(cs, -1, 1))
        g = K * (th - t0) / np.sin(th)
        fa = g * (r2 / (l1 * l2) - cs * r1 / l1 ** 2)
        fc = g * (r1 / (l1 * l2) - cs * r2 / l2 ** 2)
        F[a] += fa
        F[c_] += fc
        F[b] -= fa + fc
    return F


@pytest.mark.parametrize("pipeline", [False, True])
def test_fene_bonds_and_angles(pipeline):
    """North-star bonded terms beyond the reference (unpinned, standard
    formulas): FENE bonds and harmonic angles along 6-bead chains, no pair
    forces (a = gamma = 0), device vs fp64 -grad U; momentum conserved; the
    fused pipeline (epilogue) and the stage API (k_bonds) agree."""
    L = 9.0
    rng = np.random.default_rng(4)
    nch, m = 40, 6
    n = nch * m + 200
    X = rng.uniform(0, L, (n, 3))
    for c in range(nch):  # random walks with step 0.9 (inside R0 = 1.5)
        for b in range(1, m):
            u = rng.normal(size=3)
            X[c * m + b] = (X[c * m + b - 1] + 0.9 * u / np.linalg.norm(u)) % L
    bonds, angles = [], []
    for c in range(nch):
        for b in range(m - 1):
            i = c * m + b
            bonds.append((i, i + 1, 30.0, 1.5, 1))
        for b in range(m - 2):
            i = c * m + b
            angles.append((i, i + 1, i + 2, 5.0, 2.0))
    box = dpd.SimBox((0.0, 0.0, 0.0), (L, L, L))
    p = dpd.PairParams.make(1, 0.0, 0.0, 0.0, 1.0, 1.0, 0.01)
    z = np.zeros(n)
    e = dpd.Engine(box, p, dpd.RunConfig(), capacity=n)
    e.upload(dpd.ParticleStore.from_arrays(X[:, 0], X[:, 1], X[:, 2], z, z, z, np.arange(1, n + 1)))
    bi = np.array([b[0] + 1 for b in bonds]); bj = np.array([b[1] + 1 for b in bonds])
    e.set_bonds(bi, bj, 30.0, 1.5, style=1)
    ai, ab, ac = (np.array([a[q] + 1 for a in angles]) for q in range(3))
    e.set_angles(ai, ab, ac, 5.0, 2.0)
    if pipeline:
        e.setup()
        s = e.download()
    else:
        e.reorder_particles()
        e.build_neighbor_table()
        e.compute_forces(0)
        s = e.download()
    o = np.argsort(s.tag)
    Fg = np.stack(s.force, 1)[o]
    Fr = _bonded_reference(X, L, bonds, angles)
    assert np.linalg.norm(Fg - Fr) / np.linalg.norm(Fr) < 1e-5
    assert np.abs(Fg.sum(0)).max() < 1e-3 * np.abs(Fg).max()
    # FENE beyond R0 is a physics error
    e.set_bonds([1], [2], 30.0, 0.1, style=1)
    with pytest.raises(dpd.DPDError) as ex:
        e.compute_forces(0)
    assert ex.value.code == 2 and "FENE" in str(ex.value)
