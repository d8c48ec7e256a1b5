"""Device observables: the velocity-profile
accumulator, the pair-distance histogram behind g(r), and the statistical
acceptance runs they exist for (ideal-gas g(r), steady double-Poiseuille
viscosity)."""
import numpy as np
import pytest

import paper_1311_0402_b200 as dpd
from paper_1311_0402_b200.observables import (estimate_viscosity, radial_distribution,
                                              velocity_profile)
import dpdsys as _sys

pytestmark = pytest.mark.gpu


def engine_with_velocity(L, vfun, seed=3):
    box, obox, st = _sys.fluid(L, 3.0, seed=seed)
    st = list(st)
    st[3], st[4], st[5] = vfun(st[0], st[1], st[2])
    return _sys.engine(box, st), st


def test_profile_uniform_and_zero_flow():
    """uniform flow v = c -> every bin c; zero velocity -> 0."""
    for c in (0.375, 0.0):
        e, st = engine_with_velocity((10, 8, 12), lambda x, y, z: (np.full_like(x, c), 0 * y, 0 * z))
        e.profile_reset(12, 2, 0)
        e.profile_sample()
        e.profile_sample()
        sv, cnt, ns = e.profile()
        p = velocity_profile(sv, cnt, ns, 0.0, 12.0)
        assert ns == 2 and int(cnt.sum()) == 2 * len(st[0])
        assert np.array_equal(p.mean_v, np.full(12, c))


def test_profile_recovers_synthetic_field():
    """v_d(z) = sin(2 pi z / L) sampled at the particle positions is
    recovered slab by slab (to the 2^-24 fixed-point resolution)."""
    Lz = 16.0
    e, st = engine_with_velocity((6, 6, Lz), lambda x, y, z: (np.sin(2 * np.pi * z / Lz), 0 * y, 0 * z))
    e.profile_reset(32, 2, 0)
    e.profile_sample()
    sv, cnt, ns = e.profile()
    z, vx = st[2], st[3]
    b = np.minimum((z / (Lz / 32)).astype(int), 31)
    ref_s = np.bincount(b, weights=vx, minlength=32)
    ref_c = np.bincount(b, minlength=32)
    assert np.array_equal(cnt.astype(np.int64), ref_c)
    assert np.abs(sv - ref_s).max() <= ref_c.max() * 2.0 ** -24
    p = velocity_profile(sv, cnt, ns, 0.0, Lz)
    # slab means track the field within the binning error (|dv/dz| * w / 2)
    assert np.abs(p.mean_v - np.sin(2 * np.pi * p.centers / Lz)).max() < 2 * np.pi / Lz * (Lz / 32) / 2 + 0.05


def rdf_reference(st, L, rmax, nbins):
    """The device's arithmetic in numpy: pos4 = float32(x - box centre), fp32
    minimum image (|d| >= L/2), r2 = (dx^2 + dy^2) + dz^2, IEEE sqrt, bin =
    floor(r * float32(nbins / rmax))."""
    from scipy.spatial import cKDTree
    L = np.asarray(L, np.float64)
    P = np.stack(st[:3], 1)
    pairs = cKDTree(P, boxsize=L).query_pairs(rmax + 1e-3, output_type="ndarray")
    f = (P - L / 2).astype(np.float32)
    d = f[pairs[:, 0]] - f[pairs[:, 1]]
    Lf, Hf = L.astype(np.float32), (0.5 * L).astype(np.float32)
    d = np.where(d >= Hf, d - Lf, np.where(d < -Hf, d + Lf, d)).astype(np.float32)
    r2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]).astype(np.float32) + (d[:, 2] * d[:, 2]).astype(np.float32)
    fb = (np.sqrt(r2.astype(np.float32)) * np.float32(nbins / rmax)).astype(np.float32)
    fb = fb[fb < nbins]
    return np.bincount(fb.astype(np.int64), minlength=nbins)


@pytest.mark.parametrize("pipeline", [False, True])
def test_rdf_counts_exact(pipeline):
    """The pair histogram over the table equals a brute-force count of the
    same fp32 distances, every pair once -- for the reference split layout
    (stage API) and the range-walk layout of the step pipeline."""
    L = (20.0, 18.0, 16.0)
    box, obox, st = _sys.fluid(L, 3.0, seed=12)
    e = _sys.engine(box, st)
    if pipeline:
        e.setup()
    else:
        e.reorder_particles()
        e.build_neighbor_table()
    s = e.download()
    h = e.rdf_counts(65, 1.3)
    ref = rdf_reference([s.coord[0], s.coord[1], s.coord[2]], L, 1.3, 65)
    assert np.array_equal(h.astype(np.int64), ref)


def test_rdf_ideal_gas_is_flat():
    """a = 0 (no conservative force): uniformly placed particles have g(r) = 1
    within counting noise (98,304 particles, bins of 0.1)."""
    L = (32.0, 32.0, 32.0)
    box, obox, st = _sys.fluid(L, 3.0, seed=2)
    e = _sys.engine(box, st, params=dpd.PairParams(a=np.array([0.0])))
    e.setup()
    r, g = radial_distribution(e.rdf_counts(13, 1.3), 1.3, len(st[0]), 32.0 ** 3)
    assert np.abs(g[2:] - 1).max() < 0.02, g


def test_steady_double_poiseuille_viscosity():
    """SPEC S:649/S:678 (paper section 4.2): steady double Poiseuille flow with
    sigma = 4.5, rho = 6, kT = 0.5, dt = 0.001, g = 0.055, a = 0 in a 12 x 32 x 8
    box (the paper's 12 x 8 x 8 channel, 4x wider along the neutral y axis for
    4x the samples; drive x, profile and partition along z); the parabolic fit
    of the folded profile gives the viscosity, paper 2.089 +- 0.009.  The
    estimate of one run scatters by ~0.02 (seeds 7-14: 2.009-2.090, mean
    2.062), so the acceptance window [2.02, 2.16] is applied to the mean of
    three independent runs."""
    mus = []
    for seed in (7, 8, 9):
        L = (12.0, 32.0, 8.0)
        box, obox, st = _sys.fluid(L, 6.0, seed=seed, kbt=0.5)
        gamma = 4.5 ** 2 / (2 * 0.5)
        p = dpd.PairParams.make(1, 0.0, gamma, 0.5, 1.0, 1.0, 0.001)
        run = dpd.RunConfig(body_force=0.055, drive_axis=0, partition_axis=2)
        e = _sys.engine(box, st, params=p, run=run)
        e.setup()
        e.step(60000)  # ~1.3 viscous times d^2 / nu to steady state
        e.profile_reset(32, 2, 0)
        for _ in range(600):
            e.step(100)
            e.profile_sample()
        sv, cnt, ns = e.profile()
        prof = velocity_profile(sv, cnt, ns, 0.0, 8.0, fold=True)
        mu, se, rel = estimate_viscosity(prof.centers - 4.0, -prof.mean_v, 0.055, 6.0, 4.0)
        mus.append(mu)
    assert 2.02 <= float(np.mean(mus)) <= 2.16, mus


def poiseuille_engine(L, rho, a, sigma, kbt, dt, g, seed):
    box, obox, st = _sys.fluid(L, rho, seed=seed, kbt=kbt)
    p = dpd.PairParams.make(1, a, sigma ** 2 / (2 * kbt), kbt, 1.0, 1.0, dt)
    run = dpd.RunConfig(body_force=g, drive_axis=0, partition_axis=2)
    e = _sys.engine(box, st, params=p, run=run)
    e.setup()
    return e


def test_transient_poiseuille_matches_eq9():
    """SPEC invariant: start-up of the double Poiseuille flow
    with the paper's transient parameters (rho = 5, a = 15, sigma = 3, kT = 1,
    dt = 0.01, g = 0.055) in a 20 x 8 x 40 box (32,000 particles); the folded
    profile, averaged over t +- 0.5, deviates from Eq. (9) by <= 7% (L2) at
    t = 100, 200, 500.  nu = mu / rho from the steady fit of the same
    parameters on a 12 x 8 x 8 box (SPEC design decision)."""
    from paper_1311_0402_b200.observables import analytic_transient_profile
    g, rho = 0.055, 5.0
    s = poiseuille_engine((12.0, 8.0, 8.0), rho, 15.0, 3.0, 1.0, 0.01, g, seed=21)
    s.step(20000)
    s.profile_reset(32, 2, 0)
    for _ in range(400):
        s.step(50)
        s.profile_sample()
    prof = velocity_profile(*s.profile(), 0.0, 8.0, fold=True)
    mu, se, rel = estimate_viscosity(prof.centers - 4.0, -prof.mean_v, g, rho, 4.0)
    nu = mu / rho
    e = poiseuille_engine((20.0, 8.0, 40.0), rho, 15.0, 3.0, 1.0, 0.01, g, seed=22)
    devs = []
    t_now = 0
    for T in (100, 200, 500):
        e.step(int(round((T - 0.5) / 0.01)) - t_now)
        e.profile_reset(40, 2, 0)
        for _ in range(100):
            e.step(1)
            e.profile_sample()
        t_now = int(round((T + 0.5) / 0.01))
        p = velocity_profile(*e.profile(), 0.0, 40.0, fold=True)
        u_meas = -p.mean_v  # upper half carries the -g flow
        u_ref = analytic_transient_profile(p.centers - 30.0, float(T), g, 20.0, nu)
        devs.append(np.linalg.norm(u_meas - u_ref) / np.linalg.norm(u_ref))
    assert max(devs) <= 0.07, (mu, devs)
