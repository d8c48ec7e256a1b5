"""Host-side analysis of the observables: viscosity fit,
Eq. (9), the double-Poiseuille fold, g(r) normalisation.  CPU only."""
import numpy as np

from paper_1311_0402_b200.observables import (analytic_transient_profile, estimate_viscosity,
                                              radial_distribution, velocity_profile)


def test_viscosity_exact_parabola():
    """synthetic exact parabola with mu = 2.0 -> 2.0 within 1e-10."""
    d, g, rho = 4.0, 0.055, 6.0
    z = np.linspace(0.05, 3.95, 40)
    u = g * rho / (2 * 2.0) * z * (d - z)
    mu, se, rel = estimate_viscosity(z, u, g, rho, d)
    assert abs(mu - 2.0) <= 1e-10 and rel < 1e-12


def test_viscosity_noisy_parabola():
    """noisy parabola (1% Gaussian noise) -> mu within 2%."""
    d, g, rho = 4.0, 0.055, 6.0
    z = np.linspace(0.05, 3.95, 40)
    u = g * rho / (2 * 2.089) * z * (d - z)
    rng = np.random.default_rng(3)
    mus = [estimate_viscosity(z, u * (1 + 0.01 * rng.normal(size=z.size)), g, rho, d)[0]
           for _ in range(20)]
    assert all(abs(m - 2.089) / 2.089 < 0.02 for m in mus)


def test_eq9_limits():
    """t -> inf gives the parabola; u(+-d/2, t) = 0; u(0, 0) = 0."""
    F, d, nu = 0.055, 4.0, 0.35
    z = np.linspace(-d / 2, d / 2, 9)
    lead = F * d * d / (8 * nu)
    assert np.allclose(analytic_transient_profile(z, 1e6, F, d, nu), lead * (1 - (2 * z / d) ** 2),
                       rtol=0, atol=1e-14 * lead)
    for t in (0.0, 0.5, 5.0, 50.0):
        edge = analytic_transient_profile(np.array([-d / 2, d / 2]), t, F, d, nu)
        assert np.abs(edge).max() <= 1e-9 * lead
    assert abs(analytic_transient_profile(np.array([0.0]), 0.0, F, d, nu)[0]) <= 1e-9 * lead
    # monotone start-up at the centre line
    u = [analytic_transient_profile(np.array([0.0]), t, F, d, nu)[0] for t in (1, 5, 20, 100)]
    assert all(a < b for a, b in zip(u, u[1:])) and u[-1] < lead


def test_profile_fold():
    """Double Poiseuille: the lower half mirrors the upper half with a sign
    flip; the fold averages both onto the upper half."""
    nb, lo, hi = 8, 0.0, 8.0
    up = np.array([1.0, 2.0, 3.0, 4.0])
    sum_v = np.concatenate([-up[::-1] * 10, up * 30])
    count = np.concatenate([np.full(4, 10), np.full(4, 30)]).astype(np.uint64)
    p = velocity_profile(sum_v, count, 5, lo, hi, fold=True)
    assert np.allclose(p.centers, [4.5, 5.5, 6.5, 7.5]) and np.allclose(p.mean_v, up)
    assert list(p.count) == [40] * 4 and p.samples == 5
    q = velocity_profile(np.zeros(4), np.array([3, 0, 1, 2], np.uint64), 1, 0.0, 4.0)
    assert np.isnan(q.mean_v[1]) and q.count[1] == 0  # empty bin flagged, not an abort


def test_rdf_normalisation():
    """Uniform pair counts H = n rho / 2 * shell volume give g = 1."""
    n, vol, rmax, nb = 1000, 500.0, 1.3, 13
    edges = np.linspace(0, rmax, nb + 1)
    shell = 4 / 3 * np.pi * (edges[1:] ** 3 - edges[:-1] ** 3)
    r, g = radial_distribution(0.5 * n * (n / vol) * shell, rmax, n, vol)
    assert np.allclose(g, 1.0) and np.allclose(r, 0.5 * (edges[1:] + edges[:-1]))
