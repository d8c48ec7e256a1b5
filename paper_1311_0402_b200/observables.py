"""Host-side analysis of the device observables.

The device accumulates the raw sums (Engine.profile_*, Engine.rdf_counts); this
module turns them into the reference's ProfileSample / viscosity / Eq. (9)
quantities.  Pure numpy: no kernels here.

  velocity_profile            S:650-657  (slab means, double-Poiseuille fold)
  estimate_viscosity          S:658-665  (least-squares u(z) = g rho z (d - z) / (2 mu))
  analytic_transient_profile  S:666-672  (Eq. 9)
  radial_distribution         g(r) from the pair-distance histogram
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ProfileSample:
    """time- and slab-averaged drive-axis velocity per bin."""
    centers: np.ndarray   # bin centres along the profile axis (box coordinates)
    mean_v: np.ndarray    # mean drive-axis velocity (nan where count == 0)
    count: np.ndarray     # particle-samples per bin (0 = empty, flagged, not an abort)
    samples: int


def velocity_profile(sum_v, count, samples, lo, hi, fold=False) -> ProfileSample:
    """Slab means from the device sums.  fold=True (double Poiseuille): the
    lower half is folded onto the upper half with a sign flip, the result
    spans the upper half-box (bin i of the upper half pairs with the mirror
    bin nb-1-i of the lower half)."""
    sum_v = np.asarray(sum_v, np.float64)
    count = np.asarray(count, np.float64)
    nb = len(sum_v)
    w = (hi - lo) / nb
    centers = lo + (np.arange(nb) + 0.5) * w
    if fold:
        if nb % 2:
            raise ValueError("velocity_profile: fold needs an even bin count")
        h = nb // 2
        up_s, up_c = sum_v[h:], count[h:]
        lo_s, lo_c = sum_v[:h][::-1], count[:h][::-1]
        sum_v, count = up_s - lo_s, up_c + lo_c
        centers = centers[h:]
    with np.errstate(invalid="ignore", divide="ignore"):
        mean = np.where(count > 0, sum_v / np.maximum(count, 1), np.nan)
    return ProfileSample(centers, mean, count.astype(np.uint64), int(samples))


def estimate_viscosity(z, u, g, rho, d):
    """least-squares fit of u(z) = (g rho / (2 mu)) z (d - z) over
    one half-channel of width d (z measured from the channel wall).  Returns
    (mu, standard error, relative residual)."""
    z = np.asarray(z, np.float64)
    u = np.asarray(u, np.float64)
    ok = np.isfinite(u)
    z, u = z[ok], u[ok]
    phi = z * (d - z)  # u = c phi with c = g rho / (2 mu)
    c = float(np.dot(phi, u) / np.dot(phi, phi))
    res = u - c * phi
    dof = max(len(u) - 1, 1)
    se_c = float(np.sqrt(np.dot(res, res) / dof / np.dot(phi, phi)))
    mu = g * rho / (2.0 * c)
    se_mu = mu * se_c / abs(c)
    rel = float(np.linalg.norm(res) / max(np.linalg.norm(u), 1e-300))
    return mu, se_mu, rel


def analytic_transient_profile(z, t, F, d, nu, n_terms=None):
    """Eq. (9): start-up of plane Poiseuille flow in a channel of
    width d (z in [-d/2, d/2], no slip at +-d/2) driven by F:
      u = F d^2/(8 nu) (1 - (2z/d)^2)
          - sum_n 4 (-1)^n F d^2 / (nu pi^3 (2n+1)^3) cos((2n+1) pi z / d)
                  exp(-(2n+1)^2 pi^2 nu t / d^2)
    truncated where the remainder is below 1e-12 of the leading term."""
    z = np.asarray(z, np.float64)
    lead = F * d * d / (8.0 * nu)
    u = lead * (1.0 - (2.0 * z / d) ** 2)
    c = 4.0 * F * d * d / (nu * np.pi ** 3)
    s = np.pi ** 2 * nu * t / (d * d)
    if n_terms is None:
        # remainder after N terms: sum_{k > 2N} c e^{-k^2 s} / k^3 <= c e^{-(2N+1)^2 s} / (2 (2N)^2)
        n_terms = 1
        while c * np.exp(-((2 * n_terms + 1) ** 2) * s) / (2.0 * (2 * n_terms) ** 2) >= 1e-12 * lead:
            n_terms *= 2
            if n_terms > (1 << 24):
                break
    zz = z.reshape(-1, 1)
    for n0 in range(0, int(n_terms), 65536):
        n = np.arange(n0, min(int(n_terms), n0 + 65536), dtype=np.float64)
        k = 2.0 * n + 1.0
        w = np.where(n % 2 == 0, 1.0, -1.0) * c / k ** 3 * np.exp(-(k * k) * s)
        u = u - (np.cos(zz * (k * np.pi / d)) * w).sum(axis=1).reshape(u.shape)
    return u


def radial_distribution(hist, rmax, n, volume):
    """g(r) at the bin centres from the every-pair-once histogram of n
    particles in `volume`: g = H / (n rho / 2 * shell volume)."""
    hist = np.asarray(hist, np.float64)
    nb = len(hist)
    edges = np.linspace(0.0, rmax, nb + 1)
    shell = 4.0 / 3.0 * np.pi * (edges[1:] ** 3 - edges[:-1] ** 3)
    rho = n / volume
    return 0.5 * (edges[1:] + edges[:-1]), hist / (0.5 * n * rho * shell)
