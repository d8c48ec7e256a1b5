"""Host-side analysis of the device observables.

The device accumulates the raw sums (Engine.profile_*, Engine.rdf_counts); this
module turns them into the reference's ProfileSample / viscosity / Eq. (9)
quantities.  Pure numpy: no kernels here.

  velocity_profile            S:650-657  (slab means, double-Poiseuille fold)
  estimate_viscosity          S:658-665  (least-squares u(z) = g rho z (d - z) / (2 mu))
  analytic_transient_profile  S:666-672  (Eq. 9)
  radial_distribution         g(r) from the pair-distance histogram
  aggregate_shape             vesicle / micelle / bilayer classification of an
                              amphiphile aggregate
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


def _unwrap_cluster(P, L, periodic, rc):
    """Make a cluster spanning periodic images contiguous: breadth-first over
    the contact graph (pairs within rc), each bead placed at the minimum image
    of the neighbour it was reached from."""
    from scipy.spatial import cKDTree

    n = len(P)
    Lp = np.where(periodic, L, 0.0)
    Q = np.mod(P, np.where(periodic, L, np.inf)) if np.any(periodic) else P.copy()
    tree = cKDTree(Q, boxsize=np.where(periodic, L, 0) if np.all(periodic) else None)
    nbrs = tree.query_ball_point(Q, rc)
    out = Q.copy()
    seen = np.zeros(n, bool)
    for s in range(n):
        if seen[s]:
            continue
        seen[s] = True
        stack = [s]
        while stack:
            i = stack.pop()
            for j in nbrs[i]:
                if seen[j]:
                    continue
                d = Q[j] - Q[i]
                d -= Lp * np.round(d / np.where(Lp > 0, Lp, 1.0))
                out[j] = out[i] + d
                seen[j] = True
                stack.append(j)
    return out


@dataclass
class AggregateShape:
    """Shape of one aggregate (e.g. the tail beads of the largest cluster)."""
    n: int
    radius_of_gyration: float
    asphericity: float      # 0 sphere .. 1 rod (gyration-tensor eigenvalues)
    hollowness: float       # bead density within 0.4 Rg of the centre relative to a
                            # uniform solid ball of the same Rg (1 solid .. 0 hollow)
    closure: float          # fraction of 162 directions from the centre that hit the aggregate
    kind: str               # "vesicle" | "micelle" | "bilayer" | "irregular"


def aggregate_shape(coords, box, rc: float = 1.0) -> AggregateShape:
    """Vesicle observable ("spontaneous vesicle formation"; S:692
    cluster trace).  coords: (n, 3) bead positions of ONE aggregate (periodic
    images are joined through its contact graph).  A vesicle is a closed,
    hollow, near-spherical shell: hollowness < 0.25 (the centre is empty
    where a micelle or a solid ball is full), closure >= 0.9 (beads seen in
    almost every direction from the centre, unlike a bilayer patch or an
    open cup) and asphericity < 0.2; a micelle is closed, near-spherical and
    solid; a bilayer is flat (its smallest gyration eigenvalue < 5% of the
    largest)."""
    P = np.asarray(coords, np.float64).reshape(-1, 3)
    n = len(P)
    if n < 8:
        return AggregateShape(n, 0.0, 0.0, 1.0, 0.0, "irregular")
    L = np.array([box.length(k) for k in range(3)])
    per = np.array(box.periodic, bool)
    X = _unwrap_cluster(P - np.array(box.lo), L, per, rc)
    c = X.mean(0)
    D = X - c
    G = D.T @ D / n
    ev = np.sort(np.linalg.eigvalsh(G))
    rg = float(np.sqrt(ev.sum()))
    tr = ev.sum()
    asph = float(((ev[2] - ev[1]) ** 2 + (ev[2] - ev[0]) ** 2 + (ev[1] - ev[0]) ** 2) / (2 * tr * tr))
    r = np.linalg.norm(D, axis=1)
    # uniform solid ball with this Rg: R = Rg sqrt(5/3); fraction within a of the centre = (a/R)^3
    R = rg * np.sqrt(5.0 / 3.0)
    a = 0.4 * rg
    hollow = float((r < a).mean() / max((a / R) ** 3, 1e-12))
    # directions: a 162-vertex geodesic sphere (Fibonacci lattice)
    k = np.arange(162) + 0.5
    th = np.arccos(1 - 2 * k / 162)
    ph = np.pi * (1 + 5 ** 0.5) * k
    U = np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], 1)
    Dn = D / np.maximum(r, 1e-12)[:, None]
    cosmax = np.cos(np.deg2rad(12.0))
    closure = float(((Dn @ U.T) > cosmax).any(0).mean())
    flat = ev[0] < 0.05 * ev[2]
    if hollow < 0.25 and closure >= 0.9 and asph < 0.2:
        kind = "vesicle"
    elif flat:
        kind = "bilayer"
    elif closure >= 0.9 and asph < 0.2:
        kind = "micelle"
    else:
        kind = "irregular"
    return AggregateShape(n, rg, asph, hollow, closure, kind)
