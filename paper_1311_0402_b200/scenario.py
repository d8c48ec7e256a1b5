"""Scenario files and the runner around the engine.

parse_config(path) -> Scenario reads the flat sectioned key = value grammar
(the reference ships no config format; SPEC design decision "flat sectioned
key-value text grammar"), validating every key; Scenario.engine() creates the
device context and fills it with init_random on the device; run() executes
Alg. 1 with per-step thermo and optional profile sampling.  The paper's
parameter sets ship as configs/*.cfg.

Grammar: `[section]` lines, `key = value` lines, `#` comments.  Vectors are
whitespace separated.  Species-pair overrides are `a.X.Y = v` / `gamma.X.Y = v`
(symmetric) on top of the scalar `a` / `gamma`.

  [box]     lo (0 0 0), hi*, periodic (1 1 1), wall (0 0 0)
  [fluid]   density* or n*, kbt*, seed (1), species (S)
  [pair]    a*, sigma* or gamma*, r_c (1), s (1), a.X.Y, gamma.X.Y
  [run]     dt*, steps*, rebuild_every (10), skin (0.3), body_force (0),
            drive_axis (0), partition_axis (2), max_neighbors (128),
            wall_mode (specular | bounce_back)
  [chains]  fraction*, sequence*, r0 (0.38), k (80), solvent (first species),
            bond (harmonic | fene: FENE with maximum extension fene_r0),
            angle_k, angle_theta0 (degrees; harmonic angles along the chains)
            -- FENE and angles go beyond the reference (unpinned)
  [profile] bins (50), axis (2), every (100), start (0)
(* required; chains/profile sections optional)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import DPDError
from .engine import Engine, PairParams, RunConfig, SimBox

_KEYS = {
    "box": {"lo", "hi", "periodic", "wall"},
    "fluid": {"density", "n", "kbt", "seed", "species"},
    "pair": {"a", "sigma", "gamma", "r_c", "s"},
    "run": {"dt", "steps", "rebuild_every", "skin", "body_force", "drive_axis", "partition_axis",
            "max_neighbors", "wall_mode"},
    "chains": {"fraction", "sequence", "r0", "k", "solvent", "bond", "fene_r0", "angle_k",
               "angle_theta0"},
    "profile": {"bins", "axis", "every", "start"},
}
_REQUIRED = [("box", "hi"), ("fluid", "kbt"), ("pair", "a"), ("run", "dt"), ("run", "steps")]


@dataclass
class Scenario:
    box: SimBox
    n: int
    kbt: float
    seed: int
    species: list
    params: PairParams
    run: RunConfig
    steps: int
    chains: dict | None = None
    profile: dict | None = None
    source: str = ""
    raw: dict = field(default_factory=dict)

    @property
    def n_chains(self):
        if not self.chains:
            return 0
        return int(round(self.chains["fraction"] * self.n)) // len(self.chains["sequence"])

    def engine(self, device: int = 0, capacity: int | None = None) -> Engine:
        """Device context with init_random done on the GPU."""
        e = Engine(self.box, self.params, self.run, capacity=capacity or self.n, device=device)
        if self.chains:
            seq = [self.species.index(c) for c in self.chains["sequence"]]
            e.init_random(self.n, self.kbt, self.seed, self.n_chains, seq,
                          self.species.index(self.chains["solvent"]), self.chains["r0"],
                          self.chains["k"])
            c, m = self.chains, len(seq)
            first = np.arange(self.n_chains) * m + 1  # tags of bead 0
            if c["bond"] == "fene":
                ti = (first[:, None] + np.arange(m - 1)[None, :]).ravel()
                e.set_bonds(ti, ti + 1, c["k"], c["fene_r0"], style=Engine.BOND_FENE)
            if c["angle_k"] > 0 and m >= 3:
                ta = (first[:, None] + np.arange(m - 2)[None, :]).ravel()
                e.set_angles(ta, ta + 1, ta + 2, c["angle_k"], np.deg2rad(c["angle_theta0"]))
        else:
            e.init_random(self.n, self.kbt, self.seed)
        return e


def _floats(v, n, what):
    parts = v.split()
    if len(parts) != n:
        raise DPDError(1, f"config: {what} needs {n} values, got {len(parts)}")
    try:
        return tuple(float(p) for p in parts)
    except ValueError:
        raise DPDError(1, f"config: {what}: not a number: {v!r}") from None


def _num(v, what, cast=float):
    try:
        return cast(float(v)) if cast is int else cast(v)
    except ValueError:
        raise DPDError(1, f"config: {what}: not a number: {v!r}") from None


def parse_text(text: str, source: str = "<string>") -> Scenario:
    raw: dict = {}
    sec = None
    for ln, line in enumerate(text.splitlines(), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if line.startswith("[") and line.endswith("]"):
            sec = line[1:-1].strip()
            if sec not in _KEYS:
                raise DPDError(1, f"config {source}:{ln}: unknown section [{sec}]")
            raw.setdefault(sec, {})
            continue
        if "=" not in line or sec is None:
            raise DPDError(1, f"config {source}:{ln}: expected 'key = value' inside a [section]")
        k, v = (t.strip() for t in line.split("=", 1))
        base = k.split(".", 1)[0]
        pair_override = sec == "pair" and base in ("a", "gamma") and k.count(".") == 2
        if k not in _KEYS[sec] and not pair_override:
            raise DPDError(1, f"config {source}:{ln}: unknown key {sec}.{k}")
        if k in raw[sec]:
            raise DPDError(1, f"config {source}:{ln}: duplicate key {sec}.{k}")
        raw[sec][k] = v
    missing = [f"{s}.{k}" for s, k in _REQUIRED if k not in raw.get(s, {})]
    if "density" not in raw.get("fluid", {}) and "n" not in raw.get("fluid", {}):
        missing.append("fluid.density (or fluid.n)")
    if "sigma" not in raw.get("pair", {}) and "gamma" not in raw.get("pair", {}):
        missing.append("pair.sigma (or pair.gamma)")
    if "chains" in raw:
        missing += [f"chains.{k}" for k in ("fraction", "sequence") if k not in raw["chains"]]
    if missing:
        raise DPDError(1, "config: missing required keys: " + ", ".join(missing))

    b, f, p, r = raw["box"], raw["fluid"], raw["pair"], raw["run"]
    lo = _floats(b.get("lo", "0 0 0"), 3, "box.lo")
    hi = _floats(b["hi"], 3, "box.hi")
    per = tuple(bool(int(x)) for x in _floats(b.get("periodic", "1 1 1"), 3, "box.periodic"))
    wall = tuple(bool(int(x)) for x in _floats(b.get("wall", "0 0 0"), 3, "box.wall"))
    if any(h <= l for l, h in zip(lo, hi)):
        raise DPDError(1, "config: box.hi must exceed box.lo on every axis")
    box = SimBox(lo, hi, per, wall)
    vol = box.volume()
    if "n" in f:
        n = _num(f["n"], "fluid.n", int)
    else:
        rho = _num(f["density"], "fluid.density")
        if rho <= 0:
            raise DPDError(1, "config: fluid.density must be positive")
        n = int(round(rho * vol))
    if n <= 0:
        raise DPDError(1, "config: empty system (round(density * volume) = 0)")
    kbt = _num(f["kbt"], "fluid.kbt")
    if kbt < 0:
        raise DPDError(1, "config: fluid.kbt must be >= 0")
    species = f.get("species", "S").split()
    if len(set(species)) != len(species) or not 1 <= len(species) <= 4:
        raise DPDError(1, "config: fluid.species: 1..4 distinct names")
    ns = len(species)
    a = np.full((ns, ns), _num(p["a"], "pair.a"))
    if "gamma" in p:
        gamma = np.full((ns, ns), _num(p["gamma"], "pair.gamma"))
    else:
        sig = _num(p["sigma"], "pair.sigma")
        if kbt <= 0:
            raise DPDError(1, "config: pair.sigma needs kbt > 0 (gamma = sigma^2 / (2 kbt))")
        gamma = np.full((ns, ns), sig * sig / (2 * kbt))
    if "gamma" in p and "sigma" in p:
        sig = _num(p["sigma"], "pair.sigma")
        if not math.isclose(sig * sig, 2 * gamma[0, 0] * kbt, rel_tol=1e-9):
            raise DPDError(1, "config: pair.sigma and pair.gamma violate sigma^2 = 2 gamma kbt")
    for k, v in p.items():
        if k.count(".") != 2:
            continue
        what, x, y = k.split(".")
        if x not in species or y not in species:
            raise DPDError(1, f"config: pair.{k}: unknown species")
        m = a if what == "a" else gamma
        m[species.index(x), species.index(y)] = m[species.index(y), species.index(x)] = _num(v, f"pair.{k}")
    dt = _num(r["dt"], "run.dt")
    if dt <= 0:
        raise DPDError(1, "config: run.dt must be positive")
    params = PairParams.make(ns, a.ravel(), gamma.ravel(), kbt, _num(p.get("s", "1"), "pair.s"),
                             _num(p.get("r_c", "1"), "pair.r_c"), dt)
    run = RunConfig(rebuild_every=_num(r.get("rebuild_every", "10"), "run.rebuild_every", int),
                    skin=_num(r.get("skin", "0.3"), "run.skin"),
                    body_force=_num(r.get("body_force", "0"), "run.body_force"),
                    drive_axis=_num(r.get("drive_axis", "0"), "run.drive_axis", int),
                    partition_axis=_num(r.get("partition_axis", "2"), "run.partition_axis", int),
                    seed=_num(f.get("seed", "1"), "fluid.seed", int),
                    max_neighbors=_num(r.get("max_neighbors", "128"), "run.max_neighbors", int),
                    wall_mode={"specular": 0, "bounce_back": 1}.get(r.get("wall_mode", "specular"), -1))
    if run.wall_mode < 0:
        raise DPDError(1, "config: run.wall_mode must be specular or bounce_back")
    if run.rebuild_every < 1 or run.skin < 0:
        raise DPDError(1, "config: run.rebuild_every >= 1 and run.skin >= 0")
    steps = _num(r["steps"], "run.steps", int)
    if steps < 0:
        raise DPDError(1, "config: run.steps must be >= 0")
    chains = None
    if "chains" in raw:
        c = raw["chains"]
        seq = c["sequence"].strip()
        if any(ch not in species for ch in seq):
            raise DPDError(1, "config: chains.sequence uses an unknown species")
        frac = _num(c["fraction"], "chains.fraction")
        if not 0 < frac <= 1:
            raise DPDError(1, "config: chains.fraction must be in (0, 1]")
        chains = dict(fraction=frac, sequence=seq, r0=_num(c.get("r0", "0.38"), "chains.r0"),
                      k=_num(c.get("k", "80"), "chains.k"), solvent=c.get("solvent", species[0]),
                      bond=c.get("bond", "harmonic"),
                      fene_r0=_num(c.get("fene_r0", "1.5"), "chains.fene_r0"),
                      angle_k=_num(c.get("angle_k", "0"), "chains.angle_k"),
                      angle_theta0=_num(c.get("angle_theta0", "180"), "chains.angle_theta0"))
        if chains["bond"] not in ("harmonic", "fene"):
            raise DPDError(1, "config: chains.bond must be harmonic or fene")
        if chains["bond"] == "fene" and not chains["fene_r0"] > chains["r0"]:
            raise DPDError(1, "config: chains.fene_r0 must exceed the initial bond length r0")
        if chains["solvent"] not in species:
            raise DPDError(1, "config: chains.solvent is not a species")
    profile = None
    if "profile" in raw:
        q = raw["profile"]
        profile = dict(bins=_num(q.get("bins", "50"), "profile.bins", int),
                       axis=_num(q.get("axis", "2"), "profile.axis", int),
                       every=_num(q.get("every", "100"), "profile.every", int),
                       start=_num(q.get("start", "0"), "profile.start", int))
    return Scenario(box, n, kbt, run.seed, species, params, run, steps, chains, profile, source, raw)


def parse_config(path: str) -> Scenario:
    """parse + validate a scenario file."""
    with open(path) as fh:
        return parse_text(fh.read(), path)


def largest_cluster(coords, species, molecule, box: SimBox, members, rc: float = 1.0):
    """S:692 cluster analysis: union-find over the beads of the `members`
    species closer than rc (minimum image on periodic axes); returns (beads,
    molecules) of the largest cluster."""
    beads, mols, _ = cluster_members(coords, species, molecule, box, members, rc)
    return beads, mols


def cluster_members(coords, species, molecule, box: SimBox, members, rc: float = 1.0):
    """largest_cluster, plus the particle indices of that cluster's beads."""
    from scipy.spatial import cKDTree

    sel = np.isin(species, list(members))
    idx = np.flatnonzero(sel)
    if not len(idx):
        return 0, 0, idx
    P = np.stack([np.asarray(c)[idx] - box.lo[k] for k, c in enumerate(coords)], 1)
    L = np.array([box.length(k) for k in range(3)])
    P = np.mod(P, L)
    tree = cKDTree(P, boxsize=np.where(np.array(box.periodic), L, 0) if all(box.periodic) else None)
    pairs = tree.query_pairs(rc, output_type="ndarray")
    parent = np.arange(len(idx))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for i, j in pairs:
        ri, rj = find(i), find(j)
        if ri != rj:
            parent[max(ri, rj)] = min(ri, rj)
    roots = np.array([find(i) for i in range(len(idx))])
    best, best_idx = (0, 0), idx[:0]
    mol = np.asarray(molecule)[idx]
    for r_ in np.unique(roots):
        m = roots == r_
        cand = (int(m.sum()), len(np.unique(mol[m])))
        if (cand[1], cand[0]) > (best[1], best[0]):
            best, best_idx = cand, idx[m]
    return best[0], best[1], best_idx
