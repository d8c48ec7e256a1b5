"""Vesicle observable (P:362-374 spontaneous vesicle formation; S:692 cluster
trace): aggregate_shape classifies synthetic aggregates -- a closed hollow
shell is a vesicle, a solid ball a micelle, a flat patch a bilayer, a shell
with a large hole not closed -- including aggregates wrapped across the
periodic boundary; cluster_members returns the beads of the largest cluster."""
import numpy as np

import paper_1311_0402_b200 as dpd
from paper_1311_0402_b200.observables import aggregate_shape
from paper_1311_0402_b200.scenario import cluster_members, largest_cluster


def shell(n, R, t, rng, cap=None):
    u = rng.normal(size=(n, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    if cap is not None:  # remove the cap around +z beyond cos(theta) > cap
        u = u[u[:, 2] < cap]
    r = R + rng.uniform(-t / 2, t / 2, len(u))
    return u * r[:, None]


def test_shapes():
    rng = np.random.default_rng(0)
    box = dpd.SimBox((0.0, 0.0, 0.0), (60.0, 60.0, 60.0))
    c = np.array([30.0, 30.0, 30.0])
    ves = aggregate_shape(shell(6000, 9.0, 1.6, rng) + c, box)
    assert ves.kind == "vesicle" and ves.hollowness < 0.1 and ves.closure > 0.95, ves
    ball = rng.uniform(-1, 1, size=(20000, 3))
    ball = ball[np.linalg.norm(ball, axis=1) < 1] * 6.0
    mic = aggregate_shape(ball + c, box)
    assert mic.kind == "micelle" and mic.hollowness > 0.7, mic
    patch = np.stack([rng.uniform(-10, 10, 4000), rng.uniform(-10, 10, 4000), rng.uniform(-0.8, 0.8, 4000)], 1)
    bil = aggregate_shape(patch + c, box)
    assert bil.kind == "bilayer", bil
    cup = aggregate_shape(shell(6000, 9.0, 1.6, rng, cap=0.3) + c, box)
    assert cup.kind != "vesicle" and cup.closure < 0.9, cup


def test_shell_across_the_periodic_boundary():
    rng = np.random.default_rng(1)
    box = dpd.SimBox((0.0, 0.0, 0.0), (40.0, 40.0, 40.0))
    X = np.mod(shell(6000, 8.0, 1.6, rng) + np.array([1.0, 39.0, 20.0]), 40.0)
    s = aggregate_shape(X, box)
    assert s.kind == "vesicle" and abs(s.radius_of_gyration - 8.0) < 0.5, s


def test_cluster_members_indexes_the_largest_cluster():
    rng = np.random.default_rng(2)
    box = dpd.SimBox((0.0, 0.0, 0.0), (40.0, 40.0, 40.0))
    a = shell(3000, 6.0, 1.0, rng) + 20.0
    b = rng.uniform(0, 40, size=(200, 3))  # sparse gas of the same species
    X = np.concatenate([a, b])
    sp = np.ones(len(X), np.uint8)
    mol = np.arange(len(X)) // 4 + 1
    beads, mols, idx = cluster_members(X.T, sp, mol, box, [1], rc=1.0)
    assert beads == len(idx) and np.all(idx[: min(len(idx), 10)] < 3000)
    assert (beads, mols) == largest_cluster(X.T, sp, mol, box, [1], rc=1.0)
    assert aggregate_shape(X[idx], box).kind == "vesicle"
