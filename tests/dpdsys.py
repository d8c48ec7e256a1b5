"""Shared builders for the parity tests: the same seeded system for the
device engine and the oracle."""
import numpy as np

import oracle as O
import paper_1311_0402_b200 as dpd


def fluid(L, rho=3.0, periodic=(1, 1, 1), seed=1, kbt=1.0, wall=(0, 0, 0)):
    """Uniform DPD fluid from the oracle's counter-based init."""
    L = tuple(float(v) for v in L)
    obox = O.make_box((0, 0, 0), L, periodic, wall)
    n = int(round(rho * L[0] * L[1] * L[2]))
    st = O.init_fluid(obox, n, kbt, seed)
    box = dpd.SimBox((0.0, 0.0, 0.0), L, tuple(bool(p) for p in periodic),
                     tuple(bool(w) for w in wall))
    return box, obox, st


def engine(box, st, params=None, run=None, capacity=None):
    params = params or dpd.PairParams()
    run = run or dpd.RunConfig()
    e = dpd.Engine(box, params, run, capacity=capacity or len(st[0]))
    e.upload(dpd.ParticleStore.from_arrays(*st))
    return e


def oparams(p: "dpd.PairParams"):
    return O.make_params(a=p.a, gamma=p.gamma, kbt=p.kbt, s=p.s, r_c=p.r_c, dt=p.dt,
                         n_species=p.n_species)


def oracle_sorted(obox, st, cell_target=1.3):
    g = O.OGrid(obox, cell_target)
    x, y, z = st[0], st[1], st[2]
    order, perm = g.order(x, y, z, nthreads=8)
    return g, order, perm, [np.ascontiguousarray(a[order]) for a in st]
