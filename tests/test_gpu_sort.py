"""Device radix sort / two-level reorder / cell list / stencils vs the
reference's own outputs (golden) and the oracle -- bit-exact."""
import numpy as np
import pytest

import oracle as O
import paper_1311_0402_b200 as dpd
import dpdsys as _sys

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["s0", "s1", "s4", "s1000", "s100k"])
def test_radix_golden(golden, case):
    g = golden.sort
    k = g[case + "_keys"].copy()
    v = np.arange(len(k), dtype=np.uint32)
    dpd.radix_sort(k, v, int(g[case + "_bits"][0]))
    assert np.array_equal(k, g[case + "_skeys"]) and np.array_equal(v, g[case + "_svals"])


@pytest.mark.parametrize("n,bits", [(4095, 8), (4096, 12), (4097, 16), (1_000_003, 28),
                                    (300_000, 32), (77, 4)])
def test_radix_stable_random(n, bits):
    rng = np.random.default_rng(n)
    k = rng.integers(0, 2**bits, n, dtype=np.uint64).astype(np.uint32)
    k[: n // 3] = k[0]  # heavy duplicates exercise stability
    v = rng.permutation(n).astype(np.uint32)
    order = np.argsort(k, kind="stable")
    kk, vv = k.copy(), v.copy()
    dpd.radix_sort(kk, vv, bits)
    assert np.array_equal(kk, k[order]) and np.array_equal(vv, v[order])


CASES = ["c1small", "aniso", "walled", "tiny", "dense"]


@pytest.mark.parametrize("case", CASES)
def test_reorder_golden(golden, case):
    g = golden.cells
    p = case + "_"
    L = tuple(g[p + "L"])
    per = tuple(bool(v) for v in g[p + "per"])
    box = dpd.SimBox((0.0, 0.0, 0.0), L, per)
    x, y, z, tag = g[p + "x"], g[p + "y"], g[p + "z"], g[p + "tag"]
    n = len(x)
    zeros = np.zeros(n)
    e = dpd.Engine(box, dpd.PairParams(), dpd.RunConfig(max_neighbors=640), capacity=n)
    e.upload(dpd.ParticleStore.from_arrays(x, y, z, zeros, zeros, zeros, tag))
    assert np.array_equal(e.rank_of_cell(), g[p + "rank_of_cell"])
    info = g[p + "info_i"]
    assert e.grid.key_bits == info[12] and e.n_total_cells == info[11]
    perm = e.reorder_particles()
    assert np.array_equal(perm, g[p + "perm"])
    s = e.download()
    order = np.empty(n, np.uint32)
    order[perm] = np.arange(n, dtype=np.uint32)
    assert np.array_equal(s.coord[0], x[order]) and np.array_equal(s.tag, tag[order])
    assert np.array_equal(e.cell_start(), g[p + "cell_start"])
    coff, cc = e.coarse_stencil()
    assert np.array_equal(coff, g[p + "coff"]) and np.array_equal(cc, g[p + "ccells"])
    foff, fidx = e.fine_stencil()
    assert np.array_equal(foff, g[p + "foff"]) and np.array_equal(fidx, g[p + "fidx"])


def test_sort_keys_vs_oracle_c1():
    """C1 (98,304 particles, 32^3, rho=3): keys, permutation, cell list."""
    box, obox, st = _sys.fluid((32, 32, 32), 3.0, seed=1)
    e = _sys.engine(box, st)
    g = O.OGrid(obox, 1.3)
    assert np.array_equal(e.sort_keys(), g.keys(st[0], st[1], st[2]))
    order, perm = g.order(st[0], st[1], st[2], nthreads=8)
    assert np.array_equal(e.reorder_particles(), perm)
    xs = [a[order] for a in st[:3]]
    assert np.array_equal(e.cell_start(), g.cell_start(*xs))


def test_reorder_missed_migration_is_protocol_error():
    box, obox, st = _sys.fluid((8, 8, 8), 3.0, seed=2)
    st = list(st)
    st[0] = st[0].copy()
    st[0][5] = 8.5  # outside the slab
    e = _sys.engine(box, st)
    with pytest.raises(dpd.DPDError) as ex:
        e.reorder_particles()
    assert ex.value.code == 3
