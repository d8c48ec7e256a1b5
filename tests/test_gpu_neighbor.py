"""Device neighbor table vs the oracle's restatement of build_neighbor_table:
identical counts and identical rows (bit-exact), in the tiled split layout,
and after join / transpose (inc/neighbor_table.hpp:12-59)."""
import numpy as np
import pytest

import oracle as O
import paper_1311_0402_b200 as dpd
import dpdsys as _sys

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["range", "lane", "ballot"], autouse=True)
def builder(request, monkeypatch):
    """All device builders -- k_build_range (culled range lists, the default),
    k_build_lane (lane per row) and k_build (Alg. 3 warp ballot) -- must
    produce the reference rows."""
    monkeypatch.setenv("DPDB_BUILDER", request.param)
    return request.param


def device_table(L, rho, periodic, seed, maxn=128, wall=(0, 0, 0)):
    box, obox, st = _sys.fluid(L, rho, periodic, seed, wall=wall)
    e = _sys.engine(box, st, run=dpd.RunConfig(max_neighbors=maxn))
    e.reorder_particles()
    e.build_neighbor_table()
    return e, obox, st


def oracle_table(obox, st, maxn):
    g, order, perm, s = _sys.oracle_sorted(obox, st)
    E, core, skin = g.neighbor_table(s[0], s[1], s[2], s[6], 1.0, 0.3, maxn, nthreads=8)
    return E, core, skin, s


def assert_same(e, E, core, skin, maxn):
    t = e.neighbor_table()
    assert t.tiled and not t.joined
    n = t.n_rows
    assert np.array_equal(t.core_count, core[:n]) and np.array_equal(t.skin_count, skin[:n])
    rows = t.rows()
    Eo = np.zeros_like(rows)
    cidx = np.arange(maxn)[None, :]
    mc = cidx < core[:n, None]
    ms = cidx >= (maxn - skin[:n, None])
    Eo[:n][mc] = E[:n][mc]
    Eo[:n][ms] = E[:n][ms]
    assert np.array_equal(rows, Eo)
    return t


@pytest.mark.parametrize("L,rho,per,maxn", [
    ((32, 32, 32), 3, (1, 1, 1), 128),      # C1
    ((10.0, 7.3, 5.1), 3, (1, 0, 1), 128),  # anisotropic, one non-periodic axis
    ((6.0, 6.0, 6.0), 6, (0, 0, 0), 128),   # fully non-periodic
    ((4.0, 4.0, 4.0), 50, (1, 1, 1), 640),  # dense, 3 cells per axis (wrap everywhere)
    ((3.0, 3.0, 3.0), 3, (1, 1, 1), 128),   # 2 cells per axis
    ((9.1, 9.1, 9.1), 3, (1, 1, 1), 64),    # ncell 7: interior-cell min-image skip
])
def test_table_bitexact(L, rho, per, maxn):
    e, obox, st = device_table(L, rho, per, 3, maxn)
    E, core, skin, s = oracle_table(obox, st, maxn)
    t = assert_same(e, E, core, skin, maxn)
    # structural invariants: ascending, no self, symmetric
    rows = t.rows()
    n = t.n_rows
    for i in range(0, n, max(1, n // 500)):
        c = rows[i, : t.core_count[i]].astype(np.int64)
        sk = rows[i, maxn - t.skin_count[i]:][::-1].astype(np.int64)
        assert np.all(np.diff(c) > 0) and np.all(np.diff(sk) > 0)
        assert i not in c and i not in sk
        for j in np.concatenate([c, sk])[:5]:
            cj = rows[j, : t.core_count[j]]
            sj = rows[j, maxn - t.skin_count[j]:]
            assert i in cj or i in sj


def test_rebuild_is_stable_and_deterministic():
    e, obox, st = device_table((12, 12, 12), 3, (1, 1, 1), 8)
    t1 = e.neighbor_table()
    e.build_neighbor_table()
    t2 = e.neighbor_table()
    assert np.array_equal(t1.entries, t2.entries) and np.array_equal(t1.core_count, t2.core_count)


def test_join_and_transpose_device():
    maxn = 64
    e, obox, st = device_table((8, 8, 8), 3, (1, 1, 1), 4, maxn)
    t = e.neighbor_table()
    split_rows = t.rows()
    e.join_core_skin()
    tj = e.neighbor_table()
    assert tj.joined and tj.tiled
    rj = tj.rows()
    for i in range(t.n_rows):
        nc, ns = t.core_count[i], t.skin_count[i]
        expect = np.concatenate([split_rows[i, :nc], split_rows[i, maxn - ns:][::-1]])
        assert np.array_equal(rj[i, : nc + ns], expect)
        if ns:
            assert tj.skin_at(i, 0) == expect[nc] and tj.core_at(i, 0) == expect[0]
    e.tile_transpose()
    tu = e.neighbor_table()
    assert not tu.tiled and tu.joined
    assert np.array_equal(tu.rows(), rj)
    e.tile_transpose()
    assert e.neighbor_table().tiled


def test_pipeline_walk_layout_exports_reference_rows():
    """dpdb_setup builds the force-walk layout (half-list order); the export
    restores the reference's joined ascending rows exactly."""
    maxn = 128
    box, obox, st = _sys.fluid((14, 14, 14), 3.0, seed=9)
    e = _sys.engine(box, st)
    e.setup()
    f_walk = np.stack(e.download().force, 1)
    t = e.neighbor_table()
    assert t.joined and t.tiled
    E, core, skin, s = oracle_table(obox, st, maxn)
    assert np.array_equal(t.core_count, core[: t.n_rows]) and np.array_equal(t.skin_count, skin[: t.n_rows])
    for i in range(t.n_rows):
        assert np.array_equal(t.core_row(i), E[i, : core[i]])
        assert np.array_equal(t.skin_row(i), E[i, maxn - skin[i]:][::-1])
    # forces from the restored layout (WALK=false path) equal the walk-layout forces
    e.compute_forces(0)
    f_joined = np.stack(e.download().force, 1)
    assert np.array_equal(f_walk, f_joined)


@pytest.mark.parametrize("rho", [3.0, 6.5])
def test_pipeline_walk_layout_dense_tiles(rho, monkeypatch):
    """At rho 6.5 a tile's flat list (~1,200 items) exceeds the range
    builder's shared-memory staging (928 words), so the builder falls back to
    row order for those tiles; rows still export exactly, and the run equals
    the all-row-order one (DPDB_BUCKET=0) bit for bit."""
    maxn = 128
    box, obox, st = _sys.fluid((9.5, 9.5, 9.5), rho, seed=13)
    E, core, skin, s = oracle_table(obox, st, maxn)
    out = []
    for b in ("1", "0"):
        monkeypatch.setenv("DPDB_BUCKET", b)
        e = _sys.engine(box, st)
        e.setup()
        t = e.neighbor_table()
        assert np.array_equal(t.core_count, core[: t.n_rows]) and np.array_equal(t.skin_count, skin[: t.n_rows])
        for i in range(t.n_rows):
            assert np.array_equal(t.core_row(i), E[i, : core[i]])
            assert np.array_equal(t.skin_row(i), E[i, maxn - skin[i]:][::-1])
        e.close()
        e = _sys.engine(box, st)
        e.setup()
        e.step(12)
        out.append(e.download())
        e.close()
    for u, w in zip(out[0].coord + out[0].veloc + out[0].force, out[1].coord + out[1].veloc + out[1].force):
        assert np.array_equal(u, w)


def test_overflow_is_physics_error():
    box, obox, st = _sys.fluid((4.0, 4.0, 4.0), 50, seed=3)
    e = _sys.engine(box, st, run=dpd.RunConfig(max_neighbors=128))
    e.reorder_particles()
    with pytest.raises(dpd.DPDError) as ex:
        e.build_neighbor_table()
    assert ex.value.code == 2 and "overflow" in str(ex.value)


def test_two_particle_examples():
    for d, expect in [(0.5, (1, 0)), (1.2, (0, 1)), (1.3 + 1e-5, (0, 0))]:
        box = dpd.SimBox((0, 0, 0), (4.0, 4.0, 4.0), (False,) * 3)
        e = dpd.Engine(box, dpd.PairParams(), dpd.RunConfig(max_neighbors=32), capacity=2)
        z = np.ones(2)
        e.upload(dpd.ParticleStore.from_arrays([1.0, 1.0 + d], z, z, z * 0, z * 0, z * 0, [1, 2]))
        e.reorder_particles()
        e.build_neighbor_table()
        t = e.neighbor_table()
        assert (int(t.core_count[0]), int(t.skin_count[0])) == expect
        assert (int(t.core_count[1]), int(t.skin_count[1])) == expect


def test_builders_give_identical_runs(monkeypatch):
    """The step pipeline with either builder (different walk layouts) gives
    bit-identical trajectories: same pair sets, order-free fixed-point sums."""
    box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=17)
    out = {}
    for b in ("range", "lane", "ballot"):
        monkeypatch.setenv("DPDB_BUILDER", b)
        e = _sys.engine(box, st, run=dpd.RunConfig(rebuild_every=5))
        e.setup()
        e.step(17)
        out[b] = e.download()
    for b in ("lane", "ballot"):
        for k in range(3):
            assert np.array_equal(out["range"].coord[k], out[b].coord[k])
            assert np.array_equal(out["range"].force[k], out[b].force[k])
