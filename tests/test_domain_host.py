"""Host logic of the brick decomposition on CPU: direction
tables, slab geometry, neighbor symmetry, particle routing, and the
torch.distributed HaloExchange at world_size 2 and 4 over gloo."""
import itertools
import os
import socket

import numpy as np
import pytest

import paper_1311_0402_b200 as dpd
from paper_1311_0402_b200 import domain as D


def test_directions_roundtrip_and_opposite():
    seen = set()
    for d in range(26):
        off = D.dir_offset(d)
        assert off != (0, 0, 0)
        assert D.dir_index(*off) == d
        assert D.dir_offset(D.opposite(d)) == tuple(-o for o in off)
        seen.add(off)
    assert len(seen) == 26
    with pytest.raises(ValueError):
        D.dir_index(0, 0, 0)


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 1, 1), (2, 2, 2), (3, 2, 1), (4, 3, 2)])
@pytest.mark.parametrize("per", [(1, 1, 1), (0, 1, 0), (0, 0, 0)])
def test_neighbor_symmetry(dims, per):
    """neighbor_b(d) = a  <=>  neighbor_a(25 - d) = b -- what lets the
    transport pair sends and receives without tags."""
    for c in itertools.product(*[range(n) for n in dims]):
        for d in range(26):
            nb = D.neighbor(dims, c, per, d)
            if nb is None:
                continue
            assert all(0 <= nb[k] < dims[k] for k in range(3))
            assert nb != c  # never a self-neighbor (one brick on an axis wraps instead)
            assert D.neighbor(dims, nb, per, D.opposite(d)) == c
            off = D.dir_offset(d)
            for k in range(3):
                if dims[k] == 1:
                    assert off[k] == 0


def test_slab_bounds_tile_the_box():
    box = dpd.SimBox((-1.0, 0.5, 0.0), (10.0, 7.3, 9.9))
    dims = (3, 2, 5)
    for k in range(3):
        edges = []
        for c in range(dims[k]):
            cc = [0, 0, 0]
            cc[k] = c
            lo, hi = D.slab_bounds(box, dims, cc)
            edges.append((lo[k], hi[k]))
        assert edges[0][0] == box.lo[k] and edges[-1][1] == box.hi[k]
        for a, b in zip(edges, edges[1:]):
            assert a[1] == b[0]


def test_brick_of_respects_half_open_slabs():
    box = dpd.SimBox((0.0, 0.0, 0.0), (10.0, 9.0, 7.0))
    dims = (3, 2, 4)
    rng = np.random.default_rng(1)
    x = [rng.uniform(box.lo[k], box.hi[k], 20000) for k in range(3)]
    # exact slab edges and their neighbors
    for k in range(3):
        for c in range(dims[k]):
            cc = [0, 0, 0]
            cc[k] = c
            lo, hi = D.slab_bounds(box, dims, cc)
            x[k][c * 3: c * 3 + 3] = [lo[k], np.nextafter(lo[k], -np.inf) if c else lo[k],
                                       np.nextafter(hi[k], -np.inf)]
    b = D.brick_of(x, box, dims)
    for i in range(len(x[0])):
        lo, hi = D.slab_bounds(box, dims, b[i])
        for k in range(3):
            assert lo[k] <= x[k][i] < hi[k] or (x[k][i] == box.hi[k])


def test_split_and_gather_roundtrip():
    box = dpd.SimBox((0.0, 0.0, 0.0), (6.0, 6.0, 6.0))
    rng = np.random.default_rng(2)
    n = 1000
    st = dpd.ParticleStore.from_arrays(*[rng.uniform(0, 6, n) for _ in range(3)],
                                       *[rng.normal(size=n) for _ in range(3)],
                                       rng.permutation(n).astype(np.uint32),
                                       species=rng.integers(0, 3, n).astype(np.uint8))
    parts = D.split_store(st, box, (2, 3, 1))
    assert sum(p.n for p in parts) == n
    for p in parts:
        p.force = [np.zeros(p.n)] * 3
        p.signature = np.zeros(p.n, np.uint32)
    g = D.gather_stores(parts)
    o = np.argsort(st.tag)
    assert np.array_equal(g.tag, st.tag[o])
    assert np.array_equal(g.coord[1], st.coord[1][o])
    assert np.array_equal(g.species, st.species[o])


def test_thermo_from_sums():
    rng = np.random.default_rng(3)
    v = rng.normal(size=(999, 3)) + 0.1
    parts = np.array_split(v, 4)
    sums = [np.concatenate([p.sum(0), [(p * p).sum()]]) for p in parts]
    t = D.thermo_from_sums(sums, len(v))
    m = v.mean(0)
    assert np.allclose(t["momentum"], v.sum(0))  # total momentum, unit masses
    assert abs(t["kbt"] - ((v - m) ** 2).sum() / (3 * len(v))) < 1e-12


REC = 16  # synthetic record: (src rank, src direction, index, magic) as u32


def _exchange_worker(rank, world, port, dims, per, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        coords = D.coords_of(rank, dims)
        x = D.HaloExchange(dims, coords, per, stage_host=True)
        for rnd in range(3):
            counts = np.zeros(26, np.int64)
            recs = []
            for d in range(26):
                if x.peer[d] is None:
                    continue
                counts[d] = (rank * 7 + d * 3 + rnd) % 5
                for i in range(counts[d]):
                    recs.append((rank, d, i, 0xC0FFEE + rnd))
            payload = np.array(recs, np.uint32).reshape(-1, 4)
            send = torch.from_numpy(payload.view(np.uint8).reshape(-1).copy())
            recv, rc = x.exchange(send, counts, REC, device="cpu")
            got = recv.numpy().view(np.uint32).reshape(-1, 4)
            at = 0
            for d in range(26):
                src = x.peer[d]
                if src is None:
                    assert rc[d] == 0
                    continue
                sd = D.opposite(d)
                want = (src * 7 + sd * 3 + rnd) % 5
                assert rc[d] == want, (rank, d, rc[d], want)
                for i in range(want):
                    assert tuple(got[at]) == (src, sd, i, 0xC0FFEE + rnd), (rank, d, i)
                    at += 1
            assert at == len(got)
        q.put((rank, "ok"))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,per", [((2, 1, 1), (1, 1, 1)), ((2, 1, 1), (0, 1, 1)),
                                      ((1, 2, 1), (1, 1, 1)), ((2, 2, 1), (1, 1, 1)),
                                      ((1, 2, 2), (1, 0, 1))])
def test_halo_exchange_gloo(dims, per):
    import torch.multiprocessing as mp
    world = dims[0] * dims[1] * dims[2]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, dims, per, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
