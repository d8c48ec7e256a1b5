"""The brick protocol with GhostPackets on the wire:
in-process mailboxes and the TCP socket transport between processes both
reproduce the in-process group transport bit for bit."""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

import paper_1311_0402_b200 as dpd
from paper_1311_0402_b200 import domain as D
from paper_1311_0402_b200 import wire as W
import dpdsys as _sys

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def reference(box, st, run, dims, steps):
    g = D.BrickGroup(box, dpd.PairParams(), run, dims, capacity=len(st[0]))
    g.upload(dpd.ParticleStore.from_arrays(*st))
    g.setup()
    g.step(steps)
    out = g.download()
    g.close()
    return out


def same(a, b):
    oa, ob = np.argsort(a.tag), np.argsort(b.tag)
    assert np.array_equal(a.tag[oa], b.tag[ob])
    for u, w in zip(a.coord + a.veloc + a.force, b.coord + b.veloc + b.force):
        assert np.array_equal(u[oa], w[ob])


@pytest.mark.parametrize("dims", [(2, 1, 1), (2, 2, 2)])
def test_wire_group_matches_group(dims):
    box, obox, st = _sys.fluid((14, 13, 12), 3.0, seed=43)
    run = dpd.RunConfig(rebuild_every=4)
    w = W.WireGroup(box, dpd.PairParams(), run, dims, capacity=len(st[0]))
    w.upload(dpd.ParticleStore.from_arrays(*st))
    w.setup()
    w.step(9)
    got = w.download()
    assert w.packets > 0 and w.bytes > 0
    w.close()
    same(got, reference(box, st, run, dims, 9))


def _socket_rank(rank, dims, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import dpdsys as S
    import paper_1311_0402_b200 as P
    from paper_1311_0402_b200 import wire as WW
    box, obox, st = S.fluid((14, 13, 12), 3.0, seed=43)
    b = WW.WireBrick(box, P.PairParams(), P.RunConfig(rebuild_every=4), dims, len(st[0]), rank, port)
    b.upload_global(P.ParticleStore.from_arrays(*st))
    b.setup()
    b.step(9)
    s = b.download()
    q.put((rank, [a.copy() for a in s.coord + s.veloc + s.force], s.tag.copy()))
    b.close()


def test_socket_transport_two_processes():
    dims = (2, 1, 1)
    box, obox, st = _sys.fluid((14, 13, 12), 3.0, seed=43)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 200
    ps = [ctx.Process(target=_socket_rank, args=(r, dims, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    arrs = [np.concatenate([r[1][k] for r in res]) for k in range(9)]
    tag = np.concatenate([r[2] for r in res])
    got = dpd.ParticleStore(arrs[0:3], arrs[3:6], tag, None, None, arrs[6:9])
    same(got, reference(box, st, dpd.RunConfig(rebuild_every=4), dims, 9))
