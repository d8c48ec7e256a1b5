"""The NCCL brick driver (NcclX, domain_host.inc) with several ranks on one
GPU: N bricks of one process, one host thread per brick, each running the
unchanged dpdb_dist_* step loop, attached to an in-process stand-in of NCCL's
grouped Send / Recv and AllGather (dpdb_nccl_mock_attach: device copies with
NCCL's per-peer ordering and completion semantics).  The NCCL call sequence
-- the 26-direction count all-gather at rebuilds, sends in ascending
direction paired with receives in ascending opposite direction (the dims = 2
periodic case where one peer is reached in several directions), the halo
update on the halo stream overlapped with the interior forces -- must give
the in-process group transport's (GroupX) trajectory bit for bit, at
2x1x1, 2x2x1 and 2x2x2 (the transport must not change results)."""
import ctypes as C
import threading

import numpy as np
import pytest

import paper_1311_0402_b200 as dpd
from paper_1311_0402_b200 import domain as D
from paper_1311_0402_b200._lib import lib
import dpdsys as _sys

pytestmark = pytest.mark.gpu


def run_threads(fns):
    errs = [None] * len(fns)

    def wrap(q):
        try:
            fns[q]()
        except Exception as ex:  # noqa: BLE001
            errs[q] = ex

    ts = [threading.Thread(target=wrap, args=(q,)) for q in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    for e in errs:
        if e is not None:
            raise e


@pytest.mark.parametrize("dims", [(2, 1, 1), (2, 2, 1), (2, 2, 2)])
def test_nccl_driver_multi_rank_equals_group(dims):
    L = (14.0, 13.0, 12.0)
    box, obox, st = _sys.fluid(L, 3.0, seed=41)
    params, run = dpd.PairParams(), dpd.RunConfig(rebuild_every=5)
    nb = dims[0] * dims[1] * dims[2]
    cap = len(st[0])
    # reference: the in-process group transport
    g = D.BrickGroup(box, params, run, dims, capacity=cap)
    g.upload(dpd.ParticleStore.from_arrays(*st))
    g.setup()
    g.step(23)  # four rebuilds, fused and overlapped steps in between
    ref = g.download()
    th_ref = g.thermo()
    g.close()
    # the NCCL driver, one thread per rank
    bricks = [D._Brick(box, params, run, cap, 0, dims, D.coords_of(q, dims)) for q in range(nb)]
    parts = D.split_store(dpd.ParticleStore.from_arrays(*st), box, dims)
    for b, p in zip(bricks, parts):
        b.upload(p)
    arr = (C.c_void_p * nb)(*[b.h for b in bricks])
    assert lib().dpdb_nccl_mock_attach(arr, nb) == 0, lib().dpdb_last_error(bricks[0].h)

    def job(b):
        def f():
            for call in (lambda: lib().dpdb_dist_setup(b.h), lambda: lib().dpdb_dist_step(b.h, 23)):
                rc = call()
                if rc:
                    raise dpd.DPDError(rc, lib().dpdb_last_error(b.h).decode())
        return f

    run_threads([job(b) for b in bricks])
    got = D.gather_stores([b.download() for b in bricks])
    th = [None] * nb

    def thermo_job(q):
        def f():
            t = D.Thermo()
            rc = lib().dpdb_dist_thermo(bricks[q].h, C.byref(t))
            if rc:
                raise dpd.DPDError(rc, lib().dpdb_last_error(bricks[q].h).decode())
            th[q] = t
        return f

    run_threads([thermo_job(q) for q in range(nb)])
    for b in bricks:
        b.close()
    oa, ob = np.argsort(ref.tag), np.argsort(got.tag)
    assert np.array_equal(ref.tag[oa], got.tag[ob])
    for u, w in zip(ref.coord + ref.veloc, got.coord + got.veloc):
        assert np.array_equal(u[oa], w[ob])
    assert all(t.kbt == th[0].kbt for t in th) and th[0].n == len(st[0])
    assert abs(th[0].kbt - th_ref["kbt"]) <= 1e-12 * th_ref["kbt"]
