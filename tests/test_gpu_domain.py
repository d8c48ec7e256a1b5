"""Brick decomposition: bricks of one box driven by
the in-process group and by the torch.distributed transport reproduce the
single-domain engine -- bitwise with one brick, within the force tolerance
(1e-5 relative L2) with 2..8 bricks -- and conserve every particle across
migration."""
import os

import numpy as np
import pytest

import paper_1311_0402_b200 as dpd
from paper_1311_0402_b200 import domain as D
import dpdsys as _sys

pytestmark = pytest.mark.gpu

REL_L2 = 1e-5


def by_tag(s):
    o = np.argsort(s.tag)
    return o


def single(box, st, run, params=None, steps=0):
    e = _sys.engine(box, st, params=params, run=run)
    e.setup()
    if steps:
        e.step(steps)
    return e


def group(box, st, run, dims, params=None, steps=0):
    g = D.BrickGroup(box, params or dpd.PairParams(), run, dims, capacity=len(st[0]))
    g.upload(dpd.ParticleStore.from_arrays(*st))
    g.setup()
    if steps:
        g.step(steps)
    return g


def test_one_brick_group_is_bitwise_single_domain():
    """dims (1,1,1): the brick protocol (migrate plan, 32-bit key sort,
    walk build) is the single-domain step, bit for bit, across rebuilds."""
    box, obox, st = _sys.fluid((10, 10, 10), 3.0, seed=5)
    run = dpd.RunConfig(rebuild_every=4)
    e = single(box, st, run, steps=13)
    g = group(box, st, run, (1, 1, 1), steps=13)
    a, b = e.download(), g.download()
    oa = np.argsort(a.tag)
    for k in range(3):
        assert np.array_equal(a.coord[k][oa], b.coord[k])
        assert np.array_equal(a.veloc[k][oa], b.veloc[k])
        assert np.array_equal(a.force[k][oa], b.force[k])
    assert g.current_step == e.current_step == 13


@pytest.mark.parametrize("dims,per", [((2, 2, 2), (1, 1, 1)), ((2, 1, 1), (1, 1, 1)),
                                      ((3, 2, 1), (1, 1, 1)), ((2, 2, 1), (0, 1, 1))])
def test_setup_forces_match_single_domain(dims, per):
    L = (12.0, 12.0, 12.0) if dims != (3, 2, 1) else (12.0, 9.0, 8.0)
    box, obox, st = _sys.fluid(L, 3.0, per, seed=7)
    run = dpd.RunConfig(rebuild_every=5)
    e = single(box, st, run)
    g = group(box, st, run, dims)
    a, b = e.download(), g.download()
    oa = np.argsort(a.tag)
    assert np.array_equal(a.tag[oa], b.tag)
    Fa = np.stack([f[oa] for f in a.force], 1)
    Fb = np.stack(b.force, 1)
    rel = np.linalg.norm(Fa - Fb) / np.linalg.norm(Fa)
    assert rel <= REL_L2, rel
    # every brick holds ghosts from each neighbor; none when nothing neighbors
    gc = g.ghost_counts()
    assert all(c > 0 for c in gc)
    g.close()


def test_ghost_count_matches_geometry():
    """Border determination (Alg. 6): the ghosts a brick receives are exactly
    the neighbors' locals within r_c + skin of its slab (periodic images)."""
    box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=8)
    run = dpd.RunConfig()
    g = group(box, st, run, (2, 2, 2))
    cut = 1.0 + run.skin
    x = np.stack(st[:3], 1)
    for q, b in enumerate(g.bricks):
        lo, hi, _, _ = b.domain_info()
        lo, hi = np.array(lo), np.array(hi)
        want = 0
        # every particle image (27 shifts) outside the slab but within cut
        for sx in (-12, 0, 12):
            for sy in (-12, 0, 12):
                for sz in (-12, 0, 12):
                    y = x + np.array([sx, sy, sz])
                    inside = ((y >= lo) & (y < hi)).all(1)
                    near = ((y >= lo - cut) & (y < hi + cut)).all(1)
                    want += int((near & ~inside).sum())
        # a particle sent across a face sits within cut of it: half-open edges
        # differ from the open count only on exact ties (measure zero)
        assert b.ghost_count == want, (q, b.ghost_count, want)
    g.close()


@pytest.mark.parametrize("dims,per,wall", [((2, 2, 2), (1, 1, 1), (0, 0, 0)),
                                           ((2, 1, 2), (0, 1, 1), (1, 0, 0))])
def test_run_conserves_particles_and_temperature(dims, per, wall):
    """30 steps with rebuilds every 3: migrants move between bricks, no tag is
    lost or duplicated, everyone sits in its own slab, and the thermostat
    holds kbT like the single-domain run (C1)."""
    box, obox, st = _sys.fluid((12, 12, 12), 3.0, per, seed=9, wall=wall)
    run = dpd.RunConfig(rebuild_every=3)
    g = group(box, st, run, dims, steps=30)
    n0 = len(st[0])
    assert g.n == n0
    s = g.download()
    assert np.array_equal(s.tag, np.sort(st[6]))
    moved = 0
    b0 = D.brick_of(st[:3], box, dims)
    idx = np.argsort(st[6])
    for q, b in enumerate(g.bricks):
        lo, hi, _, c = b.domain_info()
        p = b.download()
        for k in range(3):
            assert (p.coord[k] >= lo[k]).all() and (p.coord[k] < hi[k]).all()
        at = idx[np.searchsorted(st[6][idx], p.tag)]
        moved += int((~(b0[at] == np.array(c)).all(1)).sum())
    assert moved > 0  # migration really happened
    t = g.thermo()
    e = single(box, st, run, steps=30)
    te = e.thermo()
    assert abs(t["kbt"] - te["kbt"]) < 0.05
    assert np.abs(np.array(t["momentum"]) / n0).max() < 0.05
    g.close()


@pytest.mark.parametrize("dims", [(2, 2, 2), (2, 1, 1)])
def test_trajectory_matches_single_domain_without_noise(dims):
    """Ghost updates, rebuilds and migration over 7 steps track the single
    domain.  The random force is switched off (kbT = 0, sigma = 0): with it,
    the 1e-7 force differences of the brick-centred fp32 coordinates flip a
    few velocity-signature bits after the first half kick (signatures read
    the top mantissa bits, inc/rng.hpp:43-45), which reseeds those pairs --
    the same divergence two runs of the reference on different brick
    layouts have."""
    box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=11)
    p = dpd.PairParams.make(1, 25.0, 4.5, 0.0, 1.0, 1.0, 0.01)
    run = dpd.RunConfig(rebuild_every=3)
    e = single(box, st, run, params=p)
    g = group(box, st, run, dims, params=p)
    for s in range(1, 8):
        e.step(1)
        g.step(1)
        a, b = e.download(), g.download()
        oa = np.argsort(a.tag)
        assert np.array_equal(a.tag[oa], b.tag)
        for k in range(3):  # between rebuilds a brick defers the periodic wrap
            d = a.coord[k][oa] - b.coord[k]
            assert np.abs(d - 12.0 * np.round(d / 12.0)).max() < 1e-6, s
        Fa = np.stack([f[oa] for f in a.force], 1)
        Fb = np.stack(b.force, 1)
        rel = np.linalg.norm(Fa - Fb) / np.linalg.norm(Fa)
        # 1e-7 differences grow slowly through the dissipative coupling;
        # a wrong ghost or a missed wrap shows up as ~1e-2
        assert rel <= (2 * REL_L2 if s == 1 else 1e-4), (s, rel)
    g.close()


@pytest.mark.parametrize("L,dims", [((40, 24, 24), (2, 1, 1)), ((36, 36, 36), (2, 2, 2)),
                                    ((14, 13, 12), (3, 2, 1))])
def test_overlapped_halo_update_is_bitwise_blocking(monkeypatch, L, dims):
    """Between rebuilds the ghost update runs on a halo stream while the
    interior force blocks (no ghost partner, flagged by the range builder)
    compute; the boundary blocks wait for the ghosts.  Same forces and
    trajectory bit for bit as the blocking update (DPDB_OVERLAP=0)."""
    box, obox, st = _sys.fluid(L, 3.0, seed=41)
    run = dpd.RunConfig(rebuild_every=4)
    out = []
    for ov in ("1", "0"):
        monkeypatch.setenv("DPDB_OVERLAP", ov)
        g = group(box, st, run, dims)
        g.step(9)
        if ov == "1" and L[0] >= 36:  # bricks large enough to have interior blocks
            split = [b.block_split() for b in g.bricks]
            assert all(ni < nb for nb, ni in split) and sum(ni for _, ni in split) > 0, split
        out.append(g.download())
        g.close()
    a, b = out
    assert np.array_equal(a.tag, b.tag)
    for u, w in zip(a.coord + a.veloc + a.force, b.coord + b.veloc + b.force):
        assert np.array_equal(u, w)


@pytest.mark.parametrize("L,dims", [((40, 24, 24), (2, 1, 1)), ((36, 36, 36), (2, 2, 2)),
                                    ((14, 13, 12), (3, 2, 1)), ((24, 24, 24), (2, 2, 1))])
def test_put_halo_update_is_bitwise_pack_copy_unpack(monkeypatch, L, dims):
    """The ghost update as one k_put per sender (straight into the receivers'
    ghost slots, Alg. 6) equals the pack -> peer copy -> unpack update bit
    for bit: forces, positions, velocities, thermo records, across rebuilds
    (the receiver slots and send lists change) and fused / unfused steps."""
    box, obox, st = _sys.fluid(L, 3.0, seed=43)
    run = dpd.RunConfig(rebuild_every=4)
    out = []
    for put in ("1", "0"):
        monkeypatch.setenv("DPDB_PUT", put)
        g = group(box, st, run, dims)
        rec = g.step_thermo(11)
        out.append((g.download(), rec))
        g.close()
    (a, ra), (b, rb) = out
    assert np.array_equal(a.tag, b.tag)
    for u, w in zip(a.coord + a.veloc + a.force, b.coord + b.veloc + b.force):
        assert np.array_equal(u, w)
    for k in ra:
        assert np.array_equal(ra[k], rb[k])


@pytest.mark.parametrize("dims", [(2, 1, 1), (2, 2, 2)])
def test_group_step_thermo_records(dims):
    """dpdb_group_step_thermo: per-step thermo of a brick run reduced on the
    devices (bricks combined in brick order) == the per-step group thermo;
    the trajectory equals plain group steps bit for bit."""
    box, obox, st = _sys.fluid((14, 13, 12), 3.0, seed=47)
    run = dpd.RunConfig(rebuild_every=4)
    a = group(box, st, run, dims)
    ref = []
    for _ in range(9):
        a.step(1)
        ref.append(a.thermo())
    b = group(box, st, run, dims)
    rec = b.step_thermo(9)
    assert list(rec["step"]) == list(range(1, 10))
    n = len(st[0])
    for k, t in enumerate(ref):
        assert abs(rec["kbt"][k] - t["kbt"]) <= 1e-12 * t["kbt"]
        assert np.allclose(rec["momentum"][k], t["momentum"], rtol=0, atol=1e-9 * n)
    sa, sb = a.download(), b.download()
    for u, w in zip(sa.coord + sa.veloc + sa.force, sb.coord + sb.veloc + sb.force):
        assert np.array_equal(u, w)
    a.close()
    b.close()


def test_ghosts_are_shifted_copies_of_their_owners():
    """After setup, after ghost updates and after a rebuild every ghost
    holds its owner's x (+ a periodic image shift) and v exactly."""
    box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=12)
    run = dpd.RunConfig(rebuild_every=2)
    g = group(box, st, run, (2, 2, 2))
    for s in range(4):
        b = g.download()
        idx = {int(t): i for i, t in enumerate(b.tag)}
        # ghosts were refreshed before the forces; the owners' phase-2 kick
        # after them changes v only, so positions must agree exactly (up to
        # the rounding of the fp64 image shift)
        for br in g.bricks:
            gx, gv, gt = br.ghosts()
            assert len(gt) > 0
            at = np.array([idx[int(t)] for t in gt], np.int64)
            for k in range(3):
                d = gx[k] - b.coord[k][at]
                img = np.round(d / 12.0)
                assert np.isin(img, (-1, 0, 1)).all()
                assert np.abs(d - 12.0 * img).max() <= 4e-15, s
                assert np.array_equal(d[img == 0], np.zeros((img == 0).sum()))
        g.step(1)
    g.close()


def test_device_neighbor_table_matches_host():
    import ctypes as C
    from paper_1311_0402_b200._lib import lib
    box = dpd.SimBox((0.0, 0.0, 0.0), (12.0, 9.0, 9.0), (True, False, True))
    dims = (3, 2, 2)
    g = D.BrickGroup(box, dpd.PairParams(), dpd.RunConfig(), dims, capacity=64)
    for q, b in enumerate(g.bricks):
        lo, hi, d, c = b.domain_info()
        assert d == dims and c == D.coords_of(q, dims)
        assert (lo, hi) == D.slab_bounds(box, dims, c)
        for dr in range(26):
            nb = np.zeros(3, np.int32)
            rc = lib().dpdb_md_neighbor(b.h, dr, nb.ctypes.data)
            want = D.neighbor(dims, c, box.periodic, dr)
            assert (rc == 0) == (want is not None)
            if want is not None:
                assert tuple(nb) == want
    g.close()


def test_bad_domain_config():
    box, obox, st = _sys.fluid((4, 4, 4), 3.0, seed=1)
    with pytest.raises(dpd.DPDError) as ex:  # slab thinner than r_c + skin
        D.BrickGroup(box, dpd.PairParams(), dpd.RunConfig(), (4, 1, 1), capacity=100)
    assert ex.value.code == 1
    with pytest.raises(dpd.DPDError):
        dpd.Engine(box, dpd.PairParams(), dpd.RunConfig(), 10, 0, (2, 1, 1), (2, 0, 0))


def _dist_worker(rank, world, port, dims, steps, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=13)
        run = dpd.RunConfig(rebuild_every=4)
        b = D.DistBrick(box, dpd.PairParams(), run, dims, capacity=len(st[0]), device=0)
        b.upload_global(dpd.ParticleStore.from_arrays(*st))
        b.setup()
        b.step(steps)
        s = b.download_global()
        t = b.thermo()
        if rank == 0:
            np.savez(out, tag=s.tag, x=np.stack(s.coord, 1), v=np.stack(s.veloc, 1),
                     f=np.stack(s.force, 1), kbt=t["kbt"])
    finally:
        dist.destroy_process_group()


def test_distributed_bricks_match_group(tmp_path):
    """Two ranks on one GPU over gloo (host-staged HaloExchange) run the same
    decomposition as the in-process group, bit for bit."""
    import torch.multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dims, steps = (2, 1, 1), 9
    out = str(tmp_path / "dist.npz")
    mp.start_processes(_dist_worker, args=(2, port, dims, steps, out), nprocs=2, join=True,
                       start_method="spawn")
    r = np.load(out)
    box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=13)
    g = group(box, st, dpd.RunConfig(rebuild_every=4), dims, steps=steps)
    s = g.download()
    assert np.array_equal(r["tag"], s.tag)
    assert np.array_equal(r["x"], np.stack(s.coord, 1))
    assert np.array_equal(r["v"], np.stack(s.veloc, 1))
    assert np.array_equal(r["f"], np.stack(s.force, 1))


def _nccl_worker(rank, world, port, dims, steps, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=13)
        run = dpd.RunConfig(rebuild_every=4)
        b = D.NcclBrick(box, dpd.PairParams(), run, dims, capacity=len(st[0]), device=0)
        b.upload_global(dpd.ParticleStore.from_arrays(*st))
        b.setup()
        b.step(steps)
        rec = b.step_thermo(2)
        ms, stage_ms, launches = b.step_timed(1, stages=True)
        launches = int(launches[5])
        assert abs(stage_ms[5] - ms) < 1e-6 and stage_ms[3] > 0
        s = b.download_global()
        t = b.thermo()
        if rank == 0:
            np.savez(out, tag=s.tag, x=np.stack(s.coord, 1), v=np.stack(s.veloc, 1),
                     f=np.stack(s.force, 1), kbt=t["kbt"], n=t["n"], ms=ms, launches=launches,
                     rec_step=rec["step"], rec_kbt=rec["kbt"], rec_mom=rec["momentum"])
        b.close()
    finally:
        dist.destroy_process_group()


def test_nccl_brick_single_rank_matches_group(tmp_path):
    """The engine's NCCL step loop (dlopen'ed NCCL, C++ driver) on one rank
    reproduces the in-process group bit for bit.  (NCCL cannot put two
    ranks on one GPU; the multi-rank exchange order is covered by the gloo
    tests of the same protocol.)"""
    import torch.multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "nccl.npz")
    mp.start_processes(_nccl_worker, args=(1, port, (1, 1, 1), 9, out), nprocs=1, join=True,
                       start_method="spawn")
    r = np.load(out)
    box, obox, st = _sys.fluid((12, 12, 12), 3.0, seed=13)
    g = group(box, st, dpd.RunConfig(rebuild_every=4), (1, 1, 1), steps=12)
    s = g.download()
    assert np.array_equal(r["tag"], s.tag)
    assert np.array_equal(r["x"], np.stack(s.coord, 1))
    assert np.array_equal(r["f"], np.stack(s.force, 1))
    t = g.thermo()
    assert abs(float(r["kbt"]) - t["kbt"]) < 1e-12 and int(r["n"]) == len(st[0])
    assert float(r["ms"]) > 0 and int(r["launches"]) > 0
    # dpdb_dist_step_thermo records of steps 10, 11 == the group's records
    g2 = group(box, st, dpd.RunConfig(rebuild_every=4), (1, 1, 1), steps=9)
    rg = g2.step_thermo(2)
    assert list(r["rec_step"]) == [10, 11] == list(rg["step"])
    assert np.allclose(r["rec_kbt"], rg["kbt"], rtol=1e-14, atol=0)
    assert np.allclose(r["rec_mom"], rg["momentum"], rtol=0, atol=1e-9)
