"""Brick decomposition of the DPD step (SURVEY §8 row e; spec S:539-615).

The reference's contract -- `decompose` into uniform half-open slabs
(S:554-562), `border_determination` (paper Alg. 6),
`exchange_ghosts` full / update, `migrate_strays`,
an abstract transport and the `GhostPacket` records --
is split here into

* device work per brick, in libdpdb.so (`dpdb_md_*`, include/dpdb.h): the
  migration and border masks, 26-list compaction, packing/unpacking of
  records, the one stable sort of locals + ghosts, the neighbor build and the
  forces;
* transports that only move the packed device buffers:
    - `BrickGroup`: every brick of the decomposition in this process, on one
      or several GPUs (device / NVLink peer copies inside libdpdb.so);
    - `HaloExchange` + `DistBrick`: one brick per rank over torch.distributed
      (NCCL on device buffers; gloo through host staging for CPU tests).

Directions d = 0..25 are the offsets (dx, dy, dz) in z-major order with the
centre removed; the opposite of d is 25 - d.  The brick at b receives, for
each d, the list its neighbor at b + d packed for direction 25 - d, and lays
the records out in ascending d (the receive order the ghost-update slots are
fixed to at each rebuild).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import (MD_GHOST_FULL, MD_GHOST_UPDATE, MD_MIGRANTS, NCCL_ID_BYTES, DPDError, Thermo,
                   check, lib, ptr)
from .engine import Engine, PairParams, ParticleStore, RunConfig, SimBox

N_DIRS = 26


# ------------------------------------------------------------ geometry
def dir_offset(d: int):
    """(dx, dy, dz) of direction d (z-major, centre removed)."""
    if not 0 <= d < N_DIRS:
        raise ValueError("direction out of range")
    e = d if d < 13 else d + 1
    return (e % 3 - 1, (e // 3) % 3 - 1, e // 9 - 1)


def dir_index(dx: int, dy: int, dz: int) -> int:
    e = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)
    if e == 13:
        raise ValueError("the centre is not a direction")
    return e if e < 13 else e - 1


def opposite(d: int) -> int:
    return 25 - d


def rank_of(coords, dims) -> int:
    """x-fastest linear rank of a brick."""
    return int(coords[0] + dims[0] * (coords[1] + dims[1] * coords[2]))


def coords_of(rank: int, dims):
    return (rank % dims[0], (rank // dims[0]) % dims[1], rank // (dims[0] * dims[1]))


def slab_bounds(box: SimBox, dims, coords):
    """decompose: uniform half-open slabs; the last slab ends at
    box.hi exactly.  Same arithmetic as dpdb_create."""
    lo, hi = [0.0] * 3, [0.0] * 3
    for k in range(3):
        ln = (box.hi[k] - box.lo[k]) / dims[k]
        lo[k] = box.lo[k] + coords[k] * ln
        hi[k] = box.hi[k] if coords[k] == dims[k] - 1 else box.lo[k] + (coords[k] + 1) * ln
    return tuple(lo), tuple(hi)


def neighbor(dims, coords, periodic, d):
    """Coordinates of the neighbor brick in direction d, or None (an axis
    with one brick never has a neighbor: it wraps by minimum image)."""
    off = dir_offset(d)
    nb = []
    for k in range(3):
        if off[k] == 0:
            nb.append(coords[k])
            continue
        if dims[k] == 1:
            return None
        c = coords[k] + off[k]
        if c < 0 or c >= dims[k]:
            if not periodic[k]:
                return None
            c %= dims[k]
        nb.append(c)
    return tuple(nb)


def brick_of(coord, box: SimBox, dims):
    """Brick coordinates of each particle, consistent with the device's
    half-open slab test (x >= slab_lo and x < slab_hi)."""
    out = []
    for k in range(3):
        x = np.asarray(coord[k], np.float64)
        ln = (box.hi[k] - box.lo[k]) / dims[k]
        c = np.clip(np.floor((x - box.lo[k]) / ln).astype(np.int64), 0, dims[k] - 1)
        bounds_lo = box.lo[k] + np.arange(dims[k]) * ln
        bounds_hi = np.where(np.arange(dims[k]) == dims[k] - 1, box.hi[k],
                             box.lo[k] + (np.arange(dims[k]) + 1) * ln)
        c = np.where((x < bounds_lo[c]) & (c > 0), c - 1, c)
        c = np.where((x >= bounds_hi[c]) & (c < dims[k] - 1), c + 1, c)
        out.append(c)
    return np.stack(out, 1)


def split_store(store: ParticleStore, box: SimBox, dims):
    """Scatter a global ParticleStore to the bricks (rank order)."""
    b = brick_of(store.coord, box, dims)
    r = b[:, 0] + dims[0] * (b[:, 1] + dims[1] * b[:, 2])
    parts = []
    for q in range(dims[0] * dims[1] * dims[2]):
        m = r == q
        parts.append(ParticleStore(
            [np.ascontiguousarray(a[m]) for a in store.coord],
            [np.ascontiguousarray(a[m]) for a in store.veloc],
            np.ascontiguousarray(store.tag[m]),
            None if store.species is None else np.ascontiguousarray(store.species[m]),
            None if store.molecule is None else np.ascontiguousarray(store.molecule[m])))
    return parts


def gather_stores(parts):
    """Concatenate downloaded brick stores and order them by tag."""
    tag = np.concatenate([p.tag for p in parts])
    o = np.argsort(tag, kind="stable")
    cat = lambda xs: np.concatenate(xs)[o]
    return ParticleStore([cat([p.coord[k] for p in parts]) for k in range(3)],
                         [cat([p.veloc[k] for p in parts]) for k in range(3)], tag[o],
                         cat([p.species for p in parts]), None,
                         [cat([p.force[k] for p in parts]) for k in range(3)],
                         cat([p.signature for p in parts]))


def thermo_from_sums(sums, n):
    """Global temperature/momentum from per-brick (sum v, sum |v|^2)."""
    s = np.sum(np.asarray(sums, np.float64).reshape(-1, 4), 0)
    kbt = (s[3] - float(s[:3] @ s[:3]) / n) / (3.0 * n)
    # momentum = total (unit masses), as Engine.thermo / dpdb_thermo_get
    return dict(n=int(n), kbt=float(kbt), momentum=tuple(float(v) for v in s[:3]))


class _Brick(Engine):
    """An Engine bound to one brick of a decomposition."""

    def domain_info(self):
        lo, hi = np.zeros(3), np.zeros(3)
        d, c = np.zeros(3, np.int32), np.zeros(3, np.int32)
        self._check(lib().dpdb_domain_info(self.h, ptr(lo), ptr(hi), ptr(d), ptr(c)))
        return tuple(lo), tuple(hi), tuple(int(v) for v in d), tuple(int(v) for v in c)

    @property
    def ghost_count(self):
        n = C.c_size_t()
        self._check(lib().dpdb_md_ghost_count(self.h, C.byref(n)))
        return n.value

    def block_split(self):
        """(force blocks, interior blocks) of the current table."""
        nb, ni = C.c_size_t(), C.c_size_t()
        self._check(lib().dpdb_md_block_split(self.h, C.byref(nb), C.byref(ni)))
        return nb.value, ni.value

    def ghosts(self):
        """(x[3], v[3], tag) of the ghosts this brick holds."""
        ng = self.ghost_count
        a = [np.zeros(ng) for _ in range(6)]
        tag = np.zeros(ng, np.uint32)
        self._check(lib().dpdb_md_download_ghosts(self.h, *[ptr(v) for v in a], ptr(tag)))
        return a[:3], a[3:], tag

    def sums(self):
        out = np.zeros(4)
        self._check(lib().dpdb_md_sums(self.h, ptr(out)))
        return out


# ---------------------------------------------------- in-process group
class BrickGroup:
    """All bricks of a dims[0] x dims[1] x dims[2] decomposition in this
    process.  `devices` lists the GPU of each brick (rank order); bricks on
    different GPUs exchange by cudaMemcpyPeerAsync (NVLink)."""

    def __init__(self, box: SimBox, params: PairParams, run: RunConfig | None, dims,
                 capacity: int, devices=None):
        self.box, self.params, self.run = box, params, run or RunConfig()
        self.dims = tuple(int(v) for v in dims)
        nb = self.dims[0] * self.dims[1] * self.dims[2]
        devices = list(devices) if devices is not None else [0] * nb
        if len(devices) != nb:
            raise DPDError(1, "brick group: one device per brick")
        self.bricks = [_Brick(box, params, self.run, capacity, devices[q], self.dims,
                              coords_of(q, self.dims)) for q in range(nb)]
        self._arr = (C.c_void_p * nb)(*[b.h for b in self.bricks])

    def close(self):
        for b in self.bricks:
            b.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc):
        if rc:
            msgs = [lib().dpdb_last_error(b.h).decode() for b in self.bricks]
            msg = next((m for m in msgs if m), lib().dpdb_last_error(None).decode())
            raise DPDError(rc, msg)

    def upload(self, store: ParticleStore):
        self._parts = split_store(store, self.box, self.dims)
        for b, p in zip(self.bricks, self._parts):
            b.upload(p)

    def setup(self):
        self._check(lib().dpdb_group_setup(self._arr, len(self.bricks)))

    def step(self, nsteps: int = 1):
        self._check(lib().dpdb_group_step(self._arr, len(self.bricks), int(nsteps)))

    def step_thermo(self, nsteps: int):
        """dpdb_group_step_thermo: every step's thermo line (bricks combined in
        brick order), no host sync per step."""
        k = int(nsteps)
        recs = (Thermo * max(k, 1))()
        self._check(lib().dpdb_group_step_thermo(self._arr, len(self.bricks), k, recs))
        return dict(step=np.array([recs[i].step for i in range(k)], np.int64),
                    kbt=np.array([recs[i].kbt for i in range(k)]),
                    momentum=np.array([tuple(recs[i].momentum) for i in range(k)]).reshape(k, 3))

    @property
    def n(self):
        return sum(b.n for b in self.bricks)

    def ghost_counts(self):
        return [b.ghost_count for b in self.bricks]

    def download(self) -> ParticleStore:
        return gather_stores([b.download() for b in self.bricks])

    def thermo(self):
        return thermo_from_sums([b.sums() for b in self.bricks], self.n)

    @property
    def current_step(self):
        return self.bricks[0].current_step


# ------------------------------------------- torch.distributed transport
class HaloExchange:
    """Moves packed record lists between the bricks of a torch.distributed
    job (one brick per rank, rank = rank_of(coords)).  Counts travel by one
    all-gather of 26 ints per rank; payloads by batched point-to-point ops.

    For a peer reached in several directions (dims == 2 on a periodic axis)
    the k-th send in ascending d pairs with the k-th receive in ascending
    opposite direction, which is the same list by the symmetry
    neighbor_b(d) = a  <=>  neighbor_a(25 - d) = b.
    `stage_host` copies device buffers through host memory (gloo)."""

    def __init__(self, dims, coords, periodic, group=None, stage_host=False):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.dims = tuple(dims)
        self.coords = tuple(coords)
        self.stage_host = stage_host
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world != self.dims[0] * self.dims[1] * self.dims[2]:
            raise DPDError(1, "halo exchange: world size must equal the number of bricks")
        if rank_of(self.coords, self.dims) != self.rank:
            raise DPDError(1, "halo exchange: brick coordinates do not match the rank")
        self.peer = [None] * N_DIRS
        for d in range(N_DIRS):
            nb = neighbor(self.dims, self.coords, periodic, d)
            self.peer[d] = None if nb is None else rank_of(nb, self.dims)

    def all_counts(self, counts, device):
        """[world, 26] send counts of every rank."""
        import torch
        mine = torch.as_tensor(np.asarray(counts, np.int64), device=device)
        out = torch.zeros(self.world * N_DIRS, dtype=torch.int64, device=device)
        self.dist.all_gather_into_tensor(out, mine, group=self.group)
        return out.view(self.world, N_DIRS).cpu().numpy()

    def receive_counts(self, table):
        """Per-direction receive counts from the gathered send counts."""
        rc = np.zeros(N_DIRS, np.int64)
        for d in range(N_DIRS):
            if self.peer[d] is not None:
                rc[d] = table[self.peer[d], opposite(d)]
        return rc

    def exchange(self, send, counts, rec_bytes, device=None):
        """send: uint8 tensor of the packed lists (ascending d, counts[d]
        records each).  Returns (recv uint8 tensor, receive counts[26])."""
        import torch
        device = send.device if device is None else device
        table = self.all_counts(counts, "cpu" if self.stage_host else device)
        rcnt = self.receive_counts(table)
        soff = np.concatenate([[0], np.cumsum(np.asarray(counts, np.int64))]) * rec_bytes
        roff = np.concatenate([[0], np.cumsum(rcnt)]) * rec_bytes
        recv = torch.empty(int(roff[-1]), dtype=torch.uint8, device=device)
        s_host = send.cpu() if self.stage_host else send
        r_host = torch.empty(int(roff[-1]), dtype=torch.uint8) if self.stage_host else recv
        ops = []
        P2POp, isend, irecv = self.dist.P2POp, self.dist.isend, self.dist.irecv
        for d in range(N_DIRS):  # sends: ascending d
            if self.peer[d] is not None and counts[d]:
                ops.append(P2POp(isend, s_host[int(soff[d]):int(soff[d + 1])], self.peer[d],
                                 self.group))
        for d in reversed(range(N_DIRS)):  # receives: ascending opposite direction
            if self.peer[d] is not None and rcnt[d]:
                ops.append(P2POp(irecv, r_host[int(roff[d]):int(roff[d + 1])], self.peer[d],
                                 self.group))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        if self.stage_host and len(recv):
            recv.copy_(r_host)
        return recv, rcnt


class DistBrick:
    """One brick per rank: the per-brick protocol of include/dpdb.h driven
    through a HaloExchange.  Device buffers are torch CUDA tensors on the
    brick's device (plumbing only; the records are packed and unpacked by
    the engine's kernels)."""

    def __init__(self, box: SimBox, params: PairParams, run: RunConfig | None, dims, capacity,
                 device=0, group=None, stage_host=None):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.dims = tuple(int(v) for v in dims)
        rank = dist.get_rank(group)
        self.coords = coords_of(rank, self.dims)
        self.run = run or RunConfig()
        self.brick = _Brick(box, params, self.run, capacity, device, self.dims, self.coords)
        self.box = box
        if stage_host is None:
            stage_host = dist.get_backend(group) != "nccl"
        self.x = HaloExchange(self.dims, self.coords, box.periodic, group, stage_host)
        self.dev = torch.device("cuda", device)
        self.stream = torch.cuda.ExternalStream(lib().dpdb_stream(self.brick.h), device=self.dev)
        self.gcnt = np.zeros(N_DIRS, np.int64)
        self.group = group

    @property
    def h(self):
        return self.brick.h

    def _ck(self, rc):
        check(rc, self.brick.h)

    def upload_global(self, store: ParticleStore):
        part = split_store(store, self.box, self.dims)[self.x.rank]
        self.brick.upload(part)

    def _xchg(self, what, counts):
        torch = self.torch
        rb = lib().dpdb_md_record_bytes(what)
        tot = int(np.sum(counts))
        send = torch.empty(max(tot, 1) * rb, dtype=torch.uint8, device=self.dev)
        self._ck(lib().dpdb_md_pack(self.h, what, C.c_void_p(send.data_ptr())))
        recv, rcnt = self.x.exchange(send[: tot * rb], counts, rb, self.dev)
        torch.cuda.synchronize(self.dev)
        return recv, np.ascontiguousarray(rcnt, np.int32)

    def _ptr(self, t):
        return C.c_void_p(t.data_ptr()) if t.numel() else None

    def _ghosts(self, gc):
        recv, rc = self._xchg(MD_GHOST_FULL, gc)
        self._ck(lib().dpdb_md_accept_ghosts(self.h, self._ptr(recv), ptr(rc)))
        self.gcnt = gc.astype(np.int64)

    def setup(self):
        L = lib()
        self._ck(L.dpdb_md_begin_setup(self.h))
        gc = np.zeros(N_DIRS, np.int32)
        self._ck(L.dpdb_md_accept_migrants(self.h, None, None, ptr(gc)))
        self._ghosts(gc)
        self._ck(L.dpdb_md_forces(self.h))

    def step(self, nsteps: int = 1):
        L = lib()
        for _ in range(int(nsteps)):
            if (self.brick.current_step + 1) % self.run.rebuild_every == 0:
                mc = np.zeros(N_DIRS, np.int32)
                self._ck(L.dpdb_md_begin_rebuild(self.h, ptr(mc)))
                recv, rc = self._xchg(MD_MIGRANTS, mc)
                gc = np.zeros(N_DIRS, np.int32)
                self._ck(L.dpdb_md_accept_migrants(self.h, self._ptr(recv), ptr(rc), ptr(gc)))
                self._ghosts(gc)
            else:
                self._ck(L.dpdb_md_begin_step(self.h))
                recv, rc = self._xchg(MD_GHOST_UPDATE, self.gcnt)
                self._ck(L.dpdb_md_accept_update(self.h, self._ptr(recv), ptr(rc)))
            self._ck(L.dpdb_md_forces(self.h))
        self._ck(L.dpdb_md_finish(self.h))

    def thermo(self):
        torch = self.torch
        s = torch.as_tensor(np.concatenate([self.brick.sums(), [self.brick.n]]),
                            dtype=torch.float64)
        s = s if self.x.stage_host else s.to(self.dev)
        self.x.dist.all_reduce(s, group=self.group)
        s = s.cpu().numpy()
        return thermo_from_sums(s[:4], s[4])

    def download_global(self):
        """All-gather the locals of every brick (test helper, host objects)."""
        part = self.brick.download()
        out = [None] * self.x.world
        self.x.dist.all_gather_object(out, part, group=self.group)
        return gather_stores(out)


class NcclBrick:
    """One brick per rank on the engine's own NCCL transport: the whole step
    loop (pack -> grouped ncclSend/Recv per direction -> unpack -> forces)
    runs in libdpdb.so on the brick's stream.  torch.distributed (any
    backend) only broadcasts the NCCL id and times the run."""

    def __init__(self, box: SimBox, params: PairParams, run: RunConfig | None, dims, capacity,
                 device=0, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.dims = tuple(int(v) for v in dims)
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world != self.dims[0] * self.dims[1] * self.dims[2]:
            raise DPDError(1, "nccl brick: world size must equal the number of bricks")
        self.coords = coords_of(self.rank, self.dims)
        self.box, self.run = box, run or RunConfig()
        self.brick = _Brick(box, params, self.run, capacity, device, self.dims, self.coords)
        uid = np.zeros(NCCL_ID_BYTES, np.uint8)
        if self.rank == 0:
            check(lib().dpdb_nccl_unique_id(ptr(uid)))
        obj = [uid.tobytes()]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = np.frombuffer(obj[0], np.uint8).copy()
        check(lib().dpdb_nccl_attach(self.brick.h, ptr(uid), self.world, self.rank), self.brick.h)

    @property
    def h(self):
        return self.brick.h

    def close(self):
        self.brick.close()

    def upload(self, part: ParticleStore):
        """This brick's own particles (all inside its slab)."""
        self.brick.upload(part)

    def upload_global(self, store: ParticleStore):
        self.brick.upload(split_store(store, self.box, self.dims)[self.rank])

    def setup(self):
        check(lib().dpdb_dist_setup(self.h), self.h)

    def step(self, nsteps: int = 1):
        check(lib().dpdb_dist_step(self.h, int(nsteps)), self.h)

    def step_timed(self, nsteps: int, stages: bool = False):
        """(ms, stage_ms[6] or None, stage_launches[6]) like Engine.step_timed."""
        ms = C.c_double()
        st = np.zeros(6) if stages else None
        ln = np.zeros(6, np.int64)
        check(lib().dpdb_dist_step_timed(self.h, int(nsteps), C.byref(ms), ptr(st), ptr(ln)),
              self.h)
        return ms.value, st, ln

    def thermo(self):
        t = Thermo()
        check(lib().dpdb_dist_thermo(self.h, C.byref(t)), self.h)
        return dict(step=t.step, n=t.n, kbt=t.kbt, momentum=tuple(t.momentum))

    def step_thermo(self, nsteps: int):
        """dpdb_dist_step_thermo: K steps, each rank records its per-step sums on
        the device (mapped pinned memory); one all-gather at the end adds the
        ranks' records in rank order."""
        import torch
        k = int(nsteps)
        mine = np.zeros((max(k, 1), 5))
        check(lib().dpdb_dist_step_thermo(self.h, k, ptr(mine)), self.h)
        n_loc = float(self.brick.n)
        dev = (torch.device("cuda", self.brick.device)
               if self.dist.get_backend(self.group) == "nccl" else torch.device("cpu"))
        t = torch.as_tensor(np.concatenate([mine[:k].ravel(), [n_loc]]), device=dev)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        allr = np.stack([o.cpu().numpy() for o in out])
        n = allr[:, -1].sum()
        sums = allr[:, :-1].reshape(self.world, k, 5)
        tot = np.zeros((k, 4))
        for r in range(self.world):  # rank order: deterministic
            tot += sums[r, :, 1:]
        p2 = (tot[:, :3] ** 2).sum(1)
        return dict(step=sums[0, :, 0].astype(np.int64), kbt=(tot[:, 3] - p2 / n) / (3.0 * n),
                    momentum=tot[:, :3])

    @property
    def current_step(self):
        return self.brick.current_step

    def download(self):
        return self.brick.download()

    def download_global(self):
        part = self.brick.download()
        out = [None] * self.world
        self.dist.all_gather_object(out, part, group=self.group)
        return gather_stores(out)
