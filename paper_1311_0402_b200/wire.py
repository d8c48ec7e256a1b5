"""GhostPacket wire format and a byte-stream transport for the brick protocol
(SURVEY 8(f)4).

Header: 4 little-endian u32 words -- magic 0x44504447 ("GDPD"), kind, step,
count.  Payload: `count` records, fields concatenated per particle, little
endian, no padding:

  ghost_full    tag u32, species u8, x y z f64, vx vy vz f64, molecule u32   (57 B)
  ghost_update  x y z f64, vx vy vz f64                                      (48 B)
  stray         tag u32, species u8, x y z f64, vx vy vz f64, molecule u32,
                fx fy fz f64                                                 (81 B)

Strays travel right after phase 1 of a rebuild step, before that step's
forces exist, so their force words are zero on the wire (the receiver
evaluates them).  The device packs/unpacks its own records (`dpdb_md_pack`,
`dpdb_md_accept_*`); this module converts between those records and packets,
and moves packets over any byte channel:

* `WireGroup`  -- every brick in this process, packets through in-memory
  mailboxes (the reference's default in-process channels);
* `SocketChannel` + `WireBrick` -- one brick per process, packets over
  multiprocessing connections (TCP), the reference's optional socket
  transport with the same wire format.
"""
from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from ._lib import MD_GHOST_FULL, MD_GHOST_UPDATE, MD_MIGRANTS, DPDError, check, lib, ptr
from .domain import N_DIRS, _Brick, coords_of, gather_stores, neighbor, opposite, rank_of, split_store
from .engine import PairParams, ParticleStore, RunConfig, SimBox

MAGIC = 0x44504447
KIND_GHOST_FULL, KIND_GHOST_UPDATE, KIND_STRAY = 0, 1, 2
_HDR = struct.Struct("<IIII")

# device records (domain.cuh GhostRec / GhostUpd)
DEV_REC = np.dtype([("x", "<f8", 3), ("v", "<f8", 3), ("tag", "<u4"), ("sp_mol", "<u4")])
DEV_UPD = np.dtype([("x", "<f8", 3), ("v", "<f8", 3)])
# wire payloads (packed)
WIRE_FULL = np.dtype([("tag", "<u4"), ("species", "u1"), ("x", "<f8", 3), ("v", "<f8", 3),
                      ("molecule", "<u4")])
WIRE_UPDATE = np.dtype([("x", "<f8", 3), ("v", "<f8", 3)])
WIRE_STRAY = np.dtype([("tag", "<u4"), ("species", "u1"), ("x", "<f8", 3), ("v", "<f8", 3),
                       ("molecule", "<u4"), ("f", "<f8", 3)])
_KIND_OF = {MD_GHOST_FULL: KIND_GHOST_FULL, MD_GHOST_UPDATE: KIND_GHOST_UPDATE, MD_MIGRANTS: KIND_STRAY}
_WIRE = {KIND_GHOST_FULL: WIRE_FULL, KIND_GHOST_UPDATE: WIRE_UPDATE, KIND_STRAY: WIRE_STRAY}
assert WIRE_FULL.itemsize == 57 and WIRE_UPDATE.itemsize == 48 and WIRE_STRAY.itemsize == 81
assert DEV_REC.itemsize == 56 and DEV_UPD.itemsize == 48


def encode(kind: int, step: int, dev_records: np.ndarray) -> bytes:
    """Device records of one direction -> GhostPacket bytes."""
    n = len(dev_records)
    w = np.zeros(n, _WIRE[kind])
    w["x"], w["v"] = dev_records["x"], dev_records["v"]
    if kind != KIND_GHOST_UPDATE:
        w["tag"] = dev_records["tag"]
        w["species"] = dev_records["sp_mol"] & 0xFF
        w["molecule"] = dev_records["sp_mol"] >> 8
    return _HDR.pack(MAGIC, kind, int(step) & 0xFFFFFFFF, n) + w.tobytes()


def decode(buf: bytes, expect_kind: int | None = None):
    """GhostPacket bytes -> (kind, step, device records)."""
    if len(buf) < _HDR.size:
        raise DPDError(3, "ghost packet: truncated header")
    magic, kind, step, n = _HDR.unpack_from(buf)
    if magic != MAGIC:
        raise DPDError(3, f"ghost packet: bad magic 0x{magic:08x}")
    if kind not in _WIRE:
        raise DPDError(3, f"ghost packet: unknown kind {kind}")
    if expect_kind is not None and kind != expect_kind:
        raise DPDError(3, f"ghost packet: kind {kind}, expected {expect_kind} (protocol desync)")
    wd = _WIRE[kind]
    if len(buf) != _HDR.size + n * wd.itemsize:
        raise DPDError(3, "ghost packet: count does not match the payload length")
    w = np.frombuffer(buf, wd, n, _HDR.size)
    if kind == KIND_GHOST_UPDATE:
        out = np.zeros(n, DEV_UPD)
    else:
        if np.any(w["molecule"] >= (1 << 24)):
            raise DPDError(3, "ghost packet: molecule id exceeds 24 bits")
        out = np.zeros(n, DEV_REC)
        out["tag"] = w["tag"]
        out["sp_mol"] = w["species"].astype(np.uint32) | (w["molecule"] << 8)
    out["x"], out["v"] = w["x"], w["v"]
    return kind, step, out


class _Protocol:
    """The per-brick protocol of include/dpdb.h (dpdb_md_*) with packets:
    pack on the device, split by direction, encode, post; then collect the
    packets addressed to this brick in ascending direction, decode and accept
    on the device.  Subclasses provide post()/collect()."""

    def __init__(self, brick: _Brick, dims, periodic, device):
        import torch
        self.torch = torch
        self.brick = brick
        self.dims = tuple(dims)
        self.coords = brick.domain_info()[3]
        self.rank = rank_of(self.coords, self.dims)
        self.dev = torch.device("cuda", device)
        self.peer = [None] * N_DIRS
        for d in range(N_DIRS):
            nb = neighbor(self.dims, self.coords, periodic, d)
            self.peer[d] = None if nb is None else rank_of(nb, self.dims)
        self.gcnt = np.zeros(N_DIRS, np.int64)

    def ck(self, rc):
        check(rc, self.brick.h)

    def pack_post(self, what, counts):
        torch = self.torch
        rb = lib().dpdb_md_record_bytes(what)
        tot = int(np.sum(counts))
        buf = torch.empty(max(tot, 1) * rb, dtype=torch.uint8, device=self.dev)
        self.ck(lib().dpdb_md_pack(self.brick.h, what, C.c_void_p(buf.data_ptr())))
        torch.cuda.synchronize(self.dev)
        dev = np.frombuffer(buf[: tot * rb].cpu().numpy().tobytes(),
                            DEV_UPD if what == MD_GHOST_UPDATE else DEV_REC)
        off = np.concatenate([[0], np.cumsum(np.asarray(counts, np.int64))])
        step = self.brick.current_step
        for d in range(N_DIRS):
            if self.peer[d] is not None:
                self.post(self.peer[d], opposite(d), encode(_KIND_OF[what], step, dev[off[d]:off[d + 1]]))

    def collect_accept(self, what, counts_out=None):
        torch = self.torch
        kind = _KIND_OF[what]
        parts, rc = [], np.zeros(N_DIRS, np.int32)
        for d in range(N_DIRS):
            if self.peer[d] is None:
                continue
            _, _, recs = decode(self.collect(self.peer[d], d), kind)
            parts.append(recs)
            rc[d] = len(recs)
        raw = b"".join(p.tobytes() for p in parts)
        t = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(self.dev) if raw else None
        p = C.c_void_p(t.data_ptr()) if t is not None else None
        L = lib()
        if what == MD_MIGRANTS:
            self.ck(L.dpdb_md_accept_migrants(self.brick.h, p, ptr(rc), ptr(counts_out)))
        elif what == MD_GHOST_FULL:
            self.ck(L.dpdb_md_accept_ghosts(self.brick.h, p, ptr(rc)))
        else:
            self.ck(L.dpdb_md_accept_update(self.brick.h, p, ptr(rc)))
        self.torch.cuda.synchronize(self.dev)


class WireGroup:
    """Every brick in this process; packets through in-memory mailboxes."""

    def __init__(self, box: SimBox, params: PairParams, run: RunConfig | None, dims, capacity: int,
                 device: int = 0):
        self.box, self.run = box, run or RunConfig()
        self.dims = tuple(int(v) for v in dims)
        nb = self.dims[0] * self.dims[1] * self.dims[2]
        self.bricks = [_Brick(box, params, self.run, capacity, device, self.dims,
                              coords_of(q, self.dims)) for q in range(nb)]
        self.mail = {}
        grp = self

        class P(_Protocol):
            def post(self, dest, d, pkt):
                grp.mail[(dest, d)] = pkt

            def collect(self, src, d):
                return grp.mail.pop((self.rank, d))

        self.p = [P(b, self.dims, box.periodic, device) for b in self.bricks]
        self.packets = self.bytes = 0

    def close(self):
        for b in self.bricks:
            b.close()

    def upload(self, store: ParticleStore):
        for b, part in zip(self.bricks, split_store(store, self.box, self.dims)):
            b.upload(part)

    def _round(self, what, counts):
        for p, c in zip(self.p, counts):
            p.pack_post(what, c)
        self.packets += len(self.mail)
        self.bytes += sum(len(v) for v in self.mail.values())
        outs = []
        for p in self.p:
            gc = np.zeros(N_DIRS, np.int32)
            p.collect_accept(what, gc)
            outs.append(gc)
        return outs

    def _ghosts(self, gcs):
        self._round(MD_GHOST_FULL, gcs)
        for p, g in zip(self.p, gcs):
            p.gcnt = g.astype(np.int64)

    def setup(self):
        L = lib()
        gcs = []
        for p in self.p:
            p.ck(L.dpdb_md_begin_setup(p.brick.h))
            gc = np.zeros(N_DIRS, np.int32)
            p.ck(L.dpdb_md_accept_migrants(p.brick.h, None, None, ptr(gc)))
            gcs.append(gc)
        self._ghosts(gcs)
        for p in self.p:
            p.ck(L.dpdb_md_forces(p.brick.h))

    def step(self, nsteps: int = 1):
        L = lib()
        for _ in range(int(nsteps)):
            if (self.bricks[0].current_step + 1) % self.run.rebuild_every == 0:
                mcs = []
                for p in self.p:
                    mc = np.zeros(N_DIRS, np.int32)
                    p.ck(L.dpdb_md_begin_rebuild(p.brick.h, ptr(mc)))
                    mcs.append(mc)
                self._ghosts(self._round(MD_MIGRANTS, mcs))
            else:
                for p in self.p:
                    p.ck(L.dpdb_md_begin_step(p.brick.h))
                self._round(MD_GHOST_UPDATE, [p.gcnt for p in self.p])
            for p in self.p:
                p.ck(L.dpdb_md_forces(p.brick.h))
        for p in self.p:
            p.ck(L.dpdb_md_finish(p.brick.h))

    def download(self) -> ParticleStore:
        return gather_stores([b.download() for b in self.bricks])


# ------------------------------------------------------------ sockets
class SocketChannel:
    """Byte messages between the ranks of a brick decomposition over TCP
    (multiprocessing connections on host:base_port + rank).  Every packet
    travels in an envelope carrying the direction the receiver files it
    under, so several directions to one peer cannot be confused; sends run
    on a helper thread while this rank receives (no send/send deadlock)."""

    def __init__(self, rank: int, peers, base_port: int, host: str = "127.0.0.1",
                 authkey: bytes = b"dpdb", timeout: float = 60.0):
        import time
        from multiprocessing.connection import Client, Listener
        self.rank = rank
        self.conn = {}
        peers = sorted(set(p for p in peers if p is not None and p != rank))
        lower = [p for p in peers if p < rank]
        lst = Listener((host, base_port + rank), authkey=authkey) if lower else None
        for p in peers:
            if p > rank:  # connect up, retrying until the peer listens
                t0 = time.time()
                while True:
                    try:
                        c = Client((host, base_port + p), authkey=authkey)
                        break
                    except (ConnectionRefusedError, OSError):
                        if time.time() - t0 > timeout:
                            raise DPDError(5, f"socket channel: rank {p} not reachable")
                        time.sleep(0.05)
                c.send_bytes(struct.pack("<I", rank))
                self.conn[p] = c
        for _ in lower:
            c = lst.accept()
            (p,) = struct.unpack("<I", c.recv_bytes())
            self.conn[p] = c
        if lst:
            lst.close()

    def exchange(self, outgoing, incoming):
        """outgoing: [(peer, dir_at_receiver, bytes)]; incoming: {peer: [dir, ...]}
        -> {(peer, dir): bytes}."""
        import threading

        def send_all():
            for p, d, b in outgoing:
                self.conn[p].send_bytes(struct.pack("<I", d) + b)

        th = threading.Thread(target=send_all)
        th.start()
        got = {}
        for p, dirs in incoming.items():
            for _ in dirs:
                m = self.conn[p].recv_bytes()
                (d,) = struct.unpack_from("<I", m)
                got[(p, d)] = m[4:]
        th.join()
        return got

    def close(self):
        for c in self.conn.values():
            c.close()


class WireBrick:
    """One brick per process on the socket transport: the per-brick device
    protocol with GhostPackets on the wire (rank = rank_of(coords))."""

    def __init__(self, box: SimBox, params: PairParams, run: RunConfig | None, dims, capacity: int,
                 rank: int, base_port: int, device: int = 0, host: str = "127.0.0.1"):
        self.box, self.run = box, run or RunConfig()
        self.dims = tuple(int(v) for v in dims)
        self.brick = _Brick(box, params, self.run, capacity, device, self.dims,
                            coords_of(rank, self.dims))
        outer = self
        self.out, self.inbox = [], {}

        class P(_Protocol):
            def post(self, dest, d, pkt):
                outer.out.append((dest, d, pkt))

            def collect(self, src, d):
                return outer.inbox.pop((src, d))

        self.p = P(self.brick, self.dims, box.periodic, device)
        self.chan = SocketChannel(rank, self.p.peer, base_port, host)

    def close(self):
        self.chan.close()
        self.brick.close()

    def upload_global(self, store: ParticleStore):
        self.brick.upload(split_store(store, self.box, self.dims)[self.p.rank])

    def _round(self, what, counts):
        self.out = []
        self.p.pack_post(what, counts)
        want = {}
        for d in range(N_DIRS):
            if self.p.peer[d] is not None:
                want.setdefault(self.p.peer[d], []).append(d)
        self.inbox = self.chan.exchange(self.out, want)
        gc = np.zeros(N_DIRS, np.int32)
        self.p.collect_accept(what, gc)
        return gc

    def setup(self):
        L = lib()
        self.p.ck(L.dpdb_md_begin_setup(self.brick.h))
        gc = np.zeros(N_DIRS, np.int32)
        self.p.ck(L.dpdb_md_accept_migrants(self.brick.h, None, None, ptr(gc)))
        self._round(MD_GHOST_FULL, gc)
        self.p.gcnt = gc.astype(np.int64)
        self.p.ck(L.dpdb_md_forces(self.brick.h))

    def step(self, nsteps: int = 1):
        L = lib()
        for _ in range(int(nsteps)):
            if (self.brick.current_step + 1) % self.run.rebuild_every == 0:
                mc = np.zeros(N_DIRS, np.int32)
                self.p.ck(L.dpdb_md_begin_rebuild(self.brick.h, ptr(mc)))
                gc = self._round(MD_MIGRANTS, mc)
                self._round(MD_GHOST_FULL, gc)
                self.p.gcnt = gc.astype(np.int64)
            else:
                self.p.ck(L.dpdb_md_begin_step(self.brick.h))
                self._round(MD_GHOST_UPDATE, self.p.gcnt)
            self.p.ck(L.dpdb_md_forces(self.brick.h))
        self.p.ck(L.dpdb_md_finish(self.brick.h))

    def download(self) -> ParticleStore:
        return self.brick.download()
