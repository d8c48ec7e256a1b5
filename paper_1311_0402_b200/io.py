"""Output formats of write_outputs: XYZ frames,
thermo and profile CSV, and a versioned binary restart whose reload continues
the run bitwise on one domain (save after a rebuild step; Engine.setup_at).

Restart layout (little endian):
  magic  8 bytes  b"DPDBRST\\0"
  u32    version (1)
  u32    n_species
  u64    n
  i64    step
  u32    seed
  u32    flags (bit 0: molecule ids present)
  f64[6] box lo, hi
  then n x f64 for x, y, z, vx, vy, vz, fx, fy, fz; n x u32 tags; n x u8
  species; [n x u32 molecule ids].  The forces are part of the state: step
  n+1's first half kick uses f(n), which was evaluated with the half-step
  velocity, so it cannot be recomputed from the full-step v(n).
"""
from __future__ import annotations

import struct

import numpy as np

from .engine import ParticleStore

MAGIC = b"DPDBRST\0"
VERSION = 1
_HDR = struct.Struct("<8sIIQqII6d")


def write_xyz(path, store: ParticleStore, names=("S", "A", "B", "C"), comment="", append=False):
    """One XYZ frame: count line, comment line, `name x y z` per particle."""
    sp = store.species if store.species is not None else np.zeros(len(store.tag), np.uint8)
    with open(path, "a" if append else "w") as fh:
        fh.write(f"{len(store.tag)}\n{comment}\n")
        for s_, x, y, z in zip(sp, *store.coord):
            fh.write(f"{names[int(s_)]} {x:.10g} {y:.10g} {z:.10g}\n")


def write_thermo_csv(path, records, dt, n):
    """step, time, kbt_measured, px, py, pz, n (one line per record)."""
    with open(path, "w") as fh:
        fh.write("step,time,kbt,px,py,pz,n\n")
        for s_, k, p in zip(records["step"], records["kbt"], records["momentum"]):
            fh.write(f"{int(s_)},{s_ * dt:.10g},{float(k)!r},{float(p[0])!r},{float(p[1])!r},"
                     f"{float(p[2])!r},{n}\n")


def write_profile_csv(path, prof):
    """bin_center, mean_v, count."""
    with open(path, "w") as fh:
        fh.write("bin_center,mean_v,count\n")
        for c, v, k in zip(prof.centers, prof.mean_v, prof.count):
            fh.write(f"{float(c)!r},{float(v)!r},{int(k)}\n")


def save_restart(path, engine, seed=None):
    """Full state + step + RNG seed of an Engine (single domain)."""
    s = engine.download()
    n = len(s.tag)
    mol = getattr(s, "molecule", None)
    box = engine.box
    hdr = _HDR.pack(MAGIC, VERSION, int(engine.params.n_species), n, int(engine.current_step),
                    int(engine.run.seed if seed is None else seed), 1 if mol is not None else 0,
                    *box.lo, *box.hi)
    with open(path, "wb") as fh:
        fh.write(hdr)
        for a in list(s.coord) + list(s.veloc) + list(s.force):
            fh.write(np.ascontiguousarray(a, "<f8").tobytes())
        fh.write(np.ascontiguousarray(s.tag, "<u4").tobytes())
        sp = s.species if s.species is not None else np.zeros(n, np.uint8)
        fh.write(np.ascontiguousarray(sp, "u1").tobytes())
        if mol is not None:
            fh.write(np.ascontiguousarray(mol, "<u4").tobytes())


def read_restart(path):
    """-> (ParticleStore, step, seed, header dict); raises on a bad file."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _HDR.size:
        raise ValueError(f"restart {path}: truncated header")
    magic, ver, ns, n, step, seed, flags, *b = _HDR.unpack_from(raw)
    if magic != MAGIC:
        raise ValueError(f"restart {path}: not a restart file")
    if ver != VERSION:
        raise ValueError(f"restart {path}: version {ver}, expected {VERSION}")
    need = _HDR.size + n * (9 * 8 + 4 + 1 + (4 if flags & 1 else 0))
    if len(raw) != need:
        raise ValueError(f"restart {path}: {len(raw)} bytes, expected {need}")
    off = _HDR.size
    arr = []
    for _ in range(9):
        arr.append(np.frombuffer(raw, "<f8", n, off).copy())
        off += 8 * n
    tag = np.frombuffer(raw, "<u4", n, off).copy()
    off += 4 * n
    sp = np.frombuffer(raw, "u1", n, off).copy()
    off += n
    mol = np.frombuffer(raw, "<u4", n, off).copy() if flags & 1 else None
    store = ParticleStore(arr[:3], arr[3:6], tag, sp, mol)
    store.force = arr[6:9]
    return store, step, seed, dict(n_species=ns, lo=tuple(b[:3]), hi=tuple(b[3:]))


def load_restart(path, engine):
    """Upload a restart into `engine` (same box / params) and set it up at the
    saved step; returns the step."""
    store, step, seed, hdr = read_restart(path)
    if engine.params.n_species != hdr["n_species"]:
        raise ValueError("restart: species count differs from the engine's parameters")
    engine.upload(store)
    engine.upload_forces(*store.force)
    engine.setup_at(step, keep_forces=True)
    return step
