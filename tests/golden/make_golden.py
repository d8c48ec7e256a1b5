"""Generate tests/golden/*.npz from the REFERENCE'S OWN shipped code.

Runs only where /root/reference exists: oracle/Makefile compiles the
reference sources in place into oracle/_ref/libdpdref.so (ref_shim.cpp wraps
them in extern "C").  The outputs are committed so the CPU tests and the GPU
box (which never sees /root/reference) can pin the oracle and the kernels to
the reference's bits.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def rng_kats(R):
    g = np.random.default_rng(20131102)
    out = {}
    # tea_hash(rounds, v0, v1): fixed + random
    tri = [(16, 0, 0), (4, 0, 0), (4, 1, 0), (0, 5, 6), (32, 123, 456)]
    tri += [(int(r), int(a), int(b)) for r, a, b in zip(g.integers(0, 33, 200),
                                                         g.integers(0, 2**32, 200),
                                                         g.integers(0, 2**32, 200))]
    o = np.zeros(2, np.uint32)
    res = []
    for r, a, b in tri:
        R.ref_tea_hash(r, a, b, o)
        res.append((r, a, b, int(o[0]), int(o[1])))
    out["tea"] = np.array(res, np.uint64)
    # signatures on random tags and velocities of mixed scales, plus specials
    n = 4000
    tags = g.integers(0, 2**32, n).astype(np.uint32)
    v = g.normal(size=(n, 3)) * g.choice([1e-3, 1.0, 1e3], size=(n, 1))
    v[:4] = [[0, 0, 0], [0.1, -0.2, 0.3], [-0.0, 1.0, -1.0], [1e-300, 1e300, 5e-324]]
    tags[:4] = [1, 7, 2**31, 0xFFFFFFFF]
    out["sig_tag"] = tags
    out["sig_v"] = v
    out["sig"] = np.array([R.ref_make_signature(int(t), *vv) for t, vv in zip(tags, v)], np.uint32)
    # step_mix / pair uniforms
    seeds = g.integers(0, 2**32, 300).astype(np.uint32)
    steps = g.integers(0, 10**6, 300).astype(np.uint32)
    seeds[0], steps[0] = 1, 0
    out["mix_seed"], out["mix_step"] = seeds, steps
    out["mix"] = np.array([R.ref_step_mix(int(a), int(b)) for a, b in zip(seeds, steps)], np.uint32)
    m = 3000
    pu = g.integers(0, 2**32, (m, 4)).astype(np.uint32)
    pu[0] = [0x1234, 0x5678, 3, 9]
    pu[1] = [0x5678, 0x1234, 9, 3]
    ps = g.integers(0, 2**32, m).astype(np.uint32)
    pt = g.integers(0, 10**6, m).astype(np.uint32)
    ps[:2], pt[:2] = 1, 0
    res = np.zeros((m, 2), np.uint32)
    for q in range(m):
        R.ref_pair_uniforms(*[int(x) for x in pu[q]], int(ps[q]), int(pt[q]), o)
        res[q] = o
    out["pu_in"], out["pu_seed"], out["pu_step"], out["pu_out"] = pu, ps, pt, res
    return out


def fastmath_kats(R):
    g = np.random.default_rng(1311)
    out = {}
    u = np.concatenate([np.arange(1, 2**32, 65537, dtype=np.uint64)[:50000],
                        g.integers(1, 2**32, 20000, dtype=np.uint64),
                        [1, 2, 3, 2**31, 2**32 - 1, 2**32 - 2, 3037000499, 3037000500]])
    u = u.astype(np.uint32)
    out["log_u"] = u
    out["log"] = np.array([R.ref_fastlog(int(x)) for x in u])
    c = np.concatenate([np.arange(0, 2**32, 65537, dtype=np.uint64)[:50000],
                        g.integers(0, 2**32, 20000, dtype=np.uint64),
                        [0, 2**30, 2**31, 3 * 2**30, 2**32 - 1]]).astype(np.uint32)
    out["cos_u"] = c
    out["cos"] = np.array([R.ref_fastcos2pi(int(x)) for x in c])
    ga = g.integers(0, 2**32, 20000).astype(np.uint32)
    gb = g.integers(0, 2**32, 20000).astype(np.uint32)
    ga[:3], gb[:3] = [2**31, 0, 1], [0, 5, 2**31]
    out["gauss_a"], out["gauss_b"] = ga, gb
    out["gauss"] = np.array([R.ref_gaussian(int(a), int(b)) for a, b in zip(ga, gb)])
    pa = np.concatenate([10 ** g.uniform(-10, np.log10(2), 20000), 10 ** g.uniform(-51, 51, 5000),
                         [2.0, 0.3, 1.0, 0.5]])
    pb = np.concatenate([g.uniform(0.25, 3, 20000), g.uniform(0, 6, 5000), [3.0, 0.25, 2.5, 0.0]])
    out["pow_a"], out["pow_b"] = pa, pb
    out["pow"] = np.array([R.ref_fastpow(a, b) for a, b in zip(pa, pb)])
    return out


def sort_kats(R):
    g = np.random.default_rng(7)
    out = {}
    for name, n, bits in [("s0", 0, 8), ("s1", 1, 4), ("s4", 4, 4), ("s1000", 1000, 12),
                          ("s100k", 100003, 24)]:
        if name == "s4":
            k = np.array([3, 1, 2, 1], np.uint32)
        else:
            k = g.integers(0, 2 ** bits, n).astype(np.uint32)
        v = np.arange(n, dtype=np.uint32)
        k2, v2 = k.copy(), v.copy()
        assert R.ref_radix_sort(k2, v2, n, bits, 3) == 0
        out[name + "_keys"], out[name + "_bits"] = k, np.array([bits])
        out[name + "_skeys"], out[name + "_svals"] = k2, v2
    return out


CELL_CASES = [
    # name, box, periodic, n, seed
    ("c1small", (8.0, 8.0, 8.0), (1, 1, 1), 1536, 11),
    ("aniso", (10.0, 7.3, 5.1), (1, 0, 1), 1100, 12),
    ("walled", (6.0, 6.0, 6.0), (0, 0, 0), 648, 13),
    ("tiny", (3.0, 3.0, 3.0), (1, 1, 1), 60, 14),
    ("dense", (4.0, 4.0, 4.0), (1, 1, 1), 3200, 15),
]


def cell_kats(R):
    out = {}
    for name, L, per, n, seed in CELL_CASES:
        g = np.random.default_rng(seed)
        lo = np.zeros(3)
        hi = np.array(L)
        x = g.uniform(0, L[0], n)
        y = g.uniform(0, L[1], n)
        z = g.uniform(0, L[2], n)
        tag = (g.permutation(n) + 1).astype(np.uint32)
        per = np.array(per, np.int32)
        info_i = np.zeros(13, np.int64)
        info_d = np.zeros(9)
        assert R.ref_grid_info(lo, hi, per, 1.3, 2, info_i, info_d) == 0
        ntc, nlc = int(info_i[11]), int(info_i[10])
        roc = np.zeros(ntc, np.uint32)
        R.ref_grid_ranks(lo, hi, per, 1.3, 2, roc)
        rx, ry, rz, rt = x.copy(), y.copy(), z.copy(), tag.copy()
        perm = np.zeros(n, np.uint32)
        cs = np.zeros(ntc + 1, np.uint32)
        coff = np.zeros(nlc + 1, np.uint32)
        cc = np.zeros(27 * nlc, np.uint32)
        foff = np.zeros(nlc + 1, np.uint32)
        fidx = np.zeros(28 * n * max(1, min(nlc, 27)) // 1 + 64, np.uint32)
        rc = R.ref_reorder_cells(lo, hi, per, 1.3, 2, 2, n, rx, ry, rz, rt, perm, cs, coff, cc, foff,
                                 fidx.ctypes.data, len(fidx))
        assert rc == 0, R.ref_last_error()
        p = name + "_"
        out.update({p + "L": hi, p + "per": per, p + "x": x, p + "y": y, p + "z": z, p + "tag": tag,
                    p + "info_i": info_i, p + "info_d": info_d, p + "rank_of_cell": roc,
                    p + "perm": perm, p + "cell_start": cs, p + "coff": coff,
                    p + "ccells": cc[: coff[-1]], p + "foff": foff, p + "fidx": fidx[: foff[-1]]})
    return out


def main():
    R = oracle.ref()
    if R is None:
        oracle.build()
        R = oracle.ref()
    if R is None:
        sys.exit("oracle/_ref/libdpdref.so unavailable: /root/reference is required to regenerate")
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **rng_kats(R))
    np.savez_compressed(os.path.join(OUT, "fastmath.npz"), **fastmath_kats(R))
    np.savez_compressed(os.path.join(OUT, "sort.npz"), **sort_kats(R))
    np.savez_compressed(os.path.join(OUT, "cells.npz"), **cell_kats(R))
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
