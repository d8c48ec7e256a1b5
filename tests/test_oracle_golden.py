"""Pin the CPU oracle (oracle/dpd_oracle.c) to the reference's own bits.

tests/golden/*.npz were produced by the reference's shipped code
(tests/golden/make_golden.py via oracle/_ref).  When oracle/_ref is present
(this container) the oracle is additionally cross-checked on fresh random
inputs against the reference library itself.
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O


def test_spec_kats():
    L = O.lib()
    o = np.zeros(2, np.uint32)
    L.orc_tea_hash(0, 5, 6, o)
    assert list(o) == [5, 6]  # S:285 rounds=0 identity
    L.orc_tea_hash(16, 0, 0, o)
    assert list(o) == [0x741C187D, 0x4D3E2C53]
    assert L.orc_bit_reverse(1) == 0x80000000
    assert L.orc_make_signature(1, 0.0, 0.0, 0.0) == 0xE6221E02
    assert L.orc_make_signature(7, 0.1, -0.2, 0.3) == 0xCCF8DB8C
    assert L.orc_step_mix(1, 0) == 0x8562613F
    L.orc_pair_uniforms(0x1234, 0x5678, 3, 9, L.orc_step_mix(1, 0), o)
    assert list(o) == [0x710E165A, 0xB93E1DA5]
    o2 = np.zeros(2, np.uint32)
    L.orc_pair_uniforms(0x5678, 0x1234, 9, 3, L.orc_step_mix(1, 0), o2)
    assert list(o2) == list(o)  # S:303 symmetry
    assert L.orc_gaussian(2**31, 0) == 1.1774100224905713  # S:313 (rel 2.1e-11 of closed form)
    assert abs(L.orc_gaussian(2**31, 0) / np.sqrt(-2 * np.log(0.5)) - 1) < 1e-10
    assert L.orc_fastlog(1) == -22.18070977791825
    assert L.orc_fastlog(2**31) == -0.6931471805599453
    assert L.orc_fastcos2pi(0) == pytest.approx(1.0, rel=1.1e-10)
    assert L.orc_fastcos2pi(2**31) == pytest.approx(-1.0, rel=1.1e-10)
    assert abs(L.orc_fastpow(2.0, 3.0) - 8.0) <= 6 * np.spacing(8.0)
    assert L.orc_fastpow(0.3, 0.25) == 0.3 ** 0.25
    code = C.c_uint32()
    assert L.orc_morton_encode(3, 1, 2, 2, C.byref(code)) == 0 and code.value == 43
    assert L.orc_morton_encode(1, 1, 1, 1, C.byref(code)) == 0 and code.value == 7
    assert L.orc_morton_encode(4, 0, 0, 2, C.byref(code)) == 1  # out of range -> config


def test_tea_and_signatures_golden(golden):
    L = O.lib()
    g = golden.rng
    o = np.zeros(2, np.uint32)
    for r, a, b, x, y in g["tea"]:
        L.orc_tea_hash(int(r), int(a), int(b), o)
        assert (int(o[0]), int(o[1])) == (int(x), int(y))
    v = g["sig_v"]
    sig = O.signatures(g["sig_tag"], *[np.ascontiguousarray(v[:, k]) for k in range(3)])
    assert np.array_equal(sig, g["sig"])
    mix = [L.orc_step_mix(int(a), int(b)) for a, b in zip(g["mix_seed"], g["mix_step"])]
    assert np.array_equal(np.array(mix, np.uint32), g["mix"])
    for q, (si, sj, ti, tj) in enumerate(g["pu_in"]):
        m = L.orc_step_mix(int(g["pu_seed"][q]), int(g["pu_step"][q]))
        L.orc_pair_uniforms(int(si), int(sj), int(ti), int(tj), m, o)
        assert list(o) == list(g["pu_out"][q])


def test_fastmath_golden(golden):
    L = O.lib()
    g = golden.fastmath
    assert all(L.orc_fastlog(int(u)) == r for u, r in zip(g["log_u"], g["log"]))
    assert all(L.orc_fastcos2pi(int(u)) == r for u, r in zip(g["cos_u"], g["cos"]))
    assert all(L.orc_gaussian(int(a), int(b)) == r
               for a, b, r in zip(g["gauss_a"], g["gauss_b"], g["gauss"]))
    assert all(L.orc_fastpow(a, b) == r for a, b, r in zip(g["pow_a"], g["pow_b"], g["pow"]))


def test_fastmath_error_bounds(golden):
    """Table 3 error columns on the golden sweep."""
    g = golden.fastmath
    u = g["log_u"].astype(np.float64)
    # u * 2^-32 is exact in fp64; log1p keeps the oracle accurate as u -> 2^32
    exact = np.where(u > 2.0**31, np.log1p((u - 2.0**32) * 2.0**-32), np.log(u * 2.0**-32))
    rel = np.abs(g["log"] - exact) / np.abs(np.where(exact == 0, 1, exact))
    assert rel.max() <= 4.21e-12 * 2  # float64 oracle, not 80-bit: allow 2x
    c = g["cos_u"].astype(np.float64)
    ex = np.cos(2 * np.pi * c * 2.0**-32)
    err = np.abs(g["cos"] - ex)
    big = np.abs(ex) > 1e-3
    assert (err[big] / np.abs(ex[big])).max() <= 1.1e-10 * 2
    assert err[~big].max() <= 1.1e-10 * 2 * np.pi
    a, b = g["pow_a"], g["pow_b"]
    sel = (a >= 1e-10) & (a <= 2) & (b >= 0.25) & (b <= 3)
    ex = a[sel] ** b[sel]
    ulp = np.abs(g["pow"][sel] - ex) / np.spacing(ex)
    assert ulp.max() <= 6 + 1  # vs libm pow (itself <= 1 ulp)


@pytest.mark.parametrize("case", ["s0", "s1", "s4", "s1000", "s100k"])
def test_radix_golden(golden, case):
    g = golden.sort
    k = g[case + "_keys"].copy()
    v = np.arange(len(k), dtype=np.uint32)
    for threads in (1, 2, 8):
        kk, vv = k.copy(), v.copy()
        O.check(O.lib().orc_radix_sort(kk, vv, len(kk), int(g[case + "_bits"][0]), threads))
        assert np.array_equal(kk, g[case + "_skeys"]) and np.array_equal(vv, g[case + "_svals"])
    if case == "s4":
        assert list(g[case + "_skeys"]) == [1, 1, 2, 3] and list(g[case + "_svals"]) == [1, 3, 2, 0]


def test_radix_errors():
    k = np.zeros(4, np.uint32)
    assert O.lib().orc_radix_sort(k, k.copy(), 4, 6, 1) == 1
    assert O.lib().orc_radix_sort(k, k.copy(), 4, 36, 1) == 1


CASES = ["c1small", "aniso", "walled", "tiny", "dense"]


@pytest.mark.parametrize("case", CASES)
def test_cells_golden(golden, case):
    g = golden.cells
    p = case + "_"
    per = g[p + "per"]
    box = O.make_box((0, 0, 0), tuple(g[p + "L"]), tuple(int(v) for v in per))
    grid = O.OGrid(box, 1.3)
    info = g[p + "info_i"]
    assert list(grid.g.ncell) == list(info[:3]) and list(grid.g.ncell_ext) == list(info[3:6])
    assert list(grid.g.wrapmode) == list(info[6:9]) and grid.g.bits_per_axis == info[9]
    assert grid.nlc == info[10] and grid.ntc == info[11] and grid.key_bits() == info[12]
    assert list(grid.g.cell_size) == list(g[p + "info_d"][:3])
    assert np.array_equal(grid.rank_of_cell(), g[p + "rank_of_cell"])
    x, y, z = g[p + "x"], g[p + "y"], g[p + "z"]
    order, perm = grid.order(x, y, z, nthreads=4)
    assert np.array_equal(perm, g[p + "perm"])
    xs, ys, zs = x[order], y[order], z[order]
    cs = grid.cell_start(xs, ys, zs)
    assert np.array_equal(cs, g[p + "cell_start"])
    coff, cc = grid.coarse()
    assert np.array_equal(coff, g[p + "coff"]) and np.array_equal(cc, g[p + "ccells"])
    foff, fidx = grid.fine(coff, cc, cs)
    assert np.array_equal(foff, g[p + "foff"]) and np.array_equal(fidx, g[p + "fidx"])


def test_cell_list_examples():
    L = O.lib()
    cs = np.zeros(9, np.uint32)
    O.check(L.orc_build_cell_list(8, np.array([0], np.uint32), 1, cs))
    assert list(cs) == [0, 1, 1, 1, 1, 1, 1, 1, 1]
    O.check(L.orc_build_cell_list(8, np.array([7, 7, 7], np.uint32), 3, cs))
    assert list(cs) == [0] * 7 + [0, 3]
    assert L.orc_build_cell_list(8, np.array([3, 1], np.uint32), 2, cs) == 3  # unsorted


@pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built (no /root/reference here)")
def test_oracle_vs_reference_random():
    """Fresh random inputs through both the oracle and the reference library."""
    L, R = O.lib(), O.ref()
    g = np.random.default_rng(99)
    for _ in range(3000):
        t = int(g.integers(0, 2**32))
        v = g.normal(size=3) * g.choice([1e-5, 1, 1e5])
        assert L.orc_make_signature(t, *v) == R.ref_make_signature(t, *v)
        u = int(g.integers(1, 2**32))
        assert L.orc_fastlog(u) == R.ref_fastlog(u)
        assert L.orc_fastcos2pi(u) == R.ref_fastcos2pi(u)
        a, b = 10 ** g.uniform(-12, 3), g.uniform(0, 4)
        assert L.orc_fastpow(a, b) == R.ref_fastpow(a, b)
    for n in (7, 4097, 50000):
        k = g.integers(0, 2**28, n).astype(np.uint32)
        v = np.arange(n, dtype=np.uint32)
        k1, v1, k2, v2 = k.copy(), v.copy(), k.copy(), v.copy()
        L.orc_radix_sort(k1, v1, n, 28, 3)
        R.ref_radix_sort(k2, v2, n, 28, 5)
        assert np.array_equal(v1, v2)
    dr = np.array([7.0, -6.5, 3.0])
    out = np.zeros(3)
    R.ref_minimum_image(dr, np.zeros(3), np.array([12.0, 12.0, 12.0]), np.array([1, 1, 0], np.int32), out)
    assert list(out) == [-5.0, 5.5, 3.0]
