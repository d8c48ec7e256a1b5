"""Device RNG / fastmath streams vs the reference's bits (tests/golden from the
reference's own code) -- bit-exact; plus the fp32 hot-path Gaussian bound."""
import numpy as np
import pytest

import paper_1311_0402_b200 as dpd

pytestmark = pytest.mark.gpu


def test_tea_hash_bitexact(golden):
    t = golden.rng["tea"].astype(np.uint64)
    for rounds in np.unique(t[:, 0]):
        sel = t[:, 0] == rounds
        out = dpd.tea_hash(int(rounds), t[sel, 1].astype(np.uint32), t[sel, 2].astype(np.uint32))
        assert np.array_equal(out[:, 0], t[sel, 3].astype(np.uint32))
        assert np.array_equal(out[:, 1], t[sel, 4].astype(np.uint32))


def test_signature_bitexact(golden):
    g = golden.rng
    sig = dpd.make_signature(g["sig_tag"], g["sig_v"])
    assert np.array_equal(sig, g["sig"])
    assert sig[0] == 0xE6221E02 and sig[1] == 0xCCF8DB8C


def test_step_mix_and_pair_uniforms_bitexact(golden):
    g = golden.rng
    assert np.array_equal(dpd.step_mix(g["mix_seed"], g["mix_step"]), g["mix"])
    pu = g["pu_in"]
    mix = dpd.step_mix(g["pu_seed"], g["pu_step"])
    for m in np.unique(mix)[:50]:  # the op takes one step_mix per call
        sel = mix == m
        out = dpd.pair_uniforms(pu[sel, 0], pu[sel, 1], pu[sel, 2], pu[sel, 3], int(m))
        assert np.array_equal(out, g["pu_out"][sel])
    out = dpd.pair_uniforms([0x1234, 0x5678], [0x5678, 0x1234], [3, 9], [9, 3], 0x8562613F)
    assert list(out[0]) == [0x710E165A, 0xB93E1DA5] and list(out[1]) == list(out[0])


def test_fastmath_bitexact(golden):
    g = golden.fastmath
    assert np.array_equal(dpd.fastlog(g["log_u"]), g["log"])
    assert np.array_equal(dpd.fastcos2pi(g["cos_u"]), g["cos"])
    assert np.array_equal(dpd.gaussian(g["gauss_a"], g["gauss_b"]), g["gauss"])
    assert np.array_equal(dpd.fastpow(g["pow_a"], g["pow_b"]), g["pow"])


def test_gaussian32_hot_path_accuracy(golden):
    """The force kernel's fp32 Box-Muller vs the bit-exact fp64 one."""
    g = golden.fastmath
    rng = np.random.default_rng(5)
    a = np.concatenate([g["gauss_a"], rng.integers(0, 2**32, 500000).astype(np.uint32),
                        (2**32 - np.arange(1, 5000)).astype(np.uint32)])
    b = np.concatenate([g["gauss_b"], rng.integers(0, 2**32, 500000).astype(np.uint32),
                        rng.integers(0, 2**32, 4999).astype(np.uint32)])
    ref = dpd.gaussian(a, b)
    got = dpd.gaussian(a, b, fp32=True).astype(np.float64)
    err = np.abs(got - ref)
    assert err.max() < 4e-6, err.max()
    lg = dpd.fastlog(a[a > 0], fp32=True).astype(np.float64)
    lref = dpd.fastlog(a[a > 0])
    assert (np.abs(lg - lref) / np.abs(lref)).max() < 5e-7


def test_gaussian_hot_accuracy(golden):
    """The Box-Muller the force kernels run (rcp/rsqrt/sin.approx, ftz) vs the
    bit-exact fp64 one, including u_a -> 2^32 where ln u cancels."""
    g = golden.fastmath
    rng = np.random.default_rng(6)
    a = np.concatenate([g["gauss_a"], rng.integers(0, 2**32, 1000000).astype(np.uint32),
                        (2**32 - np.arange(1, 5000)).astype(np.uint32), np.arange(0, 5000, dtype=np.uint32)])
    b = np.concatenate([g["gauss_b"], rng.integers(0, 2**32, 1000000).astype(np.uint32),
                        rng.integers(0, 2**32, 9999).astype(np.uint32)])
    ref = dpd.gaussian(a, b)
    got = dpd.gaussian(a, b, hot=True).astype(np.float64)
    assert np.abs(got - ref).max() < 4e-6, np.abs(got - ref).max()


def test_gaussian_moments():
    """moments of 2^20 Gaussians from signature-TEA + Box-Muller."""
    n = 2**20
    sig = dpd.make_signature(np.arange(1, n + 1, dtype=np.uint32),
                             np.random.default_rng(0).normal(size=(n, 3)))
    u = dpd.pair_uniforms(sig, np.roll(sig, 1), np.arange(1, n + 1), np.roll(np.arange(1, n + 1), 1),
                          0x8562613F)
    for fp32, hot in ((False, False), (True, False), (False, True)):
        xi = dpd.gaussian(u[:, 0], u[:, 1], fp32=fp32, hot=hot).astype(np.float64)
        m = xi.mean()
        v = xi.var()
        sk = ((xi - m) ** 3).mean() / v**1.5
        ku = ((xi - m) ** 4).mean() / v**2 - 3
        assert abs(m) <= 0.005 and abs(v - 1) <= 0.01 and abs(sk) <= 0.01 and abs(ku) <= 0.05


def test_morton():
    assert list(dpd.morton_encode([0, 1, 3], [0, 1, 1], [0, 1, 2], 2)) == [0, 7, 43]
    with pytest.raises(dpd.DPDError):
        dpd.morton_encode([4], [0], [0], 2)
