"""GhostPacket wire format: fixed little-endian
layout, header checks, round trips.  CPU only."""
import struct

import numpy as np
import pytest

from paper_1311_0402_b200 import DPDError
from paper_1311_0402_b200 import wire as W


def recs(n, seed=0):
    rng = np.random.default_rng(seed)
    r = np.zeros(n, W.DEV_REC)
    r["x"] = rng.normal(size=(n, 3))
    r["v"] = rng.normal(size=(n, 3))
    r["tag"] = rng.integers(1, 2**31, n)
    r["sp_mol"] = rng.integers(0, 4, n) | (rng.integers(0, 2**24, n) << 8)
    return r


def test_ghost_full_layout_and_round_trip():
    r = recs(3)
    pkt = W.encode(W.KIND_GHOST_FULL, 17, r)
    assert struct.unpack_from("<IIII", pkt) == (0x44504447, 0, 17, 3)
    assert len(pkt) == 16 + 3 * 57
    # first record: tag, species, x, v, molecule at fixed offsets
    tag, sp = struct.unpack_from("<IB", pkt, 16)
    assert tag == r["tag"][0] and sp == r["sp_mol"][0] & 0xFF
    assert struct.unpack_from("<3d", pkt, 21) == tuple(r["x"][0])
    assert struct.unpack_from("<3d", pkt, 45) == tuple(r["v"][0])
    assert struct.unpack_from("<I", pkt, 69)[0] == r["sp_mol"][0] >> 8
    kind, step, back = W.decode(pkt)
    assert kind == W.KIND_GHOST_FULL and step == 17 and back.tobytes() == r.tobytes()


def test_update_and_stray():
    u = np.zeros(4, W.DEV_UPD)
    u["x"] = np.arange(12.0).reshape(4, 3)
    u["v"] = -u["x"]
    pkt = W.encode(W.KIND_GHOST_UPDATE, 5, u)
    assert len(pkt) == 16 + 4 * 48
    assert W.decode(pkt, W.KIND_GHOST_UPDATE)[2].tobytes() == u.tobytes()
    r = recs(2, 1)
    pkt = W.encode(W.KIND_STRAY, 9, r)
    assert len(pkt) == 16 + 2 * 81
    assert struct.unpack_from("<3d", pkt, 16 + 57) == (0.0, 0.0, 0.0)  # force words
    assert W.decode(pkt)[2].tobytes() == r.tobytes()
    assert W.decode(W.encode(W.KIND_STRAY, 0, r[:0]))[2].size == 0


@pytest.mark.parametrize("mutate,needle", [
    (lambda p: b"XXXX" + p[4:], "bad magic"),
    (lambda p: p[:-1], "count does not match"),
    (lambda p: p[:8], "truncated"),
    (lambda p: struct.pack("<IIII", 0x44504447, 7, 0, 0), "unknown kind"),
])
def test_bad_packets(mutate, needle):
    pkt = W.encode(W.KIND_GHOST_FULL, 1, recs(2))
    with pytest.raises(DPDError) as ex:
        W.decode(mutate(pkt))
    assert needle in str(ex.value)


def test_kind_desync_is_an_error():
    with pytest.raises(DPDError) as ex:
        W.decode(W.encode(W.KIND_GHOST_FULL, 1, recs(1)), W.KIND_GHOST_UPDATE)
    assert "desync" in str(ex.value)
