"""Reader for the record files tests/cpp/ref_caller.cpp writes, and the
runner for its two builds (REF: oracle/_ref/ref_caller; B200:
dropin/_build/b200_caller)."""
import os
import struct
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "ref_caller")
B200_BIN = os.path.join(ROOT, "dropin", "_build", "b200_caller")
_DT = {0: np.uint32, 1: np.float64, 2: np.uint16}


def read_records(path):
    out = {}
    with open(path, "rb") as f:
        while True:
            h = f.read(4)
            if len(h) < 4:
                break
            (ln,) = struct.unpack("<I", h)
            name = f.read(ln).decode()
            dtype, cnt = struct.unpack("<IQ", f.read(12))
            dt = np.dtype(_DT[dtype])
            out[name] = np.frombuffer(f.read(cnt * dt.itemsize), dt).copy()
    return out


def run(binary, L, out, timeout=600):
    p = subprocess.run([binary, str(L), out], capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stderr, read_records(out)
