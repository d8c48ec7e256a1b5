"""The C-ABI boundary: libdpdb.so loads, exports every symbol include/dpdb.h
declares, carries sm_100a code only, and refuses to run without a B200 (no
CPU fallback).  No compute calls here -- this runs on the CPU box.
"""
import ctypes as C
import os
import re
import shutil
import subprocess

import pytest

import paper_1311_0402_b200 as dpd
from paper_1311_0402_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "dpdb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dpdb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    names = header_functions()
    assert len(names) >= 30
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_lib.SYMBOLS), set(names) ^ set(_lib.SYMBOLS)
    assert L.dpdb_version().decode().startswith("dpdb")


def test_shim_header_compiles():
    """include/dpd_b200.hpp (C++ shim mirroring the reference API) compiles."""
    gxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    src = os.path.join(ROOT, "include", "dpd_b200.hpp")
    if not os.path.exists(src):
        pytest.skip("shim header not present")
    r = subprocess.run([gxx, "-std=c++20", "-fsyntax-only", "-x", "c++", "-I",
                        os.path.join(ROOT, "include"), src], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def build_shim_example(outdir):
    """Compile + link tests/cpp/shim_smoke.cpp against libdpdb.so (no GPU needed)."""
    gxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else shutil.which("g++")
    libdir = os.path.dirname(_lib.LIB_PATH)
    exe = os.path.join(outdir, "shim_smoke")
    r = subprocess.run([gxx, "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "shim_smoke.cpp"), "-L", libdir,
                        "-ldpdb", f"-Wl,-rpath,{libdir}", "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_shim_example_links(tmp_path):
    # libdpdb.so must be linkable as -ldpdb: provide the conventional soname link
    libdir = os.path.dirname(_lib.LIB_PATH)
    assert os.path.exists(os.path.join(libdir, "libdpdb.so"))
    build_shim_example(str(tmp_path))


def test_sm100a_only():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump missing")
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_cpu_fallback_without_gpu():
    if dpd.device_count() > 0:
        pytest.skip("a B200 is present; the no-GPU refusal is tested on CPU boxes")
    with pytest.raises(dpd.DPDError) as e:
        dpd.Engine(dpd.SimBox(hi=(8, 8, 8)), dpd.PairParams(), dpd.RunConfig(), capacity=10)
    assert e.value.code == 5


def test_config_errors_before_device():
    """Configuration is validated like the reference (config = 1) before any device work."""
    with pytest.raises(dpd.DPDError) as e:
        dpd.Engine(dpd.SimBox(hi=(8, 8, 8)), dpd.PairParams(r_c=-1.0), dpd.RunConfig())
    assert e.value.code == 1
    with pytest.raises(dpd.DPDError) as e:
        dpd.Engine(dpd.SimBox(hi=(8, 8, 8)), dpd.PairParams(), dpd.RunConfig(max_neighbors=100))
    assert e.value.code == 1
    with pytest.raises(dpd.DPDError) as e:
        dpd.Engine(dpd.SimBox(hi=(8, 0.5, 8)), dpd.PairParams(), dpd.RunConfig())
    assert e.value.code == 1
    with pytest.raises(dpd.DPDError) as e:
        dpd.radix_sort(*(__import__("numpy").zeros(4, "uint32") for _ in range(2)), 6)
    assert e.value.code == 1


def test_shim_minimum_image_examples(tmp_path):
    """S:55-60 examples through the C++ shim's minimum_image (header-only, no GPU)."""
    src = tmp_path / "mi.cpp"
    src.write_text('''#include "dpd_b200.hpp"
#include <cstdio>
using namespace dpd::b200;
int main() {
    SimBox b;
    b.hi = {12.0, 8.0, 8.0};
    b.periodic = {true, true, false};
    Vec3 z = minimum_image({0, 0, 0}, b), w = minimum_image({7, -4.5, 30}, b);
    std::printf("%g %g %g %g %g %g\\n", z.x, z.y, z.z, w.x, w.y, w.z);
    return 0;
}
''')
    exe = tmp_path / "mi"
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert [float(v) for v in out] == [0, 0, 0, -5, 3.5, 30]  # L_x = 12: 7 -> -5; wall/free axis unchanged
