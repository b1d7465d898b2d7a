"""The drop-in C++ API (include/nrr/*.hpp over libnrr_b200.so) against the CPU
oracle, per module: tests/cpp/product_kats.cpp. The CPU test only proves the
headers compile and link against every exported symbol; the GPU test runs it.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2206_03410_b200")


def _build(out):
    from paper_2206_03410_b200.build import build_library

    build_library()
    cmd = ["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"), "-o", str(out),
           os.path.join(ROOT, "tests/cpp/product_kats.cpp"), "-L", LIBDIR, "-lnrr_b200",
           "-Wl,-rpath," + LIBDIR]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return str(out)


def test_product_headers_compile_and_link(tmp_path):
    assert os.path.exists(_build(tmp_path / "product_kats"))


@pytest.mark.gpu
def test_product_kats(tmp_path):
    exe = _build(tmp_path / "product_kats")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "[FAIL]" not in r.stdout
