"""Pins the CPU oracle against the reference test suite's known-answer tests
and properties. The C++ program tests/cpp/oracle_kats.cpp re-derives each
reference test (file:line in every TEST name); this wrapper builds and runs it.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path_factory):
    out = tmp_path_factory.mktemp("kat") / "oracle_kats"
    cmd = ["g++", "-O2", "-std=c++20", "-o", str(out), os.path.join(ROOT, "tests/cpp/oracle_kats.cpp")]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return str(out)


@pytest.fixture(scope="module")
def kat_binary(tmp_path_factory):
    return _build(tmp_path_factory)


def test_oracle_reference_kats(kat_binary):
    r = subprocess.run([kat_binary], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "[FAIL]" not in r.stdout
