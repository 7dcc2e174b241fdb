"""Builds and runs tests/cpp/test_gmux_dropin.cpp: the C++ drop-in header include/gmux/gmux.hpp
exercised like the reference's own Catch2 suites, linked against libgmi.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_gmux_dropin.cpp")
BIN = os.path.join(ROOT, "build", "test_gmux_dropin")
LIBDIR = os.path.join(ROOT, "paper_2206_08482_b200")


def _build():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    if os.path.exists(BIN) and os.path.getmtime(BIN) >= max(os.path.getmtime(SRC),
                                                             os.path.getmtime(os.path.join(LIBDIR, "libgmi.so"))):
        return
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", SRC, "-o", BIN, f"-L{LIBDIR}", "-lgmi",
                    f"-Wl,-rpath,{LIBDIR}"], check=True)


def test_dropin_cpu():
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_dropin_execute_on_device(cuda):
    _build()
    r = subprocess.run([BIN, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
