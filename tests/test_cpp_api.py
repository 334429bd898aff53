"""The C++ host API header (include/vecdyn_b200/vecdyn.hpp) compiles against
the C-ABI and, on a GPU, round-trips the batch API like a reference user."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "api_roundtrip.cpp")
LIBDIR = os.path.join(ROOT, "paper_2604_04310_b200", "lib")
BIN = os.path.join(ROOT, "tests", "cpp", "api_roundtrip")


def _build():
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", BIN, "-L", LIBDIR,
                    "-lvecdyn_cuda", f"-Wl,-rpath,{LIBDIR}"], check=True)


def test_cpp_header_compiles_and_links():
    _build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_api_roundtrip_on_gpu():
    if not os.path.exists(BIN):
        _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
