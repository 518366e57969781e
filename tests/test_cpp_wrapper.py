"""The header-only C++ drop-in (include/tokenselect.hpp): compiles against the
C ABI here (no GPU), and runs its reference-style checks on the GPU."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "wrapper_test.cpp")
LIBDIR = os.path.join(ROOT, "paper_2411_02886_b200", "_build")


def _gxx():
    g = shutil.which("g++")
    if not g:
        pytest.skip("g++ not available")
    return g


def test_wrapper_compiles():
    r = subprocess.run([_gxx(), "-std=c++17", "-fsyntax-only", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        SRC], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_wrapper_runs(tmp_path):
    exe = str(tmp_path / "wrapper_test")
    r = subprocess.run([_gxx(), "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                        "-L", LIBDIR, "-ltokenselect", f"-Wl,-rpath,{LIBDIR}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout + r.stderr
