"""The header-only C++ drop-in (include/kronphi_b200/kronphi.hpp): compiles
here against the reference-named forwarding headers, and runs reference-style
C++ tests on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
SRC_INTEG = os.path.join(ROOT, "tests", "cpp", "test_integrators_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2304_02327_b200", "lib")


def build(out, src=SRC):
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(ROOT, "tests", "cpp"), src, "-o", out,
           "-L", LIBDIR, "-lkronphi_b200", f"-Wl,-rpath,{LIBDIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.parametrize("src", [SRC, SRC_INTEG])
def test_cpp_dropin_compiles(tmp_path, src):
    build(str(tmp_path / "t"), src)


@pytest.mark.gpu
@pytest.mark.parametrize("src", [SRC, SRC_INTEG])
def test_cpp_dropin_runs_on_gpu(tmp_path, src):
    exe = str(tmp_path / "t")
    build(exe, src)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
