"""Builds tests/cpp/test_host_api.cpp against include/segconv_b200.hpp and the
in-tree libsegconv_b200.so and runs it (GPU).  The compile step alone is
checked on CPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_host_api.cpp")
STACK_SRC = os.path.join(ROOT, "tests", "cpp", "test_stack.cpp")
PKG = os.path.join(ROOT, "paper_2209_03704_b200")


def _build(out, src=SRC):
    cmd = ["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"),
           "-I/usr/local/cuda/include", src, "-o", out, "-L" + PKG, "-lsegconv_b200",
           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath," + PKG,
           "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_cpp_api_compiles(tmp_path):
    _build(str(tmp_path / "test_host_api"))


@pytest.mark.gpu
def test_cpp_api_runs(tmp_path):
    exe = _build(str(tmp_path / "test_host_api"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout


def test_cpp_stack_compiles(tmp_path):
    _build(str(tmp_path / "test_stack"), STACK_SRC)


@pytest.mark.gpu
def test_cpp_stack_runs(tmp_path):
    """segconv_stack_run / create / forward (C ABI multi-GPU driver) from C++ on
    every visible GPU, against a double-precision scatter chain."""
    exe = _build(str(tmp_path / "test_stack"), STACK_SRC)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout
