"""The header-only C++ mirror (paper_2006_06743_b200/cpp/include/sngb/sng.hpp)
compiles against include/sngb.h and links libsngb.so like a reference user's
program; without a GPU it throws (no CPU fallback), with one it reproduces
the SPEC example."""
import os
import subprocess

import pytest

import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = tmp_path / "demo"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(ROOT, "paper_2006_06743_b200", "cpp", "include"),
                    os.path.join(ROOT, "tests", "cpp", "cpp_mirror_demo.cpp"), "-L", libdir,
                    "-lsngb", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    return exe


def test_cpp_mirror_builds_and_fails_loudly_without_gpu(tmp_path):
    exe = _build(tmp_path)
    if sng.device_count() > 0:
        pytest.skip("a GPU is present (see the gpu-marked twin)")
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 3, r.stdout + r.stderr
    assert "no CUDA device" in r.stdout


@pytest.mark.gpu
def test_cpp_mirror_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True,
                       env={**os.environ, "DEMO_DIR": str(tmp_path)})
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fp64 via SNGD: clusters=2 ok=1" in r.stdout
    assert "exact: clusters=2 evals=6 full_edges=2" in r.stdout
    assert "multi: clusters=2 gpus=2" in r.stdout
