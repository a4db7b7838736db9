"""The C ABI library (libsngb.so): loads, exports every symbol include/sngb.h
declares, struct layouts agree with the ctypes mirror, error behaviour.
CPU only -- no compute call needs a GPU here (and must fail loudly without one)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sngb.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|void)\s+(sngb_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/sngb.h but not exported"
    assert sorted(_lib.EXPORTS) == syms


def test_exported_via_nm_dynamic():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    for s in header_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_struct_layout_matches_header(tmp_path):
    fields_info = [f for f, _ in _lib.SngbInfo._fields_]
    fields_opts = [f for f, _ in _lib.SngbOpts._fields_]
    prog = ["#include <stdio.h>", "#include <stddef.h>", '#include "sngb.h"', "int main(void){",
            'printf("%zu %zu\\n", sizeof(sngb_info), sizeof(sngb_opts));']
    for f in fields_info:
        prog.append(f'printf("%zu\\n", offsetof(sngb_info, {f}));')
    for f in fields_opts:
        prog.append(f'printf("%zu\\n", offsetof(sngb_opts, {f}));')
    prog.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(prog))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    vals = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert int(vals[0]) == C.sizeof(_lib.SngbInfo)
    assert int(vals[1]) == C.sizeof(_lib.SngbOpts)
    offs = [int(v) for v in vals[2:]]
    want = [getattr(_lib.SngbInfo, f).offset for f in fields_info] + \
        [getattr(_lib.SngbOpts, f).offset for f in fields_opts]
    assert offs == want


def test_strerror_carries_reference_messages():
    # clusterer.hpp:20-22, graph.cpp:18, dataset.hpp:22,26
    assert _lib.strerror(1) == "eps must be > 0"
    assert _lib.strerror(2) == "min_pts must be >= 1"
    assert _lib.strerror(3) == "rate must lie in (0, 1]"
    assert _lib.strerror(4) == "dataset is empty"
    assert _lib.strerror(5) == "dataset dimension must be >= 1"
    assert _lib.strerror(6) == "dataset contains a non-finite value"
    assert int(_lib.lib().sngb_abi_version()) == 4


def _call(pts, eps=1.0, min_pts=1, rate=1.0, seed=0):
    n, d = pts.shape if pts.size else (0, pts.shape[1] if pts.ndim == 2 else 1)
    labels = np.empty(max(n, 1), np.int32)
    roles = np.empty(max(n, 1), np.uint8)
    info = _lib.SngbInfo()
    return _lib.lib().sngb_dbscan_f32(
        pts.ctypes.data_as(C.POINTER(C.c_float)), n, d, eps, min_pts, rate, seed, None,
        labels.ctypes.data_as(C.POINTER(C.c_int32)), roles.ctypes.data_as(C.POINTER(C.c_uint8)),
        C.byref(info))


def test_parameter_errors_precede_device_work():
    pts = np.zeros((4, 2), np.float32)
    assert _call(pts, eps=0.0) == _lib.SNGB_ERR_EPS
    assert _call(pts, eps=float("nan")) == _lib.SNGB_ERR_EPS
    assert _call(pts, min_pts=0) == _lib.SNGB_ERR_MINPTS
    assert _call(pts, rate=0.0) == _lib.SNGB_ERR_RATE
    assert _call(pts, rate=1.0000001) == _lib.SNGB_ERR_RATE
    assert _call(np.zeros((0, 2), np.float32)) == _lib.SNGB_ERR_EMPTY


def test_no_cpu_fallback_without_gpu():
    if sng.device_count() > 0:
        pytest.skip("a GPU is present")
    pts = np.zeros((4, 2), np.float32)
    assert _call(pts) == _lib.SNGB_ERR_NO_DEVICE
    with pytest.raises(sng.GpuError, match="no CUDA device"):
        sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=1.0, min_pts=1, rate=1.0))


def _edges_call(n, d, eps, rate):
    pts = np.zeros((max(n, 1), max(d, 1)), np.float32)
    cnt = C.c_uint64(0)
    keys = np.zeros(4, np.uint64)
    return _lib.lib().sngb_sampled_edges_f32(
        pts.ctypes.data_as(C.POINTER(C.c_float)), n, d, eps, rate, 0, None,
        keys.ctypes.data_as(C.POINTER(C.c_uint64)), 4, C.byref(cnt), None)


def test_sampled_edges_validation_order_is_build_sampled_graph():
    """build_sampled_graph alone checks empty, eps, dim (graph.cpp:17-21), then the
    rate (graph.cpp:136); sng_dbscan validates its params first (clusterer.hpp:19-23)."""
    assert _edges_call(0, 2, -1.0, 7.0) == _lib.SNGB_ERR_EMPTY
    assert _edges_call(4, 2, -1.0, 7.0) == _lib.SNGB_ERR_EPS
    assert _edges_call(4, 0, 1.0, 7.0) == _lib.SNGB_ERR_DIM
    assert _edges_call(4, 2, 1.0, 7.0) == _lib.SNGB_ERR_RATE
    # sng_dbscan: params before the dataset
    assert _call(np.zeros((0, 2), np.float32), eps=-1.0) == _lib.SNGB_ERR_EPS
    assert _call(np.zeros((0, 2), np.float32), rate=2.0) == _lib.SNGB_ERR_RATE
