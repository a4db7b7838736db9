"""ctypes binding of libsngb.so (include/sngb.h).

This is the reference-side binding a maintainer would add for the
``sngdbscan`` Python module the reference planned (proj/CMakeLists.txt:11,
proj/python/CMakeLists.txt:1 is a placeholder).  There is no CPU fallback: if
the library is missing the import fails loudly, and on a host without a GPU
every compute call returns SNGB_ERR_NO_DEVICE.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SNGB_LIBRARY") or os.path.join(PKG, "lib", "libsngb.so")

SNGB_OK = 0
SNGB_ERR_EPS = 1
SNGB_ERR_MINPTS = 2
SNGB_ERR_RATE = 3
SNGB_ERR_EMPTY = 4
SNGB_ERR_DIM = 5
SNGB_ERR_NONFINITE = 6
SNGB_ERR_TOO_LARGE = 7
SNGB_ERR_ARG = 8
SNGB_ERR_NO_DEVICE = 9
SNGB_ERR_CUDA = 10
SNGB_ERR_CAPACITY = 11
SNGB_ERR_ZERO_VECTOR = 12
SNGB_FLAG_TIMING = 0x1
SNGB_FLAG_MANHATTAN = 0x2
SNGB_FLAG_COSINE = 0x4

# Every symbol include/sngb.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "sngb_dbscan_f32", "sngb_dbscan_f32_device", "sngb_sampled_edges_f32_device",
    "sngb_sampled_edges_f32", "sngb_cluster_edges_device", "sngb_strerror",
    "sngb_last_error_detail", "sngb_abi_version", "sngb_device_count", "sngb_release_pools",
    "sngb_unique_keys_device", "sngb_degrees_device", "sngb_components_device",
    "sngb_border_device", "sngb_relabel_device",
    "sngb_dbscan_f64", "sngb_dbscan_f64_device", "sngb_sampled_edges_f64",
    "sngb_dbscan_batch_f32",
    "sngb_dbscan_exact_f32", "sngb_dbscan_exact_f32_device", "sngb_dbscan_exact_f64",
    "sngb_full_edges_f32",
]


class SngbOpts(C.Structure):
    _fields_ = [("device", C.c_int32), ("flags", C.c_uint32), ("stream", C.c_void_p),
                ("row_begin", C.c_uint64), ("row_end", C.c_uint64),
                # ABI 4: GPUs of this process (0/1: one; N; -1: all) and their ordinals
                ("num_gpus", C.c_int32), ("devices", C.POINTER(C.c_int32))]


class SngbInfo(C.Structure):
    _fields_ = [
        ("distance_evals", C.c_uint64), ("edges", C.c_uint64), ("graph_bytes", C.c_uint64),
        ("cluster_count", C.c_int32), ("core_count", C.c_uint32), ("border_count", C.c_uint32),
        ("noise_count", C.c_uint32),
        ("draws", C.c_uint64), ("collisions", C.c_uint64), ("irregular_vertices", C.c_uint64),
        ("pairs_evaluated", C.c_uint64), ("band_rechecks", C.c_uint64), ("band_1e6", C.c_uint64),
        ("fp32_flips", C.c_uint64), ("directed_accepts", C.c_uint64),
        ("ms_total", C.c_float), ("ms_upload", C.c_float), ("ms_sample", C.c_float),
        ("ms_gather", C.c_float), ("ms_extras", C.c_float), ("ms_sort", C.c_float),
        ("ms_cluster", C.c_float), ("ms_download", C.c_float),
        ("gather_pairs", C.c_uint64), ("gather_bytes", C.c_uint64),
        ("kernel_launches", C.c_uint64), ("library_launches", C.c_uint64),
        ("filter_bits", C.c_uint32), ("head_bytes", C.c_uint32),
        ("num_gpus", C.c_uint32), ("merge_rounds", C.c_uint32), ("routed_keys", C.c_uint64),
        ("ms_merge", C.c_float), ("reserved", C.c_uint32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class SngbProblem(C.Structure):
    _fields_ = [("pts", C.c_void_p), ("n", C.c_uint64), ("d", C.c_uint32), ("flags", C.c_uint32),
                ("eps", C.c_double), ("rate", C.c_double), ("seed", C.c_uint64),
                ("min_pts", C.c_int32), ("status", C.c_int32), ("labels_out", C.c_void_p),
                ("roles_out", C.c_void_p), ("info_out", C.c_void_p)]


_lib = None


def lib() -> C.CDLL:
    """Load libsngb.so once.  Raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        _lib = load(LIB_PATH)
    return _lib


def load(path: str) -> C.CDLL:
    """Load and declare one build of the library (the product, or an A/B or
    test-hook build of the same sources)."""
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2006_06743_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(path)
    f32p, u64p, i32p, u8p = (C.POINTER(C.c_float), C.POINTER(C.c_uint64),
                             C.POINTER(C.c_int32), C.POINTER(C.c_uint8))
    optp, infop = C.POINTER(SngbOpts), C.POINTER(SngbInfo)
    vp = C.c_void_p
    L.sngb_dbscan_f32.restype = C.c_int
    L.sngb_dbscan_f32.argtypes = [f32p, C.c_uint64, C.c_uint32, C.c_double, C.c_int32,
                                  C.c_double, C.c_uint64, optp, i32p, u8p, infop]
    L.sngb_dbscan_f32_device.restype = C.c_int
    L.sngb_dbscan_f32_device.argtypes = [vp, C.c_uint64, C.c_uint32, C.c_double, C.c_int32,
                                         C.c_double, C.c_uint64, optp, vp, vp, infop]
    L.sngb_sampled_edges_f32_device.restype = C.c_int
    L.sngb_sampled_edges_f32_device.argtypes = [vp, C.c_uint64, C.c_uint32, C.c_double,
                                                C.c_double, C.c_uint64, optp, vp, C.c_uint64,
                                                u64p, infop]
    L.sngb_sampled_edges_f32.restype = C.c_int
    L.sngb_sampled_edges_f32.argtypes = [f32p, C.c_uint64, C.c_uint32, C.c_double,
                                         C.c_double, C.c_uint64, optp, u64p, C.c_uint64, u64p,
                                         infop]
    L.sngb_cluster_edges_device.restype = C.c_int
    L.sngb_cluster_edges_device.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_int32, optp, vp,
                                            vp, infop]
    L.sngb_unique_keys_device.restype = C.c_int
    L.sngb_unique_keys_device.argtypes = [vp, C.c_uint64, C.c_uint64, optp, vp, u64p]
    L.sngb_degrees_device.restype = C.c_int
    L.sngb_degrees_device.argtypes = [vp, C.c_uint64, C.c_uint64, optp, vp]
    L.sngb_components_device.restype = C.c_int
    L.sngb_components_device.argtypes = [vp, C.c_uint64, C.c_uint64, vp, C.c_int32, optp, vp,
                                         u64p]
    L.sngb_border_device.restype = C.c_int
    L.sngb_border_device.argtypes = [vp, C.c_uint64, C.c_uint64, vp, C.c_int32, vp, optp, vp]
    L.sngb_relabel_device.restype = C.c_int
    L.sngb_relabel_device.argtypes = [C.c_uint64, vp, C.c_int32, vp, vp, optp, vp, vp, infop]
    f64p = C.POINTER(C.c_double)
    L.sngb_dbscan_f64.restype = C.c_int
    L.sngb_dbscan_f64.argtypes = [f64p, C.c_uint64, C.c_uint32, C.c_double, C.c_int32,
                                  C.c_double, C.c_uint64, optp, i32p, u8p, infop]
    L.sngb_dbscan_f64_device.restype = C.c_int
    L.sngb_dbscan_f64_device.argtypes = [vp, C.c_uint64, C.c_uint32, C.c_double, C.c_int32,
                                         C.c_double, C.c_uint64, optp, vp, vp, infop]
    L.sngb_sampled_edges_f64.restype = C.c_int
    L.sngb_sampled_edges_f64.argtypes = [f64p, C.c_uint64, C.c_uint32, C.c_double,
                                         C.c_double, C.c_uint64, optp, u64p, C.c_uint64, u64p,
                                         infop]
    L.sngb_dbscan_batch_f32.restype = C.c_int
    L.sngb_dbscan_batch_f32.argtypes = [C.POINTER(SngbProblem), C.c_uint64, optp]
    L.sngb_dbscan_exact_f32.restype = C.c_int
    L.sngb_dbscan_exact_f32.argtypes = [f32p, C.c_uint64, C.c_uint32, C.c_double, C.c_int32,
                                        optp, i32p, u8p, infop]
    L.sngb_dbscan_exact_f32_device.restype = C.c_int
    L.sngb_dbscan_exact_f32_device.argtypes = [vp, C.c_uint64, C.c_uint32, C.c_double,
                                               C.c_int32, optp, vp, vp, infop]
    L.sngb_dbscan_exact_f64.restype = C.c_int
    L.sngb_dbscan_exact_f64.argtypes = [f64p, C.c_uint64, C.c_uint32, C.c_double, C.c_int32,
                                        optp, i32p, u8p, infop]
    L.sngb_full_edges_f32.restype = C.c_int
    L.sngb_full_edges_f32.argtypes = [f32p, C.c_uint64, C.c_uint32, C.c_double, optp, u64p,
                                      C.c_uint64, u64p, infop]
    L.sngb_strerror.restype = C.c_char_p
    L.sngb_strerror.argtypes = [C.c_int]
    L.sngb_last_error_detail.restype = C.c_char_p
    L.sngb_abi_version.restype = C.c_int
    L.sngb_device_count.restype = C.c_int
    L.sngb_release_pools.restype = None
    return L


def strerror(code: int) -> str:
    return lib().sngb_strerror(code).decode()


def last_error_detail() -> str:
    return lib().sngb_last_error_detail().decode()
