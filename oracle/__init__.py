"""ctypes loaders for the test-only checkers in oracle/.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  The product
package (paper_2006_06743_b200) never imports it and has no CPU fallback.

Two checkers:
  * ``Oracle``    -- oracle/sng_oracle.c, a C restatement of the reference hot
                     path (rng.hpp, graph.cpp:133-189, clusterer.cpp:7-65).
  * ``Reference`` -- oracle/_ref/libsngref.so, the reference's own
                     graph.cpp + clusterer.cpp compiled unmodified (oracle/Makefile).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libsng_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsngref.so")
REFERENCE_SRC = "/root/reference/proj"

_u64p = C.POINTER(C.c_uint64)


def build(quiet: bool = True) -> None:
    """Compile the restatement, and the reference shim when the sources exist."""
    targets = ["oracle"]
    if os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    subprocess.run(["make", "-C", HERE, *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


class Oracle:
    """C restatement (oracle/sng_oracle.c)."""

    ERRORS = {-1: "eps must be > 0", -2: "min_pts must be >= 1",
              -3: "rate must lie in (0, 1]", -4: "dataset is empty",
              -5: "dataset dimension must be >= 1",
              -6: "dataset contains a non-finite value"}

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_mix.restype = C.c_uint64
        L.orc_mix.argtypes = [C.c_uint64]
        L.orc_stream_key.restype = C.c_uint64
        L.orc_stream_key.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_stream_next.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.orc_stream_next_below.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.orc_draws.restype = C.c_uint64
        L.orc_draws.argtypes = [C.c_uint64, C.c_double]
        L.orc_partners.restype = C.c_uint64
        L.orc_partners.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                   C.POINTER(C.c_uint32)]
        L.orc_sampled_edges.restype = C.c_int
        L.orc_sampled_edges.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_uint32, C.c_double,
                                        C.c_double, C.c_uint64, C.c_int, C.POINTER(_u64p),
                                        _u64p, _u64p]
        L.orc_sampled_edges_rows.restype = C.c_int
        L.orc_sampled_edges_rows.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_uint32,
                                             C.c_double, C.c_double, C.c_uint64, C.c_int,
                                             C.c_uint64, C.c_uint64, C.POINTER(_u64p), _u64p,
                                             _u64p]
        L.orc_cluster_edges.restype = C.c_int
        L.orc_cluster_edges.argtypes = [_u64p, C.c_uint64, C.c_uint64, C.c_int32,
                                        C.POINTER(C.c_int32), C.POINTER(C.c_uint8),
                                        C.POINTER(C.c_int32)]
        L.orc_free.argtypes = [C.c_void_p]
        self.L = L

    def mix(self, z: int) -> int:
        return int(self.L.orc_mix(z))

    def stream_next(self, seed: int, sid: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self.L.orc_stream_next(seed, sid, count, _ptr(out, C.c_uint64))
        return out

    def stream_next_below(self, seed: int, sid: int, bound: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self.L.orc_stream_next_below(seed, sid, bound, count, _ptr(out, C.c_uint64))
        return out

    def draws(self, n: int, rate: float) -> int:
        return int(self.L.orc_draws(n, rate))

    def partners(self, n: int, draws: int, seed: int, u: int) -> np.ndarray:
        out = np.empty(max(draws, 1), np.uint32)
        k = self.L.orc_partners(n, draws, seed, u, _ptr(out, C.c_uint32))
        return out[:k]

    def sampled_edges(self, pts: np.ndarray, eps: float, rate: float, seed: int,
                      threads: int = 0):
        pts = np.ascontiguousarray(pts, np.float32)
        n, d = pts.shape
        kp = _u64p()
        nk = C.c_uint64()
        ev = C.c_uint64()
        rc = self.L.orc_sampled_edges(_ptr(pts, C.c_float), n, d, eps, rate, seed, threads,
                                      C.byref(kp), C.byref(nk), C.byref(ev))
        if rc:
            raise ValueError(self.ERRORS.get(rc, f"oracle error {rc}"))
        keys = np.ctypeslib.as_array(kp, shape=(nk.value,)).copy() if nk.value else \
            np.empty(0, np.uint64)
        self.L.orc_free(kp)
        return keys, int(ev.value)

    def sampled_edges_rows(self, pts: np.ndarray, eps: float, rate: float, seed: int,
                           row_begin: int, row_end: int, threads: int = 0):
        """Edges sampled by the query rows [row_begin, row_end) (a row shard)."""
        pts = np.ascontiguousarray(pts, np.float32)
        n, d = pts.shape
        kp = _u64p()
        nk = C.c_uint64()
        ev = C.c_uint64()
        rc = self.L.orc_sampled_edges_rows(_ptr(pts, C.c_float), n, d, eps, rate, seed, threads,
                                           row_begin, row_end, C.byref(kp), C.byref(nk),
                                           C.byref(ev))
        if rc:
            raise ValueError(self.ERRORS.get(rc, f"oracle error {rc}"))
        keys = np.ctypeslib.as_array(kp, shape=(nk.value,)).copy() if nk.value else \
            np.empty(0, np.uint64)
        self.L.orc_free(kp)
        return keys, int(ev.value)

    def cluster_edges(self, keys: np.ndarray, n: int, min_pts: int):
        keys = np.ascontiguousarray(keys, np.uint64)
        labels = np.empty(n, np.int32)
        roles = np.empty(n, np.uint8)
        cnt = C.c_int32()
        rc = self.L.orc_cluster_edges(_ptr(keys, C.c_uint64), len(keys), n, min_pts,
                                      _ptr(labels, C.c_int32), _ptr(roles, C.c_uint8),
                                      C.byref(cnt))
        if rc:
            raise ValueError(self.ERRORS.get(rc, f"oracle error {rc}"))
        return labels, roles, int(cnt.value)

    def sng_dbscan(self, pts: np.ndarray, eps: float, min_pts: int, rate: float, seed: int,
                   threads: int = 0):
        """Returns (labels, roles, info dict, keys)."""
        if not (eps > 0.0):
            raise ValueError(self.ERRORS[-1])
        if min_pts < 1:
            raise ValueError(self.ERRORS[-2])
        if not (rate > 0.0) or rate > 1.0:
            raise ValueError(self.ERRORS[-3])
        keys, evals = self.sampled_edges(pts, eps, rate, seed, threads)
        n = pts.shape[0]
        labels, roles, k = self.cluster_edges(keys, n, min_pts)
        info = {"distance_evals": evals, "edges": len(keys),
                "graph_bytes": (n + 1) * 8 + 2 * len(keys) * 4, "cluster_count": k}
        return labels, roles, info, keys


class Reference:
    """The reference's own sources compiled unmodified (oracle/_ref/libsngref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.sngref_last_error.restype = C.c_char_p
        L.sngref_hw_threads.restype = C.c_uint
        L.sngref_stream_next.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.sngref_stream_next_below.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                               _u64p]
        L.sngref_dataset_create.restype = C.c_void_p
        L.sngref_dataset_create.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_uint32]
        L.sngref_dataset_create_f64.restype = C.c_void_p
        L.sngref_dataset_create_f64.argtypes = [C.POINTER(C.c_double), C.c_uint64, C.c_uint32]
        L.sngref_dataset_free.argtypes = [C.c_void_p]
        L.sngref_dbscan.restype = C.c_int
        L.sngref_dbscan.argtypes = [C.c_void_p, C.c_double, C.c_int32, C.c_double, C.c_uint64,
                                    C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_uint8), _u64p,
                                    C.POINTER(C.c_double)]
        L.sngref_sampled_edges.restype = C.c_int
        L.sngref_sampled_edges.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_uint64,
                                           C.c_int, C.POINTER(_u64p), _u64p, _u64p,
                                           C.POINTER(C.c_double)]
        L.sngref_reference_dbscan.restype = C.c_int
        L.sngref_reference_dbscan.argtypes = [C.c_void_p, C.c_double, C.c_int32,
                                              C.POINTER(C.c_int32), C.POINTER(C.c_uint8)]
        L.sngref_free.argtypes = [C.c_void_p]
        L.sngref_set_metric.argtypes = [C.c_int]
        L.sngref_full_run.restype = C.c_int
        L.sngref_full_run.argtypes = [C.c_void_p, C.c_double, C.c_int32, C.c_double, C.c_uint64,
                                      C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_uint8), _u64p,
                                      C.POINTER(_u64p), _u64p, C.POINTER(C.c_double)]
        L.sngref_dbscan_exact.restype = C.c_int
        L.sngref_dbscan_exact.argtypes = [C.c_void_p, C.c_double, C.c_int32, C.c_int,
                                          C.POINTER(C.c_int32), C.POINTER(C.c_uint8), _u64p,
                                          C.POINTER(_u64p), _u64p, C.POINTER(C.c_double)]
        self.L = L

    def set_metric(self, name: str) -> None:
        """Distance for the next calls on this thread: euclidean / manhattan / cosine."""
        self.L.sngref_set_metric({"euclidean": 0, "manhattan": 1, "cosine": 2}[name])

    def hw_threads(self) -> int:
        return int(self.L.sngref_hw_threads())

    def _err(self):
        return ValueError(self.L.sngref_last_error().decode())

    def stream_next(self, seed, sid, count):
        out = np.empty(count, np.uint64)
        self.L.sngref_stream_next(seed, sid, count, _ptr(out, C.c_uint64))
        return out

    def stream_next_below(self, seed, sid, bound, count):
        out = np.empty(count, np.uint64)
        self.L.sngref_stream_next_below(seed, sid, bound, count, _ptr(out, C.c_uint64))
        return out

    def dataset(self, pts: np.ndarray):
        """Widen fp32 (or take fp64) rows into an sng::Dataset (outside timing)."""
        if pts.dtype == np.float64:
            pts = np.ascontiguousarray(pts)
            h = self.L.sngref_dataset_create_f64(_ptr(pts, C.c_double), pts.shape[0], pts.shape[1])
        else:
            pts = np.ascontiguousarray(pts, np.float32)
            h = self.L.sngref_dataset_create(_ptr(pts, C.c_float), pts.shape[0], pts.shape[1])
        if not h:
            raise self._err()
        return _Dataset(self, h, pts.shape[0])

    def sng_dbscan(self, ds: "_Dataset", eps, min_pts, rate, seed, threads=0):
        """Returns (labels, roles, info dict incl. wall 'ms')."""
        labels = np.empty(ds.n, np.int32)
        roles = np.empty(ds.n, np.uint8)
        info = np.zeros(4, np.uint64)
        ms = C.c_double()
        rc = self.L.sngref_dbscan(ds.h, eps, min_pts, rate, seed, threads,
                                  _ptr(labels, C.c_int32), _ptr(roles, C.c_uint8),
                                  _ptr(info, C.c_uint64), C.byref(ms))
        if rc:
            raise self._err()
        return labels, roles, {"distance_evals": int(info[0]), "edges": int(info[1]),
                               "graph_bytes": int(info[2]), "cluster_count": int(info[3]),
                               "ms": ms.value}

    def sampled_edges(self, ds: "_Dataset", eps, rate, seed, threads=0):
        kp = _u64p()
        nk = C.c_uint64()
        ev = C.c_uint64()
        ms = C.c_double()
        rc = self.L.sngref_sampled_edges(ds.h, eps, rate, seed, threads, C.byref(kp),
                                         C.byref(nk), C.byref(ev), C.byref(ms))
        if rc:
            raise self._err()
        keys = np.ctypeslib.as_array(kp, shape=(nk.value,)).copy() if nk.value else \
            np.empty(0, np.uint64)
        self.L.sngref_free(kp)
        return keys, int(ev.value), ms.value

    def _keys(self, kp, nk):
        keys = np.ctypeslib.as_array(kp, shape=(nk.value,)).copy() if nk.value else \
            np.empty(0, np.uint64)
        self.L.sngref_free(kp)
        return keys

    @staticmethod
    def _info(info, ms):
        return {"distance_evals": int(info[0]), "edges": int(info[1]),
                "graph_bytes": int(info[2]), "cluster_count": int(info[3]), "ms": ms.value}

    def full_run(self, ds: "_Dataset", eps, min_pts, rate, seed, threads=0):
        """sng_dbscan with ONE graph build that also returns the canonical edge
        keys: (labels, roles, info, keys).  Same code as sng_dbscan
        (clusterer.cpp:54-65): build_sampled_graph then cluster_graph."""
        labels = np.empty(ds.n, np.int32)
        roles = np.empty(ds.n, np.uint8)
        info = np.zeros(4, np.uint64)
        kp, nk, ms = _u64p(), C.c_uint64(), C.c_double()
        rc = self.L.sngref_full_run(ds.h, eps, min_pts, rate, seed, threads,
                                    _ptr(labels, C.c_int32), _ptr(roles, C.c_uint8),
                                    _ptr(info, C.c_uint64), C.byref(kp), C.byref(nk),
                                    C.byref(ms))
        if rc:
            raise self._err()
        return labels, roles, self._info(info, ms), self._keys(kp, nk)

    def dbscan_exact(self, ds: "_Dataset", eps, min_pts, threads=0, with_keys=True):
        """sng::dbscan_exact (clusterer.cpp:67-79): (labels, roles, info, keys|None)."""
        labels = np.empty(ds.n, np.int32)
        roles = np.empty(ds.n, np.uint8)
        info = np.zeros(4, np.uint64)
        kp, nk, ms = _u64p(), C.c_uint64(), C.c_double()
        rc = self.L.sngref_dbscan_exact(ds.h, eps, min_pts, threads, _ptr(labels, C.c_int32),
                                        _ptr(roles, C.c_uint8), _ptr(info, C.c_uint64),
                                        C.byref(kp) if with_keys else None,
                                        C.byref(nk), C.byref(ms))
        if rc:
            raise self._err()
        return labels, roles, self._info(info, ms), (self._keys(kp, nk) if with_keys else None)

    def reference_dbscan(self, ds: "_Dataset", eps, min_pts):
        labels = np.empty(ds.n, np.int32)
        core = np.empty(ds.n, np.uint8)
        rc = self.L.sngref_reference_dbscan(ds.h, eps, min_pts, _ptr(labels, C.c_int32),
                                            _ptr(core, C.c_uint8))
        if rc:
            raise self._err()
        return labels, core


class _Dataset:
    def __init__(self, ref: Reference, h, n: int):
        self.ref, self.h, self.n = ref, h, n

    def __del__(self):
        try:
            self.ref.L.sngref_dataset_free(self.h)
        except Exception:
            pass


def fnv1a64_u32(values: np.ndarray) -> int:
    """FNV-1a-64 over little-endian u32 bytes (SURVEY.md Appendix A hash)."""
    h = 1469598103934665603
    for b in np.ascontiguousarray(values, "<u4").tobytes():
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h
