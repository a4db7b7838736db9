"""sngdbscan on B200 -- Python mirror of the reference's SNG-DBSCAN entry point.

Same names, argument meaning and error behaviour as the reference C++ API
(proj/include/sng/clusterer.hpp, graph.hpp, dataset.hpp):

    from paper_2006_06743_b200 import Dataset, SngParams, ClusterRunInfo, sng_dbscan
    c = sng_dbscan(Dataset(points), SngParams(eps=0.03, min_pts=10, rate=0.1, seed=1), info)
    c.assignment, c.role, c.cluster_count

Every call runs on the GPU through the C ABI (include/sngb.h, libsngb.so).
``std::invalid_argument`` maps to :class:`InvalidArgument` (a ValueError)
with the reference's message.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import SNGB_FLAG_TIMING, SngbInfo, SngbOpts

__all__ = [
    "InvalidArgument", "GpuError", "kNoiseLabel", "PointRole", "Dataset", "Distance",
    "SngParams", "ClusterRunInfo", "BuildStats", "Clustering", "SampledGraph",
    "sng_dbscan", "build_sampled_graph", "cluster_graph", "sng_dbscan_device", "dbscan_exact",
    "build_full_graph", "dbscan_exact_device",
    "sampled_edges_device", "cluster_edges_device", "device_count",
]

kNoiseLabel = -1  # dataset.hpp:13


class InvalidArgument(ValueError):
    """std::invalid_argument of the reference (same messages)."""


class GpuError(RuntimeError):
    """CUDA failure or no usable GPU (the library has no CPU fallback)."""


class PointRole(enum.IntEnum):  # dataset.hpp:74
    Core = 0
    Border = 1
    Noise = 2


def _check(rc: int) -> None:
    if rc == _lib.SNGB_OK:
        return
    msg = _lib.strerror(rc)
    if rc in (_lib.SNGB_ERR_EPS, _lib.SNGB_ERR_MINPTS, _lib.SNGB_ERR_RATE, _lib.SNGB_ERR_EMPTY,
              _lib.SNGB_ERR_DIM, _lib.SNGB_ERR_NONFINITE, _lib.SNGB_ERR_TOO_LARGE,
              _lib.SNGB_ERR_ARG, _lib.SNGB_ERR_ZERO_VECTOR):
        raise InvalidArgument(msg)
    if rc == _lib.SNGB_ERR_CUDA:
        msg = f"{msg}: {_lib.last_error_detail()}"
    raise GpuError(msg)


def device_count() -> int:
    return int(_lib.lib().sngb_device_count())


class Distance:
    """distance.hpp: Euclidean, Manhattan and cosine run on the GPU path (the
    fp32 filter plus the reference's fp64 recheck); a Python callback (the
    reference's Metric::Custom) cannot, and raises NotImplementedError."""

    _FLAGS = {"euclidean": 0, "manhattan": 0x2, "cosine": 0x4}

    def __init__(self, kind: str = "euclidean"):
        if kind not in self._FLAGS:
            raise NotImplementedError(f"distance '{kind}' is not on the B200 hot path")
        self.kind = kind

    @property
    def flags(self) -> int:
        return self._FLAGS[self.kind]

    @staticmethod
    def euclidean() -> "Distance":
        return Distance("euclidean")

    @staticmethod
    def manhattan() -> "Distance":
        return Distance("manhattan")

    @staticmethod
    def cosine() -> "Distance":
        return Distance("cosine")

    @staticmethod
    def custom(fn, expected_dim=None) -> "Distance":
        raise NotImplementedError("a Python distance callback cannot run on the GPU path")

    @staticmethod
    def parse(name: str) -> "Distance":  # distance.hpp:37-43
        if name not in ("euclidean", "manhattan", "cosine"):
            raise InvalidArgument(
                f"unknown distance '{name}' (expected euclidean, manhattan, or cosine)")
        return Distance(name)


class Dataset:
    """Row-major n x dim matrix of finite reals (dataset.hpp:16-71).

    fp32 input, and fp64 input whose values are all exactly fp32, are stored as
    fp32 (widening back is exact).  Other fp64 input is kept in fp64
    (``values64``) and runs the fp64 entry points, which filter on rounded
    values with a widened guard band and recheck in fp64 -- the reference's
    results either way.
    """

    def __init__(self, values, dim: int | None = None):
        a = np.asarray(values)
        if dim is not None:
            if dim == 0:
                raise InvalidArgument("dataset dimension must be >= 1")
            flat = a.reshape(-1)
            if flat.size == 0 or flat.size % dim != 0:
                raise InvalidArgument("dataset values do not form n x dim rows")
            a = flat.reshape(-1, dim)
        if a.ndim != 2:
            raise InvalidArgument("dataset values do not form n x dim rows")
        if a.shape[1] == 0:
            raise InvalidArgument("dataset dimension must be >= 1")
        if a.shape[0] == 0:
            raise InvalidArgument("dataset values do not form n x dim rows")
        self.values64 = None
        if a.dtype == np.float32:
            f = np.ascontiguousarray(a)
        else:
            a64 = np.ascontiguousarray(a, np.float64)
            if not np.isfinite(a64).all():
                raise InvalidArgument("dataset contains a non-finite value")
            with np.errstate(over="ignore"):
                f = np.ascontiguousarray(a64.astype(np.float32))
            if not np.array_equal(f.astype(np.float64), a64):
                self.values64 = a64  # not exactly fp32: the fp64 path
        if not np.isfinite(f).all() and self.values64 is None:
            raise InvalidArgument("dataset contains a non-finite value")
        self.values = f
        self.truth = None

    def size(self) -> int:
        return self.values.shape[0]

    def dim(self) -> int:
        return self.values.shape[1]

    def empty(self) -> bool:
        return self.values.size == 0

    def row(self, i: int) -> np.ndarray:
        return self.values[i]


@dataclass
class SngParams:  # clusterer.hpp:11-24
    eps: float = 0.0
    min_pts: int = 1
    rate: float = 1.0
    seed: int = 0
    dist: Distance = field(default_factory=Distance.euclidean)
    threads: int = 0  # CPU worker count in the reference; ignored by the GPU path
    device: int = -1  # extension: CUDA ordinal (-1 = current)
    # extension: GPUs of this process to shard the rows over (0/1: one GPU, N, -1: all),
    # optionally their ordinals (a repeated ordinal runs several shards on one GPU)
    num_gpus: int = 0
    devices: list | None = None

    def validate(self) -> None:
        if not (self.eps > 0.0):
            raise InvalidArgument("eps must be > 0")
        if self.min_pts < 1:
            raise InvalidArgument("min_pts must be >= 1")
        if not (self.rate > 0.0) or self.rate > 1.0:
            raise InvalidArgument("rate must lie in (0, 1]")


@dataclass
class ClusterRunInfo:  # clusterer.hpp:27-31 (+ GPU counters in .gpu)
    distance_evals: int = 0
    edges: int = 0
    graph_bytes: int = 0
    gpu: dict = field(default_factory=dict)


@dataclass
class BuildStats:  # graph.hpp:56-58
    distance_evals: int = 0


@dataclass
class Clustering:  # dataset.hpp:78-91
    assignment: np.ndarray
    role: np.ndarray
    cluster_count: int = 0

    def size(self) -> int:
        return len(self.assignment)

    def count_role(self, r: PointRole) -> int:
        return int(np.count_nonzero(self.role == int(r)))


class SampledGraph:
    """Canonical edge set of the sampled graph (graph.hpp:17-54), CSR on demand."""

    def __init__(self, n: int, keys: np.ndarray):
        self.n = n
        self.keys = np.asarray(keys, np.uint64)  # sorted unique u<<32|v, u < v
        self._deg = None

    def vertex_count(self) -> int:
        return self.n

    def edge_count(self) -> int:
        return int(self.keys.size)

    def edges(self) -> list[tuple[int, int]]:
        return [(int(k >> np.uint64(32)), int(k & np.uint64(0xFFFFFFFF))) for k in self.keys]

    def edge_array(self) -> np.ndarray:
        u = (self.keys >> np.uint64(32)).astype(np.int64)
        v = (self.keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
        return np.stack([u, v], axis=1)

    def degree(self, v: int | None = None):
        if self._deg is None:
            e = self.edge_array()
            self._deg = np.bincount(e.reshape(-1), minlength=self.n).astype(np.int64)
        return self._deg if v is None else int(self._deg[v])

    def storage_bytes(self) -> int:  # graph.hpp:41-43
        return (self.n + 1) * 8 + 2 * self.edge_count() * 4


def _opts(device: int = -1, timing: bool = False, stream: int = 0, row_begin: int = 0,
          row_end: int = 0, dist: "Distance | None" = None, num_gpus: int = 0,
          devices=None) -> SngbOpts:
    flags = (SNGB_FLAG_TIMING if timing else 0) | (dist.flags if dist is not None else 0)
    o = SngbOpts(device, flags, C.c_void_p(stream or None), row_begin, row_end, int(num_gpus),
                 None)
    if devices is not None:
        devs = list(devices)
        if num_gpus in (0, 1) and len(devs) > 1:
            o.num_gpus = len(devs)
        arr = (C.c_int32 * max(len(devs), 1))(*devs)
        o.devices = C.cast(arr, C.POINTER(C.c_int32))
        o._keep = arr  # the array must outlive the call
    return o


def sng_dbscan(data: Dataset, params: SngParams, info: ClusterRunInfo | None = None,
               timing: bool = False) -> Clustering:
    """sng::sng_dbscan (clusterer.hpp:42, clusterer.cpp:54-65) on the GPU."""
    if not isinstance(data, Dataset):
        data = Dataset(data)
    params.validate()
    if not isinstance(params.dist, Distance):
        raise NotImplementedError("a Python distance callback cannot run on the GPU path")
    pts = data.values
    n, d = pts.shape
    labels = np.empty(n, np.int32)
    roles = np.empty(n, np.uint8)
    gi = SngbInfo()
    o = _opts(params.device, timing, dist=params.dist, num_gpus=params.num_gpus,
              devices=params.devices)
    if data.values64 is not None:
        fn, arg = _lib.lib().sngb_dbscan_f64, data.values64.ctypes.data_as(C.POINTER(C.c_double))
    else:
        fn, arg = _lib.lib().sngb_dbscan_f32, pts.ctypes.data_as(C.POINTER(C.c_float))
    rc = fn(arg, n, d, float(params.eps), int(params.min_pts), float(params.rate),
            int(params.seed) & 0xFFFFFFFFFFFFFFFF, C.byref(o),
            labels.ctypes.data_as(C.POINTER(C.c_int32)),
            roles.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(gi))
    _check(rc)
    if info is not None:
        info.distance_evals = gi.distance_evals
        info.edges = gi.edges
        info.graph_bytes = gi.graph_bytes
        info.gpu = gi.as_dict()
    return Clustering(labels, roles, int(gi.cluster_count))


def dbscan_exact(data: Dataset, eps: float, min_pts: int, dist: Distance | None = None,
                 threads: int = 0, info: ClusterRunInfo | None = None, device: int = -1,
                 num_gpus: int = 0, devices=None, timing: bool = False) -> Clustering:
    """sng::dbscan_exact (clusterer.hpp:46-48, clusterer.cpp:67-79) on the GPU:
    classical DBSCAN on the exact eps-graph (build_full_graph, graph.cpp:191-220),
    distance_evals = n(n-1)/2."""
    if not isinstance(data, Dataset):
        data = Dataset(data)
    if not (eps > 0.0):
        raise InvalidArgument("eps must be > 0")
    if min_pts < 1:
        raise InvalidArgument("min_pts must be >= 1")
    dist = dist or Distance.euclidean()
    if not isinstance(dist, Distance):
        raise NotImplementedError("a Python distance callback cannot run on the GPU path")
    n, d = data.values.shape
    labels = np.empty(n, np.int32)
    roles = np.empty(n, np.uint8)
    gi = SngbInfo()
    o = _opts(device, timing, dist=dist, num_gpus=num_gpus, devices=devices)
    L = _lib.lib()
    if data.values64 is not None:
        fn, arg = L.sngb_dbscan_exact_f64, data.values64.ctypes.data_as(C.POINTER(C.c_double))
    else:
        fn, arg = L.sngb_dbscan_exact_f32, data.values.ctypes.data_as(C.POINTER(C.c_float))
    _check(fn(arg, n, d, float(eps), int(min_pts), C.byref(o),
              labels.ctypes.data_as(C.POINTER(C.c_int32)),
              roles.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(gi)))
    if info is not None:
        info.distance_evals = gi.distance_evals
        info.edges = gi.edges
        info.graph_bytes = gi.graph_bytes
        info.gpu = gi.as_dict()
    return Clustering(labels, roles, int(gi.cluster_count))


def build_full_graph(data: Dataset, eps: float, dist: Distance | None = None, threads: int = 0,
                     stats: BuildStats | None = None, device: int = -1) -> SampledGraph:
    """sng::build_full_graph (graph.hpp:69-70, graph.cpp:191-220) on the GPU."""
    if not isinstance(data, Dataset):
        data = Dataset(data)
    if dist is not None and not isinstance(dist, Distance):
        raise NotImplementedError("a Python distance callback cannot run on the GPU path")
    if data.values64 is not None:  # fp64 values: the exact graph is rate-1 sampling
        g = build_sampled_graph(data, eps, 1.0, dist, 0, threads, None, device)
        if stats is not None:
            stats.distance_evals = g.n * (g.n - 1) // 2
        return g
    pts = data.values
    n, d = pts.shape
    L = _lib.lib()
    gi = SngbInfo()
    o = _opts(device, dist=dist)
    cnt = C.c_uint64(0)
    cap = 1 << 20
    while True:
        keys = np.empty(cap, np.uint64)
        rc = L.sngb_full_edges_f32(pts.ctypes.data_as(C.POINTER(C.c_float)), n, d, float(eps),
                                   C.byref(o), keys.ctypes.data_as(C.POINTER(C.c_uint64)), cap,
                                   C.byref(cnt), C.byref(gi))
        if rc == _lib.SNGB_ERR_CAPACITY:
            cap = int(cnt.value)
            continue
        _check(rc)
        break
    if stats is not None:
        stats.distance_evals = gi.distance_evals
    return SampledGraph(n, keys[: cnt.value].copy())


def build_sampled_graph(data: Dataset, eps: float, rate: float, dist: Distance | None = None,
                        seed: int = 0, threads: int = 0, stats: BuildStats | None = None,
                        device: int = -1) -> SampledGraph:
    """sng::build_sampled_graph (graph.hpp:65-66, graph.cpp:133-189) on the GPU."""
    if not isinstance(data, Dataset):
        data = Dataset(data)
    if dist is not None and not isinstance(dist, Distance):
        raise NotImplementedError("a Python distance callback cannot run on the GPU path")
    pts = data.values
    n, d = pts.shape
    L = _lib.lib()
    gi = SngbInfo()
    o = _opts(device, dist=dist)
    cnt = C.c_uint64(0)
    if data.values64 is not None:
        fn, arg = L.sngb_sampled_edges_f64, data.values64.ctypes.data_as(C.POINTER(C.c_double))
    else:
        fn, arg = L.sngb_sampled_edges_f32, pts.ctypes.data_as(C.POINTER(C.c_float))
    cap = 1 << 20
    while True:
        keys = np.empty(cap, np.uint64)
        rc = fn(arg, n, d, float(eps), float(rate), int(seed) & 0xFFFFFFFFFFFFFFFF, C.byref(o),
                keys.ctypes.data_as(C.POINTER(C.c_uint64)), cap, C.byref(cnt), C.byref(gi))
        if rc == _lib.SNGB_ERR_CAPACITY:
            cap = int(cnt.value)
            continue
        _check(rc)
        break
    if stats is not None:
        stats.distance_evals = gi.distance_evals
    return SampledGraph(n, keys[: cnt.value].copy())


def cluster_graph(g: SampledGraph, min_pts: int, device: int = -1) -> Clustering:
    """sng::cluster_graph (clusterer.hpp:38, clusterer.cpp:7-52) on the GPU."""
    if min_pts < 1:
        raise InvalidArgument("min_pts must be >= 1")
    import torch

    dev = torch.device("cuda", device if device >= 0 else torch.cuda.current_device())
    keys = torch.from_numpy(g.keys.view(np.int64)).to(dev)
    labels, roles, gi = cluster_edges_device(keys, g.n, min_pts)
    return Clustering(labels.cpu().numpy(), roles.cpu().numpy(), int(gi.cluster_count))


# ---------------------------------------------------------------------------
# Device-tensor entry points (torch is plumbing only: memory + streams).
# ---------------------------------------------------------------------------
def _check_points(points) -> None:
    import torch

    if points.dtype != torch.float32 or not points.is_cuda or points.dim() != 2:
        raise InvalidArgument("points must be a CUDA float32 [n, d] tensor")


def _check_keys(keys) -> None:
    import torch

    if keys.dtype != torch.int64 or not keys.is_cuda or keys.dim() != 1:
        raise InvalidArgument("keys must be a CUDA int64 1-D tensor (u<<32|v)")


def _check_vertex_array(t, name: str) -> None:
    import torch

    if t.dtype != torch.int32 or not t.is_cuda or t.dim() != 1:
        raise InvalidArgument(f"{name} must be a CUDA int32 1-D tensor")


def _stream_handle(t) -> int:
    import torch

    return torch.cuda.current_stream(t.device).cuda_stream


def sng_dbscan_device(points, eps: float, min_pts: int, rate: float, seed: int,
                      labels=None, roles=None, timing: bool = False, num_gpus: int = 0,
                      devices=None):
    """sng_dbscan over a CUDA float32 [n, d] tensor on torch's current stream
    (num_gpus / devices: shard the rows over several GPUs of this process; the
    points and the outputs stay on points.device, which must be devices[0]).

    Returns (labels int32[n], roles uint8[n], SngbInfo) as CUDA tensors."""
    import torch

    _check_points(points)
    points = points.contiguous()
    n, d = points.shape
    if labels is None:
        labels = torch.empty(n, dtype=torch.int32, device=points.device)
    if roles is None:
        roles = torch.empty(n, dtype=torch.uint8, device=points.device)
    gi = SngbInfo()
    o = _opts(points.device.index, timing, _stream_handle(points), num_gpus=num_gpus,
              devices=devices)
    rc = _lib.lib().sngb_dbscan_f32_device(points.data_ptr(), n, d, float(eps), int(min_pts),
                                           float(rate), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                           C.byref(o), labels.data_ptr(), roles.data_ptr(),
                                           C.byref(gi))
    _check(rc)
    return labels, roles, gi


def dbscan_exact_device(points, eps: float, min_pts: int, timing: bool = False,
                        num_gpus: int = 0, devices=None):
    """dbscan_exact over a CUDA float32 [n, d] tensor: (labels, roles, SngbInfo)."""
    import torch

    _check_points(points)
    points = points.contiguous()
    n, d = points.shape
    labels = torch.empty(n, dtype=torch.int32, device=points.device)
    roles = torch.empty(n, dtype=torch.uint8, device=points.device)
    gi = SngbInfo()
    o = _opts(points.device.index, timing, _stream_handle(points), num_gpus=num_gpus,
              devices=devices)
    _check(_lib.lib().sngb_dbscan_exact_f32_device(points.data_ptr(), n, d, float(eps),
                                                   int(min_pts), C.byref(o), labels.data_ptr(),
                                                   roles.data_ptr(), C.byref(gi)))
    return labels, roles, gi


def sampled_edges_device(points, eps: float, rate: float, seed: int, row_begin: int = 0,
                         row_end: int = 0, timing: bool = False):
    """Canonical edge keys (int64 view of u<<32|v) sampled by rows [row_begin, row_end)."""
    import torch

    _check_points(points)
    points = points.contiguous()
    n, d = points.shape
    L = _lib.lib()
    gi = SngbInfo()
    o = _opts(points.device.index, timing, _stream_handle(points), row_begin, row_end)
    cnt = C.c_uint64(0)
    rows = (row_end or n) - row_begin
    draws = min(int(np.ceil(rate * float(n))), n - 1)
    cap = int(min(max(rows * draws // 64, 1 << 20), 1 << 27))
    while True:
        keys = torch.empty(cap, dtype=torch.int64, device=points.device)
        rc = L.sngb_sampled_edges_f32_device(points.data_ptr(), n, d, float(eps), float(rate),
                                             int(seed) & 0xFFFFFFFFFFFFFFFF, C.byref(o),
                                             keys.data_ptr(), cap, C.byref(cnt), C.byref(gi))
        if rc == _lib.SNGB_ERR_CAPACITY:
            cap = int(cnt.value)
            continue
        _check(rc)
        break
    return keys[: cnt.value], gi


def cluster_edges_device(keys, n: int, min_pts: int, timing: bool = False):
    """cluster_graph over CUDA int64 keys (u<<32|v, any order, duplicates allowed)."""
    import torch

    _check_keys(keys)
    keys = keys.contiguous()
    labels = torch.empty(n, dtype=torch.int32, device=keys.device)
    roles = torch.empty(n, dtype=torch.uint8, device=keys.device)
    gi = SngbInfo()
    o = _opts(keys.device.index, timing, _stream_handle(keys))
    rc = _lib.lib().sngb_cluster_edges_device(keys.data_ptr() if keys.numel() else None,
                                              keys.numel(), n, int(min_pts), C.byref(o),
                                              labels.data_ptr(), roles.data_ptr(), C.byref(gi))
    _check(rc)
    return labels, roles, gi


# ---- multi-GPU merge steps (include/sngb.h; used by distributed.py) --------
def _ptr(t):
    return t.data_ptr() if t.numel() else None


def unique_keys_device(keys, n: int):
    """Sorted unique canonical keys (graph.cpp:34-40) of CUDA int64 keys."""
    import torch

    _check_keys(keys)
    keys = keys.contiguous()
    out = torch.empty(max(keys.numel(), 1), dtype=torch.int64, device=keys.device)
    cnt = C.c_uint64(0)
    o = _opts(keys.device.index, False, _stream_handle(keys))
    _check(_lib.lib().sngb_unique_keys_device(_ptr(keys), keys.numel(), n, C.byref(o),
                                              out.data_ptr(), C.byref(cnt)))
    return out[: cnt.value]


def degrees_device(keys, n: int, degree=None):
    """degree[v] += keys incident to v (int32[n], created zeroed when None)."""
    import torch

    _check_keys(keys)
    keys = keys.contiguous()
    if degree is None:
        degree = torch.zeros(n, dtype=torch.int32, device=keys.device)
    _check_vertex_array(degree, "degree")
    o = _opts(keys.device.index, False, _stream_handle(keys))
    _check(_lib.lib().sngb_degrees_device(_ptr(keys), keys.numel(), n, C.byref(o),
                                          degree.data_ptr()))
    return degree


def components_device(keys, n: int, degree, min_pts: int, parent) -> int:
    """Union-find step over core-core keys into `parent` (in place); returns
    the number of vertices whose entry changed."""
    _check_keys(keys)
    _check_vertex_array(degree, "degree")
    _check_vertex_array(parent, "parent")
    keys = keys.contiguous()
    changed = C.c_uint64(0)
    o = _opts(keys.device.index, False, _stream_handle(parent))
    _check(_lib.lib().sngb_components_device(_ptr(keys), keys.numel(), n, degree.data_ptr(),
                                             int(min_pts), C.byref(o), parent.data_ptr(),
                                             C.byref(changed)))
    return int(changed.value)


def border_device(keys, n: int, degree, min_pts: int, parent, border) -> None:
    """border[b] = min(border[b], parent[a]) for core a -- non-core b edges."""
    _check_keys(keys)
    for t, nm in ((degree, "degree"), (parent, "parent"), (border, "border")):
        _check_vertex_array(t, nm)
    keys = keys.contiguous()
    o = _opts(parent.device.index, False, _stream_handle(parent))
    _check(_lib.lib().sngb_border_device(_ptr(keys), keys.numel(), n, degree.data_ptr(),
                                         int(min_pts), parent.data_ptr(), C.byref(o),
                                         border.data_ptr()))


def relabel_device(n: int, degree, min_pts: int, parent, border):
    """(labels int32[n], roles uint8[n], SngbInfo) from the merged arrays."""
    import torch

    for t, nm in ((degree, "degree"), (parent, "parent"), (border, "border")):
        _check_vertex_array(t, nm)
    labels = torch.empty(n, dtype=torch.int32, device=parent.device)
    roles = torch.empty(n, dtype=torch.uint8, device=parent.device)
    gi = SngbInfo()
    o = _opts(parent.device.index, False, _stream_handle(parent))
    _check(_lib.lib().sngb_relabel_device(n, degree.data_ptr(), int(min_pts), parent.data_ptr(),
                                          border.data_ptr(), C.byref(o), labels.data_ptr(),
                                          roles.data_ptr(), C.byref(gi)))
    return labels, roles, gi


def sng_dbscan_batch(problems, device: int = -1):
    """Many small sng_dbscan calls at once (sngb_dbscan_batch_f32): `problems`
    is a sequence of (Dataset or array, SngParams); returns one Clustering per
    problem, identical to separate calls.  fp64 data that fp32 cannot hold is
    run one problem at a time through the fp64 entry point."""
    items = [(d if isinstance(d, Dataset) else Dataset(d), p) for d, p in problems]
    out = [None] * len(items)
    batch = []
    for i, (ds, p) in enumerate(items):
        p.validate()
        if ds.values64 is not None or not isinstance(p.dist, Distance):
            out[i] = sng_dbscan(ds, p)
        else:
            batch.append(i)
    arr = (_lib.SngbProblem * max(len(batch), 1))()
    keep = []
    for k, i in enumerate(batch):
        ds, p = items[i]
        n, d = ds.values.shape
        labels, roles, info = np.empty(n, np.int32), np.empty(n, np.uint8), SngbInfo()
        keep.append((labels, roles, info))
        arr[k] = _lib.SngbProblem(ds.values.ctypes.data, n, d, p.dist.flags, float(p.eps),
                                  float(p.rate), int(p.seed) & 0xFFFFFFFFFFFFFFFF,
                                  int(p.min_pts), 0, labels.ctypes.data, roles.ctypes.data,
                                  C.addressof(info))
    if batch:
        o = _opts(device)
        _lib.lib().sngb_dbscan_batch_f32(arr, len(batch), C.byref(o))
        for k, i in enumerate(batch):
            _check(arr[k].status)
            labels, roles, info = keep[k]
            out[i] = Clustering(labels, roles, int(info.cluster_count))
    return out
