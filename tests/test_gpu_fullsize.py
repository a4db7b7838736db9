"""Parity at BASELINE.json's FULL sizes, all five configs, both entry points.

tests/golden/golden_full.json holds the REFERENCE's own results on the five
synthetic workloads at full size (tests/golden/make_golden_full.py: the
reference's graph.cpp + clusterer.cpp compiled unmodified, one
build_sampled_graph + cluster_graph per config = sng_dbscan,
clusterer.cpp:54-65): SHA-256 digests of the points, the canonical edge keys,
labels and roles, and the ClusterRunInfo counters.  Here the GPU path must
reproduce them bit for bit through

  * the device entry point   (sngb_dbscan_f32_device, points resident in HBM),
  * the host-buffer entry    (sngb_dbscan_f32: chunked upload, the host-upload
                              filter plans and schedules -- what bench.py's
                              e2e times and sng::sng_dbscan / the Python
                              mirror call),
  * the edge builder         (sngb_sampled_edges_f32_device = SampledGraph::edges()).

On a mismatch the 64 per-block digests say where the labels first differ.
"""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_full.json")


def _golden(cfg):
    with open(GOLDEN) as f:
        g = json.load(f)["configs"]
    if str(cfg) not in g:
        pytest.fail(f"golden_full.json has no cfg{cfg}: run tests/golden/make_golden_full.py")
    return g[str(cfg)]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _first_bad_block(a, blocks):
    n = len(a)
    cuts = [(n * i) // len(blocks) for i in range(len(blocks) + 1)]
    for i, want in enumerate(blocks):
        if sha(a[cuts[i]:cuts[i + 1]])[:16] != want:
            return i, cuts[i], cuts[i + 1]
    return None


def _check(g, labels, roles, info, where):
    assert int(info.distance_evals) == g["distance_evals"], where
    assert int(info.edges) == g["edges"], where
    assert int(info.graph_bytes) == g["graph_bytes"], where
    assert int(info.cluster_count) == g["cluster_count"], where
    assert (int(info.core_count), int(info.border_count), int(info.noise_count)) == \
        (g["core"], g["border"], g["noise"]), where
    if sha(roles) != g["roles_sha256"]:
        pytest.fail(f"{where}: roles differ, first bad block {_first_bad_block(roles, g['roles_blocks'])}")
    if sha(labels) != g["labels_sha256"]:
        pytest.fail(f"{where}: labels differ, first bad block "
                    f"{_first_bad_block(labels, g['labels_blocks'])}")


_PTS = {}


def _points(cfg):
    if cfg not in _PTS:
        _PTS.clear()  # one full-size dataset in host memory at a time
        _PTS[cfg] = synthetic.generate(cfg)
    return _PTS[cfg]


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_generator_matches_golden_points(cfg):
    g = _golden(cfg)
    assert sha(_points(cfg)) == g["points_sha256"]


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_full_size_device_entry_equals_reference(cfg):
    import torch
    g = _golden(cfg)
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(_points(cfg)).cuda()
    labels, roles, gi = sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed)
    torch.cuda.synchronize()
    _check(g, labels.cpu().numpy(), roles.cpu().numpy(), gi, f"cfg{cfg} device entry")
    keys, ki = sng.sampled_edges_device(x, w.eps, w.rate, w.seed)
    torch.cuda.synchronize()
    assert int(ki.edges) == g["edges"]
    assert sha(keys.cpu().numpy().view(np.uint64)) == g["keys_sha256"], f"cfg{cfg} edge keys"
    del x, labels, roles, keys
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_full_size_host_entry_equals_reference(cfg):
    """The public host-buffer call (sngb_dbscan_f32 via the Python mirror), from
    pageable numpy memory -- the chunked upload and its overlapped schedules."""
    g = _golden(cfg)
    w = synthetic.CONFIGS[cfg]
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(sng.Dataset(_points(cfg)),
                       sng.SngParams(eps=w.eps, min_pts=w.min_pts, rate=w.rate, seed=w.seed), info)

    class _I:  # the fields _check reads
        pass
    gi = _I()
    for k in ("distance_evals", "edges", "graph_bytes"):
        setattr(gi, k, getattr(info, k))
    gi.cluster_count = c.cluster_count
    gi.core_count, gi.border_count, gi.noise_count = (c.count_role(sng.PointRole.Core),
                                                      c.count_role(sng.PointRole.Border),
                                                      c.count_role(sng.PointRole.Noise))
    _check(g, c.assignment, c.role, gi, f"cfg{cfg} host entry")


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_pinned_host_entry_equals_reference(cfg):
    """Same through the raw C ABI from pinned memory (bench.py's e2e leg)."""
    import ctypes as C

    import torch
    from paper_2006_06743_b200 import _lib
    g = _golden(cfg)
    w = synthetic.CONFIGS[cfg]
    host = torch.from_numpy(_points(cfg)).pin_memory()
    n, d = host.shape
    labels = torch.empty(n, dtype=torch.int32).pin_memory()
    roles = torch.empty(n, dtype=torch.uint8).pin_memory()
    gi = _lib.SngbInfo()
    rc = _lib.lib().sngb_dbscan_f32(C.cast(host.data_ptr(), C.POINTER(C.c_float)), n, d, w.eps,
                                    w.min_pts, w.rate, w.seed, None,
                                    C.cast(labels.data_ptr(), C.POINTER(C.c_int32)),
                                    C.cast(roles.data_ptr(), C.POINTER(C.c_uint8)), C.byref(gi))
    sng._check(rc)
    _check(g, labels.numpy(), roles.numpy(), gi, f"cfg{cfg} pinned host entry")


def test_cfg5_head_filter_equals_fp32_filter(monkeypatch):
    """cfg5 at full size: the auto path (head filter, 16) and the plain fp32
    gather (SNGB_HEAD=0) give the same edge list, bit for bit -- and both the
    reference's."""
    import torch
    g = _golden(5)
    w = synthetic.CONFIGS[5]
    x = torch.from_numpy(_points(5)).cuda()
    k_auto, gi = sng.sampled_edges_device(x, w.eps, w.rate, w.seed)
    torch.cuda.synchronize()
    assert gi.filter_bits == 16
    monkeypatch.setenv("SNGB_HEAD", "0")
    k_fp32, gi0 = sng.sampled_edges_device(x, w.eps, w.rate, w.seed)
    torch.cuda.synchronize()
    assert gi0.filter_bits == 32
    assert torch.equal(k_auto, k_fp32)
    assert sha(k_fp32.cpu().numpy().view(np.uint64)) == g["keys_sha256"]
