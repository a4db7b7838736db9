"""Multi-GPU through the C ABI (ABI 4: sngb_opts.num_gpus / devices;
paper_2006_06743_b200/csrc/sngb_multi.cu) -- the reference's entry point
sng::sng_dbscan (clusterer.hpp:42) with its row split (graph.cpp:45-63) over
several GPUs of one process: per-shard uploads, NVLink peer copies of the
replica, owner routing of the keys, peer-memory SUM / MIN all-reduces to a
fixed point.

This run has one GPU, so the W shards are placed on it with a repeated ordinal
(devices = [0] * W): the same code path -- per-shard contexts and streams,
cross-stream event fences, peer copies and the peer-reading reduce kernel --
with every "peer" on one device.  Results must be the reference's (golden
fixtures) and the single-GPU call's, bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402
from tests import _golden  # noqa: E402

G = _golden.load()
CASES = [c for c in G["cases"] if c["n"] >= 12]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if sng.device_count() < 1:
        pytest.fail("no CUDA device: the GPU path has no CPU fallback")


def _golden_check(c, cl, info):
    assert info.distance_evals == c["distance_evals"]
    assert info.edges == c["edges"]
    assert cl.cluster_count == c["cluster_count"]
    assert _golden.sha(cl.assignment) == c["labels_sha256"], c["name"]
    assert _golden.sha(cl.role) == c["roles_sha256"], c["name"]


@pytest.mark.parametrize("w", [2, 3, 8])
@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_multi_host_entry_equals_reference(c, w):
    pts = _golden.points(c["recipe"])
    info = sng.ClusterRunInfo()
    p = sng.SngParams(eps=c["eps"], min_pts=c["min_pts"], rate=c["rate"], seed=c["seed"],
                      devices=[0] * w)
    cl = sng.sng_dbscan(sng.Dataset(pts), p, info)
    assert info.gpu["num_gpus"] == w
    _golden_check(c, cl, info)


@pytest.mark.parametrize("w", [2, 4])
def test_multi_device_entry_equals_single(w):
    import torch
    wl = synthetic.CONFIGS[4]
    pts = synthetic.generate(4, n=60000)
    rate = 2500 / 60000
    x = torch.from_numpy(pts).cuda()
    l1, r1, g1 = sng.sng_dbscan_device(x, wl.eps, wl.min_pts, rate, wl.seed)
    lw, rw, gw = sng.sng_dbscan_device(x, wl.eps, wl.min_pts, rate, wl.seed, devices=[0] * w)
    torch.cuda.synchronize()
    assert torch.equal(l1, lw) and torch.equal(r1, rw)
    assert (gw.edges, gw.distance_evals, gw.cluster_count) == (g1.edges, g1.distance_evals,
                                                               g1.cluster_count)
    assert gw.num_gpus == w and gw.merge_rounds >= 1
    assert gw.routed_keys > 0


@pytest.mark.parametrize("cfg,n", [(2, 5000), (3, 40000), (5, 40000)])
def test_multi_filters_equal_single(cfg, n):
    """Each shard runs the same filters (8-bit rows, head filter) as one GPU."""
    w = synthetic.CONFIGS[cfg]
    pts = synthetic.generate(cfg, n=n)
    rate = min(1.0, w.draws / n)
    p1 = sng.SngParams(eps=w.eps, min_pts=w.min_pts, rate=rate, seed=w.seed)
    pw = sng.SngParams(eps=w.eps, min_pts=w.min_pts, rate=rate, seed=w.seed, devices=[0, 0, 0])
    i1, iw = sng.ClusterRunInfo(), sng.ClusterRunInfo()
    c1 = sng.sng_dbscan(sng.Dataset(pts), p1, i1)
    cw = sng.sng_dbscan(sng.Dataset(pts), pw, iw)
    np.testing.assert_array_equal(c1.assignment, cw.assignment)
    np.testing.assert_array_equal(c1.role, cw.role)
    assert i1.edges == iw.edges and i1.distance_evals == iw.distance_evals
    assert iw.gpu["filter_bits"] == i1.gpu["filter_bits"]
    assert iw.gpu["pairs_evaluated"] == i1.gpu["pairs_evaluated"]


def test_multi_exact_and_fp64():
    c = next(c for c in G["exact_cases"] if c["name"] == "exact_cfg1_n6000")
    pts = _golden.points(c["recipe"])
    info = sng.ClusterRunInfo()
    cl = sng.dbscan_exact(sng.Dataset(pts), c["eps"], c["min_pts"], info=info, devices=[0, 0, 0])
    assert info.distance_evals == c["distance_evals"] and info.edges == c["edges"]
    assert _golden.sha(cl.assignment) == c["labels_sha256"]
    assert _golden.sha(cl.role) == c["roles_sha256"]
    rng = np.random.default_rng(7)
    p64 = rng.random((3000, 4))  # fp64 values fp32 cannot hold
    prm = dict(eps=0.1, min_pts=4, rate=0.2, seed=3)
    c1 = sng.sng_dbscan(sng.Dataset(p64), sng.SngParams(**prm))
    cw = sng.sng_dbscan(sng.Dataset(p64), sng.SngParams(**prm, devices=[0, 0]))
    np.testing.assert_array_equal(c1.assignment, cw.assignment)
    np.testing.assert_array_equal(c1.role, cw.role)


def test_multi_more_shards_than_rows_and_errors():
    pts = np.arange(5, dtype=np.float32).reshape(-1, 1)
    p = sng.SngParams(eps=1.5, min_pts=1, rate=1.0, devices=[0] * 8)
    c8 = sng.sng_dbscan(sng.Dataset(pts), p)
    c1 = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=1.5, min_pts=1, rate=1.0))
    np.testing.assert_array_equal(c8.assignment, c1.assignment)
    bad = np.zeros((4, 2), np.float32)
    bad[2, 1] = np.nan
    import ctypes as C
    from paper_2006_06743_b200 import _lib
    o = sng._opts(0, devices=[0, 0])
    lab, rol = np.empty(4, np.int32), np.empty(4, np.uint8)
    rc = _lib.lib().sngb_dbscan_f32(bad.ctypes.data_as(C.POINTER(C.c_float)), 4, 2, 1.0, 1, 1.0, 0,
                                    C.byref(o), lab.ctypes.data_as(C.POINTER(C.c_int32)),
                                    rol.ctypes.data_as(C.POINTER(C.c_uint8)), None)
    assert rc == _lib.SNGB_ERR_NONFINITE
    with pytest.raises(sng.InvalidArgument):  # an ordinal that does not exist
        sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=1.5, min_pts=1, rate=1.0,
                                                       devices=[0, 99]))
    # -1: every visible GPU (here one: the single-GPU path)
    c_all = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=1.5, min_pts=1, rate=1.0,
                                                           num_gpus=-1))
    np.testing.assert_array_equal(c_all.assignment, c1.assignment)
