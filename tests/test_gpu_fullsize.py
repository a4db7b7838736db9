"""Parity at BASELINE.json's full sizes.

cfg1-cfg3: the whole pipeline against the oracle run at full size.
cfg4-cfg5 (oracle too slow for a test): size-independent properties --
  * the clustering stage is exact: the oracle's cluster_graph restatement run
    on the GPU's own edge list reproduces the GPU labels/roles bit for bit;
  * the edge set is exact on a random sample of vertices: every sampled
    vertex's Floyd partners (oracle restatement of graph.cpp:161-174) that pass
    the fp64 eps-test are edges, and every GPU edge at a sampled vertex is
    justified by one of the two endpoints' partner sets;
  * determinism (two runs identical) and distance_evals == n * draws.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if sng.device_count() < 1:
        pytest.fail("no CUDA device: the GPU path has no CPU fallback")


def _gpu(pts, w):
    import torch
    x = torch.from_numpy(pts).cuda()
    labels, roles, gi = sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed)
    keys, _ = sng.sampled_edges_device(x, w.eps, w.rate, w.seed)
    torch.cuda.synchronize()
    return labels.cpu().numpy(), roles.cpu().numpy(), gi, keys.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_full_size_equals_oracle(oracle, cfg):
    w = synthetic.CONFIGS[cfg]
    pts = synthetic.generate(cfg)
    labels, roles, gi, keys = _gpu(pts, w)
    ol, orl, oinfo, okeys = oracle.sng_dbscan(pts, w.eps, w.min_pts, w.rate, w.seed)
    assert gi.distance_evals == oinfo["distance_evals"] == w.pairs
    assert gi.edges == oinfo["edges"]
    np.testing.assert_array_equal(keys, okeys)
    np.testing.assert_array_equal(roles, orl)
    np.testing.assert_array_equal(labels, ol)
    assert gi.cluster_count == oinfo["cluster_count"]


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_properties(oracle, cfg):
    w = synthetic.CONFIGS[cfg]
    pts = synthetic.generate(cfg)
    n = pts.shape[0]
    labels, roles, gi, keys = _gpu(pts, w)
    assert gi.distance_evals == w.pairs
    # canonical, sorted, unique, in range, no self loops
    u = (keys >> np.uint64(32)).astype(np.int64)
    v = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    assert len(keys) == gi.edges
    assert np.all(np.diff(keys.astype(np.uint64)) > 0) if len(keys) > 1 else True
    assert np.all(u < v) and np.all(v < n)
    # clustering stage exact on the GPU's own edges
    cl, cr, ccount = oracle.cluster_edges(keys, n, w.min_pts)
    np.testing.assert_array_equal(cr, roles)
    np.testing.assert_array_equal(cl, labels)
    assert ccount == gi.cluster_count
    # edge set exact on sampled vertices
    rng = np.random.default_rng(cfg)
    sample = rng.choice(n, size=64, replace=False)
    eps2 = w.eps * w.eps
    edge_set = set(keys.tolist())
    partners = {}
    for s in sample:
        p = oracle.partners(n, w.draws, w.seed, int(s))
        partners[int(s)] = set(p.tolist())
        diff = pts[p].astype(np.float64) - pts[s].astype(np.float64)
        d2 = np.zeros(len(p))
        for k in range(pts.shape[1]):  # sequential in k, like distance.hpp:78-81
            d2 = d2 + diff[:, k] * diff[:, k]
        for vv, ok in zip(p.tolist(), (d2 <= eps2).tolist()):
            key = (min(s, vv) << 32) | max(s, vv)
            assert (key in edge_set) == ok, (s, vv, ok)  # within() is symmetric
    # every GPU edge at a sampled vertex is justified by a partner set
    for s in sample[:16]:
        s = int(s)
        inc = np.concatenate([v[u == s], u[v == s]])
        for x in inc.tolist():
            if x in partners[s]:
                continue
            assert s in set(oracle.partners(n, w.draws, w.seed, x).tolist()), (s, x)
    # determinism
    labels2, roles2, gi2, keys2 = _gpu(pts, w)
    np.testing.assert_array_equal(keys2, keys)
    np.testing.assert_array_equal(labels2, labels)



def test_cfg5_head_filter_equals_fp32_filter(monkeypatch):
    """cfg5 at full size: the auto path (head filter, 16) and the plain fp32
    gather (SNGB_HEAD=0) give the same edge list, bit for bit."""
    import torch
    w = synthetic.CONFIGS[5]
    x = torch.from_numpy(synthetic.generate(5)).cuda()
    k_auto, gi = sng.sampled_edges_device(x, w.eps, w.rate, w.seed)
    torch.cuda.synchronize()
    assert gi.filter_bits == 16
    monkeypatch.setenv("SNGB_HEAD", "0")
    k_fp32, gi0 = sng.sampled_edges_device(x, w.eps, w.rate, w.seed)
    torch.cuda.synchronize()
    assert gi0.filter_bits == 32
    assert torch.equal(k_auto, k_fp32)
