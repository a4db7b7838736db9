"""sng::dbscan_exact / build_full_graph on the GPU (clusterer.cpp:67-79,
graph.cpp:191-220) against the reference's own results (tests/golden/golden.json
"exact_cases", made by make_golden.py from the compiled reference): labels,
roles, the canonical edge list and distance_evals = n(n-1)/2, through the host,
device and fp64 entry points, Euclidean / Manhattan / cosine."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2006_06743_b200 as sng  # noqa: E402
from tests import _golden  # noqa: E402

CASES = _golden.load()["exact_cases"]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if sng.device_count() < 1:
        pytest.fail("no CUDA device: the GPU path has no CPU fallback")


def _check(c, labels, roles, evals, edges, clusters):
    assert evals == c["distance_evals"] == c["n"] * (c["n"] - 1) // 2
    assert edges == c["edges"]
    assert clusters == c["cluster_count"]
    assert _golden.sha(np.asarray(labels, np.int32)) == c["labels_sha256"], c["name"]
    assert _golden.sha(np.asarray(roles, np.uint8)) == c["roles_sha256"], c["name"]


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_dbscan_exact_host_entry(c):
    pts = _golden.points(c["recipe"])
    info = sng.ClusterRunInfo()
    cl = sng.dbscan_exact(sng.Dataset(pts), c["eps"], c["min_pts"], sng.Distance(c["metric"]),
                          info=info)
    _check(c, cl.assignment, cl.role, info.distance_evals, info.edges, cl.cluster_count)


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_build_full_graph_edges(c):
    pts = _golden.points(c["recipe"])
    st = sng.BuildStats()
    g = sng.build_full_graph(sng.Dataset(pts), c["eps"], sng.Distance(c["metric"]), stats=st)
    assert st.distance_evals == c["distance_evals"]
    assert g.edge_count() == c["edges"]
    assert _golden.sha(g.keys) == c["keys_sha256"], c["name"]


@pytest.mark.parametrize("c", [c for c in CASES if c["metric"] == "euclidean"],
                         ids=[c["name"] for c in CASES if c["metric"] == "euclidean"])
def test_dbscan_exact_device_entry(c):
    import torch
    pts = _golden.points(c["recipe"])
    x = torch.from_numpy(pts).cuda()
    labels, roles, gi = sng.dbscan_exact_device(x, c["eps"], c["min_pts"])
    torch.cuda.synchronize()
    _check(c, labels.cpu().numpy(), roles.cpu().numpy(), gi.distance_evals, gi.edges,
           gi.cluster_count)


def test_dbscan_exact_fp64_entry():
    """fp64 values fp32 cannot hold take sngb_dbscan_exact_f64; same result as the
    rate-1 fp64 sng_dbscan (the exact graph is the rate-1 sampled graph)."""
    rng = np.random.default_rng(5)
    pts = rng.random((700, 3))  # fp64, not fp32-exact
    ds = sng.Dataset(pts)
    assert ds.values64 is not None
    info = sng.ClusterRunInfo()
    cl = sng.dbscan_exact(ds, 0.12, 4, info=info)
    c1 = sng.sng_dbscan(ds, sng.SngParams(eps=0.12, min_pts=4, rate=1.0))
    np.testing.assert_array_equal(cl.assignment, c1.assignment)
    np.testing.assert_array_equal(cl.role, c1.role)
    assert info.distance_evals == 700 * 699 // 2


def test_dbscan_exact_validation_order():
    """clusterer.cpp:69-70 (eps, then min_pts) before graph.cpp:18 (empty)."""
    with pytest.raises(sng.InvalidArgument, match="eps must be > 0"):
        sng.dbscan_exact(sng.Dataset(np.zeros((3, 2), np.float32)), 0.0, 0)
    with pytest.raises(sng.InvalidArgument, match="min_pts must be >= 1"):
        sng.dbscan_exact(sng.Dataset(np.zeros((3, 2), np.float32)), 1.0, 0)
