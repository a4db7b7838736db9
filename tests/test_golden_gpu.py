"""CUDA path vs the REFERENCE's own outputs (tests/golden/golden.json, made
from the compiled reference sources): edge-set digest, labels, roles and the
ClusterRunInfo counters, bit-exact."""
import numpy as np
import pytest

from tests import _golden

pytestmark = pytest.mark.gpu

import paper_2006_06743_b200 as sng  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if sng.device_count() < 1:
        pytest.fail("no CUDA device: the GPU path has no CPU fallback")


@pytest.mark.parametrize("case", _golden.cases(), ids=lambda c: c["name"])
def test_cuda_matches_reference_golden(case):
    pts = _golden.points(case["recipe"])
    assert _golden.sha(pts) == case["points_sha256"]
    st = sng.BuildStats()
    g = sng.build_sampled_graph(sng.Dataset(pts), case["eps"], case["rate"], seed=case["seed"],
                                stats=st)
    assert st.distance_evals == case["edges_evals"]
    assert _golden.sha(g.keys) == case["keys_sha256"]
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=case["eps"], min_pts=case["min_pts"],
                                                       rate=case["rate"], seed=case["seed"]), info)
    assert info.distance_evals == case["distance_evals"]
    assert info.edges == case["edges"]
    assert info.graph_bytes == case["graph_bytes"]
    assert c.cluster_count == case["cluster_count"]
    assert _golden.sha(c.assignment) == case["labels_sha256"]
    assert _golden.sha(c.role) == case["roles_sha256"]
    if "labels" in case:
        assert c.assignment.tolist() == case["labels"]
        assert c.role.tolist() == case["roles"]
