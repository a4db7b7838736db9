"""The `sngdbscan` pybind11 module (reference proj/CMakeLists.txt:11:
sng_dbscan(points, eps, min_pts, rate, seed, num_gpus) -> (labels, roles,
info)) over libsngb.so."""
import numpy as np
import pytest

import sngdbscan
from tests import _golden


def test_module_loads_and_validates_before_the_gpu():
    assert sngdbscan.ABI_VERSION == 4
    pts = np.zeros((4, 2), np.float32)
    with pytest.raises(ValueError, match="eps must be > 0"):
        sngdbscan.sng_dbscan(pts, 0.0, 1)
    with pytest.raises(ValueError, match="min_pts must be >= 1"):
        sngdbscan.sng_dbscan(pts, 1.0, 0)
    with pytest.raises(ValueError, match=r"rate must lie in \(0, 1\]"):
        sngdbscan.sng_dbscan(pts, 1.0, 1, rate=1.5)
    with pytest.raises(ValueError, match="unknown distance 'l7'"):
        sngdbscan.sng_dbscan(pts, 1.0, 1, dist="l7")
    with pytest.raises(ValueError, match="2-D"):
        sngdbscan.sng_dbscan(np.zeros(4, np.float32), 1.0, 1)
    with pytest.raises(ValueError, match="dataset is empty"):
        sngdbscan.sng_dbscan(np.zeros((0, 2), np.float32), 1.0, 1)


def test_no_gpu_raises():
    if sngdbscan.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        sngdbscan.sng_dbscan(np.zeros((4, 2), np.float32), 1.0, 1)


@pytest.mark.gpu
@pytest.mark.parametrize("c", _golden.cases()[:14], ids=[c["name"] for c in _golden.cases()[:14]])
def test_golden_cases(c):
    pts = _golden.points(c["recipe"])
    labels, roles, info = sngdbscan.sng_dbscan(pts, c["eps"], c["min_pts"], c["rate"], c["seed"])
    assert labels.dtype == np.int32 and roles.dtype == np.uint8
    assert _golden.sha(labels) == c["labels_sha256"]
    assert _golden.sha(roles) == c["roles_sha256"]
    assert info["edges"] == c["edges"] and info["distance_evals"] == c["distance_evals"]
    assert info["cluster_count"] == c["cluster_count"]
    # float64 input holding fp32 values: the same result; several shards on GPU 0
    l64, r64, _ = sngdbscan.sng_dbscan(pts.astype(np.float64), c["eps"], c["min_pts"], c["rate"],
                                       c["seed"], devices=[0, 0])
    np.testing.assert_array_equal(l64, labels)
    np.testing.assert_array_equal(r64, roles)


@pytest.mark.gpu
def test_exact_and_num_gpus():
    c = next(c for c in _golden.load()["exact_cases"] if c["name"] == "exact_rand_500x3")
    pts = _golden.points(c["recipe"])
    labels, roles, info = sngdbscan.dbscan_exact(pts, c["eps"], c["min_pts"], num_gpus=-1)
    assert _golden.sha(labels) == c["labels_sha256"]
    assert info["distance_evals"] == c["distance_evals"]
    rng = np.random.default_rng(3)
    p64 = rng.random((2000, 3))  # fp64 values: the exact fp64 path
    a = sngdbscan.sng_dbscan(p64, 0.08, 4, 0.3, 5)
    b = sngdbscan.sng_dbscan(p64, 0.08, 4, 0.3, 5, devices=[0, 0, 0])
    np.testing.assert_array_equal(a[0], b[0])
    assert b[2]["num_gpus"] == 3
