"""Host-side logic of the Python mirror (no GPU): argument validation with the
reference's messages, Dataset shape rules, generator determinism."""
import numpy as np
import pytest

import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import synthetic


def test_params_validate_messages():  # clusterer.hpp:19-23
    with pytest.raises(sng.InvalidArgument, match="eps must be > 0"):
        sng.SngParams(eps=0.0).validate()
    with pytest.raises(sng.InvalidArgument, match="eps must be > 0"):
        sng.SngParams(eps=float("nan")).validate()
    with pytest.raises(sng.InvalidArgument, match="min_pts must be >= 1"):
        sng.SngParams(eps=1.0, min_pts=0).validate()
    with pytest.raises(sng.InvalidArgument, match=r"rate must lie in \(0, 1\]"):
        sng.SngParams(eps=1.0, rate=0.0).validate()
    with pytest.raises(sng.InvalidArgument, match=r"rate must lie in \(0, 1\]"):
        sng.SngParams(eps=1.0, rate=1.5).validate()
    sng.SngParams(eps=1.0, min_pts=1, rate=1.0).validate()
    assert issubclass(sng.InvalidArgument, ValueError)


def test_dataset_rules():  # dataset.hpp:21-27
    with pytest.raises(sng.InvalidArgument, match="dimension must be >= 1"):
        sng.Dataset([1.0, 2.0], dim=0)
    with pytest.raises(sng.InvalidArgument, match="do not form n x dim rows"):
        sng.Dataset([1.0, 2.0, 3.0], dim=2)
    with pytest.raises(sng.InvalidArgument, match="do not form n x dim rows"):
        sng.Dataset([], dim=2)
    with pytest.raises(sng.InvalidArgument, match="non-finite"):
        sng.Dataset(np.array([[1.0, np.inf]]))
    with pytest.raises(sng.InvalidArgument, match="non-finite"):
        sng.Dataset(np.array([[np.nan, 0.0]], np.float32))
    ds = sng.Dataset(np.arange(6, dtype=np.float64), dim=3)
    assert ds.size() == 2 and ds.dim() == 3 and ds.values.dtype == np.float32
    ds64 = sng.Dataset(np.array([[0.1, 0.2]]))  # fp64 values that fp32 cannot hold exactly
    assert ds64.values64 is not None and ds64.values64.dtype == np.float64
    assert ds.values64 is None  # fp32-exact fp64 input takes the fp32 path


def test_distance_parse():  # distance.hpp:37-43
    assert sng.Distance.parse("euclidean").kind == "euclidean"
    with pytest.raises(sng.InvalidArgument, match="unknown distance 'l7'"):
        sng.Distance.parse("l7")
    assert sng.Distance.parse("cosine").flags == 0x4
    assert sng.Distance.parse("manhattan").flags == 0x2
    with pytest.raises(NotImplementedError):
        sng.Distance.custom(lambda a, b: 0.0)


def test_point_roles_and_noise_label():  # dataset.hpp:13,74
    assert sng.kNoiseLabel == -1
    assert (int(sng.PointRole.Core), int(sng.PointRole.Border), int(sng.PointRole.Noise)) == (0, 1, 2)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_generators_deterministic_and_shaped(cfg):
    w = synthetic.CONFIGS[cfg]
    a = synthetic.generate(cfg, n=3000)
    b = synthetic.generate(cfg, n=3000)
    assert a.shape == (3000, w.d) and a.dtype == np.float32
    np.testing.assert_array_equal(a, b)
    assert np.isfinite(a).all()


def test_workload_geometry_matches_baseline():
    got = {c: (w.n, w.d, w.draws, w.pairs) for c, w in synthetic.CONFIGS.items()}
    assert got == {1: (20000, 2, 2000, 4.0e7), 2: (70000, 784, 700, 4.9e7),
                   3: (10**6, 16, 1000, 10**9), 4: (5 * 10**6, 3, 2500, 1.25e10),
                   5: (2 * 10**7, 32, 4000, 8.0e10)}


def test_device_entry_points_reject_bad_tensors():
    """CPU / wrong-dtype tensors fail with InvalidArgument before any library call
    (a host pointer handed to a kernel would poison the CUDA context)."""
    import torch
    pts = torch.zeros((8, 2), dtype=torch.float32)  # CPU
    with pytest.raises(sng.InvalidArgument, match="CUDA float32"):
        sng.sampled_edges_device(pts, 1.0, 1.0, 0)
    with pytest.raises(sng.InvalidArgument, match="CUDA float32"):
        sng.sng_dbscan_device(pts, 1.0, 1, 1.0, 0)
    keys = torch.zeros(4, dtype=torch.int64)
    with pytest.raises(sng.InvalidArgument, match="CUDA int64"):
        sng.cluster_edges_device(keys, 8, 1)
    with pytest.raises(sng.InvalidArgument, match="CUDA int64"):
        sng.unique_keys_device(keys, 8)
    with pytest.raises(sng.InvalidArgument, match="CUDA int64"):
        sng.degrees_device(keys.to(torch.int32), 8)


def test_bench_relaunch_command():
    """`bench.py --gpus N` outside torchrun re-launches itself as N local ranks."""
    import bench
    cmd = bench.relaunch_cmd(["--gpus", "4", "--steps", "3"], 4, 29511)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-port=29511" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]
    assert cmd[-5].endswith("bench.py")


def test_bench_reference_sample_rate():
    """The reference arm's bounded sample keeps the full dataset and picks a rate
    whose draws (graph.cpp:139-140) are exactly the requested count."""
    import math

    import bench
    w = synthetic.CONFIGS[5]
    for k in (1, 7, 100, 3999):
        r = bench._ref_rate(w, k)
        assert min(math.ceil(r * float(w.n)), w.n - 1) == k
