"""Randomised parity sweep: the CUDA path against the oracle on seeded random
problems that cross every internal route -- fp32 / 8-bit / head filters (auto
and forced, every head format), the bitmap / filter / generic Floyd kernels,
the 32- and 64-bit sort, host and device entry points -- over data with ties,
large offsets, tiny ranges and outliers.  Each case is a fixed seed, so a
failure reproduces exactly (the case id names the seed).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2006_06743_b200 as sng  # noqa: E402

ENVS = [
    {},
    {"SNGB_HEAD": "2", "SNGB_HEAD_KIND": "0"},
    {"SNGB_HEAD": "2", "SNGB_HEAD_KIND": "1"},
    {"SNGB_HEAD": "2", "SNGB_HEAD_KIND": "2"},
    {"SNGB_Q8": "2"},
    {"SNGB_Q8": "2", "SNGB_Q8_SPLIT": "0"},
    {"SNGB_FLOYD_NO_BITMAP": "1"},
    {"SNGB_SORT32": "0"},
    {"SNGB_HEAD": "2", "SNGB_FLOYD_NO_BITMAP": "1", "SNGB_TEST_FORCE_IRREGULAR": "3"},
    {"SNGB_Q8": "2", "SNGB_TEST_FORCE_IRREGULAR": "4"},
]


def _data(rng, n, d, kind):
    if kind == "uniform":
        return rng.random((n, d), dtype=np.float32)
    if kind == "blobs":
        k = int(rng.integers(1, 12))
        c = rng.random((k, d)).astype(np.float32) * float(rng.choice([1.0, 10.0, 100.0]))
        return (c[rng.integers(0, k, n)] +
                rng.normal(0, float(rng.choice([0.01, 0.1, 1.0])), (n, d))).astype(np.float32)
    if kind == "grid":  # many exact ties and zero distances
        return rng.integers(0, 4, (n, d)).astype(np.float32)
    if kind == "offset":  # large common offset, small spread (fp32 cancellation)
        return (np.float32(1.0e4) + rng.random((n, d), dtype=np.float32) * np.float32(0.5))
    # outlier: one far point stretching every quantised scale
    x = rng.random((n, d), dtype=np.float32)
    x[int(rng.integers(0, n)), int(rng.integers(0, d))] = np.float32(rng.choice([1e5, -3e4]))
    return x


def _cases():
    rng = np.random.default_rng(20261020)
    out = []
    for cid in range(200):
        n = int(rng.choice([2, 3, 17, 400, 1500, 4000, 9000, 70000, 130000]))
        d = int(rng.choice([1, 2, 3, 5, 8, 16, 32, 33, 64, 130, 300, 784, 1100]))
        kind = str(rng.choice(["uniform", "blobs", "grid", "offset", "outlier"]))
        rate = float(rng.choice([0.002, 0.01, 0.05, 0.2, 0.7, 1.0]))
        if n > 10000:
            rate = float(rng.choice([0.0002, 0.001, 0.003]))
        pairs = n * max(1, min(int(np.ceil(rate * n)), n - 1))
        d = max(1, min(d, 300_000_000 // pairs))  # the oracle finishes in about a second
        q = float(rng.choice([0.001, 0.02, 0.2, 0.5]))
        env = ENVS[cid % len(ENVS)]
        dev = bool(rng.integers(0, 2))
        out.append(pytest.param(cid, n, d, kind, rate, q, env, dev,
                                id=f"c{cid}-n{n}-d{d}-{kind}-r{rate}-{'dev' if dev else 'host'}"))
    return out


@pytest.mark.parametrize("cid,n,d,kind,rate,q,env,dev", _cases())
def test_fuzz_matches_oracle(oracle, monkeypatch, cid, n, d, kind, rate, q, env, dev):
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(1000 + cid)
    pts = np.ascontiguousarray(_data(rng, n, d, kind))
    # eps at a quantile of random pair distances (ties included)
    i = rng.integers(0, n, 256)
    j = rng.integers(0, n, 256)
    dist = np.sqrt(((pts[i].astype(np.float64) - pts[j]) ** 2).sum(1))
    eps = float(np.quantile(dist, q))
    if not eps > 0.0:
        eps = 0.5
    min_pts = int(rng.integers(1, 6))
    seed = int(rng.integers(0, 2**63))
    labels, roles, oinfo, okeys = oracle.sng_dbscan(pts, eps, min_pts, rate, seed)
    if dev:
        x = torch.from_numpy(pts).cuda()
        gl, gr, gi = sng.sng_dbscan_device(x, eps, min_pts, rate, seed)
        keys, _ = sng.sampled_edges_device(x, eps, rate, seed)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(keys.cpu().numpy().view(np.uint64), okeys)
        if n >= 8:  # a query-row range (the multi-GPU shard step)
            rb, re = n // 4, n - n // 3
            rkeys, _ = sng.sampled_edges_device(x, eps, rate, seed, row_begin=rb, row_end=re)
            torch.cuda.synchronize()
            orkeys, _ = oracle.sampled_edges_rows(pts, eps, rate, seed, rb, re)
            np.testing.assert_array_equal(rkeys.cpu().numpy().view(np.uint64), orkeys)
        np.testing.assert_array_equal(gl.cpu().numpy(), labels)
        np.testing.assert_array_equal(gr.cpu().numpy(), roles)
        assert gi.edges == oinfo["edges"] and gi.distance_evals == oinfo["distance_evals"]
    else:
        info = sng.ClusterRunInfo()
        c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=eps, min_pts=min_pts, rate=rate,
                                                           seed=seed), info)
        np.testing.assert_array_equal(c.assignment, labels)
        np.testing.assert_array_equal(c.role, roles)
        assert info.edges == oinfo["edges"] and info.distance_evals == oinfo["distance_evals"]
        assert c.cluster_count == oinfo["cluster_count"]


def _ref_cases():
    rng = np.random.default_rng(7_2026)
    out = []
    for cid in range(60):
        n = int(rng.choice([2, 5, 300, 2000, 6000]))
        d = int(rng.choice([1, 2, 3, 7, 16, 33, 130, 784]))
        metric = str(rng.choice(["euclidean", "manhattan", "cosine"]))
        f64 = bool(rng.integers(0, 2))
        rate = float(rng.choice([0.01, 0.05, 0.3, 1.0]))
        pairs = n * max(1, min(int(np.ceil(rate * n)), n - 1))
        d = max(1, min(d, 60_000_000 // pairs))
        kind = str(rng.choice(["uniform", "blobs", "grid", "offset", "outlier"]))
        q = float(rng.choice([0.01, 0.1, 0.4]))
        env = ENVS[cid % len(ENVS)]
        out.append(pytest.param(cid, n, d, metric, f64, rate, kind, q, env,
                                id=f"r{cid}-n{n}-d{d}-{metric}-{'f64' if f64 else 'f32'}-r{rate}"))
    return out


@pytest.mark.parametrize("cid,n,d,metric,f64,rate,kind,q,env", _ref_cases())
def test_fuzz_metrics_fp64_match_reference(monkeypatch, cid, n, d, metric, f64, rate, kind, q, env):
    """Manhattan / cosine / Euclidean on fp32 and fp64 rows against the
    reference compiled from its own sources (oracle/_ref): labels, roles,
    counters and edge lists identical."""
    import os
    from oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libsngref.so not built")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(5000 + cid)
    pts = _data(rng, n, d, kind).astype(np.float64)
    if metric == "cosine":
        pts = pts + 0.5 + np.abs(pts).max()  # no row at the origin (the reference's error)
    if f64:
        pts = pts + rng.normal(0, 1e-7, pts.shape) * (np.abs(pts) + 1.0)
    else:
        pts = pts.astype(np.float32)
    i = rng.integers(0, n, 256)
    j = rng.integers(0, n, 256)
    a, b = pts[i].astype(np.float64), pts[j].astype(np.float64)
    if metric == "manhattan":
        dist = np.abs(a - b).sum(1)
    elif metric == "cosine":
        dist = 1 - (a * b).sum(1) / np.linalg.norm(a, axis=1) / np.linalg.norm(b, axis=1)
    else:
        dist = np.sqrt(((a - b) ** 2).sum(1))
    eps = float(np.quantile(dist, q))
    if not eps > 0.0:
        eps = 1e-3
    min_pts = int(rng.integers(1, 5))
    seed = int(rng.integers(0, 2**63))
    ref = Reference()
    ref.set_metric(metric)
    try:
        rds = ref.dataset(pts)
        labels, roles, rinfo = ref.sng_dbscan(rds, eps, min_pts, rate, seed)
        keys, _, _ = ref.sampled_edges(rds, eps, rate, seed)
    finally:
        ref.set_metric("euclidean")
    ds = sng.Dataset(pts)
    dm = sng.Distance.parse(metric)
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(ds, sng.SngParams(eps=eps, min_pts=min_pts, rate=rate, seed=seed, dist=dm),
                       info)
    np.testing.assert_array_equal(c.assignment, labels)
    np.testing.assert_array_equal(c.role, roles)
    assert info.edges == rinfo["edges"] and info.distance_evals == rinfo["distance_evals"]
    g = sng.build_sampled_graph(ds, eps, rate, dist=dm, seed=seed)
    np.testing.assert_array_equal(g.keys, keys)
