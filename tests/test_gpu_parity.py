"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Bit-exact bar: edge sets, degrees/core masks, labels, roles, cluster counts
and the reference counters (distance_evals, edges, graph_bytes) must be
identical to the oracle on the same inputs and seed.  The oracle itself is
pinned to the compiled reference in tests/test_oracle.py.
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


def _run_both(oracle, pts, eps, min_pts, rate, seed):
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=eps, min_pts=min_pts, rate=rate,
                                                       seed=seed), info)
    labels, roles, oinfo, keys = oracle.sng_dbscan(pts, eps, min_pts, rate, seed)
    return c, info, labels, roles, oinfo, keys


def _assert_same(c, info, labels, roles, oinfo):
    assert info.distance_evals == oinfo["distance_evals"]
    assert info.edges == oinfo["edges"]
    assert info.graph_bytes == oinfo["graph_bytes"]
    assert c.cluster_count == oinfo["cluster_count"]
    np.testing.assert_array_equal(c.role, roles)
    np.testing.assert_array_equal(c.assignment, labels)


def test_kat_line_graph():
    """SURVEY Appendix A KAT (computed from the compiled reference)."""
    pts = np.arange(12, dtype=np.float32).reshape(12, 1)
    st = sng.BuildStats()
    g = sng.build_sampled_graph(sng.Dataset(pts), 1e9, 0.25, seed=1, stats=st)
    want = ("0-1 0-2 0-4 0-6 0-8 0-9 0-11 1-4 1-6 1-7 1-8 2-5 2-7 2-8 2-10 3-7 3-10 3-11 "
            "4-5 4-10 5-10 6-8 6-9 6-10 6-11 7-9 7-11 8-11 9-10 10-11")
    assert g.edges() == [tuple(map(int, e.split("-"))) for e in want.split()]
    assert st.distance_evals == 36
    assert list(g.degree()) == [7, 5, 5, 3, 4, 3, 6, 5, 5, 4, 7, 6]


@pytest.mark.parametrize("n,d,eps,rate,seed", [
    (3, 1, 1.0, 0.5, 0),
    (50, 2, 0.2, 0.3, 7),
    (500, 3, 0.15, 0.1, 3),
    (2000, 16, 1.5, 0.05, 11),
    (3000, 33, 2.0, 0.02, 5),
    (1500, 784, 4.5, 0.03, 2),
    (4000, 2, 0.05, 0.5, 42),
])
def test_edges_match_oracle(oracle, n, d, eps, rate, seed):
    rng = np.random.default_rng(seed)
    pts = rng.random((n, d), dtype=np.float32) * np.float32(1.0 + d ** 0.5 / 2)
    keys, evals = oracle.sampled_edges(pts, eps, rate, seed)
    st = sng.BuildStats()
    g = sng.build_sampled_graph(sng.Dataset(pts), eps, rate, seed=seed, stats=st)
    assert st.distance_evals == evals
    np.testing.assert_array_equal(g.keys, keys)


@pytest.mark.parametrize("cfg,n", [(1, 20_000), (2, 4_000), (3, 30_000), (4, 40_000), (5, 30_000)])
def test_configs_reduced_match_oracle(oracle, cfg, n):
    w = synthetic.CONFIGS[cfg]
    pts = synthetic.generate(cfg, n=n)
    # keep the per-vertex draw count of the full config where possible
    rate = min(1.0, w.draws / n) if cfg != 1 else w.rate
    c, info, labels, roles, oinfo, _ = _run_both(oracle, pts, w.eps, w.min_pts, rate, w.seed)
    _assert_same(c, info, labels, roles, oinfo)


@pytest.mark.parametrize("n,d,eps,min_pts", [(1, 2, 0.5, 1), (2, 2, 0.5, 1), (300, 2, 0.08, 4),
                                              (700, 5, 0.6, 6)])
def test_exhaustive_rate1_matches_oracle(oracle, n, d, eps, min_pts):
    rng = np.random.default_rng(n)
    pts = rng.random((n, d), dtype=np.float32)
    c, info, labels, roles, oinfo, _ = _run_both(oracle, pts, eps, min_pts, 1.0, 9)
    _assert_same(c, info, labels, roles, oinfo)


def test_spec_line_example():
    """SPEC.md clusterer example: {0, 0.5, 10, 10.5}, eps=1, min_pts=1, rate=1."""
    pts = np.array([[0.0], [0.5], [10.0], [10.5]], np.float32)
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=1.0, min_pts=1, rate=1.0))
    assert list(c.assignment) == [0, 0, 1, 1]
    assert c.cluster_count == 2


def test_errors_match_reference_messages():
    pts = np.zeros((4, 2), np.float32)
    with pytest.raises(sng.InvalidArgument, match=r"eps must be > 0"):
        sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=0.0, min_pts=1, rate=1.0))
    with pytest.raises(sng.InvalidArgument, match=r"min_pts must be >= 1"):
        sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=1.0, min_pts=0, rate=1.0))
    with pytest.raises(sng.InvalidArgument, match=r"rate must lie in \(0, 1\]"):
        sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=1.0, min_pts=1, rate=1.5))


def test_device_api_matches_host_api(oracle):
    import torch
    pts = synthetic.generate(1, n=5000)
    t = torch.from_numpy(pts).cuda()
    labels, roles, gi = sng.sng_dbscan_device(t, 0.03, 10, 0.1, 1)
    torch.cuda.synchronize()
    ol, orl, oinfo, _ = oracle.sng_dbscan(pts, 0.03, 10, 0.1, 1)
    np.testing.assert_array_equal(labels.cpu().numpy(), ol)
    np.testing.assert_array_equal(roles.cpu().numpy(), orl)
    assert gi.edges == oinfo["edges"]


@pytest.mark.parametrize("n,d,eps,rate,seed", [(6000, 3, 0.1, 0.8, 4), (9000, 2, 0.02, 0.5, 8),
                                               (40000, 2, 0.004, 0.15, 5)])
def test_large_draws_generic_sampler(oracle, monkeypatch, n, d, eps, rate, seed):
    """draws > 4096 takes the generic (regenerating) Floyd kernel (bitmap mode off)."""
    monkeypatch.setenv("SNGB_FLOYD_NO_BITMAP", "1")
    rng = np.random.default_rng(seed)
    pts = rng.random((n, d), dtype=np.float32)
    keys, evals = oracle.sampled_edges(pts, eps, rate, seed)
    st = sng.BuildStats()
    g = sng.build_sampled_graph(sng.Dataset(pts), eps, rate, seed=seed, stats=st)
    assert st.distance_evals == evals
    np.testing.assert_array_equal(g.keys, keys)


@pytest.mark.parametrize("bitmap", [True, False])
@pytest.mark.parametrize("n,d,eps,rate,seed", [(3000, 2, 0.05, 0.3, 1), (20000, 16, 1.0, 0.02, 3),
                                               (6000, 3, 0.1, 0.8, 4)])
def test_forced_irregular_vertices_exact(oracle, monkeypatch, n, d, eps, rate, seed, bitmap):
    """Force the Lemire-reject pre-condition on every 7th vertex: those vertices
    go through the exact sequential replay; the edge set must not change.
    Runs every Floyd kernel: bitmap (small n), fast (draws <= 4096), generic."""
    if not bitmap:
        monkeypatch.setenv("SNGB_FLOYD_NO_BITMAP", "1")
    rng = np.random.default_rng(seed)
    pts = rng.random((n, d), dtype=np.float32)
    keys, _ = oracle.sampled_edges(pts, eps, rate, seed)
    monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", "7")
    info = sng.ClusterRunInfo()
    g = sng.build_sampled_graph(sng.Dataset(pts), eps, rate, seed=seed)
    np.testing.assert_array_equal(g.keys, keys)
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=eps, min_pts=3, rate=rate, seed=seed),
                       info)
    assert info.gpu["irregular_vertices"] >= (n + 6) // 7  # + list-overflow replays
    ol, orl, _, _ = oracle.sng_dbscan(pts, eps, 3, rate, seed)
    np.testing.assert_array_equal(c.assignment, ol)


def test_product_library_has_no_test_hook(monkeypatch):
    """The product libsngb.so compiles SNGB_TEST_FORCE_IRREGULAR out; only the
    test build (lib/libsngb_testhooks.so, routed by conftest.py) honours it."""
    import ctypes as C
    from paper_2006_06743_b200 import _lib
    rng = np.random.default_rng(3)
    pts = np.ascontiguousarray(rng.random((5000, 3), dtype=np.float32))
    monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", "7")
    counts = []
    for L in (_lib.load(_lib.LIB_PATH), _lib.lib()):
        gi = _lib.SngbInfo()
        lab = np.empty(5000, np.int32)
        rol = np.empty(5000, np.uint8)
        rc = L.sngb_dbscan_f32(pts.ctypes.data_as(C.POINTER(C.c_float)), 5000, 3, 0.05, 3, 0.05,
                               1, None, lab.ctypes.data_as(C.POINTER(C.c_int32)),
                               rol.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(gi))
        assert rc == 0
        counts.append(gi.irregular_vertices)
    assert counts[0] == 0 and counts[1] >= 5000 // 7


def _host_edges_rows(pts, eps, rate, seed, rb, re):
    """sngb_sampled_edges_f32 (host buffers) over the query rows [rb, re)."""
    import ctypes as C
    from paper_2006_06743_b200 import _lib
    n, d = pts.shape
    cap = 1 << 22
    keys = np.empty(cap, np.uint64)
    cnt = C.c_uint64(0)
    o = _lib.SngbOpts(-1, 0, None, rb, re)
    rc = _lib.lib().sngb_sampled_edges_f32(pts.ctypes.data_as(C.POINTER(C.c_float)), n, d, eps,
                                           rate, seed, C.byref(o),
                                           keys.ctypes.data_as(C.POINTER(C.c_uint64)), cap,
                                           C.byref(cnt), None)
    sng._check(rc)
    return keys[: cnt.value]


@pytest.mark.parametrize("phases", [1, 2, 3, 4])
@pytest.mark.parametrize("cfg,n,d", [(2, 3000, 784), (3, 20000, 16)])
def test_chunked_host_upload_matches_oracle(oracle, monkeypatch, phases, cfg, n, d):
    """Host-buffer calls upload the points in row chunks on a copy stream; with
    L2 phases forced, the gather runs as the triangular (query chunk x
    partner slice) schedule as chunks arrive.  Same results as the oracle."""
    monkeypatch.setenv("SNGB_GATHER_PHASES", str(phases))
    w = synthetic.CONFIGS[cfg]
    pts = synthetic.generate(cfg, n=n)
    rate = min(1.0, 4 * w.draws / n)
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=w.eps, min_pts=w.min_pts, rate=rate,
                                                       seed=w.seed), info)
    labels, roles, oinfo, keys = oracle.sng_dbscan(pts, w.eps, w.min_pts, rate, w.seed)
    _assert_same(c, info, labels, roles, oinfo)
    rb, re = n // 3, 2 * n // 3 + 5
    okeys, _ = oracle.sampled_edges_rows(pts, w.eps, rate, w.seed, rb, re)
    np.testing.assert_array_equal(_host_edges_rows(pts, w.eps, rate, w.seed, rb, re), okeys)


def test_nonfinite_rejected_after_deferred_check():
    """The finiteness check is read at the one host sync; the error is still
    the reference's (dataset.hpp:24-26), on both the host and device paths."""
    import torch
    pts = synthetic.generate(1, n=2000)
    pts[1234, 1] = np.nan
    with pytest.raises(sng.InvalidArgument, match="non-finite"):
        _host_edges_rows(pts, 0.03, 0.1, 1, 0, 0)  # raw C ABI, host buffers
    with pytest.raises(sng.InvalidArgument, match="non-finite"):
        sng.sng_dbscan_device(torch.from_numpy(pts).cuda(), 0.03, 10, 0.1, 1)
    # the library is still usable afterwards
    pts[1234, 1] = 0.5
    labels, _, _ = sng.sng_dbscan_device(torch.from_numpy(pts).cuda(), 0.03, 10, 0.1, 1)
    assert labels.numel() == 2000


# ---- the 8-bit filter for wide rows (sngb_quant.cu) ------------------------
def _q8_case(n, d, seed, spread=1.0):
    rng = np.random.default_rng(seed)
    centers = rng.random((8, d), dtype=np.float32)
    pts = centers[rng.integers(0, 8, n)] + rng.normal(0, 0.1 * spread, (n, d)).astype(np.float32)
    return np.ascontiguousarray(pts, np.float32)


@pytest.mark.parametrize("mode", ["0", "1", "2"])
@pytest.mark.parametrize("n,d,rate,seed", [(3000, 128, 0.05, 3), (2500, 784, 0.04, 5),
                                           (2000, 1000, 0.05, 9), (2200, 131, 0.05, 6),
                                           (1800, 250, 0.06, 12)])
def test_q8_filter_matches_oracle(oracle, monkeypatch, mode, n, d, rate, seed):
    """SNGB_Q8=0 (fp32 filter), 1 (auto), 2 (forced): identical to the oracle."""
    monkeypatch.setenv("SNGB_Q8", mode)
    pts = _q8_case(n, d, seed)
    # eps at a within-cluster distance quantile: plenty of pairs near eps
    i = np.arange(0, n - 1, 7)
    dist = np.sqrt(((pts[i] - pts[i + 1]) ** 2).sum(1))
    eps = float(np.quantile(dist, 0.1))
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=eps, min_pts=3, rate=rate, seed=seed),
                       info)
    labels, roles, oinfo, keys = oracle.sng_dbscan(pts, eps, 3, rate, seed)
    _assert_same(c, info, labels, roles, oinfo)


def test_q8_band_stress_exact(oracle, monkeypatch):
    """Every pair distance within a few percent of eps: the band holds most
    pairs, which all take the exact fp64 recheck -- still bit-exact."""
    monkeypatch.setenv("SNGB_Q8", "2")
    rng = np.random.default_rng(11)
    n, d = 2000, 256
    base = rng.random(d, dtype=np.float32)
    pts = (base + rng.normal(0, 0.05, (n, d))).astype(np.float32)
    i = np.arange(0, n - 1, 3)
    eps = float(np.median(np.sqrt(((pts[i] - pts[i + 1]) ** 2).sum(1))))
    st = sng.BuildStats()
    g = sng.build_sampled_graph(sng.Dataset(pts), eps, 0.1, seed=2, stats=st)
    keys, evals = oracle.sampled_edges(pts, eps, 0.1, 2)
    np.testing.assert_array_equal(g.keys, keys)
    assert st.distance_evals == evals


def test_q8_huge_range_forced(oracle, monkeypatch):
    """A value range far wider than eps: auto keeps the fp32 filter, forcing the
    8-bit one puts nearly every pair in the band -- results unchanged."""
    pts = _q8_case(1500, 160, 4)
    pts[17, 3] = 1e6  # one far outlier stretches the 8-bit scale
    eps = 1.5
    keys, _ = oracle.sampled_edges(pts, eps, 0.05, 4)
    for mode in ("1", "2"):
        monkeypatch.setenv("SNGB_Q8", mode)
        g = sng.build_sampled_graph(sng.Dataset(pts), eps, 0.05, seed=4)
        np.testing.assert_array_equal(g.keys, keys)


def test_q8_forced_irregular_exact(oracle, monkeypatch):
    """Lemire-reject replays (test hook) through the 8-bit gather kernel."""
    pts = _q8_case(3000, 200, 8)
    eps = 1.2
    keys, _ = oracle.sampled_edges(pts, eps, 0.04, 8)
    monkeypatch.setenv("SNGB_Q8", "2")
    monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", "5")
    g = sng.build_sampled_graph(sng.Dataset(pts), eps, 0.04, seed=8)
    np.testing.assert_array_equal(g.keys, keys)


@pytest.mark.parametrize("stretch,bits", [(1.0, 8), (2.5, 8), (5.0, 32)])
def test_q8_pipelined_host_upload(oracle, stretch, bits):
    """Host-buffer call, 2 upload chunks: the 8-bit plan is made from chunk 0 and
    the gather starts before the rest arrives.  With stretch > 2 the last rows
    leave chunk 0's range, the end-of-build check fails and the build is redone
    from the global range: still 8-bit at 2.5, the fp32 filter at 5 (the band
    of the global scale is too wide) -- all bit-identical to the oracle."""
    n, d = 25000, 784
    pts = synthetic.generate(2, n=n)
    pts[n - 3000:] *= stretch
    rate, seed, eps = 100 / n, 2, 4.5
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=eps, min_pts=5, rate=rate, seed=seed),
                       info)
    labels, roles, oinfo, keys = oracle.sng_dbscan(pts, eps, 5, rate, seed)
    _assert_same(c, info, labels, roles, oinfo)
    assert info.gpu["filter_bits"] == bits


@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("n,d,rate,seed,q", [(1500, 256, 0.08, 21, 0.1), (2000, 640, 0.05, 22, 0.1),
                                             (1600, 1300, 0.05, 23, 0.1), (2500, 784, 0.04, 24, 0.5),
                                             (1800, 1000, 0.05, 25, 0.9)])
def test_q8_early_reject_matches_oracle(oracle, monkeypatch, split, n, d, rate, seed, q):
    """The head/tail gather (SNGB_Q8_SPLIT=1; tail slots 1, 2 and 3 warp widths)
    and the one-pass gather (=0) on the same wide rows: identical to the oracle,
    with eps at low and high within-cluster quantiles (few / many survivors)."""
    monkeypatch.setenv("SNGB_Q8", "2")
    monkeypatch.setenv("SNGB_Q8_SPLIT", split)
    pts = _q8_case(n, d, seed)
    i = np.arange(0, n - 1, 7)
    eps = float(np.quantile(np.sqrt(((pts[i] - pts[i + 1]) ** 2).sum(1)), q))
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=eps, min_pts=3, rate=rate, seed=seed),
                       info)
    labels, roles, oinfo, keys = oracle.sng_dbscan(pts, eps, 3, rate, seed)
    _assert_same(c, info, labels, roles, oinfo)
    assert info.gpu["filter_bits"] == 8


def test_q8_early_reject_irregular_exact(oracle, monkeypatch):
    """Lemire-reject replays through the head/tail gather."""
    pts = _q8_case(2500, 784, 8)
    eps = 3.0
    keys, _ = oracle.sampled_edges(pts, eps, 0.04, 8)
    monkeypatch.setenv("SNGB_Q8", "2")
    monkeypatch.setenv("SNGB_Q8_SPLIT", "1")
    monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", "5")
    g = sng.build_sampled_graph(sng.Dataset(pts), eps, 0.04, seed=8)
    np.testing.assert_array_equal(g.keys, keys)


def test_q8_early_reject_reads_fewer_bytes():
    """On the cfg2 data most sampled pairs are rejected by their head: the
    algorithmic bytes (head for every pair, tail for survivors) fall well below
    a full row per pair."""
    n, d = 20000, 784
    pts = synthetic.generate(2, n=n)
    info = sng.ClusterRunInfo()
    sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=4.5, min_pts=10, rate=0.01, seed=2), info)
    g = info.gpu
    assert g["filter_bits"] == 8
    assert g["gather_bytes"] < 0.6 * g["gather_pairs"] * (d + 4)


# ---- the head filter for narrow rows beyond L2 (sngb_head.cu) --------------
def _head_case(n, d, seed, k=12, spread=0.05, box=20.0):
    rng = np.random.default_rng(seed)
    centers = (rng.random((k, d)) * box).astype(np.float32)
    pts = centers[rng.integers(0, k, n)] + rng.normal(0, spread, (n, d)).astype(np.float32)
    return np.ascontiguousarray(pts, np.float32)


@pytest.mark.parametrize("bloom", [False, True, "unfused"])
@pytest.mark.parametrize("mode,kind", [("0", "99"), ("2", "0"), ("2", "1"), ("2", "2")])
@pytest.mark.parametrize("n,d,rate,seed,q", [(3000, 3, 0.05, 31, 0.3), (2500, 5, 0.06, 32, 0.5),
                                             (3000, 8, 0.05, 33, 0.2), (2800, 16, 0.05, 34, 0.6),
                                             (3000, 32, 0.04, 35, 0.3), (2000, 33, 0.06, 36, 0.9),
                                             (2200, 64, 0.05, 37, 0.4), (1800, 100, 0.06, 38, 0.5),
                                             (1500, 200, 0.08, 39, 0.3)])
def test_head_filter_matches_oracle(oracle, monkeypatch, bloom, mode, kind, n, d, rate, seed, q):
    """SNGB_HEAD=2 forces the head filter (exact reject on a head of two 16-bit,
    four 8-bit or two 8-bit coordinates -- SNGB_HEAD_KIND 0/1/2 -- fp32 test for
    survivors) on every row width it serves; =0 is the plain fp32 gather.  eps at
    low and high within-cluster quantiles (few / many survivors): all identical
    to the oracle.  bloom=True runs the large-n Floyd bookkeeping fused into the
    head gather (sngb_fused.cu), "unfused" the same as two kernels
    (k_floyd_bloom + k_gather_head), False the bitmap Floyd kernel."""
    monkeypatch.setenv("SNGB_HEAD", mode)
    monkeypatch.setenv("SNGB_HEAD_KIND", kind)
    if bloom:
        monkeypatch.setenv("SNGB_FLOYD_NO_BITMAP", "1")
    monkeypatch.setenv("SNGB_FUSED", "0" if bloom == "unfused" else "1")
    monkeypatch.setenv("SNGB_Q8", "0")
    pts = _head_case(n, d, seed)
    i = np.arange(0, n - 1, 5)
    dist = np.sqrt(((pts[i] - pts[i + 1]) ** 2).sum(1))
    dist = dist[dist < 1.0]  # within-cluster pairs
    eps = float(np.quantile(dist, q))
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=eps, min_pts=3, rate=rate, seed=seed),
                       info)
    labels, roles, oinfo, keys = oracle.sng_dbscan(pts, eps, 3, rate, seed)
    _assert_same(c, info, labels, roles, oinfo)
    assert info.gpu["filter_bits"] == (16 if mode == "2" else 32)
    if mode == "2":  # survivors read their row: the gather moves fewer bytes than fp32
        g = info.gpu
        assert g["head_bytes"] == (2 if kind == "2" else 4)
        assert g["gather_bytes"] < g["gather_pairs"] * 4 * d


def test_head_filter_band_stress_exact(oracle, monkeypatch):
    """One tight blob and eps at the median pair distance: the head rejects
    almost nothing, most pairs take the fp32 test and many its band -- exact."""
    monkeypatch.setenv("SNGB_HEAD", "2")
    rng = np.random.default_rng(41)
    n, d = 3000, 24
    pts = (rng.random(d, dtype=np.float32) + rng.normal(0, 0.05, (n, d))).astype(np.float32)
    i = np.arange(0, n - 1, 3)
    eps = float(np.median(np.sqrt(((pts[i] - pts[i + 1]) ** 2).sum(1))))
    st = sng.BuildStats()
    g = sng.build_sampled_graph(sng.Dataset(pts), eps, 0.1, seed=3, stats=st)
    keys, evals = oracle.sampled_edges(pts, eps, 0.1, 3)
    np.testing.assert_array_equal(g.keys, keys)
    assert st.distance_evals == evals


def test_head_filter_outlier_and_irregular_exact(oracle, monkeypatch):
    """A far outlier stretches the 16-bit scale (coarse head); Lemire-reject
    replays (test hook) through the head gather -- the edge set is unchanged."""
    pts = _head_case(4000, 32, 42)
    pts[77, 0] = 3e5
    eps = 0.4
    keys, _ = oracle.sampled_edges(pts, eps, 0.04, 42)
    monkeypatch.setenv("SNGB_HEAD", "2")
    for kind, bloom in (("0", False), ("1", False), ("2", False), ("0", True), ("2", True),
                        ("1", "unfused"), ("2", "unfused")):
        monkeypatch.setenv("SNGB_HEAD_KIND", kind)
        if bloom:  # the large-n Floyd bookkeeping (fused into the head gather)
            monkeypatch.setenv("SNGB_FLOYD_NO_BITMAP", "1")
        monkeypatch.setenv("SNGB_FUSED", "0" if bloom == "unfused" else "1")
        monkeypatch.delenv("SNGB_TEST_FORCE_IRREGULAR", raising=False)
        g = sng.build_sampled_graph(sng.Dataset(pts), eps, 0.04, seed=42)
        np.testing.assert_array_equal(g.keys, keys)
        monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", "5")
        g = sng.build_sampled_graph(sng.Dataset(pts), eps, 0.04, seed=42)
        np.testing.assert_array_equal(g.keys, keys)


def test_head_filter_device_api_and_row_range(oracle, monkeypatch):
    """Device-resident call and a query-row range (the multi-GPU shard step)."""
    import torch
    monkeypatch.setenv("SNGB_HEAD", "2")
    monkeypatch.setenv("SNGB_HEAD_KIND", "2")
    monkeypatch.setenv("SNGB_FLOYD_NO_BITMAP", "1")
    pts = _head_case(6000, 32, 43)
    eps, rate, seed = 0.3, 0.03, 43
    labels, roles, gi = sng.sng_dbscan_device(torch.from_numpy(pts).cuda(), eps, 4, rate, seed)
    torch.cuda.synchronize()
    ol, orl, oinfo, _ = oracle.sng_dbscan(pts, eps, 4, rate, seed)
    np.testing.assert_array_equal(labels.cpu().numpy(), ol)
    np.testing.assert_array_equal(roles.cpu().numpy(), orl)
    rb, re = 1000, 4321
    okeys, _ = oracle.sampled_edges_rows(pts, eps, rate, seed, rb, re)
    np.testing.assert_array_equal(_host_edges_rows(pts, eps, rate, seed, rb, re), okeys)


@pytest.mark.parametrize("fused", ["1", "0"])
def test_head_filter_auto_on_cfg5_shape(oracle, monkeypatch, fused):
    """cfg5's row shape (d = 32) with the fp32 table beyond half the L2: auto
    selects the head filter (fused with the Floyd bookkeeping, or the two
    kernels with SNGB_FUSED=0); labels identical to the oracle."""
    monkeypatch.setenv("SNGB_FUSED", fused)
    n = 600_000
    pts = synthetic.generate(5, n=n)
    w = synthetic.CONFIGS[5]
    rate = 60 / n
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=w.eps, min_pts=w.min_pts, rate=rate,
                                                       seed=w.seed), info)
    labels, roles, oinfo, keys = oracle.sng_dbscan(pts, w.eps, w.min_pts, rate, w.seed)
    _assert_same(c, info, labels, roles, oinfo)
    assert info.gpu["filter_bits"] == 16


# ---- fp64 input (the reference's Dataset type) -----------------------------
def _ref_or_skip():
    import os
    from oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libsngref.so not built")
    return Reference()


@pytest.mark.parametrize("q8", ["0", "1"])
@pytest.mark.parametrize("n,d,eps,rate,seed,scale", [
    (3000, 2, 0.03, 0.1, 1, 1.0), (4000, 16, 0.5, 0.05, 3, 1.0), (2500, 200, 1.4, 0.05, 7, 1.0),
    (2000, 784, 4.5, 0.05, 2, 1.0), (3000, 3, 0.1, 0.2, 4, 1e4)])
def test_fp64_input_matches_reference(monkeypatch, q8, n, d, eps, rate, seed, scale):
    """fp64 data that fp32 cannot hold: the f64 entry points (fp32 / 8-bit filter
    on rounded or requantised values, widened band, fp64 recheck on the fp64
    rows) against the reference compiled from its own sources."""
    ref = _ref_or_skip()
    monkeypatch.setenv("SNGB_Q8", q8)
    rng = np.random.default_rng(seed)
    cfg = {2: 1, 16: 3, 3: 4}.get(d, 2)
    base = synthetic.generate(cfg, n=n).astype(np.float64) if d in (2, 16, 3, 784) else \
        rng.random((n, d)) * 2.0
    pts = base * scale + rng.normal(0, 1e-7, base.shape) * scale  # break fp32 exactness
    ds = sng.Dataset(pts)
    assert ds.values64 is not None
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(ds, sng.SngParams(eps=eps * scale, min_pts=4, rate=rate, seed=seed), info)
    rds = ref.dataset(pts)
    labels, roles, rinfo = ref.sng_dbscan(rds, eps * scale, 4, rate, seed)
    np.testing.assert_array_equal(c.assignment, labels)
    np.testing.assert_array_equal(c.role, roles)
    assert info.edges == rinfo["edges"] and info.distance_evals == rinfo["distance_evals"]
    keys, evals, _ = ref.sampled_edges(rds, eps * scale, rate, seed)
    g = sng.build_sampled_graph(ds, eps * scale, rate, seed=seed)
    np.testing.assert_array_equal(g.keys, keys)


def test_fp64_band_edges_exact():
    """fp64 pairs placed within a few ulps of eps: the fp32 rounding cannot
    decide them, the fp64 recheck must, exactly as the reference."""
    ref = _ref_or_skip()
    n, d = 2000, 8
    rng = np.random.default_rng(21)
    centers = rng.random((n // 2, d))
    direction = rng.normal(size=(n // 2, d))
    direction /= np.linalg.norm(direction, axis=1, keepdims=True)
    eps = 0.3
    jitter = rng.choice([-3, -1, 0, 1, 3], size=(n // 2, 1)) * 1e-15
    pts = np.concatenate([centers, centers + direction * (eps + jitter)])
    ds = sng.Dataset(pts)
    assert ds.values64 is not None
    g = sng.build_sampled_graph(ds, eps, 1.0, seed=3)
    keys, _, _ = ref.sampled_edges(ref.dataset(pts), eps, 1.0, 3)
    np.testing.assert_array_equal(g.keys, keys)


# ---- Manhattan and cosine (distance.hpp:55-68, 91-103) ----------------------
@pytest.mark.parametrize("metric", ["manhattan", "cosine"])
@pytest.mark.parametrize("n,d,rate,seed,f64", [
    (3000, 2, 0.1, 1, False), (4000, 16, 0.05, 3, False), (2500, 200, 0.05, 7, False),
    (2000, 784, 0.05, 2, False), (3000, 16, 0.05, 5, True), (600, 8, 1.0, 9, False)])
def test_metric_matches_reference(metric, n, d, rate, seed, f64):
    ref = _ref_or_skip()
    ref.set_metric(metric)
    try:
        rng = np.random.default_rng(seed)
        cfg = {2: 1, 16: 3, 784: 2}.get(d)
        pts = synthetic.generate(cfg, n=n).astype(np.float64) if cfg else rng.random((n, d))
        if metric == "cosine":
            pts = pts + 0.5  # keep rows away from the origin
        if f64:
            pts = pts + rng.normal(0, 1e-7, pts.shape)
        else:
            pts = pts.astype(np.float32)
        # eps at a low quantile of the pair distances: plenty of accepted pairs
        i = np.arange(0, n - 1, 5)
        a, b = pts[i].astype(np.float64), pts[i + 1].astype(np.float64)
        dist = np.abs(a - b).sum(1) if metric == "manhattan" else \
            1 - (a * b).sum(1) / np.linalg.norm(a, axis=1) / np.linalg.norm(b, axis=1)
        eps = float(np.quantile(dist, 0.1))
        ds = sng.Dataset(pts)
        dm = sng.Distance.parse(metric)
        info = sng.ClusterRunInfo()
        c = sng.sng_dbscan(ds, sng.SngParams(eps=eps, min_pts=3, rate=rate, seed=seed, dist=dm),
                           info)
        rds = ref.dataset(pts)
        labels, roles, rinfo = ref.sng_dbscan(rds, eps, 3, rate, seed)
        np.testing.assert_array_equal(c.assignment, labels)
        np.testing.assert_array_equal(c.role, roles)
        assert info.edges == rinfo["edges"] and info.distance_evals == rinfo["distance_evals"]
        keys, _, _ = ref.sampled_edges(rds, eps, rate, seed)
        g = sng.build_sampled_graph(ds, eps, rate, dist=dm, seed=seed)
        np.testing.assert_array_equal(g.keys, keys)
    finally:
        ref.set_metric("euclidean")


def test_cosine_zero_vector_is_an_error():
    pts = np.random.default_rng(0).random((500, 8), dtype=np.float32)
    pts[77] = 0.0
    p = sng.SngParams(eps=0.1, min_pts=3, rate=0.1, seed=1, dist=sng.Distance.cosine())
    with pytest.raises(sng.InvalidArgument, match="cosine distance is undefined for zero vectors"):
        sng.sng_dbscan(sng.Dataset(pts), p)
    pts[77] = 1e-30  # tiny but non-zero in fp64: not an error
    sng.sng_dbscan(sng.Dataset(pts), p)


def test_batch_equals_separate_calls(oracle):
    """sngb_dbscan_batch_f32: 40 small problems of mixed shape and metric run
    concurrently; every result equals its separate call (and the oracle)."""
    rng = np.random.default_rng(5)
    problems = []
    for i in range(40):
        n = int(rng.integers(300, 6000))
        cfg = [1, 3, 4][i % 3]
        w = synthetic.CONFIGS[cfg]
        pts = synthetic.generate(cfg, n=n)
        dist = sng.Distance.euclidean() if i % 5 else sng.Distance.manhattan()
        rate = min(1.0, float(rng.uniform(0.02, 0.3)))
        problems.append((pts, sng.SngParams(eps=w.eps * (1.5 if i % 5 == 0 else 1.0),
                                             min_pts=w.min_pts, rate=rate, seed=i, dist=dist)))
    got = sng.sng_dbscan_batch(problems)
    for (pts, p), c in zip(problems, got):
        single = sng.sng_dbscan(sng.Dataset(pts), p)
        np.testing.assert_array_equal(c.assignment, single.assignment)
        np.testing.assert_array_equal(c.role, single.role)
        assert c.cluster_count == single.cluster_count
        if p.dist.kind == "euclidean":
            labels, roles, _, _ = oracle.sng_dbscan(pts, p.eps, p.min_pts, p.rate, p.seed)
            np.testing.assert_array_equal(c.assignment, labels)


# ---- edge shapes ----------------------------------------------------------
@pytest.mark.parametrize("n,d,rate", [(1, 3, 0.5), (2, 1, 1.0), (2, 5, 0.3), (3, 2000, 0.7),
                                      (1200, 1500, 0.05), (800, 3000, 1.0)])
def test_edge_shapes_match_oracle(oracle, n, d, rate):
    """n = 1 and 2 (no or one draw), and rows wider than the specialised
    gathers (d > 1024: the generic kernel), incl. the s = 1 branch."""
    rng = np.random.default_rng(n + d)
    pts = rng.random((n, d), dtype=np.float32)
    i = np.arange(0, max(n - 1, 1), 3)
    eps = float(np.quantile(np.sqrt(((pts[i] - pts[np.minimum(i + 1, n - 1)]) ** 2).sum(1)), 0.2)
                if n > 1 else 1.0) + 1e-3
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=eps, min_pts=2, rate=rate, seed=3),
                       info)
    labels, roles, oinfo, keys = oracle.sng_dbscan(pts, eps, 2, rate, 3)
    _assert_same(c, info, labels, roles, oinfo)


@pytest.mark.parametrize("n", [92682, 92683])
def test_sort32_triangular_keys_boundary(oracle, monkeypatch, n):
    """n(n-1)/2 <= 2^32 (n <= 92 682) sorts the build's keys as 32-bit
    upper-triangular indices, one more point takes the 64-bit sort: both give
    the oracle's edge list, as does SNGB_SORT32=0."""
    rng = np.random.default_rng(n)
    pts = rng.random((n, 2), dtype=np.float32)
    eps, rate, seed = 0.01, 40 / n, 7
    keys, _ = oracle.sampled_edges(pts, eps, rate, seed)
    for mode in ("1", "0"):
        monkeypatch.setenv("SNGB_SORT32", mode)
        g = sng.build_sampled_graph(sng.Dataset(pts), eps, rate, seed=seed)
        np.testing.assert_array_equal(g.keys, keys)


@pytest.mark.parametrize("pre", ["1", "0"])
@pytest.mark.parametrize("force", [None, "5"])
@pytest.mark.parametrize("chunks", ["8", "3"])
def test_q8_host_upload_bucketed_partners(oracle, monkeypatch, pre, force, chunks):
    """Host-buffer calls with the 8-bit head/tail gather over upload chunks read
    their draws' partners from lists bucketed by partner slice (SNGB_PARTNERS=1)
    instead of regenerating every earlier row's draws in each triangle launch;
    an irregular vertex's lists stop at its first fired draw; uneven slices
    (3 chunks).  Identical to the oracle either way, also for a row range."""
    monkeypatch.setenv("SNGB_Q8", "2")
    monkeypatch.setenv("SNGB_PARTNERS", pre)
    monkeypatch.setenv("SNGB_Q8_CHUNKS", chunks)
    if force:
        monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", force)
    n, d = 4001, 784
    pts = _q8_case(n, d, 61)
    i = np.arange(0, n - 1, 7)
    eps = float(np.quantile(np.sqrt(((pts[i] - pts[i + 1]) ** 2).sum(1)), 0.2))
    rate, seed = 0.05, 61
    info = sng.ClusterRunInfo()
    c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=eps, min_pts=3, rate=rate, seed=seed),
                       info)
    labels, roles, oinfo, keys = oracle.sng_dbscan(pts, eps, 3, rate, seed)
    _assert_same(c, info, labels, roles, oinfo)
    assert info.gpu["filter_bits"] == 8
    rb, re = 1000, 3100
    okeys, _ = oracle.sampled_edges_rows(pts, eps, rate, seed, rb, re)
    np.testing.assert_array_equal(_host_edges_rows(pts, eps, rate, seed, rb, re), okeys)


@pytest.mark.parametrize("host", [False, True])
def test_q8_variance_ordered_head(oracle, monkeypatch, host):
    """Rows whose first 300 coordinates are constant (an image's blank border):
    with the columns stored in order of decreasing variance the 8-bit head
    rejects as usual; in natural order it cannot (its values never differ).
    Identical to the oracle either way; the head order reads far fewer bytes."""
    import torch
    rng = np.random.default_rng(71)
    n, d = 6000, 784
    centers = rng.random((10, d - 300), dtype=np.float32)
    body = centers[rng.integers(0, 10, n)] + rng.normal(0, 0.1, (n, d - 300)).astype(np.float32)
    pts = np.ascontiguousarray(np.concatenate([np.zeros((n, 300), np.float32), body], 1))
    eps, rate, seed = 3.5, 0.05, 71
    labels, roles, oinfo, keys = oracle.sng_dbscan(pts, eps, 5, rate, seed)
    monkeypatch.setenv("SNGB_Q8", "2")
    got = {}
    for perm in ("1", "0"):
        monkeypatch.setenv("SNGB_Q8_PERM", perm)
        if host:
            info = sng.ClusterRunInfo()
            c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=eps, min_pts=5, rate=rate,
                                                               seed=seed), info)
            _assert_same(c, info, labels, roles, oinfo)
            got[perm] = info.gpu["gather_bytes"]
        else:
            x = torch.from_numpy(pts).cuda()
            gl, gr, gi = sng.sng_dbscan_device(x, eps, 5, rate, seed)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(gl.cpu().numpy(), labels)
            np.testing.assert_array_equal(gr.cpu().numpy(), roles)
            assert gi.edges == oinfo["edges"]
            got[perm] = gi.gather_bytes
    assert got["1"] < 0.6 * got["0"], got


@pytest.mark.parametrize("cfg,n,fh", [(3, 200_000, "1"), (4, 400_000, "1"), (5, 300_000, "1"),
                                      (4, 1_000_000, "1"), (5, 2_500_000, "1"), (4, 400_000, "0"),
                                      (5, 300_000, "0")])
def test_fused_floyd_head_equals_two_kernels(monkeypatch, cfg, n, fh):
    """The fused paths (sngb_fused.cu: k_floyd_head, block per vertex, for
    draws > 1024; k_sample_head, warp per vertex, below that or with SNGB_FH=0)
    against the two kernels they replace, on reduced BASELINE shapes (the bloom
    regime; the two largest with cfg4/cfg5's chain density): the same edge list,
    collisions and pair counts; also with forced Lemire replays."""
    import torch
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg, n=n)).cuda()
    rate = w.draws / n
    monkeypatch.setenv("SNGB_FH", fh)
    for force in (None, "9"):
        if force:
            monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", force)
        monkeypatch.setenv("SNGB_FUSED", "1")
        kf, gf = sng.sampled_edges_device(x, w.eps, rate, w.seed)
        monkeypatch.setenv("SNGB_FUSED", "0")
        k2, g2 = sng.sampled_edges_device(x, w.eps, rate, w.seed)
        torch.cuda.synchronize()
        assert gf.filter_bits == g2.filter_bits == 16
        assert torch.equal(kf, k2), (cfg, force)
        assert gf.collisions == g2.collisions
        assert gf.irregular_vertices == g2.irregular_vertices
        if not force:
            assert gf.gather_pairs == g2.gather_pairs == gf.draws * n
            assert gf.pairs_evaluated == g2.pairs_evaluated


@pytest.mark.parametrize("cfg,n", [(4, 400_000), (5, 300_000), (4, 1_000_000), (5, 2_500_000)])
def test_headpipe_equals_two_kernels(monkeypatch, cfg, n):
    """k_floyd_headpipe (sngb_floyd_headpipe.cuh, SNGB_FUSED=4: k_floyd_pipe's workers
    also take the head test and their survivors' fp32 test, one RNG pass) against
    the two kernels on reduced cfg4/cfg5 shapes: the same edge list, collisions,
    replayed vertices and pair counts; with forced Lemire replays and a row range."""
    import torch
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg, n=n)).cuda()
    rate = w.draws / n
    for force, rows in ((None, (0, 0)), ("9", (0, 0)), (None, (n // 4, n // 2 + 3))):
        if force:
            monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", force)
        else:
            monkeypatch.delenv("SNGB_TEST_FORCE_IRREGULAR", raising=False)
        monkeypatch.setenv("SNGB_FUSED", "4")
        kf, gf = sng.sampled_edges_device(x, w.eps, rate, w.seed, rows[0], rows[1])
        monkeypatch.setenv("SNGB_FUSED", "0")
        monkeypatch.setenv("SNGB_FLOYD_PIPE", "0")
        k2, g2 = sng.sampled_edges_device(x, w.eps, rate, w.seed, rows[0], rows[1])
        monkeypatch.delenv("SNGB_FLOYD_PIPE", raising=False)
        torch.cuda.synchronize()
        assert gf.filter_bits == g2.filter_bits == 16
        assert torch.equal(kf, k2), (cfg, force, rows)
        assert gf.collisions == g2.collisions > 0
        assert gf.irregular_vertices == g2.irregular_vertices
        assert gf.kernel_launches < g2.kernel_launches
        if not force:
            assert gf.gather_pairs == g2.gather_pairs
            assert gf.pairs_evaluated == g2.pairs_evaluated
            assert gf.band_rechecks == g2.band_rechecks


@pytest.mark.parametrize("cfg,n,split", [(4, 400_000, None), (5, 300_000, None), (4, 1_000_000, "0"),
                                         (5, 2_500_000, "0"), (5, 2_500_000, None)])
def test_duo_equals_two_kernels(monkeypatch, cfg, n, split):
    """k_duo (sngb_fused.cu, SNGB_FUSED=3: the Floyd bookkeeping and the head gather
    as two roles of one launch) against the two kernels on reduced cfg4/cfg5
    shapes: the same edge list, collisions, replayed vertices and pair counts;
    with forced Lemire replays, a row range, and both role layouts."""
    import torch
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg, n=n)).cuda()
    rate = w.draws / n
    if split is not None:
        monkeypatch.setenv("SNGB_DUO_SPLIT", split)
    for force, rows in ((None, (0, 0)), ("9", (0, 0)), (None, (n // 4, n // 2 + 3))):
        if force:
            monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", force)
        else:
            monkeypatch.delenv("SNGB_TEST_FORCE_IRREGULAR", raising=False)
        monkeypatch.setenv("SNGB_FUSED", "3")
        kf, gf = sng.sampled_edges_device(x, w.eps, rate, w.seed, rows[0], rows[1])
        monkeypatch.setenv("SNGB_FUSED", "0")
        monkeypatch.setenv("SNGB_FLOYD_PIPE", "0")
        k2, g2 = sng.sampled_edges_device(x, w.eps, rate, w.seed, rows[0], rows[1])
        monkeypatch.delenv("SNGB_FLOYD_PIPE", raising=False)
        torch.cuda.synchronize()
        assert gf.filter_bits == g2.filter_bits == 16
        assert torch.equal(kf, k2), (cfg, force, rows)
        assert gf.collisions == g2.collisions > 0
        assert gf.irregular_vertices == g2.irregular_vertices
        assert gf.gather_pairs == g2.gather_pairs
        assert gf.pairs_evaluated == g2.pairs_evaluated
        assert gf.kernel_launches < g2.kernel_launches


@pytest.mark.parametrize("cfg,n", [(4, 400_000), (5, 300_000), (4, 1_000_000), (5, 2_500_000)])
def test_floyd_lean_equals_bloom(monkeypatch, cfg, n):
    """k_floyd_lean (sngb_floyd_lean.cuh, the default above 1024 draws) against
    k_floyd_bloom (SNGB_FLOYD_LEAN=0) on reduced cfg4/cfg5 shapes: the same edge
    list, Floyd collisions and replayed vertices, with forced Lemire replays too."""
    import torch
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg, n=n)).cuda()
    rate = w.draws / n
    monkeypatch.setenv("SNGB_FUSED", "0")
    monkeypatch.setenv("SNGB_FLOYD_WARP", "0")
    monkeypatch.setenv("SNGB_FLOYD_PIPE", "0")
    for force in (None, "7"):
        if force:
            monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", force)
        monkeypatch.delenv("SNGB_FLOYD_LEAN", raising=False)
        kl, gl = sng.sampled_edges_device(x, w.eps, rate, w.seed)
        monkeypatch.setenv("SNGB_FLOYD_LEAN", "0")
        kb, gb = sng.sampled_edges_device(x, w.eps, rate, w.seed)
        torch.cuda.synchronize()
        assert gl.draws > 1024
        assert torch.equal(kl, kb), (cfg, force)
        assert gl.collisions == gb.collisions > 0
        assert gl.irregular_vertices == gb.irregular_vertices
        if force:
            assert gl.irregular_vertices >= n // 7


@pytest.mark.parametrize("cfg,n,draws", [(4, 400_000, None), (5, 300_000, None), (4, 1_000_000, None),
                                         (5, 2_500_000, None), (5, 300_000, 4096), (5, 300_000, 1025),
                                         (4, 300_000, 1281), (3, 60_000, 3000)])
def test_floyd_pipe_equals_bloom(monkeypatch, cfg, n, draws):
    """k_floyd_pipe (sngb_floyd_pipe.cuh: the workers resolve their own group
    entries, pipelined over the vertex loop) against k_floyd_bloom on reduced
    cfg3/cfg4/cfg5 shapes and the draw counts at the ends of its range: the same
    edge list, Floyd collisions and replayed vertices, with forced Lemire replays
    and a row range too."""
    import torch
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg, n=n)).cuda()
    rate = (draws or w.draws) / n
    monkeypatch.setenv("SNGB_FUSED", "0")
    monkeypatch.setenv("SNGB_FLOYD_WARP", "0")
    for force, rows in ((None, (0, 0)), ("7", (0, 0)), (None, (n // 3, n // 2 + 5))):
        if force:
            monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", force)
        else:
            monkeypatch.delenv("SNGB_TEST_FORCE_IRREGULAR", raising=False)
        monkeypatch.setenv("SNGB_FLOYD_PIPE", "1")
        kp, gp = sng.sampled_edges_device(x, w.eps, rate, w.seed, rows[0], rows[1])
        monkeypatch.setenv("SNGB_FLOYD_PIPE", "0")
        monkeypatch.setenv("SNGB_FLOYD_LEAN", "0")
        kb, gb = sng.sampled_edges_device(x, w.eps, rate, w.seed, rows[0], rows[1])
        monkeypatch.delenv("SNGB_FLOYD_LEAN", raising=False)
        torch.cuda.synchronize()
        assert gp.draws > 1024
        assert torch.equal(kp, kb), (cfg, force, rows)
        assert gp.collisions == gb.collisions > 0
        assert gp.irregular_vertices == gb.irregular_vertices
        if force:
            assert gp.irregular_vertices >= n // 7


def test_floyd_pipe_matches_oracle(monkeypatch, oracle):
    """k_floyd_pipe end to end against the oracle (labels, roles, counters) at
    1200 draws per vertex, with and without forced Lemire replays."""
    n = 40_000
    pts = synthetic.generate(3, n=n)
    w = synthetic.CONFIGS[3]
    rate = 0.03
    monkeypatch.setenv("SNGB_FLOYD_PIPE", "1")
    monkeypatch.setenv("SNGB_FLOYD_WARP", "0")
    monkeypatch.setenv("SNGB_FUSED", "0")
    labels, roles, oinfo, _ = oracle.sng_dbscan(pts, w.eps, w.min_pts, rate, w.seed)
    for force in (None, "5"):
        if force:
            monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", force)
        info = sng.ClusterRunInfo()
        c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=w.eps, min_pts=w.min_pts, rate=rate,
                                                           seed=w.seed, device=0), info)
        assert np.array_equal(c.assignment, labels) and np.array_equal(c.role, roles)
        assert info.edges == oinfo["edges"] and info.distance_evals == oinfo["distance_evals"]
        assert info.gpu["draws"] == 1200 and info.gpu["collisions"] > 0


@pytest.mark.parametrize("cfg,n,head", [(3, 200_000, "1"), (4, 400_000, "1"), (5, 300_000, "1"),
                                        (5, 300_000, "0"), (2, 120_000, "1")])
def test_floyd_warp_equals_bloom(monkeypatch, cfg, n, head):
    """k_floyd_warp (warp per vertex, sngb_floyd_warp.cuh, SNGB_FLOYD_WARP=1) against
    k_floyd_bloom (SNGB_FLOYD_BLOOM=1) on reduced BASELINE shapes: the same edge list, the same
    Floyd collisions and replayed vertices; with forced Lemire replays too, and
    draws <= 512 (cfg2 shape at n = 120 k: D = 700; cfg3: D = 1000)."""
    import torch
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg, n=n)).cuda()
    rate = w.draws / n
    monkeypatch.setenv("SNGB_FUSED", "0")
    monkeypatch.setenv("SNGB_HEAD", head)
    monkeypatch.setenv("SNGB_Q8", "0")
    for force in (None, "7"):
        if force:
            monkeypatch.setenv("SNGB_TEST_FORCE_IRREGULAR", force)
        monkeypatch.delenv("SNGB_FLOYD_BLOOM", raising=False)
        monkeypatch.setenv("SNGB_FLOYD_WARP", "1")
        kw, gw = sng.sampled_edges_device(x, w.eps, rate, w.seed)
        monkeypatch.delenv("SNGB_FLOYD_WARP", raising=False)
        monkeypatch.setenv("SNGB_FLOYD_BLOOM", "1")
        kb, gb = sng.sampled_edges_device(x, w.eps, rate, w.seed)
        torch.cuda.synchronize()
        assert torch.equal(kw, kb), (cfg, force)
        assert gw.collisions == gb.collisions
        assert gw.irregular_vertices == gb.irregular_vertices
        if force:
            assert gw.irregular_vertices >= n // 7
