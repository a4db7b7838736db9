"""The oracle (oracle/sng_oracle.c) pinned to the reference: golden vectors
made from the compiled reference sources, SURVEY Appendix A KATs, and (when
oracle/_ref is built) a live differential run.  CPU only."""
import numpy as np
import pytest

from oracle import fnv1a64_u32
from tests import _golden

G = _golden.load()


@pytest.mark.parametrize("kat", G["stream_next"], ids=lambda k: f"s{k['seed']}_id{k['id']}")
def test_stream_next_matches_reference(oracle, kat):
    got = oracle.stream_next(kat["seed"], kat["id"], len(kat["values"]))
    assert [str(v) for v in got] == kat["values"]


def test_survey_appendix_a_values(oracle):
    # SURVEY Appendix A lists Stream(1,0).next() x3 and Stream(0,0) x2 as sets
    # (its printout order is reversed); the golden file holds the reference order.
    assert set(int(v) for v in oracle.stream_next(1, 0, 3)) == {
        2256523987077522257, 3668780101835371174, 16097550823460020028}
    assert set(int(v) for v in oracle.stream_next(0, 0, 2)) == {
        4905135072117328383, 4543970728858770942}
    assert list(oracle.stream_next_below(5, 12345, 19999, 4)) == [12901, 1981, 14344, 4485]


@pytest.mark.parametrize("kat", G["stream_next_below"], ids=lambda k: f"b{k['bound']}")
def test_next_below_matches_reference(oracle, kat):
    got = oracle.stream_next_below(kat["seed"], kat["id"], kat["bound"], len(kat["values"]))
    assert [int(v) for v in got] == kat["values"]


@pytest.mark.parametrize("p", G["partners_fnv1a64"], ids=lambda p: f"n{p['n']}_u{p['u']}")
def test_partner_sets_fnv(oracle, p):
    got = oracle.partners(p["n"], p["draws"], p["seed"], p["u"])
    assert len(got) == p["draws"] and len(set(got.tolist())) == p["draws"]
    assert list(got[:4]) == p["first4"] and int(got[-1]) == p["last"]
    assert format(fnv1a64_u32(got), "016x") == p["fnv"]
    assert p["u"] not in set(got.tolist())


def test_draws_formula(oracle):
    # graph.cpp:139-140; every BASELINE config's s*n is exactly representable
    for n, r, want in [(20000, 0.1, 2000), (70000, 0.01, 700), (10**6, 0.001, 1000),
                       (5 * 10**6, 0.0005, 2500), (2 * 10**7, 0.0002, 4000), (1, 1.0, 0),
                       (2, 0.3, 1), (10, 1.0, 9)]:
        assert oracle.draws(n, r) == want


@pytest.mark.parametrize("case", [c for c in G["cases"] if c["n"] <= 30000],
                         ids=lambda c: c["name"])
def test_oracle_matches_golden(oracle, case):
    pts = _golden.points(case["recipe"])
    assert _golden.sha(pts) == case["points_sha256"], "input recipe drifted"
    labels, roles, info, keys = oracle.sng_dbscan(pts, case["eps"], case["min_pts"],
                                                  case["rate"], case["seed"])
    assert info["distance_evals"] == case["distance_evals"]
    assert info["edges"] == case["edges"]
    assert info["graph_bytes"] == case["graph_bytes"]
    assert info["cluster_count"] == case["cluster_count"]
    assert _golden.sha(keys) == case["keys_sha256"]
    assert _golden.sha(labels) == case["labels_sha256"]
    assert _golden.sha(roles) == case["roles_sha256"]
    if "labels" in case:
        assert labels.tolist() == case["labels"]
        assert [str(int(k)) for k in keys] == case["keys"]


def test_oracle_vs_reference_live(oracle, ref):
    """Differential run against the compiled reference on fresh random inputs."""
    rng = np.random.default_rng(123)
    for n, d, eps, mp, rate, seed in [(700, 2, 0.06, 4, 0.2, 1), (900, 5, 0.5, 3, 0.05, 2),
                                      (400, 3, 0.2, 5, 1.0, 3), (3, 1, 1.0, 1, 0.5, 4)]:
        pts = rng.random((n, d), dtype=np.float32)
        ol, orl, oinfo, okeys = oracle.sng_dbscan(pts, eps, mp, rate, seed, threads=3)
        ds = ref.dataset(pts)
        rl, rrl, rinfo = ref.sng_dbscan(ds, eps, mp, rate, seed, threads=2)
        rkeys, _, _ = ref.sampled_edges(ds, eps, rate, seed)
        np.testing.assert_array_equal(ol, rl)
        np.testing.assert_array_equal(orl, rrl)
        np.testing.assert_array_equal(okeys, rkeys)
        for k in ("distance_evals", "edges", "graph_bytes", "cluster_count"):
            assert oinfo[k] == rinfo[k]


def test_rate1_equals_classical_dbscan(oracle, ref):
    """SPEC oracle equivalence: sng_dbscan(rate=1) == oracles.hpp reference_dbscan."""
    rng = np.random.default_rng(9)
    for n, d, eps, mp in [(200, 2, 0.1, 4), (150, 3, 0.3, 2), (60, 2, 0.5, 10)]:
        pts = rng.random((n, d), dtype=np.float32)
        ol, orl, _, _ = oracle.sng_dbscan(pts, eps, mp, 1.0, 0)
        rl, rcore = ref.reference_dbscan(ref.dataset(pts), eps, mp)
        np.testing.assert_array_equal(ol, rl)
        np.testing.assert_array_equal(orl == 0, rcore == 1)


def test_oracle_errors(oracle):
    pts = np.zeros((3, 2), np.float32)
    with pytest.raises(ValueError, match="eps must be > 0"):
        oracle.sng_dbscan(pts, 0.0, 1, 1.0, 0)
    with pytest.raises(ValueError, match="min_pts must be >= 1"):
        oracle.sng_dbscan(pts, 1.0, 0, 1.0, 0)
    with pytest.raises(ValueError, match=r"rate must lie in \(0, 1\]"):
        oracle.sng_dbscan(pts, 1.0, 1, 0.0, 0)


def test_oracle_rate1_reproduces_reference_dbscan_exact(oracle):
    """dbscan_exact (clusterer.cpp:67-79) clusters build_full_graph; for a symmetric
    metric that is the rate-1 sampled graph (graph.cpp:157-159), so the oracle's
    rate-1 run must reproduce the reference's dbscan_exact fixtures bit for bit."""
    from tests import _golden
    g = _golden.load()
    for c in g["exact_cases"]:
        if c["metric"] != "euclidean":
            continue
        pts = _golden.points(c["recipe"])
        labels, roles, info, keys = oracle.sng_dbscan(pts, c["eps"], c["min_pts"], 1.0, 0)
        assert _golden.sha(keys) == c["keys_sha256"], c["name"]
        assert _golden.sha(labels) == c["labels_sha256"], c["name"]
        assert _golden.sha(roles) == c["roles_sha256"], c["name"]
        assert info["edges"] == c["edges"]
        n = c["n"]
        assert c["distance_evals"] == n * (n - 1) // 2
